"""VolumeFile "VRG1" I/O through the native library
(include/vreg_b200/report.hpp: save_volume / load_volume): header magic
"VRG1", u32 LE n1 n2 n3, u8 scalar kind (0 f32, 1 f64), u8 components (1 or
3), components concatenated row-major. Corrupted magic or a payload length
that disagrees with the header raise VregError(kind="io")."""
import ctypes as C

import numpy as np

from ._lib import check, lib

def _bind():
    return lib()  # signatures in _lib._SIGS


def save_volume(path, array):
    """array: (n1, n2, n3) or (3, n1, n2, n3), float32 or float64."""
    a = np.ascontiguousarray(array)
    if a.dtype not in (np.float32, np.float64):
        raise TypeError("volume data must be float32 or float64")
    if a.ndim == 3:
        ncomp, shape = 1, a.shape
    elif a.ndim == 4 and a.shape[0] == 3:
        ncomp, shape = 3, a.shape[1:]
    else:
        raise ValueError("volume shape must be (n1, n2, n3) or (3, n1, n2, n3)")
    kind = 0 if a.dtype == np.float32 else 1
    check(_bind().vreg_volume_save(str(path).encode(), shape[0], shape[1], shape[2], kind, ncomp,
                                   a.ctypes.data_as(C.c_void_p)))


def load_volume(path):
    L = _bind()
    h = (C.c_int * 5)()
    check(L.vreg_volume_header(str(path).encode(), h))
    n1, n2, n3, kind, ncomp = list(h)
    dt = np.float32 if kind == 0 else np.float64
    out = np.empty((ncomp, n1, n2, n3) if ncomp == 3 else (n1, n2, n3), dtype=dt)
    check(L.vreg_volume_load(str(path).encode(), out.ctypes.data_as(C.c_void_p), out.nbytes))
    return out
