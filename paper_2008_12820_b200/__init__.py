"""B200-native (sm_100a) Gauss-Newton Hessian-matvec path of the CLAIRE-style
LDDMM solver of arXiv 2008.12820 (reference library "vreg").

The CUDA kernels and the C++ host layer live in libvreg_b200.so (built
in-tree by paper_2008_12820_b200.build); this package binds its C ABI.
Importing `Context` requires the built library: there is no CPU fallback.
"""
from ._lib import LIB_PATH, VregError, VregGrid, exported_symbols, lib  # noqa: F401


def __getattr__(name):
    if name == "Context":
        from .engine import Context
        return Context
    raise AttributeError(name)
