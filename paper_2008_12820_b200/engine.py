"""Python-side handle on the device engine: a thin mirror of the reference's
SerialEngine member set (proj/include/vreg/engine.hpp:24-183) over the C ABI,
with torch CUDA tensors as the field storage.

Used by the tests, __graft_entry__ and bench.py. The production host layer
is the C++ CudaEngine (include/vreg_b200/cuda_engine.hpp); this module calls
the same C entry points. Fields: scalar = float32 tensor (n1_local, n2, n3),
vector = (3, n1_local, n2, n3); characteristics = (disp (3, ...), flags).
"""
from __future__ import annotations

import ctypes as C
import weakref

import torch

from ._lib import VregGrid, check, lib


def _p(t):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError("fields must be contiguous float32 CUDA tensors")
    return C.c_void_p(t.data_ptr())


def _pd(t):
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("query points must be contiguous float64 CUDA tensors")
    return C.c_void_p(t.data_ptr())


class Context:
    """One per GPU / rank (EngineState analogue, engine.hpp:14-19)."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, uid: bytes | None = None):
        self.device = device
        torch.cuda.set_device(device)
        h = C.c_void_p()
        if nranks == 1:
            check(lib().vreg_ctx_create(device, C.byref(h)))
        else:
            buf = C.create_string_buffer(bytes(uid), 128)
            check(lib().vreg_ctx_create_dist(device, rank, nranks, buf, C.byref(h)))
        self.h = h
        self._dependents = weakref.WeakSet()  # solvers on this context: closed first
        self.rank, self.nranks = rank, nranks
        # order our kernels on torch's stream so tensor ops and ours interleave safely
        check(lib().vreg_ctx_set_stream(self.h, C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().vreg_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "h", None):
            for d in list(getattr(self, "_dependents", ())):
                d.close()
            lib().vreg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- geometry -------------------------------------------------------
    @staticmethod
    def grid(n1, n2=None, n3=None, nt=4) -> VregGrid:
        n2 = n1 if n2 is None else n2
        n3 = n1 if n3 is None else n3
        return VregGrid(n1, n2, n3, nt)

    def slab(self, g):
        n1l, off = C.c_int(), C.c_int()
        check(lib().vreg_slab(self.h, C.byref(g), C.byref(n1l), C.byref(off)))
        return n1l.value, off.value

    def field(self, g, ncomp=1, zero=True):
        """This rank's slab of a device field (zero=False: uninitialised, for
        outputs the library overwrites)."""
        n1l, _ = self.slab(g)
        shape = (n1l, g.n2, g.n3) if ncomp == 1 else (ncomp, n1l, g.n2, g.n3)
        alloc = torch.zeros if zero else torch.empty
        return alloc(shape, dtype=torch.float32, device=f"cuda:{self.device}")

    def to_global(self, g, f):
        """Global field on the host (numpy float32), slabs gathered over ranks."""
        import numpy as np
        ncomp = 3 if f.dim() == 4 else 1
        shape = (g.n1, g.n2, g.n3) if ncomp == 1 else (3, g.n1, g.n2, g.n3)
        out = np.zeros(shape, dtype=np.float32)
        check(lib().vreg_to_global(self.h, C.byref(g), ncomp, _p(f),
                                   out.ctypes.data_as(C.c_void_p)))
        return out

    def from_global(self, g, a):
        """This rank's slab of a global host array, as a device field."""
        import numpy as np
        a = np.ascontiguousarray(a, dtype=np.float32)
        ncomp = 3 if a.ndim == 4 else 1
        out = self.field(g, ncomp)
        check(lib().vreg_from_global(self.h, C.byref(g), ncomp, a.ctypes.data_as(C.c_void_p),
                                     _p(out)))
        return out

    def synchronize(self):
        check(lib().vreg_ctx_synchronize(self.h))

    def set_deterministic(self, on=True):
        """Exact fixed-point transpose sweeps (bitwise reproducible and
        independent of the GPU count); default fp32 L2 reductions."""
        check(lib().vreg_ctx_set_deterministic(self.h, int(on)))

    def set_reg_order(self, order=1):
        """Regularisation order of regop / inv_regop / seminorm / h0 / the GN
        matvec: 1 = H1 (|k|^2, the reference), 2 = H2 (|k|^4)."""
        check(lib().vreg_ctx_set_reg_order(self.h, int(order)))

    def enable_timers(self, on=True):
        check(lib().vreg_ctx_enable_timers(self.h, int(on)))

    def timers(self):
        out = (C.c_double * 8)()
        check(lib().vreg_ctx_timers(self.h, out))
        names = ["fft", "fd", "sl", "ghost_comm", "interp_comm", "scatter_comm", "scatter_buffer",
                 "transpose_comm"]
        return dict(zip(names, list(out)))

    def kernel_stats(self, reset=False):
        """{name: {count, seconds}} of named kernels timed while timers were on."""
        out, i = {}, 0
        name = C.create_string_buffer(64)
        cnt, sec = C.c_uint64(), C.c_double()
        while lib().vreg_ctx_kernel_stats(self.h, i, name, C.byref(cnt), C.byref(sec)) == 0:
            out[name.value.decode()] = {"count": cnt.value, "seconds": sec.value}
            i += 1
        if reset:
            check(lib().vreg_ctx_reset_kernel_stats(self.h))
        return out

    def comm(self):
        out = (C.c_uint64 * 9)()
        check(lib().vreg_ctx_comm(self.h, out))
        names = ["ghost_fd_bytes", "ghost_interp_bytes", "scatter_points_bytes",
                 "interp_values_bytes", "fft_transpose_bytes", "spectral_gather_bytes",
                 "reduce_bytes", "p2p_messages", "alltoall_collectives"]
        return dict(zip(names, list(out)))

    def tile_stats(self):
        """(tiles built, tiles over the smem budget -> per-point fallback)."""
        a, b = C.c_uint64(), C.c_uint64()
        check(lib().vreg_ctx_tile_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def launches(self) -> int:
        out = C.c_uint64()
        check(lib().vreg_ctx_launches(self.h, C.byref(out)))
        return out.value

    # ---- pointwise / reductions (field.hpp:67-188) ----------------------
    def inner(self, g, a, b):
        out = C.c_double()
        ncomp = 3 if a.dim() == 4 else 1
        check(lib().vreg_inner(self.h, C.byref(g), ncomp, _p(a), _p(b), C.byref(out)))
        return out.value

    def norm2(self, g, a):
        return self.inner(g, a, a) ** 0.5

    def max_abs(self, g, a):
        out = C.c_double()
        ncomp = 3 if a.dim() == 4 else 1
        check(lib().vreg_max_abs(self.h, C.byref(g), ncomp, _p(a), C.byref(out)))
        return out.value

    def axpy(self, g, a, x, y):
        check(lib().vreg_axpy(self.h, C.byref(g), 3 if x.dim() == 4 else 1, a, _p(x), _p(y)))

    def scale(self, g, x, a):
        check(lib().vreg_scale(self.h, C.byref(g), 3 if x.dim() == 4 else 1, _p(x), a))

    def aypx(self, g, a, x, y):
        check(lib().vreg_aypx(self.h, C.byref(g), 3 if x.dim() == 4 else 1, a, _p(x), _p(y)))

    def fill(self, g, x, v):
        check(lib().vreg_fill(self.h, C.byref(g), 3 if x.dim() == 4 else 1, _p(x), v))

    def sub(self, g, a, b, out):
        check(lib().vreg_sub(self.h, C.byref(g), 3 if a.dim() == 4 else 1, _p(a), _p(b), _p(out)))

    def hadamard(self, g, a, b, out):
        check(lib().vreg_hadamard(self.h, C.byref(g), _p(a), _p(b), _p(out)))

    def pointwise_dot(self, g, v, w, out):
        check(lib().vreg_pointwise_dot(self.h, C.byref(g), _p(v), _p(w), _p(out)))

    def axpy_scaled_vector(self, g, a, s, w, out):
        check(lib().vreg_axpy_scaled_vector(self.h, C.byref(g), a, _p(s), _p(w), _p(out)))

    # ---- kernels (engine.hpp:77-169) -----------------------------------
    def fd_grad(self, g, f):
        out = self.field(g, 3)
        check(lib().vreg_fd_grad(self.h, C.byref(g), _p(f), _p(out)))
        return out

    def fd_div(self, g, v):
        out = self.field(g)
        check(lib().vreg_fd_div(self.h, C.byref(g), _p(v), _p(out)))
        return out

    def characteristics(self, g, v, degree=3):
        disp = self.field(g, 3)
        flags = C.c_int()
        check(lib().vreg_characteristics(self.h, C.byref(g), _p(v), degree, _p(disp), C.byref(flags)))
        return disp, flags.value

    def interp(self, g, f, chars, degree=3):
        disp, flags = chars
        out = self.field(g)
        check(lib().vreg_interp(self.h, C.byref(g), _p(f), _p(disp), flags, degree, _p(out)))
        return out

    def scatter(self, g, z, chars, degree=3):
        disp, flags = chars
        out = self.field(g)
        check(lib().vreg_scatter(self.h, C.byref(g), _p(z), _p(disp), flags, degree, _p(out)))
        return out

    def interp_points(self, g, f, xyz, degree=3):
        xyz = xyz.contiguous()
        m = xyz.numel() // 3
        out = torch.zeros(m, dtype=torch.float32, device=f.device)
        check(lib().vreg_interp_points(self.h, C.byref(g), _p(f), _pd(xyz), m, degree, _p(out)))
        return out

    def scatter_points(self, g, xyz, z, degree=3, acc=None):
        xyz = xyz.contiguous()
        m = xyz.numel() // 3
        acc = self.field(g) if acc is None else acc
        check(lib().vreg_scatter_points(self.h, C.byref(g), _pd(xyz), _p(z), m, degree, _p(acc)))
        return acc

    def solve_state(self, g, chars, m0, degree=3):
        disp, flags = chars
        n1l, _ = self.slab(g)
        m = torch.zeros((g.nt + 1, n1l, g.n2, g.n3), dtype=torch.float32, device=m0.device)
        m[0].copy_(m0)
        check(lib().vreg_solve_state(self.h, C.byref(g), _p(disp), flags, degree, _p(m)))
        return m

    def inc_state(self, g, chars, grads, vt, degree=3):
        disp, flags = chars
        n1l, _ = self.slab(g)
        mt = torch.zeros((g.nt + 1, n1l, g.n2, g.n3), dtype=torch.float32, device=vt.device)
        check(lib().vreg_inc_state(self.h, C.byref(g), _p(disp), flags, degree, _p(grads), _p(vt),
                                   _p(mt), None))
        return mt

    def transpose_assemble(self, g, chars, grads, fin, degree=3):
        disp, flags = chars
        out = self.field(g, 3)
        check(lib().vreg_transpose_assemble(self.h, C.byref(g), _p(disp), flags, degree, _p(grads),
                                            _p(fin), _p(out)))
        return out

    def gn_matvec(self, g, chars, grads, beta, vt, degree=3, out=None):
        disp, flags = chars
        out = self.field(g, 3) if out is None else out
        check(lib().vreg_gn_matvec(self.h, C.byref(g), _p(disp), flags, degree, _p(grads), beta,
                                   _p(vt), _p(out)))
        return out

    def adjoint_source_factor(self, g, v, bwd, degree=3):
        disp, flags = bwd
        q = self.field(g)
        check(lib().vreg_adjoint_source_factor(self.h, C.byref(g), _p(v), _p(disp), flags, degree,
                                               _p(q)))
        return q

    def adjoint_sweep(self, g, bwd, q, fin, degree=3):
        disp, flags = bwd
        n1l, _ = self.slab(g)
        lam = torch.zeros((g.nt + 1, n1l, g.n2, g.n3), dtype=torch.float32, device=fin.device)
        lam[g.nt].copy_(fin)
        check(lib().vreg_adjoint_sweep(self.h, C.byref(g), _p(disp), flags, degree, _p(q), _p(lam)))
        return lam

    def integrate_lambda_grad_m(self, g, lam, grads):
        out = self.field(g, 3)
        check(lib().vreg_integrate_lambda_grad_m(self.h, C.byref(g), _p(lam), _p(grads), _p(out)))
        return out

    # ---- spectral (spectral.cpp) ---------------------------------------
    def regop(self, g, v, beta, unit_zero_mode=True):
        out = self.field(g, 3)
        check(lib().vreg_regop(self.h, C.byref(g), _p(v), beta, int(unit_zero_mode), _p(out)))
        return out

    def inv_regop(self, g, v, beta):
        out = self.field(g, 3)
        check(lib().vreg_inv_regop(self.h, C.byref(g), _p(v), beta, _p(out)))
        return out

    def seminorm(self, g, v):
        out = C.c_double()
        check(lib().vreg_seminorm(self.h, C.byref(g), _p(v), C.byref(out)))
        return out.value

    def leray(self, g, v):
        out = self.field(g, 3)
        check(lib().vreg_leray(self.h, C.byref(g), _p(v), _p(out)))
        return out

    def restrict(self, g, f):
        ncomp = 3 if f.dim() == 4 else 1
        gc = VregGrid(g.n1 // 2, g.n2 // 2, g.n3 // 2, g.nt)
        out = self.field(gc, ncomp)
        check(lib().vreg_restrict(self.h, C.byref(g), ncomp, _p(f), _p(out)))
        return out

    def prolong(self, g, fc):
        ncomp = 3 if fc.dim() == 4 else 1
        out = self.field(g, ncomp)
        check(lib().vreg_prolong(self.h, C.byref(g), ncomp, _p(fc), _p(out)))
        return out

    def high_pass(self, g, f):
        ncomp = 3 if f.dim() == 4 else 1
        out = self.field(g, ncomp)
        check(lib().vreg_high_pass(self.h, C.byref(g), ncomp, _p(f), _p(out)))
        return out

    def h0_matvec(self, g, s, grad_mref, beta_pc):
        out = self.field(g, 3)
        check(lib().vreg_h0_matvec(self.h, C.byref(g), _p(s), _p(grad_mref), beta_pc, _p(out)))
        return out

    def fft_forward(self, g, f):
        out = torch.zeros((g.n1, g.n2, g.n3 // 2 + 1, 2), dtype=torch.float32, device=f.device)
        check(lib().vreg_fft_forward(self.h, C.byref(g), _p(f), _p(out)))
        return torch.view_as_complex(out)

    # ---- synthetic inputs (syn.cpp:9-44) -------------------------------
    def syn_template(self, g):
        out = self.field(g)
        check(lib().vreg_syn_template(self.h, C.byref(g), _p(out)))
        return out

    def syn_velocity(self, g):
        out = self.field(g, 3)
        check(lib().vreg_syn_velocity(self.h, C.byref(g), _p(out)))
        return out
