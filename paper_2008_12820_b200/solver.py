"""Python handle on the solver-level C ABI (include/vreg_b200.h): the
Gauss-Newton-Krylov registration and its hot path (GN Hessian matvec,
preconditioners) on the device, mirroring the reference's
register_images / gauss_newton_level / hessian_matvec_with
(proj/include/vreg/optim.hpp).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields

import torch

from . import _lib
from ._lib import VregGrid, check, lib
from .engine import Context, _p

COUNTER_NAMES = [
    "fft_forward", "fft_inverse", "fft_forward_coarse", "fft_inverse_coarse",
    "fd_gradient", "fd_divergence", "ip_eval", "ip_scatter",
    "characteristics", "characteristics_identity", "sl_state", "sl_adjoint",
    "sl_inc_state", "sl_inc_adjoint", "pc_inva_apply", "pc_h0_apply",
    "pc_h0_inner_iters", "pc_h0_inner_solves", "pc_refresh",
    "h0_inner_work_fine", "h0_inner_work_coarse",
]
REPORT_NAMES = [
    "initial_mismatch", "final_mismatch", "mism_rel", "final_g_rel", "total_gn",
    "total_pcg", "flagged", "t_pc", "t_obj", "t_grad", "t_hess", "t_total", "t_fft",
    "t_fd", "t_sl", "levels",
]
PRECOND = {"inva": 0, "invh0": 1, "2linvh0": 2}


class VregConfig(C.Structure):
    """vreg_config == RegistrationConfig (optim.hpp:16-37)."""
    _fields_ = [
        ("beta_target", C.c_double), ("beta_start", C.c_double), ("continuation", C.c_int),
        ("gamma_div", C.c_double), ("project_divfree", C.c_int), ("eps_newton", C.c_double),
        ("eps_h0", C.c_double), ("max_gn", C.c_int), ("max_pcg", C.c_int), ("precond", C.c_int),
        ("interp_degree", C.c_int), ("cache_state_gradient", C.c_int), ("fixed_gn", C.c_int),
        ("fixed_pcg", C.c_int), ("hessian_adjoint", C.c_int), ("nt", C.c_int),
        ("armijo_c", C.c_double), ("armijo_shrink", C.c_double), ("armijo_max_trials", C.c_int),
        ("h0_inner_cap", C.c_int), ("pcg_fp64", C.c_int), ("reg_order", C.c_int),
    ]


@dataclass
class Config:
    """RegistrationConfig with the reference defaults (optim.hpp:17-37)."""
    beta_target: float = 5e-4
    beta_start: float = 1.0
    continuation: bool = True
    gamma_div: float = 0.0
    project_divfree: bool = False
    eps_newton: float = 5e-2
    eps_h0: float = 1e-3
    max_gn: int = 50
    max_pcg: int = 500
    precond: str = "2linvh0"
    interp_degree: int = 3
    cache_state_gradient: bool = True
    fixed_gn: int = 0
    fixed_pcg: int = 0
    hessian_adjoint: int = 0
    nt: int = 4
    armijo_c: float = 1e-4
    armijo_shrink: float = 0.5
    armijo_max_trials: int = 10
    h0_inner_cap: int = 100
    pcg_fp64: bool = True
    reg_order: int = 1  # 1 = H1 (reference), 2 = H2 (B200 extension)

    def to_c(self) -> VregConfig:
        c = VregConfig()
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "precond":
                v = PRECOND[v]
            setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c


_SOLVER_SIGS = {
    "vreg_config_default": (None, [C.POINTER(VregConfig)]),
    "vreg_solver_create": (C.c_int, [C.c_void_p, C.POINTER(VregGrid), C.POINTER(VregConfig),
                                     C.POINTER(C.c_void_p)]),
    "vreg_solver_destroy": (C.c_int, [C.c_void_p]),
    "vreg_solver_set_images": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vreg_solver_syn_images": (C.c_int, [C.c_void_p]),
    "vreg_solver_images": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vreg_solver_linearize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double]),
    "vreg_solver_objective": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "vreg_solver_gradient": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vreg_solver_matvec": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vreg_solver_matvec_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vreg_solver_matvec_host_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vreg_solver_wait": (C.c_int, [C.c_void_p]),
    "vreg_solver_report_text": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p, C.c_size_t,
                                          C.POINTER(C.c_size_t)]),
    "vreg_solver_precond": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_void_p,
                                      C.POINTER(C.c_uint64)]),
    "vreg_solver_register": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                       C.POINTER(C.c_uint64)]),
    "vreg_solver_counters": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "vreg_solver_reset_counters": (C.c_int, [C.c_void_p]),
}
_lib._SOLVER_SIGS.update(_SOLVER_SIGS)
if _lib._lib is not None:  # already loaded: bind the late signatures
    for _n, (_r, _a) in _SOLVER_SIGS.items():
        _f = getattr(_lib._lib, _n)
        _f.restype, _f.argtypes = _r, _a


class Solver:
    """One registration problem on one grid (one per rank)."""

    def __init__(self, ctx: Context, n, cfg: Config | None = None):
        n1, n2, n3 = (n, n, n) if isinstance(n, int) else n
        self.ctx = ctx
        self.cfg = cfg or Config()
        self.grid = VregGrid(n1, n2, n3, self.cfg.nt)
        self._c = self.cfg.to_c()
        h = C.c_void_p()
        check(lib().vreg_solver_create(ctx.h, C.byref(self.grid), C.byref(self._c), C.byref(h)))
        self.h = h
        ctx._dependents.add(self)

    def close(self):
        # a solver's device state lives in its context: destroy it while the
        # context is open (Context.close closes its solvers first)
        if getattr(self, "h", None):
            if getattr(self.ctx, "h", None):
                lib().vreg_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def field(self, ncomp=1, zero=True):
        return self.ctx.field(self.grid, ncomp, zero)

    def set_images(self, m0, m1):
        check(lib().vreg_solver_set_images(self.h, _p(m0), _p(m1)))

    def syn_images(self):
        check(lib().vreg_solver_syn_images(self.h))

    def images(self):
        m0, m1 = self.field(), self.field()
        check(lib().vreg_solver_images(self.h, _p(m0), _p(m1)))
        return m0, m1

    def linearize(self, v, beta):
        check(lib().vreg_solver_linearize(self.h, _p(v), beta))

    def objective(self):
        J = (C.c_double * 4)()
        check(lib().vreg_solver_objective(self.h, J))
        return dict(total=J[0], mismatch=J[1], regularization=J[2], div_penalty=J[3])

    def gradient(self):
        g = self.field(3, zero=False)
        check(lib().vreg_solver_gradient(self.h, _p(g)))
        return g

    def matvec(self, vt, out=None):
        out = self.field(3, zero=False) if out is None else out
        check(lib().vreg_solver_matvec(self.h, _p(vt), _p(out)))
        return out

    def matvec_host(self, vt_host, out_host):
        """Same matvec on host (CPU, ideally pinned) float32 tensors."""
        assert vt_host.device.type == "cpu" and vt_host.dtype == torch.float32
        check(lib().vreg_solver_matvec_host(self.h, C.c_void_p(vt_host.data_ptr()),
                                            C.c_void_p(out_host.data_ptr())))
        return out_host

    def matvec_host_async(self, vt_host, out_host):
        """Enqueue the host-buffer matvec (pinned float32 tensors) and return;
        consecutive calls overlap upload, matvec and download. Buffers stay
        owned by the caller until wait()."""
        assert vt_host.device.type == "cpu" and vt_host.is_pinned() and out_host.is_pinned()
        check(lib().vreg_solver_matvec_host_async(self.h, C.c_void_p(vt_host.data_ptr()),
                                                  C.c_void_p(out_host.data_ptr())))
        return out_host

    def wait(self):
        check(lib().vreg_solver_wait(self.h))

    def precond(self, kind, r, eps_k):
        out = self.field(3, zero=False)
        st = (C.c_uint64 * 4)()
        check(lib().vreg_solver_precond(self.h, PRECOND[kind], _p(r), eps_k, _p(out), st))
        return out, dict(inva=st[0], h0=st[1], inner=st[2], capped=bool(st[3]))

    def register(self):
        v = self.field(3)
        rep = (C.c_double * 16)()
        cnt = (C.c_uint64 * 21)()
        check(lib().vreg_solver_register(self.h, _p(v), rep, cnt))
        return v, dict(zip(REPORT_NAMES, list(rep))), dict(zip(COUNTER_NAMES, list(cnt)))

    def report_text(self, which="report"):
        """Rendered report of the last register(): "report" (deterministic,
        no timings), "timings" or "residuals" (CSV of PCG relative residuals)
        -- include/vreg_b200/report.hpp."""
        k = {"report": 0, "timings": 1, "residuals": 2}[which]
        n = C.c_size_t()
        check(lib().vreg_solver_report_text(self.h, k, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().vreg_solver_report_text(self.h, k, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def counters(self):
        cnt = (C.c_uint64 * 21)()
        check(lib().vreg_solver_counters(self.h, cnt))
        return dict(zip(COUNTER_NAMES, list(cnt)))

    def reset_counters(self):
        check(lib().vreg_solver_reset_counters(self.h))
