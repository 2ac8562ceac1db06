"""ctypes wrapper over oracle/_ref/libvreg_ref.so (the UNMODIFIED reference).

TEST INFRASTRUCTURE ONLY. Importable solely from tests/, tests/golden/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.
The library is the reference's own C++ (fp64) compiled from
/root/reference/proj/src by oracle/Makefile; see oracle/ref_capi.cpp for the
entry points and the reference lines each one calls.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, fields

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libvreg_ref.so")

COUNTER_NAMES = [
    "fft_forward", "fft_inverse", "fft_forward_coarse", "fft_inverse_coarse",
    "fd_gradient", "fd_divergence", "ip_eval", "ip_scatter",
    "characteristics", "characteristics_identity", "sl_state", "sl_adjoint",
    "sl_inc_state", "sl_inc_adjoint", "pc_inva_apply", "pc_h0_apply",
    "pc_h0_inner_iters", "pc_h0_inner_solves", "pc_refresh",
    "h0_inner_work_fine", "h0_inner_work_coarse",
]

REPORT_NAMES = [
    "initial_mismatch", "final_mismatch", "mism_rel", "final_g_rel",
    "total_gn", "total_pcg", "flagged", "t_pc", "t_obj", "t_grad", "t_hess",
    "t_total", "t_fft", "t_fd", "t_sl", "cost_model_matches",
]

PRECOND = {"inva": 0, "invh0": 1, "2linvh0": 2}


class VrefConfig(C.Structure):
    """Mirror of RegistrationConfig (proj/include/vreg/optim.hpp:16-37)."""
    _fields_ = [
        ("beta_target", C.c_double), ("beta_start", C.c_double),
        ("continuation", C.c_int), ("gamma_div", C.c_double),
        ("project_divfree", C.c_int), ("eps_newton", C.c_double),
        ("eps_h0", C.c_double), ("max_gn", C.c_int), ("max_pcg", C.c_int),
        ("precond", C.c_int), ("interp_degree", C.c_int),
        ("cache_state_gradient", C.c_int), ("fixed_gn", C.c_int),
        ("fixed_pcg", C.c_int), ("hessian_adjoint", C.c_int), ("nt", C.c_int),
        ("armijo_c", C.c_double), ("armijo_shrink", C.c_double),
        ("armijo_max_trials", C.c_int), ("h0_inner_cap", C.c_int),
    ]


@dataclass
class Config:
    """RegistrationConfig defaults (optim.hpp:17-37)."""
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

    def to_c(self) -> VrefConfig:
        c = VrefConfig()
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "precond":
                v = PRECOND[v]
            setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"reference status {status}: {msg}")
        self.status = status


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        L.vref_last_error.restype = C.c_char_p
        L.vref_session_create.restype = C.c_void_p
        L.vref_session_create.argtypes = [C.c_int] * 3 + [
            C.POINTER(VrefConfig), C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        for name in ("vref_session_destroy", "vref_session_objective",
                     "vref_session_gradient", "vref_session_state",
                     "vref_session_chars", "vref_session_matvec",
                     "vref_session_inc_state", "vref_session_transpose_assemble",
                     "vref_session_counters", "vref_session_timers"):
            getattr(L, name).argtypes = None
        L.vref_session_precond.argtypes = [
            C.c_void_p, C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _chk(st):
    if st != 0:
        raise RefError(st, lib().vref_last_error().decode())


def _dims(shape):
    return [C.c_int(int(s)) for s in shape]


def syn(n, nt=4, degree=3):
    n1, n2, n3 = (n, n, n) if isinstance(n, int) else n
    N = n1 * n2 * n3
    m0 = np.zeros(N); v = np.zeros(3 * N); m1 = np.zeros(N)
    _chk(lib().vref_syn(n1, n2, n3, nt, degree, _p(m0), _p(v), _p(m1)))
    sh = (n1, n2, n3)
    return m0.reshape(sh), v.reshape((3,) + sh), m1.reshape(sh)


def characteristics(v3, nt, degree=3):
    sh = v3.shape[1:]
    xyz = np.zeros(3 * int(np.prod(sh)))
    ident = C.c_int(0)
    v = np.ascontiguousarray(v3, dtype=np.float64)
    _chk(lib().vref_characteristics(*_dims(sh), nt, _p(v), degree, _p(xyz), C.byref(ident)))
    return xyz.reshape(sh + (3,)), bool(ident.value)


def interp(f, xyz, degree=3):
    f = np.ascontiguousarray(f, dtype=np.float64)
    q = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(q.shape[0])
    _chk(lib().vref_interp(*_dims(f.shape), _p(f), _p(q), C.c_int64(q.shape[0]), degree, _p(out)))
    return out


def scatter(shape, xyz, z, degree=3, acc=None):
    q = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    z = np.ascontiguousarray(z, dtype=np.float64).ravel()
    a = np.zeros(shape) if acc is None else np.array(acc, dtype=np.float64)
    _chk(lib().vref_scatter(*_dims(shape), _p(q), _p(z), C.c_int64(q.shape[0]), degree, _p(a)))
    return a


def fd_grad(f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros((3,) + f.shape)
    _chk(lib().vref_fd_grad(*_dims(f.shape), _p(f), _p(out)))
    return out


def fd_div(v3):
    v = np.ascontiguousarray(v3, dtype=np.float64)
    out = np.zeros(v.shape[1:])
    _chk(lib().vref_fd_div(*_dims(v.shape[1:]), _p(v), _p(out)))
    return out


def fd8_weights():
    w = np.zeros(9)
    _chk(lib().vref_fd8_weights(_p(w)))
    return w


def regop(v3, beta, unit_zero=True):
    v = np.ascontiguousarray(v3, dtype=np.float64)
    out = np.zeros_like(v)
    _chk(lib().vref_regop(*_dims(v.shape[1:]), _p(v), C.c_double(beta), int(unit_zero), _p(out)))
    return out


def inv_regop(v3, beta):
    v = np.ascontiguousarray(v3, dtype=np.float64)
    out = np.zeros_like(v)
    _chk(lib().vref_inv_regop(*_dims(v.shape[1:]), _p(v), C.c_double(beta), _p(out)))
    return out


def seminorm(v3):
    v = np.ascontiguousarray(v3, dtype=np.float64)
    out = C.c_double(0)
    _chk(lib().vref_seminorm(*_dims(v.shape[1:]), _p(v), C.byref(out)))
    return out.value


def leray(v3):
    v = np.ascontiguousarray(v3, dtype=np.float64)
    out = np.zeros_like(v)
    _chk(lib().vref_leray(*_dims(v.shape[1:]), _p(v), _p(out)))
    return out


def restrict(f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros(tuple(s // 2 for s in f.shape))
    _chk(lib().vref_restrict(*_dims(f.shape), _p(f), _p(out)))
    return out


def prolong(fc, fine_shape):
    fc = np.ascontiguousarray(fc, dtype=np.float64)
    out = np.zeros(fine_shape)
    _chk(lib().vref_prolong(*_dims(fine_shape), _p(fc), _p(out)))
    return out


def high_pass(f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros_like(f)
    _chk(lib().vref_high_pass(*_dims(f.shape), _p(f), _p(out)))
    return out


def fft_forward(f):
    f = np.ascontiguousarray(f, dtype=np.float64)
    n1, n2, n3 = f.shape
    out = np.zeros((n1, n2, n3 // 2 + 1, 2))
    _chk(lib().vref_fft_forward(*_dims(f.shape), _p(f), _p(out)))
    return out[..., 0] + 1j * out[..., 1]


def inner(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = C.c_double(0)
    _chk(lib().vref_inner(*_dims(a.shape), _p(a), _p(b), C.byref(out)))
    return out.value


class Session:
    """A Gauss-Newton linearisation point: Flow + StateCache after objective
    and gradient, as gauss_newton_level holds them entering PCG
    (proj/include/vreg/optim.hpp:155-168)."""

    def __init__(self, m0, m1, v3, beta, cfg: Config | None = None):
        self.cfg = cfg or Config()
        self.shape = m0.shape
        self.N = int(np.prod(self.shape))
        self._m0 = np.ascontiguousarray(m0, dtype=np.float64)
        self._m1 = np.ascontiguousarray(m1, dtype=np.float64)
        self._v = np.ascontiguousarray(v3, dtype=np.float64)
        self._c = self.cfg.to_c()
        h = lib().vref_session_create(*_dims(self.shape), C.byref(self._c), C.c_double(beta),
                                      _p(self._m0), _p(self._m1), _p(self._v))
        if not h:
            raise RefError(-1, lib().vref_last_error().decode())
        self.h = C.c_void_p(h)
        self.beta = beta

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.vref_session_destroy(self.h)
            self.h = None

    def objective(self):
        J = np.zeros(4)
        lib().vref_session_objective(self.h, _p(J))
        return dict(total=J[0], mismatch=J[1], regularization=J[2], div_penalty=J[3])

    def gradient(self):
        g = np.zeros((3,) + self.shape)
        lib().vref_session_gradient(self.h, _p(g))
        return g

    def state(self):
        m = np.zeros((self.cfg.nt + 1,) + self.shape)
        lib().vref_session_state(self.h, _p(m))
        return m

    def chars(self):
        f = np.zeros(self.shape + (3,)); b = np.zeros(self.shape + (3,))
        _chk(lib().vref_session_chars(self.h, _p(f), _p(b)))
        return f, b

    def matvec(self, vt3):
        vt = np.ascontiguousarray(vt3, dtype=np.float64)
        out = np.zeros_like(vt)
        _chk(lib().vref_session_matvec(self.h, _p(vt), _p(out)))
        return out

    def inc_state(self, vt3):
        vt = np.ascontiguousarray(vt3, dtype=np.float64)
        out = np.zeros((self.cfg.nt + 1,) + self.shape)
        _chk(lib().vref_session_inc_state(self.h, _p(vt), _p(out)))
        return out

    def transpose_assemble(self, fin):
        fin = np.ascontiguousarray(fin, dtype=np.float64)
        out = np.zeros((3,) + self.shape)
        _chk(lib().vref_session_transpose_assemble(self.h, _p(fin), _p(out)))
        return out

    def precond(self, kind, r3, eps_k):
        r = np.ascontiguousarray(r3, dtype=np.float64)
        out = np.zeros_like(r)
        st = np.zeros(4, dtype=np.uint64)
        _chk(lib().vref_session_precond(self.h, PRECOND[kind], _p(r), C.c_double(eps_k),
                                        _p(out), _p(st)))
        return out, dict(inva=int(st[0]), h0=int(st[1]), inner=int(st[2]), capped=bool(st[3]))

    def counters(self):
        c = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
        lib().vref_session_counters(self.h, _p(c))
        return dict(zip(COUNTER_NAMES, (int(x) for x in c)))

    def timers(self):
        t = np.zeros(3)
        lib().vref_session_timers(self.h, _p(t))
        return dict(fft=t[0], fd=t[1], sl=t[2])


def register(m0, m1, cfg: Config):
    shape = m0.shape
    c = cfg.to_c()
    v = np.zeros((3,) + shape)
    rep = np.zeros(len(REPORT_NAMES))
    cnt = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
    m0c = np.ascontiguousarray(m0, dtype=np.float64)
    m1c = np.ascontiguousarray(m1, dtype=np.float64)
    _chk(lib().vref_register(*_dims(shape), C.byref(c), _p(m0c), _p(m1c), _p(v), _p(rep), _p(cnt)))
    return v, dict(zip(REPORT_NAMES, rep.tolist())), dict(zip(COUNTER_NAMES, (int(x) for x in cnt)))


LEVEL_KEYS = ["beta", "inva", "switched", "gn_iters", "pcg_total", "final_mismatch",
              "final_g_rel", "converged"]
ITER_KEYS = ["level", "objective", "mismatch", "g_rel", "eps_k", "alpha", "pcg_iters",
             "h0_inner_iters"]


def register_levels(m0, m1, cfg: Config):
    """register_images with its per-level and per-GN-iteration records
    (report.hpp:12-78): returns v, [level dicts], [GN-iteration dicts]."""
    shape = m0.shape
    c = cfg.to_c()
    v = np.zeros((3,) + shape)
    lev = np.zeros((64, 8))
    its = np.zeros((1024, 8))
    nl, ni = C.c_int(0), C.c_int(0)
    m0c = np.ascontiguousarray(m0, dtype=np.float64)
    m1c = np.ascontiguousarray(m1, dtype=np.float64)
    _chk(lib().vref_register_levels(*_dims(shape), C.byref(c), _p(m0c), _p(m1c), _p(v),
                                    _p(lev), 64, C.byref(nl), _p(its), 1024, C.byref(ni)))
    levels = [dict(zip(LEVEL_KEYS, r.tolist())) for r in lev[:nl.value]]
    iters = [dict(zip(ITER_KEYS, r.tolist())) for r in its[:min(ni.value, 1024)]]
    return v, levels, iters


def register_residuals(m0, m1, cfg: Config):
    """PCG relative-residual histories of register_images: rows (level,
    gn iteration, pcg iteration, relres) as render_residuals_csv."""
    shape = m0.shape
    c = cfg.to_c()
    rows = np.zeros((8192, 4))
    n = C.c_int(0)
    m0c = np.ascontiguousarray(m0, dtype=np.float64)
    m1c = np.ascontiguousarray(m1, dtype=np.float64)
    _chk(lib().vref_register_residuals(*_dims(shape), C.byref(c), _p(m0c), _p(m1c), _p(rows),
                                       8192, C.byref(n)))
    return rows[:min(n.value, 8192)]
