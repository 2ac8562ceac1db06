"""numpy restatement of the reference's GN-Hessian-matvec path (fp64).

TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured or
shipped. Importable solely from tests/, tests/golden/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg.

Each function restates the reference algorithm it cites (paths under
/root/reference/proj). Pinned against the compiled reference
(oracle/_ref/libvreg_ref.so via oracle/ref.py) in tests/test_oracle.py and
against the committed fixtures in tests/golden/.

Conventions (proj/include/vreg/grid.hpp:10-40): periodic [0, 2pi)^3, node
(i,j,k) at (i h1, j h2, k h3), arrays shaped (n1, n2, n3) with x3 innermost;
vector fields shaped (3, n1, n2, n3); nt time steps, dt = 1/nt.
"""
from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi
SNAP_TOL = 1e-12  # interp.hpp:39


# ---------------------------------------------------------------- grid ----

def spacing(shape):
    """h_a = 2 pi / n_a (grid.hpp:30)."""
    return tuple(TWO_PI / n for n in shape)


def cell_volume(shape):
    h = spacing(shape)
    return h[0] * h[1] * h[2]


def node_coords(shape):
    """Broadcastable node coordinates in radians (grid.hpp:10-11)."""
    h = spacing(shape)
    return (np.arange(shape[0])[:, None, None] * h[0],
            np.arange(shape[1])[None, :, None] * h[1],
            np.arange(shape[2])[None, None, :] * h[2])


def signed_freq(n):
    """signed_freq(k, n) = k <= n/2 ? k : k - n (fft.hpp:49)."""
    k = np.arange(n)
    return np.where(k <= n // 2, k, k - n).astype(np.float64)


# ------------------------------------------------------------- fields ----

def inner(a, b):
    """Plane-folded L2 inner product x h^3 (field.hpp:150-171)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim == 4:  # vector: inner(c1)+inner(c2)+inner(c3) (field.hpp:173-175)
        return sum(inner(a[c], b[c]) for c in range(3))
    planes = (a * b).reshape(a.shape[0], -1).sum(axis=1)
    total = 0.0
    for s in planes:
        total += s
    return total * cell_volume(a.shape)


def norm2(a):
    return math.sqrt(inner(a, a))


# ---------------------------------------------------------------- syn ----

def syn_template(shape):
    """m0 = (sin^2 x1 + sin^2 x2 + sin^2 x3)/3 (syn.cpp:9-23)."""
    x1, x2, x3 = node_coords(shape)
    s1, s2, s3 = np.sin(x1), np.sin(x2), np.sin(x3)
    return (s1 * s1 + s2 * s2 + s3 * s3) / 3.0 + np.zeros(shape)


def syn_velocity(shape):
    """Divergence-free trig velocity (syn.cpp:25-44)."""
    x1, x2, x3 = node_coords(shape)
    v = np.zeros((3,) + tuple(shape))
    v[0] = np.sin(x3) * np.cos(x2) * np.sin(x2)
    v[1] = np.sin(x1) * np.cos(x3) * np.sin(x3)
    v[2] = np.sin(x2) * np.cos(x1) * np.sin(x1)
    return v


# ------------------------------------------------------- interpolation ----

def axis_split(x, h, n):
    """Wrap into [0,n), floor, snap within 1e-12 (interp.cpp:9-24)."""
    u = x / h
    u = u - np.floor(u / n) * n
    u = np.where(u < 0, 0.0, u)
    u = np.where(u >= n, u - n, u)
    fl = np.floor(u)
    s = u - fl
    base = fl.astype(np.int64)
    lo = s < SNAP_TOL
    hi = (~lo) & (s > 1.0 - SNAP_TOL)
    s = np.where(lo | hi, 0.0, s)
    base = np.where(hi, base + 1, base)
    base = np.where(base >= n, base - n, base)
    return base, s


def cubic_weights(s):
    """Lagrange basis on offsets {-1,0,1,2} (interp.cpp:26-35)."""
    sm, sp, s2 = s - 1.0, s + 1.0, s - 2.0
    return np.stack([-s * sm * s2 / 6.0, sp * sm * s2 / 2.0,
                     -sp * s * s2 / 2.0, sp * s * sm / 6.0])


def make_stencil(shape, xyz, degree):
    """Per-axis wrapped node indices and weights (interp.cpp:39-68)."""
    if degree not in (1, 3):
        raise ValueError("interpolation degree must be 1 or 3")
    xyz = np.asarray(xyz, dtype=np.float64).reshape(-1, 3)
    if np.isnan(xyz).any():
        raise ValueError("NaN query coordinate")
    h = spacing(shape)
    idx, w = [], []
    for a in range(3):
        n = shape[a]
        base, frac = axis_split(xyz[:, a], h[a], n)
        if degree == 1:
            idx.append(np.stack([base, np.where(base + 1 == n, 0, base + 1)]))
            w.append(np.stack([1.0 - frac, frac]))
        else:
            idx.append(np.stack([(base + o) % n for o in (-1, 0, 1, 2)]))
            w.append(cubic_weights(frac))
    return idx, w


def interp(f, xyz, degree=3):
    """out[p] = sum_a w1 sum_b w2 sum_c w3 f, order a->b->c
    (interp.hpp:47-61, interp.cpp:70-82)."""
    f = np.asarray(f, dtype=np.float64)
    (i1, i2, i3), (w1, w2, w3) = make_stencil(f.shape, xyz, degree)
    nn = degree + 1
    acc1 = np.zeros(i1.shape[1])
    for a in range(nn):
        acc2 = np.zeros_like(acc1)
        for b in range(nn):
            acc3 = np.zeros_like(acc1)
            for c in range(nn):
                acc3 += w3[c] * f[i1[a], i2[b], i3[c]]
            acc2 += w2[b] * acc3
        acc1 += w1[a] * acc2
    return acc1


def scatter(shape, xyz, z, degree=3):
    """acc[node] += w1 w2 w3 z[p], the exact transpose of interp
    (interp.cpp:92-108)."""
    (i1, i2, i3), (w1, w2, w3) = make_stencil(shape, xyz, degree)
    z = np.asarray(z, dtype=np.float64).ravel()
    acc = np.zeros(shape)
    nn = degree + 1
    for a in range(nn):
        for b in range(nn):
            for c in range(nn):
                np.add.at(acc, (i1[a], i2[b], i3[c]), w1[a] * w2[b] * w3[c] * z)
    return acc


# ---------------------------------------------------- characteristics ----

def characteristics(v, nt, degree=3):
    """RK2 departure points x* = x - dt v, dep = x - dt/2 (v + v(x*)),
    interleaved (n1,n2,n3,3) radians; identity when max|v| == 0
    (engine.hpp:111-155)."""
    v = np.asarray(v, dtype=np.float64)
    shape = v.shape[1:]
    dt = 1.0 / nt
    X = [np.broadcast_to(x, shape) for x in node_coords(shape)]
    identity = float(np.abs(v).max()) == 0.0
    if identity:
        return np.stack(X, axis=-1).copy(), True
    mid = np.stack([X[a] - dt * v[a] for a in range(3)], axis=-1)
    vs = [interp(v[c], mid, degree).reshape(shape) for c in range(3)]
    dep = np.stack([X[a] - dt / 2 * (v[a] + vs[a]) for a in range(3)], axis=-1)
    return dep, False


def displacement_grid_units(dep, shape):
    """Departure point minus node in grid units, wrapped to [-n/2, n/2):
    the device stores characteristics in this form."""
    h = spacing(shape)
    idx = np.indices(shape)
    out = np.empty((3,) + tuple(shape))
    for a in range(3):
        n = shape[a]
        d = dep[..., a] / h[a] - idx[a]
        out[a] = (d + n / 2) % n - n / 2
    return out


# ------------------------------------------------------- finite diffs ----

def central_difference_weights(half_width=4, deriv=1):
    """Fornberg recursion at z = 0 on nodes -hw..hw (fd.cpp:7-48)."""
    n = 2 * half_width
    m = deriv
    x = [float(i - half_width) for i in range(n + 1)]
    c = [[0.0] * (m + 1) for _ in range(n + 1)]
    c1, c4 = 1.0, x[0]
    c[0][0] = 1.0
    for i in range(1, n + 1):
        mn = min(i, m)
        c2, c5, c4 = 1.0, c4, x[i]
        for j in range(i):
            c3 = x[i] - x[j]
            c2 *= c3
            if j == i - 1:
                for k in range(mn, 0, -1):
                    c[i][k] = c1 * (k * c[i - 1][k - 1] - c5 * c[i - 1][k]) / c2
                c[i][0] = -c1 * c5 * c[i - 1][0] / c2
            for k in range(mn, 0, -1):
                c[j][k] = (c4 * c[j][k] - k * c[j][k - 1]) / c3
            c[j][0] = c4 * c[j][0] / c3
        c1 = c2
    return np.array([c[i][m] for i in range(n + 1)])


def _fd_axis(f, axis, hinv):
    w = central_difference_weights()
    if axis == 0:  # paired antisymmetric form (fd.cpp:60-78)
        acc = np.zeros_like(f)
        for j in range(1, 5):
            acc += w[4 + j] * (np.roll(f, -j, axis=0) - np.roll(f, j, axis=0))
        return acc * hinv
    acc = np.zeros_like(f)  # unpaired 9-tap sum (fd.cpp:80-125)
    for s in range(9):
        acc += w[s] * np.roll(f, -(s - 4), axis=axis)
    return acc * hinv


def fd_grad(f):
    """8th-order periodic gradient (fd.cpp:150-162)."""
    f = np.asarray(f, dtype=np.float64)
    if min(f.shape) < 9:
        raise ValueError("fd kernels need grid sizes >= 9")
    h = spacing(f.shape)
    return np.stack([_fd_axis(f, a, 1.0 / h[a]) for a in range(3)])


def fd_div(v):
    """8th-order periodic divergence (fd.cpp:164-179)."""
    v = np.asarray(v, dtype=np.float64)
    h = spacing(v.shape[1:])
    out = _fd_axis(v[0], 0, 1.0 / h[0])
    out = out + _fd_axis(v[1], 1, 1.0 / h[1])
    out = out + _fd_axis(v[2], 2, 1.0 / h[2])
    return out


# ------------------------------------------------------------ spectral ----

def _ksq_half(shape):
    f1 = signed_freq(shape[0])[:, None, None]
    f2 = signed_freq(shape[1])[None, :, None]
    f3 = np.arange(shape[2] // 2 + 1, dtype=np.float64)[None, None, :]
    return f1, f2, f3, f1 * f1 + f2 * f2 + f3 * f3


def regop(v, beta, unit_zero_mode=True):
    """beta |k|^2 per component; k=0 -> 1 or 0 (spectral.cpp:48-70)."""
    if beta <= 0:
        raise ValueError("regularization beta must be > 0")
    v = np.asarray(v, dtype=np.float64)
    shape = v.shape[1:]
    sym = _ksq_half(shape)[3].copy()
    sym[0, 0, 0] = 1.0 if unit_zero_mode else 0.0
    return np.stack([np.fft.irfftn(np.fft.rfftn(v[c]) * (beta * sym), s=shape, axes=(0, 1, 2))
                     for c in range(3)])


def inv_regop(w, beta):
    """Divide by beta |k|^2, zero mode by beta (spectral.cpp:72-93)."""
    if beta <= 0:
        raise ValueError("regularization beta must be > 0")
    w = np.asarray(w, dtype=np.float64)
    shape = w.shape[1:]
    sym = _ksq_half(shape)[3].copy()
    sym[0, 0, 0] = 1.0
    return np.stack([np.fft.irfftn(np.fft.rfftn(w[c]) / (beta * sym), s=shape, axes=(0, 1, 2))
                     for c in range(3)])


def seminorm(v):
    """sum_c sum w3 |k|^2 |V|^2 (2pi)^3/N^2 (spectral.cpp:95-118)."""
    v = np.asarray(v, dtype=np.float64)
    shape = v.shape[1:]
    N = float(np.prod(shape))
    ksq = _ksq_half(shape)[3]
    w3 = np.full(shape[2] // 2 + 1, 2.0)
    w3[0] = 1.0
    if shape[2] % 2 == 0:
        w3[-1] = 1.0
    total = 0.0
    for c in range(3):
        F = np.fft.rfftn(v[c])
        total += float((w3 * ksq * (F.real ** 2 + F.imag ** 2)).sum())
    return total * TWO_PI ** 3 / (N * N)


def leray(v):
    """v - k (k.v)/|k|^2, zero mode untouched (spectral.cpp:120-147)."""
    v = np.asarray(v, dtype=np.float64)
    shape = v.shape[1:]
    f1, f2, f3, ksq = _ksq_half(shape)
    F = [np.fft.rfftn(v[c]) for c in range(3)]
    safe = np.where(ksq == 0, 1.0, ksq)
    kv = (f1 * F[0] + f2 * F[1] + f3 * F[2]) / safe
    kv = np.where(ksq == 0, 0.0, kv)
    return np.stack([np.fft.irfftn(F[c] - k * kv, s=shape, axes=(0, 1, 2))
                     for c, k in enumerate((f1, f2, f3))])


def _restrict_matrix(nf):
    """Coarse-from-fine selection on one axis: the coarse Nyquist line sums
    its two fine alias partners (spectral.cpp:17-28, 149-174)."""
    nc = nf // 2
    R = np.zeros((nc, nf))
    for k in range(nc):
        nu = k if k <= nc // 2 else k - nc
        if abs(nu) == nc // 2:
            R[k, (nc // 2) % nf] += 1.0
            R[k, (-(nc // 2)) % nf] += 1.0
        else:
            R[k, nu % nf] = 1.0
    return R


def _prolong_matrix(nf):
    """Fine-from-coarse split on one axis: Nyquist coarse modes split evenly
    over both fine partners (spectral.cpp:176-203)."""
    nc = nf // 2
    P = np.zeros((nf, nc))
    for k in range(nc):
        nu = k if k <= nc // 2 else k - nc
        if abs(nu) == nc // 2:
            P[(nc // 2) % nf, k] = 0.5
            P[(-(nc // 2)) % nf, k] = 0.5
        else:
            P[nu % nf, k] = 1.0
    return P


def _apply3(mats, F):
    F = np.tensordot(mats[0], F, axes=([1], [0]))
    F = np.tensordot(mats[1], F, axes=([1], [1])).transpose(1, 0, 2)
    F = np.tensordot(mats[2], F, axes=([1], [2])).transpose(1, 2, 0)
    return F


def restrict(f):
    """Spectral restriction to the half grid, amplitude preserving
    (spectral.cpp:149-174, 242-251)."""
    f = np.asarray(f, dtype=np.float64)
    if f.ndim == 4:
        return np.stack([restrict(f[c]) for c in range(3)])
    shape = f.shape
    cs = tuple(n // 2 for n in shape)
    scal = float(np.prod(cs)) / float(np.prod(shape))
    C = _apply3([_restrict_matrix(n) for n in shape], np.fft.fftn(f)) * scal
    return np.real(np.fft.ifftn(C))


def prolong(fc, fine_shape):
    """Spectral prolongation from the half grid (spectral.cpp:176-203,
    253-260)."""
    fc = np.asarray(fc, dtype=np.float64)
    if fc.ndim == 4:
        return np.stack([prolong(fc[c], fine_shape) for c in range(3)])
    scal = float(np.prod(fine_shape)) / float(np.prod(fc.shape))
    F = _apply3([_prolong_matrix(n) for n in fine_shape], np.fft.fftn(fc)) * scal
    return np.real(np.fft.ifftn(F))


def high_pass(f):
    """f minus its coarse-representable band, alias-pair averages removed on
    the coarse Nyquist lines (spectral.cpp:205-240, 262-268)."""
    f = np.asarray(f, dtype=np.float64)
    if f.ndim == 4:
        return np.stack([high_pass(f[c]) for c in range(3)])
    F = np.fft.fftn(f)
    PR = _apply3([_prolong_matrix(n) @ _restrict_matrix(n) for n in f.shape], F)
    return np.real(np.fft.ifftn(F - PR))


# ----------------------------------------------------------- transport ----

def trapezoid_weight(t, nt, dt):
    """transport.hpp:10-12."""
    return dt / 2 if t in (0, nt) else dt


def solve_state(dep, m0, nt, degree=3):
    """m(.,t+1) = I[m(.,t)] at forward chars (transport.hpp:90-102)."""
    m = [np.asarray(m0, dtype=np.float64)]
    for _ in range(nt):
        m.append(interp(m[-1], dep, degree).reshape(m0.shape))
    return m


def solve_inc_state(dep, vt, grads, nt, degree=3):
    """m~_{t+1} = I[m~_t] - dt/2 (I[u_t] + u_{t+1}), u_t = vt . grad m_t,
    m~_0 = 0 (transport.hpp:145-181)."""
    dt = 1.0 / nt
    shape = vt.shape[1:]
    mt = [np.zeros(shape)]
    u_prev = (vt * grads[0]).sum(axis=0)
    for t in range(nt):
        u_next = (vt * grads[t + 1]).sum(axis=0)
        step = interp(mt[t], dep, degree).reshape(shape)
        u_dep = interp(u_prev, dep, degree).reshape(shape)
        step = step - dt / 2 * u_dep
        step = step - dt / 2 * u_next
        mt.append(step)
        u_prev = u_next
    return mt


def adjoint_transpose_assemble(dep, grads, fin, nt, degree=3):
    """out = sum_t w_t psi_t grad m_t, psi_nt = fin, psi_{t-1} = I^T psi_t
    (transport.hpp:207-228)."""
    dt = 1.0 / nt
    shape = fin.shape
    out = np.zeros((3,) + shape)
    psi = np.asarray(fin, dtype=np.float64)
    for t in range(nt, -1, -1):
        out += trapezoid_weight(t, nt, dt) * psi[None] * grads[t]
        if t > 0:
            psi = scatter(shape, dep, psi, degree)
    return out


def adjoint_source_factor(v, bwd, nt, degree=3):
    """q = (1 + dt/2 D(dep)) / (1 - dt/2 D), D = div v (transport.hpp:49-64)."""
    dt = 1.0 / nt
    d = fd_div(v)
    if dt / 2 * np.abs(d).max() >= 0.99:
        raise ArithmeticError("divergence too large for the time step")
    d_dep = interp(d, bwd, degree).reshape(d.shape)
    return (1.0 + dt / 2 * d_dep) / (1.0 - dt / 2 * d)


def adjoint_sweep(bwd, q, fin, nt, degree=3):
    """lambda_t = I_bwd[lambda_{t+1}] .* q (transport.hpp:106-121)."""
    lam = [None] * (nt + 1)
    lam[nt] = np.asarray(fin, dtype=np.float64)
    for t in range(nt - 1, -1, -1):
        lam[t] = interp(lam[t + 1], bwd, degree).reshape(fin.shape) * q
    return lam


def integrate_lambda_grad_m(lam, grads, nt):
    """sum_t w_t lambda_t grad m_t (transport.hpp:184-201)."""
    dt = 1.0 / nt
    out = np.zeros_like(grads[0])
    for t in range(nt + 1):
        out += trapezoid_weight(t, nt, dt) * lam[t][None] * grads[t]
    return out


class Linearization:
    """Objective + gradient + cached state at velocity v; the state
    gauss_newton_level carries into PCG (optim.hpp:66-111, 155-168)."""

    def __init__(self, m0, m1, v, beta, nt=4, degree=3):
        self.nt, self.degree, self.beta = nt, degree, beta
        self.v = np.asarray(v, dtype=np.float64)
        self.m1 = np.asarray(m1, dtype=np.float64)
        self.fwd, self.fwd_identity = characteristics(self.v, nt, degree)
        self.m = solve_state(self.fwd, np.asarray(m0, dtype=np.float64), nt, degree)
        resid = self.m[-1] - self.m1
        self.mismatch = 0.5 * inner(resid, resid)
        self.regularization = beta / 2 * seminorm(self.v)
        self.J = self.mismatch + self.regularization
        self.grads = [fd_grad(mt) for mt in self.m]
        self.bwd, _ = characteristics(-self.v, nt, degree)
        q = adjoint_source_factor(self.v, self.bwd, nt, degree)
        lam = adjoint_sweep(self.bwd, q, self.m1 - self.m[-1], nt, degree)
        self.g = integrate_lambda_grad_m(lam, self.grads, nt) + regop(self.v, beta, False)

    def inc_state(self, vt):
        return solve_inc_state(self.fwd, np.asarray(vt, dtype=np.float64), self.grads,
                               self.nt, self.degree)

    def matvec(self, vt):
        """GN matvec beta A vt + transpose-adjoint data term
        (optim.hpp:115-137, HessianAdjoint::Transpose)."""
        vt = np.asarray(vt, dtype=np.float64)
        mt = self.inc_state(vt)
        h = adjoint_transpose_assemble(self.fwd, self.grads, -mt[-1], self.nt, self.degree)
        return h + regop(vt, self.beta, False)
