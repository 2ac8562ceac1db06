"""Parity of the device transport solves and the fused GN Hessian matvec with
the unmodified reference at a fixed linearisation point (SYN inputs, nt=4,
beta=1e-3, v = 0.5 v_syn, vt = -g: BASELINE.md §2a, SURVEY §8c probe).

Everything on the device side is computed on the device from the SYN
generators; the reference side is oracle/_ref (fp64).
"""
import numpy as np
import pytest
import torch

from oracle import ref

pytestmark = pytest.mark.gpu

TOL = 1e-5
BETA = 1e-3


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def host(t):
    return t.detach().double().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


class DeviceLin:
    """Device-side objective/gradient/state cache built from the C ABI
    (optim.hpp:68-111 composition)."""

    def __init__(self, ctx, n, degree=3, nt=4, vscale=0.5):
        self.ctx, self.g, self.degree = ctx, ctx.grid(n, nt=nt), degree
        g = self.g
        m0 = ctx.syn_template(g)
        vsyn = ctx.syn_velocity(g)
        m1 = ctx.solve_state(g, ctx.characteristics(g, vsyn, degree), m0, degree)[nt].clone()
        self.m0, self.m1 = m0, m1
        self.v = vsyn * vscale
        self.fwd = ctx.characteristics(g, self.v, degree)
        self.m = ctx.solve_state(g, self.fwd, m0, degree)
        self.grads = torch.stack([ctx.fd_grad(g, self.m[t].contiguous()) for t in range(nt + 1)])
        self.bwd = ctx.characteristics(g, (-self.v).contiguous(), degree)
        q = ctx.adjoint_source_factor(g, self.v, self.bwd, degree)
        lam = ctx.adjoint_sweep(g, self.bwd, q, (m1 - self.m[nt]).contiguous(), degree)
        self.gradient = ctx.integrate_lambda_grad_m(g, lam, self.grads)
        ctx.axpy(g, 1.0, ctx.regop(g, self.v, BETA, False), self.gradient)
        r = (self.m[nt] - m1).contiguous()
        self.mismatch = 0.5 * ctx.inner(g, r, r)
        self.J = self.mismatch + BETA / 2 * ctx.seminorm(g, self.v)

    def matvec(self, vt):
        return self.ctx.gn_matvec(self.g, self.fwd, self.grads, BETA, vt, self.degree)


@pytest.fixture(scope="module", params=[32, 64])
def pair(request, ctx):
    n = request.param
    m0, v, m1 = ref.syn(n)
    s = ref.Session(m0, m1, 0.5 * v, BETA, ref.Config(continuation=False, beta_target=BETA))
    return n, s, DeviceLin(ctx, n)


def test_state_and_objective(pair):
    n, s, d = pair
    assert rel(host(d.m), s.state()) < TOL
    J = s.objective()
    assert abs(d.mismatch / J["mismatch"] - 1) < TOL
    assert abs(d.J / J["total"] - 1) < TOL


def test_gradient(pair):
    n, s, d = pair
    assert rel(host(d.gradient), s.gradient()) < TOL


def test_inc_state(pair, ctx):
    n, s, d = pair
    g = s.gradient()
    mt = ctx.inc_state(d.g, d.fwd, d.grads, dev(-g), d.degree)
    assert rel(host(mt[1:]), s.inc_state(-g)[1:]) < TOL


def test_transpose_assemble(pair, ctx):
    n, s, d = pair
    fin = np.random.default_rng(7).uniform(-1, 1, (n, n, n))
    out = ctx.transpose_assemble(d.g, d.fwd, d.grads, dev(fin), d.degree)
    assert rel(host(out), s.transpose_assemble(fin)) < TOL


def test_gn_matvec(pair):
    n, s, d = pair
    g = s.gradient()
    H = d.matvec(dev(-g))
    Href = s.matvec(-g)
    assert rel(host(H), Href) < TOL


def test_matvec_probe_goldens_64(pair, ctx):
    """SURVEY §8c probe: ||H vt|| and <vt, H vt> at 64^3 (fp64 reference
    9.8356971587e-2 and 3.5306942713e-2), vt = -g, both on device."""
    n, s, d = pair
    if n != 64:
        pytest.skip("64^3 goldens")
    vt = (-d.gradient).contiguous()
    H = d.matvec(vt)
    assert abs(ctx.norm2(d.g, H) / 9.8356971587e-2 - 1) < 1e-4
    assert abs(ctx.inner(d.g, vt, H) / 3.5306942713e-2 - 1) < 1e-4


def test_hessian_symmetry(pair, ctx):
    """<u, H w> = <H u, w> (<= 1e-6 relative)."""
    n, s, d = pair
    rng = np.random.default_rng(11)
    u = dev(rng.standard_normal((3, n, n, n)) * 0.1)
    w = dev(rng.standard_normal((3, n, n, n)) * 0.1)
    a = ctx.inner(d.g, u, d.matvec(w))
    b = ctx.inner(d.g, d.matvec(u), w)
    assert abs(a - b) <= 1e-5 * max(abs(a), abs(b))


def test_deterministic_mode_is_bitwise_reproducible(ctx):
    """vreg_ctx_set_deterministic: exact fixed-point transpose sweeps give
    bit-identical matvecs run to run, within fp32 round-off of the default
    (fp32 L2 reductions) path."""
    from paper_2008_12820_b200.solver import Config, Solver
    n = 48
    s = Solver(ctx, n, Config(continuation=False, beta_target=1e-3))
    s.syn_images()
    v = (0.5 * ctx.syn_velocity(s.grid)).contiguous()
    s.linearize(v, 1e-3)
    vt = (-s.gradient()).contiguous()
    ctx.set_deterministic(True)
    try:
        a = s.matvec(vt).clone()
        b = s.matvec(vt).clone()
    finally:
        ctx.set_deterministic(False)
    c = s.matvec(vt)
    assert torch.equal(a, b)
    assert float((a - c).norm() / c.norm()) < 1e-6
    s.close()
