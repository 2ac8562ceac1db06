"""Per-kernel parity of the sm_100a path against the oracle (fp32 device vs
fp64 reference): relative L2 <= 1e-5 per kernel (BASELINE.json north_star).

Oracles: the compiled, unmodified reference (oracle/_ref/libvreg_ref.so via
oracle/ref.py) and its numpy restatement (oracle/vreg_np.py), on the SYN
inputs (proj/src/syn.cpp) and the reference's test fixtures
(proj/tests/test_util.hpp). All device calls go through the C ABI.
"""
import numpy as np
import pytest
import torch

from oracle import ref
from oracle import vreg_np as O

pytestmark = pytest.mark.gpu

TOL = 1e-5


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def host(t):
    return t.detach().double().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def syn32():
    m0, v, m1 = ref.syn(32)
    return m0, v, m1


def random_smooth(shape, seed, kmax=3, nmodes=8):
    """Band-limited random field like test_util.hpp:13-38 (numpy RNG)."""
    rng = np.random.default_rng(seed)
    x1, x2, x3 = O.node_coords(shape)
    f = np.zeros(shape)
    for _ in range(nmodes):
        a = rng.uniform(-1, 1)
        k = rng.integers(-kmax, kmax + 1, 3)
        p = rng.uniform(0, 2 * np.pi, 3)
        f += a * np.cos(k[0] * x1 + p[0]) * np.cos(k[1] * x2 + p[1]) * np.cos(k[2] * x3 + p[2])
    return f


def test_syn_inputs(ctx, syn32):
    m0, v, _ = syn32
    g = ctx.grid(32)
    assert rel(host(ctx.syn_template(g)), m0) < 1e-7
    assert rel(host(ctx.syn_velocity(g)), v) < 1e-7


@pytest.mark.parametrize("degree", [1, 3])
def test_characteristics_match_reference(ctx, syn32, degree):
    _, v, _ = syn32
    g = ctx.grid(32)
    xyz, ident = ref.characteristics(0.5 * v, 4, degree)
    disp_ref = O.displacement_grid_units(xyz, (32, 32, 32))
    disp, flags = ctx.characteristics(g, dev(0.5 * v), degree)
    assert flags & 1 == 0 and not ident
    assert np.abs(host(disp) - disp_ref).max() < 2e-5
    assert rel(host(disp), disp_ref) < TOL


def test_characteristics_identity(ctx):
    g = ctx.grid(16)
    disp, flags = ctx.characteristics(g, ctx.field(g, 3), 3)
    assert flags & 1 == 1
    assert float(disp.abs().max()) == 0.0


@pytest.mark.parametrize("degree", [1, 3])
def test_interp_and_scatter_at_characteristics(ctx, syn32, degree):
    m0, v, _ = syn32
    g = ctx.grid(32)
    xyz, _ = ref.characteristics(0.5 * v, 4, degree)
    chars = ctx.characteristics(g, dev(0.5 * v), degree)
    f = random_smooth((32, 32, 32), 5)
    out = ctx.interp(g, dev(f), chars, degree)
    assert rel(host(out), ref.interp(f, xyz, degree).reshape(32, 32, 32)) < TOL
    z = random_smooth((32, 32, 32), 9)
    sc = ctx.scatter(g, dev(z), chars, degree)
    assert rel(host(sc), ref.scatter((32, 32, 32), xyz, z, degree)) < TOL


def test_scatter_is_transpose_of_interp(ctx, syn32):
    """<I f, z> = <f, I^T z> (test_interp.cpp:154-173) on device."""
    _, v, _ = syn32
    g = ctx.grid(32)
    for degree in (1, 3):
        chars = ctx.characteristics(g, dev(0.5 * v), degree)
        f = dev(np.random.default_rng(1).uniform(-1, 1, (32, 32, 32)))
        z = dev(np.random.default_rng(2).uniform(-1, 1, (32, 32, 32)))
        lhs = ctx.inner(g, ctx.interp(g, f, chars, degree), z)
        rhs = ctx.inner(g, f, ctx.scatter(g, z, chars, degree))
        assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


def test_fd_gradient_divergence(ctx):
    g = ctx.grid(32)
    f = random_smooth((32, 32, 32), 11)
    assert rel(host(ctx.fd_grad(g, dev(f))), ref.fd_grad(f)) < TOL
    w = np.stack([random_smooth((32, 32, 32), s) for s in (12, 13, 14)])
    assert rel(host(ctx.fd_div(g, dev(w))), ref.fd_div(w)) < TOL


def test_fd_nonsquare_and_constant(ctx):
    g = ctx.grid(16, 12, 20)
    f = random_smooth((16, 12, 20), 3)
    assert rel(host(ctx.fd_grad(g, dev(f))), ref.fd_grad(f)) < TOL
    c = torch.full((16, 12, 20), 4.25, device="cuda")
    assert float(ctx.fd_grad(g, c).abs().max()) == 0.0  # paired form: exact (test_fd.cpp:72-78)


@pytest.mark.parametrize("shape", [(32, 32, 32), (64, 32, 128), (32, 256, 64), (512, 32, 32), (1024, 32, 32), (32, 32, 1024)])
def test_regop_separable_passes(ctx, shape):
    """The regop runs as three 1-D spectral passes (spec_axis.cu) on
    power-of-two grids; white noise exercises every mode incl. Nyquist, the
    per-component offsets the unit null-mode symbol (+ beta mean(v))."""
    g = ctx.grid(*shape)
    rng = np.random.default_rng(sum(shape))
    r = np.stack([random_smooth(shape, s) for s in (31, 32, 33)]) + 0.2 * rng.standard_normal((3, *shape))
    r += np.array([0.7, -0.3, 0.0])[:, None, None, None]
    rd = dev(r)
    assert rel(host(ctx.regop(g, rd, 0.37, False)), ref.regop(r, 0.37, False)) < TOL
    assert rel(host(ctx.regop(g, rd, 0.37, True)), ref.regop(r, 0.37, True)) < TOL


def test_spectral_operators(ctx):
    shape = (16, 12, 20)
    g = ctx.grid(*shape)
    r = np.stack([random_smooth(shape, s) for s in (21, 22, 23)])
    r += 0.1 * np.random.default_rng(0).uniform(-1, 1, r.shape)
    rd = dev(r)
    assert rel(host(ctx.regop(g, rd, 0.37, True)), ref.regop(r, 0.37, True)) < TOL
    assert rel(host(ctx.regop(g, rd, 0.37, False)), ref.regop(r, 0.37, False)) < TOL
    assert rel(host(ctx.inv_regop(g, rd, 5e-3)), ref.inv_regop(r, 5e-3)) < TOL
    assert abs(ctx.seminorm(g, rd) / ref.seminorm(r) - 1) < TOL
    assert rel(host(ctx.leray(g, rd)), ref.leray(r)) < TOL
    assert rel(host(ctx.restrict(g, rd)), np.stack([ref.restrict(r[c]) for c in range(3)])) < TOL
    assert rel(host(ctx.high_pass(g, rd)), np.stack([ref.high_pass(r[c]) for c in range(3)])) < TOL
    rc = r[:, :8, :6, :10].copy()
    assert rel(host(ctx.prolong(g, dev(rc))), np.stack([ref.prolong(rc[c], shape) for c in range(3)])) < TOL


def test_spectral_band_edges(ctx):
    """restrict/high_pass at the coarse Nyquist (test_spectral.cpp:200-221)."""
    shape = (64, 64, 64)
    g = ctx.grid(64)
    x1 = O.node_coords(shape)[0] + np.zeros(shape)
    for k, fn in ((16, np.cos), (16, np.sin), (15, np.sin), (17, np.sin)):
        f = fn(k * x1)
        assert rel(host(ctx.restrict(g, dev(f))), ref.restrict(f)) < 1e-5 or \
            np.abs(host(ctx.restrict(g, dev(f)))).max() < 1e-5
        hp = host(ctx.high_pass(g, dev(f)))
        assert np.abs(hp - ref.high_pass(f)).max() < 1e-5


def test_h0_matvec(ctx):
    shape = (16, 16, 16)
    g = ctx.grid(16)
    s = np.stack([random_smooth(shape, q) for q in (31, 32, 33)])
    gm = np.stack([random_smooth(shape, q) for q in (34, 35, 36)])
    expect = ref.regop(s, 0.05, True) + gm * (gm * s).sum(axis=0)[None]
    assert rel(host(ctx.h0_matvec(g, dev(s), dev(gm), 0.05)), expect) < TOL


def test_reductions_match_reference(ctx):
    shape = (16, 12, 20)
    g = ctx.grid(*shape)
    a = np.random.default_rng(3).uniform(-1, 1, shape)
    b = np.random.default_rng(4).uniform(-1, 1, shape)
    assert abs(ctx.inner(g, dev(a), dev(b)) - ref.inner(a.astype(np.float32), b.astype(np.float32))) < 1e-10
    c = torch.ones((16, 16, 16), device="cuda")
    assert abs(ctx.inner(ctx.grid(16), c, c) - (2 * np.pi) ** 3) < 1e-10  # test_fields.cpp:28-36
    assert ctx.max_abs(g, dev(a)) == float(np.abs(a.astype(np.float32)).max())


def test_node_queries_exact_and_errors(ctx):
    """test_interp.cpp:25-40 and :145-152 on device."""
    from paper_2008_12820_b200 import VregError
    shape = (16, 12, 20)
    g = ctx.grid(*shape)
    f = np.random.default_rng(3).uniform(-1, 1, shape).astype(np.float32)
    nodes = np.array([[0, 0, 0], [3, 5, 7], [15, 11, 19], [8, 0, 19], [1, 11, 0]])
    h = np.array(O.spacing(shape))
    xyz = torch.as_tensor(nodes * h, dtype=torch.float64, device="cuda")
    for degree in (1, 3):
        vals = host(ctx.interp_points(g, dev(f), xyz, degree))
        assert np.array_equal(vals, f[nodes[:, 0], nodes[:, 1], nodes[:, 2]].astype(np.float64))
    bad = xyz.clone()
    bad[0, 1] = float("nan")
    with pytest.raises(VregError) as e:
        ctx.interp_points(g, dev(f), bad, 3)
    assert e.value.kind == "input_error"
    with pytest.raises(VregError) as e:
        ctx.interp_points(g, dev(f), xyz, 2)
    assert e.value.kind == "parameter_error"


def test_point_interp_matches_reference_random_points(ctx):
    shape = (16, 16, 16)
    g = ctx.grid(16)
    f = random_smooth(shape, 41)
    q = np.random.default_rng(43).uniform(0, 2 * np.pi, (500, 3))
    xyz = torch.as_tensor(q, dtype=torch.float64, device="cuda")
    z = np.random.default_rng(83).uniform(-1, 1, 500)
    for degree in (1, 3):
        assert rel(host(ctx.interp_points(g, dev(f), xyz, degree)), ref.interp(f, q, degree)) < TOL
        acc = host(ctx.scatter_points(g, xyz, dev(z), degree))
        assert rel(acc, ref.scatter(shape, q, z, degree)) < TOL
