"""Cubic B-spline interpolation (B200 extension named by the north star; the
reference implements Lagrange cubic and trilinear only, interp.cpp:26-35,
SPEC.md:219, so there is no reference run). degree 4 = VREG_INTERP_BSPLINE3.

Independent oracle: scipy.ndimage (spline_filter + map_coordinates with
order 3, mode 'grid-wrap' -- the periodic cubic B-spline), at the departure
points of our own RK2 characteristics and at arbitrary query points; plus
the exact transpose identity <I f, z> = <f, I^T z>, interpolation of the
node values (zero displacement after a whole-cell shift), and the
registration gradient as the derivative of the objective.
"""
import math

import numpy as np
import pytest
import torch
from scipy import ndimage

from paper_2008_12820_b200 import VregGrid
from paper_2008_12820_b200.solver import Config, Solver

pytestmark = pytest.mark.gpu
BS = 4


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")


def host(t):
    return t.detach().double().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def smooth(shape, seed):
    rng = np.random.default_rng(seed)
    x = [np.arange(n) * 2 * math.pi / n for n in shape]
    X = np.meshgrid(*x, indexing="ij")
    f = np.zeros(shape)
    for _ in range(6):
        k = rng.integers(-4, 5, size=3)
        f += rng.standard_normal() * np.cos(k[0] * X[0] + k[1] * X[1] + k[2] * X[2] + rng.uniform(0, 6))
    return f


def departure_grid_units(ctx, g, shape, v):
    disp, flags = ctx.characteristics(g, dev(v), BS)
    d = host(disp)
    idx = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    return np.stack([idx[a] + d[a] for a in range(3)]), (disp, flags)


@pytest.mark.parametrize("shape", [(32, 32, 32), (24, 20, 28)])
def test_bspline_interp_matches_scipy(ctx, shape):
    g = VregGrid(*shape, 4)
    f = smooth(shape, 3)
    h = 2 * math.pi / np.array(shape)
    x = [np.arange(n) * hh for n, hh in zip(shape, h)]
    X = np.meshgrid(*x, indexing="ij")
    v = np.stack([0.4 * np.sin(X[2]) * np.cos(X[1]), 0.3 * np.cos(X[0]), 0.5 * np.sin(X[1] + X[0])])
    coords, chars = departure_grid_units(ctx, g, shape, v)
    ref = ndimage.map_coordinates(f, coords.reshape(3, -1), order=3, mode="grid-wrap").reshape(shape)
    out = host(ctx.interp(g, dev(f), chars, BS))
    assert rel(out, ref) < 1e-5


def test_bspline_transpose_identity(ctx):
    shape = (32, 32, 32)
    g = VregGrid(*shape, 4)
    X = np.meshgrid(*[np.arange(n) * 2 * math.pi / n for n in shape], indexing="ij")
    v = np.stack([0.5 * np.sin(X[2]), 0.4 * np.cos(X[0] + X[2]), 0.3 * np.sin(X[1])])
    _, chars = departure_grid_units(ctx, g, shape, v)
    f, z = smooth(shape, 11), smooth(shape, 12)
    If = host(ctx.interp(g, dev(f), chars, BS))
    ITz = host(ctx.scatter(g, dev(z), chars, BS))
    a, b = (If * z).sum(), (f * ITz).sum()
    assert abs(a / b - 1) < 1e-5


def test_bspline_points_match_scipy(ctx):
    shape = (24, 20, 28)
    g = VregGrid(*shape, 4)
    f = smooth(shape, 5)
    rng = np.random.default_rng(9)
    h = 2 * math.pi / np.array(shape)
    m = 5000
    xyz = rng.uniform(-7.0, 14.0, size=(m, 3))  # radians, several periods
    out = host(ctx.interp_points(g, dev(f), torch.as_tensor(xyz, device="cuda"), BS))
    ref = ndimage.map_coordinates(f, (xyz / h).T, order=3, mode="grid-wrap")
    assert rel(out, ref) < 1e-5
    # whole-cell shift: B-spline interpolation reproduces the node values
    nodes = np.stack(np.meshgrid(*[np.arange(n) for n in shape], indexing="ij"), -1).reshape(-1, 3)
    shifted = ((nodes + [2, -1, 3]) * h)
    out = host(ctx.interp_points(g, dev(f), torch.as_tensor(shifted, device="cuda"), BS))
    assert rel(out, np.roll(f, (-2, 1, -3), axis=(0, 1, 2)).ravel()) < 1e-5


def test_bspline_registration_gradient_is_the_derivative(ctx):
    n, beta = 32, 1e-2
    s = Solver(ctx, n, Config(continuation=False, beta_target=beta, interp_degree=BS))
    s.syn_images()
    v = (0.5 * ctx.syn_velocity(s.grid)).contiguous()
    s.linearize(v, beta)
    g = s.gradient().double()
    d = g / float(g.abs().max()) * 0.25  # along the gradient, ~1e-3 of v at eps 1e-3
    gd = float((g * d).sum() * (2 * math.pi / n) ** 3)
    eps = 1e-3
    Js = []
    for sgn in (1, -1):
        s.linearize((v.double() + sgn * eps * d).float().contiguous(), beta)
        Js.append(s.objective()["total"])
    assert abs((Js[0] - Js[1]) / (2 * eps) / gd - 1) < 1e-3
    # and a GN solve with it reduces the mismatch
    r = Solver(ctx, n, Config(continuation=False, beta_target=1e-3, interp_degree=BS,
                              fixed_gn=2, fixed_pcg=5))
    r.syn_images()
    _, rep, _ = r.register()
    assert rep["final_mismatch"] < 0.2 * rep["initial_mismatch"]
    s.close()
    r.close()
