"""Generate tests/golden/golden.npz from the UNMODIFIED reference
(oracle/_ref/libvreg_ref.so, built by `make -C oracle` from
/root/reference/proj). Inputs are seeded numpy arrays stored alongside the
outputs, so the fixtures are usable where /root/reference is absent (the GPU
box, a fresh checkout).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from oracle import vreg_np as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
BETA = 1e-3


def smooth(shape, seed):
    rng = np.random.default_rng(seed)
    x1, x2, x3 = O.node_coords(shape)
    f = np.zeros(shape)
    for _ in range(8):
        a = rng.uniform(-1, 1)
        k = rng.integers(-3, 4, 3)
        p = rng.uniform(0, 2 * np.pi, 3)
        f += a * np.cos(k[0] * x1 + p[0]) * np.cos(k[1] * x2 + p[1]) * np.cos(k[2] * x3 + p[2])
    return f


def main():
    g = {}
    # kernels on a 16^3 SYN flow
    n = 16
    m0, v, m1 = ref.syn(n)
    g["syn16_m0"], g["syn16_v"], g["syn16_m1"] = m0, v, m1
    for deg in (1, 3):
        xyz, _ = ref.characteristics(0.5 * v, 4, deg)
        g[f"chars16_deg{deg}"] = xyz
        f = smooth((n, n, n), 5)
        g["f16"] = f
        g[f"interp16_deg{deg}"] = ref.interp(f, xyz, deg).reshape(n, n, n)
        g[f"scatter16_deg{deg}"] = ref.scatter((n, n, n), xyz, f, deg)
    g["fdgrad16"] = ref.fd_grad(g["f16"])
    w = np.stack([smooth((n, n, n), s) for s in (12, 13, 14)])
    g["w16"] = w
    g["fddiv16"] = ref.fd_div(w)
    # spectral operators on a non-cubic grid (test_spectral.cpp:69 shape)
    sh = (16, 12, 20)
    r = np.stack([smooth(sh, s) for s in (21, 22, 23)])
    r += 0.1 * np.random.default_rng(0).uniform(-1, 1, r.shape)
    g["r_nc"] = r
    g["regop_nc"] = ref.regop(r, 0.37, True)
    g["regop0_nc"] = ref.regop(r, 0.37, False)
    g["invregop_nc"] = ref.inv_regop(r, 5e-3)
    g["leray_nc"] = ref.leray(r)
    g["seminorm_nc"] = np.array(ref.seminorm(r))
    g["restrict_nc"] = ref.restrict(r[0])
    g["prolong_nc"] = ref.prolong(r[0][:8, :6, :10], sh)
    g["highpass_nc"] = ref.high_pass(r[0])
    g["fd8_weights"] = ref.fd8_weights()
    # linearisation scalars + matvec at 32^3 (v = 0.5 v_syn, vt = -g)
    n = 32
    m0, v, m1 = ref.syn(n)
    s = ref.Session(m0, m1, 0.5 * v, BETA, ref.Config(continuation=False, beta_target=BETA))
    J = s.objective()
    gr = s.gradient()
    H = s.matvec(-gr)
    g["lin32_J"] = np.array([J["total"], J["mismatch"], J["regularization"]])
    g["lin32_grad"] = gr.astype(np.float32)
    g["lin32_H"] = H.astype(np.float32)
    # fixed-iteration solves at 32^3 (scalars + counters)
    for pc in ("inva", "2linvh0"):
        cfg = ref.Config(continuation=False, beta_target=BETA, fixed_gn=2, fixed_pcg=5, precond=pc)
        vv, rep, cnt = ref.register(m0, m1, cfg)
        g[f"solve32_{pc}_rep"] = np.array([rep["final_mismatch"], rep["final_g_rel"],
                                           O.norm2(vv), rep["cost_model_matches"]])
        g[f"solve32_{pc}_counters"] = np.array([cnt[k] for k in ref.COUNTER_NAMES], dtype=np.int64)
    np.savez_compressed(OUT, **g)
    print(OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
