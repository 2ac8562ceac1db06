"""Multi-GPU parity check (run under torchrun, one process per GPU):
the x1-slab decomposed run on p GPUs against a single-GPU run of the same
problem (rank 0 owns a second, non-distributed context on its GPU).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py [n]

Checks (p-independence): SYN inputs, state-derived
objective, gradient, GN matvec, InvA preconditioner, fixed-iteration solve.
Prints one JSON line on rank 0; exit status 1 on failure.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2008_12820_b200 import Context  # noqa: E402
from paper_2008_12820_b200.dist import init_from_env  # noqa: E402
from paper_2008_12820_b200.solver import Config, Solver  # noqa: E402


def run(ctx, dims, beta):
    big = dims[0] * dims[1] * dims[2] > 128 ** 3  # 512^3: kernels and operators only
    cfg = Config(continuation=False, beta_target=beta, precond="inva")
    s = Solver(ctx, dims, cfg)
    s.syn_images()
    g = s.grid
    v = (0.5 * ctx.syn_velocity(g)).contiguous()
    s.linearize(v, beta)
    J = s.objective()
    grad = s.gradient()
    vt = (-grad).contiguous()
    H = s.matvec(vt)
    ctx.set_deterministic(True)  # exact fixed-point transpose: bitwise p-independent
    Hd = s.matvec(vt)
    ctx.set_deterministic(False)
    P, _ = s.precond("inva", vt, 0.5)
    P2, _ = s.precond("2linvh0", vt, 0.5)
    m0, m1 = s.images()
    out = {"J": J, "grad": ctx.to_global(g, grad), "H": ctx.to_global(g, H),
           "Hdet": ctx.to_global(g, Hd), "P": ctx.to_global(g, P), "P2": ctx.to_global(g, P2),
           "m1": ctx.to_global(g, m1)}
    s.close()
    if big:
        return out
    # optimize-then-discretize (SL incremental adjoint) Hessian, optim.hpp:125-128
    s_sl = Solver(ctx, dims, Config(continuation=False, beta_target=beta, precond="inva",
                                    hessian_adjoint=1))
    s_sl.syn_images()
    s_sl.linearize(v, beta)
    out["H_sl"] = ctx.to_global(g, s_sl.matvec(vt))
    s_sl.close()
    cfg2 = Config(continuation=False, beta_target=beta, precond="inva", fixed_gn=2, fixed_pcg=3)
    s2 = Solver(ctx, dims, cfg2)
    s2.syn_images()
    vv, rep, cnt = s2.register()
    out["solve"] = rep
    out["v"] = ctx.to_global(g, vv)
    s2.close()
    # two-level preconditioner pieces (distributed restrict/prolong/high pass)
    rng = np.random.default_rng(5)
    fg = rng.standard_normal((3,) + tuple(dims)).astype(np.float32)
    f = ctx.from_global(g, fg)
    out["regop"] = ctx.to_global(g, ctx.regop(g, f, beta, False))  # separable passes
    out["restrict"] = ctx.to_global(VregGridC(g), ctx.restrict(g, f))
    out["high_pass"] = ctx.to_global(g, ctx.high_pass(g, f))
    cfg3 = Config(continuation=False, beta_target=beta, precond="2linvh0", fixed_gn=2, fixed_pcg=3)
    s3 = Solver(ctx, dims, cfg3)
    s3.syn_images()
    vv3, rep3, _ = s3.register()
    out["solve2l"] = rep3
    out["v2l"] = ctx.to_global(g, vv3)
    s3.close()
    return out


def run_wide(ctx, dims, beta, scale=8.0):
    """Large displacements (nt=1, scale x v_syn): ghost widths beyond the slab
    width, i.e. multi-rank ("wide") halos, csrc/dist.cu halo_chunks."""
    cfg = Config(continuation=False, beta_target=beta, precond="inva", nt=1)
    s = Solver(ctx, dims, cfg)
    s.syn_images()
    g = s.grid
    v = (scale * ctx.syn_velocity(g)).contiguous()
    s.linearize(v, beta)
    J = s.objective()
    grad = s.gradient()
    vt = (-grad).contiguous()
    H = s.matvec(vt)
    ctx.set_deterministic(True)
    Hd = s.matvec(vt)
    ctx.set_deterministic(False)
    _, flags = ctx.characteristics(g, v, 3)
    out = {"J": J, "grad": ctx.to_global(g, grad), "H": ctx.to_global(g, H),
           "Hdet": ctx.to_global(g, Hd), "G": int(flags) >> 8}
    s.close()
    return out


def wide_main(n):
    ctx, rank, world, local = init_from_env()
    dims = (n, n, n)
    beta = 1e-3
    d = run_wide(ctx, dims, beta)
    ok = True
    if rank == 0:
        single = Context(local)
        r = run_wide(single, dims, beta)
        res = {"world": world, "grid": dims, "ghost_width": d["G"] - 1, "slab_width": n // world,
               "J_rel": abs(d["J"]["total"] / r["J"]["total"] - 1)}
        for k in ("grad", "H", "Hdet"):
            res[f"{k}_rel"] = rel(d[k], r[k].astype(np.float64))
        ok = (res["ghost_width"] > res["slab_width"] and res["J_rel"] < 1e-6 and
              res["grad_rel"] < 1e-5 and res["H_rel"] < 1e-5 and res["Hdet_rel"] == 0.0)
        res["ok"] = ok
        print(json.dumps(res), flush=True)
        single.close()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0) if world > 1 else None
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) else 1)


def VregGridC(g):
    from paper_2008_12820_b200 import VregGrid
    return VregGrid(g.n1 // 2, g.n2 // 2, g.n3 // 2, g.nt)


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))


def main():
    arg = sys.argv[1] if len(sys.argv) > 1 else "64"
    if len(sys.argv) > 2 and sys.argv[2] == "wide":
        return wide_main(int(arg))
    ctx, rank, world, local = init_from_env()
    if "," in arg:  # explicit grid, e.g. 48,40,36 (non power-of-two: cuFFT slab paths)
        dims = tuple(int(x) for x in arg.split(","))
    else:
        n = int(arg)
        dims = (n, n // 2 * 2 if n >= 16 else n, n)
    beta = 1e-3
    dist_out = run(ctx, dims, beta)
    ok = True
    res = {"world": world, "grid": dims}
    if rank == 0:
        single = Context(local)  # independent single-GPU context on the same device
        ref = run(single, dims, beta)
        res["J_rel"] = abs(dist_out["J"]["total"] / ref["J"]["total"] - 1)
        res["mismatch_rel"] = abs(dist_out["J"]["mismatch"] / ref["J"]["mismatch"] - 1)
        for k in ("m1", "grad", "H", "Hdet", "H_sl", "P", "v", "regop", "restrict", "high_pass",
                  "P2", "v2l"):
            if k in dist_out:
                res[f"{k}_rel"] = rel(dist_out[k], ref[k].astype(np.float64))
        ok = (res["m1_rel"] < 1e-6 and res["J_rel"] < 1e-6 and res["grad_rel"] < 1e-5 and
              res["H_rel"] < 1e-5 and res["P_rel"] < 1e-5 and res["P2_rel"] < 1e-4 and
              res["Hdet_rel"] == 0.0)
        if "solve" in dist_out:
            res["solve_mismatch_rel"] = abs(dist_out["solve"]["final_mismatch"] /
                                            ref["solve"]["final_mismatch"] - 1)
            res["solve2l_mismatch_rel"] = abs(dist_out["solve2l"]["final_mismatch"] /
                                              ref["solve2l"]["final_mismatch"] - 1)
            ok = ok and (res["H_sl_rel"] < 1e-5 and res["v_rel"] < 1e-4 and
                         res["solve_mismatch_rel"] < 1e-4 and res["restrict_rel"] < 1e-5 and
                         res["high_pass_rel"] < 1e-5 and res["v2l_rel"] < 1e-4 and
                         res["solve2l_mismatch_rel"] < 1e-4 and res["regop_rel"] == 0.0)
        res["ok"] = ok
        print(json.dumps(res), flush=True)
        single.close()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0) if world > 1 else None
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) else 1)


if __name__ == "__main__":
    main()
