"""Stand-alone preconditioner applies: inner iterations and rel-L2 vs the reference."""
import sys, torch, numpy as np
sys.path.insert(0, ".")
from oracle import ref
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ctx = Context(0)
m0, v, m1 = ref.syn(n)
for beta in (1e-3, 5e-4, 1e-2):
    s = Solver(ctx, n, Config(continuation=False, beta_target=beta))
    s.syn_images()
    s.linearize(torch.as_tensor(0.5 * v, dtype=torch.float32, device="cuda"), beta)
    r = ref.Session(m0, m1, 0.5 * v, beta, ref.Config(continuation=False, beta_target=beta))
    g = r.gradient()
    for kind in ("2linvh0", "invh0"):
        for eps in (0.5, 0.3, 0.1, 0.03):
            out, st = s.precond(kind, torch.as_tensor(-g, dtype=torch.float32, device="cuda"), eps)
            ro, rst = r.precond(kind, -g, eps)
            o = out.double().cpu().numpy()
            print(beta, kind, eps, "inner dev", st["inner"], "ref", rst["inner"],
                  "rel %.3e" % (np.linalg.norm(o - ro) / np.linalg.norm(ro)), flush=True)
    s.close()
