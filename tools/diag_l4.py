"""Reproduce the level-4 first preconditioner apply stand-alone: the
reference's velocity after the beta = 1e-3 level, then beta = 5e-4."""
import sys, torch, numpy as np
sys.path.insert(0, ".")
from oracle import ref
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ctx = Context(0)
m0, _, m1 = ref.syn(n)
vL3, _, _ = ref.register_levels(m0, m1, ref.Config(beta_target=1e-3))
beta = 5e-4
r = ref.Session(m0, m1, vL3, beta, ref.Config(continuation=False, beta_target=beta))
g = r.gradient()
s = Solver(ctx, n, Config(continuation=False, beta_target=beta))
s.set_images(torch.as_tensor(m0, dtype=torch.float32, device="cuda"), torch.as_tensor(m1, dtype=torch.float32, device="cuda"))
s.linearize(torch.as_tensor(vL3, dtype=torch.float32, device="cuda"), beta)
gd = s.gradient().double().cpu().numpy()
print("grad rel", np.linalg.norm(gd - g) / np.linalg.norm(g))
for eps in (0.5, 0.4, 0.3, 0.2):
    for src, rr in (("refg", -g), ("devg", -gd)):
        out, st = s.precond("2linvh0", torch.as_tensor(rr, dtype=torch.float32, device="cuda"), eps)
        ro, rst = r.precond("2linvh0", rr, eps)
        o = out.double().cpu().numpy()
        print(eps, src, "inner dev", st["inner"], "ref", rst["inner"], "rel %.3e" % (np.linalg.norm(o - ro) / np.linalg.norm(ro)), flush=True)
