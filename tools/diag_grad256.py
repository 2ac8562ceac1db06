"""Where the 256^3 gradient error comes from: state, characteristics, gradient."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from oracle import ref
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = Context(0)
m0, v, m1 = ref.syn(n)
beta = 1e-3
r = ref.Session(m0, m1, 0.5 * v, beta, ref.Config(continuation=False, beta_target=beta))
s = Solver(ctx, n, Config(continuation=False, beta_target=beta))
dv = lambda a: torch.as_tensor(a, dtype=torch.float32, device="cuda")
s.set_images(dv(m0), dv(m1))
s.linearize(dv(0.5 * v), beta)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
J, Jr = s.objective(), r.objective()
print("J", J["mismatch"] / Jr["mismatch"] - 1, J["regularization"] / Jr["regularization"] - 1)
g = s.gradient().double().cpu().numpy()
gr = r.gradient()
print("grad rel", rel(g, gr), [rel(g[c], gr[c]) for c in range(3)])
# gradient at the SYN images the device builds itself
s2 = Solver(ctx, n, Config(continuation=False, beta_target=beta))
s2.syn_images()
s2.linearize(dv(0.5 * v), beta)
print("grad rel (device SYN images)", rel(s2.gradient().double().cpu().numpy(), gr))
m0d, m1d = s2.images()
print("m1 rel", rel(m1d.double().cpu().numpy(), m1))
