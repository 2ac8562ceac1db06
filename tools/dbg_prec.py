import sys, torch
sys.path.insert(0, ".")
from oracle import ref
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
import numpy as np
ctx = Context(0)
n = 32
m0, v, m1 = ref.syn(n)
s = Solver(ctx, n, Config(continuation=False, beta_target=1e-3))
s.syn_images()
s.linearize(torch.as_tensor(0.5 * v, dtype=torch.float32, device="cuda"), 1e-3)
g = s.gradient()
for kind in ("invh0", "2linvh0", "invh0"):
    try:
        out, st = s.precond(kind, (-g).contiguous(), 0.5)
        print(kind, "ok", st, float(out.norm()))
    except Exception as e:
        print(kind, "ERR", e)
