"""PCG residual histories: device solver vs compiled reference (default config)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import ref
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ctx = Context(0)
m0, _, m1 = ref.syn(n)
R = ref.register_residuals(m0, m1, ref.Config())
s = Solver(ctx, n, Config())
s.syn_images()
s.register()
rows = [ln.split(",") for ln in s.report_text("residuals").strip().splitlines()[1:]]
D = {(int(r[0]), int(r[2]), int(r[3])): float(r[4]) for r in rows}
Rd = {(int(a), int(b), int(c)): d for a, b, c, d in R}
for key in sorted(set(D) | set(Rd)):
    if key[0] >= 3:
        print(key, Rd.get(key), D.get(key))
