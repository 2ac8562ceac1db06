#!/bin/bash
# registration and 2LInvH0 timing with graph / eager Krylov loops (1 GPU, 256^3)
for mode in 1 0; do
  VREG_PCG_GRAPH=$mode python - <<'PY'
import os, sys, time, torch
sys.path.insert(0, ".")
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
ctx = Context(0)
n = 256
secs = []
for _ in range(2):
    s = Solver(ctx, n, Config())
    s.syn_images()
    torch.cuda.synchronize()
    t = time.perf_counter()
    v, rep, _ = s.register()
    torch.cuda.synchronize()
    secs.append(time.perf_counter() - t)
    s.close()
print("graph", os.environ["VREG_PCG_GRAPH"], "registration s", [round(x, 4) for x in secs], rep["total_gn"], rep["total_pcg"], "pc", round(rep["t_pc"], 4), "hess", round(rep["t_hess"], 4), "obj", round(rep["t_obj"], 4), "grad", round(rep["t_grad"], 4))
PY
  VREG_PCG_GRAPH=$mode python tools/prof_precond.py 256 7 2>&1 | tail -1
done
