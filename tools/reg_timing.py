"""Time two back-to-back registrations at 256^3 (reference defaults) with the
kernel timers on: cold (first) vs warm (second) run, per-phase and per-kernel."""
import sys
import time

import torch

from paper_2008_12820_b200.engine import Context
from paper_2008_12820_b200.solver import Config, Solver

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 256
ctx = Context(0)
timers = "--no-timers" not in sys.argv
ctx.enable_timers(timers)
for run in range(2):
    s = Solver(ctx, n, Config())
    s.syn_images()
    torch.cuda.synchronize()
    if timers:
        ctx.kernel_stats(reset=True)
    t0 = time.perf_counter()
    v, rep, cnt = s.register()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"run {run}: {dt:.3f} s", {k: round(rep[k], 3) for k in rep if k.startswith("t_")},
          "gn", rep["total_gn"], "pcg", rep["total_pcg"])
    if timers:
        ks = ctx.kernel_stats()
        top = sorted(ks.items(), key=lambda kv: -kv[1]["seconds"])[:12]
        print("   ", [(k, v["count"], round(v["seconds"] * 1e3, 1)) for k, v in top])
    s.close()
