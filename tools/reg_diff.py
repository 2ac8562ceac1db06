"""Diagnostics: per-kernel device time of two back-to-back 256^3
registrations (timers on), printed side by side."""
import time

import torch

from paper_2008_12820_b200.engine import Context
from paper_2008_12820_b200.solver import Config, Solver

ctx = Context(0)
ctx.enable_timers(True)
stats = []
for run in range(2):
    s = Solver(ctx, 256, Config())
    s.syn_images()
    torch.cuda.synchronize()
    ctx.kernel_stats(reset=True)
    t0 = time.perf_counter()
    _, rep, _ = s.register()
    torch.cuda.synchronize()
    print(f"run {run}: {time.perf_counter() - t0:.3f} s", {k: round(rep[k], 3) for k in rep if k.startswith("t_")})
    stats.append(ctx.kernel_stats())
    print("   tiles", ctx.tile_stats() if hasattr(ctx, "tile_stats") else None)
    s.close()
keys = sorted(set(stats[0]) | set(stats[1]), key=lambda k: -stats[1].get(k, {"seconds": 0})["seconds"])
for k in keys:
    a, b = stats[0].get(k, {"count": 0, "seconds": 0}), stats[1].get(k, {"count": 0, "seconds": 0})
    print(f"{k:24s} {a['count']:5d} {a['seconds']*1e3:9.2f} ms | {b['count']:5d} {b['seconds']*1e3:9.2f} ms")
