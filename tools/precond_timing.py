"""Per-kernel device time of one 2LInvH0 apply at 256^3 (kernel timers on)."""
import time

import torch

from paper_2008_12820_b200.engine import Context
from paper_2008_12820_b200.solver import Config, Solver

ctx = Context(0)
s = Solver(ctx, 256, Config(continuation=False, beta_target=1e-3))
s.syn_images()
v = (0.5 * ctx.syn_velocity(s.grid)).contiguous()
s.linearize(v, 1e-3)
r = (-s.gradient()).contiguous()
s.precond("2linvh0", r, 0.5)
torch.cuda.synchronize()
ctx.enable_timers(True)
ctx.kernel_stats(reset=True)
t0 = time.perf_counter()
for _ in range(5):
    _, st = s.precond("2linvh0", r, 0.5)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
ks = ctx.kernel_stats()
tot = sum(v["seconds"] for v in ks.values()) / 5
print(f"wall {dt*1e3:.2f} ms/apply, timed kernels {tot*1e3:.2f} ms, inner {st['inner']}")
for k, v in sorted(ks.items(), key=lambda kv: -kv[1]["seconds"])[:14]:
    print(f"  {k:24s} {v['count']/5:6.1f} x {v['seconds']/v['count']*1e6:8.1f} us")
