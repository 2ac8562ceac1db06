"""2LInvH0 apply timing in a fresh process, apply by apply (diagnoses
first-process effects: JIT / plan creation / page mapping)."""
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
for m in range(3):
    s.matvec(r)
torch.cuda.synchronize()
for i in range(12):
    t0 = time.perf_counter()
    _, st = s.precond("2linvh0", r, 0.5)
    torch.cuda.synchronize()
    print(f"apply {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms inner {st['inner']}", flush=True)
ctx.enable_timers(True)
ctx.kernel_stats(reset=True)
s.precond("2linvh0", r, 0.5)
torch.cuda.synchronize()
ks = ctx.kernel_stats()
for k, v in sorted(ks.items(), key=lambda kv: -kv[1]["seconds"])[:12]:
    print(f"  {k:24s} {v['count']:6d} x {v['seconds']/v['count']*1e6:8.1f} us")
