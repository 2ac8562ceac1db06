"""2LInvH0 apply at 256^3 (bench linearisation): timing + a launch list under ncu."""
import sys, time, torch
sys.path.insert(0, ".")
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
ctx = Context(0)
s = Solver(ctx, n, Config(continuation=False, beta_target=1e-3))
s.syn_images()
s.linearize((0.5 * ctx.syn_velocity(s.grid)).contiguous(), 1e-3)
r = (-s.gradient()).contiguous()
for _ in range(3):
    s.precond("2linvh0", r, 0.5)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    t = time.perf_counter()
    _, st = s.precond("2linvh0", r, 0.5)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t) * 1e3)
print("2linvh0 ms", sorted(ts)[len(ts) // 2], ts, st)
