"""Device time of fd_grad / fd_div at 256^3 (kernel timers)."""
import sys
import torch
sys.path.insert(0, ".")

from paper_2008_12820_b200.engine import Context

ctx = Context(0)
g = ctx.grid(256)
f = torch.randn(256, 256, 256, device="cuda")
v = torch.randn(3, 256, 256, 256, device="cuda")
for _ in range(3):
    ctx.fd_grad(g, f), ctx.fd_div(g, v)
torch.cuda.synchronize()
ctx.enable_timers(True)
ctx.kernel_stats(reset=True)
for _ in range(10):
    ctx.fd_grad(g, f), ctx.fd_div(g, v)
torch.cuda.synchronize()
for k, s in ctx.kernel_stats().items():
    us = s["seconds"] / s["count"] * 1e6
    print(f"{k:10s} {us:8.1f} us  {16 * 256**3 / (us * 1e-6) / 1e9:7.0f} GB/s (16 B/voxel)")

# characteristics of 0.5 * SYN velocity (tile-staged RK2)
v = (0.5 * ctx.syn_velocity(g)).contiguous()
for _ in range(2):
    ctx.characteristics(g, v, 3)
torch.cuda.synchronize()
ctx.kernel_stats(reset=True)
for _ in range(5):
    ctx.characteristics(g, v, 3)
torch.cuda.synchronize()
for k, s in ctx.kernel_stats().items():
    if "char" in k:
        us = s["seconds"] / s["count"] * 1e6
        print(f"{k:20s} {us:8.1f} us  {36 * 256**3 / (us * 1e-6) / 1e9:7.0f} GB/s (36 B/voxel)")
