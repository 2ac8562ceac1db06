"""Pinned host <-> device copy bandwidth (one direction, and both at once)."""
import torch

n = 201326592 // 4
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, device="cuda")
d_b = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d_a.copy_(h_in, non_blocking=True)
    h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()


def timeit(fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


gb = n * 4 / 1e9
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timeit(fn)
    print(f"{name}: {ms:.3f} ms  {gb / (ms * 1e-3):.1f} GB/s per direction")
