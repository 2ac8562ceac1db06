"""Small end-to-end case for compute-sanitizer (memcheck / racecheck): every
kernel family of the hot path at 32^3 (and the pipe kernels at 64 x 32 x 32):
characteristics, gather / scatter sweeps (both tile and TMA-pipe paths), FD8,
spectral operators, the fused GN matvec, the three preconditioners and a
fixed-iteration registration (device Krylov, conditional graphs)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver

ctx = Context(0)
for dims, deg in (((32, 32, 32), 3), ((64, 32, 32), 3), ((32, 32, 32), 1), ((24, 20, 28), 3),
                  ((32, 32, 32), 4)):
    s = Solver(ctx, dims, Config(continuation=False, beta_target=1e-3, interp_degree=deg,
                                 fixed_gn=1, fixed_pcg=2))
    s.syn_images()
    v = (0.5 * ctx.syn_velocity(s.grid)).contiguous()
    s.linearize(v, 1e-3)
    g = s.gradient()
    H = s.matvec((-g).contiguous())
    for kind in ("inva", "invh0", "2linvh0"):
        if kind == "2linvh0" and any(n % 4 for n in dims):
            continue
        s.precond(kind, (-g).contiguous(), 0.5)
    s.register()
    torch.cuda.synchronize()
    print(dims, deg, "ok", float(H.norm()), flush=True)
    s.close()
ctx.close()
