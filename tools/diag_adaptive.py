"""Diagnostic (round 2): adaptive default-config registration on the device vs
the compiled reference (register_images, optim.hpp:308-347) per level, and the
fixed 2 GN x 10 PCG InvA solve vs the SURVEY golden. Prints JSON lines."""
import json
import re
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402
from paper_2008_12820_b200 import Context  # noqa: E402
from paper_2008_12820_b200.solver import Config, Solver  # noqa: E402


def parse_levels(text):
    out = []
    for ln in text.splitlines():
        m = re.match(r"level (\d+) beta (\S+) pc (\S+) switched (\d) gn (\d+) pcg (\d+)", ln)
        if m:
            out.append(dict(beta=float(m.group(2)), pc=m.group(3), gn=int(m.group(5)),
                            pcg=int(m.group(6))))
        m = re.match(r"\s+mismatch (\S+) -> (\S+) g_rel (\S+)", ln)
        if m:
            out[-1].update(final_mismatch=float(m.group(2)), final_g_rel=float(m.group(3)))
    return out


def gnorm(x, n):
    return float(np.sqrt((np.asarray(x, dtype=np.float64) ** 2).sum() * (2 * np.pi / n) ** 3))


def main():
    ctx = Context(0)
    sizes = [int(a) for a in sys.argv[1:]] or [32, 64]
    for n in sizes:
        m0, _, m1 = ref.syn(n)
        t = time.time()
        vr, L, I = ref.register_levels(m0, m1, ref.Config())
        tr = time.time() - t
        s = Solver(ctx, n, Config())
        s.syn_images()
        t = time.time()
        v, rep, _ = s.register()
        t_dev = time.time() - t
        lv = parse_levels(s.report_text("report"))
        print(json.dumps(dict(n=n, ref_s=tr, dev_s=t_dev, ref_levels=[(l["gn_iters"], l["pcg_total"], l["final_mismatch"], l["final_g_rel"]) for l in L],
                              dev_levels=[(l["gn"], l["pcg"], l["final_mismatch"], l["final_g_rel"]) for l in lv],
                              ref_vnorm=gnorm(vr, n), dev_vnorm=gnorm(v.double().cpu().numpy(), n),
                              ref_iters=[(i["level"], i["pcg_iters"], i["alpha"], i["g_rel"]) for i in I])), flush=True)
        s.close()
    # fixed InvA 64^3 2x10 vs SURVEY golden (mismatch 6.7136229316e-3, ||v|| 3.7991080969)
    n = 64
    for pc in ("inva", "2linvh0"):
        for f64 in (True, False):
            s = Solver(ctx, n, Config(continuation=False, beta_target=1e-3, fixed_gn=2,
                                      fixed_pcg=10, precond=pc, pcg_fp64=f64))
            s.syn_images()
            t = time.time()
            v, rep, _ = s.register()
            print(json.dumps(dict(fixed=pc, pcg_fp64=f64, mismatch=rep["final_mismatch"],
                                  g_rel=rep["final_g_rel"], secs=time.time() - t,
                                  vnorm=gnorm(v.double().cpu().numpy(), n))), flush=True)
            s.close()
    ctx.close()


if __name__ == "__main__":
    main()
