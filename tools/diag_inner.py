"""Per-GN-iteration PCG and H0 inner iteration counts: device vs reference."""
import re, sys
sys.path.insert(0, ".")
from oracle import ref
from paper_2008_12820_b200 import Context
from paper_2008_12820_b200.solver import Config, Solver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ctx = Context(0)
m0, _, m1 = ref.syn(n)
_, L, I = ref.register_levels(m0, m1, ref.Config())
s = Solver(ctx, n, Config())
s.syn_images()
s.register()
dev = [(int(m.group(1)), int(m.group(2)), float(m.group(3)), float(m.group(4))) for m in
       re.finditer(r"  gn \d+ .*?g_rel (\S+) eps_k (\S+) .*? pcg (\d+) .*? h0_inner (\d+)", s.report_text("report"))
       for _ in [0]] if False else []
for ln in s.report_text("report").splitlines():
    m = re.match(r"\s+gn (\d+) .* g_rel (\S+) eps_k (\S+) alpha \S+ pcg (\d+) ls \d+ beta_pc \S+ h0_inner (\d+)", ln)
    if m:
        dev.append((int(m.group(4)), int(m.group(5)), float(m.group(2)), float(m.group(3))))
for r, d in zip(I, dev):
    print(int(r["level"]), "ref pcg", int(r["pcg_iters"]), "inner", int(r["h0_inner_iters"]),
          "g_rel %.6g" % r["g_rel"], "| dev pcg", d[0], "inner", d[1], "g_rel %.6g" % d[2])
