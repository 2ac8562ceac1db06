"""Print ms/matvec and per-launch kernel times from bench JSON lines."""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ms = d["ms_per_step"]
    per = {k: round(v * ms * 1e3 / (4 if k in ("sl_inc_step", "sl_scatter_sweep") else 1))
           for k, v in d["kernel_share"].items()}
    print(f, round(ms, 3), per)
