#!/bin/bash
# registration time: fused InvA vs the 3-D route (second-run regression check)
export PYTHONUNBUFFERED=1
for v in 0 1; do for rep in 1 2; do
  VREG_INVA_3D=$v python bench.py --steps 3 --warmup 3 --no-cpu --no-linear > gpurun_out/regab_${v}_${rep}.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/regab_${v}_${rep}.json'):
  if l.startswith('{'):
    d=json.loads(l); r=d['registration']; print('inva3d=$v rep $rep', round(r['seconds'],4), round(r['seconds_first_run'],4), {k: round(x,4) for k,x in r['phases_s'].items()})
"
done; done
