#!/bin/bash
# transpose sweep at 2 CTAs/SM (96 registers, room for the regulariser's CTAs) vs 3 CTAs/SM
export PYTHONUNBUFFERED=1
for rep in 1 2; do for o in 3 2; do
  VREG_SCATTER_OCC=$o python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/occ_o${o}_r$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/occ_o${o}_r$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); ks=d['kernel_share']; ms=d['ms_per_step']
    print('occ $o rep $rep', round(ms,4), {k: round(v*ms*1e3,1) for k,v in ks.items()})
"
done; done
VREG_SCATTER_OCC=2 VREG_SERIAL_MATVEC=1 python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/occ_o2_serial.json 2> /dev/null
python -c "
import json
for l in open('gpurun_out/occ_o2_serial.json'):
  if l.startswith('{'):
    d=json.loads(l); ks=d['kernel_share']; ms=d['ms_per_step']
    print('occ 2 serial', round(ms,4), {k: round(v*ms*1e3,1) for k,v in ks.items()})
"
