#!/bin/bash
# where the matvec's regulariser branch runs: beside the inc steps (1), beside the transpose sweeps (2), serial (0)
export PYTHONUNBUFFERED=1
for rep in 1 2; do for m in 1 2 0; do
  VREG_MATVEC_OVERLAP=$m python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/ovl_m${m}_r$rep.json 2> gpurun_out/ovl_m${m}_r$rep.err
  python -c "
import json
for l in open('gpurun_out/ovl_m${m}_r$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); ks=d['kernel_share']; ms=d['ms_per_step']
    print('mode $m rep $rep', round(ms,4), round(d['roofline']['launch_us'],1), {k: round(v*ms*1e3,1) for k,v in ks.items()})
"
done; done
