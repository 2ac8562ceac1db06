#!/bin/bash
# registration at 512^3 per GPU, p = 2: regulariser placement 1 vs 2
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
for rep in 1 2; do for m in 1 2; do
  VREG_MATVEC_OVERLAP=$m $R bench.py --gpus 2 --steps 3 --warmup 3 --size 512 --no-cpu --no-linear > gpurun_out/regmode_m${m}_r$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/regmode_m${m}_r$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); r=d['registration']; print('mode $m rep $rep', round(d['ms_per_step'],3), round(r['seconds'],3), round(r['seconds_first_run'],3), {k: round(x,3) for k,x in r['phases_s'].items()})
"
done; done
