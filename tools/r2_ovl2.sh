#!/bin/bash
# regulariser placement at p = 2 (256^3 and 512^3 per GPU)
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
for size in 256 512; do for m in 1 2; do
  VREG_MATVEC_OVERLAP=$m $R bench.py --gpus 2 --steps 10 --warmup 3 --size $size --no-cpu --no-registration --no-linear > gpurun_out/ovl2_m${m}_s$size.json 2> gpurun_out/ovl2_m${m}_s$size.err
  python -c "
import json
for l in open('gpurun_out/ovl2_m${m}_s$size.json'):
  if l.startswith('{'):
    d=json.loads(l); print('p2 s$size mode $m', round(d['ms_per_step'],4), round(d['value']))
"
done; done
