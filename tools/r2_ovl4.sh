#!/bin/bash
# regulariser placement at p = 4, 512^3 and 256^3 per GPU
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29547"
for size in 512 256; do for m in 1 2; do
  VREG_MATVEC_OVERLAP=$m $R bench.py --gpus 4 --steps 10 --warmup 3 --size $size --no-cpu --no-registration --no-linear > gpurun_out/ovl4_m${m}_s$size.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/ovl4_m${m}_s$size.json'):
  if l.startswith('{'):
    d=json.loads(l); print('p4 s$size mode $m', round(d['ms_per_step'],4), round(d['value']))
"
done; done
