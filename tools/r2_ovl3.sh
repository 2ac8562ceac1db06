#!/bin/bash
# regulariser placement: mode 3 (beside the inc pre-pass, joined before the steps) vs 2 and 1
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
for rep in 1 2; do for m in 2 3 1; do
  CUDA_VISIBLE_DEVICES=0 VREG_MATVEC_OVERLAP=$m python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/ovl3_m${m}_r$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/ovl3_m${m}_r$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); print('p1 mode $m rep $rep', round(d['ms_per_step'],4), round(d['roofline']['launch_us'],1))
"
done; done
for size in 256 512; do for m in 3 1; do
  VREG_MATVEC_OVERLAP=$m $R bench.py --gpus 2 --steps 10 --warmup 3 --size $size --no-cpu --no-registration --no-linear > gpurun_out/ovl3_p2_m${m}_s$size.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/ovl3_p2_m${m}_s$size.json'):
  if l.startswith('{'):
    d=json.loads(l); print('p2 s$size mode $m', round(d['ms_per_step'],4), round(d['value']))
"
done; done
