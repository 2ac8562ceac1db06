#!/bin/bash
# final-code weak scaling on one 4-GPU box (matvec lines only; registration/precond per N included)
export NCCL_DEBUG=WARN
for size in 256 512; do
  timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 --size $size --no-cpu > gpurun_out/scale_g1_s$size.json 2> gpurun_out/scale_g1_s$size.err
  for N in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N \
      bench.py --gpus $N --steps 10 --warmup 3 --size $size --no-cpu > gpurun_out/scale_g${N}_s$size.json 2> gpurun_out/scale_g${N}_s$size.err
  done
done
for f in gpurun_out/scale_g*_s*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), round(d['value']), (d.get('nvlink') or {}).get('frac'), d.get('registration',{}).get('seconds'), d.get('precond_2linvh0',{}).get('ms_per_apply'))" 2>&1 | tail -1; done
