#!/bin/bash
# 512^3 per GPU after the regulariser-placement rule: multi-GPU tests, scaling at 2 and 4 GPUs
export NCCL_DEBUG=WARN
timeout 1800 python -m pytest tests/test_gpu_multi.py -m gpu -q > gpurun_out/multi_tests_4gpu.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/multi_tests_4gpu.log
for N in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N \
    bench.py --gpus $N --steps 10 --warmup 3 --size 512 --no-cpu > gpurun_out/scale_g${N}_s512.json 2> gpurun_out/scale_g${N}_s512.err
  echo "bench g$N rc=$?"
done
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 --size 512 --no-cpu > gpurun_out/scale_g1_s512.json 2> gpurun_out/scale_g1_s512.err
for f in gpurun_out/scale_g*_s512.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), round(d['value']), (d.get('nvlink') or {}).get('frac'), d.get('registration',{}).get('seconds'), d.get('precond_2linvh0',{}).get('ms_per_apply'))" 2>&1 | tail -1; done
