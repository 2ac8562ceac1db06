#!/bin/bash
# 4-GPU box: multi-GPU parity tests (p = 2, 4) and weak-scaling lines
export NCCL_DEBUG=WARN
timeout 1800 python -m pytest tests/test_gpu_multi.py -m gpu -q > gpurun_out/multi_tests_4gpu.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/multi_tests_4gpu.log
for N in 4 2; do
for size in 256 512; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N \
    bench.py --gpus $N --steps 10 --warmup 3 --size $size --no-cpu > gpurun_out/scale_g${N}_s${size}.json 2> gpurun_out/scale_g${N}_s${size}.err
  echo "bench g$N s$size rc=$?"
done; done
for size in 256 512; do timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 --size $size --no-cpu > gpurun_out/scale_g1_s$size.json 2> gpurun_out/scale_g1_s$size.err; done
echo "bench g1 s512 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/mgpu_check.py 512 > gpurun_out/mgpu512_p4.log 2>&1
echo "mgpu512 p4 rc=$?"
for f in gpurun_out/scale_g*_s*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), round(d['value']), (d.get('nvlink') or {}).get('frac'), d.get('registration',{}).get('seconds'), d.get('precond_2linvh0',{}).get('ms_per_apply'))" 2>&1 | tail -1; done
