#!/bin/bash
# final multi-GPU check of the round-2 code: parity tests at p = 2 and 4 and the 512^3 check at p = 4
export NCCL_DEBUG=WARN
timeout 1800 python -m pytest tests/test_gpu_multi.py -m gpu -q > gpurun_out/multi_tests_4gpu_final.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/multi_tests_4gpu_final.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/mgpu_check.py 512 > gpurun_out/mgpu512_p4_final.log 2>&1
echo "mgpu512 p4 rc=$?"; tail -1 gpurun_out/mgpu512_p4_final.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N \
    bench.py --gpus $N --steps 10 --warmup 3 --size 256 --no-cpu > gpurun_out/scale_final_g${N}_s256.json 2> gpurun_out/scale_final_g${N}_s256.err
  echo "bench g$N rc=$?"
done
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 --size 256 --no-cpu > gpurun_out/scale_final_g1_s256.json 2> gpurun_out/scale_final_g1_s256.err
for f in gpurun_out/scale_final_g*_s256.json; do python -c "
import json; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), round(d['value']), d.get('registration',{}).get('seconds'), d.get('precond_2linvh0',{}).get('ms_per_apply'))" 2>&1 | tail -1; done
