#!/bin/bash
# multi-GPU: 512^3 p-independence + weak-scaling bench lines, hard timeouts
N=${1:-2}
export NCCL_DEBUG=WARN
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 tools/mgpu_check.py 512 > gpurun_out/mgpu512_p${N}.log 2>&1
echo "rc=$?" >> gpurun_out/mgpu512_p${N}.log
tail -3 gpurun_out/mgpu512_p${N}.log
for size in 256 512; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 \
    bench.py --gpus $N --steps 10 --warmup 3 --size $size --no-cpu > gpurun_out/scale_g${N}_s${size}.json 2> gpurun_out/scale_g${N}_s${size}.err
  echo "bench $size rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/scale_g${N}_s${size}.json')); print(round(d['ms_per_step'],3), round(d['value']), d.get('nvlink'), d.get('registration',{}).get('seconds'), d.get('precond_2linvh0',{}).get('ms_per_apply'))" 2>&1 | tail -2
done
