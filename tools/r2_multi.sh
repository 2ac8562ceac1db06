#!/bin/bash
# multi-GPU validation + weak-scaling lines on the GPUs of this box
N=${1:-2}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_multi.py -m gpu -q 2>&1 | tail -15 > gpurun_out/multi_p${N}_tests.log
for size in 256 512; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --steps 10 --warmup 3 --size $size --no-cpu > gpurun_out/scale_g${N}_s${size}.json 2> gpurun_out/scale_g${N}_s${size}.err
done
python bench.py --gpus 1 --steps 10 --warmup 3 --size 512 --no-cpu --no-registration > gpurun_out/scale_g1_s512.json 2> gpurun_out/scale_g1_s512.err
cat gpurun_out/multi_p${N}_tests.log
for f in gpurun_out/scale_g*_s*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), round(d['value']), d.get('nvlink'), d.get('registration',{}).get('seconds'), d.get('precond_2linvh0',{}).get('ms_per_apply'))" 2>&1 | tail -1; done
