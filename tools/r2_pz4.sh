#!/bin/bash
# multi-GPU A/B of the psi pre-zeroing (512^3 and 256^3 per GPU, p = 4 and 2) + NUMA-bound e2e A/B on one GPU
export PYTHONUNBUFFERED=1
for size in 512 256; do for N in 4 2; do for v in new base; do
  if [ $v = base ]; then L="$PWD/paper_2008_12820_b200/libvreg_b200_base.so"; else L=""; fi
  VREG_LIB_PATH=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N \
    bench.py --gpus $N --steps 10 --warmup 3 --size $size --no-cpu --no-registration --no-linear > gpurun_out/pz4_${v}_g${N}_s$size.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/pz4_${v}_g${N}_s$size.json'):
  if l.startswith('{'):
    d=json.loads(l); print('$v p$N s$size', round(d['ms_per_step'],3), round(d['value']))
"
done; done; done
for rep in 1 2; do for nb in 1 0; do
  CUDA_VISIBLE_DEVICES=0 VREG_BENCH_NUMA=$nb python bench.py --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/numa_${nb}_$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/numa_${nb}_$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); print('numa $nb rep $rep e2e', round(d['e2e']['value']), d['e2e'].get('host_cpus'))
"
done; done
