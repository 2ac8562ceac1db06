#!/bin/bash
# multi-rank transpose sweep: 2 CTAs/SM at 128 registers (default build) vs 3 CTAs/SM at 80 registers with fallback-path spills
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
for rep in 1 2; do for v in default dist3cta; do
  if [ $v = default ]; then L=""; else L="$PWD/paper_2008_12820_b200/libvreg_b200_dist3cta.so"; fi
  for size in 256 512; do
    VREG_LIB_PATH=$L $R bench.py --gpus 2 --steps 10 --warmup 3 --size $size --no-cpu --no-registration --no-linear > gpurun_out/d3_${v}_s${size}_r$rep.json 2> /dev/null
    python -c "
import json
for l in open('gpurun_out/d3_${v}_s${size}_r$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); ms=d['ms_per_step']; ks=d['kernel_share']
    print('$v s$size rep $rep', round(ms,4), round(d['value']), 'scatter', round(ks['sl_scatter_sweep']*ms*1e3/4,1))
"
  done
done; done
