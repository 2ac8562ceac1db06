#!/bin/bash
# psi slices zeroed by the inc-state pipeline steps (no memset per transpose sweep) vs before
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/prezero_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/prezero_tests.log
for rep in 1 2; do for v in new base; do
  if [ $v = base ]; then L="$PWD/paper_2008_12820_b200/libvreg_b200_base.so"; else L=""; fi
  CUDA_VISIBLE_DEVICES=0 VREG_LIB_PATH=$L python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/prezero_${v}_$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/prezero_${v}_$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); ks=d['kernel_share']; ms=d['ms_per_step']
    print('$v rep $rep', round(ms,4), {k: round(x*ms*1e3,1) for k,x in ks.items() if k.startswith('sl_')})
"
done; done
