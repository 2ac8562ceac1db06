#!/bin/bash
# transpose sweep with its input loads issued before the box zeroing vs the previous order
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_kernels.py -x -q > gpurun_out/scatpre_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/scatpre_tests.log
for rep in 1 2; do for v in new base; do
  if [ $v = base ]; then L="$PWD/paper_2008_12820_b200/libvreg_b200_base.so"; else L=""; fi
  VREG_LIB_PATH=$L VREG_MATVEC_OVERLAP=0 python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/scatpre_${v}_$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/scatpre_${v}_$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); ks=d['kernel_share']; ms=d['ms_per_step']
    print('$v serial rep $rep', round(ms,4), 'scatter/sweep', round(ks['sl_scatter_sweep']*ms*1e3/4,1))
"
  VREG_LIB_PATH=$L python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/scatpre_${v}_d$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/scatpre_${v}_d$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); print('$v default rep $rep', round(d['ms_per_step'],4))
"
done; done
