#!/bin/bash
# u_{t+1} formed inside the inc-state pipe steps vs the precomputed u fields
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_parity256.py tests/test_gpu_solver.py tests/test_gpu_bspline.py -x -q > gpurun_out/incu_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/incu_tests.log
for rep in 1 2; do for v in 1 0; do
  VREG_INC_U=$v python bench.py --steps 20 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/incu_${v}_$rep.json 2> /dev/null
  python -c "
import json
for l in open('gpurun_out/incu_${v}_$rep.json'):
  if l.startswith('{'):
    d=json.loads(l); ks=d['kernel_share']; ms=d['ms_per_step']
    print('inc_u_in_pipe=$v rep $rep', round(ms,4), {k: round(x*ms*1e3,1) for k,x in ks.items()})
"
done; done
