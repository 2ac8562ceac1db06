#!/bin/bash
# flat batched prolong+high-pass
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests/test_gpu_solver.py tests/test_gpu_parity256.py tests/test_gpu_h2.py tests/test_gpu_bspline.py -x -q > gpurun_out/v8_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/v8_tests.log
python tools/prof_precond.py 256 7 > gpurun_out/v8_pp.log 2>&1; echo pp rc=$?; tail -1 gpurun_out/v8_pp.log | cut -c1-80
VREG_PCG_GRAPH=0 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/v8_pp_warm.csv python tools/prof_precond.py 256 1 > gpurun_out/v8_pp_ncu.log 2>&1; echo ppn rc=$?
