#!/bin/bash
# Krylov chunks of 2048 elements; approximate reciprocal in the prolong+high-pass pass
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests/test_gpu_solver.py tests/test_gpu_parity256.py tests/test_gpu_h2.py tests/test_gpu_bspline.py tests/test_gpu_conformance.py -x -q > gpurun_out/v9_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/v9_tests.log
python tools/prof_precond.py 256 7 > gpurun_out/v9_pp.log 2>&1; echo pp rc=$?; tail -1 gpurun_out/v9_pp.log | cut -c1-80
python bench.py --steps 10 --warmup 3 --no-cpu --no-linear > gpurun_out/v9_b1.json 2> gpurun_out/v9_b1.err; echo b1 rc=$?
VREG_PCG_GRAPH=0 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/v9_pp_warm.csv python tools/prof_precond.py 256 1 > gpurun_out/v9_pp_ncu.log 2>&1; echo ppn rc=$?
