#!/bin/bash
# fused two-level end: parity tests, 2LInvH0 timing A/B
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests/test_gpu_solver.py tests/test_gpu_kernels.py tests/test_gpu_h2.py tests/test_gpu_parity256.py tests/test_gpu_switches.py -x -q > gpurun_out/tlend_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/tlend_tests.log
for v in 0 1; do VREG_TL_END_3D=$v python tools/prof_precond.py 256 7 > gpurun_out/tlend_pp_$v.log 2>&1; echo "tlend3d=$v $(tail -1 gpurun_out/tlend_pp_$v.log | cut -c1-60)"; done
VREG_PCG_GRAPH=0 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/tlend_pp_warm.csv python tools/prof_precond.py 256 1 > /dev/null 2>&1; echo ppn rc=$?
python bench.py --steps 10 --warmup 3 --no-cpu --no-linear > gpurun_out/tlend_b1.json 2> gpurun_out/tlend_b1.err; echo b1 rc=$?
