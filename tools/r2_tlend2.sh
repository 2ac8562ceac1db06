#!/bin/bash
# fused two-level end v2 (loads first): quick parity + timing A/B + end-phase kernels
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_solver.py -x -q -k "precond or fixed" > gpurun_out/tlend2_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/tlend2_tests.log
for v in 0 1; do VREG_TL_END_3D=$v python tools/prof_precond.py 256 7 > gpurun_out/tlend2_pp_$v.log 2>&1; echo "tlend3d=$v $(tail -1 gpurun_out/tlend2_pp_$v.log | cut -c1-60)"; done
VREG_PCG_GRAPH=0 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/tlend2_pp_warm.csv python tools/prof_precond.py 256 1 > /dev/null 2>&1; echo ppn rc=$?
