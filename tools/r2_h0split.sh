#!/bin/bash
# split H0 inner solves + FastDiv spectral kernels: GPU tests, 2LInvH0 timing A/B, FD tile sweep, bench
export PYTHONUNBUFFERED=1
for v in 1 0; do VREG_H0_SPLIT=$v python tools/prof_precond.py 256 7 > gpurun_out/h0s_pp_$v.log 2>&1; echo "split=$v rc=$? $(tail -1 gpurun_out/h0s_pp_$v.log | cut -c1-60)"; done
for v in 0 1 2 3 4 5; do echo "fd variant $v"; VREG_FD_TILE=$v python tools/fd_timing.py 2>&1 | head -2; done > gpurun_out/h0s_fd.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h0s_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/h0s_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/h0s_bench.json 2> gpurun_out/h0s_bench.err; echo bench rc=$?
