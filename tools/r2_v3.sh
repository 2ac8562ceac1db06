#!/bin/bash
# fused split-H0 body, row-wise prolong+high-pass, distributed two-level
# apply via InvA_f r + prolong(s_c - s_c0), DIST gather phase timers
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/v3_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/v3_tests.log
CUDA_VISIBLE_DEVICES=0 python tools/prof_precond.py 256 7 > gpurun_out/v3_pp.log 2>&1; echo pp rc=$?; tail -1 gpurun_out/v3_pp.log | cut -c1-80
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/v3_b1.json 2> gpurun_out/v3_b1.err; echo b1 rc=$?
$R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-linear > gpurun_out/v3_b2.json 2> gpurun_out/v3_b2.err; echo b2 rc=$?
CUDA_VISIBLE_DEVICES=0 VREG_PCG_GRAPH=0 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/v3_pp_warm.csv python tools/prof_precond.py 256 1 > gpurun_out/v3_pp_ncu.log 2>&1; echo ppn rc=$?
