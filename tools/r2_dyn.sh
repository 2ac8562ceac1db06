#!/bin/bash
# dynamic tile schedule of the gather pipe: tests (1 and 2 GPUs), p=2 bench with SM reserve
# variants, 1-GPU bench, warm-cache 2LInvH0 launch list, FD tile sweep
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/dyn_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/dyn_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/dyn_b1.json 2> gpurun_out/dyn_b1.err; echo b1 rc=$?
for r in 0 8; do VREG_PIPE_RESERVE=$r $R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/dyn_b2_r$r.json 2> gpurun_out/dyn_b2_r$r.err; echo b2 r=$r rc=$?; done
for v in 0 1 2 3 4 5; do echo "fd variant $v"; VREG_FD_TILE=$v python tools/fd_timing.py 2>&1 | head -2; done > gpurun_out/dyn_fd.log 2>&1
VREG_PCG_GRAPH=0 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/dyn_pp_warm.csv python tools/prof_precond.py 256 1 > gpurun_out/dyn_pp_ncu.log 2>&1; echo ppn rc=$?
