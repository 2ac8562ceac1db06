#!/bin/bash
# multi-rank scatter boundary bands beside the interior sweep
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/v5_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/v5_tests.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/v5_b1.json 2> gpurun_out/v5_b1.err; echo b1 rc=$?
$R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-linear --no-registration > gpurun_out/v5_b2.json 2> gpurun_out/v5_b2.err; echo b2 rc=$?
for r in 16; do VREG_PIPE_RESERVE=$r $R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-linear --no-registration > gpurun_out/v5_b2_r$r.json 2> gpurun_out/v5_b2_r$r.err; echo b2 r=$r rc=$?; done
