#!/bin/bash
# spill-free multi-rank transpose sweep (2 CTAs/SM) vs the 80-register build
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
$R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-linear --no-registration > gpurun_out/v6_b2.json 2> gpurun_out/v6_b2.err; echo b2 rc=$?
$R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-linear --no-registration --size 512 > gpurun_out/v6_b2_512.json 2> gpurun_out/v6_b2_512.err; echo b2_512 rc=$?
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/v6_multi.log 2>&1; echo multi rc=$?; tail -2 gpurun_out/v6_multi.log
