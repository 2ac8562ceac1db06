#!/bin/bash
# quick multi-GPU sanity: mgpu_check 64 under a hard timeout
N=${1:-2}
export NCCL_DEBUG=WARN
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/mgpu_check.py 64 > gpurun_out/mgq_${N}.log 2>&1
echo "rc=$?" >> gpurun_out/mgq_${N}.log
tail -30 gpurun_out/mgq_${N}.log
