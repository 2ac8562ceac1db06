#!/bin/bash
# p=2 matvec breakdown variants + 1-GPU 2LInvH0 launch list (eager PCG so ncu sees every kernel)
export PYTHONUNBUFFERED=1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
$R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/d2_def.json 2> gpurun_out/d2_def.err; echo def rc=$?
VREG_HALO_OVERLAP=0 $R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/d2_nov.json 2> gpurun_out/d2_nov.err; echo nov rc=$?
VREG_SERIAL_MATVEC=1 $R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/d2_ser.json 2> gpurun_out/d2_ser.err; echo ser rc=$?
export CUDA_VISIBLE_DEVICES=0
VREG_PCG_GRAPH=0 python tools/prof_precond.py 256 5 > gpurun_out/d2_pp_plain.log 2>&1; echo pp rc=$?
python tools/prof_precond.py 256 5 > gpurun_out/d2_pp_graph.log 2>&1; echo ppg rc=$?
VREG_PCG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d2_pp_launches.csv python tools/prof_precond.py 256 1 > gpurun_out/d2_pp_ncu.log 2>&1; echo ppn rc=$?
