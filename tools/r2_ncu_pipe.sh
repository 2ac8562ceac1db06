#!/bin/bash
# ncu full capture of one inc-state step launch (pipe kernel) at 256^3
python bench.py --steps 1 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/ncu_plain.json 2> gpurun_out/ncu_plain.err && \
VREG_SERIAL_MATVEC=1 ncu --set full --clock-control none --import-source on -k regex:"${1:-k_gather_pipe}" -s ${2:-12} -c 1 -o gpurun_out/${3:-prof_pipe} python bench.py --steps 1 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/ncu_run.log 2>&1
echo ncu rc=$?
