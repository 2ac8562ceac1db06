#!/bin/bash
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
$B > gpurun_out/r2p_plain.json 2> gpurun_out/r2p_plain.err || exit 1
VREG_SERIAL_MATVEC=1 ncu --set full --clock-control none --import-source on -k regex:k_gather_pipe -s 13 -c 1 -o gpurun_out/r2p_inc_step $B > /dev/null 2>&1
echo rc=$?
ncu -i gpurun_out/r2p_inc_step.ncu-rep --page raw --csv > gpurun_out/r2p_inc_step.raw.csv 2>/dev/null
ncu -i gpurun_out/r2p_inc_step.ncu-rep --page details --csv > gpurun_out/r2p_inc_step.details.csv 2>/dev/null
ncu -i gpurun_out/r2p_inc_step.ncu-rep --page source --csv --print-source sass > gpurun_out/r2p_inc_step.source.csv 2>/dev/null
du -sh gpurun_out
