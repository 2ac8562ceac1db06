#!/bin/bash
# transpose sweep: full ncu capture with source-level counters (where the sweep's time goes)
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
$B > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_scatter_tile_fp -s 4 -c 1 -o gpurun_out/scat_src $B > /dev/null 2>&1; echo cap rc=$?
ncu -i gpurun_out/scat_src.ncu-rep --page source --csv --print-source sass > gpurun_out/scat_src_sass.csv 2>/dev/null; echo src rc=$?
ncu -i gpurun_out/scat_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/scat_src_cuda.csv 2>/dev/null; echo srcc rc=$?
rm -f gpurun_out/scat_src.ncu-rep
ls -la gpurun_out/scat_src*
