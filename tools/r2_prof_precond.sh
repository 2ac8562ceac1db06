#!/bin/bash
python tools/prof_precond.py 256 3 > gpurun_out/pp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pp_launches.csv python tools/prof_precond.py 256 2 > gpurun_out/pp_ncu.log 2>&1
echo rc=$?
tail -2 gpurun_out/pp_plain.log
