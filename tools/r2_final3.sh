#!/bin/bash
# Round-2 final evidence (final code): GPU tests,
# smoke, the default bench line, its launch list, full ncu captures
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final3_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/final3_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final3_smoke.log
python bench.py > gpurun_out/final3_bench.json 2> gpurun_out/final3_bench.err; echo bench rc=$?
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final3_launches.csv $B > /dev/null 2>&1
echo launches rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gather_pipe<3, false, 2>" -s 5 -c 1 -o gpurun_out/fin3_inc_step $B > /dev/null 2>&1; echo inc rc=$?
ncu -i gpurun_out/fin3_inc_step.ncu-rep --page raw --csv > gpurun_out/fin3_inc_step.raw.csv 2>/dev/null
ncu -i gpurun_out/fin3_inc_step.ncu-rep --page details --csv > gpurun_out/fin3_inc_step.details.csv 2>/dev/null
du -sh gpurun_out
