#!/bin/bash
# final bench line and launch list (after the psi pre-zeroing)
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final6_smoke.log
python bench.py > gpurun_out/final6_bench.json 2> gpurun_out/final6_bench.err; echo bench rc=$?
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final6_launches.csv $B > /dev/null 2>&1
echo launches rc=$?
