#!/bin/bash
# Round-2 final evidence on one GPU: all GPU tests, smoke, the default bench
# line, the bench launch list and full ncu captures of the dominant kernels
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv $B > /dev/null 2>&1
echo launches rc=$?
cap() {  # name regex skip cmd...
  local name=$1 re=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c 1 -o gpurun_out/fin_$name "$@" > /dev/null 2>&1
  echo "$name rc=$?"
}
cap gather_pipe k_gather_pipe 9 $B
cap scatter k_scatter_tile_fp 4 $B
P="python tools/prof_precond.py 256 1"
cap h0_step k_h0_step 4 env VREG_PCG_GRAPH=0 $P
cap prolong_hp k_prolong_plus_hp 1 env VREG_PCG_GRAPH=0 $P
for f in gpurun_out/fin_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${f%.ncu-rep}.details.csv 2>/dev/null
done
ls -la gpurun_out/fin_*.ncu-rep
for f in gpurun_out/fin_*.ncu-rep; do case $f in *gather_pipe*) ;; *) rm -f $f ;; esac; done
du -sh gpurun_out
