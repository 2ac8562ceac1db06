#!/bin/bash
# Round-2 evidence: launch list of the default bench command and full ncu
# captures of the dominant kernels (each after a plain run exited 0).
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
$B > gpurun_out/r2p_plain.json 2> gpurun_out/r2p_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2p_launches.csv $B > /dev/null 2>&1
echo launches rc=$?
cap() {  # name regex skip [env]
  env $4 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 -o gpurun_out/r2p_$1 $B > /dev/null 2>&1
  echo "$1 rc=$?"
}
cap gather_pipe k_gather_pipe 9
cap gather_pipe_serial k_gather_pipe 9 VREG_SERIAL_MATVEC=1
cap scatter k_scatter_tile_fp 0 VREG_SERIAL_MATVEC=1
cap fd k_fd_m 1
cap chars k_chars_tile 0
cap axis k_axis_d2 1 VREG_SERIAL_MATVEC=1
# shrink for the trip back (gpurun_out <= 64 MiB): raw CSV of every capture,
# keep only the dominant kernel's report
for f in gpurun_out/r2p_*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}.raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${f%.ncu-rep}.details.csv 2>/dev/null
done
ls -la gpurun_out/r2p_*.ncu-rep
for f in gpurun_out/r2p_*.ncu-rep; do case $f in *gather_pipe_serial*) ;; *) rm -f $f ;; esac; done
du -sh gpurun_out
