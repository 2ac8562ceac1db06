# Launch list + full ncu captures of the matvec's hot kernels for the current
# code, and the reference arm; each ncu only after the same command exited 0.
set -x
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_l.log 2>&1
K="--set full --clock-control none --import-source on --kernel-name-base demangled"
ncu $K -k "regex:k_gather_tile.*int.2>" -s 2 -c 1 -o gpurun_out/prof_gather $B > gpurun_out/ncu_f1.log 2>&1
ncu $K -k "regex:k_scatter_tile.*int.3" -s 2 -c 1 -o gpurun_out/prof_scatter $B > gpurun_out/ncu_f2.log 2>&1
ncu $K -k "regex:k_axis_d2.*int.2>" -s 1 -c 1 -o gpurun_out/prof_axis $B > gpurun_out/ncu_f3.log 2>&1
ncu $K -k "regex:k_assemble" -s 1 -c 1 -o gpurun_out/prof_assemble $B > gpurun_out/ncu_f4.log 2>&1
