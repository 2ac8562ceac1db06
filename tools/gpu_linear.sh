# Launch list + full ncu captures of the trilinear (degree 1) matvec's SL kernels.
B="python bench.py --degree 1 --steps 2 --warmup 3 --no-cpu --no-registration --no-linear"
$B > gpurun_out/lin_plain.json 2> gpurun_out/lin_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lin_launches.csv $B > gpurun_out/lin_ncu_l.log 2>&1
K="--set full --clock-control none --import-source on --kernel-name-base demangled"
$B > gpurun_out/lin_plain2.json 2>/dev/null && ncu $K -k "regex:k_gather_tile<.int.1, .bool.0, .int.2>" -s 2 -c 1 -o gpurun_out/lin_gather $B > gpurun_out/lin_ncu_f1.log 2>&1
$B > gpurun_out/lin_plain2.json 2>/dev/null && ncu $K -k "regex:k_scatter_tile_fp<.int.1" -s 2 -c 1 -o gpurun_out/lin_scatter $B > gpurun_out/lin_ncu_f2.log 2>&1
