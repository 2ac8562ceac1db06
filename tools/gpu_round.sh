# One GPU round: tests, smoke, bench, launch list, full captures of the
# matvec's hot kernels (each ncu only after the same command exited 0).
set -x
python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_scatter_tile -c 1 -o gpurun_out/prof_scatter python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_f1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gather_tile -s 12 -c 1 -o gpurun_out/prof_gather python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_f2.log 2>&1
