python -m pytest tests/test_gpu_kernels.py tests/test_gpu_matvec.py tests/test_gpu_solver.py -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-registration --no-cpu > gpurun_out/q.json 2>/dev/null
VREG_SERIAL_MATVEC=1 python bench.py --steps 10 --warmup 3 --no-registration --no-cpu > gpurun_out/qs.json 2>/dev/null
