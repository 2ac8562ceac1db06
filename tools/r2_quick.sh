#!/bin/bash
# quick GPU iteration: SL parity tests + matvec bench (overlapped and serial)
set -x
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_matvec.py tests/test_gpu_solver.py -m gpu -x -q 2>&1 | tail -8
python bench.py --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
VREG_SERIAL_MATVEC=1 python bench.py --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/q_bench_serial.json 2>> gpurun_out/q_bench.err
VREG_SL_PIPE=0 VREG_SERIAL_MATVEC=1 python bench.py --steps 10 --warmup 3 --no-cpu --no-registration --no-linear > gpurun_out/q_bench_serial_nopipe.json 2>> gpurun_out/q_bench.err
python - <<'PY'
import json
for f in ("q_bench","q_bench_serial","q_bench_serial_nopipe"):
    try:
        d=json.load(open(f"gpurun_out/{f}.json"))
        print(f, round(d["ms_per_step"],3), d["value"], d["result_check"]["rel"], {k:v for k,v in d["timer_ms_per_step"].items()}, d["kernel_share"], d["roofline"]["launch_us"] if d.get("roofline") else None)
    except Exception as e: print(f, "ERR", e)
PY
tail -5 gpurun_out/q_bench.err
