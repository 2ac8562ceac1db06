B="python bench.py --steps 10 --warmup 3 --no-registration --no-cpu --no-linear"
VREG_SERIAL_MATVEC=1 $B > gpurun_out/dg_base.json 2>/dev/null
cp paper_2008_12820_b200/libvreg_b200.so /tmp/lib_base.so
VREG_NVCC_EXTRA="-DVB_DIAG_NOBOX" python -m paper_2008_12820_b200.build --force > gpurun_out/dg_b1.log 2>&1
VREG_SERIAL_MATVEC=1 $B > gpurun_out/dg_nobox.json 2>/dev/null
VREG_NVCC_EXTRA="-DVB_DIAG_NOTAPS" python -m paper_2008_12820_b200.build --force > gpurun_out/dg_b2.log 2>&1
VREG_SERIAL_MATVEC=1 $B > gpurun_out/dg_notaps.json 2>/dev/null
VREG_NVCC_EXTRA="-DVB_DIAG_NOTAPS -DVB_DIAG_NOBOX" python -m paper_2008_12820_b200.build --force > gpurun_out/dg_b3.log 2>&1
VREG_SERIAL_MATVEC=1 $B > gpurun_out/dg_none.json 2>/dev/null
