R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
$R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/mg_def.json 2> gpurun_out/mg_def.err
VREG_SERIAL_MATVEC=1 $R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/mg_ser.json 2> gpurun_out/mg_ser.err
VREG_SERIAL_MATVEC=1 VREG_HALO_OVERLAP=0 $R bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/mg_ser_nov.json 2> gpurun_out/mg_ser_nov.err
