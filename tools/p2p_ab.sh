# A/B of the fused peer-memory SL sweeps (VREG_P2P_SL) on a 2- or 4-GPU box:
# parity (mgpu_check) and the matvec bench at 256^3 and 512^3 per GPU.
G=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29513"
VREG_P2P_SL=1 timeout 300 $R tools/mgpu_check.py 64 > gpurun_out/p2p_check.json 2> gpurun_out/p2p_check.err
echo "check rc=$?"
for S in 256 512; do
  for P in 0 1; do
    VREG_P2P_SL=$P timeout 300 $R bench.py --gpus $G --size $S --steps 10 --warmup 3 --no-cpu --no-registration \
      > gpurun_out/p2p_${S}_g${G}_p$P.json 2> gpurun_out/p2p_${S}_g${G}_p$P.err
    echo "bench $S p$P rc=$?"
  done
done
