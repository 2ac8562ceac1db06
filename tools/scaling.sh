# Weak scaling of the matvec bench: 256^3 and 512^3 per GPU on 1, 2, 4 GPUs
# (one process per GPU over NCCL). Usage on a 4-GPU box: bash tools/scaling.sh <tag>
T=${1:-sc}
for S in 256 512; do
  python bench.py --size $S --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/${T}_${S}_g1.json 2> gpurun_out/${T}_${S}_g1.err
  for G in 2 4; do
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $G --size $S --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/${T}_${S}_g${G}.json 2> gpurun_out/${T}_${S}_g${G}.err
  done
done
