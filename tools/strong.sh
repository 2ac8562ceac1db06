# Strong scaling: the 512^3 matvec (cubic + trilinear) on 1, 2, 4 GPUs.
T=${1:-st}
python bench.py --grid 512,512,512 --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/${T}_g1.json 2> gpurun_out/${T}_g1.err
for G in 2 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 29541 \
    bench.py --gpus $G --grid 512,512,512 --steps 10 --warmup 3 --no-cpu --no-registration > gpurun_out/${T}_g${G}.json 2> gpurun_out/${T}_g${G}.err
done
