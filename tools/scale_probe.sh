# Weak-scaling lines of the default bench at N = 1, 2, 4 (gpurun --gpus 4);
# the NVLS and NCCL collective paths side by side at N > 1.
python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e 2>&1 | grep "^{" | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=1', d['value'], d['ms_per_step'])"
for n in 2 4; do
  for v in 1 0; do
    ESGD_NVLS=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29541 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu --no-e2e 2>&1 | grep "^{" | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=$n nvls=$v', d['value'], d['ms_per_step'], d['config']['collective'])"
  done
done
