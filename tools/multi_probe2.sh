# NVLS center-kernel grid size sweep at N=2 and N=4 (gpurun --gpus 4)
for n in 2 4; do
  for c in 8 16 32 64 148; do
    ESGD_NVLS_CTAS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29541 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu --no-e2e 2>&1 | grep "^{" | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=$n ctas=$c', d['value'], d['ms_per_step'], d['config']['collective'])"
  done
  ESGD_NVLS=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29541 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu --no-e2e 2>&1 | grep "^{" | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=$n nccl', d['value'], d['ms_per_step'], d['config']['collective'])"
done
