# Multi-GPU comparison of the round's collective paths (run with gpurun --gpus 4):
# NVLS split (default), NVLS single fused kernel, NCCL allreduce; dist_check at N=4.
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -q -s -p no:cacheprovider 2>&1 | grep -E "world=|PASS|FAIL|passed|failed"
for n in 2 4; do
  for v in 1 fused 0; do
    ESGD_NVLS=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29541 bench.py --gpus $n --steps 30 --warmup 5 --no-cpu 2>&1 | grep "^{" | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n=$n nvls=$v', d['value'], d['ms_per_step'], d['config']['collective'], d['e2e']['value'])"
  done
done
for v in 1 0; do
  ESGD_NVLS=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29561 tools/dist_check.py 2>&1 | grep -E "world=|DIST"
done
