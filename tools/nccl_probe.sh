# N=2 interference probe: NCCL algorithm/channels used by the round's allreduce
# and the step time under channel limits (run with gpurun --gpus 2)
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
          --master-port 29533 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --no-cpu 2>&1; }
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,COLL,TUNING run > gpurun_out/nccl_info.log
grep -E "NVLS|nvls|Channel|channels|algorithm|Algo|proto" gpurun_out/nccl_info.log | sort | uniq -c | sort -rn | head -30
grep "^{" gpurun_out/nccl_info.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['ms_per_step'])"
for c in 4 8 16; do
  NCCL_MAX_NCHANNELS=$c run | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('max_nchannels $c', d['ms_per_step'])"
done
NCCL_NVLS_ENABLE=0 run | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nvls off', d['ms_per_step'])"
