#!/bin/bash
# Multi-GPU bench lines (N = 2, 4 on one gpurun box): the default copy-engine
# center (ESGD_NVLS unset = ce), the multimem NVLS kernel (ESGD_NVLS=1) and
# NCCL (ESGD_NVLS=0); plus the N = 1 line. Summaries to stdout, logs in gpurun_out/.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['comm']; print('$1', d['n_gpus'], d['value'], d['ms_per_step'], 'exposed', round(c['fraction'],4), 'alone', c.get('alone'), 'e2e', (d.get('e2e') or {}).get('value'), d['clocks'])"; }
for N in ${NS:-2 4}; do
  [ $N -gt $(nvidia-smi -L | wc -l) ] && continue
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 295$N bench.py --gpus $N --steps 20 --warmup 5 --no-cpu > gpurun_out/b${N}_ce.log 2>&1; summ gpurun_out/b${N}_ce.log
  ESGD_NVLS=1 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 296$N bench.py --gpus $N --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/b${N}_nvls.log 2>&1; summ gpurun_out/b${N}_nvls.log
  ESGD_NVLS=0 timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 297$N bench.py --gpus $N --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/b${N}_nccl.log 2>&1; summ gpurun_out/b${N}_nccl.log
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/b1.log 2>&1; tail -1 gpurun_out/b1.log | cut -c1-200
