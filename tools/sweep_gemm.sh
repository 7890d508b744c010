#!/bin/bash
# Plan sweep of the tcgen05 GEMM on the AlexNet shapes: orientation x tile
# width x CTA pairs (tuning env knobs of csrc/gemm_tc.cu), one bench_gemm
# pass each; summarise with tools/sweep_gemm.py.
for sw in 0 1; do for bn in 128 192; do for pr in 0 1; do
  echo "CFG[ESGD_TC_SWAP=$sw ESGD_TC_BN=$bn ESGD_TC_PAIR=$pr]"
  ESGD_TC_SWAP=$sw ESGD_TC_BN=$bn ESGD_TC_PAIR=$pr timeout 150 python tools/bench_gemm.py 2>&1 | grep -v "^x\."
done; done; done
echo "CFG[]"; timeout 150 python tools/bench_gemm.py 2>&1 | grep -v "^x\."
