#!/bin/bash
# Targeted ncu metrics of one tcgen05 GEMM shape (tools/bench_gemm.py --only)
# for a given libesgd variant:  bash tools/ncu_gemm_metrics.sh <shape> [lib.so] [label]
shape=$1; lib=${2:-paper_1708_02983_b200/libesgd.so}; label=${3:-$(basename $lib .so)}
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,lts__t_bytes.sum.per_second,l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct
ESGD_LIB=$lib ncu --metrics $M --clock-control none -k regex:k_tc_gemm -s 3 -c 1 --csv \
  python tools/bench_gemm.py --only $shape 2>/dev/null | grep '"' | awk -F'","' -v L=$label '{gsub(/"/,"",$NF); print L, $(NF-2), $NF}'
