# Round ncu captures for profiles/ (run on the GPU box:
#   gpurun -- bash tools/capture_profiles.sh
# Reports are converted to CSV/text on the box (tools/ncu_capture.sh); only
# small files travel back. Each program first runs once without ncu.
set -x
bash tools/ncu_capture.sh r01_update k_sync_update update
bash tools/ncu_capture.sh r01_update_sum k_sync_update_sum update_sum
bash tools/ncu_capture.sh r01_tc_wgrad k_tc_gemm wgrad
bash tools/ncu_capture.sh r01_tc_dgrad k_tc_gemm dgrad
bash tools/ncu_capture.sh r01_tc_fwd k_tc_gemm fwd
cp /tmp/r01_update_sum.ncu-rep gpurun_out/ 2>/dev/null
# launch lists of the timed region only (NVTX range "timed" in bench.py)
for m in alexnet lenet; do
  python bench.py --model $m --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain_$m.log 2>&1 &&
  ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r01_launches_$m.csv python bench.py --model $m --steps 3 --warmup 3 --no-e2e --no-cpu \
      > gpurun_out/ncu_launch_$m.log 2>&1
done
ls -la gpurun_out
