# Round-1 ncu captures for profiles/ (run on the GPU box: gpurun -- bash tools/capture_profiles.sh).
# Reports are converted to CSV/text on the box; only the small update .ncu-rep travels back.
set -x
cap() { # name kernel-regex case
  python tools/ncu_case.py $3 && ncu --set full --import-source on --clock-control none -k regex:$2 -s 2 -c 1 -o /tmp/$1 python tools/ncu_case.py $3 > gpurun_out/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>&1
}
cap r01_update k_sync_update update
cap r01_tc_dgrad k_tc_gemm dgrad
cap r01_tc_wgrad k_tc_gemm wgrad
cp /tmp/r01_update.ncu-rep gpurun_out/
python bench.py --model lenet --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain34.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01_launches_lenet.csv python bench.py --model lenet --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu34d.log 2>&1
python bench.py --model alexnet --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain34e.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r01_launches_alexnet.csv python bench.py --model alexnet --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu34e.log 2>&1
du -sh gpurun_out; ls -la gpurun_out
echo done
