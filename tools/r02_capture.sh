#!/bin/bash
# Round-2 evidence run on one B200: bench (+ reference arm), the timed
# region's ncu launch list, ncu --set full of the dominant kernels.
set -x
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.log 2>&1 || exit 1
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref.log 2>&1
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02_launches.csv 2> gpurun_out/r02_launches.err
for c in update_solo dgrad fwd; do
  python tools/ncu_case.py $c || exit 1
  kre=k_tc_gemm; [ $c = update_solo ] && kre=k_sync_update_solo4
  ncu --set full --import-source on --clock-control none -k regex:$kre -s 2 -c 1 -o /tmp/r02_$c python tools/ncu_case.py $c > gpurun_out/r02_ncu_$c.log 2>&1
  ncu -i /tmp/r02_$c.ncu-rep --page raw --csv > gpurun_out/r02_ncu_${c}_raw.csv 2>&1
  ncu -i /tmp/r02_$c.ncu-rep --page details > gpurun_out/r02_ncu_${c}_details.txt 2>&1
done
