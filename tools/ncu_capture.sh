#!/bin/bash
# ncu --set full capture of one kernel of a tools/ncu_case.py case, converted
# to CSV/text on the GPU box (the .ncu-rep stays in /tmp there):
#   bash tools/ncu_capture.sh <name> <kernel-regex> <case>
name=$1; kre=$2; case=$3
python tools/ncu_case.py $case || exit 1
ncu --set full --import-source on --clock-control none -k regex:$kre -s 2 -c 1 -o /tmp/$name python tools/ncu_case.py $case > gpurun_out/$name.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>&1
ncu -i /tmp/$name.ncu-rep --page details > gpurun_out/${name}_details.txt 2>&1
ncu -i /tmp/$name.ncu-rep --page source --csv > gpurun_out/${name}_source.csv 2>&1
