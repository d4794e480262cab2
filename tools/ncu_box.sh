#!/bin/bash
# ncu --set full of selected kernels on the GPU box, condensed to CSV files in gpurun_out/
#   tools/ncu_box.sh NAME KERNEL_REGEX COUNT -- command...
set -e
name=$1; regex=$2; count=$3; shift 4
mkdir -p /tmp/nc gpurun_out
ncu -f --set full --import-source on --clock-control none -k "regex:$regex" -c "$count" -o /tmp/nc/$name "$@" > gpurun_out/ncu_$name.log 2>&1
ncu -i /tmp/nc/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv
ncu -i /tmp/nc/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_src.csv 2>&1 || true
