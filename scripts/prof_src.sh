#!/bin/bash
# Per-source-line executed instructions of one kernel launch (ncu source page):
#   prof_src.sh <cfg> <stripes> <dec|enc> <kernel regex> <skip>
cfg=$1; S=$2; what=$3; rx=$4; skip=${5:-0}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k "regex:$rx" -s $skip -c 1 -o gpurun_out/src_$cfg python scripts/prof_kernel.py $cfg $S $what > gpurun_out/src_$cfg.log 2>&1
ncu -i gpurun_out/src_$cfg.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${cfg}_cuda.csv 2>&1
ncu -i gpurun_out/src_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${cfg}_sass.csv 2>&1
rm -f gpurun_out/src_$cfg.ncu-rep
