#!/bin/bash
# On the GPU box: ncu --set full capture of one kernel, exported as the executed
# SASS mix + a few pipe metrics (the .ncu-rep itself stays on the box).
# ncu_mix_box.sh <tag> <kernel regex> <launch skip> <bench args...>
tag=$1; k=$2; s=$3; shift 3
mkdir -p gpurun_out /tmp/ncu
ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -f -o /tmp/ncu/$tag python bench.py "$@" --no-cpu-baseline --e2e-stripes 0 > /tmp/ncu/$tag.log 2>&1 || { echo "$tag ncu failed"; tail -5 /tmp/ncu/$tag.log; exit 1; }
ncu -i /tmp/ncu/$tag.ncu-rep --page source --csv --print-source sass > /tmp/ncu/$tag.src.csv 2>/dev/null
ncu -i /tmp/ncu/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
python scripts/sass_exec_mix.py /tmp/ncu/$tag.src.csv 1 40 > gpurun_out/${tag}_mix.txt
echo "$tag ok"
