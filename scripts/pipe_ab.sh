#!/bin/bash
# Pipe utilisation of one decode launch per library build: pipe_ab.sh lib1.so lib2.so ...
M=smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,gpu__time_duration.sum,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fma.sum,launch__registers_per_thread
cp paper_0907_1788_b200/libfntrs_b200.so /tmp/cur.so
for lib in "$@"; do
  cp $lib paper_0907_1788_b200/libfntrs_b200.so
  echo "== $lib"
  ncu --metrics $M --clock-control none -k regex:${KERN:-dec_fast_kernel} -s 1 -c 1 python scripts/prof_kernel.py ${CFG:-C2} ${S:-2048} ${WHAT:-dec} 2>&1 | grep -E "^\s+(smsp|sm__|gpu__|launch)" 
done
cp /tmp/cur.so paper_0907_1788_b200/libfntrs_b200.so
