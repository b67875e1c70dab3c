mkdir -p gpurun_out
P="python scripts/prof_kernel.py"
for w in sysdec sysenc; do skip=1; [ $w = sysdec ] && skip=3
ncu --set full --clock-control none -k "regex:dec_fast_kernel" -s $skip -c 1 -o gpurun_out/prof_C2_$w $P C2 8192 $w > gpurun_out/prof_C2_$w.log 2>&1; echo "$w rc=$?"
ncu -i gpurun_out/prof_C2_$w.ncu-rep --page raw --csv > gpurun_out/prof_C2_${w}_raw.csv; rm -f gpurun_out/prof_C2_$w.ncu-rep
done
