ncu --set full --import-source on --clock-control none -k "regex:dec_[1-4]_kernel" -s 4 -c 4 -o gpurun_out/src4 python scripts/prof_kernel.py C4 32 dec > gpurun_out/src4.log 2>&1
ncu -i gpurun_out/src4.ncu-rep --page source --csv --print-source sass > gpurun_out/src4_sass.csv 2>&1
rm -f gpurun_out/src4.ncu-rep
