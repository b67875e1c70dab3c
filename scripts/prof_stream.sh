export FNTRS_STREAM=1 FNTRS_STREAM_RD=8,4
ncu --set full --clock-control none -k regex:dec_stream -s 1 -c 1 -o gpurun_out/prof_stream_dec python scripts/prof_kernel.py C4 32 dec > gpurun_out/ps.log 2>&1
ncu -i gpurun_out/prof_stream_dec.ncu-rep --page raw --csv > gpurun_out/prof_stream_dec_raw.csv
ncu -i gpurun_out/prof_stream_dec.ncu-rep --page details --csv > gpurun_out/prof_stream_dec_details.csv
rm -f gpurun_out/prof_stream_dec.ncu-rep
