#!/bin/bash
# ncu --set full captures of the dominant kernels of every config (one launch
# of each kernel after warm-up), on the current build. Reports land in
# gpurun_out/prof_<cfg>_<what>_raw.csv (raw page; the .ncu-rep only with KEEP_REP=1);
# summarise them with  python scripts/ncu_summary.py gpurun_out/prof_*_raw.csv
mkdir -p gpurun_out
P="python scripts/prof_kernel.py"
run() {  # name, stripes, what, kernel regex, count
  ncu --set full --clock-control none --import-source on -k "regex:$4" -s "${6:-0}" -c "$5" -o "gpurun_out/prof_$1_$3" \
      $P "$1" "$2" "$3" > "gpurun_out/prof_$1_$3.log" 2>&1; echo "prof $1 $3 rc=$?"
  ncu -i "gpurun_out/prof_$1_$3.ncu-rep" --page raw --csv > "gpurun_out/prof_$1_$3_raw.csv"
  [ -n "$KEEP_REP" ] || rm -f "gpurun_out/prof_$1_$3.ncu-rep"
}
run C4 32 dec "dec_[1-4]_kernel" 4 4   # skip the warm-up decode's 4 launches
run C4 32 enc "enc_[ab]_kernel" 2 2
run C3 1 dec "dec_[1-4]_kernel" 4 4
run C3 1 enc "enc_[ab]_kernel" 2 2
run C5 256 dec "dec_fast_kernel" 1 1
run C5 256 enc "enc_fast_kernel" 1 1
run C2 8192 dec "dec_fast_kernel" 1 1
run C2 8192 enc "enc_fast_kernel" 1 1
run C2 8192 sysdec "dec_fast_kernel" 1 3   # skip the two MODE 4 encodes and the first decode
run C2 8192 sysenc "dec_fast_kernel" 1 1   # the systematic encode is MODE 4 of the decode kernel
