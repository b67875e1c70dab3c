#!/bin/bash
# Round measurement: default bench line, systematic line, every config, the ncu
# launch list of the default command and one --set full capture of the decode kernel.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python bench.py --codec systematic --steps 5 > gpurun_out/bench_sys.json 2> gpurun_out/bench_sys.err; echo "sys rc=$?"
./scripts/bench_all.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --stripes 8192 --no-cpu-baseline --e2e-stripes 0 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dec_fast_kernel -s 2 -c 1 -o gpurun_out/prof_dec \
    python bench.py --steps 1 --warmup 3 --stripes 8192 --no-cpu-baseline --e2e-stripes 0 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:enc_fast_kernel -s 2 -c 1 -o gpurun_out/prof_enc \
    python bench.py --steps 1 --warmup 3 --stripes 8192 --no-cpu-baseline --e2e-stripes 0 > gpurun_out/ncu_full_enc.log 2>&1; echo "full enc rc=$?"
for c in C3 C4; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$c.csv \
      python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --e2e-stripes 0 > gpurun_out/ncu_launch_$c.log 2>&1; echo "launch $c rc=$?"
done
