#!/bin/bash
# Round-2 measurement on one B200: GPU test suite, the default bench line
# (C2 headline + nested C5 strong sweep), the reference arm, every config, the
# systematic line, and the ncu launch list of the default command.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --codec systematic --steps 5 --sweep none > gpurun_out/bench_sys.json 2> gpurun_out/bench_sys.err; echo "sys rc=$?"
./scripts/bench_all.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --stripes 8192 --no-cpu-baseline --e2e-stripes 0 --sweep none > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
