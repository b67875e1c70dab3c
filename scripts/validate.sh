#!/bin/bash
# Full validation on one B200: the GPU suite, smoke(), the default bench line.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_default.json')); print(d['value'], d['encode_gbs'], d['decode_gbs'], d['e2e']['value'], d['sweep']['value'], d['cpu_baseline']['value'], d['clocks'])"
