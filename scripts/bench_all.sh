#!/bin/bash
# One bench line per BASELINE config (C2 is the default headline workload).
set -e
mkdir -p gpurun_out
for c in C1 C2 C3 C4 C5; do
  g=""; [ "$c" = C1 ] && g="--graph"  # launch-bound: whole-step CUDA-graph replay
  python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 8 --sweep none $g > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err || { echo "$c failed"; tail -5 gpurun_out/bench_$c.err; }
  python - "$c" << 'PY'
import json, sys
c = sys.argv[1]
d = json.load(open(f"gpurun_out/bench_{c}.json"))
cb = d.get("cpu_baseline", {})
print(c, "value", d["value"], "enc", d["encode_gbs"], "dec", d["decode_gbs"], "plans_ms", d["phases_ms"]["plans"],
      "dec_frac", d["roofline"]["frac"], "enc_frac", d["roofline_encode"]["frac"], "e2e", d["e2e"]["value"],
      "cpu", cb.get("value"), "clocks", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
