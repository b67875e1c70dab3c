#!/bin/bash
# End-of-round check on one B200: GPU suite, smoke, default bench, reference arm.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_default.json")); r = json.load(open("gpurun_out/bench_ref.json"))
print("value", d["value"], "enc", d["encode_gbs"], "dec", d["decode_gbs"], "e2e", d["e2e"]["value"],
      "sweep", d["sweep"]["value"], "frac", d["roofline"]["frac"], d["roofline_encode"]["frac"],
      "launches", d["gpu_launches"], "clocks", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
print("reference", r["value"], "e2e ratio", round(d["e2e"]["value"] / r["value"], 1))
PY
