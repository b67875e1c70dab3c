"""Copy the latest scripts/measure_round.sh outputs from gpurun_out/ into
profiles/ (round-tagged) and regenerate BASELINE.md's results rows.
Usage: python scripts/update_profiles.py r01"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

shutil.copy(os.path.join(G, "bench_full.json"), os.path.join(P, f"{tag}_bench_c2_full.json"))
shutil.copy(os.path.join(G, "bench_sys.json"), os.path.join(P, f"{tag}_bench_c2_systematic.json"))
with open(os.path.join(P, f"{tag}_bench_configs.jsonl"), "w") as out:
    for c in ("C1", "C2", "C3", "C4", "C5"):
        out.write(open(os.path.join(G, f"bench_{c}.json")).read().strip() + "\n")
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_launches_c2_8192.csv"))
for rep, name in (("prof_dec", f"{tag}_ncu_full_raw.csv"), ("prof_enc", f"{tag}_ncu_full_enc_raw.csv")):
    raw = subprocess.run(["ncu", "-i", os.path.join(G, rep + ".ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    open(os.path.join(P, name), "w").write(raw)

rows = []
for line in open(os.path.join(P, f"{tag}_bench_configs.jsonl")):
    d = json.loads(line)
    c = d["config"]["workload"].split(":")[0]
    cb = d.get("cpu_baseline", {})
    graph = " (CUDA graph)" if d["config"].get("cuda_graph") else ""
    rows.append(f"| {c} | 1 | {d['encode_gbs']:.1f} | {100 * d['roofline_encode']['frac']:.1f} % | "
                f"{d['decode_gbs']:.1f} / {d['decode_with_plans_gbs']:.1f} | {100 * d['roofline']['frac']:.1f} % | "
                f"{d['phases_ms']['plans']:.2f} ms | {cb.get('encode_gbs', 0):.4f} / {cb.get('decode_gbs', 0):.4f} "
                f"({cb.get('cores')} threads, Path::Auto, AVX2) | yes{graph} |")
b = open(os.path.join(ROOT, "BASELINE.md")).read()
i = b.index("| C1 | 1 |")
j = b.index("\n\n", i)
open(os.path.join(ROOT, "BASELINE.md"), "w").write(b[:i] + "\n".join(rows) + b[j:])
for r in rows:
    print(r)
d = json.load(open(os.path.join(G, "bench_full.json")))
s = json.load(open(os.path.join(G, "bench_sys.json")))
print("C2", d["value"], d["encode_gbs"], d["decode_gbs"], d["e2e"]["value"], "sys", s["value"], s["encode_gbs"],
      s["decode_gbs"], "values:", [json.loads(l)["value"] for l in open(os.path.join(P, f"{tag}_bench_configs.jsonl"))])
