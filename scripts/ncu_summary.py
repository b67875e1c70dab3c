#!/usr/bin/env python3
"""Per-kernel summary of ncu --set full reports: duration, DRAM bytes (read +
write), the issue rate and the busiest pipes, occupancy, L2 hit rate.
  python scripts/ncu_summary.py gpurun_out/prof_*.ncu-rep [--csv out.csv]"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("dur_us", "gpu__time_duration.sum", 1e-3),
    ("dram_rd_MB", "dram__bytes_read.sum", 1e-6),
    ("dram_wr_MB", "dram__bytes_write.sum", 1e-6),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("fmaheavy_pct", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("alu_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("lsu_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("l1_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("l2_hit", "lts__t_sector_hit_rate.pct", 1),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("blocks_per_sm", "launch__occupancy_limit_registers", 1),
    ("grid", "launch__grid_size", 1),
    ("smem_KB", "launch__shared_mem_per_block_dynamic", 1e-3),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "Kbyte/block": 1e3, "byte/block": 1}


def rows_of(rep):
    if rep.endswith(".csv"):  # an exported `--page raw --csv`
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return []
    h, u = r[0], r[1]
    res = []
    for v in r[2:]:
        d = {"report": rep.split("/")[-1], "kernel": v[h.index("Kernel Name")].split("(")[0][:48]}
        for name, m, sc in METRICS:
            if m not in h:
                d[name] = None
                continue
            i = h.index(m)
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                d[name] = None
                continue
            x *= SCALE.get(u[i], 1)
            d[name] = round(x * sc, 2)
        res.append(d)
    return res


def main():
    args = sys.argv[1:]
    out_csv = None
    if "--csv" in args:
        i = args.index("--csv")
        out_csv = args[i + 1]
        del args[i:i + 2]
    allrows = [d for rep in args for d in rows_of(rep)]
    cols = ["report", "kernel"] + [m[0] for m in METRICS]
    print(" ".join(f"{c:>12s}" if c not in ("kernel", "report") else f"{c:24s}" for c in cols))
    for d in allrows:
        print(" ".join(f"{str(d[c]):>12s}" if c not in ("kernel", "report") else f"{str(d[c])[:24]:24s}" for c in cols))
    if out_csv:
        with open(out_csv, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=cols)
            w.writeheader()
            w.writerows(allrows)


if __name__ == "__main__":
    main()
