#!/usr/bin/env python3
"""Benchmark: batched non-systematic FNT Reed-Solomon codec over GF(65537).

Metric (BASELINE.json): encode & decode GB/s of source data per GPU, with the
HBM-roofline fraction. One STEP is one pass of the hot path over the whole
workload resident in HBM: build the decode plans of every erasure pattern,
encode every stripe, decode every stripe from its received packets.
value = source bytes of the workload (all ranks) / step time.

Default workload: configs[1] of BASELINE.json ("C2": n=256, k=128, 65536
stripes of 128 x 4 KiB source packets = 32 GiB of source per GPU), which is
the configuration the metric is quoted on and fits one B200. Multi-GPU runs
(torchrun, one rank per GPU) are weak scaling: every rank codes its own
stripes of the same shape (seeded per rank); no collective on the data path,
NCCL is used only for the barrier and the max-over-ranks of the step time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
  python bench.py --impl reference ...   # the reference's own CPU codec
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_0907_1788_b200 import workload as W  # noqa: E402
from paper_0907_1788_b200.sharding import max_over_ranks, rank_seed, rank_stripes, sum_over_ranks  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, only if MEASURED_PEAKS.json is absent


# Committed ncu --set full captures of the current build (scripts/prof_round2.sh,
# summarised by scripts/ncu_summary.py into profiles/r02_ncu_summary.csv): one
# launch of each kernel per config, with the codewords that launch coded.
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "r02_ncu_summary.csv")
PROFILE_CODEWORDS = {"C2": 8192 * 2048, "C3": 1 * 2048, "C4": 32 * 1024, "C5": 256 * 1024}


def kernel_label(cfg, what, systematic):
    """The kernel(s) behind one encode / decode call of this config."""
    E = cfg.n.bit_length() - 1 if cfg.n & (cfg.n - 1) == 0 else cfg.n.bit_length()
    if cfg.n <= 4096:
        if what == "decode":
            return (f"dec_fast_kernel<{E}> MODE 3 (fused systematic decode: one cyclic convolution, two transforms)"
                    if systematic else f"dec_fast_kernel<{E}> (fused decode: 3 transforms, one launch per call)")
        return f"enc_fast_kernel<{E}> (fused encode, one launch per call)"
    if what == "decode":
        return "dec_1..dec_4_kernel (four-step decode: 4 launches per 32-stripe batch; values summed over the four)"
    return "enc_a + enc_b_kernel (four-step encode: 2 launches per batch; values summed over the two)"


def _summary_rows(cfg, what):
    import csv
    try:
        rows = list(csv.DictReader(open(PROFILE_SUMMARY)))
    except Exception:
        return []
    short = {"decode": "dec", "encode": "enc"}.get(what, what)
    tag = f"prof_{cfg.name}_{short}_raw.csv"
    return [r for r in rows if r["report"] == tag]


def profiled(cfg, what, systematic, codewords):
    """Per-call DRAM traffic (read + write, scaled from the captured launch(es)
    to this call's codewords) and the issue / multiplier-pipe fractions
    (duration-weighted over the kernels of the call) from the committed capture."""
    if systematic:  # the fused systematic kernels (MODE 3 decode / MODE 4 encode), captured for C2
        if cfg.name != "C2":
            return {}
        what = "sysdec" if what == "decode" else "sysenc"
    rows = _summary_rows(cfg, what)
    if not rows or cfg.name not in PROFILE_CODEWORDS:
        return {}
    dur = sum(float(r["dur_us"]) for r in rows)
    tr = sum((float(r["dram_rd_MB"]) + float(r["dram_wr_MB"])) * 1e6 for r in rows)
    wavg = lambda k: round(sum(float(r[k]) * float(r["dur_us"]) for r in rows) / dur / 100.0, 4)
    return {"traffic": int(tr * codewords / PROFILE_CODEWORDS[cfg.name]),
            "traffic_source": f"ncu --set full dram__bytes_read.sum + dram__bytes_write.sum of "
                              f"{len(rows)} kernel launch(es) coding {PROFILE_CODEWORDS[cfg.name]} codewords, scaled to "
                              f"this call (profiles/r02_ncu_summary.csv, raw pages in profiles/r02_ncu/)",
            "issue_active_frac": wavg("issue_pct"), "multiplier_pipe_busy_frac": wavg("fmaheavy_pct"),
            "profiled_kernel_us": round(dur, 2)}


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def sample_now(self):
        """One synchronous query (timed regions shorter than the 100 ms poll)."""
        try:
            r = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            for line in r.stdout.splitlines():
                self.rows.append([x.strip() for x in line.split(",")])
        except Exception:
            pass

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------ CPU reference ----
def reference_lib():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import RefLib  # checker / baseline only
    if not RefLib.available():
        return None
    return RefLib()


SYSTEMATIC = False  # --codec systematic


PATHS = {"auto": 0, "fast": 1}  # codec::Path (proj/include/fntrs/codec.hpp:39)


def cpu_reference_sample(cfg, seed, stripes, threads, path="fast"):
    """Time the reference library (oracle/_ref, the unmodified reference codec)
    on `stripes` stripes of the config, the way the reference CLI runs it
    (per-codeword encode/decode_nonsystematic -- or the systematic pair with
    --codec systematic -- threads over codewords), decoding with codec::Path
    `path`: "auto" is the CLI's default (Lagrange when k <= 256,
    proj/src/codec.cpp:21-23), "fast" the O(n log n) interpolation.
    Returns (enc_s, dec_s, source_bytes)."""
    ref = reference_lib()
    if ref is None:
        raise RuntimeError("reference library oracle/_ref not built")
    from oracle_bind import gather_received
    ref.set_systematic(SYSTEMATIC)
    src = W.symbols(seed, 0, stripes * cfg.k * cfg.L).reshape(stripes, cfg.k, cfg.L)
    pats, sp = W.patterns(cfg, seed=seed, stripes=stripes)
    t0 = time.perf_counter()
    enc, esc = ref.encode_stripes(cfg.k, cfg.n, src, threads=threads)
    t1 = time.perf_counter()
    rx, rxe = gather_received(enc, esc, pats, sp)
    t2 = time.perf_counter()
    dec, _ = ref.decode_stripes(cfg.k, cfg.n, pats, sp, rx, rxe, path=PATHS[path], threads=threads)
    t3 = time.perf_counter()
    if not np.array_equal(dec, src):
        raise RuntimeError("reference decode mismatch")
    return t1 - t0, t3 - t2, src.nbytes


def pick_cpu_sample(cfg, threads, budget_s, path="fast"):
    """Stripes (and codewords) so the reference run takes ~budget_s."""
    # calibrate on one stripe
    e, d, b = cpu_reference_sample(cfg, W.SEED, 1, threads, path)
    per = max(e + d, 1e-4)
    return max(1, min(cfg.stripes, int(budget_s / per))), per


def cpu_info(ref=None):
    """Host CPU model, logical cores and whether the reference's AVX2 kernels
    run here (the same __builtin_cpu_supports("avx2") test as
    proj/src/transform.cpp:255-279)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            model = next((line.split(":", 1)[1].strip() for line in f if line.startswith("model name")), None)
    except Exception:
        pass
    avx2 = None
    if ref is None:
        ref = reference_lib()
    if ref is not None:
        avx2 = bool(ref.lib.ref_has_avx2())
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "avx2_path": avx2}


# ------------------------------------------------------------ GPU arm ----
def rank_layout(cfg, S, rank, world, scaling):
    """Stripe range [lo, hi), data seed, and the erasure patterns (with the
    stripe -> pattern map) that rank `rank` codes.
    weak: every rank codes S stripes of its own seeded data;
    strong: rank g codes stripes [g*S/G, (g+1)*S/G) of one global workload,
    with the patterns those stripes use."""
    lo, hi = rank_stripes(S, rank, world, scaling)
    seed = rank_seed(W.SEED, rank) if scaling == "weak" else W.SEED
    if lo == 0:
        pats, sp = W.patterns(cfg, seed=seed, stripes=hi - lo)
    else:  # strong scaling: this rank's slice of the global stripes and the patterns they use
        pats_all, sp_all = W.patterns(cfg, seed=seed, stripes=S)
        used, sp = np.unique(sp_all[lo:hi], return_inverse=True)
        pats, sp = pats_all[used], sp.astype(np.uint32)
    return lo, hi, seed, pats, sp



def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_0907_1788_b200 import Codec, _lib, default_escape_capacity

    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)
    cfg = W.CONFIGS[args.config]
    S = args.stripes or cfg.stripes
    lo, hi = rank_stripes(S, rank, world, args.scaling)
    S_rank = hi - lo
    seed = rank_seed(W.SEED, rank) if args.scaling == "weak" else W.SEED
    if S_rank == 0:
        raise SystemExit(f"rank {rank}: no stripes (S={S}, world={world})")
    k, n, L = cfg.k, cfg.n, cfg.L
    lib = _lib.load()
    codec = Codec(local_rank)
    stream = torch.cuda.current_stream(dev)
    chunk = max(1, min(S_rank, args.chunk))
    nchunks = (S_rank + chunk - 1) // chunk

    # ---- workload resident in HBM (untimed setup)
    src = torch.empty((S_rank, k, L), dtype=torch.int16, device=dev)
    st = lib.fntrs_gpu_fill_symbols(seed, lo * k * L, src.numel(), C.c_void_p(src.data_ptr()),
                                    C.c_void_p(stream.cuda_stream))
    assert st == 0
    enc = torch.empty((S_rank, n, L), dtype=torch.int16, device=dev)
    esc_cap = default_escape_capacity(chunk * n * L)
    enc_esc = [torch.empty(esc_cap, dtype=torch.int64, device=dev) for _ in range(nchunks)]
    enc_cnt = torch.zeros(nchunks, dtype=torch.int64, device=dev)
    dec_cap = default_escape_capacity(chunk * k * L)
    dec_esc = torch.empty(dec_cap, dtype=torch.int64, device=dev)
    dec_cnt = torch.zeros(nchunks, dtype=torch.int64, device=dev)
    dec = torch.empty((chunk, k, L), dtype=torch.int16, device=dev)

    def encode_chunk(c):
        a, b = c * chunk, min(S_rank, (c + 1) * chunk)
        codec.encode(k, n, src[a:b], out=enc[a:b], esc_out=enc_esc[c], esc_cap=esc_cap, count=enc_cnt[c:c + 1],
                     systematic=SYSTEMATIC)

    for c in range(nchunks):
        encode_chunk(c)
    _, _, _, pats, sp = rank_layout(cfg, S, rank, world, args.scaling)
    rx = torch.empty((S_rank, k, L), dtype=torch.int16, device=dev)
    rx_esc = []
    for c in range(nchunks):
        a, b = c * chunk, min(S_rank, (c + 1) * chunk)
        sub_sp = sp[a:b]
        r, e = W.received_packets(enc[a:b], enc_esc[c], enc_cnt[c:c + 1], pats, sub_sp, n)
        rx[a:b].copy_(r)
        del r
        rx_esc.append(e)
    sp_dev = torch.from_numpy(sp.astype(np.int32)).to(dev)
    pats_pinned = torch.from_numpy(pats.astype(np.int32)).pin_memory()
    torch.cuda.synchronize(dev)

    plans_box = {}

    def build_plans():
        if "p" in plans_box:
            plans_box["p"].close()
        plans_box["p"] = codec.plans(k, n, pats_pinned)

    dec_events = []

    def decode_chunk(c, timed=False):
        a, b = c * chunk, min(S_rank, (c + 1) * chunk)
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        codec.decode(plans_box["p"], sp_dev[a:b], rx[a:b], rx_esc[c], out=dec[: b - a], esc_out=dec_esc,
                     esc_cap=dec_cap, count=dec_cnt[c:c + 1], systematic=SYSTEMATIC)
        if timed:
            e1.record(stream)
            dec_events.append((e0, e1))

    enc_events = []

    def step(timed=False, verify=False):
        ok = True
        t = {}
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        build_plans()
        ev[1].record(stream)
        for c in range(nchunks):
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            encode_chunk(c)
            if timed:
                e1.record(stream)
                enc_events.append((e0, e1))
        ev[2].record(stream)
        for c in range(nchunks):
            decode_chunk(c, timed)
            if verify:
                a, b = c * chunk, min(S_rank, (c + 1) * chunk)
                bad = int((dec[: b - a] != src[a:b]).flatten(1).any(dim=1).sum().item())
                mismatched[0] += bad
                ok &= bad == 0
        ev[3].record(stream)
        return ok, ev

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (the first also verifies decode(encode(s)) == s on every stripe; the
    # per-rank mismatch counts are summed over ranks, NCCL, outside the timed region)
    mismatched = [0]
    for w in range(args.warmup):
        step(verify=(w == 0))
    torch.cuda.synchronize(dev)
    bad_all = sum_over_ranks([mismatched[0], S_rank], device=dev)
    if bad_all[0]:
        raise RuntimeError(f"decode(encode(s)) != s during warm-up on {bad_all[0]} stripes (all ranks)")
    verified = {"stripes_checked_all_ranks": bad_all[1], "mismatched_stripes_all_ranks": bad_all[0],
                "check": "decode(encode(s)) == s on every stripe, first warm-up step; counts summed over ranks"}

    graph = None
    if args.graph:
        # one whole step (plans, encode, decode, plan release) captured once and
        # replayed: every kernel re-executes, only the host launch work is gone.
        # Phase and per-launch times come from one eager step (below).
        def graph_step():
            p = codec.plans(k, n, pats_pinned)
            plans_box["p"] = p
            for c in range(nchunks):
                encode_chunk(c)
            for c in range(nchunks):
                decode_chunk(c)
            p.close()
            plans_box.pop("p", None)

        graph_step()  # eager once on this stream (allocations cached, tables built)
        torch.cuda.synchronize(dev)
        launches_c = codec.launches
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            graph_step()
        launches_per_step = codec.launches - launches_c
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize(dev)
        dec[:].zero_()
        graph.replay()
        torch.cuda.synchronize(dev)
        if not torch.equal(dec[: min(chunk, S_rank)], src[(nchunks - 1) * chunk:(nchunks - 1) * chunk + min(chunk, S_rank)]):
            raise RuntimeError("graph replay: decode(encode(s)) != s")
        step(timed=True)  # eager step: phases and per-launch times
        torch.cuda.synchronize(dev)
        eager_evs = [step(timed=True)[1]]

    # L2 policy: workloads whose bytes exceed twice the 126 MB L2 run back to
    # back; smaller ones get a 256 MiB write between steps (outside the timed
    # ranges, each step bracketed by its own events)
    work_bytes = S_rank * (2 * k * L + 2 * n * L)
    flush = work_bytes < 2 * 126 * 10**6
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    launches0 = codec.launches
    phase_ms = np.zeros(3)
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local_rank) as clocks:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        step_evs = []
        t_start.record(stream)
        evs = []
        for _ in range(args.steps):
            if flush:
                scrub.fill_(1)
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
            if graph is not None:
                graph.replay()
            else:
                _, ev = step(timed=True)
                evs.append(ev)
            if flush:
                b_.record(stream)
                step_evs.append((a_, b_))
        t_end.record(stream)
        if not clocks.rows:
            clocks.sample_now()  # still inside the timed region (kernels queued)
        torch.cuda.synchronize(dev)
    barrier()
    gpu_launches = codec.launches - launches0
    if graph is not None:
        gpu_launches = launches_per_step * args.steps
        evs = eager_evs
    total_ms = sum(a_.elapsed_time(b_) for a_, b_ in step_evs) if flush else t_start.elapsed_time(t_end)
    for ev in evs:
        phase_ms += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])]
    phase_ms /= len(evs)
    dec_launch_ms = float(np.mean([a.elapsed_time(b) for a, b in dec_events]))
    enc_launch_ms = float(np.mean([a.elapsed_time(b) for a, b in enc_events]))
    mx = max_over_ranks([total_ms, *phase_ms, dec_launch_ms, enc_launch_ms], device=dev)
    total_ms, phase_ms, dec_launch_ms, enc_launch_ms = mx[0], np.array(mx[1:4]), mx[4], mx[5]

    ms_per_step = total_ms / args.steps
    src_bytes_rank = 2 * k * L * S_rank
    src_bytes_all = src_bytes_rank * (world if args.scaling == "weak" else 1)
    if args.scaling == "strong":
        src_bytes_all = 2 * k * L * S
    value = src_bytes_all / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant kernel (decode), per launch = one chunk
    peak, peak_src = hbm_peak()
    rows = chunk
    dec_bytes = 2 * (2 * k * L * rows)          # read 2k + write 2k per codeword
    enc_bytes = 2 * k * L * rows + 2 * n * L * rows  # read 2k + write 2n
    dec_achieved = dec_bytes / (dec_launch_ms * 1e-3) / 1e9
    enc_achieved = enc_bytes / (enc_launch_ms * 1e-3) / 1e9
    dec_prof = profiled(cfg, "decode", SYSTEMATIC, rows * L)
    enc_prof = profiled(cfg, "encode", SYSTEMATIC, rows * L)
    if args.traffic is not None:
        dec_prof["traffic"], dec_prof["traffic_source"] = args.traffic, "--traffic"
    for pr, alg in ((dec_prof, dec_bytes), (enc_prof, enc_bytes)):
        if pr.get("traffic"):
            pr["traffic_over_algorithmic"] = round(pr["traffic"] / alg, 3)
    result = {
        "metric": "encode & decode GB/s of source data per GPU (1/2/4/8 B200), % of HBM roofline",
        "codec": "systematic" if SYSTEMATIC else "non-systematic",
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": "u32 (GF(65537) in 32-bit lanes; uint16 packets)",
        "data": "synthetic (seeded splitmix64 uint16 source, seeded erasure patterns per BASELINE config)",
        "config": {
            "workload": f"{cfg.name}: n={n} k={k} L={L} stripes/GPU={S_rank} patterns/GPU={len(pats)} "
                        f"({cfg.pattern}); step = plans + encode + decode of all stripes",
            "n": n, "k": k, "L": L, "stripes_per_gpu": S_rank, "source_bytes_per_gpu": src_bytes_rank,
            "chunk_stripes": chunk,
            "l2_policy": ("L2 flushed between timed steps (256 MiB write outside per-step events): working set %.1f MB"
                          % (work_bytes / 1e6)) if flush else
                         ("inputs (%.1f GiB/GPU) far larger than L2, steps back to back" % (src_bytes_rank / 2**30)),
            "cuda_graph": bool(args.graph),
            "parallelism": f"stripes{'/rank' if args.scaling == 'weak' else ' sharded'} x {world} GPU",
        },
        "phases_ms": {"plans": round(float(phase_ms[0]), 3), "encode": round(float(phase_ms[1]), 3),
                      "decode": round(float(phase_ms[2]), 3)},
        "encode_gbs": round(src_bytes_rank / (phase_ms[1] * 1e-3) / 1e9, 2),
        "decode_gbs": round(src_bytes_rank / (phase_ms[2] * 1e-3) / 1e9, 2),
        "decode_with_plans_gbs": round(src_bytes_rank / ((phase_ms[2] + phase_ms[0]) * 1e-3) / 1e9, 2),
        "roofline": dict({
            "bound": "hbm",
            "kernel": kernel_label(cfg, "decode", SYSTEMATIC),
            "achieved": round(dec_achieved, 2), "peak": peak, "peak_source": peak_src, "unit": "GB/s",
            "frac": round(dec_achieved / peak, 4),
            "algorithmic_bytes_per_launch": dec_bytes, "avg_launch_ms": round(dec_launch_ms, 4),
            "per_unit": "read 2k + write 2k bytes per codeword (SURVEY 8(d)); a launch = one decode call of "
                        f"{rows} stripes x {L} codewords",
        }, **dec_prof),
        "roofline_encode": dict({
            "bound": "hbm", "kernel": kernel_label(cfg, "encode", SYSTEMATIC), "achieved": round(enc_achieved, 2),
            "peak": peak, "unit": "GB/s", "frac": round(enc_achieved / peak, 4),
            "algorithmic_bytes_per_launch": enc_bytes, "avg_launch_ms": round(enc_launch_ms, 4),
            "per_unit": "read 2k + write 2n bytes per codeword",
        }, **enc_prof),
        "gpu_launches": int(gpu_launches),
        "verified": verified,
        "clocks": clocks.summary(),
    }
    del rx, enc
    torch.cuda.empty_cache()
    if args.e2e_stripes:
        result["e2e"] = run_e2e(args, codec, cfg, dev, stream, seed, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds)
    return result


def run_e2e(args, codec, cfg, dev, stream, seed, world):
    """Same metric through the public API with pinned HOST buffers
    (paper_0907_1788_b200.pipeline.HostPipeline over the Codec / C-ABI calls):
    every step copies the source and the received packets (and their escape
    list) host->device and the encoded and decoded packets (and escape lists)
    device->host inside the timed region; chunks overlap H2D, kernels and D2H
    on three streams."""
    import torch
    from paper_0907_1788_b200.pipeline import HostPipeline, escape_ranges
    k, n, L = cfg.k, cfg.n, cfg.L
    S = min(args.e2e_stripes, cfg.stripes, pinned_budget_stripes(cfg, world))
    chunk = max(1, min(S, args.e2e_chunk))
    src_h = torch.from_numpy(W.symbols(seed + 7, 0, S * k * L).view(np.int16).reshape(S, k, L)).pin_memory()
    pats, sp = W.patterns(cfg, seed=seed + 7, stripes=S)
    pats_h = torch.from_numpy(pats.astype(np.int32)).pin_memory()
    # received packets prepared once (the erasure channel, not the codec)
    d_src = src_h.to(dev)
    enc0, e0, c0 = codec.encode(k, n, d_src, systematic=SYSTEMATIC)
    rx0, rxe0 = W.received_packets(enc0, e0, c0, pats, sp, n)
    rx_h = rx0.cpu().pin_memory()
    rxe_np = rxe0.cpu().numpy().view(np.uint64) if rxe0 is not None else np.zeros(0, np.uint64)
    rxe_h = torch.from_numpy(rxe_np.view(np.int64)).pin_memory() if rxe_np.size else None
    del enc0, rx0, d_src
    nch = (S + chunk - 1) // chunk
    ranges = escape_ranges(rxe_np, S, chunk, k, L)
    pipe = HostPipeline(codec, k, n, L, chunk, nstreams=args.e2e_streams, systematic=SYSTEMATIC)
    enc_h = torch.empty((S, n, L), dtype=torch.int16).pin_memory()
    dec_h = torch.empty((S, k, L), dtype=torch.int16).pin_memory()
    enc_esc_h = torch.empty((nch, pipe.cap_e), dtype=torch.int64).pin_memory()
    dec_esc_h = torch.empty((nch, pipe.cap_e), dtype=torch.int64).pin_memory()
    cnt_h = torch.zeros(2 * nch, dtype=torch.int64).pin_memory()
    sp_d = torch.from_numpy(sp.astype(np.int32)).to(dev)
    h2d = src_h.numel() * 2 + rx_h.numel() * 2 + (rxe_h.numel() * 8 if rxe_h is not None else 0) + pats_h.numel() * 4
    d2h = enc_h.numel() * 2 + dec_h.numel() * 2 + enc_esc_h.numel() * 8 + dec_esc_h.numel() * 8 + cnt_h.numel() * 8

    def step():
        rxe_d = rxe_h.to(dev, non_blocking=True) if rxe_h is not None else None
        plans = codec.plans(k, n, pats_h)
        if args.e2e_sequential:
            pipe.encode_host(src_h, enc_h, enc_esc_h, cnt_h[:nch])
            pipe.decode_host(plans, sp_d, rx_h, rxe_d, dec_h, dec_esc_h, cnt_h[nch:], ranges)
        else:  # encode and decode chunks interleaved: both copy engines busy
            pipe.code_host(src_h, enc_h, enc_esc_h, cnt_h[:nch], plans, sp_d, rx_h, rxe_d, dec_h, dec_esc_h,
                           cnt_h[nch:], ranges)
        pipe.join()
        return plans

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    assert torch.equal(dec_h, src_h), "e2e decode mismatch"
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(1, args.steps)
    keep = []
    a.record(stream)
    for _ in range(steps):
        keep.append(step())
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = max_over_ranks([a.elapsed_time(b) / steps], device=dev)[0]
    total_src = 2 * k * L * S * world
    link = pcie_peaks(dev)
    return {"value": round(total_src / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3),
            # the e2e bound: PCIe, both directions busy at once (per GPU)
            "pcie_h2d_gbs": round(h2d / (ms * 1e-3) / 1e9, 2), "pcie_d2h_gbs": round(d2h / (ms * 1e-3) / 1e9, 2),
            "pcie_peak_h2d_gbs": link[0], "pcie_peak_d2h_gbs": link[1],
            "sample": f"{S} stripes/GPU of {cfg.name} from pinned host memory via HostPipeline "
                      f"(Codec.encode/plans/decode C-ABI calls, {chunk}-stripe chunks on {args.e2e_streams} streams, "
                      f"{'encode then decode' if args.e2e_sequential else 'encode and decode chunks interleaved'})"}


def pinned_budget_stripes(cfg, world):
    """e2e sample size the host can pin: all ranks together use at most a quarter
    of MemAvailable (source, received, encoded and decoded packets per stripe)."""
    try:
        with open("/proc/meminfo") as f:
            avail = next(int(line.split()[1]) * 1024 for line in f if line.startswith("MemAvailable"))
    except Exception:
        return 1 << 30
    per_stripe = (3 * cfg.k + cfg.n) * cfg.L * 2
    return max(64, int(avail / 4 / max(1, world) / per_stripe))


def pcie_peaks(dev, nbytes=512 << 20):
    """Pinned-host copy bandwidth of this GPU's link, each direction alone (GB/s)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = []
    for fn in (lambda: d.copy_(h, non_blocking=True), lambda: h.copy_(d, non_blocking=True)):
        fn()
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            fn()
        b.record()
        torch.cuda.synchronize(dev)
        out.append(round(3 * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9, 2))
    del h, d
    return out


def cpu_baseline(cfg, budget_s):
    """The unmodified reference library on all host cores: Path::Fast (the
    faster decode, the value) and Path::Auto (the CLI default) on bounded
    samples of the workload."""
    threads = os.cpu_count() or 1
    out = {}
    try:
        for path in ("fast", "auto"):
            stripes, per = pick_cpu_sample(cfg, threads, budget_s / 2, path)
            e, d, b = cpu_reference_sample(cfg, W.SEED + 99, stripes, threads, path)
            out[path] = {"value": round(b / (e + d) / 1e9, 6), "encode_gbs": round(b / e / 1e9, 6),
                         "decode_gbs": round(b / d / 1e9, 6), "stripes": stripes}
    except Exception as ex:  # reported, never fatal for the GPU arm
        return {"value": None, "error": str(ex)[:200], **out}
    info = cpu_info()
    f = out["fast"]
    return {"value": f["value"], "unit": "GB/s", "cores": threads, "kind": "reference",
            "encode_gbs": f["encode_gbs"], "decode_gbs": f["decode_gbs"], "path": "fast",
            "paths": out, **info,
            "sample": f"{f['stripes']} stripes of {cfg.name} (encode + Path::Fast decode incl. plan build; "
                      f"Path::Auto on {out['auto']['stripes']} stripes under 'paths'), {threads} threads over "
                      f"codewords, oracle/_ref = unmodified reference library, "
                      f"AVX2 kernels {'active' if info['avx2_path'] else 'inactive'}"}


# ----------------------------------------------------- reference arm ----
def run_reference(args, rank, world):
    if rank != 0:
        return None
    cfg = W.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    ref = reference_lib()
    if ref is None:
        return {"impl": "reference", "unavailable": "reference library (oracle/_ref) not built"}
    path = args.ref_path
    stripes, per = pick_cpu_sample(cfg, threads, args.ref_step_seconds, path)
    times = []
    for i in range(args.warmup + args.steps):
        e, d, b = cpu_reference_sample(cfg, W.SEED + i, stripes, threads, path)
        if i >= args.warmup:
            times.append(e + d)
    ms = 1e3 * float(np.mean(times))
    value = 2 * cfg.k * cfg.L * stripes / (ms * 1e-3) / 1e9
    other = "auto" if path == "fast" else "fast"
    o_stripes, _ = pick_cpu_sample(cfg, threads, args.ref_step_seconds / 2, other)
    oe, od, ob = cpu_reference_sample(cfg, W.SEED + 99, o_stripes, threads, other)
    info = cpu_info(ref)
    return {
        "impl": "reference",
        "metric": "encode & decode GB/s of source data per GPU (1/2/4/8 B200), % of HBM roofline",
        "codec": "systematic" if SYSTEMATIC else "non-systematic",
        "value": round(value, 6), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "u32 (GF(65537))", "data": "synthetic (same generator and erasure classes)",
        "config": {"workload": f"{cfg.name}: n={cfg.n} k={cfg.k} L={cfg.L}; step = encode + decode "
                               f"(incl. plan build) of a {stripes}-stripe sample", "stripes_per_step": stripes,
                   "decode_path": path},
        "cpu_baseline": {"value": round(value, 6), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "path": path, **info,
                         "sample": f"{stripes} stripes per step, {threads} threads, Path::{path.capitalize()}",
                         "other_path": {"path": other, "value": round(ob / (oe + od) / 1e9, 6),
                                        "decode_gbs": round(ob / od / 1e9, 6), "stripes": o_stripes}},
        "e2e": {"value": round(value, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(W.CONFIGS))
    ap.add_argument("--stripes", type=int, default=0, help="override stripes per GPU (default: the config's)")
    ap.add_argument("--chunk", type=int, default=8192, help="stripes per kernel launch")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--e2e-stripes", type=int, default=4096)
    ap.add_argument("--e2e-chunk", type=int, default=256)
    ap.add_argument("--e2e-sequential", action="store_true", help="e2e: all encode chunks, then all decode chunks")
    ap.add_argument("--graph", action="store_true",
                    help="time CUDA-graph replays of the whole step (launch-bound small configs, e.g. C1)")
    ap.add_argument("--e2e-streams", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-step-seconds", type=float, default=6.0)
    ap.add_argument("--ref-path", default="fast", choices=sorted(PATHS),
                    help="reference arm decode path (fast = the faster; auto = the CLI default, Lagrange at k <= 256)")
    ap.add_argument("--sweep", default="C5:strong",
                    help="second workload measured after the headline and nested in the line as 'sweep' "
                         "(north_star's multi-GPU sweep: C5 sharded by stripe); 'none' to skip")
    ap.add_argument("--sweep-steps", type=int, default=5)
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU test mode: the launcher, rank layout and cross-rank reductions without a GPU")
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per decode launch (profiles/)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo = test mode for several ranks on fewer GPUs (host-side barrier/max only)")
    ap.add_argument("--codec", default="nonsystematic", choices=["nonsystematic", "systematic"],
                    help="headline: non-systematic (BASELINE north_star); systematic = the SURVEY 8(f) next row")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    args.steps = max(1, args.steps)
    global SYSTEMATIC
    SYSTEMATIC = args.codec == "systematic"

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torch.distributed.run
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if args.dry_run:
        args.dist_backend = "gloo"
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.dist_backend == "gloo":
            # test mode: ranks may share GPUs (or run on no GPU at all with --dry-run);
            # the barrier / max-over-ranks run on the host
            ndev = torch.cuda.device_count()
            if ndev:
                local_rank = local_rank % ndev
                torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    comm = communicator_report(rank, world, local_rank, args)
    if args.dry_run:
        res = run_dry(args, rank, world)
    else:
        res = run_gpu(args, rank, world, local_rank)
        sweep = parse_sweep(args.sweep)
        if sweep and (sweep[0] != args.config or sweep[1] != args.scaling):
            import torch
            torch.cuda.empty_cache()
            sub = argparse.Namespace(**vars(args))
            sub.config, sub.scaling, sub.stripes, sub.steps = sweep[0], sweep[1], 0, max(1, args.sweep_steps)
            sub.e2e_stripes, sub.no_cpu_baseline, sub.graph = 0, True, False
            r2 = run_gpu(sub, rank, world, local_rank)
            res["sweep"] = {key: r2[key] for key in ("value", "unit", "n_gpus", "ms_per_step", "scaling", "steps",
                                                     "encode_gbs", "decode_gbs", "decode_with_plans_gbs",
                                                     "phases_ms", "config", "gpu_launches", "verified", "clocks")}
            res["sweep"]["roofline_decode_frac"] = r2["roofline"]["frac"]
            res["sweep"]["roofline_encode_frac"] = r2["roofline_encode"]["frac"]
            res["sweep"]["note"] = ("north_star's multi-GPU sweep: the config's stripes sharded evenly over the ranks "
                                    "(strong scaling), value = total source bytes / max-over-ranks step time")
    res["communicator"] = comm
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def parse_sweep(spec):
    if not spec or spec == "none":
        return None
    cfg, _, scaling = spec.partition(":")
    if cfg not in W.CONFIGS or scaling not in ("weak", "strong"):
        raise SystemExit(f"bad --sweep {spec!r} (want e.g. C5:strong)")
    return cfg, scaling


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n):
    """`python bench.py --gpus N` without torchrun: start N ranks (one per GPU)
    with torch.distributed.run on 127.0.0.1, exactly as the driver does; rank 0
    prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd[1:6])} ...", file=sys.stderr, flush=True)
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "4"))
    return subprocess.call(cmd, env=env)


def communicator_report(rank, world, local_rank, args):
    """Every rank logs its place in the communicator; an all-reduce of ones
    proves how many ranks took part (outside any timed region)."""
    seen = world
    backend = None
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = dist.get_backend()
        dev = "cpu" if backend == "gloo" else torch.device(f"cuda:{local_rank}")
        t = torch.ones(1, dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        seen = int(t.item())
    dev_name = f"cuda:{local_rank}" if not args.dry_run else "cpu"
    print(f"[bench] rank {rank}/{world} on {dev_name}: backend={backend or 'none'} communicator ranks={seen}",
          file=sys.stderr, flush=True)
    return {"backend": backend or "none", "world_size": world, "ranks_seen_allreduce": seen}


def run_dry(args, rank, world):
    """The multi-rank control flow of run_gpu without a GPU (CPU tests): the
    same stripe ranges, seeds and pattern slices, a barrier-bracketed timed
    region of host work sized by the rank's stripes, max-over-ranks timing and
    the summed verification counts."""
    import torch.distributed as dist
    cfg = W.CONFIGS[args.config]
    S = args.stripes or cfg.stripes
    lo, hi, seed, pats, sp = rank_layout(cfg, S, rank, world, args.scaling)
    src = W.symbols(seed, lo * cfg.k * 4, (hi - lo) * cfg.k * 4)  # a 4-column slice of the rank's source
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        digest = int(np.bitwise_xor.reduce(src.astype(np.uint64))) if src.size else 0
    ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps)
    if world > 1:
        dist.barrier()
    mx = max_over_ranks([ms])[0]
    tot = sum_over_ranks([0, hi - lo, len(pats)])
    ranges = [None] * world
    if world > 1:
        dist.all_gather_object(ranges, (rank, lo, hi, seed, int(sp.size)))
    else:
        ranges = [(rank, lo, hi, seed, int(sp.size))]
    return {"metric": "dry run (no GPU): rank layout and reductions", "n_gpus": world, "scaling": args.scaling,
            "config": {"workload": cfg.name, "stripes": S}, "ms_per_step_max": mx, "digest_rank0": digest,
            "verified": {"stripes_checked_all_ranks": tot[1], "mismatched_stripes_all_ranks": tot[0],
                         "patterns_all_ranks": tot[2]},
            "ranks": [{"rank": r, "lo": a, "hi": b, "seed": sd, "stripes": n} for r, a, b, sd, n in ranges]}


if __name__ == "__main__":
    main()
