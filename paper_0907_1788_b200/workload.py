"""Seeded synthetic workloads for the five BASELINE.json configurations.

No public dataset is involved: the reference benches random
symbols (proj/tools/fntrs_main.cpp:248-252). Source symbols are uniform
uint16 from a splitmix64 stream (identical to fntrs_gpu_fill_symbols on the
device); erasure patterns are seeded k-subsets per stripe, in the classes
each configuration prescribes. Everything is deterministic given the seed.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED = 0x09071788
GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, index: np.ndarray) -> np.ndarray:
    """Output number `index` (0-based) of the splitmix64 stream seeded with `seed`."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (index.astype(np.uint64) + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def symbols(seed: int, first: int, count: int) -> np.ndarray:
    """uint16 source symbols first..first+count of the stream (== fntrs_gpu_fill_symbols)."""
    return (splitmix64(seed, np.arange(first, first + count, dtype=np.uint64)) & np.uint64(0xFFFF)).astype(np.uint16)


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    k: int
    L: int          # uint16 symbols per packet (= codewords per stripe)
    stripes: int
    pattern: str    # erasure-pattern class rule

    @property
    def source_bytes(self) -> int:
        return 2 * self.k * self.L * self.stripes


# BASELINE.json "configs", in order.
CONFIGS = {
    "C1": Config("C1", 2048, 1024, 512, 1, "uniform"),
    "C2": Config("C2", 256, 128, 2048, 65536, "half_shared"),
    "C3": Config("C3", 65536, 32768, 2048, 1, "split_halves"),
    "C4": Config("C4", 16384, 8192, 1024, 256, "three_classes"),
    "C5": Config("C5", 4096, 2048, 1024, 2048, "uniform"),
}


def _subset(seed: int, salt: int, n: int, k: int, lo: int = 0) -> np.ndarray:
    """Seeded uniform k-subset of [lo, lo+n), ascending (k smallest splitmix keys)."""
    keys = splitmix64(seed ^ (salt * 0x632BE59BD9B4E019 & 0xFFFFFFFFFFFFFFFF), np.arange(n, dtype=np.uint64))
    idx = np.argpartition(keys, k - 1)[:k] if k < n else np.arange(n)
    return np.sort(idx).astype(np.uint32) + np.uint32(lo)


def _bursts(seed: int, salt: int, n: int, k: int, burst: int) -> np.ndarray:
    """Erase (n-k)/burst non-overlapping bursts at seeded starts; return kept positions."""
    nb = (n - k) // burst
    cuts = np.sort(splitmix64(seed ^ (salt * 0x2545F4914F6CDD1D & 0xFFFFFFFFFFFFFFFF),
                              np.arange(nb, dtype=np.uint64)) % np.uint64(k + 1)).astype(np.int64)
    keep = np.ones(n, dtype=bool)
    for b, c in enumerate(cuts):   # b bursts and c kept symbols precede burst b
        start = int(c) + b * burst
        keep[start:start + burst] = False
    out = np.nonzero(keep)[0].astype(np.uint32)
    assert out.size == k
    return out


def patterns(cfg: Config, seed: int = SEED, stripes: int | None = None):
    """Erasure patterns for the config.

    Returns (pats [P, k] uint32 ascending received positions, stripe_pattern [S] uint32).
    """
    S = cfg.stripes if stripes is None else stripes
    n, k = cfg.n, cfg.k
    if cfg.pattern == "uniform":
        pats = np.stack([_subset(seed, s, n, k) for s in range(S)])
        return pats, np.arange(S, dtype=np.uint32)
    if cfg.pattern == "half_shared":
        # even stripes share pattern 0; odd stripe s uses its own
        npat = 1 + S // 2
        pats = np.empty((npat, k), dtype=np.uint32)
        keys = splitmix64(seed, np.arange(npat * n, dtype=np.uint64)).reshape(npat, n)
        pats[:] = np.sort(np.argsort(keys, axis=1, kind="stable")[:, :k], axis=1)
        sp = np.zeros(S, dtype=np.uint32)
        sp[1::2] = np.arange(1, 1 + S // 2, dtype=np.uint32)[: sp[1::2].size]
        return pats, sp
    if cfg.pattern == "split_halves":
        h = n // 2
        pats = np.stack([np.concatenate([_subset(seed, 2 * s, h, k // 2), _subset(seed, 2 * s + 1, h, k // 2, lo=h)])
                         for s in range(S)])
        return pats, np.arange(S, dtype=np.uint32)
    if cfg.pattern == "three_classes":
        # s % 3: 0 uniform (distinct), 1 parity only (shared), 2 bursts (distinct)
        rows, sp, shared = [], np.zeros(S, dtype=np.uint32), None
        for s in range(S):
            c = s % 3
            if c == 1:
                if shared is None:
                    shared = len(rows)
                    rows.append(np.arange(k, n, dtype=np.uint32))
                sp[s] = shared
                continue
            sp[s] = len(rows)
            rows.append(_subset(seed, s, n, k) if c == 0 else _bursts(seed, s, n, k, 1024))
        return np.stack(rows), sp
    raise ValueError(cfg.pattern)


# ------------------------------------------------ device-side stripe helpers ----
def received_packets(enc, enc_esc, enc_count, pats, stripe_pattern, n: int):
    """Gather the received packets of every stripe on the device (torch plumbing).

    enc [S, n, L] int16 CUDA tensor; enc_esc/enc_count: the encoder's escape
    list; pats [P, kp] host uint32; stripe_pattern [S] host uint32.
    Returns (rx [S, kp, L], rx_esc int64 sorted symbol indices into rx).
    """
    import torch
    S, nn, L = enc.shape
    dev = enc.device
    kp = pats.shape[1]
    rows = torch.from_numpy(pats[stripe_pattern].astype(np.int64)).to(dev)           # [S, kp]
    rx = torch.gather(enc, 1, rows[:, :, None].expand(-1, -1, L)).contiguous()
    ne = int(enc_count.item())
    if ne == 0:
        return rx, None
    keys = enc_esc[:ne]
    row, col = keys // L, keys % L
    s, pos = row // n, row % n
    inv = torch.full((pats.shape[0], n), -1, dtype=torch.int64, device=dev)
    inv.scatter_(1, torch.from_numpy(pats.astype(np.int64)).to(dev),
                 torch.arange(kp, device=dev).expand(pats.shape[0], -1).contiguous())
    spd = torch.from_numpy(stripe_pattern.astype(np.int64)).to(dev)
    i = inv[spd[s], pos]
    keep = i >= 0
    out = (s[keep] * kp + i[keep]) * L + col[keep]
    out, _ = torch.sort(out)
    return rx, (out if out.numel() else None)
