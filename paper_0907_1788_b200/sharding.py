"""Multi-GPU partitioning of stripes.

Stripes are independent, so ranks never exchange data: each rank owns a set
of stripes and codes them on its own GPU. torch.distributed (NCCL on GPUs,
gloo in the CPU tests) is used only for the barrier around the timed region
and for the max-over-ranks of the measured times.
"""
from __future__ import annotations


def rank_stripes(total: int, rank: int, world: int, scaling: str = "weak") -> tuple[int, int]:
    """Half-open stripe range [lo, hi) coded by `rank`.

    weak:   every rank codes `total` stripes of its own (per-GPU work fixed);
            the range is local to the rank (its own seeded data).
    strong: the `total` stripes are split into contiguous, near-equal ranges
            (rank g takes [g*S/G, (g+1)*S/G)).
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if scaling == "weak":
        return 0, total
    if scaling != "strong":
        raise ValueError(scaling)
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi


def rank_seed(base: int, rank: int) -> int:
    """Seed of a rank's own stripes (weak scaling)."""
    return base + 1000003 * rank


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    vals = [float(v) for v in values]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return vals
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def sum_over_ranks(values, device=None):
    """Element-wise sum of a list of integers over all ranks (identity when not
    distributed): gathers per-rank mismatch counts to every rank, outside any
    timed region (NCCL only for digests / counts)."""
    import torch
    import torch.distributed as dist
    vals = [int(v) for v in values]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return vals
    if dist.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor(vals, dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) for x in t.cpu()]
