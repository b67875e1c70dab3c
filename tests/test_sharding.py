"""Multi-rank host logic of the stripe sharding (gloo, world size 2, CPU)."""
import os
import socket

import pytest

from paper_0907_1788_b200.sharding import max_over_ranks, rank_seed, rank_stripes, sum_over_ranks


def test_strong_ranges_partition_exactly():
    for total in (0, 1, 7, 2048, 65536):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                lo, hi = rank_stripes(total, r, world, "strong")
                assert 0 <= lo <= hi <= total
                covered.extend(range(lo, hi))
            assert covered == list(range(total))
            sizes = [rank_stripes(total, r, world, "strong")[1] - rank_stripes(total, r, world, "strong")[0]
                     for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_weak_ranges_and_seeds():
    assert all(rank_stripes(65536, r, 8, "weak") == (0, 65536) for r in range(8))
    assert len({rank_seed(5, r) for r in range(8)}) == 8
    with pytest.raises(ValueError):
        rank_stripes(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = rank_stripes(2048, rank, world, "strong")
        # per-rank "times": the max over ranks must come back on every rank
        got = max_over_ranks([10.0 + rank, 100.0 - rank, float(hi - lo)])
        # per-rank mismatch / checked-stripe counts summed over ranks (bench's verification gather)
        tot = sum_over_ranks([rank, hi - lo])
        dist.barrier()
        q.put((rank, lo, hi, got, tot))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [(0, 1024), (1024, 2048)]
    for r in res:
        assert r[3] == [11.0, 100.0, 1024.0]
        assert r[4] == [1, 2048]


def _bench(*argv, timeout=300):
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *argv], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0]), r.stderr


def test_bench_gpus2_spawns_two_ranks_strong():
    """`bench.py --gpus 2` launches two ranks itself (torch.distributed.run on
    127.0.0.1); the ranks split C5's stripes evenly, share the seed, and the
    line carries the max over ranks and the counts summed over ranks."""
    res, err = _bench("--gpus", "2", "--dry-run", "--config", "C5", "--scaling", "strong", "--steps", "2")
    assert res["n_gpus"] == 2
    assert res["communicator"] == {"backend": "gloo", "world_size": 2, "ranks_seen_allreduce": 2}
    assert [(r["lo"], r["hi"]) for r in res["ranks"]] == [(0, 1024), (1024, 2048)]
    assert len({r["seed"] for r in res["ranks"]}) == 1
    assert res["verified"]["stripes_checked_all_ranks"] == 2048
    assert res["verified"]["patterns_all_ranks"] == 2048  # C5: one pattern per stripe, none shared across ranks
    assert err.count("communicator ranks=2") == 2  # logged by every rank


def test_bench_gpus2_weak_seeds_differ():
    res, _ = _bench("--gpus", "2", "--dry-run", "--config", "C4", "--scaling", "weak", "--steps", "1")
    assert [(r["lo"], r["hi"]) for r in res["ranks"]] == [(0, 256), (0, 256)]
    assert res["ranks"][0]["seed"] != res["ranks"][1]["seed"]
    assert res["verified"]["stripes_checked_all_ranks"] == 512
