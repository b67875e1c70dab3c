"""bench.py's multi-rank path on a real GPU: two ranks (gloo for the host
barrier / reductions, both on the one GPU a test box has) run run_gpu's full
control flow -- per-rank stripe ranges and seeds, warm-up verification summed
over ranks, barrier-bracketed timed steps, max over ranks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*argv):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True, text=True,
                       timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0]), r.stderr


@pytest.mark.gpu
def test_bench_two_ranks_strong_c5():
    res, err = _bench("--gpus", "2", "--dist-backend", "gloo", "--config", "C5", "--scaling", "strong",
                      "--stripes", "64", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--e2e-stripes", "0",
                      "--sweep", "none")
    assert res["n_gpus"] == 2
    assert res["communicator"]["ranks_seen_allreduce"] == 2
    assert res["config"]["stripes_per_gpu"] == 32
    assert res["verified"]["stripes_checked_all_ranks"] == 64
    assert res["verified"]["mismatched_stripes_all_ranks"] == 0
    assert res["value"] > 0 and res["gpu_launches"] > 0
    assert err.count("communicator ranks=2") == 2


@pytest.mark.gpu
def test_bench_two_ranks_weak_c2_with_sweep():
    res, _ = _bench("--gpus", "2", "--dist-backend", "gloo", "--stripes", "256", "--steps", "2", "--warmup", "3",
                    "--no-cpu-baseline", "--e2e-stripes", "0", "--sweep", "C5:strong", "--sweep-steps", "1")
    assert res["n_gpus"] == 2 and res["scaling"] == "weak"
    assert res["verified"]["stripes_checked_all_ranks"] == 512
    sw = res["sweep"]
    assert sw["n_gpus"] == 2 and sw["scaling"] == "strong"
    assert sw["config"]["stripes_per_gpu"] == 1024
    assert sw["verified"]["mismatched_stripes_all_ranks"] == 0
