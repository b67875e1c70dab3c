"""Host-side pieces of bench.py (CPU): the per-config roofline bookkeeping read
from the committed captures, the kernel labels, the sweep parser and the CPU
information block."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_kernel_labels_follow_the_path():
    import bench
    from paper_0907_1788_b200 import workload as W
    assert "dec_fast_kernel<8>" in bench.kernel_label(W.CONFIGS["C2"], "decode", False)
    assert "MODE 3" in bench.kernel_label(W.CONFIGS["C2"], "decode", True)
    assert "dec_fast_kernel<12>" in bench.kernel_label(W.CONFIGS["C5"], "decode", False)
    assert "four-step" in bench.kernel_label(W.CONFIGS["C4"], "decode", False)
    assert "enc_a" in bench.kernel_label(W.CONFIGS["C3"], "encode", False)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_profiled_traffic_scales_with_the_launch(name):
    """DRAM traffic per launch comes from the committed capture, scaled to the
    launch's codewords; the fused kernels move their algorithmic bytes."""
    import bench
    from paper_0907_1788_b200 import workload as W
    cfg = W.CONFIGS[name]
    cw = bench.PROFILE_CODEWORDS[name]
    a = bench.profiled(cfg, "decode", False, cw)
    b = bench.profiled(cfg, "decode", False, 2 * cw)
    assert a["traffic"] > 0 and abs(b["traffic"] - 2 * a["traffic"]) <= 2
    alg = cw * 4 * cfg.k  # read 2k + write 2k bytes per codeword
    ratio = a["traffic"] / alg
    if cfg.n <= 4096:
        assert 0.9 < ratio < 1.1
    else:  # the four-step chain's uint32 intermediates
        assert ratio > 4
    assert 0 < a["issue_active_frac"] <= 1 and 0 < a["multiplier_pipe_busy_frac"] <= 1


def test_sweep_parser():
    import bench
    assert bench.parse_sweep("C5:strong") == ("C5", "strong")
    assert bench.parse_sweep("none") is None
    with pytest.raises(SystemExit):
        bench.parse_sweep("C9:strong")


def test_cpu_info_block():
    import bench
    info = bench.cpu_info()
    assert info["logical_cores"] == os.cpu_count()
    assert set(info) == {"cpu_model", "logical_cores", "avx2_path"}


def test_reference_arm_line(tmp_path):
    """`bench.py --impl reference` (the reference library on the host cores)
    prints one JSON line with the contract's keys: impl, the metric and unit of
    the GPU arm, a cpu_baseline block and an e2e block with zero PCIe bytes."""
    import json
    import subprocess
    from oracle_bind import RefLib
    if not RefLib.available():
        pytest.skip("reference library (oracle/_ref) not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "3", "--ref-step-seconds", "0.3"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env={k: v for k, v in os.environ.items() if k != "WORLD_SIZE"})
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["path"] == "fast" and d["cpu_baseline"]["other_path"]["path"] == "auto"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["metric"].startswith("encode & decode GB/s")
