"""CPU checks of the C-ABI library: it loads, exports every symbol
include/fntrs_gpu.h declares, and its host-only entry points behave like the
reference (no compute calls without a GPU)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fntrs_gpu.h")).read()
    return sorted(set(re.findall(r"\b(fntrs_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_0907_1788_b200 import _lib
    lib = _lib.load()
    names = declared_symbols()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.exported_symbols())


def test_code_params_matches_reference_rules():  # proj/src/codec.cpp:112-122
    from paper_0907_1788_b200 import _lib
    lib = _lib.load()
    nd = C.c_uint32()
    assert lib.fntrs_gpu_code_params(3, 6, C.byref(nd)) == 0 and nd.value == 8
    assert lib.fntrs_gpu_code_params(16, 16, C.byref(nd)) == 0 and nd.value == 16
    assert lib.fntrs_gpu_code_params(1, 65536, C.byref(nd)) == 0 and nd.value == 65536
    for k, n in [(0, 4), (5, 4), (1, 65537)]:
        assert lib.fntrs_gpu_code_params(k, n, C.byref(nd)) == 4  # SizeMismatch


def test_python_mirror_code_params():
    import paper_0907_1788_b200 as F
    p = F.CodeParams.make(3, 6)
    assert (p.k, p.n, p.n_domain, p.systematic) == (3, 6, 8, True)
    with pytest.raises(F.SizeMismatch):
        F.CodeParams.make(5, 4)


def test_status_strings_cover_reference_errors():
    from paper_0907_1788_b200 import _lib, codec
    lib = _lib.load()
    for st, cls in codec.STATUS_CLASSES.items():
        assert lib.fntrs_gpu_status_string(st).decode() == cls.__name__


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_0907_1788_b200 import _lib
    import paper_0907_1788_b200 as F
    ctx = C.c_void_p()
    assert _lib.load().fntrs_gpu_create(0, C.byref(ctx)) == 100  # FNTRS_E_CUDA
    with pytest.raises(F.Error):
        F.Codec(0)
    with pytest.raises(F.Error):
        F.encode_nonsystematic(F.CodeParams.make(2, 4, False), [5, 7])


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_0907_1788_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("liboracle", "oracle_bind", "fntrs_oracle", "libfntrs_ref", "orc_", "import oracle"):
                    assert bad not in txt, (f, bad)


def test_subproduct_tree_layout_host_only():
    """Node lengths of the reference's tree shape (poly.cpp:216-242): leaves of
    2 coefficients, adjacent pairs multiplied, an odd last node carried."""
    from paper_0907_1788_b200 import _lib
    lib = _lib.load()
    nl, nn, nc = C.c_uint32(), C.c_uint64(), C.c_uint64()
    assert lib.fntrs_gpu_subproduct_tree_layout(5, C.byref(nl), None, 0, None, C.byref(nn), C.byref(nc)) == 0
    assert (nl.value, nn.value) == (4, 5 + 3 + 2 + 1)
    lv = (C.c_uint32 * 4)()
    lens = (C.c_uint32 * nn.value)()
    assert lib.fntrs_gpu_subproduct_tree_layout(5, C.byref(nl), lv, 4, lens, C.byref(nn), C.byref(nc)) == 0
    assert list(lv) == [5, 3, 2, 1]
    assert list(lens) == [2] * 5 + [3, 3, 2] + [5, 2] + [6]
    assert nc.value == sum(lens)
    assert lib.fntrs_gpu_subproduct_tree_layout(0, None, None, 0, None, None, None) == 4  # SizeMismatch


def test_cli_usage_errors_without_gpu(tmp_path):
    """The `fntrs` CLI rejects bad arguments with exit code 1 before touching
    a device (the reference CLI's CLI11 validation, fntrs_main.cpp:413-444),
    and a codec call without a device fails loudly with exit code 2."""
    import subprocess
    exe = os.path.join(ROOT, "build", "fntrs")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cli"], check=True, capture_output=True)
    src = tmp_path / "f.bin"
    src.write_bytes(b"abc")
    for args in (["encode", str(src), "--k", "5", "--n", "4"], ["encode", str(src), "--k", "65536", "--n", "65536"],
                 ["encode", str(src)], ["decode", str(tmp_path)], ["frobnicate"], ["bench", "--grid", "0"],
                 ["encode", str(src), "--k", "x", "--n", "4"]):
        r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=60)
        assert r.returncode == 1, (args, r.returncode, r.stderr)
        assert "usage" in r.stderr
    r = subprocess.run([exe, "decode", str(tmp_path), "-o", str(tmp_path / "o")], capture_output=True, text=True,
                       timeout=60)
    assert r.returncode == 2 and "no *.manifest.fnt" in r.stderr
