"""The rest of the reference's API through the C ABI on the GPU (poly_aux.cu):
status codes of the auxiliary entry points and values against the oracle /
Python restatements (the C++ drop-in's checks are in tests/cpp/test_dropin.cpp)."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P = 65537


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_0907_1788_b200 import Codec
    return Codec(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def ptr(t):
    return C.c_void_p(t.data_ptr())


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def test_status_codes(codec):
    from paper_0907_1788_b200 import _lib
    lib = _lib.load()
    buf = torch.zeros(64, dtype=torch.int32, device="cuda")
    assert lib.fntrs_gpu_chirp_table(codec.ctx, 6, 3, ptr(buf), ptr(buf), ptr(buf), None) == 3  # InvalidTransformSize
    assert lib.fntrs_gpu_transform_tables(codec.ctx, 12, ptr(buf), None, None, None, None, None) == 3
    assert lib.fntrs_gpu_geom_eval(codec.ctx, 8, 3, ptr(buf), 9, None, None, ptr(buf), None) == 4  # SizeMismatch
    assert lib.fntrs_gpu_geom_eval_negative(codec.ctx, 8, 3, ptr(buf), 9, None, None, ptr(buf), None) == 4
    assert lib.fntrs_gpu_subproduct_tree(codec.ctx, 0, ptr(buf), ptr(buf), None) == 4
    big = torch.zeros(1 << 17, dtype=torch.int32, device="cuda")
    # full domain: only the transform root (3) or its inverse evaluate (geom.cpp:59-71)
    assert lib.fntrs_gpu_geom_eval(codec.ctx, 65536, 5, ptr(buf), 3, None, None, ptr(big), None) == 3
    assert lib.fntrs_gpu_geom_eval(codec.ctx, 65536, 3, ptr(buf), 3, None, None, ptr(big), None) == 0


def test_naive_dft_any_root_and_lagrange(codec):
    from paper_0907_1788_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(5)
    for n in (1, 3, 17, 100):
        a = rng.integers(0, P, n).astype(np.uint32)
        root = int(rng.integers(2, P))
        d_in, d_out = dev(a), torch.zeros(n, dtype=torch.int32, device="cuda")
        assert lib.fntrs_gpu_naive_dft(codec.ctx, root, 0, n, ptr(d_in), ptr(d_out), None) == 0
        want = [sum(int(a[i]) * pow(root, i * j, P) for i in range(n)) % P for j in range(n)]
        assert host(d_out).tolist() == want
    # Lagrange through distinct points: P(x_i) = v_i, degree < k
    k = 40
    xs = rng.choice(P, k, replace=False).astype(np.uint32)
    vs = rng.integers(0, P, k).astype(np.uint32)
    out = torch.zeros(k, dtype=torch.int32, device="cuda")
    assert lib.fntrs_gpu_lagrange(codec.ctx, k, ptr(dev(xs)), ptr(dev(vs)), ptr(out), None) == 0
    c = host(out).astype(np.int64)
    for x, v in zip(xs.tolist(), vs.tolist()):
        acc = 0
        for coef in c[::-1]:
            acc = (acc * x + int(coef)) % P
        assert acc == v


def test_geom_eval_matches_horner(codec):
    from paper_0907_1788_b200 import _lib
    lib = _lib.load()
    rng = np.random.default_rng(6)
    for n, length in ((8, 8), (64, 17), (1024, 1000)):
        root = int(rng.integers(2, P))
        a = rng.integers(0, P, length).astype(np.uint32)
        out = torch.zeros(n, dtype=torch.int32, device="cuda")
        assert lib.fntrs_gpu_geom_eval(codec.ctx, n, root, ptr(dev(a)), length, None, None, ptr(out), None) == 0
        got = host(out)
        for i in (0, 1, n // 2, n - 1):
            x = pow(root, i, P)
            acc = 0
            for coef in a[::-1].tolist():
                acc = (acc * x + coef) % P
            assert int(got[i]) == acc
