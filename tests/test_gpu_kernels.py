"""Kernel-level parity on the GPU: fold (b), state gather/scatter (c), server
elementwise ops, against NumPy on the same fp32 inputs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2303_01778_b200 import _kernels
    return _kernels


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("n", [1, 3, 4, 1000, 7850, 1 << 20])
def test_fold_matches_numpy_fma(K, n):
    rng = np.random.default_rng(n)
    acc0 = rng.standard_normal(n).astype(np.float32)
    x = rng.standard_normal(n).astype(np.float32)
    acc = dev(acc0)
    K.fold(acc, dev(x), 3.0)
    want = (acc0.astype(np.float64) + 3.0 * x.astype(np.float64)).astype(np.float32)  # one rounding == fma
    assert np.array_equal(host(acc), want)


@pytest.mark.parametrize("g,n", [(1, 10), (7, 4096), (33, 7850), (300, 1003)])
def test_fold_group_equals_sequential_folds(K, g, n):
    import torch
    rng = np.random.default_rng(g * n)
    xs = rng.standard_normal((g + 3, n)).astype(np.float32)
    order = rng.permutation(g + 3)[:g].astype(np.int32)
    w = rng.integers(1, 600, g).astype(np.float32)
    acc = dev(np.zeros(n))
    K.fold_group(acc, dev(xs), torch.from_numpy(order).cuda(), dev(w))
    ref = dev(np.zeros(n))
    X = dev(xs)
    for j in range(g):
        K.fold(ref, X[int(order[j])].contiguous(), float(w[j]))
    assert np.array_equal(host(acc), host(ref))
    terms = w[:, None].astype(np.float64) * xs[order].astype(np.float64)
    bound = 1e-6 * g * np.abs(terms).sum(0)  # fp32 sequential-sum error bound (loose)
    assert np.all(np.abs(host(acc) - terms.sum(0)) <= bound + 1e-6)


def test_fold_group_column_slice(K):
    rng = np.random.default_rng(5)
    mat = rng.standard_normal((6, 50)).astype(np.float32)
    acc = dev(np.zeros(13))
    K.fold_group(acc, dev(mat)[:, 17:30], None, None)
    assert np.allclose(host(acc), mat[:, 17:30].sum(0), atol=1e-5)


def test_lincomb_and_delta_affine(K):
    rng = np.random.default_rng(3)
    x, y, z = (rng.standard_normal(1001).astype(np.float32) for _ in range(3))
    out = dev(np.zeros(1001))
    K.lincomb(out, dev(x), 2.0, dev(y), -0.5, dev(z), 0.25)
    assert np.allclose(host(out), 2 * x - 0.5 * y + 0.25 * z, atol=1e-5)
    a = rng.standard_normal((4, 257)).astype(np.float32)
    base = rng.standard_normal(257).astype(np.float32)
    c = rng.standard_normal(257).astype(np.float32)
    d = rng.standard_normal((4, 257)).astype(np.float32)
    s = np.array([1.0, -2.0, 0.5, 3.0], np.float32)
    o = dev(np.zeros((4, 257)))
    K.delta_affine(o, dev(a), dev(base), dev(s), cvec=dev(c), c=-1.0, dmat=dev(d), d=1.0)
    want = s[:, None] * (a - base) - c + d
    assert np.allclose(host(o), want, atol=1e-5)


def test_state_gather_scatter_roundtrip(K):
    import torch
    rng = np.random.default_rng(11)
    store = dev(rng.standard_normal((20, 7850)))
    slots = torch.tensor([3, -1, 17, 0], dtype=torch.int32, device="cuda")
    work = dev(np.full((4, 7850), 9.0))
    K.state_gather(work, store, slots)
    w = host(work)
    s = host(store)
    assert np.array_equal(w[0], s[3]) and np.array_equal(w[2], s[17]) and np.array_equal(w[3], s[0])
    assert not w[1].any()  # never-saved client -> zero default state
    new = rng.standard_normal((4, 7850)).astype(np.float32)
    K.state_scatter(store, dev(new), slots)
    s2 = host(store)
    assert np.array_equal(s2[3], new[0]) and np.array_equal(s2[17], new[2])
    untouched = [i for i in range(20) if i not in (0, 3, 17)]
    assert np.array_equal(s2[untouched], s[untouched])


def test_native_errors_are_loud(K):
    from paper_2303_01778_b200._lib import NativeError, lib
    with pytest.raises(NativeError, match="bad arguments"):
        lib.check(lib.pb_fold_f32(None, None, 1.0, 5, None))
