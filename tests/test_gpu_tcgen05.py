"""tcgen05 building blocks of the tensor-core scan (N5) against numpy: SW128
K-major descriptors, kind::tf32 SS and TS MMAs, TMEM st/ld, and the 3xTF32
split that makes the scan's dot products fp32-accurate."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
SO = os.path.join(os.path.dirname(__file__), "cuda", "libtcprobe.so")


def tf32_trunc(a):
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def run(A, B):
    lib = C.CDLL(SO)
    fp = C.POINTER(C.c_float)
    D1 = np.zeros((128, 32), np.float32)
    D2 = np.zeros((128, 16), np.float32)
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    rc = lib.tc_probe(A.ctypes.data_as(fp), B.ctypes.data_as(fp), A.shape[1], D1.ctypes.data_as(fp),
                      D2.ctypes.data_as(fp))
    assert rc == 0
    return D1, D2


@pytest.mark.parametrize("K", [32, 128])
def test_tf32_mma_layouts(engine, K):
    rng = np.random.default_rng(K)
    A = rng.integers(-8, 8, size=(128, K)).astype(np.float32)  # exact in tf32
    B = rng.integers(-8, 8, size=(32, K)).astype(np.float32)
    D1, D2 = run(A, B)
    np.testing.assert_array_equal(D1, A @ B.T)
    np.testing.assert_array_equal(D2, A @ B[:16].T)


def test_tf32_truncation_model(engine):
    """The scan assumes the tensor core uses x's top 19 bits (truncation)."""
    rng = np.random.default_rng(1)
    K = 128
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = tf32_trunc(rng.standard_normal((32, K)).astype(np.float32))
    D1, _ = run(A, B)
    want_trunc = tf32_trunc(A).astype(np.float64) @ B.T.astype(np.float64)
    exact = A.astype(np.float64) @ B.T.astype(np.float64)
    err_trunc = np.abs(D1 - want_trunc).max()
    err_exact = np.abs(D1 - exact).max()
    assert err_trunc < 1e-4, (err_trunc, err_exact)


def test_three_tf32_split_is_fp32_accurate(engine):
    rng = np.random.default_rng(2)
    K = 128
    x = rng.standard_normal((128, K)).astype(np.float32)
    q = rng.standard_normal((16, K)).astype(np.float32)
    qh = tf32_trunc(q)
    ql = (q - qh).astype(np.float32)
    xl = (x - tf32_trunc(x)).astype(np.float32)
    D1, _ = run(x, np.concatenate([qh, ql]))
    _, D2 = run(xl, np.concatenate([qh, ql]))
    dot = D1[:, :16] + D1[:, 16:] + D2
    exact = x.astype(np.float64) @ q.T.astype(np.float64)
    scale = np.abs(x).astype(np.float64) @ np.abs(q).T.astype(np.float64)
    assert (np.abs(dot - exact) / scale).max() < 4e-6
