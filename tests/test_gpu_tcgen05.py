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


# ---- kind::f16 (bf16 x bf16 -> fp32) accumulator: the error model the certification bound uses ----
# (paper_2504_15302_b200/csrc/ivf_kernels.cuh gamma_bf16x3; DESIGN.md §2 "Certification")
U = 2.0 ** -24


def test_bf16_accumulator_alignment_window(engine):
    """Within one K = 16 MMA step every term is aligned to the largest one and kept to 2^-25 of
    it: products of 2^-25 next to a 1 survive (their sum is then rounded), 2^-26 are dropped."""
    from tc_acc import run_acc
    for j, want in ((25, lambda n: (n // 4) * 4), (26, lambda n: 0)):
        A = np.zeros((128, 64), np.float32)
        B = np.zeros((32, 64), np.float32)
        A[:, 0], B[:, 0] = 1.0, 1.0
        A[:, 1:16] = 2.0 ** -j
        for c in range(16):
            B[c, 1:1 + c] = 1.0  # column c: c tiny products beside the 1
        D = run_acc(A, B)
        got = [int(round((D[0, c] - 1.0) / 2.0 ** -25)) for c in range(16)]
        assert got == [want(n) * (1 if j == 25 else 0) for n in range(16)], (j, got)


def test_bf16_accumulator_rounds_toward_zero(engine):
    from tc_acc import run_acc
    ulp = 2.0 ** -23
    for frac, want in ((0.75, 0.0), (1.5, 1.0), (-0.25, -0.5), (-0.75, -1.0)):
        A = np.zeros((128, 64), np.float32)
        B = np.zeros((32, 64), np.float32)
        A[:, 0], B[:, 0] = frac * ulp, 1.0
        D = run_acc(A, B, np.ones((128, 32), np.float32))
        assert (D[0, 0] - 1.0) / ulp == want, (frac, D[0, 0])


def _families(rng, K):
    yield "one_big", 2.0 ** rng.uniform(-25, -22, (128, K)), 1 + rng.random((32, K)) * 0.99, 0
    yield "loguniform", 2.0 ** rng.uniform(-30, 0, (128, K)), 2.0 ** rng.uniform(-30, 0, (32, K)), 0
    yield "mixed_sign", 2.0 ** rng.uniform(-26, 0, (128, K)), 1 + rng.random((32, K)), 1
    yield "uniform", rng.random((128, K)) + 0.5, rng.random((32, K)) + 0.5, 0


@pytest.mark.parametrize("K", [64, 512])
def test_bf16_accumulator_error_within_model(engine, K):
    """Adversarial operands (one dominant product then products just below its 2^-25 window,
    log-uniform magnitudes, mixed signs): the error stays within 10 u of each step's magnitude
    (|accumulator| + sum |products|), summed over the K / 16 steps — the model gamma_bf16x3 takes
    as 11 u per step."""
    from tc_acc import bf16_val, run_acc
    rng = np.random.default_rng(K)
    for t in range(6):
        for name, A, B, signs in _families(rng, K):
            if name == "one_big":
                A[:, rng.integers(0, K)] = 1.0
            if signs:
                A = A * rng.choice([-1.0, 1.0], A.shape)
            A, B = bf16_val(A.astype(np.float32)), bf16_val(B.astype(np.float32))
            D = run_acc(A, B).astype(np.float64)
            P = A.astype(np.float64)[:, None, :] * B.astype(np.float64)[None, :, :]  # 128 x 32 x K
            steps = P.reshape(128, 32, K // 16, 16)
            partial = np.cumsum(steps.sum(3), axis=2)  # exact running sums after each step
            acc_before = np.concatenate([np.zeros((128, 32, 1)), partial[:, :, :-1]], axis=2)
            step_mag = np.abs(acc_before) + np.abs(steps).sum(3)
            model = 10 * U * step_mag.sum(2)
            err = np.abs(D - partial[:, :, -1])
            assert (err <= model * 1.0001 + 1e-45).all(), (name, (err / model).max())
            assert (err <= 11 * U * (K // 16) * np.abs(P).sum(2) * 1.0001 + 1e-45).all(), name


@pytest.mark.parametrize("d", [64, 512])
def test_bf16x3_dot_within_certification_bound(engine, d):
    """The scan's dot product as it computes it — x1.q1, x1.q2 and x2.q1 in three accumulators,
    combined (D1 + D2) + D3 in fp32 — against exact q.x, on split-boundary operands: within
    gamma_bf16x3(d) * sum |x_t q_t|."""
    from tc_acc import bf16_val, run_acc
    rng = np.random.default_rng(d)
    gamma = (524 + 0.7 * d) * U
    worst = 0.0
    for t in range(4):
        x = (2.0 ** rng.uniform(-4, 8, (128, d)) * rng.choice([-1, 1], (128, d))).astype(np.float32)
        q = (2.0 ** rng.uniform(-4, 8, (32, d))).astype(np.float32)
        if t % 2:  # split-boundary values: residuals just under half a bf16 ulp, aligned signs
            x = np.abs(x)
            x = (bf16_val(x) * (1 + 2.0 ** -9 - 2.0 ** -17)).astype(np.float32)
            q = (bf16_val(q) * (1 + 2.0 ** -9 - 2.0 ** -17)).astype(np.float32)
        x1 = bf16_val(x)
        x2 = bf16_val((x - x1).astype(np.float32))
        q1 = bf16_val(q)
        q2 = bf16_val((q - q1).astype(np.float32))
        D1, D2, D3 = run_acc(x1, q1), run_acc(x1, q2), run_acc(x2, q1)
        dot = ((D1 + D2) + D3).astype(np.float64)  # fp32 adds, as the kernels do
        exact = x.astype(np.float64) @ q.T.astype(np.float64)
        mag = np.abs(x).astype(np.float64) @ np.abs(q).T.astype(np.float64)
        r = (np.abs(dot - exact) / mag).max()
        worst = max(worst, r)
        assert r <= gamma, (d, t, r / U)
    print(f"d={d}: worst |dot error| / sum|xq| = {worst / U:.1f} u (bound {gamma / U:.0f} u)")


@pytest.mark.parametrize("K", [64, 512])
def test_f16_accumulator_error_within_model(engine, K):
    """The residual scan's fp16 operands on the same kind::f16 datapath: the accumulator model the
    bounds use (10 u of each K = 16 step's magnitude) holds for fp16 inputs too (magnitudes kept in
    fp16's normal range, so the products are exact)."""
    from tc_acc import f16_val, run_acc
    rng = np.random.default_rng(100 + K)
    for t in range(6):
        A = 2.0 ** rng.uniform(-7, 4, (128, K)) * rng.choice([-1.0, 1.0], (128, K))
        B = 2.0 ** rng.uniform(-7, 4, (32, K))
        if t % 2:
            A[:, rng.integers(0, K)] = 2.0 ** 8  # one dominant product
        A, B = f16_val(A.astype(np.float32)), f16_val(B.astype(np.float32))
        D = run_acc(A, B, fp16=True).astype(np.float64)
        P = A.astype(np.float64)[:, None, :] * B.astype(np.float64)[None, :, :]
        steps = P.reshape(128, 32, K // 16, 16)
        partial = np.cumsum(steps.sum(3), axis=2)
        acc_before = np.concatenate([np.zeros((128, 32, 1)), partial[:, :, :-1]], axis=2)
        model = 10 * U * (np.abs(acc_before) + np.abs(steps).sum(3)).sum(2)
        err = np.abs(D - partial[:, :, -1])
        assert (err <= model * 1.0001 + 1e-45).all(), (err / model).max()


@pytest.mark.parametrize("d", [128, 512])  # (the probe's K <= 512)
def test_fp16_residual_dot_within_certification_bound(engine, d):
    """The fp16 residual scan's dot as it computes it — fp16(r) . fp16(q) in one fp32 accumulator —
    against the exact r . q, on rounding-boundary operands (components just under half an fp16 ulp
    past a representable value, aligned signs): within (2^-11 (1 + 2^-9) + 2^-11 + 16 u + 0.7 d u)
    * sum |r_t q_t| (1 + 2^-9), the terms gamma_resid16_r / _q bound with Cauchy-Schwarz."""
    from tc_acc import f16_val, run_acc
    rng = np.random.default_rng(d)
    gamma = (8192 * (1 + 2.0 ** -9) + 8192 + 16 + 0.7 * d) * U * (1 + 2.0 ** -9)
    worst = 0.0
    for t in range(4):
        r = (2.0 ** rng.uniform(-6, 2, (128, d)) * rng.choice([-1, 1], (128, d))).astype(np.float32)
        q = (2.0 ** rng.uniform(-6, 2, (32, d))).astype(np.float32)
        if t % 2:
            r = np.abs(r)
            r = (f16_val(r) * (1 + 2.0 ** -11 - 2.0 ** -20)).astype(np.float32)
            q = (f16_val(q) * (1 + 2.0 ** -11 - 2.0 ** -20)).astype(np.float32)
        D = run_acc(f16_val(r), f16_val(q), fp16=True).astype(np.float64)
        exact = r.astype(np.float64) @ q.T.astype(np.float64)
        mag = np.abs(r).astype(np.float64) @ np.abs(q).T.astype(np.float64)
        ratio = np.abs(D - exact) / (gamma * mag)
        worst = max(worst, ratio.max())
    assert worst <= 1.0, worst
