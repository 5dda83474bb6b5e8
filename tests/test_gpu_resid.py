"""The residual store (RD_STORE=resid, csrc/resid.cu): the scan reads r1 = bf16(x - c_list) against
per-(query, list) pair operands and keeps lower-bound keys; results must stay bit-identical to the
exact oracle (ids and distances) at every batch shape the scan variants cover (16-query tiles with a
streamed or resident operand, 32-query tiles incl. half-N tiles), with fallbacks counted."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RD_STORE_F32_RESID = (3, 4)  # bf16 / fp16 residual plane


@pytest.fixture(params=["bf16", "fp16"])
def resid_env(monkeypatch, request):
    """bf16 residual plane with the bf16 (q1; q2) operand, or the fp16 plane with fp16(q) alone (RD_RES16=1)."""
    monkeypatch.setenv("RD_STORE", "resid")
    monkeypatch.setenv("RD_RES16", "1" if request.param == "fp16" else "0")


def _check(engine, oracle, desc, B, nprobe, k, q0=0):
    q, src = engine.synth_queries(desc, q0, B)
    idx = engine.synthetic_index(desc)
    try:
        assert idx.info()["store"] in RD_STORE_F32_RESID
        e = idx.search(q, nprobe, k)
    finally:
        idx.close()
    o = oracle.synthetic_index(desc).search(q, nprobe, k)
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)
    assert e.stats["probe_failures"] == 0
    return e


@pytest.mark.parametrize("B", [1, 2, 8, 33, 128, 512])
def test_resid_matches_oracle(engine, oracle, resid_env, B):
    desc = engine.desc(n=200_000, d=768, nlist=256)
    e = _check(engine, oracle, desc, B, nprobe=16, k=10)
    assert e.stats["margin_failures"] <= max(1, B // 50)


@pytest.mark.parametrize("d", [128, 256, 384])
def test_resid_small_d(engine, oracle, resid_env, d):
    desc = engine.desc(n=50_000, d=d, nlist=64)
    _check(engine, oracle, desc, 64, nprobe=8, k=10)


@pytest.mark.parametrize("k", [1, 20])
def test_resid_k(engine, oracle, resid_env, k):
    desc = engine.desc(n=100_000, d=768, nlist=128)
    _check(engine, oracle, desc, 64, nprobe=16, k=k)


def test_resid_c1_full(engine, oracle, resid_env):
    from bench import CONFIGS
    c = CONFIGS["c1"]
    desc = engine.desc(c["n"], c["d"], c["nlist"])
    e = _check(engine, oracle, desc, c["batch"], c["nprobe"], c["k"])
    assert e.stats["margin_failures"] == 0


def test_fp16_overflow_keeps_the_bf16_plane_and_exactness(engine, oracle, monkeypatch):
    """Rows whose residuals leave fp16's range build the bf16 residual plane instead; queries whose
    components overflow fp16 give non-finite dots, keys of -inf, a failed certificate and the exact
    fallback: results stay the oracle's either way."""
    monkeypatch.setenv("RD_STORE", "resid")
    monkeypatch.setenv("RD_RES16", "1")
    rng = np.random.default_rng(11)
    X = rng.standard_normal((4000, 128)).astype(np.float32)
    X[:2000] *= np.float32(2e5)  # list 0: residuals beyond fp16's 65504
    offs = np.array([0, 2000, 4000], np.int64)
    C = np.stack([X[:2000].mean(0), X[2000:].mean(0)]).astype(np.float32)
    Q = (X[2000:2016] + 0.01).astype(np.float32)
    e = engine.index_from_host(X, offs, C)
    assert e.info()["store"] == 3  # residuals beyond fp16's range: the bf16 plane
    r = e.search(Q, 2, 10)
    o = oracle.index_from_host(X, offs, C).search(Q, 2, 10)
    np.testing.assert_array_equal(r.ids, o.ids)
    np.testing.assert_array_equal(r.dists, o.dists)
    # normal rows, queries with a component beyond fp16's range
    X2 = rng.standard_normal((4000, 128)).astype(np.float32)
    C2 = np.stack([X2[:2000].mean(0), X2[2000:].mean(0)]).astype(np.float32)
    Q2 = (X2[:16] + 0.01).astype(np.float32)
    Q2[:4, 3] = np.float32(1e6)
    e2 = engine.index_from_host(X2, offs, C2)
    r2 = e2.search(Q2, 2, 10)
    o2 = oracle.index_from_host(X2, offs, C2).search(Q2, 2, 10)
    np.testing.assert_array_equal(r2.ids, o2.ids)
    np.testing.assert_array_equal(r2.dists, o2.dists)
    assert r2.stats["margin_failures"] >= 4
