"""The residual store (RD_STORE=resid, csrc/resid.cu): the scan reads r1 = bf16(x - c_list) against
per-(query, list) pair operands and keeps lower-bound keys; results must stay bit-identical to the
exact oracle (ids and distances) at every batch shape the scan variants cover (16-query tiles with a
streamed or resident operand, 32-query tiles incl. half-N tiles), with fallbacks counted."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RD_STORE_F32_RESID = 3


@pytest.fixture()
def resid_env(monkeypatch):
    monkeypatch.setenv("RD_STORE", "resid")


def _check(engine, oracle, desc, B, nprobe, k, q0=0):
    q, src = engine.synth_queries(desc, q0, B)
    idx = engine.synthetic_index(desc)
    try:
        assert idx.info()["store"] == RD_STORE_F32_RESID
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
