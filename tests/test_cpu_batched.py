"""The batched CPU baseline (oracle/rd_cpu_batched.c, bench.py's cpu_baseline kind "batched") returns
the exact oracle's results bit for bit: certified fp32 ranking, canonical rerank, exact fallback."""
import numpy as np
import pytest

from oracle_ext import batched_search


@pytest.mark.parametrize("n,d,nlist,B,nprobe,k", [
    (20000, 64, 32, 17, 4, 10),
    (30000, 96, 64, 40, 8, 1),
    (12000, 770, 16, 9, 3, 24),   # d % 8 != 0: scalar tails
    (5000, 32, 64, 5, 64, 33),    # nprobe = nlist, k > 32
    (3000, 128, 200, 3, 7, 5),    # lists shorter than the rerank set, empty lists
])
def test_batched_equals_oracle(oracle, n, d, nlist, B, nprobe, k):
    desc = oracle.desc(n, d, nlist)
    idx = oracle.synthetic_index(desc)
    q, _ = oracle.synth_queries(desc, 0, B)
    want = idx.search(q, nprobe, k)
    ids, dists, fb = batched_search(oracle, idx, q, nprobe, k)
    np.testing.assert_array_equal(ids, want.ids)
    np.testing.assert_array_equal(dists, want.dists)
    assert fb == 0  # synthetic data: every query certified


def test_batched_duplicates_fall_back_exactly(oracle):
    """Exact duplicates across ranks k..m tie the certificate: those queries take the exact path."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal((300, 48)).astype(np.float32)
    vecs = np.repeat(base, 20, axis=0)  # every vector 20 times
    offs = np.linspace(0, len(vecs), 9).astype(np.int64)
    idx = oracle.index_from_host(vecs, offs, rng.standard_normal((8, 48)).astype(np.float32))
    q = base[:12] + 0.01 * rng.standard_normal((12, 48)).astype(np.float32)
    want = idx.search(q, 3, 10)
    ids, dists, fb = batched_search(oracle, idx, q, 3, 10)
    np.testing.assert_array_equal(ids, want.ids)
    np.testing.assert_array_equal(dists, want.dists)
    assert fb > 0
