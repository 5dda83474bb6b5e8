"""IVF training (rd_index_build): exact, deterministic Lloyd's k-means.
The oracle is checked against a numpy restatement on CPU; on the GPU the engine (which assigns
with its own tensor-core coarse path + certified selection) must reproduce the oracle's centroids,
list membership and search results bit for bit."""
import numpy as np
import pytest

import numpy_ref as R
from paper_2504_15302_b200.retriever import ParseError


def _numpy_kmeans(X, nlist, iters, init_rows):
    C = X[init_rows].copy()
    for it in range(iters + 1):
        dist = np.stack([R.exact_l2(c, X) for c in C], axis=1)  # canonical exact distances
        assign = np.argmin(dist, axis=1)  # first minimum: ties keep the lower id
        if it == iters:
            return C, assign
        for j in range(nlist):
            m = np.flatnonzero(assign == j)
            if m.size:
                s = np.zeros(X.shape[1])
                for r in m:  # ascending rows, fp64
                    s = s + X[r].astype(np.float64)
                C[j] = (s / m.size).astype(np.float32)


def _init_rows(lib, n, nlist, seed):
    s = lib.derive_seed(seed, 0x1006)
    rows, i = [], 0
    while len(rows) < nlist:
        r = lib.splitmix_at(s, i) % n
        i += 1
        if r not in rows:
            rows.append(r)
    return np.array(rows)


def _blobs(n, d, k, seed=0):
    rng = np.random.default_rng(seed)
    centers = rng.integers(-8, 9, size=(k, d)).astype(np.float32)
    X = centers[rng.integers(0, k, n)] + rng.standard_normal((n, d)).astype(np.float32)
    return X.astype(np.float32)


def test_oracle_build_matches_numpy(oracle):
    X = _blobs(600, 16, 5)
    nlist, iters, seed = 6, 3, 11
    idx = oracle.build_index(X, nlist, iters, seed)
    C, assign = _numpy_kmeans(X, nlist, iters, _init_rows(oracle, len(X), nlist, seed))
    np.testing.assert_array_equal(idx.centroids(), C)
    offs, ids, _ = idx.layout()
    np.testing.assert_array_equal(np.diff(offs), np.bincount(assign, minlength=nlist))
    order = np.argsort(assign, kind="stable")  # list order, ascending row within a list
    np.testing.assert_array_equal(ids, order)


def test_oracle_build_ids_and_validation(oracle):
    X = _blobs(300, 8, 3)
    ids = np.arange(300, dtype=np.int64) * 10 + 7
    idx = oracle.build_index(X, 4, 2, ids=ids)
    r = idx.search(X[:5], 4, 1)
    np.testing.assert_array_equal(r.ids[:, 0], ids[:5])
    with pytest.raises(ParseError):
        oracle.build_index(X[:3], 4, 1)  # n < nlist


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,nlist,iters", [(20000, 64, 32, 4), (30000, 768, 64, 3), (5000, 96, 16, 5)])
def test_engine_build_matches_oracle(engine, oracle, n, d, nlist, iters):
    X = _blobs(n, d, nlist // 2, seed=n)
    e = engine.build_index(X, nlist, iters, seed=5)
    o = oracle.build_index(X, nlist, iters, seed=5)
    np.testing.assert_array_equal(e.centroids(), o.centroids())
    eo, ei, _ = e.layout()
    oo, oi, _ = o.layout()
    np.testing.assert_array_equal(eo, oo)
    np.testing.assert_array_equal(ei, oi)
    q = X[::max(1, n // 40)][:40] + 0.01
    a, b = e.search(q, 4, 10), o.search(q, 4, 10)
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dists, b.dists)
