"""Certification under adversarial data (DESIGN.md §2 "Certification"): the tensor-core scan's
bf16x3 split drops x2.q2 and the split residuals, up to 2^-15 of sum |x_t q_t| independently of d.
Vectors with large norms, aligned signs and split-boundary components (residuals just under half a
bf16 ulp) make that error ~16 in squared distance at d = 64, beyond the FFMA scan's (d/2 + 8) u bound
the merge used before round 2: the true nearest row then ranks past the rerank set while the
certificate still held, a silently wrong top-k. With the per-path bound the query goes to the
exact fallback and the result is the oracle's, bit for bit (fallbacks are allowed and counted)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def split_boundary_index(G, d, ndec):
    """G lists; list g: the query's own vector A (components b_g + r1, r1 with the largest bf16x3
    residual) and ndec decoys with bf16-exact components (no residual) at exact distances
    ~4.0 + 0.5 j, all farther than A (distance 0) but ranked ahead of it by the approximation."""
    r1 = np.float32(0.25 - 2 ** -10 + 2 ** -11 - 2 ** -17)
    X, Q, C, offs = [], [], [], [0]
    for g in range(G):
        b = np.float32(64 + 4 * g)
        q = np.full(d, b + r1, np.float32)
        rows = [q.copy()]
        for j in range(ndec):
            v = np.full(d, b, np.float32)
            v[: j % d] = b + 1.0
            rows.append(v)
        X += rows
        Q.append(q)
        C.append(np.mean(rows, 0).astype(np.float32))
        offs.append(len(X))
    return np.array(X, np.float32), np.array(offs, np.int64), np.array(C, np.float32), np.array(Q, np.float32)


@pytest.mark.parametrize("store", ["split3", "resid"])
@pytest.mark.parametrize("d,k", [(64, 1), (64, 5), (128, 10), (768, 1)])
def test_split_boundary_near_ties_exact(engine, oracle, d, k, store, monkeypatch):
    # split3: the x1 | x2 scan the data is built against; resid: the residual scan over the same rows
    # (its keys are lower bounds, so the certificate holds or the fallback runs)
    monkeypatch.setenv("RD_STORE", store)
    X, offs, C, Q = split_boundary_index(8, d, ndec=k + 11)
    e = engine.index_from_host(X, offs, C).search(Q, 1, k)
    o = oracle.index_from_host(X, offs, C).search(Q, 1, k)
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)
    assert (e.ids[:, 0] == offs[:-1]).all()  # each query's own vector A is its nearest
    if d == 64 and store == "split3":  # the approximation ranks A past the rerank set: only the fallback finds it
        assert e.stats["margin_failures"] > 0


@pytest.mark.parametrize("store", ["split3", "resid"])
@pytest.mark.parametrize("B", [1, 64])
def test_split_boundary_coarse_and_seed(engine, oracle, B, store, monkeypatch):
    """The same data through every coarse path (GEMV at B <= 8, tensor-core GEMM above) with
    nprobe > 1, so the coarse certificate and the seeded pruning threshold see it too."""
    monkeypatch.setenv("RD_STORE", store)
    X, offs, C, Q = split_boundary_index(16, 64, ndec=20)
    Qb = np.repeat(Q, (B + len(Q) - 1) // len(Q), axis=0)[:B]
    e = engine.index_from_host(X, offs, C).search(Qb, 3, 10)
    o = oracle.index_from_host(X, offs, C).search(Qb, 3, 10)
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)
