"""Arguments beyond the fast path (wide.cu): any k up to 256 (the reference's Request::top_k is any
k >= 1, core/include/ragsim/domain.hpp:84-90, domain.cpp:127) through the exact query-major pass,
and nprobe up to nlist through the all-centroid exact selection — bit-exact against the oracle,
which takes the same arguments."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(e, o):
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)


@pytest.mark.parametrize("B,nprobe,k", [(1, 8, 25), (7, 16, 64), (100, 6, 128), (3, 40, 256), (33, 3, 100)])
def test_large_k(engine, oracle, B, nprobe, k):
    desc = engine.desc(60000, 256, 128)
    q, _ = engine.synth_queries(desc, 2 * k + B, B)
    _same(engine.synthetic_index(desc).search(q, nprobe, k), oracle.synthetic_index(desc).search(q, nprobe, k))


@pytest.mark.parametrize("nprobe,k", [(481, 10), (1024, 10), (2048, 20), (700, 64)])
def test_large_nprobe(engine, oracle, nprobe, k):
    desc = engine.desc(100000, 128, 2048)
    q, _ = engine.synth_queries(desc, 9, 48)
    _same(engine.synthetic_index(desc).search(q, nprobe, k), oracle.synthetic_index(desc).search(q, nprobe, k))


def test_large_nprobe_probe_order(engine, oracle):
    desc = engine.desc(40000, 64, 1024)
    q, _ = engine.synth_queries(desc, 4, 20)
    np.testing.assert_array_equal(engine.synthetic_index(desc).probe(q, 600), oracle.synthetic_index(desc).probe(q, 600))


def test_large_k_offloaded_and_fp32_store(engine, oracle, monkeypatch):
    desc = engine.desc(50000, 768, 64)
    q, _ = engine.synth_queries(desc, 1, 12)
    want = oracle.synthetic_index(desc).search(q, 10, 96)
    e = engine.synthetic_index(desc)
    e.place(offload_fraction=0.5)
    _same(e.search(q, 10, 96), want)
    monkeypatch.setenv("RD_STORE", "split3")
    monkeypatch.setenv("RD_SPLIT3", "0")
    _same(engine.synthetic_index(desc).search(q, 10, 96), want)


def test_large_k_duplicates_order_by_id(engine, oracle):
    rng = np.random.default_rng(8)
    base = rng.standard_normal((300, 64)).astype(np.float32)
    X = np.repeat(base, 10, axis=0)  # every vector ten times: ties broken by id
    offs = np.array([0, 1500, 3000], np.int64)
    C = np.stack([X[:1500].mean(0), X[1500:].mean(0)]).astype(np.float32)
    Q = base[:9] + np.float32(0.001)
    _same(engine.index_from_host(X, offs, C).search(Q, 2, 200), oracle.index_from_host(X, offs, C).search(Q, 2, 200))


def test_k_beyond_limit_rejected(engine):
    from paper_2504_15302_b200.retriever import ParseError
    desc = engine.desc(5000, 64, 8)
    q, _ = engine.synth_queries(desc, 0, 2)
    with pytest.raises(ParseError):
        engine.synthetic_index(desc).search(q, 2, 257)
