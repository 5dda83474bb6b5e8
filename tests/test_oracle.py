"""The CPU oracle (oracle/librd_cpu.so) pinned against the independent numpy
restatement's golden vectors (tests/golden/ivf_small.npz, made by
tests/make_golden.py) and against tests/numpy_ref.py directly. The reference
has no IVF implementation, so IVF parity is unpinned by the
reference itself; this is the strongest available anchor."""
import os

import numpy as np
import pytest

import numpy_ref as R
from make_golden import CASES

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ivf_small.npz"))


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_matches_golden(oracle, name):
    c = CASES[name]
    desc = oracle.desc(c["n"], c["d"], c["nlist"], shard=c.get("shard", 0), num_shards=c.get("num_shards", 1))
    idx = oracle.synthetic_index(desc)
    offs, ids, _ = idx.layout()
    np.testing.assert_array_equal(offs, GOLD[f"{name}/offs"])
    np.testing.assert_array_equal(ids[:64], GOLD[f"{name}/ids_head"][: len(ids[:64])])
    q, src = oracle.synth_queries(desc, 0, c["B"])
    np.testing.assert_array_equal(q, GOLD[f"{name}/queries"])  # bit-exact data
    np.testing.assert_array_equal(src, GOLD[f"{name}/src"])
    np.testing.assert_array_equal(idx.probe(q, c["nprobe"]), GOLD[f"{name}/probes"])
    r = idx.search(q, c["nprobe"], c["k"])
    np.testing.assert_array_equal(r.ids, GOLD[f"{name}/out_ids"])
    np.testing.assert_array_equal(r.dists, GOLD[f"{name}/out_dists"])


def test_engine_host_generator_matches(engine_lib, oracle):
    desc = oracle.desc(6000, 768, 64)
    for lib in (engine_lib, oracle):
        q, src = lib.synth_queries(desc, 0, 12)
        np.testing.assert_array_equal(q, GOLD["c1s/queries"])
        np.testing.assert_array_equal(lib.synth_vector(desc, 0), R.vectors_of([0], 768, 64)[0])


def test_exact_l2_canonical(engine_lib, oracle):
    rng = np.random.default_rng(1)
    for d in (8, 64, 768, 1000):
        a = rng.standard_normal(d).astype(np.float32) * 3
        b = rng.standard_normal(d).astype(np.float32)
        e = oracle.exact_l2(a, b)
        assert e == engine_lib.exact_l2(a, b)
        if d % 8 == 0:
            assert e == R.exact_l2(a, b[None, :])[0]
        assert e == pytest.approx(float(np.sum((a.astype(np.float64) - b) ** 2)), rel=1e-6)


def test_from_host_with_ties_and_empty_lists(oracle):
    rng = np.random.default_rng(7)
    d, nlist = 32, 10
    lens = np.array([0, 5, 0, 17, 3, 0, 40, 1, 9, 0])
    n = int(lens.sum())
    X = rng.integers(-2, 3, size=(n, d)).astype(np.float32)  # many exact ties
    X[5:10] = X[0]  # duplicates
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    C = rng.integers(-2, 3, size=(nlist, d)).astype(np.float32)
    ids = rng.permutation(n).astype(np.int64) * 3 + 11
    idx = oracle.index_from_host(X, offs, C, ids)
    Q = rng.integers(-2, 3, size=(6, d)).astype(np.float32)
    r = idx.search(Q, nprobe=nlist, k=25)
    wi, wd, _ = R.ivf_search(X, offs, C, ids, Q, nlist, 25)
    np.testing.assert_array_equal(r.ids, wi)
    np.testing.assert_array_equal(r.dists, wd)
    # fewer candidates than k -> (-1, inf) padding
    r2 = idx.search(Q, nprobe=1, k=50)
    assert (r2.ids == -1).any() and np.isinf(r2.dists[r2.ids == -1]).all()


def test_invalid_arguments_raise_parse_error(oracle):
    from paper_2504_15302_b200.retriever import ParseError
    with pytest.raises(ParseError):
        oracle.synthetic_index(oracle.desc(0, 8, 1))
    idx = oracle.synthetic_index(oracle.desc(100, 8, 4))
    with pytest.raises(ParseError):
        idx.search(np.zeros((1, 8), np.float32), nprobe=0, k=1)


@pytest.mark.parametrize("G,mask", [(1, 1), (4, 0b0101), (8, 0b11), (3, 0b111)])
def test_sampled_synth_search_matches_materialised_stripes(oracle, G, mask):
    # rd_oracle_synth_search (vectors regenerated from (seed, id), nothing materialised) equals the
    # merge of the materialised oracle stripes it selects
    from oracle_ext import synth_search
    n, d, nlist, nprobe, k = 30000, 64, 40, 6, 12
    desc = oracle.desc(n, d, nlist, num_shards=G)
    q, _ = oracle.synth_queries(desc, 11, 9)
    got_i, got_d = synth_search(oracle, desc, q, nprobe, k, mask)
    parts = [oracle.synthetic_index(oracle.desc(n, d, nlist, shard=g, num_shards=G)).search(q, nprobe, k)
             for g in range(G) if (mask >> g) & 1]
    want_i, want_d = oracle.merge_topk(np.stack([p.ids for p in parts]), np.stack([p.dists for p in parts]))
    np.testing.assert_array_equal(got_i, want_i)
    np.testing.assert_array_equal(got_d, want_d)
