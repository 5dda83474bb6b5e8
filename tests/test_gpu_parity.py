"""GPU parity: the B200 engine (librd_b200.so, called through the C-ABI)
against the CPU oracle on the same seeded inputs. The bar is bit-exact: the
engine reranks its candidates with the canonical exact distance, so ids and
distances must be identical to the oracle's, and every query's candidate
margin and probe set must be certified (SURVEY §8c parity rule, tolerance
1e-5 relative for distances is implied by bit equality)."""
import os

import numpy as np
import pytest

import numpy_ref as R
from make_golden import CASES

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "ivf_small.npz"))


def _check(res, want_ids, want_d):
    from conftest import fallbacks_allowed
    np.testing.assert_array_equal(res.ids, want_ids)
    np.testing.assert_array_equal(res.dists, want_d)
    assert res.stats["margin_failures"] <= fallbacks_allowed(*res.ids.shape)
    assert res.stats["probe_failures"] == 0


@pytest.mark.parametrize("name", list(CASES))
def test_engine_matches_golden(engine, name):
    c = CASES[name]
    desc = engine.desc(c["n"], c["d"], c["nlist"], shard=c.get("shard", 0), num_shards=c.get("num_shards", 1))
    idx = engine.synthetic_index(desc)
    offs, ids, _ = idx.layout()
    np.testing.assert_array_equal(offs, GOLD[f"{name}/offs"])
    q = GOLD[f"{name}/queries"]
    np.testing.assert_array_equal(idx.probe(q, c["nprobe"]), GOLD[f"{name}/probes"])
    _check(idx.search(q, c["nprobe"], c["k"]), GOLD[f"{name}/out_ids"], GOLD[f"{name}/out_dists"])


@pytest.mark.parametrize("store", ["resid", "split3", "fp32"])
@pytest.mark.parametrize("B,nprobe,k", [(1, 8, 10), (7, 1, 1), (32, 16, 10), (100, 64, 20), (33, 5, 24),
                                        (256, 16, 10), (300, 3, 24)])
def test_engine_vs_oracle_synthetic(engine, oracle, B, nprobe, k, store, monkeypatch):
    # resid: the residual scan (default); split3: the scan over the x1 | x2 plane; fp32: the
    # converter-warp scan over fp32 rows
    if store != "resid":
        monkeypatch.setenv("RD_STORE", "split3")
    if store == "fp32":
        monkeypatch.setenv("RD_SPLIT3", "0")
        monkeypatch.setenv("RD_PRESPLIT", "0")
    n, d, nlist = 40000, 768, 64
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 1000, B)
    e = engine.synthetic_index(desc).search(q, nprobe, k)
    o = oracle.synthetic_index(desc).search(q, nprobe, k)
    _check(e, o.ids, o.dists)


@pytest.mark.parametrize("B,nprobe", [(1, 64), (8, 64), (6, 100), (16, 64), (17, 64), (64, 64), (128, 64),
                                      (200, 64)])
def test_engine_vs_oracle_many_lists(engine, oracle, B, nprobe):
    # nlist 4096 (the C2 coarse size): small-batch GEMV coarse (B <= 8), tensor-core coarse, the
    # sorted-pairs plan (B * nprobe <= 512), the single-CTA bitmap plan (B <= 8, more pairs), the
    # multi-kernel plan, smem-staged select / rerank (B <= 2 x SMs)
    n, d, nlist = 200000, 768, 4096
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 7, B)
    e = engine.synthetic_index(desc).search(q, nprobe, 10)
    o = oracle.synthetic_index(desc).search(q, nprobe, 10)
    _check(e, o.ids, o.dists)


def test_engine_generator_bit_exact(engine, oracle):
    desc = engine.desc(5000, 96, 17)
    ei = engine.synthetic_index(desc)
    oi = oracle.synthetic_index(desc)
    eo, eids, _ = ei.layout()
    oo, oids, _ = oi.layout()
    np.testing.assert_array_equal(eo, oo)
    np.testing.assert_array_equal(eids, oids)
    # vectors: search with nprobe = nlist and k = n returns exact distances to every vector
    q, _ = engine.synth_queries(desc, 0, 3)
    want = R.vectors_of(oids[:50], 96, 17)
    np.testing.assert_array_equal(want, np.stack([engine.synth_vector(desc, int(i)) for i in oids[:50]]))
    _check(ei.search(q, 17, 24), *[getattr(oi.search(q, 17, 24), a) for a in ("ids", "dists")])


def test_from_host_ties_duplicates_empty_lists(engine, oracle):
    rng = np.random.default_rng(3)
    d, nlist = 64, 12
    lens = np.array([0, 5, 0, 700, 3, 0, 400, 1, 9, 0, 260, 33])
    n = int(lens.sum())
    X = rng.integers(-2, 3, size=(n, d)).astype(np.float32)
    X[5:40] = X[0]  # exact duplicates -> equal distances, id order decides
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    C = rng.integers(-2, 3, size=(nlist, d)).astype(np.float32)
    ids = (rng.permutation(n).astype(np.int64) * 7 + 5)
    Q = np.concatenate([X[:3], rng.integers(-2, 3, size=(9, d)).astype(np.float32)])
    for nprobe, k in [(nlist, 24), (3, 10), (1, 24)]:
        e = engine.index_from_host(X, offs, C, ids).search(Q, nprobe, k)
        o = oracle.index_from_host(X, offs, C, ids).search(Q, nprobe, k)
        np.testing.assert_array_equal(e.ids, o.ids)
        np.testing.assert_array_equal(e.dists, o.dists)


@pytest.mark.parametrize("frac,B", [(0.5, 48), (1.0, 48), (0.5, 2), (0.5, 8)])
def test_offloaded_lists_same_results(engine, oracle, frac, B):
    # B 2 / 8: the sorted-pairs planner with offloaded lists (their pairs get no device tiles)
    n, d, nlist, nprobe, k = 60000, 768, 64, 16, 10
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 77, B)
    idx = engine.synthetic_index(desc)
    idx.place(offload_fraction=frac, staging_slots=2)
    info = idx.info()
    assert info["lists_resident"] == nlist - int(np.floor(frac * nlist + 0.5))
    e = idx.search(q, nprobe, k)
    assert e.stats["h2d_list_bytes"] > 0
    o = oracle.synthetic_index(desc).search(q, nprobe, k)
    _check(e, o.ids, o.dists)
    idx.place(offload_fraction=0.0)  # back to fully resident between searches
    _check(idx.search(q, nprobe, k), o.ids, o.dists)


def test_device_shard_merge(engine):
    import torch
    rng = np.random.default_rng(5)
    G, B, k = 4, 50, 10
    d = np.sort(rng.random((G, B, k)).astype(np.float32), axis=2)
    ids = rng.integers(0, 1 << 40, size=(G, B, k)).astype(np.int64)
    ids[1, :, 5:] = -1
    want_i, want_d = engine.merge_topk(ids, d)
    ti, td = torch.from_numpy(ids).cuda(), torch.from_numpy(d).cuda()
    oi = torch.empty((B, k), dtype=torch.int64, device="cuda")
    od = torch.empty((B, k), dtype=torch.float32, device="cuda")
    engine.check(engine.lib.rd_merge_topk_device(G, B, k, ti.data_ptr(), td.data_ptr(), oi.data_ptr(),
                                                 od.data_ptr(), None))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(oi.cpu().numpy(), want_i)
    np.testing.assert_array_equal(od.cpu().numpy(), want_d)


def test_k_above_fast_path_is_exact(engine, oracle):
    # k > 24 leaves the certified fast path for the exact large-k pass (wide.cu): same results
    desc = engine.desc(2000, 64, 8)
    q, _ = engine.synth_queries(desc, 0, 2)
    e = engine.synthetic_index(desc).search(q, 4, 25)
    o = oracle.synthetic_index(desc).search(q, 4, 25)
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)


def test_search_device_matches_host_path(engine):
    import torch
    desc = engine.desc(30000, 768, 64)
    idx = engine.synthetic_index(desc)
    q, _ = engine.synth_queries(desc, 5, 64)
    h = idx.search(q, 8, 10)
    dq = torch.from_numpy(q).cuda()
    di = torch.empty((64, 10), dtype=torch.int64, device="cuda")
    dd = torch.empty((64, 10), dtype=torch.float32, device="cuda")
    st = idx.search_device(dq.data_ptr(), 64, 8, 10, di.data_ptr(), dd.data_ptr(),
                           stream=torch.cuda.current_stream().cuda_stream, sync=True)
    assert st["margin_failures"] == 0
    np.testing.assert_array_equal(di.cpu().numpy(), h.ids)
    np.testing.assert_array_equal(dd.cpu().numpy(), h.dists)


def test_search_into_pinned_buffers(engine):
    import torch
    desc = engine.desc(30000, 768, 64)
    idx = engine.synthetic_index(desc)
    q, _ = engine.synth_queries(desc, 9, 40)
    want = idx.search(q, 8, 10)
    hq = torch.from_numpy(q).pin_memory().numpy()
    hi = torch.empty((40, 10), dtype=torch.int64).pin_memory().numpy()
    hd = torch.empty((40, 10), dtype=torch.float32).pin_memory().numpy()
    idx.search_into(hq, 8, 10, hi, hd)
    np.testing.assert_array_equal(hi, want.ids)
    np.testing.assert_array_equal(hd, want.dists)


@pytest.mark.parametrize("variant", [dict(RD_TC_G="16", RD_STREAM_B="1"), dict(RD_TC_G="16", RD_STREAM_B="0"),
                                     dict(RD_TC_G="32"), dict(RD_TC_G="1", RD_STREAM_B="1"),
                                     dict(RD_TC_G="1", RD_STREAM_B="0")])
def test_every_scan_variant(engine, oracle, variant, monkeypatch):
    # one dataset through each tensor-core scan variant (16-query tiles with a streamed or resident
    # query operand, 32-query tiles, mixed widths): lists probed by 1..40 queries, so tiles of one,
    # a few and more than 16 / 32 queries all occur
    for kname, v in variant.items():
        monkeypatch.setenv(kname, v)
    n, d, nlist = 60000, 768, 96
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 321, 150)
    e = engine.synthetic_index(desc).search(q, 12, 10)
    o = oracle.synthetic_index(desc).search(q, 12, 10)
    _check(e, o.ids, o.dists)
    assert e.stats["margin_failures"] == 0 and e.stats["probe_failures"] == 0


def test_timing_stages(engine):
    # per-stage device times only while rd_timing_stages is on; whole-search times always; results
    # identical either way (the events sit between kernels, they do not change the work)
    desc = engine.desc(30000, 768, 64)
    idx = engine.synthetic_index(desc)
    q, _ = engine.synth_queries(desc, 3, 32)
    idx.timing_reset()
    off = idx.search(q, 8, 10)
    t = idx.timing_read()
    assert off.stats["scan_ms"] == 0.0 and t["searches"] == 1 and t["stage_searches"] == 0
    assert t["total_ms"] > 0.0 and t["scan_ms"] == 0.0
    idx.timing_stages(True)
    idx.timing_reset()
    on = idx.search(q, 8, 10)
    idx.search(q, 8, 10)
    t = idx.timing_read()
    idx.timing_stages(False)
    assert on.stats["scan_ms"] > 0.0 and t["searches"] == 2 and t["stage_searches"] == 2
    assert 0.0 < t["scan_ms"] < t["total_ms"]
    np.testing.assert_array_equal(on.ids, off.ids)
    np.testing.assert_array_equal(on.dists, off.dists)


@pytest.mark.parametrize("margin", ["8", "22"])
def test_duplicate_heavy_data(engine, oracle, margin, monkeypatch):
    # a corpus where each query's neighbourhood holds many exact duplicates: ties across ranks
    # k..k+margin defeat the candidate margin and send queries to the exact fallback (a wider
    # margin needs more duplicates to do so); results are the oracle's either way
    monkeypatch.setenv("RD_RERANK_MARGIN", margin)
    rng = np.random.default_rng(5)
    d, nlist = 128, 16
    C = rng.standard_normal((nlist, d)).astype(np.float32)
    base = (C[rng.integers(0, nlist, 600)] + 0.3 * rng.standard_normal((600, d))).astype(np.float32)
    X = np.repeat(base, 24, axis=0)  # every vector 24 times: ties span ranks 1..24
    assign = np.argmin(((X[:, None, :] - C[None]) ** 2).sum(-1), axis=1)
    order = np.argsort(assign, kind="stable")
    X = X[order]
    offs = np.concatenate([[0], np.cumsum(np.bincount(assign, minlength=nlist))]).astype(np.int64)
    Q = (base[:40] + 0.01 * rng.standard_normal((40, d))).astype(np.float32)
    e = engine.index_from_host(X, offs, C).search(Q, 3, 10)
    o = oracle.index_from_host(X, offs, C).search(Q, 3, 10)
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)
    if margin == "8":  # 18 reranked, the 19th ties the 10th: every query falls back to exact
        assert e.stats["margin_failures"] == len(Q)
    else:  # 32 reranked, the 33rd is another vector: certified without the fallback
        assert e.stats["margin_failures"] == 0


@pytest.mark.parametrize("store", ["resid", "split3"])
@pytest.mark.parametrize("n,nlist,B,nprobe", [(200000, 64, 300, 16), (60000, 32, 97, 8), (300000, 128, 1024, 24)])
def test_pair_scan_matches_oracle(engine, oracle, monkeypatch, n, nlist, B, nprobe, store):
    """The paired-CTA wide scan (scan_pair.cu, tcgen05 cta_group::2; opt-in RD_PAIR=1) over either
    store: lists probed by > 8 queries on average take 32-query tiles on CTA pairs, including lists
    whose last 256-row block leaves the peer CTA no rows; bit-exact against the oracle."""
    monkeypatch.setenv("RD_PAIR", "1")  # read when the index is created
    monkeypatch.setenv("RD_STORE", store)
    desc = engine.desc(n, 768, nlist)
    q, _ = engine.synth_queries(desc, 11, B)
    r = engine.synthetic_index(desc).search(q, nprobe, 10)
    o = oracle.synthetic_index(desc).search(q, nprobe, 10)
    _check(r, o.ids, o.dists)
    assert r.stats["margin_failures"] == 0
