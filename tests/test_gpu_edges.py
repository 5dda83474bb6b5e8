"""GPU edge cases against the oracle: dimension limits (FFMA paths at d % 64 != 0, the
largest d), nprobe beyond nlist, a single list, fewer candidates than k, empty batches,
scaled data, and the engine's argument validation (ragsim ParseError, exit code 2)."""
import numpy as np
import pytest

from paper_2504_15302_b200.retriever import ParseError

pytestmark = pytest.mark.gpu


def _same(e, o):
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)  # exact fallbacks may run; results must not differ


@pytest.mark.parametrize("d", [32, 96, 1024])
def test_dimension_limits(engine, oracle, d):
    desc = engine.desc(12000, d, 24)
    q, _ = engine.synth_queries(desc, 3, 20)
    _same(engine.synthetic_index(desc).search(q, 5, 10), oracle.synthetic_index(desc).search(q, 5, 10))


def test_nprobe_beyond_nlist_and_single_list(engine, oracle):
    desc = engine.desc(3000, 128, 9)
    q, _ = engine.synth_queries(desc, 0, 7)
    e, o = engine.synthetic_index(desc), oracle.synthetic_index(desc)
    _same(e.search(q, 50, 12), o.search(q, 50, 12))  # every list probed
    pe, po = e.probe(q, 12), o.probe(q, 12)
    np.testing.assert_array_equal(pe, po)
    assert (pe[:, 9:] == -1).all()
    one = engine.desc(2000, 64, 1)
    q1, _ = engine.synth_queries(one, 0, 5)
    _same(engine.synthetic_index(one).search(q1, 1, 24), oracle.synthetic_index(one).search(q1, 1, 24))


def test_fewer_candidates_than_k(engine, oracle):
    rng = np.random.default_rng(11)
    d, nlist = 64, 6
    lens = np.array([3, 0, 5, 0, 2, 1])
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    X = rng.standard_normal((int(lens.sum()), d)).astype(np.float32)
    C = rng.standard_normal((nlist, d)).astype(np.float32)
    Q = rng.standard_normal((4, d)).astype(np.float32)
    e = engine.index_from_host(X, offs, C).search(Q, 2, 20)
    o = oracle.index_from_host(X, offs, C).search(Q, 2, 20)
    _same(e, o)
    assert (e.ids == -1).any() and np.isinf(e.dists[e.ids == -1]).all()


def test_empty_batch_and_scaled_data(engine, oracle):
    desc = engine.desc(5000, 128, 16)
    idx = engine.synthetic_index(desc)
    r = idx.search(np.zeros((0, 128), np.float32), 4, 10)
    assert r.ids.shape == (0, 10)
    rng = np.random.default_rng(2)
    for scale in (1e-3, 1e3):  # the certification bounds scale with ||q|| and max ||x||
        X = (rng.standard_normal((4000, 128)) * scale).astype(np.float32)
        offs = np.linspace(0, 4000, 9).astype(np.int64)
        C = np.stack([X[offs[i]:offs[i + 1]].mean(0) for i in range(8)]).astype(np.float32)
        Q = (X[:25] + rng.standard_normal((25, 128)).astype(np.float32) * 0.1 * scale).astype(np.float32)
        _same(engine.index_from_host(X, offs, C).search(Q, 3, 10), oracle.index_from_host(X, offs, C).search(Q, 3, 10))


def test_engine_argument_validation(engine):
    idx = engine.synthetic_index(engine.desc(2000, 64, 8))
    q = np.zeros((2, 64), np.float32)
    for nprobe, k in [(0, 10), (4, 0), (4, 257)]:  # k <= 256: the exact large-k pass's widest lists
        with pytest.raises(ParseError):
            idx.search(q, nprobe, k)
    with pytest.raises(ParseError):
        engine.synthetic_index(engine.desc(100, 48, 4))  # d must be a multiple of 32
    with pytest.raises(ParseError):
        idx.migrate(promote=[0])  # already resident


def test_batch_larger_than_one_pass(engine, oracle):
    # 70000 queries > the one-pass limit (65536 at this nlist): consecutive passes, same results
    desc = engine.desc(5000, 32, 64)
    q, _ = engine.synth_queries(desc, 0, 70000)
    e = engine.synthetic_index(desc).search(q, 2, 5)
    o = oracle.synthetic_index(desc).search(q, 2, 5)
    _same(e, o)


@pytest.mark.parametrize("nprobe", [1, 5, 17, 40])
def test_probe_set_boundary_ties(engine, oracle, nprobe):
    # binary centroids and queries: whole groups of centroids at exactly the same distance, so the
    # nprobe boundary cuts through ties that only the list id decides (the set-mode certification
    # must send them to the exact path)
    rng = np.random.default_rng(nprobe)
    d, nlist = 32, 64
    C = rng.integers(0, 2, size=(nlist, d)).astype(np.float32)
    lens = rng.integers(0, 40, size=nlist)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    X = rng.integers(0, 2, size=(int(lens.sum()), d)).astype(np.float32)
    Q = rng.integers(0, 2, size=(24, d)).astype(np.float32)
    e = engine.index_from_host(X, offs, C)
    o = oracle.index_from_host(X, offs, C)
    np.testing.assert_array_equal(e.probe(Q, nprobe), o.probe(Q, nprobe))
    _same(e.search(Q, nprobe, 10), o.search(Q, nprobe, 10))


@pytest.mark.timeout(300)
def test_offloaded_device_search_beside_a_busy_stream(engine, oracle):
    """rd_search_device with offloaded lists while another thread keeps a side stream busy with GEMMs
    (the synthetic decode of bench.py): every result is the oracle's and nothing stalls. Regression
    test for the device-gate deadlock of the RD_ASYNC_TAIL path, now opt-in."""
    import threading
    import torch
    desc = engine.desc(400000, 768, 256)
    q, _ = engine.synth_queries(desc, 13, 32)
    want = oracle.synthetic_index(desc).search(q, 32, 10)
    e = engine.synthetic_index(desc)
    e.place(offload_fraction=0.5)
    dq = torch.from_numpy(q).cuda()
    stop = threading.Event()
    side = torch.cuda.Stream()
    a = torch.randn(64, 4096, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)

    def busy():
        with torch.cuda.stream(side):
            while not stop.is_set():
                for _ in range(50):
                    torch.mm(a, w)
                side.synchronize()

    t = threading.Thread(target=busy, daemon=True)
    t.start()
    try:
        stream = torch.cuda.current_stream()
        di = torch.empty((32, 10), dtype=torch.int64, device="cuda")
        dd = torch.empty((32, 10), dtype=torch.float32, device="cuda")
        for _ in range(6):
            e.search_device(dq.data_ptr(), 32, 32, 10, di.data_ptr(), dd.data_ptr(), stream=stream.cuda_stream)
        torch.cuda.synchronize()
    finally:
        stop.set()
        t.join()
    np.testing.assert_array_equal(di.cpu().numpy(), want.ids)
    np.testing.assert_array_equal(dd.cpu().numpy(), want.dists)


def test_async_search_with_offloaded_lists(engine, oracle, monkeypatch):
    """RD_ASYNC_TAIL=1: rd_search_device with offloaded lists returns once the search is enqueued —
    the offloaded part is planned and enqueued by the index's worker thread while the caller's stream
    waits on a device gate — and the results are the oracle's."""
    import time
    import torch
    monkeypatch.setenv("RD_ASYNC_TAIL", "1")  # read when the index is created
    desc = engine.desc(600000, 768, 256)
    q, _ = engine.synth_queries(desc, 12, 64)
    want = oracle.synthetic_index(desc).search(q, 32, 10)
    e = engine.synthetic_index(desc)
    e.place(offload_fraction=0.5)
    dq = torch.from_numpy(q).cuda()
    stream = torch.cuda.current_stream()
    outs = []
    for rep in range(3):  # back to back on one stream: each tail waits for the previous one
        di = torch.full((64, 10), -7, dtype=torch.int64, device="cuda")
        dd = torch.empty((64, 10), dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        t0 = time.perf_counter()
        e.search_device(dq.data_ptr(), 64, 32, 10, di.data_ptr(), dd.data_ptr(), stream=stream.cuda_stream)
        host_ms = (time.perf_counter() - t0) * 1e3
        ev1.record(stream)
        pending = not ev1.query()
        torch.cuda.synchronize()
        dev_ms = ev0.elapsed_time(ev1)
        outs.append((di.cpu().numpy(), dd.cpu().numpy(), host_ms, dev_ms, pending))
    for ids, dists, host_ms, dev_ms, pending in outs:
        np.testing.assert_array_equal(ids, want.ids)
        np.testing.assert_array_equal(dists, want.dists)
    # the call returned before the search completed (device work still pending, host time a fraction)
    assert any(p for *_, p in outs)
    assert min(h / dv for _, _, h, dv, _ in outs) < 0.5, [(h, dv) for _, _, h, dv, _ in outs]
    assert e.search(q, 32, 10).stats["h2d_list_bytes"] > 0


def test_device_read_bandwidth(engine):
    """The read-stream peak probe the bench's roofline reports against: plausible for HBM3e."""
    gbs = engine.device_read_bandwidth(0, 2 << 30)
    assert 3000.0 < gbs < 9000.0
    with pytest.raises(ParseError):
        engine.device_read_bandwidth(0, 1024)
