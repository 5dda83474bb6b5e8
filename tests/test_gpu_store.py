"""The resident store: the residual store (default while every list is resident: fp32
rows + r1 = bf16(x - c_list), 6 B per element, the scan reads 2), split3 — the exact bf16 triple
x = (x1 + x2) + x3, 6 B per element, the tensor-core scan's operand without an fp32 copy — or fp32
rows; placements choose the format by budget and relayout in place (VMM arenas grow and shrink,
never two copies of a list). Every search is checked against the CPU oracle bit for bit."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPLIT3, F32, F32_PRESPLIT = 2, 0, 1
RESID = 4  # the residual store with its default fp16 plane (3: bf16 plane)
CHUNK = 64 << 20  # largest arena chunk: what a store may hold beyond its rows, per arena


def _same(e, o):
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)


def _meta_bytes(n, nlist, d):  # norms, ids, row -> list map, coarse state (rd_index_info_get)
    return n * 16 + nlist * (d * 8 + 28)


def test_resid_is_default_and_split3_on_request(engine, oracle, monkeypatch):
    n, d, nlist = 150000, 768, 128
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 5, 64)
    want = oracle.synthetic_index(desc).search(q, 12, 10)
    r = engine.synthetic_index(desc)
    info = r.info()
    assert info["store"] == RESID
    # fp32 rows + the bf16 residual plane + ||x - c||^2 per row: 1.5 x the fp32 rows as well
    assert info["hbm_bytes"] <= 1.5 * n * d * 4 + n * 4 + 2 * CHUNK + _meta_bytes(n, nlist, d)
    _same(r.search(q, 12, 10), want)
    r.close()
    monkeypatch.setenv("RD_STORE", "split3")
    e = engine.synthetic_index(desc)
    info = e.info()
    assert info["store"] == SPLIT3
    # 1.5 x the fp32 rows, plus chunk rounding of the two arenas and the metadata
    assert info["hbm_bytes"] <= 1.5 * n * d * 4 + 2 * CHUNK + _meta_bytes(n, nlist, d)
    _same(e.search(q, 12, 10), want)
    monkeypatch.setenv("RD_SPLIT3", "0")  # the round-1 layout: fp32 rows + pre-split copy
    f = engine.synthetic_index(desc)
    assert f.info()["store"] == F32_PRESPLIT
    assert f.info()["hbm_bytes"] >= 2 * n * d * 4
    _same(f.search(q, 12, 10), want)


@pytest.mark.parametrize("store", ["resid", "split3"])
@pytest.mark.parametrize("B", [1, 40, 600])
def test_split3_every_batch_path(engine, oracle, B, store, monkeypatch):
    """Staged (small-batch) and direct rerank / seeding / fallback paths over each store."""
    monkeypatch.setenv("RD_STORE", store)
    desc = engine.desc(80000, 512, 64)
    q, _ = engine.synth_queries(desc, 77, B)
    _same(engine.synthetic_index(desc).search(q, 9, 24), oracle.synthetic_index(desc).search(q, 9, 24))


@pytest.mark.parametrize("store", ["resid", "split3"])
def test_split3_duplicates_use_the_fallback(engine, oracle, store, monkeypatch):
    """Duplicate vectors tie across ranks k..m: the exact fallback reads the store's rows."""
    monkeypatch.setenv("RD_STORE", store)
    rng = np.random.default_rng(3)
    base = rng.standard_normal((500, 128)).astype(np.float32)
    X = np.repeat(base, 40, axis=0)  # more copies than a 32-entry candidate list holds
    offs = np.array([0, 10000, 20000], np.int64)
    C = np.stack([X[:10000].mean(0), X[10000:].mean(0)]).astype(np.float32)
    Q = (base[:16] + 0.01 * rng.standard_normal((16, 128))).astype(np.float32)
    e = engine.index_from_host(X, offs, C)
    assert e.info()["store"] == (SPLIT3 if store == "split3" else RESID)
    r = e.search(Q, 2, 10)
    _same(r, oracle.index_from_host(X, offs, C).search(Q, 2, 10))
    assert r.stats["margin_failures"] > 0


def test_inexact_split_keeps_fp32_rows(engine, oracle, monkeypatch):
    """Components whose residuals fall below bf16's subnormal range do not round-trip: the index
    keeps fp32 rows and stays exact."""
    monkeypatch.setenv("RD_SPLIT3_QUIET", "1")
    monkeypatch.setenv("RD_STORE", "split3")
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3000, 64)).astype(np.float32)
    X[7, :5] = np.float32(1.2345678e-38)  # fp32 normal, its split residual is not representable
    offs = np.array([0, 1500, 3000], np.int64)
    C = np.stack([X[:1500].mean(0), X[1500:].mean(0)]).astype(np.float32)
    Q = X[:20] + np.float32(0.01)
    e = engine.index_from_host(X, offs, C)
    assert e.info()["store"] != SPLIT3
    _same(e.search(Q, 2, 10), oracle.index_from_host(X, offs, C).search(Q, 2, 10))


def test_placement_picks_the_format_by_budget(engine, oracle):
    n, d, nlist = 200000, 768, 128
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 9, 48)
    want = oracle.synthetic_index(desc).search(q, 16, 10)
    e = engine.synthetic_index(desc)
    rows = n * d
    # room for every list in the residual store (fp32 rows + bf16 residuals + ||x - c||^2), inside the
    # budget; a little less and the split3 store holds them all
    roomy = int(1.5 * rows * 4) + n * 4 + 3 * CHUNK
    e.place(hbm_budget_bytes=roomy)
    info = e.info()
    assert info["store"] == RESID and info["lists_resident"] == nlist
    assert info["hbm_bytes"] - _meta_bytes(n, nlist, d) <= roomy
    _same(e.search(q, 16, 10), want)
    roomy = int(1.5 * rows * 4) + n * 2
    e.place(hbm_budget_bytes=roomy)
    info = e.info()
    assert info["store"] == SPLIT3 and info["lists_resident"] == nlist
    assert info["hbm_bytes"] - _meta_bytes(n, nlist, d) <= roomy + 2 * CHUNK
    _same(e.search(q, 16, 10), want)
    # a budget below the split3 size but above fp32: every list resident as fp32 rows
    tight = int(1.1 * rows * 4)
    e.place(hbm_budget_bytes=tight)
    info = e.info()
    assert info["store"] == F32 and info["lists_resident"] == nlist
    assert info["hbm_bytes"] - _meta_bytes(n, nlist, d) <= tight + CHUNK
    _same(e.search(q, 16, 10), want)
    # a budget that offloads: fp32 rows, a staging ring, results unchanged
    e.place(hbm_budget_bytes=int(0.5 * rows * 4))
    info = e.info()
    assert info["store"] == F32 and 0 < info["lists_resident"] < nlist
    r = e.search(q, 16, 10)
    assert r.stats["h2d_list_bytes"] > 0
    _same(r, want)
    # no budget again: back to the residual store, all resident
    e.place(offload_fraction=0.0)
    assert e.info()["store"] == RESID and e.info()["lists_resident"] == nlist
    _same(e.search(q, 16, 10), want)


def test_migration_shrinks_and_grows_the_store(engine, oracle):
    n, d, nlist = 200000, 768, 64
    desc = engine.desc(n, d, nlist)
    e, o = engine.synthetic_index(desc), oracle.synthetic_index(desc)
    q, _ = engine.synth_queries(desc, 21, 32)
    want = o.search(q, 8, 10)
    full = e.info()["hbm_bytes"]
    half = list(range(0, nlist, 2))
    e.migrate(demote=half)
    after = e.info()
    offs = e.layout(with_ids=False)[0]
    moved = int(np.diff(offs)[half].sum()) * d * 6
    # the store gives the demoted lists' bytes back (to a chunk), the staging ring comes in
    ring = after["staging_slots"] * ((max(int(np.diff(offs)[half].max()), 16384) + 255) // 256 * 256) * d * 4
    assert after["hbm_bytes"] <= full - moved + ring + 2 * CHUNK
    _same(e.search(q, 8, 10), want)
    e.migrate(promote=half)
    assert e.info()["hbm_bytes"] <= full + 2 * CHUNK
    _same(e.search(q, 8, 10), want)


def test_migration_budget_keeps_the_ring_inside(engine):
    n, d, nlist = 100000, 256, 32
    e = engine.synthetic_index(engine.desc(n, d, nlist))
    e.place(offload_fraction=0.25, staging_slots=8)  # a deep ring
    offs = e.layout(with_ids=False)[0]
    lens = np.diff(offs)
    mask = e.layout(with_ids=False)[2].astype(bool)
    res = np.flatnonzero(mask)
    res_rows = int(lens[mask].sum()) - int(lens[res[0]])
    slot = (max(int(lens[~mask].max()), int(lens[res[0]]), 16384) + 255) // 256 * 256 * d * 4
    budget = res_rows * d * 6 + 3 * slot  # room for three slots, not eight
    e.migrate(demote=[int(res[0])], hbm_budget_bytes=budget)
    info = e.info()
    assert info["staging_slots"] == 3
    assert info["hbm_bytes"] - _meta_bytes(int(n), nlist, d) <= budget + CHUNK
