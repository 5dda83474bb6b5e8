"""Oracle parity through the unmodified production chain at the BASELINE configurations' real sizes
(BASELINE.json configs; SURVEY §8c parity rule): the engine searches the configured batch through the
C-ABI and the CPU oracle (exact IVF-Flat, the checker) recomputes a subset of it on the same
synthetic inputs. The bar is bit-exact ids and distances. Where the oracle cannot hold the knowledge
base (C4: 100M x 768 = 307 GB) it regenerates only the probed lists' rows from (seed, id)
(tests/oracle_ext.py). At full size the tests also check size-independent
properties: placement never changes results (C3 / C5 against the resident run, every query)."""
import numpy as np
import pytest

from bench import CONFIGS, c5_reservation

pytestmark = pytest.mark.gpu


def _same(got_ids, got_d, want_ids, want_d):
    np.testing.assert_array_equal(got_ids, want_ids)
    np.testing.assert_array_equal(got_d, want_d)


def test_c1_full(engine, oracle):
    c = CONFIGS["c1"]
    desc = engine.desc(c["n"], c["d"], c["nlist"])
    q, src = engine.synth_queries(desc, 0, c["batch"])
    e = engine.synthetic_index(desc).search(q, c["nprobe"], c["k"])
    o = oracle.synthetic_index(desc).search(q, c["nprobe"], c["k"])
    _same(e.ids, e.dists, o.ids, o.dists)
    assert e.stats["margin_failures"] == 0 and e.stats["probe_failures"] == 0
    assert (e.ids[:, 0] == src).all()


@pytest.fixture(scope="module")
def c2():
    """The C2 knowledge base on both sides, one B = 1024 batch, and the oracle's answer for a spread
    subset of 256 of its queries (every fourth)."""
    from paper_2504_15302_b200.retriever import Library, engine as eng_lib
    from conftest import _ensure_oracle
    eng, orc = eng_lib(), Library(_ensure_oracle())
    c = CONFIGS["c2"]
    desc = eng.desc(c["n"], c["d"], c["nlist"])
    q, _ = eng.synth_queries(desc, 0, c["batch"])
    idx = eng.synthetic_index(desc)
    sub = np.arange(0, c["batch"], 4)
    oidx = orc.synthetic_index(desc)
    want = oidx.search(q[sub], c["nprobe"], c["k"])
    # C5's oracle answer (nprobe 128, k 20, B 64) on the same knowledge base
    c5 = CONFIGS["c5"]
    q5, _ = eng.synth_queries(desc, 5_000_000, c5["batch"])
    want5 = oidx.search(q5, c5["nprobe"], c5["k"])
    cal, _ = eng.synth_queries(desc, 50_000_000, 4096)  # calibration batch for the heat placement
    oidx.close()
    yield dict(eng=eng, desc=desc, q=q, idx=idx, sub=sub, want=want, q5=q5, want5=want5, cal=cal, c=c, c5=c5)
    idx.close()


def test_c2_b1024_production_chain(c2):
    c = c2["c"]
    e = c2["idx"].search(c2["q"], c["nprobe"], c["k"])
    _same(e.ids[c2["sub"]], e.dists[c2["sub"]], c2["want"].ids, c2["want"].dists)
    assert e.stats["margin_failures"] == 0 and e.stats["probe_failures"] == 0
    c2["resident"] = e


def test_c3_half_offloaded(c2):
    c = c2["c"]
    idx = c2["idx"]
    pr = idx.probe(c2["cal"], c["nprobe"])
    heat = np.bincount(pr[pr >= 0].ravel(), minlength=c["nlist"]).astype(np.uint32)
    idx.place(offload_fraction=0.5, list_heat=heat)
    try:
        assert idx.info()["lists_resident"] == c["nlist"] // 2
        e = idx.search(c2["q"], c["nprobe"], c["k"])
        assert e.stats["h2d_list_bytes"] > 0
        _same(e.ids[c2["sub"]], e.dists[c2["sub"]], c2["want"].ids, c2["want"].dists)
        if "resident" in c2:  # every query identical to the fully resident search
            _same(e.ids, e.dists, c2["resident"].ids, c2["resident"].dists)
    finally:
        idx.place(offload_fraction=0.0)


def test_c5_llm_reservation(c2):
    import torch
    c5 = c2["c5"]
    idx = c2["idx"]
    _, total = torch.cuda.mem_get_info()
    reservation = c5_reservation(c2["eng"])
    budget = int(total - reservation - (4 << 30))
    pr = idx.probe(c2["cal"], c5["nprobe"])
    heat = np.bincount(pr[pr >= 0].ravel(), minlength=c5["nlist"]).astype(np.uint32)
    idx.place(hbm_budget_bytes=budget, list_heat=heat)
    try:
        info = idx.info()
        assert 0 < info["lists_resident"] < c5["nlist"]
        assert info["hbm_bytes"] <= budget + (1 << 30)  # lists + ring inside the budget (+ fixed metadata)
        e = idx.search(c2["q5"], c5["nprobe"], c5["k"])
        _same(e.ids, e.dists, c2["want5"].ids, c2["want5"].dists)
        assert e.stats["margin_failures"] == 0 and e.stats["probe_failures"] == 0
    finally:
        idx.place(offload_fraction=0.0)
