"""Between-batch list migration (rd_index_migrate; reference: the
retrieval worker's partition reconfiguration, simulator.cpp:331-352, costed by
plan_transfer, memory_planner.cpp:137-142, shrink before grow, simulator.cpp:323-326).

CPU tests pin the semantics on the oracle (validation, budget rule, write-once
host-copy accounting); GPU tests check that the engine's in-place compaction and
promotion keep search results bit-identical to the oracle and report the same
transfer accounting."""
import numpy as np
import pytest

from paper_2504_15302_b200.retriever import InfeasibleError, ParseError


def _mask(idx):
    return idx.layout(with_ids=False)[2].astype(bool)


def _lens(idx):
    offs = idx.layout(with_ids=False)[0]
    return np.diff(offs)


def test_oracle_migration_accounting(oracle):
    desc = oracle.desc(4000, 64, 16)
    idx = oracle.synthetic_index(desc)
    lens = _lens(idx) * 64 * 4
    # all resident, no host copies: demoting costs a device->host copy
    st = idx.migrate(demote=[1, 5])
    assert st["d2h_bytes"] == lens[1] + lens[5] and st["h2d_bytes"] == 0
    assert not _mask(idx)[[1, 5]].any() and _mask(idx).sum() == 14
    # promote back: host copies are kept (write-once), so a second demotion is free
    st = idx.migrate(promote=[5])
    assert st["h2d_bytes"] == lens[5] and st["d2h_bytes"] == 0
    st = idx.migrate(demote=[5])
    assert st["d2h_bytes"] == 0
    assert st["resident_bytes"] == lens[_mask(idx)].sum()


@pytest.mark.parametrize("bad", [dict(promote=[99]), dict(promote=[0]), dict(demote=[3, 3]),
                                 dict(promote=[2], demote=[2])])
def test_oracle_migration_invalid(oracle, bad):
    idx = oracle.synthetic_index(oracle.desc(2000, 32, 8))
    idx.migrate(demote=[2])
    with pytest.raises(ParseError):
        idx.migrate(**bad)


def test_oracle_migration_budget(oracle):
    idx = oracle.synthetic_index(oracle.desc(3000, 32, 8))
    lens = _lens(idx) * 32 * 4
    slot = 16384 * 32 * 4  # 2 slots of max(largest offloaded list, 16384 rows)
    before = _mask(idx).copy()
    need = lens.sum() - lens[0] + 2 * slot
    with pytest.raises(InfeasibleError):
        idx.migrate(demote=[0], hbm_budget_bytes=need - 1)
    np.testing.assert_array_equal(_mask(idx), before)  # nothing changed
    idx.migrate(demote=[0], hbm_budget_bytes=need)
    assert not _mask(idx)[0]


def test_oracle_results_unchanged(oracle):
    desc = oracle.desc(5000, 64, 20)
    idx = oracle.synthetic_index(desc)
    q, _ = oracle.synth_queries(desc, 0, 12)
    want = idx.search(q, 6, 10)
    idx.place(offload_fraction=0.5)
    idx.migrate(promote=np.flatnonzero(~_mask(idx))[:4], demote=np.flatnonzero(_mask(idx))[:6])
    got = idx.search(q, 6, 10)
    np.testing.assert_array_equal(got.ids, want.ids)
    np.testing.assert_array_equal(got.dists, want.dists)


@pytest.mark.gpu
def test_engine_migration_matches_oracle(engine, oracle, tmp_path):
    desc = engine.desc(60000, 768, 64)
    e, o = engine.synthetic_index(desc), oracle.synthetic_index(desc)
    q, _ = engine.synth_queries(desc, 300, 48)
    want = o.search(q, 12, 10)
    steps = [
        dict(demote=[3, 9, 10, 40]),                         # all resident: device -> host copies
        dict(promote=[9], demote=[0, 1, 2, 63]),             # mixed, compaction of the survivors
        dict(promote=[3, 10, 40, 0]),                        # host copies reused, no device->host
        dict(demote=list(range(20, 44))),                    # a large demotion, staging ring regrows
        dict(promote=list(range(20, 44)) + [1, 2, 63]),      # everything back
    ]
    for step in steps:
        se, so = e.migrate(**step), o.migrate(**step)
        for f in ("h2d_bytes", "d2h_bytes", "lists_promoted", "lists_demoted", "resident_bytes"):
            assert se[f] == so[f], (step, f, se[f], so[f])
        np.testing.assert_array_equal(_mask(e), _mask(o))
        got = e.search(q, 12, 10)
        np.testing.assert_array_equal(got.ids, want.ids)
        np.testing.assert_array_equal(got.dists, want.dists)
        assert got.stats["margin_failures"] == 0
    # the migrated index still saves the oracle's exact file
    ep, op = str(tmp_path / "e.rdidx"), str(tmp_path / "o.rdidx")
    e.save(ep)
    o.save(op)
    assert open(ep, "rb").read() == open(op, "rb").read()


@pytest.mark.gpu
def test_engine_migration_after_placement(engine, oracle):
    desc = engine.desc(40000, 768, 40)
    e, o = engine.synthetic_index(desc), oracle.synthetic_index(desc)
    for idx in (e, o):
        idx.place(offload_fraction=0.5)
    q, _ = engine.synth_queries(desc, 11, 32)
    want = o.search(q, 10, 20)
    off = np.flatnonzero(~_mask(e))
    res = np.flatnonzero(_mask(e))
    se = e.migrate(promote=off[:7], demote=res[:7])
    so = o.migrate(promote=off[:7], demote=res[:7])
    assert se["h2d_bytes"] == so["h2d_bytes"] and se["d2h_bytes"] == so["d2h_bytes"]
    got = e.search(q, 10, 20)
    np.testing.assert_array_equal(got.ids, want.ids)
    np.testing.assert_array_equal(got.dists, want.dists)
    assert got.stats["h2d_list_bytes"] > 0  # offloaded lists are still streamed
