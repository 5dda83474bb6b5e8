"""Host-side logic on CPU: the placement rule, the shard-merge algebra (the
multi-GPU exchange step), and the exported C-ABI surface."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_engine_exports_every_header_symbol(engine_lib, oracle):
    from paper_2504_15302_b200.retriever import EXPORTED_SYMBOLS
    hdr = open(os.path.join(ROOT, "include", "rd.h")).read()
    declared = set(re.findall(r"\b(rd_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(EXPORTED_SYMBOLS)
    for lib in (engine_lib, oracle):
        for sym in declared:
            assert hasattr(lib.lib, sym), (lib.path, sym)
    assert engine_lib.backend == "b200-sm100a" and oracle.backend == "cpu-oracle"


def _shard_results(oracle, G, n=3000, d=64, nlist=24, B=10, nprobe=6, k=10):
    desc = oracle.desc(n, d, nlist)
    Q, _ = oracle.synth_queries(desc, 0, B)
    full = oracle.synthetic_index(desc).search(Q, nprobe, k)
    parts = [oracle.synthetic_index(oracle.desc(n, d, nlist, shard=g, num_shards=G)).search(Q, nprobe, k)
             for g in range(G)]
    return full, np.stack([p.ids for p in parts]), np.stack([p.dists for p in parts])


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_row_striped_shards_merge_to_unsharded(oracle, engine_lib, G):
    full, sid, sd = _shard_results(oracle, G)
    for lib in (engine_lib, oracle):
        mi, md = lib.merge_topk(sid, sd)
        np.testing.assert_array_equal(mi, full.ids)
        np.testing.assert_array_equal(md, full.dists)


def test_shards_partition_the_lists(oracle):
    n, d, nlist, G = 2000, 16, 12, 3
    offs, ids, _ = oracle.synthetic_index(oracle.desc(n, d, nlist)).layout()
    parts = [oracle.synthetic_index(oracle.desc(n, d, nlist, shard=g, num_shards=G)).layout() for g in range(G)]
    for l in range(nlist):
        cat = np.concatenate([p[1][p[0][l]:p[0][l + 1]] for p in parts])
        np.testing.assert_array_equal(cat, ids[offs[l]:offs[l + 1]])


def test_placement_rule(oracle):
    from paper_2504_15302_b200.retriever import InfeasibleError
    desc = oracle.desc(4000, 32, 20)
    idx = oracle.synthetic_index(desc)
    offs, _, _ = idx.layout(with_ids=False)
    lens = np.diff(offs)
    idx.place(offload_fraction=0.5)
    _, _, mask = idx.layout(with_ids=False)
    assert mask.sum() == 10 and mask[:10].all()
    heat = np.arange(20)[::-1].copy()[::-1]  # list 19 hottest
    idx.place(offload_fraction=0.25, list_heat=heat)
    _, _, mask = idx.layout(with_ids=False)
    assert mask.sum() == 15 and mask[5:].all()
    total = int(lens.sum() * 32 * 4)
    idx.place(hbm_budget_bytes=total)  # everything fits: no staging ring needed
    assert idx.layout(with_ids=False)[2].all()
    with pytest.raises(InfeasibleError):  # one byte short: the 2-slot ring (4 MiB) does not fit
        idx.place(hbm_budget_bytes=total - 1)
    with pytest.raises(InfeasibleError):
        idx.place(hbm_budget_bytes=total - 1, resident_mask=np.ones(20, np.uint8))
    # a larger index: the budget covers the staging ring plus the first three lists
    big = oracle.synthetic_index(oracle.desc(200000, 32, 20))
    blens = np.diff(big.layout(with_ids=False)[0])
    ring = 2 * 16384 * 32 * 4  # two slots of max(largest list, 16384) rows
    assert blens.max() <= 16384
    big.place(hbm_budget_bytes=int(blens[:3].sum() * 32 * 4) + ring)
    bmask = big.layout(with_ids=False)[2]
    assert bmask[:3].all() and not bmask[3:].any()


@pytest.mark.parametrize("G", [1, 2, 3])
def test_oracle_group_equals_unsharded(oracle, G):
    # rd_group_* algebra on the CPU: stripes searched in turn and merged equal the unsharded search
    n, d, nlist, B, nprobe, k = 8000, 64, 20, 11, 4, 10
    desc = oracle.desc(n, d, nlist)
    q, _ = oracle.synth_queries(desc, 2, B)
    grp = oracle.synthetic_group(desc, [0] * G)
    assert grp.info()["num_shards"] == G and grp.info()["n"] == n
    e = grp.search(q, nprobe, k)
    o = oracle.synthetic_index(desc).search(q, nprobe, k)
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)
    from paper_2504_15302_b200.retriever import ParseError
    with pytest.raises(ParseError):  # no communicator in the CPU oracle
        oracle.group_unique_id()
    grp.close()
