"""C4 (BASELINE.json configs[3]: 100M x 768 fp32 sharded across GPUs, per-shard top-k + gather/merge):
two of the eight row stripes of the 100M knowledge base as one shard group on this GPU (the same
group code path as G GPUs, with device copies in place of NCCL because NCCL admits one rank per
device), one B = 1024 batch through rd_group_search, checked against the sampled oracle that
regenerates the probed lists' rows of those two stripes from (seed, id)."""
import numpy as np
import pytest

from bench import CONFIGS
from oracle_ext import synth_search

pytestmark = pytest.mark.gpu


def test_c4_two_stripes_of_eight(engine, oracle, monkeypatch):
    import torch
    monkeypatch.setenv("RD_PRESPLIT", "0")  # two 12.5M-row stripes plus their bf16 copies would not fit beside the test's buffers
    c = CONFIGS["c4"]
    desc = engine.desc(c["n"], c["d"], c["nlist"], num_shards=8)
    q, _ = engine.synth_queries(desc, 0, c["batch"])
    shards = [engine.synthetic_index(engine.desc(c["n"], c["d"], c["nlist"], shard=g, num_shards=8)) for g in (0, 1)]
    grp = engine.group(shards)
    try:
        info = grp.info()
        assert info["num_shards"] == 2 and info["transport"] == "copy"
        e = grp.search(q, c["nprobe"], c["k"])
        assert e.stats["margin_failures"] == 0 and e.stats["probe_failures"] == 0
        sub = np.arange(0, c["batch"], 64)  # 16 queries spread over the batch
        want_i, want_d = synth_search(oracle, desc, q[sub], c["nprobe"], c["k"], shard_mask=0b11)
        np.testing.assert_array_equal(e.ids[sub], want_i)
        np.testing.assert_array_equal(e.dists[sub], want_d)
        # every query: ascending, distinct ids, and each distance is the canonical exact distance
        assert (np.diff(e.dists, axis=1) >= 0).all()
        assert all(len(set(r)) == len(r) for r in e.ids.tolist())
        for b in range(0, c["batch"], 97):
            for j in (0, c["k"] - 1):
                x = engine.synth_vector(desc, int(e.ids[b, j]))
                assert engine.exact_l2(q[b], x) == e.dists[b, j]
        # the device entry point gives the same merged result
        dq = torch.from_numpy(q).cuda()
        di = torch.empty((c["batch"], c["k"]), dtype=torch.int64, device="cuda")
        dd = torch.empty((c["batch"], c["k"]), dtype=torch.float32, device="cuda")
        grp.search_device(dq.data_ptr(), c["batch"], c["nprobe"], c["k"], di.data_ptr(), dd.data_ptr(),
                          stream=torch.cuda.current_stream().cuda_stream, sync=True)
        np.testing.assert_array_equal(di.cpu().numpy(), e.ids)
        np.testing.assert_array_equal(dd.cpu().numpy(), e.dists)
    finally:
        grp.close()
