"""Shard groups (rd_group_*) on one GPU: G engine stripes searched as one group
and merged on the device must equal the UNSHARDED oracle; the NCCL path is exercised as a
one-rank communicator (NCCL admits one rank per device, so G ranks need G GPUs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(e, o):
    np.testing.assert_array_equal(e.ids, o.ids)
    np.testing.assert_array_equal(e.dists, o.dists)


@pytest.mark.parametrize("G,B,nprobe,k", [(2, 64, 16, 10), (3, 200, 8, 24), (2, 1, 32, 10), (4, 33, 5, 1)])
def test_group_on_one_device_equals_unsharded_oracle(engine, oracle, G, B, nprobe, k):
    n, d, nlist = 150000, 768, 256
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 17, B)
    grp = engine.synthetic_group(desc, [0] * G)
    info = grp.info()
    assert info["num_shards"] == G and info["local_shards"] == G and info["n"] == n
    assert info["transport"] == "copy"
    e = grp.search(q, nprobe, k)
    _same(e, oracle.synthetic_index(desc).search(q, nprobe, k))
    from conftest import fallbacks_allowed
    assert e.stats["margin_failures"] <= G * fallbacks_allowed(B, k) and e.stats["probe_failures"] == 0
    # the oracle's own group form agrees too
    og = oracle.synthetic_group(desc, [0] * G)
    _same(e, og.search(q, nprobe, k))
    grp.close()


def test_group_from_handles_offloaded_and_device_api(engine, oracle):
    import torch
    n, d, nlist, B, nprobe, k = 120000, 768, 128, 48, 12, 10
    full = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(full, 3, B)
    shards = [engine.synthetic_index(engine.desc(n, d, nlist, shard=g, num_shards=2)) for g in range(2)]
    grp = engine.group(shards)
    want = oracle.synthetic_index(full).search(q, nprobe, k)
    _same(grp.search(q, nprobe, k), want)
    grp.place(offload_fraction=0.5, staging_slots=2)  # every stripe half offloaded
    assert grp.shard(0).info()["lists_resident"] == nlist // 2
    e = grp.search(q, nprobe, k)
    assert e.stats["h2d_list_bytes"] > 0
    _same(e, want)
    dq = torch.from_numpy(q).cuda()
    di = torch.empty((B, k), dtype=torch.int64, device="cuda")
    dd = torch.empty((B, k), dtype=torch.float32, device="cuda")
    st = grp.search_device(dq.data_ptr(), B, nprobe, k, di.data_ptr(), dd.data_ptr(),
                           stream=torch.cuda.current_stream().cuda_stream, sync=True)
    assert st["margin_failures"] == 0
    np.testing.assert_array_equal(di.cpu().numpy(), want.ids)
    np.testing.assert_array_equal(dd.cpu().numpy(), want.dists)
    grp.close()


def test_group_one_rank_nccl(engine, oracle):
    # the per-process form through a real NCCL communicator (one rank: no peers on one GPU)
    n, d, nlist, B, nprobe, k = 50000, 768, 64, 20, 8, 10
    desc = engine.desc(n, d, nlist)
    q, _ = engine.synth_queries(desc, 5, B)
    uid = engine.group_unique_id()
    assert len(uid) == 128
    grp = engine.rank_group(engine.synthetic_index(desc), uid, 1, 0)
    info = grp.info()
    assert info["nranks"] == 1 and info["rank"] == 0
    _same(grp.search(q, nprobe, k), oracle.synthetic_index(desc).search(q, nprobe, k))
    grp.close()


@pytest.mark.parametrize("G,k", [(3, 64), (8, 128), (2, 33)])
def test_device_merge_any_k(engine, G, k):
    import torch
    rng = np.random.default_rng(G * k)
    B = 40
    d = np.sort(rng.random((G, B, k)).astype(np.float32), axis=2)
    d[0, :, :3] = d[1, :, :3] if G > 1 else d[0, :, :3]  # equal distances across shards: id order decides
    ids = rng.permutation(G * B * k).reshape(G, B, k).astype(np.int64)
    ids[-1, :, k // 2:] = -1
    want_i, want_d = engine.merge_topk(ids, d)
    ti, td = torch.from_numpy(ids).cuda(), torch.from_numpy(d).cuda()
    oi = torch.empty((B, k), dtype=torch.int64, device="cuda")
    od = torch.empty((B, k), dtype=torch.float32, device="cuda")
    engine.check(engine.lib.rd_merge_topk_device(G, B, k, ti.data_ptr(), td.data_ptr(), oi.data_ptr(),
                                                 od.data_ptr(), None))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(oi.cpu().numpy(), want_i)
    np.testing.assert_array_equal(od.cpu().numpy(), want_d)
