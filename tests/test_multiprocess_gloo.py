"""The N>1 path on CPU: two ranks (gloo, world_size 2) each search their row
stripe of every list, all-gather the local top-k, and rank 0 merges them with
the engine's host merge (rd_merge_topk) — the same exchange bench.py performs
over NCCL. Must equal the unsharded search."""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2504_15302_b200.retriever import ENGINE_PATH, Library
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle = Library(os.path.join(ROOT, "oracle", "librd_cpu.so"))
    engine = Library(ENGINE_PATH)
    n, d, nlist, B, nprobe, k = 3000, 64, 24, 9, 5, 10
    desc = oracle.desc(n, d, nlist, shard=rank, num_shards=world)
    Q, _ = oracle.synth_queries(desc, 0, B)
    r = oracle.synthetic_index(desc).search(Q, nprobe, k)
    ids = [torch.empty((B, k), dtype=torch.int64) for _ in range(world)]
    ds = [torch.empty((B, k), dtype=torch.float32) for _ in range(world)]
    dist.all_gather(ids, torch.from_numpy(r.ids))
    dist.all_gather(ds, torch.from_numpy(r.dists))
    if rank == 0:
        mi, md = engine.merge_topk(np.stack([t.numpy() for t in ids]), np.stack([t.numpy() for t in ds]))
        full = oracle.synthetic_index(oracle.desc(n, d, nlist)).search(Q, nprobe, k)
        out_q.put(bool(np.array_equal(mi, full.ids) and np.array_equal(md, full.dists)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_merge(engine_lib, oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert all(p.exitcode == 0 for p in procs)
