"""Oracle-only entry points of oracle/librd_cpu.so that are not part of include/rd.h (test
infrastructure: the checker, never the product)."""
import ctypes as C

import numpy as np

from paper_2504_15302_b200.retriever import SynthDesc


def synth_search(oracle, desc, queries, nprobe, k, shard_mask=~0):
    """rd_oracle_synth_search: exact IVF-Flat over the synthetic knowledge base `desc` restricted to
    the row stripes g of desc.num_shards with bit g of shard_mask set, regenerating only the probed
    lists' rows from (seed, id) — the check for knowledge bases too large for host memory (C4)."""
    fn = oracle.lib.rd_oracle_synth_search
    fn.restype = C.c_int
    fn.argtypes = [C.POINTER(SynthDesc), C.c_uint64, C.POINTER(C.c_float), C.c_int64, C.c_int32, C.c_int32,
                   C.POINTER(C.c_int64), C.POINTER(C.c_float)]
    q = np.ascontiguousarray(queries, dtype=np.float32)
    B = q.shape[0]
    ids = np.empty((B, k), dtype=np.int64)
    dists = np.empty((B, k), dtype=np.float32)
    oracle.check(fn(C.byref(desc), shard_mask & ((1 << 64) - 1), q.ctypes.data_as(C.POINTER(C.c_float)), B, nprobe,
                    k, ids.ctypes.data_as(C.POINTER(C.c_int64)), dists.ctypes.data_as(C.POINTER(C.c_float))),
                 "synth_search")
    return ids, dists
