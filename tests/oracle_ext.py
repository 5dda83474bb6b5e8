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


def batched_search(oracle, index, queries, nprobe, k):
    """rd_cpu_search_batched: the list-major batched CPU baseline (oracle/rd_cpu_batched.c) over an
    oracle index; returns (ids, dists, fallbacks). Prepares the row norms on first use."""
    lib = oracle.lib
    lib.rd_cpu_prepare_batched.restype = C.c_int
    lib.rd_cpu_prepare_batched.argtypes = [C.c_void_p]
    fn = lib.rd_cpu_search_batched
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                   C.POINTER(C.c_float), C.POINTER(C.c_int64)]
    if not getattr(index, "_batched_ready", False):
        assert lib.rd_cpu_prepare_batched(index.handle) == 0
        index._batched_ready = True
    q = np.ascontiguousarray(queries, dtype=np.float32)
    B = q.shape[0]
    ids = np.empty((B, k), dtype=np.int64)
    dists = np.empty((B, k), dtype=np.float32)
    fb = C.c_int64(0)
    rc = fn(index.handle, q.ctypes.data_as(C.POINTER(C.c_float)), B, nprobe, k,
            ids.ctypes.data_as(C.POINTER(C.c_int64)), dists.ctypes.data_as(C.POINTER(C.c_float)), C.byref(fb))
    assert rc == 0, f"rd_cpu_search_batched failed ({rc})"
    return ids, dists, fb.value
