"""ctypes binding of include/rd.h — the RAGDoll retriever API.

Mirrors the reference's conventions for its retrieval stage:
  - errors are the ragsim exception family (core/include/ragsim/errors.hpp:11-26):
    ``Error`` (status 4, runtime), ``InfeasibleError`` (status 3),
    ``ParseError`` (status 2, invalid input), mapped from the C status codes
    that mirror the ragsim CLI exit codes (tools/main.cpp:30);
  - ``Index.search(queries, nprobe, k)`` is the real retrieval whose wall time
    replaces ``retrieval_time(P, db)`` (core/src/cost_model.cpp:15-21);
  - ``Index.place(...)`` is per-list residency, the analogue of
    ``PlacementConfig::resident_partitions`` (core/include/ragsim/domain.hpp:78).

``Library()`` with no argument loads the B200 engine (``lib/librd_b200.so``)
and raises if it is missing: there is no CPU fallback. Tests pass an explicit
path to load the CPU oracle as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ENGINE_PATH = os.path.join(_HERE, "lib", "librd_b200.so")

RD_OK, RD_ERR_INVALID, RD_ERR_INFEASIBLE, RD_ERR_RUNTIME = 0, 2, 3, 4
DEFAULT_SEED = 250415302
STREAMS = {"centroids": 0x1001, "assign": 0x1002, "vector_noise": 0x1003,
           "query_pick": 0x1004, "query_noise": 0x1005, "train_init": 0x1006}


class Error(RuntimeError):
    """ragsim::Error — any library failure (status 4 here: runtime/CUDA)."""


class InfeasibleError(Error):
    """ragsim::InfeasibleError — a placement that cannot satisfy the HBM budget (status 3)."""


class ParseError(Error):
    """ragsim::ParseError — malformed / invalid input (status 2)."""


class SynthDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("nlist", C.c_int32), ("seed", C.c_uint64),
                ("sigma", C.c_float), ("shard", C.c_int32), ("num_shards", C.c_int32)]


class Placement(C.Structure):
    _fields_ = [("hbm_budget_bytes", C.c_uint64), ("offload_fraction", C.c_double),
                ("resident_mask", C.POINTER(C.c_uint8)), ("list_heat", C.POINTER(C.c_uint32)),
                ("staging_slots", C.c_int32), ("reserved", C.c_int32)]


class MigrationStats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("d2d_bytes", C.c_uint64), ("lists_promoted", C.c_int32), ("lists_demoted", C.c_int32),
                ("resident_bytes", C.c_uint64)]


class SearchStats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("bytes_algorithmic", C.c_uint64),
                ("bytes_lists_resident", C.c_uint64), ("h2d_list_bytes", C.c_uint64),
                ("lists_probed", C.c_uint64), ("tiles", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("scan_ms", C.c_double), ("coarse_ms", C.c_double), ("offload_ms", C.c_double),
                ("margin_failures", C.c_uint32), ("probe_failures", C.c_uint32)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class IndexInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("nlist", C.c_int32), ("n_resident", C.c_int64),
                ("hbm_bytes", C.c_uint64), ("host_pinned_bytes", C.c_uint64),
                ("lists_resident", C.c_int32), ("staging_slots", C.c_int32), ("max_norm", C.c_float),
                ("device", C.c_int32), ("store", C.c_int32), ("reserved", C.c_int32)]


class Timing(C.Structure):
    _fields_ = [("searches", C.c_int64), ("scan_ms", C.c_double), ("coarse_ms", C.c_double),
                ("tail_ms", C.c_double), ("total_ms", C.c_double), ("stage_searches", C.c_int64)]


class GroupInfo(C.Structure):
    _fields_ = [("num_shards", C.c_int32), ("local_shards", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("transport", C.c_int32), ("root_device", C.c_int32), ("n", C.c_int64), ("n_resident", C.c_int64)]


GROUP_TRANSPORTS = {0: "none", 1: "nccl", 2: "copy"}
GROUP_ID_BYTES = 128


class LlmReservation(C.Structure):
    _fields_ = [("weight_total", C.c_uint64), ("kv_bytes_per_request", C.c_uint64),
                ("workspace_bytes_per_request", C.c_uint64), ("w_gpu", C.c_double), ("c_gpu", C.c_double),
                ("gen_batch_size", C.c_int32), ("decode_phase", C.c_int32), ("workspace_fraction", C.c_double)]


_P = C.c_void_p
_FP = C.POINTER(C.c_float)
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)

_SIGS = {
    "rd_last_error": (C.c_char_p, []),
    "rd_abi_version": (C.c_int, []),
    "rd_backend": (C.c_char_p, []),
    "rd_index_create_synthetic": (C.c_int, [C.POINTER(SynthDesc), C.c_int32, C.POINTER(_P)]),
    "rd_index_create_from_host": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, _FP, _I64P, _FP, _I64P,
                                            C.c_int32, C.POINTER(_P)]),
    "rd_index_place": (C.c_int, [_P, C.POINTER(Placement)]),
    "rd_index_info_get": (C.c_int, [_P, C.POINTER(IndexInfo)]),
    "rd_index_layout": (C.c_int, [_P, _I64P, _I64P, C.POINTER(C.c_uint8)]),
    "rd_index_destroy": (None, [_P]),
    "rd_index_migrate": (C.c_int, [_P, _I32P, C.c_int32, _I32P, C.c_int32, C.c_uint64, C.c_void_p]),
    "rd_index_save": (C.c_int, [_P, C.c_char_p]),
    "rd_index_centroids": (C.c_int, [_P, _FP]),
    "rd_index_build": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, _FP, _I64P, C.c_int32, C.c_uint64, C.c_int32,
                                 C.POINTER(_P)]),
    "rd_index_load": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(_P)]),
    "rd_search": (C.c_int, [_P, _FP, C.c_int64, C.c_int32, C.c_int32, _I64P, _FP, C.POINTER(SearchStats)]),
    "rd_search_device": (C.c_int, [_P, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_int32, C.POINTER(SearchStats)]),
    "rd_probe": (C.c_int, [_P, _FP, C.c_int64, C.c_int32, _I32P]),
    "rd_merge_topk": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, _I64P, _FP, _I64P, _FP]),
    "rd_merge_topk_device": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
    "rd_timing_stages": (C.c_int, [_P, C.c_int32]),
    "rd_timing_reset": (C.c_int, [_P]),
    "rd_timing_read": (C.c_int, [_P, C.POINTER(Timing)]),
    "rd_group_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.POINTER(_P)]),
    "rd_group_create_synthetic": (C.c_int, [C.POINTER(SynthDesc), _I32P, C.c_int32, C.POINTER(_P)]),
    "rd_group_unique_id": (C.c_int, [C.c_char_p]),
    "rd_group_create_rank": (C.c_int, [_P, C.c_char_p, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "rd_group_info_get": (C.c_int, [_P, C.POINTER(GroupInfo)]),
    "rd_group_shard": (_P, [_P, C.c_int32]),
    "rd_group_place": (C.c_int, [_P, C.POINTER(Placement)]),
    "rd_group_search": (C.c_int, [_P, _FP, C.c_int64, C.c_int32, C.c_int32, _I64P, _FP, C.POINTER(SearchStats)]),
    "rd_group_search_device": (C.c_int, [_P, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int32, C.POINTER(SearchStats)]),
    "rd_group_destroy": (None, [_P]),
    "rd_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "rd_splitmix_at": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "rd_synth_queries": (C.c_int, [C.POINTER(SynthDesc), C.c_int64, C.c_int64, C.c_float, _FP, _I64P]),
    "rd_synth_vector": (C.c_int, [C.POINTER(SynthDesc), C.c_int64, _FP]),
    "rd_exact_l2": (C.c_float, [_FP, _FP, C.c_int32]),
    "rd_llm_reservation_bytes": (C.c_int, [C.POINTER(LlmReservation), C.POINTER(C.c_double)]),
    "rd_staging_depth": (C.c_int32, [C.c_double, C.c_double]),
    "rd_device_read_bandwidth": (C.c_int, [C.c_int32, C.c_uint64, C.POINTER(C.c_double)]),
}
EXPORTED_SYMBOLS = tuple(_SIGS)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_FP)


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


class Library:
    """One loaded implementation of rd.h."""

    def __init__(self, path: Optional[str] = None):
        path = path or ENGINE_PATH
        if not os.path.exists(path):
            raise Error(f"retrieval library not built: {path} (run `make` or __graft_entry__.build())")
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args
        self.backend = self.lib.rd_backend().decode()

    # -- errors
    def check(self, rc: int, what: str = "") -> None:
        if rc == RD_OK:
            return
        msg = self.lib.rd_last_error().decode(errors="replace")
        if what:
            msg = f"{what}: {msg}"
        if rc == RD_ERR_INFEASIBLE:
            raise InfeasibleError(msg)
        if rc == RD_ERR_INVALID:
            raise ParseError(msg)
        raise Error(msg)

    # -- synthetic data (shared spec)
    @staticmethod
    def desc(n: int, d: int, nlist: int, seed: int = DEFAULT_SEED, sigma: float = 0.25,
             shard: int = 0, num_shards: int = 1) -> SynthDesc:
        return SynthDesc(n, d, nlist, seed, sigma, shard, num_shards)

    def synth_queries(self, desc: SynthDesc, b0: int, B: int, qsigma: float = 0.0625):
        q = np.empty((B, desc.d), dtype=np.float32)
        src = np.empty(B, dtype=np.int64)
        self.check(self.lib.rd_synth_queries(C.byref(desc), b0, B, qsigma, _fp(q), _i64p(src)), "synth_queries")
        return q, src

    def synth_vector(self, desc: SynthDesc, i: int) -> np.ndarray:
        out = np.empty(desc.d, dtype=np.float32)
        self.check(self.lib.rd_synth_vector(C.byref(desc), i, _fp(out)), "synth_vector")
        return out

    def exact_l2(self, a: np.ndarray, b: np.ndarray) -> float:
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        return float(self.lib.rd_exact_l2(_fp(a), _fp(b), a.shape[-1]))

    def derive_seed(self, master: int, stream: int) -> int:
        return int(self.lib.rd_derive_seed(master, stream))

    def splitmix_at(self, seed: int, i: int) -> int:
        return int(self.lib.rd_splitmix_at(seed, i))

    # -- index
    def synthetic_index(self, desc: SynthDesc, device: int = 0) -> "Index":
        h = C.c_void_p()
        self.check(self.lib.rd_index_create_synthetic(C.byref(desc), device, C.byref(h)), "create_synthetic")
        return Index(self, h)

    def index_from_host(self, vectors: np.ndarray, list_offsets: np.ndarray, centroids: np.ndarray,
                        ids: Optional[np.ndarray] = None, device: int = 0) -> "Index":
        vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        list_offsets = np.ascontiguousarray(list_offsets, dtype=np.int64)
        centroids = np.ascontiguousarray(centroids, dtype=np.float32)
        n, d = vectors.shape
        nlist = centroids.shape[0]
        idp = _i64p(np.ascontiguousarray(ids, dtype=np.int64)) if ids is not None else None
        h = C.c_void_p()
        self.check(self.lib.rd_index_create_from_host(n, d, nlist, _fp(vectors), _i64p(list_offsets),
                                                      _fp(centroids), idp, device, C.byref(h)), "create_from_host")
        return Index(self, h)

    def build_index(self, vectors: np.ndarray, nlist: int, iters: int = 10, seed: int = DEFAULT_SEED,
                    ids: Optional[np.ndarray] = None, device: int = 0) -> "Index":
        """IVF training (exact, deterministic k-means) + list-order layout (rd_index_build)."""
        vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        n, d = vectors.shape
        idp = _i64p(np.ascontiguousarray(ids, dtype=np.int64)) if ids is not None else None
        h = C.c_void_p()
        self.check(self.lib.rd_index_build(n, d, nlist, _fp(vectors), idp, iters, seed, device, C.byref(h)), "build")
        return Index(self, h)

    def load_index(self, path: str, device: int = 0) -> "Index":
        """An index from the on-disk format (include/rd_format.h), fully resident."""
        h = C.c_void_p()
        self.check(self.lib.rd_index_load(os.fsencode(path), device, C.byref(h)), "load")
        return Index(self, h)

    # -- multi-GPU shard groups (rd_group_*)
    def group(self, shards) -> "Group":
        """A group over existing stripe handles (one process, any devices); the group takes them over."""
        shards = list(shards)
        arr = (_P * len(shards))(*[sh.handle for sh in shards])
        h = C.c_void_p()
        self.check(self.lib.rd_group_create(arr, len(shards), C.byref(h)), "group_create")
        for sh in shards:  # owned by the group now
            sh._h = None
        return Group(self, h)

    def synthetic_group(self, desc: SynthDesc, devices) -> "Group":
        """Stripe g of desc's knowledge base on devices[g] (one process driving every device)."""
        devs = np.ascontiguousarray(np.asarray(devices, dtype=np.int32).reshape(-1))
        h = C.c_void_p()
        self.check(self.lib.rd_group_create_synthetic(C.byref(desc), devs.ctypes.data_as(_I32P), devs.size,
                                                      C.byref(h)), "group_create_synthetic")
        return Group(self, h)

    def group_unique_id(self) -> bytes:
        buf = C.create_string_buffer(GROUP_ID_BYTES)
        self.check(self.lib.rd_group_unique_id(buf), "group_unique_id")
        return buf.raw

    def rank_group(self, shard: "Index", uid: bytes, nranks: int, rank: int) -> "Group":
        """This process's stripe as rank `rank` of `nranks` (one process per device); collective."""
        if len(uid) != GROUP_ID_BYTES:
            raise ParseError(f"group id must be {GROUP_ID_BYTES} bytes")
        h = C.c_void_p()
        self.check(self.lib.rd_group_create_rank(shard.handle, uid, nranks, rank, C.byref(h)), "group_create_rank")
        shard._h = None
        return Group(self, h)

    # -- merges and arithmetic
    def merge_topk(self, shard_ids: np.ndarray, shard_dists: np.ndarray):
        shard_ids = np.ascontiguousarray(shard_ids, dtype=np.int64)
        shard_dists = np.ascontiguousarray(shard_dists, dtype=np.float32)
        G, B, k = shard_ids.shape
        oi = np.empty((B, k), dtype=np.int64)
        od = np.empty((B, k), dtype=np.float32)
        self.check(self.lib.rd_merge_topk(G, B, k, _i64p(shard_ids), _fp(shard_dists), _i64p(oi), _fp(od)),
                   "merge_topk")
        return oi, od

    def llm_reservation_bytes(self, **kw) -> float:
        r = LlmReservation(kw.get("weight_total", 0), kw.get("kv_bytes_per_request", 0),
                           kw.get("workspace_bytes_per_request", 0), kw.get("w_gpu", 1.0), kw.get("c_gpu", 1.0),
                           kw.get("gen_batch_size", 1), kw.get("decode_phase", 0),
                           kw.get("workspace_fraction", 0.25))
        out = C.c_double()
        self.check(self.lib.rd_llm_reservation_bytes(C.byref(r), C.byref(out)), "llm_reservation_bytes")
        return out.value

    def staging_depth(self, free_bytes: float, item_bytes: float) -> int:
        return int(self.lib.rd_staging_depth(free_bytes, item_bytes))

    def device_read_bandwidth(self, device: int = 0, nbytes: int = 8 << 30) -> float:
        """HBM read-stream peak (GB/s) measured with the scan's load pattern (rd_device_read_bandwidth)."""
        out = C.c_double()
        self.check(self.lib.rd_device_read_bandwidth(device, nbytes, C.byref(out)), "device_read_bandwidth")
        return out.value


def _check_queries(queries: np.ndarray, d: int) -> np.ndarray:
    q = np.ascontiguousarray(queries, dtype=np.float32)
    if q.ndim != 2 or q.shape[1] != d:
        raise ParseError(f"queries must be (B, {d}), got {tuple(np.shape(queries))}")
    return q


def _check_into(queries, d: int, k: int, out_ids, out_dists) -> None:
    """search_into hands raw pointers to the library: shapes, dtypes and layout must be exact."""
    for name, a, dt in (("queries", queries, np.float32), ("out_ids", out_ids, np.int64),
                        ("out_dists", out_dists, np.float32)):
        if not isinstance(a, np.ndarray) or a.dtype != dt or not a.flags.c_contiguous or a.ndim != 2:
            raise ParseError(f"{name} must be a C-contiguous 2-D {np.dtype(dt).name} array")
    if queries.shape[1] != d:
        raise ParseError(f"queries must be (B, {d}), got {queries.shape}")
    if out_ids.shape != (queries.shape[0], k) or out_dists.shape != (queries.shape[0], k):
        raise ParseError(f"out_ids / out_dists must be ({queries.shape[0]}, {k})")
    if not out_ids.flags.writeable or not out_dists.flags.writeable:
        raise ParseError("output buffers must be writeable")


@dataclass
class SearchResult:
    ids: np.ndarray
    dists: np.ndarray
    stats: dict


class Index:
    """A retrieval index handle (library-owned memory; close() or GC frees it)."""

    def __init__(self, lib: Library, handle: C.c_void_p):
        self._lib = lib
        self._h = handle

    def close(self) -> None:
        if self._h and not getattr(self, "_borrowed", False):  # a group's stripe is freed by the group
            self._lib.lib.rd_index_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def info(self) -> dict:
        o = IndexInfo()
        self._lib.check(self._lib.lib.rd_index_info_get(self._h, C.byref(o)), "info")
        return {f: getattr(o, f) for f, _ in o._fields_}

    def layout(self, with_ids: bool = True):
        inf = self.info()
        offs = np.empty(inf["nlist"] + 1, dtype=np.int64)
        ids = np.empty(max(1, inf["n"]), dtype=np.int64) if with_ids else None
        mask = np.empty(inf["nlist"], dtype=np.uint8)
        self._lib.check(self._lib.lib.rd_index_layout(self._h, _i64p(offs), _i64p(ids) if with_ids else None,
                                                      mask.ctypes.data_as(C.POINTER(C.c_uint8))), "layout")
        return offs, (ids[: inf["n"]] if with_ids else None), mask

    def place(self, hbm_budget_bytes: int = 0, offload_fraction: float = 0.0,
              resident_mask: Optional[np.ndarray] = None, list_heat: Optional[np.ndarray] = None,
              staging_slots: int = 0) -> None:
        keep = []
        p = Placement(hbm_budget_bytes, offload_fraction, None, None, staging_slots, 0)
        if resident_mask is not None:
            m = np.ascontiguousarray(resident_mask, dtype=np.uint8)
            keep.append(m)
            p.resident_mask = m.ctypes.data_as(C.POINTER(C.c_uint8))
        if list_heat is not None:
            hh = np.ascontiguousarray(list_heat, dtype=np.uint32)
            keep.append(hh)
            p.list_heat = hh.ctypes.data_as(C.POINTER(C.c_uint32))
        self._lib.check(self._lib.lib.rd_index_place(self._h, C.byref(p)), "place")

    def _dim(self) -> int:
        if getattr(self, "_d", None) is None:
            self._d = self.info()["d"]
        return self._d

    def search(self, queries: np.ndarray, nprobe: int, k: int) -> SearchResult:
        q = _check_queries(queries, self._dim())
        B = q.shape[0]
        ids = np.empty((B, k), dtype=np.int64)
        dists = np.empty((B, k), dtype=np.float32)
        st = SearchStats()
        self._lib.check(self._lib.lib.rd_search(self._h, _fp(q), B, nprobe, k, _i64p(ids), _fp(dists),
                                                C.byref(st)), "search")
        return SearchResult(ids, dists, st.as_dict())

    def search_into(self, queries: np.ndarray, nprobe: int, k: int, out_ids: np.ndarray,
                    out_dists: np.ndarray) -> dict:
        """rd_search into caller-owned host buffers (page-locked buffers are copied directly)."""
        _check_into(queries, self._dim(), k, out_ids, out_dists)
        st = SearchStats()
        self._lib.check(self._lib.lib.rd_search(self._h, _fp(queries), queries.shape[0], nprobe, k, _i64p(out_ids),
                                                _fp(out_dists), C.byref(st)), "search")
        return st.as_dict()

    def search_device(self, q_ptr: int, B: int, nprobe: int, k: int, ids_ptr: int, dists_ptr: int,
                      stream: int = 0, sync: bool = False) -> dict:
        """Device-pointer search (inputs resident in HBM); enqueues on `stream`."""
        st = SearchStats()
        self._lib.check(self._lib.lib.rd_search_device(self._h, C.c_void_p(q_ptr), B, nprobe, k,
                                                       C.c_void_p(ids_ptr), C.c_void_p(dists_ptr),
                                                       C.c_void_p(stream), 1 if sync else 0, C.byref(st)),
                        "search_device")
        return st.as_dict()

    def migrate(self, promote=(), demote=(), hbm_budget_bytes: int = 0) -> dict:
        """Between-batch residency change: demote first, compact, then promote (rd_index_migrate)."""
        pr = np.ascontiguousarray(np.asarray(promote, dtype=np.int32).reshape(-1))
        de = np.ascontiguousarray(np.asarray(demote, dtype=np.int32).reshape(-1))
        st = MigrationStats()
        self._lib.check(self._lib.lib.rd_index_migrate(self._h, pr.ctypes.data_as(_I32P), pr.size,
                                                       de.ctypes.data_as(_I32P), de.size, hbm_budget_bytes,
                                                       C.cast(C.byref(st), C.c_void_p)), "migrate")
        return {f: getattr(st, f) for f, _ in st._fields_}

    def centroids(self) -> np.ndarray:
        inf = self.info()
        out = np.empty((inf["nlist"], inf["d"]), dtype=np.float32)
        self._lib.check(self._lib.lib.rd_index_centroids(self._h, _fp(out)), "centroids")
        return out

    def save(self, path: str) -> None:
        """Writes the index in the on-disk format (include/rd_format.h)."""
        self._lib.check(self._lib.lib.rd_index_save(self._h, os.fsencode(path)), "save")

    def timing_stages(self, on: bool) -> None:
        """Per-stage device timing (coarse / scan / tail) for the following searches (rd.h)."""
        self._lib.check(self._lib.lib.rd_timing_stages(self._h, 1 if on else 0), "timing_stages")

    def timing_reset(self) -> None:
        self._lib.check(self._lib.lib.rd_timing_reset(self._h), "timing_reset")

    def timing_read(self) -> dict:
        t = Timing()
        self._lib.check(self._lib.lib.rd_timing_read(self._h, C.byref(t)), "timing_read")
        return {f: getattr(t, f) for f, _ in t._fields_}

    def probe(self, queries: np.ndarray, nprobe: int) -> np.ndarray:
        q = np.ascontiguousarray(queries, dtype=np.float32)
        out = np.empty((q.shape[0], nprobe), dtype=np.int32)
        self._lib.check(self._lib.lib.rd_probe(self._h, _fp(q), q.shape[0], nprobe,
                                               out.ctypes.data_as(_I32P)), "probe")
        return out


class Group:
    """A shard group (rd_group_*): G row stripes searched together, one merged top-k per call."""

    def __init__(self, lib: Library, handle: C.c_void_p):
        self._lib = lib
        self._h = handle

    def close(self) -> None:
        if self._h:
            self._lib.lib.rd_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def info(self) -> dict:
        o = GroupInfo()
        self._lib.check(self._lib.lib.rd_group_info_get(self._h, C.byref(o)), "group_info")
        d = {f: getattr(o, f) for f, _ in o._fields_}
        d["transport"] = GROUP_TRANSPORTS.get(d["transport"], str(d["transport"]))
        return d

    def shard(self, i: int) -> "Index":
        """Borrowed view of the i-th local stripe (do not close it; the group owns it)."""
        h = self._lib.lib.rd_group_shard(self._h, i)
        if not h:
            raise ParseError(f"no local stripe {i}")
        ix = Index(self._lib, C.c_void_p(h))
        ix._borrowed = True
        return ix

    def place(self, **kw) -> None:
        p = Placement(kw.get("hbm_budget_bytes", 0), kw.get("offload_fraction", 0.0), None, None,
                      kw.get("staging_slots", 0), 0)
        keep = []
        if kw.get("list_heat") is not None:
            hh = np.ascontiguousarray(kw["list_heat"], dtype=np.uint32)
            keep.append(hh)
            p.list_heat = hh.ctypes.data_as(C.POINTER(C.c_uint32))
        if kw.get("resident_mask") is not None:
            m = np.ascontiguousarray(kw["resident_mask"], dtype=np.uint8)
            keep.append(m)
            p.resident_mask = m.ctypes.data_as(C.POINTER(C.c_uint8))
        self._lib.check(self._lib.lib.rd_group_place(self._h, C.byref(p)), "group_place")

    def search(self, queries: np.ndarray, nprobe: int, k: int) -> SearchResult:
        q = np.ascontiguousarray(queries, dtype=np.float32)
        if q.ndim != 2:
            raise ParseError("queries must be 2-D")
        B = q.shape[0]
        ids = np.empty((B, k), dtype=np.int64)
        dists = np.empty((B, k), dtype=np.float32)
        st = SearchStats()
        self._lib.check(self._lib.lib.rd_group_search(self._h, _fp(q), B, nprobe, k, _i64p(ids), _fp(dists),
                                                      C.byref(st)), "group_search")
        return SearchResult(ids, dists, st.as_dict())

    def search_into(self, queries: np.ndarray, nprobe: int, k: int, out_ids: np.ndarray,
                    out_dists: np.ndarray) -> dict:
        _check_into(queries, queries.shape[1] if getattr(queries, "ndim", 0) == 2 else -1, k, out_ids, out_dists)
        st = SearchStats()
        self._lib.check(self._lib.lib.rd_group_search(self._h, _fp(queries), queries.shape[0], nprobe, k,
                                                      _i64p(out_ids), _fp(out_dists), C.byref(st)), "group_search")
        return st.as_dict()

    def search_device(self, q_ptr: int, B: int, nprobe: int, k: int, ids_ptr: int, dists_ptr: int,
                      stream: int = 0, sync: bool = False) -> dict:
        st = SearchStats()
        self._lib.check(self._lib.lib.rd_group_search_device(self._h, C.c_void_p(q_ptr), B, nprobe, k,
                                                             C.c_void_p(ids_ptr), C.c_void_p(dists_ptr),
                                                             C.c_void_p(stream), 1 if sync else 0, C.byref(st)),
                        "group_search_device")
        return st.as_dict()


_ENGINE: Optional[Library] = None


def engine() -> Library:
    """The B200 engine library (raises if not built). RD_ENGINE_PATH points at another build of the
    same engine (A/B measurements only)."""
    global _ENGINE
    if _ENGINE is None:
        _ENGINE = Library(os.environ.get("RD_ENGINE_PATH") or ENGINE_PATH)
    return _ENGINE
