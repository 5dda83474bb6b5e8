"""bench.py — RAGDoll retrieval stage on B200: IVF-Flat top-k queries/sec.

Workload (BASELINE.json configs[1], the metric's config): 10M x 768 fp32
synthetic vectors, nlist 4096, nprobe 64, k 10, query batch 1024, fully
HBM-resident. One step = one search of one batch of synthetic queries.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1|c3|c5] [--batch B]

value       : whole-job queries/s with queries already in HBM (device timing,
              CUDA events on the search stream, max over ranks).
e2e         : same metric through the public C-ABI rd_search with host
              buffers: H2D of the queries and D2H of ids+distances every step.
roofline    : the dominant kernel (N4 list scan): algorithmic bytes of the
              probed lists' vectors per launch / its CUDA-event duration.
cpu_baseline: the exact CPU oracle (oracle/librd_cpu.so; the reference has no
              search) on a bounded query sample, rank 0, N=1;
cpu_baseline_batched: the batched list-major CPU search (oracle/rd_cpu_batched.c,
              identical results) over whole batches, and the GPU's ratio to it.
--impl reference: the batched CPU search over the whole configured batch every
              step (the exact oracle's sample rate beside it).
Inputs are larger than L2 (30.7 GB index), so no explicit flush is needed.
N>1: the config's knowledge base is split into N row stripes of every list
(strong scaling: 10M rows split N ways), one per GPU, searched as one shard group
(rd_group_*): under torchrun one process per GPU (NCCL gather of the per-stripe
top-k to rank 0 and a device merge, inside the library); `--gpus N` without
torchrun, one process driving N GPUs.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n per GPU, d, nlist, nprobe, k, batch, offload_fraction, workload label)
    "c1": dict(n=1_000_000, d=768, nlist=1024, nprobe=32, k=10, batch=32, offload=0.0,
               workload="ivf-flat 1M x 768 fp32, nlist 1024, nprobe 32, k 10, batch 32, HBM-resident"),
    "c2": dict(n=10_000_000, d=768, nlist=4096, nprobe=64, k=10, batch=1024, offload=0.0,
               workload="ivf-flat 10M x 768 fp32, nlist 4096, nprobe 64, k 10, batch 1024, HBM-resident"),
    "c3": dict(n=10_000_000, d=768, nlist=4096, nprobe=64, k=10, batch=1024, offload=0.5,
               workload="ivf-flat 10M x 768 fp32, nlist 4096, nprobe 64, k 10, batch 1024, 50% lists in pinned host DRAM"),
    # C4: 100M x 768 sharded over the GPUs of one box (nlist 16384, nprobe 64 — BASELINE leaves them
    # open; SURVEY §7 recommends these). With one GPU, one shard of 8 (12.5M rows) is run: the work
    # of one rank of the 8-GPU job.
    "c4": dict(n=100_000_000, d=768, nlist=16384, nprobe=64, k=10, batch=1024, offload=0.0, total=True,
               workload="ivf-flat 100M x 768 fp32 sharded over the box's GPUs, nlist 16384, nprobe 64, k 10, batch 1024"),
    "c5": dict(n=10_000_000, d=768, nlist=4096, nprobe=128, k=20, batch=64, offload=None, llm="70b",
               workload="ivf-flat 10M x 768 fp32, nlist 4096, nprobe 128, k 20, batch 64, under a 70B LLM-decode HBM reservation"),
    # C2's search under the reference's default 8B model (configs/default_8b.json:11-19) resident
    # beside it: the budget leaves room for the whole index in the fast (split3) store
    "c2r8b": dict(n=10_000_000, d=768, nlist=4096, nprobe=64, k=10, batch=1024, offload=None, llm="8b",
                  workload="ivf-flat 10M x 768 fp32, nlist 4096, nprobe 64, k 10, batch 1024, under an 8B LLM-decode HBM reservation"),
}
METRIC = "IVF top-k queries/sec at 10M×768 nprobe=64 k=10; achieved HBM GB/s vs peak"


def measure_h2d_gbs(nbytes: int = 1 << 30, reps: int = 5) -> float:
    """Pinned host -> device copy bandwidth (the offloaded lists' link), best of `reps`."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dbuf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dbuf.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del h, dbuf
    return best


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class DecodeStream:
    """A synthetic LLM decode running beside the retrieval (C5 / C2r8b): on its own CUDA stream, back
    to back, the decode GEMMs of a batch of 64 tokens against bf16 weight matrices carved from the
    reserved bytes (every step reads every weight once, as a w_gpu = 1 decode does). Reports the
    weight bytes it streamed per second while the timed region ran."""

    def __init__(self, hold, batch=64, dim=8192):
        import torch
        self.torch = torch
        n = hold.numel() // 2 // (dim * dim)  # whole [dim x dim] bf16 matrices in the reservation
        self.mats = [hold[i * dim * dim * 2:(i + 1) * dim * dim * 2].view(torch.bfloat16).view(dim, dim)
                     for i in range(max(0, min(n, 256)))]
        self.x = torch.randn(batch, dim, device="cuda", dtype=torch.bfloat16)
        self.stream = torch.cuda.Stream()
        self.bytes = 0
        self._stop = threading.Event()

    def __enter__(self):
        torch = self.torch
        if not self.mats:
            return self
        self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.e0.record(self.stream)

        def run():
            with torch.cuda.stream(self.stream):
                while not self._stop.is_set():
                    for w in self.mats:
                        torch.mm(self.x, w)
                        self.bytes += w.numel() * 2
                    self.stream.synchronize()  # bounded queue: at most one pass in flight

        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        if not self.mats:
            return
        self._stop.set()
        self.t.join()
        self.e1.record(self.stream)
        self.e1.synchronize()
        self.seconds = self.e0.elapsed_time(self.e1) / 1000.0

    def summary(self):
        if not self.mats:
            return None
        return {"weight_gbs": self.bytes / self.seconds / 1e9, "matrices": len(self.mats),
                "what": "bf16 decode GEMMs (64 tokens x 8192 x 8192) over the reserved bytes, back to back on "
                        "a side stream during the timed region"}


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every 10 ms) during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm, self.mx, self.flags = [], [], 0
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.mx.append(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.flags |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.01)

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted(v for k, v in self.REASONS.items() if self.flags & k)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx), "reasons": reasons,
                "samples": len(self.sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def llm_reservation(lib, model="70b"):
    """RAGDoll placement: the LLM fully on the GPU in decode at gen batch 64; reservation =
    w_gpu*W + c_gpu*C(B) + H(B)*0.25 (memory_planner.cpp:20, prefetch_timeline.cpp:85-86).
    70b: configs/ref_70b.json:11-19 (C5); 8b: configs/default_8b.json:11-19."""
    GiB, MiB = 1 << 30, 1 << 20
    W, kv, ws = (140 * GiB, 256 * MiB, 128 * MiB) if model == "70b" else (16 * GiB, 128 * MiB, 64 * MiB)
    return lib.llm_reservation_bytes(weight_total=W, kv_bytes_per_request=kv, workspace_bytes_per_request=ws,
                                     w_gpu=1.0, c_gpu=1.0, gen_batch_size=64, decode_phase=1,
                                     workspace_fraction=0.25)


def c5_reservation(lib):
    return llm_reservation(lib, "70b")


def oracle_lib():
    """The CPU oracle (exact IVF-Flat; test infrastructure), built on demand."""
    from paper_2504_15302_b200.retriever import Library
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    return Library(os.path.join(ROOT, "oracle", "librd_cpu.so"))


def cpu_desc_args(cfg, shards):
    """The knowledge base the CPU path holds: the whole config, except C4 (307 GB) where it is the
    row stripe one GPU of the N-GPU job holds (1 of 8 at N = 1)."""
    if cfg.get("total"):
        return dict(n=cfg["n"], d=cfg["d"], nlist=cfg["nlist"], shard=0, num_shards=shards)
    return dict(n=cfg["n"], d=cfg["d"], nlist=cfg["nlist"])


def cpu_baseline(cfg, desc_args, sample, steps=1, batch_of=None, batched_of=None):
    """Times the CPU oracle on `sample` queries of the same workload per step (rank 0, N=1).
    batch_of(s) gives step s's full query batch (the GPU arm's); its first `sample` queries are
    timed. Returns the per-step rates and the last step's queries and results (the parity check)."""
    oracle = oracle_lib()
    desc = oracle.desc(**desc_args)
    t0 = time.time()
    idx = oracle.synthetic_index(desc)
    build_s = time.time() - t0
    cores = len(os.sched_getaffinity(0))
    vals = []
    q = res = None
    for s in range(steps):
        q = batch_of(s)[:sample] if batch_of else oracle.synth_queries(desc, 10_000_000 + s * sample, sample)[0]
        t0 = time.perf_counter()
        res = idx.search(q, cfg["nprobe"], cfg["k"])
        vals.append(sample / (time.perf_counter() - t0))
    batched = None
    if batched_of is not None:  # the batched CPU search over whole batches, same index
        bv, bout = cpu_batched(idx, oracle, batched_of, cfg["nprobe"], cfg["k"])
        batched = {"per_step": bv, "ids": bout[0], "dists": bout[1], "fallbacks": bout[2]}
    idx.close()
    cpu = cpu_model()
    return {"value": statistics.median(vals), "unit": "queries/s", "cores": cores, "kind": "port",
            "cpu_model": cpu,
            "sample": f"first {sample} queries of each step's batch, exact IVF-Flat (fp64 canonical distances, "
                      f"query-at-a-time), {cores} threads on {cpu} (index build {build_s:.1f}s untimed)",
            "per_step": vals, "queries": q, "result": res, "batched": batched}


def cpu_batched(oracle_idx, oracle, batches, nprobe, k):
    """The batched list-major CPU search (oracle/rd_cpu_batched.c: the tuned-CPU-retriever
    baseline, results identical to the exact oracle) over whole batches: one untimed warm-up (the
    row norms), then each batch timed. Returns (per-batch q/s, last result ids/dists, fallbacks)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_ext import batched_search
    batched_search(oracle, oracle_idx, batches[0][: min(8, len(batches[0]))], nprobe, k)  # prepare
    vals, out = [], None
    for q in batches:
        t0 = time.perf_counter()
        out = batched_search(oracle, oracle_idx, q, nprobe, k)
        vals.append(len(q) / (time.perf_counter() - t0))
    return vals, out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_block(cfg, B, n_gpus, shards):
    per = cfg["n"] // shards
    return {"workload": cfg["workload"], "global_batch": B, "nprobe": cfg["nprobe"], "k": cfg["k"],
            "n_total": cfg["n"], "n_per_gpu": per, "nlist": cfg["nlist"], "d": cfg["d"],
            "parallelism": f"shard{n_gpus}" if shards == n_gpus else f"one shard of {shards} on 1 GPU",
            "l2": "inputs larger than L2 (index %.1f GB per GPU)" % (per * cfg["d"] * 4 / 1e9)}


def shards_for(cfg, n_gpus, stripe_of):
    # The knowledge base is the config's (the metric is quoted "at 10M x 768"): N GPUs split it into
    # N row stripes of every list (strong scaling). C4 (100M) does not fit one GPU: there N = 1 runs
    # one stripe of 8, the per-rank work of the 8-GPU job.
    if n_gpus > 1:
        return n_gpus
    if stripe_of > 1:
        return stripe_of
    return 8 if cfg.get("total") else 1


def run_reference(args, cfg):
    """The reference's CPU path on the box's host cores. The reference has no search of its own
    (SPEC.md:9), so its CPU path is the oracle library's: the batched list-major IVF-Flat search
    (oracle/rd_cpu_batched.c; results identical to the exact oracle) over the whole configured batch
    every step, all host threads, this arm's config. The exact query-at-a-time oracle is timed on a
    sample beside it (cpu_exact)."""
    world, rank, _ = dist_env()
    n_gpus = world if world > 1 else args.gpus
    shards = shards_for(cfg, n_gpus, args.stripe_of)
    B = cfg["batch"]
    line = {"metric": METRIC, "impl": "reference", "unit": "queries/s", "higher_is_better": True,
            "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
            "dtype": "f32 (f64 exact distances)", "data": "synthetic (splitmix64 spec, SURVEY §8d)",
            "config": config_block(cfg, B, n_gpus, shards)}
    if rank != 0:
        return
    oracle = oracle_lib()
    desc_full = oracle.desc(cfg["n"], cfg["d"], cfg["nlist"])
    nb = args.warmup + args.steps
    batches = [oracle.synth_queries(desc_full, s * B, B)[0] for s in range(nb)]
    sample = min(args.cpu_sample, B)
    res = cpu_baseline(cfg, cpu_desc_args(cfg, shards), sample, steps=1, batch_of=lambda s: batches[-1],
                       batched_of=batches)
    vals = res["batched"]["per_step"][args.warmup:]
    v = statistics.median(vals)
    line.update({"value": v, "ms_per_step": 1000.0 * B / v, "scaling": "replicas only",
                 "vs_baseline": None,
                 "cpu_baseline": {"value": v, "unit": "queries/s", "cores": res["cores"], "kind": "port",
                                  "variant": "batched list-major IVF-Flat (oracle/rd_cpu_batched.c)",
                                  "cpu_model": res["cpu_model"],
                                  "sample": f"the whole batch of {B} queries every step, {res['cores']} threads on "
                                            f"{res['cpu_model']}; exact fallbacks "
                                            f"{res['batched']['fallbacks']} in the last step"},
                 "cpu_exact": {"value": res["value"], "unit": "queries/s", "sample": res["sample"]},
                 "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import torch
    from paper_2504_15302_b200.retriever import engine

    world, rank, local = dist_env()
    lib = engine()
    B, k, nprobe, d = cfg["batch"], cfg["k"], cfg["nprobe"], cfg["d"]
    n_total = cfg["n"]
    ndev = torch.cuda.device_count()
    # Multi-GPU through the library's shard groups (rd_group_*): under torchrun one process per GPU
    # (rd_group_create_rank: NCCL gather of the per-stripe top-k to rank 0 + device merge, inside the
    # library); `--gpus N` without torchrun, one process driving N GPUs (rd_group_create_synthetic:
    # ncclCommInitAll). torch.distributed (gloo) only carries the group id, barriers and the max over
    # ranks of the device-timed step.
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        local = local % max(1, ndev)
        n_gpus = world
    else:
        dist = None
        n_gpus = args.gpus
        # RD_BENCH_DEVICES=0,0 maps the stripes onto given devices: exercises the one-process group
        # path on a one-GPU box (device copies instead of NCCL); not a scaling measurement
        devices = [int(x) for x in os.environ["RD_BENCH_DEVICES"].split(",")] if os.environ.get(
            "RD_BENCH_DEVICES") else list(range(n_gpus))
        if len(devices) != n_gpus or max(devices) >= ndev:
            raise SystemExit(f"--gpus {n_gpus}: only {ndev} CUDA devices visible")
    torch.cuda.set_device(local)
    shards = shards_for(cfg, n_gpus, args.stripe_of)
    t0 = time.time()
    grp = None
    if world > 1:
        desc = lib.desc(n_total, d, cfg["nlist"], shard=rank, num_shards=shards)
        idx0 = lib.synthetic_index(desc, device=local)
        obj = [lib.group_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        grp = lib.rank_group(idx0, obj[0], world, rank)
    elif n_gpus > 1:
        desc = lib.desc(n_total, d, cfg["nlist"], shard=0, num_shards=shards)
        grp = lib.synthetic_group(lib.desc(n_total, d, cfg["nlist"]), devices)
    else:
        desc = lib.desc(n_total, d, cfg["nlist"], shard=0, num_shards=shards)
        idx0 = lib.synthetic_index(desc, device=local)
    build_s = time.time() - t0
    searcher = grp if grp is not None else idx0
    stripe = grp.shard(0) if grp is not None else idx0  # this process's (first) stripe: stats, timing
    reservation = None
    heat = None
    if cfg["offload"] is None or cfg["offload"] > 0:
        # joint placement pins the hot lists: probe frequency from a calibration batch of queries
        # disjoint from the timed ones (north_star item 4); probe sets are the same on every stripe
        cal, _ = lib.synth_queries(desc, 50_000_000, 4096)
        pr = stripe.probe(cal, nprobe)
        heat = np.bincount(pr[pr >= 0].ravel(), minlength=cfg["nlist"]).astype(np.uint32)
    if cfg["offload"] is None:  # C5 / C2r8b: budget = device memory - LLM reservation - engine workspace
        free, total = torch.cuda.mem_get_info()
        reservation = llm_reservation(lib, cfg["llm"])
        budget = int(total - reservation - (4 << 30))
        searcher.place(hbm_budget_bytes=budget, list_heat=heat)
    elif cfg["offload"] > 0:
        searcher.place(offload_fraction=cfg["offload"], list_heat=heat)
    info = stripe.info()
    hold = None
    if reservation is not None:  # actually hold the LLM's bytes while searching
        free, _ = torch.cuda.mem_get_info()
        hold = torch.empty(int(min(reservation, free - (6 << 30))), dtype=torch.uint8, device="cuda")

    nb = args.warmup + args.steps
    full = lib.desc(n_total, d, cfg["nlist"])
    qs = [lib.synth_queries(full, i * B, B)[0] for i in range(nb)]
    dq = [torch.from_numpy(q).cuda() for q in qs]
    di = torch.empty((B, k), dtype=torch.int64, device="cuda")
    dd = torch.empty((B, k), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def step(i):  # one search of one batch; at N > 1 the merged top-k lands on rank 0 / device 0
        searcher.search_device(dq[i].data_ptr(), B, nprobe, k, di.data_ptr(), dd.data_ptr(), stream=sptr)

    def barrier():
        if dist is not None:
            dist.barrier()

    # correctness / certification and this stripe's scan bytes on one synced search
    st = searcher.search_device(dq[0].data_ptr(), B, nprobe, k, di.data_ptr(), dd.data_ptr(), stream=sptr, sync=True)
    # one stripe's counters (the roofline is per GPU): a one-process group's stats sum its stripes
    st1 = stripe.search_device(dq[0].data_ptr(), B, nprobe, k, di.data_ptr(), dd.data_ptr(), stream=sptr,
                               sync=True) if grp is not None and world == 1 else st
    # the read-only stream peak of this GPU with the scan's load pattern, measured before the timed
    # region (a copy counts read + write bytes; a pure read stream runs faster on HBM3e)
    try:
        read_peak = lib.device_read_bandwidth(local, 8 << 30)
    except Exception:
        pk = measured_peaks()
        read_peak = pk.get("hbm_read_gbs") if pk else None
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier()
    # per-stage events inside the timed region: the scan kernel's own duration for the roofline
    # (they cost the chain its launch overlap, ~12 us per search; e2e and the sweep run without)
    stripes = [grp.shard(g) for g in range(grp.info()["local_shards"])] if grp is not None else [idx0]
    for sx in stripes:
        sx.timing_stages(True)
        sx.timing_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import contextlib
    decode = DecodeStream(hold) if (hold is not None and args.decode_stream) else None
    with ClockSampler(local) as clk, (decode if decode is not None else contextlib.nullcontext()):
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        for i in range(args.warmup, nb):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    tms = [sx.timing_read() for sx in stripes]
    for sx in stripes:
        sx.timing_stages(False)
    tm = max(tms, key=lambda t: t["scan_ms"])  # the slowest stripe bounds the step
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = B * args.steps / (ms / 1000.0)

    # e2e: the public C-ABI (rd_search / rd_group_search) with pinned host buffers (H2D queries +
    # D2H ids/dists every step, inside the timed region); at N > 1 a collective group call
    hq = [torch.from_numpy(q).pin_memory().numpy() for q in qs]
    hi = torch.empty((B, k), dtype=torch.int64).pin_memory().numpy()
    hd = torch.empty((B, k), dtype=torch.float32).pin_memory().numpy()
    for i in range(min(args.warmup, 2)):
        searcher.search_into(hq[i], nprobe, k, hi, hd)
    barrier()
    with (DecodeStream(hold) if decode is not None else contextlib.nullcontext()):  # same concurrent decode
        t0 = time.perf_counter()
        for i in range(args.warmup, nb):
            searcher.search_into(hq[i], nprobe, k, hi, hd)
        barrier()
        e2e_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": B * args.steps / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": B * d * 4,
           "d2h_bytes_per_step": B * k * 12}

    # batch sweep of BASELINE configs[1] (same index, queries in HBM): q/s per batch size
    sweep = {}
    if n_gpus == 1 and not args.no_sweep and args.config == "c2":
        for Bs in (1, 8, 32, 64, 128, 256, 512, 1024):
            qs_s = torch.from_numpy(lib.synth_queries(desc, 70_000_000 + Bs, Bs)[0]).cuda()
            oi = torch.empty((Bs, k), dtype=torch.int64, device="cuda")
            od = torch.empty((Bs, k), dtype=torch.float32, device="cuda")
            for _ in range(3):
                idx0.search_device(qs_s.data_ptr(), Bs, nprobe, k, oi.data_ptr(), od.data_ptr(), stream=sptr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(reps):
                idx0.search_device(qs_s.data_ptr(), Bs, nprobe, k, oi.data_ptr(), od.data_ptr(), stream=sptr)
            e1.record(stream)
            torch.cuda.synchronize()
            sweep[str(Bs)] = Bs * reps / (e0.elapsed_time(e1) / 1000.0)

    # roofline of the dominant kernel (the resident list scan) of this process's slowest stripe
    peaks = measured_peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    scan_ms = tm["scan_ms"] / max(1, tm["stage_searches"])
    scan_bytes = st1["bytes_lists_resident"]  # probed resident rows x d x 4 (SURVEY §8d's per-row unit)
    fp32_equiv = None
    if info["store"] in (3, 4):  # residual store: the scan reads r1 (d x 2 B) and ||x - c||^2 (4 B) per row
        rows = scan_bytes // (d * 4)
        fp32_equiv = {"bytes_per_launch": scan_bytes,
                      "gbs": scan_bytes / (scan_ms * 1e-3) / 1e9 if scan_ms > 0 else 0.0,
                      "note": "the same rows at fp32 (3072 B per row): the rate an fp32 scan would need"}
        scan_bytes = rows * (d * 2 + 4)
    achieved = scan_bytes / (scan_ms * 1e-3) / 1e9 if scan_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "scan_traffic.json")
    # the captured traffic is of one unsharded launch at the config's default batch: only that
    # workload may quote it
    if os.path.exists(tpath) and shards == 1 and not args.batch:
        traffic = json.load(open(tpath)).get(args.config)
    h2d_link = None
    if st1["h2d_list_bytes"] > 0:  # offloaded lists: the host link is the roofline of that part
        link = measure_h2d_gbs()
        ach = st1["h2d_list_bytes"] / (ms_step * 1e-3) / 1e9
        h2d_link = {"achieved": ach, "peak": link, "unit": "GB/s", "frac": ach / link,
                    "bytes_per_step": st1["h2d_list_bytes"],
                    "peak_source": "measured in this run: pinned 1 GiB host->device cudaMemcpy, best of 5",
                    "note": "achieved over the whole step: the resident scan and merge overlap or follow the stream"}

    if rank != 0:
        if grp is not None:
            grp.close()
        dist.destroy_process_group()
        return
    # (read_peak: measured before the timed region, see below)
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (splitmix64 spec, SURVEY §8d), generated on device",
        "scaling": "strong",
        "config": config_block(cfg, B, n_gpus, shards),
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("ivf_scan_tc_kernel (N5 over the residual store: 16-bit r1 = x - c tiles)" if info["store"] in (3, 4)
                                else "ivf_scan_tc_kernel (N5; FFMA ivf_scan_kernel N4 when d % 64 != 0)"),
                     "peak_source": ("MEASURED_PEAKS.json hbm_gbs (a torch copy: read + write bytes); a read-only "
                                     "stream of the scan's TMA pattern reaches ~7.46 TB/s (tools/micro/bw.cu)")
                     if peaks else "fallback",
                     "bytes_per_launch": scan_bytes, "avg_launch_ms": scan_ms, "fp32_equivalent": fp32_equiv,
                     "stripe": "per GPU (this process's slowest stripe)" if n_gpus > 1 else "the index"},
        "step_breakdown_ms": {k2: tm[k2] / max(1, tm["stage_searches"]) for k2 in ("coarse_ms", "scan_ms", "tail_ms", "total_ms")},
        "step_gbps_algorithmic": st["bytes_algorithmic"] / (ms_step * 1e-3) / 1e9,
        "gpu_launches": st["kernel_launches"] * args.steps,
        "batch_sweep_qps": sweep,
        "clocks": clk.summary(),
        "certified": {"margin_failures": st["margin_failures"], "probe_failures": st["probe_failures"]},
        "h2d_link": h2d_link,
        "decode_stream": decode.summary() if decode is not None else None,
        "index": {"build_s": build_s, "lists_resident": info["lists_resident"], "hbm_bytes": info["hbm_bytes"],
                  "store": {0: "fp32", 1: "fp32 + pre-split copy", 2: "split3 (exact bf16 triple)",
                            3: "fp32 + bf16 residual plane (scan reads 2 B/element)",
                            4: "fp32 + fp16 residual plane (scan reads 2 B/element)"}.get(info["store"]),
                  "fp32_bytes": info["n"] * d * 4,
                  "host_pinned_bytes": info["host_pinned_bytes"], "h2d_list_bytes_per_step": st1["h2d_list_bytes"],
                  "llm_reservation_bytes": reservation},
    }
    if grp is not None:
        gi = grp.info()
        line["group"] = {"transport": gi["transport"], "num_shards": gi["num_shards"], "local_shards": gi["local_shards"]}
    if read_peak:
        line["roofline"]["read_peak"] = read_peak
        line["roofline"]["frac_of_read_peak"] = achieved / read_peak
        line["roofline"]["read_peak_source"] = ("rd_device_read_bandwidth in this run: persistent CTAs, 32 KiB bulk "
                                                "(TMA) stages released on arrival, 8 GiB, best of 5")
    if n_gpus == 1 and not args.no_cpu_baseline:
        # the CPU path on the first queries of the last timed batch, then the engine on those same
        # queries (outside every timed region): the parity check of this run
        sample = min(args.cpu_sample, B)
        cb = cpu_baseline(cfg, cpu_desc_args(cfg, shards), sample, batch_of=lambda s: qs[nb - 1],
                          batched_of=[qs[nb - 2], qs[nb - 1]] if nb >= 2 else [qs[nb - 1]])
        mine = idx0.search(cb["queries"], nprobe, k)
        want = cb["result"]
        line["parity"] = {"checked": int(sample),
                          "ids_equal": int((mine.ids == want.ids).all(axis=1).sum()),
                          "dists_equal": int((mine.dists == want.dists).all(axis=1).sum()),
                          "oracle": "oracle/librd_cpu.so (exact IVF-Flat, canonical fp64 distances)",
                          "data": "the whole knowledge base" if shards == 1 else f"stripe 0 of {shards}"}
        bt = cb.pop("batched")
        full = idx0.search(qs[nb - 1], nprobe, k)  # the whole last timed batch vs the batched CPU search
        line["parity_full_batch"] = {"checked": int(B),
                                     "ids_equal": int((full.ids == bt["ids"]).all(axis=1).sum()),
                                     "dists_equal": int((full.dists == bt["dists"]).all(axis=1).sum()),
                                     "oracle": "oracle/rd_cpu_batched.c (bit-identical to the exact oracle: "
                                               "tests/test_cpu_batched.py)"}
        for key in ("per_step", "queries", "result"):
            cb.pop(key, None)
        line["cpu_baseline"] = cb
        bval = statistics.median(bt["per_step"])
        line["cpu_baseline_batched"] = {
            "value": bval, "unit": "queries/s", "cores": cb["cores"], "kind": "batched",
            "cpu_model": cb["cpu_model"],
            "sample": f"the whole batch ({B} queries), list-major: probes inverted per list, each list read "
                      f"once per batch against its query group (fp32 AVX2/FMA dots), certified, exact canonical "
                      f"rerank (oracle/rd_cpu_batched.c), {cb['cores']} threads; median of "
                      f"{len(bt['per_step'])} batches; exact fallbacks {bt['fallbacks']}",
            "gpu_over_cpu": value / bval, "gpu_e2e_over_cpu": e2e["value"] / bval}
    print(json.dumps(line), flush=True)
    if grp is not None:
        grp.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=128,
                    help="exact-oracle queries timed per step (the batched CPU search takes whole batches)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--decode-stream", action="store_true",
                    help="C5 / C2r8b: run synthetic decode GEMMs over the reserved bytes on a side stream during "
                         "the timed regions")
    ap.add_argument("--stripe-of", type=int, default=0,
                    help="N = 1 only: run one row stripe of an N-way split (the per-rank work of N GPUs)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = dict(CONFIGS[args.config])
    if args.batch:
        cfg["batch"] = args.batch
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
