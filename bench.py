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
cpu_baseline: the CPU oracle (oracle/librd_cpu.so — the only CPU IVF path;
              the reference has none) on a bounded query sample, rank 0, N=1.
--impl reference: that same CPU path as the timed arm.
Inputs are larger than L2 (30.7 GB index), so no explicit flush is needed.
N>1 (torchrun): each rank holds a row stripe of every list of the config's
knowledge base (strong scaling: 10M rows split N ways), searches the same batch,
and rank 0 merges the NCCL-gathered per-shard top-k on the device.
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
    "c5": dict(n=10_000_000, d=768, nlist=4096, nprobe=128, k=20, batch=64, offload=None,
               workload="ivf-flat 10M x 768 fp32, nlist 4096, nprobe 128, k 20, batch 64, under a 70B LLM-decode HBM reservation"),
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


def c5_reservation(lib):
    """RAGDoll placement for C5: ref_70b model (configs/ref_70b.json:11-19) fully on the GPU
    in decode at gen batch 64; reservation = w_gpu*W + c_gpu*C(B) + H(B)*0.25
    (memory_planner.cpp:20, prefetch_timeline.cpp:85-86)."""
    GiB, MiB = 1 << 30, 1 << 20
    return lib.llm_reservation_bytes(weight_total=140 * GiB, kv_bytes_per_request=256 * MiB,
                                     workspace_bytes_per_request=128 * MiB, w_gpu=1.0, c_gpu=1.0,
                                     gen_batch_size=64, decode_phase=1, workspace_fraction=0.25)


def cpu_baseline(cfg, desc_args, sample, steps=1):
    """Times the CPU oracle on `sample` queries of the same workload (rank 0, N=1)."""
    from paper_2504_15302_b200.retriever import Library
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    oracle = Library(os.path.join(ROOT, "oracle", "librd_cpu.so"))
    desc = oracle.desc(**desc_args)
    t0 = time.time()
    idx = oracle.synthetic_index(desc)
    build_s = time.time() - t0
    cores = len(os.sched_getaffinity(0))
    vals = []
    for s in range(steps):
        q, _ = oracle.synth_queries(desc, 10_000_000 + s * sample, sample)
        t0 = time.perf_counter()
        idx.search(q, cfg["nprobe"], cfg["k"])
        vals.append(sample / (time.perf_counter() - t0))
    idx.close()
    return {"value": statistics.median(vals), "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": f"{sample} queries of the same workload per step, exact IVF-Flat, {cores} threads "
                      f"(index build {build_s:.1f}s untimed)", "per_step": vals}


def run_reference(args, cfg):
    world, rank, _ = dist_env()
    line = {"metric": METRIC, "impl": "reference", "unit": "queries/s", "higher_is_better": True,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "dtype": "f32 (f64 exact distances)", "data": "synthetic (splitmix64 spec, SURVEY §8d)",
            "config": {"workload": cfg["workload"], "global_batch": cfg["batch"], "nprobe": cfg["nprobe"],
                       "k": cfg["k"], "n": cfg["n"], "nlist": cfg["nlist"], "d": cfg["d"]}}
    if rank != 0:
        return
    sample = args.cpu_sample
    desc_args = dict(n=cfg["n"], d=cfg["d"], nlist=cfg["nlist"])
    res = cpu_baseline(cfg, desc_args, sample, steps=args.warmup + args.steps)
    vals = res["per_step"][args.warmup:]
    v = statistics.median(vals)
    line.update({"value": v, "ms_per_step": 1000.0 * sample / v, "scaling": "replicas only",
                 "vs_baseline": None,
                 "cpu_baseline": {"value": v, "unit": "queries/s", "cores": res["cores"], "kind": "port",
                                  "sample": res["sample"]},
                 "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_2504_15302_b200.retriever import engine

    world, rank, local = dist_env()
    # one process per GPU; RD_DIST_BACKEND=gloo (with ranks sharing a device) only exercises the
    # multi-rank code path on a single-GPU box
    backend = os.environ.get("RD_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
    torch.cuda.set_device(local)
    lib = engine()
    B, k, nprobe, d = cfg["batch"], cfg["k"], cfg["nprobe"], cfg["d"]
    # The knowledge base is the config's (the metric is quoted "at 10M x 768"): N GPUs split it into N
    # row stripes of every list (strong scaling). C4 (100M) does not fit one GPU: there N = 1 runs
    # one stripe of 8, the per-rank work of the 8-GPU job.
    n_total = cfg["n"]
    shards = world if (world > 1 or not cfg.get("total")) else 8
    if args.stripe_of > 1 and world == 1:  # one rank's share of an N-GPU run, on one GPU
        shards = args.stripe_of
    desc = lib.desc(n_total, d, cfg["nlist"], shard=rank, num_shards=shards)
    t0 = time.time()
    idx = lib.synthetic_index(desc, device=local)
    build_s = time.time() - t0
    reservation = None
    heat = None
    if cfg["offload"] is None or cfg["offload"] > 0:
        # joint placement pins the hot lists: probe frequency from a calibration batch of queries
        # disjoint from the timed ones (north_star item 4)
        cal, _ = lib.synth_queries(desc, 50_000_000, 4096)
        pr = idx.probe(cal, nprobe)
        heat = np.bincount(pr[pr >= 0].ravel(), minlength=cfg["nlist"]).astype(np.uint32)
    if cfg["offload"] is None:  # C5: budget = device memory - LLM reservation - engine workspace
        free, total = torch.cuda.mem_get_info()
        reservation = c5_reservation(lib)
        budget = int(total - reservation - (4 << 30))
        idx.place(hbm_budget_bytes=budget, list_heat=heat)
    elif cfg["offload"] > 0:
        idx.place(offload_fraction=cfg["offload"], list_heat=heat)
    info = idx.info()
    hold = None
    if reservation is not None:  # actually hold the LLM's bytes while searching
        free, _ = torch.cuda.mem_get_info()
        hold = torch.empty(int(min(reservation, free - (6 << 30))), dtype=torch.uint8, device="cuda")

    nb = args.warmup + args.steps
    qs = [lib.synth_queries(desc, i * B, B)[0] for i in range(nb)]
    dq = [torch.from_numpy(q).cuda() for q in qs]
    # one packed result buffer per rank ([B, k] ids then [B, k] distances) so the exchange is a
    # single all-gather of B * k * 12 bytes
    nbi = B * k * 8
    res8 = torch.empty(B * k * 12, dtype=torch.uint8, device="cuda")
    di = res8[:nbi].view(torch.int64).view(B, k)
    dd = res8[nbi:].view(torch.float32).view(B, k)
    gres = [torch.empty_like(res8) for _ in range(world)]
    mi = torch.empty((B, k), dtype=torch.int64, device="cuda")
    md = torch.empty((B, k), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def step(i):
        idx.search_device(dq[i].data_ptr(), B, nprobe, k, di.data_ptr(), dd.data_ptr(), stream=sptr)
        if world > 1:
            dist.all_gather(gres, res8)
            if rank == 0:
                g = torch.stack(gres)
                ti, td = g[:, :nbi].contiguous(), g[:, nbi:].contiguous()  # [G][B][k] ids, distances
                lib.check(lib.lib.rd_merge_topk_device(world, B, k, ti.data_ptr(), td.data_ptr(), mi.data_ptr(),
                                                       md.data_ptr(), sptr), "merge")

    # correctness / certification on one synced search
    st = idx.search_device(dq[0].data_ptr(), B, nprobe, k, di.data_ptr(), dd.data_ptr(), stream=sptr, sync=True)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-stage events inside the timed region: the scan kernel's own duration for the roofline
    # (they cost the chain its launch overlap, ~12 us per search; e2e and the sweep run without)
    idx.timing_stages(True)
    idx.timing_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        for i in range(args.warmup, nb):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    tm = idx.timing_read()
    idx.timing_stages(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = B * args.steps / (ms / 1000.0)

    # e2e: public C-ABI rd_search with pinned host buffers (H2D queries + D2H ids/dists every
    # step, inside the timed region); at N > 1 every rank searches its shard and rank 0 merges
    # the gathered per-shard results with rd_merge_topk (host)
    hq = [torch.from_numpy(q).pin_memory().numpy() for q in qs]
    hi = torch.empty((B, k), dtype=torch.int64).pin_memory().numpy()
    hd = torch.empty((B, k), dtype=torch.float32).pin_memory().numpy()

    def e2e_step(i):
        idx.search_into(hq[i], nprobe, k, hi, hd)
        if world > 1:
            di.copy_(torch.from_numpy(hi), non_blocking=True)
            dd.copy_(torch.from_numpy(hd), non_blocking=True)
            dist.all_gather(gres, res8)
            if rank == 0:
                g = torch.stack(gres).cpu()
                gi = g[:, :nbi].contiguous().view(torch.int64).view(world, B, k).numpy()
                gd = g[:, nbi:].contiguous().view(torch.float32).view(world, B, k).numpy()
                lib.merge_topk(gi, gd)

    for i in range(min(args.warmup, 2)):
        e2e_step(i)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.warmup, nb):
        e2e_step(i)
    if world > 1:
        dist.barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": B * args.steps / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": B * d * 4,
           "d2h_bytes_per_step": B * k * 12}

    # batch sweep of BASELINE configs[1] (same index, queries in HBM): q/s per batch size
    sweep = {}
    if world == 1 and not args.no_sweep and args.config == "c2":
        for Bs in (1, 8, 32, 64, 128, 256, 512, 1024):
            qs_s = torch.from_numpy(lib.synth_queries(desc, 70_000_000 + Bs, Bs)[0]).cuda()
            oi = torch.empty((Bs, k), dtype=torch.int64, device="cuda")
            od = torch.empty((Bs, k), dtype=torch.float32, device="cuda")
            for _ in range(3):
                idx.search_device(qs_s.data_ptr(), Bs, nprobe, k, oi.data_ptr(), od.data_ptr(), stream=sptr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(reps):
                idx.search_device(qs_s.data_ptr(), Bs, nprobe, k, oi.data_ptr(), od.data_ptr(), stream=sptr)
            e1.record(stream)
            torch.cuda.synchronize()
            sweep[str(Bs)] = Bs * reps / (e0.elapsed_time(e1) / 1000.0)

    # roofline of the dominant kernel (N4 resident list scan), measured over the timed region
    peaks = measured_peaks()
    peak = peaks["hbm_gbs"] if peaks else 6650.0
    scan_ms = tm["scan_ms"] / max(1, tm["stage_searches"])
    scan_bytes = st["bytes_lists_resident"]
    achieved = scan_bytes / (scan_ms * 1e-3) / 1e9 if scan_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "scan_traffic.json")
    # the captured traffic is of one unsharded launch at the config's default batch: only that
    # workload may quote it
    if os.path.exists(tpath) and shards == 1 and not args.batch:
        traffic = json.load(open(tpath)).get(args.config)
    launches_per_search = st["kernel_launches"]
    h2d_link = None
    if st["h2d_list_bytes"] > 0:  # offloaded lists: the host link is the roofline of that part
        link = measure_h2d_gbs()
        ach = st["h2d_list_bytes"] / (ms_step * 1e-3) / 1e9
        h2d_link = {"achieved": ach, "peak": link, "unit": "GB/s", "frac": ach / link,
                    "bytes_per_step": st["h2d_list_bytes"],
                    "peak_source": "measured in this run: pinned 1 GiB host->device cudaMemcpy, best of 5",
                    "note": "achieved over the whole step: the resident scan and merge overlap or follow the stream"}

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (splitmix64 spec, SURVEY §8d), generated on device",
        "scaling": "strong",
        "config": {"workload": cfg["workload"], "global_batch": B, "nprobe": nprobe, "k": k, "n_per_gpu": info["n"],
                   "n_total": n_total, "nlist": cfg["nlist"], "d": d,
                   "parallelism": f"shard{world}" if shards == world else f"one shard of {shards} on 1 GPU",
                   "l2": "inputs larger than L2 (index %.1f GB)" % (info["n"] * d * 4 / 1e9)},
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "ivf_scan_tc_kernel (N5; FFMA ivf_scan_kernel N4 when d % 64 != 0)", "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
                     "bytes_per_launch": scan_bytes, "avg_launch_ms": scan_ms},
        "step_breakdown_ms": {k2: tm[k2] / max(1, tm["stage_searches"]) for k2 in ("coarse_ms", "scan_ms", "tail_ms", "total_ms")},
        "step_gbps_algorithmic": st["bytes_algorithmic"] / (ms_step * 1e-3) / 1e9,
        "gpu_launches": launches_per_search * args.steps + (args.steps if world > 1 else 0),
        "batch_sweep_qps": sweep,
        "clocks": clk.summary(),
        "certified": {"margin_failures": st["margin_failures"], "probe_failures": st["probe_failures"]},
        "h2d_link": h2d_link,
        "index": {"build_s": build_s, "lists_resident": info["lists_resident"], "hbm_bytes": info["hbm_bytes"],
                  "host_pinned_bytes": info["host_pinned_bytes"], "h2d_list_bytes_per_step": st["h2d_list_bytes"],
                  "llm_reservation_bytes": reservation},
    }
    if world == 1 and not args.no_cpu_baseline:
        idx.close()
        del dq, hold
        torch.cuda.empty_cache()
        cb = cpu_baseline(cfg, dict(n=cfg["n"], d=d, nlist=cfg["nlist"]), args.cpu_sample)
        cb.pop("per_step", None)
        line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
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
