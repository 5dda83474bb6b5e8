"""Measured retrieval time T_ret(B, resident fraction) of the B200 engine through the public C ABI
(rd_search: host queries in, host ids/distances out — the call ragsim's retrieval worker makes), on
the BASELINE C2 knowledge base (10M x 768, nlist 4096, nprobe 64, k 10), for RAGDoll's retrieval
batch sizes (max_retrieval_batch 64, configs/default_8b.json:33) and partition residencies. The
offloaded lists live in pinned host DRAM and are streamed per search (heat-ordered placement from
a calibration batch). Output: JSON consumed by oracle/ragsim_measured.cpp (the reference simulator
with retrieval_time replaced by these measurements)."""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_15302_b200.retriever import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/tret/measured_tret.json")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--fractions", default="1.0,0.75,0.5,0.25,0.0")
ap.add_argument("--batches", default="1,2,4,8,16,32,64")
args = ap.parse_args()

import torch  # noqa: E402

torch.cuda.init()
lib = engine()
n, d, nlist, nprobe, k = 10_000_000, 768, 4096, 64, 10
desc = lib.desc(n, d, nlist)
idx = lib.synthetic_index(desc)
cal, _ = lib.synth_queries(desc, 50_000_000, 4096)
pr = idx.probe(cal, nprobe)
heat = np.bincount(pr[pr >= 0].ravel(), minlength=nlist).astype(np.uint32)
fractions = [float(x) for x in args.fractions.split(",")]
batches = [int(x) for x in args.batches.split(",")]
rows = []
for f in fractions:
    idx.place(offload_fraction=1.0 - f, list_heat=heat)
    info = idx.info()
    secs = []
    for B in batches:
        hq = torch.from_numpy(lib.synth_queries(desc, 0, B)[0]).pin_memory().numpy()
        hi = torch.empty((B, k), dtype=torch.int64).pin_memory().numpy()
        hd = torch.empty((B, k), dtype=torch.float32).pin_memory().numpy()
        for _ in range(2):
            idx.search_into(hq, nprobe, k, hi, hd)
        ts = []
        for r in range(args.reps):
            q = torch.from_numpy(lib.synth_queries(desc, 1000 + r * B, B)[0]).pin_memory().numpy()
            t0 = time.perf_counter()
            idx.search_into(q, nprobe, k, hi, hd)
            ts.append(time.perf_counter() - t0)
        secs.append(statistics.median(ts))
        print(f"resident {f:.2f} ({info['lists_resident']} lists) B {B}: {secs[-1] * 1e3:.3f} ms", flush=True)
    rows.append({"resident_fraction": f, "lists_resident": info["lists_resident"], "seconds": secs})
out = {"what": "median wall seconds of one rd_search (host buffers) on one B200",
       "knowledge_base": {"n": n, "d": d, "nlist": nlist, "nprobe": nprobe, "k": k, "bytes": n * d * 4},
       "batches": batches, "rows": rows, "gpu": torch.cuda.get_device_name(0)}
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
json.dump(out, open(args.out, "w"), indent=1)
print("wrote", args.out)
