"""Profiling driver: build a synthetic index and run a few searches (for ncu / nsys-less
launch lists). Not a benchmark: numbers printed under a profiler are not bench values."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_15302_b200.retriever import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--nlist", type=int, default=4096)
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--nprobe", type=int, default=64)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--searches", type=int, default=3)
ap.add_argument("--offload", type=float, default=0.0)
ap.add_argument("--stripe-of", type=int, default=1)
ap.add_argument("--no-stages", action="store_true", help="no per-stage events (as the product runs)")
args = ap.parse_args()
torch.cuda.init()
lib = engine()
desc = lib.desc(args.n, 768, args.nlist, num_shards=args.stripe_of)
idx = lib.synthetic_index(desc)
idx.timing_stages(not args.no_stages)
if args.offload:
    idx.place(offload_fraction=args.offload)
for i in range(args.searches):
    q, _ = lib.synth_queries(desc, i * args.batch, args.batch)
    r = idx.search(q, args.nprobe, args.k)
    print(i, {k: r.stats[k] for k in ("scan_ms", "coarse_ms", "total_ms", "tiles", "margin_failures", "bytes_lists_resident") if k in r.stats})
