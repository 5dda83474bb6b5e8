"""IVF training throughput (rd_index_build) on one GPU: n x d blobs, nlist lists, `iters` Lloyd
rounds. Prints one JSON line; the time includes the host->device copy of the vectors."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_15302_b200.retriever import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--d", type=int, default=768)
ap.add_argument("--nlist", type=int, default=2048)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
rng = np.random.default_rng(0)
centers = rng.standard_normal((a.nlist, a.d)).astype(np.float32)
X = np.empty((a.n, a.d), dtype=np.float32)
for s in range(0, a.n, 1 << 18):
    e = min(a.n, s + (1 << 18))
    X[s:e] = centers[rng.integers(0, a.nlist, e - s)] + 0.25 * rng.standard_normal((e - s, a.d)).astype(np.float32)
lib = engine()
lib.build_index(X[:20000], 64, 1)  # warm-up (module load, kernel attributes)
t0 = time.perf_counter()
idx = lib.build_index(X, a.nlist, a.iters)
t = time.perf_counter() - t0
rounds = a.iters + 1  # assignments
print(json.dumps({"n": a.n, "d": a.d, "nlist": a.nlist, "iters": a.iters, "seconds": t,
                  "assign_vectors_per_s": a.n * rounds / t,
                  "assign_tflops_equiv": 2.0 * a.n * a.nlist * a.d * rounds / t / 1e12,
                  "lists_nonempty": int((np.diff(idx.layout(with_ids=False)[0]) > 0).sum())}))
