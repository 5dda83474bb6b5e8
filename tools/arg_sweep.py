"""Device-timed searches over (batch, nprobe, k) on the C2 knowledge base (10M x 768, nlist 4096):
the fast path (k <= 24, nprobe <= 480), the exact large-k pass and the all-centroid selection
(wide.cu). Queries in HBM, CUDA events on the search stream, median of `reps`. One JSON line each."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_15302_b200.retriever import engine  # noqa: E402

lib = engine()
desc = lib.desc(10_000_000, 768, 4096)
idx = lib.synthetic_index(desc)
stream = torch.cuda.current_stream()
cases = [(B, 64, k) for k in (10, 32, 64, 128) for B in (1, 8, 64, 256)] + \
        [(B, npb, 10) for npb in (128, 480, 481, 1024) for B in (1, 64, 1024)]
for B, nprobe, k in cases:
    q = torch.from_numpy(lib.synth_queries(desc, 123 + B, B)[0]).cuda()
    oi = torch.empty((B, k), dtype=torch.int64, device="cuda")
    od = torch.empty((B, k), dtype=torch.float32, device="cuda")
    run = lambda: idx.search_device(q.data_ptr(), B, nprobe, k, oi.data_ptr(), od.data_ptr(), stream=stream.cuda_stream)
    for _ in range(2):
        run()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    print(json.dumps({"B": B, "nprobe": nprobe, "k": k, "ms": round(ms, 4), "qps": round(B / ms * 1e3, 1),
                      "path": ("wide" if k > 24 else "fast") + ("+select_all" if nprobe > 480 else "")}), flush=True)
