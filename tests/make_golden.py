"""Regenerates tests/golden/ivf_small.npz with the independent numpy
restatement (tests/numpy_ref.py). Run: python tests/make_golden.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy_ref as R  # noqa: E402

CASES = {
    "c1s": dict(n=6000, d=768, nlist=64, nprobe=8, k=10, B=12),
    "d128": dict(n=4000, d=128, nlist=50, nprobe=5, k=20, B=9),
    "shard1of3": dict(n=5000, d=64, nlist=40, nprobe=6, k=10, B=7, shard=1, num_shards=3),
}

if __name__ == "__main__":
    out = {}
    for name, c in CASES.items():
        X, offs, C, ids = R.synth_index(c["n"], c["d"], c["nlist"], shard=c.get("shard", 0),
                                        num_shards=c.get("num_shards", 1))
        Q, src = R.synth_queries(c["n"], c["d"], c["nlist"], 0, c["B"])
        oi, od, pr = R.ivf_search(X, offs, C, ids, Q, c["nprobe"], c["k"])
        out[f"{name}/offs"] = offs
        out[f"{name}/ids_head"] = ids[:64]
        out[f"{name}/x_row0"] = X[0]
        out[f"{name}/queries"] = Q
        out[f"{name}/src"] = src
        out[f"{name}/out_ids"] = oi
        out[f"{name}/out_dists"] = od
        out[f"{name}/probes"] = pr
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ivf_small.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, sum(v.nbytes for v in out.values()), "bytes")
