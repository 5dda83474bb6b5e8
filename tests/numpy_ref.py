"""Independent numpy restatement of the synthetic-data spec and exact IVF-Flat
search (TEST INFRASTRUCTURE). It is a second, separately written oracle used to
pin oracle/rd_oracle.c; it shares no code with it.

Spec (seeds via ragsim derive_seed, rng.hpp:52-56):
  u(s, i) = (i+1)-th output of ragsim::Rng(s).next_u64()      (rng.hpp:16-21)
  f(s, i) = (int((u >> 40) & 0xFFFFFF) - 2^23) * 2^-23
  c_j[t] = f(s_c, j*d + t);  a(i) = u(s_a, i) mod nlist
  x_i[t] = c_{a(i)}[t] + sigma * f(s_x, i*d + t)           (f32 arithmetic)
  q_b[t] = x_{r(b)}[t] + qsigma * f(s_qn, b*d + t),  r(b) = u(s_q, b) mod n
Exact distance: eight fp64 residue-class sums (t mod 8), sequential in t, fixed
combination tree, rounded to f32.
"""
import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
DS = np.uint64(0xD1B54A32D192ED03)


def splitmix_at(seed, i):
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.asarray(i, dtype=np.uint64) + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def derive_seed(master, stream):
    with np.errstate(over="ignore"):
        s = np.uint64(master) ^ (np.uint64(stream) * DS)
    return int(splitmix_at(s, 1))


def unif(seed, i):
    u = splitmix_at(seed, i)
    m = ((u >> np.uint64(40)) & np.uint64(0xFFFFFF)).astype(np.int64) - (1 << 23)
    return (m.astype(np.float32) * np.float32(2.0 ** -23)).astype(np.float32)


def seeds(master):
    return {k: derive_seed(master, v) for k, v in
            dict(c=0x1001, a=0x1002, x=0x1003, q=0x1004, qn=0x1005).items()}


def synth_index(n, d, nlist, master=250415302, sigma=0.25, shard=0, num_shards=1):
    s = seeds(master)
    C = unif(s["c"], np.arange(nlist * d, dtype=np.uint64)).reshape(nlist, d)
    a = (splitmix_at(s["a"], np.arange(n, dtype=np.uint64)) % np.uint64(nlist)).astype(np.int64)
    order = np.argsort(a, kind="stable")  # ascending id within each list
    full_len = np.bincount(a, minlength=nlist)
    starts = np.concatenate([[0], np.cumsum(full_len)])
    ids, offs = [], [0]
    for l in range(nlist):
        lo, hi = shard * full_len[l] // num_shards, (shard + 1) * full_len[l] // num_shards
        ids.append(order[starts[l] + lo: starts[l] + hi])
        offs.append(offs[-1] + (hi - lo))
    ids = np.concatenate(ids).astype(np.int64) if ids else np.zeros(0, np.int64)
    X = vectors_of(ids, d, nlist, master, sigma, C)
    return X, np.asarray(offs, dtype=np.int64), C, ids


def vectors_of(ids, d, nlist, master=250415302, sigma=0.25, C=None):
    s = seeds(master)
    if C is None:
        C = unif(s["c"], np.arange(nlist * d, dtype=np.uint64)).reshape(nlist, d)
    ids = np.asarray(ids, dtype=np.uint64)
    a = (splitmix_at(s["a"], ids) % np.uint64(nlist)).astype(np.int64)
    t = np.arange(d, dtype=np.uint64)
    noise = np.float32(sigma) * unif(s["x"], ids[:, None] * np.uint64(d) + t[None, :])
    return (C[a] + noise).astype(np.float32)


def synth_queries(n, d, nlist, b0, B, master=250415302, sigma=0.25, qsigma=0.0625):
    s = seeds(master)
    b = np.arange(b0, b0 + B, dtype=np.uint64)
    r = (splitmix_at(s["q"], b) % np.uint64(n)).astype(np.int64)
    X = vectors_of(r, d, nlist, master, sigma)
    t = np.arange(d, dtype=np.uint64)
    noise = np.float32(qsigma) * unif(s["qn"], b[:, None] * np.uint64(d) + t[None, :])
    return (X + noise).astype(np.float32), r


def exact_l2(q, X):
    """canonical distances from one query q (d,) to rows X (m, d); d % 8 == 0."""
    m, d = X.shape
    df = q.astype(np.float64)[None, :] - X.astype(np.float64)
    sq = (df * df).reshape(m, d // 8, 8)
    s = np.cumsum(sq, axis=1)[:, -1, :]  # sequential per residue class
    tot = ((s[:, 0] + s[:, 1]) + (s[:, 2] + s[:, 3])) + ((s[:, 4] + s[:, 5]) + (s[:, 6] + s[:, 7]))
    return tot.astype(np.float32)


def topk(dist, keys, k):
    order = np.lexsort((keys, dist))[:k]
    ids = np.full(k, -1, np.int64)
    ds = np.full(k, np.inf, np.float32)
    ids[: len(order)] = keys[order]
    ds[: len(order)] = dist[order]
    return ids, ds


def ivf_search(X, offs, C, ids, Q, nprobe, k):
    nlist = C.shape[0]
    out_i = np.empty((len(Q), k), np.int64)
    out_d = np.empty((len(Q), k), np.float32)
    probes = np.empty((len(Q), min(nprobe, nlist)), np.int64)
    for b, q in enumerate(Q):
        dc = exact_l2(q, C)
        pr = np.lexsort((np.arange(nlist), dc))[: min(nprobe, nlist)]
        probes[b] = pr
        rows = np.concatenate([np.arange(offs[l], offs[l + 1]) for l in pr]) if len(pr) else np.zeros(0, np.int64)
        out_i[b], out_d[b] = topk(exact_l2(q, X[rows]) if len(rows) else np.zeros(0, np.float32), ids[rows], k)
    return out_i, out_d, probes
