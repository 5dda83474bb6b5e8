/*
 * rd_cpu_batched.c — a batched, list-major CPU IVF-Flat search: the optimised CPU BASELINE that
 * bench.py reports beside the exact oracle (cpu_baseline kind "batched"). TEST / BASELINE
 * INFRASTRUCTURE ONLY, like the rest of oracle/ (see rd_oracle.c): the product library never links,
 * loads or falls back to it.
 *
 * The exact oracle (rd_search in rd_oracle.c) answers each query alone with canonical fp64
 * distances to every probed row: a correctness reference, not a CPU retriever. This file is what a
 * tuned CPU retriever does with the same batch (FAISS-style IVF-Flat): the batch's probes are
 * inverted into per-list query groups, each list is streamed once per batch and its rows are ranked
 * against the whole group with fp32 ||x||^2 - 2 q.x dot products (AVX2/FMA register blocks, 4 rows x
 * 2 queries, rows read from DRAM once per batch), each (query, list) keeps its best m + 1
 * candidates, and per query the best m are re-ranked with the canonical exact distance
 * (rd_exact_l2). The results are certified with the same rule as the GPU engine (the (m+1)-th
 * approximate distance, less a rigorous bound on the fp32 error, must exceed the k-th exact
 * distance; the coarse probe set likewise) and uncertified queries fall back to the exact oracle
 * computation, so the output is the oracle's, bit for bit (tests/test_cpu_batched.py).
 *
 * Build: gcc -O3 -march=x86-64-v3 (AVX2 + FMA; FMA contraction allowed in this unit only — every
 * approximation is covered by its error bound, and the exact distance lives in rd_oracle.c).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../include/rd.h"
#include "rd_oracle_internal.h"

typedef float v8f __attribute__((vector_size(32)));

static inline float hsum8(v8f v) {
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += v[i];
  return s;
}

static inline v8f load8(const float* p) {
  v8f v;
  memcpy(&v, p, 32);
  return v;
}

/* dot product, any d (vectorised body, scalar tail) */
static float dot(const float* a, const float* b, int d) {
  v8f acc = {0, 0, 0, 0, 0, 0, 0, 0};
  int t = 0;
  for (; t + 8 <= d; t += 8) acc += load8(a + t) * load8(b + t);
  float s = hsum8(acc);
  for (; t < d; ++t) s += a[t] * b[t];
  return s;
}

/* |approx - exact| of ||x||^2 + ||q||^2 - 2 q.x for fp32 dots of length d in any order:
 * gamma_d (d u / (1 - d u), doubled for slack) on the dot, 16 u on the norms and the adds */
static inline float err_bound(int d, float qn, float xmax) {
  const float u = 5.9604645e-8f;
  const float gamma = 2.f * (d + 4) * u;
  return 2.f * gamma * sqrtf(qn) * xmax + 16.f * u * (qn + xmax * xmax) + 1e-30f;
}

typedef struct {
  float dist;
  int64_t key; /* row (scan) or list id (coarse) */
} cand_t;

static inline int cless(float da, int64_t ka, float db, int64_t kb) { return da < db || (da == db && ka < kb); }

/* keep the cap smallest (dist, key) ascending in top[0..*cnt) */
static inline void push(cand_t* top, int* cnt, int cap, float dist, int64_t key) {
  int c = *cnt;
  if (c == cap && !cless(dist, key, top[cap - 1].dist, top[cap - 1].key)) return;
  int pos = c < cap ? c : cap - 1;
  while (pos > 0 && cless(dist, key, top[pos - 1].dist, top[pos - 1].key)) {
    top[pos] = top[pos - 1];
    --pos;
  }
  top[pos].dist = dist;
  top[pos].key = key;
  if (c < cap) *cnt = c + 1;
}

/* ---------------------------------------------------------------- prepare: norms */
typedef struct {
  rd_index* h;
} prep_ctx;

static void prep_rows(void* p, int64_t b, int64_t e) {
  rd_index* h = ((prep_ctx*)p)->h;
  for (int64_t r = b; r < e; ++r) {
    const float* x = h->vectors + r * h->d;
    double s = 0.0;
    for (int t = 0; t < h->d; ++t) s += (double)x[t] * (double)x[t];
    h->xnorm[r] = (float)s;
  }
}

int rd_cpu_prepare_batched(rd_index* h) {
  if (!h) return RD_ERR_INVALID;
  free(h->xnorm);
  free(h->cnorm);
  h->xnorm = (float*)malloc(sizeof(float) * (size_t)(h->n > 0 ? h->n : 1));
  h->cnorm = (float*)malloc(sizeof(float) * (size_t)h->nlist);
  if (!h->xnorm || !h->cnorm) return RD_ERR_RUNTIME;
  prep_ctx c = {h};
  rdo_parallel_for(h->n, 8192, prep_rows, &c);
  float cm = 0.f;
  for (int32_t j = 0; j < h->nlist; ++j) {
    const float* x = h->centroids + (int64_t)j * h->d;
    double s = 0.0;
    for (int t = 0; t < h->d; ++t) s += (double)x[t] * (double)x[t];
    h->cnorm[j] = (float)s;
    if (sqrtf((float)s) > cm) cm = sqrtf((float)s);
  }
  h->cmax = cm * (1.f + 1e-6f);
  return RD_OK;
}

/* ---------------------------------------------------------------- the batched search */
typedef struct {
  rd_index* h;
  const float* Q;
  int64_t B;
  int32_t np, k, m;
  float* qnorm;        /* B */
  int32_t* probes;     /* B x np */
  int32_t* lq_off;     /* nlist + 1: per-list query CSR */
  int32_t* lq;         /* B x np: query ids */
  int32_t* lq_slot;    /* B x np: the probe slot of that (query, list) */
  cand_t* part;        /* B x np x (m + 1) candidates per (query, probe slot) */
  int32_t* part_cnt;   /* B x np */
  int64_t* out_ids;
  float* out_dists;
  int64_t fallbacks;   /* queries recomputed exactly */
} bctx;

/* coarse: fp32 distances to every centroid, the np + 32 best refined exactly, certified */
static void coarse_range(void* p, int64_t b0, int64_t b1) {
  bctx* c = (bctx*)p;
  const rd_index* h = c->h;
  const int nl = h->nlist, d = h->d, np = c->np;
  const int C = nl < np + 32 ? nl : np + 32;
  float* approx = (float*)malloc(sizeof(float) * (size_t)nl);
  cand_t* top = (cand_t*)malloc(sizeof(cand_t) * (size_t)(C + 1));
  cand_t* ex = (cand_t*)malloc(sizeof(cand_t) * (size_t)nl);
  for (int64_t b = b0; b < b1; ++b) {
    const float* q = c->Q + b * d;
    double qs = 0.0;
    for (int t = 0; t < d; ++t) qs += (double)q[t] * (double)q[t];
    c->qnorm[b] = (float)qs;
    int cnt = 0;
    for (int j = 0; j < nl; ++j) {
      approx[j] = h->cnorm[j] - 2.f * dot(q, h->centroids + (int64_t)j * d, d);
      push(top, &cnt, C + 1 < nl ? C + 1 : nl, approx[j], j);
    }
    /* the C best exactly, ordered by (exact distance, list id) */
    const int nc = cnt < C ? cnt : C;
    int ne = 0;
    for (int i = 0; i < nc; ++i) {
      const int j = (int)top[i].key;
      push(ex, &ne, nc, rd_exact_l2(q, h->centroids + (int64_t)j * d, d), j);
    }
    int ok = 1;
    if (cnt > C) { /* something was excluded: its approx bounds its exact distance from below */
      const float eps = err_bound(d, c->qnorm[b], h->cmax);
      ok = top[C].dist + c->qnorm[b] - eps > ex[np - 1].dist;
    }
    if (!ok) { /* exact distances to every centroid */
      ne = 0;
      for (int j = 0; j < nl; ++j) push(ex, &ne, np, rd_exact_l2(q, h->centroids + (int64_t)j * d, d), j);
    }
    for (int i = 0; i < np; ++i) c->probes[b * np + i] = (int32_t)ex[i].key;
  }
  free(ex);
  free(top);
  free(approx);
}

/* scan: one list per work item. Row blocks of 4 (12 KiB at d = 768, L1-resident) outer, the list's
 * query pairs inner, so every row is read from DRAM once per batch; each (query, list) keeps its
 * m + 1 best approximate distances (||x||^2 - 2 q.x; ||q||^2 is added in the merge). */
static void scan_range(void* p, int64_t l0, int64_t l1) {
  bctx* c = (bctx*)p;
  const rd_index* h = c->h;
  const int d = h->d, cap = c->m + 1;
  cand_t** tops = (cand_t**)malloc(sizeof(cand_t*) * (size_t)(c->B > 0 ? c->B : 1));
  int** cnts = (int**)malloc(sizeof(int*) * (size_t)(c->B > 0 ? c->B : 1));
  const float** qp = (const float**)malloc(sizeof(float*) * (size_t)(c->B > 0 ? c->B + 1 : 2));
  for (int64_t l = l0; l < l1; ++l) {
    const int q0 = c->lq_off[l], nq = c->lq_off[l + 1] - q0;
    if (nq == 0) continue;
    for (int i = 0; i < nq; ++i) {
      const int b = c->lq[q0 + i];
      const int64_t sl = (int64_t)b * c->np + c->lq_slot[q0 + i];
      tops[i] = c->part + sl * cap;
      cnts[i] = &c->part_cnt[sl];
      qp[i] = c->Q + (int64_t)b * d;
    }
    qp[nq] = qp[nq - 1];  /* odd count: the last pair repeats a query, its second half is dropped */
    const int64_t r0 = h->offsets[l], r1 = h->offsets[l + 1];
    int64_t r = r0;
    for (; r + 4 <= r1; r += 4) {
      const float* x0 = h->vectors + r * d;
      for (int qi = 0; qi < nq; qi += 2) {
        const int two = qi + 1 < nq;
        const float* qa = qp[qi];
        const float* qb = qp[qi + 1];
        v8f a00 = {0}, a01 = {0}, a10 = {0}, a11 = {0}, a20 = {0}, a21 = {0}, a30 = {0}, a31 = {0};
        int t = 0;
        for (; t + 8 <= d; t += 8) {
          const v8f va = load8(qa + t), vb = load8(qb + t);
          const v8f x_0 = load8(x0 + t), x_1 = load8(x0 + d + t), x_2 = load8(x0 + 2 * d + t),
                    x_3 = load8(x0 + 3 * d + t);
          a00 += x_0 * va, a01 += x_0 * vb;
          a10 += x_1 * va, a11 += x_1 * vb;
          a20 += x_2 * va, a21 += x_2 * vb;
          a30 += x_3 * va, a31 += x_3 * vb;
        }
        float dt[4][2] = {{hsum8(a00), hsum8(a01)}, {hsum8(a10), hsum8(a11)},
                          {hsum8(a20), hsum8(a21)}, {hsum8(a30), hsum8(a31)}};
        for (; t < d; ++t)
          for (int i = 0; i < 4; ++i) {
            dt[i][0] += x0[i * d + t] * qa[t];
            dt[i][1] += x0[i * d + t] * qb[t];
          }
        for (int i = 0; i < 4; ++i)
          for (int j = 0; j <= two; ++j)
            push(tops[qi + j], cnts[qi + j], cap, h->xnorm[r + i] - 2.f * dt[i][j], r + i);
      }
    }
    for (; r < r1; ++r) {
      const float* x = h->vectors + r * d;
      for (int qi = 0; qi < nq; ++qi) push(tops[qi], cnts[qi], cap, h->xnorm[r] - 2.f * dot(x, qp[qi], d), r);
    }
  }
  free(qp);
  free(cnts);
  free(tops);
}

/* merge: per query the m + 1 best over its probes, exact rerank of m, certification, fallback */
static void merge_range(void* p, int64_t b0, int64_t b1) {
  bctx* c = (bctx*)p;
  const rd_index* h = c->h;
  const int d = h->d, np = c->np, cap = c->m + 1, k = c->k;
  cand_t* best = (cand_t*)malloc(sizeof(cand_t) * (size_t)cap);
  cand_t* ex = (cand_t*)malloc(sizeof(cand_t) * (size_t)(cap > k ? cap : k));
  for (int64_t b = b0; b < b1; ++b) {
    const float* q = c->Q + b * d;
    int nb = 0;
    for (int s = 0; s < np; ++s) {
      const cand_t* t = c->part + (b * np + s) * cap;
      for (int i = 0; i < c->part_cnt[b * np + s]; ++i) push(best, &nb, cap, t[i].dist, t[i].key);
    }
    const int nr = nb < c->m ? nb : c->m;
    int ne = 0;
    for (int i = 0; i < nr; ++i)
      push(ex, &ne, nr, rd_exact_l2(q, h->vectors + best[i].key * d, d), h->ids[best[i].key]);
    int ok = 1;
    if (nb > c->m) { /* rows not reranked: the (m+1)-th approximation bounds them */
      const float eps = err_bound(d, c->qnorm[b], h->max_norm);
      ok = ne >= k && best[c->m].dist + c->qnorm[b] - eps > ex[k - 1].dist;
    }
    if (!ok) { /* exact: every row of every probed list */
      ne = 0;
      for (int s = 0; s < np; ++s) {
        const int l = c->probes[b * np + s];
        for (int64_t r = h->offsets[l]; r < h->offsets[l + 1]; ++r)
          push(ex, &ne, k, rd_exact_l2(q, h->vectors + r * d, d), h->ids[r]);
      }
      __atomic_fetch_add(&c->fallbacks, 1, __ATOMIC_RELAXED);
    }
    for (int i = 0; i < k; ++i) {
      c->out_ids[b * k + i] = i < ne ? ex[i].key : -1;
      c->out_dists[b * k + i] = i < ne ? ex[i].dist : INFINITY;
    }
  }
  free(ex);
  free(best);
}

/* The batched search (same results as rd_search). fallbacks (optional): queries that took the
 * exact path. Requires rd_cpu_prepare_batched(h) after the index's rows last changed. */
int rd_cpu_search_batched(rd_index* h, const float* Q, int64_t B, int32_t nprobe, int32_t k, int64_t* out_ids,
                          float* out_dists, int64_t* fallbacks) {
  if (!h || B < 0 || nprobe < 1 || k < 1 || (B > 0 && (!Q || !out_ids || !out_dists))) return RD_ERR_INVALID;
  if (!h->xnorm || !h->cnorm) return RD_ERR_INVALID;
  const int np = nprobe < h->nlist ? nprobe : h->nlist;
  bctx c;
  memset(&c, 0, sizeof c);
  c.h = h, c.Q = Q, c.B = B, c.np = np, c.k = k, c.m = k + 8;
  c.out_ids = out_ids, c.out_dists = out_dists;
  const size_t P = (size_t)B * np;
  c.qnorm = (float*)malloc(sizeof(float) * (size_t)(B > 0 ? B : 1));
  c.probes = (int32_t*)malloc(sizeof(int32_t) * (P ? P : 1));
  c.lq_off = (int32_t*)calloc((size_t)h->nlist + 1, sizeof(int32_t));
  c.lq = (int32_t*)malloc(sizeof(int32_t) * (P ? P : 1));
  c.lq_slot = (int32_t*)malloc(sizeof(int32_t) * (P ? P : 1));
  c.part = (cand_t*)malloc(sizeof(cand_t) * (P ? P : 1) * (size_t)(c.m + 1));
  c.part_cnt = (int32_t*)calloc(P ? P : 1, sizeof(int32_t));
  if (!c.qnorm || !c.probes || !c.lq_off || !c.lq || !c.lq_slot || !c.part || !c.part_cnt) {
    free(c.qnorm), free(c.probes), free(c.lq_off), free(c.lq), free(c.lq_slot), free(c.part), free(c.part_cnt);
    return RD_ERR_RUNTIME;
  }
  rdo_parallel_for(B, 4, coarse_range, &c);
  /* invert: per list, its (query, probe slot) pairs in ascending query order */
  for (size_t i = 0; i < P; ++i) c.lq_off[c.probes[i] + 1]++;
  for (int32_t l = 0; l < h->nlist; ++l) c.lq_off[l + 1] += c.lq_off[l];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)h->nlist);
  memcpy(fill, c.lq_off, sizeof(int32_t) * (size_t)h->nlist);
  for (int64_t b = 0; b < B; ++b)
    for (int s = 0; s < np; ++s) {
      const int l = c.probes[b * np + s];
      c.lq[fill[l]] = (int32_t)b;
      c.lq_slot[fill[l]++] = s;
    }
  free(fill);
  rdo_parallel_for(h->nlist, 1, scan_range, &c);
  rdo_parallel_for(B, 4, merge_range, &c);
  if (fallbacks) *fallbacks = c.fallbacks;
  free(c.qnorm), free(c.probes), free(c.lq_off), free(c.lq), free(c.lq_slot), free(c.part), free(c.part_cnt);
  return RD_OK;
}
