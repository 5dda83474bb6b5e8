/*
 * rd_oracle.c — CPU ORACLE for the RAGDoll retrieval stage. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or the timed
 * CPU baseline. The product path (paper_2504_15302_b200/lib/librd_b200.so)
 * never links, loads or falls back to it.
 *
 * It implements include/rd.h with plain, exact IVF-Flat semantics restated
 * from first principles, because the reference has no search implementation
 * (its retrieval stage is retrieval_time(), /root/reference/proj/core/src/cost_model.cpp:15-21;
 * real vector search is out of the reference's scope).
 * IVF result parity is therefore UNPINNED by the reference itself; what IS
 * pinned against the compiled reference (oracle/_ref, tests/golden/) is:
 *   - the splitmix64 Rng / derive_seed streams every synthetic input derives
 *     from (/root/reference/proj/core/include/ragsim/rng.hpp:12-56), and
 *   - the placement arithmetic (memory_planner.cpp:12-35, prefetch_timeline.cpp:79-90).
 *
 * Algorithm (exact IVF-Flat, squared L2):
 *   1. coarse: exact distance from the query to every centroid;
 *   2. probes: the nprobe smallest by (distance, list id);
 *   3. scan: exact distance to every vector of the probed lists;
 *   4. top-k: the k smallest by (distance, id), ascending; pad (-1, +inf).
 * "Exact distance" is the canonical rd_exact_l2 (see below), identical
 * bit-for-bit between this file and the CUDA engine's rerank.
 *
 * Build: gcc -O3 -march=x86-64-v3 -ffp-contract=off (see oracle/Makefile).
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include "../include/rd.h"
#include "../include/rd_format.h"
#include "rd_oracle_internal.h"

/* ------------------------------------------------------------------ errors */
static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* rd_last_error(void) { return g_err; }
int rd_abi_version(void) { return RD_ABI_VERSION; }
const char* rd_backend(void) { return "cpu-oracle"; }

/* ------------------------------------------------------------------ rng
 * ragsim::Rng::next_u64 (rng.hpp:16-21): state += golden gamma, two
 * xorshift-multiply rounds. Counter form: the (i+1)-th output of Rng(seed). */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t rd_splitmix_at(uint64_t seed, uint64_t i) {
  return mix64(seed + (i + 1) * 0x9e3779b97f4a7c15ull);
}

/* ragsim::derive_seed (rng.hpp:52-56): Rng(master ^ stream*C), discard one, take one. */
uint64_t rd_derive_seed(uint64_t master, uint64_t stream) {
  uint64_t s = master ^ (stream * 0xd1b54a32d192ed03ull);
  return rd_splitmix_at(s, 1);
}

/* uniform on [-1, 1), 24-bit, exact in fp32. */
static inline float unif(uint64_t seed, uint64_t i) {
  uint64_t u = rd_splitmix_at(seed, i);
  int32_t m = (int32_t)((u >> 40) & 0xFFFFFFu) - (1 << 23);
  return (float)m * 0x1p-23f;
}

/* ------------------------------------------------------------------ canonical exact L2 */
typedef double v4d __attribute__((vector_size(32)));
typedef float v4f __attribute__((vector_size(16)));

float rd_exact_l2(const float* a, const float* b, int32_t d) {
  v4d s0 = {0, 0, 0, 0}, s1 = {0, 0, 0, 0};
  int32_t t = 0;
  for (; t + 8 <= d; t += 8) {
    v4f a0, a1, b0, b1;
    memcpy(&a0, a + t, 16);
    memcpy(&a1, a + t + 4, 16);
    memcpy(&b0, b + t, 16);
    memcpy(&b1, b + t + 4, 16);
    v4d d0 = __builtin_convertvector(a0, v4d) - __builtin_convertvector(b0, v4d);
    v4d d1 = __builtin_convertvector(a1, v4d) - __builtin_convertvector(b1, v4d);
    s0 = s0 + d0 * d0;
    s1 = s1 + d1 * d1;
  }
  double s[8] = {s0[0], s0[1], s0[2], s0[3], s1[0], s1[1], s1[2], s1[3]};
  for (; t < d; ++t) {
    double df = (double)a[t] - (double)b[t];
    s[t & 7] = s[t & 7] + df * df;
  }
  double tot = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  return (float)tot;
}

/* ------------------------------------------------------------------ threads */
int rdo_threads(void) {
  const char* e = getenv("RD_CPU_THREADS");
  if (e && atoi(e) > 0) return atoi(e);
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

typedef struct {
  work_fn fn;
  void* ctx;
  int64_t n, chunk;
  int64_t next;
  pthread_mutex_t mu;
} pool_job;

static void* pool_worker(void* p) {
  pool_job* j = (pool_job*)p;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int64_t b = j->next;
    j->next += j->chunk;
    pthread_mutex_unlock(&j->mu);
    if (b >= j->n) break;
    int64_t e = b + j->chunk < j->n ? b + j->chunk : j->n;
    j->fn(j->ctx, b, e);
  }
  return NULL;
}

void rdo_parallel_for(int64_t n, int64_t chunk, work_fn fn, void* ctx) {
  if (n <= 0) return;
  int T = rdo_threads();
  if (chunk < 1) chunk = 1;
  pool_job job = {fn, ctx, n, chunk, 0, PTHREAD_MUTEX_INITIALIZER};
  if (T == 1 || n <= chunk) {
    fn(ctx, 0, n);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)T);
  for (int i = 0; i < T; ++i) pthread_create(&th[i], NULL, pool_worker, &job);
  for (int i = 0; i < T; ++i) pthread_join(th[i], NULL);
  free(th);
}

/* ------------------------------------------------------------------ index (struct: rd_oracle_internal.h) */

static int check_desc(const rd_synth_desc* s) {
  if (!s) return fail(RD_ERR_INVALID, "null synth descriptor");
  if (s->n < 1 || s->d < 1 || s->nlist < 1)
    return fail(RD_ERR_INVALID, "synth: n, d, nlist must be >= 1");
  if (s->num_shards < 1 || s->shard < 0 || s->shard >= s->num_shards)
    return fail(RD_ERR_INVALID, "synth: shard %d of %d out of range", s->shard, s->num_shards);
  return RD_OK;
}

typedef struct {
  const rd_synth_desc* s;
  uint64_t sc, sx;
  const int64_t* ids;
  const int32_t* lists_of_rows;
  float* out;
  const float* centroids;
} gen_ctx;

static void gen_centroids(void* p, int64_t b, int64_t e) {
  gen_ctx* g = (gen_ctx*)p;
  int32_t d = g->s->d;
  for (int64_t j = b; j < e; ++j)
    for (int32_t t = 0; t < d; ++t) g->out[j * d + t] = unif(g->sc, (uint64_t)(j * d + t));
}

static void gen_rows(void* p, int64_t b, int64_t e) {
  gen_ctx* g = (gen_ctx*)p;
  int32_t d = g->s->d;
  float sigma = g->s->sigma;
  for (int64_t r = b; r < e; ++r) {
    int64_t id = g->ids[r];
    const float* c = g->centroids + (int64_t)g->lists_of_rows[r] * d;
    float* x = g->out + r * d;
    for (int32_t t = 0; t < d; ++t) {
      float noise = sigma * unif(g->sx, (uint64_t)(id * d + t));
      x[t] = c[t] + noise;
    }
  }
}

static void compute_norm_max(rd_index* h) {
  double mx = 0;
  for (int64_t r = 0; r < h->n; ++r) {
    double s = 0;
    const float* x = h->vectors + r * h->d;
    for (int32_t t = 0; t < h->d; ++t) s += (double)x[t] * x[t];
    if (s > mx) mx = s;
  }
  h->max_norm = (float)sqrt(mx);
}

int rd_index_create_synthetic(const rd_synth_desc* s, int32_t device, rd_index** out) {
  (void)device;
  int rc = check_desc(s);
  if (rc) return rc;
  if (!out) return fail(RD_ERR_INVALID, "null out");
  const int64_t n = s->n;
  const int32_t d = s->d, nl = s->nlist, G = s->num_shards, g = s->shard;
  const uint64_t sa = rd_derive_seed(s->seed, RD_STREAM_ASSIGN);
  rd_index* h = (rd_index*)calloc(1, sizeof *h);
  h->d = d;
  h->nlist = nl;
  h->centroids = (float*)malloc(sizeof(float) * (size_t)nl * d);
  gen_ctx gc = {s, rd_derive_seed(s->seed, RD_STREAM_CENTROIDS),
                rd_derive_seed(s->seed, RD_STREAM_VECTOR_NOISE), NULL, NULL, h->centroids, NULL};
  rdo_parallel_for(nl, 16, gen_centroids, &gc);

  /* list membership: a(i) = u(s_a, i) mod nlist, members ascending by id */
  int32_t* assign = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t* full_len = (int64_t*)calloc((size_t)nl, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    assign[i] = (int32_t)(rd_splitmix_at(sa, (uint64_t)i) % (uint64_t)nl);
    full_len[assign[i]]++;
  }
  /* row stripe of this shard: [g*len/G, (g+1)*len/G) */
  h->offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nl + 1));
  h->offsets[0] = 0;
  for (int32_t l = 0; l < nl; ++l) {
    int64_t lo = g * full_len[l] / G, hi = (int64_t)(g + 1) * full_len[l] / G;
    h->offsets[l + 1] = h->offsets[l] + (hi - lo);
  }
  h->n = h->offsets[nl];
  h->ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(h->n > 0 ? h->n : 1));
  int32_t* row_list = (int32_t*)malloc(sizeof(int32_t) * (size_t)(h->n > 0 ? h->n : 1));
  int64_t* cursor = (int64_t*)calloc((size_t)nl, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    int32_t l = assign[i];
    int64_t pos = cursor[l]++;
    int64_t lo = g * full_len[l] / G, hi = (int64_t)(g + 1) * full_len[l] / G;
    if (pos >= lo && pos < hi) {
      int64_t r = h->offsets[l] + (pos - lo);
      h->ids[r] = i;
      row_list[r] = l;
    }
  }
  free(cursor);
  free(full_len);
  free(assign);
  h->vectors = (float*)malloc(sizeof(float) * (size_t)(h->n > 0 ? h->n : 1) * d);
  if (!h->vectors) {
    free(row_list);
    rd_index_destroy(h);
    return fail(RD_ERR_RUNTIME, "oracle: out of host memory for %lld vectors", (long long)h->n);
  }
  gc.ids = h->ids;
  gc.lists_of_rows = row_list;
  gc.out = h->vectors;
  gc.centroids = h->centroids;
  rdo_parallel_for(h->n, 4096, gen_rows, &gc);
  free(row_list);
  h->resident = (uint8_t*)malloc((size_t)nl);
  h->hostcopy = (uint8_t*)calloc((size_t)nl, 1);
  memset(h->resident, 1, (size_t)nl);
  compute_norm_max(h);
  *out = h;
  return RD_OK;
}

/* ------------------------------------------------------------------ IVF training (rd_index_build) */
typedef struct {
  const float* X;
  const float* C;
  int32_t d, nlist;
  int32_t* assign;
} assign_ctx;

static void assign_rows(void* p, int64_t b, int64_t e) {
  const assign_ctx* a = (const assign_ctx*)p;
  for (int64_t r = b; r < e; ++r) {
    const float* x = a->X + (size_t)r * a->d;
    float best = INFINITY;
    int32_t bj = 0;
    for (int32_t j = 0; j < a->nlist; ++j) {
      const float dj = rd_exact_l2(x, a->C + (size_t)j * a->d, a->d);
      if (dj < best) { /* ties keep the lower id */
        best = dj;
        bj = j;
      }
    }
    a->assign[r] = bj;
  }
}

int rd_index_build(int64_t n, int32_t d, int32_t nlist, const float* vectors, const int64_t* ids, int32_t iters,
                   uint64_t seed, int32_t device, rd_index** out) {
  if (n < 1 || d < 1 || nlist < 1 || n < nlist || iters < 0 || !vectors || !out)
    return fail(RD_ERR_INVALID, "build: need n >= nlist >= 1, d >= 1, iters >= 0 and vectors");
  float* C = (float*)malloc(sizeof(float) * (size_t)nlist * d);
  int32_t* assign = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  uint8_t* taken = (uint8_t*)calloc((size_t)n, 1);
  const uint64_t s = rd_derive_seed(seed, RD_STREAM_TRAIN_INIT);
  uint64_t i = 0;
  for (int32_t j = 0; j < nlist;) { /* the first nlist distinct rows of u(s, i) mod n */
    const int64_t r = (int64_t)(rd_splitmix_at(s, i++) % (uint64_t)n);
    if (taken[r]) continue;
    taken[r] = 1;
    memcpy(C + (size_t)j * d, vectors + (size_t)r * d, sizeof(float) * (size_t)d);
    ++j;
  }
  free(taken);
  assign_ctx ac = {vectors, C, d, nlist, assign};
  double* sum = (double*)malloc(sizeof(double) * (size_t)nlist * d);
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)nlist);
  for (int32_t it = 0; it <= iters; ++it) {
    rdo_parallel_for(n, 256, assign_rows, &ac);
    if (it == iters) break;
    memset(sum, 0, sizeof(double) * (size_t)nlist * d);
    memset(cnt, 0, sizeof(int64_t) * (size_t)nlist);
    for (int64_t r = 0; r < n; ++r) { /* ascending rows: the canonical summation order */
      double* sl = sum + (size_t)assign[r] * d;
      const float* x = vectors + (size_t)r * d;
      for (int32_t t = 0; t < d; ++t) sl[t] = sl[t] + (double)x[t];
      cnt[assign[r]]++;
    }
    for (int32_t j = 0; j < nlist; ++j)
      if (cnt[j])
        for (int32_t t = 0; t < d; ++t) C[(size_t)j * d + t] = (float)(sum[(size_t)j * d + t] / (double)cnt[j]);
  }
  free(sum);
  /* list order, ascending row within a list (counting sort) */
  int64_t* offs = (int64_t*)calloc((size_t)nlist + 1, sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r) offs[assign[r] + 1]++;
  for (int32_t j = 0; j < nlist; ++j) offs[j + 1] += offs[j];
  memcpy(cnt, offs, sizeof(int64_t) * (size_t)nlist);
  float* Xl = (float*)malloc(sizeof(float) * (size_t)n * d);
  int64_t* idl = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t r = 0; r < n; ++r) {
    const int64_t pos = cnt[assign[r]]++;
    memcpy(Xl + (size_t)pos * d, vectors + (size_t)r * d, sizeof(float) * (size_t)d);
    idl[pos] = ids ? ids[r] : r;
  }
  const int rc = rd_index_create_from_host(n, d, nlist, Xl, offs, C, idl, device, out);
  free(Xl);
  free(idl);
  free(offs);
  free(cnt);
  free(assign);
  free(C);
  return rc;
}

int rd_index_centroids(const rd_index* h, float* out) {
  if (!h || !out) return fail(RD_ERR_INVALID, "centroids: null argument");
  memcpy(out, h->centroids, sizeof(float) * (size_t)h->nlist * h->d);
  return RD_OK;
}

int rd_index_create_from_host(int64_t n, int32_t d, int32_t nlist, const float* vectors,
                              const int64_t* list_offsets, const float* centroids,
                              const int64_t* ids, int32_t device, rd_index** out) {
  (void)device;
  if (n < 0 || d < 1 || nlist < 1 || !list_offsets || !centroids || !out || (n > 0 && !vectors))
    return fail(RD_ERR_INVALID, "create_from_host: invalid arguments");
  if (list_offsets[0] != 0 || list_offsets[nlist] != n)
    return fail(RD_ERR_INVALID, "create_from_host: list_offsets must run 0..n");
  for (int32_t l = 0; l < nlist; ++l)
    if (list_offsets[l + 1] < list_offsets[l])
      return fail(RD_ERR_INVALID, "create_from_host: list_offsets not monotone at %d", l);
  rd_index* h = (rd_index*)calloc(1, sizeof *h);
  h->n = n;
  h->d = d;
  h->nlist = nlist;
  h->vectors = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1) * d);
  if (n) memcpy(h->vectors, vectors, sizeof(float) * (size_t)n * d);
  h->offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nlist + 1));
  memcpy(h->offsets, list_offsets, sizeof(int64_t) * (size_t)(nlist + 1));
  h->centroids = (float*)malloc(sizeof(float) * (size_t)nlist * d);
  memcpy(h->centroids, centroids, sizeof(float) * (size_t)nlist * d);
  h->ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) h->ids[i] = ids ? ids[i] : i;
  h->resident = (uint8_t*)malloc((size_t)nlist);
  memset(h->resident, 1, (size_t)nlist);
  h->hostcopy = (uint8_t*)calloc((size_t)nlist, 1);
  compute_norm_max(h);
  *out = h;
  return RD_OK;
}

/* ------------------------------------------------------------------ on-disk index (rd_format.h) */
static int write_at(FILE* f, uint64_t off, const void* p, uint64_t bytes) {
  if (fseeko(f, (off_t)off, SEEK_SET) != 0) return -1;
  return bytes == 0 || fwrite(p, 1, bytes, f) == bytes ? 0 : -1;
}
static int read_at(FILE* f, uint64_t off, void* p, uint64_t bytes) {
  if (fseeko(f, (off_t)off, SEEK_SET) != 0) return -1;
  return bytes == 0 || fread(p, 1, bytes, f) == bytes ? 0 : -1;
}

int rd_index_save(const rd_index* h, const char* path) {
  if (!h || !path) return fail(RD_ERR_INVALID, "save: null argument");
  rd_file_header hd;
  rd_fmt_layout(&hd, h->n, h->d, h->nlist);
  hd.check = rd_fmt_check(&hd, h->offsets);
  FILE* f = fopen(path, "wb");
  if (!f) return fail(RD_ERR_RUNTIME, "save: cannot open %s for writing", path);
  char pad[RD_FILE_ALIGN];
  memset(pad, 0, sizeof pad);
  memcpy(pad, &hd, sizeof hd);
  int bad = write_at(f, 0, pad, sizeof pad) ||
            write_at(f, hd.off_list_offsets, h->offsets, 8ull * (uint64_t)(h->nlist + 1)) ||
            write_at(f, hd.off_ids, h->ids, 8ull * (uint64_t)h->n) ||
            write_at(f, hd.off_centroids, h->centroids, 4ull * (uint64_t)h->nlist * h->d) ||
            write_at(f, hd.off_vectors, h->vectors, 4ull * (uint64_t)h->n * h->d);
  if (fclose(f) != 0) bad = 1;
  return bad ? fail(RD_ERR_RUNTIME, "save: write to %s failed", path) : RD_OK;
}

int rd_index_load(const char* path, int32_t device, rd_index** out) {
  (void)device;
  if (!path || !out) return fail(RD_ERR_INVALID, "load: null argument");
  FILE* f = fopen(path, "rb");
  if (!f) return fail(RD_ERR_INVALID, "load: cannot open %s", path);
  rd_file_header hd;
  const char* why = NULL;
  int64_t* offs = NULL;
  if (fseeko(f, 0, SEEK_END) != 0) why = "load: cannot size file";
  const uint64_t size = why ? 0 : (uint64_t)ftello(f);
  if (!why && read_at(f, 0, &hd, sizeof hd)) why = "truncated rd index file";
  if (!why) why = rd_fmt_validate(&hd, size, NULL);
  if (!why) {
    offs = (int64_t*)malloc(8ull * (uint64_t)(hd.nlist + 1));
    if (read_at(f, hd.off_list_offsets, offs, 8ull * (uint64_t)(hd.nlist + 1))) why = "truncated rd index file";
  }
  if (!why) why = rd_fmt_validate(&hd, size, offs);
  if (why) {
    free(offs);
    fclose(f);
    return fail(RD_ERR_INVALID, "load %s: %s", path, why);
  }
  rd_index* h = (rd_index*)calloc(1, sizeof *h);
  h->n = hd.n;
  h->d = hd.d;
  h->nlist = hd.nlist;
  h->offsets = offs;
  h->ids = (int64_t*)malloc(8ull * (uint64_t)(hd.n > 0 ? hd.n : 1));
  h->centroids = (float*)malloc(4ull * (uint64_t)hd.nlist * hd.d);
  h->vectors = (float*)malloc(4ull * (uint64_t)(hd.n > 0 ? hd.n : 1) * hd.d);
  h->resident = (uint8_t*)malloc((size_t)hd.nlist);
  memset(h->resident, 1, (size_t)hd.nlist);
  h->hostcopy = (uint8_t*)calloc((size_t)hd.nlist, 1);
  const int bad = read_at(f, hd.off_ids, h->ids, 8ull * (uint64_t)hd.n) ||
                  read_at(f, hd.off_centroids, h->centroids, 4ull * (uint64_t)hd.nlist * hd.d) ||
                  read_at(f, hd.off_vectors, h->vectors, 4ull * (uint64_t)hd.n * hd.d);
  fclose(f);
  if (bad) {
    rd_index_destroy(h);
    return fail(RD_ERR_RUNTIME, "load %s: read failed", path);
  }
  compute_norm_max(h);
  *out = h;
  return RD_OK;
}

void rd_index_destroy(rd_index* h) {
  if (!h) return;
  free(h->vectors);
  free(h->offsets);
  free(h->ids);
  free(h->centroids);
  free(h->resident);
  free(h->hostcopy);
  free(h->xnorm);
  free(h->cnorm);
  free(h);
}

/* Residency does not change results; the oracle records it so the placement
 * rule (shared with the engine) can be tested on CPU. */
static int choose_resident(const rd_index* h, const rd_placement* p, uint8_t* mask) {
  const int32_t nl = h->nlist;
  const uint64_t row_bytes = (uint64_t)h->d * sizeof(float);
  if (p->resident_mask) {
    uint64_t bytes = 0;
    for (int32_t l = 0; l < nl; ++l) {
      mask[l] = p->resident_mask[l] ? 1 : 0;
      if (mask[l]) bytes += (uint64_t)(h->offsets[l + 1] - h->offsets[l]) * row_bytes;
    }
    if (p->hbm_budget_bytes && bytes > p->hbm_budget_bytes)
      return fail(RD_ERR_INFEASIBLE, "placement infeasible: resident lists need %llu bytes > budget %llu",
                  (unsigned long long)bytes, (unsigned long long)p->hbm_budget_bytes);
    return RD_OK;
  }
  if (p->offload_fraction < 0 || p->offload_fraction > 1)
    return fail(RD_ERR_INVALID, "offload_fraction must be in [0, 1]");
  /* order: heat descending, then list id ascending */
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)nl);
  for (int32_t l = 0; l < nl; ++l) order[l] = l;
  if (p->list_heat) {
    for (int32_t i = 1; i < nl; ++i) { /* stable insertion sort by heat desc */
      int32_t v = order[i], j = i - 1;
      while (j >= 0 && p->list_heat[order[j]] < p->list_heat[v]) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = v;
    }
  }
  int64_t target = nl - (int64_t)floor(p->offload_fraction * nl + 0.5);
  uint64_t bytes = 0;
  memset(mask, 0, (size_t)nl);
  /* the budget covers resident lists plus, once anything is offloaded, a staging ring of at
   * least two slots of max(largest list, 16384 rows) rounded up to 256 rows (include/rd.h) */
  uint64_t budget = p->hbm_budget_bytes;
  if (budget) {
    uint64_t all = 0;
    int64_t maxlen = 0;
    for (int32_t l = 0; l < nl; ++l)
      if (h->offsets[l + 1] - h->offsets[l] > maxlen) maxlen = h->offsets[l + 1] - h->offsets[l];
    for (int64_t i = 0; i < target; ++i) all += (uint64_t)(h->offsets[order[i] + 1] - h->offsets[order[i]]) * row_bytes;
    if (target < nl || all > budget) {
      int64_t rows = maxlen > 16384 ? maxlen : 16384;
      uint64_t slot = (uint64_t)((rows + 255) / 256 * 256) * row_bytes;
      uint64_t reserve = (uint64_t)(p->staging_slots > 2 ? p->staging_slots : 2) * slot;
      if (reserve > budget) {
        free(order);
        return fail(RD_ERR_INFEASIBLE, "placement infeasible: budget %llu below the %llu-byte staging ring",
                    (unsigned long long)budget, (unsigned long long)reserve);
      }
      budget -= reserve;
    }
  }
  for (int64_t i = 0; i < target; ++i) {
    int32_t l = order[i];
    uint64_t lb = (uint64_t)(h->offsets[l + 1] - h->offsets[l]) * row_bytes;
    if (budget && bytes + lb > budget) break;
    bytes += lb;
    mask[l] = 1;
  }
  free(order);
  return RD_OK;
}

int rd_index_place(rd_index* h, const rd_placement* p) {
  if (!h || !p) return fail(RD_ERR_INVALID, "null argument");
  uint8_t* mask = (uint8_t*)malloc((size_t)h->nlist);
  int rc = choose_resident(h, p, mask);
  if (rc == RD_OK) {
    memcpy(h->resident, mask, (size_t)h->nlist);
    for (int32_t l = 0; l < h->nlist; ++l) h->hostcopy[l] = !mask[l]; /* the relayout keeps offloaded lists only */
  }
  free(mask);
  return rc;
}

int rd_index_migrate(rd_index* h, const int32_t* promote, int32_t n_promote, const int32_t* demote,
                     int32_t n_demote, uint64_t hbm_budget_bytes, rd_migration_stats* st) {
  if (!h || n_promote < 0 || n_demote < 0 || (n_promote && !promote) || (n_demote && !demote))
    return fail(RD_ERR_INVALID, "migrate: invalid arguments");
  const int32_t nl = h->nlist;
  const uint64_t row_bytes = (uint64_t)h->d * sizeof(float);
  uint8_t* seen = (uint8_t*)calloc((size_t)nl, 1);
  for (int32_t i = 0; i < n_promote + n_demote; ++i) {
    const int is_p = i < n_promote;
    const int32_t l = is_p ? promote[i] : demote[i - n_promote];
    const char* why = NULL;
    if (l < 0 || l >= nl) why = "list id out of range";
    else if (seen[l]) why = "list named twice";
    else if (is_p && h->resident[l]) why = "promoted list is already resident";
    else if (!is_p && !h->resident[l]) why = "demoted list is not resident";
    if (why) {
      free(seen);
      return fail(RD_ERR_INVALID, "migrate: %s (%d)", why, l);
    }
    seen[l] = 1;
  }
  uint64_t res_bytes = 0;
  int64_t max_off = -1;
  for (int32_t l = 0; l < nl; ++l) {
    const int after = seen[l] ? !h->resident[l] : h->resident[l];
    const int64_t len = h->offsets[l + 1] - h->offsets[l];
    if (after) res_bytes += (uint64_t)len * row_bytes;
    else if (len > max_off) max_off = len;
  }
  free(seen);
  if (hbm_budget_bytes) {
    uint64_t need = res_bytes;
    if (max_off >= 0) {
      const int64_t rows = max_off > 16384 ? max_off : 16384;
      need += 2ull * (uint64_t)((rows + 255) / 256 * 256) * row_bytes;
    }
    if (need > hbm_budget_bytes)
      return fail(RD_ERR_INFEASIBLE, "migration infeasible: %llu bytes needed > budget %llu",
                  (unsigned long long)need, (unsigned long long)hbm_budget_bytes);
  }
  rd_migration_stats s;
  memset(&s, 0, sizeof s);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (int32_t i = 0; i < n_demote; ++i) {
    const int32_t l = demote[i];
    if (!h->hostcopy[l]) s.d2h_bytes += (uint64_t)(h->offsets[l + 1] - h->offsets[l]) * row_bytes;
    h->hostcopy[l] = 1;
    h->resident[l] = 0;
  }
  for (int32_t i = 0; i < n_promote; ++i) {
    const int32_t l = promote[i];
    s.h2d_bytes += (uint64_t)(h->offsets[l + 1] - h->offsets[l]) * row_bytes;
    h->resident[l] = 1;
  }
  s.lists_promoted = n_promote;
  s.lists_demoted = n_demote;
  s.resident_bytes = res_bytes;
  clock_gettime(CLOCK_MONOTONIC, &t1);
  s.seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec) + 1e-9;
  if (st) *st = s;
  return RD_OK;
}

int rd_index_info_get(const rd_index* h, rd_index_info* o) {
  if (!h || !o) return fail(RD_ERR_INVALID, "null argument");
  memset(o, 0, sizeof *o);
  o->n = h->n;
  o->d = h->d;
  o->nlist = h->nlist;
  for (int32_t l = 0; l < h->nlist; ++l)
    if (h->resident[l]) {
      o->lists_resident++;
      o->n_resident += h->offsets[l + 1] - h->offsets[l];
    }
  o->max_norm = h->max_norm;
  o->device = -1;
  return RD_OK;
}

int rd_index_layout(const rd_index* h, int64_t* offs, int64_t* ids, uint8_t* mask) {
  if (!h) return fail(RD_ERR_INVALID, "null index");
  if (offs) memcpy(offs, h->offsets, sizeof(int64_t) * (size_t)(h->nlist + 1));
  if (ids) memcpy(ids, h->ids, sizeof(int64_t) * (size_t)h->n);
  if (mask) memcpy(mask, h->resident, (size_t)h->nlist);
  return RD_OK;
}

/* ------------------------------------------------------------------ search */
typedef struct {
  float dist;
  int64_t id;
} cand;

static inline int cand_less(float da, int64_t ia, float db, int64_t ib) {
  return da < db || (da == db && ia < ib);
}

/* keep the k smallest (dist, id) ascending in top[0..*cnt) */
static inline void topk_push(cand* top, int32_t* cnt, int32_t k, float dist, int64_t id) {
  int32_t c = *cnt;
  if (c == k && !cand_less(dist, id, top[k - 1].dist, top[k - 1].id)) return;
  int32_t pos = c < k ? c : k - 1;
  while (pos > 0 && cand_less(dist, id, top[pos - 1].dist, top[pos - 1].id)) {
    top[pos] = top[pos - 1];
    --pos;
  }
  top[pos].dist = dist;
  top[pos].id = id;
  if (c < k) *cnt = c + 1;
}

typedef struct {
  const rd_index* h;
  const float* q;
  int32_t nprobe, k;
  int64_t* out_ids;
  float* out_dists;
  int32_t* out_lists;
} search_ctx;

static void probe_one(const rd_index* h, const float* q, int32_t nprobe, int32_t* lists) {
  cand* top = (cand*)malloc(sizeof(cand) * (size_t)nprobe);
  int32_t cnt = 0;
  for (int32_t j = 0; j < h->nlist; ++j)
    topk_push(top, &cnt, nprobe, rd_exact_l2(q, h->centroids + (int64_t)j * h->d, h->d), j);
  for (int32_t i = 0; i < nprobe; ++i) lists[i] = i < cnt ? (int32_t)top[i].id : -1;
  free(top);
}

static void search_range(void* p, int64_t b, int64_t e) {
  search_ctx* c = (search_ctx*)p;
  const rd_index* h = c->h;
  int32_t np = c->nprobe < h->nlist ? c->nprobe : h->nlist;
  int32_t* lists = (int32_t*)malloc(sizeof(int32_t) * (size_t)np);
  cand* top = (cand*)malloc(sizeof(cand) * (size_t)c->k);
  for (int64_t qi = b; qi < e; ++qi) {
    const float* q = c->q + qi * h->d;
    probe_one(h, q, np, lists);
    if (c->out_lists) {
      for (int32_t i = 0; i < c->nprobe; ++i) c->out_lists[qi * c->nprobe + i] = i < np ? lists[i] : -1;
      continue;
    }
    int32_t cnt = 0;
    for (int32_t pi = 0; pi < np; ++pi) {
      int32_t l = lists[pi];
      for (int64_t r = h->offsets[l]; r < h->offsets[l + 1]; ++r)
        topk_push(top, &cnt, c->k, rd_exact_l2(q, h->vectors + r * h->d, h->d), h->ids[r]);
    }
    for (int32_t i = 0; i < c->k; ++i) {
      c->out_ids[qi * c->k + i] = i < cnt ? top[i].id : -1;
      c->out_dists[qi * c->k + i] = i < cnt ? top[i].dist : INFINITY;
    }
  }
  free(top);
  free(lists);
}

int rd_search(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t k,
              int64_t* out_ids, float* out_dists, rd_search_stats* stats) {
  if (!h || (B > 0 && (!queries || !out_ids || !out_dists)))
    return fail(RD_ERR_INVALID, "search: null argument");
  if (B < 0 || nprobe < 1 || k < 1) return fail(RD_ERR_INVALID, "search: B >= 0, nprobe >= 1, k >= 1 required");
  search_ctx c = {h, queries, nprobe, k, out_ids, out_dists, NULL};
  rdo_parallel_for(B, 1, search_range, &c);
  if (stats) memset(stats, 0, sizeof *stats);
  return RD_OK;
}

int rd_probe(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t* out_lists) {
  if (!h || (B > 0 && (!queries || !out_lists))) return fail(RD_ERR_INVALID, "probe: null argument");
  if (B < 0 || nprobe < 1) return fail(RD_ERR_INVALID, "probe: nprobe >= 1 required");
  search_ctx c = {h, queries, nprobe, 1, NULL, NULL, out_lists};
  rdo_parallel_for(B, 1, search_range, &c);
  return RD_OK;
}

int rd_search_device(rd_index* h, const float* dq, int64_t B, int32_t nprobe, int32_t k, int64_t* di,
                     float* dd, void* stream, int32_t sync, rd_search_stats* st) {
  (void)h; (void)dq; (void)B; (void)nprobe; (void)k; (void)di; (void)dd; (void)stream; (void)sync; (void)st;
  return fail(RD_ERR_INVALID, "cpu oracle has no device search");
}

int rd_merge_topk_device(int32_t G, int64_t B, int32_t k, const int64_t* a, const float* b, int64_t* c,
                         float* d, void* s) {
  (void)G; (void)B; (void)k; (void)a; (void)b; (void)c; (void)d; (void)s;
  return fail(RD_ERR_INVALID, "cpu oracle has no device merge");
}

int rd_device_read_bandwidth(int32_t device, uint64_t bytes, double* out_gbs) {
  (void)device; (void)bytes; (void)out_gbs;
  return fail(RD_ERR_INVALID, "cpu oracle has no device");
}

int rd_timing_stages(rd_index* h, int32_t on) {
  (void)on;
  if (!h) return fail(RD_ERR_INVALID, "null index");
  return RD_OK;
}

int rd_timing_reset(rd_index* h) {
  if (!h) return fail(RD_ERR_INVALID, "null index");
  return RD_OK;
}

int rd_timing_read(rd_index* h, rd_timing* out) {
  if (!h || !out) return fail(RD_ERR_INVALID, "null argument");
  memset(out, 0, sizeof *out);
  return RD_OK;
}

int rd_merge_topk(int32_t G, int64_t B, int32_t k, const int64_t* sid, const float* sd, int64_t* oid,
                  float* od) {
  if (G < 1 || B < 0 || k < 1 || (B > 0 && (!sid || !sd || !oid || !od)))
    return fail(RD_ERR_INVALID, "merge: invalid arguments");
  cand* top = (cand*)malloc(sizeof(cand) * (size_t)k);
  for (int64_t q = 0; q < B; ++q) {
    int32_t cnt = 0;
    for (int32_t g = 0; g < G; ++g)
      for (int32_t i = 0; i < k; ++i) {
        int64_t id = sid[((int64_t)g * B + q) * k + i];
        if (id < 0) continue;
        topk_push(top, &cnt, k, sd[((int64_t)g * B + q) * k + i], id);
      }
    for (int32_t i = 0; i < k; ++i) {
      oid[q * k + i] = i < cnt ? top[i].id : -1;
      od[q * k + i] = i < cnt ? top[i].dist : INFINITY;
    }
  }
  free(top);
  return RD_OK;
}

/* ------------------------------------------------------------------ synthetic queries */
static void synth_vec(const rd_synth_desc* s, uint64_t sc, uint64_t sa, uint64_t sx, int64_t id, float* out) {
  int32_t a = (int32_t)(rd_splitmix_at(sa, (uint64_t)id) % (uint64_t)s->nlist);
  for (int32_t t = 0; t < s->d; ++t) {
    float c = unif(sc, (uint64_t)a * s->d + t);
    float noise = s->sigma * unif(sx, (uint64_t)(id * s->d + t));
    out[t] = c + noise;
  }
}

int rd_synth_vector(const rd_synth_desc* s, int64_t id, float* out) {
  int rc = check_desc(s);
  if (rc) return rc;
  if (id < 0 || id >= s->n || !out) return fail(RD_ERR_INVALID, "synth_vector: id out of range");
  synth_vec(s, rd_derive_seed(s->seed, RD_STREAM_CENTROIDS), rd_derive_seed(s->seed, RD_STREAM_ASSIGN),
            rd_derive_seed(s->seed, RD_STREAM_VECTOR_NOISE), id, out);
  return RD_OK;
}

int rd_synth_queries(const rd_synth_desc* s, int64_t b0, int64_t B, float qsigma, float* out, int64_t* src) {
  int rc = check_desc(s);
  if (rc) return rc;
  if (b0 < 0 || B < 0 || (B > 0 && !out)) return fail(RD_ERR_INVALID, "synth_queries: invalid arguments");
  uint64_t sc = rd_derive_seed(s->seed, RD_STREAM_CENTROIDS), sa = rd_derive_seed(s->seed, RD_STREAM_ASSIGN),
           sx = rd_derive_seed(s->seed, RD_STREAM_VECTOR_NOISE), sq = rd_derive_seed(s->seed, RD_STREAM_QUERY_PICK),
           sn = rd_derive_seed(s->seed, RD_STREAM_QUERY_NOISE);
  for (int64_t i = 0; i < B; ++i) {
    int64_t b = b0 + i;
    int64_t r = (int64_t)(rd_splitmix_at(sq, (uint64_t)b) % (uint64_t)s->n);
    float* q = out + i * s->d;
    synth_vec(s, sc, sa, sx, r, q);
    for (int32_t t = 0; t < s->d; ++t) q[t] = q[t] + qsigma * unif(sn, (uint64_t)(b * s->d + t));
    if (src) src[i] = r;
  }
  return RD_OK;
}

/* ------------------------------------------------------------------ placement arithmetic */
/* gpu_used of ragsim::check_feasible (memory_planner.cpp:17-20) with the decode
 * workspace share of queue_capacity (prefetch_timeline.cpp:84-86). */
int rd_llm_reservation_bytes(const rd_llm_reservation* r, double* out) {
  if (!r || !out) return fail(RD_ERR_INVALID, "null argument");
  if (r->gen_batch_size < 0 || r->w_gpu < 0 || r->w_gpu > 1 || r->c_gpu < 0 || r->c_gpu > 1)
    return fail(RD_ERR_INVALID, "reservation: fractions in [0,1] and batch >= 0 required");
  double W = (double)r->weight_total;
  double C = (double)r->kv_bytes_per_request * r->gen_batch_size;
  double H = (double)r->workspace_bytes_per_request * r->gen_batch_size;
  if (r->decode_phase) H *= r->workspace_fraction;
  *out = r->w_gpu * W + r->c_gpu * C + H;
  return RD_OK;
}

/* queue_capacity's rule (prefetch_timeline.cpp:87-89): max(1, floor(free / item)). */
int32_t rd_staging_depth(double free_bytes, double item_bytes) {
  if (item_bytes <= 0) return 1;
  double q = floor(free_bytes / item_bytes);
  if (q < 1) return 1;
  if (q > 1 << 20) return 1 << 20;
  return (int32_t)q;
}

/* ------------------------------------------------------------------ sampled oracle (oracle-only entry)
 * rd_oracle_synth_search: exact IVF-Flat (same semantics as rd_search above) over the synthetic
 * knowledge base `s` restricted to the row stripes g of s->num_shards with bit g set in
 * shard_mask, WITHOUT materialising the knowledge base: only the probed lists' rows of the selected
 * stripes are regenerated from (seed, id) ("CPU verification on a sampled query
 * subset only, with vectors regenerated from (seed, id)"). This is how a 100M x 768 (307 GB) index
 * is checked on a host that cannot hold it. s->shard is ignored. Not part of rd.h. */
typedef struct {
  const rd_synth_desc* s;
  uint64_t sc, sx;
  const float* centroids;
  const float* q;
  int32_t np, k;
  int32_t* lists;              /* B x np probes */
  const int64_t* mem_off;      /* per marked list slot: member range in mem_ids */
  const int64_t* mem_ids;      /* selected-stripe members, ascending id */
  const int32_t* mark;         /* list -> slot or -1 */
  const int32_t* marked;       /* slot -> list */
  const int64_t* pair_off;     /* slot -> range in pair_q */
  const int64_t* pair_q;       /* (query * np + probe index) pairs per slot */
  cand* part;                  /* B x np x k partial top-k */
  int32_t* part_cnt;           /* B x np */
} synth_search_ctx;

static void synth_probe_range(void* p, int64_t b, int64_t e) {
  synth_search_ctx* c = (synth_search_ctx*)p;
  const int32_t d = c->s->d, nl = c->s->nlist;
  cand* top = (cand*)malloc(sizeof(cand) * (size_t)c->np);
  for (int64_t qi = b; qi < e; ++qi) {
    int32_t cnt = 0;
    for (int32_t j = 0; j < nl; ++j)
      topk_push(top, &cnt, c->np, rd_exact_l2(c->q + qi * d, c->centroids + (int64_t)j * d, d), j);
    for (int32_t i = 0; i < c->np; ++i) c->lists[qi * c->np + i] = (int32_t)top[i].id;
  }
  free(top);
}

static void synth_scan_range(void* p, int64_t b, int64_t e) {
  synth_search_ctx* c = (synth_search_ctx*)p;
  const int32_t d = c->s->d;
  float* x = (float*)malloc(sizeof(float) * (size_t)d);
  for (int64_t slot = b; slot < e; ++slot) {
    const float* cen = c->centroids + (int64_t)c->marked[slot] * d;
    for (int64_t r = c->mem_off[slot]; r < c->mem_off[slot + 1]; ++r) {
      const int64_t id = c->mem_ids[r];
      for (int32_t t = 0; t < d; ++t) x[t] = cen[t] + c->s->sigma * unif(c->sx, (uint64_t)(id * d + t));
      for (int64_t pi = c->pair_off[slot]; pi < c->pair_off[slot + 1]; ++pi) {
        const int64_t qp = c->pair_q[pi];
        const int64_t qi = qp / c->np;
        topk_push(c->part + qp * c->k, c->part_cnt + qp, c->k, rd_exact_l2(c->q + qi * d, x, d), id);
      }
    }
  }
  free(x);
}

typedef struct {
  uint64_t sa;
  int32_t nl;
  int32_t* assign;
} assign_gen_ctx;

static void synth_assign_range(void* p, int64_t b, int64_t e) {
  assign_gen_ctx* a = (assign_gen_ctx*)p;
  for (int64_t i = b; i < e; ++i) a->assign[i] = (int32_t)(rd_splitmix_at(a->sa, (uint64_t)i) % (uint64_t)a->nl);
}

int rd_oracle_synth_search(const rd_synth_desc* s, uint64_t shard_mask, const float* queries, int64_t B,
                           int32_t nprobe, int32_t k, int64_t* out_ids, float* out_dists) {
  int rc = check_desc(s);
  if (rc) return rc;
  if (B < 0 || nprobe < 1 || k < 1 || (B > 0 && (!queries || !out_ids || !out_dists)))
    return fail(RD_ERR_INVALID, "synth_search: invalid arguments");
  if (B == 0) return RD_OK;
  const int64_t n = s->n;
  const int32_t d = s->d, nl = s->nlist, G = s->num_shards;
  const int32_t np = nprobe < nl ? nprobe : nl;
  synth_search_ctx c;
  memset(&c, 0, sizeof c);
  c.s = s;
  c.sc = rd_derive_seed(s->seed, RD_STREAM_CENTROIDS);
  c.sx = rd_derive_seed(s->seed, RD_STREAM_VECTOR_NOISE);
  c.q = queries;
  c.np = np;
  c.k = k;
  float* cen = (float*)malloc(sizeof(float) * (size_t)nl * d);
  gen_ctx gc = {s, c.sc, c.sx, NULL, NULL, cen, NULL};
  rdo_parallel_for(nl, 16, gen_centroids, &gc);
  c.centroids = cen;
  int32_t* lists = (int32_t*)malloc(sizeof(int32_t) * (size_t)B * np);
  c.lists = lists;
  rdo_parallel_for(B, 1, synth_probe_range, &c);
  /* marked lists and their (query, probe) pairs */
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * (size_t)nl);
  for (int32_t l = 0; l < nl; ++l) mark[l] = -1;
  int32_t nm = 0;
  for (int64_t i = 0; i < B * np; ++i)
    if (mark[lists[i]] < 0) mark[lists[i]] = nm++;
  int32_t* marked = (int32_t*)malloc(sizeof(int32_t) * (size_t)nm);
  for (int32_t l = 0; l < nl; ++l)
    if (mark[l] >= 0) marked[mark[l]] = l;
  int64_t* pair_off = (int64_t*)calloc((size_t)nm + 1, sizeof(int64_t));
  int64_t* pair_q = (int64_t*)malloc(sizeof(int64_t) * (size_t)B * np);
  for (int64_t i = 0; i < B * np; ++i) pair_off[mark[lists[i]] + 1]++;
  for (int32_t m = 0; m < nm; ++m) pair_off[m + 1] += pair_off[m];
  int64_t* pcur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nm > 0 ? nm : 1));
  for (int32_t m = 0; m < nm; ++m) pcur[m] = pair_off[m];
  for (int64_t i = 0; i < B * np; ++i) pair_q[pcur[mark[lists[i]]]++] = i;
  free(pcur);
  /* membership of the marked lists, ascending id, restricted to the selected stripes */
  int32_t* assign = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  if (!assign) return fail(RD_ERR_RUNTIME, "synth_search: out of host memory");
  assign_gen_ctx ac = {rd_derive_seed(s->seed, RD_STREAM_ASSIGN), nl, assign};
  rdo_parallel_for(n, 1 << 20, synth_assign_range, &ac);
  int64_t* full_len = (int64_t*)calloc((size_t)nl, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) full_len[assign[i]]++;
  int64_t* mem_off = (int64_t*)calloc((size_t)nm + 1, sizeof(int64_t));
  for (int32_t m = 0; m < nm; ++m) {
    const int64_t len = full_len[marked[m]];
    int64_t sel = 0;
    for (int32_t g = 0; g < G; ++g)
      if ((shard_mask >> (g & 63)) & 1u) sel += (int64_t)(g + 1) * len / G - (int64_t)g * len / G;
    mem_off[m + 1] = mem_off[m] + sel;
  }
  int64_t* mem_ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)(mem_off[nm] > 0 ? mem_off[nm] : 1));
  int64_t* pos = (int64_t*)calloc((size_t)nl, sizeof(int64_t));
  int64_t* mcur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nm > 0 ? nm : 1));
  for (int32_t m = 0; m < nm; ++m) mcur[m] = mem_off[m];
  for (int64_t i = 0; i < n; ++i) {
    const int32_t l = assign[i];
    const int64_t p = pos[l]++;
    if (mark[l] < 0) continue;
    const int64_t len = full_len[l];
    /* stripe of position p: the g with g*len/G <= p < (g+1)*len/G */
    int32_t g = (int32_t)((p * G) / (len > 0 ? len : 1));
    while (g + 1 < G && (int64_t)(g + 1) * len / G <= p) ++g;
    while (g > 0 && (int64_t)g * len / G > p) --g;
    if ((shard_mask >> (g & 63)) & 1u) mem_ids[mcur[mark[l]]++] = i;
  }
  free(mcur);
  free(pos);
  free(full_len);
  free(assign);
  c.mark = mark;
  c.marked = marked;
  c.mem_off = mem_off;
  c.mem_ids = mem_ids;
  c.pair_off = pair_off;
  c.pair_q = pair_q;
  c.part = (cand*)malloc(sizeof(cand) * (size_t)B * np * k);
  c.part_cnt = (int32_t*)calloc((size_t)B * np, sizeof(int32_t));
  rdo_parallel_for(nm, 1, synth_scan_range, &c);
  cand* top = (cand*)malloc(sizeof(cand) * (size_t)k);
  for (int64_t qi = 0; qi < B; ++qi) {
    int32_t cnt = 0;
    for (int32_t pi = 0; pi < np; ++pi) {
      const int64_t qp = qi * np + pi;
      for (int32_t i = 0; i < c.part_cnt[qp]; ++i) topk_push(top, &cnt, k, c.part[qp * k + i].dist, c.part[qp * k + i].id);
    }
    for (int32_t i = 0; i < k; ++i) {
      out_ids[qi * k + i] = i < cnt ? top[i].id : -1;
      out_dists[qi * k + i] = i < cnt ? top[i].dist : INFINITY;
    }
  }
  free(top);
  free(c.part);
  free(c.part_cnt);
  free(mem_ids);
  free(mem_off);
  free(pair_q);
  free(pair_off);
  free(marked);
  free(mark);
  free(lists);
  free(cen);
  return RD_OK;
}

/* ------------------------------------------------------------------ shard groups (rd.h rd_group_*)
 * Single-process forms only: every stripe is searched in turn and the per-stripe top-k are merged
 * on the host (rd_merge_topk) — the algebra the engine's NCCL gather + device merge must match. */
struct rd_group {
  rd_index** shards;
  int32_t G;
};

int rd_group_create(rd_index* const* shards, int32_t G, rd_group** out) {
  if (!shards || G < 1 || !out) return fail(RD_ERR_INVALID, "group_create: invalid arguments");
  for (int32_t g = 0; g < G; ++g) {
    if (!shards[g]) return fail(RD_ERR_INVALID, "group: null stripe %d", g);
    if (shards[g]->d != shards[0]->d || shards[g]->nlist != shards[0]->nlist)
      return fail(RD_ERR_INVALID, "group: stripes must share d and nlist");
    for (int32_t h = 0; h < g; ++h)
      if (shards[h] == shards[g]) return fail(RD_ERR_INVALID, "group: stripe handle %d given twice", g);
  }
  rd_group* grp = (rd_group*)calloc(1, sizeof *grp);
  grp->shards = (rd_index**)malloc(sizeof(rd_index*) * (size_t)G);
  memcpy(grp->shards, shards, sizeof(rd_index*) * (size_t)G);
  grp->G = G;
  *out = grp;
  return RD_OK;
}

int rd_group_create_synthetic(const rd_synth_desc* desc, const int32_t* devices, int32_t G, rd_group** out) {
  if (!desc || !devices || G < 1 || !out) return fail(RD_ERR_INVALID, "group_create_synthetic: invalid arguments");
  rd_index** s = (rd_index**)calloc((size_t)G, sizeof(rd_index*));
  for (int32_t g = 0; g < G; ++g) {
    rd_synth_desc one = *desc;
    one.shard = g;
    one.num_shards = G;
    int rc = rd_index_create_synthetic(&one, devices[g], &s[g]);
    if (rc) {
      for (int32_t h = 0; h < g; ++h) rd_index_destroy(s[h]);
      free(s);
      return rc;
    }
  }
  int rc = rd_group_create(s, G, out);
  if (rc)
    for (int32_t g = 0; g < G; ++g) rd_index_destroy(s[g]);
  free(s);
  return rc;
}

int rd_group_unique_id(uint8_t* out) {
  (void)out;
  return fail(RD_ERR_INVALID, "cpu oracle has no communicator");
}

int rd_group_create_rank(rd_index* shard, const uint8_t* id, int32_t nranks, int32_t rank, rd_group** out) {
  (void)shard; (void)id; (void)nranks; (void)rank; (void)out;
  return fail(RD_ERR_INVALID, "cpu oracle has no communicator");
}

int rd_group_info_get(const rd_group* g, rd_group_info* o) {
  if (!g || !o) return fail(RD_ERR_INVALID, "null argument");
  memset(o, 0, sizeof *o);
  o->num_shards = g->G;
  o->local_shards = g->G;
  o->nranks = 1;
  o->transport = g->G > 1 ? RD_GROUP_TRANSPORT_COPY : RD_GROUP_TRANSPORT_NONE;
  for (int32_t i = 0; i < g->G; ++i) {
    o->n += g->shards[i]->n;
    for (int32_t l = 0; l < g->shards[i]->nlist; ++l)
      if (g->shards[i]->resident[l]) o->n_resident += g->shards[i]->offsets[l + 1] - g->shards[i]->offsets[l];
  }
  return RD_OK;
}

rd_index* rd_group_shard(rd_group* g, int32_t i) {
  if (!g || i < 0 || i >= g->G) return NULL;
  return g->shards[i];
}

int rd_group_place(rd_group* g, const rd_placement* p) {
  if (!g || !p) return fail(RD_ERR_INVALID, "null argument");
  for (int32_t i = 0; i < g->G; ++i) {
    int rc = rd_index_place(g->shards[i], p);
    if (rc) return rc;
  }
  return RD_OK;
}

int rd_group_search(rd_group* g, const float* queries, int64_t B, int32_t nprobe, int32_t k, int64_t* out_ids,
                    float* out_dists, rd_search_stats* stats) {
  if (!g || B < 0 || nprobe < 1 || k < 1 || (B > 0 && (!queries || !out_ids || !out_dists)))
    return fail(RD_ERR_INVALID, "group search: invalid arguments");
  if (stats) memset(stats, 0, sizeof *stats);
  if (B == 0) return RD_OK;
  int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)g->G * B * k);
  float* dists = (float*)malloc(sizeof(float) * (size_t)g->G * B * k);
  int rc = RD_OK;
  for (int32_t i = 0; i < g->G && rc == RD_OK; ++i)
    rc = rd_search(g->shards[i], queries, B, nprobe, k, ids + (size_t)i * B * k, dists + (size_t)i * B * k, NULL);
  if (rc == RD_OK) rc = rd_merge_topk(g->G, B, k, ids, dists, out_ids, out_dists);
  free(ids);
  free(dists);
  return rc;
}

int rd_group_search_device(rd_group* g, const float* dq, int64_t B, int32_t nprobe, int32_t k, int64_t* di, float* dd,
                           void* stream, int32_t sync, rd_search_stats* st) {
  (void)g; (void)dq; (void)B; (void)nprobe; (void)k; (void)di; (void)dd; (void)stream; (void)sync; (void)st;
  return fail(RD_ERR_INVALID, "cpu oracle has no device search");
}

void rd_group_destroy(rd_group* g) {
  if (!g) return;
  for (int32_t i = 0; i < g->G; ++i) rd_index_destroy(g->shards[i]);
  free(g->shards);
  free(g);
}
