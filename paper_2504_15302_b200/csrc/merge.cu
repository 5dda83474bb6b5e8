// merge.cu — N6 per-query top-k merge and N7 exact fp32 rerank (sm_100a).
//
// One CTA per query: its warps merge the per-tile top-32 partial lists with
// warp bitonic merges, the block keeps the 32 best approximate candidates and
// recomputes their distances with the canonical exact sum (8 lanes per
// candidate), orders them by (exact distance, id) and writes the top-k. The
// result is certified when the 32nd approximate distance, less the scan's
// error bound, still exceeds the k-th exact distance: then no vector dropped
// anywhere upstream can belong to the exact top-k (SURVEY §7 "Hard parts").
#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr float kInf = __builtin_huge_valf();
constexpr long long kNoKey = 0x7fffffffffffffffll;
#ifndef RD_DECODE_BATCH
#define RD_DECODE_BATCH 12
#endif
constexpr int kDecodeBatch = RD_DECODE_BATCH;  // 8-element row chunks per thread per round trip (staged rerank; 12: the 24 candidate rows of a residual-store search in one round, B = 1 +0.8 %)

// One CTA per query. kStage (small batches, one latency chain per query): the candidate rows are
// decoded into fp32 rows in shared memory (128-bit loads, every load of a round in flight, split3
// triples summed once per element) and the canonical sums read them with q already widened to fp64;
// otherwise each group of 8 lanes streams its row from global memory (enough CTAs are resident to
// hide the latency).
template <bool kStage>
__global__ void __launch_bounds__(256, kStage ? 1 : 8) merge_rerank_kernel(const MergeParams p) {
  RD_TS(13);  // entry, before the wait on the previous kernel
  RD_PDL_PROLOGUE();
  extern __shared__ __align__(16) float dyn[];  // kStage: qd[d] (fp64), rows[32][d + kStagePad] (fp32)
  __shared__ float sd[8][kTopK];
  __shared__ long long sk[8][kTopK];
  __shared__ float ex_d[kTopK];
  __shared__ long long ex_id[kTopK];
  __shared__ const float* rowp[kTopK];   // fp32 row (offloaded list / fp32 store), or nullptr
  __shared__ long long srow[kTopK];      // split3 store row, or -1
  __shared__ float tau_s;
  RD_TS(0);
  const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cnt = min(p.part_count[b], p.part_cap);
  if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0) p.dbg[15] = (unsigned long long)cnt;
  const float* q = p.queries + (size_t)b * p.d;
  double* qd = reinterpret_cast<double*>(dyn);
  if constexpr (kStage) {
    for (int i = tid; i < (p.d >> 2); i += 256) {
      const float4 v = reinterpret_cast<const float4*>(q)[i];
      qd[4 * i] = v.x, qd[4 * i + 1] = v.y, qd[4 * i + 2] = v.z, qd[4 * i + 3] = v.w;
    }
  }

  // partial lists are ascending; read reversed to get a descending batch. Four partials per warp
  // are loaded before any is merged so their latencies overlap.
  float ld = kInf;
  long long lk = kNoKey;
  for (int i0 = warp; i0 < cnt; i0 += 32) {
    float bd[4];
    int br[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + 8 * u;
      br[u] = -1;
      if (i < cnt) {
        const size_t o = ((size_t)b * p.part_cap + i) * kTopK + (kTopK - 1 - lane);
        bd[u] = p.part_dist[o];
        br[u] = p.part_row[o];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i0 + 8 * u >= cnt) break;
      const float v = br[u] < 0 ? kInf : bd[u];
      const long long key = br[u] < 0 ? kNoKey : (long long)br[u];
      if (pair_less(v, key, ld, lk)) {
        ld = v;
        lk = key;
      }
#pragma unroll
      for (int j = 16; j > 0; j >>= 1) bitonic_step(ld, lk, lane, j, true);
    }
  }
  // the eight warps' lists: a merge tree (4, 2, 1 warps) into warp 0
  sd[warp][lane] = ld;
  sk[warp][lane] = lk;
  __syncthreads();
  for (int st = 1; st < 8; st <<= 1) {
    if ((warp & (2 * st - 1)) == 0) {
      const float v = sd[warp + st][kTopK - 1 - lane];
      const long long key = sk[warp + st][kTopK - 1 - lane];
      if (pair_less(v, key, ld, lk)) {
        ld = v;
        lk = key;
      }
#pragma unroll
      for (int j = 16; j > 0; j >>= 1) bitonic_step(ld, lk, lane, j, true);
      sd[warp][lane] = ld;
      sk[warp][lane] = lk;
    }
    __syncthreads();
  }
  RD_TS(1);
  if (warp == 0) {
    // The best m = min(32, k + margin) candidates are reranked: the (m+1)-th approximate distance
    // bounds every row not reranked (the rest of the list and everything the scan dropped), so
    // certification reads tau = that distance; the spare candidates keep it holding unless the data
    // has (near-)ties across ranks k..m (duplicates; then the exact fallback runs). Fewer rows cut
    // the rerank's HBM reads (k = 10, margin 8: 18 of 32).
    const int m = p.m_rerank;
    const float* xp = nullptr;
    long long sr = -1;
    long long id = kNoKey;
    if (lk != kNoKey && lane < m) {  // candidate rows: list of the row (row_list), address, user id
      const int l = __ldg(p.row_list + lk);
      id = __ldg(p.ids + lk);
      const float* base = p.list_base[l];
      const long long i = lk - __ldg(p.list_off + l);
      if (base)
        xp = base + (size_t)i * p.d;
      else
        sr = __ldg(p.res_row0 + l) + i;
    }
    rowp[lane] = xp;
    srow[lane] = sr;
    ex_id[lane] = id;
    if (lane == min(m, kTopK - 1)) tau_s = ld;
  }
  __syncthreads();

  RD_TS(2);
  // exact rerank: thread (c = tid/8, j = tid%8)
  const int c = tid >> 3, j8 = tid & 7;
  const float* xp = rowp[c];
  const long long sr = srow[c];
  const bool have = xp || sr >= 0;
  float e;
  if constexpr (kStage) {
    // decode: task = (row r, 8-element chunk cc) over the m candidate rows; kDecodeBatch tasks per
    // thread per round, all loads in flight (split3: x1, x2, x3 chunks; fp32: two float4 — rows of
    // offloaded lists are mapped host memory, so plain loads throughout)
    float* st = dyn + 2 * p.d;
    const int ds = p.d + kStagePad, nc = p.d >> 3;
    const int ntask = min(p.m_rerank, kTopK) * nc;
    for (int t0 = tid; t0 < ntask; t0 += 256 * kDecodeBatch) {
      uint4 a[kDecodeBatch], bb[kDecodeBatch], cc3[kDecodeBatch];
#pragma unroll
      for (int u = 0; u < kDecodeBatch; ++u) {
        const int t = t0 + u * 256;
        if (t >= ntask) break;
        const int r = t / nc, ch = t - r * nc;
        const long long rs = srow[r];
        const float* rp = rowp[r];
        if (rs >= 0) {
          a[u] = reinterpret_cast<const uint4*>(p.x12 + (size_t)rs * 2 * p.d)[ch];
          bb[u] = reinterpret_cast<const uint4*>(p.x12 + (size_t)rs * 2 * p.d + p.d)[ch];
          cc3[u] = reinterpret_cast<const uint4*>(p.x3 + (size_t)rs * p.d)[ch];
        } else if (rp) {
          a[u] = reinterpret_cast<const uint4*>(rp)[2 * ch];
          bb[u] = reinterpret_cast<const uint4*>(rp)[2 * ch + 1];
        }
      }
#pragma unroll
      for (int u = 0; u < kDecodeBatch; ++u) {
        const int t = t0 + u * 256;
        if (t >= ntask) break;
        const int r = t / nc, ch = t - r * nc;
        float4* o = reinterpret_cast<float4*>(st + r * ds + 8 * ch);
        if (srow[r] >= 0) {
          const __nv_bfloat16* h1 = reinterpret_cast<const __nv_bfloat16*>(&a[u]);
          const __nv_bfloat16* h2 = reinterpret_cast<const __nv_bfloat16*>(&bb[u]);
          const __nv_bfloat16* h3 = reinterpret_cast<const __nv_bfloat16*>(&cc3[u]);
          float xv[8];
#pragma unroll
          for (int e8 = 0; e8 < 8; ++e8)
            xv[e8] = __fadd_rn(__fadd_rn(__bfloat162float(h1[e8]), __bfloat162float(h2[e8])), __bfloat162float(h3[e8]));
          o[0] = make_float4(xv[0], xv[1], xv[2], xv[3]);
          o[1] = make_float4(xv[4], xv[5], xv[6], xv[7]);
        } else if (rowp[r]) {
          o[0] = *reinterpret_cast<const float4*>(&a[u]);
          o[1] = *reinterpret_cast<const float4*>(&bb[u]);
        }
      }
    }
    __syncthreads();
    RD_TS(3);
    e = exact_l2_group8_qd_cnt(qd, st + c * ds, have ? p.d : 0, j8);
  } else {
    // a padded slot runs zero terms so the warp stays converged for the shuffles; fp32 rows from HBM:
    // 16 loads deep (32 registers: one wave of 8 CTAs per SM); split3 rows: 128-bit loads and a
    // transpose through a per-group scratch (exact_l2_group8_split3), warp-uniform calls
    __shared__ __align__(16) float scr[8][4][72];  // [warp][group]: 64 floats + 8 of bank padding
    if (p.x12 && p.d % 64 == 0) {
      const __nv_bfloat16* x12 = p.x12 + (size_t)(sr >= 0 ? sr : 0) * 2 * p.d;
      const __nv_bfloat16* x3 = p.x3 + (size_t)(sr >= 0 ? sr : 0) * p.d;
      const float e3 = exact_l2_group8_split3(q, x12, x3, p.d, j8, sr >= 0, scr[warp][(tid >> 3) & 3]);
      const float ef = exact_l2_group8_row<16>(q, row_f32(xp ? xp : q), p.d, j8, xp ? p.d : 0);
      e = sr >= 0 ? e3 : ef;
    } else {
      const RowRef x = sr >= 0 ? row_split3(p.x12, p.x3, sr, p.d) : row_f32(xp ? xp : q);
      e = exact_l2_group8_row<16>(q, x, p.d, j8, have ? p.d : 0);
    }
  }
  if (!have) e = kInf;
  if (j8 == 0) ex_d[c] = e;
  __syncthreads();
  RD_TS(4);
  if (warp == 0) {
    float dd = ex_d[lane];
    long long kk = ex_id[lane];
    warp_sort32(dd, kk, lane, true);
    if (lane < p.k) {
      p.out_ids[(size_t)b * p.k + lane] = kk == kNoKey ? -1 : kk;
      p.out_dists[(size_t)b * p.k + lane] = kk == kNoKey ? kInf : dd;
    }
    for (int i = kTopK + lane; i < p.k; i += 32) {  // k > 32 is rejected by the host; pad defensively
      p.out_ids[(size_t)b * p.k + i] = -1;
      p.out_dists[(size_t)b * p.k + i] = kInf;
    }
    const float ek = __shfl_sync(0xffffffffu, dd, min(p.k, kTopK) - 1);
    if (lane == 0) {
      const float tau = tau_s;
      if (tau != kInf) {
        const float qn = p.qnorm[b];
        const float xm = p.xmax;
        const float eps = 2.f * p.gamma * sqrtf(qn) * xm + 16.f * kUnit * (qn + xm * xm) + 1e-30f;
        if (!(tau - eps > ek)) p.fail_list[atomicAdd(p.margin_fail, 1u)] = b;
      }
    }
  }
  RD_TS_END();
}

__global__ void shard_merge_kernel(int G, long long B, int k, const long long* __restrict__ ids,
                                   const float* __restrict__ dists, long long* __restrict__ oid,
                                   float* __restrict__ od) {
  // one warp per query; k <= 32; candidates G*k absorbed in batches of 32
  const long long q = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= B) return;
  float ld = kInf;
  long long lk = kNoKey;
  const long long tot = (long long)G * k;
  for (long long c0 = 0; c0 < tot; c0 += 32) {
    const long long c = c0 + lane;
    float v = kInf;
    long long key = kNoKey;
    if (c < tot) {
      const int g = (int)(c / k), i = (int)(c - (long long)g * k);
      const long long id = ids[((long long)g * B + q) * k + i];
      if (id >= 0) {
        v = dists[((long long)g * B + q) * k + i];
        key = id;
      }
    }
    warp_merge32(ld, lk, v, key, lane);
  }
  if (lane < k) {
    oid[q * k + lane] = lk == kNoKey ? -1 : lk;
    od[q * k + lane] = lk == kNoKey ? kInf : ld;
  }
}

// Shard merge for any k: one CTA per query sorts its G * k shard candidates by (distance, id) in
// shared memory (bitonic over the next power of two, padding +inf) and writes the first k. Shard g's
// ids / distances of query q sit at ids + g * ids_stride (bytes) + q * k, likewise the distances, so
// both the [G][B][k] arrays of rd_merge_topk_device and the packed per-shard slots of a shard group
// (group.cu: [ids B x k | dists B x k] per slot) are read in place.
__global__ void __launch_bounds__(256) shard_merge_sort_kernel(int G, long long B, int k, int P,
                                                               const char* __restrict__ ids, size_t ids_stride,
                                                               const char* __restrict__ dists, size_t d_stride,
                                                               long long* __restrict__ oid, float* __restrict__ od,
                                                               int kout) {
  RD_PDL_PROLOGUE();
  extern __shared__ __align__(16) unsigned char sm_raw[];
  long long* sk = reinterpret_cast<long long*>(sm_raw);
  float* sv = reinterpret_cast<float*>(sk + P);
  const long long q = blockIdx.x;
  const int tot = G * k;
  for (int c = threadIdx.x; c < P; c += blockDim.x) {
    float v = kInf;
    long long key = kNoKey;
    if (c < tot) {
      const int g = c / k, i = c - g * k;
      const long long id = reinterpret_cast<const long long*>(ids + (size_t)g * ids_stride)[q * k + i];
      if (id >= 0) {
        v = reinterpret_cast<const float*>(dists + (size_t)g * d_stride)[q * k + i];
        key = id;
      }
    }
    sv[c] = v;
    sk[c] = key;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int c = threadIdx.x; c < P; c += blockDim.x) {
        const int o = c ^ stride;
        if (o > c) {
          const bool up = (c & size) == 0;
          const float a = sv[c], b = sv[o];
          const long long ka = sk[c], kb = sk[o];
          if (pair_less(b, kb, a, ka) == up) {
            sv[c] = b, sv[o] = a;
            sk[c] = kb, sk[o] = ka;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < kout; i += blockDim.x) {
    const bool ok = i < P && sk[i] != kNoKey;
    oid[q * kout + i] = ok ? sk[i] : -1;
    od[q * kout + i] = ok ? sv[i] : kInf;
  }
}

// Exact fallback in one launch. Persistent: work item w -> (failed query w / nprobe, probe
// w % nprobe), the exact top-32 of that list; the last CTA to finish merges each failed query's
// nprobe partials and overwrites its result row, then re-arms the completion counter. With no
// failures (the normal case) every CTA returns at once.
__global__ void __launch_bounds__(256) fallback_kernel(const FallbackParams p) {
  RD_PDL_PROLOGUE();
  __shared__ float wd[8][kTopK];
  __shared__ long long wk[8][kTopK];
  __shared__ bool last;
  const int nf = (int)*p.fail_count;
  if (nf == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long work = (long long)nf * p.nprobe;
  for (long long w = blockIdx.x; w < work; w += gridDim.x) {
    const int q = p.fail_list[w / p.nprobe];
    const int l = p.probes[(size_t)q * p.nprobe + (w % p.nprobe)];
    float ld = kInf;
    long long lk = kNoKey;
    if (l >= 0) {
      const long long r0 = p.list_off[l], r1 = p.list_off[l + 1];
      const float* base = p.list_base[l];  // nullptr: the list's rows are in the split3 store
      const long long s0 = base ? 0 : p.res_row0[l];
      const float* qv = p.queries + (size_t)q * p.d;
      for (long long c = r0 + 32LL * warp; c < r1; c += 32LL * 8) {
        float mine = kInf;
        long long myid = kNoKey;
        for (int pass = 0; pass < 8; ++pass) {
          const long long row = c + pass * 4 + (lane >> 3);
          const bool ok = row < r1;
          const RowRef x = !ok ? row_f32(qv)
                           : base ? row_f32(base + (size_t)(row - r0) * p.d)
                                  : row_split3(p.x12, p.x3, s0 + (row - r0), p.d);
          const float e = exact_l2_group8_row(qv, x, p.d, lane & 7, ok ? p.d : 0);
          const float v = __shfl_sync(0xffffffffu, e, (lane & 3) * 8);
          if ((lane >> 2) == pass && c + lane < r1) {
            mine = v;
            myid = p.ids[c + lane];
          }
        }
        const float thr = __shfl_sync(0xffffffffu, ld, 31);
        const long long thk = __shfl_sync(0xffffffffu, lk, 31);
        const bool pass = pair_less(mine, myid, thr, thk);
        if (__any_sync(0xffffffffu, pass)) warp_merge32(ld, lk, pass ? mine : kInf, pass ? myid : kNoKey, lane);
      }
    }
    wd[warp][lane] = ld;
    wk[warp][lane] = lk;
    __syncthreads();
    if (warp == 0) {
      for (int o = 1; o < 8; ++o) warp_merge32(ld, lk, wd[o][lane], wk[o][lane], lane);
      p.fb_dist[w * kTopK + lane] = ld;
      p.fb_id[w * kTopK + lane] = lk;
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(p.done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int f = warp; f < nf; f += 8) {  // one warp per failed query
    float ld = kInf;
    long long lk = kNoKey;
    for (int i = 0; i < p.nprobe; ++i) {
      const long long w = (long long)f * p.nprobe + i;
      warp_merge32(ld, lk, __ldcg(p.fb_dist + w * kTopK + lane), __ldcg(p.fb_id + w * kTopK + lane), lane);
    }
    const int q = p.fail_list[f];
    if (lane < p.k) {
      p.out_ids[(size_t)q * p.k + lane] = lk == kNoKey ? -1 : lk;
      p.out_dists[(size_t)q * p.k + lane] = lk == kNoKey ? kInf : ld;
    }
  }
  if (threadIdx.x == 0) *p.done_ctr = 0u;
}

}  // namespace

cudaError_t launch_fallback(const FallbackParams& p, int num_sms, cudaStream_t s) {
  return launch_k(fallback_kernel, dim3(num_sms), dim3(256), 0, s, p);
}

cudaError_t launch_merge(const MergeParams& p, bool stage, cudaStream_t s) {
  if (p.B == 0) return cudaSuccess;
  if (stage && p.d % 8 == 0) {  // qd (fp64) + 32 decoded fp32 rows (8-element chunks)
    const size_t smem = sizeof(float) * (2 * (size_t)p.d + kTopK * ((size_t)p.d + kStagePad));
    return launch_k(merge_rerank_kernel<true>, dim3(p.B), dim3(256), smem, s, p);
  }
  return launch_k(merge_rerank_kernel<false>, dim3(p.B), dim3(256), 0, s, p);
}

cudaError_t launch_shard_merge(int G, long long B, int k, const long long* ids, const float* dists,
                               long long* out_ids, float* out_dists, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  if (k <= 32) {  // one warp per query, merges in registers
    const long long threads = B * 32;
    shard_merge_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(G, B, k, ids, dists, out_ids, out_dists);
    return cudaGetLastError();
  }
  return launch_shard_merge_strided(G, B, k, reinterpret_cast<const char*>(ids), (size_t)B * k * sizeof(long long),
                                    reinterpret_cast<const char*>(dists), (size_t)B * k * sizeof(float), out_ids,
                                    out_dists, s);
}

int shard_merge_max_candidates() { return 8192; }

cudaError_t launch_shard_merge_strided(int G, long long B, int k, const char* ids, size_t ids_stride,
                                       const char* dists, size_t d_stride, long long* out_ids, float* out_dists,
                                       cudaStream_t s, int kout) {
  if (B == 0) return cudaSuccess;
  if (kout <= 0) kout = k;
  const long long tot = (long long)G * k;
  if (G < 1 || k < 1 || tot > shard_merge_max_candidates()) return cudaErrorInvalidValue;
  int P = 1;
  while (P < tot) P <<= 1;
  const size_t smem = (size_t)P * (sizeof(long long) + sizeof(float));
  return launch_k(shard_merge_sort_kernel, dim3((unsigned)B), dim3(256), smem, s, G, B, k, P, ids, ids_stride, dists,
                  d_stride, out_ids, out_dists, kout);
}

}  // namespace rd
