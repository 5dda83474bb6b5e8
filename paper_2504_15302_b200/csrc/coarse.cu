// coarse.cu — N1 coarse quantization and N2 per-query nprobe selection (sm_100a).
//
// N1: Dc[b][j] = ||c_j||^2 - 2 q_b.c_j with a register-tiled FFMA GEMM
//     (64 queries x 128 centroids per CTA, 4x8 per thread, k-major smem tiles).
// N2: one CTA per query: radix-select the C = nprobe + 32 smallest approximate
//     distances, recompute those exactly (canonical fp64 sum, identical to the
//     oracle), order by (exact distance, list id) and keep nprobe. The probe set
//     is certified when every non-candidate's approximate distance, less the
//     GEMM's error bound, exceeds the nprobe-th exact distance.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <float.h>

#include "ivf_kernels.cuh"
#include "plan_device.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr int kBM = 64, kBN = 128, kBK = 16;

__global__ void __launch_bounds__(256) coarse_gemm_kernel(const float* __restrict__ Q,
                                                          const float* __restrict__ C,
                                                          const float* __restrict__ cnorm,
                                                          float* __restrict__ Dc, int B, int nlist,
                                                          int d) {
  RD_PDL_PROLOGUE();
  __shared__ __align__(16) float As[kBK][kBM + 4];
  __shared__ __align__(16) float Bs[kBK][kBN + 4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads: 4 queries x 8 centroids each
  const int qb = blockIdx.y * kBM, cb = blockIdx.x * kBN;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < d; k0 += kBK) {
    {  // A: 64 rows x 16 k = 256 float4
      const int r = tid >> 2, kq = (tid & 3) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (qb + r < B && k0 + kq < d) v = *reinterpret_cast<const float4*>(Q + (size_t)(qb + r) * d + k0 + kq);
      As[kq + 0][r] = v.x;
      As[kq + 1][r] = v.y;
      As[kq + 2][r] = v.z;
      As[kq + 3][r] = v.w;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // B: 128 rows x 16 k = 512 float4
      const int idx = tid + h * 256;
      const int r = idx >> 2, kq = (idx & 3) * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (cb + r < nlist && k0 + kq < d) v = *reinterpret_cast<const float4*>(C + (size_t)(cb + r) * d + k0 + kq);
      Bs[kq + 0][r] = v.x;
      Bs[kq + 1][r] = v.y;
      Bs[kq + 2][r] = v.z;
      Bs[kq + 3][r] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBK; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[k][tx * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[k][tx * 8 + 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = qb + ty * 4 + i;
    if (q >= B) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = cb + tx * 8 + j;
      if (c < nlist) Dc[(size_t)q * nlist + c] = __ldg(cnorm + c) - 2.f * acc[i][j];
    }
  }
}

// Small batches (B <= 8, coarse_small): Dc is a memory-bound GEMV over the centroids, so one warp
// per centroid streams its row once (float4, coalesced) against every query of the batch (through
// L1), across >= one CTA per SM — instead of the tensor-core tile kernel's 32-CTA, latency-bound K
// loop. Any summation order is covered by the select kernel's error bound ((d + 4) u 2 |q| |c|).
// Query preparation in one pass, one warp per query: ||q||^2 (fp64 lane sums and a shuffle tree;
// used only inside error-bounded approximate distances) and the bf16 (hi, lo) split rows the
// tensor-core kernels gather.
// It also zeroes the per-search counters (zero2: 2 words, zeroB: B words) so they need no memset.
__device__ __forceinline__ void qprep_rows(const QprepArgs& a, long long r0, long long rstep, bool zero2_here) {
  const int lane = threadIdx.x & 31;
  if (a.zero2 && zero2_here && threadIdx.x < 2) a.zero2[threadIdx.x] = 0u;
  constexpr int kV = 8;  // float4 per lane: d <= 1024
  const int d4 = a.d / 4;
  for (long long r = r0; r < a.B; r += rstep) {
    if (a.zeroB && lane == 0) a.zeroB[r] = 0;
    // the whole row is loaded before any use (stores to qsplit could alias it otherwise and keep
    // the loads serialised, one round trip per 32 elements)
    const float4* x = reinterpret_cast<const float4*>(a.Q + (size_t)r * a.d);
    float4 v[kV];
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      const int i = lane + 32 * k;
      v[k] = i < d4 ? __ldg(x + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      const int i = lane + 32 * k;
      if (i >= d4) break;
      const float q[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
      uint32_t hi[2], lo[2];
#pragma unroll
      for (int e = 0; e < 4; ++e) s = fma((double)q[e], (double)q[e], s);  // squares are exact in fp64
      if (a.qsplit) {
#pragma unroll
        for (int e = 0; e < 4; e += 2) {
          const __nv_bfloat162 h = __floats2bfloat162_rn(q[e], q[e + 1]);
          const __nv_bfloat162 l =
              __floats2bfloat162_rn(q[e] - __low2float(h), q[e + 1] - __high2float(h));
          hi[e / 2] = *reinterpret_cast<const uint32_t*>(&h);
          lo[e / 2] = *reinterpret_cast<const uint32_t*>(&l);
        }
        __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(a.qsplit);
        uint2* q1 = reinterpret_cast<uint2*>(qs + (size_t)(r * 2) * a.d);
        uint2* q2 = reinterpret_cast<uint2*>(qs + (size_t)(r * 2 + 1) * a.d);
        q1[i] = make_uint2(hi[0], hi[1]);
        q2[i] = make_uint2(lo[0], lo[1]);
      }
      if (a.qhalf) {  // fp16 residual scan's operand (RN; overflow to inf is caught by the scan)
        const __half2 h01 = __floats2half2_rn(q[0], q[1]), h23 = __floats2half2_rn(q[2], q[3]);
        reinterpret_cast<uint2*>(a.qhalf)[(size_t)r * (a.d / 4) + i] =
            make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) a.qnorm[r] = (float)s;
  }
}

__global__ void qprep_kernel(const QprepArgs a) {
  RD_PDL_PROLOGUE();
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  qprep_rows(a, (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5, warps, blockIdx.x == 0);
}

constexpr int kGemvThreads = 256;
constexpr int kGemvMaxV = 8;  // float4 per lane per row: d <= 1024
// one warp per centroid (grid = nlist / 8 CTAs): the row's float4 loads are all issued before any
// use; queries come through L1 (B x d x 4 <= 64 KB)
__global__ void __launch_bounds__(kGemvThreads) coarse_gemv_kernel(const float* __restrict__ Q,
                                                                   const float* __restrict__ C,
                                                                   const float* __restrict__ cnorm,
                                                                   float* __restrict__ Dc, int B, int nlist,
                                                                   int d, const QprepArgs qa) {
  RD_PDL_PROLOGUE();
  const int lane = threadIdx.x & 31;
  const int nblk = (nlist + kGemvThreads / 32 - 1) / (kGemvThreads / 32);
  if ((int)blockIdx.x >= nblk) {  // trailing CTA: the query prep (fused to save a launch)
    qprep_rows(qa, threadIdx.x >> 5, kGemvThreads / 32, true);
    return;
  }
  const int c = blockIdx.x * (kGemvThreads / 32) + (threadIdx.x >> 5);
  if (c >= nlist) return;
  const int d4 = d / 4;
  const float4* crow = reinterpret_cast<const float4*>(C + (size_t)c * d);
  float4 cv[kGemvMaxV];
#pragma unroll
  for (int k = 0; k < kGemvMaxV; ++k) {
    const int i = lane + 32 * k;
    cv[k] = i < d4 ? __ldg(crow + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float cn = __ldg(cnorm + c);
  for (int b = 0; b < B; ++b) {
    const float4* qrow = reinterpret_cast<const float4*>(Q + (size_t)b * d);
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < kGemvMaxV; ++k) {
      const int i = lane + 32 * k;
      if (i < d4) {
        const float4 qv = __ldg(qrow + i);
        acc = fmaf(qv.x, cv[k].x, fmaf(qv.y, cv[k].y, fmaf(qv.z, cv[k].z, fmaf(qv.w, cv[k].w, acc))));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) Dc[(size_t)b * nlist + c] = cn - 2.f * acc;
  }
}

__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// block-wide exclusive scan of one int per thread (NT threads, NT / 32 <= 8 warps); returns total via *total
template <int NT>
__device__ int block_excl_scan(int v, int* sh, int* total) {
  constexpr int kW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < kW ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < kW; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kW) sh[lane] = s;
  }
  __syncthreads();
  const int base = w ? sh[w - 1] : 0;
  *total = sh[kW - 1];
  __syncthreads();
  return base + x - v;
}

// small batches (staged rows, one CTA per SM): 256 threads — 1024 measured 1-2 % slower at B = 1-8
// (more threads per barrier; the phases are latency chains, not throughput)
constexpr int kSelThreadsStaged = 256;
constexpr int kSelThreads = 256;
constexpr int kSelThreadsLarge = 128;  // large batches: 7 CTAs per SM, one resident wave at B = 1024
constexpr int kSelMaxCand = 512;

// Selects the C smallest of keys[0..nlist) into cand[0..C): all keys < T plus the
// first keys == T by index (radix select, 11+11+10 bits, then an ordered compaction).
template <int NT>
__device__ uint32_t select_smallest(const uint32_t* keys, int nlist, int C, int* hist, int* scan_sh, int* cand,
                                    uint32_t* sel_prefix, uint32_t* sel_k) {
  const int tid = threadIdx.x;
  uint32_t prefix = 0, mask = 0, kk = (uint32_t)C;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
  for (int pass = 0; pass < 3; ++pass) {
    const int sh = shifts[pass], nb = 1 << widths[pass];
    for (int i = tid; i < nb; i += NT) hist[i] = 0;
    __syncthreads();
    for (int j = tid; j < nlist; j += NT) {
      const uint32_t kv = keys[j];
      if ((kv & mask) == prefix) atomicAdd(&hist[(kv >> sh) & (nb - 1)], 1);
    }
    __syncthreads();
    const int per = nb / NT;
    int local = 0;
    for (int i = 0; i < per; ++i) local += hist[tid * per + i];
    int tot;
    const int before = block_excl_scan<NT>(local, scan_sh, &tot);
    if (before < (int)kk && before + local >= (int)kk) {
      int run = before;
      for (int i = 0; i < per; ++i) {
        const int h = hist[tid * per + i];
        if (run + h >= (int)kk) {
          *sel_prefix = prefix | ((uint32_t)(tid * per + i) << sh);
          *sel_k = kk - run;
          break;
        }
        run += h;
      }
    }
    __syncthreads();
    prefix = *sel_prefix;
    kk = *sel_k;
    mask |= (uint32_t)(nb - 1) << sh;
    __syncthreads();
  }
  const uint32_t T = prefix;
  const int per = (nlist + NT - 1) / NT;
  const int j0 = tid * per, j1 = min(nlist, j0 + per);
  int nlt = 0, neq = 0;
  for (int j = j0; j < j1; ++j) {
    nlt += keys[j] < T;
    neq += keys[j] == T;
  }
  int tot_lt, tot_eq;
  int olt = block_excl_scan<NT>(nlt, scan_sh, &tot_lt);
  int oeq = block_excl_scan<NT>(neq, scan_sh, &tot_eq);
  for (int j = j0; j < j1; ++j) {
    if (keys[j] < T) {
      cand[olt++] = j;
    } else if (keys[j] == T) {
      if (oeq < (int)kk) cand[tot_lt + oeq] = j;
      ++oeq;
    }
  }
  __syncthreads();
  return T;
}

template <int NT>
__device__ __forceinline__ float block_reduce_min(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = sh[0];
  for (int i = 1; i < NT / 32; ++i) r = fminf(r, sh[i]);
  return r;
}
template <int NT>
__device__ __forceinline__ float block_reduce_max(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = sh[0];
  for (int i = 1; i < NT / 32; ++i) r = fmaxf(r, sh[i]);
  return r;
}

// dynamic smem: keys[nlist] (u32; approximate distances as floats, then exact keys in the fallback),
// q widened to fp64 [d]; kStage (small batches: one CTA per query is latency-bound) adds q as fp32
// [d] and a 32-row staging area [32][d + kStagePad] filled by bulk (TMA) row copies.
//
// Search mode (p.exact_order == 0) needs the probe SET only (the scan, the plan and the exact
// fallback are order-independent; the order only picks the seeding list). With the coarse GEMM's
// error bound eps (|approx + ||q||^2 - exact| <= eps), a candidate is
//   sure-in   if at most nprobe candidates (itself included) have approx <= its approx + 2 eps and
//             its approx + 2 eps is below every excluded centroid's approx (hi_edge),
//   sure-out  if nprobe candidates have approx < its approx - 2 eps,
//   ambiguous otherwise,
// and the excluded centroids are sure-out when nprobe candidates lie below hi_edge - 2 eps. The
// exact top-nprobe set is then the sure-in candidates plus the best ambiguous ones by (canonical
// exact distance, list id) — only those few need the fp64 sum. Exact-order mode (rd_probe) and
// uncertified queries recompute every candidate (or every centroid) exactly.
// The B = 1 plan inside the selection CTA (SelectParams::fp_tiles): the probes this CTA just wrote,
// each probed resident list cut into chunk_rows chunks (the planner's R / Rt rule), one narrow
// tensor-core tile per chunk at the block-scanned offset; list_q = query 0; counters and tile count
// as finish_counters writes them.
template <int NT>
__device__ __forceinline__ void fused_plan_b1(const SelectParams& p, int np, SmallPlanSmem& sm) {
  constexpr int PPT = (kSelMaxCand + NT - 1) / NT;
  const int tid = threadIdx.x;
  int l[PPT], len[PPT], rl[PPT], ch[PPT];
  long long g0[PPT], r0[PPT];
  int v[kTileCats] = {0, 0, 0};
  unsigned long long cc[3] = {0ull, 0ull, 0ull};
  if (tid < kTileCats) sm.carry[tid] = 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {  // thread t owns probe positions [t * PPT, (t + 1) * PPT)
    const int i = tid * PPT + k;
    l[k] = i < np ? p.probes[i] : -1;
  }
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    ch[k] = 0, len[k] = 0, rl[k] = p.fp_R, g0[k] = 0, r0[k] = -1;
    if (l[k] < 0) continue;
    g0[k] = p.list_off[l[k]];
    len[k] = (int)(p.list_off[l[k] + 1] - g0[k]);
    r0[k] = p.res_row0[l[k]];
  }
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = tid * PPT + k;
    if (l[k] < 0) continue;
    p.fp_list_q[i] = 0;
    cc[0] += 1;
    cc[r0[k] >= 0 ? 1 : 2] += (unsigned long long)len[k];
    if (r0[k] >= 0 && len[k] > 0) {
      // tiles go out in probe order, so the queue's tail is the last eighth of the probes (the
      // planner's list-id rule, tail_from, would scatter the short chunks through the queue)
      rl[k] = chunk_rows(len[k], i >= np - np / 8 ? p.fp_Rt : p.fp_R);
      ch[k] = (len[k] + rl[k] - 1) / rl[k];
      v[kCatNarrow] += ch[k];
    }
  }
  int ex[kTileCats];
  block_scan_round<NT, kTileCats>(v, ex, sm.wsum, sm.carry);
  int off = ex[kCatNarrow];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    for (int c = 0; c < ch[k]; ++c) {
      ScanTile T;
      T.src_row = r0[k] + (long long)c * rl[k];
      T.grow0 = g0[k] + (long long)c * rl[k];
      T.list = l[k];
      T.nrows = min(rl[k], len[k] - c * rl[k]);
      T.qoff = tid * PPT + k;
      T.nq = 1;
      p.fp_tiles[off + c] = T;
    }
    off += ch[k];
  }
  PlanParams fp{};
  fp.counters = p.fp_counters;
  fp.meta = p.fp_meta;
  finish_counters<NT>(fp, cc, sm.wcnt, sm.carry);
}

template <bool kStage, int NT>
__global__ void __launch_bounds__(NT) coarse_select_kernel(const SelectParams p) {
  RD_TS(13);  // entry, before the wait on the previous kernel
  RD_PDL_PROLOGUE();
  extern __shared__ __align__(16) uint32_t keys[];
  __shared__ __align__(16) int hist[2048];  // (and the B = 1 fused plan's scratch)
  __shared__ int scan_sh[32];
  __shared__ float fsh[32];
  __shared__ int cand[kSelMaxCand];
  __shared__ float cdist[kSelMaxCand];
  __shared__ uint32_t sel_prefix, sel_k;
  __shared__ int certified, ncand_s, found_bin, below_s, nin_s, na_s, lsel;
  __shared__ unsigned char lok[kSelMaxCand];  // candidate list can seed (resident, >= seed_rows rows)
  __shared__ unsigned long long amin;
  __shared__ __align__(8) uint64_t bar;
  RD_TS(0);
  const int b = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nlist = p.nlist, d = p.d;
  const float* q = p.queries + (size_t)b * d;
  const int grp = tid >> 3, j8 = tid & 7;
  const int np = min(p.nprobe, nlist);
  const float* drow = p.Dc + (size_t)b * nlist;
  float* vals = reinterpret_cast<float*>(keys);
  double* qd = reinterpret_cast<double*>(vals + ((nlist + 3) & ~3));
  float* qf = reinterpret_cast<float*>(qd + d);  // kStage
  float* st = qf + d;                            // kStage: [32][d + kStagePad]
  const int ds = d + (p.x12 ? d / 2 : 0) + kStagePad;  // staged row stride: fp32 row or split3 x12 + x3
  uint32_t bphase = 0;
  if (tid == 0) {
    amin = ~0ull;
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  float qv[1024 / NT];  // d <= 1024; stored after the distance row's loads are in flight
#pragma unroll
  for (int k = 0; k < 1024 / NT; ++k) qv[k] = tid + k * NT < d ? q[tid + k * NT] : 0.f;
  const float qn = p.qnorm[b];
  // bulk-copies rows r < nrows (row_ptr(r), device memory) into st; every thread waits
  auto stage_bulk = [&](int nrows, auto row_ptr) {
    if (warp == 0) {
      if (lane == 0) mbar_arrive_expect_tx(&bar, (uint32_t)(nrows * d * 4));
      __syncwarp();
      if (lane < nrows) bulk_g2s(st + lane * ds, row_ptr(lane), (uint32_t)(d * 4), &bar);
    }
    mbar_wait(&bar, bphase);
    bphase ^= 1;
  };
  // resident-store row sr (seeding) into staging slot i: one fp32 row, or a split3 row's x12 and x3
  auto stage_seed_row = [&](int i, long long sr) {
    if (p.x12) {
      bulk_g2s(st + i * ds, p.x12 + (size_t)sr * 2 * d, (uint32_t)(d * 4), &bar);
      bulk_g2s(st + i * ds + d, p.x3 + (size_t)sr * d, (uint32_t)(d * 2), &bar);
    } else {
      bulk_g2s(st + i * ds, p.arena + (size_t)sr * d, (uint32_t)(d * 4), &bar);
    }
  };
  // a staged seeding row as a RowRef (32 staging slots: groups beyond them read slot 31, masked)
  auto staged_ref = [&](int i) {
    const float* slot = st + min(i, 31) * ds;
    return p.x12 ? RowRef{nullptr, reinterpret_cast<const __nv_bfloat16*>(slot),
                          reinterpret_cast<const __nv_bfloat16*>(slot + d)}
                 : row_f32(slot);
  };

  float vmin = __builtin_huge_valf(), vmax = -__builtin_huge_valf();
  int jmin = 0;
  constexpr int kVB = 16;  // row loads in flight per thread
  for (int j0 = tid; j0 < nlist; j0 += kVB * NT) {
    float v[kVB];
#pragma unroll
    for (int k = 0; k < kVB; ++k) {
      const int j = j0 + k * NT;
      v[k] = j < nlist ? drow[j] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kVB; ++k) {
      const int j = j0 + k * NT;
      if (j < nlist) {
        vals[j] = v[k];
        if (v[k] < vmin) jmin = j;
        vmin = fminf(vmin, v[k]);
        vmax = fmaxf(vmax, v[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 1024 / NT; ++k)
    if (tid + k * NT < d) {
      if constexpr (kStage) {  // (large batches read q straight from global memory)
        qd[tid + k * NT] = (double)qv[k];
        qf[tid + k * NT] = qv[k];
      }
    }
  if constexpr (kStage) {  // approximate nearest centroid: warm L2 with its list's first 32 rows (the likely seed)
    __syncthreads();
    // one shared atomic per warp (a 64-bit atomicMin from every thread serialises for microseconds)
    unsigned long long key = vmin < __builtin_huge_valf() ? ((unsigned long long)f2key(vmin) << 32) | (unsigned)jmin
                                                          : ~0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
    if (lane == 0 && key != ~0ull) atomicMin(&amin, key);
  }
  vmin = block_reduce_min<NT>(vmin, fsh);
  vmax = block_reduce_max<NT>(vmax, fsh);
  // kStage: the approximately nearest list's first 32 rows (the likely seeding list) are bulk-copied
  // into the staging area now and consumed after the candidate search, off the critical path
  int seed_l = -1;  // uniform: every thread reads the same amin and list metadata
  if constexpr (kStage) {
    if (p.qthr && amin != ~0ull) {
      const int l = (int)(amin & 0xffffffffu);
      const long long r0 = p.res_row0[l];
      if (r0 >= 0 && p.list_off[l + 1] - p.list_off[l] >= p.seed_rows) {
        seed_l = l;
        if (warp == 0) {
          if (lane == 0) mbar_arrive_expect_tx(&bar, (uint32_t)(p.seed_rows * d * (p.x12 ? 6 : 4)));
          __syncwarp();
          if (lane < p.seed_rows) stage_seed_row(lane, r0 + lane);
        }
      }
    }
  }
  RD_TS(1);
  const int Cwant = min(nlist, p.nprobe + kCoarseExtra);

  // candidate set {approx < hi_edge} of size in [C, kSelMaxCand], found with value-linear 2048-bin
  // histograms (refined inside the crossing bin when it is too dense)
  int ncand = -1;
  float hi_edge = __builtin_huge_valf();
  if (Cwant == nlist && nlist <= kSelMaxCand) {
    ncand = nlist;  // every centroid is a candidate: nothing excluded
  } else if (Cwant < nlist && vmax > vmin) {
    float lo = vmin, hi = vmax;
    int below = 0;
    for (int round = 0; round < 3 && ncand < 0; ++round) {
      const float width = (hi - lo) / 2048.f;
      if (!(width > 0.f)) break;
      for (int i = tid; i < 2048; i += NT) hist[i] = 0;
      __syncthreads();
      for (int j = tid; j < nlist; j += NT) {
        const float v = vals[j];
        if (v >= lo && v < hi) atomicAdd(&hist[min(2047, (int)((v - lo) / width))], 1);
      }
      __syncthreads();
      int local = 0;
      constexpr int kPer = 2048 / NT;  // bins per thread
      for (int i = 0; i < kPer; ++i) local += hist[tid * kPer + i];
      int tot;
      const int before = block_excl_scan<NT>(local, scan_sh, &tot);
      if (tid == 0) found_bin = 2047;
      __syncthreads();
      if (below + before < Cwant && below + before + local >= Cwant) {
        int run = below + before;
        for (int i = 0; i < kPer; ++i) {
          run += hist[tid * kPer + i];
          if (run >= Cwant) {
            found_bin = tid * kPer + i;
            break;
          }
        }
      }
      __syncthreads();
      const int fb = found_bin;
      const float edge_hi = (fb == 2047) ? hi : lo + (fb + 1) * width;
      const float edge_lo = lo + fb * width;
      // exact recount of {v < edge_hi}
      int c = 0;
      for (int j = tid; j < nlist; j += NT) c += vals[j] < edge_hi;
      int total;
      block_excl_scan<NT>(c, scan_sh, &total);
      if (total >= Cwant && total <= kSelMaxCand) {
        ncand = total;
        hi_edge = edge_hi;
      } else {
        int cb = 0;
        for (int j = tid; j < nlist; j += NT) cb += vals[j] < edge_lo;
        int tb;
        block_excl_scan<NT>(cb, scan_sh, &tb);
        below = tb;
        lo = edge_lo;
        hi = edge_hi;
      }
    }
  }
  RD_TS(2);
  if (ncand >= 0) {
    if (tid == 0) ncand_s = 0;
    __syncthreads();
    for (int j0 = 0; j0 < nlist; j0 += NT) {  // warp-aggregated appends (order is irrelevant: ranked below)
      const int j = j0 + tid;
      const bool in = j < nlist && vals[j] < hi_edge;
      const unsigned m = __ballot_sync(0xffffffffu, in);
      int base = 0;
      if (lane == 0 && m) base = atomicAdd(&ncand_s, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (in) cand[base + __popc(m & ((1u << lane) - 1u))] = j;
    }
    __syncthreads();
  }
  RD_TS(3);
  if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0) p.dbg[15] = (unsigned long long)ncand;
  float seed_pre = 0.f;  // max fp32 distance to the early-staged rows (valid when seed_l >= 0)
  if constexpr (kStage) {
    if (seed_l >= 0) {
      mbar_wait(&bar, bphase);
      bphase ^= 1;
      const float e = d % 64 == 0 ? l2_group8_f32_chunks(qf, staged_ref(grp), d, j8)  // rows >= seed_rows: stale, masked
                                    : l2_group8_f32_row(qf, staged_ref(grp), d, j8);
      seed_pre = block_reduce_max<NT>(grp < p.seed_rows ? e : 0.f, fsh);
      __syncthreads();  // the staging area is free again
    }
  }
  RD_TS(4);

  const float u = kUnit;
  // |approx - exact| of a coarse distance: the GEMM's dot bound (doubled: d = ... - 2 q.c) plus the
  // norms' and the epilogue's roundings
  const float eps = 2.f * p.gamma_coarse * sqrtf(qn) * p.cmax + 16.f * u * (qn + p.cmax * p.cmax) + 1e-30f;
  bool done = false;

  // ------------------------------------------------------------ search mode: the probe set
  if (!p.exact_order && ncand >= 0) {
    const int C = ncand;
    const float e2 = 2.f * eps;
    int* state = hist;           // [512] 0 out, 1 in (sure or chosen), 2 ambiguous
    int* byrank = hist + 512;    // [512] candidate index by approximate rank
    int* ambl = hist + 1024;     // [512] ambiguous candidates in approximate-rank order
    float* adist = reinterpret_cast<float*>(hist + 1536);  // [512] their exact distances
    for (int i = tid; i < C; i += NT) {
      const int l = cand[i];
      cdist[i] = vals[l];
      // seeding eligibility, resolved here so the rank-order walk below needs no global loads
      if (p.qthr) lok[i] = p.res_row0[l] >= 0 && p.list_off[l + 1] - p.list_off[l] >= p.seed_rows;
    }
    if (tid == 0) below_s = 0;
    __syncthreads();
    RD_TS(10);
    // rank and window counts: one group of 8 lanes per candidate, lane j8 scans k = j8 (mod 8)
    int below = 0;
    for (int i0 = 0; i0 < C; i0 += NT / 8) {
      const int i = i0 + grp;
      const float vi = i < C ? cdist[i] : 0.f;
      const int ci = i < C ? cand[i] : 0;
      int r = 0, lt = 0, lo = 0;
      if (i < C)
#pragma unroll 4
        for (int k = j8; k < C; k += 8) {
          const float vk = cdist[k];
          r += vk < vi || (vk == vi && cand[k] < ci);
          lt += vk <= vi + e2;
          lo += vk < vi - e2;
        }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        r += __shfl_xor_sync(0xffffffffu, r, o);
        lt += __shfl_xor_sync(0xffffffffu, lt, o);
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
      }
      if (i < C && j8 == 0) {
        byrank[r] = i;
        state[i] = lo >= np ? 0 : (lt <= np && vi + e2 < hi_edge) ? 1 : 2;
        below += vi < hi_edge - e2;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
    if (lane == 0 && below) atomicAdd(&below_s, below);
    __syncthreads();
    RD_TS(7);
    if (warp == 0) {  // ambiguous list in rank order; sure-in count
      int nin = 0, na = 0;
      for (int r0 = 0; r0 < C; r0 += 32) {
        const int r = r0 + lane;
        const int stt = r < C ? state[byrank[r]] : 0;
        const unsigned mi = __ballot_sync(0xffffffffu, stt == 1), ma = __ballot_sync(0xffffffffu, stt == 2);
        if (stt == 2) ambl[na + __popc(ma & ((1u << lane) - 1u))] = byrank[r];
        nin += __popc(mi);
        na += __popc(ma);
      }
      if (lane == 0) {
        nin_s = nin;
        na_s = na;
      }
    }
    __syncthreads();
    RD_TS(8);
    const int nin = nin_s, na = na_s, need = np - nin;
    if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0) p.dbg[14] = (unsigned long long)na;
    if (below_s >= np && need >= 0 && need <= na) {
      if (need > 0 && need < na) {  // the best `need` ambiguous candidates by exact (distance, list id)
        constexpr int kAmb = kStage ? (NT / 8 < 32 ? NT / 8 : 32) : NT / 8;  // (32 staging slots)
        for (int a0 = 0; a0 < na; a0 += kAmb) {
          const int rows = min(kAmb, na - a0);
          const int a = a0 + grp;
          float e;
          if constexpr (kStage) {
            stage_bulk(rows, [&](int r) { return p.centroids + (size_t)cand[ambl[a0 + r]] * d; });
            e = exact_l2_group8_qd(qd, st + min(grp, 31) * ds, grp < rows ? d : 0, j8);
            __syncthreads();  // the staging area is reused by the next chunk
          } else {
            e = exact_l2_group8_impl<true, 16>(q, p.centroids + (size_t)cand[ambl[a < na ? a : na - 1]] * d, d, j8);
          }
          if (grp < rows && j8 == 0) adist[a] = e;
        }
        __syncthreads();
        for (int a = tid; a < na; a += NT) {
          const float da = adist[a];
          const int ia = cand[ambl[a]];
          int r = 0;
          for (int k = 0; k < na; ++k) {
            const float dk = adist[k];
            r += dk < da || (dk == da && cand[ambl[k]] < ia);
          }
          state[ambl[a]] = r < need ? 1 : 0;
        }
      } else {
        for (int a = tid; a < na; a += NT) state[ambl[a]] = need == na ? 1 : 0;
      }
      __syncthreads();
      RD_TS(9);
      if (warp == 0) {  // probes in approximate-rank order; seeding list = first resident one with >= 32 rows
        int n = 0, ls = -1;
        for (int r0 = 0; r0 < C; r0 += 32) {
          const int r = r0 + lane;
          const int i = r < C ? byrank[r] : 0;
          const bool in = r < C && state[i] == 1;
          const unsigned m = __ballot_sync(0xffffffffu, in);
          if (in) {
            const int l = cand[i];
            p.probes[(size_t)b * p.nprobe + n + __popc(m & ((1u << lane) - 1u))] = l;
            if (p.bitmap) atomicOr(p.bitmap + (size_t)l * p.W + (b >> 5), 1u << (b & 31));
            if (p.qthr) {
              const unsigned mo = __ballot_sync(m, lok[i] != 0);
              if (ls < 0 && mo) ls = __shfl_sync(m, l, __ffs(mo) - 1);
            }
          }
          ls = __shfl_sync(0xffffffffu, ls, __ffs(m ? m : 1u) - 1);
          n += __popc(m);
        }
        for (int i = np + lane; i < p.nprobe; i += 32) p.probes[(size_t)b * p.nprobe + i] = -1;
        if (lane == 0) lsel = ls;
      }
      done = true;
    } else if (tid == 0) {
      atomicAdd(p.probe_fail, 1u);
    }
    __syncthreads();
  }

  // ------------------------------------------------------------ exact order (rd_probe) / fallback
  if (!done) {
    for (int attempt = (ncand >= 0 && p.exact_order ? 0 : 1); attempt < 2; ++attempt) {
      int C;
      if (attempt == 0) {
        C = ncand;
      } else {
        // exact keys for every centroid, then the np smallest by (exact distance, list id)
        for (int c0 = 0; c0 < nlist; c0 += NT / 8) {
          const int c = c0 + grp;
          const int cc = c < nlist ? c : nlist - 1;
          const float e = kStage ? exact_l2_group8_qd(qd, p.centroids + (size_t)cc * d, d, j8)
                                 : exact_l2_group8_impl<true, 16>(q, p.centroids + (size_t)cc * d, d, j8);
          __syncthreads();
          if (c < nlist && j8 == 0) keys[c] = f2key(e);
        }
        __syncthreads();
        C = np;
        select_smallest<NT>(keys, nlist, C, hist, scan_sh, cand, &sel_prefix, &sel_k);
      }
      for (int c0 = 0; c0 < C; c0 += NT / 8) {
        const int c = c0 + grp;
        const int cc = c < C ? c : C - 1;
        const float e = kStage ? exact_l2_group8_qd(qd, p.centroids + (size_t)cand[cc] * d, d, j8)
                               : exact_l2_group8_impl<true, 16>(q, p.centroids + (size_t)cand[cc] * d, d, j8);
        if (c < C && j8 == 0) cdist[c] = e;
      }
      // rank sort by (exact distance, list id): keys are distinct (list ids)
      __syncthreads();
      {
        float* rd_ = reinterpret_cast<float*>(hist);  // hist is free here: [0, 512) dists, [512, 1024) ids
        int* rc_ = hist + kSelMaxCand;
        for (int i = tid; i < C; i += NT) {
          const float di = cdist[i];
          const int ii = cand[i];
          int r = 0;
          for (int jx = 0; jx < C; ++jx) {
            const float dj = cdist[jx];
            r += dj < di || (dj == di && cand[jx] < ii);
          }
          rd_[r] = di;
          rc_[r] = ii;
        }
        __syncthreads();
        for (int i = tid; i < C; i += NT) {
          cdist[i] = rd_[i];
          cand[i] = rc_[i];
        }
        __syncthreads();
      }
      if (tid == 0) {
        int ok = 1;
        if (attempt == 0) {
          // every excluded centroid has approx >= hi_edge; the GEMM's error bound turns that into
          // a lower bound on its exact distance
          ok = hi_edge + qn - eps > cdist[np - 1];
        }
        certified = ok;
        if (!ok) atomicAdd(p.probe_fail, 1u);
      }
      __syncthreads();
      if (certified) break;
    }
    for (int i = tid; i < p.nprobe; i += NT) {
      p.probes[(size_t)b * p.nprobe + i] = i < np ? cand[i] : -1;
      if (p.bitmap && i < np) atomicOr(p.bitmap + (size_t)cand[i] * p.W + (b >> 5), 1u << (b & 31));
    }
    if (p.qthr && tid == 0) {
      lsel = -1;
      for (int i = 0; i < np; ++i) {
        const int l = cand[i];
        if (p.res_row0[l] >= 0 && p.list_off[l + 1] - p.list_off[l] >= p.seed_rows) {
          lsel = l;
          break;
        }
      }
    }
    __syncthreads();
  }
  RD_TS(5);
  if (kStage && p.fp_tiles) {  // B = 1: plan the scan here (the probes are written)
    static_assert(sizeof(SmallPlanSmem) <= sizeof(hist), "fused plan scratch");
    __syncthreads();
    fused_plan_b1<NT>(p, np, *reinterpret_cast<SmallPlanSmem*>(hist));
    __syncthreads();
  }

  // fused seed: fp32 distances to the first 32 rows of the seeding list; threshold = max * (1 + rel
  // bound) + 2 eps_scan, a valid upper bound on the final 32nd-best approximate distance, so the
  // scan's certification holds (merge.cu)
  if (p.qthr) {
    __shared__ float red[NT / 32];
    const int l = lsel;
    if (l < 0) {
      if (tid == 0) p.qthr[b] = 0x7f7f7f7f;
    } else {
      const long long sr0 = p.res_row0[l];  // the list's first row in the resident store
      float e = 0.f;
      const bool pre = kStage && l == seed_l;  // computed early (uniform branch)
      if (!pre) {
        if constexpr (kStage) {
          if (warp == 0) {
            if (lane == 0) mbar_arrive_expect_tx(&bar, (uint32_t)(p.seed_rows * d * (p.x12 ? 6 : 4)));
            __syncwarp();
            if (lane < p.seed_rows) stage_seed_row(lane, sr0 + lane);
          }
          mbar_wait(&bar, bphase);
          bphase ^= 1;
          e = d % 64 == 0 ? l2_group8_f32_chunks(qf, staged_ref(grp), d, j8) : l2_group8_f32_row(qf, staged_ref(grp), d, j8);
          if (grp >= p.seed_rows) e = 0.f;  // only the first seed_rows rows bound the threshold
        } else {  // NT / 8 rows per pass (a uniform trip count keeps the group shuffles converged)
          for (int rb = 0; rb < p.seed_rows; rb += NT / 8) {
            const int r = rb + grp;
            const long long sr = sr0 + min(r, p.seed_rows - 1);
            const RowRef x = p.x12 ? row_split3(p.x12, p.x3, sr, d) : row_f32(p.arena + (size_t)sr * d);
            const float v = d % 64 == 0 ? l2_group8_f32_chunks(q, x, d, j8) : l2_group8_f32_row<16>(q, x, d, j8);
            if (r < p.seed_rows) e = fmaxf(e, v);
          }
        }
      }
      float m = e;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[warp] = m;
      __syncthreads();
      if (tid == 0) {
        float mx = red[0];
        for (int i = 1; i < NT / 32; ++i) mx = fmaxf(mx, red[i]);
        if (pre) mx = seed_pre;
        const float eps_s = 2.f * p.gamma_scan * sqrtf(qn) * p.xmax + 16.f * u * (qn + p.xmax * p.xmax) + 1e-30f;
        const float thr = mx * (1.f + 2.f * l2_f32_rel_bound(d)) + 2.f * eps_s;
        p.qthr[b] = f2ord(thr);
      }
    }
  }
  RD_TS(6);
  RD_TS_END();
}

}  // namespace

cudaError_t launch_coarse(const float* Q, const float* C, const float* cnorm, float* Dc, int B,
                          int nlist, int d, cudaStream_t s) {
  dim3 grid((nlist + kBN - 1) / kBN, (B + kBM - 1) / kBM);
  return launch_k(coarse_gemm_kernel, grid, dim3(256), 0, s, Q, C, cnorm, Dc, B, nlist, d);
}

bool coarse_small(int B) { return B <= 8; }  // measured cut-over vs the tensor-core tile kernel

cudaError_t launch_coarse_small(const float* Q, const float* C, const float* cnorm, float* Dc, int B, int nlist,
                                int d, const QprepArgs& qa, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  if (d > 4 * 32 * kGemvMaxV) return cudaErrorInvalidValue;
  const int nblk = (nlist + kGemvThreads / 32 - 1) / (kGemvThreads / 32);
  return launch_k(coarse_gemv_kernel, dim3(nblk + 1), dim3(kGemvThreads), 0, s, Q, C, cnorm, Dc, B, nlist, d, qa);
}

cudaError_t launch_qprep(const QprepArgs& a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  const long long blocks = (a.B * 32 + 255) / 256;
  return launch_k(qprep_kernel, dim3((unsigned)(blocks < 148 * 8 ? blocks : 148 * 8)), dim3(256), 0, s, a);
}

namespace {
size_t select_staged_bytes(const SelectParams& p) {
  const size_t keys = sizeof(uint32_t) * (size_t)((p.nlist + 3) & ~3);
  const size_t qd = sizeof(double) * (size_t)p.d;
  const size_t ds = (size_t)p.d + (p.x12 ? p.d / 2 : 0) + kStagePad;  // the kernel's staged row stride
  return keys + qd + sizeof(float) * ((size_t)p.d + 32 * ds);
}
}  // namespace

bool select_staged(const SelectParams& p, bool stage) { return stage && select_staged_bytes(p) <= 200 * 1024; }

cudaError_t launch_select(const SelectParams& p, bool stage, cudaStream_t s, int num_sms) {
  if (p.nprobe + kCoarseExtra > kSelMaxCand) return cudaErrorInvalidValue;
  const size_t keys = sizeof(uint32_t) * (size_t)((p.nlist + 3) & ~3);
  const size_t staged = select_staged_bytes(p);
  if (p.fp_tiles && !select_staged(p, stage)) return cudaErrorInvalidValue;  // the fused plan is staged-only
  if (select_staged(p, stage))
    return launch_k(coarse_select_kernel<true, kSelThreadsStaged>, dim3(p.B), dim3(kSelThreadsStaged), staged, s, p);
  // large batches (enough CTAs to hide latency) or very large nlist: the direct-load variant. Past
  // one resident wave of 256-thread CTAs (64 registers and ~35 KiB each: 4 per SM), 128 threads
  // and no smem copy of q fit 7 per SM (1024 queries in one wave: 65 -> 55 us on B200)
  if (p.B > 4LL * num_sms)
    return launch_k(coarse_select_kernel<false, kSelThreadsLarge>, dim3(p.B), dim3(kSelThreadsLarge), keys, s, p);
  return launch_k(coarse_select_kernel<false, kSelThreads>, dim3(p.B), dim3(kSelThreads), keys, s, p);
}

}  // namespace rd
