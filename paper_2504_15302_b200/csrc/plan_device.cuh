// plan_device.cuh — device-side pieces of the N3 planner (plan.cu): query groups, tile emission,
// block scans, counters, and the sorted-pairs plan of tiny batches for any CTA width.
#pragma once
#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

// Query groups per chunk of one list, by category. A list probed by >= tc_min_q queries goes to
// the tensor cores: in mixed mode (tc_mode 0) a list of <= 16 queries is one narrow group and a
// larger one balanced wide groups of <= 32 (usually one, so the list's bytes are read once);
// tc_mode 16 / 32 forces one width. Sparser lists form FFMA groups of <= kScanG.
struct Groups {
  int g[kTileCats];
};
__device__ __forceinline__ Groups group_split(int nq, const PlanParams& p) {
  Groups G = {{0, 0, 0}};
  if (nq >= p.tc_min_q) {
    if (p.tc_mode == 16 || (p.tc_mode == 0 && nq <= 16))
      G.g[kCatNarrow] = (nq + 15) / 16;
    else
      G.g[kCatWide] = (nq + 31) / 32;
  } else {
    G.g[kCatFfma] = (nq + kScanG - 1) / kScanG;
  }
  return G;
}

// The tiles of one list: per category, chunk-major and group-minor in that category's array;
// groups outer so each group's query split is computed once; chunks c = c0, c0 + cstep, ...
// (lanes of a warp, or one thread). toff: the list's first tile in each category's array.
__device__ __forceinline__ void emit_tiles(const PlanParams& p, int j, int nq, int qoff, int len, long long src0,
                                           long long g0, const int (&toff)[kTileCats], const Groups& G, int chunks,
                                           int rl, int c0, int cstep) {
#pragma unroll
  for (int cat = 0; cat < kTileCats; ++cat) {
    const int ng = G.g[cat];
    for (int g = 0; g < ng; ++g) {
      int tq0, tnq;
      if (cat != kCatFfma) {  // balanced tensor-core groups
        const bool s32 = nq < 46341;  // g * nq < 2^31 for g <= nq / 16 + 1
        const int q0 = s32 ? g * nq / ng : (int)((long long)g * nq / ng);
        const int q1 = s32 ? (g + 1) * nq / ng : (int)((long long)(g + 1) * nq / ng);
        tq0 = qoff + q0;
        tnq = q1 - q0;
      } else {
        tq0 = qoff + g * kScanG;
        tnq = min(kScanG, nq - g * kScanG);
      }
      ScanTile* dst = p.tiles[cat] + toff[cat] + g;
      for (int c = c0; c < chunks; c += cstep) {
        ScanTile T;
        T.src_row = src0 + (long long)c * rl;
        T.grow0 = g0 + (long long)c * rl;
        T.list = j;
        T.nrows = min(rl, len - c * rl);
        T.qoff = tq0;
        T.nq = tnq;
        dst[c * ng] = T;
      }
    }
  }
}

// Block exclusive scan of kV ints per thread (kNT threads), offset by carry[] (running totals of
// earlier rounds, updated here); wsum is [kV][32] scratch.
template <int kNT, int kV>
__device__ __forceinline__ void block_scan_round(const int (&v)[kV], int (&ex)[kV], int (*wsum)[32], int* carry) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc[kV];
#pragma unroll
  for (int i = 0; i < kV; ++i) inc[i] = v[i];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int y = __shfl_up_sync(0xffffffffu, inc[i], o);
      if (lane >= o) inc[i] += y;
    }
  if (lane == 31)
#pragma unroll
    for (int i = 0; i < kV; ++i) wsum[i][w] = inc[i];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      int a = lane < kNT / 32 ? wsum[i][lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, a, o);
        if (lane >= o) a += y;
      }
      wsum[i][lane] = a;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kV; ++i) ex[i] = carry[i] + (w ? wsum[i][w - 1] : 0) + inc[i] - v[i];
  __syncthreads();  // everyone has read carry
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < kV; ++i) carry[i] += wsum[i][kNT / 32 - 1];
  __syncthreads();
}

// block reduction of the byte counters; cat_total[cat] = tiles of each category -> counters / meta
template <int kNT>
__device__ __forceinline__ void finish_counters(const PlanParams& p, unsigned long long (&cc)[3],
                                                unsigned long long (*wcnt)[32], const int* cat_total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) cc[i] += __shfl_xor_sync(0xffffffffu, cc[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 3; ++i) wcnt[i][w] = cc[i];
  __syncthreads();
  if (w == 0) {
    unsigned long long c[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) c[i] = lane < kNT / 32 ? wcnt[i][lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) c[i] += __shfl_xor_sync(0xffffffffu, c[i], o);
    if (lane == 0) {
      for (int i = 0; i < 3; ++i) p.counters[i] = c[i];
      for (int cat = 0; cat < kTileCats; ++cat) {
        p.meta[2 * cat] = cat_total[cat];
        p.meta[2 * cat + 1] = 0;
      }
    }
  }
}

constexpr int kSmallPlanPairs = 512;  // plan_small_ok: B * nprobe <= 512

struct SmallPlanSmem {
  unsigned long long key[kSmallPlanPairs];
  int wsum[kTileCats][32];
  int carry[kTileCats];
  unsigned long long wcnt[3][32];
};

// Tiny batches (B * nprobe <= 512 pairs): plan from the probe pairs alone, in one CTA of NT threads.
// The (list, query) pairs are rank-sorted; a list's segment in sorted order IS its query CSR (list_q
// = the sorted query ids, ascending within a list), so the only passes are O(pairs) plus one
// coalesced zeroing of list_nq. Same outputs as the bitmap planners for every list. Thread t owns
// sorted positions [t * PPT, (t + 1) * PPT).
template <int NT>
__device__ __forceinline__ void plan_small_body(const PlanParams& p, SmallPlanSmem& sm) {
  constexpr int PPT = (kSmallPlanPairs + NT - 1) / NT;
  const int tid = threadIdx.x;
  const int P = p.B * p.nprobe;
  // (list, query) keys; padding / invalid probes sort last
  unsigned long long kv[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int i = tid + k * NT;
    kv[k] = ~0ull;
    if (i < P) {
      const int l = p.probes[i];
      if (l >= 0) kv[k] = ((unsigned long long)(unsigned)l << 32) | (unsigned)(i / p.nprobe);
    }
    if (i < kSmallPlanPairs) sm.key[i] = kv[k];
  }
  if (tid < kTileCats) sm.carry[tid] = 0;
  for (int j = tid; j < p.nlist; j += NT) p.list_nq[j] = 0;  // coalesced
  __syncthreads();
  int r[PPT];  // ranks of this thread's keys (valid keys are distinct)
#pragma unroll
  for (int k = 0; k < PPT; ++k) r[k] = 0;
  for (int i = 0; i < P; ++i) {
    const unsigned long long o = sm.key[i];
#pragma unroll
    for (int k = 0; k < PPT; ++k) r[k] += o < kv[k];
  }
  __syncthreads();
  int nv = 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k)
    if (kv[k] != ~0ull) {
      sm.key[r[k]] = kv[k];
      ++nv;
    }
  int valid = 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) valid += __syncthreads_count(nv > k);
  // segment starts in sorted order; per owned position: list, query count, chunking, groups
  int v[kTileCats] = {0, 0, 0};
  unsigned long long cc[3] = {0ull, 0ull, 0ull};
  int nqk[PPT], chk[PPT], lenk[PPT], rlk[PPT];
  long long src0k[PPT], g0k[PPT];
  Groups Gk[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int s = tid * PPT + k;
    const unsigned long long mine = s < valid ? sm.key[s] : ~0ull;
    const int l = (int)(mine >> 32);
    const bool start = s < valid && (s == 0 || (sm.key[s - 1] >> 32) != (mine >> 32));
    nqk[k] = 0, chk[k] = 0, lenk[k] = 0, rlk[k] = p.R, src0k[k] = -1, g0k[k] = 0;
    Gk[k] = Groups{{0, 0, 0}};
    if (s < valid) p.list_q[s] = (int)(mine & 0xffffffffu);
    if (!start) continue;
    int e = s + 1;
    while (e < valid && (sm.key[e] >> 32) == (mine >> 32)) ++e;
    nqk[k] = e - s;
    g0k[k] = p.list_off[l];
    lenk[k] = (int)(p.list_off[l + 1] - g0k[k]);
    src0k[k] = p.res_row0[l];
    if (src0k[k] >= 0 && lenk[k] > 0) {
      rlk[k] = chunk_rows(lenk[k], l >= p.tail_from ? p.Rt : p.R);
      chk[k] = (lenk[k] + rlk[k] - 1) / rlk[k];
      Gk[k] = group_split(nqk[k], p);
    }
    cc[0] += 1;
    cc[src0k[k] >= 0 ? 1 : 2] += (unsigned long long)lenk[k];
#pragma unroll
    for (int cat = 0; cat < kTileCats; ++cat) v[cat] += Gk[k].g[cat] * chk[k];
  }
  // block scan of the per-thread tile counts (the query offset is the sorted position itself)
  int ex[kTileCats];
  block_scan_round<NT, kTileCats>(v, ex, sm.wsum, sm.carry);
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    if (!nqk[k]) continue;
    const int s = tid * PPT + k;
    const int l = (int)(sm.key[s] >> 32);
    p.list_nq[l] = nqk[k];
    p.list_qoff[l] = s;
    int any = 0;
#pragma unroll
    for (int cat = 0; cat < kTileCats; ++cat) any += Gk[k].g[cat];
    if (any > 0) emit_tiles(p, l, nqk[k], s, lenk[k], src0k[k], g0k[k], ex, Gk[k], chk[k], rlk[k], 0, 1);
#pragma unroll
    for (int cat = 0; cat < kTileCats; ++cat) ex[cat] += Gk[k].g[cat] * chk[k];
  }
  finish_counters<NT>(p, cc, sm.wcnt, sm.carry);
}

}  // namespace rd
