// plan.cu — N3 probe inversion and scan work planning (sm_100a).
//
// The B x nprobe probe table is inverted into per-list query groups (queries within a list in
// ascending id, deterministically), then every probed, HBM-resident list is cut into scan tiles of
// <= R rows x one query group. Tiles fall in three categories, each with its own array and kernel:
//   kCatNarrow  tensor-core tiles of <= 16 queries (the 16-wide scan: deeper x ring)
//   kCatWide    tensor-core tiles of <= 32 queries (the 32-wide scan)
//   kCatFfma    FFMA tiles of <= kScanG queries (d % 64 != 0, d > 896, or RD_TC_MIN_Q)
// Tiles of one list are adjacent so the query groups of a chunk hit L2 for each other. Offloaded
// lists get no device tiles here; the host plans them as their bytes are staged (search.cu).
#include "ivf_kernels.cuh"
#include "plan_device.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

// warp per list: query count and resident tile counts per category (the bitmap was filled by the
// selection kernel, coarse.cu)
__global__ void list_count_kernel(const PlanParams p) {
  RD_PDL_PROLOGUE();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p.nlist) return;
  const unsigned* row = p.bitmap + (size_t)warp * p.W;
  int c = 0;
  for (int w = lane; w < p.W; w += 32) c += __popc(row[w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) {
    p.list_nq[warp] = c;
    const long long len = p.list_off[warp + 1] - p.list_off[warp];
    Groups G = {{0, 0, 0}};
    int chunks = 0;
    if (c > 0 && len > 0 && p.res_row0[warp] >= 0) {
      const int rl = chunk_rows(len, warp >= p.tail_from ? p.Rt : p.R);
      chunks = ((int)len + rl - 1) / rl;  // 32-bit: rows per list < 2^31
      G = group_split(c, p);
    }
#pragma unroll
    for (int cat = 0; cat < kTileCats; ++cat) p.list_ntile[cat * p.nlist + warp] = G.g[cat] * chunks;
  }
}

// single CTA: exclusive scans of list_nq and the tile counts; totals and byte counters. Each
// thread takes kLV consecutive lists per round (every load of the round in flight at once, then
// one block scan of the per-thread sums): one round covers 4096 lists.
constexpr int kLV = 4;
__global__ void __launch_bounds__(1024) list_scan_kernel(const PlanParams p) {
  RD_PDL_PROLOGUE();
  __shared__ int wsum[1 + kTileCats][32];
  __shared__ int carry[1 + kTileCats];
  __shared__ unsigned long long wcnt[3][32];
  const int tid = threadIdx.x;
  const int nl = p.nlist;
  if (tid <= kTileCats) carry[tid] = 0;
  unsigned long long cc[3] = {0, 0, 0};
  __syncthreads();
  for (int j0 = 0; j0 < nl; j0 += 1024 * kLV) {
    const int jb = j0 + tid * kLV;
    int v[kLV][1 + kTileCats];
    long long len[kLV], r0[kLV];
#pragma unroll
    for (int i = 0; i < kLV; ++i) {
      const int j = jb + i;
      const bool ok = j < nl;
      v[i][0] = ok ? p.list_nq[j] : 0;
#pragma unroll
      for (int cat = 0; cat < kTileCats; ++cat) v[i][1 + cat] = ok ? p.list_ntile[cat * nl + j] : 0;
      len[i] = ok ? p.list_off[j + 1] - p.list_off[j] : 0;
      r0[i] = ok ? p.res_row0[j] : 0;
    }
    int tot[1 + kTileCats] = {0, 0, 0, 0}, ex[1 + kTileCats];
#pragma unroll
    for (int i = 0; i < kLV; ++i) {
#pragma unroll
      for (int c = 0; c <= kTileCats; ++c) tot[c] += v[i][c];
      if (v[i][0] > 0) {
        ++cc[0];
        cc[r0[i] >= 0 ? 1 : 2] += len[i];
      }
    }
    block_scan_round<1024, 1 + kTileCats>(tot, ex, wsum, carry);
#pragma unroll
    for (int i = 0; i < kLV; ++i) {
      const int j = jb + i;
      if (j < nl) {
        p.list_qoff[j] = ex[0];
#pragma unroll
        for (int cat = 0; cat < kTileCats; ++cat) p.list_toff[cat * nl + j] = ex[1 + cat];
      }
#pragma unroll
      for (int c = 0; c <= kTileCats; ++c) ex[c] += v[i][c];
    }
  }
  finish_counters<1024>(p, cc, wcnt, carry + 1);
}

// warp per list: ascending query ids, then the list's tiles. Each bitmap word is zeroed once read,
// so the bitmap is all-zero again for the next search's selection.
__global__ void list_fill_kernel(const PlanParams p) {
  RD_PDL_PROLOGUE();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p.nlist) return;
  const int nq = p.list_nq[warp];
  if (nq == 0) return;  // no bit set: the list's words are zero already
  unsigned* row = p.bitmap + (size_t)warp * p.W;
  int out = p.list_qoff[warp];
  for (int w0 = 0; w0 < p.W; w0 += 32) {
    const int w = w0 + lane;
    const unsigned bits = w < p.W ? row[w] : 0u;
    if (bits) row[w] = 0u;
    const int c = __popc(bits);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = out + incl - c;
    unsigned bb = bits;
    while (bb) {
      const int bit = __ffs(bb) - 1;
      bb &= bb - 1;
      p.list_q[pos++] = w * 32 + bit;
    }
    out += __shfl_sync(0xffffffffu, incl, 31);
  }
  int total = 0;
#pragma unroll
  for (int cat = 0; cat < kTileCats; ++cat) total += p.list_ntile[cat * p.nlist + warp];
  if (total == 0) return;
  const long long len = p.list_off[warp + 1] - p.list_off[warp];
  const int rl = chunk_rows(len, warp >= p.tail_from ? p.Rt : p.R);
  const int chunks = ((int)len + rl - 1) / rl;  // 32-bit: rows per list < 2^31
  const Groups G = group_split(nq, p);
  int toff[kTileCats];
#pragma unroll
  for (int cat = 0; cat < kTileCats; ++cat) toff[cat] = p.list_toff[cat * p.nlist + warp];
  emit_tiles(p, warp, nq, p.list_qoff[warp], (int)len, p.res_row0[warp], p.list_off[warp], toff, G, chunks, rl,
             lane, 32);
}

// Small batches: the whole plan in one CTA with the list x query bitmap in shared memory (one
// launch instead of a memset and four dependent launches; same outputs as the multi-kernel path).
// Lists are visited in rounds of 1024 (thread t <-> list round * 1024 + t) so every per-list global
// access is coalesced, and each warp writes its probed lists' query ids and tiles cooperatively
// (lane = tile), since scattered per-thread stores from one SM are what bounds this kernel.
constexpr int kPlanThreads = 1024;
__global__ void __launch_bounds__(kPlanThreads) plan_fused_kernel(const PlanParams p) {
  RD_TS(13);  // entry, before the wait on the previous kernel
  RD_PDL_PROLOGUE();
  extern __shared__ unsigned bm[];  // nlist x W bitmap, then slen[nlist] (list length, ~len if offloaded)
  __shared__ int wsum[1 + kTileCats][32];
  __shared__ int carry[1 + kTileCats];
  __shared__ unsigned long long wcnt[3][32];
  const int tid = threadIdx.x, lane = tid & 31;
  RD_TS(0);
  const int W = p.W, nl = p.nlist;
  int* slen = reinterpret_cast<int*>(bm + nl * W);
  constexpr int kPB = 8;  // probes in flight per thread
  int pr[kPB];
#pragma unroll
  for (int u = 0; u < kPB; ++u) {
    const int i = tid + u * kPlanThreads;
    pr[u] = i < p.B * p.nprobe ? p.probes[i] : -1;
  }
#pragma unroll 4
  for (int j = tid; j < nl; j += kPlanThreads) {
    const int len = (int)(p.list_off[j + 1] - p.list_off[j]);
    slen[j] = p.res_row0[j] >= 0 ? len : ~len;
  }
  for (int i = tid; i < nl * W; i += kPlanThreads) bm[i] = 0u;
  if (tid <= kTileCats) carry[tid] = 0;
  __syncthreads();
  RD_TS(1);
#pragma unroll
  for (int u = 0; u < kPB; ++u) {
    const int i = tid + u * kPlanThreads;
    if (pr[u] >= 0) atomicOr(&bm[pr[u] * W + ((i / p.nprobe) >> 5)], 1u << ((i / p.nprobe) & 31));
  }
  for (int i = tid + kPB * kPlanThreads; i < p.B * p.nprobe; i += kPlanThreads) {
    const int b = i / p.nprobe, l = p.probes[i];
    if (l >= 0) atomicOr(&bm[l * W + (b >> 5)], 1u << (b & 31));
  }
  __syncthreads();
  RD_TS(2);
  unsigned long long cc[3] = {0, 0, 0};  // unique probed lists, resident rows, offloaded rows
  for (int j0 = 0; j0 < nl; j0 += kPlanThreads) {
    const int j = j0 + tid;
    int nq = 0, len = 0, chunks = 0, rl = p.R;
    Groups G = {{0, 0, 0}};
    long long src0 = 0, g0 = 0;
    if (j < nl) {
      for (int x = 0; x < W; ++x) nq += __popc(bm[j * W + x]);
      const int sl = slen[j];
      len = sl >= 0 ? sl : ~sl;
      if (nq > 0) {
        ++cc[0];
        cc[sl >= 0 ? 1 : 2] += len;
        if (sl >= 0 && len > 0) {
          rl = chunk_rows(len, j >= p.tail_from ? p.Rt : p.R);
          chunks = (len + rl - 1) / rl;
          G = group_split(nq, p);
          src0 = p.res_row0[j];
          g0 = p.list_off[j];
        }
      }
    }
    int v[1 + kTileCats], ex[1 + kTileCats];
    v[0] = nq;
#pragma unroll
    for (int cat = 0; cat < kTileCats; ++cat) v[1 + cat] = G.g[cat] * chunks;
    block_scan_round<kPlanThreads, 1 + kTileCats>(v, ex, wsum, carry);
    if (j < nl) {
      p.list_nq[j] = nq;
      p.list_qoff[j] = ex[0];
    }
    // warp-cooperative emission for the warp's probed lists
    unsigned m = __ballot_sync(0xffffffffu, nq > 0);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const int lj = __shfl_sync(0xffffffffu, j, src), lnq = __shfl_sync(0xffffffffu, nq, src);
      const int qo = __shfl_sync(0xffffffffu, ex[0], src);
      // query ids ascending: lane x < W owns bitmap word x
      const unsigned bits = lane < W ? bm[lj * W + lane] : 0u;
      int pos = __popc(bits);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pos, o);
        if (lane >= o) pos += y;
      }
      pos = qo + pos - __popc(bits);
      for (unsigned bb = bits; bb; bb &= bb - 1) p.list_q[pos++] = lane * 32 + (__ffs(bb) - 1);
      Groups LG;
      int toff[kTileCats], any = 0;
#pragma unroll
      for (int cat = 0; cat < kTileCats; ++cat) {
        LG.g[cat] = __shfl_sync(0xffffffffu, G.g[cat], src);
        toff[cat] = __shfl_sync(0xffffffffu, ex[1 + cat], src);
        any += LG.g[cat];
      }
      if (any > 0)
        emit_tiles(p, lj, lnq, qo, __shfl_sync(0xffffffffu, len, src), __shfl_sync(0xffffffffu, src0, src),
                   __shfl_sync(0xffffffffu, g0, src), toff, LG, __shfl_sync(0xffffffffu, chunks, src),
                   __shfl_sync(0xffffffffu, rl, src), lane, 32);
    }
  }
  RD_TS(3);
  finish_counters<kPlanThreads>(p, cc, wcnt, carry + 1);
  RD_TS(4);
}

constexpr int kSmallPlanThreads = 1024;
__global__ void __launch_bounds__(kSmallPlanThreads) plan_small_kernel(const PlanParams p) {
  RD_TS(13);  // entry, before the wait on the previous kernel
  RD_PDL_PROLOGUE();
  __shared__ SmallPlanSmem sm;
  RD_TS(0);
  plan_small_body<kSmallPlanThreads>(p, sm);
  RD_TS(3);
}

}  // namespace

// the rank sort is O(pairs) per thread: beyond ~512 pairs the bitmap planners win
bool plan_small_ok(int B, int nprobe) { return (long long)B * nprobe <= 512; }

bool plan_fused_ok(int B, int nlist) {
  const long long W = (B + 31) / 32;
  // one SM's issue rate bounds the fused kernel (~150 instructions per probed list): beyond a few
  // hundred probed lists the grid-wide multi-kernel plan is faster
  return B <= 8 && (long long)nlist * (W + 1) * 4 <= 96 * 1024;
}

cudaError_t launch_plan(const PlanParams& p, cudaStream_t s) {
  if (plan_small_ok(p.B, p.nprobe)) return launch_k(plan_small_kernel, dim3(1), dim3(kSmallPlanThreads), 0, s, p);
  if (plan_fused_ok(p.B, p.nlist)) {
    const int smem = p.nlist * (p.W + 1) * (int)sizeof(unsigned);
    return launch_k(plan_fused_kernel, dim3(1), dim3(kPlanThreads), smem, s, p);
  }
  // the selection filled p.bitmap (plan_uses_bitmap); count -> scan -> fill, chained with PDL
  const int blocks = (p.nlist * 32 + 255) / 256;
  cudaError_t e = launch_k(list_count_kernel, dim3(blocks), dim3(256), 0, s, p);
  if (e == cudaSuccess) e = launch_k(list_scan_kernel, dim3(1), dim3(1024), 0, s, p);
  if (e == cudaSuccess) e = launch_k(list_fill_kernel, dim3(blocks), dim3(256), 0, s, p);
  return e;
}

}  // namespace rd
