// plan.cu — N3 probe inversion and scan work planning (sm_100a).
//
// The B x nprobe probe table is inverted into per-list query groups through a
// list x query bitmap (so queries within a list come out in ascending id,
// deterministically), then every probed, HBM-resident list is cut into scan
// tiles of <= R rows x <= 16 queries. Tiles of one list are adjacent so the
// query groups of a chunk hit L2 for each other. Offloaded lists get no device
// tiles here; the host plans them as their bytes are staged (api.cu).
#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

__global__ void invert_set_kernel(const int* __restrict__ probes, unsigned* __restrict__ bitmap,
                                  int W, int B, int nprobe) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)B * nprobe) return;
  const int b = (int)(i / nprobe);
  const int l = probes[i];
  if (l >= 0) atomicOr(bitmap + (size_t)l * W + (b >> 5), 1u << (b & 31));
}

// Query groups of one list. A list probed by >= tc_min_q queries is scanned once per
// balanced group of <= kTcG queries on the tensor cores (almost always a single group, so the
// list's bytes are read once); sparser lists form one FFMA group (<= tc_min_q - 1 <= kScanG).
__device__ __forceinline__ void group_split(int nq, int tc_min_q, int& ntc, int& nff) {
  if (nq >= tc_min_q) {
    ntc = (nq + kTcG - 1) / kTcG;
    nff = 0;
  } else {
    ntc = 0;
    nff = (nq + kScanG - 1) / kScanG;
  }
}

// The tiles of one list (chunk-major, group-minor in the tile arrays): groups outer so each group's
// query split is computed once; chunks c = c0, c0 + cstep, ... (lanes of a warp, or one thread)
__device__ __forceinline__ void emit_tiles(const PlanParams& p, int j, int nq, int qoff, int len, long long src0,
                                           long long g0, int toff_tc, int toff_ff, int gtc, int gff, int chunks,
                                           int c0, int cstep) {
  for (int g = 0; g < gtc + gff; ++g) {
    int tq0, tnq, stride;
    ScanTile* dst;
    if (g < gtc) {  // balanced tensor-core groups
      const bool s32 = nq < 46341;  // g * nq < 2^31 for g <= nq / 32 + 1
      const int q0 = s32 ? g * nq / gtc : (int)((long long)g * nq / gtc);
      const int q1 = s32 ? (g + 1) * nq / gtc : (int)((long long)(g + 1) * nq / gtc);
      tq0 = qoff + q0;
      tnq = q1 - q0;
      dst = p.tiles + toff_tc + g;
      stride = gtc;
    } else {
      const int gg = g - gtc;
      tq0 = qoff + gg * kScanG;
      tnq = min(kScanG, nq - gg * kScanG);
      dst = p.ff_tiles + toff_ff + gg;
      stride = gff;
    }
    for (int c = c0; c < chunks; c += cstep) {
      ScanTile T;
      T.src_row = src0 + (long long)c * p.R;
      T.grow0 = g0 + (long long)c * p.R;
      T.list = j;
      T.nrows = min(p.R, len - c * p.R);
      T.qoff = tq0;
      T.nq = tnq;
      dst[c * stride] = T;
    }
  }
}

// warp per list: query count and resident tile counts
__global__ void list_count_kernel(const PlanParams p) {
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
    int ntc = 0, nff = 0;
    if (c > 0 && len > 0 && p.res_row0[warp] >= 0) {
      const int chunks = ((int)len + p.R - 1) / p.R;  // 32-bit: rows per list < 2^31
      group_split(c, p.tc_min_q, ntc, nff);
      ntc *= chunks;
      nff *= chunks;
    }
    p.list_ntile[warp] = ntc;
    p.list_ntile[p.nlist + warp] = nff;
  }
}

// single CTA: exclusive scans of list_nq and both tile counts; totals and byte counters
__global__ void __launch_bounds__(1024) list_scan_kernel(const PlanParams p) {
  __shared__ long long sh[3][32];
  __shared__ unsigned long long sh_c[3][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int per = (p.nlist + 1023) / 1024;
  const int j0 = tid * per, j1 = min(p.nlist, j0 + per);
  long long loc[3] = {0, 0, 0};
  unsigned long long uniq = 0, rrows = 0, orows = 0;
  for (int j = j0; j < j1; ++j) {
    const int nq = p.list_nq[j];
    loc[0] += nq;
    loc[1] += p.list_ntile[j];
    loc[2] += p.list_ntile[p.nlist + j];
    if (nq > 0) {
      const long long len = p.list_off[j + 1] - p.list_off[j];
      ++uniq;
      if (p.res_row0[j] >= 0)
        rrows += len;
      else
        orows += len;
    }
  }
  long long inc[3] = {loc[0], loc[1], loc[2]};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const long long y = __shfl_up_sync(0xffffffffu, inc[i], o);
      if (lane >= o) inc[i] += y;
    }
  unsigned long long cc[3] = {uniq, rrows, orows};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) cc[i] += __shfl_xor_sync(0xffffffffu, cc[i], o);
  if (lane == 31)
    for (int i = 0; i < 3; ++i) sh[i][w] = inc[i];
  if (lane == 0)
    for (int i = 0; i < 3; ++i) sh_c[i][w] = cc[i];
  __syncthreads();
  if (w == 0) {
    long long a[3] = {sh[0][lane], sh[1][lane], sh[2][lane]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const long long y = __shfl_up_sync(0xffffffffu, a[i], o);
        if (lane >= o) a[i] += y;
      }
    for (int i = 0; i < 3; ++i) sh[i][lane] = a[i];
    unsigned long long c[3] = {sh_c[0][lane], sh_c[1][lane], sh_c[2][lane]};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) c[i] += __shfl_xor_sync(0xffffffffu, c[i], o);
    const long long tot_tc = __shfl_sync(0xffffffffu, a[1], 31), tot_ff = __shfl_sync(0xffffffffu, a[2], 31);
    if (lane == 0) {
      for (int i = 0; i < 3; ++i) p.counters[i] = c[i];
      p.meta[0] = (int)tot_tc;
      p.meta[1] = 0;
      p.meta[2] = (int)tot_ff;
      p.meta[3] = 0;
    }
  }
  __syncthreads();
  long long o0 = (w ? sh[0][w - 1] : 0) + inc[0] - loc[0];
  long long o1 = (w ? sh[1][w - 1] : 0) + inc[1] - loc[1];
  long long o2 = (w ? sh[2][w - 1] : 0) + inc[2] - loc[2];
  for (int j = j0; j < j1; ++j) {
    p.list_qoff[j] = (int)o0;
    p.list_toff[j] = (int)o1;
    p.list_toff[p.nlist + j] = (int)o2;
    o0 += p.list_nq[j];
    o1 += p.list_ntile[j];
    o2 += p.list_ntile[p.nlist + j];
  }
}

// warp per list: ascending query ids, then the list's tiles (chunk-major, group-minor)
__global__ void list_fill_kernel(const PlanParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= p.nlist) return;
  const int nq = p.list_nq[warp];
  if (nq == 0) return;
  const unsigned* row = p.bitmap + (size_t)warp * p.W;
  int out = p.list_qoff[warp];
  for (int w0 = 0; w0 < p.W; w0 += 32) {
    const int w = w0 + lane;
    const unsigned bits = w < p.W ? row[w] : 0u;
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
  const int ntc = p.list_ntile[warp], nff = p.list_ntile[p.nlist + warp];
  if (ntc + nff == 0) return;
  const long long len = p.list_off[warp + 1] - p.list_off[warp];
  const int chunks = ((int)len + p.R - 1) / p.R;  // 32-bit: rows per list < 2^31
  const int gtc = ntc / chunks, gff = nff / chunks;
  emit_tiles(p, warp, nq, p.list_qoff[warp], (int)len, p.res_row0[warp], p.list_off[warp], p.list_toff[warp],
             p.list_toff[p.nlist + warp], gtc, gff, chunks, lane, 32);
}

// Small batches: the whole plan in one CTA with the list x query bitmap in shared memory (one
// launch instead of a memset and four dependent launches; same outputs as the multi-kernel path).
constexpr int kPlanThreads = 1024;
constexpr int kPlanMaxPer = 16;  // lists per thread (nlist <= 16384)
__global__ void __launch_bounds__(kPlanThreads) plan_fused_kernel(const PlanParams p) {
  RD_PDL_PROLOGUE();
  extern __shared__ unsigned bm[];  // nlist x W bitmap, then slen[nlist] (list length, ~len if offloaded)
  __shared__ long long sh[3][32];
  __shared__ unsigned long long sh_c[3][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int W = p.W, nl = p.nlist;
  int* slen = reinterpret_cast<int*>(bm + nl * W);
  const int per = (nl + kPlanThreads - 1) / kPlanThreads;
  const int j0 = min(nl, tid * per), j1 = min(nl, j0 + per);
  {  // every global load of the count phase in flight at once: list bounds, residency, probes
    long long off[kPlanMaxPer + 1], rr[kPlanMaxPer];
#pragma unroll
    for (int u = 0; u <= kPlanMaxPer; ++u) off[u] = j0 + u <= j1 ? p.list_off[j0 + u] : 0;
#pragma unroll
    for (int u = 0; u < kPlanMaxPer; ++u) rr[u] = j0 + u < j1 ? p.res_row0[j0 + u] : 0;
    constexpr int kPB = 8;
    int pr[kPB];
#pragma unroll
    for (int u = 0; u < kPB; ++u) {
      const int i = tid + u * kPlanThreads;
      pr[u] = i < p.B * p.nprobe ? p.probes[i] : -1;
    }
    for (int i = tid; i < nl * W; i += kPlanThreads) bm[i] = 0u;
#pragma unroll
    for (int u = 0; u < kPlanMaxPer; ++u)
      if (j0 + u < j1) {
        const int len = (int)(off[u + 1] - off[u]);
        slen[j0 + u] = rr[u] >= 0 ? len : ~len;
      }
    __syncthreads();
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
  }
  // per list: query count, resident tile counts (recomputed in the fill pass instead of kept in registers)
  auto counts = [&](int j, int& nq, int& ntc, int& nff, long long& len) {
    nq = 0;
    for (int x = 0; x < W; ++x) nq += __popc(bm[j * W + x]);
    const int sl = slen[j];
    len = sl >= 0 ? sl : ~sl;
    ntc = nff = 0;
    if (nq > 0 && len > 0 && sl >= 0) {
      const int chunks = ((int)len + p.R - 1) / p.R;  // 32-bit: rows per list < 2^31
      group_split(nq, p.tc_min_q, ntc, nff);
      ntc *= chunks;
      nff *= chunks;
    }
  };
  long long loc[3] = {0, 0, 0};
  unsigned long long cc[3] = {0, 0, 0};
  for (int j = j0; j < j1; ++j) {
    int nq, ntc, nff;
    long long len;
    counts(j, nq, ntc, nff, len);
    if (nq > 0) {
      ++cc[0];
      cc[slen[j] >= 0 ? 1 : 2] += len;
    }
    loc[0] += nq;
    loc[1] += ntc;
    loc[2] += nff;
  }
  long long inc[3] = {loc[0], loc[1], loc[2]};
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const long long y = __shfl_up_sync(0xffffffffu, inc[i], o);
      if (lane >= o) inc[i] += y;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) cc[i] += __shfl_xor_sync(0xffffffffu, cc[i], o);
  if (lane == 31)
    for (int i = 0; i < 3; ++i) sh[i][w] = inc[i];
  if (lane == 0)
    for (int i = 0; i < 3; ++i) sh_c[i][w] = cc[i];
  __syncthreads();
  if (w == 0) {
    long long a[3] = {sh[0][lane], sh[1][lane], sh[2][lane]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const long long y = __shfl_up_sync(0xffffffffu, a[i], o);
        if (lane >= o) a[i] += y;
      }
    for (int i = 0; i < 3; ++i) sh[i][lane] = a[i];
    unsigned long long c[3] = {sh_c[0][lane], sh_c[1][lane], sh_c[2][lane]};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < 3; ++i) c[i] += __shfl_xor_sync(0xffffffffu, c[i], o);
    const long long t1 = __shfl_sync(0xffffffffu, a[1], 31), t2 = __shfl_sync(0xffffffffu, a[2], 31);
    if (lane == 0) {
      for (int i = 0; i < 3; ++i) p.counters[i] = c[i];
      p.meta[0] = (int)t1;
      p.meta[1] = 0;
      p.meta[2] = (int)t2;
      p.meta[3] = 0;
    }
  }
  __syncthreads();
  long long o0 = (w ? sh[0][w - 1] : 0) + inc[0] - loc[0];
  long long o1 = (w ? sh[1][w - 1] : 0) + inc[1] - loc[1];
  long long o2 = (w ? sh[2][w - 1] : 0) + inc[2] - loc[2];
  for (int j = j0; j < j1; ++j) {
    int nq, ntc, nff;
    long long len;
    counts(j, nq, ntc, nff, len);
    p.list_nq[j] = nq;
    p.list_qoff[j] = (int)o0;
    p.list_ntile[j] = ntc;
    p.list_ntile[nl + j] = nff;
    p.list_toff[j] = (int)o1;
    p.list_toff[nl + j] = (int)o2;
    if (nq > 0) {
      int out = (int)o0;
      for (int x = 0; x < W; ++x) {
        unsigned bb = bm[j * W + x];
        while (bb) {
          const int bit = __ffs(bb) - 1;
          bb &= bb - 1;
          p.list_q[out++] = x * 32 + bit;
        }
      }
      if (ntc + nff > 0) {
        const int chunks = ((int)len + p.R - 1) / p.R;  // 32-bit: rows per list < 2^31
        const int gtc = ntc / chunks, gff = nff / chunks;
        emit_tiles(p, j, nq, (int)o0, (int)len, p.res_row0[j], p.list_off[j], (int)o1, (int)o2, gtc, gff, chunks, 0,
                   1);
      }
    }
    o0 += nq;
    o1 += ntc;
    o2 += nff;
  }
}

}  // namespace

bool plan_fused_ok(int B, int nlist) {
  const long long W = (B + 31) / 32;
  return B <= 128 && nlist <= kPlanThreads * kPlanMaxPer && (long long)nlist * (W + 1) * 4 <= 96 * 1024;
}

cudaError_t launch_plan(const PlanParams& p, cudaStream_t s) {
  if (plan_fused_ok(p.B, p.nlist)) {
    const int smem = p.nlist * (p.W + 1) * (int)sizeof(unsigned);
    static int attr = 0;
    if (smem > attr) {  // dynamic + static may exceed the 48 KiB default even below it
      cudaError_t e = cudaFuncSetAttribute(plan_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      attr = smem;
    }
    return launch_k(plan_fused_kernel, dim3(1), dim3(kPlanThreads), smem, s, p);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(p.bitmap, 0, sizeof(unsigned) * (size_t)p.nlist * p.W, s);
  if (e != cudaSuccess) return e;
  const long long np = (long long)p.B * p.nprobe;
  invert_set_kernel<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(p.probes, p.bitmap, p.W, p.B, p.nprobe);
  const int blocks = (p.nlist * 32 + 255) / 256;
  list_count_kernel<<<blocks, 256, 0, s>>>(p);
  list_scan_kernel<<<1, 1024, 0, s>>>(p);
  list_fill_kernel<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace rd
