// plan.cu — N3 probe inversion and scan work planning (sm_100a).
//
// The B x nprobe probe table is inverted into per-list query groups through a
// list x query bitmap (so queries within a list come out in ascending id,
// deterministically), then every probed, HBM-resident list is cut into scan
// tiles of <= R rows x <= 16 queries. Tiles of one list are adjacent so the
// query groups of a chunk hit L2 for each other. Offloaded lists get no device
// tiles here; the host plans them as their bytes are staged (api.cu).
#include "ivf_kernels.cuh"

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
      const int chunks = (int)((len + p.R - 1) / p.R);
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
  const int chunks = (int)((len + p.R - 1) / p.R);
  const int gtc = ntc / chunks, gff = nff / chunks;
  const int ngr = gtc + gff;
  const int toff_tc = p.list_toff[warp], toff_ff = p.list_toff[p.nlist + warp];
  for (int t = lane; t < chunks * ngr; t += 32) {
    const int c = t / ngr, g = t - c * ngr;
    ScanTile T;
    T.src_row = p.res_row0[warp] + (long long)c * p.R;
    T.grow0 = p.list_off[warp] + (long long)c * p.R;
    T.list = warp;
    T.nrows = (int)min((long long)p.R, len - (long long)c * p.R);
    if (g < gtc) {  // balanced tensor-core groups
      const int q0 = (int)((long long)g * nq / gtc), q1 = (int)((long long)(g + 1) * nq / gtc);
      T.qoff = p.list_qoff[warp] + q0;
      T.nq = q1 - q0;
      p.tiles[toff_tc + c * gtc + g] = T;
    } else {
      const int gg = g - gtc;
      T.qoff = p.list_qoff[warp] + gg * kScanG;
      T.nq = min(kScanG, nq - gg * kScanG);
      p.ff_tiles[toff_ff + c * gff + gg] = T;
    }
  }
}

}  // namespace

cudaError_t launch_plan(const PlanParams& p, cudaStream_t s) {
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
