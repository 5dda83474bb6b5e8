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

// warp per list: query count and resident tile count
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
    int nt = 0;
    if (c > 0 && len > 0 && p.res_row0[warp] >= 0)
      nt = (int)((len + p.R - 1) / p.R) * ((c + kScanG - 1) / kScanG);
    p.list_ntile[warp] = nt;
  }
}

// single CTA: exclusive scans of list_nq and list_ntile; totals and byte counters
__global__ void __launch_bounds__(1024) list_scan_kernel(const PlanParams p) {
  __shared__ long long sh_q[32], sh_t[32];
  __shared__ unsigned long long sh_c[3][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int per = (p.nlist + 1023) / 1024;
  const int j0 = tid * per, j1 = min(p.nlist, j0 + per);
  long long sq = 0, st = 0;
  unsigned long long uniq = 0, rrows = 0, orows = 0;
  for (int j = j0; j < j1; ++j) {
    const int nq = p.list_nq[j];
    sq += nq;
    st += p.list_ntile[j];
    if (nq > 0) {
      const long long len = p.list_off[j + 1] - p.list_off[j];
      ++uniq;
      if (p.res_row0[j] >= 0)
        rrows += len;
      else
        orows += len;
    }
  }
  long long xq = sq, xt = st;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long a = __shfl_up_sync(0xffffffffu, xq, o), b = __shfl_up_sync(0xffffffffu, xt, o);
    if (lane >= o) {
      xq += a;
      xt += b;
    }
  }
  unsigned long long cu = uniq, cr = rrows, co = orows;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cu += __shfl_xor_sync(0xffffffffu, cu, o);
    cr += __shfl_xor_sync(0xffffffffu, cr, o);
    co += __shfl_xor_sync(0xffffffffu, co, o);
  }
  if (lane == 31) {
    sh_q[w] = xq;
    sh_t[w] = xt;
  }
  if (lane == 0) {
    sh_c[0][w] = cu;
    sh_c[1][w] = cr;
    sh_c[2][w] = co;
  }
  __syncthreads();
  if (w == 0) {
    long long a = sh_q[lane], b = sh_t[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long ya = __shfl_up_sync(0xffffffffu, a, o), yb = __shfl_up_sync(0xffffffffu, b, o);
      if (lane >= o) {
        a += ya;
        b += yb;
      }
    }
    sh_q[lane] = a;
    sh_t[lane] = b;
    unsigned long long c0 = sh_c[0][lane], c1 = sh_c[1][lane], c2 = sh_c[2][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      c0 += __shfl_xor_sync(0xffffffffu, c0, o);
      c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    }
    if (lane == 0) {
      p.counters[0] = c0;
      p.counters[1] = c1;
      p.counters[2] = c2;
      *p.ntiles = (int)sh_t[31];
    }
  }
  __syncthreads();
  long long oq = (w ? sh_q[w - 1] : 0) + xq - sq;
  long long ot = (w ? sh_t[w - 1] : 0) + xt - st;
  for (int j = j0; j < j1; ++j) {
    p.list_qoff[j] = (int)oq;
    p.list_toff[j] = (int)ot;
    oq += p.list_nq[j];
    ot += p.list_ntile[j];
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
  const int nt = p.list_ntile[warp];
  if (nt == 0) return;
  const long long len = p.list_off[warp + 1] - p.list_off[warp];
  const int ngr = (nq + kScanG - 1) / kScanG;
  const int toff = p.list_toff[warp];
  for (int t = lane; t < nt; t += 32) {
    const int c = t / ngr, g = t - c * ngr;
    ScanTile T;
    T.src_row = p.res_row0[warp] + (long long)c * p.R;
    T.grow0 = p.list_off[warp] + (long long)c * p.R;
    T.list = warp;
    T.nrows = (int)min((long long)p.R, len - (long long)c * p.R);
    T.qoff = p.list_qoff[warp] + g * kScanG;
    T.nq = min(kScanG, nq - g * kScanG);
    p.tiles[toff + t] = T;
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
