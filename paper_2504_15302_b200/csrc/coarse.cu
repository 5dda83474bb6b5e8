// coarse.cu — N1 coarse quantization and N2 per-query nprobe selection (sm_100a).
//
// N1: Dc[b][j] = ||c_j||^2 - 2 q_b.c_j with a register-tiled FFMA GEMM
//     (64 queries x 128 centroids per CTA, 4x8 per thread, k-major smem tiles).
// N2: one CTA per query: radix-select the C = nprobe + 32 smallest approximate
//     distances, recompute those exactly (canonical fp64 sum, identical to the
//     oracle), order by (exact distance, list id) and keep nprobe. The probe set
//     is certified when every non-candidate's approximate distance, less the
//     GEMM's error bound, exceeds the nprobe-th exact distance.
#include <float.h>

#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr int kBM = 64, kBN = 128, kBK = 16;

__global__ void __launch_bounds__(256) coarse_gemm_kernel(const float* __restrict__ Q,
                                                          const float* __restrict__ C,
                                                          const float* __restrict__ cnorm,
                                                          float* __restrict__ Dc, int B, int nlist,
                                                          int d) {
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

__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// block-wide exclusive scan of one int per thread (256 threads); returns total via *total
__device__ int block_excl_scan(int v, int* sh, int* total) {
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
    int s = lane < 8 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < 8) sh[lane] = s;
  }
  __syncthreads();
  const int base = w ? sh[w - 1] : 0;
  *total = sh[7];
  __syncthreads();
  return base + x - v;
}

constexpr int kSelThreads = 256;
constexpr int kSelMaxCand = 512;

// Selects the C smallest of keys[0..nlist) into cand[0..C): all keys < T plus the
// first keys == T by index (radix select, 11+11+10 bits, then an ordered compaction).
__device__ uint32_t select_smallest(const uint32_t* keys, int nlist, int C, int* hist, int* scan_sh, int* cand,
                                    uint32_t* sel_prefix, uint32_t* sel_k) {
  const int tid = threadIdx.x;
  uint32_t prefix = 0, mask = 0, kk = (uint32_t)C;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
  for (int pass = 0; pass < 3; ++pass) {
    const int sh = shifts[pass], nb = 1 << widths[pass];
    for (int i = tid; i < nb; i += kSelThreads) hist[i] = 0;
    __syncthreads();
    for (int j = tid; j < nlist; j += kSelThreads) {
      const uint32_t kv = keys[j];
      if ((kv & mask) == prefix) atomicAdd(&hist[(kv >> sh) & (nb - 1)], 1);
    }
    __syncthreads();
    const int per = nb / kSelThreads;
    int local = 0;
    for (int i = 0; i < per; ++i) local += hist[tid * per + i];
    int tot;
    const int before = block_excl_scan(local, scan_sh, &tot);
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
  const int per = (nlist + kSelThreads - 1) / kSelThreads;
  const int j0 = tid * per, j1 = min(nlist, j0 + per);
  int nlt = 0, neq = 0;
  for (int j = j0; j < j1; ++j) {
    nlt += keys[j] < T;
    neq += keys[j] == T;
  }
  int tot_lt, tot_eq;
  int olt = block_excl_scan(nlt, scan_sh, &tot_lt);
  int oeq = block_excl_scan(neq, scan_sh, &tot_eq);
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

__device__ __forceinline__ float block_reduce_min(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = sh[0];
  for (int i = 1; i < kSelThreads / 32; ++i) r = fminf(r, sh[i]);
  return r;
}
__device__ __forceinline__ float block_reduce_max(float v, float* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = sh[0];
  for (int i = 1; i < kSelThreads / 32; ++i) r = fmaxf(r, sh[i]);
  return r;
}

// dynamic smem: keys[nlist] (u32; approximate distances as floats, then exact keys in the fallback)
__global__ void __launch_bounds__(kSelThreads) coarse_select_kernel(const SelectParams p) {
  extern __shared__ uint32_t keys[];
  __shared__ int hist[2048];
  __shared__ int scan_sh[8];
  __shared__ float fsh[8];
  __shared__ int cand[kSelMaxCand];
  __shared__ float cdist[kSelMaxCand];
  __shared__ uint32_t sel_prefix, sel_k;
  __shared__ int certified, ncand_s, found_bin;
  const int b = blockIdx.x, tid = threadIdx.x;
  const int nlist = p.nlist;
  const float* q = p.queries + (size_t)b * p.d;
  const int grp = tid >> 3, j8 = tid & 7;
  const int np = min(p.nprobe, nlist);
  const float* drow = p.Dc + (size_t)b * nlist;
  float* vals = reinterpret_cast<float*>(keys);
  float vmin = __builtin_huge_valf(), vmax = -__builtin_huge_valf();
  for (int j = tid; j < nlist; j += kSelThreads) {
    const float v = drow[j];
    vals[j] = v;
    vmin = fminf(vmin, v);
    vmax = fmaxf(vmax, v);
  }
  vmin = block_reduce_min(vmin, fsh);
  vmax = block_reduce_max(vmax, fsh);
  const int Cwant = min(nlist, p.nprobe + kCoarseExtra);

  // attempt 0: a candidate set {approx < hi} of size in [C, kSelMaxCand], found with value-linear
  // 2048-bin histograms (refined inside the crossing bin when it is too dense); exact refine;
  // certification with hi as the lower bound of every excluded approximate distance.
  // attempt 1 (uncertified or no usable threshold): exact distances to every centroid.
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
      for (int i = tid; i < 2048; i += kSelThreads) hist[i] = 0;
      __syncthreads();
      for (int j = tid; j < nlist; j += kSelThreads) {
        const float v = vals[j];
        if (v >= lo && v < hi) atomicAdd(&hist[min(2047, (int)((v - lo) / width))], 1);
      }
      __syncthreads();
      int local = 0;
      for (int i = 0; i < 8; ++i) local += hist[tid * 8 + i];
      int tot;
      const int before = block_excl_scan(local, scan_sh, &tot);
      if (tid == 0) found_bin = 2047;
      __syncthreads();
      if (below + before < Cwant && below + before + local >= Cwant) {
        int run = below + before;
        for (int i = 0; i < 8; ++i) {
          run += hist[tid * 8 + i];
          if (run >= Cwant) {
            found_bin = tid * 8 + i;
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
      for (int j = tid; j < nlist; j += kSelThreads) c += vals[j] < edge_hi;
      int total;
      block_excl_scan(c, scan_sh, &total);
      if (total >= Cwant && total <= kSelMaxCand) {
        ncand = total;
        hi_edge = edge_hi;
      } else {
        int cb = 0;
        for (int j = tid; j < nlist; j += kSelThreads) cb += vals[j] < edge_lo;
        int tb;
        block_excl_scan(cb, scan_sh, &tb);
        below = tb;
        lo = edge_lo;
        hi = edge_hi;
      }
    }
  }
  if (ncand >= 0) {
    if (tid == 0) ncand_s = 0;
    __syncthreads();
    for (int j = tid; j < nlist; j += kSelThreads)
      if (vals[j] < hi_edge) cand[atomicAdd(&ncand_s, 1)] = j;
    __syncthreads();
  }

  for (int attempt = (ncand >= 0 ? 0 : 1); attempt < 2; ++attempt) {
    int C;
    if (attempt == 0) {
      C = ncand;
    } else {
      // exact keys for every centroid, then the np smallest by (exact distance, list id)
      for (int c0 = 0; c0 < nlist; c0 += kSelThreads / 8) {
        const int c = c0 + grp;
        const int cc = c < nlist ? c : nlist - 1;
        const float e = exact_l2_group8(q, p.centroids + (size_t)cc * p.d, p.d, j8);
        __syncthreads();
        if (c < nlist && j8 == 0) keys[c] = f2key(e);
      }
      __syncthreads();
      C = np;
      select_smallest(keys, nlist, C, hist, scan_sh, cand, &sel_prefix, &sel_k);
    }
    for (int c0 = 0; c0 < C; c0 += kSelThreads / 8) {
      const int c = c0 + grp;
      const int cc = c < C ? c : C - 1;
      const float e = exact_l2_group8(q, p.centroids + (size_t)cand[cc] * p.d, p.d, j8);
      if (c < C && j8 == 0) cdist[c] = e;
    }
    int P2 = 1;
    while (P2 < C) P2 <<= 1;
    for (int c = C + tid; c < P2; c += kSelThreads) {
      cdist[c] = __builtin_huge_valf();
      cand[c] = 0x7fffffff;
    }
    __syncthreads();
    for (int size = 2; size <= P2; size <<= 1) {
      for (int jj = size >> 1; jj > 0; jj >>= 1) {
        for (int i = tid; i < P2; i += kSelThreads) {
          const int l = i ^ jj;
          if (l > i) {
            const bool up = (i & size) == 0;
            const float di = cdist[i], dl = cdist[l];
            const int ii = cand[i], il = cand[l];
            const bool l_less = dl < di || (dl == di && il < ii);
            if (l_less == up) {
              cdist[i] = dl;
              cdist[l] = di;
              cand[i] = il;
              cand[l] = ii;
            }
          }
        }
        __syncthreads();
      }
    }
    if (tid == 0) {
      int ok = 1;
      if (attempt == 0) {
        // every excluded centroid has approx >= hi_edge; the GEMM's error bound turns that into
        // a lower bound on its exact distance
        const float qn = p.qnorm[b];
        const float u = 5.9604645e-8f;
        const float eps = 2.f * ((p.d + 4) * u * 2.f * sqrtf(qn) * p.cmax + 8.f * u * (qn + p.cmax * p.cmax)) + 1e-30f;
        const float lower = hi_edge + qn - eps;
        ok = lower > cdist[np - 1];
      }
      certified = ok;
      if (!ok) atomicAdd(p.probe_fail, 1u);
    }
    __syncthreads();
    if (certified) break;
  }
  for (int i = tid; i < p.nprobe; i += kSelThreads) p.probes[(size_t)b * p.nprobe + i] = i < np ? cand[i] : -1;

  // fused seed: exact distances to the first 32 rows of the nearest resident probed list with
  // >= 32 rows; threshold = max + 2*eps_scan (valid upper bound on the final 32nd-best approximate
  // distance, so the scan's certification holds; see merge.cu seed_kernel)
  if (p.qthr) {
    __shared__ int lsel;
    __shared__ float red[kSelThreads / 32];
    if (tid == 0) {
      lsel = -1;
      for (int i = 0; i < np; ++i) {
        const int l = cand[i];
        if (p.res_row0[l] >= 0 && p.list_off[l + 1] - p.list_off[l] >= 32) {
          lsel = l;
          break;
        }
      }
    }
    __syncthreads();
    const int l = lsel;
    if (l < 0) {
      if (tid == 0) p.qthr[b] = 0x7f7f7f7f;
    } else {
      const float e = exact_l2_group8(q, p.arena + (size_t)(p.res_row0[l] + grp) * p.d, p.d, j8);
      float m = e;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((tid & 31) == 0) red[tid >> 5] = m;
      __syncthreads();
      if (tid == 0) {
        float mx = red[0];
        for (int i = 1; i < kSelThreads / 32; ++i) mx = fmaxf(mx, red[i]);
        const float qn = p.qnorm[b];
        const float u = 5.9604645e-8f;
        const float eps =
            2.f * ((p.d / 2 + 8) * u * 2.f * sqrtf(qn) * p.xmax + 8.f * u * (qn + p.xmax * p.xmax)) + 1e-30f;
        const float thr = mx + 2.f * eps;
        const int ti = __float_as_int(thr);
        p.qthr[b] = ti >= 0 ? ti : ti ^ 0x7fffffff;
      }
    }
  }
}

}  // namespace

cudaError_t launch_coarse(const float* Q, const float* C, const float* cnorm, float* Dc, int B,
                          int nlist, int d, cudaStream_t s) {
  dim3 grid((nlist + kBN - 1) / kBN, (B + kBM - 1) / kBM);
  coarse_gemm_kernel<<<grid, 256, 0, s>>>(Q, C, cnorm, Dc, B, nlist, d);
  return cudaGetLastError();
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t s) {
  if (p.nprobe + kCoarseExtra > kSelMaxCand) return cudaErrorInvalidValue;
  const size_t smem = sizeof(uint32_t) * (size_t)p.nlist;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(coarse_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  coarse_select_kernel<<<p.B, kSelThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace rd
