// resid.cu — the residual store's build and the per-search pair operands (sm_100a).
//
// The residual store keeps the fp32 rows (exact rerank, seeding, fallback) plus one bf16 plane
// r1 = bf16(x - c_l) per resident row, c_l the row's list centroid: the tensor-core scan reads
// 2 B per element instead of the split3 store's 4 (x1 | x2). Its keys are
//   key = (||q - c||^2 - eps_pair) + ||x - c||^2 - 2 r1 . (p1 + p2),   p1 + p2 ~ fl32(q - c),
// and |exact - (||q - c||^2 + ||x - c||^2 - 2 r1 . (p1 + p2))| <= eps_pair = 2 gamma_resid
// ||q - c|| max_l ||x - c|| + 32 u (||q - c||^2 + max_l ||x - c||^2), so every key is a
// lower bound on the row's exact distance: the scan's pruning, the merge's certification and the
// seeding threshold then need no error term of their own. Residuals are small against the vectors
// (IVF: rows sit near their centroid), so the bound stays well inside the gap between rank k and the
// certification rank, and exactness is the same as every other store's: exact rerank + fallback.
#include <cuda_bf16.h>

#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr int kMaxPerLane = 32;  // d <= 1024

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One CTA per list: warp per row, lanes over dimensions (coalesced); r = x - c exactly in fp64.
__global__ void __launch_bounds__(256) resid_build_kernel(const float* __restrict__ arena,
                                                          const long long* __restrict__ res_row0,
                                                          const long long* __restrict__ list_off,
                                                          const float* __restrict__ centroids, int d,
                                                          __nv_bfloat16* __restrict__ r1, float* __restrict__ rnorm,
                                                          float* __restrict__ rmax) {
  __shared__ double wmax[8];
  const int l = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long g0 = list_off[l], len = list_off[l + 1] - g0, sr0 = res_row0[l];
  const int per = d >> 5;
  double c[kMaxPerLane];
#pragma unroll
  for (int j = 0; j < kMaxPerLane; ++j) c[j] = j < per ? (double)centroids[(size_t)l * d + j * 32 + lane] : 0.0;
  double mx = 0.0;
  if (sr0 >= 0)
    for (long long i = warp; i < len; i += 8) {
      const float* x = arena + (size_t)(sr0 + i) * d;
      __nv_bfloat16* o = r1 + (size_t)(sr0 + i) * d;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < kMaxPerLane; ++j) {
        if (j >= per) break;
        const double r = (double)x[j * 32 + lane] - c[j];
        o[j * 32 + lane] = __double2bfloat16(r);
        s = fma(r, r, s);
      }
      s = warp_sum_f64(s);
      if (lane == 0) rnorm[g0 + i] = (float)s;
      mx = fmax(mx, s);
    }
  if (lane == 0) wmax[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < 8; ++w) m = fmax(m, wmax[w]);
    rmax[l] = __double2float_ru(sqrt(m) * (1.0 + 1e-12));
  }
}

// Warp per pair; lane owns 4 consecutive elements per 128-element block (float4 loads of q and c,
// all in flight before any use; 8-byte bf16x4 stores).
__global__ void __launch_bounds__(256) pair_operand_kernel(const PairParams p) {
  RD_PDL_PROLOGUE();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, d = p.d, nb = d >> 7;
  const int n16 = p.t16 ? *p.n16 : 0, n32 = p.t32 ? *p.n32 : 0;
  __nv_bfloat16* __restrict__ out = reinterpret_cast<__nv_bfloat16*>(p.pairs);
  for (int v = blockIdx.x; v < n16 + n32; v += gridDim.x) {
    const ScanTile T = v < n16 ? p.t16[v] : p.t32[v - n16];
    if (T.grow0 != __ldg(p.list_off + T.list)) continue;  // a later chunk: its first chunk wrote the pairs
    const float4* __restrict__ c = reinterpret_cast<const float4*>(p.centroids + (size_t)T.list * d);
    float4 cv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nb) cv[j] = __ldg(c + j * 32 + lane);
    const double rm = (double)__ldg(p.rmax + T.list);
    for (int g = warp; g < T.nq; g += 8) {
      const int pos = T.qoff + g;
      const float4* __restrict__ q = reinterpret_cast<const float4*>(p.queries + (size_t)__ldg(p.list_q + pos) * d);
      float4 qv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < nb) qv[j] = __ldg(q + j * 32 + lane);
      uint2* o1 = reinterpret_cast<uint2*>(out + (size_t)(2 * pos) * d);
      uint2* o2 = reinterpret_cast<uint2*>(out + (size_t)(2 * pos + 1) * d);
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= nb) break;
        const float qa[4] = {qv[j].x, qv[j].y, qv[j].z, qv[j].w}, ca[4] = {cv[j].x, cv[j].y, cv[j].z, cv[j].w};
        __nv_bfloat16 h1[4], h2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double a = (double)qa[e] - (double)ca[e];  // exact
          s = fma(a, a, s);
          const float pf = __double2float_rn(a);
          h1[e] = __float2bfloat16_rn(pf);
          h2[e] = __float2bfloat16_rn(pf - __bfloat162float(h1[e]));
        }
        o1[j * 32 + lane] = *reinterpret_cast<const uint2*>(h1);
        o2[j * 32 + lane] = *reinterpret_cast<const uint2*>(h2);
      }
      s = warp_sum_f64(s);
      if (lane == 0) {
        const double u = (double)kUnit;
        const double eps = 2.0 * (double)p.gamma * sqrt(s) * rm + 32.0 * u * (s + rm * rm) + 1e-30;
        p.pqn[pos] = __double2float_rd(s - eps);
      }
    }
  }
}

}  // namespace

cudaError_t launch_resid_build(const float* arena, const long long* res_row0, const long long* list_off,
                               const float* centroids, int nlist, int d, void* r1, float* rnorm, float* rmax,
                               cudaStream_t s) {
  if (d % 32 != 0 || d > 32 * kMaxPerLane || nlist <= 0) return cudaErrorInvalidValue;
  resid_build_kernel<<<nlist, 256, 0, s>>>(arena, res_row0, list_off, centroids, d,
                                           reinterpret_cast<__nv_bfloat16*>(r1), rnorm, rmax);
  return cudaGetLastError();
}

cudaError_t launch_pair_operand(const PairParams& p, int grid, cudaStream_t s) {
  if (p.d % 128 != 0 || p.d > 1024) return cudaErrorInvalidValue;  // (the residual scan needs d % 64 == 0)
  return launch_k(pair_operand_kernel, dim3(grid), dim3(256), 0, s, p);
}

}  // namespace rd
