// resid.cu — the residual store's build (sm_100a).
//
// The residual store keeps the fp32 rows (exact rerank, seeding, fallback) plus one bf16 plane
// r1 = bf16(x - c_l) per resident row, c_l the row's list centroid: the tensor-core scan reads
// 2 B per element instead of the split3 store's 4 (x1 | x2). With a = q - c, r = x - c:
//   ||q - x||^2 = ||a||^2 - 2 a.r + ||r||^2,   a.r1 = q.r1 - c.r1,
// so the scan keeps the split3 scan's B operand (q1; q2) and computes
//   key = (||a||^2 - eps) + (||r||^2 + 2 c.r1) - 2 r1.(q1 + q2)
// with ||a||^2 from the coarse stage (qnorm + Dc) and the row constant built here in fp64.
// |exact - (key + eps)| <= eps (scan_tc.cu resid_pair_term): the dominant term is r1's rounding,
// 2^-8 ||q - c|| max ||x - c||, small because rows sit near their centroid — so every key is a lower
// bound on the row's exact distance and the scan's pruning, the merge's certification and the
// seeding threshold need no error term of their own. Exactness is every store's: exact rerank of
// the candidates from the fp32 rows, certification, exact fallback.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

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
                                                          uint16_t* __restrict__ r1, float* __restrict__ rnorm,
                                                          float* __restrict__ rmax, bool half, unsigned* ovf) {
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
      uint16_t* o = r1 + (size_t)(sr0 + i) * d;
      double s = 0.0, t = 0.0;  // ||r||^2, c . r1
      unsigned bad = 0;
#pragma unroll
      for (int j = 0; j < kMaxPerLane; ++j) {
        if (j >= per) break;
        const double r = (double)x[j * 32 + lane] - c[j];
        double rv;
        if (half) {
          const __half h = __double2half(r);
          rv = (double)__half2float(h);
          bad += fabs(r) >= 65504.0;
          o[j * 32 + lane] = __half_as_ushort(h);
        } else {
          const __nv_bfloat16 h = __double2bfloat16(r);
          rv = (double)__bfloat162float(h);
          o[j * 32 + lane] = __bfloat16_as_ushort(h);
        }
        s = fma(r, r, s);
        t = fma(c[j], rv, t);
      }
      s = warp_sum_f64(s);
      t = warp_sum_f64(t);
      if (lane == 0) rnorm[g0 + i] = (float)(s + 2.0 * t);
      if (bad && ovf) atomicAdd(ovf, bad);
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

}  // namespace

cudaError_t launch_resid_build(const float* arena, const long long* res_row0, const long long* list_off,
                               const float* centroids, int nlist, int d, void* r1, float* rnorm, float* rmax,
                               cudaStream_t s, bool half, unsigned* ovf) {
  if (d % 32 != 0 || d > 32 * kMaxPerLane || nlist <= 0) return cudaErrorInvalidValue;
  resid_build_kernel<<<nlist, 256, 0, s>>>(arena, res_row0, list_off, centroids, d, reinterpret_cast<uint16_t*>(r1),
                                           rnorm, rmax, half, ovf);
  return cudaGetLastError();
}

}  // namespace rd
