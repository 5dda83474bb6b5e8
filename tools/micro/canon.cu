// Microbenchmark: cycles of the canonical exact distance (rd_device.cuh) and the fp32 seed distance on
// rows staged in shared memory, as the small-batch merge / select kernels run them (one CTA of 256
// threads, 32 candidates x 8 lanes, d = 768), against restructured variants.
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2504_15302_b200/csrc/rd_device.cuh"

using namespace rd;
constexpr int D = 768;
constexpr int DS = D + D / 2 + kStagePad;  // split3 staged stride (floats)

// the canonical sum with q in fp64 smem and x decoded from a split3 staged row, 16 deep
template <int kDepth>
__device__ __forceinline__ float canon_split3_qd(const double* qd, const __nv_bfloat16* x12, const __nv_bfloat16* x3,
                                                 int d, int j, int cnt) {
  double s = 0.0;
  int t = j;
  for (; t + 8 * (kDepth - 1) < cnt; t += 8 * kDepth) {
    float xv[kDepth];
    double qv[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const int u = t + 8 * i;
      xv[i] = __fadd_rn(__fadd_rn(__bfloat162float(x12[u]), __bfloat162float(x12[d + u])), __bfloat162float(x3[u]));
      qv[i] = qd[u];
    }
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const double df = __dsub_rn(qv[i], (double)xv[i]);
      s = __dadd_rn(s, __dmul_rn(df, df));
    }
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}

__global__ void k(const float* src, float* out, long long* cyc) {
  extern __shared__ __align__(16) float dyn[];
  float* q = dyn;                                  // [D]
  double* qd = reinterpret_cast<double*>(q + D);   // [D]
  float* st = reinterpret_cast<float*>(qd + D);    // [32][DS]
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    q[i] = src[i];
    qd[i] = src[i];
  }
  for (int i = threadIdx.x; i < 32 * DS; i += blockDim.x) st[i] = src[i % 4096] * 0.5f;
  __syncthreads();
  const int c = threadIdx.x >> 3, j8 = threadIdx.x & 7;
  const float* slot = st + c * DS;
  const RowRef x{nullptr, reinterpret_cast<const __nv_bfloat16*>(slot), reinterpret_cast<const __nv_bfloat16*>(slot + D)};
  float acc = 0.f;
  long long t[8];
  __syncthreads();
  t[0] = clock64();
  acc += exact_l2_group8_row(q, x, D, j8, D);  // merge kStage (current)
  __syncthreads();
  t[1] = clock64();
  acc += l2_group8_f32_row(q, x, D, j8);  // select seed (current, kDepth 1)
  __syncthreads();
  t[2] = clock64();
  acc += l2_group8_f32_row<8>(q, x, D, j8);  // seed, 8 deep
  __syncthreads();
  t[3] = clock64();
  acc += canon_split3_qd<8>(qd, x.x12, x.x3, D, j8, D);
  __syncthreads();
  t[4] = clock64();
  acc += canon_split3_qd<16>(qd, x.x12, x.x3, D, j8, D);
  __syncthreads();
  t[5] = clock64();
  acc += exact_l2_group8_qd(qd, slot, D, j8);  // fp32 row (select's ambiguous centroids)
  __syncthreads();
  t[6] = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0)
    for (int i = 0; i < 6; ++i) cyc[i] = t[i + 1] - t[i];
}

int main() {
  float* src;
  float* o;
  long long* c;
  cudaMalloc(&src, 4096 * 4);
  cudaMalloc(&o, 1024 * 4);
  cudaMallocManaged(&c, 64);
  cudaMemset(src, 0, 4096 * 4);
  const size_t smem = D * 4 + D * 8 + 32 * DS * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) k<<<1, 256, smem>>>(src, o, c);
  cudaError_t e = cudaDeviceSynchronize();
  const char* nm[6] = {"canon split3 row (merge, current)", "f32 seed kDepth1 (select, current)",
                       "f32 seed kDepth8", "canon split3 qd depth8", "canon split3 qd depth16",
                       "canon f32 row qd (select ambiguous)"};
  printf("err=%s\n", cudaGetErrorString(e));
  for (int i = 0; i < 6; ++i) printf("%-40s %6lld cycles\n", nm[i], c[i]);
  return 0;
}
