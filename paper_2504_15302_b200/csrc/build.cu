// build.cu — N10 index materialisation on the device (sm_100a): the synthetic
// knowledge base is generated straight into the HBM arena from (seed, id), so
// 30-300 GB never cross the host link; plus row norms and max-norm reductions.
#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

__global__ void gen_centroids_kernel(float* __restrict__ C, long long total, int d, uint64_t sc) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    C[i] = unif(sc, (uint64_t)i);
}

// one warp per row: x[r][t] = c[a(id)][t] + sigma * f(s_x, id*d + t), f32 round-to-nearest
__global__ void gen_vectors_kernel(float* __restrict__ X, const long long* __restrict__ ids,
                                   long long n, int d, int nlist, const float* __restrict__ C,
                                   uint64_t sa, uint64_t sx, float sigma) {
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
    const long long id = ids[r];
    const int a = (int)(splitmix_at(sa, (uint64_t)id) % (uint64_t)nlist);
    const float* c = C + (size_t)a * d;
    float* x = X + (size_t)r * d;
    for (int t = lane; t < d; t += 32) {
      const float noise = __fmul_rn(sigma, unif(sx, (uint64_t)id * d + t));
      x[t] = __fadd_rn(__ldg(c + t), noise);
    }
  }
}

__global__ void row_norms_kernel(const float* __restrict__ X, long long n, int d, float* __restrict__ out) {
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
    const float* x = X + (size_t)r * d;
    double s = 0.0;
    for (int t = lane; t < d; t += 32) {
      const double v = x[t];
      s += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = (float)s;
  }
}

__global__ void max_f32_kernel(const float* __restrict__ v, long long n, float* out) {
  float m = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = fmaxf(m, v[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));  // m >= 0
}

// one CTA per list: row_list[off[l] .. off[l+1]) = l
__global__ void row_list_kernel(const long long* __restrict__ off, int* __restrict__ row_list) {
  const int l = blockIdx.x;
  const long long r0 = off[l], r1 = off[l + 1];
  for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) row_list[r] = l;
}

}  // namespace

cudaError_t launch_row_list(const long long* off, int nlist, int* row_list, cudaStream_t s) {
  if (nlist == 0) return cudaSuccess;
  row_list_kernel<<<nlist, 256, 0, s>>>(off, row_list);
  return cudaGetLastError();
}

cudaError_t launch_gen_centroids(float* C, int nlist, int d, uint64_t sc, cudaStream_t s) {
  const long long total = (long long)nlist * d;
  gen_centroids_kernel<<<(unsigned)min((total + 255) / 256, 148LL * 32), 256, 0, s>>>(C, total, d, sc);
  return cudaGetLastError();
}
cudaError_t launch_gen_vectors(float* X, const long long* ids, long long n, int d, int nlist,
                               const float* C, uint64_t sa, uint64_t sx, float sigma, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  gen_vectors_kernel<<<148 * 16, 256, 0, s>>>(X, ids, n, d, nlist, C, sa, sx, sigma);
  return cudaGetLastError();
}
cudaError_t launch_row_norms(const float* X, long long n, int d, float* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  row_norms_kernel<<<148 * 16, 256, 0, s>>>(X, n, d, out);
  return cudaGetLastError();
}
cudaError_t launch_max_f32(const float* v, long long n, float* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float), s);
  if (e != cudaSuccess || n == 0) return e;
  max_f32_kernel<<<148 * 4, 256, 0, s>>>(v, n, out);
  return cudaGetLastError();
}

}  // namespace rd
