// train.cu — IVF training helpers for rd_index_build (sm_100a): the deterministic k-means update
// and the list-order layout. Assignment reuses the search's coarse path (index.cu, rd_index_build).
//
// Determinism: rows are stably sorted by cluster (CUB radix sort keeps equal keys in input order,
// i.e. ascending row), and each (cluster, dimension) sum runs sequentially in that order in fp64,
// so the centroids equal the oracle's (oracle/rd_oracle.c, rd_index_build) bit for bit.
#include <cub/device/device_radix_sort.cuh>

#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

__global__ void iota_kernel(int* __restrict__ v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[i] = (int)i;
}

__global__ void histogram_kernel(const int* __restrict__ keys, long long n, unsigned* __restrict__ counts) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    atomicAdd(counts + keys[i], 1u);
}

// one warp per (cluster, 32-dim slice): lane t sums dimension t over the cluster's rows in order
__global__ void centroid_update_kernel(const float* __restrict__ X, const int* __restrict__ rows,
                                       const long long* __restrict__ seg, int d, float* __restrict__ C) {
  const int l = blockIdx.x, t = blockIdx.y * 32 + threadIdx.x;
  const long long r0 = seg[l], r1 = seg[l + 1];
  if (r1 == r0 || t >= d) return;  // empty cluster keeps its centroid
  double s = 0.0;
  long long r = r0;
  for (; r + 8 <= r1; r += 8) {  // loads 8 rows ahead of the strictly sequential sum
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(X + (size_t)__ldg(rows + r + u) * d + t);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = __dadd_rn(s, (double)v[u]);
  }
  for (; r < r1; ++r) s = __dadd_rn(s, (double)__ldg(X + (size_t)__ldg(rows + r) * d + t));
  C[(size_t)l * d + t] = __double2float_rn(__ddiv_rn(s, (double)(r1 - r0)));
}

// dst row i = src row idx[i] (one warp per row, float4)
__global__ void gather_rows_kernel(const float* __restrict__ src, const int* __restrict__ idx, long long count, int d,
                                   float* __restrict__ dst) {
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31, d4 = d / 4;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; i < count; i += warps) {
    const float4* s = reinterpret_cast<const float4*>(src + (size_t)idx[i] * d);
    float4* o = reinterpret_cast<float4*>(dst + (size_t)i * d);
    for (int c = lane; c < d4; c += 32) o[c] = __ldg(s + c);
  }
}

__global__ void gather_ids_kernel(const long long* __restrict__ ids, const int* __restrict__ idx, long long count,
                                  long long* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    out[i] = ids ? ids[idx[i]] : (long long)idx[i];
}

}  // namespace

cudaError_t launch_iota(int* v, long long n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  iota_kernel<<<148 * 8, 256, 0, s>>>(v, n);
  return cudaGetLastError();
}

cudaError_t launch_histogram(const int* keys, long long n, unsigned* counts, int nbins, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(unsigned) * (size_t)nbins, s);
  if (e != cudaSuccess || n == 0) return e;
  histogram_kernel<<<148 * 8, 256, 0, s>>>(keys, n, counts);
  return cudaGetLastError();
}

cudaError_t sort_pairs(const int* keys_in, int* keys_out, const int* vals_in, int* vals_out, long long n, int end_bit,
                       void* temp, size_t* temp_bytes, cudaStream_t s) {
  return cub::DeviceRadixSort::SortPairs(temp, *temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)n, 0, end_bit,
                                         s);
}

cudaError_t launch_centroid_update(const float* X, const int* rows, const long long* seg, int nlist, int d, float* C,
                                   cudaStream_t s) {
  centroid_update_kernel<<<dim3(nlist, (d + 31) / 32), 32, 0, s>>>(X, rows, seg, d, C);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const float* src, const int* idx, long long count, int d, float* dst, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  gather_rows_kernel<<<148 * 16, 256, 0, s>>>(src, idx, count, d, dst);
  return cudaGetLastError();
}

cudaError_t launch_gather_ids(const long long* ids, const int* idx, long long count, long long* out, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  gather_ids_kernel<<<148 * 8, 256, 0, s>>>(ids, idx, count, out);
  return cudaGetLastError();
}

}  // namespace rd
