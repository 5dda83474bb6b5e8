// Microbenchmark: HBM read bandwidth of the scan's stage-load patterns on sm_100a.
//   strided : the scan today — per stage two 3D TMA boxes {64 bf16, 1 part, 128 rows} over a
//             [rows][2][768] bf16 arena (128 B from each of 128 rows, row pitch 3072 B)
//   bulk    : the same bytes stored stage-contiguous — one 32 KiB cp.async.bulk per stage
//   ldg     : plain float4 grid-stride loads (reference)
// Persistent CTAs (one per SM), a ring of `stages` 32 KiB slots, a consumer warp that only
// waits and releases. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2504_15302_b200/csrc tools/micro/bw.cu -o tools/micro/bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "rd_device.cuh"

using namespace rd;

constexpr int kRows = 128, kD = 768, kSlices = kD / 64;
constexpr int kStageBytes = 2 * kRows * 128;  // x1 + x2 tiles of one 64-dim slice

template <bool kBulk>
__global__ void __launch_bounds__(64, 1) ring_kernel(const __grid_constant__ CUtensorMap map, const char* arena,
                                                     long long ntiles, int stages, unsigned* counter,
                                                     unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      uint32_t u = 0;
      for (;;) {
        const long long t = atomicAdd(counter, 1u);
        if (t >= ntiles) break;
        for (int ks = 0; ks < kSlices; ++ks, ++u) {
          const int s = u % stages;
          mbar_wait(&empty[s], ((u / stages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], kStageBytes);
          const uint32_t dst = smem_u32(ring + (size_t)s * kStageBytes);
          if constexpr (kBulk) {
            bulk_g2s(ring + (size_t)s * kStageBytes, arena + ((size_t)t * kSlices + ks) * kStageBytes, kStageBytes,
                     &full[s]);
          } else {
            tma_load_3d_u32(dst, &map, ks * 64, 0, (int)(t * kRows), &full[s]);
            tma_load_3d_u32(dst + kRows * 128, &map, ks * 64, 1, (int)(t * kRows), &full[s]);
          }
        }
      }
      // drain: tell the consumer how many stages there were
      sink[blockIdx.x * 2] = u;
    }
  } else {
    if (lane == 0) {
      uint32_t u = 0;
      unsigned long long acc = 0;
      for (;;) {
        const int s = u % stages;
        // stop once the producer has finished and every issued stage was consumed
        volatile unsigned long long* done = sink + blockIdx.x * 2;
        while (true) {
          uint32_t ok;
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
              : "=r"(ok)
              : "r"(smem_u32(&full[s])), "r"((u / stages) & 1)
              : "memory");
          if (ok) break;
          if (*done != ~0ull && u >= *done) goto out;
        }
        acc += ring[(size_t)s * kStageBytes + (u & 127)];
        mbar_arrive(&empty[s]);
        ++u;
      }
    out:
      sink[blockIdx.x * 2 + 1] = acc;
    }
  }
}

__global__ void ldg_kernel(const float4* a, long long n4, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = __ldg(a + i);
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.x;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const long long rows = 10'000'000LL / kRows * kRows;  // C2: 10M rows x 3072 B = 30.7 GB
  const long long ntiles = rows / kRows;
  const size_t bytes = (size_t)rows * kD * 4;
  char* arena;
  if (cudaMalloc(&arena, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(arena, 1, bytes);
  unsigned* counter;
  unsigned long long* sink;
  float* out;
  cudaMalloc(&counter, 4);
  cudaMalloc(&sink, 16 * 148 * 8);
  cudaMalloc(&out, 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  std::memset(&map, 0, sizeof map);
  cuuint64_t dims[3] = {(cuuint64_t)kD, 2, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)kD * 2, (cuuint64_t)kD * 4};
  cuuint32_t box[3] = {64, 1, kRows};
  cuuint32_t estr[3] = {1, 1, 1};
  reinterpret_cast<EncodeFn>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, arena, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int stages : {2, 3, 4, 5, 6}) {
    const size_t smem = (size_t)stages * kStageBytes + 1024;
    cudaFuncSetAttribute(ring_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(ring_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int bulk = 0; bulk < 2; ++bulk) {
      float best = 1e9f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaMemset(counter, 0, 4);
        cudaMemset(sink, 0xff, 16 * 148 * 8);
        cudaEventRecord(e0);
        if (bulk)
          ring_kernel<true><<<sms, 64, smem>>>(map, arena, ntiles, stages, counter, sink);
        else
          ring_kernel<false><<<sms, 64, smem>>>(map, arena, ntiles, stages, counter, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) best = ms < best ? ms : best;
      }
      cudaError_t err = cudaGetLastError();
      printf("%-8s stages=%2d  %.3f ms  %.1f GB/s  %s\n", bulk ? "bulk" : "strided", stages, best, bytes / best / 1e6,
             cudaGetErrorString(err));
    }
  }
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    float best = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      ldg_kernel<<<blocks, 512>>>(reinterpret_cast<const float4*>(arena), (long long)(bytes / 16), out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) best = ms < best ? ms : best;
    }
    printf("ldg      blocks=%d  %.3f ms  %.1f GB/s\n", blocks, best, bytes / best / 1e6);
  }
  return 0;
}
