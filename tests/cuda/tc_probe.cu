// tc_probe.cu — TEST INFRASTRUCTURE: exercises the tcgen05 building blocks the
// tensor-core scan uses (SW128 K-major smem descriptors, kind::tf32 SS and TS
// MMAs, TMEM alloc/ld/st, commit-to-mbarrier) on one 128 x 32 x K problem so
// a unit test can compare them against numpy.
#include "../../paper_2504_15302_b200/csrc/rd_device.cuh"

using namespace rd;

// A: 128 x K (K % 32 == 0, K <= 128), B: 32 x K. Outputs:
//   D1 [128 x 32] = A . B^T            (SS, A and B from smem)
//   D2 [128 x 16] = A . B[0:16]^T      (TS, A from TMEM, written by tcgen05.st)
__global__ void __launch_bounds__(128, 1) tc_probe_kernel(const float* A, const float* B, int K, float* D1, float* D2) {
  extern __shared__ unsigned char dyn[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  unsigned char (*sa)[128 * 128] = reinterpret_cast<unsigned char (*)[128 * 128]>(base);
  unsigned char (*sb)[32 * 128] = reinterpret_cast<unsigned char (*)[32 * 128]>(base + 4 * 128 * 128);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nks = K / 32;
  for (int i = tid; i < 128 * K / 4; i += 128) {
    const int r = i / (K / 4), c4 = i % (K / 4), k = c4 * 4, ks = k >> 5, g = (k & 31) >> 2;
    *reinterpret_cast<float4*>(&sa[ks][r * 128 + ((g ^ (r & 7)) << 4)]) = reinterpret_cast<const float4*>(A)[i];
  }
  for (int i = tid; i < 32 * K / 4; i += 128) {
    const int r = i / (K / 4), c4 = i % (K / 4), k = c4 * 4, ks = k >> 5, g = (k & 31) >> 2;
    *reinterpret_cast<float4*>(&sb[ks][r * 128 + ((g ^ (r & 7)) << 4)]) = reinterpret_cast<const float4*>(B)[i];
  }
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  // A into TMEM columns [128, 128 + K) of this thread's lane (row = tid)
  for (int k0 = 0; k0 < K; k0 += 8) {
    uint32_t v[8];
    for (int e = 0; e < 8; ++e) v[e] = __float_as_uint(A[tid * K + k0 + e]);
    tmem_st8(tm + ((uint32_t)(warp * 32) << 16) + 128 + k0, v);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t id1 = idesc_tf32(128, 32), id2 = idesc_tf32(128, 16);
    for (int ks = 0; ks < nks; ++ks) {
      const uint64_t ad = umma_desc_sw128(sa[ks]), bd = umma_desc_sw128(sb[ks]);
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (ks | kk) != 0;
        mma_tf32_ss(tm, ad + (uint64_t)(kk * 2), bd + (uint64_t)(kk * 2), id1, acc);
        mma_tf32_ts(tm + 64, tm + 128 + ks * 32 + kk * 8, bd + (uint64_t)(kk * 2), id2, acc);
      }
    }
    tc_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r0[16], r1[16], r2[16];
  const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
  RD_TMEM_LD16(ta, r0);
  RD_TMEM_LD16(ta + 16, r1);
  RD_TMEM_LD16(ta + 64, r2);
  tmem_ld_wait();
  for (int j = 0; j < 16; ++j) {
    D1[tid * 32 + j] = __uint_as_float(r0[j]);
    D1[tid * 32 + 16 + j] = __uint_as_float(r1[j]);
    D2[tid * 16 + j] = __uint_as_float(r2[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 256);
  }
}

extern "C" int tc_probe(const float* hA, const float* hB, int K, float* hD1, float* hD2) {
  float *A, *B, *D1, *D2;
  cudaMalloc(&A, 128 * K * 4);
  cudaMalloc(&B, 32 * K * 4);
  cudaMalloc(&D1, 128 * 32 * 4);
  cudaMalloc(&D2, 128 * 16 * 4);
  cudaMemcpy(A, hA, 128 * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 32 * K * 4, cudaMemcpyHostToDevice);
  const int smem = 1024 + 4 * 128 * 128 + 4 * 32 * 128;
  cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc_probe_kernel<<<1, 128, smem>>>(A, B, K, D1, D2);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD1, D1, 128 * 32 * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hD2, D2, 128 * 16 * 4, cudaMemcpyDeviceToHost);
  cudaFree(A);
  cudaFree(B);
  cudaFree(D1);
  cudaFree(D2);
  return (int)e;
}

// MMA timing probe: n back-to-back MMAs (mode 0: SS N=32, 1: TS N=16, 2: SS N=32 alternating
// two accumulators, 3: SS N=256) then commit+wait; returns clock64 cycles.
__global__ void __launch_bounds__(128, 1) tc_timing_kernel(int mode, int n, long long* out) {
  extern __shared__ unsigned char dyn[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 * 128 + 256 * 128) / 4; i += 128) reinterpret_cast<float*>(base)[i] = 1.0f;
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint64_t ad = umma_desc_sw128(base), bd = umma_desc_sw128(base + 128 * 128);
    const uint32_t id32 = idesc_tf32(128, 32), id16 = idesc_tf32(128, 16), id256 = idesc_tf32(128, 256);
    long long t0 = clock64();
    if (mode >= 16) {  // bf16 TS patterns of the scan kernel: (N=64, N=32) pairs, commit every 4 MMAs?
      __shared__ uint64_t bar2;
      mbar_init(&bar2, 1);
      fence_mbar_init();
      const uint32_t ia = idesc_bf16(128, 64), ib = idesc_bf16(128, 32);
      for (int i = 0; i < n; i += 4) {
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          mma_bf16_ts(tm, tm + 256 + kk * 8, bd + kk * 2, mode == 19 ? ib : ia, 1);
          mma_bf16_ts(tm + 64, tm + 256 + 16 + kk * 8, bd + kk * 2, ib, 1);
        }
        if (mode == 17) tc_commit(&bar2);
      }
      n = 0;
    }
    if (mode >= 10 && mode < 16) {  // straight-line issue: 8 unrolled MMAs per iteration, constant descriptors
      const uint32_t idm = mode == 10 ? id32 : (mode == 11 ? id256 : mode == 13 ? idesc_tf32(64, 256) : mode == 14 ? idesc_tf32(64, 192) : mode == 15 ? idesc_tf32(64, 128) : id16);
      for (int i = 0; i < n; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (mode == 12) mma_tf32_ts(tm + 64, tm + 256 + (j & 3) * 8, bd + (j & 3) * 2, idm, 1);
          else mma_tf32_ss(tm, ad + (j & 3) * 2, bd + (j & 3) * 2, idm, 1);
        }
      }
      n = 0;
    }
    for (int i = 0; i < n; ++i) {
      const uint32_t kk = i & 3;
      if (mode == 0) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, id32, i > 0);
      else if (mode == 1) mma_tf32_ts(tm + 64, tm + 256 + kk * 8, bd + kk * 2, id16, i > 0);
      else if (mode == 2) mma_tf32_ss(tm + (i & 1) * 32, ad + kk * 2, bd + kk * 2, id32, i > 1);
      else if (mode == 3) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, id256, i > 0);
      else if (mode == 4) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, idesc_tf32(64, 256), i > 0);
      else if (mode == 5) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, idesc_tf32(64, 128), i > 0);
      else if (mode == 6) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, idesc_tf32(128, 128), i > 0);
      else if (mode == 7) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, idesc_tf32(64, 64), i > 0);
      else if (mode == 8) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, idesc_tf32(128, 64), i > 0);
      else mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, idesc_tf32(64, 32), i > 0);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

extern "C" long long tc_timing(int mode, int n) {
  long long* d;
  long long h = -1;
  cudaMalloc(&d, 8);
  const int smem = 1024 + 128 * 128 + 256 * 128;
  cudaFuncSetAttribute(tc_timing_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc_timing_kernel<<<1, 128, smem>>>(mode, n, d);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h;
}

// M=64 accumulator layout probe: D[64 x 32] = A[64 x 32] . B[32 x 32]^T (tf32, SS); dumps all
// 128 TMEM lanes x 32 columns so the test can locate where row i of D lives.
__global__ void __launch_bounds__(128, 1) tc_m64_kernel(const float* A, const float* B, float* dump) {
  extern __shared__ unsigned char dyn[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  unsigned char* sa = base;             // 64 rows x 128 B
  unsigned char* sb = base + 64 * 128;  // 32 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 8; i += 128) {
    const int r = i / 8, g = i % 8;
    *reinterpret_cast<float4*>(sa + r * 128 + ((g ^ (r & 7)) << 4)) = reinterpret_cast<const float4*>(A)[i];
  }
  for (int i = tid; i < 32 * 8; i += 128) {
    const int r = i / 8, g = i % 8;
    *reinterpret_cast<float4*>(sb + r * 128 + ((g ^ (r & 7)) << 4)) = reinterpret_cast<const float4*>(B)[i];
  }
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    // zero-initialise all 128 lanes x 32 columns first via one accumulate=0 MMA would only touch
    // the M=64 footprint, so the dump also shows which lanes are untouched (left as garbage)
    const uint64_t ad = umma_desc_sw128(sa), bd = umma_desc_sw128(sb);
    for (int kk = 0; kk < 4; ++kk) mma_tf32_ss(tm, ad + kk * 2, bd + kk * 2, idesc_tf32(64, 32), kk > 0);
    tc_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r0[16], r1[16];
  const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
  RD_TMEM_LD16(ta, r0);
  RD_TMEM_LD16(ta + 16, r1);
  tmem_ld_wait();
  for (int j = 0; j < 16; ++j) {
    dump[tid * 32 + j] = __uint_as_float(r0[j]);
    dump[tid * 32 + 16 + j] = __uint_as_float(r1[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 64);
  }
}

extern "C" int tc_m64(const float* hA, const float* hB, float* hdump) {
  float *A, *B, *D;
  cudaMalloc(&A, 64 * 32 * 4);
  cudaMalloc(&B, 32 * 32 * 4);
  cudaMalloc(&D, 128 * 32 * 4);
  cudaMemset(D, 0xff, 128 * 32 * 4);
  cudaMemcpy(A, hA, 64 * 32 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 32 * 32 * 4, cudaMemcpyHostToDevice);
  const int smem = 1024 + 96 * 128;
  cudaFuncSetAttribute(tc_m64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc_m64_kernel<<<1, 128, smem>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hdump, D, 128 * 32 * 4, cudaMemcpyDeviceToHost);
  cudaFree(A);
  cudaFree(B);
  cudaFree(D);
  return (int)e;
}

// TMA gather4 probe: rows {r0..r3}, columns [c0, c0+32) of a [R x C] fp32 tensor into a
// 128B-swizzled smem box; threads un-swizzle and return the 4 x 32 values.
__global__ void tc_gather4_kernel(const __grid_constant__ CUtensorMap map, int c0, int4 rows, float* out) {
  __shared__ __align__(1024) unsigned char buf[1024];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 512);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf)),
        "l"(&map), "r"(c0), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w), "r"(smem_u32(&bar))
        : "memory");
  }
  mbar_wait(&bar, 0);
  const int t = threadIdx.x;  // 128 threads: row t/32, col t%32
  const int r = t >> 5, c = t & 31, g = c >> 2, e = c & 3;
  out[t] = reinterpret_cast<const float*>(buf + r * 128 + ((g ^ (r & 7)) << 4))[e];
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int tc_gather4(const float* hX, int R, int Ccols, int c0, const int* rows, float* hout) {
  float *X, *O;
  cudaMalloc(&X, (size_t)R * Ccols * 4);
  cudaMalloc(&O, 128 * 4);
  cudaMemcpy(X, hX, (size_t)R * Ccols * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)Ccols, (cuuint64_t)R};
  cuuint64_t str[1] = {(cuuint64_t)Ccols * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult cr = ((EncFn)fp)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return 1000 + (int)cr;
  tc_gather4_kernel<<<1, 128>>>(m, c0, make_int4(rows[0], rows[1], rows[2], rows[3]), O);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hout, O, 128 * 4, cudaMemcpyDeviceToHost);
  cudaFree(X);
  cudaFree(O);
  return (int)e;
}

// kind::f16 (bf16 inputs, fp32 accumulate) accumulation probe: D[128 x 32] = C + A . B^T over
// K (K % 64 == 0, K <= 512), issued as K / 16 SS MMAs into ONE accumulator, exactly the way the
// scan and the coarse GEMM chain their K steps. A / B are bf16 bit patterns, row-major; C is the
// initial accumulator (stored to TMEM with tcgen05.st; has_c = 0 starts from the first product).
// The test uses it to measure the accumulator's rounding error on adversarial operands.
__global__ void __launch_bounds__(128, 1) tc_bf16_acc_kernel(const uint16_t* A, const uint16_t* B, const float* C,
                                                             int has_c, int K, float* D, int fp16) {
  extern __shared__ unsigned char dyn[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dyn) + 1023) & ~uintptr_t(1023));
  unsigned char* sa = base;                       // [K/64][128 rows x 128 B]
  unsigned char* sb = base + (K / 64) * 128 * 128;  // [K/64][32 rows x 128 B]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // 16 B chunks (8 bf16): element k of row r -> slab k / 64, chunk (k % 64) / 8 swizzled by r % 8
  for (int i = tid; i < 128 * K / 8; i += 128) {
    const int r = i / (K / 8), k = (i % (K / 8)) * 8, ks = k >> 6, g = (k & 63) >> 3;
    *reinterpret_cast<uint4*>(sa + ks * 128 * 128 + r * 128 + ((g ^ (r & 7)) << 4)) =
        reinterpret_cast<const uint4*>(A)[i];
  }
  for (int i = tid; i < 32 * K / 8; i += 128) {
    const int r = i / (K / 8), k = (i % (K / 8)) * 8, ks = k >> 6, g = (k & 63) >> 3;
    *reinterpret_cast<uint4*>(sb + ks * 32 * 128 + r * 128 + ((g ^ (r & 7)) << 4)) =
        reinterpret_cast<const uint4*>(B)[i];
  }
  fence_proxy_async();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
  if (has_c) {
    uint32_t v[16];
    for (int h = 0; h < 2; ++h) {
      for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(C[tid * 32 + h * 16 + j]);
      tmem_st16(ta + h * 16, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t id = fp16 ? idesc_f16(128, 32) : idesc_bf16(128, 32);  // fp16: the residual scan's operands
    for (int ks = 0; ks < K / 64; ++ks) {
      const uint64_t ad = umma_desc_sw128(sa + ks * 128 * 128), bd = umma_desc_sw128(sb + ks * 32 * 128);
      for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tm, ad + kk * 2, bd + kk * 2, id, (has_c | ks | kk) != 0);
    }
    tc_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r0[16], r1[16];
  RD_TMEM_LD16(ta, r0);
  RD_TMEM_LD16(ta + 16, r1);
  tmem_ld_wait();
  for (int j = 0; j < 16; ++j) {
    D[tid * 32 + j] = __uint_as_float(r0[j]);
    D[tid * 32 + 16 + j] = __uint_as_float(r1[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 32);
  }
}

static int tc_acc_impl(const uint16_t* hA, const uint16_t* hB, const float* hC, int has_c, int K, float* hD, int fp16) {
  if (K % 64 != 0 || K <= 0 || K > 512) return -1;
  uint16_t *A, *B;
  float *C, *D;
  cudaMalloc(&A, 128 * K * 2);
  cudaMalloc(&B, 32 * K * 2);
  cudaMalloc(&C, 128 * 32 * 4);
  cudaMalloc(&D, 128 * 32 * 4);
  cudaMemcpy(A, hA, 128 * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, 32 * K * 2, cudaMemcpyHostToDevice);
  if (has_c) cudaMemcpy(C, hC, 128 * 32 * 4, cudaMemcpyHostToDevice);
  const int smem = 1024 + (K / 64) * (128 + 32) * 128;
  cudaFuncSetAttribute(tc_bf16_acc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tc_bf16_acc_kernel<<<1, 128, smem>>>(A, B, C, has_c, K, D, fp16);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, 128 * 32 * 4, cudaMemcpyDeviceToHost);
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  cudaFree(D);
  return (int)e;
}

extern "C" int tc_bf16_acc(const uint16_t* hA, const uint16_t* hB, const float* hC, int has_c, int K, float* hD) {
  return tc_acc_impl(hA, hB, hC, has_c, K, hD, 0);
}
// the same probe with fp16 operands (kind::f16, a/b format F16)
extern "C" int tc_f16_acc(const uint16_t* hA, const uint16_t* hB, const float* hC, int has_c, int K, float* hD) {
  return tc_acc_impl(hA, hB, hC, has_c, K, hD, 1);
}
