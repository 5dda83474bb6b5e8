// coarse_tc.cu — N1 on the tensor cores: Dc[b][j] = ||c_j||^2 - 2 q_b.c_j (sm_100a).
//
// bf16x3 split on both sides (q = q1 + q2, c = c1 + c2, each bf16 RN; the centroid split is
// built once with the index): per 64-dim K slice, a TMA pair brings A = q1 / q2 (128 queries,
// K-major, 128 B swizzle) and B = [c1 ; c2] (2 x 128 centroids), then per 16-dim K step
//   MMA_a: D_a[128 x 256] += q1 . [c1 ; c2]^T      (kind::f16, N = 256)
//   MMA_b: D_b[128 x 128] += q2 . c1^T             (N = 128)
// q.c = D_a[c1] + D_a[c2] + D_b (missing q2.c2, ~2^-18 relative; the select kernel's error bound
// covers it). One CTA per (128 queries x 128 centroids) tile: warp 0 TMA, warp 1 MMA issuer +
// TMEM owner, warps 2-5 epilogue (tcgen05.ld, one query row per thread, float4 stores).
#include <cuda_bf16.h>

#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr int kM = 128;             // queries per tile (UMMA M)
constexpr int kNC = 128;            // centroids per tile
constexpr int kStagesC = 3;
constexpr int kABytes = kM * 128;   // one 64-dim bf16 slice of 128 rows
constexpr int kStageBytesC = 2 * kABytes + 2 * kNC * 128;  // q1, q2, c1, c2
constexpr int kThreadsC = 192;

__global__ void __launch_bounds__(kThreadsC, 1)
    coarse_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap cmap,
                     const float* __restrict__ cnorm, float* __restrict__ Dc, int B, int nlist, int d) {
  RD_PDL_PROLOGUE();
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kStagesC * kStageBytesC);
  uint64_t* empty = full + kStagesC;
  uint64_t* done = empty + kStagesC;
  uint32_t* tbase = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.y * kM, c0 = blockIdx.x * kNC;
  const int nks = d / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesC; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tbase;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&qmap);
      prefetch_tmap(&cmap);
      for (int ks = 0; ks < nks; ++ks) {
        const int s = ks % kStagesC;
        mbar_wait(&empty[s], ((ks / kStagesC) & 1) ^ 1);
        const uint32_t st = smem_u32(base + s * kStageBytesC);
        mbar_arrive_expect_tx(&full[s], kStageBytesC);
        tma_load_3d_u32(st, &qmap, ks * 64, 0, q0, &full[s]);
        tma_load_3d_u32(st + kABytes, &qmap, ks * 64, 1, q0, &full[s]);
        tma_load_3d_u32(st + 2 * kABytes, &cmap, ks * 64, 0, c0, &full[s]);
        tma_load_3d_u32(st + 2 * kABytes + kNC * 128, &cmap, ks * 64, 1, c0, &full[s]);
      }
    }
  } else if (warp == 1) {
    const uint32_t ida = idesc_bf16(kM, 2 * kNC), idb = idesc_bf16(kM, kNC);
    for (int ks = 0; ks < nks; ++ks) {
      const int s = ks % kStagesC;
      mbar_wait(&full[s], (ks / kStagesC) & 1);
      tc_fence_after();
      if (lane == 0) {
        const unsigned char* st = base + s * kStageBytesC;
        const uint64_t a1 = umma_desc_sw128(st), a2 = umma_desc_sw128(st + kABytes);
        const uint64_t bc = umma_desc_sw128(st + 2 * kABytes);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t acc = (ks | kk) != 0;
          mma_bf16_ss(tmem, a1 + kk * 2, bc + kk * 2, ida, acc);
          mma_bf16_ss(tmem + 2 * kNC, a2 + kk * 2, bc + kk * 2, idb, acc);
        }
        tc_commit(&empty[s]);
        if (ks == nks - 1) tc_commit(done);
      }
      __syncwarp();
    }
  } else {
    const int quarter = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
    const int q = q0 + quarter * 32 + lane;
    const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16);
    for (int cc = 0; cc < kNC; cc += 16) {
      uint32_t x1[16], x2[16], x3[16];
      RD_TMEM_LD16(ta + cc, x1);
      RD_TMEM_LD16(ta + kNC + cc, x2);
      RD_TMEM_LD16(ta + 2 * kNC + cc, x3);
      tmem_ld_wait();
      if (q < B) {
        float* out = Dc + (size_t)q * nlist + c0 + cc;
        if (c0 + cc + 16 <= nlist && (nlist & 3) == 0) {
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            float4 v;
            v.x = __ldg(cnorm + c0 + cc + i + 0) - 2.f * ((__uint_as_float(x1[i + 0]) + __uint_as_float(x2[i + 0])) + __uint_as_float(x3[i + 0]));
            v.y = __ldg(cnorm + c0 + cc + i + 1) - 2.f * ((__uint_as_float(x1[i + 1]) + __uint_as_float(x2[i + 1])) + __uint_as_float(x3[i + 1]));
            v.z = __ldg(cnorm + c0 + cc + i + 2) - 2.f * ((__uint_as_float(x1[i + 2]) + __uint_as_float(x2[i + 2])) + __uint_as_float(x3[i + 2]));
            v.w = __ldg(cnorm + c0 + cc + i + 3) - 2.f * ((__uint_as_float(x1[i + 3]) + __uint_as_float(x2[i + 3])) + __uint_as_float(x3[i + 3]));
            *reinterpret_cast<float4*>(out + i) = v;
          }
        } else {
          for (int i = 0; i < 16; ++i)
            if (c0 + cc + i < nlist)
              out[i] = __ldg(cnorm + c0 + cc + i) -
                       2.f * ((__uint_as_float(x1[i]) + __uint_as_float(x2[i])) + __uint_as_float(x3[i]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

size_t coarse_tc_smem_bytes() { return 1024 + (size_t)kStagesC * kStageBytesC + 8 * (2 * kStagesC + 2) + 16; }

cudaError_t launch_coarse_tc(const CUtensorMap& qmap, const CUtensorMap& cmap, const float* cnorm, float* Dc, int B,
                             int nlist, int d, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  if (d % 64 != 0) return cudaErrorInvalidValue;
  dim3 grid((nlist + kNC - 1) / kNC, (B + kM - 1) / kM);
  return launch_k(coarse_tc_kernel, grid, dim3(kThreadsC), coarse_tc_smem_bytes(), s, qmap, cmap, cnorm, Dc, B, nlist, d);
}

}  // namespace rd
