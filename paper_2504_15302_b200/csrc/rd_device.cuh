// rd_device.cuh — device-side primitives shared by the B200 retrieval kernels:
// counter-based synthetic data (ragsim splitmix64, rng.hpp:12-56), the
// canonical exact distance, mbarrier/TMA PTX wrappers, and warp-level
// bitonic top-k on (distance, row) pairs.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rd {

constexpr int kWarp = 32;
constexpr int kTopK = 32;  // candidates kept per (query, tile) and per query before rerank

// ---------------------------------------------------------------- splitmix64
// ragsim::Rng::next_u64 (rng.hpp:16-21) in counter form: the (i+1)-th output of Rng(seed).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  return mix64(seed + (i + 1) * 0x9e3779b97f4a7c15ull);
}
// uniform on [-1, 1) with 24 bits: exactly representable, identical on host and device.
__host__ __device__ __forceinline__ float unif(uint64_t seed, uint64_t i) {
  uint64_t u = splitmix_at(seed, i);
  int32_t m = (int32_t)((u >> 40) & 0xFFFFFFu) - (1 << 23);
  return (float)m * 0x1p-23f;
}

// ---------------------------------------------------------------- canonical exact L2
// Eight lanes j = lane & 7 of an aligned group each sum residue class t = j (mod 8)
// sequentially in fp64 (no contraction), then the fixed tree
// ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)); every lane of the group returns the f32 value.
__device__ __forceinline__ float exact_l2_group8(const float* __restrict__ q,
                                                 const float* __restrict__ x, int d, int j) {
  double s = 0.0;
  for (int t = j; t < d; t += 8) {
    double df = __dsub_rn((double)__ldg(q + t), (double)__ldg(x + t));
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}
// same value, x possibly in mapped host memory (no __ldg on the non-coherent path)
__device__ __forceinline__ float exact_l2_group8_any(const float* __restrict__ q, const float* x,
                                                     int d, int j) {
  double s = 0.0;
  for (int t = j; t < d; t += 8) {
    double df = __dsub_rn((double)q[t], (double)x[t]);
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}

// ---------------------------------------------------------------- PTX: smem, mbarrier, TMA
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "RD_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra RD_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- warp bitonic (dist, row)
// Lexicographic order on (distance, tie key). The tie key is the arena row for
// approximate candidates and the user id for exact candidates.
__device__ __forceinline__ bool pair_less(float da, long long ka, float db, long long kb) {
  return da < db || (da == db && ka < kb);
}

// One compare-exchange step of a 32-lane bitonic network.
__device__ __forceinline__ void bitonic_step(float& d, long long& k, int lane, int j, bool up) {
  float od = __shfl_xor_sync(0xffffffffu, d, j);
  long long ok = __shfl_xor_sync(0xffffffffu, k, j);
  bool lower = (lane & j) == 0;
  bool other_less = pair_less(od, ok, d, k);
  // ascending block: lower lane keeps min; descending: lower lane keeps max
  bool take = (lower == up) ? other_less : !other_less && !(od == d && ok == k);
  if (take) {
    d = od;
    k = ok;
  }
}
// Full sort of one element per lane; ascending if asc.
__device__ __forceinline__ void warp_sort32(float& d, long long& k, int lane, bool asc) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      bool up = ((lane & size) == 0) == asc;
      if (size == 32) up = asc;
      bitonic_step(d, k, lane, j, up);
    }
  }
}
// L ascending (one per lane) absorbs batch B (one per lane, any order): L becomes
// the 32 smallest of L ∪ B, ascending.
__device__ __forceinline__ void warp_merge32(float& ld, long long& lk, float bd, long long bk,
                                             int lane) {
  warp_sort32(bd, bk, lane, /*asc=*/false);  // descending
  if (pair_less(bd, bk, ld, lk)) {
    ld = bd;
    lk = bk;
  }
  // bitonic sequence -> ascending
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) bitonic_step(ld, lk, lane, j, true);
}

}  // namespace rd
