// rd_device.cuh — device-side primitives shared by the B200 retrieval kernels:
// counter-based synthetic data (ragsim splitmix64, rng.hpp:12-56), the
// canonical exact distance, mbarrier/TMA PTX wrappers, and warp-level
// bitonic top-k on (distance, row) pairs.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rd {

constexpr int kWarp = 32;
constexpr int kTopK = 32;  // candidates kept per (query, tile) and per query before rerank
constexpr int kMaxK = 24;  // largest k: leaves >= 8 candidates of margin for certification

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
template <bool kLdg, int kDepth = 8>
__device__ __forceinline__ float exact_l2_group8_impl(const float* __restrict__ q, const float* x, int d, int j) {
  // loads are batched kDepth deep ahead of the strictly sequential fp64 accumulation, which keeps
  // the summation order (and so the result) canonical while hiding memory latency (deeper
  // batches for rows streamed from HBM: fewer round trips per row)
  double s = 0.0;
  int t = j;
  for (; t + 8 * (kDepth - 1) < d; t += 8 * kDepth) {
    float qv[kDepth], xv[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      qv[i] = kLdg ? __ldg(q + t + 8 * i) : q[t + 8 * i];
      xv[i] = kLdg ? __ldg(x + t + 8 * i) : x[t + 8 * i];
    }
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const double df = __dsub_rn((double)qv[i], (double)xv[i]);
      s = __dadd_rn(s, __dmul_rn(df, df));
    }
  }
  for (; t < d; t += 8) {
    const double df = __dsub_rn((double)(kLdg ? __ldg(q + t) : q[t]), (double)(kLdg ? __ldg(x + t) : x[t]));
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}
// same value with q already widened to fp64 (shared memory): half the conversions
template <int kDepth = 8>
__device__ __forceinline__ float exact_l2_group8_qd(const double* qd, const float* x, int d, int j) {
  double s = 0.0;
  int t = j;
  for (; t + 8 * (kDepth - 1) < d; t += 8 * kDepth) {
    float xv[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) xv[i] = x[t + 8 * i];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const double df = __dsub_rn(qd[t + 8 * i], (double)xv[i]);
      s = __dadd_rn(s, __dmul_rn(df, df));
    }
  }
  for (; t < d; t += 8) {
    const double df = __dsub_rn(qd[t], (double)x[t]);
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}
// The canonical exact distance to a split3 row read from global memory, with 128-bit loads: per
// 64-element block, lane j of the group loads and decodes chunk 8i + j (x1, x2, x3: one uint4 each),
// the group transposes the block through its 64-float shared scratch (lane j then holds t = 64i + 8k
// + j, k = 0..7, the canonical class order) and sums exactly as exact_l2_group8_impl. Every lane of
// the warp must call it (it syncs the warp); have == false contributes nothing. d % 64 == 0.
__device__ __forceinline__ float exact_l2_group8_split3(const float* q, const __nv_bfloat16* x12,
                                                        const __nv_bfloat16* x3, int d, int j, bool have,
                                                        float* scr) {
  double s = 0.0;
  for (int i = 0; i < d / 64; ++i) {
    if (have) {
      const int c = 8 * i + j;
      const uint4 u1 = __ldg(reinterpret_cast<const uint4*>(x12) + c);
      const uint4 u2 = __ldg(reinterpret_cast<const uint4*>(x12 + d) + c);
      const uint4 u3 = __ldg(reinterpret_cast<const uint4*>(x3) + c);
      const __nv_bfloat16* h1 = reinterpret_cast<const __nv_bfloat16*>(&u1);
      const __nv_bfloat16* h2 = reinterpret_cast<const __nv_bfloat16*>(&u2);
      const __nv_bfloat16* h3 = reinterpret_cast<const __nv_bfloat16*>(&u3);
      float xv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        xv[e] = __fadd_rn(__fadd_rn(__bfloat162float(h1[e]), __bfloat162float(h2[e])), __bfloat162float(h3[e]));
      reinterpret_cast<float4*>(scr + 8 * j)[0] = make_float4(xv[0], xv[1], xv[2], xv[3]);
      reinterpret_cast<float4*>(scr + 8 * j)[1] = make_float4(xv[4], xv[5], xv[6], xv[7]);
    }
    __syncwarp();
    if (have) {
      float xv[8], qv[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        xv[k] = scr[8 * k + j];
        qv[k] = __ldg(q + 64 * i + 8 * k + j);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double df = __dsub_rn((double)qv[k], (double)xv[k]);
        s = __dadd_rn(s, __dmul_rn(df, df));
      }
    }
    __syncwarp();
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}
// exact_l2_group8_qd over the first cnt elements (cnt < d: a padded slot passes 0 and its group
// stays converged for the shuffles); x in shared memory
__device__ __forceinline__ float exact_l2_group8_qd_cnt(const double* qd, const float* x, int cnt, int j) {
  constexpr int kDepth = 8;
  double s = 0.0;
  int t = j;
  for (; t + 8 * (kDepth - 1) < cnt; t += 8 * kDepth) {
    float xv[kDepth];
    double qv[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      xv[i] = x[t + 8 * i];
      qv[i] = qd[t + 8 * i];
    }
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const double df = __dsub_rn(qv[i], (double)xv[i]);
      s = __dadd_rn(s, __dmul_rn(df, df));
    }
  }
  for (; t < cnt; t += 8) {
    const double df = __dsub_rn(qd[t], (double)x[t]);
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}
__device__ __forceinline__ float exact_l2_group8(const float* __restrict__ q, const float* __restrict__ x, int d,
                                                 int j) {
  return exact_l2_group8_impl<true>(q, x, d, j);
}
// same value, x possibly in mapped host memory (no __ldg on the non-coherent path)
__device__ __forceinline__ float exact_l2_group8_any(const float* __restrict__ q, const float* x, int d, int j) {
  return exact_l2_group8_impl<false>(q, x, d, j);
}

// ---------------------------------------------------------------- rows of the resident store
// A row is fp32 (f != nullptr: offloaded lists in mapped host memory, or an fp32 arena) or the
// exact bf16 triple split of the split3 arena (host.cuh): x = (x1 + x2) + x3 bit for bit, x1 / x2 at
// x12[t] / x12[d + t] (the scan's [rows][2][d] operand), x3 at x3[t]. at() returns the fp32 value.
struct RowRef {
  const float* f;
  const __nv_bfloat16* x12;
  const __nv_bfloat16* x3;
  __device__ __forceinline__ float at(int t, int d) const {
    if (f) return f[t];
    return __fadd_rn(__fadd_rn(__bfloat162float(x12[t]), __bfloat162float(x12[d + t])), __bfloat162float(x3[t]));
  }
};
__device__ __forceinline__ RowRef row_f32(const float* f) { return RowRef{f, nullptr, nullptr}; }
// row r of a split3 store (x12: [rows][2][d], x3: [rows][d])
__device__ __forceinline__ RowRef row_split3(const __nv_bfloat16* x12, const __nv_bfloat16* x3, long long r, int d) {
  return RowRef{nullptr, x12 + (size_t)r * 2 * d, x3 + (size_t)r * d};
}
// the canonical exact distance (exact_l2_group8_impl's order and value) to a RowRef row
// (cnt < d terms: a padded slot passes 0 and the group stays converged for the shuffles)
template <int kDepth = 8>
__device__ __forceinline__ float exact_l2_group8_row(const float* q, const RowRef& x, int d, int j, int cnt) {
  double s = 0.0;
  int t = j;
  for (; t + 8 * (kDepth - 1) < cnt; t += 8 * kDepth) {
    float qv[kDepth], xv[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      qv[i] = q[t + 8 * i];
      xv[i] = x.at(t + 8 * i, d);
    }
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const double df = __dsub_rn((double)qv[i], (double)xv[i]);
      s = __dadd_rn(s, __dmul_rn(df, df));
    }
  }
  for (; t < cnt; t += 8) {
    const double df = __dsub_rn((double)q[t], (double)x.at(t, d));
    s = __dadd_rn(s, __dmul_rn(df, df));
  }
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
  s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
  return __double2float_rn(s);
}

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the search chain starts with RD_PDL_PROLOGUE: it lets the next kernel in the
// stream begin launching (griddepcontrol.launch_dependents), then waits until every kernel it
// depends on has completed and its writes are visible (griddepcontrol.wait). Without the launch
// attribute (see launch_k) both are no-ops, so correctness never depends on PDL.
#define RD_PDL_PROLOGUE()                                              \
  do {                                                                 \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");    \
    asm volatile("griddepcontrol.wait;" ::: "memory");                 \
  } while (0)

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// profiling only (RD_DEBUG_TS): globaltimer / clock64 checkpoints of CTA 0
// profiling only: the latest end over all CTAs of a kernel at slot 12
#define RD_TS_END()                                                              \
  do {                                                                           \
    if (p.dbg && threadIdx.x == 0) atomicMax(p.dbg + 12, gtimer());              \
  } while (0)

#define RD_TS(i)                                                 \
  do {                                                           \
    if (p.dbg && blockIdx.x == 0 && threadIdx.x == 0) {          \
      p.dbg[i] = gtimer();                                       \
      p.dbg[16 + i] = clock64();                                 \
    }                                                            \
  } while (0)

// ---------------------------------------------------------------- PTX: smem, mbarrier, TMA
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- row staging for exact distances
// The canonical sum is a chain of d/8 dependent fp64 adds per lane; reading x from global memory
// inside that chain costs one memory round trip per 8-element batch (12 at d = 768). At low
// occupancy (small batches) that latency is the whole cost, so the rows are first staged into
// shared memory with every load in flight at once, then summed from smem.
constexpr int kStagePad = 8;  // floats of padding per staged row: 4 groups of a warp hit distinct banks

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// 1D bulk (TMA) copy global -> shared, completion counted on an mbarrier's tx-count
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// fp32 squared distance by groups of 8 lanes (same lane/class layout as the canonical sum);
// |result - ||q - x||^2| <= l2_f32_rel_bound(d) * ||q - x||^2
template <int kDepth = 1>
__device__ __forceinline__ float l2_group8_f32(const float* q, const float* x, int d, int j) {
  float s = 0.f;
  int t = j;
  for (; t + 8 * (kDepth - 1) < d; t += 8 * kDepth) {  // kDepth loads in flight, same summation order
    float qv[kDepth], xv[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      qv[i] = q[t + 8 * i];
      xv[i] = x[t + 8 * i];
    }
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const float df = qv[i] - xv[i];
      s = fmaf(df, df, s);
    }
  }
  for (; t < d; t += 8) {
    const float df = q[t] - x[t];
    s = fmaf(df, df, s);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  return s;
}
__host__ __device__ __forceinline__ float l2_f32_rel_bound(int d) { return 2.f * (d / 8 + 8) * 5.9604645e-8f; }
// l2_group8_f32 of a RowRef row (same order, same bound)
template <int kDepth = 1>
__device__ __forceinline__ float l2_group8_f32_row(const float* q, const RowRef& x, int d, int j) {
  float s = 0.f;
  int t = j;
  for (; t + 8 * (kDepth - 1) < d; t += 8 * kDepth) {
    float qv[kDepth], xv[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      qv[i] = q[t + 8 * i];
      xv[i] = x.at(t + 8 * i, d);
    }
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      const float df = qv[i] - xv[i];
      s = fmaf(df, df, s);
    }
  }
  for (; t < d; t += 8) {
    const float df = q[t] - x.at(t, d);
    s = fmaf(df, df, s);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  return s;
}
// Same bound as l2_group8_f32_row (each lane's chain is d/8 fp32 FMAs, then the 3-level tree), with
// lane j summing the 8-element chunks c = j (mod 8) instead of residue classes: 128-bit shared-memory
// loads (one per 8 elements and operand) instead of one load per element. q and the row are in
// shared memory, 16-byte aligned, d % 64 == 0.
__device__ __forceinline__ float l2_group8_f32_chunks(const float* q, const RowRef& x, int d, int j) {
  float s = 0.f;
  for (int c = j; c < d / 8; c += 8) {
    const float4 q0 = reinterpret_cast<const float4*>(q)[2 * c], q1 = reinterpret_cast<const float4*>(q)[2 * c + 1];
    float xv[8];
    if (x.f) {
      const float4 a = reinterpret_cast<const float4*>(x.f)[2 * c], b = reinterpret_cast<const float4*>(x.f)[2 * c + 1];
      xv[0] = a.x, xv[1] = a.y, xv[2] = a.z, xv[3] = a.w, xv[4] = b.x, xv[5] = b.y, xv[6] = b.z, xv[7] = b.w;
    } else {
      const uint4 u1 = reinterpret_cast<const uint4*>(x.x12)[c], u2 = reinterpret_cast<const uint4*>(x.x12 + d)[c],
                  u3 = reinterpret_cast<const uint4*>(x.x3)[c];
      const __nv_bfloat16* h1 = reinterpret_cast<const __nv_bfloat16*>(&u1);
      const __nv_bfloat16* h2 = reinterpret_cast<const __nv_bfloat16*>(&u2);
      const __nv_bfloat16* h3 = reinterpret_cast<const __nv_bfloat16*>(&u3);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        xv[e] = __fadd_rn(__fadd_rn(__bfloat162float(h1[e]), __bfloat162float(h2[e])), __bfloat162float(h3[e]));
    }
    const float qv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float df = qv[e] - xv[e];
      s = fmaf(df, df, s);
    }
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  return s;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// rows r < nrows of row_ptr(r) (device memory, 16 B aligned, d % 4 == 0) -> dst[r * (d + kStagePad)],
// cp.async, all in flight; the caller waits (cp_async_wait_all) and syncs
template <int NT, class RowPtr>
__device__ __forceinline__ void stage_rows_async(float* dst, int nrows, int d, RowPtr row_ptr) {
  const int v4 = d >> 2, ds = d + kStagePad;
  for (int i = threadIdx.x; i < nrows * v4; i += NT) {
    const int r = i / v4, c = i - r * v4;
    cp_async16(dst + r * ds + 4 * c, row_ptr(r) + 4 * c);
  }
}
// same with ordinary loads (rows possibly in mapped host memory), 8 loads in flight per thread
template <int NT, class RowPtr>
__device__ __forceinline__ void stage_rows_ld(float* dst, int nrows, int d, RowPtr row_ptr) {
  const int v4 = d >> 2, ds = d + kStagePad, tot = nrows * v4;
  for (int i0 = threadIdx.x; i0 < tot; i0 += 8 * NT) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * NT;
      if (i < tot) {
        const int r = i / v4, c = i - r * v4;
        v[u] = *reinterpret_cast<const float4*>(row_ptr(r) + 4 * c);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * NT;
      if (i < tot) {
        const int r = i / v4, c = i - r * v4;
        *reinterpret_cast<float4*>(dst + r * ds + 4 * c) = v[u];
      }
    }
  }
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
__device__ __forceinline__ void tma_load_2d_u32(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_u32(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// 4 arbitrary rows x box-width columns of a 2D map (box {cols, 1}) into 4 consecutive smem rows
__device__ __forceinline__ void tma_gather4_u32(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2,
                                                int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- PTX: tcgen05 / TMEM (sm_100a)
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc]^T, kind::tf32
__device__ __forceinline__ void mma_tf32_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]^T, kind::tf32
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on an mbarrier when all prior tcgen05.mma of this thread have completed
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// K-major, 128B-swizzled smem matrix descriptor (8-row x 128 B atoms, SBO = 1024 B), sm100 version 1
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem_ptr) {
  const uint32_t addr = smem_u32(smem_ptr);
  uint64_t desc = 0;
  desc |= (uint64_t)((addr >> 4) & 0x3FFF);        // start address
  desc |= (uint64_t)1 << 16;                        // LBO (ignored for swizzled K-major)
  desc |= (uint64_t)(1024 >> 4) << 32;              // SBO
  desc |= (uint64_t)1 << 46;                        // version (sm100)
  desc |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return desc;
}
// D[tmem] (+)= A[smem desc] * B[smem desc]^T, kind::f16 (BF16 inputs, F32 accumulate)
__device__ __forceinline__ void mma_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]^T, kind::f16 (BF16 inputs, F32 accumulate)
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// instruction descriptor: F32 accumulate, BF16 A/B, both K-major, M x N
// fp16 A and B (a_format = b_format = F16), fp32 D
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// explicit shared-space 128-bit accesses (generic pointers derived from aligned
// dynamic smem otherwise compile to generic LD/ST)
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// each lane stores 16 consecutive 32-bit columns of its own TMEM lane
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// instruction descriptor: F32 accumulate, TF32 A/B, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
#define RD_TMEM_LD16(taddr, r)                                                                       \
  asm volatile(                                                                                     \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
      : "r"(taddr))
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// each lane stores 8 consecutive 32-bit columns of its own TMEM lane
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
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
// Insert one candidate (broadcast in all lanes) into the ascending list L.
__device__ __forceinline__ void warp_insert1(float& ld, long long& lk, float cd, long long ck, int lane) {
  const unsigned lt = __ballot_sync(0xffffffffu, pair_less(ld, lk, cd, ck));
  const int pos = __popc(lt);
  const float ud = __shfl_up_sync(0xffffffffu, ld, 1);
  const long long uk = __shfl_up_sync(0xffffffffu, lk, 1);
  if (lane == pos) {
    ld = cd;
    lk = ck;
  } else if (lane > pos) {
    ld = ud;
    lk = uk;
  }
}
// orderable int for an atomicMin over non-negative-or-negative floats
__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

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
