// scan_pair.cu — N5 for wide tiles (<= 32 queries) on CTA PAIRS: tcgen05.mma.cta_group::2 (sm_100a).
//
// Why: the single-CTA 32-query scan (scan_tc.cu) keeps the tile's query operand B = [q1; q2]
// (64 rows x d bf16 = 96 KiB at d = 768) resident next to its x ring, which leaves room for three
// 32 KiB stages; the producer then waits for a free stage ~half the time. Here two
// CTAs of a cluster (one TPC) run one M = 256 MMA per K step: each CTA holds HALF of B — the leader
// (rank 0) q1, the peer q2 — and its own 128 x rows of every 256-row block, so the ring grows to
// five stages and the pair issues half the MMAs per byte.
//
// Per 64-dim stage (x1 | x2 of 128 rows per CTA, 32 KiB) the leader issues, for 4 K steps of 16,
//   D_a += x1 . [q1 ; q2]   (M = 256, N = 64: columns 0-31 from the leader's B half, 32-63 the peer's)
//   D_b += x2 . [q1 ; q2]   (same B; only its q1 columns are read)
// and every CTA's epilogue reads its own 128 TMEM lanes: q.x ~ (x1.q1 + x1.q2) + x2.q1 — the same
// bf16x3 dot as scan_tc.cu, so the certification bound (gamma_bf16x3) is unchanged.
//
// Roles per CTA (6 warps): warp 0 TMA producer (both CTAs load their own x rows and B half; every
// load completes on the LEADER's mbarrier, cta_group::2), warp 1 TMEM allocator (both) and MMA issuer
// (leader), warps 2-5 epilogue (both; each CTA emits its own partial lists). The leader's producer
// owns the dynamic tile queue and publishes each tile (index + descriptor) into both CTAs' shared
// memory (st.shared::cluster + a remote mbarrier arrive).
//
// Barriers (same offsets in both CTAs; "L" = only the leader's copy is used):
//   full[s]  L  1 arrival (leader producer, expect_tx of both halves) + TMA bytes of both CTAs
//   empty[s]    MMA commit multicast to both            afull[a]   MMA commit multicast to both
//   aempty[a] L 8 arrivals (4 epilogue warps per CTA)   bfull   L  expect_tx both halves' gathers
//   bempty      MMA commit multicast                     tfull[i]   leader producer (remote arrive for the peer)
//   tempty[i] L 10 arrivals (leader MMA + 4 epilogue; peer producer + 4 epilogue)
#include <cuda_bf16.h>

#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr int kPRows = 128;                 // x rows per CTA per row block (UMMA M / 2)
constexpr int kPBlock = 2 * kPRows;         // rows per pair row block
constexpr int kPG = 32;                     // queries per tile
constexpr int kPStageBytes = 2 * kPRows * 128;  // x1 | x2, 64 dims, 128 rows
constexpr int kPHalfSlice = kPG * 128;      // one CTA's B half per 64-dim slice: 32 rows x 128 B
constexpr int kPThreads = 192;
constexpr uint32_t kPTmemCols = 256;        // two accumulator buffers of D_a (64) + D_b (64)
constexpr uint32_t kPAccCols = 128;
constexpr float kPInf = __builtin_huge_valf();
constexpr long long kPNoKey = 0x7fffffffffffffffll;

// ---------------------------------------------------------------- cluster / pair PTX
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void remote_arrive(uint32_t cl_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cl_bar) : "memory");
}
// wait on a local barrier whose phase may have been completed by the peer CTA (cluster-scope acquire)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "RD_WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra RD_WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cl_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cl_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t cl_addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(cl_addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
// TMA into this CTA's smem, completion on the leader's mbarrier (cl_bar: shared::cluster address)
__device__ __forceinline__ void tma3_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t cl_bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(cl_bar)
      : "memory");
}
__device__ __forceinline__ void tma2_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t cl_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(cl_bar)
      : "memory");
}
__device__ __forceinline__ void gather4_pair(uint32_t dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                             uint32_t cl_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.cta_group::2"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(cl_bar)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void mma2_bf16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the barrier at this offset in BOTH CTAs once the leader's prior MMAs complete
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}

struct PSmem {
  uint32_t xs, bs;
  uint64_t *full, *empty, *afull, *aempty, *bfull, *bempty, *tfull, *tempty;
  int* tring;
  ScanTile* tinfo;
  uint32_t* tmem_base;
  long long* stage_k;
  float* stage_d;
  float* edist;
};

// x stage bytes per CTA: x1 | x2 (split3), or the residual store's r1 (one 16 KiB tile)
template <bool kRes>
constexpr int pstage_bytes() { return kRes ? kPRows * 128 : kPStageBytes; }

template <int kS, bool kRes>
__device__ __forceinline__ PSmem pcarve(unsigned char* raw, int d) {
  constexpr int kPStageBytes = pstage_bytes<kRes>();
  PSmem s;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  s.xs = smem_u32(base);
  s.bs = s.xs + (uint32_t)(kS * kPStageBytes);
  uint64_t* b = reinterpret_cast<uint64_t*>(base + kS * kPStageBytes + (d / 64) * kPHalfSlice);
  s.full = b;
  s.empty = s.full + kS;
  s.afull = s.empty + kS;
  s.aempty = s.afull + 2;
  s.bfull = s.aempty + 2;
  s.bempty = s.bfull + 1;
  s.tfull = s.bempty + 1;
  s.tempty = s.tfull + 2;
  s.tring = reinterpret_cast<int*>(s.tempty + 2);  // 2 ints, then padding to 16 B
  s.tinfo = reinterpret_cast<ScanTile*>(reinterpret_cast<unsigned char*>(s.tring) + 16);
  s.tmem_base = reinterpret_cast<uint32_t*>(s.tinfo + 2);
  s.stage_k = reinterpret_cast<long long*>(s.tmem_base + 2);
  s.stage_d = reinterpret_cast<float*>(s.stage_k + 4 * 32);
  s.edist = s.stage_d + 4 * 32;
  return s;
}
template <int kS, bool kRes = false>
constexpr size_t pair_smem_bytes_for(int d) {
  constexpr int kPStageBytes = pstage_bytes<kRes>();
  return 1024 + (size_t)kS * kPStageBytes + (size_t)(d / 64) * kPHalfSlice + (2 * kS + 10) * 8 + 16 +
         2 * sizeof(ScanTile) + 8 + 4 * 32 * 12 + (size_t)kPG * kPRows * 4 + 64;
}

// bytes one CTA's TMA brings for its half of row block rt (rows in 32-row boxes, x1 and x2)
template <bool kRes>
__device__ __forceinline__ uint32_t half_bytes(int nrows, int rt, int rank) {
  const int rows = min(kPRows, max(0, nrows - rt * kPBlock - rank * kPRows));
  return (uint32_t)((kRes ? 1 : 2) * ((rows + 31) >> 5) * 4096);
}

// profiling only (built with -DRD_STALL_PROF, run with RD_DEBUG_STALL): cycles a role spends blocked
// on one barrier, in the slots the host prints for the single-CTA scan (search.cu)
#ifdef RD_STALL_PROF
#define RD_PWAIT(expr, slot)                     \
  do {                                           \
    if (p.stall) {                               \
      const long long t0_ = clock64();           \
      expr;                                      \
      stall_acc[slot] += clock64() - t0_;        \
    } else {                                     \
      expr;                                      \
    }                                            \
  } while (0)
#else
#define RD_PWAIT(expr, slot) expr
#endif

// kRes: the residual store (resid.cu, scan_tc.cu): A = r1 tiles, one M = 256 MMA per K step
// (r1.[q1;q2]), lower-bound keys from resid_pair_term.
template <int kS, bool kRes>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPThreads, 1)
    ivf_scan_pair_kernel(const __grid_constant__ CUtensorMap map128, const __grid_constant__ CUtensorMap map32,
                         const __grid_constant__ CUtensorMap qmap, const TcScanParams p) {
  RD_PDL_PROLOGUE();
  extern __shared__ unsigned char smem_raw[];
  const int d = p.d, nks = d / 64;
  const PSmem sm = pcarve<kS, kRes>(smem_raw, d);
  constexpr int kPStageBytes = pstage_bytes<kRes>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.afull[i], 1);
      mbar_init(&sm.aempty[i], 8);
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 10);
    }
    mbar_init(sm.bfull, 1);
    mbar_init(sm.bempty, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2(sm.tmem_base, kPTmemCols);
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised and TMEM allocated before any remote traffic
  tc_fence_after();
  const uint32_t tmem = *sm.tmem_base;
  const int ntiles = *p.ntiles;
#ifdef RD_STALL_PROF
  long long stall_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_begin = clock64();
#endif
  // the leader's copies of the shared barriers, as shared::cluster addresses
  const uint32_t L_full0 = mapa(smem_u32(sm.full), 0), L_bfull = mapa(smem_u32(sm.bfull), 0);
  const uint32_t L_aempty0 = mapa(smem_u32(sm.aempty), 0), L_tempty0 = mapa(smem_u32(sm.tempty), 0);

  // ---------------------------------------------------------------- warp 0: TMA producer (both)
  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&map128);
      prefetch_tmap(&map32);
      prefetch_tmap(&qmap);
    }
    const int nslices = nks;
    const uint32_t P_tring0 = mapa(smem_u32(sm.tring), 1), P_tinfo0 = mapa(smem_u32(sm.tinfo), 1);
    const uint32_t P_tfull0 = mapa(smem_u32(sm.tfull), 1);
    uint32_t u = 0;
    int tn = 0;  // leader: the next tile, fetched one tile ahead
    ScanTile Tn{};
    if (leader) {
      if (lane == 0) tn = atomicAdd(p.tile_counter, 1);
      tn = __shfl_sync(0xffffffffu, tn, 0);
      if (tn < ntiles) Tn = p.tiles[tn];
    }
    for (uint32_t ti = 0;; ++ti) {
      const int slot = ti & 1;
      int t;
      ScanTile T;
      if (leader) {
        t = tn < ntiles ? tn : -1;
        T = Tn;
        if (lane == 0) {
          RD_PWAIT(mbar_wait(&sm.tempty[slot], ((ti >> 1) & 1) ^ 1), 0);
          sm.tring[slot] = t;
          sm.tinfo[slot] = T;
          st_cluster_u32(P_tring0 + 4 * slot, (uint32_t)t);
          const uint4* tv = reinterpret_cast<const uint4*>(&T);
          st_cluster_v4(P_tinfo0 + sizeof(ScanTile) * slot, tv[0]);
          st_cluster_v4(P_tinfo0 + sizeof(ScanTile) * slot + 16, tv[1]);
          mbar_arrive(&sm.tfull[slot]);
          remote_arrive(P_tfull0 + 8 * slot);
        }
        __syncwarp();
        if (t < 0) break;
        if (lane == 0) tn = atomicAdd(p.tile_counter, 1);
      } else {
        RD_PWAIT(mbar_wait_cl(&sm.tfull[slot], (ti >> 1) & 1), 0);
        t = sm.tring[slot];
        T = sm.tinfo[slot];
        __syncwarp();
        if (lane == 0) remote_arrive(L_tempty0 + 8 * slot);
        if (t < 0) break;
      }
      const int nblk = (T.nrows + kPBlock - 1) / kPBlock;
      const int nst = nblk * nks;
      auto issue_x = [&](int i) {  // lane 0
        const int rt = i / nks, ks = i - rt * nks;
        const int s = u % kS;
        RD_PWAIT(mbar_wait(&sm.empty[s], ((u / kS) & 1) ^ 1), 1);
        const uint32_t lb = L_full0 + 8 * s;
        if (leader)
          mbar_arrive_expect_tx(&sm.full[s], half_bytes<kRes>(T.nrows, rt, 0) + half_bytes<kRes>(T.nrows, rt, 1));
        const int rows = min(kPRows, T.nrows - rt * kPBlock - (int)rank * kPRows);
        if (rows > 0) {
          const uint32_t dst = sm.xs + s * kPStageBytes;
          const int row = (int)(T.src_row + rt * kPBlock + (int)rank * kPRows);
          if (kRes) {
            if (rows == kPRows)
              tma2_pair(dst, &map128, ks * 64, row, lb);
            else
              for (int b = 0; b < (rows + 31) >> 5; ++b) tma2_pair(dst + b * 4096, &map32, ks * 64, row + b * 32, lb);
          } else if (rows == kPRows) {
            tma3_pair(dst, &map128, ks * 64, 0, row, lb);
            tma3_pair(dst + kPRows * 128, &map128, ks * 64, 1, row, lb);
          } else {
            for (int b = 0; b < (rows + 31) >> 5; ++b) {
              tma3_pair(dst + b * 4096, &map32, ks * 64, 0, row + b * 32, lb);
              tma3_pair(dst + kPRows * 128 + b * 4096, &map32, ks * 64, 1, row + b * 32, lb);
            }
          }
        }
        ++u;
      };
      // this CTA's B half: rows 2 * qid + rank of the tile's queries (q1 on the leader, q2 on the
      // peer), quads of 4 rows by gather4; padding rows repeat the last query
      const int qq = (T.nq + 3) >> 2;
      const int ngrp = 32 / qq, grp = lane / qq, qi = lane - grp * qq;
      const int g0 = qi * 4;
      int r[4];
      if (grp < ngrp)
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = 2 * __ldg(p.list_q + T.qoff + min(g0 + i, T.nq - 1)) + (int)rank;
      const int npre = min(nst, kS);
      if (lane == 0)
        for (int i = 0; i < npre; ++i) issue_x(i);
      __syncwarp();
      if (leader) {  // the next tile's descriptor while this one streams
        tn = __shfl_sync(0xffffffffu, tn, 0);
        if (tn < ntiles) Tn = p.tiles[tn];
      }
      RD_PWAIT(mbar_wait(sm.bempty, (ti & 1) ^ 1), 2);
      if (leader && lane == 0) mbar_arrive_expect_tx(sm.bfull, (uint32_t)(nslices * 2 * qq * 512));
      __syncwarp();
      if (grp < ngrp)
        for (int slice = grp; slice < nslices; slice += ngrp)
          gather4_pair(sm.bs + slice * kPHalfSlice + qi * 512, &qmap, slice * 64, r[0], r[1], r[2], r[3], L_bfull);
      if (lane == 0)
        for (int i = npre; i < nst; ++i) issue_x(i);
      __syncwarp();
    }
  }
  // ---------------------------------------------------------------- warp 1: MMA issuer (leader)
  else if (warp == 1) {
    if (leader) {
      // tiles of <= 16 queries: half N (each CTA's B half holds its part's queries in rows 0..nq-1, so
      // N = 32 reads 16 rows from each CTA: x1.[q1;q2] in columns 0-31, x2.[q1;q2] from 64)
      const uint32_t idesc_full = idesc_bf16(kPBlock, 2 * kPG), idesc_half = idesc_bf16(kPBlock, kPG);
      const unsigned char* bs_ptr = reinterpret_cast<unsigned char*>(smem_raw) + (sm.bs - smem_u32(smem_raw));
      const uint64_t bdesc0 = umma_desc_sw128(bs_ptr);
      uint32_t u = 0, rtc = 0;
      for (uint32_t ti = 0;; ++ti) {
        const int slot = ti & 1;
        RD_PWAIT(mbar_wait(&sm.tfull[slot], (ti >> 1) & 1), 3);
        const int t = sm.tring[slot];
        const int nrows = sm.tinfo[slot].nrows;
        const uint32_t idesc = sm.tinfo[slot].nq <= kPG / 2 ? idesc_half : idesc_full;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[slot]);
        if (t < 0) break;
        for (int rt = 0; rt * kPBlock < nrows; ++rt, ++rtc) {
          const int a = rtc & 1;
          RD_PWAIT(mbar_wait(&sm.aempty[a], ((rtc >> 1) & 1) ^ 1), 5);
          tc_fence_after();
          const uint32_t dacc = tmem + a * kPAccCols;
          for (int ks = 0; ks < nks; ++ks, ++u) {
            if (rt == 0 && ks == 0) RD_PWAIT(mbar_wait(sm.bfull, ti & 1), 4);
            const int s = u % kS;
            RD_PWAIT(mbar_wait(&sm.full[s], (u / kS) & 1), 6);
            tc_fence_after();
            if (lane == 0) {
              const unsigned char* st =
                  reinterpret_cast<unsigned char*>(smem_raw) + (sm.xs - smem_u32(smem_raw)) + s * kPStageBytes;
              const uint64_t a1 = umma_desc_sw128(st), a2 = umma_desc_sw128(st + kPRows * 128);
              const uint64_t bd = bdesc0 + (uint64_t)(ks * (kPHalfSlice >> 4));
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t acc = (ks | kk) != 0;
                mma2_bf16_ss(dacc, a1 + kk * 2, bd + (uint64_t)(kk * 2), idesc, acc);
                if constexpr (!kRes) mma2_bf16_ss(dacc + 2 * kPG, a2 + kk * 2, bd + (uint64_t)(kk * 2), idesc, acc);
              }
              tc_commit_mc(&sm.empty[s]);
            }
            __syncwarp();
          }
          if (lane == 0) tc_commit_mc(&sm.afull[a]);
          __syncwarp();
        }
        if (lane == 0) tc_commit_mc(sm.bempty);
        __syncwarp();
      }
    }
  }
  // ---------------------------------------------------------------- warps 2-5: epilogue (both)
  else {
    constexpr int kOwn = kPG / 4;
    const int quarter = warp & 3, ew = warp - 2;
    float* edist = sm.edist;
    float* sd = sm.stage_d + ew * 32;
    long long* sk = sm.stage_k + ew * 32;
    uint32_t rtc = 0;
    for (uint32_t ti = 0;; ++ti) {
      const int slot = ti & 1;
      if (leader)
        mbar_wait(&sm.tfull[slot], (ti >> 1) & 1);
      else
        mbar_wait_cl(&sm.tfull[slot], (ti >> 1) & 1);
      const int t = sm.tring[slot];
      const ScanTile T = sm.tinfo[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&sm.tempty[slot]);
        else
          remote_arrive(L_tempty0 + 8 * slot);
      }
      if (t < 0) break;
      const int nq = T.nq;
      float qn[kOwn], ld[kOwn], qt[kOwn];
      long long lk[kOwn];
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int g = ew + 4 * j;
        const int qid = g < nq ? __ldg(p.list_q + T.qoff + g) : 0;
        qn[j] = g < nq ? __ldg(p.qnorm + qid) : 0.f;
        if (kRes && g < nq) qn[j] = resid_pair_term(p, qn[j], qid, T.list);
        qt[j] = g < nq ? ord2f(*(volatile int*)(p.qthr + qid)) : kPInf;
        ld[j] = kPInf;
        lk[j] = kPNoKey;
      }
      for (int rt = 0; rt * kPBlock < T.nrows; ++rt, ++rtc) {
        const int a = rtc & 1;
        RD_PWAIT(mbar_wait(&sm.afull[a], (rtc >> 1) & 1), 8);
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + a * kPAccCols;
        uint32_t d1[kPG], d2[kPG], d3[kPG];
        const uint32_t c2 = nq <= kPG / 2 ? kPG / 2 : kPG;  // half tiles: x1.q2 from column 16
#pragma unroll
        for (int c = 0; c < kPG; c += 16) {
          RD_TMEM_LD16(ta + c, (d1 + c));
          RD_TMEM_LD16(ta + c2 + c, (d2 + c));
          if constexpr (!kRes) RD_TMEM_LD16(ta + 2 * kPG + c, (d3 + c));
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader)
            mbar_arrive(&sm.aempty[a]);
          else
            remote_arrive(L_aempty0 + 8 * a);
        }
        const int r = quarter * 32 + lane;
        const int rloc = rt * kPBlock + (int)rank * kPRows + r;
        const bool valid = rloc < T.nrows;
        const float xn = valid ? __ldg(p.xnorm + T.grow0 + rloc) : 0.f;
        named_bar_sync(2, 128);  // every owner finished reading the previous row tile
#pragma unroll
        for (int g = 0; g < kPG; ++g) {
          const float dot = kRes ? __uint_as_float(d1[g]) + __uint_as_float(d2[g])
                                 : (__uint_as_float(d1[g]) + __uint_as_float(d2[g])) + __uint_as_float(d3[g]);
          edist[g * kPRows + r] = (valid && g < nq) ? xn - 2.f * dot : kPInf;
        }
        named_bar_sync(2, 128);
        const long long gbase = T.grow0 + (long long)rt * kPBlock + (long long)rank * kPRows;
#pragma unroll
        for (int j = 0; j < kOwn; ++j) {
          const int g = ew + 4 * j;
          if (g >= nq) break;
          float thr = fminf(__shfl_sync(0xffffffffu, ld[j], p.thr_rank), qt[j]);
          int base = 0;
#pragma unroll
          for (int m = 0; m < kPRows / 32; ++m) {
            const float v = edist[g * kPRows + m * 32 + lane] + qn[j];
            bool pass = v < thr;
            unsigned mask = __ballot_sync(0xffffffffu, pass);
            if (base + __popc(mask) > 32) {
              __syncwarp();
              const float bd = lane < base ? sd[lane] : kPInf;
              const long long bk = lane < base ? sk[lane] : kPNoKey;
              warp_merge32(ld[j], lk[j], bd, bk, lane);
              thr = fminf(__shfl_sync(0xffffffffu, ld[j], p.thr_rank), qt[j]);
              base = 0;
              pass = v < thr;
              mask = __ballot_sync(0xffffffffu, pass);
              __syncwarp();
            }
            if (pass) {
              const int pos = base + __popc(mask & ((1u << lane) - 1u));
              sd[pos] = v;
              sk[pos] = gbase + m * 32 + lane;
            }
            base += __popc(mask);
          }
          if (base > 0) {
            __syncwarp();
            if (base <= 3) {
              for (int i = 0; i < base; ++i) warp_insert1(ld[j], lk[j], sd[i], sk[i], lane);
            } else {
              const float bd = lane < base ? sd[lane] : kPInf;
              const long long bk = lane < base ? sk[lane] : kPNoKey;
              warp_merge32(ld[j], lk[j], bd, bk, lane);
            }
            __syncwarp();
          }
        }
      }
      // this CTA's per-query top-32 of the tile -> one partial list per query (slot reservations and
      // threshold updates issued together, one lane per query)
      int myqid = 0, myps = 0;
      bool myhas = false;
      float myl31 = kPInf;
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int g = ew + 4 * j;
        const float l31 = __shfl_sync(0xffffffffu, ld[j], p.thr_rank);
        const bool has = g < nq && __shfl_sync(0xffffffffu, ld[j], 0) != kPInf;
        if (lane == j) {
          myhas = has;
          myl31 = l31;
          if (g < nq) myqid = __ldg(p.list_q + T.qoff + g);
        }
      }
      if (myhas) {
        myps = atomicAdd(p.part_count + myqid, 1);
        if (myl31 != kPInf) atomicMin(p.qthr + myqid, f2ord(myl31));
      }
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int ps = __shfl_sync(0xffffffffu, myps, j);
        const int qid = __shfl_sync(0xffffffffu, myqid, j);
        const bool has = __shfl_sync(0xffffffffu, myhas ? 1 : 0, j) != 0;
        if (has && ps < p.part_cap) {
          const size_t o = ((size_t)qid * p.part_cap + ps) * kTopK + lane;
          p.part_dist[o] = ld[j];
          p.part_row[o] = lk[j] == kPNoKey ? -1 : (int)lk[j];
        }
      }
    }
  }

#ifdef RD_STALL_PROF
  if (p.stall && lane == 0 && (warp == 0 || warp == 1 || warp == 2)) {  // leader CTA's roles, like scan_tc.cu
    unsigned long long* o = p.stall + (size_t)blockIdx.x * 12;
    if (warp == 0) {
      o[0] = stall_acc[0], o[1] = stall_acc[1], o[2] = stall_acc[2], o[9] = clock64() - t_begin;
    } else if (warp == 1) {
      o[3] = stall_acc[3], o[4] = stall_acc[4], o[5] = stall_acc[5], o[6] = stall_acc[6];
    } else {
      o[8] = stall_acc[8];
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs done with the pair's TMEM and shared memory
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem, kPTmemCols);
  }
}

}  // namespace

int scan_pair_stages(int d, bool resid) {
  if (d % 64 != 0) return 0;
  if (resid) return pair_smem_bytes_for<10, true>(d) <= 227 * 1024 ? 10 : pair_smem_bytes_for<8, true>(d) <= 227 * 1024 ? 8 : 0;
  if (pair_smem_bytes_for<5>(d) <= 227 * 1024) return 5;
  if (pair_smem_bytes_for<4>(d) <= 227 * 1024) return 4;
  if (pair_smem_bytes_for<3>(d) <= 227 * 1024) return 3;
  return 0;
}

cudaError_t launch_scan_pair(const CUtensorMap& map128, const CUtensorMap& map32, const CUtensorMap& qmap,
                             const TcScanParams& p, int num_sms, cudaStream_t s, bool resid) {
  const int S = scan_pair_stages(p.d, resid);
  const dim3 grid((unsigned)(num_sms / 2 * 2));
  if (resid) {
    if (S == 10)
      return launch_k(ivf_scan_pair_kernel<10, true>, grid, dim3(kPThreads), pair_smem_bytes_for<10, true>(p.d), s,
                      map128, map32, qmap, p);
    if (S == 8)
      return launch_k(ivf_scan_pair_kernel<8, true>, grid, dim3(kPThreads), pair_smem_bytes_for<8, true>(p.d), s,
                      map128, map32, qmap, p);
    return cudaErrorInvalidValue;
  }
  switch (S) {
    case 5:
      return launch_k(ivf_scan_pair_kernel<5, false>, grid, dim3(kPThreads), pair_smem_bytes_for<5>(p.d), s, map128,
                      map32, qmap, p);
    case 4:
      return launch_k(ivf_scan_pair_kernel<4, false>, grid, dim3(kPThreads), pair_smem_bytes_for<4>(p.d), s, map128,
                      map32, qmap, p);
    case 3:
      return launch_k(ivf_scan_pair_kernel<3, false>, grid, dim3(kPThreads), pair_smem_bytes_for<3>(p.d), s, map128,
                      map32, qmap, p);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace rd
