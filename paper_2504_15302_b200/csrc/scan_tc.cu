// scan_tc.cu — N5: the inverted-list scan on the 5th-gen tensor cores (tcgen05, sm_100a),
// for tiles whose list is probed by >= kTcMinQ queries of the batch.
//
// Per 128-row tile of a list chunk, D = X . Q^T is formed in TMEM with fp32-level
// accuracy by a "bf16x3" split, x = x1 + x2 and q = q1 + q2 (each a bf16, RN):
//   MMA_a (kind::f16, A = x1 from TMEM, B = [q1 ; q2], N = 64)
//   MMA_b (kind::f16, A = x2 from TMEM, B = q1,        N = 32)
//   q.x = D_a[q1] + D_a[q2] + D_b  (missing only x2.q2 and the rounding of the
//   second terms, ~2^-17 relative — inside the margin merge.cu certifies).
// Every tcgen05.mma costs ~94+ cycles whatever its N (measured), so the design
// minimises instructions per byte of x: 4 MMAs per 16 KiB stage (128 rows x
// 32 dims), A operands in TMEM so the smem ring is released as soon as the
// converter warps have read it.
// Roles (10 warps, one persistent CTA per SM):
//   warp 0        TMA producer: [32 dims x 128 rows] fp32 boxes, 128B swizzle, 6-stage ring
//   warp 1        TMEM allocator + single-thread MMA issuer
//   warps 2-5     converter group 0 (even stages): fp32 x -> (x1, x2) bf16 pairs into an
//                 8-deep TMEM ring; also loads each tile's query operand B (bf16, K-major SW128)
//   warps 10-13   converter group 1 (odd stages)
//   warps 6-9     epilogue: tcgen05.ld of D, d~ = ||x||^2 + ||q||^2 - 2 q.x, per-query
//                 warp top-32 with threshold filter + bitonic merge, partial lists out
#include <cuda_bf16.h>

#include <algorithm>

#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr int kRows = kTcRows;               // 128 = UMMA M
constexpr int kStageBytes = kRows * 128;     // 16 KiB: 128 rows x 32 fp32
// Tile width: kG queries per tile (B operand rows: kG q1 + kG q2, 64 dims per slice).
// Pre-split path, 16-query tiles, streamed operand (kSB, chosen by the host for batches of about
// one query per probed list or fewer): every ring stage carries its own slice of the query operand
// next to the x1 / x2 tiles (x1 16 KiB | x2 16 KiB | 4 KiB B slice), re-gathered from L2 per stage,
// so no shared memory is spent on a resident operand: 6 stages (192 KiB of HBM loads in flight
// instead of 160) and tiles change without draining the ring (B200: +2 % at 1-2 queries). The
// per-stage gathers grow with the queries per tile (-4.7 % at 512 queries, ~8 per list), and for
// 32-query tiles streaming measured 11 % slower at 1024 queries: those keep a resident operand
// with 5 / 3 x 32 KiB stages. Converter path (fp32 x): 16 KiB stages, resident operand.
template <int kG>
struct TcGeom {
  static constexpr int Stages = kG == 16 ? 10 : 6;  // converter path / resident operand: 16 KiB units
  static constexpr int BRows = 2 * kG;
  static constexpr int BSlice = BRows * 128;
};
// ring depth / stage bytes of a (path, width, streamed operand) variant
#ifndef RD_RESH_S32  // fp16 residual scan: half the resident operand, deeper rings
#define RD_RESH_S32 10
#endif
#ifndef RD_RESH_S16
#define RD_RESH_S16 11
#endif
#ifndef RD_RESH_SSB
#define RD_RESH_SSB 11
#endif
#ifndef RD_RES_S32  // residual-store ring depths (16 KiB stages; A/B builds override)
#define RD_RES_S32 6
#endif
#ifndef RD_RES_S16
#define RD_RES_S16 10
#endif
#ifndef RD_RES_SSB
#define RD_RES_SSB 10
#endif
// kRes (residual plane, implies kPre): one 16 KiB r1 tile per stage instead of x1 | x2, so twice the
// stages in the same bytes
// query-operand rows per tile: [q1; q2] (bf16 split), or q1 alone for the fp16 residual scan (kH)
template <int kG, bool kH>
struct BGeom {
  static constexpr int Rows = kH ? kG : 2 * kG;
  static constexpr int Slice = Rows * 128;
};
template <bool kPre, int kG, bool kSB, bool kRes = false, bool kH = false>
struct Ring {
  static_assert(!kSB || (kPre && kG == 16), "streamed operand: pre-split 16-query tiles only");
  static_assert(!kRes || kPre, "the residual plane is read straight into smem");
  static constexpr int S = kH ? (kSB ? RD_RESH_SSB : (kG == 16 ? RD_RESH_S16 : RD_RESH_S32))
                         : kRes ? (kSB ? RD_RES_SSB : (kG == 16 ? RD_RES_S16 : RD_RES_S32))
                                : kPre ? (kSB ? 6 : TcGeom<kG>::Stages / 2) : TcGeom<kG>::Stages;
  static constexpr int B = kRes ? kRows * 128 + (kSB ? BGeom<kG, kH>::Slice : 0)
                                : kPre ? 2 * kRows * 128 + (kSB ? TcGeom<kG>::BSlice : 0) : kRows * 128;
  // converter group g owns stages / TMEM buffers with u % 2 == g; an odd ring depth would let one
  // group wait on a phase two ahead of the other group's and alias its mbarrier parity
  static_assert(TcGeom<kG>::Stages % 2 == 0, "x ring depth must be even");
  static_assert(kG == 16 || kG == 32, "tile width");
};
constexpr int kXBufs = 8;                    // TMEM ring of converted stages (32 columns each)
static_assert(kXBufs % 2 == 0, "TMEM ring depth must be even");
constexpr int kThreads = 448;                // 14 warps
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCols = 128;           // per accumulator buffer: D_a (64) + D_b (32)
constexpr uint32_t kXCol0 = 2 * kAccCols;    // first TMEM column of the x ring
constexpr float kInf = __builtin_huge_valf();
constexpr long long kNoKey = 0x7fffffffffffffffll;

struct Smem {
  uint32_t xs;  // shared-space address of stage 0
  uint32_t bs;  // shared-space address of the B operand
  uint64_t *full, *empty, *xfull, *xempty, *afull, *aempty, *bfull, *bempty, *tfull, *tempty;
  int* tring;
  uint32_t* tmem_base;
  float* edist;       // [2][kTcG][kRows] epilogue exchange
  float* stage_d;     // [4][32] per-warp compaction batch
  long long* stage_k; // [4][32]
};

template <bool kPre, int kG, bool kSB, bool kRes, bool kH>
__device__ __forceinline__ Smem carve(unsigned char* raw, int d) {
  constexpr int kStages = Ring<kPre, kG, kSB, kRes, kH>::S, kBSlice = BGeom<kG, kH>::Slice;
  // ring bytes (+ the resident operand unless the stages carry it)
  const size_t xring = (size_t)kStages * Ring<kPre, kG, kSB, kRes, kH>::B;
  const size_t ring = xring + (kSB ? 0 : (size_t)(d / 64) * kBSlice);
  Smem s;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  s.xs = smem_u32(base);
  s.bs = s.xs + (uint32_t)xring;  // resident operand (unused when streamed)
  uint64_t* b = reinterpret_cast<uint64_t*>(base + ring);
  s.full = b;
  s.empty = s.full + kStages;
  s.xfull = s.empty + kStages;
  s.xempty = s.xfull + kXBufs;
  s.afull = s.xempty + kXBufs;
  s.aempty = s.afull + 2;
  s.bfull = s.aempty + 2;
  s.bempty = s.bfull + 1;
  s.tfull = s.bempty + 1;
  s.tempty = s.tfull + 2;
  s.tring = reinterpret_cast<int*>(s.tempty + 2);
  s.tmem_base = reinterpret_cast<uint32_t*>(s.tring + 2);
  s.stage_k = reinterpret_cast<long long*>(s.tmem_base + 2);   // 8 B aligned
  s.stage_d = reinterpret_cast<float*>(s.stage_k + 4 * 32);
  s.edist = s.stage_d + 4 * 32;
  return s;
}

// profiling only (built with -DRD_STALL_PROF and run with p.stall != nullptr): cycles a role
// spends blocked on one barrier. The shipped build compiles it to a plain wait.
#ifdef RD_STALL_PROF
#define RD_TWAIT(bar, parity, slot)                                  \
  do {                                                               \
    if (p.stall) {                                                   \
      const long long t0_ = clock64();                               \
      mbar_wait(bar, parity);                                        \
      stall_acc[slot] += clock64() - t0_;                            \
    } else {                                                         \
      mbar_wait(bar, parity);                                        \
    }                                                                \
  } while (0)
#else
#define RD_TWAIT(bar, parity, slot) mbar_wait(bar, parity)
#endif

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x = lo -> low 16 bits
  return *reinterpret_cast<const uint32_t*>(&v);
}

// kPre = false: fp32 arena; converter warps split x into (x1, x2) in TMEM; TS MMAs, 32-dim stages.
// kPre = true : pre-split bf16 (x1, x2) arena ([rows][2][d], built with the index); the producer TMA-loads
//               both 64-dim tiles of a stage straight into 128B-swizzled smem and the MMAs read A from
//               smem (SS) — no conversion on the scan path; converter warps are idle.
// kRes: the residual store (resid.cu): A = r1 = bf16(x - c_list) [rows][d], B = the queries' split
//       [q1; q2] as for the split3 store, one MMA per K step (D = r1 . q); xnorm is the row constant
//       ||x - c||^2 + 2 c . r1 and the per-(query, list) term ||q - c||^2 - eps comes from the coarse
//       stage's distance (resid_pair_term), so every key is a lower bound on the exact distance:
//       key = ||q - c||^2 - eps + ||r||^2 + 2 c . r1 - 2 r1 . q.
// kH (implies kRes): the fp16 residual scan — r1 = fp16(x - c) and B = fp16(q) alone (N = G): 2^-11
//       roundings instead of bf16's 2^-9 leave q's split out; half the operand, twice the ring.
template <bool kPre, int kG, bool kSB, bool kRes, bool kH>
__global__ void __launch_bounds__(kThreads, 1)
    ivf_scan_tc_kernel(const __grid_constant__ CUtensorMap map128, const __grid_constant__ CUtensorMap map32,
                       const __grid_constant__ CUtensorMap qmap, const TcScanParams p) {
  constexpr int kTcG = kG, kStages = Ring<kPre, kG, kSB, kRes, kH>::S, kBRows = BGeom<kG, kH>::Rows,
                kBSlice = BGeom<kG, kH>::Slice;
  static_assert(!kH || kRes, "fp16 operands: residual store only");
  constexpr bool kStream = kSB;  // the query operand travels with the stages
  constexpr bool kHalfN = kPre && !kSB && kG == 32;  // half-N MMAs for tiles of <= 16 queries
  RD_PDL_PROLOGUE();
  if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 4 + 0] = gtimer();
  extern __shared__ unsigned char smem_raw[];
  const int d = p.d, nks = kPre ? d / 64 : d / 32;
  const Smem sm = carve<kPre, kG, kSB, kRes, kH>(smem_raw, d);
  // ring geometry: kStages stages of RB bytes (pre-split: x1 | x2 [| B slice]; converter: fp32 x)
  constexpr int RS = kStages;
  constexpr int RB = Ring<kPre, kG, kSB, kRes, kH>::B;
  constexpr int kXTiles = kRes ? 1 : 2;  // A tiles per stage (r1; or x1, x2)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kPre ? 1 : 4);  // MMA commit (pre-split) or the 4 converter warps
    }
    for (int i = 0; i < kXBufs; ++i) {
      mbar_init(&sm.xfull[i], 4);
      mbar_init(&sm.xempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.afull[i], 1);
      mbar_init(&sm.aempty[i], 4);
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], kPre ? 1 + 4 : 1 + 4 + 4 + 4);
    }
    mbar_init(sm.bfull, 1);
    mbar_init(sm.bempty, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(sm.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sm.tmem_base;
  const int ntiles = *p.ntiles;
#ifdef RD_STALL_PROF
  long long stall_acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_begin = clock64();
#endif
  if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 4 + 1] = gtimer();

  // ---------------------------------------------------------------- warp 0: TMA producer
  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&map128);
      prefetch_tmap(&map32);
      prefetch_tmap(&qmap);
    }
    uint32_t u = 0;
    const int nslices = d / 64;
    // The queue is read one tile ahead: the next tile's index (atomic) and descriptor are fetched
    // while the current tile's first stages go out, so a tile switch exposes no global round trip
    // (they cost ~1 us each; at small batches, with a few tiles per CTA, that showed as CTAs with
    // one more tile ending several us later).
    int tn = 0;
    ScanTile Tn{};
    if (lane == 0) tn = atomicAdd(p.tile_counter, 1);
    tn = __shfl_sync(0xffffffffu, tn, 0);
    if (tn < ntiles) Tn = p.tiles[tn];
    auto fetch_next = [&]() {  // after the current tile's first stages are issued
      tn = __shfl_sync(0xffffffffu, tn, 0);
      if (tn < ntiles) Tn = p.tiles[tn];
    };
    for (uint32_t ti = 0;; ++ti) {
      const int t = tn;
      const int slot = ti & 1;
      if (lane == 0) {
        RD_TWAIT(&sm.tempty[slot], ((ti >> 1) & 1) ^ 1, 0);
        sm.tring[slot] = t < ntiles ? t : -1;
        mbar_arrive(&sm.tfull[slot]);
      }
      __syncwarp();
      if (t >= ntiles) break;
      const ScanTile T = Tn;
      if (lane == 0) tn = atomicAdd(p.tile_counter, 1);  // consumed by fetch_next
      // x stage i of this tile: row tile i / nks, 64- (or 32-) dim slice i % nks; lane 0 issues
      const int nst = ((T.nrows + kRows - 1) / kRows) * nks;
      if constexpr (kStream) {
        // Each stage: x1 and x2 tiles of the slice (lane 0, TMA) and the slice of the query operand
        // (TMA gather4 from the L2-resident split queries: rows 0..kG-1 q1, kG..2kG-1 q2; lane qi
        // < 2 qq loads quad qi; padding rows repeat the tile's last query; quads beyond the tile's
        // queries keep stale rows whose D columns the epilogue never reads).
        const int qq = (T.nq + 3) >> 2, per = kH ? qq : 2 * qq;
        const int part = !kH && lane >= qq ? 1 : 0;
        const int g0 = (lane - part * qq) * 4;
        const uint32_t boff = kXTiles * kRows * 128 + (part * (kTcG / 4) + g0 / 4) * 512;
        int r[4] = {0, 0, 0, 0};
        if (lane < per)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            r[i] = (kH ? 1 : 2) * __ldg(p.list_q + T.qoff + min(g0 + i, T.nq - 1)) + part;
        for (int i = 0; i < nst; ++i, ++u) {
          const int rt = i / nks, ks = i - rt * nks;
          const int rows = min(kRows, T.nrows - rt * kRows);
          const int nb = (rows + 31) >> 5;
          const int row = (int)(T.src_row + rt * kRows);
          const int s = u % RS;
          const uint32_t dst = sm.xs + s * RB;
          if (lane == 0) {
            RD_TWAIT(&sm.empty[s], ((u / RS) & 1) ^ 1, 1);
            mbar_arrive_expect_tx(&sm.full[s], (uint32_t)(kXTiles * nb * 4096 + per * 512));
          }
          __syncwarp();
          if (lane < per) tma_gather4_u32(dst + boff, &qmap, ks * 64, r[0], r[1], r[2], r[3], &sm.full[s]);
          if (kRes && lane == 0) {
            if (nb == 4) {
              tma_load_2d_u32(dst, &map128, ks * 64, row, &sm.full[s]);
            } else {
              for (int b = 0; b < nb; ++b) tma_load_2d_u32(dst + b * 4096, &map32, ks * 64, row + b * 32, &sm.full[s]);
            }
          } else if (lane == 0) {
            if (nb == 4) {
              tma_load_3d_u32(dst, &map128, ks * 64, 0, row, &sm.full[s]);
              tma_load_3d_u32(dst + kRows * 128, &map128, ks * 64, 1, row, &sm.full[s]);
            } else {
              for (int b = 0; b < nb; ++b) {
                tma_load_3d_u32(dst + b * 4096, &map32, ks * 64, 0, row + b * 32, &sm.full[s]);
                tma_load_3d_u32(dst + kRows * 128 + b * 4096, &map32, ks * 64, 1, row + b * 32, &sm.full[s]);
              }
            }
          }
          if (i == 0) fetch_next();
        }
        continue;
      }
      auto issue_x = [&](int i) {
        const int rt = i / nks, ks = i - rt * nks;
        const int rows = min(kRows, T.nrows - rt * kRows);
        const int nb = (rows + 31) >> 5;
        const int row = (int)(T.src_row + rt * kRows);
        const int s = u % RS;
        RD_TWAIT(&sm.empty[s], ((u / RS) & 1) ^ 1, 1);
        const uint32_t dst = sm.xs + s * RB;
        if constexpr (kRes) {  // the r1 tile of a 64-dim slice: 16 KiB
          if (nb == 4) {
            mbar_arrive_expect_tx(&sm.full[s], kRows * 128);
            tma_load_2d_u32(dst, &map128, ks * 64, row, &sm.full[s]);
          } else {
            mbar_arrive_expect_tx(&sm.full[s], nb * 4096);
            for (int b = 0; b < nb; ++b) tma_load_2d_u32(dst + b * 4096, &map32, ks * 64, row + b * 32, &sm.full[s]);
          }
        } else if constexpr (kPre) {  // x1 and x2 tiles of a 64-dim slice: 2 x 16 KiB
          if (nb == 4) {
            mbar_arrive_expect_tx(&sm.full[s], 2 * kRows * 128);
            tma_load_3d_u32(dst, &map128, ks * 64, 0, row, &sm.full[s]);
            tma_load_3d_u32(dst + kRows * 128, &map128, ks * 64, 1, row, &sm.full[s]);
          } else {
            mbar_arrive_expect_tx(&sm.full[s], 2 * nb * 4096);
            for (int b = 0; b < nb; ++b) {
              tma_load_3d_u32(dst + b * 4096, &map32, ks * 64, 0, row + b * 32, &sm.full[s]);
              tma_load_3d_u32(dst + kRows * 128 + b * 4096, &map32, ks * 64, 1, row + b * 32, &sm.full[s]);
            }
          }
        } else {
          if (nb == 4) {
            mbar_arrive_expect_tx(&sm.full[s], kStageBytes);
            tma_load_2d_u32(dst, &map128, ks * 32, row, &sm.full[s]);
          } else {
            mbar_arrive_expect_tx(&sm.full[s], nb * 4096);
            for (int b = 0; b < nb; ++b) tma_load_2d_u32(dst + b * 4096, &map32, ks * 32, row + b * 32, &sm.full[s]);
          }
        }
        ++u;
      };
      // ---- B operand by TMA gather4: rows 0-31 q1, 32-63 q2 of the tile's queries (qsplit row
      // 2*qid + part); padding rows repeat the last query (their D columns are ignored). Only the
      // quads holding real queries are loaded; the others keep stale rows whose D columns the
      // epilogue never reads. Lane (grp, qi) owns quad qi of part qi / qq for slices grp, grp + ngrp..
      const int qq = (T.nq + 3) >> 2;  // quads per part
      const int per = kH ? qq : 2 * qq, ngrp = 32 / per, grp = lane / per, qi = lane - grp * per;
      const int part = !kH && qi >= qq ? 1 : 0;
      const int g0 = (qi - part * qq) * 4;
      int r[4];
      if (grp < ngrp)  // the ids load while the ring is refilled below
#pragma unroll
        for (int i = 0; i < 4; ++i)
          r[i] = (kH ? 1 : 2) * __ldg(p.list_q + T.qoff + min(g0 + i, T.nq - 1)) + part;
      // the first ring's worth of this tile's x stages go out before the wait for the B operand
      // buffer (free once the previous tile's MMAs are done), so HBM keeps streaming across the
      // tile boundary and only the gather's latency is exposed
      const int npre = min(nst, RS);
      if (lane == 0)
        for (int i = 0; i < npre; ++i) issue_x(i);
      __syncwarp();
      fetch_next();
      RD_TWAIT(sm.bempty, (ti & 1) ^ 1, 2);
      // one barrier for the whole gather (per-slice barriers let the first MMAs start earlier but
      // cost more than they saved: A/B on B200, 1024 queries, 206.4k vs 207.2k q/s)
      if (lane == 0) mbar_arrive_expect_tx(sm.bfull, (uint32_t)(nslices * per * 512));
      __syncwarp();
      if (grp < ngrp) {
        // half tiles (<= 16 queries of a 32-wide tile): q2 right after q1 (rows 16-31), so the MMAs run
        // at half N (see the MMA issuer)
        const bool half = kHalfN && T.nq <= kTcG / 2;
        const uint32_t dst = sm.bs + (part * (half ? kTcG / 8 : kTcG / 4) + g0 / 4) * 512;
        for (int slice = grp; slice < nslices; slice += ngrp)
          tma_gather4_u32(dst + slice * kBSlice, &qmap, slice * 64, r[0], r[1], r[2], r[3], sm.bfull);
      }
      if (lane == 0)
        for (int i = npre; i < nst; ++i) issue_x(i);
      __syncwarp();
    }
  }
  // ---------------------------------------------------------------- warp 1: MMA issuer
  else if (warp == 1) {
    // per tile: full N (x1.[q1;q2] N = 64, x2.q1 N = 32) or, for tiles of <= 16 queries in the
    // 32-wide scan, half N (32, 16) over the compacted operand — half the tensor work (and power)
    const uint32_t ida_full = kH ? idesc_f16(kRows, kBRows) : idesc_bf16(kRows, kBRows), idb_full = idesc_bf16(kRows, kTcG);
    const uint32_t ida_half = kH ? idesc_f16(kRows, kBRows / 2) : idesc_bf16(kRows, kBRows / 2),
                   idb_half = idesc_bf16(kRows, kTcG / 2);
    const unsigned char* bs_ptr = reinterpret_cast<unsigned char*>(smem_raw) + (sm.bs - smem_u32(smem_raw));
    const uint64_t bdesc0 = umma_desc_sw128(bs_ptr);
    uint32_t u = 0, rtc = 0;
    long long dbg_rows = 0;
    for (uint32_t ti = 0;; ++ti) {
      const int slot = ti & 1;
      RD_TWAIT(&sm.tfull[slot], (ti >> 1) & 1, 3);
      const int t = sm.tring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.tempty[slot]);
      if (t < 0) {
        if (p.dbg && lane == 0) {  // profiling only: tiles and rows this CTA scanned
          p.dbg[4 * gridDim.x + blockIdx.x] = ti;
          p.dbg[5 * gridDim.x + blockIdx.x] = dbg_rows;
        }
        break;
      }
      const ScanTile T = p.tiles[t];
      dbg_rows += T.nrows;
      const bool half = kHalfN && T.nq <= kTcG / 2;
      const uint32_t ida = half ? ida_half : ida_full, idb = half ? idb_half : idb_full;
      if (p.dbg && ti == 0 && lane == 0) p.dbg[blockIdx.x * 4 + 2] = gtimer();
      for (int rt = 0; rt * kRows < T.nrows; ++rt, ++rtc) {
        const int a = rtc & 1;
        RD_TWAIT(&sm.aempty[a], ((rtc >> 1) & 1) ^ 1, 5);
        tc_fence_after();
        const uint32_t dacc = tmem + a * kAccCols;
        for (int ks = 0; ks < nks; ++ks, ++u) {
          if (!kStream && rt == 0 && ks == 0) RD_TWAIT(sm.bfull, ti & 1, 4);  // the tile's queries are in B
          if constexpr (kPre) {  // (streamed: x1, x2 and the query slice all arrive with the stage)
            const int s = u % RS;
            RD_TWAIT(&sm.full[s], (u / RS) & 1, 6);
            tc_fence_after();
            if (lane == 0) {
              const unsigned char* st = reinterpret_cast<unsigned char*>(smem_raw) + (sm.xs - smem_u32(smem_raw)) +
                                        s * RB;
              const uint64_t a1 = umma_desc_sw128(st), a2 = umma_desc_sw128(st + kRows * 128);
              const uint64_t bd = kStream ? umma_desc_sw128(st + kXTiles * kRows * 128)
                                          : bdesc0 + (uint64_t)(ks * (kBSlice >> 4));
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t acc = (ks | kk) != 0;
                if (p.debug_skip & 4) continue;  // profiling only: no MMAs (RD_DEBUG_SKIP)
                mma_bf16_ss(dacc, a1 + kk * 2, bd + (uint64_t)(kk * 2), ida, acc);
                if constexpr (!kRes) mma_bf16_ss(dacc + kBRows, a2 + kk * 2, bd + (uint64_t)(kk * 2), idb, acc);
              }
              tc_commit(&sm.empty[s]);
            }
            __syncwarp();
            continue;
          }
          const int xb = u % kXBufs;
          mbar_wait(&sm.xfull[xb], (u / kXBufs) & 1);
          tc_fence_after();
          if (lane == 0) {
            // B: 64-dim bf16 slice ks/2, byte offset 64*(ks&1) + 32*kk inside the 128 B swizzle row
            const uint64_t bd = bdesc0 + (uint64_t)((ks >> 1) * (kBSlice >> 4) + (ks & 1) * 4);
            const uint32_t xa = tmem + kXCol0 + xb * 32;
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const uint32_t acc = (ks | kk) != 0;
              if (p.debug_skip & 4) continue;
              mma_bf16_ts(dacc, xa + kk * 8, bd + (uint64_t)(kk * 2), ida, acc);
              mma_bf16_ts(dacc + kBRows, xa + 16 + kk * 8, bd + (uint64_t)(kk * 2), idb, acc);
            }
            tc_commit(&sm.xempty[xb]);
          }
          __syncwarp();
        }
        if (lane == 0) tc_commit(&sm.afull[a]);
        __syncwarp();
      }
      if (!kStream && lane == 0) tc_commit(sm.bempty);  // (streamed: the operand travels with the stages)
      __syncwarp();
    }
  }
  // ------------------------------------------------- warps 2-5 / 10-13: converter groups 0 / 1
  else if (warp < 6 || warp >= 10) {
    if constexpr (kPre) goto done;  // no conversion on the pre-split path
    const int quarter = warp & 3;
    const int grp = warp >= 10;
    const int r = quarter * 32 + lane;
    uint32_t u = 0;
    // Software-pipelined: the TMEM stores of stage u complete (wait::st) while stage u+2 is being
    // converted; xfull[u] is published one iteration late (the 8-deep TMEM ring absorbs it) and
    // always before this warp blocks on the next tile.
    int pend = -1;  // TMEM buffer whose stores are in flight
    auto flush = [&]() {
      if (pend >= 0) {
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.xfull[pend]);
        pend = -1;
      }
    };
    for (uint32_t ti = 0;; ++ti) {
      const int slot = ti & 1;
      flush();
      mbar_wait(&sm.tfull[slot], (ti >> 1) & 1);
      const int t = sm.tring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.tempty[slot]);
      if (t < 0) break;
      const ScanTile T = p.tiles[t];
      for (int rt = 0; rt * kRows < T.nrows; ++rt) {
        for (int ks = 0; ks < nks; ++ks, ++u) {
          if ((int)(u & 1) != grp) continue;
          const int s = u % kStages, xb = u % kXBufs;
          mbar_wait(&sm.full[s], (u / kStages) & 1);
          const uint32_t row = sm.xs + s * kStageBytes + r * 128;
          uint32_t b1[16], b2[16];
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (p.debug_skip & 2) {
              b1[2 * g] = b1[2 * g + 1] = b2[2 * g] = b2[2 * g + 1] = 0u;
              continue;
            }
            const uint4 v = lds128(row + ((g ^ (r & 7)) << 4));
            const float x0 = __uint_as_float(v.x), x1 = __uint_as_float(v.y);
            const float x2 = __uint_as_float(v.z), x3 = __uint_as_float(v.w);
            const __nv_bfloat162 h01 = __floats2bfloat162_rn(x0, x1), h23 = __floats2bfloat162_rn(x2, x3);
            b1[2 * g] = *reinterpret_cast<const uint32_t*>(&h01);
            b1[2 * g + 1] = *reinterpret_cast<const uint32_t*>(&h23);
            b2[2 * g] = pack_bf16x2(x0 - __low2float(h01), x1 - __high2float(h01));
            b2[2 * g + 1] = pack_bf16x2(x2 - __low2float(h23), x3 - __high2float(h23));
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[s]);
          flush();  // previous stage's stores have had a whole conversion to land
          mbar_wait(&sm.xempty[xb], ((u / kXBufs) & 1) ^ 1);
          tc_fence_after();
          const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + kXCol0 + xb * 32;
          tmem_st16(ta, b1);
          tmem_st16(ta + 16, b2);
          pend = xb;
          if (p.debug_skip & 8) flush();  // A/B switch: unpipelined stores
        }
      }
    }
  }
  // ---------------------------------------------------------------- warps 6-9: epilogue
  else {
    constexpr int kOwn = kTcG / 4;  // queries owned per epilogue warp
    // Each warp reads D for its 32-lane quarter (rows), publishes d~ for all 16 queries to smem,
    // then owns queries ew, ew+4, ew+8, ew+12 over all 128 rows: candidates below the query's
    // running 32nd-best are compacted into one batch and merged (one bitonic merge per row tile
    // at most once the list has warmed up).
    const int quarter = warp & 3, ew = warp - 6;
    float* edist = sm.edist;                          // [kTcG][kRows]
    float* sd = sm.stage_d + ew * 32;                 // per-warp compaction batch
    long long* sk = sm.stage_k + ew * 32;
    uint32_t rtc = 0;
    // Per owned slot j: the query whose running top-32 the slot holds (cq, -1: none) and that list.
    // A list is written out (one partial list) only when the slot's query changes or the CTA runs
    // out of tiles: consecutive tiles of one query — the chunks of a list, and every tile at B = 1 —
    // keep one list, so the merge reads far fewer partials (B = 1: ~5 per CTA -> 1).
    float ld[kOwn];
    long long lk[kOwn];
    int cq[kOwn];
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      ld[j] = kInf;
      lk[j] = kNoKey;
      cq[j] = -1;
    }
    // writes out the lists of the slots in fmask (slot reservations issued together, one lane per
    // slot: one atomic round trip per flush) and empties them
    auto flush = [&](unsigned fmask) {
      int myqid = 0, myps = 0;
      bool myhas = false;
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const bool has = ((fmask >> j) & 1u) && cq[j] >= 0 && __shfl_sync(0xffffffffu, ld[j], 0) != kInf;
        if (lane == j) {
          myhas = has;
          myqid = cq[j];
        }
      }
      if (myhas) myps = atomicAdd(p.part_count + myqid, 1);
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int ps = __shfl_sync(0xffffffffu, myps, j);
        const bool has = __shfl_sync(0xffffffffu, myhas ? 1 : 0, j) != 0;
        if (has && ps < p.part_cap) {
          const size_t o = ((size_t)cq[j] * p.part_cap + ps) * kTopK + lane;
          p.part_dist[o] = ld[j];
          p.part_row[o] = lk[j] == kNoKey ? -1 : (int)lk[j];
        }
        if ((fmask >> j) & 1u) {
          ld[j] = kInf;
          lk[j] = kNoKey;
        }
      }
    };
    for (uint32_t ti = 0;; ++ti) {
      const int slot = ti & 1;
      RD_TWAIT(&sm.tfull[slot], (ti >> 1) & 1, 7);
      const int t = sm.tring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.tempty[slot]);
      if (t < 0) {
        flush((1u << kOwn) - 1u);
        break;
      }
      const ScanTile T = p.tiles[t];
      const int nq = T.nq;
      int nqid[kOwn];
      unsigned fmask = 0;
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const int g = ew + 4 * j;
        nqid[j] = g < nq ? __ldg(p.list_q + T.qoff + g) : -1;
        if (nqid[j] != cq[j]) fmask |= 1u << j;
      }
      if (fmask) flush(fmask);
      float qn[kOwn], qt[kOwn];  // ||q||^2 of the owned queries (added by the owner, not per row)
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        cq[j] = nqid[j];
        qn[j] = cq[j] >= 0 ? __ldg(p.qnorm + cq[j]) : 0.f;
        if (kRes && cq[j] >= 0) qn[j] = resid_pair_term(p, qn[j], cq[j], T.list);
        qt[j] = cq[j] >= 0 ? ord2f(*(volatile int*)(p.qthr + cq[j])) : kInf;
      }
      for (int rt = 0; rt * kRows < T.nrows; ++rt, ++rtc) {
        const int a = rtc & 1;
        RD_TWAIT(&sm.afull[a], (rtc >> 1) & 1, 8);
        tc_fence_after();
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + a * kAccCols;
        // D_a = [x1.q1 | x1.q2] in columns [0, 2 kTcG) (half tiles: [0, kTcG) with x1.q2 from kTcG / 2),
        // D_b = x2.q1 in [2 kTcG, 3 kTcG)
        uint32_t d1[kTcG], d2[kTcG], d3[kTcG];
        const uint32_t c2 = (kHalfN && nq <= kTcG / 2) ? kTcG / 2 : kTcG;
#pragma unroll
        for (int c = 0; c < kTcG; c += 16) {
          RD_TMEM_LD16(ta + c, (d1 + c));
          if constexpr (!kH) RD_TMEM_LD16(ta + c2 + c, (d2 + c));
          if constexpr (!kRes) RD_TMEM_LD16(ta + 2 * kTcG + c, (d3 + c));
        }
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.aempty[a]);
        const int r = quarter * 32 + lane;
        const int rloc = rt * kRows + r;
        const bool valid = rloc < T.nrows;
        const float xn = valid ? __ldg(p.xnorm + T.grow0 + rloc) : 0.f;
        float* eb = edist;
        named_bar_sync(2, 128);  // every owner finished reading the previous row tile
#pragma unroll
        for (int g = 0; g < kTcG; ++g) {
          float dot = kH     ? __uint_as_float(d1[g])
                      : kRes ? __uint_as_float(d1[g]) + __uint_as_float(d2[g])
                             : (__uint_as_float(d1[g]) + __uint_as_float(d2[g])) + __uint_as_float(d3[g]);
          // fp16 operands can overflow (|q| or |x - c| >= 65520): a non-finite dot gives the key -inf,
          // still a lower bound, so the certificate fails and the exact fallback answers the query
          if (kH && !(fabsf(dot) <= 3.0e38f)) dot = __builtin_huge_valf();
          eb[g * kRows + r] = (valid && g < nq) ? xn - 2.f * dot : kInf;
        }
        named_bar_sync(2, 128);
        const long long gbase = T.grow0 + (long long)rt * kRows;
        if (p.debug_skip & 1) continue;
#pragma unroll
        for (int j = 0; j < kOwn; ++j) {
          const int g = ew + 4 * j;
          if (g >= nq) break;
          // prune with the tighter of this list's 32nd and the query's global threshold
          float thr = fminf(__shfl_sync(0xffffffffu, ld[j], p.thr_rank), qt[j]);
          int base = 0;
#pragma unroll
          for (int m = 0; m < kRows / 32; ++m) {
            const float v = eb[g * kRows + m * 32 + lane] + qn[j];
            bool pass = v < thr;
            unsigned mask = __ballot_sync(0xffffffffu, pass);
            if (base + __popc(mask) > 32) {  // flush the staged batch first
              __syncwarp();
              const float bd = lane < base ? sd[lane] : kInf;
              const long long bk = lane < base ? sk[lane] : kNoKey;
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
              const float bd = lane < base ? sd[lane] : kInf;
              const long long bk = lane < base ? sk[lane] : kNoKey;
              warp_merge32(ld[j], lk[j], bd, bk, lane);
            }
            __syncwarp();
          }
        }
      }
      // the global pruning threshold: every tile end, fire-and-forget (the list itself waits for
      // its query to change)
      float myl31 = kInf;
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        const float l31 = __shfl_sync(0xffffffffu, ld[j], p.thr_rank);  // the bound the merge needs
        if (lane == j) myl31 = l31;
      }
      if (lane < kOwn && myl31 != kInf) {
        int myq = 0;
#pragma unroll
        for (int j = 0; j < kOwn; ++j)
          if (lane == j) myq = cq[j];
        if (myq >= 0) atomicMin(p.qthr + myq, f2ord(myl31));
      }
    }
  }

done:
#ifdef RD_STALL_PROF
  if (p.stall && (threadIdx.x & 31) == 0) {  // lane 0 of each role's first warp reports its waits
    const int w = threadIdx.x >> 5;
    unsigned long long* o = p.stall + (size_t)blockIdx.x * 12;
    if (w == 0) {
      o[0] = stall_acc[0];
      o[1] = stall_acc[1];
      o[2] = stall_acc[2];
      o[9] = clock64() - t_begin;
    } else if (w == 1) {
      o[3] = stall_acc[3];
      o[4] = stall_acc[4];
      o[5] = stall_acc[5];
      o[6] = stall_acc[6];
    } else if (w == 6) {
      o[7] = stall_acc[7];
      o[8] = stall_acc[8];
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
  if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * 4 + 3] = gtimer();
}

// q -> (q1, q2) bf16 rows: out[b][0][:] = bf16(q), out[b][1][:] = bf16(q - q1)
__global__ void qsplit_kernel(const float* __restrict__ Q, __nv_bfloat16* __restrict__ out, long long B, int d) {
  const long long total = B * d;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / d;
    const int t = (int)(i - b * d);
    const float q = Q[i];
    const __nv_bfloat16 h = __float2bfloat16_rn(q);
    out[(b * 2) * d + t] = h;
    out[(b * 2 + 1) * d + t] = __float2bfloat16_rn(q - __bfloat162float(h));
  }
}

}  // namespace

size_t scan_tc_smem_bytes(int d, int tc_g, bool presplit, bool stream, bool resid, bool half) {
  stream = stream && presplit && tc_g == 16;
  resid = resid && presplit;
  half = half && resid;
  size_t stages, sbytes;
  if (half) {
    stages = stream ? Ring<true, 16, true, true, true>::S
                    : tc_g == 16 ? Ring<true, 16, false, true, true>::S : Ring<true, 32, false, true, true>::S;
    sbytes = stream ? Ring<true, 16, true, true, true>::B : Ring<true, 16, false, true, true>::B;
  } else if (resid) {
    stages = stream ? Ring<true, 16, true, true>::S : tc_g == 16 ? Ring<true, 16, false, true>::S : Ring<true, 32, false, true>::S;
    sbytes = stream ? Ring<true, 16, true, true>::B : Ring<true, 16, false, true>::B;
  } else {
    stages = stream ? Ring<true, 16, true>::S
             : presplit ? (tc_g == 16 ? Ring<true, 16, false>::S : Ring<true, 32, false>::S)
                        : (tc_g == 16 ? Ring<false, 16, false>::S : Ring<false, 32, false>::S);
    sbytes = stream ? Ring<true, 16, true>::B : presplit ? Ring<true, 16, false>::B : Ring<false, 16, false>::B;
  }
  const size_t bslice = half ? (tc_g == 16 ? BGeom<16, true>::Slice : BGeom<32, true>::Slice)
                             : (tc_g == 16 ? TcGeom<16>::BSlice : TcGeom<32>::BSlice);
  const size_t xring = stages * sbytes;
  const size_t ring = xring + (stream ? 0 : (size_t)(d / 64) * bslice);
  return 1024 + ring +
         (2 * stages + 2 * kXBufs + 10) * sizeof(uint64_t) + 2 * sizeof(int) + 16 + 4 * 32 * 12 +
         (size_t)tc_g * kRows * sizeof(float) + 64;
}

cudaError_t launch_scan_tc(const CUtensorMap& map128, const CUtensorMap& map32, const CUtensorMap& qmap,
                           const TcScanParams& p, int grid, cudaStream_t s, bool presplit, int tc_g, bool stream,
                           bool resid, bool half) {
  if (p.d % 64 != 0 || (tc_g != 16 && tc_g != 32)) return cudaErrorInvalidValue;
  stream = stream && presplit && tc_g == 16;
  resid = resid && presplit;
  half = half && resid;
  const size_t smem = scan_tc_smem_bytes(p.d, tc_g, presplit, stream, resid, half);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (half) {
    if (tc_g == 16) {
      if (stream)
        return launch_k(ivf_scan_tc_kernel<true, 16, true, true, true>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
      return launch_k(ivf_scan_tc_kernel<true, 16, false, true, true>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
    }
    return launch_k(ivf_scan_tc_kernel<true, 32, false, true, true>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
  }
  if (resid) {
    if (tc_g == 16) {
      if (stream)
        return launch_k(ivf_scan_tc_kernel<true, 16, true, true, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
      return launch_k(ivf_scan_tc_kernel<true, 16, false, true, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
    }
    return launch_k(ivf_scan_tc_kernel<true, 32, false, true, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
  }
  if (tc_g == 16) {
    if (stream)
      return launch_k(ivf_scan_tc_kernel<true, 16, true, false, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
    if (presplit)
      return launch_k(ivf_scan_tc_kernel<true, 16, false, false, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
    return launch_k(ivf_scan_tc_kernel<false, 16, false, false, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
  }
  if (presplit)
    return launch_k(ivf_scan_tc_kernel<true, 32, false, false, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
  return launch_k(ivf_scan_tc_kernel<false, 32, false, false, false>, dim3(grid), dim3(kThreads), smem, s, map128, map32, qmap, p);
}

cudaError_t launch_qsplit(const float* Q, void* out, long long B, int d, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const long long total = B * d;
  qsplit_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 148 * 8), 256, 0, s>>>(
      Q, reinterpret_cast<__nv_bfloat16*>(out), B, d);
  return cudaGetLastError();
}

}  // namespace rd
