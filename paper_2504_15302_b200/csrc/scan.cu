// scan.cu — N4: the inverted-list scan (the hot loop), sm_100a.
//
// One persistent CTA per SM. Warp 8 is the TMA producer: it claims scan tiles
// from a global counter and streams each tile's rows through a 4-stage smem
// ring, one 2D TMA box of [32 fp32 dims x 256 rows] (32 KiB, SWIZZLE_128B) per
// stage. Warps 0-7 consume: warp w owns rows (w&3)*64 + lane + {0,32} of the
// row tile and the k-half (w>>2) (even / odd 32-dim slices), accumulating
// q.x for up to 16 queries in registers with FFMA (queries are broadcast from
// smem). The two k-halves are summed through smem, turned into
// d~ = ||x||^2 + ||q||^2 - 2 q.x, and each query's running top-32 (held
// across the tile in one warp's registers) absorbs survivors below its
// threshold with a warp bitonic merge. The tile's per-query top-32 goes to the
// partial buffer; merge.cu certifies and reranks them exactly.
#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr float kInf = __builtin_huge_valf();
constexpr long long kNoKey = 0x7fffffffffffffffll;

struct ScanSmem {
  unsigned char* xs;
  float* qs;
  float* red;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  int* tring;
  float* qn;
};

__device__ __forceinline__ ScanSmem carve(unsigned char* raw, int d) {
  ScanSmem s;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  s.xs = base;
  s.qs = reinterpret_cast<float*>(base + kScanStages * kScanStageBytes);
  s.red = s.qs + kScanG * d;
  s.full = reinterpret_cast<uint64_t*>(s.red + kScanG * kScanRows);
  s.empty = s.full + kScanStages;
  s.tfull = s.empty + kScanStages;
  s.tempty = s.tfull + 2;
  s.tring = reinterpret_cast<int*>(s.tempty + 2);
  s.qn = reinterpret_cast<float*>(s.tring + 2);
  return s;
}

// k-slices of one row tile for this warp's k-half; `it` is the global slice counter.
template <int GE>
__device__ __forceinline__ void rowtile_dots(const ScanSmem& sm, int d, int kh, int rb, int lane,
                                             uint32_t it, float (&acc)[2][kScanG]) {
  const int nks = d / kScanKSlice;
  const int r0 = rb * 64 + lane;
  const int sw = lane & 7;
#pragma unroll
  for (int g = 0; g < kScanG; ++g) acc[0][g] = acc[1][g] = 0.f;
  for (int ks = kh; ks < nks; ks += 2) {
    const uint32_t u = it + ks;
    const int stage = u & (kScanStages - 1);
    mbar_wait(&sm.full[stage], (u / kScanStages) & 1);
    const unsigned char* xst = sm.xs + stage * kScanStageBytes;
    const float* qk = sm.qs + ks * kScanKSlice;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int off = (j ^ sw) << 4;
      const float4 x0 = *reinterpret_cast<const float4*>(xst + r0 * 128 + off);
      const float4 x1 = *reinterpret_cast<const float4*>(xst + (r0 + 32) * 128 + off);
#pragma unroll
      for (int g = 0; g < GE; ++g) {
        const float4 q = *reinterpret_cast<const float4*>(qk + g * d + 4 * j);
        acc[0][g] = fmaf(x0.x, q.x, acc[0][g]);
        acc[1][g] = fmaf(x1.x, q.x, acc[1][g]);
        acc[0][g] = fmaf(x0.y, q.y, acc[0][g]);
        acc[1][g] = fmaf(x1.y, q.y, acc[1][g]);
        acc[0][g] = fmaf(x0.z, q.z, acc[0][g]);
        acc[1][g] = fmaf(x1.z, q.z, acc[1][g]);
        acc[0][g] = fmaf(x0.w, q.w, acc[0][g]);
        acc[1][g] = fmaf(x1.w, q.w, acc[1][g]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[stage]);
  }
}

__global__ void __launch_bounds__(kScanThreads, 1)
    ivf_scan_kernel(const __grid_constant__ CUtensorMap map256,
                    const __grid_constant__ CUtensorMap map32, const ScanParams p) {
  RD_PDL_PROLOGUE();
  extern __shared__ unsigned char smem_raw[];
  const ScanSmem sm = carve(smem_raw, p.d);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = p.d;
  const int nks = d / kScanKSlice;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kScanStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 4);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.tfull[s], 1);
      mbar_init(&sm.tempty[s], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = *p.ntiles;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&map256);
      prefetch_tmap(&map32);
      uint32_t it = 0;
      for (uint32_t ti = 0;; ++ti) {
        const int t = atomicAdd(p.tile_counter, 1);
        const int slot = ti & 1;
        mbar_wait(&sm.tempty[slot], ((ti >> 1) & 1) ^ 1);
        sm.tring[slot] = t < ntiles ? t : -1;
        mbar_arrive(&sm.tfull[slot]);
        if (t >= ntiles) break;
        const ScanTile T = p.tiles[t];
        for (int rt = 0; rt * kScanRows < T.nrows; ++rt) {
          const int rows = min(kScanRows, T.nrows - rt * kScanRows);
          const int nb = (rows + 31) >> 5;
          const int row = (int)(T.src_row + rt * kScanRows);
          for (int ks = 0; ks < nks; ++ks, ++it) {
            const int stage = it & (kScanStages - 1);
            mbar_wait(&sm.empty[stage], ((it / kScanStages) & 1) ^ 1);
            unsigned char* dst = sm.xs + stage * kScanStageBytes;
            if (nb == 8) {
              mbar_arrive_expect_tx(&sm.full[stage], kScanStageBytes);
              tma_load_2d(dst, &map256, ks * kScanKSlice, row, &sm.full[stage]);
            } else {
              mbar_arrive_expect_tx(&sm.full[stage], nb * 4096);
              for (int b = 0; b < nb; ++b)
                tma_load_2d(dst + b * 4096, &map32, ks * kScanKSlice, row + b * 32, &sm.full[stage]);
            }
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int tid = threadIdx.x;  // 0..255
  const int kh = warp >> 2, rb = warp & 3;
  uint32_t it = 0;
  for (uint32_t ti = 0;; ++ti) {
    const int slot = ti & 1;
    mbar_wait(&sm.tfull[slot], (ti >> 1) & 1);
    const int t = sm.tring[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.tempty[slot]);
    if (t < 0) break;
    const ScanTile T = p.tiles[t];
    const int nq = T.nq;

    named_bar_sync(1, 256);  // previous tile finished with qs / red / qn
    {
      const int d4 = d >> 2;
      float4* qs4 = reinterpret_cast<float4*>(sm.qs);
      const float4* Q4 = reinterpret_cast<const float4*>(p.queries);
      for (int i = tid; i < kScanG * d4; i += 256) {
        const int g = i / d4, c = i - g * d4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g < nq) v = __ldg(Q4 + (size_t)__ldg(p.list_q + T.qoff + g) * d4 + c);
        qs4[i] = v;
      }
      if (tid < kScanG) sm.qn[tid] = tid < nq ? __ldg(p.qnorm + __ldg(p.list_q + T.qoff + tid)) : 0.f;
    }
    named_bar_sync(1, 256);

    // running top-32 of the two queries this warp owns (g = warp, warp + 8), and their
    // global pruning thresholds (min over completed tiles' 32nd best)
    float ld0 = kInf, ld1 = kInf;
    long long lk0 = kNoKey, lk1 = kNoKey;
    const float qt0 = warp < nq ? ord2f(*(volatile int*)(p.qthr + __ldg(p.list_q + T.qoff + warp))) : kInf;
    const float qt1 = warp + 8 < nq ? ord2f(*(volatile int*)(p.qthr + __ldg(p.list_q + T.qoff + warp + 8))) : kInf;

    for (int rt = 0; rt * kScanRows < T.nrows; ++rt, it += nks) {
      float acc[2][kScanG];
      if (nq <= 4)
        rowtile_dots<4>(sm, d, kh, rb, lane, it, acc);
      else if (nq <= 8)
        rowtile_dots<8>(sm, d, kh, rb, lane, it, acc);
      else
        rowtile_dots<16>(sm, d, kh, rb, lane, it, acc);

      const int rows_valid = min(kScanRows, T.nrows - rt * kScanRows);
      const int r0 = rb * 64 + lane;
      named_bar_sync(1, 256);  // A: previous selection finished reading red
      if (kh == 1) {
#pragma unroll
        for (int g = 0; g < kScanG; ++g)
          if (g < nq) {
            sm.red[g * kScanRows + r0] = acc[0][g];
            sm.red[g * kScanRows + r0 + 32] = acc[1][g];
          }
      }
      named_bar_sync(1, 256);  // B
      if (kh == 0) {
        const long long gbase = T.grow0 + (long long)rt * kScanRows;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = r0 + 32 * i;
          const bool valid = r < rows_valid;
          const float xn = valid ? __ldg(p.xnorm + gbase + r) : 0.f;
#pragma unroll
          for (int g = 0; g < kScanG; ++g)
            if (g < nq) {
              const float dot = acc[i][g] + sm.red[g * kScanRows + r];
              sm.red[g * kScanRows + r] = valid ? (xn + sm.qn[g]) - 2.f * dot : kInf;
            }
        }
      }
      named_bar_sync(1, 256);  // C
      // selection: warp owns queries warp and warp+8
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int g = warp + 8 * h;
        if (g >= nq) break;
        float& ld = h ? ld1 : ld0;
        long long& lk = h ? lk1 : lk0;
        const float qt = h ? qt1 : qt0;
        float thr = fminf(__shfl_sync(0xffffffffu, ld, p.thr_rank), qt);
        const long long gbase = T.grow0 + (long long)rt * kScanRows;
#pragma unroll 1
        for (int m = 0; m < kScanRows / 32; ++m) {
          const float v = sm.red[g * kScanRows + m * 32 + lane];
          const bool pass = v < thr;
          if (__any_sync(0xffffffffu, pass)) {
            warp_merge32(ld, lk, pass ? v : kInf, pass ? gbase + m * 32 + lane : kNoKey, lane);
            thr = fminf(__shfl_sync(0xffffffffu, ld, p.thr_rank), qt);
          }
        }
      }
    }

    // emit this tile's per-query top-32
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = warp + 8 * h;
      if (g >= nq) break;
      const int qid = __ldg(p.list_q + T.qoff + g);
      const float ld = h ? ld1 : ld0;
      const long long lk = h ? lk1 : lk0;
      if (__shfl_sync(0xffffffffu, ld, 0) == kInf) continue;  // nothing survived: no partial
      const float l31 = __shfl_sync(0xffffffffu, ld, p.thr_rank);
      int pslot = 0;
      if (lane == 0) {
        pslot = atomicAdd(p.part_count + qid, 1);
        if (l31 != kInf) atomicMin(p.qthr + qid, f2ord(l31));
      }
      pslot = __shfl_sync(0xffffffffu, pslot, 0);
      if (pslot < p.part_cap) {
        const size_t o = ((size_t)qid * p.part_cap + pslot) * kTopK + lane;
        p.part_dist[o] = ld;
        p.part_row[o] = lk == kNoKey ? -1 : (int)lk;
      }
    }
  }
}

}  // namespace

size_t scan_smem_bytes(int d) {
  return 1024 /*alignment slack*/ + (size_t)kScanStages * kScanStageBytes +
         (size_t)kScanG * d * sizeof(float) + (size_t)kScanG * kScanRows * sizeof(float) +
         (2 * kScanStages + 4) * sizeof(uint64_t) + 2 * sizeof(int) + kScanG * sizeof(float) + 64;
}

cudaError_t launch_scan(const CUtensorMap& map256, const CUtensorMap& map32, const ScanParams& p,
                        int grid, cudaStream_t s) {
  const size_t smem = scan_smem_bytes(p.d);
  return launch_k(ivf_scan_kernel, dim3(grid), dim3(kScanThreads), smem, s, map256, map32, p);
}

}  // namespace rd
