// wide.cu — the search beyond the fast path's limits (sm_100a), so the engine takes every argument
// the reference's Request::top_k (core/include/ragsim/domain.hpp:84-90, validated at domain.cpp:127)
// and the CPU oracle take:
//
//   nprobe + 32 > 512 (the certified selection's candidate buffer): the probe set straight from the
//     canonical exact distance to every centroid, a stable segmented radix sort by (distance, list
//     id) — the oracle's order — and the first nprobe of each query;
//   k > kMaxK (24, the certified rerank's margin inside 32-wide candidate lists): an exact
//     query-major pass over the probed lists — per query, split over S CTAs, each warp keeps the
//     32R best rows by (canonical distance, id) in R cascaded 32-lists (R = ceil(k / 32)); rows are
//     filtered first by an fp32 distance against the running 32R-th exact distance (the fp32 value
//     is within l2_f32_rel_bound of the exact one), so only contenders pay the fp64 canonical sum;
//     the S x 32R survivors of a query are merged by (distance, id) on the device.
//
// Both are exact by construction (no certification). The large-k pass reads each probed list once
// per query (no reuse across the batch), so it suits RAG-sized batches; k <= 24 keeps the
// list-major tensor-core scan.
#include <cub/device/device_segmented_radix_sort.cuh>

#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace rd {

namespace {

constexpr float kInf = __builtin_huge_valf();
constexpr long long kNoKey = 0x7fffffffffffffffll;

// ---------------------------------------------------------------- all-centroid exact selection
// One CTA per query: canonical exact distance to every centroid (8 lanes per centroid), as the
// sort's (key, value) pairs; distances are >= 0, so their bit patterns order like the values.
__global__ void __launch_bounds__(256) centroid_exact_kernel(const float* __restrict__ Q, const float* __restrict__ C,
                                                             int nlist, int d, unsigned* __restrict__ keys,
                                                             int* __restrict__ vals) {
  extern __shared__ __align__(16) float qs[];
  const int b = blockIdx.x, tid = threadIdx.x;
  for (int t = tid; t < d; t += 256) qs[t] = Q[(size_t)b * d + t];
  __syncthreads();
  const int grp = tid >> 3, j8 = tid & 7;
  for (int c0 = 0; c0 < nlist; c0 += 32) {  // uniform trip count: the groups' shuffles stay converged
    const int c = c0 + grp;
    const float e = exact_l2_group8_impl<false>(qs, C + (size_t)min(c, nlist - 1) * d, c < nlist ? d : 0, j8);
    if (j8 == 0 && c < nlist) {
      keys[(size_t)b * nlist + c] = __float_as_uint(e);
      vals[(size_t)b * nlist + c] = c;
    }
  }
}

__global__ void segment_offsets_kernel(int* __restrict__ off, int nseg, int len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= nseg) off[i] = i * len;
}

// the first np sorted lists of each query -> probes (the rest -1), and the plan's bitmap bits
__global__ void take_probes_kernel(const int* __restrict__ sorted, int nlist, int B, int nprobe, int np, long long b0,
                                   int* __restrict__ probes, unsigned* __restrict__ bitmap, int W) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)B * nprobe) return;
  const int bl = (int)(i / nprobe), j = (int)(i - (long long)bl * nprobe);
  const long long b = b0 + bl;
  const int l = j < np ? sorted[(size_t)bl * nlist + j] : -1;
  probes[(size_t)b * nprobe + j] = l;
  if (bitmap && l >= 0) atomicOr(bitmap + (size_t)l * W + (b >> 5), 1u << (b & 31));
}

// ---------------------------------------------------------------- large-k exact pass
// fp32 squared distance of a row for the prefilter, 8 lanes per row: lane j sums the 8-element
// chunks j, j + 8, ... (16-byte loads, all of a lane's chunks in flight), then the 3-level shuffle
// tree. Each lane still sums d / 8 terms, so |result - exact| <= l2_f32_rel_bound(d) * exact, as
// for l2_group8_f32. q in shared memory; d % 8 == 0.
__device__ __forceinline__ float l2_prefilter(const float* q, const RowRef& x, int d, int j) {
  float s = 0.f;
  constexpr int kU = 4;  // chunks in flight per lane
  for (int c0 = j * 8; c0 < d; c0 += 64 * kU) {
    float xv[kU][8];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = c0 + u * 64;
      if (t < d) {
        if (x.f) {
          const float4 a = *reinterpret_cast<const float4*>(x.f + t), b = *reinterpret_cast<const float4*>(x.f + t + 4);
          xv[u][0] = a.x, xv[u][1] = a.y, xv[u][2] = a.z, xv[u][3] = a.w;
          xv[u][4] = b.x, xv[u][5] = b.y, xv[u][6] = b.z, xv[u][7] = b.w;
        } else {
          const uint4 h1 = *reinterpret_cast<const uint4*>(x.x12 + t), h2 = *reinterpret_cast<const uint4*>(x.x12 + d + t),
                      h3 = *reinterpret_cast<const uint4*>(x.x3 + t);
          const __nv_bfloat16* a1 = reinterpret_cast<const __nv_bfloat16*>(&h1);
          const __nv_bfloat16* a2 = reinterpret_cast<const __nv_bfloat16*>(&h2);
          const __nv_bfloat16* a3 = reinterpret_cast<const __nv_bfloat16*>(&h3);
#pragma unroll
          for (int e = 0; e < 8; ++e)
            xv[u][e] = __fadd_rn(__fadd_rn(__bfloat162float(a1[e]), __bfloat162float(a2[e])), __bfloat162float(a3[e]));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = c0 + u * 64;
      if (t < d) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float df = q[t + e] - xv[u][e];
          s = fmaf(df, df, s);
        }
      }
    }
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  return s;
}

// L (R ascending 32-lists, L[0] <= L[1] <= ..., one sorted 32R list across lanes and registers)
// absorbs a batch of 32 candidates (any order, one per lane).
template <int R>
__device__ __forceinline__ void absorb32(float (&ld)[R], long long (&lk)[R], float bd, long long bk, int lane) {
  warp_sort32(bd, bk, lane, /*asc=*/false);  // descending: pairs with L[r] ascending
#pragma unroll
  for (int r = 0; r < R; ++r) {
    // lane-wise min / max of an ascending and a descending list: two bitonic halves, the 32
    // smallest of L[r] u batch and the 32 largest
    const bool take = pair_less(bd, bk, ld[r], lk[r]);
    const float lo_d = take ? bd : ld[r], hi_d = take ? ld[r] : bd;
    const long long lo_k = take ? bk : lk[r], hi_k = take ? lk[r] : bk;
    ld[r] = lo_d, lk[r] = lo_k;
    bd = hi_d, bk = hi_k;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) bitonic_step(ld[r], lk[r], lane, j, true);
    if (r + 1 < R) {
#pragma unroll
      for (int j = 16; j > 0; j >>= 1) bitonic_step(bd, bk, lane, j, false);  // descending for the next level
    }
  }
}

// grid (B, S): the 8 S warps of query b stride over the rows of every probed list, 4 rows (8 lanes
// per row) at a time, each keeping its 32R best; a row is dropped without its exact distance when its
// fp32 distance places it beyond the query's running threshold — the min over warps of their 32R-th
// exact distance (qthr[b], atomicMin: any warp's 32R-th bounds the query's from above). The CTA's
// 32R best go to out[s][b][32R] (the [G][B][k] layout of the shard merge).
template <int R>
__global__ void __launch_bounds__(256) wide_exact_kernel(const WideParams p) {
  RD_PDL_PROLOGUE();
  extern __shared__ __align__(16) float qs[];  // q[d]
  __shared__ float wd[8][32 * R];
  __shared__ long long wk[8][32 * R];
  const int b = blockIdx.x, s = blockIdx.y, S = gridDim.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 3, j8 = lane & 7;
  const int d = p.d;
  for (int t = tid; t < d; t += 256) qs[t] = p.queries[(size_t)b * d + t];
  __syncthreads();
  float ld[R];
  long long lk[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ld[r] = kInf, lk[r] = kNoKey;
  const float rel = l2_f32_rel_bound(d);
  float bd = kInf;  // batch being gathered: lane (pass * 4 + group) holds one row
  long long bk = kNoKey;
  int filled = 0;
  const int gw = s * 8 + warp;  // this warp among the query's 8 S
  int* qthr = p.qthr + b;
  float thr = kInf;  // min(own 32R-th, the query's threshold), refreshed after every batch
  for (int pi = 0; pi < p.nprobe; ++pi) {
    const int l = p.probes[(size_t)b * p.nprobe + pi];
    if (l < 0) continue;
    const long long r0 = p.list_off[l], r1 = p.list_off[l + 1];
    const float* base = p.list_base[l];  // nullptr: rows in the split3 store from res_row0
    const long long s0 = base ? 0 : p.res_row0[l];
    for (long long c = r0 + 4LL * gw; c < r1; c += 32LL * S) {  // uniform per warp
      const long long row = c + g;
      const bool ok = row < r1;
      const RowRef x = !ok ? row_f32(qs)
                           : base ? row_f32(base + (size_t)(row - r0) * d)
                                  : row_split3(p.x12, p.x3, s0 + (row - r0), d);
      const float e32 = l2_prefilter(qs, x, d, j8);
      // exact only where the fp32 distance does not already place the row beyond the 32R-th best
      const bool need = ok && !(e32 > thr * (1.f + rel) * (1.f + rel));
      const float e = exact_l2_group8_row(qs, x, d, j8, need ? d : 0);
      const long long id = need ? p.ids[row] : kNoKey;
      // gather into the batch: pass `filled` fills lanes filled * 4 .. filled * 4 + 3
      const float ev = __shfl_sync(0xffffffffu, e, (lane & 3) * 8);
      const long long iv = __shfl_sync(0xffffffffu, id, (lane & 3) * 8);
      const bool nv = __shfl_sync(0xffffffffu, need, (lane & 3) * 8);
      if ((lane >> 2) == filled) {
        bd = nv ? ev : kInf;
        bk = nv ? iv : kNoKey;
      }
      if (++filled == 8) {
        const float t2 = __shfl_sync(0xffffffffu, ld[R - 1], 31);
        const long long tk = __shfl_sync(0xffffffffu, lk[R - 1], 31);
        if (__any_sync(0xffffffffu, pair_less(bd, bk, t2, tk))) {
          absorb32<R>(ld, lk, bd, bk, lane);
          const float mine = __shfl_sync(0xffffffffu, ld[R - 1], 31);
          if (lane == 0 && mine < kInf) atomicMin(qthr, f2ord(mine));
        }
        thr = fminf(__shfl_sync(0xffffffffu, ld[R - 1], 31), ord2f(*(volatile int*)qthr));
        bd = kInf, bk = kNoKey, filled = 0;
      }
    }
  }
  if (__any_sync(0xffffffffu, bk != kNoKey)) absorb32<R>(ld, lk, bd, bk, lane);
#pragma unroll
  for (int r = 0; r < R; ++r) wd[warp][r * 32 + lane] = ld[r], wk[warp][r * 32 + lane] = lk[r];
  __syncthreads();
  if (warp == 0) {  // the CTA's best 32R: warp 0 absorbs the other warps' lists 32 at a time
    for (int w = 1; w < 8; ++w)
      for (int r = 0; r < R; ++r) {
        const float v = wd[w][r * 32 + lane];
        const long long kk = wk[w][r * 32 + lane];
        if (!__any_sync(0xffffffffu, kk != kNoKey)) break;  // the rest of this warp's list is empty
        absorb32<R>(ld, lk, v, kk, lane);
      }
    const size_t o = ((size_t)s * gridDim.x + b) * 32 * R;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      p.out_d[o + r * 32 + lane] = ld[r];
      p.out_id[o + r * 32 + lane] = lk[r] == kNoKey ? -1 : lk[r];
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ host side
size_t select_all_scratch_bytes(long long Bsub, int nlist) {
  size_t temp = 0;
  const long long n = Bsub * nlist;
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp, (const unsigned*)nullptr, (unsigned*)nullptr,
                                           (const int*)nullptr, (int*)nullptr, (int)n, (int)Bsub, (const int*)nullptr,
                                           (const int*)nullptr, 0, 32);
  return temp + (size_t)n * 16 + (size_t)(Bsub + 1) * 4 + 1024;
}

long long select_all_batch(int nlist) {  // queries per sort pass: ~64M (key, value) pairs
  return std::max<long long>(1, std::min<long long>(65536, (64LL << 20) / std::max(1, nlist)));
}

cudaError_t launch_select_all(const float* Q, const float* C, long long B, int nlist, int d, int nprobe, int* probes,
                              unsigned* bitmap, int W, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const long long Bsub = std::min(B, select_all_batch(nlist));
  const long long n = Bsub * nlist;
  char* base = reinterpret_cast<char*>(scratch);
  auto carve = [&](size_t bytes) {
    char* p = base;
    base += (bytes + 255) / 256 * 256;
    return p;
  };
  unsigned* kin = reinterpret_cast<unsigned*>(carve((size_t)n * 4));
  unsigned* kout = reinterpret_cast<unsigned*>(carve((size_t)n * 4));
  int* vin = reinterpret_cast<int*>(carve((size_t)n * 4));
  int* vout = reinterpret_cast<int*>(carve((size_t)n * 4));
  int* off = reinterpret_cast<int*>(carve((size_t)(Bsub + 1) * 4));
  size_t temp = 0;
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp, kin, kout, vin, vout, (int)n, (int)Bsub, off,
                                                           off + 1, 0, 32, s);
  if (e != cudaSuccess) return e;
  if ((size_t)(base - reinterpret_cast<char*>(scratch)) + temp > scratch_bytes) return cudaErrorInvalidValue;
  void* tmp = base;
  const int np = std::min(nprobe, nlist);
  for (long long b0 = 0; b0 < B; b0 += Bsub) {
    const long long nb = std::min(Bsub, B - b0);
    segment_offsets_kernel<<<(unsigned)((nb + 256) / 256), 256, 0, s>>>(off, (int)nb, nlist);
    e = launch_k(centroid_exact_kernel, dim3((unsigned)nb), dim3(256), sizeof(float) * (size_t)d, s,
                 Q + (size_t)b0 * d, C, nlist, d, kin, vin);
    if (e != cudaSuccess) return e;
    size_t t2 = temp;
    e = cub::DeviceSegmentedRadixSort::SortPairs(tmp, t2, kin, kout, vin, vout, (int)(nb * nlist), (int)nb, off,
                                                 off + 1, 0, 32, s);
    if (e != cudaSuccess) return e;
    const long long tot = nb * nprobe;
    take_probes_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(vout, nlist, (int)nb, nprobe, np, b0, probes,
                                                                       bitmap, W);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int wide_lists(int k) {  // R: 32-lists per warp for top-k
  const int r = (k + 31) / 32;
  return r <= 1 ? 1 : r <= 2 ? 2 : r <= 4 ? 4 : 8;
}

int wide_splits(long long B, int nprobe, int k, int num_sms) {  // S: CTAs per query
  (void)nprobe;
  const long long want = (2LL * num_sms + B - 1) / B;
  const long long cap = shard_merge_max_candidates() / (32LL * wide_lists(k));  // the final merge's buffer
  return (int)std::max<long long>(1, std::min<long long>(want, cap));
}

cudaError_t launch_wide(const WideParams& p, int S, cudaStream_t s) {
  if (p.B == 0) return cudaSuccess;
  const dim3 grid((unsigned)p.B, (unsigned)S);
  const size_t smem = sizeof(float) * (size_t)p.d;
  switch (wide_lists(p.k)) {
    case 1: return launch_k(wide_exact_kernel<1>, grid, dim3(256), smem, s, p);
    case 2: return launch_k(wide_exact_kernel<2>, grid, dim3(256), smem, s, p);
    case 4: return launch_k(wide_exact_kernel<4>, grid, dim3(256), smem, s, p);
    default: return launch_k(wide_exact_kernel<8>, grid, dim3(256), smem, s, p);
  }
}

}  // namespace rd
