// ivf_kernels.cuh — launch interface of the IVF-Flat search kernels (sm_100a).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

namespace rd {

// Kernel launch with programmatic stream serialization (PDL): the kernel may be scheduled while
// its predecessor in the stream drains; the kernel's RD_PDL_PROLOGUE waits for the predecessor's
// results. RD_PDL=0 in the environment launches them plainly (A/B).
bool pdl_enabled();
cudaError_t ensure_smem(const void* kern, size_t smem);  // per (device, kernel) dynamic smem limit

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  const cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Scan geometry (see DESIGN.md §Kernels / N4):
constexpr int kScanRows = 256;      // rows of one row tile (one TMA box)
constexpr int kScanKSlice = 32;     // fp32 dims per stage: 128 B rows, SWIZZLE_128B
constexpr int kScanStages = 4;      // smem ring depth (32 KiB per stage)
constexpr int kScanG = 16;          // max queries per tile
constexpr int kScanThreads = 288;   // 8 consumer warps + 1 TMA producer warp
constexpr int kScanStageBytes = kScanRows * 128;
constexpr int kCoarseExtra = 32;    // approximate coarse candidates beyond nprobe
// tensor-core scan (N5)
constexpr int kTcRows = 128;        // UMMA M: rows per accumulator tile
constexpr int kTcGMax = 32;         // widest tensor-core tile (queries); 16- and 32-wide variants exist
constexpr int kTcMinQ = 1;          // lists probed by >= this many queries use the tensor cores
constexpr int kPartsPerTile = 1;    // partial lists one scan tile emits per query

// One unit of scan work: rows [row0, row0+nrows) of one list against <= 16 queries.
struct __align__(16) ScanTile {
  long long src_row;  // TMA row coordinate of the first row in the source arena
  long long grow0;    // global (list-order) row index of the first row
  int list;
  int nrows;
  int qoff;           // offset into list_q (query ids probing `list`)
  int nq;
};

struct ScanParams {
  const ScanTile* tiles;
  const int* ntiles;       // device scalar
  int* tile_counter;       // device scalar, zeroed before launch
  const float* queries;    // B x d
  const float* qnorm;      // B
  const int* list_q;       // query ids grouped by list
  const float* xnorm;      // n (global row order)
  float* part_dist;        // B x cap x 32
  int* part_row;           // B x cap x 32
  int* part_count;         // B
  int part_cap;
  int d;
  int* qthr;               // B: per-query pruning threshold (f2ord), min over completed tiles' 32nd
  // 0-based rank whose distance bounds what the merge needs (min(31, k + 8): it reranks k + 8 and
  // certifies against the next): rows beyond a tile's (thr_rank+1)-th best can be dropped
  int thr_rank = 31;
};

struct TcScanParams {
  const ScanTile* tiles;
  const int* ntiles;
  int* tile_counter;
  const void* qsplit;      // B x 2 x d bf16: (q1, q2) per query, q1 = bf16(q), q2 = bf16(q - q1)
  const float* qnorm;
  const int* list_q;
  const float* xnorm;
  float* part_dist;
  int* part_row;
  int* part_count;
  int part_cap;
  int d;
  int* qthr;               // B: per-query pruning threshold (f2ord), min over completed tiles' 32nd
  int debug_skip;          // profiling only (RD_DEBUG_SKIP): 1 = no epilogue selection, 2 = no conversion, 4 = no MMA
  unsigned long long* stall = nullptr;  // profiling only (RD_DEBUG_STALL): per CTA x 12 barrier-wait cycles
  unsigned long long* dbg = nullptr;  // profiling only (RD_DEBUG_TS): per CTA [entry, ready, first tile, end] globaltimer
  int thr_rank = 31;       // as ScanParams::thr_rank
  // residual store only (scan_tc.cu resid_pair_term): the coarse distances and their bound, ||c||^2
  // and max ||x - c|| per list, the scan's error factors (gamma_resid_r, gamma_resid_q)
  const float* Dc = nullptr;
  int nlist = 0;
  const float* cnorm = nullptr;
  const float* rmax = nullptr;
  float gamma_coarse = 0.f, cmax = 0.f, gamma_res = 0.f, gamma_q = 0.f, abs_res = 0.f;
};

size_t scan_smem_bytes(int d);
size_t scan_tc_smem_bytes(int d, int tc_g, bool presplit, bool stream = false, bool resid = false, bool half = false);
// 32-query tiles over the x1 | x2 plane on CTA pairs (scan_pair.cu, cta_group::2): ring depth for
// this d (0: unsupported), and the launch (grid = the SMs rounded down to pairs)
int scan_pair_stages(int d, bool resid = false);
cudaError_t launch_scan_pair(const CUtensorMap& map128, const CUtensorMap& map32, const CUtensorMap& qmap,
                             const TcScanParams& p, int num_sms, cudaStream_t s, bool resid = false);
// qmap: 2D bf16 map over the qsplit buffer as [2B rows x d], box {64, 1} (gather4 source)
// presplit: map128 / map32 are 3D bf16 maps over the pre-split [rows][2][d] arena, box {64, 1, 128|32}
// tc_g: queries per tile, 16 or 32 (the planner grouped the tiles with the same width)
cudaError_t launch_scan_tc(const CUtensorMap& map128, const CUtensorMap& map32, const CUtensorMap& qmap,
                           const TcScanParams& p, int grid, cudaStream_t s, bool presplit, int tc_g,
                           bool stream = false, bool resid = false, bool half = false);

// Residual store (resid.cu). r1 = bf16(x - c_list) per resident row ([rows][d], the scan's A
// operand), rnorm[global row] = ||x - c_list||^2 + 2 c_list . r1 (fp64 sums, RN), rmax[list] =
// max ||x - c_list|| rounded up. One CTA per list.
// half: r1 as fp16 (the fp16 residual scan); *ovf counts components beyond fp16's range
cudaError_t launch_resid_build(const float* arena, const long long* res_row0, const long long* list_off,
                               const float* centroids, int nlist, int d, void* r1, float* rnorm, float* rmax,
                               cudaStream_t s, bool half = false, unsigned* ovf = nullptr);

cudaError_t launch_qsplit(const float* Q, void* out, long long B, int d, cudaStream_t s);
cudaError_t launch_scan(const CUtensorMap& map256, const CUtensorMap& map32, const ScanParams& p,
                        int grid, cudaStream_t s);

// Coarse quantization: Dc[b][j] = ||c_j||^2 - 2 q_b . c_j (the query norm is
// constant per query and added where an absolute distance is needed).
cudaError_t launch_coarse(const float* Q, const float* C, const float* cnorm, float* Dc, int B,
                          int nlist, int d, cudaStream_t s);
// Query preparation: ||q||^2 and (when qsplit != nullptr) the bf16 (hi, lo) split rows of a query
// batch in one pass; zero2 (2 words) and zeroB (B words) are zeroed on the way when non-null.
struct QprepArgs {
  const float* Q;
  long long B;
  int d;
  float* qnorm;
  void* qsplit;
  unsigned* zero2;
  int* zeroB;
  void* qhalf = nullptr;  // fp16 residual scan: q as fp16 rows [B][d]
};
cudaError_t launch_qprep(const QprepArgs& a, cudaStream_t s);
// small batches: FFMA GEMV over the centroids (memory-bound; see coarse_small for the cut-over), with
// the query preparation `qa` fused into one trailing CTA
bool coarse_small(int B);
cudaError_t launch_coarse_small(const float* Q, const float* C, const float* cnorm, float* Dc, int B, int nlist,
                                int d, const QprepArgs& qa, cudaStream_t s);
// tensor-core variant (d % 64 == 0): qmap / cmap are 3D bf16 maps over the (hi, lo) splits,
// dims {d, 2, rows}, box {64, 1, 128}, 128 B swizzle
size_t coarse_tc_smem_bytes();
cudaError_t launch_coarse_tc(const CUtensorMap& qmap, const CUtensorMap& cmap, const float* cnorm, float* Dc, int B,
                             int nlist, int d, cudaStream_t s);

// Error bounds of the approximate dot products the certification relies on (DESIGN.md §2
// "Certification"): |computed q.x - exact q.x| <= gamma * ||q|| * max||x||, by path. u = 2^-24.
//  - FFMA scan: two d/2-long fp32 FFMA chains, gamma = (d/2 + 8) u, kept with a factor 2 of slack;
//  - FFMA coarse GEMM / GEMV: gamma = (d + 4) u, factor 2 of slack;
//  - bf16x3 on tcgen05 kind::f16 (scan and coarse): the dropped x2.q2 term and the two split
//    residuals, |x - x1 - x2| <= 2^-17 |x| (same for q), total <= 2^-15 (1 + 2^-7) sum|x_t q_t| ~ 516 u,
//    plus the accumulator: per K = 16 MMA step each of the 16 products not of the largest magnitude
//    is truncated to 2^-25 of the step's largest term (accumulator included) and the result is rounded
//    toward zero (measured on B200: tests/test_gpu_tcgen05.py), <= 10 u of the step's magnitude, taken
//    as 11 u per step over d / 16 steps on each of the three accumulators (1.02 x the x1.q1 mass),
//    plus the two fp32 adds that combine them: gamma = (524 + 0.7 d) u.
constexpr float kUnit = 5.9604645e-8f;
inline float gamma_ffma_scan(int d) { return 2.f * (d / 2 + 8) * kUnit; }
inline float gamma_ffma_coarse(int d) { return 2.f * (d + 4) * kUnit; }
inline float gamma_bf16x3(int d) { return (524.f + 0.7f * d) * kUnit; }
// residual scan (scan_tc.cu resid_pair_term): r1 = bf16(x - c) is within 2^-9 |x - c| (against
// ||q - c||); D = r1 . (q1 + q2) carries q's split (2^-17) and the measured fp32 accumulation term of
// the bf16x3 model (against ||q|| max ||r1||, r1 <= (1 + 2^-9) r)
inline float gamma_resid_r(int) { return 2.f * 16384.f * kUnit * (1.f + 1.f / 128.f); }
inline float gamma_resid_q(int d) { return (128.f + 16.f + 0.7f * d) * kUnit * (1.f + 1.f / 256.f); }
// fp16 residual scan (r1 = fp16(x - c), B = fp16(q), no split): 2^-11 for each rounding (r1 against
// ||q - c||; q1 against ||q|| max ||r1||, with the accumulation term); subnormals: abs_resid16
inline float gamma_resid16_r(int) { return 8192.f * kUnit * (1.f + 1.f / 512.f); }
inline float gamma_resid16_q(int d) { return (8192.f + 16.f + 0.7f * d) * kUnit * (1.f + 1.f / 256.f); }
// fp16 subnormals (|v| < 2^-14) round with an absolute error <= 2^-25 per element: with Cauchy-Schwarz
// <= 2^-25 sqrt(d) (||q - c|| + max ||r1||) on the dot, doubled in the distance
inline float abs_resid16(int d) { return 2.f * 2.9802322e-8f * sqrtf((float)d) * 1.01f; }

#ifdef __CUDACC__
// Residual store: ||q - c_l||^2 - eps for query b and list l, from ||q||^2 (qq) and the coarse
// distance Dc = ||c||^2 - 2 q.c (error <= ec, the selection's bound). eps bounds |key - exact| with
// key = that + rnorm_row - 2 D, D = r1 . (q1 + q2) in fp32 (resid.cu): the coarse error, the bf16
// rounding of r (2^-9 |r|, against ||q - c||), D's split and accumulation error (against ||q||) and
// the fp32 roundings of the terms; every bound inflated by 1 %.
__device__ __forceinline__ float resid_pair_term(const TcScanParams& p, float qq, int b, int l) {
  const float Q = qq + __ldg(p.Dc + (size_t)b * p.nlist + l);
  const float nq = sqrtf(qq), rm = __ldg(p.rmax + l), cn = sqrtf(__ldg(p.cnorm + l)) * 1.0001f;
  const float ec = 2.f * p.gamma_coarse * nq * p.cmax + 16.f * kUnit * (qq + p.cmax * p.cmax);
  const float na = sqrtf(fmaxf(Q + ec, 0.f)) * 1.0001f;
  const float eps = 1.01f * (ec + 2.f * p.gamma_res * na * rm + 2.f * p.gamma_q * rm * nq + p.abs_res * (na + rm)) +
                    8.f * kUnit * (fabsf(Q) + rm * rm + 2.f * cn * rm + 2.f * rm * nq + qq) + 1e-30f;
  return Q - eps;
}

#endif


// Scan tile categories (plan.cu): tensor-core tiles of <= 16 queries (16-wide scan), of <= 32
// queries (32-wide scan), and FFMA tiles.
constexpr int kTileCats = 3;
constexpr int kCatNarrow = 0, kCatWide = 1, kCatFfma = 2;

struct PlanParams {
  const int* probes;          // B x nprobe
  unsigned* bitmap;           // nlist x W
  int W;                      // words per list = ceil(B / 32)
  const long long* list_off;  // nlist + 1 (global rows)
  const long long* res_row0;  // nlist: row in the resident arena, -1 = offloaded
  int* list_nq;               // nlist
  int* list_qoff;             // nlist
  int* list_ntile;            // kTileCats x nlist: resident tiles per category
  int* list_toff;             // kTileCats x nlist
  int* list_q;                // B x nprobe
  ScanTile* tiles[kTileCats]; // tile arrays per category
  int* meta;                  // per category c: [2c] #tiles, [2c + 1] the scan's tile counter
  unsigned long long* counters;  // [0] unique lists, [1] resident rows probed, [2] offloaded rows probed
  int B, nlist, nprobe, R, tc_min_q;
  int tc_mode;                // 0: lists of <= 16 queries narrow, others wide; 16 / 32: one width
  // lists j >= tail_from are cut at Rt (<= R) rows: the scan's dynamic queue hands out tiles in
  // list order, so its last tiles are the short ones and the CTAs finish closer together
  int Rt, tail_from;
  unsigned long long* dbg = nullptr;  // RD_DEBUG_TS: globaltimer checkpoints of CTA 0
};
struct SelectParams {
  const float* Dc;         // B x nlist
  const float* queries;    // B x d
  const float* qnorm;      // B
  const float* centroids;  // nlist x d
  int* probes;             // B x nprobe
  unsigned* probe_fail;    // device scalar
  int B, nlist, nprobe, d;
  float cmax;              // max ||c||
  // fused seeding of the scan's pruning threshold (coarse.cu, seed phase); qthr == nullptr skips it
  const long long* list_off;
  const long long* res_row0;
  const float* arena;
  float xmax;
  int* qthr;
  int exact_order;         // 1: probes in exact (distance, list id) order (rd_probe); 0: the set (search)
  unsigned long long* dbg = nullptr;  // RD_DEBUG_TS: globaltimer checkpoints of CTA 0
  // the multi-kernel plan's list x query bitmap (nlist x W words, zero on entry): the selection
  // sets each probe's bit as it writes the probe, so the plan needs no inversion pass
  unsigned* bitmap = nullptr;
  int W = 0;
  // seeding rows: the threshold must bound the (seed_rows)-th best distance (= thr_rank + 1 of the
  // scans), so a list with at least that many rows can seed
  int seed_rows = 32;
  float gamma_coarse = 0.f;  // dot-product bound of the coarse path that filled Dc (gamma_* above)
  float gamma_scan = 0.f;    // dot-product bound of the scans the seed threshold prunes
  // split3 resident store (host.cuh; arena == nullptr then): seeding rows are rebuilt from it
  const __nv_bfloat16* x12 = nullptr;
  const __nv_bfloat16* x3 = nullptr;
  // B = 1 without offloaded lists, every list a tensor-core list: the selection CTA also plans the
  // scan (fp_tiles != nullptr: the narrow tile array; no plan launch): one tile per chunk of each
  // probed list, list_q, the byte counters and the tile count (the sorted-pairs plan's outputs)
  ScanTile* fp_tiles = nullptr;
  int* fp_list_q = nullptr;
  int* fp_meta = nullptr;
  unsigned long long* fp_counters = nullptr;
  int fp_R = 0, fp_Rt = 0;
};
// stage: q and candidate rows go through shared memory (latency-bound small batches)
// num_sms: batches beyond one resident wave of 256-thread CTAs (4 per SM) use 128-thread CTAs
cudaError_t launch_select(const SelectParams& p, bool stage, cudaStream_t s, int num_sms = 148);
bool select_staged(const SelectParams& p, bool stage);  // the staged (small-batch) variant will run


// Rows per scan chunk of a list of `len` rows under the plan's cap R (a multiple of kTcRows): the
// fewest chunks of <= R rows, balanced and rounded up to the tensor-core tile, so a list is not cut
// into full chunks plus a short remainder (2441 rows at R = 1152: 896 + 896 + 649, not
// 1152 + 1152 + 137) — every tile costs the scan a fixed overhead, whatever its length.
__host__ __device__ __forceinline__ int chunk_rows(long long len, int R) {
  if (len <= R) return R;
  const long long n = (len + R - 1) / R;
  const long long r = (len + n - 1) / n;
  const long long rr = (r + kTcRows - 1) / kTcRows * kTcRows;
  return (int)(rr < R ? rr : R);
}

cudaError_t launch_plan(const PlanParams& p, cudaStream_t s);
bool plan_fused_ok(int B, int nlist);  // the single-CTA bitmap plan applies
bool plan_small_ok(int B, int nprobe);  // the single-CTA sorted-pairs plan applies (B * nprobe <= 512)
// the multi-kernel plan reads the bitmap the selection filled (SelectParams::bitmap) and leaves it
// zero again for the next search
inline bool plan_uses_bitmap(int B, int nprobe, int nlist) { return !plan_small_ok(B, nprobe) && !plan_fused_ok(B, nlist); }

struct MergeParams {
  const float* part_dist;
  const int* part_row;
  const int* part_count;
  int part_cap;
  const float* queries;
  const float* qnorm;
  const long long* list_off;       // nlist + 1
  const float* const* list_base;   // nlist: device-visible pointer to the list's first row
  const long long* ids;            // n (global row order)
  const int* row_list;             // n: list of each global row
  const float* arena_lo;           // resident arena [lo, hi): rows there are bulk-copied (TMA), others
  const float* arena_hi;           // (mapped host memory of offloaded lists) are loaded by the threads
  int nlist, d, k;
  float xmax;
  long long* out_ids;              // B x k
  float* out_dists;                // B x k
  unsigned* margin_fail;            // device scalar: number of uncertified queries
  int* fail_list;                  // B: ids of uncertified queries (exact fallback work list)
  int B;
  // candidates reranked exactly (min(32, k + margin)); the next one's distance certifies
  int m_rerank = 32;
  unsigned long long* dbg = nullptr;  // RD_DEBUG_TS: globaltimer checkpoints of CTA 0
  float gamma = 0.f;               // dot-product bound of the scans that produced the candidates
  // split3 resident store: a list whose list_base is nullptr has its rows at res_row0 in x12 / x3
  const long long* res_row0 = nullptr;
  const __nv_bfloat16* x12 = nullptr;
  const __nv_bfloat16* x3 = nullptr;
};
// stage: the 32 rerank rows go through shared memory (latency-bound small batches)
cudaError_t launch_merge(const MergeParams& p, bool stage, cudaStream_t s);


// Exact fallback for uncertified queries: every row of every probed list is compared
// with the canonical exact distance and ordered by (distance, id).
struct FallbackParams {
  const int* fail_list;
  const unsigned* fail_count;
  const int* probes;               // B x nprobe
  int nprobe;
  const float* queries;
  const long long* list_off;
  const float* const* list_base;
  const long long* ids;
  int nlist, d, k;
  float* fb_dist;                  // B x nprobe x 32
  long long* fb_id;
  long long* out_ids;
  float* out_dists;
  unsigned* done_ctr;              // device scalar, 0 between launches (the kernel re-arms it)
  const long long* res_row0 = nullptr;  // split3 store, as MergeParams
  const __nv_bfloat16* x12 = nullptr;
  const __nv_bfloat16* x3 = nullptr;
};
cudaError_t launch_fallback(const FallbackParams& p, int num_sms, cudaStream_t s);

// Beyond the fast path (wide.cu): nprobe + 32 > 512 takes the probe set from the exact distance to
// every centroid (sorted by (distance, list id)); k > kMaxK an exact query-major pass over the probed
// lists whose per-query S x 32R survivors [S][B][32R] the shard merge reduces to the top-k.
size_t select_all_scratch_bytes(long long Bsub, int nlist);
long long select_all_batch(int nlist);
cudaError_t launch_select_all(const float* Q, const float* C, long long B, int nlist, int d, int nprobe, int* probes,
                              unsigned* bitmap, int W, void* scratch, size_t scratch_bytes, cudaStream_t s);
struct WideParams {
  const float* queries;
  const int* probes;  // B x nprobe
  int nprobe;
  const long long* list_off;
  const float* const* list_base;
  const long long* res_row0;
  const __nv_bfloat16* x12;
  const __nv_bfloat16* x3;
  const long long* ids;
  int d, k;
  long long B;
  float* out_d;       // S x B x 32R
  long long* out_id;
  int* qthr;          // B: running per-query threshold (f2ord), huge on entry
};
int wide_lists(int k);
int wide_splits(long long B, int nprobe, int k, int num_sms);
cudaError_t launch_wide(const WideParams& p, int S, cudaStream_t s);

// [G][B][k] shard results -> [B][k] (device), any k with G * k <= shard_merge_max_candidates()
cudaError_t launch_shard_merge(int G, long long B, int k, const long long* ids, const float* dists,
                               long long* out_ids, float* out_dists, cudaStream_t s);
int shard_merge_max_candidates();
// the same with shard g's B x k ids at ids + g * ids_stride bytes and distances at dists + g * d_stride
// (kout: results per query written, <= G * k; 0 = k)
cudaError_t launch_shard_merge_strided(int G, long long B, int k, const char* ids, size_t ids_stride,
                                       const char* dists, size_t d_stride, long long* out_ids, float* out_dists,
                                       cudaStream_t s, int kout = 0);

// Index build helpers
cudaError_t launch_gen_centroids(float* C, int nlist, int d, uint64_t sc, cudaStream_t s);
cudaError_t launch_gen_vectors(float* X, const long long* ids, long long n, int d, int nlist,
                               const float* C, uint64_t sa, uint64_t sx, float sigma, cudaStream_t s);
cudaError_t launch_row_norms(const float* X, long long n, int d, float* out, cudaStream_t s);
cudaError_t launch_max_f32(const float* v, long long n, float* out, cudaStream_t s);
// split3 resident store (host.cuh): x12 [rows][2][d] bf16 (x1, x2), x3 [rows][d] bf16, (x1 + x2) + x3 == x
// bit for bit; elements that do not round-trip are added to *inexact (device counter)
cudaError_t launch_split3(const float* X, long long rows, int d, void* x12, void* x3, unsigned* inexact,
                          cudaStream_t s);
cudaError_t launch_join3(const void* x12, const void* x3, long long rows, int d, float* X, cudaStream_t s);
// IVF training (train.cu)
cudaError_t launch_iota(int* v, long long n, cudaStream_t s);
cudaError_t launch_histogram(const int* keys, long long n, unsigned* counts, int nbins, cudaStream_t s);
// stable radix sort of (key, value) pairs on bits [0, end_bit); temp == nullptr queries *temp_bytes
cudaError_t sort_pairs(const int* keys_in, int* keys_out, const int* vals_in, int* vals_out, long long n, int end_bit,
                       void* temp, size_t* temp_bytes, cudaStream_t s);
// C[l] = fp64 sum of X[rows[seg[l] .. seg[l+1])] in order / count (empty clusters untouched)
cudaError_t launch_centroid_update(const float* X, const int* rows, const long long* seg, int nlist, int d, float* C,
                                   cudaStream_t s);
cudaError_t launch_gather_rows(const float* src, const int* idx, long long count, int d, float* dst, cudaStream_t s);
// out[i] = ids ? ids[idx[i]] : idx[i]
cudaError_t launch_gather_ids(const long long* ids, const int* idx, long long count, long long* out, cudaStream_t s);
// row_list[r] = l for off[l] <= r < off[l + 1]
cudaError_t launch_row_list(const long long* off, int nlist, int* row_list, cudaStream_t s);

}  // namespace rd
