// api.cu — host side of the B200 retrieval engine behind include/rd.h.
//
// Owns the index in HBM (list-order arena, norms, ids, centroids), the pinned
// host arena of offloaded lists, the H2D staging ring, per-search workspaces,
// streams and events, and orchestrates one search:
//
//   qnorm -> N1 coarse GEMM -> N2 select+exact refine -> N3 plan
//     -> N4 resident scan (persistent, main stream)
//     || N9 offloaded lists: cudaMemcpyAsync pinned->staging on a copy stream,
//        event-gated scans of staged slots on a side stream
//   -> N6/N7 merge + exact rerank -> results
//
// Reference seam: retrieval_time(P, db) (cost_model.cpp:15-21), called by the
// retrieval worker (simulator.cpp:359,560). Error model: ragsim exit codes
// (tools/main.cpp:30) with the message in rd_last_error().
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rd.h"
#include "../../include/rd_format.h"
#include "ivf_kernels.cuh"
#include "rd_device.cuh"

namespace {

thread_local std::string g_err;

struct RdError : std::runtime_error {
  int code;
  RdError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_rd(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw RdError(code, buf);
}

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw_rd(RD_ERR_RUNTIME, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
               __LINE__);                                                                       \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return RD_OK;
  } catch (const RdError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return RD_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RD_ERR_RUNTIME;
  }
}

// ------------------------------------------------------------------ device buffers
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      throw_rd(RD_ERR_RUNTIME, "cudaMalloc(%zu bytes) failed: %s", count * sizeof(T), cudaGetErrorString(e));
    }
    n = count;
  }
  void ensure(size_t count) {
    if (count > n) alloc(std::max(count, n + n / 2));
  }
};

template <class T>
struct HBuf {  // pinned, mapped host memory
  T* p = nullptr;
  size_t n = 0;
  HBuf() = default;
  HBuf(const HBuf&) = delete;
  HBuf& operator=(const HBuf&) = delete;
  ~HBuf() { reset(); }
  void reset() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    reset();
    if (count == 0) count = 1;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), count * sizeof(T),
                                  cudaHostAllocPortable | cudaHostAllocMapped);
    if (e != cudaSuccess) {
      p = nullptr;
      throw_rd(RD_ERR_RUNTIME, "cudaHostAlloc(%zu bytes) failed: %s", count * sizeof(T), cudaGetErrorString(e));
    }
    n = count;
  }
  void ensure(size_t count) {
    if (count > n) alloc(std::max(count, n + n / 2));
  }
};

// ------------------------------------------------------------------ tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !ptr) throw_rd(RD_ERR_RUNTIME, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

// 3D bf16 map over a [rows][2][d] (hi, lo) split buffer, box {64 dims, 1 part, 128 rows}, 128B swizzle.
CUtensorMap make_split_map(const void* base, long long rows, int d, int box_rows = 128) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  if (rows < 1) rows = 1;
  cuuint64_t dims[3] = {(cuuint64_t)d, 2, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)d * 4};
  cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw_rd(RD_ERR_RUNTIME, "cuTensorMapEncodeTiled (split) failed (%d)", (int)r);
  return m;
}

// 2D bf16 map over the [rows][2][d] split buffer viewed as [2*rows x d], box {64, 1} (gather4 source).
CUtensorMap make_gather_map(const void* base, long long rows, int d) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  if (rows < 1) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)(2 * rows)};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw_rd(RD_ERR_RUNTIME, "cuTensorMapEncodeTiled (gather) failed (%d)", (int)r);
  return m;
}

// 2D fp32 map over rows x d, box [32 dims x box_rows], 128B swizzle.
CUtensorMap make_row_map(const float* base, long long rows, int d, int box_rows) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  if (rows < 1) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)rd::kScanKSlice, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw_rd(RD_ERR_RUNTIME, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return m;
}

// ------------------------------------------------------------------ host arithmetic
inline uint64_t derive_seed(uint64_t master, uint64_t stream) {
  return rd::splitmix_at(master ^ (stream * 0xd1b54a32d192ed03ull), 1);
}

void parallel_for(long long n, const std::function<void(long long, long long)>& fn) {
  unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 65536 || T == 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  const long long chunk = (n + T - 1) / T;
  for (unsigned i = 0; i < T; ++i) {
    const long long b = i * chunk, e = std::min(n, b + chunk);
    if (b < e) th.emplace_back(fn, b, e);
  }
  for (auto& t : th) t.join();
}

}  // namespace

// ====================================================================== the index
constexpr size_t kStatBytes = 64;  // per-search counter block (see rd_index::Ws::blk)

struct rd_index {
  int device = 0;
  int num_sms = 148;
  int tc_min_q = rd::kTcMinQ;
  int debug_skip = 0;  // profiling only
  bool dbg_ts = std::getenv("RD_DEBUG_TS") != nullptr;  // profiling only: select checkpoints to stderr
  int stage_max_b = -1;  // batches up to this size stage exact-distance rows in smem (-1: 2 x SMs)
  int tiles_per_sm = 8;  // scan tiles per SM the planner aims for (RD_TILES_PER_SM)
  long long seed_max_b = 1LL << 40;  // batches up to this size seed the scan's pruning threshold (RD_SEED_MAX_B)
  bool no_inner_events = std::getenv("RD_NO_INNER_EVENTS") != nullptr;  // A/B: no per-stage timing events
  // the tensor-core scan stages 64-dim bf16 query slices of up to 32 queries in shared memory:
  // d % 64 == 0 and d <= 896 (beyond, its B operand does not fit next to the x ring); else FFMA
  bool tc_scan() const { return d % 64 == 0 && rd::scan_tc_smem_bytes(d) <= 227 * 1024; }
  bool stage_rows(long long B) const { return B <= (stage_max_b >= 0 ? stage_max_b : 2LL * num_sms); }
  long long n = 0;
  int d = 0, nlist = 0;
  std::vector<long long> list_off;  // host copy, nlist + 1
  long long max_len = 0;
  float cmax = 0.f, xmax = 0.f;

  DBuf<float> centroids, cnorm, xnorm, arena;
  DBuf<float> csplit;  // nlist x 2 x d bf16 (c1, c2) for the tensor-core coarse GEMM
  CUtensorMap cmap{};
  // pre-split bf16 (x1, x2) copy of the resident arena for the conversion-free tensor-core scan;
  // kept only while every list is resident and device memory allows (RD_PRESPLIT=0 disables)
  DBuf<float> xsplit;
  CUtensorMap xmap128{}, xmap32{};
  bool presplit = false;
  bool budgeted = false;  // last placement had an HBM byte budget
  DBuf<long long> d_list_off, d_ids, d_res_row0;
  DBuf<int> d_row_list;  // list of each global row (merge: row -> list without a search)
  DBuf<const float*> d_list_base;
  std::vector<uint8_t> resident;      // host mask
  std::vector<long long> res_row0;    // host: row in arena or -1
  std::vector<long long> host_row0;   // host: row in host arena or -1
  long long n_resident = 0;
  HBuf<float> host_arena;
  long long host_used = 0;            // rows of host_arena holding list copies (write-once per list)
  CUtensorMap map256{}, map128{}, map32{};

  // staging ring for offloaded lists
  int slots = 0;
  long long slot_rows = 0;
  DBuf<float> staging;
  CUtensorMap smap256{}, smap128{}, smap32{};

  // per-search workspace
  struct Ws {
    DBuf<float> qnorm, Dc, q, qsplit;
    DBuf<int> probes, list_nq, list_qoff, list_ntile, list_toff, list_q, part_count, part_row, off_meta;
    DBuf<unsigned> bitmap, fb_ctr;
    DBuf<rd::ScanTile> tiles, ff_tiles, off_tiles;
    DBuf<float> part_dist;
    DBuf<long long> fb_id;
    DBuf<int> fail_list, qthr;
    DBuf<float> fb_dist;
    HBuf<float> hq;
    HBuf<int> h_nq, h_qoff, h_meta;
    // per-search counters in one block so a synced search reads them back with one copy:
    // [0, 24) counters (u64 x 3), [24, 32) fails (u32 x 2), [32, 48) meta (i32 x 4); the host path
    // places its result ids / distances right after (kStatBytes) and copies everything at once
    DBuf<char> blk;
    HBuf<char> h_blk;
    unsigned long long* counters() const { return reinterpret_cast<unsigned long long*>(blk.p); }
    unsigned* fails() const { return reinterpret_cast<unsigned*>(blk.p + 24); }
    int* meta() const { return reinterpret_cast<int*>(blk.p + 32); }
    HBuf<rd::ScanTile> h_tiles;
  } ws;

  cudaStream_t copy_stream = nullptr, off_stream = nullptr;
  cudaEvent_t ev[8] = {};
  // device-time accounting: 4 events per search (start, plan done, resident scan done, end)
  static constexpr int kRing = 64;
  cudaEvent_t tev[kRing][4] = {};
  long long t_recorded = 0, t_accounted = 0;
  rd_timing t_acc{};

  void account(long long i) {  // fold search i's events into t_acc (synchronizes on them)
    cudaEvent_t* e = tev[i % kRing];
    CK(cudaEventSynchronize(e[3]));
    float a = 0, b = 0, c = 0, t = 0;
    if (!no_inner_events) {
      CK(cudaEventElapsedTime(&a, e[0], e[1]));
      CK(cudaEventElapsedTime(&b, e[1], e[2]));
      CK(cudaEventElapsedTime(&c, e[2], e[3]));
    }
    CK(cudaEventElapsedTime(&t, e[0], e[3]));
    t_acc.searches += 1;
    t_acc.coarse_ms += a;
    t_acc.scan_ms += b;
    t_acc.tail_ms += c;
    t_acc.total_ms += t;
  }
  cudaEvent_t* next_timing_slot() {
    if (t_recorded - t_accounted >= kRing) account(t_accounted++);
    return tev[t_recorded++ % kRing];
  }
  std::vector<cudaEvent_t> slot_ready, slot_done;

  ~rd_index() {
    cudaSetDevice(device);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (off_stream) cudaStreamDestroy(off_stream);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    for (auto e : slot_ready) cudaEventDestroy(e);
    for (auto e : slot_done) cudaEventDestroy(e);
    for (auto& r : tev)
      for (auto e : r)
        if (e) cudaEventDestroy(e);
  }

  void init_runtime() {
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
    int major = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) throw_rd(RD_ERR_RUNTIME, "librd_b200 requires an sm_100 (B200) device, found sm_%d.x", major);
    CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&off_stream, cudaStreamNonBlocking));
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (auto& r : tev)
      for (auto& e : r) CK(cudaEventCreate(&e));
    if (const char* v = std::getenv("RD_TC_MIN_Q")) tc_min_q = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("RD_DEBUG_SKIP")) debug_skip = std::atoi(v);
    if (const char* v = std::getenv("RD_STAGE_MAX_B")) stage_max_b = std::atoi(v);
    if (const char* v = std::getenv("RD_TILES_PER_SM")) tiles_per_sm = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("RD_SEED_MAX_B")) seed_max_b = std::atoll(v);
    // the tensor-core scan stages bf16 query slices of 64 dims
  }

  void finish_layout() {
    max_len = 0;
    for (int l = 0; l < nlist; ++l) max_len = std::max(max_len, list_off[l + 1] - list_off[l]);
    d_list_off.alloc(nlist + 1);
    CK(cudaMemcpy(d_list_off.p, list_off.data(), sizeof(long long) * (nlist + 1), cudaMemcpyHostToDevice));
    d_row_list.alloc(n);
    CK(rd::launch_row_list(d_list_off.p, nlist, d_row_list.p, 0));
    // all lists resident in list order
    resident.assign(nlist, 1);
    res_row0.resize(nlist);
    host_row0.assign(nlist, -1);
    for (int l = 0; l < nlist; ++l) res_row0[l] = list_off[l];
    n_resident = n;
    upload_residency();
    prepare_centroids();
    DBuf<float> tmp;
    tmp.alloc(1);
    float m2 = 0;
    CK(rd::launch_max_f32(xnorm.p, n, tmp.p, 0));
    CK(cudaMemcpy(&m2, tmp.p, sizeof(float), cudaMemcpyDeviceToHost));
    xmax = std::sqrt(m2) * (1.f + 1e-6f);
    CK(cudaDeviceSynchronize());
    build_presplit();
  }

  // coarse-stage state derived from the centroids: ||c||^2, the bf16 (hi, lo) split and its TMA
  // map for the tensor-core coarse GEMM, and max ||c|| for the selection's error bound
  void prepare_centroids() {
    if (cnorm.n < (size_t)nlist) cnorm.alloc(nlist);
    CK(launch_row_norms_wrap(centroids.p, nlist, cnorm.p));
    if (d % 64 == 0) {
      if (csplit.n < (size_t)nlist * d) csplit.alloc((size_t)nlist * d);  // 2 x bf16 per element = one float
      CK(rd::launch_qsplit(centroids.p, csplit.p, nlist, d, 0));
      cmap = make_split_map(csplit.p, nlist, d);
    }
    DBuf<float> tmp;
    tmp.alloc(1);
    CK(rd::launch_max_f32(cnorm.p, nlist, tmp.p, 0));
    float m2 = 0;
    CK(cudaMemcpy(&m2, tmp.p, sizeof(float), cudaMemcpyDeviceToHost));
    cmax = std::sqrt(m2) * (1.f + 1e-6f);
  }

  void build_presplit() {
    presplit = false;
    xsplit.reset();
    const char* env = std::getenv("RD_PRESPLIT");
    // a byte budget (e.g. the LLM reservation, C5) must not be exceeded by a second copy
    if (!tc_scan() || (env && std::atoi(env) == 0) || n_resident == 0 || budgeted) return;
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const size_t need = (size_t)n_resident * d * 4;
    if (need + (size_t(4) << 30) > fr) return;  // not enough room: the converter path stays
    xsplit.alloc((size_t)n_resident * d);
    CK(rd::launch_qsplit(arena.p, xsplit.p, n_resident, d, 0));
    CK(cudaDeviceSynchronize());
    xmap128 = make_split_map(xsplit.p, n_resident, d, rd::kTcRows);
    xmap32 = make_split_map(xsplit.p, n_resident, d, 32);
    presplit = true;
  }

  // Profiling only (RD_DEBUG_TS): runs `launch` with its kernel's CTA-0 checkpoint buffer attached
  // (globaltimer at [i], clock64 at [16 + i], RD_TS in rd_device.cuh), waits, and prints the clock64
  // offsets of each checkpoint from the first. Otherwise just launches.
  template <class F>
  void traced(const char* name, cudaStream_t s, unsigned long long*& slot, F&& launch) {
    if (!dbg_ts) {
      launch();
      return;
    }
    if (!dbg_buf.p) dbg_buf.alloc(32);
    CK(cudaMemsetAsync(dbg_buf.p, 0, 32 * sizeof(unsigned long long), s));
    slot = dbg_buf.p;
    launch();
    slot = nullptr;
    unsigned long long t[32];
    CK(cudaMemcpyAsync(t, dbg_buf.p, sizeof t, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    fprintf(stderr, "%s [14]=%lld [15]=%lld cycles:", name, (long long)t[14], (long long)t[15]);
    for (int i = 1; i < 14; ++i)
      if (t[16 + i]) fprintf(stderr, " %d:%lld", i, (long long)(t[16 + i] - t[16]));
    fprintf(stderr, "\n");
  }
  DBuf<unsigned long long> dbg_buf, dbg_scan;

  // H2D staging ring for offloaded lists: `slots` slots of `slot_rows` rows (0 slots: none)
  void set_staging(int nslots, long long nrows) {
    for (auto e : slot_ready) cudaEventDestroy(e);
    for (auto e : slot_done) cudaEventDestroy(e);
    slot_ready.clear();
    slot_done.clear();
    staging.reset();
    slots = nslots;
    slot_rows = nrows;
    if (!slots) return;
    staging.alloc((size_t)slots * slot_rows * d);
    smap256 = make_row_map(staging.p, (long long)slots * slot_rows, d, rd::kScanRows);
    smap128 = make_row_map(staging.p, (long long)slots * slot_rows, d, rd::kTcRows);
    smap32 = make_row_map(staging.p, (long long)slots * slot_rows, d, 32);
    slot_ready.resize(slots);
    slot_done.resize(slots);
    for (int s = 0; s < slots; ++s) {
      CK(cudaEventCreateWithFlags(&slot_ready[s], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&slot_done[s], cudaEventDisableTiming));
    }
  }

  cudaError_t launch_row_norms_wrap(const float* X, long long rows, float* out) {
    return rd::launch_row_norms(X, rows, d, out, 0);
  }

  void upload_residency() {
    d_res_row0.alloc(nlist);
    CK(cudaMemcpy(d_res_row0.p, res_row0.data(), sizeof(long long) * nlist, cudaMemcpyHostToDevice));
    xsplit.reset();  // any relayout invalidates the pre-split copy (rebuilt by build_presplit)
    presplit = false;
    std::vector<const float*> base(nlist);
    for (int l = 0; l < nlist; ++l)
      base[l] = resident[l] ? arena.p + (size_t)res_row0[l] * d : host_arena.p + (size_t)host_row0[l] * d;
    d_list_base.alloc(nlist);
    CK(cudaMemcpy(d_list_base.p, base.data(), sizeof(const float*) * nlist, cudaMemcpyHostToDevice));
    map256 = make_row_map(arena.p, std::max(1LL, n_resident), d, rd::kScanRows);
    map128 = make_row_map(arena.p, std::max(1LL, n_resident), d, rd::kTcRows);
    map32 = make_row_map(arena.p, std::max(1LL, n_resident), d, 32);
  }
};

namespace {

void check_dims(int d) {
  if (d < 32 || d % 32 != 0 || d > 1024)
    throw_rd(RD_ERR_INVALID, "d must be a multiple of 32 in [32, 1024], got %d", d);
}

std::unique_ptr<rd_index> new_index(int device) {
  auto h = std::make_unique<rd_index>();
  h->device = device;
  h->init_runtime();
  return h;
}

}  // namespace

extern "C" {

const char* rd_last_error(void) { return g_err.c_str(); }
int rd_abi_version(void) { return RD_ABI_VERSION; }
const char* rd_backend(void) { return "b200-sm100a"; }

uint64_t rd_splitmix_at(uint64_t seed, uint64_t i) { return rd::splitmix_at(seed, i); }
uint64_t rd_derive_seed(uint64_t master, uint64_t stream) { return derive_seed(master, stream); }

float rd_exact_l2(const float* a, const float* b, int32_t d) {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int32_t t = 0; t < d; ++t) {
    volatile double df = (double)a[t] - (double)b[t];  // volatile: no contraction into an FMA
    volatile double sq = df * df;
    s[t & 7] = s[t & 7] + sq;
  }
  return (float)(((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7])));
}

static void validate_desc(const rd_synth_desc* s) {
  if (!s) throw_rd(RD_ERR_INVALID, "null synth descriptor");
  if (s->n < 1 || s->d < 1 || s->nlist < 1) throw_rd(RD_ERR_INVALID, "synth: n, d, nlist must be >= 1");
  if (s->num_shards < 1 || s->shard < 0 || s->shard >= s->num_shards)
    throw_rd(RD_ERR_INVALID, "synth: shard %d of %d out of range", s->shard, s->num_shards);
}

static void synth_vec_host(const rd_synth_desc* s, uint64_t sc, uint64_t sa, uint64_t sx, int64_t id, float* out) {
  const int a = (int)(rd::splitmix_at(sa, (uint64_t)id) % (uint64_t)s->nlist);
  for (int t = 0; t < s->d; ++t) {
    volatile float noise = s->sigma * rd::unif(sx, (uint64_t)id * s->d + t);
    out[t] = rd::unif(sc, (uint64_t)a * s->d + t) + noise;
  }
}

int rd_synth_vector(const rd_synth_desc* s, int64_t id, float* out) {
  return guarded([&] {
    validate_desc(s);
    if (id < 0 || id >= s->n || !out) throw_rd(RD_ERR_INVALID, "synth_vector: id out of range");
    synth_vec_host(s, derive_seed(s->seed, RD_STREAM_CENTROIDS), derive_seed(s->seed, RD_STREAM_ASSIGN),
                   derive_seed(s->seed, RD_STREAM_VECTOR_NOISE), id, out);
  });
}

int rd_synth_queries(const rd_synth_desc* s, int64_t b0, int64_t B, float qsigma, float* out, int64_t* src) {
  return guarded([&] {
    validate_desc(s);
    if (b0 < 0 || B < 0 || (B > 0 && !out)) throw_rd(RD_ERR_INVALID, "synth_queries: invalid arguments");
    const uint64_t sc = derive_seed(s->seed, RD_STREAM_CENTROIDS), sa = derive_seed(s->seed, RD_STREAM_ASSIGN),
                   sx = derive_seed(s->seed, RD_STREAM_VECTOR_NOISE),
                   sq = derive_seed(s->seed, RD_STREAM_QUERY_PICK), sn = derive_seed(s->seed, RD_STREAM_QUERY_NOISE);
    parallel_for(B * 64, [&](long long lo, long long hi) {
      for (long long i = (lo + 63) / 64; i < (hi + 63) / 64 && i < B; ++i) {
        const int64_t b = b0 + i;
        const int64_t r = (int64_t)(rd::splitmix_at(sq, (uint64_t)b) % (uint64_t)s->n);
        float* q = out + i * s->d;
        synth_vec_host(s, sc, sa, sx, r, q);
        for (int t = 0; t < s->d; ++t) {
          volatile float noise = qsigma * rd::unif(sn, (uint64_t)b * s->d + t);
          q[t] = q[t] + noise;
        }
        if (src) src[i] = r;
      }
    });
  });
}

int rd_index_create_synthetic(const rd_synth_desc* s, int32_t device, rd_index** out) {
  return guarded([&] {
    validate_desc(s);
    check_dims(s->d);
    if (!out) throw_rd(RD_ERR_INVALID, "null out");
    auto h = new_index(device);
    h->d = s->d;
    h->nlist = s->nlist;
    const long long n = s->n;
    const int nl = s->nlist, G = s->num_shards, g = s->shard;
    const uint64_t sa = derive_seed(s->seed, RD_STREAM_ASSIGN);
    // list membership on the host (counting sort, ids ascending within a list)
    std::vector<int32_t> assign(n);
    parallel_for(n, [&](long long lo, long long hi) {
      for (long long i = lo; i < hi; ++i) assign[i] = (int32_t)(rd::splitmix_at(sa, (uint64_t)i) % (uint64_t)nl);
    });
    std::vector<long long> full_len(nl, 0);
    for (long long i = 0; i < n; ++i) full_len[assign[i]]++;
    h->list_off.assign(nl + 1, 0);
    for (int l = 0; l < nl; ++l) {
      const long long lo = g * full_len[l] / G, hi = (long long)(g + 1) * full_len[l] / G;
      h->list_off[l + 1] = h->list_off[l] + (hi - lo);
    }
    h->n = h->list_off[nl];
    std::vector<long long> ids(std::max(1LL, h->n));
    {
      std::vector<long long> cursor(nl, 0);
      for (long long i = 0; i < n; ++i) {
        const int l = assign[i];
        const long long pos = cursor[l]++;
        const long long lo = g * full_len[l] / G, hi = (long long)(g + 1) * full_len[l] / G;
        if (pos >= lo && pos < hi) ids[h->list_off[l] + (pos - lo)] = i;
      }
    }
    std::vector<int32_t>().swap(assign);
    h->centroids.alloc((size_t)nl * h->d);
    h->cnorm.alloc(nl);
    CK(rd::launch_gen_centroids(h->centroids.p, nl, h->d, derive_seed(s->seed, RD_STREAM_CENTROIDS), 0));
    h->d_ids.alloc(h->n);
    CK(cudaMemcpy(h->d_ids.p, ids.data(), sizeof(long long) * h->n, cudaMemcpyHostToDevice));
    h->arena.alloc((size_t)h->n * h->d);
    CK(rd::launch_gen_vectors(h->arena.p, h->d_ids.p, h->n, h->d, nl, h->centroids.p, sa,
                              derive_seed(s->seed, RD_STREAM_VECTOR_NOISE), s->sigma, 0));
    h->xnorm.alloc(h->n);
    CK(rd::launch_row_norms(h->arena.p, h->n, h->d, h->xnorm.p, 0));
    h->finish_layout();
    *out = h.release();
  });
}

int rd_index_create_from_host(int64_t n, int32_t d, int32_t nlist, const float* vectors, const int64_t* list_offsets,
                              const float* centroids, const int64_t* ids, int32_t device, rd_index** out) {
  return guarded([&] {
    if (n < 0 || nlist < 1 || !list_offsets || !centroids || !out || (n > 0 && !vectors))
      throw_rd(RD_ERR_INVALID, "create_from_host: invalid arguments");
    check_dims(d);
    if (list_offsets[0] != 0 || list_offsets[nlist] != n)
      throw_rd(RD_ERR_INVALID, "create_from_host: list_offsets must run 0..n");
    for (int l = 0; l < nlist; ++l)
      if (list_offsets[l + 1] < list_offsets[l])
        throw_rd(RD_ERR_INVALID, "create_from_host: list_offsets not monotone at %d", l);
    if (n >= (1LL << 31)) throw_rd(RD_ERR_INVALID, "create_from_host: at most 2^31-1 vectors per handle");
    auto h = new_index(device);
    h->n = n;
    h->d = d;
    h->nlist = nlist;
    h->list_off.assign(list_offsets, list_offsets + nlist + 1);
    h->centroids.alloc((size_t)nlist * d);
    h->cnorm.alloc(nlist);
    CK(cudaMemcpy(h->centroids.p, centroids, sizeof(float) * (size_t)nlist * d, cudaMemcpyHostToDevice));
    h->arena.alloc((size_t)n * d);
    if (n) CK(cudaMemcpy(h->arena.p, vectors, sizeof(float) * (size_t)n * d, cudaMemcpyHostToDevice));
    h->d_ids.alloc(n);
    std::vector<long long> idv(std::max<int64_t>(1, n));
    for (long long i = 0; i < n; ++i) idv[i] = ids ? ids[i] : i;
    CK(cudaMemcpy(h->d_ids.p, idv.data(), sizeof(long long) * n, cudaMemcpyHostToDevice));
    h->xnorm.alloc(n);
    CK(rd::launch_row_norms(h->arena.p, n, d, h->xnorm.p, 0));
    h->finish_layout();
    *out = h.release();
  });
}

void rd_index_destroy(rd_index* h) { delete h; }

int rd_index_centroids(const rd_index* h, float* out) {
  return guarded([&] {
    if (!h || !out) throw_rd(RD_ERR_INVALID, "centroids: null argument");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpy(out, h->centroids.p, sizeof(float) * (size_t)h->nlist * h->d, cudaMemcpyDeviceToHost));
  });
}

// ---------------------------------------------------------------- IVF training (N10)
// Lloyd's k-means, exact and deterministic (include/rd.h, rd_index_build): assignment is the
// search's own coarse path with nprobe = 1 — tensor-core (or FFMA) distances, certified selection,
// canonical fp64 distances for ambiguous centroids — over batches of the vectors; the update is
// train.cu's ordered fp64 mean.
int rd_index_build(int64_t n, int32_t d, int32_t nlist, const float* vectors, const int64_t* ids, int32_t iters,
                   uint64_t seed, int32_t device, rd_index** out) {
  return guarded([&] {
    if (n < 1 || nlist < 1 || n < nlist || iters < 0 || !vectors || !out)
      throw_rd(RD_ERR_INVALID, "build: need n >= nlist >= 1, iters >= 0 and vectors");
    check_dims(d);
    if (n >= (1LL << 31)) throw_rd(RD_ERR_INVALID, "build: at most 2^31-1 vectors per handle");
    auto h = new_index(device);
    h->n = n;
    h->d = d;
    h->nlist = nlist;
    cudaStream_t s = 0;
    DBuf<float> X;  // input order
    X.alloc((size_t)n * d);
    CK(cudaMemcpy(X.p, vectors, sizeof(float) * (size_t)n * d, cudaMemcpyHostToDevice));
    {  // init: the first nlist distinct rows of u(s, i) mod n
      const uint64_t si = derive_seed(seed, RD_STREAM_TRAIN_INIT);
      std::vector<uint8_t> taken((size_t)n, 0);
      std::vector<int> pick;
      for (uint64_t i = 0; (int)pick.size() < nlist; ++i) {
        const long long r = (long long)(rd::splitmix_at(si, i) % (uint64_t)n);
        if (!taken[r]) {
          taken[r] = 1;
          pick.push_back((int)r);
        }
      }
      DBuf<int> dpick;
      dpick.alloc(nlist);
      CK(cudaMemcpy(dpick.p, pick.data(), sizeof(int) * nlist, cudaMemcpyHostToDevice));
      h->centroids.alloc((size_t)nlist * d);
      CK(rd::launch_gather_rows(X.p, dpick.p, nlist, d, h->centroids.p, s));
    }
    DBuf<int> assign, keys_sorted, rows, rows_sorted;
    DBuf<unsigned> counts;
    DBuf<long long> seg;
    DBuf<char> temp;
    assign.alloc(n);
    keys_sorted.alloc(n);
    rows.alloc(n);
    rows_sorted.alloc(n);
    counts.alloc(nlist);
    seg.alloc(nlist + 1);
    int end_bit = 1;
    while ((1LL << end_bit) < nlist) ++end_bit;
    size_t temp_bytes = 0;
    CK(rd::sort_pairs(nullptr, nullptr, nullptr, nullptr, n, end_bit, nullptr, &temp_bytes, s));
    temp.alloc(temp_bytes);
    std::vector<unsigned> hcount(nlist);
    std::vector<long long> hseg(nlist + 1);
    auto& w = h->ws;
    const long long chunk = std::max<long long>(1024, std::min<long long>(65536, (1LL << 28) / nlist));
    auto assign_all = [&] {
      h->prepare_centroids();
      w.qnorm.ensure(chunk);
      w.qsplit.ensure((size_t)chunk * d);
      w.Dc.ensure((size_t)chunk * nlist);
      w.blk.ensure(kStatBytes);
      for (long long b0 = 0; b0 < n; b0 += chunk) {
        const int B = (int)std::min(chunk, n - b0);
        const float* q = X.p + (size_t)b0 * d;
        CK(rd::launch_qprep(q, B, d, w.qnorm.p, d % 64 == 0 ? w.qsplit.p : nullptr, w.fails(), nullptr, s));
        if (d % 64 == 0) {
          const CUtensorMap qmap = make_split_map(w.qsplit.p, B, d);
          CK(rd::launch_coarse_tc(qmap, h->cmap, h->cnorm.p, w.Dc.p, B, nlist, d, s));
        } else {
          CK(rd::launch_coarse(q, h->centroids.p, h->cnorm.p, w.Dc.p, B, nlist, d, s));
        }
        rd::SelectParams sp{w.Dc.p, q, w.qnorm.p, h->centroids.p, assign.p + b0, w.fails(), B, nlist, 1, d,
                            h->cmax, nullptr, nullptr, nullptr, 0.f, nullptr, 0};
        CK(rd::launch_select(sp, false, s));
      }
    };
    auto group = [&] {  // rows stably sorted by cluster; per-cluster segments
      CK(rd::launch_iota(rows.p, n, s));
      CK(rd::sort_pairs(assign.p, keys_sorted.p, rows.p, rows_sorted.p, n, end_bit, temp.p, &temp_bytes, s));
      CK(rd::launch_histogram(assign.p, n, counts.p, nlist, s));
      CK(cudaMemcpyAsync(hcount.data(), counts.p, sizeof(unsigned) * nlist, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      hseg[0] = 0;
      for (int l = 0; l < nlist; ++l) hseg[l + 1] = hseg[l] + hcount[l];
      CK(cudaMemcpy(seg.p, hseg.data(), sizeof(long long) * (nlist + 1), cudaMemcpyHostToDevice));
    };
    for (int it = 0; it < iters; ++it) {
      assign_all();
      group();
      CK(rd::launch_centroid_update(X.p, rows_sorted.p, seg.p, nlist, d, h->centroids.p, s));
    }
    assign_all();
    group();
    // list-order layout
    h->list_off = hseg;
    h->arena.alloc((size_t)n * d);
    CK(rd::launch_gather_rows(X.p, rows_sorted.p, n, d, h->arena.p, s));
    DBuf<long long> uids;
    if (ids) {
      uids.alloc(n);
      CK(cudaMemcpy(uids.p, ids, sizeof(long long) * (size_t)n, cudaMemcpyHostToDevice));
    }
    h->d_ids.alloc(n);
    CK(rd::launch_gather_ids(ids ? uids.p : nullptr, rows_sorted.p, n, h->d_ids.p, s));
    CK(cudaStreamSynchronize(s));
    X.reset();
    h->xnorm.alloc(n);
    CK(rd::launch_row_norms(h->arena.p, n, d, h->xnorm.p, 0));
    h->finish_layout();
    *out = h.release();
  });
}

// ---------------------------------------------------------------- on-disk index (include/rd_format.h)
namespace {

void pwrite_all(int fd, const void* p, size_t bytes, uint64_t off, const char* path) {
  const char* b = static_cast<const char*>(p);
  while (bytes) {
    const ssize_t w = ::pwrite(fd, b, bytes, (off_t)off);
    if (w <= 0) throw_rd(RD_ERR_RUNTIME, "save: write to %s failed", path);
    b += w;
    off += (uint64_t)w;
    bytes -= (size_t)w;
  }
}
void pread_all(int fd, void* p, size_t bytes, uint64_t off, const char* path) {
  char* b = static_cast<char*>(p);
  while (bytes) {
    const ssize_t r = ::pread(fd, b, bytes, (off_t)off);
    if (r <= 0) throw_rd(RD_ERR_RUNTIME, "load: read from %s failed", path);
    b += r;
    off += (uint64_t)r;
    bytes -= (size_t)r;
  }
}
struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};
constexpr size_t kIoChunk = size_t(64) << 20;  // pinned bounce buffer (bytes)

}  // namespace

int rd_index_save(const rd_index* h, const char* path) {
  return guarded([&] {
    if (!h || !path) throw_rd(RD_ERR_INVALID, "save: null argument");
    CK(cudaSetDevice(h->device));
    rd_file_header hd;
    rd_fmt_layout(&hd, h->n, h->d, h->nlist);
    hd.check = rd_fmt_check(&hd, reinterpret_cast<const int64_t*>(h->list_off.data()));
    Fd f;
    f.fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) throw_rd(RD_ERR_RUNTIME, "save: cannot open %s for writing", path);
    std::vector<char> head(RD_FILE_ALIGN, 0);
    std::memcpy(head.data(), &hd, sizeof hd);
    pwrite_all(f.fd, head.data(), head.size(), 0, path);
    pwrite_all(f.fd, h->list_off.data(), 8 * (size_t)(h->nlist + 1), hd.off_list_offsets, path);
    {
      std::vector<long long> ids(std::max<long long>(1, h->n));
      if (h->n) CK(cudaMemcpy(ids.data(), h->d_ids.p, 8 * (size_t)h->n, cudaMemcpyDeviceToHost));
      pwrite_all(f.fd, ids.data(), 8 * (size_t)h->n, hd.off_ids, path);
      std::vector<float> c((size_t)h->nlist * h->d);
      CK(cudaMemcpy(c.data(), h->centroids.p, 4 * c.size(), cudaMemcpyDeviceToHost));
      pwrite_all(f.fd, c.data(), 4 * c.size(), hd.off_centroids, path);
    }
    // vectors in list order, gathered from HBM (resident lists) or pinned host memory (offloaded)
    HBuf<float> bounce;
    const size_t row_bytes = 4 * (size_t)h->d;
    const long long chunk_rows = std::max<long long>(1, (long long)(kIoChunk / row_bytes));
    bounce.alloc((size_t)chunk_rows * h->d);
    long long fill = 0, row = 0;  // rows in the bounce buffer; global row of its first row
    auto flush = [&] {
      if (!fill) return;
      pwrite_all(f.fd, bounce.p, (size_t)fill * row_bytes, hd.off_vectors + (uint64_t)row * row_bytes, path);
      row += fill;
      fill = 0;
    };
    for (int l = 0; l < h->nlist; ++l) {
      const long long len = h->list_off[l + 1] - h->list_off[l];
      const float* src = h->resident[l] ? h->arena.p + (size_t)h->res_row0[l] * h->d
                                        : h->host_arena.p + (size_t)h->host_row0[l] * h->d;
      for (long long r = 0; r < len;) {
        const long long take = std::min(len - r, chunk_rows - fill);
        CK(cudaMemcpy(bounce.p + (size_t)fill * h->d, src + (size_t)r * h->d, (size_t)take * row_bytes,
                      cudaMemcpyDefault));
        fill += take;
        r += take;
        if (fill == chunk_rows) flush();
      }
    }
    flush();
    if (::fsync(f.fd) != 0) throw_rd(RD_ERR_RUNTIME, "save: fsync of %s failed", path);
  });
}

int rd_index_load(const char* path, int32_t device, rd_index** out) {
  return guarded([&] {
    if (!path || !out) throw_rd(RD_ERR_INVALID, "load: null argument");
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) throw_rd(RD_ERR_INVALID, "load: cannot open %s", path);
    struct stat stt;
    if (::fstat(f.fd, &stt) != 0) throw_rd(RD_ERR_RUNTIME, "load: cannot stat %s", path);
    const uint64_t size = (uint64_t)stt.st_size;
    rd_file_header hd;
    if (size < sizeof hd) throw_rd(RD_ERR_INVALID, "load %s: truncated rd index file", path);
    pread_all(f.fd, &hd, sizeof hd, 0, path);
    if (const char* why = rd_fmt_validate(&hd, size, nullptr)) throw_rd(RD_ERR_INVALID, "load %s: %s", path, why);
    std::vector<long long> offs((size_t)hd.nlist + 1);
    pread_all(f.fd, offs.data(), 8 * offs.size(), hd.off_list_offsets, path);
    if (const char* why = rd_fmt_validate(&hd, size, reinterpret_cast<const int64_t*>(offs.data())))
      throw_rd(RD_ERR_INVALID, "load %s: %s", path, why);
    check_dims(hd.d);
    if (hd.n >= (1LL << 31)) throw_rd(RD_ERR_INVALID, "load: at most 2^31-1 vectors per handle");
    auto h = new_index(device);
    h->n = hd.n;
    h->d = hd.d;
    h->nlist = hd.nlist;
    h->list_off = offs;
    const int d = hd.d;
    {
      std::vector<float> c((size_t)hd.nlist * d);
      pread_all(f.fd, c.data(), 4 * c.size(), hd.off_centroids, path);
      h->centroids.alloc(c.size());
      h->cnorm.alloc(hd.nlist);
      CK(cudaMemcpy(h->centroids.p, c.data(), 4 * c.size(), cudaMemcpyHostToDevice));
      std::vector<long long> ids(std::max<long long>(1, hd.n));
      pread_all(f.fd, ids.data(), 8 * (size_t)hd.n, hd.off_ids, path);
      h->d_ids.alloc(hd.n);
      if (hd.n) CK(cudaMemcpy(h->d_ids.p, ids.data(), 8 * (size_t)hd.n, cudaMemcpyHostToDevice));
    }
    // vectors: file -> two pinned bounce buffers -> HBM; the read of chunk i+1 overlaps the copy of chunk i
    h->arena.alloc((size_t)hd.n * d);
    const uint64_t total = 4ull * (uint64_t)hd.n * d;
    HBuf<char> buf[2];
    cudaEvent_t done[2];
    for (int i = 0; i < 2; ++i) {
      buf[i].alloc(kIoChunk);
      CK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    try {
      for (uint64_t o = 0, i = 0; o < total; o += kIoChunk, ++i) {
        const size_t bytes = (size_t)std::min<uint64_t>(kIoChunk, total - o);
        if (i >= 2) CK(cudaEventSynchronize(done[i & 1]));
        pread_all(f.fd, buf[i & 1].p, bytes, hd.off_vectors + o, path);
        CK(cudaMemcpyAsync(reinterpret_cast<char*>(h->arena.p) + o, buf[i & 1].p, bytes, cudaMemcpyHostToDevice,
                           h->copy_stream));
        CK(cudaEventRecord(done[i & 1], h->copy_stream));
      }
      CK(cudaStreamSynchronize(h->copy_stream));
    } catch (...) {
      cudaStreamSynchronize(h->copy_stream);
      for (auto e : done) cudaEventDestroy(e);
      throw;
    }
    for (auto e : done) cudaEventDestroy(e);
    h->xnorm.alloc(hd.n);
    CK(rd::launch_row_norms(h->arena.p, hd.n, d, h->xnorm.p, 0));
    h->finish_layout();
    *out = h.release();
  });
}

int rd_index_info_get(const rd_index* h, rd_index_info* o) {
  return guarded([&] {
    if (!h || !o) throw_rd(RD_ERR_INVALID, "null argument");
    std::memset(o, 0, sizeof *o);
    o->n = h->n;
    o->d = h->d;
    o->nlist = h->nlist;
    o->n_resident = h->n_resident;
    for (int l = 0; l < h->nlist; ++l) o->lists_resident += h->resident[l];
    o->hbm_bytes = (uint64_t)h->n_resident * h->d * 4 + (uint64_t)h->n * 16 + (uint64_t)h->nlist * (h->d + 1) * 4 +
                   (uint64_t)h->slots * h->slot_rows * h->d * 4 + (uint64_t)h->xsplit.n * 4;
    o->host_pinned_bytes = (uint64_t)h->host_arena.n * 4;
    o->staging_slots = h->slots;
    o->max_norm = h->xmax;
    o->device = h->device;
  });
}

int rd_index_layout(const rd_index* h, int64_t* offs, int64_t* ids, uint8_t* mask) {
  return guarded([&] {
    if (!h) throw_rd(RD_ERR_INVALID, "null index");
    CK(cudaSetDevice(h->device));
    if (offs) std::memcpy(offs, h->list_off.data(), sizeof(int64_t) * (h->nlist + 1));
    if (ids && h->n) CK(cudaMemcpy(ids, h->d_ids.p, sizeof(int64_t) * h->n, cudaMemcpyDeviceToHost));
    if (mask) std::memcpy(mask, h->resident.data(), h->nlist);
  });
}

// ---------------------------------------------------------------- placement (N8)
int rd_index_place(rd_index* h, const rd_placement* p) {
  return guarded([&] {
    if (!h || !p) throw_rd(RD_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    const int nl = h->nlist;
    const uint64_t row_bytes = (uint64_t)h->d * sizeof(float);
    std::vector<uint8_t> mask(nl, 0);
    uint64_t res_bytes = 0;
    if (p->resident_mask) {
      for (int l = 0; l < nl; ++l) {
        mask[l] = p->resident_mask[l] ? 1 : 0;
        if (mask[l]) res_bytes += (uint64_t)(h->list_off[l + 1] - h->list_off[l]) * row_bytes;
      }
      if (p->hbm_budget_bytes && res_bytes > p->hbm_budget_bytes)
        throw_rd(RD_ERR_INFEASIBLE, "placement infeasible: resident lists need %llu bytes > budget %llu",
                 (unsigned long long)res_bytes, (unsigned long long)p->hbm_budget_bytes);
    } else {
      if (p->offload_fraction < 0 || p->offload_fraction > 1)
        throw_rd(RD_ERR_INVALID, "offload_fraction must be in [0, 1]");
      std::vector<int> order(nl);
      for (int l = 0; l < nl; ++l) order[l] = l;
      if (p->list_heat)
        std::stable_sort(order.begin(), order.end(),
                         [&](int a, int b) { return p->list_heat[a] > p->list_heat[b]; });
      const long long target = nl - (long long)std::floor(p->offload_fraction * nl + 0.5);
      // the budget covers the resident lists and, once anything is offloaded, a staging ring of
      // at least two slots of max(largest list, 16384 rows) (include/rd.h, rd_placement)
      uint64_t budget = p->hbm_budget_bytes;
      if (budget) {
        uint64_t all = 0;
        for (long long i = 0; i < target; ++i)
          all += (uint64_t)(h->list_off[order[i] + 1] - h->list_off[order[i]]) * row_bytes;
        if (target < nl || all > budget) {
          const uint64_t slot = (uint64_t)((std::max<long long>(h->max_len, 16384) + 255) / 256 * 256) * row_bytes;
          const uint64_t reserve = (uint64_t)std::max(2, p->staging_slots) * slot;
          if (reserve > budget)
            throw_rd(RD_ERR_INFEASIBLE, "placement infeasible: budget %llu below the %llu-byte staging ring",
                     (unsigned long long)budget, (unsigned long long)reserve);
          budget -= reserve;
        }
      }
      for (long long i = 0; i < target; ++i) {
        const int l = order[i];
        const uint64_t lb = (uint64_t)(h->list_off[l + 1] - h->list_off[l]) * row_bytes;
        if (budget && res_bytes + lb > budget) break;
        res_bytes += lb;
        mask[l] = 1;
      }
    }
    // relayout: resident lists compact into a new arena, the rest to pinned host memory
    long long n_res = 0, n_off = 0, max_off = 0;
    for (int l = 0; l < nl; ++l) {
      const long long len = h->list_off[l + 1] - h->list_off[l];
      if (mask[l])
        n_res += len;
      else {
        n_off += len;
        max_off = std::max(max_off, len);
      }
    }
    // staging ring: slots of >= the largest offloaded list; depth by the queue_capacity rule
    long long slot_rows = 0;
    int slots = 0;
    if (n_off > 0) {
      slot_rows = std::max<long long>(max_off, 16384);
      slot_rows = (slot_rows + 255) / 256 * 256;
      const double slot_bytes = (double)slot_rows * row_bytes;
      double free_bytes;
      if (p->hbm_budget_bytes) {
        free_bytes = (double)p->hbm_budget_bytes - (double)res_bytes;
      } else {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        free_bytes = (double)fr - (double)(1ull << 30);
      }
      slots = p->staging_slots > 0 ? p->staging_slots : std::min(8, rd_staging_depth(free_bytes, slot_bytes));
      if (p->hbm_budget_bytes && res_bytes + slots * slot_bytes > (double)p->hbm_budget_bytes)
        throw_rd(RD_ERR_INFEASIBLE, "placement infeasible: no room for one %.0f-byte staging slot in the budget",
                 slot_bytes);
    }
    HBuf<float> new_host;
    std::vector<long long> new_res(nl, -1), new_host_row(nl, -1);
    if (n_off) new_host.alloc((size_t)n_off * h->d);
    DBuf<float> new_arena;
    new_arena.alloc((size_t)std::max(1LL, n_res) * h->d);
    long long rr = 0, hr = 0;
    for (int l = 0; l < nl; ++l) {
      const long long len = h->list_off[l + 1] - h->list_off[l];
      const float* src = h->resident[l] ? h->arena.p + (size_t)h->res_row0[l] * h->d
                                        : h->host_arena.p + (size_t)h->host_row0[l] * h->d;
      if (mask[l]) {
        new_res[l] = rr;
        if (len) CK(cudaMemcpy(new_arena.p + (size_t)rr * h->d, src, len * row_bytes, cudaMemcpyDefault));
        rr += len;
      } else {
        new_host_row[l] = hr;
        if (len) CK(cudaMemcpy(new_host.p + (size_t)hr * h->d, src, len * row_bytes, cudaMemcpyDefault));
        hr += len;
      }
    }
    CK(cudaDeviceSynchronize());
    std::swap(h->arena.p, new_arena.p);
    std::swap(h->arena.n, new_arena.n);
    std::swap(h->host_arena.p, new_host.p);
    std::swap(h->host_arena.n, new_host.n);
    h->resident = mask;
    h->res_row0 = new_res;
    h->host_row0 = new_host_row;
    h->n_resident = n_res;
    h->host_used = n_off;
    h->budgeted = p->hbm_budget_bytes != 0;
    h->upload_residency();
    h->build_presplit();
    h->set_staging(slots, slot_rows);
  });
}

// ---------------------------------------------------------------- migration
int rd_index_migrate(rd_index* h, const int32_t* promote, int32_t n_promote, const int32_t* demote, int32_t n_demote,
                     uint64_t hbm_budget_bytes, rd_migration_stats* st) {
  return guarded([&] {
    if (!h || n_promote < 0 || n_demote < 0 || (n_promote && !promote) || (n_demote && !demote))
      throw_rd(RD_ERR_INVALID, "migrate: invalid arguments");
    CK(cudaSetDevice(h->device));
    const auto t0 = std::chrono::steady_clock::now();
    const int nl = h->nlist, d = h->d;
    const size_t row_bytes = (size_t)d * sizeof(float);
    auto len_of = [&](int l) { return h->list_off[l + 1] - h->list_off[l]; };
    std::vector<uint8_t> seen(nl, 0);
    for (int i = 0; i < n_promote + n_demote; ++i) {
      const bool is_p = i < n_promote;
      const int l = is_p ? promote[i] : demote[i - n_promote];
      const char* why = nullptr;
      if (l < 0 || l >= nl)
        why = "list id out of range";
      else if (seen[l])
        why = "list named twice";
      else if (is_p && h->resident[l])
        why = "promoted list is already resident";
      else if (!is_p && !h->resident[l])
        why = "demoted list is not resident";
      if (why) throw_rd(RD_ERR_INVALID, "migrate: %s (%d)", why, l);
      seen[l] = 1;
    }
    std::vector<uint8_t> after(h->resident);
    for (int l = 0; l < nl; ++l)
      if (seen[l]) after[l] = !after[l];
    long long res_rows = 0, max_off = -1;
    for (int l = 0; l < nl; ++l) {
      if (after[l])
        res_rows += len_of(l);
      else
        max_off = std::max(max_off, len_of(l));
    }
    const long long slot_rows = max_off >= 0 ? (std::max<long long>(max_off, 16384) + 255) / 256 * 256 : 0;
    if (hbm_budget_bytes) {
      const uint64_t need = (uint64_t)res_rows * row_bytes + (max_off >= 0 ? 2ull * slot_rows * row_bytes : 0);
      if (need > hbm_budget_bytes)
        throw_rd(RD_ERR_INFEASIBLE, "migration infeasible: %llu bytes needed > budget %llu",
                 (unsigned long long)need, (unsigned long long)hbm_budget_bytes);
    }
    rd_migration_stats ms;
    std::memset(&ms, 0, sizeof ms);
    cudaStream_t cs = h->copy_stream;
    // 1. demote: lists without a host copy go to pinned host memory (write-once copies)
    long long need_host = h->host_used;
    for (int i = 0; i < n_demote; ++i)
      if (h->host_row0[demote[i]] < 0) need_host += len_of(demote[i]);
    if ((size_t)need_host * d > h->host_arena.n) {  // grow the host arena, keeping its contents
      HBuf<float> grown;
      grown.alloc((size_t)std::max<long long>(need_host, h->host_used + h->host_used / 2) * d);
      if (h->host_used) std::memcpy(grown.p, h->host_arena.p, (size_t)h->host_used * row_bytes);
      std::swap(h->host_arena.p, grown.p);
      std::swap(h->host_arena.n, grown.n);
    }
    for (int i = 0; i < n_demote; ++i) {
      const int l = demote[i];
      if (h->host_row0[l] >= 0) continue;
      const size_t bytes = (size_t)len_of(l) * row_bytes;
      CK(cudaMemcpyAsync(h->host_arena.p + (size_t)h->host_used * d, h->arena.p + (size_t)h->res_row0[l] * d, bytes,
                         cudaMemcpyDeviceToHost, cs));
      h->host_row0[l] = h->host_used;
      h->host_used += len_of(l);
      ms.d2h_bytes += bytes;
    }
    CK(cudaStreamSynchronize(cs));
    // 2. compact the lists that stay resident, in arena order, toward row 0 (forward chunked copies
    //    never overlap: a chunk is at most the shift)
    std::vector<int> keep;
    for (int l = 0; l < nl; ++l)
      if (h->resident[l] && after[l]) keep.push_back(l);
    std::sort(keep.begin(), keep.end(), [&](int a, int b) { return h->res_row0[a] < h->res_row0[b]; });
    long long tail = 0;
    for (int l : keep) {
      const long long old = h->res_row0[l], len = len_of(l);
      if (old != tail && len > 0) {
        const long long chunk = std::min(len, old - tail);
        for (long long r = 0; r < len; r += chunk) {
          const long long c = std::min(chunk, len - r);
          CK(cudaMemcpyAsync(h->arena.p + (size_t)(tail + r) * d, h->arena.p + (size_t)(old + r) * d, (size_t)c * row_bytes,
                             cudaMemcpyDeviceToDevice, cs));
        }
        ms.d2d_bytes += (size_t)len * row_bytes;
      }
      h->res_row0[l] = tail;
      tail += len;
    }
    for (int i = 0; i < n_demote; ++i) h->res_row0[demote[i]] = -1;
    // 3. promote into the freed space (the arena grows only if the resident set outgrows it)
    if ((size_t)res_rows * d > h->arena.n) {
      DBuf<float> grown;
      grown.alloc((size_t)res_rows * d);
      if (tail) CK(cudaMemcpyAsync(grown.p, h->arena.p, (size_t)tail * row_bytes, cudaMemcpyDeviceToDevice, cs));
      CK(cudaStreamSynchronize(cs));
      std::swap(h->arena.p, grown.p);
      std::swap(h->arena.n, grown.n);
    }
    for (int i = 0; i < n_promote; ++i) {
      const int l = promote[i];
      const size_t bytes = (size_t)len_of(l) * row_bytes;
      if (bytes)
        CK(cudaMemcpyAsync(h->arena.p + (size_t)tail * d, h->host_arena.p + (size_t)h->host_row0[l] * d, bytes,
                           cudaMemcpyHostToDevice, cs));
      h->res_row0[l] = tail;
      tail += len_of(l);
      ms.h2d_bytes += bytes;
    }
    CK(cudaStreamSynchronize(cs));
    h->resident = after;
    h->n_resident = tail;
    if (hbm_budget_bytes) h->budgeted = true;
    // 4. staging ring for the new offloaded set (slot >= its largest list)
    if (max_off < 0)
      h->set_staging(0, 0);
    else if (h->slots == 0 || h->slot_rows < slot_rows)
      h->set_staging(std::max(2, h->slots), slot_rows);
    h->upload_residency();
    h->build_presplit();
    ms.lists_promoted = n_promote;
    ms.lists_demoted = n_demote;
    ms.resident_bytes = (uint64_t)tail * row_bytes;
    ms.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (st) *st = ms;
  });
}

// ---------------------------------------------------------------- search
namespace {

struct Plan {
  int R;
  int max_chunks;
  int cap;
  long long max_tiles;
};

Plan make_plan(const rd_index* h, long long B, int nprobe) {
  Plan pl;
  const int np = std::min(nprobe, h->nlist);
  const double avg = h->nlist ? (double)h->n / h->nlist : 0.0;
  const double est_rows = std::min((double)h->n, (double)B * np * avg);
  // ~tiles_per_sm tiles per SM so the dynamic tile queue's tail (at most one tile per SM) stays
  // short; rows rounded to the tensor-core tile (128), at least one 256-row TMA box of the FFMA scan
  // when that path is in use
  const long long gran = rd::kTcRows;
  long long R = (long long)std::ceil(est_rows / ((double)h->num_sms * h->tiles_per_sm));
  R = std::max<long long>(h->tc_min_q > 1 || !h->tc_scan() ? rd::kScanRows : gran,
                          std::min<long long>(4096, (R + gran - 1) / gran * gran));
  pl.R = (int)R;
  pl.max_chunks = (int)std::max<long long>(1, (h->max_len + R - 1) / R);
  pl.cap = np * pl.max_chunks * rd::kPartsPerTile;
  pl.max_tiles = std::min<long long>(B * np, B * np / rd::kScanG + h->nlist) * pl.max_chunks + 1;
  return pl;
}

// result_bytes: bytes after the stat block that the sync copy brings back too (the host path's results)
void do_search(rd_index* h, const float* d_q, long long B, int nprobe, int k, long long* d_ids, float* d_dists,
               cudaStream_t s, bool sync, rd_search_stats* st, size_t result_bytes = 0,
               const std::function<void()>& before_sync = {}) {
  if (nprobe < 1 || k < 1) throw_rd(RD_ERR_INVALID, "search: nprobe >= 1 and k >= 1 required");
  if (k > rd::kMaxK) throw_rd(RD_ERR_INVALID, "search: k <= %d supported, got %d", rd::kMaxK, k);
  if (std::min(nprobe, h->nlist) + rd::kCoarseExtra > 512) throw_rd(RD_ERR_INVALID, "search: nprobe <= 480 supported");
  CK(cudaSetDevice(h->device));
  auto& w = h->ws;
  const int nl = h->nlist, d = h->d;
  const Plan pl = make_plan(h, B, nprobe);
  const int W = (int)((B + 31) / 32);
  w.qnorm.ensure(B);
  w.Dc.ensure((size_t)B * nl);
  w.probes.ensure((size_t)B * nprobe);
  w.bitmap.ensure((size_t)nl * W);
  w.list_nq.ensure(nl);
  w.list_qoff.ensure(nl);
  w.list_ntile.ensure(2 * (size_t)nl);
  w.list_toff.ensure(2 * (size_t)nl);
  w.list_q.ensure((size_t)B * nprobe);
  w.tiles.ensure(pl.max_tiles);
  w.ff_tiles.ensure(pl.max_tiles);
  w.qsplit.ensure((size_t)B * 2 * d);
  w.blk.ensure(kStatBytes + result_bytes);
  w.h_blk.ensure(kStatBytes + result_bytes);
  w.part_count.ensure(B);
  w.part_dist.ensure((size_t)B * pl.cap * rd::kTopK);
  w.part_row.ensure((size_t)B * pl.cap * rd::kTopK);


  cudaEvent_t* te = h->next_timing_slot();
  cudaEvent_t e0 = te[0], e1 = te[1], e2 = te[2], e3 = h->ev[3], e_plan = h->ev[4], e_off = h->ev[5];
  unsigned long long launches = 0;
  CK(cudaEventRecord(e0, s));
  // ||q||^2 and the query split (the tensor-core scan's operand) in one pass
  CK(rd::launch_qprep(d_q, B, d, w.qnorm.p, d % 64 == 0 ? w.qsplit.p : nullptr, w.fails(), w.part_count.p, s));
  if (rd::coarse_small((int)B)) {
    CK(rd::launch_coarse_small(d_q, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, h->num_sms, s));
  } else if (d % 64 == 0) {
    const CUtensorMap qmap = make_split_map(w.qsplit.p, B, d);
    CK(rd::launch_coarse_tc(qmap, h->cmap, h->cnorm.p, w.Dc.p, (int)B, nl, d, s));
  } else {
    CK(rd::launch_coarse(d_q, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, s));
  }
  w.qthr.ensure(B);
  const bool seed = B <= h->seed_max_b;
  if (!seed) CK(cudaMemsetAsync(w.qthr.p, 0x7f, sizeof(int) * B, s));  // no threshold: huge
  rd::SelectParams sp{w.Dc.p, d_q, w.qnorm.p, h->centroids.p, w.probes.p, w.fails(), (int)B, nl, nprobe, d, h->cmax,
                      h->d_list_off.p, h->d_res_row0.p, h->arena.p, h->xmax, seed ? w.qthr.p : nullptr, 0};
  h->traced("select", s, sp.dbg, [&] { CK(rd::launch_select(sp, h->stage_rows(B), s)); });
  launches += 3;
  rd::PlanParams pp{w.probes.p, w.bitmap.p, W, h->d_list_off.p, h->d_res_row0.p, w.list_nq.p, w.list_qoff.p,
                    w.list_ntile.p, w.list_toff.p, w.list_q.p, w.tiles.p, w.ff_tiles.p, w.meta(), w.counters(),
                    (int)B, nl, nprobe, pl.R, h->tc_scan() ? h->tc_min_q : 1 << 30};
  h->traced("plan", s, pp.dbg, [&] { CK(rd::launch_plan(pp, s)); });
  launches += rd::plan_small_ok((int)B, nprobe) || rd::plan_fused_ok((int)B, nl) ? 1 : 4;
  if (!h->no_inner_events) CK(cudaEventRecord(e1, s));

  const bool has_off = h->slots > 0;
  if (has_off) {  // fetch the probe histogram for host-side staging decisions
    w.h_nq.ensure(nl);
    w.h_qoff.ensure(nl);
    CK(cudaMemcpyAsync(w.h_nq.p, w.list_nq.p, sizeof(int) * nl, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(w.h_qoff.p, w.list_qoff.p, sizeof(int) * nl, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaEventRecord(e_plan, s));
  const CUtensorMap gmap = make_gather_map(w.qsplit.p, B, d);
  rd::ScanParams sc{w.ff_tiles.p, w.meta() + 2, w.meta() + 3, d_q, w.qnorm.p, w.list_q.p, h->xnorm.p,
                    w.part_dist.p, w.part_row.p, w.part_count.p, pl.cap, d, w.qthr.p};
  rd::TcScanParams tc{w.tiles.p, w.meta(), w.meta() + 1, w.qsplit.p, w.qnorm.p, w.list_q.p, h->xnorm.p,
                      w.part_dist.p, w.part_row.p, w.part_count.p, pl.cap, d, w.qthr.p, h->debug_skip};
  if (!h->tc_scan() || h->tc_min_q > 1) {  // FFMA tiles exist only in these cases
    CK(rd::launch_scan(h->map256, h->map32, sc, h->num_sms, s));
    launches += 1;
  }
  if (h->tc_scan()) {  // otherwise every tile is FFMA
    if (h->dbg_ts) {  // profiling only: per-CTA entry / ready / first tile / end times
      if (h->dbg_scan.n < 4 * (size_t)h->num_sms) h->dbg_scan.alloc(4 * (size_t)h->num_sms);
      CK(cudaMemsetAsync(h->dbg_scan.p, 0, 8 * 4 * (size_t)h->num_sms, s));
      tc.dbg = h->dbg_scan.p;
    }
    CK(rd::launch_scan_tc(h->presplit ? h->xmap128 : h->map128, h->presplit ? h->xmap32 : h->map32, gmap, tc,
                          h->num_sms, s, h->presplit));
    launches += 1;
    if (h->dbg_ts) {
      std::vector<unsigned long long> t(4 * (size_t)h->num_sms);
      CK(cudaMemcpyAsync(t.data(), h->dbg_scan.p, 8 * t.size(), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      unsigned long long t0 = ~0ull, mx[4] = {0, 0, 0, 0};
      for (int c = 0; c < h->num_sms; ++c) t0 = std::min(t0, t[4 * c]);
      double mean[4] = {0, 0, 0, 0};
      for (int c = 0; c < h->num_sms; ++c)
        for (int j = 0; j < 4; ++j) {
          const unsigned long long v = t[4 * c + j] ? t[4 * c + j] - t0 : 0;
          mx[j] = std::max(mx[j], v);
          mean[j] += (double)v / h->num_sms;
        }
      fprintf(stderr, "scan ns from first CTA entry: entry mean %.0f max %llu | ready mean %.0f max %llu | "
              "first tile mean %.0f max %llu | end mean %.0f max %llu\n", mean[0], mx[0], mean[1], mx[1], mean[2],
              mx[2], mean[3], mx[3]);
    }
  }
  if (!h->no_inner_events) CK(cudaEventRecord(e2, s));

  unsigned long long h2d = 0;
  if (has_off) {
    CK(cudaEventSynchronize(e_plan));
    // offloaded, probed lists in ascending id, packed into staging slots
    std::vector<std::vector<int>> batches;
    long long fill = 0;
    for (int l = 0; l < nl; ++l) {
      if (h->resident[l] || w.h_nq.p[l] == 0) continue;
      const long long len = h->list_off[l + 1] - h->list_off[l];
      if (len == 0) continue;
      if (batches.empty() || fill + len > h->slot_rows) {
        batches.emplace_back();
        fill = 0;
      }
      batches.back().push_back(l);
      fill += len;
    }
    // host-planned tiles of every batch (tensor-core and FFMA groups), uploaded once
    const size_t nb = batches.size();
    std::vector<rd::ScanTile> tv;  // per batch: [tc tiles][ff tiles]
    std::vector<int> tstart(nb + 1, 0), ntc(nb, 0);
    for (size_t bi = 0; bi < nb; ++bi) {
      tstart[bi] = (int)tv.size();
      std::vector<rd::ScanTile> ff;
      long long srow = (long long)(bi % h->slots) * h->slot_rows;
      for (int l : batches[bi]) {
        const long long len = h->list_off[l + 1] - h->list_off[l];
        const int nq = w.h_nq.p[l];
        const bool tcl = nq >= h->tc_min_q && h->tc_scan();
        const int ngr = tcl ? (nq + rd::kTcG - 1) / rd::kTcG : (nq + rd::kScanG - 1) / rd::kScanG;
        for (long long c = 0; c * pl.R < len; ++c)
          for (int g = 0; g < ngr; ++g) {
            rd::ScanTile T;
            T.src_row = srow + c * pl.R;
            T.grow0 = h->list_off[l] + c * pl.R;
            T.list = l;
            T.nrows = (int)std::min<long long>(pl.R, len - c * pl.R);
            if (tcl) {
              const int q0 = (int)((long long)g * nq / ngr), q1 = (int)((long long)(g + 1) * nq / ngr);
              T.qoff = w.h_qoff.p[l] + q0;
              T.nq = q1 - q0;
              tv.push_back(T);
            } else {
              T.qoff = w.h_qoff.p[l] + g * rd::kScanG;
              T.nq = std::min(rd::kScanG, nq - g * rd::kScanG);
              ff.push_back(T);
            }
          }
        srow += len;
      }
      ntc[bi] = (int)tv.size() - tstart[bi];
      tv.insert(tv.end(), ff.begin(), ff.end());
    }
    tstart[nb] = (int)tv.size();
    if (nb) {
      w.h_tiles.ensure(tv.size());
      std::memcpy(w.h_tiles.p, tv.data(), sizeof(rd::ScanTile) * tv.size());
      w.off_tiles.ensure(tv.size());
      w.h_meta.ensure(4 * nb);
      for (size_t bi = 0; bi < nb; ++bi) {
        w.h_meta.p[4 * bi + 0] = ntc[bi];
        w.h_meta.p[4 * bi + 1] = 0;
        w.h_meta.p[4 * bi + 2] = tstart[bi + 1] - tstart[bi] - ntc[bi];
        w.h_meta.p[4 * bi + 3] = 0;
      }
      DBuf<int>& dmeta = w.off_meta;
      dmeta.ensure(4 * nb);
      CK(cudaStreamWaitEvent(h->off_stream, e_plan, 0));
      CK(cudaMemcpyAsync(w.off_tiles.p, w.h_tiles.p, sizeof(rd::ScanTile) * tv.size(), cudaMemcpyHostToDevice,
                         h->off_stream));
      CK(cudaMemcpyAsync(dmeta.p, w.h_meta.p, sizeof(int) * 4 * nb, cudaMemcpyHostToDevice, h->off_stream));
      CK(cudaEventRecord(e3, h->off_stream));
      CK(cudaStreamWaitEvent(h->copy_stream, e_plan, 0));
      for (size_t bi = 0; bi < nb; ++bi) {
        const int slot = (int)(bi % h->slots);
        if (bi >= (size_t)h->slots) CK(cudaStreamWaitEvent(h->copy_stream, h->slot_done[slot], 0));
        long long srow = (long long)slot * h->slot_rows;
        for (int l : batches[bi]) {
          const long long len = h->list_off[l + 1] - h->list_off[l];
          const size_t bytes = (size_t)len * d * sizeof(float);
          CK(cudaMemcpyAsync(h->staging.p + (size_t)srow * d, h->host_arena.p + (size_t)h->host_row0[l] * d, bytes,
                             cudaMemcpyHostToDevice, h->copy_stream));
          h2d += bytes;
          srow += len;
        }
        CK(cudaEventRecord(h->slot_ready[slot], h->copy_stream));
        CK(cudaStreamWaitEvent(h->off_stream, h->slot_ready[slot], 0));
        const int nt_tc = ntc[bi], nt_ff = tstart[bi + 1] - tstart[bi] - ntc[bi];
        if (nt_ff) {
          rd::ScanParams so = sc;
          so.tiles = w.off_tiles.p + tstart[bi] + nt_tc;
          so.ntiles = dmeta.p + 4 * bi + 2;
          so.tile_counter = dmeta.p + 4 * bi + 3;
          CK(rd::launch_scan(h->smap256, h->smap32, so, std::min(h->num_sms, nt_ff), h->off_stream));
          launches += 1;
        }
        if (nt_tc) {
          rd::TcScanParams to = tc;
          to.tiles = w.off_tiles.p + tstart[bi];
          to.ntiles = dmeta.p + 4 * bi + 0;
          to.tile_counter = dmeta.p + 4 * bi + 1;
          CK(rd::launch_scan_tc(h->smap128, h->smap32, gmap, to, std::min(h->num_sms, nt_tc), h->off_stream, false));
          launches += 1;
        }
        CK(cudaEventRecord(h->slot_done[slot], h->off_stream));
      }
    }
    CK(cudaEventRecord(e_off, h->off_stream));
    CK(cudaStreamWaitEvent(s, e_off, 0));
  }

  if (!w.fb_ctr.p) {  // the fallback kernel's completion counter: zeroed once, re-armed by the kernel
    w.fb_ctr.alloc(1);
    CK(cudaMemset(w.fb_ctr.p, 0, sizeof(unsigned)));
  }
  w.fail_list.ensure(B);
  w.fb_dist.ensure((size_t)B * nprobe * rd::kTopK);
  w.fb_id.ensure((size_t)B * nprobe * rd::kTopK);
  rd::MergeParams mp{w.part_dist.p, w.part_row.p, w.part_count.p, pl.cap, d_q, w.qnorm.p, h->d_list_off.p,
                     h->d_list_base.p, h->d_ids.p, h->d_row_list.p, h->arena.p,
                     h->arena.p + (size_t)h->n_resident * d, nl, d, k, h->xmax, d_ids, d_dists,
                     w.fails() + 1, w.fail_list.p, (int)B};
  h->traced("merge", s, mp.dbg, [&] { CK(rd::launch_merge(mp, h->stage_rows(B), s)); });
  rd::FallbackParams fp{w.fail_list.p, w.fails() + 1, w.probes.p, nprobe, d_q, h->d_list_off.p, h->d_list_base.p,
                        h->d_ids.p, nl, d, k, w.fb_dist.p, w.fb_id.p, d_ids, d_dists, w.fb_ctr.p};
  CK(rd::launch_fallback(fp, h->num_sms, s));
  launches += 2;
  CK(cudaEventRecord(te[3], s));
  if (st) {
    std::memset(st, 0, sizeof *st);
    st->kernel_launches = launches;
  }
  if (before_sync) before_sync();  // e.g. the host path's result copies, ordered before the one sync
  if (sync) {
    // counters (and, on the host path, the results placed after them) in one copy
    CK(cudaMemcpyAsync(w.h_blk.p, w.blk.p, kStatBytes + result_bytes, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const auto* hc = reinterpret_cast<const unsigned long long*>(w.h_blk.p);
    const auto* hf = reinterpret_cast<const unsigned*>(w.h_blk.p + 24);
    const auto* hm = reinterpret_cast<const int*>(w.h_blk.p + 32);
    if (st) {
      float ms = 0;
      const unsigned long long row_bytes = (unsigned long long)d * 4;
      st->lists_probed = hc[0];
      st->bytes_lists_resident = hc[1] * row_bytes;
      st->h2d_list_bytes = h2d;
      st->bytes_algorithmic = (hc[1] + hc[2]) * row_bytes + (unsigned long long)nl * row_bytes +
                              (unsigned long long)B * row_bytes + (unsigned long long)B * k * 12ull;
      st->tiles = (uint64_t)hm[0] + (uint64_t)hm[2];
      if (!h->no_inner_events) {
        CK(cudaEventElapsedTime(&ms, e1, e2));
        st->scan_ms = ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        st->coarse_ms = ms;
      }
      if (has_off) {
        CK(cudaEventElapsedTime(&ms, e_plan, e_off));
        st->offload_ms = ms;
      }
      st->probe_failures = hf[0];
      st->margin_failures = hf[1];
    }
  }
}

}  // namespace

namespace {
// Largest batch searched in one pass: bounds the B x nlist coarse-distance workspace (2 GiB).
long long search_chunk(const rd_index* h) {
  return std::max<long long>(1024, std::min<long long>(65536, (1LL << 31) / (4LL * h->nlist)));
}
void add_stats(rd_search_stats* acc, const rd_search_stats& s) {  // counters summed over chunks
  acc->bytes_algorithmic += s.bytes_algorithmic;
  acc->bytes_lists_resident += s.bytes_lists_resident;
  acc->h2d_list_bytes += s.h2d_list_bytes;
  acc->lists_probed += s.lists_probed;
  acc->tiles += s.tiles;
  acc->kernel_launches += s.kernel_launches;
  acc->scan_ms += s.scan_ms;
  acc->coarse_ms += s.coarse_ms;
  acc->offload_ms += s.offload_ms;
  acc->margin_failures += s.margin_failures;
  acc->probe_failures += s.probe_failures;
}
}  // namespace

int rd_search_device(rd_index* h, const float* d_q, int64_t B, int32_t nprobe, int32_t k, int64_t* d_ids,
                     float* d_dists, void* stream, int32_t sync, rd_search_stats* st) {
  return guarded([&] {
    if (!h || B < 0 || (B > 0 && (!d_q || !d_ids || !d_dists))) throw_rd(RD_ERR_INVALID, "search: invalid arguments");
    if (st) std::memset(st, 0, sizeof *st);
    if (B == 0) return;
    const auto t0 = std::chrono::steady_clock::now();
    const long long chunk = search_chunk(h);
    for (long long b0 = 0; b0 < B; b0 += chunk) {  // very large batches run as consecutive passes
      const long long nb = std::min<long long>(chunk, B - b0);
      rd_search_stats part{};
      do_search(h, d_q + (size_t)b0 * h->d, nb, nprobe, k, reinterpret_cast<long long*>(d_ids) + (size_t)b0 * k,
                d_dists + (size_t)b0 * k, (cudaStream_t)stream, sync != 0, st ? &part : nullptr);
      if (st) add_stats(st, part);
    }
    if (st) st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int rd_search(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t k, int64_t* out_ids,
              float* out_dists, rd_search_stats* st) {
  if (h && B > search_chunk(h) && queries && out_ids && out_dists && h->d > 0 && k > 0) {
    // very large batches: consecutive passes of the one-pass path below
    const auto t0 = std::chrono::steady_clock::now();
    rd_search_stats acc{};
    const long long chunk = search_chunk(h);
    for (long long b0 = 0; b0 < B; b0 += chunk) {
      rd_search_stats part{};
      const int rc = rd_search(h, queries + (size_t)b0 * h->d, std::min<long long>(chunk, B - b0), nprobe, k,
                               out_ids + (size_t)b0 * k, out_dists + (size_t)b0 * k, &part);
      if (rc != RD_OK) return rc;
      add_stats(&acc, part);
    }
    acc.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (st) *st = acc;
    return RD_OK;
  }
  return guarded([&] {
    if (!h || B < 0 || (B > 0 && (!queries || !out_ids || !out_dists)))
      throw_rd(RD_ERR_INVALID, "search: invalid arguments");
    if (nprobe < 1 || k < 1) throw_rd(RD_ERR_INVALID, "search: nprobe >= 1 and k >= 1 required");
    const auto t0 = std::chrono::steady_clock::now();
    if (B == 0) {
      if (st) std::memset(st, 0, sizeof *st);
      return;
    }
    CK(cudaSetDevice(h->device));
    auto& w = h->ws;
    const size_t qn = (size_t)B * h->d, rn = (size_t)B * k;
    w.q.ensure(qn);
    // caller buffers that are already page-locked are copied directly; others go through the
    // handle's pinned staging buffers
    auto pinned = [](const void* ptr) {
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      return a.type == cudaMemoryTypeHost;
    };
    const bool pq = pinned(queries), pi = pinned(out_ids), pd = pinned(out_dists);
    const float* qsrc = queries;
    if (!pq) {
      w.hq.ensure(qn);
      std::memcpy(w.hq.p, queries, qn * sizeof(float));
      qsrc = w.hq.p;
    }
    cudaStream_t s = 0;
    CK(cudaMemcpyAsync(w.q.p, qsrc, qn * sizeof(float), cudaMemcpyHostToDevice, s));
    // results live right after the stat block: pinned caller buffers get direct copies, otherwise
    // stats and results come back in the sync's single copy
    const bool direct = pi && pd;
    const size_t res_bytes = rn * (sizeof(long long) + sizeof(float));
    w.blk.ensure(kStatBytes + res_bytes);
    long long* d_ids = reinterpret_cast<long long*>(w.blk.p + kStatBytes);
    float* d_dists = reinterpret_cast<float*>(w.blk.p + kStatBytes + rn * sizeof(long long));
    do_search(h, w.q.p, B, nprobe, k, d_ids, d_dists, s, true, st, direct ? 0 : res_bytes, [&] {
      if (!direct) return;
      CK(cudaMemcpyAsync(out_ids, d_ids, rn * sizeof(long long), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(out_dists, d_dists, rn * sizeof(float), cudaMemcpyDeviceToHost, s));
    });
    if (!direct) {
      std::memcpy(out_ids, w.h_blk.p + kStatBytes, rn * sizeof(long long));
      std::memcpy(out_dists, w.h_blk.p + kStatBytes + rn * sizeof(long long), rn * sizeof(float));
    }
    if (st) st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int rd_probe(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t* out_lists) {
  return guarded([&] {
    if (!h || B < 0 || (B > 0 && (!queries || !out_lists))) throw_rd(RD_ERR_INVALID, "probe: invalid arguments");
    if (nprobe < 1 || std::min(nprobe, h->nlist) + rd::kCoarseExtra > 512)
      throw_rd(RD_ERR_INVALID, "probe: 1 <= nprobe <= 480 required");
    if (B == 0) return;
    CK(cudaSetDevice(h->device));
    auto& w = h->ws;
    const int nl = h->nlist, d = h->d;
    w.q.ensure((size_t)B * d);
    w.qnorm.ensure(B);
    w.Dc.ensure((size_t)B * nl);
    w.probes.ensure((size_t)B * nprobe);
    w.blk.ensure(kStatBytes);
    CK(cudaMemcpy(w.q.p, queries, sizeof(float) * B * d, cudaMemcpyHostToDevice));
    CK(cudaMemset(w.fails(), 0, 2 * sizeof(unsigned)));
    w.qsplit.ensure((size_t)B * d);
    CK(rd::launch_qprep(w.q.p, B, d, w.qnorm.p, d % 64 == 0 ? w.qsplit.p : nullptr, nullptr, nullptr, 0));
    if (rd::coarse_small((int)B)) {
      CK(rd::launch_coarse_small(w.q.p, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, h->num_sms, 0));
    } else if (d % 64 == 0) {
      const CUtensorMap qmap = make_split_map(w.qsplit.p, B, d);
      CK(rd::launch_coarse_tc(qmap, h->cmap, h->cnorm.p, w.Dc.p, (int)B, nl, d, 0));
    } else {
      CK(rd::launch_coarse(w.q.p, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, 0));
    }
    rd::SelectParams sp{w.Dc.p, w.q.p, w.qnorm.p, h->centroids.p, w.probes.p, w.fails(), (int)B, nl, nprobe, d, h->cmax,
                        h->d_list_off.p, h->d_res_row0.p, h->arena.p, h->xmax, nullptr, 1};
    CK(rd::launch_select(sp, h->stage_rows(B), 0));
    CK(cudaMemcpy(out_lists, w.probes.p, sizeof(int) * B * nprobe, cudaMemcpyDeviceToHost));
  });
}

int rd_timing_reset(rd_index* h) {
  return guarded([&] {
    if (!h) throw_rd(RD_ERR_INVALID, "null index");
    CK(cudaSetDevice(h->device));
    while (h->t_accounted < h->t_recorded) {  // drain so the ring's events are free again
      CK(cudaEventSynchronize(h->tev[h->t_accounted % rd_index::kRing][3]));
      ++h->t_accounted;
    }
    h->t_acc = rd_timing{};
  });
}

int rd_timing_read(rd_index* h, rd_timing* out) {
  return guarded([&] {
    if (!h || !out) throw_rd(RD_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    while (h->t_accounted < h->t_recorded) h->account(h->t_accounted++);
    *out = h->t_acc;
  });
}

// ---------------------------------------------------------------- shard merge
int rd_merge_topk(int32_t G, int64_t B, int32_t k, const int64_t* sid, const float* sd, int64_t* oid, float* od) {
  return guarded([&] {
    if (G < 1 || B < 0 || k < 1 || (B > 0 && (!sid || !sd || !oid || !od)))
      throw_rd(RD_ERR_INVALID, "merge: invalid arguments");
    std::vector<std::pair<float, int64_t>> c;
    for (int64_t q = 0; q < B; ++q) {
      c.clear();
      for (int g = 0; g < G; ++g)
        for (int i = 0; i < k; ++i) {
          const size_t o = ((size_t)g * B + q) * k + i;
          if (sid[o] >= 0) c.emplace_back(sd[o], sid[o]);
        }
      const size_t m = std::min<size_t>(k, c.size());
      std::partial_sort(c.begin(), c.begin() + m, c.end());
      for (int i = 0; i < k; ++i) {
        oid[q * k + i] = (size_t)i < m ? c[i].second : -1;
        od[q * k + i] = (size_t)i < m ? c[i].first : INFINITY;
      }
    }
  });
}

int rd_merge_topk_device(int32_t G, int64_t B, int32_t k, const int64_t* ids, const float* dists, int64_t* oid,
                         float* od, void* stream) {
  return guarded([&] {
    if (G < 1 || B < 0 || k < 1 || k > 32) throw_rd(RD_ERR_INVALID, "merge_device: invalid arguments (k <= 32)");
    CK(rd::launch_shard_merge(G, B, k, reinterpret_cast<const long long*>(ids), dists,
                              reinterpret_cast<long long*>(oid), od, (cudaStream_t)stream));
  });
}

// ---------------------------------------------------------------- placement arithmetic
int rd_llm_reservation_bytes(const rd_llm_reservation* r, double* out) {
  return guarded([&] {
    if (!r || !out) throw_rd(RD_ERR_INVALID, "null argument");
    if (r->gen_batch_size < 0 || r->w_gpu < 0 || r->w_gpu > 1 || r->c_gpu < 0 || r->c_gpu > 1)
      throw_rd(RD_ERR_INVALID, "reservation: fractions in [0,1] and batch >= 0 required");
    const double W = (double)r->weight_total;
    const double C = (double)r->kv_bytes_per_request * r->gen_batch_size;
    double H = (double)r->workspace_bytes_per_request * r->gen_batch_size;
    if (r->decode_phase) H *= r->workspace_fraction;
    *out = r->w_gpu * W + r->c_gpu * C + H;
  });
}

int32_t rd_staging_depth(double free_bytes, double item_bytes) {
  if (item_bytes <= 0) return 1;
  const double q = std::floor(free_bytes / item_bytes);
  if (q < 1) return 1;
  if (q > (double)(1 << 20)) return 1 << 20;
  return (int32_t)q;
}

}  // extern "C"
