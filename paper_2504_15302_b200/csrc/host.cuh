// host.cuh — host-side core of the B200 retrieval engine behind include/rd.h: error model,
// device / pinned buffers, TMA tensor maps, and the index object (index.cu: lifecycle,
// placement, migration, files, training; search.cu: the search itself).
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
#pragma once
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
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/rd.h"
#include "../../include/rd_format.h"
#include "ivf_kernels.cuh"
#include "rd_device.cuh"

// message of the last failure on this thread (rd_last_error), defined in index.cu
extern thread_local std::string g_err;

namespace {

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

// ------------------------------------------------------------------ growable device arenas (CUDA VMM)
// Driver entry points of the virtual memory management API, bound at run time like the tensor-map
// encoder (no link-time libcuda dependency).
struct VmmApi {
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) free_range = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
};
const VmmApi& vmm() {
  static VmmApi api = [] {
    VmmApi a;
    auto get = [](const char* name) {
      void* ptr = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        ptr = nullptr;
      return ptr;
    };
    a.reserve = reinterpret_cast<decltype(a.reserve)>(get("cuMemAddressReserve"));
    a.free_range = reinterpret_cast<decltype(a.free_range)>(get("cuMemAddressFree"));
    a.create = reinterpret_cast<decltype(a.create)>(get("cuMemCreate"));
    a.release = reinterpret_cast<decltype(a.release)>(get("cuMemRelease"));
    a.map = reinterpret_cast<decltype(a.map)>(get("cuMemMap"));
    a.unmap = reinterpret_cast<decltype(a.unmap)>(get("cuMemUnmap"));
    a.set_access = reinterpret_cast<decltype(a.set_access)>(get("cuMemSetAccess"));
    a.granularity = reinterpret_cast<decltype(a.granularity)>(get("cuMemGetAllocationGranularity"));
    return a;
  }();
  if (!api.reserve || !api.create || !api.map || !api.unmap || !api.set_access || !api.granularity || !api.release ||
      !api.free_range)
    throw_rd(RD_ERR_RUNTIME, "CUDA virtual memory management entry points unavailable");
  return api;
}
#define CUK(x)                                                                                  \
  do {                                                                                          \
    CUresult r_ = (x);                                                                          \
    if (r_ != CUDA_SUCCESS) throw_rd(RD_ERR_RUNTIME, "%s failed (%d) (%s:%d)", #x, (int)r_, __FILE__, __LINE__); \
  } while (0)

// A device arena over one reserved virtual range, backed by physical memory in fixed-size chunks
// mapped on demand (CUDA VMM): resize() grows or shrinks the usable prefix in place and map_range()
// backs any window, so a relayout never holds two copies of the rows (format conversions run
// tail-first: the destination's tail is mapped as the source's tail is released), the base pointer
// — and every TMA map encoded over it — stays valid, and the HBM held is what is mapped.
// n = elements usable (the resident store's rows x row elements).
template <class T>
struct VArena {
  T* p = nullptr;
  size_t n = 0;            // elements usable
  size_t cap = 0;          // elements the reserved range can hold
  size_t chunk = 0;        // bytes per physical chunk
  int device = -1;
  std::vector<CUmemGenericAllocationHandle> h;  // per chunk of the range
  std::vector<uint8_t> on;                      // chunk mapped
  VArena() = default;
  VArena(const VArena&) = delete;
  VArena& operator=(const VArena&) = delete;
  ~VArena() { reset(); }
  size_t mapped_bytes() const {
    size_t c = 0;
    for (uint8_t b : on) c += b;
    return c * chunk;
  }
  void unmap_chunk(size_t i) {
    const auto& v = vmm();
    CUK(v.unmap(reinterpret_cast<CUdeviceptr>(p) + i * chunk, chunk));
    CUK(v.release(h[i]));
    on[i] = 0;
  }
  void reset() {
    if (!p) return;
    const auto& v = vmm();
    for (size_t i = 0; i < on.size(); ++i)
      if (on[i]) {
        v.unmap(reinterpret_cast<CUdeviceptr>(p) + i * chunk, chunk);
        v.release(h[i]);
      }
    v.free_range(reinterpret_cast<CUdeviceptr>(p), on.size() * chunk);
    h.clear();
    on.clear();
    p = nullptr;
    n = cap = 0;
  }
  // reserves room for `capacity` elements on the current device (contents dropped); chunks hold whole
  // rows of row_elems elements, so no row (one TMA box row, one bulk copy) spans two physical
  // allocations
  void reserve(size_t capacity, size_t row_elems = 1) {
    reset();
    const auto& v = vmm();
    CK(cudaGetDevice(&device));
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    size_t gran = 0;
    CUK(v.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    if (!gran) gran = size_t(2) << 20;
    const size_t bytes = std::max<size_t>(1, capacity) * sizeof(T);
    // chunks of at most 64 MiB (the most a store holds beyond its rows), at least one granule,
    // ~1/512 of the range for large arenas
    const size_t rb = std::max<size_t>(1, row_elems) * sizeof(T);
    size_t g = gran, r = rb;  // unit = lcm(granule, row bytes)
    while (r) {
      const size_t t = g % r;
      g = r;
      r = t;
    }
    const size_t unit = gran / g * rb;
    chunk = std::min<size_t>(std::max<size_t>(size_t(64) << 20, unit), std::max(unit, bytes / 512));
    chunk = (chunk + unit - 1) / unit * unit;
    const size_t nchunks = (bytes + chunk - 1) / chunk;
    CUdeviceptr base = 0;
    CUK(v.reserve(&base, nchunks * chunk, 0, 0, 0));  // default alignment (chunk need not be a power of two)
    p = reinterpret_cast<T*>(base);
    cap = nchunks * chunk / sizeof(T);
    h.assign(nchunks, 0);
    on.assign(nchunks, 0);
    n = 0;
  }
  // backs elements [lo, hi) with physical memory (chunks already mapped are kept)
  void map_range(size_t lo, size_t hi) {
    if (hi > cap) throw_rd(RD_ERR_RUNTIME, "arena window beyond its reservation (%zu > %zu)", hi, cap);
    if (hi <= lo) return;
    const auto& v = vmm();
    const CUdeviceptr base = reinterpret_cast<CUdeviceptr>(p);
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    const size_t c0 = lo * sizeof(T) / chunk, c1 = (hi * sizeof(T) + chunk - 1) / chunk;
    for (size_t i = c0; i < c1; ++i) {
      if (on[i]) continue;
      const CUresult r = v.create(&h[i], chunk, &prop, 0);
      if (r != CUDA_SUCCESS)
        throw_rd(RD_ERR_RUNTIME, "device memory exhausted backing an arena window of %zu bytes (cuMemCreate %d)",
                 (hi - lo) * sizeof(T), (int)r);
      const CUresult m = v.map(base + i * chunk, chunk, 0, h[i], 0);
      if (m != CUDA_SUCCESS) {
        v.release(h[i]);
        throw_rd(RD_ERR_RUNTIME, "cuMemMap failed (%d)", (int)m);
      }
      on[i] = 1;
      CUK(v.set_access(base + i * chunk, chunk, &acc, 1));
    }
  }
  // releases every chunk that lies wholly at or beyond element `from`
  void unmap_from(size_t from) {
    const size_t c0 = (from * sizeof(T) + chunk - 1) / chunk;
    for (size_t i = c0; i < on.size(); ++i)
      if (on[i]) unmap_chunk(i);
  }
  // `count` usable elements from the start: contents below min(old, new) kept
  void resize(size_t count) {
    if (count > cap) throw_rd(RD_ERR_RUNTIME, "arena resize beyond its reservation (%zu > %zu)", count, cap);
    unmap_from(count);
    map_range(0, count);
    n = count;
  }
  // reserve(capacity) + resize(count): a fresh arena of `count` usable elements
  void alloc(size_t count, size_t capacity = 0) {
    reserve(std::max(count, capacity));
    resize(count);
  }
};

// ------------------------------------------------------------------ stream memory operations
// cuStreamWaitValue32 / cuStreamWriteValue32 (driver API, bound at run time): an asynchronous search
// with offloaded lists gates the caller's stream on a device word that a host worker releases once
// it has enqueued the offloaded part (search.cu).
struct StreamMemApi {
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
};
const StreamMemApi& stream_mem() {
  static StreamMemApi api = [] {
    StreamMemApi a;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      a.wait32 = reinterpret_cast<decltype(a.wait32)>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      a.write32 = reinterpret_cast<decltype(a.write32)>(p);
    return a;
  }();
  return api;
}

// One host thread that runs posted jobs one at a time (an asynchronous search's offloaded part).
// wait() blocks until the last job finished and rethrows its error.
class TailWorker {
 public:
  TailWorker() : th_([this] { loop(); }) {}
  ~TailWorker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void post(std::function<void()> f) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !busy_; });
    job_ = std::move(f);
    busy_ = true;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !busy_; });
    if (err_) {
      std::exception_ptr e = err_;
      err_ = nullptr;
      std::rethrow_exception(e);
    }
  }

 private:
  void loop() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return quit_ || (busy_ && job_); });
      if (quit_ && !busy_) return;
      auto f = std::move(job_);
      job_ = nullptr;
      lk.unlock();
      std::exception_ptr e;
      try {
        f();
      } catch (...) {
        e = std::current_exception();
      }
      lk.lock();
      if (e && !err_) err_ = e;
      busy_ = false;
      cv_.notify_all();
      if (quit_) return;
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::function<void()> job_;
  bool busy_ = false, quit_ = false;
  std::exception_ptr err_;
  std::thread th_;
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

// 2D bf16 map over a [rows][d] plane (the residual store's r1), box {64 dims, box_rows}, 128B swizzle:
// the same smem tile as one part of the split map's box.
CUtensorMap make_bf16_row_map(const void* base, long long rows, int d, int box_rows, bool fp16 = false) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  if (rows < 1) rows = 1;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw_rd(RD_ERR_RUNTIME, "cuTensorMapEncodeTiled (16-bit rows) failed (%d)", (int)r);
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
  // profiling only: checkpoints of every kernel of one search, taken without serialising the chain
  bool dbg_chain = std::getenv("RD_DEBUG_CHAIN") != nullptr;
  int stage_max_b = -1;  // batches up to this size stage exact-distance rows in smem (-1: 2 x SMs)
  int tiles_per_sm = 0;  // scan tiles per SM the planner aims for (RD_TILES_PER_SM; 0 = by batch, make_plan)
  // rd_search_device with offloaded lists: return before the plan completes (a device gate released by
  // the worker thread) only with RD_ASYNC_TAIL=1 — a stream-memory wait can deadlock when the caller's
  // stream shares a hardware queue with the side streams (seen with a concurrent decode stream, C5)
  bool async_tail = std::getenv("RD_ASYNC_TAIL") && std::atoi(std::getenv("RD_ASYNC_TAIL")) == 1;
  bool fuse_plan = !(std::getenv("RD_FUSE_PLAN") && std::atoi(std::getenv("RD_FUSE_PLAN")) == 0);  // B = 1 plan in the selection
  // scan_pair.cu for wide tiles: opt-in (RD_PAIR=1) — measured 6 % slower at B = 1024
  bool pair_scan = std::getenv("RD_PAIR") && std::atoi(std::getenv("RD_PAIR")) == 1;
  long long seed_max_b = 1LL << 40;  // batches up to this size seed the scan's pruning threshold (RD_SEED_MAX_B)
  bool stage_events = false;  // rd_timing_stages: per-stage events between the chain's kernels
  // the tensor-core scan stages 64-dim bf16 query slices of up to 32 queries in shared memory:
  // d % 64 == 0 and d <= 896 (beyond, its B operand does not fit next to the x ring); else FFMA
  // the converter variant (offloaded lists, or no pre-split copy) must fit: its operand is resident
  bool tc_scan() const { return d % 64 == 0 && rd::scan_tc_smem_bytes(d, 32, false) <= 227 * 1024; }
  // dot-product error bound of the scans whose candidates the merge certifies (ivf_kernels.cuh): the
  // tensor-core and FFMA scans may both run in one search (offloaded or sparse lists)
  // (a search over the residual store passes 0 instead: its keys are lower bounds already, resid.cu)
  float scan_gamma_base() const {
    return tc_scan() ? std::max(rd::gamma_bf16x3(d), rd::gamma_ffma_scan(d)) : rd::gamma_ffma_scan(d);
  }
  // Tensor-core tile width for a batch: 16-query tiles (the 16-wide scan's deeper ring) when the
  // probed lists see <= 8 queries on average, else 32-query tiles (lists read once). Measured: mixing
  // both widths in one batch (RD_TC_G=1: lists of <= 16 queries narrow, others wide) does not beat
  // all-wide at B = 1024 and loses at short lists. RD_TC_G=16|32 forces one width.
  int tc_mode_for(long long B, int nprobe) const {
    if (tc_g_force == 16 || tc_g_force == 32) return tc_g_force;
    if (tc_g_force == 1) return 0;
    const double per_list = (double)B * std::min(nprobe, nlist) / std::max(1, nlist);
    return per_list <= 8.0 ? 16 : 32;
  }
  int tc_g_force = std::getenv("RD_TC_G") ? std::atoi(std::getenv("RD_TC_G")) : 0;
  // streamed query operand for the 16-query scan (scan_tc.cu): -1 by batch, RD_STREAM_B=0|1 forces
  int stream_force = std::getenv("RD_STREAM_B") ? std::atoi(std::getenv("RD_STREAM_B")) : -1;
  // spare candidates reranked beyond k (RD_RERANK_MARGIN, 8..32): more tolerate more duplicate
  // vectors around rank k before a query needs the exact fallback, at more rerank reads and a
  // looser scan pruning rank
  // (-1: by store — 14 over the residual store, whose keys sit up to eps_pair below the exact
  // distances, so rank k + 15 clears rank k's near-ties; 8 otherwise)
  int rerank_margin_env = std::getenv("RD_RERANK_MARGIN")
                              ? std::max(8, std::min(32, std::atoi(std::getenv("RD_RERANK_MARGIN"))))
                              : -1;
  // (fp16 residual scan from 512 queries: 21 — its slightly wider bound sent ~1 query in a few
  // thousand to the exact fallback at margin 14, which at B = 1024 costs more than the wider rerank:
  // +3-4 % measured; below 512 queries 14 is as fast or faster)
  int rerank_margin(bool res, bool res16, long long B) const {
    return rerank_margin_env >= 0 ? rerank_margin_env : res ? (res16 && B >= 512 ? 21 : 14) : 8;
  }
  bool stage_rows(long long B) const { return B <= (stage_max_b >= 0 ? stage_max_b : 2LL * num_sms); }
  long long n = 0;
  int d = 0, nlist = 0;
  std::vector<long long> list_off;  // host copy, nlist + 1
  long long max_len = 0;
  float cmax = 0.f, xmax = 0.f;

  DBuf<float> centroids, cnorm, xnorm;
  DBuf<float> csplit;  // nlist x 2 x d bf16 (c1, c2) for the tensor-core coarse GEMM
  CUtensorMap cmap{};
  // Resident store: the rows of the HBM-resident lists (a list's rows contiguous from res_row0), in
  // one of two formats:
  //  split3 (whenever the tensor-core scan applies and the split round-trips): the exact bf16 triple
  //    x = (x1 + x2) + x3 — xsplit [rows][2][d] (x1, x2), the scan's operand, and x3 [rows][d], read
  //    only by the exact rerank / fallback / seeding, which rebuild x bit for bit: 6 B per element;
  //  fp32: arena [rows][d] (the FFMA scan's input: d % 64 != 0, RD_SPLIT3=0, data whose split does
  //    not round-trip), plus, while no byte budget applies and memory allows, a pre-split xsplit copy
  //    for the conversion-free scan (8 B per element; RD_PRESPLIT=0 disables).
  // Every store is a VArena: relayouts grow and shrink it in place.
  bool split3 = false;
  VArena<float> arena;
  VArena<float> xsplit;  // 2 bf16 per float slot
  VArena<uint16_t> x3;
  CUtensorMap xmap128{}, xmap32{};
  bool presplit = false;
  // Residual store (RD_STORE=resid, resid.cu): the fp32 arena plus r1 = bf16(x - c_list) [rows][d]
  // (2 B per element: the scan's only operand), ||x - c||^2 per row and max ||x - c|| per list. Built
  // while every list is resident and no byte budget applies; any relayout drops it (build_presplit
  // rebuilds it).
  bool resid = false;
  DBuf<uint16_t> rplane;
  DBuf<float> rnorm, rmax;
  CUtensorMap rmap128{}, rmap32{};
  // RD_STORE=split3 keeps the round-2 stores (split3 / fp32 by budget) for fully resident indexes too
  static bool resid_wanted() {
    const char* v = std::getenv("RD_STORE");
    return !(v && std::strcmp(v, "split3") == 0);
  }
  bool resid_ok = true;  // the last placement chose the residual store (materialize: always)
  // the residual store applies: wanted, the tensor-core scan for every list, 128-dim pair-operand blocks
  bool resid_fmt() const { return resid_wanted() && tc_scan() && tc_min_q == 1 && d % 128 == 0; }
  void drop_resid() {
    resid = false;
    rplane.reset();
    rnorm.reset();
    rmax.reset();
  }
  // fp16 residual plane and fp16(q) operand (default; RD_RES16=0: bf16 plane with the (q1; q2) split)
  // unless a component leaves fp16's range
  bool res16 = false;
  static bool res16_wanted() {
    const char* v = std::getenv("RD_RES16");
    return !(v && std::atoi(v) == 0);
  }
  bool build_resid() {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const size_t need = (size_t)n * d * 2 + (size_t)n * 4 + (size_t)nlist * 4;
    if (need + (size_t(1) << 30) > fr) return false;
    rplane.alloc((size_t)n * d);
    rnorm.alloc(n);
    rmax.alloc(nlist);
    res16 = res16_wanted();
    if (res16) {
      DBuf<unsigned> ovf;
      ovf.alloc(1);
      CK(cudaMemset(ovf.p, 0, sizeof(unsigned)));
      CK(rd::launch_resid_build(arena.p, d_res_row0.p, d_list_off.p, centroids.p, nlist, d, rplane.p, rnorm.p,
                                rmax.p, 0, true, ovf.p));
      unsigned bad = 0;
      CK(cudaMemcpy(&bad, ovf.p, sizeof bad, cudaMemcpyDeviceToHost));
      res16 = bad == 0;
    }
    if (!res16)
      CK(rd::launch_resid_build(arena.p, d_res_row0.p, d_list_off.p, centroids.p, nlist, d, rplane.p, rnorm.p, rmax.p, 0));
    CK(cudaDeviceSynchronize());
    rmap128 = make_bf16_row_map(rplane.p, n_resident, d, rd::kTcRows, res16);
    rmap32 = make_bf16_row_map(rplane.p, n_resident, d, 32, res16);
    resid = true;
    return true;
  }
  DBuf<unsigned> inexact_ctr;  // split3_kernel's count of elements that did not round-trip
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
    DBuf<uint16_t> qhalf;  // fp16 residual scan: q as fp16 [B][d]
    DBuf<int> probes, list_nq, list_qoff, list_ntile, list_toff, list_q, part_count, part_row, off_meta;
    DBuf<unsigned> bitmap, fb_ctr;
    bool bitmap_clean = false;  // the bitmap is all-zero (the plan's list_fill re-zeroes it)
    DBuf<rd::ScanTile> tiles, tiles16, ff_tiles, off_tiles;  // wide / narrow tensor-core, FFMA, offloaded
    DBuf<float> part_dist;
    DBuf<long long> fb_id;
    DBuf<int> fail_list, qthr;
    DBuf<float> fb_dist;
    DBuf<char> sel_scratch;          // the all-centroid selection (large nprobe)
    DBuf<float> wide_d;              // the large-k pass: S x B x 32R per-split survivors
    DBuf<long long> wide_id;
    HBuf<int> h_nq, h_qoff, h_meta;
    // per-search counters in one block so a synced search reads them back with one copy:
    // [0, 24) counters (u64 x 3), [24, 32) fails (u32 x 2), [32, 56) meta (i32 x 6); the host path
    // places its result ids / distances right after (kStatBytes) and copies everything at once
    DBuf<char> blk;
    HBuf<char> h_blk;
    // (re)allocates the block; its unused padding is zeroed once so every byte the sync copy
    // brings back has been written
    void ensure_blk(size_t n) {
      if (blk.n >= n) return;
      blk.ensure(n);
      CK(cudaMemset(blk.p, 0, kStatBytes));
    }
    unsigned long long* counters() const { return reinterpret_cast<unsigned long long*>(blk.p); }
    unsigned* fails() const { return reinterpret_cast<unsigned*>(blk.p + 24); }
    int* meta() const { return reinterpret_cast<int*>(blk.p + 32); }
    HBuf<rd::ScanTile> h_tiles;
  } ws;

  // the search whose stat block copy do_search enqueued last (rdh::finish_stats reads it back)
  struct Pending {
    long long B = 0;
    int k = 0;
    unsigned long long h2d = 0, launches = 0;
    bool staged = false, has_off = false;
    cudaEvent_t e0{}, e1{}, e2{};
  } pend;

  cudaStream_t copy_stream = nullptr, off_stream = nullptr;
  cudaEvent_t ev[8] = {};
  // device-time accounting: 4 events per search (start, plan done, resident scan done, end)
  static constexpr int kRing = 64;
  cudaEvent_t tev[kRing][4] = {};
  bool tev_staged[kRing] = {};
  long long t_recorded = 0, t_accounted = 0;
  rd_timing t_acc{};

  void account(long long i) {  // fold search i's events into t_acc (synchronizes on them)
    cudaEvent_t* e = tev[i % kRing];
    CK(cudaEventSynchronize(e[3]));
    float a = 0, b = 0, c = 0, t = 0;
    if (tev_staged[i % kRing]) {
      t_acc.stage_searches += 1;
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
    tev_staged[t_recorded % kRing] = stage_events;
    return tev[t_recorded++ % kRing];
  }
  std::vector<cudaEvent_t> slot_ready, slot_done;

  // asynchronous searches with offloaded lists (search.cu): the caller's stream waits on gate >= seq
  // until the tail worker has enqueued the offloaded part and the merge
  DBuf<unsigned> gate;
  unsigned gate_seq = 0;
  std::unique_ptr<TailWorker> tailw;
  // every entry point that touches the index first lets a pending tail finish enqueueing
  void tail_wait() {
    if (tailw) tailw->wait();
  }

  ~rd_index() {
    if (tailw) {
      try {
        tailw->wait();
      } catch (...) {
      }
      tailw.reset();
    }
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

  // ---- the resident store (format-agnostic row operations; rows are resident-store rows)
  bool split3_eligible() const {
    const char* env = std::getenv("RD_SPLIT3");
    return tc_scan() && tc_min_q == 1 && !(env && std::atoi(env) == 0);
  }
  size_t res_row_bytes() const { return (size_t)d * (split3 ? 6 : 4); }
  void store_reserve(long long rows_cap) {  // capacity for rows_cap rows, contents dropped
    if (split3) {
      arena.reset();
      xsplit.reserve((size_t)std::max(1LL, rows_cap) * d, d);
      x3.reserve((size_t)std::max(1LL, rows_cap) * d, d);
    } else {
      xsplit.reset();
      x3.reset();
      arena.reserve((size_t)std::max(1LL, rows_cap) * d, d);
    }
  }
  void store_resize(long long rows) {
    if (split3) {
      xsplit.resize((size_t)rows * d);
      x3.resize((size_t)rows * d);
    } else {
      arena.resize((size_t)rows * d);
    }
  }
  uint64_t store_bytes() const { return arena.mapped_bytes() + xsplit.mapped_bytes() + x3.mapped_bytes(); }
  // fp32 device rows -> store rows [row0, row0 + rows)
  void store_put(long long row0, const float* src, long long rows, cudaStream_t s) {
    if (!rows) return;
    if (split3) {
      if (!inexact_ctr.p) {
        inexact_ctr.alloc(1);
        CK(cudaMemset(inexact_ctr.p, 0, sizeof(unsigned)));
      }
      CK(rd::launch_split3(src, rows, d, xsplit.p + (size_t)row0 * d, x3.p + (size_t)row0 * d, inexact_ctr.p, s));
    } else {
      CK(cudaMemcpyAsync(arena.p + (size_t)row0 * d, src, (size_t)rows * d * 4, cudaMemcpyDeviceToDevice, s));
    }
  }
  // store rows [row0, row0 + rows) -> fp32 device rows
  void store_get(long long row0, long long rows, float* dst, cudaStream_t s) const {
    if (!rows) return;
    if (split3)
      CK(rd::launch_join3(xsplit.p + (size_t)row0 * d, x3.p + (size_t)row0 * d, rows, d, dst, s));
    else
      CK(cudaMemcpyAsync(dst, arena.p + (size_t)row0 * d, (size_t)rows * d * 4, cudaMemcpyDeviceToDevice, s));
  }
  // store rows [src, src + rows) -> [dst, dst + rows), dst < src (compaction): chunks never overlap
  void store_move_down(long long dst, long long src, long long rows, cudaStream_t s) {
    if (!rows || dst == src) return;
    const long long chunk = std::min(rows, src - dst);
    for (long long r = 0; r < rows; r += chunk) {
      const long long c = std::min(chunk, rows - r);
      if (split3) {
        CK(cudaMemcpyAsync(xsplit.p + (size_t)(dst + r) * d, xsplit.p + (size_t)(src + r) * d, (size_t)c * d * 4,
                           cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(x3.p + (size_t)(dst + r) * d, x3.p + (size_t)(src + r) * d, (size_t)c * d * 2,
                           cudaMemcpyDeviceToDevice, s));
      } else {
        CK(cudaMemcpyAsync(arena.p + (size_t)(dst + r) * d, arena.p + (size_t)(src + r) * d, (size_t)c * d * 4,
                           cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  // In-place format change of the resident store (placements), tail-first: the destination's window
  // for rows [lo, hi) is mapped, the rows converted, and the source's chunks above lo released, so
  // device memory peaks at max(source, destination) plus about a chunk each. To split3 only when
  // every element round-trips (checked before anything is released); returns whether it converted.
  bool convert_store(bool to3) {
    if (to3 == split3) return true;
    const long long rows = n_resident;
    const long long cr = conv_rows();
    if (to3) {
      if (!inexact_ctr.p) inexact_ctr.alloc(1);
      CK(cudaMemset(inexact_ctr.p, 0, sizeof(unsigned)));
      CK(rd::launch_split3(arena.p, rows, d, nullptr, nullptr, inexact_ctr.p, 0));
      unsigned bad = 0;
      CK(cudaMemcpy(&bad, inexact_ctr.p, sizeof bad, cudaMemcpyDeviceToHost));
      if (bad) return false;
      xsplit.reserve((size_t)std::max(1LL, n) * d, d);
      x3.reserve((size_t)std::max(1LL, n) * d, d);
      for (long long hi = rows; hi > 0;) {
        const long long lo = std::max(0LL, hi - cr);
        xsplit.map_range((size_t)lo * d, (size_t)hi * d);
        x3.map_range((size_t)lo * d, (size_t)hi * d);
        CK(rd::launch_split3(arena.p + (size_t)lo * d, hi - lo, d, xsplit.p + (size_t)lo * d, x3.p + (size_t)lo * d,
                             inexact_ctr.p, 0));
        CK(cudaStreamSynchronize(0));
        arena.unmap_from((size_t)lo * d);
        hi = lo;
      }
      arena.reset();
      xsplit.n = x3.n = (size_t)rows * d;
    } else {
      arena.reserve((size_t)std::max(1LL, n) * d, d);
      for (long long hi = rows; hi > 0;) {
        const long long lo = std::max(0LL, hi - cr);
        arena.map_range((size_t)lo * d, (size_t)hi * d);
        CK(rd::launch_join3(xsplit.p + (size_t)lo * d, x3.p + (size_t)lo * d, hi - lo, d, arena.p + (size_t)lo * d, 0));
        CK(cudaStreamSynchronize(0));
        xsplit.unmap_from((size_t)lo * d);
        x3.unmap_from((size_t)lo * d);
        hi = lo;
      }
      xsplit.reset();
      x3.reset();
      arena.n = (size_t)rows * d;
    }
    split3 = to3;
    return true;
  }

  // rows that fit one conversion buffer (host <-> split3 transfers, materialize)
  long long conv_rows() const { return std::max<long long>(1, (long long)((size_t(64) << 20) / ((size_t)d * 4))); }

  // Builds the store of a fully resident index from fp32 rows produced chunk by chunk
  // (produce(r0, rows, dst): rows [r0, r0 + rows) in list order into the device buffer dst), with the
  // row norms on the way: split3 when eligible (the fp32 rows never exist in HBM all at once); if any
  // element does not round-trip, the rows are produced again into an fp32 store.
  void materialize(const std::function<void(long long, long long, float*)>& produce) {
    xnorm.alloc(n);
    DBuf<float> tmp;
    const long long cr = std::min<long long>(std::max(1LL, n), conv_rows());
    tmp.alloc((size_t)cr * d);
    for (int attempt = 0; attempt < 2; ++attempt) {
      split3 = attempt == 0 && split3_eligible() && !resid_fmt();
      resid_ok = true;
      if (attempt == 1 && !std::getenv("RD_SPLIT3_QUIET"))
        fprintf(stderr, "rd: split3 store inexact for this data (%s); using fp32 rows\n", "residual out of bf16 range");
      store_reserve(n);
      store_resize(n);
      if (split3) {
        if (!inexact_ctr.p) inexact_ctr.alloc(1);
        CK(cudaMemset(inexact_ctr.p, 0, sizeof(unsigned)));
      }
      for (long long r0 = 0; r0 < n; r0 += cr) {
        const long long c = std::min(cr, n - r0);
        produce(r0, c, tmp.p);
        CK(rd::launch_row_norms(tmp.p, c, d, xnorm.p + r0, 0));
        store_put(r0, tmp.p, c, 0);
      }
      if (!split3) break;
      unsigned bad = 0;
      CK(cudaMemcpy(&bad, inexact_ctr.p, sizeof bad, cudaMemcpyDeviceToHost));
      if (bad == 0) break;
    }
    CK(cudaDeviceSynchronize());
    finish_layout();
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

  // After every (re)layout: the scan's operand for the resident store. Default (RD_STORE unset):
  // every list resident and the last placement chose it -> the residual store (fp32 rows + r1 plane;
  // a split3 store is converted back to fp32 rows in place first); otherwise split3 unless a byte
  // budget already chose fp32 rows. RD_STORE=split3: the round-2 rule (split3 by placement, a
  // pre-split copy beside fp32 rows only without a budget).
  void build_presplit() {
    drop_resid();
    const char* env = std::getenv("RD_PRESPLIT");
    const bool pre_off = env && std::atoi(env) == 0;
    if (resid_fmt() && !pre_off && n_resident > 0) {
      if (resid_ok && n_resident == n) {
        if (split3 && convert_store(false)) upload_residency();
        if (!split3) {
          presplit = false;
          xsplit.reset();
          if (build_resid()) return;
        }
      }
      // not every list resident, or no room for the residual plane: split3 in place (1.5 x the fp32
      // rows) unless a budget chose fp32 rows
      if (!split3 && !budgeted && split3_eligible() && convert_store(true)) upload_residency();
    }
    if (split3) {  // the store is the scan's operand
      presplit = n_resident > 0;
      return;
    }
    presplit = false;
    xsplit.reset();
    // a byte budget (e.g. the LLM reservation, C5) must not be exceeded by a second copy
    if (!tc_scan() || pre_off || n_resident == 0 || budgeted) return;
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
  DBuf<unsigned long long> dbg_buf, dbg_scan, dbg_stall, dbg_chain_buf;

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

  // Device-side residency tables after any relayout: res_row0, each list's row base (fp32 rows:
  // the fp32 arena or mapped host memory; nullptr for a list in the split3 store, whose rows the
  // kernels address through res_row0) and the scans' tensor maps.
  void upload_residency() {
    d_res_row0.alloc(nlist);
    CK(cudaMemcpy(d_res_row0.p, res_row0.data(), sizeof(long long) * nlist, cudaMemcpyHostToDevice));
    if (!split3) {
      xsplit.reset();  // any relayout invalidates the pre-split copy (rebuilt by build_presplit)
      presplit = false;
      drop_resid();
    }
    std::vector<const float*> base(nlist);
    for (int l = 0; l < nlist; ++l)
      base[l] = resident[l] ? (split3 ? nullptr : arena.p + (size_t)res_row0[l] * d)
                            : host_arena.p + (size_t)host_row0[l] * d;
    d_list_base.alloc(nlist);
    CK(cudaMemcpy(d_list_base.p, base.data(), sizeof(const float*) * nlist, cudaMemcpyHostToDevice));
    if (split3) {
      if (n_resident > 0) {
        xmap128 = make_split_map(xsplit.p, n_resident, d, rd::kTcRows);
        xmap32 = make_split_map(xsplit.p, n_resident, d, 32);
      }
      presplit = n_resident > 0;
    } else if (arena.p) {
      map256 = make_row_map(arena.p, std::max(1LL, n_resident), d, rd::kScanRows);
      map128 = make_row_map(arena.p, std::max(1LL, n_resident), d, rd::kTcRows);
      map32 = make_row_map(arena.p, std::max(1LL, n_resident), d, 32);
    }
  }
  // device pointers the kernels take for the split3 store (nullptr in fp32 mode)
  const __nv_bfloat16* x12_dev() const { return split3 ? reinterpret_cast<const __nv_bfloat16*>(xsplit.p) : nullptr; }
  const __nv_bfloat16* x3_dev() const { return split3 ? reinterpret_cast<const __nv_bfloat16*>(x3.p) : nullptr; }
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

// One search (search.cu), shared by the single-index entry points and the shard groups (group.cu).
namespace rdh {
enum SearchMode { kAsync = 0, kSync = 1, kStatsAsync = 2 };
void validate_search(const rd_index* h, int nprobe, int k);
bool select_all_needed(const rd_index* h, int nprobe);
void* select_all_scratch(rd_index* h, long long B, size_t* bytes);
// Enqueues one search of B device queries on stream s. kAsync: nothing is read back; kSync: the
// counters are copied back and `st` filled before returning; kStatsAsync: the counter copy is
// enqueued, the caller synchronizes s and then calls finish_stats. result_bytes: bytes after the
// stat block the counter copy brings along (the host path's results); before_sync runs before it.
void do_search(rd_index* h, const float* d_q, long long B, int nprobe, int k, long long* d_ids, float* d_dists,
               cudaStream_t s, int mode, rd_search_stats* st, size_t result_bytes = 0,
               const std::function<void()>& before_sync = {});
void finish_stats(rd_index* h, rd_search_stats* st);
}  // namespace rdh
