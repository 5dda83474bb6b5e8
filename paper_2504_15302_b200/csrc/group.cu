// group.cu — multi-GPU shard groups behind include/rd.h (rd_group_*), SURVEY §8e / row N11.
//
// A group is G row stripes of one knowledge base (stripe g holds rows [g*len/G, (g+1)*len/G) of
// every list), each an ordinary rd_index on its own device. One search:
//
//   root device queries --(peer copy over NVLink)--> every stripe's device
//   every stripe: the full single-device chain (search.cu), its exact top-k into a result slot
//   -> NCCL gather of the slots to the root device (grouped ncclSend / ncclRecv: NCCL 2.27 has no
//      ncclGather) -> one device merge by (distance, id) -> the merged top-k
//
// so the caller gets one merged result per retrieval call, as the reference's retrieval worker
// expects (core/src/simulator.cpp:359, serial :560). Stripes that share a device (NCCL admits one
// rank per device) gather by device copies instead; so does RD_GROUP_TRANSPORT=copy (A/B).
//
// Two ways to form a group:
//   one process, G devices (rd_group_create / rd_group_create_synthetic): ncclCommInitAll, one host
//     worker thread per stripe enqueues its search so the G chains start together;
//   one process per device (rd_group_create_rank, e.g. under torchrun): ncclCommInitRank with a
//     unique id the caller broadcasts; rank 0 is the root and receives the merged result.
//
// NCCL is bound at run time (dlopen of libnccl.so.2 — the copy a host framework already loaded, or
// the system one): the library has no link-time NCCL dependency to clash with another NCCL build in
// the same process, and a group that needs NCCL fails loudly if it is missing.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <exception>
#include <mutex>

#include "host.cuh"

namespace {

// ------------------------------------------------------------------ NCCL, bound at run time
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetVersion) get_version = nullptr;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      const char* e = dlerror();
      a.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(lib, name));
      if (!fp && a.why.empty()) a.why = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.init_rank, "ncclCommInitRank");
    sym(a.init_all, "ncclCommInitAll");
    sym(a.destroy, "ncclCommDestroy");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.error_string, "ncclGetErrorString");
    sym(a.get_version, "ncclGetVersion");
    return a;
  }();
  if (!api.why.empty()) throw_rd(RD_ERR_RUNTIME, "NCCL unavailable: %s", api.why.c_str());
  return api;
}

#define NK(x)                                                                                           \
  do {                                                                                                  \
    ncclResult_t r_ = (x);                                                                              \
    if (r_ != ncclSuccess)                                                                              \
      throw_rd(RD_ERR_RUNTIME, "%s failed: %s (%s:%d)", #x, nccl().error_string(r_), __FILE__, __LINE__); \
  } while (0)

// One persistent host thread per stripe: enqueueing a search is ~10 launches of host work, so G
// stripes enqueued from one thread would start up to G times that apart.
class Worker {
 public:
  Worker() : th_([this] { loop(); }) {}
  ~Worker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void post(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = std::move(f);
      busy_ = true;
      err_ = nullptr;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !busy_; });
    if (err_) std::rethrow_exception(err_);
  }

 private:
  void loop() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return quit_ || (busy_ && job_); });
      if (quit_) return;
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
      err_ = e;
      busy_ = false;
      cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::function<void()> job_;
  bool busy_ = false, quit_ = false;
  std::exception_ptr err_;
  std::thread th_;
};

}  // namespace

// ====================================================================== the group
struct rd_group {
  struct Lane {
    rd_index* h = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_done = nullptr;
    DBuf<float> q;     // this stripe's copy of the queries (lane 0: the host path's query buffer)
    DBuf<char> res;    // result slots: lane 0 holds all G (the gather target), others their own
    ncclComm_t comm = nullptr;
    std::unique_ptr<Worker> worker;
    rd_search_stats st{};
  };
  std::vector<Lane> lanes;  // local stripes: G in one process, 1 per rank
  int G = 1;                // stripes in the whole group
  int rank = 0, nranks = 1; // one process per device: this process's rank (root = 0)
  bool multiproc = false;
  int transport = RD_GROUP_TRANSPORT_NONE;
  bool owns = true;
  cudaEvent_t ev_in = nullptr;  // queries ready on the root device
  DBuf<long long> out_ids;      // host path: merged result on the root device
  DBuf<float> out_dists;
  HBuf<char> h_out;
  size_t slot_bytes = 0;

  int root_device() const { return lanes[0].h->device; }
  static size_t slot_for(long long B, int k) { return ((size_t)B * k * 12 + 255) / 256 * 256; }

  ~rd_group() {
    for (auto& l : lanes) l.worker.reset();
    for (auto& l : lanes) {
      if (l.h) cudaSetDevice(l.h->device);
      if (l.comm) nccl().destroy(l.comm);
      if (l.stream) cudaStreamDestroy(l.stream);
      if (l.ev_done) cudaEventDestroy(l.ev_done);
      l.q.reset();
      l.res.reset();
    }
    if (ev_in) {
      cudaSetDevice(root_device());
      cudaEventDestroy(ev_in);
    }
    out_ids.reset();
    out_dists.reset();
    h_out.reset();
    if (owns)
      for (auto& l : lanes) delete l.h;
  }

  void init_lanes(const std::vector<rd_index*>& shards) {
    lanes = std::vector<Lane>(shards.size());
    for (size_t g = 0; g < shards.size(); ++g) {
      Lane& L = lanes[g];
      L.h = shards[g];
      CK(cudaSetDevice(L.h->device));
      CK(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&L.ev_done, cudaEventDisableTiming));
      if (shards.size() > 1) L.worker = std::make_unique<Worker>();
    }
    CK(cudaSetDevice(root_device()));
    CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
  }

  // runs f(g) for every local stripe: on the stripes' worker threads when there are several
  void each(const std::function<void(int)>& f) {
    if (lanes.size() == 1) {
      f(0);
      return;
    }
    for (size_t g = 0; g < lanes.size(); ++g) lanes[g].worker->post([&f, g] { f((int)g); });
    std::exception_ptr first;
    for (auto& L : lanes) {
      try {
        L.worker->wait();
      } catch (...) {
        if (!first) first = std::current_exception();
      }
    }
    if (first) std::rethrow_exception(first);
  }

  // One group search: d_q (B x d) on the root device / this rank's device, ready in stream s;
  // the merged top-k into d_ids / d_dists on s (multi-process non-root ranks: their own top-k).
  void search(const float* d_q, long long B, int nprobe, int k, long long* d_ids, float* d_dists, cudaStream_t s,
              bool stats) {
    for (auto& L : lanes) rdh::validate_search(L.h, nprobe, k);
    if ((long long)G * k > rd::shard_merge_max_candidates())
      throw_rd(RD_ERR_INVALID, "group search: stripes x k <= %d", rd::shard_merge_max_candidates());
    const int d = lanes[0].h->d;
    const size_t slot = slot_for(B, k);
    slot_bytes = slot;
    const bool gather_here = !multiproc || rank == 0;
    CK(cudaSetDevice(root_device()));
    lanes[0].res.ensure(gather_here ? slot * G : slot);
    CK(cudaEventRecord(ev_in, s));
    each([&](int g) {
      Lane& L = lanes[g];
      CK(cudaSetDevice(L.h->device));
      const float* q = d_q;
      cudaStream_t ls = g == 0 ? s : L.stream;
      if (g > 0) {  // this stripe's copy of the queries, from the root device (NVLink peer copy)
        L.res.ensure(slot);
        L.q.ensure((size_t)B * d);
        CK(cudaStreamWaitEvent(ls, ev_in, 0));
        CK(cudaMemcpyPeerAsync(L.q.p, L.h->device, d_q, root_device(), (size_t)B * d * sizeof(float), ls));
        q = L.q.p;
      }
      char* r = L.res.p;
      rdh::do_search(L.h, q, B, nprobe, k, reinterpret_cast<long long*>(r), reinterpret_cast<float*>(r + (size_t)B * k * 8),
                     ls, stats ? rdh::kStatsAsync : rdh::kAsync, stats ? &L.st : nullptr);
    });
    // gather the result slots on the root device
    if (G > 1 && transport == RD_GROUP_TRANSPORT_NCCL) {
      const auto& api = nccl();
      NK(api.group_start());
      if (multiproc) {
        if (rank == 0) {
          for (int r = 1; r < nranks; ++r)
            NK(api.recv(lanes[0].res.p + (size_t)r * slot, slot, ncclUint8, r, lanes[0].comm, s));
        } else {
          NK(api.send(lanes[0].res.p, slot, ncclUint8, 0, lanes[0].comm, s));
        }
      } else {
        for (int g = 1; g < G; ++g) {
          NK(api.send(lanes[g].res.p, slot, ncclUint8, 0, lanes[g].comm, lanes[g].stream));
          NK(api.recv(lanes[0].res.p + (size_t)g * slot, slot, ncclUint8, g, lanes[0].comm, s));
        }
      }
      NK(api.group_end());
    } else if (G > 1) {  // device copies (stripes sharing a device, or forced)
      for (int g = 1; g < G; ++g) {
        Lane& L = lanes[g];
        CK(cudaSetDevice(L.h->device));
        CK(cudaMemcpyPeerAsync(lanes[0].res.p + (size_t)g * slot, root_device(), L.res.p, L.h->device, slot, L.stream));
        CK(cudaEventRecord(L.ev_done, L.stream));
        CK(cudaSetDevice(root_device()));
        CK(cudaStreamWaitEvent(s, L.ev_done, 0));
      }
    }
    CK(cudaSetDevice(root_device()));
    const char* base = lanes[0].res.p;
    if (gather_here && G > 1) {
      CK(rd::launch_shard_merge_strided(G, B, k, base, slot, base + (size_t)B * k * 8, slot, d_ids, d_dists, s));
    } else {  // one stripe, or a non-root rank: its own top-k
      CK(cudaMemcpyAsync(d_ids, base, (size_t)B * k * 8, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(d_dists, base + (size_t)B * k * 8, (size_t)B * k * 4, cudaMemcpyDeviceToDevice, s));
    }
  }

  // after the root stream synchronized: every stripe's counters summed
  void collect(rd_search_stats* st) {
    std::memset(st, 0, sizeof *st);
    for (auto& L : lanes) {
      CK(cudaSetDevice(L.h->device));
      CK(cudaStreamSynchronize(L.stream));
      rd_search_stats one{};
      rdh::finish_stats(L.h, &one);
      st->bytes_algorithmic += one.bytes_algorithmic;
      st->bytes_lists_resident += one.bytes_lists_resident;
      st->h2d_list_bytes += one.h2d_list_bytes;
      st->lists_probed += one.lists_probed;
      st->tiles += one.tiles;
      st->kernel_launches += one.kernel_launches + 1;  // + the merge (or result copy)
      st->scan_ms = std::max(st->scan_ms, one.scan_ms);
      st->coarse_ms = std::max(st->coarse_ms, one.coarse_ms);
      st->offload_ms = std::max(st->offload_ms, one.offload_ms);
      st->margin_failures += one.margin_failures;
      st->probe_failures += one.probe_failures;
    }
    CK(cudaSetDevice(root_device()));
  }
};

namespace {

void init_transport(rd_group* g) {
  const int n = (int)g->lanes.size();
  g->transport = RD_GROUP_TRANSPORT_NONE;
  if (g->G == 1) return;
  const char* force = std::getenv("RD_GROUP_TRANSPORT");
  bool distinct = true;
  for (int a = 0; a < n; ++a)
    for (int b = a + 1; b < n; ++b)
      if (g->lanes[a].h->device == g->lanes[b].h->device) distinct = false;
  if (!distinct || (force && std::strcmp(force, "copy") == 0)) {
    g->transport = RD_GROUP_TRANSPORT_COPY;
    for (int a = 1; a < n; ++a) {  // NVLink peer access where the devices differ
      const int da = g->lanes[a].h->device, d0 = g->root_device();
      if (da == d0) continue;
      int ok = 0;
      CK(cudaDeviceCanAccessPeer(&ok, d0, da));
      if (!ok) continue;
      CK(cudaSetDevice(d0));
      cudaError_t e = cudaDeviceEnablePeerAccess(da, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      CK(cudaSetDevice(da));
      e = cudaDeviceEnablePeerAccess(d0, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
      cudaGetLastError();
    }
    return;
  }
  std::vector<int> devs(n);
  std::vector<ncclComm_t> comms(n);
  for (int a = 0; a < n; ++a) devs[a] = g->lanes[a].h->device;
  NK(nccl().init_all(comms.data(), n, devs.data()));
  for (int a = 0; a < n; ++a) g->lanes[a].comm = comms[a];
  g->transport = RD_GROUP_TRANSPORT_NCCL;
  for (int a = 1; a < n; ++a) {  // the query broadcast is a peer copy
    int ok = 0;
    CK(cudaDeviceCanAccessPeer(&ok, g->root_device(), devs[a]));
    if (!ok) continue;
    CK(cudaSetDevice(g->root_device()));
    cudaError_t e = cudaDeviceEnablePeerAccess(devs[a], 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
    CK(cudaSetDevice(devs[a]));
    e = cudaDeviceEnablePeerAccess(g->root_device(), 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
    cudaGetLastError();
  }
}

void check_stripes(const std::vector<rd_index*>& s) {
  for (size_t g = 0; g < s.size(); ++g) {
    if (!s[g]) throw_rd(RD_ERR_INVALID, "group: null stripe %zu", g);
    if (s[g]->d != s[0]->d || s[g]->nlist != s[0]->nlist)
      throw_rd(RD_ERR_INVALID, "group: stripes must share d and nlist");
    for (size_t h = 0; h < g; ++h)
      if (s[h] == s[g]) throw_rd(RD_ERR_INVALID, "group: stripe handle %zu given twice", g);
  }
}

}  // namespace

extern "C" {

int rd_group_create(rd_index* const* shards, int32_t G, rd_group** out) {
  return guarded([&] {
    if (!shards || G < 1 || !out) throw_rd(RD_ERR_INVALID, "group_create: invalid arguments");
    std::vector<rd_index*> s(shards, shards + G);
    check_stripes(s);
    auto g = std::make_unique<rd_group>();
    g->owns = false;  // adopted only once everything below succeeded
    g->G = G;
    g->init_lanes(s);
    init_transport(g.get());
    g->owns = true;
    *out = g.release();
  });
}

int rd_group_create_synthetic(const rd_synth_desc* desc, const int32_t* devices, int32_t G, rd_group** out) {
  return guarded([&] {
    if (!desc || !devices || G < 1 || !out) throw_rd(RD_ERR_INVALID, "group_create_synthetic: invalid arguments");
    std::vector<rd_index*> s(G, nullptr);
    std::vector<int> rc(G, RD_OK);
    std::vector<std::string> msg(G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)  // stripes built concurrently, one host thread per device
      th.emplace_back([&, g] {
        rd_synth_desc one = *desc;
        one.shard = g;
        one.num_shards = G;
        rc[g] = rd_index_create_synthetic(&one, devices[g], &s[g]);
        if (rc[g] != RD_OK) msg[g] = rd_last_error();
      });
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g)
      if (rc[g] != RD_OK) {
        for (auto* h : s) delete h;
        throw_rd(rc[g], "stripe %d: %s", g, msg[g].c_str());
      }
    const int r = rd_group_create(s.data(), G, out);
    if (r != RD_OK) {
      const std::string m = rd_last_error();
      for (auto* h : s) delete h;
      throw_rd(r, "%s", m.c_str());
    }
  });
}

int rd_group_unique_id(uint8_t* out) {
  return guarded([&] {
    if (!out) throw_rd(RD_ERR_INVALID, "null out");
    ncclUniqueId id;
    static_assert(sizeof id == RD_GROUP_ID_BYTES, "NCCL unique id size");
    NK(nccl().get_unique_id(&id));
    std::memcpy(out, &id, sizeof id);
  });
}

int rd_group_create_rank(rd_index* shard, const uint8_t* id, int32_t nranks, int32_t rank, rd_group** out) {
  return guarded([&] {
    if (!shard || !id || nranks < 1 || rank < 0 || rank >= nranks || !out)
      throw_rd(RD_ERR_INVALID, "group_create_rank: invalid arguments");
    auto g = std::make_unique<rd_group>();
    g->owns = false;
    g->G = nranks;
    g->rank = rank;
    g->nranks = nranks;
    g->multiproc = true;
    g->init_lanes({shard});
    if (nranks > 1) {
      ncclUniqueId uid;
      std::memcpy(&uid, id, sizeof uid);
      CK(cudaSetDevice(shard->device));
      NK(nccl().init_rank(&g->lanes[0].comm, nranks, uid, rank));
      g->transport = RD_GROUP_TRANSPORT_NCCL;
    }
    g->owns = true;
    *out = g.release();
  });
}

int rd_group_info_get(const rd_group* g, rd_group_info* o) {
  return guarded([&] {
    if (!g || !o) throw_rd(RD_ERR_INVALID, "null argument");
    std::memset(o, 0, sizeof *o);
    o->num_shards = g->G;
    o->local_shards = (int32_t)g->lanes.size();
    o->rank = g->rank;
    o->nranks = g->nranks;
    o->transport = g->transport;
    o->root_device = g->root_device();
    for (auto& L : g->lanes) {
      o->n += L.h->n;
      o->n_resident += L.h->n_resident;
    }
  });
}

rd_index* rd_group_shard(rd_group* g, int32_t i) {
  if (!g || i < 0 || i >= (int32_t)g->lanes.size()) return nullptr;
  return g->lanes[i].h;
}

int rd_group_place(rd_group* g, const rd_placement* p) {
  return guarded([&] {
    if (!g || !p) throw_rd(RD_ERR_INVALID, "null argument");
    for (size_t i = 0; i < g->lanes.size(); ++i) {
      const int rc = rd_index_place(g->lanes[i].h, p);
      if (rc != RD_OK) throw_rd(rc, "stripe %zu: %s", i, rd_last_error());
    }
  });
}

int rd_group_search_device(rd_group* g, const float* d_q, int64_t B, int32_t nprobe, int32_t k, int64_t* d_ids,
                           float* d_dists, void* stream, int32_t sync, rd_search_stats* st) {
  return guarded([&] {
    if (!g || B < 0 || (B > 0 && (!d_q || !d_ids || !d_dists))) throw_rd(RD_ERR_INVALID, "group search: invalid arguments");
    if (st) std::memset(st, 0, sizeof *st);
    if (B == 0) return;
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t s = (cudaStream_t)stream;
    g->search(d_q, B, nprobe, k, reinterpret_cast<long long*>(d_ids), d_dists, s, sync != 0 && st);
    if (sync) {
      CK(cudaStreamSynchronize(s));
      if (st) g->collect(st);
    }
    if (st) st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int rd_group_search(rd_group* g, const float* queries, int64_t B, int32_t nprobe, int32_t k, int64_t* out_ids,
                    float* out_dists, rd_search_stats* st) {
  return guarded([&] {
    if (!g || B < 0 || (B > 0 && (!queries || !out_ids || !out_dists)))
      throw_rd(RD_ERR_INVALID, "group search: invalid arguments");
    if (st) std::memset(st, 0, sizeof *st);
    if (B == 0) return;
    const auto t0 = std::chrono::steady_clock::now();
    auto& L0 = g->lanes[0];
    CK(cudaSetDevice(L0.h->device));
    const size_t qn = (size_t)B * L0.h->d, rn = (size_t)B * k;
    L0.q.ensure(qn);
    g->out_ids.ensure(rn);
    g->out_dists.ensure(rn);
    cudaStream_t s = L0.stream;
    CK(cudaMemcpyAsync(L0.q.p, queries, qn * sizeof(float), cudaMemcpyHostToDevice, s));
    g->search(L0.q.p, B, nprobe, k, g->out_ids.p, g->out_dists.p, s, st != nullptr);
    CK(cudaMemcpyAsync(out_ids, g->out_ids.p, rn * sizeof(long long), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out_dists, g->out_dists.p, rn * sizeof(float), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (st) {
      g->collect(st);
      st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

void rd_group_destroy(rd_group* g) { delete g; }

}  // extern "C"
