// rd_ragsim.hpp — C++17 adapter that puts the rd.h retrieval engine behind the
// reference's (ragsim) retrieval-stage conventions. Header-only; link either
// implementation of rd.h (librd_b200.so, or oracle/librd_cpu.so for CPU tests).
//
// Reference seam (§8f rows 1 and 4):
//   R2  retrieval_time(P, db)          core/src/cost_model.cpp:15-21   -> RetrievalIndex::search() wall time,
//                                                                          MeasuredRetrievalCost::seconds(B)
//   R3  choose_retrieval_batch         core/src/scheduler.cpp:80-83    -> choose_retrieval_batch()
//   R4  retrieval worker               core/src/simulator.cpp:273-289, 328-368 -> RetrievalWorker
//   R9  profiler cost inputs           core/src/scheduler.cpp:123-131;
//       fit_power_law / predict        core/src/cost_model.cpp:97-136  -> fit_power_law(), PowerLawFit::predict()
//   R6  partition reconfiguration      core/src/simulator.cpp:331-352  -> RetrievalWorker::reconfigure()
// Errors follow ragsim's model (core/include/ragsim/errors.hpp:11-26): Error, InfeasibleError,
// ParseError, raised from the rd.h status codes exactly as the ragsim CLI maps exit codes
// (tools/main.cpp:30).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <deque>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rd.h"

namespace ragsim {
namespace rd {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InfeasibleError : Error {
  using Error::Error;
};
struct ParseError : Error {
  using Error::Error;
};

inline void check(int rc, const char* what) {
  if (rc == RD_OK) return;
  const std::string msg = std::string(what) + ": " + rd_last_error();
  if (rc == RD_ERR_INFEASIBLE) throw InfeasibleError(msg);
  if (rc == RD_ERR_INVALID) throw ParseError(msg);
  throw Error(msg);
}

struct SearchResult {
  std::vector<int64_t> ids;  // B x k, per query ascending (distance, id)
  std::vector<float> dists;
  rd_search_stats stats{};
};

// RAII owner of one rd_index handle (one in-flight search, as ragsim's single retrieval worker).
class RetrievalIndex {
 public:
  static RetrievalIndex synthetic(const rd_synth_desc& desc, int device = 0) {
    rd_index* h = nullptr;
    check(rd_index_create_synthetic(&desc, device, &h), "rd_index_create_synthetic");
    return RetrievalIndex(h);
  }
  static RetrievalIndex load(const std::string& path, int device = 0) {
    rd_index* h = nullptr;
    check(rd_index_load(path.c_str(), device, &h), "rd_index_load");
    return RetrievalIndex(h);
  }
  RetrievalIndex(RetrievalIndex&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  RetrievalIndex& operator=(RetrievalIndex&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  RetrievalIndex(const RetrievalIndex&) = delete;
  RetrievalIndex& operator=(const RetrievalIndex&) = delete;
  ~RetrievalIndex() { reset(); }

  rd_index* handle() const { return h_; }
  rd_index_info info() const {
    rd_index_info i{};
    check(rd_index_info_get(h_, &i), "rd_index_info_get");
    return i;
  }
  void place(const rd_placement& p) { check(rd_index_place(h_, &p), "rd_index_place"); }
  rd_migration_stats migrate(const std::vector<int32_t>& promote, const std::vector<int32_t>& demote,
                             uint64_t hbm_budget_bytes = 0) {
    rd_migration_stats st{};
    check(rd_index_migrate(h_, promote.data(), (int32_t)promote.size(), demote.data(), (int32_t)demote.size(),
                           hbm_budget_bytes, &st),
          "rd_index_migrate");
    return st;
  }
  void save(const std::string& path) const { check(rd_index_save(h_, path.c_str()), "rd_index_save"); }

  // queries: B x d row-major (host). The returned stats.seconds is the measured stage time that
  // replaces retrieval_time(P, db).
  SearchResult search(const float* queries, int64_t B, int nprobe, int k) {
    SearchResult r;
    r.ids.resize((size_t)(B * k));
    r.dists.resize((size_t)(B * k));
    check(rd_search(h_, queries, B, nprobe, k, r.ids.data(), r.dists.data(), &r.stats), "rd_search");
    return r;
  }

 private:
  explicit RetrievalIndex(rd_index* h) : h_(h) {}
  void reset() {
    if (h_) rd_index_destroy(h_);
    h_ = nullptr;
  }
  rd_index* h_ = nullptr;
};

// Greedy drain of the retrieval queue (scheduler.cpp:80-83): the whole backlog up to the cap.
inline int choose_retrieval_batch(int backlog, int max_retrieval_batch) {
  if (backlog < 1) throw Error("choose_retrieval_batch: empty backlog");
  if (max_retrieval_batch < 1) throw Error("choose_retrieval_batch: max_retrieval_batch must be >= 1");
  return backlog < max_retrieval_batch ? backlog : max_retrieval_batch;
}

// T(B) = a * B^c fitted by least squares in log-log space, the form the reference's profiler
// consumes (cost_model.cpp:97-136): a negative slope is clamped to a constant (c = 0, a = the
// geometric mean), residual = RMS log error.
struct BatchTime {
  double batch_size;
  double seconds;
};
struct PowerLawFit {
  double a = 0.0, c = 0.0, residual = 0.0;
  int samples = 0;
  bool exponent_clamped = false;
  double predict(double batch_size) const { return a * std::pow(batch_size, c); }
};
inline PowerLawFit fit_power_law(const std::vector<BatchTime>& s) {
  std::vector<double> xs;
  for (const auto& v : s) {
    if (!(v.batch_size > 0.0) || !(v.seconds > 0.0)) throw Error("fit_power_law: samples must be positive");
    if (std::find(xs.begin(), xs.end(), v.batch_size) == xs.end()) xs.push_back(v.batch_size);
  }
  if (s.size() < 2 || xs.size() < 2) throw Error("fit_power_law: underdetermined fit");
  double mx = 0, my = 0;
  for (const auto& v : s) {
    mx += std::log(v.batch_size);
    my += std::log(v.seconds);
  }
  mx /= (double)s.size();
  my /= (double)s.size();
  double sxy = 0, sxx = 0;
  for (const auto& v : s) {
    const double dx = std::log(v.batch_size) - mx;
    sxy += dx * (std::log(v.seconds) - my);
    sxx += dx * dx;
  }
  PowerLawFit f;
  f.samples = (int)s.size();
  const double slope = sxy / sxx;
  if (slope < 0.0) {
    f.c = 0.0;
    f.exponent_clamped = true;
    f.a = std::exp(my);
  } else {
    f.c = slope;
    f.a = std::exp(my - slope * mx);
  }
  double sq = 0;
  for (const auto& v : s) {
    const double e = std::log(v.seconds) - std::log(f.predict(v.batch_size));
    sq += e * e;
  }
  f.residual = std::sqrt(sq / (double)s.size());
  return f;
}

// Calibrates T_ret(B) for the index's current placement by timing real searches (median of
// `reps` after one warm-up per size). Re-calibrate after place() / migrate(): the resident
// fraction is what the reference's retrieval_time(P, db) models.
class MeasuredRetrievalCost {
 public:
  MeasuredRetrievalCost(RetrievalIndex& idx, std::vector<float> query_pool, int d, int nprobe, int k)
      : idx_(idx), pool_(std::move(query_pool)), d_(d), nprobe_(nprobe), k_(k) {
    if (d_ < 1 || pool_.size() < (size_t)d_) throw ParseError("MeasuredRetrievalCost: empty query pool");
  }
  const PowerLawFit& calibrate(const std::vector<int>& batch_sizes, int reps = 3) {
    samples_.clear();
    for (int B : batch_sizes) {
      std::vector<double> t;
      for (int r = 0; r <= reps; ++r) {
        const double s = time_batch(B, r);
        if (r) t.push_back(s);  // r == 0 warms up
      }
      std::nth_element(t.begin(), t.begin() + (long)t.size() / 2, t.end());
      samples_.push_back({(double)B, t[t.size() / 2]});
    }
    fit_ = fit_power_law(samples_);
    return fit_;
  }
  double seconds(int batch) const { return fit_.predict(batch); }  // replaces retrieval_time(P, db)
  const std::vector<BatchTime>& samples() const { return samples_; }
  // one real search of B pool queries (cycled from offset `salt`), wall seconds
  double time_batch(int B, int salt = 0) {
    const int64_t pool_n = (int64_t)(pool_.size() / d_);
    std::vector<float> q((size_t)B * d_);
    for (int b = 0; b < B; ++b) {
      const int64_t src = (b + (int64_t)salt * B) % pool_n;
      std::copy(pool_.begin() + src * d_, pool_.begin() + (src + 1) * d_, q.begin() + (int64_t)b * d_);
    }
    const auto t0 = std::chrono::steady_clock::now();
    idx_.search(q.data(), B, nprobe_, k_);
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

 private:
  RetrievalIndex& idx_;
  std::vector<float> pool_;
  int d_, nprobe_, k_;
  std::vector<BatchTime> samples_;
  PowerLawFit fit_;
};

// The retrieval worker of RAGDoll's pipeline (simulator.cpp:273-289, 328-368) driven by real
// searches: requests queue on arrival; whenever the worker is free it drains a greedy batch
// (choose_retrieval_batch), runs one rd_search over the batch's queries and is busy for the
// measured seconds; reconfigurations (list migrations) queued with reconfigure() are applied
// between batches, charging their measured time to the worker first (simulator.cpp:331-352).
struct Request {
  double arrival = 0.0;   // seconds
  int64_t query = 0;      // row of the query pool
  double dispatched = 0.0, completed = 0.0;
  std::vector<int64_t> ids;  // its top-k
};
struct WorkerReport {
  int batches = 0;
  double busy_seconds = 0.0, reconfig_seconds = 0.0, makespan = 0.0;
  std::vector<int> batch_sizes;
};

class RetrievalWorker {
 public:
  RetrievalWorker(RetrievalIndex& idx, const float* query_pool, int d, int nprobe, int k, int max_retrieval_batch)
      : idx_(idx), pool_(query_pool), d_(d), nprobe_(nprobe), k_(k), max_batch_(max_retrieval_batch) {}

  void reconfigure(std::vector<int32_t> promote, std::vector<int32_t> demote, uint64_t budget = 0) {
    pending_.push_back({std::move(promote), std::move(demote), budget});
  }

  // Runs every request (sorted by arrival) to completion; fills dispatched / completed / ids.
  WorkerReport run(std::vector<Request>& reqs) {
    std::sort(reqs.begin(), reqs.end(), [](const Request& a, const Request& b) { return a.arrival < b.arrival; });
    WorkerReport rep;
    std::deque<size_t> queue;
    size_t next = 0;
    double now = 0.0;
    while (next < reqs.size() || !queue.empty()) {
      if (queue.empty()) now = std::max(now, reqs[next].arrival);
      while (next < reqs.size() && reqs[next].arrival <= now) queue.push_back(next++);
      for (auto& m : pending_) {  // between batches only
        const rd_migration_stats st = idx_.migrate(m.promote, m.demote, m.budget);
        now += st.seconds;
        rep.reconfig_seconds += st.seconds;
      }
      pending_.clear();
      const int B = choose_retrieval_batch((int)queue.size(), max_batch_);
      std::vector<float> q((size_t)B * d_);
      for (int b = 0; b < B; ++b)
        std::copy(pool_ + reqs[queue[b]].query * d_, pool_ + (reqs[queue[b]].query + 1) * d_, q.begin() + (size_t)b * d_);
      const auto t0 = std::chrono::steady_clock::now();
      SearchResult r = idx_.search(q.data(), B, nprobe_, k_);
      const double dur = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      for (int b = 0; b < B; ++b) {
        Request& rq = reqs[queue.front()];
        queue.pop_front();
        rq.dispatched = now;
        rq.completed = now + dur;
        rq.ids.assign(r.ids.begin() + (size_t)b * k_, r.ids.begin() + (size_t)(b + 1) * k_);
      }
      now += dur;
      rep.batches += 1;
      rep.busy_seconds += dur;
      rep.batch_sizes.push_back(B);
    }
    rep.makespan = now;
    return rep;
  }

 private:
  struct Reconfig {
    std::vector<int32_t> promote, demote;
    uint64_t budget;
  };
  RetrievalIndex& idx_;
  const float* pool_;
  int d_, nprobe_, k_, max_batch_;
  std::vector<Reconfig> pending_;
};

}  // namespace rd
}  // namespace ragsim
