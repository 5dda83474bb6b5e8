// ragsim_measured.cpp — TEST / EVALUATION INFRASTRUCTURE. Runs the reference's
// own, unmodified simulator (core/src/simulator.cpp, scheduler.cpp, cost_model.cpp, workload.cpp,
// config_io.cpp, ...; compiled in place by oracle/build_ref_sim.sh, output only into oracle/_ref/)
// with its retrieval-stage cost replaced by MEASURED B200 search times.
//
// The seam is the reference's retrieval_time(P, db) (core/src/cost_model.cpp:15-21), called by the
// retrieval worker (simulator.cpp:359, serial :560) and the profiler (scheduler.cpp:126). The binary
// is linked with -Wl,--wrap on its mangled name, so every such call lands in
// __wrap_ragsim_retrieval_time below; with RAGSIM_TRET unset it forwards to the reference's formula
// (__real_), with RAGSIM_TRET=<table.json> (tools/measure_tret.py: median wall time of one rd_search
// through the C ABI on one B200, per batch size and resident fraction) it returns the measured time.
// The formula has no batch-size argument; the batch the worker just took is captured by wrapping
// choose_retrieval_batch (scheduler.cpp:80-83) the same way, and the profiler's evaluations (no batch
// taken) use the largest retrieval batch. Between measured points: the reference's own
// fit_power_law / predict (cost_model.cpp:97-136) over the batch sizes, linear in the resident
// fraction.
//
// Usage: ragsim_measured SCENARIO.json [SEED]   (prints one JSON object)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "ragsim/config_io.hpp"
#include "ragsim/cost_model.hpp"
#include "ragsim/rng.hpp"
#include "ragsim/scheduler.hpp"
#include "ragsim/simulator.hpp"
#include "ragsim/workload.hpp"

using namespace ragsim;

// the wrapped originals (--wrap resolves __real_<sym> to the reference's definitions)
extern "C" double __real__ZN6ragsim14retrieval_timeEiRKNS_15DatabaseProfileE(int, const DatabaseProfile&);
extern "C" int __real__ZN6ragsim22choose_retrieval_batchEii(int, int);

namespace {

struct Measured {
  std::vector<double> fractions;        // resident fraction per row, descending or any order
  std::vector<CostModelFit> fits;       // T(B) per row: the reference's power-law fit
  std::vector<std::vector<BatchTimeSample>> samples;
  bool on = false;
} g_meas;

int g_last_batch = 0;        // the batch choose_retrieval_batch just returned (0: none pending)
int g_default_batch = 64;    // the profiler's evaluations: the largest retrieval batch
long g_calls_measured = 0, g_calls_modelled = 0;
bool g_use_measured = false;

void load_table(const std::string& path) {
  std::ifstream f(path);
  if (!f) {
    std::fprintf(stderr, "cannot open %s\n", path.c_str());
    std::exit(2);
  }
  nlohmann::json j = nlohmann::json::parse(f);
  const auto batches = j.at("batches").get<std::vector<int>>();
  for (const auto& row : j.at("rows")) {
    const auto secs = row.at("seconds").get<std::vector<double>>();
    std::vector<BatchTimeSample> s;
    for (size_t i = 0; i < batches.size(); ++i) s.push_back({(double)batches[i], secs[i]});
    g_meas.fractions.push_back(row.at("resident_fraction").get<double>());
    g_meas.fits.push_back(fit_power_law(s));
    g_meas.samples.push_back(s);
  }
  g_meas.on = true;
}

double measured_seconds(double frac, int batch) {
  // rows bracketing frac; predict each at the batch, interpolate linearly in the fraction
  int lo = -1, hi = -1;
  for (size_t i = 0; i < g_meas.fractions.size(); ++i) {
    const double f = g_meas.fractions[i];
    if (f <= frac && (lo < 0 || f > g_meas.fractions[lo])) lo = (int)i;
    if (f >= frac && (hi < 0 || f < g_meas.fractions[hi])) hi = (int)i;
  }
  if (lo < 0) lo = hi;
  if (hi < 0) hi = lo;
  const double tl = predict(g_meas.fits[lo], batch), th = predict(g_meas.fits[hi], batch);
  const double fl = g_meas.fractions[lo], fh = g_meas.fractions[hi];
  if (fh == fl) return tl;
  return tl + (th - tl) * (frac - fl) / (fh - fl);
}

}  // namespace

extern "C" double __wrap__ZN6ragsim14retrieval_timeEiRKNS_15DatabaseProfileE(int resident, const DatabaseProfile& db) {
  const int batch = g_last_batch > 0 ? g_last_batch : g_default_batch;
  g_last_batch = 0;
  if (!g_use_measured) {
    ++g_calls_modelled;
    return __real__ZN6ragsim14retrieval_timeEiRKNS_15DatabaseProfileE(resident, db);
  }
  if (resident < 0 || resident > db.num_partitions)  // the reference's own argument check
    return __real__ZN6ragsim14retrieval_timeEiRKNS_15DatabaseProfileE(resident, db);
  ++g_calls_measured;
  return measured_seconds((double)resident / db.num_partitions, batch);
}

extern "C" int __wrap__ZN6ragsim22choose_retrieval_batchEii(int backlog, int max_batch) {
  const int take = __real__ZN6ragsim22choose_retrieval_batchEii(backlog, max_batch);
  g_last_batch = take;
  return take;
}

namespace {

nlohmann::json run_once(const Scenario& s, const std::vector<Request>& requests, std::uint64_t seed) {
  ProfilerOptions options;
  options.w_step = s.profiler.w_step;
  options.prefetch_mode = s.prefetch_mode;
  options.cost = s.cost;
  PolicyTable table =
      active_profile(s.hardware, s.model, s.database, s.profiler.probe_batches, s.profiler.partition_candidates, options);
  SimConfig cfg = make_sim_config(s, SimMode::Pipelined, seed);
  cfg.policy = table;
  SimOutcome out = run(requests, cfg);
  // retrieval-stage times per batch, from the trace
  std::vector<double> ret;
  for (const auto& t : out.traces) ret.push_back(t.retrieval_end - t.retrieval_start);
  std::sort(ret.begin(), ret.end());
  auto pct = [&](double p) { return ret.empty() ? 0.0 : percentile_nearest_rank(ret, p); };
  nlohmann::json entries = nlohmann::json::array();
  for (const auto& e : table.entries)
    entries.push_back({{"backlog_min", e.backlog_min}, {"gen_batch", e.config.gen_batch_size},
                       {"resident_partitions", e.config.resident_partitions}, {"w_gpu", e.config.w_gpu},
                       {"c_gpu", e.config.c_gpu}});
  return {{"latency", {{"average", out.aggregates.average}, {"p50", out.aggregates.p50}, {"p90", out.aggregates.p90},
                       {"p99", out.aggregates.p99}, {"max", out.aggregates.max}}},
          {"breakdown", {{"waiting", out.breakdown.waiting}, {"retrieval", out.breakdown.retrieval},
                         {"generation", out.breakdown.generation}}},
          {"retrieval_stage", {{"p50", pct(50)}, {"p99", pct(99)}, {"max", ret.empty() ? 0.0 : ret.back()}}},
          {"makespan", out.makespan}, {"requests", out.traces.size()}, {"policy", entries},
          {"report", metrics_report(out)}};
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s SCENARIO.json [SEED]\n", argv[0]);
    return 2;
  }
  const std::uint64_t seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
  Scenario s = load_scenario(argv[1]);
  g_default_batch = s.max_retrieval_batch;
  std::vector<Request> requests = generate_poisson(s.schedule, derive_seed(seed, 1), s.top_k);
  nlohmann::json out;
  out["scenario"] = argv[1];
  out["seed"] = seed;
  g_use_measured = false;
  out["modelled"] = run_once(s, requests, seed);
  out["modelled"]["retrieval_time_calls"] = g_calls_modelled;
  if (const char* t = std::getenv("RAGSIM_TRET")) {
    load_table(t);
    g_use_measured = true;
    out["measured"] = run_once(s, requests, seed);
    out["measured"]["retrieval_time_calls"] = g_calls_measured;
    out["measured"]["table"] = t;
    nlohmann::json fits = nlohmann::json::array();
    for (size_t i = 0; i < g_meas.fits.size(); ++i)
      fits.push_back({{"resident_fraction", g_meas.fractions[i]}, {"a", g_meas.fits[i].a}, {"c", g_meas.fits[i].c},
                      {"residual", g_meas.fits[i].residual}});
    out["measured"]["fits"] = fits;
  }
  std::printf("%s\n", out.dump(1).c_str());
  return 0;
}
