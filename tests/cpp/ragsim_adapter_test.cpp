// Test driver for include/rd_ragsim.hpp (the ragsim-side adapter). Linked against either
// implementation of rd.h: the CPU oracle (tests, no GPU) or the B200 engine (-m gpu tests).
// Prints one JSON line with the calibrated retrieval cost and exits 0 when every check holds.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "rd_ragsim.hpp"

using namespace ragsim::rd;

static int failures = 0;
#define EXPECT(c)                                                          \
  do {                                                                     \
    if (!(c)) {                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 20000;
  const int d = argc > 2 ? std::atoi(argv[2]) : 128;
  const int nlist = argc > 3 ? std::atoi(argv[3]) : 64;
  const int nreq = argc > 4 ? std::atoi(argv[4]) : 200;

  // R3: greedy drain
  EXPECT(choose_retrieval_batch(5, 64) == 5);
  EXPECT(choose_retrieval_batch(100, 64) == 64);
  EXPECT(throws<Error>([] { choose_retrieval_batch(0, 64); }));

  // R9: power-law fit
  {
    std::vector<BatchTime> s;
    for (int B : {1, 4, 16, 64}) s.push_back({(double)B, 2e-3 * std::pow((double)B, 0.5)});
    const PowerLawFit f = fit_power_law(s);
    EXPECT(std::fabs(f.a - 2e-3) < 1e-9 && std::fabs(f.c - 0.5) < 1e-9 && f.residual < 1e-9);
    EXPECT(std::fabs(f.predict(256) - 2e-3 * 16) < 1e-9);
    const PowerLawFit g = fit_power_law({{1, 4.0}, {2, 2.0}, {4, 1.0}});
    EXPECT(g.exponent_clamped && g.c == 0.0 && std::fabs(g.a - 2.0) < 1e-12);
    EXPECT(throws<Error>([] { fit_power_law({{1, 1.0}, {1, 2.0}}); }));
    EXPECT(throws<Error>([] { fit_power_law({{1, 1.0}, {2, -1.0}}); }));
  }

  // status -> exception mapping (tools/main.cpp:30)
  EXPECT(throws<ParseError>([] { RetrievalIndex::load("/nonexistent/kb.rdidx"); }));

  rd_synth_desc desc{n, d, nlist, RD_DEFAULT_SEED, 0.25f, 0, 1};
  RetrievalIndex idx = RetrievalIndex::synthetic(desc);
  std::vector<float> pool((size_t)nreq * d);
  std::vector<int64_t> src(nreq);
  check(rd_synth_queries(&desc, 0, nreq, 0.0625f, pool.data(), src.data()), "rd_synth_queries");
  EXPECT(throws<InfeasibleError>([&] { idx.migrate({}, {0}, /*budget=*/1024); }));
  EXPECT(throws<ParseError>([&] { idx.migrate({0}, {}); }));  // already resident

  // R4 + R6: the retrieval worker over real searches, with one between-batch reconfiguration
  std::vector<Request> reqs(nreq);
  double t = 0.0;
  const uint64_t s_arr = rd_derive_seed(RD_DEFAULT_SEED, 0x2001u);
  for (int i = 0; i < nreq; ++i) {  // exponential inter-arrivals, mean 50 us
    const double u = ((double)(rd_splitmix_at(s_arr, (uint64_t)i) >> 11) + 0.5) / 9007199254740992.0;
    t += -50e-6 * std::log(u);
    reqs[i].arrival = t;
    reqs[i].query = i;
  }
  RetrievalWorker worker(idx, pool.data(), d, /*nprobe=*/8, /*k=*/10, /*max_retrieval_batch=*/64);
  worker.reconfigure({}, {1, 2});
  const WorkerReport rep = worker.run(reqs);
  int correct = 0;
  for (const auto& r : reqs) {
    EXPECT(r.completed >= r.dispatched && r.dispatched >= r.arrival);
    correct += !r.ids.empty() && r.ids[0] == src[r.query];
  }
  EXPECT(correct == nreq);  // each query's source vector is its nearest neighbour
  // digest of every request's top-k ids (FNV-1a): the results do not depend on how the worker
  // batched them, so the engine-linked and oracle-linked drivers must print the same digest
  uint64_t digest = 1469598103934665603ull;
  for (const auto& r : reqs)
    for (int64_t id : r.ids)
      for (int byte = 0; byte < 8; ++byte) digest = (digest ^ ((uint64_t)id >> (8 * byte) & 0xffu)) * 1099511628211ull;
  for (int b : rep.batch_sizes) EXPECT(b >= 1 && b <= 64);
  EXPECT(rep.reconfig_seconds > 0.0 && idx.info().lists_resident == nlist - 2);

  // R2: the measured cost that replaces retrieval_time(P, db), for this placement
  MeasuredRetrievalCost cost(idx, pool, d, 8, 10);
  const PowerLawFit f = cost.calibrate({1, 8, 32, 64}, 3);
  EXPECT(f.a > 0.0 && f.samples == 4);
  std::printf("{\"backend\": \"%s\", \"requests\": %d, \"batches\": %d, \"makespan_s\": %.6g, "
              "\"busy_s\": %.6g, \"reconfig_s\": %.6g, \"t_ret_fit\": {\"a\": %.6g, \"c\": %.4f, \"residual\": %.4f}, "
              "\"t_ret_64_s\": %.6g, \"results_digest\": \"%016llx\", \"failures\": %d}\n",
              rd_backend(), nreq, rep.batches, rep.makespan, rep.busy_seconds, rep.reconfig_seconds, f.a, f.c,
              f.residual, cost.seconds(64), (unsigned long long)digest, failures);
  return failures ? 1 : 0;
}
