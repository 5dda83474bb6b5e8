// ref_harness.cpp — TEST INFRASTRUCTURE. Links the reference's own sources
// (compiled in place from /root/reference/proj/core/src by oracle/build_ref.sh,
// outputs only into oracle/_ref/) and prints golden vectors for the pieces of
// the reference this repo restates:
//   - ragsim::Rng / derive_seed         (core/include/ragsim/rng.hpp:12-56)
//   - ragsim::check_feasible gpu_used   (core/src/memory_planner.cpp:12-35)
//   - ragsim::queue_capacity            (core/src/prefetch_timeline.cpp:79-90)
//   - ragsim::retrieval_time            (core/src/cost_model.cpp:15-21)
//   - ragsim::fit_power_law / predict   (core/src/cost_model.cpp:97-136)
// The JSON it prints is committed as tests/golden/ref_golden.json.
#include <cinttypes>
#include <cstdio>
#include <vector>

#include "ragsim/cost_model.hpp"
#include "ragsim/domain.hpp"
#include "ragsim/memory_planner.hpp"
#include "ragsim/prefetch_timeline.hpp"
#include "ragsim/rng.hpp"
#include "ragsim/units.hpp"

using namespace ragsim;

int main() {
  std::printf("{\n  \"rng\": [\n");
  const std::uint64_t seeds[] = {0ull, 1ull, 250415302ull, 0xdeadbeefcafef00dull};
  bool first = true;
  for (std::uint64_t s : seeds) {
    Rng r(s);
    std::printf("%s    {\"seed\": \"%" PRIu64 "\", \"outputs\": [", first ? "" : ",\n", s);
    for (int i = 0; i < 16; ++i) std::printf("%s\"%" PRIu64 "\"", i ? ", " : "", r.next_u64());
    std::printf("]}");
    first = false;
  }
  std::printf("\n  ],\n  \"derive_seed\": [\n");
  const std::uint64_t masters[] = {250415302ull, 7ull};
  const std::uint64_t streams[] = {1, 2, 0x1001, 0x1002, 0x1003, 0x1004, 0x1005, 0x100000005ull};
  first = true;
  for (std::uint64_t m : masters)
    for (std::uint64_t st : streams) {
      std::printf("%s    {\"master\": \"%" PRIu64 "\", \"stream\": \"%" PRIu64 "\", \"seed\": \"%" PRIu64 "\"}",
                  first ? "" : ",\n", m, st, derive_seed(m, st));
      first = false;
    }

  // memory planner / queue capacity on reference-shaped profiles
  ModelProfile m8;  // configs/default_8b.json model block
  m8.num_layers = 32; m8.weight_total = 16 * GiB; m8.kv_bytes_per_request = 128 * MiB;
  m8.workspace_bytes_per_request = 64 * MiB; m8.output_tokens = 64;
  ModelProfile m70;  // configs/ref_70b.json model block
  m70.num_layers = 80; m70.weight_total = 140 * GiB; m70.kv_bytes_per_request = 256 * MiB;
  m70.workspace_bytes_per_request = 128 * MiB; m70.output_tokens = 64;
  DatabaseProfile db; db.num_partitions = 32; db.partition_bytes = 8 * GiB;
  db.search_seconds_per_partition = 0.5; db.load_seconds_per_partition = 5.5;
  HardwareProfile b200 = pf_high();
  b200.gpu_mem = 191502876672ll;  // B200 cudaMemGetInfo total seen on the box
  struct Case { const char* model; ModelProfile* m; HardwareProfile hw; double w_gpu, c_gpu; int batch; };
  std::vector<Case> cases = {
      {"8b", &m8, pf_high(), 0.75, 1.0, 32}, {"8b", &m8, pf_high(), 1.0, 1.0, 8},
      {"8b", &m8, pf_low(), 0.5, 0.5, 16},   {"70b", &m70, b200, 1.0, 1.0, 64},
      {"70b", &m70, b200, 0.5, 1.0, 48},     {"70b", &m70, pf_high(), 0.05, 0.0, 8},
      {"8b", &m8, b200, 1.0, 1.0, 64},       {"70b", &m70, b200, 0.8, 0.5, 1}};
  std::printf("\n  ],\n  \"placement\": [\n");
  first = true;
  for (auto& c : cases) {
    PlacementConfig cfg;
    cfg.w_gpu = c.w_gpu; cfg.w_cpu = 1.0 - c.w_gpu; cfg.c_gpu = c.c_gpu; cfg.c_cpu = 1.0 - c.c_gpu;
    cfg.resident_partitions = 8; cfg.gen_batch_size = c.batch;
    FeasibilityReport rep = check_feasible(cfg, c.hw, *c.m, db);
    int qp = queue_capacity(cfg, c.hw, *c.m, Phase::Prefill, 0.25);
    int qd = queue_capacity(cfg, c.hw, *c.m, Phase::Decode, 0.25);
    std::printf("%s    {\"model\": \"%s\", \"weight_total\": %lld, \"kv_bytes_per_request\": %lld, "
                "\"workspace_bytes_per_request\": %lld, \"num_layers\": %d, \"gpu_mem\": %lld, "
                "\"w_gpu\": %.17g, \"c_gpu\": %.17g, \"batch\": %d, \"gpu_used\": %.17g, "
                "\"gpu_slack\": %.17g, \"queue_capacity_prefill\": %d, \"queue_capacity_decode\": %d}",
                first ? "" : ",\n", c.model, (long long)c.m->weight_total,
                (long long)c.m->kv_bytes_per_request, (long long)c.m->workspace_bytes_per_request,
                c.m->num_layers, (long long)c.hw.gpu_mem, c.w_gpu, c.c_gpu, c.batch, rep.gpu_used,
                rep.gpu_slack, qp, qd);
    first = false;
  }
  std::printf("\n  ],\n  \"retrieval_time\": [");
  for (int p = 0; p <= 32; p += 8)
    std::printf("%s{\"resident\": %d, \"seconds\": %.17g}", p ? ", " : "", p, retrieval_time(p, db));
  // fit_power_law (cost_model.cpp:97-136) on sample sets: B200 measured T_ret rows
  // (profiles/round2_measured_tret.json, resident fractions 1.0 and 0.0), a decreasing set (exponent
  // clamped to 0), repeated batch sizes, two points
  const std::vector<std::vector<BatchTimeSample>> sets = {
      {{1, 0.000181}, {2, 0.000241}, {4, 0.000362}, {8, 0.000588}, {16, 0.000968}, {32, 0.001521}, {64, 0.002264}},
      {{1, 0.009134}, {2, 0.017783}, {4, 0.034356}, {8, 0.064310}, {16, 0.114713}, {32, 0.186829}, {64, 0.284393}},
      {{1, 4.0}, {2, 2.0}, {4, 1.0}},
      {{8, 0.1}, {8, 0.12}, {16, 0.2}, {64, 0.5}},
      {{1, 1e-3}, {1000, 2.0}}};
  std::printf("],\n  \"fit_power_law\": [");
  for (size_t i = 0; i < sets.size(); ++i) {
    const CostModelFit f = fit_power_law(sets[i]);
    std::printf("%s\n    {\"samples\": [", i ? "," : "");
    for (size_t j = 0; j < sets[i].size(); ++j)
      std::printf("%s[%.17g, %.17g]", j ? ", " : "", sets[i][j].batch_size, sets[i][j].seconds);
    std::printf("], \"a\": %.17g, \"c\": %.17g, \"residual\": %.17g, \"clamped\": %s, \"predict_256\": %.17g}",
                f.a, f.c, f.residual, f.exponent_clamped ? "true" : "false", predict(f, 256));
  }
  std::printf("\n  ]\n}\n");
  return 0;
}
