// End-to-end latency of rd_search through the C ABI from C++ (how a ragsim retrieval worker calls
// it: host queries in, host ids / distances out, one blocking call per batch), without the Python
// binding in the way. C2 knowledge base (10M x 768, nlist 4096, nprobe 64, k 10), page-locked host
// buffers. Prints one line per batch size: p50 / p90 latency and queries/s at p50.
// Build: make tools/e2e_latency   Run: tools/e2e_latency [reps]
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rd.h"

static void check(int rc, const char* what) {
  if (rc != RD_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, rd_last_error());
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 50;
  rd_synth_desc desc{10'000'000, 768, 4096, 250415302ull, 0.25f, 0, 1};
  rd_index* idx = nullptr;
  check(rd_index_create_synthetic(&desc, 0, &idx), "create");
  const int nprobe = 64, k = 10, d = desc.d;
  const int batches[] = {1, 2, 8, 32, 64, 256, 1024};
  const int bmax = 1024, pool = 8;  // 8 pre-generated batches, cycled: back-to-back calls
  float* q = nullptr;
  int64_t* ids = nullptr;
  float* dists = nullptr;
  // portable: page-locked for every CUDA context (the engine links its own static runtime)
  const unsigned fl = cudaHostAllocPortable;
  if (cudaHostAlloc(&q, sizeof(float) * pool * bmax * d, fl) != cudaSuccess ||
      cudaHostAlloc(&ids, sizeof(int64_t) * bmax * k, fl) != cudaSuccess ||
      cudaHostAlloc(&dists, sizeof(float) * bmax * k, fl) != cudaSuccess) {
    std::fprintf(stderr, "cudaHostAlloc failed\n");
    return 1;
  }
  std::printf("rd_search from C++ (page-locked host buffers), C2: 10M x 768, nlist 4096, nprobe 64, k 10\n");
  for (int B : batches) {
    std::vector<double> us;
    for (int i = 0; i < pool; ++i)
      check(rd_synth_queries(&desc, 1'000'000 + (int64_t)i * B, B, 0.0625f, q + (size_t)i * bmax * d, nullptr),
            "queries");
    for (int r = -3; r < reps; ++r) {  // 3 warm-up calls
      const float* qb = q + (size_t)((r + 3) % pool) * bmax * d;
      const auto t0 = std::chrono::steady_clock::now();
      check(rd_search(idx, qb, B, nprobe, k, ids, dists, nullptr), "search");
      const auto t1 = std::chrono::steady_clock::now();
      if (r >= 0) us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    std::sort(us.begin(), us.end());
    const double p50 = us[us.size() / 2], p90 = us[us.size() * 9 / 10];
    std::printf("B=%5d  p50 %9.1f us  p90 %9.1f us  %10.0f queries/s at p50\n", B, p50, p90, B / (p50 * 1e-6));
  }
  rd_index_destroy(idx);
  cudaFreeHost(q);
  cudaFreeHost(ids);
  cudaFreeHost(dists);
  return 0;
}
