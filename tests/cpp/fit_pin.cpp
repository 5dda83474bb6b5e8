// Test driver: include/rd_ragsim.hpp's fit_power_law / predict on the samples given as arguments
// ("B,seconds" pairs), printed as JSON for tests/test_golden_reference.py to compare with the
// reference's own fit (tests/golden/ref_golden.json "fit_power_law", cost_model.cpp:97-136).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rd_ragsim.hpp"

int main(int argc, char** argv) {
  std::vector<ragsim::rd::BatchTime> s;
  for (int i = 1; i < argc; ++i) {
    char* end = nullptr;
    const double b = std::strtod(argv[i], &end);
    const double t = std::strtod(end + 1, nullptr);
    s.push_back({b, t});
  }
  const ragsim::rd::PowerLawFit f = ragsim::rd::fit_power_law(s);
  std::printf("{\"a\": %.17g, \"c\": %.17g, \"residual\": %.17g, \"clamped\": %s, \"predict_256\": %.17g}\n", f.a, f.c,
              f.residual, f.exponent_clamped ? "true" : "false", f.predict(256));
  return 0;
}
