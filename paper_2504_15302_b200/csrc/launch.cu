// launch.cu — launch policy shared by every search kernel (see launch_k in ivf_kernels.cuh):
// programmatic dependent launch on/off, and the per-(device, kernel) dynamic shared-memory limit.
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "ivf_kernels.cuh"

namespace rd {

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("RD_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is raised whenever a launch needs more than the kernel
// was last configured for on this device: dynamic + static smem can exceed the 48 KiB default even
// when the dynamic part alone does not, so there is no "small enough" shortcut.
cudaError_t ensure_smem(const void* kern, size_t smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> configured;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = configured[{dev, kern}];
  if (smem > cur) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cur = smem;
  }
  return cudaSuccess;
}

}  // namespace rd
