// peak.cu — the HBM read-stream peak of this device, measured the way the list scan reads: persistent
// CTAs (one per SM), a 4-deep ring of 32 KiB shared-memory stages filled by 1D bulk (TMA) copies of
// consecutive chunks from a dynamic queue, released as soon as they land. bench.py reports the scan's
// roofline fraction against this figure beside the (read + write) copy bandwidth of
// MEASURED_PEAKS.json: a pure read stream runs above a copy's rate on HBM3e.
#include <chrono>

#include "host.cuh"

namespace {

constexpr int kPkStages = 4, kPkChunk = 32 * 1024;

__global__ void __launch_bounds__(64, 1) read_stream_kernel(const char* src, long long nchunks, unsigned* counter,
                                                            unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char ring_raw[];  // kPkStages x kPkChunk
  auto ring = reinterpret_cast<unsigned char(*)[kPkChunk]>(ring_raw);
  __shared__ uint64_t full[kPkStages], empty[kPkStages];
  __shared__ unsigned long long issued;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPkStages; ++i) {
      rd::mbar_init(&full[i], 1);
      rd::mbar_init(&empty[i], 1);
    }
    rd::fence_mbar_init();
    issued = ~0ull;
  }
  __syncthreads();
  if (warp == 0 && lane == 0) {  // producer
    uint32_t u = 0;
    for (;;) {
      const long long c = atomicAdd(counter, 1u);
      if (c >= nchunks) break;
      const int s = u % kPkStages;
      rd::mbar_wait(&empty[s], ((u / kPkStages) & 1) ^ 1);
      rd::mbar_arrive_expect_tx(&full[s], kPkChunk);
      rd::bulk_g2s(ring[s], src + (size_t)c * kPkChunk, kPkChunk, &full[s]);
      ++u;
    }
    *(volatile unsigned long long*)&issued = u;
  } else if (warp == 1 && lane == 0) {  // consumer: wait, touch one byte, release
    unsigned long long acc = 0;
    for (uint32_t u = 0;; ++u) {
      const int s = u % kPkStages;
      for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(rd::smem_u32(&full[s])), "r"((u / kPkStages) & 1)
            : "memory");
        if (ok) break;
        const unsigned long long n = *(volatile unsigned long long*)&issued;
        if (n != ~0ull && u >= n) goto done;
      }
      acc += ring[s][u & 127];
      rd::mbar_arrive(&empty[s]);
    }
  done:
    sink[blockIdx.x] = acc;
  }
}

}  // namespace

extern "C" int rd_device_read_bandwidth(int32_t device, uint64_t bytes, double* out_gbs) {
  return guarded([&] {
    if (!out_gbs || bytes < (uint64_t)kPkChunk * 1024) throw_rd(RD_ERR_INVALID, "read bandwidth: >= 32 MiB and an output");
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const long long nchunks = (long long)(bytes / kPkChunk);
    DBuf<char> buf;
    buf.alloc((size_t)nchunks * kPkChunk);
    CK(cudaMemset(buf.p, 1, (size_t)nchunks * kPkChunk));
    DBuf<unsigned> counter;
    counter.alloc(1);
    DBuf<unsigned long long> sink;
    sink.alloc((size_t)sms);
    CK(rd::ensure_smem(reinterpret_cast<const void*>(read_stream_kernel), kPkStages * kPkChunk));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best = 0.0;
    for (int rep = 0; rep < 6; ++rep) {  // the first is a warm-up
      CK(cudaMemset(counter.p, 0, sizeof(unsigned)));
      CK(cudaEventRecord(e0));
      read_stream_kernel<<<sms, 64, kPkStages * kPkChunk>>>(buf.p, nchunks, counter.p, sink.p);
      CK(cudaGetLastError());
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0) best = std::max(best, (double)nchunks * kPkChunk / (ms * 1e-3) / 1e9);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out_gbs = best;
  });
}
