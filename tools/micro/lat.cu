// Microbenchmark: dependent-latency of DADD / DMUL / F2F.F64.F32 / LDS on sm_100a (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const float* x, double* out, long long* cyc, int n) {
  __shared__ float sx[1024];
  __shared__ double sq[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sx[i] = x[i]; sq[i] = x[i] * 0.5; }
  __syncthreads();
  double s = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, 1.0000001);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) s = __dmul_rn(s, 0.9999999);
  long long t2 = clock64();
  float f = (float)s;
  for (int i = 0; i < n; ++i) { double d = (double)f; f = (float)(d * 1.0000001); }
  long long t3 = clock64();
  // canonical exact inner loop from smem, one lane chain of n elements
  double a = 0;
  int j = threadIdx.x & 7;
  for (int t = j; t < 8 * n; t += 8) { double df = __dsub_rn(sq[t & 1023], (double)sx[t & 1023]); a = __dadd_rn(a, __dmul_rn(df, df)); }
  long long t4 = clock64();
  out[threadIdx.x] = s + f + a;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  float* x; double* o; long long* c;
  cudaMalloc(&x, 4096 * 4); cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  cudaMemset(x, 0, 4096 * 4);
  for (int threads : {32, 256, 1024}) {
    for (int rep = 0; rep < 2; ++rep) k<<<1, threads>>>(x, o, c, 96);
    cudaDeviceSynchronize();
    printf("threads=%4d per-op cycles: dadd %.1f dmul %.1f f2f+mul+f2f %.1f canon-elem %.1f\n", threads, c[0] / 96.0,
           c[1] / 96.0, c[2] / 96.0, c[3] / 96.0);
  }
  return 0;
}
