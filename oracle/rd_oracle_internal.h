/* rd_oracle_internal.h — shared internals of the CPU library (TEST / BASELINE INFRASTRUCTURE, see
 * rd_oracle.c): the index object, the thread pool and the canonical exact distance, used by the
 * exact oracle (rd_oracle.c) and the batched CPU baseline (rd_cpu_batched.c). */
#pragma once
#include <stdint.h>

struct rd_index {
  int64_t n;
  int32_t d, nlist;
  float* vectors;   /* n x d, list order */
  int64_t* offsets; /* nlist + 1 */
  int64_t* ids;     /* n */
  float* centroids; /* nlist x d */
  uint8_t* resident;
  uint8_t* hostcopy; /* list has a (write-once) pinned host copy: offloaded at some point */
  float max_norm;
  /* batched baseline only (rd_cpu_prepare_batched): fp32 squared norms of rows / centroids */
  float* xnorm;
  float* cnorm;
  float cmax;
};

typedef void (*work_fn)(void* ctx, int64_t begin, int64_t end);
int rdo_threads(void);
void rdo_parallel_for(int64_t n, int64_t chunk, work_fn fn, void* ctx);
float rd_exact_l2(const float* a, const float* b, int32_t d);
