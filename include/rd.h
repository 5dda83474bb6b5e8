/*
 * rd.h — C-ABI of the RAGDoll retrieval stage: batched IVF-Flat search over an
 * inverted-list index that is partly resident in GPU memory (HBM) and partly
 * offloaded to pinned host DRAM.
 *
 * Two libraries implement this header:
 *   paper_2504_15302_b200/lib/librd_b200.so  — the B200 engine (product; sm_100a CUDA)
 *   oracle/librd_cpu.so                      — the CPU oracle (test infrastructure only)
 * so the engine is a literal drop-in for a CPU retrieval stage.
 *
 * What this replaces in the reference (/root/reference/proj):
 *   The reference (ragsim) has no search implementation; its retrieval stage is
 *   the closed-form cost `retrieval_time(P, db)` (core/src/cost_model.cpp:15-21,
 *   decl core/include/ragsim/cost_model.hpp:27-29), called by the retrieval
 *   worker (core/src/simulator.cpp:359, serial mode :560) and the profiler
 *   (core/src/scheduler.cpp:126). `rd_search` is the real computation whose
 *   measured wall time replaces that number. The reference's "index" is
 *   `DatabaseProfile` (core/include/ragsim/domain.hpp:57-68) and its placement
 *   knob is `PlacementConfig::resident_partitions` (domain.hpp:78): here a
 *   partition is an inverted list and residency is per list (rd_index_place).
 *
 * Conventions follow the reference:
 *   - status codes are the ragsim CLI exit codes (tools/main.cpp:30, 424-440;
 *     SPEC.md:540): 0 ok, 2 invalid argument / parse, 3 infeasible placement
 *     (ragsim::InfeasibleError, core/include/ragsim/errors.hpp:16-19),
 *     4 runtime (CUDA) failure. No exception crosses the ABI; the message of
 *     the last failure on the calling thread is in rd_last_error().
 *   - one in-flight search per handle (the single retrieval worker,
 *     SPEC.md:432); residency changes only between searches.
 *   - synthetic data derives from one master seed through ragsim's splitmix64
 *     Rng / derive_seed (core/include/ragsim/rng.hpp:12-56).
 *
 * Output ordering: per query ascending (distance, id); id = -1 and
 * distance = +inf pad when fewer than k candidates exist. Distances are squared
 * L2, the canonical exact value (see rd_exact_l2).
 */
#ifndef RD_H_
#define RD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RD_ABI_VERSION 1

/* Status codes (ragsim CLI exit codes, tools/main.cpp:30). */
#define RD_OK 0
#define RD_ERR_INVALID 2
#define RD_ERR_INFEASIBLE 3
#define RD_ERR_RUNTIME 4

/* Synthetic-data stream ids under the master seed. They avoid
 * the reference's own streams 1, 2 (tools/main.cpp:101,316) and
 * 0x100000000|n (core/src/simulator.cpp:204). */
#define RD_STREAM_CENTROIDS 0x1001u
#define RD_STREAM_ASSIGN 0x1002u
#define RD_STREAM_VECTOR_NOISE 0x1003u
#define RD_STREAM_QUERY_PICK 0x1004u
#define RD_STREAM_QUERY_NOISE 0x1005u
#define RD_STREAM_TRAIN_INIT 0x1006u
#define RD_DEFAULT_SEED 250415302ull

typedef struct rd_index rd_index; /* opaque, library-owned */

/* Counter-based synthetic knowledge base. Vector i belongs to list
 * a(i) = u(s_a, i) mod nlist and x_i[t] = c_{a(i)}[t] + sigma * f(s_x, i*d + t).
 * shard/num_shards row-stripe every list: shard g keeps rows
 * [g*len/G, (g+1)*len/G) of each list. */
typedef struct {
  int64_t n;          /* vectors in the whole (unsharded) knowledge base */
  int32_t d;          /* dimension */
  int32_t nlist;      /* inverted lists ("partitions") */
  uint64_t seed;      /* master seed */
  float sigma;        /* vector noise scale around its centroid (0.25) */
  int32_t shard;      /* this handle's stripe, 0 <= shard < num_shards */
  int32_t num_shards; /* 1 = unsharded */
} rd_synth_desc;

/* Placement between searches (reference analogue: PlacementConfig, domain.hpp:75-82).
 * Lists not resident live in pinned host memory and are streamed per search. The engine keeps the
 * resident rows as RD_STORE_F32_RESID (fp32 rows + bf16 residuals: 6 B per element + 4 B per row) when
 * every list stays resident within the budget (d % 128 == 0), else as RD_STORE_SPLIT3 (6 B per
 * element) when the tensor-core scan applies and the budget does not cut the resident set at that
 * size, else as fp32 (4 B per element: under a tight budget
 * residency beats scan speed, since every list left out streams over the host link per search).
 * Relayouts happen in place: the store grows or shrinks in chunks (<= 64 MiB) and never holds two
 * copies of a list; a 64 MiB conversion buffer is the only transient. Waits for searches in flight. */
typedef struct {
  uint64_t hbm_budget_bytes;     /* 0 = no byte budget; else covers resident lists plus (once any list
                                    is offloaded) a staging ring of >= 2 slots of
                                    max(largest list, 16384 rows), rows rounded up to 256 */
  double offload_fraction;       /* fraction of lists (by count) to offload; 0 = none */
  const uint8_t* resident_mask;  /* nullable; nlist bytes, 1 = HBM-resident. Overrides the two above */
  const uint32_t* list_heat;     /* nullable; nlist probe counts: hottest lists stay resident */
  int32_t staging_slots;         /* depth of the H2D staging ring; 0 = derive (queue_capacity rule) */
  int32_t reserved;
} rd_placement;

typedef struct {
  double seconds;               /* wall time of the call */
  uint64_t bytes_algorithmic;   /* unique probed lists' vectors + centroids + queries + results */
  uint64_t bytes_lists_resident;/* vector bytes of probed resident lists */
  uint64_t h2d_list_bytes;      /* vector bytes of probed offloaded lists streamed from host */
  uint64_t lists_probed;        /* unique lists probed by the batch */
  uint64_t tiles;               /* scan work items */
  uint64_t kernel_launches;     /* device kernels launched by this call */
  double scan_ms;               /* device time of the resident list-scan kernel (CUDA events; 0 unless
                                   rd_timing_stages is on) */
  double coarse_ms;             /* device time of coarse quantization + probe selection (likewise) */
  double offload_ms;            /* device time from first H2D to last offloaded scan */
  uint32_t margin_failures;     /* queries whose candidate margin could not be certified */
  uint32_t probe_failures;      /* queries whose probe set could not be certified */
} rd_search_stats;

typedef struct {
  int64_t n;            /* vectors held by this handle (its shard) */
  int32_t d, nlist;
  int64_t n_resident;   /* vectors resident in HBM */
  uint64_t hbm_bytes;   /* device bytes held by the index */
  uint64_t host_pinned_bytes;
  int32_t lists_resident;
  int32_t staging_slots;
  float max_norm;       /* max ||x|| over the index (used by the margin bound) */
  int32_t device;
  int32_t store;        /* resident-row format: RD_STORE_* (engine; the CPU oracle reports 0) */
  int32_t reserved;
} rd_index_info;
/* Resident-row formats. */
#define RD_STORE_F32 0          /* fp32 rows (FFMA scan, or the tensor-core scan converting on the fly) */
#define RD_STORE_F32_PRESPLIT 1 /* fp32 rows plus a bf16 (x1, x2) copy for the scan: 8 B per element */
#define RD_STORE_SPLIT3 2       /* the exact bf16 triple x = (x1 + x2) + x3 only: 6 B per element */
#define RD_STORE_F32_RESID 3    /* fp32 rows plus a bf16 residual plane r1 = bf16(x - c_list) for the scan
                                   (every list resident): 6 B per element, scan reads 2 */
#define RD_STORE_F32_RESID16 4  /* the same with an fp16 residual plane (default; RD_RES16=0 for bf16) */

/* LLM-side memory reservation for the retrieval GPU (C5). Mirrors
 * ragsim::ModelProfile (domain.hpp:37-55) and the PlacementConfig weight/KV
 * shares. Reservation = w_gpu*W + c_gpu*C(B) + H(B)*workspace_fraction
 * (core/src/memory_planner.cpp:20, decode workspace core/src/prefetch_timeline.cpp:85-86). */
typedef struct {
  uint64_t weight_total;
  uint64_t kv_bytes_per_request;
  uint64_t workspace_bytes_per_request;
  double w_gpu;
  double c_gpu;
  int32_t gen_batch_size;
  int32_t decode_phase;          /* 1: H(B) scaled by workspace_fraction (decode) */
  double workspace_fraction;     /* cost.decode_workspace_fraction (0.25) */
} rd_llm_reservation;

/* ---- library ---- */
const char* rd_last_error(void);
int rd_abi_version(void);
const char* rd_backend(void); /* "b200-sm100a" or "cpu-oracle" */

/* ---- index lifecycle (reference: DatabaseProfile, domain.hpp:57-68) ---- */
int rd_index_create_synthetic(const rd_synth_desc* desc, int32_t device, rd_index** out);
/* vectors: n x d row-major in list order; list_offsets: nlist+1 prefix offsets;
 * ids: nullable (default: row index). All host pointers, copied in. */
int rd_index_create_from_host(int64_t n, int32_t d, int32_t nlist, const float* vectors,
                              const int64_t* list_offsets, const float* centroids,
                              const int64_t* ids, int32_t device, rd_index** out);
int rd_index_place(rd_index* h, const rd_placement* placement);
int rd_index_info_get(const rd_index* h, rd_index_info* out);
/* Copies list_offsets (nlist+1) and optionally ids (n) / resident mask (nlist) to host. */
int rd_index_layout(const rd_index* h, int64_t* list_offsets, int64_t* ids, uint8_t* resident_mask);
/* Copies the nlist x d centroids to host. */
int rd_index_centroids(const rd_index* h, float* out);

/* IVF training from raw vectors (index build): Lloyd's k-means with exact,
 * deterministic arithmetic, so both libraries produce the same centroids and lists bit for bit:
 *   init    centroid j = the vector at row r_j, r_0, r_1, ... the first nlist distinct values of
 *           u(s, i) mod n for i = 0, 1, ... (s = rd_derive_seed(seed, RD_STREAM_TRAIN_INIT));
 *   assign  every vector to its nearest centroid by (canonical exact distance, centroid id),
 *           the order rd_probe uses;
 *   update  centroid = (fp64 sum of its members' components in ascending row order) / count,
 *           rounded to f32; an empty cluster keeps its centroid;
 * `iters` rounds of (assign, update), then a final assign; rows are laid out in list order,
 * ascending row within a list; ids default to the row index. Requires n >= nlist.
 * The engine assigns with its own coarse path (tensor-core GEMM + certified selection). */
int rd_index_build(int64_t n, int32_t d, int32_t nlist, const float* vectors, const int64_t* ids,
                   int32_t iters, uint64_t seed, int32_t device, rd_index** out);
void rd_index_destroy(rd_index* h);

/* ---- between-batch list migration ----
 * Reference analogue: the retrieval worker's partition reconfiguration between batches
 * (core/src/simulator.cpp:331-352), costed |dP| * M_p / bw by plan_transfer
 * (core/src/memory_planner.cpp:137-142), with loads gated behind weight shrinks
 * ("shrink before grow", core/src/simulator.cpp:323-326). Here a partition is an inverted list:
 * `demote` lists leave HBM first (copied to pinned host memory unless a host copy already exists:
 * host copies are write-once and kept), the remaining resident lists are compacted in place, then
 * `promote` lists are copied host -> HBM into the freed space, so the HBM footprint never exceeds
 * max(before, after). hbm_budget_bytes (0 = none) must cover the resident lists after the move
 * plus, while any list is offloaded, two staging slots of max(largest offloaded list, 16384 rows)
 * rounded up to 256 rows; otherwise RD_ERR_INFEASIBLE and nothing changes. Invalid ids, promoting
 * a resident list, demoting an offloaded one or naming a list twice: RD_ERR_INVALID.
 * Only between searches: waits for searches enqueued with rd_search_device first. With a budget, the
 * staging ring keeps as many slots (>= 2) as the budget leaves room for. */
typedef struct {
  double seconds;            /* wall time of the migration */
  uint64_t h2d_bytes;        /* promoted list bytes, pinned host -> HBM */
  uint64_t d2h_bytes;        /* demoted list bytes without a host copy yet, HBM -> pinned host */
  uint64_t d2d_bytes;        /* resident bytes moved by the in-place compaction (engine only) */
  int32_t lists_promoted;
  int32_t lists_demoted;
  uint64_t resident_bytes;   /* resident list bytes after the migration */
} rd_migration_stats;
int rd_index_migrate(rd_index* h, const int32_t* promote, int32_t n_promote, const int32_t* demote,
                     int32_t n_demote, uint64_t hbm_budget_bytes, rd_migration_stats* stats);

/* ---- on-disk index (format in include/rd_format.h, shared by both libraries) ----
 * save: every list in list order (resident lists from HBM, offloaded ones from pinned host memory).
 * load: header, offsets, ids and centroids, then the vectors streamed file -> pinned bounce
 * buffers -> HBM with the reads overlapped with the copies; the loaded index is fully resident.
 * Errors: RD_ERR_INVALID for a missing / malformed file, RD_ERR_RUNTIME for I/O or device failure. */
int rd_index_save(const rd_index* h, const char* path);
int rd_index_load(const char* path, int32_t device, rd_index** out);

/* ---- search (reference seam: retrieval_time, cost_model.cpp:15-21) ---- */
/* Host buffers: queries B x d row-major; out_ids / out_dists B x k. */
int rd_search(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t k,
              int64_t* out_ids, float* out_dists, rd_search_stats* stats);
/* Device buffers on the index's device, stream = cudaStream_t (NULL = legacy
 * default). Asynchronous: returns after enqueueing; stats device times are
 * filled only when sync != 0. With offloaded lists the host plans the staging
 * copies from the device plan, so the call returns once the plan is done (the
 * resident scan is already running). RD_ASYNC_TAIL=1 (set before the index is
 * created) returns at once instead: the caller's stream waits on a device gate
 * (cuStreamWaitValue32) that the index's worker thread releases — only safe
 * when that stream cannot share a hardware queue with the index's side
 * streams (CUDA_DEVICE_MAX_CONNECTIONS); otherwise the gate can deadlock.
 * CPU oracle: returns RD_ERR_INVALID. */
int rd_search_device(rd_index* h, const float* d_queries, int64_t B, int32_t nprobe, int32_t k,
                     int64_t* d_ids, float* d_dists, void* stream, int32_t sync,
                     rd_search_stats* stats);
/* Probe sets only (coarse quantization + selection): out_lists B x nprobe,
 * ascending (exact centroid distance, list id). */
int rd_probe(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t* out_lists);

/* ---- device-time accounting (CUDA events on each search's stream) ----
 * Every search records events around the whole chain. Per-stage events (the
 * coarse / scan / tail split) sit between kernels and cost the chain its
 * programmatic-dependent-launch overlap (~6 us per event at small batches), so
 * they are recorded only while rd_timing_stages(h, 1) is on (default off). */
typedef struct {
  int64_t searches; /* searches accounted since the last reset */
  double scan_ms;   /* summed device time of the resident list scan (N4) */
  double coarse_ms; /* summed device time of qnorm + N1 coarse + N2 select + N3 plan */
  double tail_ms;   /* summed device time after the resident scan: offload wait, N6/N7 merge */
  double total_ms;  /* summed device time of whole searches */
  int64_t stage_searches; /* of those, searches with per-stage events (scan/coarse/tail sums cover these) */
} rd_timing;
int rd_timing_stages(rd_index* h, int32_t on);
int rd_timing_reset(rd_index* h);
int rd_timing_read(rd_index* h, rd_timing* out); /* synchronizes the recorded searches */

/* ---- shard merge (multi-GPU) ----
 * G shard results, each B x k ascending, laid out [G][B][k]; writes the merged
 * per-query top-k ascending (distance, id). Host-side; used by rank 0. */
int rd_merge_topk(int32_t G, int64_t B, int32_t k, const int64_t* shard_ids,
                  const float* shard_dists, int64_t* out_ids, float* out_dists);
/* Device-side merge of [G][B][k] device buffers. CPU oracle: RD_ERR_INVALID. */
int rd_merge_topk_device(int32_t G, int64_t B, int32_t k, const int64_t* d_shard_ids,
                         const float* d_shard_dists, int64_t* d_out_ids, float* d_out_dists,
                         void* stream);

/* HBM read-stream peak of a device (GB/s), measured with the scan's load pattern (persistent
 * CTAs, 32 KiB bulk-copy stages, released on arrival) over `bytes` of device memory, best of 5 after
 * a warm-up: the denominator for a read-only kernel's roofline beside the copy bandwidth.
 * CPU oracle: RD_ERR_INVALID. */
int rd_device_read_bandwidth(int32_t device, uint64_t bytes, double* out_gbs);

/* ---- multi-GPU shard groups ----
 * north_star: "the lists shard across the GPUs of one 8xB200 box, each shard returns a local
 * top-k, and the results are merged with an NCCL gather over NVLink". A group holds G row stripes
 * of one knowledge base (stripe g = rows [g*len/G, (g+1)*len/G) of every list; rd_synth_desc
 * shard/num_shards, or any stripe handles the caller built), searches every stripe with the same
 * batch, gathers the per-stripe top-k to the root stripe's device (NCCL grouped send/recv; stripes
 * sharing one device gather by device copies, as NCCL admits one rank per device) and merges them
 * there by (distance, id). One call returns one merged result, which is what the reference's
 * retrieval worker consumes per batch (core/src/simulator.cpp:359, serial :560).
 * Two forms:
 *   - one process driving G devices: rd_group_create / rd_group_create_synthetic;
 *   - one process per device (e.g. torchrun): rank 0 calls rd_group_unique_id, the caller
 *     broadcasts the bytes, every rank calls rd_group_create_rank with its own stripe; rank 0 is
 *     the root and receives the merged result, other ranks receive their own stripe's top-k.
 * Group searches are collective in the second form: every rank calls with the same batch.
 * CPU oracle: the single-process forms search the stripes in turn and merge on the host;
 * rd_group_unique_id / rd_group_create_rank / rd_group_search_device return RD_ERR_INVALID. */
#define RD_GROUP_ID_BYTES 128
#define RD_GROUP_TRANSPORT_NONE 0 /* one stripe */
#define RD_GROUP_TRANSPORT_NCCL 1 /* NCCL send/recv to the root device */
#define RD_GROUP_TRANSPORT_COPY 2 /* device-to-device copies (stripes sharing a device; RD_GROUP_TRANSPORT=copy) */
typedef struct rd_group rd_group;
typedef struct {
  int32_t num_shards;   /* stripes in the whole group */
  int32_t local_shards; /* stripes driven by this process */
  int32_t rank, nranks; /* one process per device: this rank (root = 0); else 0, 1 */
  int32_t transport;    /* RD_GROUP_TRANSPORT_* */
  int32_t root_device;
  int64_t n;            /* vectors held by this process's stripes */
  int64_t n_resident;
} rd_group_info;
/* G stripe handles on any devices; the group owns them from a successful call on (destroying the
 * group destroys them). */
int rd_group_create(rd_index* const* shards, int32_t G, rd_group** out);
/* Stripe g of desc's knowledge base (desc->shard / num_shards ignored) on devices[g]. */
int rd_group_create_synthetic(const rd_synth_desc* desc, const int32_t* devices, int32_t G, rd_group** out);
int rd_group_unique_id(uint8_t* out /* RD_GROUP_ID_BYTES */);
/* This process's stripe (owned by the group from a successful call on) as rank `rank` of `nranks`. */
int rd_group_create_rank(rd_index* shard, const uint8_t* id, int32_t nranks, int32_t rank, rd_group** out);
int rd_group_info_get(const rd_group* g, rd_group_info* out);
/* Borrowed handle of the i-th local stripe (NULL if out of range): info, timing, migration. */
rd_index* rd_group_shard(rd_group* g, int32_t i);
/* rd_index_place on every local stripe (an HBM budget applies per device). */
int rd_group_place(rd_group* g, const rd_placement* placement);
/* Host buffers; stats sum the stripes' counters (device times: the slowest stripe). */
int rd_group_search(rd_group* g, const float* queries, int64_t B, int32_t nprobe, int32_t k,
                    int64_t* out_ids, float* out_dists, rd_search_stats* stats);
/* Device buffers on the root device (one process) or this rank's device, stream on that device. */
int rd_group_search_device(rd_group* g, const float* d_queries, int64_t B, int32_t nprobe, int32_t k,
                           int64_t* d_ids, float* d_dists, void* stream, int32_t sync, rd_search_stats* stats);
void rd_group_destroy(rd_group* g);

/* ---- synthetic data and canonical arithmetic (shared spec) ---- */
uint64_t rd_derive_seed(uint64_t master, uint64_t stream); /* rng.hpp:52-56 */
uint64_t rd_splitmix_at(uint64_t seed, uint64_t i);       /* (i+1)-th Rng(seed).next_u64(), rng.hpp:16-21 */
/* Queries b0..b0+B-1: q_b = x_{r(b)} + qsigma * f(s_qn, b*d+t), r(b) = u(s_q, b) mod n
 * (r over the unsharded knowledge base). src_ids nullable (B). */
int rd_synth_queries(const rd_synth_desc* desc, int64_t b0, int64_t B, float qsigma,
                     float* out_queries, int64_t* out_src_ids);
/* Vector x_id of the synthetic knowledge base (d floats). */
int rd_synth_vector(const rd_synth_desc* desc, int64_t id, float* out);
/* Canonical exact squared L2: eight fp64 residue-class sums over t mod 8, no
 * FMA contraction, combined ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)), rounded to f32. */
float rd_exact_l2(const float* a, const float* b, int32_t d);

/* ---- placement arithmetic (reference: memory_planner.cpp:12-35, prefetch_timeline.cpp:79-90) ---- */
int rd_llm_reservation_bytes(const rd_llm_reservation* r, double* out_bytes);
/* Staging-ring depth: max(1, floor(free_bytes / item_bytes)) (queue_capacity rule). */
int32_t rd_staging_depth(double free_bytes, double item_bytes);

#ifdef __cplusplus
}
#endif
#endif /* RD_H_ */
