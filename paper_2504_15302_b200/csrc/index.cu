// index.cu — index lifecycle behind include/rd.h: creation (synthetic, host arrays, file,
// IVF training), placement (N8), between-batch migration, save / load, introspection, and the
// placement arithmetic shared with the reference (memory_planner.cpp, prefetch_timeline.cpp).
#include "host.cuh"

thread_local std::string g_err;

extern "C" {

const char* rd_last_error(void) { return g_err.c_str(); }
int rd_abi_version(void) { return RD_ABI_VERSION; }
const char* rd_backend(void) { return "b200-sm100a"; }

uint64_t rd_splitmix_at(uint64_t seed, uint64_t i) { return rd::splitmix_at(seed, i); }
uint64_t rd_derive_seed(uint64_t master, uint64_t stream) { return derive_seed(master, stream); }

float rd_exact_l2(const float* a, const float* b, int32_t d) {
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int32_t t = 0; t < d; ++t) {
    volatile double df = (double)a[t] - (double)b[t];  // volatile: no contraction into an FMA
    volatile double sq = df * df;
    s[t & 7] = s[t & 7] + sq;
  }
  return (float)(((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7])));
}

static void validate_desc(const rd_synth_desc* s) {
  if (!s) throw_rd(RD_ERR_INVALID, "null synth descriptor");
  if (s->n < 1 || s->d < 1 || s->nlist < 1) throw_rd(RD_ERR_INVALID, "synth: n, d, nlist must be >= 1");
  if (s->num_shards < 1 || s->shard < 0 || s->shard >= s->num_shards)
    throw_rd(RD_ERR_INVALID, "synth: shard %d of %d out of range", s->shard, s->num_shards);
}

static void synth_vec_host(const rd_synth_desc* s, uint64_t sc, uint64_t sa, uint64_t sx, int64_t id, float* out) {
  const int a = (int)(rd::splitmix_at(sa, (uint64_t)id) % (uint64_t)s->nlist);
  for (int t = 0; t < s->d; ++t) {
    volatile float noise = s->sigma * rd::unif(sx, (uint64_t)id * s->d + t);
    out[t] = rd::unif(sc, (uint64_t)a * s->d + t) + noise;
  }
}

int rd_synth_vector(const rd_synth_desc* s, int64_t id, float* out) {
  return guarded([&] {
    validate_desc(s);
    if (id < 0 || id >= s->n || !out) throw_rd(RD_ERR_INVALID, "synth_vector: id out of range");
    synth_vec_host(s, derive_seed(s->seed, RD_STREAM_CENTROIDS), derive_seed(s->seed, RD_STREAM_ASSIGN),
                   derive_seed(s->seed, RD_STREAM_VECTOR_NOISE), id, out);
  });
}

int rd_synth_queries(const rd_synth_desc* s, int64_t b0, int64_t B, float qsigma, float* out, int64_t* src) {
  return guarded([&] {
    validate_desc(s);
    if (b0 < 0 || B < 0 || (B > 0 && !out)) throw_rd(RD_ERR_INVALID, "synth_queries: invalid arguments");
    const uint64_t sc = derive_seed(s->seed, RD_STREAM_CENTROIDS), sa = derive_seed(s->seed, RD_STREAM_ASSIGN),
                   sx = derive_seed(s->seed, RD_STREAM_VECTOR_NOISE),
                   sq = derive_seed(s->seed, RD_STREAM_QUERY_PICK), sn = derive_seed(s->seed, RD_STREAM_QUERY_NOISE);
    parallel_for(B * 64, [&](long long lo, long long hi) {
      for (long long i = (lo + 63) / 64; i < (hi + 63) / 64 && i < B; ++i) {
        const int64_t b = b0 + i;
        const int64_t r = (int64_t)(rd::splitmix_at(sq, (uint64_t)b) % (uint64_t)s->n);
        float* q = out + i * s->d;
        synth_vec_host(s, sc, sa, sx, r, q);
        for (int t = 0; t < s->d; ++t) {
          volatile float noise = qsigma * rd::unif(sn, (uint64_t)b * s->d + t);
          q[t] = q[t] + noise;
        }
        if (src) src[i] = r;
      }
    });
  });
}

int rd_index_create_synthetic(const rd_synth_desc* s, int32_t device, rd_index** out) {
  return guarded([&] {
    validate_desc(s);
    check_dims(s->d);
    if (!out) throw_rd(RD_ERR_INVALID, "null out");
    auto h = new_index(device);
    h->d = s->d;
    h->nlist = s->nlist;
    const long long n = s->n;
    const int nl = s->nlist, G = s->num_shards, g = s->shard;
    const uint64_t sa = derive_seed(s->seed, RD_STREAM_ASSIGN);
    // list membership on the host (counting sort, ids ascending within a list)
    std::vector<int32_t> assign(n);
    parallel_for(n, [&](long long lo, long long hi) {
      for (long long i = lo; i < hi; ++i) assign[i] = (int32_t)(rd::splitmix_at(sa, (uint64_t)i) % (uint64_t)nl);
    });
    std::vector<long long> full_len(nl, 0);
    for (long long i = 0; i < n; ++i) full_len[assign[i]]++;
    h->list_off.assign(nl + 1, 0);
    for (int l = 0; l < nl; ++l) {
      const long long lo = g * full_len[l] / G, hi = (long long)(g + 1) * full_len[l] / G;
      h->list_off[l + 1] = h->list_off[l] + (hi - lo);
    }
    h->n = h->list_off[nl];
    std::vector<long long> ids(std::max(1LL, h->n));
    {
      std::vector<long long> cursor(nl, 0);
      for (long long i = 0; i < n; ++i) {
        const int l = assign[i];
        const long long pos = cursor[l]++;
        const long long lo = g * full_len[l] / G, hi = (long long)(g + 1) * full_len[l] / G;
        if (pos >= lo && pos < hi) ids[h->list_off[l] + (pos - lo)] = i;
      }
    }
    std::vector<int32_t>().swap(assign);
    h->centroids.alloc((size_t)nl * h->d);
    h->cnorm.alloc(nl);
    CK(rd::launch_gen_centroids(h->centroids.p, nl, h->d, derive_seed(s->seed, RD_STREAM_CENTROIDS), 0));
    h->d_ids.alloc(h->n);
    CK(cudaMemcpy(h->d_ids.p, ids.data(), sizeof(long long) * h->n, cudaMemcpyHostToDevice));
    const uint64_t sx = derive_seed(s->seed, RD_STREAM_VECTOR_NOISE);
    const float sigma = s->sigma;
    rd_index* hp = h.get();
    h->materialize([&](long long r0, long long c, float* dst) {
      CK(rd::launch_gen_vectors(dst, hp->d_ids.p + r0, c, hp->d, nl, hp->centroids.p, sa, sx, sigma, 0));
    });
    *out = h.release();
  });
}

int rd_index_create_from_host(int64_t n, int32_t d, int32_t nlist, const float* vectors, const int64_t* list_offsets,
                              const float* centroids, const int64_t* ids, int32_t device, rd_index** out) {
  return guarded([&] {
    if (n < 0 || nlist < 1 || !list_offsets || !centroids || !out || (n > 0 && !vectors))
      throw_rd(RD_ERR_INVALID, "create_from_host: invalid arguments");
    check_dims(d);
    if (list_offsets[0] != 0 || list_offsets[nlist] != n)
      throw_rd(RD_ERR_INVALID, "create_from_host: list_offsets must run 0..n");
    for (int l = 0; l < nlist; ++l)
      if (list_offsets[l + 1] < list_offsets[l])
        throw_rd(RD_ERR_INVALID, "create_from_host: list_offsets not monotone at %d", l);
    if (n >= (1LL << 31)) throw_rd(RD_ERR_INVALID, "create_from_host: at most 2^31-1 vectors per handle");
    auto h = new_index(device);
    h->n = n;
    h->d = d;
    h->nlist = nlist;
    h->list_off.assign(list_offsets, list_offsets + nlist + 1);
    h->centroids.alloc((size_t)nlist * d);
    h->cnorm.alloc(nlist);
    CK(cudaMemcpy(h->centroids.p, centroids, sizeof(float) * (size_t)nlist * d, cudaMemcpyHostToDevice));
    h->d_ids.alloc(n);
    std::vector<long long> idv(std::max<int64_t>(1, n));
    for (long long i = 0; i < n; ++i) idv[i] = ids ? ids[i] : i;
    CK(cudaMemcpy(h->d_ids.p, idv.data(), sizeof(long long) * n, cudaMemcpyHostToDevice));
    h->materialize([&](long long r0, long long c, float* dst) {
      CK(cudaMemcpy(dst, vectors + (size_t)r0 * d, sizeof(float) * (size_t)c * d, cudaMemcpyHostToDevice));
    });
    *out = h.release();
  });
}

void rd_index_destroy(rd_index* h) { delete h; }

int rd_index_centroids(const rd_index* h, float* out) {
  return guarded([&] {
    if (!h || !out) throw_rd(RD_ERR_INVALID, "centroids: null argument");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpy(out, h->centroids.p, sizeof(float) * (size_t)h->nlist * h->d, cudaMemcpyDeviceToHost));
  });
}

// ---------------------------------------------------------------- IVF training (N10)
// Lloyd's k-means, exact and deterministic (include/rd.h, rd_index_build): assignment is the
// search's own coarse path with nprobe = 1 — tensor-core (or FFMA) distances, certified selection,
// canonical fp64 distances for ambiguous centroids — over batches of the vectors; the update is
// train.cu's ordered fp64 mean.
int rd_index_build(int64_t n, int32_t d, int32_t nlist, const float* vectors, const int64_t* ids, int32_t iters,
                   uint64_t seed, int32_t device, rd_index** out) {
  return guarded([&] {
    if (n < 1 || nlist < 1 || n < nlist || iters < 0 || !vectors || !out)
      throw_rd(RD_ERR_INVALID, "build: need n >= nlist >= 1, iters >= 0 and vectors");
    check_dims(d);
    if (n >= (1LL << 31)) throw_rd(RD_ERR_INVALID, "build: at most 2^31-1 vectors per handle");
    auto h = new_index(device);
    h->n = n;
    h->d = d;
    h->nlist = nlist;
    cudaStream_t s = 0;
    DBuf<float> X;  // input order
    X.alloc((size_t)n * d);
    CK(cudaMemcpy(X.p, vectors, sizeof(float) * (size_t)n * d, cudaMemcpyHostToDevice));
    {  // init: the first nlist distinct rows of u(s, i) mod n
      const uint64_t si = derive_seed(seed, RD_STREAM_TRAIN_INIT);
      std::vector<uint8_t> taken((size_t)n, 0);
      std::vector<int> pick;
      for (uint64_t i = 0; (int)pick.size() < nlist; ++i) {
        const long long r = (long long)(rd::splitmix_at(si, i) % (uint64_t)n);
        if (!taken[r]) {
          taken[r] = 1;
          pick.push_back((int)r);
        }
      }
      DBuf<int> dpick;
      dpick.alloc(nlist);
      CK(cudaMemcpy(dpick.p, pick.data(), sizeof(int) * nlist, cudaMemcpyHostToDevice));
      h->centroids.alloc((size_t)nlist * d);
      CK(rd::launch_gather_rows(X.p, dpick.p, nlist, d, h->centroids.p, s));
    }
    DBuf<int> assign, keys_sorted, rows, rows_sorted;
    DBuf<unsigned> counts;
    DBuf<long long> seg;
    DBuf<char> temp;
    assign.alloc(n);
    keys_sorted.alloc(n);
    rows.alloc(n);
    rows_sorted.alloc(n);
    counts.alloc(nlist);
    seg.alloc(nlist + 1);
    int end_bit = 1;
    while ((1LL << end_bit) < nlist) ++end_bit;
    size_t temp_bytes = 0;
    CK(rd::sort_pairs(nullptr, nullptr, nullptr, nullptr, n, end_bit, nullptr, &temp_bytes, s));
    temp.alloc(temp_bytes);
    std::vector<unsigned> hcount(nlist);
    std::vector<long long> hseg(nlist + 1);
    auto& w = h->ws;
    const long long chunk = std::max<long long>(1024, std::min<long long>(65536, (1LL << 28) / nlist));
    auto assign_all = [&] {
      h->prepare_centroids();
      w.qnorm.ensure(chunk);
      w.qsplit.ensure((size_t)chunk * d);
      w.Dc.ensure((size_t)chunk * nlist);
      w.blk.ensure(kStatBytes);
      for (long long b0 = 0; b0 < n; b0 += chunk) {
        const int B = (int)std::min(chunk, n - b0);
        const float* q = X.p + (size_t)b0 * d;
        CK(rd::launch_qprep(rd::QprepArgs{q, B, d, w.qnorm.p, d % 64 == 0 ? w.qsplit.p : nullptr, w.fails(), nullptr},
                            s));
        if (d % 64 == 0) {
          const CUtensorMap qmap = make_split_map(w.qsplit.p, B, d);
          CK(rd::launch_coarse_tc(qmap, h->cmap, h->cnorm.p, w.Dc.p, B, nlist, d, s));
        } else {
          CK(rd::launch_coarse(q, h->centroids.p, h->cnorm.p, w.Dc.p, B, nlist, d, s));
        }
        rd::SelectParams sp{w.Dc.p, q, w.qnorm.p, h->centroids.p, assign.p + b0, w.fails(), B, nlist, 1, d,
                            h->cmax, nullptr, nullptr, nullptr, 0.f, nullptr, 0};
        sp.gamma_coarse = d % 64 == 0 ? rd::gamma_bf16x3(d) : rd::gamma_ffma_coarse(d);
        CK(rd::launch_select(sp, false, s, h->num_sms));
      }
    };
    auto group = [&] {  // rows stably sorted by cluster; per-cluster segments
      CK(rd::launch_iota(rows.p, n, s));
      CK(rd::sort_pairs(assign.p, keys_sorted.p, rows.p, rows_sorted.p, n, end_bit, temp.p, &temp_bytes, s));
      CK(rd::launch_histogram(assign.p, n, counts.p, nlist, s));
      CK(cudaMemcpyAsync(hcount.data(), counts.p, sizeof(unsigned) * nlist, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      hseg[0] = 0;
      for (int l = 0; l < nlist; ++l) hseg[l + 1] = hseg[l] + hcount[l];
      CK(cudaMemcpy(seg.p, hseg.data(), sizeof(long long) * (nlist + 1), cudaMemcpyHostToDevice));
    };
    for (int it = 0; it < iters; ++it) {
      assign_all();
      group();
      CK(rd::launch_centroid_update(X.p, rows_sorted.p, seg.p, nlist, d, h->centroids.p, s));
    }
    assign_all();
    group();
    // list-order layout
    h->list_off = hseg;
    DBuf<long long> uids;
    if (ids) {
      uids.alloc(n);
      CK(cudaMemcpy(uids.p, ids, sizeof(long long) * (size_t)n, cudaMemcpyHostToDevice));
    }
    h->d_ids.alloc(n);
    CK(rd::launch_gather_ids(ids ? uids.p : nullptr, rows_sorted.p, n, h->d_ids.p, s));
    CK(cudaStreamSynchronize(s));
    h->materialize([&](long long r0, long long c, float* dst) {
      CK(rd::launch_gather_rows(X.p, rows_sorted.p + r0, c, d, dst, s));
    });
    X.reset();
    *out = h.release();
  });
}

// ---------------------------------------------------------------- on-disk index (include/rd_format.h)
namespace {

void pwrite_all(int fd, const void* p, size_t bytes, uint64_t off, const char* path) {
  const char* b = static_cast<const char*>(p);
  while (bytes) {
    const ssize_t w = ::pwrite(fd, b, bytes, (off_t)off);
    if (w <= 0) throw_rd(RD_ERR_RUNTIME, "save: write to %s failed", path);
    b += w;
    off += (uint64_t)w;
    bytes -= (size_t)w;
  }
}
void pread_all(int fd, void* p, size_t bytes, uint64_t off, const char* path) {
  char* b = static_cast<char*>(p);
  while (bytes) {
    const ssize_t r = ::pread(fd, b, bytes, (off_t)off);
    if (r <= 0) throw_rd(RD_ERR_RUNTIME, "load: read from %s failed", path);
    b += r;
    off += (uint64_t)r;
    bytes -= (size_t)r;
  }
}
struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};
constexpr size_t kIoChunk = size_t(64) << 20;  // pinned bounce buffer (bytes)

}  // namespace

int rd_index_save(const rd_index* h, const char* path) {
  return guarded([&] {
    if (!h || !path) throw_rd(RD_ERR_INVALID, "save: null argument");
    CK(cudaSetDevice(h->device));
    const_cast<rd_index*>(h)->tail_wait();
    CK(cudaDeviceSynchronize());
    rd_file_header hd;
    rd_fmt_layout(&hd, h->n, h->d, h->nlist);
    hd.check = rd_fmt_check(&hd, reinterpret_cast<const int64_t*>(h->list_off.data()));
    Fd f;
    f.fd = ::open(path, O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) throw_rd(RD_ERR_RUNTIME, "save: cannot open %s for writing", path);
    std::vector<char> head(RD_FILE_ALIGN, 0);
    std::memcpy(head.data(), &hd, sizeof hd);
    pwrite_all(f.fd, head.data(), head.size(), 0, path);
    pwrite_all(f.fd, h->list_off.data(), 8 * (size_t)(h->nlist + 1), hd.off_list_offsets, path);
    {
      std::vector<long long> ids(std::max<long long>(1, h->n));
      if (h->n) CK(cudaMemcpy(ids.data(), h->d_ids.p, 8 * (size_t)h->n, cudaMemcpyDeviceToHost));
      pwrite_all(f.fd, ids.data(), 8 * (size_t)h->n, hd.off_ids, path);
      std::vector<float> c((size_t)h->nlist * h->d);
      CK(cudaMemcpy(c.data(), h->centroids.p, 4 * c.size(), cudaMemcpyDeviceToHost));
      pwrite_all(f.fd, c.data(), 4 * c.size(), hd.off_centroids, path);
    }
    // vectors in list order, gathered from HBM (resident lists) or pinned host memory (offloaded)
    HBuf<float> bounce;
    const size_t row_bytes = 4 * (size_t)h->d;
    const long long chunk_rows = std::max<long long>(1, (long long)(kIoChunk / row_bytes));
    bounce.alloc((size_t)chunk_rows * h->d);
    long long fill = 0, row = 0;  // rows in the bounce buffer; global row of its first row
    auto flush = [&] {
      if (!fill) return;
      pwrite_all(f.fd, bounce.p, (size_t)fill * row_bytes, hd.off_vectors + (uint64_t)row * row_bytes, path);
      row += fill;
      fill = 0;
    };
    DBuf<float> conv;  // resident rows in fp32 (the split3 store rebuilt by join3)
    if (h->split3) conv.alloc((size_t)std::min(chunk_rows, h->conv_rows()) * h->d);
    for (int l = 0; l < h->nlist; ++l) {
      const long long len = h->list_off[l + 1] - h->list_off[l];
      for (long long r = 0; r < len;) {
        long long take = std::min(len - r, chunk_rows - fill);
        float* dst = bounce.p + (size_t)fill * h->d;
        if (!h->resident[l]) {
          std::memcpy(dst, h->host_arena.p + (size_t)(h->host_row0[l] + r) * h->d, (size_t)take * row_bytes);
        } else if (!h->split3) {
          CK(cudaMemcpy(dst, h->arena.p + (size_t)(h->res_row0[l] + r) * h->d, (size_t)take * row_bytes,
                        cudaMemcpyDeviceToHost));
        } else {
          take = std::min<long long>(take, (long long)(conv.n / h->d));
          h->store_get(h->res_row0[l] + r, take, conv.p, 0);
          CK(cudaMemcpy(dst, conv.p, (size_t)take * row_bytes, cudaMemcpyDeviceToHost));
        }
        fill += take;
        r += take;
        if (fill == chunk_rows) flush();
      }
    }
    flush();
    if (::fsync(f.fd) != 0) throw_rd(RD_ERR_RUNTIME, "save: fsync of %s failed", path);
  });
}

int rd_index_load(const char* path, int32_t device, rd_index** out) {
  return guarded([&] {
    if (!path || !out) throw_rd(RD_ERR_INVALID, "load: null argument");
    Fd f;
    f.fd = ::open(path, O_RDONLY);
    if (f.fd < 0) throw_rd(RD_ERR_INVALID, "load: cannot open %s", path);
    struct stat stt;
    if (::fstat(f.fd, &stt) != 0) throw_rd(RD_ERR_RUNTIME, "load: cannot stat %s", path);
    const uint64_t size = (uint64_t)stt.st_size;
    rd_file_header hd;
    if (size < sizeof hd) throw_rd(RD_ERR_INVALID, "load %s: truncated rd index file", path);
    pread_all(f.fd, &hd, sizeof hd, 0, path);
    if (const char* why = rd_fmt_validate(&hd, size, nullptr)) throw_rd(RD_ERR_INVALID, "load %s: %s", path, why);
    std::vector<long long> offs((size_t)hd.nlist + 1);
    pread_all(f.fd, offs.data(), 8 * offs.size(), hd.off_list_offsets, path);
    if (const char* why = rd_fmt_validate(&hd, size, reinterpret_cast<const int64_t*>(offs.data())))
      throw_rd(RD_ERR_INVALID, "load %s: %s", path, why);
    check_dims(hd.d);
    if (hd.n >= (1LL << 31)) throw_rd(RD_ERR_INVALID, "load: at most 2^31-1 vectors per handle");
    auto h = new_index(device);
    h->n = hd.n;
    h->d = hd.d;
    h->nlist = hd.nlist;
    h->list_off = offs;
    const int d = hd.d;
    {
      std::vector<float> c((size_t)hd.nlist * d);
      pread_all(f.fd, c.data(), 4 * c.size(), hd.off_centroids, path);
      h->centroids.alloc(c.size());
      h->cnorm.alloc(hd.nlist);
      CK(cudaMemcpy(h->centroids.p, c.data(), 4 * c.size(), cudaMemcpyHostToDevice));
      std::vector<long long> ids(std::max<long long>(1, hd.n));
      pread_all(f.fd, ids.data(), 8 * (size_t)hd.n, hd.off_ids, path);
      h->d_ids.alloc(hd.n);
      if (hd.n) CK(cudaMemcpy(h->d_ids.p, ids.data(), 8 * (size_t)hd.n, cudaMemcpyHostToDevice));
    }
    // vectors: file -> two pinned bounce buffers -> the conversion buffer -> the resident store; the
    // read of bounce chunk i+1 overlaps the copy of chunk i
    const size_t row_bytes = 4 * (size_t)d;
    const long long bounce_rows = std::max<long long>(1, (long long)(kIoChunk / row_bytes));
    HBuf<char> buf[2];
    cudaEvent_t done[2];
    for (int i = 0; i < 2; ++i) {
      buf[i].alloc((size_t)bounce_rows * row_bytes);
      CK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    long long nchunk = 0;
    try {
      h->materialize([&](long long r0, long long c, float* dst) {
        for (long long r = 0; r < c; r += bounce_rows, ++nchunk) {
          const long long take = std::min(bounce_rows, c - r);
          const int slot = (int)(nchunk & 1);
          if (nchunk >= 2) CK(cudaEventSynchronize(done[slot]));
          pread_all(f.fd, buf[slot].p, (size_t)take * row_bytes, hd.off_vectors + (uint64_t)(r0 + r) * row_bytes, path);
          CK(cudaMemcpyAsync(dst + (size_t)r * d, buf[slot].p, (size_t)take * row_bytes, cudaMemcpyHostToDevice,
                             h->copy_stream));
          CK(cudaEventRecord(done[slot], h->copy_stream));
        }
        CK(cudaStreamSynchronize(h->copy_stream));
      });
    } catch (...) {
      cudaStreamSynchronize(h->copy_stream);
      for (auto e : done) cudaEventDestroy(e);
      throw;
    }
    for (auto e : done) cudaEventDestroy(e);
    *out = h.release();
  });
}

int rd_index_info_get(const rd_index* h, rd_index_info* o) {
  return guarded([&] {
    if (!h || !o) throw_rd(RD_ERR_INVALID, "null argument");
    std::memset(o, 0, sizeof *o);
    o->n = h->n;
    o->d = h->d;
    o->nlist = h->nlist;
    o->n_resident = h->n_resident;
    for (int l = 0; l < h->nlist; ++l) o->lists_resident += h->resident[l];
    // what the index holds on the device: the resident store as mapped (rows rounded up to its
    // arena chunks), the staging ring, per-row norms / ids / list map and the coarse-stage state
    o->hbm_bytes = h->store_bytes() + (uint64_t)h->rplane.n * 2 + (uint64_t)h->rnorm.n * 4 + (uint64_t)h->staging.n * 4 + (uint64_t)h->n * (4 + 8 + 4) +
                   (uint64_t)h->nlist * ((uint64_t)h->d * 8 + 4 + 8 + 8 + 8);
    o->host_pinned_bytes = (uint64_t)h->host_arena.n * 4;
    o->staging_slots = h->slots;
    o->max_norm = h->xmax;
    o->device = h->device;
    o->store = h->split3 ? RD_STORE_SPLIT3 : h->resid ? (h->res16 ? RD_STORE_F32_RESID16 : RD_STORE_F32_RESID) : h->presplit ? RD_STORE_F32_PRESPLIT : RD_STORE_F32;
  });
}

int rd_index_layout(const rd_index* h, int64_t* offs, int64_t* ids, uint8_t* mask) {
  return guarded([&] {
    if (!h) throw_rd(RD_ERR_INVALID, "null index");
    CK(cudaSetDevice(h->device));
    if (offs) std::memcpy(offs, h->list_off.data(), sizeof(int64_t) * (h->nlist + 1));
    if (ids && h->n) CK(cudaMemcpy(ids, h->d_ids.p, sizeof(int64_t) * h->n, cudaMemcpyDeviceToHost));
    if (mask) std::memcpy(mask, h->resident.data(), h->nlist);
  });
}

// ---------------------------------------------------------------- relayout (placement and migration)
namespace {

// Residency change of an index between searches ("shrink before grow",
// core/src/simulator.cpp:323-326): lists leaving HBM get a pinned host copy unless they have one
// (copies are write-once and kept), the lists staying resident are compacted in store order toward
// row 0, the store shrinks (or grows) in place to the new resident rows — its VArenas unmap or map
// chunks at the tail — and the lists coming in are copied from their host copies into the tail.
// Device memory never holds more than max(before, after) of the store plus one conversion buffer
// (split3 stores only: fp32 <-> split rows). A list is resident in the store's current format.
void relayout(rd_index* h, const std::vector<uint8_t>& after, rd_migration_stats* ms) {
  const int nl = h->nlist, d = h->d;
  const size_t row_f32 = (size_t)d * 4;
  auto len_of = [&](int l) { return h->list_off[l + 1] - h->list_off[l]; };
  cudaStream_t cs = h->copy_stream;
  DBuf<float> conv;
  auto conv_buf = [&] {
    if (!conv.p) conv.alloc((size_t)std::min<long long>(h->conv_rows(), std::max(1LL, h->max_len)) * d);
    return (long long)(conv.n / d);
  };
  // 1. host copies of lists leaving HBM
  long long need_host = h->host_used;
  for (int l = 0; l < nl; ++l)
    if (h->resident[l] && !after[l] && h->host_row0[l] < 0) need_host += len_of(l);
  if ((size_t)need_host * d > h->host_arena.n) {  // grow the host arena, keeping its contents
    HBuf<float> grown;
    grown.alloc((size_t)std::max<long long>(need_host, h->host_used + h->host_used / 2) * d);
    if (h->host_used) std::memcpy(grown.p, h->host_arena.p, (size_t)h->host_used * row_f32);
    std::swap(h->host_arena.p, grown.p);
    std::swap(h->host_arena.n, grown.n);  // host_row0 are row offsets: unchanged by the move
  }
  for (int l = 0; l < nl; ++l) {
    if (!(h->resident[l] && !after[l]) || h->host_row0[l] >= 0) continue;
    const long long len = len_of(l);
    float* dst = h->host_arena.p + (size_t)h->host_used * d;
    if (!h->split3) {
      CK(cudaMemcpyAsync(dst, h->arena.p + (size_t)h->res_row0[l] * d, (size_t)len * row_f32,
                         cudaMemcpyDeviceToHost, cs));
    } else {
      const long long cr = conv_buf();
      for (long long r = 0; r < len; r += cr) {
        const long long c = std::min(cr, len - r);
        h->store_get(h->res_row0[l] + r, c, conv.p, cs);
        CK(cudaMemcpyAsync(dst + (size_t)r * d, conv.p, (size_t)c * row_f32, cudaMemcpyDeviceToHost, cs));
      }
    }
    h->host_row0[l] = h->host_used;
    h->host_used += len;
    if (ms) ms->d2h_bytes += (size_t)len * row_f32;
  }
  CK(cudaStreamSynchronize(cs));
  // 2. compact the lists that stay, in store order, toward row 0
  std::vector<int> keep;
  for (int l = 0; l < nl; ++l)
    if (h->resident[l] && after[l]) keep.push_back(l);
  std::sort(keep.begin(), keep.end(), [&](int a, int b) { return h->res_row0[a] < h->res_row0[b]; });
  long long tail = 0;
  for (int l : keep) {
    const long long old = h->res_row0[l], len = len_of(l);
    if (old != tail && len > 0) {
      h->store_move_down(tail, old, len, cs);
      if (ms) ms->d2d_bytes += (size_t)len * h->res_row_bytes();
    }
    h->res_row0[l] = tail;
    tail += len;
  }
  for (int l = 0; l < nl; ++l)
    if (h->resident[l] && !after[l]) h->res_row0[l] = -1;
  CK(cudaStreamSynchronize(cs));
  // 3. the store to the new resident size, in place
  long long res_rows = tail;
  for (int l = 0; l < nl; ++l)
    if (!h->resident[l] && after[l]) res_rows += len_of(l);
  h->store_resize(res_rows);
  // 4. lists coming in, from their host copies into the tail
  for (int l = 0; l < nl; ++l) {
    if (h->resident[l] || !after[l]) continue;
    const long long len = len_of(l);
    const float* src = h->host_arena.p + (size_t)h->host_row0[l] * d;
    if (!h->split3) {
      if (len)
        CK(cudaMemcpyAsync(h->arena.p + (size_t)tail * d, src, (size_t)len * row_f32, cudaMemcpyHostToDevice, cs));
    } else {
      const long long cr = conv_buf();
      for (long long r = 0; r < len; r += cr) {
        const long long c = std::min(cr, len - r);
        CK(cudaMemcpyAsync(conv.p, src + (size_t)r * d, (size_t)c * row_f32, cudaMemcpyHostToDevice, cs));
        h->store_put(tail + r, conv.p, c, cs);
      }
    }
    h->res_row0[l] = tail;
    tail += len;
    if (ms) ms->h2d_bytes += (size_t)len * row_f32;
  }
  CK(cudaStreamSynchronize(cs));
  h->resident = after;
  h->n_resident = tail;
}

// A placement keeps host copies of the offloaded lists only (the oracle's rule, rd_oracle.c
// rd_index_place): the pinned host arena is rebuilt with just those, in list order.
void compact_host(rd_index* h) {
  const int nl = h->nlist, d = h->d;
  long long n_off = 0;
  for (int l = 0; l < nl; ++l)
    if (!h->resident[l]) n_off += h->list_off[l + 1] - h->list_off[l];
  HBuf<float> fresh;
  if (n_off) fresh.alloc((size_t)n_off * d);
  long long hr = 0;
  for (int l = 0; l < nl; ++l) {
    const long long len = h->list_off[l + 1] - h->list_off[l];
    if (h->resident[l]) {
      h->host_row0[l] = -1;
      continue;
    }
    if (len) std::memcpy(fresh.p + (size_t)hr * d, h->host_arena.p + (size_t)h->host_row0[l] * d, (size_t)len * d * 4);
    h->host_row0[l] = hr;
    hr += len;
  }
  std::swap(h->host_arena.p, fresh.p);
  std::swap(h->host_arena.n, fresh.n);
  h->host_used = hr;
}

// staging-ring rows for an offloaded set whose largest list has max_off rows (rd.h, rd_placement)
long long ring_slot_rows(long long max_off) { return (std::max<long long>(max_off, 16384) + 255) / 256 * 256; }

}  // namespace

// ---------------------------------------------------------------- placement (N8)
int rd_index_place(rd_index* h, const rd_placement* p) {
  return guarded([&] {
    if (!h || !p) throw_rd(RD_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    h->tail_wait();
    CK(cudaDeviceSynchronize());  // searches enqueued with rd_search_device read the store
    const int nl = h->nlist;
    const uint64_t budget0 = p->hbm_budget_bytes;
    auto len_of = [&](int l) { return h->list_off[l + 1] - h->list_off[l]; };
    // The resident set for a store format (bytes per resident row): the mask, or the hottest lists
    // up to the offload fraction and the budget; `cut` when the budget, not the fraction, stopped it.
    auto choose = [&](uint64_t row_bytes, std::vector<uint8_t>& mask, uint64_t& res_bytes, bool& cut) {
      mask.assign(nl, 0);
      res_bytes = 0;
      cut = false;
      if (p->resident_mask) {
        for (int l = 0; l < nl; ++l) {
          mask[l] = p->resident_mask[l] ? 1 : 0;
          if (mask[l]) res_bytes += (uint64_t)len_of(l) * row_bytes;
        }
        return;
      }
      std::vector<int> order(nl);
      for (int l = 0; l < nl; ++l) order[l] = l;
      if (p->list_heat)
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return p->list_heat[a] > p->list_heat[b]; });
      const long long target = nl - (long long)std::floor(p->offload_fraction * nl + 0.5);
      // the budget covers the resident lists and, once anything is offloaded, a staging ring of at
      // least two slots of max(largest list, 16384 rows) (include/rd.h, rd_placement)
      uint64_t budget = budget0;
      if (budget) {
        uint64_t all = 0;
        for (long long i = 0; i < target; ++i) all += (uint64_t)len_of(order[i]) * row_bytes;
        if (target < nl || all > budget) {
          const uint64_t reserve = (uint64_t)std::max(2, p->staging_slots) * ring_slot_rows(h->max_len) * h->d * 4;
          if (reserve > budget)
            throw_rd(RD_ERR_INFEASIBLE, "placement infeasible: budget %llu below the %llu-byte staging ring",
                     (unsigned long long)budget, (unsigned long long)reserve);
          budget -= reserve;
        }
      }
      for (long long i = 0; i < target; ++i) {
        const int l = order[i];
        const uint64_t lb = (uint64_t)len_of(l) * row_bytes;
        if (budget && res_bytes + lb > budget) {
          cut = true;
          break;
        }
        res_bytes += lb;
        mask[l] = 1;
      }
    };
    if (!p->resident_mask && (p->offload_fraction < 0 || p->offload_fraction > 1))
      throw_rd(RD_ERR_INVALID, "offload_fraction must be in [0, 1]");
    // Store format: split3 (the fast scan) unless a byte budget would then hold fewer lists than
    // fp32 rows can — under a tight budget (an LLM co-tenant, C5) residency is worth more than scan
    // speed, since every list left out streams over the host link on every search.
    std::vector<uint8_t> mask;
    uint64_t res_bytes = 0;
    bool cut = false, fmt3 = false, fmt_res = false;
    // the residual store (fp32 rows + bf16 residual plane + ||x - c||^2: 6 B + 4 B per row) when every
    // list stays resident in it — the fastest scan (2 B per element read)
    if (h->resid_fmt()) {
      choose((uint64_t)h->d * 6 + 4, mask, res_bytes, cut);
      bool all = !cut;
      for (int l = 0; l < nl && all; ++l) all = mask[l] != 0;
      fmt_res = all && !(budget0 && res_bytes > budget0);
    }
    if (!fmt_res && h->split3_eligible()) {
      choose((uint64_t)h->d * 6, mask, res_bytes, cut);
      fmt3 = !cut && !(p->resident_mask && budget0 && res_bytes > budget0);
    }
    if (!fmt3 && !fmt_res) choose((uint64_t)h->d * 4, mask, res_bytes, cut);
    if (p->resident_mask && budget0 && res_bytes > budget0)
      throw_rd(RD_ERR_INFEASIBLE, "placement infeasible: resident lists need %llu bytes > budget %llu",
               (unsigned long long)res_bytes, (unsigned long long)budget0);
    // staging ring: slots of >= the largest offloaded list; depth by the queue_capacity rule
    long long n_off = 0, max_off = 0, n_res = 0;
    for (int l = 0; l < nl; ++l) {
      if (mask[l])
        n_res += len_of(l);
      else {
        n_off += len_of(l);
        max_off = std::max(max_off, len_of(l));
      }
    }
    long long slot_rows = 0;
    int slots = 0;
    const uint64_t row_bytes = (uint64_t)h->d * (fmt3 || fmt_res ? 6 : 4);
    if (n_off > 0) {
      slot_rows = ring_slot_rows(max_off);
      const double slot_bytes = (double)slot_rows * h->d * 4;
      double free_bytes;
      if (budget0) {
        free_bytes = (double)budget0 - (double)res_bytes;
      } else {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        // free now, plus what the store gives back, minus what it grows by
        free_bytes = (double)fr + (double)h->store_bytes() - (double)n_res * row_bytes - (double)(1ull << 30);
      }
      slots = p->staging_slots > 0 ? p->staging_slots : std::min(8, rd_staging_depth(free_bytes, slot_bytes));
      if (budget0 && res_bytes + slots * slot_bytes > (double)budget0)
        throw_rd(RD_ERR_INFEASIBLE, "placement infeasible: no room for one %.0f-byte staging slot in the budget",
                 slot_bytes);
    }
    {  // the device must hold the new store next to what stays: fail before touching anything
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      const double grow = (double)n_res * row_bytes + (double)slots * slot_rows * h->d * 4 -
                          (double)h->store_bytes() - (double)h->staging.n * 4;
      if (grow > (double)fr)
        throw_rd(RD_ERR_INFEASIBLE, "placement infeasible: needs %.0f more device bytes, %zu free", grow, fr);
    }
    h->set_staging(0, 0);  // the ring is rebuilt for the new offloaded set
    // a format change converts the store in place on the side where it is smaller: fp32 rows
    // (4 B per element) before the relayout when leaving split3, after it when entering
    if (!fmt3 && h->split3) h->convert_store(false);
    relayout(h, mask, nullptr);
    if (fmt3 && !h->split3) h->convert_store(true);  // stays fp32 if the split does not round-trip
    compact_host(h);
    h->budgeted = budget0 != 0;
    h->resid_ok = fmt_res;
    h->upload_residency();
    h->build_presplit();
    h->set_staging(slots, slot_rows);
  });
}

// ---------------------------------------------------------------- migration
int rd_index_migrate(rd_index* h, const int32_t* promote, int32_t n_promote, const int32_t* demote, int32_t n_demote,
                     uint64_t hbm_budget_bytes, rd_migration_stats* st) {
  return guarded([&] {
    if (!h || n_promote < 0 || n_demote < 0 || (n_promote && !promote) || (n_demote && !demote))
      throw_rd(RD_ERR_INVALID, "migrate: invalid arguments");
    CK(cudaSetDevice(h->device));
    const auto t0 = std::chrono::steady_clock::now();
    const int nl = h->nlist, d = h->d;
    auto len_of = [&](int l) { return h->list_off[l + 1] - h->list_off[l]; };
    std::vector<uint8_t> seen(nl, 0);
    for (int i = 0; i < n_promote + n_demote; ++i) {
      const bool is_p = i < n_promote;
      const int l = is_p ? promote[i] : demote[i - n_promote];
      const char* why = nullptr;
      if (l < 0 || l >= nl)
        why = "list id out of range";
      else if (seen[l])
        why = "list named twice";
      else if (is_p && h->resident[l])
        why = "promoted list is already resident";
      else if (!is_p && !h->resident[l])
        why = "demoted list is not resident";
      if (why) throw_rd(RD_ERR_INVALID, "migrate: %s (%d)", why, l);
      seen[l] = 1;
    }
    std::vector<uint8_t> after(h->resident);
    for (int l = 0; l < nl; ++l)
      if (seen[l]) after[l] = !after[l];
    long long res_rows = 0, max_off = -1;
    for (int l = 0; l < nl; ++l) {
      if (after[l])
        res_rows += len_of(l);
      else
        max_off = std::max(max_off, len_of(l));
    }
    // the ring after the move: slots of >= the largest offloaded list; with a budget, as many slots
    // as it leaves room for (at least two), otherwise the current depth (at least two)
    const long long slot_rows = max_off >= 0 ? ring_slot_rows(max_off) : 0;
    const uint64_t slot_bytes = (uint64_t)slot_rows * d * 4;
    const uint64_t res_bytes = (uint64_t)res_rows * h->res_row_bytes();
    int slots = max_off >= 0 ? std::max(2, h->slots) : 0;
    if (hbm_budget_bytes) {
      const uint64_t need = res_bytes + (max_off >= 0 ? 2ull * slot_bytes : 0);
      if (need > hbm_budget_bytes)
        throw_rd(RD_ERR_INFEASIBLE, "migration infeasible: %llu bytes needed > budget %llu",
                 (unsigned long long)need, (unsigned long long)hbm_budget_bytes);
      if (max_off >= 0)
        slots = (int)std::max<uint64_t>(2, std::min<uint64_t>(slots, (hbm_budget_bytes - res_bytes) / slot_bytes));
    }
    h->tail_wait();
    CK(cudaDeviceSynchronize());  // searches enqueued with rd_search_device read the store
    rd_migration_stats ms;
    std::memset(&ms, 0, sizeof ms);
    const bool ring_changes = slots != h->slots || (slots && slot_rows != h->slot_rows);
    if (ring_changes) h->set_staging(0, 0);  // shrink before grow: the old ring goes first
    relayout(h, after, &ms);
    if (hbm_budget_bytes) {
      h->budgeted = true;
      h->resid_ok = false;  // the budget rule counted the store's own row bytes only
    }
    if (ring_changes) h->set_staging(slots, slot_rows);
    h->upload_residency();
    h->build_presplit();
    ms.lists_promoted = n_promote;
    ms.lists_demoted = n_demote;
    ms.resident_bytes = (uint64_t)h->n_resident * d * 4;
    ms.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (st) *st = ms;
  });
}

// ---------------------------------------------------------------- placement arithmetic
int rd_llm_reservation_bytes(const rd_llm_reservation* r, double* out) {
  return guarded([&] {
    if (!r || !out) throw_rd(RD_ERR_INVALID, "null argument");
    if (r->gen_batch_size < 0 || r->w_gpu < 0 || r->w_gpu > 1 || r->c_gpu < 0 || r->c_gpu > 1)
      throw_rd(RD_ERR_INVALID, "reservation: fractions in [0,1] and batch >= 0 required");
    const double W = (double)r->weight_total;
    const double C = (double)r->kv_bytes_per_request * r->gen_batch_size;
    double H = (double)r->workspace_bytes_per_request * r->gen_batch_size;
    if (r->decode_phase) H *= r->workspace_fraction;
    *out = r->w_gpu * W + r->c_gpu * C + H;
  });
}

int32_t rd_staging_depth(double free_bytes, double item_bytes) {
  if (item_bytes <= 0) return 1;
  const double q = std::floor(free_bytes / item_bytes);
  if (q < 1) return 1;
  if (q > (double)(1 << 20)) return 1 << 20;
  return (int32_t)q;
}

}  // extern "C"
