// search.cu — one search behind include/rd.h (rd_search, rd_search_device, rd_probe):
//
//   qprep -> N1 coarse (GEMV / tensor-core GEMM) -> N2 select + seed -> N3 plan
//     -> N4/N5 resident scan (persistent, main stream)
//     || N9 offloaded lists: cudaMemcpyAsync pinned->staging on a copy stream,
//        event-gated scans of staged slots on a side stream
//   -> N6/N7 merge + exact rerank -> (exact fallback) -> results
//
// plus device-time accounting and the shard merges (N11). Reference seam: retrieval_time(P, db)
// (cost_model.cpp:15-21), called by the retrieval worker (simulator.cpp:359,560).
#include "host.cuh"

// ---------------------------------------------------------------- search
namespace {

struct Plan {
  int R, Rt, tail_from;
  int max_chunks;
  int cap;
  long long max_tiles;
};

Plan make_plan(const rd_index* h, long long B, int nprobe, bool pair, bool res) {
  Plan pl;
  const int np = std::min(nprobe, h->nlist);
  const double avg = h->nlist ? (double)h->n / h->nlist : 0.0;
  const double est_rows = std::min((double)h->n, (double)B * np * avg);
  // ~tiles_per_sm tiles per SM so the dynamic tile queue's tail (at most one tile per SM) stays
  // short, against a fixed cost per tile (query-operand gather, partial top-k records). Measured on
  // B200 (C2): 32 per SM up to a few hundred queries (+0.4-1.5 % over 8), 8 from 512 queries on,
  // where one chunk per list keeps the partial records few. Rows rounded to the tensor-core tile
  // (128), at least 256 (shorter tiles lost at one query), and at least one 256-row TMA box of the
  // FFMA scan when that path is in use; chunk_rows then balances each list's chunks. The residual
  // scan reads half the bytes per row, so a tile's fixed cost weighs twice as much: 8 per SM at every
  // batch (B = 8 +3.8 %, 128 +2 %, 256 +2.4 % over 32; B = 1 unchanged).
  const long long gran = rd::kTcRows;
  const int tps = h->tiles_per_sm > 0 ? h->tiles_per_sm : (B >= 512 || res ? 8 : 32);
  long long R = (long long)std::ceil(est_rows / ((double)h->num_sms * tps));
  static const long long floor_r = std::getenv("RD_MIN_ROWS") ? std::atoll(std::getenv("RD_MIN_ROWS")) : rd::kScanRows;
  // tail chunks: one tensor-core row tile (128) when every tile is a tensor-core tile (B200, B = 1:
  // 150 -> 146 us), else one FFMA box; smaller tail tiles measured slower (each tile's fixed latency)
  static const char* tail_env = std::getenv("RD_TAIL_ROWS");
  const bool all_tc = h->split3 || (h->tc_scan() && h->tc_min_q <= 1);
  const long long floor_t = tail_env ? std::atoll(tail_env) : all_tc ? rd::kTcRows : rd::kScanRows;
  R = std::max<long long>(floor_r, std::min<long long>(4096, (R + gran - 1) / gran * gran));
  pl.R = (int)R;
  // the last eighth of the lists (in id order, the order the scan's queue hands tiles out) in
  // quarter-size chunks: a shorter tail at one more tile per list there
  {
    const long long tg = floor_t < gran ? 32 : gran;
    pl.Rt = (int)std::max<long long>(floor_t, (R / 4 + tg - 1) / tg * tg);
  }
  pl.tail_from = h->nlist - h->nlist / 8;
  if (const char* v = std::getenv("RD_TAIL_FRAC")) pl.tail_from = h->nlist - (int)(h->nlist * std::atof(v));
  pl.max_chunks = (int)std::max<long long>(1, (h->max_len + pl.Rt - 1) / pl.Rt);
  // a CTA pair (scan_pair.cu) emits one partial list per CTA and query of a tile
  pl.cap = np * pl.max_chunks * rd::kPartsPerTile * (pair ? 2 : 1);
  pl.max_tiles = std::min<long long>(B * np, B * np / rd::kScanG + h->nlist) * pl.max_chunks + 1;
  return pl;
}

}  // namespace

namespace rdh {

// the coarse path a batch of B queries takes (do_search, rd_probe) and its dot-product bound
float coarse_gamma(long long B, int d) {
  return !rd::coarse_small((int)B) && d % 64 == 0 ? rd::gamma_bf16x3(d) : rd::gamma_ffma_coarse(d);
}

constexpr int kMaxWideK = 256;  // the exact large-k pass keeps up to 8 x 32 rows per warp (wide.cu)

void validate_search(const rd_index* h, int nprobe, int k) {
  (void)h;
  if (nprobe < 1 || k < 1) throw_rd(RD_ERR_INVALID, "search: nprobe >= 1 and k >= 1 required");
  if (k > kMaxWideK) throw_rd(RD_ERR_INVALID, "search: k <= %d supported, got %d", kMaxWideK, k);
}

// nprobe beyond the certified selection's candidate buffer: the all-centroid exact selection
bool select_all_needed(const rd_index* h, int nprobe) { return std::min(nprobe, h->nlist) + rd::kCoarseExtra > 512; }

// the all-centroid selection's scratch (sort keys, values, offsets, CUB temp) for a batch of B
void* select_all_scratch(rd_index* h, long long B, size_t* bytes) {
  *bytes = rd::select_all_scratch_bytes(std::min<long long>(B, rd::select_all_batch(h->nlist)), h->nlist);
  h->ws.sel_scratch.ensure(*bytes);
  return h->ws.sel_scratch.p;
}

// Counters of the search whose stat block copy do_search enqueued (mode kSync / kStatsAsync), read
// after its stream synchronized.
void finish_stats(rd_index* h, rd_search_stats* st) {
  const auto& pd = h->pend;
  std::memset(st, 0, sizeof *st);
  st->kernel_launches = pd.launches;
  const auto& w = h->ws;
  const auto* hc = reinterpret_cast<const unsigned long long*>(w.h_blk.p);
  const auto* hf = reinterpret_cast<const unsigned*>(w.h_blk.p + 24);
  const auto* hm = reinterpret_cast<const int*>(w.h_blk.p + 32);
  float ms = 0;
  const unsigned long long row_bytes = (unsigned long long)h->d * 4;
  st->lists_probed = hc[0];
  st->bytes_lists_resident = hc[1] * row_bytes;
  st->h2d_list_bytes = pd.h2d;
  st->bytes_algorithmic = (hc[1] + hc[2]) * row_bytes + (unsigned long long)h->nlist * row_bytes +
                          (unsigned long long)pd.B * row_bytes + (unsigned long long)pd.B * pd.k * 12ull;
  st->tiles = (uint64_t)hm[0] + (uint64_t)hm[2] + (uint64_t)hm[4];
  if (pd.staged) {
    CK(cudaEventElapsedTime(&ms, pd.e1, pd.e2));
    st->scan_ms = ms;
    CK(cudaEventElapsedTime(&ms, pd.e0, pd.e1));
    st->coarse_ms = ms;
  }
  if (pd.has_off) {
    CK(cudaEventElapsedTime(&ms, h->ev[4], h->ev[5]));
    st->offload_ms = ms;
  }
  st->probe_failures = hf[0];
  st->margin_failures = hf[1];
}

// result_bytes: bytes after the stat block that the stats copy brings back too (the host path's results)
void do_search(rd_index* h, const float* d_q, long long B, int nprobe, int k, long long* d_ids, float* d_dists,
               cudaStream_t s, int mode, rd_search_stats* st, size_t result_bytes,
               const std::function<void()>& before_sync) {
  validate_search(h, nprobe, k);
  CK(cudaSetDevice(h->device));
  h->tail_wait();  // the previous asynchronous search's tail is enqueued (it shares the workspace)
  auto& w = h->ws;
  const int nl = h->nlist, d = h->d;
  // tensor-core tile widths: mixed (<= 16-query lists narrow, others wide) or one width; the
  // offloaded lists' host-planned tiles use one width
  const int tc_mode = h->tc_mode_for(B, nprobe);
  // wide tiles over the x1 | x2 plane on CTA pairs (cta_group::2): RD_PAIR=1 only (slower)
  const bool sel_all = select_all_needed(h, nprobe);  // probes from exact distances to every centroid
  // residual store: the scan's keys need the coarse distances (not computed by the all-centroid
  // selection: those searches take the converter scan over the fp32 rows, with its error bound);
  // k > 18 as well: its rerank margin (32 - k) no longer clears the residual keys' bound, so a few
  // percent of queries would take the exact fallback (measured 4 % at k = 24)
  const bool res = h->resid && h->tc_scan() && h->slots == 0 && !sel_all && k + 14 <= rd::kTopK;
  const bool res16 = res && h->res16;  // fp16 residual scan (B = fp16(q) alone)
  const bool pair = tc_mode != 16 && h->tc_scan() && (h->presplit || res) && !res16 && h->pair_scan &&
                    rd::scan_pair_stages(h->d, res) > 0;
  const Plan pl = make_plan(h, B, nprobe, pair, res);
  const int tc_g = tc_mode == 16 ? 16 : 32;
  const int W = (int)((B + 31) / 32);
  w.qnorm.ensure(B);
  w.Dc.ensure((size_t)B * nl);
  w.probes.ensure((size_t)B * nprobe);
  w.list_nq.ensure(nl);
  w.list_qoff.ensure(nl);
  w.list_ntile.ensure(rd::kTileCats * (size_t)nl);
  w.list_toff.ensure(rd::kTileCats * (size_t)nl);
  w.list_q.ensure((size_t)B * nprobe);
  w.tiles.ensure(pl.max_tiles);
  w.tiles16.ensure(pl.max_tiles);
  w.ff_tiles.ensure(pl.max_tiles);
  w.qsplit.ensure((size_t)B * 2 * d);
  w.ensure_blk(kStatBytes + result_bytes);
  w.h_blk.ensure(kStatBytes + result_bytes);
  w.part_count.ensure(B);
  w.part_dist.ensure((size_t)B * pl.cap * rd::kTopK);
  w.part_row.ensure((size_t)B * pl.cap * rd::kTopK);


  cudaEvent_t* te = h->next_timing_slot();
  cudaEvent_t e0 = te[0], e1 = te[1], e2 = te[2], e3 = h->ev[3], e_plan = h->ev[4], e_off = h->ev[5];
  unsigned long long launches = 0;
  CK(cudaEventRecord(e0, s));
  // ||q||^2 and the query split (the tensor-core scan's operand) in one pass; at small batches it
  // rides in a trailing CTA of the GEMV coarse kernel
  rd::QprepArgs qa{d_q, B, d, w.qnorm.p, d % 64 == 0 ? w.qsplit.p : nullptr, w.fails(), w.part_count.p};
  if (res16) {
    w.qhalf.ensure((size_t)B * d);
    qa.qhalf = w.qhalf.p;
  }
  const float scan_gamma = res ? 0.f : h->scan_gamma_base();
  const bool wide = k > rd::kMaxK;                      // the exact large-k pass instead of scan + rerank
  if (sel_all) {
    CK(rd::launch_qprep(qa, s));
  } else if (rd::coarse_small((int)B)) {
    CK(rd::launch_coarse_small(d_q, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, qa, s));
  } else if (d % 64 == 0) {
    CK(rd::launch_qprep(qa, s));
    const CUtensorMap qmap = make_split_map(w.qsplit.p, B, d);
    CK(rd::launch_coarse_tc(qmap, h->cmap, h->cnorm.p, w.Dc.p, (int)B, nl, d, s));
  } else {
    CK(rd::launch_qprep(qa, s));
    CK(rd::launch_coarse(d_q, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, s));
  }
  w.qthr.ensure(B);
  const bool seed = B <= h->seed_max_b && !sel_all && !wide;
  if (!seed) CK(cudaMemsetAsync(w.qthr.p, 0x7f, sizeof(int) * B, s));  // no threshold: huge
  rd::SelectParams sp{w.Dc.p, d_q, w.qnorm.p, h->centroids.p, w.probes.p, w.fails(), (int)B, nl, nprobe, d, h->cmax,
                      h->d_list_off.p, h->d_res_row0.p, h->arena.p, h->xmax, seed ? w.qthr.p : nullptr, 0};
  sp.gamma_coarse = coarse_gamma(B, d);
  sp.gamma_scan = scan_gamma;
  sp.x12 = h->x12_dev();
  sp.x3 = h->x3_dev();
  unsigned long long* chain = nullptr;  // profiling only (RD_DEBUG_CHAIN): [select 32][plan 32][merge 32][scan 4/CTA + tiles, rows]
  if (h->dbg_chain) {
    const size_t n = 96 + 6 * (size_t)h->num_sms;
    if (h->dbg_chain_buf.n < n) h->dbg_chain_buf.alloc(n);
    chain = h->dbg_chain_buf.p;
    CK(cudaMemsetAsync(chain, 0, 8 * n, s));
    sp.dbg = chain;
  }
  const bool use_bm = !wide && rd::plan_uses_bitmap((int)B, nprobe, nl);
  if (use_bm) {  // zeroed on (re)allocation or after a search that stopped before its plan
    if (w.bitmap.n < (size_t)nl * W || !w.bitmap_clean) {
      w.bitmap.ensure((size_t)nl * W);
      CK(cudaMemsetAsync(w.bitmap.p, 0, sizeof(unsigned) * w.bitmap.n, s));
    }
    w.bitmap_clean = false;
    sp.bitmap = w.bitmap.p;
    sp.W = W;
  }
  // the merge reranks m = min(32, k + margin) candidates and certifies against the next: scans
  // prune with, and the seed bounds, that rank's distance
  const int m_rerank = std::min(rd::kTopK, k + h->rerank_margin(res, res16, B));
  const int thr_rank = std::min(rd::kTopK - 1, m_rerank);
  sp.seed_rows = thr_rank + 1;
  rd::PlanParams pp{w.probes.p, w.bitmap.p, W, h->d_list_off.p, h->d_res_row0.p, w.list_nq.p, w.list_qoff.p,
                    w.list_ntile.p, w.list_toff.p, w.list_q.p, {w.tiles16.p, w.tiles.p, w.ff_tiles.p}, w.meta(),
                    w.counters(), (int)B, nl, nprobe, pl.R, h->tc_scan() ? h->tc_min_q : 1 << 30, tc_mode,
                    pl.Rt, pl.tail_from};
  // B = 1, every list resident and a tensor-core list: the selection CTA plans the scan itself
  // (one launch and one kernel boundary fewer; RD_FUSE_PLAN=0 for A/B)
  const bool fuse_plan = B == 1 && !wide && !sel_all && h->slots == 0 && h->tc_scan() && h->tc_min_q <= 1 &&
                         tc_mode != 32 && h->fuse_plan && rd::select_staged(sp, h->stage_rows(B));
  if (fuse_plan) {
    sp.fp_tiles = w.tiles16.p;
    sp.fp_list_q = w.list_q.p;
    sp.fp_meta = w.meta();
    sp.fp_counters = w.counters();
    sp.fp_R = pl.R;
    sp.fp_Rt = pl.Rt;
  }
  if (sel_all) {
    size_t sb = 0;
    void* scratch = select_all_scratch(h, B, &sb);
    CK(rd::launch_select_all(d_q, h->centroids.p, B, nl, d, nprobe, w.probes.p, use_bm ? w.bitmap.p : nullptr, W,
                             scratch, sb, s));
    launches += 1 + 4 * ((B + rd::select_all_batch(nl) - 1) / rd::select_all_batch(nl));
  } else {
    h->traced("select", s, sp.dbg, [&] { CK(rd::launch_select(sp, h->stage_rows(B), s, h->num_sms)); });
    launches += rd::coarse_small((int)B) ? 2 : 3;  // (query prep +) coarse + select
  }
  if (wide) {  // exact query-major pass over the probed lists, then the per-query merge of its splits
    const int R = rd::wide_lists(k), S = rd::wide_splits(B, nprobe, k, h->num_sms);
    w.wide_d.ensure((size_t)S * B * 32 * R);
    w.wide_id.ensure((size_t)S * B * 32 * R);
    const rd::WideParams wp{d_q, w.probes.p, nprobe, h->d_list_off.p, h->d_list_base.p, h->d_res_row0.p,
                            h->x12_dev(), h->x3_dev(), h->d_ids.p, d, k, B, w.wide_d.p, w.wide_id.p, w.qthr.p};
    CK(rd::launch_wide(wp, S, s));
    const int K = 32 * R;
    CK(rd::launch_shard_merge_strided(S, B, K, reinterpret_cast<const char*>(w.wide_id.p), (size_t)B * K * 8,
                                      reinterpret_cast<const char*>(w.wide_d.p), (size_t)B * K * 4, d_ids, d_dists, s,
                                      k));
    launches += 2;
    if (h->stage_events) {
      CK(cudaEventRecord(e1, s));
      CK(cudaEventRecord(e2, s));
    }
    CK(cudaEventRecord(te[3], s));
    if (before_sync) before_sync();
    if (mode != kAsync) {
      CK(cudaMemcpyAsync(w.h_blk.p, w.blk.p, kStatBytes + result_bytes, cudaMemcpyDeviceToHost, s));
      h->pend = rd_index::Pending{B, k, 0, launches, h->stage_events, false, e0, e1, e2};
      if (mode == kSync) {
        CK(cudaStreamSynchronize(s));
        if (st) finish_stats(h, st);
      }
    } else if (st) {
      std::memset(st, 0, sizeof *st);
      st->kernel_launches = launches;
    }
    return;
  }
  if (!fuse_plan) {
    if (chain) pp.dbg = chain + 32;
    h->traced("plan", s, pp.dbg, [&] { CK(rd::launch_plan(pp, s)); });
    if (use_bm) w.bitmap_clean = true;  // list_fill, now enqueued, clears every bit the selection sets
    launches += use_bm ? 3 : 1;
  }
  const bool staged = h->stage_events;
  if (staged) CK(cudaEventRecord(e1, s));

  const bool has_off = h->slots > 0;
  if (has_off) {  // fetch the probe histogram for host-side staging decisions
    w.h_nq.ensure(nl);
    w.h_qoff.ensure(nl);
    CK(cudaMemcpyAsync(w.h_nq.p, w.list_nq.p, sizeof(int) * nl, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(w.h_qoff.p, w.list_qoff.p, sizeof(int) * nl, cudaMemcpyDeviceToHost, s));
  }
  if (has_off) CK(cudaEventRecord(e_plan, s));  // an event between two kernels costs their PDL overlap
  const CUtensorMap gmap = res16 ? make_bf16_row_map(w.qhalf.p, B, d, 1, true) : make_gather_map(w.qsplit.p, B, d);
  rd::ScanParams sc{w.ff_tiles.p, w.meta() + 2 * rd::kCatFfma, w.meta() + 2 * rd::kCatFfma + 1, d_q, w.qnorm.p,
                    w.list_q.p, h->xnorm.p, w.part_dist.p, w.part_row.p, w.part_count.p, pl.cap, d, w.qthr.p};
  rd::TcScanParams tc{w.tiles.p, w.meta() + 2 * rd::kCatWide, w.meta() + 2 * rd::kCatWide + 1, w.qsplit.p, w.qnorm.p,
                      w.list_q.p, h->xnorm.p,
                      w.part_dist.p, w.part_row.p, w.part_count.p, pl.cap, d, w.qthr.p, h->debug_skip};
  sc.thr_rank = thr_rank;
  tc.thr_rank = thr_rank;
  if (res) {  // residual store: lower-bound keys from the coarse distances (scan_tc.cu resid_pair_term)
    tc.xnorm = h->rnorm.p;
    tc.Dc = w.Dc.p;
    tc.nlist = nl;
    tc.cnorm = h->cnorm.p;
    tc.rmax = h->rmax.p;
    tc.gamma_coarse = coarse_gamma(B, d);
    tc.cmax = h->cmax;
    tc.gamma_res = res16 ? rd::gamma_resid16_r(d) : rd::gamma_resid_r(d);
    tc.gamma_q = res16 ? rd::gamma_resid16_q(d) : rd::gamma_resid_q(d);
    tc.abs_res = res16 ? rd::abs_resid16(d) : 0.f;
  }
  if (!h->split3 && (!h->tc_scan() || h->tc_min_q > 1)) {  // FFMA tiles exist only in these cases (fp32 store)
    CK(rd::launch_scan(h->map256, h->map32, sc, h->num_sms, s));
    launches += 1;
  }
  if (h->tc_scan()) {  // otherwise every tile is FFMA
    if (chain) tc.dbg = chain + 96;
    if (h->dbg_ts) {  // profiling only: per-CTA entry / ready / first tile / end times
      if (h->dbg_scan.n < 6 * (size_t)h->num_sms) h->dbg_scan.alloc(6 * (size_t)h->num_sms);
      CK(cudaMemsetAsync(h->dbg_scan.p, 0, 8 * 6 * (size_t)h->num_sms, s));
      tc.dbg = h->dbg_scan.p;
    }
    const bool stall = std::getenv("RD_DEBUG_STALL") != nullptr;  // profiling only (scan_tc.cu built with -DRD_STALL_PROF)
    if (stall) {
      if (h->dbg_stall.n < 12 * (size_t)h->num_sms) h->dbg_stall.alloc(12 * (size_t)h->num_sms);
      CK(cudaMemsetAsync(h->dbg_stall.p, 0, 8 * 12 * (size_t)h->num_sms, s));
      tc.stall = h->dbg_stall.p;
    }
    const CUtensorMap& xm128 = res ? h->rmap128 : h->presplit ? h->xmap128 : h->map128;
    const CUtensorMap& xm32 = res ? h->rmap32 : h->presplit ? h->xmap32 : h->map32;
    if (tc_mode != 32) {  // narrow tiles: the 16-wide scan (deeper ring)
      rd::TcScanParams tn = tc;
      tn.tiles = w.tiles16.p;
      tn.ntiles = w.meta() + 2 * rd::kCatNarrow;
      tn.tile_counter = w.meta() + 2 * rd::kCatNarrow + 1;
      // streamed query operand for about one query per probed list or fewer (scan_tc.cu)
      const bool stream =
          h->stream_force >= 0 ? h->stream_force != 0 : (long long)B * std::min(nprobe, nl) <= nl;

      CK(rd::launch_scan_tc(xm128, xm32, gmap, tn, h->num_sms, s, h->presplit || res, 16, stream, res, res16));
      launches += 1;
    }
    if (tc_mode != 16) {  // wide tiles: the 32-wide scan
      if (pair)
        CK(rd::launch_scan_pair(xm128, xm32, gmap, tc, h->num_sms, s, res));
      else
        CK(rd::launch_scan_tc(xm128, xm32, gmap, tc, h->num_sms, s, h->presplit || res, 32, false, res, res16));
      launches += 1;
    }
    if (stall) {
      std::vector<unsigned long long> v(12 * (size_t)h->num_sms);
      CK(cudaMemcpyAsync(v.data(), h->dbg_stall.p, 8 * v.size(), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      static const char* nm[10] = {"P.tempty", "P.empty", "P.bempty", "M.tfull", "M.bfull", "M.aempty", "M.full",
                                   "E.tfull", "E.afull", "total"};
      fprintf(stderr, "scan stall cycles (mean over CTAs):");
      for (int k2 = 0; k2 < 10; ++k2) {
        double m = 0;
        for (int c = 0; c < h->num_sms; ++c) m += (double)v[12 * c + k2] / h->num_sms;
        fprintf(stderr, " %s=%.0f", nm[k2], m);
      }
      fprintf(stderr, "\n");
    }
    if (h->dbg_ts) {
      std::vector<unsigned long long> t(6 * (size_t)h->num_sms);
      CK(cudaMemcpyAsync(t.data(), h->dbg_scan.p, 8 * t.size(), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      {  // CTAs by end time: (end ns from the first entry, tiles, rows), earliest and latest five
        const int G = h->num_sms;
        unsigned long long e0 = ~0ull;
        for (int c = 0; c < G; ++c) e0 = std::min(e0, t[4 * c]);
        std::vector<int> ord(G);
        for (int c = 0; c < G; ++c) ord[c] = c;
        std::sort(ord.begin(), ord.end(), [&](int a, int b) { return t[4 * a + 3] < t[4 * b + 3]; });
        fprintf(stderr, "scan CTA ends (ns, tiles, rows):");
        for (int i = 0; i < G; ++i)
          if (i < 5 || i >= G - 5)
            fprintf(stderr, " [%lld %llu %llu]", (long long)(t[4 * ord[i] + 3] - e0), t[4 * G + ord[i]], t[5 * G + ord[i]]);
        fprintf(stderr, "\n");
      }
      unsigned long long t0 = ~0ull, mx[4] = {0, 0, 0, 0};
      for (int c = 0; c < h->num_sms; ++c) t0 = std::min(t0, t[4 * c]);
      double mean[4] = {0, 0, 0, 0};
      for (int c = 0; c < h->num_sms; ++c)
        for (int j = 0; j < 4; ++j) {
          const unsigned long long v = t[4 * c + j] ? t[4 * c + j] - t0 : 0;
          mx[j] = std::max(mx[j], v);
          mean[j] += (double)v / h->num_sms;
        }
      fprintf(stderr, "scan ns from first CTA entry: entry mean %.0f max %llu | ready mean %.0f max %llu | "
              "first tile mean %.0f max %llu | end mean %.0f max %llu\n", mean[0], mx[0], mean[1], mx[1], mean[2],
              mx[2], mean[3], mx[3]);
    }
  }
  if (staged) CK(cudaEventRecord(e2, s));

  // The tail: offloaded lists (host-planned staging copies and scans on the side streams), then the
  // merge + exact rerank and the fallback on stream ms. ms = s runs it inline; an asynchronous search
  // with offloaded lists runs it on a host worker with ms = off_stream, while s waits on the gate.
  cudaEvent_t te3 = te[3], e_res = h->ev[6];
  auto tail = [=, &w](cudaStream_t ms, unsigned long long& launches) -> unsigned long long {
    unsigned long long h2d = 0;
    if (has_off) {
      CK(cudaEventSynchronize(e_plan));
      // offloaded, probed lists in ascending id, packed into staging slots
      std::vector<std::vector<int>> batches;
      long long fill = 0;
      for (int l = 0; l < nl; ++l) {
        if (h->resident[l] || w.h_nq.p[l] == 0) continue;
        const long long len = h->list_off[l + 1] - h->list_off[l];
        if (len == 0) continue;
        if (batches.empty() || fill + len > h->slot_rows) {
          batches.emplace_back();
          fill = 0;
        }
        batches.back().push_back(l);
        fill += len;
      }
      // host-planned tiles of every batch (tensor-core and FFMA groups), uploaded once
      const size_t nb = batches.size();
      std::vector<rd::ScanTile> tv;  // per batch: [tc tiles][ff tiles]
      std::vector<int> tstart(nb + 1, 0), ntc(nb, 0);
      for (size_t bi = 0; bi < nb; ++bi) {
        tstart[bi] = (int)tv.size();
        std::vector<rd::ScanTile> ff;
        long long srow = (long long)(bi % h->slots) * h->slot_rows;
        for (int l : batches[bi]) {
          const long long len = h->list_off[l + 1] - h->list_off[l];
          const int nq = w.h_nq.p[l];
          const bool tcl = nq >= h->tc_min_q && h->tc_scan();
          const int ngr = tcl ? (nq + tc_g - 1) / tc_g : (nq + rd::kScanG - 1) / rd::kScanG;
          const int rl = rd::chunk_rows(len, pl.R);
          for (long long c = 0; c * rl < len; ++c)
            for (int g = 0; g < ngr; ++g) {
              rd::ScanTile T;
              T.src_row = srow + c * rl;
              T.grow0 = h->list_off[l] + c * rl;
              T.list = l;
              T.nrows = (int)std::min<long long>(rl, len - c * rl);
              if (tcl) {
                const int q0 = (int)((long long)g * nq / ngr), q1 = (int)((long long)(g + 1) * nq / ngr);
                T.qoff = w.h_qoff.p[l] + q0;
                T.nq = q1 - q0;
                tv.push_back(T);
              } else {
                T.qoff = w.h_qoff.p[l] + g * rd::kScanG;
                T.nq = std::min(rd::kScanG, nq - g * rd::kScanG);
                ff.push_back(T);
              }
            }
          srow += len;
        }
        ntc[bi] = (int)tv.size() - tstart[bi];
        tv.insert(tv.end(), ff.begin(), ff.end());
      }
      tstart[nb] = (int)tv.size();
      if (nb) {
        w.h_tiles.ensure(tv.size());
        std::memcpy(w.h_tiles.p, tv.data(), sizeof(rd::ScanTile) * tv.size());
        w.off_tiles.ensure(tv.size());
        w.h_meta.ensure(4 * nb);
        for (size_t bi = 0; bi < nb; ++bi) {
          w.h_meta.p[4 * bi + 0] = ntc[bi];
          w.h_meta.p[4 * bi + 1] = 0;
          w.h_meta.p[4 * bi + 2] = tstart[bi + 1] - tstart[bi] - ntc[bi];
          w.h_meta.p[4 * bi + 3] = 0;
        }
        DBuf<int>& dmeta = w.off_meta;
        dmeta.ensure(4 * nb);
        CK(cudaStreamWaitEvent(h->off_stream, e_plan, 0));
        CK(cudaMemcpyAsync(w.off_tiles.p, w.h_tiles.p, sizeof(rd::ScanTile) * tv.size(), cudaMemcpyHostToDevice,
                           h->off_stream));
        CK(cudaMemcpyAsync(dmeta.p, w.h_meta.p, sizeof(int) * 4 * nb, cudaMemcpyHostToDevice, h->off_stream));
        CK(cudaEventRecord(e3, h->off_stream));
        CK(cudaStreamWaitEvent(h->copy_stream, e_plan, 0));
        for (size_t bi = 0; bi < nb; ++bi) {
          const int slot = (int)(bi % h->slots);
          if (bi >= (size_t)h->slots) CK(cudaStreamWaitEvent(h->copy_stream, h->slot_done[slot], 0));
          long long srow = (long long)slot * h->slot_rows;
          // lists adjacent in the host arena (and so in the slot) go out as one copy: fewer, larger
          // DMAs keep the host link closer to its peak than one copy per list
          long long run_src = -1, run_dst = 0, run_rows = 0;
          auto flush = [&] {
            if (run_rows == 0) return;
            const size_t bytes = (size_t)run_rows * d * sizeof(float);
            CK(cudaMemcpyAsync(h->staging.p + (size_t)run_dst * d, h->host_arena.p + (size_t)run_src * d, bytes,
                               cudaMemcpyHostToDevice, h->copy_stream));
            h2d += bytes;
            run_rows = 0;
          };
          for (int l : batches[bi]) {
            const long long len = h->list_off[l + 1] - h->list_off[l];
            if (run_rows && h->host_row0[l] != run_src + run_rows) flush();
            if (run_rows == 0) {
              run_src = h->host_row0[l];
              run_dst = srow;
            }
            run_rows += len;
            srow += len;
          }
          flush();
          CK(cudaEventRecord(h->slot_ready[slot], h->copy_stream));
          CK(cudaStreamWaitEvent(h->off_stream, h->slot_ready[slot], 0));
          const int nt_tc = ntc[bi], nt_ff = tstart[bi + 1] - tstart[bi] - ntc[bi];
          if (nt_ff) {
            rd::ScanParams so = sc;
            so.tiles = w.off_tiles.p + tstart[bi] + nt_tc;
            so.ntiles = dmeta.p + 4 * bi + 2;
            so.tile_counter = dmeta.p + 4 * bi + 3;
            CK(rd::launch_scan(h->smap256, h->smap32, so, std::min(h->num_sms, nt_ff), h->off_stream));
            launches += 1;
          }
          if (nt_tc) {
            rd::TcScanParams to = tc;
            to.tiles = w.off_tiles.p + tstart[bi];
            to.ntiles = dmeta.p + 4 * bi + 0;
            to.tile_counter = dmeta.p + 4 * bi + 1;
            CK(rd::launch_scan_tc(h->smap128, h->smap32, gmap, to, std::min(h->num_sms, nt_tc), h->off_stream, false,
                                  tc_g));
            launches += 1;
          }
          CK(cudaEventRecord(h->slot_done[slot], h->off_stream));
        }
      }
      CK(cudaEventRecord(e_off, h->off_stream));
      CK(cudaStreamWaitEvent(ms, e_off, 0));
    }
    if (ms != s) CK(cudaStreamWaitEvent(ms, e_res, 0));  // the resident scan, on the caller's stream

    if (!w.fb_ctr.p) {  // the fallback kernel's completion counter: zeroed once, re-armed by the kernel
      w.fb_ctr.alloc(1);
      CK(cudaMemset(w.fb_ctr.p, 0, sizeof(unsigned)));
    }
    w.fail_list.ensure(B);
    w.fb_dist.ensure((size_t)B * nprobe * rd::kTopK);
    w.fb_id.ensure((size_t)B * nprobe * rd::kTopK);
    rd::MergeParams mp{w.part_dist.p, w.part_row.p, w.part_count.p, pl.cap, d_q, w.qnorm.p, h->d_list_off.p,
                       h->d_list_base.p, h->d_ids.p, h->d_row_list.p, h->arena.p,
                       h->arena.p ? h->arena.p + (size_t)h->n_resident * d : nullptr, nl, d, k, h->xmax, d_ids, d_dists,
                       w.fails() + 1, w.fail_list.p, (int)B};
    mp.m_rerank = m_rerank;
    mp.gamma = scan_gamma;
    mp.res_row0 = h->d_res_row0.p;
    mp.x12 = h->x12_dev();
    mp.x3 = h->x3_dev();
    if (chain) mp.dbg = chain + 64;
    h->traced("merge", ms, mp.dbg, [&] { CK(rd::launch_merge(mp, h->stage_rows(B), ms)); });
    rd::FallbackParams fp{w.fail_list.p, w.fails() + 1, w.probes.p, nprobe, d_q, h->d_list_off.p, h->d_list_base.p,
                          h->d_ids.p, nl, d, k, w.fb_dist.p, w.fb_id.p, d_ids, d_dists, w.fb_ctr.p};
    fp.res_row0 = h->d_res_row0.p;
    fp.x12 = h->x12_dev();
    fp.x3 = h->x3_dev();
    CK(rd::launch_fallback(fp, h->num_sms, ms));
    launches += 2;
    CK(cudaEventRecord(te3, ms));
    if (chain) {  // ns from select's entry: [13] = entry (before the PDL wait), [0] = past the wait
      std::vector<unsigned long long> t(96 + 6 * (size_t)h->num_sms);
      CK(cudaMemcpyAsync(t.data(), chain, 8 * t.size(), cudaMemcpyDeviceToHost, ms));
      CK(cudaStreamSynchronize(ms));
      const long long t0 = (long long)t[13];
      const char* nm[3] = {"select", "plan", "merge"};
      for (int kk = 0; kk < 3; ++kk) {
        fprintf(stderr, "%s:", nm[kk]);
        if (t[32 * kk + 13]) fprintf(stderr, " entry=%lld", (long long)t[32 * kk + 13] - t0);
        for (int i = 0; i < 13; ++i)
          if (t[32 * kk + i]) fprintf(stderr, " %d=%lld", i, (long long)t[32 * kk + i] - t0);
        fprintf(stderr, "\n");
      }
      long long mn[4], mx[4];
      double mean[4];
      for (int j = 0; j < 4; ++j) {
        mn[j] = 1LL << 62, mx[j] = -(1LL << 62), mean[j] = 0;
        int cnt = 0;
        for (int c = 0; c < h->num_sms; ++c) {
          const unsigned long long v = t[96 + 4 * c + j];
          if (!v) continue;
          const long long r = (long long)v - t0;
          mn[j] = std::min(mn[j], r), mx[j] = std::max(mx[j], r), mean[j] += r, ++cnt;
        }
        if (cnt) mean[j] /= cnt;
      }
      fprintf(stderr, "scan: entry %lld/%.0f/%lld ready %lld/%.0f/%lld first %lld/%.0f/%lld end %lld/%.0f/%lld (min/mean/max)\n",
              mn[0], mean[0], mx[0], mn[1], mean[1], mx[1], mn[2], mean[2], mx[2], mn[3], mean[3], mx[3]);
    }
    return h2d;
  };
  unsigned long long h2d = 0;
  const bool async_tail =
      h->async_tail && has_off && mode == kAsync && !chain && stream_mem().wait32 && stream_mem().write32;
  if (!async_tail) {
    h2d = tail(s, launches);
  } else {
    // rd_search_device's contract: return once enqueued. The caller's stream s waits on gate >= seq;
    // the worker waits for the plan, enqueues the offloaded part, the merge and the fallback on the
    // side streams, then releases the gate from off_stream.
    CK(cudaEventRecord(e_res, s));
    if (!h->gate.p) {
      h->gate.alloc(1);
      CK(cudaMemset(h->gate.p, 0, sizeof(unsigned)));
    }
    if (!h->tailw) h->tailw = std::make_unique<TailWorker>();
    const unsigned seq = ++h->gate_seq;
    const CUdeviceptr gate = reinterpret_cast<CUdeviceptr>(h->gate.p);
    const CUresult r = stream_mem().wait32((CUstream)s, gate, seq, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw_rd(RD_ERR_RUNTIME, "cuStreamWaitValue32 failed (%d)", (int)r);
    h->tailw->post([=]() mutable {
      unsigned long long n = 0;
      std::exception_ptr err;
      try {
        CK(cudaSetDevice(h->device));
        tail(h->off_stream, n);
      } catch (...) {
        err = std::current_exception();
      }
      // released even after a failure, so the caller's stream never waits forever
      stream_mem().write32((CUstream)h->off_stream, gate, seq, 0);
      if (err) std::rethrow_exception(err);
    });
  }
  if (before_sync) before_sync();  // e.g. the host path's result copies, ordered before the one sync
  if (mode != kAsync) {
    // counters (and, on the host path, the results placed after them) in one copy
    CK(cudaMemcpyAsync(w.h_blk.p, w.blk.p, kStatBytes + result_bytes, cudaMemcpyDeviceToHost, s));
    h->pend = rd_index::Pending{B, k, h2d, launches, staged, has_off, e0, e1, e2};
    if (mode == kSync) {
      CK(cudaStreamSynchronize(s));
      if (st) finish_stats(h, st);
    }
  } else if (st) {
    std::memset(st, 0, sizeof *st);
    st->kernel_launches = launches;
  }
}

}  // namespace rdh

namespace {
// Largest batch searched in one pass: bounds the B x nlist coarse-distance workspace (2 GiB).
long long search_chunk(const rd_index* h) {
  return std::max<long long>(1024, std::min<long long>(65536, (1LL << 31) / (4LL * h->nlist)));
}
void add_stats(rd_search_stats* acc, const rd_search_stats& s) {  // counters summed over chunks
  acc->bytes_algorithmic += s.bytes_algorithmic;
  acc->bytes_lists_resident += s.bytes_lists_resident;
  acc->h2d_list_bytes += s.h2d_list_bytes;
  acc->lists_probed += s.lists_probed;
  acc->tiles += s.tiles;
  acc->kernel_launches += s.kernel_launches;
  acc->scan_ms += s.scan_ms;
  acc->coarse_ms += s.coarse_ms;
  acc->offload_ms += s.offload_ms;
  acc->margin_failures += s.margin_failures;
  acc->probe_failures += s.probe_failures;
}
}  // namespace

extern "C" {

int rd_search_device(rd_index* h, const float* d_q, int64_t B, int32_t nprobe, int32_t k, int64_t* d_ids,
                     float* d_dists, void* stream, int32_t sync, rd_search_stats* st) {
  return guarded([&] {
    if (!h || B < 0 || (B > 0 && (!d_q || !d_ids || !d_dists))) throw_rd(RD_ERR_INVALID, "search: invalid arguments");
    if (st) std::memset(st, 0, sizeof *st);
    if (B == 0) return;
    const auto t0 = std::chrono::steady_clock::now();
    const long long chunk = search_chunk(h);
    for (long long b0 = 0; b0 < B; b0 += chunk) {  // very large batches run as consecutive passes
      const long long nb = std::min<long long>(chunk, B - b0);
      rd_search_stats part{};
      rdh::do_search(h, d_q + (size_t)b0 * h->d, nb, nprobe, k, reinterpret_cast<long long*>(d_ids) + (size_t)b0 * k,
                d_dists + (size_t)b0 * k, (cudaStream_t)stream, sync != 0 ? rdh::kSync : rdh::kAsync, st ? &part : nullptr);
      if (st) add_stats(st, part);
    }
    if (st) st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int rd_search(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t k, int64_t* out_ids,
              float* out_dists, rd_search_stats* st) {
  if (h && B > search_chunk(h) && queries && out_ids && out_dists && h->d > 0 && k > 0) {
    // very large batches: consecutive passes of the one-pass path below
    const auto t0 = std::chrono::steady_clock::now();
    rd_search_stats acc{};
    const long long chunk = search_chunk(h);
    for (long long b0 = 0; b0 < B; b0 += chunk) {
      rd_search_stats part{};
      const int rc = rd_search(h, queries + (size_t)b0 * h->d, std::min<long long>(chunk, B - b0), nprobe, k,
                               out_ids + (size_t)b0 * k, out_dists + (size_t)b0 * k, &part);
      if (rc != RD_OK) return rc;
      add_stats(&acc, part);
    }
    acc.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (st) *st = acc;
    return RD_OK;
  }
  return guarded([&] {
    if (!h || B < 0 || (B > 0 && (!queries || !out_ids || !out_dists)))
      throw_rd(RD_ERR_INVALID, "search: invalid arguments");
    if (nprobe < 1 || k < 1) throw_rd(RD_ERR_INVALID, "search: nprobe >= 1 and k >= 1 required");
    const auto t0 = std::chrono::steady_clock::now();
    if (B == 0) {
      if (st) std::memset(st, 0, sizeof *st);
      return;
    }
    CK(cudaSetDevice(h->device));
    auto& w = h->ws;
    const size_t qn = (size_t)B * h->d, rn = (size_t)B * k;
    w.q.ensure(qn);
    // cudaMemcpyAsync copies straight from the caller's buffer: DMA when it is page-locked, a staged
    // copy by the driver otherwise (both correct; no pointer-attribute queries on the hot path)
    cudaStream_t s = 0;
    CK(cudaMemcpyAsync(w.q.p, queries, qn * sizeof(float), cudaMemcpyHostToDevice, s));
    // results live right after the stat block: small results come back with the counters in the
    // sync's single copy; large ones go straight into the caller's buffers
    const size_t res_bytes = rn * (sizeof(long long) + sizeof(float));
    const bool direct = res_bytes > (size_t(64) << 10);
    w.ensure_blk(kStatBytes + res_bytes);
    long long* d_ids = reinterpret_cast<long long*>(w.blk.p + kStatBytes);
    float* d_dists = reinterpret_cast<float*>(w.blk.p + kStatBytes + rn * sizeof(long long));
    rdh::do_search(h, w.q.p, B, nprobe, k, d_ids, d_dists, s, rdh::kSync, st, direct ? 0 : res_bytes, [&] {
      if (!direct) return;
      CK(cudaMemcpyAsync(out_ids, d_ids, rn * sizeof(long long), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(out_dists, d_dists, rn * sizeof(float), cudaMemcpyDeviceToHost, s));
    });
    if (!direct) {
      std::memcpy(out_ids, w.h_blk.p + kStatBytes, rn * sizeof(long long));
      std::memcpy(out_dists, w.h_blk.p + kStatBytes + rn * sizeof(long long), rn * sizeof(float));
    }
    if (st) st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int rd_probe(rd_index* h, const float* queries, int64_t B, int32_t nprobe, int32_t* out_lists) {
  return guarded([&] {
    if (!h || B < 0 || (B > 0 && (!queries || !out_lists))) throw_rd(RD_ERR_INVALID, "probe: invalid arguments");
    if (nprobe < 1) throw_rd(RD_ERR_INVALID, "probe: nprobe >= 1 required");
    if (B == 0) return;
    CK(cudaSetDevice(h->device));
    h->tail_wait();
    auto& w = h->ws;
    const int nl = h->nlist, d = h->d;
    w.q.ensure((size_t)B * d);
    w.qnorm.ensure(B);
    w.Dc.ensure((size_t)B * nl);
    w.probes.ensure((size_t)B * nprobe);
    w.ensure_blk(kStatBytes);
    CK(cudaMemcpy(w.q.p, queries, sizeof(float) * B * d, cudaMemcpyHostToDevice));
    CK(cudaMemset(w.fails(), 0, 2 * sizeof(unsigned)));
    if (rdh::select_all_needed(h, nprobe)) {  // large nprobe: already in exact order
      size_t sb = 0;
      void* scratch = rdh::select_all_scratch(h, B, &sb);
      CK(rd::launch_select_all(w.q.p, h->centroids.p, B, nl, d, nprobe, w.probes.p, nullptr, 0, scratch, sb, 0));
      CK(cudaMemcpy(out_lists, w.probes.p, sizeof(int) * B * nprobe, cudaMemcpyDeviceToHost));
      return;
    }
    w.qsplit.ensure((size_t)B * d);
    const rd::QprepArgs qa{w.q.p, B, d, w.qnorm.p, d % 64 == 0 ? w.qsplit.p : nullptr, nullptr, nullptr};
    if (rd::coarse_small((int)B)) {
      CK(rd::launch_coarse_small(w.q.p, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, qa, 0));
    } else if (d % 64 == 0) {
      CK(rd::launch_qprep(qa, 0));
      const CUtensorMap qmap = make_split_map(w.qsplit.p, B, d);
      CK(rd::launch_coarse_tc(qmap, h->cmap, h->cnorm.p, w.Dc.p, (int)B, nl, d, 0));
    } else {
      CK(rd::launch_qprep(qa, 0));
      CK(rd::launch_coarse(w.q.p, h->centroids.p, h->cnorm.p, w.Dc.p, (int)B, nl, d, 0));
    }
    rd::SelectParams sp{w.Dc.p, w.q.p, w.qnorm.p, h->centroids.p, w.probes.p, w.fails(), (int)B, nl, nprobe, d, h->cmax,
                        h->d_list_off.p, h->d_res_row0.p, h->arena.p, h->xmax, nullptr, 1};
    sp.gamma_coarse = rdh::coarse_gamma(B, d);
    CK(rd::launch_select(sp, h->stage_rows(B), 0, h->num_sms));
    CK(cudaMemcpy(out_lists, w.probes.p, sizeof(int) * B * nprobe, cudaMemcpyDeviceToHost));
  });
}

int rd_timing_stages(rd_index* h, int32_t on) {
  return guarded([&] {
    if (!h) throw_rd(RD_ERR_INVALID, "null index");
    h->stage_events = on != 0;
  });
}

int rd_timing_reset(rd_index* h) {
  return guarded([&] {
    if (!h) throw_rd(RD_ERR_INVALID, "null index");
    CK(cudaSetDevice(h->device));
    h->tail_wait();
    while (h->t_accounted < h->t_recorded) {  // drain so the ring's events are free again
      CK(cudaEventSynchronize(h->tev[h->t_accounted % rd_index::kRing][3]));
      ++h->t_accounted;
    }
    h->t_acc = rd_timing{};
  });
}

int rd_timing_read(rd_index* h, rd_timing* out) {
  return guarded([&] {
    if (!h || !out) throw_rd(RD_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    h->tail_wait();
    while (h->t_accounted < h->t_recorded) h->account(h->t_accounted++);
    *out = h->t_acc;
  });
}

// ---------------------------------------------------------------- shard merge
int rd_merge_topk(int32_t G, int64_t B, int32_t k, const int64_t* sid, const float* sd, int64_t* oid, float* od) {
  return guarded([&] {
    if (G < 1 || B < 0 || k < 1 || (B > 0 && (!sid || !sd || !oid || !od)))
      throw_rd(RD_ERR_INVALID, "merge: invalid arguments");
    std::vector<std::pair<float, int64_t>> c;
    for (int64_t q = 0; q < B; ++q) {
      c.clear();
      for (int g = 0; g < G; ++g)
        for (int i = 0; i < k; ++i) {
          const size_t o = ((size_t)g * B + q) * k + i;
          if (sid[o] >= 0) c.emplace_back(sd[o], sid[o]);
        }
      const size_t m = std::min<size_t>(k, c.size());
      std::partial_sort(c.begin(), c.begin() + m, c.end());
      for (int i = 0; i < k; ++i) {
        oid[q * k + i] = (size_t)i < m ? c[i].second : -1;
        od[q * k + i] = (size_t)i < m ? c[i].first : INFINITY;
      }
    }
  });
}

int rd_merge_topk_device(int32_t G, int64_t B, int32_t k, const int64_t* ids, const float* dists, int64_t* oid,
                         float* od, void* stream) {
  return guarded([&] {
    if (G < 1 || B < 0 || k < 1 || (long long)G * k > rd::shard_merge_max_candidates())
      throw_rd(RD_ERR_INVALID, "merge_device: invalid arguments (G * k <= %d)", rd::shard_merge_max_candidates());
    CK(rd::launch_shard_merge(G, B, k, reinterpret_cast<const long long*>(ids), dists,
                              reinterpret_cast<long long*>(oid), od, (cudaStream_t)stream));
  });
}

}  // extern "C"
