// capi.cu — pp_ctx and the C-ABI entry points (include/pipeplan_b200.h).
//
// Host-side orchestration of one planning call over n_seg independent
// mini-batches (the reference plans each with order_samples -> make_slice_cost
// -> dp_partition, src/planner.cpp:42,64-65; batches come from run_plan's
// worker pool, src/driver.cpp:222-242):
//
//   1. segmented sort                       (sort.cu)     order_samples(Sort)
//   2. cost pass A: Rm(i), singleton check,  (cost.cu)     microbatch.cpp:228-251
//      candidate statistics
//   3. band offsets, cost pass B: band +     (cost.cu)     microbatch.cpp:237-243,253-269
//      candidate bitmap / raw list
//   4. candidate compaction                  (cost.cu/sort.cu)
//   5. bound + minimax pass (c > 1)          (dp.cu)       microbatch.cpp:274-279
//   6. candidate waves: DP per (mb, t) +     (dp.cu)       microbatch.cpp:289-318
//      in-order selection, until every
//      mini-batch hit the reference's break
//   7. assembly                              (dp.cu)       microbatch.cpp:322-335
//
// The host only sizes buffers and decides wave membership from a few
// per-segment words read back between phases; all planning arithmetic is on
// the device.  There is no CPU fallback: without a device every entry point
// returns PP_ERR_NO_DEVICE.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pp_internal.cuh"

namespace ppb {
// sort.cu
cudaError_t launch_segmented_sort(const pp_sample* d_in, const int64_t* d_seg_off,
                                  const int64_t* h_seg_off, int n_seg, int64_t total,
                                  int presorted, unsigned long long* d_range,
                                  unsigned long long* h_range, unsigned long long* d_keys,
                                  uint32_t* d_vals, pp_sample* d_out, double* d_in_len,
                                  double* d_tgt_len, cudaStream_t st);
cudaError_t launch_segmented_sort_u64(unsigned long long* keys, unsigned long long* tmp,
                                      const int64_t* off, const unsigned long long* cnt,
                                      const int* seg_mode, int want_mode, int* in_tmp, int n_seg,
                                      cudaStream_t st);
// cost.cu
cudaError_t launch_row_scan(const GridDev& g, const double* tabT, const double* tabM,
                            const double* in_d, const double* tgt_d, const int64_t* seg_off,
                            int n_seg, int64_t total_rows, double cap, double interval, int* row_w,
                            SegStats* stats, cudaStream_t st);
cudaError_t launch_row_offsets(const int* row_w, const int64_t* seg_off, int n_seg, int64_t* row_off,
                               SegStats* stats, cudaStream_t st);
cudaError_t launch_band(const GridDev& g, const double* tabT, const double* tabM, const double* in_d,
                        const double* tgt_d, const int64_t* seg_off, int n_seg, int64_t total_rows,
                        double cap, double interval, int* row_w, SegStats* stats,
                        const int64_t* row_off, const int64_t* seg_band_base, double* band,
                        unsigned int* bitmap, const int64_t* bitmap_off, const int* seg_mode,
                        unsigned long long* cand_raw, const int64_t* cand_raw_off,
                        unsigned long long* cand_raw_cnt, cudaStream_t st);
cudaError_t launch_cand_bitmap(const unsigned int* bitmap, const int64_t* bitmap_off,
                               const SegStats* stats, const int* seg_mode, int n_seg,
                               double interval, const int64_t* cand_off, double* cand, int* cand_n,
                               cudaStream_t st);
cudaError_t launch_cand_unique(const unsigned long long* keys_a, const unsigned long long* keys_b,
                               const int* in_b, const int64_t* raw_off,
                               const unsigned long long* raw_cnt, const int* seg_mode, int n_seg,
                               const int64_t* cand_off, double* cand, int* cand_n, cudaStream_t st);
// dp.cu
size_t dp_smem_bytes(int mode, int n);
cudaError_t launch_dp_pass(int mode, const WorkItem* items, int n_items, size_t smem,
                           const int64_t* seg_off, const int* row_w, const int64_t* row_off,
                           const int64_t* seg_band_base, const double* band, const double* cand,
                           const int64_t* cand_off, ItemResult* res, int* next_buf, double* gstate,
                           cudaStream_t st);
cudaError_t launch_seg_init(const ItemResult* bound_res, int has_bound, int replicas,
                            const int64_t* cand_off, const int* cand_n, const double* cand,
                            const int* active, SegDP* dp, int n_seg, cudaStream_t st);
cudaError_t launch_select(const WorkItem* items, const ItemResult* res, const int* seg_item_start,
                          const int* seg_item_cnt, const int* next_buf, int* best_next,
                          const int64_t* seg_off, const double* cand, const int64_t* cand_off,
                          int stage_count, int replicas, SegDP* dps, int n_seg, cudaStream_t st);
cudaError_t launch_finalize(const SegDP* dps, const int* best_next, const int64_t* seg_off,
                            const int* row_w, const int64_t* row_off, const int64_t* seg_band_base,
                            const double* band, const SegStats* stats, const pp_sample* ordered,
                            int stage_count, int replicas, int max_n, int n_seg, int32_t* splits,
                            double* mb_times, int32_t* count, double* t_max_used, double* objective,
                            int32_t* status, int64_t* err_id, cudaStream_t st);
}  // namespace ppb

using namespace ppb;

namespace {

constexpr size_t kDpSmemLimit = 200 * 1024;  // per-CTA state budget before spilling to global

// Grow-only device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

struct pp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  pp_tuning tuning{};
  pp_stats stats{};
  cudaEvent_t ev[4]{};
  // device scratch
  DevBuf samples, seg_off, ordered, in_d, tgt_d, sort_keys, sort_vals, range;
  DevBuf grid_ax, grid_cells, layouts, tabT, tabM;
  DevBuf row_w, row_off, stats_d, band_base, band, bitmap, bitmap_off, seg_mode, raw, raw_tmp,
      raw_off, raw_cnt, raw_in_tmp, cand, cand_off, cand_n, active;
  DevBuf items, results, next_buf, gstate, seg_item_start, seg_item_cnt, segdp, best_next,
      bound_items, bound_res;
  DevBuf out_splits, out_times, out_count, out_tmax, out_obj, out_status, out_err;
  PinBuf h_range, h_stats, h_segdp, h_misc;
};

namespace {

#define PP_CUDA(x)                                                                   \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_);                    \
      return PP_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

int fail(pp_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

// Everything one planning call needs, all device pointers unless h_*.
struct PlanCall {
  const pp_sample* d_samples = nullptr;  // grid path
  const double* d_tabT = nullptr;        // table path
  const double* d_tabM = nullptr;
  const int64_t* d_seg_off = nullptr;
  const int64_t* h_seg_off = nullptr;
  int n_seg = 0;
  int presorted = 0;
  const pp_grid_desc* grid = nullptr;
  const pp_model_desc* model = nullptr;
  pp_dp_options opts{};
  // outputs (device)
  pp_sample* d_ordered = nullptr;
  int32_t* d_splits = nullptr;
  double* d_times = nullptr;
  int32_t* d_count = nullptr;
  double* d_tmax = nullptr;
  double* d_obj = nullptr;
  int32_t* d_status = nullptr;
  int64_t* d_err = nullptr;
};

int validate_opts(pp_ctx* ctx, const pp_dp_options& o) {
  if (o.stage_count < 1 || o.replica_count < 1)
    return fail(ctx, PP_ERR_INVALID, "stage and replica counts must be >= 1");
  if (o.t_max_interval < 0 || std::isnan(o.t_max_interval))
    return fail(ctx, PP_ERR_INVALID, "t_max_interval must be >= 0");
  return PP_OK;
}

// Upload the grid restricted to the recompute strategy, plus the distinct
// stage layouts.  Returns the device descriptor.
int upload_grid(pp_ctx* ctx, const pp_grid_desc* g, const pp_model_desc* m, GridDev* out) {
  if (!g || !m) return fail(ctx, PP_ERR_INVALID, "grid and model descriptors are required");
  if (g->n_mbs < 1 || g->n_seq < 1) return fail(ctx, PP_ERR_INVALID, "grid axis is empty");
  if (m->n_stages < 1) return fail(ctx, PP_ERR_INVALID, "stage and layer counts must be >= 1");
  if (m->recompute < 0 || m->recompute > 2) return fail(ctx, PP_ERR_INVALID, "unknown recompute strategy");
  const int nm = g->n_mbs, ns = g->n_seq;
  std::vector<double> ax((size_t)nm + ns);
  for (int k = 0; k < nm; ++k) ax[k] = static_cast<double>(g->mbs_axis[k]);
  for (int k = 0; k < ns; ++k) ax[nm + k] = static_cast<double>(g->seq_axis[k]);
  const size_t per = (size_t)nm * ns * 3;
  std::vector<double> cells(2 * per);
  for (int kind = 0; kind < 2; ++kind)
    std::memcpy(&cells[kind * per], g->cells + ((size_t)kind * 3 + m->recompute) * per,
                per * sizeof(double));
  std::vector<Layout> lay;
  for (int s = 0; s < m->n_stages; ++s) {
    Layout l{m->encoder_layers[s] > 0 ? m->encoder_layers[s] : 0,
             m->decoder_layers[s] > 0 ? m->decoder_layers[s] : 0};
    if (l.enc == 0 && l.dec == 0) continue;  // contributes (0, 0): max() unaffected
    bool seen = false;
    for (const auto& x : lay) seen |= (x.enc == l.enc && x.dec == l.dec);
    if (!seen) lay.push_back(l);
  }
  PP_CUDA(ctx->grid_ax.ensure(ax.size() * sizeof(double)));
  PP_CUDA(ctx->grid_cells.ensure(cells.size() * sizeof(double)));
  PP_CUDA(ctx->layouts.ensure(std::max<size_t>(lay.size(), 1) * sizeof(Layout)));
  PP_CUDA(cudaMemcpyAsync(ctx->grid_ax.p, ax.data(), ax.size() * sizeof(double),
                          cudaMemcpyHostToDevice, ctx->stream));
  PP_CUDA(cudaMemcpyAsync(ctx->grid_cells.p, cells.data(), cells.size() * sizeof(double),
                          cudaMemcpyHostToDevice, ctx->stream));
  if (!lay.empty())
    PP_CUDA(cudaMemcpyAsync(ctx->layouts.p, lay.data(), lay.size() * sizeof(Layout),
                            cudaMemcpyHostToDevice, ctx->stream));
  out->n_mbs = nm;
  out->n_seq = ns;
  out->n_layouts = (int)lay.size();
  out->is_encdec = m->is_encoder_decoder ? 1 : 0;
  out->mbs_ax = ctx->grid_ax.as<double>();
  out->seq_ax = ctx->grid_ax.as<double>() + nm;
  out->cells = ctx->grid_cells.as<double>();
  out->layouts = ctx->layouts.as<Layout>();
  // The host staging vectors die at return: make the copies complete first.
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  return PP_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// The planning pipeline (steps 1-7 above).
int run_plan(pp_ctx* ctx, const PlanCall& c) {
  cudaStream_t st = ctx->stream;
  const int n_seg = c.n_seg;
  const int64_t total = c.h_seg_off[n_seg] - c.h_seg_off[0];
  pp_stats S{};
  int max_n = 0;
  for (int s = 0; s < n_seg; ++s)
    max_n = std::max<int>(max_n, (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]));
  if (c.h_seg_off[0] != 0) return fail(ctx, PP_ERR_INVALID, "seg_offsets[0] must be 0");
  for (int s = 0; s < n_seg; ++s)
    if (c.h_seg_off[s + 1] < c.h_seg_off[s]) return fail(ctx, PP_ERR_INVALID, "seg_offsets must be non-decreasing");
  if (total >= INT_MAX) return fail(ctx, PP_ERR_INVALID, "too many samples in one call");

  GridDev g{};
  const bool table = c.d_tabT != nullptr;
  if (!table) {
    int rc = upload_grid(ctx, c.grid, c.model, &g);
    if (rc) return rc;
  }
  PP_CUDA(cudaEventRecord(ctx->ev[0], st));

  // ---- 1. order_samples(Sort)
  PP_CUDA(ctx->in_d.ensure(std::max<int64_t>(total, 1) * sizeof(double)));
  PP_CUDA(ctx->tgt_d.ensure(std::max<int64_t>(total, 1) * sizeof(double)));
  if (!table) {
    PP_CUDA(ctx->range.ensure(6 * sizeof(unsigned long long)));
    PP_CUDA(ctx->h_range.ensure(6 * sizeof(unsigned long long)));
    PP_CUDA(ctx->sort_keys.ensure(std::max<int64_t>(total, 1) * 6 * sizeof(unsigned long long)));
    PP_CUDA(ctx->sort_vals.ensure(std::max<int64_t>(total, 1) * 2 * sizeof(uint32_t)));
    if (total > 0)
      PP_CUDA(launch_segmented_sort(c.d_samples, c.d_seg_off, c.h_seg_off, n_seg, total, c.presorted,
                                    ctx->range.as<unsigned long long>(),
                                    ctx->h_range.as<unsigned long long>(),
                                    ctx->sort_keys.as<unsigned long long>(),
                                    ctx->sort_vals.as<uint32_t>(), c.d_ordered, ctx->in_d.as<double>(),
                                    ctx->tgt_d.as<double>(), st));
  }
  PP_CUDA(cudaEventRecord(ctx->ev[1], st));

  // ---- 2. cost pass A
  const double cap = c.opts.per_mb_mem_cap;
  const double I = c.opts.t_max_interval;
  PP_CUDA(ctx->row_w.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
  PP_CUDA(ctx->row_off.ensure(std::max<int64_t>(total, 1) * sizeof(int64_t)));
  PP_CUDA(ctx->stats_d.ensure(n_seg * sizeof(SegStats)));
  PP_CUDA(ctx->h_stats.ensure(n_seg * sizeof(SegStats)));
  {
    SegStats* hs = ctx->h_stats.as<SegStats>();
    for (int s = 0; s < n_seg; ++s) hs[s] = SegStats{~0ULL, 0ULL, 0ULL, INT_MAX, 0, 0};
    PP_CUDA(cudaMemcpyAsync(ctx->stats_d.p, hs, n_seg * sizeof(SegStats), cudaMemcpyHostToDevice, st));
  }
  SegStats* d_stats = ctx->stats_d.as<SegStats>();
  if (total > 0) {
    PP_CUDA(launch_row_scan(g, c.d_tabT, c.d_tabM, ctx->in_d.as<double>(), ctx->tgt_d.as<double>(),
                            c.d_seg_off, n_seg, total, cap, I, ctx->row_w.as<int>(), d_stats, st));
    PP_CUDA(launch_row_offsets(ctx->row_w.as<int>(), c.d_seg_off, n_seg, ctx->row_off.as<int64_t>(),
                               d_stats, st));
  }
  PP_CUDA(cudaMemcpyAsync(ctx->h_stats.p, d_stats, n_seg * sizeof(SegStats), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));

  // ---- 3. sizing: band, candidate modes
  const SegStats* hs = ctx->h_stats.as<SegStats>();
  const bool single = c.opts.stage_count == 1;  // candidates = {+inf} (microbatch.cpp:255-257)
  std::vector<int64_t> band_base(n_seg), bm_off(n_seg + 1, 0), raw_off(n_seg + 1, 0),
      cand_off(n_seg + 1, 0);
  std::vector<int> mode(n_seg, 2), active(n_seg, 0);
  int64_t band_total = 0;
  for (int s = 0; s < n_seg; ++s) {
    const int n = (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]);
    band_base[s] = band_total;
    band_total += hs[s].band;
    active[s] = (n > 0 && hs[s].err_row == INT_MAX) ? 1 : 0;
    int64_t ncap = 1;
    bm_off[s + 1] = bm_off[s];
    raw_off[s + 1] = raw_off[s];
    if (!single && active[s]) {
      bool bitmap_ok = false;
      if (I > 0 && hs[s].kmin != ~0ULL) {
        // host mirror of dkey_inv
        auto inv = [](unsigned long long k) {
          unsigned long long u = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
          double d;
          std::memcpy(&d, &u, 8);
          return d;
        };
        const double kmn = inv(hs[s].kmin), kmx = inv(hs[s].kmax);
        if (std::fabs(kmn) < 4.0e15 && std::fabs(kmx) < 4.0e15 && kmx - kmn < (double)(1 << 26)) {
          const int64_t range = (int64_t)(kmx - kmn) + 1;
          bm_off[s + 1] = bm_off[s] + (range + 31) / 32;
          ncap = range + 2;
          bitmap_ok = true;
        }
      }
      if (bitmap_ok) {
        mode[s] = 0;
      } else {
        mode[s] = 1;
        raw_off[s + 1] = raw_off[s] + (int64_t)hs[s].nraw;
        ncap = (int64_t)hs[s].nraw + 1;
      }
    }
    cand_off[s + 1] = cand_off[s] + ncap;
  }
  S.slices_costed = 0;
  for (int s = 0; s < n_seg; ++s) {
    const int64_t n = c.h_seg_off[s + 1] - c.h_seg_off[s];
    S.slices_costed += n * (n + 1) / 2 + hs[s].band;
  }
  PP_CUDA(ctx->band_base.ensure(n_seg * sizeof(int64_t)));
  PP_CUDA(ctx->band.ensure(std::max<int64_t>(band_total, 1) * sizeof(double)));
  PP_CUDA(ctx->bitmap_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->bitmap.ensure(std::max<int64_t>(bm_off[n_seg], 1) * sizeof(unsigned int)));
  PP_CUDA(ctx->seg_mode.ensure(n_seg * sizeof(int)));
  PP_CUDA(ctx->active.ensure(n_seg * sizeof(int)));
  PP_CUDA(ctx->raw_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->raw.ensure(std::max<int64_t>(raw_off[n_seg], 1) * sizeof(unsigned long long)));
  PP_CUDA(ctx->raw_tmp.ensure(std::max<int64_t>(raw_off[n_seg], 1) * sizeof(unsigned long long)));
  PP_CUDA(ctx->raw_cnt.ensure(n_seg * sizeof(unsigned long long)));
  PP_CUDA(ctx->raw_in_tmp.ensure(n_seg * sizeof(int)));
  PP_CUDA(ctx->cand_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->cand.ensure(std::max<int64_t>(cand_off[n_seg], 1) * sizeof(double)));
  PP_CUDA(ctx->cand_n.ensure(n_seg * sizeof(int)));
  PP_CUDA(cudaMemcpyAsync(ctx->band_base.p, band_base.data(), n_seg * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->bitmap_off.p, bm_off.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->seg_mode.p, mode.data(), n_seg * sizeof(int), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->active.p, active.data(), n_seg * sizeof(int), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->raw_off.p, raw_off.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->cand_off.p, cand_off.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if (bm_off[n_seg] > 0) PP_CUDA(cudaMemsetAsync(ctx->bitmap.p, 0, bm_off[n_seg] * sizeof(unsigned int), st));
  PP_CUDA(cudaMemsetAsync(ctx->raw_cnt.p, 0, n_seg * sizeof(unsigned long long), st));
  PP_CUDA(cudaMemsetAsync(ctx->raw_in_tmp.p, 0, n_seg * sizeof(int), st));
  PP_CUDA(cudaMemsetAsync(ctx->cand_n.p, 0, n_seg * sizeof(int), st));

  if (total > 0)
    PP_CUDA(launch_band(g, c.d_tabT, c.d_tabM, ctx->in_d.as<double>(), ctx->tgt_d.as<double>(),
                        c.d_seg_off, n_seg, total, cap, I, ctx->row_w.as<int>(), d_stats,
                        ctx->row_off.as<int64_t>(), ctx->band_base.as<int64_t>(),
                        ctx->band.as<double>(), ctx->bitmap.as<unsigned int>(),
                        ctx->bitmap_off.as<int64_t>(), ctx->seg_mode.as<int>(),
                        ctx->raw.as<unsigned long long>(), ctx->raw_off.as<int64_t>(),
                        ctx->raw_cnt.as<unsigned long long>(), st));
  // ---- 4. candidate lists
  if (single) {
    std::vector<double> infs(cand_off[n_seg], INFINITY);
    std::vector<int> ones(n_seg, 1);
    PP_CUDA(cudaMemcpyAsync(ctx->cand.p, infs.data(), infs.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    PP_CUDA(cudaMemcpyAsync(ctx->cand_n.p, ones.data(), n_seg * sizeof(int), cudaMemcpyHostToDevice, st));
    PP_CUDA(cudaStreamSynchronize(st));  // host vectors die here
  } else {
    PP_CUDA(launch_cand_bitmap(ctx->bitmap.as<unsigned int>(), ctx->bitmap_off.as<int64_t>(), d_stats,
                               ctx->seg_mode.as<int>(), n_seg, I, ctx->cand_off.as<int64_t>(),
                               ctx->cand.as<double>(), ctx->cand_n.as<int>(), st));
    if (raw_off[n_seg] > 0) {
      PP_CUDA(launch_segmented_sort_u64(ctx->raw.as<unsigned long long>(),
                                        ctx->raw_tmp.as<unsigned long long>(),
                                        ctx->raw_off.as<int64_t>(),
                                        ctx->raw_cnt.as<unsigned long long>(), ctx->seg_mode.as<int>(),
                                        1, ctx->raw_in_tmp.as<int>(), n_seg, st));
      PP_CUDA(launch_cand_unique(ctx->raw.as<unsigned long long>(),
                                 ctx->raw_tmp.as<unsigned long long>(), ctx->raw_in_tmp.as<int>(),
                                 ctx->raw_off.as<int64_t>(), ctx->raw_cnt.as<unsigned long long>(),
                                 ctx->seg_mode.as<int>(), n_seg, ctx->cand_off.as<int64_t>(),
                                 ctx->cand.as<double>(), ctx->cand_n.as<int>(), st));
    }
  }
  PP_CUDA(cudaEventRecord(ctx->ev[2], st));

  // ---- 5. bound + minimax pass
  PP_CUDA(ctx->segdp.ensure(n_seg * sizeof(SegDP)));
  PP_CUDA(ctx->h_segdp.ensure(n_seg * sizeof(SegDP)));
  PP_CUDA(ctx->best_next.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
  PP_CUDA(ctx->bound_res.ensure(n_seg * sizeof(ItemResult)));
  const int64_t* d_cand_off = ctx->cand_off.as<int64_t>();
  const double* d_cand = ctx->cand.as<double>();
  int64_t bound_transitions = 0;
  if (!single) {
    std::vector<WorkItem> bi(n_seg);
    int64_t goff = 0;
    size_t smem_max = 0;
    for (int s = 0; s < n_seg; ++s) {
      const int n = (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]);
      bi[s].seg = s;
      bi[s].cand = -1;
      bi[s].next_off = 0;
      const size_t need = dp_smem_bytes(1, n);
      if (need <= kDpSmemLimit) {
        bi[s].state_off = -1;
        smem_max = std::max(smem_max, need);
      } else {
        bi[s].state_off = goff;
        goff += 2 * (int64_t)(n + 1);
      }
      if (active[s]) bound_transitions += hs[s].band;
    }
    // inactive segments still launch (cheap: they walk their band) but
    // their results are ignored by seg_init.
    PP_CUDA(ctx->bound_items.ensure(n_seg * sizeof(WorkItem)));
    PP_CUDA(ctx->gstate.ensure(std::max<int64_t>(goff, 1) * sizeof(double)));
    PP_CUDA(ctx->next_buf.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
    PP_CUDA(cudaMemcpyAsync(ctx->bound_items.p, bi.data(), n_seg * sizeof(WorkItem), cudaMemcpyHostToDevice, st));
    PP_CUDA(launch_dp_pass(1, ctx->bound_items.as<WorkItem>(), n_seg, smem_max, c.d_seg_off,
                           ctx->row_w.as<int>(), ctx->row_off.as<int64_t>(),
                           ctx->band_base.as<int64_t>(), ctx->band.as<double>(), d_cand, d_cand_off,
                           ctx->bound_res.as<ItemResult>(), ctx->next_buf.as<int>(),
                           ctx->gstate.as<double>(), st));
    PP_CUDA(cudaStreamSynchronize(st));  // bi dies here
  }
  PP_CUDA(launch_seg_init(ctx->bound_res.as<ItemResult>(), single ? 0 : 1, c.opts.replica_count,
                          d_cand_off, ctx->cand_n.as<int>(), d_cand, ctx->active.as<int>(),
                          ctx->segdp.as<SegDP>(), n_seg, st));

  // ---- 6. candidate waves
  int wave = std::max(1, ctx->tuning.first_wave);
  const int max_wave = std::max(wave, ctx->tuning.max_wave > 0 ? ctx->tuning.max_wave : 16);
  int64_t transitions = bound_transitions, evaluated = 0, waves = 0;
  std::vector<WorkItem> items;
  std::vector<int> item_start(n_seg), item_cnt(n_seg);
  for (;;) {
    PP_CUDA(cudaMemcpyAsync(ctx->h_segdp.p, ctx->segdp.p, n_seg * sizeof(SegDP), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaStreamSynchronize(st));
    const SegDP* hd = ctx->h_segdp.as<SegDP>();
    items.clear();
    int64_t noff = 0, goff = 0;
    size_t smem_max = 0;
    for (int s = 0; s < n_seg; ++s) {
      item_start[s] = (int)items.size();
      item_cnt[s] = 0;
      if (hd[s].done) continue;
      const int n = (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]);
      const int k = std::min(wave, hd[s].n_cand - hd[s].next_cand);
      const size_t need = dp_smem_bytes(0, n);
      for (int q = 0; q < k; ++q) {
        WorkItem w;
        w.seg = s;
        w.cand = hd[s].next_cand + q;
        w.next_off = noff;
        noff += n;
        if (need <= kDpSmemLimit) {
          w.state_off = -1;
          smem_max = std::max(smem_max, need);
        } else {
          w.state_off = goff;
          goff += 2 * (int64_t)(n + 1);
        }
        items.push_back(w);
        transitions += hs[s].band;
      }
      item_cnt[s] = k;
    }
    if (items.empty()) break;
    ++waves;
    evaluated += (int64_t)items.size();
    const int ni = (int)items.size();
    PP_CUDA(ctx->items.ensure(ni * sizeof(WorkItem)));
    PP_CUDA(ctx->results.ensure(ni * sizeof(ItemResult)));
    PP_CUDA(ctx->next_buf.ensure(std::max<int64_t>(noff, 1) * sizeof(int)));
    PP_CUDA(ctx->gstate.ensure(std::max<int64_t>(goff, 1) * sizeof(double)));
    PP_CUDA(ctx->seg_item_start.ensure(n_seg * sizeof(int)));
    PP_CUDA(ctx->seg_item_cnt.ensure(n_seg * sizeof(int)));
    PP_CUDA(cudaMemcpyAsync(ctx->items.p, items.data(), ni * sizeof(WorkItem), cudaMemcpyHostToDevice, st));
    PP_CUDA(cudaMemcpyAsync(ctx->seg_item_start.p, item_start.data(), n_seg * sizeof(int), cudaMemcpyHostToDevice, st));
    PP_CUDA(cudaMemcpyAsync(ctx->seg_item_cnt.p, item_cnt.data(), n_seg * sizeof(int), cudaMemcpyHostToDevice, st));
    PP_CUDA(launch_dp_pass(0, ctx->items.as<WorkItem>(), ni, smem_max, c.d_seg_off,
                           ctx->row_w.as<int>(), ctx->row_off.as<int64_t>(),
                           ctx->band_base.as<int64_t>(), ctx->band.as<double>(), d_cand, d_cand_off,
                           ctx->results.as<ItemResult>(), ctx->next_buf.as<int>(),
                           ctx->gstate.as<double>(), st));
    PP_CUDA(launch_select(ctx->items.as<WorkItem>(), ctx->results.as<ItemResult>(),
                          ctx->seg_item_start.as<int>(), ctx->seg_item_cnt.as<int>(),
                          ctx->next_buf.as<int>(), ctx->best_next.as<int>(), c.d_seg_off, d_cand,
                          d_cand_off, c.opts.stage_count, c.opts.replica_count,
                          ctx->segdp.as<SegDP>(), n_seg, st));
    wave = std::min(wave * 2, max_wave);
  }
  PP_CUDA(cudaEventRecord(ctx->ev[3], st));

  // ---- 7. assembly
  PP_CUDA(launch_finalize(ctx->segdp.as<SegDP>(), ctx->best_next.as<int>(), c.d_seg_off,
                          ctx->row_w.as<int>(), ctx->row_off.as<int64_t>(),
                          ctx->band_base.as<int64_t>(), ctx->band.as<double>(), d_stats, c.d_ordered,
                          c.opts.stage_count, c.opts.replica_count, std::max(max_n, 1), n_seg,
                          c.d_splits, c.d_times, c.d_count, c.d_tmax, c.d_obj, c.d_status, c.d_err,
                          st));
  PP_CUDA(cudaStreamSynchronize(st));
  PP_CUDA(cudaGetLastError());

  // stats
  const SegDP* hd = ctx->h_segdp.as<SegDP>();
  int64_t ref_tr = 0, gen = 0;
  for (int s = 0; s < n_seg; ++s) {
    const int64_t n = c.h_seg_off[s + 1] - c.h_seg_off[s];
    if (!active[s]) continue;
    gen += hd[s].n_cand;
    ref_tr += n * (n + 1) / 2 * ((int64_t)hd[s].ref_evals + (single ? 0 : 1));
  }
  S.candidates_generated = gen;
  S.candidates_evaluated = evaluated;
  S.transitions_executed = transitions;
  S.transitions_reference = ref_tr;
  S.waves = waves;
  S.ms_sort = elapsed(ctx->ev[0], ctx->ev[1]);
  S.ms_cost = elapsed(ctx->ev[1], ctx->ev[2]);
  S.ms_dp = elapsed(ctx->ev[2], ctx->ev[3]);
  S.ms_total = elapsed(ctx->ev[0], ctx->ev[3]);
  ctx->stats = S;
  return PP_OK;
}

int check_ctx(pp_ctx* ctx) {
  if (!ctx) return PP_ERR_INVALID;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return fail(ctx, PP_ERR_CUDA, cudaGetErrorString(e));
  return PP_OK;
}

}  // namespace

extern "C" {

int pp_abi_version(void) { return PP_ABI_VERSION; }

int pp_ctx_create(int device, pp_ctx** out) {
  if (!out) return PP_ERR_INVALID;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return PP_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= n) return PP_ERR_INVALID;
  if (cudaSetDevice(device) != cudaSuccess) return PP_ERR_CUDA;
  pp_ctx* ctx = new pp_ctx();
  ctx->device = device;
  ctx->tuning.first_wave = 1;
  ctx->tuning.max_wave = 16;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return PP_ERR_CUDA;
  }
  ctx->own_stream = true;
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  *out = ctx;
  return PP_OK;
}

int pp_ctx_destroy(pp_ctx* ctx) {
  if (!ctx) return PP_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (DevBuf* b : {&ctx->samples, &ctx->seg_off, &ctx->ordered, &ctx->in_d, &ctx->tgt_d,
                    &ctx->sort_keys, &ctx->sort_vals, &ctx->range, &ctx->grid_ax, &ctx->grid_cells,
                    &ctx->layouts, &ctx->tabT, &ctx->tabM, &ctx->row_w, &ctx->row_off, &ctx->stats_d,
                    &ctx->band_base, &ctx->band, &ctx->bitmap, &ctx->bitmap_off, &ctx->seg_mode,
                    &ctx->raw, &ctx->raw_tmp, &ctx->raw_off, &ctx->raw_cnt, &ctx->raw_in_tmp,
                    &ctx->cand, &ctx->cand_off, &ctx->cand_n, &ctx->active, &ctx->items,
                    &ctx->results, &ctx->next_buf, &ctx->gstate, &ctx->seg_item_start,
                    &ctx->seg_item_cnt, &ctx->segdp, &ctx->best_next, &ctx->bound_items,
                    &ctx->bound_res, &ctx->out_splits, &ctx->out_times, &ctx->out_count,
                    &ctx->out_tmax, &ctx->out_obj, &ctx->out_status, &ctx->out_err})
    b->release();
  for (PinBuf* b : {&ctx->h_range, &ctx->h_stats, &ctx->h_segdp, &ctx->h_misc}) b->release();
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PP_OK;
}

const char* pp_ctx_last_error(const pp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int pp_ctx_set_tuning(pp_ctx* ctx, const pp_tuning* t) {
  if (!ctx || !t || t->first_wave < 1) return PP_ERR_INVALID;
  ctx->tuning = *t;
  return PP_OK;
}

int pp_ctx_get_stats(const pp_ctx* ctx, pp_stats* out) {
  if (!ctx || !out) return PP_ERR_INVALID;
  *out = ctx->stats;
  return PP_OK;
}

int pp_ctx_set_stream(pp_ctx* ctx, void* stream) {
  if (!ctx) return PP_ERR_INVALID;
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  ctx->stream = static_cast<cudaStream_t>(stream);
  ctx->own_stream = false;
  return PP_OK;
}

int pp_eval_objective(const double* times, int64_t m, int32_t c, int32_t d, double* out) {
  // eval_objective (microbatch.cpp:109-120); host helper for the C++ API.
  if (!times || !out || m <= 0) return PP_ERR_INVALID;
  if (c < 1 || d < 1) return PP_ERR_INVALID;
  double max_t = 0.0, sum = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    max_t = (max_t < times[i]) ? times[i] : max_t;
    sum += times[i];
  }
  *out = static_cast<double>(c - 1) * max_t + sum / static_cast<double>(d);
  return PP_OK;
}

int pp_plan_grid_device(pp_ctx* ctx, const pp_sample* d_samples, const int64_t* d_seg_offsets,
                        const int64_t* h_seg_offsets, int32_t n_seg, int32_t presorted,
                        const pp_grid_desc* grid, const pp_model_desc* model,
                        const pp_dp_options* opts, pp_plan_out* d_out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!opts || !d_out || n_seg < 1 || !h_seg_offsets || !d_seg_offsets)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if ((rc = validate_opts(ctx, *opts))) return rc;
  PlanCall c;
  c.d_samples = d_samples;
  c.d_seg_off = d_seg_offsets;
  c.h_seg_off = h_seg_offsets;
  c.n_seg = n_seg;
  c.presorted = presorted;
  c.grid = grid;
  c.model = model;
  c.opts = *opts;
  c.d_ordered = d_out->ordered;
  c.d_splits = d_out->splits;
  c.d_times = d_out->mb_times;
  c.d_count = d_out->count;
  c.d_tmax = d_out->t_max_used;
  c.d_obj = d_out->objective;
  c.d_status = d_out->status;
  c.d_err = d_out->err_sample_id;
  return run_plan(ctx, c);
}

int pp_plan_grid(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets, int32_t n_seg,
                 int32_t presorted, const pp_grid_desc* grid, const pp_model_desc* model,
                 const pp_dp_options* opts, pp_plan_out* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!samples || !seg_offsets || n_seg < 1 || !opts || !out)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if ((rc = validate_opts(ctx, *opts))) return rc;
  const int64_t total = seg_offsets[n_seg];
  cudaStream_t st = ctx->stream;
  PP_CUDA(ctx->samples.ensure(std::max<int64_t>(total, 1) * sizeof(pp_sample)));
  PP_CUDA(ctx->seg_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->ordered.ensure(std::max<int64_t>(total, 1) * sizeof(pp_sample)));
  PP_CUDA(ctx->out_splits.ensure(std::max<int64_t>(total, 1) * sizeof(int32_t)));
  PP_CUDA(ctx->out_times.ensure(std::max<int64_t>(total, 1) * sizeof(double)));
  PP_CUDA(ctx->out_count.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->out_tmax.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->out_obj.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->out_status.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->out_err.ensure(n_seg * sizeof(int64_t)));
  if (total > 0)
    PP_CUDA(cudaMemcpyAsync(ctx->samples.p, samples, total * sizeof(pp_sample), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->seg_off.p, seg_offsets, (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  pp_plan_out d{};
  d.ordered = ctx->ordered.as<pp_sample>();
  d.splits = ctx->out_splits.as<int32_t>();
  d.mb_times = ctx->out_times.as<double>();
  d.count = ctx->out_count.as<int32_t>();
  d.t_max_used = ctx->out_tmax.as<double>();
  d.objective = ctx->out_obj.as<double>();
  d.status = ctx->out_status.as<int32_t>();
  d.err_sample_id = ctx->out_err.as<int64_t>();
  rc = pp_plan_grid_device(ctx, ctx->samples.as<pp_sample>(), ctx->seg_off.as<int64_t>(), seg_offsets,
                           n_seg, presorted, grid, model, opts, &d);
  if (rc) return rc;
  auto d2h = [&](void* dst, const void* src, size_t bytes) {
    return dst && bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) : cudaSuccess;
  };
  PP_CUDA(d2h(out->ordered, d.ordered, total * sizeof(pp_sample)));
  PP_CUDA(d2h(out->splits, d.splits, total * sizeof(int32_t)));
  PP_CUDA(d2h(out->mb_times, d.mb_times, total * sizeof(double)));
  PP_CUDA(d2h(out->count, d.count, n_seg * sizeof(int32_t)));
  PP_CUDA(d2h(out->t_max_used, d.t_max_used, n_seg * sizeof(double)));
  PP_CUDA(d2h(out->objective, d.objective, n_seg * sizeof(double)));
  PP_CUDA(d2h(out->status, d.status, n_seg * sizeof(int32_t)));
  PP_CUDA(d2h(out->err_sample_id, d.err_sample_id, n_seg * sizeof(int64_t)));
  PP_CUDA(cudaStreamSynchronize(st));
  return PP_OK;
}

int pp_order_samples(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets, int32_t n_seg,
                     pp_sample* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!samples || !seg_offsets || n_seg < 1 || !out) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  for (int s = 0; s < n_seg; ++s)
    if (seg_offsets[s + 1] <= seg_offsets[s]) return fail(ctx, PP_ERR_INVALID, "mini-batch is empty");
  const int64_t total = seg_offsets[n_seg];
  cudaStream_t st = ctx->stream;
  PP_CUDA(ctx->samples.ensure(total * sizeof(pp_sample)));
  PP_CUDA(ctx->seg_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->ordered.ensure(total * sizeof(pp_sample)));
  PP_CUDA(ctx->in_d.ensure(total * sizeof(double)));
  PP_CUDA(ctx->tgt_d.ensure(total * sizeof(double)));
  PP_CUDA(ctx->range.ensure(6 * sizeof(unsigned long long)));
  PP_CUDA(ctx->h_range.ensure(6 * sizeof(unsigned long long)));
  PP_CUDA(ctx->sort_keys.ensure(total * 6 * sizeof(unsigned long long)));
  PP_CUDA(ctx->sort_vals.ensure(total * 2 * sizeof(uint32_t)));
  PP_CUDA(cudaMemcpyAsync(ctx->samples.p, samples, total * sizeof(pp_sample), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->seg_off.p, seg_offsets, (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(launch_segmented_sort(ctx->samples.as<pp_sample>(), ctx->seg_off.as<int64_t>(), seg_offsets,
                                n_seg, total, 0, ctx->range.as<unsigned long long>(),
                                ctx->h_range.as<unsigned long long>(),
                                ctx->sort_keys.as<unsigned long long>(), ctx->sort_vals.as<uint32_t>(),
                                ctx->ordered.as<pp_sample>(), ctx->in_d.as<double>(),
                                ctx->tgt_d.as<double>(), st));
  PP_CUDA(cudaMemcpyAsync(out, ctx->ordered.p, total * sizeof(pp_sample), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  return PP_OK;
}

int pp_candidate_range(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets,
                       int32_t n_seg, int32_t presorted, const pp_grid_desc* grid,
                       const pp_model_desc* model, double cap, double* t_min, double* t_max) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!samples || !seg_offsets || n_seg < 1 || !t_min || !t_max)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  const int64_t total = seg_offsets[n_seg];
  if (total <= 0) return fail(ctx, PP_ERR_INVALID, "mini-batch is empty");
  cudaStream_t st = ctx->stream;
  GridDev g{};
  if ((rc = upload_grid(ctx, grid, model, &g))) return rc;
  PP_CUDA(ctx->samples.ensure(total * sizeof(pp_sample)));
  PP_CUDA(ctx->seg_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->ordered.ensure(total * sizeof(pp_sample)));
  PP_CUDA(ctx->in_d.ensure(total * sizeof(double)));
  PP_CUDA(ctx->tgt_d.ensure(total * sizeof(double)));
  PP_CUDA(ctx->range.ensure(6 * sizeof(unsigned long long)));
  PP_CUDA(ctx->h_range.ensure(6 * sizeof(unsigned long long)));
  PP_CUDA(ctx->sort_keys.ensure(total * 6 * sizeof(unsigned long long)));
  PP_CUDA(ctx->sort_vals.ensure(total * 2 * sizeof(uint32_t)));
  PP_CUDA(ctx->row_w.ensure(total * sizeof(int)));
  PP_CUDA(ctx->stats_d.ensure(n_seg * sizeof(SegStats)));
  PP_CUDA(ctx->h_stats.ensure(n_seg * sizeof(SegStats)));
  PP_CUDA(cudaMemcpyAsync(ctx->samples.p, samples, total * sizeof(pp_sample), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->seg_off.p, seg_offsets, (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(launch_segmented_sort(ctx->samples.as<pp_sample>(), ctx->seg_off.as<int64_t>(), seg_offsets,
                                n_seg, total, presorted, ctx->range.as<unsigned long long>(),
                                ctx->h_range.as<unsigned long long>(),
                                ctx->sort_keys.as<unsigned long long>(), ctx->sort_vals.as<uint32_t>(),
                                ctx->ordered.as<pp_sample>(), ctx->in_d.as<double>(),
                                ctx->tgt_d.as<double>(), st));
  SegStats* hs = ctx->h_stats.as<SegStats>();
  for (int s = 0; s < n_seg; ++s) hs[s] = SegStats{~0ULL, 0ULL, 0ULL, INT_MAX, 0, 0};
  PP_CUDA(cudaMemcpyAsync(ctx->stats_d.p, hs, n_seg * sizeof(SegStats), cudaMemcpyHostToDevice, st));
  // interval 0: the statistics are over the raw slice times
  PP_CUDA(launch_row_scan(g, nullptr, nullptr, ctx->in_d.as<double>(), ctx->tgt_d.as<double>(),
                          ctx->seg_off.as<int64_t>(), n_seg, total, cap, 0.0, ctx->row_w.as<int>(),
                          ctx->stats_d.as<SegStats>(), st));
  PP_CUDA(cudaMemcpyAsync(hs, ctx->stats_d.p, n_seg * sizeof(SegStats), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  auto inv = [](unsigned long long k) {
    unsigned long long u = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
    double d;
    std::memcpy(&d, &u, 8);
    return d;
  };
  for (int s = 0; s < n_seg; ++s) {
    const bool any = hs[s].kmin != ~0ULL;
    t_min[s] = (hs[s].flags & 2) ? -INFINITY : any ? inv(hs[s].kmin) : (hs[s].flags & 1) ? INFINITY : NAN;
    t_max[s] = (hs[s].flags & 1) ? INFINITY : any ? inv(hs[s].kmax) : (hs[s].flags & 2) ? -INFINITY : NAN;
  }
  return PP_OK;
}

int pp_plan_tables(pp_ctx* ctx, const double* slice_time, const double* slice_mem, int64_t n,
                   const pp_dp_options* opts, int32_t* splits, double* mb_times, int32_t* count,
                   double* t_max_used, double* objective, int64_t* err_index) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!opts) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if (n <= 0) return fail(ctx, PP_ERR_INVALID, "cannot partition an empty sample list");
  if ((rc = validate_opts(ctx, *opts))) return rc;
  if (!slice_time || !slice_mem || !splits || !count || !t_max_used || !objective)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if (n >= (1 << 30)) return fail(ctx, PP_ERR_INVALID, "too many samples");
  const int64_t tri = n * (n + 1) / 2;
  cudaStream_t st = ctx->stream;
  PP_CUDA(ctx->tabT.ensure(tri * sizeof(double)));
  PP_CUDA(ctx->tabM.ensure(tri * sizeof(double)));
  PP_CUDA(ctx->seg_off.ensure(2 * sizeof(int64_t)));
  PP_CUDA(ctx->ordered.ensure(n * sizeof(pp_sample)));
  PP_CUDA(ctx->out_splits.ensure(n * sizeof(int32_t)));
  PP_CUDA(ctx->out_times.ensure(n * sizeof(double)));
  PP_CUDA(ctx->out_count.ensure(sizeof(int32_t)));
  PP_CUDA(ctx->out_tmax.ensure(sizeof(double)));
  PP_CUDA(ctx->out_obj.ensure(sizeof(double)));
  PP_CUDA(ctx->out_status.ensure(sizeof(int32_t)));
  PP_CUDA(ctx->out_err.ensure(sizeof(int64_t)));
  std::vector<pp_sample> ids(n);
  for (int64_t k = 0; k < n; ++k) ids[k] = pp_sample{k, 1, 0};  // err_id == ordered index
  const int64_t so[2] = {0, n};
  PP_CUDA(cudaMemcpyAsync(ctx->tabT.p, slice_time, tri * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->tabM.p, slice_mem, tri * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->seg_off.p, so, sizeof(so), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->ordered.p, ids.data(), n * sizeof(pp_sample), cudaMemcpyHostToDevice, st));
  PlanCall c;
  c.d_tabT = ctx->tabT.as<double>();
  c.d_tabM = ctx->tabM.as<double>();
  c.d_seg_off = ctx->seg_off.as<int64_t>();
  c.h_seg_off = so;
  c.n_seg = 1;
  c.presorted = 1;
  c.opts = *opts;
  c.d_ordered = ctx->ordered.as<pp_sample>();
  c.d_splits = ctx->out_splits.as<int32_t>();
  c.d_times = ctx->out_times.as<double>();
  c.d_count = ctx->out_count.as<int32_t>();
  c.d_tmax = ctx->out_tmax.as<double>();
  c.d_obj = ctx->out_obj.as<double>();
  c.d_status = ctx->out_status.as<int32_t>();
  c.d_err = ctx->out_err.as<int64_t>();
  rc = run_plan(ctx, c);
  if (rc) return rc;
  int32_t status = 0;
  int64_t err = -1;
  PP_CUDA(cudaMemcpyAsync(&status, c.d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(&err, c.d_err, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(count, c.d_count, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(t_max_used, c.d_tmax, sizeof(double), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(objective, c.d_obj, sizeof(double), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(splits, c.d_splits, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (mb_times) PP_CUDA(cudaMemcpyAsync(mb_times, c.d_times, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  if (err_index) *err_index = err;
  if (status == PP_ERR_INFEASIBLE_SAMPLE)
    return fail(ctx, status, "sample does not fit the per-micro-batch memory cap alone");
  if (status == PP_ERR_INFEASIBLE) return fail(ctx, status, "no feasible partition under the memory cap");
  return status;
}

}  // extern "C"
