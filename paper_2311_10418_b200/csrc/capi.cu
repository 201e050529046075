// capi.cu — pp_ctx and the C-ABI entry points (include/pipeplan_b200.h).
//
// Host-side orchestration of one planning call over n_seg independent
// mini-batches (the reference plans each with order_samples -> make_slice_cost
// -> dp_partition, src/planner.cpp:42,64-65; batches come from run_plan's
// worker pool, src/driver.cpp:222-242):
//
//   1. segmented sort                          (sort.cu)  order_samples(Sort)
//   2. cost pass A: Rm(i), singleton check,     (cost.cu)  microbatch.cpp:228-251
//      candidate statistics, tile widths
//   3. tile offsets, cost pass B: band tiles + (cost.cu)  microbatch.cpp:237-243,253-269
//      candidate bitmap / raw list
//   4. candidate compaction                     (cost.cu/sort.cu)
//   5. bound + minimax pass (c > 1)             (dp.cu)    microbatch.cpp:274-279
//   6. candidate waves: DP per (mb, t) +        (dp.cu)    microbatch.cpp:289-318
//      in-order selection, until every
//      mini-batch hit the reference's break
//   7. assembly                                 (dp.cu)    microbatch.cpp:322-335
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
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <string>
#include <chrono>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "pp_internal.cuh"

namespace ppb {
// sort.cu
cudaError_t launch_segmented_sort(const pp_sample* d_in, const int64_t* d_seg_off,
                                  const int64_t* h_seg_off, int n_seg, int64_t total,
                                  int presorted, unsigned long long* d_range,
                                  unsigned long long* h_range, unsigned long long* d_keys,
                                  uint32_t* d_vals, pp_sample* d_out, double* d_in_len,
                                  double* d_tgt_len, int32_t* d_perm, cudaStream_t st);
cudaError_t launch_segmented_sort_u64(unsigned long long* keys, unsigned long long* tmp,
                                      const int64_t* off, const unsigned long long* cnt,
                                      const int* seg_mode, int want_mode, int* in_tmp, int n_seg,
                                      cudaStream_t st);
// cost.cu
cudaError_t launch_brackets(const CostGrid& g, int max_n, AxisPos* mbp, const double* in_d,
                            const double* tgt_d, int64_t total, AxisPos* pin, AxisPos* ptg,
                            cudaStream_t st);
cudaError_t launch_cost_pass(int pass, const CostGrid& g, const double* tabT, const double* tabM,
                             const double* in_d, const double* tgt_d, const AxisPos* pin,
                             const AxisPos* ptg, const int64_t* seg_off, const int* blk_base, int n_seg,
                             int total_blocks, int max_n, const AxisPos* mbp, double cap,
                             double interval, int* row_w, int* row_fb, int* blk_W, SegStats* stats,
                             const int64_t* tile_off, const int64_t* seg_band_base, double* band,
                             double exit_thresh, unsigned int* small_bm, const double* tau,
                             double lo_thresh, int bisect, int sorted_in, int reuse, double* cmin,
                             short* colbase, int* chunk_nv, int* wrote_cmin, int nostore, cudaStream_t st);
bool band_run_applies(const CostGrid& g, const double* tabT, int reuse, const double* tau, int sorted_in);
// gtab.cu
cudaError_t launch_gtab_need(const int64_t* seg_off, const int* blk_base, int n_seg, int total_blocks,
                             int max_blocks, const int* blk_W, const double* in_d, int* need, cudaStream_t st);
cudaError_t launch_gtab_offsets(const int* need, int nK, int64_t* row_off, long long* total, cudaStream_t st);
cudaError_t launch_gtab_fill(const CostGrid& g, double cap, const AxisPos* mbp, int nK, const int* need,
                             const int64_t* row_off, double* G, double* G1, cudaStream_t st);
cudaError_t launch_gtab_gbase(const double* in_d, int64_t total, const int64_t* row_off, int* gbase,
                              cudaStream_t st);
cudaError_t launch_gtab_bins(const int64_t* seg_off, int n_seg, const double* in_d, const int* gbase,
                             const int* need, const double* G, double interval, const double* tau,
                             unsigned int* small_bm, SegStats* stats, int nK, const int64_t* row_off, int* rf,
                             double* rlo, int max_n, cudaStream_t st);
cudaError_t launch_full_rows(const int64_t* seg_off, const int* blk_base, int n_seg, int total_blocks,
                             int* row_w, int* blk_W, cudaStream_t st);
cudaError_t launch_band_cand(const int64_t* seg_off, const int* blk_base, int n_seg, int total_blocks,
                             const int* blk_W, const int64_t* tile_off, const int64_t* seg_band_base,
                             const double* band, double interval, const SegStats* stats,
                             unsigned int* bitmap, const int64_t* bitmap_off, const int* seg_mode,
                             unsigned long long* cand_raw, const int64_t* cand_raw_off,
                             unsigned long long* cand_raw_cnt, const short* colbase, const int* row_w,
                             cudaStream_t st);
cudaError_t launch_tile_offsets(const int* blk_W, const int* blk_base, int n_seg, int64_t* tile_off,
                                SegStats* stats, cudaStream_t st);
cudaError_t launch_cand_bitmap(const unsigned int* bitmap, const int64_t* bitmap_off,
                               const SegStats* stats, const int* seg_mode, int n_seg,
                               const unsigned int* small_bm, double interval,
                               const int64_t* cand_off, double* cand, int* cand_n, cudaStream_t st);
cudaError_t launch_cand_unique(const unsigned long long* keys_a, const unsigned long long* keys_b,
                               const int* in_b, const int64_t* raw_off,
                               const unsigned long long* raw_cnt, const int* seg_mode, int n_seg,
                               const int64_t* cand_off, double* cand, int* cand_n, cudaStream_t st);
// dp.cu
size_t dp_smem_fixed();
size_t dp_state_bytes(int mode, int entries);
int dp_state_stride(int entries);
cudaError_t launch_dp_pass(int mode, const WorkItem* items, int n_items, size_t smem_state,
                           int state_global, int sanitize, size_t smem_budget, const int64_t* seg_off,
                           const int* blk_base, const int* blk_W, const int64_t* tile_off,
                           const int64_t* seg_band_base, const double* band, const double* cand,
                           const int64_t* cand_off, ItemResult* res, int* next_buf, double* gstate,
                           int res_by_seg, const double* cmin, double t_margin,
                           unsigned long long* cols_streamed, ItemResult* res2, const int* gbase,
                           cudaStream_t st);
cudaError_t launch_seg_set_bound(const ItemResult* bound_res, int replicas, SegDP* dp, int n_seg,
                                 cudaStream_t st);
cudaError_t launch_mb_shapes(const pp_sample* ordered, const int64_t* seg_off, const int32_t* splits,
                             const int64_t* mb_off, int n_seg, int64_t n_mb, pp_padded_shape* shapes,
                             cudaStream_t st);
cudaError_t launch_op_costs(const CostGrid& g, const double* le_st, const double* ld_st, int stages,
                            const pp_padded_shape* shapes, int64_t n, double* t_f, double* t_b,
                            double* act, cudaStream_t st);
cudaError_t launch_recompute_select(const int64_t* mb_off, int n_seg, int C, int n_tries, const int* tries,
                                    int64_t n_mb, const double* tf_all, const double* tb_all,
                                    const double* act_all, const double* limits, int32_t* strategy,
                                    int32_t* violating, double* t_f, double* t_b, double* act, cudaStream_t st);
size_t dp_coop_parts_bytes(int grid);
size_t order_search_slot_bytes(int64_t max_m, int C);
int order_search_warps(int64_t n_items, int C, size_t slot_bytes, size_t budget);
size_t order_search_item_bytes();
cudaError_t launch_emit_plans(const double* tf, const double* tb, const double* act, const int64_t* mb_off, int n_seg,
                              int C, const double* limits, double comm_latency, int64_t max_m, const int* order,
                              int f1b, char* scratch, size_t slot_bytes, int warps, void* items, int* ok, int* seen,
                              int* out_ins, int* out_nins, double* makespan, double* bubble, int* deadlock,
                              double* dev_stats, int* status, cudaStream_t st);
size_t order_search_best_bytes();
size_t ingest_scratch_bytes(int64_t n_bytes);
cudaError_t launch_load_records(const unsigned char* d_bytes, int64_t n, long long max_seq_len, char* scratch,
                                size_t scratch_bytes, pp_sample* d_out, int64_t capacity, int64_t* n_records,
                                int64_t* n_lines_out, int64_t* err_line, int32_t* err_kind, int64_t* err_byte,
                                cudaStream_t st);
size_t draw_scratch_bytes(int64_t n);
cudaError_t launch_sim_1f1b(const double* tf, const double* tb, const double* act, const int64_t* mb_off,
                            int n_seg, int C, double comm_latency, int64_t max_m, char* scratch,
                            size_t slot_bytes, int warps, void* items, cudaStream_t st);
cudaError_t launch_truncate(const pp_sample* in, int64_t n, long long max_len, pp_sample* out, cudaStream_t st);
cudaError_t launch_minibatch_stats(const pp_sample* s, const int64_t* off, int n_seg, long long max_len,
                                   long long* bins, long long* st6, pp_padded_shape* naive, cudaStream_t st);
cudaError_t launch_dp_padded(const pp_padded_shape* sh, const int64_t* mb_off, int n_seg, long long* st6,
                             cudaStream_t st);
cudaError_t launch_broadcast_rows(const double* tf1, const double* tb1, const double* ac1, int C, int64_t rows,
                                  double* tf, double* tb, double* ac, cudaStream_t st);
cudaError_t launch_draw_minibatches(const pp_sample* d_samples, int64_t n, long long budget, char* scratch,
                                    size_t scratch_bytes, int64_t* d_seg_offsets, int64_t* n_seg, cudaStream_t st);
cudaError_t launch_order_search(const double* tf, const double* tb, const double* act,
                                const int64_t* mb_off, int n_seg, int C, const double* limits,
                                int k, int kfact, double comm_latency, int64_t max_m, double* pred,
                                int* assign, int* cl_idx, int* cl_off, int* cl_k, char* scratch,
                                size_t slot_bytes, int warps, void* items, double* item_stats,
                                int* order, double* makespan, double* bubble, int* deadlock,
                                double* dev_stats, int* status, int rwin, void* best, double* best_stats, cudaStream_t st);
int dp_coop_grid(int device);
cudaError_t launch_pack_slots(const int32_t* count, const int32_t* status, const double* tmax,
                              const double* obj, const int32_t* splits, const int32_t* order,
                              const int64_t* seg_off, int n_seg, int n_max, long long* slots,
                              cudaStream_t st);
cudaError_t launch_dp_coop(int mode, int sanitize, const WorkItem& it, int grid, const int64_t* seg_off,
                           const int* blk_base, const int* blk_W, const int64_t* tile_off,
                           const int64_t* seg_band_base, const double* band, const double* cand,
                           const int64_t* cand_off, ItemResult* res, int res_slot, int* next_buf,
                           double* gstate, void* parts, cudaStream_t st);
cudaError_t launch_seg_init(const ItemResult* bound_res, int has_bound, int replicas,
                            const int64_t* cand_off, const int* cand_n, const double* cand,
                            const int* active, const SegStats* tsingle, double margin, SegDP* dp,
                            int n_seg, cudaStream_t st);
cudaError_t launch_select(const WorkItem* items, const ItemResult* res, const int* seg_item_start,
                          const int* seg_item_cnt, const int* next_buf, int* best_next,
                          const int64_t* seg_off, const double* cand, const int64_t* cand_off,
                          int stage_count, int replicas, SegDP* dps, int n_seg, cudaStream_t st);
cudaError_t launch_finalize(const SegDP* dps, const int* best_next, const int64_t* seg_off,
                            const int* blk_base, const int64_t* tile_off, const int64_t* seg_band_base,
                            const double* band, const SegStats* stats, const short* colbase,
                            const pp_sample* ordered, int stage_count, int replicas, int max_n, int n_seg,
                            int32_t* splits, double* mb_times, int32_t* count, double* t_max_used,
                            double* objective, int32_t* status, int64_t* err_id, const DpPrice* price,
                            int price_lay, cudaStream_t st);
}  // namespace ppb

using namespace ppb;

namespace {

constexpr size_t kDpSmemLimit = 190 * 1024;
// A DP launch over few, very long mini-batches (C5: 65,536 samples, rows up
// to n wide) runs each pass as one cooperative kernel over the whole GPU
// (dp_coop.cu) instead of one CTA per pass.
constexpr int kCoopMinN = 16384;
constexpr int kCoopMaxItems = 8;
  // fixed + state budget before DP state spills to global

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

// Small transfers of the planning path (offsets, work lists, per-segment
// statistics, read-backs) run as a one-CTA copy kernel through mapped pinned
// memory (UVA: a cudaMallocHost pointer is valid on the device), never on a
// copy engine: a host-buffer call keeps the engines busy with tens of MB of
// samples and plans, and a small cudaMemcpyAsync — pageable or not — can
// queue behind them for milliseconds while the planning stream waits on it.
// Every thread issues its (up to four) 16-byte loads before any store, so a
// copy of up to 64 KB costs one PCIe round trip, not one per 1 KB.
__global__ void __launch_bounds__(1024) small_copy_kernel(const unsigned int* __restrict__ src,
                                                          unsigned int* __restrict__ dst, size_t words) {
  size_t done = 0;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const size_t nv = words / 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (size_t k = threadIdx.x; k < nv; k += 4 * (size_t)blockDim.x) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t q = k + (size_t)u * blockDim.x;
        if (q < nv) v[u] = s4[q];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t q = k + (size_t)u * blockDim.x;
        if (q < nv) d4[q] = v[u];
      }
    }
    done = nv * 4;
  }
  for (size_t k = done + threadIdx.x; k < words; k += blockDim.x) dst[k] = src[k];
}
cudaError_t small_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  const size_t words = (bytes + 3) / 4;
  const unsigned threads = words >= 4096 ? 1024u : words >= 512 ? 256u : 64u;
  small_copy_kernel<<<1, threads, 0, st>>>(static_cast<const unsigned int*>(src), static_cast<unsigned int*>(dst),
                                           words);
  return cudaGetLastError();
}

// Pinned staging arena for small_copy uploads: bump-allocated within a
// planning call (every call ends with its stream synchronised, so the next
// call starts over); a request that does not fit waits for the stream.
struct PinArena {
  PinBuf buf;
  size_t off = 0;
  void* take(size_t bytes, cudaStream_t st) {
    bytes = (bytes + 15) / 16 * 16;
    if (off + bytes > buf.cap) {
      if (cudaStreamSynchronize(st) != cudaSuccess) return nullptr;
      off = 0;
      if (bytes > buf.cap && buf.ensure(std::max<size_t>(bytes, (size_t)1 << 20)) != cudaSuccess) return nullptr;
    }
    void* p = static_cast<char*>(buf.p) + off;
    off += bytes;
    return p;
  }
};

// One staging set of a pipelined host-buffer worker (plan_host_chunks):
// device inputs and outputs of one chunk, the pinned segment offsets, and the
// events that order its copies against the compute stream.
struct HostSet {
  DevBuf samples, seg, ordered, order, splits, times, count, tmax, obj, status, err;
  PinBuf hoff;
  cudaEvent_t h2d = nullptr, d2h = nullptr;
  bool d2h_pending = false;
};

}  // namespace

struct pp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t pstream = nullptr;             // plan_host_pieces: this worker's prioritised stream
  std::string err;
  pp_tuning tuning{};
  pp_stats stats{};
  cudaEvent_t ev[4]{};
  // device scratch
  DevBuf samples, seg_off, ordered, in_d, tgt_d, sort_keys, sort_vals, range;
  DevBuf grid_ax, grid_cells, layouts, tabT, tabM, mbp, pin, ptg, tau;
  int64_t band_total = 0;
  DevBuf row_w, row_fb, blk_base, blk_W, tile_off, stats_d, band_base, band, bitmap, bitmap_off, seg_mode,
      raw, raw_tmp, raw_off, raw_cnt, raw_in_tmp, cand, cand_off, cand_n, active;
  DevBuf items, results, next_buf, gstate, seg_item_start, seg_item_cnt, segdp, best_next,
      bound_items, bound_res;
  DevBuf out_splits, out_times, out_count, out_tmax, out_obj, out_status, out_err;
  PinBuf h_range, h_stats, h_segdp;
  DevBuf small_bm, coop_state, coop_parts, shapes, stage_lay, mb_off, oc_tf, oc_tb, oc_act, cmin, dp_cols,
      colbase, chunk_nv, perm;
  // injection-order search (sched.cu)
  DevBuf os_tf, os_tb, os_act, os_off, os_lim, os_pred, os_assign, os_idx, os_cloff, os_clk, os_scratch,
      os_items, os_istats, os_order, os_ms, os_bub, os_dl, os_ds, os_status, os_best, os_bstats, em_ins, em_nins;
  // dataset ingest (ingest.cu)
  DevBuf ing_bytes, ing_scratch, ing_out, ing_off;
  // padding report (report.cu)
  DevBuf rp_samples, rp_trunc, rp_off, rp_ordered, rp_splits, rp_times, rp_count, rp_tmax, rp_obj, rp_status,
      rp_err, rp_tf, rp_tb, rp_act, rp_mboff, rp_st6, rp_bins, rp_naive, rp_items, rp_row;
  // host copy of the uploaded grid (restricted to the recompute strategy)
  // for the monotonicity certificate of cost pass A
  std::vector<double> h_ax, h_cells;
  std::vector<Layout> h_lay;
  int h_nm = 0, h_ns = 0, h_encdec = 0;
  double exit_thresh = INFINITY;  // last call's pass-A row-exit threshold
  double trunc_margin = INFINITY; // candidate-pass truncation margin 2E (+inf: off)
  bool compact = false;           // the band holds compact chunk records (pp_internal.cuh)
  bool priced = false;            // no band: the DP prices its slices in-kernel (dp.cu PRICE)
  bool gtab = false;              // no band: the call's shared slice table (gtab.cu)
  DevBuf gt_need, gt_off, gt_total, gt_G, gt_base, gt_rf, gt_rlo;
  DevBuf rc_tab, rc_lim, rc_out;  // select_recomputation
  PinBuf h_gt_total;
  int64_t gtab_entries = 0;
  DpPrice price{};                // its inputs
  int price_lay = 0;              // its layout class (kLayDec1 / kLayEncDec2)
  // pipelined host-buffer worker (plan_host_chunks): copy stream + two sets
  cudaStream_t cstream = nullptr;
  cudaStream_t ostream = nullptr;             // plan_host_pieces: device->host copies
  PinArena arena;                             // small_copy uploads of the planning path
  PinBuf h_word;                              // small_copy read-back scratch
  std::vector<cudaEvent_t> piece_ev;          // plan_host_pieces: inputs in / part planned
  PinBuf piece_off;                           // plan_host_pieces: part-relative offsets (pinned)
  HostSet hset[2];
  CostGrid grid_dev{};            // device view of the uploaded grid
  bool grid_valid = false;
  double tau_interval = -1.0;     // interval the device bin thresholds were built for
  // concurrent sub-batch contexts (pp_tuning::streams), created on demand
  std::vector<pp_ctx*> subs;
  cudaEvent_t ev_in = nullptr;
  cudaEvent_t ev_done = nullptr;  // (sub-context) its stream's work of a plan_split part
  // per-launch event pairs for kernel timing (pp_stats::ms_kernel)
  std::vector<cudaEvent_t> kev;
  std::vector<int> kcat;
  size_t kused = 0;
  std::vector<DevBuf*> all_bufs() {
    return {&samples, &seg_off, &ordered, &in_d, &tgt_d, &sort_keys, &sort_vals, &range, &grid_ax,
            &grid_cells, &layouts, &tabT, &tabM, &mbp, &pin, &ptg, &tau, &row_w, &row_fb, &blk_base, &blk_W, &tile_off,
            &stats_d, &band_base, &band, &bitmap, &bitmap_off, &seg_mode, &raw, &raw_tmp, &raw_off,
            &raw_cnt, &raw_in_tmp, &cand, &cand_off, &cand_n, &active, &items, &results, &next_buf,
            &gstate, &seg_item_start, &seg_item_cnt, &segdp, &best_next, &bound_items, &bound_res,
            &out_splits, &out_times, &out_count, &out_tmax, &out_obj, &out_status, &out_err,
            &small_bm, &coop_state, &coop_parts, &shapes, &stage_lay, &mb_off, &oc_tf, &oc_tb, &oc_act,
            &cmin, &dp_cols, &colbase, &chunk_nv, &perm, &gt_need, &gt_off, &gt_total, &gt_G, &gt_base, &gt_rf, &gt_rlo, &rc_tab, &rc_lim, &rc_out,
            &os_tf, &os_tb, &os_act, &os_off, &os_lim, &os_pred, &os_assign, &os_idx, &os_cloff, &os_clk,
            &os_scratch, &os_items, &os_istats, &os_order, &os_ms, &os_bub, &os_dl, &os_ds, &os_status, &os_best, &os_bstats, &em_ins, &em_nins,
            &ing_bytes, &ing_scratch, &ing_out, &ing_off,
            &rp_samples, &rp_trunc, &rp_off, &rp_ordered, &rp_splits, &rp_times, &rp_count, &rp_tmax, &rp_obj,
            &rp_status, &rp_err, &rp_tf, &rp_tb, &rp_act, &rp_mboff, &rp_st6, &rp_bins, &rp_naive, &rp_items,
            &rp_row,
            &hset[0].samples, &hset[0].seg, &hset[0].ordered, &hset[0].order, &hset[0].splits,
            &hset[0].times, &hset[0].count, &hset[0].tmax, &hset[0].obj, &hset[0].status, &hset[0].err,
            &hset[1].samples, &hset[1].seg, &hset[1].ordered, &hset[1].order, &hset[1].splits,
            &hset[1].times, &hset[1].count, &hset[1].tmax, &hset[1].obj, &hset[1].status, &hset[1].err};
  }
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

// Record an event pair around one kernel launch (category = pp_stats
// ms_kernel index, see include/pipeplan_b200.h) so pp_stats reports
// per-kernel device time measured on the launching stream.
cudaError_t timed_begin(pp_ctx* ctx, int cat) {
  if (ctx->kused + 2 > ctx->kev.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      ctx->kev.push_back(e);
    }
  }
  ctx->kcat.push_back(cat);
  return cudaEventRecord(ctx->kev[ctx->kused++], ctx->stream);
}
cudaError_t timed_end(pp_ctx* ctx) { return cudaEventRecord(ctx->kev[ctx->kused++], ctx->stream); }

// NVTX ranges (header-only NVTX v3: free without a profiler attached): one
// per planning call / part / run_plan phase, and one per kernel launch named
// by its pp_stats category, so an Nsight Systems timeline shows the phases.
const char* const kNvtxCat[8] = {"pp sort", "pp cost setup", "pp cost pass A", "pp slice table / pass B",
                                 "pp DP bound (+first candidate)", "pp DP candidates", "pp candidate compaction",
                                 "pp selection / assembly"};
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

#define PP_TIMED(cat, x)            \
  do {                              \
    NvtxRange nvtx_(kNvtxCat[cat]); \
    PP_CUDA(timed_begin(ctx, cat)); \
    PP_CUDA(x);                     \
    PP_CUDA(timed_end(ctx));        \
  } while (0)

// PP_E2E_TRACE=1: host timestamps (µs since the first mark) of planning
// phases, to stderr (development aid).
void trace_mark(const char* what) {
  static const bool on = std::getenv("PP_E2E_TRACE") != nullptr;
  if (!on) return;
  static const auto t0 = std::chrono::steady_clock::now();
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  std::fprintf(stderr, "phase %9.1f us  %s\n", us, what);
}

int fail(pp_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

// Upload `bytes` of host memory to device memory on the ctx stream through
// the pinned arena and small_copy (see small_copy_kernel).
cudaError_t up(pp_ctx* ctx, void* d_dst, const void* h_src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  void* stage = ctx->arena.take(bytes, ctx->stream);
  if (!stage) return cudaErrorMemoryAllocation;
  std::memcpy(stage, h_src, bytes);
  return small_copy(d_dst, stage, bytes, ctx->stream);
}
// Device memory into PINNED host memory (a PinBuf) on the ctx stream; the
// caller synchronises the stream before reading it.
cudaError_t down(pp_ctx* ctx, void* h_pinned, const void* d_src, size_t bytes) {
  return small_copy(h_pinned, d_src, bytes, ctx->stream);
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
  int32_t* d_order = nullptr;
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
  // (a NaN interval is not rejected: the reference's `< 0` test passes it and
  // its `> 0` test then selects the exact candidate set, microbatch.cpp:225,263)
  if (o.t_max_interval < 0) return fail(ctx, PP_ERR_INVALID, "t_max_interval must be >= 0");
  return PP_OK;
}

// Upload the grid restricted to the recompute strategy, plus the distinct
// stage layouts.
int upload_grid(pp_ctx* ctx, const pp_grid_desc* g, const pp_model_desc* m, CostGrid* out) {
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
  std::vector<Layout> lay0;
  for (int s = 0; s < m->n_stages; ++s) {
    Layout l{m->encoder_layers[s] > 0 ? m->encoder_layers[s] : 0,
             m->decoder_layers[s] > 0 ? m->decoder_layers[s] : 0};
    if (l.enc == 0 && l.dec == 0) continue;
    bool seen = false;
    for (const auto& x : lay0) seen |= (x.enc == l.enc && x.dec == l.dec);
    if (!seen) lay0.push_back(l);
  }
  // Same grid, strategy and layouts as the previous call: the device tables
  // are current (planning the same model call after call is the common case).
  const int encdec = m->is_encoder_decoder ? 1 : 0;
  if (ctx->grid_valid && ctx->h_nm == nm && ctx->h_ns == ns && ctx->h_encdec == encdec &&
      ctx->h_ax == ax && ctx->h_cells == cells && ctx->h_lay.size() == lay0.size() &&
      std::equal(lay0.begin(), lay0.end(), ctx->h_lay.begin(),
                 [](const Layout& a, const Layout& b) { return a.enc == b.enc && a.dec == b.dec; })) {
    *out = ctx->grid_dev;
    return PP_OK;
  }
  ctx->grid_valid = false;
  // cost-kernel tables: values + mbs-direction differences (see CostGrid)
  std::vector<double4> tt(2 * (size_t)nm * ns);
  std::vector<double2> am(2 * (size_t)nm * ns);
  for (int kind = 0; kind < 2; ++kind)
    for (int mi = 0; mi < nm; ++mi)
      for (int si = 0; si < ns; ++si) {
        const int m1 = std::min(mi + 1, nm - 1);
        const double* c0 = &cells[kind * per + ((size_t)mi * ns + si) * 3];
        const double* c1 = &cells[kind * per + ((size_t)m1 * ns + si) * 3];
        volatile double d[3];  // IEEE subtraction, exactly the reference's c10 - c00
        for (int f = 0; f < 3; ++f) d[f] = c1[f] - c0[f];
        const size_t o = (size_t)kind * nm * ns + (size_t)mi * ns + si;
        tt[o] = make_double4(c0[0], c0[1], d[0], d[1]);
        am[o] = make_double2(c0[2], d[2]);
      }
  const std::vector<Layout>& lay = lay0;  // stages with (0, 0) layers contribute nothing to max()
  std::vector<LayoutD> layd;
  int used = 0;
  for (const auto& l : lay) {
    layd.push_back(LayoutD{(double)l.enc, (double)l.dec});
    used |= (l.enc > 0 ? 1 : 0) | (l.dec > 0 ? 2 : 0);
  }
  PP_CUDA(ctx->grid_ax.ensure(ax.size() * sizeof(double)));
  PP_CUDA(ctx->grid_cells.ensure(tt.size() * sizeof(double4) + am.size() * sizeof(double2)));
  PP_CUDA(ctx->layouts.ensure(std::max<size_t>(layd.size(), 1) * sizeof(LayoutD)));
  double4* d_tt = ctx->grid_cells.as<double4>();
  double2* d_am = reinterpret_cast<double2*>(d_tt + tt.size());
  PP_CUDA(cudaMemcpyAsync(ctx->grid_ax.p, ax.data(), ax.size() * sizeof(double),
                          cudaMemcpyHostToDevice, ctx->stream));
  PP_CUDA(cudaMemcpyAsync(d_tt, tt.data(), tt.size() * sizeof(double4), cudaMemcpyHostToDevice,
                          ctx->stream));
  PP_CUDA(cudaMemcpyAsync(d_am, am.data(), am.size() * sizeof(double2), cudaMemcpyHostToDevice,
                          ctx->stream));
  if (!layd.empty())
    PP_CUDA(cudaMemcpyAsync(ctx->layouts.p, layd.data(), layd.size() * sizeof(LayoutD),
                            cudaMemcpyHostToDevice, ctx->stream));
  ctx->h_ax = ax;
  ctx->h_cells = cells;
  ctx->h_lay = lay;
  ctx->h_nm = nm;
  ctx->h_ns = ns;
  ctx->h_encdec = m->is_encoder_decoder ? 1 : 0;
  out->nm = nm;
  out->ns = ns;
  out->n_lay = (int)layd.size();
  out->is_encdec = m->is_encoder_decoder ? 1 : 0;
  out->used = used;
  out->lay_class = kLayGeneric;
  out->le = 0.0;
  out->ld = 0.0;
  if (lay.size() == 1 && lay[0].enc == 0 && lay[0].dec > 0) {
    out->lay_class = kLayDec1;
    out->ld = (double)lay[0].dec;
  } else if (lay.size() == 2) {
    for (int k = 0; k < 2; ++k) {
      const Layout& e = lay[k];
      const Layout& d = lay[1 - k];
      if (e.enc > 0 && e.dec == 0 && d.enc == 0 && d.dec > 0) {
        out->lay_class = kLayEncDec2;
        out->le = (double)e.enc;
        out->ld = (double)d.dec;
      }
    }
  }
  out->mbs_ax = ctx->grid_ax.as<double>();
  out->seq_ax = ctx->grid_ax.as<double>() + nm;
  out->tt = d_tt;
  out->am = d_am;
  out->lay = ctx->layouts.as<LayoutD>();
  // The host staging vectors die at return: make the copies complete first.
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->grid_dev = *out;
  ctx->grid_valid = true;
  return PP_OK;
}

// Candidate-bin thresholds for cost pass B: tau[k] = the largest double
// T >= 0 with fl(T / I) <= k, k < 32 * kSmallBmWords.  Correctly rounded
// division by I > 0 is monotone in T, so ceil(fl(T / I)) = min{k : T <=
// tau[k]} for every T in [0, tau[last]] — the device then bins a slice time
// with compares only (microbatch.cpp:264 quantisation, no division).  Found by
// bisection over the ordered bit patterns of non-negative doubles, with the
// host's IEEE division.
void bin_thresholds(double I, std::vector<double>& tau) {
  tau.resize(32 * kSmallBmWords);
  for (int k = 0; k < (int)tau.size(); ++k) {
    const double kk = (double)k;
    uint64_t lo = 0, hi = 0x7ff0000000000000ULL;  // P(lo) true (0 / I = 0 <= k), P(+inf) false
    while (hi - lo > 1) {
      const uint64_t mid = lo + (hi - lo) / 2;
      double t;
      std::memcpy(&t, &mid, 8);
      volatile double q = t / I;
      if (q <= kk) lo = mid; else hi = mid;
    }
    std::memcpy(&tau[k], &lo, 8);
  }
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

double dkey_inv_host(unsigned long long k) {
  const unsigned long long u = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}

// ---------------------------------------------------------------------------
// Row-exit certificate for cost pass A (act_mem only).
//
// Pass A needs Rm(i) = the last j with !(M[i,j] > cap).  The reference prices
// every slice.  For slice [i, j) the padded shape is (mbs = j - i, running max
// of the lengths), both non-decreasing in j for ANY sample order, so if the
// exact (real-arithmetic) act_mem surface is non-decreasing in mbs and in the
// sequence length over the ranges this call can reach, the exact M[i,j] is
// non-decreasing in j.  The device value M~ differs from the exact M by at
// most E (bound below), hence once M~[i,j0] > cap + 2E every j >= j0 has
// M~[i,j] >= M[i,j] - E >= M[i,j0] - E >= M~[i,j0] - 2E > cap: the rest of the
// row is infeasible and pass A stops scanning it.  No result changes; only
// slices that provably fail the cap are skipped.
//
// Exact surface per field and kind (ProfileGrid::per_layer,
// cost_model.cpp:126-150): on cell (mi, si) with corners c00, c10 (mbs+1),
// c01 (seq+1), c11 the blend is bilinear in (tm, ts); tm, ts lie in [0, 1]
// inside the axes and leave it only in the first / last segment
// (extrapolation).  It is non-decreasing in tm iff (1-ts)(c10-c00) +
// ts(c11-c01) >= 0 over the reachable ts, and in ts iff (1-tm)(c01-c00) +
// tm(c11-c10) >= 0 over the reachable tm; both are linear, so the axis
// differences (ts, tm in [0, 1]) plus the two extrapolated end points are
// checked.  Adjacent cells agree on shared edges (continuity), max(0, .),
// non-negative layer multiples, sums and max over stages preserve order.
//
// Rounding bound: every field evaluation is ~10 IEEE operations on values of
// magnitude <= A (1 + 2|tm|)(1 + 2|ts|), A = max |cell|; a forward error
// analysis gives |v~ - v| <= 72 u A (1 + |tm|)(1 + |ts|) per weighted field,
// u = 2^-53; we use 128 u.  Returns +inf (no certificate: full scan) when a
// condition fails or is within 1e-12 relative of failing.
// Certified forward error bound of a slice value priced on the grid: the sum
// over `fields` [f0, f1] of the cell surfaces (0 t_f, 1 t_b, 2 act), scaled
// by the layer multiples of every stage layout.  Returns E with
// |computed - exact| <= E for every slice of the call, PROVIDED each used
// kind's surfaces are nondecreasing along both grid axes (checked here,
// including the extrapolated ends the call's micro-batch sizes and lengths
// reach) — so the exact value is nondecreasing in the slice end j of a row of
// a length-sorted segment.  +inf when not certified.  `k_ulp` sizes the
// per-value rounding budget (the blends, the layer products and the sums).
long double surface_error_bound(const pp_ctx* ctx, int max_n, const double seq_lo[2], const double seq_hi[2],
                                int f0, int f1, long double k_ulp) {
  const long double BAD = INFINITY;
  const int nm = ctx->h_nm, ns = ctx->h_ns;
  const double* mbs_ax = ctx->h_ax.data();
  const double* seq_ax = ctx->h_ax.data() + nm;
  auto tpos = [](const double* ax, int size, double x, int& seg) -> long double {
    seg = 0;
    if (size == 1) return 0.0L;
    while (seg + 2 < size && x >= ax[seg + 1]) ++seg;
    return ((long double)x - ax[seg]) / ((long double)ax[seg + 1] - ax[seg]);
  };
  int sg;
  const long double tm_lo = tpos(mbs_ax, nm, 1.0, sg);
  const int tm_lo_seg = sg;
  const long double tm_hi = tpos(mbs_ax, nm, (double)std::max(max_n, 1), sg);
  const int tm_hi_seg = sg;
  const long double tm_abs = std::max({1.0L, std::fabs(tm_lo), std::fabs(tm_hi)});
  bool used[2] = {false, false};
  for (const Layout& l : ctx->h_lay) {
    used[0] |= l.enc > 0;
    used[1] |= l.dec > 0;
  }
  long double A[2] = {0.0L, 0.0L}, ts_abs[2] = {1.0L, 1.0L};
  const size_t per = (size_t)nm * ns * 3;
  for (int k = 0; k < 2; ++k) {
    if (!used[k]) continue;
    // kind k reads the input length (encoder, or decoder of a decoder-only
    // model) or the target length (decoder of an encoder-decoder model)
    const int fld = (k == 1 && ctx->h_encdec) ? 1 : 0;
    const double lo = std::max(0.0, seq_lo[fld]), hi = std::max(0.0, seq_hi[fld]);
    const long double ts_lo = tpos(seq_ax, ns, lo, sg);
    const int ts_lo_seg = sg;
    const long double ts_hi = tpos(seq_ax, ns, hi, sg);
    const int ts_hi_seg = sg;
    ts_abs[k] = std::max({1.0L, std::fabs(ts_lo), std::fabs(ts_hi)});
    for (int f = f0; f <= f1; ++f) {
      auto c = [&](int mi, int si) -> long double {
        return ctx->h_cells[k * per + ((size_t)mi * ns + si) * 3 + f];
      };
      auto nonneg = [](long double v, long double scale) { return v >= 1e-12L * scale; };
      long double af = 0.0L;
      for (int mi = 0; mi < nm; ++mi)
        for (int si = 0; si < ns; ++si) {
          const long double v = c(mi, si);
          if (!std::isfinite((double)v)) return BAD;
          af = std::max(af, std::fabs(v));
          if (mi + 1 < nm && !(c(mi + 1, si) >= v)) return BAD;
          if (si + 1 < ns && !(c(mi, si + 1) >= v)) return BAD;
        }
      A[k] += af;
      // extrapolated sequence positions: d/dtm >= 0 at ts_lo (first segment)
      // and ts_hi (last segment), for every mbs segment
      for (int mi = 0; mi + 1 < nm && ns > 1; ++mi) {
        for (int e = 0; e < 2; ++e) {
          const long double ts = e ? ts_hi : ts_lo;
          if (ts >= 0.0L && ts <= 1.0L) continue;
          const int si = e ? ts_hi_seg : ts_lo_seg;
          const long double d0 = c(mi + 1, si) - c(mi, si), d1 = c(mi + 1, si + 1) - c(mi, si + 1);
          if (!nonneg((1.0L - ts) * d0 + ts * d1, (std::fabs(d0) + std::fabs(d1)) * (1.0L + std::fabs(ts))))
            return BAD;
        }
      }
      // extrapolated micro-batch sizes: d/dts >= 0 at tm_lo / tm_hi
      for (int si = 0; si + 1 < ns && nm > 1; ++si) {
        for (int e = 0; e < 2; ++e) {
          const long double tm = e ? tm_hi : tm_lo;
          if (tm >= 0.0L && tm <= 1.0L) continue;
          const int mi = e ? tm_hi_seg : tm_lo_seg;
          const long double e0 = c(mi, si + 1) - c(mi, si), e1 = c(mi + 1, si + 1) - c(mi + 1, si);
          if (!nonneg((1.0L - tm) * e0 + tm * e1, (std::fabs(e0) + std::fabs(e1)) * (1.0L + std::fabs(tm))))
            return BAD;
        }
      }
    }
  }
  long double worst = 0.0L;
  for (const Layout& l : ctx->h_lay) {
    long double w = 0.0L;
    if (l.enc > 0) w += (long double)l.enc * A[0] * ts_abs[0];
    if (l.dec > 0) w += (long double)l.dec * A[1] * ts_abs[1];
    worst = std::max(worst, w);
  }
  const long double u = std::ldexp(1.0L, -53);
  return k_ulp * u * (1.0L + tm_abs) * 2.0L * worst + 1e-300L;
}

double mem_exit_threshold(const pp_ctx* ctx, double cap, int max_n, double seq_lo[2],
                          double seq_hi[2], double* lo_thresh) {
  const double INF = INFINITY;
  *lo_thresh = -INF;
  if (!(cap < INF) || std::isnan(cap)) return INF;
  const long double E = surface_error_bound(ctx, max_n, seq_lo, seq_hi, 2, 2, 128.0L);
  if (!std::isfinite((double)E)) return INF;
  double th = (double)((long double)cap + 2.0L * E);
  th = std::nextafter(std::nextafter(th, INF), INF);
  if (!std::isfinite(th)) return INF;
  // cap - 2E, rounded down: a slice at or below it is certified feasible along
  // with every shorter slice of its row (rowexit_kernel)
  double tl = (double)((long double)cap - 2.0L * E);
  *lo_thresh = std::nextafter(std::nextafter(tl, -INF), -INF);
  return th;
}

// Margin 2E of the candidate passes' band truncation (dp.cu): a far chunk
// whose first column prices above t + 2E on every live row has, on a
// length-sorted segment, only slices above t from there on.  +inf: not
// certified (no truncation).
double time_trunc_margin(const pp_ctx* ctx, int max_n, const double seq_lo[2], const double seq_hi[2]) {
  // the slice time sums two blends per kind (t_f, t_b) through the layer
  // products: a doubled rounding budget over the act_mem certificate's
  const long double E = surface_error_bound(ctx, max_n, seq_lo, seq_hi, 0, 1, 256.0L);
  if (!std::isfinite((double)E)) return INFINITY;
  const double m = std::nextafter((double)(2.0L * E), (double)INFINITY);
  return std::isfinite(m) ? m : INFINITY;
}

// Steps 1-2 (+ tile offsets): sort, block bookkeeping, cost pass A.  Leaves
// the per-segment statistics in ctx->h_stats (synchronised) and the block
// table in host vector `blk_base`.
int cost_pass_a(pp_ctx* ctx, const PlanCall& c, const CostGrid& g, double interval,
                std::vector<int>& blk_base, int& max_n) {
  cudaStream_t st = ctx->stream;
  const int n_seg = c.n_seg;
  const int64_t total = c.h_seg_off[n_seg];
  const bool table = c.d_tabT != nullptr;
  blk_base.assign(n_seg + 1, 0);
  max_n = 0;
  for (int s = 0; s < n_seg; ++s) {
    const int n = (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]);
    max_n = std::max(max_n, n);
    blk_base[s + 1] = blk_base[s] + (n + kRB - 1) / kRB;
  }
  const int total_blocks = blk_base[n_seg];
  PP_CUDA(ctx->in_d.ensure(std::max<int64_t>(total, 1) * sizeof(double)));
  PP_CUDA(ctx->tgt_d.ensure(std::max<int64_t>(total, 1) * sizeof(double)));
  if (!table) {
    PP_CUDA(ctx->range.ensure(8 * sizeof(unsigned long long)));
    PP_CUDA(ctx->h_range.ensure(8 * sizeof(unsigned long long)));
    PP_CUDA(ctx->sort_keys.ensure(std::max<int64_t>(total, 1) * 6 * sizeof(unsigned long long)));
    PP_CUDA(ctx->sort_vals.ensure(std::max<int64_t>(total, 1) * 2 * sizeof(uint32_t)));
    if (total > 0)
      PP_TIMED(0, launch_segmented_sort(c.d_samples, c.d_seg_off, c.h_seg_off, n_seg, total, c.presorted,
                                        ctx->range.as<unsigned long long>(),
                                        ctx->h_range.as<unsigned long long>(),
                                        ctx->sort_keys.as<unsigned long long>(),
                                        ctx->sort_vals.as<uint32_t>(), c.d_ordered,
                                        ctx->in_d.as<double>(), ctx->tgt_d.as<double>(), c.d_order, st));
    PP_CUDA(ctx->mbp.ensure((size_t)(max_n + 1) * sizeof(AxisPos)));
    PP_CUDA(ctx->pin.ensure(std::max<int64_t>(total, 1) * sizeof(AxisPos)));
    PP_CUDA(ctx->ptg.ensure(std::max<int64_t>(total, 1) * sizeof(AxisPos)));
    PP_TIMED(1, launch_brackets(g, max_n, ctx->mbp.as<AxisPos>(), ctx->in_d.as<double>(),
                                ctx->tgt_d.as<double>(), total, ctx->pin.as<AxisPos>(),
                                ctx->ptg.as<AxisPos>(), st));
  }
  PP_CUDA(cudaEventRecord(ctx->ev[1], st));
  PP_CUDA(ctx->row_w.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
  PP_CUDA(ctx->row_fb.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
  PP_CUDA(ctx->blk_base.ensure((n_seg + 1) * sizeof(int)));
  PP_CUDA(ctx->blk_W.ensure(std::max(total_blocks, 1) * sizeof(int)));
  PP_CUDA(ctx->tile_off.ensure(std::max(total_blocks, 1) * sizeof(int64_t)));
  PP_CUDA(ctx->stats_d.ensure(n_seg * sizeof(SegStats)));
  PP_CUDA(ctx->h_stats.ensure(n_seg * sizeof(SegStats)));
  PP_CUDA(ctx->band_base.ensure(n_seg * sizeof(int64_t)));
  SegStats* hs = ctx->h_stats.as<SegStats>();
  for (int s = 0; s < n_seg; ++s) hs[s] = SegStats{~0ULL, 0ULL, 0ULL, INT_MAX, 0, 0, 0, 0, 0ULL, 0ULL, 0ULL};
  PP_CUDA(up(ctx, ctx->stats_d.p, hs, n_seg * sizeof(SegStats)));
  PP_CUDA(up(ctx, ctx->blk_base.p, blk_base.data(), (n_seg + 1) * sizeof(int)));
  const double cap = c.opts.per_mb_mem_cap;
  // Pass A (or its closed form when every slice is memory-feasible).
  const bool full_rows = !table && cap == INFINITY;
  double exit_thresh = INFINITY, lo_thresh = -INFINITY;
  int bisect = 0;
  if (!table && !full_rows && total > 0) {
    const unsigned long long* hr = ctx->h_range.as<unsigned long long>();
    double lo[2], hi[2];
    for (int q = 0; q < 2; ++q) {
      lo[q] = (double)(long long)(hr[q] ^ 0x8000000000000000ULL);
      hi[q] = (double)(long long)(hr[3 + q] ^ 0x8000000000000000ULL);
    }
    exit_thresh = mem_exit_threshold(ctx, cap, max_n, lo, hi, &lo_thresh);
    // bisection needs O(1) slice pricing: every segment sorted by input (our
    // sort) and every priced kind reading the input length
    bisect = !c.presorted && std::isfinite(exit_thresh) && (!g.is_encdec || !(g.used & 2));
  }
  ctx->exit_thresh = exit_thresh;
  unsigned int* small_bm = nullptr;
  if (interval > 0 && total > 0) {
    PP_CUDA(ctx->small_bm.ensure((size_t)n_seg * kSmallBmWords * sizeof(unsigned int)));
    PP_CUDA(cudaMemsetAsync(ctx->small_bm.p, 0, (size_t)n_seg * kSmallBmWords * sizeof(unsigned int), st));
    small_bm = ctx->small_bm.as<unsigned int>();
  }
  const double* tau_d = nullptr;
  if (interval > 0 && total > 0 && !table) {
    if (ctx->tau_interval != interval) {
      std::vector<double> tau;
      bin_thresholds(interval, tau);
      PP_CUDA(ctx->tau.ensure(tau.size() * sizeof(double)));
      PP_CUDA(up(ctx, ctx->tau.p, tau.data(), tau.size() * sizeof(double)));
      PP_CUDA(cudaStreamSynchronize(st));  // tau dies at scope exit
      trace_mark("passA tau sync");
      ctx->tau_interval = interval;
    }
    tau_d = ctx->tau.as<double>();
  }
  if (total > 0) {
    if (full_rows)
      PP_TIMED(1, launch_full_rows(c.d_seg_off, ctx->blk_base.as<int>(), n_seg, total_blocks,
                                   ctx->row_w.as<int>(), ctx->blk_W.as<int>(), st));
    else
      PP_TIMED(2, launch_cost_pass(0, g, c.d_tabT, c.d_tabM, ctx->in_d.as<double>(), ctx->tgt_d.as<double>(),
                                   ctx->pin.as<AxisPos>(), ctx->ptg.as<AxisPos>(), c.d_seg_off,
                                   ctx->blk_base.as<int>(), n_seg, total_blocks, max_n, ctx->mbp.as<AxisPos>(),
                                   cap, interval, ctx->row_w.as<int>(), ctx->row_fb.as<int>(), ctx->blk_W.as<int>(),
                                   ctx->stats_d.as<SegStats>(), nullptr, nullptr, nullptr, exit_thresh,
                                   nullptr, nullptr, lo_thresh, bisect, 0, 0, nullptr, nullptr, nullptr,
                                   nullptr, 0, st));
    PP_TIMED(1, launch_tile_offsets(ctx->blk_W.as<int>(), ctx->blk_base.as<int>(), n_seg,
                                    ctx->tile_off.as<int64_t>(), ctx->stats_d.as<SegStats>(), st));
  }
  PP_CUDA(down(ctx, hs, ctx->stats_d.p, n_seg * sizeof(SegStats)));
  PP_CUDA(cudaStreamSynchronize(st));
  trace_mark("passA stats sync");
  // Band allocation (tiles are NaN-filled: masked / unused entries).
  std::vector<int64_t> band_base(n_seg);
  int64_t band_total = 0;
  for (int s = 0; s < n_seg; ++s) {
    band_base[s] = band_total;
    band_total += hs[s].band;
  }
  ctx->band_total = band_total;
  // In-kernel DP pricing (dp.cu PRICE): pass B takes band_run_kernel (sorted
  // single-input mini-batches, quantised candidates) and no pass runs
  // cooperatively (dp_coop.cu streams the band): then the band is never
  // materialised — pass B only marks candidates, the DP prices its slices.
  const int64_t coop_n = ctx->tuning.coop_min_n > 0 ? ctx->tuning.coop_min_n : kCoopMinN;
  const bool sorted_gpt = !table && total > 0 && !ctx->tuning.compact_band && !c.presorted &&
                          band_run_applies(g, nullptr, ctx->tuning.no_slice_reuse ? 0 : 1, tau_d, 1) &&
                          !(n_seg <= kCoopMaxItems && max_n >= coop_n);
  // The call's shared slice table (gtab.cu) instead of a band per
  // mini-batch: lengths index its rows, so they must be bounded
  const int64_t max_len = (int64_t)(long long)(ctx->h_range.as<unsigned long long>()[3] ^ 0x8000000000000000ULL);
  bool use_gtab = sorted_gpt && !ctx->tuning.no_slice_table && !ctx->tuning.dp_pricing &&
                  max_len <= (int64_t)1 << 22 && max_n <= kGtabMaxN;
  const bool price_in_dp = sorted_gpt && !use_gtab && ctx->tuning.dp_pricing;
  ctx->gtab = false;
  if (use_gtab) {
    const int nK = (int)std::max<int64_t>(max_len, 0) + 1;
    PP_CUDA(ctx->gt_need.ensure((size_t)nK * sizeof(int)));
    PP_CUDA(ctx->gt_off.ensure((size_t)nK * sizeof(int64_t)));
    PP_CUDA(ctx->gt_total.ensure(sizeof(long long)));
    PP_CUDA(ctx->h_gt_total.ensure(sizeof(long long)));
    PP_CUDA(ctx->gt_base.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
    PP_CUDA(ctx->gt_rf.ensure((size_t)nK * sizeof(int)));
    PP_CUDA(ctx->gt_rlo.ensure((size_t)nK * sizeof(double)));
    PP_CUDA(cudaMemsetAsync(ctx->gt_need.p, 0, (size_t)nK * sizeof(int), st));
    PP_TIMED(3, launch_gtab_need(c.d_seg_off, ctx->blk_base.as<int>(), n_seg, total_blocks,
                                 (int)((max_n + kRB - 1) / kRB), ctx->blk_W.as<int>(),
                                 ctx->in_d.as<double>(), ctx->gt_need.as<int>(), st));
    PP_TIMED(3, launch_gtab_offsets(ctx->gt_need.as<int>(), nK, ctx->gt_off.as<int64_t>(),
                                    ctx->gt_total.as<long long>(), st));
    PP_CUDA(down(ctx, ctx->h_gt_total.p, ctx->gt_total.p, sizeof(long long)));
    PP_CUDA(cudaStreamSynchronize(st));
    trace_mark("gtab total sync");
    const int64_t entries = *ctx->h_gt_total.as<long long>();
    ctx->gtab_entries = entries;
    // row bases are int32 (dp.cu reads G[base - r]): a larger table takes the band
    if (entries + 64 >= (int64_t)INT_MAX) use_gtab = false;
  }
  if (use_gtab) {
    const int nK = (int)std::max<int64_t>(max_len, 0) + 1;
    const int64_t entries = ctx->gtab_entries;
    // G, then its copy shifted by one entry (starting 16 B aligned)
    const int64_t g1_at = (entries + 2) & ~(int64_t)1;
    PP_CUDA(ctx->gt_G.ensure((size_t)(g1_at + entries + 2) * sizeof(double)));
    PP_TIMED(3, launch_gtab_fill(g, cap, ctx->mbp.as<AxisPos>(), nK, ctx->gt_need.as<int>(), ctx->gt_off.as<int64_t>(),
                                 ctx->gt_G.as<double>(), ctx->gt_G.as<double>() + g1_at, st));
    PP_TIMED(3, launch_gtab_gbase(ctx->in_d.as<double>(), total, ctx->gt_off.as<int64_t>(),
                                  ctx->gt_base.as<int>(), st));
    PP_TIMED(3, launch_gtab_bins(c.d_seg_off, n_seg, ctx->in_d.as<double>(), ctx->gt_base.as<int>(),
                                 ctx->gt_need.as<int>(), ctx->gt_G.as<double>(), interval, tau_d, small_bm,
                                 ctx->stats_d.as<SegStats>(), nK, ctx->gt_off.as<int64_t>(),
                                 ctx->tuning.no_bin_intervals ? nullptr : ctx->gt_rf.as<int>(),
                                 ctx->gt_rlo.as<double>(), max_n, st));
    ctx->gtab = true;
    ctx->price = DpPrice{};
    ctx->price.gbase = ctx->gt_base.as<int>();
    ctx->price.g_odd = ctx->gt_G.as<double>() + g1_at;
  }
  if (!price_in_dp && !use_gtab) PP_CUDA(ctx->band.ensure(std::max<int64_t>(band_total, 1) * sizeof(double)));
  PP_CUDA(up(ctx, ctx->band_base.p, band_base.data(), n_seg * sizeof(int64_t)));
  // (no fill: pass B writes every tile entry, NaN where no slice is feasible)
  // Per-chunk minimum slice times for the candidate passes' truncation (dp.cu):
  // one slot per 1024 band entries plus one per block bounds every tile's chunks.
  double* cmin = nullptr;
  short* colbase = nullptr;
  int* chunk_nv = nullptr;
  if (!table && total > 0) {
    const int64_t ids = (band_total >> 10) + 2 * (int64_t)total_blocks + 64;  // chunk_id0 range
    PP_CUDA(ctx->cmin.ensure(ids * sizeof(double)));
    cmin = ctx->cmin.as<double>();
    if (ctx->tuning.compact_band) {
      PP_CUDA(ctx->colbase.ensure(ids * 32 * sizeof(short)));
      PP_CUDA(ctx->chunk_nv.ensure(ids * sizeof(int)));
      colbase = ctx->colbase.as<short>();
      chunk_nv = ctx->chunk_nv.as<int>();
    }
  }
  int wrote_cmin = 0;
  // Pass B: band + candidate statistics.
  if (total > 0 && !use_gtab)
    PP_TIMED(3, launch_cost_pass(1, g, c.d_tabT, c.d_tabM, ctx->in_d.as<double>(), ctx->tgt_d.as<double>(),
                                 ctx->pin.as<AxisPos>(), ctx->ptg.as<AxisPos>(), c.d_seg_off,
                                 ctx->blk_base.as<int>(), n_seg, total_blocks, max_n, ctx->mbp.as<AxisPos>(),
                                 cap, interval, ctx->row_w.as<int>(), ctx->row_fb.as<int>(), ctx->blk_W.as<int>(),
                                 ctx->stats_d.as<SegStats>(), ctx->tile_off.as<int64_t>(),
                                 ctx->band_base.as<int64_t>(), ctx->band.as<double>(), INFINITY, small_bm,
                                 tau_d, -INFINITY, 0, c.presorted ? 0 : 1,
                                 ctx->tuning.no_slice_reuse ? 0 : 1, cmin, colbase, chunk_nv, &wrote_cmin,
                                 price_in_dp ? 1 : 0, st));
  ctx->trunc_margin = INFINITY;
  ctx->compact = (wrote_cmin & 2) != 0;
  ctx->priced = (wrote_cmin & 4) != 0;
  if (price_in_dp && !ctx->priced) return fail(ctx, PP_ERR_CUDA, "internal: pass B did not take the in-DP pricing path");
  if (ctx->priced) {
    DpPrice& p = ctx->price;
    const int per = g.nm * g.ns;
    p.P.tt_e = g.tt;
    p.P.tt_d = g.tt + per;
    p.P.am_e = g.am;
    p.P.am_d = g.am + per;
    p.P.ns = g.ns;
    p.P.le = g.le;
    p.P.ld = g.ld;
    p.P.cap = cap;
    p.P.need_mem = !(cap == INFINITY);
    p.cells = per;
    p.mbp = ctx->mbp.as<AxisPos>();
    p.pin = ctx->pin.as<AxisPos>();
    p.in_d = ctx->in_d.as<double>();
    p.max_n = max_n;
    // bracket(seq axis, 0.0) (cost_model.cpp:46-53) on the host: the same
    // IEEE operations as the device's bracket() (band_run_kernel's p0)
    const double* sx = ctx->h_ax.data() + g.nm;
    int sg = 0;
    double tz = 0.0;
    if (g.ns > 1) {
      while (sg + 2 < g.ns && 0.0 >= sx[sg + 1]) ++sg;
      volatile double num = 0.0 - sx[sg], den = sx[sg + 1] - sx[sg];
      tz = num / den;
    }
    p.p0.t = tz;
    p.p0.seg = sg;
    p.p0.pad = 0;
    ctx->price_lay = g.lay_class;
  }
  if (((wrote_cmin & 1) || use_gtab) && !ctx->tuning.no_band_trunc) {
    // (the slice-time certificate; the table path records no chunk minima,
    // so only the bound pass / first wave use it, not the truncation)
    const unsigned long long* hr = ctx->h_range.as<unsigned long long>();
    double lo[2], hi[2];
    for (int q = 0; q < 2; ++q) {
      lo[q] = (double)(long long)(hr[q] ^ 0x8000000000000000ULL);
      hi[q] = (double)(long long)(hr[3 + q] ^ 0x8000000000000000ULL);
    }
    ctx->trunc_margin = time_trunc_margin(ctx, max_n, lo, hi);
  }
  PP_CUDA(down(ctx, hs, ctx->stats_d.p, n_seg * sizeof(SegStats)));
  PP_CUDA(cudaStreamSynchronize(st));
  trace_mark("passB stats sync");
  return PP_OK;
}

// DP state placement for one pass over a segment of n samples whose tiles
// are at most wmax columns wide: a ring of R >= wmax + 64 entries (dp.cu)
// when that is smaller than the full n + 1.
// Shared memory per DP CTA: deep chunk rings when the launch has at most one
// CTA per SM, two CTAs per SM otherwise.
size_t dp_budget(int n_items) { return n_items <= 148 ? 220 * 1024 : 110 * 1024; }

void state_layout(int mode, int n, int wmax, unsigned& mask, int& entries, size_t& smem) {
  // R slots, a multiple of 32, indexed (j + shift) mod R (dp.cu, shift < 32):
  // a ring of R >= W_max + 64 (the live states), or the whole row range
  const int R_ring = (wmax + 64 + 31) / 32 * 32;
  const int R_full = (n + 32 + 31) / 32 * 32;
  entries = std::min(R_ring, R_full);
  mask = entries < R_full ? (unsigned)(entries - 1) : ~0u;  // (informational)
  smem = dp_smem_fixed() + dp_state_bytes(mode, entries);
}

// A DP launch keeps every item's state in shared memory, or (when any
// item's state does not fit) every item's state in an L2-resident global
// ring: the kernel is specialised on the placement.
void place_states(std::vector<WorkItem>& items, int mode, size_t& smem_state, int& state_global,
                  int64_t& goff) {
  smem_state = 0;
  state_global = 0;
  goff = 0;
  for (const WorkItem& w : items)
    if (dp_smem_fixed() + dp_state_bytes(mode, w.state_entries) > kDpSmemLimit) state_global = 1;
  for (WorkItem& w : items) {
    if (state_global) {
      w.state_off = goff;  // (16-byte aligned: the DP's vector state loads)
      goff += ((int64_t)((dp_state_bytes(mode, w.state_entries) + 7) / 8) + 1) & ~(int64_t)1;
    } else {
      w.state_off = -1;
      smem_state = std::max(smem_state, dp_state_bytes(mode, w.state_entries));
    }
  }
}


bool use_coop(const pp_ctx* ctx, const std::vector<WorkItem>& items, const int64_t* h_seg_off) {
  if (items.empty() || (int)items.size() > kCoopMaxItems) return false;
  if (ctx->compact || ctx->priced || ctx->gtab) return false;  // the cooperative pass reads the dense band
  const int64_t min_n = ctx->tuning.coop_min_n > 0 ? ctx->tuning.coop_min_n : kCoopMinN;
  for (const WorkItem& w : items)
    if (h_seg_off[w.seg + 1] - h_seg_off[w.seg] < min_n) return false;
  return true;
}

int run_coop(pp_ctx* ctx, int mode, int sanitize, const std::vector<WorkItem>& items, const PlanCall& c,
             ItemResult* res, int res_by_seg, cudaStream_t st) {
  const int grid = dp_coop_grid(ctx->device);
  int64_t nmax = 0;
  for (const WorkItem& w : items) nmax = std::max<int64_t>(nmax, c.h_seg_off[w.seg + 1] - c.h_seg_off[w.seg]);
  PP_CUDA(ctx->coop_state.ensure((size_t)2 * (nmax + 1) * sizeof(double)));
  PP_CUDA(ctx->coop_parts.ensure(dp_coop_parts_bytes(grid)));
  for (size_t k = 0; k < items.size(); ++k) {
    WorkItem w = items[k];
    w.state_off = 0;  // passes run one after another on the stream: one state array
    PP_CUDA(launch_dp_coop(mode, sanitize, w, grid, c.d_seg_off, ctx->blk_base.as<int>(), ctx->blk_W.as<int>(),
                           ctx->tile_off.as<int64_t>(), ctx->band_base.as<int64_t>(), ctx->band.as<double>(),
                           ctx->cand.as<double>(), ctx->cand_off.as<int64_t>(), res,
                           res_by_seg ? w.seg : (int)k, ctx->next_buf.as<int>(), ctx->coop_state.as<double>(),
                           ctx->coop_parts.p, st));
  }
  return PP_OK;
}

// What the DP passes and the assembly read: the band, or (gtab) the call's
// shared slice table with its per-sample row bases, or (priced) nothing.
const double* dp_band(const pp_ctx* ctx) { return ctx->gtab ? ctx->gt_G.as<double>() : ctx->band.as<double>(); }
const DpPrice* dp_price(const pp_ctx* ctx) { return (ctx->gtab || ctx->priced) ? &ctx->price : nullptr; }
int dp_lay(const pp_ctx* ctx) { return ctx->gtab ? kGtab : ctx->price_lay; }
// The DP's per-sample slice-table row bases (slice-table path), or null (band).
const int* dp_gbase(const pp_ctx* ctx) { return ctx->gtab ? ctx->gt_base.as<int>() : nullptr; }

// The planning pipeline (steps 1-7 above).
int run_plan(pp_ctx* ctx, const PlanCall& c) {
  NvtxRange nvtx("pp run_plan");
  ctx->arena.off = 0;  // (the previous call ended with its stream synchronised)
  cudaStream_t st = ctx->stream;
  const int n_seg = c.n_seg;
  if (c.h_seg_off[0] != 0) return fail(ctx, PP_ERR_INVALID, "seg_offsets[0] must be 0");
  for (int s = 0; s < n_seg; ++s)
    if (c.h_seg_off[s + 1] < c.h_seg_off[s])
      return fail(ctx, PP_ERR_INVALID, "seg_offsets must be non-decreasing");
  const int64_t total = c.h_seg_off[n_seg];
  if (total >= INT_MAX) return fail(ctx, PP_ERR_INVALID, "too many samples in one call");
  ctx->kused = 0;
  ctx->kcat.clear();
  pp_stats S{};

  CostGrid g{};
  if (!c.d_tabT) {
    int rc = upload_grid(ctx, c.grid, c.model, &g);
    if (rc) return rc;
  }
  PP_CUDA(cudaEventRecord(ctx->ev[0], st));
  // NaN -> 0: exact candidate set, as the reference's `interval > 0` test (microbatch.cpp:263)
  const double I = c.opts.t_max_interval > 0 ? c.opts.t_max_interval : 0.0;
  const bool table = c.d_tabT != nullptr;
  std::vector<int> blk_base;
  int max_n = 0;
  {
    int rc = cost_pass_a(ctx, c, g, I, blk_base, max_n);
    if (rc) return rc;
  }
  const int total_blocks = blk_base[n_seg];

  // ---- 3. sizing: band, candidate modes
  const SegStats* hs = ctx->h_stats.as<SegStats>();
  const bool single = c.opts.stage_count == 1;  // candidates = {+inf} (microbatch.cpp:255-257)
  std::vector<int64_t> bm_off(n_seg + 1, 0), raw_off(n_seg + 1, 0), cand_off(n_seg + 1, 0);
  std::vector<int> mode(n_seg, 2), active(n_seg, 0);
  for (int s = 0; s < n_seg; ++s) {
    const int n = (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]);
    active[s] = (n > 0 && hs[s].err_row == INT_MAX) ? 1 : 0;
    int64_t ncap = 1;
    bm_off[s + 1] = bm_off[s];
    raw_off[s + 1] = raw_off[s];
    if (!single && active[s]) {
      bool bitmap_ok = false;
      bool small_ok = false;
      if (I > 0) {
        // every finite bin in [0, 32 * kSmallBmWords): pass B marked them all
        small_ok = hs[s].kmin == ~0ULL ||
                   (dkey_inv_host(hs[s].kmin) >= 0.0 && dkey_inv_host(hs[s].kmax) < 32.0 * kSmallBmWords);
      }
      if (small_ok) {
        mode[s] = 3;
        ncap = 32 * kSmallBmWords + 2;
      } else if (I > 0 && hs[s].kmin != ~0ULL) {
        const double kmn = dkey_inv_host(hs[s].kmin), kmx = dkey_inv_host(hs[s].kmax);
        if (std::fabs(kmn) < 4.0e15 && std::fabs(kmx) < 4.0e15 && kmx - kmn < (double)(1 << 26)) {
          const int64_t range = (int64_t)(kmx - kmn) + 1;
          bm_off[s + 1] = bm_off[s] + (range + 31) / 32;
          ncap = range + 2;
          bitmap_ok = true;
        }
      }
      if (small_ok) {
      } else if (bitmap_ok) {
        mode[s] = 0;
      } else {
        mode[s] = 1;
        raw_off[s + 1] = raw_off[s] + (int64_t)hs[s].nraw;
        ncap = (int64_t)hs[s].nraw + 1;
      }
    }
    cand_off[s + 1] = cand_off[s] + ncap;
  }
  for (int s = 0; s < n_seg; ++s) {
    const int64_t n = c.h_seg_off[s + 1] - c.h_seg_off[s];
    (void)n;
    S.slices_costed += (int64_t)hs[s].priced + (int64_t)hs[s].priced_b;
  }
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
  PP_CUDA(up(ctx, ctx->bitmap_off.p, bm_off.data(), (n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(up(ctx, ctx->seg_mode.p, mode.data(), n_seg * sizeof(int)));
  PP_CUDA(up(ctx, ctx->active.p, active.data(), n_seg * sizeof(int)));
  PP_CUDA(up(ctx, ctx->raw_off.p, raw_off.data(), (n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(up(ctx, ctx->cand_off.p, cand_off.data(), (n_seg + 1) * sizeof(int64_t)));
  if (bm_off[n_seg] > 0) PP_CUDA(cudaMemsetAsync(ctx->bitmap.p, 0, bm_off[n_seg] * sizeof(unsigned int), st));
  PP_CUDA(cudaMemsetAsync(ctx->raw_cnt.p, 0, n_seg * sizeof(unsigned long long), st));
  PP_CUDA(cudaMemsetAsync(ctx->raw_in_tmp.p, 0, n_seg * sizeof(int), st));
  PP_CUDA(cudaMemsetAsync(ctx->cand_n.p, 0, n_seg * sizeof(int), st));

  // pass C: candidate values from the band (segments pass B did not cover)
  bool need_pass_c = false;
  for (int s = 0; s < n_seg; ++s) need_pass_c |= (mode[s] == 0 || mode[s] == 1);
  if ((ctx->priced || ctx->gtab) && total > 0 && !single && need_pass_c) {
    // candidate bins past pass B's bitmap: pass C reads them from the band,
    // so this call materialises it after all (pass B again, storing; its
    // candidate marks are idempotent) and the DP streams it
    PP_CUDA(ctx->band.ensure(std::max<int64_t>(ctx->band_total, 1) * sizeof(double)));
    int wrote = 0;
    PP_TIMED(3, launch_cost_pass(1, g, nullptr, nullptr, ctx->in_d.as<double>(), ctx->tgt_d.as<double>(),
                                 ctx->pin.as<AxisPos>(), ctx->ptg.as<AxisPos>(), c.d_seg_off,
                                 ctx->blk_base.as<int>(), n_seg, total_blocks, max_n, ctx->mbp.as<AxisPos>(),
                                 c.opts.per_mb_mem_cap, I, ctx->row_w.as<int>(), ctx->row_fb.as<int>(),
                                 ctx->blk_W.as<int>(), ctx->stats_d.as<SegStats>(), ctx->tile_off.as<int64_t>(),
                                 ctx->band_base.as<int64_t>(), ctx->band.as<double>(), INFINITY,
                                 ctx->small_bm.as<unsigned int>(), ctx->tau.as<double>(), -INFINITY, 0, 1,
                                 ctx->tuning.no_slice_reuse ? 0 : 1, ctx->cmin.as<double>(), nullptr, nullptr,
                                 &wrote, 0, st));
    ctx->priced = false;
    ctx->gtab = false;
  }
  if (total > 0 && !single && need_pass_c)
    PP_TIMED(6, launch_band_cand(c.d_seg_off, ctx->blk_base.as<int>(), n_seg, total_blocks,
                                 ctx->blk_W.as<int>(), ctx->tile_off.as<int64_t>(),
                                 ctx->band_base.as<int64_t>(), ctx->band.as<double>(), I,
                                 ctx->stats_d.as<SegStats>(), ctx->bitmap.as<unsigned int>(),
                                 ctx->bitmap_off.as<int64_t>(), ctx->seg_mode.as<int>(),
                                 ctx->raw.as<unsigned long long>(), ctx->raw_off.as<int64_t>(),
                                 ctx->raw_cnt.as<unsigned long long>(),
                                 ctx->compact ? ctx->colbase.as<short>() : nullptr, ctx->row_w.as<int>(), st));
  // ---- 4. candidate lists
  if (single) {
    std::vector<double> infs(cand_off[n_seg], INFINITY);
    std::vector<int> ones(n_seg, 1);
    PP_CUDA(up(ctx, ctx->cand.p, infs.data(), infs.size() * sizeof(double)));
    PP_CUDA(up(ctx, ctx->cand_n.p, ones.data(), n_seg * sizeof(int)));
    PP_CUDA(cudaStreamSynchronize(st));  // host vectors die here
    trace_mark("dp setup sync");
  } else {
    PP_TIMED(6, launch_cand_bitmap(ctx->bitmap.as<unsigned int>(), ctx->bitmap_off.as<int64_t>(),
                                   ctx->stats_d.as<SegStats>(), ctx->seg_mode.as<int>(), n_seg,
                                   ctx->small_bm.as<unsigned int>(), I, ctx->cand_off.as<int64_t>(),
                                   ctx->cand.as<double>(), ctx->cand_n.as<int>(), st));
    if (raw_off[n_seg] > 0) {
      PP_TIMED(6, launch_segmented_sort_u64(ctx->raw.as<unsigned long long>(),
                                            ctx->raw_tmp.as<unsigned long long>(),
                                            ctx->raw_off.as<int64_t>(),
                                            ctx->raw_cnt.as<unsigned long long>(), ctx->seg_mode.as<int>(),
                                            1, ctx->raw_in_tmp.as<int>(), n_seg, st));
      PP_TIMED(6, launch_cand_unique(ctx->raw.as<unsigned long long>(),
                                     ctx->raw_tmp.as<unsigned long long>(), ctx->raw_in_tmp.as<int>(),
                                     ctx->raw_off.as<int64_t>(), ctx->raw_cnt.as<unsigned long long>(),
                                     ctx->seg_mode.as<int>(), n_seg, ctx->cand_off.as<int64_t>(),
                                     ctx->cand.as<double>(), ctx->cand_n.as<int>(), st));
    }
  }
  PP_CUDA(cudaEventRecord(ctx->ev[2], st));

  // ---- 5. bound + minimax pass (one CTA per active segment)
  PP_CUDA(ctx->segdp.ensure(n_seg * sizeof(SegDP)));
  PP_CUDA(ctx->h_segdp.ensure(n_seg * sizeof(SegDP)));
  PP_CUDA(ctx->best_next.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
  PP_CUDA(ctx->bound_res.ensure(n_seg * sizeof(ItemResult)));
  const int64_t* d_cand_off = ctx->cand_off.as<int64_t>();
  const double* d_cand = ctx->cand.as<double>();
  int64_t bound_transitions = 0;
  // with a certified slice-time surface (pass B's truncation certificate), t*
  // is bounded below by the singleton slices: the bound pass then skips the
  // minimax (MODE 2) and the first wave starts at that bound
  const double* t_lo = nullptr;  // (non-null: the margin 2E; the bound is pass B's singleton maximum)
  bool fused = false;
  if (!single) {
    std::vector<WorkItem> bi;
    int64_t goff = 0;
    for (int s = 0; s < n_seg; ++s) {
      if (!active[s]) continue;
      const int n = (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]);
      WorkItem w{};
      w.seg = s;
      w.cand = -1;
      w.next_off = 0;
      size_t need;
      state_layout(1, n, hs[s].wmax, w.state_mask, w.state_entries, need);
      bound_transitions += hs[s].band;
      bi.push_back(w);
    }
    size_t smem_state = 0;
    int state_global = 0;
    place_states(bi, 1, smem_state, state_global, goff);
    if (!bi.empty()) {
      PP_CUDA(ctx->bound_items.ensure(bi.size() * sizeof(WorkItem)));
      PP_CUDA(ctx->gstate.ensure(std::max<int64_t>(goff, 1) * sizeof(double)));
      PP_CUDA(ctx->next_buf.ensure(std::max<int64_t>(total, 1) * sizeof(int)));
      PP_CUDA(up(ctx, ctx->bound_items.p, bi.data(), bi.size() * sizeof(WorkItem)));
      const bool coop = use_coop(ctx, bi, c.h_seg_off);
      // (pass B recorded the largest singleton time per segment, SegStats::tsingle)
      const int bmode = std::isfinite(ctx->trunc_margin) && !table ? 2 : 1;
      if (bmode == 2 && !coop) t_lo = &ctx->trunc_margin;
      // the first wave's candidate is then known before the bound: one fused
      // pass runs both (MODE 3, in the wave loop below)
      fused = t_lo != nullptr && std::max(1, ctx->tuning.first_wave) == 1;
      if (coop) {
        PP_CUDA(timed_begin(ctx, 4));
        int rc = run_coop(ctx, 1, table ? 1 : 0, bi, c, ctx->bound_res.as<ItemResult>(), 1, st);
        if (rc) return rc;
        PP_CUDA(timed_end(ctx));
      } else if (!fused) {
        PP_TIMED(4, launch_dp_pass(bmode, ctx->bound_items.as<WorkItem>(), (int)bi.size(), smem_state,
                                   state_global, table ? 1 : 0, dp_budget((int)bi.size()), c.d_seg_off,
                                   ctx->blk_base.as<int>(), ctx->blk_W.as<int>(), ctx->tile_off.as<int64_t>(),
                                   ctx->band_base.as<int64_t>(), dp_band(ctx), d_cand, d_cand_off,
                                   ctx->bound_res.as<ItemResult>(), ctx->next_buf.as<int>(),
                                   ctx->gstate.as<double>(), 1, nullptr, 0.0, nullptr, nullptr,
                                   dp_gbase(ctx), st));
      }
      PP_CUDA(cudaStreamSynchronize(st));  // bi dies here
      trace_mark("wave sync");
    }
  }
  PP_TIMED(7, launch_seg_init(ctx->bound_res.as<ItemResult>(), single ? 0 : fused ? 2 : 1, c.opts.replica_count,
                              d_cand_off, ctx->cand_n.as<int>(), d_cand, ctx->active.as<int>(),
                              t_lo ? ctx->stats_d.as<SegStats>() : nullptr, t_lo ? *t_lo : 0.0,
                              ctx->segdp.as<SegDP>(), n_seg, st));

  // ---- 6. candidate waves
  int wave = std::max(1, ctx->tuning.first_wave);
  const int max_wave = std::max(wave, ctx->tuning.max_wave > 0 ? ctx->tuning.max_wave : 16);
  int64_t transitions = bound_transitions, evaluated = 0, waves = 0;
  // candidate passes on certified tiles stream only the chunks that can hold
  // a slice <= t: their transitions are counted on the device
  const bool trunc = std::isfinite(ctx->trunc_margin);
  PP_CUDA(ctx->dp_cols.ensure(sizeof(unsigned long long)));
  PP_CUDA(cudaMemsetAsync(ctx->dp_cols.p, 0, sizeof(unsigned long long), st));
  bool counted = false;
  std::vector<WorkItem> items;
  std::vector<int> item_start(n_seg), item_cnt(n_seg);
  for (;;) {
    PP_CUDA(down(ctx, ctx->h_segdp.p, ctx->segdp.p, n_seg * sizeof(SegDP)));
    PP_CUDA(cudaStreamSynchronize(st));
    trace_mark("wave end sync");
    const SegDP* hd = ctx->h_segdp.as<SegDP>();
    items.clear();
    int64_t noff = 0, goff = 0;
    for (int s = 0; s < n_seg; ++s) {
      item_start[s] = (int)items.size();
      item_cnt[s] = 0;
      if (hd[s].done) continue;
      const int n = (int)(c.h_seg_off[s + 1] - c.h_seg_off[s]);
      const int k = std::min(fused ? 1 : wave, hd[s].n_cand - hd[s].next_cand);
      WorkItem proto{};
      size_t need;
      state_layout(fused ? 3 : 0, n, hs[s].wmax, proto.state_mask, proto.state_entries, need);
      for (int q = 0; q < k; ++q) {
        WorkItem w = proto;
        w.seg = s;
        w.cand = hd[s].next_cand + q;
        w.next_off = noff;
        noff += n;
        items.push_back(w);
      }
      item_cnt[s] = k;
    }
    if (items.empty()) break;
    size_t smem_state = 0;
    int state_global = 0;
    place_states(items, fused ? 3 : 0, smem_state, state_global, goff);
    ++waves;
    evaluated += (int64_t)items.size();
    const int ni = (int)items.size();
    PP_CUDA(ctx->items.ensure(ni * sizeof(WorkItem)));
    PP_CUDA(ctx->results.ensure(ni * sizeof(ItemResult)));
    PP_CUDA(ctx->next_buf.ensure(std::max<int64_t>(noff, 1) * sizeof(int)));
    PP_CUDA(ctx->gstate.ensure(std::max<int64_t>(goff, 1) * sizeof(double)));
    PP_CUDA(ctx->seg_item_start.ensure(n_seg * sizeof(int)));
    PP_CUDA(ctx->seg_item_cnt.ensure(n_seg * sizeof(int)));
    PP_CUDA(up(ctx, ctx->items.p, items.data(), ni * sizeof(WorkItem)));
    PP_CUDA(up(ctx, ctx->seg_item_start.p, item_start.data(), n_seg * sizeof(int)));
    PP_CUDA(up(ctx, ctx->seg_item_cnt.p, item_cnt.data(), n_seg * sizeof(int)));
    if (fused) {
      // the bound pass and the first wave in one band stream (MODE 3): the
      // candidate results per item, the bounds per segment
      PP_TIMED(4, launch_dp_pass(3, ctx->items.as<WorkItem>(), ni, smem_state, state_global, 0, dp_budget(ni),
                                 c.d_seg_off, ctx->blk_base.as<int>(), ctx->blk_W.as<int>(),
                                 ctx->tile_off.as<int64_t>(), ctx->band_base.as<int64_t>(),
                                 dp_band(ctx), d_cand, d_cand_off, ctx->results.as<ItemResult>(),
                                 ctx->next_buf.as<int>(), ctx->gstate.as<double>(), 0, nullptr, 0.0, nullptr,
                                 ctx->bound_res.as<ItemResult>(), dp_gbase(ctx), st));
      PP_TIMED(7, launch_seg_set_bound(ctx->bound_res.as<ItemResult>(), c.opts.replica_count,
                                       ctx->segdp.as<SegDP>(), n_seg, st));
    } else if (use_coop(ctx, items, c.h_seg_off)) {
      PP_CUDA(timed_begin(ctx, 5));
      int rc = run_coop(ctx, 0, table ? 1 : 0, items, c, ctx->results.as<ItemResult>(), 0, st);
      if (rc) return rc;
      PP_CUDA(timed_end(ctx));
      for (const WorkItem& w : items) transitions += hs[w.seg].band;
    } else {
      PP_TIMED(5, launch_dp_pass(0, ctx->items.as<WorkItem>(), ni, smem_state, state_global, table ? 1 : 0,
                                 dp_budget(ni), c.d_seg_off, ctx->blk_base.as<int>(),
                                 ctx->blk_W.as<int>(), ctx->tile_off.as<int64_t>(), ctx->band_base.as<int64_t>(),
                                 dp_band(ctx), d_cand, d_cand_off, ctx->results.as<ItemResult>(),
                                 ctx->next_buf.as<int>(), ctx->gstate.as<double>(), 0,
                                 (trunc && !ctx->gtab) ? ctx->cmin.as<double>() : nullptr, ctx->trunc_margin,
                                 ctx->dp_cols.as<unsigned long long>(), nullptr, dp_gbase(ctx), st));
      counted = true;
    }
    PP_TIMED(7, launch_select(ctx->items.as<WorkItem>(), ctx->results.as<ItemResult>(),
                              ctx->seg_item_start.as<int>(), ctx->seg_item_cnt.as<int>(),
                              ctx->next_buf.as<int>(), ctx->best_next.as<int>(), c.d_seg_off, d_cand,
                              d_cand_off, c.opts.stage_count, c.opts.replica_count,
                              ctx->segdp.as<SegDP>(), n_seg, st));
    if (fused) fused = false;  // (wave 1 done; the doubling goes on from it)
    wave = std::min(wave * 2, max_wave);
  }
  PP_CUDA(cudaEventRecord(ctx->ev[3], st));

  // ---- 7. assembly
  PP_TIMED(7, launch_finalize(ctx->segdp.as<SegDP>(), ctx->best_next.as<int>(), c.d_seg_off,
                              ctx->blk_base.as<int>(), ctx->tile_off.as<int64_t>(),
                              ctx->band_base.as<int64_t>(), dp_band(ctx),
                              ctx->stats_d.as<SegStats>(), ctx->compact ? ctx->colbase.as<short>() : nullptr,
                              c.d_ordered, c.opts.stage_count,
                              c.opts.replica_count, std::max(max_n, 1), n_seg, c.d_splits, c.d_times,
                              c.d_count, c.d_tmax, c.d_obj, c.d_status, c.d_err,
                              dp_price(ctx), dp_lay(ctx), st));
  unsigned long long dp_cols = 0;
  if (counted) {
    PP_CUDA(ctx->h_word.ensure(sizeof(dp_cols)));
    PP_CUDA(down(ctx, ctx->h_word.p, ctx->dp_cols.p, sizeof(dp_cols)));
  }
  PP_CUDA(cudaStreamSynchronize(st));
  trace_mark("run_plan end sync");
  if (counted) dp_cols = *ctx->h_word.as<unsigned long long>();
  PP_CUDA(cudaGetLastError());
  transitions += (int64_t)dp_cols * kRB;

  // stats
  const SegDP* hd = ctx->h_segdp.as<SegDP>();
  int64_t ref_tr = 0, gen = 0, ref_ev = 0;
  for (int s = 0; s < n_seg; ++s) {
    const int64_t n = c.h_seg_off[s + 1] - c.h_seg_off[s];
    if (!active[s]) continue;
    gen += hd[s].n_cand;
    ref_ev += hd[s].ref_evals;
    ref_tr += n * (n + 1) / 2 * ((int64_t)hd[s].ref_evals + (single ? 0 : 1));
  }
  S.candidates_generated = gen;
  S.candidates_ref_evaluated = ref_ev;
  S.candidates_evaluated = evaluated;
  S.transitions_executed = transitions;
  S.transitions_reference = ref_tr;
  S.waves = waves;
  S.ms_sort = elapsed(ctx->ev[0], ctx->ev[1]);
  S.ms_cost = elapsed(ctx->ev[1], ctx->ev[2]);
  S.ms_dp = elapsed(ctx->ev[2], ctx->ev[3]);
  S.ms_total = elapsed(ctx->ev[0], ctx->ev[3]);
  for (size_t k = 0; k < ctx->kcat.size(); ++k) {
    S.ms_kernel[ctx->kcat[k]] += elapsed(ctx->kev[2 * k], ctx->kev[2 * k + 1]);
    S.launches[ctx->kcat[k]] += 1;
  }
  S.dp_band_bytes = transitions * (int64_t)sizeof(double);
  S.band_bytes = (ctx->priced || ctx->gtab) ? 0 : ctx->band_total * (int64_t)sizeof(double);
  S.exit_thresh = ctx->exit_thresh;
  for (int s = 0; s < n_seg; ++s) {
    S.slices_pass_a += (int64_t)hs[s].priced;
    S.slices_pass_b += (int64_t)hs[s].priced_b;
  }
  S.bound_transitions = bound_transitions;
  ctx->stats = S;
  return PP_OK;
}

int check_ctx(pp_ctx* ctx) {
  if (!ctx) return PP_ERR_INVALID;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return fail(ctx, PP_ERR_CUDA, cudaGetErrorString(e));
  return PP_OK;
}

// Stage host samples + offsets into the ctx buffers.
int stage_inputs(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets, int n_seg) {
  const int64_t total = seg_offsets[n_seg];
  cudaStream_t st = ctx->stream;
  PP_CUDA(ctx->samples.ensure(std::max<int64_t>(total, 1) * sizeof(pp_sample)));
  PP_CUDA(ctx->seg_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->ordered.ensure(std::max<int64_t>(total, 1) * sizeof(pp_sample)));
  if (total > 0)
    PP_CUDA(cudaMemcpyAsync(ctx->samples.p, samples, total * sizeof(pp_sample), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->seg_off.p, seg_offsets, (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  return PP_OK;
}

// pp_tuning::streams > 1: contiguous sub-batches of segments, each planned by
// its own sub-context (stream + scratch) from its own host thread, all on the
// caller's device.  Sub-streams start after the caller stream's pending work
// (the inputs) and the caller stream waits for all of them, so the call keeps
// its single-stream semantics.  Results are written in place (outputs are
// indexed by sample / segment, so each part writes a disjoint slice).
int plan_split(pp_ctx* ctx, const PlanCall& c, int parts) {
  const int n_seg = c.n_seg;
  parts = std::min(parts, n_seg);
  while ((int)ctx->subs.size() < parts) {
    pp_ctx* sub = nullptr;
    const int rc = pp_ctx_create(ctx->device, &sub);
    if (rc != PP_OK) return fail(ctx, rc, "cannot create a sub-context");
    ctx->subs.push_back(sub);
  }
  if (!ctx->ev_in) PP_CUDA(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
  PP_CUDA(cudaEventRecord(ctx->ev_in, ctx->stream));
  // split by sample count
  const int64_t total = c.h_seg_off[n_seg];
  std::vector<int> cut(parts + 1, 0);
  cut[parts] = n_seg;
  for (int p = 1; p < parts; ++p) {
    const int64_t target = total * p / parts;
    int s = cut[p - 1] + 1;
    while (s < n_seg - (parts - p) && c.h_seg_off[s] < target) ++s;
    cut[p] = s;
  }
  std::vector<int> rcs(parts, PP_OK);
  std::vector<std::thread> th;
  for (int p = 0; p < parts; ++p) {
    th.emplace_back([&, p]() {
      pp_ctx* sub = ctx->subs[p];
      cudaSetDevice(sub->device);
      sub->tuning = ctx->tuning;
      sub->tuning.streams = 1;
      const int s0 = cut[p], s1 = cut[p + 1];
      const int64_t base = c.h_seg_off[s0];
      std::vector<int64_t> off(s1 - s0 + 1);
      for (int s = s0; s <= s1; ++s) off[s - s0] = c.h_seg_off[s] - base;
      int rc = PP_OK;
      auto cu = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == PP_OK) {
          sub->err = cudaGetErrorString(e);
          rc = PP_ERR_CUDA;
        }
      };
      cu(cudaStreamWaitEvent(sub->stream, ctx->ev_in, 0));
      cu(sub->seg_off.ensure(off.size() * sizeof(int64_t)));
      cu(cudaMemcpyAsync(sub->seg_off.p, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                         sub->stream));
      if (rc == PP_OK) {
        PlanCall cc = c;
        cc.d_samples = c.d_samples ? c.d_samples + base : nullptr;
        cc.d_seg_off = sub->seg_off.as<int64_t>();
        cc.h_seg_off = off.data();
        cc.n_seg = s1 - s0;
        cc.d_ordered = c.d_ordered + base;
        cc.d_order = c.d_order ? c.d_order + base : nullptr;
        cc.d_splits = c.d_splits ? c.d_splits + base : nullptr;
        cc.d_times = c.d_times ? c.d_times + base : nullptr;
        cc.d_count = c.d_count ? c.d_count + s0 : nullptr;
        cc.d_tmax = c.d_tmax ? c.d_tmax + s0 : nullptr;
        cc.d_obj = c.d_obj ? c.d_obj + s0 : nullptr;
        cc.d_status = c.d_status ? c.d_status + s0 : nullptr;
        cc.d_err = c.d_err ? c.d_err + s0 : nullptr;
        rc = run_plan(sub, cc);
      }
      // the sub-stream's completion, for the caller's stream below (run_plan
      // happens to synchronise its stream today; the event keeps the
      // single-stream semantics if it stops doing so)
      if (!sub->ev_done) cu(cudaEventCreateWithFlags(&sub->ev_done, cudaEventDisableTiming));
      cu(cudaEventRecord(sub->ev_done, sub->stream));
      rcs[p] = rc;
    });
  }
  for (auto& t : th) t.join();
  for (int p = 0; p < parts; ++p)
    if (ctx->subs[p]->ev_done) PP_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->subs[p]->ev_done, 0));
  pp_stats S{};
  S.exit_thresh = INFINITY;
  for (int p = 0; p < parts; ++p) {
    pp_ctx* sub = ctx->subs[p];
    if (rcs[p] != PP_OK) return fail(ctx, rcs[p], sub->err);
    const pp_stats& t = sub->stats;
    S.candidates_generated += t.candidates_generated;
    S.candidates_ref_evaluated += t.candidates_ref_evaluated;
    S.candidates_evaluated += t.candidates_evaluated;
    S.transitions_executed += t.transitions_executed;
    S.transitions_reference += t.transitions_reference;
    S.slices_costed += t.slices_costed;
    S.waves = std::max(S.waves, t.waves);
    S.ms_sort = std::max(S.ms_sort, t.ms_sort);
    S.ms_cost = std::max(S.ms_cost, t.ms_cost);
    S.ms_dp = std::max(S.ms_dp, t.ms_dp);
    S.ms_total = std::max(S.ms_total, t.ms_total);
    for (int k = 0; k < 8; ++k) {
      S.ms_kernel[k] += t.ms_kernel[k];
      S.launches[k] += t.launches[k];
    }
    S.dp_band_bytes += t.dp_band_bytes;
    S.slices_pass_a += t.slices_pass_a;
    S.slices_pass_b += t.slices_pass_b;
    S.band_bytes += t.band_bytes;
    S.bound_transitions += t.bound_transitions;
    S.exit_thresh = std::min(S.exit_thresh, t.exit_thresh);
  }
  ctx->stats = S;
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
  for (pp_ctx* sub : ctx->subs) pp_ctx_destroy(sub);
  ctx->subs.clear();
  cudaSetDevice(ctx->device);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_done) cudaEventDestroy(ctx->ev_done);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->ostream) {
    cudaStreamSynchronize(ctx->ostream);
    cudaStreamDestroy(ctx->ostream);
  }
  for (cudaEvent_t e : ctx->piece_ev) cudaEventDestroy(e);
  if (ctx->cstream) {
    cudaStreamSynchronize(ctx->cstream);
    cudaStreamDestroy(ctx->cstream);
  }
  for (HostSet& h : ctx->hset) {
    if (h.h2d) cudaEventDestroy(h.h2d);
    if (h.d2h) cudaEventDestroy(h.d2h);
    h.hoff.release();
  }
  for (DevBuf* b : ctx->all_bufs()) b->release();
  for (PinBuf* b : {&ctx->h_range, &ctx->h_stats, &ctx->h_segdp, &ctx->h_gt_total, &ctx->arena.buf, &ctx->h_word})
    b->release();
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->kev) cudaEventDestroy(e);
  if (ctx->pstream) cudaStreamDestroy(ctx->pstream);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PP_OK;
}

const char* pp_ctx_last_error(const pp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int pp_ctx_set_tuning(pp_ctx* ctx, const pp_tuning* t) {
  if (!ctx || !t || t->first_wave < 1 || t->streams < 0 || t->streams > 16) return PP_ERR_INVALID;
  ctx->tuning = *t;
  // retired knobs (the DP reads dense tiles or the slice table only): the
  // compact band records and the in-DP pricing were measured slower
  // and the DP kernel no longer has those variants
  ctx->tuning.compact_band = 0;
  ctx->tuning.dp_pricing = 0;
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

int pp_pack_plan_slots(pp_ctx* ctx, const int32_t* d_count, const int32_t* d_status, const double* d_t_max_used,
                       const double* d_objective, const int32_t* d_splits, const int32_t* d_order,
                       const int64_t* d_seg_offsets, int32_t n_seg, int32_t n_max, int64_t* d_slots) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n_seg < 0 || n_max < 1 || !d_count || !d_status || !d_t_max_used || !d_objective || !d_splits ||
      !d_seg_offsets || !d_slots)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  PP_CUDA(launch_pack_slots(d_count, d_status, d_t_max_used, d_objective, d_splits, d_order, d_seg_offsets,
                            n_seg, n_max, reinterpret_cast<long long*>(d_slots), ctx->stream));
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
  NvtxRange nvtx("pp_plan_grid_device");
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
  c.d_order = d_out->order;
  c.d_splits = d_out->splits;
  c.d_times = d_out->mb_times;
  c.d_count = d_out->count;
  c.d_tmax = d_out->t_max_used;
  c.d_obj = d_out->objective;
  c.d_status = d_out->status;
  c.d_err = d_out->err_sample_id;
  if (!c.d_ordered) {  // the sort output is needed internally
    const int64_t total = h_seg_offsets[n_seg];
    PP_CUDA(ctx->ordered.ensure(std::max<int64_t>(total, 1) * sizeof(pp_sample)));
    c.d_ordered = ctx->ordered.as<pp_sample>();
  }
  if (ctx->tuning.streams > 1 && n_seg > 1) {
    if (h_seg_offsets[0] != 0) return fail(ctx, PP_ERR_INVALID, "seg_offsets[0] must be 0");
    for (int s = 0; s < n_seg; ++s)
      if (h_seg_offsets[s + 1] < h_seg_offsets[s])
        return fail(ctx, PP_ERR_INVALID, "seg_offsets must be non-decreasing");
    return plan_split(ctx, c, ctx->tuning.streams);
  }
  return run_plan(ctx, c);
}

}  // extern "C"

namespace {

// One host-buffer planning call on one context: stage the samples, plan on
// the device, copy the plans back (caller's buffers), synchronise.
int plan_host(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets, int32_t n_seg,
              int32_t presorted, const pp_grid_desc* grid, const pp_model_desc* model,
              const pp_dp_options* opts, const pp_plan_out* out) {
  const int64_t total = seg_offsets[n_seg];
  cudaStream_t st = ctx->stream;
  int rc;
  if ((rc = stage_inputs(ctx, samples, seg_offsets, n_seg))) return rc;
  PP_CUDA(ctx->out_splits.ensure(std::max<int64_t>(total, 1) * sizeof(int32_t)));
  PP_CUDA(ctx->out_times.ensure(std::max<int64_t>(total, 1) * sizeof(double)));
  PP_CUDA(ctx->out_count.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->out_tmax.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->out_obj.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->out_status.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->out_err.ensure(n_seg * sizeof(int64_t)));
  pp_plan_out d{};
  d.ordered = ctx->ordered.as<pp_sample>();
  if (out->order) {
    PP_CUDA(ctx->perm.ensure(std::max<int64_t>(total, 1) * sizeof(int32_t)));
    d.order = ctx->perm.as<int32_t>();
  }
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
  PP_CUDA(d2h(out->order, d.order, total * sizeof(int32_t)));
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

// pp_tuning::streams > 1 with host buffers: the batch is cut into 2 x streams
// contiguous chunks that `streams` host threads (each with its own
// sub-context and stream) take from a queue; a chunk is staged, planned and
// copied back on its own stream, so one chunk's copies overlap another's
// planning.
// A worker's chunk queue with its copies overlapped: while the compute stream
// plans chunk k, the copy stream stages chunk k+1's samples and drains chunk
// k-1's plans, through two alternating sets of device buffers (each set's
// outputs are reused only after their device->host copy completed).
// `claim` hands out chunk indices (-1: none left); chunk q covers segments
// [cut[q], cut[q + 1]).
// PP_E2E_TRACE=1: host timestamps of the host-buffer pipeline's phases,
// printed to stderr per call (development aid; no effect otherwise).
struct E2eTrace {
  bool on = std::getenv("PP_E2E_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(int worker, int chunk, const char* what) const {
    if (!on) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "e2e %9.1f us  w%d c%d %s\n", us, worker, chunk, what);
  }
};

// Large host<->device copies of the host-buffer pipeline go out in pieces of
// at most 4 MB, so the planning calls' small staging copies and read-backs on
// the other streams interleave with them in the copy engines instead of
// queueing behind tens of MB.
cudaError_t copy_pieces(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
  constexpr size_t kPiece = (size_t)4 << 20;
  for (size_t o = 0; o < bytes; o += kPiece) {
    const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                                          std::min(kPiece, bytes - o), kind, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// The valid prefix of each segment's splits / mb_times (count[s] entries, the
// API's contract: pp_plan_out) written straight into the caller's pinned
// buffers through their device alias — 12 B per micro-batch over PCIe
// instead of 12 B per sample through the copy engines (C3: ~1 MB instead of
// 87 MB per 888 mini-batches).  One CTA per segment; seg_off and the device
// arrays are relative to the part, the aliases already offset to it.
__global__ void prefix_out_kernel(const int64_t* __restrict__ seg_off, const int32_t* __restrict__ count,
                                  const int32_t* __restrict__ splits, const double* __restrict__ times,
                                  int32_t* h_splits, double* h_times) {
  const int s = blockIdx.x;
  const int64_t b = seg_off[s], n = seg_off[s + 1] - b;
  const int64_t cs = count[s] > 0 ? (int64_t)count[s] : 0;
  const int c = (int)(cs < n ? cs : n);
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    if (h_splits) h_splits[b + i] = splits[b + i];
    if (h_times) h_times[b + i] = times[b + i];
  }
}

// Device alias of a caller's host array when it is pinned (cudaHostAlloc /
// cudaHostRegister memory is mapped under UVA), else null: pageable output
// keeps the full-length copies.
template <class T>
T* device_alias(T* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer ? static_cast<T*>(a.devicePointer) : nullptr;
}

template <class Claim, class Done>
int plan_host_chunks(pp_ctx* sub, const pp_sample* samples, const int64_t* seg_offsets, const int* cut,
                     int32_t presorted, const pp_grid_desc* grid, const pp_model_desc* model,
                     const pp_dp_options* opts, const pp_plan_out* out, Claim claim, Done done,
                     const E2eTrace& tr, int wid) {
  pp_ctx* ctx = sub;  // (PP_CUDA reports on ctx)
  if (!sub->cstream) PP_CUDA(cudaStreamCreateWithFlags(&sub->cstream, cudaStreamNonBlocking));
  int32_t* const as_splits = device_alias(out->splits);
  double* const as_times = device_alias(out->mb_times);
  for (HostSet& h : sub->hset) {
    if (!h.h2d) PP_CUDA(cudaEventCreateWithFlags(&h.h2d, cudaEventDisableTiming));
    if (!h.d2h) PP_CUDA(cudaEventCreateWithFlags(&h.d2h, cudaEventDisableTiming));
    h.d2h_pending = false;
  }
  cudaStream_t cs = sub->cstream;
  auto stage = [&](int set, int q) -> int {
    HostSet& h = sub->hset[set];
    const int s0 = cut[q], s1 = cut[q + 1], ns = s1 - s0;
    const int64_t base = seg_offsets[s0], n = seg_offsets[s1] - base;
    PP_CUDA(h.hoff.ensure((ns + 1) * sizeof(int64_t)));
    int64_t* ho = h.hoff.as<int64_t>();
    for (int s = s0; s <= s1; ++s) ho[s - s0] = seg_offsets[s] - base;
    PP_CUDA(h.samples.ensure(std::max<int64_t>(n, 1) * sizeof(pp_sample)));
    PP_CUDA(h.seg.ensure((ns + 1) * sizeof(int64_t)));
    if (n > 0) PP_CUDA(copy_pieces(h.samples.p, samples + base, n * sizeof(pp_sample), cudaMemcpyHostToDevice, cs));
    PP_CUDA(cudaMemcpyAsync(h.seg.p, ho, (ns + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, cs));
    PP_CUDA(cudaEventRecord(h.h2d, cs));
    return PP_OK;
  };
  int rc = PP_OK;
  int q = claim(), set = 0;
  if (q >= 0 && (rc = stage(set, q))) return rc;
  tr.mark(wid, q, "staged");
  while (q >= 0) {
    const int qn = claim();
    // prefetch the next chunk's inputs — after this chunk's arrived, so the
    // first chunks of all workers cross PCIe ahead of any prefetch
    PP_CUDA(cudaEventSynchronize(sub->hset[set].h2d));
    tr.mark(wid, q, "h2d done");
    if (qn >= 0 && (rc = stage(set ^ 1, qn))) return rc;
    HostSet& h = sub->hset[set];
    const int s0 = cut[q], s1 = cut[q + 1], ns = s1 - s0;
    const int64_t base = seg_offsets[s0], n = seg_offsets[s1] - base;
    PP_CUDA(cudaStreamWaitEvent(sub->stream, h.h2d, 0));
    if (h.d2h_pending) PP_CUDA(cudaStreamWaitEvent(sub->stream, h.d2h, 0));
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    PP_CUDA(h.splits.ensure(nn * sizeof(int32_t)));
    PP_CUDA(h.times.ensure(nn * sizeof(double)));
    PP_CUDA(h.count.ensure(ns * sizeof(int32_t)));
    PP_CUDA(h.tmax.ensure(ns * sizeof(double)));
    PP_CUDA(h.obj.ensure(ns * sizeof(double)));
    PP_CUDA(h.status.ensure(ns * sizeof(int32_t)));
    PP_CUDA(h.err.ensure(ns * sizeof(int64_t)));
    pp_plan_out d{};
    if (out->ordered) {
      PP_CUDA(h.ordered.ensure(nn * sizeof(pp_sample)));
      d.ordered = h.ordered.as<pp_sample>();
    }
    if (out->order) {
      PP_CUDA(h.order.ensure(nn * sizeof(int32_t)));
      d.order = h.order.as<int32_t>();
    }
    d.splits = h.splits.as<int32_t>();
    d.mb_times = h.times.as<double>();
    d.count = h.count.as<int32_t>();
    d.t_max_used = h.tmax.as<double>();
    d.objective = h.obj.as<double>();
    d.status = h.status.as<int32_t>();
    d.err_sample_id = h.err.as<int64_t>();
    rc = pp_plan_grid_device(sub, h.samples.as<pp_sample>(), h.seg.as<int64_t>(), h.hoff.as<int64_t>(), ns,
                             presorted, grid, model, opts, &d);
    tr.mark(wid, q, "planned");
    if (rc) {
      cudaStreamSynchronize(cs);  // no copy into the caller's buffers after the call
      return rc;
    }
    done(q);
    // drain this chunk's plans on the copy stream (the compute stream is idle:
    // the planning call synchronised it)
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      return dst && bytes ? copy_pieces(dst, src, bytes, cudaMemcpyDeviceToHost, cs) : cudaSuccess;
    };
    PP_CUDA(d2h(out->ordered ? out->ordered + base : nullptr, d.ordered, n * sizeof(pp_sample)));
    PP_CUDA(d2h(out->order ? out->order + base : nullptr, d.order, n * sizeof(int32_t)));
    if (ns > 0 && (as_splits || as_times)) {
      prefix_out_kernel<<<ns, 128, 0, cs>>>(h.seg.as<int64_t>(), d.count, d.splits, d.mb_times,
                                            as_splits ? as_splits + base : nullptr,
                                            as_times ? as_times + base : nullptr);
      PP_CUDA(cudaGetLastError());
    }
    PP_CUDA(d2h(out->splits && !as_splits ? out->splits + base : nullptr, d.splits, n * sizeof(int32_t)));
    PP_CUDA(d2h(out->mb_times && !as_times ? out->mb_times + base : nullptr, d.mb_times, n * sizeof(double)));
    PP_CUDA(d2h(out->count ? out->count + s0 : nullptr, d.count, ns * sizeof(int32_t)));
    PP_CUDA(d2h(out->t_max_used ? out->t_max_used + s0 : nullptr, d.t_max_used, ns * sizeof(double)));
    PP_CUDA(d2h(out->objective ? out->objective + s0 : nullptr, d.objective, ns * sizeof(double)));
    PP_CUDA(d2h(out->status ? out->status + s0 : nullptr, d.status, ns * sizeof(int32_t)));
    PP_CUDA(d2h(out->err_sample_id ? out->err_sample_id + s0 : nullptr, d.err_sample_id, ns * sizeof(int64_t)));
    PP_CUDA(cudaEventRecord(h.d2h, cs));
    h.d2h_pending = true;
    q = qn;
    set ^= 1;
  }
  PP_CUDA(cudaStreamSynchronize(cs));
  tr.mark(wid, -1, "drained");
  return PP_OK;
}

// Host buffers, cut into `parts` parts by sample count: every part's
// samples go out at once, in part order, on one copy stream (one event per
// part), and `workers` host threads (sub-contexts with their own stream and
// scratch) plan parts w, w + workers, ... each as soon as its samples are in,
// then send its plans back on the worker's own copy stream while the worker
// plans its next part.  What stays exposed is the first part's upload and
// the last parts' download.  All small transfers inside a planning call are
// copy kernels through mapped pinned memory (small_copy), so they never wait
// behind these bulk copies in the copy engines.
int plan_host_pieces(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets, int32_t n_seg,
                     int32_t presorted, const pp_grid_desc* grid, const pp_model_desc* model,
                     const pp_dp_options* opts, const pp_plan_out* out, int parts, int workers) {
  parts = std::max(1, std::min(parts, (int)n_seg));
  workers = std::max(1, std::min(workers, parts));
  const int64_t total = seg_offsets[n_seg];
  std::vector<int> cut(parts + 1, 0);
  cut[parts] = n_seg;
  for (int p = 1; p < parts; ++p) {
    const int64_t target = total * p / parts;
    int s = cut[p - 1] + 1;
    while (s < n_seg - (parts - p) && seg_offsets[s] < target) ++s;
    cut[p] = s;
  }
  while ((int)ctx->subs.size() < workers) {
    pp_ctx* sub = nullptr;
    const int rc = pp_ctx_create(ctx->device, &sub);
    if (rc != PP_OK) return fail(ctx, rc, "cannot create a sub-context");
    ctx->subs.push_back(sub);
  }
  // later parts plan on higher-priority streams: their samples arrive last,
  // so their kernels go ahead of earlier parts' when both are ready and the
  // call's tail (the last part's planning + download) shrinks
  static const bool prio_on = std::getenv("PP_HOST_NO_PRIO") == nullptr;
  int p_least = 0, p_greatest = 0;
  if (prio_on) PP_CUDA(cudaDeviceGetStreamPriorityRange(&p_least, &p_greatest));
  std::vector<cudaStream_t> wstream(workers);
  for (int w = 0; w < workers; ++w) {
    pp_ctx* sub = ctx->subs[w];
    if (prio_on && !sub->pstream) {
      const int span = p_least - p_greatest;  // (priorities count down)
      const int prio = p_least - (workers > 1 ? w * span / (workers - 1) : 0);
      PP_CUDA(cudaStreamCreateWithPriority(&sub->pstream, cudaStreamNonBlocking, prio));
    }
    wstream[w] = prio_on ? sub->pstream : sub->stream;
  }
  if (!ctx->cstream) PP_CUDA(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  while ((int)ctx->piece_ev.size() < parts) {
    cudaEvent_t e;
    PP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->piece_ev.push_back(e);
  }
  int32_t* const as_splits = device_alias(out->splits);
  double* const as_times = device_alias(out->mb_times);
  const size_t nn = (size_t)std::max<int64_t>(total, 1);
  PP_CUDA(ctx->samples.ensure(nn * sizeof(pp_sample)));
  PP_CUDA(ctx->ordered.ensure(nn * sizeof(pp_sample)));
  PP_CUDA(ctx->seg_off.ensure((n_seg + parts) * sizeof(int64_t)));
  PP_CUDA(ctx->piece_off.ensure((n_seg + parts) * sizeof(int64_t)));
  PP_CUDA(ctx->out_splits.ensure(nn * sizeof(int32_t)));
  PP_CUDA(ctx->out_times.ensure(nn * sizeof(double)));
  PP_CUDA(ctx->out_count.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->out_tmax.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->out_obj.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->out_status.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->out_err.ensure(n_seg * sizeof(int64_t)));
  if (out->order) PP_CUDA(ctx->perm.ensure(nn * sizeof(int32_t)));
  // part-relative segment offsets, part p at [cut[p] + p, cut[p + 1] + p]
  int64_t* ho = ctx->piece_off.as<int64_t>();
  for (int p = 0; p < parts; ++p)
    for (int s = cut[p]; s <= cut[p + 1]; ++s) ho[s + p] = seg_offsets[s] - seg_offsets[cut[p]];
  cudaStream_t ci = ctx->cstream;
  for (int p = 0; p < parts; ++p) {
    const int64_t base = seg_offsets[cut[p]], n = seg_offsets[cut[p + 1]] - base;
    PP_CUDA(cudaMemcpyAsync(ctx->seg_off.as<int64_t>() + cut[p] + p, ho + cut[p] + p,
                            (cut[p + 1] - cut[p] + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, ci));
    if (n > 0)
      PP_CUDA(copy_pieces(ctx->samples.as<pp_sample>() + base, samples + base, n * sizeof(pp_sample),
                          cudaMemcpyHostToDevice, ci));
    PP_CUDA(cudaEventRecord(ctx->piece_ev[p], ci));
  }
  const E2eTrace tr;
  std::vector<int> rcs(workers, PP_OK);
  std::vector<pp_stats> acc(workers);
  std::vector<std::thread> th;
  for (int w = 0; w < workers; ++w) {
    th.emplace_back([&, w]() {
      pp_ctx* sub = ctx->subs[w];
      cudaSetDevice(sub->device);
      sub->tuning = ctx->tuning;
      sub->tuning.streams = 1;
      struct Restore {  // the sub-context's own stream back after the call
        pp_ctx* c;
        cudaStream_t s;
        ~Restore() { c->stream = s; }
      } restore{sub, sub->stream};
      sub->stream = wstream[w];
      pp_stats S{};
      S.exit_thresh = INFINITY;
      int rc = PP_OK;
      auto cu = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == PP_OK) {
          sub->err = cudaGetErrorString(e);
          rc = PP_ERR_CUDA;
        }
      };
      if (!sub->ostream) cu(cudaStreamCreateWithFlags(&sub->ostream, cudaStreamNonBlocking));
      while (rc == PP_OK && (int)sub->piece_ev.size() < 1) {
        cudaEvent_t e;
        cu(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        sub->piece_ev.push_back(e);
      }
      for (int p = w; p < parts && rc == PP_OK; p += workers) {
        const int s0 = cut[p], s1 = cut[p + 1];
        const int64_t base = seg_offsets[s0], n = seg_offsets[s1] - base;
        cu(cudaStreamWaitEvent(sub->stream, ctx->piece_ev[p], 0));
        if (tr.on) {
          cudaEventSynchronize(ctx->piece_ev[p]);
          tr.mark(w, p, "in");
        }
        PlanCall c;
        c.d_samples = ctx->samples.as<pp_sample>() + base;
        c.d_seg_off = ctx->seg_off.as<int64_t>() + s0 + p;
        c.h_seg_off = ho + s0 + p;
        c.n_seg = s1 - s0;
        c.presorted = presorted;
        c.grid = grid;
        c.model = model;
        c.opts = *opts;
        c.d_ordered = ctx->ordered.as<pp_sample>() + base;
        c.d_order = out->order ? ctx->perm.as<int32_t>() + base : nullptr;
        c.d_splits = ctx->out_splits.as<int32_t>() + base;
        c.d_times = ctx->out_times.as<double>() + base;
        c.d_count = ctx->out_count.as<int32_t>() + s0;
        c.d_tmax = ctx->out_tmax.as<double>() + s0;
        c.d_obj = ctx->out_obj.as<double>() + s0;
        c.d_status = ctx->out_status.as<int32_t>() + s0;
        c.d_err = ctx->out_err.as<int64_t>() + s0;
        if (rc == PP_OK) {
          NvtxRange nvtx("pp host part");
          rc = run_plan(sub, c);
        }
        tr.mark(w, p, "planned");
        if (rc != PP_OK) break;
        const pp_stats& t = sub->stats;
        S.candidates_generated += t.candidates_generated;
        S.candidates_ref_evaluated += t.candidates_ref_evaluated;
        S.candidates_evaluated += t.candidates_evaluated;
        S.transitions_executed += t.transitions_executed;
        S.transitions_reference += t.transitions_reference;
        S.slices_costed += t.slices_costed;
        S.waves = std::max(S.waves, t.waves);
        S.ms_sort += t.ms_sort;
        S.ms_cost += t.ms_cost;
        S.ms_dp += t.ms_dp;
        S.ms_total += t.ms_total;
        for (int q = 0; q < 8; ++q) {
          S.ms_kernel[q] += t.ms_kernel[q];
          S.launches[q] += t.launches[q];
        }
        S.dp_band_bytes += t.dp_band_bytes;
        S.slices_pass_a += t.slices_pass_a;
        S.slices_pass_b += t.slices_pass_b;
        S.band_bytes += t.band_bytes;
        S.bound_transitions += t.bound_transitions;
        S.exit_thresh = std::min(S.exit_thresh, t.exit_thresh);
        // this part's plans back to the caller while the worker plans its next part
        cudaStream_t co = sub->ostream;
        cu(cudaEventRecord(sub->piece_ev[0], sub->stream));
        cu(cudaStreamWaitEvent(co, sub->piece_ev[0], 0));
        auto d2h = [&](void* dst, const void* src, size_t bytes) {
          if (dst && bytes) cu(copy_pieces(dst, src, bytes, cudaMemcpyDeviceToHost, co));
        };
        d2h(out->ordered ? out->ordered + base : nullptr, c.d_ordered, n * sizeof(pp_sample));
        d2h(out->order ? out->order + base : nullptr, c.d_order, n * sizeof(int32_t));
        if (s1 > s0 && (as_splits || as_times)) {
          prefix_out_kernel<<<s1 - s0, 128, 0, co>>>(c.d_seg_off, c.d_count, c.d_splits, c.d_times,
                                                     as_splits ? as_splits + base : nullptr,
                                                     as_times ? as_times + base : nullptr);
          cu(cudaGetLastError());
        }
        d2h(out->splits && !as_splits ? out->splits + base : nullptr, c.d_splits, n * sizeof(int32_t));
        d2h(out->mb_times && !as_times ? out->mb_times + base : nullptr, c.d_times, n * sizeof(double));
        d2h(out->count ? out->count + s0 : nullptr, c.d_count, (s1 - s0) * sizeof(int32_t));
        d2h(out->t_max_used ? out->t_max_used + s0 : nullptr, c.d_tmax, (s1 - s0) * sizeof(double));
        d2h(out->objective ? out->objective + s0 : nullptr, c.d_obj, (s1 - s0) * sizeof(double));
        d2h(out->status ? out->status + s0 : nullptr, c.d_status, (s1 - s0) * sizeof(int32_t));
        d2h(out->err_sample_id ? out->err_sample_id + s0 : nullptr, c.d_err, (s1 - s0) * sizeof(int64_t));
      }
      // no copy into the caller's buffers after the call, failed or not
      if (sub->ostream) cudaStreamSynchronize(sub->ostream);
      tr.mark(w, -1, "drained");
      rcs[w] = rc;
      acc[w] = S;
    });
  }
  for (auto& t : th) t.join();
  cudaStreamSynchronize(ci);
  pp_stats S{};
  S.exit_thresh = INFINITY;
  for (int w = 0; w < workers; ++w) {
    if (rcs[w] != PP_OK) return fail(ctx, rcs[w], ctx->subs[w]->err);
    const pp_stats& t = acc[w];
    S.candidates_generated += t.candidates_generated;
    S.candidates_ref_evaluated += t.candidates_ref_evaluated;
    S.candidates_evaluated += t.candidates_evaluated;
    S.transitions_executed += t.transitions_executed;
    S.transitions_reference += t.transitions_reference;
    S.slices_costed += t.slices_costed;
    S.waves = std::max(S.waves, t.waves);
    S.ms_sort = std::max(S.ms_sort, t.ms_sort);
    S.ms_cost = std::max(S.ms_cost, t.ms_cost);
    S.ms_dp = std::max(S.ms_dp, t.ms_dp);
    S.ms_total = std::max(S.ms_total, t.ms_total);
    for (int q = 0; q < 8; ++q) {
      S.ms_kernel[q] += t.ms_kernel[q];
      S.launches[q] += t.launches[q];
    }
    S.dp_band_bytes += t.dp_band_bytes;
    S.slices_pass_a += t.slices_pass_a;
    S.slices_pass_b += t.slices_pass_b;
    S.band_bytes += t.band_bytes;
    S.bound_transitions += t.bound_transitions;
    S.exit_thresh = std::min(S.exit_thresh, t.exit_thresh);
  }
  ctx->stats = S;
  return PP_OK;
}

int plan_host_split(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets, int32_t n_seg,
                    int32_t presorted, const pp_grid_desc* grid, const pp_model_desc* model,
                    const pp_dp_options* opts, const pp_plan_out* out, int workers) {
  workers = std::min(workers, (int)n_seg);
  // >= two chunks per worker: one is planned while the next one's inputs and
  // the previous one's plans cross PCIe (plan_host_chunks)
  const int per_worker = -ctx->tuning.host_chunks >= 1 ? -ctx->tuning.host_chunks : 2;
  std::vector<int> wts(std::min<int>(n_seg, per_worker * workers), 1);
  const int chunks = (int)wts.size();
  while ((int)ctx->subs.size() < workers) {
    pp_ctx* sub = nullptr;
    const int rc = pp_ctx_create(ctx->device, &sub);
    if (rc != PP_OK) return fail(ctx, rc, "cannot create a sub-context");
    ctx->subs.push_back(sub);
  }
  const int64_t total = seg_offsets[n_seg];
  std::vector<int> cut(chunks + 1, 0);
  cut[chunks] = n_seg;
  int64_t wsum = 0, wacc = 0;
  for (int wt : wts) wsum += wt;
  for (int p = 1; p < chunks; ++p) {
    wacc += wts[p - 1];
    const int64_t target = total * wacc / wsum;
    int s = cut[p - 1] + 1;
    while (s < n_seg - (chunks - p) && seg_offsets[s] < target) ++s;
    cut[p] = s;
  }
  std::vector<int> rcs(workers, PP_OK);
  std::vector<pp_stats> acc(workers);
  std::vector<std::thread> th;
  const E2eTrace tr;
  for (int w = 0; w < workers; ++w) {
    th.emplace_back([&, w]() {
      pp_ctx* sub = ctx->subs[w];
      cudaSetDevice(sub->device);
      sub->tuning = ctx->tuning;
      sub->tuning.streams = 1;
      pp_stats S{};
      S.exit_thresh = INFINITY;
      // chunks w, w + workers, w + 2 workers, ... (static round robin: a
      // worker claims its next chunk early, to prefetch its inputs, so a
      // shared queue would let the first workers take chunks an idle worker
      // could have started on)
      int mine = w;
      auto claim = [&]() {
        const int k = mine;
        mine += workers;
        return k < chunks ? k : -1;
      };
      auto done = [&](int) {
        const pp_stats& t = sub->stats;
        S.candidates_generated += t.candidates_generated;
        S.candidates_ref_evaluated += t.candidates_ref_evaluated;
        S.candidates_evaluated += t.candidates_evaluated;
        S.transitions_executed += t.transitions_executed;
        S.transitions_reference += t.transitions_reference;
        S.slices_costed += t.slices_costed;
        S.waves = std::max(S.waves, t.waves);
        S.ms_sort += t.ms_sort;
        S.ms_cost += t.ms_cost;
        S.ms_dp += t.ms_dp;
        S.ms_total += t.ms_total;
        for (int q = 0; q < 8; ++q) {
          S.ms_kernel[q] += t.ms_kernel[q];
          S.launches[q] += t.launches[q];
        }
        S.dp_band_bytes += t.dp_band_bytes;
        S.slices_pass_a += t.slices_pass_a;
        S.slices_pass_b += t.slices_pass_b;
        S.band_bytes += t.band_bytes;
        S.bound_transitions += t.bound_transitions;
        S.exit_thresh = std::min(S.exit_thresh, t.exit_thresh);
      };
      rcs[w] = plan_host_chunks(sub, samples, seg_offsets, cut.data(), presorted, grid, model, opts, out,
                                claim, done, tr, w);
      acc[w] = S;
    });
  }
  for (auto& t : th) t.join();
  pp_stats S{};
  S.exit_thresh = INFINITY;
  for (int w = 0; w < workers; ++w) {
    if (rcs[w] != PP_OK) return fail(ctx, rcs[w], ctx->subs[w]->err);
    const pp_stats& t = acc[w];
    S.candidates_generated += t.candidates_generated;
    S.candidates_ref_evaluated += t.candidates_ref_evaluated;
    S.candidates_evaluated += t.candidates_evaluated;
    S.transitions_executed += t.transitions_executed;
    S.transitions_reference += t.transitions_reference;
    S.slices_costed += t.slices_costed;
    S.waves = std::max(S.waves, t.waves);
    S.ms_sort = std::max(S.ms_sort, t.ms_sort);
    S.ms_cost = std::max(S.ms_cost, t.ms_cost);
    S.ms_dp = std::max(S.ms_dp, t.ms_dp);
    S.ms_total = std::max(S.ms_total, t.ms_total);
    for (int q = 0; q < 8; ++q) {
      S.ms_kernel[q] += t.ms_kernel[q];
      S.launches[q] += t.launches[q];
    }
    S.dp_band_bytes += t.dp_band_bytes;
    S.slices_pass_a += t.slices_pass_a;
    S.slices_pass_b += t.slices_pass_b;
    S.band_bytes += t.band_bytes;
    S.bound_transitions += t.bound_transitions;
    S.exit_thresh = std::min(S.exit_thresh, t.exit_thresh);
  }
  ctx->stats = S;
  return PP_OK;
}

}  // namespace

extern "C" {

int pp_plan_grid(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets, int32_t n_seg,
                 int32_t presorted, const pp_grid_desc* grid, const pp_model_desc* model,
                 const pp_dp_options* opts, pp_plan_out* out) {
  NvtxRange nvtx("pp_plan_grid");
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!samples || !seg_offsets || n_seg < 1 || !opts || !out)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if ((rc = validate_opts(ctx, *opts))) return rc;
  if (seg_offsets[0] != 0) return fail(ctx, PP_ERR_INVALID, "seg_offsets[0] must be 0");
  for (int s = 0; s < n_seg; ++s)
    if (seg_offsets[s + 1] < seg_offsets[s]) return fail(ctx, PP_ERR_INVALID, "seg_offsets must be non-decreasing");
  if (ctx->tuning.streams > 1 && n_seg > 1) {
    if (ctx->tuning.host_chunks < 0)  // the concurrent-worker pipeline (A/B)
      return plan_host_split(ctx, samples, seg_offsets, n_seg, presorted, grid, model, opts, out,
                             ctx->tuning.streams);
    // parts: host_chunks per worker (default 1: smaller parts plan less
    // efficiently than the upload they hide, profiles/r02/e2e), workers: streams
    // default: 2 x streams workers with one part each — the parts start
    // staggered by their uploads, and more, smaller concurrent parts keep
    // the GPU busier at both ends of the call (C3, 888 mini-batches,
    // streams 3: 8.95 ms with 3 workers, 8.30 ms with 6; profiles/r02/e2e)
    if (ctx->tuning.host_chunks > 0)
      return plan_host_pieces(ctx, samples, seg_offsets, n_seg, presorted, grid, model, opts, out,
                              ctx->tuning.host_chunks * ctx->tuning.streams, ctx->tuning.streams);
    return plan_host_pieces(ctx, samples, seg_offsets, n_seg, presorted, grid, model, opts, out,
                            2 * ctx->tuning.streams, 2 * ctx->tuning.streams);
  }
  return plan_host(ctx, samples, seg_offsets, n_seg, presorted, grid, model, opts, out);
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
  if ((rc = stage_inputs(ctx, samples, seg_offsets, n_seg))) return rc;
  PP_CUDA(ctx->in_d.ensure(total * sizeof(double)));
  PP_CUDA(ctx->tgt_d.ensure(total * sizeof(double)));
  PP_CUDA(ctx->range.ensure(8 * sizeof(unsigned long long)));
  PP_CUDA(ctx->h_range.ensure(8 * sizeof(unsigned long long)));
  PP_CUDA(ctx->sort_keys.ensure(total * 6 * sizeof(unsigned long long)));
  PP_CUDA(ctx->sort_vals.ensure(total * 2 * sizeof(uint32_t)));
  PP_CUDA(launch_segmented_sort(ctx->samples.as<pp_sample>(), ctx->seg_off.as<int64_t>(), seg_offsets,
                                n_seg, total, 0, ctx->range.as<unsigned long long>(),
                                ctx->h_range.as<unsigned long long>(),
                                ctx->sort_keys.as<unsigned long long>(), ctx->sort_vals.as<uint32_t>(),
                                ctx->ordered.as<pp_sample>(), ctx->in_d.as<double>(),
                                ctx->tgt_d.as<double>(), nullptr, st));
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
  if (seg_offsets[0] != 0 || seg_offsets[n_seg] <= 0) return fail(ctx, PP_ERR_INVALID, "mini-batch is empty");
  ctx->kused = 0;
  ctx->kcat.clear();
  CostGrid g{};
  if ((rc = upload_grid(ctx, grid, model, &g))) return rc;
  if ((rc = stage_inputs(ctx, samples, seg_offsets, n_seg))) return rc;
  PlanCall c;
  c.d_samples = ctx->samples.as<pp_sample>();
  c.d_seg_off = ctx->seg_off.as<int64_t>();
  c.h_seg_off = seg_offsets;
  c.n_seg = n_seg;
  c.presorted = presorted;
  c.opts.stage_count = 2;
  c.opts.replica_count = 1;
  c.opts.per_mb_mem_cap = cap;
  c.opts.t_max_interval = 0.0;
  c.d_ordered = ctx->ordered.as<pp_sample>();
  std::vector<int> blk_base;
  int max_n = 0;
  // interval 0: the statistics are over the raw slice times
  if ((rc = cost_pass_a(ctx, c, g, 0.0, blk_base, max_n))) return rc;
  const SegStats* hs = ctx->h_stats.as<SegStats>();
  for (int s = 0; s < n_seg; ++s) {
    const bool any = hs[s].kmin != ~0ULL;
    t_min[s] = (hs[s].flags & 2) ? -INFINITY : any ? dkey_inv_host(hs[s].kmin) : (hs[s].flags & 1) ? INFINITY : NAN;
    t_max[s] = (hs[s].flags & 1) ? INFINITY : any ? dkey_inv_host(hs[s].kmax) : (hs[s].flags & 2) ? -INFINITY : NAN;
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


int pp_op_costs(pp_ctx* ctx, const pp_padded_shape* shapes, int64_t n, const pp_grid_desc* grid,
                const pp_model_desc* model, double* t_f, double* t_b, double* act_mem) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!shapes || !t_f || !t_b || !act_mem))) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  for (int64_t k = 0; k < n; ++k)
    if (shapes[k].mbs < 1) return fail(ctx, PP_ERR_INVALID, "micro-batch size must be >= 1");  // :299
  CostGrid g{};
  if ((rc = upload_grid(ctx, grid, model, &g))) return rc;
  if (n == 0) return PP_OK;
  const int C = model->n_stages;
  cudaStream_t st = ctx->stream;
  std::vector<double> lay(2 * (size_t)C);
  for (int j = 0; j < C; ++j) {
    lay[j] = model->encoder_layers[j] > 0 ? (double)model->encoder_layers[j] : 0.0;
    lay[C + j] = model->decoder_layers[j] > 0 ? (double)model->decoder_layers[j] : 0.0;
  }
  PP_CUDA(ctx->stage_lay.ensure(lay.size() * sizeof(double)));
  PP_CUDA(ctx->shapes.ensure(n * sizeof(pp_padded_shape)));
  PP_CUDA(ctx->oc_tf.ensure(n * C * sizeof(double)));
  PP_CUDA(ctx->oc_tb.ensure(n * C * sizeof(double)));
  PP_CUDA(ctx->oc_act.ensure(n * C * sizeof(double)));
  PP_CUDA(cudaMemcpyAsync(ctx->stage_lay.p, lay.data(), lay.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->shapes.p, shapes, n * sizeof(pp_padded_shape), cudaMemcpyHostToDevice, st));
  PP_CUDA(launch_op_costs(g, ctx->stage_lay.as<double>(), ctx->stage_lay.as<double>() + C, C,
                          ctx->shapes.as<pp_padded_shape>(), n, ctx->oc_tf.as<double>(), ctx->oc_tb.as<double>(),
                          ctx->oc_act.as<double>(), st));
  PP_CUDA(cudaMemcpyAsync(t_f, ctx->oc_tf.p, n * C * sizeof(double), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(t_b, ctx->oc_tb.p, n * C * sizeof(double), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(act_mem, ctx->oc_act.p, n * C * sizeof(double), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));  // lay dies here
  return PP_OK;
}

int pp_plan_op_costs_device(pp_ctx* ctx, const pp_sample* d_ordered, const int64_t* d_seg_offsets,
                            const int64_t* h_seg_offsets, int32_t n_seg, const int32_t* d_splits,
                            const int32_t* d_count, const pp_grid_desc* grid,
                            const pp_model_desc* model, int64_t capacity, int64_t* mb_offset,
                            double* d_t_f, double* d_t_b, double* d_act_mem) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n_seg < 1 || !d_ordered || !d_seg_offsets || !h_seg_offsets || !d_splits || !d_count || !mb_offset)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  CostGrid g{};
  if ((rc = upload_grid(ctx, grid, model, &g))) return rc;
  cudaStream_t st = ctx->stream;
  std::vector<int32_t> cnt(n_seg);
  PP_CUDA(cudaMemcpyAsync(cnt.data(), d_count, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  mb_offset[0] = 0;
  for (int s = 0; s < n_seg; ++s) mb_offset[s + 1] = mb_offset[s] + std::max(cnt[s], 0);
  const int64_t n_mb = mb_offset[n_seg];
  if (n_mb > capacity) return fail(ctx, PP_ERR_INVALID, "op-cost table capacity too small");
  if (n_mb == 0) return PP_OK;
  const int C = model->n_stages;
  std::vector<double> lay(2 * (size_t)C);
  for (int j = 0; j < C; ++j) {
    lay[j] = model->encoder_layers[j] > 0 ? (double)model->encoder_layers[j] : 0.0;
    lay[C + j] = model->decoder_layers[j] > 0 ? (double)model->decoder_layers[j] : 0.0;
  }
  PP_CUDA(ctx->stage_lay.ensure(lay.size() * sizeof(double)));
  PP_CUDA(ctx->mb_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->shapes.ensure(n_mb * sizeof(pp_padded_shape)));
  PP_CUDA(cudaMemcpyAsync(ctx->stage_lay.p, lay.data(), lay.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->mb_off.p, mb_offset, (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(launch_mb_shapes(d_ordered, d_seg_offsets, d_splits, ctx->mb_off.as<int64_t>(), n_seg, n_mb,
                           ctx->shapes.as<pp_padded_shape>(), st));
  PP_CUDA(launch_op_costs(g, ctx->stage_lay.as<double>(), ctx->stage_lay.as<double>() + C, C,
                          ctx->shapes.as<pp_padded_shape>(), n_mb, d_t_f, d_t_b, d_act_mem, st));
  PP_CUDA(cudaStreamSynchronize(st));  // lay and the offsets die here
  return PP_OK;
}

}  // extern "C"

namespace {

// select_recomputation over device-resident shapes (ctx->shapes, n_mb rows,
// ctx->mb_off per table): one op-cost table per allowed strategy, then the
// per-table choice (opcost.cu recompute_select_kernel).
int select_recompute_run(pp_ctx* ctx, const pp_grid_desc* grid, const pp_model_desc* model, int32_t mask,
                         const double* limits, int32_t n_seg, int64_t n_mb, double* d_t_f, double* d_t_b,
                         double* d_act, int32_t* d_strategy, int32_t* d_violating) {
  cudaStream_t st = ctx->stream;
  int tries[3], n_tries = 0;
  for (int r = 0; r < 3; ++r)  // the reference's canonical order (schedule.cpp:332-336)
    if (mask & (1 << r)) tries[n_tries++] = r;
  const int C = model->n_stages;
  std::vector<double> lay(2 * (size_t)C);
  for (int j = 0; j < C; ++j) {
    lay[j] = model->encoder_layers[j] > 0 ? (double)model->encoder_layers[j] : 0.0;
    lay[C + j] = model->decoder_layers[j] > 0 ? (double)model->decoder_layers[j] : 0.0;
  }
  const size_t tab = (size_t)std::max<int64_t>(n_mb, 1) * C;
  PP_CUDA(ctx->stage_lay.ensure(lay.size() * sizeof(double)));
  PP_CUDA(ctx->rc_tab.ensure(3 * (size_t)n_tries * tab * sizeof(double)));
  PP_CUDA(ctx->rc_lim.ensure((size_t)C * sizeof(double)));
  PP_CUDA(cudaMemcpyAsync(ctx->stage_lay.p, lay.data(), lay.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->rc_lim.p, limits, (size_t)C * sizeof(double), cudaMemcpyHostToDevice, st));
  double* tf_all = ctx->rc_tab.as<double>();
  double* tb_all = tf_all + (size_t)n_tries * tab;
  double* act_all = tb_all + (size_t)n_tries * tab;
  for (int q = 0; q < n_tries; ++q) {
    pp_model_desc m = *model;
    m.recompute = tries[q];
    CostGrid g{};
    int rc = upload_grid(ctx, grid, &m, &g);
    if (rc) return rc;
    PP_CUDA(launch_op_costs(g, ctx->stage_lay.as<double>(), ctx->stage_lay.as<double>() + C, C,
                            ctx->shapes.as<pp_padded_shape>(), n_mb, tf_all + q * tab, tb_all + q * tab,
                            act_all + q * tab, st));
  }
  PP_CUDA(launch_recompute_select(ctx->mb_off.as<int64_t>(), n_seg, C, n_tries, tries, n_mb, tf_all, tb_all,
                                  act_all, ctx->rc_lim.as<double>(), d_strategy, d_violating, d_t_f, d_t_b,
                                  d_act, st));
  return PP_OK;
}

int select_recompute_check(pp_ctx* ctx, int32_t n_seg, const pp_model_desc* model, int32_t mask,
                           const double* limits) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n_seg < 1 || !model || !limits) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if ((mask & 7) == 0) return fail(ctx, PP_ERR_INVALID, "no recompute strategies to try");  // schedule.cpp:323
  if (model->n_stages < 1) return fail(ctx, PP_ERR_INVALID, "stage and layer counts must be >= 1");
  return PP_OK;
}

}  // namespace

extern "C" {

int pp_select_recomputation(pp_ctx* ctx, const pp_padded_shape* shapes, const int64_t* mb_offset, int32_t n_seg,
                            const pp_grid_desc* grid, const pp_model_desc* model, int32_t strategies_mask,
                            const double* limits, double* t_f, double* t_b, double* act_mem, int32_t* strategy,
                            int32_t* violating_stage) {
  int rc = select_recompute_check(ctx, n_seg, model, strategies_mask, limits);
  if (rc) return rc;
  if (!mb_offset || !strategy || !violating_stage || (mb_offset[n_seg] > 0 && (!shapes || !t_f || !t_b || !act_mem)))
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  cudaStream_t st = ctx->stream;
  const int64_t n_mb = mb_offset[n_seg];
  const int C = model->n_stages;
  PP_CUDA(ctx->shapes.ensure(std::max<int64_t>(n_mb, 1) * sizeof(pp_padded_shape)));
  PP_CUDA(ctx->mb_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->oc_tf.ensure(std::max<int64_t>(n_mb, 1) * C * sizeof(double)));
  PP_CUDA(ctx->oc_tb.ensure(std::max<int64_t>(n_mb, 1) * C * sizeof(double)));
  PP_CUDA(ctx->oc_act.ensure(std::max<int64_t>(n_mb, 1) * C * sizeof(double)));
  PP_CUDA(ctx->rc_out.ensure(2 * (size_t)n_seg * sizeof(int32_t)));
  if (n_mb > 0)
    PP_CUDA(cudaMemcpyAsync(ctx->shapes.p, shapes, n_mb * sizeof(pp_padded_shape), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->mb_off.p, mb_offset, (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  int32_t* d_sv = ctx->rc_out.as<int32_t>();
  if ((rc = select_recompute_run(ctx, grid, model, strategies_mask, limits, n_seg, n_mb, ctx->oc_tf.as<double>(),
                                 ctx->oc_tb.as<double>(), ctx->oc_act.as<double>(), d_sv, d_sv + n_seg)))
    return rc;
  if (n_mb > 0) {
    PP_CUDA(cudaMemcpyAsync(t_f, ctx->oc_tf.p, n_mb * C * sizeof(double), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaMemcpyAsync(t_b, ctx->oc_tb.p, n_mb * C * sizeof(double), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaMemcpyAsync(act_mem, ctx->oc_act.p, n_mb * C * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  PP_CUDA(cudaMemcpyAsync(strategy, d_sv, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(violating_stage, d_sv + n_seg, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  return PP_OK;
}

int pp_select_recomputation_device(pp_ctx* ctx, const pp_sample* d_ordered, const int64_t* d_seg_offsets,
                                   const int64_t* h_seg_offsets, int32_t n_seg, const int32_t* d_splits,
                                   const int32_t* d_count, const pp_grid_desc* grid, const pp_model_desc* model,
                                   int32_t strategies_mask, const double* limits, int64_t capacity,
                                   int64_t* mb_offset, double* d_t_f, double* d_t_b, double* d_act_mem,
                                   int32_t* d_strategy, int32_t* d_violating_stage) {
  int rc = select_recompute_check(ctx, n_seg, model, strategies_mask, limits);
  if (rc) return rc;
  if (!d_ordered || !d_seg_offsets || !h_seg_offsets || !d_splits || !d_count || !mb_offset || !d_strategy ||
      !d_violating_stage)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  cudaStream_t st = ctx->stream;
  std::vector<int32_t> cnt(n_seg);
  PP_CUDA(cudaMemcpyAsync(cnt.data(), d_count, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  mb_offset[0] = 0;
  for (int s = 0; s < n_seg; ++s) mb_offset[s + 1] = mb_offset[s] + std::max(cnt[s], 0);
  const int64_t n_mb = mb_offset[n_seg];
  if (n_mb > capacity) return fail(ctx, PP_ERR_INVALID, "op-cost table capacity too small");
  PP_CUDA(ctx->mb_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->shapes.ensure(std::max<int64_t>(n_mb, 1) * sizeof(pp_padded_shape)));
  PP_CUDA(cudaMemcpyAsync(ctx->mb_off.p, mb_offset, (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(launch_mb_shapes(d_ordered, d_seg_offsets, d_splits, ctx->mb_off.as<int64_t>(), n_seg, n_mb,
                           ctx->shapes.as<pp_padded_shape>(), st));
  if ((rc = select_recompute_run(ctx, grid, model, strategies_mask, limits, n_seg, n_mb, d_t_f, d_t_b, d_act_mem,
                                 d_strategy, d_violating_stage)))
    return rc;
  PP_CUDA(cudaStreamSynchronize(st));  // the host offsets and limits die here
  return PP_OK;
}

}  // extern "C"

namespace {

// Shared body of pp_order_search{,_device}: every pointer is device memory
// except h_off and limits.
int order_search_run(pp_ctx* ctx, const double* d_tf, const double* d_tb, const double* d_act,
                     const int64_t* d_off, const int64_t* h_off, int32_t n_seg, int32_t C,
                     const double* limits, int32_t k, double comm_latency, int32_t* d_order,
                     double* d_ms, double* d_bub, int32_t* d_dl, double* d_ds, int32_t* d_status) {
  cudaStream_t st = ctx->stream;
  int64_t max_m = 1;
  std::vector<int32_t> stat(n_seg, PP_OK);
  for (int s = 0; s < n_seg; ++s) {
    const int64_t m = h_off[s + 1] - h_off[s];
    if (m < 1) stat[s] = PP_ERR_INVALID;  // "need at least one micro-batch" (schedule.cpp:281)
    if (m >= (int64_t)1 << 26) return fail(ctx, PP_ERR_INVALID, "micro-batch count too large");
    max_m = std::max(max_m, m);
  }
  int kfact = 1;
  for (int q = 2; q <= k; ++q) kfact *= q;
  const int64_t n_mb = h_off[n_seg] - h_off[0];
  // permutations per launch: all of them, or windows of at most ~4 M
  // (table, permutation) evaluations whose results fold into a running best
  constexpr int64_t kWindowItems = (int64_t)1 << 22;
  const int rwin = (int64_t)n_seg * kfact <= kWindowItems
                       ? kfact
                       : (int)std::max<int64_t>(1, kWindowItems / std::max<int32_t>(n_seg, 1));
  const int64_t n_items = (int64_t)n_seg * rwin;
  const size_t slot = order_search_slot_bytes(max_m, C);
  // scratch budget: half the free memory, at most 32 GB (one slot per
  // resident (mini-batch, permutation) evaluation; L2-resident when small)
  size_t free_b = 0, total_b = 0;
  PP_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const size_t budget = std::min<size_t>(free_b / 2, (size_t)32 << 30);
  const int warps = order_search_warps(n_items, C, slot, budget);
  int G = 1;
  while (G < C) G *= 2;
  PP_CUDA(ctx->os_lim.ensure(C * sizeof(double)));
  PP_CUDA(ctx->os_pred.ensure(std::max<int64_t>(n_mb + h_off[0], 1) * sizeof(double)));
  PP_CUDA(ctx->os_assign.ensure(std::max<int64_t>(n_mb + h_off[0], 1) * sizeof(int)));
  PP_CUDA(ctx->os_idx.ensure(std::max<int64_t>(n_mb + h_off[0], 1) * sizeof(int)));
  PP_CUDA(ctx->os_cloff.ensure((size_t)n_seg * (k + 1) * sizeof(int)));
  PP_CUDA(ctx->os_clk.ensure(n_seg * sizeof(int)));
  PP_CUDA(ctx->os_scratch.ensure((size_t)warps * (32 / G) * slot));
  PP_CUDA(ctx->os_items.ensure(n_items * order_search_item_bytes()));
  PP_CUDA(ctx->os_istats.ensure(n_items * 5 * C * sizeof(double)));
  if (rwin < kfact) {
    PP_CUDA(ctx->os_best.ensure((size_t)n_seg * order_search_best_bytes()));
    PP_CUDA(ctx->os_bstats.ensure((size_t)n_seg * 5 * C * sizeof(double)));
  }
  PP_CUDA(cudaMemcpyAsync(ctx->os_lim.p, limits, C * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(d_status, stat.data(), n_seg * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  // tables with no micro-batch are skipped by the kernels (cl_k = 0)
  PP_CUDA(ctx->os_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(cudaMemcpyAsync(ctx->os_off.p, d_off, (n_seg + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  PP_CUDA(launch_order_search(d_tf, d_tb, d_act, ctx->os_off.as<int64_t>(), n_seg, C, ctx->os_lim.as<double>(), k,
                              kfact, comm_latency, max_m, ctx->os_pred.as<double>(), ctx->os_assign.as<int>(),
                              ctx->os_idx.as<int>(), ctx->os_cloff.as<int>(), ctx->os_clk.as<int>(),
                              ctx->os_scratch.as<char>(), slot, warps, ctx->os_items.p,
                              d_ds ? ctx->os_istats.as<double>() : nullptr, d_order, d_ms, d_bub, d_dl, d_ds,
                              d_status, rwin, ctx->os_best.p, d_ds ? ctx->os_bstats.as<double>() : nullptr, st));
  PP_CUDA(cudaStreamSynchronize(st));  // stat / limits die here
  return PP_OK;
}

int order_search_check(pp_ctx* ctx, const int64_t* h_off, int32_t n_seg, int32_t C, const double* limits,
                       int32_t k) {
  if (n_seg < 0 || (n_seg > 0 && (!h_off || !limits))) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if (C < 1 || C > 32) return fail(ctx, PP_ERR_INVALID, "the device order search supports 1..32 stages");
  if (k < 1) return fail(ctx, PP_ERR_INVALID, "n_clusters must be >= 1");  // schedule.cpp:284
  if (k > 12) return fail(ctx, PP_ERR_INVALID, "the device order search supports n_clusters <= 12");
  for (int s = 0; s < n_seg; ++s)
    if (h_off[s + 1] < h_off[s]) return fail(ctx, PP_ERR_INVALID, "mb_offset must be non-decreasing");
  return PP_OK;
}

}  // namespace

extern "C" {

int pp_order_search(pp_ctx* ctx, const double* t_f, const double* t_b, const double* act_mem,
                    const int64_t* mb_offset, int32_t n_seg, int32_t n_stages, const double* limits,
                    int32_t n_clusters, double comm_latency, int32_t* order, double* makespan,
                    double* bubble_ratio, int32_t* deadlock, double* device_stats, int32_t* status) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if ((rc = order_search_check(ctx, mb_offset, n_seg, n_stages, limits, n_clusters))) return rc;
  if (n_seg == 0) return PP_OK;
  if (!t_f || !t_b || !act_mem || !order || !makespan || !status) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  const int C = n_stages;
  const int64_t o0 = mb_offset[0], n_mb = mb_offset[n_seg] - o0;
  std::vector<int64_t> off(n_seg + 1);
  for (int s = 0; s <= n_seg; ++s) off[s] = mb_offset[s] - o0;
  cudaStream_t st = ctx->stream;
  const size_t tb_bytes = std::max<int64_t>(n_mb, 1) * C * sizeof(double);
  PP_CUDA(ctx->os_tf.ensure(tb_bytes));
  PP_CUDA(ctx->os_tb.ensure(tb_bytes));
  PP_CUDA(ctx->os_act.ensure(tb_bytes));
  PP_CUDA(ctx->mb_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->os_order.ensure(std::max<int64_t>(n_mb, 1) * sizeof(int32_t)));
  PP_CUDA(ctx->os_ms.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->os_bub.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->os_dl.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->os_ds.ensure((size_t)n_seg * 5 * C * sizeof(double)));
  PP_CUDA(ctx->os_status.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(cudaMemcpyAsync(ctx->os_tf.p, t_f + o0 * C, n_mb * C * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->os_tb.p, t_b + o0 * C, n_mb * C * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->os_act.p, act_mem + o0 * C, n_mb * C * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->mb_off.p, off.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if ((rc = order_search_run(ctx, ctx->os_tf.as<double>(), ctx->os_tb.as<double>(), ctx->os_act.as<double>(),
                             ctx->mb_off.as<int64_t>(), off.data(), n_seg, C, limits, n_clusters, comm_latency,
                             ctx->os_order.as<int32_t>(), ctx->os_ms.as<double>(), ctx->os_bub.as<double>(),
                             ctx->os_dl.as<int32_t>(), device_stats ? ctx->os_ds.as<double>() : nullptr,
                             ctx->os_status.as<int32_t>())))
    return rc;
  PP_CUDA(cudaMemcpyAsync(order + o0, ctx->os_order.p, n_mb * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(makespan, ctx->os_ms.p, n_seg * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (bubble_ratio)
    PP_CUDA(cudaMemcpyAsync(bubble_ratio, ctx->os_bub.p, n_seg * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (deadlock)
    PP_CUDA(cudaMemcpyAsync(deadlock, ctx->os_dl.p, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (device_stats)
    PP_CUDA(cudaMemcpyAsync(device_stats, ctx->os_ds.p, (size_t)n_seg * 5 * C * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(status, ctx->os_status.p, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  return PP_OK;
}

int pp_order_search_device(pp_ctx* ctx, const double* d_t_f, const double* d_t_b,
                           const double* d_act_mem, const int64_t* d_mb_offset,
                           const int64_t* h_mb_offset, int32_t n_seg, int32_t n_stages,
                           const double* limits, int32_t n_clusters, double comm_latency,
                           int32_t* d_order, double* d_makespan, double* d_bubble_ratio,
                           int32_t* d_deadlock, double* d_device_stats, int32_t* d_status) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if ((rc = order_search_check(ctx, h_mb_offset, n_seg, n_stages, limits, n_clusters))) return rc;
  if (n_seg == 0) return PP_OK;
  if (!d_t_f || !d_t_b || !d_act_mem || !d_mb_offset || !d_order || !d_makespan || !d_status)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  return order_search_run(ctx, d_t_f, d_t_b, d_act_mem, d_mb_offset, h_mb_offset, n_seg, n_stages, limits,
                          n_clusters, comm_latency, d_order, d_makespan, d_bubble_ratio, d_deadlock,
                          d_device_stats, d_status);
}


}  // extern "C"

namespace {

// Emission of the chosen plans (device tables, orders and outputs).
int emit_plans_run(pp_ctx* ctx, const double* d_tf, const double* d_tb, const double* d_act, const int64_t* d_off,
                   const int64_t* h_off, int32_t n_seg, int32_t C, const double* limits, double comm_latency,
                   int32_t f1b, const int32_t* d_order, int32_t* d_ins, int32_t* d_nins, double* d_ms, double* d_bub,
                   int32_t* d_dl, double* d_ds, int32_t* d_status) {
  cudaStream_t st = ctx->stream;
  int64_t max_m = 1;
  for (int s = 0; s < n_seg; ++s) {
    const int64_t m = h_off[s + 1] - h_off[s];
    if (m >= (int64_t)1 << 26) return fail(ctx, PP_ERR_INVALID, "micro-batch count too large");
    max_m = std::max(max_m, m);
  }
  const int64_t rows = h_off[n_seg] - h_off[0];
  const size_t slot = order_search_slot_bytes(max_m, C);
  size_t free_b = 0, total_b = 0;
  PP_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const int warps = order_search_warps(n_seg, C, slot, std::min<size_t>(free_b / 2, (size_t)32 << 30));
  int G = 1;
  while (G < C) G *= 2;
  PP_CUDA(ctx->os_lim.ensure(C * sizeof(double)));
  PP_CUDA(ctx->os_scratch.ensure((size_t)warps * (32 / G) * slot));
  PP_CUDA(ctx->os_items.ensure((size_t)n_seg * order_search_item_bytes()));
  PP_CUDA(ctx->os_idx.ensure(std::max<int64_t>(rows + h_off[0], 1) * sizeof(int)));
  PP_CUDA(ctx->os_clk.ensure(n_seg * sizeof(int)));
  if (!f1b) PP_CUDA(up(ctx, ctx->os_lim.p, limits, C * sizeof(double)));
  PP_CUDA(launch_emit_plans(d_tf, d_tb, d_act, d_off, n_seg, C, ctx->os_lim.as<double>(), comm_latency, max_m,
                            d_order, f1b, ctx->os_scratch.as<char>(), slot, warps, ctx->os_items.p,
                            ctx->os_clk.as<int>(), ctx->os_idx.as<int>(), d_ins, d_nins, d_ms, d_bub, d_dl, d_ds,
                            d_status, st));
  PP_CUDA(cudaStreamSynchronize(st));
  return PP_OK;
}

}  // namespace

extern "C" {

int pp_emit_plans(pp_ctx* ctx, const double* t_f, const double* t_b, const double* act_mem, const int64_t* mb_offset,
                  int32_t n_seg, int32_t n_stages, const double* limits, double comm_latency, int32_t one_f_one_b,
                  const int32_t* order, int32_t* instructions, int32_t* n_instructions, double* makespan,
                  double* bubble_ratio, int32_t* deadlock, double* device_stats, int32_t* status) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n_seg < 0 || n_stages < 1 || n_stages > 32 || (n_seg > 0 && !mb_offset))
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if (n_seg == 0) return PP_OK;
  if (!t_f || !t_b || !act_mem || (!one_f_one_b && (!order || !limits)) || !instructions || !n_instructions ||
      !makespan || !status)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  for (int s = 0; s < n_seg; ++s)
    if (mb_offset[s + 1] < mb_offset[s]) return fail(ctx, PP_ERR_INVALID, "mb_offset must be non-decreasing");
  const int C = n_stages;
  const int64_t o0 = mb_offset[0], n_mb = mb_offset[n_seg] - o0;
  std::vector<int64_t> off(n_seg + 1);
  for (int s = 0; s <= n_seg; ++s) off[s] = mb_offset[s] - o0;
  cudaStream_t st = ctx->stream;
  const size_t tb_bytes = std::max<int64_t>(n_mb, 1) * C * sizeof(double);
  PP_CUDA(ctx->os_tf.ensure(tb_bytes));
  PP_CUDA(ctx->os_tb.ensure(tb_bytes));
  PP_CUDA(ctx->os_act.ensure(tb_bytes));
  PP_CUDA(ctx->mb_off.ensure((n_seg + 1) * sizeof(int64_t)));
  PP_CUDA(ctx->os_order.ensure(std::max<int64_t>(n_mb, 1) * sizeof(int32_t)));
  PP_CUDA(ctx->em_ins.ensure(std::max<int64_t>(n_mb, 1) * 10 * C * sizeof(int32_t)));
  PP_CUDA(ctx->em_nins.ensure((size_t)n_seg * C * sizeof(int32_t)));
  PP_CUDA(ctx->os_ms.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->os_bub.ensure(n_seg * sizeof(double)));
  PP_CUDA(ctx->os_dl.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(ctx->os_ds.ensure((size_t)n_seg * 5 * C * sizeof(double)));
  PP_CUDA(ctx->os_status.ensure(n_seg * sizeof(int32_t)));
  PP_CUDA(cudaMemcpyAsync(ctx->os_tf.p, t_f + o0 * C, n_mb * C * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->os_tb.p, t_b + o0 * C, n_mb * C * sizeof(double), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->os_act.p, act_mem + o0 * C, n_mb * C * sizeof(double), cudaMemcpyHostToDevice, st));
  if (!one_f_one_b)
    PP_CUDA(cudaMemcpyAsync(ctx->os_order.p, order + o0, n_mb * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  PP_CUDA(cudaMemcpyAsync(ctx->mb_off.p, off.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if ((rc = emit_plans_run(ctx, ctx->os_tf.as<double>(), ctx->os_tb.as<double>(), ctx->os_act.as<double>(),
                           ctx->mb_off.as<int64_t>(), off.data(), n_seg, C, limits, comm_latency, one_f_one_b,
                           ctx->os_order.as<int32_t>(), ctx->em_ins.as<int32_t>(), ctx->em_nins.as<int32_t>(),
                           ctx->os_ms.as<double>(), ctx->os_bub.as<double>(), ctx->os_dl.as<int32_t>(),
                           ctx->os_ds.as<double>(), ctx->os_status.as<int32_t>())))
    return rc;
  PP_CUDA(cudaMemcpyAsync(instructions + o0 * 10 * C, ctx->em_ins.p, n_mb * 10 * C * sizeof(int32_t),
                          cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(n_instructions, ctx->em_nins.p, (size_t)n_seg * C * sizeof(int32_t), cudaMemcpyDeviceToHost,
                          st));
  PP_CUDA(cudaMemcpyAsync(makespan, ctx->os_ms.p, n_seg * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (bubble_ratio)
    PP_CUDA(cudaMemcpyAsync(bubble_ratio, ctx->os_bub.p, n_seg * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (deadlock) PP_CUDA(cudaMemcpyAsync(deadlock, ctx->os_dl.p, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  if (device_stats)
    PP_CUDA(cudaMemcpyAsync(device_stats, ctx->os_ds.p, (size_t)n_seg * 5 * C * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaMemcpyAsync(status, ctx->os_status.p, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PP_CUDA(cudaStreamSynchronize(st));
  return PP_OK;
}

int pp_emit_plans_device(pp_ctx* ctx, const double* d_t_f, const double* d_t_b, const double* d_act_mem,
                         const int64_t* d_mb_offset, const int64_t* h_mb_offset, int32_t n_seg, int32_t n_stages,
                         const double* limits, double comm_latency, int32_t one_f_one_b, const int32_t* d_order,
                         int32_t* d_instructions, int32_t* d_n_instructions, double* d_makespan,
                         double* d_bubble_ratio, int32_t* d_deadlock, double* d_device_stats, int32_t* d_status) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n_seg < 0 || n_stages < 1 || n_stages > 32 || (n_seg > 0 && !h_mb_offset))
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if (n_seg == 0) return PP_OK;
  if (!d_t_f || !d_t_b || !d_act_mem || !d_mb_offset || (!one_f_one_b && (!d_order || !limits)) || !d_instructions ||
      !d_n_instructions || !d_makespan || !d_status)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  return emit_plans_run(ctx, d_t_f, d_t_b, d_act_mem, d_mb_offset, h_mb_offset, n_seg, n_stages, limits,
                        comm_latency, one_f_one_b, d_order, d_instructions, d_n_instructions, d_makespan,
                        d_bubble_ratio, d_deadlock, d_device_stats, d_status);
}

static const char* parse_msg(int kind) {
  switch (kind) {
    case PP_PARSE_MISSING_TAB: return "dataset record missing tab separator";
    case PP_PARSE_NOT_INTEGERS: return "dataset record is not a pair of integers";
    case PP_PARSE_INPUT_LT_1: return "dataset record has input_len < 1";
    default: return "dataset record has target_len < 0";
  }
}

int pp_load_records_device(pp_ctx* ctx, const char* d_bytes, int64_t n_bytes, int64_t max_seq_len,
                           pp_sample* d_out, int64_t capacity, int64_t* n_records, int64_t* err_line,
                           int64_t* err_byte, int32_t* err_kind) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n_bytes < 0 || (n_bytes > 0 && !d_bytes) || !n_records || !err_line || !err_byte || !err_kind ||
      capacity < 0)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  *n_records = 0;
  *err_line = -1;
  *err_byte = 0;
  *err_kind = 0;
  if (max_seq_len < 1) return fail(ctx, PP_ERR_INVALID, "max_seq_len must be >= 1");  // workload.cpp:110
  if (n_bytes >= ((int64_t)1 << 31) - 1) return fail(ctx, PP_ERR_INVALID, "record file too large (< 2 GiB)");
  const size_t need = ingest_scratch_bytes(n_bytes);
  PP_CUDA(ctx->ing_scratch.ensure(need));
  int64_t nrec = 0, nlines = 0, el = -1, eb = 0;
  int32_t ek = 0;
  PP_CUDA(launch_load_records(reinterpret_cast<const unsigned char*>(d_bytes), n_bytes, max_seq_len,
                              ctx->ing_scratch.as<char>(), ctx->ing_scratch.cap, d_out, capacity, &nrec, &nlines,
                              &el, &ek, &eb, ctx->stream));
  if (el >= 0) {
    *err_line = el + 1;
    *err_byte = eb;
    *err_kind = ek;
    return fail(ctx, PP_ERR_PARSE, std::string(parse_msg(ek)) + " (line " + std::to_string(el + 1) + ", byte " +
                                        std::to_string(eb) + ")");
  }
  *n_records = nrec;
  if (nrec == 0) return fail(ctx, PP_ERR_INVALID, "dataset is empty");  // workload.cpp:121
  if (nrec > capacity) return fail(ctx, PP_ERR_INVALID, "sample capacity too small");
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  return PP_OK;
}

int pp_load_records(pp_ctx* ctx, const char* bytes, int64_t n_bytes, int64_t max_seq_len, pp_sample* out,
                    int64_t capacity, int64_t* n_records, int64_t* err_line, int64_t* err_byte,
                    int32_t* err_kind) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n_bytes < 0 || (n_bytes > 0 && !bytes) || capacity < 0) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  PP_CUDA(ctx->ing_bytes.ensure(std::max<int64_t>(n_bytes, 1)));
  if (n_bytes > 0)
    PP_CUDA(cudaMemcpyAsync(ctx->ing_bytes.p, bytes, n_bytes, cudaMemcpyHostToDevice, ctx->stream));
  PP_CUDA(ctx->ing_out.ensure(std::max<int64_t>(capacity, 1) * sizeof(pp_sample)));
  rc = pp_load_records_device(ctx, ctx->ing_bytes.as<char>(), n_bytes, max_seq_len, ctx->ing_out.as<pp_sample>(),
                              capacity, n_records, err_line, err_byte, err_kind);
  if (rc) return rc;
  if (out && *n_records > 0)
    PP_CUDA(cudaMemcpyAsync(out, ctx->ing_out.p, *n_records * sizeof(pp_sample), cudaMemcpyDeviceToHost, ctx->stream));
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  return PP_OK;
}

int pp_draw_minibatches_device(pp_ctx* ctx, const pp_sample* d_samples, int64_t n, int64_t token_budget,
                               int64_t* d_seg_offsets, int64_t* n_seg) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!d_samples || !d_seg_offsets)) || !n_seg) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  if (token_budget < 1) return fail(ctx, PP_ERR_INVALID, "token_budget must be >= 1");  // workload.cpp:131
  if (n >= ((int64_t)1 << 31) - 2) return fail(ctx, PP_ERR_INVALID, "too many samples");
  PP_CUDA(ctx->ing_scratch.ensure(draw_scratch_bytes(n)));
  PP_CUDA(launch_draw_minibatches(d_samples, n, token_budget, ctx->ing_scratch.as<char>(), ctx->ing_scratch.cap,
                                  d_seg_offsets, n_seg, ctx->stream));
  return PP_OK;
}

int pp_draw_minibatches(pp_ctx* ctx, const pp_sample* samples, int64_t n, int64_t token_budget,
                        int64_t* seg_offsets, int64_t* n_seg) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!samples || !seg_offsets)) || !n_seg) return fail(ctx, PP_ERR_INVALID, "bad arguments");
  PP_CUDA(ctx->ing_out.ensure(std::max<int64_t>(n, 1) * sizeof(pp_sample)));
  PP_CUDA(ctx->ing_off.ensure((n + 1) * sizeof(int64_t)));
  if (n > 0)
    PP_CUDA(cudaMemcpyAsync(ctx->ing_out.p, samples, n * sizeof(pp_sample), cudaMemcpyHostToDevice, ctx->stream));
  rc = pp_draw_minibatches_device(ctx, ctx->ing_out.as<pp_sample>(), n, token_budget, ctx->ing_off.as<int64_t>(),
                                  n_seg);
  if (rc) return rc;
  if (n > 0)
    PP_CUDA(cudaMemcpyAsync(seg_offsets, ctx->ing_off.p, (*n_seg + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                            ctx->stream));
  else
    seg_offsets[0] = 0;
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  return PP_OK;
}


// padding_vs_packing_report, one max_seq_len at a time (simulate.cpp:296-403)
int pp_padding_report(pp_ctx* ctx, const pp_sample* samples, int64_t n, const int64_t* max_seq_lens,
                      int32_t n_lens, const pp_grid_desc* grid, const pp_model_desc* model,
                      int64_t token_budget, double t_max_interval, int32_t max_iterations,
                      int32_t recompute, pp_padding_row* rows) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (n < 1 || !samples) return fail(ctx, PP_ERR_INVALID, "padding report needs a non-empty dataset");  // :293
  if (n_lens < 0 || (n_lens > 0 && (!max_seq_lens || !rows)) || !grid || !model || model->n_stages < 1 ||
      model->n_stages > 32)
    return fail(ctx, PP_ERR_INVALID, "bad arguments");
  cudaStream_t st = ctx->stream;
  const int C = model->n_stages;
  PP_CUDA(ctx->rp_samples.ensure(n * sizeof(pp_sample)));
  PP_CUDA(ctx->rp_trunc.ensure(n * sizeof(pp_sample)));
  PP_CUDA(ctx->rp_off.ensure((n + 1) * sizeof(int64_t)));
  PP_CUDA(cudaMemcpyAsync(ctx->rp_samples.p, samples, n * sizeof(pp_sample), cudaMemcpyHostToDevice, st));
  pp_model_desc dpm = *model;
  dpm.recompute = recompute;
  pp_model_desc nm = *model;
  nm.recompute = 0;  // run_iteration prices with Recompute::None (:279)
  std::vector<int32_t> pe(C), pd(C);
  for (int j = 0; j < C; ++j) {  // packing merges both streams into one sequence (:357-364)
    pe[j] = model->is_encoder_decoder ? 0 : model->encoder_layers[j];
    pd[j] = model->is_encoder_decoder ? model->decoder_layers[j] + model->encoder_layers[j] : model->decoder_layers[j];
  }
  pp_model_desc pm = nm;
  pm.encoder_layers = pe.data();
  pm.decoder_layers = pd.data();
  pm.is_encoder_decoder = 0;
  const size_t ib = order_search_item_bytes();
  for (int L = 0; L < n_lens; ++L) {
    const int64_t max_len = max_seq_lens[L];
    PP_CUDA(launch_truncate(ctx->rp_samples.as<pp_sample>(), n, max_len, ctx->rp_trunc.as<pp_sample>(), st));
    int64_t n_seg64 = 0;
    if ((rc = pp_draw_minibatches_device(ctx, ctx->rp_trunc.as<pp_sample>(), n, token_budget,
                                         ctx->rp_off.as<int64_t>(), &n_seg64)))
      return rc;
    if (max_iterations > 0) n_seg64 = std::min<int64_t>(n_seg64, max_iterations);
    const int n_seg = (int)n_seg64;
    std::vector<int64_t> h_off(n_seg + 1);
    PP_CUDA(cudaMemcpyAsync(h_off.data(), ctx->rp_off.p, (n_seg + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaStreamSynchronize(st));
    const int64_t total = h_off[n_seg];
    // ---- DP micro-batching of every mini-batch (:310-326) ----
    PP_CUDA(ctx->rp_ordered.ensure(total * sizeof(pp_sample)));
    PP_CUDA(ctx->rp_splits.ensure(total * sizeof(int32_t)));
    PP_CUDA(ctx->rp_times.ensure(total * sizeof(double)));
    for (DevBuf* b : {&ctx->rp_count, &ctx->rp_status}) PP_CUDA(b->ensure(n_seg * sizeof(int32_t)));
    for (DevBuf* b : {&ctx->rp_tmax, &ctx->rp_obj}) PP_CUDA(b->ensure(n_seg * sizeof(double)));
    PP_CUDA(ctx->rp_err.ensure(n_seg * sizeof(int64_t)));
    pp_plan_out out{};
    out.ordered = ctx->rp_ordered.as<pp_sample>();
    out.splits = ctx->rp_splits.as<int32_t>();
    out.mb_times = ctx->rp_times.as<double>();
    out.count = ctx->rp_count.as<int32_t>();
    out.t_max_used = ctx->rp_tmax.as<double>();
    out.objective = ctx->rp_obj.as<double>();
    out.status = ctx->rp_status.as<int32_t>();
    out.err_sample_id = ctx->rp_err.as<int64_t>();
    const pp_dp_options opts{C, 1, INFINITY, t_max_interval};
    if ((rc = pp_plan_grid_device(ctx, ctx->rp_trunc.as<pp_sample>(), ctx->rp_off.as<int64_t>(), h_off.data(), n_seg,
                                  0, grid, &dpm, &opts, &out)))
      return rc;
    std::vector<int32_t> stv(n_seg);
    PP_CUDA(cudaMemcpyAsync(stv.data(), out.status, n_seg * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaStreamSynchronize(st));
    for (int q = 0; q < n_seg; ++q)
      if (stv[q] != PP_OK) return fail(ctx, stv[q], "dp_partition failed on a mini-batch of the report");
    // op costs of the DP micro-batches at Recompute::None
    std::vector<int64_t> mbo(n_seg + 1);
    for (DevBuf* b : {&ctx->rp_tf, &ctx->rp_tb, &ctx->rp_act}) PP_CUDA(b->ensure(std::max<int64_t>(total, 1) * C * sizeof(double)));
    if ((rc = pp_plan_op_costs_device(ctx, out.ordered, ctx->rp_off.as<int64_t>(), h_off.data(), n_seg, out.splits,
                                      out.count, grid, &nm, total, mbo.data(), ctx->rp_tf.as<double>(),
                                      ctx->rp_tb.as<double>(), ctx->rp_act.as<double>())))
      return rc;
    PP_CUDA(ctx->rp_st6.ensure((size_t)n_seg * 6 * sizeof(long long)));
    PP_CUDA(launch_dp_padded(ctx->shapes.as<pp_padded_shape>(), ctx->mb_off.as<int64_t>(), n_seg,
                             ctx->rp_st6.as<long long>(), st));
    // ---- packing / naive integer work (:328-379) ----
    PP_CUDA(ctx->rp_bins.ensure(std::max<int64_t>(total, 1) * sizeof(long long)));
    PP_CUDA(ctx->rp_naive.ensure(std::max(n_seg, 1) * sizeof(pp_padded_shape)));
    PP_CUDA(launch_minibatch_stats(ctx->rp_trunc.as<pp_sample>(), ctx->rp_off.as<int64_t>(), n_seg, max_len,
                                   ctx->rp_bins.as<long long>(), ctx->rp_st6.as<long long>(),
                                   ctx->rp_naive.as<pp_padded_shape>(), st));
    std::vector<long long> st6((size_t)n_seg * 6);
    PP_CUDA(cudaMemcpyAsync(st6.data(), ctx->rp_st6.p, st6.size() * sizeof(long long), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaStreamSynchronize(st));
    // ---- the three table sets, each simulated as one 1F1B iteration per mini-batch ----
    std::vector<int64_t> pko(n_seg + 1, 0), nvo(n_seg + 1);
    for (int q = 0; q < n_seg; ++q) pko[q + 1] = pko[q] + st6[6 * q + 3];
    for (int q = 0; q <= n_seg; ++q) nvo[q] = q;
    const int64_t n_dp = mbo[n_seg], n_pk = pko[n_seg];
    const int64_t rows_all = n_dp + n_pk + n_seg;
    PP_CUDA(ctx->rp_row.ensure(((size_t)rows_all * C * 3 + 3 * C) * sizeof(double)));
    double* pk_tf = ctx->rp_row.as<double>();
    double* pk_tb = pk_tf + n_pk * C;
    double* pk_ac = pk_tb + n_pk * C;
    double* nv_tf = pk_ac + n_pk * C;
    double* nv_tb = nv_tf + (int64_t)n_seg * C;
    double* nv_ac = nv_tb + (int64_t)n_seg * C;
    double* one = nv_ac + (int64_t)n_seg * C;  // the packed micro-batch's row
    CostGrid g{};
    std::vector<double> lay(2 * (size_t)C);
    // naive: one micro-batch per mini-batch under the model (Recompute::None)
    if ((rc = upload_grid(ctx, grid, &nm, &g))) return rc;
    for (int j = 0; j < C; ++j) {
      lay[j] = nm.encoder_layers[j] > 0 ? (double)nm.encoder_layers[j] : 0.0;
      lay[C + j] = nm.decoder_layers[j] > 0 ? (double)nm.decoder_layers[j] : 0.0;
    }
    PP_CUDA(ctx->stage_lay.ensure(lay.size() * sizeof(double)));
    PP_CUDA(cudaMemcpyAsync(ctx->stage_lay.p, lay.data(), lay.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    PP_CUDA(launch_op_costs(g, ctx->stage_lay.as<double>(), ctx->stage_lay.as<double>() + C, C,
                            ctx->rp_naive.as<pp_padded_shape>(), n_seg, nv_tf, nv_tb, nv_ac, st));
    PP_CUDA(cudaStreamSynchronize(st));  // lay is reused below
    // packing: every bin is {1, max_len, 0} under the merged-stream model
    if ((rc = upload_grid(ctx, grid, &pm, &g))) return rc;
    for (int j = 0; j < C; ++j) {
      lay[j] = pm.encoder_layers[j] > 0 ? (double)pm.encoder_layers[j] : 0.0;
      lay[C + j] = pm.decoder_layers[j] > 0 ? (double)pm.decoder_layers[j] : 0.0;
    }
    const pp_padded_shape pshape{1, max_len, 0};
    PP_CUDA(ctx->shapes.ensure(sizeof(pp_padded_shape)));
    PP_CUDA(cudaMemcpyAsync(ctx->stage_lay.p, lay.data(), lay.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    PP_CUDA(cudaMemcpyAsync(ctx->shapes.p, &pshape, sizeof(pshape), cudaMemcpyHostToDevice, st));
    PP_CUDA(launch_op_costs(g, ctx->stage_lay.as<double>(), ctx->stage_lay.as<double>() + C, C,
                            ctx->shapes.as<pp_padded_shape>(), 1, one, one + C, one + 2 * C, st));
    PP_CUDA(launch_broadcast_rows(one, one + C, one + 2 * C, C, n_pk, pk_tf, pk_tb, pk_ac, st));
    // offsets of the three sets, one device array
    PP_CUDA(ctx->rp_mboff.ensure(3 * (size_t)(n_seg + 1) * sizeof(int64_t)));
    int64_t* d_dpo = ctx->rp_mboff.as<int64_t>();
    int64_t* d_pko = d_dpo + n_seg + 1;
    int64_t* d_nvo = d_pko + n_seg + 1;
    PP_CUDA(cudaMemcpyAsync(d_dpo, mbo.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    PP_CUDA(cudaMemcpyAsync(d_pko, pko.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    PP_CUDA(cudaMemcpyAsync(d_nvo, nvo.data(), (n_seg + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    int64_t max_m = 1;
    for (int q = 0; q < n_seg; ++q) max_m = std::max({max_m, mbo[q + 1] - mbo[q], pko[q + 1] - pko[q]});
    const size_t slot = order_search_slot_bytes(max_m, C);
    size_t free_b = 0, total_b = 0;
    PP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const int warps = order_search_warps(n_seg, C, slot, std::min<size_t>(free_b / 2, (size_t)32 << 30));
    int G = 1;
    while (G < C) G *= 2;
    PP_CUDA(ctx->os_scratch.ensure((size_t)warps * (32 / G) * slot));
    PP_CUDA(ctx->rp_items.ensure(3 * (size_t)std::max(n_seg, 1) * ib));
    char* items = ctx->rp_items.as<char>();
    PP_CUDA(launch_sim_1f1b(ctx->rp_tf.as<double>(), ctx->rp_tb.as<double>(), ctx->rp_act.as<double>(), d_dpo, n_seg, C,
                            0.0, max_m, ctx->os_scratch.as<char>(), slot, warps, items, st));
    PP_CUDA(launch_sim_1f1b(pk_tf, pk_tb, pk_ac, d_pko, n_seg, C, 0.0, max_m, ctx->os_scratch.as<char>(), slot,
                            warps, items + (size_t)n_seg * ib, st));
    PP_CUDA(launch_sim_1f1b(nv_tf, nv_tb, nv_ac, d_nvo, n_seg, C, 0.0, max_m, ctx->os_scratch.as<char>(), slot,
                            warps, items + 2 * (size_t)n_seg * ib, st));
    std::vector<char> hi(3 * (size_t)n_seg * ib);
    PP_CUDA(cudaMemcpyAsync(hi.data(), items, hi.size(), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaStreamSynchronize(st));
    // accumulate in iteration order (:319-378), emit (:384-403)
    struct Acc {
      long long ai = 0, pi = 0, at = 0, pt = 0;
      double sim = 0.0;
    } acc[3];
    for (int q = 0; q < n_seg; ++q) {
      const long long* v = st6.data() + 6 * q;
      double ms[3];
      for (int m = 0; m < 3; ++m) {
        const char* it = hi.data() + ((size_t)m * n_seg + q) * ib;
        std::memcpy(&ms[m], it, sizeof(double));
        int32_t flags = 0;
        std::memcpy(&flags, it + 2 * sizeof(double), sizeof(int32_t));
        if ((flags >> 8) & 0xff) return fail(ctx, PP_ERR_NOT_EXECUTABLE, "1F1B plan not executable");
      }
      acc[0].ai += v[0]; acc[0].pi += v[4]; acc[0].at += v[1]; acc[0].pt += v[5]; acc[0].sim += ms[0];
      acc[1].ai += v[2]; acc[1].pi += v[3] * max_len; acc[1].sim += ms[1];
      acc[2].ai += v[0]; acc[2].at += v[1]; acc[2].sim += ms[2];
    }
    // naive padded sums: count * max lengths, from the naive shapes
    std::vector<pp_padded_shape> nsh(n_seg);
    PP_CUDA(cudaMemcpyAsync(nsh.data(), ctx->rp_naive.p, n_seg * sizeof(pp_padded_shape), cudaMemcpyDeviceToHost, st));
    PP_CUDA(cudaStreamSynchronize(st));
    for (int q = 0; q < n_seg; ++q) {
      acc[2].pi += nsh[q].mbs * nsh[q].input_len;
      acc[2].pt += nsh[q].mbs * nsh[q].target_len;
    }
    for (int m = 0; m < 3; ++m) {
      pp_padding_row& r = rows[3 * L + m];
      r.method = m;
      r.reserved = 0;
      r.max_seq_len = max_len;
      r.padding_eff_input = acc[m].pi == 0 ? 1.0 : (double)acc[m].ai / (double)acc[m].pi;
      r.padding_eff_target = acc[m].pt == 0 ? 1.0 : (double)acc[m].at / (double)acc[m].pt;
      r.tokens = acc[m].ai + acc[m].at;
      r.sim_time = acc[m].sim;
      r.throughput_proxy = acc[m].sim > 0 ? (double)r.tokens / acc[m].sim : 0.0;
    }
  }
  return PP_OK;
}

}  // extern "C"
