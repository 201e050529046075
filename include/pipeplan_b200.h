/* pipeplan_b200.h — C-ABI of the B200 micro-batch planner.
 *
 * This is the drop-in boundary underneath the reference planner's C++ API
 * (include/pipeplan/microbatch.h, cost_model.h).  Every signature uses plain
 * pointers, sizes and POD descriptors — no C++ or torch types — so a ctypes /
 * cgo / JNI stub can bind it directly (INTEGRATION.md shows the bindings).
 *
 * What each entry point replaces in the reference (/root/reference/proj):
 *
 *   pp_order_samples     order_samples(mb, OrderMethod::Sort)
 *                          src/microbatch.cpp:97-105, include/pipeplan/microbatch.h:59-63
 *   pp_plan_grid         order_samples(Sort) -> make_slice_cost(grid, cfg, ordered, r)
 *                          -> dp_partition(ordered, cost, opts), batched over
 *                          independent mini-batches (the run_plan worker pool,
 *                          src/driver.cpp:222-242).  Slice costing is
 *                          estimate()/ProfileGrid::per_layer (src/cost_model.cpp:126-150,
 *                          294-319) evaluated on the device, bit-exact.
 *                          include/pipeplan/microbatch.h:64-95
 *   pp_plan_grid_device  same, device-resident inputs/outputs on a caller stream
 *   pp_plan_tables       dp_partition() with an arbitrary SliceCostFn: the caller
 *                          evaluates the callback into the triangular tables the
 *                          reference builds at src/microbatch.cpp:228-243.
 *
 * Errors: a C-ABI cannot throw.  Every call returns a pp_status; per
 * mini-batch results carry their own status.  The C++ wrapper
 * (pipeplan::dp_partition) re-throws the reference's exception types with the
 * reference's messages (src/microbatch.cpp:98,222-226,248-250,320).
 *
 * Threading: a pp_ctx owns a CUDA stream and scratch buffers.  Calls on one
 * ctx are serialised by the caller; use one ctx per host thread (the C++
 * wrapper keeps a thread_local ctx), which matches the reference's reentrant,
 * thread-pooled use (src/driver.cpp:222-242).
 */
#ifndef PIPEPLAN_B200_H_
#define PIPEPLAN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_ABI_VERSION 1

typedef enum pp_status {
  PP_OK = 0,
  PP_ERR_INVALID = 1,          /* std::invalid_argument in the reference     */
  PP_ERR_INFEASIBLE_SAMPLE = 2,/* InfeasibleError(sample_id, -1), :248-250   */
  PP_ERR_INFEASIBLE = 3,       /* InfeasibleError(-1, -1), :320              */
  PP_ERR_CUDA = 4,             /* device error (distinct from domain errors) */
  PP_ERR_NO_DEVICE = 5,        /* no CUDA device: the product never falls back to CPU */
  PP_ERR_OUT_OF_RANGE = 6,     /* std::out_of_range (cost_model.cpp:297-298) */
  PP_ERR_NOT_CONVERGED = 7,    /* std::logic_error, schedule.cpp:81-82        */
  PP_ERR_NOT_EXECUTABLE = 8,   /* std::logic_error, schedule.cpp:155-156      */
  PP_ERR_PARSE = 9             /* ParseError (errors.h:25-40), workload.cpp:77-98 */
} pp_status;

/* ParseError kinds of load_record_file (src/workload.cpp:79-97), in the
 * reference's check order; the messages are the reference's. */
#define PP_PARSE_MISSING_TAB 0   /* "dataset record missing tab separator"     */
#define PP_PARSE_NOT_INTEGERS 1  /* "dataset record is not a pair of integers" */
#define PP_PARSE_INPUT_LT_1 2    /* "dataset record has input_len < 1"         */
#define PP_PARSE_TARGET_LT_0 3   /* "dataset record has target_len < 0"        */

/* Same layout as pipeplan::Sample (include/pipeplan/workload.h:27-33). */
typedef struct pp_sample {
  int64_t id;
  int64_t input_len;
  int64_t target_len;
} pp_sample;

/* A profile grid (reference ProfileGrid, cost_model.h:74-105).  cells holds
 * [kind(2)][recompute(3)][n_mbs][n_seq][3] doubles, fields (t_f, t_b, act_mem),
 * in the reference's cell_index order (src/cost_model.cpp:69-73). */
typedef struct pp_grid_desc {
  int32_t n_mbs;
  int32_t n_seq;
  const int64_t* mbs_axis;
  const int64_t* seq_axis;
  const double* cells;
} pp_grid_desc;

/* Reference ModelConfig (cost_model.h:113-127) reduced to what costing reads,
 * plus the recompute strategy passed to make_slice_cost. */
typedef struct pp_model_desc {
  int32_t n_stages;
  const int32_t* encoder_layers; /* [n_stages] */
  const int32_t* decoder_layers; /* [n_stages] */
  int32_t is_encoder_decoder;
  int32_t recompute;             /* 0 None, 1 Selective, 2 Full */
} pp_model_desc;

/* Reference PaddedShape (cost_model.h:52-56). */
typedef struct pp_padded_shape {
  int64_t mbs;
  int64_t input_len;
  int64_t target_len;
} pp_padded_shape;

/* Reference DpOptions (microbatch.h:79-86). */
typedef struct pp_dp_options {
  int32_t stage_count;
  int32_t replica_count;
  double per_mb_mem_cap;   /* +inf = no cap */
  double t_max_interval;   /* 0 = exact candidate set */
} pp_dp_options;

/* Planner knobs that never change results, only the schedule of work. */
typedef struct pp_tuning {
  int32_t first_wave;      /* t_max candidates evaluated in the first wave (>=1) */
  int32_t max_wave;        /* cap on a wave's candidates per mini-batch */
  int32_t streams;         /* >1: a batched call is split into this many contiguous
                              sub-batches planned concurrently on their own streams
                              and host threads (one sub-batch's latency-bound DP
                              overlaps another's cost passes); 0/1 = one stream */
  int32_t coop_min_n;      /* a DP launch of <= 8 passes whose mini-batches all have at
                              least this many samples runs each pass as one cooperative
                              kernel over the whole GPU; 0 = default (16384) */
  int32_t no_slice_reuse;  /* 1: price every band slice; 0 (default): sorted single-input
                              mini-batches price each distinct (micro-batch size, padded
                              length) pair once and copy it along the band's diagonal */
  int32_t no_band_trunc;   /* 1: candidate DP passes stream every tile column; 0 (default):
                              on certified length-sorted tiles they stop at the first
                              32-column chunk whose slices all exceed the candidate */
  int32_t compact_band;    /* retired (ignored): compact far-chunk records were measured slower
                              than dense tiles; the DP no longer reads them */
  int32_t host_chunks;     /* host-buffer calls with streams > 1: the call's samples are
                              uploaded part by part on one copy stream while workers plan
                              parts as they arrive and send plans back on their own copy
                              streams.  0 (default): 2 x streams workers, one part each;
                              k > 0: `streams` workers, k parts each.  Negative values
                              select the earlier concurrent-worker pipeline with -host_chunks
                              chunks per worker (A/B only) */
  int32_t dp_pricing;      /* retired (ignored): in-DP slice pricing was measured slower than
                              the shared slice table (no_slice_table = 0) */
  int32_t no_slice_table;  /* 1: length-sorted single-input mini-batches get a per-mini-batch
                              band from cost pass B; 0 (default): ONE slice table per call,
                              G[length][d] (a slice of such a mini-batch depends on its size
                              and padded length only), priced once, L2-resident, read by the
                              DP and the candidate scan — no band (gtab.cu) */
  int32_t no_bin_intervals; /* 1: the slice-table candidate scan reads every table entry a
                              mini-batch reaches; 0 (default): rows whose bins form an
                              interval for every prefix are marked from two entries */
} pp_tuning;

/* Per-call result arrays, all caller-owned.  Arrays sized [total samples] are
 * indexed like the input (segment s occupies [seg_offsets[s], seg_offsets[s+1])).
 *   ordered   : the order_samples(Sort) permutation of the segment (may be NULL)
 *   splits    : exclusive end of each micro-batch, relative to the segment start
 *               (the reference's Best::splits, microbatch.cpp:284); first
 *               count[s] entries valid
 *   mb_times  : slice time of each chosen micro-batch (microbatch.cpp:328)
 *   count, t_max_used, objective, status, err_sample_id : per segment
 *   (objective is eval_objective over mb_times, microbatch.cpp:333-334;
 *    t_max_used follows microbatch.cpp:335). */
typedef struct pp_plan_out {
  pp_sample* ordered;
  int32_t* splits;
  double* mb_times;
  int32_t* count;
  double* t_max_used;
  double* objective;
  int32_t* status;
  int64_t* err_sample_id;
  int32_t* order;  /* optional (may be NULL): the same ordering as `ordered`, as the
                      index (within the segment) of the input sample placed at each
                      position — 4 bytes per sample instead of a 24-byte copy */
} pp_plan_out;

/* Work counters for the last call (for benchmarks / rooflines). */
typedef struct pp_stats {
  int64_t candidates_generated;   /* sum over segments of |unique candidates| */
  int64_t candidates_evaluated;   /* DP passes actually run on the device      */
  int64_t transitions_executed;   /* DP transitions visited on the device      */
  int64_t transitions_reference;  /* n(n+1)/2 x passes the reference would run */
  int64_t slices_costed;          /* fused slice-cost evaluations              */
  int64_t waves;                  /* candidate waves launched                  */
  double  ms_sort, ms_cost, ms_dp, ms_total;  /* device time per phase          */
  /* per-kernel device time (CUDA events around each launch, on the ctx
   * stream) and launch counts: [0] segmented sort, [1] cost setup (axis
   * brackets, row widths, tile offsets), [2] cost pass A (act_mem, row
   * widths), [3] cost pass B (band tiles + candidate bins), [4] DP bound
   * pass (t = +inf; fused with the first candidate pass on certified sorted
   * GPT mini-batches), [5] DP candidate passes, [6] candidate compaction,
   * [7] selection / assembly */
  double  ms_kernel[8];
  int64_t launches[8];
  int64_t dp_band_bytes;          /* band bytes the DP passes read (8 B / transition) */
  int64_t slices_pass_a;          /* act_mem-only slices priced by cost pass A        */
  double  exit_thresh;            /* pass-A certified row-exit threshold (+inf: none) */
  int64_t slices_pass_b;          /* memory-feasible band slices priced by cost pass B */
  int64_t bound_transitions;      /* DP transitions of the bound pass (t = +inf)       */
  int64_t band_bytes;             /* band written by cost pass B (32-row tiles, 8 B/entry) */
  int64_t candidates_ref_evaluated; /* sum over segments of the candidates the reference's
                                       loop visits before its break (microbatch.cpp:289-292) */
} pp_stats;

typedef struct pp_ctx pp_ctx;

int pp_abi_version(void);
int pp_ctx_create(int device, pp_ctx** out);
int pp_ctx_destroy(pp_ctx* ctx);
const char* pp_ctx_last_error(const pp_ctx* ctx);
int pp_ctx_set_tuning(pp_ctx* ctx, const pp_tuning* tuning);
int pp_ctx_get_stats(const pp_ctx* ctx, pp_stats* out);
/* Optional: let the planner run on a caller-owned cudaStream_t. */
int pp_ctx_set_stream(pp_ctx* ctx, void* cuda_stream);

/* Segmented order_samples(Sort): host in, host out. */
int pp_order_samples(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets,
                     int32_t n_seg, pp_sample* out);

/* order_samples(Sort) + make_slice_cost + dp_partition for n_seg independent
 * mini-batches.  Host buffers in and out.  presorted != 0 skips the sort and
 * treats each segment as already ordered (the dp_partition(span) entry). */
int pp_plan_grid(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets,
                 int32_t n_seg, int32_t presorted, const pp_grid_desc* grid,
                 const pp_model_desc* model, const pp_dp_options* opts, pp_plan_out* out);

/* Same computation; samples / seg_offsets / every pp_plan_out array are
 * DEVICE pointers.  grid / model / opts descriptors are host structs. */
int pp_plan_grid_device(pp_ctx* ctx, const pp_sample* d_samples, const int64_t* d_seg_offsets,
                        const int64_t* h_seg_offsets, int32_t n_seg, int32_t presorted,
                        const pp_grid_desc* grid, const pp_model_desc* model,
                        const pp_dp_options* opts, pp_plan_out* d_out);

/* Fixed-size plan slots of n_seg planned mini-batches (pp_plan_grid_device
 * outputs, DEVICE pointers) for the multi-GPU epoch gather that replaces the
 * per-thread results of run_plan's pool (driver.cpp:222-242).  Slot s =
 * d_slots[s * words ..], words = 4 + ceil(n_max / 2) * (d_order ? 2 : 1):
 * [0] count [1] status [2] t_max_used bits [3] objective bits, then the
 * splits as packed int32, then (d_order non-NULL) the ordering as packed
 * int32 per-segment sample indices (micro-batch k = samples order[splits[k-1]
 * .. splits[k]), i.e. make_micro_batch's sample_ids, microbatch.cpp:122-134).
 * Enqueued on the ctx stream. */
int pp_pack_plan_slots(pp_ctx* ctx, const int32_t* d_count, const int32_t* d_status, const double* d_t_max_used,
                       const double* d_objective, const int32_t* d_splits, const int32_t* d_order,
                       const int64_t* d_seg_offsets, int32_t n_seg, int32_t n_max, int64_t* d_slots);

/* dp_partition over host-evaluated triangular slice tables: row i holds
 * slices [i, j) for j in (i, n] at index row_offset(i) + (j - i - 1)
 * (src/microbatch.cpp:228-243).  On PP_ERR_INFEASIBLE_SAMPLE, *err_index is
 * the ordered index of the offending sample. */
int pp_plan_tables(pp_ctx* ctx, const double* slice_time, const double* slice_mem, int64_t n,
                   const pp_dp_options* opts, int32_t* splits, double* mb_times, int32_t* count,
                   double* t_max_used, double* objective, int64_t* err_index);

/* Per segment: min / max slice time over memory-feasible slices (the
 * unquantized candidate range, microbatch.cpp:260-266 with I = 0), computed by
 * the device cost pass.  Used to map "K candidates" onto t_max_interval. */
int pp_candidate_range(pp_ctx* ctx, const pp_sample* samples, const int64_t* seg_offsets,
                       int32_t n_seg, int32_t presorted, const pp_grid_desc* grid,
                       const pp_model_desc* model, double per_mb_mem_cap, double* t_min,
                       double* t_max);

/* OpCostTable::from_shapes (src/cost_model.cpp:360-382, per shape and stage
 * estimate(), :294-319): t_f / t_b / act_mem of every (shape, stage) at
 * [shape * n_stages + stage], priced on the device, bit-exact.  Host buffers.
 * model->recompute selects the strategy (the planner may price a replica
 * with a different one than it partitioned with, planner.cpp:73-130). */
int pp_op_costs(pp_ctx* ctx, const pp_padded_shape* shapes, int64_t n, const pp_grid_desc* grid,
                const pp_model_desc* model, double* t_f, double* t_b, double* act_mem);

/* The same table for every micro-batch of plans already on the device
 * (pp_plan_grid_device outputs: ordered samples, splits, count): micro-batch
 * k of segment s is row mb_offset[s] + k at its padded shape (microbatch_cost
 * over the micro-batch's samples, cost_model.cpp:331-341).  mb_offset (host,
 * n_seg + 1 entries) is filled; the d_* tables are device arrays of
 * capacity x n_stages doubles (PP_ERR_INVALID if capacity is too small). */
int pp_plan_op_costs_device(pp_ctx* ctx, const pp_sample* d_ordered, const int64_t* d_seg_offsets,
                            const int64_t* h_seg_offsets, int32_t n_seg, const int32_t* d_splits,
                            const int32_t* d_count, const pp_grid_desc* grid,
                            const pp_model_desc* model, int64_t capacity, int64_t* mb_offset,
                            double* d_t_f, double* d_t_b, double* d_act_mem);

/* select_recomputation (src/schedule.cpp:319-364, include/pipeplan/
 * schedule.h:114-120; called per replica at planner.cpp:83-84), batched over
 * n_seg partitions: for each, the first strategy of {None, Selective, Full}
 * (in that order) whose bit is set in strategies_mask (1 << Recompute) and
 * whose OpCostTable::from_shapes has every act_mem(mb, j) < limits[j]
 * (limits: n_stages host doubles).  Per partition: strategy (the Recompute
 * value, or -1 when none fits — the reference's InfeasibleError) and
 * violating_stage (-1, or the lowest stage violated by the LAST strategy
 * tried: the exception's stage); rows mb_offset[s]..mb_offset[s+1] of the
 * t_f / t_b / act_mem tables hold the chosen strategy's costs.
 * PP_ERR_INVALID "no recompute strategies to try" for an empty mask
 * (schedule.cpp:323).  The reference's RecomputeSelection::schedule
 * (schedule_adaptive over the identity order) is not returned: plan_iteration
 * never reads it, and the order search evaluates the identity order itself.
 * Host buffers: shapes as pp_op_costs, mb_offset n_seg + 1 entries. */
int pp_select_recomputation(pp_ctx* ctx, const pp_padded_shape* shapes, const int64_t* mb_offset, int32_t n_seg,
                            const pp_grid_desc* grid, const pp_model_desc* model, int32_t strategies_mask,
                            const double* limits, double* t_f, double* t_b, double* act_mem, int32_t* strategy,
                            int32_t* violating_stage);
/* The same for plans already on the device (pp_plan_grid_device outputs),
 * like pp_plan_op_costs_device: mb_offset (host) is filled, the d_* outputs
 * are device arrays (tables of capacity x n_stages doubles, n_seg int32s). */
int pp_select_recomputation_device(pp_ctx* ctx, const pp_sample* d_ordered, const int64_t* d_seg_offsets,
                                   const int64_t* h_seg_offsets, int32_t n_seg, const int32_t* d_splits,
                                   const int32_t* d_count, const pp_grid_desc* grid, const pp_model_desc* model,
                                   int32_t strategies_mask, const double* limits, int64_t capacity,
                                   int64_t* mb_offset, double* d_t_f, double* d_t_b, double* d_act_mem,
                                   int32_t* d_strategy, int32_t* d_violating_stage);

/* Injection-order search of the per-replica planner:
 * order_microbatches(predicted, costs, limits, n_clusters, evaluator)
 * (src/schedule.cpp:277-317, include/pipeplan/schedule.h:101-108) with the
 * evaluator plan_iteration passes (src/planner.cpp:94-105): the makespan of
 * simulate(plan_communication(schedule_adaptive(costs, limits, order)),
 * costs, {noise_sigma 0, comm_latency}) (schedule.cpp:55-122,
 * comm_plan.cpp:115-233, simulate.cpp:78-213).  Batched over n_seg
 * independent op-cost tables (mini-batches / replicas): table s holds rows
 * [mb_offset[s], mb_offset[s+1]) of t_f / t_b / act_mem, [row * n_stages +
 * stage] (OpCostTable layout, cost_model.h:148-171; pp_op_costs output);
 * predicted times are OpCostTable::scalar_time (cost_model.cpp:344-348).
 * Outputs per table: order (n_s entries at mb_offset[s], the chosen
 * injection order; all -1 when no order is selectable, where the reference
 * returns an empty vector), makespan, bubble_ratio and deadlock of the chosen
 * order's SimReport (simulate.cpp:186-197), device_stats (optional,
 * [s][stage][5] = busy, idle, blocked, peak_mem, final_mem: DeviceStats,
 * simulate.h:30-36), status (PP_ERR_INVALID: no micro-batch or a negative /
 * NaN duration; PP_ERR_NOT_CONVERGED / PP_ERR_NOT_EXECUTABLE: the
 * reference's logic_errors).  Device limits: n_stages <= 32, n_clusters <= 12 (permutations beyond 8 clusters are
 * evaluated in windows folded into a running best).
 * Host buffers. */
int pp_order_search(pp_ctx* ctx, const double* t_f, const double* t_b, const double* act_mem,
                    const int64_t* mb_offset, int32_t n_seg, int32_t n_stages, const double* limits,
                    int32_t n_clusters, double comm_latency, int32_t* order, double* makespan,
                    double* bubble_ratio, int32_t* deadlock, double* device_stats, int32_t* status);

/* The same on device-resident tables (e.g. pp_plan_op_costs_device output)
 * on the ctx stream: d_* are device pointers, h_mb_offset / limits host. */
int pp_order_search_device(pp_ctx* ctx, const double* d_t_f, const double* d_t_b,
                           const double* d_act_mem, const int64_t* d_mb_offset,
                           const int64_t* h_mb_offset, int32_t n_seg, int32_t n_stages,
                           const double* limits, int32_t n_clusters, double comm_latency,
                           int32_t* d_order, double* d_makespan, double* d_bubble_ratio,
                           int32_t* d_deadlock, double* d_device_stats, int32_t* d_status);

/* The chosen plan of every replica, emitted on the device: for each table
 * s (op costs as pp_order_search) and its GIVEN injection order (order, n_s
 * entries at mb_offset[s]; e.g. pp_order_search's output), the
 * ExecutionPlan instruction lists of plan_communication(schedule_adaptive(
 * costs, limits, order)) (src/comm_plan.cpp:115-233, schedule.cpp:55-122) —
 * or of schedule_1f1b(n_s, C) when one_f_one_b (schedule.cpp:29-53; order
 * and limits unused) — with the zero-noise SimReport summary of that plan
 * (simulate.cpp:78-213) as pp_order_search reports it.  Device j's list of
 * table s is instructions[10 C mb_offset[s] + 10 n_s j ..] (capacity 10 x
 * n_stages x rows ints), n_instructions[s * n_stages + j] entries, each
 * (micro_batch << 4) | InstrKind with the reference's InstrKind numbering
 * (comm_plan.h:28-39: ForwardPass 0 ... WaitRecvGrad 9); the peer of a
 * transfer is the neighbouring stage (SendAct / WaitSendAct / RecvGrad /
 * WaitRecvGrad: j + 1, the others j - 1) and its shape boundary_shape() of
 * the micro-batch (comm_plan.cpp:104-113), so the plan file (save_plan,
 * comm_plan.cpp:313-342) is a formatting of these lists.  status:
 * PP_ERR_INVALID (no micro-batch, a negative / NaN duration, an order that
 * is not a permutation), PP_ERR_NOT_CONVERGED / PP_ERR_NOT_EXECUTABLE (the
 * reference's logic_errors).  Host buffers. */
int pp_emit_plans(pp_ctx* ctx, const double* t_f, const double* t_b, const double* act_mem, const int64_t* mb_offset,
                  int32_t n_seg, int32_t n_stages, const double* limits, double comm_latency, int32_t one_f_one_b,
                  const int32_t* order, int32_t* instructions, int32_t* n_instructions, double* makespan,
                  double* bubble_ratio, int32_t* deadlock, double* device_stats, int32_t* status);
/* save_plan's text (src/comm_plan.cpp:313-342) of ONE table of a
 * pp_emit_plans result: instructions / n_instructions of that table (device
 * j's list at instructions[10 * micro_batches * j]), the micro-batches'
 * padded shapes, the model's stage layouts and recompute strategy, and the
 * PlanMeta fields (src/planner.cpp:86-95); into out (cap bytes, NUL
 * terminated), *len = the full text length.  Host code (plan_file.cpp). */
int pp_format_plan(const int32_t* instructions, const int32_t* n_instructions, int32_t n_stages,
                   int32_t micro_batches, const pp_padded_shape* shapes, const pp_model_desc* model,
                   int64_t iteration, int32_t replica, int64_t hidden_dim, char* out, int64_t cap, int64_t* len);
/* The same on device-resident tables, orders and outputs (ctx stream). */
int pp_emit_plans_device(pp_ctx* ctx, const double* d_t_f, const double* d_t_b, const double* d_act_mem,
                         const int64_t* d_mb_offset, const int64_t* h_mb_offset, int32_t n_seg, int32_t n_stages,
                         const double* limits, double comm_latency, int32_t one_f_one_b, const int32_t* d_order,
                         int32_t* d_instructions, int32_t* d_n_instructions, double* d_makespan,
                         double* d_bubble_ratio, int32_t* d_deadlock, double* d_device_stats, int32_t* d_status);

/* Dataset ingest on the device: load_dataset over a
 * record file (src/workload.cpp:65-103 load_record_file + :109-127
 * truncation to max_seq_len), given the file's bytes.  out receives the
 * samples (id = record index) when capacity allows; *n_records is set either
 * way.  PP_ERR_PARSE: the first malformed line, *err_line 1-based,
 * *err_byte its offset, *err_kind a PP_PARSE_* kind.  PP_ERR_INVALID:
 * max_seq_len < 1, "dataset is empty" (no record), or capacity too small.
 * Host buffers (the bytes are copied to the device). */
int pp_load_records(pp_ctx* ctx, const char* bytes, int64_t n_bytes, int64_t max_seq_len, pp_sample* out,
                    int64_t capacity, int64_t* n_records, int64_t* err_line, int64_t* err_byte,
                    int32_t* err_kind);
/* The same with the bytes and the output on the device (ctx stream). */
int pp_load_records_device(pp_ctx* ctx, const char* d_bytes, int64_t n_bytes, int64_t max_seq_len,
                           pp_sample* d_out, int64_t capacity, int64_t* n_records, int64_t* err_line,
                           int64_t* err_byte, int32_t* err_kind);

/* The mini-batches run_plan draws over a sample stream (src/driver.cpp:211,
 * draw_minibatch src/workload.cpp:129-146, cursor 0 onwards): consecutive
 * samples until the running total_tokens reaches token_budget, the crossing
 * sample included.  seg_offsets (capacity n + 1) receives the n_seg + 1
 * boundaries, directly usable as pp_plan_grid's seg_offsets.
 * PP_ERR_INVALID: token_budget < 1. */
int pp_draw_minibatches(pp_ctx* ctx, const pp_sample* samples, int64_t n, int64_t token_budget,
                        int64_t* seg_offsets, int64_t* n_seg);
int pp_draw_minibatches_device(pp_ctx* ctx, const pp_sample* d_samples, int64_t n, int64_t token_budget,
                               int64_t* d_seg_offsets, int64_t* n_seg);

/* One row of padding_vs_packing_report (PaddingRow, include/pipeplan/simulate.h:92-100). */
typedef struct pp_padding_row {
  int32_t method;            /* 0 DpMicrobatch, 1 Packing, 2 NaivePadding (BatchingMethod) */
  int32_t reserved;
  int64_t max_seq_len;
  double padding_eff_input;
  double padding_eff_target;
  int64_t tokens;
  double sim_time;
  double throughput_proxy;
} pp_padding_row;

/* padding_vs_packing_report (src/simulate.cpp:288-406, the second production
 * caller of dp_partition) on the device: per max_seq_len, truncation, the
 * token-budgeted draw (pp_draw_minibatches), the DP partition of every
 * mini-batch in one batched call (order_samples(Sort) -> make_slice_cost(grid,
 * model, ordered, recompute) -> dp_partition with t_max_interval), first-fit
 * packing and naive padding, and one zero-noise 1F1B simulate() per mini-batch
 * and method (schedule_1f1b -> plan_communication -> simulate over
 * OpCostTable::from_shapes at Recompute::None).  rows receives 3 * n_lens rows
 * in the reference's order (DP, packing, naive per max_seq_len).  model's
 * recompute field is ignored (the DP uses `recompute`, the simulations None).
 * Host buffers; errors as the reference (PP_ERR_INVALID for an empty dataset or
 * token_budget < 1; the DP's own errors). */
int pp_padding_report(pp_ctx* ctx, const pp_sample* samples, int64_t n, const int64_t* max_seq_lens,
                      int32_t n_lens, const pp_grid_desc* grid, const pp_model_desc* model,
                      int64_t token_budget, double t_max_interval, int32_t max_iterations,
                      int32_t recompute, pp_padding_row* rows);

/* Diagnostics: measured FP64 add issue rate of `device` (adds/s), the
 * roofline denominator of the FP64-bound cost kernels (calib.cu). */
int pp_calibrate_fp64(int device, double* dadd_per_s);

/* ---- host helpers (no device work): the drop-in C++ API exposed to C ---- */
/* eval_objective (microbatch.cpp:109-120) */
int pp_eval_objective(const double* times, int64_t m, int32_t stage_count, int32_t replica_count,
                      double* out);
/* dp_partition's tail (microbatch.cpp:337-348): replica_assignment of the m
 * planned micro-batches (balance_replicas when m >= replica_count, else
 * micro-batch k -> replica k) and max_replica_load, from their times. */
int pp_assign_replicas(const double* times, int64_t m, int32_t replica_count, int32_t* replica,
                       double* max_load);
/* ProfileGrid::synthetic (cost_model.cpp:91-124).  params = {alpha, beta, gamma,
 * full_mem_factor, selective_mem_factor, full_tb_penalty, selective_tb_penalty};
 * empty axes (n = 0) select the defaults.  out_mbs/out_seq need 64 entries,
 * out_cells 2*3*n_mbs*n_seq*3; out_sizes receives (n_mbs, n_seq). */
int pp_synthetic_grid(const double* params, int32_t tp_degree, const int64_t* mbs_axis,
                      int32_t n_mbs, const int64_t* seq_axis, int32_t n_seq, int64_t* out_mbs,
                      int64_t* out_seq, int32_t* out_sizes, double* out_cells);
/* load_dataset with a synthetic descriptor (workload.cpp:50-63,109-127).
 * dist = {family(0 lognormal,1 uniform,2 mixture), log_mean, log_sigma,
 *         uniform_lo, uniform_hi, lognormal_weight}; tgt_dist may be NULL. */
int pp_synthetic_dataset(int64_t n, const double* in_dist, const double* tgt_dist,
                         int64_t max_seq_len, uint64_t seed, pp_sample* out);
/* The make_slice_cost lambda on the host for one slice [begin, end). */
int pp_slice_cost_host(const pp_grid_desc* grid, const pp_model_desc* model,
                       const pp_sample* ordered, int64_t begin, int64_t end, double* time,
                       double* act_mem);

#ifdef __cplusplus
}
#endif
#endif /* PIPEPLAN_B200_H_ */
