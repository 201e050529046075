/* pp_oracle.h — CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the CHECKER.  The product library never
 * links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * reference's own known-answer tests (tests/golden/known_answers.json, transcribed
 * from proj/tests/test_microbatch.cpp and test_cost_model.cpp) and against the
 * unmodified reference compiled into oracle/_ref/ (tests/golden/*.json were
 * generated from it by tests/golden/make_golden.py).
 */
#ifndef PP_ORACLE_H_
#define PP_ORACLE_H_
#include <stdint.h>

#include "pipeplan_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

int orc_order_samples(const pp_sample* in, int64_t n, pp_sample* out);
int orc_per_layer(const pp_grid_desc* g, int32_t kind, int32_t r, double mbs, double seqlen,
                  double out[3]);
int orc_estimate(const pp_grid_desc* g, const pp_model_desc* m, int32_t stage, int64_t mbs,
                 int64_t max_in, int64_t max_tgt, double out[3]);
int orc_slice_cost(const pp_grid_desc* g, const pp_model_desc* m, const pp_sample* ordered,
                   int64_t begin, int64_t end, double* time, double* act_mem);
int orc_dp_tables(const double* slice_time, const double* slice_mem, int64_t n,
                  const pp_dp_options* o, int32_t* splits, double* mb_times, int32_t* count,
                  double* t_max_used, double* objective, int64_t* err_index,
                  int64_t* n_candidates, int64_t* n_evaluated);
int orc_plan_grid(const pp_sample* samples, int64_t n, int32_t presorted, const pp_grid_desc* g,
                  const pp_model_desc* m, const pp_dp_options* o, pp_sample* ordered,
                  int32_t* splits, double* mb_times, int32_t* count, double* t_max_used,
                  double* objective, int64_t* err_sample_id, int64_t* n_candidates,
                  int64_t* n_evaluated);
int orc_slice_extrema(const pp_sample* ordered, int64_t n, const pp_grid_desc* g,
                      const pp_model_desc* m, double cap, double* t_capmax, double* single_act_max);
/* Streaming restatement (pp_stream.c): no O(n^2) tables, slices priced on the
 * fly, `threads` OpenMP threads.  Same outputs as orc_plan_grid. */
int orc_plan_grid_stream(const pp_sample* samples, int64_t n, int32_t presorted, const pp_grid_desc* g,
                         const pp_model_desc* m, const pp_dp_options* o, int32_t threads,
                         pp_sample* ordered, int32_t* splits, double* mb_times, int32_t* count,
                         double* t_max_used, double* objective, int64_t* err_sample_id,
                         int64_t* n_candidates, int64_t* n_evaluated);
int orc_eval_objective(const double* times, int64_t m, int32_t c, int32_t d, double* out);

#ifdef __cplusplus
}
#endif
#endif
