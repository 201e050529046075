/* pp_oracle.c — plain-C restatement of the reference micro-batch planner hot
 * path (DynaPipe arXiv 2311.10418, /root/reference/proj).
 *
 * TEST INFRASTRUCTURE ONLY (see pp_oracle.h).  It is deliberately a literal,
 * sequential restatement: same operation order, same comparisons, same
 * tie-breaks, no FMA contraction (built with -ffp-contract=off), so its
 * output is bit-identical to the reference.  Each function cites the
 * reference lines it restates.
 */
#include "pp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- order_samples(Sort): src/microbatch.cpp:97-105 ---------------------- */
static int cmp_sample(const void* pa, const void* pb) {
  const pp_sample* a = (const pp_sample*)pa;
  const pp_sample* b = (const pp_sample*)pb;
  /* std::tie(input_len, target_len, id) < ... (microbatch.cpp:101-103) */
  if (a->input_len != b->input_len) return a->input_len < b->input_len ? -1 : 1;
  if (a->target_len != b->target_len) return a->target_len < b->target_len ? -1 : 1;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return 0;
}

int orc_order_samples(const pp_sample* in, int64_t n, pp_sample* out) {
  if (n <= 0) return PP_ERR_INVALID; /* "mini-batch is empty" (:98) */
  memcpy(out, in, (size_t)n * sizeof(pp_sample));
  qsort(out, (size_t)n, sizeof(pp_sample), cmp_sample);
  return PP_OK;
}

/* ---- bracket: src/cost_model.cpp:46-53 ----------------------------------- */
static void bracket(const int64_t* axis, int32_t size, double x, int32_t* seg_out, double* t_out) {
  if (size == 1) {
    *seg_out = 0;
    *t_out = 0.0;
    return;
  }
  int32_t seg = 0;
  while (seg + 2 < size && x >= (double)axis[seg + 1]) ++seg;
  const double x0 = (double)axis[seg];
  const double x1 = (double)axis[seg + 1];
  *seg_out = seg;
  *t_out = (x - x0) / (x1 - x0);
}

/* ---- ProfileGrid::per_layer: src/cost_model.cpp:126-150 ------------------ */
int orc_per_layer(const pp_grid_desc* g, int32_t kind, int32_t r, double mbs, double seqlen,
                  double out[3]) {
  int32_t mi, si;
  double tm, ts;
  bracket(g->mbs_axis, g->n_mbs, mbs, &mi, &tm);
  bracket(g->seq_axis, g->n_seq, seqlen, &si, &ts);
  const size_t per_table = (size_t)g->n_mbs * (size_t)g->n_seq;
  const size_t base = ((size_t)kind * 3 + (size_t)r) * per_table;
  /* corner(dm, ds): min(mi + dm, size - 1), cost_model.cpp:132-136 */
  const int32_t m0 = mi, m1 = (mi + 1 < g->n_mbs - 1) ? mi + 1 : g->n_mbs - 1;
  const int32_t s0 = si, s1 = (si + 1 < g->n_seq - 1) ? si + 1 : g->n_seq - 1;
  const double* a = g->cells + 3 * (base + (size_t)m0 * g->n_seq + s0); /* corner(0,0) */
  const double* b = g->cells + 3 * (base + (size_t)m1 * g->n_seq + s0); /* corner(1,0) */
  const double* c = g->cells + 3 * (base + (size_t)m0 * g->n_seq + s1); /* corner(0,1) */
  const double* d = g->cells + 3 * (base + (size_t)m1 * g->n_seq + s1); /* corner(1,1) */
  for (int f = 0; f < 3; ++f) {
    /* blend, cost_model.cpp:138-142; std::max(0.0, v) returns 0.0 unless 0.0 < v */
    const double lo = a[f] + tm * (b[f] - a[f]);
    const double hi = c[f] + tm * (d[f] - c[f]);
    const double v = lo + ts * (hi - lo);
    out[f] = (0.0 < v) ? v : 0.0;
  }
  return PP_OK;
}

/* ---- estimate: src/cost_model.cpp:294-319 -------------------------------- */
int orc_estimate(const pp_grid_desc* g, const pp_model_desc* m, int32_t stage, int64_t mbs,
                 int64_t max_in, int64_t max_tgt, double out[3]) {
  if (stage < 0 || stage >= m->n_stages) return PP_ERR_OUT_OF_RANGE;
  if (mbs < 1) return PP_ERR_INVALID;
  const int32_t enc = m->encoder_layers[stage];
  const int32_t dec = m->decoder_layers[stage];
  const double decoder_len = (double)(m->is_encoder_decoder ? max_tgt : max_in);
  double est[3] = {0.0, 0.0, 0.0};
  double c[3];
  if (enc > 0) {
    orc_per_layer(g, 0, m->recompute, (double)mbs, (double)max_in, c);
    for (int f = 0; f < 3; ++f) est[f] += enc * c[f]; /* int * double -> double */
  }
  if (dec > 0) {
    orc_per_layer(g, 1, m->recompute, (double)mbs, decoder_len, c);
    for (int f = 0; f < 3; ++f) est[f] += dec * c[f];
  }
  memcpy(out, est, sizeof(est));
  return PP_OK;
}

/* ---- make_slice_cost lambda: src/microbatch.cpp:136-158 ------------------- */
static void slice_cost_shape(const pp_grid_desc* g, const pp_model_desc* m, int64_t mbs,
                             int64_t in, int64_t tgt, double* time, double* act) {
  double t = 0.0, a = 0.0, est[3];
  for (int32_t j = 0; j < m->n_stages; ++j) {
    orc_estimate(g, m, j, mbs, in, tgt, est);
    const double tt = est[0] + est[1];
    t = (t < tt) ? tt : t; /* std::max(cost.time, ...) keeps the first on ties */
    a = (a < est[2]) ? est[2] : a;
  }
  *time = t;
  *act = a;
}

int orc_slice_cost(const pp_grid_desc* g, const pp_model_desc* m, const pp_sample* ordered,
                   int64_t begin, int64_t end, double* time, double* act_mem) {
  int64_t in = 0, tgt = 0; /* shape.input_len = 0, target_len = 0 (:143-144) */
  for (int64_t k = begin; k < end; ++k) {
    if (ordered[k].input_len > in) in = ordered[k].input_len;
    if (ordered[k].target_len > tgt) tgt = ordered[k].target_len;
  }
  if (end - begin < 1) return PP_ERR_INVALID;
  slice_cost_shape(g, m, end - begin, in, tgt, time, act_mem);
  return PP_OK;
}

/* ---- eval_objective: src/microbatch.cpp:109-120 -------------------------- */
int orc_eval_objective(const double* times, int64_t m, int32_t c, int32_t d, double* out) {
  if (m <= 0) return PP_ERR_INVALID;
  if (c < 1 || d < 1) return PP_ERR_INVALID;
  double max_t = 0.0, sum = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    max_t = (max_t < times[i]) ? times[i] : max_t;
    sum += times[i];
  }
  *out = (double)(c - 1) * max_t + sum / (double)d;
  return PP_OK;
}

/* ---- run_suffix_dp: src/microbatch.cpp:162-189 --------------------------- */
typedef struct {
  double sum;
  int32_t count;
} suffix_state;

static int run_suffix_dp(int64_t n, const double* T, const double* M, const int64_t* row_off,
                         double t_max, double cap, suffix_state* st) {
  for (int64_t k = 0; k <= n; ++k) {
    st[k].sum = INFINITY;
    st[k].count = 0;
  }
  st[n].sum = 0.0;
  st[n].count = 0;
  for (int64_t i = n - 1; i >= 0; --i) {
    suffix_state best = {INFINITY, 0};
    for (int64_t j = i + 1; j <= n; ++j) {
      const int64_t idx = row_off[i] + (j - i - 1);
      if (M[idx] > cap || T[idx] > t_max) continue;
      if (!isfinite(st[j].sum)) continue;
      const double sum = T[idx] + st[j].sum;
      const int32_t cnt = 1 + st[j].count;
      if (sum < best.sum || (sum == best.sum && cnt < best.count)) {
        best.sum = sum;
        best.count = cnt;
      }
    }
    st[i] = best;
  }
  return isfinite(st[0].sum);
}

/* ---- reconstruct_splits: src/microbatch.cpp:194-215 ---------------------- */
static int64_t reconstruct(int64_t n, const double* T, const double* M, const int64_t* row_off,
                           double t_max, double cap, const suffix_state* st, int32_t* splits) {
  int64_t m = 0, i = 0;
  while (i < n) {
    for (int64_t j = i + 1; j <= n; ++j) {
      const int64_t idx = row_off[i] + (j - i - 1);
      if (M[idx] > cap || T[idx] > t_max) continue;
      if (!isfinite(st[j].sum)) continue;
      if (T[idx] + st[j].sum == st[i].sum && 1 + st[j].count == st[i].count) {
        splits[m++] = (int32_t)j;
        i = j;
        break;
      }
    }
  }
  return m;
}

static int cmp_double(const void* pa, const void* pb) {
  const double a = *(const double*)pa, b = *(const double*)pb;
  return (a < b) ? -1 : (b < a) ? 1 : 0;
}

/* lexicographic std::vector<size_t> operator< */
static int splits_less(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {
  const int64_t k = na < nb ? na : nb;
  for (int64_t i = 0; i < k; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return na < nb;
}

/* ---- dp_partition: src/microbatch.cpp:219-350 (tables given) -------------- */
int orc_dp_tables(const double* T, const double* M, int64_t n, const pp_dp_options* o,
                  int32_t* splits_out, double* mb_times, int32_t* count_out,
                  double* t_max_used, double* objective, int64_t* err_index,
                  int64_t* n_candidates, int64_t* n_evaluated) {
  if (n <= 0) return PP_ERR_INVALID;                                   /* :222 */
  if (o->stage_count < 1 || o->replica_count < 1) return PP_ERR_INVALID; /* :223-224 */
  if (o->t_max_interval < 0) return PP_ERR_INVALID;                    /* :225-226 */
  int64_t* row_off = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    row_off[i] = total;
    total += n - i;
  }
  const double cap = o->per_mb_mem_cap;
  for (int64_t k = 0; k < n; ++k) { /* singleton check, :245-251 */
    if (M[row_off[k]] > cap) {
      if (err_index) *err_index = k;
      free(row_off);
      return PP_ERR_INFEASIBLE_SAMPLE;
    }
  }
  /* candidate set, :253-269 */
  double* cand;
  int64_t nc = 0;
  if (o->stage_count == 1) {
    cand = (double*)malloc(sizeof(double));
    cand[nc++] = INFINITY;
  } else {
    cand = (double*)malloc((size_t)total * sizeof(double));
    for (int64_t idx = 0; idx < total; ++idx) {
      if (M[idx] > cap) continue;
      double t = T[idx];
      if (o->t_max_interval > 0) t = ceil(t / o->t_max_interval) * o->t_max_interval;
      /* std::sort leaves the order of -0.0 and +0.0 unspecified, so which zero
       * std::unique keeps is too; the checker (and the device) keep +0.0. */
      if (t == 0.0) t = 0.0;
      cand[nc++] = t;
    }
    qsort(cand, (size_t)nc, sizeof(double), cmp_double);
    int64_t u = 0; /* std::unique with operator== */
    for (int64_t k = 0; k < nc; ++k)
      if (u == 0 || !(cand[u - 1] == cand[k])) cand[u++] = cand[k];
    nc = u;
  }
  if (n_candidates) *n_candidates = nc;
  suffix_state* st = (suffix_state*)malloc((size_t)(n + 1) * sizeof(suffix_state));
  double min_sum_bound = 0.0; /* :274-279 */
  int64_t evaluated = 0;
  if (o->stage_count > 1) {
    run_suffix_dp(n, T, M, row_off, INFINITY, cap, st);
    min_sum_bound = st[0].sum / (double)o->replica_count;
  }
  /* candidate loop, :281-318 */
  double best_obj = INFINITY, best_t = 0.0;
  int32_t best_count = 0;
  int valid = 0;
  int32_t* best_splits = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int32_t* tmp = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int64_t best_m = 0;
  const double ramp = (double)(o->stage_count - 1);
  for (int64_t ci = 0; ci < nc; ++ci) {
    const double t_max = cand[ci];
    if (valid && ramp * t_max + min_sum_bound > best_obj) break;
    ++evaluated;
    if (!run_suffix_dp(n, T, M, row_off, t_max, cap, st)) continue;
    const double obj = (o->stage_count > 1 ? ramp * t_max : 0.0) +
                       st[0].sum / (double)o->replica_count;
    int take = 0;
    if (!valid || obj < best_obj) {
      take = 1;
    } else if (obj == best_obj) {
      if (st[0].count < best_count) {
        take = 1;
      } else if (st[0].count == best_count) {
        const int64_t m = reconstruct(n, T, M, row_off, t_max, cap, st, tmp);
        if (splits_less(tmp, m, best_splits, best_m)) {
          memcpy(best_splits, tmp, (size_t)m * sizeof(int32_t));
          best_m = m;
          best_t = t_max;
          continue;
        }
      }
    }
    if (take) {
      best_obj = obj;
      best_count = st[0].count;
      best_m = reconstruct(n, T, M, row_off, t_max, cap, st, best_splits);
      best_t = t_max;
      valid = 1;
    }
  }
  if (n_evaluated) *n_evaluated = evaluated;
  int rc = PP_OK;
  if (!valid) {
    rc = PP_ERR_INFEASIBLE; /* :319-320 */
    if (err_index) *err_index = -1;
  } else {
    /* assembly, :322-335 */
    int64_t begin = 0;
    double realized_max = 0.0;
    for (int64_t k = 0; k < best_m; ++k) {
      const int64_t split = best_splits[k];
      const double t = T[row_off[begin] + (split - begin - 1)];
      mb_times[k] = t;
      splits_out[k] = (int32_t)split;
      realized_max = (realized_max < t) ? t : realized_max;
      begin = split;
    }
    *count_out = (int32_t)best_m;
    orc_eval_objective(mb_times, best_m, o->stage_count, o->replica_count, objective);
    *t_max_used = isfinite(best_t) ? best_t : realized_max;
  }
  free(row_off);
  free(cand);
  free(st);
  free(best_splits);
  free(tmp);
  return rc;
}

/* ---- the production path: order -> make_slice_cost -> dp_partition -------- */
int orc_plan_grid(const pp_sample* samples, int64_t n, int32_t presorted, const pp_grid_desc* g,
                  const pp_model_desc* m, const pp_dp_options* o, pp_sample* ordered,
                  int32_t* splits, double* mb_times, int32_t* count, double* t_max_used,
                  double* objective, int64_t* err_sample_id, int64_t* n_candidates,
                  int64_t* n_evaluated) {
  if (n <= 0) return PP_ERR_INVALID;
  if (presorted)
    memcpy(ordered, samples, (size_t)n * sizeof(pp_sample));
  else
    orc_order_samples(samples, n, ordered);
  const int64_t total = n * (n + 1) / 2;
  double* T = (double*)malloc((size_t)total * sizeof(double));
  double* M = (double*)malloc((size_t)total * sizeof(double));
  if (!T || !M) {
    free(T);
    free(M);
    return PP_ERR_INVALID;
  }
  /* table build, microbatch.cpp:228-243; the padded max over [i, j) is kept
   * as a running max along the row (identical value, O(1) per slice). */
  int64_t idx = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t in = 0, tgt = 0;
    for (int64_t j = i + 1; j <= n; ++j) {
      if (ordered[j - 1].input_len > in) in = ordered[j - 1].input_len;
      if (ordered[j - 1].target_len > tgt) tgt = ordered[j - 1].target_len;
      slice_cost_shape(g, m, j - i, in, tgt, &T[idx], &M[idx]);
      ++idx;
    }
  }
  int64_t err_index = -1;
  const int rc = orc_dp_tables(T, M, n, o, splits, mb_times, count, t_max_used, objective,
                               &err_index, n_candidates, n_evaluated);
  if (rc == PP_ERR_INFEASIBLE_SAMPLE && err_sample_id) *err_sample_id = ordered[err_index].id;
  if (rc == PP_ERR_INFEASIBLE && err_sample_id) *err_sample_id = -1;
  free(T);
  free(M);
  return rc;
}

/* Largest slice time over memory-feasible slices (!(M > cap)) and the largest
 * singleton act_mem: the two quantities the K -> t_max_interval mapping of the
 * benchmark configs needs (mapping A').  Running maxima along
 * each row give the same padded shape as microbatch.cpp:145-148. */
int orc_slice_extrema(const pp_sample* ordered, int64_t n, const pp_grid_desc* g,
                      const pp_model_desc* m, double cap, double* t_capmax, double* single_act_max) {
  double best = -INFINITY, sa = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    int64_t in = 0, tgt = 0;
    for (int64_t j = i + 1; j <= n; ++j) {
      if (ordered[j - 1].input_len > in) in = ordered[j - 1].input_len;
      if (ordered[j - 1].target_len > tgt) tgt = ordered[j - 1].target_len;
      double t, a;
      slice_cost_shape(g, m, j - i, in, tgt, &t, &a);
      if (j == i + 1 && sa < a) sa = a;
      if (!(a > cap) && best < t) best = t;
    }
  }
  *t_capmax = best;
  *single_act_max = sa;
  return PP_OK;
}
