/* pp_stream.c — STREAMING restatement of the reference planner's hot path
 * (order_samples(Sort) -> make_slice_cost -> dp_partition), for mini-batches
 * whose triangular tables do not fit in memory (BASELINE config C5: n = 65,536,
 * 2 x 2.1 G slices = 34 GB of tables in the reference).
 *
 * TEST INFRASTRUCTURE ONLY (see pp_oracle.h): the checker that pins the
 * device path at C5 scale.  Same arithmetic as pp_oracle.c (which is pinned
 * against the unmodified reference); what changes is only WHEN a slice is
 * priced — on the fly, inside each sweep, instead of once into the tables of
 * microbatch.cpp:228-243:
 *
 *   * slice [i, j) is priced from its padded shape (j - i, max in[i..j),
 *     max tgt[i..j)) (microbatch.cpp:141-148); the two maxima come from a
 *     sparse range-max table (the max of a set is exact, any evaluation order);
 *   * estimate() (cost_model.cpp:294-319) runs once per DISTINCT stage layout:
 *     stages with equal (encoder, decoder) layer counts yield equal values and
 *     max() over equal values returns that value (microbatch.cpp:149-155);
 *   * bracket() (cost_model.cpp:46-53) is a pure function of its argument, so
 *     it is evaluated once per micro-batch size and once per length value;
 *   * the candidate set (microbatch.cpp:253-269) is collected with a hash set
 *     instead of a vector + sort + unique (same set, then sorted ascending);
 *   * candidates below t* = min over partitions of the max slice time are not
 *     run: run_suffix_dp(t) is feasible iff some partition keeps every slice
 *     <= t (and under the cap), i.e. iff t >= t*, so the reference's loop only
 *     `continue`s there (microbatch.cpp:292).  They still count in n_evaluated
 *     exactly as the reference's loop visits them.  t* comes from one minimax
 *     sweep fused with the bound pass (microbatch.cpp:274-279).
 *   * each DP row's scan over j (microbatch.cpp:177-185) is split across
 *     threads into contiguous j ranges whose partial (sum, count, first j)
 *     minima are combined in ascending range order with the reference's
 *     strict-improvement rule — the same winner as the sequential scan
 *     (every candidate sum is one rounded add, independent of the order).
 *
 * Pinned: tests/test_oracle.py compares it with the unmodified reference
 * (oracle/_ref) and with pp_oracle.c for n <= 2048 (GPT / T5, capped and
 * uncapped, I in {0, 5, 1e3}); tests/golden/c5.json was generated with it.
 */
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "pp_oracle.h"

typedef struct {
  double t;
  int32_t seg;
} axpos;

/* bracket: src/cost_model.cpp:46-53 */
static axpos bracket_pos(const int64_t* axis, int32_t size, double x) {
  axpos p;
  if (size == 1) {
    p.seg = 0;
    p.t = 0.0;
    return p;
  }
  int32_t seg = 0;
  while (seg + 2 < size && x >= (double)axis[seg + 1]) ++seg;
  const double x0 = (double)axis[seg];
  const double x1 = (double)axis[seg + 1];
  p.seg = seg;
  p.t = (x - x0) / (x1 - x0);
  return p;
}

/* ProfileGrid::per_layer with pre-bracketed axes: src/cost_model.cpp:126-150 */
static void per_layer_at(const pp_grid_desc* g, int32_t kind, int32_t r, axpos pm, axpos ps,
                         double out[3]) {
  const size_t per_table = (size_t)g->n_mbs * (size_t)g->n_seq;
  const size_t base = ((size_t)kind * 3 + (size_t)r) * per_table;
  const int32_t m0 = pm.seg, m1 = (pm.seg + 1 < g->n_mbs - 1) ? pm.seg + 1 : g->n_mbs - 1;
  const int32_t s0 = ps.seg, s1 = (ps.seg + 1 < g->n_seq - 1) ? ps.seg + 1 : g->n_seq - 1;
  const double* a = g->cells + 3 * (base + (size_t)m0 * g->n_seq + s0);
  const double* b = g->cells + 3 * (base + (size_t)m1 * g->n_seq + s0);
  const double* c = g->cells + 3 * (base + (size_t)m0 * g->n_seq + s1);
  const double* d = g->cells + 3 * (base + (size_t)m1 * g->n_seq + s1);
  const double tm = pm.t, ts = ps.t;
  for (int f = 0; f < 3; ++f) {
    const double lo = a[f] + tm * (b[f] - a[f]);
    const double hi = c[f] + tm * (d[f] - c[f]);
    const double v = lo + ts * (hi - lo);
    out[f] = (0.0 < v) ? v : 0.0;
  }
}

typedef struct {
  /* inputs */
  const pp_grid_desc* g;
  int32_t recompute, encdec;
  int32_t n_lay;
  int32_t lay_enc[64], lay_dec[64];
  int64_t n;
  const pp_sample* o; /* ordered */
  /* caches */
  axpos* mbs_pos;     /* [n + 1] bracket of double(mbs) */
  axpos* len_pos;     /* [max_len + 1] bracket of double(len) */
  int64_t max_len;
  int32_t levels;
  int64_t** rin;      /* sparse range-max tables of input / target lengths */
  int64_t** rtg;
} coster;

static int64_t range_max(int64_t* const* tab, int64_t lo, int64_t hi /* exclusive */) {
  const int64_t len = hi - lo;
  int k = 63 - __builtin_clzll((unsigned long long)len);
  const int64_t a = tab[k][lo], b = tab[k][hi - (1LL << k)];
  return a > b ? a : b;
}

/* make_slice_cost lambda (microbatch.cpp:136-158) over estimate
 * (cost_model.cpp:294-319): time = max over stages of t_f + t_b, act_mem =
 * max of act, from 0.0; padded lengths start at 0 (:143-144). */
static void slice_cost(const coster* k, int64_t i, int64_t j, double* time, double* act) {
  int64_t in = range_max(k->rin, i, j), tgt = range_max(k->rtg, i, j);
  if (in < 0) in = 0;
  if (tgt < 0) tgt = 0;
  const axpos pm = k->mbs_pos[j - i];
  const axpos pin = k->len_pos[in];
  const axpos pdec = k->len_pos[k->encdec ? tgt : in];
  double t = 0.0, a = 0.0;
  for (int l = 0; l < k->n_lay; ++l) {
    double est[3] = {0.0, 0.0, 0.0}, c[3];
    if (k->lay_enc[l] > 0) {
      per_layer_at(k->g, 0, k->recompute, pm, pin, c);
      for (int f = 0; f < 3; ++f) est[f] += k->lay_enc[l] * c[f];
    }
    if (k->lay_dec[l] > 0) {
      per_layer_at(k->g, 1, k->recompute, pm, pdec, c);
      for (int f = 0; f < 3; ++f) est[f] += k->lay_dec[l] * c[f];
    }
    const double tt = est[0] + est[1];
    t = (t < tt) ? tt : t;
    a = (a < est[2]) ? est[2] : a;
  }
  *time = t;
  *act = a;
}

static int coster_init(coster* k, const pp_grid_desc* g, const pp_model_desc* m, const pp_sample* o,
                       int64_t n) {
  memset(k, 0, sizeof(*k));
  k->g = g;
  k->recompute = m->recompute;
  k->encdec = m->is_encoder_decoder;
  k->n = n;
  k->o = o;
  for (int32_t s = 0; s < m->n_stages; ++s) {
    const int32_t e = m->encoder_layers[s], d = m->decoder_layers[s];
    int seen = 0;
    for (int l = 0; l < k->n_lay; ++l) seen |= (k->lay_enc[l] == e && k->lay_dec[l] == d);
    if (!seen) {
      if (k->n_lay == 64) return PP_ERR_INVALID;
      k->lay_enc[k->n_lay] = e;
      k->lay_dec[k->n_lay] = d;
      k->n_lay++;
    }
  }
  k->mbs_pos = (axpos*)malloc((size_t)(n + 1) * sizeof(axpos));
  for (int64_t d = 1; d <= n; ++d) k->mbs_pos[d] = bracket_pos(g->mbs_axis, g->n_mbs, (double)d);
  int64_t mx = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (o[i].input_len > mx) mx = o[i].input_len;
    if (o[i].target_len > mx) mx = o[i].target_len;
  }
  k->max_len = mx;
  k->len_pos = (axpos*)malloc((size_t)(mx + 1) * sizeof(axpos));
  for (int64_t v = 0; v <= mx; ++v) k->len_pos[v] = bracket_pos(g->seq_axis, g->n_seq, (double)v);
  int levels = 1;
  while ((1LL << levels) <= n) ++levels;
  k->levels = levels;
  k->rin = (int64_t**)malloc(sizeof(int64_t*) * levels);
  k->rtg = (int64_t**)malloc(sizeof(int64_t*) * levels);
  for (int L = 0; L < levels; ++L) {
    k->rin[L] = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    k->rtg[L] = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  }
  for (int64_t i = 0; i < n; ++i) {
    k->rin[0][i] = o[i].input_len;
    k->rtg[0][i] = o[i].target_len;
  }
  for (int L = 1; L < levels; ++L)
    for (int64_t i = 0; i + (1LL << L) <= n; ++i) {
      const int64_t h = 1LL << (L - 1);
      k->rin[L][i] = k->rin[L - 1][i] > k->rin[L - 1][i + h] ? k->rin[L - 1][i] : k->rin[L - 1][i + h];
      k->rtg[L][i] = k->rtg[L - 1][i] > k->rtg[L - 1][i + h] ? k->rtg[L - 1][i] : k->rtg[L - 1][i + h];
    }
  return PP_OK;
}

static void coster_free(coster* k) {
  free(k->mbs_pos);
  free(k->len_pos);
  for (int L = 0; L < k->levels; ++L) {
    free(k->rin[L]);
    free(k->rtg[L]);
  }
  free(k->rin);
  free(k->rtg);
}

/* ---- open-addressing set of doubles (bit patterns) ----------------------- */
typedef struct {
  uint64_t* keys;
  int64_t cap, count;
} dset;
#define DSET_EMPTY 0xfff8dead00000001ULL /* a NaN payload no candidate can have */

static void dset_init(dset* s, int64_t cap) {
  s->cap = cap;
  s->count = 0;
  s->keys = (uint64_t*)malloc((size_t)cap * sizeof(uint64_t));
  for (int64_t k = 0; k < cap; ++k) s->keys[k] = DSET_EMPTY;
}
static void dset_add(dset* s, double v);
static void dset_grow(dset* s) {
  dset t;
  dset_init(&t, s->cap * 2);
  for (int64_t k = 0; k < s->cap; ++k)
    if (s->keys[k] != DSET_EMPTY) {
      double v;
      memcpy(&v, &s->keys[k], 8);
      dset_add(&t, v);
    }
  free(s->keys);
  *s = t;
}
static void dset_add(dset* s, double v) {
  uint64_t u;
  memcpy(&u, &v, 8);
  uint64_t h = u * 0x9e3779b97f4a7c15ULL;
  int64_t p = (int64_t)(h >> 17) & (s->cap - 1);
  while (s->keys[p] != DSET_EMPTY) {
    if (s->keys[p] == u) return;
    p = (p + 1) & (s->cap - 1);
  }
  s->keys[p] = u;
  if (++s->count * 2 > s->cap) dset_grow(s);
}

static int cmp_dbl(const void* pa, const void* pb) {
  const double a = *(const double*)pa, b = *(const double*)pb;
  return (a < b) ? -1 : (b < a) ? 1 : 0;
}

/* ---- one DP sweep ---------------------------------------------------------
 * mode 0: run_suffix_dp(t_max) (microbatch.cpp:162-189), state (sum, count)
 * mode 1: bound pass (t = +inf, the sums) fused with the minimax t*:
 *         mm[i] = min over feasible j of max(T[i,j], mm[j]).
 * Returns state[0].sum finite. */
typedef struct {
  double sum;
  int32_t count;
} sstate;

typedef struct {
  double s;
  int32_t c;
  double m;
} part;

static int sweep(const coster* k, int mode, double t_max, double cap, sstate* st, double* mm,
                 int threads) {
  const int64_t n = k->n;
  for (int64_t q = 0; q <= n; ++q) {
    st[q].sum = INFINITY;
    st[q].count = 0;
    if (mm) mm[q] = INFINITY;
  }
  st[n].sum = 0.0;
  st[n].count = 0;
  if (mm) mm[n] = -INFINITY;
  part* parts = (part*)malloc(sizeof(part) * (size_t)threads);
#pragma omp parallel num_threads(threads)
  {
    const int tid = omp_get_thread_num();
    const int nt = omp_get_num_threads();
    for (int64_t i = n - 1; i >= 0; --i) {
      const int64_t span = n - i;  /* j in (i, n] */
      const int64_t per = (span + nt - 1) / nt;
      const int64_t j0 = i + 1 + (int64_t)tid * per;
      const int64_t j1 = (j0 + per - 1 < n) ? j0 + per - 1 : n;
      part p = {INFINITY, 0, INFINITY};
      for (int64_t j = j0; j <= j1; ++j) {
        double T, M;
        slice_cost(k, i, j, &T, &M);
        if (M > cap || T > t_max) continue; /* :179 */
        if (!isfinite(st[j].sum)) continue;  /* :180 */
        const double sum = T + st[j].sum;    /* :182 */
        const int32_t cnt = 1 + st[j].count;
        if (sum < p.s || (sum == p.s && cnt < p.c)) { /* :184 */
          p.s = sum;
          p.c = cnt;
        }
        if (mode == 1) {
          const double v = (T < mm[j]) ? mm[j] : T;
          p.m = (v < p.m) ? v : p.m;
        }
      }
      parts[tid] = p;
#pragma omp barrier
#pragma omp single
      {
        part b = {INFINITY, 0, INFINITY};
        for (int q = 0; q < nt; ++q) { /* ascending j ranges: first minimum wins */
          if (parts[q].s < b.s || (parts[q].s == b.s && parts[q].c < b.c)) {
            b.s = parts[q].s;
            b.c = parts[q].c;
          }
          b.m = (parts[q].m < b.m) ? parts[q].m : b.m;
        }
        st[i].sum = b.s;
        st[i].count = b.c;
        if (mode == 1) mm[i] = b.m;
      } /* implicit barrier */
    }
  }
  free(parts);
  return isfinite(st[0].sum);
}

/* reconstruct_splits (microbatch.cpp:194-215), front to back */
static int64_t reconstruct(const coster* k, double t_max, double cap, const sstate* st, int32_t* splits) {
  const int64_t n = k->n;
  int64_t m = 0, i = 0;
  while (i < n) {
    int64_t nx = -1;
    for (int64_t j = i + 1; j <= n; ++j) {
      double T, M;
      slice_cost(k, i, j, &T, &M);
      if (M > cap || T > t_max) continue;
      if (!isfinite(st[j].sum)) continue;
      if (T + st[j].sum == st[i].sum && 1 + st[j].count == st[i].count) {
        nx = j;
        break;
      }
    }
    if (nx < 0) return -1; /* cannot happen for a feasible state */
    splits[m++] = (int32_t)nx;
    i = nx;
  }
  return m;
}

static int splits_less(const int32_t* a, int64_t na, const int32_t* b, int64_t nb) {
  const int64_t q = na < nb ? na : nb;
  for (int64_t i = 0; i < q; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return na < nb;
}

int orc_plan_grid_stream(const pp_sample* samples, int64_t n, int32_t presorted, const pp_grid_desc* g,
                         const pp_model_desc* m, const pp_dp_options* o, int32_t threads,
                         pp_sample* ordered, int32_t* splits_out, double* mb_times, int32_t* count_out,
                         double* t_max_used, double* objective, int64_t* err_sample_id,
                         int64_t* n_candidates, int64_t* n_evaluated) {
  if (n <= 0) return PP_ERR_INVALID;                                     /* :222 */
  if (o->stage_count < 1 || o->replica_count < 1) return PP_ERR_INVALID; /* :223-224 */
  if (o->t_max_interval < 0) return PP_ERR_INVALID;                      /* :225-226 */
  if (threads < 1) threads = 1;
  if (presorted)
    memcpy(ordered, samples, (size_t)n * sizeof(pp_sample));
  else
    orc_order_samples(samples, n, ordered);
  coster k;
  if (coster_init(&k, g, m, ordered, n) != PP_OK) return PP_ERR_INVALID;
  const double cap = o->per_mb_mem_cap;
  /* singleton check, :245-251 */
  for (int64_t q = 0; q < n; ++q) {
    double T, M;
    slice_cost(&k, q, q + 1, &T, &M);
    if (M > cap) {
      if (err_sample_id) *err_sample_id = ordered[q].id;
      coster_free(&k);
      return PP_ERR_INFEASIBLE_SAMPLE;
    }
  }
  /* candidate set, :253-269 */
  double* cand = NULL;
  int64_t nc = 0;
  const double I = o->t_max_interval;
  if (o->stage_count == 1) {
    cand = (double*)malloc(sizeof(double));
    cand[nc++] = INFINITY;
  } else {
    dset* sets = (dset*)malloc(sizeof(dset) * (size_t)threads);
#pragma omp parallel num_threads(threads)
    {
      const int tid = omp_get_thread_num();
      dset_init(&sets[tid], 1024);
#pragma omp for schedule(dynamic, 16)
      for (int64_t i = 0; i < n; ++i) {
        double last = NAN;
        for (int64_t j = i + 1; j <= n; ++j) {
          double T, M;
          slice_cost(&k, i, j, &T, &M);
          if (M > cap) continue;
          double t = T;
          if (I > 0) t = ceil(t / I) * I;
          if (t == 0.0) t = 0.0; /* (-0.0 and +0.0 are one value; keep +0.0, as pp_oracle.c) */
          if (t == last) continue; /* (a repeat of the previous value: already in the set) */
          last = t;
          dset_add(&sets[tid], t);
        }
      }
    }
    dset all;
    dset_init(&all, 1024);
    for (int q = 0; q < threads; ++q) {
      for (int64_t p = 0; p < sets[q].cap; ++p)
        if (sets[q].keys[p] != DSET_EMPTY) {
          double v;
          memcpy(&v, &sets[q].keys[p], 8);
          dset_add(&all, v);
        }
      free(sets[q].keys);
    }
    free(sets);
    cand = (double*)malloc((size_t)(all.count + 1) * sizeof(double));
    for (int64_t p = 0; p < all.cap; ++p)
      if (all.keys[p] != DSET_EMPTY) memcpy(&cand[nc++], &all.keys[p], 8);
    free(all.keys);
    qsort(cand, (size_t)nc, sizeof(double), cmp_dbl);
  }
  if (n_candidates) *n_candidates = nc;
  sstate* st = (sstate*)malloc((size_t)(n + 1) * sizeof(sstate));
  double* mm = (double*)malloc((size_t)(n + 1) * sizeof(double));
  double min_sum_bound = 0.0, tstar = -INFINITY;
  if (o->stage_count > 1) { /* bound pass :274-279, fused with the minimax t* */
    sweep(&k, 1, INFINITY, cap, st, mm, threads);
    min_sum_bound = st[0].sum / (double)o->replica_count;
    tstar = mm[0];
  }
  double best_obj = INFINITY, best_t = 0.0;
  int32_t best_count = 0;
  int valid = 0;
  int32_t* best_splits = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int32_t* tmp = (int32_t*)malloc((size_t)n * sizeof(int32_t));
  int64_t best_m = 0, evaluated = 0;
  const double ramp = (double)(o->stage_count - 1);
  for (int64_t ci = 0; ci < nc; ++ci) { /* candidate loop :281-318 */
    const double t_max = cand[ci];
    if (valid && ramp * t_max + min_sum_bound > best_obj) break; /* :291 */
    ++evaluated;
    if (t_max < tstar) continue; /* infeasible (see header): run_suffix_dp fails, :292 */
    if (!sweep(&k, 0, t_max, cap, st, NULL, threads)) continue;
    const double obj = (o->stage_count > 1 ? ramp * t_max : 0.0) + st[0].sum / (double)o->replica_count;
    int take = 0;
    if (!valid || obj < best_obj) {
      take = 1;
    } else if (obj == best_obj) {
      if (st[0].count < best_count) {
        take = 1;
      } else if (st[0].count == best_count) {
        const int64_t mm2 = reconstruct(&k, t_max, cap, st, tmp);
        if (splits_less(tmp, mm2, best_splits, best_m)) {
          memcpy(best_splits, tmp, (size_t)mm2 * sizeof(int32_t));
          best_m = mm2;
          best_t = t_max;
          continue;
        }
      }
    }
    if (take) {
      best_obj = obj;
      best_count = st[0].count;
      best_m = reconstruct(&k, t_max, cap, st, best_splits);
      best_t = t_max;
      valid = 1;
    }
  }
  if (n_evaluated) *n_evaluated = evaluated;
  int rc = PP_OK;
  if (!valid) {
    rc = PP_ERR_INFEASIBLE; /* :319-320 */
    if (err_sample_id) *err_sample_id = -1;
  } else { /* assembly :322-335 */
    int64_t begin = 0;
    double realized_max = 0.0;
    for (int64_t q = 0; q < best_m; ++q) {
      const int64_t split = best_splits[q];
      double T, M;
      slice_cost(&k, begin, split, &T, &M);
      mb_times[q] = T;
      splits_out[q] = (int32_t)split;
      realized_max = (realized_max < T) ? T : realized_max;
      begin = split;
    }
    *count_out = (int32_t)best_m;
    orc_eval_objective(mb_times, best_m, o->stage_count, o->replica_count, objective);
    *t_max_used = isfinite(best_t) ? best_t : realized_max;
  }
  free(cand);
  free(st);
  free(mm);
  free(best_splits);
  free(tmp);
  coster_free(&k);
  return rc;
}
