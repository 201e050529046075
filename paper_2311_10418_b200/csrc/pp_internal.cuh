// pp_internal.cuh — device-side building blocks shared by the planner kernels.
//
// Bit-exactness contract: every FP64 operation on the
// slice-cost path is an explicit round-to-nearest intrinsic (__dadd_rn,
// __dsub_rn, __dmul_rn, __ddiv_rn) so nvcc can never contract a*b+c into a
// DFMA; the whole library is also built with --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pipeplan_b200.h"

namespace ppb {

constexpr int kWarp = 32;
constexpr int kMaxLayouts = 64;  // distinct (encoder, decoder) layer layouts

// One distinct stage layout; stages with equal layouts yield equal costs and
// max() over equal values is exact, so dedup is parity-safe
// (microbatch.cpp:150-155).
struct Layout {
  int32_t enc;
  int32_t dec;
};

// Profile grid restricted to the recompute strategy in use
// (ProfileGrid::per_layer, cost_model.cpp:126-150).
struct GridDev {
  int32_t n_mbs;
  int32_t n_seq;
  int32_t n_layouts;
  int32_t is_encdec;
  const double* mbs_ax;  // double(axis[k]) — the reference converts at :50-51
  const double* seq_ax;
  const double* cells;   // [kind 2][n_mbs][n_seq][3]
  const Layout* layouts; // [n_layouts]
};

// bracket(): linear segment scan + IEEE divide (cost_model.cpp:46-53).
__device__ __forceinline__ void bracket(const double* ax, int size, double x, int& seg,
                                        double& t) {
  if (size == 1) {
    seg = 0;
    t = 0.0;
    return;
  }
  int s = 0;
  while (s + 2 < size && x >= ax[s + 1]) ++s;
  const double x0 = ax[s];
  const double x1 = ax[s + 1];
  seg = s;
  t = __ddiv_rn(__dsub_rn(x, x0), __dsub_rn(x1, x0));
}

// blend + std::max(0.0, v) (cost_model.cpp:138-142).
__device__ __forceinline__ double blend(double tm, double ts, double c00, double c10, double c01,
                                        double c11) {
  const double lo = __dadd_rn(c00, __dmul_rn(tm, __dsub_rn(c10, c00)));
  const double hi = __dadd_rn(c01, __dmul_rn(tm, __dsub_rn(c11, c01)));
  const double v = __dadd_rn(lo, __dmul_rn(ts, __dsub_rn(hi, lo)));
  return (0.0 < v) ? v : 0.0;
}

struct Cell3 {
  double tf, tb, act;
};

// ProfileGrid::per_layer for one kind given pre-bracketed axes.
__device__ __forceinline__ Cell3 per_layer(const GridDev& g, int kind, int mi, double tm, int si,
                                           double ts) {
  const int m1 = min(mi + 1, g.n_mbs - 1);
  const int s1 = min(si + 1, g.n_seq - 1);
  const double* base = g.cells + (size_t)kind * g.n_mbs * g.n_seq * 3;
  const double* a = base + ((size_t)mi * g.n_seq + si) * 3;
  const double* b = base + ((size_t)m1 * g.n_seq + si) * 3;
  const double* c = base + ((size_t)mi * g.n_seq + s1) * 3;
  const double* d = base + ((size_t)m1 * g.n_seq + s1) * 3;
  Cell3 r;
  r.tf = blend(tm, ts, a[0], b[0], c[0], d[0]);
  r.tb = blend(tm, ts, a[1], b[1], c[1], d[1]);
  r.act = blend(tm, ts, a[2], b[2], c[2], d[2]);
  return r;
}

// The make_slice_cost lambda for a padded shape (microbatch.cpp:141-155 with
// estimate(), cost_model.cpp:294-319).  in_len / tgt_len are the padded
// maxima as doubles (already max(0, .)).
__device__ __forceinline__ void slice_cost(const GridDev& g, double mbs, double in_len,
                                           double tgt_len, double& time, double& act) {
  int mi, si_in, si_dec;
  double tm, ts_in, ts_dec;
  bracket(g.mbs_ax, g.n_mbs, mbs, mi, tm);
  bracket(g.seq_ax, g.n_seq, in_len, si_in, ts_in);
  const double dec_len = g.is_encdec ? tgt_len : in_len;
  if (g.is_encdec) {
    bracket(g.seq_ax, g.n_seq, dec_len, si_dec, ts_dec);
  } else {
    si_dec = si_in;
    ts_dec = ts_in;
  }
  double t_best = 0.0, a_best = 0.0;
  for (int l = 0; l < g.n_layouts; ++l) {
    const Layout lay = g.layouts[l];
    double ef = 0.0, eb = 0.0, ea = 0.0;
    if (lay.enc > 0) {
      const Cell3 c = per_layer(g, 0, mi, tm, si_in, ts_in);
      const double L = (double)lay.enc;
      ef = __dadd_rn(ef, __dmul_rn(L, c.tf));
      eb = __dadd_rn(eb, __dmul_rn(L, c.tb));
      ea = __dadd_rn(ea, __dmul_rn(L, c.act));
    }
    if (lay.dec > 0) {
      const Cell3 c = per_layer(g, 1, mi, tm, si_dec, ts_dec);
      const double L = (double)lay.dec;
      ef = __dadd_rn(ef, __dmul_rn(L, c.tf));
      eb = __dadd_rn(eb, __dmul_rn(L, c.tb));
      ea = __dadd_rn(ea, __dmul_rn(L, c.act));
    }
    const double tt = __dadd_rn(ef, eb);
    t_best = (t_best < tt) ? tt : t_best;
    a_best = (a_best < ea) ? ea : a_best;
  }
  time = t_best;
  act = a_best;
}

// Masked band entry for a slice excluded by the memory cap.  NaN makes every
// DP test `t <= t_max` false, exactly like the reference's `continue` at
// microbatch.cpp:179, and is never a candidate.
__device__ __forceinline__ double masked() { return __longlong_as_double(0x7ff8000000000000LL); }

// Order-preserving map of doubles to uint64 (for radix sort / atomics).
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u & 0x8000000000000000ULL) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long u = (k & 0x8000000000000000ULL) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)u);
}

// Per-segment statistics written by cost pass A.
struct SegStats {
  unsigned long long kmin;   // dkey of min finite candidate key
  unsigned long long kmax;   // dkey of max finite candidate key
  unsigned long long nraw;   // memory-feasible, non-NaN slices (candidate capacity)
  int err_row;               // lowest ordered index whose singleton violates the cap
  int flags;                 // bit0: +inf candidate, bit1: -inf candidate
  long long band;            // band entries of the segment
};

// One DP pass: (mini-batch, t_max candidate).
struct WorkItem {
  int seg;
  int cand;            // candidate index within the segment (-1: bound pass, t = +inf)
  long long next_off;  // offset of this item's next[] (rows) in the next buffer
  long long state_off; // offset of global state scratch (or -1: shared memory)
};

struct ItemResult {
  double sum0;
  int count0;
  int feasible;
  double aux;     // bound pass: minimax t*
};

struct SegDP {
  double bound;     // min_sum_bound (microbatch.cpp:278)
  double tstar;     // min over partitions of the max slice time (feasibility threshold)
  double best_obj;
  double best_t;
  int best_count;
  int valid;
  int done;
  int next_cand;    // next candidate index to evaluate
  int n_cand;
  int ref_evals;    // candidates the reference's loop runs (for stats)
  int pad[2];
};


__device__ __forceinline__ double item_t(const WorkItem& it, const double* cand,
                                         const int64_t* cand_off) {
  return it.cand < 0 ? __longlong_as_double(0x7ff0000000000000LL) : cand[cand_off[it.seg] + it.cand];
}

}  // namespace ppb
