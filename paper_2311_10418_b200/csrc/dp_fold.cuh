// dp_fold.cuh — the DP's per-transition arithmetic (one row accumulator,
// the reference's lexicographic update rule), shared by dp.cu and the chain
// micro-benchmark (tools/chain_probe.cu).  run_suffix_dp's update
// (microbatch.cpp:176-186): take (T + S, 1 + C) when T <= t, M <= cap and
// it is lexicographically smaller, lowest j on ties.
#pragma once
#include <cuda_runtime.h>

namespace ppb {

// One row's running state: sum s, second value x (bound sum / minimax),
// count c and argmin j (CAND modes).
struct Acc {
  double s, x;
  int c, j;
};

__device__ __forceinline__ int shfl_i32(int v, int src) {
  int r;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v), "r"(src));
  return r;
}
__device__ __forceinline__ double shfl_f64(double v, int src) {
  int lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
  lo = shfl_i32(lo, src);
  hi = shfl_i32(hi, src);
  double r;
  asm("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
  return r;
}

// Lexicographic (sum, count) select of a descending-column fold: (hs, hc)
// <- (cs, cn) when pre and (cs < hs or cs == hs and cn <= hc); returns the
// decision.  Written in PTX so both compares of cs hang off the add in
// parallel and one predicate OR feeds the selects — ptxas otherwise chains
// the compares, pre and the count tie one after another behind the add,
// which is the chain warp's critical path (the triangle's state step).
__device__ __forceinline__ unsigned lex_select_desc(double cs, int cn, unsigned pre, double& hs, int& hc) {
  unsigned u;
  asm("{\n\t"
      ".reg .pred pp, pt, pl, pe;\n\t"
      "setp.ne.u32 pp, %5, 0;\n\t"
      "setp.le.and.s32 pt, %4, %2, pp;\n\t"
      "setp.lt.and.f64 pl, %3, %1, pp;\n\t"
      "setp.eq.and.f64 pe, %3, %1, pt;\n\t"
      "or.pred pl, pl, pe;\n\t"
      "selp.f64 %1, %3, %1, pl;\n\t"
      "selp.s32 %2, %4, %2, pl;\n\t"
      "selp.u32 %0, 1, 0, pl;\n\t"
      "}"
      : "=r"(u), "+d"(hs), "+r"(hc)
      : "d"(cs), "r"(cn), "r"(pre));
  return u;
}

// The DP transition of one tile entry into a row accumulator, for the mode's
// recurrences (microbatch.cpp:176-186; the bound pass :274-279).  `ss`, `sx`,
// `sc` are state[j]; DESC: columns arrive in descending j, so an equal
// (sum, count) takes the new (lower) j; otherwise ascending j keeps the old.
//   CAND (MODE 0 / 3): (x + S, 1 + C) when x <= t and it is lexicographically
//     smaller.  NaN entries (infeasible slices) and +inf states fail every
//     compare against the (+inf, 0) identity or any taken value.
//   MODE 3 also: bound sum min(x + B);  MODE 1: min sum and min over
//     max(x, M) (the minimax t*);  MODE 2: min sum.
// fold_c takes the count through j already incremented (cn = 1 + C): the
// DP state arrays store 1 + count, so the far-far loop adds nothing.
template <int MODE, bool DESC>
__device__ __forceinline__ void fold_c(Acc& a, double xv, double ss, double sx, int cn, int j, bool okb,
                                       double t) {
  constexpr bool CAND = MODE == 0 || MODE == 3;
  const double cs = __dadd_rn(xv, ss);
  if (CAND && DESC) {
    const unsigned pre = (okb & (xv <= t)) ? 1u : 0u;
    const unsigned u = lex_select_desc(cs, cn, pre, a.s, a.c);
    a.j = u ? j : a.j;
  } else if (CAND) {
    const bool tie = DESC ? (cn <= a.c) : (cn < a.c);
    const bool upd = okb & (xv <= t) & ((cs < a.s) | ((cs == a.s) & tie));
    a.s = upd ? cs : a.s;
    a.c = upd ? cn : a.c;
    a.j = upd ? j : a.j;
  } else {
    a.s = (okb & (cs < a.s)) ? cs : a.s;
  }
  if (MODE == 3) {
    const double cb = __dadd_rn(xv, sx);
    a.x = (okb & (cb < a.x)) ? cb : a.x;
  } else if (MODE == 1) {
    const double v = (xv < sx) ? sx : xv;
    a.x = (okb & (v < a.x)) ? v : a.x;
  }
}
template <int MODE, bool DESC>
__device__ __forceinline__ void fold(Acc& a, double xv, double ss, double sx, int sc, int j, bool okb,
                                     double t) {
  fold_c<MODE, DESC>(a, xv, ss, sx, 1 + sc, j, okb, t);
}

// Keyed form for the slice-table far-far loop: the state's count and column
// travel as one key ((1 + C) << 16 | j, dp.cu kKeyShift; n <= kKeyMaxN), so
// (sum, count) lexicographic order with lowest-j ties is (sum, key) order
// with a strict key compare in either column order, and a.c carries the key
// (a.j unused): one select fewer per transition.
template <int MODE>
__device__ __forceinline__ void fold_k(Acc& a, double xv, double ss, double sx, int key, double t) {
  const double cs = __dadd_rn(xv, ss);
  const bool upd = (xv <= t) & ((cs < a.s) | ((cs == a.s) & (key < a.c)));
  a.s = upd ? cs : a.s;
  a.c = upd ? key : a.c;
  if (MODE == 3) {
    const double cb = __dadd_rn(xv, sx);
    a.x = (cb < a.x) ? cb : a.x;
  }
}
template <int MODE>
__device__ __forceinline__ void combine_k(Acc& a, const Acc& o) {
  const bool tk = o.s < a.s || (o.s == a.s && o.c < a.c);
  a.s = tk ? o.s : a.s;
  a.c = tk ? o.c : a.c;
  if (MODE == 3) a.x = (o.x < a.x) ? o.x : a.x;
}

// (s, c, j) lexmin with lowest-j ties.
__device__ __forceinline__ bool better(double s1, int c1, int j1, double s0, int c0, int j0) {
  return s1 < s0 || (s1 == s0 && (c1 < c0 || (c1 == c0 && j1 < j0)));
}
// Combine two partial accumulators over disjoint column sets (associative).
template <int MODE>
__device__ __forceinline__ void combine(Acc& a, const Acc& o) {
  constexpr bool CAND = MODE == 0 || MODE == 3;
  if (CAND) {
    const bool tk = better(o.s, o.c, o.j, a.s, a.c, a.j);
    a.s = tk ? o.s : a.s;
    a.c = tk ? o.c : a.c;
    a.j = tk ? o.j : a.j;
  } else {
    a.s = (o.s < a.s) ? o.s : a.s;
  }
  if (MODE == 1 || MODE == 3) a.x = (o.x < a.x) ? o.x : a.x;
}

}  // namespace ppb
