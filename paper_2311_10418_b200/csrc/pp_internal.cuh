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
// Candidate bins k = ceil(T / I) < 32 * kSmallBmWords are marked directly by
// cost pass B into a per-segment bitmap (segment mode 3, capi.cu).
constexpr int kSmallBmWords = 8;

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

// One field (0 t_f, 1 t_b, 2 act_mem) of ProfileGrid::per_layer for one kind
// given pre-bracketed axes (cost_model.cpp:126-150).
__device__ __forceinline__ double per_layer_field(const GridDev& g, int kind, int mi, double tm,
                                                  int si, double ts, int f) {
  const int m1 = min(mi + 1, g.n_mbs - 1);
  const int s1 = min(si + 1, g.n_seq - 1);
  const double* base = g.cells + (size_t)kind * g.n_mbs * g.n_seq * 3 + f;
  const double c00 = base[((size_t)mi * g.n_seq + si) * 3];
  const double c10 = base[((size_t)m1 * g.n_seq + si) * 3];
  const double c01 = base[((size_t)mi * g.n_seq + s1) * 3];
  const double c11 = base[((size_t)m1 * g.n_seq + s1) * 3];
  return blend(tm, ts, c00, c10, c01, c11);
}

// Pre-bracketed query of one slice: mbs bracket (mi, tm), the encoder's
// sequence bracket (input length) and the decoder's (target length for
// encoder-decoder models, else the input length) — estimate(),
// cost_model.cpp:301-317.
struct Query {
  int mi, si_enc, si_dec;
  double tm, ts_enc, ts_dec;
};

// act_mem of the slice: max over distinct stage layouts of
// 0.0 + L_enc * act(enc) + L_dec * act(dec) (microbatch.cpp:154).
__device__ __forceinline__ double slice_mem(const GridDev& g, const Query& q) {
  double best = 0.0;
  for (int l = 0; l < g.n_layouts; ++l) {
    const Layout lay = g.layouts[l];
    double ea = 0.0;
    if (lay.enc > 0)
      ea = __dadd_rn(ea, __dmul_rn((double)lay.enc, per_layer_field(g, 0, q.mi, q.tm, q.si_enc, q.ts_enc, 2)));
    if (lay.dec > 0)
      ea = __dadd_rn(ea, __dmul_rn((double)lay.dec, per_layer_field(g, 1, q.mi, q.tm, q.si_dec, q.ts_dec, 2)));
    best = (best < ea) ? ea : best;
  }
  return best;
}

// time of the slice: max over layouts of (t_f + t_b) (microbatch.cpp:153).
__device__ __forceinline__ double slice_time(const GridDev& g, const Query& q) {
  double best = 0.0;
  for (int l = 0; l < g.n_layouts; ++l) {
    const Layout lay = g.layouts[l];
    double ef = 0.0, eb = 0.0;
    if (lay.enc > 0) {
      const double L = (double)lay.enc;
      ef = __dadd_rn(ef, __dmul_rn(L, per_layer_field(g, 0, q.mi, q.tm, q.si_enc, q.ts_enc, 0)));
      eb = __dadd_rn(eb, __dmul_rn(L, per_layer_field(g, 0, q.mi, q.tm, q.si_enc, q.ts_enc, 1)));
    }
    if (lay.dec > 0) {
      const double L = (double)lay.dec;
      ef = __dadd_rn(ef, __dmul_rn(L, per_layer_field(g, 1, q.mi, q.tm, q.si_dec, q.ts_dec, 0)));
      eb = __dadd_rn(eb, __dmul_rn(L, per_layer_field(g, 1, q.mi, q.tm, q.si_dec, q.ts_dec, 1)));
    }
    const double tt = __dadd_rn(ef, eb);
    best = (best < tt) ? tt : best;
  }
  return best;
}

// Rows per band tile (= rows per DP block).  The band of a segment is stored
// as one tile per block of 32 rows, top-down (block b holds rows
// [max(0, n-32(b+1)), n-32b)); tile column c holds the 32 rows' values for
// slice end j = i0 + c, contiguous (256 B per column).
constexpr int kRB = 32;

__device__ __forceinline__ int seg_of(const int* __restrict__ base, int n_seg, int g) {
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (base[mid] <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
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
  long long band;            // band entries of the segment (sum of 32 x W_b)
  int wmax;                  // max tile width W_b of the segment
  int pad;
  unsigned long long priced;   // slices priced by cost pass A
  unsigned long long priced_b; // band slices priced by cost pass B
};

// ---- TMA bulk copies + mbarriers (sm_90+ PTX, used on sm_100a) ----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completion reported on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Order prior generic-proxy accesses of shared memory before async-proxy (TMA) writes.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Named barrier for a subset of warps.
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// One DP pass: (mini-batch, t_max candidate).
struct WorkItem {
  int seg;
  int cand;            // candidate index within the segment (-1: bound pass, t = +inf)
  long long next_off;  // offset of this item's next[] (rows) in the next buffer
  long long state_off; // offset of global state scratch (or -1: shared memory)
  unsigned state_mask; // state index = j & mask (ring of mask+1 entries, or ~0u: no ring)
  int state_entries;   // entries per state array
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
