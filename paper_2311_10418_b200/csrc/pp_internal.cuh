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

#include <mutex>
#include <unordered_map>

namespace ppb {

// cudaFuncAttributeMaxDynamicSharedMemorySize is process-wide per (function,
// device) while contexts plan on many host threads at once (the reference's
// run_plan pool, driver.cpp:222-242): a thread that LOWERED the limit for its
// small launch would fail another thread's larger launch in flight with
// "invalid argument".  So the limit only ever rises, under a lock.
inline cudaError_t ensure_dyn_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> lim[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = lim[dev & 63][fn];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

constexpr int kWarp = 32;
constexpr int kMaxLayouts = 64;  // distinct (encoder, decoder) layer layouts
// Candidate bins k = ceil(T / I) < 32 * kSmallBmWords are marked directly by
// cost pass B into a per-segment bitmap (segment mode 3, capi.cu).
constexpr int kSmallBmWords = 16;

// One distinct stage layout as FP64 layer multiples (0 = kind absent).
// Stages with equal layouts yield equal costs and max() over equal values is
// exact, so dedup is parity-safe (microbatch.cpp:150-155).  The multiples are
// converted once on the host, so the slice loops issue no int->double
// conversions (those run on the narrow XU pipe).
struct Layout {
  int32_t enc;
  int32_t dec;
};
struct LayoutD {
  double le;
  double ld;
};

// Profile grid of ONE recompute strategy, prepared on the host (capi.cu
// upload_grid) for the cost kernels.  Per kind and cell (mi, si):
//   tt = {t_f, t_b, dt_f, dt_b},  am = {act, dact}
// where dX(mi, si) = X(min(mi+1, nm-1), si) - X(mi, si) is the mbs-direction
// difference the reference evaluates inside every blend
// (cost_model.cpp:138-142: c10 - c00 and c11 - c01).  It depends on the
// cells only, so computing it once (IEEE subtraction on the host) gives the
// same double the reference computes per query.
struct CostGrid {
  int32_t nm, ns;          // axis sizes
  int32_t n_lay;           // distinct stage layouts
  int32_t is_encdec;
  int32_t used;            // bit0: encoder kind priced, bit1: decoder kind priced
  int32_t lay_class;       // kLayGeneric / kLayDec1 / kLayEncDec2 (see slice_cost_lay)
  double le, ld;           // the class's encoder / decoder layer multiples
  const double* mbs_ax;    // double(axis[k]) — the reference converts at :50-51
  const double* seq_ax;
  const double4* tt;       // [2][nm][ns]
  const double2* am;       // [2][nm][ns]
  const LayoutD* lay;      // [n_lay]
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

// A pre-bracketed axis position: segment and interpolation weight.
struct AxisPos {
  double t;
  int32_t seg;
  int32_t pad;
};

// std::max(0.0, v) = (0.0 < v) ? v : 0.0 (NaN -> 0.0), as one compare and a
// select: left to itself nvcc lowers the ternary to DSETP.MAX plus NaN
// fix-ups (7 instructions).
__device__ __forceinline__ double clamp0(double v) {
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, 0d0000000000000000;\n\t"
      "selp.f64 %0, %1, 0d0000000000000000, p;\n\t}"
      : "=d"(r)
      : "d"(v));
  return r;
}

// blend + std::max(0.0, v) (cost_model.cpp:138-142) with the mbs-direction
// differences d0 = c10 - c00, d1 = c11 - c01 precomputed (see CostGrid).
__device__ __forceinline__ double blend_d(double tm, double ts, double c00, double d0, double c01,
                                          double d1) {
  const double lo = __dadd_rn(c00, __dmul_rn(tm, d0));
  const double hi = __dadd_rn(c01, __dmul_rn(tm, d1));
  const double v = __dadd_rn(lo, __dmul_rn(ts, __dsub_rn(hi, lo)));
  return clamp0(v);
}

// ProfileGrid::per_layer (cost_model.cpp:126-150) of one kind: corners
// (mi, si) and (mi, s1) carry the mbs-direction differences to (m1, .).
struct KindCost {
  double tf, tb, act;
};
template <bool TIME, bool MEM>
__device__ __forceinline__ KindCost kind_cost(const double4* __restrict__ tt,
                                              const double2* __restrict__ am, int ns, int mi,
                                              double tm, int si, double ts) {
  const int s1 = min(si + 1, ns - 1);
  const int i0 = mi * ns + si, i1 = mi * ns + s1;
  KindCost v;
  if (TIME) {
    const double4 a = tt[i0], b = tt[i1];
    v.tf = blend_d(tm, ts, a.x, a.z, b.x, b.z);
    v.tb = blend_d(tm, ts, a.y, a.w, b.y, b.w);
  }
  if (MEM) {
    const double2 a = am[i0], b = am[i1];
    v.act = blend_d(tm, ts, a.x, a.y, b.x, b.y);
  }
  return v;
}

// Slice cost (make_slice_cost lambda, microbatch.cpp:149-155 over estimate,
// cost_model.cpp:301-317): per distinct stage layout
//   est.X = 0.0 + L_enc * enc.X (+ L_dec * dec.X)
// then time = max over stages of t_f + t_b, act_mem = max of act, both from
// 0.0.  Every per_layer value is in [+0, +inf] (the clamp maps NaN to 0.0),
// so 0.0 + L * x == L * x bit for bit and the leading add is skipped.
template <bool TIME, bool MEM>
__device__ __forceinline__ void slice_cost(const double4* __restrict__ tt,
                                           const double2* __restrict__ am,
                                           const LayoutD* __restrict__ lay, int n_lay, int used,
                                           int nm, int ns, int mi, double tm, int se, double tse,
                                           int sd, double tsd, double& T, double& M) {
  KindCost E{0.0, 0.0, 0.0}, D{0.0, 0.0, 0.0};
  const int per = nm * ns;
  if (used & 1) E = kind_cost<TIME, MEM>(tt, am, ns, mi, tm, se, tse);
  if (used & 2) D = kind_cost<TIME, MEM>(tt + per, am + per, ns, mi, tm, sd, tsd);
  double bt = 0.0, bm = 0.0;
  for (int l = 0; l < n_lay; ++l) {
    const LayoutD L = lay[l];
    if (MEM) {
      double ea;
      if (L.le > 0.0) {
        ea = __dmul_rn(L.le, E.act);
        if (L.ld > 0.0) ea = __dadd_rn(ea, __dmul_rn(L.ld, D.act));
      } else {
        ea = __dmul_rn(L.ld, D.act);
      }
      bm = (bm < ea) ? ea : bm;
    }
    if (TIME) {
      double ef, eb;
      if (L.le > 0.0) {
        ef = __dmul_rn(L.le, E.tf);
        eb = __dmul_rn(L.le, E.tb);
        if (L.ld > 0.0) {
          ef = __dadd_rn(ef, __dmul_rn(L.ld, D.tf));
          eb = __dadd_rn(eb, __dmul_rn(L.ld, D.tb));
        }
      } else {
        ef = __dmul_rn(L.ld, D.tf);
        eb = __dmul_rn(L.ld, D.tb);
      }
      const double t = __dadd_rn(ef, eb);
      bt = (bt < t) ? t : bt;
    }
  }
  T = bt;
  M = bm;
}

// Stage-layout classes with a branch-free slice-cost path (capi.cu picks one
// per call; results are identical to slice_cost, max() over non-NaN values
// being order-free):
//   kLayGeneric  any layouts
//   kLayDec1     one layout, decoder layers only (decoder-only models: GPT)
//   kLayEncDec2  two layouts, one encoder-only and one decoder-only
//                (ModelConfig::uniform encoder-decoder split, T5)
constexpr int kLayGeneric = 0, kLayDec1 = 1, kLayEncDec2 = 2;

template <int LAY, bool TIME, bool MEM>
__device__ __forceinline__ void slice_cost_lay(const double4* __restrict__ tt,
                                               const double2* __restrict__ am,
                                               const LayoutD* __restrict__ lay, int n_lay, int used,
                                               int nm, int ns, int mi, double tm, int se, double tse,
                                               int sd, double tsd, double le, double ld, double& T,
                                               double& M) {
  if (LAY == kLayGeneric) {
    slice_cost<TIME, MEM>(tt, am, lay, n_lay, used, nm, ns, mi, tm, se, tse, sd, tsd, T, M);
    return;
  }
  const int per = nm * ns;
  const KindCost D = kind_cost<TIME, MEM>(tt + per, am + per, ns, mi, tm, sd, tsd);
  // per_layer values are in [+0, +inf] (clamped), so L * x and sums of them
  // are too (no NaN: L >= 1 is finite): max(0.0, .) of the first layout's
  // value is the value itself
  if (LAY == kLayDec1) {
    if (TIME) T = __dadd_rn(__dmul_rn(ld, D.tf), __dmul_rn(ld, D.tb));
    if (MEM) M = __dmul_rn(ld, D.act);
  } else {
    const KindCost E = kind_cost<TIME, MEM>(tt, am, ns, mi, tm, se, tse);
    if (TIME) {
      const double t1 = __dadd_rn(__dmul_rn(le, E.tf), __dmul_rn(le, E.tb));
      const double t2 = __dadd_rn(__dmul_rn(ld, D.tf), __dmul_rn(ld, D.tb));
      T = (t1 < t2) ? t2 : t1;
    }
    if (MEM) {
      const double a1 = __dmul_rn(le, E.act), a2 = __dmul_rn(ld, D.act);
      M = (a1 < a2) ? a2 : a1;
    }
  }
}

// Slice pricing of length-sorted single-input segments (GPT; band_run_kernel
// and the DP's in-kernel pricing, dp.cu): slice [i, j) pads to (d = j - i,
// in[j-1]), so its value depends on (d, length) only.  price_time is the
// make_slice_cost time (microbatch.cpp:149-155 over estimate,
// cost_model.cpp:301-317) with the operations of band3_kernel; price_slice
// also evaluates act_mem and returns NaN when it exceeds the cap (the
// reference's `continue` at microbatch.cpp:179).  Cells: per kind the
// CostGrid tt / am tables with row base mb.pad = mi * ns.
struct SlicePricer {
  const double4* tt_e;  // encoder kind (kLayEncDec2 only)
  const double4* tt_d;  // decoder kind
  const double2* am_e;
  const double2* am_d;
  int ns;
  double le, ld, cap;
  bool need_mem;
};

template <int LAY>
__device__ __forceinline__ double price_time(const SlicePricer& P, const AxisPos& mb, const AxisPos& pe) {
  const int s1 = min(pe.seg + 1, P.ns - 1);
  const double4 c0 = P.tt_d[mb.pad + pe.seg], c1 = P.tt_d[mb.pad + s1];
  const double df = blend_d(mb.t, pe.t, c0.x, c0.z, c1.x, c1.z);
  const double db = blend_d(mb.t, pe.t, c0.y, c0.w, c1.y, c1.w);
  const double t2 = __dadd_rn(__dmul_rn(P.ld, df), __dmul_rn(P.ld, db));
  if (LAY == kLayDec1) return t2;
  const double4 e0 = P.tt_e[mb.pad + pe.seg], e1 = P.tt_e[mb.pad + s1];
  const double ef = blend_d(mb.t, pe.t, e0.x, e0.z, e1.x, e1.z);
  const double eb = blend_d(mb.t, pe.t, e0.y, e0.w, e1.y, e1.w);
  const double t1 = __dadd_rn(__dmul_rn(P.le, ef), __dmul_rn(P.le, eb));
  return (t1 < t2) ? t2 : t1;
}

template <int LAY>
__device__ __forceinline__ double price_slice(const SlicePricer& P, const AxisPos& mb, const AxisPos& pe) {
  double T = price_time<LAY>(P, mb, pe);
  if (P.need_mem) {
    const int s1 = min(pe.seg + 1, P.ns - 1);
    const double2 c0 = P.am_d[mb.pad + pe.seg], c1 = P.am_d[mb.pad + s1];
    double M = __dmul_rn(P.ld, blend_d(mb.t, pe.t, c0.x, c0.y, c1.x, c1.y));
    if (LAY != kLayDec1) {
      const double2 e0 = P.am_e[mb.pad + pe.seg], e1 = P.am_e[mb.pad + s1];
      const double a1 = __dmul_rn(P.le, blend_d(mb.t, pe.t, e0.x, e0.y, e1.x, e1.y));
      M = (a1 < M) ? M : a1;
    }
    T = (M > P.cap) ? __longlong_as_double(0x7ff8000000000000LL) : T;
  }
  return T;
}

// In-kernel pricing inputs of the DP (dp.cu, PRICE != 0): the pricer's
// cells live in global memory here and are staged into shared memory by
// each DP CTA; per micro-batch size the mbs bracket, per ordered sample the
// sequence bracket of its input length and the length itself.
// PRICE / price_lay value of the shared-table path (gtab.cu): the DP's tiles
// come from the call's table G[length][d] instead of the band or in-kernel
// pricing.
constexpr int kGtab = 3;

struct DpPrice {
  SlicePricer P;          // global-memory cells
  int cells;              // cells per kind (nm * ns)
  const AxisPos* mbp;     // [max_n + 1]
  const AxisPos* pin;     // [total]
  const double* in_d;     // [total]
  int max_n;
  AxisPos p0;             // bracket of length 0 (padded lengths start at 0)
  const int* gbase;       // kGtab: per ordered sample, its length's table row at d = 0
                          // (int32: the call keeps G below 2^31 entries)
  const double* g_odd;    // kGtab: the table shifted by one entry (g_odd[k + 1] = G[k]), so
                          // every 32-entry window starts 16 B aligned in one of the copies
};

// Rows per band tile (= rows per DP block).  The band of a segment is stored
// as one tile per block of 32 rows, top-down (block b holds rows
// [max(0, n-32(b+1)), n-32b)); tile column c holds the 32 rows' values for
// slice end j = i0 + c, contiguous (256 B per column).
constexpr int kRB = 32;
// Slice-table DP state key (dp.cu KEYED): (1 + count) << kKeyShift | column,
// a positive int32 while the column and 1 + count stay below 2^16 and 2^15:
// the slice table serves mini-batches of at most kGtabMaxN samples.
constexpr int kKeyShift = 16;
constexpr int kGtabMaxN = 32766;

// Compact band (length-sorted single-input mini-batches: cost.cu
// band_run_kernel<.., true> writes it, dp.cu dp_pass_kernel<.., .., .., true>
// and finalize read it).  A tile's near tile (columns [0, 64): the DP's
// serial triangle) stays dense; each far 32-column chunk kk >= 2 keeps, IN
// PLACE of its dense region (columns [32 kk, 32 kk + 32) x 32 rows), a record: the values
// of the distinct (micro-batch size d, padded length) pairs its columns use —
// one window d in [cs - 31, ce] per run of equal lengths [cs, ce] — nv =
// chunk_nv[id] doubles (nv <= 32 x columns, so the record fits the region),
// and colbase[id][q] (int16) with
//     T(row r, column 32 kk + q) = vals[colbase[q] - r]
// for every slice of an existing row r: far columns have d = column - r >= 33,
// and d > w_r reads NaN exactly like the dense band (past the row's last
// feasible j every act_mem exceeds the cap; with no cap every d fits).
// Readers mask rows past the top tile's last row and d <= 0 (band_cand).
// NaN values: act_mem > cap.
// Record ids: chunk kk of the tile at band offset `off` (doubles) of block gb
// is chunk_id0(off, gb) + kk — disjoint across tiles (ceil(W / 32) <=
// floor(32 W / 1024) + 1).  Also indexes the per-chunk minima (cmin).
__host__ __device__ inline int64_t chunk_id0(int64_t off, int gb) { return (off >> 10) + gb; }

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
  unsigned long long tsingle;  // dkey of the largest feasible singleton slice time (band_run_kernel; 0: none)
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
// Shared-memory load the compiler may not hoist or cache in registers (keeps
// per-step operands out of the register file of latency-bound loops).
__device__ __forceinline__ double lds_f64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// Plain arrive (release.cta): a consumer hands a buffer back to the producer.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
// 8-byte asynchronous global -> shared copy (LDGSTS): no register staging,
// so one warp keeps a whole unit's loads in flight; cp_async_wait_all makes
// the calling thread's copies complete (and visible to it) before it arrives
// on the consumers' barrier.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Producer side of a named-barrier hand-off (release; the consumer's
// named_bar on the same id and count completes it).
__device__ __forceinline__ void named_bar_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
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
