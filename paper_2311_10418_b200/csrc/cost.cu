// cost.cu — fused slice costing on sm_100a.  Produces, on the device, the
// slice-time table the reference builds with n(n+1)/2 std::function calls
// (microbatch.cpp:228-243), stored as a compact *band* of 32-row tiles.
//
// Mapping: one warp per 32-row block, lane r <-> row i = i0 + r, and a
// warp-uniform loop over tile columns c (slice end j = i0 + c) in chunks of
// 32.  Per chunk the warp stages in shared memory the 32 padded-length
// candidates in[j-1], tgt[j-1] with their pre-bracketed sequence-axis
// positions, and the 63 micro-batch-size brackets the lanes need, so the
// inner loop issues no global loads.  Each lane keeps its own running maxima
// of the padded lengths (microbatch.cpp:143-148), so unsorted spans are
// priced exactly like the reference; tile writes are 256 B coalesced columns.
//
// Pass A (cap < +inf): act_mem only, every j in (i, n]:
//   Rm(i) = max{ j : !(M[i,j] > cap) } (the last memory-feasible end), the
//   singleton check (microbatch.cpp:245-251) and the tile width
//   W_b = max_r (r + w_r) + 1.  With cap = +inf every slice is feasible,
//   Rm(i) = n, and pass A is replaced by full_rows_kernel.
// Pass B: T for c in [r+1, r+w_r] into the tile (NaN where M > cap: it never
//   passes `T <= t_max`, exactly like the reference's `continue` at
//   microbatch.cpp:179), plus the candidate statistics (microbatch.cpp:253-269).
// Pass C (band_cand_kernel): reads the band back and marks candidate values
//   k = ceil(T / I) in a per-segment bitmap, or appends raw values for a
//   segmented sort (exact mode I == 0, or very wide k ranges).
// Every slice outside (i, Rm(i)] has M > cap, so the DP never needs it; no
// monotonicity of the cost model is assumed anywhere.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "pp_internal.cuh"

namespace ppb {

namespace {

constexpr int kCostWarps = 8;

// Shared-memory image of the cost grid + candidate-bin thresholds.
struct GridSmem {
  size_t tt, am, lay, tau, bytes;
};
__host__ __device__ inline GridSmem grid_smem_layout(int nm, int ns, int n_lay, int n_tau) {
  GridSmem g;
  const size_t cells = 2 * (size_t)nm * ns;
  g.tt = 0;
  g.am = g.tt + cells * sizeof(double4);
  g.lay = g.am + cells * sizeof(double2);
  g.tau = g.lay + (size_t)n_lay * sizeof(LayoutD);
  g.bytes = g.tau + (size_t)n_tau * sizeof(double);
  return g;
}

// bracket() of the mbs axis for every micro-batch size 1..max_n.
__global__ void mbs_bracket_kernel(CostGrid g, int max_n, AxisPos* __restrict__ out) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m <= max_n; m += gridDim.x * blockDim.x) {
    AxisPos p;
    bracket(g.mbs_ax, g.nm, (double)m, p.seg, p.t);
    p.pad = p.seg * g.ns;  // row base of the cell table (band_kernel)
    out[m] = p;
  }
}

// bracket() of the sequence axis at every ordered sample's input / target length.
__global__ void seq_bracket_kernel(CostGrid g, const double* __restrict__ in_d,
                                   const double* __restrict__ tgt_d, int64_t total,
                                   AxisPos* __restrict__ pin, AxisPos* __restrict__ ptg) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    AxisPos p;
    p.pad = 0;
    bracket(g.seq_ax, g.ns, in_d[k], p.seg, p.t);
    pin[k] = p;
    bracket(g.seq_ax, g.ns, tgt_d[k], p.seg, p.t);
    ptg[k] = p;
  }
}

struct CostArgs {
  CostGrid g;
  const double* tabT;
  const double* tabM;
  const double* in_d;
  const double* tgt_d;
  const AxisPos* pin;
  const AxisPos* ptg;
  const int64_t* seg_off;
  const int* blk_base;
  int n_seg;
  int total_blocks;
  int max_n;
  const AxisPos* mbp;
  double cap;
  double interval;
  int* row_w;
  int* row_fb;  // pass A -> B: first memory-infeasible j of the row (INT_MAX: none)
  int* blk_W;
  SegStats* stats;
  const int64_t* tile_off;
  const int64_t* seg_band_base;
  double* band;
  // pass A: certified row exit (capi.cu mem_exit_threshold): once a slice's
  // act_mem exceeds this, every longer slice of the row exceeds the cap
  // (+inf = no certificate, scan every j like the reference).
  double exit_thresh;
  // pass B: 256-bit candidate bitmap per segment for k = ceil(T / I) < 256
  // (null when I == 0), and the bin thresholds tau[k] = the largest double T
  // with fl(T / I) <= k, so k = ceil(fl(T / I)) = min{k : T <= tau[k]} needs
  // no division (monotone, correctly rounded division; capi.cu bin_thresholds)
  unsigned int* small_bm;
  const double* tau;
  // pass B (band_run_kernel): per far chunk k of a tile (the DP's columns
  // [64 + 32k, 96 + 32k)), the least slice time (act_mem ignored) over the
  // live rows at its first column; slot ((tile base) >> 10) + k.  Lets the DP
  // candidate passes stop streaming a tile where every row has passed t
  // (dp.cu; capi.cu time_trunc_margin).  Null: not recorded.
  double* cmin;
  // pass B (band_run_kernel<.., true>): compact chunk records instead of the
  // dense band (pp_internal.cuh "compact band"); null: dense band
  short* colbase;
  int* chunk_nv;
};

// SRC: 0 = fused grid costing, grid staged in shared memory
//      1 = fused grid costing, grid read from global memory (oversized grids)
//      2 = host-evaluated triangular tables (generic SliceCostFn)
// PASS 0 = A (act_mem, Rm, singleton check, W_b); PASS 1 = B (band + candidates).
template <int PASS, int SRC, int LAY>
__global__ void __launch_bounds__(32 * kCostWarps)
    block_kernel(CostArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ double s_x[kCostWarps][32], s_y[kCostWarps][32];
  __shared__ AxisPos s_px[kCostWarps][32], s_py[kCostWarps][32];
  __shared__ AxisPos s_mb[kCostWarps][64];
  __shared__ unsigned int s_bm[kCostWarps][kSmallBmWords];
  constexpr bool kGrid = SRC != 2;
  const int nm = a.g.nm, ns = a.g.ns, n_lay = a.g.n_lay, used = a.g.used;
  const double4* tt = a.g.tt;
  const double2* am = a.g.am;
  const LayoutD* lay = a.g.lay;
  const double* tau = a.tau;
  if (SRC == 0) {
    const GridSmem L = grid_smem_layout(nm, ns, n_lay, a.tau ? kSmallBmWords * 32 : 0);
    double4* stt = reinterpret_cast<double4*>(dsm + L.tt);
    double2* sam = reinterpret_cast<double2*>(dsm + L.am);
    LayoutD* slay = reinterpret_cast<LayoutD*>(dsm + L.lay);
    double* stau = reinterpret_cast<double*>(dsm + L.tau);
    const int cells = 2 * nm * ns;
    for (int k = threadIdx.x; k < cells; k += blockDim.x) {
      stt[k] = a.g.tt[k];
      sam[k] = a.g.am[k];
    }
    for (int k = threadIdx.x; k < n_lay; k += blockDim.x) slay[k] = a.g.lay[k];
    if (a.tau)
      for (int k = threadIdx.x; k < kSmallBmWords * 32; k += blockDim.x) stau[k] = a.tau[k];
    __syncthreads();
    tt = stt;
    am = sam;
    lay = slay;
    tau = a.tau ? stau : nullptr;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warps = gridDim.x * kCostWarps;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const bool need_mem = PASS == 0 || !(a.cap == INF);
  const bool encdec = a.g.is_encdec != 0;
  constexpr int kTau = kSmallBmWords * 32;
  // bracket of the initial padded length 0.0 (shape.input_len = 0, :143-144)
  AxisPos p0{0.0, 0, 0};
  if (kGrid) bracket(a.g.seq_ax, ns, 0.0, p0.seg, p0.t);
  for (int gb = blockIdx.x * kCostWarps + wid; gb < a.total_blocks; gb += warps) {
    const int s = seg_of(a.blk_base, a.n_seg, gb);
    const int64_t b0 = a.seg_off[s];
    const int n = (int)(a.seg_off[s + 1] - b0);
    const int bl = gb - a.blk_base[s];
    const int i1 = n - kRB * bl;
    const int i0 = max(0, i1 - kRB);
    const int nb = i1 - i0;
    const int r = lane;
    const bool rowv = r < nb;
    const int i = i0 + r;
    int wr = 0, cend, fb = INT_MAX;
    double* tile = nullptr;
    if (PASS == 1) {
      wr = rowv ? a.row_w[b0 + i] : 0;
      if (need_mem && SRC != 2 && rowv) fb = a.row_fb[b0 + i];
      cend = a.blk_W[gb] - 1;
      tile = a.band + a.seg_band_base[s] + a.tile_off[gb];
    } else {
      cend = n - i0;
    }
    // running padded maxima and their sequence brackets
    double pin = 0.0, ptg = 0.0;
    AxisPos pe = p0, pd = p0;
    int last_ok = i;
    bool done = !rowv;  // pass A: row certified finished (or no row)
    double kmn = INF, kmx = -INF;
    unsigned long long nraw = 0;
    int flags = 0;
    int last_k = -1, kw = 0;
    // the lane's current bin kw and its bounds: T in (tlo, thi] <=> bin kw
    double tlo = -INF, thi = (PASS == 1 && tau) ? tau[0] : -INF;
    bool any_binned = false;
    unsigned int npriced = 0;
    if (PASS == 1 && a.small_bm) {
      if (lane < kSmallBmWords) s_bm[wid][lane] = 0u;
      __syncwarp();
    }
    const int64_t trow = SRC == 2 ? (int64_t)i * n - (int64_t)i * (i - 1) / 2 - (i + 1) : 0;
    if (PASS == 1) tile[r] = masked();  // column 0: j = i0 <= i is never a slice
    for (int c0 = 1; c0 <= cend; c0 += 32) {
      if (kGrid) {
        // stage the chunk: column c0 + q reads sample index i0 + c0 + q - 1
        const int cq = c0 + lane;
        if (cq <= cend) {
          const int64_t k = b0 + i0 + cq - 1;
          s_x[wid][lane] = a.in_d[k];
          s_px[wid][lane] = a.pin[k];
          if (encdec) {
            s_y[wid][lane] = a.tgt_d[k];
            s_py[wid][lane] = a.ptg[k];
          }
        }
        // micro-batch sizes m = c - r in [c0 - 31, c0 + 31] -> slot m - (c0 - 32)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int p = lane + 32 * h;
          s_mb[wid][p] = a.mbp[min(max(c0 - 32 + p, 1), a.max_n)];
        }
        __syncwarp();
      }
      const int qend = min(32, cend - c0 + 1);
      for (int q = 0; q < qend; ++q) {
        const int c = c0 + q;
        const int j = i0 + c;
        const bool live = rowv && c >= r + 1 && (PASS == 0 ? !done : c <= r + wr);
        // pass B writes every tile entry: NaN outside the row's feasible span,
        // so the band needs no separate fill
        double outv = masked();
        if (live) {
        double T = 0.0, M = 0.0;
        bool ok = true;
        if (SRC == 2) {
          T = a.tabT[trow + j];
          M = a.tabM[trow + j];
          ok = !(M > a.cap);
        } else {
          const double x = s_x[wid][q];
          const AxisPos px = s_px[wid][q];
          const bool upx = pin < x;
          pin = upx ? x : pin;
          pe.t = upx ? px.t : pe.t;
          pe.seg = upx ? px.seg : pe.seg;
          if (encdec) {
            const double y = s_y[wid][q];
            const AxisPos py = s_py[wid][q];
            const bool upy = ptg < y;
            ptg = upy ? y : ptg;
            pd.t = upy ? py.t : pd.t;
            pd.seg = upy ? py.seg : pd.seg;
          }
          const AxisPos mb = s_mb[wid][q - r + 32];
          // the decoder reads the target length of encoder-decoder models (:301-302)
          const int sd = encdec ? pd.seg : pe.seg;
          const double tsd = encdec ? pd.t : pe.t;
          if (PASS == 0) {
            slice_cost_lay<LAY, false, true>(tt, am, lay, n_lay, used, nm, ns, mb.seg, mb.t, pe.seg, pe.t,
                                             sd, tsd, a.g.le, a.g.ld, T, M);
            ok = !(M > a.cap);
          } else {
            slice_cost_lay<LAY, true, false>(tt, am, lay, n_lay, used, nm, ns, mb.seg, mb.t, pe.seg, pe.t,
                                             sd, tsd, a.g.le, a.g.ld, T, M);
            // act_mem only from the row's first infeasible slice on (pass A):
            // every earlier slice of the row is feasible
            if (j >= fb) {
              double T2;
              slice_cost_lay<LAY, false, true>(tt, am, lay, n_lay, used, nm, ns, mb.seg, mb.t, pe.seg,
                                               pe.t, sd, tsd, a.g.le, a.g.ld, T2, M);
              ok = !(M > a.cap);
            }
          }
        }
        ++npriced;
        if (PASS == 0) {
          if (ok) last_ok = j;
          fb = (!ok & (j < fb)) ? j : fb;
          if (c == r + 1 && !ok) atomicMin(&a.stats[s].err_row, i);
          if (M > a.exit_thresh) done = true;
        } else {
          outv = ok ? T : masked();
          if (ok && !isnan(T)) {
            ++nraw;
            bool binned = false;
            if (kGrid && tau && T >= 0.0) {
              // k = min{k : T <= tau[k]}; a row's bins change rarely, so the
              // common case is two compares against the cached bounds
              if (!(T > tlo && T <= thi)) {
                int k = kw;
                while (k < kTau && !(T <= tau[k])) ++k;
                while (k > 0 && T <= tau[k - 1]) --k;
                kw = min(k, kTau - 1);
                tlo = kw > 0 ? tau[kw - 1] : -INF;
                thi = tau[kw];
              }
              if (T <= thi) {  // else beyond the last threshold: exact division below
                binned = true;
                any_binned = true;
                if (kw != last_k) {  // a row's bins repeat in runs
                  atomicOr(&s_bm[wid][kw >> 5], 1u << (kw & 31));
                  last_k = kw;
                }
              }
            }
            double qv = T;
            if (!binned && a.interval > 0) qv = ceil(__ddiv_rn(T, a.interval));
            if (binned) {
            } else if (isinf(qv)) {
              flags |= (qv > 0) ? 1 : 2;
            } else {
              kmn = (qv < kmn) ? qv : kmn;
              kmx = (kmx < qv) ? qv : kmx;
              if (a.small_bm && qv >= 0.0 && qv < (double)kTau) {
                const int k = (int)qv;
                if (k != last_k) {  // a row's bins repeat in runs
                  atomicOr(&s_bm[wid][k >> 5], 1u << (k & 31));
                  last_k = k;
                }
              }
            }
          }
        }
        }  // live
        if (PASS == 1) tile[(size_t)c * kRB + r] = outv;
      }
      if (kGrid) __syncwarp();
      if (PASS == 0 && !__any_sync(0xffffffffu, !done)) break;  // every row certified done
    }
    unsigned long long np = npriced;
#pragma unroll
    for (int o = 16; o; o >>= 1) np += __shfl_xor_sync(0xffffffffu, np, o);
    if (PASS == 0) {
      const int w = rowv ? last_ok - i : 0;
      if (rowv) {
        a.row_w[b0 + i] = w;
        a.row_fb[b0 + i] = fb;
      }
      int wmax = rowv ? r + w : 0;
#pragma unroll
      for (int o = 16; o; o >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
      if (lane == 0) {
        a.blk_W[gb] = wmax + 1;
        atomicAdd(&a.stats[s].priced, np);
      }
    } else {
      if (any_binned) {  // binned values lie in [0, kTau): widen the range to a superset
        kmn = (0.0 < kmn) ? 0.0 : kmn;
        kmx = (kmx < (double)(kTau - 1)) ? (double)(kTau - 1) : kmx;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, kmn, o);
        const double y = __shfl_xor_sync(0xffffffffu, kmx, o);
        kmn = (x < kmn) ? x : kmn;
        kmx = (kmx < y) ? y : kmx;
        nraw += __shfl_xor_sync(0xffffffffu, nraw, o);
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
      }
      if (lane == 0) {
        atomicAdd(&a.stats[s].priced_b, np);
        if (nraw) {
          atomicAdd(&a.stats[s].nraw, nraw);
          if (!isinf(kmn)) {
            atomicMin(&a.stats[s].kmin, dkey(kmn));
            atomicMax(&a.stats[s].kmax, dkey(kmx));
          }
        }
        if (flags) atomicOr(&a.stats[s].flags, flags);
      }
      if (a.small_bm) {
        __syncwarp();
        if (lane < kSmallBmWords) {
          const unsigned int w = s_bm[wid][lane];
          if (w) atomicOr(&a.small_bm[(size_t)s * kSmallBmWords + lane], w);
        }
        __syncwarp();
      }
    }
  }
}

// Pass A by certified bisection.  Applies when every segment is sorted by
// input length and every priced stage kind reads the input length (decoder-
// only models, or encoder-decoder models without decoder layers): the padded
// shape of slice [i, j) is then (j - i, max(0, in[j-1])), so any slice can be
// priced in O(1).  With the monotonicity certificate (capi.cu
// mem_exit_threshold: exact act_mem non-decreasing in j, device error <= E):
//   * a j with M~(i,j) > cap + 2E makes every longer slice infeasible (jx);
//   * a j with M~(i,j) <= cap - 2E makes every shorter slice feasible (jlo);
// bisection finds such crossing points in ~2 log2(n) pricings, and only the
// few slices strictly between them are priced one by one.  Rm(i), the first
// infeasible end fb(i) and the singleton check come out exactly as from the
// full scan of block_kernel<0>.
template <int SRC, int LAY>
__global__ void __launch_bounds__(32 * kCostWarps)
    rowexit_kernel(CostArgs a, double lo_thresh) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int nm = a.g.nm, ns = a.g.ns, n_lay = a.g.n_lay, used = a.g.used;
  const double4* tt = a.g.tt;
  const double2* am = a.g.am;
  const LayoutD* lay = a.g.lay;
  if (SRC == 0) {
    const GridSmem L = grid_smem_layout(nm, ns, n_lay, 0);
    double4* stt = reinterpret_cast<double4*>(dsm + L.tt);
    double2* sam = reinterpret_cast<double2*>(dsm + L.am);
    LayoutD* slay = reinterpret_cast<LayoutD*>(dsm + L.lay);
    const int cells = 2 * nm * ns;
    for (int k = threadIdx.x; k < cells; k += blockDim.x) {
      stt[k] = a.g.tt[k];
      sam[k] = a.g.am[k];
    }
    for (int k = threadIdx.x; k < n_lay; k += blockDim.x) slay[k] = a.g.lay[k];
    __syncthreads();
    tt = stt;
    am = sam;
    lay = slay;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warps = gridDim.x * kCostWarps;
  const double cap = a.cap, hi_thresh = a.exit_thresh;
  AxisPos p0{0.0, 0, 0};
  bracket(a.g.seq_ax, ns, 0.0, p0.seg, p0.t);
  for (int gb = blockIdx.x * kCostWarps + wid; gb < a.total_blocks; gb += warps) {
    const int s = seg_of(a.blk_base, a.n_seg, gb);
    const int64_t b0 = a.seg_off[s];
    const int n = (int)(a.seg_off[s + 1] - b0);
    const int bl = gb - a.blk_base[s];
    const int i1 = n - kRB * bl;
    const int i0 = max(0, i1 - kRB);
    const int r = lane;
    const bool rowv = r < i1 - i0;
    const int i = i0 + r;
    unsigned int npriced = 0;
    int w = 0;
    if (rowv) {
      // act_mem of slice [i, j): shape (j - i, max(0, in[j-1]))
      auto mem_of = [&](int j) -> double {
        ++npriced;
        const AxisPos mb = a.mbp[min(j - i, a.max_n)];
        const bool pos = 0.0 < a.in_d[b0 + j - 1];
        const AxisPos px = a.pin[b0 + j - 1];
        const int se = pos ? px.seg : p0.seg;
        const double ts = pos ? px.t : p0.t;
        double T, M;
        slice_cost_lay<LAY, false, true>(tt, am, lay, n_lay, used, nm, ns, mb.seg, mb.t, se, ts, se, ts,
                                         a.g.le, a.g.ld, T, M);
        return M;
      };
      const double m1 = mem_of(i + 1);
      if (m1 > cap) atomicMin(&a.stats[s].err_row, i);  // microbatch.cpp:245-251
      // jx: every slice [i, j >= jx) is infeasible
      int jx = n + 1;
      if (mem_of(n) > hi_thresh) {
        int lo = i, hi = n;  // mem_of(hi) > hi_thresh; lo: empty or <= hi_thresh
        while (hi - lo > 1) {
          const int mid = lo + ((hi - lo) >> 1);
          if (mem_of(mid) > hi_thresh) hi = mid; else lo = mid;
        }
        jx = hi;
      }
      // jlo: every slice [i, j <= jlo) is feasible
      int jlo = i;
      if (m1 <= lo_thresh) {
        int lo = i + 1, hi = jx;  // hi: virtual (> lo_thresh) or jx
        while (hi - lo > 1) {
          const int mid = lo + ((hi - lo) >> 1);
          if (mem_of(mid) <= lo_thresh) lo = mid; else hi = mid;
        }
        jlo = lo;
      }
      int last_ok = jlo, fb = INT_MAX;
      for (int j = jlo + 1; j < min(jx, n + 1); ++j) {
        const double m = (j == i + 1) ? m1 : mem_of(j);
        const bool ok = !(m > cap);
        last_ok = ok ? j : last_ok;
        fb = (!ok & (j < fb)) ? j : fb;
      }
      if (jx <= n) fb = min(fb, jx);
      w = last_ok - i;
      a.row_w[b0 + i] = w;
      a.row_fb[b0 + i] = fb;
    }
    int wmax = rowv ? r + w : 0;
    unsigned long long np = npriced;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
      np += __shfl_xor_sync(0xffffffffu, np, o);
    }
    if (lane == 0) {
      a.blk_W[gb] = wmax + 1;
      atomicAdd(&a.stats[s].priced, np);
    }
  }
}

// Cells of the cost grid the lean band kernel keeps in STATIC shared memory
// (statically shared addresses: plain LDS with immediate offsets, no generic
// address conversion in the loop); larger grids take band_kernel.
constexpr int kBandCells = 384;  // 2 kinds x 192 (mbs x seq) cells: 18 KB

// Pass B, quantised candidates (I > 0), grid staged in static shared memory:
// the leanest column loop.  ENC: encoder-decoder model (decoder reads the
// target length; its running maximum is tracked).  SIN: segments sorted by
// input length (padded input = max(0, in[j-1]), no running maximum).
// Candidate bins: a lane's slice times grow along its row, so the bins it
// hits through the fast path form a contiguous run [run_lo, kw]; runs are
// written to the warp's bitmap only when they end (a miss or the block end).
template <int LAY, bool SIN, bool ENC>
__global__ void __launch_bounds__(32 * kCostWarps)
    band3_kernel(CostArgs a) {
  __shared__ double4 s_tt[kBandCells];
  __shared__ double2 s_am[kBandCells];
  __shared__ double s_tau[kSmallBmWords * 32];
  __shared__ double s_x[kCostWarps][32], s_y[kCostWarps][32];
  __shared__ AxisPos s_px[kCostWarps][32], s_py[kCostWarps][32];
  __shared__ AxisPos s_mb[kCostWarps][64];
  __shared__ unsigned int s_bm[kCostWarps][kSmallBmWords];
  const int nm = a.g.nm, ns = a.g.ns;
  {
    const int cells = 2 * nm * ns;
    for (int k = threadIdx.x; k < cells; k += blockDim.x) {
      s_tt[k] = a.g.tt[k];
      s_am[k] = a.g.am[k];
    }
    for (int k = threadIdx.x; k < kSmallBmWords * 32; k += blockDim.x) s_tau[k] = a.tau[k];
    __syncthreads();
  }
  const int per = nm * ns;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warps = gridDim.x * kCostWarps;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);
  const bool need_mem = !(a.cap == INF);
  constexpr int kTau = kSmallBmWords * 32;
  const double le = a.g.le, ld = a.g.ld, ival = a.interval, cap = a.cap;
  AxisPos p0{0.0, 0, 0};
  bracket(a.g.seq_ax, ns, 0.0, p0.seg, p0.t);
  // one kind's (t_f, t_b) at cell row mb (mi * ns) and sequence segment sg
  auto kind_time = [&](int base, int mb, double tm, int sg, double ts, double& tf, double& tb) {
    const int s1 = min(sg + 1, ns - 1);
    const double4 c0 = s_tt[base + mb + sg], c1 = s_tt[base + mb + s1];
    tf = blend_d(tm, ts, c0.x, c0.z, c1.x, c1.z);
    tb = blend_d(tm, ts, c0.y, c0.w, c1.y, c1.w);
  };
  auto kind_mem = [&](int base, int mb, double tm, int sg, double ts) {
    const int s1 = min(sg + 1, ns - 1);
    const double2 c0 = s_am[base + mb + sg], c1 = s_am[base + mb + s1];
    return blend_d(tm, ts, c0.x, c0.y, c1.x, c1.y);
  };
  // bits [lo, hi] of the warp's bin bitmap
  auto mark_run = [&](int lo, int hi) {
    for (int w = lo >> 5; w <= (hi >> 5); ++w) {
      const int b_lo = max(lo - 32 * w, 0), b_hi = min(hi - 32 * w, 31);
      const unsigned int m = (b_hi == 31 ? 0xffffffffu : ((1u << (b_hi + 1)) - 1u)) & ~((1u << b_lo) - 1u);
      atomicOr(&s_bm[wid][w], m);
    }
  };
  for (int gb = blockIdx.x * kCostWarps + wid; gb < a.total_blocks; gb += warps) {
    const int s = seg_of(a.blk_base, a.n_seg, gb);
    const int64_t b0 = a.seg_off[s];
    const int n = (int)(a.seg_off[s + 1] - b0);
    const int bl = gb - a.blk_base[s];
    const int i1 = n - kRB * bl;
    const int i0 = max(0, i1 - kRB);
    const int r = lane;
    const bool rowv = r < i1 - i0;
    const int i = i0 + r;
    const int wr = rowv ? a.row_w[b0 + i] : 0;  // 0: never live
    const int fb = (need_mem && rowv) ? a.row_fb[b0 + i] : INT_MAX;
    int cfb = (fb != INT_MAX && fb <= i + wr) ? fb - i0 : INT_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) cfb = min(cfb, __shfl_xor_sync(0xffffffffu, cfb, o));
    const int W = a.blk_W[gb];
    double* tile = a.band + a.seg_band_base[s] + a.tile_off[gb];
    tile[r] = QNAN;  // column 0: j = i0 <= i is never a slice
    double pin = 0.0, ptg = 0.0;
    AxisPos pe = p0, pd = p0;
    int kw = -1, run_lo = -1;
    double tlo = INF, thi = -INF, tnx = -INF;
    double kmn = INF, kmx = -INF;
    int flags = 0;
    unsigned int npriced = 0;
    if (lane < kSmallBmWords) s_bm[wid][lane] = 0u;
    __syncwarp();
    for (int c0 = 1; c0 < W; c0 += 32) {
      const int cq = c0 + lane;
      if (cq < W) {
        const int64_t k = b0 + i0 + cq - 1;
        s_x[wid][lane] = a.in_d[k];
        s_px[wid][lane] = a.pin[k];
        if (ENC) {
          s_y[wid][lane] = a.tgt_d[k];
          s_py[wid][lane] = a.ptg[k];
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = lane + 32 * h;
        s_mb[wid][p] = a.mbp[min(max(c0 - 32 + p, 1), a.max_n)];
      }
      __syncwarp();
      const int qend = min(32, W - c0);
      for (int q = 0; q < qend; ++q) {
        const int c = c0 + q;
        const bool inrow = c > r;  // sample j-1 belongs to slice [i, j)
        const bool live = inrow & (c <= r + wr);
        if (SIN) {
          const AxisPos px = s_px[wid][q];
          const bool pos = 0.0 < s_x[wid][q];
          pe.t = pos ? px.t : p0.t;
          pe.seg = pos ? px.seg : p0.seg;
        } else {
          const double x = s_x[wid][q];
          const AxisPos px = s_px[wid][q];
          const bool upx = inrow & (pin < x);
          pin = upx ? x : pin;
          pe.t = upx ? px.t : pe.t;
          pe.seg = upx ? px.seg : pe.seg;
        }
        if (ENC) {
          const double y = s_y[wid][q];
          const AxisPos py = s_py[wid][q];
          const bool upy = inrow & (ptg < y);
          ptg = upy ? y : ptg;
          pd.t = upy ? py.t : pd.t;
          pd.seg = upy ? py.seg : pd.seg;
        }
        const AxisPos mb = s_mb[wid][q - r + 32];
        const int sd = ENC ? pd.seg : pe.seg;
        const double tsd = ENC ? pd.t : pe.t;
        double T;
        {
          double df, db;
          kind_time(per, mb.pad, mb.t, sd, tsd, df, db);
          const double t2 = __dadd_rn(__dmul_rn(ld, df), __dmul_rn(ld, db));
          if (LAY == kLayDec1) {
            T = t2;
          } else {  // kLayEncDec2
            double ef, eb;
            kind_time(0, mb.pad, mb.t, pe.seg, pe.t, ef, eb);
            const double t1 = __dadd_rn(__dmul_rn(le, ef), __dmul_rn(le, eb));
            T = (t1 < t2) ? t2 : t1;
          }
        }
        bool ok = true;
        if (c >= cfb) {  // act_mem near the cap: warp-uniform, rare
          const bool chk = live & (i0 + c >= fb);
          double M = __dmul_rn(ld, kind_mem(per, mb.pad, mb.t, sd, tsd));
          if (LAY != kLayDec1) {
            const double a1 = __dmul_rn(le, kind_mem(0, mb.pad, mb.t, pe.seg, pe.t));
            M = (a1 < M) ? M : a1;
          }
          ok = !(chk & (M > cap));
        }
        const bool feas = live & ok;
        tile[(size_t)c * kRB + r] = feas ? T : QNAN;
        npriced += live ? 1u : 0u;
        // bin fast path: same bin, or the next one
        const bool step = feas & (T > thi) & (T <= tnx) & (kw + 1 < kTau);
        kw += step ? 1 : 0;
        tlo = step ? thi : tlo;
        thi = step ? tnx : thi;
        {
          const double nx = s_tau[min(kw + 1, kTau - 1)];
          tnx = step ? ((kw + 1 < kTau) ? nx : INF) : tnx;
        }
        const bool miss = feas & !((T > tlo) & (T <= thi));
        if (__any_sync(0xffffffffu, miss)) {
          if (miss) {
            if (run_lo >= 0) mark_run(run_lo, kw);
            run_lo = -1;
            int k = max(kw, 0);
            while (k < kTau && !(T <= s_tau[k])) ++k;
            while (k > 0 && T <= s_tau[k - 1]) --k;
            if (k < kTau) {
              kw = k;
              run_lo = k;
              tlo = k > 0 ? s_tau[k - 1] : -INF;
              thi = s_tau[k];
              tnx = (k + 1 < kTau) ? s_tau[k + 1] : INF;
            } else {  // beyond the thresholds (or +inf): exact quantisation
              const double qv = ceil(__ddiv_rn(T, ival));
              if (isinf(qv)) {
                flags |= (qv > 0) ? 1 : 2;
              } else {
                kmn = (qv < kmn) ? qv : kmn;
                kmx = (kmx < qv) ? qv : kmx;
              }
            }
          }
        }
      }
      __syncwarp();
    }
    if (run_lo >= 0) mark_run(run_lo, kw);
    const bool any_binned = __any_sync(0xffffffffu, kw >= 0);
    if (any_binned) {  // binned values lie in [0, kTau): widen the range to a superset
      kmn = (0.0 < kmn) ? 0.0 : kmn;
      kmx = (kmx < (double)(kTau - 1)) ? (double)(kTau - 1) : kmx;
    }
    unsigned long long np = npriced;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, kmn, o);
      const double y = __shfl_xor_sync(0xffffffffu, kmx, o);
      kmn = (x < kmn) ? x : kmn;
      kmx = (kmx < y) ? y : kmx;
      np += __shfl_xor_sync(0xffffffffu, np, o);
      flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if (lane == 0) {
      atomicAdd(&a.stats[s].priced_b, np);
      if (np) atomicAdd(&a.stats[s].nraw, np);  // >= the raw count; only sizes the raw fallback
      if (!isinf(kmn)) {
        atomicMin(&a.stats[s].kmin, dkey(kmn));
        atomicMax(&a.stats[s].kmax, dkey(kmx));
      }
      if (flags) atomicOr(&a.stats[s].flags, flags);
    }
    __syncwarp();
    if (lane < kSmallBmWords) {
      const unsigned int w = s_bm[wid][lane];
      if (w) atomicOr(&a.small_bm[(size_t)s * kSmallBmWords + lane], w);
    }
    __syncwarp();
  }
}

// Pass B for segments sorted by input length with one sequence input (GPT):
// the slice [i, j) pads to in[j-1], so its time and act_mem depend only on
// (d = j - i, in[j-1]).  Sorted mini-batches repeat lengths (C3: ~1550
// distinct lengths in 8192 samples, and the wide rows are the short, dense
// ones), so along a diagonal of the band the same value recurs for every
// column of a run of equal lengths: only ~11% of C3's band slices are
// distinct (d, run) pairs.  Each pair is priced ONCE, with exactly the
// operations of band3_kernel, into a per-warp ring indexed by d, and every
// column of the run reads its 32 entries back (lane r: d = c - r):
//   * a column chunk splits into pieces of equal length (a ballot over the
//     staged lengths); a piece prices the diagonals it reaches that the run
//     has not priced yet, 32 per batch (lane l: d = next + l), then stores
//     its columns (one coalesced 256 B column per step);
//   * the ring holds the last 128 priced diagonals, enough for a piece of up
//     to 32 columns (needs d in [cs - 31, ce]) after a batch overshoot.
// Feasibility is (live) & !(act_mem > cap) per entry: act_mem > cap implies
// j >= the row's first infeasible j (pass A), which is exactly band3's test.
// A pair's candidate bin is recorded iff some LIVE slice of the tile carries
// it (a range-max over the tile's row widths: rows r' with d <= w_r' whose
// column r' + d lies in the run), so the candidate set is the reference's
// exactly.  The store stream is the kernel's bound rather than FP64 issue.
// NOSTORE: the band is not written at all — the DP prices its slices itself
// (dp.cu, PRICE != 0); this pass then only marks the candidate bins, the
// per-chunk minima and the singleton maximum (no tile, no record).
template <int LAY, bool COMPACT, bool NOSTORE>
__global__ void __launch_bounds__(32 * kCostWarps, 4)  // 4 CTAs (32 warps) per SM: more stores in flight
    band_run_kernel(CostArgs a) {
  __shared__ double4 s_tt[kBandCells];
  __shared__ double2 s_am[kBandCells];
  __shared__ double s_tau[kSmallBmWords * 32];
  __shared__ double s_x[kCostWarps][32];
  __shared__ AxisPos s_px[kCostWarps][32];
  __shared__ double s_ring[kCostWarps][160];  // 128 diagonals + a mirror of the first 32 (no wrap on reads)
  __shared__ short s_cb[kCostWarps][32];
  __shared__ int s_rmq[kCostWarps][5][32];
  __shared__ unsigned int s_bm[kCostWarps][kSmallBmWords];
  const int nm = a.g.nm, ns = a.g.ns;
  {
    const int cells = 2 * nm * ns;
    for (int k = threadIdx.x; k < cells; k += blockDim.x) {
      s_tt[k] = a.g.tt[k];
      s_am[k] = a.g.am[k];
    }
    for (int k = threadIdx.x; k < kSmallBmWords * 32; k += blockDim.x) s_tau[k] = a.tau[k];
    __syncthreads();
  }
  const int per = nm * ns;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warps = gridDim.x * kCostWarps;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);
  const bool need_mem = !(a.cap == INF);
  constexpr int kTau = kSmallBmWords * 32;
  const double ival = a.interval;
  AxisPos p0{0.0, 0, 0};
  bracket(a.g.seq_ax, ns, 0.0, p0.seg, p0.t);
  SlicePricer SP{s_tt, s_tt + per, s_am, s_am + per, ns, a.g.le, a.g.ld, a.cap, need_mem};
  // slice time (band3_kernel's operations) ...
  auto price_t = [&](const AxisPos& mb, const AxisPos& pe) { return price_time<LAY>(SP, mb, pe); };
  // ... NaN where act_mem exceeds the cap
  auto price = [&](const AxisPos& mb, const AxisPos& pe) { return price_slice<LAY>(SP, mb, pe); };
  for (int gb = blockIdx.x * kCostWarps + wid; gb < a.total_blocks; gb += warps) {
    const int s = seg_of(a.blk_base, a.n_seg, gb);
    const int64_t b0 = a.seg_off[s];
    const int n = (int)(a.seg_off[s + 1] - b0);
    const int bl = gb - a.blk_base[s];
    const int i1 = n - kRB * bl;
    const int i0 = max(0, i1 - kRB);
    const int r = lane;
    const bool rowv = r < i1 - i0;
    const int wr = rowv ? a.row_w[b0 + i0 + r] : 0;  // 0: never live
    // the last tile column on which every row of the tile is live
    int minlive = r + wr;
#pragma unroll
    for (int o = 16; o; o >>= 1) minlive = min(minlive, __shfl_xor_sync(0xffffffffu, minlive, o));
    // range-max table over the tile's row widths (levels 0..4: windows of 2^L rows)
    {
      int m = wr;
      s_rmq[wid][0][lane] = m;
#pragma unroll
      for (int L = 1; L < 5; ++L) {
        m = max(m, __shfl_down_sync(0xffffffffu, m, 1 << (L - 1)));
        s_rmq[wid][L][lane] = m;
      }
    }
    if (lane < kSmallBmWords) s_bm[wid][lane] = 0u;
    __syncwarp();
    auto rmq = [&](int lo, int hi) {  // max of the row widths r' in [lo, hi], 0 <= lo <= hi <= 31
      const int L = min(31 - __clz(hi - lo + 1), 4);  // two windows of 2^L cover the range
      return max(s_rmq[wid][L][lo], s_rmq[wid][L][hi - (1 << L) + 1]);
    };
    // candidate bins of the priced pairs: k = ceil(T / I) exactly as the
    // reference computes it, one division per bin change of the lane (its bin
    // (tlo, thi] = (tau[k-1], tau[k]] is cached); bits gather in one register
    // word until the word changes
    double tlo = INF, thi = -INF;
    int cw = -1;
    unsigned int cbits = 0u;
    double kmn = INF, kmx = -INF;
    int flags = 0;
    bool any_binned = false;
    auto bin = [&](double T) {
      if ((T > tlo) & (T <= thi)) return;  // the lane's current bin: already marked
      const double qv = ceil(__ddiv_rn(T, ival));
      if (qv < (double)kTau) {  // T >= +0: qv in [0, kTau)
        const int k = (int)qv;
        tlo = k > 0 ? s_tau[k - 1] : -INF;
        thi = s_tau[k];
        any_binned = true;
        if ((k >> 5) != cw) {
          if (cbits) atomicOr(&s_bm[wid][cw], cbits);
          cw = k >> 5;
          cbits = 0u;
        }
        cbits |= 1u << (k & 31);
      } else if (isinf(qv)) {
        flags |= (qv > 0) ? 1 : 2;
      } else {
        kmn = (qv < kmn) ? qv : kmn;
        kmx = (kmx < qv) ? qv : kmx;
      }
    };
    const int W = a.blk_W[gb];
    double* tile = a.band + a.seg_band_base[s] + a.tile_off[gb];
    const int64_t cid = chunk_id0(a.seg_band_base[s] + a.tile_off[gb], gb);  // record of column chunk 0
    double* ring = s_ring[wid];
    double prev_x = QNAN;  // NaN: the first column starts a run
    AxisPos pe = p0;       // sequence bracket of the current run
    int ca = 0, cb = 0;    // the run's first and last column (within the tile)
    int done = 0;          // the run's diagonals up to `done` are in the ring
    // 32-column chunks aligned with the DP's (column 0 = the never-live
    // diagonal, a one-column run of its own)
    for (int c0 = 0; c0 < W; c0 += 32) {
      const int kk = c0 >> 5;
      const int cq = c0 + lane;
      double xq = QNAN;
      AxisPos pxq = p0;
      if (cq < W && cq > 0) {
        const int64_t k = b0 + i0 + cq - 1;
        xq = a.in_d[k];
        pxq = a.pin[k];
      }
      s_x[wid][lane] = xq;
      s_px[wid][lane] = pxq;
      // bit q: column c0 + q ends its run (the next column differs or is past the tile)
      double xn = __shfl_down_sync(0xffffffffu, xq, 1);
      if (lane == 31) xn = (cq + 1 < W) ? a.in_d[b0 + i0 + cq] : QNAN;
      const unsigned int run_end = __ballot_sync(0xffffffffu, !(xn == xq));
      __syncwarp();
      const int qend = min(32, W - c0);
      // far chunks (kk >= 2) of a COMPACT band hold records; the near tile
      // (columns [0, 64), the DP's serial triangle) stays dense
      const bool rec = COMPACT && kk >= 2;
      double* vals = tile + (size_t)c0 * kRB;  // the chunk's region: its record
      int voff = 0;                            // values written to the record
      double vfirst = QNAN;                    // the lane's entry at the chunk's first column
      for (int q = 0; q < qend;) {
        const unsigned int e = run_end >> q;
        const int qe = min(e ? q + __ffs(e) - 1 : 31, qend - 1);
        const int cs = c0 + q, ce = c0 + qe;
        const double x = s_x[wid][q];
        if (!(x == prev_x)) {  // warp-uniform: column cs starts a run of equal lengths
          prev_x = x;
          const AxisPos px = s_px[wid][q];
          const bool pos = 0.0 < x;
          pe.t = pos ? px.t : p0.t;
          pe.seg = pos ? px.seg : p0.seg;
          ca = cs;
          if (e) {
            cb = c0 + q + __ffs(e) - 1;
          } else {  // the run continues past this chunk
            cb = W - 1;
            for (int base = c0 + 32; base < W; base += 32) {
              const int cc = base + lane;
              const bool same = (cc < W) && (a.in_d[b0 + i0 + cc - 1] == x);
              const unsigned int diff = __ballot_sync(0xffffffffu, !same);
              if (diff) {
                cb = base + __ffs(diff) - 2;
                break;
              }
            }
          }
          if (cb == cs) {  // a one-column run: lane r prices its own slice (r, cs), d = cs - r
            const int d = cs - r;
            const double F = price(a.mbp[min(max(d, 1), a.max_n)], pe);
            const bool live = (unsigned)(d - 1) < (unsigned)wr;
            if (rec) {
              vals[voff + 31 - r] = F;  // window d in [cs - 31, cs]
              if (lane == 0) s_cb[wid][q] = (short)(voff + 31);
              voff += 32;
            } else if (!NOSTORE) {
              tile[(size_t)cs * kRB + r] = live ? F : QNAN;
            }
            if (live && !isnan(F)) bin(F);
            if (q == 0) vfirst = F;
            q = qe + 1;
            continue;
          }
          done = cs - 32;
        }
        // price the run's diagonals (done, ce] (d <= 0 entries are never live)
        while (done < ce) {
          const int d = done + 1 + lane;
          const double F = price(a.mbp[min(max(d, 1), a.max_n)], pe);
          ring[d & 127] = F;
          if ((d & 127) < 32) ring[(d & 127) + 128] = F;
          // live slices carrying (d, run): rows r' in [ca - d, cb - d] with w_r' >= d
          const int lo = max(ca - d, 0), hi = min(cb - d, 31);
          if ((d >= 1) && (lo <= hi) && !isnan(F) && rmq(lo, hi) >= d) bin(F);
          done += 32;
        }
        __syncwarp();
        if (q == 0) vfirst = ring[(cs - r) & 127];
        if (rec) {
          // the piece's window d in [cs - 31, ce]; column c reads it at c - cs + 31 - r
          const int L = ce - cs + 32;
          for (int idx = lane; idx < L; idx += 32) vals[voff + idx] = ring[(cs - 31 + idx) & 127];
          if (lane <= qe - q) s_cb[wid][q + lane] = (short)(voff + lane + 31);
          voff += L;
        } else if (!NOSTORE) {
          // column c: lane r stores ring[d = c - r], live iff 1 <= d <= w_r
          double* out = tile + (size_t)cs * kRB + r;
          // the lane's diagonals of the piece sit at ring[b .. b + ce - cs]
          // without wrapping (the ring's mirrored upper half)
          const double* src = ring + ((cs - r) & 127);
          if (cs >= kRB && ce <= minlive) {
            // every row live on every column of the piece: a plain copy
            const int L = ce - cs + 1;
            int k = 0;
            for (; k + 4 <= L; k += 4) {
              const double v0 = src[k], v1 = src[k + 1], v2 = src[k + 2], v3 = src[k + 3];
              out[(size_t)k * kRB] = v0;
              out[(size_t)(k + 1) * kRB] = v1;
              out[(size_t)(k + 2) * kRB] = v2;
              out[(size_t)(k + 3) * kRB] = v3;
            }
            for (; k < L; ++k) out[(size_t)k * kRB] = src[k];
          } else {
            int d = cs - r;
#pragma unroll 2
            for (int c = cs; c <= ce; ++c) {
              const double v = *src++;
              *out = ((unsigned)(d - 1) < (unsigned)wr) ? v : QNAN;
              out += kRB;
              ++d;
            }
          }
        }
        __syncwarp();
        q = qe + 1;
      }
      if (rec) {
        __syncwarp();
        a.colbase[(cid + kk) * 32 + lane] = lane < qend ? s_cb[wid][lane] : (short)0;
        if (lane == 0) a.chunk_nv[cid + kk] = voff;
      }
      // far chunk (kk >= 2): least slice time over the live rows at its first
      // column (act_mem-masked entries re-priced), for the DP's truncation
      if (a.cmin && kk >= 2) {
        const int d = c0 - r;
        double v = vfirst;
        const bool live = (unsigned)(d - 1) < (unsigned)wr;
        if (live && isnan(v)) v = price_t(a.mbp[min(max(d, 1), a.max_n)], pe);
        v = live ? v : INF;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double y = __shfl_xor_sync(0xffffffffu, v, o);
          v = (y < v) ? y : v;
        }
        if (lane == 0) a.cmin[cid + kk] = v;
      }
      __syncwarp();
    }
    {
      // the tile's singleton slices [i, i+1) (column r + 1 <= 32, in the dense
      // near tile, written by this lane): their largest feasible time bounds
      // t* from below (dp.cu seg_init_kernel)
      double v;
      if (NOSTORE) {  // no tile: price the singleton (d = 1, in[i]) directly
        const double x = rowv ? a.in_d[b0 + i0 + r] : QNAN;
        const AxisPos px = rowv ? a.pin[b0 + i0 + r] : p0;
        v = (r + 1 < W) ? price(a.mbp[1], (0.0 < x) ? px : p0) : QNAN;
      } else {
        v = (r + 1 < W) ? tile[(size_t)(r + 1) * kRB + r] : QNAN;
      }
      v = (wr > 0 && !isnan(v)) ? v : -INF;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, v, o);
        v = (v < y) ? y : v;
      }
      if (lane == 0 && v > -INF) atomicMax(&a.stats[s].tsingle, dkey(v));
    }
    const unsigned int npriced = (unsigned int)wr;  // live slices of the row: columns r+1 .. r+wr
    if (cbits) atomicOr(&s_bm[wid][cw], cbits);
    const bool any_b = __any_sync(0xffffffffu, any_binned);
    if (any_b) {  // binned values lie in [0, kTau): widen the range to a superset
      kmn = (0.0 < kmn) ? 0.0 : kmn;
      kmx = (kmx < (double)(kTau - 1)) ? (double)(kTau - 1) : kmx;
    }
    unsigned long long np = npriced;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, kmn, o);
      const double y = __shfl_xor_sync(0xffffffffu, kmx, o);
      kmn = (x < kmn) ? x : kmn;
      kmx = (kmx < y) ? y : kmx;
      np += __shfl_xor_sync(0xffffffffu, np, o);
      flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if (lane == 0) {
      atomicAdd(&a.stats[s].priced_b, np);
      if (np) atomicAdd(&a.stats[s].nraw, np);  // >= the raw count; only sizes the raw fallback
      if (!isinf(kmn)) {
        atomicMin(&a.stats[s].kmin, dkey(kmn));
        atomicMax(&a.stats[s].kmax, dkey(kmx));
      }
      if (flags) atomicOr(&a.stats[s].flags, flags);
    }
    __syncwarp();
    if (lane < kSmallBmWords) {
      const unsigned int w = s_bm[wid][lane];
      if (w) atomicOr(&a.small_bm[(size_t)s * kSmallBmWords + lane], w);
    }
    __syncwarp();
  }
}

// Pass B, fused grid costing with quantised candidates (I > 0): the lean
// form of block_kernel<1, SRC, LAY>.  Every lane prices every column of its
// warp's tile unconditionally and masks the result (no divergence in the
// column loop); act_mem is priced only where some lane of the warp reaches
// its row's first infeasible slice (pass A), and candidate bins only leave
// the two-compare fast path when a lane's slice time crosses into another bin.
template <int SRC, int LAY, bool SIN>
__global__ void __launch_bounds__(32 * kCostWarps)
    band_kernel(CostArgs a) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ double s_x[kCostWarps][32], s_y[kCostWarps][32];
  __shared__ AxisPos s_px[kCostWarps][32], s_py[kCostWarps][32];
  __shared__ AxisPos s_mb[kCostWarps][64];
  __shared__ unsigned int s_bm[kCostWarps][kSmallBmWords];
  const int nm = a.g.nm, ns = a.g.ns, n_lay = a.g.n_lay, used = a.g.used;
  const double4* tt = a.g.tt;
  const double2* am = a.g.am;
  const LayoutD* lay = a.g.lay;
  const double* tau = a.tau;
  if (SRC == 0) {
    const GridSmem L = grid_smem_layout(nm, ns, n_lay, kSmallBmWords * 32);
    double4* stt = reinterpret_cast<double4*>(dsm + L.tt);
    double2* sam = reinterpret_cast<double2*>(dsm + L.am);
    LayoutD* slay = reinterpret_cast<LayoutD*>(dsm + L.lay);
    double* stau = reinterpret_cast<double*>(dsm + L.tau);
    const int cells = 2 * nm * ns;
    for (int k = threadIdx.x; k < cells; k += blockDim.x) {
      stt[k] = a.g.tt[k];
      sam[k] = a.g.am[k];
    }
    for (int k = threadIdx.x; k < n_lay; k += blockDim.x) slay[k] = a.g.lay[k];
    for (int k = threadIdx.x; k < kSmallBmWords * 32; k += blockDim.x) stau[k] = a.tau[k];
    __syncthreads();
    tt = stt;
    am = sam;
    lay = slay;
    tau = stau;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int warps = gridDim.x * kCostWarps;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);
  const bool need_mem = !(a.cap == INF);
  const bool encdec = a.g.is_encdec != 0;
  constexpr int kTau = kSmallBmWords * 32;
  AxisPos p0{0.0, 0, 0};
  bracket(a.g.seq_ax, ns, 0.0, p0.seg, p0.t);
  for (int gb = blockIdx.x * kCostWarps + wid; gb < a.total_blocks; gb += warps) {
    const int s = seg_of(a.blk_base, a.n_seg, gb);
    const int64_t b0 = a.seg_off[s];
    const int n = (int)(a.seg_off[s + 1] - b0);
    const int bl = gb - a.blk_base[s];
    const int i1 = n - kRB * bl;
    const int i0 = max(0, i1 - kRB);
    const int r = lane;
    const bool rowv = r < i1 - i0;
    const int i = i0 + r;
    const int wr = rowv ? a.row_w[b0 + i] : 0;  // 0: never live
    const int fb = (need_mem && rowv) ? a.row_fb[b0 + i] : INT_MAX;
    // first tile column at which any row of the warp reaches its first
    // infeasible slice: only from there on is act_mem priced (warp-uniform)
    // (a lane needs it only when an infeasible slice lies INSIDE its feasible
    // span, i.e. fb <= i + wr: act_mem not monotone along the row)
    int cfb = (fb != INT_MAX && fb <= i + wr) ? fb - i0 : INT_MAX;
#pragma unroll
    for (int o = 16; o; o >>= 1) cfb = min(cfb, __shfl_xor_sync(0xffffffffu, cfb, o));
    const double le = a.g.le, ld = a.g.ld, ival = a.interval;
    const int W = a.blk_W[gb];
    double* tile = a.band + a.seg_band_base[s] + a.tile_off[gb];
    tile[r] = QNAN;  // column 0: j = i0 <= i is never a slice
    double pin = 0.0, ptg = 0.0;
    AxisPos pe = p0, pd = p0;
    // candidate bin of the lane: T in (tlo, thi] <=> bin kw (first slice always
    // misses); bins seen are kept in a 64-bit window [kb, kb + 64) and
    // flushed to the warp's shared bitmap only when the window moves
    int kw = -1, kb = 0;
    double tlo = INF, thi = -INF, tnx = -INF;  // tnx = tau[kw + 1]
    unsigned long long win = 0ull;
    double kmn = INF, kmx = -INF;
    int flags = 0;
    bool any_binned = false;
    unsigned int npriced = 0;
    if (lane < kSmallBmWords) s_bm[wid][lane] = 0u;
    __syncwarp();
    for (int c0 = 1; c0 < W; c0 += 32) {
      const int cq = c0 + lane;
      if (cq < W) {
        const int64_t k = b0 + i0 + cq - 1;
        s_x[wid][lane] = a.in_d[k];
        s_px[wid][lane] = a.pin[k];
        if (encdec) {
          s_y[wid][lane] = a.tgt_d[k];
          s_py[wid][lane] = a.ptg[k];
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = lane + 32 * h;
        s_mb[wid][p] = a.mbp[min(max(c0 - 32 + p, 1), a.max_n)];
      }
      __syncwarp();
      const int qend = min(32, W - c0);
#pragma unroll 2
      for (int q = 0; q < qend; ++q) {
        const int c = c0 + q;
        const int j = i0 + c;
        const bool inrow = c > r;  // sample j-1 belongs to slice [i, j)
        const bool live = inrow & (c <= r + wr);
        if (SIN) {
          // sorted by input: the padded input of [i, j) is max(0, in[j-1])
          const AxisPos px = s_px[wid][q];
          const bool pos = 0.0 < s_x[wid][q];
          pe.t = pos ? px.t : p0.t;
          pe.seg = pos ? px.seg : p0.seg;
        } else {
          const double x = s_x[wid][q];
          const AxisPos px = s_px[wid][q];
          const bool upx = inrow & (pin < x);
          pin = upx ? x : pin;
          pe.t = upx ? px.t : pe.t;
          pe.seg = upx ? px.seg : pe.seg;
        }
        if (encdec) {
          const double y = s_y[wid][q];
          const AxisPos py = s_py[wid][q];
          const bool upy = inrow & (ptg < y);
          ptg = upy ? y : ptg;
          pd.t = upy ? py.t : pd.t;
          pd.seg = upy ? py.seg : pd.seg;
        }
        const AxisPos mb = s_mb[wid][q - r + 32];
        const int sd = encdec ? pd.seg : pe.seg;
        const double tsd = encdec ? pd.t : pe.t;
        double T, M;
        slice_cost_lay<LAY, true, false>(tt, am, lay, n_lay, used, nm, ns, mb.seg, mb.t, pe.seg, pe.t, sd,
                                         tsd, le, ld, T, M);
        bool ok = true;
        if (c >= cfb) {  // act_mem near the cap: warp-uniform, rare
          const bool chk = live & (j >= fb);
          double T2;
          slice_cost_lay<LAY, false, true>(tt, am, lay, n_lay, used, nm, ns, mb.seg, mb.t, pe.seg, pe.t,
                                           sd, tsd, le, ld, T2, M);
          ok = !(chk & (M > a.cap));
        }
        const bool feas = live & ok;
        tile[(size_t)c * kRB + r] = feas ? T : QNAN;
        npriced += live ? 1u : 0u;
        // candidate bin k = ceil(fl(T / I)) = min{k : T <= tau[k]} (microbatch.cpp:264).
        // Fast path, branch-free: same bin, or the next one (slice times grow
        // along a row).
        const bool step = feas & (T > thi) & (T <= tnx) & (kw + 1 < kb + 64) & (kw + 1 < kTau);
        kw = step ? kw + 1 : kw;
        tlo = step ? thi : tlo;
        thi = step ? tnx : thi;
        win |= step ? (1ull << (kw - kb)) : 0ull;
        {
          const double nx = tau[min(kw + 1, kTau - 1)];  // unconditional: no branch
          tnx = step ? ((kw + 1 < kTau) ? nx : INF) : tnx;
        }
        const bool miss = feas & !((T > tlo) & (T <= thi));
        if (__any_sync(0xffffffffu, miss)) {
          if (miss) {
            int k = max(kw, 0);
            while (k < kTau && !(T <= tau[k])) ++k;
            while (k > 0 && T <= tau[k - 1]) --k;
            if (k < kTau) {
              if (k < kb || k >= kb + 64) {  // move the window
                for (int w = 0; w < 2; ++w) {
                  const unsigned int part = (unsigned int)(win >> (32 * w));
                  if (part) atomicOr(&s_bm[wid][(kb >> 5) + w], part);
                }
                win = 0ull;
                kb = k & ~31;
              }
              kw = k;
              tlo = k > 0 ? tau[k - 1] : -INF;
              thi = tau[k];
              tnx = (k + 1 < kTau) ? tau[k + 1] : INF;
              win |= 1ull << (k - kb);
              any_binned = true;
            } else {  // beyond the thresholds (or +inf): exact quantisation
              const double qv = ceil(__ddiv_rn(T, ival));
              if (isinf(qv)) {
                flags |= (qv > 0) ? 1 : 2;
              } else {
                kmn = (qv < kmn) ? qv : kmn;
                kmx = (kmx < qv) ? qv : kmx;
              }
            }
          }
        }
      }
      __syncwarp();
    }
    for (int w = 0; w < 2; ++w) {  // flush the bin window
      const unsigned int part = (unsigned int)(win >> (32 * w));
      if (part) atomicOr(&s_bm[wid][(kb >> 5) + w], part);
    }
    if (any_binned) {  // binned values lie in [0, kTau): widen the range to a superset
      kmn = (0.0 < kmn) ? 0.0 : kmn;
      kmx = (kmx < (double)(kTau - 1)) ? (double)(kTau - 1) : kmx;
    }
    unsigned long long np = npriced;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, kmn, o);
      const double y = __shfl_xor_sync(0xffffffffu, kmx, o);
      kmn = (x < kmn) ? x : kmn;
      kmx = (kmx < y) ? y : kmx;
      np += __shfl_xor_sync(0xffffffffu, np, o);
      flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    }
    if (lane == 0) {
      atomicAdd(&a.stats[s].priced_b, np);
      if (np) atomicAdd(&a.stats[s].nraw, np);  // >= the raw count; only sizes the raw fallback
      if (!isinf(kmn)) {
        atomicMin(&a.stats[s].kmin, dkey(kmn));
        atomicMax(&a.stats[s].kmax, dkey(kmx));
      }
      if (flags) atomicOr(&a.stats[s].flags, flags);
    }
    __syncwarp();
    if (lane < kSmallBmWords) {
      const unsigned int w = s_bm[wid][lane];
      if (w) atomicOr(&a.small_bm[(size_t)s * kSmallBmWords + lane], w);
    }
    __syncwarp();
  }
}

// cap = +inf: every slice is memory-feasible (!(M > inf) holds for every M,
// NaN included), so Rm(i) = n and W_b = n - i0 + 1 without costing anything.
__global__ void full_rows_kernel(const int64_t* __restrict__ seg_off, const int* __restrict__ blk_base,
                                 int n_seg, int total_blocks, int* __restrict__ row_w,
                                 int* __restrict__ blk_W) {
  for (int gb = blockIdx.x * blockDim.x + threadIdx.x; gb < total_blocks;
       gb += gridDim.x * blockDim.x) {
    const int s = seg_of(blk_base, n_seg, gb);
    const int64_t b0 = seg_off[s];
    const int n = (int)(seg_off[s + 1] - b0);
    const int bl = gb - blk_base[s];
    const int i1 = n - kRB * bl;
    const int i0 = max(0, i1 - kRB);
    for (int i = i0; i < i1; ++i) row_w[b0 + i] = n - i;
    blk_W[gb] = n - i0 + 1;
  }
}

// Pass C: candidate values from the band (microbatch.cpp:259-266).
__global__ void __launch_bounds__(256)
    band_cand_kernel(const int64_t* __restrict__ seg_off, const int* __restrict__ blk_base, int n_seg,
                     int total_blocks, const int* __restrict__ blk_W,
                     const int64_t* __restrict__ tile_off, const int64_t* __restrict__ seg_band_base,
                     const double* __restrict__ band, double interval,
                     const SegStats* __restrict__ stats, unsigned int* __restrict__ bitmap,
                     const int64_t* __restrict__ bitmap_off, const int* __restrict__ seg_mode,
                     unsigned long long* __restrict__ cand_raw,
                     const int64_t* __restrict__ cand_raw_off,
                     unsigned long long* __restrict__ cand_raw_cnt, const short* __restrict__ colbase,
                     const int* __restrict__ row_w) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int gb = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gb < total_blocks; gb += warps) {
    const int s = seg_of(blk_base, n_seg, gb);
    const int mode = seg_mode[s];
    if (mode > 1) continue;
    const double* tile = band + seg_band_base[s] + tile_off[gb];
    const int W = blk_W[gb];
    const double kmin = mode == 0 ? dkey_inv(stats[s].kmin) : 0.0;
    unsigned int* bm = bitmap + bitmap_off[s];
    long long last_bit = -1;
    // compact band (pp_internal.cuh): entry (lane, c) of a live slice is
    // record value colbase[c] - lane; other entries are masked here
    int wr = 0;
    int64_t cid = 0;
    if (colbase) {
      const int n = (int)(seg_off[s + 1] - seg_off[s]);
      const int i1 = n - kRB * (gb - blk_base[s]);
      const int i0 = max(0, i1 - kRB);
      wr = lane < i1 - i0 ? row_w[seg_off[s] + i0 + lane] : 0;
      cid = chunk_id0(seg_band_base[s] + tile_off[gb], gb);
    }
    for (int c = 1; c < W; ++c) {
      double T;
      if (colbase && c >= 64) {
        const int kk = c >> 5;
        T = (unsigned)(c - lane - 1) < (unsigned)wr
                ? tile[(size_t)kk * (32 * kRB) + colbase[(cid + kk) * 32 + (c & 31)] - lane]
                : __longlong_as_double(0x7ff8000000000000LL);
      } else {
        T = tile[(size_t)c * kRB + lane];
      }
      if (isnan(T)) continue;
      double q = T;
      if (interval > 0) q = ceil(__ddiv_rn(T, interval));
      if (mode == 0) {
        if (isinf(q)) continue;  // +-inf candidates come from the flags
        const long long bit = (long long)(q - kmin);
        if (bit != last_bit) {
          atomicOr(&bm[bit >> 5], 1u << (bit & 31));
          last_bit = bit;
        }
      } else {
        double qq = interval > 0 ? __dmul_rn(q, interval) : T;
        if (qq == 0.0) qq = 0.0;  // +0.0: the reference's order of equal +-0 is unspecified
        const unsigned long long slot = atomicAdd(&cand_raw_cnt[s], 1ULL);
        cand_raw[cand_raw_off[s] + slot] = dkey(qq);
      }
    }
  }
}

// Per-segment exclusive scan of tile sizes (32 x W_b doubles) -> tile offsets.
__global__ void __launch_bounds__(1024)
    tile_offsets_kernel(const int* __restrict__ blk_W, const int* __restrict__ blk_base,
                        int64_t* __restrict__ tile_off, SegStats* __restrict__ stats) {
  __shared__ long long warp_tot[32];
  __shared__ int wmax;
  const int s = blockIdx.x;
  const int b = blk_base[s];
  const int nbk = blk_base[s + 1] - b;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) wmax = 0;
  __syncthreads();
  long long carry = 0;
  for (int t0 = 0; t0 < nbk; t0 += blockDim.x) {
    const int k = t0 + threadIdx.x;
    if (k < nbk) atomicMax(&wmax, blk_W[b + k]);
    const long long v = k < nbk ? (long long)kRB * blk_W[b + k] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      long long w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;
    }
    __syncthreads();
    const long long before = wid ? warp_tot[wid - 1] : 0;
    if (k < nbk) tile_off[b + k] = carry + before + x - v;
    carry += warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    stats[s].band = carry;
    stats[s].wmax = wmax;
  }
}

// Bitmap -> ascending candidate list (k * I), with the +/-inf flags.
__global__ void __launch_bounds__(1024)
    cand_bitmap_kernel(const unsigned int* __restrict__ bitmap, const int64_t* __restrict__ bitmap_off,
                       const SegStats* __restrict__ stats, const int* __restrict__ seg_mode,
                       const unsigned int* __restrict__ small_bm, double interval,
                       const int64_t* __restrict__ cand_off, double* __restrict__ cand,
                       int* __restrict__ cand_n) {
  __shared__ int warp_tot[32];
  const int s = blockIdx.x;
  const int mode = seg_mode[s];
  if (mode != 0 && mode != 3) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // mode 0: bitmap over [kmin, kmax] filled by band_cand_kernel;
  // mode 3: the 256-bit bitmap over [0, 256) filled by cost pass B.
  const int64_t nw = mode == 3 ? kSmallBmWords : bitmap_off[s + 1] - bitmap_off[s];
  const unsigned int* bm = mode == 3 ? small_bm + (size_t)s * kSmallBmWords : bitmap + bitmap_off[s];
  double* out = cand + cand_off[s];
  const SegStats st = stats[s];
  int carry = 0;
  if (st.flags & 2) carry = 1;  // -inf first
  if (threadIdx.x == 0 && (st.flags & 2)) out[0] = -__longlong_as_double(0x7ff0000000000000LL);
  const double kmin = (mode == 0 && st.nraw && st.kmin != ~0ULL) ? dkey_inv(st.kmin) : 0.0;
  for (int64_t t0 = 0; t0 < nw; t0 += blockDim.x) {
    const int64_t k = t0 + threadIdx.x;
    const unsigned int w = k < nw ? bm[k] : 0u;
    const int v = __popc(w);
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int ww = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ww, o);
        if (lane >= o) ww += y;
      }
      warp_tot[lane] = ww;
    }
    __syncthreads();
    int pos = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
    unsigned int rem = w;
    while (rem) {
      const int bit = __ffs(rem) - 1;
      rem &= rem - 1;
      const double kk = kmin + (double)(k * 32 + bit);  // exact: integers < 2^52
      double q = __dmul_rn(kk, interval);               // ceil(t / I) * I (:264)
      if (q == 0.0) q = 0.0;                            // canonical +0.0 (see band_cand_kernel)
      out[pos++] = q;
    }
    carry += warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (st.flags & 1) out[carry++] = __longlong_as_double(0x7ff0000000000000LL);
    cand_n[s] = carry;
  }
}

// After the segmented sort of raw keys: std::unique with operator== on the
// doubles, one CTA per segment.
__global__ void __launch_bounds__(1024)
    cand_unique_kernel(const unsigned long long* __restrict__ keys_a,
                       const unsigned long long* __restrict__ keys_b, const int* __restrict__ in_b,
                       const int64_t* __restrict__ raw_off,
                       const unsigned long long* __restrict__ raw_cnt, const int* __restrict__ seg_mode,
                       const int64_t* __restrict__ cand_off, double* __restrict__ cand,
                       int* __restrict__ cand_n) {
  __shared__ int warp_tot[32];
  const int s = blockIdx.x;
  if (seg_mode[s] != 1) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t n = (int64_t)raw_cnt[s];
  const unsigned long long* kk = (in_b[s] ? keys_b : keys_a) + raw_off[s];
  double* out = cand + cand_off[s];
  int carry = 0;
  for (int64_t t0 = 0; t0 < n; t0 += blockDim.x) {
    const int64_t k = t0 + threadIdx.x;
    double v = 0.0;
    int keep = 0;
    if (k < n) {
      v = dkey_inv(kk[k]);
      keep = (k == 0) || !(dkey_inv(kk[k - 1]) == v);
    }
    int x = keep;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int ww = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, ww, o);
        if (lane >= o) ww += y;
      }
      warp_tot[lane] = ww;
    }
    __syncthreads();
    if (keep) out[carry + (wid ? warp_tot[wid - 1] : 0) + x - 1] = v;
    carry += warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) cand_n[s] = carry;
}

}  // namespace

// ---------------------------------------------------------------- launchers
cudaError_t launch_brackets(const CostGrid& g, int max_n, AxisPos* mbp, const double* in_d,
                            const double* tgt_d, int64_t total, AxisPos* pin, AxisPos* ptg,
                            cudaStream_t st) {
  mbs_bracket_kernel<<<(max_n + 256) / 256, 256, 0, st>>>(g, max_n, mbp);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  if (total > 0)
    seq_bracket_kernel<<<std::max(blocks, 1), 256, 0, st>>>(g, in_d, tgt_d, total, pin, ptg);
  return cudaGetLastError();
}

// pass: 0 = A, 1 = B.  tabT != null selects the table source.
// Pass B takes band_run_kernel (diagonal reuse) for length-sorted
// single-input segments with quantised candidates and a grid that fits its
// static shared memory; only then can the DP price its own slices
// (band_run_kernel<.., NOSTORE>, dp.cu PRICE).
bool band_run_applies(const CostGrid& g, const double* tabT, int reuse, const double* tau, int sorted_in) {
  const GridSmem L = grid_smem_layout(g.nm, g.ns, g.n_lay, tau ? kSmallBmWords * 32 : 0);
  const int src = tabT ? 2 : (L.bytes <= 160 * 1024 ? 0 : 1);
  return reuse && tau && src != 2 && 2 * g.nm * g.ns <= kBandCells && sorted_in && !g.is_encdec &&
         (g.lay_class == kLayDec1 || g.lay_class == kLayEncDec2);
}

cudaError_t launch_cost_pass(int pass, const CostGrid& g, const double* tabT, const double* tabM,
                             const double* in_d, const double* tgt_d, const AxisPos* pin,
                             const AxisPos* ptg, const int64_t* seg_off, const int* blk_base, int n_seg,
                             int total_blocks, int max_n, const AxisPos* mbp, double cap,
                             double interval, int* row_w, int* row_fb, int* blk_W, SegStats* stats,
                             const int64_t* tile_off, const int64_t* seg_band_base, double* band,
                             double exit_thresh, unsigned int* small_bm, const double* tau,
                             double lo_thresh, int bisect, int sorted_in, int reuse, double* cmin,
                             short* colbase, int* chunk_nv, int* wrote_cmin, int nostore, cudaStream_t st) {
  CostArgs a{g, tabT, tabM, in_d, tgt_d, pin, ptg, seg_off, blk_base, n_seg, total_blocks, max_n, mbp,
             cap, interval, row_w, row_fb, blk_W, stats, tile_off, seg_band_base, band, exit_thresh,
             small_bm, tau, cmin, colbase, chunk_nv};
  if (wrote_cmin) *wrote_cmin = 0;
  const GridSmem L = grid_smem_layout(g.nm, g.ns, g.n_lay, tau ? kSmallBmWords * 32 : 0);
  const int src = tabT ? 2 : (L.bytes <= 160 * 1024 ? 0 : 1);
  const size_t sm = src == 0 ? L.bytes : 0;
  const int blocks = std::max(1, std::min((total_blocks + kCostWarps - 1) / kCostWarps, 148 * 32));
#define PP_COST_LAUNCH(P, S, L)                                                                        \
  do {                                                                                                 \
    ensure_dyn_smem((const void*)block_kernel<P, S, L>, sm);                                           \
    block_kernel<P, S, L><<<blocks, 32 * kCostWarps, sm, st>>>(a);                                     \
  } while (0)
#define PP_COST_LAUNCH_L(P, S)                                                  \
  do {                                                                           \
    if (g.lay_class == kLayDec1) PP_COST_LAUNCH(P, S, kLayDec1);                 \
    else if (g.lay_class == kLayEncDec2) PP_COST_LAUNCH(P, S, kLayEncDec2);      \
    else PP_COST_LAUNCH(P, S, kLayGeneric);                                      \
  } while (0)
#define PP_BAND_LAUNCH2(S, L, Z)                                                                      \
  do {                                                                                                 \
    ensure_dyn_smem((const void*)band_kernel<S, L, Z>, sm);                                            \
    band_kernel<S, L, Z><<<blocks, 32 * kCostWarps, sm, st>>>(a);                                      \
  } while (0)
#define PP_BAND_LAUNCH(S, L)                                 \
  do {                                                       \
    if (sorted_in) PP_BAND_LAUNCH2(S, L, true);              \
    else PP_BAND_LAUNCH2(S, L, false);                       \
  } while (0)
#define PP_ROWEXIT_LAUNCH(S, L)                                                                        \
  do {                                                                                                 \
    const size_t smr = S == 0 ? grid_smem_layout(g.nm, g.ns, g.n_lay, 0).bytes : 0;                   \
    ensure_dyn_smem((const void*)rowexit_kernel<S, L>, smr);                                           \
    rowexit_kernel<S, L><<<blocks, 32 * kCostWarps, smr, st>>>(a, lo_thresh);                          \
  } while (0)
  if (pass == 0 && bisect && src != 2) {
    if (src == 0) {
      if (g.lay_class == kLayDec1) PP_ROWEXIT_LAUNCH(0, kLayDec1);
      else if (g.lay_class == kLayEncDec2) PP_ROWEXIT_LAUNCH(0, kLayEncDec2);
      else PP_ROWEXIT_LAUNCH(0, kLayGeneric);
    } else {
      if (g.lay_class == kLayDec1) PP_ROWEXIT_LAUNCH(1, kLayDec1);
      else if (g.lay_class == kLayEncDec2) PP_ROWEXIT_LAUNCH(1, kLayEncDec2);
      else PP_ROWEXIT_LAUNCH(1, kLayGeneric);
    }
  } else if (pass == 0) {
    if (src == 0) PP_COST_LAUNCH_L(0, 0); else if (src == 1) PP_COST_LAUNCH_L(0, 1); else PP_COST_LAUNCH(0, 2, 0);
  } else if (band_run_applies(g, tabT, reuse, tau, sorted_in)) {
    const bool compact = colbase != nullptr && !nostore;
    if (!compact) {
      a.colbase = nullptr;
      a.chunk_nv = nullptr;
    }
    if (g.lay_class == kLayDec1) {
      if (nostore) band_run_kernel<kLayDec1, false, true><<<blocks, 32 * kCostWarps, 0, st>>>(a);
      else if (compact) band_run_kernel<kLayDec1, true, false><<<blocks, 32 * kCostWarps, 0, st>>>(a);
      else band_run_kernel<kLayDec1, false, false><<<blocks, 32 * kCostWarps, 0, st>>>(a);
    } else {
      if (nostore) band_run_kernel<kLayEncDec2, false, true><<<blocks, 32 * kCostWarps, 0, st>>>(a);
      else if (compact) band_run_kernel<kLayEncDec2, true, false><<<blocks, 32 * kCostWarps, 0, st>>>(a);
      else band_run_kernel<kLayEncDec2, false, false><<<blocks, 32 * kCostWarps, 0, st>>>(a);
    }
    if (wrote_cmin) *wrote_cmin = (cmin ? 1 : 0) | (compact && !nostore ? 2 : 0) | (nostore ? 4 : 0);
  } else if (tau && src != 2 && 2 * g.nm * g.ns <= kBandCells &&
             (g.lay_class == kLayDec1 || g.lay_class == kLayEncDec2)) {
#define PP_BAND3(L, Z, E)                                              \
  band3_kernel<L, Z, E><<<blocks, 32 * kCostWarps, 0, st>>>(a)
    const bool enc = g.is_encdec != 0;
    if (g.lay_class == kLayDec1) {
      if (sorted_in) { if (enc) PP_BAND3(kLayDec1, true, true); else PP_BAND3(kLayDec1, true, false); }
      else { if (enc) PP_BAND3(kLayDec1, false, true); else PP_BAND3(kLayDec1, false, false); }
    } else {
      if (sorted_in) { if (enc) PP_BAND3(kLayEncDec2, true, true); else PP_BAND3(kLayEncDec2, true, false); }
      else { if (enc) PP_BAND3(kLayEncDec2, false, true); else PP_BAND3(kLayEncDec2, false, false); }
    }
#undef PP_BAND3
  } else if (tau && src != 2) {
    if (src == 0) {
      if (g.lay_class == kLayDec1) PP_BAND_LAUNCH(0, kLayDec1);
      else if (g.lay_class == kLayEncDec2) PP_BAND_LAUNCH(0, kLayEncDec2);
      else PP_BAND_LAUNCH(0, kLayGeneric);
    } else {
      if (g.lay_class == kLayDec1) PP_BAND_LAUNCH(1, kLayDec1);
      else if (g.lay_class == kLayEncDec2) PP_BAND_LAUNCH(1, kLayEncDec2);
      else PP_BAND_LAUNCH(1, kLayGeneric);
    }
  } else {
    if (src == 0) PP_COST_LAUNCH_L(1, 0); else if (src == 1) PP_COST_LAUNCH_L(1, 1); else PP_COST_LAUNCH(1, 2, 0);
  }
#undef PP_COST_LAUNCH_L
#undef PP_BAND_LAUNCH
#undef PP_BAND_LAUNCH2
#undef PP_ROWEXIT_LAUNCH
#undef PP_COST_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_full_rows(const int64_t* seg_off, const int* blk_base, int n_seg, int total_blocks,
                             int* row_w, int* blk_W, cudaStream_t st) {
  full_rows_kernel<<<std::max(1, (total_blocks + 127) / 128), 128, 0, st>>>(seg_off, blk_base, n_seg,
                                                                             total_blocks, row_w, blk_W);
  return cudaGetLastError();
}

cudaError_t launch_band_cand(const int64_t* seg_off, const int* blk_base, int n_seg, int total_blocks,
                             const int* blk_W, const int64_t* tile_off, const int64_t* seg_band_base,
                             const double* band, double interval, const SegStats* stats,
                             unsigned int* bitmap, const int64_t* bitmap_off, const int* seg_mode,
                             unsigned long long* cand_raw, const int64_t* cand_raw_off,
                             unsigned long long* cand_raw_cnt, const short* colbase, const int* row_w,
                             cudaStream_t st) {
  const int blocks = std::max(1, std::min((total_blocks + 7) / 8, 148 * 32));
  band_cand_kernel<<<blocks, 256, 0, st>>>(seg_off, blk_base, n_seg, total_blocks, blk_W, tile_off,
                                           seg_band_base, band, interval, stats, bitmap, bitmap_off,
                                           seg_mode, cand_raw, cand_raw_off, cand_raw_cnt, colbase, row_w);
  return cudaGetLastError();
}

cudaError_t launch_tile_offsets(const int* blk_W, const int* blk_base, int n_seg, int64_t* tile_off,
                                SegStats* stats, cudaStream_t st) {
  tile_offsets_kernel<<<n_seg, 1024, 0, st>>>(blk_W, blk_base, tile_off, stats);
  return cudaGetLastError();
}

cudaError_t launch_cand_bitmap(const unsigned int* bitmap, const int64_t* bitmap_off,
                               const SegStats* stats, const int* seg_mode, int n_seg,
                               const unsigned int* small_bm, double interval,
                               const int64_t* cand_off, double* cand, int* cand_n, cudaStream_t st) {
  cand_bitmap_kernel<<<n_seg, 1024, 0, st>>>(bitmap, bitmap_off, stats, seg_mode, small_bm, interval,
                                             cand_off, cand, cand_n);
  return cudaGetLastError();
}

cudaError_t launch_cand_unique(const unsigned long long* keys_a, const unsigned long long* keys_b,
                               const int* in_b, const int64_t* raw_off,
                               const unsigned long long* raw_cnt, const int* seg_mode, int n_seg,
                               const int64_t* cand_off, double* cand, int* cand_n, cudaStream_t st) {
  cand_unique_kernel<<<n_seg, 1024, 0, st>>>(keys_a, keys_b, in_b, raw_off, raw_cnt, seg_mode, cand_off,
                                             cand, cand_n);
  return cudaGetLastError();
}

}  // namespace ppb
