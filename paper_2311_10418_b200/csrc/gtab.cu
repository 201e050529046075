// gtab.cu — the shared slice table of length-sorted single-input (GPT)
// mini-batches: the band's replacement.
//
// On a mini-batch sorted by input length (order_samples(Sort),
// microbatch.cpp:97-105) with one sequence input per stage kind, slice
// [i, j) pads to (d = j - i, L = max(0, in[j-1])) (microbatch.cpp:141-148),
// so its time and act_mem (make_slice_cost, :149-155, over estimate,
// cost_model.cpp:294-319) depend on (d, L) only — identically in every
// mini-batch priced with the same grid, model and cap.  Instead of a per
// mini-batch band (2.9 M entries, 23 MB at BASELINE config C3) this file
// builds ONE table for the whole call:
//     G[L][d] = slice time of (d, L), NaN when its act_mem exceeds the cap
// for every length L present and every d some DP tile reads (d up to the
// widest tile column that ends on a sample of length L, need[L]); rows start
// 31 entries before d = 1 so a tile column's 32 rows (d = c - r, r < 32) are
// one contiguous read.  Each (d, L) pair is priced ONCE per call instead of
// once per mini-batch and tile (C3: ~1.5 M table entries per 296 mini-batches
// instead of ~95 M pricings), the DP streams its tile columns from this
// L2-resident table (dp.cu GTAB) instead of HBM, and the candidate bins,
// the singleton maximum and the per-mini-batch statistics come from a scan
// of the table rows a mini-batch's runs of equal lengths reach (gtab_bins):
//     candidates = { ceil(G[L][d] / I) * I : run of length L ending at j,
//                    1 <= d <= min(j, need[L]), G[L][d] not NaN }
// which is exactly the reference's set (microbatch.cpp:253-269): slice
// (j - d, j) is memory-feasible iff act(d, L) <= cap, and every feasible d
// is <= need[L] (a feasible slice lies inside its row's width, hence inside
// the row block's tile).
//
// Values are priced with price_slice (pp_internal.cuh), the operations of
// cost pass B's band_run_kernel, so G holds the band's values bit for bit.
// A second copy shifted by one entry (G1[k + 1] = G[k]) makes every tile
// column's 32-entry window start 16 B aligned in one of the two, so the DP's
// producer moves each column with ONE 256 B cp.async.bulk (TMA) copy.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "pp_internal.cuh"

namespace ppb {

namespace {

constexpr int kGWarps = 8;
constexpr int kGCells = 384;  // cells staged per kind pair (2 kinds x nm x ns <= 384, band_run_applies)

__device__ __forceinline__ int len_key(double x) { return 0.0 < x ? (int)x : 0; }

// need[K] = the widest tile column (slice size d from a block's first row)
// ending on a sample of length K: one warp per 32-row block, the last column
// of each run of equal lengths inside the tile.
__global__ void gtab_need_kernel(const int64_t* __restrict__ seg_off, const int* __restrict__ blk_base, int n_seg,
                                 int total_blocks, const int* __restrict__ blk_W, const double* __restrict__ in_d,
                                 int* __restrict__ need) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int gb = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gb < total_blocks; gb += warps) {
    const int s = seg_of(blk_base, n_seg, gb);
    const int64_t b0 = seg_off[s];
    const int n = (int)(seg_off[s + 1] - b0);
    const int bl = gb - blk_base[s];
    const int i1 = n - kRB * bl;
    const int i0 = max(0, i1 - kRB);
    const int W = blk_W[gb];
    for (int c = 1 + lane; c < W; c += 32) {
      const int64_t p = b0 + i0 + c - 1;  // sample of column c (slice end j = i0 + c)
      const double x = in_d[p];
      const bool last = c + 1 >= W || !(in_d[p + 1] == x);
      if (last) atomicMax(&need[len_key(x)], c);
    }
  }
}

// need[K] by runs (one CTA per segment; the same values as gtab_need_kernel
// with one atomic per run instead of one per tile column that ends a run).
// Block bl's tile covers slice ends j in [i0 + 1, E], E = i0 + W - 1, and a
// run of equal lengths on positions [ps, pe] (slice ends [ps + 1, pe + 1])
// meets it in its last column min(pe + 1, E) - i0 when i0 <= pe and
// E >= max(ps, i0) + 1.  Over the blocks in ascending i0, the first one
// that can meet the run is found by bisection on the prefix maximum of E;
// the walk stops at the first block with E >= pe + 1 (every later block has
// a larger i0, hence a smaller column).  No monotonicity is assumed.
constexpr int kNeedMaxBlocks = 4096;
__global__ void __launch_bounds__(1024) gtab_need_runs_kernel(const int64_t* __restrict__ seg_off,
                                                             const int* __restrict__ blk_base,
                                                             const int* __restrict__ blk_W,
                                                             const double* __restrict__ in_d,
                                                             int* __restrict__ need) {
  extern __shared__ int s_need[];
  const int s = blockIdx.x;
  const int64_t b0 = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b0);
  const int gb0 = blk_base[s];
  const int nblk = blk_base[s + 1] - gb0;
  int* s_i0 = s_need;             // ascending block a: i0
  int* s_E = s_i0 + nblk;         // its tile's last slice end (i0 - 1 + W)
  int* s_pm = s_E + nblk;         // prefix max of s_E
  for (int a = threadIdx.x; a < nblk; a += blockDim.x) {
    const int bl = nblk - 1 - a;
    const int i0 = max(0, n - kRB * (bl + 1));
    s_i0[a] = i0;
    s_E[a] = i0 + blk_W[gb0 + bl] - 1;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    int carry = INT_MIN;
    for (int a0 = 0; a0 < nblk; a0 += 32) {
      int v = a0 + lane < nblk ? s_E[a0 + lane] : INT_MIN;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = max(v, y);
      }
      v = max(v, carry);
      if (a0 + lane < nblk) s_pm[a0 + lane] = v;
      carry = __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  const double* in = in_d + b0;
  for (int pe = threadIdx.x; pe < n; pe += blockDim.x) {
    const double x = in[pe];
    if (pe + 1 < n && in[pe + 1] == x) continue;  // not the run's last position
    // ps = the run's first position (the segment is sorted ascending)
    int lo = 0, hi = pe;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (in[mid] < x) lo = mid + 1; else hi = mid;
    }
    const int ps = lo;
    // first ascending block whose prefix-max end reaches ps + 1
    int a = 0, ah = nblk;
    while (a < ah) {
      const int mid = (a + ah) >> 1;
      if (s_pm[mid] < ps + 1) a = mid + 1; else ah = mid;
    }
    int best = 0;
    for (; a < nblk; ++a) {
      const int i0 = s_i0[a], E = s_E[a];
      if (i0 > pe) break;
      if (E >= max(ps, i0) + 1) best = max(best, min(pe + 1, E) - i0);
      if (E >= pe + 1) break;
    }
    if (best > 0) atomicMax(&need[len_key(x)], best);
  }
}

// Row offsets: rows of lengths with need > 0, each need + 32 entries
// (d in [-31, need]); a 32-entry NaN row at offset 0 serves column 0 of the
// top tiles (never a slice).  One CTA.
__global__ void __launch_bounds__(1024) gtab_offsets_kernel(const int* __restrict__ need, int nK,
                                                            int64_t* __restrict__ row_off,
                                                            long long* __restrict__ total) {
  __shared__ long long warp_tot[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long carry = 32;  // the NaN row
  for (int k0 = 0; k0 < nK; k0 += blockDim.x) {
    const int k = k0 + threadIdx.x;
    const long long v = (k < nK && need[k] > 0) ? (long long)need[k] + 32 : 0;
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
    const long long before = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
    if (k < nK) row_off[k] = v ? before : -1;
    carry += warp_tot[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// G rows: one warp per length, lanes over d in [-31, need]; the cells in
// shared memory like band_run_kernel's.
template <int LAY>
__global__ void __launch_bounds__(32 * kGWarps) gtab_fill_kernel(CostGrid g, double cap, const AxisPos* __restrict__ mbp,
                                                                 int nK, const int* __restrict__ need,
                                                                 const int64_t* __restrict__ row_off,
                                                                 double* __restrict__ G, double* __restrict__ G1) {
  __shared__ double4 s_tt[kGCells];
  __shared__ double2 s_am[kGCells];
  const int nm = g.nm, ns = g.ns, per = nm * ns;
  for (int k = threadIdx.x; k < 2 * per; k += blockDim.x) {
    s_tt[k] = g.tt[k];
    s_am[k] = g.am[k];
  }
  __syncthreads();
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // the NaN row, in both copies
    G[threadIdx.x] = QNAN;
    G1[threadIdx.x + 1] = QNAN;
  }
  const SlicePricer SP{s_tt, s_tt + per, s_am, s_am + per, ns, g.le, g.ld, cap,
                       !(cap == __longlong_as_double(0x7ff0000000000000LL))};
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * kGWarps;
  for (int K = blockIdx.x * kGWarps + (threadIdx.x >> 5); K < nK; K += warps) {
    const int D = need[K];
    if (D <= 0) continue;
    // bracket of the padded length (band_run_kernel: pin of in[j-1], or the
    // bracket of 0.0 for non-positive lengths — K = max(0, L))
    AxisPos pe;
    pe.pad = 0;
    bracket(g.seq_ax, ns, (double)K, pe.seg, pe.t);
    double* row = G + row_off[K];
    double* row1 = G1 + row_off[K] + 1;
    for (int e = lane; e < D + 32; e += 32) {
      const int d = e - 31;
      const double v = d >= 1 ? price_slice<LAY>(SP, mbp[d], pe) : QNAN;
      row[e] = v;
      row1[e] = v;
    }
  }
}

// Per ordered sample: the offset of its length's row at d = 0.
__global__ void gtab_gbase_kernel(const double* __restrict__ in_d, int64_t total, const int64_t* __restrict__ row_off,
                                  int* __restrict__ gbase) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x)
    gbase[k] = (int)(row_off[len_key(in_d[k])] + 31);
}

// Per table row K (after the fill): when the row's candidate bins are an
// interval for every prefix — ival > 0, the non-NaN entries of d in
// [1, need] are a prefix [1, f] of finite values whose bins q(d) =
// ceil(G[K][d] / I) (microbatch.cpp:264) are finite and step by 0 or +1 —
// then the bins of any prefix [1, D] are exactly [q(1), q(min(D, f))], and
// gtab_bins_kernel marks them without scanning the row: rf[K] = f, rlo[K] =
// q(1).  Otherwise rf[K] = -1 and the row is scanned entry by entry.
__global__ void __launch_bounds__(32 * kGWarps) gtab_rowinfo_kernel(int nK, const int* __restrict__ need,
                                                                    const int64_t* __restrict__ row_off,
                                                                    const double* __restrict__ G, double ival,
                                                                    int* __restrict__ rf, double* __restrict__ rlo) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * kGWarps;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  for (int K = blockIdx.x * kGWarps + (threadIdx.x >> 5); K < nK; K += warps) {
    const int D = need[K];
    if (D <= 0) continue;
    const double* row = G + row_off[K] + 31;  // row[d]
    int first_nan = D + 1, last_ok = 0;
    bool bad = !(ival > 0.0);
    for (int d = 1 + lane; d <= D && !bad; d += 32) {
      const double T = row[d];
      if (isnan(T)) {
        first_nan = min(first_nan, d);
        continue;
      }
      last_ok = max(last_ok, d);
      const double q = ceil(__ddiv_rn(T, ival));
      if (!(q < INF) || !(T < INF)) bad = true;
      if (d < D) {
        const double T2 = row[d + 1];
        if (!isnan(T2)) {
          const double q2 = ceil(__ddiv_rn(T2, ival));
          if (!(q2 >= q && q2 <= q + 1.0)) bad = true;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      first_nan = min(first_nan, __shfl_xor_sync(0xffffffffu, first_nan, o));
      last_ok = max(last_ok, __shfl_xor_sync(0xffffffffu, last_ok, o));
    }
    bad = __any_sync(0xffffffffu, bad) || last_ok > first_nan;
    if (lane == 0) {
      rf[K] = bad ? -1 : last_ok;
      rlo[K] = (!bad && last_ok >= 1) ? ceil(__ddiv_rn(row[1], ival)) : 0.0;
    }
  }
}

// Candidate bins and statistics of each mini-batch from the table (the part
// of cost pass B's band_run_kernel that the DP needs before its passes):
// per run of equal lengths ending at position j (1-based slice end), the
// row's entries d in [1, min(j, need)] — the bins ceil(T / I) of the
// non-NaN ones (one division per bin change of a lane, thresholds tau), the
// largest singleton time (SegStats::tsingle, dp.cu seg_init_kernel), the
// range of out-of-bitmap bins (then the call falls back to the band).
// One CTA per segment, up to 32 warps: the row loop is a chain of dependent
// loads (length, run key, table base, row entries), so occupancy hides it
// (8 warps per CTA left the SMs at a quarter of their warp slots on C3).
constexpr int kBinsThreads = 1024;
__global__ void __launch_bounds__(kBinsThreads) gtab_bins_kernel(const int64_t* __restrict__ seg_off,
                                                        const double* __restrict__ in_d,
                                                        const int* __restrict__ gbase,
                                                        const int* __restrict__ need,
                                                        const double* __restrict__ G, double ival,
                                                        const double* __restrict__ tau,
                                                        unsigned int* __restrict__ small_bm,
                                                        SegStats* __restrict__ stats,
                                                        const int* __restrict__ rf,
                                                        const double* __restrict__ rlo) {
  constexpr int kTau = kSmallBmWords * 32;
  __shared__ double s_tau[kTau];
  __shared__ unsigned int s_bm[kSmallBmWords];
  const int s = blockIdx.x;
  const int64_t b0 = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b0);
  for (int k = threadIdx.x; k < kTau; k += blockDim.x) s_tau[k] = tau[k];
  if (threadIdx.x < kSmallBmWords) s_bm[threadIdx.x] = 0u;
  __syncthreads();
  if (stats[s].err_row != INT_MAX) return;  // infeasible singleton: the segment is inactive (block-uniform)
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double tlo = INF, thi = -INF;
  int cw = -1;
  unsigned int cbits = 0u;
  double kmn = INF, kmx = -INF, tsing = -INF;
  int flags = 0;
  bool any_binned = false;
  unsigned long long scanned = 0;
  for (int p0 = wid * 32; p0 < n; p0 += nw * 32) {
    const int p = p0 + lane;
    const double x = p < n ? in_d[b0 + p] : 0.0;
    bool end = p < n && (p + 1 == n || !(in_d[b0 + p + 1] == x));
    if (end && rf != nullptr) {
      // interval rows (gtab_rowinfo_kernel): this lane marks its run alone
      const int K = len_key(x);
      const int f = rf[K];
      if (f >= 0) {
        end = false;
        const int Dp = min(min(p + 1, need[K]), f);
        if (Dp >= 1) {
          const double* row = G + gbase[b0 + p];
          const double t1 = row[1];  // the singleton of the run's samples
          tsing = (tsing < t1) ? t1 : tsing;
          scanned += (unsigned long long)Dp;
          const double lo = rlo[K];
          const double hi = ceil(__ddiv_rn(row[Dp], ival));
          if (lo < (double)kTau) {
            const int k0 = (int)lo, k1 = hi < (double)kTau ? (int)hi : kTau - 1;
            any_binned = true;
            for (int wd = k0 >> 5; wd <= (k1 >> 5); ++wd) {
              const int a0 = max(k0, wd * 32) - wd * 32, a1 = min(k1, wd * 32 + 31) - wd * 32;
              const unsigned int m = (a1 == 31 ? 0xffffffffu : ((1u << (a1 + 1)) - 1u)) & ~((1u << a0) - 1u);
              atomicOr(&s_bm[wd], m);
            }
          }
          if (!(hi < (double)kTau)) {
            const double kl = (lo < (double)kTau) ? (double)kTau : lo;
            kmn = (kl < kmn) ? kl : kmn;
            kmx = (kmx < hi) ? hi : kmx;
          }
        }
      }
    }
    unsigned int ends = __ballot_sync(0xffffffffu, end);
    while (ends) {
      const int q = __ffs(ends) - 1;
      ends &= ends - 1;
      const int j = p0 + q + 1;  // the run's last slice end
      const double xq = __shfl_sync(0xffffffffu, x, q);
      const int gb = gbase[b0 + j - 1];
      const int D = min(j, need[len_key(xq)]);
      const double* row = G + gb;
      if (lane == 0) {
        const double t1 = row[1];  // the singleton of the run's samples
        if (!isnan(t1)) tsing = (tsing < t1) ? t1 : tsing;
      }
      for (int d = 1 + lane; d <= D; d += 32) {
        const double T = row[d];
        if (isnan(T)) continue;
        ++scanned;
        if ((T > tlo) & (T <= thi)) continue;  // the lane's current bin: already marked
        const double qv = ceil(__ddiv_rn(T, ival));  // microbatch.cpp:264
        if (qv < (double)kTau) {  // T >= +0: qv in [0, kTau)
          const int k = (int)qv;
          tlo = k > 0 ? s_tau[k - 1] : -INF;
          thi = s_tau[k];
          any_binned = true;
          if ((k >> 5) != cw) {
            if (cbits) atomicOr(&s_bm[cw], cbits);
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
      }
    }
  }
  if (cbits) atomicOr(&s_bm[cw], cbits);
  if (any_binned) {  // binned values lie in [0, kTau): widen the range to a superset
    kmn = (0.0 < kmn) ? 0.0 : kmn;
    kmx = (kmx < (double)(kTau - 1)) ? (double)(kTau - 1) : kmx;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double a = __shfl_xor_sync(0xffffffffu, kmn, o);
    const double b = __shfl_xor_sync(0xffffffffu, kmx, o);
    const double c = __shfl_xor_sync(0xffffffffu, tsing, o);
    kmn = (a < kmn) ? a : kmn;
    kmx = (kmx < b) ? b : kmx;
    tsing = (tsing < c) ? c : tsing;
    flags |= __shfl_xor_sync(0xffffffffu, flags, o);
    scanned += __shfl_xor_sync(0xffffffffu, scanned, o);
  }
  if (lane == 0) {
    if (!isinf(kmn)) {
      atomicMin(&stats[s].kmin, dkey(kmn));
      atomicMax(&stats[s].kmax, dkey(kmx));
    }
    if (flags) atomicOr(&stats[s].flags, flags);
    if (tsing > -INF) atomicMax(&stats[s].tsingle, dkey(tsing));
    atomicAdd(&stats[s].priced_b, scanned);
  }
  __syncthreads();
  if (threadIdx.x < kSmallBmWords && s_bm[threadIdx.x])
    atomicOr(&small_bm[(size_t)s * kSmallBmWords + threadIdx.x], s_bm[threadIdx.x]);
  // raw-candidate capacity (only sizes the band fallback's raw mode): the
  // segment's band entries bound its feasible slices
  if (threadIdx.x == 0) stats[s].nraw = (unsigned long long)stats[s].band;
}

}  // namespace

cudaError_t launch_gtab_need(const int64_t* seg_off, const int* blk_base, int n_seg, int total_blocks,
                             int max_blocks, const int* blk_W, const double* in_d, int* need, cudaStream_t st) {
  if (n_seg > 0 && max_blocks <= kNeedMaxBlocks) {
    const size_t smem = (size_t)3 * max_blocks * sizeof(int);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(gtab_need_runs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // (long segments: 32 warps to hide the dependent bisection loads, as gtab_bins_kernel)
    gtab_need_runs_kernel<<<n_seg, max_blocks >= 128 ? 1024 : 256, smem, st>>>(seg_off, blk_base, blk_W, in_d, need);
    return cudaGetLastError();
  }
  const int blocks = std::max(1, std::min((total_blocks + 7) / 8, 148 * 16));
  gtab_need_kernel<<<blocks, 256, 0, st>>>(seg_off, blk_base, n_seg, total_blocks, blk_W, in_d, need);
  return cudaGetLastError();
}

cudaError_t launch_gtab_offsets(const int* need, int nK, int64_t* row_off, long long* total, cudaStream_t st) {
  gtab_offsets_kernel<<<1, 1024, 0, st>>>(need, nK, row_off, total);
  return cudaGetLastError();
}

cudaError_t launch_gtab_fill(const CostGrid& g, double cap, const AxisPos* mbp, int nK, const int* need,
                             const int64_t* row_off, double* G, double* G1, cudaStream_t st) {
  const int blocks = std::max(1, std::min((nK + kGWarps - 1) / kGWarps, 148 * 8));
  if (g.lay_class == kLayDec1)
    gtab_fill_kernel<kLayDec1><<<blocks, 32 * kGWarps, 0, st>>>(g, cap, mbp, nK, need, row_off, G, G1);
  else
    gtab_fill_kernel<kLayEncDec2><<<blocks, 32 * kGWarps, 0, st>>>(g, cap, mbp, nK, need, row_off, G, G1);
  return cudaGetLastError();
}

cudaError_t launch_gtab_gbase(const double* in_d, int64_t total, const int64_t* row_off, int* gbase,
                              cudaStream_t st) {
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
  gtab_gbase_kernel<<<blocks, 256, 0, st>>>(in_d, total, row_off, gbase);
  return cudaGetLastError();
}

cudaError_t launch_gtab_bins(const int64_t* seg_off, int n_seg, const double* in_d, const int* gbase,
                             const int* need, const double* G, double interval, const double* tau,
                             unsigned int* small_bm, SegStats* stats, int nK, const int64_t* row_off, int* rf,
                             double* rlo, int max_n, cudaStream_t st) {
  if (rf) {
    const int blocks = std::max(1, std::min((nK + kGWarps - 1) / kGWarps, 148 * 8));
    gtab_rowinfo_kernel<<<blocks, 32 * kGWarps, 0, st>>>(nK, need, row_off, G, interval, rf, rlo);
  }
  // long segments take 32 warps (C3: 0.15 -> 0.11 ms per 296); short ones 8
  // (C1's 256-sample segments were slower at 32)
  if (n_seg > 0)
    gtab_bins_kernel<<<n_seg, max_n >= 4096 ? kBinsThreads : 256, 0, st>>>(seg_off, in_d, gbase, need, G, interval,
                                                                           tau, small_bm, stats, rf, rlo);
  return cudaGetLastError();
}

}  // namespace ppb
