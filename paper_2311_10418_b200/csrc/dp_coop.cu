// dp_coop.cu — one DP pass spread over the whole GPU, for mini-batches too
// long for one CTA (BASELINE config C5: 65,536 samples, no memory cap, so
// every row is up to n columns wide and a pass is ~2.1 G transitions).
//
// Same recurrence, tie rules and results as dp_pass_kernel (dp.cu; reference
// run_suffix_dp, src/microbatch.cpp:162-189).  A cooperative launch of G
// CTAs walks the 32-row blocks; iteration b:
//   * CTA 0, warp 0 (the chain): folds block b's partials and runs the
//     32-step in-block triangle (shuffle broadcast of each newly final row),
//     then publishes the block's states to global memory (L2);
//   * CTA 0, warps 1..7: block b's near-far columns [nb, 64) and the fold of
//     the far-far partials the other CTAs produced for block b;
//   * CTAs 1..G-1: the far-far columns [64, W) of block b+1, whose states
//     (rows of blocks <= b-1) are final, one contiguous column range per
//     warp, folded per CTA into one partial per row;
//   * one grid-wide barrier.
// States live in an L2-resident global array (read with ld.global.cg: they
// are written by CTA 0 on another SM); the band tiles are read straight from
// HBM, coalesced (a tile column is 256 contiguous bytes).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "pp_internal.cuh"

namespace cg = cooperative_groups;

namespace ppb {

namespace {

constexpr int kCoopWarps = 8;
constexpr int kCoopThreads = 32 * kCoopWarps;

struct Acc {
  double s;  // MODE 0: sum; MODE 1: min sum
  double m;  // MODE 1: minimax
  int c;     // MODE 0: count
  int j;     // MODE 0: argmin j (lowest on ties)
};

__device__ __forceinline__ Acc acc_id() {
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  return Acc{INF, INF, 0, INT_MAX};
}

// full lexicographic merge (order-free)
template <int MODE>
__device__ __forceinline__ void merge(Acc& a, const Acc& b) {
  if (MODE == 0) {
    const bool tk = b.s < a.s || (b.s == a.s && (b.c < a.c || (b.c == a.c && b.j < a.j)));
    if (tk) a = b;
  } else {
    a.s = (b.s < a.s) ? b.s : a.s;
    a.m = (b.m < a.m) ? b.m : a.m;
  }
}

// one column (x = T[i, j]) into an accumulator scanning ascending j
template <int MODE>
__device__ __forceinline__ void take(Acc& a, double x, int j, double sj, int cj, double mj, double t) {
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double cs = __dadd_rn(x, sj);
  if (MODE == 0) {
    const int cn = 1 + cj;
    const bool upd = (x <= t) & ((cs < a.s) | ((cs == a.s) & (cn < a.c)));
    a.s = upd ? cs : a.s;
    a.c = upd ? cn : a.c;
    a.j = upd ? j : a.j;
  } else {
    const bool ok = !isnan(x);
    a.s = (ok & (cs < a.s)) ? cs : a.s;
    const double v = (x < mj) ? mj : x;
    a.m = (ok & (x < INF) & (mj < INF) & (v < a.m)) ? v : a.m;
  }
}

template <int MODE, bool SANITIZE>
__global__ void __launch_bounds__(kCoopThreads, 1)
    dp_coop_kernel(WorkItem it, const int64_t* __restrict__ seg_off, const int* __restrict__ blk_base,
                   const int* __restrict__ blk_W, const int64_t* __restrict__ tile_off,
                   const int64_t* __restrict__ seg_band_base, const double* __restrict__ band,
                   const double* __restrict__ cand, const int64_t* __restrict__ cand_off,
                   ItemResult* __restrict__ res, int res_slot, int* __restrict__ next_buf,
                   double* __restrict__ gstate, Acc* __restrict__ parts /* [2][G][32] */) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Acc s_part[kCoopWarps][32];
  const int s = it.seg;
  const int64_t b0 = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b0);
  const int gb0 = blk_base[s];
  const int nblk = blk_base[s + 1] - gb0;
  const double t = item_t(it, cand, cand_off);
  const double* bseg = band + seg_band_base[s];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int G = gridDim.x;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);
  // state: S[j] (sum), X[j] (count as int bits, or minimax) for j in [0, n]
  double* S = gstate + it.state_off;
  double* X = S + (n + 1);
  int* nxt = next_buf + it.next_off;
  auto ldS = [&](int j) { return __ldcg(S + j); };
  auto ldX = [&](int j) { return __ldcg(X + j); };
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S[n] = 0.0;  // state[n] = {0.0, 0} (microbatch.cpp:174)
    X[n] = MODE == 0 ? __longlong_as_double(0) : -INF;
  }
  grid.sync();
  double row0_s = INF, row0_x = MODE == 0 ? 0.0 : INF;

  for (int b = 0; b < nblk; ++b) {
    const int i1 = n - kRB * b;
    const int i0 = max(0, i1 - kRB);
    const int nb = i1 - i0;
    const int W = blk_W[gb0 + b];
    const double* tile = bseg + tile_off[gb0 + b];
    const int r = lane;
    if (blockIdx.x == 0) {
      // ---- CTA 0: near-far + fold of the far-far CTA partials, then the chain
      if (wid > 0) {
        Acc a = acc_id();
        // near-far columns [nb, min(64, W)): warp w takes nb + (w-1), +7, ...
        const int cnf = min(64, W);
        for (int c = nb + (wid - 1); c < cnf; c += kCoopWarps - 1) {
          const int j = i0 + c;
          const double x = tile[(size_t)c * kRB + r];
          const double xs = ldS(j), xx = ldX(j);
          take<MODE>(a, x, j, xs, __double_as_longlong(xx) & 0xffffffff, xx, t);
        }
        // far-far partials of block b from CTAs 1..G-1 (iteration b-1),
        // four independent L2 loads in flight per step
        if (b > 0) {
          const Acc* pp = parts + (size_t)(b & 1) * G * kRB;
          const int step = kCoopWarps - 1;
          int g = wid;
          for (; g + 3 * step < G; g += 4 * step) {
            const Acc p0 = pp[(size_t)g * kRB + r], p1 = pp[(size_t)(g + step) * kRB + r];
            const Acc p2 = pp[(size_t)(g + 2 * step) * kRB + r], p3 = pp[(size_t)(g + 3 * step) * kRB + r];
            merge<MODE>(a, p0);
            merge<MODE>(a, p1);
            merge<MODE>(a, p2);
            merge<MODE>(a, p3);
          }
          for (; g < G; g += step) merge<MODE>(a, pp[(size_t)g * kRB + r]);
        }
        s_part[wid][r] = a;
      }
      __syncthreads();
      if (wid == 0) {
        Acc a = acc_id();
#pragma unroll
        for (int w = 1; w < kCoopWarps; ++w) merge<MODE>(a, s_part[w][r]);
        // in-block triangle: T[i0 + r, i0 + jj] for jj in (r, nb)
        double tn[kRB];
#pragma unroll
        for (int jj = 0; jj < kRB; ++jj) tn[jj] = (jj < W) ? tile[(size_t)jj * kRB + r] : QNAN;
        double as = a.s, am = a.m;
        int ac = a.c, aj = a.j;
        if (r >= nb) {
          as = INF;
          ac = 0;
          am = INF;
        }
#pragma unroll
        for (int jj = kRB - 1; jj >= 0; --jj) {
          if (jj < nb) {
            double sj = __shfl_sync(0xffffffffu, as, jj);
            if (SANITIZE) sj = isfinite(sj) ? sj : INF;
            const double x = tn[jj];
            const double cs = __dadd_rn(x, sj);
            const bool ok = (r < jj) & (MODE == 0 ? (x <= t) : !isnan(x));
            if (MODE == 0) {
              const int cn = 1 + __shfl_sync(0xffffffffu, ac, jj);
              const bool upd = ok & ((cs < as) | ((cs == as) & (cn <= ac)));
              as = upd ? cs : as;
              ac = upd ? cn : ac;
              aj = upd ? i0 + jj : aj;
            } else {
              const double mj = __shfl_sync(0xffffffffu, am, jj);
              as = (ok & (cs < as)) ? cs : as;
              const double v = (x < mj) ? mj : x;
              am = (ok & (x < INF) & (mj < INF) & (v < am)) ? v : am;
            }
          }
        }
        if (r < nb) {
          const int row = i0 + r;
          const bool f = isfinite(as);
          __stcg(S + row, (SANITIZE && !f) ? INF : as);
          if (MODE == 0) {
            __stcg(X + row, __longlong_as_double(f ? ac : 0));
            nxt[row] = f ? aj : -1;
          } else {
            __stcg(X + row, am);
          }
          if (row == 0) {
            row0_s = as;
            row0_x = MODE == 0 ? (double)ac : am;
          }
        }
      }
    } else if (b + 1 < nblk) {
      // ---- CTAs 1..G-1: far-far columns [64, W') of block b+1
      const int bn = b + 1;
      const int j1 = n - kRB * bn;
      const int k0 = max(0, j1 - kRB);
      const int Wn = blk_W[gb0 + bn];
      const double* tn_ = bseg + tile_off[gb0 + bn];
      const int nw = (G - 1) * kCoopWarps;
      const int gw = (blockIdx.x - 1) * kCoopWarps + wid;
      const int ncol = max(Wn - 64, 0);
      const int per = (ncol + nw - 1) / nw;
      const int c_lo = 64 + gw * per, c_hi = min(Wn, c_lo + per);
      Acc a = acc_id();
      for (int c = c_lo; c < c_hi; ++c) {
        const int j = k0 + c;
        const double x = tn_[(size_t)c * kRB + r];
        const double xs = ldS(j), xx = ldX(j);
        take<MODE>(a, x, j, xs, __double_as_longlong(xx) & 0xffffffff, xx, t);
      }
      s_part[wid][r] = a;
      __syncthreads();
      if (wid == 0) {
#pragma unroll
        for (int w = 1; w < kCoopWarps; ++w) merge<MODE>(a, s_part[w][r]);
        parts[((size_t)(bn & 1) * G + blockIdx.x) * kRB + r] = a;
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ItemResult rr;
    rr.sum0 = row0_s;
    rr.count0 = MODE == 0 ? (int)row0_x : 0;
    rr.feasible = isfinite(row0_s) ? 1 : 0;
    rr.aux = MODE == 1 ? row0_x : 0.0;
    res[res_slot] = rr;
  }
}

}  // namespace

// Bytes of global scratch one cooperative pass needs besides its state.
size_t dp_coop_parts_bytes(int grid) { return (size_t)2 * grid * kRB * sizeof(Acc); }

// Grid size of the cooperative pass on `device` (one CTA per SM).
int dp_coop_grid(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return std::max(sms, 2);
}

cudaError_t launch_dp_coop(int mode, int sanitize, const WorkItem& it, int grid, const int64_t* seg_off,
                           const int* blk_base, const int* blk_W, const int64_t* tile_off,
                           const int64_t* seg_band_base, const double* band, const double* cand,
                           const int64_t* cand_off, ItemResult* res, int res_slot, int* next_buf,
                           double* gstate, void* parts, cudaStream_t st) {
  WorkItem w = it;
  Acc* pa = static_cast<Acc*>(parts);
  void* args[] = {&w,        &seg_off,  &blk_base, &blk_W,    &tile_off, &seg_band_base, &band,
                  &cand,     &cand_off, &res,      &res_slot, &next_buf, &gstate,        &pa};
  const void* fn;
  if (mode == 0)
    fn = sanitize ? (const void*)dp_coop_kernel<0, true> : (const void*)dp_coop_kernel<0, false>;
  else
    fn = sanitize ? (const void*)dp_coop_kernel<1, true> : (const void*)dp_coop_kernel<1, false>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kCoopThreads), args, 0, st);
}

}  // namespace ppb
