// cost.cu — fused slice costing on sm_100a: the triangular slice tables the
// reference builds with n(n+1)/2 std::function calls (microbatch.cpp:228-243),
// produced on the device as a compact *band*.
//
// Pass A (row_scan_kernel): one warp per row i scans every j in (i, n],
//   prices the slice [i, j) bit-exactly (pp_internal.cuh::slice_cost, the
//   make_slice_cost lambda microbatch.cpp:136-158 + estimate cost_model.cpp:294-319),
//   and records
//     - the last memory-feasible end  Rm(i) = max{ j : !(M[i,j] > cap) }
//     - singleton infeasibility (microbatch.cpp:245-251)
//     - candidate statistics (microbatch.cpp:253-269).
//   The padded maxima are running maxima along the row (warp max-scan), so
//   unsorted spans are priced exactly like the reference's O(j-i) loop.
// Row offsets (row_offsets_kernel): per-segment exclusive scan of widths.
// Pass B (band_kernel): rewrites T for j in (i, Rm(i)] into the band; slices
//   with M > cap become NaN (never pass `T <= t_max`).  Candidate values are
//   set in a per-segment bitmap over k = ceil(T / I) or, for the exact mode
//   (I == 0) or very wide k ranges, appended for a segmented sort.
// Candidate compaction (cand_bitmap_kernel / cand_unique_kernel): ascending,
//   unique candidate t_max list per segment.
//
// Every slice outside (i, Rm(i)] has M > cap, so the DP never needs it: the
// band carries every slice the reference's DP can use, nothing is assumed
// about monotonicity of the cost model.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "pp_internal.cuh"

namespace ppb {

__device__ __forceinline__ int seg_of_row(const int64_t* seg_off, int n_seg, int64_t r) {
  int lo = 0, hi = n_seg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_off[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Stage the (small) grid tables in shared memory.
__device__ __forceinline__ GridDev stage_grid(const GridDev& g, double* sm, Layout* sl) {
  const int nm = g.n_mbs, ns = g.n_seq, nc = 2 * nm * ns * 3;
  for (int k = threadIdx.x; k < nm; k += blockDim.x) sm[k] = g.mbs_ax[k];
  for (int k = threadIdx.x; k < ns; k += blockDim.x) sm[nm + k] = g.seq_ax[k];
  for (int k = threadIdx.x; k < nc; k += blockDim.x) sm[nm + ns + k] = g.cells[k];
  for (int k = threadIdx.x; k < g.n_layouts; k += blockDim.x) sl[k] = g.layouts[k];
  __syncthreads();
  GridDev s = g;
  s.mbs_ax = sm;
  s.seq_ax = sm + nm;
  s.cells = sm + nm + ns;
  s.layouts = sl;
  return s;
}

__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }

// Inclusive warp max-scan.
__device__ __forceinline__ double warp_max_scan(double x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = dmax(x, y);
  }
  return x;
}

// kTable: slice costs come from host-evaluated triangular tables (the generic
// SliceCostFn path, microbatch.cpp:237-243) instead of the fused grid coster.
template <bool kBand, bool kTable>
__global__ void __launch_bounds__(256)
    row_kernel(GridDev g, int stage, const double* __restrict__ tabT, const double* __restrict__ tabM, const double* __restrict__ in_d, const double* __restrict__ tgt_d,
               const int64_t* __restrict__ seg_off, int n_seg, int64_t total_rows, double cap,
               double interval, int* __restrict__ row_w, SegStats* __restrict__ stats,
               const int64_t* __restrict__ row_off, const int64_t* __restrict__ seg_band_base,
               double* __restrict__ band, unsigned int* __restrict__ bitmap,
               const int64_t* __restrict__ bitmap_off, const int* __restrict__ seg_mode,
               unsigned long long* __restrict__ cand_raw, const int64_t* __restrict__ cand_raw_off,
               unsigned long long* __restrict__ cand_raw_cnt) {
  extern __shared__ __align__(16) double sm_grid[];
  __shared__ Layout sm_lay[kMaxLayouts];
  // Small grids (every realistic profile: 648 cells) are staged in shared
  // memory; oversized ones are read through L1 from global memory.
  const GridDev G = stage ? stage_grid(g, sm_grid, sm_lay) : g;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < total_rows;
       r += warps) {
    const int s = seg_of_row(seg_off, n_seg, r);
    const int64_t b = seg_off[s];
    const int n = (int)(seg_off[s + 1] - b);
    const int i = (int)(r - b);
    int jend = n;
    if (kBand) jend = i + row_w[r];
    double cin = 0.0, ctg = 0.0;  // shape.input_len = 0 / target_len = 0 (:143-144)
    int last_ok = i;
    double kmn = __longlong_as_double(0x7ff0000000000000LL), kmx = -kmn;  // +inf / -inf
    unsigned long long nraw = 0;
    int flags = 0;
    double* brow = nullptr;
    int mode = 0;
    if (kBand) {
      brow = band + seg_band_base[s] + row_off[r] - (i + 1);
      mode = seg_mode[s];
    }
    for (int j0 = i + 1; j0 <= jend; j0 += 32) {
      const int j = j0 + lane;
      const bool valid = j <= jend;
      double xi = -__longlong_as_double(0x7ff0000000000000LL), xt = xi;
      if (valid && !kTable) {
        xi = in_d[b + j - 1];
        xt = tgt_d[b + j - 1];
      }
      const double pin = dmax(cin, warp_max_scan(xi, lane));
      const double ptg = dmax(ctg, warp_max_scan(xt, lane));
      cin = __shfl_sync(0xffffffffu, pin, 31);
      ctg = __shfl_sync(0xffffffffu, ptg, 31);
      double T = 0.0, M = 0.0;
      bool ok = false;
      if (valid) {
        if (kTable) {
          const int64_t idx = (int64_t)i * n - (int64_t)i * (i - 1) / 2 + (j - i - 1);
          T = tabT[idx];
          M = tabM[idx];
        } else {
          slice_cost(G, (double)(j - i), pin, ptg, T, M);
        }
        ok = !(M > cap);
        if (!kBand) {
          if (ok) last_ok = j;
          if (j == i + 1 && !ok) atomicMin(&stats[s].err_row, i);
        } else {
          brow[j] = ok ? T : masked();
        }
      }
      const bool is_cand = valid && ok && !isnan(T);
      double q = T;
      if (is_cand && interval > 0) q = ceil(__ddiv_rn(T, interval));
      if (!kBand) {
        if (is_cand) {
          ++nraw;
          if (isinf(q)) flags |= (q > 0) ? 1 : 2;
          else {
            kmn = (q < kmn) ? q : kmn;
            kmx = (kmx < q) ? q : kmx;
          }
        }
      } else if (mode == 0) {  // bitmap over k
        const bool fin = is_cand && !isinf(q);
        long long bit = -1;
        if (fin) bit = (long long)(q - dkey_inv(stats[s].kmin));
        const long long prev = __shfl_up_sync(0xffffffffu, bit, 1);
        if (fin && (lane == 0 || prev != bit))
          atomicOr(&bitmap[bitmap_off[s] + (bit >> 5)], 1u << (bit & 31));
      } else if (mode == 1) {  // raw list for the segmented sort (mode 2: c == 1, no candidates)
        const unsigned int m = __ballot_sync(0xffffffffu, is_cand);
        unsigned long long base = 0;
        if (lane == 0 && m) base = atomicAdd(&cand_raw_cnt[s], (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (is_cand) {
          const double qq = interval > 0 ? __dmul_rn(q, interval) : T;
          cand_raw[cand_raw_off[s] + base + __popc(m & ((1u << lane) - 1))] = dkey(qq);
        }
      }
    }
    if (!kBand) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        last_ok = max(last_ok, __shfl_xor_sync(0xffffffffu, last_ok, o));
        const double a = __shfl_xor_sync(0xffffffffu, kmn, o);
        const double c = __shfl_xor_sync(0xffffffffu, kmx, o);
        kmn = (a < kmn) ? a : kmn;
        kmx = (kmx < c) ? c : kmx;
        nraw += __shfl_xor_sync(0xffffffffu, nraw, o);
        flags |= __shfl_xor_sync(0xffffffffu, flags, o);
      }
      if (lane == 0) {
        row_w[r] = last_ok - i;
        if (nraw) {
          atomicAdd(&stats[s].nraw, nraw);
          if (!isinf(kmn)) {
            atomicMin(&stats[s].kmin, dkey(kmn));
            atomicMax(&stats[s].kmax, dkey(kmx));
          }
        }
        if (flags) atomicOr(&stats[s].flags, flags);
      }
    }
  }
}

// Per-segment exclusive scan of the row widths -> band offsets.
__global__ void __launch_bounds__(1024)
    row_offsets_kernel(const int* __restrict__ row_w, const int64_t* __restrict__ seg_off,
                       int64_t* __restrict__ row_off, SegStats* __restrict__ stats) {
  __shared__ long long warp_tot[32];
  const int s = blockIdx.x;
  const int64_t b = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long carry = 0;
  for (int t0 = 0; t0 < n; t0 += blockDim.x) {
    const int k = t0 + threadIdx.x;
    const long long v = k < n ? row_w[b + k] : 0;
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
    if (k < n) row_off[b + k] = carry + before + x - v;
    carry += warp_tot[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) stats[s].band = carry;
}

// Bitmap -> ascending candidate list (k * I), with the +/-inf flags.
__global__ void __launch_bounds__(1024)
    cand_bitmap_kernel(const unsigned int* __restrict__ bitmap, const int64_t* __restrict__ bitmap_off,
                       const SegStats* __restrict__ stats, const int* __restrict__ seg_mode,
                       double interval, const int64_t* __restrict__ cand_off,
                       double* __restrict__ cand, int* __restrict__ cand_n) {
  __shared__ int warp_tot[32];
  const int s = blockIdx.x;
  if (seg_mode[s] != 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nw = bitmap_off[s + 1] - bitmap_off[s];
  const unsigned int* bm = bitmap + bitmap_off[s];
  double* out = cand + cand_off[s];
  const SegStats st = stats[s];
  int carry = 0;
  if (st.flags & 2) carry = 1;  // -inf first
  if (threadIdx.x == 0 && (st.flags & 2)) out[0] = -__longlong_as_double(0x7ff0000000000000LL);
  const double kmin = st.nraw && st.kmin != ~0ULL ? dkey_inv(st.kmin) : 0.0;
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
      out[pos++] = __dmul_rn(kk, interval);             // ceil(t / I) * I (:264)
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
// doubles (so -0.0 and +0.0 collapse, keeping the first), one CTA per segment.
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

// ---------------------------------------------------------------- launchers
static size_t grid_smem(const GridDev& g) {
  return sizeof(double) * ((size_t)g.n_mbs + g.n_seq + 2 * (size_t)g.n_mbs * g.n_seq * 3);
}
static bool grid_fits(const GridDev& g) {
  return grid_smem(g) <= 160 * 1024 && g.n_layouts <= kMaxLayouts;
}

cudaError_t launch_row_scan(const GridDev& g, const double* tabT, const double* tabM,
                            const double* in_d, const double* tgt_d,
                            const int64_t* seg_off, int n_seg, int64_t total_rows, double cap,
                            double interval, int* row_w, SegStats* stats, cudaStream_t st) {
  const int stage = grid_fits(g) ? 1 : 0;
  const size_t sm = stage ? grid_smem(g) : 0;
  const int64_t blocks = std::max<int64_t>(std::min<int64_t>((total_rows + 7) / 8, 148 * 64), 1);
  if (tabT) {
    row_kernel<false, true><<<(int)blocks, 256, 0, st>>>(
        g, 0, tabT, tabM, in_d, tgt_d, seg_off, n_seg, total_rows, cap, interval, row_w, stats,
        nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    return cudaGetLastError();
  }
  cudaFuncSetAttribute(row_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  row_kernel<false, false><<<(int)blocks, 256, sm, st>>>(
      g, stage, nullptr, nullptr, in_d, tgt_d, seg_off, n_seg, total_rows, cap, interval, row_w, stats, nullptr, nullptr,
      nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_row_offsets(const int* row_w, const int64_t* seg_off, int n_seg, int64_t* row_off,
                               SegStats* stats, cudaStream_t st) {
  row_offsets_kernel<<<n_seg, 1024, 0, st>>>(row_w, seg_off, row_off, stats);
  return cudaGetLastError();
}

cudaError_t launch_band(const GridDev& g, const double* tabT, const double* tabM, const double* in_d, const double* tgt_d,
                        const int64_t* seg_off, int n_seg, int64_t total_rows, double cap,
                        double interval, int* row_w, SegStats* stats, const int64_t* row_off,
                        const int64_t* seg_band_base, double* band, unsigned int* bitmap,
                        const int64_t* bitmap_off, const int* seg_mode,
                        unsigned long long* cand_raw, const int64_t* cand_raw_off,
                        unsigned long long* cand_raw_cnt, cudaStream_t st) {
  const int stage = grid_fits(g) ? 1 : 0;
  const size_t sm = stage ? grid_smem(g) : 0;
  const int64_t blocks = std::max<int64_t>(std::min<int64_t>((total_rows + 7) / 8, 148 * 64), 1);
  if (tabT) {
    row_kernel<true, true><<<(int)blocks, 256, 0, st>>>(
        g, 0, tabT, tabM, in_d, tgt_d, seg_off, n_seg, total_rows, cap, interval, row_w, stats,
        row_off, seg_band_base, band, bitmap, bitmap_off, seg_mode, cand_raw, cand_raw_off,
        cand_raw_cnt);
    return cudaGetLastError();
  }
  cudaFuncSetAttribute(row_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  row_kernel<true, false><<<(int)blocks, 256, sm, st>>>(
      g, stage, nullptr, nullptr, in_d, tgt_d, seg_off, n_seg, total_rows, cap, interval, row_w, stats, row_off,
      seg_band_base, band, bitmap, bitmap_off, seg_mode, cand_raw, cand_raw_off, cand_raw_cnt);
  return cudaGetLastError();
}

cudaError_t launch_cand_bitmap(const unsigned int* bitmap, const int64_t* bitmap_off,
                               const SegStats* stats, const int* seg_mode, int n_seg,
                               double interval, const int64_t* cand_off, double* cand, int* cand_n,
                               cudaStream_t st) {
  cand_bitmap_kernel<<<n_seg, 1024, 0, st>>>(bitmap, bitmap_off, stats, seg_mode, interval, cand_off,
                                             cand, cand_n);
  return cudaGetLastError();
}

cudaError_t launch_cand_unique(const unsigned long long* keys_a, const unsigned long long* keys_b,
                               const int* in_b, const int64_t* raw_off,
                               const unsigned long long* raw_cnt, const int* seg_mode, int n_seg,
                               const int64_t* cand_off, double* cand, int* cand_n, cudaStream_t st) {
  cand_unique_kernel<<<n_seg, 1024, 0, st>>>(keys_a, keys_b, in_b, raw_off, raw_cnt, seg_mode, cand_off, cand, cand_n);
  return cudaGetLastError();
}

}  // namespace ppb
