// dp.cu — the suffix DP of dp_partition on sm_100a, one CTA per
// (mini-batch, t_max candidate), plus the per-mini-batch candidate selection.
//
// Reference: run_suffix_dp (src/microbatch.cpp:162-189), the candidate loop
// (:281-318), reconstruct_splits (:194-215) and assembly (:322-335).
//
// Row recurrence for a candidate t (state[n] = (0, 0)):
//   state[i] = lexmin over j in (i, n] with  T[i,j] <= t, M[i,j] <= cap,
//              state[j] finite  of  (T[i,j] + state[j].sum, 1 + state[j].count)
// with the reference's strict-improvement rule, i.e. the lowest j among equal
// (sum, count) pairs; that j is recorded as next[i].  next[] then *is* the
// reference's reconstruct_splits: its front-to-back scan picks the smallest j
// with T + state[j].sum == state[i].sum && 1 + state[j].count == state[i].count,
// which is exactly the lowest-index argmin of the row.
//
// Only finite sums can ever be taken (inf/NaN sums fail both `<` and the
// count tie-break against the initial (inf, 0)), so the parallel reduction
// uses only finite candidates; lexmin over (sum, count, j) is associative and
// commutative, so any reduction order gives the reference's answer.
//
// Blocking (the CTA's schedule; never changes results): rows are processed
// top-down in blocks of 32.  For a block [i0, i0+32):
//   phase 1 (all 8 warps): the "far" transitions j >= i0+32, whose states are
//     final, reduced per row with warp shuffles;
//   phase 2 (warp 0, lane r <-> row i0+r): the in-block triangle.  Walking
//     jj = 31..0, lane jj finalises its row, broadcasts (sum, count) with two
//     shuffles and the lanes below fold T[i0+r, i0+jj] + state into their
//     accumulators (descending j, so equal pairs take the lower j).
// The band gives T for j in (i, Rm(i)] (cost.cu), NaN where M > cap.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "pp_internal.cuh"

namespace ppb {

constexpr int kDpThreads = 256;
constexpr int kBlk = 32;

__device__ __forceinline__ bool isfin(double x) { return isfinite(x); }

struct Acc {
  double s;
  int c;
  int j;
};

// (s, c, j) lexmin with lowest-j ties.
__device__ __forceinline__ bool better(double s1, int c1, int j1, const Acc& a) {
  if (s1 < a.s) return true;
  if (s1 == a.s) {
    if (c1 < a.c) return true;
    if (c1 == a.c && j1 < a.j) return true;
  }
  return false;
}

// MODE 0: candidate pass.  MODE 1: bound pass (t = +inf, sum only) fused with
// the minimax pass that yields the feasibility threshold t*.
template <int MODE>
__global__ void __launch_bounds__(kDpThreads)
    dp_pass_kernel(const WorkItem* __restrict__ items, const int64_t* __restrict__ seg_off,
                   const int* __restrict__ row_w, const int64_t* __restrict__ row_off,
                   const int64_t* __restrict__ seg_band_base, const double* __restrict__ band,
                   const double* __restrict__ cand, const int64_t* __restrict__ cand_off,
                   ItemResult* __restrict__ res, int* __restrict__ next_buf,
                   double* __restrict__ gstate) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double p_s[kBlk];
  __shared__ double p_m[kBlk];
  __shared__ int p_c[kBlk];
  __shared__ int p_j[kBlk];
  const WorkItem it = items[blockIdx.x];
  const int64_t b = seg_off[it.seg];
  const int n = (int)(seg_off[it.seg + 1] - b);
  const double t = item_t(it, cand, cand_off);
  double* st_s;  // state sums  [n+1]
  int* st_c;     // MODE 0: counts [n+1];  MODE 1: aliases st_m
  double* st_m;  // MODE 1: minimax [n+1]
  if (it.state_off < 0) {
    st_s = reinterpret_cast<double*>(smem);
    st_m = st_s + (n + 1);
  } else {
    st_s = gstate + it.state_off;
    st_m = st_s + (n + 1);
  }
  st_c = reinterpret_cast<int*>(st_m);
  int* nxt = next_buf + it.next_off;
  const double* bseg = band + seg_band_base[it.seg];
  const int* wseg = row_w + b;
  const int64_t* oseg = row_off + b;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);

  if (threadIdx.x == 0) {
    st_s[n] = 0.0;  // state[n] = {0.0, 0} (microbatch.cpp:174)
    if (MODE == 0) st_c[n] = 0; else st_m[n] = -INF;
  }
  __syncthreads();

  for (int top = n; top > 0; top -= kBlk) {
    const int i0 = max(0, top - kBlk);
    const int nb = top - i0;
    // ---- phase 1: far transitions j in [top, i + w(i)] ----
    for (int r = wid; r < nb; r += kDpThreads / 32) {
      const int i = i0 + r;
      const int jmax = i + wseg[i];
      const double* brow = bseg + oseg[i] - (i + 1);
      Acc a{INF, 0, 0x7fffffff};
      double mm = INF;
      for (int j = top + lane; j <= jmax; j += 32) {
        const double x = brow[j];
        const double sj = st_s[j];
        if (MODE == 0) {
          if (x <= t && isfin(sj)) {
            const double cs = __dadd_rn(x, sj);
            const int cc = 1 + st_c[j];
            if (isfin(cs) && better(cs, cc, j, a)) a = Acc{cs, cc, j};
          }
        } else {
          if (!isnan(x)) {
            if (isfin(sj)) {
              const double cs = __dadd_rn(x, sj);
              if (isfin(cs) && cs < a.s) a.s = cs;
            }
            const double mj = st_m[j];
            if (x < INF && mj < INF) {
              const double v = (x < mj) ? mj : x;
              mm = (v < mm) ? v : mm;
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, a.s, o);
        if (MODE == 0) {
          const int oc = __shfl_xor_sync(0xffffffffu, a.c, o);
          const int oj = __shfl_xor_sync(0xffffffffu, a.j, o);
          if (better(os, oc, oj, a)) a = Acc{os, oc, oj};
        } else {
          a.s = (os < a.s) ? os : a.s;
          const double om = __shfl_xor_sync(0xffffffffu, mm, o);
          mm = (om < mm) ? om : mm;
        }
      }
      if (lane == 0) {
        p_s[r] = a.s;
        if (MODE == 0) {
          p_c[r] = a.c;
          p_j[r] = a.j;
        } else {
          p_m[r] = mm;
        }
      }
    }
    __syncthreads();
    // ---- phase 2: in-block triangle, serial over rows ----
    if (wid == 0) {
      const int i = i0 + lane;
      const bool row_ok = lane < nb;
      const int jmax = row_ok ? i + wseg[i] : -1;
      const double* brow = row_ok ? bseg + oseg[i] - (i + 1) : bseg;
      double tn[kBlk];
#pragma unroll
      for (int jj = 0; jj < kBlk; ++jj) {
        const int j = i0 + jj;
        tn[jj] = (row_ok && j > i && j <= jmax) ? brow[j] : __longlong_as_double(0x7ff8000000000000LL);
      }
      Acc a{INF, 0, 0x7fffffff};
      double mm = INF;
      if (row_ok) {
        a.s = p_s[lane];
        if (MODE == 0) {
          a.c = p_c[lane];
          a.j = p_j[lane];
        } else {
          mm = p_m[lane];
        }
      }
#pragma unroll
      for (int jj = kBlk - 1; jj >= 0; --jj) {
        if (jj < nb) {
          const double sj = __shfl_sync(0xffffffffu, a.s, jj);
          int cj = 0;
          double mj = 0.0;
          if (MODE == 0) cj = __shfl_sync(0xffffffffu, a.c, jj);
          else mj = __shfl_sync(0xffffffffu, mm, jj);
          if (lane == jj) {
            const int row = i0 + jj;
            if (MODE == 0) {
              const bool f = isfin(a.s);
              st_s[row] = f ? a.s : INF;
              st_c[row] = f ? a.c : 0;
              nxt[row] = f ? a.j : -1;
            } else {
              st_s[row] = a.s;
              st_m[row] = mm;
            }
          }
          if (lane < jj) {
            const double x = tn[jj];
            const int j = i0 + jj;
            if (MODE == 0) {
              if (x <= t && isfin(sj)) {
                const double cs = __dadd_rn(x, sj);
                const int cc = 1 + cj;
                // descending j: equal (sum, count) takes the lower j
                if (isfin(cs) && (cs < a.s || (cs == a.s && cc <= a.c))) a = Acc{cs, cc, j};
              }
            } else {
              if (!isnan(x)) {
                if (isfin(sj)) {
                  const double cs = __dadd_rn(x, sj);
                  if (isfin(cs) && cs < a.s) a.s = cs;
                }
                if (x < INF && mj < INF) {
                  const double v = (x < mj) ? mj : x;
                  mm = (v < mm) ? v : mm;
                }
              }
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ItemResult r;
    r.sum0 = st_s[0];
    r.count0 = MODE == 0 ? st_c[0] : 0;
    r.feasible = isfin(st_s[0]) ? 1 : 0;
    r.aux = MODE == 1 ? st_m[0] : 0.0;
    res[blockIdx.x] = r;
  }
}

// After the bound pass: record bound / t* and the first candidate >= t*.
__global__ void seg_init_kernel(const ItemResult* __restrict__ bound_res, int has_bound, int replicas,
                                const int64_t* __restrict__ cand_off, const int* __restrict__ cand_n,
                                const double* __restrict__ cand, const int* __restrict__ active,
                                SegDP* __restrict__ dp, int n_seg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  SegDP d;
  d.best_obj = __longlong_as_double(0x7ff0000000000000LL);
  d.best_t = 0.0;
  d.best_count = 0;
  d.valid = 0;
  d.n_cand = cand_n[s];
  d.ref_evals = 0;
  d.pad[0] = d.pad[1] = 0;
  if (!active[s]) {
    d.done = 1;
    d.next_cand = d.n_cand;
    d.bound = 0.0;
    d.tstar = 0.0;
    dp[s] = d;
    return;
  }
  d.done = 0;
  if (has_bound) {
    const ItemResult r = bound_res[s];
    d.bound = r.sum0 / (double)replicas;  // microbatch.cpp:278
    d.tstar = r.aux;
    // first candidate >= t*: every candidate below it is infeasible (no
    // partition keeps all slices <= t), so the reference only `continue`s
    // there (microbatch.cpp:292) before any best exists.
    const double* c = cand + cand_off[s];
    int lo = 0, hi = d.n_cand;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (c[mid] < d.tstar) lo = mid + 1; else hi = mid;
    }
    d.next_cand = lo;
  } else {
    d.bound = 0.0;
    d.tstar = -__longlong_as_double(0x7ff0000000000000LL);
    d.next_cand = 0;
  }
  if (d.next_cand >= d.n_cand) {
    d.done = 1;
    d.ref_evals = d.n_cand;
  }
  dp[s] = d;
}

// Lexicographic compare of two split vectors given as next[] chains from 0
// (std::vector<size_t> operator<, microbatch.cpp:304).  Same counts.
__device__ bool chain_less(const int* a, const int* bb, int n) {
  int i = 0, k = 0;
  while (i < n) {
    const int x = a[i], y = bb[k];
    if (x != y) return x < y;
    i = x;
    k = y;
  }
  return false;
}

// The candidate loop (microbatch.cpp:289-318) over this wave's items of one
// segment, in ascending t.  One CTA per segment.
__global__ void __launch_bounds__(256)
    select_kernel(const WorkItem* __restrict__ items, const ItemResult* __restrict__ res,
                  const int* __restrict__ seg_item_start, const int* __restrict__ seg_item_cnt,
                  const int* __restrict__ next_buf, int* __restrict__ best_next,
                  const int64_t* __restrict__ seg_off, const double* __restrict__ cand,
                  const int64_t* __restrict__ cand_off, int stage_count, int replicas,
                  SegDP* __restrict__ dps) {
  const int s = blockIdx.x;
  const int cnt = seg_item_cnt[s];
  if (cnt == 0) return;
  __shared__ SegDP d;
  __shared__ int copy_from;  // item index whose next[] becomes best (-1 none)
  const int64_t b = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b);
  int* bn = best_next + b;
  if (threadIdx.x == 0) d = dps[s];
  __syncthreads();
  const double ramp = (double)(stage_count - 1);
  const int first = seg_item_start[s];
  for (int k = 0; k < cnt; ++k) {
    const WorkItem it = items[first + k];
    if (threadIdx.x == 0) {
      copy_from = -1;
      const double tm = item_t(it, cand, cand_off);
      if (d.done) {
      } else if (d.valid && __dadd_rn(__dmul_rn(ramp, tm), d.bound) > d.best_obj) {  // :291
        d.done = 1;
        d.ref_evals = it.cand;
      } else {
        const ItemResult r = res[first + k];
        d.next_cand = it.cand + 1;
        if (r.feasible) {
          const double obj = __dadd_rn(stage_count > 1 ? __dmul_rn(ramp, tm) : 0.0,
                                       __ddiv_rn(r.sum0, (double)replicas));  // :293-294
          bool take = false;
          if (!d.valid || obj < d.best_obj) {
            take = true;
          } else if (obj == d.best_obj) {
            if (r.count0 < d.best_count) {
              take = true;
            } else if (r.count0 == d.best_count) {
              if (chain_less(next_buf + it.next_off, bn, n)) {  // :302-308
                copy_from = first + k;
                d.best_t = tm;
              }
            }
          }
          if (take) {
            d.best_obj = obj;
            d.best_count = r.count0;
            d.best_t = tm;
            d.valid = 1;
            copy_from = first + k;
          }
        }
      }
    }
    __syncthreads();
    if (copy_from >= 0) {
      const int* src = next_buf + items[copy_from].next_off;
      for (int q = threadIdx.x; q < n; q += blockDim.x) bn[q] = src[q];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (!d.done) {
      if (d.next_cand >= d.n_cand) {
        d.done = 1;
        d.ref_evals = d.n_cand;
      } else if (d.valid) {
        const double tn = cand[cand_off[s] + d.next_cand];
        if (__dadd_rn(__dmul_rn(ramp, tn), d.bound) > d.best_obj) {
          d.done = 1;
          d.ref_evals = d.next_cand;
        }
      }
    }
    dps[s] = d;
  }
}

// Assembly (microbatch.cpp:322-335): splits, per-micro-batch times,
// eval_objective (front-to-back, :109-120) and t_max_used.
__global__ void __launch_bounds__(256)
    finalize_kernel(const SegDP* __restrict__ dps, const int* __restrict__ best_next,
                    const int64_t* __restrict__ seg_off, const int* __restrict__ row_w,
                    const int64_t* __restrict__ row_off, const int64_t* __restrict__ seg_band_base,
                    const double* __restrict__ band, const SegStats* __restrict__ stats,
                    const pp_sample* __restrict__ ordered, int chain_in_smem, int stage_count, int replicas,
                    int32_t* __restrict__ splits, double* __restrict__ mb_times,
                    int32_t* __restrict__ count, double* __restrict__ t_max_used,
                    double* __restrict__ objective, int32_t* __restrict__ status,
                    int64_t* __restrict__ err_id) {
  extern __shared__ int chain[];
  const int s = blockIdx.x;
  const int64_t b = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b);
  const SegDP d = dps[s];
  if (n <= 0) {
    if (threadIdx.x == 0) {
      status[s] = PP_ERR_INVALID;
      count[s] = 0;
      err_id[s] = -1;
    }
    return;
  }
  const int err = stats[s].err_row;
  if (err != INT_MAX) {
    if (threadIdx.x == 0) {
      status[s] = PP_ERR_INFEASIBLE_SAMPLE;
      err_id[s] = ordered[b + err].id;
      count[s] = 0;
    }
    return;
  }
  if (!d.valid) {
    if (threadIdx.x == 0) {
      status[s] = PP_ERR_INFEASIBLE;
      err_id[s] = -1;
      count[s] = 0;
    }
    return;
  }
  const int* bn = best_next + b;
  const int* ch = bn;
  if (chain_in_smem) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) chain[q] = bn[q];
    __syncthreads();
    ch = chain;
  }
  if (threadIdx.x == 0) {
    const double* bseg = band + seg_band_base[s];
    int i = 0, m = 0;
    double max_t = 0.0, sum = 0.0;
    while (i < n) {
      const int j = ch[i];
      const double tt = bseg[row_off[b + i] + (j - i - 1)];
      splits[b + m] = j;
      mb_times[b + m] = tt;
      max_t = (max_t < tt) ? tt : max_t;
      sum = __dadd_rn(sum, tt);
      ++m;
      i = j;
    }
    count[s] = m;
    objective[s] = __dadd_rn(__dmul_rn((double)(stage_count - 1), max_t),
                             __ddiv_rn(sum, (double)replicas));
    t_max_used[s] = isfinite(d.best_t) ? d.best_t : max_t;
    status[s] = PP_OK;
    err_id[s] = -1;
  }
}

// ---------------------------------------------------------------- launchers
size_t dp_smem_bytes(int mode, int n) {
  // MODE 0: sums (8) + counts (4, aliased into the second array of 8)
  // MODE 1: sums (8) + minimax (8)
  (void)mode;
  return (size_t)(n + 1) * 16;
}

cudaError_t launch_dp_pass(int mode, const WorkItem* items, int n_items, size_t smem,
                           const int64_t* seg_off, const int* row_w, const int64_t* row_off,
                           const int64_t* seg_band_base, const double* band, const double* cand,
                           const int64_t* cand_off, ItemResult* res, int* next_buf, double* gstate,
                           cudaStream_t st) {
  if (n_items == 0) return cudaSuccess;
  if (mode == 0) {
    cudaFuncSetAttribute(dp_pass_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dp_pass_kernel<0><<<n_items, kDpThreads, smem, st>>>(items, seg_off, row_w, row_off,
                                                         seg_band_base, band, cand, cand_off, res, next_buf, gstate);
  } else {
    cudaFuncSetAttribute(dp_pass_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dp_pass_kernel<1><<<n_items, kDpThreads, smem, st>>>(items, seg_off, row_w, row_off,
                                                         seg_band_base, band, cand, cand_off, res, next_buf, gstate);
  }
  return cudaGetLastError();
}

cudaError_t launch_seg_init(const ItemResult* bound_res, int has_bound, int replicas,
                            const int64_t* cand_off, const int* cand_n, const double* cand,
                            const int* active, SegDP* dp, int n_seg, cudaStream_t st) {
  seg_init_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(bound_res, has_bound, replicas, cand_off,
                                                       cand_n, cand, active, dp, n_seg);
  return cudaGetLastError();
}

cudaError_t launch_select(const WorkItem* items, const ItemResult* res, const int* seg_item_start,
                          const int* seg_item_cnt, const int* next_buf, int* best_next,
                          const int64_t* seg_off, const double* cand, const int64_t* cand_off,
                          int stage_count, int replicas, SegDP* dps, int n_seg, cudaStream_t st) {
  select_kernel<<<n_seg, 256, 0, st>>>(items, res, seg_item_start, seg_item_cnt, next_buf, best_next,
                                       seg_off, cand, cand_off, stage_count, replicas, dps);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const SegDP* dps, const int* best_next, const int64_t* seg_off,
                            const int* row_w, const int64_t* row_off, const int64_t* seg_band_base,
                            const double* band, const SegStats* stats, const pp_sample* ordered,
                            int stage_count, int replicas, int max_n, int n_seg, int32_t* splits,
                            double* mb_times, int32_t* count, double* t_max_used, double* objective,
                            int32_t* status, int64_t* err_id, cudaStream_t st) {
  const int in_smem = (size_t)max_n * sizeof(int) <= 200 * 1024 ? 1 : 0;
  const size_t smem = in_smem ? (size_t)max_n * sizeof(int) : 0;
  cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  finalize_kernel<<<n_seg, 256, smem, st>>>(dps, best_next, seg_off, row_w, row_off, seg_band_base,
                                            band, stats, ordered, in_smem, stage_count, replicas, splits,
                                            mb_times, count, t_max_used, objective, status, err_id);
  return cudaGetLastError();
}

}  // namespace ppb
