// dp.cu — the suffix DP of dp_partition on sm_100a: one CTA per
// (mini-batch, t_max candidate), plus the per-mini-batch candidate selection
// and assembly.
//
// Reference: run_suffix_dp (src/microbatch.cpp:162-189), the candidate loop
// (:281-318), reconstruct_splits (:194-215) and assembly (:322-335).
//
// Row recurrence for a candidate t (state[n] = (0, 0)):
//   state[i] = lexmin over j in (i, n] with T[i,j] <= t, M[i,j] <= cap and
//              state[j] finite of (T[i,j] + state[j].sum, 1 + state[j].count)
// with the reference's strict-improvement rule, i.e. the lowest j among equal
// (sum, count) pairs; that j is next[i].  next[] then *is* reconstruct_splits:
// its front-to-back scan picks the smallest j with T + state[j].sum ==
// state[i].sum && 1 + state[j].count == state[i].count — the lowest-index
// argmin of the row.  Only finite sums can ever be taken (inf/NaN fail both
// `<` and the count tie-break against the initial (inf, 0)), and lexmin over
// (sum, count, j) is associative and commutative, so any reduction order
// yields the reference's state bit-for-bit.
//
// CTA schedule (never changes results).  Rows are processed top-down in
// 32-row blocks; the band of a block is one tile (cost.cu): column c holds
// T[i0 + r, i0 + c] for the 32 rows r.  For block b:
//   * warp 0 (the chain warp) folds the far-far partials, the near-far
//     columns [nb, 64) and then runs the in-block triangle serially: lane r
//     owns row i0 + r; walking jj = nb-1 .. 0, lane jj finalises its row and
//     broadcasts (sum, count) with shuffles, the lanes below fold
//     T[i0 + r, i0 + jj] + state into their accumulators;
//   * warps 1..8 (workers) meanwhile reduce the far-far columns [64, W) of
//     block b+1, whose states (j >= i1(b)) are already final;
//   * the near tile (columns [0, 64)) of each block and the far-far columns in
//     32-column chunks are streamed global -> shared by TMA bulk copies
//     (cp.async.bulk, mbarrier completion), issued by one worker thread ahead
//     of use through a ring of chunk buffers, so the serial chain never waits
//     on global memory.
// DP state lives in shared memory, as a ring of R >= W_max + 64 entries when
// the memory cap bounds the row widths.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "pp_internal.cuh"

namespace ppb {

constexpr int kWorkers = 8;
constexpr int kDpThreads = 32 * (1 + kWorkers);
constexpr int kNearCols = 64;
constexpr int kChunkCols = 32;
constexpr int kMaxRing = 24;
constexpr uint32_t kColBytes = kRB * sizeof(double);  // 256 B
constexpr size_t kChunkBytes = (size_t)kChunkCols * kColBytes;  // 8 KB

__device__ __forceinline__ bool isfin(double x) { return isfinite(x); }

// (s, c, j) lexmin with lowest-j ties.
__device__ __forceinline__ bool better(double s1, int c1, int j1, double s0, int c0, int j0) {
  if (s1 < s0) return true;
  if (s1 == s0) {
    if (c1 < c0) return true;
    if (c1 == c0 && j1 < j0) return true;
  }
  return false;
}

// Shared-memory layout of dp_pass_kernel (offsets in bytes): fixed part,
// then the DP state (when it lives in shared memory), then the ring of far
// chunk buffers, whose depth the launcher sizes to the remaining space.
struct DpSmem {
  static constexpr size_t near = 0;                                  // [2][64][32] double
  static constexpr size_t ffs = near + 2 * kNearCols * kColBytes;    // [2][8][32] double
  static constexpr size_t ffx = ffs + 2 * kWorkers * kRB * 8;        // [2][8][32] double/int
  static constexpr size_t ffj = ffx + 2 * kWorkers * kRB * 8;        // [2][8][32] int
  static constexpr size_t bars = ffj + 2 * kWorkers * kRB * 4;       // mbarriers
  static constexpr size_t state = bars + 8 * (2 + kMaxRing);         // state arrays
};

size_t dp_smem_fixed() { return DpSmem::state; }
size_t dp_state_bytes(int mode, int entries) { return (size_t)entries * (mode == 0 ? 12 : 16); }
size_t dp_chunk_bytes() { return kChunkBytes; }
int dp_max_ring() { return kMaxRing; }

// Far-far chunk sequence helpers: block b has max(0, ceil((W_b - 64) / 32))
// chunks of up to 32 columns starting at column 64.
__device__ __forceinline__ int n_chunks(int W) {
  return W > kNearCols ? (W - kNearCols + kChunkCols - 1) / kChunkCols : 0;
}

template <int MODE>
__global__ void __launch_bounds__(kDpThreads, 1)
    dp_pass_kernel(const WorkItem* __restrict__ items, const int64_t* __restrict__ seg_off,
                   const int* __restrict__ blk_base, const int* __restrict__ blk_W,
                   const int64_t* __restrict__ tile_off, const int64_t* __restrict__ seg_band_base,
                   const double* __restrict__ band, const double* __restrict__ cand,
                   const int64_t* __restrict__ cand_off, ItemResult* __restrict__ res,
                   int* __restrict__ next_buf, double* __restrict__ gstate, int res_by_seg,
                   int ring_off, int kRing) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* near = reinterpret_cast<double*>(smem + DpSmem::near);
  double* ring = reinterpret_cast<double*>(smem + ring_off);
  double* ffs = reinterpret_cast<double*>(smem + DpSmem::ffs);
  double* ffm = reinterpret_cast<double*>(smem + DpSmem::ffx);  // MODE 1
  int* ffc = reinterpret_cast<int*>(smem + DpSmem::ffx);        // MODE 0
  int* ffj = reinterpret_cast<int*>(smem + DpSmem::ffj);
  uint64_t* bar_near = reinterpret_cast<uint64_t*>(smem + DpSmem::bars);
  uint64_t* bar_ring = bar_near + 2;

  const WorkItem it = items[blockIdx.x];
  const int s = it.seg;
  const int64_t b0 = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b0);
  const int gb0 = blk_base[s];
  const int nblk = blk_base[s + 1] - gb0;
  const double t = item_t(it, cand, cand_off);
  const double* bseg = band + seg_band_base[s];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);

  // state: ring of R = mask + 1 entries (mask = ~0 when not a ring)
  const unsigned mask = it.state_mask;
  const int entries = it.state_entries;
  double* st_s;
  unsigned char* st_x_raw;
  if (it.state_off < 0) {
    st_s = reinterpret_cast<double*>(smem + DpSmem::state);
  } else {
    st_s = gstate + it.state_off;
  }
  st_x_raw = reinterpret_cast<unsigned char*>(st_s + entries);
  int* st_c = reinterpret_cast<int*>(st_x_raw);        // MODE 0
  double* st_m = reinterpret_cast<double*>(st_x_raw);  // MODE 1
  int* nxt = next_buf + it.next_off;

  // ---- prologue
  if (threadIdx.x == 0) {
    mbar_init(&bar_near[0], 1);
    mbar_init(&bar_near[1], 1);
    for (int k = 0; k < kRing; ++k) mbar_init(&bar_ring[k], 1);
    mbar_fence_init();
    st_s[n & mask] = 0.0;  // state[n] = {0.0, 0} (microbatch.cpp:174)
    if (MODE == 0) st_c[n & mask] = 0; else st_m[n & mask] = -INF;
  }
  // block 0 has no far-far columns (j <= n < i0 + 64)
  if (wid >= 1) {
    const int w = wid - 1;
    ffs[(0 * kWorkers + w) * kRB + lane] = INF;
    if (MODE == 0) {
      ffc[(0 * kWorkers + w) * kRB + lane] = 0;
      ffj[(0 * kWorkers + w) * kRB + lane] = INT_MAX;
    } else {
      ffm[(0 * kWorkers + w) * kRB + lane] = INF;
    }
  }
  __syncthreads();

  // producer state (thread 32): next far chunk to issue, in consumption order
  const bool producer = threadIdx.x == 32;
  int pb = 1, pk = 0;     // block / chunk cursor of the next chunk to issue
  int issued = 0;         // chunks issued so far
  int consumed = 0;       // chunks consumed so far (workers, uniform)
  auto issue_chunks = [&](int limit) {
    while (issued < limit && pb < nblk) {
      const int gb = gb0 + pb;
      const int W = blk_W[gb];
      const int nc = n_chunks(W);
      if (pk >= nc) {
        ++pb;
        pk = 0;
        continue;
      }
      const int c0 = kNearCols + pk * kChunkCols;
      const int cols = min(kChunkCols, W - c0);
      const int slot = issued % kRing;
      mbar_expect_tx(&bar_ring[slot], cols * kColBytes);
      tma_load_1d(ring + (size_t)slot * kChunkCols * kRB, bseg + tile_off[gb] + (size_t)c0 * kRB,
                  cols * kColBytes, &bar_ring[slot]);
      ++issued;
      ++pk;
    }
  };
  auto issue_near = [&](int b) {
    const int gb = gb0 + b;
    const int cols = min(kNearCols, blk_W[gb]);
    mbar_expect_tx(&bar_near[b & 1], cols * kColBytes);
    tma_load_1d(near + (size_t)(b & 1) * kNearCols * kRB, bseg + tile_off[gb], cols * kColBytes,
                &bar_near[b & 1]);
  };
  if (producer && nblk > 0) {
    issue_near(0);
    issue_chunks(kRing);
  }

  for (int b = 0; b < nblk; ++b) {
    const int i1 = n - kRB * b;
    const int i0 = max(0, i1 - kRB);
    const int nb = i1 - i0;
    const int W = blk_W[gb0 + b];
    if (producer && b + 1 < nblk) issue_near(b + 1);

    if (wid == 0) {
      // ================= chain warp: block b =================
      mbar_wait(&bar_near[b & 1], (b >> 1) & 1);
      const double* nt = near + (size_t)(b & 1) * kNearCols * kRB;
      const int r = lane;
      const bool rowv = r < nb;
      // far-far partials (workers, previous iteration)
      double as = INF, am = INF;
      int ac = 0, aj = INT_MAX;
#pragma unroll
      for (int w = 0; w < kWorkers; ++w) {
        const int o = ((b & 1) * kWorkers + w) * kRB + r;
        const double ps = ffs[o];
        if (MODE == 0) {
          const int pc = ffc[o], pj = ffj[o];
          if (better(ps, pc, pj, as, ac, aj)) {
            as = ps;
            ac = pc;
            aj = pj;
          }
        } else {
          as = (ps < as) ? ps : as;
          const double pm = ffm[o];
          am = (pm < am) ? pm : am;
        }
      }
      // near-far columns [nb, min(64, W)): states final
      const int cnf = min(kNearCols, W);
      for (int c = nb; c < cnf; ++c) {
        const double x = nt[c * kRB + r];
        const int j = i0 + c;
        const double sj = st_s[j & mask];
        if (MODE == 0) {
          if (x <= t && isfin(sj)) {
            const double cs = __dadd_rn(x, sj);
            const int cc = 1 + st_c[j & mask];
            if (isfin(cs) && better(cs, cc, j, as, ac, aj)) {
              as = cs;
              ac = cc;
              aj = j;
            }
          }
        } else if (!isnan(x)) {
          if (isfin(sj)) {
            const double cs = __dadd_rn(x, sj);
            if (isfin(cs) && cs < as) as = cs;
          }
          const double mj = st_m[j & mask];
          if (x < INF && mj < INF) {
            const double v = (x < mj) ? mj : x;
            am = (v < am) ? v : am;
          }
        }
      }
      // in-block triangle: T[i0 + r, i0 + jj] for jj in (r, nb)
      double tn[kRB];
#pragma unroll
      for (int jj = 0; jj < kRB; ++jj) tn[jj] = (jj < W) ? nt[jj * kRB + r] : QNAN;
      if (!rowv) {
        as = INF;
        ac = 0;
        am = INF;
      }
#pragma unroll
      for (int jj = kRB - 1; jj >= 0; --jj) {
        if (jj < nb) {
          const double sj = __shfl_sync(0xffffffffu, as, jj);
          int cj = 0;
          double mj = 0.0;
          if (MODE == 0) cj = __shfl_sync(0xffffffffu, ac, jj);
          else mj = __shfl_sync(0xffffffffu, am, jj);
          if (lane == jj) {
            const int row = i0 + jj;
            if (MODE == 0) {
              const bool f = isfin(as);
              st_s[row & mask] = f ? as : INF;
              st_c[row & mask] = f ? ac : 0;
              nxt[row] = f ? aj : -1;
            } else {
              st_s[row & mask] = as;
              st_m[row & mask] = am;
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
                if (isfin(cs) && (cs < as || (cs == as && cc <= ac))) {
                  as = cs;
                  ac = cc;
                  aj = j;
                }
              }
            } else if (!isnan(x)) {
              if (isfin(sj)) {
                const double cs = __dadd_rn(x, sj);
                if (isfin(cs) && cs < as) as = cs;
              }
              if (x < INF && mj < INF) {
                const double v = (x < mj) ? mj : x;
                am = (v < am) ? v : am;
              }
            }
          }
        }
      }
    } else {
      // ================= workers: far-far of block b+1 =================
      const int w = wid - 1;
      const int bn = b + 1;
      if (bn < nblk) {
        const int j1 = n - kRB * bn;
        const int k0 = max(0, j1 - kRB);  // i0 of block b+1
        const int Wn = blk_W[gb0 + bn];
        const int nc = n_chunks(Wn);
        double as = INF, am = INF;
        int ac = 0, aj = INT_MAX;
        const int r = lane;
        for (int k = 0; k < nc; ++k) {
          const int slot = consumed % kRing;
          mbar_wait(&bar_ring[slot], (consumed / kRing) & 1);
          const double* ch = ring + (size_t)slot * kChunkCols * kRB;
          const int c0 = kNearCols + k * kChunkCols;
          const int cols = min(kChunkCols, Wn - c0);
#pragma unroll
          for (int q0 = 0; q0 < kChunkCols; q0 += kWorkers) {
            const int q = q0 + w;
            if (q < cols) {
              const double x = ch[q * kRB + r];
              const int j = k0 + c0 + q;
              const double sj = st_s[j & mask];
              if (MODE == 0) {
                if (x <= t && isfin(sj)) {
                  const double cs = __dadd_rn(x, sj);
                  const int cc = 1 + st_c[j & mask];
                  if (isfin(cs) && better(cs, cc, j, as, ac, aj)) {
                    as = cs;
                    ac = cc;
                    aj = j;
                  }
                }
              } else if (!isnan(x)) {
                if (isfin(sj)) {
                  const double cs = __dadd_rn(x, sj);
                  if (isfin(cs) && cs < as) as = cs;
                }
                const double mj = st_m[j & mask];
                if (x < INF && mj < INF) {
                  const double v = (x < mj) ? mj : x;
                  am = (v < am) ? v : am;
                }
              }
            }
          }
          ++consumed;
          named_bar(1, 32 * kWorkers);  // every worker is done with this slot
          if (producer) {
            fence_proxy_async();
            issue_chunks(consumed + kRing);
          }
        }
        const int o = ((bn & 1) * kWorkers + w) * kRB + r;
        ffs[o] = as;
        if (MODE == 0) {
          ffc[o] = ac;
          ffj[o] = aj;
        } else {
          ffm[o] = am;
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ItemResult rr;
    rr.sum0 = st_s[0];
    rr.count0 = MODE == 0 ? st_c[0] : 0;
    rr.feasible = isfin(st_s[0]) ? 1 : 0;
    rr.aux = MODE == 1 ? st_m[0] : 0.0;
    res[res_by_seg ? s : blockIdx.x] = rr;
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
// eval_objective (front-to-back, :109-120) and t_max_used.  The split chain
// is walked in shared memory; the slice times are fetched in parallel; the
// objective's sum is accumulated front-to-back by one thread (same rounding
// order as the reference).
__global__ void __launch_bounds__(256)
    finalize_kernel(const SegDP* __restrict__ dps, const int* __restrict__ best_next,
                    const int64_t* __restrict__ seg_off, const int* __restrict__ blk_base,
                    const int64_t* __restrict__ tile_off, const int64_t* __restrict__ seg_band_base,
                    const double* __restrict__ band, const SegStats* __restrict__ stats,
                    const pp_sample* __restrict__ ordered, int chain_in_smem, int stage_count,
                    int replicas, int32_t* __restrict__ splits, double* __restrict__ mb_times,
                    int32_t* __restrict__ count, double* __restrict__ t_max_used,
                    double* __restrict__ objective, int32_t* __restrict__ status,
                    int64_t* __restrict__ err_id) {
  extern __shared__ int chain[];
  __shared__ int m_sh;
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
  int32_t* sp = splits + b;
  if (threadIdx.x == 0) {
    int i = 0, m = 0;
    while (i < n) {
      const int j = ch[i];
      sp[m++] = j;
      i = j;
    }
    m_sh = m;
  }
  __syncthreads();
  const int m = m_sh;
  const double* bseg = band + seg_band_base[s];
  const int gb0 = blk_base[s];
  double* tt = mb_times + b;
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    const int j = sp[k];
    const int i = k ? sp[k - 1] : 0;
    const int bl = (n - 1 - i) / kRB;  // block of row i
    const int i0 = max(0, n - kRB * (bl + 1));
    tt[k] = bseg[tile_off[gb0 + bl] + (int64_t)(j - i0) * kRB + (i - i0)];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double max_t = 0.0, sum = 0.0;
    for (int k = 0; k < m; ++k) {
      const double v = tt[k];
      max_t = (max_t < v) ? v : max_t;
      sum = __dadd_rn(sum, v);
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
// smem_state = the largest shared-memory DP state of the launch's items.
// The chunk ring gets the rest of `smem_budget` (4..kMaxRing chunks of 8 KB).
cudaError_t launch_dp_pass(int mode, const WorkItem* items, int n_items, size_t smem_state,
                           size_t smem_budget, const int64_t* seg_off, const int* blk_base,
                           const int* blk_W, const int64_t* tile_off, const int64_t* seg_band_base,
                           const double* band, const double* cand, const int64_t* cand_off,
                           ItemResult* res, int* next_buf, double* gstate, int res_by_seg,
                           cudaStream_t st) {
  if (n_items == 0) return cudaSuccess;
  const size_t ring_off = (DpSmem::state + smem_state + 127) / 128 * 128;
  int ring = (int)std::min<size_t>(kMaxRing, (smem_budget - std::min(smem_budget, ring_off)) / kChunkBytes);
  ring = std::max(ring, 4);
  const size_t smem = ring_off + (size_t)ring * kChunkBytes;
  if (mode == 0) {
    cudaFuncSetAttribute(dp_pass_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dp_pass_kernel<0><<<n_items, kDpThreads, smem, st>>>(items, seg_off, blk_base, blk_W, tile_off,
                                                         seg_band_base, band, cand, cand_off, res,
                                                         next_buf, gstate, res_by_seg, (int)ring_off,
                                                         ring);
  } else {
    cudaFuncSetAttribute(dp_pass_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dp_pass_kernel<1><<<n_items, kDpThreads, smem, st>>>(items, seg_off, blk_base, blk_W, tile_off,
                                                         seg_band_base, band, cand, cand_off, res,
                                                         next_buf, gstate, res_by_seg, (int)ring_off,
                                                         ring);
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
                            const int* blk_base, const int64_t* tile_off, const int64_t* seg_band_base,
                            const double* band, const SegStats* stats, const pp_sample* ordered,
                            int stage_count, int replicas, int max_n, int n_seg, int32_t* splits,
                            double* mb_times, int32_t* count, double* t_max_used, double* objective,
                            int32_t* status, int64_t* err_id, cudaStream_t st) {
  const int in_smem = (size_t)max_n * sizeof(int) <= 200 * 1024 ? 1 : 0;
  const size_t smem = in_smem ? (size_t)max_n * sizeof(int) : 0;
  cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  finalize_kernel<<<n_seg, 256, smem, st>>>(dps, best_next, seg_off, blk_base, tile_off, seg_band_base,
                                            band, stats, ordered, in_smem, stage_count, replicas,
                                            splits, mb_times, count, t_max_used, objective, status,
                                            err_id);
  return cudaGetLastError();
}

}  // namespace ppb
