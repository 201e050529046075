// sched.cu — the per-replica step after the partition:
// the injection-order search of the reference planner.
//
// plan_iteration (planner.cpp:94-108) calls
//   order_microbatches(predicted, costs, limits, n_clusters, evaluator)
// (schedule.cpp:277-317) with
//   evaluator(sched) = simulate(plan_communication(sched, costs, meta),
//                               costs, {noise 0, comm_latency}).makespan
// i.e. per candidate order: schedule_adaptive (schedule.cpp:55-122) ->
// replay_schedule (:124-183) -> plan_communication's Start/Wait placement
// (comm_plan.cpp:115-233) -> the rendezvous simulator (simulate.cpp:78-213).
// The reference runs those n_clusters! evaluations one after another per
// mini-batch; here every (mini-batch, permutation) pair is one WARP whose
// lane j plays pipeline device j (C <= 32):
//
//  * schedule_adaptive: a cycle is one warp step.  Device j only touches its
//    own queues, memory ledger and the two one-entry "unlocked" buffers
//    (new_fwd[j+1], new_bwd[j-1]), so the reference's loop over devices inside
//    a cycle is exactly a lane-parallel step plus two shuffles.
//  * replay_schedule and simulate: each device walks its own list; the values
//    (start/end times, clocks, transfer completions) are fixed points of a
//    dependency graph, so rounds of "every lane advances as far as it can,
//    __syncwarp" compute the same doubles as the reference's sequential sweep
//    (every value is produced by the same operation on the same operands) and
//    stall exactly where it stalls (a round with no progress = the
//    reference's circular-dependency / deadlock condition).
//  * plan_communication: the global sort of transfers by (end, device,
//    op_index) restricted to one device is a 3-way merge of already sorted
//    streams (own producing ops, device j-1's forwards, device j+1's
//    backwards: op ends are non-decreasing along a device's order because
//    durations are >= 0), so each lane emits its instruction list alone.
//
// Clustering (cluster_by_time, schedule.cpp:187-275) is one CTA per
// mini-batch; the k-means centre sums run sequentially per cluster in index
// order (the reference's summation order), everything else in parallel.
// Selection (one CTA per mini-batch) applies the reference's
// "strictly smaller, or equal and identity" rule over permutations in
// std::next_permutation (lexicographic) order.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pp_internal.cuh"

namespace ppb {

// Largest n_clusters the device search takes: 12! = 479,001,600 permutations
// still index with int; beyond 8 clusters the permutations are evaluated in
// windows whose results fold into a running best per table (order_merge_kernel).
constexpr int kMaxClusters = 12;

namespace {

constexpr unsigned kFull = 0xffffffffu;

// InstrKind numbering of comm_plan.h:28-39
enum : int {
  kFwd = 0, kBwd = 1, kSendActStart = 2, kRecvActStart = 3, kSendGradStart = 4,
  kRecvGradStart = 5, kWaitSendAct = 6, kWaitRecvAct = 7, kWaitSendGrad = 8, kWaitRecvGrad = 9
};

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000LL); }

}  // namespace

// Per-warp scratch carve-up.  fq/bq (phase 1) alias the instruction area
// (phases 3-4); fend/bend (phase 2) alias the channel area (phase 4).
struct SchedSlot {
  int* ord;      // [C][2M]   packed mb << 1 | is_backward
  double* st;    // [C][2M]   replay start
  double* en;    // [C][2M]   replay end
  int* ins;      // [C][10M]  packed mb << 4 | InstrKind
  int* fq;       // [C][M]    (alias ins)
  int* bq;       // [C][M]    (alias ins)
  double* fend;  // [M][C]    (alias chan)
  double* bend;  // [M][C]
  int* sq_mb;    // [2(C-1)][M]
  int* rq_mb;
  double* sq_t;
  double* rq_t;
  double* comp;  // [2(C-1)][M] completion by micro-batch, NaN = pending
};

__host__ __device__ inline size_t sched_slot_bytes(int64_t M, int C) {
  const size_t cm = (size_t)M * (size_t)C;
  const size_t chan = (size_t)2 * (size_t)(C > 1 ? C - 1 : 1) * (size_t)M;
  size_t b = 0;
  b += 2 * cm * sizeof(int);       // ord
  b += 2 * cm * sizeof(double);    // st
  b += 2 * cm * sizeof(double);    // en
  b += 10 * cm * sizeof(int);      // ins (>= fq + bq)
  const size_t ch = chan * (2 * sizeof(int) + 3 * sizeof(double));
  b += ch > 2 * cm * sizeof(double) ? ch : 2 * cm * sizeof(double);  // channels (>= fend + bend)
  return (b + 255) & ~(size_t)255;
}

__device__ inline SchedSlot carve(char* base, int64_t M, int C) {
  SchedSlot s;
  const size_t cm = (size_t)M * (size_t)C;
  const size_t chan = (size_t)2 * (size_t)(C > 1 ? C - 1 : 1) * (size_t)M;
  char* p = base;
  s.st = (double*)p; p += 2 * cm * sizeof(double);
  s.en = (double*)p; p += 2 * cm * sizeof(double);
  char* chan_base = p;
  s.sq_t = (double*)p; p += chan * sizeof(double);
  s.rq_t = (double*)p; p += chan * sizeof(double);
  s.comp = (double*)p; p += chan * sizeof(double);
  s.sq_mb = (int*)p; p += chan * sizeof(int);
  s.rq_mb = (int*)p; p += chan * sizeof(int);
  const size_t ch = chan * (2 * sizeof(int) + 3 * sizeof(double));
  p = chan_base + (ch > 2 * cm * sizeof(double) ? ch : 2 * cm * sizeof(double));
  s.fend = (double*)chan_base;
  s.bend = s.fend + cm;
  s.ord = (int*)p; p += 2 * cm * sizeof(int);
  s.ins = (int*)p;
  s.fq = s.ins;
  s.bq = s.ins + cm;
  return s;
}

// ---------------------------------------------------------------------------
// 1. predicted times (OpCostTable::scalar_time, cost_model.cpp:344-348) and
//    cluster_by_time (schedule.cpp:187-275), one CTA per mini-batch.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) cluster_kernel(
    const double* __restrict__ tf, const double* __restrict__ tb, const int64_t* __restrict__ mb_off,
    int C, int k, double* __restrict__ pred, int* __restrict__ assign_g, int* __restrict__ cl_idx,
    int* __restrict__ cl_off, int* __restrict__ cl_k, int* __restrict__ status) {
  __shared__ double centers[32];
  __shared__ double tile[1024];
  __shared__ int changed, bad;
  __shared__ int cnt[32], front[32], start_of[32];
  __shared__ double minv[32];
  const int s = blockIdx.x;
  const int64_t base = mb_off[s];
  const int M = (int)(mb_off[s + 1] - base);
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int i = tid; i < M; i += blockDim.x) {
    double worst = 0.0;
    for (int j = 0; j < C; ++j) {
      const double f = tf[(base + i) * C + j], b = tb[(base + i) * C + j];
      // the emission merge relies on op ends being non-decreasing along a
      // device's order: durations must be >= 0 and not NaN
      if (!(f >= 0.0) || !(b >= 0.0)) bad = 1;
      const double x = __dadd_rn(f, b);
      worst = worst < x ? x : worst;  // std::max(worst, x)
    }
    pred[base + i] = worst;
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) { status[s] = PP_ERR_INVALID; cl_k[s] = 0; }
    return;
  }
  if (M <= k) {  // one cluster per micro-batch (schedule.cpp:285-287)
    for (int i = tid; i < M; i += blockDim.x) cl_idx[base + i] = i;
    for (int c = tid; c <= M; c += blockDim.x) cl_off[(int64_t)s * (k + 1) + c] = c;
    if (tid == 0) cl_k[s] = M;
    return;
  }
  const double* v = pred + base;
  int* assign = assign_g + base;
  // quantile seeding: centers[c] = value of rank (2c+1)n/(2k) in (value, index) order
  for (int i0 = 0; i0 < M; i0 += blockDim.x) {
    const int i = i0 + tid;
    const double vi = i < M ? v[i] : 0.0;
    int rank = 0;
    for (int t0 = 0; t0 < M; t0 += 1024) {
      const int tn = min(1024, M - t0);
      __syncthreads();
      for (int q = tid; q < tn; q += blockDim.x) tile[q] = v[t0 + q];
      __syncthreads();
      if (i < M)
        for (int q = 0; q < tn; ++q) {
          const double w = tile[q];
          rank += (w < vi) || (w == vi && t0 + q < i);
        }
    }
    if (i < M)
      for (int c = 0; c < k; ++c)
        if (rank == min(M - 1, (2 * c + 1) * M / (2 * k))) centers[c] = vi;
  }
  for (int i = tid; i < M; i += blockDim.x) assign[i] = 0;
  __syncthreads();
  for (int iter = 0; iter < 100; ++iter) {
    if (tid == 0) changed = 0;
    __syncthreads();
    for (int i = tid; i < M; i += blockDim.x) {
      const double vi = v[i];
      int best = 0;
      double best_d = fabs(__dsub_rn(vi, centers[0]));
      for (int c = 1; c < k; ++c) {
        const double d = fabs(__dsub_rn(vi, centers[c]));
        if (d < best_d) { best = c; best_d = d; }
      }
      if (assign[i] != best) { assign[i] = best; changed = 1; }
    }
    __syncthreads();
    // centre update: per-cluster sums in index order (schedule.cpp:226-234)
    if (tid < k) {
      double sum = 0.0;
      int n = 0;
      for (int i = 0; i < M; ++i)
        if (assign[i] == tid) { sum = __dadd_rn(sum, v[i]); ++n; }
      if (n > 0) centers[tid] = __ddiv_rn(sum, (double)n);
    }
    __syncthreads();
    if (!changed) break;
  }
  // clusters: members ascending, empties dropped, sorted by (min value, front)
  if (tid < k) {
    int n = 0, fr = -1;
    double mv = 0.0;
    for (int i = 0; i < M; ++i)
      if (assign[i] == tid) {
        if (n == 0) { fr = i; mv = v[i]; }
        else mv = v[i] < mv ? v[i] : mv;  // std::min(v, x)
        ++n;
      }
    cnt[tid] = n; front[tid] = fr; minv[tid] = mv;
  }
  __syncthreads();
  if (tid == 0) {
    int order[32], kk = 0;
    for (int c = 0; c < k; ++c)
      if (cnt[c] > 0) {
        int p = kk++;
        while (p > 0) {  // insertion by (min value, front)
          const int o = order[p - 1];
          const bool less = minv[c] < minv[o] || (minv[c] == minv[o] && front[c] < front[o]);
          if (!less) break;
          order[p] = o;
          --p;
        }
        order[p] = c;
      }
    int off = 0;
    for (int r = 0; r < kk; ++r) {
      start_of[order[r]] = off;
      cl_off[(int64_t)s * (k + 1) + r] = off;
      off += cnt[order[r]];
    }
    cl_off[(int64_t)s * (k + 1) + kk] = off;
    cl_k[s] = kk;
  }
  __syncthreads();
  if (tid < k && cnt[tid] > 0) {
    int o = start_of[tid];
    for (int i = 0; i < M; ++i)
      if (assign[i] == tid) cl_idx[base + o++] = i;
  }
}

// r-th permutation of 0..k-1 in lexicographic (std::next_permutation) order
__device__ inline void nth_perm(int r, int k, int* perm) {
  int pool[kMaxClusters];
  for (int i = 0; i < k; ++i) pool[i] = i;
  for (int i = 0; i < k; ++i) {
    int f = 1;  // (k - 1 - i)!
    for (int q = 2; q <= k - 1 - i; ++q) f *= q;
    const int d = r / f;
    r -= d * f;
    perm[i] = pool[d];
    for (int q = d; q < k - 1 - i; ++q) pool[q] = pool[q + 1];
  }
}

// ---------------------------------------------------------------------------
// 2. one warp per (mini-batch, permutation): adaptive schedule -> replay ->
//    Start/Wait placement -> rendezvous simulation.
// ---------------------------------------------------------------------------
struct ItemOut {
  double makespan;
  double bubble;
  int32_t flags;  // bit0 identity order, bit1 deadlock, bits 8..15 error code
  int32_t pad;
};

// Lanes are packed in groups of G = next power of two >= C: 32 / G
// (mini-batch, permutation) items per warp, lane j of a group = device j.
// Loop exits are warp-wide (every group steps until all groups are done);
// per-group conditions (convergence, no progress) use ballots masked to the
// group.  Cross-lane data goes through global scratch written and read with
// CTA-scope relaxed accesses (coherent in the SM's L1: every lane of a group
// is in the same CTA), ordered by __syncwarp between rounds.
__device__ __forceinline__ double ld_cta(const double* p) {
  double v;
  asm volatile("ld.relaxed.cta.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_cta(double* p, double v) {
  asm volatile("st.relaxed.cta.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// F1B: the schedule is schedule_1f1b (schedule.cpp:29-53) of table s (one
// item per table, no clustering): the simulate() makespan of a fixed 1F1B
// plan, as padding_vs_packing_report's run_iteration needs (simulate.cpp:277-286).
// EMIT: one item per table with its injection order GIVEN (`given`, M_s
// entries at mb_off[s]; ignored with F1B, whose order is the identity): the
// plan_communication instruction lists of that schedule (comm_plan.cpp:115-233)
// are copied out — device j's at out_ins[10 C mb_off[s] + 10 M_s j], packed
// (mb << 4 | InstrKind), their count at out_nins[s C + j] — next to the
// SimReport summary, so the chosen plan of every replica comes off the device.
template <bool F1B, bool EMIT = false>
__global__ void __launch_bounds__(128, 6) perm_eval_kernel(
    const double* __restrict__ tf, const double* __restrict__ tb, const double* __restrict__ act,
    const int64_t* __restrict__ mb_off, const double* __restrict__ limits, int C, int G, int k, int kfact,
    double comm_latency, int n_seg, const int* __restrict__ cl_idx, const int* __restrict__ cl_off,
    const int* __restrict__ cl_k, char* __restrict__ scratch, size_t slot_bytes, int64_t Mcap,
    ItemOut* __restrict__ items, double* __restrict__ dev_stats, int r0, int rwin,
    const int* __restrict__ given = nullptr, int* __restrict__ out_ins = nullptr,
    int* __restrict__ out_nins = nullptr) {
  __shared__ int sqn_s[4][64], rqn_s[4][64];
  __shared__ int perm_s[4][32][kMaxClusters];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int IPW = 32 / G;                 // items per warp
  const int grp = lane / G, j = lane % G;  // item slot in the warp, device
  const unsigned gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << (grp * G);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  SchedSlot S = carve(scratch + (gw * IPW + grp) * slot_bytes, Mcap, C);
  int* sqn = sqn_s[wib] + grp * 2 * G;
  int* rqn = rqn_s[wib] + grp * 2 * G;
  int* perm = perm_s[wib][grp];
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double lim = (!F1B && j < C) ? limits[j] : 0.0;
  // this launch evaluates permutations [r0, r0 + rwin) of every table; item
  // = s * rwin + (r - r0), the window-local output slot
  const int64_t n_items = (int64_t)n_seg * rwin;

  for (int64_t ib = gw * IPW; ib < n_items; ib += nw * IPW) {
    const int64_t item = ib + grp;
    int s = 0, r = 0, kk = 0, kkf = 0;
    if (item < n_items) {
      s = (int)(item / rwin);
      r = r0 + (int)(item - (int64_t)s * rwin);
      if (F1B || EMIT) {
        kk = (mb_off[s + 1] > mb_off[s] && (!EMIT || cl_k[s] > 0)) ? 1 : 0;  // EMIT: cl_k = the table's check
        kkf = 1;
      } else {
        kk = cl_k[s];
        kkf = 1;
        for (int q = 2; q <= kk; ++q) kkf *= q;
      }
    }
    // (kk == 0: no micro-batch or bad input, status set by cluster_kernel)
    const bool valid = item < n_items && kk > 0 && r < kkf;
    const bool active = valid && j < C;
    const int64_t base = valid ? mb_off[s] : 0;
    const int M = valid ? (int)(mb_off[s + 1] - base) : 0;
    const int M2 = 2 * M;
    const double* TF = tf + base * C;
    const double* TB = tb + base * C;
    const double* AC = act + base * C;

    // injection order = clusters concatenated in permutation order, written
    // straight into device 0's forward queue
    if (!F1B && !EMIT && valid && j == 0) nth_perm(r, kk, perm);
    __syncwarp();
    bool ident = true;
    if (EMIT && !F1B && valid) {  // the given injection order
      for (int t = j; t < M; t += G) {
        const int mb = given[base + t];
        S.fq[t] = mb;
        ident &= (mb == t);
      }
    } else if (!F1B && valid) {
      const int* idx = cl_idx + base;
      const int* off = cl_off + (int64_t)s * (k + 1);
      int pos = 0;
      for (int q = 0; q < kk; ++q) {
        const int c = perm[q];
        const int a = off[c], n = off[c + 1] - off[c];
        for (int t = j; t < n; t += G) {
          const int mb = idx[a + t];
          S.fq[pos + t] = mb;
          ident &= (mb == pos + t);
        }
        pos += n;
      }
    }
    ident = (__ballot_sync(kFull, !ident) & gmask) == 0;
    __syncwarp();
    int err = 0;  // group-uniform

    // ---- phase 1 (1F1B): stage j runs min(C - j, M) warm-up forwards, then
    // backward b / forward warmup + b, then drains (schedule.cpp:40-49) ----
    if (F1B) {
      if (active) {
        int* ORD = S.ord + (int64_t)j * M2;
        const int warm = min(C - j, M);
        int n_ord = 0;
        for (int i = 0; i < warm; ++i) ORD[n_ord++] = 2 * i;
        for (int b2 = 0; b2 < M; ++b2) {
          ORD[n_ord++] = 2 * b2 + 1;
          if (warm + b2 < M) ORD[n_ord++] = 2 * (warm + b2);
        }
      }
    } else
    // ---- phase 1: schedule_adaptive (schedule.cpp:55-122) ----
    {
      int n_ord = 0, fh = 0, ft = (j == 0) ? M : 0, bh = 0, bt = 0;
      double mem = 0.0;
      int* FQ = S.fq + (int64_t)j * M;
      int* BQ = S.bq + (int64_t)j * M;
      int* ORD = S.ord + (int64_t)j * M2;
      const long long cap = 4LL * M * C;
      long long cycle = 0;
      bool gdone = !valid;
      while (true) {
        if (!gdone) gdone = (__ballot_sync(gmask, active && n_ord != M2) & gmask) == 0;
        if (__all_sync(kFull, gdone)) break;
        if (!gdone && cycle > cap) { err = 3; gdone = true; }  // logic_error: failed to converge
        int fo = -1, bo = -1, selfb = -1;
        if (!gdone) {
          ++cycle;
          if (active) {
            if (bh < bt) {
              const int i = BQ[bh++];
              mem = __dsub_rn(mem, AC[(int64_t)i * C + j]);
              ORD[n_ord++] = 2 * i + 1;
              if (j > 0) bo = i;
            }
            if (fh < ft) {
              const int i = FQ[fh];
              const double a = AC[(int64_t)i * C + j];
              if (__dadd_rn(mem, a) < lim) {
                ++fh;
                mem = __dadd_rn(mem, a);
                ORD[n_ord++] = 2 * i;
                if (j + 1 < C) fo = i; else selfb = i;
              }
            }
          }
        }
        const int in_f = __shfl_up_sync(kFull, fo, 1, G);
        const int in_b = __shfl_down_sync(kFull, bo, 1, G);
        if (active && !gdone) {
          if (j > 0 && in_f >= 0) FQ[ft++] = in_f;
          const int nb = (j == C - 1) ? selfb : in_b;
          if (nb >= 0) BQ[bt++] = nb;
        }
      }
    }
    __syncwarp();

    // ---- phase 2: replay_schedule (schedule.cpp:124-183) ----
    {
      if (valid && !err)
        for (int64_t q = j; q < (int64_t)M * C; q += G) { S.fend[q] = qnan(); S.bend[q] = qnan(); }
      __syncwarp();
      int p = 0;
      double dev_free = 0.0;
      const int* ORD = S.ord + (int64_t)j * M2;
      double* ST = S.st + (int64_t)j * M2;
      double* EN = S.en + (int64_t)j * M2;
      bool gdone = !valid || err;
      while (true) {
        bool prog = false;
        if (active && !gdone)
          while (p < M2) {
            // four ops at a time: their orders, producer ends and durations are
            // loaded together; an end still NaN when loaded is re-read when its
            // op is reached (it may have been written since, e.g. by this lane)
            constexpr int kG = 4;
            const int ng = min(kG, M2 - p);
            int og[kG];
            double rd[kG], du[kG];
#pragma unroll
            for (int q = 0; q < kG; ++q) og[q] = q < ng ? ORD[p + q] : 0;
            auto ready_ptr = [&](int o) -> const double* {
              const int mb = o >> 1;
              if (!(o & 1)) return j == 0 ? nullptr : S.fend + (int64_t)mb * C + j - 1;
              return j == C - 1 ? S.fend + (int64_t)mb * C + j : S.bend + (int64_t)mb * C + j + 1;
            };
#pragma unroll
            for (int q = 0; q < kG; ++q) {
              rd[q] = -INF;
              du[q] = 0.0;
              if (q < ng) {
                const double* rp = ready_ptr(og[q]);
                if (rp) rd[q] = ld_cta(rp);
                const int mb = og[q] >> 1;
                du[q] = (og[q] & 1) ? TB[(int64_t)mb * C + j] : TF[(int64_t)mb * C + j];
              }
            }
            bool stop = false;
#pragma unroll
            for (int q = 0; q < kG; ++q) {
              if (q >= ng || stop) break;
              const int o = og[q];
              const int mb = o >> 1;
              const bool bwd = o & 1;
              double ready = rd[q];
              if (ready != ready) ready = ld_cta(ready_ptr(o));
              if (ready != ready) { stop = true; break; }
              const double start = dev_free < ready ? ready : dev_free;  // std::max(dev_free, ready)
              const double end = __dadd_rn(start, du[q]);
              ST[p] = start;
              EN[p] = end;
              st_cta((bwd ? S.bend : S.fend) + (int64_t)mb * C + j, end);
              dev_free = end;
              ++p;
              prog = true;
            }
            if (stop) break;
          }
        __syncwarp();
        const unsigned pend = __ballot_sync(kFull, active && !gdone && p != M2) & gmask;
        const unsigned anyp = __ballot_sync(kFull, prog) & gmask;
        if (!gdone && pend == 0) gdone = true;
        if (!gdone && anyp == 0) { err = 4; gdone = true; }  // logic_error: not executable
        if (__all_sync(kFull, gdone)) break;
      }
    }
    __syncwarp();

    // ---- phase 3: plan_communication's per-device emission (comm_plan.cpp:115-233) ----
    int n_ins = 0;
    if (!err && active) {
      int* INS = S.ins + (int64_t)j * 10 * M;
      const int* ORD = S.ord + (int64_t)j * M2;
      const int* ORDP = j > 0 ? S.ord + (int64_t)(j - 1) * M2 : nullptr;
      const int* ORDN = j + 1 < C ? S.ord + (int64_t)(j + 1) * M2 : nullptr;
      const double* EN = S.en + (int64_t)j * M2;
      const double* ENP = j > 0 ? S.en + (int64_t)(j - 1) * M2 : nullptr;
      const double* ENN = j + 1 < C ? S.en + (int64_t)(j + 1) * M2 : nullptr;
      const double* ST = S.st + (int64_t)j * M2;
      auto adv_own = [&](int q) {
        while (q < M2) {
          const bool b = ORD[q] & 1;
          if ((!b && j + 1 < C) || (b && j > 0)) break;
          ++q;
        }
        return q;
      };
      auto adv_prev = [&](int q) {  // device j-1 forwards -> RecvActStart
        if (!ORDP) return M2;
        while (q < M2 && (ORDP[q] & 1)) ++q;
        return q;
      };
      auto adv_next = [&](int q) {  // device j+1 backwards -> RecvGradStart
        if (!ORDN) return M2;
        while (q < M2 && !(ORDN[q] & 1)) ++q;
        return q;
      };
      int po = adv_own(0), pp = adv_prev(0), pn = adv_next(0);
      // stream heads cached in registers (end time, +inf sentinel via flags)
      double ep = pp < M2 ? ENP[pp] : 0.0, eo = po < M2 ? EN[po] : 0.0, en_ = pn < M2 ? ENN[pn] : 0.0;
      // lazily placed send Waits: channel 0 = (j+1, SendAct), 1 = (j-1, SendGrad)
      bool pend[2] = {false, false};
      int pend_mb[2] = {0, 0}, stamp[2] = {0, 0}, ctr = 0;
      auto emit = [&](int kind, int mb) { INS[n_ins++] = (mb << 4) | kind; };
      // next pending Start in (end, device, op_index) order: 0 prev, 1 own, 2 next, -1 none
      auto head = [&](double& e) {
        int w = -1;
        if (pp < M2) { w = 0; e = ep; }
        if (po < M2 && (w < 0 || eo < e)) { w = 1; e = eo; }
        if (pn < M2 && (w < 0 || en_ < e)) { w = 2; e = en_; }
        return w;
      };
      auto emit_head = [&](int w) {
        if (w == 0) {
          emit(kRecvActStart, ORDP[pp] >> 1);
          pp = adv_prev(pp + 1);
          if (pp < M2) ep = ENP[pp];
        } else if (w == 2) {
          emit(kRecvGradStart, ORDN[pn] >> 1);
          pn = adv_next(pn + 1);
          if (pn < M2) en_ = ENN[pn];
        } else {
          const int o = ORD[po];
          const int ch = (o & 1) ? 1 : 0;
          if (pend[ch]) { emit(ch ? kWaitSendGrad : kWaitSendAct, pend_mb[ch]); pend[ch] = false; }
          emit(ch ? kSendGradStart : kSendActStart, o >> 1);
          pend[ch] = true; pend_mb[ch] = o >> 1; stamp[ch] = ++ctr;
          po = adv_own(po + 1);
          if (po < M2) eo = EN[po];
        }
      };
      for (int p = 0; p < M2; ++p) {
        const double op_start = ST[p];
        double e;
        int w;
        while ((w = head(e)) >= 0 && e <= op_start) emit_head(w);
        const int o = ORD[p];
        if (!(o & 1)) {
          if (j > 0) emit(kWaitRecvAct, o >> 1);
          emit(kFwd, o >> 1);
        } else {
          if (j + 1 < C) emit(kWaitRecvGrad, o >> 1);
          emit(kBwd, o >> 1);
        }
      }
      double e;
      int w;
      while ((w = head(e)) >= 0) emit_head(w);
      if (pend[0] && pend[1]) {
        const int a = stamp[0] < stamp[1] ? 0 : 1;
        emit(a ? kWaitSendGrad : kWaitSendAct, pend_mb[a]);
        emit(a ? kWaitSendAct : kWaitSendGrad, pend_mb[1 - a]);
      } else if (pend[0]) emit(kWaitSendAct, pend_mb[0]);
      else if (pend[1]) emit(kWaitSendGrad, pend_mb[1]);
      if (EMIT) {
        int* dst = out_ins + (int64_t)10 * C * base + (int64_t)10 * M * j;
        for (int q = 0; q < n_ins; ++q) dst[q] = INS[q];
      }
    }
    if (EMIT && active) out_nins[(int64_t)s * C + j] = err ? 0 : n_ins;
    __syncwarp();

    // ---- phase 4: simulate at zero noise (simulate.cpp:78-213) ----
    double clock = 0.0, busy = 0.0, blocked = 0.0, mem = 0.0, peak = 0.0;
    bool deadlock = false;
    {
      const bool run = valid && !err;
      if (run) {
        const int nch = 2 * (C - 1);
        for (int64_t q = j; q < (int64_t)nch * M; q += G) S.comp[q] = qnan();
        for (int q = j; q < 2 * G; q += G) { sqn[q] = 0; rqn[q] = 0; }
      }
      __syncwarp();
      const int* INS = S.ins + (int64_t)j * 10 * M;
      // queues this lane appends to: send (j, act), send (j-1, grad), recv (j-1, act), recv (j, grad)
      int n_sa = 0, n_sg = 0, n_ra = 0, n_rg = 0;
      int matched[2] = {0, 0};
      double free_at[2] = {0.0, 0.0};
      int ip = 0;
      bool gdone = !run;
      while (true) {
        bool prog = false;
        if (active && !gdone)
          while (ip < n_ins) {
            // a group of up to 4 instructions: their loads (kind, duration,
            // act_mem, transfer completion) are issued together, then the
            // group is executed in order (completions do not change during
            // the advance half of a round, so the early loads see the same
            // values the one-by-one walk would)
            constexpr int kG = 4;
            const int ng = min(kG, n_ins - ip);
            int wk[kG];
            double v0[kG], v1[kG];
#pragma unroll
            for (int q = 0; q < kG; ++q) wk[q] = q < ng ? INS[ip + q] : 0;
#pragma unroll
            for (int q = 0; q < kG; ++q) {
              const int kind = wk[q] & 15, mb = wk[q] >> 4;
              v0[q] = 0.0;
              v1[q] = 0.0;
              if (q < ng) {
                if (kind <= kBwd) {
                  v0[q] = (kind == kFwd ? TF : TB)[(int64_t)mb * C + j];
                  v1[q] = AC[(int64_t)mb * C + j];
                } else if (kind >= kWaitSendAct) {
                  const int ch = kind == kWaitSendAct ? 2 * j
                                 : kind == kWaitRecvAct ? 2 * (j - 1)
                                 : kind == kWaitSendGrad ? 2 * (j - 1) + 1
                                                         : 2 * j + 1;
                  v0[q] = ld_cta(S.comp + (int64_t)ch * M + mb);
                }
              }
            }
            bool stop = false;
#pragma unroll
            for (int q = 0; q < kG; ++q) {
              if (q >= ng || stop) break;
              const int kind = wk[q] & 15, mb = wk[q] >> 4;
              if (kind <= kBwd) {
                const double dur = v0[q], a = v1[q];
                clock = __dadd_rn(clock, dur);
                busy = __dadd_rn(busy, dur);
                if (kind == kFwd) {
                  mem = __dadd_rn(mem, a);
                  peak = peak < mem ? mem : peak;
                } else {
                  mem = __dsub_rn(mem, a);
                }
              } else if (kind <= kRecvGradStart) {
                int ch, qq;
                if (kind == kSendActStart) { ch = 2 * j; qq = n_sa++; }
                else if (kind == kSendGradStart) { ch = 2 * (j - 1) + 1; qq = n_sg++; }
                else if (kind == kRecvActStart) { ch = 2 * (j - 1); qq = n_ra++; }
                else { ch = 2 * j + 1; qq = n_rg++; }
                const bool send = kind == kSendActStart || kind == kSendGradStart;
                (send ? S.sq_mb : S.rq_mb)[(int64_t)ch * M + qq] = mb;
                (send ? S.sq_t : S.rq_t)[(int64_t)ch * M + qq] = clock;
              } else {
                const double c = v0[q];
                if (c != c) { stop = true; break; }  // blocked until the transfer lands
                if (c > clock) {
                  blocked = __dadd_rn(blocked, __dsub_rn(c, clock));
                  clock = c;
                }
              }
              ++ip;
              prog = true;
            }
            if (stop) break;
          }
        // publish queue lengths, then resolve channels (lane l owns link l)
        if (active && !gdone) {
          if (j + 1 < C) sqn[2 * j] = n_sa;
          if (j > 0) sqn[2 * (j - 1) + 1] = n_sg;
          if (j > 0) rqn[2 * (j - 1)] = n_ra;
          if (j + 1 < C) rqn[2 * j + 1] = n_rg;
        }
        __syncwarp();
        if (active && !gdone && j + 1 < C)
          for (int a = 0; a < 2; ++a) {
            const int ch = 2 * j + a;
            const int ns = sqn[ch], nr = rqn[ch];
            while (matched[a] < ns && matched[a] < nr &&
                   S.sq_mb[(int64_t)ch * M + matched[a]] == S.rq_mb[(int64_t)ch * M + matched[a]]) {
              const int mb = S.sq_mb[(int64_t)ch * M + matched[a]];
              double st = S.sq_t[(int64_t)ch * M + matched[a]];
              const double rt = S.rq_t[(int64_t)ch * M + matched[a]];
              if (st < rt) st = rt;
              if (st < free_at[a]) st = free_at[a];  // std::max({send, recv, free_at})
              const double en = __dadd_rn(st, comm_latency);
              st_cta(S.comp + (int64_t)ch * M + mb, en);
              free_at[a] = en;
              ++matched[a];
              prog = true;
            }
          }
        __syncwarp();
        const unsigned pendm = __ballot_sync(kFull, active && !gdone && ip != n_ins) & gmask;
        const unsigned anyp = __ballot_sync(kFull, prog) & gmask;
        if (!gdone && pendm == 0) gdone = true;
        if (!gdone && anyp == 0) { deadlock = true; gdone = true; }
        if (__all_sync(kFull, gdone)) break;
      }
    }
    // report (simulate.cpp:186-197): device order j = 0..C-1 on lane 0 of the group
    double makespan = 0.0, non_busy = 0.0;
    for (int q = 0; q < C; ++q) {
      const double c = __shfl_sync(kFull, clock, q, G);
      makespan = makespan < c ? c : makespan;
    }
    double* ds = (dev_stats && valid) ? dev_stats + item * 5 * C : nullptr;
    for (int q = 0; q < C; ++q) {
      const double bz = __shfl_sync(kFull, busy, q, G), bl = __shfl_sync(kFull, blocked, q, G);
      const double pk = __shfl_sync(kFull, peak, q, G), fm = __shfl_sync(kFull, mem, q, G);
      const double idle = __dsub_rn(__dsub_rn(makespan, bz), bl);
      non_busy = __dadd_rn(non_busy, __dadd_rn(idle, bl));
      if (ds && j == 0) {
        ds[5 * q + 0] = bz; ds[5 * q + 1] = idle; ds[5 * q + 2] = bl;
        ds[5 * q + 3] = pk; ds[5 * q + 4] = fm;
      }
    }
    if (valid && j == 0) {
      ItemOut o;
      o.makespan = makespan;
      o.bubble = makespan > 0 ? __ddiv_rn(non_busy, __dmul_rn((double)C, makespan)) : 0.0;
      o.flags = (ident ? 1 : 0) | (deadlock ? 2 : 0) | (err << 8);
      o.pad = 0;
      items[item] = o;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// 3. selection (schedule.cpp:297-316) and the chosen order, one CTA per mini-batch
// ---------------------------------------------------------------------------
__global__ void order_select_kernel(const int64_t* __restrict__ mb_off, int k, int kfact, int C,
                                    const int* __restrict__ cl_idx, const int* __restrict__ cl_off,
                                    const int* __restrict__ cl_k, const ItemOut* __restrict__ items,
                                    const double* __restrict__ item_stats, int* __restrict__ order,
                                    double* __restrict__ makespan, double* __restrict__ bubble,
                                    int* __restrict__ deadlock, double* __restrict__ dev_stats,
                                    int* __restrict__ status) {
  __shared__ int best_s, perm[kMaxClusters];
  const int s = blockIdx.x;
  const int64_t base = mb_off[s];
  const int M = (int)(mb_off[s + 1] - base);
  const int kk = cl_k[s];
  if (threadIdx.x == 0) {
    int best = -1;
    if (kk > 0 && status[s] == PP_OK) {
      int nf = 1;
      for (int q = 2; q <= kk; ++q) nf *= q;
      double best_ms = __longlong_as_double(0x7ff0000000000000LL);
      bool best_id = false;
      for (int r = 0; r < nf; ++r) {
        const ItemOut it = items[(int64_t)s * kfact + r];
        const int e = (it.flags >> 8) & 0xff;
        if (e) { status[s] = e == 3 ? PP_ERR_NOT_CONVERGED : PP_ERR_NOT_EXECUTABLE; best = -1; break; }
        const bool id = it.flags & 1;
        if (it.makespan < best_ms || (it.makespan == best_ms && id && !best_id)) {
          best_ms = it.makespan;
          best = r;
          best_id = id;
        }
      }
    }
    best_s = best;
    if (best >= 0) {
      const ItemOut it = items[(int64_t)s * kfact + best];
      makespan[s] = it.makespan;
      if (bubble) bubble[s] = it.bubble;
      if (deadlock) deadlock[s] = (it.flags >> 1) & 1;
      nth_perm(best, kk, perm);
    } else {
      makespan[s] = __longlong_as_double(0x7ff8000000000000LL);
      if (bubble) bubble[s] = 0.0;
      if (deadlock) deadlock[s] = 0;
    }
  }
  __syncthreads();
  const int best = best_s;
  if (best < 0) {  // no order: the reference returns an empty vector
    for (int i = threadIdx.x; i < M; i += blockDim.x) order[base + i] = -1;
    return;
  }
  if (dev_stats && item_stats)
    for (int q = threadIdx.x; q < 5 * C; q += blockDim.x)
      dev_stats[s * 5 * C + q] = item_stats[((int64_t)s * kfact + best) * 5 * C + q];
  const int* off = cl_off + (int64_t)s * (k + 1);
  int pos = 0;
  for (int q = 0; q < kk; ++q) {
    const int c = perm[q];
    const int a = off[c], n = off[c + 1] - off[c];
    for (int t = threadIdx.x; t < n; t += blockDim.x) order[base + pos + t] = cl_idx[base + a + t];
    pos += n;
  }
}

// Windowed selection (n_clusters > 8 or too many items for one launch): the
// reference's rule (schedule.cpp:297-316: smaller makespan, the identity
// order on a tie; the first failing evaluation throws) applied to each
// window of permutations in order, against a running best per table.
struct OrderBest {
  double makespan, bubble;
  int r, flags, err, pad;
};

__global__ void order_merge_kernel(int n_seg, int C, int r0, int rwin, const int* __restrict__ cl_k,
                                   const ItemOut* __restrict__ items, const double* __restrict__ item_stats,
                                   OrderBest* __restrict__ best, double* __restrict__ best_stats,
                                   const int* __restrict__ status) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  OrderBest b = best[s];
  const int kk = cl_k[s];
  if (kk <= 0 || status[s] != PP_OK || b.err) return;
  int nf = 1;
  for (int q = 2; q <= kk; ++q) nf *= q;
  int won = -1;
  for (int r = r0; r < r0 + rwin && r < nf; ++r) {
    const ItemOut it = items[(int64_t)s * rwin + (r - r0)];
    const int e = (it.flags >> 8) & 0xff;
    if (e) {
      b.err = e;
      break;
    }
    const bool id = it.flags & 1;
    const bool bid = b.r >= 0 && (b.flags & 1);
    if (it.makespan < b.makespan || (it.makespan == b.makespan && id && !bid)) {
      b.makespan = it.makespan;
      b.bubble = it.bubble;
      b.flags = it.flags;
      b.r = r;
      won = r - r0;
    }
  }
  if (won >= 0 && item_stats)
    for (int q = 0; q < 5 * C; ++q) best_stats[(int64_t)s * 5 * C + q] = item_stats[((int64_t)s * rwin + won) * 5 * C + q];
  best[s] = b;
}

__global__ void order_final_kernel(const int64_t* __restrict__ mb_off, int k, int C, const int* __restrict__ cl_idx,
                                   const int* __restrict__ cl_off, const int* __restrict__ cl_k,
                                   const OrderBest* __restrict__ bestv, const double* __restrict__ best_stats,
                                   int* __restrict__ order, double* __restrict__ makespan, double* __restrict__ bubble,
                                   int* __restrict__ deadlock, double* __restrict__ dev_stats,
                                   int* __restrict__ status) {
  __shared__ int perm[kMaxClusters];
  const int s = blockIdx.x;
  const int64_t base = mb_off[s];
  const int M = (int)(mb_off[s + 1] - base);
  const int kk = cl_k[s];
  const OrderBest b = bestv[s];
  int best = (kk > 0 && status[s] == PP_OK) ? b.r : -1;
  if (kk > 0 && status[s] == PP_OK && b.err) best = -1;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (kk > 0 && status[s] == PP_OK && b.err) status[s] = b.err == 3 ? PP_ERR_NOT_CONVERGED : PP_ERR_NOT_EXECUTABLE;
    if (best >= 0) {
      makespan[s] = b.makespan;
      if (bubble) bubble[s] = b.bubble;
      if (deadlock) deadlock[s] = (b.flags >> 1) & 1;
      nth_perm(best, kk, perm);
    } else {
      makespan[s] = __longlong_as_double(0x7ff8000000000000LL);
      if (bubble) bubble[s] = 0.0;
      if (deadlock) deadlock[s] = 0;
    }
  }
  __syncthreads();
  if (best < 0) {
    for (int i = threadIdx.x; i < M; i += blockDim.x) order[base + i] = -1;
    return;
  }
  if (dev_stats && best_stats)
    for (int q = threadIdx.x; q < 5 * C; q += blockDim.x) dev_stats[s * 5 * C + q] = best_stats[(int64_t)s * 5 * C + q];
  const int* off = cl_off + (int64_t)s * (k + 1);
  int pos = 0;
  for (int q = 0; q < kk; ++q) {
    const int c = perm[q];
    const int a = off[c], n = off[c + 1] - off[c];
    for (int t = threadIdx.x; t < n; t += blockDim.x) order[base + pos + t] = cl_idx[base + a + t];
    pos += n;
  }
}

__global__ void order_best_init_kernel(int n_seg, OrderBest* best) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_seg) best[s] = OrderBest{__longlong_as_double(0x7ff0000000000000LL), 0.0, -1, 0, 0, 0};
}

size_t order_search_best_bytes() { return sizeof(OrderBest); }

size_t order_search_slot_bytes(int64_t max_m, int C) { return sched_slot_bytes(max_m, C); }

// warps for the evaluation grid; the scratch holds warps * (32 / G) slots
int order_search_warps(int64_t n_items, int C, size_t slot_bytes, size_t budget) {
  int G = 1;
  while (G < C) G *= 2;
  const int ipw = 32 / G;
  int64_t w = std::min<int64_t>((n_items + ipw - 1) / ipw, (int64_t)148 * 64);
  const int64_t by_mem = std::max<int64_t>(4, (int64_t)(budget / std::max<size_t>(slot_bytes * ipw, 1)));
  w = std::max<int64_t>(std::min(w, by_mem), 1);
  return (int)((w + 3) / 4 * 4);  // whole 4-warp CTAs: every warp owns a slot
}

cudaError_t launch_order_search(const double* tf, const double* tb, const double* act,
                                const int64_t* mb_off, int n_seg, int C, const double* limits,
                                int k, int kfact, double comm_latency, int64_t max_m, double* pred,
                                int* assign, int* cl_idx, int* cl_off, int* cl_k, char* scratch,
                                size_t slot_bytes, int warps, void* items, double* item_stats,
                                int* order, double* makespan, double* bubble, int* deadlock,
                                double* dev_stats, int* status, int rwin, void* best, double* best_stats,
                                cudaStream_t st) {
  if (n_seg <= 0) return cudaSuccess;
  cluster_kernel<<<n_seg, 256, 0, st>>>(tf, tb, mb_off, C, k, pred, assign, cl_idx, cl_off, cl_k, status);
  int G = 1;
  while (G < C) G *= 2;
  const int blocks = (warps + 3) / 4;
  if (rwin >= kfact) {  // every permutation in one launch
    perm_eval_kernel<false><<<blocks, 128, 0, st>>>(tf, tb, act, mb_off, limits, C, G, k, kfact, comm_latency, n_seg,
                                                    cl_idx, cl_off, cl_k, scratch, slot_bytes, max_m,
                                                    (ItemOut*)items, item_stats, 0, kfact);
    order_select_kernel<<<n_seg, 128, 0, st>>>(mb_off, k, kfact, C, cl_idx, cl_off, cl_k, (const ItemOut*)items,
                                               item_stats, order, makespan, bubble, deadlock, dev_stats, status);
    return cudaGetLastError();
  }
  OrderBest* bv = static_cast<OrderBest*>(best);
  order_best_init_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(n_seg, bv);
  for (int r0 = 0; r0 < kfact; r0 += rwin) {
    const int w = std::min(rwin, kfact - r0);
    perm_eval_kernel<false><<<blocks, 128, 0, st>>>(tf, tb, act, mb_off, limits, C, G, k, kfact, comm_latency, n_seg,
                                                    cl_idx, cl_off, cl_k, scratch, slot_bytes, max_m,
                                                    (ItemOut*)items, item_stats, r0, w);
    order_merge_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(n_seg, C, r0, w, cl_k, (const ItemOut*)items, item_stats,
                                                            bv, best_stats, status);
  }
  order_final_kernel<<<n_seg, 128, 0, st>>>(mb_off, k, C, cl_idx, cl_off, cl_k, bv, best_stats, order, makespan,
                                            bubble, deadlock, dev_stats, status);
  return cudaGetLastError();
}

size_t order_search_item_bytes() { return sizeof(ItemOut); }

// Emission inputs per table: at least one micro-batch, durations >= 0 and
// not NaN (the emission merge), and (adaptive) an injection order that is a
// permutation of 0..M-1 (schedule_adaptive's precondition, schedule.cpp:62-66).
__global__ void __launch_bounds__(256) emit_check_kernel(const double* __restrict__ tf, const double* __restrict__ tb,
                                                         const int64_t* __restrict__ mb_off, int C,
                                                         const int* __restrict__ order, int f1b, int* __restrict__ ok,
                                                         int* __restrict__ seen, int* __restrict__ status,
                                                         int* __restrict__ out_nins) {
  __shared__ int bad;
  const int s = blockIdx.x;
  const int64_t base = mb_off[s];
  const int M = (int)(mb_off[s + 1] - base);
  if (threadIdx.x == 0) bad = M < 1;
  for (int i = threadIdx.x; i < M; i += blockDim.x) seen[base + i] = 0;
  for (int j = threadIdx.x; j < C; j += blockDim.x) out_nins[(int64_t)s * C + j] = 0;
  __syncthreads();
  for (int64_t q = threadIdx.x; q < (int64_t)M * C; q += blockDim.x)
    if (!(tf[base * C + q] >= 0.0) || !(tb[base * C + q] >= 0.0)) bad = 1;
  if (!f1b)
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      const int mb = order[base + i];
      if (mb < 0 || mb >= M || atomicExch(&seen[base + mb], 1)) bad = 1;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    ok[s] = bad ? 0 : 1;
    status[s] = bad ? PP_ERR_INVALID : PP_OK;
  }
}

__global__ void emit_final_kernel(int n_seg, const int* __restrict__ ok, const ItemOut* __restrict__ items,
                                  double* __restrict__ makespan, double* __restrict__ bubble, int* __restrict__ deadlock,
                                  int* __restrict__ status) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  if (!ok[s]) {
    makespan[s] = __longlong_as_double(0x7ff8000000000000LL);
    if (bubble) bubble[s] = 0.0;
    if (deadlock) deadlock[s] = 0;
    return;
  }
  const ItemOut it = items[s];
  const int e = (it.flags >> 8) & 0xff;
  status[s] = e ? (e == 3 ? PP_ERR_NOT_CONVERGED : PP_ERR_NOT_EXECUTABLE) : PP_OK;
  makespan[s] = it.makespan;
  if (bubble) bubble[s] = it.bubble;
  if (deadlock) deadlock[s] = (it.flags >> 1) & 1;
}

// plan_communication of each table's schedule_adaptive(costs, limits, order)
// (or schedule_1f1b with f1b) for GIVEN injection orders: instruction lists,
// counts, and the SimReport summary (makespan, bubble, deadlock, device
// stats [s][C][5]); status PP_ERR_INVALID / NOT_CONVERGED / NOT_EXECUTABLE.
cudaError_t launch_emit_plans(const double* tf, const double* tb, const double* act, const int64_t* mb_off, int n_seg,
                              int C, const double* limits, double comm_latency, int64_t max_m, const int* order,
                              int f1b, char* scratch, size_t slot_bytes, int warps, void* items, int* ok, int* seen,
                              int* out_ins, int* out_nins, double* makespan, double* bubble, int* deadlock,
                              double* dev_stats, int* status, cudaStream_t st) {
  if (n_seg <= 0) return cudaSuccess;
  int G = 1;
  while (G < C) G *= 2;
  const int blocks = (warps + 3) / 4;
  emit_check_kernel<<<n_seg, 256, 0, st>>>(tf, tb, mb_off, C, order, f1b, ok, seen, status, out_nins);
  if (f1b)
    perm_eval_kernel<true, true><<<blocks, 128, 0, st>>>(tf, tb, act, mb_off, limits, C, G, 1, 1, comm_latency,
                                                         n_seg, nullptr, nullptr, ok, scratch, slot_bytes, max_m,
                                                         (ItemOut*)items, dev_stats, 0, 1, order, out_ins, out_nins);
  else
    perm_eval_kernel<false, true><<<blocks, 128, 0, st>>>(tf, tb, act, mb_off, limits, C, G, 1, 1, comm_latency,
                                                          n_seg, nullptr, nullptr, ok, scratch, slot_bytes,
                                                          max_m, (ItemOut*)items, dev_stats, 0, 1, order, out_ins,
                                                          out_nins);
  emit_final_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(n_seg, ok, (const ItemOut*)items, makespan, bubble, deadlock,
                                                          status);
  return cudaGetLastError();
}

// simulate() makespans of schedule_1f1b over every table (run_iteration,
// simulate.cpp:277-286): items[s].makespan, zero noise, comm_latency.
cudaError_t launch_sim_1f1b(const double* tf, const double* tb, const double* act, const int64_t* mb_off,
                            int n_seg, int C, double comm_latency, int64_t max_m, char* scratch,
                            size_t slot_bytes, int warps, void* items, cudaStream_t st) {
  if (n_seg <= 0) return cudaSuccess;
  int G = 1;
  while (G < C) G *= 2;
  const int blocks = (warps + 3) / 4;
  perm_eval_kernel<true><<<blocks, 128, 0, st>>>(tf, tb, act, mb_off, nullptr, C, G, 1, 1, comm_latency, n_seg,
                                                 nullptr, nullptr, nullptr, scratch, slot_bytes, max_m,
                                                 (ItemOut*)items, nullptr, 0, 1);
  return cudaGetLastError();
}

}  // namespace ppb
