// opcost.cu — the step after the partition: per (micro-batch, stage) op
// costs, the table the reference's planner hands to its scheduler,
// communication planner and simulator (OpCostTable::from_shapes /
// microbatch_cost, src/cost_model.cpp:321-382, over estimate :294-319;
// called at planner.cpp:73-130 once per replica).  SURVEY.md §8f row 2.
//
// One thread per (micro-batch, stage): bracket the padded shape on the grid
// axes, blend the per-layer cell values (pp_internal.cuh blend_d: the same
// operation order and rounding as ProfileGrid::per_layer) and accumulate the
// stage's encoder then decoder layers exactly like estimate():
//   est.X = 0.0; est.X += L_enc * enc.X; est.X += L_dec * dec.X.
// Shapes come from the caller (from_shapes) or straight from device-resident
// plans (the padded shape of each planned micro-batch, microbatch_cost over
// a span of samples).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pp_internal.cuh"

namespace ppb {

namespace {

// padded shape of micro-batch g of the planned segments (microbatch_cost
// over samples, cost_model.cpp:331-341: max of the lengths from 0)
__global__ void mb_shape_kernel(const pp_sample* __restrict__ ordered, const int64_t* __restrict__ seg_off,
                                const int32_t* __restrict__ splits, const int64_t* __restrict__ mb_off,
                                int n_seg, int64_t n_mb, pp_padded_shape* __restrict__ shapes) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_mb;
       g += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_seg - 1;  // segment of micro-batch g: last s with mb_off[s] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (mb_off[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const int s = lo;
    const int64_t b0 = seg_off[s];
    const int64_t k = g - mb_off[s];
    const int64_t a = k == 0 ? 0 : splits[b0 + k - 1];
    const int64_t e = splits[b0 + k];
    long long in = 0, tg = 0;
    for (int64_t q = b0 + a; q < b0 + e; ++q) {
      in = max(in, (long long)ordered[q].input_len);
      tg = max(tg, (long long)ordered[q].target_len);
    }
    shapes[g] = pp_padded_shape{e - a, in, tg};
  }
}

__global__ void op_cost_kernel(CostGrid g, const double* __restrict__ le_st, const double* __restrict__ ld_st,
                               int stages, const pp_padded_shape* __restrict__ shapes, int64_t n,
                               double* __restrict__ t_f, double* __restrict__ t_b,
                               double* __restrict__ act) {
  const int per = g.nm * g.ns;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * stages;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = q / stages;
    const int st = (int)(q - k * stages);
    const pp_padded_shape sh = shapes[k];
    int mi, se, sd;
    double tm, tse, tsd;
    bracket(g.mbs_ax, g.nm, (double)sh.mbs, mi, tm);
    bracket(g.seq_ax, g.ns, (double)sh.input_len, se, tse);
    // the decoder reads the target length of encoder-decoder models (:301-302)
    bracket(g.seq_ax, g.ns, (double)(g.is_encdec ? sh.target_len : sh.input_len), sd, tsd);
    const double le = le_st[st], ld = ld_st[st];
    double ef = 0.0, eb = 0.0, ea = 0.0;
    if (le > 0.0) {
      const KindCost c = kind_cost<true, true>(g.tt, g.am, g.ns, mi, tm, se, tse);
      ef = __dadd_rn(ef, __dmul_rn(le, c.tf));
      eb = __dadd_rn(eb, __dmul_rn(le, c.tb));
      ea = __dadd_rn(ea, __dmul_rn(le, c.act));
    }
    if (ld > 0.0) {
      const KindCost c = kind_cost<true, true>(g.tt + per, g.am + per, g.ns, mi, tm, sd, tsd);
      ef = __dadd_rn(ef, __dmul_rn(ld, c.tf));
      eb = __dadd_rn(eb, __dmul_rn(ld, c.tb));
      ea = __dadd_rn(ea, __dmul_rn(ld, c.act));
    }
    t_f[q] = ef;
    t_b[q] = eb;
    act[q] = ea;
  }
}

// select_recomputation (src/schedule.cpp:319-364) over n_seg op-cost
// tables at once, one CTA per table: the first allowed strategy, in the
// reference's cheapest-compute-first order (None, Selective, Full), whose
// every act_mem(mb, j) < limits[j]; the violating stage of a strategy that
// does not fit is the smallest j holding an act >= limit (the reference's
// j-major scan with its break), and a table that fits no strategy reports
// the LAST tried strategy's stage (InfeasibleError's stage).  The chosen
// strategy's rows are copied to the output tables.
__global__ void __launch_bounds__(256) recompute_select_kernel(
    const int64_t* __restrict__ mb_off, int C, int n_tries, int3 tries, int64_t n_mb,
    const double* __restrict__ tf_all, const double* __restrict__ tb_all, const double* __restrict__ act_all,
    const double* __restrict__ limits, int32_t* __restrict__ strategy, int32_t* __restrict__ violating,
    double* __restrict__ t_f, double* __restrict__ t_b, double* __restrict__ act) {
  __shared__ int s_min;
  const int s = blockIdx.x;
  const int64_t r0 = mb_off[s] * C, r1 = mb_off[s + 1] * C;
  int chosen = -1, viol = -1;
  for (int q = 0; q < n_tries; ++q) {
    if (threadIdx.x == 0) s_min = C;
    __syncthreads();
    const double* a = act_all + (size_t)q * n_mb * C;
    int m = C;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
      const int j = (int)(i % C);
      if (a[i] >= limits[j]) m = min(m, j);
    }
    if (m < C) atomicMin(&s_min, m);
    __syncthreads();
    const int vj = s_min;
    __syncthreads();
    if (vj == C) {
      chosen = q;
      break;
    }
    viol = vj;
  }
  if (threadIdx.x == 0) {
    strategy[s] = chosen < 0 ? -1 : (chosen == 0 ? tries.x : chosen == 1 ? tries.y : tries.z);
    violating[s] = chosen < 0 ? viol : -1;
  }
  if (chosen < 0) return;
  const size_t o = (size_t)chosen * n_mb * C;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    t_f[i] = tf_all[o + i];
    t_b[i] = tb_all[o + i];
    act[i] = act_all[o + i];
  }
}

}  // namespace

cudaError_t launch_recompute_select(const int64_t* mb_off, int n_seg, int C, int n_tries, const int* tries,
                                    int64_t n_mb, const double* tf_all, const double* tb_all,
                                    const double* act_all, const double* limits, int32_t* strategy,
                                    int32_t* violating, double* t_f, double* t_b, double* act, cudaStream_t st) {
  if (n_seg <= 0) return cudaSuccess;
  const int3 tr = make_int3(tries[0], n_tries > 1 ? tries[1] : -1, n_tries > 2 ? tries[2] : -1);
  recompute_select_kernel<<<n_seg, 256, 0, st>>>(mb_off, C, n_tries, tr, n_mb, tf_all, tb_all, act_all, limits,
                                                 strategy, violating, t_f, t_b, act);
  return cudaGetLastError();
}

cudaError_t launch_mb_shapes(const pp_sample* ordered, const int64_t* seg_off, const int32_t* splits,
                             const int64_t* mb_off, int n_seg, int64_t n_mb, pp_padded_shape* shapes,
                             cudaStream_t st) {
  if (n_mb <= 0) return cudaSuccess;
  const int blocks = (int)std::min<int64_t>((n_mb + 255) / 256, 148 * 8);
  mb_shape_kernel<<<blocks, 256, 0, st>>>(ordered, seg_off, splits, mb_off, n_seg, n_mb, shapes);
  return cudaGetLastError();
}

cudaError_t launch_op_costs(const CostGrid& g, const double* le_st, const double* ld_st, int stages,
                            const pp_padded_shape* shapes, int64_t n, double* t_f, double* t_b,
                            double* act, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t work = n * stages;
  const int blocks = (int)std::min<int64_t>((work + 255) / 256, 148 * 16);
  op_cost_kernel<<<blocks, 256, 0, st>>>(g, le_st, ld_st, stages, shapes, n, t_f, t_b, act);
  return cudaGetLastError();
}

}  // namespace ppb
