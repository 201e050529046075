// report.cu — the second production caller of dp_partition (SURVEY.md §8f
// row 4): padding_vs_packing_report (src/simulate.cpp:288-406) on the device.
// Per max_seq_len: truncate, draw the token-budgeted mini-batches, plan every
// mini-batch with the DP (pp_plan_grid_device), and simulate one 1F1B
// iteration per mini-batch and method (sched.cu, F1B variant).  This file
// holds the per-mini-batch integer work of the two baselines:
//  * first-fit packing of min(total_tokens, max_len) into max_len bins
//    (:333-353), one thread per mini-batch, bins in global scratch;
//  * naive padding: the mini-batch as one micro-batch (:366-378);
//  * token sums of the DP micro-batches (:318-324).
#include <cuda_runtime.h>
#include <stdint.h>

#include "pp_internal.cuh"

namespace ppb {

namespace {

__global__ void truncate_kernel(const pp_sample* __restrict__ in, int64_t n, long long max_len,
                                pp_sample* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    pp_sample v = in[k];
    v.input_len = min((long long)v.input_len, max_len);  // simulate.cpp:301-304
    v.target_len = min((long long)v.target_len, max_len);
    out[k] = v;
  }
}

// one thread per mini-batch, samples in mini-batch (input) order
__global__ void minibatch_stats_kernel(const pp_sample* __restrict__ s, const int64_t* __restrict__ off, int n_seg,
                                       long long max_len, long long* __restrict__ bins, long long* __restrict__ st,
                                       pp_padded_shape* __restrict__ naive) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_seg; q += gridDim.x * blockDim.x) {
    const int64_t a = off[q], e = off[q + 1];
    long long sum_in = 0, sum_tg = 0, mx_in = 0, mx_tg = 0, used = 0;
    long long* b = bins + a;
    int64_t nb = 0;
    for (int64_t k = a; k < e; ++k) {
      const long long in = s[k].input_len, tg = s[k].target_len;
      sum_in += in;
      sum_tg += tg;
      mx_in = max(mx_in, in);  // PaddedShape starts at 0 (simulate.cpp:368-372)
      mx_tg = max(mx_tg, tg);
      const long long tok = min(in + tg, max_len);  // first fit (:336-351)
      used += tok;
      int64_t p = 0;
      while (p < nb && !(b[p] + tok <= max_len)) ++p;
      if (p < nb) b[p] += tok;
      else b[nb++] = tok;
    }
    st[6 * q + 0] = sum_in;
    st[6 * q + 1] = sum_tg;
    st[6 * q + 2] = used;
    st[6 * q + 3] = nb;
    naive[q] = pp_padded_shape{e - a, mx_in, mx_tg};
  }
}

// padded token sums of the DP micro-batches: sum over micro-batches of
// mbs * padded_input_len and mbs * padded_target_len (:318-324)
__global__ void dp_padded_kernel(const pp_padded_shape* __restrict__ sh, const int64_t* __restrict__ mb_off,
                                 int n_seg, long long* __restrict__ st) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_seg; q += gridDim.x * blockDim.x) {
    long long pi = 0, pt = 0;
    for (int64_t m = mb_off[q]; m < mb_off[q + 1]; ++m) {
      pi += sh[m].mbs * sh[m].input_len;
      pt += sh[m].mbs * sh[m].target_len;
    }
    st[6 * q + 4] = pi;
    st[6 * q + 5] = pt;
  }
}

// every packed bin is the same micro-batch {1, max_len, 0}: replicate row 0
__global__ void broadcast_rows_kernel(const double* __restrict__ tf1, const double* __restrict__ tb1,
                                      const double* __restrict__ ac1, int C, int64_t rows, double* __restrict__ tf,
                                      double* __restrict__ tb, double* __restrict__ ac) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < rows * C; q += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(q % C);
    tf[q] = tf1[j];
    tb[q] = tb1[j];
    ac[q] = ac1[j];
  }
}

int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

cudaError_t launch_truncate(const pp_sample* in, int64_t n, long long max_len, pp_sample* out, cudaStream_t st) {
  if (n > 0) truncate_kernel<<<blocks_for(n), 256, 0, st>>>(in, n, max_len, out);
  return cudaGetLastError();
}

cudaError_t launch_minibatch_stats(const pp_sample* s, const int64_t* off, int n_seg, long long max_len,
                                   long long* bins, long long* st6, pp_padded_shape* naive, cudaStream_t st) {
  if (n_seg > 0) minibatch_stats_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(s, off, n_seg, max_len, bins, st6, naive);
  return cudaGetLastError();
}

cudaError_t launch_dp_padded(const pp_padded_shape* sh, const int64_t* mb_off, int n_seg, long long* st6,
                             cudaStream_t st) {
  if (n_seg > 0) dp_padded_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(sh, mb_off, n_seg, st6);
  return cudaGetLastError();
}

cudaError_t launch_broadcast_rows(const double* tf1, const double* tb1, const double* ac1, int C, int64_t rows,
                                  double* tf, double* tb, double* ac, cudaStream_t st) {
  if (rows > 0) broadcast_rows_kernel<<<blocks_for(rows * C), 256, 0, st>>>(tf1, tb1, ac1, C, rows, tf, tb, ac);
  return cudaGetLastError();
}

}  // namespace ppb
