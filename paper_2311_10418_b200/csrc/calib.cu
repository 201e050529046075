// calib.cu — in-run FP64 pipe calibration for the roofline denominators.
//
// The planner's cost and DP kernels are bound by the FP64 pipe and by
// instruction issue, not by HBM or tensor cores.
// MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks, so bench.py
// measures the FP64 add rate on the same box, in the same process, at the
// clock the run sees: every thread runs 8 independent __dadd_rn chains (the
// explicit-rounding add the planner uses), enough warps per SM to hide the
// pipe latency, grid = 8 CTAs per SM.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pipeplan_b200.h"

namespace {

constexpr int kChains = 8;
constexpr int kIters = 2048;

__global__ void __launch_bounds__(256) dadd_peak_kernel(double* out, double step) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = (double)(threadIdx.x + c);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __dadd_rn(x[c], step);
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc = __dadd_rn(acc, x[c]);
  if (acc == -1.0) out[0] = acc;  // never true; keeps the chains live
}

}  // namespace

extern "C" int pp_calibrate_fp64(int device, double* dadd_per_s) {
  if (!dadd_per_s) return PP_ERR_INVALID;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return PP_ERR_NO_DEVICE;
  }
  if (cudaSetDevice(device) != cudaSuccess) return PP_ERR_CUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = std::max(sms, 1) * 8;
  double* d = nullptr;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return PP_ERR_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaMalloc(&d, sizeof(double));
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, st);
    dadd_peak_kernel<<<blocks, 256, 0, st>>>(d, 1e-3);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0) best = std::min(best, ms);  // first launch warms up
  }
  const cudaError_t err = cudaGetLastError();
  cudaFree(d);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  if (err != cudaSuccess) return PP_ERR_CUDA;
  const double ops = (double)blocks * 256.0 * kIters * kChains;
  *dadd_per_s = ops / (best * 1e-3);
  return PP_OK;
}
