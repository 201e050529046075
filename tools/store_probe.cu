// Store-bandwidth probe: how fast can a kernel stream 8-byte stores (the
// band's write pattern: one coalesced 256 B column per warp step) into HBM?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/store_probe.cu -o /tmp/store_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int VEC>
__global__ void store_kernel(double* __restrict__ out, size_t n, double v) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * VEC;
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC; i < n; i += stride) {
    if (VEC == 1) out[i] = v;
    else reinterpret_cast<double2*>(out)[i / 2] = make_double2(v, v);
  }
}

// warp writes 32-row columns one after another, like pass B (tile = 32 x W)
__global__ void column_kernel(double* __restrict__ out, size_t tiles, int W, double v) {
  const int lane = threadIdx.x & 31;
  const size_t warps = (size_t)gridDim.x * (blockDim.x >> 5);
  for (size_t t = (size_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < tiles; t += warps) {
    double* tile = out + t * (size_t)W * 32;
    for (int c = 0; c < W; ++c) tile[(size_t)c * 32 + lane] = v + c;
  }
}

int main() {
  const size_t bytes = 6ull << 30;
  const size_t n = bytes / 8;
  double* d;
  cudaMalloc(&d, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep) {
    for (int mode = 0; mode < 4; ++mode) {
      cudaEventRecord(a);
      if (mode == 0) store_kernel<1><<<sms * 8, 256>>>(d, n, 1.0);
      if (mode == 1) store_kernel<2><<<sms * 8, 256>>>(d, n, 1.0);
      if (mode == 2) column_kernel<<<sms * 4, 256>>>(d, n / (322 * 32), 322, 1.0);
      if (mode == 3) cudaMemsetAsync(d, 0, bytes);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const char* nm[] = {"STG.64 grid-stride", "STG.128 grid-stride", "pass-B columns (W=322)", "cudaMemset"};
      if (rep) printf("%-26s %8.3f ms  %7.1f GB/s\n", nm[mode], ms, bytes / ms / 1e6);
    }
  }
  return 0;
}
