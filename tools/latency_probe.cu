// latency_probe.cu — dependent-chain latencies of the instructions on the DP
// chain's critical path (development tool; run on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/latency_probe tools/latency_probe.cu
//   ./build/latency_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k_dadd(double* out, double a, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
__global__ void k_dsetp_sel(double* out, double a, long long* cyc) {
  double x = a, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = (x < y) ? y : __dadd_rn(x, 0.0);  // compare -> select chain
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x + y; }
}
__global__ void k_shfl_d(double* out, double a, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
__global__ void k_shfl_i(double* out, double a, long long* cyc) {
  int x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (x + 1) & 31);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
__global__ void k_lds(double* out, double a, long long* cyc) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = s[x];
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
// one triangle step as the DP writes it: shfl(sum) -> dadd -> compare -> select
__global__ void k_step(double* out, double a, long long* cyc) {
  double as = 1e9 + threadIdx.x, x = a + threadIdx.x;
  int ac = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
    const int jj = i & 31;
    const double sj = __shfl_sync(0xffffffffu, as, jj);
    const int cn = 1 + __shfl_sync(0xffffffffu, ac, jj);
    const double cs = __dadd_rn(x, sj);
    const bool upd = (threadIdx.x < jj) && (cs < as || (cs == as && cn <= ac));
    as = upd ? cs : as;
    ac = upd ? cn : ac;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = as + ac; }
}

template <typename K>
void run(const char* name, K k) {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 8);
  k<<<1, 32>>>(o, 1.000001, c);
  k<<<1, 32>>>(o, 1.000001, c);
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.1f cycles / iteration\n", name, (double)h / N);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run("dadd chain", k_dadd);
  run("dsetp+select+dadd chain", k_dsetp_sel);
  run("shfl double chain", k_shfl_d);
  run("shfl int chain", k_shfl_i);
  run("lds chain", k_lds);
  run("dp triangle step", k_step);
  return 0;
}
