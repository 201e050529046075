// Dependent-chain latencies of the operations on the DP's serial path
// (development tool; one warp, clock64 around N dependent operations).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cstdint>

constexpr int N = 4096;

__global__ void probe(double* out_d, long long* out_t, double a, double b, int ia, int ib) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = a + lane;
  sm[lane + 32] = b;
  __syncwarp();
  long long t[16];
  double x = a, y = b;
  // 0: DADD chain
  long long c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) x = __dadd_rn(x, y);
  long long c1 = clock64();
  t[0] = c1 - c0;
  // 1: DSETP + FSEL chain (x = (x < y) ? x' : y' with the result feeding the compare)
  double p = x, q = y + 1.0;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) p = (p < q) ? q : p - 1.0 * 0.0 + 0.0;
  c1 = clock64();
  t[1] = c1 - c0;
  // 2: DADD + DSETP + FSEL (one DP row step: s = min(s, s + y))
  double s = x;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) {
    const double cs = __dadd_rn(s, y);
    s = (cs < q) ? cs : q;
    q = __dadd_rn(q, 0.0);
  }
  c1 = clock64();
  t[2] = c1 - c0;
  // 3: integer 64-bit compare + select chain on double bits
  unsigned long long u = __double_as_longlong(x), v = __double_as_longlong(y);
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) u = (u < v) ? v - 1 : u;
  c1 = clock64();
  t[3] = c1 - c0;
  // 4: SHFL chain (double: two SHFLs)
  double sh = x;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) sh = __shfl_sync(0xffffffffu, sh, (lane + 1) & 31);
  c1 = clock64();
  t[4] = c1 - c0;
  // 5: SHFL int chain
  int si = ia;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) si = __shfl_sync(0xffffffffu, si, (si + lane) & 31);
  c1 = clock64();
  t[5] = c1 - c0;
  // 6: LDS chain (address from the loaded value)
  int idx = lane;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) idx = ((int)sm[idx & 63]) & 63;
  c1 = clock64();
  t[6] = c1 - c0;
  // 7: ISETP + SEL int chain
  int ii = ia;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) ii = (ii < ib) ? ii + 3 : ii - 5;
  c1 = clock64();
  t[7] = c1 - c0;
  // 8: DADD + 64-bit integer compare on the bits + select (the candidate chain alternative)
  double s2 = x;
  unsigned long long qb = __double_as_longlong(q);
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) {
    const double cs = __dadd_rn(s2, y);
    const unsigned long long cb = __double_as_longlong(cs);
    s2 = (cb < qb) ? cs : __longlong_as_double(qb);
    qb += 1;
  }
  c1 = clock64();
  t[8] = c1 - c0;
  // 9: DMUL chain
  double m = x;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) m = __dmul_rn(m, y);
  c1 = clock64();
  t[9] = c1 - c0;
  // 10: FADD chain (fp32)
  float f = (float)x, g = (float)y;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) f = __fadd_rn(f, g);
  c1 = clock64();
  t[10] = c1 - c0;
  // 11: DSETP only chain feeding a predicate combine (ISETP-free): p2 = p2 & (x < y)
  bool pb = true;
  double z = x;
  c0 = clock64();
#pragma unroll 16
  for (int k = 0; k < N; ++k) {
    pb = pb & (z < y);
    z = pb ? y : z;
  }
  c1 = clock64();
  t[11] = c1 - c0;
  if (lane == 0) {
    for (int k = 0; k < 12; ++k) out_t[k] = t[k];
    out_d[0] = x + p + s + (double)u + sh + si + idx + ii + s2 + m + f + z + pb;
  }
}

int main() {
  double* d;
  long long* t;
  cudaMalloc(&d, 64);
  cudaMalloc(&t, 16 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) probe<<<1, 32>>>(d, t, 1.0, 1e-9, 3, 1000000);
  cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"DADD", "DSETP+FSEL", "DADD+DSETP+FSEL", "u64 cmp+sel", "SHFL f64", "SHFL i32",
                         "LDS (dependent)", "ISETP+SEL i32", "DADD+u64cmp+sel", "DMUL", "FADD", "DSETP+PLOP+FSEL"};
  for (int k = 0; k < 12; ++k) printf("%-20s %7.2f cycles/step\n", names[k], (double)h[k] / N);
  return 0;
}
