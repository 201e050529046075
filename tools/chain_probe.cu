// Cycles per triangle step of the DP chain warp (development tool).
//   nvcc -std=c++17 -O3 --fmad=false -gencode arch=compute_100a,code=sm_100a \
//        -Ipaper_2311_10418_b200/csrc -Iinclude -o build/chain_probe tools/chain_probe.cu
// One warp alone on the GPU runs NB 32-row triangles of MODE 3 (bound +
// candidate) over a fixed shared-memory unit, with the dp_fold.cuh
// arithmetic; each variant reports clock64 cycles per step.
//   V0  dp.cu's redundant chain: every lane recomputes state[k] from H_k
//       (lane k's accumulator shuffled two steps ahead) and T[k, k+1]
//   V1  V0 with plain shared loads instead of volatile ld.shared asm
//   V2  broadcast: lane k's row is complete after folding column k+1, its
//       state is shuffled to every lane (one shuffle round trip per step)
//   V3  V2 with plain shared loads;  V4  V3 without the next block's fold
#include <cstdio>
#include <cstdint>

#include "dp_fold.cuh"
#include "pp_internal.cuh"

using namespace ppb;

constexpr int NB = 64;

template <int V>
__global__ void probe(const double* init, double t, long long* out, double* sink) {
  __shared__ double U[64 * 32];
  const int r = threadIdx.x;
  for (int q = r; q < 64 * 32; q += 32) U[q] = init[q];
  __syncwarp();
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const Acc kIdent{INF, INF, 0, 0x7fffffff};
  Acc A{1e9 + r, 1e9 + r, 5, 0}, N = kIdent;
  const int W = 64, cnx = 32, i0 = 1000;
  auto lds = [&](int idx) {
    if (V == 1 || V == 3 || V == 4) return U[idx];
    return lds_f64(U + idx);
  };
  long long c0 = clock64();
  for (int b = 0; b < NB; ++b) {
    if (V >= 2) {
      double Ss = 0.0, Sx = 0.0;
      int Sc = 0;
#pragma unroll
      for (int k = 31; k >= 0; --k) {
        // fold column k + 1 (state[k+1]) into every row l < k + 1
        if (k + 1 < 32) fold<3, true>(A, lds((k + 1) * 32 + r), Ss, Sx, Sc, i0 + k + 1, r < k + 1, t);
        // lane k's row is complete: state[k]
        const double ns = shfl_f64(A.s, k), nx = shfl_f64(A.x, k);
        const int nc = shfl_i32(A.c, k);
        if (V != 4) fold<3, true>(N, lds((32 + k) * 32 + r), ns, nx, nc, i0 + k, k < cnx, t);
        Ss = ns;
        Sx = nx;
        Sc = nc;
      }
      A.s = __dadd_rn(A.s, Ss * 1e-30);  // keep the block's result live
    } else {
      auto shfl_acc = [&](const Acc& a, int src) {
        Acc h;
        h.s = shfl_f64(a.s, src);
        h.x = shfl_f64(a.x, src);
        h.c = shfl_i32(a.c, src);
        h.j = 0;
        return h;
      };
      Acc H1 = shfl_acc(A, 31), H2 = shfl_acc(A, 30);
      double Ss = 0.0, Sx = 0.0;
      int Sc = 0;
      double x1n = 0.0, xon = lds(31 * 32 + r), xnn = lds((32 + 31) * 32 + r);
#pragma unroll
      for (int k = 31; k >= 0; --k) {
        const double x1 = x1n, xo = xon, xn = xnn;
        if (k > 0) {
          x1n = lds(k * 32 + k - 1);
          xon = lds((k - 1) * 32 + r);
          xnn = lds((32 + k - 1) * 32 + r);
        }
        Acc h = H1;
        if (k + 1 < 32) {
          const unsigned pre = ((k + 1 < W) & (x1 <= t)) ? 1u : 0u;
          const double cs = __dadd_rn(x1, Ss);
          lex_select_desc(cs, 1 + Sc, pre, h.s, h.c);
          const double cb = __dadd_rn(x1, Sx);
          h.x = ((k + 1 < W) & (cb < h.x)) ? cb : h.x;
        }
        const double ns = h.s, nx = h.x;
        fold<3, true>(A, xo, ns, nx, h.c, i0 + k, (r < k) & (k < W), t);
        fold<3, true>(N, xn, ns, nx, h.c, i0 + k, k < cnx, t);
        Ss = ns;
        Sx = nx;
        Sc = h.c;
        H1 = H2;
        if (k >= 2) H2 = shfl_acc(A, k - 2);
      }
      A.s = __dadd_rn(A.s, Ss * 1e-30);
    }
  }
  long long c1 = clock64();
  if (r == 0) out[V] = c1 - c0;
  sink[r] = A.s + N.s + A.x + N.x + A.c + N.c + A.j + N.j;
}

int main() {
  double h[64 * 32];
  unsigned s = 12345;
  for (auto& v : h) {
    s = s * 1664525u + 1013904223u;
    v = 1.0 + (s >> 8) % 1000;
  }
  double *d_init, *d_sink;
  long long* d_out;
  cudaMalloc(&d_init, sizeof h);
  cudaMalloc(&d_sink, 32 * sizeof(double));
  cudaMalloc(&d_out, 8 * sizeof(long long));
  cudaMemcpy(d_init, h, sizeof h, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    probe<0><<<1, 32>>>(d_init, 1e12, d_out, d_sink);
    probe<1><<<1, 32>>>(d_init, 1e12, d_out, d_sink);
    probe<2><<<1, 32>>>(d_init, 1e12, d_out, d_sink);
    probe<3><<<1, 32>>>(d_init, 1e12, d_out, d_sink);
    probe<4><<<1, 32>>>(d_init, 1e12, d_out, d_sink);
    cudaDeviceSynchronize();
  }
  long long o[8];
  cudaMemcpy(o, d_out, sizeof o, cudaMemcpyDeviceToHost);
  const char* names[5] = {"V0 redundant chain (dp.cu)", "V1 V0 + plain smem loads", "V2 broadcast by shuffle",
                          "V3 V2 + plain smem loads", "V4 V3 without the next-block fold"};
  for (int v = 0; v < 5; ++v) printf("%-32s %8.1f cycles/step\n", names[v], (double)o[v] / (NB * 32));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
