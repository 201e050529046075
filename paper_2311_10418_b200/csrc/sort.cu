// sort.cu — segmented order_samples(Sort) for sm_100a.
//
// Reference: order_samples(mb, OrderMethod::Sort), src/microbatch.cpp:97-105:
// std::sort by std::tie(input_len, target_len, id).  A stable LSD radix sort
// over the key (input, target, id) reproduces that order exactly: the key is
// a strict total order whenever ids are unique, and fully-equal keys are
// indistinguishable samples.
//
// Key construction: each field is biased by its minimum over the call, so any
// int64 values work.  When the three bias-ed widths fit 64 bits (every
// BASELINE config: 13+13+23 bits) the key is packed into one word; otherwise
// the sort runs over three words (id, then target, then input — LSD order).
//
// One CTA per segment.  Keys and the index payload live in shared memory when
// the segment fits (n <= 8192 with one key word), otherwise in a global
// scratch ping-pong buffer.  2-bit digits; the per-tile digit ranks come from
// one block-wide exclusive scan of four packed 16-bit counters.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "pp_internal.cuh"

namespace ppb {

namespace {

constexpr int kSortThreads = 512;
constexpr int kSortIPT = 8;  // items per thread per tile
constexpr int kTile = kSortThreads * kSortIPT;

struct FieldRange {
  long long mn[3];  // input, target, id
  long long mx[3];
};

__global__ void range_init_kernel(unsigned long long* r) {
  if (threadIdx.x < 7) r[threadIdx.x] = threadIdx.x < 3 ? ~0ULL : 0ULL;
}
__global__ void range_out_kernel(const unsigned long long* r, unsigned long long* h) {
  if (threadIdx.x < 7) h[threadIdx.x] = r[threadIdx.x];
}

__global__ void field_range_kernel(const pp_sample* __restrict__ s, int64_t n,
                                   unsigned long long* out /* 6 words, biased; [6]: ids unordered */) {
  long long mn[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
  long long mx[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  int unordered = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const pp_sample v = s[k];
    if (k + 1 < n) unordered |= s[k + 1].id <= v.id;
    const long long f[3] = {v.input_len, v.target_len, v.id};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      mn[q] = min(mn[q], f[q]);
      mx[q] = max(mx[q], f[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    for (int o = 16; o; o >>= 1) {
      mn[q] = min(mn[q], __shfl_xor_sync(0xffffffffu, mn[q], o));
      mx[q] = max(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], o));
    }
  }
  // block reduction first: one atomic per block and field (the 7 words are
  // shared by every block of the call)
  __shared__ long long wmn[32][3], wmx[32][3];
  __shared__ int wuo[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int uo = __any_sync(0xffffffffu, unordered);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      wmn[wid][q] = mn[q];
      wmx[wid][q] = mx[q];
    }
    wuo[wid] = uo;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    const int q = threadIdx.x;
    long long a = wmn[0][q], b = wmx[0][q];
    for (int w = 1; w < nw; ++w) {
      a = min(a, wmn[w][q]);
      b = max(b, wmx[w][q]);
    }
    // signed -> order-preserving unsigned
    atomicMin(&out[q], (unsigned long long)a ^ 0x8000000000000000ULL);
    atomicMax(&out[3 + q], (unsigned long long)b ^ 0x8000000000000000ULL);
  } else if (threadIdx.x == 3) {
    int any = 0;
    for (int w = 0; w < nw; ++w) any |= wuo[w];
    if (any) atomicOr(&out[6], 1ULL);
  }
}

__device__ __forceinline__ int bit_width(unsigned long long range) {
  return range == 0 ? 0 : 64 - __clzll(range);
}

// Exclusive block scan of one uint64 per thread (packed counters).
__device__ __forceinline__ unsigned long long block_exscan(unsigned long long v,
                                                           unsigned long long* warp_tot,
                                                           unsigned long long& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    unsigned long long w = lane < nw ? warp_tot[lane] : 0ULL;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_tot[lane] = w;  // inclusive
  }
  __syncthreads();
  const unsigned long long before = wid ? warp_tot[wid - 1] : 0ULL;
  total = warp_tot[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before + x - v;
}

// One stable LSD pass on `n` items: digit = (key[item*W + w] >> sh) & 3.
template <int W, bool V = true, class KT = unsigned long long, class VT = uint32_t>
__device__ void radix_pass(const KT* __restrict__ kin, const VT* __restrict__ vin,
                           KT* __restrict__ kout, VT* __restrict__ vout, int n,
                           int w, int sh, unsigned long long* warp_tot, int* bucket) {
  // bucket totals
  if (threadIdx.x < 4) bucket[threadIdx.x] = 0;
  __syncthreads();
  int c[4] = {0, 0, 0, 0};
  for (int k = threadIdx.x; k < n; k += blockDim.x) ++c[(kin[(size_t)k * W + w] >> sh) & 3];
#pragma unroll
  for (int d = 0; d < 4; ++d)
    if (c[d]) atomicAdd(&bucket[d], c[d]);
  __syncthreads();
  int base[4];
  base[0] = 0;
  base[1] = bucket[0];
  base[2] = base[1] + bucket[1];
  base[3] = base[2] + bucket[2];
  __syncthreads();
  int running[4] = {0, 0, 0, 0};
  for (int t0 = 0; t0 < n; t0 += kTile) {
    const int beg = t0 + threadIdx.x * kSortIPT;
    uint8_t dig[kSortIPT];
    unsigned long long cnt = 0;  // four 16-bit counters
#pragma unroll
    for (int q = 0; q < kSortIPT; ++q) {
      const int k = beg + q;
      dig[q] = 0xff;
      if (k < n) {
        dig[q] = (uint8_t)((kin[(size_t)k * W + w] >> sh) & 3);
        cnt += 1ULL << (16 * dig[q]);
      }
    }
    unsigned long long tot;
    unsigned long long pre = block_exscan(cnt, warp_tot, tot);
#pragma unroll
    for (int q = 0; q < kSortIPT; ++q) {
      const int k = beg + q;
      if (k < n) {
        const int d = dig[q];
        const int pos = base[d] + running[d] + (int)((pre >> (16 * d)) & 0xffff);
        pre += 1ULL << (16 * d);
#pragma unroll
        for (int x = 0; x < W; ++x) kout[(size_t)pos * W + x] = kin[(size_t)k * W + x];
        if (V) vout[pos] = vin[k];
      }
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) running[d] += (int)((tot >> (16 * d)) & 0xffff);
  }
  __syncthreads();
}

// One stable LSD pass with a 7-bit digit (one key word): warp w owns the
// contiguous item range [w * per, (w + 1) * per) and ranks its items 32 at a
// time with __match_any_sync (peers with the same digit; rank = peers below
// this lane) against warp-private counters in shared memory; an exclusive
// scan over (digit, warp) in digit-major order turns the counts into
// starting positions, and a second sweep scatters.  Items keep their order
// within a digit (warps own contiguous ranges, ranks follow lane order), so
// the pass is stable: two passes sort a 14-bit key where 2-bit passes took
// seven block scans each.  cnt: [warps][kDig7] ints.
constexpr int kDig7 = 128;
template <class KT, class VT>
__device__ void radix_pass7(const KT* __restrict__ kin, const VT* __restrict__ vin, KT* __restrict__ kout,
                            VT* __restrict__ vout, int n, int sh, int* cnt, unsigned long long* warp_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int per = (n + nw - 1) / nw;
  const int wb = min(n, wid * per), we = min(n, wb + per);
  int* my = cnt + wid * kDig7;
  for (int d = lane; d < kDig7; d += 32) my[d] = 0;
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int k0 = wb; k0 < we; k0 += 32) {
    const int k = k0 + lane;
    const unsigned d = k < we ? (unsigned)((kin[k] >> sh) & (kDig7 - 1)) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d != 0xffffffffu && (peers & lt) == 0) my[d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan over entries e = d * nw + w (digit-major), 4 per thread
  {
    const int total = kDig7 * nw;
    const int e0 = threadIdx.x * 4;
    int v[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = e0 + q;
      v[q] = e < total ? cnt[(e % nw) * kDig7 + e / nw] : 0;
      sum += v[q];
    }
    unsigned long long tot;
    int run = (int)block_exscan((unsigned long long)sum, warp_tot, tot);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = e0 + q;
      if (e < total) cnt[(e % nw) * kDig7 + e / nw] = run;
      run += v[q];
    }
  }
  __syncthreads();
  for (int k0 = wb; k0 < we; k0 += 32) {
    const int k = k0 + lane;
    const bool ok = k < we;
    const unsigned d = ok ? (unsigned)((kin[k] >> sh) & (kDig7 - 1)) : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    int pos = 0;
    if (ok) pos = my[d] + __popc(peers & lt);
    __syncwarp();
    if (ok) {
      kout[pos] = kin[k];
      vout[pos] = vin[k];
      if ((peers & lt) == 0) my[d] += __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
}

// Builds keys for segment `seg`, sorts, and gathers ordered samples + SoA
// double lengths.  `range` holds the biased field minima/maxima of the call.
// KT / VT: key and index types.  uint32 keys + uint16 indices (12 B per
// item, two 8192-item CTAs per SM) when the launcher certified that every
// key fits 32 bits (input + target bits <= 32, ids increasing) and n <= 65536.
template <int W, class KT = unsigned long long, class VT = uint32_t>
__global__ void __launch_bounds__(kSortThreads)
    seg_sort_kernel(const pp_sample* __restrict__ in, const int64_t* __restrict__ seg_off,
                    const unsigned long long* __restrict__ range, KT* gkeys,
                    VT* gvals, int use_smem, pp_sample* __restrict__ out,
                    double* __restrict__ in_d, double* __restrict__ tgt_d, int32_t* __restrict__ perm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long warp_tot[kSortThreads / 32];
  __shared__ int bucket[4];
  __shared__ int dig_cnt[W == 1 ? (kSortThreads / 32) * kDig7 : 1];
  const int s = blockIdx.x;
  const int64_t b = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b);
  if (n <= 0) return;
  // field ranges of THIS segment (each is within the call's range, so the
  // key still fits the word count the launcher chose from the call's range):
  // ids of a mini-batch usually span far fewer bits than the call's ids
  __shared__ long long s_rng[kSortThreads / 32][6];
  // ids strictly increasing in input order (the common case: ids are indices):
  // a stable sort on (input, target) alone then yields the (input, target, id)
  // order, with the id bits out of the key
  bool ids_in_order;
  {
    long long lo[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX};
    long long hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
    int unordered = 0;  // some id is not above its predecessor's
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
      const pp_sample v = in[b + k];
      if (k + 1 < n) unordered |= in[b + k + 1].id <= v.id;
      const long long f[3] = {v.input_len, v.target_len, v.id};
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        lo[q] = min(lo[q], f[q]);
        hi[q] = max(hi[q], f[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      for (int o = 16; o; o >>= 1) {
        lo[q] = min(lo[q], __shfl_xor_sync(0xffffffffu, lo[q], o));
        hi[q] = max(hi[q], __shfl_xor_sync(0xffffffffu, hi[q], o));
      }
    }
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        s_rng[threadIdx.x >> 5][q] = lo[q];
        s_rng[threadIdx.x >> 5][3 + q] = hi[q];
      }
    }
    ids_in_order = !__syncthreads_or(unordered);
  }
  long long mn[3];
  int bits[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    long long lo = s_rng[0][q], hi = s_rng[0][3 + q];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = min(lo, s_rng[w][q]);
      hi = max(hi, s_rng[w][3 + q]);
    }
    mn[q] = lo;
    bits[q] = bit_width((unsigned long long)hi - (unsigned long long)lo);
  }
  if (ids_in_order) bits[2] = 0;
  (void)range;
  KT *k0, *k1;
  VT *v0, *v1;
  if (use_smem) {
    k0 = reinterpret_cast<KT*>(smem_raw);
    k1 = k0 + (size_t)n * W;
    v0 = reinterpret_cast<VT*>(k1 + (size_t)n * W);
    v1 = v0 + n;
  } else {
    k0 = gkeys + (size_t)b * W * 2;
    k1 = k0 + (size_t)n * W;
    v0 = gvals + (size_t)b * 2;
    v1 = v0 + n;
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const pp_sample v = in[b + k];
    const unsigned long long fi = (unsigned long long)v.input_len - (unsigned long long)mn[0];
    const unsigned long long ft = (unsigned long long)v.target_len - (unsigned long long)mn[1];
    const unsigned long long fd = ids_in_order ? 0ULL : (unsigned long long)v.id - (unsigned long long)mn[2];
    if (W == 1) {
      // caller checked bits[0]+bits[1]+bits[2] <= 64; guard the 64-bit shifts
      const int s1 = bits[1] + bits[2];
      k0[k] = (KT)((s1 < 64 ? (fi << s1) : 0ULL) | (bits[2] < 64 ? (ft << bits[2]) : 0ULL) | fd);
    } else {
      k0[(size_t)k * W + 0] = fd;
      k0[(size_t)k * W + 1] = ft;
      k0[(size_t)k * W + 2] = fi;
    }
    v0[k] = (VT)k;
  }
  __syncthreads();
  if (W == 1) {
    const int total = bits[0] + bits[1] + bits[2];
    for (int sh = 0; sh < total; sh += 7) {
      radix_pass7<KT, VT>(k0, v0, k1, v1, n, sh, dig_cnt, warp_tot);
      KT* tk = k0; k0 = k1; k1 = tk;
      VT* tv = v0; v0 = v1; v1 = tv;
    }
  } else {
    const int word_bits[3] = {bits[2], bits[1], bits[0]};
    for (int w = 0; w < 3; ++w)
      for (int sh = 0; sh < word_bits[w]; sh += 2) {
        radix_pass<W, true, KT, VT>(k0, v0, k1, v1, n, w, sh, warp_tot, bucket);
        KT* tk = k0; k0 = k1; k1 = tk;
        VT* tv = v0; v0 = v1; v1 = tv;
      }
  }
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const uint32_t src = v0[k];
    const pp_sample v = in[b + src];
    out[b + k] = v;
    in_d[b + k] = (double)v.input_len;
    tgt_d[b + k] = (double)v.target_len;
    if (perm) perm[b + k] = (int32_t)src;
  }
}

// Segmented ascending sort of raw 64-bit keys (candidate t_max values mapped
// by dkey(), exact mode), global-memory ping-pong, one CTA per segment.  Only
// the bits that differ within the segment are sorted.
__global__ void __launch_bounds__(kSortThreads)
    seg_sort_u64_kernel(unsigned long long* keys, unsigned long long* tmp,
                        const int64_t* __restrict__ off, const unsigned long long* __restrict__ cnt,
                        const int* __restrict__ seg_mode, int want_mode, int* __restrict__ in_tmp) {
  __shared__ unsigned long long warp_tot[kSortThreads / 32];
  __shared__ int bucket[4];
  __shared__ unsigned long long diff;
  const int s = blockIdx.x;
  if (seg_mode[s] != want_mode) return;
  const int n = (int)cnt[s];
  unsigned long long* k0 = keys + off[s];
  unsigned long long* k1 = tmp + off[s];
  if (threadIdx.x == 0) diff = 0;
  __syncthreads();
  if (n > 0) {
    const unsigned long long ref = k0[0];
    unsigned long long d = 0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) d |= k0[k] ^ ref;
    for (int o = 16; o; o >>= 1) d |= __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0 && d) atomicOr(&diff, d);
  }
  __syncthreads();
  const int bits = diff ? 64 - __clzll(diff) : 0;
  int parity = 0;
  for (int sh = 0; sh < bits; sh += 2) {
    radix_pass<1, false>(k0, (const uint32_t*)nullptr, k1, (uint32_t*)nullptr, n, 0, sh, warp_tot, bucket);
    unsigned long long* tk = k0; k0 = k1; k1 = tk;
    parity ^= 1;
  }
  if (threadIdx.x == 0) in_tmp[s] = parity;
}

// presorted path: copy + SoA lengths.
// presorted order: position k of a segment holds its sample k
__global__ void iota_seg_kernel(const int64_t* __restrict__ seg_off, int32_t* __restrict__ perm) {
  const int64_t b = seg_off[blockIdx.x], e = seg_off[blockIdx.x + 1];
  for (int64_t k = b + threadIdx.x; k < e; k += blockDim.x) perm[k] = (int32_t)(k - b);
}

__global__ void copy_soa_kernel(const pp_sample* __restrict__ in, int64_t n, pp_sample* out,
                                double* in_d, double* tgt_d) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const pp_sample v = in[k];
    out[k] = v;
    in_d[k] = (double)v.input_len;
    tgt_d[k] = (double)v.target_len;
  }
}

}  // namespace

// Sorts each mode-`want_mode` segment's keys in place (result may end in tmp:
// in_tmp[s] = 1 then).
cudaError_t launch_segmented_sort_u64(unsigned long long* keys, unsigned long long* tmp,
                                      const int64_t* off, const unsigned long long* cnt,
                                      const int* seg_mode, int want_mode, int* in_tmp, int n_seg,
                                      cudaStream_t st) {
  seg_sort_u64_kernel<<<n_seg, kSortThreads, 0, st>>>(keys, tmp, off, cnt, seg_mode, want_mode,
                                                      in_tmp);
  return cudaGetLastError();
}

// Host launcher.  range_buf: 6 device words.  Scratch (gkeys/gvals) must hold
// 2*3*total words / 2*total indices when any segment takes the global path.
cudaError_t launch_segmented_sort(const pp_sample* d_in, const int64_t* d_seg_off,
                                  const int64_t* h_seg_off, int n_seg, int64_t total,
                                  int presorted, unsigned long long* d_range,
                                  unsigned long long* h_range, unsigned long long* d_keys,
                                  uint32_t* d_vals, pp_sample* d_out, double* d_in_len,
                                  double* d_tgt_len, int32_t* d_perm, cudaStream_t st) {
  // Field ranges of the call: they size the sort key and feed the host's
  // monotonicity certificate for the cost passes (capi.cu), so they are
  // computed for presorted calls too.
  // (initialised and read back by one-thread kernels, h_range being pinned:
  // no copy-engine transfer on the planning stream, capi.cu small_copy)
  range_init_kernel<<<1, 32, 0, st>>>(d_range);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
  field_range_kernel<<<blocks, 256, 0, st>>>(d_in, total, d_range);
  range_out_kernel<<<1, 32, 0, st>>>(d_range, h_range);  // 7 words
  if (presorted) {
    const int cb = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    copy_soa_kernel<<<cb, 256, 0, st>>>(d_in, total, d_out, d_in_len, d_tgt_len);
    if (d_perm && n_seg > 0) iota_seg_kernel<<<n_seg, 256, 0, st>>>(d_seg_off, d_perm);
    return cudaStreamSynchronize(st);
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  int bits = 0, fbits[3];
  for (int q = 0; q < 3; ++q) {
    const unsigned long long r = (h_range[3 + q] ^ 0x8000000000000000ULL) -
                                 (h_range[q] ^ 0x8000000000000000ULL);
    fbits[q] = r == 0 ? 0 : 64 - __builtin_clzll(r);
    bits += fbits[q];
  }
  const int W = bits <= 64 ? 1 : 3;
  int64_t max_n = 0;
  for (int s = 0; s < n_seg; ++s) max_n = std::max<int64_t>(max_n, h_seg_off[s + 1] - h_seg_off[s]);
  // ids increasing over the call => increasing in every segment, so each
  // segment's key is (input, target) only: 32-bit keys when those fit
  const bool key32 = h_range[6] == 0 && fbits[0] + fbits[1] <= 32 && max_n <= 65536;
  // one-word keys (radix_pass7, any warp count): small segments take
  // smaller CTAs, more of them per SM (C1: 256 samples per segment)
  const int t1 = max_n <= 1024 ? 128 : max_n <= 4096 ? 256 : kSortThreads;
  if (key32) {
    const size_t need = (size_t)max_n * (2 * 4 + 2 * 2);
    const int sm = need <= 200 * 1024 ? 1 : 0;
    ensure_dyn_smem((const void*)seg_sort_kernel<1, uint32_t, uint16_t>, sm ? need : 0);
    seg_sort_kernel<1, uint32_t, uint16_t><<<n_seg, t1, sm ? need : 0, st>>>(
        d_in, d_seg_off, d_range, reinterpret_cast<uint32_t*>(d_keys), reinterpret_cast<uint16_t*>(d_vals), sm,
        d_out, d_in_len, d_tgt_len, d_perm);
    return cudaGetLastError();
  }
  const size_t smem_need = (size_t)max_n * (2 * 8 * W + 2 * 4);
  const int use_smem = smem_need <= 200 * 1024 ? 1 : 0;
  const size_t smem = use_smem ? smem_need : 0;
  if (W == 1) {
    ensure_dyn_smem((const void*)seg_sort_kernel<1>, smem);
    seg_sort_kernel<1><<<n_seg, t1, smem, st>>>(d_in, d_seg_off, d_range, d_keys, d_vals,
                                                          use_smem, d_out, d_in_len, d_tgt_len, d_perm);
  } else {
    ensure_dyn_smem((const void*)seg_sort_kernel<3>, smem);
    seg_sort_kernel<3><<<n_seg, kSortThreads, smem, st>>>(d_in, d_seg_off, d_range, d_keys, d_vals,
                                                          use_smem, d_out, d_in_len, d_tgt_len, d_perm);
  }
  return cudaGetLastError();
}

}  // namespace ppb
