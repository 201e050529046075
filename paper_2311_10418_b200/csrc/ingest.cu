// ingest.cu — the data format on the input side of the path (SURVEY.md §8f
// row 3): dataset record files and token-budgeted mini-batches, on the device.
//
//  * load_record_file + load_dataset's truncation (src/workload.cpp:65-103,
//    109-127): `input_len<TAB>target_len` lines, '#' comments and empty lines
//    skipped, ids = record index, std::stoll field semantics (leading
//    whitespace, optional sign, every character consumed, int64 range), the
//    first malformed line reported with its 1-based line number and byte
//    offset (ParseError, include/pipeplan/errors.h:25-40).
//  * the draw_minibatch loop of run_plan (src/driver.cpp:211,
//    src/workload.cpp:129-146): consecutive samples until the running token
//    count reaches the budget (the crossing sample stays).
//
// Byte work, HBM-bound: line starts are found with 16-byte loads and a block
// scan per 32 KB chunk; each line is parsed by one thread (lines are a few
// bytes); record ids come from a device-wide scan.  The mini-batch cut is a
// chain c -> next(c) (binary search on the token prefix sums); the chain
// through 0 is marked by pointer doubling (log2 n rounds of O(n) parallel
// work) instead of a serial walk.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "pp_internal.cuh"

namespace ppb {

namespace {

constexpr int kIngThreads = 256;
constexpr int kBytesPerThread = 128;
constexpr int64_t kChunk = (int64_t)kIngThreads * kBytesPerThread;  // 32 KB per block

__device__ __forceinline__ bool is_start(const unsigned char* b, int64_t p) {
  return p == 0 || b[p - 1] == '\n';
}

// Counts (pass 0) or writes (pass 1) the line starts of one 32 KB chunk.
template <bool WRITE>
__global__ void __launch_bounds__(kIngThreads)
    line_start_kernel(const unsigned char* __restrict__ b, int64_t n, int64_t* __restrict__ block_cnt,
                      const int64_t* __restrict__ block_off, int64_t* __restrict__ starts) {
  using Scan = cub::BlockScan<int, kIngThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t p0 = (int64_t)blockIdx.x * kChunk + (int64_t)threadIdx.x * kBytesPerThread;
  // flags of positions p0 .. p0+127: p is a start iff p == 0 or b[p-1] == '\n'
  uint32_t mask[kBytesPerThread / 32] = {0, 0, 0, 0};
  int cnt = 0;
  if (p0 < n) {
    if (p0 + kBytesPerThread <= n && p0 > 0) {
      const unsigned char prev = b[p0 - 1];
      const uint4* v = reinterpret_cast<const uint4*>(b + p0);
#pragma unroll
      for (int q = 0; q < kBytesPerThread / 16; ++q) {
        const uint4 w = __ldg(v + q);
        const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int k = q * 16 + t * 4 + c;  // byte p0 + k is '\n' -> p0 + k + 1 is a start
            if (((words[t] >> (8 * c)) & 0xff) == '\n' && k + 1 < kBytesPerThread)
              mask[(k + 1) >> 5] |= 1u << ((k + 1) & 31);
          }
      }
      if (prev == '\n') mask[0] |= 1u;
    } else {
      for (int k = 0; k < kBytesPerThread && p0 + k < n; ++k)
        if (is_start(b, p0 + k)) mask[k >> 5] |= 1u << (k & 31);
    }
#pragma unroll
    for (int q = 0; q < kBytesPerThread / 32; ++q) cnt += __popc(mask[q]);
  }
  int before = 0, total = 0;
  Scan(tmp).ExclusiveSum(cnt, before, total);
  if (!WRITE) {
    if (threadIdx.x == 0) block_cnt[blockIdx.x] = total;
    return;
  }
  int64_t o = block_off[blockIdx.x] + before;
#pragma unroll
  for (int q = 0; q < kBytesPerThread / 32; ++q) {
    uint32_t m = mask[q];
    while (m) {
      const int k = __ffs(m) - 1;
      m &= m - 1;
      starts[o++] = p0 + q * 32 + k;
    }
  }
}

__device__ __forceinline__ bool is_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// std::stoll(field, &used) with used == field length (workload.cpp:83-88):
// whitespace* [+-]? digit+ and nothing after; false on no digits, trailing
// characters or int64 overflow (std::out_of_range).
__device__ bool parse_ll(const unsigned char* s, int64_t len, long long& out) {
  int64_t k = 0;
  while (k < len && is_space(s[k])) ++k;
  bool neg = false;
  if (k < len && (s[k] == '+' || s[k] == '-')) {
    neg = s[k] == '-';
    ++k;
  }
  if (k >= len || s[k] < '0' || s[k] > '9') return false;
  // accumulate the magnitude as unsigned; LLONG_MIN's magnitude is 2^63
  unsigned long long mag = 0;
  const unsigned long long lim = neg ? 9223372036854775808ULL : 9223372036854775807ULL;
  for (; k < len && s[k] >= '0' && s[k] <= '9'; ++k) {
    const unsigned d = s[k] - '0';
    if (mag > (lim - d) / 10) return false;  // overflow
    mag = mag * 10 + d;
  }
  if (k != len) return false;
  out = neg ? (long long)(0ULL - mag) : (long long)mag;
  return true;
}

// One thread per line: kind 0 skipped (empty / '#'), 1 record, 2.. errors
// (PP_PARSE_*), the first erroneous line via atomicMin.
// COMPACT = false: records are written at out[L] (ids = line index, right
// when no line is skipped, the common case) and skipped lines are counted.
// COMPACT = true (only when some line was skipped): records are re-parsed
// and written at out[id[L]].
template <bool COMPACT>
__global__ void parse_lines_kernel(const unsigned char* __restrict__ b, int64_t n,
                                   const int64_t* __restrict__ starts, int64_t n_lines, int8_t* __restrict__ kind,
                                   const int32_t* __restrict__ id, long long max_seq_len, int64_t capacity,
                                   pp_sample* __restrict__ out, unsigned long long* __restrict__ first_err,
                                   unsigned long long* __restrict__ skipped) {
  int my_skip = 0;
  for (int64_t L = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; L < n_lines;
       L += (int64_t)gridDim.x * blockDim.x) {
    if (COMPACT && kind[L] != 1) continue;
    const int64_t a = starts[L];
    const int64_t e = L + 1 < n_lines ? starts[L + 1] - 1 : (b[n - 1] == '\n' ? n - 1 : n);
    const unsigned char* s = b + a;
    const int64_t len = e - a;
    int k = 0;
    long long x = 0, y = 0;
    if (len == 0 || s[0] == '#') {
      k = 0;
    } else {
      int64_t tab = -1;
      for (int64_t q = 0; q < len; ++q)
        if (s[q] == '\t') { tab = q; break; }
      if (tab < 0) k = 2 + PP_PARSE_MISSING_TAB;
      else if (!parse_ll(s, tab, x) || !parse_ll(s + tab + 1, len - tab - 1, y)) k = 2 + PP_PARSE_NOT_INTEGERS;
      else if (x < 1) k = 2 + PP_PARSE_INPUT_LT_1;
      else if (y < 0) k = 2 + PP_PARSE_TARGET_LT_0;
      else k = 1;
    }
    const int64_t r = COMPACT ? (int64_t)id[L] : L;
    // load_dataset truncates input and target independently (workload.cpp:123-126)
    if (k == 1 && r < capacity) out[r] = pp_sample{r, min(x, max_seq_len), min(y, max_seq_len)};
    if (!COMPACT) {
      kind[L] = (int8_t)k;
      my_skip += k == 0;
      if (k >= 2) atomicMin(first_err, (unsigned long long)L);
    }
  }
  if (!COMPACT) {
    for (int o = 16; o; o >>= 1) my_skip += __shfl_xor_sync(0xffffffffu, my_skip, o);
    if ((threadIdx.x & 31) == 0 && my_skip) atomicAdd(skipped, (unsigned long long)my_skip);
  }
}

__global__ void record_flag_kernel(const int8_t* __restrict__ kind, int64_t n_lines, int32_t* __restrict__ flag) {
  for (int64_t L = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; L < n_lines;
       L += (int64_t)gridDim.x * blockDim.x)
    flag[L] = kind[L] == 1 ? 1 : 0;
}

// ---- draw_minibatch chain ----
__global__ void tokens_kernel(const pp_sample* __restrict__ s, int64_t n, long long* __restrict__ tok) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    tok[k] = (long long)s[k].input_len + (long long)s[k].target_len;  // Sample::total_tokens
}

// next(c): the cursor after the mini-batch drawn at c: the smallest m > c
// with P[m] - P[c] >= budget (the crossing sample m-1 stays), else n.
// P is the inclusive-from-0 prefix (P[0] = 0, n+1 entries).  The running sum
// of the reference is P[m] - P[c] exactly (int64 sums of the same terms).
__global__ void next_cursor_kernel(const long long* __restrict__ P, int64_t n, long long budget,
                                   int64_t* __restrict__ nxt, uint8_t* __restrict__ mark) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= n; c += (int64_t)gridDim.x * blockDim.x) {
    if (c == n) { nxt[c] = n; mark[c] = 0; continue; }
    const long long want = P[c] + budget;
    int64_t lo = c + 1, hi = n;  // answer in [c+1, n]
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (P[mid] >= want) hi = mid; else lo = mid + 1;
    }
    nxt[c] = lo;
    mark[c] = c == 0 ? 1 : 0;
  }
}

// one doubling round: marked c marks J(c); J2 = J o J.  Marks set during the
// round are path nodes too, so the race is benign.
__global__ void chain_round_kernel(const int64_t* __restrict__ J, int64_t n, uint8_t* mark, int64_t* __restrict__ J2) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= n; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = J[c];
    if (mark[c] && j < n) mark[j] = 1;
    J2[c] = j < n ? J[j] : n;
  }
}

int grid_for(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 32));
}

}  // namespace

// Scratch needs of ingest (bytes), for the ctx to size one buffer.
size_t ingest_scratch_bytes(int64_t n_bytes) {
  const int64_t blocks = (n_bytes + kChunk - 1) / kChunk;
  const int64_t max_lines = n_bytes + 1;
  size_t t1 = 0, t2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, (int64_t*)nullptr, (int64_t*)nullptr, (int)(blocks + 1));
  cub::DeviceScan::ExclusiveSum(nullptr, t2, (int32_t*)nullptr, (int32_t*)nullptr,
                                (int)std::min<int64_t>(max_lines + 1, INT32_MAX));
  size_t b = 0;
  b += (size_t)(blocks + 1) * 8 * 2;                 // block counts / offsets
  b += (size_t)max_lines * (8 + 1) + 2 * ((size_t)max_lines + 1) * 4;  // starts, kind, flag, id
  b += std::max(t1, t2) + 32 * 256;                  // cub temp + alignment slack
  return b;
}

// Parses `n` bytes at d_bytes into d_out (capacity samples).  Fills
// n_records, n_lines, first_err_line (-1: none, 0-based), its kind and byte.
cudaError_t launch_load_records(const unsigned char* d_bytes, int64_t n, long long max_seq_len, char* scratch,
                                size_t scratch_bytes, pp_sample* d_out, int64_t capacity, int64_t* n_records,
                                int64_t* n_lines_out, int64_t* err_line, int32_t* err_kind, int64_t* err_byte,
                                cudaStream_t st) {
  *n_records = 0;
  *n_lines_out = 0;
  *err_line = -1;
  *err_kind = 0;
  *err_byte = 0;
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = (n + kChunk - 1) / kChunk;
  char* p = scratch;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  int64_t* bcnt = (int64_t*)take((blocks + 1) * 8);
  int64_t* boff = (int64_t*)take((blocks + 1) * 8);
  unsigned long long* ctr = (unsigned long long*)take(16);  // first error, skipped lines
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, bcnt, boff, (int)(blocks + 1), st);
  void* tmp = take(tb);
  if ((size_t)(p - scratch) > scratch_bytes) return cudaErrorInvalidValue;
  line_start_kernel<false><<<(int)blocks, kIngThreads, 0, st>>>(d_bytes, n, bcnt, nullptr, nullptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(bcnt + blocks, 0, 8, st);
  cub::DeviceScan::ExclusiveSum(tmp, tb, bcnt, boff, (int)(blocks + 1), st);
  int64_t n_lines = 0;
  e = cudaMemcpyAsync(&n_lines, boff + blocks, 8, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *n_lines_out = n_lines;
  if (n_lines == 0) return cudaSuccess;
  int64_t* starts = (int64_t*)take(n_lines * 8);
  int8_t* kind = (int8_t*)take(n_lines);
  if ((size_t)(p - scratch) > scratch_bytes) return cudaErrorInvalidValue;
  line_start_kernel<true><<<(int)blocks, kIngThreads, 0, st>>>(d_bytes, n, nullptr, boff, starts);
  cudaMemsetAsync(ctr, 0xff, 8, st);
  cudaMemsetAsync(ctr + 1, 0, 8, st);
  parse_lines_kernel<false><<<grid_for(n_lines), 256, 0, st>>>(d_bytes, n, starts, n_lines, kind, nullptr,
                                                               max_seq_len, capacity, d_out, ctr, ctr + 1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  unsigned long long h[2] = {0, 0};
  cudaMemcpyAsync(h, ctr, 16, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (h[0] != ~0ULL) {
    *err_line = (int64_t)h[0];
    int8_t k = 0;
    cudaMemcpyAsync(&k, kind + h[0], 1, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(err_byte, starts + h[0], 8, cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    *err_kind = k - 2;
    return cudaSuccess;
  }
  if (h[1] == 0) {  // no skipped line: records were written in place
    *n_records = n_lines;
    return cudaSuccess;
  }
  // some lines skipped: record ids by a scan, then a compacting re-parse
  int32_t* flag = (int32_t*)take((n_lines + 1) * 4);
  int32_t* id = (int32_t*)take((n_lines + 1) * 4);
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, flag, id, (int)(n_lines + 1), st);
  if (tb2 > tb) tmp = take(tb2);
  if ((size_t)(p - scratch) > scratch_bytes) return cudaErrorInvalidValue;
  record_flag_kernel<<<grid_for(n_lines), 256, 0, st>>>(kind, n_lines, flag);
  cudaMemsetAsync(flag + n_lines, 0, 4, st);
  cub::DeviceScan::ExclusiveSum(tmp, tb2, flag, id, (int)(n_lines + 1), st);
  parse_lines_kernel<true><<<grid_for(n_lines), 256, 0, st>>>(d_bytes, n, starts, n_lines, kind, id, max_seq_len,
                                                              capacity, d_out, nullptr, nullptr);
  int32_t nrec = 0;
  cudaMemcpyAsync(&nrec, id + n_lines, 4, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *n_records = nrec;
  return cudaGetLastError();
}

size_t draw_scratch_bytes(int64_t n) {
  size_t t = 0, t2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, t, (long long*)nullptr, (long long*)nullptr, (int)std::min<int64_t>(n + 1, INT32_MAX));
  cub::DeviceSelect::Flagged(nullptr, t2, thrust::counting_iterator<int64_t>(0), (uint8_t*)nullptr,
                             (int64_t*)nullptr, (int64_t*)nullptr, (int)std::min<int64_t>(n + 1, INT32_MAX));
  return (size_t)(n + 2) * (8 + 8 + 8 + 1) + std::max(t, t2) + 32 * 256;
}

// seg_offsets[0..n_seg] of the mini-batches run_plan draws (cursor 0, budget)
cudaError_t launch_draw_minibatches(const pp_sample* d_samples, int64_t n, long long budget, char* scratch,
                                    size_t scratch_bytes, int64_t* d_seg_offsets, int64_t* n_seg, cudaStream_t st) {
  *n_seg = 0;
  if (n <= 0) return cudaSuccess;
  char* p = scratch;
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) & ~(size_t)255;
    return r;
  };
  long long* P = (long long*)take((n + 1) * 8);
  int64_t* J = (int64_t*)take((n + 1) * 8);
  int64_t* J2 = (int64_t*)take((n + 1) * 8);
  uint8_t* mark = (uint8_t*)take(n + 1);
  int64_t* nsel = (int64_t*)take(8);
  cudaMemsetAsync(P, 0, 8, st);
  tokens_kernel<<<grid_for(n), 256, 0, st>>>(d_samples, n, P + 1);
  size_t tb = 0, tb2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tb, P + 1, P + 1, (int)n, st);
  cub::DeviceSelect::Flagged(nullptr, tb2, thrust::counting_iterator<int64_t>(0), mark, d_seg_offsets, nsel,
                             (int)(n + 1), st);
  void* tmp = take(std::max(tb, tb2));
  if ((size_t)(p - scratch) > scratch_bytes) return cudaErrorInvalidValue;
  cub::DeviceScan::InclusiveSum(tmp, tb, P + 1, P + 1, (int)n, st);
  next_cursor_kernel<<<grid_for(n + 1), 256, 0, st>>>(P, n, budget, J, mark);
  for (int64_t hop = 1; hop < n; hop *= 2) {
    chain_round_kernel<<<grid_for(n + 1), 256, 0, st>>>(J, n, mark, J2);
    int64_t* t = J; J = J2; J2 = t;
  }
  cudaMemsetAsync(mark + n, 1, 1, st);  // the end cursor closes the last mini-batch
  cub::DeviceSelect::Flagged(tmp, tb2, thrust::counting_iterator<int64_t>(0), mark, d_seg_offsets, nsel,
                             (int)(n + 1), st);
  int64_t k = 0;
  cudaMemcpyAsync(&k, nsel, 8, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  *n_seg = k - 1;
  return cudaGetLastError();
}

}  // namespace ppb
