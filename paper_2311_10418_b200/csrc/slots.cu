// slots.cu — fixed-size plan slots for the multi-GPU epoch gather.
//
// The reference plans an epoch's mini-batches on run_plan's thread pool and
// keeps each MicroBatchPartition (driver.cpp:222-242): per micro-batch the
// sample ids in order (make_micro_batch, microbatch.cpp:122-134), the
// objective and t_max_used.  Across GPUs every rank plans a contiguous block
// of mini-batches; one all_gather of equal-size slots then gives every rank
// the epoch's plans.  A slot (int64 words) is
//     [0] micro-batch count  [1] status  [2] t_max_used bits  [3] objective bits
//     [4, 4 + h)            splits, int32 packed (h = ceil(n_max / 2))
//     [4 + h, 4 + 2h)       (with order) the ordering as per-segment sample
//                           indices, int32 packed: micro-batch k holds the
//                           samples order[splits[k-1] .. splits[k]) — the
//                           reference's sample_ids with the input samples
// written by ONE kernel straight from the planner's device outputs (no host
// round trip, no per-field framework copies).
#include <cuda_runtime.h>
#include <stdint.h>

namespace ppb {

__global__ void __launch_bounds__(256)
    pack_slots_kernel(const int32_t* __restrict__ count, const int32_t* __restrict__ status,
                      const double* __restrict__ tmax, const double* __restrict__ obj,
                      const int32_t* __restrict__ splits, const int32_t* __restrict__ order,
                      const int64_t* __restrict__ seg_off, int h, int words,
                      long long* __restrict__ slots) {
  const int s = blockIdx.x;
  const int64_t b0 = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b0);
  long long* row = slots + (size_t)s * words;
  const int st = status[s];
  const int m = st == 0 ? count[s] : 0;
  if (threadIdx.x == 0) {
    row[0] = m;
    row[1] = st;
    row[2] = st == 0 ? __double_as_longlong(tmax[s]) : 0;
    row[3] = st == 0 ? __double_as_longlong(obj[s]) : 0;
  }
  // int32 view of the payload: splits at [0, 2h), the ordering at [2h, 4h)
  int32_t* w = reinterpret_cast<int32_t*>(row + 4);
  for (int k = threadIdx.x; k < 2 * h; k += blockDim.x) w[k] = k < m ? splits[b0 + k] : 0;
  if (order)
    for (int k = threadIdx.x; k < 2 * h; k += blockDim.x) w[2 * h + k] = k < n ? order[b0 + k] : 0;
}

cudaError_t launch_pack_slots(const int32_t* count, const int32_t* status, const double* tmax,
                              const double* obj, const int32_t* splits, const int32_t* order,
                              const int64_t* seg_off, int n_seg, int n_max, long long* slots,
                              cudaStream_t st) {
  const int h = (n_max + 1) / 2;
  const int words = 4 + (order ? 2 : 1) * h;
  if (n_seg > 0)
    pack_slots_kernel<<<n_seg, 256, 0, st>>>(count, status, tmax, obj, splits, order, seg_off, h, words,
                                             slots);
  return cudaGetLastError();
}

}  // namespace ppb
