// dp.cu — the suffix DP of dp_partition on sm_100a: one CTA per
// (mini-batch, t_max candidate), plus the per-mini-batch candidate selection
// and assembly.
//
// Reference: run_suffix_dp (src/microbatch.cpp:162-189), the candidate loop
// (:281-318), reconstruct_splits (:194-215) and assembly (:322-335).
//
// Row recurrence for a candidate t (state[n] = (0, 0)):
//   state[i] = lexmin over j in (i, n] with T[i,j] <= t, M[i,j] <= cap and
//              state[j] finite of (T[i,j] + state[j].sum, 1 + state[j].count)
// with the reference's strict-improvement rule, i.e. the lowest j among equal
// (sum, count) pairs; that j is next[i].  next[] then *is* reconstruct_splits:
// its front-to-back scan picks the smallest j with T + state[j].sum ==
// state[i].sum && 1 + state[j].count == state[i].count — the lowest-index
// argmin of the row.  Only finite sums can ever be taken (inf/NaN fail both
// `<` and the count tie-break against the initial (inf, 0)), and lexmin over
// (sum, count, j) is associative and commutative, so any reduction order
// yields the reference's state bit-for-bit.
//
// CTA schedule (never changes results).  Rows are processed top-down in
// 32-row blocks; the band of a block is one tile (cost.cu): column c holds
// T[i0 + r, i0 + c] for the 32 rows r.  For block b:
//   * warp 0 (the chain warp) takes the folded far-far partial, the near-far
//     columns [nb, 64) (four interleaved accumulators) and then runs the
//     in-block triangle serially: lane r owns row i0 + r; walking
//     jj = nb-1 .. 0, lane jj's row is final and is broadcast with shuffles,
//     the lanes below fold T[i0 + r, i0 + jj] + state into their
//     accumulators with predicated selects (no divergence, no stores until
//     the block ends);
//   * warps 1..8 (workers) meanwhile reduce the far-far columns [64, W) of
//     block b+1, whose states (j >= i1(b)) are already final, and fold their
//     eight partials into one per row off the chain's critical path;
//   * the near tile (columns [0, 64)) of each block and the far-far columns in
//     32-column chunks are streamed global -> shared by TMA bulk copies
//     (cp.async.bulk, mbarrier completion), issued by one worker thread ahead
//     of use through a ring of chunk buffers, so the serial chain never waits
//     on global memory.
// DP state lives in shared memory, as a ring of R >= W_max + 64 entries when
// the memory cap bounds the row widths.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>

#include "pp_internal.cuh"

namespace ppb {

constexpr int kWorkers = 8;
constexpr int kDpThreads = 32 * (2 + kWorkers);      // chain + workers + producer warp
constexpr int kSyncThreads = 32 * (1 + kWorkers);    // chain + workers (block barrier)
// Warp roles.  The SM sub-partition scheduler picks the highest warp id
// first among eligible warps, so the serial chain warp gets the highest id:
// it is the critical path and must never lose an issue slot to a worker.
constexpr int kProducerWarp = kWorkers;      // warp 8
constexpr int kChainWarp = kWorkers + 1;     // warp 9

#ifdef PP_DP_TRACE
__device__ long long* g_dp_trace = nullptr;  // [block][16] clock64 stamps of CTA 0
#define PP_TRACE(slot)                                                           \
  do {                                                                            \
    if (g_dp_trace && blockIdx.x == 0 && lane == 0) g_dp_trace[b * 16 + (slot)] = clock64(); \
  } while (0)
#else
#define PP_TRACE(slot) \
  do {                 \
  } while (0)
#endif
constexpr int kNearCols = 64;
constexpr int kChunkCols = 32;
constexpr int kMaxRing = 24;
constexpr int kNearBufs = 2;  // near tile of block b in use, b+1 in flight
constexpr uint32_t kColBytes = kRB * sizeof(double);  // 256 B
constexpr size_t kChunkBytes = (size_t)kChunkCols * kColBytes;  // 8 KB

// Shared-memory layout of dp_pass_kernel (offsets in bytes): fixed part,
// then the DP state (when it lives in shared memory), then the ring of far
// chunk buffers, whose depth the launcher sizes to the remaining space.
struct DpSmem {
  static constexpr size_t near = 0;                                   // [3][64][32] double
  static constexpr size_t wps = near + kNearBufs * kNearCols * kColBytes;  // [8][32] double worker partials
  static constexpr size_t wpx = wps + kWorkers * kRB * 8;             // [8][32] double / int
  static constexpr size_t wpj = wpx + kWorkers * kRB * 8;             // [8][32] int
  static constexpr size_t ps = wpj + kWorkers * kRB * 4;              // [2][32] double  folded partial
  static constexpr size_t px = ps + 2 * kRB * 8;                      // [2][32] double / int
  static constexpr size_t pj = px + 2 * kRB * 8;                      // [2][32] int
  static constexpr size_t nps = pj + 2 * kRB * 4;                     // [8][32] double  near-far partials
  static constexpr size_t npx = nps + kWorkers * kRB * 8;             // [8][32] double / int
  static constexpr size_t npj = npx + kWorkers * kRB * 8;             // [8][32] int
  // MODE 3 (fused bound + candidate): the bound sums' partials
  static constexpr size_t npb = npj + kWorkers * kRB * 4;             // [8][32] double  near-far
  static constexpr size_t wpb = npb + kWorkers * kRB * 8;             // [8][32] double  worker
  static constexpr size_t pb = wpb + kWorkers * kRB * 8;              // [2][32] double  folded
  static constexpr size_t row0 = pb + 2 * kRB * 8;                    // raw state[0] (sum, aux, bound)
  // compact band: column -> window index tables of the near tiles and the
  // ring chunks (int16), and the row widths of the current / next block
  static constexpr size_t cbn = (row0 + 32 + 15) / 16 * 16;           // [2][64] short
  static constexpr size_t cbr = cbn + kNearBufs * kNearCols * 2;      // [kMaxRing][32] short
  static constexpr size_t wrs = cbr + kMaxRing * kChunkCols * 2;      // [2][32] int
  static constexpr size_t bars = (wrs + 2 * kRB * 4 + 15) / 16 * 16;  // mbarriers: near full/empty
  static constexpr size_t state = (bars + 8 * (2 * kNearBufs + 2 * kMaxRing) + 127) / 128 * 128;  // + ring
};

size_t dp_smem_fixed() { return DpSmem::state; }
// DP state arrays (sum; count or minimax) of E = entries + kStatePad slots:
// a ring (R = mask + 1 entries) mirrors its first kStatePad entries after its
// end, so the far-far loop reads a chunk's 32 states at base + q with no
// per-column wrap or clamp; a full array (mask = ~0) just gets the slack.
constexpr int kStatePad = 32;
int dp_state_stride(int entries) { return entries + kStatePad; }
size_t dp_state_bytes(int mode, int entries) {
  return (size_t)(entries + kStatePad) * (mode == 0 ? 12 : mode == 3 ? 20 : 16);
}
size_t dp_chunk_bytes() { return kChunkBytes; }
int dp_max_ring() { return kMaxRing; }

// Far-far chunk sequence helpers: block b has max(0, ceil((W_b - 64) / 32))
// chunks of up to 32 columns starting at column 64.
__device__ __forceinline__ int n_chunks(int W) {
  return W > kNearCols ? (W - kNearCols + kChunkCols - 1) / kChunkCols : 0;
}

// Far-far chunks of a tile that a candidate pass (MODE 0, threshold t) needs:
// all nc of them, or those before the first chunk k whose opening column
// prices above thr = t + 2E on every live row (cost.cu band_run_kernel's
// cmin; capi.cu time_trunc_margin): on a length-sorted segment the exact
// slice time is nondecreasing along a row, so every slice from that column
// on exceeds t and can never pass `x <= t`.  Warp-cooperative (all lanes).
__device__ __forceinline__ int far_chunks_needed(int nc, const double* __restrict__ cmin_blk, double thr,
                                                 int lane) {
  for (int base = 0; base < nc; base += 32) {
    const bool over = (base + lane < nc) && (cmin_blk[base + lane] > thr);
    const unsigned int m = __ballot_sync(0xffffffffu, over);
    if (m) return base + __ffs(m) - 1;
  }
  return nc;
}

// ---- cp.async (8-byte, generic proxy) with mbarrier completion ------------
__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// the mbarrier's phase counts this thread's prior cp.async copies as one of its
// expected arrivals, delivered when they have all landed
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---- in-kernel slice pricing (PRICE != 0) ---------------------------------
// On length-sorted single-input mini-batches (GPT) the band is never
// materialised: slice [i, j) depends only on (d = j - i, in[j-1])
// (pp_internal.cuh SlicePricer), and sorted mini-batches repeat lengths, so
// along a diagonal the same value recurs for every column of a run of equal
// lengths.  A warp walks a range of tile columns of the block whose first row
// is k0; per run it prices the diagonals the run reaches (32 per batch, lane l:
// d = next + l) into a 128-entry ring indexed by d, and lane r reads its entry
// of column c at d = c - r; one-column runs are priced in place (lane r: its
// own slice).  f(c, x, parity) receives lane r's T(k0 + r, k0 + c), NaN when
// the slice's act_mem exceeds the cap.  Same operations as cost pass B's
// band_run_kernel, so the values are the band's bit for bit.
struct WalkScratch {
  double* ring;   // [128]
  double* x;      // [32] staged lengths
  AxisPos* px;    // [32] their sequence brackets
};

template <int LAY, class F>
__device__ __forceinline__ void walk_columns(const DpPrice& pr, const SlicePricer& SP, const double* __restrict__ len,
                                             const AxisPos* __restrict__ pos, int cb, int ce,
                                             const WalkScratch& ws, int lane, F&& f) {
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);
  double prev_x = QNAN;
  AxisPos pe = pr.p0;
  int done = 0;
  for (int c0 = cb; c0 < ce; c0 += 32) {
    const int cq = c0 + lane;
    double xq = QNAN;
    AxisPos pxq = pr.p0;
    if (cq < ce && cq > 0) {
      xq = len[cq];
      pxq = pos[cq];
    }
    ws.x[lane] = xq;
    ws.px[lane] = pxq;
    double xn = __shfl_down_sync(0xffffffffu, xq, 1);
    if (lane == 31) xn = (cq + 1 < ce) ? len[cq + 1] : QNAN;
    // bit q: column c0 + q ends its run (the next column differs or is past the range)
    const unsigned int run_end = __ballot_sync(0xffffffffu, !(xn == xq));
    __syncwarp();
    const int qend = min(32, ce - c0);
    for (int q = 0; q < qend;) {
      const unsigned int e = run_end >> q;
      const int qe = min(e ? q + __ffs(e) - 1 : 31, qend - 1);
      const int cs = c0 + q, cend = c0 + qe;
      const double x = ws.x[q];
      if (!(x == prev_x)) {  // warp-uniform: column cs starts a run of equal lengths
        prev_x = x;
        const AxisPos px = ws.px[q];
        if (0.0 < x) pe = px; else pe = pr.p0;
        if (e & 1u) {  // a one-column run: lane r prices its own slice, d = cs - r
          const int d = cs - lane;
          f(cs, price_slice<LAY>(SP, pr.mbp[min(max(d, 1), pr.max_n)], pe), 0);
          q = qe + 1;
          continue;
        }
        done = cs - 32;
      }
      // price the run's diagonals (done, cend] (d <= 0 entries are never used)
      while (done < cend) {
        const int d = done + 1 + lane;
        ws.ring[d & 127] = price_slice<LAY>(SP, pr.mbp[min(max(d, 1), pr.max_n)], pe);
        done += 32;
      }
      __syncwarp();
      int c = cs;
      for (; c + 1 <= cend; c += 2) {
        const double x0 = ws.ring[(c - lane) & 127];
        const double x1 = ws.ring[(c + 1 - lane) & 127];
        f(c, x0, 0);
        f(c + 1, x1, 1);
      }
      if (c <= cend) f(c, ws.ring[(c - lane) & 127], 0);
      __syncwarp();
      q = qe + 1;
    }
  }
}

// (s, c, j) lexmin with lowest-j ties.
__device__ __forceinline__ bool better(double s1, int c1, int j1, double s0, int c0, int j0) {
  return s1 < s0 || (s1 == s0 && (c1 < c0 || (c1 == c0 && j1 < j0)));
}

// MODE 0: DP pass of one t_max candidate: (sum, count, next) per row.
// MODE 1: bound pass (t = +inf): min sum (microbatch.cpp:274-279) and the
//         minimax slice time t* per row (the feasibility threshold).
// MODE 2: the bound pass without the minimax, when a certified lower bound of
//         t* comes from the singleton slices instead (seg_init_kernel).
// MODE 3: MODE 2 fused with the first candidate pass (MODE 0): that candidate
//         (the first >= the singleton bound) is known before the bound, so
//         one pass streams the band once and runs both recurrences — two
//         independent chains interleaved in the same triangle steps.  The
//         candidate result goes to res[item], the bound to res2[segment].
// SMEM_STATE: DP state in shared memory (else an L2-resident global ring).
// SANITIZE: slice times may be -inf (generic SliceCostFn tables).  The
//   reference skips non-finite state[j] (microbatch.cpp:180); states are stored
//   with non-finite sums as +inf, which can never improve a row (x + inf is
//   +inf or NaN), so the hot loops need no finiteness test.  Grid-priced
//   times are >= 0 and never -inf, so only the table path pays for this.
//
// Update rule (microbatch.cpp:183-184): take (x + S[j], 1 + C[j]) when it is
// lexicographically smaller; equal (sum, count) keeps the lowest j.  No
// finiteness test on the sum is needed: +inf or NaN never compares smaller
// than the (+inf, 0) identity or any taken value, -inf is taken exactly when
// the reference takes it.
// PRICE (kLayDec1 / kLayEncDec2; 0 = read the band): no band — the workers
//   price every tile entry themselves (walk_columns above): the near tile of
//   block b+1 into the dense near buffer and the far-far columns of block b+1
//   straight into their reductions, during block b; the producer warp idles.
// PRICE == kGtab: the producer streams the tiles from the call's shared
//   slice table G (gtab.cu: `band` points at G, pr.gbase per sample) with
//   cp.async, 8 B per lane and one tile column per warp instruction; the
//   table is L2-resident, the band does not exist.
template <int MODE, bool SMEM_STATE, bool SANITIZE, bool COMPACT, int PRICE>
__global__ void __launch_bounds__(kDpThreads, 2)
    dp_pass_kernel(const WorkItem* __restrict__ items, const int64_t* __restrict__ seg_off,
                   const int* __restrict__ blk_base, const int* __restrict__ blk_W,
                   const int64_t* __restrict__ tile_off, const int64_t* __restrict__ seg_band_base,
                   const double* __restrict__ band, const double* __restrict__ cand,
                   const int64_t* __restrict__ cand_off, ItemResult* __restrict__ res,
                   int* __restrict__ next_buf, double* __restrict__ gstate, int res_by_seg,
                   int ring_off, int kRing, const double* __restrict__ cmin, double t_margin,
                   unsigned long long* __restrict__ cols_streamed, const short* __restrict__ colbase,
                   const int* __restrict__ chunk_nv, const int* __restrict__ row_w,
                   ItemResult* __restrict__ res2, DpPrice pr) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr bool INK = PRICE == kLayDec1 || PRICE == kLayEncDec2;  // in-kernel pricing
  constexpr bool GTAB = PRICE == kGtab;                           // tiles from the shared table
  double* near = reinterpret_cast<double*>(smem + DpSmem::near);
  double* ring = reinterpret_cast<double*>(smem + ring_off);
  double* wps = reinterpret_cast<double*>(smem + DpSmem::wps);
  int* wpc = reinterpret_cast<int*>(smem + DpSmem::wpx);        // MODE 0
  double* wpm = reinterpret_cast<double*>(smem + DpSmem::wpx);  // MODE 1
  int* wpj = reinterpret_cast<int*>(smem + DpSmem::wpj);
  double* ps = reinterpret_cast<double*>(smem + DpSmem::ps);
  int* pc = reinterpret_cast<int*>(smem + DpSmem::px);          // MODE 0
  double* pm = reinterpret_cast<double*>(smem + DpSmem::px);    // MODE 1
  int* pj = reinterpret_cast<int*>(smem + DpSmem::pj);
  double* nps = reinterpret_cast<double*>(smem + DpSmem::nps);
  int* npc = reinterpret_cast<int*>(smem + DpSmem::npx);        // MODE 0
  double* npm = reinterpret_cast<double*>(smem + DpSmem::npx);  // MODE 1
  int* npj = reinterpret_cast<int*>(smem + DpSmem::npj);
  double* npb = reinterpret_cast<double*>(smem + DpSmem::npb);  // MODE 3
  double* wpb = reinterpret_cast<double*>(smem + DpSmem::wpb);  // MODE 3
  double* pb = reinterpret_cast<double*>(smem + DpSmem::pb);    // MODE 3
  double* row0 = reinterpret_cast<double*>(smem + DpSmem::row0);
  short* cbn = reinterpret_cast<short*>(smem + DpSmem::cbn);
  short* cbr = reinterpret_cast<short*>(smem + DpSmem::cbr);
  int* wrs = reinterpret_cast<int*>(smem + DpSmem::wrs);
  uint64_t* near_full = reinterpret_cast<uint64_t*>(smem + DpSmem::bars);
  uint64_t* near_empty = near_full + kNearBufs;
  uint64_t* ring_full = near_full + 2 * kNearBufs;
  uint64_t* ring_empty = ring_full + kMaxRing;

  const WorkItem it = items[blockIdx.x];
  const int s = it.seg;
  const int64_t b0 = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b0);
  const int gb0 = blk_base[s];
  const int nblk = blk_base[s + 1] - gb0;
  const double t = item_t(it, cand, cand_off);
  const double* bseg = band + seg_band_base[s];
  // candidate passes on certified tiles stream only the far chunks that can
  // hold a slice time <= t (thr = +inf or cmin == null: all of them)
  const bool trunc = MODE == 0 && cmin != nullptr;
  const double thr = trunc ? __dadd_ru(t, t_margin) : __longlong_as_double(0x7ff0000000000000LL);
  auto far_nc = [&](int gb, int W) {
    const int nc = n_chunks(W);
    return trunc ? far_chunks_needed(nc, cmin + chunk_id0(seg_band_base[s] + tile_off[gb], gb) + 2, thr,
                                     threadIdx.x & 31)
                 : nc;
  };
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  const double QNAN = __longlong_as_double(0x7ff8000000000000LL);
  // CAND: the candidate recurrence (lexmin of (sum, count, j) over T <= t);
  // BSUM: MODE 3's extra bound recurrence (min sum, t = +inf)
  constexpr bool CAND = MODE == 0 || MODE == 3;
  constexpr bool BSUM = MODE == 3;

  // state: ring of R = mask + 1 entries (mask = ~0 when not a ring)
  const unsigned mask = it.state_mask;
  const int entries = it.state_entries;
  double* st_s = SMEM_STATE ? reinterpret_cast<double*>(smem + DpSmem::state) : gstate + it.state_off;
  int* st_c = reinterpret_cast<int*>(st_s + (BSUM ? 2 : 1) * (entries + kStatePad));  // CAND
  double* st_m = st_s + entries + kStatePad;                                         // MODE 1
  double* st_b = st_s + entries + kStatePad;                                         // MODE 3
  const bool ring_state = mask != ~0u;
  // state slot of row j: j mod R on a ring of R = entries slots (R is only a
  // multiple of 32 sized to the widest tile, not a power of two): one modulo
  // per block and role; offsets below R from a block's base wrap once
  auto slot = [&](int j) { return ring_state ? j % entries : j; };
  auto wrap = [&](int e) { return (ring_state && e >= entries) ? e - entries : e; };
  int* nxt = next_buf + it.next_off;

  // ---- prologue
  if (threadIdx.x == 0) {
    for (int k = 0; k < kNearBufs; ++k) {
      mbar_init(&near_full[k], GTAB ? 32 : 1);  // GTAB: one cp.async arrive per producer lane
      mbar_init(&near_empty[k], 1);   // the chain warp releases a near tile
    }
    for (int k = 0; k < kRing; ++k) {
      mbar_init(&ring_full[k], GTAB ? 32 : 1);
      mbar_init(&ring_empty[k], kWorkers);  // every worker warp releases a chunk
    }
    mbar_fence_init();
    // state[n] = {0.0, 0} (microbatch.cpp:174), and its ring mirror
    for (int e = slot(n); ; e += entries) {
      st_s[e] = 0.0;
      if (CAND) st_c[e] = 0; else if (MODE == 1) st_m[e] = -INF;
      if (BSUM) st_b[e] = 0.0;
      if (!(ring_state && e < kStatePad)) break;
    }
    row0[0] = INF;
    row0[1] = CAND ? 0.0 : INF;
    row0[2] = INF;
  }
  if (wid == 0) {  // block 0 has no far-far columns (j <= n < i0 + 64)
    ps[lane] = INF;
    if (BSUM) pb[lane] = INF;
    if (CAND) {
      pc[lane] = 0;
      pj[lane] = INT_MAX;
    } else {
      if (MODE == 1) pm[lane] = INF;
    }
  }
  // PRICE: the pricer's cells (decoder kind, + encoder kind for kLayEncDec2)
  // staged in shared memory at ring_off, then per worker warp a diagonal ring
  // and the staged lengths of its current columns
  SlicePricer SP{};
  WalkScratch ws{};
  if (INK) {
    const int cells = pr.cells;
    double4* s_tt = reinterpret_cast<double4*>(smem + ring_off);
    double2* s_am = reinterpret_cast<double2*>(s_tt + (PRICE == kLayEncDec2 ? 2 : 1) * cells);
    for (int k = threadIdx.x; k < cells; k += blockDim.x) {
      s_tt[k] = pr.P.tt_d[k];
      s_am[k] = pr.P.am_d[k];
      if (PRICE == kLayEncDec2) {
        s_tt[cells + k] = pr.P.tt_e[k];
        s_am[cells + k] = pr.P.am_e[k];
      }
    }
    SP = pr.P;
    SP.tt_d = s_tt;
    SP.am_d = s_am;
    SP.tt_e = s_tt + cells;
    SP.am_e = s_am + cells;
    double* wbase = reinterpret_cast<double*>(s_am + (PRICE == kLayEncDec2 ? 2 : 1) * cells);
    const int w = wid < kWorkers ? wid : 0;
    ws.ring = wbase + w * (128 + 32 + 64);
    ws.x = ws.ring + 128;
    ws.px = reinterpret_cast<AxisPos*>(ws.x + 32);
  }
  __syncthreads();
  const double* seg_len = INK ? pr.in_d + b0 - 1 : nullptr;  // + row i0 + column c: in[i0 + c - 1]
  const AxisPos* seg_pos = INK ? pr.pin + b0 - 1 : nullptr;
  // PRICE: the dense near tile (columns [0, min(64, W)) of block bb, first
  // row k0) into near buffer bb % 2; worker w prices columns [8w, 8w + 8)
  auto price_near = [&](int bb) {
    const int kk0 = max(0, n - kRB * (bb + 1));
    const int cmax = min(kNearCols, blk_W[gb0 + bb]);
    const int c_lo = min(8 * wid, cmax), c_hi = min(8 * wid + 8, cmax);
    double* dst = near + (size_t)(bb % kNearBufs) * kNearCols * kRB;
    if (c_lo < c_hi)
      walk_columns<INK ? PRICE : kLayDec1>(pr, SP, seg_len + kk0, seg_pos + kk0, c_lo, c_hi, ws, lane,
                                            [&](int c, double x, int) { dst[c * kRB + lane] = x; });
  };
  if (INK) {
    if (wid == kProducerWarp) return;  // (no band to stream)
    if (wid == 0 && lane == 0 && cols_streamed && nblk > 0)
      atomicAdd(cols_streamed, (unsigned long long)min(kNearCols, blk_W[gb0]));
    if (wid < kWorkers && nblk > 0) price_near(0);
    named_bar(1, kSyncThreads);
  }

  // ================= producer warp: TMA bulk copies, in consumption order
  // (near tile of block b, then the far-far chunks of block b, which the
  // workers consume during block b-1), each into a buffer its consumers
  // released through the matching "empty" mbarrier.  It never joins the
  // block barrier, so it runs ahead by up to the ring depth.
  if (!INK && wid == kProducerWarp) {
    // Issue order = consumption order: near tile of block b (used during
    // block b), then the far-far chunks of block b+1 (used by the workers
    // during block b), so far chunks never queue behind a near-buffer wait.
    if (GTAB) {
      // tile column c of the block whose first row is ii0: lane r's entry is
      // G[gbase[sample j - 1] + (c - r)] (d = c - r), column 0 the NaN row
      const double* G = band;
      auto issue_cols = [&](double* dst, int ii0, int c0, int cols) {
        const int c = c0 + lane;
        const long long bq = lane < cols ? (c == 0 ? 31LL : (long long)pr.gbase[b0 + ii0 + c - 1] + c) : 0LL;
        for (int q = 0; q < cols; ++q) {
          const long long base = __shfl_sync(0xffffffffu, bq, q);
          cp_async_8(dst + q * kRB + lane, G + base - lane);
        }
      };
      int islot = 0, iround = 0;
      long long ncols_total = 0;
      for (int b = 0; b < nblk; ++b) {
        const int gb = gb0 + b;
        const int W = blk_W[gb];
        const int nsl = b % kNearBufs;
        const int ncols = min(kNearCols, W);
        const int ii0 = max(0, n - kRB * (b + 1));
        ncols_total += ncols;
        if (b >= kNearBufs) mbar_wait(&near_empty[nsl], ((b / kNearBufs) - 1) & 1);
        issue_cols(near + (size_t)nsl * kNearCols * kRB, ii0, 0, min(ncols, 32));
        if (ncols > 32) issue_cols(near + (size_t)nsl * kNearCols * kRB + 32 * kRB, ii0, 32, ncols - 32);
        cp_async_arrive_noinc(&near_full[nsl]);
        if (b + 1 >= nblk) break;
        const int gn = gb + 1;
        const int Wn = blk_W[gn];
        const int k0n = max(0, n - kRB * (b + 2));
        const int nc = far_nc(gn, Wn);
        ncols_total += nc > 0 ? min(Wn, kNearCols + nc * kChunkCols) - kNearCols : 0;
        for (int k = 0; k < nc; ++k) {
          const int c0 = kNearCols + k * kChunkCols;
          const int cols = min(kChunkCols, Wn - c0);
          if (iround > 0) mbar_wait(&ring_empty[islot], (iround - 1) & 1);
          issue_cols(ring + (size_t)islot * kChunkCols * kRB, k0n, c0, cols);
          cp_async_arrive_noinc(&ring_full[islot]);
          if (++islot == kRing) {
            islot = 0;
            ++iround;
          }
        }
      }
      if (lane == 0 && cols_streamed) atomicAdd(cols_streamed, (unsigned long long)ncols_total);
      return;
    }
    int islot = 0, iround = 0;
    long long ncols_total = 0;  // tile columns streamed (the transitions this pass visits / 32)
    for (int b = 0; b < nblk; ++b) {
      const int gb = gb0 + b;
      const int W = blk_W[gb];
      const int nsl = b % kNearBufs;
      const int ncols = min(kNearCols, W);
      ncols_total += ncols;
      if (lane == 0) {
        if (b >= kNearBufs) mbar_wait(&near_empty[nsl], ((b / kNearBufs) - 1) & 1);
        mbar_expect_tx(&near_full[nsl], ncols * kColBytes);
        tma_load_1d(near + (size_t)nsl * kNearCols * kRB, bseg + tile_off[gb], ncols * kColBytes,
                    &near_full[nsl]);
      }
      if (b + 1 >= nblk) break;
      const int gn = gb + 1;
      const int Wn = blk_W[gn];
      // (the whole warp: far_nc is warp-cooperative; lane 0 issues)
      const int nc = far_nc(gn, Wn);
      ncols_total += nc > 0 ? min(Wn, kNearCols + nc * kChunkCols) - kNearCols : 0;
      if (COMPACT) {
        // far chunks kk = 2 .. nc + 1 are records (pp_internal.cuh); their
        // sizes are read 32 at a time by the whole warp
        const int64_t cid = chunk_id0(seg_band_base[s] + tile_off[gn], gn) + kNearCols / kChunkCols;
        const double* tb = bseg + tile_off[gn] + (size_t)kNearCols * kRB;
        int mynv = 0;
        for (int k = 0; k < nc; ++k) {
          if ((k & 31) == 0) mynv = k + lane < nc ? chunk_nv[cid + k + lane] : 0;
          const int nv = __shfl_sync(0xffffffffu, mynv, k & 31);
          const uint32_t vbytes = (uint32_t)((nv + 1) & ~1) * 8u;  // a multiple of 16 B
          if (lane == 0) {
            if (iround > 0) mbar_wait(&ring_empty[islot], (iround - 1) & 1);
            mbar_expect_tx(&ring_full[islot], vbytes + 64u);
            tma_load_1d(ring + (size_t)islot * kChunkCols * kRB, tb + (size_t)k * kChunkCols * kRB, vbytes,
                        &ring_full[islot]);
            tma_load_1d(cbr + islot * kChunkCols, colbase + (cid + k) * kChunkCols, 64u, &ring_full[islot]);
          }
          if (++islot == kRing) {
            islot = 0;
            ++iround;
          }
        }
      } else if (lane == 0) {
        for (int k = 0; k < nc; ++k) {
          const int c0 = kNearCols + k * kChunkCols;
          const int cols = min(kChunkCols, Wn - c0);
          if (iround > 0) mbar_wait(&ring_empty[islot], (iround - 1) & 1);
          mbar_expect_tx(&ring_full[islot], cols * kColBytes);
          tma_load_1d(ring + (size_t)islot * kChunkCols * kRB, bseg + tile_off[gn] + (size_t)c0 * kRB,
                      cols * kColBytes, &ring_full[islot]);
          if (++islot == kRing) {
            islot = 0;
            ++iround;
          }
        }
      }
    }
    if (lane == 0 && cols_streamed) atomicAdd(cols_streamed, (unsigned long long)ncols_total);
    return;
  }
  int cslot = 0;
  uint32_t cphase = 0;

  for (int b = 0; b < nblk; ++b) {
    const int i1 = n - kRB * b;
    const int i0 = max(0, i1 - kRB);
    const int nb = i1 - i0;

    // ---- phase 1 (workers): near-far columns [nb, min(64, W)) of block b;
    // their states (rows of blocks b-1, b-2 and state[n]) are final.  Worker
    // w takes columns nb + w, nb + w + 8, ...; the chain folds the eight
    // partials.  A few hundred cycles instead of a serial 32-column loop on
    // the chain.
    const double* nt = near + (size_t)(b % kNearBufs) * kNearCols * kRB;
    const int si0 = slot(i0);  // state slot of the block's first row
    if (wid < kWorkers) {
      const int W = blk_W[gb0 + b];
      const int r = lane;
      if (!INK) mbar_wait(&near_full[b % kNearBufs], (b / kNearBufs) & 1);
      double s1 = INF, m1 = INF, b1 = INF;
      int c1 = 0, j1 = INT_MAX;
      const int cnf = min(kNearCols, W);
      for (int c = nb + wid; c < cnf; c += kWorkers) {
        const double x = nt[c * kRB + r];
        const int j = i0 + c;
        const int sj = wrap(si0 + c);  // (c < 64 < R)
        const double cs = __dadd_rn(x, st_s[sj]);
        if (BSUM) {
          const double cb = __dadd_rn(x, st_b[sj]);
          b1 = (cb < b1) ? cb : b1;
        }
        if (CAND) {
          const int cn = 1 + st_c[sj];
          const bool upd = (x <= t) & ((cs < s1) | ((cs == s1) & (cn < c1)));
          s1 = upd ? cs : s1;
          c1 = upd ? cn : c1;
          j1 = upd ? j : j1;
        } else {
          // (NaN / +inf entries never pass the compares: see the far-far loop)
          s1 = (cs < s1) ? cs : s1;
          const double mj = MODE == 1 ? st_m[sj] : 0.0;
          const double v = (x < mj) ? mj : x;
          if (MODE == 1) m1 = (v < m1) ? v : m1;
        }
      }
      const int o = wid * kRB + r;
      nps[o] = s1;
      if (BSUM) npb[o] = b1;
      if (CAND) {
        npc[o] = c1;
        npj[o] = j1;
      } else {
        if (MODE == 1) npm[o] = m1;
      }
    }
    // ---- the chain warp meanwhile loads its far-far partial, waits for its tile
    const int W = blk_W[gb0 + b];
    const int r = lane;
    double as = INF, am = INF, ab = INF;
    int ac = 0, aj = INT_MAX;
    if (wid == kChainWarp) {
      PP_TRACE(0);
      const int pbuf = (b & 1) * kRB + r;
      as = ps[pbuf];
      if (BSUM) ab = pb[pbuf];
      if (CAND) {
        ac = pc[pbuf];
        aj = pj[pbuf];
      } else {
        if (MODE == 1) am = pm[pbuf];
      }
      if (!INK) mbar_wait(&near_full[b % kNearBufs], (b / kNearBufs) & 1);
    }
    named_bar(3, kSyncThreads);

    if (wid == kChainWarp) {
      // ================= chain warp: block b =================
      PP_TRACE(1);
      // fold the 8 near-far partials: a pairwise tree (ILP), lexmin with j
      // ties is associative
      {
        double s8[kWorkers], m8[kWorkers], b8[kWorkers];
        int c8[kWorkers], j8[kWorkers];
#pragma unroll
        for (int v = 0; v < kWorkers; ++v) {
          const int o = v * kRB + r;
          s8[v] = nps[o];
          b8[v] = BSUM ? npb[o] : INF;
          if (CAND) {
            c8[v] = npc[o];
            j8[v] = npj[o];
          } else {
            m8[v] = MODE == 1 ? npm[o] : INF;
          }
        }
#pragma unroll
        for (int h = kWorkers / 2; h >= 1; h /= 2) {
#pragma unroll
          for (int v = 0; v < h; ++v) {
            if (BSUM) b8[v] = (b8[v + h] < b8[v]) ? b8[v + h] : b8[v];
            if (CAND) {
              const bool tk = better(s8[v + h], c8[v + h], j8[v + h], s8[v], c8[v], j8[v]);
              s8[v] = tk ? s8[v + h] : s8[v];
              c8[v] = tk ? c8[v + h] : c8[v];
              j8[v] = tk ? j8[v + h] : j8[v];
            } else {
              s8[v] = (s8[v + h] < s8[v]) ? s8[v + h] : s8[v];
              if (MODE == 1) m8[v] = (m8[v + h] < m8[v]) ? m8[v + h] : m8[v];
            }
          }
        }
        if (BSUM) ab = (b8[0] < ab) ? b8[0] : ab;
        if (CAND) {
          const bool tk = better(s8[0], c8[0], j8[0], as, ac, aj);
          as = tk ? s8[0] : as;
          ac = tk ? c8[0] : ac;
          aj = tk ? j8[0] : aj;
        } else {
          as = (s8[0] < as) ? s8[0] : as;
          if (MODE == 1) am = (m8[0] < am) ? m8[0] : am;
        }
      }
      PP_TRACE(2);
      if (r >= nb) {
        as = INF;
        ac = 0;
        am = INF;
        ab = INF;
      }
      // Step jj: lane jj's row is final; broadcast it, the lanes below absorb
      // T[i0 + r, i0 + jj] + state.  Descending j: equal (sum, count) takes
      // the lower j.  Rows >= nb hold (+inf, 0), which can never be taken, so
      // a full block runs all 32 steps unconditionally.
      // the triangle's tile column jj is read from shared memory inside its
      // step (independent of the chain, so its latency hides under the
      // shuffle) — 32 doubles fewer live registers
      auto tri_step = [&](int jj) {
        const double x = lds_f64(nt + jj * kRB + r);
        double sj = __shfl_sync(0xffffffffu, as, jj);
        if (SANITIZE) sj = isfinite(sj) ? sj : INF;
        const double cs = __dadd_rn(x, sj);
        const bool okb = (jj < W) & (r < jj);
        const bool ok = okb & (CAND ? (x <= t) : true);  // (NaN: fails the `<`s)
        if (BSUM) {  // the bound chain, independent of the candidate chain
          const double bj = __shfl_sync(0xffffffffu, ab, jj);
          const double cb = __dadd_rn(x, bj);
          ab = (okb & (cb < ab)) ? cb : ab;
        }
        if (CAND) {
          const int cn = 1 + __shfl_sync(0xffffffffu, ac, jj);
          const bool upd = ok & ((cs < as) | ((cs == as) & (cn <= ac)));
          as = upd ? cs : as;
          ac = upd ? cn : ac;
          aj = upd ? i0 + jj : aj;
        } else {
          const double mj = MODE == 1 ? __shfl_sync(0xffffffffu, am, jj) : 0.0;
          as = (ok & (cs < as)) ? cs : as;
          const double v = (x < mj) ? mj : x;
          if (MODE == 1) am = (ok & (v < am)) ? v : am;
        }
      };
      if (nb == kRB) {  // every block but the top one of a segment
#pragma unroll
        for (int jj = kRB - 1; jj >= 0; --jj) tri_step(jj);
      } else {
#pragma unroll
        for (int jj = kRB - 1; jj >= 0; --jj)
          if (jj < nb) tri_step(jj);
      }
      // near tile of block b consumed: the warp's reads are ordered before the
      // release (__syncwarp + mbarrier arrive), and the producer's next TMA
      // write into the buffer waits for it (the TMA pipeline WAR pattern)
      __syncwarp();
      if (!INK && lane == 0) mbar_arrive(&near_empty[b % kNearBufs]);
      PP_TRACE(3);
      if (r < nb) {
        const int row = i0 + r;
        const bool f = isfinite(as);
        const int e = wrap(si0 + r);
        const int em = (ring_state && e < kStatePad) ? e + entries : e;  // the ring mirror
        const double sv = (SANITIZE && !f) ? INF : as;
        st_s[e] = sv;
        st_s[em] = sv;
        if (BSUM) {
          st_b[e] = ab;
          st_b[em] = ab;
        }
        if (CAND) {
          st_c[e] = f ? ac : 0;
          st_c[em] = f ? ac : 0;
          nxt[row] = f ? aj : -1;
        } else {
          if (MODE == 1) st_m[e] = am;
          if (MODE == 1) st_m[em] = am;
        }
        if (row == 0) {
          row0[0] = as;
          row0[1] = CAND ? (double)ac : am;
          row0[2] = ab;
        }
      }
    } else {
      // ================= workers: far-far of block b+1 =================
      const int w = wid;
      const int bn = b + 1;
      if (w == 0) PP_TRACE(8);
      if (bn < nblk) {
        const int j1 = n - kRB * bn;
        const int k0 = max(0, j1 - kRB);  // i0 of block b+1
        const int Wn = blk_W[gb0 + bn];
        const int nc = far_nc(gb0 + bn, Wn);
        const int sk0 = slot(k0);  // state slot of block b+1's first row
        double as = INF, am = INF, as2 = INF, am2 = INF, ab = INF, ab2 = INF;
        int ac = 0, aj = INT_MAX, ac2 = 0, aj2 = INT_MAX;
        const int r = lane;

        if (INK) {
          // block b+1's near tile for the chain and phase 1 of the next block ...
          price_near(bn);
          // ... and its far-far columns [64, Weff), worker w a contiguous share
          // of them, priced on the fly into its reductions
          const int Weff = nc > 0 ? min(Wn, kNearCols + nc * kChunkCols) : min(Wn, kNearCols);
          const int F = Weff - kNearCols;
          const int per = F > 0 ? (F + kWorkers - 1) / kWorkers : 0;
          const int cw0 = kNearCols + min(F, w * per), cw1 = kNearCols + min(F, (w + 1) * per);
          if (w == 0 && lane == 0 && cols_streamed)
            atomicAdd(cols_streamed, (unsigned long long)(min(kNearCols, Wn) + max(F, 0)));
          int ecur = wrap(sk0 + cw0), ccur = cw0;  // state slot of the current column
          auto upd = [&](int c, double x, int par) {
            int e = ecur + (c - ccur);
            if (ring_state && e >= entries) e -= entries;
            ecur = e;
            ccur = c;
            const int j = k0 + c;
            const double cs = __dadd_rn(x, st_s[e]);
            double& s_ = par ? as2 : as;
            int& c_ = par ? ac2 : ac;
            int& j_ = par ? aj2 : aj;
            double& m_ = par ? am2 : am;
            if (BSUM) {
              double& b_ = par ? ab2 : ab;
              const double cb = __dadd_rn(x, st_b[e]);
              b_ = (cb < b_) ? cb : b_;
            }
            if (CAND) {
              const int cn = 1 + st_c[e];
              const bool u = (x <= t) & ((cs < s_) | ((cs == s_) & (cn < c_)));
              s_ = u ? cs : s_;
              c_ = u ? cn : c_;
              j_ = u ? j : j_;
            } else {
              s_ = (cs < s_) ? cs : s_;
              const double mj = MODE == 1 ? st_m[e] : 0.0;
              const double v = (x < mj) ? mj : x;
              if (MODE == 1) m_ = (v < m_) ? v : m_;
            }
          };
          if (cw0 < cw1)
            walk_columns<INK ? PRICE : kLayDec1>(pr, SP, seg_len + k0, seg_pos + k0, cw0, cw1, ws, lane, upd);
        }
        for (int k = 0; k < (INK ? 0 : nc); ++k) {
          mbar_wait(&ring_full[cslot], cphase);
          const double* ch = ring + (size_t)cslot * kChunkCols * kRB;
          const int c0 = kNearCols + k * kChunkCols;
          const int cols = min(kChunkCols, Wn - c0);
          // the chunk's states: slots jb .. jb + 31 (ring mirror / slack: no wrap)
          const int jb = wrap(sk0 + c0) + w;  // (c0 < W <= R - 63)
          const double* ss = st_s + jb;
          const int* sc = st_c + jb;
          const double* sm = st_m + jb;
          const double* sb = st_b + jb;
#pragma unroll
          for (int q0 = 0; q0 < kChunkCols; q0 += kWorkers) {
            const int q = q0 + w;
            const int j = k0 + c0 + q;
            // columns past the chunk are masked (NaN never passes x <= t)
            double x;
            if (COMPACT) {  // record of a far chunk (pp_internal.cuh: no masking needed)
              x = (q < cols) ? ch[cbr[cslot * kChunkCols + q] - r] : QNAN;
            } else {
              x = (q < cols) ? ch[q * kRB + r] : QNAN;
            }
            const double cs = __dadd_rn(x, ss[q0]);
            // two accumulators (even / odd q0 step) for ILP; ascending j in each
            double& s_ = (q0 / kWorkers) & 1 ? as2 : as;
            int& c_ = (q0 / kWorkers) & 1 ? ac2 : ac;
            int& j_ = (q0 / kWorkers) & 1 ? aj2 : aj;
            double& m_ = (q0 / kWorkers) & 1 ? am2 : am;
            if (BSUM) {
              double& b_ = (q0 / kWorkers) & 1 ? ab2 : ab;
              const double cb = __dadd_rn(x, sb[q0]);
              b_ = (cb < b_) ? cb : b_;
            }
            if (CAND) {
              const int cn = 1 + sc[q0];
              const bool upd = (x <= t) & ((cs < s_) | ((cs == s_) & (cn < c_)));
              s_ = upd ? cs : s_;
              c_ = upd ? cn : c_;
              j_ = upd ? j : j_;
            } else {
              // an infeasible entry (x NaN) gives cs = NaN and v = NaN, which
              // fail every `<`; x = +inf or state = +inf gives v = +inf, which
              // never beats the running minimum (<= +inf): no separate tests
              s_ = (cs < s_) ? cs : s_;
              const double mj = MODE == 1 ? sm[q0] : 0.0;
              const double v = (x < mj) ? mj : x;
              if (MODE == 1) m_ = (v < m_) ? v : m_;
            }
          }
          __syncwarp();  // the warp's reads of the slot, then its release
          if (lane == 0) mbar_arrive(&ring_empty[cslot]);  // this warp is done with the chunk
          if (++cslot == kRing) {
            cslot = 0;
            cphase ^= 1u;
          }
        }
        if (BSUM) ab = (ab2 < ab) ? ab2 : ab;
        if (CAND) {
          const bool tk = better(as2, ac2, aj2, as, ac, aj);
          as = tk ? as2 : as;
          ac = tk ? ac2 : ac;
          aj = tk ? aj2 : aj;
        } else {
          as = (as2 < as) ? as2 : as;
          if (MODE == 1) am = (am2 < am) ? am2 : am;
        }
        if (w == 0) PP_TRACE(9);
        const int o = w * kRB + r;
        wps[o] = as;
        if (BSUM) wpb[o] = ab;
        if (CAND) {
          wpc[o] = ac;
          wpj[o] = aj;
        } else {
          if (MODE == 1) wpm[o] = am;
        }
        named_bar(2, 32 * kWorkers);
        if (w == 0) {  // fold the 8 worker partials for the chain
#pragma unroll
          for (int v = 1; v < kWorkers; ++v) {
            const int p = v * kRB + r;
            if (BSUM) ab = (wpb[p] < ab) ? wpb[p] : ab;
            if (CAND) {
              if (better(wps[p], wpc[p], wpj[p], as, ac, aj)) {
                as = wps[p];
                ac = wpc[p];
                aj = wpj[p];
              }
            } else {
              as = (wps[p] < as) ? wps[p] : as;
              if (MODE == 1) am = (wpm[p] < am) ? wpm[p] : am;
            }
          }
          const int pb2 = (bn & 1) * kRB + r;
          ps[pb2] = as;
          if (BSUM) pb[pb2] = ab;
          if (CAND) {
            pc[pb2] = ac;
            pj[pb2] = aj;
          } else {
            if (MODE == 1) pm[pb2] = am;
          }
        }
      }
    }
    if (wid == kChainWarp) PP_TRACE(4);
    if (wid == 0) PP_TRACE(10);
    named_bar(1, kSyncThreads);  // chain + workers: block b's states and block b+1's partials
    if (wid == kChainWarp) PP_TRACE(5);
  }
  if (threadIdx.x == 0) {  // after the last block barrier: row0 is final
    ItemResult rr;
    rr.sum0 = row0[0];
    rr.count0 = CAND ? (int)row0[1] : 0;
    rr.feasible = isfinite(row0[0]) ? 1 : 0;
    rr.aux = MODE == 1 ? row0[1] : -__longlong_as_double(0x7ff0000000000000LL);  // (MODE 2: no t*)
    res[res_by_seg ? s : blockIdx.x] = rr;
    if (BSUM) {  // the fused bound pass's result, by segment
      ItemResult rb;
      rb.sum0 = row0[2];
      rb.count0 = 0;
      rb.feasible = isfinite(row0[2]) ? 1 : 0;
      rb.aux = -__longlong_as_double(0x7ff0000000000000LL);
      res2[s] = rb;
    }
  }
}

// After the bound pass: record bound / t* and the first candidate >= t*.
__global__ void seg_init_kernel(const ItemResult* __restrict__ bound_res, int has_bound, int replicas,
                                const int64_t* __restrict__ cand_off, const int* __restrict__ cand_n,
                                const double* __restrict__ cand, const int* __restrict__ active,
                                const SegStats* __restrict__ tsingle, double margin,
                                SegDP* __restrict__ dp, int n_seg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg) return;
  SegDP d;
  d.best_obj = __longlong_as_double(0x7ff0000000000000LL);
  d.best_t = 0.0;
  d.best_count = 0;
  d.valid = 0;
  d.n_cand = cand_n[s];
  d.ref_evals = 0;
  d.pad[0] = d.pad[1] = 0;
  if (!active[s]) {
    d.done = 1;
    d.next_cand = d.n_cand;
    d.bound = 0.0;
    d.tstar = 0.0;
    dp[s] = d;
    return;
  }
  d.done = 0;
  if (has_bound) {
    // has_bound 2: before a fused (MODE 3) pass — the bound arrives with the
    // first wave's results (seg_set_bound_kernel); t* comes from the singletons
    const ItemResult r = has_bound == 1 ? bound_res[s] : ItemResult{};
    d.bound = r.sum0 / (double)replicas;  // microbatch.cpp:278
    // t*, or (MODE 2 bound pass) its certified lower bound: on a length-sorted
    // segment with a certified slice-time surface every slice [a, b) costs at
    // least (exactly) the singleton [i, i+1) of any sample it holds, so
    // t* >= max_i T(i, i+1) exactly and >= (computed max) - 2E as computed;
    // candidates below it are infeasible just the same
    d.tstar = tsingle ? __dsub_rd(dkey_inv(tsingle[s].tsingle), margin) : r.aux;
    // first candidate >= t*: every candidate below it is infeasible (no
    // partition keeps all slices <= t), so the reference only `continue`s
    // there (microbatch.cpp:292) before any best exists.
    const double* c = cand + cand_off[s];
    int lo = 0, hi = d.n_cand;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (c[mid] < d.tstar) lo = mid + 1; else hi = mid;
    }
    d.next_cand = lo;
  } else {
    d.bound = 0.0;
    d.tstar = -__longlong_as_double(0x7ff0000000000000LL);
    d.next_cand = 0;
  }
  if (d.next_cand >= d.n_cand) {
    d.done = 1;
    d.ref_evals = d.n_cand;
  }
  dp[s] = d;
}

// After a fused (MODE 3) pass: the bound of every segment still in the loop.
__global__ void seg_set_bound_kernel(const ItemResult* __restrict__ bound_res, int replicas,
                                     SegDP* __restrict__ dp, int n_seg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seg || dp[s].done) return;
  dp[s].bound = bound_res[s].sum0 / (double)replicas;  // microbatch.cpp:278
}

// Lexicographic compare of two split vectors given as next[] chains from 0
// (std::vector<size_t> operator<, microbatch.cpp:304).  Same counts.
__device__ bool chain_less(const int* a, const int* bb, int n) {
  int i = 0, k = 0;
  while (i < n) {
    const int x = a[i], y = bb[k];
    if (x != y) return x < y;
    i = x;
    k = y;
  }
  return false;
}

// The candidate loop (microbatch.cpp:289-318) over this wave's items of one
// segment, in ascending t.  One CTA per segment.
__global__ void __launch_bounds__(256)
    select_kernel(const WorkItem* __restrict__ items, const ItemResult* __restrict__ res,
                  const int* __restrict__ seg_item_start, const int* __restrict__ seg_item_cnt,
                  const int* __restrict__ next_buf, int* __restrict__ best_next,
                  const int64_t* __restrict__ seg_off, const double* __restrict__ cand,
                  const int64_t* __restrict__ cand_off, int stage_count, int replicas,
                  SegDP* __restrict__ dps) {
  const int s = blockIdx.x;
  const int cnt = seg_item_cnt[s];
  if (cnt == 0) return;
  __shared__ SegDP d;
  __shared__ int copy_from;  // item index whose next[] becomes best (-1 none)
  const int64_t b = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b);
  int* bn = best_next + b;
  if (threadIdx.x == 0) d = dps[s];
  __syncthreads();
  const double ramp = (double)(stage_count - 1);
  const int first = seg_item_start[s];
  for (int k = 0; k < cnt; ++k) {
    const WorkItem it = items[first + k];
    if (threadIdx.x == 0) {
      copy_from = -1;
      const double tm = item_t(it, cand, cand_off);
      if (d.done) {
      } else if (d.valid && __dadd_rn(__dmul_rn(ramp, tm), d.bound) > d.best_obj) {  // :291
        d.done = 1;
        d.ref_evals = it.cand;
      } else {
        const ItemResult r = res[first + k];
        d.next_cand = it.cand + 1;
        if (r.feasible) {
          const double obj = __dadd_rn(stage_count > 1 ? __dmul_rn(ramp, tm) : 0.0,
                                       __ddiv_rn(r.sum0, (double)replicas));  // :293-294
          bool take = false;
          if (!d.valid || obj < d.best_obj) {
            take = true;
          } else if (obj == d.best_obj) {
            if (r.count0 < d.best_count) {
              take = true;
            } else if (r.count0 == d.best_count) {
              if (chain_less(next_buf + it.next_off, bn, n)) {  // :302-308
                copy_from = first + k;
                d.best_t = tm;
              }
            }
          }
          if (take) {
            d.best_obj = obj;
            d.best_count = r.count0;
            d.best_t = tm;
            d.valid = 1;
            copy_from = first + k;
          }
        }
      }
    }
    __syncthreads();
    if (copy_from >= 0) {
      const int* src = next_buf + items[copy_from].next_off;
      for (int q = threadIdx.x; q < n; q += blockDim.x) bn[q] = src[q];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (!d.done) {
      if (d.next_cand >= d.n_cand) {
        d.done = 1;
        d.ref_evals = d.n_cand;
      } else if (d.valid) {
        const double tn = cand[cand_off[s] + d.next_cand];
        if (__dadd_rn(__dmul_rn(ramp, tn), d.bound) > d.best_obj) {
          d.done = 1;
          d.ref_evals = d.next_cand;
        }
      }
    }
    dps[s] = d;
  }
}

// Assembly (microbatch.cpp:322-335): splits, per-micro-batch times,
// eval_objective (front-to-back, :109-120) and t_max_used.  The split chain
// is walked in shared memory; the slice times are fetched in parallel; the
// objective's sum is accumulated front-to-back by one thread (same rounding
// order as the reference).
__global__ void __launch_bounds__(256)
    finalize_kernel(const SegDP* __restrict__ dps, const int* __restrict__ best_next,
                    const int64_t* __restrict__ seg_off, const int* __restrict__ blk_base,
                    const int64_t* __restrict__ tile_off, const int64_t* __restrict__ seg_band_base,
                    const double* __restrict__ band, const SegStats* __restrict__ stats,
                    const short* __restrict__ colbase, const pp_sample* __restrict__ ordered,
                    int chain_in_smem, int stage_count,
                    int replicas, int32_t* __restrict__ splits, double* __restrict__ mb_times,
                    int32_t* __restrict__ count, double* __restrict__ t_max_used,
                    double* __restrict__ objective, int32_t* __restrict__ status,
                    int64_t* __restrict__ err_id, DpPrice pr, int price_lay) {
  extern __shared__ int chain[];
  __shared__ int m_sh;
  const int s = blockIdx.x;
  const int64_t b = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b);
  const SegDP d = dps[s];
  if (n <= 0) {
    if (threadIdx.x == 0) {
      status[s] = PP_ERR_INVALID;
      count[s] = 0;
      err_id[s] = -1;
    }
    return;
  }
  const int err = stats[s].err_row;
  if (err != INT_MAX) {
    if (threadIdx.x == 0) {
      status[s] = PP_ERR_INFEASIBLE_SAMPLE;
      err_id[s] = ordered[b + err].id;
      count[s] = 0;
    }
    return;
  }
  if (!d.valid) {
    if (threadIdx.x == 0) {
      status[s] = PP_ERR_INFEASIBLE;
      err_id[s] = -1;
      count[s] = 0;
    }
    return;
  }
  const int* bn = best_next + b;
  const int* ch = bn;
  if (chain_in_smem) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) chain[q] = bn[q];
    __syncthreads();
    ch = chain;
  }
  int32_t* sp = splits + b;
  if (chain_in_smem == 2) {
    // hop tables next^2, next^4, next^8 (built in parallel); one thread walks
    // the chain 8 splits per dependent shared-memory load, leaving a
    // checkpoint every 8 splits, and the block expands the checkpoints in
    // parallel (8 dependent loads each)
    // three n-int buffers (two CTAs per SM at n = 8192): h2 and h8 share
    // one, and the checkpoints reuse h4's once h8 is built
    int* h1 = chain;
    int* h2 = chain + n;
    int* h4 = chain + 2 * n;
    int* h8 = h2;
    int* ck = h4;  // checkpoints: the node before splits 8k .. 8k + 7
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const int a = h1[q];
      h2[q] = a < n ? h1[a] : n;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const int a = h2[q];
      h4[q] = a < n ? h2[a] : n;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const int a = h4[q];
      h8[q] = a < n ? h4[a] : n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int i = 0, k = 0;
      while (i < n) {
        ck[k++] = i;
        i = h8[i];
      }
      m_sh = k;  // checkpoint count for now
    }
    __syncthreads();
    const int K = m_sh;
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      int node = ck[k];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int nx = h1[node];
        sp[8 * k + q] = nx;
        if (nx >= n) {
          m_sh = 8 * k + q + 1;  // only the last checkpoint reaches n
          break;
        }
        node = nx;
      }
    }
  } else if (threadIdx.x == 0) {  // one dependent load per split
    int i = 0, m = 0;
    while (i < n) {
      const int j = ch[i];
      sp[m++] = j;
      i = j;
    }
    m_sh = m;
  }
  __syncthreads();
  const int m = m_sh;
  const double* bseg = band + seg_band_base[s];
  const int gb0 = blk_base[s];
  double* tt = mb_times + b;
  // slice times of the chosen micro-batches, fetched in parallel; staged in
  // shared memory (over the chain, which is no longer needed) when they fit
  double* tsh = chain_in_smem ? reinterpret_cast<double*>(chain) : nullptr;
  const bool t_in_smem = chain_in_smem && (size_t)m * sizeof(double) <= (size_t)n * sizeof(int) * (chain_in_smem == 2 ? 3 : 1);
  double mx = 0.0;
  // four micro-batches per thread and step: their band loads are independent
  constexpr int kU = 4;
  for (int kb = threadIdx.x; kb < m; kb += kU * blockDim.x) {
    int64_t at[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int k = kb + u * blockDim.x;
      at[u] = -1;
      if (k < m) {
        const int j = sp[k];
        const int i = k ? sp[k - 1] : 0;
        const int bl = (n - 1 - i) / kRB;  // block of row i
        const int i0 = max(0, n - kRB * (bl + 1));
        const int64_t to = __ldg(tile_off + gb0 + bl);
        if (colbase && j - i0 >= 64) {  // compact band: the record of far column chunk (j - i0) / 32
          const int c = j - i0, kk = c >> 5;
          const int64_t id = chunk_id0(seg_band_base[s] + to, gb0 + bl) + kk;
          at[u] = to + (int64_t)kk * (32 * kRB) + __ldg(colbase + id * 32 + (c & 31)) - (i - i0);
        } else {
          at[u] = to + (int64_t)(j - i0) * kRB + (i - i0);
        }
      }
    }
    double v[kU];
    if (price_lay == kGtab) {  // the shared slice table (gtab.cu): G[gbase(j - 1) + (j - i)]
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int k = kb + u * blockDim.x;
        v[u] = 0.0;
        if (k < m) {
          const int j = sp[k];
          const int i = k ? sp[k - 1] : 0;
          v[u] = __ldg(band + __ldg(pr.gbase + b + j - 1) + (j - i));
        }
      }
    } else if (price_lay) {  // no band: price the chosen slices like the DP did (walk_columns)
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int k = kb + u * blockDim.x;
        v[u] = 0.0;
        if (k < m) {
          const int j = sp[k];
          const int i = k ? sp[k - 1] : 0;
          const double x = __ldg(pr.in_d + b + j - 1);
          const AxisPos pe = (0.0 < x) ? pr.pin[b + j - 1] : pr.p0;
          const AxisPos mb = pr.mbp[j - i];
          v[u] = price_lay == kLayDec1 ? price_slice<kLayDec1>(pr.P, mb, pe) : price_slice<kLayEncDec2>(pr.P, mb, pe);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = at[u] >= 0 ? __ldg(bseg + at[u]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int k = kb + u * blockDim.x;
      if (k < m) {
        tt[k] = v[u];
        mx = (mx < v[u]) ? v[u] : mx;
      }
    }
  }
  __syncthreads();  // every thread is past its last chain read
  if (t_in_smem)
    for (int k = threadIdx.x; k < m; k += blockDim.x) tsh[k] = tt[k];
  // max slice time (order-free) ...
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (mx < y) ? y : mx;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double max_t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) max_t = (max_t < red[w]) ? red[w] : max_t;
    // ... and the front-to-back sum of eval_objective (microbatch.cpp:109-120):
    // one dependent add per micro-batch, loads issued ahead of the chain
    const double* src = t_in_smem ? tsh : tt;
    double sum = 0.0;
    int k = 0;
    for (; k + 8 <= m; k += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = src[k + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) sum = __dadd_rn(sum, v[q]);
    }
    for (; k < m; ++k) sum = __dadd_rn(sum, src[k]);
    count[s] = m;
    objective[s] = __dadd_rn(__dmul_rn((double)(stage_count - 1), max_t),
                             __ddiv_rn(sum, (double)replicas));
    t_max_used[s] = isfinite(d.best_t) ? d.best_t : max_t;
    status[s] = PP_OK;
    err_id[s] = -1;
  }
}

// ---------------------------------------------------------------- launchers
#ifdef PP_DP_TRACE
extern "C" int pp_debug_dp_trace(long long* d_buf) {
  return cudaMemcpyToSymbol(g_dp_trace, &d_buf, sizeof(d_buf)) == cudaSuccess ? 0 : 4;
}
#endif
// smem_state = the largest shared-memory DP state of the launch's items
// (0 with state_global: every item's state then lives in gstate).  The chunk
// ring gets the rest of `smem_budget` (4..kMaxRing chunks of 8 KB).
// PRICE shared memory after the fixed part / state: the pricer's cells and
// per worker a 128-entry diagonal ring + 32 staged lengths and brackets.
size_t dp_price_smem(int lay, int cells) {
  return (size_t)(lay == kLayEncDec2 ? 2 : 1) * cells * (sizeof(double4) + sizeof(double2)) +
         (size_t)kWorkers * (128 + 32 + 64) * sizeof(double);
}

// smem_state = the largest shared-memory DP state of the launch's items
// (0 with state_global: every item's state then lives in gstate).  The chunk
// ring gets the rest of `smem_budget` (4..kMaxRing chunks of 8 KB); with
// `price` (in-kernel pricing, no band) there is no chunk ring.
cudaError_t launch_dp_pass(int mode, const WorkItem* items, int n_items, size_t smem_state,
                           int state_global, int sanitize, size_t smem_budget, const int64_t* seg_off,
                           const int* blk_base, const int* blk_W, const int64_t* tile_off,
                           const int64_t* seg_band_base, const double* band, const double* cand,
                           const int64_t* cand_off, ItemResult* res, int* next_buf, double* gstate,
                           int res_by_seg, const double* cmin, double t_margin,
                           unsigned long long* cols_streamed, const short* colbase, const int* chunk_nv,
                           const int* row_w, ItemResult* res2, const DpPrice* price, int price_lay,
                           cudaStream_t st) {
  if (n_items == 0) return cudaSuccess;
  const size_t ring_off = (DpSmem::state + (state_global ? 0 : smem_state) + 127) / 128 * 128;
  int ring = 0;
  size_t smem;
  DpPrice pr{};
  if (price && price_lay != kGtab) {
    pr = *price;
    smem = ring_off + dp_price_smem(price_lay, pr.cells);
  } else {
    if (price) pr = *price;
    ring = (int)std::min<size_t>(kMaxRing, (smem_budget - std::min(smem_budget, ring_off)) / kChunkBytes);
    ring = std::max(ring, 4);
    smem = ring_off + (size_t)ring * kChunkBytes;
  }
  const bool compact = colbase != nullptr;
#define PP_DP_LAUNCH(M, S, Z, C, P)                                                                   \
  do {                                                                                                \
    ensure_dyn_smem((const void*)dp_pass_kernel<M, S, Z, C, P>, smem);                                \
    dp_pass_kernel<M, S, Z, C, P><<<n_items, kDpThreads, smem, st>>>(                                 \
        items, seg_off, blk_base, blk_W, tile_off, seg_band_base, band, cand, cand_off, res, next_buf, \
        gstate, res_by_seg, (int)ring_off, ring, cmin, t_margin, cols_streamed, colbase, chunk_nv,    \
        row_w, res2, pr);                                                                             \
  } while (0)
#define PP_DP_LAUNCH_Z(M, S)                                                 \
  do {                                                                       \
    if (price && price_lay == kGtab) PP_DP_LAUNCH(M, S, false, false, kGtab);              \
    else if (price && price_lay == kLayDec1) PP_DP_LAUNCH(M, S, false, false, kLayDec1);   \
    else if (price) PP_DP_LAUNCH(M, S, false, false, kLayEncDec2);           \
    else if (compact) PP_DP_LAUNCH(M, S, false, true, 0);                    \
    else if (sanitize) PP_DP_LAUNCH(M, S, true, false, 0);                   \
    else PP_DP_LAUNCH(M, S, false, false, 0);                                \
  } while (0)
  if (mode == 0) {
    if (state_global) PP_DP_LAUNCH_Z(0, false); else PP_DP_LAUNCH_Z(0, true);
  } else if (mode == 1) {
    if (state_global) PP_DP_LAUNCH_Z(1, false); else PP_DP_LAUNCH_Z(1, true);
  } else if (mode == 2) {
    if (state_global) PP_DP_LAUNCH_Z(2, false); else PP_DP_LAUNCH_Z(2, true);
  } else {
    if (state_global) PP_DP_LAUNCH_Z(3, false); else PP_DP_LAUNCH_Z(3, true);
  }
#undef PP_DP_LAUNCH_Z
#undef PP_DP_LAUNCH
  return cudaGetLastError();
}

cudaError_t launch_seg_init(const ItemResult* bound_res, int has_bound, int replicas,
                            const int64_t* cand_off, const int* cand_n, const double* cand,
                            const int* active, const SegStats* tsingle, double margin, SegDP* dp,
                            int n_seg, cudaStream_t st) {
  seg_init_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(bound_res, has_bound, replicas, cand_off,
                                                       cand_n, cand, active, tsingle, margin, dp, n_seg);
  return cudaGetLastError();
}


cudaError_t launch_seg_set_bound(const ItemResult* bound_res, int replicas, SegDP* dp, int n_seg,
                                 cudaStream_t st) {
  seg_set_bound_kernel<<<(n_seg + 127) / 128, 128, 0, st>>>(bound_res, replicas, dp, n_seg);
  return cudaGetLastError();
}

cudaError_t launch_select(const WorkItem* items, const ItemResult* res, const int* seg_item_start,
                          const int* seg_item_cnt, const int* next_buf, int* best_next,
                          const int64_t* seg_off, const double* cand, const int64_t* cand_off,
                          int stage_count, int replicas, SegDP* dps, int n_seg, cudaStream_t st) {
  select_kernel<<<n_seg, 256, 0, st>>>(items, res, seg_item_start, seg_item_cnt, next_buf, best_next,
                                       seg_off, cand, cand_off, stage_count, replicas, dps);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const SegDP* dps, const int* best_next, const int64_t* seg_off,
                            const int* blk_base, const int64_t* tile_off, const int64_t* seg_band_base,
                            const double* band, const SegStats* stats, const short* colbase,
                            const pp_sample* ordered, int stage_count, int replicas, int max_n, int n_seg,
                            int32_t* splits,
                            double* mb_times, int32_t* count, double* t_max_used, double* objective,
                            int32_t* status, int64_t* err_id, const DpPrice* price, int price_lay,
                            cudaStream_t st) {
  // 2: the chain and its hop tables (three n-int buffers) in shared memory; 1: the chain only
  const size_t hop_bytes = ((size_t)max_n * 3 + 2) * sizeof(int);
  const int in_smem = hop_bytes <= 200 * 1024 ? 2 : (size_t)max_n * sizeof(int) <= 200 * 1024 ? 1 : 0;
  const size_t smem = in_smem == 2 ? hop_bytes : in_smem ? (size_t)max_n * sizeof(int) : 0;
  ensure_dyn_smem((const void*)finalize_kernel, smem);
  finalize_kernel<<<n_seg, 256, smem, st>>>(dps, best_next, seg_off, blk_base, tile_off, seg_band_base,
                                            band, stats, colbase, ordered, in_smem, stage_count, replicas,
                                            splits, mb_times, count, t_max_used, objective, status,
                                            err_id, price ? *price : DpPrice{}, price ? price_lay : 0);
  return cudaGetLastError();
}

}  // namespace ppb
