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
// 32-row blocks; block b's tile (cost.cu band, or the call's slice table G,
// gtab.cu) has column c = T[i0 + r, i0 + c] for its 32 rows r.  Columns split
// into the triangle [0, nb) (in-block j), the near-far columns [nb, nb + 32)
// (j = the previous block's rows), and the far-far columns [64, W).
//   * workers (warps 0..7) reduce the far-far columns of block b+1 while the
//     chain runs block b (their states are final), four contiguous columns per
//     warp and 32-column chunk, and fold their eight partials into one;
//   * the chain warp (warp 9) runs block b's triangle.  Its critical path is
//     the row-to-row dependency state[k] <- T[k, k+1] + state[k+1]: instead of
//     broadcasting each newly final row with a shuffle (a shuffle round trip
//     per row), EVERY lane recomputes state[k] itself from
//       H_k = lane k's accumulator over columns >= k+2 (shuffled one row ahead,
//             off the critical path) and the tile entry T[k, k+1] (a
//             broadcast shared load),
//     with exactly lane k's own operations, so the copies are bit-identical
//     to what lane k stores.  As each state[k] appears, lane l folds
//     T[l, k] + state[k] into its own row (l < k) AND T'[l, nb' + k] into row
//     l of the NEXT block — the next block's near-far columns are reduced on
//     the fly, so no separate near-far phase or partial fold sits between
//     blocks;
//   * the producer warp (warp 8) stages, per block, a 64-column "unit" (the
//     triangle of block u and the near-far columns of block u+1) and, on the
//     band path, the far-far chunks through a ring, with TMA bulk copies and
//     mbarriers; on the slice-table path it fills the units with coalesced
//     loads of G and the workers read their far-far entries from G directly
//     (L2/L1-resident, no ring).
// DP state lives in shared memory (or an L2-resident global array), indexed
// slot(j) = (j + shift) mod R with shift = -n mod 32, so every far-far chunk
// starts at a 32-aligned slot and a worker's four columns load with 16-byte
// vector loads.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <climits>
#include <type_traits>

#include "pp_internal.cuh"
#include "dp_fold.cuh"

namespace ppb {

constexpr int kWorkers = 8;
constexpr int kDpThreads = 32 * (2 + kWorkers);      // workers + producer + chain
// The slice-table path has no producer warp: the workers fill the chain's
// next unit with cp.async at the start of each block (an eighth each) and
// the block barrier hands it over, so the CTA is 9 warps and the register
// cap at two CTAs per SM is 112 instead of 96.
template <bool GTAB>
constexpr int dp_threads() { return GTAB ? 32 * (1 + kWorkers) : kDpThreads; }
constexpr int kSyncThreads = 32 * (1 + kWorkers);    // workers + chain (block barrier)
// Warp roles.  The SM sub-partition scheduler picks the highest warp id
// first among eligible warps, so the serial chain warp gets the highest id:
// it is the critical path and must never lose an issue slot to a worker.
constexpr int kProducerWarp = kWorkers;      // warp 8 (band path)
constexpr int kChainWarp = kWorkers + 1;     // warp 9 (band path; warp 8 on the slice-table path)
// Named barriers: 1 = block barrier (chain + workers; on the slice-table path
// it also hands the chain the unit the workers copied with cp.async);
// 7 + w (w < 4): worker w + 4 hands its far-far partial to worker w.  The
// band path orders its TMA unit and chunk copies through mbarriers.
constexpr int kBarPair = 7;
// 11 + w (w < 2): worker w + 2 hands its (already paired) partial to worker w.
constexpr int kBarPair2 = 11;

#ifdef PP_DP_TRACE
__device__ long long* g_dp_trace = nullptr;  // [block][16] clock64 stamps of CTA 0
__device__ int g_dp_flags = 0;               // bit 0: workers skip the far-far columns (timing only)
#define PP_TRACE(slot)                                                           \
  do {                                                                            \
    if (g_dp_trace && blockIdx.x == 0 && lane == 0) g_dp_trace[b * 16 + (slot)] = clock64(); \
  } while (0)
#else
#define PP_TRACE(slot) \
  do {                 \
  } while (0)
#endif
constexpr int kUnitCols = 64;   // unit u: triangle of block u [0, 32) + near-far of block u+1 [32, 64)
constexpr int kNearCols = 64;   // a tile's far-far columns start here
constexpr int kChunkCols = 32;
constexpr int kMaxRing = 24;
constexpr uint32_t kColBytes = kRB * sizeof(double);  // 256 B
constexpr size_t kChunkBytes = (size_t)kChunkCols * kColBytes;  // 8 KB

// Shared-memory layout of dp_pass_kernel (offsets in bytes): fixed part,
// then the DP state (when it lives in shared memory), then (band path) the
// ring of far chunk buffers, whose depth the launcher sizes to what is left.
// "x" is the second double of a state: the bound sum (MODE 3) or the
// minimax (MODE 1).
struct DpSmem {
  static constexpr size_t unit = 0;                                   // [2][64][32] double
  // worker partials of a block's far-far columns, double-buffered by block
  // parity: [2][8][32] each (the chain folds a block's eight partials)
  static constexpr size_t wps = unit + 2 * kUnitCols * kColBytes;     // double sum
  static constexpr size_t wpx = wps + 2 * kWorkers * kRB * 8;         // double x
  static constexpr size_t wpc = wpx + 2 * kWorkers * kRB * 8;         // int count
  static constexpr size_t wpj = wpc + 2 * kWorkers * kRB * 4;         // int argmin
  static constexpr size_t row0 = wpj + 2 * kWorkers * kRB * 4;        // state[0]: sum, aux, x
  static constexpr size_t bars = (row0 + 32 + 15) / 16 * 16;          // unit full/empty, ring full/empty
  static constexpr size_t state = (bars + 8 * (4 + 2 * kMaxRing) + 127) / 128 * 128;
};

size_t dp_smem_fixed() { return DpSmem::state; }
// DP state: arrays of SE = entries + kStatePad slots (entries a multiple of
// 32): sum (double), x (double: MODE 1 / 3), count (int: MODE 0 / 3).  The
// first kStatePad slots are mirrored after the end, so a chunk's 32 states
// read at base + q with no wrap.
constexpr int kStatePad = 32;
int dp_state_stride(int entries) { return entries + kStatePad; }
size_t dp_state_bytes(int mode, int entries) {
  return (size_t)(entries + kStatePad) * (mode == 0 ? 12 : mode == 1 ? 16 : mode == 2 ? 8 : 20);
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

// MODE 0: DP pass of one t_max candidate: (sum, count, next) per row.
// MODE 1: bound pass (t = +inf): min sum (microbatch.cpp:274-279) and the
//         minimax slice time t* per row (the feasibility threshold).
// MODE 2: the bound pass without the minimax, when a certified lower bound of
//         t* comes from the singleton slices instead (seg_init_kernel).
// MODE 3: MODE 2 fused with the first candidate pass (MODE 0): that candidate
//         (the first >= the singleton bound) is known before the bound, so
//         one pass streams the tiles once and runs both recurrences.  The
//         candidate result goes to res[item], the bound to res2[segment].
// SMEM_STATE: DP state in shared memory (else an L2-resident global array).
// SANITIZE: slice times may be -inf (generic SliceCostFn tables).  The
//   reference skips non-finite state[j] (microbatch.cpp:180); states are used
//   and stored with non-finite sums as +inf, which can never improve a row
//   (x + inf is +inf or NaN), so the hot loops need no finiteness test.
// GTAB: the tiles are views of the call's shared slice table G (gtab.cu:
//   `band` points at G, pr.gbase per ordered sample): column c of the block
//   whose first row is i0 is G[gbase[i0 + c - 1] + c - r] for row r.
template <int MODE, bool SMEM_STATE, bool SANITIZE, bool GTAB>
__global__ void __launch_bounds__(dp_threads<GTAB>(), 2)
    dp_pass_kernel(const WorkItem* __restrict__ items, const int64_t* __restrict__ seg_off,
                   const int* __restrict__ blk_base, const int* __restrict__ blk_W,
                   const int64_t* __restrict__ tile_off, const int64_t* __restrict__ seg_band_base,
                   const double* __restrict__ band, const double* __restrict__ cand,
                   const int64_t* __restrict__ cand_off, ItemResult* __restrict__ res,
                   int* __restrict__ next_buf, double* __restrict__ gstate, int res_by_seg,
                   int ring_off, int kRing, const double* __restrict__ cmin, double t_margin,
                   unsigned long long* __restrict__ cols_streamed, ItemResult* __restrict__ res2,
                   const int* __restrict__ gbase) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr bool CAND = MODE == 0 || MODE == 3;
  constexpr bool X2 = MODE == 1 || MODE == 3;
  // slice-table candidate passes store a state's count as the key
  // (1 + C) << kKeyShift | j (dp_fold.cuh fold_k; the launcher keeps n <= kGtabMaxN)
  constexpr bool KEYED = GTAB && CAND;
  auto cnt_of = [](int v) { return KEYED ? v >> kKeyShift : v; };
  double* unit = reinterpret_cast<double*>(smem + DpSmem::unit);
  double* ring = reinterpret_cast<double*>(smem + ring_off);
  double* wps = reinterpret_cast<double*>(smem + DpSmem::wps);
  double* wpx = reinterpret_cast<double*>(smem + DpSmem::wpx);
  int* wpc = reinterpret_cast<int*>(smem + DpSmem::wpc);
  int* wpj = reinterpret_cast<int*>(smem + DpSmem::wpj);
  double* row0 = reinterpret_cast<double*>(smem + DpSmem::row0);
  uint64_t* unit_full = reinterpret_cast<uint64_t*>(smem + DpSmem::bars);
  uint64_t* unit_empty = unit_full + 2;
  uint64_t* ring_full = unit_full + 4;
  uint64_t* ring_empty = ring_full + kMaxRing;

  const WorkItem it = items[blockIdx.x];
  const int s = it.seg;
  const int64_t b0 = seg_off[s];
  const int n = (int)(seg_off[s + 1] - b0);
  const int gb0 = blk_base[s];
  const int nblk = blk_base[s + 1] - gb0;
  const double t = item_t(it, cand, cand_off);
  const double* bseg = GTAB ? band : band + seg_band_base[s];
  const int* gb_seg = GTAB ? gbase + b0 : nullptr;  // per ordered sample of the segment
  // candidate passes on certified tiles stream only the far chunks that can
  // hold a slice time <= t (thr = +inf or cmin == null: all of them)
  const bool trunc = MODE == 0 && !GTAB && cmin != nullptr;
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
  const Acc kIdent{INF, INF, 0, INT_MAX};

  // state slots: slot(j) = (j + shift) mod R, R = entries (a multiple of 32)
  const int R = it.state_entries;
  const int SE = R + kStatePad;
  const int shift = (32 - (n & 31)) & 31;
  double* st_s = SMEM_STATE ? reinterpret_cast<double*>(smem + DpSmem::state) : gstate + it.state_off;
  double* st_x = st_s + SE;                                                   // X2
  int* st_c = reinterpret_cast<int*>(st_s + (X2 ? 2 : 1) * SE);               // CAND: 1 + count
  auto slot = [&](int j) {
    const int e = j + shift;
    return e >= R ? e % R : e;
  };
  int* nxt = next_buf + it.next_off;
  // tile column base of column c of the block whose first row is i0 (GTAB):
  // row r's entry is G[colbase - r]
  auto gcol = [&](int i0, int c) -> int { return c == 0 ? 31 : __ldg(gb_seg + i0 + c - 1) + c; };

  // ---- prologue
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init(&unit_full[k], 1);  // (band path; the slice-table path hands units over by named barriers)
      mbar_init(&unit_empty[k], 1);             // the chain warp releases a unit
    }
    for (int k = 0; k < kRing; ++k) {
      mbar_init(&ring_full[k], 1);
      mbar_init(&ring_empty[k], kWorkers);  // every worker warp releases a chunk
    }
    mbar_fence_init();
    // state[n] = {0.0, 0} (microbatch.cpp:174), and its mirror
    const int e = slot(n);
    for (int q = 0; q < 2; ++q) {
      const int ee = q ? e + R : e;
      if (q && e >= kStatePad) break;
      st_s[ee] = 0.0;
      if (CAND) st_c[ee] = KEYED ? (1 << kKeyShift) | n : 1;
      if (MODE == 1) st_x[ee] = -INF;
      if (MODE == 3) st_x[ee] = 0.0;
    }
    row0[0] = INF;
    row0[1] = CAND ? 0.0 : INF;
    row0[2] = INF;
  }
  if (wid < kWorkers) {  // block 0 has no far-far columns (j <= n < i0 + 64): identity partials
    const int o = wid * kRB + lane;
    wps[o] = INF;
    wpx[o] = INF;
    wpc[o] = 0;
    wpj[o] = INT_MAX;
  }
  // (slice-table path) unit u — the triangle columns of block u and the
  // near-far columns of block u + 1 — into buffer (u + 1) & 1, worker w
  // copying the unit's columns w, w + 8, ... with cp.async (lane = row).
  // Columns [0, 32): triangle column q; [32, 64): near-far column q - 32.
  auto fill_unit = [&](int u) {
    double* U = unit + (size_t)((u + 1) & 1) * kUnitCols * kRB;
    int ct = 0, cn = 0, i0 = 0, i0n = 0, nbn = 0;
    if (u >= 0) {
      const int i1 = n - kRB * u;
      i0 = max(0, i1 - kRB);
      ct = min(i1 - i0, blk_W[gb0 + u]);
    }
    if (u + 1 < nblk) {
      const int i1n = n - kRB * (u + 1);
      i0n = max(0, i1n - kRB);
      nbn = i1n - i0n;
      cn = max(0, min(kRB, blk_W[gb0 + u + 1] - nbn));
    }
    const int q = wid + kWorkers * (lane & 7);  // lane m < 8: the base of column wid + 8m
    const bool ok = q < kRB ? q < ct : q - kRB < cn;
    const int g = ok ? (q < kRB ? gcol(i0, q) : gcol(i0n, nbn + q - kRB)) : 0;
    const unsigned m = __ballot_sync(0xffffffffu, ok && lane < 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int gk = __shfl_sync(0xffffffffu, g, k);
      if (m & (1u << k)) cp_async8(U + (wid + kWorkers * k) * kRB + lane, band + (gk - lane));
    }
  };
  if (GTAB && wid < kWorkers && nblk > 0) {
    fill_unit(-1);
    fill_unit(0);
    cp_async_wait_all();
  }
  __syncthreads();

  // ================= producer warp: the units (and, band path, the far-far
  // ring) in consumption order.  Unit u goes to buffer (u + 1) & 1; unit -1
  // holds only block 0's near-far columns.  It never joins the block barrier.
  if (!GTAB && wid == kProducerWarp) {
    long long ncols_total = 0;  // tile columns visited (transitions / 32)
    auto unit_geom = [&](int u, int& i0, int& nb, int& W) {
      const int i1 = n - kRB * u;
      i0 = max(0, i1 - kRB);
      nb = i1 - i0;
      W = blk_W[gb0 + u];
    };
    auto load_unit = [&](int u) {
      const int k = (u + 1) & 1;
      double* U = unit + (size_t)k * kUnitCols * kRB;
      int ct = 0, cn = 0, i0 = 0, nb = 0, W = 0, i0n = 0, nbn = 0, Wn = 0;
      if (u >= 0) {
        unit_geom(u, i0, nb, W);
        ct = min(nb, W);
      }
      if (u + 1 < nblk) {
        unit_geom(u + 1, i0n, nbn, Wn);
        cn = max(0, min(kRB, Wn - nbn));
      }
      if (lane == 0) {
        mbar_expect_tx(&unit_full[k], (uint32_t)(ct + cn) * kColBytes);
        if (ct > 0) tma_load_1d(U, bseg + tile_off[gb0 + u], ct * kColBytes, &unit_full[k]);
        if (cn > 0)
          tma_load_1d(U + kRB * kRB, bseg + tile_off[gb0 + u + 1] + (size_t)nbn * kRB, cn * kColBytes,
                      &unit_full[k]);
      }
    };
    load_unit(-1);
    if (nblk > 0) load_unit(0);
    int islot = 0, iround = 0;
    for (int b = 0; b < nblk; ++b) {
      const int W = blk_W[gb0 + b];
      ncols_total += min(kNearCols, W);
      if (b + 1 >= nblk) break;
      // unit b+1 into the buffer of unit b-1, once the chain released it
      const int u = b + 1, k = (u + 1) & 1, f = (u + 1) >> 1;
      PP_TRACE(11);
      mbar_wait(&unit_empty[k], (f - 1) & 1);
      PP_TRACE(12);
      load_unit(u);
      PP_TRACE(13);
      // far-far chunks of block b+1 (the workers reduce them during block b)
      const int gn = gb0 + b + 1;
      const int Wn = blk_W[gn];
      const int nc = far_nc(gn, Wn);
      ncols_total += nc > 0 ? min(Wn, kNearCols + nc * kChunkCols) - kNearCols : 0;
      if (lane == 0) {
        for (int q = 0; q < nc; ++q) {
          const int c0 = kNearCols + q * kChunkCols;
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

  // ================= chain warp
  if (wid == (GTAB ? kWorkers : kChainWarp)) {
    const int r = lane;
    Acc N = kIdent;  // this lane's row of the NEXT block: its near-far columns so far
    // block 0's near-far columns (unit -1: j = n, ...), from the stored states
    if (nblk > 0) {
      if (!GTAB) mbar_wait(&unit_full[0], 0);
      const int nb0 = n - max(0, n - kRB);
      const int cnf = max(0, min(kRB, blk_W[gb0] - nb0));
      const double* U = unit;
      for (int k = cnf - 1; k >= 0; --k) {
        const int j = n - kRB * 0 + k;  // i1 of block 0 is n
        const int e = slot(j);
        fold_c<MODE, true>(N, U[(kRB + k) * kRB + r], st_s[e], X2 ? st_x[e] : 0.0, CAND ? cnt_of(st_c[e]) : 1, j,
                           true, t);
      }
      __syncwarp();
      if (!GTAB && lane == 0) mbar_arrive(&unit_empty[0]);
    }
    // (slice-table path) unit -1 read: the workers may refill its buffer
    if (GTAB) named_bar(1, kSyncThreads);
    for (int b = 0; b < nblk; ++b) {
      PP_TRACE(0);
      const int i1 = n - kRB * b;
      const int i0 = max(0, i1 - kRB);
      const int nb = i1 - i0;
      const int W = blk_W[gb0 + b];
      const bool has_next = b + 1 < nblk;
      const int i0n = max(0, i0 - kRB);
      const int nbn = i0 - i0n;
      const int cnx = has_next ? max(0, min(kRB, blk_W[gb0 + b + 1] - nbn)) : 0;  // valid next near-far cols
      const int ub = (b + 1) & 1;
      const double* U = unit + (size_t)ub * kUnitCols * kRB;
      // this row's accumulator: the near-far columns (folded during the
      // previous block) and the workers' far-far partial
      Acc A = N;
      {  // the worker partials of this block's far-far columns (four: workers
         // 0-3 folded in 4-7's), a pairwise tree
        constexpr int kParts = kWorkers / 4;
        Acc v[kParts];
#pragma unroll
        for (int q = 0; q < kParts; ++q) {
          const int p = ((b & 1) * kWorkers + q) * kRB + r;
          v[q].s = wps[p];
          v[q].x = X2 ? wpx[p] : INF;
          v[q].c = CAND ? wpc[p] : 0;
          v[q].j = CAND && !KEYED ? wpj[p] : INT_MAX;
        }
#pragma unroll
        for (int h = kParts / 2; h >= 1; h /= 2)
#pragma unroll
          for (int q = 0; q < h; ++q) {
            if (KEYED) combine_k<MODE>(v[q], v[q + h]);
            else combine<MODE>(v[q], v[q + h]);
          }
        if (KEYED) {  // key -> (count, argmin)
          v[0].j = v[0].c & ((1 << kKeyShift) - 1);
          v[0].c >>= kKeyShift;
        }
        combine<MODE>(A, v[0]);
      }
      // the last block of a segment whose n is not a multiple of 32 has
      // near-far columns past the previous block's rows: fold them from the
      // tile in global memory and the stored states (once per pass)
      if (nb < kRB && b > 0) {
        const int chi = min(kNearCols, W);
        for (int c = chi - 1; c >= nb + kRB; --c) {
          const int j = i0 + c;
          const double xv = GTAB ? __ldg(band + gcol(i0, c) - r) : __ldg(bseg + tile_off[gb0 + b] + (size_t)c * kRB + r);
          const int e = slot(j);
          fold_c<MODE, true>(A, xv, st_s[e], X2 ? st_x[e] : 0.0, CAND ? cnt_of(st_c[e]) : 1, j, true, t);
        }
      }
      if (r >= nb) A = kIdent;
      N = kIdent;
      if (!GTAB) mbar_wait(&unit_full[ub], ((b + 1) >> 1) & 1);
      PP_TRACE(1);
      PP_TRACE(2);
      // ---- the triangle.  Iteration k: every lane l <= k folds the slice
      // (l, k+1) with state[k+1] (lane k's row is then complete: state[k]),
      // lane k's accumulator is shuffled to every lane, and every lane folds
      // state[k] into its row of the NEXT block (near-far column k).  The
      // serial path per row is one fold and one shuffle round trip
      // (tools/chain_probe.cu: ~64 cycles per row alone on an SM, against
      // ~110 for recomputing each state redundantly from accumulators
      // shuffled two rows ahead).
      auto triangle = [&](auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        double Ss = 0.0, Sx = 0.0;  // state[k+1] (every lane)
        int Sc = 0;
        auto lda = [&](int k) { return (FULL ? (k + 1 < kRB) : (k + 1 < nb)) ? lds_f64(U + (k + 1) * kRB + r) : 0.0; };
        auto ldn = [&](int k) { return lds_f64(U + (kRB + k) * kRB + r); };
        const int kst = FULL ? kRB - 1 : nb - 1;  // the first step
        double xan = lda(kst), xnn = ldn(kst);
#pragma unroll
        for (int k = kRB - 1; k >= 0; --k) {
          if (FULL || k < nb) {
            const double xa = xan, xn = xnn;
            if (k > 0) {  // the next step's entries, one step ahead
              xan = lda(k - 1);
              xnn = ldn(k - 1);
            }
            if (FULL ? (k + 1 < kRB) : (k + 1 < nb))
              fold<MODE, true>(A, xa, Ss, Sx, Sc, i0 + k + 1, (r <= k) & (k + 1 < W), t);
            double ns = shfl_f64(A.s, k);
            double nx = X2 ? shfl_f64(A.x, k) : INF;
            const int nc = CAND ? shfl_i32(A.c, k) : 0;
            if (SANITIZE) {
              ns = isfinite(ns) ? ns : INF;
              if (MODE == 3) nx = isfinite(nx) ? nx : INF;
            }
            // (k < cnx is false without a next block; ldn then reads the idle buffer half)
            fold<MODE, true>(N, xn, ns, nx, nc, i0 + k, k < cnx, t);
            Ss = ns;
            Sx = nx;
            Sc = nc;
          }
        }
      };
      if (nb == kRB) triangle(std::true_type{}); else triangle(std::false_type{});
      // unit b consumed: the warp's reads are ordered before the release
      // (__syncwarp + mbarrier arrive), and the producer's next write into the
      // buffer waits for it
      __syncwarp();
      if (!GTAB && lane == 0) mbar_arrive(&unit_empty[ub]);
      PP_TRACE(3);
      if (r < nb) {
        const int row = i0 + r;
        const bool f = isfinite(A.s);
        const int e = slot(row);
        const double sv = (SANITIZE && !f) ? INF : A.s;
        const double xv = (SANITIZE && MODE == 3 && !isfinite(A.x)) ? INF : A.x;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q && e >= kStatePad) break;
          const int ee = q ? e + R : e;  // the mirror
          st_s[ee] = sv;
          if (X2) st_x[ee] = xv;
          if (CAND) st_c[ee] = KEYED ? ((f ? A.c + 1 : 1) << kKeyShift) | row : (f ? A.c + 1 : 1);
        }
        if (CAND) nxt[row] = f ? A.j : -1;
        if (row == 0) {
          row0[0] = A.s;
          row0[1] = CAND ? (double)A.c : A.x;
          row0[2] = A.x;
        }
      }
      PP_TRACE(4);
      __syncwarp();  // (reconverge: lanes >= nb skipped the stores)
      named_bar(1, kSyncThreads);  // chain + workers: block b's states and block b+1's partial
      PP_TRACE(5);
    }
  } else {
    // ================= workers: far-far columns of block b+1 during block b
    const int w = wid;
    int cslot = 0;
    uint32_t cphase = 0;
    if (GTAB) named_bar(1, kSyncThreads);  // (the chain has read unit -1)
    for (int b = 0; b < nblk; ++b) {
      const int bn = b + 1;
      if (w == 0) PP_TRACE(8);
      // the chain's unit for block b + 1 (its buffer held unit b - 1, read
      // before the last block barrier); complete at the next one
      if (GTAB && bn < nblk) fill_unit(bn);
      if (bn < nblk) {
        const int j1 = n - kRB * bn;
        const int k0 = max(0, j1 - kRB);  // i0 of block b+1
        const int Wn = blk_W[gb0 + bn];
#ifdef PP_DP_TRACE
        const int nc = (g_dp_flags & 1) ? 0 : (GTAB ? n_chunks(Wn) : far_nc(gb0 + bn, Wn));
#else
        const int nc = GTAB ? n_chunks(Wn) : far_nc(gb0 + bn, Wn);
#endif
        Acc a0 = kIdent, a1 = kIdent;
        // a multiple of 32 (k0 + 64 == n mod 32) except on the last block of a
        // segment whose n is not a multiple of 32: then scalar state loads
        const int sb0 = slot(k0 + kNearCols);
        const int q0 = 4 * w;
        // one chunk step: the four columns' states (sb = the chunk's first
        // slot) and entries x folded into the two accumulators (even / odd
        // column, ascending j in each).  VEC: 16-byte state loads (sb + q0 is
        // a multiple of 4; the mirror covers sb + 31 >= R).  The stored count
        // is already 1 + count (fold_c).
        auto reduce4 = [&](auto vec_tag, int sb, int j, const double* x) {
          constexpr bool VEC = decltype(vec_tag)::value;
          double2 s01, s23, x01{0.0, 0.0}, x23{0.0, 0.0};
          int4 cc{1, 1, 1, 1};
          const int e = sb + q0;
          if (VEC) {
            s01 = *reinterpret_cast<const double2*>(st_s + e);
            s23 = *reinterpret_cast<const double2*>(st_s + e + 2);
            if (X2) {
              x01 = *reinterpret_cast<const double2*>(st_x + e);
              x23 = *reinterpret_cast<const double2*>(st_x + e + 2);
            }
            if (CAND) cc = *reinterpret_cast<const int4*>(st_c + e);
          } else {
            s01 = double2{st_s[e], st_s[e + 1]};
            s23 = double2{st_s[e + 2], st_s[e + 3]};
            if (X2) {
              x01 = double2{st_x[e], st_x[e + 1]};
              x23 = double2{st_x[e + 2], st_x[e + 3]};
            }
            if (CAND) cc = int4{st_c[e], st_c[e + 1], st_c[e + 2], st_c[e + 3]};
          }
          fold_c<MODE, false>(a0, x[0], s01.x, x01.x, cc.x, j, true, t);
          fold_c<MODE, false>(a1, x[1], s01.y, x01.y, cc.y, j + 1, true, t);
          fold_c<MODE, false>(a0, x[2], s23.x, x23.x, cc.z, j + 2, true, t);
          fold_c<MODE, false>(a1, x[3], s23.y, x23.y, cc.w, j + 3, true, t);
        };
        auto next_sb = [&](int sb) {
          sb += kChunkCols;
          return sb >= R ? sb - R : sb;
        };
        if (GTAB) {
          // lane q holds the table base of column 64 + 32k + q of chunk k (one
          // coalesced int32 load per chunk; 31 = the NaN row past the tile),
          // a worker takes its four columns' bases by shuffles.  Entries run
          // one chunk ahead of their use.  The state ring wraps at most once
          // in a block's far-far range (R >= W + 64): chunks [0, kw) read
          // slots sb0 + 32k, the rest 32k - (R - sb0), so the loop walks
          // plain pointers and steps them back by R once, between two runs.
          const int* gp = gb_seg + k0 - 1 + kNearCols + lane;  // column 64 + lane of chunk 0
          int cw = kNearCols + lane;                             // this lane's column
          auto colb = [&]() -> int {
            const int v = cw < Wn ? __ldg(gp) + cw : 31;
            gp += kChunkCols;
            cw += kChunkCols;
            return v;
          };
          auto load_x = [&](int lb, double* x) {  // row `lane` of a column: band[base - lane]
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = __ldg(band + (shfl_i32(lb, q0 + i) - lane));
          };
          auto loop = [&](auto vec_tag) {
            constexpr bool VEC = decltype(vec_tag)::value;
            double xa[4], xb[4];
            int j = k0 + kNearCols + q0;
            const double* ps = st_s + sb0 + q0;
            const double* px = st_x + sb0 + q0;
            const int* pc = st_c + sb0 + q0;
            auto step = [&](const double* x) {  // one chunk: this worker's four columns
              double2 s01, s23, x01{0.0, 0.0}, x23{0.0, 0.0};
              int4 cc{1, 1, 1, 1};
              if (VEC) {
                s01 = *reinterpret_cast<const double2*>(ps);
                s23 = *reinterpret_cast<const double2*>(ps + 2);
                if (X2) {
                  x01 = *reinterpret_cast<const double2*>(px);
                  x23 = *reinterpret_cast<const double2*>(px + 2);
                }
                if (CAND) cc = *reinterpret_cast<const int4*>(pc);
              } else {
                s01 = double2{ps[0], ps[1]};
                s23 = double2{ps[2], ps[3]};
                if (X2) {
                  x01 = double2{px[0], px[1]};
                  x23 = double2{px[2], px[3]};
                }
                if (CAND) cc = int4{pc[0], pc[1], pc[2], pc[3]};
              }
              if (KEYED) {
                fold_k<MODE>(a0, x[0], s01.x, x01.x, cc.x, t);
                fold_k<MODE>(a1, x[1], s01.y, x01.y, cc.y, t);
                fold_k<MODE>(a0, x[2], s23.x, x23.x, cc.z, t);
                fold_k<MODE>(a1, x[3], s23.y, x23.y, cc.w, t);
              } else {
                fold_c<MODE, false>(a0, x[0], s01.x, x01.x, cc.x, j, true, t);
                fold_c<MODE, false>(a1, x[1], s01.y, x01.y, cc.y, j + 1, true, t);
                fold_c<MODE, false>(a0, x[2], s23.x, x23.x, cc.z, j + 2, true, t);
                fold_c<MODE, false>(a1, x[3], s23.y, x23.y, cc.w, j + 3, true, t);
              }
              ps += kChunkCols;
              px += kChunkCols;
              pc += kChunkCols;
              j += kChunkCols;
            };
            load_x(colb(), xa);
            int k = 0;
            // chunks [k, kend) with no ring wrap; entries of chunk k in xa on entry and exit
            auto run = [&](int kend) {
              for (; k + 2 <= kend; k += 2) {
                load_x(colb(), xb);
                step(xa);
                load_x(colb(), xa);
                step(xb);
              }
              if (k < kend) {
                load_x(colb(), xb);
                step(xa);
#pragma unroll
                for (int i = 0; i < 4; ++i) xa[i] = xb[i];
                ++k;
              }
            };
            const int kw = min(nc, (R - sb0 + kChunkCols - 1) / kChunkCols);
            run(kw);
            ps -= R;
            px -= R;
            pc -= R;
            run(nc);
          };
          if ((sb0 & 3) == 0) loop(std::true_type{}); else loop(std::false_type{});
        } else {
          int sb = sb0;
          for (int k = 0; k < nc; ++k) {
            const int c0 = kNearCols + k * kChunkCols;
            double x[4];
            mbar_wait(&ring_full[cslot], cphase);
            const double* ch = ring + (size_t)cslot * kChunkCols * kRB;
            const int cols = min(kChunkCols, Wn - c0);
#pragma unroll
            for (int i = 0; i < 4; ++i) x[i] = (q0 + i < cols) ? ch[(q0 + i) * kRB + lane] : QNAN;
            if ((sb0 & 3) == 0) reduce4(std::true_type{}, sb, k0 + c0 + q0, x);
            else reduce4(std::false_type{}, sb, k0 + c0 + q0, x);
            __syncwarp();  // the warp's reads of the slot, then its release
            if (lane == 0) mbar_arrive(&ring_empty[cslot]);
            if (++cslot == kRing) {
              cslot = 0;
              cphase ^= 1u;
            }
            sb = next_sb(sb);
          }
        }
        if (KEYED) combine_k<MODE>(a0, a1);
        else combine<MODE>(a0, a1);
        if (w == 0) PP_TRACE(9);
        // this worker's partial of block b+1, for the chain to fold when it
        // starts that block (slot parity bn: the chain is reading block b's).
        // Workers w + 4 hand theirs to worker w (a named barrier per pair),
        // which folds it in: the chain folds four partials, not eight.
        const int half = kWorkers / 2;
        auto put = [&](int slot, const Acc& a) {
          const int o = ((bn & 1) * kWorkers + slot) * kRB + lane;
          wps[o] = a.s;
          if (X2) wpx[o] = a.x;
          if (CAND) wpc[o] = a.c;
          if (CAND && !KEYED) wpj[o] = a.j;
        };
        if (w >= half) {
          put(w, a0);
          __syncwarp();
          named_bar_arrive(kBarPair + (w - half), 64);
        } else {
          named_bar(kBarPair + w, 64);
          auto take = [&](int from) {
            const int o = ((bn & 1) * kWorkers + from) * kRB + lane;
            Acc p{wps[o], X2 ? wpx[o] : INF, CAND ? wpc[o] : 0, CAND && !KEYED ? wpj[o] : INT_MAX};
            if (KEYED) combine_k<MODE>(a0, p);
            else combine<MODE>(a0, p);
          };
          take(w + half);
          // a second level: workers 2-3 hand theirs to 0-1, the chain folds two
          if (w >= 2) {
            put(w, a0);
            __syncwarp();
            named_bar_arrive(kBarPair2 + (w - 2), 64);
          } else {
            named_bar(kBarPair2 + w, 64);
            take(w + 2);
            put(w, a0);
          }
        }
        if (w == 0) PP_TRACE(10);
      }
      if (GTAB) cp_async_wait_all();
      __syncwarp();
      named_bar(1, kSyncThreads);  // chain + workers: block b's states and block b+1's partial
    }
  }
  if (threadIdx.x == 0) {  // (worker 0) after the last block barrier: row0 is final
    ItemResult rr;
    rr.sum0 = row0[0];
    rr.count0 = CAND ? (int)row0[1] : 0;
    rr.feasible = isfinite(row0[0]) ? 1 : 0;
    rr.aux = MODE == 1 ? row0[1] : -INF;  // (MODE 2: no t*)
    res[res_by_seg ? s : blockIdx.x] = rr;
    if (MODE == 3) {  // the fused bound pass's result, by segment
      ItemResult rb;
      rb.sum0 = row0[2];
      rb.count0 = 0;
      rb.feasible = isfinite(row0[2]) ? 1 : 0;
      rb.aux = -INF;
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
extern "C" int pp_debug_dp_flags(int flags) {
  return cudaMemcpyToSymbol(g_dp_flags, &flags, sizeof(flags)) == cudaSuccess ? 0 : 4;
}
#endif
// smem_state = the largest shared-memory DP state of the launch's items
// (0 with state_global: every item's state then lives in gstate).  Band path:
// the chunk ring gets the rest of `smem_budget` (4..kMaxRing chunks of 8 KB);
// slice-table path (gbase != null): no ring, the workers read G directly.
cudaError_t launch_dp_pass(int mode, const WorkItem* items, int n_items, size_t smem_state,
                           int state_global, int sanitize, size_t smem_budget, const int64_t* seg_off,
                           const int* blk_base, const int* blk_W, const int64_t* tile_off,
                           const int64_t* seg_band_base, const double* band, const double* cand,
                           const int64_t* cand_off, ItemResult* res, int* next_buf, double* gstate,
                           int res_by_seg, const double* cmin, double t_margin,
                           unsigned long long* cols_streamed, ItemResult* res2, const int* gbase,
                           cudaStream_t st) {
  if (n_items == 0) return cudaSuccess;
  const size_t ring_off = (DpSmem::state + (state_global ? 0 : smem_state) + 127) / 128 * 128;
  int ring = 0;
  size_t smem = ring_off;
  if (!gbase) {
    ring = (int)std::min<size_t>(kMaxRing, (smem_budget - std::min(smem_budget, ring_off)) / kChunkBytes);
    ring = std::max(ring, 4);
    smem = ring_off + (size_t)ring * kChunkBytes;
  }
#define PP_DP_LAUNCH(M, S, Z, G)                                                                      \
  do {                                                                                                \
    ensure_dyn_smem((const void*)dp_pass_kernel<M, S, Z, G>, smem);                                   \
    dp_pass_kernel<M, S, Z, G><<<n_items, dp_threads<G>(), smem, st>>>(                              \
        items, seg_off, blk_base, blk_W, tile_off, seg_band_base, band, cand, cand_off, res, next_buf, \
        gstate, res_by_seg, (int)ring_off, ring, cmin, t_margin, cols_streamed, res2, gbase);         \
  } while (0)
#define PP_DP_LAUNCH_Z(M, S)                          \
  do {                                                \
    if (gbase) PP_DP_LAUNCH(M, S, false, true);       \
    else if (sanitize) PP_DP_LAUNCH(M, S, true, false); \
    else PP_DP_LAUNCH(M, S, false, false);            \
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
