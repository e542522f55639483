// msp_common.cuh -- shared device types and helpers for the B200 market-split solver.
//
// Data layout in HBM:
//   quarter table t in {A,B,C,D}: sorted row-0 weights (u64), subset masks (u32) and the
//   companion rows 1..m-1 packed two u16 per u32 word ("P16"), SW words per entry (AoS, 16 B at
//   m <= 9) so one LDG.128 brings a whole companion vector.
//   Dense per-weight run arrays (start, end) index every equal-weight run of a table.
// The enumeration space of one alpha-batch is a union of rectangles X-run(alpha - w) x Y-run(w)
// (SURVEY.md §0 restatement); a warp tile covers 32 entries of the longer run x TQ of the other.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace msp {

constexpr int kTQ = 32;            // loop entries per warp tile
constexpr int kMaxMC = 15;         // companion coordinates supported by P16 (m <= 16); P32: m <= 9
constexpr uint64_t kFnvOffset = 0xCBF29CE484222325ull;  // validate.py:34, fastval.py:42
constexpr uint64_t kFnvPrime = 0x100000001B3ull;         // validate.py:35, fastval.py:43
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kHitFlag = 1ull << 63;

// Host-side FNV fold step (validate.py:40-42) -- also used for the per-batch constant h0.
__host__ __device__ inline uint64_t fnv_step64(uint64_t h, uint64_t v) { return (h ^ v) * kFnvPrime; }

// One FNV-1a-style fold step on a 64-bit state held as two u32 halves, for a coordinate value
// v < 2^32:  (h ^ v) * (2^40 + 435)  mod 2^64.  Four integer ops: LOP3, IMAD.WIDE.U32, IMAD, LEA.
__device__ __forceinline__ void fnv_step(uint32_t &lo, uint32_t &hi, uint32_t v) {
  const uint32_t x = lo ^ v;
  const uint64_t p = (uint64_t)x * 435u;
  hi = hi * 435u + (uint32_t)(p >> 32) + (x << 8);
  lo = (uint32_t)p;
}

struct TableDev {
  const uint64_t *w;         // row-0 weights in table order
  const uint32_t *mask;      // subset masks (bit t <-> column start+t)
  const uint32_t *comp;      // packed companions, sw words per entry
  const uint32_t *run_start; // dense over [0, S]
  const uint32_t *run_end;   // dense over [0, S]; run empty iff end == start
  uint32_t S;                // largest row-0 weight (block row-0 sum)
  uint32_t size;
};

struct YRuns {               // distinct weights of a Y table (B for left, D for right)
  const uint32_t *w;
  const uint32_t *start;
  const uint32_t *len;
  uint32_t n;
};

// One (batch, side[, pass]) unit of a launch.
struct UnitDesc {
  uint64_t tile_base;        // first launch tile of the unit
  uint64_t h0;               // FNV state after coordinate 0 (= alpha on both sides)
  uint32_t xw_total;         // alpha (left) / beta (right): X weight = xw_total - Y weight
  uint32_t side;             // 0 left (A x B), 1 right (C x D)
  uint32_t rect_base;        // first rectangle of this (batch, side) in the rectangle list
  uint32_t gid;              // batch index within the solve
  uint32_t slot;             // wave-local batch slot (global-table zero-key counts)
  uint32_t region_base;      // global table / hit-set region base, or wave bucket base
  uint32_t region_log2;      // log2 capacity of the region, or bucket bits of the batch
  uint32_t pass, npass;      // hash-range pass filter (npass == 1: all keys)
  uint32_t count_filter;     // count overshooting right pairs in this unit
  uint32_t flags;            // bit0: hit set contains key 0; bit1: probe role (partitioned join)
  uint32_t nrect;            // rectangles of this (batch, side)
};

// One nonempty rectangle X-run(w_x) x Y-run(w_y) of a batch side, oriented for the warp tile:
// the longer run goes across lanes.  tile_off = warp tiles before it within its (batch, side).
struct RectDesc {
  uint32_t lane_start, loop_start, L, Q;
  uint32_t tile_off;
  uint32_t gs_x;             // (2 * batch + side) << 1 | lane_is_x
  uint32_t nl, nq;
  __device__ __forceinline__ bool lane_is_x() const { return gs_x & 1u; }
  __device__ __forceinline__ uint32_t gs() const { return gs_x >> 1; }
};

struct EnumArgs {
  TableDev tab[4];
  YRuns yr[2];               // [0] = B runs, [1] = D runs
  const RectDesc *rects;     // rectangle lists of all (batch, side)
  const UnitDesc *units;
  uint32_t nunits;
  uint64_t total_tiles;
  uint64_t chunk_tiles;      // tiles per warp work item
  uint64_t nchunks;
  uint32_t dpack[8];         // d rows 1..m-1 packed, +0x8000 guard per half (right side)
  uint32_t diag;             // MSP_FLAG_DIAG_HASH_ONLY: hash without staging (timing only)
  uint64_t key_mask;         // keys & key_mask (~0; MSP_FLAG_DEGENERATE_HASH: 0, every pair collides)
  unsigned long long *batch_filtered; // per batch (gid)
  unsigned long long *batch_hits;     // per batch (gid)
};

__device__ __forceinline__ uint32_t pass_of(uint64_t key, uint32_t npass) {
  return (uint32_t)(((key >> 32) * (uint64_t)npass) >> 32);
}

__device__ __forceinline__ uint32_t home_slot(uint64_t key, uint32_t log2cap) {
  return (uint32_t)((key * kGolden) >> (64 - log2cap));
}

template <int SW>
__device__ __forceinline__ void load_vec(const uint32_t *__restrict__ base, uint32_t idx, uint32_t (&v)[SW]) {
  const uint32_t *p = base + (size_t)idx * SW;
  if constexpr (SW == 1) {
    v[0] = __ldg(p);
  } else if constexpr (SW == 2) {
    const uint2 t = __ldg(reinterpret_cast<const uint2 *>(p));
    v[0] = t.x; v[1] = t.y;
  } else {
#pragma unroll
    for (int k = 0; k < SW; k += 4) {
      const uint4 t = __ldg(reinterpret_cast<const uint4 *>(p + k));
      v[k] = t.x; v[k + 1] = t.y; v[k + 2] = t.z; v[k + 3] = t.w;
    }
  }
}

// Companion layouts, selected by the kernels' compile-time MCX = MC (+ kWide):
//   P16 (MCX = MC <= 15): two companion coordinates per u32 word, 16 bits each; exact while every
//        block row sum is <= 16384 and d_j <= 32767 (right residual d - s kept with a guard bit
//        per half: (d + 0x8000) - s keeps bit 15 iff s <= d);
//   P32 (MCX = MC + kWide, MC <= 8): one coordinate per word, 31-bit values; exact while every
//        block row sum is < 2^30 and d_j < 2^31 (guard bit 31).
constexpr int kWide = 16;
constexpr int kMaxWideMC = 8;
__host__ __device__ constexpr int mc_of(int mcx) { return mcx & (kWide - 1); }
__host__ __device__ constexpr bool wide_of(int mcx) { return mcx >= kWide; }
__host__ __device__ constexpr int words_for(int mcx) { return wide_of(mcx) ? mc_of(mcx) : (mc_of(mcx) + 1) / 2; }
__host__ __device__ constexpr int stride_for(int mcx) {
  return words_for(mcx) <= 1 ? 1 : words_for(mcx) <= 2 ? 2 : words_for(mcx) <= 4 ? 4 : 8;
}
__host__ __device__ constexpr uint32_t guard_mask(int mcx) { return wide_of(mcx) ? 0x80000000u : 0x80008000u; }
// Coordinate c (< MC) of a companion word vector: left (a plain sum) or right (the guarded residual).
template <int MCX, bool RIGHT>
__host__ __device__ __forceinline__ uint32_t coord(const uint32_t *w, int c) {
  if constexpr (wide_of(MCX)) return RIGHT ? (w[c] & 0x7FFFFFFFu) : w[c];
  else return ((c & 1) ? (w[c >> 1] >> 16) : w[c >> 1]) & (RIGHT ? 0x7FFFu : 0xFFFFu);
}

// Lane-step slots a warp-tile orientation spends on an L x Q rectangle (L across 32-lane tiles, Q
// looped in steps of 4 keys within tiles of kTQ); the rectangle lists orient each rectangle the
// cheaper way (longer-run-across-lanes alone leaves ~3% more slots idle at (7,60)).
__host__ __device__ inline uint64_t tile_slots(uint32_t L, uint32_t Q) {
  return (uint64_t)((L + 31) / 32) * 32 * ((Q / 32) * 32 + (((Q % 32) + 3) / 4) * 4);
}
__host__ __device__ inline bool lanes_over_x(uint32_t xl, uint32_t yl) { return tile_slots(xl, yl) <= tile_slots(yl, xl); }

// The warp-tile pieces of one rectangle X[xs, xs + xl) x Y[ys, ys + yl) of batch side gs: oriented
// the cheaper way; when the lane run is not a multiple of 32, its full 32-lane tiles form one piece
// and the remainder (r < 32 lane entries x the loop run) a second piece, itself oriented the cheaper
// way (usually lanes over the loop run): (7,60) lane use 84% -> 88% (tools/tile_sim.py).
// Returns the piece count (0..2); pieces get every RectDesc field but tile_off.
#ifndef MSP_SPLIT_REMAINDER
#define MSP_SPLIT_REMAINDER 1
#endif
__host__ __device__ inline RectDesc rect_piece(uint32_t gs, bool lx, uint32_t xs, uint32_t xl, uint32_t ys, uint32_t yl) {
  RectDesc R;
  R.gs_x = (gs << 1) | (lx ? 1u : 0u);
  R.lane_start = lx ? xs : ys;
  R.loop_start = lx ? ys : xs;
  R.L = lx ? xl : yl;
  R.Q = lx ? yl : xl;
  R.tile_off = 0;
  R.nl = (R.L + 31) / 32;
  R.nq = (R.Q + kTQ - 1) / kTQ;
  return R;
}
__host__ __device__ inline uint32_t rect_pieces(uint32_t gs, uint32_t xs, uint32_t xl, uint32_t ys, uint32_t yl,
                                                RectDesc (&out)[2]) {
  if (!xl || !yl) return 0;
  const bool lx = lanes_over_x(xl, yl);
  const uint32_t A = lx ? xl : yl, full = A & ~31u, r = A - full;
  if (!MSP_SPLIT_REMAINDER || full == 0 || r == 0) {
    out[0] = rect_piece(gs, lx, xs, xl, ys, yl);
    return 1;
  }
  if (lx) {  // X across lanes: X[xs, xs + full) x Y, then X[xs + full, xs + xl) x Y
    out[0] = rect_piece(gs, true, xs, full, ys, yl);
    out[1] = rect_piece(gs, lanes_over_x(r, yl), xs + full, r, ys, yl);
  } else {   // Y across lanes: X x Y[ys, ys + full), then X x Y[ys + full, ys + yl)
    out[0] = rect_piece(gs, false, xs, xl, ys, full);
    out[1] = rect_piece(gs, lanes_over_x(xl, r), xs, xl, ys + full, r);
  }
  return 2;
}

struct HitRec { uint32_t gid, pad; uint64_t key; };
struct PairRec { uint32_t gid, side, xidx, yidx, xmask, ymask; uint64_t key; };

}  // namespace msp
