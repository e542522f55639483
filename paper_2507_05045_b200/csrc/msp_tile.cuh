// msp_tile.cuh -- warp tile walker shared by the enumeration kernels.
//
// A batch side is a union of rectangles X-run(alpha - w) x Y-run(w) (SURVEY.md §0 restatement of
// the heap stream, fastenum.py:87-147).  A warp tile covers 32 entries of the rectangle's longer run
// (one per lane, companion vector held in registers) x up to kTQ entries of the shorter run (loaded
// warp-uniformly, i.e. broadcast).  Tiles of a launch are numbered contiguously across its units;
// a warp walks a contiguous range of them through the compacted rectangle lists built by k_rects.
#pragma once
#include "msp_common.cuh"

namespace msp {

__device__ __forceinline__ uint32_t find_unit(const UnitDesc *u, uint32_t n, uint64_t T) {
  uint32_t lo = 0, hi = n;  // last u with tile_base <= T
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (u[mid].tile_base <= T) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t find_rect(const RectDesc *r, uint32_t n, uint32_t t) {
  uint32_t lo = 0, hi = n;  // last rectangle with tile_off <= t
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(&r[mid].tile_off) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ RectDesc load_rect(const RectDesc *p) {
  const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p));
  const uint4 b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
  return RectDesc{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}

// Walks tiles [T, Tend) of a launch for one warp: rectangle after rectangle of the compacted
// rectangle lists, one 32-byte descriptor load per rectangle.
struct TileWalker {
  uint64_t T, Tend;
  uint32_t u, ri, lc, qc;
  UnitDesc d;
  RectDesc R;

  __device__ __forceinline__ void init(const EnumArgs &A, uint64_t t0, uint64_t t1) {
    T = t0;
    Tend = t1;
    if (T >= Tend) return;
    u = find_unit(A.units, A.nunits, T);
    d = A.units[u];
    const uint32_t tl = (uint32_t)(T - d.tile_base);
    ri = find_rect(A.rects + d.rect_base, d.nrect, tl);
    R = load_rect(A.rects + d.rect_base + ri);
    const uint32_t local = tl - R.tile_off;
    lc = local / R.nq;
    qc = local - lc * R.nq;
  }

  __device__ __forceinline__ bool valid() const { return T < Tend; }

  // Advance to the next tile; returns true when the unit changed (caller flushes counters first).
  __device__ __forceinline__ bool advance(const EnumArgs &A, uint32_t &old_unit) {
    old_unit = u;
    if (++T >= Tend) return false;
    if (++qc < R.nq) return false;
    qc = 0;
    if (++lc < R.nl) return false;
    lc = 0;
    bool changed = false;
    if (++ri >= d.nrect) {
      while (u + 1 < A.nunits && T >= A.units[u + 1].tile_base) ++u;
      d = A.units[u];
      ri = 0;
      changed = true;
    }
    R = load_rect(A.rects + d.rect_base + ri);
    return changed;
  }

  // (constant indices only: a runtime index into the parameter struct would copy it to local memory)
  __device__ __forceinline__ const uint32_t *x_comp(const EnumArgs &A) const {
    return d.side ? A.tab[2].comp : A.tab[0].comp;
  }
  __device__ __forceinline__ const uint32_t *y_comp(const EnumArgs &A) const {
    return d.side ? A.tab[3].comp : A.tab[1].comp;
  }
  __device__ __forceinline__ const uint32_t *lane_comp(const EnumArgs &A) const {
    return R.lane_is_x() ? x_comp(A) : y_comp(A);
  }
  __device__ __forceinline__ const uint32_t *loop_comp(const EnumArgs &A) const {
    return R.lane_is_x() ? y_comp(A) : x_comp(A);
  }
};

// Resumable per-lane state of the walker's current tile: the lane's companion vector, the tile's
// loop vectors (staged once per tile in the warp's shared-memory slot `ybuf`, one coalesced load)
// and the next loop entry.  step_keys() produces up to kU keys per call (warp-uniform), so a
// consumer can stop mid-tile (e.g. when its staging buffer is full) and resume later.
constexpr int kU = 4;
template <int SW>
struct TileCursor {
  uint32_t lv[SW];
  uint32_t q, q0, q1, lidx;
  bool lok;
  uint32_t *ybuf;  // kTQ * SW words of shared memory owned by this warp
};

template <int MC, class Walker>
__device__ __forceinline__ void begin_tile(const EnumArgs &A, const Walker &W, uint32_t lane,
                                           TileCursor<stride_for(MC)> &C) {
  constexpr int SW = stride_for(MC);
  const RectDesc &R = W.R;
  const uint32_t loff = W.lc * 32 + lane;
  C.lok = loff < R.L;
  C.lidx = R.lane_start + (C.lok ? loff : 0);
  load_vec<SW>(W.lane_comp(A), C.lidx, C.lv);
  C.q0 = C.q = W.qc * kTQ;
  C.q1 = min(R.Q, C.q + kTQ);
  __syncwarp();
  if (lane < C.q1 - C.q0) {
    uint32_t yv[SW];
    load_vec<SW>(W.loop_comp(A), R.loop_start + C.q0 + lane, yv);
#pragma unroll
    for (int k = 0; k < SW; ++k) C.ybuf[lane * SW + k] = yv[k];
  }
  __syncwarp();
}

template <int SW>
__device__ __forceinline__ void lds_vec(const uint32_t *p, uint32_t (&v)[SW]) {
  if constexpr (SW == 1) {
    v[0] = p[0];
  } else if constexpr (SW == 2) {
    const uint2 t = *reinterpret_cast<const uint2 *>(p);
    v[0] = t.x; v[1] = t.y;
  } else {
#pragma unroll
    for (int k = 0; k < SW; k += 4) {
      const uint4 t = *reinterpret_cast<const uint4 *>(p + k);
      v[k] = t.x; v[k + 1] = t.y; v[k + 2] = t.z; v[k + 3] = t.w;
    }
  }
}

// Keys of loop entries [C.q, min(C.q + kU, C.q1)): fn(u, key, ok, lidx, qidx) for each of them, in
// order.  ok is false for lanes past the run end and for right pairs that overshoot d (counted into
// `filt` when the unit counts filters).  The kU entries are folded together so each thread carries
// kU independent FNV chains (the fold itself is a serial dependency chain).
template <int MC, class Walker, class Fn>
__device__ __forceinline__ void step_keys(const Walker &W, TileCursor<stride_for(MC)> &C,
                                          const uint32_t (&dg)[words_for(MC) > 0 ? words_for(MC) : 1],
                                          unsigned long long &filt, uint64_t kmask, Fn &&fn) {
  constexpr int NW0 = words_for(MC);           // companion words (0 when m == 1)
  constexpr int NW = NW0 > 0 ? NW0 : 1;        // array extent
  constexpr int SW = stride_for(MC);
  constexpr int U = kU;
  const uint32_t q = C.q;
  const uint32_t h0lo = (uint32_t)W.d.h0, h0hi = (uint32_t)(W.d.h0 >> 32);
  const bool right = W.d.side != 0, cf = W.d.count_filter != 0;
  uint32_t sv[U][NW];
  bool ok[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool in = q + u < C.q1;
    uint32_t yv[SW];
    lds_vec<SW>(C.ybuf + (in ? q + u - C.q0 : 0) * SW, yv);
#pragma unroll
    for (int k = 0; k < NW; ++k) sv[u][k] = C.lv[k] + yv[k];
    ok[u] = C.lok && in;
  }
  uint32_t lo[U], hi[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { lo[u] = h0lo; hi[u] = h0hi; }
  if (right) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < NW0; ++k) { sv[u][k] = dg[k] - sv[u][k]; acc &= sv[u][k]; }
      const bool fit = (acc & guard_mask(MC)) == guard_mask(MC);
      if (ok[u] && !fit && cf) ++filt;
      ok[u] = ok[u] && fit;
    }
#pragma unroll
    for (int c = 0; c < mc_of(MC); ++c)
#pragma unroll
      for (int u = 0; u < U; ++u) fnv_step(lo[u], hi[u], coord<MC, true>(sv[u], c));
  } else {
#pragma unroll
    for (int c = 0; c < mc_of(MC); ++c)
#pragma unroll
      for (int u = 0; u < U; ++u) fnv_step(lo[u], hi[u], coord<MC, false>(sv[u], c));
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (q + u < C.q1) fn(u, (((uint64_t)hi[u] << 32) | lo[u]) & kmask, ok[u], C.lidx, W.R.loop_start + q + u);
  C.q = q + U;
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace msp
