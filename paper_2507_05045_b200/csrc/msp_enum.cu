// msp_enum.cu -- K3/K4/K5: enumerate every candidate pair of a launch's batches, fold its residual
// into the 64-bit FNV hash and hand the key to a join sink.
//
// Replaces fastenum._expand (fastenum.py:150-158) + fastval._join_pairs (fastval.py:47-108):
//   left  pair (i, j): residual = cA[i] + cB[j]                          (fastval.py:66-74)
//   right pair (k, l): s = cC[k] + cD[l]; filtered if any s_c > d_c;     (fastval.py:83-99)
//                      residual = d - s
//   key = FNV fold over all m coordinates, coordinate 0 = alpha          (validate.py:34-50)
// Coordinate 0 is alpha on both sides, so its fold step is the per-batch constant h0 and the warp
// only folds the m-1 companion coordinates.  Companions arrive packed two u16 per u32 word; a
// single 32-bit add sums both halves, and on the right side a guard bit per half
// ((d + 0x8000) - s keeps bit 15 iff s <= d) turns the overshoot filter into one AND per word.
//
// Work decomposition: a batch is a union of rectangles X-run(alpha - w) x Y-run(w).  A warp tile is
// 32 entries of the rectangle's longer run (one per lane, companion vector in registers) x up to
// kTQ entries of the shorter run (warp-uniform loads, broadcast).  Each warp takes a contiguous
// chunk of tiles; rectangles are located by binary search over per-batch Y-run tile prefixes.
#include <cstdint>
#include "msp_common.cuh"
#include "msp_kernels.h"

namespace msp {

__device__ __forceinline__ uint32_t find_unit(const UnitDesc *u, uint32_t n, uint64_t T) {
  uint32_t lo = 0, hi = n;  // last u with tile_base <= T
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (u[mid].tile_base <= T) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t find_run(const uint32_t *P, uint32_t ny, uint32_t t) {
  uint32_t lo = 0, hi = ny;  // last r in [0, ny) with P[r] <= t  (P[ny] = total > t)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(P + mid) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

struct Rect {
  const uint32_t *lane_comp, *loop_comp;
  uint32_t lane_start, loop_start, L, Q, nl, nq;
  bool lane_is_x;
};

__device__ __forceinline__ void set_rect(const EnumArgs &A, const UnitDesc &d, uint32_t r, Rect &R) {
  const YRuns &yr = A.yr[d.side];
  const TableDev &X = A.tab[d.side ? 2 : 0];
  const TableDev &Y = A.tab[d.side ? 3 : 1];
  const uint32_t wy = __ldg(yr.w + r), ys = __ldg(yr.start + r), yl = __ldg(yr.len + r);
  const uint32_t wx = d.xw_total - wy;
  const uint32_t xs = __ldg(X.run_start + wx), xl = __ldg(X.run_end + wx) - xs;
  R.lane_is_x = xl >= yl;
  if (R.lane_is_x) {
    R.lane_comp = X.comp; R.loop_comp = Y.comp;
    R.lane_start = xs; R.L = xl; R.loop_start = ys; R.Q = yl;
  } else {
    R.lane_comp = Y.comp; R.loop_comp = X.comp;
    R.lane_start = ys; R.L = yl; R.loop_start = xs; R.Q = xl;
  }
  R.nl = (R.L + 31) >> 5;
  R.nq = (R.Q + kTQ - 1) / kTQ;
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- sinks (global hash table)

__device__ __forceinline__ bool table_find(const JoinTable &jt, const UnitDesc &d, uint64_t key,
                                           uint32_t &slot_out) {
  const uint32_t mask = (1u << d.region_log2) - 1;
  uint32_t s = home_slot(key, d.region_log2);
  const unsigned long long *K = jt.keys + d.region_base;
  for (uint32_t p = 0; p <= mask; ++p) {
    const unsigned long long k = K[s];
    if (k == key) { slot_out = d.region_base + s; return true; }
    if (k == 0) return false;
    s = (s + 1) & mask;
  }
  return false;
}

template <int KIND>
__device__ __forceinline__ void sink(const JoinTable &jt, const UnitDesc &d, uint64_t key, bool ok,
                                     const Rect &R, uint32_t lidx, uint32_t qidx, const EnumArgs &A,
                                     unsigned long long &hits) {
  if (!ok) return;
  if (d.npass > 1 && pass_of(key, d.npass) != d.pass) return;
  if constexpr (KIND == SINK_BUILD) {
    if (key == 0) { atomicAdd(jt.zero + d.slot, 1ull); return; }
    const uint32_t mask = (1u << d.region_log2) - 1;
    uint32_t s = home_slot(key, d.region_log2);
    unsigned long long *K = jt.keys + d.region_base;
    for (uint32_t p = 0; p <= mask; ++p) {
      const unsigned long long old = atomicCAS(K + s, 0ull, (unsigned long long)key);
      if (old == 0) return;                       // fresh key: stored count-1 stays 0
      if (old == key) { atomicAdd(jt.cnt + d.region_base + s, 1ull); return; }
      s = (s + 1) & mask;
    }
    atomicOr(jt.err, 1);                          // region full: host retries with more passes
  } else if constexpr (KIND == SINK_PROBE) {
    if (key == 0) {
      const unsigned long long z = jt.zero[d.slot];
      if (z) {
        hits += z;
        if (atomicExch(jt.zero_hit + d.slot, 1u) == 0u) {
          const unsigned long long i = atomicAdd(jt.nhits, 1ull);
          if (i < jt.hit_cap) jt.hits[i] = HitRec{d.gid, 0u, 0ull};
        }
      }
      return;
    }
    uint32_t slot;
    if (table_find(jt, d, key, slot)) {
      const unsigned long long c = jt.cnt[slot];
      hits += (c & ~kHitFlag) + 1;
      if (!(c & kHitFlag)) {
        const unsigned long long old = atomicOr(jt.cnt + slot, kHitFlag);
        if (!(old & kHitFlag)) {
          const unsigned long long i = atomicAdd(jt.nhits, 1ull);
          if (i < jt.hit_cap) jt.hits[i] = HitRec{d.gid, 0u, key};
        }
      }
    }
  } else {  // SINK_RECOVER: emit every pair whose key is in the batch's hit set
    bool present;
    if (key == 0) {
      present = d.flags & 1u;
    } else {
      uint32_t slot;
      present = table_find(jt, d, key, slot);
    }
    if (present) {
      const unsigned long long i = atomicAdd(jt.nrecs, 1ull);
      if (i < jt.rec_cap) {
        const uint32_t xi = R.lane_is_x ? lidx : qidx, yi = R.lane_is_x ? qidx : lidx;
        const TableDev &X = A.tab[d.side ? 2 : 0];
        const TableDev &Y = A.tab[d.side ? 3 : 1];
        jt.recs[i] = PairRec{d.gid, d.side, xi, yi, __ldg(X.mask + xi), __ldg(Y.mask + yi), key};
      }
    }
  }
}

// ---------------------------------------------------------------- enumeration kernel

template <int MC, int KIND>
__global__ void __launch_bounds__(256) k_enum(const EnumArgs A, const JoinTable jt) {
  constexpr int NW = words_for(MC);
  constexpr int SW = stride_for(MC);
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;

  uint32_t dg[NW > 0 ? NW : 1];
#pragma unroll
  for (int k = 0; k < NW; ++k) dg[k] = A.dpack[k];

  for (uint64_t chunk = wid; chunk < A.nchunks; chunk += nwarps) {
    uint64_t T = chunk * A.chunk_tiles;
    const uint64_t Tend = min(T + A.chunk_tiles, A.total_tiles);
    uint32_t u = find_unit(A.units, A.nunits, T);
    UnitDesc d = A.units[u];
    const uint32_t *P = A.prefix + d.prefix_off;
    uint32_t ny = A.yr[d.side].n;
    uint32_t tl = (uint32_t)(T - d.tile_base);
    uint32_t r = find_run(P, ny, tl);
    Rect R;
    set_rect(A, d, r, R);
    uint32_t local = tl - __ldg(P + r);
    uint32_t lc = local / R.nq, qc = local - lc * R.nq;
    unsigned long long filt = 0, hits = 0;

    while (true) {
      // ---------------- one warp tile: 32 lane entries x up to kTQ loop entries
      const uint32_t loff = lc * 32 + lane;
      const bool lok = loff < R.L;
      const uint32_t lidx = R.lane_start + (lok ? loff : 0);
      uint32_t lv[SW];
      load_vec<SW>(R.lane_comp, lidx, lv);
      const uint32_t q0 = qc * kTQ, q1 = min(R.Q, q0 + kTQ);
      const uint32_t h0lo = (uint32_t)d.h0, h0hi = (uint32_t)(d.h0 >> 32);
      const bool right = d.side != 0, cf = d.count_filter != 0;
      for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t qidx = R.loop_start + q;
        uint32_t yv[SW];
        load_vec<SW>(R.loop_comp, qidx, yv);
        uint32_t lo = h0lo, hi = h0hi;
        bool ok = lok;
        if (right) {
          uint32_t g[NW > 0 ? NW : 1];
          uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
          for (int k = 0; k < NW; ++k) { g[k] = dg[k] - (lv[k] + yv[k]); acc &= g[k]; }
          const bool fit = (acc & 0x80008000u) == 0x80008000u;
          if (lok && !fit && cf) ++filt;
          ok = ok && fit;
#pragma unroll
          for (int c = 0; c < MC; ++c) fnv_step(lo, hi, (g[c >> 1] >> (16 * (c & 1))) & 0x7FFFu);
        } else {
#pragma unroll
          for (int c = 0; c < MC; ++c)
            fnv_step(lo, hi, ((lv[c >> 1] + yv[c >> 1]) >> (16 * (c & 1))) & 0xFFFFu);
        }
        const uint64_t key = ((uint64_t)hi << 32) | lo;
        sink<KIND>(jt, d, key, ok, R, lidx, qidx, A, hits);
      }
      // ---------------- advance to the next tile of the chunk
      if (++T >= Tend) break;
      if (++qc < R.nq) continue;
      qc = 0;
      if (++lc < R.nl) continue;
      lc = 0;
      if (u + 1 < A.nunits && T >= A.units[u + 1].tile_base) {
        const unsigned long long f = warp_sum(filt), h = warp_sum(hits);
        if (lane == 0) {
          if (f) atomicAdd(A.unit_filtered + u, f);
          if (h) atomicAdd(A.unit_hits + u, h);
        }
        filt = hits = 0;
        while (u + 1 < A.nunits && T >= A.units[u + 1].tile_base) ++u;
        d = A.units[u];
        P = A.prefix + d.prefix_off;
        ny = A.yr[d.side].n;
      }
      tl = (uint32_t)(T - d.tile_base);
      r = find_run(P, ny, tl);
      set_rect(A, d, r, R);
    }
    const unsigned long long f = warp_sum(filt), h = warp_sum(hits);
    if (lane == 0) {
      if (f) atomicAdd(A.unit_filtered + u, f);
      if (h) atomicAdd(A.unit_hits + u, h);
    }
  }
}

template <int MC>
static void launch_mc(SinkKind kind, const EnumArgs &a, const JoinTable &jt, int grid, cudaStream_t st) {
  switch (kind) {
    case SINK_BUILD: k_enum<MC, SINK_BUILD><<<grid, 256, 0, st>>>(a, jt); break;
    case SINK_PROBE: k_enum<MC, SINK_PROBE><<<grid, 256, 0, st>>>(a, jt); break;
    default: k_enum<MC, SINK_RECOVER><<<grid, 256, 0, st>>>(a, jt); break;
  }
}

int launch_enum(int mc, SinkKind kind, const EnumArgs &args, const JoinTable &jt, int num_sms,
                cudaStream_t st) {
  if (args.nchunks == 0) return 0;
  uint64_t want = (args.nchunks + 7) / 8;  // 8 warps per block
  const uint64_t cap = (uint64_t)num_sms * 8;
  const int grid = (int)(want < cap ? (want ? want : 1) : cap);
  switch (mc) {
#define MSP_CASE(N) case N: launch_mc<N>(kind, args, jt, grid, st); break;
    MSP_CASE(0) MSP_CASE(1) MSP_CASE(2) MSP_CASE(3) MSP_CASE(4) MSP_CASE(5) MSP_CASE(6) MSP_CASE(7)
    MSP_CASE(8) MSP_CASE(9) MSP_CASE(10) MSP_CASE(11) MSP_CASE(12) MSP_CASE(13) MSP_CASE(14)
    MSP_CASE(15)
#undef MSP_CASE
    default: return -1;
  }
  return 0;
}

}  // namespace msp
