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
// chunk of tiles through the compacted rectangle lists (k_rects).
#include <cstdint>
#include "msp_common.cuh"
#include "msp_kernels.h"
#include "msp_tile.cuh"

namespace msp {

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
                                     const RectDesc &R, uint32_t lidx, uint32_t qidx, const EnumArgs &A,
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
        const uint32_t *xm = d.side ? A.tab[2].mask : A.tab[0].mask;
        const uint32_t *ym = d.side ? A.tab[3].mask : A.tab[1].mask;
        jt.recs[i] = PairRec{d.gid, d.side, xi, yi, __ldg(xm + xi), __ldg(ym + yi), key};
      }
    }
  }
}

// ---------------------------------------------------------------- enumeration kernel

template <int MC, int KIND>
__global__ void __launch_bounds__(256) k_enum(const EnumArgs A, const JoinTable jt) {
  constexpr int NW = words_for(MC);
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t dg[NW > 0 ? NW : 1];
#pragma unroll
  for (int k = 0; k < NW; ++k) dg[k] = A.dpack[k];

  __shared__ __align__(16) uint32_t ybuf_all[8][kTQ * 8];
  for (uint64_t chunk = wid; chunk < A.nchunks; chunk += nwarps) {
    TileWalker W;
    W.init(A, chunk * A.chunk_tiles, min(chunk * A.chunk_tiles + A.chunk_tiles, A.total_tiles));
    unsigned long long filt = 0, hits = 0;
    TileCursor<stride_for(MC)> C;
    C.ybuf = ybuf_all[threadIdx.x >> 5];
    while (W.valid()) {
      begin_tile<MC>(A, W, lane, C);
      while (C.q < C.q1)
        step_keys<MC>(W, C, dg, filt, [&](int, uint64_t key, bool ok, uint32_t lidx, uint32_t qidx) {
          sink<KIND>(jt, W.d, key, ok, W.R, lidx, qidx, A, hits);
        });
      uint32_t old;
      if (W.advance(A, old)) {
        const unsigned long long f = warp_sum(filt), h = warp_sum(hits);
        if (lane == 0) {
          if (f) atomicAdd(A.batch_filtered + A.units[old].gid, f);
          if (h) atomicAdd(A.batch_hits + A.units[old].gid, h);
        }
        filt = hits = 0;
      }
    }
    const unsigned long long f = warp_sum(filt), h = warp_sum(hits);
    if (lane == 0) {
      if (f) atomicAdd(A.batch_filtered + W.d.gid, f);
      if (h) atomicAdd(A.batch_hits + W.d.gid, h);
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
