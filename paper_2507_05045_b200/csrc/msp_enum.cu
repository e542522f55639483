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
#include <algorithm>
#include <cstdint>
#include "msp_common.cuh"
#include "msp_kernels.h"
#include "msp_tile.cuh"

namespace msp {

// ---------------------------------------------------------------- sinks (global hash table)
//
// The table lives in L2 (<= 8M 64-bit key slots per wave, 64 MB).  Random L2 atomics and loads are
// throughput-bound only when many are in flight, so a warp step's kU keys are issued as kU
// independent CAS / loads before any result is inspected; collisions fall to a linear-probe slow
// path.  Duplicate counts and hit flags live in an epoch-tagged side array that never needs
// clearing: only the key array is reset per wave.

constexpr unsigned long long kCntMask = (1ull << 39) - 1;
constexpr unsigned long long kCntFlag = 1ull << 39;

__device__ __forceinline__ bool table_find(const JoinTable &jt, const UnitDesc &d, uint64_t key,
                                           uint32_t s, uint32_t &slot_out) {
  const uint32_t mask = (1u << d.region_log2) - 1;
  const unsigned long long *K = jt.keys + d.region_base;
  for (uint32_t p = 0; p <= mask; ++p) {
    const unsigned long long k = K[s];
    if (k == key) { slot_out = d.region_base + s; return true; }
    if (k == 0) return false;
    s = (s + 1) & mask;
  }
  return false;
}

__device__ __forceinline__ void count_duplicate(const JoinTable &jt, uint32_t slot) {
  unsigned long long *c = jt.cnt + slot;
  unsigned long long old = *c, assumed;
  do {
    assumed = old;
    const unsigned long long nv = (assumed >> 40) == jt.epoch ? assumed + 1 : (jt.epoch << 40) | 1ull;
    old = atomicCAS(c, assumed, nv);
  } while (old != assumed);
}

// hits += multiplicity of the build key in `slot`; the first probe to hit it records (gid, key).
__device__ __forceinline__ void register_hit(const JoinTable &jt, uint32_t gid, uint32_t slot, uint64_t key,
                                             unsigned long long &hits) {
  unsigned long long *c = jt.cnt + slot;
  unsigned long long cur = *c;
  const bool valid = (cur >> 40) == jt.epoch;
  hits += (valid ? (cur & kCntMask) : 0ull) + 1;
  if (valid && (cur & kCntFlag)) return;
  unsigned long long assumed;
  do {
    assumed = cur;
    const bool v = (assumed >> 40) == jt.epoch;
    if (v && (assumed & kCntFlag)) return;  // someone else recorded it
    const unsigned long long nv = v ? (assumed | kCntFlag) : ((jt.epoch << 40) | kCntFlag);
    cur = atomicCAS(c, assumed, nv);
  } while (cur != assumed);
  const unsigned long long i = atomicAdd(jt.nhits, 1ull);
  if (i < jt.hit_cap) jt.hits[i] = HitRec{gid, 0u, key};
}

template <int KIND>
__device__ __forceinline__ void sink_batch(const JoinTable &jt, const UnitDesc &d, const uint64_t (&key)[kU],
                                           bool (&ok)[kU], const RectDesc &R, const uint32_t (&lidx)[kU],
                                           const uint32_t (&qidx)[kU], const EnumArgs &A,
                                           unsigned long long &hits, const uint32_t *rfilt = nullptr) {
#pragma unroll
  for (int u = 0; u < kU; ++u)
    if (ok[u] && d.npass > 1 && pass_of(key[u], d.npass) != d.pass) ok[u] = false;
  if constexpr (KIND == SINK_BUILD) {
    const uint32_t mask = (1u << d.region_log2) - 1;
    unsigned long long *K = jt.keys + d.region_base;
    uint32_t s[kU];
    unsigned long long old[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {  // kU independent CAS in flight
      s[u] = home_slot(key[u], d.region_log2);
      old[u] = (ok[u] && key[u] != 0) ? atomicCAS(K + s[u], 0ull, (unsigned long long)key[u]) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!ok[u]) continue;
      if (key[u] == 0) { atomicAdd(jt.zero + d.slot, 1ull); continue; }
      if (old[u] == 0) continue;                            // fresh key
      if (old[u] == key[u]) { count_duplicate(jt, d.region_base + s[u]); continue; }
      uint32_t t = (s[u] + 1) & mask;                       // collision: linear probe
      bool placed = false;
      for (uint32_t p = 0; p < mask; ++p) {
        const unsigned long long o = atomicCAS(K + t, 0ull, (unsigned long long)key[u]);
        if (o == 0) { placed = true; break; }
        if (o == key[u]) { count_duplicate(jt, d.region_base + t); placed = true; break; }
        t = (t + 1) & mask;
      }
      if (!placed) atomicOr(jt.err, 1);                     // region full
    }
  } else if constexpr (KIND == SINK_PROBE) {
    const uint32_t mask = (1u << d.region_log2) - 1;
    const unsigned long long *K = jt.keys + d.region_base;
    uint32_t s[kU];
    unsigned long long t[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {  // kU independent loads in flight
      s[u] = home_slot(key[u], d.region_log2);
      t[u] = (ok[u] && key[u] != 0) ? K[s[u]] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!ok[u]) continue;
      if (key[u] == 0) {
        const unsigned long long z = jt.zero[d.slot];
        if (z) {
          hits += z;
          if (atomicExch(jt.zero_hit + d.slot, 1u) == 0u) {
            const unsigned long long i = atomicAdd(jt.nhits, 1ull);
            if (i < jt.hit_cap) jt.hits[i] = HitRec{d.gid, 0u, 0ull};
          }
        }
        continue;
      }
      if (t[u] == key[u]) { register_hit(jt, d.gid, d.region_base + s[u], key[u], hits); continue; }
      if (t[u] == 0) continue;                              // miss
      uint32_t slot;
      if (table_find(jt, d, key[u], (s[u] + 1) & mask, slot)) register_hit(jt, d.gid, slot, key[u], hits);
    }
  } else if constexpr (KIND == SINK_NONE) {  // diagnostic: keep the keys live, touch nothing
#pragma unroll
    for (int u = 0; u < kU; ++u) hits ^= ok[u] ? key[u] : 0ull;
  } else {  // SINK_RECOVER: emit every pair whose key is in the batch's hit set
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!ok[u]) continue;
      bool present;
      if (key[u] == 0) {
        present = d.flags & 1u;
      } else if (!((rfilt[key[u] >> 53] >> ((key[u] >> 48) & 31u)) & 1u)) {
        present = false;  // no hit key of the launch starts with these 16 bits (shared-memory filter)
      } else {
        uint32_t slot;
        present = table_find(jt, d, key[u], home_slot(key[u], d.region_log2), slot);
      }
      if (present) {
        const unsigned long long i = atomicAdd(jt.nrecs, 1ull);
        if (i < jt.rec_cap) {
          const uint32_t xi = R.lane_is_x() ? lidx[u] : qidx[u], yi = R.lane_is_x() ? qidx[u] : lidx[u];
          const uint32_t *xm = d.side ? A.tab[2].mask : A.tab[0].mask;
          const uint32_t *ym = d.side ? A.tab[3].mask : A.tab[1].mask;
          jt.recs[i] = PairRec{d.gid, d.side, xi, yi, __ldg(xm + xi), __ldg(ym + yi), key[u]};
        }
      }
    }
  }
}

// Bulk table operations for one unit's staged keys (one warp): 8 keys per lane are loaded from
// the warp's shared-memory stage and their CAS / loads are all issued before any result is used,
// so each warp keeps 256 L2 operations in flight while the other warps keep hashing.
template <int KIND>
__device__ __forceinline__ void sink_bulk(const JoinTable &jt, const UnitDesc &d, const unsigned long long *stage,
                                          uint32_t cnt, uint32_t lane, unsigned long long &hits) {
  constexpr int V = 8;
  const uint32_t mask = (1u << d.region_log2) - 1;
  unsigned long long *K = jt.keys + d.region_base;
  for (uint32_t j0 = 0; j0 < cnt; j0 += 32 * V) {
    unsigned long long k[V];
    uint32_t s[V];
    unsigned long long r[V];
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const uint32_t j = j0 + u * 32 + lane;
      k[u] = j < cnt ? stage[j] : 0ull;
      s[u] = home_slot(k[u], d.region_log2);
    }
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const bool live = j0 + u * 32 + lane < cnt && k[u] != 0;
      if constexpr (KIND == SINK_BUILD) r[u] = live ? atomicCAS(K + s[u], 0ull, k[u]) : 0ull;
      else r[u] = live ? K[s[u]] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < V; ++u) {
      if (j0 + u * 32 + lane >= cnt) continue;
      if constexpr (KIND == SINK_BUILD) {
        if (k[u] == 0) { atomicAdd(jt.zero + d.slot, 1ull); continue; }
        if (r[u] == 0) continue;
        if (r[u] == k[u]) { count_duplicate(jt, d.region_base + s[u]); continue; }
        uint32_t t = (s[u] + 1) & mask;
        bool placed = false;
        for (uint32_t p = 0; p < mask; ++p) {
          const unsigned long long o = atomicCAS(K + t, 0ull, k[u]);
          if (o == 0) { placed = true; break; }
          if (o == k[u]) { count_duplicate(jt, d.region_base + t); placed = true; break; }
          t = (t + 1) & mask;
        }
        if (!placed) atomicOr(jt.err, 1);
      } else {
        if (k[u] == 0) {
          const unsigned long long z = jt.zero[d.slot];
          if (z) {
            hits += z;
            if (atomicExch(jt.zero_hit + d.slot, 1u) == 0u) {
              const unsigned long long i = atomicAdd(jt.nhits, 1ull);
              if (i < jt.hit_cap) jt.hits[i] = HitRec{d.gid, 0u, 0ull};
            }
          }
          continue;
        }
        if (r[u] == k[u]) { register_hit(jt, d.gid, d.region_base + s[u], k[u], hits); continue; }
        if (r[u] == 0) continue;
        uint32_t slot;
        if (table_find(jt, d, k[u], (s[u] + 1) & mask, slot)) register_hit(jt, d.gid, slot, k[u], hits);
      }
    }
  }
}

// ---------------------------------------------------------------- enumeration kernel

constexpr uint32_t kEnumStage = 512;  // keys a warp stages before a bulk table pass

template <int MC, int KIND>
__global__ void __launch_bounds__(256, 2) k_enum(const EnumArgs A, const JoinTable jt) {
  constexpr int NW = words_for(MC);
  constexpr bool kBulk = KIND == SINK_BUILD || KIND == SINK_PROBE;
  const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint64_t wid = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t dg[NW > 0 ? NW : 1];
#pragma unroll
  for (int k = 0; k < NW; ++k) dg[k] = A.dpack[k];

  __shared__ __align__(16) uint32_t ybuf_all[8][kTQ * stride_for(MC)];
  __shared__ unsigned long long stage_all[kBulk ? 8 : 1][kBulk ? kEnumStage : 1];
  // hit recovery: a 64K-bit filter of the hit keys' top 16 bits, so almost every key is rejected
  // by one shared load instead of a global hash-table probe
  __shared__ uint32_t rfilt[KIND == SINK_RECOVER ? 2048 : 1];
  if constexpr (KIND == SINK_RECOVER) {
    for (uint32_t i = threadIdx.x; i < 2048u; i += blockDim.x) rfilt[i] = 0u;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < jt.nkeys; i += blockDim.x) {
      const unsigned long long k = jt.keys[i];
      if (k) atomicOr(&rfilt[k >> 53], 1u << ((k >> 48) & 31u));
    }
    __syncthreads();
  }
  unsigned long long *stage = stage_all[kBulk ? wl : 0];
  for (uint64_t chunk = wid; chunk < A.nchunks; chunk += nwarps) {
    TileWalker W;
    W.init(A, chunk * A.chunk_tiles, min(chunk * A.chunk_tiles + A.chunk_tiles, A.total_tiles));
    unsigned long long filt = 0, hits = 0;
    uint32_t cnt = 0;
    TileCursor<stride_for(MC)> C;
    C.ybuf = ybuf_all[wl];
    while (W.valid()) {
      begin_tile<MC>(A, W, lane, C);
      while (C.q < C.q1) {
        if constexpr (kBulk) {
          step_keys<MC>(W, C, dg, filt, A.key_mask, [&](int, uint64_t key, bool ok, uint32_t, uint32_t) {
            if (ok && W.d.npass > 1 && pass_of(key, W.d.npass) != W.d.pass) ok = false;
            const uint32_t m = __ballot_sync(0xffffffffu, ok);
            if (ok) stage[cnt + __popc(m & lt_mask)] = key;
            cnt += __popc(m);
          });
          if (cnt + 32 * kU > kEnumStage) {
            __syncwarp();
            sink_bulk<KIND>(jt, W.d, stage, cnt, lane, hits);
            __syncwarp();
            cnt = 0;
          }
        } else {
          uint64_t kk[kU];
          bool okk[kU];
          uint32_t li[kU], qi[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) { okk[u] = false; kk[u] = 0; li[u] = qi[u] = 0; }
          step_keys<MC>(W, C, dg, filt, A.key_mask, [&](int u, uint64_t key, bool ok, uint32_t lidx, uint32_t qidx) {
            kk[u] = key; okk[u] = ok; li[u] = lidx; qi[u] = qidx;
          });
          sink_batch<KIND>(jt, W.d, kk, okk, W.R, li, qi, A, hits, rfilt);
        }
      }
      const UnitDesc dprev = W.d;
      uint32_t old;
      const bool changed = W.advance(A, old);
      if constexpr (kBulk) {
        if ((changed || !W.valid()) && cnt) {  // the stage holds one unit's keys
          __syncwarp();
          sink_bulk<KIND>(jt, dprev, stage, cnt, lane, hits);
          __syncwarp();
          cnt = 0;
        }
      }
      if (changed) {
        const unsigned long long f = warp_sum(filt), h = warp_sum(hits);
        if (lane == 0) {
          if (f) atomicAdd(A.batch_filtered + dprev.gid, f);
          if (h) atomicAdd(A.batch_hits + dprev.gid, h);
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

// Table clear with ordinary 16-byte stores so the cleared lines stay resident in L2 for the build
// (a DMA memset does not leave the 64 MB table in L2; measured 33% L2 hit rate on the CAS).
__global__ void k_clear(uint4 *p, size_t n16) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) p[i] = z;
}

void launch_clear(void *p, size_t bytes, int num_sms, cudaStream_t st) {
  const size_t n16 = bytes / 16;
  if (n16) k_clear<<<num_sms * 4, 512, 0, st>>>(reinterpret_cast<uint4 *>(p), n16);
  if (bytes % 16) cudaMemsetAsync(reinterpret_cast<char *>(p) + n16 * 16, 0, bytes % 16, st);
}

template <int MC>
static void launch_mc(SinkKind kind, const EnumArgs &a, const JoinTable &jt, int grid, cudaStream_t st) {
  switch (kind) {
    case SINK_BUILD: k_enum<MC, SINK_BUILD><<<grid, 256, 0, st>>>(a, jt); break;
    case SINK_PROBE: k_enum<MC, SINK_PROBE><<<grid, 256, 0, st>>>(a, jt); break;
    case SINK_NONE: k_enum<MC, SINK_NONE><<<grid, 256, 0, st>>>(a, jt); break;
    default: k_enum<MC, SINK_RECOVER><<<grid, 256, 0, st>>>(a, jt); break;
  }
}

// ---------------------------------------------------------------- one-sided hit recovery

// Hash of a table entry's (row-0 weight, companion words): build and lookup must agree.
__device__ __forceinline__ uint64_t entry_hash(uint64_t w, const uint32_t *words, int nw) {
  uint64_t h = w * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  for (int k = 0; k < nw; ++k) {
    h ^= words[k];
    h *= 0x100000001B3ull;
    h ^= h >> 29;
  }
  return h;
}

// Every Y entry into an open-addressing table of 2^log2 slots (entry + 1; 0 = empty).
__global__ void k_vhash_build(const LookupArgs a, uint32_t *slots) {
  const uint32_t msk = (1u << a.log2) - 1u;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.Y.n; v += gridDim.x * blockDim.x) {
    uint32_t s = (uint32_t)(entry_hash(a.Y.w[v], a.Y.comp + (size_t)v * a.sw, a.nw) >> (64 - a.log2));
    while (atomicCAS(slots + s, 0u, v + 1u) != 0u) s = (s + 1u) & msk;
  }
}

// Target t (blockIdx.y stride) x X entry x: the Y entries equal to target - X[x] (row 0 and every
// companion coordinate, exactly), emitted as pairs of the target's side.
__global__ void k_lookup(const LookupArgs a) {
  const uint32_t msk = (1u << a.log2) - 1u;
  for (uint32_t t = blockIdx.y; t < a.ntg; t += gridDim.y) {
    const LookupTarget &T = a.tg[t];
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < a.X.n; x += gridDim.x * blockDim.x) {
      const uint64_t wx = a.X.w[x];
      if (T.w0 < wx) continue;
      const uint64_t wt = T.w0 - wx;
      const uint32_t *cx = a.X.comp + (size_t)x * a.sw;
      uint32_t words[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      bool ok = true;
      for (int c = 0; c < a.mc; ++c) {
        const uint32_t v = a.wide ? cx[c] : (((c & 1) ? cx[c >> 1] >> 16 : cx[c >> 1]) & 0xFFFFu);
        if (T.tc[c] < v) { ok = false; break; }
        const uint32_t r = T.tc[c] - v;
        if (a.wide) words[c] = r;
        else if (r > 0xFFFFu) { ok = false; break; }
        else words[c >> 1] |= r << (16 * (c & 1));
      }
      if (!ok) continue;
      uint32_t s = (uint32_t)(entry_hash(wt, words, a.nw) >> (64 - a.log2));
      for (uint32_t e; (e = a.slots[s]) != 0u; s = (s + 1u) & msk) {
        const uint32_t y = e - 1u;
        if (a.Y.w[y] != wt) continue;
        const uint32_t *cy = a.Y.comp + (size_t)y * a.sw;
        bool eq = true;
        for (int k = 0; k < a.nw; ++k) eq = eq && cy[k] == words[k];
        if (!eq) continue;
        const unsigned long long o = atomicAdd(a.nout, 1ull);
        if (o < a.cap) a.out[o] = PairRec{T.gid, T.side, x, y, a.X.mask[x], a.Y.mask[y], T.key};
      }
    }
  }
}

void launch_vhash_build(const LookupArgs &a, uint32_t *slots, cudaStream_t st) {
  k_vhash_build<<<(unsigned)std::min<uint64_t>((a.Y.n + 255) / 256, 4096), 256, 0, st>>>(a, slots);
}

void launch_lookup(const LookupArgs &a, cudaStream_t st) {
  if (!a.ntg) return;
  const dim3 grid((unsigned)std::min<uint64_t>((a.X.n + 255) / 256, 1024), std::min<uint32_t>(a.ntg, 65535));
  k_lookup<<<grid, 256, 0, st>>>(a);
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
    MSP_CASE(15) MSP_CASE(17) MSP_CASE(18) MSP_CASE(19) MSP_CASE(20) MSP_CASE(21) MSP_CASE(22)
    MSP_CASE(23) MSP_CASE(24)
#undef MSP_CASE
    default: return -1;
  }
  return 0;
}

}  // namespace msp
