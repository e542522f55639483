// msp_part.cu -- K4/K5 as a radix-partitioned shared-memory hash join (the default join path).
//
// Same semantics as fastval._join_pairs (fastval.py:47-108): every left key is joined with every
// unfiltered right key of the same batch and all full-64-bit-hash-equal pairs are counted
// (hash_hits) and reported for exact confirmation.  Instead of bucket chains in DRAM, one wave of
// batches is joined in two launches:
//
//   k_scatter  enumerate + hash (msp_tile.cuh), stage 4096 keys per CTA round in shared memory,
//              counting-sort them by bucket (top bits of the key within the batch), reserve space
//              per bucket with one global atomic, and write bucket-contiguous runs into an
//              L2-resident scratch.  Right pairs that overshoot d are counted, not written.
//   k_join     one CTA per bucket: insert the build side's keys (the smaller side of the batch)
//              into a 16K-slot (key, count) table in shared memory, stream the probe side's keys
//              through it, count hash hits, record each hit key once for recovery.
//
// The per-bucket capacity is sized from the exact batch counts (mean + 7 sigma); a bucket that
// overflows (duplicate-heavy instances) marks its batch, which the host re-joins with the global
// table path (msp_enum.cu), so results never depend on the partitioning.
#include <cstdint>
#include <type_traits>
#include "msp_common.cuh"
#include "msp_kernels.h"
#include "msp_tile.cuh"

namespace msp {

constexpr int kScatterWarps = 16;
constexpr int kWarpStage = 512;                         // keys a warp stages per round
constexpr int kStage = kScatterWarps * kWarpStage;      // keys staged per CTA round
constexpr uint32_t kOvf = 0x80000000u;
constexpr int kHistEntries = 2 * kMaxWaveBuckets;       // (role, bucket)

size_t scatter_smem_bytes() {
  return (size_t)kStage * (8 + 8 + 2 + 2 + 2) + (size_t)kHistEntries * 4 * 3 + 64;
}

// Shared-memory views of one CTA's staging area.
struct Stage {
  unsigned long long *skey, *sorted;
  uint16_t *sbkt, *rank, *sortb;
  uint32_t *hist, *off, *abase;
  uint8_t *ovf;
  uint32_t *warp_tot;
};

__device__ __forceinline__ Stage stage_views(unsigned char *smem, uint8_t *ovf, uint32_t *warp_tot) {
  Stage g;
  g.skey = reinterpret_cast<unsigned long long *>(smem);
  g.sorted = g.skey + kStage;
  g.sbkt = reinterpret_cast<uint16_t *>(g.sorted + kStage);
  g.rank = g.sbkt + kStage;
  g.sortb = g.rank + kStage;
  g.hist = reinterpret_cast<uint32_t *>(g.sortb + kStage);
  g.off = g.hist + kHistEntries;
  g.abase = g.off + kHistEntries;
  g.ovf = ovf;
  g.warp_tot = warp_tot;
  return g;
}

// Append one warp-step of keys densely to the warp's stage (ballot + popc) and rank each key
// within its (role, bucket) with one shared-memory atomic.
__device__ __forceinline__ void stage_key(const Stage &g, uint32_t warp, uint32_t lane_lt, uint32_t &cnt,
                                          uint64_t key, uint32_t b, bool ok) {
  const uint32_t m = __ballot_sync(0xffffffffu, ok);
  if (ok) {
    const uint32_t pos = warp * kWarpStage + cnt + __popc(m & lane_lt);
    g.skey[pos] = key;
    g.sbkt[pos] = (uint16_t)b;
    g.rank[pos] = (uint16_t)atomicAdd(g.hist + b, 1u);
  }
  cnt += __popc(m);
}

// After a __syncthreads: scan the round's bucket counts, reserve one global range per nonempty
// bucket (the thread's kPer reservations are independent atomics issued back to back), reorder the
// staged keys into bucket-sorted runs and write the runs out coalesced.  Ends synchronised, with
// the histogram zeroed for the next round.
__device__ __forceinline__ void flush_round(const Stage &g, const PartArgs &S, uint32_t cnt) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nbw = S.nb, nent = 2 * nbw;
  constexpr int kPer = kHistEntries / (kScatterWarps * 32);
  const uint32_t j0 = tid * kPer;
  uint32_t hv[kPer], local = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    hv[k] = j0 + k < nent ? g.hist[j0 + k] : 0u;
    g.hist[j0 + k] = 0u;  // ready for the next fill
    local += hv[k];
  }
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) g.warp_tot[warp] = incl;
  uint32_t gres[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t j = j0 + k, role = j >= nbw;
    gres[k] = hv[k] ? atomicAdd((role ? S.fill[1] : S.fill[0]) + (j - role * nbw), hv[k]) : 0u;
  }
  __syncthreads();
  uint32_t run = incl - local;
  for (uint32_t w = 0; w < warp; ++w) run += g.warp_tot[w];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t j = j0 + k;
    if (j < nent) {
      g.off[j] = run;
      g.ovf[j] = 0;
      if (hv[k]) {
        const uint32_t role = j >= nbw, b = j - role * nbw;
        if (gres[k] + hv[k] > __ldg((role ? S.cap[1] : S.cap[0]) + b)) {
          g.ovf[j] = 1;
          atomicOr(S.batch_ovf + __ldg(S.gid + b), 1u);
        } else {
          g.abase[j] = __ldg((role ? S.start[1] : S.start[0]) + b) + gres[k] - run;
        }
      }
    }
    run += hv[k];
  }
#ifndef MSP_SCATTER_DIRECT
  uint32_t total = 0;
  for (int w = 0; w < kScatterWarps; ++w) total += g.warp_tot[w];
  __syncthreads();
  for (uint32_t j = lane; j < cnt; j += 32) {  // each warp reorders its own staged keys
    const uint32_t i = warp * kWarpStage + j;
    const uint16_t b = g.sbkt[i];
    const uint32_t pos = g.off[b] + g.rank[i];
    g.sorted[pos] = g.skey[i];
    g.sortb[pos] = b;
  }
  __syncthreads();
  for (uint32_t pos = tid; pos < total; pos += blockDim.x) {
    const uint16_t b = g.sortb[pos];
    if (!g.ovf[b]) S.scratch[g.abase[b] + pos] = g.sorted[pos];
  }
  __syncthreads();
#else
  __syncthreads();
  for (uint32_t j = lane; j < cnt; j += 32) {  // direct: each key to its final slot
    const uint32_t i = warp * kWarpStage + j;
    const uint16_t b = g.sbkt[i];
    if (!g.ovf[b]) S.scratch[g.abase[b] + g.off[b] + g.rank[i]] = g.skey[i];
  }
  __syncthreads();
#endif
}

template <int MC, bool ITEMS>
__global__ void __launch_bounds__(kScatterWarps * 32) k_scatter(const EnumArgs A, const PartArgs S) {
  constexpr int NW = words_for(MC);
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t warp_tot[kScatterWarps];
  __shared__ uint8_t ovf[kHistEntries];
  __shared__ __align__(16) uint32_t ybuf_all[kScatterWarps][kTQ * stride_for(MC)];
  const Stage g = stage_views(smem, ovf, warp_tot);

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t nbw = S.nb;
  uint32_t dg[NW > 0 ? NW : 1];
#pragma unroll
  for (int k = 0; k < NW; ++k) dg[k] = A.dpack[k];
  for (uint32_t i = tid; i < kHistEntries; i += blockDim.x) g.hist[i] = 0;
  __syncthreads();

  // ITEMS: one-tile work items statically strided over the grid (small waves, balanced);
  // else: contiguous tile chunks per warp (huge batches: large chunks amortise the search).
  using Walker = typename std::conditional<ITEMS, ItemWalker, TileWalker>::type;
  Walker W;
  uint64_t chunk = (uint64_t)blockIdx.x * kScatterWarps + warp;
  const uint64_t nwarps = (uint64_t)gridDim.x * kScatterWarps;
  if constexpr (ITEMS) {
    W.init(A, chunk, nwarps);
  } else {
    W.init(A, min(chunk * A.chunk_tiles, A.total_tiles), min(chunk * A.chunk_tiles + A.chunk_tiles, A.total_tiles));
  }
  TileCursor<stride_for(MC)> C;
  C.ybuf = ybuf_all[warp];
  bool have;
  if constexpr (ITEMS) have = W.grab(A, lane); else have = W.valid();
  if (have) begin_tile<MC>(A, W, lane, C);
  unsigned long long filt = 0, diag_acc = 0;
  while (true) {
    uint32_t cnt = 0;
    while (have && cnt + 32 * kU <= (uint32_t)kWarpStage) {
      const uint32_t bbase = ((W.d.flags >> 1) & 1u) * nbw + W.d.region_base;
      const uint32_t bits = W.d.region_log2;
      if (A.diag) {  // diagnostic timing: hash only, no staging / partition
        step_keys<MC>(W, C, dg, filt, [&](int, uint64_t key, bool ok, uint32_t, uint32_t) {
          if (ok) diag_acc ^= key;
        });
      } else {
        step_keys<MC>(W, C, dg, filt, [&](int, uint64_t key, bool ok, uint32_t, uint32_t) {
          stage_key(g, warp, lt_mask, cnt, key, bbase + (bits ? (uint32_t)(key >> (64 - bits)) : 0u), ok);
        });
      }
      if (C.q >= C.q1) {
        uint32_t old_gid;
        bool changed;
        if constexpr (ITEMS) {
          changed = W.advance(A, lane, old_gid);
        } else {
          uint32_t old_u;
          changed = W.advance(A, old_u);
          old_gid = A.units[old_u].gid;
          if (!W.valid()) {  // next contiguous chunk of this warp
            chunk += nwarps;
            changed = true;
            W.init(A, min(chunk * A.chunk_tiles, A.total_tiles), min(chunk * A.chunk_tiles + A.chunk_tiles, A.total_tiles));
          }
        }
        if (changed) {
          const unsigned long long f = warp_sum(filt);
          if (lane == 0 && f) atomicAdd(A.batch_filtered + old_gid, f);
          filt = 0;
        }
        have = W.valid();
        if (have) begin_tile<MC>(A, W, lane, C);
      }
    }
    if (!__syncthreads_or(cnt > 0)) break;
    flush_round(g, S, cnt);
  }
  if (diag_acc == 0x123456789ull) A.batch_filtered[0] = diag_acc;  // keep the diagnostic keys live
}

// Level 2 of the huge-batch path: stream already-hashed keys back from coarse bucket regions
// (HBM) and re-partition them into fine buckets (L2 scratch) for k_join.  Each CTA round takes
// kStage consecutive input slots; slots past a region's fill are empty.
__global__ void __launch_bounds__(kScatterWarps * 32) k_rescatter(const RescatterArgs R, const PartArgs S) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t warp_tot[kScatterWarps];
  __shared__ uint8_t ovf[kHistEntries];
  const Stage g = stage_views(smem, ovf, warp_tot);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t nbw = S.nb;
  for (uint32_t i = tid; i < kHistEntries; i += blockDim.x) g.hist[i] = 0;
  __syncthreads();
  for (uint64_t chunk = blockIdx.x; chunk * kStage < R.total; chunk += gridDim.x) {
    const uint64_t base = chunk * kStage + (uint64_t)warp * kWarpStage;
    uint32_t s = 0;
    {
      uint32_t lo = 0, hi = R.nsrc;  // last source with in_base <= base
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (R.src[mid].in_base <= base) lo = mid; else hi = mid;
      }
      s = lo;
    }
    uint32_t cnt = 0;
#pragma unroll 4
    for (int k = 0; k < kWarpStage / 32; ++k) {
      const uint64_t idx = base + (uint64_t)k * 32 + lane;
      uint32_t sl = s;
      while (sl + 1 < R.nsrc && idx >= R.src[sl + 1].in_base) ++sl;
      const RescatterSrc &src = R.src[sl];
      const uint64_t local = idx - src.in_base;
      const bool ok = idx < R.total && local < min(*src.fill, src.cap);
      const uint64_t key = ok ? src.keys[local] : 0ull;
      const uint32_t fb = src.fbits ? (uint32_t)((key << src.coarse_bits) >> (64 - src.fbits)) : 0u;
      stage_key(g, warp, lt_mask, cnt, key, src.role * nbw + src.fine_base + fb, ok);
    }
    __syncthreads();
    flush_round(g, S, cnt);
  }
}

constexpr int kJoinThreads = 1024;
constexpr int kJoinSlots = 1 << kJoinSlotsLog2;        // 16K key slots
constexpr int kJBuckets = kJoinSlots / 4;               // 4K buckets of 4 slots
constexpr int kStash = 256;                             // keys whose two buckets were both full
constexpr int kHitWords = (kJoinSlots + kStash) / 32;

// Shared-memory join table of one bucket: two-choice hashing into 4-slot buckets.  Each slot keeps
// the full 64-bit key and, in a packed word per bucket, a 16-bit fingerprint, so a probe reads two
// fingerprint words and two counts and compares four fingerprints per word with one SIMD compare;
// the full keys are read only on a fingerprint match (~1e-4 of probes plus the true hits).  No
// probe ever loops, so warps do not diverge on chain lengths.  Only the counts are cleared per
// bucket (slots past a bucket's count are never read).
struct JoinSmem {
  unsigned long long key[kJBuckets][4];
  unsigned long long fp[kJBuckets];     // four 16-bit fingerprints
  uint32_t cnt[kJBuckets];              // claims (may exceed 4: failed claims spill over)
  unsigned long long stash[kStash];
  uint32_t hitbits[kHitWords];
  unsigned long long bhits[kJoinThreads / 32];
  uint32_t nstash, zb, zhit, ovf;
};

size_t join_smem_bytes() { return sizeof(JoinSmem); }

struct JoinHash { uint32_t b1, b2, fp; };
__device__ __forceinline__ JoinHash join_hash(unsigned long long k) {
  const unsigned long long m = k * kGolden;  // odd multiplier: a bijection on 64-bit keys
  JoinHash h;
  h.b1 = (uint32_t)(m >> 52);
  h.b2 = (uint32_t)(m >> 40) & (kJBuckets - 1);
  if (h.b2 == h.b1) h.b2 ^= 1u;
  h.fp = (uint32_t)(m >> 24) & 0xFFFFu;
  return h;
}

// Lanes of `w` (four 16-bit fingerprints) equal to fp, as a 4-bit mask, restricted to n slots.
__device__ __forceinline__ uint32_t fp_match(unsigned long long w, uint32_t fp, uint32_t n) {
  const uint32_t f2 = fp * 0x10001u;
  const uint32_t lo = __vcmpeq2((uint32_t)w, f2), hi = __vcmpeq2((uint32_t)(w >> 32), f2);
  const uint32_t m = (lo & 1u) | ((lo >> 15) & 2u) | ((hi & 1u) << 2) | ((hi >> 13) & 8u);
  return m & ((1u << n) - 1u);
}

__device__ __forceinline__ void join_insert(JoinSmem &T, unsigned long long k) {
  const JoinHash h = join_hash(k);
  const uint32_t c1 = T.cnt[h.b1], c2 = T.cnt[h.b2];
  uint32_t b = c1 <= c2 ? h.b1 : h.b2, o = c1 <= c2 ? h.b2 : h.b1;
  uint32_t s = atomicAdd(&T.cnt[b], 1u);
  if (s >= 4) { b = o; s = atomicAdd(&T.cnt[b], 1u); }
  if (s < 4) {
    T.key[b][s] = k;
    atomicOr(reinterpret_cast<unsigned long long *>(&T.fp[b]), (unsigned long long)h.fp << (16 * s));
  } else {
    const uint32_t i = atomicAdd(&T.nstash, 1u);
    if (i < (uint32_t)kStash) T.stash[i] = k; else T.ovf = 1u;
  }
}

// Multiplicity of k in the table; *first = slot id of its first copy (bucket-major, then stash).
__device__ __forceinline__ uint32_t join_count(const JoinSmem &T, unsigned long long k, uint32_t nstash,
                                               uint32_t &first) {
  const JoinHash h = join_hash(k);
  const uint32_t n1 = min(T.cnt[h.b1], 4u), n2 = min(T.cnt[h.b2], 4u);
  uint32_t m1 = fp_match(T.fp[h.b1], h.fp, n1), m2 = fp_match(T.fp[h.b2], h.fp, n2);
  uint32_t c = 0;
  first = 0xFFFFFFFFu;
  if (m1 | m2) {  // rare: fingerprint hit, compare full keys
    while (m1) {
      const uint32_t s = __ffs(m1) - 1;
      m1 &= m1 - 1;
      if (T.key[h.b1][s] == k) { if (!c) first = h.b1 * 4 + s; ++c; }
    }
    while (m2) {
      const uint32_t s = __ffs(m2) - 1;
      m2 &= m2 - 1;
      if (T.key[h.b2][s] == k) { if (!c) first = h.b2 * 4 + s; ++c; }
    }
  }
  for (uint32_t i = 0; i < nstash; ++i)
    if (T.stash[i] == k) { if (!c) first = kJoinSlots + i; ++c; }
  return c;
}

__global__ void __launch_bounds__(kJoinThreads, 1) k_join(const PartArgs S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JoinSmem &T = *reinterpret_cast<JoinSmem *>(smem_raw);
  const uint32_t tid = threadIdx.x;
  constexpr int U = 8;  // keys loaded per thread before the table operations

  for (uint32_t b = blockIdx.x; b < S.nb; b += gridDim.x) {
    for (uint32_t i = tid; i < (uint32_t)kJBuckets; i += kJoinThreads) { T.cnt[i] = 0u; T.fp[i] = 0ull; }
    for (uint32_t i = tid; i < (uint32_t)kHitWords; i += kJoinThreads) T.hitbits[i] = 0u;
    if (tid == 0) { T.nstash = 0; T.zb = 0; T.zhit = 0; T.ovf = 0; }
    const uint32_t gid = __ldg(S.gid + b);
    const uint32_t nbuild = min(S.fill[0][b], __ldg(S.cap[0] + b));
    const uint32_t nprobe = min(S.fill[1][b], __ldg(S.cap[1] + b));
    const unsigned long long *bk = S.scratch + __ldg(S.start[0] + b);
    const unsigned long long *pk = S.scratch + __ldg(S.start[1] + b);
    unsigned long long kv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // first build keys in flight across the clear
      const uint32_t i = u * kJoinThreads + tid;
      kv[u] = i < nbuild ? __ldcs(bk + i) : 0ull;
    }
    __syncthreads();
    for (uint32_t base = 0; base < nbuild; base += kJoinThreads * U) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (base + u * kJoinThreads + tid >= nbuild) continue;
        if (kv[u] == 0) { atomicAdd(&T.zb, 1u); continue; }
        join_insert(T, kv[u]);
      }
      const uint32_t nb2 = base + kJoinThreads * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = nb2 + u * kJoinThreads + tid;
        kv[u] = i < nbuild ? __ldcs(bk + i) : 0ull;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {  // first probe keys in flight across the barrier
      const uint32_t i = u * kJoinThreads + tid;
      kv[u] = i < nprobe ? __ldcs(pk + i) : 0ull;
    }
    __syncthreads();
    const uint32_t nstash = min(T.nstash, (uint32_t)kStash);
    const uint32_t zb = T.zb;
    if (T.ovf && tid == 0) atomicOr(S.batch_ovf + gid, 1u);
    unsigned long long hits = 0;
    for (uint32_t base = 0; base < nprobe; base += kJoinThreads * U) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned long long k = kv[u];
        if (base + u * kJoinThreads + tid >= nprobe) continue;
        if (k == 0) {
          if (zb) {
            hits += zb;
            if (atomicExch(&T.zhit, 1u) == 0u) {
              const unsigned long long h = atomicAdd(S.nhits, 1ull);
              if (h < S.hit_cap) S.hits[h] = HitRec{gid, 0u, 0ull};
            }
          }
          continue;
        }
        uint32_t first;
        const uint32_t c = join_count(T, k, nstash, first);
        if (c) {
          hits += c;
          if (!(atomicOr(T.hitbits + (first >> 5), 1u << (first & 31)) & (1u << (first & 31)))) {
            const unsigned long long h = atomicAdd(S.nhits, 1ull);
            if (h < S.hit_cap) S.hits[h] = HitRec{gid, 0u, k};
          }
        }
      }
      const uint32_t nb2 = base + kJoinThreads * U;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = nb2 + u * kJoinThreads + tid;
        kv[u] = i < nprobe ? __ldcs(pk + i) : 0ull;
      }
    }
    hits = warp_sum(hits);
    if ((tid & 31) == 0) T.bhits[tid >> 5] = hits;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < kJoinThreads / 32; ++w) t += T.bhits[w];
      if (t) atomicAdd(S.batch_hits + gid, t);
      S.fill[0][b] = 0;
      S.fill[1][b] = 0;
    }
    __syncthreads();
  }
}

template <int MC, bool ITEMS>
static cudaError_t launch_scatter_mi(const EnumArgs &a, const PartArgs &p, int grid, cudaStream_t st) {
  static bool configured = false;
  const size_t sm = scatter_smem_bytes();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_scatter<MC, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_scatter<MC, ITEMS><<<grid, kScatterWarps * 32, sm, st>>>(a, p);
  return cudaGetLastError();
}
template <int MC>
static cudaError_t launch_scatter_mc(const EnumArgs &a, const PartArgs &p, int grid, cudaStream_t st) {
  return a.items ? launch_scatter_mi<MC, true>(a, p, grid, st) : launch_scatter_mi<MC, false>(a, p, grid, st);
}

cudaError_t launch_scatter(int mc, const EnumArgs &args, const PartArgs &p, int num_sms, cudaStream_t st) {
  const uint64_t work = args.items ? args.item_hi - args.item_lo : args.nchunks;
  if (args.items ? args.item_hi <= args.item_lo : args.nchunks == 0) return cudaSuccess;
  const uint64_t blocks = (work + kScatterWarps - 1) / kScatterWarps;
  const int grid = (int)(blocks < (uint64_t)num_sms ? blocks : (uint64_t)num_sms);
  switch (mc) {
#define MSP_CASE(N) case N: return launch_scatter_mc<N>(args, p, grid, st);
    MSP_CASE(0) MSP_CASE(1) MSP_CASE(2) MSP_CASE(3) MSP_CASE(4) MSP_CASE(5) MSP_CASE(6) MSP_CASE(7)
    MSP_CASE(8) MSP_CASE(9) MSP_CASE(10) MSP_CASE(11) MSP_CASE(12) MSP_CASE(13) MSP_CASE(14)
    MSP_CASE(15)
#undef MSP_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rescatter(const RescatterArgs &r, const PartArgs &p, int num_sms, cudaStream_t st) {
  static bool configured = false;
  const size_t sm = scatter_smem_bytes();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_rescatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const uint64_t chunks = (r.total + kStage - 1) / kStage;
  if (!chunks) return cudaSuccess;
  const int grid = (int)(chunks < (uint64_t)num_sms ? chunks : (uint64_t)num_sms);
  k_rescatter<<<grid, kScatterWarps * 32, sm, st>>>(r, p);
  return cudaGetLastError();
}

cudaError_t launch_join(const PartArgs &p, int num_sms, cudaStream_t st) {
  static bool configured = false;
  const size_t sm = join_smem_bytes();
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_join, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (p.nb == 0) return cudaSuccess;
  const uint32_t grid = p.nb < (uint32_t)num_sms ? p.nb : (uint32_t)num_sms;
  k_join<<<grid, kJoinThreads, sm, st>>>(p);
  return cudaGetLastError();
}

}  // namespace msp
