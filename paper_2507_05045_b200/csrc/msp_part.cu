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
constexpr int kWarpStage = 448;                         // keys a warp stages per round
constexpr int kStage = kScatterWarps * kWarpStage;      // keys staged per CTA round
constexpr int kHistEntries = 2 * kMaxWaveBuckets;       // (role, bucket)
constexpr int kPer = kHistEntries / (kScatterWarps * 32);

// Reservation of n slots at *p, result left in flight in r (predicated: no-op when n == 0, so no
// select has to wait for the atomic's return value).
__device__ __forceinline__ void reserve_async(uint32_t &r, uint32_t *p, uint32_t n) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q atom.global.add.u32 %0, [%1], %2;\n\t}"
               : "+r"(r)
               : "l"(p), "r"(n)
               : "memory");
}

// Shared memory of a scatter CTA (k_scatter / k_rescatter); the producers' loop-vector buffers
// follow it (k_scatter only).
struct __align__(16) Stage {
  unsigned long long skey[kStage];   // staged keys (warp-private slot ranges)
  unsigned long long sorted[kStage]; // the round's keys sorted by (role, bucket)
  uint16_t sbkt[kStage], rank[kStage], sortb[kStage];
  uint32_t hist[kHistEntries];       // keys per entry in the round being filled
  uint32_t off[kHistEntries];        // sorted position of each entry's run
  uint32_t abase[kHistEntries];      // scratch index of sorted position 0 of the run, or kDrop
  uint32_t est[kHistEntries];        // scratch start of each entry's bucket region
  uint32_t ecap[kHistEntries];       // its capacity
  UnitInfo units[kMaxUnits];
  uint32_t warp_tot[kScatterWarps];
  uint32_t round_end;                // set by the first warp whose stage is full
};

size_t scatter_smem_bytes(int sw) { return sizeof(Stage) + (size_t)kScatterWarps * (kTQ + kU) * sw * 4; }

__device__ __forceinline__ void stage_init(Stage &g, const PartArgs &S, const UnitInfo *units, uint32_t nunits) {
  const uint32_t nbw = S.nb;
  for (uint32_t i = threadIdx.x; i < kHistEntries; i += blockDim.x) g.hist[i] = 0;
  for (uint32_t j = threadIdx.x; j < 2 * nbw; j += blockDim.x) {
    const uint32_t role = j >= nbw, b = j - role * nbw;
    g.est[j] = __ldg((role ? S.start[1] : S.start[0]) + b);
    g.ecap[j] = __ldg((role ? S.cap[1] : S.cap[0]) + b);
  }
  for (uint32_t u = threadIdx.x; u < nunits; u += blockDim.x) g.units[u] = units[u];
  if (threadIdx.x == 0) g.round_end = 0;
}

// Append one warp-step of keys densely to the warp's stage (ballot + popc) and rank each key
// within its (role, bucket) entry with one shared-memory atomic.
__device__ __forceinline__ void stage_key(Stage &g, uint32_t warp, uint32_t lane_lt, uint32_t &cnt,
                                          uint64_t key, uint32_t e, bool ok) {
  const uint32_t m = __ballot_sync(0xffffffffu, ok);
  if (ok) {
    const uint32_t pos = warp * kWarpStage + cnt + __popc(m & lane_lt);
    g.skey[pos] = key;
    g.sbkt[pos] = (uint16_t)e;
    g.rank[pos] = (uint16_t)atomicAdd(g.hist + e, 1u);
  }
  cnt += __popc(m);
}

// After a __syncthreads: scan the round's entry counts and reserve one scratch range per nonempty
// entry (global atomics, left in flight), sort each warp's staged keys into bucket-contiguous runs
// (hiding the atomics' latency), then turn the reservations into run bases and write the runs out
// coalesced.  The histogram is zeroed for the next fill.
__device__ __forceinline__ void flush_round(Stage &g, const PartArgs &S, uint32_t cnt) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nbw = S.nb, nent = 2 * nbw;
  const uint32_t j0 = tid * kPer;
  uint32_t hv[kPer], gres[kPer], local = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    hv[k] = j0 + k < nent ? g.hist[j0 + k] : 0u;
    g.hist[j0 + k] = 0u;  // ready for the next fill
    local += hv[k];
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t j = j0 + k, role = j >= nbw;
    gres[k] = 0u;
    reserve_async(gres[k], (role ? S.fill[1] : S.fill[0]) + (j - role * nbw), hv[k]);
  }
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) g.warp_tot[warp] = incl;
  __syncthreads();
  uint32_t run = incl - local, total = 0;
#pragma unroll
  for (int w = 0; w < kScatterWarps; ++w) {
    const uint32_t t = g.warp_tot[w];
    if ((uint32_t)w < warp) run += t;
    total += t;
  }
  uint32_t offs[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) { offs[k] = run; g.off[j0 + k] = run; run += hv[k]; }
  __syncthreads();
  for (uint32_t j = lane; j < cnt; j += 32) {  // each warp sorts its own staged keys
    const uint32_t i = warp * kWarpStage + j;
    const uint16_t b = g.sbkt[i];
    const uint32_t pos = g.off[b] + g.rank[i];
    g.sorted[pos] = g.skey[i];
    g.sortb[pos] = b;
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const uint32_t j = j0 + k;
    if (hv[k]) {
      if (gres[k] + hv[k] > g.ecap[j]) {  // overflow: the run goes to the sink, the batch is re-joined
        g.abase[j] = S.sink - offs[k];
        const uint32_t role = j >= nbw;
        atomicOr(S.batch_ovf + __ldg(S.gid + (j - role * nbw)), 1u);
      } else {
        g.abase[j] = g.est[j] + gres[k] - offs[k];
      }
    }
  }
  __syncthreads();
  for (uint32_t pos = tid; pos < total; pos += blockDim.x) S.scratch[g.abase[g.sortb[pos]] + pos] = g.sorted[pos];
}

// ---------------------------------------------------------------- tile descriptors

__global__ void k_tiles(const TileGenArgs a) {
  for (uint32_t r = a.rect_lo + blockIdx.x * blockDim.x + threadIdx.x; r < a.rect_hi; r += gridDim.x * blockDim.x) {
    const RectDesc R = a.rects[r];
    const uint32_t gs = R.gs();
    const uint32_t unit = a.gs_unit ? a.gs_unit[gs] : 0u;
    if (unit == 0xFFFFFFFFu) continue;
    TileDesc *out = a.out + (a.gs_tile_base ? a.gs_tile_base[gs] : 0ull) + R.tile_off;
    const uint32_t lx = R.lane_is_x() ? 1u : 0u;
    for (uint32_t lc = 0; lc < R.nl; ++lc) {
      const uint32_t ln = min(32u, R.L - lc * 32);
      for (uint32_t qc = 0; qc < R.nq; ++qc) {
        const uint32_t qn = min((uint32_t)kTQ, R.Q - qc * kTQ);
        TileDesc t;
        t.lane0 = R.lane_start + lc * 32;
        t.loop0 = R.loop_start + qc * kTQ;
        t.meta = unit | ((ln - 1) << 8) | ((qn - 1) << 13) | (lx << 18);
        t.pad = 0;
        *out++ = t;
      }
    }
  }
}

void launch_tiles(const TileGenArgs &a, cudaStream_t st) {
  const uint32_t n = a.rect_hi - a.rect_lo;
  if (!n) return;
  const uint32_t blocks = (n + 127) / 128;
  k_tiles<<<blocks < 1184 ? blocks : 1184, 128, 0, st>>>(a);
}

// ---------------------------------------------------------------- scatter (enumerate + hash + partition)

__device__ __forceinline__ uint4 ld_tile(const TileDesc *t, uint32_t i, uint32_t n) {
  return i < n ? __ldg(reinterpret_cast<const uint4 *>(t + i)) : make_uint4(0, 0, 0, 0);
}

// FNV fold step (validate.py:40-42) on (lo, hi) for v < 2^32: (h ^ v) * (2^40 + 435) mod 2^64.
__device__ __forceinline__ void fold(uint32_t &lo, uint32_t &hi, uint32_t v) {
  const uint32_t x = lo ^ v;
  hi = hi * 435u + __umulhi(x, 435u) + (x << 8);
  lo = x * 435u;
}

// Companion-vector loads of one tile for this lane: its lane entry and its (lane-th) loop entry.
template <int SW>
__device__ __forceinline__ void tile_vecs(const ScatterArgs &A, const Stage &g, const uint4 d, uint32_t lane,
                                          uint32_t (&lv)[SW], uint32_t (&yv)[SW]) {
  const uint32_t meta = d.z;
  const uint32_t side = (g.units[meta & 0xFFu].ent >> 16) & 1u;
  const bool lx = (meta >> 18) & 1u;
  const uint32_t ln = ((meta >> 8) & 31u) + 1u, qn = ((meta >> 13) & 31u) + 1u;
  const uint32_t *lt = side ? (lx ? A.comp[2] : A.comp[3]) : (lx ? A.comp[0] : A.comp[1]);
  const uint32_t *yt = side ? (lx ? A.comp[3] : A.comp[2]) : (lx ? A.comp[1] : A.comp[0]);
  load_vec<SW>(lt, d.x + min(lane, ln - 1u), lv);
  load_vec<SW>(yt, d.y + min(lane, qn - 1u), yv);
}

// kU keys of the current tile (loop entries q .. q+kU-1) into the stage.
template <int MC, bool RIGHT>
__device__ __forceinline__ void hash_step(Stage &g, const uint32_t *ybuf, const uint32_t (&lv)[stride_for(MC)],
                                          const uint32_t (&dg)[words_for(MC) > 0 ? words_for(MC) : 1],
                                          uint32_t warp, uint32_t lane_lt, uint32_t &cnt, uint32_t q, uint32_t qn,
                                          bool lok, const UnitInfo &ui, uint32_t diag,
                                          unsigned long long &filt, unsigned long long &dacc) {
  constexpr int SW = stride_for(MC), NW0 = words_for(MC), NW = NW0 > 0 ? NW0 : 1;
  const uint32_t ebase = ui.ent & 0xFFFu, bits = (ui.ent >> 12) & 0xFu;
  uint64_t key[kU];
  uint32_t e[kU];
  bool ok[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    uint32_t yv[SW];
    lds_vec<SW>(ybuf + (q + u) * SW, yv);  // ybuf holds kTQ + kU entries: reads past qn are padding
    uint32_t sv[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) sv[k] = lv[k] + yv[k];
    bool in = lok && q + u < qn;
    if (RIGHT) {
      uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < NW0; ++k) { sv[k] = dg[k] - sv[k]; acc &= sv[k]; }
      const bool fit = (acc & 0x80008000u) == 0x80008000u;
      filt += (in && !fit) ? 1u : 0u;
      in = in && fit;
    }
    uint32_t lo = ui.h0lo, hi = ui.h0hi;
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const uint32_t w = sv[c >> 1];
      fold(lo, hi, (c & 1) ? (w >> 16) & (RIGHT ? 0x7FFFu : 0xFFFFu) : w & (RIGHT ? 0x7FFFu : 0xFFFFu));
    }
    key[u] = ((uint64_t)hi << 32) | lo;
    ok[u] = in;
    e[u] = ebase + (uint32_t)(((uint64_t)hi << bits) >> 32);  // top `bits` bits of the key
  }
  if (diag) {
#pragma unroll
    for (int u = 0; u < kU; ++u) dacc ^= ok[u] ? key[u] : 0ull;
  } else {
#pragma unroll
    for (int u = 0; u < kU; ++u) stage_key(g, warp, lane_lt, cnt, key[u], e[u], ok[u]);
  }
}

// Enumerate + hash + partition the launch's tiles.  Each warp walks tiles warp, warp + W, ... with
// the descriptor two tiles ahead and the companion vectors one tile ahead in flight, so a tile
// change never waits on a load.  A full warp stage suspends the tile mid-way for a CTA round.
template <int MC>
__global__ void __launch_bounds__(kScatterWarps * 32, 1) k_scatter(const ScatterArgs A, const PartArgs S) {
  constexpr int SW = stride_for(MC), NW0 = words_for(MC), NW = NW0 > 0 ? NW0 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Stage &g = *reinterpret_cast<Stage *>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lane_lt = (1u << lane) - 1u;
  uint32_t *ybuf = reinterpret_cast<uint32_t *>(smem_raw + sizeof(Stage)) + warp * (kTQ + kU) * SW;
  stage_init(g, S, A.units, A.nunits);
  for (uint32_t i = lane; i < (uint32_t)((kTQ + kU) * SW); i += 32) ybuf[i] = 0;
  uint32_t dg[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) dg[k] = A.dpack[k];
  __syncthreads();

  const uint32_t nw = gridDim.x * kScatterWarps, n = A.ntiles;
  uint32_t t = blockIdx.x * kScatterWarps + warp;
  uint4 dcur = ld_tile(A.tiles, t, n), dnxt = ld_tile(A.tiles, t + nw, n), dnn = ld_tile(A.tiles, t + 2 * nw, n);
  uint32_t lvc[SW], yvc[SW], lvn[SW], yvn[SW];
  if (t < n) tile_vecs<SW>(A, g, dcur, lane, lvc, yvc);
  if (t + nw < n) tile_vecs<SW>(A, g, dnxt, lane, lvn, yvn);
  bool have = t < n;
  uint32_t q = 0, qn = 0, fgid = 0xFFFFFFFFu;
  bool lok = false, right = false;
  UnitInfo ui{};
  unsigned long long filt = 0, dacc = 0;
  auto begin_tile = [&]() {
    const uint32_t meta = dcur.z;
    ui = g.units[meta & 0xFFu];
    right = (ui.ent >> 16) & 1u;
    qn = ((meta >> 13) & 31u) + 1u;
    lok = lane <= ((meta >> 8) & 31u);
    q = 0;
    __syncwarp();
    if (lane < qn) {
#pragma unroll
      for (int k = 0; k < SW; ++k) ybuf[lane * SW + k] = yvc[k];
    }
    __syncwarp();
    if (ui.gid != fgid) {
      if (fgid != 0xFFFFFFFFu) {
        const unsigned long long f = warp_sum(filt);
        if (lane == 0 && f) atomicAdd(A.batch_filtered + fgid, f);
      }
      filt = 0;
      fgid = ui.gid;
    }
  };
  if (have) begin_tile();
  uint32_t cnt = 0;
  volatile uint32_t *round_end = &g.round_end;
  while (true) {
    // a round ends as soon as one warp's stage is full: the others stop within one step, so no
    // warp idles at the barrier while a slow one fills up
    while (have && !*round_end) {
      if (cnt + 32 * kU > (uint32_t)kWarpStage) { *round_end = 1u; break; }
      if (right)
        hash_step<MC, true>(g, ybuf, lvc, dg, warp, lane_lt, cnt, q, qn, lok, ui, A.diag, filt, dacc);
      else
        hash_step<MC, false>(g, ybuf, lvc, dg, warp, lane_lt, cnt, q, qn, lok, ui, A.diag, filt, dacc);
      q += kU;
      if (q >= qn) {  // next tile: everything it needs was loaded one (vectors) or two tiles ago
        t += nw;
        have = t < n;
        if (have) {
          dcur = dnxt;
#pragma unroll
          for (int k = 0; k < SW; ++k) { lvc[k] = lvn[k]; yvc[k] = yvn[k]; }
          dnxt = dnn;
          if (t + nw < n) tile_vecs<SW>(A, g, dnxt, lane, lvn, yvn);
          dnn = ld_tile(A.tiles, t + 2 * nw, n);
          begin_tile();
        }
      }
    }
    if (!__syncthreads_or(cnt > 0 || have)) break;
    if (tid == 0) *round_end = 0u;  // ordered before the next fill by the flush's barriers
    flush_round(g, S, cnt);
    cnt = 0;
  }
  if (fgid != 0xFFFFFFFFu) {
    const unsigned long long f = warp_sum(filt);
    if (lane == 0 && f) atomicAdd(A.batch_filtered + fgid, f);
  }
  if (dacc == 0x123456789ull) A.batch_filtered[0] = dacc;  // keep the diagnostic keys live
}

// Level 2 of the huge-batch path: stream already-hashed keys back from coarse bucket regions
// (HBM) and re-partition them into fine buckets (L2 scratch) for k_join.  Each CTA round takes
// kStage consecutive input slots; slots past a region's fill are empty.
__global__ void __launch_bounds__(kScatterWarps * 32) k_rescatter(const RescatterArgs R, const PartArgs S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Stage &g = *reinterpret_cast<Stage *>(smem_raw);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t nbw = S.nb;
  stage_init(g, S, nullptr, 0);
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
#pragma unroll 2
    for (int k = 0; k < kWarpStage / 32; ++k) {
      const uint64_t idx = base + (uint64_t)k * 32 + lane;
      uint32_t sl = s;
      while (sl + 1 < R.nsrc && idx >= R.src[sl + 1].in_base) ++sl;
      const RescatterSrc &src = R.src[sl];
      const uint64_t local = idx - src.in_base;
      const bool ok = idx < R.total && local < min(*src.fill, src.cap);
      const uint64_t key = ok ? __ldcs(src.keys + local) : 0ull;
      const uint32_t fb = src.fbits ? (uint32_t)((key << src.coarse_bits) >> (64 - src.fbits)) : 0u;
      stage_key(g, warp, lt_mask, cnt, key, src.role * nbw + src.fine_base + fb, ok);
    }
    __syncthreads();
    flush_round(g, S, cnt);
    __syncthreads();
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
  if (h.fp == 0) h.fp = 1;  // 0 marks an empty slot: a probe needs no slot counts
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
    reinterpret_cast<uint16_t *>(&T.fp[b])[s] = (uint16_t)h.fp;  // slot s is this thread's alone
  } else {
    const uint32_t i = atomicAdd(&T.nstash, 1u);
    if (i < (uint32_t)kStash) T.stash[i] = k; else T.ovf = 1u;
  }
}

// Multiplicity of k in the table; *first = slot id of its first copy (bucket-major, then stash).
// Fast path: two fingerprint words, one zero-lane test each (no slot counts, no loop).
__device__ __forceinline__ uint32_t join_count(const JoinSmem &T, unsigned long long k, uint32_t nstash,
                                               uint32_t &first) {
  constexpr unsigned long long kL = 0x0001000100010001ull, kH = 0x8000800080008000ull;
  const JoinHash h = join_hash(k);
  const unsigned long long w1 = T.fp[h.b1], w2 = T.fp[h.b2], pat = h.fp * kL;
  const unsigned long long x1 = w1 ^ pat, x2 = w2 ^ pat;
  uint32_t c = 0;
  first = 0xFFFFFFFFu;
  if ((((x1 - kL) & ~x1) | ((x2 - kL) & ~x2)) & kH) {  // some lane may hold fp: compare full keys
#pragma unroll
    for (int s = 0; s < 4; ++s)
      if (((w1 >> (16 * s)) & 0xFFFFu) == h.fp && T.key[h.b1][s] == k) { if (!c) first = h.b1 * 4 + s; ++c; }
#pragma unroll
    for (int s = 0; s < 4; ++s)
      if (((w2 >> (16 * s)) & 0xFFFFu) == h.fp && T.key[h.b2][s] == k) { if (!c) first = h.b2 * 4 + s; ++c; }
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

template <int MC>
static cudaError_t launch_scatter_mc(const ScatterArgs &a, const PartArgs &p, int grid, cudaStream_t st) {
  static bool configured = false;
  const size_t sm = scatter_smem_bytes(stride_for(MC));
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_scatter<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k_scatter<MC><<<grid, kScatterWarps * 32, sm, st>>>(a, p);
  return cudaGetLastError();
}

cudaError_t launch_scatter(int mc, const ScatterArgs &args, const PartArgs &p, int num_sms, cudaStream_t st) {
  if (args.ntiles == 0) return cudaSuccess;
  const uint32_t blocks = (args.ntiles + kScatterWarps - 1) / kScatterWarps;
  const int grid = (int)(blocks < (uint32_t)num_sms ? blocks : (uint32_t)num_sms);
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
  const size_t sm = sizeof(Stage);
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
