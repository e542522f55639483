// msp_part.cu -- K4/K5 as a radix-partitioned shared-memory hash join (the default join path).
//
// Same semantics as fastval._join_pairs (fastval.py:47-108): every left key is joined with every
// unfiltered right key of the same batch and all full-64-bit-hash-equal pairs are counted
// (hash_hits) and reported for exact confirmation.  Instead of bucket chains in DRAM, waves of
// batches are partitioned and joined:
//
//   scatter_chunk  enumerate + hash (msp_tile.cuh) a chunk of one batch side's tiles and partition
//                  the keys by bucket (top of the key) through a shared-memory stage in which a
//                  key's slot is its rank inside its bucket entry (no sort), flushing each round
//                  as one coalesced run per bucket into the wave's scratch.  Right pairs that
//                  overshoot d are counted, not written.
//   join_group     one CTA per bucket: insert the build side's keys (the smaller side of the batch)
//                  into a 16K-slot table in shared memory, stream the probe side's keys through
//                  it, count hash hits, record each hit key once for recovery.
//   k_waves        the persistent pipeline that runs both as tasks of one launch (one CTA per SM).
//
// The per-bucket capacity is sized from the exact batch counts (mean + 7 sigma); a bucket that
// overflows (duplicate-heavy instances) marks its batch, which the host re-joins with the global
// table path (msp_enum.cu), so results never depend on the partitioning.
#include <cstdint>
#include <algorithm>
#include <cstddef>
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>
#include "msp_common.cuh"
#include "msp_kernels.h"
#include "msp_tile.cuh"


namespace msp {

// Scatter CTA shape: kScatterCtas resident CTAs per SM, so one CTA's flush (reservation atomics +
// write-out) overlaps the other's enumeration.
constexpr int kScatterCtas = MSP_SCATTER_CTAS;
static_assert(kScatterCtas == kScatterCtasHost, "scatter CTAs per SM: msp_kernels.h and msp_part.cu disagree");
#ifndef MSP_SCATTER_WARPS
#define MSP_SCATTER_WARPS (16 / MSP_SCATTER_CTAS)
#endif
constexpr int kScatterWarps = MSP_SCATTER_WARPS;
constexpr int kScatterThreads = kScatterWarps * 32;
constexpr int kStageKeys = kScatterStageKeys;                   // stage slots of a CTA
constexpr int kMaxNB = kMaxUnitBuckets;                         // entries of one unit
#ifndef MSP_STAGE_FILL_PCT
#define MSP_STAGE_FILL_PCT 75
#endif
// (the huge-batch passes stage over ~500 coarse / fine entries, where a fuller stage spills more
// keys past C; each spill is a global atomic the warp -- and the next barrier -- waits on)
#ifndef MSP_L1STAGE_FILL_PCT
#define MSP_L1STAGE_FILL_PCT 62
#endif
#ifndef MSP_RSTAGE_FILL_PCT
#define MSP_RSTAGE_FILL_PCT 62
#endif
#ifndef MSP_RESCATTER_N
#define MSP_RESCATTER_N 4
#endif
#ifndef MSP_SCATTER_KEYS
#define MSP_SCATTER_KEYS 4
#endif
constexpr int kUS = MSP_SCATTER_KEYS;                           // keys per lane per scatter step

// Shared memory of a scatter CTA (k_scatter / k_rescatter / scatter tasks of k_waves).  A CTA works
// on one CHUNK at a time: consecutive tiles of ONE unit (one batch side), whose keys spread
// uniformly over the unit's NB bucket entries.  A round's keys are bucketed in place: entry j owns
// slots [j*C, j*C + C) (C even), C = kStageKeys / NB, and a key's slot is its rank within the
// entry (one shared atomic), so the round needs no sort.  The round ends once a lane has staged its
// share of MSP_STAGE_FILL_PCT % of the stage (no shared counter on the hot path); a key ranked past
// C -- rare at that fill -- goes straight to its bucket region (one global atomic).  The flush
// moves each entry's run to its bucket region with ONE bulk copy (cp.async.bulk, TMA): runs are
// padded to an even length with key 0 so both ends stay 16-byte aligned; real keys equal to 0 are
// never staged but counted per (batch, side) (zero_keys), and every reader skips key 0.
// The producers' loop-vector buffers follow the struct (scatter only).
#ifndef MSP_SPILL_LIST
#define MSP_SPILL_LIST 64
#endif
constexpr int kSpillList = MSP_SPILL_LIST;  // keys ranked past C parked in shared memory until the flush
struct SpillRec { unsigned long long key; uint32_t e, pad; };
struct __align__(16) Stage {
  unsigned long long key[kStageKeys];
  uint32_t cnt[kMaxNB + 32];         // keys ranked into each entry this round (> C: the rest spilled);
                                     // + one dummy counter per lane (never read)
  uint32_t round_end, chunk, tctr, nstaged;
  uint32_t nspill, sbase, spad[2];   // spills so far (monotonic) and at the round's start: this
                                     // round's list holds spills [sbase, nspill) (past kSpillList: global)
  SpillRec spill[kSpillList];
};

// Reservation of n slots at *p, result left in flight in r (predicated: no-op when n == 0, so no
// select has to wait for the atomic's return value).
__device__ __forceinline__ void reserve_async(uint32_t &r, uint32_t *p, uint32_t n) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q atom.global.add.u32 %0, [%1], %2;\n\t}"
               : "+r"(r)
               : "l"(p), "r"(n)
               : "memory");
}

size_t scatter_smem_bytes(int sw) { return sizeof(Stage) + (size_t)kScatterWarps * (kTQ + kUS) * sw * 4; }

__device__ __forceinline__ void stage_init(Stage &g) {
  for (uint32_t i = threadIdx.x; i < (uint32_t)kMaxNB; i += blockDim.x) g.cnt[i] = 0;
  if (threadIdx.x == 0) { g.round_end = 0; g.nstaged = 0; g.nspill = 0; g.sbase = 0; }
}

// The CTA's next work chunk (dynamic: one global atomic per chunk), broadcast through shared memory.
__device__ __forceinline__ uint32_t next_chunk(Stage &g, unsigned int *ctr) {
  if (threadIdx.x == 0) g.chunk = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t c = g.chunk;
  __syncthreads();
  return c;
}

// Role-indexed member of a 2-array by select (a runtime index into the argument struct's array would
// put the struct in local memory).
template <class T>
__device__ __forceinline__ T sel(T const (&a)[2], uint32_t role) { return role ? a[1] : a[0]; }

// A key ranked past its entry's C slots: straight to its bucket region (one global atomic, the key
// and a pad).
__device__ __forceinline__ void stage_spill(const PartArgs &S, uint32_t e, unsigned long long key) {
  const uint32_t role = e >= S.nb, b = e - role * S.nb;
  const uint32_t pos = atomicAdd(sel(S.fill, role) + b, 2u);  // (even: the regions stay 16-byte aligned)
  if (pos + 2 <= __ldg(sel(S.cap, role) + b)) {
    unsigned long long *p = S.scratch + __ldg(sel(S.start, role) + b) + pos;
    __stcg(p, key);
    __stcg(p + 1, 0ull);
  } else {
    atomicOr(S.batch_ovf + __ldg(S.gid + b), 1u);
  }
  if (S.dbg) atomicAdd(S.dbg + 13, 1ull);
}


// Stage N keys per lane into their entries j (local to the chunk's unit): rank (shared atomics,
// all issued before any dependent store), then store into the entry's slots; keys ranked past C
// (rare) are spilled in a separate, warp-uniform pass so the common path stays branch-free.
// `staged` counts this lane's keys of the round; at `budget` the lane ends the round for the CTA
// (lanes stage at similar rates, so the stage is then ~half full and keys ranked past C stay rare:
// an exact CTA-wide count to a fuller stage measured slower, its spills cost more than its rounds).
template <int N>
__device__ __forceinline__ void stage_keys(Stage &g, const PartArgs &S, uint32_t ebase, uint32_t C,
                                           uint32_t &staged, uint32_t budget,
                                           const unsigned long long (&key)[N], const uint32_t (&j)[N],
                                           const bool (&ok)[N]) {
  // every lane ranks every key (no predicated atomic, which would become a branch): a key that is
  // not staged ranks itself in the lane's own dummy counter past the entries instead
  const uint32_t dummy = kMaxNB + (threadIdx.x & 31);
  uint32_t r[N];
#pragma unroll
  for (int u = 0; u < N; ++u) r[u] = atomicAdd(&g.cnt[ok[u] ? j[u] : dummy], 1u);
  bool spill = false;
#pragma unroll
  for (int u = 0; u < N; ++u) {
    if (ok[u] && r[u] < C) g.key[j[u] * C + r[u]] = key[u];
    spill |= ok[u] && r[u] >= C;
    staged += ok[u] ? 1u : 0u;
  }
  if (__any_sync(0xffffffffu, spill)) {  // park them in the spill list (shared), flushed with the round
#pragma unroll
    for (int u = 0; u < N; ++u)
      if (ok[u] && r[u] >= C) {
        const uint32_t q = atomicAdd(&g.nspill, 1u) - g.sbase;
        if (q < (uint32_t)kSpillList) g.spill[q] = SpillRec{key[u], ebase + j[u], 0u};
        else stage_spill(S, ebase + j[u], key[u]);  // (list full: straight to the bucket region)
      }
  }
  if (staged >= budget) *(volatile uint32_t *)&g.round_end = 1u;
}

// Generic-proxy shared-memory writes (the staged keys) made visible to the async proxy (TMA).
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Bulk copy (TMA) of `bytes` (multiple of 16) from shared memory to global memory, 16-byte aligned
// ends; the issuing thread waits for it with bulk_wait_read() before the source is rewritten.
__device__ __forceinline__ void bulk_store(unsigned long long *dst, const unsigned long long *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst), "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// Every thread, before the CTA publishes a chunk's keys (task counter / kernel end): its bulk copies
// have fully completed (not just read the stage) and are ordered before its later generic accesses.
__device__ __forceinline__ void bulk_complete() {
  asm volatile("cp.async.bulk.wait_group 0;\n\tfence.proxy.async.global;" ::: "memory");
  __threadfence();
}

// Called by every thread after a barrier that ends the round (every thread fenced its staged
// writes for the async proxy before it): one lane per nonempty entry reserves the entry's run,
// padded to even length with key 0, in its bucket region (global atomics, all in flight at once)
// and moves it with one bulk copy; the issuing lanes wait until the copies have read the stage,
// then the stage is free again.  Ends with a barrier.
__device__ __forceinline__ void flush_round(Stage &g, const PartArgs &S, uint32_t ebase, uint32_t NB, uint32_t C) {
  const uint32_t tid = threadIdx.x;
  const uint32_t nb = S.nb;
  bool issued = false;
  for (uint32_t j = tid; j < NB; j += kScatterThreads) {
    uint32_t n = min(g.cnt[j], C);
    g.cnt[j] = 0u;
    if (!n) continue;
    const uint32_t e = ebase + j, role = e >= nb, b = e - role * nb;
    const uint32_t ne = (n + 1u) & ~1u;
    const uint32_t pos = atomicAdd(sel(S.fill, role) + b, ne);
    if (pos + ne <= __ldg(sel(S.cap, role) + b)) {
      unsigned long long *src = g.key + j * C;
      if (ne != n) { src[n] = 0ull; fence_proxy_async_smem(); }  // the pad (n odd => n < C)
      bulk_store(S.scratch + __ldg(sel(S.start, role) + b) + pos, src, ne * 8u);
      issued = true;
    } else {
      atomicOr(S.batch_ovf + __ldg(S.gid + b), 1u);
      if (S.dbg) atomicAdd(S.dbg + 12, 1ull);
    }
    if (S.dbg) atomicAdd(S.dbg + 1, (unsigned long long)n);
  }
  if (tid < 32) {  // warp 0 writes the round's parked spills and alone moves the list base
    const uint32_t nend = g.nspill, nsp = min(nend - g.sbase, (uint32_t)kSpillList);
    for (uint32_t i = tid; i < nsp; i += 32) stage_spill(S, g.spill[i].e, g.spill[i].key);
    __syncwarp();
    if (tid == 0) g.sbase = nend;
  }
  if (issued) {
    bulk_commit();
    bulk_wait_read();
  }
  if (S.dbg && tid == 0) atomicAdd(S.dbg + 0, 1ull);
  if (tid == 0) { g.round_end = 0u; g.nstaged = 0u; }
  __syncthreads();
}

// Stage slots per entry of a unit with NB buckets, and each lane's share of a round.
__device__ __forceinline__ void stage_geometry(uint32_t NB, uint32_t &C, uint32_t &budget,
                                               uint32_t fill_pct = MSP_STAGE_FILL_PCT) {
  C = (kStageKeys / NB) & ~1u;  // even: every entry's run starts 16-byte aligned
  budget = max(1u, NB * C * fill_pct / (100u * kScatterThreads));
}

// ---------------------------------------------------------------- tile descriptors

// A warp takes 32 rectangles at a time (one per lane: their descriptors load in parallel), scans
// their tile counts, and writes the group's tiles as one flat range: lane l writes tile t0 + l of the
// range, found in its rectangle by a 5-step search over the scanned counts.  Most rectangles hold
// one or two tiles, so a warp per rectangle left the lanes idle behind its dependent loads.
__global__ void k_tiles(const TileGenArgs a) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t n = a.rect_hi - a.rect_lo;
  for (uint32_t base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32u; base < n; base += nw * 32u) {
    uint32_t nt = 0, ls = 0, qs = 0, L = 0, Q = 0, nq = 1, w2 = 0;
    unsigned long long obase = 0;
    if (base + lane < n) {
      const RectDesc R = a.rects[a.rect_lo + base + lane];
      const uint32_t gs = R.gs();
      const uint32_t unit = a.gs_unit ? a.gs_unit[gs] : 0u;
      if (unit != 0xFFFFFFFFu) {
        nt = R.nl * R.nq;
        ls = R.lane_start; qs = R.loop_start; L = R.L; Q = R.Q; nq = R.nq;
        w2 = unit | ((R.lane_is_x() ? 1u : 0u) << 18);
        obase = (unsigned long long)(a.out + (a.gs_tile_base ? a.gs_tile_base[gs] : 0ull) + R.tile_off);
      }
    }
    uint32_t inc = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(~0u, inc, o);
      if (lane >= (uint32_t)o) inc += v;
    }
    const uint32_t total = __shfl_sync(~0u, inc, 31), exc = inc - nt;
    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
      const uint32_t t = t0 + lane;
      uint32_t k = 0;  // first lane whose inclusive count exceeds t
#pragma unroll
      for (uint32_t s = 16; s; s >>= 1) {
        const uint32_t v = __shfl_sync(~0u, inc, k + s - 1);
        if (v <= t) k += s;
      }
      const uint32_t kk = min(k, 31u);
      const uint32_t tl = t - __shfl_sync(~0u, exc, kk);
      const uint32_t knq = __shfl_sync(~0u, nq, kk), kls = __shfl_sync(~0u, ls, kk), kqs = __shfl_sync(~0u, qs, kk);
      const uint32_t kL = __shfl_sync(~0u, L, kk), kQ = __shfl_sync(~0u, Q, kk), kw2 = __shfl_sync(~0u, w2, kk);
      const unsigned long long ko = __shfl_sync(~0u, obase, kk);
      if (t < total) {
        const uint32_t lc = tl / knq, qc = tl - lc * knq;
        const uint32_t ln = min(32u, kL - lc * 32);
        const uint32_t qn = min((uint32_t)kTQ, kQ - qc * kTQ);
        const uint4 v = make_uint4(kls + lc * 32, kqs + qc * kTQ, kw2 | ((ln - 1) << 8) | ((qn - 1) << 13), 0u);
        *reinterpret_cast<uint4 *>(reinterpret_cast<TileDesc *>(ko) + tl) = v;
      }
    }
  }
}

// One warp per rectangle, lanes over its nl x nq warp tiles: for the few large rectangles of a huge
// batch side (~1000 tiles each), where 32 rectangles per warp would leave too few warps.
__global__ void k_tiles_wide(const TileGenArgs a) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wpg = gridDim.x * (blockDim.x >> 5);
  for (uint32_t r = a.rect_lo + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < a.rect_hi; r += wpg) {
    const RectDesc R = a.rects[r];
    const uint32_t gs = R.gs();
    const uint32_t unit = a.gs_unit ? a.gs_unit[gs] : 0u;
    if (unit == 0xFFFFFFFFu) continue;
    TileDesc *out = a.out + (a.gs_tile_base ? a.gs_tile_base[gs] : 0ull) + R.tile_off;
    const uint32_t w2 = unit | ((R.lane_is_x() ? 1u : 0u) << 18);
    const uint32_t nt = R.nl * R.nq;
    for (uint32_t t = lane; t < nt; t += 32) {
      const uint32_t lc = t / R.nq, qc = t - lc * R.nq;
      const uint32_t ln = min(32u, R.L - lc * 32);
      const uint32_t qn = min((uint32_t)kTQ, R.Q - qc * kTQ);
      const uint4 v = make_uint4(R.lane_start + lc * 32, R.loop_start + qc * kTQ, w2 | ((ln - 1) << 8) | ((qn - 1) << 13), 0u);
      *reinterpret_cast<uint4 *>(out + t) = v;
    }
  }
}

void launch_tiles(const TileGenArgs &a, cudaStream_t st) {
  const uint32_t n = a.rect_hi - a.rect_lo;
  if (!n) return;
  if (a.tiles > 8ull * n) {  // large rectangles: a warp each
    const uint32_t blocks = (n + 7) / 8;
    k_tiles_wide<<<blocks < 2368 ? blocks : 2368, 256, 0, st>>>(a);
    return;
  }
  const uint32_t blocks = (n + 255) / 256;  // 8 warps per block, 32 rectangles per warp
  k_tiles<<<blocks < 2368 ? blocks : 2368, 256, 0, st>>>(a);
}

// One block per batch: its buckets' region starts, capacities and batch id.
__global__ void k_expand_buckets(const BucketRun *runs, uint32_t nruns, uint32_t *out, uint32_t nbt) {
  for (uint32_t r = blockIdx.x; r < nruns; r += gridDim.x) {
    const BucketRun R = runs[r];
    for (uint32_t k = threadIdx.x; k < R.nb; k += blockDim.x) {
      const uint32_t b = R.b0 + k, s0 = R.base + k * (R.cb + R.cp);
      out[b] = s0;
      out[nbt + b] = s0 + R.cb;
      out[2 * nbt + b] = R.cb;
      out[3 * nbt + b] = R.cp;
      out[4 * nbt + b] = R.gid;
    }
  }
}

void launch_expand_buckets(const BucketRun *runs, uint32_t nruns, uint32_t *out, uint32_t nbt, cudaStream_t st) {
  if (!nruns) return;
  k_expand_buckets<<<nruns < 4096 ? nruns : 4096, 256, 0, st>>>(runs, nruns, out, nbt);
}

// ---------------------------------------------------------------- scatter (enumerate + hash + partition)

__device__ __forceinline__ uint4 ld_tile(const TileDesc *t, uint32_t i, uint32_t n) {
  return i < n ? __ldg(reinterpret_cast<const uint4 *>(t + i)) : make_uint4(0, 0, 0, 0);
}

// FNV fold step (validate.py:40-42) on (lo, hi) for v < 2^32: (h ^ v) * (2^40 + 435) mod 2^64.
// Written so that each state word has a two-instruction dependency chain per step: lo' = low(x *
// 435) after x = lo ^ v; hi' = hi * 435 + high(x * 435) + (x << 8), where hi * 435 does not wait
// for x and the shift is a byte permute (ALU pipe, not an IMAD the FMA pipe would also carry).
#ifndef MSP_FOLD_PTX
#define MSP_FOLD_PTX 0
#endif
__device__ __forceinline__ void fold(uint32_t &lo, uint32_t &hi, uint32_t v) {
#if MSP_FOLD_PTX == 2
  // LOP3 (x), IMAD.WIDE (x * 435), IMAD (hi * 435 + carry), LEA ((x << 8) + that): two FMA-pipe and
  // two ALU-pipe instructions per step (the plain C++ form compiles the shift-add to a third IMAD,
  // leaving the hash steps FMA-pipe bound)
  asm("{\n\t.reg .u32 x, u, s, c;\n\t.reg .u64 p;\n\t"
      "xor.b32 x, %0, %2;\n\t"
      "mul.wide.u32 p, x, 435;\n\t"
      "mov.b64 {%0, c}, p;\n\t"
      "mad.lo.u32 u, %1, 435, c;\n\t"
      "shl.b32 s, x, 8;\n\t"
      "add.u32 %1, u, s;\n\t}"
      : "+r"(lo), "+r"(hi) : "r"(v));
#elif MSP_FOLD_PTX
  asm("{\n\t.reg .u32 x, t1, t3, c;\n\t.reg .u64 p;\n\t"
      "xor.b32 x, %0, %2;\n\t"
      "mul.lo.u32 t1, %1, 435;\n\t"
      "mul.wide.u32 p, x, 435;\n\t"
      "prmt.b32 t3, x, 0, 0x2104;\n\t"
      "mov.b64 {%0, c}, p;\n\t"
      "add.u32 t1, t1, c;\n\t"
      "add.u32 %1, t1, t3;\n\t}"
      : "+r"(lo), "+r"(hi) : "r"(v));
#else
  const uint32_t x = lo ^ v;
  hi = hi * 435u + __umulhi(x, 435u) + (x << 8);
  lo = x * 435u;
#endif
}

// Companion-vector loads of one tile for this lane: its lane entry and its (lane-th) loop entry.
template <int SW>
__device__ __forceinline__ void tile_vecs(const ScatterArgs &A, uint32_t side, const uint4 d, uint32_t lane,
                                          uint32_t (&lv)[SW], uint32_t (&yv)[SW]) {
  const uint32_t meta = d.z;
  const bool lx = (meta >> 18) & 1u;
  const uint32_t ln = ((meta >> 8) & 31u) + 1u, qn = ((meta >> 13) & 31u) + 1u;
  const uint32_t *lt = side ? (lx ? A.comp[2] : A.comp[3]) : (lx ? A.comp[0] : A.comp[1]);
  const uint32_t *yt = side ? (lx ? A.comp[3] : A.comp[2]) : (lx ? A.comp[1] : A.comp[0]);
  load_vec<SW>(lt, d.x + min(lane, ln - 1u), lv);
  load_vec<SW>(yt, d.y + min(lane, qn - 1u), yv);
}

// kUS keys of the current tile (loop entries q .. q+kUS-1) into the stage.  (MC: the companion
// layout MCX of msp_common.cuh -- coordinate count plus kWide for P32.)
template <int MC, bool RIGHT>
__device__ __forceinline__ void hash_step(Stage &g, const PartArgs &S, const uint32_t *ybuf,
                                          const uint32_t (&lv)[stride_for(MC)],
                                          const uint32_t (&dg)[words_for(MC) > 0 ? words_for(MC) : 1],
                                          uint32_t C, uint32_t budget, uint32_t &staged, uint32_t q,
                                          uint32_t qn, bool lok, const UnitInfo &ui, uint32_t nbk, uint32_t diag,
                                          unsigned long long &filt, unsigned long long &dacc) {
  constexpr int SW = stride_for(MC), NW0 = words_for(MC), NW = NW0 > 0 ? NW0 : 1;
  unsigned long long key[kUS];
  uint32_t j[kUS];
  bool ok[kUS];
  uint32_t nzero = 0;
#pragma unroll
  for (int u = 0; u < kUS; ++u) {
    uint32_t yv[SW];
    lds_vec<SW>(ybuf + (q + u) * SW, yv);  // ybuf holds kTQ + kUS entries: reads past qn are padding
    uint32_t sv[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) sv[k] = lv[k] + yv[k];
    bool in = lok && q + u < qn;
    if (RIGHT) {
      uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < NW0; ++k) { sv[k] = dg[k] - sv[k]; acc &= sv[k]; }
      const bool fit = (acc & guard_mask(MC)) == guard_mask(MC);
      filt += (in && !fit) ? 1u : 0u;
      in = in && fit;
    }
    uint32_t lo = ui.h0lo, hi = ui.h0hi;
#pragma unroll
    for (int c = 0; c < mc_of(MC); ++c) fold(lo, hi, coord<MC, RIGHT>(sv, c));
    key[u] = ((unsigned long long)hi << 32) | lo;
    const bool z = in && (hi | lo) == 0u;  // a real key 0: counted per (batch, side), never staged
    nzero += z ? 1u : 0u;
    ok[u] = in && !z;
    j[u] = __umulhi(hi, nbk);  // bucket within the unit = floor(hi * NB / 2^32)
  }
  if (__any_sync(0xffffffffu, nzero != 0u) && nzero)
    atomicAdd(S.zero_keys + 2 * ui.gid + (RIGHT ? 1u : 0u), (unsigned long long)nzero);
  if (diag) {
#pragma unroll
    for (int u = 0; u < kUS; ++u) dacc ^= ok[u] ? key[u] : 0ull;
  } else {
    stage_keys<kUS>(g, S, ui.ent & 0x1FFFu, C, staged, budget, key, j, ok);
  }
}

// One work chunk: tiles [t0, n) of ONE unit (one batch side), enumerated + hashed + partitioned by
// the CTA.  Warps take their first two tiles statically and later ones from a shared counter (so
// they finish within one tile of each other), with the descriptor two tiles ahead and the
// companion vectors one tile ahead in flight.  A round ends for every warp as soon as some lane
// has staged its share (the CTA flushes, then resumes mid-tile) and at the end of the chunk.
// Filtered right pairs go to batch_filtered.  Ends with a barrier (the last flush).
template <int MC>
__device__ __forceinline__ void scatter_chunk(Stage &g, uint32_t *ybuf, const ScatterArgs &A, const PartArgs &S,
                                              const uint32_t (&dg)[words_for(MC) > 0 ? words_for(MC) : 1],
                                              const UnitInfo ui, uint32_t t0, uint32_t n, unsigned long long &dacc,
                                              uint32_t fill_pct = MSP_STAGE_FILL_PCT) {
  constexpr int SW = stride_for(MC);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  volatile uint32_t *round_end = &g.round_end;
  const uint32_t ebase = ui.ent & 0x1FFFu, nbk = (ui.ent >> 13) & 0x7FFu, side = (ui.ent >> 24) & 1u;
  const bool right = side != 0;
  uint32_t C, budget, staged = 0;
  stage_geometry(nbk, C, budget, fill_pct);
  if (tid == 0) g.tctr = 0;
  __syncthreads();
  auto grab = [&]() {
    uint32_t x = 0;
    if (lane == 0) x = atomicAdd(&g.tctr, 1u);
    return t0 + 2 * kScatterWarps + __shfl_sync(0xffffffffu, x, 0);
  };
  uint32_t t = t0 + warp, tn = t + kScatterWarps, tnn = grab();
  uint4 dcur = ld_tile(A.tiles, t, n), dnxt = ld_tile(A.tiles, tn, n), dnn = ld_tile(A.tiles, tnn, n);
  uint32_t lvc[SW], yvc[SW], lvn[SW], yvn[SW];
  if (t < n) tile_vecs<SW>(A, side, dcur, lane, lvc, yvc);
  if (tn < n) tile_vecs<SW>(A, side, dnxt, lane, lvn, yvn);
  bool have = t < n;
  uint32_t q = 0, qn = 0;
  bool lok = false;
  unsigned long long filt = 0;
  auto begin_tile = [&]() {
    const uint32_t meta = dcur.z;
    qn = ((meta >> 13) & 31u) + 1u;
    lok = lane <= ((meta >> 8) & 31u);
    q = 0;
    __syncwarp();
    if (lane < qn) {
#pragma unroll
      for (int k = 0; k < SW; ++k) ybuf[lane * SW + k] = yvc[k];
    }
    __syncwarp();
  };
  if (have) begin_tile();
  while (true) {
    while (have && !*round_end) {
      if (right)
        hash_step<MC, true>(g, S, ybuf, lvc, dg, C, budget, staged, q, qn, lok, ui, nbk, A.diag, filt, dacc);
      else
        hash_step<MC, false>(g, S, ybuf, lvc, dg, C, budget, staged, q, qn, lok, ui, nbk, A.diag, filt, dacc);
      q += kUS;
      if (q >= qn) {  // next tile: everything it needs was loaded one (vectors) or two tiles ago
        t = tn;
        tn = tnn;
        have = t < n;
        if (have) {
          dcur = dnxt;
#pragma unroll
          for (int k = 0; k < SW; ++k) { lvc[k] = lvn[k]; yvc[k] = yvn[k]; }
          dnxt = dnn;
          if (tn < n) tile_vecs<SW>(A, side, dnxt, lane, lvn, yvn);
          tnn = tn < n ? grab() : n;
          dnn = ld_tile(A.tiles, tnn, n);
          begin_tile();
        }
      }
    }
    fence_proxy_async_smem();  // the round's staged keys -> the flush's bulk copies
    const bool more = __syncthreads_or(have);
    flush_round(g, S, ebase, nbk, C);
    staged = 0;
    if (!more) break;
  }
  bulk_complete();
  if (right) {
    const unsigned long long f = warp_sum(filt);
    if (lane == 0 && f) atomicAdd(A.batch_filtered + ui.gid, f);
  }
}

// Enumerate + hash + partition one launch (the huge-batch level-1 pass, and the per-wave launch
// path used under MSP_FLAG_PROFILE): CTA b runs chunks [cta_first[b], cta_first[b+1]).
template <int MC>
__global__ void __launch_bounds__(kScatterThreads, kScatterCtas) k_scatter(const ScatterArgs A, const PartArgs S) {
  constexpr int SW = stride_for(MC), NW0 = words_for(MC), NW = NW0 > 0 ? NW0 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Stage &g = *reinterpret_cast<Stage *>(smem_raw);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *ybuf = reinterpret_cast<uint32_t *>(smem_raw + sizeof(Stage)) + warp * (kTQ + kUS) * SW;
  stage_init(g);
  for (uint32_t i = lane; i < (uint32_t)((kTQ + kUS) * SW); i += 32) ybuf[i] = 0;
  uint32_t dg[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) dg[k] = A.dpack[k];
  unsigned long long dacc = 0;
  __syncthreads();
  const uint32_t cend = __ldg(A.cta_first + blockIdx.x + 1);
  __shared__ int s_stop;
  for (uint32_t c = __ldg(A.cta_first + blockIdx.x); c < cend; ++c) {
    if (A.abort_dev) {  // stop (deadline / cancel): checked per chunk
      if (threadIdx.x == 0) s_stop = *(volatile int *)A.abort_dev;
      __syncthreads();
      if (s_stop) break;
    }
    const unsigned long long cw = __ldg(A.chunks + c);
    const uint32_t t0 = (uint32_t)cw, n = t0 + (uint32_t)((cw >> 32) & 0xFFFFu), unit = (uint32_t)(cw >> 48);
    scatter_chunk<MC>(g, ybuf, A, S, dg, A.units[unit], t0, n, dacc, MSP_L1STAGE_FILL_PCT);
  }
  if (dacc == 0x123456789ull) A.batch_filtered[0] = dacc;  // keep the diagnostic keys live
}

// Level 2 of the huge-batch path: stream already-hashed keys back from coarse bucket regions
// (HBM) and re-partition them into fine buckets (L2 scratch) for the join.  One work chunk: slots
// [s0, s1) of ONE source (a coarse region of one role, holding `fill` keys and run pads, which
// spread uniformly over its NF fine buckets), re-partitioned by the CTA.  Fine bucket = floor(frac *
// NF / 2^32), frac = the key's position inside its coarse bucket (the low word of hi * NC).  The
// keys arrive by TMA bulk copies in steps of kRStep keys through two shared buffers behind the
// stage (the next step always in flight), each step prefetched into L2 kRPrefetch steps earlier
// (cp.async.bulk.prefetch.L2), so a step copy waits on L2, not on HBM.
// Ends with a barrier.
#ifndef MSP_RSTEP
#define MSP_RSTEP 2048
#endif
#ifndef MSP_RFENCE_AT_END
#define MSP_RFENCE_AT_END 1
#endif
#ifndef MSP_RBUFS
#define MSP_RBUFS 2
#endif
constexpr uint32_t kRStep = MSP_RSTEP;            // keys per step
constexpr uint32_t kRBufs = MSP_RBUFS;            // step buffers behind the stage
#ifndef MSP_RPREFETCH
#define MSP_RPREFETCH 8
#endif
constexpr uint32_t kRPrefetch = MSP_RPREFETCH;    // steps prefetched into L2 (TMA prefetch) ahead of the step copies
constexpr int kRPerThread = (kRStep + kScatterThreads - 1) / kScatterThreads;
size_t rescatter_smem_bytes() { return sizeof(Stage) + (size_t)kRBufs * kRStep * 8; }

__device__ __forceinline__ void rescatter_chunk(Stage &g, const PartArgs &S, const RescatterSrc &src, uint32_t s0,
                                                uint32_t s1) {
  const uint32_t tid = threadIdx.x;
  const uint32_t ebase = src.role * S.nb + src.fine_base, NB = src.nf, nc = src.nc;
  uint32_t C, budget, staged = 0;
  stage_geometry(NB, C, budget, MSP_RSTAGE_FILL_PCT);
  unsigned long long *buf = reinterpret_cast<unsigned long long *>(&g + 1);  // kRBufs x kRStep keys
  __shared__ unsigned long long s_rbar[kRBufs];
  const uint32_t nstep = s1 > s0 ? (s1 - s0 + kRStep - 1) / kRStep : 0;
  auto prefetch = [&](uint32_t c) {  // thread 0: step c into L2 (TMA prefetch, no shared memory)
    if (kRPrefetch == 0 || c >= nstep) return;
    const uint32_t a = s0 + c * kRStep, n = min(s1 - a, kRStep);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src.keys + a), "r"(8u * ((n + 1u) & ~1u)) : "memory");
  };
  auto issue = [&](uint32_t c) {  // thread 0: step c into buffer c % kRBufs
    prefetch(c + kRPrefetch);
    const uint32_t a = s0 + c * kRStep, n = min(s1 - a, kRStep);
    fence_proxy_async_smem();
    const uint32_t bi = c % kRBufs;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&s_rbar[bi])), "r"(8u * ((n + 1u) & ~1u)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((uint32_t)__cvta_generic_to_shared(buf + bi * kRStep)), "l"(src.keys + a),
                    "r"(8u * ((n + 1u) & ~1u)), "r"((uint32_t)__cvta_generic_to_shared(&s_rbar[bi])) : "memory");
  };
  if (tid == 0) {
    for (uint32_t k = 0; k < kRBufs; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&s_rbar[k])) : "memory");
    for (uint32_t c = kRBufs; c < kRPrefetch; ++c) prefetch(c);
    for (uint32_t c = 0; c < kRBufs && c < nstep; ++c) issue(c);
  }
  __syncthreads();
  uint32_t phm = 0;  // bit k: the parity buffer k's barrier completes next
  for (uint32_t c = 0; c < nstep; ++c) {
    const uint32_t bsel = c % kRBufs;
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(&s_rbar[bsel])), "r"((phm >> bsel) & 1u) : "memory");
    phm ^= 1u << bsel;
    const uint32_t n = min(s1 - (s0 + c * kRStep), kRStep);
    const unsigned long long *bk = buf + bsel * kRStep;
    unsigned long long key[kRPerThread];
    uint32_t j[kRPerThread];
    bool ok[kRPerThread];
#pragma unroll
    for (int u = 0; u < kRPerThread; ++u) {
      const uint32_t i = tid + u * kScatterThreads;
      key[u] = bk[min(i, kRStep - 1)];
      ok[u] = i < n && key[u] != 0ull;  // (0: a run pad)
      j[u] = __umulhi((uint32_t)(key[u] >> 32) * nc, NB);
    }
    stage_keys<kRPerThread>(g, S, ebase, C, staged, budget, key, j, ok);
    if (!MSP_RFENCE_AT_END) fence_proxy_async_smem();  // (the staged keys -> a flush's bulk copies)
    const bool end = __syncthreads_or(g.round_end != 0u) || c + 1 == nstep;  // (the buffer is free)
    if (tid == 0 && c + kRBufs < nstep) issue(c + kRBufs);
    if (end) {
      if (MSP_RFENCE_AT_END) {  // the proxy fence once per round, not per step
        fence_proxy_async_smem();
        __syncthreads();
      }
      flush_round(g, S, ebase, NB, C);
      staged = 0;
    }
  }
  if (tid == 0)
    for (uint32_t k = 0; k < kRBufs; ++k)
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&s_rbar[k])) : "memory");
  bulk_complete();
  __syncthreads();
}

// Level 2 of the huge-batch path as its own launch (MSP_FLAG_WAVE_LAUNCHES): stream already-hashed
// keys back from coarse bucket regions (HBM) and re-partition them into fine buckets (L2 scratch)
// for k_join; chunks from a global counter.
__global__ void __launch_bounds__(kScatterThreads, kScatterCtas) k_rescatter(const RescatterArgs R, const PartArgs S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Stage &g = *reinterpret_cast<Stage *>(smem_raw);
  stage_init(g);
  __syncthreads();
  for (uint32_t c = next_chunk(g, R.chunk_ctr); c < R.nchunks; c = next_chunk(g, R.chunk_ctr)) {
    const unsigned long long cw = __ldg(R.chunks + c);
    const RescatterSrc &src = R.src[(uint32_t)(cw >> 48)];
    const uint32_t s0 = (uint32_t)cw, s1 = min(s0 + (uint32_t)((cw >> 32) & 0xFFFFu) * 32u, min(*src.fill, src.cap));
    rescatter_chunk(g, S, src, s0, s1);
  }
}

constexpr int kJoinThreads = 1024;
constexpr int kJoinSlots = 1 << kJoinSlotsLog2;        // 16K table slots
constexpr int kJWays = 8;                               // slots per table bucket
constexpr int kJBuckets = kJoinSlots / kJWays;          // 2K buckets of 8 slots
constexpr int kStash = 256;                             // keys whose two buckets were both full
constexpr int kHitWords = (kJoinSlots + kStash) / 32;
constexpr int kJQueue = 512;                            // deferred probes (per-warp segments)
#ifndef MSP_JOIN_CHUNK
#define MSP_JOIN_CHUNK 4000
#endif
constexpr int kJChunk = MSP_JOIN_CHUNK;                 // keys per streamed chunk (two buffers)
static_assert(kJChunk % 2 == 0, "chunks start 16-byte aligned");

// Shared-memory join of one partition bucket.  The table has 8-slot buckets, first fit in bucket
// b1, then b2, then a small stash; a slot holds the full 64-bit key and a fingerprint byte 0x80 | 7
// key bits (0 = empty; the eight of a bucket are one 64-bit word).  An insert is one shared atomic
// + two stores; a probe reads ONE fingerprint word and tests all eight bytes at once (branch-free);
// the few probes whose test does not rule a match out are queued in the warp's segment and counted
// exactly later (full keys, in shared memory).  A key sits in b2 only if b1 was full (slot 7's
// marker bit, the word's sign bit).  b1/b2 come from a multiplicative mix of the key's low word, the
// fingerprint from its high word (whose top bits chose the partition bucket).
// Keys arrive by TMA bulk copies (cp.async.bulk + mbarrier) as ONE stream of chunks through two
// buffers: each bucket's build chunks then its probe chunks, the next chunk always in flight while
// the current one is processed -- across bucket boundaries too.
struct JoinSmem {
  unsigned long long key[kJBuckets][kJWays];
  unsigned long long fp[kJBuckets];     // eight fingerprint bytes
  uint32_t cnt[kJBuckets];              // claims (may exceed 8: failed claims move on)
  unsigned long long stash[kStash];
  uint32_t hitbits[kHitWords];
  unsigned long long queue[kJQueue];    // per-warp segments of deferred probes
  unsigned long long bhits[kJoinThreads / 32];
  unsigned long long mbar[2];           // one per chunk buffer
  uint32_t nstash, ovf, pad[2];
  alignas(16) unsigned long long buf[2][kJChunk + 64];  // (bulk-copy destinations: 16-byte aligned;
                                                          // +64: unrolled warps read past a chunk's end)
};
static_assert(offsetof(JoinSmem, buf) % 16 == 0, "bulk copy alignment");

size_t join_smem_bytes() { return sizeof(JoinSmem); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long *b) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" :: "r"(smem_u32(b)) : "memory");
}
// Thread 0: expect `bytes` on barrier b and copy them from global src to shared dst (one bulk copy,
// 16-byte aligned ends).
__device__ __forceinline__ void bulk_load(unsigned long long *dst, const unsigned long long *src, uint32_t bytes,
                                          unsigned long long *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// Every thread: wait for the completion of phase `parity` of barrier b.
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
}

__device__ __forceinline__ uint32_t jmix(unsigned long long k) { return (uint32_t)k * 0x9E3779B1u; }
__device__ __forceinline__ uint32_t jb1(uint32_t t) { return t >> 21; }
__device__ __forceinline__ uint32_t jb2(uint32_t t) { return (t >> 21) ^ (((t >> 10) & (kJBuckets - 1)) | 1u); }
// fingerprint byte replicated into all four bytes of a word
__device__ __forceinline__ uint32_t jfp4(unsigned long long k) {
  return __byte_perm((uint32_t)(k >> 32), 0u, 0x1111u) | 0x80808080u;
}
// 0x80 in exactly the bytes of x that are zero (exact per byte; the halves are independent).
__device__ __forceinline__ uint32_t zero_byte_mask32(uint32_t x) {
  return ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);
}
// Some byte of x is zero (exact for presence).
__device__ __forceinline__ uint32_t has_zero_byte(uint32_t x) { return (x - 0x01010101u) & ~x & 0x80808080u; }
// 64-bit load from a 32-bit shared-window address (keeps the compiler from re-deriving the
// window base from a generic pointer on every access in the join's inner loops)
__device__ __forceinline__ unsigned long long lds64(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void join_insert(JoinSmem &T, unsigned long long k) {
  const uint32_t t = jmix(k), fpb = jfp4(k) & 0xFFu;
  uint32_t b = jb1(t), s = atomicAdd(&T.cnt[b], 1u);
  if (s >= (uint32_t)kJWays) { b = jb2(t); s = atomicAdd(&T.cnt[b], 1u); }
  if (s < (uint32_t)kJWays) {
    T.key[b][s] = k;
    reinterpret_cast<uint8_t *>(&T.fp[b])[s] = (uint8_t)fpb;  // slot s is this thread's alone
  } else {
    const uint32_t q = atomicAdd(&T.nstash, 1u);
    if (q < (uint32_t)kStash) T.stash[q] = k; else T.ovf = 1u;
  }
}

// Copies of k among the slots of bucket b whose fingerprint byte matches.
__device__ __forceinline__ void count_in_bucket(const JoinSmem &T, uint32_t b, unsigned long long w, uint32_t pat,
                                                unsigned long long k, uint32_t &c, uint32_t &first) {
  unsigned long long m = ((unsigned long long)zero_byte_mask32((uint32_t)(w >> 32) ^ pat) << 32) |
                         zero_byte_mask32((uint32_t)w ^ pat);
  while (m) {
    const uint32_t s = (uint32_t)(__ffsll((long long)m) - 1) >> 3;
    if (T.key[b][s] == k) {
      if (!c) first = b * kJWays + s;
      ++c;
    }
    m &= m - 1;
  }
}

// Multiplicity of k among the build keys (b1, b2 if b1 is full, the stash if b2 is full too);
// `first` = slot id of its first copy.
__device__ __forceinline__ uint32_t join_count_slow(const JoinSmem &T, unsigned long long k, uint32_t nstash,
                                                    uint32_t &first) {
  const uint32_t t = jmix(k), b1 = jb1(t), pat = jfp4(k);
  const unsigned long long w1 = T.fp[b1];
  first = 0xFFFFFFFFu;
  uint32_t c = 0;
  count_in_bucket(T, b1, w1, pat, k, c, first);
  if ((long long)w1 < 0) {  // b1 full: k may have moved on to b2 (and, if b2 is full too, the stash)
    const uint32_t b2 = jb2(t);
    const unsigned long long w2 = T.fp[b2];
    count_in_bucket(T, b2, w2, pat, k, c, first);
    if ((long long)w2 < 0)
      for (uint32_t i = 0; i < nstash; ++i)
        if (T.stash[i] == k) { if (!c) first = kJoinSlots + i; ++c; }
  }
  return c;
}

// The chunk stream of a join task: for each bucket, its build chunks then its probe chunks.
struct ChunkCursor {
  uint32_t b, c, nbc, npc;  // bucket, chunk within the bucket, build / probe chunks of the bucket
};

// Join of buckets [b0, b1) of a wave by one CTA of NT threads (fastval.py:75-107 semantics: every
// full-64-bit-hash-equal (build, probe) pair is a hit; each hit key is recorded once for the exact
// confirmation), resetting each bucket's fill counters for the next use of the scratch buffer.  The
// regions hold min(fill, cap) keys, run pads (key 0) among them (fill > cap flagged the batch).
// Ends with a barrier.
#ifndef MSP_JOIN_INLINE
#define MSP_JOIN_INLINE __forceinline__
#endif
template <int NT>
__device__ MSP_JOIN_INLINE void join_group(JoinSmem &T, const PartArgs &S, uint32_t b0, uint32_t b1) {
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  auto nbuild_of = [&](uint32_t b) { return min(S.fill[0][b], __ldg(S.cap[0] + b)); };
  auto nprobe_of = [&](uint32_t b) { return min(S.fill[1][b], __ldg(S.cap[1] + b)); };
  // thread 0: issue chunk `cur` of the stream into buffer `bf` (and advance the issue cursor)
  auto issue = [&](ChunkCursor &ic, uint32_t bf) {
    while (ic.b < b1 && ic.c >= ic.nbc + ic.npc) {
      if (++ic.b >= b1) return;
      ic.c = 0;
      ic.nbc = (nbuild_of(ic.b) + kJChunk - 1) / kJChunk;
      ic.npc = (nprobe_of(ic.b) + kJChunk - 1) / kJChunk;
    }
    if (ic.b >= b1) return;
    const bool build = ic.c < ic.nbc;
    const uint32_t n = build ? nbuild_of(ic.b) : nprobe_of(ic.b);
    const uint32_t c0 = (build ? ic.c : ic.c - ic.nbc) * kJChunk;
    const uint32_t len = min(n - c0, (uint32_t)kJChunk);
    const unsigned long long *src = S.scratch + __ldg((build ? S.start[0] : S.start[1]) + ic.b) + c0;
    fence_proxy_async_smem();  // (generic accesses of the buffer before -> async write)
    bulk_load(T.buf[bf], src, 8u * ((len + 1u) & ~1u), &T.mbar[bf]);  // (odd: one slot past, < cap)
    ++ic.c;
  };
  if (tid == 0) { mbar_init(&T.mbar[0]); mbar_init(&T.mbar[1]); }
  __syncthreads();
  ChunkCursor ic{b0, 0, (nbuild_of(b0) + kJChunk - 1) / kJChunk, (nprobe_of(b0) + kJChunk - 1) / kJChunk};
  if (tid == 0) { issue(ic, 0); issue(ic, 1); }
  uint32_t k_chunk = 0;           // stream position of the next chunk to process (buffer k & 1)
  uint32_t ph0 = 0, ph1 = 0;      // barrier phases (every thread tracks them alike)
  constexpr uint32_t kQW = kJQueue / (NT / 32);
  unsigned long long *qw = T.queue + (tid >> 5) * kQW;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t b = b0; b < b1; ++b) {
    long long tp0 = 0, tp1 = 0, tp2 = 0;
    if (S.dbg && tid == 0) tp0 = clock64();
    const uint32_t gid = __ldg(S.gid + b);
    const uint32_t nbuild = nbuild_of(b), nprobe = nprobe_of(b);
    const uint32_t nbc = (nbuild + kJChunk - 1) / kJChunk, npc = (nprobe + kJChunk - 1) / kJChunk;
    for (uint32_t i = tid; i < (uint32_t)kJBuckets / 4; i += NT) reinterpret_cast<uint4 *>(T.cnt)[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t i = tid; i < (uint32_t)kJBuckets / 2; i += NT) reinterpret_cast<uint4 *>(T.fp)[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t i = tid; i < (uint32_t)kHitWords; i += NT) T.hitbits[i] = 0u;
    if (tid == 0) { T.nstash = 0; T.ovf = 0; }
    __syncthreads();
    uint32_t hits = 0, nqw = 0, nstash = 0;  // (nqw: warp-uniform)
    auto probe_slow = [&](unsigned long long k) {  // a possible hit: count it, record the key once
      uint32_t first;
      const uint32_t c = join_count_slow(T, k, nstash, first);
      if (c) {
        hits += c;
        if (!(atomicOr(T.hitbits + (first >> 5), 1u << (first & 31)) & (1u << (first & 31)))) {
          const unsigned long long h = atomicAdd(S.nhits, 1ull);
          if (h < S.hit_cap) S.hits[h] = HitRec{gid, 0u, k};
        }
      }
    };
    for (uint32_t c = 0; c < nbc + npc; ++c, ++k_chunk) {
      const uint32_t bf = k_chunk & 1u;
      mbar_wait(&T.mbar[bf], bf ? ph1 : ph0);
      if (bf) ph1 ^= 1u; else ph0 ^= 1u;
      const unsigned long long *ck = T.buf[bf];
      const uint32_t cks = smem_u32(ck);
      if (c < nbc) {  // ---- build chunk: insert (two keys per thread per step)
        const uint32_t n = min(nbuild - c * kJChunk, (uint32_t)kJChunk);
        for (uint32_t i = tid; i < n; i += 2 * NT) {
          const unsigned long long k0 = lds64(cks + 8u * i), k1 = lds64(cks + 8u * min(i + NT, (uint32_t)kJChunk));
          if (k0 != 0ull) join_insert(T, k0);  // (0: a run pad)
          if (k1 != 0ull && i + NT < n) join_insert(T, k1);
        }
        __syncthreads();  // buffer released; after the last build chunk the table is complete
        if (c + 1 == nbc) {
          nstash = min(T.nstash, (uint32_t)kStash);
          if (T.ovf && tid == 0) { atomicOr(S.batch_ovf + gid, 1u); if (S.dbg) atomicAdd(S.dbg + 14, 1ull); }
          if (S.dbg && tid == 0) tp1 = clock64();
        }
      } else {        // ---- probe chunk: fast test, branch-free; possible hits to the warp's queue
        const uint32_t n = min(nprobe - (c - nbc) * kJChunk, (uint32_t)kJChunk);
        const uint32_t fps = smem_u32(T.fp);
        for (uint32_t i = tid; i - lane < n; i += NT) {  // (whole warps iterate: the exit is warp-uniform)
          // (a pad -- key 0 -- may be probed: pads are never inserted and real zero keys never reach
          // the scratch, so its count is 0)
          const unsigned long long k = lds64(cks + 8u * i);
          const uint32_t pat = jfp4(k);
          const unsigned long long w = lds64(fps + 8u * jb1(jmix(k)));
          const bool maybe = ((has_zero_byte((uint32_t)w ^ pat) | has_zero_byte((uint32_t)(w >> 32) ^ pat)) != 0u ||
                              (long long)w < 0) && i < n;
          const uint32_t mm = __ballot_sync(0xffffffffu, maybe);
          if (nqw + __popc(mm) > kQW) {  // the warp's segment is full: count its queued probes now
            for (uint32_t q = lane; q < nqw; q += 32) probe_slow(qw[q]);
            nqw = 0;
            __syncwarp();
          }
          if (maybe) qw[nqw + __popc(mm & lt)] = k;
          nqw += __popc(mm);
        }
        __syncthreads();  // buffer released
      }
      if (tid == 0) issue(ic, bf);  // the chunk after next into the released buffer
    }
    if (nbc == 0 && S.dbg && tid == 0) tp1 = clock64();
    for (uint32_t q = lane; q < nqw; q += 32) probe_slow(qw[q]);
    const unsigned long long wh = warp_sum((unsigned long long)hits);
    if (lane == 0) T.bhits[tid >> 5] = wh;
    __syncthreads();
    if (S.dbg && tid == 0) {
      tp2 = clock64();
      atomicAdd(S.dbg + 8, (unsigned long long)(tp1 - tp0));
      atomicAdd(S.dbg + 9, (unsigned long long)(tp2 - tp1));
      atomicAdd(S.dbg + 10, (unsigned long long)nstash);
      atomicAdd(S.dbg + 11, 1ull);
    }
    if (tid == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < NT / 32; ++w) t += T.bhits[w];
      if (t) atomicAdd(S.batch_hits + gid, t);
      S.fill[0][b] = 0;
      S.fill[1][b] = 0;
    }
  }
  __syncthreads();
  if (tid == 0) { mbar_inval(&T.mbar[0]); mbar_inval(&T.mbar[1]); }
  __syncthreads();
}

__global__ void __launch_bounds__(kJoinThreads, 1) k_join(const PartArgs S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JoinSmem &T = *reinterpret_cast<JoinSmem *>(smem_raw);
  for (uint32_t b = blockIdx.x; b < S.nb; b += gridDim.x) join_group<kJoinThreads>(T, S, b, b + 1);
}

// ---------------------------------------------------------------- persistent wave pipeline

// All partitioned waves of a solve in ONE launch, one CTA per SM: CTAs pull tasks in queue order
// S(0) S(1) S(2) J(0) S(3) J(1) ... where S(w) are wave w's scatter chunks and J(w) its join bucket
// groups, ordered S(w + 2) before J(w).  J(w) waits for every chunk of S(w) (scat_done[w]); S(w)
// waits for J(w-4) (join_done), the last reader of its scratch buffer w % 4 (four buffers, so S(w)
// never waits on the joins handed out just before it).  Every wait points at tasks earlier in the queue,
// already held by resident CTAs, so the pipeline cannot deadlock; joins of wave w run on some SMs
// while others scatter wave w + 1, and no wave ends in a launch tail.
template <int MC>
__global__ void __launch_bounds__(kScatterThreads, 1) k_waves(const WavesArgs W) {
  constexpr int SW = stride_for(MC), NW0 = words_for(MC), NW = NW0 > 0 ? NW0 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Stage &g = *reinterpret_cast<Stage *>(smem_raw);
  JoinSmem &T = *reinterpret_cast<JoinSmem *>(smem_raw);  // (union with the stage)
  __shared__ unsigned long long s_task;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t *ybuf = reinterpret_cast<uint32_t *>(smem_raw + sizeof(Stage)) + warp * (kTQ + kUS) * SW;
  for (uint32_t i = lane; i < (uint32_t)((kTQ + kUS) * SW); i += 32) ybuf[i] = 0;
  uint32_t dg[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) dg[k] = W.sc.dpack[k];
  unsigned long long dacc = 0;
  long long t_prev = clock64();
  // Thread 0 fetches the NEXT task at each switch: queue index (atomic), task word, then its wave
  // descriptor, chunk word (the task word holds the chunk's global index, so both load in parallel),
  // dependency target and the stop word, handed over through shared memory at the following switch.
  // (Deeper lookahead -- tasks reserved two or three ahead, every load off the switch's critical
  // path -- measured slower: reserved-but-unstarted scatter chunks delay the joins that wait on them.)
  struct Next { unsigned long long tk, cw; WaveDesc wd; uint32_t need; const unsigned int *ctr; int stop; };
  __shared__ unsigned long long s_cw;
  __shared__ WaveDesc s_wd;
  auto task_word = [&](uint32_t i) -> unsigned long long { return i < W.ntasks ? W.tasks[i] : ~0ull; };
  auto fetch = [&](unsigned long long tk, Next &x) {
    // the stop word (device memory, set by the host watchdog's copy): read a task ahead, so its
    // latency overlaps the current task
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(x.stop) : "l"(W.abort_dev));
    x.tk = tk;
    x.ctr = nullptr;
    x.need = 0;
    x.cw = 0;
    if (tk == ~0ull) return;
    const uint32_t w = (uint32_t)(tk >> 32) & 0x7FFFFFFFu;
    x.wd = W.waves[w];
    if (tk >> 63) {
      x.ctr = W.scat_done + w;
      x.need = W.waves[w].nchunks;
    } else {
      x.cw = __ldg(W.chunks + (uint32_t)tk);
      if (w >= kWaveBuffers) {  // the last wave on this scratch buffer must be fully joined
        x.ctr = W.join_done + w - kWaveBuffers;
        x.need = W.waves[w - kWaveBuffers].njoin;
      }
    }
  };
  Next nc;
  uint32_t na = 0;  // (fetch_ahead: the queue index of the task after next, reserved a task early)
  if (tid == 0) {
    fetch(task_word(atomicAdd(W.task_ctr, 1u)), nc);
    if (W.fetch_ahead) na = atomicAdd(W.task_ctr, 1u);
  }
  while (true) {
    if (tid == 0) {
      const Next cur = nc;
      if (cur.tk != ~0ull) {
        if (W.fetch_ahead) {
          fetch(task_word(na), nc);
          na = atomicAdd(W.task_ctr, 1u);
        } else {
          fetch(task_word(atomicAdd(W.task_ctr, 1u)), nc);
        }
      }
      // stop (deadline / cancel, MSP_OPTIONS): every CTA leaves at its next task switch, waits included
      bool stop = cur.stop != 0;
      if (cur.ctr && !stop) {
        const long long tw = clock64();
        uint32_t v;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cur.ctr) : "memory");
          if (v >= cur.need) break;
          if (*(volatile int *)W.abort_dev) { stop = true; break; }
          __nanosleep(256);
        }
        if (W.pa.dbg) atomicAdd(W.pa.dbg + ((cur.tk >> 63) ? 6 : 7), (unsigned long long)(clock64() - tw));
      }
      s_task = stop ? ~0ull : cur.tk;
      s_cw = cur.cw;
      s_wd = cur.wd;
    }
    __syncthreads();
    const unsigned long long tk = s_task;
    if (tk == ~0ull) break;
    const uint32_t w = (uint32_t)(tk >> 32) & 0x7FFFFFFFu, idx = (uint32_t)tk;
    const WaveDesc wd = s_wd;
    PartArgs S = W.pa;
    const uint32_t buf = w % kWaveBuffers;
    S.scratch = W.scratch + buf * W.scratch_stride;
    S.fill[0] = W.fill + buf * (2 * kMaxWaveBuckets);
    S.fill[1] = S.fill[0] + kMaxWaveBuckets;
    S.start[0] = W.bstart0 + wd.b0;
    S.start[1] = W.bstart1 + wd.b0;
    S.cap[0] = W.bcap0 + wd.b0;
    S.cap[1] = W.bcap1 + wd.b0;
    S.gid = W.bgid + wd.b0;
    S.nb = wd.nb;
    S.roles = 2;
    if (tk >> 63) {  // join: buckets [idx, idx + kJoinGroup) of the wave
      const uint32_t b1 = min(idx + (uint32_t)kJoinGroup, wd.nb);
      join_group<kScatterThreads>(T, S, idx, b1);  // (ends with a barrier: the CTA's writes are ordered before the release)
      if (tid == 0) { __threadfence(); atomicAdd(W.join_done + w, 1u); }
      if (tid == 0 && W.pa.dbg) { const long long now = clock64(); atomicAdd(W.pa.dbg + 5, (unsigned long long)(now - t_prev)); t_prev = now; }
    } else {  // scatter chunk idx of the wave (tiles, or a level-2 slot range of a coarse region)
      stage_init(g);
      __syncthreads();
      const unsigned long long cw = s_cw;
      if (wd.kind) {
        const RescatterSrc &src = W.srcs[wd.src0 + (uint32_t)(cw >> 48)];
        const uint32_t s0 = (uint32_t)cw;
        const uint32_t s1 = min(s0 + (uint32_t)((cw >> 32) & 0xFFFFu) * 32u, min(*src.fill, src.cap));
        rescatter_chunk(g, S, src, s0, s1);
      } else {
        ScatterArgs A = W.sc;
        A.tiles = W.sc.tiles + wd.tile0;
        const uint32_t t0 = (uint32_t)cw, n = t0 + (uint32_t)((cw >> 32) & 0xFFFFu), unit = (uint32_t)(cw >> 48);
        scatter_chunk<MC>(g, ybuf, A, S, dg, W.sc.units[wd.unit0 + unit], t0, n, dacc);
      }
      __syncthreads();
      if (tid == 0) { __threadfence(); atomicAdd(W.scat_done + w, 1u); }
      if (tid == 0 && W.pa.dbg) { const long long now = clock64(); atomicAdd(W.pa.dbg + 4, (unsigned long long)(now - t_prev)); t_prev = now; }
    }
  }
  if (dacc == 0x123456789ull) W.sc.batch_filtered[0] = dacc;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel): the attribute belongs
// to each device's context, so a process that solves on several devices must set it on each.
cudaError_t smem_attr(const void *fn, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void *>> done;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, fn})) return cudaSuccess;
  if (cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)) return e;
  done.insert({dev, fn});
  return cudaSuccess;
}

template <int MC>
static cudaError_t launch_scatter_mc(const ScatterArgs &a, const PartArgs &p, int grid, cudaStream_t st) {
  const size_t sm = scatter_smem_bytes(stride_for(MC));
  if (cudaError_t e = smem_attr((const void *)k_scatter<MC>, sm)) return e;
  k_scatter<MC><<<grid, kScatterThreads, sm, st>>>(a, p);
  return cudaGetLastError();
}

cudaError_t launch_scatter(int mc, const ScatterArgs &args, const PartArgs &p, int num_sms, cudaStream_t st) {
  if (args.nchunks == 0) return cudaSuccess;
  const uint32_t slots = (uint32_t)num_sms * kScatterCtas;
  const int grid = args.cta_first ? (int)slots : (int)(args.nchunks < slots ? args.nchunks : slots);
  switch (mc) {
#define MSP_CASE(N) case N: return launch_scatter_mc<N>(args, p, grid, st);
    MSP_CASE(0) MSP_CASE(1) MSP_CASE(2) MSP_CASE(3) MSP_CASE(4) MSP_CASE(5) MSP_CASE(6) MSP_CASE(7)
    MSP_CASE(8) MSP_CASE(9) MSP_CASE(10) MSP_CASE(11) MSP_CASE(12) MSP_CASE(13) MSP_CASE(14)
    MSP_CASE(15) MSP_CASE(17) MSP_CASE(18) MSP_CASE(19) MSP_CASE(20) MSP_CASE(21) MSP_CASE(22)
    MSP_CASE(23) MSP_CASE(24)
#undef MSP_CASE
    default: return cudaErrorInvalidValue;
  }
}

template <int MC>
static cudaError_t launch_waves_mc(const WavesArgs &w, int grid, cudaStream_t st) {
  const size_t sm = std::max({scatter_smem_bytes(stride_for(MC)), sizeof(JoinSmem), rescatter_smem_bytes()});
  if (cudaError_t e = smem_attr((const void *)k_waves<MC>, sm)) return e;
  k_waves<MC><<<grid, kScatterThreads, sm, st>>>(w);
  return cudaGetLastError();
}

cudaError_t launch_waves(int mc, const WavesArgs &w, int num_sms, cudaStream_t st) {
  if (w.ntasks == 0) return cudaSuccess;
  switch (mc) {
#define MSP_CASE(N) case N: return launch_waves_mc<N>(w, num_sms, st);
    MSP_CASE(0) MSP_CASE(1) MSP_CASE(2) MSP_CASE(3) MSP_CASE(4) MSP_CASE(5) MSP_CASE(6) MSP_CASE(7)
    MSP_CASE(8) MSP_CASE(9) MSP_CASE(10) MSP_CASE(11) MSP_CASE(12) MSP_CASE(13) MSP_CASE(14)
    MSP_CASE(15) MSP_CASE(17) MSP_CASE(18) MSP_CASE(19) MSP_CASE(20) MSP_CASE(21) MSP_CASE(22)
    MSP_CASE(23) MSP_CASE(24)
#undef MSP_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rescatter(const RescatterArgs &r, const PartArgs &p, int num_sms, cudaStream_t st) {
  const size_t sm = rescatter_smem_bytes();
  if (cudaError_t e = smem_attr((const void *)k_rescatter, sm)) return e;
  if (!r.nchunks) return cudaSuccess;
  const uint32_t slots = (uint32_t)num_sms * kScatterCtas;
  const int grid = (int)(r.nchunks < slots ? r.nchunks : slots);
  k_rescatter<<<grid, kScatterThreads, sm, st>>>(r, p);
  return cudaGetLastError();
}

cudaError_t launch_join(const PartArgs &p, int num_sms, cudaStream_t st) {
  const size_t sm = join_smem_bytes();
  if (cudaError_t e = smem_attr((const void *)k_join, sm)) return e;
  if (p.nb == 0) return cudaSuccess;
  const uint32_t grid = p.nb < (uint32_t)num_sms ? p.nb : (uint32_t)num_sms;
  k_join<<<grid, kJoinThreads, sm, st>>>(p);
  return cudaGetLastError();
}

}  // namespace msp
