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
//   join_bucket    one CTA per bucket: insert the build side's keys (the smaller side of the batch)
//                  into a 16K-slot table in shared memory, stream the probe side's keys through
//                  it, count hash hits, record each hit key once for recovery.
//   k_waves        the persistent pipeline that runs both as tasks of one launch (one CTA per SM).
//
// The per-bucket capacity is sized from the exact batch counts (mean + 7 sigma); a bucket that
// overflows (duplicate-heavy instances) marks its batch, which the host re-joins with the global
// table path (msp_enum.cu), so results never depend on the partitioning.
#include <cstdint>
#include <algorithm>
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
#ifndef MSP_OVF_KEYS
#define MSP_OVF_KEYS (1024 / MSP_SCATTER_CTAS)
#endif
constexpr int kOvf = MSP_OVF_KEYS;                              // keys ranked past their entry's C slots
constexpr int kOvfTrigger = kOvf * 3 / 8;                       // a round ends at this many (default)
constexpr int kMaxNB = kMaxUnitBuckets;                         // entries of one unit
constexpr uint32_t kDrop = 0xFFFFFFFFu;
#ifndef MSP_RESCATTER_N
#define MSP_RESCATTER_N 4
#endif
#ifndef MSP_SCATTER_KEYS
#define MSP_SCATTER_KEYS 4
#endif
constexpr int kUS = MSP_SCATTER_KEYS;                           // keys per lane per scatter step

// Reservation of n slots at *p, result left in flight in r (predicated: no-op when n == 0, so no
// select has to wait for the atomic's return value).
__device__ __forceinline__ void reserve_async(uint32_t &r, uint32_t *p, uint32_t n) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q atom.global.add.u32 %0, [%1], %2;\n\t}"
               : "+r"(r)
               : "l"(p), "r"(n)
               : "memory");
}

// Shared memory of a scatter CTA (k_scatter / k_rescatter).  A CTA works on one CHUNK at a time:
// consecutive tiles of ONE unit (one batch side), whose keys spread uniformly over the unit's NB
// bucket entries.  The round's keys are bucketed in place: entry j owns slots [j*C, j*C + C),
// C = kStageKeys / NB, and a key's slot is its rank within the entry (one shared atomic), so the
// round needs no sort.  Keys ranked past C go to the overflow list with their (entry, rank); the
// round ends when that list passes kOvfTrigger, or at the end of the chunk.  The producers'
// loop-vector buffers follow the struct (k_scatter only).
struct __align__(16) Stage {
  unsigned long long key[kStageKeys];
  unsigned long long ovk[kOvf];
  uint32_t ove[kOvf];                // entry | rank << 11
  uint32_t cnt[kMaxNB];              // keys ranked into each entry this round
  uint2 run[kMaxNB];                 // flush: (scratch index of rank 0, staged keys to write)
  uint32_t novf, round_end, chunk, ove_spill;  // ove_spill: some rank past C has no key this round
  uint32_t tctr;                     // tiles of the chunk handed out past the first 2 per warp
  uint32_t nstaged, pad[2];          // keys staged this round (fill trigger)
};

size_t scatter_smem_bytes(int sw) { return sizeof(Stage) + (size_t)kScatterWarps * (kTQ + kUS) * sw * 4; }

__device__ __forceinline__ void stage_init(Stage &g) {
  for (uint32_t i = threadIdx.x; i < (uint32_t)kMaxNB; i += blockDim.x) g.cnt[i] = 0;
  if (threadIdx.x == 0) { g.novf = 0; g.round_end = 0; g.ove_spill = 0; g.nstaged = 0; }
}

// The CTA's next work chunk (dynamic: one global atomic per chunk), broadcast through shared memory.
__device__ __forceinline__ uint32_t next_chunk(Stage &g, unsigned int *ctr) {
  if (threadIdx.x == 0) g.chunk = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t c = g.chunk;
  __syncthreads();
  return c;
}

// Spill of an overflow key that found the overflow list full: straight to its bucket region (one
// global atomic + store); its rank slot of the round stays empty (the flush pads it).
__device__ __noinline__ void stage_spill(Stage &g, const PartArgs &S, uint32_t e, unsigned long long key) {
  const uint32_t role = e >= S.nb, b = e - role * S.nb;
  const uint32_t pos = atomicAdd(S.fill[role] + b, 1u);
  if (pos < __ldg(S.cap[role] + b)) __stcg(S.scratch + __ldg(S.start[role] + b) + pos, key);
  else atomicOr(S.batch_ovf + __ldg(S.gid + b), 1u);
  g.ove_spill = 1u;
  if (S.dbg) atomicAdd(S.dbg + 13, 1ull);
}

// Stage N keys per lane into their entries j (local to the chunk's unit): rank (shared atomics,
// all issued before any dependent store), store into the entry's slots.  Keys ranked past C go to
// the overflow list with (entry, rank): one warp-aggregated reservation per warp step.  The round
// ends once the list passes `trig` (few big entries... many small ones overflow early) or the stage
// holds `ftrig` keys (few big entries all fill at once: stop before the warps in flight overflow).
template <int N>
__device__ __forceinline__ void stage_keys(Stage &g, const PartArgs &S, uint32_t ebase, uint32_t lane, uint32_t C,
                                           uint32_t trig, uint32_t ftrig,
                                           const unsigned long long (&key)[N], const uint32_t (&j)[N],
                                           const bool (&ok)[N]) {
  uint32_t r[N], nok = 0;
#pragma unroll
  for (int u = 0; u < N; ++u) {
    r[u] = ok[u] ? atomicAdd(&g.cnt[j[u]], 1u) : 0u;
    nok += ok[u] ? 1u : 0u;
  }
  const uint32_t wok = __reduce_add_sync(0xffffffffu, nok);
  if (lane == 0 && wok && atomicAdd(&g.nstaged, wok) + wok >= ftrig) *(volatile uint32_t *)&g.round_end = 1u;
  uint32_t nov = 0;
#pragma unroll
  for (int u = 0; u < N; ++u) {
    if (ok[u] && r[u] < C) g.key[j[u] * C + r[u]] = key[u];
    nov += (ok[u] && r[u] >= C) ? 1u : 0u;
  }
  if (__any_sync(0xffffffffu, nov != 0u)) {
    uint32_t inc = nov;  // warp inclusive scan of the lanes' overflow counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (uint32_t)o) inc += y;
    }
    uint32_t ob = 0;
    if (lane == 31) ob = atomicAdd(&g.novf, inc);
    ob = __shfl_sync(0xffffffffu, ob, 31);
    const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    uint32_t o = ob + inc - nov;
#pragma unroll
    for (int u = 0; u < N; ++u) {
      if (!(ok[u] && r[u] >= C)) continue;
      if (o < (uint32_t)kOvf) {
        g.ovk[o] = key[u];
        g.ove[o] = j[u] | (r[u] << 11);
      } else {
        stage_spill(g, S, ebase + j[u], key[u]);
      }
      ++o;
    }
    if (lane == 31 && ob + tot >= trig) *(volatile uint32_t *)&g.round_end = 1u;
  }
}

// After a barrier: reserve one scratch range per nonempty entry of the chunk's unit (entries
// ebase .. ebase + NB - 1 of the launch; global atomics, one thread per entry), write the round's
// runs out (slot-major, so consecutive threads store consecutive keys of a run) and the overflow
// keys, reset the round.  Ends with a barrier.
__device__ __forceinline__ void flush_round(Stage &g, const PartArgs &S, uint32_t ebase, uint32_t NB, uint32_t C,
                                            uint32_t cmagic) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nb = S.nb;
  constexpr int kPerT = (kMaxNB + kScatterThreads - 1) / kScatterThreads;
  uint32_t res[kPerT], cn[kPerT];
#pragma unroll
  for (int k = 0; k < kPerT; ++k) {
    const uint32_t j = tid + k * kScatterThreads;
    cn[k] = j < NB ? g.cnt[j] : 0u;
    res[k] = 0u;
    if (j < NB) {
      const uint32_t e = ebase + j, role = e >= nb;
      reserve_async(res[k], S.fill[role] + (e - role * nb), cn[k]);
    }
  }
  unsigned long long nstaged = 0;
#pragma unroll
  for (int k = 0; k < kPerT; ++k) {
    const uint32_t j = tid + k * kScatterThreads;
    if (j >= NB) continue;
    if (!cn[k]) { g.run[j] = make_uint2(kDrop, 0u); continue; }
    nstaged += cn[k];
    const uint32_t e = ebase + j, role = e >= nb, b = e - role * nb;
    uint2 run = make_uint2(kDrop, 0u);
    if (res[k] + cn[k] <= __ldg(S.cap[role] + b)) run = make_uint2(__ldg(S.start[role] + b) + res[k], min(cn[k], C));
    else { atomicOr(S.batch_ovf + __ldg(S.gid + b), 1u); if (S.dbg) atomicAdd(S.dbg + 12, 1ull); }
    g.run[j] = run;
  }
  if (S.dbg) {  // diagnostics: rounds, staged keys, overflow keys
    nstaged = warp_sum(nstaged);
    if ((tid & 31) == 0 && nstaged) atomicAdd(S.dbg + 1, nstaged);
    if (tid == 0) { atomicAdd(S.dbg + 0, 1ull); atomicAdd(S.dbg + 2, (unsigned long long)g.novf); }
  }
  __syncthreads();
  const uint32_t tot = NB * C;  // (NB * C <= kStageKeys; a dropped entry has run.y == 0)
  for (uint32_t s0 = tid; s0 < tot; s0 += 2 * kScatterThreads) {  // two slots in flight per thread
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t s = s0 + h * kScatterThreads;
      const uint32_t j = __umulhi(s, cmagic), i = s - j * C;
      const uint2 run = s < tot ? g.run[j] : make_uint2(0u, 0u);
      if (i < run.y) __stcg(S.scratch + run.x + i, g.key[s]);
    }
  }
  if (g.ove_spill) {  // ranks past C whose keys were spilled stay empty: pad every rank past C
    __syncthreads();   // with key 0 (readers skip it), then write the listed overflow keys
    for (uint32_t j = warp; j < NB; j += kScatterWarps) {
      const uint32_t n = g.cnt[j], b = g.run[j].x;
      if (b == kDrop) continue;
      for (uint32_t i = C + lane; i < n; i += 32) __stcg(S.scratch + b + i, 0ull);
    }
    __syncthreads();
  }
  const uint32_t no = min(g.novf, (uint32_t)kOvf);
  for (uint32_t o = tid; o < no; o += kScatterThreads) {
    const uint32_t w = g.ove[o], j = w & 0x7FFu;
    const uint32_t b = g.run[j].x;
    if (b != kDrop) __stcg(S.scratch + b + (w >> 11), g.ovk[o]);
  }
  __syncthreads();
  for (uint32_t j = tid; j < NB; j += kScatterThreads) g.cnt[j] = 0u;
  if (tid == 0) { g.novf = 0u; g.round_end = 0u; g.ove_spill = 0u; g.nstaged = 0u; }
  __syncthreads();
}

// Per-chunk stage geometry: C slots per entry and ceil(2^32 / C) (s / C == umulhi(s, cmagic) for
// every slot index s < kStageKeys).
__device__ __forceinline__ void stage_geometry(uint32_t NB, uint32_t &C, uint32_t &cmagic) {
  C = kStageKeys / NB;
  cmagic = (uint32_t)((0xFFFFFFFFull + C) / C);
}

// ---------------------------------------------------------------- tile descriptors

// One warp per rectangle, lanes over its nl x nq warp tiles (consecutive lanes write consecutive
// 16-byte descriptors: coalesced).
__global__ void k_tiles(const TileGenArgs a) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t wpg = gridDim.x * (blockDim.x >> 5);
  for (uint32_t r = a.rect_lo + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < a.rect_hi; r += wpg) {
    const RectDesc R = a.rects[r];
    const uint32_t gs = R.gs();
    const uint32_t unit = a.gs_unit ? a.gs_unit[gs] : 0u;
    if (unit == 0xFFFFFFFFu) continue;
    TileDesc *out = a.out + (a.gs_tile_base ? a.gs_tile_base[gs] : 0ull) + R.tile_off;
    const uint32_t lx = R.lane_is_x() ? 1u : 0u;
    const uint32_t nt = R.nl * R.nq;
    for (uint32_t t = lane; t < nt; t += 32) {
      const uint32_t lc = t / R.nq, qc = t - lc * R.nq;
      const uint32_t ln = min(32u, R.L - lc * 32);
      const uint32_t qn = min((uint32_t)kTQ, R.Q - qc * kTQ);
      const uint4 v = make_uint4(R.lane_start + lc * 32, R.loop_start + qc * kTQ,
                                 unit | ((ln - 1) << 8) | ((qn - 1) << 13) | (lx << 18), 0u);
      *reinterpret_cast<uint4 *>(out + t) = v;
    }
  }
}

void launch_tiles(const TileGenArgs &a, cudaStream_t st) {
  const uint32_t n = a.rect_hi - a.rect_lo;
  if (!n) return;
  const uint32_t blocks = (n + 7) / 8;  // 8 warps per block
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
__device__ __forceinline__ void fold(uint32_t &lo, uint32_t &hi, uint32_t v) {
  const uint32_t x = lo ^ v;
  hi = hi * 435u + __umulhi(x, 435u) + (x << 8);
  lo = x * 435u;
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

// kUS keys of the current tile (loop entries q .. q+kUS-1) into the stage.
template <int MC, bool RIGHT>
__device__ __forceinline__ void hash_step(Stage &g, const PartArgs &S, const uint32_t *ybuf,
                                          const uint32_t (&lv)[stride_for(MC)],
                                          const uint32_t (&dg)[words_for(MC) > 0 ? words_for(MC) : 1],
                                          uint32_t lane, uint32_t C, uint32_t q, uint32_t qn, bool lok,
                                          const UnitInfo &ui, uint32_t nbk, uint32_t diag,
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
    key[u] = ((unsigned long long)hi << 32) | lo;
    const bool z = in && (hi | lo) == 0u;  // a real key 0: counted per (batch, side), never staged
    nzero += z ? 1u : 0u;
    ok[u] = in && !z;
    j[u] = __umulhi(hi, nbk);  // bucket within the unit = floor(hi * NB / 2^32)
  }
  if (nzero) atomicAdd(S.zero_keys + 2 * ui.gid + (RIGHT ? 1u : 0u), (unsigned long long)nzero);
  if (diag) {
#pragma unroll
    for (int u = 0; u < kUS; ++u) dacc ^= ok[u] ? key[u] : 0ull;
  } else {
    stage_keys<kUS>(g, S, ui.ent & 0x1FFFu, lane, C, S.ovf_trigger ? S.ovf_trigger : kOvfTrigger, nbk * C * 7 / 8,
                   key, j, ok);
  }
}

// One work chunk: tiles [t0, n) of ONE unit (one batch side), enumerated + hashed + partitioned by
// the CTA.  Warps take their first two tiles statically and later ones from a shared counter (so
// they finish within one tile of each other), with the descriptor two tiles ahead and the
// companion vectors one tile ahead in flight.  A round ends for every warp as soon as the overflow
// list passes its trigger (the CTA flushes, then resumes mid-tile) and at the end of the chunk.
// Filtered right pairs go to batch_filtered.  Ends with a barrier (the last flush).
template <int MC>
__device__ __forceinline__ void scatter_chunk(Stage &g, uint32_t *ybuf, const ScatterArgs &A, const PartArgs &S,
                                              const uint32_t (&dg)[words_for(MC) > 0 ? words_for(MC) : 1],
                                              const UnitInfo ui, uint32_t t0, uint32_t n, unsigned long long &dacc) {
  constexpr int SW = stride_for(MC);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  volatile uint32_t *round_end = &g.round_end;
  const uint32_t ebase = ui.ent & 0x1FFFu, nbk = (ui.ent >> 13) & 0x7FFu, side = (ui.ent >> 24) & 1u;
  const bool right = side != 0;
  uint32_t C, cmagic;
  stage_geometry(nbk, C, cmagic);
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
        hash_step<MC, true>(g, S, ybuf, lvc, dg, lane, C, q, qn, lok, ui, nbk, A.diag, filt, dacc);
      else
        hash_step<MC, false>(g, S, ybuf, lvc, dg, lane, C, q, qn, lok, ui, nbk, A.diag, filt, dacc);
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
    const bool more = __syncthreads_or(have);
    flush_round(g, S, ebase, nbk, C, cmagic);
    if (!more) break;
  }
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
  for (uint32_t c = __ldg(A.cta_first + blockIdx.x); c < cend; ++c) {
    const unsigned long long cw = __ldg(A.chunks + c);
    const uint32_t t0 = (uint32_t)cw, n = t0 + (uint32_t)((cw >> 32) & 0xFFFFu), unit = (uint32_t)(cw >> 48);
    scatter_chunk<MC>(g, ybuf, A, S, dg, A.units[unit], t0, n, dacc);
  }
  if (dacc == 0x123456789ull) A.batch_filtered[0] = dacc;  // keep the diagnostic keys live
}

// Level 2 of the huge-batch path: stream already-hashed keys back from coarse bucket regions
// (HBM) and re-partition them into fine buckets (L2 scratch) for k_join.  Work chunks are slot
// ranges of ONE source (a coarse region of one role, whose keys spread uniformly over its NF fine
// buckets); slots past the region's fill are empty.  Fine bucket = floor(frac * NF / 2^32), frac
// = the key's position inside its coarse bucket (the low word of hi * NC).
// One level-2 work chunk: slots [s0, s1) of ONE source (a coarse region of one role, whose keys
// spread uniformly over its NF fine buckets), re-partitioned by the CTA.  Ends with a barrier.
__device__ __forceinline__ void rescatter_chunk(Stage &g, const PartArgs &S, const RescatterSrc &src, uint32_t s0,
                                                uint32_t s1) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  volatile uint32_t *round_end = &g.round_end;
  constexpr int N = MSP_RESCATTER_N;  // keys per lane per step; the next step's keys are in flight meanwhile (HBM)
  const uint32_t ebase = src.role * S.nb + src.fine_base, NB = src.nf, nc = src.nc;
  uint32_t C, cmagic;
  stage_geometry(NB, C, cmagic);
  const uint32_t stride = kScatterThreads;
  uint32_t idx = s0 + warp * 32 + lane;
  unsigned long long nxt[N];
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const uint32_t x = idx + u * stride;
    nxt[u] = x < s1 ? __ldcs(src.keys + x) : 0ull;
  }
  while (true) {
    while (idx - lane < s1 && !*round_end) {
      unsigned long long key[N];
      uint32_t j[N];
      bool ok[N];
#pragma unroll
      for (int u = 0; u < N; ++u) {
        key[u] = nxt[u];
        const uint32_t x = idx + (N + u) * stride;
        nxt[u] = x < s1 ? __ldcs(src.keys + x) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < N; ++u) {
        ok[u] = key[u] != 0ull;  // past the fill, or a run pad
        j[u] = __umulhi((uint32_t)(key[u] >> 32) * nc, NB);
      }
      stage_keys<N>(g, S, ebase, lane, C, S.ovf_trigger ? S.ovf_trigger : kOvfTrigger, NB * C * 7 / 8, key, j, ok);
      idx += N * stride;
    }
    const bool more = __syncthreads_or(idx - lane < s1);
    flush_round(g, S, ebase, NB, C, cmagic);
    if (!more) break;
  }
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

#ifndef MSP_JOIN_U
#define MSP_JOIN_U 4
#endif
constexpr int kJoinThreads = 1024;
constexpr int kJoinSlots = 1 << kJoinSlotsLog2;        // 16K key slots
constexpr int kJWays = 8;                               // slots per table bucket
constexpr int kJBuckets = kJoinSlots / kJWays;          // 2K buckets of 8 slots
constexpr int kStash = 256;                             // keys whose two buckets were both full
constexpr int kHitWords = (kJoinSlots + kStash) / 32;

// Shared-memory join table of one bucket: 8-slot buckets, first fit in bucket b1, then b2, then a
// small stash.  Each slot keeps the full 64-bit key and an 8-bit fingerprint (0 = empty); the eight
// fingerprints of a bucket are one 64-bit word.  An insert is one shared atomic + two stores; a
// probe reads ONE fingerprint word and tests all eight lanes at once (zero-byte test), reading
// full keys only on a fingerprint match (~3% of probes plus the true hits).  A key can sit in b2
// only if b1 is full (no zero lane), so b2 is read only by probes whose b1 is full.  Keys arriving
// here are FNV outputs whose top bits chose the bucket; b1/b2 come from a multiplicative mix of the
// low word, the fingerprint from the middle of the high word.  Only counts and fingerprints are
// cleared per bucket.
struct JoinSmem {
  unsigned long long key[kJBuckets][kJWays];
  unsigned long long fp[kJBuckets];     // eight 8-bit fingerprints
  uint32_t cnt[kJBuckets];              // claims (may exceed 8: failed claims move on)
  unsigned long long stash[kStash];
  uint32_t hitbits[kHitWords];
  unsigned long long bhits[kJoinThreads / 32];
  uint32_t nstash, ovf;
};

size_t join_smem_bytes() { return sizeof(JoinSmem); }

struct JoinHash { uint32_t b1, b2, fp; };
__device__ __forceinline__ JoinHash join_hash(unsigned long long k) {
  const uint32_t t = (uint32_t)k * 0x9E3779B1u, hi = (uint32_t)(k >> 32);
  JoinHash h;
  h.b1 = t >> 21;
  h.b2 = h.b1 ^ (((t >> 10) & (kJBuckets - 1)) | 1u);  // != b1
  h.fp = (hi >> 8) & 0xFFu;
  if (h.fp == 0) h.fp = 1;  // 0 marks an empty slot
  return h;
}

// 0x80 in exactly the bytes of x that are zero (no false positives, unlike the borrow trick).  Per
// 32-bit half: (x & 0x7F..) + 0x7F.. never carries across a byte, so the halves are independent.
__device__ __forceinline__ uint32_t zero_byte_mask32(uint32_t x) {
  return ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);
}
__device__ __forceinline__ unsigned long long zero_byte_mask(unsigned long long x) {
  return ((unsigned long long)zero_byte_mask32((uint32_t)(x >> 32)) << 32) | zero_byte_mask32((uint32_t)x);
}
// Bucket full: slots are claimed in order 0..7 (one atomic count per bucket) and every claim below 8
// writes its fingerprint before the build/probe barrier, so the bucket is full iff slot 7 is set.
__device__ __forceinline__ bool bucket_full(unsigned long long w) { return (uint32_t)(w >> 56) != 0u; }
__device__ __forceinline__ void join_insert(JoinSmem &T, unsigned long long k) {
  const JoinHash h = join_hash(k);
  uint32_t b = h.b1, s = atomicAdd(&T.cnt[b], 1u);
  if (s >= (uint32_t)kJWays) { b = h.b2; s = atomicAdd(&T.cnt[b], 1u); }
  if (s < (uint32_t)kJWays) {
    T.key[b][s] = k;
    reinterpret_cast<uint8_t *>(&T.fp[b])[s] = (uint8_t)h.fp;  // slot s is this thread's alone
  } else {
    const uint32_t i = atomicAdd(&T.nstash, 1u);
    if (i < (uint32_t)kStash) T.stash[i] = k; else T.ovf = 1u;
  }
}

// Copies of k among the slots of bucket b whose fingerprint byte matches (one iteration per match:
// usually none, so a warp rarely runs the key comparisons at all).
__device__ __forceinline__ void count_in_bucket(const JoinSmem &T, uint32_t b, unsigned long long w,
                                                unsigned long long pat, unsigned long long k, uint32_t &c,
                                                uint32_t &first) {
  unsigned long long m = zero_byte_mask(w ^ pat);
  while (m) {
    const uint32_t s = (uint32_t)(__ffsll((long long)m) - 1) >> 3;
    if (T.key[b][s] == k) {
      if (!c) first = b * kJWays + s;
      ++c;
    }
    m &= m - 1;
  }
}

// Some byte of x is zero: the borrow trick, exact for presence (not for which bytes).
__device__ __forceinline__ bool any_zero_byte(unsigned long long x) {
  const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  return (((lo - 0x01010101u) & ~lo) | ((hi - 0x01010101u) & ~hi)) & 0x80808080u;
}

// Multiplicity of k in the table; `first` = slot id of its first copy (b1, then b2, then stash).
// Fast path (almost every probe): no fingerprint byte of b1 matches and b1 is not full.
__device__ __forceinline__ uint32_t join_count(const JoinSmem &T, unsigned long long k, uint32_t nstash,
                                               uint32_t &first) {
  const JoinHash h = join_hash(k);
  const unsigned long long pat = h.fp * 0x0101010101010101ull;
  const unsigned long long w1 = T.fp[h.b1];
  first = 0xFFFFFFFFu;
  if (!any_zero_byte(w1 ^ pat) && !bucket_full(w1)) return 0u;
  uint32_t c = 0;
  count_in_bucket(T, h.b1, w1, pat, k, c, first);
  if (bucket_full(w1)) {  // b1 full: k may have moved on to b2 (and, if b2 is full too, the stash)
    const unsigned long long w2 = T.fp[h.b2];
    count_in_bucket(T, h.b2, w2, pat, k, c, first);
    if (bucket_full(w2))
      for (uint32_t i = 0; i < nstash; ++i)
        if (T.stash[i] == k) { if (!c) first = kJoinSlots + i; ++c; }
  }
  return c;
}

// Join of bucket b of a wave by one CTA of NT threads: clear the table, insert the build keys,
// probe with the probe keys (fastval.py:75-107 semantics: every full-64-bit-hash-equal pair is a
// hit), record each hit key once, reset the bucket's fill counters for the next use of the buffer.
// Key 0 only pads runs (real zero keys are counted by the scatter) and is skipped, as are the
// zero-filled loads past the bucket's end.  Ends with a barrier.
template <int NT>
__device__ __forceinline__ void join_bucket(JoinSmem &T, const PartArgs &S, uint32_t b) {
  const uint32_t tid = threadIdx.x;
  constexpr int U = MSP_JOIN_U;  // keys loaded per thread before the table operations
  long long tp0 = 0, tp1 = 0, tp2 = 0;
  if (S.dbg && tid == 0) tp0 = clock64();
  for (uint32_t i = tid; i < (uint32_t)kJBuckets; i += NT) { T.cnt[i] = 0u; T.fp[i] = 0ull; }
  for (uint32_t i = tid; i < (uint32_t)kHitWords; i += NT) T.hitbits[i] = 0u;
  if (tid == 0) { T.nstash = 0; T.ovf = 0; }
  const uint32_t gid = __ldg(S.gid + b);
  const uint32_t nbuild = min(S.fill[0][b], __ldg(S.cap[0] + b));
  const uint32_t nprobe = min(S.fill[1][b], __ldg(S.cap[1] + b));
  const unsigned long long *bk = S.scratch + __ldg(S.start[0] + b);
  const unsigned long long *pk = S.scratch + __ldg(S.start[1] + b);
  unsigned long long kv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {  // first build keys in flight across the clear
    const uint32_t i = u * NT + tid;
    kv[u] = i < nbuild ? __ldcs(bk + i) : 0ull;
  }
  __syncthreads();
  for (uint32_t base = 0; base < nbuild; base += NT * U) {
    unsigned long long nx[U];  // next keys in flight while this batch is inserted
    const uint32_t nb2 = base + NT * U;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = nb2 + u * NT + tid;
      nx[u] = i < nbuild ? __ldcs(bk + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (kv[u]) join_insert(T, kv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) kv[u] = nx[u];
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {  // first probe keys in flight across the barrier
    const uint32_t i = u * NT + tid;
    kv[u] = i < nprobe ? __ldcs(pk + i) : 0ull;
  }
  __syncthreads();
  if (S.dbg && tid == 0) tp1 = clock64();
  const uint32_t nstash = min(T.nstash, (uint32_t)kStash);
  if (T.ovf && tid == 0) { atomicOr(S.batch_ovf + gid, 1u); if (S.dbg) atomicAdd(S.dbg + 14, 1ull); }
  unsigned long long hits = 0;
  for (uint32_t base = 0; base < nprobe; base += NT * U) {
    unsigned long long nx[U];  // next keys in flight while this batch is probed
    const uint32_t nb2 = base + NT * U;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = nb2 + u * NT + tid;
      nx[u] = i < nprobe ? __ldcs(pk + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned long long k = kv[u];
      if (!k) continue;
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
#pragma unroll
    for (int u = 0; u < U; ++u) kv[u] = nx[u];
  }
  hits = warp_sum(hits);
  if ((tid & 31) == 0) T.bhits[tid >> 5] = hits;
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
  __syncthreads();
}

__global__ void __launch_bounds__(kJoinThreads, 1) k_join(const PartArgs S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JoinSmem &T = *reinterpret_cast<JoinSmem *>(smem_raw);
  for (uint32_t b = blockIdx.x; b < S.nb; b += gridDim.x) join_bucket<kJoinThreads>(T, S, b);
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
  // Thread 0 keeps the NEXT task in flight while the CTA works: its index (atomic), word, wave
  // descriptor, chunk word and dependency target are loaded a whole task ahead; at the switch it
  // waits for the dependency (acquire load) and hands everything over through shared memory.
  struct Next { unsigned long long tk, cw; WaveDesc wd; uint32_t need; const unsigned int *ctr; };
  __shared__ unsigned long long s_cw;
  __shared__ WaveDesc s_wd;
  auto fetch = [&](Next &x) {
    const uint32_t i = atomicAdd(W.task_ctr, 1u);
    x.tk = i < W.ntasks ? W.tasks[i] : ~0ull;
    x.ctr = nullptr;
    x.need = 0;
    x.cw = 0;
    if (x.tk == ~0ull) return;
    const uint32_t w = (uint32_t)(x.tk >> 32) & 0x7FFFFFFFu;
    x.wd = W.waves[w];
    if (x.tk >> 63) {
      x.ctr = W.scat_done + w;
      x.need = x.wd.nchunks;
    } else {
      x.cw = __ldg(W.chunks + x.wd.chunk0 + (uint32_t)x.tk);
      if (w >= kWaveBuffers) {  // the last wave on this scratch buffer must be fully joined
        x.ctr = W.join_done + w - kWaveBuffers;
        x.need = W.waves[w - kWaveBuffers].njoin;
      }
    }
  };
  Next nx;
  if (tid == 0) fetch(nx);
  while (true) {
    if (tid == 0) {
      const Next cur = nx;
      if (cur.tk != ~0ull) fetch(nx);
      if (cur.ctr) {
        const long long tw = clock64();
        uint32_t v;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cur.ctr) : "memory");
          if (v >= cur.need) break;
          __nanosleep(256);
        }
        if (W.pa.dbg) atomicAdd(W.pa.dbg + 6, (unsigned long long)(clock64() - tw));
      }
      s_task = cur.tk;
      s_cw = cur.cw;
      s_wd = cur.wd;
    }
    __syncthreads();
    const unsigned long long tk = s_task;
    if (tk == ~0ull) break;
    const uint32_t w = (uint32_t)(tk >> 32) & 0x7FFFFFFFu, idx = (uint32_t)tk;
    const WaveDesc wd = s_wd;
    PartArgs S = W.pa;
    S.scratch = W.scratch[w % kWaveBuffers];
    S.fill[0] = W.fill[w % kWaveBuffers];
    S.fill[1] = W.fill[w % kWaveBuffers] + kMaxWaveBuckets;
    S.start[0] = W.bstart0 + wd.b0;
    S.start[1] = W.bstart1 + wd.b0;
    S.cap[0] = W.bcap0 + wd.b0;
    S.cap[1] = W.bcap1 + wd.b0;
    S.gid = W.bgid + wd.b0;
    S.nb = wd.nb;
    S.roles = 2;
    if (tk >> 63) {  // join: buckets [idx, idx + kJoinGroup) of the wave
      const uint32_t b1 = min(idx + (uint32_t)kJoinGroup, wd.nb);
      for (uint32_t b = idx; b < b1; ++b) join_bucket<kScatterThreads>(T, S, b);
      __syncthreads();  // (join_bucket ended with one; the CTA's writes are ordered before the release)
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
    MSP_CASE(15)
#undef MSP_CASE
    default: return cudaErrorInvalidValue;
  }
}

template <int MC>
static cudaError_t launch_waves_mc(const WavesArgs &w, int grid, cudaStream_t st) {
  const size_t sm = std::max(scatter_smem_bytes(stride_for(MC)), sizeof(JoinSmem));
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
    MSP_CASE(15)
#undef MSP_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_rescatter(const RescatterArgs &r, const PartArgs &p, int num_sms, cudaStream_t st) {
  const size_t sm = sizeof(Stage);
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
