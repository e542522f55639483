// msp_kernels.h -- host-visible argument structs and launch wrappers of the solver kernels.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "msp_common.cuh"

namespace msp {

struct MergeStep {
  const uint64_t *sw; const uint32_t *sm;  // sorted list of n entries
  uint64_t *dw; uint32_t *dm;              // merged list of 2n entries
  uint32_t n;                              // 0: table already complete
  uint64_t a;                              // row-0 coefficient of the new column
  uint32_t bit;                            // mask bit of the new column
  int asc;
};
struct MergeArgs { MergeStep s[4]; };

struct PackTable { const uint32_t *mask; uint32_t *comp; uint32_t size; int start, b; };
struct PackArgs { PackTable t[4]; const uint64_t *a; int m, n, sw, wide; };  // wide: P32 layout

struct RunTable { const uint64_t *w; uint32_t *run_start, *run_end; uint32_t size; };
struct RunArgs { RunTable t[4]; };

struct YRunTable {
  const uint32_t *run_start, *run_end; uint32_t S;
  uint32_t *out_w, *out_start, *out_len, *out_n;
};
struct YRunArgs { YRunTable t[2]; };

struct ConvSide {
  const uint32_t *x_start, *x_end; uint32_t SX;  // X table dense runs (A or C)
  const uint32_t *yw, *ylen; const uint32_t *ny; // Y runs (B or D)
  uint32_t vmax; unsigned long long *out;
};
struct ConvArgs { ConvSide s[2]; };

struct GroupArgs {
  const unsigned long long *hl, *hr; uint64_t amax, bmax, target, alpha_lo, alpha_hi;
  uint64_t *alpha; unsigned long long *nl, *nr; uint32_t *count; uint32_t max_groups;
};

struct RectSide {
  const uint32_t *x_start, *x_end; uint32_t SX;  // X table dense runs (A or C)
  const uint32_t *yw, *ys, *ylen; const uint32_t *ny;  // Y runs (B or D)
};
struct RectArgs {
  RectSide s[2]; const uint64_t *alpha; uint64_t target; const uint32_t *count;
  unsigned long long *tiles; uint32_t *nrect;  // count mode outputs, per (batch, side)
  const uint32_t *rect_base; RectDesc *rects;  // write mode (rects != nullptr)
  int *err;
};

struct BruteArgs {
  const uint64_t *a, *d; int m, n;
  unsigned long long *count; uint64_t *out; uint64_t cap;
};

// Global-hash-table join sinks (build / probe / recover), see msp_enum.cu.
struct JoinTable {
  unsigned long long *keys;    // 0 = empty (cleared per wave)
  unsigned long long *cnt;     // epoch-tagged: (epoch << 40) | hit flag << 39 | (count - 1); a
                               // slot whose tag is not this wave's epoch has count 1, no hit yet
  unsigned long long epoch;    // 24-bit tag of the current wave (never 0)
  unsigned long long *zero;    // per wave slot: count of key 0
  unsigned int *zero_hit;      // per wave slot
  HitRec *hits; unsigned long long *nhits; uint64_t hit_cap;
  PairRec *recs; unsigned long long *nrecs; uint64_t rec_cap;
  int *err;
  uint32_t nkeys;              // recovery: slots of `keys` (all regions), scanned for the filter
};

// Sparse alpha plan (msp_plan.cu) for arbitrary u64 row-0 weights: batch headers in alpha order,
// per (batch, side) rectangle bases / counts / tile totals, and the rectangle list on the device
// (owned by the plan's per-device workspace, valid until its next call).
struct SparsePlanIn {
  const uint64_t *w[4];                // sorted table weights (device)
  uint32_t size[4];
  uint64_t target, alpha_lo, alpha_hi; // alpha band [lo, hi) of this shard (hi = ~0: unbounded)
};
struct SparsePlanOut {
  std::vector<uint64_t> alpha, nl, nr, tiles;   // tiles: [2g + side]
  std::vector<uint32_t> rect_base, nrect;       // [2g + side]
  RectDesc *rects = nullptr;
};
int sparse_plan(int device, const SparsePlanIn &in, SparsePlanOut &out, cudaStream_t st, int64_t &launches,
                std::string &err);

void launch_merge_step(const MergeArgs &a, uint32_t max_n, cudaStream_t st);
void launch_pack(const PackArgs &a, uint32_t max_size, cudaStream_t st);
void launch_runs(const RunArgs &a, uint32_t max_size, cudaStream_t st);
void launch_yruns(const YRunArgs &a, cudaStream_t st);
void launch_conv(const ConvArgs &a, uint32_t vmax, cudaStream_t st);
void launch_groups(const GroupArgs &a, cudaStream_t st);
void launch_rects(const RectArgs &a, uint32_t max_groups, cudaStream_t st);
void launch_brute(const BruteArgs &a, cudaStream_t st);

// Partitioned join (msp_part.cu).  Buckets of one wave, per role (0 = build, 1 = probe).
#ifndef MSP_MAX_WAVE_BUCKETS
#define MSP_MAX_WAVE_BUCKETS 2048
#endif
constexpr int kMaxWaveBuckets = MSP_MAX_WAVE_BUCKETS;  // buckets per role per wave (ebase: 13 bits)
constexpr int kMaxUnitBuckets = 1024;  // buckets of one batch side (stage entries; UnitInfo: 11 bits)
static_assert(2 * kMaxWaveBuckets <= 8192 && kMaxUnitBuckets < 2048, "UnitInfo.ent field widths");
#ifndef MSP_SCATTER_CTAS
#define MSP_SCATTER_CTAS 1
#endif
constexpr int kScatterCtasHost = MSP_SCATTER_CTAS;  // resident k_scatter CTAs per SM (grid = SMs x this)
#ifndef MSP_STAGE_KEYS
#define MSP_STAGE_KEYS (23552 / MSP_SCATTER_CTAS)
#endif
constexpr int kScatterStageKeys = MSP_STAGE_KEYS;  // stage slots of a scatter CTA
constexpr int kJoinSlotsLog2 = 14;     // shared-memory join table: 16K (key, count) slots
#ifndef MSP_BUCKET_TARGET
#define MSP_BUCKET_TARGET 6144u
#endif
constexpr uint32_t kBucketTarget = MSP_BUCKET_TARGET;  // mean build keys per bucket (16K-slot table: load 3/8; 4K/5K/8K/10K/12K measured slower)
// Largest mean per bucket (table load 1/2): a batch side whose build keys need more than
// kMaxUnitBuckets buckets of this size takes the two-level path, whose fine buckets use this size.
constexpr uint32_t kBucketTargetMax = 1u << (kJoinSlotsLog2 - 1);
struct PartArgs {
  unsigned long long *scratch;
  const uint32_t *start[2];   // bucket region start in scratch
  const uint32_t *cap[2];     // bucket region capacity
  uint32_t *fill[2];          // keys written (reset by k_join)
  const uint32_t *gid;        // batch of each bucket
  uint32_t nb;                // buckets per role
  uint32_t roles;             // roles present in the launch's entries (0 means 2)
  unsigned long long *zero_keys;  // per (batch, side): real keys equal to 0 (never staged: 0 pads runs)
  unsigned long long *dbg;    // diagnostics (MSP_DEBUG_STATS): rounds, staged, overflow, pads
  unsigned int *batch_ovf;    // per batch: a bucket overflowed -> re-join with the global table
  HitRec *hits; unsigned long long *nhits; uint64_t hit_cap;
  unsigned long long *batch_hits;
};
constexpr uint32_t kSinkSlots = 64;    // scratch slack past the last region
// One (batch, side) unit of a scatter launch, kept in shared memory by k_scatter.
constexpr int kMaxUnits = 128;         // units per scatter launch (64 batches per wave)
struct UnitInfo {
  uint32_t h0lo, h0hi;                 // FNV state after coordinate 0 (alpha)
  uint32_t ent;                        // first (role, bucket) entry | buckets NB << 13 | side << 24
                                       // (bucket of a key = floor(hi32 * NB / 2^32))
  uint32_t gid;                        // batch index within the solve
};
// One warp tile: up to 32 lane entries x up to 32 loop entries of one rectangle (16 B, one load).
struct TileDesc {
  uint32_t lane0, loop0;               // first lane entry / first loop entry (table indices)
  uint32_t meta;                       // unit | (lane_n - 1) << 8 | (loop_n - 1) << 13 | lane_is_x << 18
  uint32_t pad;
};
struct TileGenArgs {
  const RectDesc *rects; uint32_t rect_lo, rect_hi;  // rectangles to expand (global indices)
  const uint64_t *gs_tile_base;        // by (batch, side): first tile in `out` (nullptr: 0)
  const uint32_t *gs_unit;             // by (batch, side): unit within its scatter launch, or
                                       // 0xFFFFFFFF to skip the rectangle (nullptr: unit 0)
  TileDesc *out;
  uint64_t tiles;                      // total tiles written (picks the kernel: few rectangles with
                                       // many tiles each take a warp per rectangle)
};
void launch_tiles(const TileGenArgs &a, cudaStream_t st);

// Bucket regions of one partitioned batch in its wave's scratch: buckets [b0, b0 + nb) of the launch;
// bucket k's build region starts at base + k(cb + cp) (cb slots), its probe region right after (cp).
struct BucketRun { uint32_t b0, nb, base, cb, cp, gid; };
// Expands BucketRuns into the five per-bucket arrays (start build, start probe, cap build, cap probe,
// batch id) at out, out + nbt, ..., out + 4 nbt.
void launch_expand_buckets(const BucketRun *runs, uint32_t nruns, uint32_t *out, uint32_t nbt, cudaStream_t st);
struct ScatterArgs {
  const uint32_t *comp[4];             // companion tables A, B, C, D
  uint32_t dpack[8];                   // d rows 1..m-1 packed, +0x8000 guard per half
  const TileDesc *tiles;
  const unsigned long long *chunks;    // work chunks: first tile | tile count << 32 | unit << 48
  uint32_t nchunks;
  unsigned int *chunk_ctr;             // next chunk (zeroed before the launch)
  const uint32_t *cta_first;           // static mode: CTA b runs chunks [cta_first[b], cta_first[b+1])
  const UnitInfo *units; uint32_t nunits;
  unsigned long long *batch_filtered;  // per batch (gid)
  uint32_t diag;                       // MSP_FLAG_DIAG_HASH_ONLY: hash without staging
  const int *abort_dev;                // (k_scatter) the stop word, polled per chunk
};
cudaError_t launch_scatter(int mc, const ScatterArgs &args, const PartArgs &p, int num_sms, cudaStream_t st);
// Huge batches, level 2: re-partition coarse bucket regions (already hashed keys) into fine buckets.
struct RescatterSrc {
  const unsigned long long *keys;  // coarse bucket region
  const uint32_t *fill;            // keys written into it (device counter)
  uint32_t cap, role;              // region capacity; 0 build, 1 probe
  uint32_t fine_base, nf;          // first fine bucket (per role) and fine buckets of this source
  uint32_t nc, pad;                // coarse buckets of the level-1 partition
  uint64_t in_base;                // first input slot of this source
};
struct RescatterArgs {
  const RescatterSrc *src;
  const unsigned long long *chunks;  // first slot | 32-slot groups << 32 | source << 48
  uint32_t nchunks;
  unsigned int *chunk_ctr;           // next chunk (zeroed before the launch)
};
cudaError_t launch_rescatter(const RescatterArgs &r, const PartArgs &p, int num_sms, cudaStream_t st);
cudaError_t launch_join(const PartArgs &p, int num_sms, cudaStream_t st);

// Persistent pipeline of partitioned waves (msp_part.cu k_waves): scatter chunks of wave w + 1 and
// join bucket groups of wave w from one task queue, one CTA per SM.
#ifndef MSP_JOIN_GROUP
#define MSP_JOIN_GROUP 6
#endif
constexpr uint32_t kJoinGroup = MSP_JOIN_GROUP;  // buckets per join task
constexpr uint32_t kWaveBuffers = 4;   // scratch buffers of the pipeline
#ifndef MSP_WAVE_LOOKAHEAD
#define MSP_WAVE_LOOKAHEAD 2
#endif
constexpr uint32_t kWaveLookahead = MSP_WAVE_LOOKAHEAD;  // task order S(w + 2) J(w): joins trail scatters by 2 waves
static_assert(kWaveLookahead + 1 <= kWaveBuffers, "S(w + L) must follow J(w - 1) in the queue");
struct WaveDesc {
  uint32_t tile0;                      // first tile of the wave in the tile array
  uint32_t chunk0, nchunks;            // its scatter chunks (wave-relative tiles) in the chunk array
  uint32_t unit0;                      // its units in the UnitInfo array
  uint32_t b0, nb;                     // its buckets (per role) in the bucket arrays
  uint32_t njoin;                      // its join tasks (ceil(nb / kJoinGroup))
  uint32_t kind;                       // 0: tile scatter chunks; 1: level-2 (coarse region) chunks
  uint32_t src0;                       // kind 1: its sources in the RescatterSrc array
  uint32_t pad;
};
struct WavesArgs {
  ScatterArgs sc;                      // comp, dpack, tiles (all waves), units (all waves), filters
  PartArgs pa;                         // hit list, per-batch counters, zero keys, diagnostics
  const uint32_t *bstart0, *bstart1, *bcap0, *bcap1, *bgid;  // bucket arrays of all waves
  unsigned long long *scratch;         // kWaveBuffers buffers of scratch_stride keys: wave w uses
  uint64_t scratch_stride;             //   buffer w % kWaveBuffers (no runtime-indexed param array)
  uint32_t *fill;                      // kWaveBuffers x 2 x kMaxWaveBuckets fill counters
  const WaveDesc *waves;
  const RescatterSrc *srcs;            // level-2 sources (kind 1 waves)
  const unsigned long long *chunks;    // scatter chunks of all waves
  const unsigned long long *tasks;     // join << 63 | wave << 32 | first bucket, or wave << 32 | chunk (index into chunks)
  uint32_t ntasks;
  unsigned int *task_ctr, *scat_done, *join_done;  // zeroed before the launch
  uint32_t fetch_ahead;                // 1: reserve the task after next one task early (level-2 launches)
  int *abort_dev;                      // stop word (deadline / cross-rank cancel): zeroed per solve, set
                                       // by the host watchdog with an async copy while kernels run
};
cudaError_t launch_waves(int mc, const WavesArgs &w, int num_sms, cudaStream_t st);

void launch_clear(void *p, size_t bytes, int num_sms, cudaStream_t st);

// One-sided hit recovery (msp_enum.cu): the pairs of the OTHER side of a batch whose companion
// vector (row 0 included) equals a target exactly -- d minus a recovered pair's sums -- found by
// X-entry x hash lookup of (target - X[x]) among the Y entries.
constexpr int kLookupMaxMC = 16;
struct LookupTarget { uint64_t w0, key; uint32_t tc[kLookupMaxMC]; uint32_t gid, side; };
struct LookupTable { const uint64_t *w; const uint32_t *comp; const uint32_t *mask; uint32_t n; };
struct LookupArgs {
  LookupTable X, Y;                    // X scanned, Y hashed (slots: entry + 1, 0 empty)
  const uint32_t *slots; uint32_t log2;
  int sw, nw, mc, wide;                // companion layout of the tables
  const LookupTarget *tg; uint32_t ntg;
  PairRec *out; unsigned long long *nout; uint64_t cap;
};
void launch_vhash_build(const LookupArgs &a, uint32_t *slots, cudaStream_t st);
void launch_lookup(const LookupArgs &a, cudaStream_t st);

enum SinkKind { SINK_BUILD = 0, SINK_PROBE = 1, SINK_RECOVER = 2, SINK_NONE = 3 /* diagnostic: hash only */ };
// Enumerate every pair of the launch's units, hash it, and hand the key to the sink.
int launch_enum(int mc, SinkKind kind, const EnumArgs &args, const JoinTable &jt, int num_sms,
                cudaStream_t st);

}  // namespace msp
