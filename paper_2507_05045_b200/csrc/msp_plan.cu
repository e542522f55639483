// msp_plan.cu -- the SPARSE alpha plan: batch headers and rectangle lists for arbitrary u64 row-0
// weights (surrogate-reduced rows, K >> 100), where the dense per-weight histograms of msp_tables.cu
// (k_conv over 0..S) do not fit.
//
// The reference's heap stream (fastenum.py:87-147) emits, for every alpha in S_L n (t - S_R) in
// ascending order, the left pairs with wa + wb = alpha and the right pairs with wc + wd = t - alpha
// (SURVEY.md §0 restatement).  With distinct-weight runs of the four sorted quarter tables, a batch
// side is the union of rectangles A-run x B-run whose run weights sum to alpha.  So:
//   1. distinct-weight runs of each table (flag + compact),
//   2. every (A-run, B-run) pair's weight sum, sorted (radix sort of u64 sums, the pair as payload);
//      the same for (C-run, D-run),
//   3. run-length encode the sorted sums: distinct alpha (beta) with n_left (n_right) = sum of the
//      run-length products, and the segment of pairs = the batch side's rectangles,
//   4. a batch per distinct alpha whose beta = t - alpha is a right sum (binary search), in the
//      alpha band of this shard,
//   5. the oriented rectangle lists (RectDesc, as the dense k_rects writes them) of every batch side.
// Work is O(runs_A * runs_B + runs_C * runs_D) pair sums, streamed through alpha WINDOWS: the alpha
// range is cut into consecutive windows [lo, hi) each holding at most a budget of run pairs per side
// (left sums in [lo, hi), right sums in (t - hi, t - lo]; default 2^27, MSP_SPARSE_WINDOW_PAIRS),
// found by binary search on the per-side pair-count function; steps 2-5 run per window and append.
// The sort, scans and compactions are CUB device primitives (library code for the plan stage; the
// hot path stays hand-written).
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cstdlib>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "msp_common.cuh"
#include "msp_kernels.h"

namespace msp {
namespace {

struct Buf {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t c = bytes + bytes / 4 + 256;
    cudaError_t e = cudaMalloc(&p, c);
    if (e == cudaSuccess) cap = c;
    return e;
  }
  // grow to at least `bytes`, keeping the first `keep` bytes (stream-ordered copy)
  cudaError_t grow_keep(size_t bytes, size_t keep, cudaStream_t st) {
    if (bytes <= cap) return cudaSuccess;
    void *q = nullptr;
    const size_t c = bytes + bytes / 2 + 256;
    cudaError_t e = cudaMalloc(&q, c);
    if (e != cudaSuccess) return e;
    if (keep) e = cudaMemcpyAsync(q, p, keep, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { cudaFree(q); return e; }
    if (p) cudaFree(p);
    p = q;
    cap = c;
    return cudaSuccess;
  }
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct Work {
  Buf flag, starts, cnt1;                      // run compaction
  Buf rw[4], rs[4], rl[4];                     // distinct-weight runs of each table
  Buf k0, k1, v0, v1, pc, tmp;                 // pair sort and pair counts (scratch)
  Buf xcnt, xoff, wtot;                        // window: pairs per X-run, their offsets, side totals
  Buf ids[2], ukey[2], usum[2], ulen[2], uoff[2], nun[2], ukey2;  // per side
  Buf bflag, ridx, sel, nb, hdr, rbase, tiles, rects, err;        // batches
};
std::mutex g_mu;
std::map<int, Work *> g_work;

#define PCK(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) { err = std::string(#x) + ": " + cudaGetErrorString(e_); return MSP_CUDA_ERROR_CODE; } \
  } while (0)
constexpr int MSP_CUDA_ERROR_CODE = 3;
constexpr int MSP_UNSUPPORTED_CODE = 5;

__global__ void k_run_flags(const uint64_t *w, uint32_t n, uint8_t *flag) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
    flag[e] = (e == 0 || w[e - 1] != w[e]) ? 1 : 0;
}

// Run r of a table: weight, first entry, length (from the compacted run starts).
__global__ void k_run_info(const uint64_t *w, uint32_t n, const uint32_t *starts, const uint32_t *nruns,
                           uint64_t *rw, uint32_t *rs, uint32_t *rl) {
  const uint32_t nr = *nruns;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    const uint32_t s = starts[r], e = r + 1 < nr ? starts[r + 1] : n;
    rw[r] = w[s];
    rs[r] = s;
    rl[r] = e - s;
  }
}

// Y-runs y with wx + wy in [lo, hi): an index range of the sorted Y run weights (ascending for B,
// descending for D).
template <bool DESC>
__device__ __forceinline__ void y_range(const uint64_t *yw, uint32_t ny, uint64_t wx, uint64_t lo, uint64_t hi,
                                        uint32_t &b, uint32_t &e) {
  b = e = 0;
  if (wx >= hi) return;
  const uint64_t a = lo > wx ? lo - wx : 0, z = hi - wx;  // wy in [a, z)
  auto first = [&](uint64_t v) {  // ASC: first wy >= v; DESC: first wy < v
    uint32_t l = 0, h = ny;
    while (l < h) {
      const uint32_t m = (l + h) >> 1;
      if (DESC ? (yw[m] >= v) : (yw[m] < v)) l = m + 1; else h = m;
    }
    return l;
  };
  if (DESC) { b = first(z); e = first(a); } else { b = first(a); e = first(z); }
  if (e < b) e = b;
}

// Pairs of one side whose sum lies in [lo, hi): per X-run count (optional) and the side total.
template <bool DESC>
__global__ void k_window_count(const uint64_t *xw, uint32_t nx, const uint64_t *yw, uint32_t ny, uint64_t lo,
                               uint64_t hi, uint64_t *xcnt, unsigned long long *total) {
  uint64_t acc = 0;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < nx; x += gridDim.x * blockDim.x) {
    uint32_t b, e;
    y_range<DESC>(yw, ny, xw[x], lo, hi, b, e);
    if (xcnt) xcnt[x] = e - b;
    acc += e - b;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc && total) atomicAdd(total, (unsigned long long)acc);
}

// Window search: pairs of one side with sums in [a[c], z[c]) for up to kProbe candidate windows at
// once (blockIdx.y = candidate), one 64-bit total per candidate.
constexpr int kProbe = 32;
struct WinProbe { uint64_t a[kProbe], z[kProbe]; };
template <bool DESC>
__global__ void k_window_probe(const uint64_t *xw, uint32_t nx, const uint64_t *yw, uint32_t ny, WinProbe pr,
                               unsigned long long *total) {
  const int c = blockIdx.y;
  uint64_t acc = 0;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < nx; x += gridDim.x * blockDim.x) {
    uint32_t b, e;
    y_range<DESC>(yw, ny, xw[x], pr.a[c], pr.z[c], b, e);
    acc += e - b;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(total + c, (unsigned long long)acc);
}

// The window's pairs of one side: weight sum (key) and pair id x * ny + y (payload), X-run x at xoff[x]
// (one warp per X-run).
template <bool DESC>
__global__ void k_window_pairs(const uint64_t *xw, uint32_t nx, const uint64_t *yw, uint32_t ny, uint64_t lo,
                               uint64_t hi, const uint64_t *xoff, uint64_t *key, uint64_t *val) {
  const uint32_t lane = threadIdx.x & 31, nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t x = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); x < nx; x += nw) {
    const uint64_t wx = xw[x];
    uint32_t b, e;
    y_range<DESC>(yw, ny, wx, lo, hi, b, e);
    const uint64_t o = xoff[x];
    for (uint32_t y = b + lane; y < e; y += 32) {
      key[o + (y - b)] = wx + yw[y];
      val[o + (y - b)] = (uint64_t)x * ny + y;
    }
  }
}

// Pair count (run-length product) of each sorted pair, for the per-sum totals.
__global__ void k_pair_counts(const uint64_t *val, uint64_t np, const uint32_t *xl, const uint32_t *yl, uint32_t ny,
                              uint64_t *cnt) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < np; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = val[i];
    const uint32_t x = (uint32_t)(p / ny), y = (uint32_t)(p - (uint64_t)x * ny);
    cnt[i] = (uint64_t)xl[x] * yl[y];
  }
}

// Batches: distinct left sums alpha (ascending) in [alpha_lo, alpha_hi) whose beta = t - alpha is
// a distinct right sum; flag + the right sum's index.
__global__ void k_match(const uint64_t *ua, const uint32_t *na, const uint64_t *ub, const uint32_t *nbp,
                        uint64_t target, uint64_t lo, uint64_t hi, uint8_t *flag, uint32_t *ridx) {
  const uint32_t n = *na, nb = *nbp;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t a = ua[i];
    bool ok = a <= target && a >= lo && a < hi;
    uint32_t j = 0;
    if (ok) {
      const uint64_t b = target - a;
      uint32_t l = 0, h = nb;  // first index with ub >= b
      while (l < h) { const uint32_t m = (l + h) >> 1; if (ub[m] < b) l = m + 1; else h = m; }
      ok = l < nb && ub[l] == b;
      j = l;
    }
    flag[i] = ok ? 1 : 0;
    ridx[i] = j;
  }
}

// Batch g's header: (alpha, n_left, n_right, left segment offset, count, right segment offset, count).
__global__ void k_batch_headers(const uint32_t *sel, const uint32_t *nsel, const uint32_t *ridx,
                                const uint64_t *ua, const uint64_t *ca, const uint32_t *oa, const uint32_t *cnta,
                                const uint64_t *cb, const uint32_t *ob, const uint32_t *cntb, uint64_t *hdr) {
  const uint32_t G = *nsel;
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    const uint32_t i = sel[g], j = ridx[i];
    uint64_t *h = hdr + 7 * (size_t)g;
    h[0] = ua[i]; h[1] = ca[i]; h[2] = cb[j]; h[3] = oa[i]; h[4] = cnta[i]; h[5] = ob[j]; h[6] = cntb[j];
  }
}

__device__ uint32_t block_scan_excl(uint32_t v, uint32_t &total) {
  __shared__ uint32_t ws[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < nw ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const uint32_t y = __shfl_up_sync(0xffffffffu, s, o); if (lane >= o) s += y; }
    ws[lane] = s;
  }
  __syncthreads();
  const uint32_t base = wid ? ws[wid - 1] : 0;
  total = ws[nw - 1];
  __syncthreads();
  return base + x - v;
}

struct RectSparseSide {
  const uint64_t *val;                 // sorted pair ids
  const uint32_t *xs, *xl, *ys, *yl;   // X / Y run starts and lengths
  uint32_t ny;
};

// Block (g, side): the batch side's rectangles X-run x Y-run, oriented for the warp tile (lanes_over_x:
// the cheaper orientation) with their tile offsets -- the records k_rects writes for the dense plan.
__global__ void k_rects_sparse(RectSparseSide L, RectSparseSide R, const uint64_t *hdr, const uint32_t *rbase,
                               uint32_t g0, RectDesc *rects, unsigned long long *tiles, int *err) {
  const uint32_t g = blockIdx.x;  // batch g0 + g of the plan
  const int side = blockIdx.y;
  const RectSparseSide &S = side ? R : L;
  const uint64_t *h = hdr + 7 * (size_t)g;
  const uint32_t off = (uint32_t)h[side ? 5 : 3], cnt = (uint32_t)h[side ? 6 : 4];
  RectDesc *out = rects + rbase[2 * (size_t)g + side];
  uint64_t tbase = 0;
  for (uint32_t r0 = 0; r0 < cnt; r0 += blockDim.x) {
    const uint32_t r = r0 + threadIdx.x;
    uint32_t t = 0;
    RectDesc D{};
    if (r < cnt) {
      const uint64_t p = S.val[off + r];
      const uint32_t x = (uint32_t)(p / S.ny), y = (uint32_t)(p - (uint64_t)x * S.ny);
      const uint32_t xs = S.xs[x], xl = S.xl[x], ys = S.ys[y], yl = S.yl[y];
      // one piece per run pair (the segment counts fixed the rectangle bases): the cheaper orientation
      D = rect_piece((g0 + g) * 2 + side, lanes_over_x(xl, yl), xs, xl, ys, yl);
      t = D.nl * D.nq;
    }
    uint32_t tot;
    const uint32_t pos = block_scan_excl(t, tot);
    if (r < cnt) {
      D.tile_off = (uint32_t)(tbase + pos);
      out[r] = D;
    }
    tbase += tot;
  }
  if (threadIdx.x == 0) {
    tiles[2 * (size_t)g + side] = tbase;
    if (tbase > 0xFFFFFFFFull) atomicOr(err, 2);
  }
}

unsigned grid_for(uint64_t n) { return (unsigned)std::min<uint64_t>((n + 255) / 256, 4096); }

// One alpha window [lo, hi): steps 2-5 on its pair sums (cnt[side] pairs per side), batches and
// rectangles appended to `out` (batch index from Gtot, rectangle index from nrt).
template <class CountF>
int sparse_window(Work *W, const SparsePlanIn &in, const uint32_t nr[4], uint64_t lo, uint64_t hi,
                  const uint64_t cnt[2], CountF &launch_count, cudaStream_t st, int64_t &launches,
                  SparsePlanOut &out, uint64_t &nrt, uint32_t &Gtot, std::string &err) {
  thrust::counting_iterator<uint32_t> ci(0);
  size_t tb = 0;
  const uint64_t t = in.target;
  uint32_t nu[2];
  // ---- 2./3. per side: the window's run-pair sums, sorted; distinct sums with their n and segment
  for (int side = 0; side < 2; ++side) {
    const int X = side ? 2 : 0, Y = side ? 3 : 1;
    const uint64_t P = cnt[side];
    if (P >= (1ull << 31)) {
      char b[200];
      snprintf(b, sizeof b, "sparse alpha plan: %llu run pairs of one alpha window side", (unsigned long long)P);
      err = b;
      return MSP_UNSUPPORTED_CODE;
    }
    PCK(W->k0.ensure(8 * P)); PCK(W->k1.ensure(8 * P)); PCK(W->v0.ensure(8 * P)); PCK(W->v1.ensure(8 * P));
    PCK(W->pc.ensure(8 * P));
    PCK(W->xcnt.ensure(8ull * nr[X] + 8)); PCK(W->xoff.ensure(8ull * nr[X] + 8));
    launch_count(side, lo, hi, W->xcnt.as<uint64_t>(), nullptr);
    tb = 0;
    PCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, W->xcnt.as<uint64_t>(), W->xoff.as<uint64_t>(), (int)nr[X], st));
    PCK(W->tmp.ensure(tb));
    PCK(cub::DeviceScan::ExclusiveSum(W->tmp.p, tb, W->xcnt.as<uint64_t>(), W->xoff.as<uint64_t>(), (int)nr[X], st));
    const uint64_t a = side ? t + 1 - hi : lo, z = side ? t + 1 - lo : hi;
    const unsigned gp = (unsigned)std::min<uint64_t>((nr[X] + 7) / 8, 4096);
    if (side)
      k_window_pairs<true><<<gp, 256, 0, st>>>(W->rw[X].as<uint64_t>(), nr[X], W->rw[Y].as<uint64_t>(), nr[Y], a, z,
                                               W->xoff.as<uint64_t>(), W->k0.as<uint64_t>(), W->v0.as<uint64_t>());
    else
      k_window_pairs<false><<<gp, 256, 0, st>>>(W->rw[X].as<uint64_t>(), nr[X], W->rw[Y].as<uint64_t>(), nr[Y], a, z,
                                                W->xoff.as<uint64_t>(), W->k0.as<uint64_t>(), W->v0.as<uint64_t>());
    cub::DoubleBuffer<uint64_t> dk(W->k0.as<uint64_t>(), W->k1.as<uint64_t>());
    cub::DoubleBuffer<uint64_t> dv(W->v0.as<uint64_t>(), W->v1.as<uint64_t>());
    tb = 0;
    PCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)P, 0, 64, st));
    PCK(W->tmp.ensure(tb));
    PCK(cub::DeviceRadixSort::SortPairs(W->tmp.p, tb, dk, dv, (int)P, 0, 64, st));
    const uint64_t *skey = dk.Current();
    PCK(W->ids[side].ensure(8 * P));
    PCK(cudaMemcpyAsync(W->ids[side].p, dv.Current(), 8 * P, cudaMemcpyDeviceToDevice, st));  // the rectangles
    k_pair_counts<<<grid_for(P), 256, 0, st>>>(W->ids[side].as<uint64_t>(), P, W->rl[X].as<uint32_t>(),
                                               W->rl[Y].as<uint32_t>(), nr[Y], W->pc.as<uint64_t>());
    PCK(W->ukey[side].ensure(8 * P)); PCK(W->usum[side].ensure(8 * P)); PCK(W->ulen[side].ensure(4 * P));
    PCK(W->uoff[side].ensure(4 * P)); PCK(W->nun[side].ensure(8)); PCK(W->ukey2.ensure(8 * P));
    PCK(W->cnt1.ensure(8));
    tb = 0;  // distinct sums with their total pair counts (n_left / n_right)
    PCK(cub::DeviceReduce::ReduceByKey(nullptr, tb, skey, W->ukey[side].as<uint64_t>(), W->pc.as<uint64_t>(),
                                       W->usum[side].as<uint64_t>(), W->nun[side].as<uint32_t>(), cub::Sum(), (int)P, st));
    PCK(W->tmp.ensure(tb));
    PCK(cub::DeviceReduce::ReduceByKey(W->tmp.p, tb, skey, W->ukey[side].as<uint64_t>(), W->pc.as<uint64_t>(),
                                       W->usum[side].as<uint64_t>(), W->nun[side].as<uint32_t>(), cub::Sum(), (int)P, st));
    tb = 0;  // ... and their pair segments (run lengths, exclusive scan)
    PCK(cub::DeviceRunLengthEncode::Encode(nullptr, tb, skey, W->ukey2.as<uint64_t>(), W->ulen[side].as<uint32_t>(),
                                           W->cnt1.as<uint32_t>(), (int)P, st));
    PCK(W->tmp.ensure(tb));
    PCK(cub::DeviceRunLengthEncode::Encode(W->tmp.p, tb, skey, W->ukey2.as<uint64_t>(), W->ulen[side].as<uint32_t>(),
                                           W->cnt1.as<uint32_t>(), (int)P, st));
    PCK(cudaMemcpyAsync(&nu[side], W->nun[side].p, 4, cudaMemcpyDeviceToHost, st));
    PCK(cudaStreamSynchronize(st));
    tb = 0;
    PCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, W->ulen[side].as<uint32_t>(), W->uoff[side].as<uint32_t>(),
                                      (int)nu[side], st));
    PCK(W->tmp.ensure(tb));
    PCK(cub::DeviceScan::ExclusiveSum(W->tmp.p, tb, W->ulen[side].as<uint32_t>(), W->uoff[side].as<uint32_t>(),
                                      (int)nu[side], st));
    launches += 4;
  }
  // ---- 4. batches: distinct alpha (ascending) of the window with t - alpha a right sum
  PCK(W->bflag.ensure(nu[0] + 16));
  PCK(W->ridx.ensure(4ull * nu[0] + 4));
  PCK(W->sel.ensure(4ull * nu[0] + 4));
  PCK(W->nb.ensure(8));
  k_match<<<grid_for(nu[0]), 256, 0, st>>>(W->ukey[0].as<uint64_t>(), W->nun[0].as<uint32_t>(),
                                            W->ukey[1].as<uint64_t>(), W->nun[1].as<uint32_t>(), t, lo, hi,
                                            W->bflag.as<uint8_t>(), W->ridx.as<uint32_t>());
  tb = 0;
  PCK(cub::DeviceSelect::Flagged(nullptr, tb, ci, W->bflag.as<uint8_t>(), W->sel.as<uint32_t>(), W->nb.as<uint32_t>(),
                                 (int)nu[0], st));
  PCK(W->tmp.ensure(tb));
  PCK(cub::DeviceSelect::Flagged(W->tmp.p, tb, ci, W->bflag.as<uint8_t>(), W->sel.as<uint32_t>(), W->nb.as<uint32_t>(),
                                 (int)nu[0], st));
  uint32_t G = 0;
  PCK(cudaMemcpyAsync(&G, W->nb.p, 4, cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  launches += 2;
  if (!G) return 0;
  if ((uint64_t)Gtot + G >= (1u << 30)) { err = "sparse alpha plan: more than 2^30 batches"; return MSP_UNSUPPORTED_CODE; }
  PCK(W->hdr.ensure(8ull * 7 * G));
  k_batch_headers<<<grid_for(G), 256, 0, st>>>(W->sel.as<uint32_t>(), W->nb.as<uint32_t>(), W->ridx.as<uint32_t>(),
                                                W->ukey[0].as<uint64_t>(), W->usum[0].as<uint64_t>(),
                                                W->uoff[0].as<uint32_t>(), W->ulen[0].as<uint32_t>(),
                                                W->usum[1].as<uint64_t>(), W->uoff[1].as<uint32_t>(),
                                                W->ulen[1].as<uint32_t>(), W->hdr.as<uint64_t>());
  std::vector<uint64_t> h(7 * (size_t)G);
  PCK(cudaMemcpyAsync(h.data(), W->hdr.p, 8ull * 7 * G, cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  const size_t g0 = Gtot, nrt0 = nrt;
  out.alpha.resize(g0 + G);
  out.nl.resize(g0 + G);
  out.nr.resize(g0 + G);
  out.tiles.resize(2 * (g0 + G), 0);
  out.rect_base.resize(2 * (g0 + G), 0);
  out.nrect.resize(2 * (g0 + G), 0);
  for (uint32_t g = 0; g < G; ++g) {
    const uint64_t *r = &h[7 * (size_t)g];
    out.alpha[g0 + g] = r[0];
    out.nl[g0 + g] = r[1];
    out.nr[g0 + g] = r[2];
    for (int side = 0; side < 2; ++side) {
      out.rect_base[2 * (g0 + g) + side] = (uint32_t)nrt;
      out.nrect[2 * (g0 + g) + side] = (uint32_t)r[side ? 6 : 4];
      nrt += r[side ? 6 : 4];
    }
  }
  if (nrt > 0xFFFFFFFFull) { err = "rectangle list too large"; return MSP_UNSUPPORTED_CODE; }
  // ---- 5. the oriented rectangle lists of the window's batch sides, after the earlier windows' ones
  PCK(W->rects.grow_keep(sizeof(RectDesc) * std::max<uint64_t>(nrt, 1), sizeof(RectDesc) * nrt0, st));
  PCK(W->rbase.ensure(4ull * 2 * G));
  PCK(cudaMemcpyAsync(W->rbase.p, out.rect_base.data() + 2 * g0, 4ull * 2 * G, cudaMemcpyHostToDevice, st));
  PCK(W->tiles.ensure(8ull * 2 * G));
  PCK(W->err.ensure(8));
  PCK(cudaMemsetAsync(W->err.p, 0, 4, st));
  RectSparseSide L{W->ids[0].as<uint64_t>(), W->rs[0].as<uint32_t>(), W->rl[0].as<uint32_t>(), W->rs[1].as<uint32_t>(),
                   W->rl[1].as<uint32_t>(), nr[1]};
  RectSparseSide R{W->ids[1].as<uint64_t>(), W->rs[2].as<uint32_t>(), W->rl[2].as<uint32_t>(), W->rs[3].as<uint32_t>(),
                   W->rl[3].as<uint32_t>(), nr[3]};
  k_rects_sparse<<<dim3(G, 2), 256, 0, st>>>(L, R, W->hdr.as<uint64_t>(), W->rbase.as<uint32_t>(), (uint32_t)g0,
                                              W->rects.as<RectDesc>(), W->tiles.as<unsigned long long>(), W->err.as<int>());
  launches += 2;
  int rerr = 0;
  static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "tiles");
  PCK(cudaMemcpyAsync(out.tiles.data() + 2 * g0, W->tiles.p, 8ull * 2 * G, cudaMemcpyDeviceToHost, st));
  PCK(cudaMemcpyAsync(&rerr, W->err.p, 4, cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  PCK(cudaGetLastError());
  if (rerr) { err = "tile count of one batch side exceeds 2^32"; return MSP_UNSUPPORTED_CODE; }
  Gtot += G;
  return 0;
}

}  // namespace

int sparse_plan(int device, const SparsePlanIn &in, SparsePlanOut &out, cudaStream_t st, int64_t &launches,
                std::string &err) {
  Work *W;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_work.find(device);
    if (it == g_work.end()) it = g_work.emplace(device, new Work()).first;
    W = it->second;
  }
  out = SparsePlanOut();
  thrust::counting_iterator<uint32_t> ci(0);
  size_t tb = 0;
  // ---- 1. distinct-weight runs of each table
  uint32_t nr[4];
  for (int t = 0; t < 4; ++t) {
    const uint32_t n = in.size[t];
    PCK(W->flag.ensure(n));
    PCK(W->starts.ensure(4ull * n));
    PCK(W->cnt1.ensure(8));
    k_run_flags<<<grid_for(n), 256, 0, st>>>(in.w[t], n, W->flag.as<uint8_t>());
    tb = 0;
    PCK(cub::DeviceSelect::Flagged(nullptr, tb, ci, W->flag.as<uint8_t>(), W->starts.as<uint32_t>(),
                                   W->cnt1.as<uint32_t>(), (int)n, st));
    PCK(W->tmp.ensure(tb));
    PCK(cub::DeviceSelect::Flagged(W->tmp.p, tb, ci, W->flag.as<uint8_t>(), W->starts.as<uint32_t>(),
                                   W->cnt1.as<uint32_t>(), (int)n, st));
    PCK(W->rw[t].ensure(8ull * n));
    PCK(W->rs[t].ensure(4ull * n));
    PCK(W->rl[t].ensure(4ull * n));
    k_run_info<<<grid_for(n), 256, 0, st>>>(in.w[t], n, W->starts.as<uint32_t>(), W->cnt1.as<uint32_t>(),
                                             W->rw[t].as<uint64_t>(), W->rs[t].as<uint32_t>(), W->rl[t].as<uint32_t>());
    launches += 3;
    PCK(cudaMemcpyAsync(&nr[t], W->cnt1.p, 4, cudaMemcpyDeviceToHost, st));
    PCK(cudaStreamSynchronize(st));
  }
  // ---- the alpha windows: [lo, hi) within the band and alpha <= t, at most `budget` run pairs per side
  const uint64_t t = in.target;
  if (t == ~0ull) { err = "sparse alpha plan: target 2^64 - 1"; return MSP_UNSUPPORTED_CODE; }
  const uint64_t A0 = in.alpha_lo, A1 = std::min<uint64_t>(in.alpha_hi, t + 1);
  uint64_t budget = 1ull << 27;
  if (const char *e = getenv("MSP_SPARSE_WINDOW_PAIRS")) {
    const unsigned long long v = strtoull(e, nullptr, 0);
    if (v) budget = v;
  }
  PCK(W->wtot.ensure(16));
  // side 0: left sums in [lo, hi); side 1: right sums in [t + 1 - hi, t + 1 - lo)
  auto sums_lo = [&](int side, uint64_t lo, uint64_t hi) { return side ? t + 1 - hi : lo; };
  auto sums_hi = [&](int side, uint64_t lo, uint64_t hi) { return side ? t + 1 - lo : hi; };
  auto launch_count = [&](int side, uint64_t lo, uint64_t hi, uint64_t *xcnt, unsigned long long *tot) {
    const int X = side ? 2 : 0, Y = side ? 3 : 1;
    const uint64_t a = sums_lo(side, lo, hi), z = sums_hi(side, lo, hi);
    if (side)
      k_window_count<true><<<grid_for(nr[X]), 256, 0, st>>>(W->rw[X].as<uint64_t>(), nr[X], W->rw[Y].as<uint64_t>(),
                                                             nr[Y], a, z, xcnt, tot);
    else
      k_window_count<false><<<grid_for(nr[X]), 256, 0, st>>>(W->rw[X].as<uint64_t>(), nr[X], W->rw[Y].as<uint64_t>(),
                                                              nr[Y], a, z, xcnt, tot);
    ++launches;
  };
  // pair totals of both sides for the windows [lo, his[c]), c < nc (kProbe candidates per launch)
  PCK(W->wtot.ensure(16 * kProbe));
  uint64_t pc[2][kProbe];
  auto probe = [&](uint64_t lo, const uint64_t *his, int nc) -> cudaError_t {
    cudaError_t e = cudaMemsetAsync(W->wtot.p, 0, 16 * kProbe, st);
    if (e != cudaSuccess) return e;
    for (int side = 0; side < 2; ++side) {
      const int X = side ? 2 : 0, Y = side ? 3 : 1;
      WinProbe pr{};
      for (int c = 0; c < nc; ++c) { pr.a[c] = sums_lo(side, lo, his[c]); pr.z[c] = sums_hi(side, lo, his[c]); }
      const dim3 grid((unsigned)std::min<uint64_t>((nr[X] + 255) / 256, 256), nc);
      unsigned long long *tot = W->wtot.as<unsigned long long>() + side * kProbe;
      if (side)
        k_window_probe<true><<<grid, 256, 0, st>>>(W->rw[X].as<uint64_t>(), nr[X], W->rw[Y].as<uint64_t>(), nr[Y], pr, tot);
      else
        k_window_probe<false><<<grid, 256, 0, st>>>(W->rw[X].as<uint64_t>(), nr[X], W->rw[Y].as<uint64_t>(), nr[Y], pr, tot);
      ++launches;
    }
    e = cudaMemcpyAsync(pc, W->wtot.p, 16 * kProbe, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e;
  };
  uint64_t nrt = 0;  // rectangles written so far (the rect_base of the next batch side)
  uint32_t Gtot = 0;
  for (uint64_t lo = A0; lo < A1;) {
    uint64_t hi = A1, cnt[2];
    PCK(probe(lo, &hi, 1));
    cnt[0] = pc[0][0]; cnt[1] = pc[1][0];
    if (cnt[0] > budget || cnt[1] > budget) {
      // the largest hi with both sides within budget (at least one alpha: lo + 1); the counts are
      // monotone in hi, so a kProbe-ary search: `good` fits (or is lo + 1), `bad` does not
      uint64_t good = lo + 1, bad = A1;
      PCK(probe(lo, &good, 1));
      cnt[0] = pc[0][0]; cnt[1] = pc[1][0];
      while (bad - good > 1) {
        uint64_t his[kProbe];
        const uint64_t span = bad - good;
        int nc = 0;
        for (int c = 1; c <= kProbe; ++c) {
          const uint64_t h = good + (uint64_t)((unsigned __int128)span * c / (kProbe + 1));
          if (h > good && h < bad && (nc == 0 || h > his[nc - 1])) his[nc++] = h;
        }
        if (!nc) break;
        PCK(probe(lo, his, nc));
        for (int c = 0; c < nc; ++c) {
          if (pc[0][c] <= budget && pc[1][c] <= budget) {
            good = his[c];
            cnt[0] = pc[0][c]; cnt[1] = pc[1][c];
          } else {
            bad = his[c];
            break;
          }
        }
      }
      hi = good;
    }
    if (cnt[0] && cnt[1]) {
      const int rc = sparse_window(W, in, nr, lo, hi, cnt, launch_count, st, launches, out, nrt, Gtot, err);
      if (rc) return rc;
    }
    lo = hi;
  }
  PCK(cudaGetLastError());
  out.rects = W->rects.as<RectDesc>();
  return 0;
}

}  // namespace msp
