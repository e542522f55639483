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
// Work is O(runs_A * runs_B + runs_C * runs_D); bounded here at 2^27 pair sums per side.
// The sort, scans and compactions are CUB device primitives (library code for the plan stage; the
// hot path stays hand-written).
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <vector>

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
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
};

struct Work {
  Buf flag, starts, cnt1;                      // run compaction
  Buf rw[4], rs[4], rl[4];                     // distinct-weight runs of each table
  Buf k0, k1, v0, v1, pc, tmp;                 // pair sort and pair counts (scratch)
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

// Every (X-run, Y-run) pair: its weight sum (key) and the pair id x * ny + y (payload).
__global__ void k_pair_sums(const uint64_t *xw, uint32_t nx, const uint64_t *yw, uint32_t ny, uint64_t *key,
                            uint64_t *val) {
  const uint64_t np = (uint64_t)nx * ny;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < np; p += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = (uint32_t)(p / ny), y = (uint32_t)(p - (uint64_t)x * ny);
    key[p] = xw[x] + yw[y];
    val[p] = p;
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
                               RectDesc *rects, unsigned long long *tiles, int *err) {
  const uint32_t g = blockIdx.x;
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
      D = rect_piece(g * 2 + side, lanes_over_x(xl, yl), xs, xl, ys, yl);
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
  // ---- 2./3. per side: every run pair's weight sum, sorted; distinct sums with their n and segment
  uint32_t nu[2];
  for (int side = 0; side < 2; ++side) {
    const int X = side ? 2 : 0, Y = side ? 3 : 1;
    const uint64_t P = (uint64_t)nr[X] * nr[Y];
    if (P > (1ull << 27)) {
      char b[200];
      snprintf(b, sizeof b, "sparse alpha plan: %llu run pairs on one side exceed 2^27", (unsigned long long)P);
      err = b;
      return MSP_UNSUPPORTED_CODE;
    }
    PCK(W->k0.ensure(8 * P)); PCK(W->k1.ensure(8 * P)); PCK(W->v0.ensure(8 * P)); PCK(W->v1.ensure(8 * P));
    PCK(W->pc.ensure(8 * P));
    k_pair_sums<<<grid_for(P), 256, 0, st>>>(W->rw[X].as<uint64_t>(), nr[X], W->rw[Y].as<uint64_t>(), nr[Y],
                                             W->k0.as<uint64_t>(), W->v0.as<uint64_t>());
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
    launches += 2;
  }
  // ---- 4. batches: distinct alpha (ascending) in the band with t - alpha a right sum
  PCK(W->bflag.ensure(nu[0] + 16));
  PCK(W->ridx.ensure(4ull * nu[0] + 4));
  PCK(W->sel.ensure(4ull * nu[0] + 4));
  PCK(W->nb.ensure(8));
  k_match<<<grid_for(nu[0]), 256, 0, st>>>(W->ukey[0].as<uint64_t>(), W->nun[0].as<uint32_t>(),
                                            W->ukey[1].as<uint64_t>(), W->nun[1].as<uint32_t>(), in.target,
                                            in.alpha_lo, in.alpha_hi, W->bflag.as<uint8_t>(), W->ridx.as<uint32_t>());
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
  out.alpha.resize(G);
  out.nl.resize(G);
  out.nr.resize(G);
  out.tiles.assign(2 * (size_t)G, 0);
  out.rect_base.assign(2 * (size_t)G, 0);
  out.nrect.assign(2 * (size_t)G, 0);
  if (!G) return 0;
  PCK(W->hdr.ensure(8ull * 7 * G));
  k_batch_headers<<<grid_for(G), 256, 0, st>>>(W->sel.as<uint32_t>(), W->nb.as<uint32_t>(), W->ridx.as<uint32_t>(),
                                                W->ukey[0].as<uint64_t>(), W->usum[0].as<uint64_t>(),
                                                W->uoff[0].as<uint32_t>(), W->ulen[0].as<uint32_t>(),
                                                W->usum[1].as<uint64_t>(), W->uoff[1].as<uint32_t>(),
                                                W->ulen[1].as<uint32_t>(), W->hdr.as<uint64_t>());
  std::vector<uint64_t> h(7 * (size_t)G);
  PCK(cudaMemcpyAsync(h.data(), W->hdr.p, 8ull * 7 * G, cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  uint64_t nrt = 0;
  for (uint32_t g = 0; g < G; ++g) {
    const uint64_t *r = &h[7 * (size_t)g];
    out.alpha[g] = r[0];
    out.nl[g] = r[1];
    out.nr[g] = r[2];
    for (int side = 0; side < 2; ++side) {
      out.rect_base[2 * (size_t)g + side] = (uint32_t)nrt;
      out.nrect[2 * (size_t)g + side] = (uint32_t)r[side ? 6 : 4];
      nrt += r[side ? 6 : 4];
    }
  }
  if (nrt > 0xFFFFFFFFull) { err = "rectangle list too large"; return MSP_UNSUPPORTED_CODE; }
  // ---- 5. the oriented rectangle lists of every batch side
  PCK(W->rects.ensure(sizeof(RectDesc) * std::max<uint64_t>(nrt, 1)));
  PCK(W->rbase.ensure(4ull * 2 * G));
  PCK(cudaMemcpyAsync(W->rbase.p, out.rect_base.data(), 4ull * 2 * G, cudaMemcpyHostToDevice, st));
  PCK(W->tiles.ensure(8ull * 2 * G));
  PCK(W->err.ensure(8));
  PCK(cudaMemsetAsync(W->err.p, 0, 4, st));
  RectSparseSide L{W->ids[0].as<uint64_t>(), W->rs[0].as<uint32_t>(), W->rl[0].as<uint32_t>(), W->rs[1].as<uint32_t>(),
                   W->rl[1].as<uint32_t>(), nr[1]};
  RectSparseSide R{W->ids[1].as<uint64_t>(), W->rs[2].as<uint32_t>(), W->rl[2].as<uint32_t>(), W->rs[3].as<uint32_t>(),
                   W->rl[3].as<uint32_t>(), nr[3]};
  k_rects_sparse<<<dim3(G, 2), 256, 0, st>>>(L, R, W->hdr.as<uint64_t>(), W->rbase.as<uint32_t>(),
                                              W->rects.as<RectDesc>(), W->tiles.as<unsigned long long>(), W->err.as<int>());
  launches += 2;
  int rerr = 0;
  PCK(cudaMemcpyAsync(out.tiles.data(), W->tiles.p, 8ull * 2 * G, cudaMemcpyDeviceToHost, st));
  PCK(cudaMemcpyAsync(&rerr, W->err.p, 4, cudaMemcpyDeviceToHost, st));
  PCK(cudaStreamSynchronize(st));
  PCK(cudaGetLastError());
  if (rerr) { err = "tile count of one batch side exceeds 2^32"; return MSP_UNSUPPORTED_CODE; }
  out.rects = W->rects.as<RectDesc>();
  return 0;
}

}  // namespace msp
