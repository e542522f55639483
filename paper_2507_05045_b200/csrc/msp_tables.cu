// msp_tables.cu -- K1 quarter tables (merge-doubling) and K2/K3 alpha plan kernels.
//
// K1 replaces build_quarter_tables (enumerate1d.py:86-135): each block's power set is grown one
// column at a time by merging the sorted list L with L + a_col, the new column taking the next
// mask bit and ties taking the old half first.  That reproduces numpy's lexsort((masks, key))
// order exactly (ascending weight for A,B; descending for C,D; ties by mask ascending), so table
// indices equal the reference's.  Companion rows are then packed two u16 per u32 word.
//
// K2/K3 replace the heap stream (fastenum.py:87-147): with dense per-weight runs, the left count
// of alpha is sum_w |A_w| * |B_{alpha-w}| (histogram convolution) and every batch is the union
// of rectangles A-run(alpha - w_B) x B-run(w_B) -- no heap needed.
#include <cstdint>
#include "msp_common.cuh"
#include "msp_kernels.h"

namespace msp {

// ------------------------------------------------------------------ merge-doubling

__device__ __forceinline__ uint32_t lb_asc(const uint64_t *a, uint32_t n, uint64_t x) {  // #a[i] < x
  uint32_t lo = 0, hi = n;
  while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (a[mid] < x) lo = mid + 1; else hi = mid; }
  return lo;
}
__device__ __forceinline__ uint32_t ub_asc(const uint64_t *a, uint32_t n, uint64_t x) {  // #a[i] <= x
  uint32_t lo = 0, hi = n;
  while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (a[mid] <= x) lo = mid + 1; else hi = mid; }
  return lo;
}
__device__ __forceinline__ uint32_t gt_desc(const uint64_t *a, uint32_t n, uint64_t x) { // #a[i] > x
  uint32_t lo = 0, hi = n;
  while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (a[mid] > x) lo = mid + 1; else hi = mid; }
  return lo;
}
__device__ __forceinline__ uint32_t ge_desc(const uint64_t *a, uint32_t n, uint64_t x) { // #a[i] >= x
  uint32_t lo = 0, hi = n;
  while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (a[mid] >= x) lo = mid + 1; else hi = mid; }
  return lo;
}

__global__ void k_merge_step(MergeArgs args) {
  const MergeStep s = args.s[blockIdx.y];
  if (s.n == 0) return;
  const uint32_t total = 2 * s.n;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    if (i < s.n) {  // old element: after every new element strictly before it
      const uint64_t v = s.sw[i];
      uint32_t before;
      if (s.asc) before = v >= s.a ? lb_asc(s.sw, s.n, v - s.a) : 0;
      else before = v < s.a ? s.n : gt_desc(s.sw, s.n, v - s.a);
      s.dw[i + before] = v;
      s.dm[i + before] = s.sm[i];
    } else {        // new element: after every old element before-or-equal (old half first on ties)
      const uint32_t q = i - s.n;
      const uint64_t v = s.sw[q] + s.a;
      const uint32_t before = s.asc ? ub_asc(s.sw, s.n, v) : ge_desc(s.sw, s.n, v);
      s.dw[q + before] = v;
      s.dm[q + before] = s.sm[q] | (1u << s.bit);
    }
  }
}

// Companion rows 1..m-1 of every entry, packed P16 (two u16 per word, low half = lower row) or P32.
__global__ void k_pack(PackArgs args) {
  const PackTable t = args.t[blockIdx.y];
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < t.size; e += gridDim.x * blockDim.x) {
    const uint32_t mk = t.mask[e];
    uint32_t words[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int r = 1; r < args.m; ++r) {
      uint32_t s = 0;
      for (int b = 0; b < t.b; ++b)
        if ((mk >> b) & 1u) s += (uint32_t)args.a[(size_t)r * args.n + t.start + b];
      const int j = r - 1;
      if (args.wide) words[j] = s;  // P32 (block sums < 2^30, checked on the host)
      else words[j >> 1] |= (s & 0xFFFFu) << (16 * (j & 1));
    }
    for (int k = 0; k < args.sw; ++k) t.comp[(size_t)e * args.sw + k] = words[k];
  }
}

// Dense run bounds per weight (the _run_ends information, enumerate1d.py:138-145, keyed by weight).
__global__ void k_runs(RunArgs args) {
  const RunTable t = args.t[blockIdx.y];
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < t.size; e += gridDim.x * blockDim.x) {
    const uint32_t w = (uint32_t)t.w[e];
    if (e == 0 || t.w[e - 1] != t.w[e]) t.run_start[w] = e;
    if (e + 1 == t.size || t.w[e + 1] != t.w[e]) t.run_end[w] = e + 1;
  }
}

// Block-wide exclusive scan of one value per thread (blockDim.x multiple of 32, <= 1024).
template <class T>
__device__ T block_excl_scan(T v, T &total) {
  __shared__ T warp_sums[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_sums[lane] = s;  // inclusive
  }
  __syncthreads();
  const T base = wid ? warp_sums[wid - 1] : 0;
  total = warp_sums[nw - 1];
  __syncthreads();
  return base + x - v;
}

// Distinct-weight run lists of B (y=0) and D (y=1), in ascending weight order.
__global__ void k_yruns(YRunArgs args) {
  const YRunTable t = args.t[blockIdx.x];
  uint32_t base = 0;
  for (uint32_t w0 = 0; w0 <= t.S; w0 += blockDim.x) {
    const uint32_t w = w0 + threadIdx.x;
    const uint32_t len = w <= t.S ? t.run_end[w] - t.run_start[w] : 0;
    uint32_t tot;
    const uint32_t pos = block_excl_scan<uint32_t>(len > 0, tot);
    if (len > 0) {
      t.out_w[base + pos] = w;
      t.out_start[base + pos] = t.run_start[w];
      t.out_len[base + pos] = len;
    }
    base += tot;
  }
  if (threadIdx.x == 0) *t.out_n = base;
}

// hl[alpha] = sum_r |A_{alpha - w_r}| |B_r| (left) and hr[beta] = sum_r |C_{beta - w_r}| |D_r|.
// One warp per value v, lanes over the Y runs, then a warp sum (a thread per v left the GPU nearly
// empty: ~3000 values at (7,60), each a loop over ~1500 runs).
__global__ void k_conv(ConvArgs args) {
  const ConvSide s = args.s[blockIdx.y];
  const uint32_t ny = *s.ny, lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t v = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); v <= s.vmax; v += nw) {
    unsigned long long acc = 0;
    for (uint32_t r = lane; r < ny; r += 32) {
      const uint32_t wy = s.yw[r];
      if (wy > v) continue;
      const uint32_t wx = v - wy;
      if (wx > s.SX) continue;
      acc += (unsigned long long)(s.x_end[wx] - s.x_start[wx]) * s.ylen[r];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
    if (lane == 0) s.out[v] = acc;
  }
}

// Batches: alpha ascending with hl[alpha] > 0 and hr[t - alpha] > 0, restricted to the band.
__global__ void k_groups(GroupArgs g) {
  uint32_t base = 0;
  for (uint64_t a0 = 0; a0 <= g.amax; a0 += blockDim.x) {
    const uint64_t al = a0 + threadIdx.x;
    bool ok = al <= g.amax && al >= g.alpha_lo && al < g.alpha_hi && g.hl[al] > 0 && al <= g.target;
    uint64_t be = ok ? g.target - al : 0;
    ok = ok && be <= g.bmax && g.hr[be] > 0;
    uint32_t tot;
    const uint32_t pos = block_excl_scan<uint32_t>(ok, tot);
    if (ok && base + pos < g.max_groups) {
      g.alpha[base + pos] = al;
      g.nl[base + pos] = g.hl[al];
      g.nr[base + pos] = g.hr[be];
    }
    base += tot;
  }
  if (threadIdx.x == 0) *g.count = base;
}

// Per (batch, side): the nonempty rectangles X-run(xw_total - w) x Y-run(w) over the Y runs w,
// oriented for the warp tile (lanes_over_x: the cheaper way) with their warp-tile offsets.  Count mode
// (rects == nullptr) only produces the per-(batch, side) tile and rectangle totals the host needs
// to plan waves; write mode fills the compacted rectangle list at rect_base[2g + side].
__global__ void k_rects(RectArgs p) {
  const uint32_t g = blockIdx.x;
  if (g >= *p.count) return;
  const int side = blockIdx.y;
  const RectSide s = p.s[side];
  const uint32_t ny = *s.ny;
  const uint64_t xw_total = side == 0 ? p.alpha[g] : p.target - p.alpha[g];
  const bool write = p.rects != nullptr;
  RectDesc *out = write ? p.rects + p.rect_base[(size_t)g * 2 + side] : nullptr;
  uint64_t tbase = 0;
  uint32_t rbase = 0;
  const size_t gs = (size_t)g * 2 + side;
  for (uint32_t r0 = 0; r0 < ny; r0 += blockDim.x) {
    const uint32_t r = r0 + threadIdx.x;
    uint32_t tiles = 0, np = 0;
    RectDesc pc[2];
    if (r < ny) {
      const uint32_t wy = s.yw[r];
      if (wy <= xw_total && xw_total - wy <= s.SX) {
        const uint32_t wx = (uint32_t)(xw_total - wy);
        const uint32_t xs = s.x_start[wx];
        np = rect_pieces((uint32_t)gs, xs, s.x_end[wx] - xs, s.ys[r], s.ylen[r], pc);
        for (uint32_t k = 0; k < np; ++k) tiles += pc[k].nl * pc[k].nq;
      }
    }
    // one scan of both counts: tiles in the low 48 bits, rectangles (<= 2 per thread) in the high 16
    unsigned long long tot;
    const unsigned long long pos = block_excl_scan<unsigned long long>(tiles | (unsigned long long)np << 48, tot);
    const unsigned long long kLow = (1ull << 48) - 1;
    const uint64_t tpos = pos & kLow, ttot = tot & kLow;
    const uint32_t rpos = (uint32_t)(pos >> 48), rtot = (uint32_t)(tot >> 48);
    if (write) {
      uint32_t t = (uint32_t)(tbase + tpos);
      for (uint32_t k = 0; k < np; ++k) {
        pc[k].tile_off = t;
        t += pc[k].nl * pc[k].nq;
        out[rbase + rpos + k] = pc[k];
      }
    }
    tbase += ttot;
    rbase += rtot;
  }
  if (!write && threadIdx.x == 0) {
    p.tiles[gs] = tbase;
    p.nrect[gs] = rbase;
    if (tbase > 0xFFFFFFFFull) atomicOr(p.err, 2);
  }
}

// n <= 12 branch (solver.py:197-211, oracle.py:27-75): every assignment, x_1 = MSB of enc.
__global__ void k_brute(BruteArgs b) {
  const uint64_t total = 1ull << b.n;
  for (uint64_t enc = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; enc < total;
       enc += (uint64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    for (int i = 0; i < b.m && ok; ++i) {
      unsigned long long s = 0;
      for (int j = 0; j < b.n; ++j)
        if ((enc >> (b.n - 1 - j)) & 1) s += b.a[(size_t)i * b.n + j];
      ok = s == b.d[i];
    }
    if (ok) {
      const unsigned long long k = atomicAdd(b.count, 1ull);
      if (k < b.cap) b.out[k] = enc;
    }
  }
}

// ------------------------------------------------------------------ launch wrappers

void launch_merge_step(const MergeArgs &a, uint32_t max_n, cudaStream_t st) {
  const uint32_t threads = 256;
  uint32_t blocks = (2 * max_n + threads - 1) / threads;
  if (blocks > 4096) blocks = 4096;
  k_merge_step<<<dim3(blocks, 4), threads, 0, st>>>(a);
}
void launch_pack(const PackArgs &a, uint32_t max_size, cudaStream_t st) {
  uint32_t blocks = (max_size + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_pack<<<dim3(blocks, 4), 256, 0, st>>>(a);
}
void launch_runs(const RunArgs &a, uint32_t max_size, cudaStream_t st) {
  uint32_t blocks = (max_size + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_runs<<<dim3(blocks, 4), 256, 0, st>>>(a);
}
void launch_yruns(const YRunArgs &a, cudaStream_t st) { k_yruns<<<2, 1024, 0, st>>>(a); }
void launch_conv(const ConvArgs &a, uint32_t vmax, cudaStream_t st) {
  uint32_t blocks = (vmax + 8) / 8;  // 8 warps per block, a warp per value
  if (blocks > 8192) blocks = 8192;
  k_conv<<<dim3(blocks, 2), 256, 0, st>>>(a);
}
void launch_groups(const GroupArgs &a, cudaStream_t st) { k_groups<<<1, 1024, 0, st>>>(a); }
void launch_rects(const RectArgs &a, uint32_t max_groups, cudaStream_t st) {
  if (max_groups) k_rects<<<dim3(max_groups, 2), 256, 0, st>>>(a);
}
void launch_brute(const BruteArgs &a, cudaStream_t st) {
  const uint64_t total = 1ull << a.n;
  uint32_t blocks = (uint32_t)((total + 255) / 256);
  if (blocks > 8192) blocks = 8192;
  k_brute<<<blocks, 256, 0, st>>>(a);
}

}  // namespace msp
