// msp_solve.cu -- host orchestration and the C-ABI of libmsp_b200.so.
//
// One msp_solve call = the reference's table path (solver.py:213-245) on one GPU:
//   K1 quarter tables -> K2 plan (runs, convolution, batch list, rectangle lists) -> one host sync
//   -> join waves (build / probe launches over the global hash table) -> hit recovery -> exact
//   confirmation on the host (validate.py:285-313) -> solution bit vectors.
// All arithmetic on the hot path runs in the kernels of msp_tables.cu / msp_enum.cu; the host only
// plans waves and confirms the (rare) full-hash hits exactly, as the reference does on its CPU.
#include <algorithm>
#include <tuple>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "msp_b200.h"
#include "msp_common.cuh"
#include "msp_kernels.h"

namespace msp {
namespace {

thread_local std::string g_err;

void set_err(const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      set_err("%s failed: %s", #x, cudaGetErrorString(e_));                   \
      return MSP_CUDA_ERROR;                                                  \
    }                                                                         \
  } while (0)

struct DBuf {
  void *p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    const size_t grow = cap < (256ull << 20) ? 2 * cap : 0;  // geometric for small buffers: few regrowths
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t c = std::max<size_t>(std::max(bytes + bytes / 4, grow), 256);
    cudaError_t e = cudaMalloc(&p, c);
    if (e == cudaSuccess) cap = c;
    return e;
  }
  template <class T> T *as() const { return reinterpret_cast<T *>(p); }
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

struct Device {
  int dev = -1;
  // host staging vectors of the partitioned-wave path, kept across solves: their capacity (up to a
  // few hundred KB each) would otherwise be fresh mmap'd memory that page-faults on every solve
  std::vector<unsigned long long> h_tasks, h_tch;
  std::vector<UnitDesc> h_units;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::mutex mu;
  DBuf a, d;
  DBuf tw[4], tm[4], tw2[4], tm2[4], comp[4], rs[4], re[4];
  DBuf yw[2], ys[2], yl[2], yn;
  DBuf hl, hr, galpha, gnl, gnr, gcount, rects, nrect, rbase, tiles, err;
  DBuf units, ufilt, uhits;
  DBuf keys, cnt, zero, zhit, hits, nhits, recs, nrecs;
  DBuf bout, bcnt;
  DBuf rkeys, runits, rfilt, rhits;
  DBuf vslots, ltg, lout, lnout;  // one-sided recovery: hashed Y table, targets, matches
  DBuf bfilt, bhits, bovf, scratch, bk, bruns, fill, zkeys, dbg;
  DBuf cscratch[2], cfill, cbk, hunits, l2bk, l2src;
  uint64_t epoch = 0;  // tag of the last global-table wave (JoinTable::cnt)
  uint64_t hit_cap = 0;  // distinct hit keys the hit list holds (grown on overflow, fastval.py:126-139)
  volatile int *abort_h = nullptr;  // why the watchdog stopped the solve: 1 deadline, 2 cancel (pinned)
  int *abort_one = nullptr;         // pinned source of the stop copy
  cudaStream_t stream_wd = nullptr; // the watchdog's copy stream (runs beside the kernels)
  DBuf abort_dev;                   // the stop word the kernels poll (device memory)
  cudaStream_t stream2 = nullptr;        // join stream (overlaps the next wave's scatter)
  cudaEvent_t ev_s[2] = {nullptr, nullptr}, ev_j[2] = {nullptr, nullptr}, ev_x = nullptr;
  uint64_t wstride = 0;  // keys per wave scratch buffer (D.scratch holds kWaveBuffers of them)
  DBuf tdesc, gstb, gsu, uinfo, chunks, cchunks, l2chunks, cctr, cfirst, ccfirst, tchunks, wdesc, wctr, tasks;
  uint32_t cctr_next = 0;  // next unused chunk counter in cctr (zeroed per solve)
  // pinned staging ring for the per-launch metadata uploads: a cudaMemcpyAsync from pageable memory
  // waits for the stream to drain first, which would idle the GPU between launches
  unsigned char *ring = nullptr;
  size_t ring_cap = 0, ring_off = 0;
  // pinned landing area of the end-of-join readback (per-batch counters, flags): pageable
  // destinations make each copy a staged, synchronous transfer
  unsigned char *pin = nullptr;
  size_t pin_cap = 0;
  unsigned char *pinned(size_t bytes) {
    if (bytes <= pin_cap) return pin;
    if (pin) cudaFreeHost(pin);
    pin = nullptr;
    pin_cap = 0;
    if (cudaMallocHost(&pin, bytes) != cudaSuccess) { pin = nullptr; return nullptr; }
    pin_cap = bytes;
    return pin;
  }
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t pev[2] = {nullptr, nullptr};
  void release_all() {
    if (ring) cudaFreeHost(ring);
    ring = nullptr;
    ring_cap = ring_off = 0;
    if (pin) cudaFreeHost(pin);
    pin = nullptr;
    pin_cap = 0;
    DBuf *all[] = {&a, &d, &yn, &hl, &hr, &galpha, &gnl, &gnr, &gcount, &rects, &nrect, &rbase, &tiles, &err,
                   &units, &ufilt, &uhits, &keys, &cnt, &zero, &zhit, &hits, &nhits, &recs,
                   &nrecs, &bout, &bcnt, &rkeys, &runits, &rfilt, &rhits,
                   &bfilt, &bhits, &bovf, &zkeys, &scratch, &bk, &bruns, &fill, &cscratch[0], &cscratch[1],
                   &cfill, &cbk, &hunits, &l2bk, &l2src, &tdesc, &gstb, &gsu, &uinfo,
                   &chunks, &cchunks, &l2chunks, &cctr, &cfirst, &ccfirst, &tchunks, &wdesc, &wctr, &tasks};
    for (DBuf *b : all) b->release();
    for (int i = 0; i < 4; ++i) { tw[i].release(); tm[i].release(); tw2[i].release(); tm2[i].release();
                                  comp[i].release(); rs[i].release(); re[i].release(); }
    for (int i = 0; i < 2; ++i) { yw[i].release(); ys[i].release(); yl[i].release(); }
  }
};

std::mutex g_devices_mu;
std::map<int, Device *> g_devices;

int get_device(int dev, Device **out, double *t_init = nullptr) {
  std::lock_guard<std::mutex> lk(g_devices_mu);
  auto it = g_devices.find(dev);
  if (it != g_devices.end()) { *out = it->second; return MSP_OK; }
  const double t0 = now_s();
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (dev < 0 || dev >= ndev) { set_err("device %d out of range (%d devices)", dev, ndev); return MSP_INVALID_ARGUMENT; }
  CK(cudaSetDevice(dev));
  CK(cudaFree(nullptr));  // create the primary context now (its cost is reported as t_init)
  Device *D = new Device();
  D->dev = dev;
  CK(cudaStreamCreateWithFlags(&D->stream, cudaStreamNonBlocking));
  CK(cudaDeviceGetAttribute(&D->num_sms, cudaDevAttrMultiProcessorCount, dev));
  for (auto &e : D->ev) CK(cudaEventCreate(&e));
  for (auto &e : D->pev) CK(cudaEventCreate(&e));
  CK(cudaStreamCreateWithFlags(&D->stream2, cudaStreamNonBlocking));
  for (auto &e : D->ev_s) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto &e : D->ev_j) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&D->ev_x, cudaEventDisableTiming));
  {
    void *h = nullptr;
    CK(cudaHostAlloc(&h, 64, cudaHostAllocDefault));
    D->abort_h = reinterpret_cast<volatile int *>(h);
    D->abort_one = reinterpret_cast<int *>(h) + 4;
    *D->abort_h = 0;
    D->abort_one[0] = 1;
    CK(cudaStreamCreateWithFlags(&D->stream_wd, cudaStreamNonBlocking));
  }
  g_devices[dev] = D;
  *out = D;
  if (t_init) *t_init = now_s() - t0;
  return MSP_OK;
}

void block_sizes(int n, int out[4]) {  // enumerate1d.py:81-83
  const int q = n / 4, r = n % 4;
  for (int i = 0; i < 4; ++i) out[i] = i < r ? q + 1 : q;
}

uint32_t pow2ceil(uint64_t v) {
  uint32_t l = 0;
  while ((1ull << l) < v) ++l;
  return l;
}

// Keys per partitioned wave (both roles).  Bigger waves mean fewer two-level batches and fewer,
// fuller pipeline stages; the bucket limit (kMaxWaveBuckets per role) caps a wave near 8M build
// keys anyway.  Four pipeline buffers of this size live in HBM (~1.4 GB).
constexpr uint64_t kDefaultWaveKeys = 40ull << 20;

// Everything msp_solve needs after K1 + K2.
struct Plan {
  int m = 0, n = 0, mc = 0, sw = 1;
  int mcx = 0;            // companion layout (msp_common.cuh): mc, + kWide for P32
  bool wide = false;      // P32 companions
  bool sparse = false;    // sparse (sorted pair-sum) alpha plan instead of the dense histograms
  uint64_t S64[4] = {0, 0, 0, 0};  // exact block row-0 sums
  int b[4] = {0, 0, 0, 0}, start[4] = {0, 0, 0, 0};
  uint32_t S[4] = {0, 0, 0, 0};
  uint64_t target = 0;
  uint32_t ny[2] = {0, 0};
  uint32_t G = 0;
  std::vector<uint64_t> alpha, nl, nr, tiles;  // tiles[2g + side]
  std::vector<uint32_t> rect_base, nrect;      // [2g + side]
  EnumArgs base{};
  int merge_w_cur[4] = {0, 0, 0, 0};  // which ping-pong buffer holds the final table
};

const uint64_t *table_w(Device &D, const Plan &P, int t) {
  return P.merge_w_cur[t] ? D.tw2[t].as<uint64_t>() : D.tw[t].as<uint64_t>();
}
const uint32_t *table_m(Device &D, const Plan &P, int t) {
  return P.merge_w_cur[t] ? D.tm2[t].as<uint32_t>() : D.tm[t].as<uint32_t>();
}

// Dense row-0 plan limits: block row-0 sums up to kDenseMaxWeight and a convolution of at most
// kDenseMaxWork (weight, Y-run) steps; beyond them the sparse plan (msp_plan.cu) takes over.
constexpr uint64_t kDenseMaxWeight = 1ull << 24;
constexpr double kDenseMaxWork = 4.0e9;
bool force_sparse_plan() {
  const char *e = getenv("MSP_SPARSE_PLAN");
  return e && atoi(e) != 0;
}

// Checks the arithmetic mode preconditions (companion layout, row-0 plan).
int check_instance(const msp_problem *pr, Plan &P) {
  P.m = pr->m;
  P.n = pr->n;
  if (P.m < 1 || P.n < 1 || !pr->a || !pr->d) { set_err("invalid problem"); return MSP_INVALID_ARGUMENT; }
  if (P.n < 4) { set_err("four-block split needs n >= 4, got n=%d", P.n); return MSP_INVALID_ARGUMENT; }
  block_sizes(P.n, P.b);
  for (int t = 0, s = 0; t < 4; ++t) { P.start[t] = s; s += P.b[t]; }
  if (P.b[0] > 24) { set_err("block size %d > 24 unsupported", P.b[0]); return MSP_UNSUPPORTED; }
  P.mc = P.m - 1;
  if (P.mc > kMaxMC) { set_err("m=%d > %d rows unsupported", P.m, kMaxMC + 1); return MSP_UNSUPPORTED; }
  // companion layout: P16 when every block row sum fits 16384 and d_j <= 32767, else P32
  unsigned __int128 cmax = 0, dmax = 0;
  for (int t = 0; t < 4; ++t) {
    for (int r = 1; r < P.m; ++r) {
      unsigned __int128 s = 0;
      for (int j = 0; j < P.b[t]; ++j) s += pr->a[(size_t)r * P.n + P.start[t] + j];
      cmax = std::max(cmax, s);
    }
  }
  for (int r = 1; r < P.m; ++r) dmax = std::max<unsigned __int128>(dmax, pr->d[r]);
  P.wide = !(cmax <= 16384 && dmax <= 32767);
  if (P.wide && (P.mc > kMaxWideMC || cmax >= (1u << 30) || dmax >= (1u << 31))) {
    set_err("companion rows outside the packed layouts (P16: block sums <= 16384, d <= 32767; P32: m <= %d, "
            "block sums < 2^30, d < 2^31)", kMaxWideMC + 1);
    return MSP_UNSUPPORTED;
  }
  P.mcx = P.mc + (P.wide ? kWide : 0);
  P.sw = stride_for(P.mcx);
  // row-0 plan: dense per-weight histograms while the block sums are small, else the sparse plan
  bool big = false;
  for (int t = 0; t < 4; ++t) {
    unsigned __int128 s0 = 0;
    for (int j = 0; j < P.b[t]; ++j) s0 += pr->a[P.start[t] + j];
    if (s0 > kDenseMaxWeight) big = true;
    P.S[t] = (uint32_t)std::min<unsigned __int128>(s0, 0xFFFFFFFFu);
    P.S64[t] = (uint64_t)std::min<unsigned __int128>(s0, ~0ull);
  }
  {  // dense plan cost: the convolution loops over (S_X + 1) x (distinct Y weights <= min(S_Y + 1, 2^b_Y))
    const double nyB = std::min<double>((double)P.S[1] + 1, (double)(1ull << P.b[1]));
    const double nyD = std::min<double>((double)P.S[3] + 1, (double)(1ull << P.b[3]));
    const double work = ((double)P.S[0] + P.S[1] + 1) * nyB + ((double)P.S[2] + P.S[3] + 1) * nyD;
    if (work > kDenseMaxWork) big = true;
  }
  P.sparse = big || (force_sparse_plan());
  P.target = pr->d[0];
  return MSP_OK;
}

void fill_enum_base(Device &D, Plan &P, const msp_problem *pr, const RectDesc *rects);

// K1 + K2 on the device; ends with the batch list and tile totals on the host.
int build_plan(Device &D, const msp_problem *pr, Plan &P, uint64_t alpha_lo, uint64_t alpha_hi,
               cudaStream_t st, int64_t &launches, double *t_tables = nullptr) {
  const int m = P.m, n = P.n;
  CK(D.a.ensure(sizeof(uint64_t) * m * n));
  CK(D.d.ensure(sizeof(uint64_t) * m));
  CK(cudaMemcpyAsync(D.a.p, pr->a, sizeof(uint64_t) * m * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(D.d.p, pr->d, sizeof(uint64_t) * m, cudaMemcpyHostToDevice, st));
  uint32_t maxsize = 0;
  for (int t = 0; t < 4; ++t) {
    const size_t sz = (size_t)1 << P.b[t];
    maxsize = std::max<uint32_t>(maxsize, (uint32_t)sz);
    CK(D.tw[t].ensure(8 * sz)); CK(D.tw2[t].ensure(8 * sz));
    CK(D.tm[t].ensure(4 * sz)); CK(D.tm2[t].ensure(4 * sz));
    CK(D.comp[t].ensure(4 * sz * P.sw));
    if (!P.sparse) { CK(D.rs[t].ensure(4 * ((size_t)P.S[t] + 1))); CK(D.re[t].ensure(4 * ((size_t)P.S[t] + 1))); }
    CK(cudaMemsetAsync(D.tw[t].p, 0, 8, st));  // the empty subset: weight 0, mask 0
    CK(cudaMemsetAsync(D.tm[t].p, 0, 4, st));
    P.merge_w_cur[t] = 0;
  }
  // ---- K1: merge-doubling, one launch per column step over all four tables
  const int bmax = *std::max_element(P.b, P.b + 4);
  for (int step = 0; step < bmax; ++step) {
    MergeArgs ma{};
    uint32_t mx = 0;
    for (int t = 0; t < 4; ++t) {
      MergeStep &s = ma.s[t];
      if (step >= P.b[t]) { s.n = 0; continue; }
      const int cur = P.merge_w_cur[t];
      s.sw = cur ? D.tw2[t].as<uint64_t>() : D.tw[t].as<uint64_t>();
      s.sm = cur ? D.tm2[t].as<uint32_t>() : D.tm[t].as<uint32_t>();
      s.dw = cur ? D.tw[t].as<uint64_t>() : D.tw2[t].as<uint64_t>();
      s.dm = cur ? D.tm[t].as<uint32_t>() : D.tm2[t].as<uint32_t>();
      s.n = 1u << step;
      s.a = pr->a[P.start[t] + step];
      s.bit = step;
      s.asc = t < 2;
      mx = std::max(mx, s.n);
      P.merge_w_cur[t] ^= 1;
    }
    launch_merge_step(ma, mx, st);
    ++launches;
  }
  PackArgs pa{};
  RunArgs ra{};
  for (int t = 0; t < 4; ++t) {
    pa.t[t] = PackTable{table_m(D, P, t), D.comp[t].as<uint32_t>(), 1u << P.b[t], P.start[t], P.b[t]};
    if (P.sparse) continue;
    ra.t[t] = RunTable{table_w(D, P, t), D.rs[t].as<uint32_t>(), D.re[t].as<uint32_t>(), 1u << P.b[t]};
    CK(cudaMemsetAsync(D.rs[t].p, 0, 4 * ((size_t)P.S[t] + 1), st));
    CK(cudaMemsetAsync(D.re[t].p, 0, 4 * ((size_t)P.S[t] + 1), st));
  }
  pa.a = D.a.as<uint64_t>(); pa.m = m; pa.n = n; pa.sw = P.sw; pa.wide = P.wide;
  launch_pack(pa, maxsize, st);
  ++launches;
  if (!P.sparse) { launch_runs(ra, maxsize, st); ++launches; }
  if (t_tables) {  // K1 done: the stats split t_build (tables) from t_enumerate (the plan)
    CK(cudaStreamSynchronize(st));
    *t_tables = now_s();
  }
  if (P.sparse) {  // ---- K2/K3 for arbitrary weights: the sorted pair-sum plan (msp_plan.cu)
    SparsePlanIn si{};
    for (int t = 0; t < 4; ++t) { si.w[t] = table_w(D, P, t); si.size[t] = 1u << P.b[t]; }
    si.target = P.target;
    si.alpha_lo = alpha_lo;
    si.alpha_hi = alpha_hi ? alpha_hi : ~0ull;
    SparsePlanOut so;
    std::string perr;
    const int prc = sparse_plan(D.dev, si, so, st, launches, perr);
    if (prc) { set_err("%s", perr.c_str()); return prc; }
    P.G = (uint32_t)so.alpha.size();
    P.alpha = so.alpha; P.nl = so.nl; P.nr = so.nr; P.tiles = so.tiles;
    P.rect_base = so.rect_base; P.nrect = so.nrect;
    P.ny[0] = P.ny[1] = 0;
    fill_enum_base(D, P, pr, so.rects);
    return MSP_OK;
  }
  // ---- K2: Y-run lists, convolution, batch list
  CK(D.yn.ensure(8));
  YRunArgs ya{};
  for (int s = 0; s < 2; ++s) {
    const int t = s ? 3 : 1;
    const size_t cap = (size_t)P.S[t] + 1;
    CK(D.yw[s].ensure(4 * cap)); CK(D.ys[s].ensure(4 * cap)); CK(D.yl[s].ensure(4 * cap));
    ya.t[s] = YRunTable{D.rs[t].as<uint32_t>(), D.re[t].as<uint32_t>(), P.S[t], D.yw[s].as<uint32_t>(),
                        D.ys[s].as<uint32_t>(), D.yl[s].as<uint32_t>(), D.yn.as<uint32_t>() + s};
  }
  launch_yruns(ya, st);
  const uint64_t vmaxL = (uint64_t)P.S[0] + P.S[1], vmaxR = (uint64_t)P.S[2] + P.S[3];
  CK(D.hl.ensure(8 * (vmaxL + 1)));
  CK(D.hr.ensure(8 * (vmaxR + 1)));
  ConvArgs ca{};
  ca.s[0] = ConvSide{D.rs[0].as<uint32_t>(), D.re[0].as<uint32_t>(), P.S[0], D.yw[0].as<uint32_t>(),
                     D.yl[0].as<uint32_t>(), D.yn.as<uint32_t>(), (uint32_t)vmaxL, D.hl.as<unsigned long long>()};
  ca.s[1] = ConvSide{D.rs[2].as<uint32_t>(), D.re[2].as<uint32_t>(), P.S[2], D.yw[1].as<uint32_t>(),
                     D.yl[1].as<uint32_t>(), D.yn.as<uint32_t>() + 1, (uint32_t)vmaxR, D.hr.as<unsigned long long>()};
  launch_conv(ca, (uint32_t)std::max(vmaxL, vmaxR), st);
  const uint32_t maxG = (uint32_t)(vmaxL + 1);
  CK(D.galpha.ensure(8 * maxG)); CK(D.gnl.ensure(8 * maxG)); CK(D.gnr.ensure(8 * maxG));
  CK(D.gcount.ensure(8));
  GroupArgs ga{D.hl.as<unsigned long long>(), D.hr.as<unsigned long long>(), vmaxL, vmaxR, P.target,
               alpha_lo, alpha_hi ? alpha_hi : ~0ull, D.galpha.as<uint64_t>(),
               D.gnl.as<unsigned long long>(), D.gnr.as<unsigned long long>(), D.gcount.as<uint32_t>(), maxG};
  launch_groups(ga, st);
  launches += 3;
  uint32_t hdr[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(hdr, D.gcount.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hdr + 2, D.yn.p, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  P.G = hdr[0];
  P.ny[0] = hdr[2];
  P.ny[1] = hdr[3];
  P.alpha.resize(P.G); P.nl.resize(P.G); P.nr.resize(P.G); P.tiles.assign(2 * (size_t)P.G, 0);
  if (P.G == 0) return MSP_OK;
  // ---- rectangle lists per (batch, side): count pass, one sync, write pass
  CK(D.tiles.ensure(16 * (size_t)P.G));
  CK(D.nrect.ensure(8 * (size_t)P.G));
  CK(D.rbase.ensure(8 * (size_t)P.G));
  CK(D.err.ensure(16));
  CK(cudaMemsetAsync(D.err.p, 0, 16, st));
  RectArgs ra2{};
  for (int s = 0; s < 2; ++s) {
    const int X = s ? 2 : 0;
    ra2.s[s] = RectSide{D.rs[X].as<uint32_t>(), D.re[X].as<uint32_t>(), P.S[X], D.yw[s].as<uint32_t>(),
                        D.ys[s].as<uint32_t>(), D.yl[s].as<uint32_t>(), D.yn.as<uint32_t>() + s};
  }
  ra2.alpha = D.galpha.as<uint64_t>();
  ra2.target = P.target;
  ra2.count = D.gcount.as<uint32_t>();
  ra2.tiles = D.tiles.as<unsigned long long>();
  ra2.nrect = D.nrect.as<uint32_t>();
  ra2.err = D.err.as<int>();
  launch_rects(ra2, P.G, st);
  ++launches;
  int err = 0;
  std::vector<uint32_t> nrect(2 * (size_t)P.G);
  CK(cudaMemcpyAsync(P.alpha.data(), D.galpha.p, 8 * (size_t)P.G, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(P.nl.data(), D.gnl.p, 8 * (size_t)P.G, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(P.nr.data(), D.gnr.p, 8 * (size_t)P.G, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(P.tiles.data(), D.tiles.p, 16 * (size_t)P.G, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(nrect.data(), D.nrect.p, 8 * (size_t)P.G, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&err, D.err.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (err) { set_err("tile count of one batch side exceeds 2^32"); return MSP_UNSUPPORTED; }
  P.rect_base.assign(2 * (size_t)P.G, 0);
  P.nrect = nrect;
  uint64_t nrt = 0;
  for (size_t i = 0; i < 2 * (size_t)P.G; ++i) { P.rect_base[i] = (uint32_t)nrt; nrt += nrect[i]; }
  if (nrt > 0xFFFFFFFFull) { set_err("rectangle list too large"); return MSP_UNSUPPORTED; }
  CK(D.rects.ensure(sizeof(RectDesc) * std::max<uint64_t>(nrt, 1)));
  CK(cudaMemcpyAsync(D.rbase.p, P.rect_base.data(), 4 * 2 * (size_t)P.G, cudaMemcpyHostToDevice, st));
  ra2.rect_base = D.rbase.as<uint32_t>();
  ra2.rects = D.rects.as<RectDesc>();
  launch_rects(ra2, P.G, st);
  ++launches;
  fill_enum_base(D, P, pr, D.rects.as<RectDesc>());
  return MSP_OK;
}

// Launch-invariant enumeration arguments (tables, rectangle list, packed d).
void fill_enum_base(Device &D, Plan &P, const msp_problem *pr, const RectDesc *rects) {
  const int m = P.m;
  EnumArgs &A = P.base;
  for (int t = 0; t < 4; ++t)
    A.tab[t] = TableDev{table_w(D, P, t), table_m(D, P, t), D.comp[t].as<uint32_t>(),
                        P.sparse ? nullptr : D.rs[t].as<uint32_t>(), P.sparse ? nullptr : D.re[t].as<uint32_t>(),
                        P.S[t], 1u << P.b[t]};
  for (int s = 0; s < 2; ++s)
    A.yr[s] = P.sparse ? YRuns{nullptr, nullptr, nullptr, 0}
                       : YRuns{D.yw[s].as<uint32_t>(), D.ys[s].as<uint32_t>(), D.yl[s].as<uint32_t>(), P.ny[s]};
  A.rects = rects;
  for (int k = 0; k < 8; ++k) {
    const int c0 = 2 * k + 1, c1 = 2 * k + 2;  // rows c0, c1 (1-based companion rows)
    if (P.wide) {  // P32: word k = d[k + 1] + 2^31 (guard bit 31)
      A.dpack[k] = (k + 1 < m ? (uint32_t)pr->d[k + 1] : 0u) + 0x80000000u;
      continue;
    }
    const uint32_t lo = (c0 < m ? (uint32_t)pr->d[c0] : 0u) + 0x8000u;
    const uint32_t hi = (c1 < m ? (uint32_t)pr->d[c1] : 0u) + 0x8000u;
    A.dpack[k] = lo | (hi << 16);
  }
}

struct Wave {
  size_t ub0 = 0, ub1 = 0;   // build units [ub0, ub1) in the global unit array
  size_t up0 = 0, up1 = 0;   // probe units
  uint64_t slots = 0;        // table slots used
  uint32_t nslot = 0;        // batches (zero-key slots)
  uint64_t build_tiles = 0, probe_tiles = 0;
  uint64_t pairs = 0;        // candidate pairs enumerated by the wave
};

UnitDesc make_unit(const Plan &P, uint32_t g, int side, uint64_t tile_base) {
  UnitDesc u{};
  u.tile_base = tile_base;
  u.h0 = fnv_step64(kFnvOffset, P.alpha[g]);
  u.xw_total = (uint32_t)(side == 0 ? P.alpha[g] : P.target - P.alpha[g]);
  u.side = side;
  u.rect_base = P.rect_base[2 * (size_t)g + side];
  u.nrect = P.nrect[2 * (size_t)g + side];
  u.gid = g;
  u.npass = 1;
  return u;
}

// The shared-memory unit record of k_scatter for a unit of a wave with `nb` buckets per role; the
// unit's batch owns buckets [region_base, region_base + region_log2) of its role (for partitioned
// units region_log2 holds the bucket COUNT NB, not a log).
UnitInfo make_info(const UnitDesc &u, uint32_t nb) {
  UnitInfo i;
  i.h0lo = (uint32_t)u.h0;
  i.h0hi = (uint32_t)(u.h0 >> 32);
  const uint32_t ebase = ((u.flags >> 1) & 1u) * nb + u.region_base;
  i.ent = ebase | (u.region_log2 << 13) | (u.side << 24);  // 13 | 11 | 1 bits
  i.gid = u.gid;
  return i;
}

ScatterArgs scatter_base(const Plan &P, const EnumArgs &A) {
  ScatterArgs s{};
  for (int t = 0; t < 4; ++t) s.comp[t] = P.base.tab[t].comp;
  for (int k = 0; k < 8; ++k) s.dpack[k] = P.base.dpack[k];
  s.batch_filtered = A.batch_filtered;
  s.diag = A.diag;
  return s;
}

void set_enum_range(EnumArgs &A, const UnitDesc *units_dev, size_t nunits, uint64_t total_tiles,
                    int num_sms) {
  A.units = units_dev;
  A.nunits = (uint32_t)nunits;
  A.total_tiles = total_tiles;
  const uint64_t warps = (uint64_t)num_sms * 64;
  uint64_t ct = total_tiles / (warps * 4);
  ct = std::max<uint64_t>(1, std::min<uint64_t>(ct, 64));
  A.chunk_tiles = ct;
  A.nchunks = (total_tiles + ct - 1) / ct;
}

struct Residual { std::vector<unsigned __int128> v; };

// Exact confirmation of full-hash hits (validate.py:285-313 + assemble_solution enumerate1d.py:313-327).
int confirm(const msp_problem *pr, const Plan &P, const std::vector<PairRec> &recs,
            std::vector<std::vector<uint8_t>> &sols, int64_t &host_hash_hits) {
  const int m = P.m, n = P.n;
  auto block_sum = [&](int t, uint32_t mask, int row) {
    unsigned __int128 s = 0;
    for (int b = 0; b < P.b[t]; ++b)
      if ((mask >> b) & 1u) s += pr->a[(size_t)row * n + P.start[t] + b];
    return s;
  };
  struct Key { uint32_t gid; uint64_t key; bool operator<(const Key &o) const { return gid != o.gid ? gid < o.gid : key < o.key; } };
  std::map<Key, std::pair<std::vector<const PairRec *>, std::vector<const PairRec *>>> by;
  for (const PairRec &r : recs) {
    auto &e = by[Key{r.gid, r.key}];
    (r.side ? e.second : e.first).push_back(&r);
  }
  host_hash_hits = 0;
  for (auto &kv : by) {
    auto &L = kv.second.first;
    auto &R = kv.second.second;
    host_hash_hits += (int64_t)L.size() * (int64_t)R.size();
    if (L.empty() || R.empty()) continue;
    std::map<std::vector<unsigned __int128>, std::vector<const PairRec *>> lv;
    for (const PairRec *l : L) {
      std::vector<unsigned __int128> v(m);
      for (int i = 0; i < m; ++i) v[i] = block_sum(0, l->xmask, i) + block_sum(1, l->ymask, i);
      lv[v].push_back(l);
    }
    for (const PairRec *r : R) {
      std::vector<unsigned __int128> v(m);
      bool ok = true;
      for (int i = 0; i < m && ok; ++i) {
        const unsigned __int128 s = block_sum(2, r->xmask, i) + block_sum(3, r->ymask, i);
        if (s > pr->d[i]) ok = false; else v[i] = (unsigned __int128)pr->d[i] - s;
      }
      if (!ok) return MSP_INTERNAL;  // a filtered pair reached the join
      auto it = lv.find(v);
      if (it == lv.end()) continue;  // full-hash collision, not a solution
      for (const PairRec *l : it->second) {
        std::vector<uint8_t> x(n, 0);
        const uint32_t mk[4] = {l->xmask, l->ymask, r->xmask, r->ymask};
        for (int t = 0; t < 4; ++t)
          for (int b = 0; b < P.b[t]; ++b) x[P.start[t] + b] = (mk[t] >> b) & 1u;
        for (int i = 0; i < m; ++i) {  // verify_solution (instances.py:322-336)
          unsigned __int128 s = 0;
          for (int j = 0; j < n; ++j) if (x[j]) s += pr->a[(size_t)i * n + j];
          if (s != pr->d[i]) { set_err("internal error: residual match failed full verification"); return MSP_INTERNAL; }
        }
        sols.push_back(std::move(x));
      }
    }
  }
  return MSP_OK;
}

int brute_force(Device &D, const msp_problem *pr, cudaStream_t st, std::vector<std::vector<uint8_t>> &sols,
                int64_t &launches) {
  const int m = pr->m, n = pr->n;
  if (n > 28) { set_err("brute force capped at n <= 28, got n=%d", n); return MSP_INVALID_ARGUMENT; }
  for (int i = 0; i < m; ++i) {
    unsigned __int128 s = 0;
    for (int j = 0; j < n; ++j) s += pr->a[(size_t)i * n + j];
    if (s > ~0ull) { set_err("row sum overflow"); return MSP_INVALID_ARGUMENT; }
  }
  uint64_t cap = 1 << 16;
  for (int attempt = 0; attempt < 2; ++attempt) {
    CK(D.a.ensure(8 * (size_t)m * n)); CK(D.d.ensure(8 * (size_t)m));
    CK(D.bout.ensure(8 * cap)); CK(D.bcnt.ensure(8));
    CK(cudaMemcpyAsync(D.a.p, pr->a, 8 * (size_t)m * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(D.d.p, pr->d, 8 * (size_t)m, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(D.bcnt.p, 0, 8, st));
    BruteArgs ba{D.a.as<uint64_t>(), D.d.as<uint64_t>(), m, n, D.bcnt.as<unsigned long long>(), D.bout.as<uint64_t>(), cap};
    launch_brute(ba, st);
    ++launches;
    CK(cudaGetLastError());
    unsigned long long cnt = 0;
    CK(cudaMemcpyAsync(&cnt, D.bcnt.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (cnt > cap) { cap = cnt; continue; }
    std::vector<uint64_t> enc(cnt);
    if (cnt) CK(cudaMemcpy(enc.data(), D.bout.p, 8 * cnt, cudaMemcpyDeviceToHost));
    std::sort(enc.begin(), enc.end());
    for (uint64_t e : enc) {
      std::vector<uint8_t> x(n);
      for (int j = 0; j < n; ++j) x[j] = (e >> (n - 1 - j)) & 1;
      sols.push_back(std::move(x));
    }
    return MSP_OK;
  }
  set_err("brute force result buffer overflow");
  return MSP_INTERNAL;
}

float elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) return 0;
  return ms;
}

uint32_t even_up(double x) { const uint32_t v = (uint32_t)x; return v + (v & 1u); }

// Capacity of a bucket region holding `mean` keys on average (multinomial spread: mean + 7 sigma)
// plus the key-0 pads of the scatter's even-length bulk-copy runs: every round of every chunk of
// the side pads each bucket at most once, about half of the time.  `side_keys` / `chunks`: the
// partitioned side's keys and work chunks (rounds hold >= ~1/3 of a stage).
uint32_t region_cap(double mean, double side_keys, double chunks) {
  const double rounds = side_keys / (kScatterStageKeys / 3.0) + chunks;
  return even_up(mean + 7.0 * std::sqrt(mean) + 16 + 0.5 * rounds + 4.0 * std::sqrt(rounds) + 16);
}

constexpr uint32_t kChunkCounters = 1u << 16;
// Level-1 coarse buckets of a huge batch side: at most 2^kCoarseBitsMax (each stage entry of the
// level-1 scatter then keeps >= 46 slots, so its runs stay long and its rank overflow rare)
#ifndef MSP_COARSE_BITS_MAX
#define MSP_COARSE_BITS_MAX 9
#endif
constexpr uint32_t kCoarseBitsMax = MSP_COARSE_BITS_MAX;
// Internal status: the hit list overflowed; msp_solve re-runs the (deterministic) solve with the
// grown list, as fastval.join_pairs regrows its output buffer (fastval.py:126-139).
constexpr int kRetryHits = 100;
// Tiles per scatter task of the persistent wave pipeline: a wave's tiles over about one task per SM
// (fewer, longer tasks: fewer partial rounds and task switches, every SM still scatters the wave),
// at least kTaskTilesMin.  MSP_TASK_TILES fixes it (tuning).
#ifndef MSP_TASK_TILES
#define MSP_TASK_TILES 0
#endif
constexpr uint64_t kTaskTiles = MSP_TASK_TILES;
constexpr uint64_t kTaskTilesMin = 96;
#ifndef MSP_L2_CHUNK
#define MSP_L2_CHUNK 65536
#endif
constexpr uint64_t kL2ChunkSlots = MSP_L2_CHUNK;  // slots of a coarse region per level-2 task (multiple of 32)
static_assert(kL2ChunkSlots % 32 == 0 && kL2ChunkSlots / 32 <= 0xFFFF, "level-2 chunk word");
#ifndef MSP_TASKS_PER_SM
#define MSP_TASKS_PER_SM 1
#endif

// Static split of a launch's tiles (units given as consecutive tile ranges [ub[i], ub[i+1])) over
// `nct` CTAs: CTA b gets tiles [b*T/nct, (b+1)*T/nct), cut at unit boundaries into chunks.
void static_chunks(const std::vector<uint64_t> &ub, uint32_t nct, std::vector<unsigned long long> &chunks,
                   std::vector<uint32_t> &first) {
  const uint64_t T = ub.back();
  size_t u = 0;
  for (uint32_t b = 0; b < nct; ++b) {
    first.push_back((uint32_t)chunks.size());
    uint64_t t = T * b / nct;
    const uint64_t te = T * (b + 1) / nct;
    while (t < te) {
      while (ub[u + 1] <= t) ++u;
      const uint64_t e = std::min<uint64_t>({te, ub[u + 1], t + 65535});
      chunks.push_back(t | ((e - t) << 32) | ((unsigned long long)u << 48));
      t = e;
    }
  }
  first.push_back((uint32_t)chunks.size());
}

int solve_impl(const msp_problem *pr, const msp_options *opt, msp_result *res) {
  const double t0 = now_s();
  memset(res, 0, sizeof(*res));
  if (!pr || !opt || !res) { set_err("null argument"); return MSP_INVALID_ARGUMENT; }
  res->n = pr->n;
  Device *Dp = nullptr;
  int rc = get_device(opt->device, &Dp, &res->stats.t_init);
  if (rc) return rc;
  Device &D = *Dp;
  std::lock_guard<std::mutex> lk(D.mu);
  CK(cudaSetDevice(D.dev));
  cudaStream_t st = opt->stream ? (cudaStream_t)opt->stream : D.stream;
  msp_stats &S = res->stats;
  std::vector<std::vector<uint8_t>> sols;
  const bool profile = opt->flags & MSP_FLAG_PROFILE;
  // MSP_TIMELINE: host time and stream time of the solve's phase boundaries (GPU idle = gaps)
  struct TLMark { const char *name; double host_ms; cudaEvent_t ev; };
  std::vector<TLMark> tl;
  const bool tl_on = getenv("MSP_TIMELINE") != nullptr;
  auto hmark = [&](const char *name) {  // host-only timestamp
    if (tl_on) fprintf(stderr, "[msp timeline]   %-16s host %8.3f ms\n", name, 1e3 * (now_s() - t0));
  };
  auto mark = [&](const char *name) {
    if (!tl_on) return;
    TLMark m{name, 1e3 * (now_s() - t0), nullptr};
    if (cudaEventCreate(&m.ev) == cudaSuccess && cudaEventRecord(m.ev, st) == cudaSuccess) tl.push_back(m);
  };
  const int bf_max = opt->brute_force_max_n < 0 ? 12 : opt->brute_force_max_n;
  auto emit = [&](void) -> int {
    res->n_solutions = (int64_t)sols.size();
    if (!sols.empty()) {
      res->xbits = (uint8_t *)malloc(sols.size() * (size_t)pr->n);
      for (size_t i = 0; i < sols.size(); ++i) memcpy(res->xbits + i * pr->n, sols[i].data(), pr->n);
    }
    S.t_total = now_s() - t0;
    return MSP_OK;
  };
  if (!(opt->flags & MSP_FLAG_FORCE_TABLE_PATH) && pr->n <= bf_max) {
    CK(cudaEventRecord(D.ev[0], st));
    rc = brute_force(D, pr, st, sols, S.kernel_launches);
    if (rc) return rc;
    CK(cudaEventRecord(D.ev[1], st));
    CK(cudaEventSynchronize(D.ev[1]));
    S.dev_ms_total = elapsed_ms(D.ev[0], D.ev[1]);
    if (opt->mode == MSP_MODE_FIRST && sols.size() > 1) sols.resize(1);
    S.fallback = 1;
    S.exact_hits = (int64_t)sols.size();
    return emit();
  }
  Plan P;
  rc = check_instance(pr, P);
  if (rc) return rc;
  const double deadline = opt->time_limit_s > 0 ? t0 + opt->time_limit_s : 0;
  // Watchdog: a host thread turns the deadline and the cross-rank cancel word into the device stop
  // word the running kernels poll (k_waves at every task switch, k_scatter per chunk) -- one async
  // copy on its own stream, which runs beside the kernels -- so a solve stops within one task instead
  // of at the next host checkpoint.
  *D.abort_h = 0;
  CK(D.abort_dev.ensure(64));
  CK(cudaMemsetAsync(D.abort_dev.p, 0, 4, st));
  struct Watchdog {
    std::atomic<bool> done{false};
    std::thread th;
    ~Watchdog() { done = true; if (th.joinable()) th.join(); }
  } wd;
  if (deadline > 0 || opt->cancel) {
    CK(cudaStreamSynchronize(st));  // (the stop word is zero before the watchdog can set it)
    volatile int *word = D.abort_h;
    const volatile int32_t *cancel = opt->cancel;
    int *dev_word = D.abort_dev.as<int>(), *one = D.abort_one;
    cudaStream_t wst = D.stream_wd;
    const int devno = D.dev;
    wd.th = std::thread([&wd, word, cancel, deadline, dev_word, one, wst, devno]() {
      while (!wd.done.load()) {
        int why = 0;
        if (deadline > 0 && now_s() > deadline) why = 1;
        else if (cancel && *cancel) why = 2;
        if (why) {
          *word = why;
          cudaSetDevice(devno);
          cudaMemcpyAsync(dev_word, one, 4, cudaMemcpyHostToDevice, wst);
          cudaStreamSynchronize(wst);
          return;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
      }
    });
  }
  // the stop word's verdict after a sync: timeout / cancelled / none
  auto stop_state = [&]() { return *D.abort_h; };
  CK(cudaEventRecord(D.ev[0], st));
  const uint64_t key_budget = opt->wave_keys ? std::max<uint64_t>(4096, opt->wave_keys) : kDefaultWaveKeys;
  double t_tables = 0;
  rc = build_plan(D, pr, P, opt->alpha_lo, opt->alpha_hi, st, S.kernel_launches, &t_tables);
  if (rc) return rc;
  CK(cudaGetLastError());
  CK(cudaEventRecord(D.ev[1], st));
  mark("plan done");
  S.t_build = t_tables - t0;
  S.t_enumerate = now_s() - t_tables;
  S.peak_table_entries = 0;
  for (int t = 0; t < 4; ++t) S.peak_table_entries += (int64_t)1 << P.b[t];
  S.peak_heap1 = (int64_t)1 << P.b[1];
  S.peak_heap2 = (int64_t)1 << P.b[3];
  S.batches = P.G;
  unsigned __int128 row1 = 0;
  for (uint32_t g = 0; g < P.G; ++g) {
    S.candidates_left += (int64_t)P.nl[g];
    S.candidates_right += (int64_t)P.nr[g];
    row1 += (unsigned __int128)P.nl[g] * P.nr[g];
  }
  S.row1_pairs_lo = (uint64_t)row1;
  S.row1_pairs_hi = (uint64_t)(row1 >> 64);
  if (deadline && now_s() > deadline) { set_err("time limit exceeded"); return MSP_TIMEOUT; }
  if (opt->cancel && *opt->cancel) {
    S.cancelled = 1;
    return emit();
  }

  // ---- per-batch counters, hit list
  const size_t G1 = std::max<size_t>(1, P.G);
  CK(D.bfilt.ensure(8 * G1));
  CK(D.bhits.ensure(8 * G1));
  CK(D.bovf.ensure(4 * G1));
  CK(cudaMemsetAsync(D.bfilt.p, 0, 8 * G1, st));
  CK(cudaMemsetAsync(D.bhits.p, 0, 8 * G1, st));
  CK(cudaMemsetAsync(D.bovf.p, 0, 4 * G1, st));
  CK(D.zkeys.ensure(16 * G1));
  CK(cudaMemsetAsync(D.zkeys.p, 0, 16 * G1, st));
  if (!D.hit_cap) {
    D.hit_cap = 1 << 20;
    if (const char *ev = getenv("MSP_HIT_CAP")) D.hit_cap = std::max<uint64_t>(16, strtoull(ev, nullptr, 10));  // (tests)
  }
  const uint64_t hit_cap = D.hit_cap;
  CK(D.hits.ensure(sizeof(HitRec) * hit_cap));
  CK(D.nhits.ensure(8));
  CK(D.nrecs.ensure(8));
  CK(cudaMemsetAsync(D.nhits.p, 0, 8, st));
  CK(cudaMemsetAsync(D.err.p, 0, 16, st));
  hmark("counters zeroed");
  JoinTable jt{};
  jt.hits = D.hits.as<HitRec>();
  jt.nhits = D.nhits.as<unsigned long long>();
  jt.hit_cap = hit_cap;
  jt.err = D.err.as<int>();
  P.base.key_mask = (opt->flags & MSP_FLAG_DEGENERATE_HASH) ? 0ull : ~0ull;  // (every k_enum launch)
  EnumArgs A = P.base;
  A.diag = (opt->flags & MSP_FLAG_DIAG_HASH_ONLY) ? 1u : 0u;
  A.batch_filtered = D.bfilt.as<unsigned long long>();
  A.batch_hits = D.bhits.as<unsigned long long>();
  double hot_ms = 0;
  const double t_join0 = now_s();
  uint64_t hits_done = 0;
  bool stopped = false;
  std::vector<uint8_t> dropped(P.G, 0);  // batches whose partitioned join overflowed

  bool fill_zeroed = false;  // wave fill counters (reset by k_join after each bucket)
  // Double-buffered waves: wave k scatters into buffer k&1 on `st` while wave k-1 joins on
  // stream2; ordering is carried by events (scatter k waits for join k-2, join k for scatter k).
  const bool overlap = !profile;  // (per-wave launch path and huge batches)
  auto join_streams = [&]() -> int {
    CK(cudaEventRecord(D.ev_x, D.stream2));
    CK(cudaStreamWaitEvent(st, D.ev_x, 0));
    return MSP_OK;
  };
  auto launch_pair = [&](size_t wi, auto &&scatter_fn, PartArgs &pa) -> int {
    const int buf = (int)(wi & 1);
    pa.scratch = D.scratch.as<unsigned long long>() + buf * D.wstride;
    pa.fill[0] = D.fill.as<uint32_t>() + buf * (2 * kMaxWaveBuckets);
    pa.fill[1] = pa.fill[0] + kMaxWaveBuckets;
    if (!overlap) {
      CK(scatter_fn(pa, st));
      CK(launch_join(pa, D.num_sms, st));
      return MSP_OK;
    }
    if (wi >= 2) CK(cudaStreamWaitEvent(st, D.ev_j[buf], 0));
    CK(scatter_fn(pa, st));
    CK(cudaEventRecord(D.ev_s[buf], st));
    CK(cudaStreamWaitEvent(D.stream2, D.ev_s[buf], 0));
    CK(launch_join(pa, D.num_sms, D.stream2));
    CK(cudaEventRecord(D.ev_j[buf], D.stream2));
    return MSP_OK;
  };
  // kWaveBuffers scratch buffers of >= scratch_keys keys each, and their fill counters (zeroed per
  // solve and after a reallocation; the joins reset them after every bucket)
  auto ensure_wave_buffers = [&](uint64_t scratch_keys) -> int {
    const uint64_t stride = (scratch_keys + kSinkSlots + 31) & ~31ull;
    if (stride > D.wstride || !D.scratch.p) {
      CK(D.scratch.ensure(8 * kWaveBuffers * stride));
      D.wstride = D.scratch.cap / (8 * kWaveBuffers) & ~31ull;
    }
    void *f0 = D.fill.p;
    CK(D.fill.ensure(4 * kWaveBuffers * 2 * kMaxWaveBuckets));
    if (f0 != D.fill.p || !fill_zeroed) {
      CK(cudaMemsetAsync(D.fill.p, 0, 4 * kWaveBuffers * 2 * kMaxWaveBuckets, st));
      fill_zeroed = true;
    }
    return MSP_OK;
  };
  // Recovery of a set of hit keys (validate.py:285-313): re-enumerate ONE side of each hit batch (the
  // one with fewer pairs) and emit its pairs whose key is a hit key; then, per recovered pair, find
  // the other side's pairs whose companion vector is exactly d minus the pair's (an X-entry x hash
  // lookup among the Y entries: k_lookup) -- a pair of the other side with the same key but another
  // vector is an FNV collision, which the join already counted and which confirms nothing.  The
  // exact pairs are confirmed on the host in 128-bit arithmetic.  When the one side yields more
  // than kLookupMaxTargets pairs (degenerate multiplicities), the other side is enumerated too and
  // every (left, right) pair of a hit key is compared, as before.  Own buffers: waves can resume.
  int64_t recovered_hh = 0;
  bool recovered_one_sided = false;
  constexpr size_t kLookupMaxTargets = 1u << 16;
  auto recover = [&](const std::vector<HitRec> &hv) -> int {
    if (hv.empty()) return MSP_OK;
    std::map<uint32_t, std::vector<uint64_t>> byg;
    for (const HitRec &h : hv) byg[h.gid].push_back(h.key);
    std::vector<UnitDesc> ru[2];  // [0]: each batch's side with fewer pairs, [1]: the other side
    uint64_t tb[2] = {0, 0};
    std::vector<unsigned long long> himg;
    uint64_t slots = 0;
    for (auto &kv : byg) {
      const uint32_t g = kv.first;
      std::vector<uint64_t> ks = kv.second;
      std::sort(ks.begin(), ks.end());
      ks.erase(std::unique(ks.begin(), ks.end()), ks.end());
      const uint32_t l2 = std::max<uint32_t>(6, pow2ceil(4 * ks.size()));
      const uint64_t cap = 1ull << l2;
      himg.resize(slots + cap, 0);
      bool has_zero = false;
      for (uint64_t k : ks) {
        if (k == 0) { has_zero = true; continue; }
        uint32_t sl = (uint32_t)((k * kGolden) >> (64 - l2));
        while (himg[slots + sl]) sl = (sl + 1) & (uint32_t)(cap - 1);
        himg[slots + sl] = k;
      }
      const int small = P.nl[g] <= P.nr[g] ? 0 : 1;
      for (int side = 0; side < 2; ++side) {
        const int pass = side == small ? 0 : 1;
        UnitDesc u = make_unit(P, g, side, tb[pass]);
        u.region_base = (uint32_t)slots;
        u.region_log2 = l2;
        u.flags = has_zero ? 1u : 0u;
        tb[pass] += P.tiles[2 * g + side];
        ru[pass].push_back(u);
      }
      slots += cap;
    }
    CK(D.rkeys.ensure(8 * std::max<uint64_t>(slots, 1)));
    CK(D.rfilt.ensure(8 * P.G));
    CK(D.rhits.ensure(8 * P.G));
    CK(cudaMemcpyAsync(D.rkeys.p, himg.data(), 8 * slots, cudaMemcpyHostToDevice, st));
    JoinTable rj = jt;
    rj.keys = D.rkeys.as<unsigned long long>();
    rj.nkeys = (uint32_t)slots;
    EnumArgs RA = P.base;
    RA.batch_filtered = D.rfilt.as<unsigned long long>();
    RA.batch_hits = D.rhits.as<unsigned long long>();
    std::vector<PairRec> recs;
    auto run_pass = [&](int pass) -> int {  // enumerate the units ru[pass], append their hit pairs
      if (ru[pass].empty()) return MSP_OK;
      CK(D.runits.ensure(sizeof(UnitDesc) * ru[pass].size()));
      CK(cudaMemcpyAsync(D.runits.p, ru[pass].data(), sizeof(UnitDesc) * ru[pass].size(), cudaMemcpyHostToDevice, st));
      uint64_t rec_cap = std::max<uint64_t>(4096, 4 * hv.size());
      for (int attempt = 0; attempt < 2; ++attempt) {
        CK(D.recs.ensure(sizeof(PairRec) * rec_cap));
        CK(cudaMemsetAsync(D.nrecs.p, 0, 8, st));
        rj.recs = D.recs.as<PairRec>();
        rj.nrecs = D.nrecs.as<unsigned long long>();
        rj.rec_cap = rec_cap;
        set_enum_range(RA, D.runits.as<UnitDesc>(), ru[pass].size(), tb[pass], D.num_sms);
        launch_enum(P.mcx, SINK_RECOVER, RA, rj, D.num_sms, st);
        ++S.kernel_launches;
        CK(cudaGetLastError());
        unsigned long long nr = 0;
        CK(cudaMemcpyAsync(&nr, D.nrecs.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (nr > rec_cap) { rec_cap = nr; continue; }
        const size_t r0 = recs.size();
        recs.resize(r0 + nr);
        if (nr) CK(cudaMemcpy(recs.data() + r0, D.recs.p, sizeof(PairRec) * nr, cudaMemcpyDeviceToHost));
        return MSP_OK;
      }
      set_err("hit recovery buffer overflow");
      return MSP_INTERNAL;
    };
    if (int r = run_pass(0)) return r;
    if (recs.size() > kLookupMaxTargets || getenv("MSP_RECOVER_TWO_SIDED")) {
      // degenerate multiplicities (or the test seam): both sides, all pairs of a hit key compared
      if (int r = run_pass(1)) return r;
      int64_t hh = 0;
      if (int r = confirm(pr, P, recs, sols, hh)) return r;
      recovered_hh += hh;
      return MSP_OK;
    }
    // targets per recovered pair: d minus its sums (128-bit; a negative row cannot be matched)
    const int m = P.m, n = P.n;
    std::vector<LookupTarget> tg[2];  // by the side to look up
    for (const PairRec &r : recs) {
      LookupTarget T{};
      bool ok = true;
      for (int i = 0; i < m && ok; ++i) {
        unsigned __int128 sum = 0;
        const uint32_t mk[2] = {r.xmask, r.ymask};
        for (int h = 0; h < 2; ++h) {
          const int t = 2 * (int)r.side + h;
          for (int b = 0; b < P.b[t]; ++b)
            if ((mk[h] >> b) & 1u) sum += pr->a[(size_t)i * n + P.start[t] + b];
        }
        if (sum > pr->d[i]) { ok = false; break; }
        const unsigned __int128 rem = (unsigned __int128)pr->d[i] - sum;
        if (i == 0) T.w0 = (uint64_t)rem;
        else if (rem > 0xFFFFFFFFu) ok = false;  // past any companion sum of two table entries
        else T.tc[i - 1] = (uint32_t)rem;
      }
      if (!ok) continue;
      T.key = r.key;
      T.gid = r.gid;
      T.side = 1u - r.side;
      tg[T.side].push_back(T);
    }
    const size_t nrec_side = recs.size();
    for (int o = 0; o < 2; ++o) {
      if (tg[o].empty()) continue;
      const int tx = 2 * o, ty = 2 * o + 1;
      LookupArgs la{};
      la.X = LookupTable{table_w(D, P, tx), D.comp[tx].as<uint32_t>(), table_m(D, P, tx), 1u << P.b[tx]};
      la.Y = LookupTable{table_w(D, P, ty), D.comp[ty].as<uint32_t>(), table_m(D, P, ty), 1u << P.b[ty]};
      la.log2 = (uint32_t)P.b[ty] + 1;
      la.sw = P.sw;
      la.nw = words_for(P.mcx);
      la.mc = m - 1;
      la.wide = P.wide ? 1 : 0;
      CK(D.vslots.ensure(4ull << la.log2));
      CK(cudaMemsetAsync(D.vslots.p, 0, 4ull << la.log2, st));
      launch_vhash_build(la, D.vslots.as<uint32_t>(), st);
      la.slots = D.vslots.as<uint32_t>();
      CK(D.ltg.ensure(sizeof(LookupTarget) * tg[o].size()));
      CK(cudaMemcpyAsync(D.ltg.p, tg[o].data(), sizeof(LookupTarget) * tg[o].size(), cudaMemcpyHostToDevice, st));
      la.tg = D.ltg.as<LookupTarget>();
      la.ntg = (uint32_t)tg[o].size();
      CK(D.lnout.ensure(8));
      uint64_t cap = std::max<uint64_t>(1024, 4 * tg[o].size());
      for (int attempt = 0;; ++attempt) {
        CK(D.lout.ensure(sizeof(PairRec) * cap));
        CK(cudaMemsetAsync(D.lnout.p, 0, 8, st));
        la.out = D.lout.as<PairRec>();
        la.nout = D.lnout.as<unsigned long long>();
        la.cap = cap;
        launch_lookup(la, st);
        S.kernel_launches += 2;
        CK(cudaGetLastError());
        unsigned long long no = 0;
        CK(cudaMemcpyAsync(&no, D.lnout.p, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (no > cap) {
          if (attempt) { set_err("hit lookup buffer overflow"); return MSP_INTERNAL; }
          cap = no;
          continue;
        }
        const size_t r0 = recs.size();
        recs.resize(r0 + no);
        if (no) CK(cudaMemcpy(recs.data() + r0, D.lout.p, sizeof(PairRec) * no, cudaMemcpyDeviceToHost));
        break;
      }
    }
    {  // recovered pairs with equal vectors share a target: keep each looked-up pair once
      auto lt = [](const PairRec &a, const PairRec &b) {
        return std::tie(a.gid, a.side, a.xidx, a.yidx) < std::tie(b.gid, b.side, b.xidx, b.yidx);
      };
      auto eq = [](const PairRec &a, const PairRec &b) {
        return a.gid == b.gid && a.side == b.side && a.xidx == b.xidx && a.yidx == b.yidx;
      };
      std::sort(recs.begin() + nrec_side, recs.end(), lt);
      recs.erase(std::unique(recs.begin() + nrec_side, recs.end(), eq), recs.end());
    }
    int64_t hh = 0;  // (counts only the exact pairs of the looked-up side: no hash-hit cross-check)
    if (int r = confirm(pr, P, recs, sols, hh)) return r;
    recovered_one_sided = true;
    return MSP_OK;
  };
  auto fetch_hits = [&](uint64_t from, uint64_t to, std::vector<HitRec> &out) -> int {
    out.clear();
    if (to <= from) return MSP_OK;
    std::vector<HitRec> hv(to - from);
    CK(cudaMemcpy(hv.data(), D.hits.as<HitRec>() + from, sizeof(HitRec) * hv.size(), cudaMemcpyDeviceToHost));
    for (const HitRec &h : hv) if (!dropped[h.gid]) out.push_back(h);
    return MSP_OK;
  };
  // Sync point: deadline, hit-list capacity and (first mode) early recovery.
  auto checkpoint = [&](bool &stop_now) -> int {
    if (int r0 = join_streams()) return r0;
    unsigned long long nh = 0;
    CK(cudaMemcpyAsync(&nh, D.nhits.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    if ((deadline && now_s() > deadline) || stop_state() == 1) { set_err("time limit exceeded"); return MSP_TIMEOUT; }
    if (nh > hit_cap) { D.hit_cap = 2 * nh; return kRetryHits; }  // regrow the hit list and re-run
    if ((opt->cancel && *opt->cancel) || stop_state() == 2) {  // another rank confirmed a solution (first mode)
      S.cancelled = 1;
      stop_now = true;
      return MSP_OK;
    }
    if (opt->mode == MSP_MODE_FIRST && nh > hits_done) {
      std::vector<HitRec> hv;
      int r2 = fetch_hits(hits_done, nh, hv);
      if (r2) return r2;
      r2 = recover(hv);
      if (r2) return r2;
      hits_done = nh;
      if (!sols.empty()) stop_now = true;
    }
    return MSP_OK;
  };
  // host checkpoints between pipeline segments: first mode only (its solutions are confirmed on the
  // host); deadlines and cancels reach the running kernels through the watchdog's stop word
  const bool periodic = opt->mode == MSP_MODE_FIRST;
  // asynchronous metadata upload through the pinned ring (wraps after a stream sync)
  auto upload = [&](void *dst, const void *src, size_t bytes) -> int {
    if (!bytes) return MSP_OK;
    constexpr size_t kRing = 64ull << 20;
    if (bytes > kRing) {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
      return MSP_OK;
    }
    if (!D.ring) {
      CK(cudaMallocHost(&D.ring, kRing));
      D.ring_cap = kRing;
      D.ring_off = 0;
    }
    if (D.ring_off + bytes > D.ring_cap) {  // every earlier copy out of the ring is done after this
      CK(cudaStreamSynchronize(st));
      D.ring_off = 0;
    }
    memcpy(D.ring + D.ring_off, src, bytes);
    CK(cudaMemcpyAsync(dst, D.ring + D.ring_off, bytes, cudaMemcpyHostToDevice, st));
    D.ring_off = (D.ring_off + bytes + 255) & ~(size_t)255;
    return MSP_OK;
  };
  // Room for `bytes` in the pinned upload ring, to be filled in place and sent with ring_send (no
  // staging copy); nullptr when the ring cannot hold it (the caller then uses upload).
  auto ring_take = [&](size_t bytes) -> char * {
    constexpr size_t kRing = 64ull << 20;
    if (!bytes || bytes > kRing) return nullptr;
    if (!D.ring) {
      if (cudaMallocHost(&D.ring, kRing) != cudaSuccess) { D.ring = nullptr; return nullptr; }
      D.ring_cap = kRing;
      D.ring_off = 0;
    }
    if (D.ring_off + bytes > D.ring_cap) {
      if (cudaStreamSynchronize(st) != cudaSuccess) return nullptr;
      D.ring_off = 0;
    }
    return reinterpret_cast<char *>(D.ring) + D.ring_off;
  };
  auto ring_send = [&](void *dst, size_t bytes) -> int {
    CK(cudaMemcpyAsync(dst, D.ring + D.ring_off, bytes, cudaMemcpyHostToDevice, st));
    D.ring_off = (D.ring_off + bytes + 255) & ~(size_t)255;
    return MSP_OK;
  };
  // buckets per role of one partitioned wave (scatter entries = 2x): fewer entries give longer
  // runs per round; MSP_WAVE_BUCKETS overrides for tuning
  uint32_t wave_buckets = kMaxWaveBuckets;
  unsigned long long *dbg_stats = nullptr;
  CK(D.cctr.ensure(4 * kChunkCounters));
  CK(cudaMemsetAsync(D.cctr.p, 0, 4 * kChunkCounters, st));
  D.cctr_next = 0;
  // a zeroed chunk counter for the next scatter launch (stream-ordered reuse after a wrap)
  auto take_counter = [&](unsigned int **out) -> int {
    if (D.cctr_next == kChunkCounters) {
      CK(cudaMemsetAsync(D.cctr.p, 0, 4 * kChunkCounters, st));
      D.cctr_next = 0;
    }
    *out = D.cctr.as<unsigned int>() + D.cctr_next++;
    return MSP_OK;
  };
  if (getenv("MSP_DEBUG_STATS")) {
    CK(D.dbg.ensure(3 * 128));
    CK(cudaMemsetAsync(D.dbg.p, 0, 3 * 128, st));
    dbg_stats = D.dbg.as<unsigned long long>();
  }
  if (const char *ev = getenv("MSP_WAVE_BUCKETS")) wave_buckets = (uint32_t)std::max(1, std::min(kMaxWaveBuckets, atoi(ev)));

  // Launches of the persistent wave pipeline (msp_part.cu k_waves) over `wds` (descriptors and
  // chunks already on the device in W): tasks S(0) S(1) J(0) S(2) J(1) ... J(last), one launch per
  // segment of waves (16 when checkpoints are due, else all).  `pairs` per wave for profiling.
  auto run_pipeline = [&](WavesArgs &W, const std::vector<WaveDesc> &wds, const std::vector<uint64_t> &pairs,
                          bool timed) -> int {
    CK(D.wctr.ensure(4 * (1 + 2 * wds.size())));
    CK(cudaMemsetAsync(D.wctr.p, 0, 4 * (1 + 2 * wds.size()), st));
    W.task_ctr = D.wctr.as<unsigned int>();
    W.abort_dev = D.abort_dev.as<int>();
    W.scat_done = W.task_ctr + 1;
    W.join_done = W.scat_done + wds.size();
    const size_t seg = periodic ? 16 : wds.size();
    for (size_t s0 = 0; s0 < wds.size() && !stopped; s0 += seg) {
      const size_t s1 = std::min(wds.size(), s0 + seg);
      // task list S(s0) S(s0+1) S(s0+2) J(s0) S(s0+3) J(s0+1) ... J(s1-1), written in place into the
      // pinned upload ring (ranges filled by index: no per-task push)
      size_t nt = 0;
      for (size_t w = s0; w < s1; ++w) nt += wds[w].nchunks + (wds[w].nb + kJoinGroup - 1) / kJoinGroup;
      unsigned long long *tasks = reinterpret_cast<unsigned long long *>(ring_take(8 * nt));
      std::vector<unsigned long long> &tv = D.h_tasks;
      if (!tasks) { tv.resize(nt); tasks = tv.data(); }
      size_t o = 0;
      auto put_join = [&](size_t w) {
        const unsigned long long hi = (1ull << 63) | ((unsigned long long)w << 32);
        for (uint32_t b = 0; b < wds[w].nb; b += kJoinGroup) tasks[o++] = hi | b;
      };
      for (size_t w = s0; w < s1; ++w) {
        const unsigned long long hi = (unsigned long long)w << 32, c0 = wds[w].chunk0;
        for (uint32_t c = 0; c < wds[w].nchunks; ++c) tasks[o + c] = hi | (c0 + c);
        o += wds[w].nchunks;
        if (w >= s0 + kWaveLookahead) put_join(w - kWaveLookahead);
      }
      for (size_t w = s1 > s0 + kWaveLookahead ? s1 - kWaveLookahead : s0; w < s1; ++w) put_join(w);
      hmark("task list built");
      CK(D.tasks.ensure(8 * nt));
      if (tasks == tv.data()) {
        if (int ru_ = upload(D.tasks.p, tasks, 8 * nt)) return ru_;
      } else if (int ru_ = ring_send(D.tasks.p, 8 * nt)) {
        return ru_;
      }
      hmark("task list uploaded");
      CK(cudaMemsetAsync(W.task_ctr, 0, 4, st));
      W.tasks = D.tasks.as<unsigned long long>();
      W.ntasks = (uint32_t)nt;
      if (profile && timed) CK(cudaEventRecord(D.pev[0], st));
      mark("k_waves launch");
      CK(launch_waves(P.mcx, W, D.num_sms, st));
      mark("k_waves returned");
      S.kernel_launches += 1;
      if (profile && timed) {
        CK(cudaEventRecord(D.pev[1], st));
        CK(cudaEventSynchronize(D.pev[1]));
        hot_ms += elapsed_ms(D.pev[0], D.pev[1]);
        S.hot_launches += 1;
        for (size_t w = s0; w < s1; ++w) S.hot_pairs += (int64_t)pairs[w];
      }
      if (periodic) {
        bool stop_now = false;
        const int r1 = checkpoint(stop_now);
        if (r1) return r1;
        if (stop_now) stopped = true;
      }
    }
    return MSP_OK;
  };
  auto pipeline_base = [&](WavesArgs &W) {
    W.scratch = D.scratch.as<unsigned long long>();
    W.scratch_stride = D.wstride;
    W.fill = D.fill.as<uint32_t>();
  };

  // ---- classify batches: partitioned shared-memory join (default) or global-table join
  std::vector<uint32_t> part_b, huge_b, global_b;
  for (uint32_t g = 0; g < P.G; ++g) {
    const uint64_t nb = std::min(P.nl[g], P.nr[g]), np = std::max(P.nl[g], P.nr[g]);
    const uint64_t nbk = std::max<uint64_t>(1, (nb + kBucketTargetMax - 1) / kBucketTargetMax);
    if (opt->flags & (MSP_FLAG_JOIN_GLOBAL | MSP_FLAG_DEGENERATE_HASH))
      global_b.push_back(g);
    else if (nbk > (uint64_t)std::min<uint32_t>(wave_buckets, kMaxUnitBuckets) || nb + np > key_budget)
      huge_b.push_back(g);
    else
      part_b.push_back(g);
  }

  hmark("classified");
  // ---- partitioned waves
  {
    struct PWave { size_t u0, u1, b0, nb; uint64_t t0, ntiles, scratch, pairs; uint32_t g0, g1; };
    std::vector<PWave> pw;
    std::vector<UnitDesc> &units = D.h_units;
    units.clear();
    std::vector<BucketRun> bruns;  // per batch: its buckets' regions (expanded on the device)
    uint32_t nbt_all = 0;
    PWave cur{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint64_t cur_keys = 0;
    // tile list of every partitioned batch side, in (batch, side) order
    std::vector<uint64_t> gs_tb(2 * (size_t)P.G, 0);
    std::vector<uint32_t> gs_unit(2 * (size_t)P.G, 0xFFFFFFFFu);
    uint64_t all_tiles = 0;
    auto flush = [&]() {
      if (cur.nb == 0) return;
      cur.u1 = units.size();
      pw.push_back(cur);
      cur = PWave{units.size(), units.size(), nbt_all, 0, all_tiles, 0, 0, 0, 0, 0};
      cur_keys = 0;
    };
    for (uint32_t g : part_b) {
      const int bside = P.nr[g] <= P.nl[g] ? 1 : 0;
      const uint64_t nb = bside ? P.nr[g] : P.nl[g], np = bside ? P.nl[g] : P.nr[g];
      const uint32_t NB = (uint32_t)std::max<uint64_t>(  // <= kMaxUnitBuckets by the classification
          1, std::min<uint64_t>(std::min<uint32_t>(wave_buckets, kMaxUnitBuckets), (nb + kBucketTarget - 1) / kBucketTarget));
      if (cur.nb + NB > wave_buckets || cur_keys + nb + np > key_budget ||
          (cur.nb && g != cur.g1) ||  // waves hold consecutive batches (contiguous tile ranges)
          units.size() - cur.u0 + 2 > (size_t)kMaxUnits) {
        flush();
      }
      if (cur.nb == 0) { cur.g0 = g; cur.t0 = all_tiles; }
      const double mb = (double)nb / NB, mp = (double)np / NB;
      // capacities even: bucket regions start 16-byte aligned for the scatter's bulk copies
      const double chb = (double)P.tiles[2 * (size_t)g + bside] / kTaskTilesMin + 2.0 * D.num_sms;
      const double chp = (double)P.tiles[2 * (size_t)g + 1 - bside] / kTaskTilesMin + 2.0 * D.num_sms;
      const uint32_t cb = region_cap(mb, (double)nb, chb), cp = region_cap(mp, (double)np, chp);
      // bucket k of the batch: build region at base + k(cb + cp), probe region right after it
      bruns.push_back(BucketRun{nbt_all, NB, (uint32_t)cur.scratch, cb, cp, g});
      cur.scratch += (uint64_t)NB * (cb + cp);
      nbt_all += NB;
      for (int side = 0; side < 2; ++side) {
        UnitDesc u = make_unit(P, g, side, 0);
        u.region_base = cur.nb;
        u.region_log2 = NB;
        u.flags = (side == bside ? 0u : 1u) << 1;  // role: 0 build, 1 probe
        const size_t gs = 2 * (size_t)g + side;
        gs_unit[gs] = (uint32_t)(units.size() - cur.u0);
        gs_tb[gs] = all_tiles;
        all_tiles += P.tiles[gs];
        cur.ntiles += P.tiles[gs];
        units.push_back(u);
      }
      cur.nb += NB;
      cur.g1 = g + 1;
      cur.pairs += P.nl[g] + P.nr[g];
      cur_keys += nb + np;
    }
    flush();
    if (all_tiles > 0xFFFFFFFFull) {  // WaveDesc.tile0 and the chunk words index tiles with 32 bits
      set_err("partitioned batches hold %llu warp tiles (> 2^32)", (unsigned long long)all_tiles);
      return MSP_UNSUPPORTED;
    }
    hmark("waves packed");
    S.waves += (int32_t)pw.size();
    if (!pw.empty()) {
      uint64_t max_scratch = 0;
      for (const PWave &w : pw) max_scratch = std::max(max_scratch, w.scratch);
      const size_t nbt = nbt_all;
      rc = ensure_wave_buffers(max_scratch);
      if (rc) return rc;
      std::vector<UnitInfo> uinfo(units.size());
      for (const PWave &w : pw)
        for (size_t i = w.u0; i < w.u1; ++i) uinfo[i] = make_info(units[i], (uint32_t)w.nb);
      CK(D.uinfo.ensure(sizeof(UnitInfo) * uinfo.size()));
      if (int ru_ = upload(D.uinfo.p, uinfo.data(), sizeof(UnitInfo) * uinfo.size())) return ru_;
      CK(D.bk.ensure(4 * 5 * nbt));
      CK(D.bruns.ensure(sizeof(BucketRun) * bruns.size()));
      if (int ru_ = upload(D.bruns.p, bruns.data(), sizeof(BucketRun) * bruns.size())) return ru_;
      launch_expand_buckets(D.bruns.as<BucketRun>(), (uint32_t)bruns.size(), D.bk.as<uint32_t>(), (uint32_t)nbt, st);
      ++S.kernel_launches;
      hmark("buckets uploaded");
      // per wave: each CTA's equal share of the wave's tiles, cut at unit boundaries
      const uint32_t nct = (uint32_t)D.num_sms * kScatterCtasHost;
      std::vector<unsigned long long> chimg;
      std::vector<uint32_t> cfirst;
      std::vector<size_t> choff, cfoff;
      const bool per_wave = opt->flags & MSP_FLAG_WAVE_LAUNCHES;
      for (const PWave &w : pw) {
        if (!per_wave) break;  // (static CTA chunks: per-wave launch path only)
        choff.push_back(chimg.size());
        cfoff.push_back(cfirst.size());
        std::vector<uint64_t> ub{0};
        for (size_t i = w.u0; i < w.u1; ++i) {
          const UnitDesc &u = units[i];
          ub.push_back(ub.back() + P.tiles[2 * (size_t)u.gid + u.side]);
        }
        std::vector<uint32_t> f;
        static_chunks(ub, nct, chimg, f);
        for (uint32_t &x : f) x -= (uint32_t)choff.back();
        cfirst.insert(cfirst.end(), f.begin(), f.end());
      }
      hmark("chunks built");
      CK(D.chunks.ensure(8 * std::max<size_t>(1, chimg.size())));
      if (int ru_ = upload(D.chunks.p, chimg.data(), 8 * chimg.size())) return ru_;
      CK(D.cfirst.ensure(4 * std::max<size_t>(1, cfirst.size())));
      if (int ru_ = upload(D.cfirst.p, cfirst.data(), 4 * cfirst.size())) return ru_;
      // K3b: every partitioned batch side's warp tiles, one launch
      CK(D.tdesc.ensure(sizeof(TileDesc) * std::max<uint64_t>(all_tiles, 1)));
      CK(D.gstb.ensure(8 * gs_tb.size()));
      CK(D.gsu.ensure(4 * gs_unit.size()));
      if (int ru_ = upload(D.gstb.p, gs_tb.data(), 8 * gs_tb.size())) return ru_;
      if (int ru_ = upload(D.gsu.p, gs_unit.data(), 4 * gs_unit.size())) return ru_;
      TileGenArgs tg{};
      tg.rects = P.base.rects;
      tg.rect_lo = 0;
      tg.rect_hi = P.rect_base.empty() ? 0 : P.rect_base.back() + P.nrect.back();
      tg.gs_tile_base = D.gstb.as<uint64_t>();
      tg.gs_unit = D.gsu.as<uint32_t>();
      tg.out = D.tdesc.as<TileDesc>();
      tg.tiles = all_tiles;
      mark("tiles launch");
      launch_tiles(tg, st);
      ++S.kernel_launches;
      const uint32_t *bkd = D.bk.as<uint32_t>();
      PartArgs pa{};
      pa.scratch = D.scratch.as<unsigned long long>();
      pa.fill[0] = D.fill.as<uint32_t>();
      pa.fill[1] = D.fill.as<uint32_t>() + kMaxWaveBuckets;
      pa.batch_ovf = D.bovf.as<unsigned int>();
      pa.zero_keys = D.zkeys.as<unsigned long long>();
      pa.dbg = dbg_stats;
      pa.hits = D.hits.as<HitRec>();
      pa.nhits = D.nhits.as<unsigned long long>();
      pa.hit_cap = hit_cap;
      pa.batch_hits = D.bhits.as<unsigned long long>();
      hmark("tiles launched");
      ScatterArgs sa = scatter_base(P, A);
        sa.abort_dev = D.abort_dev.as<int>();
      if (!per_wave) {  // one persistent launch per segment of waves (msp_part.cu k_waves)
        // task chunks (<= tt tiles of one unit each): counted per wave, then written in place into the
        // pinned upload ring
        std::vector<WaveDesc> wds(pw.size());
        std::vector<uint64_t> wtt(pw.size());
        size_t ntch = 0;
        for (size_t wi = 0; wi < pw.size(); ++wi) {
          const PWave &w = pw[wi];
          WaveDesc &wd = wds[wi];
          const uint64_t ntask = (uint64_t)D.num_sms * MSP_TASKS_PER_SM;
          const uint64_t tt = kTaskTiles ? kTaskTiles
                                         : std::min<uint64_t>(0xFFFF, std::max(kTaskTilesMin, (w.ntiles + ntask - 1) / ntask));
          wtt[wi] = tt;
          wd.tile0 = (uint32_t)w.t0;
          wd.chunk0 = (uint32_t)ntch;
          for (size_t i = w.u0; i < w.u1; ++i) ntch += (P.tiles[2 * (size_t)units[i].gid + units[i].side] + tt - 1) / tt;
          wd.nchunks = (uint32_t)(ntch - wd.chunk0);
          wd.unit0 = (uint32_t)w.u0;
          wd.b0 = (uint32_t)w.b0;
          wd.nb = (uint32_t)w.nb;
          wd.njoin = (uint32_t)((w.nb + kJoinGroup - 1) / kJoinGroup);
        }
        unsigned long long *tch = reinterpret_cast<unsigned long long *>(ring_take(8 * ntch));
        std::vector<unsigned long long> &tcv = D.h_tch;
        if (!tch) { tcv.resize(std::max<size_t>(1, ntch)); tch = tcv.data(); }
        for (size_t wi = 0, o = 0; wi < pw.size(); ++wi) {
          const PWave &w = pw[wi];
          const uint64_t tt = wtt[wi];
          uint64_t t = 0;
          for (size_t i = w.u0; i < w.u1; ++i) {
            const uint64_t nt = P.tiles[2 * (size_t)units[i].gid + units[i].side];
            const unsigned long long hi = (unsigned long long)(i - w.u0) << 48;
            for (uint64_t k = 0; k < nt; k += tt) tch[o++] = (t + k) | (std::min<uint64_t>(tt, nt - k) << 32) | hi;
            t += nt;
          }
        }
        hmark("task chunks built");
        CK(D.tchunks.ensure(8 * std::max<size_t>(1, ntch)));
        if (tch == tcv.data()) {
          if (int ru_ = upload(D.tchunks.p, tch, 8 * ntch)) return ru_;
        } else if (int ru_ = ring_send(D.tchunks.p, 8 * ntch)) {
          return ru_;
        }
        CK(D.wdesc.ensure(sizeof(WaveDesc) * wds.size()));
        if (int ru_ = upload(D.wdesc.p, wds.data(), sizeof(WaveDesc) * wds.size())) return ru_;
        rc = ensure_wave_buffers(max_scratch);
        if (rc) return rc;
        hmark("chunks uploaded");
        WavesArgs W{};
        W.sc = sa;
        W.sc.tiles = D.tdesc.as<TileDesc>();
        W.sc.units = D.uinfo.as<UnitInfo>();
        W.pa = pa;
        W.bstart0 = bkd; W.bstart1 = bkd + nbt; W.bcap0 = bkd + 2 * nbt; W.bcap1 = bkd + 3 * nbt; W.bgid = bkd + 4 * nbt;
        pipeline_base(W);
        W.waves = D.wdesc.as<WaveDesc>();
        W.chunks = D.tchunks.as<unsigned long long>();
        std::vector<uint64_t> wpairs;
        for (const PWave &w : pw) wpairs.push_back(w.pairs);
        rc = run_pipeline(W, wds, wpairs, true);
        if (rc) return rc;
      }
      for (size_t wi = 0; per_wave && wi < pw.size(); ++wi) {
        const PWave &w = pw[wi];
        pa.start[0] = bkd + w.b0;
        pa.start[1] = bkd + nbt + w.b0;
        pa.cap[0] = bkd + 2 * nbt + w.b0;
        pa.cap[1] = bkd + 3 * nbt + w.b0;
        pa.gid = bkd + 4 * nbt + w.b0;
        pa.nb = (uint32_t)w.nb;
        sa.tiles = D.tdesc.as<TileDesc>() + w.t0;
        sa.chunks = D.chunks.as<unsigned long long>() + choff[wi];
        sa.cta_first = D.cfirst.as<uint32_t>() + cfoff[wi];
        sa.nchunks = 1;  // (static mode: the launch runs a full grid)
        sa.units = D.uinfo.as<UnitInfo>() + w.u0;
        sa.nunits = (uint32_t)(w.u1 - w.u0);
        if (profile) CK(cudaEventRecord(D.pev[0], st));
        rc = launch_pair(wi, [&](const PartArgs &p2, cudaStream_t s2) { return launch_scatter(P.mcx, sa, p2, D.num_sms, s2); }, pa);
        if (rc) return rc;
        S.kernel_launches += 2;
        if (profile) {
          CK(cudaEventRecord(D.pev[1], st));
          CK(cudaEventSynchronize(D.pev[1]));
          hot_ms += elapsed_ms(D.pev[0], D.pev[1]);
          S.hot_launches += 2;
          S.hot_pairs += (int64_t)w.pairs;
        }
        if (periodic && (wi % 16 == 15 || wi + 1 == pw.size())) {
          bool stop_now = false;
          rc = checkpoint(stop_now);
          if (rc) return rc;
          if (stop_now) { stopped = true; break; }
        }
      }
    }
  }

  rc = join_streams();
  if (rc) return rc;

  // ---- huge batches: two-level partitioned join.  Level 1 hashes the batch once and partitions
  //      each side into <= 1024 coarse buckets in HBM (one k_scatter launch per side, so each
  //      side's region indices stay 32-bit); level 2 streams coarse buckets back, re-partitions
  //      them into fine buckets in the L2 scratch and joins them (k_rescatter + k_join).
  if (!stopped && !huge_b.empty()) {
    uint64_t kCoarseTarget = 2ull << 20;  // build keys per coarse bucket (MSP_COARSE_TARGET: tuning)
    if (const char *ev = getenv("MSP_COARSE_TARGET")) kCoarseTarget = std::max<uint64_t>(65536, strtoull(ev, nullptr, 10));
    CK(D.cfill.ensure(4 * 2 * kMaxWaveBuckets));
    {  // size the big per-batch buffers once for the largest batch (a regrowth stalls the stream)
      uint64_t mcb = 0, mcp = 0, mt = 0;
      for (uint32_t g : huge_b) {
        const int bs = P.nr[g] <= P.nl[g] ? 1 : 0;
        const uint64_t nb = bs ? P.nr[g] : P.nl[g], np = bs ? P.nl[g] : P.nr[g];
        uint32_t cbits = pow2ceil((nb + kCoarseTarget - 1) / kCoarseTarget);
        cbits = std::max<uint32_t>(1, std::min<uint32_t>(cbits, kCoarseBitsMax));
        const double mb = (double)nb / (1u << cbits), mp = (double)np / (1u << cbits);
        mcb = std::max<uint64_t>(mcb, (uint64_t)region_cap(mb, (double)nb, 4.0 * D.num_sms) << cbits);
        mcp = std::max<uint64_t>(mcp, (uint64_t)region_cap(mp, (double)np, 4.0 * D.num_sms) << cbits);
        mt = std::max<uint64_t>(mt, std::max(P.tiles[2 * (size_t)g], P.tiles[2 * (size_t)g + 1]));
      }
      {  // the coarse regions of the largest batch must fit next to everything else
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        const uint64_t need = 8 * (mcb + mcp + 2 * kSinkSlots), have = free_b + D.cscratch[0].cap + D.cscratch[1].cap;
        if (need > have) {
          set_err("largest batch needs %.1f GB of coarse scratch, %.1f GB available", need / 1e9, have / 1e9);
          return MSP_UNSUPPORTED;
        }
      }
      CK(D.cscratch[0].ensure(8 * (mcb + kSinkSlots)));
      CK(D.cscratch[1].ensure(8 * (mcp + kSinkSlots)));
      CK(D.tdesc.ensure(sizeof(TileDesc) * std::max<uint64_t>(1, mt)));
      rc = ensure_wave_buffers(2 * key_budget + 4 * kMaxWaveBuckets * 64ull);
      if (rc) return rc;
    }
    for (size_t hi_ = 0; hi_ < huge_b.size() && !stopped; ++hi_) {
      if (stop_state()) { stopped = true; break; }  // deadline / cancel (reported after the sync)
      rc = join_streams();  // the previous batch's joins still read the wave buffers
      if (rc) return rc;
      const uint32_t g = huge_b[hi_];
      const int bside = P.nr[g] <= P.nl[g] ? 1 : 0;
      const uint64_t nb = bside ? P.nr[g] : P.nl[g], np = bside ? P.nl[g] : P.nr[g];
      uint32_t cbits = pow2ceil((nb + kCoarseTarget - 1) / kCoarseTarget);
      cbits = std::max<uint32_t>(1, std::min<uint32_t>(cbits, kCoarseBitsMax));
      const uint32_t NC = 1u << cbits;
      const double mb = (double)nb / NC, mp = (double)np / NC;
      const uint64_t cb = region_cap(mb, (double)nb, 4.0 * D.num_sms), cp = region_cap(mp, (double)np, 4.0 * D.num_sms);
      if (cb * NC > 0xFFFFFFF0ull || cp * NC > 0xFFFFFFF0ull) {
        set_err("batch side too large for 32-bit coarse regions");
        return MSP_UNSUPPORTED;
      }
      // coarse bucket arrays: start[0] | start[1] | cap[0] | cap[1] | gid
      std::vector<uint32_t> cbk(5 * (size_t)NC);
      for (uint32_t c = 0; c < NC; ++c) {
        cbk[c] = (uint32_t)(c * cb);
        cbk[NC + c] = (uint32_t)(c * cp);
        cbk[2 * NC + c] = (uint32_t)cb;
        cbk[3 * NC + c] = (uint32_t)cp;
        cbk[4 * NC + c] = g;
      }
      CK(D.cscratch[0].ensure(8 * (cb * NC + kSinkSlots)));
      CK(D.cscratch[1].ensure(8 * (cp * NC + kSinkSlots)));
      CK(D.cbk.ensure(4 * cbk.size()));
      if (int ru_ = upload(D.cbk.p, cbk.data(), 4 * cbk.size())) return ru_;
      CK(cudaMemsetAsync(D.cfill.p, 0, 4 * 2 * kMaxWaveBuckets, st));
      UnitDesc lu[2];
      uint64_t ltiles[2];
      for (int side = 0; side < 2; ++side) {
        const uint32_t role = side == bside ? 0u : 1u;
        lu[role] = make_unit(P, g, side, 0);
        lu[role].region_base = 0;
        lu[role].region_log2 = NC;
        lu[role].flags = 0;  // each side is scattered by its own launch as role 0 (roles = 1)
        lu[role].count_filter = side == 1;
        ltiles[role] = P.tiles[2 * g + side];
      }
      UnitInfo li[2] = {make_info(lu[0], NC), make_info(lu[1], NC)};
      CK(D.hunits.ensure(sizeof(UnitInfo) * 2));
      if (int ru_ = upload(D.hunits.p, li, sizeof(UnitInfo) * 2)) return ru_;
      const uint32_t *cbkd = D.cbk.as<uint32_t>();
      PartArgs c1{};
      c1.gid = cbkd + 4 * NC;
      c1.nb = NC;
      c1.roles = 1;
      std::vector<unsigned long long> cch;  // level-1 chunks (static split): role 0's, then role 1's
      std::vector<uint32_t> ccf;
      const uint32_t nct = (uint32_t)D.num_sms * kScatterCtasHost;
      static_chunks({0, ltiles[0]}, nct, cch, ccf);
      const size_t cch1 = cch.size(), ccf1 = ccf.size();
      {
        std::vector<uint32_t> f;
        static_chunks({0, ltiles[1]}, nct, cch, f);
        for (uint32_t &x : f) x -= (uint32_t)cch1;
        ccf.insert(ccf.end(), f.begin(), f.end());
      }
      CK(D.cchunks.ensure(8 * std::max<size_t>(1, cch.size())));
      if (int ru_ = upload(D.cchunks.p, cch.data(), 8 * cch.size())) return ru_;
      CK(D.ccfirst.ensure(4 * ccf.size()));
      if (int ru_ = upload(D.ccfirst.p, ccf.data(), 4 * ccf.size())) return ru_;
      c1.batch_ovf = D.bovf.as<unsigned int>();
      c1.zero_keys = D.zkeys.as<unsigned long long>();
      c1.dbg = dbg_stats ? dbg_stats + 16 : nullptr;
      if (profile) CK(cudaEventRecord(D.pev[0], st));
      mark("huge: level 1");
      CK(D.tdesc.ensure(sizeof(TileDesc) * std::max<uint64_t>(1, std::max(ltiles[0], ltiles[1]))));
      for (int role = 0; role < 2; ++role) {
        const int side = role == 0 ? bside : 1 - bside;
        const size_t gs = 2 * (size_t)g + side;
        TileGenArgs tg{};
        tg.rects = P.base.rects;
        tg.rect_lo = P.rect_base[gs];
        tg.rect_hi = P.rect_base[gs] + P.nrect[gs];
        tg.out = D.tdesc.as<TileDesc>();
        tg.tiles = P.tiles[gs];
        launch_tiles(tg, st);
        c1.scratch = D.cscratch[role].as<unsigned long long>();
        c1.start[0] = cbkd + role * NC;
        c1.cap[0] = cbkd + (2 + role) * NC;
        c1.fill[0] = D.cfill.as<uint32_t>() + role * kMaxWaveBuckets;
        ScatterArgs sa = scatter_base(P, A);
        sa.abort_dev = D.abort_dev.as<int>();
        sa.tiles = D.tdesc.as<TileDesc>();
        sa.chunks = D.cchunks.as<unsigned long long>() + (role ? cch1 : 0);
        sa.cta_first = D.ccfirst.as<uint32_t>() + (role ? ccf1 : 0);
        sa.nchunks = 1;
        sa.units = D.hunits.as<UnitInfo>() + role;
        sa.nunits = 1;
        CK(launch_scatter(P.mcx, sa, c1, D.num_sms, st));
        S.kernel_launches += 2;
      }
      // level 2 waves over the coarse buckets
      hmark("L1 launched");
      mark("huge: level 2 setup");
      const uint32_t NF = (uint32_t)std::max<uint64_t>(1, (uint64_t)std::ceil(mb / kBucketTargetMax));
      if (NF > (uint32_t)kMaxUnitBuckets) { set_err("coarse bucket too large for one level-2 wave"); return MSP_UNSUPPORTED; }
      const double fmb = mb / NF, fmp = mp / NF;
      // level-2 sources: one coarse region per role, read in kL2ChunkSlots-slot chunks
      const uint32_t fcb = region_cap(fmb, (double)cb, (double)cb / kL2ChunkSlots + 2), fcp = region_cap(fmp, (double)cp, (double)cp / kL2ChunkSlots + 2);
      struct L2Wave { size_t s0, ns, b0, nb; uint64_t total, scratch; };
      std::vector<L2Wave> lw;
      std::vector<RescatterSrc> srcs;
      std::vector<uint32_t> fst0, fst1, fcap0, fcap1, fgid;
      L2Wave cw{0, 0, 0, 0, 0, 0};
      for (uint32_t c = 0; c < NC; ++c) {
        if (cw.nb && (cw.nb + NF > (uint32_t)kMaxWaveBuckets || cw.total + cb + cp > key_budget)) {
          lw.push_back(cw);
          cw = L2Wave{srcs.size(), 0, fgid.size(), 0, 0, 0};
        }
        for (int role = 0; role < 2; ++role) {
          RescatterSrc r{};
          r.keys = D.cscratch[role].as<unsigned long long>() + (size_t)c * (role ? cp : cb);
          r.fill = D.cfill.as<uint32_t>() + role * kMaxWaveBuckets + c;
          r.cap = (uint32_t)(role ? cp : cb);
          r.role = role;
          r.fine_base = (uint32_t)cw.nb;
          r.nf = NF;
          r.nc = NC;
          r.in_base = cw.total;
          cw.total += r.cap;
          srcs.push_back(r);
          cw.ns++;
        }
        for (uint32_t k = 0; k < NF; ++k) {
          fst0.push_back((uint32_t)cw.scratch); fcap0.push_back(fcb); cw.scratch += fcb;
          fst1.push_back((uint32_t)cw.scratch); fcap1.push_back(fcp); cw.scratch += fcp;
          fgid.push_back(g);
        }
        cw.nb += NF;
      }
      lw.push_back(cw);
      const size_t nft = fgid.size();
      uint64_t max_scr = 0;
      for (const L2Wave &w : lw) max_scr = std::max(max_scr, w.scratch);
      std::vector<uint32_t> fimg;
      fimg.reserve(5 * nft);
      for (auto *v : {&fst0, &fst1, &fcap0, &fcap1, &fgid}) fimg.insert(fimg.end(), v->begin(), v->end());
      rc = ensure_wave_buffers(max_scr);
      if (rc) return rc;
      CK(D.l2bk.ensure(4 * fimg.size()));
      CK(D.l2src.ensure(sizeof(RescatterSrc) * srcs.size()));
      if (int ru_ = upload(D.l2bk.p, fimg.data(), 4 * fimg.size())) return ru_;
      if (int ru_ = upload(D.l2src.p, srcs.data(), sizeof(RescatterSrc) * srcs.size())) return ru_;
      const uint32_t *fb = D.l2bk.as<uint32_t>();
      PartArgs pa{};
      pa.scratch = D.scratch.as<unsigned long long>();
      pa.fill[0] = D.fill.as<uint32_t>();
      pa.fill[1] = D.fill.as<uint32_t>() + kMaxWaveBuckets;
      pa.batch_ovf = D.bovf.as<unsigned int>();
      pa.zero_keys = D.zkeys.as<unsigned long long>();
      pa.dbg = dbg_stats ? dbg_stats + 32 : nullptr;
      pa.hits = D.hits.as<HitRec>();
      pa.nhits = D.nhits.as<unsigned long long>();
      pa.hit_cap = hit_cap;
      pa.batch_hits = D.bhits.as<unsigned long long>();
      std::vector<unsigned long long> l2ch;  // per wave: kL2ChunkSlots-slot chunks of each source region
      std::vector<size_t> l2off;
      for (const L2Wave &w : lw) {
        l2off.push_back(l2ch.size());
        for (size_t si = 0; si < w.ns; ++si) {
          const uint64_t cap = srcs[w.s0 + si].cap;
          for (uint64_t o = 0; o < cap; o += kL2ChunkSlots) {
            const uint64_t grp = std::min<uint64_t>(kL2ChunkSlots / 32, (cap - o + 31) / 32);
            l2ch.push_back(o | (grp << 32) | ((unsigned long long)si << 48));
          }
        }
      }
      l2off.push_back(l2ch.size());
      hmark("L2 lists built");
      CK(D.l2chunks.ensure(8 * std::max<size_t>(1, l2ch.size())));
      if (int ru_ = upload(D.l2chunks.p, l2ch.data(), 8 * l2ch.size())) return ru_;
      if (!(opt->flags & MSP_FLAG_WAVE_LAUNCHES)) {  // level-2 waves through the persistent pipeline
        rc = join_streams();  // (the previous batch's joins may still read the wave buffers)
        if (rc) return rc;
        rc = ensure_wave_buffers(max_scr);
        if (rc) return rc;
        std::vector<WaveDesc> wds(lw.size());
        for (size_t wi = 0; wi < lw.size(); ++wi) {
          WaveDesc &wd = wds[wi];
          wd.kind = 1;
          wd.chunk0 = (uint32_t)l2off[wi];
          wd.nchunks = (uint32_t)(l2off[wi + 1] - l2off[wi]);
          wd.src0 = (uint32_t)lw[wi].s0;
          wd.b0 = (uint32_t)lw[wi].b0;
          wd.nb = (uint32_t)lw[wi].nb;
          wd.njoin = (uint32_t)((lw[wi].nb + kJoinGroup - 1) / kJoinGroup);
        }
        CK(D.wdesc.ensure(sizeof(WaveDesc) * wds.size()));
        if (int ru_ = upload(D.wdesc.p, wds.data(), sizeof(WaveDesc) * wds.size())) return ru_;
        WavesArgs W{};
        W.sc = scatter_base(P, A);
        W.pa = pa;
        W.bstart0 = fb; W.bstart1 = fb + nft; W.bcap0 = fb + 2 * nft; W.bcap1 = fb + 3 * nft; W.bgid = fb + 4 * nft;
        pipeline_base(W);
        W.waves = D.wdesc.as<WaveDesc>();
        W.srcs = D.l2src.as<RescatterSrc>();
        W.fetch_ahead = 1;  // level-2 tasks have no scatter -> join order to upset (measured -0.3%)
        if (const char *ev = getenv("MSP_L2_FETCH_AHEAD")) W.fetch_ahead = (uint32_t)atoi(ev);
        W.chunks = D.l2chunks.as<unsigned long long>();
        hmark("L2 pipeline start");
        rc = run_pipeline(W, wds, std::vector<uint64_t>(lw.size(), 0), false);  // (timed per batch below)
        hmark("L2 pipeline queued");
        if (rc) return rc;
      }
      for (size_t wi = 0; (opt->flags & MSP_FLAG_WAVE_LAUNCHES) && wi < lw.size(); ++wi) {
        const L2Wave &w = lw[wi];

        pa.start[0] = fb + w.b0;
        pa.start[1] = fb + nft + w.b0;
        pa.cap[0] = fb + 2 * nft + w.b0;
        pa.cap[1] = fb + 3 * nft + w.b0;
        pa.gid = fb + 4 * nft + w.b0;
        pa.nb = (uint32_t)w.nb;
        RescatterArgs ra{};
        ra.src = D.l2src.as<RescatterSrc>() + w.s0;
        ra.chunks = D.l2chunks.as<unsigned long long>() + l2off[wi];
        ra.nchunks = (uint32_t)(l2off[wi + 1] - l2off[wi]);
        if (int r0 = take_counter(&ra.chunk_ctr)) return r0;
        rc = launch_pair(wi, [&](const PartArgs &p2, cudaStream_t s2) { return launch_rescatter(ra, p2, D.num_sms, s2); }, pa);
        if (rc) return rc;
        S.kernel_launches += 2;
      }
      S.waves += (int32_t)lw.size() + 1;
      if (profile) {
        CK(cudaEventRecord(D.pev[1], st));
        CK(cudaEventSynchronize(D.pev[1]));
        hot_ms += elapsed_ms(D.pev[0], D.pev[1]);
        S.hot_launches += 2 + 2 * (int64_t)lw.size();
        S.hot_pairs += (int64_t)(P.nl[g] + P.nr[g]);
      }
      if (periodic) {
        bool stop_now = false;
        rc = checkpoint(stop_now);
        if (rc) return rc;
        if (stop_now) stopped = true;
      }
    }
  }

  rc = join_streams();
  if (rc) return rc;
  mark("joins queued");

  // ---- overflowed partitioned batches are re-joined with the global table.  The per-batch totals
  //      are read back in the same round trip: without global-table batches they are final.
  unsigned long long n_v2_hits = 0;
  std::vector<unsigned long long> bf(P.G), bh(P.G), zk(2 * (size_t)P.G);
  unsigned long long nh = 0;
  int err = 0;
  bool totals_read = false;
  // pinned layout: bf | bh | zk (2G) | ovf (G x 4 B) | nh | n_v2_hits | err
  const size_t G8 = 8 * (size_t)P.G;
  unsigned char *pin = D.pinned(4 * G8 + 4 * (size_t)P.G + 32);
  if (!pin) { set_err("cudaMallocHost failed"); return MSP_CUDA_ERROR; }
  unsigned long long *p_nh = reinterpret_cast<unsigned long long *>(pin + 4 * G8 + ((4 * (size_t)P.G + 7) & ~(size_t)7));
  unsigned long long *p_nv2 = p_nh + 1;
  int *p_err = reinterpret_cast<int *>(p_nh + 2);
  auto read_totals = [&]() -> int {
    CK(cudaEventRecord(D.ev[2], st));
    if (P.G) {
      CK(cudaMemcpyAsync(pin, D.bfilt.p, G8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(pin + G8, D.bhits.p, G8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(pin + 2 * G8, D.zkeys.p, 2 * G8, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(p_nh, D.nhits.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(p_err, D.err.p, 4, cudaMemcpyDeviceToHost, st));
    return MSP_OK;
  };
  auto take_totals = [&]() {  // after the stream synchronised
    if (P.G) {
      memcpy(bf.data(), pin, G8);
      memcpy(bh.data(), pin + G8, G8);
      memcpy(zk.data(), pin + 2 * G8, 2 * G8);
    }
    nh = *p_nh;
    err = *p_err;
  };
  if (!stopped && (!part_b.empty() || !huge_b.empty())) {
    std::vector<uint32_t> ovf(P.G);
    if (P.G) CK(cudaMemcpyAsync(pin + 4 * G8, D.bovf.p, 4 * (size_t)P.G, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(p_nv2, D.nhits.p, 8, cudaMemcpyDeviceToHost, st));
    if (global_b.empty()) {
      if (int r_ = read_totals()) return r_;
      totals_read = true;
    }
    CK(cudaStreamSynchronize(st));
    if (P.G) memcpy(ovf.data(), pin + 4 * G8, 4 * (size_t)P.G);
    n_v2_hits = *p_nv2;
    if (totals_read) take_totals();
    if (stop_state()) stopped = true;  // the kernels stopped early: nothing left to re-join
    for (uint32_t g = 0; g < P.G && !stopped; ++g) {
      if (!ovf[g]) continue;
      totals_read = false;  // the re-joined batches change them
      dropped[g] = 1;
      global_b.push_back(g);
      CK(cudaMemsetAsync(D.bfilt.as<unsigned long long>() + g, 0, 8, st));
      CK(cudaMemsetAsync(D.bhits.as<unsigned long long>() + g, 0, 8, st));
    }
    std::sort(global_b.begin(), global_b.end());
  }

  // ---- global-table waves (huge batches by hash-range passes; overflow fallback)
  if (!stopped && !global_b.empty()) {
    const uint64_t slot_budget = opt->wave_keys ? std::max<uint64_t>(1024, 2 * opt->wave_keys) : (1ull << 23);
    std::vector<UnitDesc> units;
    std::vector<Wave> waves;
    Wave cur;
    uint64_t tb_build = 0, tb_probe = 0;
    std::vector<UnitDesc> pend_build, pend_probe;
    auto flush = [&]() {
      if (pend_build.empty()) return;
      cur.ub0 = units.size();
      units.insert(units.end(), pend_build.begin(), pend_build.end());
      cur.ub1 = units.size();
      cur.up0 = units.size();
      units.insert(units.end(), pend_probe.begin(), pend_probe.end());
      cur.up1 = units.size();
      cur.build_tiles = tb_build;
      cur.probe_tiles = tb_probe;
      waves.push_back(cur);
      cur = Wave();
      pend_build.clear();
      pend_probe.clear();
      tb_build = tb_probe = 0;
    };
    for (uint32_t g : global_b) {
      const int bside = P.nr[g] <= P.nl[g] ? 1 : 0;
      const uint64_t nb = bside ? P.nr[g] : P.nl[g];
      const uint64_t need = 1ull << std::max<uint32_t>(6, pow2ceil(2 * nb));
      uint32_t npass = 1;
      uint64_t cap = need;
      if (need > slot_budget) {
        npass = (uint32_t)((2 * nb + slot_budget - 1) / slot_budget);
        do {
          ++npass;
          cap = 1ull << std::max<uint32_t>(6, pow2ceil((uint64_t)(2.2 * (double)nb / npass) + 64));
        } while (cap > slot_budget);
        flush();
      }
      for (uint32_t p = 0; p < npass; ++p) {
        if (npass == 1 && cur.slots + cap > slot_budget) flush();
        UnitDesc ub = make_unit(P, g, bside, tb_build);
        UnitDesc up = make_unit(P, g, 1 - bside, tb_probe);
        for (UnitDesc *u : {&ub, &up}) {
          u->slot = cur.nslot;
          u->region_base = (uint32_t)cur.slots;
          u->region_log2 = pow2ceil(cap);
          u->pass = p;
          u->npass = npass;
          u->count_filter = (u->side == 1 && p == 0);
        }
        tb_build += P.tiles[2 * g + bside];
        tb_probe += P.tiles[2 * g + 1 - bside];
        cur.pairs += P.nl[g] + P.nr[g];
        pend_build.push_back(ub);
        pend_probe.push_back(up);
        cur.slots += cap;
        cur.nslot++;
        if (npass > 1) flush();
      }
    }
    flush();
    S.waves += (int32_t)waves.size();
    uint32_t max_nslot = 1;
    uint64_t max_slots = 64;
    for (const Wave &w : waves) { max_nslot = std::max(max_nslot, w.nslot); max_slots = std::max(max_slots, w.slots); }
    CK(D.units.ensure(sizeof(UnitDesc) * std::max<size_t>(1, units.size())));
    CK(D.keys.ensure(8 * max_slots));
    {
      void *before = D.cnt.p;
      CK(D.cnt.ensure(8 * max_slots));
      if (D.cnt.p != before) {  // fresh memory: no stale tag may look like a live epoch
        CK(cudaMemsetAsync(D.cnt.p, 0, D.cnt.cap, st));
        D.epoch = 0;
      }
    }
    CK(D.zero.ensure(8 * max_nslot));
    CK(D.zhit.ensure(4 * max_nslot));
    CK(cudaMemcpyAsync(D.units.p, units.data(), sizeof(UnitDesc) * units.size(), cudaMemcpyHostToDevice, st));
    jt.keys = D.keys.as<unsigned long long>();
    jt.cnt = D.cnt.as<unsigned long long>();
    jt.zero = D.zero.as<unsigned long long>();
    jt.zero_hit = D.zhit.as<unsigned int>();
    const UnitDesc *udev = D.units.as<UnitDesc>();
    for (size_t wi = 0; wi < waves.size(); ++wi) {
      if (stop_state()) { stopped = true; break; }
      const Wave &w = waves[wi];
      launch_clear(D.keys.p, 8 * w.slots, D.num_sms, st);
      if (++D.epoch >= (1ull << 24)) {  // tag space exhausted: clear and restart
        CK(cudaMemsetAsync(D.cnt.p, 0, D.cnt.cap, st));
        D.epoch = 1;
      }
      jt.epoch = D.epoch;
      CK(cudaMemsetAsync(D.zero.p, 0, 8 * w.nslot, st));
      CK(cudaMemsetAsync(D.zhit.p, 0, 4 * w.nslot, st));
      if (profile) CK(cudaEventRecord(D.pev[0], st));
      set_enum_range(A, udev + w.ub0, w.ub1 - w.ub0, w.build_tiles, D.num_sms);
      const bool diag = opt->flags & MSP_FLAG_DIAG_HASH_ONLY;
      if (launch_enum(P.mcx, diag ? SINK_NONE : SINK_BUILD, A, jt, D.num_sms, st)) { set_err("unsupported m"); return MSP_INTERNAL; }
      set_enum_range(A, udev + w.up0, w.up1 - w.up0, w.probe_tiles, D.num_sms);
      launch_enum(P.mcx, diag ? SINK_NONE : SINK_PROBE, A, jt, D.num_sms, st);
      S.kernel_launches += 2;
      if (profile) {
        CK(cudaEventRecord(D.pev[1], st));
        CK(cudaEventSynchronize(D.pev[1]));
        hot_ms += elapsed_ms(D.pev[0], D.pev[1]);
        S.hot_launches += 2;
        S.hot_pairs += (int64_t)w.pairs;
      }
      if (periodic && (wi % 16 == 15 || wi + 1 == waves.size())) {
        bool stop_now = false;
        rc = checkpoint(stop_now);
        if (rc) return rc;
        if (stop_now) { stopped = true; break; }
      }
    }
  }

  // ---- totals
  if (!totals_read || stopped) {
    if (int r_ = read_totals()) return r_;
    CK(cudaStreamSynchronize(st));
    take_totals();
  }
  S.t_validate = now_s() - t_join0;
  S.dev_ms_tables = elapsed_ms(D.ev[0], D.ev[1]);
  S.dev_ms_join = elapsed_ms(D.ev[1], D.ev[2]);
  S.dev_ms_hot = hot_ms;
  S.hot_bytes = 8 * S.hot_pairs;  // algorithmic bytes: one 64-bit key written or read per candidate pair
  if (err) { set_err("join table region overflow (err=%d)", err); return MSP_INTERNAL; }
  // real zero keys never reach the partitioned join (0 pads the runs): their hash hits are the
  // per-batch product, and key 0 joins the recovery set (global-table batches count their own
  // zeros and never touch zkeys)
  std::vector<HitRec> zero_hits;
  for (uint32_t g = 0; g < P.G; ++g) {
    const unsigned long long zz = dropped[g] ? 0ull : zk[2 * (size_t)g] * zk[2 * (size_t)g + 1];
    if (zz) { bh[g] += zz; zero_hits.push_back(HitRec{g, 0u, 0ull}); }
  }
  for (uint32_t g = 0; g < P.G; ++g) { S.filtered_residuals += (int64_t)bf[g]; S.hash_hits += (int64_t)bh[g]; }
  if ((opt->flags & MSP_FLAG_BATCH_STATS) && P.G) {  // per-batch ValidationStats (validate.py:63-71)
    res->batch_stats = (int64_t *)malloc(sizeof(int64_t) * 5 * (size_t)P.G);
    if (!res->batch_stats) { set_err("out of host memory"); return MSP_INTERNAL; }
    res->n_batch_stats = P.G;
    for (uint32_t g = 0; g < P.G; ++g) {
      int64_t *r = res->batch_stats + 5 * (size_t)g;
      r[0] = (int64_t)P.alpha[g]; r[1] = (int64_t)P.nl[g]; r[2] = (int64_t)P.nr[g];
      r[3] = (int64_t)bf[g]; r[4] = (int64_t)bh[g];
    }
  }
  if (stop_state() == 1 || (deadline && now_s() > deadline)) { set_err("time limit exceeded"); return MSP_TIMEOUT; }
  if (stop_state() == 2) {  // cancelled mid-solve by another rank: counters are partial
    S.cancelled = 1;
    return emit();
  }
  if (nh > hit_cap) { D.hit_cap = 2 * nh; return kRetryHits; }  // regrow the hit list and re-run
  if (!stopped) {
    // hits recorded by the partitioned join of dropped batches are superseded by their re-join
    std::vector<HitRec> hv;
    rc = fetch_hits(hits_done, n_v2_hits > hits_done ? n_v2_hits : hits_done, hv);
    if (rc) return rc;
    std::vector<HitRec> tail(0);
    if (nh > std::max<uint64_t>(hits_done, n_v2_hits)) {
      const uint64_t from = std::max<uint64_t>(hits_done, n_v2_hits);
      std::vector<HitRec> t2(nh - from);
      CK(cudaMemcpy(t2.data(), D.hits.as<HitRec>() + from, sizeof(HitRec) * t2.size(), cudaMemcpyDeviceToHost));
      hv.insert(hv.end(), t2.begin(), t2.end());
    }
    hv.insert(hv.end(), zero_hits.begin(), zero_hits.end());
    mark("recovery start");
    rc = recover(hv);
    if (rc) return rc;
    mark("recovery done");
    if (opt->mode == MSP_MODE_ALL && !recovered_one_sided && recovered_hh != S.hash_hits) {
      set_err("internal error: recovered hash hits %lld != join hash hits %lld", (long long)recovered_hh,
              (long long)S.hash_hits);
      return MSP_INTERNAL;
    }
  }
  CK(cudaEventRecord(D.ev[3], st));
  CK(cudaEventSynchronize(D.ev[3]));
  for (const TLMark &m : tl) {
    float g = 0;
    cudaEventElapsedTime(&g, D.ev[0], m.ev);
    fprintf(stderr, "[msp timeline] %-18s host %8.3f ms  stream %8.3f ms\n", m.name, m.host_ms, g);
    cudaEventDestroy(m.ev);
  }
  if (tl_on) fprintf(stderr, "[msp timeline] %-18s host %8.3f ms  stream %8.3f ms\n", "end", 1e3 * (now_s() - t0),
                     elapsed_ms(D.ev[0], D.ev[3]));
  if (dbg_stats) {
    unsigned long long dva[48];
    CK(cudaMemcpy(dva, dbg_stats, 3 * 128, cudaMemcpyDeviceToHost));
    for (int blk = 1; blk < 3; ++blk)
      fprintf(stderr, "[msp dbg] %s: rounds %llu staged %llu overflow %llu spilled %llu capacity-overflow %llu; "
              "SM-ms (pipeline) scatter %.1f join %.1f wait %.1f + %.1f, join phases %.1f / %.1f\n",
              blk == 1 ? "level-1 scatter" : "level-2", dva[16 * blk], dva[16 * blk + 1], dva[16 * blk + 2],
              dva[16 * blk + 13], dva[16 * blk + 12], dva[16 * blk + 4] / 1.965e6, dva[16 * blk + 5] / 1.965e6,
              dva[16 * blk + 6] / 1.965e6, dva[16 * blk + 7] / 1.965e6, dva[16 * blk + 8] / 1.965e6, dva[16 * blk + 9] / 1.965e6);
    unsigned long long *dv = dva;
    int nov = 0;
    for (uint32_t g = 0; g < P.G; ++g) nov += dropped[g];
    fprintf(stderr, "[msp dbg] scatter rounds %llu staged %llu overflow %llu; keys/round %.0f; overflowed batches %d of %u; "
            "SM-ms scatter %.1f join %.1f (incl. waits: joins for their scatters %.1f, scatters for their buffer %.1f)\n",
            dv[0], dv[1], dv[2], dv[0] ? (double)dv[1] / dv[0] : 0.0, nov, P.G, dv[4] / 1.965e6, dv[5] / 1.965e6,
            dv[6] / 1.965e6, dv[7] / 1.965e6);
    fprintf(stderr, "[msp dbg] join buckets %llu: build phase %.1f SM-ms, probe phase %.1f SM-ms, mean stash %.2f\n",
            dv[11], dv[8] / 1.965e6, dv[9] / 1.965e6, dv[11] ? (double)dv[10] / dv[11] : 0.0);
    fprintf(stderr, "[msp dbg] overflow events: region capacity %llu, spilled keys %llu, join stash %llu\n",
            dv[12], dv[13], dv[14]);
  }
  S.dev_ms_total = elapsed_ms(D.ev[0], D.ev[3]);
  S.exact_hits = (int64_t)sols.size();
  if (opt->mode == MSP_MODE_FIRST && sols.size() > 1) sols.resize(1);
  return emit();
}

}  // namespace
}  // namespace msp

// ====================================================================== C-ABI

extern "C" {

int msp_solve(const msp_problem *prob, const msp_options *opt, msp_result *res) {
  try {
    int rc = msp::solve_impl(prob, opt, res);
    for (int attempt = 0; rc == msp::kRetryHits && attempt < 8; ++attempt) {
      msp_result_free(res);
      rc = msp::solve_impl(prob, opt, res);
    }
    if (rc == msp::kRetryHits) { msp::set_err("hit list regrowth did not converge"); rc = MSP_INTERNAL; }
    if (rc && res) msp_result_free(res);
    return rc;
  } catch (const std::exception &e) {
    msp::set_err("exception: %s", e.what());
    return MSP_INTERNAL;
  }
}

void msp_result_free(msp_result *res) {
  if (!res) return;
  free(res->xbits);
  res->xbits = nullptr;
  res->n_solutions = 0;
  free(res->batch_stats);
  res->batch_stats = nullptr;
  res->n_batch_stats = 0;
}

int msp_join_alpha(const msp_problem *prob, const msp_options *opt, uint64_t alpha, msp_result *res) {
  if (!opt) { msp::set_err("null options"); return MSP_INVALID_ARGUMENT; }
  msp_options o = *opt;
  o.alpha_lo = alpha;
  o.alpha_hi = alpha + 1;
  o.mode = MSP_MODE_ALL;
  o.flags |= MSP_FLAG_FORCE_TABLE_PATH;
  return msp_solve(prob, &o, res);
}

int64_t msp_alpha_plan(const msp_problem *prob, int32_t device, int64_t max_batches, uint64_t *alpha,
                       uint64_t *beta, uint64_t *n_left, uint64_t *n_right) {
  using namespace msp;
  Device *D = nullptr;
  int rc = get_device(device, &D);
  if (rc) return -rc;
  std::lock_guard<std::mutex> lk(D->mu);
  if (cudaSetDevice(D->dev) != cudaSuccess) return -MSP_CUDA_ERROR;
  Plan P;
  rc = check_instance(prob, P);
  if (rc) return -rc;
  int64_t launches = 0;
  rc = build_plan(*D, prob, P, 0, 0, D->stream, launches);
  if (rc) return -rc;
  for (uint32_t g = 0; g < P.G && (int64_t)g < max_batches; ++g) {
    alpha[g] = P.alpha[g];
    beta[g] = P.target - P.alpha[g];
    n_left[g] = P.nl[g];
    n_right[g] = P.nr[g];
  }
  return P.G;
}

int msp_build_tables(const msp_problem *prob, int32_t device, uint64_t **weights, uint32_t **masks,
                     uint64_t **contribs, int64_t **run_end) {
  using namespace msp;
  Device *D = nullptr;
  int rc = get_device(device, &D);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(D->mu);
  CK(cudaSetDevice(D->dev));
  Plan P;
  rc = check_instance(prob, P);
  if (rc) return rc;
  int64_t launches = 0;
  rc = build_plan(*D, prob, P, 0, 0, D->stream, launches);
  if (rc) return rc;
  const int m = P.m;
  for (int t = 0; t < 4; ++t) {
    const size_t sz = (size_t)1 << P.b[t];
    std::vector<uint32_t> comp(sz * P.sw);
    CK(cudaMemcpy(weights[t], table_w(*D, P, t), 8 * sz, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(masks[t], table_m(*D, P, t), 4 * sz, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(comp.data(), D->comp[t].p, 4 * sz * P.sw, cudaMemcpyDeviceToHost));
    for (size_t e = 0; e < sz; ++e) {
      contribs[t][e * m] = weights[t][e];
      for (int c = 0; c < P.mc; ++c)
        contribs[t][e * m + 1 + c] = P.wide ? comp[e * P.sw + c] : (comp[e * P.sw + (c >> 1)] >> (16 * (c & 1))) & 0xFFFFu;
    }
    int64_t end = (int64_t)sz;
    for (int64_t i = (int64_t)sz - 1; i >= 0; --i) {
      if (i + 1 < (int64_t)sz && weights[t][i] != weights[t][i + 1]) end = i + 1;
      run_end[t][i] = end;
    }
  }
  return MSP_OK;
}

void msp_release(int32_t device) {
  std::lock_guard<std::mutex> lk(msp::g_devices_mu);
  auto it = msp::g_devices.find(device);
  if (it == msp::g_devices.end()) return;
  {
    std::lock_guard<std::mutex> lk2(it->second->mu);
    cudaSetDevice(device);
    it->second->release_all();
  }
}

const char *msp_last_error(void) { return msp::g_err.c_str(); }
void msp_abi_sizes(int32_t *out) {
  out[0] = (int32_t)sizeof(msp_problem);
  out[1] = (int32_t)sizeof(msp_options);
  out[2] = (int32_t)sizeof(msp_stats);
  out[3] = (int32_t)sizeof(msp_result);
}
int32_t msp_version(void) { return 1; }

}  // extern "C"
