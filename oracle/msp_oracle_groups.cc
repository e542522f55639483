// msp_oracle_groups.cc -- CPU oracle for ONE alpha-group of a large instance (TEST INFRASTRUCTURE).
//
// The reference validates a batch with validate_chunked -> fastval.join_pairs (validate.py:316-379,
// fastval.py:47-108): every left pair (A idx, B idx) of the batch and every right pair (C idx,
// D idx) whose residual d - s does not overshoot are hashed with the 64-bit FNV fold over all m
// coordinates (validate.py:34-60); every (left, right) pair with equal hashes is a hash hit, and the
// hits whose residual vectors are equal are the solutions (_confirm_hits, validate.py:285-313).
//
// The reference (and oracle_solve in msp_oracle.c) materialise the batch's pair arrays (16 B per
// pair) and a bucket-chain index (16 B per left pair): ~45 GB for the largest (9,80) batches, out of
// reach of this container.  This restatement computes the same counters without materialising
// pairs: the batch is the union of rectangles A-run(alpha - w) x B-run(w) and C-run(beta - w) x
// D-run(w), keys are generated per rectangle (threads over rectangles), and the join
// runs in P hash-range passes (pass p keeps the keys whose top bits equal p: every key lives in
// exactly one pass) as a sort-merge equi-join -- the count of equal-key (left, right) pairs is the
// reference's hash_hits by definition.  Exact confirmation re-enumerates the pairs whose key is a
// hit key.  Pinned against oracle_solve's per-batch records and the reference-generated alpha-group
// goldens (tests/test_oracle.py).
//
// oracle_groups_run(..., method 1) computes the same counters by a FILTER JOIN, fast enough to run
// every batch of a (9,80) instance on this container's 8 cores: left keys set a bit in a map indexed
// by their top bits; right keys that hit a set bit are the candidates (kept, sorted); candidates set
// a second map indexed by their low bits; left keys that hit it are the survivors (kept, sorted); the
// sort-merge of survivors against candidates counts every equal-key (left, right) pair.  A pair with
// equal keys always passes both maps, so the count is exact (the maps only drop pairs whose keys
// differ).  Pinned against method 0 and the reference-generated goldens (tests/test_oracle.py).
#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

extern "C" {
void oracle_block_sizes(int n, int32_t out[4]);
int oracle_build_tables(int m, int n, const uint64_t *a, int row, uint64_t **weights, uint64_t **masks,
                        uint64_t **contribs, int64_t **run_end);
}

namespace {

constexpr uint64_t kOffset = 0xCBF29CE484222325ull;  // validate.py:34
constexpr uint64_t kPrime = 0x100000001B3ull;         // validate.py:35

struct Table {
  int b = 0, start = 0;
  int64_t size = 0;
  std::vector<uint64_t> w, mask, contrib;  // contrib: size x m
  std::vector<int64_t> run_end;
};

struct Rect { int64_t x0, xn, y0, yn; };  // X-run [x0, x0+xn) x Y-run [y0, y0+yn)

// Rectangles X-run(total - w) x Y-run(w) over the distinct weights w of Y (enumerate1d.py:241-310
// restated: a batch holds every pair whose row-0 weights sum to total).
std::vector<Rect> rects_for(const Table &X, const Table &Y, uint64_t total) {
  std::unordered_map<uint64_t, std::pair<int64_t, int64_t>> xr;
  for (int64_t i = 0; i < X.size; i = X.run_end[i]) xr[X.w[i]] = {i, X.run_end[i] - i};
  std::vector<Rect> out;
  for (int64_t j = 0; j < Y.size; j = Y.run_end[j]) {
    const uint64_t wy = Y.w[j];
    if (wy > total) continue;
    auto it = xr.find(total - wy);
    if (it == xr.end()) continue;
    out.push_back(Rect{it->second.first, it->second.second, j, Y.run_end[j] - j});
  }
  return out;
}

struct Ctx {
  int m = 0, n = 0;
  const uint64_t *d = nullptr;
  Table t[4];
  uint64_t alpha = 0, beta = 0;
  std::vector<Rect> left, right;
  int threads = 1;
};

// Key of left pair (i in A, j in B): FNV over v = cA[i] + cB[j] (fastval.py:66-74).
inline uint64_t left_key(const Ctx &c, int64_t i, int64_t j) {
  const uint64_t *va = &c.t[0].contrib[(size_t)i * c.m], *vb = &c.t[1].contrib[(size_t)j * c.m];
  uint64_t h = kOffset;
  for (int k = 0; k < c.m; ++k) h = (h ^ (va[k] + vb[k])) * kPrime;
  return h;
}

// Key of right pair (i in C, j in D): FNV over d - (cC[i] + cD[j]); false when some coordinate
// overshoots d (filtered, fastval.py:83-99).
inline bool right_key(const Ctx &c, int64_t i, int64_t j, uint64_t &h) {
  const uint64_t *vc = &c.t[2].contrib[(size_t)i * c.m], *vd = &c.t[3].contrib[(size_t)j * c.m];
  h = kOffset;
  for (int k = 0; k < c.m; ++k) {
    const uint64_t s = vc[k] + vd[k];
    if (s > c.d[k]) return false;
    h = (h ^ (c.d[k] - s)) * kPrime;
  }
  return true;
}

// right_key without the per-coordinate early exit (the overshoot test is folded into one flag, so
// the loop has no data-dependent branch); same key and verdict.
inline bool right_key_flat(const Ctx &c, int64_t i, int64_t j, uint64_t &h) {
  const uint64_t *vc = &c.t[2].contrib[(size_t)i * c.m], *vd = &c.t[3].contrib[(size_t)j * c.m];
  uint64_t x = kOffset;
  bool over = false;
  for (int k = 0; k < c.m; ++k) {
    const uint64_t s = vc[k] + vd[k];
    over |= s > c.d[k];
    x = (x ^ (c.d[k] - s)) * kPrime;
  }
  h = x;
  return !over;
}

// Runs fn(thread, rect) over the rectangles with dynamic scheduling.
template <class F>
void for_rects(const std::vector<Rect> &rs, int threads, F &&fn) {
  std::atomic<size_t> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t)
    th.emplace_back([&, t]() {
      for (size_t r = next.fetch_add(1); r < rs.size(); r = next.fetch_add(1)) fn(t, rs[r]);
    });
  for (auto &x : th) x.join();
}

// Sort of keys that share their top `pbits` bits: one counting-scatter pass on the next 10 bits,
// then the 1024 buckets sorted by `threads` threads.
void psort(std::vector<uint64_t> &v, int pbits, int threads) {
  if (v.size() < 1u << 16) { std::sort(v.begin(), v.end()); return; }
  const int shift = 64 - pbits - 10;
  std::vector<size_t> cnt(1025, 0);
  for (uint64_t k : v) cnt[((k >> shift) & 1023) + 1]++;
  for (int i = 0; i < 1024; ++i) cnt[i + 1] += cnt[i];
  std::vector<uint64_t> tmp(v.size());
  {
    std::vector<size_t> pos(cnt.begin(), cnt.end() - 1);
    for (uint64_t k : v) tmp[pos[(k >> shift) & 1023]++] = k;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t)
    th.emplace_back([&]() {
      for (int b = next.fetch_add(1); b < 1024; b = next.fetch_add(1)) std::sort(tmp.begin() + cnt[b], tmp.begin() + cnt[b + 1]);
    });
  for (auto &x : th) x.join();
  v.swap(tmp);
}

}  // namespace

extern "C" {
typedef struct {
  int64_t n_left, n_right, filtered, hash_hits, exact_hits;
  int64_t passes;
  int64_t n_hit_keys;
  uint64_t *hit_keys;      // distinct keys with at least one (left, right) full-hash-equal pair
  int64_t n_solutions;
  uint8_t *xbits;          // n_solutions x n
} oracle_group_result;
}

namespace {

// Byte maps of the filter join: one anonymous mapping (huge pages where the kernel gives them),
// grown on demand and zeroed by all threads before each use.
struct ByteMap {
  uint8_t *p = nullptr;
  size_t bytes = 0;
  ~ByteMap() { if (p) munmap(p, bytes); }
  bool reserve(size_t want) {
    if (want <= bytes) return true;
    if (p) munmap(p, bytes);
    p = nullptr;
    bytes = 0;
    void *q = mmap(nullptr, want, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (q == MAP_FAILED) return false;
    madvise(q, want, MADV_HUGEPAGE);
    p = (uint8_t *)q;
    bytes = want;
    return true;
  }
  void clear(size_t used, int threads) {
    std::vector<std::thread> th;
    const size_t per = (used + threads - 1) / threads;
    for (int t = 0; t < threads; ++t)
      th.emplace_back([=]() {
        const size_t lo = std::min(used, per * t), hi = std::min(used, lo + per);
        if (hi > lo) memset(p + lo, 0, hi - lo);
      });
    for (auto &x : th) x.join();
  }
};

// An instance's tables, shared by every alpha-group run on it.
struct Groups {
  Ctx c;
  std::vector<uint64_t> d;
  ByteMap map;
};

// Sort-merge count of equal keys of two sorted vectors: hash_hits += |L(k)| x |R(k)| per key k.
void merge_count(const std::vector<uint64_t> &L, const std::vector<uint64_t> &R, int64_t &hash_hits,
                 std::vector<uint64_t> &hits) {
  size_t i = 0, j = 0;
  while (i < L.size() && j < R.size()) {
    if (L[i] < R[j]) { ++i; continue; }
    if (R[j] < L[i]) { ++j; continue; }
    const uint64_t k = L[i];
    size_t i1 = i, j1 = j;
    while (i1 < L.size() && L[i1] == k) ++i1;
    while (j1 < R.size() && R[j1] == k) ++j1;
    hash_hits += (int64_t)((i1 - i) * (j1 - j));
    hits.push_back(k);
    i = i1;
    j = j1;
  }
}

std::vector<uint64_t> concat(std::vector<std::vector<uint64_t>> &parts) {
  std::vector<uint64_t> v;
  size_t n = 0;
  for (auto &x : parts) n += x.size();
  v.reserve(n);
  for (auto &x : parts) { v.insert(v.end(), x.begin(), x.end()); std::vector<uint64_t>().swap(x); }
  return v;
}

// Method 0: P hash-range passes (pass p keeps the keys whose top bits equal p), each a sort-merge.
void join_sortmerge(Ctx &c, int passes, oracle_group_result *out, std::vector<uint64_t> &hits) {
  int P = passes;
  if (P <= 0) {
    const int64_t big = std::max(out->n_left, out->n_right);
    P = 1;
    while (big / P > 400000000ll) P *= 2;
  }
  int pbits = 0;
  while ((1 << pbits) < P) ++pbits;
  P = 1 << pbits;
  out->passes = P;
  auto part = [pbits](uint64_t k) -> uint64_t { return pbits ? k >> (64 - pbits) : 0; };
  std::atomic<int64_t> filtered{0};
  for (int p = 0; p < P; ++p) {
    std::vector<std::vector<uint64_t>> lk(c.threads), rk(c.threads);
    for_rects(c.left, c.threads, [&](int t, const Rect &r) {
      for (int64_t j = r.y0; j < r.y0 + r.yn; ++j)
        for (int64_t i = r.x0; i < r.x0 + r.xn; ++i) {
          const uint64_t k = left_key(c, i, j);
          if (part(k) == (uint64_t)p) lk[t].push_back(k);
        }
    });
    for_rects(c.right, c.threads, [&](int t, const Rect &r) {
      int64_t f = 0;
      for (int64_t j = r.y0; j < r.y0 + r.yn; ++j)
        for (int64_t i = r.x0; i < r.x0 + r.xn; ++i) {
          uint64_t k;
          if (!right_key(c, i, j, k)) { ++f; continue; }
          if (part(k) == (uint64_t)p) rk[t].push_back(k);
        }
      if (p == 0) filtered += f;
    });
    std::vector<uint64_t> L = concat(lk), R = concat(rk);
    psort(L, pbits, c.threads);
    psort(R, pbits, c.threads);
    merge_count(L, R, out->hash_hits, hits);
  }
  out->filtered = filtered;
}

// A hashed pair: key and the pair's table indices (i in X, j in Y).
struct Hit { uint64_t key; int64_t i, j; };

// Exact confirmation (validate.py:285-313) of the pairs whose key is a hit key: residuals compared in
// full; equal residual vectors are solutions, the rest full-hash collisions.
void confirm_pairs(const Ctx &c, const std::vector<Hit> &lh, const std::vector<Hit> &rh,
                   std::vector<uint64_t> &hits, oracle_group_result *out) {
  const int m = c.m, n = c.n;
  std::vector<uint8_t> xs;
  for (const Hit &l : lh)
    for (const Hit &r : rh) {
      if (l.key != r.key) continue;
      bool eq = true;
      for (int k = 0; k < m && eq; ++k) {
        const uint64_t v = c.t[0].contrib[(size_t)l.i * m + k] + c.t[1].contrib[(size_t)l.j * m + k];
        const uint64_t s = c.t[2].contrib[(size_t)r.i * m + k] + c.t[3].contrib[(size_t)r.j * m + k];
        eq = v == c.d[k] - s;
      }
      if (!eq) continue;  // full-hash collision
      const uint64_t mk[4] = {c.t[0].mask[l.i], c.t[1].mask[l.j], c.t[2].mask[r.i], c.t[3].mask[r.j]};
      std::vector<uint8_t> x(n, 0);
      for (int t = 0; t < 4; ++t)
        for (int b = 0; b < c.t[t].b; ++b) x[c.t[t].start + b] = (mk[t] >> b) & 1u;
      xs.insert(xs.end(), x.begin(), x.end());
      out->exact_hits++;
    }
  out->n_solutions = out->exact_hits;
  if (!xs.empty()) {
    out->xbits = (uint8_t *)malloc(xs.size());
    memcpy(out->xbits, xs.data(), xs.size());
  }
  std::sort(hits.begin(), hits.end());
  out->n_hit_keys = (int64_t)hits.size();
  if (!hits.empty()) {
    out->hit_keys = (uint64_t *)malloc(8 * hits.size());
    memcpy(out->hit_keys, hits.data(), 8 * hits.size());
  }
}

// Method 0's confirmation: re-enumerates both sides for the pairs whose key is a hit key.
void confirm(const Ctx &c, std::vector<uint64_t> &hits, oracle_group_result *out) {
  std::sort(hits.begin(), hits.end());
  std::vector<Hit> lh, rh;
  std::mutex mu;
  auto is_hit = [&](uint64_t k) { return std::binary_search(hits.begin(), hits.end(), k); };
  if (!hits.empty()) {
    for_rects(c.left, c.threads, [&](int, const Rect &r) {
      for (int64_t j = r.y0; j < r.y0 + r.yn; ++j)
        for (int64_t i = r.x0; i < r.x0 + r.xn; ++i) {
          const uint64_t k = left_key(c, i, j);
          if (is_hit(k)) { std::lock_guard<std::mutex> g(mu); lh.push_back(Hit{k, i, j}); }
        }
    });
    for_rects(c.right, c.threads, [&](int, const Rect &r) {
      for (int64_t j = r.y0; j < r.y0 + r.yn; ++j)
        for (int64_t i = r.x0; i < r.x0 + r.xn; ++i) {
          uint64_t k;
          if (right_key(c, i, j, k) && is_hit(k)) { std::lock_guard<std::mutex> g(mu); rh.push_back(Hit{k, i, j}); }
        }
    });
  }
  confirm_pairs(c, lh, rh, hits, out);
}

// Method 1: filter join (see the header), with bit maps: the power of two >= 16 bits per left key
// (<= 6.25% of right keys survive the first map), capped at 2^35 bits; the second map has the same
// size.  Candidates and survivors keep their pair indices,
// so the confirmation needs no third enumeration.
constexpr int kProbe = 32;  // keys hashed before their map bytes are read (the loads overlap)

std::vector<Hit> concat_hits(std::vector<std::vector<Hit>> &parts) {
  std::vector<Hit> v;
  size_t n = 0;
  for (auto &x : parts) n += x.size();
  v.reserve(n);
  for (auto &x : parts) { v.insert(v.end(), x.begin(), x.end()); std::vector<Hit>().swap(x); }
  return v;
}

int join_filter(Groups &g, oracle_group_result *out) {
  Ctx &c = g.c;
  const bool tm = getenv("ORACLE_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char *what) {
    if (!tm) return;
    auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "  %s %.2f s\n", what, std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  };
  // bit maps: >= 16 bits per key (<= 6.25% false positives), at most 2^35 bits (4 GB)
  auto bits_for = [](int64_t keys) {
    int b = 23;
    while (b < 35 && ((int64_t)1 << b) < 16 * keys) ++b;
    return b;
  };
  const int mb = bits_for(out->n_left);
  if (!g.map.reserve((size_t)1 << (mb - 3))) return -1;
  uint64_t *map = (uint64_t *)g.map.p;
  auto set_bit = [map](uint64_t idx) { __atomic_fetch_or(&map[idx >> 6], (uint64_t)1 << (idx & 63), __ATOMIC_RELAXED); };
  auto get_bit = [map](uint64_t idx) { return (__atomic_load_n(&map[idx >> 6], __ATOMIC_RELAXED) >> (idx & 63)) & 1; };
  auto pf_bit = [map](uint64_t idx) { __builtin_prefetch(&map[idx >> 6]); };
  out->passes = 1;
  // 1. left keys set bit (top mb bits)
  g.map.clear((size_t)1 << (mb - 3), c.threads);
  for_rects(c.left, c.threads, [&](int, const Rect &r) {
    for (int64_t j = r.y0; j < r.y0 + r.yn; ++j)
      for (int64_t i = r.x0; i < r.x0 + r.xn; ++i) set_bit(left_key(c, i, j) >> (64 - mb));
  });
  lap("left set");
  // 2. right keys that hit it are the candidates; overshooting right pairs are the filtered count
  std::vector<std::vector<Hit>> parts(c.threads);
  std::atomic<int64_t> filtered{0};
  for_rects(c.right, c.threads, [&](int t, const Rect &r) {
    int64_t f = 0;
    uint64_t kb[kProbe];
    int64_t ib[kProbe];
    for (int64_t j = r.y0; j < r.y0 + r.yn; ++j)
      for (int64_t i0 = r.x0; i0 < r.x0 + r.xn; i0 += kProbe) {
        const int nk = (int)std::min<int64_t>(kProbe, r.x0 + r.xn - i0);
        int nv = 0;
        for (int q = 0; q < nk; ++q) {
          uint64_t k;
          const bool ok = right_key_flat(c, i0 + q, j, k);
          f += !ok;
          pf_bit(k >> (64 - mb));
          ib[nv] = i0 + q;
          kb[nv] = k;
          nv += ok;
        }
        for (int q = 0; q < nv; ++q)
          if (get_bit(kb[q] >> (64 - mb))) parts[t].push_back(Hit{kb[q], ib[q], j});
      }
    filtered += f;
  });
  out->filtered = filtered;
  std::vector<Hit> R = concat_hits(parts);
  lap("right test");
  std::vector<uint64_t> hits;
  std::vector<Hit> lh, rh;
  if (!R.empty()) {
    // 3. candidates set map2[low mb2 bits]; left keys that hit it are the survivors
    const int mb2 = mb;  // survivors ~ n_left x candidates / 2^mb: a few per mille
    const uint64_t lo_mask = ((uint64_t)1 << mb2) - 1;
    g.map.clear((size_t)1 << (mb2 - 3), c.threads);
    {
      std::vector<std::thread> th;
      for (int t = 0; t < c.threads; ++t)
        th.emplace_back([&, t]() {
          for (size_t q = t; q < R.size(); q += c.threads) set_bit(R[q].key & lo_mask);
        });
      for (auto &x : th) x.join();
    }
    for_rects(c.left, c.threads, [&](int t, const Rect &r) {
      uint64_t kb[kProbe];
      for (int64_t j = r.y0; j < r.y0 + r.yn; ++j)
        for (int64_t i0 = r.x0; i0 < r.x0 + r.xn; i0 += kProbe) {
          const int nk = (int)std::min<int64_t>(kProbe, r.x0 + r.xn - i0);
          for (int q = 0; q < nk; ++q) {
            kb[q] = left_key(c, i0 + q, j);
            pf_bit(kb[q] & lo_mask);
          }
          for (int q = 0; q < nk; ++q)
            if (get_bit(kb[q] & lo_mask)) parts[t].push_back(Hit{kb[q], i0 + q, j});
        }
    });
    std::vector<Hit> L = concat_hits(parts);
    lap("left test");
    // 4. every (left survivor, right candidate) pair with equal keys: survivors sorted by key, each
    // candidate's equal range counted (hash_hits += |L(k)| per candidate with key k)
    auto by_key = [](const Hit &x, const Hit &y) { return x.key < y.key; };
    std::sort(L.begin(), L.end(), by_key);
    std::vector<uint64_t> Lk(L.size());
    for (size_t q = 0; q < L.size(); ++q) Lk[q] = L[q].key;
    // a third, cache-sized map over the survivors' middle bits: only its hits are searched
    constexpr int kB3 = 26;
    std::vector<uint8_t> map3((size_t)1 << kB3, 0);
    auto mid = [](uint64_t k) { return (k >> 20) & (((uint64_t)1 << kB3) - 1); };
    for (uint64_t k : Lk) map3[mid(k)] = 1;
    std::vector<int64_t> hh(c.threads, 0);
    std::vector<std::vector<Hit>> rparts(c.threads);
    {
      std::atomic<size_t> next{0};
      std::vector<std::thread> th;
      const size_t step = 1 << 16;
      for (int t = 0; t < c.threads; ++t)
        th.emplace_back([&, t]() {
          for (size_t lo = next.fetch_add(step); lo < R.size(); lo = next.fetch_add(step))
            for (size_t q = lo; q < std::min(R.size(), lo + step); ++q) {
              if (!map3[mid(R[q].key)]) continue;
              auto er = std::equal_range(Lk.begin(), Lk.end(), R[q].key);
              if (er.first == er.second) continue;
              hh[t] += er.second - er.first;
              rparts[t].push_back(R[q]);
            }
        });
      for (auto &x : th) x.join();
    }
    for (int64_t v : hh) out->hash_hits += v;
    rh = concat_hits(rparts);
    for (const Hit &h : rh) hits.push_back(h.key);
    std::sort(hits.begin(), hits.end());
    hits.erase(std::unique(hits.begin(), hits.end()), hits.end());
    for (const Hit &h : L)
      if (std::binary_search(hits.begin(), hits.end(), h.key)) lh.push_back(h);
    lap("equal keys");
    if (tm) fprintf(stderr, "  mb %d/%d candidates %zu survivors %zu\n", mb, mb2, R.size(), L.size());
  }
  confirm_pairs(c, lh, rh, hits, out);
  return 0;
}

}  // namespace

extern "C" {

void oracle_group_result_free(oracle_group_result *r);

// Builds the row-0 quarter tables of instance (m, n, a, d) once, for any number of alpha-group runs.
// Returns nullptr on bad input.
void *oracle_groups_open(int m, int n, const uint64_t *a, const uint64_t *d) {
  if (m < 1 || n < 4 || !a || !d) return nullptr;
  Groups *g = new Groups();
  Ctx &c = g->c;
  c.m = m;
  c.n = n;
  g->d.assign(d, d + m);
  c.d = g->d.data();
  int32_t bs[4];
  oracle_block_sizes(n, bs);
  uint64_t *wp[4], *mp[4], *cp[4];
  int64_t *rp[4];
  for (int t = 0, s = 0; t < 4; ++t) {
    Table &T = c.t[t];
    T.b = bs[t];
    T.start = s;
    s += bs[t];
    T.size = (int64_t)1 << bs[t];
    T.w.resize(T.size); T.mask.resize(T.size); T.contrib.resize((size_t)T.size * m); T.run_end.resize(T.size);
    wp[t] = T.w.data(); mp[t] = T.mask.data(); cp[t] = T.contrib.data(); rp[t] = T.run_end.data();
  }
  if (oracle_build_tables(m, n, a, 0, wp, mp, cp, rp)) { delete g; return nullptr; }
  return g;
}

void oracle_groups_close(void *h) { delete (Groups *)h; }

// One alpha-group (batch) of an opened instance.  method 0: sort-merge in `passes` hash-range passes
// (passes <= 0: chosen so that a pass holds <= 4e8 keys per side); method 1: filter join.  threads
// <= 0: hardware concurrency.  A group that is not a batch (an empty side) returns all-zero
// counters.  Returns 0, or -1 on bad input / allocation failure.
int oracle_groups_run(void *h, uint64_t alpha, int threads, int method, int passes, oracle_group_result *out) {
  memset(out, 0, sizeof(*out));
  if (!h || method < 0 || method > 1) return -1;
  Groups &g = *(Groups *)h;
  Ctx &c = g.c;
  c.threads = threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
  c.alpha = alpha;
  if (alpha > c.d[0]) return 0;  // no right side: empty batch
  c.beta = c.d[0] - alpha;
  c.left = rects_for(c.t[0], c.t[1], alpha);
  c.right = rects_for(c.t[2], c.t[3], c.beta);
  for (const Rect &r : c.left) out->n_left += r.xn * r.yn;
  for (const Rect &r : c.right) out->n_right += r.xn * r.yn;
  if (!out->n_left || !out->n_right) { out->n_left = out->n_right = 0; return 0; }  // not a batch
  if (method == 1) return join_filter(g, out);
  std::vector<uint64_t> hits;
  join_sortmerge(c, passes, out, hits);
  confirm(c, hits, out);
  return 0;
}

// One alpha-group of instance (m, n, a, d), sort-merge method (the original single-call entry).
int oracle_alpha_group(int m, int n, const uint64_t *a, const uint64_t *d, uint64_t alpha, int threads,
                       int passes, oracle_group_result *out) {
  memset(out, 0, sizeof(*out));
  void *h = oracle_groups_open(m, n, a, d);
  if (!h) return -1;
  const int rc = oracle_groups_run(h, alpha, threads, 0, passes, out);
  oracle_groups_close(h);
  return rc;
}

void oracle_group_result_free(oracle_group_result *r) {
  if (!r) return;
  free(r->hit_keys);
  free(r->xbits);
  r->hit_keys = nullptr;
  r->xbits = nullptr;
}

}  // extern "C"
