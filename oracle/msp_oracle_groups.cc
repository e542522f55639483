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
#include <algorithm>
#include <atomic>
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

// One alpha-group of instance (m, n, a, d), enumerated row 0.  passes <= 0: chosen so that a pass
// holds <= 4e8 keys per side; threads <= 0: hardware concurrency.  Returns 0, or -1 on bad input.
int oracle_alpha_group(int m, int n, const uint64_t *a, const uint64_t *d, uint64_t alpha, int threads,
                       int passes, oracle_group_result *out) {
  memset(out, 0, sizeof(*out));
  if (m < 1 || n < 4 || !a || !d) return -1;
  Ctx c;
  c.m = m;
  c.n = n;
  c.d = d;
  c.threads = threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
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
  if (oracle_build_tables(m, n, a, 0, wp, mp, cp, rp)) return -1;
  c.alpha = alpha;
  if (alpha > d[0]) return 0;  // no right side: empty batch
  c.beta = d[0] - alpha;
  c.left = rects_for(c.t[0], c.t[1], alpha);
  c.right = rects_for(c.t[2], c.t[3], c.beta);
  for (const Rect &r : c.left) out->n_left += r.xn * r.yn;
  for (const Rect &r : c.right) out->n_right += r.xn * r.yn;
  if (!out->n_left || !out->n_right) { out->n_left = out->n_right = 0; return 0; }  // not a batch
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
  std::vector<uint64_t> hits;
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
    std::vector<uint64_t> L, R;
    for (auto &v : lk) { L.insert(L.end(), v.begin(), v.end()); std::vector<uint64_t>().swap(v); }
    for (auto &v : rk) { R.insert(R.end(), v.begin(), v.end()); std::vector<uint64_t>().swap(v); }
    psort(L, pbits, c.threads);
    psort(R, pbits, c.threads);
    size_t i = 0, j = 0;
    while (i < L.size() && j < R.size()) {
      if (L[i] < R[j]) { ++i; continue; }
      if (R[j] < L[i]) { ++j; continue; }
      const uint64_t k = L[i];
      size_t i1 = i, j1 = j;
      while (i1 < L.size() && L[i1] == k) ++i1;
      while (j1 < R.size() && R[j1] == k) ++j1;
      out->hash_hits += (int64_t)((i1 - i) * (j1 - j));
      hits.push_back(k);
      i = i1;
      j = j1;
    }
  }
  out->filtered = filtered;
  std::sort(hits.begin(), hits.end());
  // exact confirmation (validate.py:285-313): pairs whose key is a hit key, residuals compared
  struct Hit { uint64_t key; int64_t i, j; };
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
  std::vector<uint8_t> xs;
  for (const Hit &l : lh)
    for (const Hit &r : rh) {
      if (l.key != r.key) continue;
      bool eq = true;
      for (int k = 0; k < m && eq; ++k) {
        const uint64_t v = c.t[0].contrib[(size_t)l.i * m + k] + c.t[1].contrib[(size_t)l.j * m + k];
        const uint64_t s = c.t[2].contrib[(size_t)r.i * m + k] + c.t[3].contrib[(size_t)r.j * m + k];
        eq = v == d[k] - s;
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
  out->n_hit_keys = (int64_t)hits.size();
  if (!hits.empty()) {
    out->hit_keys = (uint64_t *)malloc(8 * hits.size());
    memcpy(out->hit_keys, hits.data(), 8 * hits.size());
  }
  return 0;
}

void oracle_group_result_free(oracle_group_result *r) {
  if (!r) return;
  free(r->hit_keys);
  free(r->xbits);
  r->hit_keys = nullptr;
  r->xbits = nullptr;
}

}  // extern "C"
