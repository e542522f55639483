/*
 * msp_oracle.c -- CPU restatement of the reference market-split solver.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU baseline
 * ("cpu_baseline.kind = port").  Only tests/, __graft_entry__.smoke() and bench.py's
 * reference/cpu_baseline legs may load it.  The product path (paper_2507_05045_b200/)
 * never links or calls it.
 *
 * It restates, function by function, the reference package
 * (/root/reference/pkg/src/marketsplit, pure Python + numba):
 *
 *   splitmix64 / below            instances.py:222-247
 *   fnv fold                      validate.py:34-50, fastval.py:42-43,70-73
 *   build_quarter_tables          enumerate1d.py:81-135  (lexsort((masks, key)))
 *   _run_ends                     enumerate1d.py:138-145
 *   heap pair-sum enumerator      fastenum.py:44-147     (array heaps, complemented H2 keys)
 *   _expand                       fastenum.py:150-158    (done lazily per chunk here)
 *   fused join _join_pairs        fastval.py:47-113      (bucket chains, 2^22 cap)
 *   validate_chunked + stats      validate.py:316-385    (quadratic chunk loop, first-sweep stats)
 *   _confirm_hits / assemble      validate.py:285-313, enumerate1d.py:313-327
 *   brute force (n <= 12)         oracle.py:27-75, solver.py:197-211
 *   pipeline_run                  solver.py:292-419      (1 enumerator thread + W workers)
 *
 * Parity of this restatement is pinned against fixtures generated from the reference itself
 * (JSON fixtures under tests/golden/, script tests/golden/make_golden.py); see tests/test_oracle.py.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#define FNV_OFFSET 0xCBF29CE484222325ULL
#define FNV_PRIME 0x100000001B3ULL

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ---------------------------------------------------------------- KATs */

uint64_t oracle_splitmix64_next(uint64_t *state) { /* instances.py:230-235 */
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t oracle_splitmix64_below(uint64_t *state, uint64_t k) { /* instances.py:237-247 */
  /* limit = 2^64 - (2^64 mod k); u < limit accepted */
  uint64_t rem = (uint64_t)(((unsigned __int128)1 << 64) % k);
  for (;;) {
    uint64_t u = oracle_splitmix64_next(state);
    if (rem == 0 || u < (uint64_t)(0 - rem)) return u % k;
  }
}

uint64_t oracle_fnv_fold(const uint64_t *v, int m) { /* validate.py:45-50 */
  uint64_t h = FNV_OFFSET;
  for (int j = 0; j < m; ++j) h = (h ^ v[j]) * FNV_PRIME;
  return h;
}

/* ---------------------------------------------------------------- tables */

typedef struct {
  int b;            /* block size (columns) */
  int start;        /* first column */
  int ascending;
  int64_t size;     /* 2^b */
  uint64_t *weights;
  uint64_t *masks;
  uint64_t *contribs; /* size x m, row-major, coordinate 0 = enumerated row */
  int64_t *run_end;
} qtable;

typedef struct { uint64_t key, mask; } kv_t;

static int kv_cmp(const void *x, const void *y) {
  const kv_t *a = (const kv_t *)x, *b = (const kv_t *)y;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->mask < b->mask ? -1 : (a->mask > b->mask);
}

static void block_sizes(int n, int out[4]) { /* enumerate1d.py:81-83 */
  int q = n / 4, r = n % 4;
  for (int i = 0; i < 4; ++i) out[i] = i < r ? q + 1 : q;
}

/* enumerate1d.py:86-135 */
static int build_tables(int m, int n, const uint64_t *a, int row, qtable t[4]) {
  if (n < 4 || row < 0 || row >= m) return -1;
  int sizes[4];
  block_sizes(n, sizes);
  int *row_map = (int *)malloc(sizeof(int) * m);
  row_map[0] = row;
  for (int i = 0, c = 1; i < m; ++i)
    if (i != row) row_map[c++] = i;
  int start = 0;
  for (int bi = 0; bi < 4; ++bi) {
    int b = sizes[bi];
    int64_t size = (int64_t)1 << b;
    uint64_t *contrib_mask_order = (uint64_t *)calloc((size_t)size * m, 8);
    for (int ci = 0; ci < m; ++ci) {
      const uint64_t *arow = a + (size_t)row_map[ci] * n;
      /* doubling: sums = concat(sums, sums + a[ri, col]); bit t <-> column start+t */
      for (int64_t mask = 0; mask < size; ++mask) {
        uint64_t s = 0;
        for (int tb = 0; tb < b; ++tb)
          if ((mask >> tb) & 1) s += arow[start + tb];
        contrib_mask_order[(size_t)mask * m + ci] = s;
      }
    }
    int asc = bi < 2;
    kv_t *kv = (kv_t *)malloc(sizeof(kv_t) * size);
    for (int64_t mask = 0; mask < size; ++mask) {
      uint64_t w = contrib_mask_order[(size_t)mask * m];
      kv[mask].key = asc ? w : (~0ULL - w);
      kv[mask].mask = (uint64_t)mask;
    }
    qsort(kv, (size_t)size, sizeof(kv_t), kv_cmp); /* == np.lexsort((masks, key)) */
    t[bi].b = b;
    t[bi].start = start;
    t[bi].ascending = asc;
    t[bi].size = size;
    t[bi].weights = (uint64_t *)malloc(8 * size);
    t[bi].masks = (uint64_t *)malloc(8 * size);
    t[bi].contribs = (uint64_t *)malloc(8 * (size_t)size * m);
    t[bi].run_end = (int64_t *)malloc(8 * size);
    for (int64_t e = 0; e < size; ++e) {
      uint64_t mk = kv[e].mask;
      t[bi].masks[e] = mk;
      memcpy(t[bi].contribs + (size_t)e * m, contrib_mask_order + (size_t)mk * m, 8 * (size_t)m);
      t[bi].weights[e] = t[bi].contribs[(size_t)e * m];
    }
    /* _run_ends: end of maximal equal-weight run (enumerate1d.py:138-145) */
    int64_t e = size;
    for (int64_t i = size - 1; i >= 0; --i) {
      if (i + 1 < size && t[bi].weights[i] != t[bi].weights[i + 1]) e = i + 1;
      t[bi].run_end[i] = e;
    }
    free(kv);
    free(contrib_mask_order);
    start += b;
  }
  free(row_map);
  return 0;
}

static void free_tables(qtable t[4]) {
  for (int i = 0; i < 4; ++i) {
    free(t[i].weights);
    free(t[i].masks);
    free(t[i].contribs);
    free(t[i].run_end);
  }
}

/* Exported for table-parity tests: caller passes 4 x (weights, masks, contribs, run_end) buffers
 * sized from oracle_block_sizes. */
void oracle_block_sizes(int n, int32_t out[4]) {
  int s[4];
  block_sizes(n, s);
  for (int i = 0; i < 4; ++i) out[i] = s[i];
}

int oracle_build_tables(int m, int n, const uint64_t *a, int row, uint64_t **weights,
                        uint64_t **masks, uint64_t **contribs, int64_t **run_end) {
  qtable t[4];
  if (build_tables(m, n, a, row, t)) return -1;
  for (int i = 0; i < 4; ++i) {
    memcpy(weights[i], t[i].weights, 8 * t[i].size);
    memcpy(masks[i], t[i].masks, 8 * t[i].size);
    memcpy(contribs[i], t[i].contribs, 8 * (size_t)t[i].size * m);
    memcpy(run_end[i], t[i].run_end, 8 * t[i].size);
  }
  free_tables(t);
  return 0;
}

/* ---------------------------------------------------------------- heap enumerator */
/* fastenum.py:44-147: two array heaps ordered by (key, fixed index). */

typedef struct {
  uint64_t *k;
  int64_t *f, *r;
  int64_t n;
} heap_t;

static inline int hless(uint64_t k1, int64_t f1, uint64_t k2, int64_t f2) {
  return k1 != k2 ? k1 < k2 : f1 < f2;
}

static void sift_down(heap_t *h, int64_t size, int64_t i) { /* fastenum.py:51-68 */
  uint64_t k = h->k[i];
  int64_t f = h->f[i], r = h->r[i];
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= size) break;
    int64_t rc = c + 1;
    if (rc < size && hless(h->k[rc], h->f[rc], h->k[c], h->f[c])) c = rc;
    if (hless(h->k[c], h->f[c], k, f)) {
      h->k[i] = h->k[c];
      h->f[i] = h->f[c];
      h->r[i] = h->r[c];
      i = c;
    } else
      break;
  }
  h->k[i] = k;
  h->f[i] = f;
  h->r[i] = r;
}

static void heap_pop(heap_t *h) { /* fastenum.py:71-77 */
  h->n -= 1;
  if (h->n > 0) {
    h->k[0] = h->k[h->n];
    h->f[0] = h->f[h->n];
    h->r[0] = h->r[h->n];
    sift_down(h, h->n, 0);
  }
}

static void heap_replace(heap_t *h, uint64_t k, int64_t f, int64_t r) {
  h->k[0] = k;
  h->f[0] = f;
  h->r[0] = r;
  sift_down(h, h->n, 0);
}

static void heapify(heap_t *h) {
  for (int64_t i = h->n / 2 - 1; i >= 0; --i) sift_down(h, h->n, i);
}

typedef struct {
  const qtable *t;
  uint64_t target;
  heap_t h1, h2;
  int64_t peak1, peak2;
  int exhausted;
} enum_t;

/* Seed at alpha >= alpha_lo: every B partner sits at the first A run reaching alpha_lo, and every
 * D partner at the first C run with weight <= target - alpha_lo.  With alpha_lo = 0 this is exactly
 * the reference seeding (i = 0 / k = 0 for every partner, fastenum.py:179-188).  For alpha_lo > 0 it
 * is the state the reference heap holds when its top first reaches alpha_lo (entries only advance
 * while they are the minimum), so the emitted batches for alpha >= alpha_lo are unchanged. */
static void enum_init(enum_t *e, const qtable t[4], uint64_t target, uint64_t alpha_lo) {
  e->t = t;
  e->target = target;
  int64_t nb = t[1].size, nd = t[3].size;
  e->h1.k = (uint64_t *)malloc(8 * nb);
  e->h1.f = (int64_t *)malloc(8 * nb);
  e->h1.r = (int64_t *)malloc(8 * nb);
  e->h2.k = (uint64_t *)malloc(8 * nd);
  e->h2.f = (int64_t *)malloc(8 * nd);
  e->h2.r = (int64_t *)malloc(8 * nd);
  e->h1.n = 0;
  for (int64_t j = 0; j < nb; ++j) {
    int64_t i = 0;
    if (alpha_lo > 0) { /* first i with wa[i] + wb[j] >= alpha_lo (A ascending) */
      int64_t lo = 0, hi = t[0].size;
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (t[0].weights[mid] + t[1].weights[j] < alpha_lo) lo = mid + 1; else hi = mid;
      }
      i = lo;
      if (i >= t[0].size) continue;
    }
    e->h1.k[e->h1.n] = t[0].weights[i] + t[1].weights[j];
    e->h1.f[e->h1.n] = j;
    e->h1.r[e->h1.n] = i;
    e->h1.n++;
  }
  e->h2.n = 0;
  uint64_t beta_hi = target >= alpha_lo ? target - alpha_lo : 0;
  for (int64_t l = 0; l < nd; ++l) {
    int64_t k = 0;
    if (alpha_lo > 0) { /* first k with wc[k] + wd[l] <= beta_hi (C descending) */
      if (target < alpha_lo) break;
      int64_t lo = 0, hi = t[2].size;
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (t[2].weights[mid] + t[3].weights[l] > beta_hi) lo = mid + 1; else hi = mid;
      }
      k = lo;
      if (k >= t[2].size) continue;
    }
    e->h2.k[e->h2.n] = ~0ULL - (t[2].weights[k] + t[3].weights[l]);
    e->h2.f[e->h2.n] = l;
    e->h2.r[e->h2.n] = k;
    e->h2.n++;
  }
  heapify(&e->h1);
  heapify(&e->h2);
  e->peak1 = nb;
  e->peak2 = nd;
  e->exhausted = 0;
}

static void enum_free(enum_t *e) {
  free(e->h1.k); free(e->h1.f); free(e->h1.r);
  free(e->h2.k); free(e->h2.f); free(e->h2.r);
}

typedef struct {
  uint64_t alpha, beta;
  int64_t nlseg, nrseg;
  int64_t *lseg; /* (start, end, fixed) triples */
  int64_t *rseg;
  int64_t nl, nr;
  int64_t seq;
} batch_t;

/* fastenum.py:87-147: returns 1 and fills *b on a batch, 0 when exhausted. */
static int enum_next(enum_t *e, batch_t *b) {
  const qtable *t = e->t;
  const uint64_t *wa = t[0].weights, *wb = t[1].weights, *wc = t[2].weights, *wd = t[3].weights;
  const int64_t *rea = t[0].run_end, *rec = t[2].run_end;
  int64_t na = t[0].size, nc = t[2].size;
  heap_t *h1 = &e->h1, *h2 = &e->h2;
  while (h1->n > 0 && h2->n > 0) {
    uint64_t alpha = h1->k[0];
    uint64_t beta = ~0ULL - h2->k[0];
    uint64_t combined = alpha + beta;
    if (combined < e->target) {
      int64_t j = h1->f[0], ni = rea[h1->r[0]];
      if (ni < na) heap_replace(h1, wa[ni] + wb[j], j, ni); else heap_pop(h1);
    } else if (combined > e->target) {
      int64_t l = h2->f[0], nk = rec[h2->r[0]];
      if (nk < nc) heap_replace(h2, ~0ULL - (wc[nk] + wd[l]), l, nk); else heap_pop(h2);
    } else {
      int64_t nl = 0, nlp = 0;
      while (h1->n > 0 && h1->k[0] == alpha) {
        int64_t j = h1->f[0], i = h1->r[0], end = rea[i];
        b->lseg[3 * nl] = i; b->lseg[3 * nl + 1] = end; b->lseg[3 * nl + 2] = j;
        nl++; nlp += end - i;
        if (end < na) heap_replace(h1, wa[end] + wb[j], j, end); else heap_pop(h1);
      }
      int64_t nr = 0, nrp = 0;
      uint64_t cb = h2->k[0];
      while (h2->n > 0 && h2->k[0] == cb) {
        int64_t l = h2->f[0], k = h2->r[0], end = rec[k];
        b->rseg[3 * nr] = k; b->rseg[3 * nr + 1] = end; b->rseg[3 * nr + 2] = l;
        nr++; nrp += end - k;
        if (end < nc) heap_replace(h2, ~0ULL - (wc[end] + wd[l]), l, end); else heap_pop(h2);
      }
      b->alpha = alpha; b->beta = beta;
      b->nlseg = nl; b->nrseg = nr; b->nl = nlp; b->nr = nrp;
      return 1;
    }
  }
  e->exhausted = 1;
  return 0;
}

/* Expand pairs [s, s+cnt) of a segment list into out (x idx, y idx) -- fastenum.py:150-158,
 * materialised one chunk at a time instead of the whole batch. */
static void expand_range(const int64_t *seg, int64_t nseg, int64_t s, int64_t cnt, int64_t *out) {
  int64_t pos = 0, si = 0;
  while (si < nseg && pos + (seg[3 * si + 1] - seg[3 * si]) <= s) { pos += seg[3 * si + 1] - seg[3 * si]; si++; }
  int64_t off = s - pos, w = 0;
  while (w < cnt && si < nseg) {
    int64_t st = seg[3 * si], en = seg[3 * si + 1], fx = seg[3 * si + 2];
    for (int64_t x = st + off; x < en && w < cnt; ++x) { out[2 * w] = x; out[2 * w + 1] = fx; w++; }
    off = 0; si++;
  }
}

/* ---------------------------------------------------------------- fused join */

static int bucket_bits(int64_t nl, int cap) { /* fastval.py:111-113 */
  int64_t v = (nl > 1 ? nl : 1) - 1;
  int bl = 0;
  while (v) { bl++; v >>= 1; }
  int bits = bl + 1;
  if (bits < 10) bits = 10;
  if (bits > cap) bits = cap;
  return bits;
}

typedef struct {
  int64_t *heads; int64_t heads_cap;
  int64_t *links; uint64_t *lh; int64_t lcap;
  int64_t *hits; int64_t hits_cap;
  int64_t *lp, *rp; int64_t pcap;
} join_ws;

/* fastval.py:47-108 + join_pairs wrapper :116-139.  Returns number of hits (all stored). */
static int64_t join_pairs(const qtable t[4], int m, const uint64_t *d, uint64_t alpha,
                          const int64_t *lp, int64_t nl, const int64_t *rp, int64_t nr,
                          int bits_cap, join_ws *ws, int64_t *filtered_out, int *bad_out) {
  int bits = bucket_bits(nl, bits_cap);
  int64_t nb = (int64_t)1 << bits;
  if (ws->heads_cap < nb) { free(ws->heads); ws->heads = (int64_t *)malloc(8 * nb); ws->heads_cap = nb; }
  if (ws->lcap < nl) {
    free(ws->links); free(ws->lh);
    ws->links = (int64_t *)malloc(8 * (nl + 1)); ws->lh = (uint64_t *)malloc(8 * (nl + 1)); ws->lcap = nl;
  }
  for (int64_t i = 0; i < nb; ++i) ws->heads[i] = -1;
  uint64_t mask = (uint64_t)nb - 1;
  const uint64_t *cA = t[0].contribs, *cB = t[1].contribs, *cC = t[2].contribs, *cD = t[3].contribs;
  int bad = 0;
  for (int64_t q = 0; q < nl; ++q) {
    const uint64_t *va = cA + (size_t)lp[2 * q] * m, *vb = cB + (size_t)lp[2 * q + 1] * m;
    if (va[0] + vb[0] != alpha) bad++;
    uint64_t h = FNV_OFFSET;
    for (int j = 0; j < m; ++j) h = (h ^ (va[j] + vb[j])) * FNV_PRIME;
    ws->lh[q] = h;
  }
  for (int64_t q = nl - 1; q >= 0; --q) { /* head-insert in reverse: chains ascend */
    uint64_t bk = ws->lh[q] & mask;
    ws->links[q] = ws->heads[bk];
    ws->heads[bk] = q;
  }
  int64_t nout = 0, filtered = 0;
  for (int64_t r = 0; r < nr; ++r) {
    const uint64_t *vc = cC + (size_t)rp[2 * r] * m, *vd = cD + (size_t)rp[2 * r + 1] * m;
    int keep = 1;
    uint64_t h = FNV_OFFSET;
    for (int j = 0; j < m; ++j) {
      uint64_t s = vc[j] + vd[j];
      if (s > d[j]) { keep = 0; break; }
      uint64_t res = d[j] - s;
      if (j == 0 && res != alpha) bad++;
      h = (h ^ res) * FNV_PRIME;
    }
    if (!keep) { filtered++; continue; }
    for (int64_t q = ws->heads[h & mask]; q != -1; q = ws->links[q]) {
      if (ws->lh[q] == h) {
        if (nout >= ws->hits_cap) {
          ws->hits_cap = ws->hits_cap ? 2 * ws->hits_cap : 1024;
          ws->hits = (int64_t *)realloc(ws->hits, 16 * ws->hits_cap);
        }
        ws->hits[2 * nout] = q; ws->hits[2 * nout + 1] = r;
        nout++;
      }
    }
  }
  *filtered_out = filtered;
  *bad_out = bad;
  return nout;
}

/* ---------------------------------------------------------------- solve */

typedef struct {
  int32_t mode;          /* 0 first, 1 all */
  int32_t workers;       /* 0 -> cpu_count - 1 (solver.py:143-146) */
  int64_t chunk_pairs;   /* 0 -> default_chunk_pairs(m) (validate.py:382-385) */
  int32_t bucket_bits_cap; /* 0 -> 22 (fastval.py:111-113) */
  int32_t record_batches;
  uint64_t alpha_lo, alpha_hi; /* validate only batches with alpha in [lo, hi); hi=0 -> no bound */
  int32_t row;           /* enumerated row (0 in solve) */
  int32_t brute_force_max_n; /* -1 -> 12 (solver.py:48) */
} oracle_options;

typedef struct {
  int64_t batches, candidates_left, candidates_right, filtered_residuals, hash_hits, exact_hits;
  uint64_t row1_pairs_lo, row1_pairs_hi;
  int64_t peak_table_entries, peak_heap1, peak_heap2;
  double t_build, t_enumerate, t_validate, t_total;
  int32_t fallback; /* 0 none, 1 brute-force, 2 zero-rhs */
  int32_t threads_used;
  int64_t n_solutions;
  uint8_t *xbits;          /* n_solutions x n */
  int64_t n_batch_records;
  int64_t *batch_records;  /* per batch: alpha, n_left, n_right, filtered, hash_hits, exact_hits */
} oracle_result;

typedef struct {
  int m, n;
  const uint64_t *a, *d_orig;
  uint64_t *dperm;
  qtable t[4];
  oracle_options opt;
  int64_t chunk;
  /* queue */
  pthread_mutex_t mu;
  pthread_cond_t cv_put, cv_get;
  batch_t **q; int qcap, qhead, qcount;
  int done, stop;
  /* results */
  pthread_mutex_t rmu;
  uint8_t *xbits; int64_t nsol, solcap;
  int64_t *brec; int64_t nbrec, brcap;
  int64_t batches, cl, cr, filt, hh, eh;
  unsigned __int128 row1;
  double t_enum, t_val;
  int error;
} solve_ctx;

static void add_solution(solve_ctx *c, const int64_t idx[4]) {
  uint8_t *x = (uint8_t *)calloc(c->n, 1);
  for (int ti = 0; ti < 4; ++ti) {
    uint64_t mk = c->t[ti].masks[idx[ti]];
    for (int bt = 0; bt < c->t[ti].b; ++bt) x[c->t[ti].start + bt] = (mk >> bt) & 1;
  }
  /* verify on the instance (instances.py:322-336); failure is an internal error */
  for (int i = 0; i < c->m; ++i) {
    unsigned __int128 s = 0;
    for (int j = 0; j < c->n; ++j) if (x[j]) s += c->a[(size_t)i * c->n + j];
    if (s != c->d_orig[i]) c->error = 4;
  }
  if (c->nsol >= c->solcap) {
    c->solcap = c->solcap ? 2 * c->solcap : 64;
    c->xbits = (uint8_t *)realloc(c->xbits, (size_t)c->solcap * c->n);
  }
  memcpy(c->xbits + (size_t)c->nsol * c->n, x, c->n);
  c->nsol++;
  free(x);
}

/* validate_chunked (validate.py:316-379) on one batch; returns exact hits */
static void validate_batch(solve_ctx *c, batch_t *b, join_ws *ws) {
  int m = c->m;
  int64_t chunk = c->chunk;
  int64_t cl = 0, cr = 0, filt = 0, hh = 0, eh = 0;
  int64_t pneed = chunk < b->nl ? chunk : b->nl;
  int64_t pneed2 = chunk < b->nr ? chunk : b->nr;
  if (pneed2 > pneed) pneed = pneed2;
  if (ws->pcap < pneed) {
    free(ws->lp); free(ws->rp);
    ws->lp = (int64_t *)malloc(16 * (pneed + 1)); ws->rp = (int64_t *)malloc(16 * (pneed + 1));
    ws->pcap = pneed;
  }
  int first_sweep = 1;
  int64_t lmax = b->nl > 1 ? b->nl : 1, rmax = b->nr > 1 ? b->nr : 1;
  for (int64_t ls = 0; ls < lmax; ls += chunk) {
    int64_t lc = b->nl - ls < chunk ? b->nl - ls : chunk;
    if (lc < 0) lc = 0;
    expand_range(b->lseg, b->nlseg, ls, lc, ws->lp);
    cl += lc;
    for (int64_t rs = 0; rs < rmax; rs += chunk) {
      int64_t rc = b->nr - rs < chunk ? b->nr - rs : chunk;
      if (rc < 0) rc = 0;
      expand_range(b->rseg, b->nrseg, rs, rc, ws->rp);
      int64_t f = 0;
      int bad = 0;
      int64_t nh = join_pairs(c->t, m, c->dperm, b->alpha, ws->lp, lc, ws->rp, rc,
                              c->opt.bucket_bits_cap, ws, &f, &bad);
      if (bad) c->error = 4; /* AssertionError: residual coordinate 0 disagrees with alpha */
      if (first_sweep) { cr += rc; filt += f; }
      hh += nh;
      for (int64_t hi = 0; hi < nh; ++hi) { /* _confirm_hits: exact residual equality */
        int64_t q = ws->hits[2 * hi], r = ws->hits[2 * hi + 1];
        int64_t idx[4] = {ws->lp[2 * q], ws->lp[2 * q + 1], ws->rp[2 * r], ws->rp[2 * r + 1]};
        const uint64_t *va = c->t[0].contribs + (size_t)idx[0] * m, *vb = c->t[1].contribs + (size_t)idx[1] * m;
        const uint64_t *vc = c->t[2].contribs + (size_t)idx[2] * m, *vd = c->t[3].contribs + (size_t)idx[3] * m;
        int eq = 1;
        for (int j = 0; j < m; ++j) if (va[j] + vb[j] != c->dperm[j] - (vc[j] + vd[j])) { eq = 0; break; }
        if (eq) {
          pthread_mutex_lock(&c->rmu);
          add_solution(c, idx);
          pthread_mutex_unlock(&c->rmu);
          eh++;
        }
      }
    }
    first_sweep = 0;
  }
  pthread_mutex_lock(&c->rmu);
  c->cl += cl; c->cr += cr; c->filt += filt; c->hh += hh; c->eh += eh;
  if (c->opt.record_batches) {
    if (c->nbrec >= c->brcap) {
      c->brcap = c->brcap ? 2 * c->brcap : 1024;
      c->brec = (int64_t *)realloc(c->brec, 8 * 7 * c->brcap);
    }
    int64_t *r = c->brec + 7 * c->nbrec++;
    r[0] = (int64_t)b->alpha; r[1] = b->nl; r[2] = b->nr; r[3] = filt; r[4] = hh; r[5] = eh; r[6] = b->seq;
  }
  if (c->opt.mode == 0 && eh > 0) c->stop = 1;
  pthread_mutex_unlock(&c->rmu);
}

static void *producer(void *arg) { /* solver.py:318-355 */
  solve_ctx *c = (solve_ctx *)arg;
  enum_t e;
  double t0 = now_s();
  enum_init(&e, c->t, c->dperm[0], c->opt.alpha_lo);
  int64_t seq = 0;
  for (;;) {
    batch_t *b = (batch_t *)malloc(sizeof(batch_t));
    b->lseg = (int64_t *)malloc(24 * (c->t[1].size + 1));
    b->rseg = (int64_t *)malloc(24 * (c->t[3].size + 1));
    pthread_mutex_lock(&c->mu);
    int stop = c->stop;
    pthread_mutex_unlock(&c->mu);
    int got = stop ? 0 : enum_next(&e, b);
    if (got && c->opt.alpha_hi && b->alpha >= c->opt.alpha_hi) got = 0;
    if (!got) { free(b->lseg); free(b->rseg); free(b); break; }
    b->seq = seq++;
    pthread_mutex_lock(&c->mu);
    c->batches++;
    c->row1 += (unsigned __int128)b->nl * (unsigned __int128)b->nr;
    while (c->qcount == c->qcap && !c->stop) pthread_cond_wait(&c->cv_put, &c->mu);
    if (c->stop) { pthread_mutex_unlock(&c->mu); free(b->lseg); free(b->rseg); free(b); break; }
    c->q[(c->qhead + c->qcount) % c->qcap] = b;
    c->qcount++;
    pthread_cond_signal(&c->cv_get);
    pthread_mutex_unlock(&c->mu);
  }
  pthread_mutex_lock(&c->mu);
  c->done = 1;
  c->t_enum = now_s() - t0;
  pthread_cond_broadcast(&c->cv_get);
  pthread_mutex_unlock(&c->mu);
  enum_free(&e);
  return NULL;
}

static void *worker(void *arg) { /* solver.py:357-399 */
  solve_ctx *c = (solve_ctx *)arg;
  join_ws ws;
  memset(&ws, 0, sizeof(ws));
  for (;;) {
    pthread_mutex_lock(&c->mu);
    while (c->qcount == 0 && !c->done && !c->stop) pthread_cond_wait(&c->cv_get, &c->mu);
    if (c->qcount == 0 || c->stop) { pthread_mutex_unlock(&c->mu); break; }
    batch_t *b = c->q[c->qhead];
    c->qhead = (c->qhead + 1) % c->qcap;
    c->qcount--;
    pthread_cond_signal(&c->cv_put);
    pthread_mutex_unlock(&c->mu);
    double t0 = now_s();
    validate_batch(c, b, &ws);
    double dt = now_s() - t0;
    pthread_mutex_lock(&c->mu);
    c->t_val += dt;
    if (c->stop) pthread_cond_broadcast(&c->cv_put);
    pthread_mutex_unlock(&c->mu);
    free(b->lseg); free(b->rseg); free(b);
  }
  free(ws.heads); free(ws.links); free(ws.lh); free(ws.hits); free(ws.lp); free(ws.rp);
  return NULL;
}

/* oracle.py:27-75 restated: all x with A x = d, n <= 28 */
static void brute_force(solve_ctx *c) {
  int n = c->n, m = c->m;
  for (uint64_t enc = 0; enc < ((uint64_t)1 << n); ++enc) {
    int ok = 1;
    for (int i = 0; i < m && ok; ++i) {
      unsigned __int128 s = 0;
      for (int j = 0; j < n; ++j) /* x_1 is the MSB of the encoding */
        if ((enc >> (n - 1 - j)) & 1) s += c->a[(size_t)i * n + j];
      ok = s == c->d_orig[i];
    }
    if (ok) {
      if (c->nsol >= c->solcap) {
        c->solcap = c->solcap ? 2 * c->solcap : 64;
        c->xbits = (uint8_t *)realloc(c->xbits, (size_t)c->solcap * n);
      }
      for (int j = 0; j < n; ++j) c->xbits[(size_t)c->nsol * n + j] = (enc >> (n - 1 - j)) & 1;
      c->nsol++;
    }
  }
}

int oracle_solve(int m, int n, const uint64_t *a, const uint64_t *d, const oracle_options *opt_in,
                 oracle_result *res) {
  double t_start = now_s();
  memset(res, 0, sizeof(*res));
  solve_ctx *c = (solve_ctx *)calloc(1, sizeof(solve_ctx));
  c->m = m; c->n = n; c->a = a; c->d_orig = d;
  c->opt = *opt_in;
  if (c->opt.bucket_bits_cap <= 0) c->opt.bucket_bits_cap = 22;
  int bf_max = c->opt.brute_force_max_n < 0 ? 12 : c->opt.brute_force_max_n;
  int any_d = 0;
  for (int i = 0; i < m; ++i) any_d |= d[i] != 0;
  if (c->opt.mode == 0 && !any_d) { /* solver.py:190-195 */
    res->fallback = 2;
    res->n_solutions = 1;
    res->xbits = (uint8_t *)calloc(n, 1);
    res->t_total = now_s() - t_start;
    free(c);
    return 0;
  }
  if (n <= bf_max) { /* solver.py:197-211 */
    if (n > 28) { free(c); return 2; }
    brute_force(c);
    if (c->opt.mode == 0 && c->nsol > 1) c->nsol = 1;
    res->fallback = 1;
    res->exact_hits = c->nsol;
    res->n_solutions = c->nsol;
    res->xbits = c->xbits;
    res->t_total = now_s() - t_start;
    free(c);
    return 0;
  }
  double t0 = now_s();
  if (build_tables(m, n, a, c->opt.row, c->t)) { free(c); return 2; }
  res->t_build = now_s() - t0;
  c->dperm = (uint64_t *)malloc(8 * m);
  c->dperm[0] = d[c->opt.row];
  for (int i = 0, k = 1; i < m; ++i) if (i != c->opt.row) c->dperm[k++] = d[i];
  c->chunk = c->opt.chunk_pairs > 0 ? c->opt.chunk_pairs : (int64_t)((512LL << 20) / (2 * (8 * m + 32)));
  int workers = c->opt.workers;
  if (workers <= 0) {
    long nc = sysconf(_SC_NPROCESSORS_ONLN);
    workers = nc > 2 ? (int)nc - 1 : 1;
  }
  c->qcap = 8;
  c->q = (batch_t **)calloc(c->qcap, sizeof(batch_t *));
  pthread_mutex_init(&c->mu, NULL);
  pthread_mutex_init(&c->rmu, NULL);
  pthread_cond_init(&c->cv_put, NULL);
  pthread_cond_init(&c->cv_get, NULL);
  pthread_t prod, *wk = (pthread_t *)malloc(sizeof(pthread_t) * workers);
  pthread_create(&prod, NULL, producer, c);
  for (int w = 0; w < workers; ++w) pthread_create(&wk[w], NULL, worker, c);
  pthread_join(prod, NULL);
  for (int w = 0; w < workers; ++w) pthread_join(wk[w], NULL);
  /* drain anything left in the queue after a first-mode stop */
  while (c->qcount) {
    batch_t *b = c->q[c->qhead];
    c->qhead = (c->qhead + 1) % c->qcap; c->qcount--;
    free(b->lseg); free(b->rseg); free(b);
  }
  res->batches = c->batches;
  res->candidates_left = c->cl;
  res->candidates_right = c->cr;
  res->filtered_residuals = c->filt;
  res->hash_hits = c->hh;
  res->exact_hits = c->eh;
  res->row1_pairs_lo = (uint64_t)c->row1;
  res->row1_pairs_hi = (uint64_t)(c->row1 >> 64);
  res->peak_table_entries = c->t[0].size + c->t[1].size + c->t[2].size + c->t[3].size;
  res->peak_heap1 = c->t[1].size;
  res->peak_heap2 = c->t[3].size;
  res->t_enumerate = c->t_enum;
  res->t_validate = c->t_val;
  res->threads_used = workers + 1;
  res->n_solutions = c->nsol;
  res->xbits = c->xbits;
  res->n_batch_records = c->nbrec;
  res->batch_records = c->brec;
  int err = c->error;
  free_tables(c->t);
  free(c->dperm);
  free(c->q);
  free(wk);
  pthread_mutex_destroy(&c->mu);
  pthread_mutex_destroy(&c->rmu);
  pthread_cond_destroy(&c->cv_put);
  pthread_cond_destroy(&c->cv_get);
  free(c);
  res->t_total = now_s() - t_start;
  return err;
}

void oracle_result_free(oracle_result *r) {
  free(r->xbits);
  free(r->batch_records);
  memset(r, 0, sizeof(*r));
}

/* Batch stream for stream-parity tests: writes per batch (alpha, beta, nl, nr) and the expanded
 * pairs into caller buffers; returns number of batches (or -needed when buffers are short). */
int64_t oracle_stream(int m, int n, const uint64_t *a, const uint64_t *d, int64_t max_batches,
                      int64_t *hdr, int64_t max_pairs, int64_t *pairs) {
  qtable t[4];
  if (build_tables(m, n, a, 0, t)) return -1;
  enum_t e;
  enum_init(&e, t, d[0], 0);
  batch_t b;
  b.lseg = (int64_t *)malloc(24 * (t[1].size + 1));
  b.rseg = (int64_t *)malloc(24 * (t[3].size + 1));
  int64_t nb = 0, np = 0;
  while (enum_next(&e, &b)) {
    if (nb < max_batches) {
      hdr[4 * nb] = (int64_t)b.alpha; hdr[4 * nb + 1] = (int64_t)b.beta;
      hdr[4 * nb + 2] = b.nl; hdr[4 * nb + 3] = b.nr;
    }
    if (np + b.nl + b.nr <= max_pairs) {
      expand_range(b.lseg, b.nlseg, 0, b.nl, pairs + 2 * np);
      expand_range(b.rseg, b.nrseg, 0, b.nr, pairs + 2 * (np + b.nl));
    }
    np += b.nl + b.nr;
    nb++;
  }
  free(b.lseg); free(b.rseg);
  enum_free(&e);
  free_tables(t);
  return (nb <= max_batches && np <= max_pairs) ? nb : -nb - 1;
}
