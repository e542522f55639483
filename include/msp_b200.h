/*
 * msp_b200.h -- C-ABI of the B200-native market-split solver (libmsp_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary.
 *
 * The reference (/root/reference/pkg/src/marketsplit) is pure Python, so its "FFI" for this path is
 * the Python call it makes at the engine dispatch point.  Each entry point
 * below replaces one reference interface:
 *
 *   msp_solve        <- the table path of solve() after reduction/zero-RHS handling:
 *                       build_quarter_tables (enumerate1d.py:86-135) + _make_enumerator
 *                       (solver.py:158-167) + _run_sequential / pipeline_run
 *                       (solver.py:227-234,256-419) + validate_chunked (validate.py:316-379) +
 *                       fastval.join_pairs (fastval.py:116-139) + _confirm_hits (validate.py:285-313),
 *                       and the n <= 12 brute-force branch (solver.py:197-211, oracle.py:27-75).
 *                       Stats mirror SolveStats (solver.py:94-129).
 *   msp_build_tables <- build_quarter_tables (enumerate1d.py:86-135) + _run_ends (:138-145)
 *   msp_alpha_plan   <- the batch stream headers of JitPairSumEnumerator.next_batch
 *                       (fastenum.py:199-218): (alpha, beta, n_left, n_right) per batch
 *   msp_join_alpha   <- validate_chunked(...) on the single batch alpha (validate.py:316-379)
 *
 * Error behaviour mirrors the reference exceptions (solver.py:54-91, validate.py:248-251,274-277,
 * fastval.py:134-135): the return code selects the Python exception the host raises.
 */
#ifndef MSP_B200_H
#define MSP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum msp_status {
  MSP_OK = 0,
  MSP_TIMEOUT = 1,          /* -> SolveTimeout        (solver.py:54-56) */
  MSP_INVALID_ARGUMENT = 2, /* -> ValueError          (solver.py:77-91)  */
  MSP_CUDA_ERROR = 3,       /* -> RuntimeError                           */
  MSP_INTERNAL = 4,         /* -> AssertionError / RuntimeError (fastval.py:134-135, validate.py:274-277) */
  MSP_UNSUPPORTED = 5       /* instance outside the implemented arithmetic modes -> ValueError */
};

enum msp_mode { MSP_MODE_FIRST = 0, MSP_MODE_ALL = 1 };

enum msp_flags {
  MSP_FLAG_PROFILE = 1u << 0,      /* time the dominant kernel per launch with CUDA events */
  MSP_FLAG_FORCE_TABLE_PATH = 1u << 1, /* never take the n <= brute_force_max_n branch */
  MSP_FLAG_JOIN_GLOBAL = 1u << 2,  /* force the global-hash-table join (fallback path) */
  MSP_FLAG_DIAG_HASH_ONLY = 1u << 3, /* diagnostic timing: global path kernels hash but do not join
                                       (results invalid; never set in a real solve) */
  MSP_FLAG_WAVE_LAUNCHES = 1u << 4, /* partitioned waves as per-wave scatter + join launches instead
                                       of the persistent pipeline (parity testing) */
  MSP_FLAG_BATCH_STATS = 1u << 5,   /* fill msp_result.batch_stats: one row per batch, the per-batch
                                       ValidationStats of validate_chunked (validate.py:63-71,316-379) */
  MSP_FLAG_DEGENERATE_HASH = 1u << 6 /* test seam: every key hashes to 0 (the reference's encode_fn
                                       injection, validate.py:161-162,208-216): hash_hits = every
                                       unfiltered (left, right) pair; exact confirmation unchanged.
                                       Runs the global-table join. */
};

typedef struct {
  int32_t m, n;
  const uint64_t *a; /* m x n, row-major; row 0 is the enumerated row (solver.py:214) */
  const uint64_t *d; /* m */
} msp_problem;

typedef struct {
  int32_t mode;              /* msp_mode */
  int32_t device;            /* CUDA ordinal */
  double time_limit_s;       /* <= 0: none (cooperative, checked between waves) */
  uint64_t alpha_lo;         /* shard band: only batches with alpha in [alpha_lo, alpha_hi) */
  uint64_t alpha_hi;         /* 0 = unbounded */
  uint32_t flags;            /* msp_flags */
  int32_t brute_force_max_n; /* < 0 -> 12 (solver.py:48) */
  uint64_t wave_keys;        /* 0 -> default join wave budget (keys per wave) */
  void *stream;              /* cudaStream_t to run on, NULL -> library stream */
  const volatile int32_t *cancel; /* optional cross-rank early exit (first mode): when *cancel != 0
                                     at a wave checkpoint, the solve stops and returns what it has
                                     confirmed so far with stats.cancelled = 1 */
} msp_options;

typedef struct {
  /* SolveStats counters (solver.py:94-129); deterministic in all-mode */
  int64_t batches, candidates_left, candidates_right, filtered_residuals, hash_hits, exact_hits;
  uint64_t row1_pairs_lo, row1_pairs_hi; /* sum over batches of n_left*n_right (128-bit) */
  int64_t peak_table_entries, peak_heap1, peak_heap2;
  double t_build, t_enumerate, t_validate, t_total; /* host wall seconds: t_build = K1 quarter tables
                              (incl. t_init), t_enumerate = the alpha plan (replaces the heap stream),
                              t_validate = join waves + recovery + confirmation */
  int32_t fallback;  /* 0 none, 1 brute-force */
  int32_t waves;     /* join waves executed */
  int64_t kernel_launches; /* kernels this call launched */
  double dev_ms_total;     /* CUDA-event time of the whole device pipeline */
  double dev_ms_tables;    /* table build + plan */
  double dev_ms_join;      /* enumeration + join waves */
  double dev_ms_hot;       /* summed event time of the dominant kernel (MSP_FLAG_PROFILE) */
  int64_t hot_launches;    /* launches of the dominant kernel */
  int64_t hot_pairs;       /* candidate pairs the dominant kernel processed */
  int64_t hot_bytes;       /* algorithmic HBM/L2 bytes of those launches */
  int32_t cancelled;       /* 1: stopped early by msp_options.cancel (counters are partial) */
  int32_t reserved;
  double t_init;           /* host seconds of one-time CUDA init inside this call (context + device
                              state of a first call on the device; 0 afterwards) */
} msp_stats;

typedef struct {
  int64_t n_solutions;
  int32_t n;               /* solution length */
  uint8_t *xbits;          /* n_solutions x n, 0/1, unsorted (host sorts by solution_encoding) */
  msp_stats stats;
  int64_t n_batch_stats;   /* MSP_FLAG_BATCH_STATS: rows of batch_stats (= stats.batches), else 0 */
  int64_t *batch_stats;    /* n_batch_stats x 5, alpha-ascending: (alpha, n_left, n_right,
                              filtered_residuals, hash_hits) of each batch of the stream */
} msp_result;

/* Full solve of one instance (or of the alpha band of one shard).  Blocking. */
int msp_solve(const msp_problem *prob, const msp_options *opt, msp_result *res);
void msp_result_free(msp_result *res);

/* Parity exports. Buffers are caller-owned: weights/contribs u64, masks u32, run_end i64, each
 * sized 2^b_t for the block sizes of _block_sizes(n) (contribs: 2^b_t x m, row-major). */
int msp_build_tables(const msp_problem *prob, int32_t device, uint64_t **weights, uint32_t **masks,
                     uint64_t **contribs, int64_t **run_end);
/* Batch headers in alpha-ascending order; returns the number of batches (may exceed max_batches:
 * only the first max_batches are written), or a negative msp_status. */
int64_t msp_alpha_plan(const msp_problem *prob, int32_t device, int64_t max_batches, uint64_t *alpha,
                       uint64_t *beta, uint64_t *n_left, uint64_t *n_right);
/* Join of the single batch alpha (msp_solve restricted to [alpha, alpha+1)). */
int msp_join_alpha(const msp_problem *prob, const msp_options *opt, uint64_t alpha, msp_result *res);

/* INT32 ops/s of the FNV fold instruction mix on `device` (roofline denominator), or < 0 on error. */
double msp_int32_peak(int32_t device);

/* sizeof(msp_problem), sizeof(msp_options), sizeof(msp_stats), sizeof(msp_result) -> out[0..3]
 * (lets bindings check their struct mirrors without a GPU). */
void msp_abi_sizes(int32_t *out);

/* Free the cached per-device workspace. */
void msp_release(int32_t device);
const char *msp_last_error(void);
int32_t msp_version(void);

#ifdef __cplusplus
}
#endif
#endif
