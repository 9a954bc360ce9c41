/*
 * messi.h -- C-ABI of the B200-native MESSI exact 1-NN hot path (libmessi.so).
 *
 * Paper: Peng, Fatourou, Palpanas, "Fast Data Series Indexing for In-Memory Data",
 * arXiv 2110.07519; "P:<line>" cites /root/reference/PAPER.md (section / algorithm).
 *
 * The operation (sec. 2.1): "given a query series S_q of length n, and a
 * collection S of sequences of the same length, n, identify the series S_c in S that has
 * the smallest distance to S_q", under Euclidean distance or DTW with a
 * Sakoe-Chiba band of reach r (sec. 3.4).  The index is the iSAX
 * summary of every series (PAA means -> 8-bit N(0,1)-region symbols) plus an
 * approximate-search order (Alg. 5 line "approxSearch").  Answers are EXACT:
 * the id is the lexicographic minimum of (squared distance in fp64, id) over all rows
 * (ties -> lowest id), and dist = sqrt of that fp64 squared distance (R11-R13).
 *
 * Conventions for every call:
 *   - returns messi_status; MESSI_OK == 0; never aborts; on failure a thread-local message
 *     is available from messi_last_error().
 *   - pointers named *_dev are CUDA device pointers on the index's device; *_host are host
 *     pointers; "query" pointers may be either (detected with cudaPointerGetAttributes).
 *   - work is enqueued on cfg.stream (a cudaStream_t, e.g. torch's current stream); the
 *     non-batch calls synchronise that stream before returning.
 *   - float data is row-major fp32 [count][length]; ids are 0-based, global ids are
 *     cfg.row_begin + local row.
 *
 * Deviations from the contract SURVEY.md 8(b) proposed (all additive): messi_result also
 * carries the exact fp64 d2 (the cross-shard merge key: sqrt loses the order of near-ties)
 * and a reserved word (32-byte records); messi_stats has per-stage counters of this design
 * (tiles, coarse / fine survivors, quantised-bound survivors) instead of the proposed list;
 * messi_config has keep_paa (tests only).  Beyond the four north-star calls the library
 * exports batched and k-NN forms, the shard-linking calls, per-kernel timing and the
 * inspection entry points at the end of this file.
 */
#ifndef MESSI_H
#define MESSI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MESSI_OK = 0,
    MESSI_EINVAL = 1, /* null pointer, bad length/segments/card_bits, reach outside [0, n], count too large */
    MESSI_EEMPTY = 2, /* count == 0 (empty dataset is an error) */
    MESSI_ENOMEM = 3, /* device allocation failed */
    MESSI_ECUDA = 4   /* any other CUDA error (message in messi_last_error()) */
} messi_status;

typedef struct messi_index messi_index; /* opaque; owned by the library until messi_free */

typedef struct {
    int32_t length;    /* n: points per series; n >= 16, n % segments == 0, n <= 8192 */
    int32_t segments;  /* w: PAA segments; 16 only ("w is fixed to 16") */
    int32_t card_bits; /* bits per iSAX symbol; 8 only (256 symbols) */
    int32_t window;    /* approximate-search leaf size; 0 -> 2000 (P:2064-2065 leaf capacity) */
    int32_t device;    /* CUDA ordinal that holds rows_dev and runs every kernel */
    int32_t keep_paa;  /* 1: also keep the fp32 PAA [count][16] (tests); 0: symbols only */
    int64_t row_begin; /* global id of local row 0 (row sharding over GPUs; 0 unsharded) */
    void* stream;      /* cudaStream_t to enqueue on; NULL = legacy default stream */
} messi_config;

typedef struct {
    double dist;      /* sqrt of d2 (fp64, correctly rounded) */
    int64_t id;       /* global id of the nearest series; -1 only if no row has a finite distance */
    double d2;        /* the exact fp64 squared distance (ED^2 or DTW^2): the cross-shard merge key */
    int64_t reserved; /* 0 */
} messi_result;

typedef struct {
    int64_t lb_computed;  /* series lower bounds evaluated (the members of the scanned tiles) */
    int64_t tiles_scanned; /* 512-series tiles whose box bound <= BSF0 * (1 + eps) (scanned) */
    int64_t candidates;   /* series whose iSAX bound <= BSF0 * (1 + eps) */
    int64_t lbk_pass;     /* DTW: candidates passing the LB_Keogh filter against BSF0: the bound
                             from the quantised row, (sqrt(LBK(x^)) - e)^2, at reaches served by
                             the strip refine (r >= 7), the raw LB_Keogh otherwise; where the
                             filter has the reverse bound (n, reach in MESSI_REV_SPECS) that too */
    int64_t refined;      /* real distances computed (fp32) in the refine step */
    int64_t abandoned;    /* real distance computations abandoned early */
    int64_t near_best;    /* fp32 near-ties re-ranked exactly in fp64 */
    int64_t dtw_cells;    /* DTW: valid band cells (|i - j| <= r inside the n x n matrix) of the rows the
                             fp32 refine evaluated -- n(2r+1) - r(r+1) per completed candidate, the
                             rows done for an abandoned one */
    int64_t exact;        /* ED: real distances over the raw fp32 rows = candidates whose
                             quantised-row bound did not prune them; DTW: reverse
                             LB_Keogh bounds evaluated (forward survivors; 0 without that filter) */
    int64_t tiles_listed; /* tiles whose box bound <= BSF0 * (1 + eps) (the filter's list); ED scans
                             those still within the CURRENT BSF when reached (tiles_scanned) */
    int64_t coarse;       /* series whose cardinality-16 bound passed (their 8-bit bound evaluated) */
    double seed_d2;       /* BSF0: squared distance found by the approximate search */
    double bsf_d2;        /* final fp32 best-so-far (squared) before the exact re-rank */
    int64_t rev_paa_pass; /* DTW at strip reaches: candidates that also passed the reverse envelope-PAA
                             bound (the rows' envelope-PAA symbols against the query PAA, DESIGN.md
                             5) -- the series the LB_Keogh filter reads; otherwise = candidates */
} messi_stats;

/* Build the index over `count` rows of length cfg->length (device pointer, borrowed: the
 * caller keeps it alive and unmodified until messi_free; no copy is made).  Runs the iSAX
 * summarisation (Alg. 3, ConvertToiSAX P:710) and the approximate-search key
 * sort on the device.  count must be < 2^31.  *out receives the new index. */
messi_status messi_build(const float* rows_dev, int64_t count, const messi_config* cfg, messi_index** out);

/* Exact 1-NN under ED (Alg. 5 ExactSearch P:933-961 with Alg. 9) of one query
 * of length n (host or device pointer).  *local_best (host) receives this index's best;
 * stats (host, nullable) the per-query counters.  Synchronous. */
messi_status messi_query_ed(messi_index* idx, const float* query, messi_result* local_best, messi_stats* stats);

/* Exact 1-NN under DTW with reach `reach` points, 0 <= reach <= n (Alg. 10). */
messi_status messi_query_dtw(messi_index* idx, const float* query, int32_t reach, messi_result* local_best,
                             messi_stats* stats);

/* Batched, asynchronous forms: nq queries [nq][n] in device memory, answered one after the
 * other (the paper's sequential query model) entirely on cfg.stream with no
 * host synchronisation; results_dev[nq] and stats_dev[nq] (nullable) are device arrays.
 * The caller synchronises the stream before reading them. */
messi_status messi_query_ed_batch(messi_index* idx, const float* queries_dev, int32_t nq,
                                  messi_result* results_dev, messi_stats* stats_dev);
messi_status messi_query_dtw_batch(messi_index* idx, const float* queries_dev, int32_t nq, int32_t reach,
                                   messi_result* results_dev, messi_stats* stats_dev);

/* ---- shards of one row-sharded collection (north_star: "each GPU returns a local (dist,
 * id) minimum") -------------------------------------------------------------------------
 * Linked indexes share each query's best-so-far while the batched ED kernels and the DTW
 * path run (MESSI's single shared BSF): every new local best is also raised into
 * the peers' state for the same query (atomicMax of an epoch-tagged key, over NVLink peer
 * memory between GPUs), and every bound test reads the smallest of them.  Exactness is
 * unchanged: a shard may then prune its own rows down to "no row within the global BSF" (its
 * local answer is then (inf, -1)), and the cross-shard lexicographic min of the local answers
 * (dist.py) is the global one.  Linked shards must make the same sequence of query calls after
 * linking: the epoch = link generation (high byte) | ED launch groups / DTW queries since the
 * link, so a value written for another query or under an earlier link never matches.
 *
 * messi_batch_state_ipc: the CUDA IPC handle (64 bytes into handle_out) of one of this index's
 *   state arrays: set 0 or 1 = the batched ED path's query states, set 2 = the DTW slots.
 * messi_link_peers_ipc: open the handles of npeers (<= 8) peers, handles = npeers x 3 x 64
 *   bytes (peer-major, sets 0, 1, 2), replacing earlier links; npeers = 0 unlinks.
 * messi_link_peers_local: the same for indexes of this process (same or peer-accessible
 *   GPUs; used by the tests to emulate shards on one GPU). */
messi_status messi_batch_state_ipc(messi_index* idx, int32_t set, void* handle_out);
messi_status messi_link_peers_ipc(messi_index* idx, const void* handles, int32_t npeers);
messi_status messi_link_peers_local(messi_index* idx, messi_index* const* peers, int32_t npeers);

/* Exact k-NN under ED (the paper's k-NN variant: the BSF becomes
 * the k-th best distance), 1 <= k <= 64 (k > 1 needs cfg.window <= 4096).  The pruning
 * threshold is the k-th smallest fp32 distance of the rows refined so far (seeded with the
 * k-th smallest of the approximate-search window); every row within it is re-ranked in fp64,
 * and the answer is the k lexicographically smallest (d2, id): ascending, ties to the lowest
 * id; fewer than k rows -> the remaining entries are (inf, -1).
 * messi_query_ed_knn: one query (host or device pointer), results = k messi_result in host
 *   memory, stats (host, nullable).  Synchronous.
 * messi_query_ed_knn_batch: nq queries [nq][n] on the device, results_dev[nq][k] and
 *   stats_dev[nq] (nullable) device arrays; asynchronous on cfg.stream like the 1-NN batch. */
messi_status messi_query_ed_knn(messi_index* idx, const float* query, int32_t k, messi_result* results,
                                messi_stats* stats);
messi_status messi_query_ed_knn_batch(messi_index* idx, const float* queries_dev, int32_t nq, int32_t k,
                                      messi_result* results_dev, messi_stats* stats_dev);

/* Exact k-NN under DTW with reach `reach` (the paper's k-NN for both measures, P:2604-2611,
 * DTW priced at P:2718-2719), 1 <= k <= 64 (k > 1 needs cfg.window <= 4096): BSF0 = the k-th
 * smallest window distance; the refine keeps the k smallest fp32 distances (their k-th is the
 * pruning threshold); every completed candidate within it is re-ranked in fp64 and the answer
 * is the k lexicographically smallest (d2, id), ascending, ties to the lowest id; fewer than k
 * rows -> the remaining entries are (inf, -1).  Same forms as the ED k-NN calls. */
messi_status messi_query_dtw_knn(messi_index* idx, const float* query, int32_t reach, int32_t k, messi_result* results,
                                 messi_stats* stats);
messi_status messi_query_dtw_knn_batch(messi_index* idx, const float* queries_dev, int32_t nq, int32_t reach, int32_t k,
                                       messi_result* results_dev, messi_stats* stats_dev);

/* Exact 1-NN under ED of nq queries [nq][n] (device) by the tensor-core pass (SURVEY 8(f) f4:
 * one stream of the quantised rows per <= 256 queries; tcgen05.mma kind::i8 computes every
 * (row, query) int8 dot product exactly, the epilogue keeps the rows whose quantised-row bound
 * does not exceed the approximate search's BSF0, and those are re-refined exactly:
 * fp32 ED on the raw row, fp64 re-rank).  Same answers as messi_query_ed_batch.  n must be 128
 * or 256 (EINVAL otherwise).  results_dev[nq], stats_dev[nq] (nullable) device arrays;
 * asynchronous on cfg.stream. */
messi_status messi_query_ed_tc_batch(messi_index* idx, const float* queries_dev, int32_t nq, messi_result* results_dev,
                                     messi_stats* stats_dev);

/* Release everything the library allocated for idx.  NULL-safe. */
void messi_free(messi_index* idx);

/* Thread-local text of the last failure ("" if none). */
const char* messi_last_error(void);

/* Kernel launches the library enqueued so far on this index (for bench accounting). */
int64_t messi_launch_count(const messi_index* idx);

/* Per-kernel device timing (bench accounting): with bit 0 of `enable` set the library brackets
 * every launch of the query path with CUDA events on the stream it is launched on; with bit 1
 * set every stage of the per-query (DTW) path runs on cfg.stream, with no overlap between
 * stages or queries (so per-kernel times add up to the step).  kind: 0 seed (prologue +
 * approximate search + tile filter), 1 lower-bound scan (ED: the fused scan + refine
 * kernel), 2 refine (DTW), 3 DTW LB_Keogh filter, 4 exact resolve.  messi_profile_enable
 * resets the accumulators; messi_profile_read synchronises and returns the summed
 * milliseconds and the launch count. */
messi_status messi_profile_enable(messi_index* idx, int32_t enable);
messi_status messi_profile_read(messi_index* idx, int32_t kind, double* total_ms, int64_t* launches);

/* Device time of the build phases (CUDA events on cfg.stream inside messi_build), ms_out[5]:
 * 0 breakpoints + summarisation (PAA, symbols, keys: Alg. 3), 1 the CUB key sort,
 * 2 sorted layout (tiles, 8-bit words, boxes, super-boxes), 3 quantised rows; 4 the last
 * reverse-envelope symbol pass of the DTW path (k_renv, per reach, run by the first strip-reach
 * DTW query of that reach; 0 if none). */
messi_status messi_build_times(const messi_index* idx, double* ms_out);

/* Scan throughput in isolation: one query's prologue and tile filter, then `reps` scans back
 * to back, each timed with CUDA events; *ms_out = summed kernel milliseconds, *coarse_out
 * (nullable) = candidates of the last repetition | (tiles scanned << 32). */
messi_status messi_debug_scan_repeat(messi_index* idx, const float* query_dev, int32_t reps, double* ms_out,
                                     int64_t* coarse_out);

/* ---- inspection entry points (tests) -------------------------------------------------
 * Each runs the QUERY PATH'S OWN KERNELS with their pruning thresholds at +inf (nothing is
 * pruned, nothing abandoned) and scatters what they produce back to row / id order; only the
 * ED refine's inner passes, which live inside the fused kernel, are reached through a small
 * kernel calling the same device functions.  All outputs are device buffers; entries a call
 * did not produce are left NaN.  Synchronous. */

/* The 255 fp32 N(0,1) breakpoints the device derived (O3 reading), into host memory. */
messi_status messi_debug_breakpoints(int32_t device, float* beta32_host);

/* iSAX symbols [count][16] (u8) and, if cfg.keep_paa, PAA [count][16] (fp32) of every row,
 * de-tiled into caller device buffers (paa_dev may be NULL). */
messi_status messi_debug_summaries(messi_index* idx, uint8_t* sym_dev, float* paa_dev);

/* The quantised copy of the rows used by the refine's distance bounds (DESIGN.md §5/§7),
 * back in row order: q8_dev[count][n] int8 c = rint(x / s) in [-127, 127] and meta_dev[count][2]
 * fp32 {s, e}: s a power of two, e >= ||x - s c||_2.  Device buffers. */
messi_status messi_debug_quantised(messi_index* idx, uint8_t* q8_dev, float* meta_dev);

/* Sorted approximate-search keys and the row permutation (device pointers owned by idx). */
messi_status messi_debug_order(messi_index* idx, const uint64_t** skey_dev, const uint32_t** perm_dev);

/* 8-bit iSAX lower bound of every row against one query (device pointer), lb_dev[count]:
 * the scan kernel k_scan (coarse pass, then fine_lb -- the device function the fused ED
 * kernel's fine pass calls) over every tile, with the scan table of the query path: ED
 * (reach < 0) -> mindist (Property 1) from k_prologue_batch's table; DTW
 * (reach >= 0) -> the envelope-PAA bound from k_seed_dtw's.  Squared, fp32, table
 * entries rounded down and summed rounding down. */
messi_status messi_debug_lower_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev);
/* The reverse envelope-PAA bound (the DTW path's filter between the scan and
 * LB_Keogh at strip reaches) of every row for `reach` >= 1, lb_dev[N] in row order:
 * m sum_s max(0, qbar_s - hi(u_s), lo(l_s) - qbar_s)^2 in fp32 rounded down, u_s / l_s the
 * row's envelope-PAA symbols (k_renv).  Reverse LB_Keogh (P:1392-1405 with the series' roles
 * swapped) reduced by PAA as P:1411 does for the query envelope: <= DTW(q, x). */
messi_status messi_debug_rev_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev);

/* Coarse (cardinality-16, the top 4 bits of every symbol) bound of every row against one
 * query with the scan kernel's own arithmetic (coarse_acc, called by scan_tile_coarse):
 * squared, fp32, rounded down, <= the 8-bit bound (the coarse boxes contain the fine ones). */
messi_status messi_debug_coarse_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev);

/* Box bound of every tile (512 consecutive series in approximate-search order; members are
 * rows perm[512*t .. 512*t+511]), lb_dev[ntiles]: ED (reach < 0) -> the batch filter kernel
 * k_filter_batch (fp32 box_lb over the zero runs of the filter table, rounded down); DTW ->
 * the per-query filter k_tile_filter (fp64 bound, rounded to fp32). */
messi_status messi_debug_tile_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev);

/* ED box bound of every super-tile (16 consecutive tiles, the union box) with the filter's
 * box_lb, lb_dev[ceil(ntiles / 16)]. */
messi_status messi_debug_super_bounds(messi_index* idx, const float* query_dev, float* lb_dev);

/* ED refine of `k` local row ids (device u32, distinct), with the query path's device code and
 * nothing pruned: q8_dev[k][2] fp64 = (dh2, L) -- dh2 a lower bound (fp64, error margin
 * subtracted) of ||q^ - x^||^2 between the quantised query and the quantised row, L =
 * sqrt(dh2) - e_q - e_x its lower bound of ||q - x|| (q8i_bound_pass);
 * d32_dev[k] the fp32 squared ED of the exact pass (ed2_group); d64_dev[k] the fp64 canonical
 * re-rank (ed2_exact_g).  The quantised query is the batch path's (k_prologue_batch). */
messi_status messi_debug_ed_refine(messi_index* idx, const float* query_dev, const uint32_t* ids_dev, int32_t k,
                                   double* q8_dev, float* d32_dev, double* d64_dev);

/* DTW filter + refine of `k` local row ids (device u32, distinct) with reach `reach`: the ids
 * are handed to the query path's LB_Keogh filter kernel (threshold +inf) and refine kernel
 * (frozen: threshold +inf, no BSF update, no abandon).  lbk_dev[k] (nullable) = the filter's
 * LB_Keogh -- of the QUANTISED row x^ = s c at reaches served by the strip refine
 * (*quantised = 1), of the raw row otherwise (*quantised = 0); d32_dev[k] (nullable) = the
 * refine kernel's fp32 DTW^2; lbrev_dev[k] (nullable) = the filter's lower bound of the
 * REVERSE LB_Keogh (the query's points against the candidate's envelope, from the quantised
 * row; lbk_rev_q8) where the filter computes one -- strip reaches with (n, reach) in
 * MESSI_REV_SPECS (refine.cuh) -- else NaN (all bits set).  quantised may be NULL. */
messi_status messi_debug_dtw_stages(messi_index* idx, const float* query_dev, int32_t reach, const uint32_t* ids_dev,
                                    int32_t k, float* lbk_dev, float* d32_dev, int32_t* quantised, float* lbrev_dev);

/* For `k` local row ids: d32 = the refine's fp32 squared distance (ED: ed2_group; DTW: the
 * refine kernel via messi_debug_dtw_stages), d64 = the exact fp64 re-rank (ED: ed2_exact_g;
 * DTW: the resolve kernel's dtw_warp_any<double>), lbk (DTW) = the filter kernel's LB_Keogh as
 * in messi_debug_dtw_stages.  reach < 0 -> ED.  Any output pointer may be NULL. */
messi_status messi_debug_distances(messi_index* idx, const float* query_dev, int32_t reach, const uint32_t* ids_dev,
                                   int32_t k, float* d32_dev, double* d64_dev, float* lbk_dev);

#ifdef __cplusplus
}
#endif
#endif /* MESSI_H */
