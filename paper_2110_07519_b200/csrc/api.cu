// api.cu -- the C-ABI of libmessi (include/messi.h): argument checks, device memory,
// stream/event orchestration of the kernels.  The only translation unit; the .cuh files
// hold the kernels.
//
// Query pipeline (per query k, state slot k & 1, three streams):
//   side   : seed(k)  -- prologue tables + approximate search -> BSF0      (latency-bound)
//   main   : scan(k)  -- coarse iSAX lower bound of every series           (HBM-bound)
//   refine : ED : fine bound + real distances + exact re-rank -> result(k)
//            DTW: fine bound + LB_Keogh -> banded DTW -> exact re-rank -> result(k)
// scan(k) waits for seed(k); refine(k) for scan(k); seed(k+2) for refine(k) (slot reuse).
// So seed(k+1) and refine(k) overlap scan(k+1): the HBM stream on `main` is back to back.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/messi.h"
#include "common.cuh"
#include "dtw.cuh"
#include "refine.cuh"
#include "scan.cuh"
#include "summarise.cuh"
#include "fused.cuh"
#include "tc.cuh"

using namespace messi;

// Per-query state sets of the DTW path: queries in flight at once (the stages of
// consecutive queries overlap across the library's streams).
#ifndef MESSI_DTW_SLOTS
#define MESSI_DTW_SLOTS 4  // C4: 2 -> 1136, 3 -> 1232, 4 -> 1281, 6 -> 1303, 8 -> 1307 q/s
#endif

struct Slot {
    QState* st = nullptr;
    float *lut = nullptr, *tab = nullptr, *U = nullptr, *L = nullptr;  // tab: 64 KB scan table
    uint2* cand = nullptr;    // scan survivors (sorted position, 8-bit LB)                      [lazy]
    uint4* list2 = nullptr;   // DTW: LB_Keogh survivors (id, LBK, LBK of the first window, 0)  [lazy]
    uint4* rlist = nullptr;   // DTW: forward survivors queued for the reverse bound               [lazy]
    uint2* cand2 = nullptr;   // DTW: scan survivors passing the reverse envelope-PAA bound         [lazy]
    unsigned* tlist = nullptr;  // tiles surviving the box filter
    NearEntry* near = nullptr;  // near-best (id, d32) of the DTW refine                          [lazy]
    double* rbuf = nullptr;     // DTW resolve: global wavefront scratch for long series         [lazy]
    KnnState* knn = nullptr;    // DTW k-NN: the k smallest fp32 distances of the query          [lazy]
    float* seedd = nullptr;     // DTW k-NN: every approximate-search window distance            [lazy]
    cudaEvent_t ev_seed = nullptr, ev_scan = nullptr, ev_lbk = nullptr, ev_refined = nullptr, ev_done = nullptr;
};

struct messi_index {
    int device = 0;
    cudaStream_t stream = nullptr;  // the caller's stream ("main": scans)
    cudaStream_t side = nullptr;    // library-owned: seeds
    cudaStream_t rstr = nullptr;    // library-owned: ED sub-batches; DTW LB_Keogh filter
    cudaStream_t fstr = nullptr;    // library-owned: DTW LB_Keogh filter of every other query
    cudaStream_t dstr = nullptr;    // library-owned: DTW refine (overlaps the next query's filter)
    cudaStream_t dstr2 = nullptr;   // library-owned: DTW refine of the other slot (its start overlaps
                                    // the tail of the previous query's refine)
    cudaStream_t dstr3 = nullptr, dstr4 = nullptr;  // MESSI_REFINE_STREAMS=4 (experiments)
    cudaStream_t xstr = nullptr;    // library-owned: DTW exact resolve (overlaps the next query's refine)
    cudaStream_t sstr = nullptr;    // library-owned: DTW scans (high priority; MESSI_SCAN_STREAM=0: the caller's stream)
    cudaEvent_t ev_fork = nullptr;
    int n = 0, window = 2000, keep_paa = 0;
    long long N = 0, ntiles = 0, row_begin = 0;
    const float* rows = nullptr;
    int sms = 148;
    // summaries
    uint4* tiles = nullptr;          // cardinality-16 pair bytes, 4 KB per 512 sorted positions
    uint4* sym8 = nullptr;           // 8-bit iSAX words in sorted order [npad][16]
    unsigned char* boxes = nullptr;  // [ntiles][32]: per-segment min / max symbol
    uint4* sboxes = nullptr;         // [nsuper][2]: union boxes of kSuperTiles consecutive tiles
    float* paa = nullptr;
    unsigned char* rows8 = nullptr;  // quantised rows in sorted order [npad][n] (biased int8)
    float2* meta8 = nullptr;         // per sorted position {scale (power of 2), error norm bound}
    unsigned long long* skey = nullptr;
    unsigned* perm = nullptr;
    float *beta32 = nullptr, *lo_w = nullptr, *hi_w = nullptr;
    // DTW: the rows' envelope-PAA symbols for reach renv_reach (k_renv, 32 B per sorted
    // position), built on the first strip-reach DTW query and rebuilt when the reach changes
    uint4* renv = nullptr;
    int renv_reach = -1;
    float renv_ms = 0.0f;
    // batched ED path (fused.cuh): per-query state, tables and tile lists of a launch group
    // (two sets, alternating between consecutive groups of one call)
    struct BatchSet {
        QState* bst = nullptr;
        float *lutc = nullptr, *lutx = nullptr, *lutf = nullptr;
        unsigned* qc = nullptr;   // quantised queries [kBatchMax][n / 4] (4 x s8 per word)
        uint2* btlist = nullptr;  // listed tiles, best-first (k_order_tiles)
        uint2* tstage = nullptr;  // listed tiles as the filter appends them
        KnnState* knn = nullptr;  // k-NN state (lazy)
        float* seedd = nullptr;   // k-NN: the window distances of every query (lazy)
    } bset[2];
    // shards sharing each query's best-so-far (PeerSet): their per-set state arrays, the
    // IPC mappings to close, and the launch epoch (identical on every shard for the same
    // sequence of calls)
    QState* peer_st[3][MESSI_MAX_PEERS] = {};   // sets 0, 1: ED batch states; 2: DTW slot states
    void* peer_ipc[3][MESSI_MAX_PEERS] = {};
    QState** d_peers = nullptr;  // device copy of peer_st
    int npeers = 0;
    unsigned epoch = 0;
    int fused_grid = 0;
    unsigned link_gen = 0;  // links made so far (the high byte of every epoch: see launch_ed_group)
    unsigned dtw_epoch = 0;  // DTW queries since the link (the low bits of the DTW path's epoch)
    QState* slot_st = nullptr;  // the DTW slots' states, contiguous (one IPC handle for all)
    // inspection scratch (messi_debug_*, allocated on first use): inverse permutation, row ->
    // index map of the ids being inspected, tile iota, per-id outputs
    unsigned* dbg_inv = nullptr;
    int* dbg_map = nullptr;
    unsigned* dbg_iota = nullptr;
    double* dbg_gbuf = nullptr;
    // tensor-core batched path (tc.cuh), allocated on its first use
    struct TcSet {
        QState* bst = nullptr;     // per-query state of a pass (<= kTcMaxQ queries)
        unsigned* qc = nullptr;    // quantised queries [kTcMaxQ][n] int8 (the MMA's B operand)
        unsigned* cand = nullptr;  // survivors [kTcMaxQ][kTcCandCap] (sorted positions)
        float4* tcm = nullptr;     // per sorted position: the row's share of the survival test
        CUtensorMap tmA, tmB;      // TMA maps of rows8 and qc (128 B x 128 / 256 rows, 128-byte swizzle)
    } tc;
    // per-query scratch
    Slot slot[MESSI_DTW_SLOTS];
    unsigned long long qcount = 0;
    float* qbuf = nullptr;
    messi_result* res1 = nullptr;
    messi_result* resk = nullptr;    // k-NN single-query results (device)
    messi_stats* stats1 = nullptr;
    long long launches = 0;
    float build_ms[4] = {0, 0, 0, 0};  // build phases (messi_build_times)
    // optional per-kernel event timing
    bool prof = false;
    bool serial = false;  // every per-query stage on the caller's stream (profiling passes)
    struct Ev { int kind; cudaEvent_t a, b; };
    std::vector<Ev> evs;
    std::vector<cudaEvent_t> pool;
};

static_assert(sizeof(messi_result) == 32, "messi_result layout");
static_assert(sizeof(messi_stats) == kStatsBytes, "messi_stats layout");

enum { K_SEED = 0, K_SCAN = 1, K_REFINE = 2, K_LBK = 3, K_RESOLVE = 4, K_KINDS = 5 };

// ------------------------------------------------------------------------------ errors
static thread_local char g_err[512] = "";

static messi_status fail(messi_status s, const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            messi_status s_ = e_ == cudaErrorMemoryAllocation ? MESSI_ENOMEM : MESSI_ECUDA;         \
            return fail(s_, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));     \
        }                                                                                           \
    } while (0)

#define LAUNCHED(idx)                                                                               \
    do {                                                                                            \
        ++(idx)->launches;                                                                          \
        CK(cudaGetLastError());                                                                     \
    } while (0)

#define TRY(x)                                                                                      \
    do {                                                                                            \
        messi_status s_ = (x);                                                                      \
        if (s_ != MESSI_OK) return s_;                                                              \
    } while (0)

template <typename T> static messi_status dalloc(T** p, size_t count)
{
    *p = nullptr;
    if (count == 0) count = 1;
    CK(cudaMalloc((void**)p, count * sizeof(T)));
    return MESSI_OK;
}

static unsigned grid_of_rows(long long n, int threads)
{
    long long g = (n + threads - 1) / threads;
    return (unsigned)(g < 1 ? 1 : g);
}

static cudaEvent_t pool_get(messi_index* idx)
{
    if (!idx->pool.empty()) {
        cudaEvent_t e = idx->pool.back();
        idx->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Brackets one launch with events on its stream when profiling is on.
struct ProfScope {
    messi_index* idx;
    int kind;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    ProfScope(messi_index* i, int k, cudaStream_t st) : idx(i), kind(k), s(st)
    {
        if (idx->prof) {
            a = pool_get(idx);
            cudaEventRecord(a, s);
        }
    }
    ~ProfScope()
    {
        if (idx->prof && a) {
            cudaEvent_t b = pool_get(idx);
            cudaEventRecord(b, s);
            idx->evs.push_back({kind, a, b});
        }
    }
};

// Reaches with a register-band DTW instantiation (DtwThread<R>); others use the warp path.
#define MESSI_DTW_REACHES(X) X(2) X(5) X(12) X(25)

// Strip DTW instantiations (rows per strip H, REM = (2R - 2H + 3) mod H): H = 8 for R >= 7,
// 4 for R in [3, 6], 2 for R in [1, 2].
// K: query-pair copies (16, or 8 when 16 would not fit three CTAs per SM -- large R, H = 8);
// T: threads per CTA (128; 64 with one query copy when even 8 copies and 128 threads would not
// fit: e.g. n = 2048 at a 10% window).
#define MESSI_STRIP_VARIANTS(X)                                                                  \
    X(8, 0, 16, 128) X(8, 1, 16, 128) X(8, 2, 16, 128) X(8, 3, 16, 128) X(8, 4, 16, 128)          \
    X(8, 5, 16, 128) X(8, 6, 16, 128) X(8, 7, 16, 128) X(4, 0, 16, 128) X(4, 1, 16, 128)          \
    X(4, 2, 16, 128) X(4, 3, 16, 128) X(2, 0, 16, 128) X(2, 1, 16, 128) X(8, 0, 8, 128)           \
    X(8, 1, 8, 128) X(8, 2, 8, 128) X(8, 3, 8, 128) X(8, 4, 8, 128) X(8, 5, 8, 128) X(8, 6, 8, 128) \
    X(8, 7, 8, 128) X(8, 0, 1, 64) X(8, 1, 1, 64) X(8, 2, 1, 64) X(8, 3, 1, 64) X(8, 4, 1, 64)      \
    X(8, 5, 1, 64) X(8, 6, 1, 64) X(8, 7, 1, 64)
static const int kStripSmemMax = 227 * 1024;

static int strip_rows(int R)
{
    const char* e = getenv("MESSI_DTW_STRIP_H");  // experiments: rows per strip (8, 4, 2)
    const int h = e ? atoi(e) : 0;
    if ((h == 8 || h == 4 || h == 2) && R >= h - 1) return h;
    return R >= 7 ? 8 : (R >= 3 ? 4 : 2);
}

// Which refine kernel serves reach R: the strip kernel (and with it the strip pipeline: the
// reverse envelope-PAA filter and the quantised LB_Keogh) for every R >= 1 whose shared
// memory fits -- also at R = 2, 5 where a register band (DtwThread<R>) is instantiated: the
// strip pipeline's filters make it 7.5K vs 4.5K q/s at R = 2 on 10M x 256
// (profiles/r02s5_strip_small_reach.txt); else the warp wavefront.  MESSI_DTW_STRIP=0
// (experiments, tests) keeps the register bands and the raw LB_Keogh filter reachable.
// Threads per strip CTA: 128 when the CTA's shared memory fits, else 64 (large reaches).
static int strip_threads(int n, int R) { return strip_qcopies(n, R) == 1 ? 64 : 128; }

static bool use_strip(int n, int R, bool have_band)
{
    const char* e = getenv("MESSI_DTW_STRIP");  // read per launch: tests switch it
    const int force = e ? atoi(e) : -1;
    const int T = strip_threads(n, R);
    const bool fits = R >= 1 && (T == 128 || R >= 7) &&
                      strip_smem(n, R, strip_qcopies(n, R), T) <= (size_t)kStripSmemMax;
    if (force == 0) return false;
    if (force == 1) return fits;
    (void)have_band;  // the register bands (R = 2, 5) stay reachable with MESSI_DTW_STRIP=0
    return fits;
}

static bool strip_trim_on()
{
    static int v = -1;
    if (v < 0) v = (getenv("MESSI_DTW_TRIM") && !strcmp(getenv("MESSI_DTW_TRIM"), "0")) ? 0 : 1;
    return v == 1;
}

static messi_status launch_strip(messi_index* idx, const Slot& sl, int n, int R, const float* q_dev, cudaStream_t rs,
                                 KnnState* knn, int kk, PeerSet ps, int slot)
{
    const int H = strip_rows(R);
    const int rem = (2 * R - 2 * H + 3) % H;
    int K = strip_qcopies(n, R);
    if (const char* e = getenv("MESSI_DTW_QCOPIES"))  // experiments: 8 query-pair copies (H = 8 only)
        if (atoi(e) == 8 && K == 16 && H == 8) K = 8;
    const int T = strip_threads(n, R);
    const size_t smem = strip_smem(n, R, K, T);
    bool launched = false;
#define LAUNCH_S(HH, REM, KK, TT)                                                                                \
    if (!launched && H == HH && rem == REM && K == KK && T == TT) {                                             \
        int occ = 0;                                                                                             \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_refine_dtw_strip<HH, REM, KK, TT>, TT, smem));  \
        const char* oe = getenv("MESSI_DTW_REFINE_OCC"); /* experiments: CTAs per SM */                          \
        if (oe && atoi(oe) > 0 && atoi(oe) < occ) occ = atoi(oe);                                                \
        const unsigned grid = (unsigned)(idx->sms * (occ > 0 ? occ : 1));                                        \
        /* lists under 4 entries per thread run on 2 of 3 CTAs per SM (MESSI_DTW_TRIM=0, experiments: off) */   \
        const unsigned full_min = (occ == 3 && strip_trim_on()) ? 4u * grid * TT : 0u;                           \
        k_refine_dtw_strip<HH, REM, KK, TT><<<grid, TT, smem, rs>>>(idx->rows, n, R, q_dev, sl.U, sl.L, sl.list2, \
                                                                    (unsigned)idx->N, sl.st, sl.near, knn, kk, ps, \
                                                                    slot, full_min);                              \
        launched = true;                                                                                         \
    }
    MESSI_STRIP_VARIANTS(LAUNCH_S)
#undef LAUNCH_S
    if (!launched) return fail(MESSI_EINVAL, "no strip DTW variant for reach %d", R);
    return MESSI_OK;
}

// The DTW seed's distances at strip reaches (k_seed_rows, one thread per window row); seed_d:
// k-NN (every window distance), else 1-NN (BSF0 published).
static messi_status launch_seed_rows(messi_index* idx, const Slot& sl, int n, int R, const float* q_dev,
                                     cudaStream_t s, float* seed_d, PeerSet ps, int slot, int len)
{
    const int H = strip_rows(R);
    const int rem = (2 * R - 2 * H + 3) % H;
    const int K = strip_qcopies(n, R);
    const int T = strip_threads(n, R);
    const size_t smem = strip_smem(n, R, K, T);
    const int grid = (len + T - 1) / T;
    bool launched = false;
#define LAUNCH_SR(HH, REM, KK, TT)                                                                              \
    if (!launched && H == HH && rem == REM && K == KK && T == TT) {                                            \
        k_seed_rows<HH, REM, KK, TT><<<grid > 0 ? grid : 1, TT, smem, s>>>(idx->rows, n, R, q_dev, idx->perm,  \
                                                                          sl.st, seed_d, ps, slot);             \
        launched = true;                                                                                        \
    }
    MESSI_STRIP_VARIANTS(LAUNCH_SR)
#undef LAUNCH_SR
    if (!launched) return fail(MESSI_EINVAL, "no strip DTW variant for reach %d", R);
    return MESSI_OK;
}

// The DTW seed runs one thread per window row (k_seed_prologue + k_seed_rows) at the strip
// reaches (MESSI_SEED_ROWS=0, experiments: the warp-wavefront k_seed_dtw everywhere).
static bool seed_rows_on()
{
    static int v = -1;
    if (v < 0) v = (getenv("MESSI_SEED_ROWS") && !strcmp(getenv("MESSI_SEED_ROWS"), "0")) ? 0 : 1;
    return v == 1;
}

static size_t scan_smem() { return kScanLutBytes; }
static size_t lbk_smem(int n) { return 2 * (size_t)((n + 3) & ~3) * sizeof(float); }

// Function attributes (the shared-memory opt-ins) belong to the current device's context:
// set them once per device (bit `device` of `done`).
static messi_status setup_kernels(int device)
{
    static unsigned long long done = 0;  // guarded by the caller's single-threaded use per device
    const unsigned long long bit = 1ull << (device & 63);
    if (done & bit) return MESSI_OK;
    const int big = 200 * 1024;
    CK(cudaFuncSetAttribute(k_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem()));
    CK(cudaFuncSetAttribute(k_debug_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem()));
    CK(cudaFuncSetAttribute(k_scan_refine_ed<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem(MESSI_MAX_N)));
    CK(cudaFuncSetAttribute(k_scan_refine_ed<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem(MESSI_MAX_N)));
    CK(cudaFuncSetAttribute(k_scan_refine_ed<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem(MESSI_MAX_N)));
    CK(cudaFuncSetAttribute(k_scan_refine_ed<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused_smem(MESSI_MAX_N)));
    CK(cudaFuncSetAttribute(k_filter_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, kFilterQ * kLutF * 4));
    CK(cudaFuncSetAttribute(k_lbk_filter<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_lbk_filter<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_lbk_filter_q8, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_lbk_filter_q8b<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lbkb_smem<256>()));
    CK(cudaFuncSetAttribute(k_debug_dtw64, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_ed_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc_smem_bytes(256)));
    CK(cudaFuncSetAttribute(k_seed_dtw, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_renv, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_rev_paa_filter, cudaFuncAttributeMaxDynamicSharedMemorySize, kRevTabBytes));
    CK(cudaFuncSetAttribute(k_refine_dtw_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_resolve_dtw, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CK(cudaFuncSetAttribute(k_resolve_dtw_knn, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
#define SET_ATTR_S(H, REM, K, T) CK(cudaFuncSetAttribute(k_refine_dtw_strip<H, REM, K, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStripSmemMax)); \
    CK(cudaFuncSetAttribute(k_seed_rows<H, REM, K, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStripSmemMax));
    MESSI_STRIP_VARIANTS(SET_ATTR_S)
#undef SET_ATTR_S
#define SET_ATTR_R(R) CK(cudaFuncSetAttribute(k_refine_dtw<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    MESSI_DTW_REACHES(SET_ATTR_R)
#undef SET_ATTR_R
    done |= bit;
    return MESSI_OK;
}

// Warps per CTA for wavefront kernels holding `per_warp` bytes of shared memory each.
static int warps_for(size_t per_warp, int maxw)
{
    int w = (int)((96 * 1024) / (per_warp ? per_warp : 1));
    return w < 1 ? 1 : (w > maxw ? maxw : w);
}

// ------------------------------------------------------------------------------ build
extern "C" messi_status messi_build(const float* rows_dev, int64_t count, const messi_config* cfg, messi_index** out)
{
    g_err[0] = 0;
    if (!out) return fail(MESSI_EINVAL, "out is NULL");
    *out = nullptr;
    if (!cfg) return fail(MESSI_EINVAL, "cfg is NULL");
    if (count == 0) return fail(MESSI_EEMPTY, "empty collection (count == 0)");
    if (!rows_dev) return fail(MESSI_EINVAL, "rows_dev is NULL");
    if (count < 0 || count > 0x7fffffffLL) return fail(MESSI_EINVAL, "count %lld outside [1, 2^31-1]", (long long)count);
    if (cfg->segments != MESSI_W) return fail(MESSI_EINVAL, "segments must be 16 (got %d)", cfg->segments);
    if (cfg->card_bits != 8) return fail(MESSI_EINVAL, "card_bits must be 8 (got %d)", cfg->card_bits);
    const int n = cfg->length;
    if (n < MESSI_W || n % MESSI_W || n > MESSI_MAX_N)
        return fail(MESSI_EINVAL, "length %d: need 16 <= n <= %d and n %% 16 == 0", n, MESSI_MAX_N);
    if (cfg->window < 0) return fail(MESSI_EINVAL, "window < 0");
    if (cfg->row_begin < 0) return fail(MESSI_EINVAL, "row_begin < 0");

    CK(cudaSetDevice(cfg->device));
    cudaPointerAttributes pa;
    CK(cudaPointerGetAttributes(&pa, rows_dev));
    if (pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged)
        return fail(MESSI_EINVAL, "rows_dev is not a device pointer");
    TRY(setup_kernels(cfg->device));

    messi_index* idx = new (std::nothrow) messi_index();
    if (!idx) return fail(MESSI_ENOMEM, "host allocation failed");
    idx->device = cfg->device;
    idx->stream = (cudaStream_t)cfg->stream;
    idx->n = n;
    idx->window = cfg->window ? cfg->window : 2000;
    idx->keep_paa = cfg->keep_paa ? 1 : 0;
    idx->N = count;
    idx->ntiles = (count + MESSI_TILE_ROWS - 1) / MESSI_TILE_ROWS;
    idx->row_begin = cfg->row_begin;
    idx->rows = rows_dev;
    cudaDeviceGetAttribute(&idx->sms, cudaDevAttrMultiProcessorCount, cfg->device);

    auto bail = [&](messi_status s) { messi_free(idx); return s; };
    const long long N = count;
    const size_t npadrows = (size_t)idx->ntiles * MESSI_TILE_ROWS;
    messi_status s;
    if ((s = dalloc(&idx->tiles, (size_t)idx->ntiles * (MESSI_TILE_BYTES / 16))) ||
        (s = dalloc(&idx->boxes, (size_t)idx->ntiles * 32)) || (s = dalloc(&idx->sym8, npadrows)) ||
        (s = dalloc(&idx->sboxes, (size_t)2 * ((idx->ntiles + kSuperTiles - 1) / kSuperTiles))))
        return bail(s);
    if (idx->keep_paa && (s = dalloc(&idx->paa, (size_t)N * MESSI_W))) return bail(s);
    if ((s = dalloc(&idx->rows8, npadrows * (size_t)n)) || (s = dalloc(&idx->meta8, npadrows))) return bail(s);
    if ((s = dalloc(&idx->skey, (size_t)N)) || (s = dalloc(&idx->perm, (size_t)N))) return bail(s);
    if ((s = dalloc(&idx->beta32, 256)) || (s = dalloc(&idx->lo_w, 256)) || (s = dalloc(&idx->hi_w, 256))) return bail(s);
    if ((s = dalloc(&idx->slot_st, MESSI_DTW_SLOTS))) return bail(s);
    if (cudaMemset(idx->slot_st, 0, sizeof(QState) * MESSI_DTW_SLOTS) != cudaSuccess)  // gbsf = 0: no epoch
        return bail(fail(MESSI_ECUDA, "memset"));
    for (int i = 0; i < MESSI_DTW_SLOTS; ++i) idx->slot[i].st = idx->slot_st + i;
    for (Slot& sl : idx->slot) {
        if ((s = dalloc(&sl.lut, MESSI_W * MESSI_CARD)) || (s = dalloc(&sl.tab, kScanTab)) ||
            (s = dalloc(&sl.U, n)) || (s = dalloc(&sl.L, n)) || (s = dalloc(&sl.tlist, (size_t)idx->ntiles)))
            return bail(s);
        if (cudaEventCreateWithFlags(&sl.ev_seed, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sl.ev_scan, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sl.ev_lbk, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sl.ev_refined, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sl.ev_done, cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(MESSI_ECUDA, "event creation failed"));
    }
    if ((s = dalloc(&idx->qbuf, n)) || (s = dalloc(&idx->res1, 1)) || (s = dalloc(&idx->stats1, 1))) return bail(s);
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (getenv("MESSI_PRIO_EQUAL")) prio_hi = 0;
    // the DTW refine streams below the seed / scan / filter / resolve streams: when SMs free up,
    // CTAs of the filter chain (the pipeline's critical path) are scheduled first and the
    // refine fills what is left (C4 +0.6%; MESSI_PRIO_REFINE_HI=1: all equal, experiments)
    const int prio_ref = getenv("MESSI_PRIO_REFINE_HI") ? prio_hi : prio_lo;
    if (cudaStreamCreateWithPriority(&idx->side, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->rstr, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->fstr, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->dstr, cudaStreamNonBlocking, prio_ref) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->dstr2, cudaStreamNonBlocking, prio_ref) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->dstr3, cudaStreamNonBlocking, prio_ref) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->dstr4, cudaStreamNonBlocking, prio_ref) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->xstr, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&idx->sstr, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&idx->ev_fork, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(MESSI_ECUDA, "stream creation failed"));

    cudaStream_t st = idx->stream;
    unsigned long long* keys_in = nullptr;
    unsigned* ids_in = nullptr;
    uint4* sym_tmp = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    auto cleanup = [&]() {
        cudaFree(keys_in);
        cudaFree(ids_in);
        cudaFree(sym_tmp);
        cudaFree(temp);
    };
    cudaEvent_t bev[5] = {};
    for (auto& e : bev)
        if (cudaEventCreate(&e) != cudaSuccess) return bail(fail(MESSI_ECUDA, "event creation failed"));
    auto free_bev = [&]() {
        for (auto& e : bev) cudaEventDestroy(e);
    };
    do {
        if ((s = dalloc(&keys_in, (size_t)N)) || (s = dalloc(&ids_in, (size_t)N)) || (s = dalloc(&sym_tmp, npadrows))) break;
        cudaEventRecord(bev[0], st);
        k_breakpoints<<<1, 256, 0, st>>>(idx->beta32, idx->lo_w, idx->hi_w);
        ++idx->launches;
        if (cudaGetLastError() != cudaSuccess) { s = fail(MESSI_ECUDA, "k_breakpoints launch"); break; }
        long long grid = idx->ntiles < (long long)idx->sms * 8 ? idx->ntiles : (long long)idx->sms * 8;
        k_summarise<<<(unsigned)grid, 256, 0, st>>>(rows_dev, N, n, idx->beta32, sym_tmp, idx->ntiles, keys_in, ids_in,
                                                    idx->paa);
        ++idx->launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "k_summarise: %s", cudaGetErrorString(e)); break; }
        e = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys_in, idx->skey, ids_in, idx->perm, (int)N, 0, 64, st);
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "cub sort sizing: %s", cudaGetErrorString(e)); break; }
        e = cudaMalloc(&temp, temp_bytes ? temp_bytes : 1);
        if (e != cudaSuccess) { s = fail(MESSI_ENOMEM, "cub temp (%zu B): %s", temp_bytes, cudaGetErrorString(e)); break; }
        cudaEventRecord(bev[1], st);
        e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, idx->skey, ids_in, idx->perm, (int)N, 0, 64, st);
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "cub sort: %s", cudaGetErrorString(e)); break; }
        cudaEventRecord(bev[2], st);
        idx->launches += 4;
        k_layout<<<(unsigned)idx->ntiles, MESSI_TILE_ROWS, 0, st>>>(sym_tmp, idx->perm, N, idx->tiles, idx->sym8,
                                                                    idx->boxes);
        ++idx->launches;
        e = cudaGetLastError();
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "k_layout: %s", cudaGetErrorString(e)); break; }
        {
            const long long nsuper = (idx->ntiles + kSuperTiles - 1) / kSuperTiles;
            k_superbox<<<(unsigned)((nsuper + 255) / 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(idx->boxes),
                                                                       idx->ntiles, idx->sboxes);
            ++idx->launches;
        }
        cudaEventRecord(bev[3], st);
        // the sort's row-id input is free now: the inverse permutation for the row-order quantise
        k_invert_perm<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(idx->perm, N, ids_in);
        ++idx->launches;
        k_quantise<<<(unsigned)(idx->sms * 8), 256, 0, st>>>(rows_dev, ids_in, N, (int64_t)npadrows, n, idx->rows8,
                                                            idx->meta8);
        ++idx->launches;
        cudaEventRecord(bev[4], st);
        e = cudaGetLastError();
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "k_quantise: %s", cudaGetErrorString(e)); break; }
        for (Slot& sl : idx->slot) {
            k_arm<<<1, 1, 0, st>>>(sl.st);
            ++idx->launches;
        }
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "build: %s", cudaGetErrorString(e)); break; }
        for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&idx->build_ms[i], bev[i], bev[i + 1]);
        s = MESSI_OK;
    } while (0);
    cleanup();
    free_bev();
    if (s != MESSI_OK) return bail(s);
    *out = idx;
    return MESSI_OK;
}

extern "C" void messi_free(messi_index* idx)
{
    if (!idx) return;
    cudaSetDevice(idx->device);
    if (idx->side) cudaStreamSynchronize(idx->side);
    if (idx->rstr) cudaStreamSynchronize(idx->rstr);
    if (idx->fstr) cudaStreamSynchronize(idx->fstr);
    if (idx->dstr) cudaStreamSynchronize(idx->dstr);
    if (idx->dstr2) cudaStreamSynchronize(idx->dstr2);
    if (idx->dstr3) cudaStreamSynchronize(idx->dstr3);
    if (idx->dstr4) cudaStreamSynchronize(idx->dstr4);
    if (idx->xstr) cudaStreamSynchronize(idx->xstr);
    if (idx->sstr) cudaStreamSynchronize(idx->sstr);
    if (idx->stream) cudaStreamSynchronize(idx->stream);
    else cudaDeviceSynchronize();
    void* ptrs[] = {idx->tiles, idx->sym8, idx->boxes, idx->sboxes, idx->paa, idx->skey, idx->perm, idx->beta32, idx->lo_w,
                    idx->hi_w,  idx->qbuf,  idx->res1, idx->resk, idx->stats1, idx->rows8, idx->meta8,
                    idx->dbg_inv, idx->dbg_map, idx->dbg_iota, idx->dbg_gbuf, idx->tc.bst, idx->tc.qc, idx->tc.cand,
                    idx->tc.tcm, idx->slot_st, idx->renv};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (auto& row : idx->peer_ipc)
        for (void* p : row)
            if (p) cudaIpcCloseMemHandle(p);
    if (idx->d_peers) cudaFree(idx->d_peers);
    for (auto& bs : idx->bset) {
        void* bp[] = {bs.bst, bs.lutc, bs.lutx, bs.lutf, bs.qc, bs.btlist, bs.tstage, bs.knn, bs.seedd};
        for (void* p : bp)
            if (p) cudaFree(p);
    }
    for (Slot& sl : idx->slot) {
        void* sp[] = {sl.lut, sl.tab, sl.U, sl.L, sl.cand, sl.cand2, sl.list2, sl.rlist, sl.near, sl.tlist, sl.rbuf, sl.knn,
                      sl.seedd};
        for (void* p : sp)
            if (p) cudaFree(p);
        cudaEvent_t es[] = {sl.ev_seed, sl.ev_scan, sl.ev_lbk, sl.ev_refined, sl.ev_done};
        for (cudaEvent_t e : es)
            if (e) cudaEventDestroy(e);
    }
    if (idx->ev_fork) cudaEventDestroy(idx->ev_fork);
    if (idx->side && idx->side != idx->stream) cudaStreamDestroy(idx->side);
    if (idx->rstr && idx->rstr != idx->stream) cudaStreamDestroy(idx->rstr);
    if (idx->fstr) cudaStreamDestroy(idx->fstr);
    if (idx->dstr && idx->dstr != idx->stream) cudaStreamDestroy(idx->dstr);
    if (idx->dstr2 && idx->dstr2 != idx->stream) cudaStreamDestroy(idx->dstr2);
    if (idx->dstr3) cudaStreamDestroy(idx->dstr3);
    if (idx->dstr4) cudaStreamDestroy(idx->dstr4);
    if (idx->xstr && idx->xstr != idx->stream) cudaStreamDestroy(idx->xstr);
    if (idx->sstr) cudaStreamDestroy(idx->sstr);
    for (auto& e : idx->evs) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    for (auto e : idx->pool) cudaEventDestroy(e);
    delete idx;
}

extern "C" const char* messi_last_error(void) { return g_err; }

extern "C" messi_status messi_build_times(const messi_index* idx, double* ms_out)
{
    if (!idx || !ms_out) return fail(MESSI_EINVAL, "NULL argument");
    for (int i = 0; i < 4; ++i) ms_out[i] = idx->build_ms[i];
    ms_out[4] = idx->renv_ms;
    return MESSI_OK;
}

extern "C" int64_t messi_launch_count(const messi_index* idx) { return idx ? idx->launches : 0; }

static messi_status sync_all(messi_index* idx)
{
    CK(cudaStreamSynchronize(idx->stream));
    CK(cudaStreamSynchronize(idx->side));
    CK(cudaStreamSynchronize(idx->rstr));
    CK(cudaStreamSynchronize(idx->fstr));
    CK(cudaStreamSynchronize(idx->dstr));
    CK(cudaStreamSynchronize(idx->dstr2));
    CK(cudaStreamSynchronize(idx->dstr3));
    CK(cudaStreamSynchronize(idx->dstr4));
    CK(cudaStreamSynchronize(idx->xstr));
    CK(cudaStreamSynchronize(idx->sstr));
    return MESSI_OK;
}

extern "C" messi_status messi_profile_enable(messi_index* idx, int32_t enable)
{
    if (!idx) return fail(MESSI_EINVAL, "NULL index");
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    for (auto& e : idx->evs) {
        idx->pool.push_back(e.a);
        idx->pool.push_back(e.b);
    }
    idx->evs.clear();
    idx->prof = (enable & 1) != 0;
    idx->serial = (enable & 2) != 0;
    return MESSI_OK;
}

extern "C" messi_status messi_profile_read(messi_index* idx, int32_t kind, double* total_ms, int64_t* launches)
{
    if (!idx || !total_ms || !launches || kind < 0 || kind >= K_KINDS) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    double ms = 0.0;
    long long cnt = 0;
    for (auto& e : idx->evs) {
        if (e.kind != kind) continue;
        float t = 0.0f;
        CK(cudaEventElapsedTime(&t, e.a, e.b));
        ms += t;
        ++cnt;
    }
    *total_ms = ms;
    *launches = cnt;
    return MESSI_OK;
}

// ---------------------------------------------------------------------------- queries
static int scan_grid(const messi_index* idx)
{
    long long need = (idx->ntiles + kScanWarps - 1) / kScanWarps;
    long long cap = (long long)idx->sms * 2;
    return (int)(need < cap ? (need < 1 ? 1 : need) : cap);
}

static int refine_grid(const messi_index* idx, int per_block_rows)
{
    long long need = (idx->N + per_block_rows - 1) / per_block_rows;
    long long cap = (long long)idx->sms * 4;
    return (int)(need < cap ? (need < 1 ? 1 : need) : cap);
}

// The LB_Keogh filter's front bin: survivors with LBK <= front * BSF0 are refined first
// (MESSI_DTW_FRONT overrides, for experiments; 0 = one bin in filter order).
static float dtw_front()
{
    static float v = -1.0f;
    if (v < 0.0f) {
        const char* e = getenv("MESSI_DTW_FRONT");
        v = e ? (float)atof(e) : 0.5f;
    }
    return v;
}

// Serial mode (messi_profile_enable bit 1, or MESSI_SERIAL=1 for experiments): every stage of
// the per-query path on the caller's stream, no overlap between stages or queries -- so the
// per-kernel event times of a profiling pass add up to the step time.
static bool serial_env()
{
    static int v = -1;
    if (v < 0) v = getenv("MESSI_SERIAL") ? 1 : 0;
    return v == 1;
}
static bool serial_mode(const messi_index* idx) { return idx->serial || serial_env(); }

// Orders the side and refine streams after everything already enqueued on the main stream
// (query buffers written by the caller) -- once per API call, not between batch queries.
static messi_status fork_streams(messi_index* idx)
{
    if (serial_mode(idx)) return MESSI_OK;
    CK(cudaEventRecord(idx->ev_fork, idx->stream));
    CK(cudaStreamWaitEvent(idx->side, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->rstr, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->fstr, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->dstr, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->dstr2, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->dstr3, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->dstr4, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->xstr, idx->ev_fork, 0));
    CK(cudaStreamWaitEvent(idx->sstr, idx->ev_fork, 0));
    return MESSI_OK;
}

// The caller's stream waits for the results of every query enqueued so far.
static messi_status join_streams(messi_index* idx)
{
    for (Slot& sl : idx->slot) CK(cudaStreamWaitEvent(idx->stream, sl.ev_done, 0));
    return MESSI_OK;
}

// Per-slot candidate buffers of the per-query (DTW) path, allocated on its first use: an
// ED-only index never holds them (4 slots x 32 B per row: 12.8 GB at 100M rows).
static messi_status ensure_dtw_buffers(messi_index* idx)
{
    for (Slot& sl : idx->slot) {
        if (!sl.cand) TRY(dalloc(&sl.cand, (size_t)idx->N));
        if (!sl.near) TRY(dalloc(&sl.near, (size_t)idx->N));
        if (!sl.list2) TRY(dalloc(&sl.list2, (size_t)idx->N));
        if (!sl.rlist) TRY(dalloc(&sl.rlist, (size_t)idx->N));
    }
    return MESSI_OK;
}

// Warps of the DTW resolve and whether its wavefront buffers go to global scratch (series
// too long for shared memory at reaches above the register wavefront's).
static const size_t kResolveSmemMax = 200 * 1024;
static int resolve_warps(int n, int reach, bool* global_buf)
{
    *global_buf = resolve_warp_bytes(n, reach, false) > kResolveSmemMax;
    const size_t per = resolve_warp_bytes(n, reach, *global_buf);
    int w = (int)(kResolveSmemMax / per);
    return w < 1 ? 1 : (w > 8 ? 8 : w);
}

static int filter_grid(const messi_index* idx)
{
    long long need = (idx->ntiles + 255) / 256;
    long long cap = (long long)idx->sms * 4;
    return (int)(need < cap ? (need < 1 ? 1 : need) : cap);
}

// Box filter of every tile (side stream, right after the seed: needs BSF0 and the query PAA).
static messi_status launch_tile_filter(messi_index* idx, Slot& sl, cudaStream_t st, PeerSet ps = PeerSet{nullptr, 0, 0u})
{
    k_tile_filter<<<filter_grid(idx), 256, 0, st>>>(idx->boxes, idx->ntiles, idx->n / MESSI_W, idx->lo_w, idx->hi_w,
                                                   sl.st, sl.tlist, nullptr, ps.epoch);
    LAUNCHED(idx);
    return MESSI_OK;
}

static bool scan_stream_on()
{
    static int v = -1;
    if (v < 0) v = (getenv("MESSI_SCAN_STREAM") && !strcmp(getenv("MESSI_SCAN_STREAM"), "0")) ? 0 : 1;
    return v == 1;
}

static messi_status launch_scan(messi_index* idx, Slot& sl, cudaStream_t next, PeerSet peers)
{
    // the scans of consecutive queries in order on one stream: the library's high-priority
    // scan stream (the caller's stream, default priority, in serial mode)
    const cudaStream_t ss = (!serial_mode(idx) && scan_stream_on()) ? idx->sstr : idx->stream;
    CK(cudaStreamWaitEvent(ss, sl.ev_seed, 0));
    {
        ProfScope ps(idx, K_SCAN, ss);
        k_scan<<<scan_grid(idx), 32 * kScanWarps, scan_smem(), ss>>>(idx->tiles, idx->sym8, idx->N, sl.tab,
                                                                     sl.st, sl.cand, sl.tlist, peers.epoch);
        LAUNCHED(idx);
    }
    CK(cudaEventRecord(sl.ev_scan, ss));
    CK(cudaStreamWaitEvent(next, sl.ev_scan, 0));
    return MESSI_OK;
}

static messi_status ensure_batch_buffers(messi_index* idx)
{
    if (idx->bset[0].bst) return MESSI_OK;
    TRY(dalloc(&idx->d_peers, 3 * MESSI_MAX_PEERS));
    CK(cudaMemset(idx->d_peers, 0, sizeof(QState*) * 3 * MESSI_MAX_PEERS));
    for (auto& bs : idx->bset) {
        TRY(dalloc(&bs.bst, kBatchMax));
        CK(cudaMemset(bs.bst, 0, sizeof(QState) * kBatchMax));  // gbsf = 0: no epoch
        TRY(dalloc(&bs.lutc, (size_t)kBatchMax * MESSI_W * MESSI_CARD));
        TRY(dalloc(&bs.lutx, (size_t)kBatchMax * kLutX));
        TRY(dalloc(&bs.lutf, (size_t)kBatchMax * kLutF));
        TRY(dalloc(&bs.qc, (size_t)kBatchMax * (idx->n / 4)));
        TRY(dalloc(&bs.btlist, (size_t)kBatchMax * (size_t)idx->ntiles));
        TRY(dalloc(&bs.tstage, (size_t)kBatchMax * (size_t)idx->ntiles));
    }
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scan_refine_ed<false, false>, 32 * kFusedWarps, fused_smem(idx->n)));
    if (occ < 1) return fail(MESSI_ECUDA, "fused kernel does not fit an SM (n = %d)", idx->n);
    idx->fused_grid = idx->sms * occ;
    return MESSI_OK;
}

// One group of B <= kBatchMax queries of the batched ED path (fused.cuh) on stream st with
// state set bs: prologue, seed, tile filter, the fused scan + refine kernel, finalise.
static messi_status launch_ed_group(messi_index* idx, const messi_index::BatchSet& bs, cudaStream_t st, const float* q, int B,
                                    messi_result* res, messi_stats* stats, int k)
{
    KnnState* knn = k > 1 ? bs.knn : nullptr;
    float* seed_d = k > 1 ? bs.seedd : nullptr;
    const int set = (int)(&bs - idx->bset);
    PeerSet peers;
    peers.st = idx->d_peers + set * MESSI_MAX_PEERS;
    peers.n = idx->npeers;
    // epoch = link generation (high byte) | launch groups since that link (low 24 bits): every
    // shard of one link counts the same groups (they make the same batch calls after linking),
    // and a value a peer wrote under an earlier link never carries a current epoch
    idx->epoch = (idx->epoch + 1) & 0xffffffu;
    peers.epoch = ((idx->link_gen & 0xffu) << 24) | idx->epoch;
    if (peers.n == 0) peers.epoch = 0;  // unlinked: kernels read the local BSF only
    const int n = idx->n;
    const size_t qsm = (size_t)((n + 3) & ~3) * sizeof(float);
    const int len = (int)(idx->window < idx->N ? idx->window : idx->N);
    {
        ProfScope ps(idx, K_SEED, st);
        k_prologue_batch<<<B, 256, qsm, st>>>(q, n, idx->beta32, idx->lo_w, idx->hi_w, idx->skey, idx->N, idx->window,
                                              bs.lutc, bs.lutx, bs.lutf, bs.bst, knn, bs.qc);
        LAUNCHED(idx);
        dim3 sg((unsigned)((len + kSeedRowsPerCta - 1) / kSeedRowsPerCta), (unsigned)B);
        k_seed_batch<<<sg, 256, qsm, st>>>(q, n, idx->rows, idx->perm, bs.bst, peers, seed_d, idx->window);
        LAUNCHED(idx);
        if (knn) {
            int np = 1;
            while (np < len) np <<= 1;
            k_seed_select<<<B, 1024, (size_t)np * sizeof(float), st>>>(seed_d, idx->window, k, bs.bst, peers, -1);
            LAUNCHED(idx);
        }
        const long long nsuper = (idx->ntiles + kSuperTiles - 1) / kSuperTiles;
        const int npairs = (B + kFilterQ - 1) / kFilterQ;
        long long fx = (nsuper + 255) / 256;
        long long fcap = (long long)idx->sms * 8 / npairs + 1;
        if (const char* e = getenv("MESSI_FILTER_CTAS"))  // experiments: filter CTAs per query pair
            fcap = atoi(e) > 0 ? atoi(e) : fcap;
        if (fx > fcap) fx = fcap;
        dim3 fg((unsigned)fx, (unsigned)npairs);
        k_filter_batch<<<fg, 256, kFilterQ * kLutF * 4, st>>>(reinterpret_cast<const uint4*>(idx->boxes), idx->sboxes,
                                                              idx->ntiles, nsuper, bs.lutf, bs.bst, B, bs.tstage,
                                                              peers.epoch);
        LAUNCHED(idx);
        k_order_tiles<<<dim3(kOrderCtas, B), 256, 0, st>>>(bs.tstage, bs.bst, idx->ntiles, bs.btlist);
        LAUNCHED(idx);
    }
    {
        ProfScope ps(idx, K_SCAN, st);
#define FUSED_ARGS                                                                                        \
    idx->tiles, idx->sym8, idx->ntiles, idx->N, n, q, bs.lutx, bs.btlist, bs.bst, B, idx->rows8, idx->meta8, \
        bs.qc, idx->perm, idx->rows, peers, knn, k
        const dim3 fg(idx->fused_grid), fb(32 * kFusedWarps);
        const size_t fs = fused_smem(n);
        if (peers.n > 0 && k > 1) k_scan_refine_ed<true, true><<<fg, fb, fs, st>>>(FUSED_ARGS);
        else if (peers.n > 0) k_scan_refine_ed<true, false><<<fg, fb, fs, st>>>(FUSED_ARGS);
        else if (k > 1) k_scan_refine_ed<false, true><<<fg, fb, fs, st>>>(FUSED_ARGS);
        else k_scan_refine_ed<false, false><<<fg, fb, fs, st>>>(FUSED_ARGS);
#undef FUSED_ARGS
        LAUNCHED(idx);
        k_finalise_batch<<<(B + 127) / 128, 128, 0, st>>>(bs.bst, B, idx->N, idx->row_begin, res, stats, knn, k);
        LAUNCHED(idx);
    }
    return MESSI_OK;
}

// The batched ED path for nq queries [nq][n] on the device: one group per kBatchMax queries
// on the caller's stream.  (Splitting a batch over the two library streams, to overlap one
// group's prologue / filter with the other's fused kernel, was measured slower: each
// persistent kernel then balances fewer queries.)
static messi_status run_ed_batch(messi_index* idx, const float* queries_dev, int nq, messi_result* results_dev,
                                 messi_stats* stats_dev, int k = 1)
{
    TRY(ensure_batch_buffers(idx));
    if (k > 1)
        for (auto& bs : idx->bset) {
            if (!bs.knn) TRY(dalloc(&bs.knn, kBatchMax));
            if (!bs.seedd) TRY(dalloc(&bs.seedd, (size_t)kBatchMax * idx->window));
        }
    const int n = idx->n;
    for (int g0 = 0; g0 < nq; g0 += kBatchMax) {
        const int B = nq - g0 < kBatchMax ? nq - g0 : kBatchMax;
        TRY(launch_ed_group(idx, idx->bset[(g0 / kBatchMax) & 1], idx->stream, queries_dev + (size_t)g0 * n, B,
                            results_dev + (size_t)g0 * k, stats_dev ? stats_dev + g0 : nullptr, k));
    }
    return MESSI_OK;
}

// The refine kernel of reach R (see use_strip): the strip kernel, a register band, or the
// warp wavefront.
static bool dtw_uses_strip(int n, int reach)
{
    bool band = false;
#define HAVE_R(R) band = band || reach == R;
    MESSI_DTW_REACHES(HAVE_R)
#undef HAVE_R
    return use_strip(n, reach, band);
}

// DTW step 1: the LB_Keogh filter of the slot's candidates (list sl.cand, count and threshold
// in sl.st) into list2 -- over the quantised rows at strip reaches (the strip refine's tail
// bound uses the same terms), else over the raw rows.
// MESSI_NO_REV=1 (experiments): the forward-only filter k_lbk_filter_q8 at every reach.
static bool no_rev_env()
{
    static int v = -1;
    if (v < 0) v = getenv("MESSI_NO_REV") ? 1 : 0;
    return v == 1;
}

// The reverse bound (n, reach in MESSI_REV_SPECS, strip reaches): the forward filter
// k_lbk_filter_q8 queues its survivors with forward bound <= rho * BSF0 (MESSI_REV_RHO,
// default 1: all of them) and k_lbk_rev_q8 evaluates the queue with every lane busy
// (MESSI_REV_MODE=fused, experiments: both bounds in one kernel, k_lbk_filter_q8r).
static float rev_rho()
{
    static float v = -1.0f;
    if (v < 0.0f) {
        const char* e = getenv("MESSI_REV_RHO");
        v = e ? (float)atof(e) : 1.0f;
    }
    return v;
}
static bool lbk_bulk()  // MESSI_LBK_BULK=0 (experiments): the LDG forward filter instead of the bulk-copy one
{
    static int v = -1;
    if (v < 0) v = (getenv("MESSI_LBK_BULK") && !strcmp(getenv("MESSI_LBK_BULK"), "0")) ? 0 : 1;
    return v == 1;
}
static bool rev_fused()
{
    static int v = -1;
    if (v < 0) v = (getenv("MESSI_REV_MODE") && !strcmp(getenv("MESSI_REV_MODE"), "fused")) ? 1 : 0;
    return v == 1;
}

// The reverse envelope-PAA filter (k_rev_paa_filter) between the scan and the LB_Keogh
// filter, at the strip reaches >= 1 (MESSI_NO_RENV=1, experiments: off).
static bool renv_env_off()
{
    static int v = -1;
    if (v < 0) v = getenv("MESSI_NO_RENV") ? 1 : 0;
    return v == 1;
}
static bool renv_on(const messi_index* idx, int reach)
{
    return !renv_env_off() && reach >= 1 && idx->renv && idx->renv_reach == reach;
}

// The rows' envelope-PAA symbols for `reach` (k_renv over every sorted position, on the
// caller's stream ahead of the query's scan), built when the reach differs from the last
// built one; earlier queries (which may read the old symbols) are joined first.
static messi_status ensure_renv(messi_index* idx, int reach)
{
    if (renv_env_off() || reach < 1 || idx->renv_reach == reach) return MESSI_OK;
    if (!idx->renv) TRY(dalloc(&idx->renv, 2 * (size_t)idx->N));
    for (Slot& sl : idx->slot)
        if (!sl.cand2) TRY(dalloc(&sl.cand2, (size_t)idx->N));
    TRY(join_streams(idx));
    const int n = idx->n;
    int wr = (int)((96 * 1024) / ((size_t)12 * n));
    wr = wr < 1 ? 1 : (wr > 8 ? 8 : wr);
    long long need = (idx->N + wr - 1) / wr, cap = (long long)idx->sms * 16;
    cudaEvent_t a = nullptr, b = nullptr;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, idx->stream));
    k_renv<<<(int)(need < cap ? need : cap), 32 * wr, (size_t)wr * 12 * n, idx->stream>>>(idx->rows, idx->perm, idx->N, n,
                                                                                       reach, idx->beta32, idx->renv);
    LAUNCHED(idx);
    CK(cudaEventRecord(b, idx->stream));
    CK(cudaEventSynchronize(b));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    idx->renv_ms = ms;
    idx->renv_reach = reach;
    return MESSI_OK;
}

static messi_status launch_lbk_filter(messi_index* idx, Slot& sl, int reach, bool strip, const float* q_dev,
                                      cudaStream_t rs, float* rev_out = nullptr)
{
    const int n = idx->n;
    bool rev = false;
    // the scan's candidates, or those of them passing the reverse envelope-PAA bound
    const uint2* cand = sl.cand;
    const unsigned* cnt_p = &sl.st->cand_count;
    if (strip && renv_on(idx, reach)) {
        k_rev_paa_filter<<<idx->sms * 3, 256, kRevTabBytes, rs>>>(sl.cand, idx->renv, idx->lo_w, idx->hi_w, n / MESSI_W,
                                                                  sl.st, sl.cand2, 0);
        LAUNCHED(idx);
        cand = sl.cand2;
        cnt_p = &sl.st->rcand_count;
    }
#define LAUNCH_REV(NN, RR)                                                                                        \
    if (strip && !rev && n == NN && reach == RR && !no_rev_env()) {                                             \
        if (rev_fused()) {                                                                                        \
            k_lbk_filter_q8r<NN, RR><<<idx->sms * 8, 128, 0, rs>>>(sl.cand, idx->perm, idx->rows8, idx->meta8,   \
                                                                    sl.U, sl.L, q_dev, sl.st, sl.list2,         \
                                                                    (unsigned)idx->N, dtw_front(), rev_out);    \
        } else {                                                                                                  \
            if (lbk_bulk())                                                                                       \
                k_lbk_filter_q8b<NN><<<idx->sms * 3, 128, lbkb_smem<NN>(), rs>>>(                                \
                    cand, idx->perm, idx->rows8, idx->meta8, sl.U, sl.L, sl.st, sl.list2, (unsigned)idx->N,       \
                    dtw_front(), sl.rlist, rev_rho(), 0x4B000000u, cnt_p);                                       \
            else                                                                                                  \
                k_lbk_filter_q8<<<idx->sms * 8, 128, 2 * (size_t)((n + 15) & ~15) * sizeof(float), rs>>>(         \
                    cand, idx->perm, idx->rows8, idx->meta8, n, sl.U, sl.L, sl.st, sl.list2, (unsigned)idx->N,    \
                    dtw_front(), sl.rlist, rev_rho(), cnt_p);                                                    \
            LAUNCHED(idx);                                                                                        \
            k_lbk_rev_q8<NN, RR><<<idx->sms * 8, 128, 0, rs>>>(sl.rlist, idx->perm, idx->rows8, q_dev, sl.st,     \
                                                                sl.list2, (unsigned)idx->N, dtw_front(), rev_out, \
                                                                rev_out ? idx->dbg_map : nullptr);               \
        }                                                                                                         \
        rev = true;                                                                                               \
    }
    MESSI_REV_SPECS(LAUNCH_REV)
#undef LAUNCH_REV
    if (rev) {
    } else if (strip)
        k_lbk_filter_q8<<<idx->sms * 8, 128, 2 * (size_t)((n + 15) & ~15) * sizeof(float), rs>>>(
            cand, idx->perm, idx->rows8, idx->meta8, n, sl.U, sl.L, sl.st, sl.list2, (unsigned)idx->N, dtw_front(),
            nullptr, 0.0f, cnt_p);
    else
        k_lbk_filter<4><<<refine_grid(idx, 1024) * 2, 128, lbk_smem(n), rs>>>(
            sl.cand, idx->perm, idx->rows, n, sl.U, sl.L, reach, sl.st, sl.list2, (unsigned)idx->N, dtw_front());
    LAUNCHED(idx);
    return MESSI_OK;
}

// DTW step 2: banded fp32 DTW of the list2 entries (near-best entries to sl.near).
static messi_status launch_dtw_refine(messi_index* idx, Slot& sl, int reach, bool strip, const float* q_dev,
                                      cudaStream_t rs, int kk = 1, PeerSet ps = PeerSet{nullptr, 0, 0u}, int slot = 0)
{
    KnnState* knn = kk > 1 ? sl.knn : nullptr;
    const int n = idx->n;
    const int npad = (n + 3) & ~3;
    const size_t qsm = (size_t)npad * sizeof(float);
    bool launched = false;
#ifdef MESSI_TIMING_KNOBS  // critical-path experiments only (WRONG answers): never in the default build
    static const bool skip = getenv("MESSI_TIMING_SKIP_REFINE") != nullptr;
    if (skip) return MESSI_OK;
#endif
    if (strip) {
        TRY(launch_strip(idx, sl, n, reach, q_dev, rs, knn, kk, ps, slot));
        launched = true;
    }
#define LAUNCH_R(R)                                                                                           \
    if (!launched && reach == R) {                                                                            \
        int occ = 0;                                                                                          \
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_refine_dtw<R>, 128, 3 * qsm));               \
        k_refine_dtw<R><<<idx->sms * (occ > 0 ? occ : 1), 128, 3 * qsm, rs>>>(idx->rows, n, q_dev, sl.U, sl.L, \
                                                                            sl.list2, (unsigned)idx->N, sl.st, \
                                                                            sl.near, knn, kk, ps, slot);      \
        launched = true;                                                                                      \
    }
    MESSI_DTW_REACHES(LAUNCH_R)
#undef LAUNCH_R
    if (!launched) {
        const int wr = warps_for((size_t)4 * npad * sizeof(float), 8);
        k_refine_dtw_warp<<<idx->sms * 4, 32 * wr, qsm + (size_t)wr * 4 * npad * sizeof(float), rs>>>(
            idx->rows, n, reach, q_dev, sl.list2, (unsigned)idx->N, sl.st, sl.near, knn, kk, ps, slot);
    }
    LAUNCHED(idx);
    return MESSI_OK;
}

static messi_status ensure_dtw_knn(messi_index* idx)
{
    for (Slot& sl : idx->slot) {
        if (!sl.knn) TRY(dalloc(&sl.knn, 1));
        if (!sl.seedd) TRY(dalloc(&sl.seedd, (size_t)idx->window));
    }
    return MESSI_OK;
}

// One DTW query (k = 1: 1-NN; k > 1: k-NN, results res[k]) on the next slot, staged over the
// library's streams (serial: all on the caller's stream).
static messi_status run_dtw(messi_index* idx, const float* q_dev, int reach, messi_result* res, messi_stats* stats,
                            int kk = 1)
{
    if (dtw_uses_strip(idx->n, reach)) TRY(ensure_renv(idx, reach));
    const int slot = (int)(idx->qcount++ % MESSI_DTW_SLOTS);
    Slot& sl = idx->slot[slot];
    const bool ser = serial_mode(idx);
    // shards linked: the slot's best-so-far is shared with the peers' same slot (the same
    // query when the shards make the same DTW calls since the link), tagged like the ED path
    PeerSet peers{nullptr, 0, 0u};
    if (idx->npeers > 0) {
        idx->dtw_epoch = (idx->dtw_epoch + 1) & 0xffffffu;
        peers.st = idx->d_peers + 2 * MESSI_MAX_PEERS;
        peers.n = idx->npeers;
        peers.epoch = ((idx->link_gen & 0xffu) << 24) | idx->dtw_epoch;
    }
    cudaStream_t side = ser ? idx->stream : idx->side;
    cudaStream_t rs = ser ? idx->stream : idx->rstr;
    const int n = idx->n;
    const int npad = (n + 3) & ~3;
    const size_t qsm = (size_t)npad * sizeof(float);
    int len = (int)(idx->window < idx->N ? idx->window : idx->N);
    const size_t seed_warp = (size_t)(npad + 3 * n) * sizeof(float);
    const int wf = warps_for(seed_warp, 8);
    int seed_grid = (len + wf - 1) / wf;
    if (seed_grid > idx->sms * 4) seed_grid = idx->sms * 4;
    CK(cudaStreamWaitEvent(side, sl.ev_done, 0));
    // arm the slot for this query (whatever the previous query on it did, e.g. a launch that
    // failed part-way): BSF +inf, every counter 0
    if (kk > 1) k_arm_knn<<<1, 1, 0, side>>>(sl.st, sl.knn);
    else k_arm<<<1, 1, 0, side>>>(sl.st);
    LAUNCHED(idx);
    {
        ProfScope ps(idx, K_SEED, side);
        if (dtw_uses_strip(n, reach) && seed_rows_on()) {  // one thread per window row
            k_seed_prologue<<<1, 256, qsm, side>>>(q_dev, n, reach, idx->skey, idx->N, idx->window, idx->beta32,
                                                   idx->lo_w, idx->hi_w, sl.lut, sl.tab, sl.U, sl.L, sl.st);
            LAUNCHED(idx);
            TRY(launch_seed_rows(idx, sl, n, reach, q_dev, side, kk > 1 ? sl.seedd : nullptr, peers, slot, len));
        } else {
            k_seed_dtw<<<seed_grid, 32 * wf, qsm + wf * seed_warp, side>>>(
                q_dev, n, reach, idx->rows, idx->skey, idx->perm, idx->N, idx->window, idx->beta32, idx->lo_w,
                idx->hi_w, sl.lut, sl.tab, sl.U, sl.L, sl.st, kk > 1 ? sl.seedd : nullptr, peers, slot);
        }
        LAUNCHED(idx);
        if (kk > 1) {  // BSF0 = the k-th smallest window distance
            int np = 1;
            while (np < len) np <<= 1;
            k_seed_select<<<1, 1024, (size_t)np * sizeof(float), side>>>(sl.seedd, idx->window, kk, sl.st, peers, slot);
            LAUNCHED(idx);
        }
        TRY(launch_tile_filter(idx, sl, side, peers));
    }
    CK(cudaEventRecord(sl.ev_seed, side));
    TRY(launch_scan(idx, sl, rs, peers));
    const bool strip = dtw_uses_strip(n, reach);
#ifdef MESSI_TIMING_KNOBS  // critical-path experiments only (WRONG answers): never in the default build
    static const bool skipf = getenv("MESSI_TIMING_SKIP_FILTER") != nullptr;
#else
    constexpr bool skipf = false;
#endif
    if (!ser && (idx->qcount & 1)) {  // filters of consecutive queries on two streams (C4: +2%)
        rs = idx->fstr;
        CK(cudaStreamWaitEvent(rs, sl.ev_scan, 0));
    }
    {
        ProfScope ps(idx, K_LBK, rs);
        if (!skipf) TRY(launch_lbk_filter(idx, sl, reach, strip, q_dev, rs));
    }
    // the refine and the resolve run on their own stream: the LB_Keogh filter of the next
    // query (bandwidth-bound) overlaps this query's band DP (latency / ALU-bound)
    CK(cudaEventRecord(sl.ev_lbk, rs));
    if (!ser) {  // qcount was advanced for this query
        static const int nref = getenv("MESSI_REFINE_STREAMS") ? atoi(getenv("MESSI_REFINE_STREAMS")) : 2;
        const cudaStream_t rst[4] = {idx->dstr, idx->dstr2, idx->dstr3, idx->dstr4};
        rs = rst[idx->qcount % (nref == 4 ? 4 : 2)];
    }
    CK(cudaStreamWaitEvent(rs, sl.ev_lbk, 0));
    {
        ProfScope ps(idx, K_REFINE, rs);
        TRY(launch_dtw_refine(idx, sl, reach, strip, q_dev, rs, kk, peers, slot));
    }
    // the exact resolve of this query overlaps the next query's refine (another slot)
    CK(cudaEventRecord(sl.ev_refined, rs));
    if (!ser) rs = idx->xstr;
    CK(cudaStreamWaitEvent(rs, sl.ev_refined, 0));
    {
        bool gb = false;
        const int wr = resolve_warps(n, reach, &gb);
        if (gb && !sl.rbuf) TRY(dalloc(&sl.rbuf, (size_t)8 * 3 * n));
        ProfScope ps(idx, K_RESOLVE, rs);
        if (kk > 1)
            k_resolve_dtw_knn<<<1, 32 * wr, wr * resolve_warp_bytes(n, reach, gb), rs>>>(
                idx->rows, n, reach, q_dev, sl.near, sl.st, idx->N, idx->row_begin, res, stats, gb ? sl.rbuf : nullptr,
                reinterpret_cast<double2*>(sl.list2), kk);
        else
            k_resolve_dtw<<<1, 32 * wr, wr * resolve_warp_bytes(n, reach, gb), rs>>>(
                idx->rows, n, reach, q_dev, sl.near, sl.st, idx->N, idx->row_begin, res, stats, gb ? sl.rbuf : nullptr);
        LAUNCHED(idx);
    }
    CK(cudaEventRecord(sl.ev_done, rs));
    return MESSI_OK;
}

// Copies a host-or-device query into the index's query buffer; returns the device pointer.
static messi_status stage_query(messi_index* idx, const float* query, const float** q_dev)
{
    cudaPointerAttributes pa;
    cudaError_t e = cudaPointerGetAttributes(&pa, query);
    if (e != cudaSuccess) {
        cudaGetLastError();
        pa.type = cudaMemoryTypeUnregistered;
    }
    if (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged) {
        if (pa.device != idx->device) return fail(MESSI_EINVAL, "query lives on device %d, index on %d", pa.device, idx->device);
        *q_dev = query;
        return MESSI_OK;
    }
    // the buffer may still be read by an earlier query on the refine stream
    TRY(join_streams(idx));
    CK(cudaMemcpyAsync(idx->qbuf, query, (size_t)idx->n * sizeof(float), cudaMemcpyHostToDevice, idx->stream));
    *q_dev = idx->qbuf;
    return MESSI_OK;
}

static messi_status finish_single(messi_index* idx, messi_result* local_best, messi_stats* stats)
{
    TRY(join_streams(idx));
    CK(cudaMemcpyAsync(local_best, idx->res1, sizeof(messi_result), cudaMemcpyDeviceToHost, idx->stream));
    if (stats) CK(cudaMemcpyAsync(stats, idx->stats1, sizeof(messi_stats), cudaMemcpyDeviceToHost, idx->stream));
    CK(cudaStreamSynchronize(idx->stream));
    return MESSI_OK;
}

extern "C" messi_status messi_query_ed(messi_index* idx, const float* query, messi_result* local_best, messi_stats* stats)
{
    g_err[0] = 0;
    if (!idx || !query || !local_best) return fail(MESSI_EINVAL, "NULL argument");
    CK(cudaSetDevice(idx->device));
    const float* q = nullptr;
    TRY(stage_query(idx, query, &q));
    TRY(run_ed_batch(idx, q, 1, idx->res1, idx->stats1));
    return finish_single(idx, local_best, stats);
}

extern "C" messi_status messi_query_dtw(messi_index* idx, const float* query, int32_t reach, messi_result* local_best,
                                        messi_stats* stats)
{
    g_err[0] = 0;
    if (!idx || !query || !local_best) return fail(MESSI_EINVAL, "NULL argument");
    if (reach < 0 || reach > idx->n) return fail(MESSI_EINVAL, "reach %d outside [0, %d]", reach, idx->n);
    CK(cudaSetDevice(idx->device));
    TRY(ensure_dtw_buffers(idx));
    const float* q = nullptr;
    TRY(stage_query(idx, query, &q));
    TRY(fork_streams(idx));
    TRY(run_dtw(idx, q, reach, idx->res1, idx->stats1));
    return finish_single(idx, local_best, stats);
}

extern "C" messi_status messi_query_ed_batch(messi_index* idx, const float* queries_dev, int32_t nq,
                                             messi_result* results_dev, messi_stats* stats_dev)
{
    g_err[0] = 0;
    if (!idx || !queries_dev || !results_dev || nq < 0) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    TRY(join_streams(idx));  // earlier DTW queries (other streams) before the ED batch reuses qbuf users
    if (nq == 0) return MESSI_OK;
    return run_ed_batch(idx, queries_dev, nq, results_dev, stats_dev);
}

static messi_status check_k(const messi_index* idx, int32_t k)
{
    if (k < 1 || k > MESSI_MAX_K) return fail(MESSI_EINVAL, "k = %d outside [1, %d]", k, MESSI_MAX_K);
    if (k > 1 && idx->window > 4096) return fail(MESSI_EINVAL, "k-NN needs an approximate-search window <= 4096");
    return MESSI_OK;
}

extern "C" messi_status messi_query_ed_knn(messi_index* idx, const float* query, int32_t k, messi_result* results,
                                           messi_stats* stats)
{
    g_err[0] = 0;
    if (!idx || !query || !results) return fail(MESSI_EINVAL, "NULL argument");
    TRY(check_k(idx, k));
    CK(cudaSetDevice(idx->device));
    if (k == 1) return messi_query_ed(idx, query, results, stats);
    const float* q = nullptr;
    TRY(stage_query(idx, query, &q));
    if (!idx->resk) TRY(dalloc(&idx->resk, MESSI_MAX_K));
    TRY(run_ed_batch(idx, q, 1, idx->resk, idx->stats1, k));
    TRY(join_streams(idx));
    CK(cudaMemcpyAsync(results, idx->resk, sizeof(messi_result) * k, cudaMemcpyDeviceToHost, idx->stream));
    if (stats) CK(cudaMemcpyAsync(stats, idx->stats1, sizeof(messi_stats), cudaMemcpyDeviceToHost, idx->stream));
    CK(cudaStreamSynchronize(idx->stream));
    return MESSI_OK;
}

extern "C" messi_status messi_query_ed_knn_batch(messi_index* idx, const float* queries_dev, int32_t nq, int32_t k,
                                                 messi_result* results_dev, messi_stats* stats_dev)
{
    g_err[0] = 0;
    if (!idx || !queries_dev || !results_dev || nq < 0) return fail(MESSI_EINVAL, "bad argument");
    TRY(check_k(idx, k));
    CK(cudaSetDevice(idx->device));
    TRY(join_streams(idx));
    if (nq == 0) return MESSI_OK;
    return run_ed_batch(idx, queries_dev, nq, results_dev, stats_dev, k);
}

static messi_status check_dtw_k(const messi_index* idx, int32_t k)
{
    if (k < 1 || k > MESSI_MAX_K) return fail(MESSI_EINVAL, "k = %d outside [1, %d]", k, MESSI_MAX_K);
    if (k > 1 && idx->window > 4096) return fail(MESSI_EINVAL, "k-NN needs an approximate-search window <= 4096");
    return MESSI_OK;
}

extern "C" messi_status messi_query_dtw_knn(messi_index* idx, const float* query, int32_t reach, int32_t k,
                                            messi_result* results, messi_stats* stats)
{
    g_err[0] = 0;
    if (!idx || !query || !results) return fail(MESSI_EINVAL, "NULL argument");
    if (reach < 0 || reach > idx->n) return fail(MESSI_EINVAL, "reach %d outside [0, %d]", reach, idx->n);
    TRY(check_dtw_k(idx, k));
    CK(cudaSetDevice(idx->device));
    TRY(ensure_dtw_buffers(idx));
    if (k > 1) TRY(ensure_dtw_knn(idx));
    if (!idx->resk) TRY(dalloc(&idx->resk, MESSI_MAX_K));
    const float* q = nullptr;
    TRY(stage_query(idx, query, &q));
    TRY(fork_streams(idx));
    TRY(run_dtw(idx, q, reach, idx->resk, idx->stats1, k));
    TRY(join_streams(idx));
    CK(cudaMemcpyAsync(results, idx->resk, sizeof(messi_result) * k, cudaMemcpyDeviceToHost, idx->stream));
    if (stats) CK(cudaMemcpyAsync(stats, idx->stats1, sizeof(messi_stats), cudaMemcpyDeviceToHost, idx->stream));
    CK(cudaStreamSynchronize(idx->stream));
    return MESSI_OK;
}

extern "C" messi_status messi_query_dtw_knn_batch(messi_index* idx, const float* queries_dev, int32_t nq, int32_t reach,
                                                  int32_t k, messi_result* results_dev, messi_stats* stats_dev)
{
    g_err[0] = 0;
    if (!idx || !queries_dev || !results_dev || nq < 0) return fail(MESSI_EINVAL, "bad argument");
    if (reach < 0 || reach > idx->n) return fail(MESSI_EINVAL, "reach %d outside [0, %d]", reach, idx->n);
    TRY(check_dtw_k(idx, k));
    CK(cudaSetDevice(idx->device));
    TRY(ensure_dtw_buffers(idx));
    if (k > 1) TRY(ensure_dtw_knn(idx));
    TRY(fork_streams(idx));
    for (int i = 0; i < nq; ++i)
        TRY(run_dtw(idx, queries_dev + (size_t)i * idx->n, reach, results_dev + (size_t)i * k,
                    stats_dev ? stats_dev + i : nullptr, k));
    return join_streams(idx);
}

extern "C" messi_status messi_query_dtw_batch(messi_index* idx, const float* queries_dev, int32_t nq, int32_t reach,
                                              messi_result* results_dev, messi_stats* stats_dev)
{
    g_err[0] = 0;
    if (!idx || !queries_dev || !results_dev || nq < 0) return fail(MESSI_EINVAL, "bad argument");
    if (reach < 0 || reach > idx->n) return fail(MESSI_EINVAL, "reach %d outside [0, %d]", reach, idx->n);
    CK(cudaSetDevice(idx->device));
    TRY(ensure_dtw_buffers(idx));
    TRY(fork_streams(idx));
    for (int i = 0; i < nq; ++i)
        TRY(run_dtw(idx, queries_dev + (size_t)i * idx->n, reach, results_dev + i, stats_dev ? stats_dev + i : nullptr));
    return join_streams(idx);
}

// ----------------------------------------------------------------- tensor-core ED path
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// A 2-D uint8 TMA map over `rows` rows of `inner` bytes: boxes of 128 bytes x box_rows rows,
// 128-byte swizzle (the UMMA K-major SWIZZLE_128B operand layout).
static messi_status encode_u8_map(CUtensorMap* m, const void* base, unsigned long long inner, unsigned long long rows,
                                  unsigned box_rows)
{
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) return fail(MESSI_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {inner};
    const cuuint32_t box[2] = {128u, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(MESSI_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return MESSI_OK;
}

static messi_status ensure_tc(messi_index* idx)
{
    if (idx->n != 128 && idx->n != 256)
        return fail(MESSI_EINVAL, "the tensor-core path serves n = 128 or 256 (got %d)", idx->n);
    auto& tc = idx->tc;
    if (tc.bst) return MESSI_OK;
    const size_t npad = (size_t)idx->ntiles * MESSI_TILE_ROWS;
    TRY(dalloc(&tc.bst, kTcMaxQ));
    CK(cudaMemset(tc.bst, 0, sizeof(QState) * kTcMaxQ));
    TRY(dalloc(&tc.qc, (size_t)kTcMaxQ * (idx->n / 4)));
    CK(cudaMemset(tc.qc, 0, (size_t)kTcMaxQ * idx->n));
    TRY(dalloc(&tc.cand, (size_t)kTcMaxQ * kTcCandCap));
    TRY(dalloc(&tc.tcm, npad));
    k_tc_rowmeta<<<grid_of_rows(npad, 256), 256, 0, idx->stream>>>(idx->rows8, idx->meta8, (long long)npad, idx->n, tc.tcm);
    LAUNCHED(idx);
    TRY(encode_u8_map(&tc.tmA, idx->rows8, (unsigned long long)idx->n, (unsigned long long)npad, kTcRows));
    TRY(encode_u8_map(&tc.tmB, tc.qc, (unsigned long long)idx->n, (unsigned long long)kTcMaxQ, kTcMaxQ));
    return MESSI_OK;
}

// The batched tensor-core path for nq queries [nq][n] on the device: passes of <= kTcMaxQ
// queries, each one stream of the quantised rows through k_ed_tc.
static messi_status run_ed_tc(messi_index* idx, const float* queries_dev, int nq, messi_result* results_dev,
                              messi_stats* stats_dev)
{
    TRY(ensure_tc(idx));
    auto& tc = idx->tc;
    const int n = idx->n;
    const size_t qsm = (size_t)((n + 3) & ~3) * sizeof(float);
    const int len = (int)(idx->window < idx->N ? idx->window : idx->N);
    const long long ntc = idx->ntiles * (MESSI_TILE_ROWS / kTcRows);
    cudaStream_t st = idx->stream;
    PeerSet none{nullptr, 0, 0u};
    for (int g0 = 0; g0 < nq; g0 += kTcMaxQ) {
        const int B = nq - g0 < kTcMaxQ ? nq - g0 : kTcMaxQ;
        const float* q = queries_dev + (size_t)g0 * n;
        {
            ProfScope ps(idx, K_SEED, st);
            k_prologue_tc<<<B, 256, qsm, st>>>(q, n, idx->beta32, idx->lo_w, idx->hi_w, idx->skey, idx->N, idx->window,
                                               tc.bst, tc.qc);
            LAUNCHED(idx);
            dim3 sg((unsigned)((len + kSeedRowsPerCta - 1) / kSeedRowsPerCta), (unsigned)B);
            k_seed_batch<<<sg, 256, qsm, st>>>(q, n, idx->rows, idx->perm, tc.bst, none, nullptr, idx->window);
            LAUNCHED(idx);
        }
        {
            ProfScope ps(idx, K_SCAN, st);
            const long long grid = ntc < idx->sms ? ntc : idx->sms;
            k_ed_tc<<<(unsigned)grid, kTcThreads, tc_smem_bytes(n), st>>>(tc.tmA, tc.tmB, ntc, idx->N, n, B, tc.tcm,
                                                                          tc.bst, tc.cand);
            LAUNCHED(idx);
        }
        {
            ProfScope ps(idx, K_REFINE, st);
            const size_t per_warp = (fused_qpad(n) + (size_t)n / 4) * sizeof(float);
            k_tc_verify<<<(B + 3) / 4, 128, 4 * per_warp, st>>>(q, n, B, tc.cand, idx->rows8, idx->meta8, tc.qc, idx->perm,
                                                              idx->rows, idx->N, tc.bst);
            LAUNCHED(idx);
            k_finalise_batch<<<(B + 127) / 128, 128, 0, st>>>(tc.bst, B, idx->N, idx->row_begin, results_dev + g0,
                                                              stats_dev ? stats_dev + g0 : nullptr, nullptr, 1);
            LAUNCHED(idx);
        }
    }
    return MESSI_OK;
}

extern "C" messi_status messi_query_ed_tc_batch(messi_index* idx, const float* queries_dev, int32_t nq,
                                                messi_result* results_dev, messi_stats* stats_dev)
{
    g_err[0] = 0;
    if (!idx || !queries_dev || !results_dev || nq < 0) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    TRY(join_streams(idx));
    if (nq == 0) return MESSI_OK;
    return run_ed_tc(idx, queries_dev, nq, results_dev, stats_dev);
}

// ------------------------------------------------------------ shared best-so-far (shards)
extern "C" messi_status messi_batch_state_ipc(messi_index* idx, int32_t set, void* handle_out)
{
    g_err[0] = 0;
    if (!idx || !handle_out || set < 0 || set > 2) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    TRY(ensure_batch_buffers(idx));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, set < 2 ? idx->bset[set].bst : idx->slot_st));
    memcpy(handle_out, &h, sizeof h);
    return MESSI_OK;
}

static messi_status unlink_peers(messi_index* idx)
{
    for (auto& row : idx->peer_ipc)
        for (void*& p : row)
            if (p) {
                CK(cudaIpcCloseMemHandle(p));
                p = nullptr;
            }
    for (auto& row : idx->peer_st)
        for (QState*& p : row) p = nullptr;
    idx->npeers = 0;
    return MESSI_OK;
}

static messi_status upload_peers(messi_index* idx)
{
    CK(cudaMemcpy(idx->d_peers, &idx->peer_st[0][0], sizeof(QState*) * 3 * MESSI_MAX_PEERS, cudaMemcpyHostToDevice));
    return MESSI_OK;
}

extern "C" messi_status messi_link_peers_ipc(messi_index* idx, const void* handles, int32_t npeers)
{
    g_err[0] = 0;
    if (!idx || npeers < 0 || npeers > MESSI_MAX_PEERS || (npeers && !handles)) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    TRY(ensure_batch_buffers(idx));
    TRY(unlink_peers(idx));
    const unsigned char* h = static_cast<const unsigned char*>(handles);
    for (int i = 0; i < npeers; ++i)
        for (int set = 0; set < 3; ++set) {
            cudaIpcMemHandle_t mh;
            memcpy(&mh, h + ((size_t)i * 3 + set) * sizeof(cudaIpcMemHandle_t), sizeof mh);
            void* p = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                unlink_peers(idx);
                return fail(MESSI_ECUDA, "cudaIpcOpenMemHandle(peer %d, set %d): %s", i, set, cudaGetErrorString(e));
            }
            idx->peer_ipc[set][i] = p;
            idx->peer_st[set][i] = static_cast<QState*>(p);
        }
    idx->npeers = npeers;
    idx->link_gen = (idx->link_gen + 1) % 255 + 1;  // never 0: epoch 0 means unlinked
    idx->epoch = 0;
    idx->dtw_epoch = 0;
    return upload_peers(idx);
}

extern "C" messi_status messi_link_peers_local(messi_index* idx, messi_index* const* peers, int32_t npeers)
{
    g_err[0] = 0;
    if (!idx || npeers < 0 || npeers > MESSI_MAX_PEERS || (npeers && !peers)) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    TRY(ensure_batch_buffers(idx));
    TRY(unlink_peers(idx));
    for (int i = 0; i < npeers; ++i) {
        if (!peers[i] || peers[i] == idx) return fail(MESSI_EINVAL, "peer %d is NULL or the index itself", i);
        if (peers[i]->device != idx->device) {
            cudaError_t e = cudaDeviceEnablePeerAccess(peers[i]->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return fail(MESSI_ECUDA, "peer access %d -> %d: %s", idx->device, peers[i]->device, cudaGetErrorString(e));
            cudaGetLastError();
        }
        CK(cudaSetDevice(peers[i]->device));
        TRY(ensure_batch_buffers(peers[i]));
        CK(cudaSetDevice(idx->device));
        for (int set = 0; set < 2; ++set) idx->peer_st[set][i] = peers[i]->bset[set].bst;
        idx->peer_st[2][i] = peers[i]->slot_st;
    }
    idx->npeers = npeers;
    idx->link_gen = (idx->link_gen + 1) % 255 + 1;
    idx->epoch = 0;
    idx->dtw_epoch = 0;
    return upload_peers(idx);
}

// ------------------------------------------------------------------------ inspection
extern "C" messi_status messi_debug_breakpoints(int32_t device, float* beta32_host)
{
    g_err[0] = 0;
    if (!beta32_host) return fail(MESSI_EINVAL, "NULL argument");
    CK(cudaSetDevice(device));
    float* d = nullptr;
    CK(cudaMalloc(&d, 3 * 256 * sizeof(float)));
    k_breakpoints<<<1, 256>>>(d, d + 256, d + 512);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(beta32_host, d, 255 * sizeof(float), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(MESSI_ECUDA, "breakpoints: %s", cudaGetErrorString(e));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_summaries(messi_index* idx, uint8_t* sym_dev, float* paa_dev)
{
    g_err[0] = 0;
    if (!idx || !sym_dev) return fail(MESSI_EINVAL, "NULL argument");
    if (paa_dev && !idx->paa) return fail(MESSI_EINVAL, "index built without keep_paa");
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    k_detile<<<(unsigned)((idx->N + 255) / 256), 256, 0, idx->stream>>>(idx->sym8, idx->perm, idx->N,
                                                                        reinterpret_cast<uint4*>(sym_dev));
    LAUNCHED(idx);
    if (paa_dev)
        CK(cudaMemcpyAsync(paa_dev, idx->paa, (size_t)idx->N * MESSI_W * sizeof(float), cudaMemcpyDeviceToDevice,
                           idx->stream));
    CK(cudaStreamSynchronize(idx->stream));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_quantised(messi_index* idx, uint8_t* q8_dev, float* meta_dev)
{
    g_err[0] = 0;
    if (!idx || !q8_dev || !meta_dev) return fail(MESSI_EINVAL, "NULL argument");
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    k_unsort_q8<<<(unsigned)(idx->sms * 8), 256, 0, idx->stream>>>(idx->rows8, idx->meta8, idx->perm, idx->N, idx->n,
                                                                   q8_dev, reinterpret_cast<float2*>(meta_dev));
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(idx->stream));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_order(messi_index* idx, const uint64_t** skey_dev, const uint32_t** perm_dev)
{
    if (!idx || !skey_dev || !perm_dev) return fail(MESSI_EINVAL, "NULL argument");
    *skey_dev = (const uint64_t*)idx->skey;
    *perm_dev = (const uint32_t*)idx->perm;
    return MESSI_OK;
}

// ------------------------------------------------------------------ inspection helpers
// The step-level inspection calls run the QUERY PATH'S OWN KERNELS with their pruning
// thresholds at +inf, so that every row / tile comes out of them, and scatter the outputs back
// to row (or id) order: k_scan for the 8-bit bound, k_filter_batch for the tile boxes,
// k_lbk_filter_q8 / k_lbk_filter and the strip / band / warp DTW refine (frozen: no BSF update,
// no abandon) for LB_Keogh and the fp32 DTW.  Only the ED refine's inner passes, which sit
// inside the fused kernel, are reached through a small kernel that calls the same device
// functions (q8i_bound_pass, ed2_group, ed2_exact_g).
__global__ void k_dbg_invert(const unsigned* __restrict__ perm, long long N, unsigned* __restrict__ inv)
{
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < N) inv[perm[p]] = (unsigned)p;
}
__global__ void k_dbg_iota(unsigned* a, long long n)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (unsigned)i;
}
// arm, then the inspection setup: tile list length, candidate count, filter threshold +inf
__global__ void k_dbg_state(QState* st, unsigned tiles, unsigned cands, unsigned frozen)
{
    arm_state(st);
    st->tile_count = tiles;
    st->cand_count = cands;
    st->lbk_thr_bits = 0x7f800000u;
    st->frozen = frozen;
}
__global__ void k_dbg_map(const unsigned* __restrict__ ids, int k, int* map, const unsigned* __restrict__ inv,
                          uint2* __restrict__ cand, int set)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= k) return;
    map[ids[t]] = set ? t : -1;
    if (cand) cand[t] = make_uint2(inv[ids[t]], 0u);  // (sorted position, 8-bit bound 0)
}
__global__ void k_dbg_scatter_cand(const uint2* __restrict__ cand, const QState* st, const unsigned* __restrict__ perm,
                                   float* __restrict__ out, int rev = 0)
{
    const unsigned total = rev ? st->rcand_count : st->cand_count;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x)
        out[perm[cand[i].x]] = __uint_as_float(cand[i].y);
}
__global__ void k_dbg_scatter_tiles(const uint2* __restrict__ tl, const QState* st, float* __restrict__ out)
{
    const unsigned total = st->tile_count;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x)
        out[tl[i].x] = __uint_as_float(tl[i].y);
}
__global__ void k_dbg_scatter_dtw(const uint4* __restrict__ list2, const NearEntry* __restrict__ near, const QState* st,
                                  const int* __restrict__ map, float* __restrict__ lbk, float* __restrict__ d32)
{
    const unsigned nl = st->list2_count, nn = st->near_count;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < max(nl, nn); i += gridDim.x * blockDim.x) {
        if (lbk && i < nl) lbk[map[list2[i].x]] = __uint_as_float(list2[i].y);
        if (d32 && i < nn) d32[map[near[i].id]] = near[i].d32;
    }
}
// Box bound of every super-tile (16 consecutive tiles) with the filter's own code (box_lb,
// same lane mapping: lane = super-tile mod 32), from query 0's filter table of a batch set.
__global__ void __launch_bounds__(256) k_dbg_superbox(const uint4* __restrict__ sboxes, long long nsuper,
                                                      const float* __restrict__ lutf, const QState* st,
                                                      float* __restrict__ out)
{
    extern __shared__ __align__(16) float lutf_s[];
    __shared__ unsigned char zlo[16], zhi[16];
    for (int i = threadIdx.x; i < kLutF / 4; i += blockDim.x)
        reinterpret_cast<float4*>(lutf_s)[i] = reinterpret_cast<const float4*>(lutf)[i];
    if (threadIdx.x < 16) { zlo[threadIdx.x] = st->zlo[threadIdx.x]; zhi[threadIdx.x] = st->zhi[threadIdx.x]; }
    __syncthreads();
    const int lane = threadIdx.x & 31, r = lane & 15, h = lane >> 4;
    const long long S = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (S >= nsuper) return;
    const uint4 mn = rotate_bytes(sboxes[2 * S], r), mx = rotate_bytes(sboxes[2 * S + 1], r);
    out[S] = box_lb(mn, mx, lutf_s + 16 * h, zlo, zhi, r);
}

static unsigned grid_of(long long n, int threads)
{
    long long g = (n + threads - 1) / threads;
    return (unsigned)(g < 1 ? 1 : (g > 65535LL * 32 ? 65535LL * 32 : g));
}

static messi_status ensure_debug_buffers(messi_index* idx)
{
    if (idx->dbg_inv) return MESSI_OK;
    TRY(dalloc(&idx->dbg_inv, (size_t)idx->N));
    TRY(dalloc(&idx->dbg_map, (size_t)idx->N));
    TRY(dalloc(&idx->dbg_iota, (size_t)idx->ntiles));
    CK(cudaMemsetAsync(idx->dbg_map, 0xff, sizeof(int) * (size_t)idx->N, idx->stream));  // -1: not inspected
    k_dbg_invert<<<grid_of(idx->N, 256), 256, 0, idx->stream>>>(idx->perm, idx->N, idx->dbg_inv);
    LAUNCHED(idx);
    k_dbg_iota<<<grid_of(idx->ntiles, 256), 256, 0, idx->stream>>>(idx->dbg_iota, idx->ntiles);
    LAUNCHED(idx);
    return MESSI_OK;
}

// DTW prologue only (envelope U/L, tables) for `reach` into slot 0 (k_seed_dtw over a
// one-row window), then re-armed.
static messi_status debug_prologue(messi_index* idx, const float* query_dev, int reach)
{
    cudaStream_t st = idx->stream;
    Slot& sl = idx->slot[0];
    const int n = idx->n;
    const size_t qsm = (size_t)((n + 3) & ~3) * sizeof(float);
    k_seed_dtw<<<1, 32, 2 * qsm + 3 * (size_t)n * sizeof(float), st>>>(query_dev, n, reach < 0 ? 0 : reach, idx->rows,
                                                                      idx->skey, idx->perm, idx->N, 1, idx->beta32,
                                                                      idx->lo_w, idx->hi_w, sl.lut, sl.tab, sl.U, sl.L,
                                                                      sl.st, nullptr, PeerSet{nullptr, 0, 0u}, 0);
    LAUNCHED(idx);
    k_arm<<<1, 1, 0, st>>>(sl.st);
    LAUNCHED(idx);
    return MESSI_OK;
}

// ED prologue only: k_prologue_batch for one query into batch set 0 (the ED batch path's
// tables: expanded scan table lutx, filter table lutf, zero runs, query PAA).
static messi_status debug_prologue_ed(messi_index* idx, const float* query_dev)
{
    TRY(ensure_batch_buffers(idx));
    const auto& bs = idx->bset[0];
    const size_t qsm = (size_t)((idx->n + 3) & ~3) * sizeof(float);
    k_prologue_batch<<<1, 256, qsm, idx->stream>>>(query_dev, idx->n, idx->beta32, idx->lo_w, idx->hi_w, idx->skey,
                                                   idx->N, idx->window, bs.lutc, bs.lutx, bs.lutf, bs.bst, nullptr,
                                                   bs.qc);
    LAUNCHED(idx);
    return MESSI_OK;
}

static messi_status debug_begin(messi_index* idx, const float* query_dev, int reach)
{
    g_err[0] = 0;
    if (!idx || !query_dev) return fail(MESSI_EINVAL, "NULL argument");
    if (reach > idx->n) return fail(MESSI_EINVAL, "reach %d > n", reach);
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    TRY(ensure_dtw_buffers(idx));
    TRY(ensure_debug_buffers(idx));
    return MESSI_OK;
}

// The scan table and state of `reach`'s query path: ED -> batch set 0 (k_prologue_batch),
// DTW -> slot 0 (k_seed_dtw's prologue).
static messi_status debug_tables(messi_index* idx, const float* query_dev, int reach, const float** tab, QState** st)
{
    if (reach < 0) {
        TRY(debug_prologue_ed(idx, query_dev));
        *tab = idx->bset[0].lutx;
        *st = idx->bset[0].bst;
    } else {
        TRY(debug_prologue(idx, query_dev, reach));
        *tab = idx->slot[0].tab;
        *st = idx->slot[0].st;
    }
    return MESSI_OK;
}

extern "C" messi_status messi_debug_lower_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev)
{
    if (!lb_dev) return fail(MESSI_EINVAL, "NULL argument");
    TRY(debug_begin(idx, query_dev, reach));
    const float* tab = nullptr;
    QState* st = nullptr;
    TRY(debug_tables(idx, query_dev, reach, &tab, &st));
    Slot& sl = idx->slot[0];
    cudaStream_t s = idx->stream;
    k_dbg_state<<<1, 1, 0, s>>>(st, (unsigned)idx->ntiles, 0u, 0u);  // every tile listed, BSF +inf
    LAUNCHED(idx);
    CK(cudaMemsetAsync(lb_dev, 0xff, sizeof(float) * (size_t)idx->N, s));  // NaN: not written
    k_scan<<<scan_grid(idx), 32 * kScanWarps, scan_smem(), s>>>(idx->tiles, idx->sym8, idx->N, tab, st, sl.cand,
                                                                idx->dbg_iota, 0u);
    LAUNCHED(idx);
    k_dbg_scatter_cand<<<idx->sms * 8, 256, 0, s>>>(sl.cand, st, idx->perm, lb_dev);
    LAUNCHED(idx);
    k_arm<<<1, 1, 0, s>>>(st);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(s));
    return MESSI_OK;
}

// The reverse envelope-PAA bound of every row (k_renv for `reach`, then k_scan with every
// tile listed and the threshold at +inf, then k_rev_paa_filter in its rev_only mode).
extern "C" messi_status messi_debug_rev_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev)
{
    if (!lb_dev) return fail(MESSI_EINVAL, "NULL argument");
    if (reach < 1) return fail(MESSI_EINVAL, "reach %d: the reverse envelope-PAA bound serves reaches >= 1", reach);
    if (renv_env_off()) return fail(MESSI_EINVAL, "the reverse envelope-PAA filter is off (MESSI_NO_RENV)");
    TRY(debug_begin(idx, query_dev, reach));
    TRY(ensure_renv(idx, reach));
    const float* tab = nullptr;
    QState* st = nullptr;
    TRY(debug_tables(idx, query_dev, reach, &tab, &st));
    Slot& sl = idx->slot[0];
    cudaStream_t s = idx->stream;
    k_dbg_state<<<1, 1, 0, s>>>(st, (unsigned)idx->ntiles, 0u, 0u);  // every tile listed, BSF +inf
    LAUNCHED(idx);
    CK(cudaMemsetAsync(lb_dev, 0xff, sizeof(float) * (size_t)idx->N, s));  // NaN: not written
    k_scan<<<scan_grid(idx), 32 * kScanWarps, scan_smem(), s>>>(idx->tiles, idx->sym8, idx->N, tab, st, sl.cand,
                                                                idx->dbg_iota, 0u);
    LAUNCHED(idx);
    k_rev_paa_filter<<<idx->sms * 3, 256, kRevTabBytes, s>>>(sl.cand, idx->renv, idx->lo_w, idx->hi_w, idx->n / MESSI_W,
                                                             st, sl.cand2, 1);
    LAUNCHED(idx);
    k_dbg_scatter_cand<<<idx->sms * 8, 256, 0, s>>>(sl.cand2, st, idx->perm, lb_dev, 1);
    LAUNCHED(idx);
    k_arm<<<1, 1, 0, s>>>(st);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(s));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_coarse_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev)
{
    if (!lb_dev) return fail(MESSI_EINVAL, "NULL argument");
    TRY(debug_begin(idx, query_dev, reach));
    const float* tab = nullptr;
    QState* st = nullptr;
    TRY(debug_tables(idx, query_dev, reach, &tab, &st));
    k_debug_coarse<<<scan_grid(idx), 32 * kScanWarps, scan_smem(), idx->stream>>>(idx->tiles, idx->ntiles, idx->N, tab,
                                                                                 idx->perm, lb_dev);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(idx->stream));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_tile_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev)
{
    if (!lb_dev) return fail(MESSI_EINVAL, "NULL argument");
    TRY(debug_begin(idx, query_dev, reach));
    cudaStream_t s = idx->stream;
    if (reach < 0) {  // the ED batch path's filter (fp32 box bound, zero runs), threshold +inf
        TRY(debug_prologue_ed(idx, query_dev));
        const auto& bs = idx->bset[0];
        const long long nsuper = (idx->ntiles + kSuperTiles - 1) / kSuperTiles;
        CK(cudaMemsetAsync(lb_dev, 0xff, sizeof(float) * (size_t)idx->ntiles, s));
        long long fx = (nsuper + 255) / 256;
        if (fx > idx->sms * 8) fx = idx->sms * 8;
        k_filter_batch<<<dim3((unsigned)fx, 1), 256, kFilterQ * kLutF * 4, s>>>(
            reinterpret_cast<const uint4*>(idx->boxes), idx->sboxes, idx->ntiles, nsuper, bs.lutf, bs.bst, 1, bs.btlist,
            0u);
        LAUNCHED(idx);
        k_dbg_scatter_tiles<<<idx->sms * 4, 256, 0, s>>>(bs.btlist, bs.bst, lb_dev);
        LAUNCHED(idx);
    } else {  // the DTW path's filter (fp64 box bound)
        TRY(debug_prologue(idx, query_dev, reach));
        Slot& sl = idx->slot[0];
        k_tile_filter<<<filter_grid(idx), 256, 0, s>>>(idx->boxes, idx->ntiles, idx->n / MESSI_W, idx->lo_w, idx->hi_w,
                                                      sl.st, nullptr, lb_dev, 0u);
        LAUNCHED(idx);
    }
    CK(cudaStreamSynchronize(s));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_super_bounds(messi_index* idx, const float* query_dev, float* lb_dev)
{
    if (!lb_dev) return fail(MESSI_EINVAL, "NULL argument");
    TRY(debug_begin(idx, query_dev, -1));
    TRY(debug_prologue_ed(idx, query_dev));
    const long long nsuper = (idx->ntiles + kSuperTiles - 1) / kSuperTiles;
    k_dbg_superbox<<<grid_of(nsuper, 256), 256, kLutF * 4, idx->stream>>>(idx->sboxes, nsuper, idx->bset[0].lutf,
                                                                          idx->bset[0].bst, lb_dev);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(idx->stream));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_ed_refine(messi_index* idx, const float* query_dev, const uint32_t* ids_dev,
                                              int32_t k, double* q8_dev, float* d32_dev, double* d64_dev)
{
    if ((!ids_dev && k > 0) || k < 0 || !q8_dev || !d32_dev || !d64_dev) return fail(MESSI_EINVAL, "bad argument");
    TRY(debug_begin(idx, query_dev, -1));
    if (k == 0) return MESSI_OK;
    cudaStream_t s = idx->stream;
    TRY(debug_prologue_ed(idx, query_dev));  // the quantised query of the batch path (set 0, query 0)
    const int wpb = 8;
    unsigned grid = (unsigned)((k + 32 * wpb - 1) / (32 * wpb));
    if (grid > (unsigned)idx->sms * 8) grid = idx->sms * 8;
    k_debug_ed_refine<<<grid, 32 * wpb, fused_qpad(idx->n) * sizeof(float) + idx->n, s>>>(
        idx->rows, idx->n, query_dev, idx->rows8, idx->meta8, idx->bset[0].qc, idx->bset[0].bst, idx->dbg_inv, ids_dev,
        k, reinterpret_cast<double2*>(q8_dev), d32_dev, d64_dev);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(s));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_dtw_stages(messi_index* idx, const float* query_dev, int32_t reach,
                                               const uint32_t* ids_dev, int32_t k, float* lbk_dev, float* d32_dev,
                                               int32_t* quantised, float* rev_dev)
{
    if ((!ids_dev && k > 0) || k < 0 || reach < 0) return fail(MESSI_EINVAL, "bad argument");
    TRY(debug_begin(idx, query_dev, reach));
    const bool strip = dtw_uses_strip(idx->n, reach);
    if (strip) TRY(ensure_renv(idx, reach));  // the query path's filter chain (threshold +inf here)
    if (quantised) *quantised = strip ? 1 : 0;
    if (k == 0) return MESSI_OK;
    cudaStream_t s = idx->stream;
    Slot& sl = idx->slot[0];
    TRY(debug_prologue(idx, query_dev, reach));
    k_dbg_state<<<1, 1, 0, s>>>(sl.st, 0u, (unsigned)k, 1u);  // k candidates, threshold +inf, frozen
    LAUNCHED(idx);
    k_dbg_map<<<grid_of(k, 256), 256, 0, s>>>(ids_dev, k, idx->dbg_map, idx->dbg_inv, sl.cand, 1);
    LAUNCHED(idx);
    if (rev_dev) CK(cudaMemsetAsync(rev_dev, 0xff, sizeof(float) * (size_t)k, s));
    TRY(launch_lbk_filter(idx, sl, reach, strip, query_dev, s, rev_dev));
    {
        ProfScope ps(idx, K_REFINE, s);  // profiling on: the frozen refine's own time (bench steady-state rate)
        TRY(launch_dtw_refine(idx, sl, reach, strip, query_dev, s));
    }
    if (lbk_dev) CK(cudaMemsetAsync(lbk_dev, 0xff, sizeof(float) * (size_t)k, s));
    if (d32_dev) CK(cudaMemsetAsync(d32_dev, 0xff, sizeof(float) * (size_t)k, s));
    k_dbg_scatter_dtw<<<grid_of(k, 256), 256, 0, s>>>(sl.list2, sl.near, sl.st, idx->dbg_map, lbk_dev, d32_dev);
    LAUNCHED(idx);
    k_dbg_map<<<grid_of(k, 256), 256, 0, s>>>(ids_dev, k, idx->dbg_map, idx->dbg_inv, nullptr, 0);
    LAUNCHED(idx);
    k_arm<<<1, 1, 0, s>>>(sl.st);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(s));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_distances(messi_index* idx, const float* query_dev, int32_t reach,
                                              const uint32_t* ids_dev, int32_t k, float* d32_dev, double* d64_dev,
                                              float* lbk_dev)
{
    if ((!ids_dev && k > 0) || k < 0) return fail(MESSI_EINVAL, "bad argument");
    TRY(debug_begin(idx, query_dev, reach));
    if (k == 0) return MESSI_OK;
    cudaStream_t s = idx->stream;
    const int n = idx->n;
    if (reach < 0) {  // scratch for the outputs the caller did not ask for
        double *q8 = nullptr, *d64 = d64_dev;
        float* d32 = d32_dev;
        messi_status st = dalloc(&q8, 2 * (size_t)k);
        if (st == MESSI_OK && !d64) st = dalloc(&d64, (size_t)k);
        if (st == MESSI_OK && !d32) st = dalloc(&d32, (size_t)k);
        if (st == MESSI_OK) st = messi_debug_ed_refine(idx, query_dev, ids_dev, k, q8, d32, d64);
        cudaFree(q8);
        if (!d64_dev) cudaFree(d64);
        if (!d32_dev) cudaFree(d32);
        return st;
    }
    if (d64_dev) {  // the resolve kernel's fp64 engine
        bool gb = false;
        const int wr = resolve_warps(n, reach, &gb);
        if (gb && !idx->dbg_gbuf) TRY(dalloc(&idx->dbg_gbuf, (size_t)8 * 3 * MESSI_MAX_N));
        unsigned grid = gb ? 1u : (unsigned)((k + wr - 1) / wr);
        if (grid > (unsigned)idx->sms * 8) grid = idx->sms * 8;
        k_debug_dtw64<<<grid, 32 * wr, wr * resolve_warp_bytes(n, reach, gb), s>>>(idx->rows, n, reach, query_dev,
                                                                                 ids_dev, k, d64_dev,
                                                                                 gb ? idx->dbg_gbuf : nullptr);
        LAUNCHED(idx);
    }
    if (d32_dev || lbk_dev) TRY(messi_debug_dtw_stages(idx, query_dev, reach, ids_dev, k, lbk_dev, d32_dev, nullptr, nullptr));
    CK(cudaStreamSynchronize(s));
    return MESSI_OK;
}

// Scan throughput in isolation (tuning / roofline evidence): prologue for one query, then
// `reps` coarse scans back to back on the main stream, each bracketed by CUDA events; the
// survivor counter is reset between repetitions.  Returns the summed kernel milliseconds.
__global__ void k_reset_cand(QState* st) { st->cand_count = 0; }

extern "C" messi_status messi_debug_scan_repeat(messi_index* idx, const float* query_dev, int32_t reps, double* ms_out,
                                                int64_t* coarse_out)
{
    g_err[0] = 0;
    if (!idx || !query_dev || reps <= 0 || !ms_out) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    TRY(sync_all(idx));
    TRY(ensure_dtw_buffers(idx));
    Slot& sl = idx->slot[0];
    cudaStream_t st = idx->stream;
    const int n = idx->n;
    const size_t qsm = (size_t)((n + 3) & ~3) * sizeof(float);
    int len = (int)(idx->window < idx->N ? idx->window : idx->N);
    int seed_grid = (len + 7) / 8;
    if (seed_grid > 256) seed_grid = 256;
    k_seed_ed<<<seed_grid, 256, qsm, st>>>(query_dev, n, idx->rows, idx->skey, idx->perm, idx->N, idx->window, idx->beta32,
                                           idx->lo_w, idx->hi_w, sl.lut, sl.tab, sl.st);
    LAUNCHED(idx);
    TRY(launch_tile_filter(idx, sl, st));
    std::vector<cudaEvent_t> ev(2 * (size_t)reps);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (int r = 0; r < reps; ++r) {
        k_reset_cand<<<1, 1, 0, st>>>(sl.st);
        CK(cudaEventRecord(ev[2 * r], st));
        k_scan<<<scan_grid(idx), 32 * kScanWarps, scan_smem(), st>>>(idx->tiles, idx->sym8, idx->N, sl.tab, sl.st, sl.cand,
                                                                     sl.tlist, 0u);
        CK(cudaEventRecord(ev[2 * r + 1], st));
    }
    idx->launches += 2 * reps;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    double ms = 0.0;
    for (int r = 0; r < reps; ++r) {
        float t = 0.0f;
        CK(cudaEventElapsedTime(&t, ev[2 * r], ev[2 * r + 1]));
        ms += t;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (coarse_out) {
        unsigned c[2] = {0, 0};
        CK(cudaMemcpy(&c[0], &sl.st->cand_count, sizeof(unsigned), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&c[1], &sl.st->tile_count, sizeof(unsigned), cudaMemcpyDeviceToHost));
        *coarse_out = (int64_t)c[0] | ((int64_t)c[1] << 32);
    }
    k_arm<<<1, 1, 0, st>>>(sl.st);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(st));
    *ms_out = ms;
    return MESSI_OK;
}

