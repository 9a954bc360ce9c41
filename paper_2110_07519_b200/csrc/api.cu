// api.cu -- the C-ABI of libmessi (include/messi.h): argument checks, device memory,
// kernel orchestration.  The only translation unit; the .cuh files hold the kernels.
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/messi.h"
#include "common.cuh"
#include "dtw.cuh"
#include "refine.cuh"
#include "scan.cuh"
#include "summarise.cuh"

using namespace messi;

struct messi_index {
    int device = 0;
    cudaStream_t stream = nullptr;
    int n = 0, window = 2000, keep_paa = 0;
    long long N = 0, ntiles = 0, row_begin = 0;
    const float* rows = nullptr;
    int sms = 148;
    // summaries
    uint4* tiles = nullptr;
    float* paa = nullptr;
    unsigned long long* skey = nullptr;
    unsigned* perm = nullptr;
    float *beta32 = nullptr, *lo_w = nullptr, *hi_w = nullptr;
    // per-query scratch
    float *lut = nullptr, *U = nullptr, *L = nullptr, *qbuf = nullptr;
    uint2* cand = nullptr;
    unsigned* list2 = nullptr;
    NearEntry* near = nullptr;
    QState* st = nullptr;
    messi_result* res1 = nullptr;
    messi_stats* stats1 = nullptr;
    long long launches = 0;
    // optional per-kernel event timing
    bool prof = false;
    struct Ev { int kind; cudaEvent_t a, b; };
    std::vector<Ev> evs;
    std::vector<cudaEvent_t> pool;
};

enum { K_SEED = 0, K_SCAN = 1, K_REFINE = 2, K_LBK = 3, K_RESOLVE = 4, K_KINDS = 5 };

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

// Brackets one launch with events when profiling is on.
struct ProfScope {
    messi_index* idx;
    int kind;
    cudaEvent_t a = nullptr;
    ProfScope(messi_index* i, int k) : idx(i), kind(k)
    {
        if (idx->prof) {
            a = pool_get(idx);
            cudaEventRecord(a, idx->stream);
        }
    }
    ~ProfScope()
    {
        if (idx->prof && a) {
            cudaEvent_t b = pool_get(idx);
            cudaEventRecord(b, idx->stream);
            idx->evs.push_back({kind, a, b});
        }
    }
};

static_assert(sizeof(messi_result) == 32, "messi_result layout");
static_assert(sizeof(messi_stats) == 64, "messi_stats layout");

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

template <typename T> static messi_status dalloc(T** p, size_t count)
{
    *p = nullptr;
    if (count == 0) count = 1;
    CK(cudaMalloc((void**)p, count * sizeof(T)));
    return MESSI_OK;
}

#define TRY(x)                                                                                      \
    do {                                                                                            \
        messi_status s_ = (x);                                                                      \
        if (s_ != MESSI_OK) return s_;                                                              \
    } while (0)

// Reaches with a register-band DTW instantiation (DtwThread<R>); others use the warp path.
#define MESSI_DTW_REACHES(X) X(2) X(5) X(12) X(25)

static size_t scan_smem() { return (size_t)MESSI_CARD * 64 * sizeof(float); }

static messi_status setup_kernels()
{
    static bool done = false;
    if (done) return MESSI_OK;
    CK(cudaFuncSetAttribute(k_scan<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem()));
    CK(cudaFuncSetAttribute(k_scan<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem()));
    CK(cudaFuncSetAttribute(k_seed_dtw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_refine_dtw_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_resolve_dtw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_debug_dist<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
#define SET_ATTR(R) CK(cudaFuncSetAttribute(k_debug_dist<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    MESSI_DTW_REACHES(SET_ATTR)
#undef SET_ATTR
    done = true;
    return MESSI_OK;
}

// warps per CTA for kernels holding 3*n elements of `esize` bytes per warp in smem
static int wavefront_warps(int n, size_t esize, int maxw)
{
    size_t per = 3 * (size_t)n * esize;
    int w = (int)((96 * 1024) / per);
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
    TRY(setup_kernels());

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
    messi_status s;
    if ((s = dalloc(&idx->tiles, (size_t)idx->ntiles * (MESSI_TILE_BYTES / 16)))) return bail(s);
    if (idx->keep_paa && (s = dalloc(&idx->paa, (size_t)N * MESSI_W))) return bail(s);
    if ((s = dalloc(&idx->skey, (size_t)N)) || (s = dalloc(&idx->perm, (size_t)N))) return bail(s);
    if ((s = dalloc(&idx->beta32, 256)) || (s = dalloc(&idx->lo_w, 256)) || (s = dalloc(&idx->hi_w, 256))) return bail(s);
    if ((s = dalloc(&idx->lut, MESSI_W * MESSI_CARD)) || (s = dalloc(&idx->U, n)) || (s = dalloc(&idx->L, n)) ||
        (s = dalloc(&idx->qbuf, n)))
        return bail(s);
    if ((s = dalloc(&idx->cand, (size_t)N)) || (s = dalloc(&idx->list2, (size_t)N)) || (s = dalloc(&idx->near, (size_t)N)))
        return bail(s);
    if ((s = dalloc(&idx->st, 1)) || (s = dalloc(&idx->res1, 1)) || (s = dalloc(&idx->stats1, 1))) return bail(s);

    cudaStream_t st = idx->stream;
    unsigned long long* keys_in = nullptr;
    unsigned* ids_in = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    auto cleanup = [&]() {
        cudaFree(keys_in);
        cudaFree(ids_in);
        cudaFree(temp);
    };
    do {
        if ((s = dalloc(&keys_in, (size_t)N)) || (s = dalloc(&ids_in, (size_t)N))) break;
        k_breakpoints<<<1, 256, 0, st>>>(idx->beta32, idx->lo_w, idx->hi_w);
        ++idx->launches;
        if (cudaGetLastError() != cudaSuccess) { s = fail(MESSI_ECUDA, "k_breakpoints launch"); break; }
        long long grid = idx->ntiles < (long long)idx->sms * 8 ? idx->ntiles : (long long)idx->sms * 8;
        k_summarise<<<(unsigned)grid, 256, 0, st>>>(rows_dev, N, n, idx->beta32, idx->tiles, idx->ntiles, keys_in,
                                                    ids_in, idx->paa);
        ++idx->launches;
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "k_summarise: %s", cudaGetErrorString(e)); break; }
        e = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys_in, idx->skey, ids_in, idx->perm, (int)N, 0, 64, st);
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "cub sort sizing: %s", cudaGetErrorString(e)); break; }
        e = cudaMalloc(&temp, temp_bytes ? temp_bytes : 1);
        if (e != cudaSuccess) { s = fail(MESSI_ENOMEM, "cub temp (%zu B): %s", temp_bytes, cudaGetErrorString(e)); break; }
        e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, idx->skey, ids_in, idx->perm, (int)N, 0, 64, st);
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "cub sort: %s", cudaGetErrorString(e)); break; }
        idx->launches += 4;
        k_arm<<<1, 1, 0, st>>>(idx->st);
        ++idx->launches;
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { s = fail(MESSI_ECUDA, "build: %s", cudaGetErrorString(e)); break; }
        s = MESSI_OK;
    } while (0);
    cleanup();
    if (s != MESSI_OK) return bail(s);
    *out = idx;
    return MESSI_OK;
}

extern "C" void messi_free(messi_index* idx)
{
    if (!idx) return;
    cudaSetDevice(idx->device);
    if (idx->stream) cudaStreamSynchronize(idx->stream);
    else cudaDeviceSynchronize();
    void* ptrs[] = {idx->tiles, idx->paa,   idx->skey, idx->perm, idx->beta32, idx->lo_w,  idx->hi_w,
                    idx->lut,   idx->U,     idx->L,    idx->qbuf, idx->cand,   idx->list2, idx->near,
                    idx->st,    idx->res1,  idx->stats1};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (auto& e : idx->evs) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    for (auto e : idx->pool) cudaEventDestroy(e);
    delete idx;
}

extern "C" const char* messi_last_error(void) { return g_err; }

extern "C" int64_t messi_launch_count(const messi_index* idx) { return idx ? idx->launches : 0; }

extern "C" messi_status messi_profile_enable(messi_index* idx, int32_t enable)
{
    if (!idx) return fail(MESSI_EINVAL, "NULL index");
    CK(cudaSetDevice(idx->device));
    CK(cudaStreamSynchronize(idx->stream));
    for (auto& e : idx->evs) {
        idx->pool.push_back(e.a);
        idx->pool.push_back(e.b);
    }
    idx->evs.clear();
    idx->prof = enable != 0;
    return MESSI_OK;
}

extern "C" messi_status messi_profile_read(messi_index* idx, int32_t kind, double* total_ms, int64_t* launches)
{
    if (!idx || !total_ms || !launches || kind < 0 || kind >= K_KINDS) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    CK(cudaStreamSynchronize(idx->stream));
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
    long long need = (idx->ntiles + 7) / 8;
    long long cap = (long long)idx->sms * 2;
    return (int)(need < cap ? (need < 1 ? 1 : need) : cap);
}

// One ED query, fully on the stream: seed (+prologue) -> scan -> refine -> resolve.
static messi_status run_ed(messi_index* idx, const float* q_dev, messi_result* res, messi_stats* stats)
{
    cudaStream_t st = idx->stream;
    const int n = idx->n;
    const size_t qsm = (size_t)((n + 3) & ~3) * sizeof(float);
    int len = (int)(idx->window < idx->N ? idx->window : idx->N);
    int seed_grid = (len + 7) / 8;
    if (seed_grid > 256) seed_grid = 256;
    {
        ProfScope ps(idx, K_SEED);
        k_seed_ed<<<seed_grid, 256, qsm, st>>>(q_dev, n, idx->rows, idx->skey, idx->perm, idx->N, idx->window,
                                               idx->beta32, idx->lo_w, idx->hi_w, idx->lut, idx->st);
        LAUNCHED(idx);
    }
    {
        ProfScope ps(idx, K_SCAN);
        k_scan<false><<<scan_grid(idx), 256, scan_smem(), st>>>(idx->tiles, idx->ntiles, idx->N, idx->lut, idx->st,
                                                                idx->cand, nullptr);
        LAUNCHED(idx);
    }
    {
        ProfScope ps(idx, K_REFINE);
        k_refine_ed<<<idx->sms * 4, 256, qsm, st>>>(idx->rows, n, q_dev, idx->cand, idx->st, idx->near);
        LAUNCHED(idx);
    }
    {
        ProfScope ps(idx, K_RESOLVE);
        k_resolve_ed<<<1, 256, 0, st>>>(idx->rows, n, q_dev, idx->near, idx->st, idx->N, idx->row_begin, res, stats);
        LAUNCHED(idx);
    }
    return MESSI_OK;
}

static messi_status run_dtw(messi_index* idx, const float* q_dev, int reach, messi_result* res, messi_stats* stats)
{
    cudaStream_t st = idx->stream;
    const int n = idx->n;
    const int npad = (n + 3) & ~3;
    const size_t qsm = (size_t)npad * sizeof(float);
    int len = (int)(idx->window < idx->N ? idx->window : idx->N);
    const int wf = wavefront_warps(n, sizeof(float), 8);
    int seed_grid = (len + wf - 1) / wf;
    if (seed_grid > idx->sms * 4) seed_grid = idx->sms * 4;
    {
        ProfScope ps(idx, K_SEED);
        k_seed_dtw<<<seed_grid, 32 * wf, qsm + (size_t)wf * 3 * n * sizeof(float), st>>>(
            q_dev, n, reach, idx->rows, idx->skey, idx->perm, idx->N, idx->window, idx->beta32, idx->lo_w, idx->hi_w,
            idx->lut, idx->U, idx->L, idx->st);
        LAUNCHED(idx);
    }
    {
        ProfScope ps(idx, K_SCAN);
        k_scan<false><<<scan_grid(idx), 256, scan_smem(), st>>>(idx->tiles, idx->ntiles, idx->N, idx->lut, idx->st,
                                                                idx->cand, nullptr);
        LAUNCHED(idx);
    }
    {
        ProfScope ps(idx, K_LBK);
        k_lbk_filter<<<idx->sms * 4, 256, 2 * qsm, st>>>(idx->rows, n, idx->U, idx->L, idx->cand, idx->st, idx->list2);
        LAUNCHED(idx);
    }
    ProfScope* ref_scope = new ProfScope(idx, K_REFINE);
    bool launched = false;
#define LAUNCH_R(R)                                                                                           \
    if (!launched && reach == R) {                                                                            \
        k_refine_dtw<R><<<idx->sms * 8, 128, qsm, st>>>(idx->rows, n, q_dev, idx->list2, idx->st, idx->near); \
        ++idx->launches;                                                                                      \
        launched = true;                                                                                      \
    }
    MESSI_DTW_REACHES(LAUNCH_R)
#undef LAUNCH_R
    if (!launched) {
        k_refine_dtw_warp<<<idx->sms * 4, 32 * wf, qsm + (size_t)wf * 3 * n * sizeof(float), st>>>(
            idx->rows, n, reach, q_dev, idx->list2, idx->st, idx->near);
        ++idx->launches;
    }
    delete ref_scope;
    CK(cudaGetLastError());
    const int wr = wavefront_warps(n, sizeof(double), 8);
    {
        ProfScope ps(idx, K_RESOLVE);
        k_resolve_dtw<<<1, 32 * wr, (size_t)wr * 3 * n * sizeof(double), st>>>(idx->rows, n, reach, q_dev, idx->near,
                                                                              idx->st, idx->N, idx->row_begin, res, stats);
        LAUNCHED(idx);
    }
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
    CK(cudaMemcpyAsync(idx->qbuf, query, (size_t)idx->n * sizeof(float), cudaMemcpyHostToDevice, idx->stream));
    *q_dev = idx->qbuf;
    return MESSI_OK;
}

static messi_status finish_single(messi_index* idx, messi_result* local_best, messi_stats* stats)
{
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
    TRY(run_ed(idx, q, idx->res1, idx->stats1));
    return finish_single(idx, local_best, stats);
}

extern "C" messi_status messi_query_dtw(messi_index* idx, const float* query, int32_t reach, messi_result* local_best,
                                        messi_stats* stats)
{
    g_err[0] = 0;
    if (!idx || !query || !local_best) return fail(MESSI_EINVAL, "NULL argument");
    if (reach < 0 || reach > idx->n) return fail(MESSI_EINVAL, "reach %d outside [0, %d]", reach, idx->n);
    CK(cudaSetDevice(idx->device));
    const float* q = nullptr;
    TRY(stage_query(idx, query, &q));
    TRY(run_dtw(idx, q, reach, idx->res1, idx->stats1));
    return finish_single(idx, local_best, stats);
}

extern "C" messi_status messi_query_ed_batch(messi_index* idx, const float* queries_dev, int32_t nq,
                                             messi_result* results_dev, messi_stats* stats_dev)
{
    g_err[0] = 0;
    if (!idx || !queries_dev || !results_dev || nq < 0) return fail(MESSI_EINVAL, "bad argument");
    CK(cudaSetDevice(idx->device));
    for (int i = 0; i < nq; ++i)
        TRY(run_ed(idx, queries_dev + (size_t)i * idx->n, results_dev + i, stats_dev ? stats_dev + i : nullptr));
    return MESSI_OK;
}

extern "C" messi_status messi_query_dtw_batch(messi_index* idx, const float* queries_dev, int32_t nq, int32_t reach,
                                              messi_result* results_dev, messi_stats* stats_dev)
{
    g_err[0] = 0;
    if (!idx || !queries_dev || !results_dev || nq < 0) return fail(MESSI_EINVAL, "bad argument");
    if (reach < 0 || reach > idx->n) return fail(MESSI_EINVAL, "reach %d outside [0, %d]", reach, idx->n);
    CK(cudaSetDevice(idx->device));
    for (int i = 0; i < nq; ++i)
        TRY(run_dtw(idx, queries_dev + (size_t)i * idx->n, reach, results_dev + i, stats_dev ? stats_dev + i : nullptr));
    return MESSI_OK;
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
    long long total = idx->N * MESSI_W;
    k_detile<<<(unsigned)((total + 255) / 256), 256, 0, idx->stream>>>((const unsigned char*)idx->tiles, idx->N, sym_dev);
    LAUNCHED(idx);
    if (paa_dev)
        CK(cudaMemcpyAsync(paa_dev, idx->paa, (size_t)total * sizeof(float), cudaMemcpyDeviceToDevice, idx->stream));
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

extern "C" messi_status messi_debug_lower_bounds(messi_index* idx, const float* query_dev, int32_t reach, float* lb_dev)
{
    g_err[0] = 0;
    if (!idx || !query_dev || !lb_dev) return fail(MESSI_EINVAL, "NULL argument");
    if (reach > idx->n) return fail(MESSI_EINVAL, "reach %d > n", reach);
    CK(cudaSetDevice(idx->device));
    cudaStream_t st = idx->stream;
    const int n = idx->n;
    const size_t qsm = (size_t)((n + 3) & ~3) * sizeof(float);
    if (reach < 0) {
        k_seed_ed<<<1, 256, qsm, st>>>(query_dev, n, idx->rows, idx->skey, idx->perm, idx->N, 1, idx->beta32, idx->lo_w,
                                       idx->hi_w, idx->lut, idx->st);
    } else {
        k_seed_dtw<<<1, 32, qsm + 3 * (size_t)n * sizeof(float), st>>>(query_dev, n, reach, idx->rows, idx->skey, idx->perm,
                                                                      idx->N, 1, idx->beta32, idx->lo_w, idx->hi_w,
                                                                      idx->lut, idx->U, idx->L, idx->st);
    }
    LAUNCHED(idx);
    k_scan<true><<<scan_grid(idx), 256, scan_smem(), st>>>(idx->tiles, idx->ntiles, idx->N, idx->lut, idx->st, idx->cand,
                                                           lb_dev);
    LAUNCHED(idx);
    k_arm<<<1, 1, 0, st>>>(idx->st);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(st));
    return MESSI_OK;
}

extern "C" messi_status messi_debug_distances(messi_index* idx, const float* query_dev, int32_t reach,
                                              const uint32_t* ids_dev, int32_t k, float* d32_dev, double* d64_dev,
                                              float* lbk_dev)
{
    g_err[0] = 0;
    if (!idx || !query_dev || (!ids_dev && k > 0) || k < 0) return fail(MESSI_EINVAL, "bad argument");
    if (reach > idx->n) return fail(MESSI_EINVAL, "reach %d > n", reach);
    CK(cudaSetDevice(idx->device));
    cudaStream_t st = idx->stream;
    const int n = idx->n;
    const int npad = (n + 3) & ~3;
    if (reach >= 0) {  // envelope for LB_Keogh (prologue only)
        k_seed_dtw<<<1, 32, (size_t)npad * sizeof(float) + 3 * (size_t)n * sizeof(float), st>>>(
            query_dev, n, reach, idx->rows, idx->skey, idx->perm, idx->N, 1, idx->beta32, idx->lo_w, idx->hi_w, idx->lut,
            idx->U, idx->L, idx->st);
        LAUNCHED(idx);
        k_arm<<<1, 1, 0, st>>>(idx->st);
        LAUNCHED(idx);
    }
    const int wr = wavefront_warps(n, sizeof(double), 4);
    const size_t smem = 3 * (size_t)npad * sizeof(float) + (size_t)wr * 3 * n * sizeof(double);
    int grid = (k + wr - 1) / wr;
    if (grid > idx->sms * 8) grid = idx->sms * 8;
    if (grid < 1) grid = 1;
    bool launched = false;
#define LAUNCH_D(R)                                                                                          \
    if (!launched && reach == R) {                                                                           \
        k_debug_dist<R><<<grid, 32 * wr, smem, st>>>(idx->rows, n, reach, query_dev, idx->U, idx->L, ids_dev, k, \
                                                     d32_dev, d64_dev, lbk_dev);                             \
        launched = true;                                                                                     \
    }
    MESSI_DTW_REACHES(LAUNCH_D)
#undef LAUNCH_D
    if (!launched)
        k_debug_dist<-1><<<grid, 32 * wr, smem, st>>>(idx->rows, n, reach, query_dev, idx->U, idx->L, ids_dev, k, d32_dev,
                                                      d64_dev, lbk_dev);
    LAUNCHED(idx);
    CK(cudaStreamSynchronize(st));
    return MESSI_OK;
}
