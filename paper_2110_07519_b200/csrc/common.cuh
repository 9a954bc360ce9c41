// common.cuh -- shared device definitions of libmessi (the CUDA product path).
// Independent of oracle/ (no shared code, tables or constants).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define MESSI_W 16                 // PAA segments ("w is fixed to 16")
#define MESSI_CARD 256             // 8-bit iSAX symbols
#define MESSI_TILE_ROWS 512        // series per tile (32 blocks x 16 series)
#define MESSI_TILE_BYTES 4096      // tile: 8 tile rows x 512 B of cardinality-16 pair bytes
#define MESSI_MAX_N 8192
#define MESSI_MAX_PEERS 8          // shards that share each query's best-so-far (batched ED)

// Bounds checks of the checked build (-DMESSI_CHECKED, tools/checked.sh): every computed
// index into a list, buffer or shared array is asserted against its capacity and a violation
// traps the kernel (the CUDA call then fails loudly).  No code in the normal build.
#ifdef MESSI_CHECKED
#define MESSI_CHECK(cond)                                                                                         \
    do {                                                                                                          \
        if (!(cond)) {                                                                                            \
            printf("MESSI_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, blockIdx.x,   \
                   threadIdx.x);                                                                                  \
            __trap();                                                                                             \
        }                                                                                                         \
    } while (0)
#else
#define MESSI_CHECK(cond) \
    do {                  \
    } while (0)
#endif

namespace messi {

// Relative slack on every prune / abandon / near-tie test:
// thr = BSF * (1 + 2^-12), rounded up.  > 10x the fp32 error of any distance we compare.
__device__ __forceinline__ float slack_up(float bsf) { return __fmul_ru(bsf, 1.000244140625f); }

// Per-query device state.  bsf_bits holds a non-negative fp32 whose bit pattern orders
// like the value, so atomicMin on the bits is a monotone BSF update (Observation 1,
// BSF only decreases).  The resolve kernel re-arms it for the next query.
struct QState {
    unsigned bsf_bits;      // current best-so-far (fp32 bits), +inf when armed
    unsigned seed_bits;     // BSF0 after the approximate search
    unsigned cand_count;    // series-bound survivors appended by the scan
    unsigned list2_count;   // DTW: LB_Keogh survivors
    unsigned near_count;    // near-best entries (d32 <= thr at refine time)
    unsigned refined;       // real distances started
    unsigned abandoned;     // real distances abandoned early
    unsigned done;          // CTAs of the refine stage that finished (last one resolves)
    unsigned tile_count;    // tiles whose box bound <= BSF0 * (1 + eps) (batch ED: those <= BSF0 / 2)
    unsigned tile_back;     // batch ED: the listed tiles with box bound > BSF0 / 2 (list back end)
    unsigned exact;         // ED: fp32 distances over the raw rows (quantised bound passed)
    unsigned tiles_scanned; // batch ED: tiles whose box bound still passed the CURRENT BSF
    unsigned coarse_count;  // series whose cardinality-16 bound passed (fine bound evaluated)
    unsigned tiles_done;    // batch ED: listed tiles finished (the warp finishing the last finalises)
    unsigned lock;          // batch ED: guards best_d / best_id
    unsigned tile_hist[16]; // batch ED: listed tiles per best-first bin (k_filter_batch -> k_order_tiles)
    unsigned tile_cur[16];  // batch ED: k_order_tiles' per-bin fill cursors
    // batch ED: next pair of listed tiles to hand out -- the fused kernel's hot claim counter,
    // alone on its 128-byte line: loads of the fields above (the BSF every warp reads once per
    // pair) would otherwise queue behind the claims at the L2 slice that owns the line
    alignas(128) unsigned next_tile;
    unsigned next_tile_pad[31];
    unsigned long long dtw_cells;  // DTW band cells evaluated in fp32 (refine)
    unsigned long long gbsf; // batch ED: the epoch-tagged best-so-far of all shards (PeerSet)
    double best_d;          // batch ED: lexicographic min (d64, id) over the fp64 re-ranked rows
    long long best_id;
    unsigned long long qkey;  // query's approximate-search key
    int window_start;       // first sorted position of the approximate-search window
    int window_len;
    double ubar[16], lbar[16];  // query PAA (ED: both) or envelope PAA (DTW), fp64
    unsigned char zlo[16], zhi[16];  // batch ED: per segment, the symbols whose table entry is 0
    unsigned lbk_thr_bits;  // DTW: the scan's threshold (BSF0), used by the LB_Keogh filter
    unsigned list2_back;    // DTW: LB_Keogh survivors appended from the back of list2 (larger LBK)
    unsigned rev_count;     // DTW: forward survivors queued for the reverse LB_Keogh (rlist)
    // DTW: the query's own PAA per segment, fp32 bounds below / above (directed fp64 sums), for
    // the scan's reverse envelope-PAA bound against the rows' envelope symbols (renv)
    float qlo[16], qhi[16];
    unsigned rcand_count;   // DTW: scan candidates that also passed the reverse envelope-PAA bound
    unsigned rev_paa;       // DTW: 1 when k_rev_paa_filter ran for this query
    // batch ED: the query quantised like the rows ("quantised-row bound"):
    // c_q = rint(q / s_q) in [-127, 127], s_q a power of two; q8e >= ||q - s_q c_q||;
    // q8sum = sum c_q, q8s2ss = s_q^2 sum c_q^2 (exact in fp64); the words go to qc_all
    float q8s;
    int q8sum;
    double q8e, q8s2ss;
    unsigned frozen;        // inspection only (messi_debug_dtw_stages): the DTW refine kernels keep
                            // their threshold at its start value and never lower the BSF, so every
                            // candidate runs to completion (no abandon) and reports its fp32 DTW
};

struct NearEntry { unsigned id; float d32; };

// k-NN (k > 1) state of one query of the batched ED path, under QState::lock: the k smallest
// fp32 distances of the rows refined so far (their k-th is the pruning threshold, held in
// bsf_bits) and the k lexicographically smallest (fp64 d2, id) of the rows re-ranked.
#define MESSI_MAX_K 64
constexpr size_t kStatsBytes = 112;  // sizeof(messi_stats) (include/messi.h; asserted in api.cu)
struct KnnState {
    float d32[MESSI_MAX_K];
    double d64[MESSI_MAX_K];
    long long id[MESSI_MAX_K];
    int n32, n64;
};

// Best-so-far shared with the other shards of a row-sharded collection (batched ED path):
// the per-query states of up to MESSI_MAX_PEERS peer indexes (peer GPUs' memory reached over
// NVLink, or other indexes of this process) and the launch epoch every shard tags its
// updates with.  gbsf = epoch << 32 | (0xffffffff - fp32 bits) is raised with atomicMax: a
// newer epoch wins, within an epoch the smaller distance wins, and a reader ignores other
// epochs -- so a peer running a batch ahead can never lower this batch's threshold.
struct PeerSet {
    QState* const* st;  // device array of the n peers' per-query state arrays
    int n;
    unsigned epoch;
};

__device__ __forceinline__ void arm_state(QState* st)
{
    st->bsf_bits = 0x7f800000u;
    st->seed_bits = 0x7f800000u;
    st->cand_count = 0;
    st->list2_count = 0;
    st->list2_back = 0;
    st->rev_count = 0;
    st->rcand_count = 0;
    st->rev_paa = 0;
    st->near_count = 0;
    st->refined = 0;
    st->abandoned = 0;
    st->done = 0;
    st->tile_count = 0;
    st->tile_back = 0;
    st->exact = 0;
    st->tiles_scanned = 0;
    st->next_tile = 0;
    st->coarse_count = 0;
    st->tiles_done = 0;
    for (int j = 0; j < 16; ++j) st->tile_hist[j] = st->tile_cur[j] = 0;
    st->lock = 0;
    st->best_d = (double)INFINITY;
    st->best_id = -1;
    st->dtw_cells = 0;
    st->frozen = 0;
}

// mbarrier (TMA / bulk-copy completion) wrappers.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Waits for the phase of parity `parity` to complete; the suspend-time hint lets the hardware
// park the waiting thread until then instead of spinning on issue slots the epilogue needs.
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity)
{
    const unsigned a = smem_u32(b);
    unsigned ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 1000000;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

// Bulk copy (TMA, non-tensor) of `bytes` (a multiple of 16, 16-byte aligned ends) from global
// to shared memory, completing on mbarrier b, in chunks of at most 32 KB; one thread issues.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b)
{
    for (unsigned off = 0; off < bytes; off += 32768u) {
        const unsigned len = min(32768u, bytes - off);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(static_cast<char*>(dst) + off)),
                     "l"(static_cast<const char*>(src) + off), "r"(len), "r"(smem_u32(b))
                     : "memory");
    }
}

// Paired fp32 arithmetic (Blackwell FADD2 / FFMA2: two lanes of fp32 per instruction on the
// FMA pipe -- half the issue slots of two scalar ops).
__device__ __forceinline__ float2 fadd2_rd(float2 a, float2 b)
{
    float2 r;
    asm("{\n .reg .b64 x, y, z;\n mov.b64 x, {%2, %3};\n mov.b64 y, {%4, %5};\n add.rm.f32x2 z, x, y;\n"
        " mov.b64 {%0, %1}, z;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 fsub2_rd(float2 a, float2 b)
{
    float2 r;
    asm("{\n .reg .b64 x, y, z;\n mov.b64 x, {%2, %3};\n mov.b64 y, {%4, %5};\n sub.rm.f32x2 z, x, y;\n"
        " mov.b64 {%0, %1}, z;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b)
{
    float2 r;
    asm("{\n .reg .b64 x, y, z;\n mov.b64 x, {%2, %3};\n mov.b64 y, {%4, %5};\n add.rn.f32x2 z, x, y;\n"
        " mov.b64 {%0, %1}, z;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c)
{
    float2 r;
    asm("{\n .reg .b64 x, y, z, w;\n mov.b64 x, {%2, %3};\n mov.b64 y, {%4, %5};\n mov.b64 z, {%6, %7};\n"
        " fma.rn.f32x2 w, x, y, z;\n mov.b64 {%0, %1}, w;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

// Four-way byte dot products with 32-bit accumulation (IDP.4A): exact integer arithmetic.
__device__ __forceinline__ int dp4a_us(unsigned a, unsigned b, int c)  // a: 4 x u8, b: 4 x s8
{
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int dp4a_ss(unsigned a, unsigned b, int c)  // a, b: 4 x s8
{
    int d;
    asm("dp4a.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ unsigned dp4a_uu(unsigned a, unsigned b, unsigned c)  // a, b: 4 x u8
{
    unsigned d;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ float2 ffma2_rd(float2 a, float2 b, float2 c)
{
    float2 r;
    asm("{\n .reg .b64 x, y, z, w;\n mov.b64 x, {%2, %3};\n mov.b64 y, {%4, %5};\n mov.b64 z, {%6, %7};\n"
        " fma.rm.f32x2 w, x, y, z;\n mov.b64 {%0, %1}, w;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
__device__ __forceinline__ float max3f(float a, float b, float c)
{
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__device__ __forceinline__ float warp_sum(float v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_min(float v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float ld_bsf(const QState* st)
{
    return __uint_as_float(*(volatile const unsigned*)&st->bsf_bits);
}

__device__ __forceinline__ void bsf_update(QState* st, float d)
{
    if (d >= 0.0f) atomicMin(&st->bsf_bits, __float_as_uint(d));
}

// The threshold source of the batched ED path: the local BSF, lowered by the shards' shared
// one when it carries this launch's epoch (epoch 0 = unlinked: gbsf is not read).
// (GPU-scope relaxed load: a stale value is a valid, larger threshold; a volatile load
// compiles to a system-scope strong load, which was measured to wait behind the warp's
// in-flight claim atomic.)
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <bool LINKED>
__device__ __forceinline__ float ld_bsf_l(const QState* st, unsigned epoch)
{
    if (!LINKED) return __uint_as_float(ld_relaxed_gpu(&st->bsf_bits));
    const float loc = __uint_as_float(*(volatile const unsigned*)&st->bsf_bits);
    const unsigned long long g = *(volatile const unsigned long long*)&st->gbsf;
    if ((unsigned)(g >> 32) == epoch) return fminf(loc, __uint_as_float(0xffffffffu - (unsigned)g));
    return loc;
}

__device__ __forceinline__ float ld_bsf_eff(const QState* st, unsigned epoch)
{
    const float loc = __uint_as_float(*(volatile const unsigned*)&st->bsf_bits);
    if (epoch == 0u) return loc;  // unlinked: the local BSF only (one load)
    const unsigned long long g = *(volatile const unsigned long long*)&st->gbsf;
    if ((unsigned)(g >> 32) == epoch) return fminf(loc, __uint_as_float(0xffffffffu - (unsigned)g));
    return loc;
}

// A new local best d of query b: the local BSF, and (linked) every peer's shared one.
// The peer fan-out is out of line (rare: a few BSF improvements per query) and uses global-
// space atomics explicitly, so the hot kernels do not carry generic-address atomic code.
__device__ __noinline__ void bsf_publish_peers(PeerSet ps, int b, float d)
{
    const unsigned long long key = ((unsigned long long)ps.epoch << 32) | (0xffffffffu - __float_as_uint(d));
    for (int i = 0; i < ps.n; ++i) {
        unsigned long long* a = &ps.st[i][b].gbsf;
        asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(a)), "l"(key) : "memory");
    }
}

__device__ __forceinline__ void bsf_publish(QState* st, PeerSet ps, int b, float d)
{
    bsf_update(st, d);
    if (ps.n > 0 && d >= 0.0f) bsf_publish_peers(ps, b, d);
}

// Symbol of a fp32 PAA value: #{k : beta32_k <= x} over the 255 ascending breakpoints
// (reading R3/R4: ascending, ties go to the region above).  Branch-free binary search.
__device__ __forceinline__ int symbol_of(float x, const float* beta)
{
    int pos = 0;
#pragma unroll
    for (int step = 128; step; step >>= 1)
        if (pos + step <= 255 && beta[pos + step - 1] <= x) pos += step;
    return pos;
}

}  // namespace messi
