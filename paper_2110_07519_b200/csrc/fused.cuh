// fused.cuh -- the batched ED query path: B queries per launch group, four kernels.
//
//   k_prologue_batch  (B CTAs)        query PAA, key, lower-bound tables (A3), and the
//                                     approximate-search position of the key (A4 part 1)
//   k_seed_batch      (S x B CTAs)    real distances of the window rows -> BSF0 (A4)
//   k_filter_batch    (tiles x B/2)   box bound of every tile for every query (Alg. 7 node
//                                     pruning on the flat tile array) -> per-query tile lists
//   k_scan_refine_ed  (persistent)    work chunks of (query, 16 listed tiles) in query order:
//                                     box re-check against the CURRENT BSF, series bounds
//                                     (A5), quantised-row bound, fp32 distance (A7), fp64
//                                     re-rank of near-best rows (A9) -- all in one pass, as
//                                     Alg. 9's workers do; the CTA finishing a
//                                     query's last chunk writes its result.
//
// The batch replaces MESSI's one-query-at-a-time loop by one persistent pass
// over the work of all B queries (results per query are unchanged: every query is exact).
#pragma once
#include "common.cuh"
#include "dtw.cuh"
#include "refine.cuh"
#include "scan.cuh"

namespace messi {

constexpr int kLutX = MESSI_CARD * 64;   // expanded scan table: word v*64 + 16h + s (64 KB)
constexpr int kLutF = MESSI_CARD * 32;   // filter table: word v*32 + 16h + s (32 KB)
constexpr int kChunkTiles = 16;          // tiles per work chunk (2 per warp)
#ifndef MESSI_FUSED_WARPS
#define MESSI_FUSED_WARPS 12
#endif
constexpr int kFusedWarps = MESSI_FUSED_WARPS;  // 2 CTAs of 12 warps per SM (64 KB table each)
#ifndef MESSI_FUSED_MINB
#define MESSI_FUSED_MINB 2
#endif
constexpr int kCandBuf = 64;            // per-warp buffer of fine survivors awaiting the refine
constexpr int kBatchMax = 128;           // queries per launch group
constexpr int kFilterQ = 2;              // queries per filter CTA
constexpr int kTileBins = 16;            // best-first bins of a query's tile list (k_order_tiles)
constexpr unsigned kTileMask = 0x0fffffffu;    // list entry .x: tile | bin << 28
constexpr unsigned kClaimsDone = 0x40000000u;  // next_tile raised to this: no listed pair left

// Best-first bins of a query's listed tiles: bin j = min(15, (int)fl(lb * sc)) with sc = 16 /
// (BSF0 (1 + eps)) from the query's local seed (the same value in every kernel: the filter
// keeps lb <= BSF (1 + eps) <= that, so bins cover [0, 15]); sc = 0 (no finite seed): bin 0.
__device__ __forceinline__ float tile_bin_scale(const QState* st)
{
    const float t = slack_up(__uint_as_float(*(volatile const unsigned*)&st->seed_bits));
    return (t > 0.0f && t < INFINITY) ? (float)kTileBins / t : 0.0f;
}
__device__ __forceinline__ int tile_bin(float lb, float sc) { return min(kTileBins - 1, (int)(lb * sc)); }
// A lower bound of every bound in bin j: fl(lb sc) >= j, so lb sc >= j (1 - 2^-24) and
// lb >= j / sc (1 - 2^-24) >= fl_rd(j / sc) (1 - 2^-20).
__device__ __forceinline__ float tile_bin_floor(int j, float sc)
{
    return (j == 0 || sc == 0.0f) ? 0.0f : __fdiv_rd((float)j, sc) * (1.0f - 0x1p-20f);
}

// ------------------------------------------------------------------------ prologue
// One CTA per query: arms the query's state, runs the prologue (prologue_block: PAA in fp64,
// key, T[s][v] rounded down) into the compact table, then lays the table out for the scan
// (expanded, conflict-free) and the filter, finds the per-segment zero runs
// [zlo_s, zhi_s] of T (T[s][.] is non-increasing, zero on one run, non-decreasing: the box
// of a symbol moves monotonically past the query mean), and locates the query's key in the
// sorted keys (the approximate-search window, reading R14).
// The query quantised like the rows (k_quantise's recipe): s_q the smallest power of two with
// max |q_i| <= 127 s_q, c_q = rint(q / s_q); e_q >= ||q - s_q c_q|| (fp64 sum, sqrt inflated by
// 2^-30 and rounded up); words qc[n/4] = 4 x s8 each.  A query that cannot be quantised (non-
// finite values, scale outside 2^+-100) gets e_q = +inf: the quantised bound then never prunes.
__device__ void quantise_query_block(const float* q_s, int n, unsigned* __restrict__ qc, QState* st)
{
    __shared__ float mx_s[32];
    __shared__ double er_s[32];
    __shared__ int sm_s[32], ss_s[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    float mx = 0.0f;
    for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmaxf(mx, fabsf(q_s[i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) mx_s[w] = mx;
    __syncthreads();
    mx = mx_s[0];
    for (int k = 1; k < nw; ++k) mx = fmaxf(mx, mx_s[k]);
    bool usable = isfinite(mx);
    int kq = 0;
    if (usable && mx > 0.0f) {
        int e;
        const float f = frexpf(mx, &e);
        kq = (f * 128.0f <= 127.0f) ? e - 7 : e - 6;
        if (kq < -100 || kq > 100) usable = false;
    }
    const float sq = ldexpf(1.0f, kq);
    double err = 0.0;
    int sum = 0, ss = 0;
    for (int wd = threadIdx.x; wd < n / 4; wd += blockDim.x) {
        unsigned word = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float x = q_s[4 * wd + j];
            const int c = usable ? (int)rintf(ldexpf(x, -kq)) : 0;
            const double r = __dsub_rn((double)x, (double)c * (double)sq);
            err = __dadd_rn(err, __dmul_rn(r, r));
            sum += c;
            ss += c * c;
            word |= (unsigned)(c & 255) << (8 * j);
        }
        qc[wd] = word;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        err = __dadd_rn(err, __shfl_xor_sync(0xffffffffu, err, o));
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if (lane == 0) { er_s[w] = err; sm_s[w] = sum; ss_s[w] = ss; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < nw; ++k) { err = __dadd_rn(err, er_s[k]); sum += sm_s[k]; ss += ss_s[k]; }
        st->q8s = sq;
        st->q8sum = sum;
        st->q8s2ss = (double)sq * (double)sq * (double)ss;
        st->q8e = usable ? sqrt(err) * (1.0 + 0x1p-30) : (double)INFINITY;
    }
}

__global__ void __launch_bounds__(256) k_prologue_batch(const float* __restrict__ queries, int n,
                                                        const float* __restrict__ beta_g, const float* __restrict__ lo_w,
                                                        const float* __restrict__ hi_w,
                                                        const unsigned long long* __restrict__ skey, long long N,
                                                        int window, float* __restrict__ lutc_all,
                                                        float* __restrict__ lutx_all, float* __restrict__ lutf_all,
                                                        QState* st_all, KnnState* knn, unsigned* __restrict__ qc_all)
{
    extern __shared__ __align__(16) float q_s[];
    __shared__ unsigned long long qkey_s;
    const int b = blockIdx.x;
    QState* st = st_all + b;
    const float* q = queries + (size_t)b * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q[i];
    if (threadIdx.x == 0) {
        arm_state(st);
        if (knn) knn[b].n32 = knn[b].n64 = 0;
    }
    __syncthreads();
    if (qc_all) quantise_query_block(q_s, n, qc_all + (size_t)b * (n / 4), st);
    float* lutc = lutc_all + (size_t)b * (MESSI_W * MESSI_CARD);
    prologue_block(q_s, n, -1, beta_g, lo_w, hi_w, lutc, lutx_all + (size_t)b * kLutX, nullptr, nullptr, &qkey_s, st);
    __syncthreads();
    float* lutf = lutf_all + (size_t)b * kLutF;
    for (int i = threadIdx.x; i < MESSI_W * MESSI_CARD; i += blockDim.x) {
        const int s = i >> 8, v = i & 255;
        const float val = lutc[i];
        lutf[v * 32 + s] = val;
        lutf[v * 32 + 16 + s] = val;
    }
    if (threadIdx.x < MESSI_W) {
        const int s = threadIdx.x;
        int lo = 256, hi = -1;
        for (int v = 0; v < 256; ++v)
            if (lutc[s * 256 + v] == 0.0f) { lo = min(lo, v); hi = max(hi, v); }
        if (hi < 0) { lo = 255; hi = 0; }  // cannot happen (boxes tile the line); empty run is still safe
        st->zlo[s] = (unsigned char)lo;
        st->zhi[s] = (unsigned char)hi;
    }
    const unsigned long long qkey = qkey_s;
    const long long a = block_lower_bound(skey, N, qkey);
    if (threadIdx.x == 0) {
        const int len = (int)min((long long)window, N);
        st->qkey = qkey;
        st->window_start = (int)max(0LL, min(a - len / 2, N - len));
        st->window_len = len;
    }
}

// ------------------------------------------------------------------------------ seed
// Real distances of the approximate-search window (Alg. 5 approxSearch): CTA
// (j, b) takes rows [j*per, (j+1)*per) of query b's window, one warp per group of four rows
// (four rows in flight), and lowers BSF0 with atomicMin (fp32 bits).
constexpr int kSeedRowsPerCta = 64;
__global__ void __launch_bounds__(256) k_seed_batch(const float* __restrict__ queries, int n,
                                                    const float* __restrict__ rows, const unsigned* __restrict__ perm,
                                                    QState* st_all, PeerSet ps, float* __restrict__ seed_d, int seed_cap)
{
    extern __shared__ __align__(16) float q_s[];
    const int b = blockIdx.y;
    QState* st = st_all + b;
    const float* q = queries + (size_t)b * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q[i];
    __syncthreads();
    const int start = st->window_start, len = st->window_len;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int k0 = blockIdx.x * kSeedRowsPerCta;
    float best = INFINITY;
    for (int g = k0 + 4 * w; g < min(len, k0 + kSeedRowsPerCta); g += 4 * (blockDim.x >> 5)) {
        unsigned id[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            ok[u] = g + u < min(len, k0 + kSeedRowsPerCta);
            id[u] = ok[u] ? perm[start + g + u] : 0u;
        }
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int j = lane * 4; j < n; j += 128) {
            const float4 qv = *reinterpret_cast<const float4*>(q_s + j);
            float4 cv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                cv[u] = ok[u] ? __ldg(reinterpret_cast<const float4*>(rows + (long long)id[u] * n + j))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float d;
                d = qv.x - cv[u].x; acc[u] = fmaf(d, d, acc[u]);
                d = qv.y - cv[u].y; acc[u] = fmaf(d, d, acc[u]);
                d = qv.z - cv[u].z; acc[u] = fmaf(d, d, acc[u]);
                d = qv.w - cv[u].w; acc[u] = fmaf(d, d, acc[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float d = warp_sum(acc[u]);
            if (ok[u]) {
                best = fminf(best, d);
                if (seed_d && lane == 0) seed_d[(size_t)b * seed_cap + g + u] = d;  // k-NN: every window distance
            }
        }
    }
    if (!seed_d && lane == 0 && best < INFINITY) {  // 1-NN: the window's best is BSF0
        bsf_publish(st, ps, b, best);
        atomicMin(&st->seed_bits, __float_as_uint(best));
    }
}

// k-NN seed: the k-th smallest fp32 distance of the window (a distance k rows achieve) is
// BSF0; one CTA per query sorts the window's distances in shared memory (bitonic).
__global__ void __launch_bounds__(1024) k_seed_select(const float* __restrict__ seed_d, int seed_cap, int k,
                                                      QState* st_all, PeerSet ps, int slot)
{
    extern __shared__ float sv[];
    const int b = blockIdx.x;
    QState* st = st_all + b;
    const int len = st->window_len;
    int np = 1;
    while (np < len) np <<= 1;
    for (int i = threadIdx.x; i < np; i += blockDim.x) sv[i] = i < len ? seed_d[(size_t)b * seed_cap + i] : INFINITY;
    __syncthreads();
    for (int size = 2; size <= np; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < np; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const float a = sv[i], c = sv[j];
                    if ((a > c) == up) { sv[i] = c; sv[j] = a; }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x == 0 && len >= k && sv[k - 1] < INFINITY) {
        bsf_publish(st, ps, slot >= 0 ? slot : b, sv[k - 1]);  // slot: a DTW slot (its peers' index)
        atomicMin(&st->seed_bits, __float_as_uint(sv[k - 1]));
    }
}

// --------------------------------------------------------------------------- filter
// Box bound of a tile for one query (Alg. 7 line "FindDist(node) > BSF -> prune"):
// per segment the tile's symbols lie in [vmin, vmax]; the smallest table entry over that
// range is 0 if it meets the zero run [zlo, zhi], else T[vmax] (range below the run) or
// T[vmin] (above it) -- so sum_s of it (round-down adds) lower-bounds every member's bound.
// mn / mx are the box bytes rotated by r = lane & 15, so that at step s lane l reads
// segment (s + l) mod 16 from table copy l >> 4 (T = table + 16 (l >> 4)): 32 distinct banks.
__device__ __forceinline__ float box_lb(uint4 mn, uint4 mx, const float* T, const unsigned char* zlo,
                                        const unsigned char* zhi, int r)
{
    const unsigned a[4] = {mn.x, mn.y, mn.z, mn.w}, c[4] = {mx.x, mx.y, mx.z, mx.w};
    float acc = 0.0f;
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const int sg = (s + r) & 15;
        const unsigned vmin = (a[s >> 2] >> (8 * (s & 3))) & 255u, vmax = (c[s >> 2] >> (8 * (s & 3))) & 255u;
        const unsigned zl = zlo[sg], zh = zhi[sg];
        const unsigned v = vmax < zl ? vmax : vmin;
        const float term = T[v * 32 + sg];
        acc = __fadd_rd(acc, (vmin <= zh && vmax >= zl) ? 0.0f : term);
    }
    return acc;
}

// Super-tile boxes: the union box of kSuperTiles consecutive tiles (a node one level up the
// key-sorted "tree"), bytewise min of the mins / max of the maxes.
constexpr int kSuperTiles = 16;
__global__ void k_superbox(const uint4* __restrict__ boxes, long long ntiles, uint4* __restrict__ sboxes)
{
    const long long S = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long t0 = S * kSuperTiles;
    if (t0 >= ntiles) return;
    uint4 mn = boxes[2 * t0], mx = boxes[2 * t0 + 1];
    for (long long t = t0 + 1; t < min(ntiles, t0 + kSuperTiles); ++t) {
        const uint4 a = boxes[2 * t], c = boxes[2 * t + 1];
        mn = make_uint4(__vminu4(mn.x, a.x), __vminu4(mn.y, a.y), __vminu4(mn.z, a.z), __vminu4(mn.w, a.w));
        mx = make_uint4(__vmaxu4(mx.x, c.x), __vmaxu4(mx.y, c.y), __vmaxu4(mx.z, c.z), __vmaxu4(mx.w, c.w));
    }
    sboxes[2 * S] = mn;
    sboxes[2 * S + 1] = mx;
}

// Two-level filter, kFilterQ queries per CTA: a warp tests 32 super-tiles (one per lane);
// the tiles of every super-tile that passes are tested 16 at a time (half-warps), and the
// kept tiles are appended as (tile, bound) to the query's staging list (k_order_tiles then
// lays the list out best-first for the fused kernel).
__global__ void __launch_bounds__(256, 3) k_filter_batch(const uint4* __restrict__ boxes, const uint4* __restrict__ sboxes,
                                                      long long ntiles, long long nsuper,
                                                      const float* __restrict__ lutf_all, QState* st_all, int B,
                                                      uint2* __restrict__ tlist_all, unsigned epoch)
{
    extern __shared__ __align__(16) float lutf_s[];  // kFilterQ * kLutF
    __shared__ unsigned char zlo[kFilterQ][16], zhi[kFilterQ][16];
    __shared__ float thr_s[kFilterQ], sc_s[kFilterQ];
    __shared__ unsigned hist_s[kFilterQ][kTileBins];
    __shared__ __align__(8) unsigned long long tab_bar;
    const int b0 = blockIdx.y * kFilterQ;
    const int nq = min(kFilterQ, B - b0);
    if (threadIdx.x == 0) {  // the queries' tables: one bulk copy, overlapped with the set-up below
        mbar_init(&tab_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&tab_bar, (unsigned)(nq * kLutF * 4));
        bulk_g2s(lutf_s, lutf_all + (size_t)b0 * kLutF, (unsigned)(nq * kLutF * 4), &tab_bar);
    }
    if (threadIdx.x < nq * 16) {
        const int qq = threadIdx.x >> 4, s = threadIdx.x & 15;
        zlo[qq][s] = st_all[b0 + qq].zlo[s];
        zhi[qq][s] = st_all[b0 + qq].zhi[s];
    }
    if (threadIdx.x < nq) {
        thr_s[threadIdx.x] = slack_up(ld_bsf_eff(st_all + b0 + threadIdx.x, epoch));
        sc_s[threadIdx.x] = tile_bin_scale(st_all + b0 + threadIdx.x);
    }
    if (threadIdx.x < kFilterQ * kTileBins) hist_s[threadIdx.x / kTileBins][threadIdx.x % kTileBins] = 0u;
    __syncthreads();
    mbar_wait(&tab_bar, 0);
    const int lane = threadIdx.x & 31, r = lane & 15, h = lane >> 4;
    const int wpb = blockDim.x >> 5;
    for (long long s0 = ((long long)blockIdx.x * wpb + (threadIdx.x >> 5)) * 32; s0 < nsuper;
         s0 += (long long)gridDim.x * wpb * 32) {
        const long long S = s0 + lane;
        const bool sval = S < nsuper;
        uint4 smn = make_uint4(0, 0, 0, 0), smx = make_uint4(0, 0, 0, 0);
        if (sval) {
            smn = rotate_bytes(sboxes[2 * S], r);
            smx = rotate_bytes(sboxes[2 * S + 1], r);
        }
        for (int qq = 0; qq < nq; ++qq) {
            const float* T = lutf_s + qq * kLutF + 16 * h;
            const float thr = thr_s[qq];
            const bool skeep = sval && box_lb(smn, smx, T, zlo[qq], zhi[qq], r) <= thr;
            unsigned m = __ballot_sync(0xffffffffu, skeep);
            QState* st = st_all + b0 + qq;
            while (m) {
                const int S1 = __ffs(m) - 1;
                m &= m - 1;
                const int S2 = m ? __ffs(m) - 1 : -1;
                if (m) m &= m - 1;
                const int mine = h == 0 ? S1 : S2;
                const long long t = mine >= 0 ? (s0 + mine) * kSuperTiles + r : ntiles;
                const bool tval = t < ntiles;
                bool keep = false;
                float lb = 0.0f;
                if (tval) {
                    const uint4 mn = rotate_bytes(boxes[2 * t], r), mx = rotate_bytes(boxes[2 * t + 1], r);
                    lb = box_lb(mn, mx, T, zlo[qq], zhi[qq], r);
                    keep = lb <= thr;
                }
                // kept tiles are appended (tile, bound) to the query's staging list; k_order_tiles
                // then lays them out best-first
                const unsigned mk = __ballot_sync(0xffffffffu, keep);
                if (mk) {
                    unsigned base = 0;
                    if (lane == 0) base = atomicAdd(&st->tile_count, (unsigned)__popc(mk));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    uint2* tl = tlist_all + (size_t)(b0 + qq) * ntiles;
                    MESSI_CHECK(!keep || base + __popc(mk & ((1u << lane) - 1)) < (unsigned)ntiles);
                    if (keep) {
                        tl[base + __popc(mk & ((1u << lane) - 1))] = make_uint2((unsigned)t, __float_as_uint(lb));
                        atomicAdd(&hist_s[qq][tile_bin(lb, sc_s[qq])], 1u);
                    }
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < nq * kTileBins) {
        const unsigned c = hist_s[threadIdx.x / kTileBins][threadIdx.x % kTileBins];
        if (c) atomicAdd(&st_all[b0 + threadIdx.x / kTileBins].tile_hist[threadIdx.x % kTileBins], c);
    }
}

// Best-first layout of a query's listed tiles (kOrderCtas CTAs per query, each a contiguous
// slice of the staging list): a counting sort by bin (tile_bin; bin sizes from the filter's
// histogram): bin 0, bin 1, ... (order inside a bin arbitrary), each entry (tile | j << 28,
// lb).  fl(lb sc) is monotone in lb, so every tile of a later bin has a larger bound than any
// tile of an earlier one: once the best-so-far drops below tile_bin_floor(j) for the bin j of
// a claimed tile, every tile from there on is box-pruned and the fused kernel voids the
// query's remaining claims.  A CTA counts its slice per bin (shared memory), reserves one
// range per bin in the query's list (global cursor), then scatters its slice; lanes of one
// warp with the same bin take consecutive slots (__match_any_sync).  Tiles are < 2^28
// (sorted positions are 32-bit: ntiles < 2^23).
constexpr int kOrderCtas = 64;
__global__ void __launch_bounds__(256) k_order_tiles(const uint2* __restrict__ stage_all, QState* st_all,
                                                     long long ntiles, uint2* __restrict__ tlist_all)
{
    __shared__ unsigned cnt[kTileBins], cur[kTileBins];
    const int b = blockIdx.y;
    QState* st = st_all + b;
    const unsigned count = st->tile_count;
    const unsigned per = (count + kOrderCtas - 1) / kOrderCtas;
    const unsigned lo = min(count, blockIdx.x * per), hi = min(count, lo + per);
    if (lo >= hi) return;
    const float sc = tile_bin_scale(st);
    const uint2* in = stage_all + (size_t)b * ntiles;
    uint2* out = tlist_all + (size_t)b * ntiles;
    if (threadIdx.x < kTileBins) cnt[threadIdx.x] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (unsigned i0 = lo + (threadIdx.x & ~31u); i0 < hi; i0 += blockDim.x) {
        const unsigned i = i0 + lane;
        const int j = i < hi ? tile_bin(__uint_as_float(in[i].y), sc) : kTileBins;
        const unsigned peers = __match_any_sync(0xffffffffu, j);
        if (j < kTileBins && lane == __ffs(peers) - 1) atomicAdd(&cnt[j], (unsigned)__popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < kTileBins) {
        const int j = threadIdx.x;
        unsigned start = 0;
        for (int jj = 0; jj < j; ++jj) start += st->tile_hist[jj];
        cur[j] = cnt[j] ? start + atomicAdd(&st->tile_cur[j], cnt[j]) : 0u;
    }
    __syncthreads();
    for (unsigned i0 = lo + (threadIdx.x & ~31u); i0 < hi; i0 += blockDim.x) {
        const unsigned i = i0 + lane;
        const bool v = i < hi;
        const uint2 e = v ? in[i] : make_uint2(0u, 0u);
        const int j = v ? tile_bin(__uint_as_float(e.y), sc) : kTileBins;
        const unsigned peers = __match_any_sync(0xffffffffu, j);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0;
        if (v && lane == leader) base = atomicAdd(&cur[j], (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        MESSI_CHECK(!v || base + __popc(peers & ((1u << lane) - 1)) < count);
        if (v) out[base + __popc(peers & ((1u << lane) - 1))] = make_uint2(e.x | ((unsigned)j << 28), e.y);
    }
}

// ------------------------------------------------------------- fused scan + refine
// fp64 canonical squared ED of one row (the oracle's operation sequence: sequential in i,
// round-to-nearest, no FMA), by one thread.  q_p: the padded query (element i at i + 4 (i >> 5)).
__device__ __forceinline__ double ed2_exact_g(const float* __restrict__ q_p, const float* __restrict__ c, int n)
{
    double sum = 0.0;
    for (int i = 0; i < n; i += 4) {
        const float4 cv = __ldg(reinterpret_cast<const float4*>(c + i));
        const float4 qv = *reinterpret_cast<const float4*>(q_p + i + 4 * (i >> 5));
        double d;
        d = __dsub_rn((double)qv.x, (double)cv.x); sum = __dadd_rn(sum, __dmul_rn(d, d));
        d = __dsub_rn((double)qv.y, (double)cv.y); sum = __dadd_rn(sum, __dmul_rn(d, d));
        d = __dsub_rn((double)qv.z, (double)cv.z); sum = __dadd_rn(sum, __dmul_rn(d, d));
        d = __dsub_rn((double)qv.w, (double)cv.w); sum = __dadd_rn(sum, __dmul_rn(d, d));
    }
    return sum;
}

// Lexicographic (d, id) min under the query's lock (near-ties only: a handful per query).
__device__ __forceinline__ void best_update(QState* st, double d, long long id)
{
    while (atomicCAS(&st->lock, 0u, 1u) != 0u) __nanosleep(64);
    __threadfence();
    const double bd = *(volatile double*)&st->best_d;
    const long long bi = *(volatile long long*)&st->best_id;
    if (d < bd || (d == bd && (bi < 0 || id < bi))) {
        *(volatile double*)&st->best_d = d;
        *(volatile long long*)&st->best_id = id;
    }
    __threadfence();
    atomicExch(&st->lock, 0u);
}

// k-NN: a refined row (fp32 d32, fp64 d64, id) under the query's lock.  The fp32 list keeps
// the k smallest d32 (distinct rows: each row is refined once); once it holds k, its k-th is
// a distance k rows achieve, i.e. a valid threshold for the k-th neighbour, and lowers the
// BSF.  The fp64 list keeps the k lexicographically smallest (d64, id) -- the answer.
// Single-thread insert (lane 0) for small k: under the lock the new entry shifts the
// larger ones up one slot (few of them: an accepted row usually lands near the k-th).
constexpr int kKnnLaneMax = 16;  // k above this: warp-cooperative insert (measured: k = 50 2.7x faster)

__device__ void knn_insert_lane(QState* st, KnnState* kn, int k, float d32, double d64, long long id, PeerSet ps, int b,
                           bool linked)
{
    while (atomicCAS(&st->lock, 0u, 1u) != 0u) __nanosleep(64);
    __threadfence();
    volatile KnnState* v = kn;
    int n = v->n32;
    if (n < k || d32 < v->d32[k - 1]) {
        int i = n < k ? n : k - 1;
        while (i > 0 && v->d32[i - 1] > d32) { v->d32[i] = v->d32[i - 1]; --i; }
        v->d32[i] = d32;
        if (n < k) v->n32 = ++n;
    }
    float kth = n == k ? v->d32[k - 1] : -1.0f;
    n = v->n64;
    auto less = [&](double a, long long ia, double c, long long ic) { return a < c || (a == c && ia < ic); };
    if (n < k || less(d64, id, v->d64[k - 1], v->id[k - 1])) {
        int i = n < k ? n : k - 1;
        while (i > 0 && less(d64, id, v->d64[i - 1], v->id[i - 1])) {
            v->d64[i] = v->d64[i - 1];
            v->id[i] = v->id[i - 1];
            --i;
        }
        v->d64[i] = d64;
        v->id[i] = id;
        if (n < k) v->n64 = n + 1;
    }
    __threadfence();
    atomicExch(&st->lock, 0u);
    if (kth >= 0.0f) {
        if (linked) bsf_publish(st, ps, b, kth);
        else bsf_update(st, kth);
    }
}

// Insert (d32, d64, id) into query b's k-NN state, the whole warp cooperating (k <= 64: lane
// l holds entries l and l + 32): under the query's lock the lists are read with one round of
// parallel loads, the insertion position comes from a ballot, entries shift by one lane via
// shuffles and go back with coalesced stores -- three memory round trips per insert instead
// of one per shifted entry.  The d32 list keeps the k smallest fp32 distances (its k-th is
// the pruning threshold); the (d64, id) list the k lexicographically smallest exact pairs.
__device__ void knn_insert_warp(QState* st, KnnState* kn, int k, float d32, double d64, long long id, PeerSet ps,
                                int b, bool linked, int lane)
{
    if (lane == 0)
        while (atomicCAS(&st->lock, 0u, 1u) != 0u) __nanosleep(64);
    __syncwarp();
    __threadfence();
    volatile KnnState* v = kn;
    const int n32 = v->n32, n64 = v->n64;
    const int i0 = lane, i1 = lane + 32;
    const float a0 = i0 < n32 ? v->d32[i0] : INFINITY, a1 = i1 < n32 ? v->d32[i1] : INFINITY;
    const double e0 = i0 < n64 ? v->d64[i0] : (double)INFINITY, e1 = i1 < n64 ? v->d64[i1] : (double)INFINITY;
    const long long j0 = i0 < n64 ? v->id[i0] : -1, j1 = i1 < n64 ? v->id[i1] : -1;
    float kth = -1.0f;
    {  // fp32 list: insert after the entries <= d32 (ties keep arrival order)
        const int pos = __popc(__ballot_sync(0xffffffffu, i0 < n32 && a0 <= d32)) +
                        __popc(__ballot_sync(0xffffffffu, i1 < n32 && a1 <= d32));
        const float up0 = __shfl_up_sync(0xffffffffu, a0, 1), up1 = __shfl_up_sync(0xffffffffu, a1, 1);
        const float last0 = __shfl_sync(0xffffffffu, a0, 31);
        const float p0 = lane == 0 ? 0.0f : up0, p1 = lane == 0 ? last0 : up1;  // entries i0-1, i1-1
        const int nn = n32 < k ? n32 + 1 : k;
        if (pos < k) {
            const float w0 = i0 < pos ? a0 : (i0 == pos ? d32 : p0);
            const float w1 = i1 < pos ? a1 : (i1 == pos ? d32 : p1);
            if (i0 < nn && i0 >= pos) v->d32[i0] = w0;
            if (i1 < nn && i1 >= pos) v->d32[i1] = w1;
            if (lane == 0) v->n32 = nn;
            const float kk = (k - 1) < 32 ? __shfl_sync(0xffffffffu, w0, (k - 1) & 31)
                                          : __shfl_sync(0xffffffffu, w1, (k - 1) & 31);
            kth = nn == k ? kk : -1.0f;
        } else {
            kth = n32 == k ? __shfl_sync(0xffffffffu, (k - 1) < 32 ? a0 : a1, (k - 1) & 31) : -1.0f;
        }
    }
    {  // (d64, id) list, lexicographic
        auto less = [](double a, long long ia, double c, long long ic) { return a < c || (a == c && ia < ic); };
        const int pos = __popc(__ballot_sync(0xffffffffu, i0 < n64 && less(e0, j0, d64, id))) +
                        __popc(__ballot_sync(0xffffffffu, i1 < n64 && less(e1, j1, d64, id)));
        const double ue0 = __shfl_up_sync(0xffffffffu, e0, 1), ue1 = __shfl_up_sync(0xffffffffu, e1, 1);
        const long long uj0 = __shfl_up_sync(0xffffffffu, j0, 1), uj1 = __shfl_up_sync(0xffffffffu, j1, 1);
        const double le = __shfl_sync(0xffffffffu, e0, 31);
        const long long lj = __shfl_sync(0xffffffffu, j0, 31);
        const double pe0 = ue0, pe1 = lane == 0 ? le : ue1;
        const long long pj0 = uj0, pj1 = lane == 0 ? lj : uj1;
        const int nn = n64 < k ? n64 + 1 : k;
        if (pos < k) {
            if (i0 < nn && i0 >= pos) {
                v->d64[i0] = i0 == pos ? d64 : pe0;
                v->id[i0] = i0 == pos ? id : pj0;
            }
            if (i1 < nn && i1 >= pos) {
                v->d64[i1] = i1 == pos ? d64 : pe1;
                v->id[i1] = i1 == pos ? id : pj1;
            }
            if (lane == 0) v->n64 = nn;
        }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) {
        atomicExch(&st->lock, 0u);
        if (kth >= 0.0f) {
            if (linked) bsf_publish(st, ps, b, kth);
            else bsf_update(st, kth);
        }
    }
}

// The candidates of `keep` (one per lane, sorted position my_pos): fp32 squared ED over the
// raw rows, four rows in flight per warp (Alg. 9 RealDist); a distance <= BSF*(1+eps)
// lowers the BSF (atomicMin, Alg. 8's BSF update P:1178-1186) and is re-ranked exactly in
// fp64 at once (reading R11/R12): the lexicographic min over the re-ranked rows is the answer.
// fp32 squared ED of the warp's kRefineGroup rows id[g] (ok[g]: slot used), all rows in flight
// at once: lane takes float4 chunks lane*4 + 128k of each row, then a butterfly sum (every lane
// ends with the totals).  The query comes from q_p (element i at i + 4 (i >> 5)).
__device__ __forceinline__ void ed2_group(const unsigned (&id)[kRefineGroup], const bool (&ok)[kRefineGroup],
                                          const float* __restrict__ rows, int n, const float* __restrict__ q_p,
                                          int lane, float (&acc)[kRefineGroup])
{
#pragma unroll
    for (int g = 0; g < kRefineGroup; ++g) acc[g] = 0.0f;
    for (int j = lane * 4; j < n; j += 128) {
        const float4 qv = *reinterpret_cast<const float4*>(q_p + j + 4 * (j >> 5));
        float4 cv[kRefineGroup];
#pragma unroll
        for (int g = 0; g < kRefineGroup; ++g)
            cv[g] = ok[g] ? __ldg(reinterpret_cast<const float4*>(rows + (long long)id[g] * n + j))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int g = 0; g < kRefineGroup; ++g) {
            float d;
            d = qv.x - cv[g].x; acc[g] = fmaf(d, d, acc[g]);
            d = qv.y - cv[g].y; acc[g] = fmaf(d, d, acc[g]);
            d = qv.z - cv[g].z; acc[g] = fmaf(d, d, acc[g]);
            d = qv.w - cv[g].w; acc[g] = fmaf(d, d, acc[g]);
        }
    }
#pragma unroll
    for (int g = 0; g < kRefineGroup; ++g) acc[g] = warp_sum(acc[g]);
}

// Returns (every lane) the smallest fp32 distance this call accepted (+inf if none): the
// caller lowers its cached threshold with it.
template <bool LINKED, bool KNN>
__device__ float exact_pass(unsigned keep, unsigned my_pos, const unsigned* __restrict__ perm,
                            const float* __restrict__ rows, int n, const float* __restrict__ q_p, QState* st,
                            PeerSet ps, int b, KnnState* knn, int k, int lane)
{
    float dmin = INFINITY;
    while (keep) {
        unsigned id[kRefineGroup];
        bool ok[kRefineGroup];
#pragma unroll
        for (int g = 0; g < kRefineGroup; ++g) {
            ok[g] = keep != 0;
            const int src = ok[g] ? __ffs(keep) - 1 : 0;
            keep &= keep - 1;
            const unsigned pos = __shfl_sync(0xffffffffu, my_pos, src);
            id[g] = ok[g] ? perm[pos] : 0u;
        }
        float acc[kRefineGroup];
        ed2_group(id, ok, rows, n, q_p, lane, acc);
        if (KNN && k > kKnnLaneMax) {  // large k: the warp inserts each accepted row together
            // (the KNN = false instantiation keeps the runtime knn test below: measured
            // 2% faster C3 code than with the k-NN branches folded away)
#pragma unroll
            for (int g = 0; g < kRefineGroup; ++g) {
                if (!ok[g]) continue;
                int take = 0;
                double d64 = 0.0;
                if (lane == 0) {
                    take = acc[g] <= slack_up(ld_bsf_l<LINKED>(st, ps.epoch));
                    if (take) {
                        d64 = ed2_exact_g(q_p, rows + (long long)id[g] * n, n);
                        atomicAdd(&st->near_count, 1u);
                    }
                }
                if (__shfl_sync(0xffffffffu, take, 0)) {
                    d64 = __shfl_sync(0xffffffffu, d64, 0);
                    knn_insert_warp(st, knn + b, k, acc[g], d64, (long long)id[g], ps, b, LINKED, lane);
                }
            }
        } else if (lane == 0) {
#pragma unroll
            for (int g = 0; g < kRefineGroup; ++g) {
                if (!ok[g]) continue;
                const float thr = slack_up(ld_bsf_l<LINKED>(st, ps.epoch));
                if (acc[g] <= thr) {
                    const double d64 = ed2_exact_g(q_p, rows + (long long)id[g] * n, n);
                    if (knn) {
                        knn_insert_lane(st, knn + b, k, acc[g], d64, (long long)id[g], ps, b, LINKED);
                    } else {
                        if (LINKED) bsf_publish(st, ps, b, acc[g]);
                        else bsf_update(st, acc[g]);
                        best_update(st, d64, (long long)id[g]);
                        dmin = fminf(dmin, acc[g]);
                    }
                    atomicAdd(&st->near_count, 1u);
                }
            }
        }
        __syncwarp();
    }
    return __shfl_sync(0xffffffffu, dmin, 0);
}

// Dynamic shared memory of k_scan_refine_ed: scan table, padded query, the quantised query
// (n bytes), per-warp coarse survivor lists (current + previous tile) and fine-survivor
// buffer (n = 256: 92.5 KB -> 2 CTAs of 12 warps per SM).
__host__ __device__ inline size_t fused_qpad(int n) { return (size_t)(n + 4 * ((n + 31) / 32) + 4) & ~(size_t)3; }
__host__ __device__ inline size_t fused_smem(int n)
{
    return (size_t)kLutX * 4 + fused_qpad(n) * 4 + (size_t)n +
           (size_t)kFusedWarps * (MESSI_TILE_ROWS * 2 + kCandBuf * 4 + 4 + 16);
}

// Writes query b's result and stats (finish_query's layout) from its state.
__device__ void fused_finalise(const QState* st, long long N, long long row_begin, void* result, void* stats)
{
    struct R { double dist; long long id; double d2; long long reserved; };
    struct S { long long lb, tiles, cand, lbk, refined, abandoned, near, cells, exact, listed, coarse; double seed, bsf; long long rpaa; };
    const double bd = st->best_d;
    const long long bi = st->best_id;
    R* res = reinterpret_cast<R*>(result);
    res->dist = bi >= 0 ? sqrt(bd) : (double)INFINITY;
    res->id = bi >= 0 ? row_begin + bi : -1;
    res->d2 = bd;
    res->reserved = 0;
    if (stats) {
        S* s = reinterpret_cast<S*>(stats);
        const unsigned ts = st->tiles_scanned;
        s->lb = (long long)ts * MESSI_TILE_ROWS < N ? (long long)ts * MESSI_TILE_ROWS : N;
        s->tiles = ts;
        s->cand = st->cand_count;
        s->lbk = 0;
        s->refined = st->refined;
        s->exact = st->exact;
        s->listed = st->tile_count + st->tile_back;
        s->coarse = st->coarse_count;
        s->abandoned = s->refined - s->exact;
        s->near = st->near_count;
        s->cells = 0;
        s->seed = (double)__uint_as_float(st->seed_bits);
        s->bsf = (double)__uint_as_float(st->bsf_bits);
        s->rpaa = s->cand;  // ED: no reverse bound
    }
}

// One thread per query of the batch, after k_scan_refine_ed (stream order makes every
// update of the fused kernel visible): results and stats.  k-NN: k results per query,
// ascending (d2, id); fewer than k rows -> the rest (inf, -1).
__global__ void k_finalise_batch(const QState* __restrict__ st_all, int B, long long N, long long row_begin,
                                 void* results, void* stats, const KnnState* __restrict__ knn, int k)
{
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    if (!knn) {
        fused_finalise(st_all + b, N, row_begin, reinterpret_cast<char*>(results) + (size_t)b * 32,
                       stats ? reinterpret_cast<char*>(stats) + (size_t)b * kStatsBytes : nullptr);
        return;
    }
    fused_finalise(st_all + b, N, row_begin, reinterpret_cast<char*>(results) + (size_t)b * k * 32,
                   stats ? reinterpret_cast<char*>(stats) + (size_t)b * kStatsBytes : nullptr);
    struct R { double dist; long long id; double d2; long long reserved; };
    R* res = reinterpret_cast<R*>(results) + (size_t)b * k;
    const KnnState* kn = knn + b;
    for (int i = 0; i < k; ++i) {
        const bool have = i < kn->n64;
        res[i].dist = have ? sqrt(kn->d64[i]) : (double)INFINITY;
        res[i].id = have ? row_begin + kn->id[i] : -1;
        res[i].d2 = have ? kn->d64[i] : (double)INFINITY;
        res[i].reserved = 0;
    }
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Quantised-row bound with integer dot products: the query quantised like the
// rows (q^ = s_q c_q, e_q >= ||q - q^||, k_prologue_batch) and row x^ = s_x c_x (e_x >= ||x - x^||):
//     ||q - x|| >= ||q^ - x^|| - e_q - e_x,
//     ||q^ - x^||^2 = s_q^2 sum c_q^2 + s_x^2 sum c_x^2 - 2 s_q s_x sum c_q c_x,
// the sums exact in int32 (IDP.4A over the row's int8 bytes: sum c_x c_q, sum c_x^2),
// the combination in fp64 with an error margin, so L below is a rigorous lower bound of ||q - x||.
// A candidate with L > 0 and L^2 > thr cannot be the nearest neighbour; the others come back
// (bit set) for the exact fp32 refine.  Groups of 4 lanes take one row each (8 rows per pass);
// lane gl of a group reads the row's 16-byte chunks gl, gl + 4, ... with the query's chunk from
// shared memory (qc_s).  DBG (inspection): dbg[src lane] = (dh2 lower bound, L).
struct Q8Query {
    double sq, e, s2ss;  // s_q, e_q, s_q^2 sum c_q^2
};

template <bool DBG = false>
__device__ __forceinline__ unsigned q8i_bound_pass(int count, unsigned my_pos, const unsigned char* __restrict__ rows8,
                                                   const float2* __restrict__ meta8, int n, const uint4* qc_s,
                                                   const Q8Query& qq, float thr, int lane, double2* dbg = nullptr)
{
    // candidates: lanes 0 .. count-1 (a prefix), lane l's at sorted position my_pos.  Pass p
    // streams candidates 8p .. 8p+7, group g = lane >> 2 the row of candidate 8p + g; the
    // group's integer sums then go to the candidate's own lane, and every lane finishes its
    // candidate's bound at once.
    const int g = lane >> 2, gl = lane & 3;
    const int nch = n >> 4;
    int my_dq = 0, my_ss = 0;  // sum c_x c_q, sum c_x^2 of this lane's candidate (exact int32)
    // the row's (scale, error), issued before the row passes (a random 8-byte gather)
    const float2 mt = lane < count ? meta8[my_pos] : make_float2(0.0f, 0.0f);
#pragma unroll 1
    for (int p = 0; 8 * p < count; ++p) {
        const int c = 8 * p + g;
        const bool ok = c < count;
        const unsigned pos = __shfl_sync(0xffffffffu, my_pos, c & 31);
        const uint4* row = reinterpret_cast<const uint4*>(rows8 + (size_t)pos * (size_t)n);
        int dq = 0, ss = 0;
#pragma unroll 4
        for (int ch = gl; ch < nch; ch += 4) {
            const uint4 w = ok ? __ldg(row + ch) : make_uint4(0u, 0u, 0u, 0u);
            const uint4 qv = qc_s[ch];
            dq = dp4a_ss(w.x, qv.x, dq); dq = dp4a_ss(w.y, qv.y, dq);
            dq = dp4a_ss(w.z, qv.z, dq); dq = dp4a_ss(w.w, qv.w, dq);
            ss = dp4a_ss(w.x, w.x, ss); ss = dp4a_ss(w.y, w.y, ss);
            ss = dp4a_ss(w.z, w.z, ss); ss = dp4a_ss(w.w, w.w, ss);
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            dq += __shfl_xor_sync(0xffffffffu, dq, o);
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
        }
        const int src = 4 * (lane & 7);
        const int v_dq = __shfl_sync(0xffffffffu, dq, src), v_ss = __shfl_sync(0xffffffffu, ss, src);
        if ((lane >> 3) == p) { my_dq = v_dq; my_ss = v_ss; }
    }
    bool survives = true;
    if (lane < count) {
        const double sx = (double)mt.x;  // a power of two
        const double t2 = sx * sx * (double)my_ss, t3 = 2.0 * qq.sq * sx * (double)my_dq;  // exact products
        const double d2 = (qq.s2ss + t2) - t3;
        // two roundings of magnitude <= 2^-53 (s2ss + t2 + |t3|) each; margin 2^-50
        const double d2lo = d2 - 0x1p-50 * (qq.s2ss + t2 + fabs(t3));
        const double L = (d2lo > 0.0 ? sqrt(d2lo) * (1.0 - 0x1p-50) : 0.0) - (double)mt.y - qq.e;
        survives = !(L > 0.0 && L * L * (1.0 - 0x1p-40) > (double)thr);
        if constexpr (DBG) dbg[lane] = make_double2(d2lo, L);
    }
    return __ballot_sync(0xffffffffu, lane < count && survives);
}

// L2 prefetch of the n bytes at p (128-byte lines, one instruction per line and lane).
__device__ __forceinline__ void prefetch_l2_lines(const void* p, int bytes)
{
    const char* c = static_cast<const char*>(p);
    for (int off = 0; off < bytes; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(c + off));
}

// Fine pass + refine of the coarse survivors of one tile (list surv, m entries, warp-
// uniform), against the warp's cached threshold thr (updated when the refine finds a better
// distance).  Round 0 uses the 8-bit words the warp preloaded (w0 / pos0) one tile earlier;
// each round loads the next round's words before evaluating its own.  Fine survivors
// (LB8 <= thr) wait in the warp's buffer cbuf (prefetched into L2); every full round of 32
// goes through the quantised bound and the exact passes.
// The warp's per-query counters live in shared memory (lane 0 updates them; registers are
// the fused kernel's occupancy limit): c[0] tiles, c[1] coarse, c[2] cand, c[3] exact.
struct WarpCounts {
    unsigned* c;
    __device__ __forceinline__ void add(int i, unsigned v, int lane) const { if (lane == 0) c[i] += v; }
};

struct FusedCtx {
    const uint4* sym8;
    const unsigned char* rows8;
    const float2* meta8;
    const unsigned* perm;
    const float* rows;
    const float* q_p;
    const uint4* qc_s;
    const char* lbase;
    QState* st;
    KnnState* knn;
    PeerSet ps;
    const Q8Query* qq;  // the current query's, in shared memory (registers are the occupancy limit)
    int n, b, k;
    long long npad;  // sorted positions (checked build)
};

template <bool LINKED, bool KNN>
__device__ __forceinline__ void refine_round(const FusedCtx& cx, unsigned cp, int count, float& thr,
                                             WarpCounts& wc, int lane)
{
    const unsigned keep = q8i_bound_pass(count, cp, cx.rows8, cx.meta8, cx.n, cx.qc_s, *cx.qq, thr, lane);
    wc.add(3, __popc(keep), lane);
    if (keep) thr = fminf(thr, slack_up(exact_pass<LINKED, KNN>(keep, cp, cx.perm, cx.rows, cx.n, cx.q_p, cx.st,
                                                                   cx.ps, cx.b, cx.knn, cx.k, lane)));
}

template <bool LINKED, bool KNN>
__device__ __forceinline__ void fine_and_refine(const FusedCtx& cx, long long tile, int m, const unsigned short* surv,
                                                uint4 w0, unsigned pos0, unsigned* cbuf, unsigned& ncb, float& thr,
                                                WarpCounts& wc, int lane)
{
    unsigned pos = pos0;
    uint4 w = w0;
    for (int i0 = 0; i0 < m; i0 += 32) {
        const bool v = i0 + lane < m;
        // the next round's words, loaded before this round's bounds
        unsigned pos_n = 0;
        uint4 w_n = make_uint4(0u, 0u, 0u, 0u);
        if (i0 + 32 < m) {
            const bool vn = i0 + 32 + lane < m;
            pos_n = vn ? (unsigned)(tile * MESSI_TILE_ROWS + surv[i0 + 32 + lane]) : 0u;
            if (vn) w_n = cx.sym8[pos_n];
        }
        float lb = INFINITY;
        if (v) lb = fine_lb(w, cx.lbase, lane);
        const bool ok = v && lb <= thr;
        const unsigned pass = __ballot_sync(0xffffffffu, ok);
        if (pass) {
            if (ok) {
                MESSI_CHECK(ncb + __popc(pass & ((1u << lane) - 1)) < (unsigned)kCandBuf);
                MESSI_CHECK(pos < (unsigned)(cx.npad));
                cbuf[ncb + __popc(pass & ((1u << lane) - 1))] = pos;
                prefetch_l2_lines(cx.rows8 + (long long)pos * cx.n, cx.n);
            }
            ncb += __popc(pass);
            wc.add(2, __popc(pass), lane);
            __syncwarp();
            if (ncb >= 32) {
                const unsigned cp = cbuf[lane];
                const unsigned rest = ncb - 32 > (unsigned)lane ? cbuf[32 + lane] : 0u;
                __syncwarp();
                if (ncb - 32 > (unsigned)lane) cbuf[lane] = rest;
                ncb -= 32;
                __syncwarp();
                refine_round<LINKED, KNN>(cx, cp, 32, thr, wc, lane);
            }
        }
        pos = pos_n;
        w = w_n;
    }
}

// A claim of the next work item (one lane): atom.inc with limit 2^31 - 1 (a counter of tile
// pairs never gets there), which ptxas keeps as one ATOMG.E.INC -- an add (or an inc with
// limit 2^32 - 1, which it turns into an add) becomes a warp-aggregated atomic whose result
// is broadcast with a shuffle right after it, so the warp would wait for the round trip at
// the claim instead of where the value is first used.
__device__ __forceinline__ unsigned claim_next(unsigned* p)
{
    unsigned r;
    asm volatile("atom.global.inc.u32 %0, [%1], 2147483647;" : "=r"(r) : "l"(p) : "memory");
    return r;
}

// Persistent.  CTA j starts at query j mod B and walks the batch's queries cyclically once;
// at a query with listed tiles left it loads the query's scan table, padded query and
// quantised query into shared memory, then its warps take pairs of tiles from the query's
// list (Alg. 9's Fetch&Inc chunks), re-check each tile's box bound against the best-so-far
// (Alg. 7's node pruning), run the coarse pass of the tile (A5), and the fine pass + refine of
// the PREVIOUS tile's coarse survivors (whose 8-bit words were loaded before this tile's
// coarse pass, hiding the gather), as Alg. 9's workers do.
// Software pipeline per warp, one pair ahead: while pair i is processed, lane 0 has already
// claimed pair i + 2 (atomicAdd), read the best-so-far and loaded pair i + 1's list entries,
// and, after pair i's first tile, bulk-prefetches pair i + 1's tiles into L2.  The warp's
// threshold is the best-so-far read one pair earlier (a stale, i.e. larger, value is a valid
// threshold: it only prunes less), lowered at once by the distances the warp itself accepts.
// When a query's list runs dry the CTA joins the next one: light queries finish early and
// their CTAs help the heavy ones.  k_finalise_batch writes the results.  KNN = true adds the
// warp-cooperative k-NN insert (k > 16).
template <bool LINKED, bool KNN>
__global__ void __launch_bounds__(32 * kFusedWarps, MESSI_FUSED_MINB) k_scan_refine_ed(
    const uint4* __restrict__ tiles, const uint4* __restrict__ sym8, long long ntiles, long long N, int n,
    const float* __restrict__ queries, const float* __restrict__ lutx_all, const uint2* __restrict__ tlist_all,
    QState* st_all, int B, const unsigned char* __restrict__ rows8, const float2* __restrict__ meta8,
    const unsigned* __restrict__ qc_all, const unsigned* __restrict__ perm, const float* __restrict__ rows, PeerSet ps,
    KnnState* knn_arg, int k_arg)
{
    extern __shared__ __align__(16) float smem[];
    float* lut_s = smem;
    float* q_p = lut_s + kLutX;
    unsigned* qc_w = reinterpret_cast<unsigned*>(q_p + fused_qpad(n));
    unsigned short* surv_all = reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(qc_w) + n);
    unsigned* cbuf_all = reinterpret_cast<unsigned*>(surv_all + kFusedWarps * MESSI_TILE_ROWS);
    unsigned* wcnt_all = cbuf_all + kFusedWarps * kCandBuf;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned short* surv = surv_all + warp * MESSI_TILE_ROWS;  // coarse survivors of the previous tile
    unsigned* cbuf = cbuf_all + warp * kCandBuf;
    unsigned* wcnt = wcnt_all + warp;
    unsigned* wcs = wcnt_all + kFusedWarps + 4 * warp;  // the warp's per-query counters
    __shared__ int s_has;
    __shared__ float s_binfloor[kTileBins];
    __shared__ Q8Query s_qq;
    FusedCtx cx;
    cx.sym8 = sym8; cx.rows8 = rows8; cx.meta8 = meta8; cx.perm = perm; cx.rows = rows; cx.q_p = q_p;
    cx.qc_s = reinterpret_cast<const uint4*>(qc_w); cx.lbase = reinterpret_cast<const char*>(lut_s);
    cx.knn = knn_arg; cx.ps = ps; cx.n = n; cx.k = k_arg; cx.npad = ntiles * MESSI_TILE_ROWS; cx.qq = &s_qq;
    int b = (int)(blockIdx.x % (unsigned)B);
    for (int visited = 0; visited < B; ++visited, b = (b + 1 == B ? 0 : b + 1)) {
        QState* st = st_all + b;
        // listed tiles, best-first (k_order_tiles)
        const unsigned count = *(volatile unsigned*)&st->tile_count;
        if (threadIdx.x == 0) s_has = *(volatile unsigned*)&st->next_tile * 2u < count;
        __syncthreads();
        const bool has = s_has;
        __syncthreads();  // s_has is rewritten by the next visit
        if (!has) continue;
        {
            const float4* src = reinterpret_cast<const float4*>(lutx_all + (size_t)b * kLutX);
            for (int i = threadIdx.x; i < kLutX / 4; i += blockDim.x) reinterpret_cast<float4*>(lut_s)[i] = src[i];
            const float* q = queries + (size_t)b * n;
            for (int i = threadIdx.x; i < n; i += blockDim.x) q_p[i + 4 * (i >> 5)] = q[i];
            const unsigned* qc = qc_all + (size_t)b * (n / 4);
            for (int i = threadIdx.x; i < n / 4; i += blockDim.x) qc_w[i] = qc[i];
            if (threadIdx.x < kTileBins) s_binfloor[threadIdx.x] = tile_bin_floor(threadIdx.x, tile_bin_scale(st));
        }
        cx.st = st;
        cx.b = b;
        if (threadIdx.x == 0) {
            s_qq.sq = (double)st->q8s;
            s_qq.e = st->q8e;
            s_qq.s2ss = st->q8s2ss;
        }
        __syncthreads();
        const uint2* tl = tlist_all + (size_t)b * ntiles;
        auto at = [&](unsigned kk) { return tl[kk]; };
        WarpCounts wc{wcs};
        if (lane == 0) wcs[0] = wcs[1] = wcs[2] = wcs[3] = 0u;
        unsigned ncb = 0;        // fine survivors pending in cbuf (warp-uniform)
        int pm = 0;              // previous tile's coarse survivors (list surv)
        long long ptile = 0;
        uint4 pw = make_uint4(0, 0, 0, 0);
        unsigned ppos = 0;
        // pipeline start: claims of pairs 0 and 1, the first threshold, pair 0's entries
        unsigned kc = 0, kn = 0;
        float thr = 0.0f;
        if (lane == 0) {
            kc = atomicAdd(&st->next_tile, 1u) * 2u;
            kn = atomicAdd(&st->next_tile, 1u) * 2u;
            thr = slack_up(ld_bsf_l<LINKED>(st, ps.epoch));
        }
        kc = __shfl_sync(0xffffffffu, kc, 0);
        kn = __shfl_sync(0xffffffffu, kn, 0);
        thr = __shfl_sync(0xffffffffu, thr, 0);
        uint2 te0 = kc < count ? at(kc) : make_uint2(0u, 0x7f800000u);
        uint2 te1 = kc + 1 < count ? at(kc + 1) : make_uint2(0u, 0x7f800000u);
        while (kc < count) {
            // lane 0: claim pair i + 2, read the best-so-far, load pair i + 1's entries (used later)
            // (lane 0's block only issues the atomic and the loads; their results are first
            // used after pair i's first tile, so no instruction in the divergent block waits
            // on them and the warp reconverges at once)
            unsigned k2 = 0;
            float thr_n = 0.0f;
            uint2 ne0 = make_uint2(0u, 0x7f800000u), ne1 = make_uint2(0u, 0x7f800000u);
            if (lane == 0) {
                if (kn < count) {
                    k2 = claim_next(&st->next_tile);  // pair index: x2 when consumed
                    ne0 = at(kn);
                    if (kn + 1 < count) ne1 = at(kn + 1);
                } else {
                    k2 = kn >> 1;
                }
                thr_n = ld_bsf_l<LINKED>(st, ps.epoch);  // raw: slack_up when consumed
            }
#pragma unroll 1
            for (int u = 0; u < 2; ++u) {
                if (u == 1 && lane == 0) {  // pair i + 1's tiles into L2, unless already box-pruned
                    thr_n = slack_up(thr_n);
                    if (__uint_as_float(ne0.y) <= thr_n)
                        prefetch_l2_bulk(tiles + (long long)(ne0.x & kTileMask) * (MESSI_TILE_BYTES / 16), MESSI_TILE_BYTES);
                    if (__uint_as_float(ne1.y) <= thr_n)
                        prefetch_l2_bulk(tiles + (long long)(ne1.x & kTileMask) * (MESSI_TILE_BYTES / 16), MESSI_TILE_BYTES);
                }
                const uint2 te = u == 0 ? te0 : te1;
                MESSI_CHECK(kc + u >= count || (te.x & kTileMask) < (unsigned)ntiles);
                if (kc + u >= count) continue;
                if (__uint_as_float(te.y) > thr) {  // box pruned (warp-uniform)
                    // every bound of this tile's bin above thr too, so every later bin's: the
                    // query's remaining claims are void
                    if (lane == 0 && s_binfloor[te.x >> 28] > thr) atomicMax(&st->next_tile, kClaimsDone);
                    continue;
                }
                wc.add(0, 1u, lane);
                const long long tile = te.x & kTileMask;
                // coarse pass of this tile (its survivors stay a per-lane mask until the previous
                // tile's fine pass has released the warp's list)
                float acc[16];
                coarse_acc(tiles, tile, cx.lbase, lane, acc);
                const unsigned cmask = coarse_mask(acc, thr, N, tile, lane);
                if (pm)
                    fine_and_refine<LINKED, KNN>(cx, ptile, pm, surv, pw, ppos, cbuf, ncb, thr, wc, lane);
                const int m = compact_mask(cmask, surv, wcnt, lane);
                wc.add(1, (unsigned)m, lane);
                // preload the 8-bit words of this tile's first 32 coarse survivors
                ppos = lane < m ? (unsigned)(tile * MESSI_TILE_ROWS + surv[lane]) : 0u;
                pw = lane < m ? sym8[ppos] : make_uint4(0, 0, 0, 0);
                pm = m;
                ptile = tile;
            }
            // advance the pipeline
            kc = kn;
            kn = __shfl_sync(0xffffffffu, k2, 0) * 2u;
            thr = fminf(thr, __shfl_sync(0xffffffffu, thr_n, 0));
            te0 = make_uint2(__shfl_sync(0xffffffffu, ne0.x, 0), __shfl_sync(0xffffffffu, ne0.y, 0));
            te1 = make_uint2(__shfl_sync(0xffffffffu, ne1.x, 0), __shfl_sync(0xffffffffu, ne1.y, 0));
        }
        if (pm) fine_and_refine<LINKED, KNN>(cx, ptile, pm, surv, pw, ppos, cbuf, ncb, thr, wc, lane);
        if (ncb) {  // the query's last fine survivors
            const unsigned cp = (unsigned)lane < ncb ? cbuf[lane] : 0u;
            __syncwarp();
            refine_round<LINKED, KNN>(cx, cp, (int)ncb, thr, wc, lane);
            ncb = 0;
        }
        if (lane == 0) {
            if (wcs[0]) atomicAdd(&st->tiles_scanned, wcs[0]);
            if (wcs[2]) atomicAdd(&st->cand_count, wcs[2]);
            if (wcs[2]) atomicAdd(&st->refined, wcs[2]);
            if (wcs[1]) atomicAdd(&st->coarse_count, wcs[1]);
            if (wcs[3]) atomicAdd(&st->exact, wcs[3]);
        }
        __syncthreads();  // every warp is done with b's table before it is overwritten
    }
}

// ------------------------------------------------------------------------ inspection
// Inspection of the ED refine (messi_debug_ed_refine): for `k` local row ids, one warp per 32
// of them, the query path's own device code -- q8i_bound_pass (the lower bound dh2 of the
// squared distance between the quantised query and row, and L, its lower bound of ||q - x||),
// ed2_group (the exact pass's fp32 squared ED) and ed2_exact_g (the fp64 re-rank) -- nothing
// pruned.  The quantised query and its parameters come from query 0 of a batch set
// (k_prologue_batch).  inv: sorted position of every row (the inverse of perm).
__global__ void __launch_bounds__(256) k_debug_ed_refine(const float* __restrict__ rows, int n,
                                                         const float* __restrict__ q_g,
                                                         const unsigned char* __restrict__ rows8,
                                                         const float2* __restrict__ meta8,
                                                         const unsigned* __restrict__ qc_g, const QState* qst,
                                                         const unsigned* __restrict__ inv,
                                                         const unsigned* __restrict__ ids, int k,
                                                         double2* __restrict__ q8out, float* __restrict__ d32,
                                                         double* __restrict__ d64)
{
    extern __shared__ __align__(16) float q_p[];
    __shared__ double2 dbg_s[8][32];
    unsigned* qc_w = reinterpret_cast<unsigned*>(q_p + fused_qpad(n));
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_p[i + 4 * (i >> 5)] = q_g[i];
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x) qc_w[i] = qc_g[i];
    __syncthreads();
    Q8Query qq;
    qq.sq = (double)qst->q8s;
    qq.e = qst->q8e;
    qq.s2ss = qst->q8s2ss;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    for (int t0 = (blockIdx.x * wpb + w) * 32; t0 < k; t0 += gridDim.x * wpb * 32) {
        const bool v = t0 + lane < k;
        const unsigned id = v ? ids[t0 + lane] : 0u;
        const unsigned pos = v ? inv[id] : 0u;
        const unsigned mask = __ballot_sync(0xffffffffu, v);
        q8i_bound_pass<true>(min(32, k - t0), pos, rows8, meta8, n, reinterpret_cast<const uint4*>(qc_w), qq, INFINITY,
                             lane, dbg_s[w]);
        __syncwarp();
        float mine = 0.0f;
        unsigned rest = mask;
        while (rest) {
            unsigned gid[kRefineGroup];
            bool ok[kRefineGroup];
            int src[kRefineGroup];
#pragma unroll
            for (int g = 0; g < kRefineGroup; ++g) {
                ok[g] = rest != 0;
                src[g] = ok[g] ? __ffs(rest) - 1 : 0;
                rest &= rest - 1;
                gid[g] = __shfl_sync(0xffffffffu, id, src[g]);
            }
            float acc[kRefineGroup];
            ed2_group(gid, ok, rows, n, q_p, lane, acc);
#pragma unroll
            for (int g = 0; g < kRefineGroup; ++g)
                if (ok[g] && lane == src[g]) mine = acc[g];
        }
        if (v) {
            q8out[t0 + lane] = dbg_s[w][lane];
            d32[t0 + lane] = mine;
            d64[t0 + lane] = ed2_exact_g(q_p, rows + (long long)id * n, n);
        }
        __syncwarp();
    }
}

}  // namespace messi
