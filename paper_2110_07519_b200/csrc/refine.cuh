// refine.cuh -- refinement of the scan's candidates (A7 ED, A8 DTW) and the exact
// resolution of near-ties (A9).
#pragma once
#include "common.cuh"
#include "dtw.cuh"

namespace messi {

__device__ __forceinline__ void append_near(QState* st, NearEntry* near, unsigned id, float d)
{
    unsigned pos = atomicAdd(&st->near_count, 1u);
    near[pos] = NearEntry{id, d};
}

// Valid band cells of the first J rows of an n x n DTW matrix with reach R (|i - j| <= R,
// 0 <= i, j < n): sum_{j < J} (min(n - 1, j + R) - max(0, j - R) + 1); J = n gives
// n(2R + 1) - R(R + 1) (SURVEY 8(d)'s cell count).  The refine kernels report the cells of
// the rows they evaluated (an abandoned candidate counts the rows done).
__device__ __forceinline__ unsigned long long band_cells(long long n, long long R, long long J)
{
    if (J <= 0) return 0ull;
    if (J > n) J = n;
    if (R > n - 1) R = n - 1;
    const long long J1 = J < n - R ? J : n - R;  // rows whose band end j + R stays inside
    const long long A = J1 * (J1 - 1) / 2 + J1 * (R + 1) + (J - J1) * n;
    const long long K = J - R - 1 > 0 ? J - R - 1 : 0;  // rows whose band start j - R > 0
    return (unsigned long long)(A - K * (K + 1) / 2);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v)
{
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Rows in flight per warp in the fp32 distance loops (four 1 KB rows at n = 256).
constexpr int kRefineGroup = 4;

struct Best { double d; long long id; };

// DTW k-NN (the paper's k-NN: the BSF becomes the k-th best distance): a refined
// candidate's fp32 distance into the query's list of the k smallest fp32 distances so far,
// under the query's lock (one thread; completions within the threshold are rare).  Once the
// list holds k distances its k-th is a distance k distinct rows achieve -- a valid threshold
// for the k-th neighbour -- and lowers the BSF.
__device__ __noinline__ void knn32_insert(QState* st, KnnState* kn, int k, float d, PeerSet ps, int slot)
{
    while (atomicCAS(&st->lock, 0u, 1u) != 0u) __nanosleep(32);
    __threadfence();
    volatile KnnState* v = kn;
    int cnt = v->n32;
    if (cnt < k || d < v->d32[k - 1]) {
        int i = cnt < k ? cnt : k - 1;
        while (i > 0 && v->d32[i - 1] > d) { v->d32[i] = v->d32[i - 1]; --i; }
        v->d32[i] = d;
        if (cnt < k) v->n32 = ++cnt;
    }
    const float kth = cnt == k ? v->d32[k - 1] : -1.0f;
    __threadfence();
    atomicExch(&st->lock, 0u);
    if (kth >= 0.0f) bsf_publish(st, ps, slot, kth);
}

// The refine's acceptance of a completed candidate at fp32 distance d <= thr: the near-best
// list, and (unless inspecting, frozen) the BSF -- 1-NN: d itself (the thread's own threshold
// drops with it); k-NN: the k-th of the list.
__device__ __forceinline__ void dtw_accept(QState* st, NearEntry* near, KnnState* knn, int kk, bool frozen,
                                           unsigned id, float d, float& thr, PeerSet ps, int slot)
{
    append_near(st, near, id, d);
    if (frozen) return;
    if (knn) {
        knn32_insert(st, knn, kk, d, ps, slot);
    } else {
        bsf_publish(st, ps, slot, d);
        thr = fminf(thr, slack_up(d));
    }
}

// DTW step 1 (Alg. 10 line LB_Keogh): the scan's candidates (sorted position,
// envelope-PAA bound) whose bound still does not exceed the BSF get the raw LB_Keogh
// against the query envelope, four rows in flight per warp; survivors go to list2 as
// (row id, LBK, LBK of columns 0 .. reach+3 -- the columns the DP's first window holds).
// Best-first in two bins (the priority-queue order of MESSI, coarsened):
// survivors with LBK <= front * BSF0 are appended at the front of list2, the others from
// its back end (capacity cap), so the refine -- which hands entries out in list order --
// starts the candidates most likely to be near (and to run longest) first.
__device__ __forceinline__ uint4 list2_at(const uint4* __restrict__ list2, unsigned k, unsigned nfront, unsigned cap)
{
    return k < nfront ? list2[k] : list2[cap - 1u - (k - nfront)];
}

template <int G>
__global__ void __launch_bounds__(G == 8 ? 256 : 128, G == 8 ? 1 : 8) k_lbk_filter(const uint2* __restrict__ cand, const unsigned* __restrict__ perm,
                                                    const float* __restrict__ rows, int n, const float* __restrict__ U_g,
                                                    const float* __restrict__ L_g, int reach, QState* st,
                                                    uint4* __restrict__ list2, unsigned cap, float front)
{
    extern __shared__ __align__(16) float env[];
    float* U = env;
    float* L = U + ((n + 3) & ~3);
    for (int i = threadIdx.x; i < n; i += blockDim.x) { U[i] = U_g[i]; L[i] = L_g[i]; }
    __syncthreads();
    const unsigned total = *(volatile unsigned*)&st->cand_count;
    const int lane = threadIdx.x & 31;
    const unsigned wpb = blockDim.x >> 5;
    const float thr = __uint_as_float(st->lbk_thr_bits);  // the scan's threshold (BSF0, fixed)
    for (unsigned k0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * 32; k0 < total; k0 += gridDim.x * wpb * 32) {
        const bool valid = k0 + lane < total;
        const uint2 e = valid ? cand[k0 + lane] : make_uint2(0u, 0x7f800000u);
        const bool ok = valid && __uint_as_float(e.y) <= thr;
        const unsigned rid = ok ? perm[e.x] : 0u;
        unsigned todo = __ballot_sync(0xffffffffu, ok);
        unsigned passmask = 0, frontmask = 0;
        float mylbk = 0.0f, myhead = 0.0f;
        // G rows in flight per warp; per element d = c - clamp(c, L, U) (the LB_Keogh term
        // c - U above the envelope, c - L below it, 0 inside: P:1392-1405), squares summed
        // in element pairs with FFMA2.  G = 4: 128-thread CTAs of <= 64 registers, which fit
        // beside the resident refine kernel of the previous query (its 2 CTAs per SM leave
        // 8.7K registers).
        while (todo) {
            int src[G];
            unsigned id[G];
            bool gok[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                gok[g] = todo != 0;
                src[g] = gok[g] ? __ffs(todo) - 1 : 0;
                todo &= todo - 1;
                id[g] = __shfl_sync(0xffffffffu, rid, src[g]);
            }
            float2 acc[G];
            float head[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                acc[g] = make_float2(0.0f, 0.0f);
                head[g] = 0.0f;
            }
            for (int j = lane * 4; j < n; j += 128) {
                const float4 uv = *reinterpret_cast<const float4*>(U + j);
                const float4 lv = *reinterpret_cast<const float4*>(L + j);
                float4 cv[G];
#pragma unroll
                for (int g = 0; g < G; ++g)
                    cv[g] = gok[g] ? __ldg(reinterpret_cast<const float4*>(rows + (long long)id[g] * n + j))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                const bool in_head = j <= reach + 3;  // the columns of the DP's first window
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float d0 = cv[g].x - fminf(fmaxf(cv[g].x, lv.x), uv.x);
                    const float d1 = cv[g].y - fminf(fmaxf(cv[g].y, lv.y), uv.y);
                    const float d2 = cv[g].z - fminf(fmaxf(cv[g].z, lv.z), uv.z);
                    const float d3 = cv[g].w - fminf(fmaxf(cv[g].w, lv.w), uv.w);
                    acc[g] = ffma2(make_float2(d0, d1), make_float2(d0, d1), acc[g]);
                    acc[g] = ffma2(make_float2(d2, d3), make_float2(d2, d3), acc[g]);
                    if (in_head) {
                        const float dd[4] = {d0, d1, d2, d3};
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (j + k <= reach + 3) head[g] = fmaf(dd[k], dd[k], head[g]);
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float a = warp_sum(acc[g].x + acc[g].y);
                const float h = warp_sum(head[g]);
                if (gok[g] && a <= thr) {
                    passmask |= 1u << src[g];
                    if (a <= thr * front) frontmask |= 1u << src[g];
                    if (lane == src[g]) { mylbk = a; myhead = h; }
                }
            }
        }
        if (passmask) {
            const unsigned backmask = passmask & ~frontmask;
            unsigned fb = 0, bb = 0;
            if (lane == 0) {
                if (frontmask) fb = atomicAdd(&st->list2_count, (unsigned)__popc(frontmask));
                if (backmask) bb = atomicAdd(&st->list2_back, (unsigned)__popc(backmask));
            }
            fb = __shfl_sync(0xffffffffu, fb, 0);
            bb = __shfl_sync(0xffffffffu, bb, 0);
            const unsigned lt = (1u << lane) - 1u;
            const uint4 e = make_uint4(rid, __float_as_uint(mylbk), __float_as_uint(myhead), 0u);
            MESSI_CHECK(!(frontmask & (1u << lane)) || fb + __popc(frontmask & lt) + bb < cap);
            MESSI_CHECK(!(backmask & (1u << lane)) || bb + __popc(backmask & lt) + fb < cap);
            if (frontmask & (1u << lane)) list2[fb + __popc(frontmask & lt)] = e;
            if (backmask & (1u << lane)) list2[cap - 1u - (bb + __popc(backmask & lt))] = e;
        }
    }
}

// Lower bound of sqrt(LB_Keogh(x)) from the quantised row x^ = s c: the
// per-point term x -> dist(x, [L_i, U_i]) is 1-Lipschitz, so for any set S of points
//     sqrt(sum_S lbk(x_i)) >= sqrt(sum_S lbk(x^_i)) - ||x - x^||_2 >= sqrt(tq) - e
// for tq <= sum_S lbk(x^_i) and e >= ||x - x^||_2 (meta8).  Returns the squared bound,
// rounded down (tq is reduced by 2^-10 for the fp32 summation order).
__device__ __forceinline__ float q8_lbk_bound(float tq, float e)
{
    const float r = __fsub_rd(__fsqrt_rd(fmaxf(0.0f, tq * 0.9990234375f)), e);
    return r > 0.0f ? __fmul_rd(r, r) : 0.0f;
}

// DTW step 1 over the QUANTISED rows (strip refine reaches): the scan's candidates whose
// bound does not exceed BSF0 get the LB_Keogh of their quantised row x^ (n bytes + s, e
// instead of 4n bytes), kept when q8_lbk_bound(LBK(x^), e) <= BSF0 -- a lower bound of
// the raw LB_Keogh, hence of DTW.  list2 entries: (row id, LBK(x^), s, e);
// the strip refine computes its tail bound from the same quantised terms.  One lane per
// candidate: a lane streams its row's bytes 64 at a time (all lanes read the same U, L
// words: shared-memory broadcasts); two best-first bins as k_lbk_filter.  (G lanes per
// candidate with coalesced 16-byte chunks, G = 2..16, measured slower on C4: 22-64 ms vs
// 15.5 ms per 100 queries in the serial pass -- the four 16-byte loads a lane keeps in flight
// here matter more than the lines a warp load touches.)
__global__ void __launch_bounds__(128) k_lbk_filter_q8(const uint2* __restrict__ cand, const unsigned* __restrict__ perm,
                                                       const unsigned char* __restrict__ rows8,
                                                       const float2* __restrict__ meta8, int n,
                                                       const float* __restrict__ U_g, const float* __restrict__ L_g,
                                                       QState* st, uint4* __restrict__ list2, unsigned cap, float front,
                                                       uint4* __restrict__ rlist, float rho, const unsigned* cnt_p)
{
    extern __shared__ __align__(16) float env[];
    float* U = env;
    float* L = U + ((n + 15) & ~15);
    for (int i = threadIdx.x; i < n; i += blockDim.x) { U[i] = U_g[i]; L[i] = L_g[i]; }
    __syncthreads();
    const unsigned total = *(volatile const unsigned*)cnt_p;  // QState::cand_count or ::rcand_count
    const int lane = threadIdx.x & 31;
    const float thr = __uint_as_float(st->lbk_thr_bits);
    unsigned mf;  // 0x4B000000 (2^23) in a register the compiler cannot fold: PRMT keeps an immediate selector
    asm volatile("mov.b32 %0, 0x4B000000;" : "=r"(mf));
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k - lane < total; k += gridDim.x * blockDim.x) {
        const bool valid = k < total;
        const uint2 ce = valid ? cand[k] : make_uint2(0u, 0x7f800000u);
        const bool ok = valid && __uint_as_float(ce.y) <= thr;
        float a = 0.0f;
        float2 meta = make_float2(1.0f, INFINITY);
        if (ok) {
            meta = __ldg(meta8 + ce.x);
            const float qoff = -8388736.0f * meta.x;  // -(2^23 + 128) s, exact (s a power of two)
            const uint4* src = reinterpret_cast<const uint4*>(rows8 + (long long)ce.x * n);
            float2 acc = make_float2(0.0f, 0.0f);
            for (int j0 = 0; j0 < n; j0 += 64) {  // 64 bytes in flight per lane
                uint4 raw4[4];
#pragma unroll
                for (int h = 0; h < 4; ++h)
                    raw4[h] = j0 + 16 * h < n ? __ldg(src + (j0 >> 4) + h) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                const int j = j0 + 16 * h;
                if (j >= n) break;
                const uint4 raw = raw4[h];
                // int8 c -> biased byte c + 128 (flip each sign bit), for the 2^23 conversion below
                const unsigned wd[4] = {raw.x ^ 0x80808080u, raw.y ^ 0x80808080u, raw.z ^ 0x80808080u,
                                        raw.w ^ 0x80808080u};
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const float4 uu = *reinterpret_cast<const float4*>(U + j + 4 * g);
                    const float4 ll = *reinterpret_cast<const float4*>(L + j + 4 * g);
                    const float us[4] = {uu.x, uu.y, uu.z, uu.w}, ls[4] = {ll.x, ll.y, ll.z, ll.w};
                    float d[4];
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        // 2^23 + byte via PRMT, then (2^23 + byte - 2^23 - 128) * s in one exact FFMA
                        const float fm = __uint_as_float(__byte_perm(wd[g], mf, 0x7650u | b));
                        const float xq = fmaf(fm, meta.x, qoff);
                        d[b] = xq - fminf(fmaxf(xq, ls[b]), us[b]);
                    }
                    acc = ffma2(make_float2(d[0], d[1]), make_float2(d[0], d[1]), acc);
                    acc = ffma2(make_float2(d[2], d[3]), make_float2(d[2], d[3]), acc);
                }
                }
            }
            a = acc.x + acc.y;
        }
        const float bnd = q8_lbk_bound(a, meta.y);
        bool pass = ok && bnd <= thr;
        // survivors whose forward bound is <= rho * BSF0 (the ones the refine would run longest)
        // queue for the reverse bound (k_lbk_rev_q8) instead of going to list2
        const bool rq = rlist && pass && bnd <= rho * thr;
        const unsigned rmask = __ballot_sync(0xffffffffu, rq);
        if (rmask) {
            unsigned rb = 0;
            if (lane == 0) rb = atomicAdd(&st->rev_count, (unsigned)__popc(rmask));
            rb = __shfl_sync(0xffffffffu, rb, 0);
            MESSI_CHECK(!rq || rb + __popc(rmask & ((1u << lane) - 1u)) < cap);
            if (rq) rlist[rb + __popc(rmask & ((1u << lane) - 1u))] =
                make_uint4(ce.x, __float_as_uint(a), __float_as_uint(meta.x), __float_as_uint(meta.y));
            pass = pass && !rq;
        }
        const bool fr = pass && bnd <= thr * front;
        const unsigned passmask = __ballot_sync(0xffffffffu, pass), frontmask = __ballot_sync(0xffffffffu, fr);
        if (passmask) {
            const unsigned backmask = passmask & ~frontmask;
            unsigned fb = 0, bb = 0;
            if (lane == 0) {
                if (frontmask) fb = atomicAdd(&st->list2_count, (unsigned)__popc(frontmask));
                if (backmask) bb = atomicAdd(&st->list2_back, (unsigned)__popc(backmask));
            }
            fb = __shfl_sync(0xffffffffu, fb, 0);
            bb = __shfl_sync(0xffffffffu, bb, 0);
            const unsigned lt = (1u << lane) - 1u;
            if (pass) {
                const uint4 e = make_uint4(perm[ce.x], __float_as_uint(a), __float_as_uint(meta.x), __float_as_uint(meta.y));
                MESSI_CHECK(fb + __popc(frontmask & lt) + bb + __popc(backmask & lt) < cap);
                if (fr) list2[fb + __popc(frontmask & lt)] = e;
                else list2[cap - 1u - (bb + __popc(backmask & lt))] = e;
            }
        }
    }
}

// Reverse LB_Keogh of a quantised row ("reverse LB_Keogh"): LB_Keogh is
// defined for either series against the envelope of the other (every point of
// a series lies on the warping path, matched to a point of the other within the reach), so
//     LBrev(x) = sum_i dist(q_i, [L^x_i, U^x_i])^2 <= DTW(q, x),
// U^x_i / L^x_i = max / min of x over |k - i| <= R (clipped to [0, n)).  From the quantised
// row x^ = s c (|x_k - x^_k| <= s/2 per point, k_quantise): U^x <= U^x^ + s/2 and
// L^x >= L^x^ - s/2, so in code units (q' = q / s, exact: s is a power of two)
//     dist(q_i, [L^x_i, U^x_i]) / s >= max(q'_i - Uc_i - 1/2, Lc_i - q'_i - 1/2, 0),
// Uc / Lc the max / min code over the window.  Every rounding is DOWNWARD, so the result
// (times s^2, exact) lower-bounds LBrev(x) with no margin.
//
// Envelope: the codes as biased bytes b = c + 128 paired with their complements in one
// u16x2 word (b * 257, (255 - b) * 257), so ONE lanewise max (VIMNMX.U16x2) updates the
// max of b and the min of b (as 255 - max(255 - b)); absent points are 0 in both lanes.
// Points go in blocks of 8: the window of point 8b + t covers the suffix of block
// b - A - [t < R0] from offset (t - R0) mod 8, the whole blocks between, and the prefix of
// block b + A + [t + R0 >= 8] to offset (t + R0) mod 8 (A = R / 8, R0 = R mod 8), so each
// block's prefix / suffix maxima are computed once, when the block is loaded (A + 1 blocks
// ahead), into a ring of P = 2A + 3 register slots (the loop body is P blocks: the slot of a
// block is static), and every envelope value is one 3-input max.
// Term, per point: the byte pairs into floats 2^15 + b (PRMT into a magic exponent), then
// (RD(q' + 2^15 + 127.5) - (2^15 + Ub), RD(2^15 + 126.5 - q') - (2^15 + 255 - Lb)) --
// = (q' - Uc - 1/2, Lc - q' - 1/2), rounded down -- in one FFMA2 + one FSUB2.
template <int NN, int RR>
__device__ __forceinline__ float lbk_rev_q8(const unsigned* row, float s, const float* __restrict__ Q, unsigned mg)
{
    static_assert(NN % 16 == 0 && RR >= 8 && 2 * RR + 1 < NN, "lbk_rev_q8: unsupported (n, reach)");
    constexpr int NB = NN / 8, A = RR / 8, R0 = RR % 8, P = 2 * A + 3;
    unsigned pre[P][8], suf[P][8];
    auto vmax = [](unsigned x, unsigned y) { return __vmaxu2(x, y); };
    // block k into ring slot SL: its pairs, prefix and suffix maxima; VALID (compile-time)
    // says whether k is inside [0, NB) -- outside, the block is absent (all pairs 0)
    auto load = [&](int k, auto SL, auto VALID) {
        constexpr int sl = decltype(SL)::value;
        unsigned x[8];
        if constexpr (decltype(VALID)::value) {
            unsigned w0, w1;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                         : "=r"(w0), "=r"(w1)
                         : "r"((unsigned)__cvta_generic_to_shared(row + 2 * k)));
            const unsigned b0 = w0 ^ 0x80808080u, b1 = w1 ^ 0x80808080u;
            const unsigned c0 = ~b0, c1 = ~b1;
            static_for<4>([&](auto T) {
                constexpr int t = decltype(T)::value;
                constexpr unsigned sel = t | (t << 4) | ((4 + t) << 8) | ((4 + t) << 12);
                x[t] = __byte_perm(b0, c0, sel);
                x[4 + t] = __byte_perm(b1, c1, sel);
            });
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) x[t] = 0u;
        }
        pre[sl][0] = x[0];
#pragma unroll
        for (int t = 1; t < 8; ++t) pre[sl][t] = vmax(pre[sl][t - 1], x[t]);
        suf[sl][7] = x[7];
#pragma unroll
        for (int t = 6; t >= 0; --t) suf[sl][t] = vmax(suf[sl][t + 1], x[t]);
    };
    static_for<2 * A + 2>([&](auto I) {  // blocks -A-1 .. A
        constexpr int k = decltype(I)::value - A - 1;
        load(k, std::integral_constant<int, (k + P) % P>{}, std::integral_constant<bool, (k >= 0 && k < NB)>{});
    });
    const float inv = __frcp_rn(s);  // exact: s is a power of two
    const float2 sc2 = make_float2(inv, -inv), kk2 = make_float2(32895.5f, 32894.5f);
    float2 acc = make_float2(0.0f, 0.0f);
    // output block b (ring position j = b mod P): loads block b + A + 1 (present iff LV), then
    // the envelope and terms of points 8b .. 8b+7
    auto step = [&](int b, auto J, auto LV) {
        constexpr int j = decltype(J)::value;
        load(b + A + 1, std::integral_constant<int, (j + A + 1) % P>{}, LV);
        unsigned core = pre[(j - A + 1 + P) % P][7];
        static_for<2 * A - 2>([&](auto D) {
            constexpr int d = decltype(D)::value - A + 2;
            core = vmax(core, pre[(j + d + P) % P][7]);
        });
        const unsigned ml = vmax(core, pre[(j - A + P) % P][7]), mr = vmax(core, pre[(j + A) % P][7]);
        const unsigned mlr = vmax(ml, pre[(j + A) % P][7]);
        const float4 qa = *reinterpret_cast<const float4*>(Q + 8 * b);
        const float4 qb = *reinterpret_cast<const float4*>(Q + 8 * b + 4);
        const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        float dd[8];
        static_for<8>([&](auto T) {
            constexpr int t = decltype(T)::value;
            constexpr bool lft = t < R0, rgt = t + R0 >= 8;
            constexpr int sl_l = (j - A - (lft ? 1 : 0) + 2 * P) % P, ol = (t - R0 + 8) % 8;
            constexpr int sl_h = (j + A + (rgt ? 1 : 0)) % P, oh = (t + R0) % 8;
            const unsigned mid = lft ? (rgt ? mlr : ml) : (rgt ? mr : core);
            const unsigned e = __vimax3_u16x2(suf[sl_l][ol], mid, pre[sl_h][oh]);
            // (2^15 + Ub, 2^15 + 255 - Lb) as floats
            float2 f;
            asm("prmt.b32 %0, %1, %2, 0x7614;" : "=r"(*reinterpret_cast<unsigned*>(&f.x)) : "r"(e), "r"(mg));
            asm("prmt.b32 %0, %1, %2, 0x7634;" : "=r"(*reinterpret_cast<unsigned*>(&f.y)) : "r"(e), "r"(mg));
            const float2 qk = ffma2_rd(make_float2(qv[t], qv[t]), sc2, kk2);
            const float2 ac = fsub2_rd(qk, f);
            dd[t] = max3f(ac.x, ac.y, 0.0f);
        });
#pragma unroll
        for (int p = 0; p < 4; ++p)
            acc = ffma2_rd(make_float2(dd[2 * p], dd[2 * p + 1]), make_float2(dd[2 * p], dd[2 * p + 1]), acc);
    };
    // ring periods whose every step is inside [0, NB) and loads a present block run as a
    // loop; the rest (the last < 2P steps) are unrolled with their bounds known at compile time
    constexpr int CLEAN = NB - A - P > 0 ? (NB - A - P + P - 1) / P : 0;  // periods b0 < NB - A - P
#pragma unroll 1
    for (int b0 = 0; b0 < CLEAN * P; b0 += P)
        static_for<P>([&](auto J) { step(b0 + decltype(J)::value, J, std::true_type{}); });
    static_for<2 * P>([&](auto I) {
        constexpr int b = CLEAN * P + decltype(I)::value;
        if constexpr (b < NB)
            step(b, std::integral_constant<int, b % P>{}, std::integral_constant<bool, (b + A + 1 < NB)>{});
    });
    return __fmul_rd(__fadd_rd(acc.x, acc.y), s * s);
}

// The reverse LB_Keogh over the forward filter's queue (rlist: sorted position, LBK(x^), s, e;
// QState::rev_count entries), one thread per entry with every lane busy: the row's n bytes in
// flight, a copy in this thread's shared-memory slot for lbk_rev_q8; entries whose reverse
// bound is <= the threshold join list2 (front bin by the larger of the two bounds).
// rev_out / dbg_map: inspection only (the bound per inspected id).
template <int NN, int RR>
__global__ void __launch_bounds__(128) k_lbk_rev_q8(const uint4* __restrict__ rlist, const unsigned* __restrict__ perm,
                                                    const unsigned char* __restrict__ rows8, const float* __restrict__ q_g,
                                                    QState* st, uint4* __restrict__ list2, unsigned cap, float front,
                                                    float* __restrict__ rev_out, const int* __restrict__ dbg_map)
{
    __shared__ __align__(16) float Q[NN];
    __shared__ __align__(16) unsigned rowbuf[128 * (NN / 4 + 2)];
    unsigned* myrow = rowbuf + threadIdx.x * (NN / 4 + 2);
    __shared__ unsigned magic;
    if (threadIdx.x == 0) magic = 0x47000000u;
    for (int i = threadIdx.x; i < NN; i += blockDim.x) Q[i] = q_g[i];
    __syncthreads();
    const unsigned mg = magic;
    const unsigned total = *(volatile unsigned*)&st->rev_count;
    const int lane = threadIdx.x & 31;
    const float thr = __uint_as_float(st->lbk_thr_bits);
    const unsigned stride = gridDim.x * blockDim.x;
    const uint4 none = make_uint4(0u, 0u, 0x3f800000u, 0x7f800000u);
    // the next entry's row is prefetched into L1 while this one is evaluated
    auto prefetch = [&](const uint4& e) {
        const char* r = reinterpret_cast<const char*>(rows8) + (long long)e.x * NN;
#pragma unroll
        for (int c = 0; c < NN; c += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(r + c));
    };
    unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k + stride < total) prefetch(rlist[k + stride]);
    uint4 nxt;
    for (; k - lane < total; k += stride) {
        const bool valid = k < total;
        const uint4 e = valid ? rlist[k] : none;
        if (k + 2 * stride < total) {  // the entry after next: its row to L1
            nxt = rlist[k + 2 * stride];
            prefetch(nxt);
        }
        const float a = __uint_as_float(e.y), s = __uint_as_float(e.z), ee = __uint_as_float(e.w);
        float rev = INFINITY;
        if (valid) {
            if (isinf(ee) || !(s >= 0x1p-60f && s <= 0x1p60f)) {
                rev = 0.0f;  // an unusable row (all-zero codes): not filtered here
            } else {
                const uint4* src = reinterpret_cast<const uint4*>(rows8 + (long long)e.x * NN);
                uint4 raw[NN / 16];
#pragma unroll
                for (int h = 0; h < NN / 16; ++h) raw[h] = __ldg(src + h);
#pragma unroll
                for (int h = 0; h < NN / 16; ++h) {
                    *reinterpret_cast<uint2*>(myrow + 4 * h) = make_uint2(raw[h].x, raw[h].y);
                    *reinterpret_cast<uint2*>(myrow + 4 * h + 2) = make_uint2(raw[h].z, raw[h].w);
                }
                rev = lbk_rev_q8<NN, RR>(myrow, s, Q, mg);
            }
            if (rev_out) rev_out[dbg_map[perm[e.x]]] = rev;
        }
        const float bnd = q8_lbk_bound(a, ee);
        const bool pass = valid && rev <= thr;
        const bool fr = pass && fmaxf(bnd, rev) <= thr * front;
        const unsigned passmask = __ballot_sync(0xffffffffu, pass), frontmask = __ballot_sync(0xffffffffu, fr);
        if (passmask) {
            const unsigned backmask = passmask & ~frontmask;
            unsigned fb = 0, bb = 0;
            if (lane == 0) {
                if (frontmask) fb = atomicAdd(&st->list2_count, (unsigned)__popc(frontmask));
                if (backmask) bb = atomicAdd(&st->list2_back, (unsigned)__popc(backmask));
            }
            fb = __shfl_sync(0xffffffffu, fb, 0);
            bb = __shfl_sync(0xffffffffu, bb, 0);
            const unsigned lt = (1u << lane) - 1u;
            if (pass) {
                const uint4 o = make_uint4(perm[e.x], e.y, e.z, e.w);
                MESSI_CHECK(fb + __popc(frontmask & lt) + bb + __popc(backmask & lt) < cap);
                if (fr) list2[fb + __popc(frontmask & lt)] = o;
                else list2[cap - 1u - (bb + __popc(backmask & lt))] = o;
            }
        }
    }
}

// k_lbk_filter_q8 with the reverse bound, for the (n, reach) pairs it is compiled for
// (MESSI_REV_SPECS): a lane loads its whole row (n bytes in flight), computes the forward
// quantised LB_Keogh exactly as k_lbk_filter_q8, and -- when that passes -- lbk_rev_q8; the
// candidate is kept when both bounds are <= the threshold (rev_out, inspection only: the
// reverse bound per candidate position, +inf when not computed).
#define MESSI_REV_SPECS(X) X(256, 12) X(256, 25) X(256, 51)
template <int NN, int RR>
__global__ void __launch_bounds__(128) k_lbk_filter_q8r(const uint2* __restrict__ cand, const unsigned* __restrict__ perm,
                                                        const unsigned char* __restrict__ rows8,
                                                        const float2* __restrict__ meta8, const float* __restrict__ U_g,
                                                        const float* __restrict__ L_g, const float* __restrict__ q_g,
                                                        QState* st, uint4* __restrict__ list2, unsigned cap, float front,
                                                        float* __restrict__ rev_out)
{
    __shared__ __align__(16) float U[NN], L[NN], Q[NN];
    // per-thread row copies, NN + 8 bytes apart: the 8-byte loads of a half-warp hit 16
    // distinct bank pairs
    __shared__ __align__(16) unsigned rowbuf[128 * (NN / 4 + 2)];
    unsigned* myrow = rowbuf + threadIdx.x * (NN / 4 + 2);
    // the PRMT magic exponents read back from shared memory, so the compiler cannot fold them
    // into PRMT's immediate (which would put each byte selector in a register instead)
    __shared__ unsigned magic[2];
    if (threadIdx.x == 0) { magic[0] = 0x4B000000u; magic[1] = 0x47000000u; }
    for (int i = threadIdx.x; i < NN; i += blockDim.x) { U[i] = U_g[i]; L[i] = L_g[i]; Q[i] = q_g[i]; }
    __syncthreads();
    const unsigned mf = magic[0], mg = magic[1];
    const unsigned total = *(volatile unsigned*)&st->cand_count;
    const int lane = threadIdx.x & 31;
    const float thr = __uint_as_float(st->lbk_thr_bits);
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k - lane < total; k += gridDim.x * blockDim.x) {
        const bool valid = k < total;
        const uint2 ce = valid ? cand[k] : make_uint2(0u, 0x7f800000u);
        const bool ok = valid && __uint_as_float(ce.y) <= thr;
        float a = 0.0f, rev = INFINITY;
        float2 meta = make_float2(1.0f, INFINITY);
        if (ok) {
            meta = __ldg(meta8 + ce.x);
            const float qoff = -8388736.0f * meta.x;
            const uint4* src = reinterpret_cast<const uint4*>(rows8 + (long long)ce.x * NN);
            uint4 raw[NN / 16];
#pragma unroll
            for (int h = 0; h < NN / 16; ++h) raw[h] = __ldg(src + h);
#pragma unroll
            for (int h = 0; h < NN / 16; ++h) {  // this thread's copy for the reverse bound
                *reinterpret_cast<uint2*>(myrow + 4 * h) = make_uint2(raw[h].x, raw[h].y);
                *reinterpret_cast<uint2*>(myrow + 4 * h + 2) = make_uint2(raw[h].z, raw[h].w);
            }
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll 4
            for (int h = 0; h < NN / 16; ++h) {
                // back from the thread's copy (volatile: the registers of the loads are free)
                uint4 rw;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%4];\n\tld.shared.v2.u32 {%2, %3}, [%4+8];"
                             : "=r"(rw.x), "=r"(rw.y), "=r"(rw.z), "=r"(rw.w)
                             : "r"((unsigned)__cvta_generic_to_shared(myrow + 4 * h)));
                const unsigned wd[4] = {rw.x ^ 0x80808080u, rw.y ^ 0x80808080u, rw.z ^ 0x80808080u, rw.w ^ 0x80808080u};
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const float4 uu = *reinterpret_cast<const float4*>(U + 16 * h + 4 * g);
                    const float4 ll = *reinterpret_cast<const float4*>(L + 16 * h + 4 * g);
                    const float us[4] = {uu.x, uu.y, uu.z, uu.w}, ls[4] = {ll.x, ll.y, ll.z, ll.w};
                    float d[4];
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const float fm = __uint_as_float(__byte_perm(wd[g], mf, 0x7650u | b));
                        const float xq = fmaf(fm, meta.x, qoff);
                        d[b] = xq - fminf(fmaxf(xq, ls[b]), us[b]);
                    }
                    acc = ffma2(make_float2(d[0], d[1]), make_float2(d[0], d[1]), acc);
                    acc = ffma2(make_float2(d[2], d[3]), make_float2(d[2], d[3]), acc);
                }
            }
            a = acc.x + acc.y;
            // the reverse bound where the forward one passes (an unusable row, e = +inf, has
            // all-zero codes: no per-point bound, so it is not filtered here)
            if (q8_lbk_bound(a, meta.y) <= thr) rev = (isinf(meta.y) || !(meta.x >= 0x1p-60f && meta.x <= 0x1p60f))
                          ? 0.0f : lbk_rev_q8<NN, RR>(myrow, meta.x, Q, mg);
        }
        if (rev_out && valid) rev_out[k] = rev;
        const float bnd = q8_lbk_bound(a, meta.y);
        const bool pass = ok && bnd <= thr && rev <= thr;
        const bool fr = pass && bnd <= thr * front;
        const unsigned passmask = __ballot_sync(0xffffffffu, pass), frontmask = __ballot_sync(0xffffffffu, fr);
        if (passmask) {
            const unsigned backmask = passmask & ~frontmask;
            unsigned fb = 0, bb = 0;
            if (lane == 0) {
                if (frontmask) fb = atomicAdd(&st->list2_count, (unsigned)__popc(frontmask));
                if (backmask) bb = atomicAdd(&st->list2_back, (unsigned)__popc(backmask));
            }
            fb = __shfl_sync(0xffffffffu, fb, 0);
            bb = __shfl_sync(0xffffffffu, bb, 0);
            const unsigned lt = (1u << lane) - 1u;
            if (pass) {
                const uint4 e = make_uint4(perm[ce.x], __float_as_uint(a), __float_as_uint(meta.x), __float_as_uint(meta.y));
                MESSI_CHECK(fb + __popc(frontmask & lt) + bb + __popc(backmask & lt) < cap);
                if (fr) list2[fb + __popc(frontmask & lt)] = e;
                else list2[cap - 1u - (bb + __popc(backmask & lt))] = e;
            }
        }
    }
}

// k_lbk_filter_q8 for compile-time n with the rows brought in by the bulk-copy (TMA) engine:
// each lane of a warp issues one cp.async.bulk of its candidate's n bytes into its own slot
// of a per-warp double buffer in shared memory (completion on the warp's mbarrier), so a
// row costs one instruction and no L1 wavefronts (one lane per row, n/16 LDG.128 per lane,
// made the L1 the limiter), and the next 32 rows are in flight while these are evaluated.
// Same values, list2 / rlist appends and result as k_lbk_filter_q8 (the per-point term as
// max(x^ - U, L - x^, 0), paired FADD2 + one FMNMX3, instead of x^ - clamp(x^, L, U)).
// mf = 0x4B000000 as a parameter: a value the compiler cannot fold into PRMT's immediate,
// which would leave every byte selector in a register.
template <int NN>
__host__ __device__ constexpr size_t lbkb_smem()
{
    return (size_t)2 * NN * 4 + 8 * 8 + (size_t)2 * 128 * (NN + 16);
}
template <int NN>
__global__ void __launch_bounds__(128) k_lbk_filter_q8b(const uint2* __restrict__ cand, const unsigned* __restrict__ perm,
                                                        const unsigned char* __restrict__ rows8,
                                                        const float2* __restrict__ meta8, const float* __restrict__ U_g,
                                                        const float* __restrict__ L_g, QState* st,
                                                        uint4* __restrict__ list2, unsigned cap, float front,
                                                        uint4* __restrict__ rlist, float rho, unsigned mf,
                                                        const unsigned* cnt_p)
{
    constexpr int RS = NN + 16;  // slot stride: 16-byte aligned, LDS.128 quarter-warps conflict-free
    extern __shared__ __align__(128) unsigned char lsm[];
    float* U = reinterpret_cast<float*>(lsm);
    float* L = U + NN;
    unsigned long long* mb = reinterpret_cast<unsigned long long*>(L + NN);  // [warp][buffer]
    unsigned char* rowsm = reinterpret_cast<unsigned char*>(mb + 8);           // [buffer][thread][RS]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        mbar_init(&mb[2 * w], 1);
        mbar_init(&mb[2 * w + 1], 1);
    }
    for (int i = threadIdx.x; i < NN; i += blockDim.x) { U[i] = U_g[i]; L[i] = L_g[i]; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const unsigned total = *(volatile const unsigned*)cnt_p;  // QState::cand_count or ::rcand_count
    const float thr = __uint_as_float(st->lbk_thr_bits);
    const uint2 none = make_uint2(0u, 0x7f800000u);
    struct Cur { uint2 ce; bool ok; float2 meta; unsigned id; };
    // warp-uniform: rows of the candidates ce (k0 + lane, loaded one batch earlier) into
    // buffer b (lanes without a usable one copy nothing; the warp's mbarrier expects the
    // bytes of the others); their scale / error bound and row id load meanwhile
    auto issue = [&](uint2 ce, unsigned k0, int b) {
        Cur c;
        c.ce = ce;
        c.ok = k0 + lane < total && __uint_as_float(ce.y) <= thr;
        const unsigned cnt = __popc(__ballot_sync(0xffffffffu, c.ok));
        unsigned long long* bar = &mb[2 * w + b];
        if (lane == 0) mbar_expect_tx(bar, cnt * NN);
        __syncwarp();
        if (c.ok) {
            const unsigned dst = smem_u32(rowsm + ((size_t)b * 128 + threadIdx.x) * RS);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                "l"(rows8 + (long long)ce.x * NN), "r"(NN), "r"(smem_u32(bar))
                : "memory");
        }
        c.meta = c.ok ? __ldg(meta8 + ce.x) : make_float2(1.0f, INFINITY);
        c.id = c.ok ? __ldg(perm + ce.x) : 0u;
        return c;
    };
    // appends of one batch: the atomics are issued after its evaluation and their results
    // consumed after the NEXT batch's (their latency hidden behind it)
    struct Pend { unsigned rmask, passmask, frontmask, rb, fb, bb; uint4 e; bool rq, pass, fr; };
    auto flush = [&](const Pend& pd) {
        const unsigned lt = (1u << lane) - 1u;
        if (pd.rmask) {
            const unsigned rb = __shfl_sync(0xffffffffu, pd.rb, 0);
            MESSI_CHECK(!pd.rq || rb + __popc(pd.rmask & lt) < cap);
            if (pd.rq) rlist[rb + __popc(pd.rmask & lt)] = pd.e;
        }
        if (pd.passmask) {
            const unsigned backmask = pd.passmask & ~pd.frontmask;
            const unsigned fb = __shfl_sync(0xffffffffu, pd.fb, 0), bb = __shfl_sync(0xffffffffu, pd.bb, 0);
            MESSI_CHECK(!pd.pass || fb + __popc(pd.frontmask & lt) + bb + __popc(backmask & lt) < cap);
            if (pd.fr) list2[fb + __popc(pd.frontmask & lt)] = pd.e;
            else if (pd.pass) list2[cap - 1u - (bb + __popc(backmask & lt))] = pd.e;
        }
    };
    const unsigned kstep = gridDim.x * blockDim.x;
    unsigned k0 = (blockIdx.x * 4 + w) * 32;
    auto entry = [&](unsigned kb) { return kb + lane < total ? cand[kb + lane] : none; };
    Cur cur = {none, false, make_float2(1.0f, INFINITY), 0u};
    if (k0 < total) cur = issue(entry(k0), k0, 0);
    uint2 ce_n = entry(k0 + kstep);  // candidates of the next batch (their rows issued next iteration)
    Pend pend = {0u, 0u, 0u, 0u, 0u, 0u, make_uint4(0u, 0u, 0u, 0u), false, false, false};
    for (int it = 0; k0 < total; ++it, k0 += kstep) {
        const int b = it & 1;
        Cur nxt = {none, false, make_float2(1.0f, INFINITY), 0u};
        if (k0 + kstep < total) nxt = issue(ce_n, k0 + kstep, b ^ 1);
        ce_n = entry(k0 + 2 * kstep);
        mbar_wait(&mb[2 * w + b], (it >> 1) & 1);
        const bool ok = cur.ok;
        const float2 meta = cur.meta;
        float a = 0.0f;
        if (ok) {
            const unsigned char* row = rowsm + ((size_t)b * 128 + threadIdx.x) * RS;
            const float qoff = -8388736.0f * meta.x;  // -(2^23 + 128) s, exact (s a power of two)
            const float2 s2 = make_float2(meta.x, meta.x), qoff2 = make_float2(qoff, qoff);
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll 4
            for (int h = 0; h < NN / 16; ++h) {
                const uint4 raw = *reinterpret_cast<const uint4*>(row + 16 * h);
                const unsigned wd[4] = {raw.x ^ 0x80808080u, raw.y ^ 0x80808080u, raw.z ^ 0x80808080u,
                                        raw.w ^ 0x80808080u};
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const float4 uu = *reinterpret_cast<const float4*>(U + 16 * h + 4 * g);
                    const float4 ll = *reinterpret_cast<const float4*>(L + 16 * h + 4 * g);
                    float fm[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) fm[q] = __uint_as_float(__byte_perm(wd[g], mf, 0x7650u | q));
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        // x^ = (2^23 + byte - 2^23 - 128) s exactly; dist = max(x^ - U, L - x^, 0)
                        const float2 xq = ffma2(make_float2(fm[2 * p], fm[2 * p + 1]), s2, qoff2);
                        const float2 up = p ? make_float2(uu.z, uu.w) : make_float2(uu.x, uu.y);
                        const float2 lo = p ? make_float2(ll.z, ll.w) : make_float2(ll.x, ll.y);
                        const float2 da = fadd2(xq, make_float2(-up.x, -up.y));
                        const float2 db = fadd2(lo, make_float2(-xq.x, -xq.y));
                        const float2 d = make_float2(max3f(da.x, db.x, 0.0f), max3f(da.y, db.y, 0.0f));
                        acc = ffma2(d, d, acc);
                    }
                }
            }
            a = acc.x + acc.y;
        }
        flush(pend);  // the previous batch's appends (its atomics have long returned)
        const float bnd = q8_lbk_bound(a, meta.y);
        Pend pd;
        pd.pass = ok && bnd <= thr;
        pd.rq = rlist && pd.pass && bnd <= rho * thr;
        pd.pass = pd.pass && !pd.rq;
        pd.fr = pd.pass && bnd <= thr * front;
        pd.rmask = __ballot_sync(0xffffffffu, pd.rq);
        pd.passmask = __ballot_sync(0xffffffffu, pd.pass);
        pd.frontmask = __ballot_sync(0xffffffffu, pd.fr);
        pd.rb = pd.fb = pd.bb = 0u;
        if (lane == 0) {
            if (pd.rmask) pd.rb = atomicAdd(&st->rev_count, (unsigned)__popc(pd.rmask));
            if (pd.frontmask) pd.fb = atomicAdd(&st->list2_count, (unsigned)__popc(pd.frontmask));
            if (pd.passmask & ~pd.frontmask) pd.bb = atomicAdd(&st->list2_back, (unsigned)__popc(pd.passmask & ~pd.frontmask));
        }
        pd.e = pd.rq ? make_uint4(cur.ce.x, __float_as_uint(a), __float_as_uint(meta.x), __float_as_uint(meta.y))
                     : make_uint4(cur.id, __float_as_uint(a), __float_as_uint(meta.x), __float_as_uint(meta.y));
        pend = pd;
        __syncwarp();  // every lane is done with buffer b before the next issue refills it
        cur = nxt;
    }
    flush(pend);
}

// Work distribution of the per-thread refine kernels: a lane that finishes (or skips) a
// candidate takes the next one from its warp's chunk of list2 entries; chunks of kClaimChunk
// consecutive entries are claimed with one atomicAdd on QState::next_tile, the next chunk one
// chunk ahead so the warp never waits on the atomic.  Lanes thus stay busy until the list is
// exhausted, whatever the spread of candidate lifetimes (early abandon after a few rows vs
// the full n), where a static lane stride left most lanes of a warp idle behind its slowest.
#ifndef MESSI_STRIP_DEPTH1  // strip refine: list2 entries held ahead per lane (1; 0: two, the round-2 session-3 kernel)
#define MESSI_STRIP_DEPTH1 1
#endif
#ifndef MESSI_STRIP_INTERLEAVE  // strip refine: chunk halves from the two ends of list2 (see k_refine_dtw_strip)
#define MESSI_STRIP_INTERLEAVE 1
#endif
#ifndef MESSI_CLAIM_CHUNK
#define MESSI_CLAIM_CHUNK 64
#endif
constexpr unsigned kClaimChunk = MESSI_CLAIM_CHUNK;

struct WarpClaim {
    unsigned cbase, cused;  // warp-uniform: current chunk, entries used
    unsigned nraw;          // lane 0: the next chunk (its atomic's result, read one chunk later)

    __device__ __forceinline__ void init(unsigned* ctr, int lane)
    {
        unsigned a = 0;
        nraw = 0;
        if (lane == 0) { a = atomicAdd(ctr, kClaimChunk); nraw = atomicAdd(ctr, kClaimChunk); }
        cbase = __shfl_sync(0xffffffffu, a, 0);
        cused = 0;
    }

    // Lanes of `m` (ballot of the lanes asking) get distinct entry indices.
    __device__ __forceinline__ unsigned take(unsigned* ctr, unsigned m, int lane)
    {
        const unsigned cnt = __popc(m);
        const unsigned pos = cused + __popc(m & ((1u << lane) - 1u));
        unsigned k = cbase + pos;
        if (cused + cnt > kClaimChunk) {  // warp-uniform: the chunk runs out
            const unsigned nbase = __shfl_sync(0xffffffffu, nraw, 0);
            if (pos >= kClaimChunk) k = nbase + (pos - kClaimChunk);
            cbase = nbase;
            cused = cused + cnt - kClaimChunk;
            if (lane == 0) nraw = atomicAdd(ctr, kClaimChunk);  // consumed at the next overflow
        } else {
            cused += cnt;
        }
        return k;
    }
};

// DTW step 2 (Alg. 10 line RealDist, P:1425 / P:1453 "true DTW distance"): banded fp32
// DTW, one thread per LB_Keogh survivor (band in registers, DtwThread<R>), entries handed
// out by WarpClaim.  Each lane holds its current candidate and the next two list2 entries
// (nxt loaded, nxt2 in flight); the row of nxt is prefetched into L1.
template <int R>
__global__ void __launch_bounds__(128) k_refine_dtw(const float* __restrict__ rows, int n, const float* __restrict__ q_g,
                                                    const float* __restrict__ U_g, const float* __restrict__ L_g,
                                                    const uint4* __restrict__ list2, unsigned cap, QState* st,
                                                    NearEntry* near, KnnState* knn, int kk, PeerSet ps, int slot)
{
    extern __shared__ __align__(16) float dsm[];
    const int npad = (n + 3) & ~3;
    float* q_s = dsm;
    float* U = dsm + npad;
    float* L = dsm + 2 * npad;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { q_s[i] = q_g[i]; U[i] = U_g[i]; L[i] = L_g[i]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned nfront = *(volatile unsigned*)&st->list2_count;
    const unsigned total = nfront + *(volatile unsigned*)&st->list2_back;
    unsigned* ctr = &st->next_tile;
    WarpClaim wc;
    wc.init(ctr, lane);
    const uint4 none = make_uint4(0xffffffffu, 0u, 0u, 0u);  // .x = ~0: no entry
    auto fetch = [&](unsigned k) { return k < total ? list2_at(list2, k, nfront, cap) : none; };
    uint4 nxt = fetch(wc.take(ctr, 0xffffffffu, lane));
    uint4 nxt2 = fetch(wc.take(ctr, 0xffffffffu, lane));
    auto prefetch_row = [&](unsigned rid) {
        const char* pr = reinterpret_cast<const char*>(rows + (long long)rid * n);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pr));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pr + 128));
    };
    if (nxt.x != 0xffffffffu) prefetch_row(nxt.x);
    DtwThread<R> dp;
    const float* c = rows;
    unsigned id = 0, refined = 0, abandoned = 0, skipped = 0;
    unsigned long long cells = 0;
    float lbk_total = 0.0f;
    float thr = slack_up(ld_bsf_eff(st, ps.epoch));  // linked shards: the shared BSF too
    const bool frozen = *(volatile const unsigned*)&st->frozen != 0u;  // inspection: no BSF updates
    bool running = false;
    for (;;) {
        // lanes without a candidate take their next entry (a candidate whose LB_Keogh
        // already exceeds the threshold is skipped unstarted)
        const bool need = !running && nxt.x != 0xffffffffu;
        const unsigned m = __ballot_sync(0xffffffffu, need);
        if (m) {
            const unsigned k = wc.take(ctr, m, lane);
            if (need) {
                id = nxt.x;
                lbk_total = __uint_as_float(nxt.y);
                const float head = __uint_as_float(nxt.z);
                nxt = nxt2;
                nxt2 = fetch(k);
                if (nxt.x != 0xffffffffu) prefetch_row(nxt.x);
                if (lbk_total * 0.9990234375f <= thr) {
                    c = rows + (long long)id * n;
                    dp.start(c, n, head);
                    ++refined;
                    running = true;
                } else {
                    ++skipped;
                }
            }
        }
        if (!__any_sync(0xffffffffu, running || nxt.x != 0xffffffffu)) break;
        if (running) {
            const float bsf_now = ld_bsf_eff(st, ps.epoch);  // consumed after the step
            const float rowmin = dp.step4(c, n, q_s, U, L);
            thr = fminf(thr, slack_up(bsf_now));
            const float tail = fmaxf(0.0f, lbk_total * 0.9990234375f - dp.seen_lo * 1.0009765625f);
            const float bound = (rowmin + tail) * 0.9990234375f;
            if (bound > thr) {
                running = false;
                ++abandoned;
                cells += band_cells(n, R, dp.i);
            } else if (dp.i >= n) {
                running = false;
                cells += band_cells(n, R, n);
                const float d = dp.result();
                if (d <= thr) dtw_accept(st, near, knn, kk, frozen, id, d, thr, ps, slot);
            }
        }
    }
    refined = __reduce_add_sync(0xffffffffu, refined);
    abandoned = __reduce_add_sync(0xffffffffu, abandoned + skipped);
    cells = warp_sum_u64(cells);
    if ((threadIdx.x & 31) == 0) {
        if (refined) atomicAdd(&st->refined, refined);
        if (abandoned) atomicAdd(&st->abandoned, abandoned);
        if (cells) atomicAdd(&st->dtw_cells, cells);
    }
}

// Shared memory of k_refine_dtw_strip: the boundary arrays (2R+2 slots x T threads), the
// query pairs padded by R points of +inf on each side in K lane copies, U, L.
__host__ __device__ inline size_t strip_smem(int n, int R, int K, int T = kStripThreads)
{
    const size_t npad = (size_t)((n + 3) & ~3);
    return ((size_t)(2 * R + 2) * T + (size_t)(n + 2 * R) * K * 2 + 2 * npad) * sizeof(float);
}

// Query copies: 16 while the CTA's shared memory stays <= 76 KB (three CTAs per SM; C4: 68 KB;
// with 8 copies of single points the loads conflicted on 46% of wavefronts: 1277 vs 1305
// q/s), else 8.
__host__ __device__ inline int strip_qcopies(int n, int R)
{
    if (strip_smem(n, R, 16) <= 76 * 1024 || R < 7) return 16;
    if (strip_smem(n, R, 8) <= 227 * 1024) return 8;  // K = 8 variants exist for H = 8
    return 1;  // large n and R: one copy, 64-thread CTAs (strip_threads)
}

// DTW step 2 for any reach (DtwStrip<H>, one thread per LB_Keogh survivor), the same
// candidate hand-out, BSF sharing and early abandon as k_refine_dtw: after each strip of
// H rows every warping path still has to cross its last row (>= rmin) and visit every
// later candidate point j at least once, at a cost >= that point's LB_Keogh term against
// the query envelope, so the candidate is dropped when rmin + (LBK_total -
// LBK of the rows done) exceeds the threshold (2^-10 margins for the fp32 sums).
template <int H, int REM, int K, int T>
__global__ void __launch_bounds__(T) k_refine_dtw_strip(const float* __restrict__ rows, int n, int R,
                                                                   const float* __restrict__ q_g,
                                                                   const float* __restrict__ U_g,
                                                                   const float* __restrict__ L_g,
                                                                   const uint4* __restrict__ list2, unsigned cap,
                                                                   QState* st, NearEntry* near, KnnState* knn, int kk,
                                                                   PeerSet ps, int slot, unsigned full_min)
{
    extern __shared__ __align__(16) float dsm[];
    // Short lists (fewer than full_min entries: under ~4 per thread of the full grid) run on two
    // thirds of the CTAs: with so few entries per lane they are all bound at the first claim, and
    // fewer, longer-lived warps balance them better (C4: serial refine 25.1 -> 22.7 ms per 100
    // queries at 2 CTAs per SM, 24.5 at 1); long lists keep every CTA.
    if (blockIdx.x * 3u >= gridDim.x * 2u &&
        *(volatile unsigned*)&st->list2_count + *(volatile unsigned*)&st->list2_back < full_min)
        return;
    const int npad = (n + 3) & ~3;
    float2* qrep = reinterpret_cast<float2*>(dsm + (size_t)(2 * R + 2) * T);  // 8-byte aligned: 2R+2 even
    float* U = reinterpret_cast<float*>(qrep + (size_t)(n + 2 * R) * K);
    float* L = U + npad;
    for (int x = threadIdx.x; x < (n + 2 * R) * K; x += T) {
        const int i = x / K - R;
        qrep[x] = make_float2((i >= 0 && i < n) ? q_g[i] : INFINITY, (i >= 1 && i <= n) ? q_g[i - 1] : INFINITY);
    }
    for (int i = threadIdx.x; i < n; i += T) { U[i] = U_g[i]; L[i] = L_g[i]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float* Bt = dsm + threadIdx.x;
    const float2* qlane = qrep + (lane & (K - 1));
    const int nfull = (2 * R - 2 * H + 3) / H;
    const unsigned nfront = *(volatile unsigned*)&st->list2_count;
    const unsigned total = nfront + *(volatile unsigned*)&st->list2_back;
    unsigned* ctr = &st->next_tile;
    WarpClaim wc;
    wc.init(ctr, lane);
    const uint4 none = make_uint4(0xffffffffu, 0u, 0u, 0u);
#if MESSI_STRIP_INTERLEAVE
    // Hand-out order: the first half of every 64-entry chunk comes from the START of the list
    // (the front bin: small LB_Keogh, the candidates that run deep), the second half from its
    // END (large LB_Keogh: abandoned after a strip or two).  A warp's first claim gives every
    // lane one entry of each half -- its current candidate and the one it holds ahead -- so no
    // lane starts with two deep candidates in a row while other warps run out of work (the
    // front bin then set the kernel's time: two full DPs back to back on ~F/64 warps).
    // Entry k: a = 32 (k / 64) + k mod 32; k mod 64 < 32: position a (a < ceil(total/2)),
    // else position total-1-a (a < floor(total/2)); other k below kmax are holes (skipped).
    static_assert(kClaimChunk == 64, "the interleaved hand-out splits 64-entry chunks in halves");
    static_assert(MESSI_STRIP_DEPTH1 == 1, "holes of the interleaved order need the has_nxt flag");
    const unsigned kmax = ((total + 63u) >> 6) << 6, half_lo = (total + 1u) >> 1, half_hi = total >> 1;
    auto fetch = [&](unsigned k) {
        const unsigned a = ((k >> 6) << 5) | (k & 31u);
        const bool hi = (k & 32u) != 0u;
        if (k >= kmax || a >= (hi ? half_hi : half_lo)) return none;
        return list2_at(list2, hi ? total - 1u - a : a, nfront, cap);
    };
#else
    const unsigned kmax = total;
    auto fetch = [&](unsigned k) { return k < total ? list2_at(list2, k, nfront, cap) : none; };
#endif
#if MESSI_STRIP_DEPTH1
    // one list2 entry ahead per lane (claimed when the lane starts a candidate, its row
    // prefetched one strip later), so few entries are tied to a lane when the list is short
    unsigned k1 = wc.take(ctr, 0xffffffffu, lane);
    bool has_nxt = k1 < kmax, pf = false;
    uint4 nxt = fetch(k1);
#else
    uint4 nxt = fetch(wc.take(ctr, 0xffffffffu, lane));
    uint4 nxt2 = fetch(wc.take(ctr, 0xffffffffu, lane));
#endif
    auto prefetch_row = [&](unsigned rid) {
        const char* pr = reinterpret_cast<const char*>(rows + (long long)rid * n);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pr));
    };
    if (nxt.x != 0xffffffffu) prefetch_row(nxt.x);
    auto load_h = [&](const float* c, int j, float (&dst)[H]) {
        if constexpr (H % 4 == 0) {
#pragma unroll
            for (int b = 0; b < H / 4; ++b) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(c + j) + b);
                dst[4 * b] = v.x; dst[4 * b + 1] = v.y; dst[4 * b + 2] = v.z; dst[4 * b + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int u = 0; u < H; ++u) dst[u] = __ldg(c + j + u);
        }
    };
    DtwStrip<H> dp;
    float cnext[H];
    const float* c = rows;
    int j0 = 0;
    unsigned id = 0, refined = 0, abandoned = 0, skipped = 0;
    unsigned long long cells = 0;
    // list2 entries of k_lbk_filter_q8: (id, LB_Keogh of the quantised row x^, s, e); the
    // tail bound uses the quantised terms of the rows not done yet (q8_lbk_bound), with
    // x^_j = s rint(x_j / s) recomputed from the raw point (bit-identical to k_quantise)
    float lbk_total = 0.0f, seen = 0.0f, qs = 1.0f, qinv = 1.0f, qe = INFINITY;
    float thr = slack_up(ld_bsf_eff(st, ps.epoch));  // linked shards: the shared BSF too
    const bool frozen = *(volatile const unsigned*)&st->frozen != 0u;  // inspection: no BSF updates
    bool running = false;
    for (;;) {
        // lanes without a candidate take list2 entries until one passes its bound (up to four
        // rounds: a lane whose entry is skipped does not sit out a whole strip), then start it
        bool start = false;
#if MESSI_STRIP_DEPTH1
        if (pf) {  // the entry claimed a strip ago has landed
            if (has_nxt && nxt.x != 0xffffffffu) prefetch_row(nxt.x);
            pf = false;
        }
#endif
#pragma unroll 1
        for (int tries = 0; tries < 4; ++tries) {
#if MESSI_STRIP_DEPTH1
            const bool need = !running && !start && has_nxt;
#else
            const bool need = !running && !start && nxt.x != 0xffffffffu;
#endif
            const unsigned m = __ballot_sync(0xffffffffu, need);
            if (!m) break;
            const unsigned k = wc.take(ctr, m, lane);
            if (need) {
                id = nxt.x;
                lbk_total = __uint_as_float(nxt.y);
                qs = __uint_as_float(nxt.z);
                qe = __uint_as_float(nxt.w);
#if MESSI_STRIP_DEPTH1
                has_nxt = k < kmax;
                nxt = fetch(k);
                pf = true;
#else
                nxt = nxt2;
                nxt2 = fetch(k);
                if (nxt.x != 0xffffffffu) prefetch_row(nxt.x);
#endif
                if (id == 0xffffffffu) {  // a hole of the interleaved order: nothing to refine
                } else if (q8_lbk_bound(lbk_total, qe) <= thr) start = true;
                else ++skipped;
            }
        }
        if (start) {
            qinv = __frcp_rn(qs);  // exact: s is a power of two
            c = rows + (long long)id * n;
            load_h(c, 0, cnext);
            // virtual row -1: D(-1, -1) = 0 (slot R), +inf elsewhere
            for (int x = 0; x < 2 * R + 2; ++x) Bt[x * T] = x == R ? 0.0f : INFINITY;
            j0 = 0;
            seen = 0.0f;
            ++refined;
            running = true;
        }
#if MESSI_STRIP_DEPTH1
        if (!__any_sync(0xffffffffu, running || has_nxt)) break;
#else
        if (!__any_sync(0xffffffffu, running || nxt.x != 0xffffffffu)) break;
#endif
        if (running) {
            const float bsf_now = ld_bsf_eff(st, ps.epoch);  // consumed after the strip
#pragma unroll
            for (int u = 0; u < H; ++u) dp.cv[u] = cnext[u];
            if (j0 + H < n) load_h(c, j0 + H, cnext);  // the next strip's points, one strip ahead
            dp.template run<REM, K, T>(Bt, qlane + (size_t)j0 * K, R, nfull);
#pragma unroll
            for (int u = 0; u < H; ++u) {
                const float v = rintf(dp.cv[u] * qinv) * qs, uu = U[j0 + u], ll = L[j0 + u];
                const float d = v - fminf(fmaxf(v, ll), uu);
                seen = fmaf(d, d, seen);
            }
            j0 += H;
            thr = fminf(thr, slack_up(bsf_now));
            const float tail = q8_lbk_bound(fmaxf(0.0f, lbk_total - seen * 1.0009765625f), qe);
            const float bound = (dp.rmin + tail) * 0.9990234375f;
            if (bound > thr) {
                running = false;
                ++abandoned;
                cells += band_cells(n, R, j0);
            } else if (j0 >= n) {
                running = false;
                cells += band_cells(n, R, n);
                const float d = Bt[R * T];  // D(n-1, n-1): column n-1 of the last row
                if (d <= thr) dtw_accept(st, near, knn, kk, frozen, id, d, thr, ps, slot);
            }
        }
    }
    refined = __reduce_add_sync(0xffffffffu, refined);
    abandoned = __reduce_add_sync(0xffffffffu, abandoned + skipped);
    cells = warp_sum_u64(cells);
    if (lane == 0) {
        if (refined) atomicAdd(&st->refined, refined);
        if (abandoned) atomicAdd(&st->abandoned, abandoned);
        if (cells) atomicAdd(&st->dtw_cells, cells);
    }
}

// DTW seed, step 2, at the strip reaches: ONE THREAD PER WINDOW ROW (k_seed_prologue's
// window, R14; BSF0 rule as k_seed_dtw): the strip DP of k_refine_dtw_strip (DtwStrip<H>) over
// the row, abandoned once the strip's row minimum exceeds the best finished window distance
// (every warping path crosses that row, and costs are >= 0: the row cannot be the window's
// minimum); finished rows publish their fp32 DTW (1-NN) or, with seed_d (k-NN), every row runs
// to the end and its distance goes to seed_d for k_seed_select.  The DP costs ~2.5
// instructions per cell where the warp wavefront (k_seed_dtw) spends ~45 per anti-diagonal
// step, so the seed holds ceil(window / T) CTAs instead of the whole GPU.
template <int H, int REM, int K, int T>
__global__ void __launch_bounds__(T) k_seed_rows(const float* __restrict__ rows, int n, int R,
                                                 const float* __restrict__ q_g, const unsigned* __restrict__ perm,
                                                 QState* st, float* __restrict__ seed_d, PeerSet ps, int slot)
{
    extern __shared__ __align__(16) float dsm[];
    float2* qrep = reinterpret_cast<float2*>(dsm + (size_t)(2 * R + 2) * T);
    for (int x = threadIdx.x; x < (n + 2 * R) * K; x += T) {
        const int i = x / K - R;
        qrep[x] = make_float2((i >= 0 && i < n) ? q_g[i] : INFINITY, (i >= 1 && i <= n) ? q_g[i - 1] : INFINITY);
    }
    __syncthreads();
    const int len = st->window_len;
    const int k = blockIdx.x * T + threadIdx.x;
    if (k >= len) return;
    const int lane = threadIdx.x & 31;
    float* Bt = dsm + threadIdx.x;
    const float2* qlane = qrep + (lane & (K - 1));
    const int nfull = (2 * R - 2 * H + 3) / H;
    const float* c = rows + (long long)perm[st->window_start + k] * n;
    for (int x = 0; x < 2 * R + 2; ++x) Bt[x * T] = x == R ? 0.0f : INFINITY;  // virtual row -1
    auto load_h = [&](int j, float (&dst)[H]) {
        if constexpr (H % 4 == 0) {
#pragma unroll
            for (int b = 0; b < H / 4; ++b) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(c + j) + b);
                dst[4 * b] = v.x; dst[4 * b + 1] = v.y; dst[4 * b + 2] = v.z; dst[4 * b + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int u = 0; u < H; ++u) dst[u] = __ldg(c + j + u);
        }
    };
    DtwStrip<H> dp;
    float cnext[H];
    load_h(0, cnext);
    for (int j0 = 0; j0 < n; j0 += H) {
#pragma unroll
        for (int u = 0; u < H; ++u) dp.cv[u] = cnext[u];
        if (j0 + H < n) load_h(j0 + H, cnext);
        dp.template run<REM, K, T>(Bt, qlane + (size_t)j0 * K, R, nfull);
        if (!seed_d && dp.rmin * 0.9990234375f > slack_up(ld_bsf_eff(st, ps.epoch))) return;
    }
    const float d = Bt[R * T];  // D(n-1, n-1)
    if (seed_d) {
        seed_d[k] = d;
    } else {
        bsf_publish(st, ps, slot, d);
        atomicMin(&st->seed_bits, __float_as_uint(d));
    }
}

// Stage one row into a warp's shared buffer (float4, n % 4 == 0).
__device__ __forceinline__ void stage_row(float* dst, const float* __restrict__ src, int n, int lane)
{
    for (int j = lane * 4; j < n; j += 128)
        *reinterpret_cast<float4*>(dst + j) = __ldg(reinterpret_cast<const float4*>(src + j));
    __syncwarp();
}

// DTW step 2 for reaches without a register-band instantiation: one warp per candidate,
// fp32 anti-diagonal wavefront (dtw_warp<float>) over the row staged in shared memory.
// Per-warp shared memory: n floats of row + 3n floats of anti-diagonals.
__global__ void k_refine_dtw_warp(const float* __restrict__ rows, int n, int reach, const float* __restrict__ q_g,
                                  const uint4* __restrict__ list2, unsigned cap, QState* st, NearEntry* near,
                                  KnnState* knn, int kk, PeerSet ps, int slot)
{
    extern __shared__ __align__(16) float dsm[];
    const int npad = (n + 3) & ~3;
    float* q_s = dsm;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    float* c_s = dsm + npad + (size_t)w * 4 * npad;
    float* buf = c_s + npad;
    const unsigned nfront = *(volatile unsigned*)&st->list2_count;
    const unsigned total = nfront + *(volatile unsigned*)&st->list2_back;
    unsigned refined = 0;
    for (unsigned k = blockIdx.x * wpb + w; k < total; k += gridDim.x * wpb) {
        const unsigned id = list2_at(list2, k, nfront, cap).x;
        stage_row(c_s, rows + (long long)id * n, n, lane);
        const float d = dtw_warp_any<float>(q_s, c_s, n, reach, buf, lane);
        ++refined;
        float thr = slack_up(ld_bsf_eff(st, ps.epoch));
        if (lane == 0 && d <= thr)
            dtw_accept(st, near, knn, kk, *(volatile const unsigned*)&st->frozen != 0u, id, d, thr, ps, slot);
    }
    if (lane == 0 && refined) {
        atomicAdd(&st->refined, refined);
        atomicAdd(&st->dtw_cells, (unsigned long long)refined * band_cells(n, reach, n));
    }
}

// ------------------------------------------------------------------- exact resolution

__device__ __forceinline__ bool better(double d, long long id, double bd, long long bid)
{
    return d < bd || (d == bd && id >= 0 && (bid < 0 || id < bid));
}

// Writes the query's result and stats, then re-arms the state for the next query.
__device__ void finish_query(Best b, unsigned nb, QState* st, long long N, long long row_begin,
                             void* result, void* stats)
{
    struct R { double dist; long long id; double d2; long long reserved; };
    struct S { long long lb, tiles, cand, lbk, refined, abandoned, near, cells, exact, listed, coarse; double seed, bsf; long long rpaa; };
    R* res = reinterpret_cast<R*>(result);
    res->dist = b.id >= 0 ? sqrt(b.d) : (double)INFINITY;
    res->id = b.id >= 0 ? row_begin + b.id : -1;
    res->d2 = b.d;
    res->reserved = 0;
    if (stats) {
        S* s = reinterpret_cast<S*>(stats);
        s->lb = (long long)st->tile_count * MESSI_TILE_ROWS < N ? (long long)st->tile_count * MESSI_TILE_ROWS : N;
        s->tiles = st->tile_count;
        s->cand = st->cand_count;
        s->lbk = st->list2_count + st->list2_back;
        s->refined = st->refined;
        s->abandoned = st->abandoned;
        s->near = nb;
        s->cells = (long long)st->dtw_cells;
        s->exact = st->rev_count;  // DTW: reverse LB_Keogh evaluations
        s->listed = st->tile_count;
        s->coarse = st->coarse_count;
        s->seed = (double)__uint_as_float(st->seed_bits);
        s->bsf = (double)__uint_as_float(st->bsf_bits);
        s->rpaa = st->rev_paa ? st->rcand_count : st->cand_count;
    }
    arm_state(st);
}

__device__ Best block_best(Best b, int* cnt_io)
{
    __shared__ double sd[32];
    __shared__ long long si[32];
    __shared__ int sc[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int cnt = *cnt_io;
    for (int o = 16; o; o >>= 1) {
        double od = __shfl_xor_sync(0xffffffffu, b.d, o);
        long long oi = __shfl_xor_sync(0xffffffffu, b.id, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (better(od, oi, b.d, b.id)) { b.d = od; b.id = oi; }
    }
    if (lane == 0) { sd[w] = b.d; si[w] = b.id; sc[w] = cnt; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < nw; ++k) {
            if (better(sd[k], si[k], b.d, b.id)) { b.d = sd[k]; b.id = si[k]; }
            cnt += sc[k];
        }
    }
    *cnt_io = cnt;
    return b;
}

// DTW exact resolution (A9): every near-best entry with d32 <= BSF_final*(1+eps) is
// recomputed in fp64 with the warp wavefront (bit-identical to the row-by-row DP of the
// oracle: every cell is fl(fl(d*d) + min) whatever the order).  Per-warp shared memory:
// q and the row (2 npad floats), then (reach > kShflMaxReach and gbuf == NULL) the 3n
// doubles of the shared-memory wavefront; with gbuf the wavefront lives in global scratch
// (gbuf + 3n per warp: long series whose buffers do not fit shared memory).
__host__ __device__ inline size_t resolve_warp_bytes(int n, int reach, bool global_buf)
{
    const size_t npad = (size_t)((n + 3) & ~3);
    return 2 * npad * sizeof(float) + ((reach > kShflMaxReach && !global_buf) ? (size_t)3 * n * sizeof(double) : 0);
}

__global__ void k_resolve_dtw(const float* __restrict__ rows, int n, int reach, const float* __restrict__ q_g,
                              const NearEntry* __restrict__ near, QState* st, long long N, long long row_begin,
                              void* result, void* stats, double* gbuf)
{
    extern __shared__ __align__(16) double dbuf[];
    const int npad = (n + 3) & ~3;
    const float thr = slack_up(ld_bsf(st));
    const unsigned total = *(volatile unsigned*)&st->near_count;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    char* mine = reinterpret_cast<char*>(dbuf) + (size_t)w * resolve_warp_bytes(n, reach, gbuf != nullptr);
    float* qc = reinterpret_cast<float*>(mine);  // q then c
    double* buf = gbuf ? gbuf + (size_t)w * 3 * n : reinterpret_cast<double*>(mine + 2 * (size_t)npad * sizeof(float));
    for (int i = lane; i < n; i += 32) qc[i] = q_g[i];
    Best b{(double)INFINITY, -1};
    int cnt = 0;
    for (unsigned k = w; k < total; k += wpb) {
        const NearEntry e = near[k];
        if (!(e.d32 <= thr)) continue;
        if (lane == 0) ++cnt;
        stage_row(qc + npad, rows + (long long)e.id * n, n, lane);
        const double d = dtw_warp_any<double>(qc, qc + npad, n, reach, buf, lane);
        if (better(d, e.id, b.d, b.id)) { b.d = d; b.id = e.id; }
    }
    b = block_best(b, &cnt);
    if (threadIdx.x == 0) finish_query(b, (unsigned)cnt, st, N, row_begin, result, stats);
}

// DTW k-NN exact resolution: every near-best entry with d32 <= BSF_final * (1 + eps) (BSF =
// the k-th smallest fp32 distance) is recomputed in fp64 (warp wavefront, as k_resolve_dtw)
// into scratch (d64, id) pairs; then k rounds of a block-wide lexicographic argmin, each over
// the pairs strictly greater than the previous pick (ids are distinct), give the k smallest
// (d64, id) in order: results[k] (fewer rows -> (inf, -1)), stats, and the slot is re-armed.
// Same per-warp memory layout as k_resolve_dtw.
__global__ void k_resolve_dtw_knn(const float* __restrict__ rows, int n, int reach, const float* __restrict__ q_g,
                                  const NearEntry* __restrict__ near, QState* st, long long N, long long row_begin,
                                  void* result, void* stats, double* gbuf, double2* __restrict__ scratch, int kk)
{
    extern __shared__ __align__(16) double dbuf[];
    __shared__ unsigned cnt_s;
    __shared__ double rd[MESSI_MAX_K];
    __shared__ long long ri[MESSI_MAX_K];
    __shared__ double wd[32];
    __shared__ long long wi[32];
    const int npad = (n + 3) & ~3;
    const float thr = slack_up(ld_bsf(st));
    const unsigned total = *(volatile unsigned*)&st->near_count;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    if (threadIdx.x == 0) cnt_s = 0;
    __syncthreads();
    char* mine = reinterpret_cast<char*>(dbuf) + (size_t)w * resolve_warp_bytes(n, reach, gbuf != nullptr);
    float* qc = reinterpret_cast<float*>(mine);
    double* buf = gbuf ? gbuf + (size_t)w * 3 * n : reinterpret_cast<double*>(mine + 2 * (size_t)npad * sizeof(float));
    for (int i = lane; i < n; i += 32) qc[i] = q_g[i];
    for (unsigned k = w; k < total; k += wpb) {
        const NearEntry e = near[k];
        if (!(e.d32 <= thr)) continue;
        stage_row(qc + npad, rows + (long long)e.id * n, n, lane);
        const double d = dtw_warp_any<double>(qc, qc + npad, n, reach, buf, lane);
        if (lane == 0) scratch[atomicAdd(&cnt_s, 1u)] = make_double2(d, __longlong_as_double((long long)e.id));
    }
    for (int r = threadIdx.x; r < kk; r += blockDim.x) { rd[r] = (double)INFINITY; ri[r] = -1; }
    __syncthreads();
    const unsigned cnt = cnt_s;
    double pd = -1.0;
    long long pi = -1;
    for (int r = 0; r < kk && r < (int)cnt; ++r) {
        double bd = (double)INFINITY;
        long long bi = -1;
        for (unsigned i = threadIdx.x; i < cnt; i += blockDim.x) {
            const double2 e = scratch[i];
            const long long id = __double_as_longlong(e.y);
            const bool after = e.x > pd || (e.x == pd && id > pi);
            if (after && (e.x < bd || (e.x == bd && (bi < 0 || id < bi)))) { bd = e.x; bi = id; }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (better(od, oi, bd, bi)) { bd = od; bi = oi; }
        }
        if (lane == 0) { wd[w] = bd; wi[w] = bi; }
        __syncthreads();
        bd = wd[0];
        bi = wi[0];
        for (int j = 1; j < wpb; ++j)
            if (better(wd[j], wi[j], bd, bi)) { bd = wd[j]; bi = wi[j]; }
        if (threadIdx.x == 0) { rd[r] = bd; ri[r] = bi; }
        __syncthreads();
        pd = bd;
        pi = bi;
    }
    if (threadIdx.x == 0) {
        struct Rr { double dist; long long id; double d2; long long reserved; };
        Rr* res = reinterpret_cast<Rr*>(result);
        for (int r = 1; r < kk; ++r) {
            const bool have = ri[r] >= 0;
            res[r].dist = have ? sqrt(rd[r]) : (double)INFINITY;
            res[r].id = have ? row_begin + ri[r] : -1;
            res[r].d2 = have ? rd[r] : (double)INFINITY;
            res[r].reserved = 0;
        }
        finish_query(Best{ri[0] >= 0 ? rd[0] : (double)INFINITY, ri[0]}, cnt, st, N, row_begin, result, stats);
    }
}

__global__ void k_arm(QState* st) { arm_state(st); }

__global__ void k_arm_knn(QState* st, KnnState* kn)
{
    arm_state(st);
    kn->n32 = 0;
    kn->n64 = 0;
}

// --------------------------------------------------------------------- inspection
// fp64 DTW of `k` local row ids with the resolve kernel's engine (dtw_warp_any<double>,
// one warp per id; same per-warp memory layout as k_resolve_dtw).
__global__ void k_debug_dtw64(const float* __restrict__ rows, int n, int reach, const float* __restrict__ q_g,
                              const unsigned* __restrict__ ids, int k, double* __restrict__ d64, double* gbuf)
{
    extern __shared__ __align__(16) double dbuf[];
    const int npad = (n + 3) & ~3;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    char* mine = reinterpret_cast<char*>(dbuf) + (size_t)w * resolve_warp_bytes(n, reach, gbuf != nullptr);
    float* qc = reinterpret_cast<float*>(mine);
    double* buf = gbuf ? gbuf + ((size_t)blockIdx.x * wpb + w) * 3 * n
                       : reinterpret_cast<double*>(mine + 2 * (size_t)npad * sizeof(float));
    for (int i = lane; i < n; i += 32) qc[i] = q_g[i];
    for (int t = blockIdx.x * wpb + w; t < k; t += gridDim.x * wpb) {
        stage_row(qc + npad, rows + (long long)ids[t] * n, n, lane);
        const double d = dtw_warp_any<double>(qc, qc + npad, n, reach, buf, lane);
        if (lane == 0) d64[t] = d;
        __syncwarp();
    }
}

}  // namespace messi
