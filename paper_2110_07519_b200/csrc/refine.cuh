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

// ED refine (Alg. 9; Alg. 8 BSF update P:1178-1186): one warp per candidate.
// Skip when the candidate's LB already exceeds the current BSF (the BSF has dropped since
// the scan); else the fp32 squared ED; a result <= BSF*(1+eps) lowers the BSF (atomicMin,
// the lock-free form of the paper's BSF lock) and joins the near-best list.
__global__ void __launch_bounds__(256) k_refine_ed(const float* __restrict__ rows, int n, const float* __restrict__ q_g,
                                                   const uint2* __restrict__ cand, QState* st, NearEntry* near)
{
    extern __shared__ __align__(16) float q_s[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    const unsigned total = *(volatile unsigned*)&st->cand_count;
    const int lane = threadIdx.x & 31;
    const unsigned wpb = blockDim.x >> 5;
    unsigned refined = 0;
    for (unsigned k = blockIdx.x * wpb + (threadIdx.x >> 5); k < total; k += gridDim.x * wpb) {
        const uint2 e = cand[k];
        float thr = slack_up(ld_bsf(st));
        if (__uint_as_float(e.y) > thr) continue;
        const float d = ed2_warp(q_s, rows + (long long)e.x * n, n, lane);
        ++refined;
        thr = slack_up(ld_bsf(st));
        if (lane == 0 && d <= thr) {
            bsf_update(st, d);
            append_near(st, near, e.x, d);
        }
    }
    if (lane == 0 && refined) atomicAdd(&st->refined, refined);
}

// DTW step 1 (Alg. 10 line LB_Keogh): raw LB_Keogh of each scan survivor against
// the query envelope; survivors with LBK <= BSF*(1+eps) go to list2.  One warp per
// candidate, 32 candidates per round, one atomicAdd per round.
__global__ void __launch_bounds__(256) k_lbk_filter(const float* __restrict__ rows, int n, const float* __restrict__ U_g,
                                                    const float* __restrict__ L_g, const uint2* __restrict__ cand,
                                                    QState* st, unsigned* __restrict__ list2)
{
    extern __shared__ __align__(16) float env[];
    float* U = env;
    float* L = env + ((n + 3) & ~3);
    for (int i = threadIdx.x; i < n; i += blockDim.x) { U[i] = U_g[i]; L[i] = L_g[i]; }
    __syncthreads();
    const unsigned total = *(volatile unsigned*)&st->cand_count;
    const int lane = threadIdx.x & 31;
    const unsigned wpb = blockDim.x >> 5;
    const float thr = slack_up(ld_bsf(st));
    for (unsigned k0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * 32; k0 < total; k0 += gridDim.x * wpb * 32) {
        const unsigned cnt = min(32u, total - k0);
        const uint2 mine = lane < (int)cnt ? cand[k0 + lane] : make_uint2(0, 0x7f800000u);
        unsigned pass = 0;
        for (unsigned j = 0; j < cnt; ++j) {
            const unsigned id = __shfl_sync(0xffffffffu, mine.x, j);
            const float lb = __uint_as_float(__shfl_sync(0xffffffffu, mine.y, j));
            if (lb > thr) continue;
            const float v = lbk_warp(U, L, rows + (long long)id * n, n, lane);
            if (v <= thr) pass |= 1u << j;
        }
        if (pass) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&st->list2_count, (unsigned)__popc(pass));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (pass & (1u << lane)) list2[base + __popc(pass & ((1u << lane) - 1))] = mine.x;
        }
    }
}

// DTW step 2 (Alg. 10 line RealDist, P:1425 / P:1453 "true DTW distance"): banded fp32
// DTW, one thread per LB_Keogh survivor (band in registers, DtwThread<R>), lanes striding
// over list2.  Each lane keeps its own candidate; the loop runs while any lane has one, so
// a lane that abandons early simply starts its next candidate.
template <int R>
__global__ void __launch_bounds__(128) k_refine_dtw(const float* __restrict__ rows, int n, const float* __restrict__ q_g,
                                                    const unsigned* __restrict__ list2, QState* st, NearEntry* near)
{
    extern __shared__ __align__(16) float q_s[];
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    const unsigned total = *(volatile unsigned*)&st->list2_count;
    const unsigned nthreads = gridDim.x * blockDim.x;
    unsigned k = blockIdx.x * blockDim.x + threadIdx.x;
    DtwThread<R> dp;
    bool have = k < total;
    const float* c = rows;
    unsigned id = 0, refined = 0, abandoned = 0;
    if (have) {
        id = list2[k];
        c = rows + (long long)id * n;
        dp.start(c, n);
        ++refined;
    }
    float thr = slack_up(ld_bsf(st));
    while (__any_sync(0xffffffffu, have)) {
        if (have) {
            const float rowmin = dp.step4(c, n, q_s);
            bool done = false;
            if (rowmin > thr) {
                thr = slack_up(ld_bsf(st));
                if (rowmin > thr) { done = true; ++abandoned; }
            }
            if (!done && dp.i >= n) {
                done = true;
                const float d = dp.result();
                thr = slack_up(ld_bsf(st));
                if (d <= thr) {
                    bsf_update(st, d);
                    append_near(st, near, id, d);
                }
            }
            if (done) {
                k += nthreads;
                have = k < total;
                if (have) {
                    id = list2[k];
                    c = rows + (long long)id * n;
                    dp.start(c, n);
                    ++refined;
                    thr = slack_up(ld_bsf(st));
                }
            }
        }
    }
    refined = __reduce_add_sync(0xffffffffu, refined);
    abandoned = __reduce_add_sync(0xffffffffu, abandoned);
    if ((threadIdx.x & 31) == 0) {
        if (refined) atomicAdd(&st->refined, refined);
        if (abandoned) atomicAdd(&st->abandoned, abandoned);
    }
}

// DTW step 2 for reaches without a register-band instantiation: one warp per candidate,
// fp32 anti-diagonal wavefront (dtw_warp<float>).
__global__ void k_refine_dtw_warp(const float* __restrict__ rows, int n, int reach, const float* __restrict__ q_g,
                                  const unsigned* __restrict__ list2, QState* st, NearEntry* near)
{
    extern __shared__ __align__(16) float dsm[];
    float* q_s = dsm;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    float* buf = dsm + ((n + 3) & ~3) + w * 3 * n;
    const unsigned total = *(volatile unsigned*)&st->list2_count;
    unsigned refined = 0;
    for (unsigned k = blockIdx.x * wpb + w; k < total; k += gridDim.x * wpb) {
        const unsigned id = list2[k];
        const float d = dtw_warp<float>(q_s, rows + (long long)id * n, n, reach, buf, lane);
        ++refined;
        const float thr = slack_up(ld_bsf(st));
        if (lane == 0 && d <= thr) {
            bsf_update(st, d);
            append_near(st, near, id, d);
        }
    }
    if (lane == 0 && refined) atomicAdd(&st->refined, refined);
}

// ------------------------------------------------------------------- exact resolution
struct Best { double d; long long id; };

__device__ __forceinline__ bool better(double d, long long id, double bd, long long bid)
{
    return d < bd || (d == bd && id >= 0 && (bid < 0 || id < bid));
}

// Writes the query's result and stats, then re-arms the state for the next query.
__device__ void finish_query(Best b, unsigned nb, QState* st, long long N, long long row_begin,
                             void* result, void* stats)
{
    struct R { double dist; long long id; double d2; long long reserved; };
    struct S { long long lb, cand, lbk, refined, abandoned, near; double seed, bsf; };
    R* res = reinterpret_cast<R*>(result);
    res->dist = b.id >= 0 ? sqrt(b.d) : (double)INFINITY;
    res->id = b.id >= 0 ? row_begin + b.id : -1;
    res->d2 = b.d;
    res->reserved = 0;
    if (stats) {
        S* s = reinterpret_cast<S*>(stats);
        s->lb = N;
        s->cand = st->cand_count;
        s->lbk = st->list2_count;
        s->refined = st->refined;
        s->abandoned = st->abandoned;
        s->near = nb;
        s->seed = (double)__uint_as_float(st->seed_bits);
        s->bsf = (double)__uint_as_float(st->bsf_bits);
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

// ED: every near-best entry with d32 <= BSF_final*(1+eps) is recomputed canonically in
// fp64; the lexicographic min over (d64, id) is the answer (reading R11/R12; Thm. 2
// P:1881-1913 exactness).  One CTA.
__global__ void __launch_bounds__(256) k_resolve_ed(const float* __restrict__ rows, int n, const float* __restrict__ q_g,
                                                    const NearEntry* __restrict__ near, QState* st, long long N,
                                                    long long row_begin, void* result, void* stats)
{
    const float thr = slack_up(ld_bsf(st));
    const unsigned total = *(volatile unsigned*)&st->near_count;
    Best b{(double)INFINITY, -1};
    int cnt = 0;
    for (unsigned k = threadIdx.x; k < total; k += blockDim.x) {
        const NearEntry e = near[k];
        if (!(e.d32 <= thr)) continue;
        ++cnt;
        const double d = ed2_exact(q_g, rows + (long long)e.id * n, n);
        if (better(d, e.id, b.d, b.id)) { b.d = d; b.id = e.id; }
    }
    b = block_best(b, &cnt);
    if (threadIdx.x == 0) finish_query(b, (unsigned)cnt, st, N, row_begin, result, stats);
}

// DTW: same, with the fp64 warp wavefront (bit-identical to the row-by-row DP of the
// oracle: every cell is fl(fl(d*d) + min) whatever the order).  buf: 3*n doubles per warp.
__global__ void k_resolve_dtw(const float* __restrict__ rows, int n, int reach, const float* __restrict__ q_g,
                              const NearEntry* __restrict__ near, QState* st, long long N, long long row_begin,
                              void* result, void* stats)
{
    extern __shared__ __align__(16) double dbuf[];
    const float thr = slack_up(ld_bsf(st));
    const unsigned total = *(volatile unsigned*)&st->near_count;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    double* buf = dbuf + (size_t)w * 3 * n;
    Best b{(double)INFINITY, -1};
    int cnt = 0;
    for (unsigned k = w; k < total; k += wpb) {
        const NearEntry e = near[k];
        if (!(e.d32 <= thr)) continue;
        if (lane == 0) ++cnt;
        const double d = dtw_warp<double>(q_g, rows + (long long)e.id * n, n, reach, buf, lane);
        if (better(d, e.id, b.d, b.id)) { b.d = d; b.id = e.id; }
    }
    b = block_best(b, &cnt);
    if (threadIdx.x == 0) finish_query(b, (unsigned)cnt, st, N, row_begin, result, stats);
}

__global__ void k_arm(QState* st) { arm_state(st); }

// --------------------------------------------------------------------- inspection
// Per id: refine-kernel fp32 distance (no abandoning), exact fp64 distance, and (DTW) the
// fp32 LB_Keogh -- the same device routines the query path runs.  One warp per id.
template <int R>
__global__ void k_debug_dist(const float* __restrict__ rows, int n, int reach, const float* __restrict__ q_g,
                             const float* __restrict__ U_g, const float* __restrict__ L_g,
                             const unsigned* __restrict__ ids, int k, float* d32, double* d64, float* lbk)
{
    extern __shared__ __align__(16) float dsm[];
    const int npad = (n + 3) & ~3;
    float* q_s = dsm;
    float* U = dsm + npad;
    float* L = dsm + 2 * npad;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    double* buf = reinterpret_cast<double*>(dsm + 3 * npad) + (size_t)w * 3 * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        q_s[i] = q_g[i];
        if (reach >= 0) { U[i] = U_g[i]; L[i] = L_g[i]; }
    }
    __syncthreads();
    for (int t = blockIdx.x * wpb + w; t < k; t += gridDim.x * wpb) {
        const float* c = rows + (long long)ids[t] * n;
        if (reach < 0) {
            float v = ed2_warp(q_s, c, n, lane);
            if (lane == 0) {
                if (d32) d32[t] = v;
                if (d64) d64[t] = ed2_exact(q_s, c, n);
            }
        } else {
            if (lbk) {
                float v = lbk_warp(U, L, c, n, lane);
                if (lane == 0) lbk[t] = v;
            }
            if (d64) {
                double v = dtw_warp<double>(q_s, c, n, reach, buf, lane);
                if (lane == 0) d64[t] = v;
            }
            if (d32) {
                float v;
                if (R >= 0 && reach == R) {
                    v = INFINITY;
                    if (lane == 0) {
                        DtwThread<(R >= 0 ? R : 0)> dp;
                        dp.start(c, n);
                        while (dp.i < n) dp.step4(c, n, q_s);
                        v = dp.result();
                    }
                } else {
                    v = dtw_warp<float>(q_s, c, n, reach, reinterpret_cast<float*>(buf), lane);
                }
                if (lane == 0) d32[t] = v;
            }
        }
    }
}

}  // namespace messi
