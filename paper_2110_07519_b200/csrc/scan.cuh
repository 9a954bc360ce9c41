// scan.cuh -- query prologue (A3), approximate-search seed (A4) and the lower-bound scan
// with candidate compaction (A5): the HBM-roofline step.
#pragma once
#include "common.cuh"
#include "dtw.cuh"

namespace messi {

// ----------------------------------------------------------------------------- prologue
// One CTA.  Query PAA (fp64 means; the fp32-rounded copy gives the query's iSAX word and
// key, same rule as the data, "calculate iSAX summary for QDS"), and the per-query
// lower-bound table T[s][v] = m * max(0, lo_w(v) - Ubar_s, Lbar_s - hi_w(v))^2 evaluated in
// fp64 and rounded DOWN to fp32.  ED: Ubar = Lbar = query PAA, so T is mindist's per-segment
// term (Property 1).  DTW (reach >= 0): U, L = the LB_Keogh envelope
// (clamped windows) and Ubar, Lbar their PAA, T = the ABOVE / BELOW /
// IN cases of Fig. fig:dtwsimd as one branch-free max.
__device__ void prologue_block(const float* __restrict__ q, int n, int reach, const float* __restrict__ beta_g,
                               const float* __restrict__ lo_w, const float* __restrict__ hi_w,
                               float* __restrict__ lut_g, float* __restrict__ U_g, float* __restrict__ L_g,
                               unsigned long long* key_out)
{
    __shared__ double ubar[MESSI_W], lbar[MESSI_W];
    __shared__ float beta[256];
    const int m = n / MESSI_W, tid = threadIdx.x;
    for (int i = tid; i < 255; i += blockDim.x) beta[i] = beta_g[i];
    if (reach >= 0) {
        for (int i = tid; i < n; i += blockDim.x) {
            int a = max(0, i - reach), b = min(n - 1, i + reach);
            float u = q[a], l = q[a];
            for (int j = a + 1; j <= b; ++j) { u = fmaxf(u, q[j]); l = fminf(l, q[j]); }
            U_g[i] = u;
            L_g[i] = l;
        }
    }
    __syncthreads();  // U_g / L_g visible to the block (global writes, same block)
    if (tid < 32) {
        const int s = tid & 15;
        int sym = 0;
        if (tid < 16) {
            double sq = 0.0, su = 0.0, sl = 0.0;
            for (int j = 0; j < m; ++j) {
                sq = __dadd_rn(sq, (double)q[s * m + j]);
                if (reach >= 0) {
                    su = __dadd_rn(su, (double)U_g[s * m + j]);
                    sl = __dadd_rn(sl, (double)L_g[s * m + j]);
                }
            }
            double qbar = __ddiv_rn(sq, (double)m);
            ubar[s] = reach >= 0 ? __ddiv_rn(su, (double)m) : qbar;
            lbar[s] = reach >= 0 ? __ddiv_rn(sl, (double)m) : qbar;
            sym = symbol_of(__double2float_rn(qbar), beta);
        }
        unsigned long long key = 0;
#pragma unroll
        for (int bit = 7; bit >= 4; --bit) {
            unsigned plane = __ballot_sync(0xffffffffu, tid < 16 && ((sym >> bit) & 1));
            key = (key << 16) | (plane & 0xffffu);
        }
        if (tid == 0 && key_out) *key_out = key;
    }
    __syncthreads();
    if (lut_g) {
        const double md = (double)m;
        for (int i = tid; i < MESSI_W * MESSI_CARD; i += blockDim.x) {
            int s = i >> 8, v = i & 255;
            double lo = (double)lo_w[v], hi = (double)hi_w[v];
            double d = fmax(0.0, fmax(lo - ubar[s], lbar[s] - hi));
            lut_g[i] = __double2float_rd(md * d * d);
        }
    }
}

// Cooperative lower_bound over the sorted keys: first position whose key >= qkey.
// 256-ary search, one global load per thread per level (~4 levels for 100M keys).
__device__ long long block_lower_bound(const unsigned long long* __restrict__ skey, long long N,
                                       unsigned long long qkey)
{
    long long lo = 0, hi = N;
    const int nt = blockDim.x;
    while (hi - lo > nt) {
        long long stride = (hi - lo + nt - 1) / nt;
        long long idx = lo + (long long)threadIdx.x * stride;
        int pred = idx < hi && skey[idx] < qkey;
        int cnt = __syncthreads_count(pred);
        long long nlo = cnt == 0 ? lo : lo + (long long)(cnt - 1) * stride + 1;
        long long nhi = min(hi, lo + (long long)cnt * stride);
        lo = nlo;
        hi = nhi;
    }
    long long idx = lo + threadIdx.x;
    int pred = idx < hi && skey[idx] < qkey;
    int cnt = __syncthreads_count(pred);
    return lo + cnt;
}

// Approximate search (Alg. 5 line approxSearch; the leaf "closest" to the query,
// P:562-567): the `window` rows around the query's key in approximate-search order stand
// in for MESSI's leaf (reading R14).  BSF0 = min real distance over them (fp32).  Every
// CTA repeats the search; CTA 0 also runs the prologue.  ED: one warp per window row.
__global__ void __launch_bounds__(256) k_seed_ed(const float* __restrict__ q_g, int n, const float* __restrict__ rows,
                                                 const unsigned long long* __restrict__ skey,
                                                 const unsigned* __restrict__ perm, long long N, int window,
                                                 const float* __restrict__ beta_g, const float* __restrict__ lo_w,
                                                 const float* __restrict__ hi_w, float* __restrict__ lut_g,
                                                 QState* st)
{
    extern __shared__ __align__(16) float q_s[];
    __shared__ unsigned long long qkey_s;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    prologue_block(q_s, n, -1, beta_g, lo_w, hi_w, blockIdx.x == 0 ? lut_g : nullptr, nullptr, nullptr, &qkey_s);
    __syncthreads();
    const unsigned long long qkey = qkey_s;
    long long a = block_lower_bound(skey, N, qkey);
    int len = (int)min((long long)window, N);
    long long start = max(0LL, min(a - len / 2, N - len));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->qkey = qkey;
        st->window_start = (int)start;
        st->window_len = len;
    }
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    float best = INFINITY;
    for (int k = blockIdx.x * wpb + (threadIdx.x >> 5); k < len; k += gridDim.x * wpb) {
        const float* c = rows + (long long)perm[start + k] * n;
        best = fminf(best, ed2_warp(q_s, c, n, lane));
    }
    if (lane == 0 && best < INFINITY) {
        bsf_update(st, best);
        atomicMin(&st->seed_bits, __float_as_uint(best));
    }
}

// DTW seed: prologue (envelope, envelope PAA, table) in CTA 0, then the window rows' fp32
// banded DTW, one warp per row (anti-diagonal wavefront, dtw.cuh).
__global__ void k_seed_dtw(const float* __restrict__ q_g, int n, int reach, const float* __restrict__ rows,
                           const unsigned long long* __restrict__ skey, const unsigned* __restrict__ perm,
                           long long N, int window, const float* __restrict__ beta_g,
                           const float* __restrict__ lo_w, const float* __restrict__ hi_w,
                           float* __restrict__ lut_g, float* __restrict__ U_g, float* __restrict__ L_g, QState* st)
{
    extern __shared__ __align__(16) float dsm[];
    float* q_s = dsm;
    __shared__ unsigned long long qkey_s;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    if (blockIdx.x == 0)
        prologue_block(q_s, n, reach, beta_g, lo_w, hi_w, lut_g, U_g, L_g, &qkey_s);
    else
        prologue_block(q_s, n, -1, beta_g, lo_w, hi_w, nullptr, nullptr, nullptr, &qkey_s);
    __syncthreads();
    const unsigned long long qkey = qkey_s;
    long long a = block_lower_bound(skey, N, qkey);
    int len = (int)min((long long)window, N);
    long long start = max(0LL, min(a - len / 2, N - len));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->qkey = qkey;
        st->window_start = (int)start;
        st->window_len = len;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    float* buf = dsm + ((n + 3) & ~3) + w * 3 * n;
    float best = INFINITY;
    for (int k = blockIdx.x * wpb + w; k < len; k += gridDim.x * wpb) {
        const float* c = rows + (long long)perm[start + k] * n;
        best = fminf(best, dtw_warp<float>(q_s, c, n, reach, buf, lane));
    }
    if (lane == 0 && best < INFINITY) {
        bsf_update(st, best);
        atomicMin(&st->seed_bits, __float_as_uint(best));
    }
}

// ---------------------------------------------------------------------- lower-bound scan
// Every series' lower bound LB = sum_s T[s][sym_s] (round-down adds), kept iff
// LB <= BSF0 * (1 + eps): Alg. 9 line LowerBound_SIMD / Alg. 10 line
// LowerBound_DTW_SIMD over the whole summary array, like ParIS+'s SIMS scan
// (P:432-443).  Shared-memory LUT, 64 KB: word v*64 + 16h + s holds T[s][v]; the lane that
// owns block b = 2p + h reads segment s = (t + p) mod 16 at step t, so the 32 lanes hit 32
// distinct banks for any symbol values.  PRMT builds the byte address (v << 8 | base) from
// the packed symbols in one instruction.  Survivors are compacted with a warp ballot/scan
// and one atomicAdd per warp-tile.  WRITE_ALL (inspection) writes every LB instead.
template <bool WRITE_ALL>
__global__ void __launch_bounds__(256, 2) k_scan(const uint4* __restrict__ tiles, long long ntiles, long long N,
                                                 const float* __restrict__ lut_g, QState* st,
                                                 uint2* __restrict__ cand, float* __restrict__ lb_all)
{
    extern __shared__ __align__(16) float lut_s[];  // 256 * 64 floats
    for (int i = threadIdx.x; i < MESSI_W * MESSI_CARD; i += blockDim.x) {
        int s = i >> 8, v = i & 255;
        float val = lut_g[i];
        lut_s[v * 64 + s] = val;
        lut_s[v * 64 + 16 + s] = val;
    }
    __syncthreads();
    const float thr = WRITE_ALL ? INFINITY : slack_up(ld_bsf(st));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int p = lane >> 1, h = lane & 1;
    const char* lbase = reinterpret_cast<const char*>(lut_s);
    for (long long tl = (long long)blockIdx.x * 8 + warp; tl < ntiles; tl += (long long)gridDim.x * 8) {
        const uint4* tp = tiles + tl * (MESSI_TILE_BYTES / 16) + lane;
        uint4 data[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) data[t] = __ldcs(tp + t * 32);
        float acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0.0f;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const unsigned base = (unsigned)((16 * h + ((t + p) & 15)) * 4);
            const unsigned wv[4] = {data[t].x, data[t].y, data[t].z, data[t].w};
#pragma unroll
            for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    unsigned addr = __byte_perm(wv[wi], base, 0x5504 | (b << 4));
                    acc[wi * 4 + b] = __fadd_rd(acc[wi * 4 + b], *reinterpret_cast<const float*>(lbase + addr));
                }
            }
        }
        const long long id0 = tl * MESSI_TILE_ROWS + lane * 16;
        if (WRITE_ALL) {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (id0 + k < N) lb_all[id0 + k] = acc[k];
        } else {
            unsigned mask = 0;
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (acc[k] <= thr && id0 + k < N) mask |= 1u << k;
            if (__any_sync(0xffffffffu, mask)) {
                int cnt = __popc(mask), incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int total = __shfl_sync(0xffffffffu, incl, 31);
                unsigned base = 0;
                if (lane == 0) base = atomicAdd(&st->cand_count, (unsigned)total);
                base = __shfl_sync(0xffffffffu, base, 0);
                unsigned pos = base + incl - cnt;
                while (mask) {
                    int k = __ffs(mask) - 1;
                    mask &= mask - 1;
                    float lb = 0.0f;
#pragma unroll
                    for (int kk = 0; kk < 16; ++kk)
                        if (kk == k) lb = acc[kk];
                    cand[pos++] = make_uint2((unsigned)(id0 + k), __float_as_uint(lb));
                }
            }
        }
    }
}

}  // namespace messi
