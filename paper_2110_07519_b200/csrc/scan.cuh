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
// fp64 and rounded DOWN to fp32.  Ubar / Lbar also go to the query state (tile filter).  ED: Ubar = Lbar = query PAA, so T is mindist's per-segment
// term (Property 1).  DTW (reach >= 0): U, L = the LB_Keogh envelope
// (clamped windows) and Ubar, Lbar their PAA, T = the ABOVE / BELOW /
// IN cases of Fig. fig:dtwsimd as one branch-free max.
__device__ void prologue_block(const float* __restrict__ q, int n, int reach, const float* __restrict__ beta_g,
                               const float* __restrict__ lo_w, const float* __restrict__ hi_w,
                               float* __restrict__ lut_g, float* __restrict__ tab, float* __restrict__ U_g,
                               float* __restrict__ L_g, unsigned long long* key_out, QState* st)
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
            if (lut_g) {  // for the tile filter
                st->ubar[s] = ubar[s];
                st->lbar[s] = lbar[s];
            }
            if (lut_g && reach >= 0) {  // the reverse envelope-PAA bound: qlo <= mean(q_seg) <= qhi
                double lo = 0.0, hi = 0.0;
                for (int j = 0; j < m; ++j) {
                    lo = __dadd_rd(lo, (double)q[s * m + j]);
                    hi = __dadd_ru(hi, (double)q[s * m + j]);
                }
                st->qlo[s] = __double2float_rd(__ddiv_rd(lo, (double)m));
                st->qhi[s] = __double2float_ru(__ddiv_ru(hi, (double)m));
            }
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
            const float t8 = __double2float_rd(md * d * d);
            lut_g[i] = t8;
            if (tab) {
                tab[v * 64 + 32 + s] = t8;
                tab[v * 64 + 48 + s] = t8;
            }
        }
        // scan table, coarse part: pair byte v = (a << 4 | c) of segments (2j, 2j+1) at
        // cardinality 16 -- the box of 4-bit symbol a is the union of the 8-bit boxes
        // 16a .. 16a+15, so T16 <= T8 of every refinement (Property 1 holds per level)
        if (tab) {
            for (int i = tid; i < MESSI_CARD * 8; i += blockDim.x) {
                const int v = i >> 3, j = i & 7, a = v >> 4, c = v & 15;
                const double da = fmax(0.0, fmax((double)lo_w[16 * a] - ubar[2 * j], lbar[2 * j] - (double)hi_w[16 * a + 15]));
                const double dc = fmax(0.0, fmax((double)lo_w[16 * c] - ubar[2 * j + 1],
                                                 lbar[2 * j + 1] - (double)hi_w[16 * c + 15]));
                const float pt = __double2float_rd(md * da * da + md * dc * dc);
#pragma unroll
                for (int cp = 0; cp < 4; ++cp) tab[v * 64 + 4 * j + cp] = pt;
            }
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
                                                 float* __restrict__ tab, QState* st)
{
    extern __shared__ __align__(16) float q_s[];
    __shared__ unsigned long long qkey_s;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    prologue_block(q_s, n, -1, beta_g, lo_w, hi_w, blockIdx.x == 0 ? lut_g : nullptr, blockIdx.x == 0 ? tab : nullptr,
                   nullptr, nullptr, &qkey_s, st);
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
// banded DTW, one warp per row (anti-diagonal wavefront, dtw.cuh) over the row staged in
// shared memory; BSF0 = their minimum (1-NN) or, with seed_d, every distance goes to seed_d
// for k_seed_select (k-NN: BSF0 = the k-th smallest).  Dynamic shared memory: q (npad) + per
// warp row (npad) + 3n floats.
__global__ void k_seed_dtw(const float* __restrict__ q_g, int n, int reach, const float* __restrict__ rows,
                           const unsigned long long* __restrict__ skey, const unsigned* __restrict__ perm,
                           long long N, int window, const float* __restrict__ beta_g,
                           const float* __restrict__ lo_w, const float* __restrict__ hi_w,
                           float* __restrict__ lut_g, float* __restrict__ tab, float* __restrict__ U_g,
                           float* __restrict__ L_g, QState* st, float* __restrict__ seed_d, PeerSet ps, int slot)
{
    extern __shared__ __align__(16) float dsm[];
    float* q_s = dsm;
    __shared__ unsigned long long qkey_s;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    if (blockIdx.x == 0)
        prologue_block(q_s, n, reach, beta_g, lo_w, hi_w, lut_g, tab, U_g, L_g, &qkey_s, st);
    else
        prologue_block(q_s, n, -1, beta_g, lo_w, hi_w, nullptr, nullptr, nullptr, nullptr, &qkey_s, st);
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
    const int npad = (n + 3) & ~3;
    float* c_s = dsm + npad + (size_t)w * (npad + 3 * n);
    float* buf = c_s + npad;
    float best = INFINITY;
    for (int k = blockIdx.x * wpb + w; k < len; k += gridDim.x * wpb) {
        for (int j = lane * 4; j < n; j += 128)
            *reinterpret_cast<float4*>(c_s + j) =
                __ldg(reinterpret_cast<const float4*>(rows + (long long)perm[start + k] * n + j));
        __syncwarp();
        const float d = dtw_warp_any<float>(q_s, c_s, n, reach, buf, lane);
        best = fminf(best, d);
        if (seed_d && lane == 0) seed_d[k] = d;  // k-NN: every window distance (k_seed_select)
    }
    if (!seed_d && lane == 0 && best < INFINITY) {
        bsf_publish(st, ps, slot, best);  // linked shards: also the peers' same slot
        atomicMin(&st->seed_bits, __float_as_uint(best));
    }
}

// DTW seed, step 1 (k_seed_rows does the distances): one CTA runs k_seed_dtw's prologue
// (envelope, tables) and window search and records the window in the query state.
__global__ void __launch_bounds__(256) k_seed_prologue(const float* __restrict__ q_g, int n, int reach,
                                                       const unsigned long long* __restrict__ skey, long long N,
                                                       int window, const float* __restrict__ beta_g,
                                                       const float* __restrict__ lo_w, const float* __restrict__ hi_w,
                                                       float* __restrict__ lut_g, float* __restrict__ tab,
                                                       float* __restrict__ U_g, float* __restrict__ L_g, QState* st)
{
    extern __shared__ __align__(16) float q_s[];
    __shared__ unsigned long long qkey_s;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q_g[i];
    __syncthreads();
    prologue_block(q_s, n, reach, beta_g, lo_w, hi_w, lut_g, tab, U_g, L_g, &qkey_s, st);
    __syncthreads();
    const unsigned long long qkey = qkey_s;
    const long long a = block_lower_bound(skey, N, qkey);
    const int len = (int)min((long long)window, N);
    if (threadIdx.x == 0) {
        st->qkey = qkey;
        st->window_start = (int)max(0LL, min(a - len / 2, N - len));
        st->window_len = len;
    }
}

// ---------------------------------------------------------------------- tile filter
// MESSI's node pruning (Alg. 7 TraverseRootSubtree: "if FindDist(node) > BSF then prune",
// P:1117-1143) on the flat tile array: the box of a tile (per segment the min and max
// 8-bit symbol of its 512 sorted series) contains every member's symbol box, so
// m * sum_s max(0, lo(min_s) - Ubar_s, Lbar_s - hi(max_s))^2 (fp64) lower-bounds every
// member's bound and distance (Property 1/2).  Tiles whose bound exceeds
// BSF0 * (1 + eps) are skipped; the others are listed (one thread per tile) for the scan.
__global__ void k_tile_filter(const unsigned char* __restrict__ boxes, long long ntiles, int m,
                              const float* __restrict__ lo_w, const float* __restrict__ hi_w, QState* st,
                              unsigned* __restrict__ list, float* __restrict__ lb_all, unsigned epoch)
{
    __shared__ float lo[256], hi[256];
    __shared__ double ub[16], lb[16];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) { lo[i] = lo_w[i]; hi[i] = hi_w[i]; }
    if (threadIdx.x < 16) { ub[threadIdx.x] = st->ubar[threadIdx.x]; lb[threadIdx.x] = st->lbar[threadIdx.x]; }
    __syncthreads();
    const double thr = (double)slack_up(ld_bsf_eff(st, epoch));  // linked shards: the shared BSF too
    const int lane = threadIdx.x & 31;
    for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < ntiles; t0 += (long long)gridDim.x * blockDim.x) {
        const long long t = t0 + threadIdx.x;
        bool keep = false;
        double acc = 0.0;
        if (t < ntiles) {
            const uint4 mn = *reinterpret_cast<const uint4*>(boxes + t * 32);
            const uint4 mx = *reinterpret_cast<const uint4*>(boxes + t * 32 + 16);
            const unsigned a[4] = {mn.x, mn.y, mn.z, mn.w}, b[4] = {mx.x, mx.y, mx.z, mx.w};
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                const unsigned vmin = (a[s >> 2] >> (8 * (s & 3))) & 255u, vmax = (b[s >> 2] >> (8 * (s & 3))) & 255u;
                const double d = fmax(0.0, fmax((double)lo[vmin] - ub[s], lb[s] - (double)hi[vmax]));
                acc += d * d;
            }
            acc *= (double)m;
            keep = acc <= thr;
            if (lb_all) lb_all[t] = (float)acc;
        }
        if (list) {
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            unsigned base = 0;
            if (lane == 0 && msk) base = atomicAdd(&st->tile_count, (unsigned)__popc(msk));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (keep) list[base + __popc(msk & ((1u << lane) - 1))] = (unsigned)t;
        }
    }
}

// Rotates the 16 bytes of x down by r (byte s of the result = byte (s + r) mod 16 of x).
__device__ __forceinline__ uint4 rotate_bytes(uint4 x, int r)
{
    // branch-free (lane-dependent r): two predicated word rotations, then one funnel shift
    const bool r1 = (r & 4) != 0, r2 = (r & 8) != 0;
    unsigned a0 = r1 ? x.y : x.x, a1 = r1 ? x.z : x.y, a2 = r1 ? x.w : x.z, a3 = r1 ? x.x : x.w;
    const unsigned b0 = r2 ? a2 : a0, b1 = r2 ? a3 : a1, b2 = r2 ? a0 : a2, b3 = r2 ? a1 : a3;
    const int rb = (r & 3) * 8;
    uint4 y;
    y.x = __funnelshift_r(b0, b1, rb);
    y.y = __funnelshift_r(b1, b2, rb);
    y.z = __funnelshift_r(b2, b3, rb);
    y.w = __funnelshift_r(b3, b0, rb);
    return y;
}

// ---------------------------------------------------------------------- lower-bound scan
// The HBM-roofline step (A5): Alg. 9 line LowerBound_SIMD / Alg. 10 line
// LowerBound_DTW_SIMD, in two resolutions of the same iSAX word (variable
// cardinality):
//   coarse: every series of a tile, from its cardinality-16 pair bytes (4 KB per tile):
//           LB16 = sum_j PT[j][H_j] (round-down adds), PT[j][.] = T16[2j] + T16[2j+1]
//   fine:   the coarse survivors, from their 8-bit words (sym8, 16 B each):
//           LB8 = sum_s T8[s][sym_s] >= LB16 (T16 = min of T8 over the 16 refinements)
// Shared-memory scan table (64 KB, built by the prologue, copied per CTA), word v*64 + w:
//   w = 4j + c (c < 4): PT[j][v]      -- lane b reads pair (t + b) mod 8 at tile row t from
//                                        copy b >> 3: 32 distinct banks for any bytes
//   w = 32 + 16x + s  : T8[s][v]      -- lane l reads segment (s + l) mod 16 at step s from
//                                        copy l >> 4: 32 distinct banks for any symbols
// PRMT builds every byte address (v << 8 | w * 4) in one instruction.
constexpr int kScanWarps = 8;
constexpr int kScanTab = MESSI_CARD * 64;                 // floats per scan table
constexpr size_t kScanLutBytes = (size_t)kScanTab * sizeof(float);

// Coarse bounds acc[k] of the lane's 16 series 16*lane + k of a tile from its 8 rows
// (data[t] = tile row t, 16 bytes per lane).
__device__ __forceinline__ void coarse_acc_data(const uint4 (&data)[8], const char* lbase, int lane, float acc[16])
{
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 0.0f;
    const int bl = lane & 7, cp = lane >> 3;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const unsigned base = (unsigned)((4 * ((t + bl) & 7) + cp) * 4);
        const unsigned wv[4] = {data[t].x, data[t].y, data[t].z, data[t].w};
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
#pragma unroll
            for (int bb = 0; bb < 4; bb += 2) {
                const unsigned a0 = __byte_perm(wv[wi], base, 0x5504 | (bb << 4));
                const unsigned a1 = __byte_perm(wv[wi], base, 0x5504 | ((bb + 1) << 4));
                const float2 t = make_float2(*reinterpret_cast<const float*>(lbase + a0),
                                             *reinterpret_cast<const float*>(lbase + a1));
                const float2 r = fadd2_rd(make_float2(acc[wi * 4 + bb], acc[wi * 4 + bb + 1]), t);
                acc[wi * 4 + bb] = r.x;
                acc[wi * 4 + bb + 1] = r.y;
            }
        }
    }
}

// Coarse bounds acc[k] of the lane's 16 series 16*lane + k of tile `tile`.
__device__ __forceinline__ void coarse_acc(const uint4* __restrict__ tiles, long long tile, const char* lbase, int lane,
                                           float acc[16])
{
    const uint4* tp = tiles + tile * (MESSI_TILE_BYTES / 16) + lane;
    uint4 data[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) data[t] = __ldcs(tp + t * 32);
    coarse_acc_data(data, lbase, lane, acc);
}

// The lane's survivors (bit k: series 16*lane + k has LB16 <= thr and lies inside the
// collection -- series past the end exist in the last tile only: one 64-bit test per lane).
__device__ __forceinline__ unsigned coarse_mask(const float acc[16], float thr, long long N, long long tile, int lane)
{
    unsigned mask = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k)
        if (acc[k] <= thr) mask |= 1u << k;
    const long long left = N - (tile * MESSI_TILE_ROWS + lane * 16);
    if (left < 16) mask &= left > 0 ? (1u << left) - 1u : 0u;
    return mask;
}

// Compaction of the lanes' survivor masks into the warp's list surv (tile-local indices):
// each lane reserves its survivors' slots with one shared-memory atomic on the warp's counter
// (the list order across lanes is free: every later pass is order-free); returns their
// number (warp-uniform).
__device__ __forceinline__ int compact_mask(unsigned mask, unsigned short* surv, unsigned* wcnt, int lane)
{
    const int cnt = __popc(mask);
    if (lane == 0) *wcnt = 0u;
    __syncwarp();
    int off = cnt ? (int)atomicAdd(wcnt, (unsigned)cnt) : 0;
    __syncwarp();
    const int m = (int)*(volatile unsigned*)wcnt;
    while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        MESSI_CHECK(off < MESSI_TILE_ROWS);
        surv[off++] = (unsigned short)(lane * 16 + k);
    }
    __syncwarp();
    return m;
}

// Coarse bounds of the 512 series of tile `tile`; the series with LB16 <= thr are written to
// the warp's list surv (tile-local index); returns their number (warp-uniform).
__device__ __forceinline__ int scan_tile_coarse(const uint4* __restrict__ tiles, long long tile, const char* lbase,
                                                float thr, long long N, unsigned short* surv, unsigned* wcnt, int lane)
{
    float acc[16];
    coarse_acc(tiles, tile, lbase, lane, acc);
    return compact_mask(coarse_mask(acc, thr, N, tile, lane), surv, wcnt, lane);
}

// Fine bound of one series from its 8-bit word (16 symbols, segment s in byte s); the lane
// sums the segments in the order (s + lane) mod 16 (any order gives a valid bound).
__device__ __forceinline__ float fine_lb(uint4 w, const char* lbase, int lane)
{
    const int r = lane & 15;
    const uint4 x = rotate_bytes(w, r);  // byte s of x = symbol of segment (s + r) mod 16
    const unsigned xv[4] = {x.x, x.y, x.z, x.w};
    const unsigned cbase = 128u + 64u * (unsigned)(lane >> 4);
    float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int s = 0; s < 16; s += 2) {
        const unsigned b0 = cbase + 4u * (unsigned)((s + r) & 15), b1 = cbase + 4u * (unsigned)((s + 1 + r) & 15);
        const unsigned a0 = __byte_perm(xv[s >> 2], b0, 0x5504 | ((s & 3) << 4));
        const unsigned a1 = __byte_perm(xv[s >> 2], b1, 0x5504 | (((s + 1) & 3) << 4));
        acc = fadd2_rd(acc, make_float2(*reinterpret_cast<const float*>(lbase + a0),
                                        *reinterpret_cast<const float*>(lbase + a1)));
    }
    return __fadd_rd(acc.x, acc.y);
}

// Per-query scan for the DTW path (and the scan-throughput probe): the tiles the box filter
// listed, coarse + fine bounds, survivors (LB8 <= BSF0 * (1 + eps)) appended as (sorted
// position, LB8) with one atomicAdd per warp-round.
// Latency structure (a warp's tile is a chain of dependent loads: list entry -> tile rows ->
// 8-bit words -> append): the next tile's rows are loaded while this tile's fine pass runs,
// the list entry two tiles ahead; a tile's fine survivors are compacted in place in the
// warp's shared list and appended with ONE atomic per tile (not one per 32-series round).
__global__ void __launch_bounds__(32 * kScanWarps, 2) k_scan(const uint4* __restrict__ tiles, const uint4* __restrict__ sym8,
                                                             long long N, const float* __restrict__ tab_g, QState* st,
                                                             uint2* __restrict__ out, const unsigned* __restrict__ tlist,
                                                             unsigned epoch)
{
    extern __shared__ __align__(16) float tab_s[];
    __shared__ unsigned short surv_all[kScanWarps][MESSI_TILE_ROWS];
    __shared__ float lbs_all[kScanWarps][MESSI_TILE_ROWS];
    __shared__ unsigned wcnt_all[kScanWarps];
    for (int i = threadIdx.x; i < kScanTab / 4; i += blockDim.x)
        reinterpret_cast<float4*>(tab_s)[i] = reinterpret_cast<const float4*>(tab_g)[i];
    __syncthreads();
    const float thr = slack_up(ld_bsf_eff(st, epoch));  // linked shards: the shared BSF too
    if (blockIdx.x == 0 && threadIdx.x == 0) st->lbk_thr_bits = __float_as_uint(thr);  // for the DTW filter
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned short* surv = surv_all[warp];
    float* lbs = lbs_all[warp];
    const char* lbase = reinterpret_cast<const char*>(tab_s);
    const long long count = (long long)*(volatile unsigned*)&st->tile_count;
    const long long stride = (long long)gridDim.x * kScanWarps;
    long long it = (long long)blockIdx.x * kScanWarps + warp;
    if (it >= count) return;
    long long tl = (long long)tlist[it];
    long long tl_n = it + stride < count ? (long long)tlist[it + stride] : 0;
    uint4 data[8];
    {
        const uint4* tp = tiles + tl * (MESSI_TILE_BYTES / 16) + lane;
#pragma unroll
        for (int t = 0; t < 8; ++t) data[t] = __ldcs(tp + t * 32);
    }
    unsigned coarse = 0;
    for (; it < count; it += stride) {
        float acc[16];
        coarse_acc_data(data, lbase, lane, acc);
        const int m = compact_mask(coarse_mask(acc, thr, N, tl, lane), surv, &wcnt_all[warp], lane);
        coarse += (unsigned)m;
        // the next tile's rows and the list entry after it, in flight during the fine pass
        if (it + stride < count) {
            const uint4* tp = tiles + tl_n * (MESSI_TILE_BYTES / 16) + lane;
#pragma unroll
            for (int t = 0; t < 8; ++t) data[t] = __ldcs(tp + t * 32);
        }
        const long long tl_nn = it + 2 * stride < count ? (long long)tlist[it + 2 * stride] : 0;
        // rounds of 32 coarse survivors; the next round's 8-bit words are loaded before this
        // round's bounds are evaluated (DTW: ~40% of a tile survives the coarse bound); the
        // survivors of a round overwrite list slots already read (cnt <= i0)
        unsigned pos_n = lane < m ? (unsigned)(tl * MESSI_TILE_ROWS + surv[lane]) : 0u;
        uint4 w_n = lane < m ? sym8[pos_n] : make_uint4(0u, 0u, 0u, 0u);
        int cnt = 0;
        for (int i0 = 0; i0 < m; i0 += 32) {
            const bool v = i0 + lane < m;
            const unsigned pos = pos_n;
            const uint4 w = w_n;
            if (i0 + 32 < m) {
                const bool vn = i0 + 32 + lane < m;
                pos_n = vn ? (unsigned)(tl * MESSI_TILE_ROWS + surv[i0 + 32 + lane]) : 0u;
                if (vn) w_n = sym8[pos_n];
            }
            float lb = INFINITY;
            if (v) lb = fine_lb(w, lbase, lane);
            const bool ok = v && lb <= thr;
            const unsigned msk = __ballot_sync(0xffffffffu, ok);
            __syncwarp();  // every lane read its slot i0 + lane before the slots below are rewritten
            if (ok) {
                const int o = cnt + __popc(msk & ((1u << lane) - 1));
                surv[o] = (unsigned short)(pos - (unsigned)(tl * MESSI_TILE_ROWS));
                lbs[o] = lb;
            }
            cnt += __popc(msk);
        }
        if (cnt) {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(&st->cand_count, (unsigned)cnt);
            base = __shfl_sync(0xffffffffu, base, 0);
            __syncwarp();
            MESSI_CHECK(base + (unsigned)cnt <= (unsigned)N);
            for (int i = lane; i < cnt; i += 32)
                out[base + i] = make_uint2((unsigned)(tl * MESSI_TILE_ROWS + surv[i]), __float_as_uint(lbs[i]));
        }
        __syncwarp();  // the list is rewritten by the next tile's compaction
        tl = tl_n;
        tl_n = tl_nn;
    }
    if (lane == 0 && coarse) atomicAdd(&st->coarse_count, coarse);
}

// ------------------------------------------------- reverse envelope-PAA bound (DTW)
// LB_Keogh holds for either series against the envelope of the other (every
// point of a series lies on the warping path, matched to a point of the other within the
// reach), and the envelope-PAA reduction of P:1411 applies to either side too: per segment s
// of m points, Jensen on the convex f(q, L, U)^2 = max(0, q - U, L - q)^2 gives
//     sum_{i in s} dist(q_i, [L^x_i, U^x_i])^2 >= m dist(qbar_s, [Lbar^x_s, Ubar^x_s])^2,
// and the left side summed over s is the reverse LB_Keogh (<= DTW).  The rows' envelope PAA
// is kept per reach as 8-bit symbols whose regions contain it (renv, k_renv), so
//     LBrp(x) = m sum_s max(0, qbar_s - hi(u_s), lo(l_s) - qbar_s)^2 <= DTW(q, x).
//
// k_renv: for the row at sorted position p, u_s = symbol of an fp32 value >= mean(U^x over s)
// and l_s = symbol of one <= mean(L^x over s) (fp64 sums and quotient rounded up / down), so
// hi_w(u_s) > Ubar and lo_w(l_s) < Lbar (symbol_of puts x in [beta_{v-1}, beta_v)).
// out[2p] = u_0..u_15, out[2p+1] = l_0..l_15.  One warp per row staged in shared memory
// (row, U, L: 3n floats per warp), a lane per point for the clipped-window max / min.
__global__ void __launch_bounds__(256) k_renv(const float* __restrict__ rows, const unsigned* __restrict__ perm,
                                              long long N, int n, int R, const float* __restrict__ beta_g,
                                              uint4* __restrict__ out)
{
    extern __shared__ __align__(16) float rsm[];
    __shared__ float beta[256];
    for (int i = threadIdx.x; i < 255; i += blockDim.x) beta[i] = beta_g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    float* x = rsm + (size_t)w * 3 * n;
    float* U = x + n;
    float* L = U + n;
    const int m = n / MESSI_W;
    for (long long p = (long long)blockIdx.x * nw + w; p < N; p += (long long)gridDim.x * nw) {
        const float* src = rows + (long long)perm[p] * n;
        for (int j = lane * 4; j < n; j += 128)
            *reinterpret_cast<float4*>(x + j) = __ldg(reinterpret_cast<const float4*>(src + j));
        __syncwarp();
        for (int i = lane; i < n; i += 32) {
            const int a = max(0, i - R), b = min(n - 1, i + R);
            float u = x[a], l = x[a];
            for (int j = a + 1; j <= b; ++j) { u = fmaxf(u, x[j]); l = fminf(l, x[j]); }
            U[i] = u;
            L[i] = l;
        }
        __syncwarp();
        const int s = lane & 15;
        double acc = 0.0;
        float v;
        if (lane < 16) {
            for (int j = 0; j < m; ++j) acc = __dadd_ru(acc, (double)U[s * m + j]);
            v = __double2float_ru(__ddiv_ru(acc, (double)m));
        } else {
            for (int j = 0; j < m; ++j) acc = __dadd_rd(acc, (double)L[s * m + j]);
            v = __double2float_rd(__ddiv_rd(acc, (double)m));
        }
        unsigned word = (unsigned)symbol_of(v, beta) << (8 * (lane & 3));
        word |= __shfl_xor_sync(0xffffffffu, word, 1);
        word |= __shfl_xor_sync(0xffffffffu, word, 2);
        if ((lane & 3) == 0) reinterpret_cast<unsigned*>(out)[8 * p + (lane >> 2)] = word;
        __syncwarp();  // x, U, L are rewritten by the next row
    }
}

// The reverse envelope-PAA filter over the scan's candidates (cand, QState::cand_count): the
// ones with LBrp(x) <= the threshold go to out (QState::rcand_count) with LB = max(scan LB,
// LBrp) (rev_only, inspection: LBrp, every candidate kept).  Table per CTA (64 KB), word
// v * 64 + c: c = 16x + s: TU[s][v] = m max(0, qlo_s - hi_w(v))^2, c = 32 + 16x + s:
// TL[s][v] = m max(0, lo_w(v) - qhi_s)^2 (two copies x; fp32 rounded down, qlo / qhi the
// query's segment means rounded down / up) -- lane l reads segment (s + l) mod 16 of copy
// l >> 4, 32 distinct banks for any symbols.  At most one of TU, TL is nonzero per segment
// (u_s >= l_s), so TU + TL is the max form exactly.  A warp takes 128 candidates at a time
// (their rows' 32-byte words all in flight) and appends its survivors with one atomic.
constexpr int kRevTabBytes = 256 * 64 * 4;
__global__ void __launch_bounds__(256) k_rev_paa_filter(const uint2* __restrict__ cand, const uint4* __restrict__ renv,
                                                        const float* __restrict__ lo_w, const float* __restrict__ hi_w,
                                                        int m, QState* st, uint2* __restrict__ out, int rev_only)
{
    extern __shared__ __align__(16) float rtab[];
    __shared__ uint2 buf_all[8][128];
    for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
        const int v = i >> 4, s = i & 15;
        const float du = fmaxf(0.0f, __fsub_rd(st->qlo[s], hi_w[v]));  // hi_w(255) = +inf: 0
        const float dl = fmaxf(0.0f, __fsub_rd(lo_w[v], st->qhi[s]));  // lo_w(0) = -inf: 0
        const float tu = __fmul_rd((float)m, __fmul_rd(du, du)), tl = __fmul_rd((float)m, __fmul_rd(dl, dl));
        rtab[v * 64 + s] = tu;
        rtab[v * 64 + 16 + s] = tu;
        rtab[v * 64 + 32 + s] = tl;
        rtab[v * 64 + 48 + s] = tl;
    }
    __syncthreads();
    const float thr = __uint_as_float(st->lbk_thr_bits);
    const unsigned total = *(volatile unsigned*)&st->cand_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) st->rev_paa = 1u;
    const int lane = threadIdx.x & 31, r = lane & 15;
    uint2* buf = buf_all[threadIdx.x >> 5];
    const char* tb = reinterpret_cast<const char*>(rtab);
    const unsigned cbase = 64u * (unsigned)(lane >> 4);  // byte offset of copy x
    const unsigned nwarp = gridDim.x * (blockDim.x >> 5);
    for (unsigned k0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 128u; k0 < total; k0 += nwarp * 128u) {
        uint2 ce[4];
        bool ok[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const unsigned k = k0 + 32u * b + lane;
            ce[b] = k < total ? cand[k] : make_uint2(0u, 0x7f800000u);
            ok[b] = k < total && (rev_only || __uint_as_float(ce[b].y) <= thr);
        }
        uint4 wu[4], wl[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            wu[b] = ok[b] ? renv[2 * (size_t)ce[b].x] : make_uint4(0u, 0u, 0u, 0u);
            wl[b] = ok[b] ? renv[2 * (size_t)ce[b].x + 1] : make_uint4(0u, 0u, 0u, 0u);
        }
        int cnt = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint4 xu = rotate_bytes(wu[b], r), xl = rotate_bytes(wl[b], r);
            const unsigned uv[4] = {xu.x, xu.y, xu.z, xu.w}, lv[4] = {xl.x, xl.y, xl.z, xl.w};
            float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int s = 0; s < 16; s += 2) {
                // byte address of (symbol, column): symbol * 256 + (copy + segment) * 4
                const unsigned c0 = cbase + 4u * (unsigned)((s + r) & 15), c1 = cbase + 4u * (unsigned)((s + 1 + r) & 15);
                const unsigned au0 = __byte_perm(uv[s >> 2], c0, 0x5504 | ((s & 3) << 4));
                const unsigned au1 = __byte_perm(uv[s >> 2], c1, 0x5504 | (((s + 1) & 3) << 4));
                const unsigned al0 = __byte_perm(lv[s >> 2], c0 + 128u, 0x5504 | ((s & 3) << 4));
                const unsigned al1 = __byte_perm(lv[s >> 2], c1 + 128u, 0x5504 | (((s + 1) & 3) << 4));
                const float2 tu = make_float2(*reinterpret_cast<const float*>(tb + au0), *reinterpret_cast<const float*>(tb + au1));
                const float2 tl = make_float2(*reinterpret_cast<const float*>(tb + al0), *reinterpret_cast<const float*>(tb + al1));
                acc = fadd2_rd(fadd2_rd(acc, tu), tl);
            }
            const float rb = __fadd_rd(acc.x, acc.y);
            const bool pass = ok[b] && (rev_only || rb <= thr);
            const unsigned msk = __ballot_sync(0xffffffffu, pass);
            if (pass)
                buf[cnt + __popc(msk & ((1u << lane) - 1u))] =
                    make_uint2(ce[b].x, __float_as_uint(rev_only ? rb : fmaxf(__uint_as_float(ce[b].y), rb)));
            cnt += __popc(msk);
        }
        __syncwarp();
        if (cnt) {
            unsigned o = 0;
            if (lane == 0) o = atomicAdd(&st->rcand_count, (unsigned)cnt);
            o = __shfl_sync(0xffffffffu, o, 0);
            for (int i = lane; i < cnt; i += 32) out[o + i] = buf[i];
        }
        __syncwarp();
    }
}

// Inspection: the coarse (cardinality-16) bound of every series with the scan's own
// arithmetic (coarse_acc), scattered back to row order.
__global__ void __launch_bounds__(32 * kScanWarps) k_debug_coarse(const uint4* __restrict__ tiles, long long ntiles,
                                                                  long long N, const float* __restrict__ tab_g,
                                                                  const unsigned* __restrict__ perm, float* __restrict__ lb_all)
{
    extern __shared__ __align__(16) float tab_s[];
    for (int i = threadIdx.x; i < kScanTab / 4; i += blockDim.x)
        reinterpret_cast<float4*>(tab_s)[i] = reinterpret_cast<const float4*>(tab_g)[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long tl = (long long)blockIdx.x * kScanWarps + warp; tl < ntiles; tl += (long long)gridDim.x * kScanWarps) {
        float acc[16];
        coarse_acc(tiles, tl, reinterpret_cast<const char*>(tab_s), lane, acc);
        const long long id0 = tl * MESSI_TILE_ROWS + lane * 16;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (id0 + k < N) lb_all[perm[id0 + k]] = acc[k];
    }
}

}  // namespace messi
