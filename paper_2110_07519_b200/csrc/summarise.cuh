// summarise.cuh -- index build: breakpoints, iSAX summarisation (A1), approximate-search
// key (A2).  Paper: ConvertToiSAX inside CalculateiSAXSummaries, Alg. 3 P:696-718;
// PAA P:378-381; iSAX P:383-392.
#pragma once
#include "common.cuh"

namespace messi {

// Breakpoints beta_k = Phi^{-1}(k/256), k = 1..255 (reading R2: N(0,1) quantiles, the iSAX
// convention the paper cites at P:384-387), computed on the device with normcdfinv in fp64
// and rounded to nearest fp32.  Also the symbol boxes used by the lower-bound tables:
// box(v) = [beta32_v, beta32_{v+1}) widened outward by one fp32 ulp (lo_w, hi_w), so that
// the box contains the exact (unrounded) segment mean of every series that received v
// (keeps LB <= true distance although the PAA was rounded to fp32).
__global__ void k_breakpoints(float* beta32, float* lo_w, float* hi_w)
{
    __shared__ float b[256];
    int k = threadIdx.x;  // 256 threads
    if (k >= 1) {
        double p = (double)k / 256.0;
        b[k - 1] = __double2float_rn(normcdfinv(p));
        beta32[k - 1] = b[k - 1];
    }
    __syncthreads();
    int v = k;
    lo_w[v] = v == 0 ? -INFINITY : nextafterf(b[v - 1], -INFINITY);
    hi_w[v] = v == 255 ? INFINITY : nextafterf(b[v], INFINITY);
}

// Summaries in APPROXIMATE-SEARCH ORDER.  After the key sort every 8-bit iSAX word is
// stored at its sorted position p (row = perm[p]).  Consecutive positions share the leading
// bit planes of the interleaved key, i.e. they sit in the same subtree of the variable-
// cardinality iSAX tree; a tile of 512 consecutive positions plays the role of a
// leaf node, and its box -- per segment the min and max symbol of its members -- is the
// node's iSAX summary used to prune it (Alg. 7's FindDist).
//  * tiles (4 KB per 512 positions): the cardinality-16 word of each series (the top 4 bits
//    of its 8-bit symbols: iSAX is variable-cardinality by construction), as 8
//    pair bytes H_j = hi4(sym_2j) << 4 | hi4(sym_2j+1).  Skewed: block b = 16 series
//    (b < 32); tile row t (512 B) holds at byte 16b + k the pair byte j = (t + b) mod 8 of
//    series 16b + k.  A warp reading tile row t (lane b loads 16 B) holds all 8 pairs, each
//    for 4 lanes; with the pair table stored 4 times (copy b >> 3) the 32 lanes hit 32
//    distinct shared-memory banks whatever the bytes.
//  * sym8 [npad][16] u8: the full 8-bit words, series-major (one 16 B load per series) --
//    read only for the few series whose coarse bound survives.
//  * boxes [ntiles][32] u8: per segment min (bytes 0..15) and max (16..31) symbol.
__device__ __forceinline__ int tile_offset(int rr, int j)
{
    const int b = rr >> 4, k = rr & 15;
    const int t = (j - b) & 7;
    return t * 512 + b * 16 + k;
}

// One CTA (256 threads) summarises 512 rows per iteration (row order).  Lane (h2, s) of a
// warp takes segment s of row 2*pair + h2; the segment mean is an fp64 sequential sum
// (reading R5: the same operation order as the oracle, so PAA and symbols are bit-exact),
// divided by m and rounded once to fp32.  The approximate-search key interleaves the top
// 4 bits of the 16 symbols, most significant bit plane first: bits 63..48 are the root
// subtree of P:711 (one bit per segment), each further plane refines it like a split.
__global__ void __launch_bounds__(256) k_summarise(const float* __restrict__ rows, int64_t N, int n,
                                                   const float* __restrict__ beta_g, uint4* __restrict__ symrows_tmp,
                                                   int64_t ntiles, unsigned long long* __restrict__ keys,
                                                   unsigned* __restrict__ ids, float* __restrict__ paa)
{
    __shared__ float beta[256];
    __shared__ __align__(16) unsigned char srow[MESSI_TILE_ROWS * MESSI_W];
    const int m = n / MESSI_W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = lane & 15, h2 = lane >> 4;
    if (threadIdx.x < 255) beta[threadIdx.x] = beta_g[threadIdx.x];
    for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        __syncthreads();
        const int64_t row0 = tl * MESSI_TILE_ROWS;
#pragma unroll 2
        for (int pr = 0; pr < 32; ++pr) {
            const int rr = warp * 64 + pr * 2 + h2;
            const int64_t row = row0 + rr;
            const bool valid = row < N;
            int sym = 0;
            if (valid) {
                const float* x = rows + row * (int64_t)n + (int64_t)s * m;
                double sum = 0.0;
                if ((m & 3) == 0) {
                    for (int j = 0; j < m; j += 4) {
                        float4 v = __ldg(reinterpret_cast<const float4*>(x + j));
                        sum = __dadd_rn(sum, (double)v.x);
                        sum = __dadd_rn(sum, (double)v.y);
                        sum = __dadd_rn(sum, (double)v.z);
                        sum = __dadd_rn(sum, (double)v.w);
                    }
                } else {
                    for (int j = 0; j < m; ++j) sum = __dadd_rn(sum, (double)__ldg(x + j));
                }
                float p32 = __double2float_rn(__ddiv_rn(sum, (double)m));
                sym = symbol_of(p32, beta);
                if (paa) paa[row * MESSI_W + s] = p32;
            }
            srow[rr * MESSI_W + s] = (unsigned char)sym;
            unsigned long long key = 0;
#pragma unroll
            for (int bit = 7; bit >= 4; --bit) {
                unsigned plane = __ballot_sync(0xffffffffu, (sym >> bit) & 1);
                key = (key << 16) | ((plane >> (16 * h2)) & 0xffffu);
            }
            if (valid && s == 0) {
                keys[row] = key;
                ids[row] = (unsigned)row;
            }
        }
        __syncthreads();
        uint4* sdst = symrows_tmp + tl * MESSI_TILE_ROWS;
        for (int i = threadIdx.x; i < MESSI_TILE_ROWS; i += blockDim.x)
            sdst[i] = reinterpret_cast<const uint4*>(srow)[i];
    }
}

// Lays the summaries out in sorted order: one CTA (512 threads) per tile of 512 sorted
// positions gathers its rows' 8-bit words, writes them series-major (sym8), the skewed
// coarse tile and the box.
__global__ void __launch_bounds__(512) k_layout(const uint4* __restrict__ symrows_tmp, const unsigned* __restrict__ perm,
                                                int64_t N, uint4* __restrict__ tiles, uint4* __restrict__ sym8,
                                                unsigned char* __restrict__ boxes)
{
    __shared__ __align__(16) unsigned char tile[MESSI_TILE_BYTES];
    __shared__ unsigned bmin[MESSI_W], bmax[MESSI_W];
    const int i = threadIdx.x;
    const int64_t tl = blockIdx.x;
    const int64_t p = tl * MESSI_TILE_ROWS + i;
    if (i < MESSI_W) { bmin[i] = 255; bmax[i] = 0; }
    __syncthreads();
    const bool valid = p < N;
    const uint4 sr = valid ? symrows_tmp[perm[p]] : make_uint4(0, 0, 0, 0);
    sym8[p] = sr;
    const unsigned w[4] = {sr.x, sr.y, sr.z, sr.w};
#pragma unroll
    for (int j = 0; j < MESSI_W / 2; ++j) {
        const unsigned a = (w[(2 * j) >> 2] >> (8 * ((2 * j) & 3))) & 255u;
        const unsigned c = (w[(2 * j + 1) >> 2] >> (8 * ((2 * j + 1) & 3))) & 255u;
        tile[tile_offset(i, j)] = (unsigned char)((a & 0xF0u) | (c >> 4));
    }
#pragma unroll
    for (int sg = 0; sg < MESSI_W; ++sg) {
        const unsigned sym = (w[sg >> 2] >> (8 * (sg & 3))) & 255u;
        if (valid) {
            atomicMin(&bmin[sg], sym);
            atomicMax(&bmax[sg], sym);
        }
    }
    __syncthreads();
    if (i < MESSI_TILE_BYTES / 16) {
        uint4* dst = tiles + tl * (MESSI_TILE_BYTES / 16);
        dst[i] = reinterpret_cast<const uint4*>(tile)[i];
    }
    if (i < MESSI_W) {
        boxes[tl * 32 + i] = (unsigned char)bmin[i];
        boxes[tl * 32 + 16 + i] = (unsigned char)bmax[i];
    }
}

// Quantised copy of the rows for the refine's distance bound (DESIGN.md §7 "quantised
// rows"; not in the paper, whose refine reads every candidate's raw series, Alg. 9).
// Sorted position p (row perm[p]) gets n bytes c_i (two's-complement int8), c_i = rint(x_i / s),
// s = the smallest power of two with max_i |x_i| <= 127 s (so x_i / s and s * c_i are exact
// in fp32), and meta[p] = {s, e}, e >= ||x - s c||_2 (round-up fp32 sum of exact terms).  By the triangle
// inequality ||q - x|| >= ||q - s c|| - e: a lower bound of the true ED from n bytes instead
// of 4n.  Rows whose scale would leave the normal range, or with non-finite values, get
// e = +inf (never pruned by the bound).  One warp per position.
// The rows are read in ROW order (inv: sorted position of every row), so the 4n-byte reads
// stream linearly and only the n-byte writes scatter (round 1 gathered the rows in sorted
// order: 1.3 TB/s).
__global__ void k_invert_perm(const unsigned* __restrict__ perm, int64_t N, unsigned* __restrict__ inv)
{
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < N) inv[perm[p]] = (unsigned)p;
}

__global__ void __launch_bounds__(256) k_quantise(const float* __restrict__ rows, const unsigned* __restrict__ inv,
                                                  int64_t N, int64_t npad, int n, unsigned char* __restrict__ rows8,
                                                  float2* __restrict__ meta8)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < npad; r += warps) {
        if (r >= N) {  // padding positions (N .. npad-1): never candidates; zero them for determinism
            unsigned char* dst = rows8 + r * n;
            for (int j = lane * 16; j < n; j += 512) *reinterpret_cast<uint4*>(dst + j) = make_uint4(0, 0, 0, 0);
            if (lane == 0) meta8[r] = make_float2(1.0f, INFINITY);
            continue;
        }
        const int64_t p = inv[r];
        unsigned char* dst = rows8 + p * n;
        const float* x = rows + r * n;
        float mx = 0.0f;
        for (int j = lane * 4; j < n; j += 128) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(x + j));
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        bool usable = isfinite(mx);
        int k = 0;
        if (usable && mx > 0.0f) {
            int e;
            const float f = frexpf(mx, &e);           // mx = f * 2^e, f in [0.5, 1)
            k = (f * 128.0f <= 127.0f) ? e - 7 : e - 6;  // 127 * 2^k >= mx, smallest k
            if (k < -100 || k > 100) usable = false;
        }
        const float s = ldexpf(1.0f, k), sinv = ldexpf(1.0f, -k);  // exact powers of two
        // r = x - c s is exact in fp32 (|r| <= s / 2 and c s within a factor 2 of x when c != 0:
        // Sterbenz), and summing r^2 with round-UP fmas / adds gives a value >= the exact sum
        float err = 0.0f;
        for (int j = lane * 4; j < n; j += 128) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(x + j));
            const float xv[4] = {v.x, v.y, v.z, v.w};
            unsigned word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const float c = usable ? rintf(xv[b] * sinv) : 0.0f;  // |c| <= 127
                const float rr = xv[b] - c * s;
                err = __fmaf_ru(rr, rr, err);
                word |= ((unsigned)(int)c & 255u) << (8 * b);
            }
            *reinterpret_cast<unsigned*>(dst + j) = word;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) err = __fadd_ru(err, __shfl_xor_sync(0xffffffffu, err, o));
        if (lane == 0) meta8[p] = make_float2(s, usable ? __fsqrt_ru(err) : INFINITY);
    }
}

// Inspection: the quantised rows and their {scale, error bound} back in row order.
__global__ void k_unsort_q8(const unsigned char* __restrict__ rows8, const float2* __restrict__ meta8,
                            const unsigned* __restrict__ perm, int64_t N, int n, unsigned char* __restrict__ out,
                            float2* __restrict__ meta_out)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < N; p += warps) {
        const unsigned r = perm[p];
        for (int j = lane; j < n; j += 32) out[(int64_t)r * n + j] = rows8[p * n + j];
        if (lane == 0) meta_out[r] = meta8[p];
    }
}

// Inspection: the 8-bit words back in row order, out[row][16].
__global__ void k_detile(const uint4* __restrict__ sym8, const unsigned* __restrict__ perm, int64_t N,
                         uint4* __restrict__ out)
{
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < N) out[perm[p]] = sym8[p];
}

}  // namespace messi
