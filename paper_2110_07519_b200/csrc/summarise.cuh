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

// Two resolutions of the same iSAX words (the bit-prefix property of variable-cardinality
// iSAX, P:387-392 / P:408-417: the first b bits of an 8-bit symbol are the symbol at
// cardinality 2^b):
//  * symrows [Npad][16] u8: the full 8-bit word of every series, series-major (16 B).
//  * coarse tiles (4 KB per 512 series): the top nibble of every symbol, two segments per
//    byte -- byte = hi(sym_2p) << 4 | hi(sym_2p+1) for pair p -- 8 B per series, in a
//    skewed tile layout.  Block b = 16 series (b < 32); tile row t (512 B) holds, at byte
//    offset 16*b, the pair bytes of pair p = (t + b) mod 8 of block b's 16 series.  A warp
//    reading tile row t (lane b loads 16 B) therefore gets 8 different pairs across each
//    group of 8 lanes; with the coarse table replicated 4 times (copy b >> 3) the 32 lanes
//    hit 32 distinct shared-memory banks whatever the symbol values.
__device__ __forceinline__ int coarse_offset(int rr, int pair)
{
    int b = rr >> 4, k = rr & 15;
    int t = (pair - b) & 7;
    return t * 512 + b * 16 + k;
}

// One CTA (256 threads) summarises one tile of 512 rows per iteration.  Lane (h2, s) of a
// warp takes segment s of row 2*pair + h2; the segment mean is an fp64 sequential sum
// (reading R5: the same operation order as the oracle, so PAA and symbols are bit-exact),
// divided by m and rounded once to fp32.  The approximate-search key interleaves the top
// 4 bits of the 16 symbols, most significant bit plane first: bits 63..48 are the root
// subtree of P:711 (one bit per segment), each further plane refines it like a split.
__global__ void __launch_bounds__(256) k_summarise(const float* __restrict__ rows, int64_t N, int n,
                                                   const float* __restrict__ beta_g, uint4* __restrict__ tiles,
                                                   uint4* __restrict__ symrows, int64_t ntiles,
                                                   unsigned long long* __restrict__ keys, unsigned* __restrict__ ids,
                                                   float* __restrict__ paa)
{
    __shared__ float beta[256];
    __shared__ __align__(16) unsigned char tile[MESSI_TILE_BYTES];
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
            // pair byte: even lane s takes its odd neighbour's top nibble
            const int nb = __shfl_down_sync(0xffffffffu, sym, 1);
            if ((s & 1) == 0) tile[coarse_offset(rr, s >> 1)] = (unsigned char)((sym & 0xf0) | (nb >> 4));
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
        uint4* dst = tiles + tl * (MESSI_TILE_BYTES / 16);
        for (int i = threadIdx.x; i < MESSI_TILE_BYTES / 16; i += blockDim.x)
            dst[i] = reinterpret_cast<const uint4*>(tile)[i];
        uint4* sdst = symrows + tl * MESSI_TILE_ROWS;
        for (int i = threadIdx.x; i < MESSI_TILE_ROWS; i += blockDim.x)
            sdst[i] = reinterpret_cast<const uint4*>(srow)[i];
    }
}

// Inverse of the coarse layout (inspection): the pair bytes of every row, [N][8].
__global__ void k_detile_coarse(const unsigned char* __restrict__ tiles, int64_t N, unsigned char* __restrict__ out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * MESSI_PAIRS) return;
    int64_t row = i / MESSI_PAIRS;
    int pair = (int)(i % MESSI_PAIRS);
    out[i] = tiles[(row / MESSI_TILE_ROWS) * MESSI_TILE_BYTES + coarse_offset((int)(row % MESSI_TILE_ROWS), pair)];
}

}  // namespace messi
