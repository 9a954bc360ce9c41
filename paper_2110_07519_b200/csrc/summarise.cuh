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

// Tile layout of the symbols (what the LB scan streams).  A tile holds 512 consecutive
// rows = 32 blocks of 16 rows; block b = 2p + h (pair p = b>>1, half h = b&1).  Tile row t
// (512 B) holds, for every block b, the 16 symbols of segment s = (t + p) mod 16 of that
// block's 16 rows at byte offset 16*b.  So one warp reading tile row t with lane b loading
// 16 B gets 16 different segments across the 16 pairs -- what makes the LUT lookups of the
// scan bank-conflict free -- while the warp's load is one contiguous 512 B line set.
__device__ __forceinline__ int tile_offset(int rr, int s)
{
    int b = rr >> 4, k = rr & 15, p = b >> 1;
    int t = (s - p) & 15;
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
                                                   int64_t ntiles, unsigned long long* __restrict__ keys,
                                                   unsigned* __restrict__ ids, float* __restrict__ paa)
{
    __shared__ float beta[256];
    __shared__ __align__(16) unsigned char tile[MESSI_TILE_BYTES];
    const int m = n / MESSI_W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int s = lane & 15, h2 = lane >> 4;
    if (threadIdx.x < 255) beta[threadIdx.x] = beta_g[threadIdx.x];
    for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
        for (int i = threadIdx.x; i < MESSI_TILE_BYTES / 16; i += blockDim.x)
            reinterpret_cast<uint4*>(tile)[i] = make_uint4(0, 0, 0, 0);
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
                tile[tile_offset(rr, s)] = (unsigned char)sym;
            }
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
        __syncthreads();
    }
}

// Inverse of the tile layout, for inspection: sym[row][s].
__global__ void k_detile(const unsigned char* __restrict__ tiles, int64_t N, unsigned char* __restrict__ sym)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * MESSI_W) return;
    int64_t row = i / MESSI_W;
    int s = (int)(i % MESSI_W);
    int64_t tl = row / MESSI_TILE_ROWS;
    int rr = (int)(row % MESSI_TILE_ROWS);
    sym[i] = tiles[tl * MESSI_TILE_BYTES + tile_offset(rr, s)];
}

}  // namespace messi
