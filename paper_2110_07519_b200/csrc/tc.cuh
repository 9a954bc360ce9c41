// tc.cuh -- SURVEY 8(f) f4 (i) + (ii): the batched-query ED path on the tensor cores.
//
// One pass over the quantised rows answers up to kTcMaxQ queries at once (f4 (i): one
// summary pass for Q' queries).  The dense part is a real contraction: for every row x (int8
// c_x, scale s_x) and query q (int8 c_q, scale s_q, k_prologue_tc) the tensor cores compute
// D = sum_t c_x,t c_q,t EXACTLY (tcgen05.mma kind::i8, int32 accumulators in TMEM), so
//     ||q^ - x^||^2 = s_q^2 sum c_q^2 + s_x^2 sum c_x^2 - 2 s_q s_x D
// is known exactly, and with e_q >= ||q - q^||, e_x >= ||x - x^||
//     ||q - x|| >= ||q^ - x^|| - e_q - e_x  =: L.
// A row survives iff NOT (L > sqrt(thr)), thr = BSF0 (1 + eps) from the approximate search
// (A4) -- the same rule as the fused kernel's quantised bound, so the prescreen never drops
// the nearest neighbour.  The survivors (a few per query) are re-refined exactly: fp32 ED on
// the raw row, the fp64 canonical re-rank of every near tie (k_tc_verify: q8i_bound_pass +
// exact_pass of the fused path), i.e. "exactly re-refined in fp32" (north_star).
//
// Kernel k_ed_tc (persistent, one CTA per SM, 10 warps):
//   warp 0      TMA producer: 128-row tiles of rows8 (SWIZZLE_128B, n/128 boxes of 128 x 128
//               bytes per tile) into a kTcStages-deep shared-memory ring; the queries' int8
//               block (<= 256 x n bytes) once.
//   warp 1      MMA issuer (one lane): M = 128 rows x N = nq (padded to 16) queries, K = 32
//               bytes per tcgen05.mma, into one of two TMEM accumulators (2 x 256 columns).
//   warps 2..9  epilogue (two groups of four, one per TMEM accumulator, i.e. alternate tiles;
//               warp & 3 = its TMEM lane quarter): tcgen05.ld
//               of the tile's dot products (thread = TMEM lane = row), the survival test in
//               paired fp32 with directed rounding (every quantity that enters the threshold
//               is rounded towards keeping), survivors appended to the query's candidate list.
// Shapes: n = 128 or 256 (one or two 128-byte K chunks); <= 256 queries per pass.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "fused.cuh"

namespace messi {

constexpr int kTcRows = 128;     // rows per tile (UMMA M)
constexpr int kTcMaxQ = 256;     // queries per pass (UMMA N <= 256)
constexpr int kTcStages = 4;     // A-tile ring depth
constexpr int kTcEpiWarps = 8;   // two groups of four (one per accumulator, alternate tiles)
constexpr int kTcThreads = 32 * (2 + kTcEpiWarps);  // warp 0 TMA, warp 1 MMA, then the epilogue
constexpr unsigned kTcCandCap = 65536;  // candidates per query; more -> exhaustive fallback

__host__ __device__ inline size_t tc_smem_bytes(int n)
{
    const size_t kch = (size_t)n / 128;
    // 1024 B alignment slack + B block + A ring
    return 1024 + kch * kTcMaxQ * 128 + (size_t)kTcStages * kch * kTcRows * 128;
}

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, 128-byte-swizzled operand tile (the TMA SWIZZLE_128B layout): rows of 128 bytes,
// 8-row groups 1024 bytes apart (SBO), LBO unused (1), version 1 (sm_100), layout 2.
__device__ __forceinline__ unsigned long long sw128_desc(unsigned saddr)
{
    return (unsigned long long)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((unsigned long long)(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}

// tcgen05.mma kind::i8 instruction descriptor: D s32, A s8, B s8, both K-major, M = 128, N.
__device__ __forceinline__ unsigned idesc_i8(int N)
{
    return (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(N >> 3) << 17) | ((unsigned)(kTcRows >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(unsigned d_tmem, unsigned long long a_desc, unsigned long long b_desc, unsigned idesc,
                                        unsigned accumulate)
{
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(
            d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(unsigned long long* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// tcgen05.ld of 32 columns without the wait (the registers are valid only after tmem_wait).
__device__ __forceinline__ void tmem_ld32_async(unsigned taddr, int (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
// tcgen05.wait::ld, with v as read-write operands so no use of v is scheduled before it.
__device__ __forceinline__ void tmem_wait(int (&v)[32])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]),
                   "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]),
                   "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]),
                   "+r"(v[30]), "+r"(v[31])
                 :
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(unsigned taddr, int (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ----------------------------------------------------------------- build-time row terms
// Per sorted position p: {u = 2 s_x, v = s_x^2 sum c_x^2 - e_x^2 (rounded down), nw = -e_x, 0}
// -- the row's share of the survival test.  Rows whose quantisation is unusable (e_x = inf)
// get v = -inf, nw = 0: always kept.  One thread per position.
__global__ void k_tc_rowmeta(const unsigned char* __restrict__ rows8, const float2* __restrict__ meta8, long long npad,
                             int n, float4* __restrict__ tcm)
{
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npad) return;
    const float2 mt = meta8[p];
    const uint4* r = reinterpret_cast<const uint4*>(rows8 + p * n);
    int ss = 0;
    for (int c = 0; c < n / 16; ++c) {
        const uint4 w = __ldg(r + c);
        ss = dp4a_ss(w.x, w.x, ss); ss = dp4a_ss(w.y, w.y, ss);
        ss = dp4a_ss(w.z, w.z, ss); ss = dp4a_ss(w.w, w.w, ss);
    }
    float4 out;
    if (!(mt.y < INFINITY)) {
        out = make_float4(1.0f, -INFINITY, 0.0f, 0.0f);
    } else {
        const double s = (double)mt.x, e = (double)mt.y;
        const double v = s * s * (double)ss - e * e;  // exact product terms, one rounding
        out = make_float4(2.0f * mt.x, __double2float_rd(v - fabs(v) * 0x1p-50), -mt.y, 0.0f);
    }
    tcm[p] = out;
}

// ----------------------------------------------------------------------- prologue
// One CTA per query of the pass: arm, quantise (as the fused path), query PAA / key and the
// approximate-search window (for k_seed_batch's BSF0).
__global__ void __launch_bounds__(256) k_prologue_tc(const float* __restrict__ queries, int n,
                                                     const float* __restrict__ beta_g, const float* __restrict__ lo_w,
                                                     const float* __restrict__ hi_w,
                                                     const unsigned long long* __restrict__ skey, long long N, int window,
                                                     QState* st_all, unsigned* __restrict__ qc_all)
{
    extern __shared__ __align__(16) float q_s[];
    __shared__ unsigned long long qkey_s;
    const int b = blockIdx.x;
    QState* st = st_all + b;
    const float* q = queries + (size_t)b * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) q_s[i] = q[i];
    if (threadIdx.x == 0) arm_state(st);
    __syncthreads();
    quantise_query_block(q_s, n, qc_all + (size_t)b * (n / 4), st);
    prologue_block(q_s, n, -1, beta_g, lo_w, hi_w, nullptr, nullptr, nullptr, nullptr, &qkey_s, st);
    __syncthreads();
    const long long a = block_lower_bound(skey, N, qkey_s);
    if (threadIdx.x == 0) {
        const int len = (int)min((long long)window, N);
        st->qkey = qkey_s;
        st->window_start = (int)max(0LL, min(a - len / 2, N - len));
        st->window_len = len;
    }
}

// ----------------------------------------------------------------------- GEMM + test
// Query j's share of the survival test (fp32, directed rounding so the threshold only drops):
//   keep iff u_x D >= fma(v_x, r_j, fma(nw_x, b_j, a_j)),
//   a_j = (A_j - T_j^2) / s_j (down), r_j = 1 / s_j (exact), b_j = 2 T_j / s_j (up),
//   T_j = sqrt(thr_j) + e_q (up), A_j = s_j^2 sum c_q^2,  thr_j = BSF0_j (1 + eps).
// Derivation: u_x D s_j >= A_j + B_x - (T_j + e_x)^2  <=>  ||q^ - x^|| <= T_j + e_x  <=>  L <= sqrt(thr).
__device__ __forceinline__ float4 tc_query_params(const QState* st)
{
    const float thr = slack_up(__uint_as_float(*(volatile const unsigned*)&st->bsf_bits));
    const double sq = (double)st->q8s;
    const double T = (double)__fsqrt_ru(thr) * (1.0 + 0x1p-50) + st->q8e * (1.0 + 0x1p-50);
    if (!(T < (double)INFINITY)) return make_float4(-INFINITY, (float)(1.0 / sq), 0.0f, 0.0f);
    const double alpha = st->q8s2ss - T * T * (1.0 + 0x1p-50);
    const double a = alpha / sq, bq = 2.0 * T / sq;
    return make_float4(__double2float_rd(a - fabs(a) * 0x1p-50), (float)(1.0 / sq), __double2float_ru(bq * (1.0 + 0x1p-50)),
                       0.0f);
}

// The survival test of a row against two columns (queries j, j+1) at once, paired fp32 ops with
// directed rounding.  With X = float(D + C) (C = 1.5 * 2^23: exact for |D| < 2^22, n <= 256),
//   t1 = fma_rd(nw, b_j, a_j) <= a_j + nw b_j,   T2 = fma_rd(v, r_j, u C) <= v r_j + u C,
//   diff = (u X - T2) - t1  (round to nearest),
// u X - T2 >= u D - v r_j exactly, so whenever the exact test u D >= a_j + v r_j + nw b_j holds,
// the rounded diff is >= 0 (rounding is monotone and t1 is representable).  UNIFORM_R: every
// query of the pass has the same scale, so T2 is one value per row (hoisted).
constexpr float kTcMagic = 12582912.0f;  // 1.5 * 2^23
template <bool UNIFORM_R>
__device__ __forceinline__ float2 tc_diff2(int d0, int d1, float2 a, float2 r, float2 bq, float u, float v, float nw,
                                           float uC, float T2u)
{
    const float2 t1 = ffma2_rd(make_float2(nw, nw), bq, a);
    const float2 T2 = UNIFORM_R ? make_float2(T2u, T2u) : ffma2_rd(make_float2(v, v), r, make_float2(uC, uC));
    const float2 X = make_float2(__int_as_float(d0 + 0x4B400000), __int_as_float(d1 + 0x4B400000));
    const float2 y = ffma2(make_float2(u, u), X, make_float2(-T2.x, -T2.y));
    return fadd2(y, make_float2(-t1.x, -t1.y));
}

// Epilogue of one 32-column chunk: the chunk's max diff over its columns; survivors (diff >= 0,
// rare) appended to their queries' candidate lists.
template <bool UNIFORM_R>
__device__ __forceinline__ void tc_chunk(const int (&d)[32], int c0, const float* qa, const float* qr, const float* qb,
                                        float u, float v, float nw, float uC, float T2u, bool valid, long long pos, int nq,
                                        QState* st_all, unsigned* __restrict__ cand)
{
    float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
    for (int jj = 0; jj < 32; jj += 4) {
        const float2 df0 = tc_diff2<UNIFORM_R>(d[jj], d[jj + 1], *reinterpret_cast<const float2*>(qa + c0 + jj),
                                               *reinterpret_cast<const float2*>(qr + c0 + jj),
                                               *reinterpret_cast<const float2*>(qb + c0 + jj), u, v, nw, uC, T2u);
        const float2 df1 = tc_diff2<UNIFORM_R>(d[jj + 2], d[jj + 3], *reinterpret_cast<const float2*>(qa + c0 + jj + 2),
                                               *reinterpret_cast<const float2*>(qr + c0 + jj + 2),
                                               *reinterpret_cast<const float2*>(qb + c0 + jj + 2), u, v, nw, uC, T2u);
        m0 = max3f(m0, df0.x, df0.y);
        m1 = max3f(m1, df1.x, df1.y);
    }
    if (valid && fmaxf(m0, m1) >= 0.0f) {  // rare: a survivor in this chunk -- find and append it
        for (int jj = 0; jj < 32; jj += 2) {
            const float2 df = tc_diff2<UNIFORM_R>(d[jj], d[jj + 1], *reinterpret_cast<const float2*>(qa + c0 + jj),
                                                  *reinterpret_cast<const float2*>(qr + c0 + jj),
                                                  *reinterpret_cast<const float2*>(qb + c0 + jj), u, v, nw, uC, T2u);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = c0 + jj + h;
                if ((h ? df.y : df.x) >= 0.0f && j < nq) {
                    const unsigned slot = atomicAdd(&st_all[j].cand_count, 1u);
                    MESSI_CHECK(j < kTcMaxQ);
                    if (slot < kTcCandCap) cand[(size_t)j * kTcCandCap + slot] = (unsigned)pos;
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kTcThreads, 1) k_ed_tc(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB, long long ntc,
                                                          long long N, int n, int nq, const float4* __restrict__ tcm,
                                                          QState* st_all, unsigned* __restrict__ cand)
{
    extern __shared__ __align__(16) unsigned char tc_dsm[];
    __shared__ unsigned long long full_a[kTcStages], empty_a[kTcStages], full_b, tm_full[2], tm_empty[2];
    __shared__ unsigned tmem_base_s;
    __shared__ __align__(16) float qa_s[kTcMaxQ], qr_s[kTcMaxQ], qb_s[kTcMaxQ];  // a_j, r_j, b_j
    __shared__ int nonuniform_s;
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<size_t>(tc_dsm) + 1023) & ~(size_t)1023);
    const int kch = n / 128;
    unsigned char* B_s = base;                                   // kch x [256 rows x 128 B]
    unsigned char* A_s = B_s + (size_t)kch * kTcMaxQ * 128;      // kTcStages x kch x [128 rows x 128 B]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Nm = max(16, (nq + 15) & ~15);  // MMA N
    const unsigned stage_bytes = (unsigned)kch * kTcRows * 128;

    if (threadIdx.x == 0) {
        nonuniform_s = 0;
        for (int s = 0; s < kTcStages; ++s) { mbar_init(&full_a[s], 1); mbar_init(&empty_a[s], 1); }
        mbar_init(&full_b, 1);
        for (int a = 0; a < 2; ++a) { mbar_init(&tm_full[a], 1); mbar_init(&tm_empty[a], kTcEpiWarps / 2); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // two accumulators of 256 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    for (int j = threadIdx.x; j < kTcMaxQ; j += blockDim.x) {
        // columns past the batch: a = +inf makes rhs +inf, diff -inf (never kept)
        const float4 qp = j < nq ? tc_query_params(st_all + j) : make_float4(INFINITY, 1.0f, 0.0f, 0.0f);
        qa_s[j] = qp.x;
        qr_s[j] = qp.y;
        qb_s[j] = qp.z;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nq; j += blockDim.x)
        if (qr_s[j] != qr_s[0]) nonuniform_s = 1;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = tmem_base_s;
    const bool uniform_r = nonuniform_s == 0;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            mbar_expect_tx(&full_b, (unsigned)kch * kTcMaxQ * 128);
            for (int c = 0; c < kch; ++c) tma_load_2d(B_s + (size_t)c * kTcMaxQ * 128, &tmB, c * 128, 0, &full_b);
            long long it = 0;
            for (long long t = blockIdx.x; t < ntc; t += gridDim.x, ++it) {
                const int s = (int)(it % kTcStages);
                const unsigned ph = (unsigned)((it / kTcStages) & 1);
                mbar_wait(&empty_a[s], ph ^ 1u);
                mbar_expect_tx(&full_a[s], stage_bytes);
                unsigned char* dst = A_s + (size_t)s * stage_bytes;
                for (int c = 0; c < kch; ++c)
                    tma_load_2d(dst + (size_t)c * kTcRows * 128, &tmA, c * 128, (int)(t * kTcRows), &full_a[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            const unsigned idesc = idesc_i8(Nm);
            mbar_wait(&full_b, 0);
            long long it = 0;
            for (long long t = blockIdx.x; t < ntc; t += gridDim.x, ++it) {
                const int s = (int)(it % kTcStages);
                const unsigned ph = (unsigned)((it / kTcStages) & 1);
                const int acc = (int)(it & 1);
                const unsigned aph = (unsigned)((it >> 1) & 1);
                mbar_wait(&tm_empty[acc], aph ^ 1u);
                mbar_wait(&full_a[s], ph);
                tc_fence_after();
                const unsigned a0 = smem_u32(A_s + (size_t)s * stage_bytes), b0 = smem_u32(B_s);
                for (int c = 0; c < kch; ++c) {
                    const unsigned long long ad = sw128_desc(a0 + c * kTcRows * 128);
                    const unsigned long long bd = sw128_desc(b0 + c * kTcMaxQ * 128);
#pragma unroll
                    for (int k = 0; k < 4; ++k)  // 32 bytes of K per instruction: +2 in the 16-byte address field
                        umma_i8(tmem + (unsigned)acc * 256u, ad + 2ull * k, bd + 2ull * k, idesc, (c | k) != 0);
                }
                umma_commit(&empty_a[s]);
                umma_commit(&tm_full[acc]);
            }
        }
    } else {  // ---------------- epilogue: group g = (warp - 2) / 4 takes the tiles of accumulator g (every
              // other tile), warp & 3 is its TMEM lane quarter; the two groups overlap their tiles
        const int qtr = warp & 3, grp = (warp - 2) >> 2;
        const int nchunks = (Nm + 31) / 32;
        long long it = grp;
        long long t = (long long)blockIdx.x + (long long)grp * gridDim.x;
        const long long step = 2LL * gridDim.x;
        // the row terms (u, v, nw, 0) of this thread's row, loaded one tile ahead
        float4 rm_next = t < ntc ? tcm[t * kTcRows + qtr * 32 + lane] : make_float4(0, 0, 0, 0);
        for (; t < ntc; t += step, it += 2) {
            const int acc = grp;
            const unsigned aph = (unsigned)((it >> 1) & 1);
            const long long pos = t * kTcRows + qtr * 32 + lane;
            const bool valid = pos < N;
            const float4 rm = rm_next;
            if (t + step < ntc) rm_next = tcm[(t + step) * kTcRows + qtr * 32 + lane];
            const float u = rm.x, v = rm.y, nw = rm.z, uC = rm.x * kTcMagic;
            const float T2u = __fmaf_rd(v, qr_s[0], uC);  // the row's T2 when every query has scale 1/qr_s[0]
            mbar_wait(&tm_full[acc], aph);
            tc_fence_after();
            const unsigned taddr = tmem + ((unsigned)(qtr * 32) << 16) + (unsigned)acc * 256u;
            // two chunks in flight: the next chunk's tcgen05.ld overlaps this chunk's test
            int dA[32], dB[32];
            auto test = [&](const int (&d)[32], int c0) {
                if (uniform_r)
                    tc_chunk<true>(d, c0, qa_s, qr_s, qb_s, u, v, nw, uC, T2u, valid, pos, nq, st_all, cand);
                else
                    tc_chunk<false>(d, c0, qa_s, qr_s, qb_s, u, v, nw, uC, T2u, valid, pos, nq, st_all, cand);
            };
            tmem_ld32_async(taddr, dA);
            tmem_wait(dA);
            for (int ch = 0; ch < nchunks; ch += 2) {
                const bool more = ch + 1 < nchunks;
                if (more) tmem_ld32_async(taddr + (unsigned)((ch + 1) * 32), dB);
                test(dA, ch * 32);
                if (!more) break;
                tmem_wait(dB);
                const bool more2 = ch + 2 < nchunks;
                if (more2) tmem_ld32_async(taddr + (unsigned)((ch + 2) * 32), dA);
                test(dB, (ch + 1) * 32);
                if (!more2) break;
                tmem_wait(dA);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tm_empty[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
    }
}

// ------------------------------------------------------------------- exact re-refine
// One warp per query: the candidate list in rounds of 32 through the fused path's own
// quantised bound (q8i_bound_pass, against the current BSF) and exact pass (fp32 ED on the raw
// row, fp64 canonical re-rank of every near tie, best_update).  A query whose list overflowed
// the capacity is answered by every row instead (exhaustive exact pass; correct, slow).
__global__ void __launch_bounds__(128) k_tc_verify(const float* __restrict__ queries, int n, int nq,
                                                   const unsigned* __restrict__ cand, const unsigned char* __restrict__ rows8,
                                                   const float2* __restrict__ meta8, const unsigned* __restrict__ qc_all,
                                                   const unsigned* __restrict__ perm, const float* __restrict__ rows,
                                                   long long N, QState* st_all)
{
    extern __shared__ __align__(16) float tv_dsm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    const size_t per_warp = fused_qpad(n) + (size_t)n / 4;  // floats: padded query + quantised query words
    float* q_p = tv_dsm + (size_t)w * per_warp;
    unsigned* qc_w = reinterpret_cast<unsigned*>(q_p + fused_qpad(n));
    const int b = blockIdx.x * wpb + w;
    if (b >= nq) return;
    QState* st = st_all + b;
    for (int i = lane; i < n; i += 32) q_p[i + 4 * (i >> 5)] = queries[(size_t)b * n + i];
    for (int i = lane; i < n / 4; i += 32) qc_w[i] = qc_all[(size_t)b * (n / 4) + i];
    __syncwarp();
    Q8Query qq;
    qq.sq = (double)st->q8s;
    qq.e = st->q8e;
    qq.s2ss = st->q8s2ss;
    PeerSet none{nullptr, 0, 0u};
    const unsigned total = *(volatile unsigned*)&st->cand_count;
    const bool overflow = total > kTcCandCap;
    const long long cnt = overflow ? N : (long long)total;
    unsigned exact = 0;
    for (long long i0 = 0; i0 < cnt; i0 += 32) {
        const bool v = i0 + lane < cnt;
        unsigned pos = 0;
        if (v) pos = overflow ? (unsigned)(i0 + lane) : cand[(size_t)b * kTcCandCap + i0 + lane];
        const float thr = slack_up(ld_bsf(st));
        const unsigned keep = overflow ? __ballot_sync(0xffffffffu, v)
                                       : q8i_bound_pass((int)min(32LL, cnt - i0), pos, rows8, meta8, n,
                                                        reinterpret_cast<const uint4*>(qc_w), qq, thr, lane);
        exact += __popc(keep);
        if (keep) exact_pass<false, false>(keep, pos, perm, rows, n, q_p, st, none, b, nullptr, 1, lane);
    }
    if (lane == 0) {
        st->refined = (unsigned)min(cnt, (long long)0xffffffffLL);
        st->exact = exact;
        st->tiles_scanned = (unsigned)((N + MESSI_TILE_ROWS - 1) / MESSI_TILE_ROWS);  // every row was bounded
    }
}

}  // namespace messi
