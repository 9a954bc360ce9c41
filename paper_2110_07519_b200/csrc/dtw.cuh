// dtw.cuh -- real-distance engines: fp32 ED (warp), fp32/fp64 banded DTW (warp
// wavefront), fp32 banded DTW (one thread per candidate: band in registers, or strips of
// candidate rows for any reach).
#pragma once
#include "common.cuh"

#include <utility>

namespace messi {

// Squared ED in fp32, one warp: lane handles float4 chunks lane*4 + 128k, then a butterfly
// sum (commutative pairs -> every lane holds the same total).  RealDist_SIMD.
__device__ __forceinline__ float ed2_warp(const float* __restrict__ q_s, const float* __restrict__ c, int n, int lane)
{
    float acc = 0.0f;
    for (int j = lane * 4; j < n; j += 128) {
        float4 cv = __ldg(reinterpret_cast<const float4*>(c + j));
        float4 qv = *reinterpret_cast<const float4*>(q_s + j);
        float d;
        d = qv.x - cv.x; acc = fmaf(d, d, acc);
        d = qv.y - cv.y; acc = fmaf(d, d, acc);
        d = qv.z - cv.z; acc = fmaf(d, d, acc);
        d = qv.w - cv.w; acc = fmaf(d, d, acc);
    }
    return warp_sum(acc);
}

template <typename T> __device__ __forceinline__ T inf_of();
template <> __device__ __forceinline__ float inf_of<float>() { return INFINITY; }
template <> __device__ __forceinline__ double inf_of<double>() { return (double)INFINITY; }

// Three-input fp32 minimum: one FMNMX3 on sm_100a (min is exact, so the DP values are the
// same as with two fminf).
__device__ __forceinline__ float min3f(float a, float b, float c)
{
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__device__ __forceinline__ float cell_cost_add(float q, float c, float m) { float d = q - c; return fmaf(d, d, m); }
__device__ __forceinline__ double cell_cost_add(float q, float c, double m)
{
    double d = __dsub_rn((double)q, (double)c);
    return __dadd_rn(__dmul_rn(d, d), m);
}

// Banded DTW (reach r: |i - j| <= r; D(0,0) = cost; D = cost + min(diag, up, left)),
// P:323-324 / P:1379, one warp, anti-diagonal wavefront: anti-diagonal t = i + j holds the
// cells i in [ilo, ihi]; lanes take them 32 at a time; three rotating buffers indexed by i
// (buf: 3*n of T).  Cells just outside the band are written +inf so later reads see +inf.
// q and c must already be in shared memory (the step loop is latency-bound otherwise).
// With T = double and cell_cost_add's _rn ops every cell is fl(fl(d*d) + min(...)): the
// same value in any evaluation order, i.e. bit-identical to a row-by-row DP.
template <typename T>
__device__ T dtw_warp(const float* __restrict__ q, const float* __restrict__ c, int n, int r, T* buf, int lane)
{
    T* Dm2 = buf;
    T* Dm1 = buf + n;
    T* D0 = buf + 2 * n;
    const T INF = inf_of<T>();
    for (int t = 0; t <= 2 * n - 2; ++t) {
        const int ilo = max(max(0, t - (n - 1)), (t - r + 1) >> 1);
        const int ihi = min(min(n - 1, t), (t + r) >> 1);
        for (int i = ilo - 1 + lane; i <= ihi + 1; i += 32) {
            if (i < 0 || i >= n) continue;
            T val = INF;
            if (i >= ilo && i <= ihi) {
                const int j = t - i;
                T mn;
                if (t == 0) {
                    mn = (T)0;
                } else {
                    T up = i > 0 ? Dm1[i - 1] : INF;
                    T left = j > 0 ? Dm1[i] : INF;
                    T diag = (i > 0 && j > 0) ? Dm2[i - 1] : INF;
                    mn = diag < up ? diag : up;
                    mn = left < mn ? left : mn;
                }
                val = cell_cost_add(q[i], c[j], mn);
            }
            D0[i] = val;
        }
        __syncwarp();
        T* tmp = Dm2;
        Dm2 = Dm1;
        Dm1 = D0;
        D0 = tmp;
    }
    T out = Dm1[n - 1];
    __syncwarp();
    return out;
}

// Same banded DTW with the anti-diagonal in REGISTERS: for reach r <= 30 an anti-diagonal
// holds at most r+1 <= 31 band cells, so lane l owns cell i = ilo(t) + l of anti-diagonal t.
// Its three predecessors live on anti-diagonals t-1 (up, left) and t-2 (diag) in lanes
// shifted by the (warp-uniform) change of ilo: three shuffles per step, no shared memory,
// no barriers.  Lanes outside [ilo, ihi] hold +inf, which is what out-of-band reads must
// see.  Same cell arithmetic as dtw_warp (cell_cost_add), so the fp64 result is identical.
constexpr int kShflMaxReach = 30;

template <typename T>
__device__ T dtw_warp_shfl(const float* __restrict__ q, const float* __restrict__ c, int n, int r, int lane)
{
    const T INF = inf_of<T>();
    T cur = INF, prev = INF;  // this lane's cell on anti-diagonals t-1 and t-2
    int ilo1 = 0, ilo2 = 0;   // ilo(t-1), ilo(t-2)
    for (int t = 0; t <= 2 * n - 2; ++t) {
        const int ilo = max(max(0, t - (n - 1)), (t - r + 1) >> 1);
        const int ihi = min(min(n - 1, t), (t + r) >> 1);
        const int i = ilo + lane, j = t - i;
        const int su = lane + (ilo - ilo1) - 1;  // (i-1, j)   on t-1
        const int sl = lane + (ilo - ilo1);      // (i,   j-1) on t-1
        const int sd = lane + (ilo - ilo2) - 1;  // (i-1, j-1) on t-2
        T up = __shfl_sync(0xffffffffu, cur, su & 31);
        T left = __shfl_sync(0xffffffffu, cur, sl & 31);
        T diag = __shfl_sync(0xffffffffu, prev, sd & 31);
        up = su >= 0 && su < 32 ? up : INF;
        left = sl < 32 ? left : INF;
        diag = sd >= 0 && sd < 32 ? diag : INF;
        T mn = diag < up ? diag : up;
        mn = left < mn ? left : mn;
        if (t == 0) mn = (T)0;
        const bool valid = i <= ihi;
        const T val = valid ? cell_cost_add(q[valid ? i : 0], c[valid ? j : 0], mn) : INF;
        prev = cur;
        cur = val;
        ilo2 = ilo1;
        ilo1 = ilo;
    }
    return __shfl_sync(0xffffffffu, cur, 0);  // t = 2n-2: ilo = n-1, lane 0 holds D(n-1, n-1)
}

// Dispatch: register wavefront when the band fits a warp, shared-memory wavefront otherwise.
template <typename T>
__device__ __forceinline__ T dtw_warp_any(const float* __restrict__ q, const float* __restrict__ c, int n, int r,
                                          T* buf, int lane)
{
    return r <= kShflMaxReach ? dtw_warp_shfl<T>(q, c, n, r, lane) : dtw_warp<T>(q, c, n, r, buf, lane);
}

// Banded DTW in fp32, ONE THREAD per candidate, band of width W = 2R+1 held in registers.
// Row i, band slot d <-> column j = i + d - R.  D[d] is updated in place left to right:
// before the update D[d] = D(i-1, j-1), D[d+1] = D(i-1, j), `left` = D(i, j-1).  Columns
// outside [0, n) read c = +inf, so their cells are +inf without branches.  Rows advance
// four at a time over a sliding register window cw[e] = c[i - R + e], e < W + 3; the four
// columns entering the window each step come from two aligned float4 blocks held in
// registers, the block after them being loaded one step ahead.
// Early abandon (Alg. 10's "< BSF" test, exact for non-negative costs): after rows i..i+3
// every warping path still has to cross row i+3 (>= its row minimum) and every column
// j >= i+R+4 (>= that column's LB_Keogh term against the query envelope), so
// the candidate is dropped when rowmin + (LBK_total - LBK of the columns seen) exceeds the
// threshold (the UCR-suite cumulative bound, with fp32 margins of 2^-10).
template <int R>
struct DtwThread {
    static constexpr int W = 2 * R + 1;
    static constexpr int CW = W + 3;
    static constexpr int T = R & 3;  // offset of column i+R+4 inside its float4 block
    float D[W + 1];
    float cw[CW];
    float4 hold, h2;
    float seen;     // sum of the LB_Keogh terms of the columns that entered the window
    float seen_lo;  // the same before the last step's four columns: columns < i + R (i after step4)
    int i;

    __device__ __forceinline__ static float4 block(const float* __restrict__ c, int n, int b)
    {
        return (b >= 0 && 4 * b < n) ? __ldg(reinterpret_cast<const float4*>(c) + b)
                                     : make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
    }

    __device__ __forceinline__ static float lbk_term(float v, float u, float l)
    {
        float d = v > u ? v - u : (v < l ? v - l : 0.0f);
        return d * d;
    }

    // head_lbk: the LB_Keogh terms of columns 0 .. R+3 (the first window), summed by the
    // filter kernel (any summation order: the tail bound carries 2^-10 margins)
    __device__ __forceinline__ void start(const float* __restrict__ c, int n, float head_lbk)
    {
#pragma unroll
        for (int d = 0; d <= W; ++d) D[d] = INFINITY;
        D[R] = 0.0f;  // virtual D(-1, -1) = 0 so that D(0, 0) = cost(0, 0)
        constexpr int NB = (R + 4 + 3) / 4;  // blocks covering columns 0 .. R+3
        float f[NB * 4];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            float4 v = block(c, n, b);
            f[4 * b] = v.x; f[4 * b + 1] = v.y; f[4 * b + 2] = v.z; f[4 * b + 3] = v.w;
        }
        seen = head_lbk;
        seen_lo = 0.0f;
#pragma unroll
        for (int e = 0; e < CW; ++e) {
            const int j = e - R;
            cw[e] = j < 0 ? INFINITY : f[j];
        }
        hold = block(c, n, (R + 4) >> 2);
        h2 = block(c, n, ((R + 4) >> 2) + 1);
        i = 0;
    }

    // Rows i..i+3.  Returns min over the band of row i+3 (+inf cells included).
    __device__ __forceinline__ float step4(const float* __restrict__ c, int n, const float* __restrict__ q_s,
                                           const float* __restrict__ U, const float* __restrict__ L)
    {
        const int p = i + R + 4;  // first column entering the window
        const float4 nx4 = block(c, n, (p >> 2) + 2);  // for the next step
        const float hv[8] = {hold.x, hold.y, hold.z, hold.w, h2.x, h2.y, h2.z, h2.w};
        float nx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) nx[u] = hv[T + u];
        const float4 qv = *reinterpret_cast<const float4*>(q_s + i);
        const float qq[4] = {qv.x, qv.y, qv.z, qv.w};
        // rows (0, 1) then (2, 3), each pair as a skewed wavefront: row u+1 runs two cells
        // behind row u (its cell c needs row u's cells c and c+1), so one paired FFMA2
        // finishes a cell of each row (Blackwell f32x2: half the FMA-pipe issue).  In-place:
        // row u+1 overwrites D[c] only after row u has read it.
#pragma unroll
        for (int u = 0; u < 4; u += 2) {
            float lu = INFINITY, lv = INFINITY;
#pragma unroll
            for (int dd = 0; dd < W + 2; ++dd) {
                const int a = dd, c2 = dd - 2;
                if (a < W && c2 >= 0) {
                    const float mna = min3f(D[a], D[a + 1], lu);
                    const float mnc = min3f(D[c2], D[c2 + 1], lv);
                    const float dfa = qq[u] - cw[a + u];
                    const float dfc = qq[u + 1] - cw[c2 + u + 1];
                    const float2 r = ffma2(make_float2(dfa, dfc), make_float2(dfa, dfc), make_float2(mna, mnc));
                    lu = r.x;
                    lv = r.y;
                    D[a] = lu;
                    D[c2] = lv;
                } else if (a < W) {
                    const float mna = min3f(D[a], D[a + 1], lu);
                    const float dfa = qq[u] - cw[a + u];
                    lu = fmaf(dfa, dfa, mna);
                    D[a] = lu;
                } else {
                    const float mnc = min3f(D[c2], D[c2 + 1], lv);
                    const float dfc = qq[u + 1] - cw[c2 + u + 1];
                    lv = fmaf(dfc, dfc, mnc);
                    D[c2] = lv;
                }
            }
        }
        float mn = D[0];
#pragma unroll
        for (int d = 1; d + 1 < W; d += 2) mn = min3f(mn, D[d], D[d + 1]);
        if ((W & 1) == 0) mn = fminf(mn, D[W - 1]);
        seen_lo = seen;
#pragma unroll
        for (int e = 0; e < CW - 4; ++e) cw[e] = cw[e + 4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            cw[CW - 4 + u] = nx[u];
            const int j = p + u;
            if (j < n) seen += lbk_term(nx[u], U[j], L[j]);
        }
        hold = h2;
        h2 = nx4;
        i += 4;
        return mn;
    }

    __device__ __forceinline__ float result() const { return D[R]; }
};


// ------------------------------------------------------------------ strip DTW (any reach)
// Banded DTW in fp32, one thread per candidate, for ANY reach R >= H - 1, with O(H)
// registers.  DTW is symmetric in its two series, so the thread walks the CANDIDATE's points
// as rows j (read from global memory, H at a time) and the query's as columns i:
//     D(j, i) = (q_i - c_j)^2 + min(D(j-1, i-1), D(j-1, i), D(j, i-1)),  |i - j| <= R,
// the same cell arithmetic as DtwThread (fl(d*d + min) with d = fl(q_i - c_j)), so the fp32
// value of every cell -- and the distance -- is the same as there.
// Rows go in strips of H.  Inside a strip row u runs one column behind row u-1 (at step t
// row u is at column j0 - R + t - u), so the H cells of a step are independent (paired
// FFMA2) and each needs only values of the previous two steps, held in registers:
//     left = row u at t-1, up = row u-1 at t-1, diag = row u-1 at t-2.
// Row 0 reads the previous strip's last row, and row H-1 writes this strip's, from/to a
// per-thread boundary array B of 2R+2 slots in shared memory (slot x of strip j0 = column
// j0 - R - 1 + x; thread-interleaved, so conflict-free); slot 2R+1 stays +inf (the cell
// right of the band).  The query comes from shared memory padded with +inf outside
// [0, n) (so cells outside the matrix are +inf), in 8 lane-interleaved copies.  Row u is
// active at steps [2u, 2u + 2R]: the first 2H-2 steps (prologue) and the last 2H-2
// (epilogue) are unrolled with their active rows fixed at compile time, the 2R - 2H + 3
// steps between them run in H-step chunks (the query window rotates through H registers)
// plus REM = (2R - 2H + 3) mod H single steps (a template parameter).
constexpr int kStripThreads = 128;  // threads per CTA (64 for reaches whose boundary arrays need it)
// Lane copies of the padded query pairs (q[c], q[c-1]): 16 (a 64-bit load serves a half-warp
// per wavefront: conflict-free) when they fit beside the boundary arrays, else 8 (chosen
// per launch; strip_qcopies in refine.cuh).

template <int... Is, class F>
__device__ __forceinline__ void static_for_impl(std::integer_sequence<int, Is...>, F&& f)
{
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f)
{
    static_for_impl(std::make_integer_sequence<int, N>{}, f);
}

template <int H>
struct DtwStrip {
    float S[2][H];  // row values at steps of parity 0 / 1
    float2 Qp[H];   // query window: Qp[t % H] = (q[c], q[c-1]), c = row 0's column at step t
    float cv[H];    // candidate points of the strip's rows
    float2 ncv[H / 2];  // (-cv[2p], -cv[2p+1]): row pairs subtract with one FADD2
    float bprev;    // row 0's diagonal input (boundary slot of the previous step)
    float rmin;     // min over row H-1 (the strip's last row)

    // One step t (compile-time facts: PH = t % H, PAR = t & 1, active rows [LO, HI],
    // whether row H-1 writes the boundary).  bsrc: boundary slot t+1 (read when row 0 is
    // active), q: the pair (q[c], q[c-1]) at column c = j0 - R + t, bdst: boundary slot t - 2H + 2.
    // Rows go in aligned pairs (2p, 2p+1): the pair loaded u steps ago holds exactly the two
    // query points rows u and u+1 need now, so both differences are one FADD2 and both cells
    // one FFMA2.
    template <int PH, int PAR, int LO, int HI>
    __device__ __forceinline__ void step(const float* bsrc, const float2* q, float* bdst)
    {
        float up0 = 0.0f, dg0 = 0.0f;
        if constexpr (LO == 0) {
            up0 = *bsrc;
            dg0 = bprev;
            bprev = up0;
        }
        Qp[PH] = *q;
        float nv[H];
        static_for<HI / 2 - LO / 2 + 1>([&](auto P) {
            constexpr int u = 2 * (LO / 2 + decltype(P)::value);
            constexpr int v = u + 1;
            constexpr bool au = u >= LO && u <= HI, av = v >= LO && v <= HI;
            const float2 qq = Qp[(PH - u + 2 * H) % H];  // (q[c-u], q[c-u-1])
            float mnu = 0.0f;
            if constexpr (au) {
                const float upu = u == 0 ? up0 : S[PAR ^ 1][u == 0 ? 0 : u - 1];
                const float dgu = u == 0 ? dg0 : S[PAR][u == 0 ? 0 : u - 1];
                mnu = min3f(dgu, upu, S[PAR ^ 1][u]);
            }
            if constexpr (au && av) {
                const float mnv = min3f(S[PAR][u], S[PAR ^ 1][u], S[PAR ^ 1][v]);
                const float2 df = fadd2(qq, ncv[u / 2]);
                const float2 r = ffma2(df, df, make_float2(mnu, mnv));
                nv[u] = r.x;
                nv[v] = r.y;
            } else if constexpr (au) {
                const float dfu = qq.x - cv[u];
                nv[u] = fmaf(dfu, dfu, mnu);
            } else if constexpr (av) {
                const float mnv = min3f(S[PAR][u], S[PAR ^ 1][u], S[PAR ^ 1][v]);
                const float dfv = qq.y - cv[v];
                nv[v] = fmaf(dfv, dfv, mnv);
            }
        });
#pragma unroll
        for (int u = 0; u < H; ++u) {
            if (u >= LO && u <= HI) S[PAR][u] = nv[u];
            else if (u < LO) S[PAR][u] = INFINITY;  // finished rows read as out of band
        }
        if constexpr (HI == H - 1) {
            *bdst = nv[H - 1];
            rmin = fminf(rmin, nv[H - 1]);
        }
    }

    // All steps of the strip of rows j0 .. j0+H-1 (cv loaded).  Bt: this thread's boundary
    // slot 0; qt: the query pairs' copy at column j0 - R (K copies per column); nfull =
    // (2R - 2H + 3) / H.
    template <int REM, int K, int T>
    __device__ __forceinline__ void run(float* Bt, const float2* qt, int R, int nfull)
    {
#pragma unroll
        for (int u = 0; u < H; ++u) S[0][u] = S[1][u] = INFINITY;
#pragma unroll
        for (int p = 0; p < H / 2; ++p) ncv[p] = make_float2(-cv[2 * p], -cv[2 * p + 1]);
        bprev = Bt[0];
        rmin = INFINITY;
        static_for<2 * H - 2>([&](auto I) {  // prologue: rows 0 .. t/2
            constexpr int t = decltype(I)::value;
            step<t % H, t & 1, 0, t / 2>(Bt + (t + 1) * T, qt + t * K, nullptr);
        });
        float* bp = Bt + (2 * H - 1) * T;
        float* wp = Bt;
        const float2* qp = qt + (2 * H - 2) * K;
        for (int c = 0; c < nfull; ++c) {
            static_for<H>([&](auto I) {
                constexpr int k = decltype(I)::value;
                step<(2 * H - 2 + k) % H, k & 1, 0, H - 1>(bp + k * T, qp + k * K, wp + k * T);
            });
            bp += H * T;
            qp += H * K;
            wp += H * T;
        }
        static_for<REM>([&](auto I) {
            constexpr int k = decltype(I)::value;
            step<(2 * H - 2 + k) % H, k & 1, 0, H - 1>(bp + k * T, qp + k * K, wp + k * T);
        });
        float* we = wp + REM * T;                 // boundary slot of step 2R+1
        const float2* qe = qt + 2 * R * K;        // query column of step 2R
        static_for<2 * H - 2>([&](auto I) {  // epilogue: rows (t+1)/2 .. H-1 at step 2R + t
            constexpr int t = decltype(I)::value + 1;
            step<(REM + 3 * H - 3 + t) % H, t & 1, (t + 1) / 2, H - 1>(nullptr, qe + t * K, we + (t - 1) * T);
        });
    }
};

}  // namespace messi
