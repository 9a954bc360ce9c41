/*
 * messi_oracle.c -- plain, serial, fp64 CPU oracle for the MESSI exact 1-NN hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this file.  The CUDA product
 * path (paper_2110_07519_b200/) shares no code, header, table or constant with it and
 * never calls it.
 *
 * Paper: Peng, Fatourou, Palpanas, "Fast Data Series Indexing for In-Memory Data"
 * (arXiv 2110.07519), cited as PAPER.md line numbers "P:<line>" with the section /
 * equation / algorithm they sit in.  Readings of silent or garbled passages follow
 * SURVEY.md section 8(c) and are listed in DESIGN.md ("Readings").
 *
 * Every function is the plain definition, written out, with no pruning, no blocking,
 * no reordering: sums are sequential in index order, in fp64, and this file must be
 * compiled with -ffp-contract=off (no FMA contraction) and without -ffast-math, so
 * the fp64 results are a fixed, checkable sequence of IEEE operations.
 *
 * Pins (tests/test_oracle_pins.py): closed-form breakpoints vs scipy.special.ndtri
 * and statistics.NormalDist; hand-computed PAA/iSAX worked example; SPEC examples;
 * Property 1 and the LB_Keogh chain as invariants;
 * DTW brute force over all warping paths on tiny inputs; 1-NN brute force against
 * a numpy scan.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

/* ---------------------------------------------------------------- breakpoints --
 * O3.  iSAX divides the value axis into regions "with just 256 symbols, the maximum
 * alphabet cardinality ... 8 bits" (sec. 2.2 "iSAX Representation").  The
 * paper does not restate the breakpoints; reading R2: the N(0,1) quantiles
 * beta_k = Phi^{-1}(k/card), k = 1..card-1, inverted by plain bisection to the last
 * representable double.  Phi(x) - p is evaluated as erf(x/sqrt 2)/2 - (p - 1/2) near the
 * median (where erf keeps full relative precision) and as erfc(-x/sqrt 2)/2 - p in the
 * lower tail; the upper half uses the symmetry Phi^{-1}(p) = -Phi^{-1}(1-p) of N(0,1).
 */
static double oracle_phi_minus(double x, double p)
{
    if (p >= 0.25) return 0.5 * erf(x / sqrt(2.0)) - (p - 0.5);
    return 0.5 * erfc(-x / sqrt(2.0)) - p;
}

double oracle_inv_phi(double p)
{
    if (p > 0.5) return -oracle_inv_phi(1.0 - p);
    if (p == 0.5) return 0.0; /* the same symmetry at the median: x = -x */
    double lo = -40.0, hi = 40.0;
    for (int it = 0; it < 2000; ++it) {
        double mid = 0.5 * (lo + hi);
        if (mid == lo || mid == hi) break;
        if (oracle_phi_minus(mid, p) < 0.0) lo = mid; else hi = mid;
    }
    /* lo: largest double seen with Phi < p; hi: smallest with Phi >= p; take the closer */
    return (fabs(oracle_phi_minus(lo, p)) < fabs(oracle_phi_minus(hi, p))) ? lo : hi;
}

/* beta64[k-1] = Phi^{-1}(k/card), beta32[k-1] = round-to-nearest float of it. */
int oracle_breakpoints(int card, double* beta64, float* beta32)
{
    if (card < 2 || card > 256 || (card & (card - 1))) return -1;
    for (int k = 1; k < card; ++k) {
        double b = oracle_inv_phi((double)k / (double)card);
        beta64[k - 1] = b;
        beta32[k - 1] = (float)b;
    }
    return 0;
}

/* ------------------------------------------------------------------------ PAA --
 * O2.  PAA "divides the data series in w segments of equal length, and uses the mean
 * value of the points in each segment".  Reading R5: fp64 sequential sum
 * over the segment, divided by m = n/w, rounded once to fp32 (paa32) -- this fp32 mean
 * is what the iSAX symbol is taken from.  n % w != 0 is rejected (DESIGN.md R-n%w).
 */
int oracle_paa32(const float* x, int n, int w, float* paa32)
{
    if (w <= 0 || n < w || n % w) return -1;
    int m = n / w;
    for (int s = 0; s < w; ++s) {
        double sum = 0.0;
        for (int j = 0; j < m; ++j) sum = sum + (double)x[s * m + j];
        paa32[s] = (float)(sum / (double)m);
    }
    return 0;
}

/* Same mean, kept in fp64: the query-side PAA used by the lower bounds (O6, O11). */
int oracle_paa64(const float* x, int n, int w, double* paa64)
{
    if (w <= 0 || n < w || n % w) return -1;
    int m = n / w;
    for (int s = 0; s < w; ++s) {
        double sum = 0.0;
        for (int j = 0; j < m; ++j) sum = sum + (double)x[s * m + j];
        paa64[s] = sum / (double)m;
    }
    return 0;
}

/* ---------------------------------------------------------------------- iSAX --
 * O4.  "represents each of the w segments ... with the symbol of the region the PAA
 * falls into".  Reading R3/R4: ascending symbols (0 = lowest region), a
 * value equal to a breakpoint goes to the region above: sym = #{k : beta32_k <= paa32}.
 */
int oracle_symbol(float paa32, const float* beta32, int card)
{
    int count = 0;
    for (int k = 0; k < card - 1; ++k)
        if (beta32[k] <= paa32) count = count + 1;
    return count;
}

int oracle_isax(const float* x, int n, int w, const float* beta32, int card, float* paa32,
                uint8_t* sym)
{
    if (oracle_paa32(x, n, w, paa32)) return -1;
    for (int s = 0; s < w; ++s) sym[s] = (uint8_t)oracle_symbol(paa32[s], beta32, card);
    return 0;
}

/* O5.  Region box of symbol v: [lo, hi) = [beta32_v, beta32_{v+1}), beta_0 = -inf,
 * beta_card = +inf (the "iSAX box" of Fig. fig:dtwsimd). */
static double box_lo(int v, const float* beta32) { return v == 0 ? -INFINITY : (double)beta32[v - 1]; }
static double box_hi(int v, const float* beta32, int card)
{
    return v == card - 1 ? INFINITY : (double)beta32[v];
}

/* ------------------------------------------------------------------- mindist --
 * O6.  Property 1: the distance between the PAA of the query and the
 * iSAX summary lower-bounds the real distance.  Reading R6/R7 (the iSAX literature
 * form): LB^2 = m * sum_s max(0, lo(sym_s) - qpaa_s, qpaa_s - hi(sym_s))^2, squared.
 */
double oracle_mindist2(const double* qpaa, const uint8_t* sym, int w, int n, const float* beta32,
                       int card)
{
    double m = (double)(n / w);
    double sum = 0.0;
    for (int s = 0; s < w; ++s) {
        double lo = box_lo(sym[s], beta32), hi = box_hi(sym[s], beta32, card);
        double d = 0.0;
        if (lo - qpaa[s] > d) d = lo - qpaa[s];
        if (qpaa[s] - hi > d) d = qpaa[s] - hi;
        sum = sum + d * d;
    }
    return m * sum;
}

/* ------------------------------------------------------------------------ ED --
 * O7.  Euclidean distance (sec. 2.1; reading R1: sqrt of the sum of squared
 * point differences), kept squared: d2 = sum_i ((double)a_i - (double)b_i)^2, in i order.
 */
double oracle_ed2(const float* a, const float* b, int n)
{
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        double d = (double)a[i] - (double)b[i];
        sum = sum + d * d;
    }
    return sum;
}

/* ------------------------------------------------------------------ envelope --
 * O9.  U_i = max(q_{i-r} : q_{i+r}), L_i = min(...) (sec. 3.4 DTW);
 * reading R9: the window is clamped to [0, n-1].
 */
int oracle_envelope(const float* q, int n, int r, float* U, float* L)
{
    if (r < 0 || r > n) return -1;
    for (int i = 0; i < n; ++i) {
        int a = i - r < 0 ? 0 : i - r;
        int b = i + r > n - 1 ? n - 1 : i + r;
        float u = q[a], l = q[a];
        for (int j = a; j <= b; ++j) {
            if (q[j] > u) u = q[j];
            if (q[j] < l) l = q[j];
        }
        U[i] = u;
        L[i] = l;
    }
    return 0;
}

/* O10.  LB_Keogh(Q, C) = sqrt(sum_i (c_i-U_i)^2 if c_i>U_i; (c_i-L_i)^2 if c_i<L_i; 0)
 * (P:1392-1405), kept squared. */
double oracle_lb_keogh2(const float* U, const float* L, const float* c, int n)
{
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        double d = 0.0;
        if (c[i] > U[i]) d = (double)c[i] - (double)U[i];
        else if (c[i] < L[i]) d = (double)c[i] - (double)L[i];
        sum = sum + d * d;
    }
    return sum;
}

/* O11.  Envelope-PAA vs iSAX ("the PAA of the LB_Keogh envelope"; the ABOVE /
 * BELOW / IN cases of Fig. fig:dtwsimd): per segment ABOVE = lo - Upaa
 * when the box lies above the upper envelope PAA, BELOW = Lpaa - hi when it lies below
 * the lower envelope PAA, IN = 0; squared, summed, scaled by m. */
double oracle_lb_env_paa2(const double* Upaa, const double* Lpaa, const uint8_t* sym, int w, int n,
                          const float* beta32, int card)
{
    double m = (double)(n / w);
    double sum = 0.0;
    for (int s = 0; s < w; ++s) {
        double lo = box_lo(sym[s], beta32), hi = box_hi(sym[s], beta32, card);
        double d = 0.0;                     /* IN */
        if (lo > Upaa[s]) d = lo - Upaa[s]; /* ABOVE */
        else if (hi < Lpaa[s]) d = Lpaa[s] - hi; /* BELOW */
        sum = sum + d * d;
    }
    return m * sum;
}

/* O11b.  Reverse envelope-PAA bound (reading R19).  LB_Keogh holds with
 * the roles of the two series swapped (the query against the envelope of the
 * candidate), and the PAA reduction of P:1411 applies to that envelope as it does to the
 * query's.  oracle_renv_sym: the candidate's envelope (O9), the mean of U and of L over
 * each segment (fp64), and the symbol of the box containing each mean (O4's rule,
 * #{k : beta32_k <= mean}). */
int oracle_renv_sym(const float* x, int n, int r, int w, const float* beta32, int card, uint8_t* usym,
                    uint8_t* lsym)
{
    if (w <= 0 || n % w || r < 0 || r > n) return -1;
    float* U = (float*)malloc(sizeof(float) * (size_t)n);
    float* L = (float*)malloc(sizeof(float) * (size_t)n);
    if (!U || !L) { free(U); free(L); return -1; }
    oracle_envelope(x, n, r, U, L);
    int m = n / w;
    for (int s = 0; s < w; ++s) {
        double su = 0.0, sl = 0.0;
        for (int j = 0; j < m; ++j) {
            su = su + (double)U[s * m + j];
            sl = sl + (double)L[s * m + j];
        }
        double ubar = su / (double)m, lbar = sl / (double)m;
        int cu = 0, cl = 0;
        for (int k = 0; k < card - 1; ++k) {
            if ((double)beta32[k] <= ubar) cu = cu + 1;
            if ((double)beta32[k] <= lbar) cl = cl + 1;
        }
        usym[s] = (uint8_t)cu;
        lsym[s] = (uint8_t)cl;
    }
    free(U);
    free(L);
    return 0;
}

int oracle_renv_sym_rows(const float* data, int64_t rows, int n, int r, int w, const float* beta32, int card,
                         uint8_t* usym, uint8_t* lsym)
{
    for (int64_t i = 0; i < rows; ++i)
        if (oracle_renv_sym(data + i * n, n, r, w, beta32, card, usym + i * w, lsym + i * w)) return -1;
    return 0;
}

/* LB^2 = m * sum_s max(0, qpaa_s - hi(usym_s), lo(lsym_s) - qpaa_s)^2: the distance of the
 * query's segment mean to the box spanning [lo(lsym_s), hi(usym_s)] (O5's boxes), which
 * contains [Lbar_s, Ubar_s]. */
double oracle_lb_rev_paa2(const double* qpaa, const uint8_t* usym, const uint8_t* lsym, int w, int n,
                          const float* beta32, int card)
{
    double m = (double)(n / w);
    double sum = 0.0;
    for (int s = 0; s < w; ++s) {
        double hi = box_hi(usym[s], beta32, card), lo = box_lo(lsym[s], beta32);
        double d = 0.0;                       /* inside */
        if (qpaa[s] > hi) d = qpaa[s] - hi;   /* query mean above the upper envelope's box */
        else if (qpaa[s] < lo) d = lo - qpaa[s]; /* below the lower envelope's box */
        sum = sum + d * d;
    }
    return m * sum;
}

void oracle_lb_rev_paa2_rows(const double* qpaa, const uint8_t* usym, const uint8_t* lsym, int64_t rows, int w,
                             int n, const float* beta32, int card, double* out)
{
    for (int64_t i = 0; i < rows; ++i) out[i] = oracle_lb_rev_paa2(qpaa, usym + i * w, lsym + i * w, w, n, beta32, card);
}

/* ----------------------------------------------------------------------- DTW --
 * O12.  DTW with a Sakoe-Chiba band of reach r ("reach ... allowed
 * range of warping"; reading R8): D(0,0) = c(0,0); D(i,j) = c(i,j) + min(D(i-1,j-1),
 * D(i-1,j), D(i,j-1)) for |i-j| <= r, +inf outside the band; c(i,j) = (q_i - c_j)^2 in
 * fp64; result D(n-1,n-1) (squared DTW).  Plain full-width rows, row by row.
 */
double oracle_dtw2(const float* q, const float* c, int n, int r)
{
    double* prev = (double*)malloc(sizeof(double) * (size_t)n);
    double* cur = (double*)malloc(sizeof(double) * (size_t)n);
    if (!prev || !cur) { free(prev); free(cur); return NAN; }
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            if (j - i > r || i - j > r) { cur[j] = INFINITY; continue; }
            double d = (double)q[i] - (double)c[j];
            double cost = d * d;
            if (i == 0 && j == 0) { cur[j] = cost; continue; }
            double best = INFINITY;
            if (i > 0 && j > 0 && prev[j - 1] < best) best = prev[j - 1];
            if (i > 0 && prev[j] < best) best = prev[j];
            if (j > 0 && cur[j - 1] < best) best = cur[j - 1];
            cur[j] = cost + best;
        }
        double* t = prev; prev = cur; cur = t;
    }
    double out = prev[n - 1];
    free(prev);
    free(cur);
    return out;
}

/* --------------------------------------------------------------------- 1-NN --
 * O8 / O13.  "given a query series S_q of length n, and a collection S of sequences
 * of the same length, n, we want to identify the series S_c in S that has the smallest
 * distance to S_q" (sec. 2.1).  Brute force over every row, lexicographic
 * min over (d2, id): strict '<' keeps the lowest id on ties (reading R11).  row_begin
 * offsets the ids (a chunk of a larger collection).
 */
void oracle_nn_ed(const float* data, int64_t rows, int n, const float* q, int64_t row_begin,
                  double* best_d2, int64_t* best_id)
{
    double bd = INFINITY;
    int64_t bi = -1;
    for (int64_t k = 0; k < rows; ++k) {
        double d = oracle_ed2(q, data + (size_t)k * (size_t)n, n);
        if (d < bd) { bd = d; bi = row_begin + k; }
    }
    *best_d2 = bd;
    *best_id = bi;
}

void oracle_nn_dtw(const float* data, int64_t rows, int n, const float* q, int r, int64_t row_begin,
                   double* best_d2, int64_t* best_id)
{
    double bd = INFINITY;
    int64_t bi = -1;
    for (int64_t k = 0; k < rows; ++k) {
        double d = oracle_dtw2(q, data + (size_t)k * (size_t)n, n, r);
        if (d < bd) { bd = d; bi = row_begin + k; }
    }
    *best_d2 = bd;
    *best_id = bi;
}

/* Same definition for nq queries over one row chunk: out[qi] = min over rows, per query. */
void oracle_nn_ed_multi(const float* data, int64_t rows, int n, const float* queries, int nq,
                        int64_t row_begin, double* best_d2, int64_t* best_id)
{
    for (int qi = 0; qi < nq; ++qi)
        oracle_nn_ed(data, rows, n, queries + (size_t)qi * (size_t)n, row_begin, &best_d2[qi],
                     &best_id[qi]);
}

void oracle_nn_dtw_multi(const float* data, int64_t rows, int n, const float* queries, int nq, int r,
                         int64_t row_begin, double* best_d2, int64_t* best_id)
{
    for (int qi = 0; qi < nq; ++qi)
        oracle_nn_dtw(data, rows, n, queries + (size_t)qi * (size_t)n, r, row_begin, &best_d2[qi],
                      &best_id[qi]);
}

/* Per-row distances (for element-by-element parity of single steps). */
void oracle_ed2_rows(const float* data, int64_t rows, int n, const float* q, double* out)
{
    for (int64_t k = 0; k < rows; ++k) out[k] = oracle_ed2(q, data + (size_t)k * (size_t)n, n);
}

void oracle_dtw2_rows(const float* data, int64_t rows, int n, const float* q, int r, double* out)
{
    for (int64_t k = 0; k < rows; ++k) out[k] = oracle_dtw2(q, data + (size_t)k * (size_t)n, n, r);
}

/* O2 + O4 for `rows` consecutive series (a loop over oracle_isax; no new arithmetic). */
int oracle_isax_rows(const float* data, int64_t rows, int n, int w, const float* beta32, int card, float* paa32,
                     uint8_t* sym)
{
    for (int64_t k = 0; k < rows; ++k)
        if (oracle_isax(data + (size_t)k * (size_t)n, n, w, beta32, card, paa32 + (size_t)k * (size_t)w,
                        sym + (size_t)k * (size_t)w))
            return -1;
    return 0;
}
