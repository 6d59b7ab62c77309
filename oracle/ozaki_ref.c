/*
 * oracle/ozaki_ref.c -- CPU ORACLE for the Ozaki scheme on integer matrix units
 * (Ootomo, Ozaki, Yokota, arXiv 2306.11975).
 *
 * *** TEST INFRASTRUCTURE ONLY. ***
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (libozimmu.so and the
 * paper_2306_11975_b200 package) never links, imports or calls it, and this file
 * shares no code, header, table or helper with the CUDA path.
 *
 * It is a plain, slow, obviously-correct restatement of the paper's algorithm in
 * the paper's order and notation.  Citations are "P:<line>" into PAPER.md and
 * name the section / algorithm / equation.  Where the paper is silent or garbled
 * the reading taken is the one listed in SURVEY.md s8(c) and DESIGN.md s3
 * ("reading A<n>").
 *
 * Build: gcc -std=c99 -O2 -fopenmp -ffp-contract=off -fPIC -shared  (no -ffast-math:
 * every floating-point operation below is an IEEE-754 binary64 operation with
 * round-to-nearest-even, and the order of operations is the order written).
 *
 * Layout conventions (BLAS, column-major):
 *   op(A) is m x k, op(A)(i,l) = transA==0 ? A[i + l*lda] : A[l + i*lda]
 *   op(B) is k x n, op(B)(l,j) = transB==0 ? B[l + j*ldb] : B[j + l*ldb]
 *   C     is m x n, C(i,j)    = C[i + j*ldc]
 * (trans codes: 0 = N, 1 = T, 2 = C; C is identical to T for real data.)
 *
 * Pins: see tests/test_oracle_*.py.  Every function below is pinned by a test
 * against something other than itself (SPEC/paper worked examples, exact
 * rational arithmetic, big-integer brute force, closed forms, invariants).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OZR_OK 0
#define OZR_ERR_ARG 1
#define OZR_ERR_BUDGET 2   /* k * (2^w - 1)^2 exceeds INT32 (would break exactness) */
#define OZR_ERR_OVERFLOW 3 /* an INT32 partial product left the INT32 range (must never happen) */

/* ------------------------------------------------------------------------- */
/* A1: slice width.                                                           */
/* ------------------------------------------------------------------------- */

/* Eq. alpha (s2.3.1) in the integer-unit form of s3.2.1:
 *     alpha = floor((l_acc - log2 k) / 2)
 * with l_acc the accumulator mantissa length (31 for INT32, Table 2).
 * The real-valued log2 is used exactly as printed. */
int oz_ref_alpha(int l_acc, int64_t k)
{
    return (int)floor(((double)l_acc - log2((double)k)) / 2.0);
}

/* BPS = min(alpha, l_in) (s3.2.1); for INT8-INT32, l_in = 7, l_acc = 31
 * (Table 2).  Returns <= 0 when no exact accumulation is possible. */
int oz_ref_bps(int l_in, int l_acc, int64_t k)
{
    int a = oz_ref_alpha(l_acc, k);
    return a < l_in ? a : l_in;
}

/* Slice width used by the method on INT8-INT32 (reading A2: the positional
 * scale of Alg. 3 line 7 uses w = BPS, not alpha). */
int oz_ref_slice_width(int64_t k)
{
    return oz_ref_bps(7, 31, k);
}

/* No-overflow budget ("absence of rounding errors ... absence of
 * overflow"): k products of two w-bit magnitudes must fit in INT32. */
int oz_ref_budget_ok(int w, int64_t k)
{
    int64_t d = ((int64_t)1 << w) - 1;
    return (double)k * (double)(d * d) <= 2147483647.0;
}

/* #GEMM = s(s+1)/2 (s3.2.4): pairs with i + j <= s + 1. */
int64_t oz_ref_gemm_count(int s)
{
    return (int64_t)s * (s + 1) / 2;
}

/* ------------------------------------------------------------------------- */
/* A2 + A3: SplitInt (Alg. 4).                                     */
/* ------------------------------------------------------------------------- */

/* Split `rows` vectors of length `kdim`; vector r, element l is
 *     v(r,l) = trans==0 ? M[r + l*ld] : M[l + r*ld].
 * For op(A) call with trans = transA; for the columns of op(B) call with
 * trans = !transB (column j of op(B) is row j of op(B)^T).
 *
 * Alg. 4 line 2 (reading A3): e_r = 2^E_r with E_r the frexp exponent of
 * max_l |v(r,l)|, so that |v| / 2^E_r < 1 strictly; E_r = 0 for an all-zero row.
 * Alg. 4 lines 3-5 (readings A4, A5): slice p (p = 1..s) of v holds, with the
 * sign of v, the bits of |v| / 2^E_r at positions (p-1)w+1 .. pw after the
 * binary point:
 *     d_p = sgn(v) * ( floor( |v| * 2^(w p - E_r) ) mod 2^w ).
 * Each digit is computed from |v| with ONE ldexp (exact: the result is either
 * >= 1, hence normal, or < 1 where floor gives 0 regardless of rounding),
 * then floor and fmod, all exact in binary64.
 * Reading A9: a row containing a NaN or Inf gets nonfinite[r] = 1 and zero
 * digits; the final result is NaN for every output in that row / column.
 *
 * digits: int8 array [s][rows][kdim] (digit p of v(r,l) at ((p-1)*rows + r)*kdim + l).
 * E:      int32 [rows];  nonfinite: uint8 [rows] (may be NULL). */
int oz_ref_split(int trans, int64_t rows, int64_t kdim, const double *M, int64_t ld,
                 int s, int w, int8_t *digits, int32_t *E, uint8_t *nonfinite)
{
    if (rows < 0 || kdim < 0 || s < 1 || w < 1 || w > 7) return OZR_ERR_ARG;
    const double two_w = ldexp(1.0, w);
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
        double vmax = 0.0;
        int bad = 0;
        for (int64_t l = 0; l < kdim; ++l) {
            double v = trans == 0 ? M[r + l * ld] : M[l + r * ld];
            if (!isfinite(v)) bad = 1;
            else if (fabs(v) > vmax) vmax = fabs(v);
        }
        int Er = 0;
        if (vmax != 0.0) (void)frexp(vmax, &Er); /* vmax = f * 2^Er, f in [0.5, 1) */
        if (bad) Er = 0;
        E[r] = Er;
        if (nonfinite) nonfinite[r] = (uint8_t)bad;
        for (int p = 1; p <= s; ++p) {
            int8_t *dp = digits + ((int64_t)(p - 1) * rows + r) * kdim;
            for (int64_t l = 0; l < kdim; ++l) {
                double v = trans == 0 ? M[r + l * ld] : M[l + r * ld];
                if (bad || v == 0.0) { dp[l] = 0; continue; }
                double t = floor(ldexp(fabs(v), w * p - Er));
                double d = fmod(t, two_w);           /* in [0, 2^w - 1] */
                dp[l] = (int8_t)(v < 0.0 ? -d : d);
            }
        }
    }
    return OZR_OK;
}

/* ------------------------------------------------------------------------- */
/* A4: one INT8 x INT8 -> INT32 slice product (Alg. 3 line 6).         */
/* ------------------------------------------------------------------------- */

/* P(i,j) = sum_l a(i,l) * b(j,l) where a is [ra][kdim] and b is [rb][kdim]
 * (b holds the columns of op(B)).  The sum is formed in int64 and checked to
 * lie in INT32 at every partial step -- that check IS the paper's claim that
 * the integer GEMM is error-free.  Output P is [ra][rb] row-major
 * INT32.  Returns OZR_ERR_OVERFLOW if any partial sum leaves INT32. */
int oz_ref_int_gemm(int64_t ra, int64_t rb, int64_t kdim, const int8_t *a,
                    const int8_t *b, int32_t *P)
{
    int err = 0;
#pragma omp parallel for schedule(static) reduction(| : err)
    for (int64_t i = 0; i < ra; ++i) {
        for (int64_t j = 0; j < rb; ++j) {
            int64_t acc = 0;
            for (int64_t l = 0; l < kdim; ++l) {
                acc += (int64_t)a[i * kdim + l] * (int64_t)b[j * kdim + l];
                if (acc > INT32_MAX || acc < INT32_MIN) err = 1;
            }
            P[i * rb + j] = (int32_t)acc;
        }
    }
    return err ? OZR_ERR_OVERFLOW : OZR_OK;
}

/* ------------------------------------------------------------------------- */
/* A5: accumulation and output (Alg. 3 line 7), readings A6-A9.         */
/* ------------------------------------------------------------------------- */

/* Result of the split + pair products for a block of output elements: the exact
 * level sums L_g = sum_{p+q=g} P_pq (g = 2..s+1), in int64 (exact: |L_g| <=
 * s k (2^w-1)^2 < 2^53).  Stored as Lg[(g-2)][i][j], i over the `nr` selected
 * rows, j over the `nc` selected columns (row-major within a level). */
static int level_sums(int s, int64_t nr, int64_t nc, int64_t kdim,
                      const int8_t *dA, const int8_t *dB, int64_t *Lg)
{
    int err = 0;
    int32_t *P = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nr * nc > 0 ? nr * nc : 1));
    if (!P) return OZR_ERR_ARG;
    memset(Lg, 0, sizeof(int64_t) * (size_t)(s * nr * nc));
    /* Alg. 3 lines 4-6: i = 1..s, j = 1..(s - i + 1). */
    for (int p = 1; p <= s; ++p) {
        for (int q = 1; q <= s - p + 1; ++q) {
            int e = oz_ref_int_gemm(nr, nc, kdim, dA + (int64_t)(p - 1) * nr * kdim,
                                    dB + (int64_t)(q - 1) * nc * kdim, P);
            if (e) err = e;
            int64_t *L = Lg + (int64_t)(p + q - 2) * nr * nc;
            for (int64_t t = 0; t < nr * nc; ++t) L[t] += P[t];
        }
    }
    free(P);
    return err;
}

/* Reading A8 (BLAS semantics, alpha/beta not in the paper):
 *   alpha == 0          : C = beta * C_in          (C = 0 when beta == 0)
 *   beta  == 0          : C = alpha * X            (C_in never read)
 *   otherwise           : C = fma(alpha, X, beta * C_in)  with beta*C_in rounded first. */
static double apply_alpha_beta(double alpha, double X, double beta, double cin)
{
    if (beta == 0.0) return alpha * X;
    return fma(alpha, X, beta * cin);
}

/* Full method for the sub-block of C given by row indices `ri` (nr of them)
 * and column indices `cj` (nc of them).  Writes C[ri[a] + cj[b]*ldc] only.
 * mode 0 = canonical order (reading A6, "mode L"): exact level sums, then
 *          acc = +0; for g = s+1 down to 2: acc = acc + L_g * 2^(-w g)
 *          (one rounding per add; the product is exact);
 * mode 1 = paper-literal Alg. 3 order ("mode P"): for i = 1..s, for
 *          j = 1..s-i+1: acc = acc + P_ij * 2^(-w(i+j))  (accuracy comparison only).
 * Then (reading A7) X = ldexp(acc, E_A[i] + E_B[j]) -- one ldexp, i.e. one
 * correctly-rounded scaling, applied once -- and reading A8 for alpha/beta.
 * Reading A9: non-finite input in row i of op(A) or column j of op(B) -> X = NaN. */
int oz_ref_dgemm_sub(int transA, int transB, int64_t m, int64_t n, int64_t k,
                     double alpha, const double *A, int64_t lda, const double *B,
                     int64_t ldb, double beta, double *C, int64_t ldc, int s, int mode,
                     const int64_t *ri, int64_t nr, const int64_t *cj, int64_t nc)
{
    if (m < 0 || n < 0 || k < 0 || s < 1 || nr < 0 || nc < 0) return OZR_ERR_ARG;
    if (nr == 0 || nc == 0) return OZR_OK;
    for (int64_t a = 0; a < nr; ++a) if (ri[a] < 0 || ri[a] >= m) return OZR_ERR_ARG;
    for (int64_t b = 0; b < nc; ++b) if (cj[b] < 0 || cj[b] >= n) return OZR_ERR_ARG;

    if (alpha == 0.0 || k == 0) {           /* A and B are not read (BLAS quick return) */
        for (int64_t b = 0; b < nc; ++b)
            for (int64_t a = 0; a < nr; ++a) {
                double *c = &C[ri[a] + cj[b] * ldc];
                *c = beta == 0.0 ? 0.0 : beta * *c;
            }
        return OZR_OK;
    }
    int w = oz_ref_slice_width(k);
    if (w < 1 || !oz_ref_budget_ok(w, k)) return OZR_ERR_BUDGET;

    /* Gather the selected rows of op(A) and columns of op(B) into dense
     * row-vector form, then split them (Alg. 3 lines 1-2). */
    double *Ar = (double *)malloc(sizeof(double) * (size_t)(nr * k));
    double *Bc = (double *)malloc(sizeof(double) * (size_t)(nc * k));
    int8_t *dA = (int8_t *)malloc((size_t)(s * nr * k));
    int8_t *dB = (int8_t *)malloc((size_t)(s * nc * k));
    int32_t *EA = (int32_t *)malloc(sizeof(int32_t) * (size_t)nr);
    int32_t *EB = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
    uint8_t *bA = (uint8_t *)malloc((size_t)nr), *bB = (uint8_t *)malloc((size_t)nc);
    int64_t *Lg = (int64_t *)malloc(sizeof(int64_t) * (size_t)(s * nr * nc));
    int32_t *P = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nr * nc));
    int err = OZR_OK;
    if (!Ar || !Bc || !dA || !dB || !EA || !EB || !bA || !bB || !Lg || !P) { err = OZR_ERR_ARG; goto done; }
    for (int64_t a = 0; a < nr; ++a)
        for (int64_t l = 0; l < k; ++l)
            Ar[a * k + l] = transA == 0 ? A[ri[a] + l * lda] : A[l + ri[a] * lda];
    for (int64_t b = 0; b < nc; ++b)
        for (int64_t l = 0; l < k; ++l)
            Bc[b * k + l] = transB == 0 ? B[l + cj[b] * ldb] : B[cj[b] + l * ldb];
    /* Ar / Bc are row-major [n][k]: row r element l at r*k + l, i.e. trans=1, ld=k. */
    if ((err = oz_ref_split(1, nr, k, Ar, k, s, w, dA, EA, bA))) goto done;
    if ((err = oz_ref_split(1, nc, k, Bc, k, s, w, dB, EB, bB))) goto done;

    if (mode == 0) {
        if ((err = level_sums(s, nr, nc, k, dA, dB, Lg))) goto done;
#pragma omp parallel for schedule(static)
        for (int64_t a = 0; a < nr; ++a)
            for (int64_t b = 0; b < nc; ++b) {
                double acc = 0.0;
                for (int g = s + 1; g >= 2; --g) {
                    double term = (double)Lg[(int64_t)(g - 2) * nr * nc + a * nc + b] * ldexp(1.0, -w * g);
                    acc = acc + term;
                }
                double X = (bA[a] || bB[b]) ? NAN : ldexp(acc, EA[a] + EB[b]);
                double *c = &C[ri[a] + cj[b] * ldc];
                *c = apply_alpha_beta(alpha, X, beta, beta == 0.0 ? 0.0 : *c);
            }
    } else {
        double *acc = (double *)calloc((size_t)(nr * nc), sizeof(double));
        if (!acc) { err = OZR_ERR_ARG; goto done; }
        for (int p = 1; p <= s && !err; ++p)
            for (int q = 1; q <= s - p + 1; ++q) {
                int e = oz_ref_int_gemm(nr, nc, k, dA + (int64_t)(p - 1) * nr * k,
                                        dB + (int64_t)(q - 1) * nc * k, P);
                if (e) { err = e; break; }
                double sc = ldexp(1.0, -w * (p + q));
                for (int64_t t = 0; t < nr * nc; ++t) acc[t] = acc[t] + (double)P[t] * sc;
            }
        if (!err)
            for (int64_t a = 0; a < nr; ++a)
                for (int64_t b = 0; b < nc; ++b) {
                    double X = (bA[a] || bB[b]) ? NAN : ldexp(acc[a * nc + b], EA[a] + EB[b]);
                    double *c = &C[ri[a] + cj[b] * ldc];
                    *c = apply_alpha_beta(alpha, X, beta, beta == 0.0 ? 0.0 : *c);
                }
        free(acc);
    }
done:
    free(Ar); free(Bc); free(dA); free(dB); free(EA); free(EB); free(bA); free(bB); free(Lg); free(P);
    return err;
}

/* Exact level sums for a sub-block (test hook for the GPU's
 * ozimmu_debug_level_sums).  Lg_out: int64 [s][nr][nc] row-major, level g at
 * index g-2. */
int oz_ref_level_sums_sub(int transA, int transB, int64_t m, int64_t n, int64_t k,
                          const double *A, int64_t lda, const double *B, int64_t ldb,
                          int s, const int64_t *ri, int64_t nr, const int64_t *cj,
                          int64_t nc, int64_t *Lg_out)
{
    if (m < 0 || n < 0 || k < 1 || s < 1 || nr < 1 || nc < 1) return OZR_ERR_ARG;
    int w = oz_ref_slice_width(k);
    if (w < 1 || !oz_ref_budget_ok(w, k)) return OZR_ERR_BUDGET;
    double *Ar = (double *)malloc(sizeof(double) * (size_t)(nr * k));
    double *Bc = (double *)malloc(sizeof(double) * (size_t)(nc * k));
    int8_t *dA = (int8_t *)malloc((size_t)(s * nr * k));
    int8_t *dB = (int8_t *)malloc((size_t)(s * nc * k));
    int32_t *EA = (int32_t *)malloc(sizeof(int32_t) * (size_t)nr);
    int32_t *EB = (int32_t *)malloc(sizeof(int32_t) * (size_t)nc);
    int err = OZR_ERR_ARG;
    if (Ar && Bc && dA && dB && EA && EB) {
        for (int64_t a = 0; a < nr; ++a)
            for (int64_t l = 0; l < k; ++l)
                Ar[a * k + l] = transA == 0 ? A[ri[a] + l * lda] : A[l + ri[a] * lda];
        for (int64_t b = 0; b < nc; ++b)
            for (int64_t l = 0; l < k; ++l)
                Bc[b * k + l] = transB == 0 ? B[l + cj[b] * ldb] : B[cj[b] + l * ldb];
        err = oz_ref_split(1, nr, k, Ar, k, s, w, dA, EA, NULL);
        if (!err) err = oz_ref_split(1, nc, k, Bc, k, s, w, dB, EB, NULL);
        if (!err) err = level_sums(s, nr, nc, k, dA, dB, Lg_out);
    }
    free(Ar); free(Bc); free(dA); free(dB); free(EA); free(EB);
    return err;
}

/* ------------------------------------------------------------------------- */
/* f1: complex GEMM ("We can compute a complex GEMM by separating   */
/* the real and imaginary parts ... while splitting").  Reading A16 (DESIGN): */
/* the real embedding with interleaved K                                       */
/*   Ahat(i, 2l) = Re op(A)(i,l),   Ahat(i, 2l+1) = Im op(A)(i,l)              */
/*   Bhat(2l, 2j) = Re op(B)(l,j),  Bhat(2l+1, 2j)   = -Im op(B)(l,j)          */
/*   Bhat(2l, 2j+1) = Im op(B)(l,j), Bhat(2l+1, 2j+1) = Re op(B)(l,j)          */
/* so that (Ahat Bhat)(i,2j) = Re(op(A)op(B))(i,j) and (i,2j+1) = Im; the     */
/* Ozaki method (mode L, K' = 2k) is applied to the real product, i.e. one    */
/* shared exponent per complex row of op(A) / complex column of op(B).        */
/* Complex data is interleaved (re, im) doubles; op 2 = conjugate transpose. */
/* Then with X = Xre + i Xim (reading A8 generalised):                        */
/*   alpha == 0: C = beta C (complex product below; beta == 0 -> C = 0)       */
/*   T = alpha X:  Tre = fma(ar, Xre, -(ai*Xim)),  Tim = fma(ar, Xim, ai*Xre)  */
/*   beta == 0: C = T; else U = beta C_in (same form), C = T + U per part.     */
/* ------------------------------------------------------------------------- */
static void cmul(double ar, double ai, double xr, double xi, double *zr, double *zi)
{
    double t = ai * xi;
    *zr = fma(ar, xr, -t);
    double u = ai * xr;
    *zi = fma(ar, xi, u);
}

int oz_ref_zgemm_sub(int transA, int transB, int64_t m, int64_t n, int64_t k,
                     const double *alpha, const double *A, int64_t lda, const double *B,
                     int64_t ldb, const double *beta, double *C, int64_t ldc, int s,
                     const int64_t *ri, int64_t nr, const int64_t *cj, int64_t nc)
{
    if (m < 0 || n < 0 || k < 0 || s < 1 || nr < 0 || nc < 0) return OZR_ERR_ARG;
    if (nr == 0 || nc == 0) return OZR_OK;
    const int alpha_zero = alpha[0] == 0.0 && alpha[1] == 0.0;
    const int beta_zero = beta[0] == 0.0 && beta[1] == 0.0;
    if (alpha_zero || k == 0) {
        for (int64_t b = 0; b < nc; ++b)
            for (int64_t a = 0; a < nr; ++a) {
                double *c = &C[2 * (ri[a] + cj[b] * ldc)];
                if (beta_zero) { c[0] = 0.0; c[1] = 0.0; }
                else { double zr, zi; cmul(beta[0], beta[1], c[0], c[1], &zr, &zi); c[0] = zr; c[1] = zi; }
            }
        return OZR_OK;
    }
    const int64_t K2 = 2 * k;
    /* Ahat restricted to the selected rows: nr x K2 (row-major), Bhat columns 2j, 2j+1 for
     * the selected j as a K2 x (2 nc) column-major real matrix. */
    double *Ah = (double *)malloc(sizeof(double) * (size_t)(nr * K2));
    double *Bh = (double *)malloc(sizeof(double) * (size_t)(K2 * 2 * nc));
    double *Xh = (double *)calloc((size_t)(nr * 2 * nc), sizeof(double));
    int64_t *rr = (int64_t *)malloc(sizeof(int64_t) * (size_t)nr);
    int64_t *cc = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * nc));
    int err = OZR_ERR_ARG;
    if (Ah && Bh && Xh && rr && cc) {
        for (int64_t a = 0; a < nr; ++a) {
            rr[a] = a;
            for (int64_t l = 0; l < k; ++l) {
                const double *z = transA == 0 ? &A[2 * (ri[a] + l * lda)] : &A[2 * (l + ri[a] * lda)];
                Ah[a * K2 + 2 * l] = z[0];
                Ah[a * K2 + 2 * l + 1] = transA == 2 ? -z[1] : z[1];
            }
        }
        for (int64_t b = 0; b < nc; ++b) {
            cc[2 * b] = 2 * b;
            cc[2 * b + 1] = 2 * b + 1;
            for (int64_t l = 0; l < k; ++l) {
                const double *z = transB == 0 ? &B[2 * (l + cj[b] * ldb)] : &B[2 * (cj[b] + l * ldb)];
                const double re = z[0], im = transB == 2 ? -z[1] : z[1];
                Bh[(2 * b) * K2 + 2 * l] = re;
                Bh[(2 * b) * K2 + 2 * l + 1] = -im;
                Bh[(2 * b + 1) * K2 + 2 * l] = im;
                Bh[(2 * b + 1) * K2 + 2 * l + 1] = re;
            }
        }
        /* X = Ahat Bhat by the real method (mode L), alpha = 1, beta = 0.
         * Ahat is row-major nr x K2 = column-major with trans = T, ld = K2. */
        err = oz_ref_dgemm_sub(1, 0, nr, 2 * nc, K2, 1.0, Ah, K2, Bh, K2, 0.0, Xh, nr, s, 0,
                               rr, nr, cc, 2 * nc);
    }
    if (!err) {
        for (int64_t b = 0; b < nc; ++b)
            for (int64_t a = 0; a < nr; ++a) {
                const double xr = Xh[a + (2 * b) * nr], xi = Xh[a + (2 * b + 1) * nr];
                double tr, ti;
                cmul(alpha[0], alpha[1], xr, xi, &tr, &ti);
                double *c = &C[2 * (ri[a] + cj[b] * ldc)];
                if (beta_zero) { c[0] = tr; c[1] = ti; }
                else {
                    double ur, ui;
                    cmul(beta[0], beta[1], c[0], c[1], &ur, &ui);
                    c[0] = tr + ur;
                    c[1] = ti + ui;
                }
            }
    }
    free(Ah); free(Bh); free(Xh); free(rr); free(cc);
    return err;
}

/* ------------------------------------------------------------------------- */
/* f2: INT8-AUTO split selection ("we select the number of splits   */
/* so that the average mantissa loss in the splitting process is equal to or  */
/* smaller than a threshold T"; Discussion P:713-734).  Reading A17:          */
/* for a nonzero finite element x of a vector with exponent E, write          */
/* |x| / 2^E = sum_t b_t 2^-t; its significant bits occupy positions          */
/* lead = E - ilogb(x) ... t_last = lead + vlen - 1, vlen = number of bits    */
/* from the MSB to the last 1 of the significand ("valid mantissa   */
/* length").  The s digits keep positions 1..s*w, so the bits lost are        */
/*     loss_s(x) = min(vlen, max(0, t_last - s*w)).                           */
/* mean_loss(M, s) = mean over the nonzero finite elements of M (0 if none). */
/* ------------------------------------------------------------------------- */

static int valid_len(double x) /* bits from MSB to last 1 of |x|'s significand */
{
    int e;
    double f = frexp(fabs(x), &e); /* f in [0.5, 1) */
    int v = 0;
    while (f != floor(f)) { f = f * 2.0; v++; }
    return v;
}

/* Sum of loss_s over the vectors of op(M) as in oz_ref_split (trans, rows, kdim, ld),
 * for s = 1..s_max (loss_sum[s-1]); nnz = number of nonzero finite elements. */
int oz_ref_mantissa_loss(int trans, int64_t rows, int64_t kdim, const double *M, int64_t ld,
                         int w, int s_max, int64_t *loss_sum, int64_t *nnz)
{
    if (rows < 0 || kdim < 0 || s_max < 1 || w < 1) return OZR_ERR_ARG;
    for (int s = 0; s < s_max; ++s) loss_sum[s] = 0;
    *nnz = 0;
    for (int64_t r = 0; r < rows; ++r) {
        double vmax = 0.0;
        int bad = 0;
        for (int64_t l = 0; l < kdim; ++l) {
            double v = trans == 0 ? M[r + l * ld] : M[l + r * ld];
            if (!isfinite(v)) bad = 1;
            else if (fabs(v) > vmax) vmax = fabs(v);
        }
        if (bad || vmax == 0.0) continue;
        int E;
        (void)frexp(vmax, &E);
        for (int64_t l = 0; l < kdim; ++l) {
            double v = trans == 0 ? M[r + l * ld] : M[l + r * ld];
            if (v == 0.0) continue;
            int lead = E - ilogb(v);
            int vlen = valid_len(v);
            int t_last = lead + vlen - 1;
            *nnz += 1;
            for (int s = 1; s <= s_max; ++s) {
                int over = t_last - s * w;
                int loss = over < 0 ? 0 : (over > vlen ? vlen : over);
                loss_sum[s - 1] += loss;
            }
        }
    }
    return OZR_OK;
}

/* Smallest s in [1, s_max] with mean_loss(op(A) rows, s) <= T and mean_loss(op(B)
 * columns, s) <= T (mean = (double)loss_sum / (double)nnz, 0 if nnz = 0); s_max if none.
 * w is the method's slice width for this k (A1). */
int oz_ref_auto_splits(int transA, int transB, int64_t m, int64_t n, int64_t k,
                       const double *A, int64_t lda, const double *B, int64_t ldb, double T,
                       int s_max)
{
    if (k < 1 || s_max < 1 || s_max > 64) return -1;
    int w = oz_ref_slice_width(k);
    int64_t la[64], lb[64], na = 0, nb = 0;
    if (oz_ref_mantissa_loss(transA == 0 ? 0 : 1, m, k, A, lda, w, s_max, la, &na)) return -1;
    if (oz_ref_mantissa_loss(transB == 0 ? 1 : 0, n, k, B, ldb, w, s_max, lb, &nb)) return -1;
    for (int s = 1; s <= s_max; ++s) {
        double ma = na ? (double)la[s - 1] / (double)na : 0.0;
        double mb = nb ? (double)lb[s - 1] / (double)nb : 0.0;
        if (ma <= T && mb <= T) return s;
    }
    return s_max;
}

/* ---- f2 INT8-AUTO, accuracy-targeted selection (reading A18) -----------
 *
 * The Discussion says the loss criterion "does not yield the optimal number of
 * splits", because the DGEMM rounding error grows with the accumulation length while the
 * Ozaki error does not ("the accumulation length should be one of the key factors").
 * Reading A18 writes the error of the method (Alg. 3 keeps the pairs p + q <= s + 1)
 * elementwise: with a^(t) the first t digits of a (Alg. 4), R_a(t) = a - a^(t)
 * and R_a(0) = a,
 *     C - C_s = sum_l sum_{q=1..s} b_q-part (a - a^(s+1-q)) + a (b - b^(s)),
 * |b_q-part| <= |R_b(q-1)|, hence |C - C_s|_ij <= sum_{t=0..s} (|R_A(t)| |R_B(s-t)|)_ij.
 * With magnitudes independent along l, (|X||Y|)_ij ~ ||x_i||_1 ||y_j||_1 / k, so relative to
 * (|A||B|)_ij the predicted error is eta(s) = sum_{t=0..s} rho_A(t) rho_B(s-t), where
 * rho_v(t) = ||R_v(t)||_1 / ||v||_1 for one vector (row of op(A) / column of op(B)) and
 * rho_A(t) = max over the rows (rho_B: over the columns), rho(0) = 1.  FP64 DGEMM's own
 * error in the same units is u sqrt(k) (probabilistic form of gamma_k |A||B|, u = 2^-53), so
 * s = the smallest s <= s_max with eta(s) <= tau u sqrt(k) (tau = 1: "FP64-equivalent").
 *
 * Evaluation, exact and order-free so that any implementation takes the same decision: the
 * l1 sums are taken in 32-bit fixed point relative to 2^E, the residual terms rounded UP and
 * the norm terms rounded DOWN (so rho is an upper estimate), as integers:
 *     N_t(v) = sum_x ceil(frac(|x| 2^(wt - E)) 2^32),   D(v) = sum_x floor(|x| 2^(32 - E)),
 *     rho_v(t) = ((double)N_t / (double)D) 2^(-wt)   (N, D < 2^53: exact conversions).
 * Vectors holding NaN/Inf or only zeros are skipped; an operand with no other vector has
 * rho(t) = 0 for all t (its product is exactly zero or NaN).                           */

/* |x| = M 2^(e - 53) with M an integer, 2^52 <= M < 2^53 (normal) or < 2^52 (subnormal) */
static void sig_exp(double x, uint64_t *M, int *e)
{
    double f = frexp(fabs(x), e); /* |x| = f 2^e, f in [0.5, 1) */
    *M = (uint64_t)ldexp(f, 53);  /* exact: f has at most 53 significant bits */
}

/* ceil(frac(|x| 2^(wt - E)) 2^32): |x| 2^(wt-E) = M 2^-z with z = 53 + E - e - wt fraction bits */
static uint64_t resid_up32(double x, int E, int w, int t)
{
    uint64_t M;
    int e;
    sig_exp(x, &M, &e);
    int z = 53 + E - e - w * t;
    if (z <= 0) return 0; /* |x| 2^(wt-E) is an integer: nothing left after t digits */
    unsigned __int128 R = z >= 64 ? (unsigned __int128)M : (unsigned __int128)(M % ((uint64_t)1 << z));
    if (z <= 32) return (uint64_t)(R << (32 - z)); /* exact */
    int d = z - 32;                                 /* ceil(R / 2^d) */
    if (d >= 64) return R != 0;
    return (uint64_t)((R + (((unsigned __int128)1 << d) - 1)) >> d);
}

/* floor(|x| 2^(32 - E)) = floor(M 2^(e - 53 + 32 - E)) */
static uint64_t norm_dn32(double x, int E)
{
    uint64_t M;
    int e;
    sig_exp(x, &M, &e);
    int d = 53 + E - e - 32; /* >= 21 since e <= E */
    return d >= 64 ? 0 : M >> d;
}

/* rho[t], t = 0..s_max, of the vectors of op(M): trans = 0 -> vector r = M[r + l ld]
 * (rows of op(A) with transA = N), trans = 1 -> M[l + r ld]. */
int oz_ref_trunc_residual(int trans, int64_t rows, int64_t kdim, const double *M, int64_t ld,
                          int w, int s_max, double *rho)
{
    if (rows < 0 || kdim < 0 || s_max < 1 || s_max > 64 || w < 1) return OZR_ERR_ARG;
    for (int t = 0; t <= s_max; ++t) rho[t] = 0.0;
    /* per-vector values (vectors are independent; the max below is order-free) */
    double *rv = (double *)calloc((size_t)(rows > 0 ? rows : 1) * (size_t)(s_max + 1), sizeof(double));
    if (!rv) return OZR_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t r = 0; r < rows; ++r) {
        double *out = rv + r * (s_max + 1);
        double vmax = 0.0;
        int bad = 0;
        for (int64_t l = 0; l < kdim; ++l) {
            double v = trans == 0 ? M[r + l * ld] : M[l + r * ld];
            if (!isfinite(v)) bad = 1;
            else if (fabs(v) > vmax) vmax = fabs(v);
        }
        if (bad || vmax == 0.0) continue; /* skipped: out stays 0 */
        int E;
        (void)frexp(vmax, &E);
        uint64_t D = 0, N[65];
        for (int t = 1; t <= s_max; ++t) N[t] = 0;
        for (int64_t l = 0; l < kdim; ++l) {
            double v = trans == 0 ? M[r + l * ld] : M[l + r * ld];
            if (v == 0.0) continue;
            D += norm_dn32(v, E);
            for (int t = 1; t <= s_max; ++t) N[t] += resid_up32(v, E, w, t);
        }
        out[0] = 1.0;
        for (int t = 1; t <= s_max; ++t) out[t] = ldexp((double)N[t] / (double)D, -w * t);
    }
    for (int64_t r = 0; r < rows; ++r)
        for (int t = 0; t <= s_max; ++t)
            if (rv[r * (s_max + 1) + t] > rho[t]) rho[t] = rv[r * (s_max + 1) + t];
    free(rv);
    return OZR_OK;
}

/* eta(s) = sum_{t=0..s} rho_A(t) rho_B(s - t), summed in the order t = 0, 1, .., s. */
double oz_ref_acc_eta(const double *rhoA, const double *rhoB, int s)
{
    double eta = 0.0;
    for (int t = 0; t <= s; ++t) eta = eta + rhoA[t] * rhoB[s - t];
    return eta;
}

/* Smallest s in [1, s_max] with eta(s) <= tau u sqrt(k), u = 2^-53 (reading A18); s_max if
 * none (then *capped = 1).  k is the accumulation length (2k for the complex embedding A16). */
int oz_ref_auto_splits_acc(int transA, int transB, int64_t m, int64_t n, int64_t k,
                           const double *A, int64_t lda, const double *B, int64_t ldb,
                           double tau, int s_max, int *capped)
{
    if (k < 1 || s_max < 1 || s_max > 64 || !(tau > 0.0)) return -1;
    int w = oz_ref_slice_width(k);
    double ra[65], rb[65];
    if (oz_ref_trunc_residual(transA == 0 ? 0 : 1, m, k, A, lda, w, s_max, ra)) return -1;
    if (oz_ref_trunc_residual(transB == 0 ? 1 : 0, n, k, B, ldb, w, s_max, rb)) return -1;
    double target = tau * ldexp(sqrt((double)k), -53);
    if (capped) *capped = 0;
    for (int s = 1; s <= s_max; ++s)
        if (oz_ref_acc_eta(ra, rb, s) <= target) return s;
    if (capped) *capped = 1;
    return s_max;
}
