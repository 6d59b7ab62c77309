/*
 * oracle/dd_ref.c -- double-double ("DD") reference GEMM used as the
 * high-precision ground truth C^DD of the paper's relative-error metric
 * (s4.2.1 Eq. relative-error: "reference ... computed in higher
 * precision, the double-double precision").
 *
 * *** TEST INFRASTRUCTURE ONLY. *** (same rules as oracle/ozaki_ref.c: only
 * tests/, smoke() and bench.py's CPU baseline may load it; it shares nothing
 * with the CUDA path.)
 *
 * Standard error-free transformations (Knuth two_sum, FMA-based two_prod) and
 * the accurate DD addition (two two_sums + renormalisation).  Build with
 * -ffp-contract=off so that no a*b+c is silently fused except the explicit fma
 * inside two_prod.
 */
#include <math.h>
#include <stdint.h>

typedef struct { double hi, lo; } dd_t;

/* hi = fl(a+b), hi + lo = a + b exactly (Knuth, no branch). */
void dd_two_sum(double a, double b, double *hi, double *lo)
{
    double s = a + b;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    *hi = s;
    *lo = e;
}

/* hi = fl(a*b), hi + lo = a * b exactly (barring under/overflow). */
void dd_two_prod(double a, double b, double *hi, double *lo)
{
    double p = a * b;
    *hi = p;
    *lo = fma(a, b, -p);
}

static dd_t quick_two_sum(double a, double b)
{
    dd_t r;
    double s = a + b;
    r.lo = b - (s - a);
    r.hi = s;
    return r;
}

/* Accurate DD + DD (relative error O(2^-104)). */
static dd_t dd_add(dd_t x, dd_t y)
{
    double s1, s2, t1, t2;
    dd_two_sum(x.hi, y.hi, &s1, &s2);
    dd_two_sum(x.lo, y.lo, &t1, &t2);
    s2 = s2 + t1;
    dd_t r = quick_two_sum(s1, s2);
    s2 = r.lo + t2;
    return quick_two_sum(r.hi, s2);
}

/* C^DD = op(A) op(B) with every product formed exactly (two_prod) and the
 * k-term sum accumulated in DD in ascending l (fixed order, deterministic).
 * Column-major BLAS layout as in ozaki_ref.c.  Only the rows ri[0..nr) and
 * columns cj[0..nc) are computed; output Chi/Clo are [nr][nc] row-major. */
int dd_gemm_sub(int transA, int transB, int64_t m, int64_t n, int64_t k,
                const double *A, int64_t lda, const double *B, int64_t ldb,
                const int64_t *ri, int64_t nr, const int64_t *cj, int64_t nc,
                double *Chi, double *Clo)
{
    if (m < 0 || n < 0 || k < 0 || nr < 0 || nc < 0) return 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t a = 0; a < nr; ++a) {
        int64_t i = ri[a];
        for (int64_t b = 0; b < nc; ++b) {
            int64_t j = cj[b];
            dd_t acc = {0.0, 0.0};
            for (int64_t l = 0; l < k; ++l) {
                double x = transA == 0 ? A[i + l * lda] : A[l + i * lda];
                double y = transB == 0 ? B[l + j * ldb] : B[j + l * ldb];
                dd_t p;
                dd_two_prod(x, y, &p.hi, &p.lo);
                acc = dd_add(acc, p);
            }
            Chi[a * nc + b] = acc.hi;
            Clo[a * nc + b] = acc.lo;
        }
    }
    return 0;
}

/* Plain binary64 GEMM in ascending-l recursive summation (no FMA): a CPU
 * stand-in for "DGEMM" when no GPU is present (accuracy trend tests only). */
int fp64_gemm_sub(int transA, int transB, int64_t m, int64_t n, int64_t k,
                  const double *A, int64_t lda, const double *B, int64_t ldb,
                  const int64_t *ri, int64_t nr, const int64_t *cj, int64_t nc, double *Cout)
{
    if (m < 0 || n < 0 || k < 0) return 1;
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < nr; ++a) {
        int64_t i = ri[a];
        for (int64_t b = 0; b < nc; ++b) {
            int64_t j = cj[b];
            double acc = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                double x = transA == 0 ? A[i + l * lda] : A[l + i * lda];
                double y = transB == 0 ? B[l + j * ldb] : B[j + l * ldb];
                acc = acc + x * y;
            }
            Cout[a * nc + b] = acc;
        }
    }
    return 0;
}

/* Complex DD reference: Re and Im of op(A) op(B) accumulated in DD (each of the four
 * real products formed exactly by two_prod), ascending l.  Interleaved complex data;
 * op 2 = conjugate transpose.  Outputs [nr][nc] row-major hi/lo per part. */
int dd_zgemm_sub(int transA, int transB, int64_t m, int64_t n, int64_t k,
                 const double *A, int64_t lda, const double *B, int64_t ldb,
                 const int64_t *ri, int64_t nr, const int64_t *cj, int64_t nc,
                 double *Rhi, double *Rlo, double *Ihi, double *Ilo)
{
    if (m < 0 || n < 0 || k < 0) return 1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t a = 0; a < nr; ++a) {
        for (int64_t b = 0; b < nc; ++b) {
            dd_t re = {0.0, 0.0}, im = {0.0, 0.0};
            for (int64_t l = 0; l < k; ++l) {
                const double *x = transA == 0 ? &A[2 * (ri[a] + l * lda)] : &A[2 * (l + ri[a] * lda)];
                const double *y = transB == 0 ? &B[2 * (l + cj[b] * ldb)] : &B[2 * (cj[b] + l * ldb)];
                const double xr = x[0], xi = transA == 2 ? -x[1] : x[1];
                const double yr = y[0], yi = transB == 2 ? -y[1] : y[1];
                dd_t p;
                dd_two_prod(xr, yr, &p.hi, &p.lo); re = dd_add(re, p);
                dd_two_prod(-xi, yi, &p.hi, &p.lo); re = dd_add(re, p);
                dd_two_prod(xr, yi, &p.hi, &p.lo); im = dd_add(im, p);
                dd_two_prod(xi, yr, &p.hi, &p.lo); im = dd_add(im, p);
            }
            Rhi[a * nc + b] = re.hi; Rlo[a * nc + b] = re.lo;
            Ihi[a * nc + b] = im.hi; Ilo[a * nc + b] = im.lo;
        }
    }
    return 0;
}
