/* oracle.c -- plain, slow, obviously correct CPU oracle.  See oracle.h for the contract.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs; never by the product library.
 *
 * Every function below is the textbook definition written out; the only "algorithmic"
 * choice is evaluating the 2D DFT separably (rows, then columns), which is an identity
 * of the definition (sum over n1 inside the sum over n0), not an approximation.
 */
#include "oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_threads(int threads) {
#ifdef _OPENMP
    return threads > 0 ? threads : omp_get_max_threads();
#else
    (void)threads;
    return 1;
#endif
}

/* complex element j of x as double (exact promotion from float). */
static inline void load_c(const void* x, int in_type, int64_t j, double* re, double* im) {
    if (in_type == ORACLE_IN_F32) {
        const float* f = (const float*)x;
        *re = (double)f[2 * j];
        *im = (double)f[2 * j + 1];
    } else {
        const double* d = (const double*)x;
        *re = d[2 * j];
        *im = d[2 * j + 1];
    }
}

static inline double load_r(const void* x, int in_type, int64_t j) {
    return in_type == ORACLE_IN_F32 ? (double)((const float*)x)[j] : ((const double*)x)[j];
}

/* w[j] = exp(sign * 2 pi i j / n) for j in [0, n), from the exactly reduced index j
 * (all callers pass j = (k*t) mod n computed in integers), angle in long double. */
static double* make_twiddles(int64_t n, int sign) {
    double* w = (double*)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    if (!w) return NULL;
    const long double half_pi = 1.570796326794896619231321691639751442L;
    for (int64_t j = 0; j < n; ++j) {
        /* quadrant reduction in integers: 2 pi j/n = q pi/2 + (pi/2) rem/n, 4j = q n + rem,
         * so multiples of pi/2 give exactly 0 and +-1. */
        int64_t q = (4 * j) / n, rem = (4 * j) % n;
        long double a = half_pi * (long double)rem / (long double)n;
        long double c = cosl(a), s = sinl(a), cr, sr;
        switch (q & 3) {
            case 0: cr = c; sr = s; break;
            case 1: cr = -s; sr = c; break;
            case 2: cr = -c; sr = -s; break;
            default: cr = s; sr = -c; break;
        }
        w[2 * j] = (double)cr;
        w[2 * j + 1] = (double)(sign * sr);
    }
    return w;
}

/* Naive 1D DFT of length n: out[k] = sum_t in[t] * w[(k t) mod n].
 * in/out are complex128 with element strides (in complex units). */
static void dft1d(const double* in, int64_t is, double* out, int64_t os, int64_t n,
                  const double* w) {
    for (int64_t k = 0; k < n; ++k) {
        double sr = 0.0, si = 0.0;
        for (int64_t t = 0; t < n; ++t) {
            int64_t j = (int64_t)(((unsigned __int128)k * (unsigned __int128)t) % (unsigned __int128)n);
            double ar = in[2 * t * is], ai = in[2 * t * is + 1];
            double wr = w[2 * j], wi = w[2 * j + 1];
            sr += ar * wr - ai * wi;
            si += ar * wi + ai * wr;
        }
        out[2 * k * os] = sr;
        out[2 * k * os + 1] = si;
    }
}

int oracle_dft2d(const void* x, int in_type, double* X, int64_t n0, int64_t n1, int sign,
                 int threads) {
    if (n0 <= 0 || n1 <= 0 || (sign != -1 && sign != 1)) return 1;
    double* w0 = make_twiddles(n0, sign);
    double* w1 = make_twiddles(n1, sign);
    double* tmp = (double*)malloc(sizeof(double) * 2 * (size_t)(n0 * n1));
    if (!w0 || !w1 || !tmp) { free(w0); free(w1); free(tmp); return 2; }
    int nt = oracle_threads(threads);
    (void)nt;
    /* Stage 1: for every row n0, the 1D DFT over n1 (inner sum of the definition). */
#pragma omp parallel num_threads(nt)
    {
        double* row = (double*)malloc(sizeof(double) * 2 * (size_t)n1);
#pragma omp for schedule(dynamic, 1)
        for (int64_t r = 0; r < n0; ++r) {
            for (int64_t c = 0; c < n1; ++c) load_c(x, in_type, r * n1 + c, &row[2 * c], &row[2 * c + 1]);
            dft1d(row, 1, tmp + 2 * r * n1, 1, n1, w1);
        }
        free(row);
    }
    /* Stage 2: for every output column k1, the 1D DFT over n0 (outer sum). */
    double scale = (sign == 1) ? 1.0 / ((double)n0 * (double)n1) : 1.0;
#pragma omp parallel num_threads(nt)
    {
        double* col = (double*)malloc(sizeof(double) * 2 * (size_t)n0);
        double* res = (double*)malloc(sizeof(double) * 2 * (size_t)n0);
#pragma omp for schedule(dynamic, 1)
        for (int64_t c = 0; c < n1; ++c) {
            for (int64_t r = 0; r < n0; ++r) {
                col[2 * r] = tmp[2 * (r * n1 + c)];
                col[2 * r + 1] = tmp[2 * (r * n1 + c) + 1];
            }
            dft1d(col, 1, res, 1, n0, w0);
            for (int64_t r = 0; r < n0; ++r) {
                X[2 * (r * n1 + c)] = res[2 * r] * scale;
                X[2 * (r * n1 + c) + 1] = res[2 * r + 1] * scale;
            }
        }
        free(col);
        free(res);
    }
    free(w0); free(w1); free(tmp);
    return 0;
}

int oracle_dft1d_rows(const void* x, int in_type, double* X, int64_t batch, int64_t n, int sign,
                      int threads) {
    if (batch <= 0 || n <= 0 || (sign != -1 && sign != 1)) return 1;
    double* w = make_twiddles(n, sign);
    if (!w) return 2;
    int nt = oracle_threads(threads);
    (void)nt;
    const double scale = (sign == 1) ? 1.0 / (double)n : 1.0;
#pragma omp parallel num_threads(nt)
    {
        double* row = (double*)malloc(sizeof(double) * 2 * (size_t)n);
#pragma omp for schedule(dynamic, 1)
        for (int64_t b = 0; b < batch; ++b) {
            for (int64_t t = 0; t < n; ++t) load_c(x, in_type, b * n + t, &row[2 * t], &row[2 * t + 1]);
            dft1d(row, 1, X + 2 * b * n, 1, n, w);
            for (int64_t k = 0; k < 2 * n; ++k) X[2 * b * n + k] *= scale;
        }
        free(row);
    }
    free(w);
    return 0;
}

int oracle_dft2d_bruteforce(const void* x, int in_type, double* X, int64_t n0, int64_t n1,
                            int sign) {
    if (n0 <= 0 || n1 <= 0 || (sign != -1 && sign != 1)) return 1;
    /* Common denominator N0*N1: exp(s 2 pi i (k0 t0/N0 + k1 t1/N1))
     *   = exp(s 2 pi i ((k0 t0 N1 + k1 t1 N0) mod N0N1) / (N0 N1)). */
    int64_t nn = n0 * n1;
    double* w = make_twiddles(nn, sign);
    if (!w) return 2;
    double scale = (sign == 1) ? 1.0 / (double)nn : 1.0;
    for (int64_t k0 = 0; k0 < n0; ++k0)
        for (int64_t k1 = 0; k1 < n1; ++k1) {
            double sr = 0.0, si = 0.0;
            for (int64_t t0 = 0; t0 < n0; ++t0)
                for (int64_t t1 = 0; t1 < n1; ++t1) {
                    int64_t j = (k0 * t0 % n0 * n1 + k1 * t1 % n1 * n0) % nn;
                    double ar, ai;
                    load_c(x, in_type, t0 * n1 + t1, &ar, &ai);
                    sr += ar * w[2 * j] - ai * w[2 * j + 1];
                    si += ar * w[2 * j + 1] + ai * w[2 * j];
                }
            X[2 * (k0 * n1 + k1)] = sr * scale;
            X[2 * (k0 * n1 + k1) + 1] = si * scale;
        }
    free(w);
    return 0;
}

int oracle_dft2d_col(const void* x, int in_type, int64_t n0, int64_t n1, int64_t k1, int sign,
                     double* out, int threads) {
    if (n0 <= 0 || n1 <= 0 || k1 < 0 || k1 >= n1 || (sign != -1 && sign != 1)) return 1;
    double* w0 = make_twiddles(n0, sign);
    double* w1 = make_twiddles(n1, sign);
    double* y = (double*)malloc(sizeof(double) * 2 * (size_t)n0);
    if (!w0 || !w1 || !y) { free(w0); free(w1); free(y); return 2; }
    int nt = oracle_threads(threads);
    (void)nt;
    /* y[t0] = sum_t1 x[t0, t1] w1[(k1 t1) mod n1]  (the inner sum, for this k1 only) */
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t t0 = 0; t0 < n0; ++t0) {
        double sr = 0.0, si = 0.0;
        for (int64_t t1 = 0; t1 < n1; ++t1) {
            int64_t j = (k1 * t1) % n1;
            double ar, ai;
            load_c(x, in_type, t0 * n1 + t1, &ar, &ai);
            sr += ar * w1[2 * j] - ai * w1[2 * j + 1];
            si += ar * w1[2 * j + 1] + ai * w1[2 * j];
        }
        y[2 * t0] = sr;
        y[2 * t0 + 1] = si;
    }
    double scale = (sign == 1) ? 1.0 / ((double)n0 * (double)n1) : 1.0;
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t k0 = 0; k0 < n0; ++k0) {
        double sr = 0.0, si = 0.0;
        for (int64_t t0 = 0; t0 < n0; ++t0) {
            int64_t j = (int64_t)(((unsigned __int128)k0 * (unsigned __int128)t0) % (unsigned __int128)n0);
            sr += y[2 * t0] * w0[2 * j] - y[2 * t0 + 1] * w0[2 * j + 1];
            si += y[2 * t0] * w0[2 * j + 1] + y[2 * t0 + 1] * w0[2 * j];
        }
        out[2 * k0] = sr * scale;
        out[2 * k0 + 1] = si * scale;
    }
    free(w0); free(w1); free(y);
    return 0;
}

int oracle_dft2d_row(const void* x, int in_type, int64_t n0, int64_t n1, int64_t k0, int sign,
                     double* out, int threads) {
    if (n0 <= 0 || n1 <= 0 || k0 < 0 || k0 >= n0 || (sign != -1 && sign != 1)) return 1;
    double* w0 = make_twiddles(n0, sign);
    double* w1 = make_twiddles(n1, sign);
    double* z = (double*)calloc(2 * (size_t)n1, sizeof(double));
    if (!w0 || !w1 || !z) { free(w0); free(w1); free(z); return 2; }
    int nt = oracle_threads(threads);
    (void)nt;
    /* z[t1] = sum_t0 x[t0, t1] w0[(k0 t0) mod n0]  (the outer sum, for this k0 only) */
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t t1 = 0; t1 < n1; ++t1) {
        double sr = 0.0, si = 0.0;
        for (int64_t t0 = 0; t0 < n0; ++t0) {
            int64_t j = (k0 * t0) % n0;
            double ar, ai;
            load_c(x, in_type, t0 * n1 + t1, &ar, &ai);
            sr += ar * w0[2 * j] - ai * w0[2 * j + 1];
            si += ar * w0[2 * j + 1] + ai * w0[2 * j];
        }
        z[2 * t1] = sr;
        z[2 * t1 + 1] = si;
    }
    double scale = (sign == 1) ? 1.0 / ((double)n0 * (double)n1) : 1.0;
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t k1 = 0; k1 < n1; ++k1) {
        double sr = 0.0, si = 0.0;
        for (int64_t t1 = 0; t1 < n1; ++t1) {
            int64_t j = (int64_t)(((unsigned __int128)k1 * (unsigned __int128)t1) % (unsigned __int128)n1);
            sr += z[2 * t1] * w1[2 * j] - z[2 * t1 + 1] * w1[2 * j + 1];
            si += z[2 * t1] * w1[2 * j + 1] + z[2 * t1 + 1] * w1[2 * j];
        }
        out[2 * k1] = sr * scale;
        out[2 * k1 + 1] = si * scale;
    }
    free(w0); free(w1); free(z);
    return 0;
}

int oracle_matmul(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                  int64_t ldb, int in_type, double* C, int64_t ldc, int threads) {
    if (m < 0 || n < 0 || k < 0) return 1;
    int nt = oracle_threads(threads);
    (void)nt;
    /* C[i][j] = sum_p A[i][p] B[p][j], i-k-j order, double accumulation. */
#pragma omp parallel for num_threads(nt) schedule(dynamic, 4)
    for (int64_t i = 0; i < m; ++i) {
        double* c = C + i * ldc;
        for (int64_t j = 0; j < n; ++j) c[j] = 0.0;
        for (int64_t p = 0; p < k; ++p) {
            double a = load_r(A, in_type, i * lda + p);
            if (in_type == ORACLE_IN_F32) {
                const float* b = (const float*)B + p * ldb;
                for (int64_t j = 0; j < n; ++j) c[j] += a * (double)b[j];
            } else {
                const double* b = (const double*)B + p * ldb;
                for (int64_t j = 0; j < n; ++j) c[j] += a * b[j];
            }
        }
    }
    return 0;
}

int oracle_matmul_rows(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                       const void* B, int64_t ldb, int in_type, const int64_t* rows,
                       int64_t nrows, double* C_rows, int threads) {
    for (int64_t r = 0; r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= m) return 1;
    int nt = oracle_threads(threads);
    (void)nt;
    /* Split the j range across threads so one long row still uses every core. */
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        double* c = C_rows + r * n;
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t j0 = 0; j0 < n; j0 += 256) {
            int64_t j1 = j0 + 256 < n ? j0 + 256 : n;
            for (int64_t j = j0; j < j1; ++j) c[j] = 0.0;
            for (int64_t p = 0; p < k; ++p) {
                double a = load_r(A, in_type, i * lda + p);
                for (int64_t j = j0; j < j1; ++j) c[j] += a * load_r(B, in_type, p * ldb + j);
            }
        }
    }
    return 0;
}

int oracle_matmul_cols(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                       const void* B, int64_t ldb, int in_type, const int64_t* cols,
                       int64_t ncols, double* C_cols, int threads) {
    for (int64_t c = 0; c < ncols; ++c)
        if (cols[c] < 0 || cols[c] >= n) return 1;
    int nt = oracle_threads(threads);
    (void)nt;
    for (int64_t c = 0; c < ncols; ++c) {
        int64_t j = cols[c];
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            double s = 0.0;
            for (int64_t p = 0; p < k; ++p)
                s += load_r(A, in_type, i * lda + p) * load_r(B, in_type, p * ldb + j);
            C_cols[c * m + i] = s;
        }
    }
    return 0;
}

int oracle_lu(int64_t n, double* A, int64_t lda, int32_t* ipiv, int threads) {
    if (n < 0 || lda < n) return -1;
    int nt = oracle_threads(threads);
    (void)nt;
    int info = 0;
    for (int64_t k = 0; k < n; ++k) {
        /* pivot: first row with the largest magnitude in column k */
        int64_t p = k;
        double best = fabs(A[k * lda + k]);
        for (int64_t i = k + 1; i < n; ++i) {
            double v = fabs(A[i * lda + k]);
            if (v > best) { best = v; p = i; }
        }
        ipiv[k] = (int32_t)p;
        if (p != k)
            for (int64_t j = 0; j < n; ++j) {
                double t = A[k * lda + j];
                A[k * lda + j] = A[p * lda + j];
                A[p * lda + j] = t;
            }
        double piv = A[k * lda + k];
        if (piv == 0.0) {
            if (!info) info = (int)(k + 1);
            continue;
        }
        /* multipliers, then the rank-1 update of the trailing matrix.  As LAPACK dgetf2 (and
           dgetrf2): scale by the reciprocal 1/piv when |piv| >= sfmin (the smallest normal,
           DBL_MIN), divide otherwise */
        const int use_recip = fabs(piv) >= DBL_MIN;
        const double rpiv = 1.0 / piv;
#pragma omp parallel for num_threads(nt) schedule(static)
        for (int64_t i = k + 1; i < n; ++i) {
            double l = use_recip ? A[i * lda + k] * rpiv : A[i * lda + k] / piv;
            A[i * lda + k] = l;
            for (int64_t j = k + 1; j < n; ++j) A[i * lda + j] -= l * A[k * lda + j];
        }
    }
    return info;
}
