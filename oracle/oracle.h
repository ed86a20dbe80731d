/* oracle.h -- CPU oracle for the two function blocks of Yamato, "Proposal of Automatic
 * Offloading for Function Blocks of Applications" (arXiv 2004.09883).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2004_09883_b200/, libfb.so) never includes, links or calls it, and this file
 * shares no code, header, table or constant with it.
 *
 * What is computed (PAPER.md gives no formulas; it names the blocks only):
 *   - P:149-151: the "Fourier transform" block, replaced by cuFFT, run on a
 *     2048*2048 grid.  Oracle: the plain 2D DFT definition:
 *        X[k0,k1] = sum_{n0,n1} x[n0,n1] exp(s*2*pi*i*(k0 n0/N0 + k1 n1/N1)),  s = -1
 *     inverse: s = +1 and a factor 1/(N0 N1) (readings R1, R2).
 *   - P:153, P:165 (+ BASELINE.json north_star, reading R9): the "matrix
 *     calculation" block as a dense product C[i,j] = sum_k A[i,k] B[k,j].
 *
 * Precision: every sum is accumulated in IEEE double; twiddles exp(s*2*pi*i*j/N) are
 * formed from the exactly reduced integer j mod N in long double and rounded to double.
 * Layout: row-major, complex = interleaved (re, im) (reading R3).
 *
 * Parity pins (tests/test_oracle_pins.py): worked 2x2 example, delta and tone closed
 * forms, Parseval, linearity, shift theorem, Hermitian symmetry, inverse(forward)=id,
 * non-separable brute force, numpy.fft (independent library); for the product:
 * identity/permutation (exact), Sylvester-Hadamard H H^T = N I (exact), DCT-II Q Q^T = I,
 * exact small-integer products, numpy float64 matmul.
 */
#ifndef FB_ORACLE_H
#define FB_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Element type of an input array handed to the oracle. */
enum { ORACLE_IN_F64 = 0, ORACLE_IN_F32 = 1 };

/* 2D DFT of x[n0][n1] (complex, interleaved; element type in_type) into X[n0][n1]
 * (complex128 interleaved).  sign = -1 forward (unscaled), +1 inverse (scaled by
 * 1/(n0 n1)).  Evaluated separably (rows, then columns), each 1D transform as the
 * O(N^2) definition.  threads <= 0 means "all available".  Returns 0 on success. */
int oracle_dft2d(const void* x, int in_type, double* X, int64_t n0, int64_t n1,
                 int sign, int threads);

/* The same definition evaluated as the non-separable quadruple sum (brute force).
 * O((n0 n1)^2): tiny sizes only. */
int oracle_dft2d_bruteforce(const void* x, int in_type, double* X, int64_t n0, int64_t n1,
                            int sign);

/* Batched 1D DFT (the 1D transform the paper's Fourier block applies per
 * signal): X[b][k] = sum_t x[b][t] exp(sign 2 pi i k t / n) for each of `batch`
 * contiguous lines of length n (inverse, sign +1: times 1/n).  Same O(n^2) definition and
 * twiddles as one stage of oracle_dft2d. */
int oracle_dft1d_rows(const void* x, int in_type, double* X, int64_t batch, int64_t n, int sign,
                      int threads);

/* One output column X[:, k1] (n0 complex values) of the 2D DFT of x[n0][n1]. */
int oracle_dft2d_col(const void* x, int in_type, int64_t n0, int64_t n1, int64_t k1,
                     int sign, double* out, int threads);

/* One output row X[k0, :] (n1 complex values) of the 2D DFT of x[n0][n1]. */
int oracle_dft2d_row(const void* x, int in_type, int64_t n0, int64_t n1, int64_t k0,
                     int sign, double* out, int threads);

/* C[m][n] = A[m][k] * B[k][n]; row-major with leading dimensions in elements.
 * A, B of element type in_type; C is double.  i-k-j triple loop, double accumulate. */
int oracle_matmul(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                  const void* B, int64_t ldb, int in_type, double* C, int64_t ldc,
                  int threads);

/* Selected rows: C_rows[r][:] = A[rows[r]][:] * B  (C_rows is nrows x n, ld = n). */
int oracle_matmul_rows(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                       const void* B, int64_t ldb, int in_type, const int64_t* rows,
                       int64_t nrows, double* C_rows, int threads);

/* Selected columns: C_cols[c][:] = (A * B[:, cols[c]])^T  (nc x m, ld = m). */
int oracle_matmul_cols(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                       const void* B, int64_t ldb, int in_type, const int64_t* cols,
                       int64_t ncols, double* C_cols, int threads);

/* LU factorisation with partial pivoting ("LU decomposition processing of 2048*2048
 * orthogonal matrix data", replaced by cuSOLVER getrf; reading R19):
 * P A = L U in place on the row-major n x n double matrix A (lda), right-looking, column by
 * column exactly as LAPACK's unblocked dgetf2: at step k the pivot is the FIRST row p >= k
 * with the largest |A[p][k]|, rows k and p are swapped (whole rows), the column below the
 * diagonal is scaled by the pivot's reciprocal (divided instead when |pivot| < DBL_MIN, the
 * sfmin rule of dgetf2), and the trailing matrix receives the rank-1 update.
 * ipiv[k] = p (0-based).  Returns 0, or k+1 for the first exactly-zero pivot (the step is
 * then skipped, as in LAPACK). */
int oracle_lu(int64_t n, double* A, int64_t lda, int32_t* ipiv, int threads);

/* Number of OpenMP threads a call with `threads` would use. */
int oracle_threads(int threads);

#ifdef __cplusplus
}
#endif
#endif
