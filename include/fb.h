/* fb.h -- C ABI of libfb.so: the two "function blocks" of Yamato, "Proposal of Automatic
 * Offloading for Function Blocks of Applications" (arXiv 2004.09883), rebuilt for B200
 * (sm_100a).  PAPER.md (P:n = line n) names the blocks; BASELINE.json's north_star fixes
 * their semantics; DESIGN.md lists every reading taken where the paper is silent.
 *
 *   Fourier-transform block  ("grid size 2048*2048", replaced by
 *                             cuFFT)                        -> fb_fft2d / fb_ifft2d
 *   Matrix-calculation block ("linear algebra ... cuBLAS"; GEMM per the
 *                             north_star, reading R9) -> fb_matmul
 *   Interface with the host program (C-1: "the replacement library ... is installed
 *   ... and a host (CPU) program is connected"; P:43 transfer overhead)
 *                                                           -> fb_*_host variants
 *   Multi-GPU partitioning (north_star (4)) -> fb_comm_*, fb_fft2d_slab, fb_matmul_rowblock
 *
 * Conventions (all entry points)
 *   - Every parameter is a plain pointer or integer; there are no CUDA or torch types.
 *     `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - Device pointers are owned by the caller.  The library never allocates or frees
 *     caller-visible memory; it keeps only immutable per-device state (a 16384-entry FP32
 *     twiddle table and a TMA descriptor scratch), created by fb_init (or lazily, on the
 *     first call on a device, outside any stream capture).
 *   - All work is enqueued on `stream`; no call synchronises the host except fb_init,
 *     fb_comm_init/destroy and the *_host variants (which return after the D2H copy).
 *   - Layout: row-major.  complex64 = {float re, im} interleaved (== torch.complex64).
 *   - Validation happens before anything is enqueued; on error NOTHING is enqueued and a
 *     status != FB_OK is returned, with a thread-local message in fb_last_error_detail().
 *     Asynchronous device faults surface at the caller's next synchronisation.
 *   - Determinism: for a fixed (shape, world size, build) every result is bitwise
 *     reproducible run to run (no atomics in any reduction, no split-K).
 */
#ifndef FB_H
#define FB_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FB_OK = 0,
    FB_ERR_INVALID_VALUE = 1,    /* null pointer, bad flag, partial overlap, n % P != 0 ... */
    FB_ERR_UNSUPPORTED_SIZE = 2, /* FFT length > 2^14, or not a power of two and > 8192 */
    FB_ERR_MISALIGNED = 3,       /* pointer not 16-byte aligned / leading dim breaks TMA rule */
    FB_ERR_WORKSPACE = 4,        /* workspace pointer null or smaller than *_workspace_bytes */
    FB_ERR_NOT_INITIALIZED = 5,  /* fb_comm_* on a null or destroyed communicator */
    FB_ERR_CUDA = 6,             /* a CUDA runtime call or kernel launch failed */
    FB_ERR_NCCL = 7,             /* an NCCL call failed (detail from ncclGetLastError) */
    FB_ERR_ARCH = 8              /* device is not sm_100 (the kernels are sm_100a only) */
} fb_status;

typedef enum { FB_F32 = 0, FB_F64 = 1 } fb_dtype;

/* Library version (major*10000 + minor*100 + patch). */
int fb_version(void);
/* Static string for a status code. */
const char* fb_status_string(int status);
/* Thread-local detail of the last error returned on this thread ("" if none). */
const char* fb_last_error_detail(void);
/* Number of kernels libfb has launched in this process (all devices).  Lets a harness
 * count the library's own launches inside a timed region. */
uint64_t fb_launch_count(void);
/* Re-read the FB_* A/B tuning knobs from the environment (normally read once per process, on
 * first use; no launch path calls getenv).  For tests and tuning tools that change the
 * environment inside one process.  Not thread-safe against concurrent launches. */
void fb_reload_knobs(void);

/* Once per device: checks sm_100, builds the twiddle table W[j] = exp(-2 pi i j/16384)
 * (computed in FP64 with sincospi, RN-rounded to FP32; exact at multiples of pi/2),
 * resolves cuTensorMapEncodeTiled.  Synchronous.  Idempotent. */
fb_status fb_init(int device);

/* ------------------------------------------------------------------ Fourier block
 * Y = DFT2(X) over an n0 x n1 complex64 array (n0 rows, n1 contiguous columns):
 *   Y[k0,k1] = sum_{t0,t1} X[t0,t1] exp(-2 pi i (k0 t0/n0 + k1 t1/n1))      (unscaled)
 * fb_ifft2d: sign +1 and the factor 1/(n0 n1) (exact when n0 n1 is a power of two, else the
 * FP32 rounding of the FP64 reciprocal).
 * Reading R1 (sign -1 forward, cuFFT/numpy convention), R2 (inverse scaled), R3 (layout),
 * R4 / R22 (sizes): each of n0, n1 a power of two <= 16384, or any other length <= 8192
 * (lengths that factor into 2, 3, 5, 7: mixed-radix Stockham lines; others: Bluestein's
 * chirp-z over power-of-two passes).
 * x and y: device pointers, 16-byte aligned, n0*n1*8 bytes each; x == y (in place) is
 * allowed, partial overlap is FB_ERR_INVALID_VALUE.
 * ws: device workspace of fb_fft2d_workspace_bytes(n0, n1) bytes (may be NULL when that
 * is 0: power-of-two n0 < 512 or n0 == 4096; the 2 x n0/2 column split for 512 <= n0 <= 2048
 * and the four-step split for n0 > 4096 use n0*n1*8 bytes; other sizes a transpose buffer,
 * the convolution lines and the chirp / twiddle tables).  Not read before written; contents
 * undefined afterwards.
 * Accuracy (north_star): rel-L2 <= 1e-5 * log2(n0 n1) vs the exact DFT; internal gate
 * 5e-7 (reading R6). */
size_t fb_fft2d_workspace_bytes(int64_t n0, int64_t n1);
fb_status fb_fft2d(const void* x, void* y, int64_t n0, int64_t n1, void* ws, size_t ws_bytes,
                   void* stream);
fb_status fb_ifft2d(const void* x, void* y, int64_t n0, int64_t n1, void* ws, size_t ws_bytes,
                    void* stream);

/* Batched 1D transform: `batch` independent lines of length n, line b at
 * x + b*n complex64 elements (contiguous rows of a batch x n array):
 *   Y[b][k] = sum_t X[b][t] exp(-2 pi i k t / n)   (unscaled);  fb_ifft1d_batched: +1, 1/n.
 * One pass of the same line kernels as fb_fft2d.  n a power of two <= 16384, batch >= 1,
 * x and y 16-byte aligned, in place allowed (partial overlap: FB_ERR_INVALID_VALUE); no
 * workspace.  Accuracy as fb_fft2d with N = n. */
fb_status fb_fft1d_batched(const void* x, void* y, int64_t n, int64_t batch, void* stream);
fb_status fb_ifft1d_batched(const void* x, void* y, int64_t n, int64_t batch, void* stream);

/* Real-input 2D transform (the paper's vibration signals are real):
 * x is an n0 x n1 row-major float32 array, y the Hermitian half of its DFT, an n0 x (n1/2+1)
 * row-major complex64 array (numpy rfft2 / cuFFT R2C layout):
 *   y[k0][k1] = sum_{t0,t1} x[t0][t1] exp(-2 pi i (k0 t0/n0 + k1 t1/n1)), 0 <= k1 <= n1/2.
 * fb_irfft2d is the exact inverse (sign +1, 1/(n0 n1); y read, never written).  n0, n1 powers
 * of two, 1 <= n0 <= 16384, 2 <= n1 <= 16384.  x, y, ws 16-byte aligned and pairwise
 * disjoint; ws: fb_rfft2d_workspace_bytes(n0, n1) bytes.  Accuracy as fb_fft2d. */
size_t fb_rfft2d_workspace_bytes(int64_t n0, int64_t n1);
fb_status fb_rfft2d(const void* x, void* y, int64_t n0, int64_t n1, void* ws, size_t ws_bytes, void* stream);
fb_status fb_irfft2d(const void* y, void* x, int64_t n0, int64_t n1, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ matrix block
 * C[m][n] = A[m][k] * B[k][n]  (row-major, leading dimensions in ELEMENTS, C overwritten).
 * FB_F64: IEEE FP64 (DMMA tensor-core FMAs, RN); accuracy rel-L2 <= 1e-12.
 * FB_F32: FP32 via 3xTF32 on tcgen05 tensor cores (hi*hi + hi*lo + lo*hi; B split RN into
 *         hi/lo, A used raw as hi -- the tensor core truncates it to TF32, reading R21 -- with
 *         lo = rn(a - trunc(a)); FP32 accumulation in TMEM promoted to RN registers every
 *         128 k); accuracy rel-L2 <= 1e-5 (reading R11).  Bitwise deterministic for a fixed
 *         shape; not bitwise equal to an FP32 SIMT GEMM.
 * m, n, k >= 1 (any value: ragged edges are handled).  A, B, C 16-byte aligned;
 * lda, ldb, ldc >= the row width and lda*esize, ldb*esize, ldc*esize multiples of 16 B.
 * ws: device workspace of fb_matmul_workspace_bytes(...) bytes (FP32: the TF32 hi/lo
 * split operands; FP64: 0).  C must not overlap A, B or ws. */
size_t fb_matmul_workspace_bytes(int dtype, int64_t m, int64_t n, int64_t k);

/* BF16 GEMM: C[m][n] (float32) = A[m][k] * op(B), A and B bfloat16 (raw
 * 16-bit storage), exact BF16 products accumulated in FP32 on tcgen05 (kind::f16, CTA pairs),
 * partial sums promoted to round-to-nearest FP32 registers every 1024 k (FB_BF16_KP = 16 k-blocks
 * of 64).  b_transposed = 1: B is
 * given K-major as [n][k] (ldb >= k); 0: B is [k][n] (ldb >= n) and is transposed into ws.
 * A, B, C 16-byte aligned; lda*2, ldb*2, ldc*4 multiples of 16.  ws:
 * fb_matmul_bf16_workspace_bytes(b_transposed, m, n, k) bytes (0 when b_transposed). */
size_t fb_matmul_bf16_workspace_bytes(int b_transposed, int64_t m, int64_t n, int64_t k);
fb_status fb_matmul_bf16(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                         int b_transposed, void* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream);

/* BLAS-style variant: C = alpha op(A) op(B) + beta C, op(X) = X (trans 0) or
 * X^T (trans 1); op(A) is m x k (A stored m x k, lda >= k; or k x m, lda >= m), op(B) is k x n
 * (B stored k x n, ldb >= n; or n x k, ldb >= k).  Same arithmetic and accuracy as fb_matmul
 * (the same kernels: a transposed operand is read in its stored orientation -- by the FP64
 * kernel's tile loads, by the FP32 TF32 split -- and alpha, beta are applied in the kernels'
 * epilogue in FP32 / FP64; (alpha, beta) = (1, 0) with no transposes is bitwise fb_matmul).
 * beta == 0: C is not read (NaN in C does not propagate); alpha == 0: A and B are not read
 * (C = beta C).  Alignment rules as fb_matmul.  ws: fb_gemm_workspace_bytes(...) bytes (the
 * fb_matmul workspace: FP32 split operands; 0 for FP64, ws may then be NULL). */
size_t fb_gemm_workspace_bytes(int dtype, int transA, int transB, int64_t m, int64_t n, int64_t k);
fb_status fb_gemm(int dtype, int transA, int transB, int64_t m, int64_t n, int64_t k, double alpha,
                  const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                  int64_t ldc, void* ws, size_t ws_bytes, void* stream);
fb_status fb_matmul(int dtype, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                    const void* B, int64_t ldb, void* C, int64_t ldc, void* ws,
                    size_t ws_bytes, void* stream);

/* The two steps of the FB_F32 path, exposed so a caller can reuse a split operand (e.g. a
 * broadcast B) and a harness can time the tensor-core kernel alone.
 * fb_tf32_split: X (rows x cols, ldx) -> hi, lo with hi = rna_tf32(x), lo = rna_tf32(x - hi)
 *   (FP32 bit patterns with the low 13 mantissa bits zero).  transpose = 0 writes hi/lo as
 *   rows x cols with leading dim ld_out (>= cols); transpose = 1 writes them as cols x rows
 *   (ld_out >= rows).  ld_out*4 must be a multiple of 16.
 * fb_matmul_3xtf32_presplit: C[m][n] = Ah*Bh^T + Ah*Bl^T + Al*Bh^T where Ah/Al are m x k
 *   (ld lda) and Bh/Bl are n x k (ld ldb), i.e. both K-major, as produced by fb_tf32_split
 *   (A with transpose = 0, B with transpose = 1).  lda*4, ldb*4, ldc*4 multiples of 16. */
fb_status fb_tf32_split(int transpose, int64_t rows, int64_t cols, const float* X, int64_t ldx,
                        float* hi, float* lo, int64_t ld_out, void* stream);
fb_status fb_matmul_3xtf32_presplit(int64_t m, int64_t n, int64_t k, const float* Ah,
                                    const float* Al, int64_t lda, const float* Bh,
                                    const float* Bl, int64_t ldb, float* C, int64_t ldc,
                                    void* stream);

/* ------------------------------------------------------------------ host interface
 * The C-1 "connect the host program" form including the CPU<->GPU transfer the
 * paper names as the overhead of naive offload: HOST input -> H2D -> the block ->
 * D2H -> HOST output, all on `stream`; returns after the result is in host memory.
 * Host buffers should be pinned (cudaHostAlloc / torch pin_memory) for full bandwidth.
 * dev: caller-owned DEVICE scratch of *_host_workspace_bytes bytes (holds the device
 * copies and the block's own workspace). */
size_t fb_fft2d_host_workspace_bytes(int64_t n0, int64_t n1);
fb_status fb_fft2d_host(const void* x_host, void* y_host, int64_t n0, int64_t n1, int inverse,
                        void* dev, size_t dev_bytes, void* stream);
/* Streaming host form: `batch` independent n0 x n1 transforms, x_host/y_host hold them back to
 * back (batch * n0 * n1 complex64 each, pinned for overlap).  Two device slots (dev: caller-owned
 * DEVICE scratch of fb_fft2d_host_batch_workspace_bytes = 2 x the fb_fft2d_host scratch) alternate
 * between `stream` and a library-owned auxiliary stream, so transform i+1's H2D copy overlaps
 * transform i's D2H copy (PCIe is full duplex) with the kernels in between: the offload pipeline
 * that hides the transfer overhead P:43 names.  Ordered after prior work on `stream`; returns
 * after every result is in host memory.  Errors: as fb_fft2d_host; batch < 1 is
 * FB_ERR_INVALID_VALUE.  Calls are serialised per process (one pipeline at a time). */
size_t fb_fft2d_host_batch_workspace_bytes(int64_t n0, int64_t n1);
fb_status fb_fft2d_host_batch(const void* x_host, void* y_host, int64_t n0, int64_t n1, int64_t batch,
                              int inverse, void* dev, size_t dev_bytes, void* stream);
size_t fb_matmul_host_workspace_bytes(int dtype, int64_t m, int64_t n, int64_t k);
fb_status fb_matmul_host(int dtype, int64_t m, int64_t n, int64_t k, const void* A_host,
                         const void* B_host, void* C_host, void* dev, size_t dev_bytes,
                         void* stream);

/* ------------------------------------------------------------------ LU block
 * The paper's actual matrix workload: "LU decomposition processing of 2048*2048 orthogonal
 * matrix data", replaced there by cuSOLVER getrf; reading R19.
 * P A = L U in place on the row-major n x n matrix A (device, leading dim lda, 16-byte
 * aligned, lda even): L unit lower (strictly below the diagonal), U upper.  LAPACK getrf
 * pivoting: at step k the pivot is the FIRST row p >= k of largest |A[p][k]|; whole rows are
 * swapped; ipiv[k] = p (device int32[n], 0-based).  *info (device int32) = 0, or k+1 for the
 * first exactly-zero pivot (that step is skipped, as LAPACK).  Multipliers are formed with the
 * pivot's reciprocal when |pivot| >= DBL_MIN (dgetf2's sfmin rule).  dtype FB_F64 only;
 * n <= 4096.  ws: fb_lu_workspace_bytes(dtype, n) bytes (currently 0).
 * Execution: a look-ahead schedule on the caller's stream and an internal per-thread stream
 * (joined back before return, in stream order), captured on first use for each (A, n, lda,
 * ipiv, info) into a cached CUDA graph and replayed on later calls with the same buffers. */
size_t fb_lu_workspace_bytes(int dtype, int64_t n);
fb_status fb_lu(int dtype, int64_t n, void* A, int64_t lda, int32_t* ipiv, int32_t* info, void* ws,
                size_t ws_bytes, void* stream);

/* NR-compatible shim (the paper's C-1/C-2 interface matching, for the
 * Numerical Recipes in C applications it offloads): the argument list of NR's
 *     void fourn(float data[], unsigned long nn[], int ndim, int isign)
 * so a rewritten call site needs no other change.  NR conventions: 1-based arrays (data[1] is
 * the real part of the first element, nn[1..ndim] are the sizes, nn[1] the slowest index),
 * complex interleaved, isign = +1 computes sum x exp(+2 pi i k.n/N) and isign = -1 the
 * exp(-2 pi i ...) transform, both UNSCALED, in place on the host array.  ndim is 1 or 2;
 * sizes powers of two <= 16384.  Host data is copied to the GPU, transformed with the same
 * kernels as fb_fft2d, and copied back (the transfers the paper counts); the shim owns
 * a cached device staging buffer (it has no way to receive one) and synchronises the host.
 * Returns an fb_status (NR's fourn returns void; callers that ignore it keep NR semantics). */
fb_status fb_nr_fourn(float data[], const unsigned long nn[], int ndim, int isign);

/* ------------------------------------------------------------------ multi-GPU
 * One process per GPU.  Rank 0 calls fb_comm_unique_id and the caller distributes the
 * 128 bytes (e.g. torch.distributed broadcast); every rank then calls fb_comm_init.
 * An fb_comm wraps an NCCL communicator bound to `device`; use it from one stream at a
 * time. */
typedef struct fb_comm fb_comm;
size_t fb_comm_unique_id_bytes(void);
fb_status fb_comm_unique_id(void* uid_out /* fb_comm_unique_id_bytes() bytes */);
fb_status fb_comm_init(fb_comm** comm, int nranks, int rank, const void* uid, int device);
fb_status fb_comm_destroy(fb_comm* comm);
int fb_comm_rank(const fb_comm* comm);
int fb_comm_size(const fb_comm* comm);

/* Slab-sharded 2D FFT over P = comm size ranks (north_star (4), reading R8).
 * Rank r owns rows [r n0/P, (r+1) n0/P) of the natural n0 x n1 array, stored as an
 * (n0/P) x n1 row-major slab.  The forward transform returns the COLUMN slab: rank r
 * receives all n0 rows of columns [r n1/P, (r+1) n1/P) of Y, stored row-major as an
 * n0 x (n1/P) array.  fb_ifft2d_slab is the exact inverse: column slab in, natural row
 * slab out (scaled by 1/(n0 n1)).  Requires n0 % P == 0 and n1 % P == 0.  x and out must
 * not overlap.  ws: fb_fft2d_slab_workspace_bytes(P, n0, n1) device bytes.
 *
 * The global transpose runs one of two ways (same kernels, same results bit for bit):
 *   fused (default when every rank is NVLink/NVSwitch load-store reachable -- NCCL LSA team =
 *     world -- and NCCL symmetric memory is available): the row pass stores each column block
 *     straight into its owner's symmetric receive window (forward), or loads it from there
 *     (inverse), over NVLink; two NCCL device-API LSA barriers per call order the windows.
 *     The window (n0 n1 / P elements per rank) is owned by the communicator, allocated
 *     collectively on the first call that needs it (every rank must make the same calls).
 *   NCCL: row pass packs per-peer blocks into ws, one ncclAlltoAll, column pass.
 * fb_comm_fused reports the mode (1 fused, 0 NCCL; env FB_SLAB_FUSED=0 forces NCCL) and
 * fb_comm_fused_detail why fused is off. */
size_t fb_fft2d_slab_workspace_bytes(int nranks, int64_t n0, int64_t n1);
fb_status fb_fft2d_slab(fb_comm* comm, const void* x_rows, void* y_cols, int64_t n0, int64_t n1,
                        void* ws, size_t ws_bytes, void* stream);
fb_status fb_ifft2d_slab(fb_comm* comm, const void* y_cols, void* x_rows, int64_t n0, int64_t n1,
                         void* ws, size_t ws_bytes, void* stream);
int fb_comm_fused(fb_comm* comm);
const char* fb_comm_fused_detail(const fb_comm* comm);

/* Single-GPU model of the fused slab path for P virtual ranks (test hook, no communicator):
 * runs, rank after rank on `stream`, exactly the kernels and peer addressing the P ranks run,
 * with rank d's receive window = win + d * (n0 n1 / P) elements (win: n0 n1 complex64).
 * Forward: x = the full n0 x n1 array (rank r's slab = rows [r n0/P, (r+1) n0/P)); y = the P
 * column slabs one after another ([d][n0][n1/P]).  Inverse (inverse = 1): y in, x out.
 * ws: fb_fft2d_slab_workspace_bytes(P, n0, n1) bytes (four-step scratch). */
fb_status fb_fft2d_slab_model(int nranks, int inverse, void* x, void* y, int64_t n0, int64_t n1, void* win,
                              void* ws, size_t ws_bytes, void* stream);

/* Row-block GEMM (north_star (4), reading R18): rank r owns A rows and C rows
 * [r m/P, (r+1) m/P) as (m/P) x k and (m/P) x n row-major blocks; B (k x n) lives on
 * `root` and is broadcast (ncclBroadcast, inside the call) into every rank's B buffer
 * (on non-root ranks B is a receive buffer of k x n elements with leading dim ldb).
 * Requires m % P == 0.  ws: fb_matmul_rowblock_workspace_bytes(...) device bytes. */
size_t fb_matmul_rowblock_workspace_bytes(int nranks, int dtype, int64_t m, int64_t n, int64_t k);
fb_status fb_matmul_rowblock(fb_comm* comm, int dtype, int64_t m, int64_t n, int64_t k,
                             const void* A_rows, int64_t lda, void* B, int64_t ldb, int root,
                             void* C_rows, int64_t ldc, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FB_H */
