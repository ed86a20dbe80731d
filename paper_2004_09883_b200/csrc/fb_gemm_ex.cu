// fb_gemm_ex.cu -- BLAS-style variant of the matrix block: C = alpha op(A)
// op(B) + beta C with op = identity or transpose, FP32 (3xTF32) and FP64 (DMMA).
//
// No extra HBM pass for either feature: a transposed operand is read in its stored orientation
// (FP64: the DMMA kernel's tile loads; FP32: the TF32 split, which writes K-major hi/lo from
// either orientation), and alpha/beta are applied in the GEMM kernels' epilogue
// (gemm_ex_device, fb_gemm.cu).  C is not read when beta == 0, as in BLAS, so NaN/Inf in an
// uninitialised C do not propagate; alpha == 0 skips the product and A, B are not read
// (C = beta C in one streaming pass).
#include <stdint.h>

#include "fb_common.cuh"

namespace fb {

// C = beta C (beta == 0: C = 0, C not read) -- the alpha == 0 case
template <typename T>
__global__ void __launch_bounds__(256) scale_kernel(T* __restrict__ C, int64_t ldc, int64_t m, int64_t n, T beta) {
    const int64_t total = m * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        C[i * ldc + j] = (beta == T(0)) ? T(0) : beta * C[i * ldc + j];
    }
}

static size_t gemm_ex_ws(int dtype, int64_t m, int64_t n, int64_t k) { return gemm_ws_bytes(dtype, m, n, k); }

template <typename T>
static fb_status gemm_ex_typed(int dtype, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
                               const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                               int64_t ldc, void* ws, size_t ws_bytes, const DeviceState* st, cudaStream_t s) {
    if (alpha != 0.0)
        return gemm_ex_device(dtype, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st, s);
    const int64_t total = m * n;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 4 * 148 * 8) blocks = 4 * 148 * 8;
    scale_kernel<T><<<(unsigned)blocks, 256, 0, s>>>((T*)C, ldc, m, n, (T)beta);
    FB_LAUNCH_CHECK("scale_kernel");
    return FB_OK;
}

}  // namespace fb

using namespace fb;

extern "C" {

size_t fb_gemm_workspace_bytes(int dtype, int transA, int transB, int64_t m, int64_t n, int64_t k) {
    if ((dtype != FB_F32 && dtype != FB_F64) || m <= 0 || n <= 0 || k <= 0) return 0;
    return gemm_ex_ws(dtype, m, n, k);
}

fb_status fb_gemm(int dtype, int transA, int transB, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                  int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc, void* ws,
                  size_t ws_bytes, void* stream) {
    clear_error();
    if (dtype != FB_F32 && dtype != FB_F64) {
        set_error("dtype must be FB_F32 or FB_F64");
        return FB_ERR_INVALID_VALUE;
    }
    if ((transA != 0 && transA != 1) || (transB != 0 && transB != 1)) {
        set_error("transA / transB must be 0 or 1");
        return FB_ERR_INVALID_VALUE;
    }
    if (m <= 0 || n <= 0 || k <= 0) {
        set_error("m, n, k must be >= 1");
        return FB_ERR_INVALID_VALUE;
    }
    if (!A || !B || !C) {
        set_error("null operand");
        return FB_ERR_INVALID_VALUE;
    }
    const int64_t a_cols = transA ? m : k, a_rows = transA ? k : m;
    const int64_t b_cols = transB ? k : n, b_rows = transB ? n : k;
    if (lda < a_cols || ldb < b_cols || ldc < n) {
        set_error("leading dimensions too small");
        return FB_ERR_INVALID_VALUE;
    }
    const int64_t es = dtype == FB_F32 ? 4 : 8;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C) || (lda * es) % 16 || (ldb * es) % 16 || (ldc * es) % 16) {
        set_error("operands must be 16-byte aligned and ld*elemsize a multiple of 16");
        return FB_ERR_MISALIGNED;
    }
    const size_t cbytes = (size_t)((m - 1) * ldc + n) * es;
    if (ranges_overlap(C, cbytes, A, (size_t)((a_rows - 1) * lda + a_cols) * es) ||
        ranges_overlap(C, cbytes, B, (size_t)((b_rows - 1) * ldb + b_cols) * es)) {
        set_error("C overlaps A or B");
        return FB_ERR_INVALID_VALUE;
    }
    const size_t need = gemm_ex_ws(dtype, m, n, k);
    if ((need && !ws) || ws_bytes < need || !aligned16(ws)) {
        set_error("workspace of %zu bytes (16B aligned) required, got %zu", need, ws_bytes);
        return FB_ERR_WORKSPACE;
    }
    if (need && ranges_overlap(ws, need, C, cbytes)) {
        set_error("workspace overlaps C");
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    if (dtype == FB_F32)
        return gemm_ex_typed<float>(dtype, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st,
                                    (cudaStream_t)stream);
    return gemm_ex_typed<double>(dtype, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, ws_bytes, st,
                                 (cudaStream_t)stream);
}

}  // extern "C"
