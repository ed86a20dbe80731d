// fb_gemm_ex.cu -- BLAS-style variant of the matrix block: C = alpha op(A)
// op(B) + beta C with op = identity or transpose, FP32 (3xTF32) and FP64 (DMMA).
//
// Built from the fb_matmul core (gemm_device): a transposed operand is first materialised in
// the workspace (32x32 shared-memory tile transpose, coalesced on both sides), the product
// goes straight to C when (alpha, beta) = (1, 0) and otherwise to a workspace tile T, then
// C = alpha T + beta C in one streaming pass (C is not read when beta == 0, as in BLAS, so
// NaN/Inf in an uninitialised C do not propagate; alpha == 0 skips the product).
#include <stdint.h>

#include "fb_common.cuh"

namespace fb {

template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(const T* __restrict__ X, int64_t rows, int64_t cols,
                                                        int64_t ldx, T* __restrict__ Y, int64_t ldy) {
    __shared__ T tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t r = r0 + ty + j, c = c0 + tx;
        if (r < rows && c < cols) tile[ty + j][tx] = X[r * ldx + c];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t c = c0 + ty + j, r = r0 + tx;  // Y[c][r] = X[r][c]
        if (c < cols && r < rows) Y[c * ldy + r] = tile[tx][ty + j];
    }
}

template <typename T>
__global__ void __launch_bounds__(256) axpby_kernel(const T* __restrict__ P, int64_t ldp, T* __restrict__ C,
                                                    int64_t ldc, int64_t m, int64_t n, T alpha, T beta,
                                                    int use_p) {
    const int64_t total = m * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / n, j = e % n;
        const T p = use_p ? alpha * P[i * ldp + j] : T(0);
        C[i * ldc + j] = (beta == T(0)) ? p : p + beta * C[i * ldc + j];
    }
}

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
// leading dimension (elements) of a workspace temporary: rows padded to 16 bytes, the row
// alignment the fb_matmul kernels assume (float4 / TMA rows)
static int64_t ld16(int64_t x, size_t es) {
    const int64_t q = (int64_t)(16 / es);
    return (x + q - 1) / q * q;
}

struct GemmExLayout {
    size_t core, opa, opb, t, total;
};
static GemmExLayout gemm_ex_layout(int dtype, int ta, int tb, int64_t m, int64_t n, int64_t k) {
    const size_t es = dtype == FB_F32 ? 4 : 8;
    GemmExLayout L;
    L.core = align256(gemm_ws_bytes(dtype, m, n, k));
    L.opa = ta ? align256((size_t)m * (size_t)ld16(k, es) * es) : 0;
    L.opb = tb ? align256((size_t)k * (size_t)ld16(n, es) * es) : 0;
    L.t = align256((size_t)m * (size_t)ld16(n, es) * es);
    L.total = L.core + L.opa + L.opb + L.t;
    return L;
}

template <typename T>
static fb_status launch_transpose(const T* X, int64_t rows, int64_t cols, int64_t ldx, T* Y, int64_t ldy,
                                  cudaStream_t s) {
    dim3 g((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    if (g.y > 65535) {
        set_error("operand too tall for the transpose grid");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    transpose_kernel<T><<<g, 256, 0, s>>>(X, rows, cols, ldx, Y, ldy);
    FB_LAUNCH_CHECK("transpose_kernel");
    return FB_OK;
}

template <typename T>
static fb_status gemm_ex_typed(int dtype, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
                               const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                               int64_t ldc, void* ws, const GemmExLayout& L, const DeviceState* st,
                               cudaStream_t s) {
    char* w = (char*)ws;
    const T* a = (const T*)A;
    const T* b = (const T*)B;
    int64_t la = lda, lb = ldb;
    if (alpha != 0.0) {
        if (ta) {  // A stored k x m -> op(A) m x k
            T* at = (T*)(w + L.core);
            la = ld16(k, sizeof(T));
            FB_TRY(launch_transpose<T>(a, k, m, lda, at, la, s));
            a = at;
        }
        if (tb) {  // B stored n x k -> op(B) k x n
            T* bt = (T*)(w + L.core + L.opa);
            lb = ld16(n, sizeof(T));
            FB_TRY(launch_transpose<T>(b, n, k, ldb, bt, lb, s));
            b = bt;
        }
    }
    const bool plain = alpha == 1.0 && beta == 0.0;
    if (plain) return gemm_device(dtype, m, n, k, a, la, b, lb, C, ldc, ws, L.core, st, s);
    T* t = (T*)(w + L.core + L.opa + L.opb);
    const int64_t lt = ld16(n, sizeof(T));
    if (alpha != 0.0) FB_TRY(gemm_device(dtype, m, n, k, a, la, b, lb, t, lt, ws, L.core, st, s));
    const int64_t total = m * n;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 4 * 148 * 8) blocks = 4 * 148 * 8;
    axpby_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(t, lt, (T*)C, ldc, m, n, (T)alpha, (T)beta, alpha != 0.0);
    FB_LAUNCH_CHECK("axpby_kernel");
    return FB_OK;
}

}  // namespace fb

using namespace fb;

extern "C" {

size_t fb_gemm_workspace_bytes(int dtype, int transA, int transB, int64_t m, int64_t n, int64_t k) {
    if ((dtype != FB_F32 && dtype != FB_F64) || m <= 0 || n <= 0 || k <= 0) return 0;
    return gemm_ex_layout(dtype, transA != 0, transB != 0, m, n, k).total;
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
    const GemmExLayout L = gemm_ex_layout(dtype, transA, transB, m, n, k);
    if (!ws || ws_bytes < L.total || !aligned16(ws)) {
        set_error("workspace of %zu bytes (16B aligned) required, got %zu", L.total, ws_bytes);
        return FB_ERR_WORKSPACE;
    }
    if (ranges_overlap(ws, L.total, C, cbytes)) {
        set_error("workspace overlaps C");
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    if (dtype == FB_F32)
        return gemm_ex_typed<float>(dtype, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, L, st,
                                    (cudaStream_t)stream);
    return gemm_ex_typed<double>(dtype, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, L, st,
                                 (cudaStream_t)stream);
}

}  // extern "C"
