// fb_common.cuh -- shared host/device plumbing for libfb (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>

#include "../../include/fb.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libfb kernels are written for sm_100a only (compile with -gencode arch=compute_100a,code=sm_100a)"
#endif

namespace fb {

// ---------------------------------------------------------------- error reporting
void set_error(const char* fmt, ...);
void clear_error();
extern std::atomic<uint64_t> g_launches;

#define FB_CUDA_TRY(expr)                                                                  \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess) {                                                           \
            ::fb::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                            __LINE__);                                                     \
            return FB_ERR_CUDA;                                                            \
        }                                                                                  \
    } while (0)

// Check the launch that was just enqueued and count it.
#define FB_LAUNCH_CHECK(name)                                                              \
    do {                                                                                   \
        cudaError_t _e = cudaGetLastError();                                               \
        if (_e != cudaSuccess) {                                                           \
            ::fb::set_error("launch of %s failed: %s", name, cudaGetErrorString(_e));       \
            return FB_ERR_CUDA;                                                            \
        }                                                                                  \
        ::fb::g_launches.fetch_add(1, std::memory_order_relaxed);                          \
    } while (0)

#define FB_TRY(expr)                      \
    do {                                  \
        fb_status _s = (expr);            \
        if (_s != FB_OK) return _s;       \
    } while (0)

// ---------------------------------------------------------------- A/B knobs
// Tuning switches for A/B measurements (defaults = the tuned configuration).  They are read
// from the environment ONCE per process (first use, or fb_reload_knobs() -- the tests call it
// after changing the environment); no launch path calls getenv.  Result-altering timing
// decompositions (FB_FFT_DEBUG, FB_LU_DEBUG) are honoured only in builds compiled with
// -DFB_DEBUG_BUILD=1 (tools), never in the product library.
#ifndef FB_DEBUG_BUILD
#define FB_DEBUG_BUILD 0
#endif
struct Knobs {
    // FFT (fb_fft.cu, fb_fft_kern.cuh)
    int fft_stagger_ns = 600, fft_col_stg = -1, fft_pair2 = 2, fft_colpair = 0, fft_col_max_log2 = 12;
    int fft_4step_lb = -1, fft_pair = 1, fft_pair_max_log2 = 11, fft_no_tma_col = 0, fft_col_c = 0;
    int fft_no_tma_row = 0, fft_col_nb = 0, fft_row_nb = 0, fft_no_tma = 0, fft_longrow = 1, fft_pair_tma = 1;
    int fft_no_pdl = 0, fft_debug = 0, fft_sub = 0;  // FB_FFT_SUB: 0 auto, 1 / 3 forced
    int fft_sub_ilv = 0, fft_col32 = 1, fft_row16k = 1, fft_row16k_cps = 2;
    int fft_mixed = 1, fft_mr_small = 1024;  // 7-smooth non-power-of-two lines as mixed-radix Stockham (0: Bluestein)
    int fft_stagger_col = 300;  // radix-32 column pass stagger (ns; -1: as FB_FFT_STAGGER); 2048^2: 600 ns 32.68, 300 ns 32.37-32.53, 150 ns 32.39 us
    int fft_small = 16;  // 256 x 256 as one cluster kernel: cluster size 16 (8), 0 = two-pass path
    // multi-GPU (fb_comm.cu)
    int slab_fused = 1;
    int64_t rowblock_panel = 2048;  // same width as fb_matmul's N-panel launches (32768^3 at world 1: 307 -> 301 ms)
    // GEMM (fb_gemm.cu, fb_gemm_bf16.cu)
    int f64_cfg = 0, gemm_split2 = 0, gemm_splitv = 0, gemm_split_pdl = 0, gemm_1cta = 0, bf16_cluster = 2;
    int gemm_fused = 0, gemm_lo_prepass = 1, gemm_streamk = 0, gemm_lo_overlap = 0, gemm_persist = 0;
    int gemm_npanel = -1, gemm_raster_panel = 0, gemm_nt = 0, gemm_ahi_raw = 1;  // -1: auto N-panels (fb_gemm.cu)
    int bf16_persist = 1;  // 8192^3 0.820 -> 0.790 ms, 4096^3 0.145 -> 0.124 ms (interleaved A/B)
    // LU (fb_lu.cu)
    int lu_tma = 1, lu_debug = 0, lu_rank_simt = 1, lu_serial = 0, lu_lookahead = 1, lu_graph = 1;
};
const Knobs& knobs();
void reload_knobs();

// Per-device "done once" bit mask for cudaFuncSetAttribute and similar per-context setup
// (devices 0..31); atomic, so concurrent first calls at worst repeat the idempotent setup.
struct DevOnce {
    std::atomic<uint32_t> mask{0};
    static int dev() {
        int d = 0;
        cudaGetDevice(&d);
        return d & 31;
    }
    bool done(int d) const { return (mask.load() >> d) & 1u; }
    void set(int d) { mask.fetch_or(1u << d); }
};

// Per-device immutable state (twiddle table pointer, SM count, ...).
struct DeviceState {
    bool ready = false;
    int sm_count = 0;
    float2* twiddles = nullptr;  // 16384 entries, W[j] = exp(-2 pi i j / 16384)
    float2* stage_tw = nullptr;  // per-(line length, stage) contiguous twiddles (fb_fft.cu)
    cudaStream_t aux = nullptr;  // second slot of the host-batch copy/compute pipeline
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};  // copy-order chain
};
int64_t stage_tw_total();
void stage_tw_index(int32_t* idx);
fb_status ensure_device(int* dev_out, DeviceState** st_out);

constexpr int kTwLog2 = 14;
constexpr int kTwN = 1 << kTwLog2;  // twiddle table resolution (max line length)

inline bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
inline int ilog2(int64_t n) {
    int l = 0;
    while ((int64_t(1) << l) < n) ++l;
    return l;
}
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool ranges_partially_overlap(const void* a, size_t na, const void* b, size_t nb) {
    uintptr_t a0 = (uintptr_t)a, a1 = a0 + na, b0 = (uintptr_t)b, b1 = b0 + nb;
    bool overlap = a0 < b1 && b0 < a1;
    return overlap && !(a0 == b0 && na == nb);
}
inline bool ranges_overlap(const void* a, size_t na, const void* b, size_t nb) {
    uintptr_t a0 = (uintptr_t)a, a1 = a0 + na, b0 = (uintptr_t)b, b1 = b0 + nb;
    return na && nb && a0 < b1 && b0 < a1;
}

// ---------------------------------------------------------------- FFT internals
// One "pass" = length-L FFTs along a set of lines (see fb_fft.cu for the addressing).
struct LineMap {
    // line g -> base = (g >> g_shift) * hi + (g & ((1<<g_shift)-1)) * lo
    int64_t hi, lo;
    // element k -> (k & ((1<<kb_shift)-1)) * es + (k >> kb_shift) * bs
    int kb_shift;
    int64_t es, bs;
};
constexpr int kMaxPeers = 8;  // one NVLink/NVSwitch node
struct FftPass {
    const float2* in;
    float2* out;
    int log2L;
    int64_t nlines;
    int g_shift;
    LineMap lin, lout;
    int conj_in, conj_out;
    float scale;
    int tw4_log2N;  // >0: four-step twiddle W_N^{(g >> g_shift) * k} on the output, N = 2^tw4_log2N
    int col_like;   // 1: adjacent lines are adjacent in memory (pick a wide C for coalescing)
    int debug;      // timing decomposition only (FB_FFT_DEBUG): 1 skip stages, 2 skip loads, 4 skip stores
    int stagger_ns; // persistent TMA pass: CTA slot s (= blockIdx / SMs) delays its first load by s * this
    int sm_count;   //   (set by launch_fft_pass)
    int pair_half_shfl; // pair step: 0 lane exchange per element, 1 per element pair, 2 fused into the
                        //   last row stage, no exchange (default; knob FB_FFT_PAIR2)
    int col_pair_last; // column pass: last stage on column pairs with 16-byte shared accesses (knob)
    int col_stg;    // persistent column pass: 1 outputs by direct stores, 0 X + TMA store, -1 auto
    int pair_log2N; // >0: lines come in pairs (g = 2q + c, rows q and q + N/2 of an N-long column);
                    // after the row FFT, the radix-2 column butterfly across the pair and the
                    // four-step twiddle W_N^{q k_a} are applied (first step of a 2 x N/2 split)
    // Peer mode of the fused slab transpose (fb_comm.cu): element k of a line lives in the
    // column block d = k >> kb_shift, and block d is addressed from its own base peer[d] (a
    // pointer into GPU d's symmetric window, NVLink load/store) instead of base + d * bs.
    int peer_out, peer_in;
    float2* peer[kMaxPeers];
    // FB_FFT_TRACE builds only (tools/fft_trace.py): per-CTA timeline of the persistent pass,
    // 32 u64 per CTA at trace + (trace_slot * 1024 + blockIdx) * 32 (null: off)
    unsigned long long* trace;
    int trace_slot;
    int sub_ilv;  // persistent pass with sub-CTAs: warps interleaved across sub-CTAs (knob)
};
#ifndef FB_FFT_TRACE
#define FB_FFT_TRACE 0
#endif
extern unsigned long long* g_fft_trace_host;  // set by fb_debug_fft_trace (trace builds)
fb_status launch_fft_pass(const FftPass& p, const DeviceState* st, cudaStream_t s);

// Full single-GPU 2D FFT on device buffers (used by the API and the host/slab variants).
size_t fft2d_ws_bytes(int64_t n0, int64_t n1);
fb_status fft2d_device(const void* x, void* y, int64_t n0, int64_t n1, bool inverse, void* ws,
                       size_t ws_bytes, const DeviceState* st, cudaStream_t s, bool unscaled = false);
// Non-power-of-two sizes (fb_bluestein.cu): each dimension a power of two <= 16384 or any
// length <= 8192 (Bluestein chirp-z over power-of-two passes)
bool fft_size_ok(int64_t n);
// 256 x 256 in one thread-block-cluster kernel (fb_fft_small.cu)
bool fft_small_eligible(int64_t n0, int64_t n1);
fb_status fft2d_small(const float2* x, float2* y, bool inverse, float scale, const DeviceState* st, cudaStream_t s);
size_t bluestein_ws_bytes(int64_t n0, int64_t n1);
fb_status fft2d_bluestein(const void* x, void* y, int64_t n0, int64_t n1, bool inverse, void* ws, size_t ws_bytes,
                          const DeviceState* st, cudaStream_t s, bool unscaled);
// Column transform of an n0 x ncols block with leading dimension ld (in place allowed when
// n0 <= 4096); used by 2D and slab paths.
fb_status fft_columns(const float2* in, float2* out, int64_t n0, int64_t ncols, int64_t ld_in,
                      int64_t ld_out, bool conj_in, bool conj_out, float scale, float2* tmp,
                      const DeviceState* st, cudaStream_t s);

// ---------------------------------------------------------------- GEMM internals
size_t gemm_ws_bytes(int dtype, int64_t m, int64_t n, int64_t k);
fb_status gemm_device(int dtype, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                      const void* B, int64_t ldb, void* C, int64_t ldc, void* ws,
                      size_t ws_bytes, const DeviceState* st, cudaStream_t s);
// fb_gemm's core: C = alpha op(A) op(B) + beta C, op(A) = A (ta = 0, stored m x k) or A^T (ta = 1,
// stored k x m), op(B) likewise (stored k x n / n x k).  The orientation is taken by the operand
// loads (FP64) or the TF32 split (FP32), alpha/beta by the kernels' epilogue (C is not read when
// beta == 0); alpha must be nonzero.  ws: gemm_ws_bytes.
fb_status gemm_ex_device(int dtype, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                         int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc, void* ws,
                         size_t ws_bytes, const DeviceState* st, cudaStream_t s);

// G1: TF32 split (transpose=0: X[rows][cols] -> hi/lo [rows][ldo]; transpose=1: -> [cols][ldo])
fb_status tf32_split_device(int transpose, int64_t rows, int64_t cols, const float* X, int64_t ldx, float* hi,
                            float* lo, int64_t ldo, const DeviceState* st, cudaStream_t s, bool trunc_hi = false);
// raw-hi mode of G1: lo = rna(x - trunc(x)) only (the raw X is the hi operand; reading R21)
fb_status tf32_lo_device(int64_t rows, int64_t cols, const float* X, int64_t ldx, float* lo, int64_t ldo,
                         cudaStream_t s);
// G2-G4: C = Ah*Bh^T + Ah*Bl^T + Al*Bh^T with K-major split operands (A: m x k, B^T: n x k)
// G1-G4 fused: C = A B (row-major FP32 A [m][k], B [k][n]), no workspace (fb_gemm_fused.cu)
size_t gemm_3xtf32_fused_ws_bytes(int64_t m, int64_t n, int64_t k);
fb_status gemm_3xtf32_fused_device(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                                   int64_t ldb, float* C, int64_t ldc, void* ws, size_t ws_bytes, cudaStream_t s);
fb_status gemm_3xtf32_presplit_device(int64_t m, int64_t n, int64_t k, const float* Ah, const float* Al,
                                      int64_t lda, const float* Bh, const float* Bl, int64_t ldb, float* C,
                                      int64_t ldc, cudaStream_t s, float alpha = 1.f, float beta = 0.f,
                                      int64_t lda_hi = -1);  // lda_hi: row pitch of Ah if != lda

}  // namespace fb
