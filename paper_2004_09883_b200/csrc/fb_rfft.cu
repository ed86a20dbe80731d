// fb_rfft.cu -- real-input 2D FFT (the paper's vibration signals are real,
// P:149).  X[k0][k1] for k1 = 0..n1/2 (the Hermitian half, numpy rfft2 / cuFFT R2C layout).
//
// Forward: a real row of length n1 is read as h = n1/2 complex values z[t] = x[2t] + i x[2t+1]
// (the same bytes, no copy) -> length-h row FFT Z -> per row the split
//   E[k] = (Z[k] + conj Z[h-k]) / 2,  O[k] = (Z[k] - conj Z[h-k]) / (2i),  X[k] = E[k] + W_n1^k O[k]
// for k = 0..h (Z periodic in h) -> length-n0 column FFTs over the h+1 columns.
// Inverse: column inverse FFTs (unscaled) -> per row E[k] = (Y[k] + conj Y[h-k]) / 2,
// O[k] = (Y[k] - conj Y[h-k]) W_n1^-k / 2, Z[k] = E[k] + i O[k] -> length-h inverse row FFT
// with the exact power-of-two scale 2/(n0 n1) -> the complex values are the real row pairs.
// The line passes are the fb_fft2d kernels; the split/merge is one streaming kernel each.
#include <stdint.h>

#include "fb_common.cuh"

namespace fb {

__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cmulf2(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Z [n0][h] -> X [n0][h + 1]
__global__ void __launch_bounds__(256) rfft_split_kernel(const float2* __restrict__ Z, float2* __restrict__ X,
                                                         int64_t n0, int64_t h, int tw_shift,
                                                         const float2* __restrict__ tw) {
    const int64_t w = h + 1, total = n0 * w;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / w, k = e % w;
        const float2 a = Z[r * h + (k == h ? 0 : k)];
        const float2 b = conjf2(Z[r * h + (k == 0 ? 0 : h - k)]);
        const float2 E = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
        const float2 d = make_float2(0.5f * (a.x - b.x), 0.5f * (a.y - b.y));  // (Z - conj Z') / 2
        const float2 O = make_float2(d.y, -d.x);                                 // d / i
        const float2 wk = __ldg(tw + ((k << tw_shift) & (kTwN - 1)));            // W_n1^k (k = h: -1)
        const float2 t = (k == h) ? make_float2(-O.x, -O.y) : cmulf2(wk, O);
        X[r * w + k] = make_float2(E.x + t.x, E.y + t.y);
    }
}

// Y [n0][h + 1] -> Z [n0][h]
__global__ void __launch_bounds__(256) rfft_merge_kernel(const float2* __restrict__ Y, float2* __restrict__ Z,
                                                         int64_t n0, int64_t h, int tw_shift,
                                                         const float2* __restrict__ tw) {
    const int64_t w = h + 1, total = n0 * h;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / h, k = e % h;
        const float2 a = Y[r * w + k];
        const float2 b = conjf2(Y[r * w + (h - k)]);
        const float2 E = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
        const float2 d = make_float2(0.5f * (a.x - b.x), 0.5f * (a.y - b.y));
        const float2 wk = __ldg(tw + ((k << tw_shift) & (kTwN - 1)));
        const float2 O = cmulf2(d, conjf2(wk));                        // d W_n1^-k
        Z[r * h + k] = make_float2(E.x - O.y, E.y + O.x);              // E + i O
    }
}

static size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

static fb_status check_rfft(int64_t n0, int64_t n1) {
    if (n0 < 1 || n1 < 2) {
        set_error("rfft2d needs n0 >= 1 and n1 >= 2");
        return FB_ERR_INVALID_VALUE;
    }
    if (!is_pow2(n0) || !is_pow2(n1) || n0 > kTwN || n1 > kTwN) {
        set_error("FFT sizes must be powers of two in [1, %d] (n1 >= 2)", kTwN);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    return FB_OK;
}

struct RfftWs {
    size_t z, t, f, total;
};
static RfftWs rfft_ws(int64_t n0, int64_t n1) {
    const int64_t h = n1 / 2;
    RfftWs L;
    L.z = al256((size_t)n0 * h * sizeof(float2));
    L.t = al256((size_t)n0 * (h + 1) * sizeof(float2));
    L.f = (ilog2(n0) > 12) ? L.t : 0;  // four-step column split scratch
    L.total = L.z + L.t + L.f;
    return L;
}

static fb_status row_pass(const float2* in, float2* out, int64_t n0, int64_t h, bool inverse, float scale,
                          const DeviceState* st, cudaStream_t s) {
    FftPass p{};
    p.in = in;
    p.out = out;
    p.log2L = ilog2(h);
    p.nlines = n0;
    p.g_shift = 0;
    p.lin.hi = p.lout.hi = h;
    p.lin.kb_shift = p.lout.kb_shift = 30;
    p.lin.es = p.lout.es = 1;
    p.conj_in = inverse;
    p.conj_out = inverse;
    p.scale = scale;
    return launch_fft_pass(p, st, s);
}

static int64_t grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    return b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b);
}

}  // namespace fb

using namespace fb;

extern "C" {

size_t fb_rfft2d_workspace_bytes(int64_t n0, int64_t n1) {
    if (check_rfft(n0, n1) != FB_OK) return 0;
    return rfft_ws(n0, n1).total;
}

fb_status fb_rfft2d(const void* x, void* y, int64_t n0, int64_t n1, void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    FB_TRY(check_rfft(n0, n1));
    if (!x || !y) {
        set_error("null x or y");
        return FB_ERR_INVALID_VALUE;
    }
    if (!aligned16(x) || !aligned16(y) || !aligned16(ws)) {
        set_error("x, y and ws must be 16-byte aligned");
        return FB_ERR_MISALIGNED;
    }
    const int64_t h = n1 / 2;
    const RfftWs L = rfft_ws(n0, n1);
    const size_t xb = (size_t)n0 * n1 * sizeof(float), yb = (size_t)n0 * (h + 1) * sizeof(float2);
    if (!ws || ws_bytes < L.total) {
        set_error("workspace of %zu bytes required, got %zu", L.total, ws_bytes);
        return FB_ERR_WORKSPACE;
    }
    if (ranges_overlap(x, xb, y, yb) || ranges_overlap(ws, L.total, x, xb) || ranges_overlap(ws, L.total, y, yb)) {
        set_error("x, y and ws must not overlap");
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    float2* Z = (float2*)ws;
    FB_TRY(row_pass((const float2*)x, Z, n0, h, false, 1.f, st, s));
    const int64_t tot = n0 * (h + 1);
    rfft_split_kernel<<<(unsigned)grid_for(tot), 256, 0, s>>>(Z, (float2*)y, n0, h, kTwLog2 - ilog2(n1),
                                                              st->twiddles);
    FB_LAUNCH_CHECK("rfft_split_kernel");
    float2* F = L.f ? (float2*)((char*)ws + L.z + L.t) : nullptr;
    return fft_columns((const float2*)y, (float2*)y, n0, h + 1, h + 1, h + 1, false, false, 1.f, F, st, s);
}

fb_status fb_irfft2d(const void* y, void* x, int64_t n0, int64_t n1, void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    FB_TRY(check_rfft(n0, n1));
    if (!x || !y) {
        set_error("null x or y");
        return FB_ERR_INVALID_VALUE;
    }
    if (!aligned16(x) || !aligned16(y) || !aligned16(ws)) {
        set_error("x, y and ws must be 16-byte aligned");
        return FB_ERR_MISALIGNED;
    }
    const int64_t h = n1 / 2;
    const RfftWs L = rfft_ws(n0, n1);
    const size_t xb = (size_t)n0 * n1 * sizeof(float), yb = (size_t)n0 * (h + 1) * sizeof(float2);
    if (!ws || ws_bytes < L.total) {
        set_error("workspace of %zu bytes required, got %zu", L.total, ws_bytes);
        return FB_ERR_WORKSPACE;
    }
    if (ranges_overlap(x, xb, y, yb) || ranges_overlap(ws, L.total, x, xb) || ranges_overlap(ws, L.total, y, yb)) {
        set_error("x, y and ws must not overlap");
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    float2* Z = (float2*)ws;
    float2* T = (float2*)((char*)ws + L.z);
    float2* F = L.f ? (float2*)((char*)ws + L.z + L.t) : nullptr;
    // column inverse FFTs (unscaled; conj in, conj out) of the h+1 columns into T
    FB_TRY(fft_columns((const float2*)y, T, n0, h + 1, h + 1, h + 1, true, true, 1.f, F, st, s));
    rfft_merge_kernel<<<(unsigned)grid_for(n0 * h), 256, 0, s>>>(T, Z, n0, h, kTwLog2 - ilog2(n1), st->twiddles);
    FB_LAUNCH_CHECK("rfft_merge_kernel");
    const float scale = (float)(2.0 / ((double)n0 * (double)n1));  // power of two: exact
    return row_pass(Z, (float2*)x, n0, h, true, scale, st, s);
}

}  // extern "C"
