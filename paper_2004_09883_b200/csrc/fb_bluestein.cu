// fb_bluestein.cu -- the Fourier-transform block for sizes that are NOT
// powers of two (vibration records have arbitrary lengths).
//
// A length-n DFT along a line is evaluated with Bluestein's chirp-z identity
//     j k = (j^2 + k^2 - (k - j)^2) / 2  =>
//     X[k] = c[k] * sum_j (x[j] c[j]) * conj(c[k - j]),   c[j] = exp(-pi i j^2 / n),
// i.e. a linear convolution of length 2n - 1, done as a circular convolution of power-of-two
// length M >= 2n - 1 with the power-of-two passes of fb_fft_kern.cuh:
//     a = pad_M(x * c);  A = FFT_M(a);  B = A * H;  b = IFFT_M(B);  X = c * b[0 .. n)
// with H = FFT_M(h), h[j] = conj(c[j]) for 0 <= j < n, h[M - j] = conj(c[j]) for 0 < j < n.
// The chirp is formed from the exactly reduced integer j^2 mod 2n in FP64 (sincospi) and rounded
// once to FP32.  The inverse (sign +1) uses conj(DFT(conj X)); its 1/(n0 n1) is applied in the
// last step.  A 2D transform runs the rows, a tiled transpose, the (former) columns as rows, and
// a transpose back; a power-of-two dimension takes the ordinary pass.  Sizes: any n0, n1 with
// each non-power-of-two dimension <= 8192 (M <= 16384, the longest power-of-two pass).
#include <math.h>

#include "fb_common.cuh"

namespace fb {

constexpr int64_t kBluesteinMax = 8192;

static int64_t bs_len(int64_t n) {  // power-of-two convolution length for a length-n line
    int64_t m = 1;
    while (m < 2 * n - 1) m <<= 1;
    return m;
}

bool fft_size_ok(int64_t n) { return n >= 1 && (is_pow2(n) ? n <= kTwN : n <= kBluesteinMax); }

// workspace (float2 elements): P (batch x M conv rows, the larger dimension), T (transpose),
// chirp c and spectrum H for each non-power-of-two dimension
static int64_t bs_ws_elems(int64_t n0, int64_t n1) {
    const int64_t m0 = is_pow2(n0) ? 0 : bs_len(n0), m1 = is_pow2(n1) ? 0 : bs_len(n1);
    const int64_t p = (n0 * m1 > n1 * m0) ? n0 * m1 : n1 * m0;
    return p + n0 * n1 + (m0 + n0) + (m1 + n1) + 64;
}
size_t bluestein_ws_bytes(int64_t n0, int64_t n1) { return (size_t)bs_ws_elems(n0, n1) * sizeof(float2) + 256; }

// c[j] = exp(-pi i j^2 / n) (FP64, exact reduction of j^2 mod 2n), h = the wrapped conj chirp
__global__ void bs_chirp_kernel(float2* __restrict__ c, float2* __restrict__ h, int64_t n, int64_t M) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
        float2 hv = make_float2(0.f, 0.f);
        const int64_t jj = (j < n) ? j : ((M - j < n) ? M - j : -1);
        if (jj >= 0) {
            const int64_t e = (jj * jj) % (2 * n);
            double sn, cs;
            sincospi((double)e / (double)n, &sn, &cs);
            const float2 cv = make_float2((float)cs, (float)(-sn));  // exp(-pi i e / n)
            if (j < n) c[j] = cv;
            hv = make_float2(cv.x, -cv.y);                           // conj(c)
        }
        h[j] = hv;
    }
}

// P[b][j] = (conj? x : x)[b][j] * c[j] for j < n, 0 for n <= j < M
__global__ void bs_pad_kernel(const float2* __restrict__ x, int64_t batch, int64_t n, int64_t M,
                              const float2* __restrict__ c, float2* __restrict__ P, int conj_in) {
    const int64_t total = batch * M;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / M, j = e - b * M;
        float2 v = make_float2(0.f, 0.f);
        if (j < n) {
            float2 a = x[b * n + j];
            if (conj_in) a.y = -a.y;
            const float2 w = c[j];
            v = make_float2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
        }
        P[e] = v;
    }
}

// P[b][k] *= H[k]
__global__ void bs_mul_kernel(float2* __restrict__ P, int64_t batch, int64_t M, const float2* __restrict__ H) {
    const int64_t total = batch * M;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const float2 a = P[e], w = H[e % M];
        P[e] = make_float2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
    }
}

// y[b][k] = s * (conj?)(c[k] * P[b][k]) for k < n
__global__ void bs_crop_kernel(const float2* __restrict__ P, int64_t batch, int64_t n, int64_t M,
                               const float2* __restrict__ c, float2* __restrict__ y, int conj_out, float s) {
    const int64_t total = batch * n;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / n, k = e - b * n;
        const float2 a = P[b * M + k], w = c[k];
        float2 v = make_float2(a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x);
        if (conj_out) v.y = -v.y;
        y[e] = make_float2(v.x * s, v.y * s);
    }
}

// Y[c][r] = X[r][c] (rows x cols complex64), 32 x 32 tiles through shared memory
__global__ void __launch_bounds__(256) bs_transpose_kernel(const float2* __restrict__ X, int64_t rows, int64_t cols,
                                                           float2* __restrict__ Y) {
    __shared__ float2 tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t r = r0 + ty + j, cc = c0 + tx;
        if (r < rows && cc < cols) tile[ty + j][tx] = X[r * cols + cc];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t cc = c0 + ty + j, r = r0 + tx;
        if (cc < cols && r < rows) Y[cc * rows + r] = tile[tx][ty + j];
    }
}

static unsigned grid_for(int64_t work) {
    int64_t b = (work + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

// power-of-two FFT of `batch` contiguous lines of length L (in place allowed)
static fb_status pow2_rows(const float2* in, float2* out, int64_t batch, int64_t L, bool conj_in, bool conj_out,
                           float scale, const DeviceState* st, cudaStream_t s) {
    FftPass p{};
    p.in = in;
    p.out = out;
    p.log2L = ilog2(L);
    p.nlines = batch;
    p.g_shift = 0;
    p.lin.hi = L, p.lin.lo = 0, p.lin.kb_shift = 30, p.lin.es = 1, p.lin.bs = 0;
    p.lout = p.lin;
    p.conj_in = conj_in;
    p.conj_out = conj_out;
    p.scale = scale;
    return launch_fft_pass(p, st, s);
}

// DFT (sign -1, or +1 with inverse) of `batch` contiguous rows of length n: x -> y, times `scale`
static fb_status dft_rows(const float2* x, float2* y, int64_t batch, int64_t n, bool inverse, float scale,
                          float2* P, float2* c, float2* H, const DeviceState* st, cudaStream_t s) {
    if (is_pow2(n)) return pow2_rows(x, y, batch, n, inverse, inverse, scale, st, s);
    const int64_t M = bs_len(n);
    // chirp and filter spectrum H = FFT_M(h) (recomputed per call: one line of length M)
    bs_chirp_kernel<<<grid_for(M), 256, 0, s>>>(c, H, n, M);
    FB_LAUNCH_CHECK("bs_chirp_kernel");
    FB_TRY(pow2_rows(H, H, 1, M, false, false, 1.f, st, s));
    bs_pad_kernel<<<grid_for(batch * M), 256, 0, s>>>(x, batch, n, M, c, P, inverse ? 1 : 0);
    FB_LAUNCH_CHECK("bs_pad_kernel");
    FB_TRY(pow2_rows(P, P, batch, M, false, false, 1.f, st, s));
    bs_mul_kernel<<<grid_for(batch * M), 256, 0, s>>>(P, batch, M, H);
    FB_LAUNCH_CHECK("bs_mul_kernel");
    // IFFT_M = conj(FFT_M(conj)) / M  (M a power of two: the scale is exact)
    FB_TRY(pow2_rows(P, P, batch, M, true, true, 1.0f / (float)M, st, s));
    bs_crop_kernel<<<grid_for(batch * n), 256, 0, s>>>(P, batch, n, M, c, y, inverse ? 1 : 0, scale);
    FB_LAUNCH_CHECK("bs_crop_kernel");
    return FB_OK;
}

fb_status fft2d_bluestein(const void* x, void* y, int64_t n0, int64_t n1, bool inverse, void* ws, size_t ws_bytes,
                          const DeviceState* st, cudaStream_t s, bool unscaled) {
    if (ws_bytes < bluestein_ws_bytes(n0, n1) || !ws) {
        set_error("workspace of %zu bytes required for a non-power-of-two FFT", bluestein_ws_bytes(n0, n1));
        return FB_ERR_WORKSPACE;
    }
    const int64_t m0 = is_pow2(n0) ? 0 : bs_len(n0), m1 = is_pow2(n1) ? 0 : bs_len(n1);
    float2* P = (float2*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    const int64_t pe = (n0 * m1 > n1 * m0) ? n0 * m1 : n1 * m0;
    float2* T = P + pe;
    float2* c0 = T + n0 * n1;
    float2* H0 = c0 + n0;
    float2* c1 = H0 + m0;
    float2* H1 = c1 + n1;
    const float sc = (inverse && !unscaled) ? (float)(1.0 / ((double)n0 * (double)n1)) : 1.0f;
    // rows (length n1) x -> y, then y^T -> T, columns as rows of T, T^T -> y
    FB_TRY(dft_rows((const float2*)x, (float2*)y, n0, n1, inverse, n0 == 1 ? sc : 1.0f, P, c1, H1, st, s));
    if (n0 == 1) return FB_OK;
    dim3 tg((unsigned)((n1 + 31) / 32), (unsigned)((n0 + 31) / 32));
    bs_transpose_kernel<<<tg, 256, 0, s>>>((const float2*)y, n0, n1, T);
    FB_LAUNCH_CHECK("bs_transpose_kernel");
    FB_TRY(dft_rows(T, T, n1, n0, inverse, sc, P, c0, H0, st, s));
    dim3 tg2((unsigned)((n0 + 31) / 32), (unsigned)((n1 + 31) / 32));
    bs_transpose_kernel<<<tg2, 256, 0, s>>>(T, n1, n0, (float2*)y);
    FB_LAUNCH_CHECK("bs_transpose_kernel");
    return FB_OK;
}

}  // namespace fb
