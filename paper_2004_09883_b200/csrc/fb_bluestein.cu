// fb_bluestein.cu -- the Fourier-transform block for sizes that are NOT
// powers of two (vibration records have arbitrary lengths).
//
// Lines whose length n <= 8192 factors into 2, 3, 5 and 7 run as a mixed-radix Stockham
// transform in shared memory (one CTA per line, radix-8/4/2/3/5/7 stages, mr_lines_kernel below);
// every other length uses Bluestein's identity:
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

#include "fb_fft_kern.cuh"

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

// ------------------------------------------------------------------ mixed radix (2, 3, 5, 7)
// Stockham autosort, one CTA per line held in shared memory (two n-element buffers).  Stage s
// with radix R and Ns = product of the earlier radices: for every j < n / R, with k = j mod Ns,
//   a[r] = src[j + r n / R] * W_{Ns R}^{r k}   (r < R),   b = DFT_R(a),
//   dst[(j / Ns) Ns R + k + q Ns] = b[q]       (q < R);
// after the last stage the line is in natural order.  W_{Ns R}^{r k} = W_n^{r k n / (Ns R)} comes
// from a per-call FP64-computed table W_n^j (j < n) rounded once to FP32.
struct MrPlan {
    int nst;
    int r[24];
};

static bool smooth7(int64_t n) {
    for (int p : {2, 3, 5, 7})
        while (n % p == 0) n /= p;
    return n == 1;
}

static MrPlan mr_plan(int64_t n) {
    MrPlan pl{};
    auto push = [&](int r) { pl.r[pl.nst++] = r; n /= r; };
    while (n % 8 == 0) push(8);
    while (n % 4 == 0) push(4);
    while (n % 2 == 0) push(2);
    while (n % 7 == 0) push(7);
    while (n % 5 == 0) push(5);
    while (n % 3 == 0) push(3);
    return pl;
}

__global__ void mr_twiddle_kernel(float2* __restrict__ W, int64_t n) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        double sn, cs;
        sincospi(2.0 * (double)j / (double)n, &sn, &cs);
        W[j] = make_float2((float)cs, (float)(-sn));  // exp(-2 pi i j / n)
    }
}

// cos / sin of 2 pi j / R for the odd radices, RN FP32 constants
template <int R>
__device__ __forceinline__ constexpr float cosR(int j);
template <int R>
__device__ __forceinline__ constexpr float sinR(int j);
template <>
__device__ __forceinline__ constexpr float cosR<3>(int j) { return j == 0 ? 1.f : -0.5f; }
template <>
__device__ __forceinline__ constexpr float sinR<3>(int j) {
    return j == 0 ? 0.f : j == 1 ? 0.866025403784438646763723170752936183f : -0.866025403784438646763723170752936183f;
}
template <>
__device__ __forceinline__ constexpr float cosR<5>(int j) {
    return j == 0 ? 1.f : (j == 1 || j == 4) ? 0.309016994374947424102293417182819059f
                                             : -0.809016994374947424102293417182819059f;
}
template <>
__device__ __forceinline__ constexpr float sinR<5>(int j) {
    return j == 0 ? 0.f : j == 1 ? 0.951056516295153572116439333379382143f
         : j == 2 ? 0.587785252292473129168705954639072769f : j == 3 ? -0.587785252292473129168705954639072769f
                  : -0.951056516295153572116439333379382143f;
}
template <>
__device__ __forceinline__ constexpr float cosR<7>(int j) {
    return j == 0 ? 1.f : (j == 1 || j == 6) ? 0.623489801858733530525004884004239810f
         : (j == 2 || j == 5) ? -0.222520933956314404288902564496794759f : -0.900968867902419126236102319507445051f;
}
template <>
__device__ __forceinline__ constexpr float sinR<7>(int j) {
    return j == 0 ? 0.f : j == 1 ? 0.781831482468029808708444526674057750f
         : j == 2 ? 0.974927912181823607018131682993931217f : j == 3 ? 0.433883739117558120475768332848358754f
         : j == 4 ? -0.433883739117558120475768332848358754f : j == 5 ? -0.974927912181823607018131682993931217f
                  : -0.781831482468029808708444526674057750f;
}

// b[q] = sum_r a[r] exp(-2 pi i r q / R): power-of-two radices through the radix-2 DIT template,
// 3 / 5 / 7 directly (pairs r, R - r combined: a[r] + a[R-r] and a[r] - a[R-r])
template <int R>
__device__ __forceinline__ void dft_any(float2* a) {
    if constexpr ((R & (R - 1)) == 0) {
        dft<R>(a);
    } else {
        float2 sp[R / 2 + 1], sm[R / 2 + 1];
#pragma unroll
        for (int r = 1; r <= R / 2; ++r) {
            sp[r] = make_float2(a[r].x + a[R - r].x, a[r].y + a[R - r].y);
            sm[r] = make_float2(a[r].x - a[R - r].x, a[r].y - a[R - r].y);
        }
        float2 b[R];
        b[0] = a[0];
#pragma unroll
        for (int r = 1; r <= R / 2; ++r) b[0] = make_float2(b[0].x + sp[r].x, b[0].y + sp[r].y);
#pragma unroll
        for (int q = 1; q <= R / 2; ++q) {
            // X[q] = a0 + sum_r (sp[r] cos - i sm[r] sin),  X[R-q] = a0 + sum_r (sp[r] cos + i sm[r] sin)
            float re = a[0].x, im = a[0].y, tre = 0.f, tim = 0.f;
#pragma unroll
            for (int r = 1; r <= R / 2; ++r) {
                const float c = cosR<R>((r * q) % R), sn = sinR<R>((r * q) % R);
                re = fmaf(sp[r].x, c, re);
                im = fmaf(sp[r].y, c, im);
                tre = fmaf(sm[r].y, sn, tre);
                tim = fmaf(-sm[r].x, sn, tim);
            }
            b[q] = make_float2(re + tre, im + tim);
            b[R - q] = make_float2(re - tre, im - tim);
        }
#pragma unroll
        for (int q = 0; q < R; ++q) a[q] = b[q];
    }
}

// one stage over C interleaved lines: element i of line c at i * C + c
template <int R, bool COLS>
__device__ __forceinline__ void mr_stage(const float2* __restrict__ src, float2* __restrict__ dst, int n, int Ns,
                                         int Cr, const float2* __restrict__ W) {
    const int C = COLS ? Cr : 1;  // rows: one contiguous line, no index division
    const int m = n / R, tstep = n / (Ns * R);
    for (int u = threadIdx.x; u < m * C; u += blockDim.x) {
        const int j = COLS ? u / C : u, c = COLS ? u - j * C : 0;
        const int k = j % Ns;
        float2 a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) a[r] = src[(j + r * m) * C + c];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) a[r] = cmul(a[r], __ldg(W + r * k * tstep));
        }
        dft_any<R>(a);
        const int o = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int q = 0; q < R; ++q) dst[(o + q * Ns) * C + c] = a[q];
    }
}

// C lines per CTA: rows (C = 1, line b = row b, contiguous) or columns (line c of CTA b = column
// b C + c, elements ld apart; the C columns are loaded and stored as C-wide row segments).
// Every element of the CTA's lines is in shared memory before the first store: in place is safe.
template <bool COLS>
__global__ void __launch_bounds__(256) mr_lines_kernel(const float2* __restrict__ x, float2* __restrict__ y, int n,
                                                       int Cr, int64_t ld, int64_t ncols, MrPlan pl,
                                                       const float2* __restrict__ W, int conj_in, int conj_out,
                                                       float scale) {
    const int C = COLS ? Cr : 1;
    constexpr bool cols = COLS;
    extern __shared__ float2 mr_sm[];
    float2* A = mr_sm;
    float2* B = mr_sm + (int64_t)n * C;
    const int64_t c0 = (int64_t)blockIdx.x * C;  // first line of this CTA (rows: C = 1, ld = n)
    const float2* xs = cols ? x + c0 : x + c0 * n;
    float2* ys = cols ? y + c0 : y + c0 * n;
    const int64_t step = cols ? ld : 1;  // element stride along a line
    const int cw = (int)((ncols - c0) < C ? (ncols - c0) : C);
    for (int u = threadIdx.x; u < n * C; u += blockDim.x) {
        const int i = COLS ? u / C : u, c = COLS ? u - i * C : 0;
        float2 v = make_float2(0.f, 0.f);
        if (c < cw) v = xs[(int64_t)i * step + c];
        if (conj_in) v.y = -v.y;
        A[u] = v;
    }
    __syncthreads();
    int Ns = 1;
    for (int st = 0; st < pl.nst; ++st) {
        const int R = pl.r[st];
        switch (R) {
            case 8: mr_stage<8, COLS>(A, B, n, Ns, C, W); break;
            case 4: mr_stage<4, COLS>(A, B, n, Ns, C, W); break;
            case 2: mr_stage<2, COLS>(A, B, n, Ns, C, W); break;
            case 3: mr_stage<3, COLS>(A, B, n, Ns, C, W); break;
            case 5: mr_stage<5, COLS>(A, B, n, Ns, C, W); break;
            default: mr_stage<7, COLS>(A, B, n, Ns, C, W); break;
        }
        __syncthreads();
        float2* t = A;
        A = B;
        B = t;
        Ns *= R;
    }
    for (int u = threadIdx.x; u < n * C; u += blockDim.x) {
        const int i = COLS ? u / C : u, c = COLS ? u - i * C : 0;
        if (c >= cw) continue;
        float2 v = A[u];
        if (conj_out) v.y = -v.y;
        ys[(int64_t)i * step + c] = make_float2(v.x * scale, v.y * scale);
    }
}

static bool use_mixed_radix(int64_t n) { return knobs().fft_mixed != 0 && n <= kBluesteinMax && smooth7(n); }

// lines of length n: `batch` contiguous rows (cols == false), or the ncols columns of an n x ncols
// row-major array (cols == true, row pitch ncols); W: n-entry scratch for the W_n table
static fb_status mixed_lines(const float2* x, float2* y, int64_t batch, int64_t n, bool cols, int64_t ncols,
                             bool inverse, float scale, float2* W, cudaStream_t s) {
    constexpr size_t kMaxSmem = (size_t)2 * kBluesteinMax * sizeof(float2);  // 128 KiB
    static DevOnce once;
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(mr_lines_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMaxSmem));
        FB_CUDA_TRY(cudaFuncSetAttribute(mr_lines_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kMaxSmem));
        once.set(dev);
    }
    // columns per CTA: up to 8 (64-byte row segments), as many as fit 128 KiB of line buffers
    int C = 1;
    if (cols)
        while (C < 8 && (size_t)2 * n * (2 * C) * sizeof(float2) <= kMaxSmem) C *= 2;
    const int64_t ctas = cols ? (ncols + C - 1) / C : batch;
    if (ctas > INT32_MAX) {
        set_error("too many lines for the mixed-radix kernel");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    mr_twiddle_kernel<<<grid_for(n), 256, 0, s>>>(W, n);
    FB_LAUNCH_CHECK("mr_twiddle_kernel");
    const size_t smem = (size_t)2 * n * C * sizeof(float2);
    if (cols)
        mr_lines_kernel<true><<<(unsigned)ctas, 256, smem, s>>>(x, y, (int)n, C, ncols, ncols, mr_plan(n), W,
                                                               inverse ? 1 : 0, inverse ? 1 : 0, scale);
    else
        // rows: 128 threads for n <= 1024 (a radix-8 stage has <= 128 butterflies; 256-thread CTAs
        // were register-limited to 4 per SM, 1.69 waves at 1000^2), else 256
        mr_lines_kernel<false><<<(unsigned)ctas, n <= knobs().fft_mr_small ? 128 : 256, smem, s>>>(
            x, y, (int)n, 1, n, batch, mr_plan(n), W, inverse ? 1 : 0, inverse ? 1 : 0, scale);
    FB_LAUNCH_CHECK("mr_lines_kernel");
    return FB_OK;
}

// DFT (sign -1, or +1 with inverse) of `batch` contiguous rows of length n: x -> y, times `scale`
static fb_status dft_rows(const float2* x, float2* y, int64_t batch, int64_t n, bool inverse, float scale,
                          float2* P, float2* c, float2* H, const DeviceState* st, cudaStream_t s) {
    if (is_pow2(n)) return pow2_rows(x, y, batch, n, inverse, inverse, scale, st, s);
    if (use_mixed_radix(n)) return mixed_lines(x, y, batch, n, false, 1, inverse, scale, c, s);  // c: W_n table
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
    // FB_FFT_MIXED=2: 7-smooth columns in place, C <= 8 at a time (no transposes) -- measured
    // slower than the transposed route (1000^2 53.6 -> 59.5 us, 2000 x 3000 176 -> 279 us, 2187^2
    // 150 -> 189 us: 64-byte segments and 128 KiB of line buffers per CTA), so off by default
    if (knobs().fft_mixed == 2 && use_mixed_radix(n0))
        return mixed_lines((const float2*)y, (float2*)y, 0, n0, true, n1, inverse, sc, c0, s);
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
