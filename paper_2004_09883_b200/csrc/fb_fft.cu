// fb_fft.cu -- the Fourier-transform function block on sm_100a.
//
// A 2D DFT is computed as passes of batched 1D FFTs along "lines" (rows, then columns),
// which is the separable identity of the DFT definition (oracle/oracle.c evaluates the
// same definition naively).  One pass = one kernel launch:
//
//   * a CTA owns C whole lines, so every pass may run in place (the CTA reads all of its
//     lines before it writes any of them, and no other CTA touches them);
//   * lines are addressed through a LineMap (row lines, column lines, the per-peer blocks of
//     the slab all-to-all, the strided sub-lines of a four-step split), so packing and
//     unpacking are fused into the loads/stores of a pass instead of extra HBM passes;
//   * thread (c, t) of a line of length L = 16*T holds 16 elements k = t + m*T in registers.
//     The first Stockham stage runs straight from global memory, the last one stores
//     straight to global memory, and only the 1-2 middle exchanges go through shared memory
//     (padded k + k/16 layout, interleaved by line: conflict-free for every stage);
//   * radix-16 (and one radix-2/4/8 tail stage) butterflies are fully unrolled in registers;
//     twiddles come from one 16384-entry FP32 table built in FP64 (fb_api.cu);
//   * the inverse uses conj(FFT(conj x)) / N, so one kernel serves both signs and the exact
//     power-of-two scale 1/(n0 n1) is fused into the last pass.
//
// Stockham autosort (mixed radix): stage with radix R after Ns = product of earlier radices,
// butterfly j reads x[j + r L/R] (r < R), multiplies by W_{Ns R}^{(j mod Ns) r}, applies the
// radix-R DFT, writes y[(j / Ns) Ns R + (j mod Ns) + r Ns].  Output is in natural order.
#include "fb_common.cuh"

namespace fb {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

// x * exp(-2 pi i K / R) for 0 <= K < R/2 with compile-time K, R <= 16.
// Multiples of pi/4 are applied exactly (swaps / one scalar), the rest with RN constants.
template <int K, int R>
__device__ __forceinline__ float2 mul_wR(float2 x) {
    constexpr float kS = 0.707106781186547524400844362104849039f;  // cos(pi/4)
    constexpr float kC1 = 0.923879532511286756128183189396788933f;  // cos(pi/8)
    constexpr float kS1 = 0.382683432365089771728459984030398866f;  // sin(pi/8)
    if constexpr (K == 0) {
        return x;
    } else if constexpr (4 * K == R) {  // -i
        return make_float2(x.y, -x.x);
    } else if constexpr (8 * K == R) {  // exp(-i pi/4)
        return make_float2((x.x + x.y) * kS, (x.y - x.x) * kS);
    } else if constexpr (8 * K == 3 * R) {  // exp(-3 i pi/4)
        return make_float2((x.y - x.x) * kS, -(x.x + x.y) * kS);
    } else {
        static_assert(R == 16, "only R=16 needs pi/8 constants");
        // theta = 2 pi K / 16 = K pi / 8 with K odd in {1,3,5,7}
        constexpr float c = (K == 1) ? kC1 : (K == 3) ? kS1 : (K == 5) ? -kS1 : -kC1;
        constexpr float s = (K == 1) ? kS1 : (K == 3) ? kC1 : (K == 5) ? kC1 : kS1;
        // x * (c - i s)
        return make_float2(x.x * c + x.y * s, x.y * c - x.x * s);
    }
}

template <int R, int K>
struct Combine {
    __device__ __forceinline__ static void run(float2* v, const float2* e, const float2* o) {
        if constexpr (K < R / 2) {
            float2 tt = mul_wR<K, R>(o[K]);
            v[K] = cadd(e[K], tt);
            v[K + R / 2] = csub(e[K], tt);
            Combine<R, K + 1>::run(v, e, o);
        }
    }
};

// In-register DFT: v[k] <- sum_r v[r] exp(-2 pi i r k / R), natural order in and out.
template <int R>
__device__ __forceinline__ void dft(float2* v) {
    if constexpr (R == 1) {
        return;
    } else if constexpr (R == 2) {
        float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else {
        float2 e[R / 2], o[R / 2];
#pragma unroll
        for (int i = 0; i < R / 2; ++i) {
            e[i] = v[2 * i];
            o[i] = v[2 * i + 1];
        }
        dft<R / 2>(e);
        dft<R / 2>(o);
        Combine<R, 0>::run(v, e, o);
    }
}

template <int LOG2L>
struct LineGeom {
    static constexpr int L = 1 << LOG2L;
    static constexpr int E = L < 16 ? L : 16;       // elements per thread
    static constexpr int T = L / E;                 // threads per line
    static constexpr int S16 = LOG2L >= 4 ? LOG2L / 4 : 0;
    static constexpr int REM = LOG2L >= 4 ? LOG2L % 4 : LOG2L;
    // stage radices: S16 stages of 16, then one stage of 2^REM (if REM > 0)
    static constexpr int NSTAGES = S16 + (REM > 0 ? 1 : 0);
    static constexpr int PADL = L + (L >> 4);       // padded line length in smem
};

// Padded shared-memory position of element k of a line (one pad slot per 16 elements).
__host__ __device__ constexpr int padk(int k) { return k + (k >> 4); }

// ---- per-stage twiddle tables (built once per device by fb_init, see stage_tw_index()):
// for line length 2^l and stage s >= 1 (radix R, Ns = 16^s), entries [jm][r] = W_{Ns R}^{jm r},
// jm < Ns, r < R, stored contiguously so a thread fetches its R twiddles with R/2 16-byte
// loads at immediate offsets from one base pointer.
__host__ __device__ constexpr int stage_radix(int l, int s) {
    return (s < (l >= 4 ? l / 4 : 0)) ? 16 : (1 << (l >= 4 ? l % 4 : l));
}
__host__ __device__ constexpr int stage_count(int l) {
    return (l >= 4 ? l / 4 : 0) + (((l >= 4 ? l % 4 : l) > 0) ? 1 : 0);
}
__host__ __device__ constexpr int64_t stage_tw_size(int l, int s) {
    return (s == 0) ? 0 : (int64_t(1) << (4 * s)) * stage_radix(l, s);
}
__host__ __device__ constexpr int64_t stage_tw_offset(int l, int s) {
    int64_t off = 0;
    for (int ll = 0; ll < l; ++ll)
        for (int ss = 1; ss < stage_count(ll); ++ss) off += stage_tw_size(ll, ss);
    for (int ss = 1; ss < s; ++ss) off += stage_tw_size(l, ss);
    return off;
}
int64_t stage_tw_total() { return stage_tw_offset(kTwLog2 + 1, 0); }
// master-table index (W_16384^idx) of every stage-table entry, in table order
void stage_tw_index(int32_t* idx) {
    int64_t e = 0;
    for (int l = 0; l <= kTwLog2; ++l)
        for (int s = 1; s < stage_count(l); ++s) {
            const int R = stage_radix(l, s);
            const int64_t Ns = int64_t(1) << (4 * s);
            const int64_t step = kTwN / (Ns * R);
            for (int64_t jm = 0; jm < Ns; ++jm)
                for (int r = 0; r < R; ++r) idx[e++] = (int32_t)(jm * r * step);
        }
}

// Stage `S` (0-based): radix R, Ns = 16^S.  v[m] holds element t + m T of the stage input
// on entry (stage 0: loaded from global by the caller) and of the stage output on exit.
template <int LOG2L, int C, int S>
struct Stages {
    using G = LineGeom<LOG2L>;
    __device__ __forceinline__ static void run(float2* v, float2* sm, int t, int c,
                                               const float2* __restrict__ stw) {
        if constexpr (S < G::NSTAGES) {
            constexpr int R = stage_radix(LOG2L, S);
            constexpr int Ns = 1 << (4 * S);
            constexpr int Q = G::E / R;  // butterflies per thread in this stage
            constexpr int T = G::T;
            constexpr bool first = (S == 0);
            constexpr bool last = (S == G::NSTAGES - 1);
            if constexpr (!first) {
                // read x[t + m T]
                if constexpr (T % 16 == 0) {
                    const float2* rp = sm + padk(t) * C + c;
#pragma unroll
                    for (int m = 0; m < G::E; ++m) v[m] = rp[m * (T + T / 16) * C];
                } else {
#pragma unroll
                    for (int m = 0; m < G::E; ++m) v[m] = sm[padk(t + m * T) * C + c];
                }
            }
            // butterflies j = t + q T (q < Q), inputs v[q + r Q] = x[j + r L/R]
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                float2 b[R];
#pragma unroll
                for (int r = 0; r < R; ++r) b[r] = v[q + r * Q];
                if constexpr (!first) {
                    const int jm = (t + q * T) & (Ns - 1);
                    const float4* tw4 = reinterpret_cast<const float4*>(
                        stw + stage_tw_offset(LOG2L, S) + (int64_t)jm * R);
#pragma unroll
                    for (int r2 = 0; r2 < R / 2; ++r2) {
                        const float4 w = __ldg(tw4 + r2);
                        if (r2 > 0) b[2 * r2] = cmul(b[2 * r2], make_float2(w.x, w.y));
                        b[2 * r2 + 1] = cmul(b[2 * r2 + 1], make_float2(w.z, w.w));
                    }
                }
                dft<R>(b);
#pragma unroll
                for (int r = 0; r < R; ++r) v[q + r * Q] = b[r];
            }
            if constexpr (!last) {
                static_assert(Q == 1 && R == 16, "only the last stage may be a tail stage");
                if constexpr (!first) __syncthreads();  // everyone has read the buffer
                // write y[(t / Ns) Ns R + (t mod Ns) + r Ns]
                if constexpr (Ns == 1) {
                    float2* wp = sm + (17 * t) * C + c;
#pragma unroll
                    for (int r = 0; r < R; ++r) wp[r * C] = v[r];
                } else {
                    const int kb = (t / Ns) * Ns * R + (t & (Ns - 1));
                    float2* wp = sm + padk(kb) * C + c;
#pragma unroll
                    for (int r = 0; r < R; ++r) wp[r * (Ns + Ns / 16) * C] = v[r];
                }
                __syncthreads();
                Stages<LOG2L, C, S + 1>::run(v, sm, t, c, stw);
            }
        }
    }
};

// PLAIN: both line maps unblocked (element k at k*es) -> incremental 64-bit addressing.
template <int LOG2L, int C, bool PLAIN>
__global__ void __launch_bounds__(C * LineGeom<LOG2L>::T,
                                  (C * LineGeom<LOG2L>::T >= 1024) ? 1 : 1024 / (C * LineGeom<LOG2L>::T))
    fft_pass_kernel(const FftPass p, const float2* __restrict__ tw, const float2* __restrict__ stw) {
    using G = LineGeom<LOG2L>;
    extern __shared__ float2 sm[];
    const int tid = threadIdx.x;
    const int c = tid % C;
    const int t = tid / C;
    const int64_t g = (int64_t)blockIdx.x * C + c;
    const bool valid = g < p.nlines;
    const int64_t gh = (p.g_shift >= 62) ? 0 : (g >> p.g_shift);
    const int64_t gl = (p.g_shift >= 62) ? g : (g & ((int64_t(1) << p.g_shift) - 1));

    const float2* src = p.in + gh * p.lin.hi + gl * p.lin.lo;
    float2* dst = p.out + gh * p.lout.hi + gl * p.lout.lo;

    float2 v[G::E];
    if constexpr (PLAIN) {
        const float2* sp = src + (int64_t)t * p.lin.es;
        const int64_t sstride = (int64_t)G::T * p.lin.es;
#pragma unroll
        for (int m = 0; m < G::E; ++m) v[m] = valid ? sp[m * sstride] : make_float2(0.f, 0.f);
    } else {
        const int in_kmask = (1 << p.lin.kb_shift) - 1;
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            const int k = t + m * G::T;
            const int64_t off = (int64_t)(k & in_kmask) * p.lin.es + (int64_t)(k >> p.lin.kb_shift) * p.lin.bs;
            v[m] = valid ? src[off] : make_float2(0.f, 0.f);
        }
    }
    if (p.conj_in) {
#pragma unroll
        for (int m = 0; m < G::E; ++m) v[m].y = -v[m].y;
    }

    Stages<LOG2L, C, 0>::run(v, sm, t, c, stw);

    if (!valid) return;
    if (p.tw4_log2N > 0) {
        // four-step twiddle W_N^{gh k}, N = 2^tw4 (the master table has resolution 2^14)
        const int tw4 = p.tw4_log2N;
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            const int k = t + m * G::T;
            const int64_t e = (gh * (int64_t)k) & ((int64_t(1) << tw4) - 1);
            v[m] = cmul(v[m], __ldg(tw + (e << (kTwLog2 - tw4))));
        }
    }
    if (p.conj_out) {
#pragma unroll
        for (int m = 0; m < G::E; ++m) v[m].y = -v[m].y;
    }
    if (p.scale != 1.0f) {
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            v[m].x *= p.scale;
            v[m].y *= p.scale;
        }
    }
    if constexpr (PLAIN) {
        float2* dp = dst + (int64_t)t * p.lout.es;
        const int64_t dstride = (int64_t)G::T * p.lout.es;
#pragma unroll
        for (int m = 0; m < G::E; ++m) dp[m * dstride] = v[m];
    } else {
        const int out_kmask = (1 << p.lout.kb_shift) - 1;
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            const int k = t + m * G::T;
            const int64_t off = (int64_t)(k & out_kmask) * p.lout.es + (int64_t)(k >> p.lout.kb_shift) * p.lout.bs;
            dst[off] = v[m];
        }
    }
}

template <int LOG2L, int C, bool PLAIN>
static fb_status launch_one(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    using G = LineGeom<LOG2L>;
    constexpr int threads = C * G::T;
    static_assert(threads <= 1024, "CTA too large");
    const size_t smem = (G::NSTAGES > 1) ? (size_t)C * G::PADL * sizeof(float2) : 0;
    static int attr_done_mask = 0;  // per-device bit (devices 0..31)
    int dev = 0;
    cudaGetDevice(&dev);
    if (smem > 48 * 1024 && !(attr_done_mask & (1 << (dev & 31)))) {
        FB_CUDA_TRY(cudaFuncSetAttribute(fft_pass_kernel<LOG2L, C, PLAIN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_done_mask |= 1 << (dev & 31);
    }
    const int64_t blocks = (p.nlines + C - 1) / C;
    if (blocks > 0x7fffffff) {
        set_error("FFT pass grid too large (%lld CTAs)", (long long)blocks);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    fft_pass_kernel<LOG2L, C, PLAIN><<<(unsigned)blocks, threads, smem, s>>>(p, st->twiddles, st->stage_tw);
    FB_LAUNCH_CHECK("fft_pass_kernel");
    return FB_OK;
}

template <int LOG2L, int C>
static fb_status launch_LC(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    const bool plain = p.lin.kb_shift >= LOG2L && p.lout.kb_shift >= LOG2L;
    return plain ? launch_one<LOG2L, C, true>(p, st, s) : launch_one<LOG2L, C, false>(p, st, s);
}

template <int LOG2L>
static fb_status launch_L(const FftPass& p, int C, const DeviceState* st, cudaStream_t s) {
    constexpr int T = LineGeom<LOG2L>::T;
    switch (C) {
        case 8:
            if constexpr (8 * T <= 1024) return launch_LC<LOG2L, 8>(p, st, s);
            break;
        case 4:
            if constexpr (4 * T <= 1024) return launch_LC<LOG2L, 4>(p, st, s);
            break;
        case 2:
            if constexpr (2 * T <= 1024) return launch_LC<LOG2L, 2>(p, st, s);
            break;
        case 1:
            return launch_LC<LOG2L, 1>(p, st, s);
    }
    set_error("internal: no FFT instantiation for L=2^%d C=%d", LOG2L, C);
    return FB_ERR_UNSUPPORTED_SIZE;
}

// Lines per CTA.  Column-like passes (adjacent lines adjacent in memory) want C*8 >= 32 B
// row segments -> C = 4 (or 8 for short lines); row passes want small CTAs (many per SM so
// the load / compute / store phases of different CTAs overlap), at least one full warp.
static int pick_C(int log2L, bool col_like) {
    const int T = (1 << log2L) < 16 ? 1 : (1 << log2L) / 16;
    int C;
    if (col_like)
        C = (T <= 64) ? 8 : (T <= 256 ? 4 : 1024 / T);
    else
        C = (T >= 32) ? 1 : 32 / T;
    if (C > 8) C = 8;
    if (C < 1) C = 1;
    return C;
}

fb_status launch_fft_pass(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    if (p.nlines <= 0) return FB_OK;
    const int C = pick_C(p.log2L, p.col_like != 0);
    switch (p.log2L) {
        case 0: return launch_L<0>(p, C, st, s);
        case 1: return launch_L<1>(p, C, st, s);
        case 2: return launch_L<2>(p, C, st, s);
        case 3: return launch_L<3>(p, C, st, s);
        case 4: return launch_L<4>(p, C, st, s);
        case 5: return launch_L<5>(p, C, st, s);
        case 6: return launch_L<6>(p, C, st, s);
        case 7: return launch_L<7>(p, C, st, s);
        case 8: return launch_L<8>(p, C, st, s);
        case 9: return launch_L<9>(p, C, st, s);
        case 10: return launch_L<10>(p, C, st, s);
        case 11: return launch_L<11>(p, C, st, s);
        case 12: return launch_L<12>(p, C, st, s);
        case 13: return launch_L<13>(p, C, st, s);
        case 14: return launch_L<14>(p, C, st, s);
    }
    set_error("FFT line length 2^%d unsupported", p.log2L);
    return FB_ERR_UNSUPPORTED_SIZE;
}

static LineMap plain_map(int64_t hi, int64_t lo, int64_t es) {
    LineMap m;
    m.hi = hi;
    m.lo = lo;
    m.kb_shift = 30;  // no blocking
    m.es = es;
    m.bs = 0;
    return m;
}

static constexpr int kMaxOnChipCol = 12;  // column lines up to 4096 in one pass

fb_status fft_columns(const float2* in, float2* out, int64_t n0, int64_t ncols, int64_t ld_in,
                      int64_t ld_out, bool conj_in, bool conj_out, float scale, float2* tmp,
                      const DeviceState* st, cudaStream_t s) {
    const int l0 = ilog2(n0);
    const int lc = ilog2(ncols);
    if (l0 <= kMaxOnChipCol) {
        FftPass p{};
        p.in = in;
        p.out = out;
        p.log2L = l0;
        p.nlines = ncols;
        p.g_shift = 62;
        p.lin = plain_map(0, 1, ld_in);
        p.lout = plain_map(0, 1, ld_out);
        p.conj_in = conj_in;
        p.conj_out = conj_out;
        p.scale = scale;
        p.tw4_log2N = 0;
        p.col_like = 1;
        return launch_fft_pass(p, st, s);
    }
    // Four-step split of the column length n0 = a * b (b = 128 contiguous sub-line rows):
    //   step 1: for each n2 < b: length-a FFTs over rows b*n1 + n2, times W_n0^{n2 k1}
    //           (tmp rows b*k1 + n2)
    //   step 3: for each k1 < a: length-b FFTs over rows b*k1 + n2 -> out rows k1 + a*k2
    if (!tmp) {
        set_error("internal: four-step column FFT needs a workspace");
        return FB_ERR_WORKSPACE;
    }
    const int lb = 7;
    const int la = l0 - lb;
    const int64_t a = int64_t(1) << la, b = int64_t(1) << lb;
    FftPass p1{};
    p1.in = in;
    p1.out = tmp;
    p1.log2L = la;
    p1.nlines = b * ncols;
    p1.g_shift = lc;  // g = n2 * ncols + c
    p1.lin = plain_map(ld_in, 1, b * ld_in);
    p1.lout = plain_map(ncols, 1, b * ncols);
    p1.conj_in = conj_in;
    p1.conj_out = 0;
    p1.scale = 1.f;
    p1.tw4_log2N = l0;
    p1.col_like = 1;
    FB_TRY(launch_fft_pass(p1, st, s));
    FftPass p3{};
    p3.in = tmp;
    p3.out = out;
    p3.log2L = lb;
    p3.nlines = a * ncols;
    p3.g_shift = lc;  // g = k1 * ncols + c
    p3.lin = plain_map(b * ncols, 1, ncols);
    p3.lout = plain_map(ld_out, 1, a * ld_out);
    p3.conj_in = 0;
    p3.conj_out = conj_out;
    p3.scale = scale;
    p3.tw4_log2N = 0;
    p3.col_like = 1;
    return launch_fft_pass(p3, st, s);
}

size_t fft2d_ws_bytes(int64_t n0, int64_t n1) {
    if (ilog2(n0) <= kMaxOnChipCol) return 0;
    return (size_t)n0 * (size_t)n1 * sizeof(float2);
}

fb_status fft2d_device(const void* x, void* y, int64_t n0, int64_t n1, bool inverse, void* ws,
                       size_t ws_bytes, const DeviceState* st, cudaStream_t s) {
    const float scale = inverse ? 1.0f / (float)((double)n0 * (double)n1) : 1.0f;
    const bool four_step = ilog2(n0) > kMaxOnChipCol;
    float2* rowout = four_step ? (float2*)ws : (float2*)y;
    if (four_step && ws_bytes < fft2d_ws_bytes(n0, n1)) {
        set_error("workspace too small");
        return FB_ERR_WORKSPACE;
    }
    // pass 1: row FFTs (length n1) x -> rowout
    FftPass p{};
    p.in = (const float2*)x;
    p.out = rowout;
    p.log2L = ilog2(n1);
    p.nlines = n0;
    p.g_shift = 0;
    p.lin = plain_map(n1, 0, 1);
    p.lout = plain_map(n1, 0, 1);
    p.conj_in = inverse;
    p.conj_out = 0;
    p.scale = 1.f;
    p.tw4_log2N = 0;
    p.col_like = 0;
    FB_TRY(launch_fft_pass(p, st, s));
    // pass 2: column FFTs (length n0) rowout -> y (in place when on-chip)
    return fft_columns(rowout, (float2*)y, n0, n1, n1, n1, false, inverse, scale,
                       four_step ? (float2*)ws : nullptr, st, s);
}

}  // namespace fb
