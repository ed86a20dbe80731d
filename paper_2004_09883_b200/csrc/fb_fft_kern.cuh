// fb_fft_kern.cuh -- kernels of the Fourier-transform function block on sm_100a.
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
#pragma once
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include "fb_common.cuh"
#include "fb_ptx.cuh"

namespace fb {

// Complex arithmetic on interleaved (re, im) pairs with the sm_100 packed-FP32 instructions
// (FADD2 / FMUL2 / FFMA2; operand broadcast, lane swap and per-lane negation are free
// operand modifiers), so a complex add is one instruction and a complex multiply two.
// Every lane is IEEE RN, identical to the scalar forms.
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __ffma2_rn(b, bc2(-1.f), a); }
// a * w  = a.x (w.x, w.y) + a.y (-w.y, w.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
    const float2 t = __fmul2_rn(bc2(a.x), w);
    return __ffma2_rn(make_float2(-w.y, w.x), bc2(a.y), t);
}
// a + (-i) b = (a.x + b.y, a.y - b.x)   and   a - (-i) b = (a.x - b.y, a.y + b.x)
__device__ __forceinline__ float2 cadd_mi(float2 a, float2 b) {
    return __ffma2_rn(make_float2(b.y, b.x), make_float2(1.f, -1.f), a);
}
__device__ __forceinline__ float2 csub_mi(float2 a, float2 b) {
    return __ffma2_rn(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a);
}
// x * (c - i s) = c x + s (x.y, -x.x)
__device__ __forceinline__ float2 cmul_cs(float2 x, float c, float s) {
    const float2 t = __fmul2_rn(x, bc2(c));
    return __ffma2_rn(make_float2(x.y, x.x), make_float2(s, -s), t);
}

// cos(j pi / 16) and sin(j pi / 16), j = 0..16, as RN FP32 constants (the radix-2..32 internal
// twiddles; the values for R <= 16 are the same constants as before the table existed)
__device__ __forceinline__ constexpr float cos16(int j) {
    constexpr float c1 = 0.980785280403230449126182236134239037f, c2 = 0.923879532511286756128183189396788933f,
                    c3 = 0.831469612302545237078788377617905756f, c4 = 0.707106781186547524400844362104849039f,
                    c5 = 0.555570233019602224742830813948532874f, c6 = 0.382683432365089771728459984030398866f,
                    c7 = 0.195090322016128267848284868477022240f;
    return j == 0 ? 1.f : j == 1 ? c1 : j == 2 ? c2 : j == 3 ? c3 : j == 4 ? c4 : j == 5 ? c5 : j == 6 ? c6
         : j == 7 ? c7 : j == 8 ? 0.f : j == 9 ? -c7 : j == 10 ? -c6 : j == 11 ? -c5 : j == 12 ? -c4
         : j == 13 ? -c3 : j == 14 ? -c2 : j == 15 ? -c1 : -1.f;
}
__device__ __forceinline__ constexpr float sin16(int j) { return j <= 8 ? cos16(8 - j) : cos16(j - 8); }

// Radix-2 combine of the DIT recursion with the compile-time twiddle W_R^K = exp(-2 pi i K/R):
// v[K] = e + W o, v[K + R/2] = e - W o.  K = 0 and K = R/4 (-i) need no multiply.
template <int K, int R>
__device__ __forceinline__ void butterfly(float2* v, float2 e, float2 o) {
    static_assert(R <= 32, "radix > 32 not supported");
    if constexpr (K == 0) {
        v[K] = cadd(e, o);
        v[K + R / 2] = csub(e, o);
    } else if constexpr (4 * K == R) {
        v[K] = cadd_mi(e, o);
        v[K + R / 2] = csub_mi(e, o);
    } else {
        // theta = 2 pi K / R = j pi / 16 in (0, pi), K != R/4
        constexpr int j = 32 * K / R;
        constexpr float c = cos16(j), s = sin16(j);
        const float2 t = cmul_cs(o, c, s);
        v[K] = cadd(e, t);
        v[K + R / 2] = csub(e, t);
    }
}

template <int R, int K>
struct Combine {
    __device__ __forceinline__ static void run(float2* v, const float2* e, const float2* o) {
        if constexpr (K < R / 2) {
            butterfly<K, R>(v, e[K], o[K]);
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
        const float2 a = v[0], b = v[1];
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
// for line length 2^l and stage s >= 1 (radix R, Ns = 16^s), entries [r][jm] = W_{Ns R}^{jm r},
// r < R, jm < Ns: a warp's lanes (consecutive jm) read consecutive entries for each r, and a
// thread reaches its R twiddles at immediate offsets r*Ns from one base pointer.
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

// Twiddles of stage S for this thread's butterflies j = t + q T: W_{Ns R}^{(j mod Ns) r}, r < R.
// FB_FFT_TWREC = 1 (default): only the log2(R) "bases" W^{jm 2^i} are loaded per butterfly
// (tw[q][i]); tw_expand forms the other R - 1 - log2(R) powers by products of at most
// popcount(r) - 1 complex multiplies (<= 3 for R = 16), so each radix-16 stage issues 4
// table loads per butterfly instead of 15 (the loads were the largest stall of both 2048^2
// passes: long scoreboard 22 % / 28 % of warp samples, profiles/r1_fft2048_full.txt).
// FB_FFT_TWREC = 0: all R - 1 twiddles are loaded (tw[q][r-1]), each RN of the FP64 value.
#ifndef FB_FFT_TWREC
#define FB_FFT_TWREC 1
#endif
__host__ __device__ constexpr int ilog2c(int r) { return r <= 1 ? 0 : 1 + ilog2c(r / 2); }  // floor(log2 r)
template <int R>
struct TwCount {
    static constexpr int value = FB_FFT_TWREC ? ilog2c(R) : R - 1;
};
// full[r - 1] = W^{jm r} for r = 1 .. R-1 from the loaded values `b` (bases or, without
// FB_FFT_TWREC, all of them).  r = hb + rest (hb = highest power of two <= r):
// W^{jm r} = W^{jm rest} * W^{jm hb}.
template <int R, int r = 1>
__device__ __forceinline__ void pow_expand(float2* full, const float2* b) {  // always from bases
    if constexpr (r < R) {
        constexpr int i = ilog2c(r), hb = 1 << i;
        if constexpr (r == hb)
            full[r - 1] = b[i];
        else
            full[r - 1] = cmul(full[r - hb - 1], b[i]);
        pow_expand<R, r + 1>(full, b);
    }
}
template <int R>
__device__ __forceinline__ void tw_expand(float2* full, const float2* b) {
    if constexpr (FB_FFT_TWREC) {
        pow_expand<R>(full, b);
    } else {
#pragma unroll
        for (int r = 1; r < R; ++r) full[r - 1] = b[r - 1];
    }
}
// load this butterfly's stored twiddles from the [r][jm] table row base twp (= table + jm)
template <int R, int Ns>
__device__ __forceinline__ void tw_load(float2* b, const float2* __restrict__ twp) {
#pragma unroll
    for (int i = 0; i < TwCount<R>::value; ++i) b[i] = __ldg(twp + (FB_FFT_TWREC ? (1 << i) : (i + 1)) * Ns);
}

// Four-step twiddles W_N^{gh k} for this thread's elements k = t + m T (m < E), N = 2^log2N:
// one scattered load a = W^{gh t} and log2(E) warp-uniform bases W^{gh T 2^i}; the powers
// b^m = W^{gh T m} come from tw_expand, then v[m] *= a b^m (FB_FFT_TW4REC = 1, default).  With
// FB_FFT_TW4REC = 0 every element loads its own twiddle (E scattered loads per thread; the
// 16384^2 first four-step pass ran at 70 % of the copy bandwidth that way).
#ifndef FB_FFT_TW4REC
#define FB_FFT_TW4REC 1
#endif
template <int E, int T>
__device__ __forceinline__ void apply_tw4(float2* v, int64_t gh, int t, int log2N, const float2* __restrict__ tw) {
    const int64_t msk = (int64_t(1) << log2N) - 1;
    const int sh = kTwLog2 - log2N;
    if constexpr (FB_FFT_TW4REC && E >= 2) {
        constexpr int LE = ilog2c(E);
        const float2 a = __ldg(tw + (((gh * (int64_t)t) & msk) << sh));
        float2 b[LE], full[E - 1];
#pragma unroll
        for (int i = 0; i < LE; ++i) b[i] = __ldg(tw + (((gh * (int64_t)(T << i)) & msk) << sh));
        pow_expand<E>(full, b);
        v[0] = cmul(v[0], a);
#pragma unroll
        for (int m = 1; m < E; ++m) v[m] = cmul(v[m], cmul(a, full[m - 1]));
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int64_t e = (gh * (int64_t)(t + m * T)) & msk;
            v[m] = cmul(v[m], __ldg(tw + (e << sh)));
        }
    }
}

template <int LOG2L, int S>
struct StageTw {
    static constexpr int R = stage_radix(LOG2L, S);
    static constexpr int Q = LineGeom<LOG2L>::E / R;
    static constexpr int NB = TwCount<R>::value;  // stored twiddles per butterfly
    static constexpr int NT = (S == 0) ? 1 : Q * NB;
    __device__ __forceinline__ static void load(float2* tw, int t, const float2* __restrict__ stw) {
        if constexpr (S > 0) {
            constexpr int Ns = 1 << (4 * S);
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const int jm = (t + q * LineGeom<LOG2L>::T) & (Ns - 1);
                tw_load<R, Ns>(tw + q * NB, stw + stage_tw_offset(LOG2L, S) + jm);
            }
        }
    }
};

// Barrier of the threads that share one exchange buffer: the whole CTA (id 0, __syncthreads)
// or one sub-CTA of a multi-group persistent CTA (named barrier `id` over `n` threads).
struct Sync {
    int id, n;
    __device__ __forceinline__ void operator()() const {
        if (id == 0)
            __syncthreads();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    }
};

// Stage `S` (0-based): radix R, Ns = 16^S.  v[m] holds element t + m T of the stage input
// on entry (stage 0: loaded by the caller) and of the stage output on exit.  `tw` holds this
// stage's twiddles, prefetched by the previous stage just before its barrier (the element
// registers are dead there, so the loads overlap the barrier and the exchange reads).
// STOP < NSTAGES: return at the start of stage STOP (its input exchange is written and past the
// barrier; the caller runs that stage itself, see pair_last_stage).
template <int LOG2L, int C, int S, int STOP = 64>
struct Stages {
    using G = LineGeom<LOG2L>;
    __device__ __forceinline__ static void run(float2* v, float2* sm, int t, int c,
                                               const float2* __restrict__ stw, const float2* tw,
                                               Sync sy = Sync{0, 0}) {
        if constexpr (S < G::NSTAGES && S != STOP) {
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
                    float2 full[R - 1];
                    tw_expand<R>(full, tw + q * StageTw<LOG2L, S>::NB);
#pragma unroll
                    for (int r = 1; r < R; ++r) b[r] = cmul(b[r], full[r - 1]);
                }
                dft<R>(b);
#pragma unroll
                for (int r = 0; r < R; ++r) v[q + r * Q] = b[r];
            }
            if constexpr (!last) {
                static_assert(Q == 1 && R == 16, "only the last stage may be a tail stage");
                if constexpr (!first) sy();  // everyone has read the buffer
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
                float2 twn[StageTw<LOG2L, S + 1>::NT];
                if constexpr (S + 1 != STOP) StageTw<LOG2L, S + 1>::load(twn, t, stw);
                sy();
                Stages<LOG2L, C, S + 1, STOP>::run(v, sm, t, c, stw, twn, sy);
            }
        }
    }
};

#ifndef FB_FFT_THREADS_PER_SM
#define FB_FFT_THREADS_PER_SM 1024  // occupancy target -> register cap 65536 / this
#endif
// First step of a 2 x (N/2) four-step split of the column length, fused into the row pass:
// lane pairs (c = 0, 1) hold rows q and q + N/2 of the same column positions; X[0] = x0 + x1
// goes to row q, X[1] = (x0 - x1) W_N^q to row q + N/2.
__device__ __forceinline__ float2 pair_twiddle(int64_t q, int log2N, const float2* __restrict__ tw) {
    return __ldg(tw + ((q << (kTwLog2 - log2N)) & (kTwN - 1)));
}
// Branch-free: lane c computes (o + s v) * w_c with s = +1, w_0 = 1 for c = 0 and s = -1,
// w_1 = W_N^q for c = 1 (FFMA2 with s is exact; multiplying by (1, 0) is exact for finite
// values), so both lanes run the same three packed instructions per element.
template <int E>
__device__ __forceinline__ void pair_radix2(float2* v, int c, float2 w) {
    const float2 sgn = bc2(c == 0 ? 1.f : -1.f);
    const float2 wc = (c == 0) ? make_float2(1.f, 0.f) : w;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, v[m].x, 1), __shfl_xor_sync(0xffffffffu, v[m].y, 1));
        v[m] = cmul(__ffma2_rn(v[m], sgn, o), wc);
    }
}

// Last row stage of the pair plan fused with the pair step (C = 2 lines q, q + N/2 interleaved in
// the exchange buffer): thread (c, t) runs butterflies j = 2t + c + 2T qq (qq < Q/2) of BOTH
// lines (same butterfly arithmetic and twiddles as Stages), so the radix-2 across the pair is
// thread-local (no lane exchange) and each twiddle serves two lines; X0 = x0 + x1 goes to row q,
// X1 = (x0 - x1) W_N^q to row q + N/2 (the formulas of pair_radix2, bitwise).  Interleaved A/B
// at 2048^2 (4 x 200 reps): 37.80 us (one exchange per element pair) -> 36.97 us (butterfly
// j = t + cT, 8-byte loads) -> 35.99 us (j = 2t + c, 16-byte loads of both rows' element k).
template <int LOG2L>
struct PairLast {
    using G = LineGeom<LOG2L>;
    static constexpr int S = G::NSTAGES - 1;
    static constexpr int R = stage_radix(LOG2L, S);
    static constexpr int Ns = 1 << (4 * S);
    static constexpr int Q = G::E / R;
    static constexpr bool ok = (G::NSTAGES >= 2) && (Q % 2 == 0);
    __device__ __forceinline__ static void run(const float2* X, int t, int c, const float2* __restrict__ stw,
                                               float2 w, float2* row0, float2* row1) {
        if constexpr (ok) {
            constexpr int T = G::T, L = G::L, QH = Q / 2;
#pragma unroll
            for (int qq = 0; qq < QH; ++qq) {
                // butterfly j = 2t + c + 2T qq: adjacent lanes take adjacent butterflies, so each
                // 16-byte load (element k of both rows, interleaved in X) and each store is
                // contiguous across the warp
                const int j = 2 * t + c + qq * 2 * T;
                const float2* twp = stw + stage_tw_offset(LOG2L, S) + (j & (Ns - 1));
                float2 b0[R], b1[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 x01 = *reinterpret_cast<const float4*>(X + padk(j + r * (L / R)) * 2);
                    b0[r] = make_float2(x01.x, x01.y);
                    b1[r] = make_float2(x01.z, x01.w);
                }
                float2 tb[TwCount<R>::value], full[R - 1];
                tw_load<R, Ns>(tb, twp);
                tw_expand<R>(full, tb);
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    b0[r] = cmul(b0[r], full[r - 1]);
                    b1[r] = cmul(b1[r], full[r - 1]);
                }
                dft<R>(b0);
                dft<R>(b1);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int k = j + r * (L / R);
                    row0[k] = cadd(b0[r], b1[r]);
                    row1[k] = cmul(csub(b0[r], b1[r]), w);
                }
            }
        }
    }
};

// Last stage of a column pass (C interleaved columns, C even) with 16-byte shared accesses:
// thread (c, t) runs butterflies j = 2t + (c & 1) + 2T qq (qq < Q/2) of the column PAIR
// (2 (c >> 1), 2 (c >> 1) + 1) -- both columns' element k are adjacent in the exchange buffer and
// in the dense output staging [k][C], so inputs and outputs move as float4 (half the shared-memory
// instructions) and each twiddle serves two columns.  Same butterfly arithmetic as Stages, then
// the conj/scale epilogue; writes the results to X as the TMA store expects (after a barrier:
// other threads may still be reading their inputs).  Knob FB_FFT_COLPAIR=1; A/B neutral at
// 2048^2 (35.99 vs 35.99 us) and 4096^2, so it is off by default.
template <int LOG2L, int C>
struct ColPairLast {
    using G = LineGeom<LOG2L>;
    static constexpr int S = G::NSTAGES - 1;
    static constexpr int R = stage_radix(LOG2L, S);
    static constexpr int Ns = 1 << (4 * S);
    static constexpr int Q = G::E / R;
    static constexpr bool ok = (G::NSTAGES >= 2) && (Q % 2 == 0) && (C % 2 == 0);
    __device__ __forceinline__ static void run(float2* X, int t, int c, const float2* __restrict__ stw,
                                               int conj_out, float scale, Sync sy = Sync{0, 0}) {
        if constexpr (ok) {
            constexpr int T = G::T, L = G::L, QH = Q / 2;
            const int cp = c & ~1;  // first column of the pair
            float2 b0[QH][R], b1[QH][R];
#pragma unroll
            for (int qq = 0; qq < QH; ++qq) {
                const int j = 2 * t + (c & 1) + qq * 2 * T;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4 x01 = *reinterpret_cast<const float4*>(X + padk(j + r * (L / R)) * C + cp);
                    b0[qq][r] = make_float2(x01.x, x01.y);
                    b1[qq][r] = make_float2(x01.z, x01.w);
                }
            }
            sy();  // every thread has read its last-stage inputs; X becomes the output staging
#pragma unroll
            for (int qq = 0; qq < QH; ++qq) {
                const int j = 2 * t + (c & 1) + qq * 2 * T;
                const float2* twp = stw + stage_tw_offset(LOG2L, S) + (j & (Ns - 1));
                float2 tb[TwCount<R>::value], full[R - 1];
                tw_load<R, Ns>(tb, twp);
                tw_expand<R>(full, tb);
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    b0[qq][r] = cmul(b0[qq][r], full[r - 1]);
                    b1[qq][r] = cmul(b1[qq][r], full[r - 1]);
                }
                dft<R>(b0[qq]);
                dft<R>(b1[qq]);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float2 y0 = b0[qq][r], y1 = b1[qq][r];
                    if (conj_out) {
                        y0.y = -y0.y;
                        y1.y = -y1.y;
                    }
                    if (scale != 1.0f) {
                        y0 = __fmul2_rn(y0, bc2(scale));
                        y1 = __fmul2_rn(y1, bc2(scale));
                    }
                    *reinterpret_cast<float4*>(X + (j + r * (L / R)) * C + cp) = make_float4(y0.x, y0.y, y1.x, y1.y);
                }
            }
        }
    }
};

template <int LOG2L, int C, int MODE>
__global__ void __launch_bounds__(C * LineGeom<LOG2L>::T,
                                  (C * LineGeom<LOG2L>::T >= FB_FFT_THREADS_PER_SM) ? 1
                                  : (FB_FFT_THREADS_PER_SM / (C * LineGeom<LOG2L>::T) > 32)
                                      ? 32
                                      : FB_FFT_THREADS_PER_SM / (C * LineGeom<LOG2L>::T))
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
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();  // PDL: the previous pass's output is complete and visible

    float2 v[G::E];
    if constexpr (MODE == 1) {
        const float2* sp = src + t;
#pragma unroll
        for (int m = 0; m < G::E; ++m) v[m] = valid ? sp[m * G::T] : make_float2(0.f, 0.f);
    } else if constexpr (MODE == 2) {
        const char* sp = reinterpret_cast<const char*>(src + (int64_t)t * p.lin.es);
        const int64_t step = (int64_t)G::T * p.lin.es * (int64_t)sizeof(float2);
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            v[m] = valid ? *reinterpret_cast<const float2*>(sp) : make_float2(0.f, 0.f);
            sp += step;
        }
    } else {
        const int in_kmask = (1 << p.lin.kb_shift) - 1;
        const int64_t row = gh * p.lin.hi + gl * p.lin.lo;
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            const int k = t + m * G::T;
            if (p.peer_in) {  // block k >> kb_shift from its owner's window (NVLink load)
                const float2* b = p.peer[k >> p.lin.kb_shift] + row;
                v[m] = valid ? b[(int64_t)(k & in_kmask) * p.lin.es] : make_float2(0.f, 0.f);
            } else {
                const int64_t off = (int64_t)(k & in_kmask) * p.lin.es + (int64_t)(k >> p.lin.kb_shift) * p.lin.bs;
                v[m] = valid ? src[off] : make_float2(0.f, 0.f);
            }
        }
    }
    if (p.conj_in) {
#pragma unroll
        for (int m = 0; m < G::E; ++m) v[m].y = -v[m].y;
    }

    float2 wpair = make_float2(1.f, 0.f);
    if constexpr (C % 2 == 0) {
        if (p.pair_log2N > 0) wpair = pair_twiddle(gh, p.pair_log2N, tw);
    }
    Stages<LOG2L, C, 0>::run(v, sm, t, c, stw, nullptr);
    if constexpr (C % 2 == 0) {
        if (p.pair_log2N > 0) pair_radix2<G::E>(v, c & 1, wpair);  // nlines even: both lanes valid
    }

    if (!valid) return;
    if (p.tw4_log2N > 0) apply_tw4<G::E, G::T>(v, gh, t, p.tw4_log2N, tw);  // four-step twiddle W_N^{gh k}
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
    if constexpr (MODE == 1) {
        float2* dp = dst + t;
#pragma unroll
        for (int m = 0; m < G::E; ++m) dp[m * G::T] = v[m];
    } else if constexpr (MODE == 2) {
        char* dp = reinterpret_cast<char*>(dst + (int64_t)t * p.lout.es);
        const int64_t step = (int64_t)G::T * p.lout.es * (int64_t)sizeof(float2);
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            *reinterpret_cast<float2*>(dp) = v[m];
            dp += step;
        }
    } else {
        const int out_kmask = (1 << p.lout.kb_shift) - 1;
        const int64_t row = gh * p.lout.hi + gl * p.lout.lo;
#pragma unroll
        for (int m = 0; m < G::E; ++m) {
            const int k = t + m * G::T;
            if (p.peer_out) {  // block k >> kb_shift into its owner's window (NVLink store)
                p.peer[k >> p.lout.kb_shift][row + (int64_t)(k & out_kmask) * p.lout.es] = v[m];
            } else {
                const int64_t off = (int64_t)(k & out_kmask) * p.lout.es + (int64_t)(k >> p.lout.kb_shift) * p.lout.bs;
                dst[off] = v[m];
            }
        }
    }
}

static bool fft_pdl_enabled() { return knobs().fft_no_pdl == 0; }

// Launch with programmatic stream serialization: the kernel may start while the previous
// kernel on the stream drains; every FFT kernel calls pdl_wait() before touching global memory.
template <typename Kern, typename... Args>
static fb_status launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = fft_pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
    FB_LAUNCH_CHECK("fft pass");
    return FB_OK;
}

template <int LOG2L, int C, int MODE>
static fb_status launch_one(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    using G = LineGeom<LOG2L>;
    constexpr int threads = C * G::T;
    static_assert(threads <= 1024, "CTA too large");
    const size_t smem = (G::NSTAGES > 1) ? (size_t)C * G::PADL * sizeof(float2) : 0;
    static DevOnce once;
    const int dev = DevOnce::dev();
    if (smem > 48 * 1024 && !once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(fft_pass_kernel<LOG2L, C, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        once.set(dev);
    }
    const int64_t blocks = (p.nlines + C - 1) / C;
    if (blocks > 0x7fffffff) {
        set_error("FFT pass grid too large (%lld CTAs)", (long long)blocks);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    FB_TRY(launch_pdl(fft_pass_kernel<LOG2L, C, MODE>, dim3((unsigned)blocks), dim3(threads), smem, s, p,
                      (const float2*)st->twiddles, (const float2*)st->stage_tw));
    return FB_OK;
}

template <int LOG2L, int C>
static fb_status launch_LC(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    const bool plain = p.lin.kb_shift >= LOG2L && p.lout.kb_shift >= LOG2L;
    if (plain && p.lin.es == 1 && p.lout.es == 1) return launch_one<LOG2L, C, 1>(p, st, s);
    if (plain) return launch_one<LOG2L, C, 2>(p, st, s);
    return launch_one<LOG2L, C, 0>(p, st, s);
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

// =====================================================================================
// Persistent, TMA-pipelined pass (the fast path).  Each CTA loops over groups of C lines;
// while group i is transformed, the async proxy is already filling the other staging buffer
// with group i+1 (two staging buffers, one mbarrier each), so global-load latency is hidden
// and no LSU instruction touches the strided input:
//   KIND_ROW: lines (or per-peer line segments) are contiguous -> 1D bulk copies
//             (cp.async.bulk) into S[c][k]; outputs leave by coalesced direct stores.
//   KIND_COL: lines are adjacent columns -> one 3D TMA tensor box per 256 elements into
//             S[k][c] (32 B or 16 B row segments gathered by the TMA engine); outputs are
//             written densely to the exchange buffer and leave by TMA tensor stores.
// Stage 1 reads S, later stages exchange through the padded buffer X exactly as in
// fft_pass_kernel (same arithmetic, same results bit for bit).
// =====================================================================================
enum { KIND_ROW = 1, KIND_COL = 2 };

template <int LOG2L, int C, int KIND, int NB = 2>
struct TmaGeom {
    using G = LineGeom<LOG2L>;
    static constexpr int PADS = (KIND == KIND_ROW && C > 1) ? 16 / C : 0;  // S line pad (row kind)
    static constexpr int SLINE = G::L + PADS;
    static constexpr int S_ELEMS = (KIND == KIND_ROW) ? C * SLINE : C * G::L;
    static constexpr int X_ELEMS = C * G::PADL;
    static constexpr size_t SMEM = (size_t)(NB * S_ELEMS + X_ELEMS) * sizeof(float2) + 64;
    static constexpr int BOX = G::L < 256 ? G::L : 256;  // COL: elements per TMA box
};

// Occupancy policy of the persistent pass: CTAs of <= 256 threads are compiled for 3 per SM
// (register cap 85; the 16-element line code needs ~80 without spills) and get one staging
// buffer when that lets 3 fit in shared memory (A/B at 2048^2: 39 us vs 42 us with 2 CTAs/SM
// and two buffers); larger CTAs keep 1 per SM minimum and two buffers.
#ifndef FB_FFT_TMA_SMALL_MINB
#define FB_FFT_TMA_SMALL_MINB 3
#endif
template <int THREADS>
constexpr int tma_minb() { return THREADS <= 256 ? FB_FFT_TMA_SMALL_MINB : 1; }
template <int LOG2L, int C, int KIND>
constexpr int tma_nb() {
    return (C * LineGeom<LOG2L>::T <= 256 && 3 * (TmaGeom<LOG2L, C, KIND, 1>::SMEM + 1024) <= 228 * 1024) ? 1 : 2;
}

// SUB > 1: one CTA per SM made of SUB independent sub-CTAs (C*T threads each, own staging and
// exchange buffers, own mbarriers, named barrier 1 + sub), which take the CTA's groups
// {blockIdx + i gridDim} from a shared-memory counter as they free up.  With SUB separate CTAs
// per SM instead, each CTA had a fixed share and the warp arbiter starves some of them: in
// the 2048^2 trace (tools/fft_trace.py) an SM's three CTAs finished 3-4 us apart and the last
// one ran alone; the SM-local queue hands the remaining groups to whichever sub-CTA is free.
template <int LOG2L, int C, int KIND, bool OUT_GENERIC, int NB, int SUB = 1>
__global__ void __launch_bounds__(SUB * C * LineGeom<LOG2L>::T,
                                  SUB == 1 ? tma_minb<C * LineGeom<LOG2L>::T>() : 1)
    fft_pass_tma_kernel(const FftPass p, const __grid_constant__ CUtensorMap tin,
                        const __grid_constant__ CUtensorMap tout, const float2* __restrict__ tw,
                        const float2* __restrict__ stw, int64_t ngroups, int64_t nh_in) {
    using G = LineGeom<LOG2L>;
    using TG = TmaGeom<LOG2L, C, KIND, NB>;
    static_assert(NB == 1 || NB == 2, "one or two staging buffers");
    constexpr int L = G::L, T = G::T, E = G::E;
    constexpr int NT = C * T;  // threads of one (sub-)CTA
    extern __shared__ __align__(128) float2 smf[];
    // sub-CTA of this warp: interleaved (warp w -> sub w % SUB) so that every sub-CTA holds warps
    // of every scheduler-priority level (the arbiter favours high warp ids; contiguous warp
    // ranges would let one sub-CTA starve the others), or contiguous (knob FB_FFT_SUB_ILV=0)
    const int wid = (int)(threadIdx.x >> 5);
    const int sub = (SUB == 1) ? 0 : (p.sub_ilv ? wid % SUB : wid / (NT / 32));
    float2* Sbuf = smf + sub * (NB * TG::S_ELEMS + TG::X_ELEMS);
    float2* X = Sbuf + NB * TG::S_ELEMS;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smf + SUB * (NB * TG::S_ELEMS + TG::X_ELEMS)) + 2 * sub;
    __shared__ int64_t slot_grp[SUB][2];  // SUB > 1: group staged in buffer b of sub-CTA sub
    __shared__ unsigned int q_next;        // SUB > 1: next index into this CTA's group list
    const Sync sy{SUB == 1 ? 0 : 1 + sub, NT};
    const int tid = (SUB == 1) ? (int)threadIdx.x
                               : (p.sub_ilv ? (wid / SUB) * 32 + (int)(threadIdx.x & 31) : (int)threadIdx.x - sub * NT);
    const int c = tid % C;
    const int t = tid / C;
    const int gshift = p.g_shift >= 62 ? 62 : p.g_shift;
    const int64_t gmask = (gshift >= 62) ? -1 : ((int64_t(1) << gshift) - 1);

    if (tid == 0) {
        ptx::mbar_init(ptx::smem_u32(&bars[0]), 1);
        ptx::mbar_init(ptx::smem_u32(&bars[1]), 1);
        ptx::fence_mbar_init();
        if (sub == 0) {
            q_next = 0;
            if constexpr (KIND == KIND_COL) {
                ptx::tma_prefetch_desc(&tin);
                ptx::tma_prefetch_desc(&tout);
            }
        }
    }
    __syncthreads();
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();  // PDL: everything above overlapped the previous grid's tail
#if FB_FFT_TRACE
    unsigned long long* tr =
        p.trace ? p.trace + ((size_t)p.trace_slot * 1024 + blockIdx.x * SUB + sub) * 32 : nullptr;
    auto gtime = []() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    };
    if (tid == 0 && tr) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        tr[0] = smid;
        tr[1] = gtime();
    }
#endif

    // thread 0: start the asynchronous fill of staging buffer `buf` with group `grp`
    auto issue = [&](int64_t grp, int buf) {
        float2* S = Sbuf + buf * TG::S_ELEMS;
        const uint32_t bar = ptx::smem_u32(&bars[buf]);
        const int64_t g0 = grp * C;
        if constexpr (KIND == KIND_COL) {
            ptx::mbar_arrive_expect_tx(bar, (uint32_t)(C * L * sizeof(float2)));
            const int64_t gh = (gshift >= 62) ? 0 : (g0 >> gshift);
            const int gl = (int)(g0 & gmask);
#pragma unroll 1
            for (int kb = 0; kb < L; kb += TG::BOX)
                ptx::tma_load_3d(ptx::smem_u32(S + kb * C), &tin, bar, gl, kb, (int)gh);
        } else {
            const int64_t nv = (p.nlines - g0) < C ? (p.nlines - g0) : C;
            const int seg = (p.lin.kb_shift >= LOG2L) ? L : (1 << p.lin.kb_shift);
            ptx::mbar_arrive_expect_tx(bar, (uint32_t)(nv * L * sizeof(float2)));
            for (int cl = 0; cl < nv; ++cl) {
                const int64_t g = g0 + cl;
                const int64_t gh = (gshift >= 62) ? 0 : (g >> gshift);
                const float2* src = p.in + gh * p.lin.hi + (g & gmask) * p.lin.lo;
#pragma unroll 1
                for (int k0 = 0; k0 < L; k0 += seg)
                    ptx::bulk_load(ptx::smem_u32(S + cl * TG::SLINE + k0), src + (int64_t)(k0 / seg) * p.lin.bs,
                                   (uint32_t)(seg * sizeof(float2)), bar);
            }
        }
    };

    const int dbg = FB_DEBUG_BUILD ? p.debug : 0;  // timing decomposition (debug builds only)
    const bool dbg_noload = (dbg & 2) != 0;
    // SUB > 1: thread 0 of a sub-CTA takes the next group of this CTA's list from q_next and
    // publishes it in slot_grp before the buffer's mbarrier phase completes (the arrive has
    // release semantics); "no more work" completes the phase with a plain arrive.
    volatile int64_t* vslot = slot_grp[sub];
    auto take = [&]() -> int64_t {
        const int64_t g = blockIdx.x + (int64_t)atomicAdd(&q_next, 1u) * gridDim.x;
        if constexpr (C % 2 == 0) {  // the pair twiddle is read right after the wait: warm it
            if (p.pair_log2N > 0 && g < ngroups) {
                const int64_t gq = (g * C) >> ((gshift >= 62) ? 62 : gshift);
                asm volatile("prefetch.global.L2 [%0];" ::"l"(tw + ((gq << (kTwLog2 - p.pair_log2N)) & (kTwN - 1))));
            }
        }
        return g;
    };
    auto feed = [&](int64_t grp, int buf) {
        vslot[buf] = grp;
        if (grp < ngroups && !dbg_noload)
            issue(grp, buf);
        else
            ptx::mbar_arrive(ptx::smem_u32(&bars[buf]));
    };
    if (tid == 0) {
        // Staggered start: CTA slot s (the s-th CTA placed on an SM, or sub-CTA s) issues its
        // first load s * stagger_ns later, so the slot-0 CTAs get their first group from a less
        // crowded memory system and start computing earlier (interleaved A/B at 2048^2, 4 x 150
        // reps: 38.74 -> 38.21 us at 300 ns; no effect at 1024^2 / 4096^2).  Knob FB_FFT_STAGGER
        // (ns); default 600 since the fused pair stage (3 x 200 reps interleaved, 2048^2: 300 ns
        // 36.20, 600 ns 35.87, 900 ns 35.86, 1200 ns 35.95 us; 1024^2 / 4096^2 within 0.05 us).
        if (p.stagger_ns > 0 && p.sm_count > 0) {
            const int slot = (SUB > 1) ? sub : (int)(blockIdx.x / (unsigned)p.sm_count);
            for (int i = 0; i < slot; ++i) __nanosleep((unsigned)p.stagger_ns);
        }
        if constexpr (SUB > 1) {
            feed(take(), 0);
            if (NB == 2) feed(take(), 1);
        } else if (!dbg_noload) {
            if ((int64_t)blockIdx.x < ngroups) issue(blockIdx.x, 0);
            if (NB == 2 && (int64_t)blockIdx.x + gridDim.x < ngroups) issue((int64_t)blockIdx.x + gridDim.x, 1);
        }
    }
    (void)nh_in;

    int it = 0;
    for (int64_t grp = blockIdx.x; SUB > 1 || grp < ngroups; grp += gridDim.x, ++it) {
        float2 wpair = make_float2(1.f, 0.f);  // pair-plan twiddle, loaded before the data wait
        if constexpr (C % 2 == 0 && SUB == 1) {
            if (p.pair_log2N > 0) {
                const int64_t gq = (grp * C + c) >> ((gshift >= 62) ? 62 : gshift);
                wpair = pair_twiddle(gq, p.pair_log2N, tw);
            }
        }
        const int buf = (NB == 2) ? (it & 1) : 0;
        const float2* S = Sbuf + buf * TG::S_ELEMS;
#if FB_FFT_TRACE
        if (tid == 0 && tr && it < 14) tr[2 + 2 * it] = gtime();
#endif
        if (SUB > 1 || !dbg_noload)
            ptx::mbar_wait(ptx::smem_u32(&bars[buf]), (uint32_t)((NB == 2) ? (it >> 1) : it) & 1u);
#if FB_FFT_TRACE
        if (tid == 0 && tr && it < 14) tr[3 + 2 * it] = gtime();
#endif
        if constexpr (SUB > 1) {
            grp = vslot[buf];
            if (grp >= ngroups) break;  // uniform across the sub-CTA
            if constexpr (C % 2 == 0) {
                if (p.pair_log2N > 0) {
                    const int64_t gq = (grp * C + c) >> ((gshift >= 62) ? 62 : gshift);
                    wpair = pair_twiddle(gq, p.pair_log2N, tw);
                }
            }
        }
        float2 v[E];
        if constexpr (KIND == KIND_COL) {
            const float2* sp = S + t * C + c;
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = sp[m * T * C];
        } else {
            const float2* sp = S + c * TG::SLINE + t;
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = sp[m * T];
        }
        if (p.conj_in) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m].y = -v[m].y;
        }
        // order this thread's generic-proxy reads of S[buf] before the async-proxy (TMA)
        // refill of S[buf] that thread 0 issues after the barrier
        ptx::fence_proxy_async_smem();
        if constexpr (KIND == KIND_COL) {
            if (tid == 0) ptx::bulk_wait_read0();  // previous group's TMA store has read X
        }
        sy();  // S[buf] consumed by everyone; X free
        if (tid == 0) {
            if constexpr (SUB > 1) {
                feed(take(), buf);
            } else if (!dbg_noload) {
                const int64_t nxt = grp + NB * (int64_t)gridDim.x;
                if (nxt < ngroups) issue(nxt, buf);
            }
        }

        if constexpr (KIND == KIND_ROW && C == 2 && !OUT_GENERIC && PairLast<LOG2L>::ok) {
            if (p.pair_log2N > 0 && p.pair_half_shfl == 2 && p.tw4_log2N == 0 && !p.conj_out && p.scale == 1.0f &&
                !dbg) {
                Stages<LOG2L, C, 0, PairLast<LOG2L>::S>::run(v, X, t, c, stw, nullptr, sy);
                const int64_t gq = (grp * C) >> ((gshift >= 62) ? 62 : gshift);
                float2* row0 = p.out + gq * p.lout.hi;
                PairLast<LOG2L>::run(X, t, c, stw, wpair, row0, row0 + p.lout.lo);
                continue;
            }
        }
        if constexpr (KIND == KIND_COL && ColPairLast<LOG2L, C>::ok) {
            if (p.col_pair_last && !p.col_stg && p.tw4_log2N == 0 && p.pair_log2N == 0 && !dbg) {
                Stages<LOG2L, C, 0, ColPairLast<LOG2L, C>::S>::run(v, X, t, c, stw, nullptr, sy);
                ColPairLast<LOG2L, C>::run(X, t, c, stw, p.conj_out, p.scale, sy);
                ptx::fence_proxy_async_smem();
                sy();
                if (tid == 0) {
                    const int64_t g0 = grp * C;
                    const int64_t gh0 = (gshift >= 62) ? 0 : (g0 >> gshift);
                    const int gl0 = (int)(g0 & gmask);
#pragma unroll 1
                    for (int kb = 0; kb < L; kb += TG::BOX)
                        ptx::tma_store_3d(&tout, ptx::smem_u32(X + kb * C), gl0, kb, (int)gh0);
                    ptx::bulk_commit();
                }
                continue;
            }
        }
        if (!(dbg & 1)) Stages<LOG2L, C, 0>::run(v, X, t, c, stw, nullptr, sy);
        if (dbg & 4) continue;

        const int64_t g = grp * C + c;
        const int64_t gh = (gshift >= 62) ? 0 : (g >> gshift);
        if constexpr (KIND == KIND_ROW && C == 2 && !OUT_GENERIC) {
            // Pair step with half the lane exchanges: lane c keeps the elements m = 2i + c of
            // BOTH rows (one shuffle per element pair instead of one per element) and writes
            // X0 = x0 + x1 to row q and X1 = (x0 - x1) W_N^q to row q + N/2.  Lane 1 forms
            // (x1 + x0) and (x1 - x0)(-W): bitwise the same values as lane 0's formulas.
            // Interleaved A/B at 2048^2 (6 x 200 reps): 38.39 -> 37.55 us; 512^2 11.44 -> 11.30 us.
            if (p.pair_log2N > 0 && p.pair_half_shfl && p.tw4_log2N == 0 && !p.conj_out && p.scale == 1.0f) {
                const float2 sw = (c == 0) ? wpair : make_float2(-wpair.x, -wpair.y);
                float2* row0 = p.out + gh * p.lout.hi;
                float2* row1 = row0 + p.lout.lo;
#pragma unroll
                for (int i = 0; i < E / 2; ++i) {
                    const float2 a = v[2 * i], b = v[2 * i + 1];
                    const float2 snd = c ? a : b;
                    const float2 mine = c ? b : a;
                    const float2 r = make_float2(__shfl_xor_sync(0xffffffffu, snd.x, 1),
                                                 __shfl_xor_sync(0xffffffffu, snd.y, 1));
                    const int k = t + (2 * i + c) * T;
                    row0[k] = cadd(mine, r);
                    row1[k] = cmul(csub(mine, r), sw);
                }
                continue;
            }
        }
        if constexpr (C % 2 == 0) {
            if (p.pair_log2N > 0) pair_radix2<E>(v, c & 1, wpair);
        }
        if (p.tw4_log2N > 0) apply_tw4<E, T>(v, gh, t, p.tw4_log2N, tw);  // four-step twiddle W_N^{gh k}
        if (p.conj_out) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m].y = -v[m].y;
        }
        if (p.scale != 1.0f) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = __fmul2_rn(v[m], bc2(p.scale));
        }
        if (KIND == KIND_COL && p.col_stg) {
            // column results straight from registers (C-wide row segments per warp store)
            const int64_t row = gh * p.lout.hi + (g & gmask) * p.lout.lo;
            float2* dp = p.out + row + (int64_t)t * p.lout.es;
            const int64_t step = (int64_t)T * p.lout.es;
#pragma unroll
            for (int m = 0; m < E; ++m) dp[m * step] = v[m];
        } else if constexpr (KIND == KIND_COL) {
            sy();  // last stage finished reading X
            float2* xp = X + t * C + c;
#pragma unroll
            for (int m = 0; m < E; ++m) xp[m * T * C] = v[m];
            ptx::fence_proxy_async_smem();
            sy();
            if (tid == 0) {
                const int64_t g0 = grp * C;
                const int64_t gh0 = (gshift >= 62) ? 0 : (g0 >> gshift);
                const int gl0 = (int)(g0 & gmask);
#pragma unroll 1
                for (int kb = 0; kb < L; kb += TG::BOX)
                    ptx::tma_store_3d(&tout, ptx::smem_u32(X + kb * C), gl0, kb, (int)gh0);
                ptx::bulk_commit();
            }
        } else {
            if (g < p.nlines) {
                float2* dst = p.out + gh * p.lout.hi + (g & gmask) * p.lout.lo;
                if constexpr (!OUT_GENERIC) {
                    float2* dp = dst + t;
#pragma unroll
                    for (int m = 0; m < E; ++m) dp[m * T] = v[m];
                } else {
                    const int out_kmask = (1 << p.lout.kb_shift) - 1;
                    const int64_t row = gh * p.lout.hi + (g & gmask) * p.lout.lo;
#pragma unroll
                    for (int m = 0; m < E; ++m) {
                        const int k = t + m * T;
                        if (p.peer_out)  // block k >> kb_shift into its owner's window (NVLink store)
                            p.peer[k >> p.lout.kb_shift][row + (int64_t)(k & out_kmask) * p.lout.es] = v[m];
                        else
                            dst[(int64_t)(k & out_kmask) * p.lout.es + (int64_t)(k >> p.lout.kb_shift) * p.lout.bs] =
                                v[m];
                    }
                }
            }
        }
    }
    if constexpr (KIND == KIND_COL) {
        if (tid == 0) ptx::bulk_wait0();
    }
#if FB_FFT_TRACE
    if (tid == 0 && tr) {
        tr[30] = gtime();
        tr[31] = it;
    }
#endif
}

// ------------------------------------------------------------ host side of the TMA path
typedef CUresult (*EncodeTiledFnFFT)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFnFFT fft_encoder() {
    static EncodeTiledFnFFT fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFnFFT)f;
    }
    return fn;
}

// 3D view {line-lo (contiguous lines), element k (stride es), line-hi (stride hi)} of 8-byte
// complex elements; box {C, min(L,256), 1}.
static bool make_col_map(CUtensorMap* m, const void* base, int64_t glo, int64_t L, int64_t nh, int64_t es,
                         int64_t hi, int C) {
    EncodeTiledFnFFT enc = fft_encoder();
    if (!enc) return false;
    if (nh <= 1) hi = es * L;  // unused dimension; any legal stride
    cuuint64_t dims[3] = {(cuuint64_t)glo, (cuuint64_t)L, (cuuint64_t)(nh < 1 ? 1 : nh)};
    cuuint64_t strides[2] = {(cuuint64_t)(es * 8), (cuuint64_t)(hi * 8)};
    cuuint32_t box[3] = {(cuuint32_t)C, (cuuint32_t)(L < 256 ? L : 256), 1u};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LOG2L, int C, int KIND, bool OUT_GENERIC, int NB = 2, int SUB = 1>
static fb_status launch_tma_one(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    using TG = TmaGeom<LOG2L, C, KIND, NB>;
    constexpr int threads = SUB * C * LineGeom<LOG2L>::T;
    constexpr size_t SMEM = (size_t)SUB * (NB * TG::S_ELEMS + TG::X_ELEMS) * sizeof(float2) + 64;
    auto kern = fft_pass_tma_kernel<LOG2L, C, KIND, OUT_GENERIC, NB, SUB>;
    static DevOnce once;
    static std::atomic<int> occ[32];
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
        int nb = 0;
        FB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, SMEM));
        occ[dev].store(nb < 1 ? 1 : nb);
        once.set(dev);
    }
    const int64_t ngroups = (p.nlines + C - 1) / C;
    int64_t grid = (int64_t)st->sm_count * occ[dev].load();
    if (grid > ngroups) grid = ngroups;
    CUtensorMap tin, tout;
    memset(&tin, 0, sizeof(tin));
    memset(&tout, 0, sizeof(tout));
    int64_t nh = 1;
    if (KIND == KIND_COL) {
        const int gshift = p.g_shift >= 62 ? 62 : p.g_shift;
        const int64_t glo = (gshift >= 62) ? p.nlines : (int64_t(1) << gshift);
        nh = (p.nlines + glo - 1) / glo;
        if (!make_col_map(&tin, p.in, glo, int64_t(1) << LOG2L, nh, p.lin.es, p.lin.hi, C) ||
            !make_col_map(&tout, p.out, glo, int64_t(1) << LOG2L, nh, p.lout.es, p.lout.hi, C)) {
            set_error("cuTensorMapEncodeTiled failed for an FFT column pass");
            return FB_ERR_CUDA;
        }
    }
    // Column outputs: direct stores from registers when a warp store covers whole 128-byte row
    // segments (C = 16), else the exchange buffer + TMA tensor store (A/B, means of 3 x 100:
    // 512^2 12.06 -> 11.36 us and 16384^2 2.892 -> 2.870 ms with direct stores; 2048^2
    // (C = 4, 32-byte segments) 37.84 -> 40.13 us and 4096^2 157.7 -> 167.1 us, so those keep
    // the TMA store).  Knob FB_FFT_COL_STG = 0 / 1 forces.
    FftPass pk = p;
    pk.sub_ilv = knobs().fft_sub_ilv;
    if (KIND == KIND_COL) pk.col_stg = (p.col_stg >= 0) ? p.col_stg : (C >= 16 ? 1 : 0);
    FB_TRY(launch_pdl(kern, dim3((unsigned)grid), dim3(threads), SMEM, s, pk, tin, tout,
                      (const float2*)st->twiddles, (const float2*)st->stage_tw, ngroups, nh));
    return FB_OK;
}


// Picks the TMA path when the pass is expressible; returns false to fall back.
static bool tma_eligible(const FftPass& p, int& kind, int& C, bool& out_generic) {
    const int l = p.log2L;
    if (l < 6 || l > 12) return false;  // >= 64 elements, staging fits for <= 4096
    if (p.peer_in) return false;        // peer loads take the LSU path (no bulk copies from peers)
    if (p.peer_out && p.col_like) return false;
    const bool al_in = ((uintptr_t)p.in & 15) == 0, al_out = ((uintptr_t)p.out & 15) == 0;
    if (!al_in || !al_out) return false;
    const bool in_plain = p.lin.kb_shift >= l, out_plain = p.lout.kb_shift >= l;
    const int gshift = p.g_shift >= 62 ? 62 : p.g_shift;
    if (p.col_like && p.lin.lo == 1 && p.lout.lo == 1 && in_plain && out_plain) {
        if (knobs().fft_no_tma_col) return false;
        // widest row segment (up to 128 B = 16 columns) whose double-buffered staging plus
        // exchange buffer stays near 100 KiB (two CTAs per SM)
        // widest row segment whose staging stays small: 128-long columns (the 16384^2 four-step
        // passes) take 32 columns = 256-byte segments (A/B 2721 -> 2534 us at 16384^2: the first
        // four-step pass gathers rows 16 MiB apart, where longer DRAM bursts pay)
        C = (l == 6 || l == 7) ? 32 : (l <= 8) ? 16 : (l == 9 ? 8 : (l == 10 ? 4 : 2));
        const int kc = knobs().fft_col_c;
        if (kc == 2 || kc == 4 || kc == 8 || kc == 16 || (kc == 32 && (l == 6 || l == 7))) C = kc;
        if (C * (1 << l) / 16 > 1024 || (size_t)C * (1 << l) * 8 * 3 > 200 * 1024) return false;
        const int64_t glo = (gshift >= 62) ? p.nlines : (int64_t(1) << gshift);
        if (glo % C) return false;
        if ((p.lin.es * 8) % 16 || (p.lout.es * 8) % 16) return false;
        const int64_t nh = (p.nlines + glo - 1) / glo;
        if (nh > 1 && ((p.lin.hi * 8) % 16 || (p.lout.hi * 8) % 16)) return false;
        if (glo > (int64_t(1) << 31) || nh > (int64_t(1) << 31)) return false;
        kind = KIND_COL;
        out_generic = false;
        return true;
    }
    // row lines; the pair plan addresses line g = 2q + c at q*hi + c*lo (lo = n0/2 rows)
    const bool lo_ok = (p.lout.lo == 0 && p.lin.lo == 0) ||
                       (p.pair_log2N > 0 && (p.lin.lo * 8) % 16 == 0 && (p.lout.lo * 8) % 16 == 0);
    if (!p.col_like && p.lin.es == 1 && lo_ok) {
        if (knobs().fft_no_tma_row) return false;
        const int seg = in_plain ? (1 << l) : (1 << p.lin.kb_shift);
        if (seg < 2) return false;
        if ((p.lin.hi * 8) % 16) return false;
        if (!in_plain && (p.lin.bs * 8) % 16) return false;
        if (p.lout.es != 1) return false;
        C = p.pair_log2N > 0 ? 2 : 1;
        kind = KIND_ROW;
        out_generic = !out_plain;
        return true;
    }
    return false;
}

// Staging-buffer count: one buffer (3 CTAs/SM) when the tma_nb policy allows it and every
// CTA then still has >= 2 groups to stream (A/B: 2048^2 38 us vs 42, 16384^2 2.97 ms vs
// 3.05); with fewer groups per CTA (<= 1024^2) two buffers and 2 CTAs/SM avoid a serial
// second group on a third of the CTAs (17.4 us vs 19.0 at 1024^2).  Knob (1 or 2) forces.
template <int LOG2L, int C, int KIND>
static fb_status launch_tma_nb(const FftPass& p, const DeviceState* st, cudaStream_t s, int knob_nb) {
    constexpr int D = tma_nb<LOG2L, C, KIND>();
    int nb = D;
    if constexpr (D == 1) {
        constexpr int occ1 = (int)((228 * 1024) / (TmaGeom<LOG2L, C, KIND, 1>::SMEM + 1024));
        const int64_t ngroups = (p.nlines + C - 1) / C;
        if (ngroups < 2 * (int64_t)st->sm_count * (occ1 < 3 ? occ1 : 3)) nb = 2;
    }
    if (knob_nb == 1 || knob_nb == 2) nb = knob_nb;
    if (nb == 3 - D) return launch_tma_one<LOG2L, C, KIND, false, 3 - D>(p, st, s);
    if constexpr (D == 1 && (C * LineGeom<LOG2L>::T) % 32 == 0) {
        // the one-buffer configuration runs as SUB = 3 sub-CTAs of one CTA per SM (SM-local
        // group queue, see fft_pass_tma_kernel) when every sub-CTA streams many groups;
        // knob FB_FFT_SUB=1: three separate CTAs always, 3: sub-CTAs always
        const int64_t ngroups = (p.nlines + C - 1) / C;
        const int sub = knobs().fft_sub;
        if (sub == 3 || (sub == 0 && ngroups >= 48 * (int64_t)st->sm_count))
            return launch_tma_one<LOG2L, C, KIND, false, 1, 3>(p, st, s);
    }
    return launch_tma_one<LOG2L, C, KIND, false, D>(p, st, s);
}

template <int LOG2L>
static fb_status launch_tma_L(const FftPass& p, int kind, int C, bool og, const DeviceState* st, cudaStream_t s) {
    constexpr int T = LineGeom<LOG2L>::T;
    if (kind == KIND_COL) {
        if (C == 2) return launch_tma_nb<LOG2L, 2, KIND_COL>(p, st, s, knobs().fft_col_nb);
        if (C == 4) return launch_tma_nb<LOG2L, 4, KIND_COL>(p, st, s, knobs().fft_col_nb);
        if constexpr (8 * T <= 1024 && LOG2L <= 11)
            if (C == 8) return launch_tma_nb<LOG2L, 8, KIND_COL>(p, st, s, knobs().fft_col_nb);
        if constexpr (16 * T <= 1024 && LOG2L <= 10)
            if (C == 16) return launch_tma_nb<LOG2L, 16, KIND_COL>(p, st, s, knobs().fft_col_nb);
        if constexpr (32 * T <= 256 && (LOG2L == 6 || LOG2L == 7))
            if (C == 32) return launch_tma_nb<LOG2L, 32, KIND_COL>(p, st, s, knobs().fft_col_nb);
    } else {
        if (C == 2) return launch_tma_nb<LOG2L, 2, KIND_ROW>(p, st, s, knobs().fft_row_nb);
        if (!og) return launch_tma_nb<LOG2L, 1, KIND_ROW>(p, st, s, knobs().fft_row_nb);
        return launch_tma_one<LOG2L, 1, KIND_ROW, true>(p, st, s);
    }
    set_error("internal: no TMA FFT instantiation");
    return FB_ERR_UNSUPPORTED_SIZE;
}

static bool g_fft_tma_disabled() { return knobs().fft_no_tma == 1; }


// =====================================================================================
// Long rows (L = 16384, one line per CTA, 1024 threads): the padded exchange buffer alone is
// 139 KB, so a second full staging buffer does not fit and the plain kernel leaves the SM idle
// while each line loads.  This persistent kernel streams the NEXT line in two halves while the
// current one is transformed: elements [0, L/2) go to a 64 KB staging buffer as soon as stage 1
// has read it, elements [L/2, L) into the (dense) start of the exchange buffer once the last
// exchange has been read.  Stage 1 reads the dense halves directly (thread t: k = t + 1024 m).
// =====================================================================================
template <bool OUT_GENERIC>
__global__ void __launch_bounds__(1024, 1)
    fft_longrow_kernel(const FftPass p, const float2* __restrict__ tw, const float2* __restrict__ stw) {
    constexpr int LOG2L = 14;
    using G = LineGeom<LOG2L>;
    constexpr int L = G::L, T = G::T, E = G::E, H = L / 2;
    extern __shared__ __align__(128) float2 smf[];
    float2* X = smf;                  // [PADL] exchange; its first H elements also stage the second half
    float2* S = smf + G::PADL;        // [H] first-half staging
    uint64_t* bars = reinterpret_cast<uint64_t*>(S + H);
    const int t = threadIdx.x;
    const uint32_t bar_a = ptx::smem_u32(&bars[0]), bar_b = ptx::smem_u32(&bars[1]);
    if (t == 0) {
        ptx::mbar_init(bar_a, 1);
        ptx::mbar_init(bar_b, 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    auto line_src = [&](int64_t g) { return p.in + g * p.lin.hi; };
    const int64_t nl = p.nlines;
    int64_t g = blockIdx.x;
    if (t == 0 && g < nl) {
        ptx::mbar_arrive_expect_tx(bar_a, H * sizeof(float2));
        ptx::bulk_load(ptx::smem_u32(S), line_src(g), H * sizeof(float2), bar_a);
        ptx::mbar_arrive_expect_tx(bar_b, H * sizeof(float2));
        ptx::bulk_load(ptx::smem_u32(X), line_src(g) + H, H * sizeof(float2), bar_b);
    }
    for (int it = 0; g < nl; g += gridDim.x, ++it) {
        const int64_t gn = g + gridDim.x;
        ptx::mbar_wait(bar_a, (uint32_t)it & 1u);
        ptx::mbar_wait(bar_b, (uint32_t)it & 1u);
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = (m < E / 2) ? S[t + m * T] : X[t + (m - E / 2) * T];
        if (p.conj_in) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m].y = -v[m].y;
        }
        ptx::fence_proxy_async_smem();
        __syncthreads();  // S and X consumed
        if (t == 0 && gn < nl) {
            ptx::mbar_arrive_expect_tx(bar_a, H * sizeof(float2));
            ptx::bulk_load(ptx::smem_u32(S), line_src(gn), H * sizeof(float2), bar_a);
        }
        Stages<LOG2L, 1, 0>::run(v, X, t, 0, stw, nullptr);
        ptx::fence_proxy_async_smem();
        __syncthreads();  // the last exchange has been read
        if (t == 0 && gn < nl) {
            ptx::mbar_arrive_expect_tx(bar_b, H * sizeof(float2));
            ptx::bulk_load(ptx::smem_u32(X), line_src(gn) + H, H * sizeof(float2), bar_b);
        }
        if (p.conj_out) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m].y = -v[m].y;
        }
        if (p.scale != 1.0f) {
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = __fmul2_rn(v[m], bc2(p.scale));
        }
        float2* dst = p.out + g * p.lout.hi;
        if constexpr (!OUT_GENERIC) {
#pragma unroll
            for (int m = 0; m < E; ++m) dst[t + m * T] = v[m];
        } else {
            const int out_kmask = (1 << p.lout.kb_shift) - 1;
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int k = t + m * T;
                if (p.peer_out)
                    p.peer[k >> p.lout.kb_shift][g * p.lout.hi + (int64_t)(k & out_kmask) * p.lout.es] = v[m];
                else
                    dst[(int64_t)(k & out_kmask) * p.lout.es + (int64_t)(k >> p.lout.kb_shift) * p.lout.bs] = v[m];
            }
        }
    }
}

static bool longrow_eligible(const FftPass& p) {
    if (p.log2L != 14 || p.col_like || p.pair_log2N || p.peer_in || p.tw4_log2N || p.lin.lo || p.lout.lo) return false;
    if (p.g_shift != 0 && p.g_shift < 62) return false;
    if (p.lin.es != 1 || p.lin.kb_shift < 14 || p.lout.es != 1) return false;
    if (((uintptr_t)p.in & 15) || ((uintptr_t)p.out & 15) || (p.lin.hi * 8) % 16) return false;
    return knobs().fft_longrow != 0 && !g_fft_tma_disabled();
}

// =====================================================================================
// 16384-long rows as a 32 x 32 x 16 four-step inside one 512-thread CTA (one line at a time,
// one CTA per SM), 32 elements per thread:
//   A  thread t < 512: length-32 DFT of x[t + 512 m] (loaded straight from global memory: each
//      warp load is 256 contiguous bytes; the next line was prefetched into L2 by one bulk
//      prefetch), times W_16384^{t k1} -> E1[k1][t] (pitch 513: conflict-free both ways);
//   B  thread (k1 = lane, t1 = warp): length-32 DFT over t2 of y[t1 + 16 t2][k1], times
//      W_512^{t1 k2b} -> E2[k2b][t1][k1];
//   C  thread (k1 = lane, warp w): for k2b in {2w, 2w+1} the length-16 DFT over t1 ->
//      X[k1 + 32 k2b + 1024 k2c], stored as 256-byte warp segments.
// Two shared-memory exchanges and three barriers per line, against four stages / three
// exchanges and a half-line staging scheme in fft_longrow_kernel.
// =====================================================================================
// v[r] *= W^r (r = 1..31) from the bases b[i] = W^{2^i} (i < 5) with few live registers:
// W^r = W^{4a} W^{b}, r = 4a + b, from the 3 low and 7 high powers (10 values, 5 products).
__device__ __forceinline__ void apply_pow32(float2* v, const float2* b) {
    float2 lo[4], hi[8];
    lo[1] = b[0];
    lo[2] = b[1];
    lo[3] = cmul(b[0], b[1]);
    hi[1] = b[2];
    hi[2] = b[3];
    hi[3] = cmul(b[2], b[3]);
    hi[4] = b[4];
    hi[5] = cmul(b[2], b[4]);
    hi[6] = cmul(b[3], b[4]);
    hi[7] = cmul(hi[3], b[4]);
#pragma unroll
    for (int r = 1; r < 32; ++r) {
        const int a = r >> 2, bb = r & 3;
        const float2 w = (a == 0) ? lo[bb] : (bb == 0) ? hi[a] : cmul(hi[a], lo[bb]);
        v[r] = cmul(v[r], w);
    }
}

constexpr int kL14Threads = 512;
constexpr int kL14P1 = 513;
constexpr int kL14Half = 8192;  // first half of the next line, staged by one bulk copy (3/4: 2451 vs 2437 us)
constexpr size_t kL14Smem = (size_t)(32 * kL14P1 + kL14Half) * sizeof(float2) + 64;

template <bool OUT_GENERIC>
__global__ void __launch_bounds__(kL14Threads, 1)
    fft_row16384_kernel(const FftPass p, const float2* __restrict__ tw) {
    extern __shared__ __align__(128) float2 smf[];
    float2* E = smf;
    float2* S = smf + 32 * kL14P1;  // 16-byte aligned: 32 * 513 * 8 is a multiple of 16
    uint64_t* bar = reinterpret_cast<uint64_t*>(S + kL14Half);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) {
        ptx::mbar_init(ptx::smem_u32(bar), 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const int64_t nl = p.nlines;
    int64_t g = blockIdx.x;
    // the first kL14Half elements of each line arrive by a bulk copy into S issued one line
    // ahead; the rest is read straight from global memory (L2-prefetched)
    auto stage_first_half = [&](int64_t line) {
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(bar), kL14Half * sizeof(float2));
        ptx::bulk_load(ptx::smem_u32(S), p.in + line * p.lin.hi, kL14Half * sizeof(float2), ptx::smem_u32(bar));
    };
    if (tid == 0 && g < nl) {
        stage_first_half(g);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.in + g * p.lin.hi + kL14Half),
                     "r"((uint32_t)(16384 - kL14Half) * 8u)
                     : "memory");
    }
    int it = 0;
    for (; g < nl; g += gridDim.x, ++it) {
        const int64_t gn = g + gridDim.x;
        if (tid == 0 && gn < nl)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.in + gn * p.lin.hi), "r"(16384u * 8u)
                         : "memory");
        float2 v[32];
        {
            const float2* src = p.in + g * p.lin.hi + tid;
#pragma unroll
            for (int m = kL14Half / 512; m < 32; ++m) v[m] = __ldcs(src + 512 * m);
        }
        ptx::mbar_wait(ptx::smem_u32(bar), (uint32_t)it & 1u);
#pragma unroll
        for (int m = 0; m < kL14Half / 512; ++m) v[m] = S[tid + 512 * m];
        ptx::fence_proxy_async_smem();  // generic reads of S before its bulk refill
        __syncthreads();
        if (tid == 0 && gn < nl) stage_first_half(gn);
        if (p.conj_in) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m].y = -v[m].y;
        }
        // ---- A
        dft<32>(v);
        {
            float2 bA[5];  // W_16384^{tid 2^i} (reloaded per line: L1 hits, fewer live registers)
#pragma unroll
            for (int i = 0; i < 5; ++i) bA[i] = __ldg(tw + ((tid << i) & (kTwN - 1)));
            apply_pow32(v, bA);
        }
        __syncthreads();  // the previous line's stage C has read E
#pragma unroll
        for (int k = 0; k < 32; ++k) E[k * kL14P1 + tid] = v[k];
        __syncthreads();
        // ---- B: (k1 = lane, t1 = w), values over t2
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = E[lane * kL14P1 + w + 16 * m];
        dft<32>(v);
        {
            float2 bB[5];  // W_512^{w 2^i}
#pragma unroll
            for (int i = 0; i < 5; ++i) bB[i] = __ldg(tw + (((w << i) << 5) & (kTwN - 1)));
            apply_pow32(v, bB);
        }
        __syncthreads();  // every thread has read E1
#pragma unroll
        for (int k = 0; k < 32; ++k) E[(k * 16 + w) * 32 + lane] = v[k];  // E2[k2b][t1][k1]
        __syncthreads();
        // ---- C: k2b in {2w, 2w + 1}, length-16 DFT over t1
        float2* dst = p.out + g * p.lout.hi;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k2b = 2 * w + h;
            float2 u[16];
#pragma unroll
            for (int t1 = 0; t1 < 16; ++t1) u[t1] = E[(k2b * 16 + t1) * 32 + lane];
            dft<16>(u);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                float2 o = u[c];
                if (p.conj_out) o.y = -o.y;
                if (p.scale != 1.0f) o = __fmul2_rn(o, bc2(p.scale));
                const int k = lane + 32 * k2b + 1024 * c;
                if constexpr (!OUT_GENERIC) {
                    dst[k] = o;
                } else {  // per-peer column blocks (the slab transpose), as fft_longrow_kernel
                    const int out_kmask = (1 << p.lout.kb_shift) - 1;
                    if (p.peer_out)
                        p.peer[k >> p.lout.kb_shift][g * p.lout.hi + (int64_t)(k & out_kmask) * p.lout.es] = o;
                    else
                        dst[(int64_t)(k & out_kmask) * p.lout.es + (int64_t)(k >> p.lout.kb_shift) * p.lout.bs] = o;
                }
            }
        }
    }
}

template <bool OG>
static fb_status launch_row16384(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    static DevOnce once;
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(fft_row16384_kernel<OG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kL14Smem));
        once.set(dev);
    }
    int64_t grid = st->sm_count;
    if (grid > p.nlines) grid = p.nlines;
    return launch_pdl(fft_row16384_kernel<OG>, dim3((unsigned)grid), dim3(kL14Threads), kL14Smem, s, p,
                      (const float2*)st->twiddles);
}

// -------------------------------------------------------------------------------------
// The same 32 x 32 x 16 four-step with each line split over a CTA PAIR (cluster of 2,
// 256 threads each), so that two or three half-line CTAs of different lines share an SM and
// their load / exchange / store phases interleave (one 512-thread CTA per SM holding a whole
// 128 KiB line cannot overlap them).  CTA r:
//   A  thread j: t = 256 r + j, the length-32 DFT over m of x[t + 512 m], times
//      W_16384^{t k1}; y[t][k1] goes to the CTA owning k1 (k1 >> 4): E1[k1 & 15][t] (pitch
//      513), half of it through distributed shared memory;
//   B  thread (k1l = j & 15, t1 = j >> 4), k1 = 16 r + k1l: the length-32 DFT over t2 of
//      E1[k1l][t1 + 16 t2], times W_512^{t1 k2b} -> E2[k2b][t1][k1l] (aliases E1);
//   C  thread (k1l, k2b in {2 (j >> 4), 2 (j >> 4) + 1}): the length-16 DFT over t1 ->
//      X[k1 + 32 k2b + 1024 c].
// Per element the operations are those of fft_row16384_kernel, so the results are bitwise
// equal.  Two cluster barriers per line: after the remote writes (release / acquire), and a
// split one whose arrive follows stage C's reads of E2 and whose wait precedes the next line's
// remote writes, so the peer's reads of the previous line overlap this CTA's loads and stage A.
constexpr int kL14cThreads = 256;
constexpr int kL14cP1 = 513;
constexpr size_t kL14cSmem = (size_t)16 * kL14cP1 * sizeof(float2) + 16;

template <bool OUT_GENERIC, int CPS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kL14cThreads, CPS)
    fft_row16384c_kernel(const FftPass p, const float2* __restrict__ tw) {
    extern __shared__ __align__(128) float2 smf[];
    float2* E = smf;
    const int j = threadIdx.x;
    const uint32_t r = ptx::cluster_ctarank();
    const uint32_t e_loc = ptx::smem_u32(E);
    const uint32_t e_peer = ptx::mapa_shared(e_loc, r ^ 1u);
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    const int64_t nl = p.nlines;
    const int64_t ncl = gridDim.x >> 1;
    const int t = 256 * (int)r + j;
    ptx::cluster_arrive_release();  // "E free" for the first line
    for (int64_t g = blockIdx.x >> 1; g < nl; g += ncl) {
        const int64_t gn = g + ncl;
        if (j == 0 && gn < nl)  // this CTA's half of the next line into L2
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.in + gn * p.lin.hi + 8192 * r),
                         "r"(8192u * 8u)
                         : "memory");
        float2 v[32];
        {
            const float2* src = p.in + g * p.lin.hi + t;
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = __ldcs(src + 512 * m);
        }
        if (p.conj_in) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m].y = -v[m].y;
        }
        // ---- A
        dft<32>(v);
        {
            float2 bA[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) bA[i] = __ldg(tw + ((t << i) & (kTwN - 1)));
            apply_pow32(v, bA);
        }
        ptx::cluster_wait_acquire();  // both CTAs finished reading E (previous line's stage C)
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t off = (uint32_t)(((k & 15) * kL14cP1 + t) * 8);
            if ((uint32_t)(k >> 4) == r)
                E[(k & 15) * kL14cP1 + t] = v[k];
            else
                ptx::st_cluster_f2(e_peer + off, v[k]);
        }
        ptx::cluster_arrive_release();
        ptx::cluster_wait_acquire();  // E1 complete in both CTAs
        // ---- B: (k1l, t1), values over t2
        const int k1l = j & 15, t1 = j >> 4;
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = E[k1l * kL14cP1 + t1 + 16 * m];
        dft<32>(v);
        {
            float2 bB[5];  // W_512^{t1 2^i}
#pragma unroll
            for (int i = 0; i < 5; ++i) bB[i] = __ldg(tw + (((t1 << i) << 5) & (kTwN - 1)));
            apply_pow32(v, bB);
        }
        __syncthreads();  // every thread has read E1
#pragma unroll
        for (int k = 0; k < 32; ++k) E[(k * 16 + t1) * 16 + k1l] = v[k];  // E2[k2b][t1][k1l]
        __syncthreads();
        // ---- C: k2b in {2 (j >> 4), 2 (j >> 4) + 1}, length-16 DFT over t1
        float2* dst = p.out + g * p.lout.hi;
        const int k1 = 16 * (int)r + k1l;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int k2b = 2 * (j >> 4) + h;
            float2 u[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) u[q] = E[(k2b * 16 + q) * 16 + k1l];
            dft<16>(u);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                float2 o = u[c];
                if (p.conj_out) o.y = -o.y;
                if (p.scale != 1.0f) o = __fmul2_rn(o, bc2(p.scale));
                const int k = k1 + 32 * k2b + 1024 * c;
                if constexpr (!OUT_GENERIC) {
                    dst[k] = o;
                } else {
                    const int out_kmask = (1 << p.lout.kb_shift) - 1;
                    if (p.peer_out)
                        p.peer[k >> p.lout.kb_shift][g * p.lout.hi + (int64_t)(k & out_kmask) * p.lout.es] = o;
                    else
                        dst[(int64_t)(k & out_kmask) * p.lout.es + (int64_t)(k >> p.lout.kb_shift) * p.lout.bs] = o;
                }
            }
        }
        ptx::cluster_arrive_release();  // this CTA is done reading E for this line
    }
    ptx::cluster_wait_acquire();  // no peer writes into E after this CTA exits
}

template <bool OG, int CPS>
static fb_status launch_row16384c_cps(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    static DevOnce once;
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(fft_row16384c_kernel<OG, CPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kL14cSmem));
        once.set(dev);
    }
    int64_t clusters = (int64_t)st->sm_count * CPS / 2;
    if (clusters > p.nlines) clusters = p.nlines;
    return launch_pdl(fft_row16384c_kernel<OG, CPS>, dim3((unsigned)(2 * clusters)), dim3(kL14cThreads), kL14cSmem,
                      s, p, (const float2*)st->twiddles);
}
// CTAs per SM (knob FB_FFT_ROW16K_CPS): 2 (128 registers) or 3 (85 registers)
template <bool OG>
static fb_status launch_row16384c(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    return knobs().fft_row16k_cps == 3 ? launch_row16384c_cps<OG, 3>(p, st, s) : launch_row16384c_cps<OG, 2>(p, st, s);
}

template <bool OG>
static fb_status launch_longrow(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    using G = LineGeom<14>;
    constexpr size_t SMEM = (size_t)(G::PADL + G::L / 2) * sizeof(float2) + 64;
    static DevOnce once;
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(fft_longrow_kernel<OG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
        once.set(dev);
    }
    int64_t grid = st->sm_count;
    if (grid > p.nlines) grid = p.nlines;
    return launch_pdl(fft_longrow_kernel<OG>, dim3((unsigned)grid), dim3(1024), SMEM, s, p,
                      (const float2*)st->twiddles, (const float2*)st->stage_tw);
}

// =====================================================================================
// Column pass of 1024-long lines with 32 elements per thread (radix 32 x 32, one exchange).
// 1024 = 32 x 32 four-step inside the CTA: thread (w, l) of a 4-column group (C = 4, 128
// threads) owns column c = l & 3 and residue t = 8 w + (l >> 2); stage 1 is the length-32 DFT
// of x[t + 32 m] (m < 32) in registers, then y[t][k1] *= W_1024^{t k1}; one shared-memory
// transpose later the same thread owns (c, k1 = t) and runs the length-32 DFT over t, which
// yields X[k1 + 32 k2].  Compared with the radix-16 pass (16 x 16 x 4: two exchanges, three
// stages) it moves each element through shared memory once instead of twice and has one
// barrier per exchange less.  All shared-memory patterns are conflict-free: the staging read
// S[(t + 32 m) 4 + c] and the output staging [k][c] are contiguous per warp, and the exchange
// E[c][k1][t] uses a 33-element row pitch and a 1060-element column pitch.
// =====================================================================================
constexpr int kC32Cols = 4, kC32Threads = 128;
constexpr int kC32EPitch = 32 * 33 + 4;  // float2 per column in the exchange buffer
constexpr int kC32S = kC32Cols * 1024;  // staging (float2)
constexpr int kC32E = kC32Cols * kC32EPitch;
constexpr size_t kC32Smem = (size_t)(kC32S + kC32E) * sizeof(float2) + 64;

// W_1024^{t k} for k = 1..31 from the bases W_1024^{t 2^i} (i < 5; master table, resolution 2^14)
__device__ __forceinline__ void c32_twiddles(float2* full, int t, const float2* __restrict__ tw) {
    float2 b[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) b[i] = __ldg(tw + (((t << i) << 4) & (kTwN - 1)));
    pow_expand<32>(full, b);
}

template <int UNUSED = 0>  // a template so that every translation unit may include the definition
__global__ void __launch_bounds__(kC32Threads, 3)
    fft_col1024_kernel(const FftPass p, const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
                       const float2* __restrict__ tw, int64_t ngroups) {
    constexpr int C = kC32Cols, L = 1024, BOX = 256;
    extern __shared__ __align__(128) float2 smf[];
    float2* S = smf;
    float2* E = smf + kC32S;  // exchange, then the output staging [k][c] (4096 float2)
    uint64_t* bar = reinterpret_cast<uint64_t*>(E + kC32E);
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    const int c = l & 3, t = 8 * w + (l >> 2);
    const int gshift = p.g_shift >= 62 ? 62 : p.g_shift;
    const int64_t gmask = (gshift >= 62) ? -1 : ((int64_t(1) << gshift) - 1);
    if (tid == 0) {
        ptx::mbar_init(ptx::smem_u32(bar), 1);
        ptx::fence_mbar_init();
        ptx::tma_prefetch_desc(&tin);
        ptx::tma_prefetch_desc(&tout);
    }
    __syncthreads();
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    auto issue = [&](int64_t grp) {
        const uint32_t b = ptx::smem_u32(bar);
        ptx::mbar_arrive_expect_tx(b, (uint32_t)(C * L * sizeof(float2)));
        const int64_t g0 = grp * C;
        const int64_t gh = (gshift >= 62) ? 0 : (g0 >> gshift);
        const int gl = (int)(g0 & gmask);
#pragma unroll 1
        for (int kb = 0; kb < L; kb += BOX) ptx::tma_load_3d(ptx::smem_u32(S + kb * C), &tin, b, gl, kb, (int)gh);
    };
    if (tid == 0) {
        if (p.stagger_ns > 0 && p.sm_count > 0) {
            const int slot = (int)(blockIdx.x / (unsigned)p.sm_count);
            for (int i = 0; i < slot; ++i) __nanosleep((unsigned)p.stagger_ns);
        }
        if ((int64_t)blockIdx.x < ngroups) issue(blockIdx.x);
    }
    // this thread's four-step twiddles W_1024^{t k1}, fixed for every group
    float2 twf[31];
    c32_twiddles(twf, t, tw);
    int it = 0;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++it) {
        ptx::mbar_wait(ptx::smem_u32(bar), (uint32_t)it & 1u);
        float2 v[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = S[(t + 32 * m) * C + c];
        if (p.conj_in) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m].y = -v[m].y;
        }
        ptx::fence_proxy_async_smem();          // generic reads of S before its TMA refill
        if (tid == 0) ptx::bulk_wait_read0();   // the previous group's TMA store has read E
        __syncthreads();
        if (tid == 0 && grp + gridDim.x < ngroups) issue(grp + gridDim.x);
        // stage 1: length-32 DFT over m, then the four-step twiddle
        dft<32>(v);
#pragma unroll
        for (int k = 1; k < 32; ++k) v[k] = cmul(v[k], twf[k - 1]);
        // transpose: E[c][k1][t]
        float2* ew = E + c * kC32EPitch + t;
#pragma unroll
        for (int k = 0; k < 32; ++k) ew[k * 33] = v[k];
        __syncthreads();
        // stage 2: this thread owns (c, k1 = t): length-32 DFT over the residues t'
        const float2* er = E + c * kC32EPitch + t * 33;
#pragma unroll
        for (int m = 0; m < 32; ++m) v[m] = er[m];
        dft<32>(v);
        if (p.conj_out) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m].y = -v[m].y;
        }
        if (p.scale != 1.0f) {
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = __fmul2_rn(v[m], bc2(p.scale));
        }
        __syncthreads();  // every thread has read its exchange row: E becomes the output staging
        // X[k1 + 32 k2] -> staging [k][c]
#pragma unroll
        for (int m = 0; m < 32; ++m) E[(t + 32 * m) * C + c] = v[m];
        ptx::fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            const int64_t g0 = grp * C;
            const int64_t gh0 = (gshift >= 62) ? 0 : (g0 >> gshift);
            const int gl0 = (int)(g0 & gmask);
#pragma unroll 1
            for (int kb = 0; kb < L; kb += BOX) ptx::tma_store_3d(&tout, ptx::smem_u32(E + kb * C), gl0, kb, (int)gh0);
            ptx::bulk_commit();
        }
    }
    if (tid == 0) ptx::bulk_wait0();
}

static fb_status launch_col1024(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    static DevOnce once;
    static std::atomic<int> occ[32];
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(fft_col1024_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kC32Smem));
        int nb = 0;
        FB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fft_col1024_kernel<0>, kC32Threads, kC32Smem));
        occ[dev].store(nb < 1 ? 1 : nb);
        once.set(dev);
    }
    const int64_t ngroups = (p.nlines + kC32Cols - 1) / kC32Cols;
    int64_t grid = (int64_t)st->sm_count * occ[dev].load();
    if (grid > ngroups) grid = ngroups;
    const int gshift = p.g_shift >= 62 ? 62 : p.g_shift;
    const int64_t glo = (gshift >= 62) ? p.nlines : (int64_t(1) << gshift);
    const int64_t nh = (p.nlines + glo - 1) / glo;
    CUtensorMap tin, tout;
    if (!make_col_map(&tin, p.in, glo, 1024, nh, p.lin.es, p.lin.hi, kC32Cols) ||
        !make_col_map(&tout, p.out, glo, 1024, nh, p.lout.es, p.lout.hi, kC32Cols)) {
        set_error("cuTensorMapEncodeTiled failed for the radix-32 column pass");
        return FB_ERR_CUDA;
    }
    FftPass pk = p;
    if (knobs().fft_stagger_col >= 0) pk.stagger_ns = knobs().fft_stagger_col;  // A/B knob
    return launch_pdl(fft_col1024_kernel<0>, dim3((unsigned)grid), dim3(kC32Threads), kC32Smem, s, pk, tin, tout,
                      (const float2*)st->twiddles, ngroups);
}

// All launches of one line length (explicitly instantiated per length in fb_fft_k*.cu so the
// kernel variants compile in parallel translation units).
template <int LOG2L>
fb_status launch_pass_L(const FftPass& p, const DeviceState* st, cudaStream_t s) {
    int kind = 0, tc = 0;
    bool og = false;
    constexpr bool has_tma = LOG2L >= 6 && LOG2L <= 12;
    if (p.pair_log2N > 0) {
        // pair-plan row pass: lane pairs c = 0, 1 hold rows q, q + n0/2.  TMA kernel when the
        // pass is expressible (A/B at 2048^2: 22 us vs 28 us for the plain kernel with C = 2);
        // FB_FFT_PAIR_TMA=0 forces the plain kernel.
        if constexpr (has_tma) {
            if (knobs().fft_pair_tma && !g_fft_tma_disabled() && tma_eligible(p, kind, tc, og) && tc == 2 &&
                !og)
                return launch_tma_L<LOG2L>(p, kind, tc, og, st, s);
        }
        const int pc = pick_C(LOG2L, false);
        if constexpr (LOG2L >= 6 && LOG2L <= 12) return launch_L<LOG2L>(p, pc < 2 ? 2 : pc, st, s);
        set_error("internal: pair-plan row length 2^%d", LOG2L);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    if constexpr (has_tma) {
        if (!g_fft_tma_disabled() && tma_eligible(p, kind, tc, og)) {
            if constexpr (LOG2L == 10) {
                // 1024-long column lines in 4-column groups: the radix-32 one-exchange pass
                // (knob FB_FFT_COL32=0: the radix-16 persistent pass)
                if (kind == KIND_COL && tc == 4 && p.tw4_log2N == 0 && p.pair_log2N == 0 && knobs().fft_col32 &&
                    !(p.col_stg > 0))
                    return launch_col1024(p, st, s);
            }
            return launch_tma_L<LOG2L>(p, kind, tc, og, st, s);
        }
    }
    if constexpr (LOG2L == 14) {
        if (longrow_eligible(p)) {
            // the 32 x 32 x 16 four-step kernel, plain or per-peer outputs (knob FB_FFT_ROW16K=0:
            // the radix-16 half-line-streaming kernel)
            if (knobs().fft_row16k == 2)  // each line over a CTA pair (DSMEM exchange)
                return p.lout.kb_shift >= 14 && !p.peer_out ? launch_row16384c<false>(p, st, s)
                                                            : launch_row16384c<true>(p, st, s);
            if (knobs().fft_row16k)
                return p.lout.kb_shift >= 14 && !p.peer_out ? launch_row16384<false>(p, st, s)
                                                            : launch_row16384<true>(p, st, s);
            return p.lout.kb_shift >= 14 && !p.peer_out ? launch_longrow<false>(p, st, s) : launch_longrow<true>(p, st, s);
        }
    }
    return launch_L<LOG2L>(p, pick_C(LOG2L, p.col_like != 0), st, s);
}

#define FB_FFT_EXTERN_L(L) extern template fb_status launch_pass_L<L>(const FftPass&, const DeviceState*, cudaStream_t);
#define FB_FFT_INSTANTIATE_L(L) template fb_status launch_pass_L<L>(const FftPass&, const DeviceState*, cudaStream_t);

}  // namespace fb
