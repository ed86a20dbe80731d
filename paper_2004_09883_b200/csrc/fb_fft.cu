// fb_fft.cu -- plans of the Fourier-transform function block:
// which passes (fb_fft_kern.cuh) a 2D transform, a column batch or a four-step split runs.
#include "fb_fft_kern.cuh"

namespace fb {

int64_t stage_tw_total() { return stage_tw_offset(kTwLog2 + 1, 0); }
// master-table index (W_16384^idx) of every stage-table entry, in table order
void stage_tw_index(int32_t* idx) {
    int64_t e = 0;
    for (int l = 0; l <= kTwLog2; ++l)
        for (int s = 1; s < stage_count(l); ++s) {
            const int R = stage_radix(l, s);
            const int64_t Ns = int64_t(1) << (4 * s);
            const int64_t step = kTwN / (Ns * R);
            for (int r = 0; r < R; ++r)
                for (int64_t jm = 0; jm < Ns; ++jm) idx[e++] = (int32_t)(jm * r * step);
        }
}

FB_FFT_EXTERN_L(0) FB_FFT_EXTERN_L(1) FB_FFT_EXTERN_L(2) FB_FFT_EXTERN_L(3) FB_FFT_EXTERN_L(4)
FB_FFT_EXTERN_L(5) FB_FFT_EXTERN_L(6) FB_FFT_EXTERN_L(7) FB_FFT_EXTERN_L(8) FB_FFT_EXTERN_L(9)
FB_FFT_EXTERN_L(10) FB_FFT_EXTERN_L(11) FB_FFT_EXTERN_L(12) FB_FFT_EXTERN_L(13) FB_FFT_EXTERN_L(14)

unsigned long long* g_fft_trace_host = nullptr;

fb_status launch_fft_pass(const FftPass& p_in, const DeviceState* st, cudaStream_t s) {
    if (p_in.nlines <= 0) return FB_OK;
    FftPass p = p_in;
    p.trace = FB_FFT_TRACE ? g_fft_trace_host : nullptr;
    const Knobs& kn = knobs();
    p.debug = kn.fft_debug;  // 0 unless built with FB_DEBUG_BUILD
    p.stagger_ns = kn.fft_stagger_ns;
    p.sm_count = st->sm_count;
    p.col_stg = kn.fft_col_stg;
    p.pair_half_shfl = kn.fft_pair2;
    p.col_pair_last = kn.fft_colpair;
    switch (p.log2L) {
        case 0: return launch_pass_L<0>(p, st, s);
        case 1: return launch_pass_L<1>(p, st, s);
        case 2: return launch_pass_L<2>(p, st, s);
        case 3: return launch_pass_L<3>(p, st, s);
        case 4: return launch_pass_L<4>(p, st, s);
        case 5: return launch_pass_L<5>(p, st, s);
        case 6: return launch_pass_L<6>(p, st, s);
        case 7: return launch_pass_L<7>(p, st, s);
        case 8: return launch_pass_L<8>(p, st, s);
        case 9: return launch_pass_L<9>(p, st, s);
        case 10: return launch_pass_L<10>(p, st, s);
        case 11: return launch_pass_L<11>(p, st, s);
        case 12: return launch_pass_L<12>(p, st, s);
        case 13: return launch_pass_L<13>(p, st, s);
        case 14: return launch_pass_L<14>(p, st, s);
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

// column lines up to 2^12 in one pass (knob FB_FFT_COL_MAX_LOG2 for A/B; longer ones use the
// four-step split)
static int max_onchip_col() { return knobs().fft_col_max_log2; }

fb_status fft_columns(const float2* in, float2* out, int64_t n0, int64_t ncols, int64_t ld_in,
                      int64_t ld_out, bool conj_in, bool conj_out, float scale, float2* tmp,
                      const DeviceState* st, cudaStream_t s) {
    const int l0 = ilog2(n0);
    const int lc = ilog2(ncols);
    if (l0 <= max_onchip_col()) {
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
    // the four-step line numbering (g = n2 * ncols + c) needs a power-of-two column count:
    // other counts run as power-of-two column blocks
    if (!is_pow2(ncols)) {
        int64_t c0 = 0;
        for (int bit = 62; bit >= 0; --bit) {
            const int64_t w = int64_t(1) << bit;
            if (!(ncols & w)) continue;
            FB_TRY(fft_columns(in + c0, out + c0, n0, w, ld_in, ld_out, conj_in, conj_out, scale, tmp, st, s));
            c0 += w;
        }
        return FB_OK;
    }
    // Four-step split of the column length n0 = a * b (b = 128 contiguous sub-line rows):
    //   step 1: for each n2 < b: length-a FFTs over rows b*n1 + n2, times W_n0^{n2 k1}
    //           (tmp rows b*k1 + n2)
    //   step 3: for each k1 < a: length-b FFTs over rows b*k1 + n2 -> out rows k1 + a*k2
    if (!tmp) {
        set_error("internal: four-step column FFT needs a workspace");
        return FB_ERR_WORKSPACE;
    }
    const int lb = knobs().fft_4step_lb > 0 ? knobs().fft_4step_lb : (l0 >= 14 ? 7 : (l0 + 1) / 2);
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

// "Pair" plan for 2^9 <= n0 <= 2^12 (knob FB_FFT_PAIR=0 disables): the column length splits as
// 2 x n0/2; the radix-2 step rides in the row pass (lane shuffle + twiddle), so the column
// pass works on n0/2-long lines with twice as wide TMA rows (A/B at 2048^2: 16-byte rows
// cost 22 us, 32-byte rows 16.5 us).  Needs an n0 x n1 workspace (out-of-place column pass).
static bool use_pair_plan(int64_t n0, int64_t n1) {
    const int l0 = ilog2(n0), l1 = ilog2(n1);
    return knobs().fft_pair != 0 && l0 >= 9 && l0 <= knobs().fft_pair_max_log2 &&
           l0 <= max_onchip_col() && l1 >= 6 && l1 <= 12;
}

size_t fft2d_ws_bytes(int64_t n0, int64_t n1) {
    if (!is_pow2(n0) || !is_pow2(n1)) return bluestein_ws_bytes(n0, n1);
    if (ilog2(n0) <= max_onchip_col() && !use_pair_plan(n0, n1)) return 0;
    return (size_t)n0 * (size_t)n1 * sizeof(float2);
}

fb_status fft2d_device(const void* x, void* y, int64_t n0, int64_t n1, bool inverse, void* ws,
                       size_t ws_bytes, const DeviceState* st, cudaStream_t s, bool unscaled) {
    if (!is_pow2(n0) || !is_pow2(n1)) return fft2d_bluestein(x, y, n0, n1, inverse, ws, ws_bytes, st, s, unscaled);
    const float scale = (inverse && !unscaled) ? 1.0f / (float)((double)n0 * (double)n1) : 1.0f;
    if (fft_small_eligible(n0, n1) && aligned16(x) && aligned16(y))
        return fft2d_small((const float2*)x, (float2*)y, inverse, scale, st, s);
    if (use_pair_plan(n0, n1) && aligned16(x) && aligned16(y) && aligned16(ws)) {
        if (ws_bytes < fft2d_ws_bytes(n0, n1)) {
            set_error("workspace too small");
            return FB_ERR_WORKSPACE;
        }
        const int64_t half = n0 / 2;
        float2* w = (float2*)ws;
        // pass 1: row FFTs of the pair (q, q + n0/2) + radix-2 across the pair + W_n0^{q k_a}
        FftPass p{};
        p.in = (const float2*)x;
        p.out = w;
        p.log2L = ilog2(n1);
        p.nlines = n0;
        p.g_shift = 1;  // g = 2q + c -> row q + c n0/2
        p.lin = plain_map(n1, half * n1, 1);
        p.lout = plain_map(n1, half * n1, 1);
        p.conj_in = inverse;
        p.scale = 1.f;
        p.col_like = 0;
        p.pair_log2N = ilog2(n0);
        p.trace_slot = 0;
        FB_TRY(launch_fft_pass(p, st, s));
        // pass 2: for k_a in {0, 1}: length-n0/2 column FFTs over rows n0/2 k_a + n_b,
        // output X[k_a + 2 k_b] at row k_a + 2 k_b
        const int lc = ilog2(n1);
        FftPass p3{};
        p3.in = w;
        p3.out = (float2*)y;
        p3.log2L = ilog2(half);
        p3.nlines = 2 * n1;
        p3.g_shift = lc;  // g = k_a * n1 + c
        p3.lin = plain_map(half * n1, 1, n1);
        p3.lout = plain_map(n1, 1, 2 * n1);
        p3.conj_out = inverse;
        p3.scale = scale;
        p3.col_like = 1;
        p3.trace_slot = 1;
        return launch_fft_pass(p3, st, s);
    }
    const bool four_step = ilog2(n0) > max_onchip_col();
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

#if FB_FFT_TRACE
extern "C" int fb_debug_fft_trace(void* buf) {  // trace builds only: device buffer or null
    fb::g_fft_trace_host = (unsigned long long*)buf;
    return 0;
}
#endif
