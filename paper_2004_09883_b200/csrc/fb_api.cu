// fb_api.cu -- the C ABI of libfb.so (include/fb.h): validation, per-device state, entry points.
#include <stdarg.h>
#include <string.h>

#include <mutex>

#include "fb_common.cuh"

namespace fb {

std::atomic<uint64_t> g_launches{0};
static thread_local char t_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_err, sizeof(t_err), fmt, ap);
    va_end(ap);
}
void clear_error() { t_err[0] = 0; }

// ---------------------------------------------------------------- knobs (fb_common.cuh)
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return (e && e[0]) ? atoi(e) : dflt;
}
static Knobs read_knobs() {
    Knobs k;
    k.fft_stagger_ns = env_int("FB_FFT_STAGGER", k.fft_stagger_ns);
    k.fft_col_stg = env_int("FB_FFT_COL_STG", k.fft_col_stg);
    k.fft_pair2 = env_int("FB_FFT_PAIR2", k.fft_pair2);
    k.fft_colpair = env_int("FB_FFT_COLPAIR", k.fft_colpair);
    k.fft_col_max_log2 = env_int("FB_FFT_COL_MAX_LOG2", k.fft_col_max_log2);
    k.fft_4step_lb = env_int("FB_FFT_4STEP_LB", k.fft_4step_lb);
    k.fft_pair = env_int("FB_FFT_PAIR", k.fft_pair);
    k.fft_pair_max_log2 = env_int("FB_FFT_PAIR_MAX_LOG2", k.fft_pair_max_log2);
    k.fft_no_tma_col = env_int("FB_FFT_NO_TMA_COL", k.fft_no_tma_col);
    k.fft_col_c = env_int("FB_FFT_COL_C", k.fft_col_c);
    k.fft_no_tma_row = env_int("FB_FFT_NO_TMA_ROW", k.fft_no_tma_row);
    k.fft_col_nb = env_int("FB_FFT_COL_NB", k.fft_col_nb);
    k.fft_row_nb = env_int("FB_FFT_ROW_NB", k.fft_row_nb);
    k.fft_no_tma = env_int("FB_FFT_NO_TMA", k.fft_no_tma);
    k.fft_longrow = env_int("FB_FFT_LONGROW", k.fft_longrow);
    k.fft_pair_tma = env_int("FB_FFT_PAIR_TMA", k.fft_pair_tma);
    k.fft_no_pdl = env_int("FB_FFT_NO_PDL", k.fft_no_pdl);
    k.fft_sub = env_int("FB_FFT_SUB", k.fft_sub);
    k.fft_sub_ilv = env_int("FB_FFT_SUB_ILV", k.fft_sub_ilv);
    k.fft_col32 = env_int("FB_FFT_COL32", k.fft_col32);
    k.fft_row16k = env_int("FB_FFT_ROW16K", k.fft_row16k);
    k.fft_row16k_cps = env_int("FB_FFT_ROW16K_CPS", k.fft_row16k_cps);
    k.fft_small = env_int("FB_FFT_SMALL", k.fft_small);
    k.fft_stagger_col = env_int("FB_FFT_STAGGER_COL", k.fft_stagger_col);
    k.fft_mixed = env_int("FB_FFT_MIXED", k.fft_mixed);
    k.fft_mr_small = env_int("FB_FFT_MR_SMALL", k.fft_mr_small);
    k.slab_fused = env_int("FB_SLAB_FUSED", k.slab_fused);
    const char* pk = getenv("FB_ROWBLOCK_PANEL");
    if (pk && pk[0]) k.rowblock_panel = atoll(pk);
    k.f64_cfg = env_int("FB_F64_CFG", k.f64_cfg);
    k.gemm_split2 = env_int("FB_GEMM_SPLIT2", k.gemm_split2);
    k.gemm_splitv = env_int("FB_GEMM_SPLITV", k.gemm_splitv);
    k.gemm_split_pdl = env_int("FB_GEMM_SPLIT_PDL", k.gemm_split_pdl);
    k.gemm_1cta = env_int("FB_GEMM_1CTA", k.gemm_1cta);
    k.gemm_persist = env_int("FB_GEMM_PERSIST", k.gemm_persist);
    k.bf16_persist = env_int("FB_BF16_PERSIST", k.bf16_persist);
    k.gemm_npanel = env_int("FB_GEMM_NPANEL", k.gemm_npanel);
    k.gemm_nt = env_int("FB_GEMM_NT", k.gemm_nt);
    k.gemm_ahi_raw = env_int("FB_GEMM_AHI_RAW", k.gemm_ahi_raw);
    k.gemm_raster_panel = env_int("FB_GEMM_RASTER_PANEL", k.gemm_raster_panel);
    k.gemm_fused = env_int("FB_GEMM_FUSED", k.gemm_fused);
    k.gemm_lo_prepass = env_int("FB_GEMM_LO_PREPASS", k.gemm_lo_prepass);
    k.gemm_streamk = env_int("FB_GEMM_STREAMK", k.gemm_streamk);
    k.gemm_lo_overlap = env_int("FB_GEMM_LO_OVERLAP", k.gemm_lo_overlap);

    k.bf16_cluster = env_int("FB_BF16_CLUSTER", k.bf16_cluster);
    k.lu_tma = env_int("FB_LU_TMA", k.lu_tma);
    k.lu_rank_simt = env_int("FB_LU_RANK_SIMT", k.lu_rank_simt);
    k.lu_serial = env_int("FB_LU_SERIAL", k.lu_serial);
    k.lu_lookahead = env_int("FB_LU_LOOKAHEAD", k.lu_lookahead);
    k.lu_graph = env_int("FB_LU_GRAPH", k.lu_graph);
#if FB_DEBUG_BUILD
    k.fft_debug = env_int("FB_FFT_DEBUG", 0);
    k.lu_debug = env_int("FB_LU_DEBUG", 0);
#endif
    return k;
}
static std::atomic<const Knobs*> g_knobs{nullptr};
static std::mutex g_knobs_mu;
void reload_knobs() {
    std::lock_guard<std::mutex> lk(g_knobs_mu);
    g_knobs.store(new Knobs(read_knobs()));  // the previous snapshot is kept alive (tiny, rare)
}
const Knobs& knobs() {
    const Knobs* k = g_knobs.load();
    if (!k) {
        std::lock_guard<std::mutex> lk(g_knobs_mu);
        if (!g_knobs.load()) g_knobs.store(new Knobs(read_knobs()));
        k = g_knobs.load();
    }
    return *k;
}

static constexpr int kMaxDev = 64;
static DeviceState g_dev[kMaxDev];
static std::mutex g_dev_mu;

// W[j] = exp(-2 pi i j / 16384): FP64 sincospi of the exact rational 2j/16384, RN to FP32.
// sincospi is exact at multiples of 1/2, so +-1 and 0 are exact.
__global__ void build_twiddles_kernel(float2* w) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < kTwN) {
        double s, c;
        sincospi((double)(2 * j) / (double)kTwN, &s, &c);
        w[j] = make_float2((float)c, (float)(-s));
    }
}

// Stage tables: entry e = master[idx[e]] (same FP32 values as the master table).
__global__ void gather_twiddles_kernel(const float2* __restrict__ w, const int32_t* __restrict__ idx,
                                       float2* __restrict__ out, int64_t n) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) out[e] = w[idx[e]];
}

static fb_status init_device_locked(int dev) {
    DeviceState& st = g_dev[dev];
    if (st.ready) return FB_OK;
    cudaDeviceProp prop;
    FB_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10 || prop.minor != 0) {
        set_error("device %d is sm_%d%d; libfb is built for sm_100a only", dev, prop.major, prop.minor);
        return FB_ERR_ARCH;
    }
    int cur = 0;
    FB_CUDA_TRY(cudaGetDevice(&cur));
    FB_CUDA_TRY(cudaSetDevice(dev));
    fb_status rc = FB_OK;
    float2* tw = nullptr;
    float2* stw = nullptr;
    int32_t* didx = nullptr;
    const int64_t nst = stage_tw_total();
    int32_t* hidx = new int32_t[nst];
    stage_tw_index(hidx);
    cudaError_t e = cudaMalloc(&tw, sizeof(float2) * kTwN);
    if (e == cudaSuccess) e = cudaMalloc(&stw, sizeof(float2) * nst);
    if (e == cudaSuccess) e = cudaMalloc(&didx, sizeof(int32_t) * nst);
    if (e == cudaSuccess) e = cudaMemcpy(didx, hidx, sizeof(int32_t) * nst, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        build_twiddles_kernel<<<kTwN / 256, 256>>>(tw);
        gather_twiddles_kernel<<<(unsigned)((nst + 255) / 256), 256>>>(tw, didx, stw, nst);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    delete[] hidx;
    if (didx) cudaFree(didx);
    if (e != cudaSuccess) {
        set_error("fb_init(%d): %s", dev, cudaGetErrorString(e));
        rc = FB_ERR_CUDA;
    } else {
        st.twiddles = tw;
        st.stage_tw = stw;
        if (cudaStreamCreateWithFlags(&st.aux, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&st.ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&st.ev_join, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&st.ev_h2d[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&st.ev_h2d[1], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&st.ev_d2h[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&st.ev_d2h[1], cudaEventDisableTiming) != cudaSuccess) {
            set_error("fb_init(%d): stream/event creation failed", dev);
            cudaSetDevice(cur);
            return FB_ERR_CUDA;
        }
        st.sm_count = prop.multiProcessorCount;
        st.ready = true;
    }
    cudaSetDevice(cur);
    return rc;
}

fb_status ensure_device(int* dev_out, DeviceState** st_out) {
    int dev = 0;
    FB_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDev) {
        set_error("device ordinal %d out of range", dev);
        return FB_ERR_INVALID_VALUE;
    }
    if (!g_dev[dev].ready) {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        FB_TRY(init_device_locked(dev));
    }
    if (dev_out) *dev_out = dev;
    *st_out = &g_dev[dev];
    return FB_OK;
}

static fb_status check_fft_dims(int64_t n0, int64_t n1) {
    if (n0 <= 0 || n1 <= 0) {
        set_error("n0=%lld n1=%lld must be >= 1", (long long)n0, (long long)n1);
        return FB_ERR_INVALID_VALUE;
    }
    if (!fft_size_ok(n0) || !fft_size_ok(n1)) {
        set_error("FFT sizes must be powers of two in [1, %d] or other lengths in [1, 8192] (got %lld x %lld)",
                  kTwN, (long long)n0, (long long)n1);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    return FB_OK;
}

static fb_status fft_entry(const void* x, void* y, int64_t n0, int64_t n1, void* ws,
                           size_t ws_bytes, void* stream, bool inverse) {
    clear_error();
    FB_TRY(check_fft_dims(n0, n1));
    if (!x || !y) {
        set_error("null x or y");
        return FB_ERR_INVALID_VALUE;
    }
    if (!aligned16(x) || !aligned16(y)) {
        set_error("x and y must be 16-byte aligned");
        return FB_ERR_MISALIGNED;
    }
    const size_t bytes = (size_t)n0 * (size_t)n1 * sizeof(float2);
    if (ranges_partially_overlap(x, bytes, y, bytes)) {
        set_error("x and y partially overlap (exact aliasing is allowed)");
        return FB_ERR_INVALID_VALUE;
    }
    const size_t need = fft2d_ws_bytes(n0, n1);
    if (need && (!ws || ws_bytes < need)) {
        set_error("workspace of %zu bytes required, got %zu", need, ws_bytes);
        return FB_ERR_WORKSPACE;
    }
    if (need && (ranges_overlap(ws, need, x, bytes) || ranges_overlap(ws, need, y, bytes))) {
        set_error("workspace overlaps x or y");
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    return fft2d_device(x, y, n0, n1, inverse, ws, ws_bytes, st, (cudaStream_t)stream);
}

}  // namespace fb

using namespace fb;

extern "C" {

int fb_version(void) { return 100; }

const char* fb_status_string(int s) {
    switch (s) {
        case FB_OK: return "FB_OK";
        case FB_ERR_INVALID_VALUE: return "FB_ERR_INVALID_VALUE";
        case FB_ERR_UNSUPPORTED_SIZE: return "FB_ERR_UNSUPPORTED_SIZE";
        case FB_ERR_MISALIGNED: return "FB_ERR_MISALIGNED";
        case FB_ERR_WORKSPACE: return "FB_ERR_WORKSPACE";
        case FB_ERR_NOT_INITIALIZED: return "FB_ERR_NOT_INITIALIZED";
        case FB_ERR_CUDA: return "FB_ERR_CUDA";
        case FB_ERR_NCCL: return "FB_ERR_NCCL";
        case FB_ERR_ARCH: return "FB_ERR_ARCH";
    }
    return "FB_ERR_UNKNOWN";
}

const char* fb_last_error_detail(void) { return t_err; }

uint64_t fb_launch_count(void) { return g_launches.load(); }

void fb_reload_knobs(void) { reload_knobs(); }

fb_status fb_init(int device) {
    clear_error();
    if (device < 0 || device >= kMaxDev) {
        set_error("device ordinal %d out of range", device);
        return FB_ERR_INVALID_VALUE;
    }
    int n = 0;
    FB_CUDA_TRY(cudaGetDeviceCount(&n));
    if (device >= n) {
        set_error("device %d does not exist (%d devices)", device, n);
        return FB_ERR_INVALID_VALUE;
    }
    std::lock_guard<std::mutex> lk(g_dev_mu);
    return init_device_locked(device);
}

size_t fb_fft2d_workspace_bytes(int64_t n0, int64_t n1) {
    if (check_fft_dims(n0, n1) != FB_OK) return 0;
    return fft2d_ws_bytes(n0, n1);
}

fb_status fb_fft2d(const void* x, void* y, int64_t n0, int64_t n1, void* ws, size_t ws_bytes,
                   void* stream) {
    return fft_entry(x, y, n0, n1, ws, ws_bytes, stream, false);
}

fb_status fb_ifft2d(const void* x, void* y, int64_t n0, int64_t n1, void* ws, size_t ws_bytes,
                    void* stream) {
    return fft_entry(x, y, n0, n1, ws, ws_bytes, stream, true);
}

static fb_status fft1d_entry(const void* x, void* y, int64_t n, int64_t batch, void* stream, bool inverse) {
    clear_error();
    if (batch < 1 || n < 1) {
        set_error("n and batch must be >= 1");
        return FB_ERR_INVALID_VALUE;
    }
    if (!is_pow2(n) || n > kTwN) {
        set_error("line length must be a power of two in [1, %d] (got %lld)", kTwN, (long long)n);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    if (!x || !y) {
        set_error("null x or y");
        return FB_ERR_INVALID_VALUE;
    }
    if (!aligned16(x) || !aligned16(y)) {
        set_error("x and y must be 16-byte aligned");
        return FB_ERR_MISALIGNED;
    }
    const size_t bytes = (size_t)n * (size_t)batch * sizeof(float2);
    if (ranges_partially_overlap(x, bytes, y, bytes)) {
        set_error("x and y partially overlap (exact aliasing is allowed)");
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    FftPass p{};
    p.in = (const float2*)x;
    p.out = (float2*)y;
    p.log2L = ilog2(n);
    p.nlines = batch;
    p.g_shift = 0;
    p.lin.hi = p.lout.hi = n;
    p.lin.lo = p.lout.lo = 0;
    p.lin.kb_shift = p.lout.kb_shift = 30;
    p.lin.es = p.lout.es = 1;
    p.lin.bs = p.lout.bs = 0;
    p.conj_in = inverse;
    p.conj_out = inverse;
    p.scale = inverse ? 1.0f / (float)n : 1.0f;
    return launch_fft_pass(p, st, (cudaStream_t)stream);
}

fb_status fb_fft1d_batched(const void* x, void* y, int64_t n, int64_t batch, void* stream) {
    return fft1d_entry(x, y, n, batch, stream, false);
}

fb_status fb_ifft1d_batched(const void* x, void* y, int64_t n, int64_t batch, void* stream) {
    return fft1d_entry(x, y, n, batch, stream, true);
}

size_t fb_matmul_workspace_bytes(int dtype, int64_t m, int64_t n, int64_t k) {
    if ((dtype != FB_F32 && dtype != FB_F64) || m <= 0 || n <= 0 || k <= 0) return 0;
    return gemm_ws_bytes(dtype, m, n, k);
}

fb_status fb_matmul(int dtype, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                    const void* B, int64_t ldb, void* C, int64_t ldc, void* ws, size_t ws_bytes,
                    void* stream) {
    clear_error();
    if (dtype != FB_F32 && dtype != FB_F64) {
        set_error("dtype must be FB_F32 or FB_F64");
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
    if (lda < k || ldb < n || ldc < n) {
        set_error("leading dimensions too small");
        return FB_ERR_INVALID_VALUE;
    }
    const int64_t es = dtype == FB_F32 ? 4 : 8;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C) || (lda * es) % 16 || (ldb * es) % 16 ||
        (ldc * es) % 16) {
        set_error("operands must be 16-byte aligned and ld*elemsize a multiple of 16");
        return FB_ERR_MISALIGNED;
    }
    const size_t cbytes = (size_t)((m - 1) * ldc + n) * es;
    if (ranges_overlap(C, cbytes, A, (size_t)((m - 1) * lda + k) * es) ||
        ranges_overlap(C, cbytes, B, (size_t)((k - 1) * ldb + n) * es)) {
        set_error("C overlaps A or B");
        return FB_ERR_INVALID_VALUE;
    }
    const size_t need = gemm_ws_bytes(dtype, m, n, k);
    if (need && (!ws || ws_bytes < need || !aligned16(ws))) {
        set_error("workspace of %zu bytes (16B aligned) required, got %zu", need, ws_bytes);
        return FB_ERR_WORKSPACE;
    }
    if (need && ranges_overlap(ws, need, C, cbytes)) {
        set_error("workspace overlaps C");
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    return gemm_device(dtype, m, n, k, A, lda, B, ldb, C, ldc, ws, ws_bytes, st,
                       (cudaStream_t)stream);
}

fb_status fb_tf32_split(int transpose, int64_t rows, int64_t cols, const float* X, int64_t ldx, float* hi,
                        float* lo, int64_t ld_out, void* stream) {
    clear_error();
    if (rows <= 0 || cols <= 0 || !X || !hi || !lo || (transpose != 0 && transpose != 1) || ldx < cols ||
        ld_out < (transpose ? rows : cols)) {
        set_error("bad fb_tf32_split arguments");
        return FB_ERR_INVALID_VALUE;
    }
    if (!aligned16(hi) || !aligned16(lo) || (ld_out * 4) % 16) {
        set_error("hi/lo must be 16-byte aligned with ld_out*4 a multiple of 16");
        return FB_ERR_MISALIGNED;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    return tf32_split_device(transpose, rows, cols, X, ldx, hi, lo, ld_out, st, (cudaStream_t)stream);
}

fb_status fb_matmul_3xtf32_presplit(int64_t m, int64_t n, int64_t k, const float* Ah, const float* Al,
                                    int64_t lda, const float* Bh, const float* Bl, int64_t ldb, float* C,
                                    int64_t ldc, void* stream) {
    clear_error();
    if (m <= 0 || n <= 0 || k <= 0 || !Ah || !Al || !Bh || !Bl || !C || lda < k || ldb < k || ldc < n) {
        set_error("bad fb_matmul_3xtf32_presplit arguments");
        return FB_ERR_INVALID_VALUE;
    }
    if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) {
        set_error("dimension exceeds int32");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    if (!aligned16(Ah) || !aligned16(Al) || !aligned16(Bh) || !aligned16(Bl) || !aligned16(C) || (lda * 4) % 16 ||
        (ldb * 4) % 16 || (ldc * 4) % 16) {
        set_error("operands must be 16-byte aligned, ld*4 multiples of 16");
        return FB_ERR_MISALIGNED;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    return gemm_3xtf32_presplit_device(m, n, k, Ah, Al, lda, Bh, Bl, ldb, C, ldc, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- host interface
static size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t fb_fft2d_host_workspace_bytes(int64_t n0, int64_t n1) {
    if (check_fft_dims(n0, n1) != FB_OK) return 0;
    return round_up((size_t)n0 * n1 * sizeof(float2), 256) + fft2d_ws_bytes(n0, n1);
}

fb_status fb_fft2d_host(const void* x_host, void* y_host, int64_t n0, int64_t n1, int inverse,
                        void* dev, size_t dev_bytes, void* stream) {
    clear_error();
    FB_TRY(check_fft_dims(n0, n1));
    if (!x_host || !y_host || !dev) {
        set_error("null pointer");
        return FB_ERR_INVALID_VALUE;
    }
    const size_t need = fb_fft2d_host_workspace_bytes(n0, n1);
    if (dev_bytes < need || !aligned16(dev)) {
        set_error("device scratch of %zu bytes (16B aligned) required, got %zu", need, dev_bytes);
        return FB_ERR_WORKSPACE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)n0 * n1 * sizeof(float2);
    char* d = (char*)dev;
    void* ws = d + round_up(bytes, 256);
    FB_CUDA_TRY(cudaMemcpyAsync(d, x_host, bytes, cudaMemcpyHostToDevice, s));
    FB_TRY(fft2d_device(d, d, n0, n1, inverse != 0, ws, fft2d_ws_bytes(n0, n1), st, s));
    FB_CUDA_TRY(cudaMemcpyAsync(y_host, d, bytes, cudaMemcpyDeviceToHost, s));
    FB_CUDA_TRY(cudaStreamSynchronize(s));
    return FB_OK;
}

size_t fb_fft2d_host_batch_workspace_bytes(int64_t n0, int64_t n1) {
    const size_t one = fb_fft2d_host_workspace_bytes(n0, n1);
    return one ? 2 * round_up(one, 256) : 0;
}

// Streaming form of fb_fft2d_host: `batch` independent transforms x_host[i] -> y_host[i]
// through two device slots, slot i % 2 on the caller's stream (even i) or the library's
// auxiliary stream (odd i), so the H2D copy of transform i + 1 and the D2H copy of transform i
// run on the two copy directions at once while the kernels run between them.  Ordered after
// prior work on `stream`; returns after every result is in host memory.
static std::mutex g_host_batch_mu;
fb_status fb_fft2d_host_batch(const void* x_host, void* y_host, int64_t n0, int64_t n1, int64_t batch,
                              int inverse, void* dev, size_t dev_bytes, void* stream) {
    clear_error();
    FB_TRY(check_fft_dims(n0, n1));
    if (!x_host || !y_host || !dev || batch < 1) {
        set_error(batch < 1 ? "batch must be >= 1" : "null pointer");
        return FB_ERR_INVALID_VALUE;
    }
    const size_t need = fb_fft2d_host_batch_workspace_bytes(n0, n1);
    if (dev_bytes < need || !aligned16(dev)) {
        set_error("device scratch of %zu bytes (16B aligned) required, got %zu", need, dev_bytes);
        return FB_ERR_WORKSPACE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    std::lock_guard<std::mutex> lk(g_host_batch_mu);  // one pipeline (aux stream, events) at a time
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)n0 * n1 * sizeof(float2);
    const size_t slot = need / 2;
    FB_CUDA_TRY(cudaEventRecord(st->ev_fork, s));
    FB_CUDA_TRY(cudaStreamWaitEvent(st->aux, st->ev_fork, 0));
    for (int64_t i = 0; i < batch; ++i) {
        cudaStream_t ss = (i & 1) ? st->aux : s;
        char* d = (char*)dev + (i & 1) * slot;
        void* ws = d + round_up(bytes, 256);
        // copies of one direction run one at a time, in transform order (each at the full link
        // rate), so transform i's D2H overlaps transform i+1's H2D from the first pair on
        if (i > 0) FB_CUDA_TRY(cudaStreamWaitEvent(ss, st->ev_h2d[(i - 1) & 1], 0));
        FB_CUDA_TRY(cudaMemcpyAsync(d, (const char*)x_host + i * bytes, bytes, cudaMemcpyHostToDevice, ss));
        FB_CUDA_TRY(cudaEventRecord(st->ev_h2d[i & 1], ss));
        FB_TRY(fft2d_device(d, d, n0, n1, inverse != 0, ws, fft2d_ws_bytes(n0, n1), st, ss));
        if (i > 0) FB_CUDA_TRY(cudaStreamWaitEvent(ss, st->ev_d2h[(i - 1) & 1], 0));
        FB_CUDA_TRY(cudaMemcpyAsync((char*)y_host + i * bytes, d, bytes, cudaMemcpyDeviceToHost, ss));
        FB_CUDA_TRY(cudaEventRecord(st->ev_d2h[i & 1], ss));
    }
    FB_CUDA_TRY(cudaEventRecord(st->ev_join, st->aux));
    FB_CUDA_TRY(cudaStreamWaitEvent(s, st->ev_join, 0));
    FB_CUDA_TRY(cudaStreamSynchronize(s));
    return FB_OK;
}

size_t fb_matmul_host_workspace_bytes(int dtype, int64_t m, int64_t n, int64_t k) {
    if ((dtype != FB_F32 && dtype != FB_F64) || m <= 0 || n <= 0 || k <= 0) return 0;
    const size_t es = dtype == FB_F32 ? 4 : 8;
    return round_up(m * k * es, 256) + round_up(k * n * es, 256) + round_up(m * n * es, 256) +
           gemm_ws_bytes(dtype, m, n, k);
}

fb_status fb_matmul_host(int dtype, int64_t m, int64_t n, int64_t k, const void* A_host,
                         const void* B_host, void* C_host, void* dev, size_t dev_bytes,
                         void* stream) {
    clear_error();
    if ((dtype != FB_F32 && dtype != FB_F64) || m <= 0 || n <= 0 || k <= 0) {
        set_error("bad dtype or size");
        return FB_ERR_INVALID_VALUE;
    }
    if (!A_host || !B_host || !C_host || !dev) {
        set_error("null pointer");
        return FB_ERR_INVALID_VALUE;
    }
    const size_t es = dtype == FB_F32 ? 4 : 8;
    if ((k * es) % 16 || (n * es) % 16) {
        set_error("host variant packs rows densely: k*esize and n*esize must be multiples of 16");
        return FB_ERR_MISALIGNED;
    }
    const size_t need = fb_matmul_host_workspace_bytes(dtype, m, n, k);
    if (dev_bytes < need || !aligned16(dev)) {
        set_error("device scratch of %zu bytes required, got %zu", need, dev_bytes);
        return FB_ERR_WORKSPACE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    char* d = (char*)dev;
    char* dA = d;
    char* dB = dA + round_up(m * k * es, 256);
    char* dC = dB + round_up(k * n * es, 256);
    char* ws = dC + round_up(m * n * es, 256);
    FB_CUDA_TRY(cudaMemcpyAsync(dA, A_host, m * k * es, cudaMemcpyHostToDevice, s));
    FB_CUDA_TRY(cudaMemcpyAsync(dB, B_host, k * n * es, cudaMemcpyHostToDevice, s));
    FB_TRY(gemm_device(dtype, m, n, k, dA, k, dB, n, dC, n, ws, gemm_ws_bytes(dtype, m, n, k), st, s));
    FB_CUDA_TRY(cudaMemcpyAsync(C_host, dC, m * n * es, cudaMemcpyDeviceToHost, s));
    FB_CUDA_TRY(cudaStreamSynchronize(s));
    return FB_OK;
}

// ---------------------------------------------------------------- NR-compatible shim (N3)
fb_status fb_nr_fourn(float data[], const unsigned long nn[], int ndim, int isign) {
    clear_error();
    if (!data || !nn || (ndim != 1 && ndim != 2) || (isign != 1 && isign != -1)) {
        set_error("fb_nr_fourn: need data, nn, ndim in {1,2}, isign = +-1");
        return FB_ERR_INVALID_VALUE;
    }
    const int64_t n0 = ndim == 2 ? (int64_t)nn[1] : 1;
    const int64_t n1 = ndim == 2 ? (int64_t)nn[2] : (int64_t)nn[1];
    FB_TRY(check_fft_dims(n0, n1));
    if (!is_pow2(n0) || !is_pow2(n1)) {  // NR fourn's contract: every nn[i] a power of two
        set_error("fourn: every nn[i] must be a power of two (got %lld x %lld)", (long long)n0, (long long)n1);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    DeviceState* st;
    int dev = 0;
    FB_TRY(ensure_device(&dev, &st));
    static std::mutex mu;
    static void* buf[kMaxDev] = {nullptr};
    static size_t cap[kMaxDev] = {0};
    std::lock_guard<std::mutex> lk(mu);
    const size_t bytes = (size_t)n0 * n1 * sizeof(float2);
    const size_t need = round_up(bytes, 256) + fft2d_ws_bytes(n0, n1);
    if (cap[dev] < need) {
        if (buf[dev]) cudaFree(buf[dev]);
        buf[dev] = nullptr;
        cap[dev] = 0;
        FB_CUDA_TRY(cudaMalloc(&buf[dev], need));
        cap[dev] = need;
    }
    char* d = (char*)buf[dev];
    void* ws = d + round_up(bytes, 256);
    float* host = data + 1;  // NR 1-based: data[1] is the first real part
    // NR isign = -1 is our forward (exp(-2 pi i)); isign = +1 our inverse, left unscaled
    FB_CUDA_TRY(cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice));
    FB_TRY(fft2d_device(d, d, n0, n1, isign == 1, ws, fft2d_ws_bytes(n0, n1), st, 0, /*unscaled=*/true));
    FB_CUDA_TRY(cudaMemcpy(host, d, bytes, cudaMemcpyDeviceToHost));
    return FB_OK;
}

}  // extern "C"
