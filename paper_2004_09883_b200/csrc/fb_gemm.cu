// fb_gemm.cu -- the matrix-calculation function block (north_star: dense
// GEMM C = A B, reading R9) on sm_100a.
//
// FB_F64: FP64 tensor-core FMAs (DMMA, mma.sync m16n8k8 f64; tcgen05 has no f64 kind), a
//         3-stage cp.async pipeline into padded, bank-conflict-free shared-memory tiles.
// FB_F32: 3xTF32 on the 5th-generation tensor cores.  A pre-pass splits every operand into
//         RN-rounded TF32 hi and lo parts (hi = rna(x), lo = rna(x - hi)) and writes B
//         transposed, so both operands are K-major.  The main kernel is warp specialised:
//         one TMA producer thread streams 128B-swizzled {Ahi, Alo, Bhi, Blo} k-blocks through
//         an mbarrier ring; one thread issues tcgen05.mma kind::tf32 (hi*hi + hi*lo + lo*hi)
//         into an FP32 accumulator in TMEM; four epilogue warps drain TMEM with tcgen05.ld.
#include <cuda.h>

#include "fb_common.cuh"
#include "fb_ptx.cuh"

namespace fb {

// =============================================================================== FP64 (DMMA)
namespace f64 {
constexpr int BM = 128, BN = 128, BK = 16, STAGES = 3, THREADS = 256;
constexpr int LDA_S = BK + 4;  // doubles; row stride 160 B -> conflict-free fragment loads
constexpr int LDB_S = BN + 4;  // doubles
constexpr int A_STAGE = BM * LDA_S;
constexpr int B_STAGE = BK * LDB_S;
constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);

__device__ __forceinline__ void dmma_16x8x8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

__device__ __forceinline__ void load_stage(double* As, double* Bs, const double* __restrict__ A,
                                           const double* __restrict__ B, int64_t M, int64_t N,
                                           int64_t K, int64_t lda, int64_t ldb, int64_t m0,
                                           int64_t n0, int64_t k0, int tid) {
    // A tile BM x BK: 128 rows x 8 chunks of 16 B (2 doubles)
#pragma unroll
    for (int i = 0; i < (BM * BK / 2) / THREADS; ++i) {
        const int c = tid + i * THREADS;
        const int r = c / (BK / 2), kc = (c % (BK / 2)) * 2;
        const int64_t gr = m0 + r, gk = k0 + kc;
        uint32_t bytes = 0;
        const double* src = A;
        if (gr < M && gk < K) {
            bytes = (gk + 1 < K) ? 16 : 8;
            src = A + gr * lda + gk;
        }
        ptx::cp_async_16(ptx::smem_u32(As + r * LDA_S + kc), src, bytes);
    }
    // B tile BK x BN: 16 rows x 64 chunks
#pragma unroll
    for (int i = 0; i < (BK * BN / 2) / THREADS; ++i) {
        const int c = tid + i * THREADS;
        const int r = c / (BN / 2), nc = (c % (BN / 2)) * 2;
        const int64_t gk = k0 + r, gn = n0 + nc;
        uint32_t bytes = 0;
        const double* src = B;
        if (gk < K && gn < N) {
            bytes = (gn + 1 < N) ? 16 : 8;
            src = B + gk * ldb + gn;
        }
        ptx::cp_async_16(ptx::smem_u32(Bs + r * LDB_S + nc), src, bytes);
    }
}

// 8 warps as 2 (M) x 4 (N); warp tile 64 x 32 = 4 m16 x 4 n8 DMMA tiles.
__global__ void __launch_bounds__(THREADS, 1)
    gemm_f64_dmma_kernel(const double* __restrict__ A, const double* __restrict__ B,
                         double* __restrict__ C, int64_t M, int64_t N, int64_t K, int64_t lda,
                         int64_t ldb, int64_t ldc) {
    extern __shared__ __align__(128) double smem_d[];
    double* As = smem_d;
    double* Bs = smem_d + STAGES * A_STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2, wn = warp & 3;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int KT = (int)((K + BK - 1) / BK);

    double acc[4][4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < KT)
            load_stage(As + s * A_STAGE, Bs + s * B_STAGE, A, B, M, N, K, lda, ldb, m0, n0,
                       (int64_t)s * BK, tid);
        ptx::cp_async_commit();
    }
    const int g = lane >> 2, tq = lane & 3;
    for (int kt = 0; kt < KT; ++kt) {
        ptx::cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < KT)
                load_stage(As + (nk % STAGES) * A_STAGE, Bs + (nk % STAGES) * B_STAGE, A, B, M, N,
                           K, lda, ldb, m0, n0, (int64_t)nk * BK, tid);
            ptx::cp_async_commit();
        }
        const double* as = As + (kt % STAGES) * A_STAGE + (wm * 64) * LDA_S;
        const double* bs = Bs + (kt % STAGES) * B_STAGE + wn * 32;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 8) {
            double af[4][4], bf[4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    af[i][v] = as[(i * 16 + g + 8 * (v & 1)) * LDA_S + kk + tq + 4 * (v >> 1)];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int v = 0; v < 2; ++v) bf[j][v] = bs[(kk + tq + 4 * v) * LDB_S + j * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_16x8x8(acc[i][j], af[i], bf[j]);
        }
    }
    ptx::cp_async_wait<0>();
    // epilogue: c[v] at row g + 8*(v>>1), col 2*tq + (v&1)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + wm * 64 + i * 16 + g + 8 * h;
                const int64_t c = n0 + wn * 32 + j * 8 + 2 * tq;
                if (r < M) {
                    double* dst = C + r * ldc + c;
                    if (c + 1 < N) {
                        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][2 * h], acc[i][j][2 * h + 1]);
                    } else if (c < N) {
                        dst[0] = acc[i][j][2 * h];
                    }
                }
            }
}
}  // namespace f64

// =============================================================================== FP32 (3xTF32)
namespace tf32 {
constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3;
constexpr int NUM_THREADS = 192;                    // w0 TMA, w1 MMA+TMEM, w2..5 epilogue
constexpr uint32_t TILE_A_BYTES = BM * BK * 4;      // 16 KiB
constexpr uint32_t TILE_B_BYTES = BN * BK * 4;      // 16 KiB
constexpr uint32_t STAGE_BYTES = 2 * TILE_A_BYTES + 2 * TILE_B_BYTES;
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t TMEM_COLS = 2 * BN;              // two FP32 accumulators, 128 lanes x BN columns
constexpr int NUM_EPI_WARPS = 4;
// Promotion interval: TMEM partial sums span KP_BLOCKS*BK = 128 k before they are added (RN)
// into register accumulators (error ~3e-9 * k_p under truncating accumulation).
constexpr int KP_BLOCKS = 4;
constexpr int GROUP_M = 8;                          // tile rasterisation for L2 reuse

inline int64_t kpad(int64_t k) { return (k + 3) / 4 * 4; }  // 16-byte rows for TMA

// Operand split (G1): hi = rna_tf32(x), lo = rna_tf32(x - hi), both stored as FP32 bit patterns
// with the low 13 mantissa bits zero.  A: [M][K] -> [M][Kp] (same orientation).
__global__ void split_rows_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ldx,
                                  float* __restrict__ hi, float* __restrict__ lo, int64_t ldo) {
    const int64_t total = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - r * cols;
        const float x = X[r * ldx + c];
        const uint32_t h = ptx::f32_to_tf32_rna(x);
        const float hf = __uint_as_float(h);
        const uint32_t l = ptx::f32_to_tf32_rna(x - hf);
        hi[r * ldo + c] = hf;
        lo[r * ldo + c] = __uint_as_float(l);
    }
}

// B: [K][N] -> hi/lo [N][Kp] (transposed through a 32x33 smem tile so both sides coalesce).
__global__ void split_transpose_kernel(const float* __restrict__ X, int64_t rows, int64_t cols,
                                       int64_t ldx, float* __restrict__ hi, float* __restrict__ lo,
                                       int64_t ldo) {
    __shared__ float th[32][33], tl[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t r = r0 + ty + j, c = c0 + tx;
        float x = (r < rows && c < cols) ? X[r * ldx + c] : 0.f;
        const uint32_t h = ptx::f32_to_tf32_rna(x);
        const float hf = __uint_as_float(h);
        th[ty + j][tx] = hf;
        tl[ty + j][tx] = __uint_as_float(ptx::f32_to_tf32_rna(x - hf));
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t c = c0 + ty + j, r = r0 + tx;  // output row c (= column of X), col r
        if (c < cols && r < rows) {
            hi[c * ldo + r] = th[tx][ty + j];
            lo[c * ldo + r] = tl[tx][ty + j];
        }
    }
}

__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& tm, int& tn) {
    const int per_group = GROUP_M * tiles_n;
    const int grp = tile / per_group;
    const int first_m = grp * GROUP_M;
    const int gm = min(GROUP_M, tiles_m - first_m);
    const int in = tile - grp * per_group;
    tm = first_m + in % gm;
    tn = in / gm;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                       const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
                       float* __restrict__ C, int M, int N, int K, int64_t ldc, int tiles_m, int tiles_n) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms
    const uint32_t raw_u32 = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_u32 + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_u32);
    const uint32_t bar_base = base + STAGES * STAGE_BYTES;
    // barriers: full[STAGES], empty[STAGES], tmem_full[2], tmem_empty[2]; then the TMEM slot
    auto full_bar = [&](int s) { return bar_base + 8u * s; };
    auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
    auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + b); };
    auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + 2 + b); };
    const uint32_t tmem_slot = bar_base + 8u * (2 * STAGES + 4);
    const uint32_t* tmem_slot_ptr =
        reinterpret_cast<const uint32_t*>(smem + STAGES * STAGE_BYTES + 8 * (2 * STAGES + 4));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int tm, tn;
    tile_coords(blockIdx.x, tiles_m, tiles_n, tm, tn);
    const int m0 = tm * BM, n0 = tn * BN;
    const int KB = (K + BK - 1) / BK;
    const int NCHUNK = (KB + KP_BLOCKS - 1) / KP_BLOCKS;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmAh);
        ptx::tma_prefetch_desc(&tmAl);
        ptx::tma_prefetch_desc(&tmBh);
        ptx::tma_prefetch_desc(&tmBl);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(tfull_bar(b), 1);
            ptx::mbar_init(tempty_bar(b), NUM_EPI_WARPS);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc(tmem_slot, TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            for (int kb = 0; kb < KB; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
                ptx::mbar_wait(empty_bar(s), ph ^ 1u);
                const uint32_t st = base + s * STAGE_BYTES;
                ptx::mbar_arrive_expect_tx(full_bar(s), STAGE_BYTES);
                const int kc = kb * BK;
                ptx::tma_load_2d(st, &tmAh, full_bar(s), kc, m0);
                ptx::tma_load_2d(st + TILE_A_BYTES, &tmAl, full_bar(s), kc, m0);
                ptx::tma_load_2d(st + 2 * TILE_A_BYTES, &tmBh, full_bar(s), kc, n0);
                ptx::tma_load_2d(st + 2 * TILE_A_BYTES + TILE_B_BYTES, &tmBl, full_bar(s), kc, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread)
            // instruction descriptor: D f32, A/B tf32, both K-major, N = BN, M = BM
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                   ((uint32_t)(BM >> 4) << 24);
            for (int c = 0; c < NCHUNK; ++c) {
                const int buf = c & 1;
                // wait until the epilogue has drained this accumulator buffer (chunk c-2)
                ptx::mbar_wait(tempty_bar(buf), ((uint32_t)(c >> 1) & 1u) ^ 1u);
                ptx::tc_fence_after();
                const uint32_t tmem_d = tmem_base + (uint32_t)(buf * BN);
                const int kb_end = min(KB, (c + 1) * KP_BLOCKS);
                for (int kb = c * KP_BLOCKS; kb < kb_end; ++kb) {
                    const int s = kb % STAGES;
                    const uint32_t ph = (uint32_t)(kb / STAGES) & 1u;
                    ptx::mbar_wait(full_bar(s), ph);
                    ptx::tc_fence_after();
                    const uint32_t st = base + s * STAGE_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 8; ++kk) {
                        const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes inside the swizzle atom
                        const uint64_t ah = ptx::smem_desc_sw128_kmajor(st + off);
                        const uint64_t al = ptx::smem_desc_sw128_kmajor(st + TILE_A_BYTES + off);
                        const uint64_t bh = ptx::smem_desc_sw128_kmajor(st + 2 * TILE_A_BYTES + off);
                        const uint64_t bl =
                            ptx::smem_desc_sw128_kmajor(st + 2 * TILE_A_BYTES + TILE_B_BYTES + off);
                        const uint32_t acc0 = (kb > c * KP_BLOCKS || kk > 0) ? 1u : 0u;
                        ptx::mma_tf32(tmem_d, al, bh, idesc, acc0);  // small terms first
                        ptx::mma_tf32(tmem_d, ah, bl, idesc, 1u);
                        ptx::mma_tf32(tmem_d, ah, bh, idesc, 1u);
                    }
                    ptx::mma_commit(empty_bar(s));  // frees the smem slot once these MMAs finish
                }
                ptx::mma_commit(tfull_bar(buf));    // chunk partial sum ready in TMEM
            }
        }
    } else {
        // ---------------- epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31, one row each.
        // The tensor core accumulates with truncation (measured; R11), so each
        // KP_BLOCKS*BK-deep partial sum is promoted into round-to-nearest FP32 registers.
        const int q = warp & 3;
        float acc[BN];
#pragma unroll
        for (int j = 0; j < BN; ++j) acc[j] = 0.f;
        for (int c = 0; c < NCHUNK; ++c) {
            const int buf = c & 1;
            ptx::mbar_wait(tfull_bar(buf), (uint32_t)(c >> 1) & 1u);
            ptx::tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * BN);
#pragma unroll
            for (int cb = 0; cb < BN; cb += 32) {
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(taddr + (uint32_t)cb, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[cb + j] += __uint_as_float(r[j]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty_bar(buf));
        }
        const int row = m0 + q * 32 + lane;
        if (row < M) {
            float* dst = C + (int64_t)row * ldc + n0;
            const int valid = N - n0;
            if (valid >= BN) {
#pragma unroll
                for (int j = 0; j < BN; j += 4)
                    *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < BN; ++j)
                    if (j < valid) dst[j] = acc[j];
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ------------------------------------------------------------ host: TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// rows x K fp32 matrix with row pitch ld_elems, box 128 rows x 32 (128 B) with 128B swizzle.
static fb_status make_kmajor_map(CUtensorMap* map, const float* ptr, int64_t rows, int64_t K,
                                 int64_t ld_elems, int box_rows) {
    EncodeTiledFn enc = get_encode();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return FB_ERR_CUDA;
    }
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 4)};
    cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld K=%lld ld=%lld", (int)r, (long long)rows,
                  (long long)K, (long long)ld_elems);
        return FB_ERR_CUDA;
    }
    return FB_OK;
}
}  // namespace tf32

size_t gemm_ws_bytes(int dtype, int64_t m, int64_t n, int64_t k) {
    if (dtype == FB_F64) return 0;
    const int64_t kp = tf32::kpad(k);
    return (size_t)(2 * m * kp + 2 * n * kp) * sizeof(float);
}

fb_status gemm_device(int dtype, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                      const void* B, int64_t ldb, void* C, int64_t ldc, void* ws, size_t ws_bytes,
                      const DeviceState* st, cudaStream_t s) {
    if (dtype == FB_F64) {
        static int attr_mask = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_mask & (1 << (dev & 31)))) {
            FB_CUDA_TRY(cudaFuncSetAttribute(f64::gemm_f64_dmma_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f64::SMEM));
            attr_mask |= 1 << (dev & 31);
        }
        dim3 grid((unsigned)((n + f64::BN - 1) / f64::BN), (unsigned)((m + f64::BM - 1) / f64::BM));
        if (grid.y > 65535) {
            set_error("m too large for the FP64 grid");
            return FB_ERR_UNSUPPORTED_SIZE;
        }
        f64::gemm_f64_dmma_kernel<<<grid, f64::THREADS, f64::SMEM, s>>>(
            (const double*)A, (const double*)B, (double*)C, m, n, k, lda, ldb, ldc);
        FB_LAUNCH_CHECK("gemm_f64_dmma_kernel");
        return FB_OK;
    }
    // ---- FP32 via 3xTF32: split A (same orientation), split B transposed, then the MMA kernel
    if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) {
        set_error("dimension exceeds int32");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    const int64_t kp = tf32::kpad(k);
    if (ws_bytes < gemm_ws_bytes(dtype, m, n, k)) {
        set_error("workspace too small");
        return FB_ERR_WORKSPACE;
    }
    float* Ah = (float*)ws;
    float* Al = Ah + m * kp;
    float* Bh = Al + m * kp;
    float* Bl = Bh + n * kp;
    FB_TRY(tf32_split_device(0, m, k, (const float*)A, lda, Ah, Al, kp, st, s));
    FB_TRY(tf32_split_device(1, k, n, (const float*)B, ldb, Bh, Bl, kp, st, s));
    return gemm_3xtf32_presplit_device(m, n, k, Ah, Al, kp, Bh, Bl, kp, (float*)C, ldc, s);
}

fb_status tf32_split_device(int transpose, int64_t rows, int64_t cols, const float* X, int64_t ldx, float* hi,
                            float* lo, int64_t ldo, const DeviceState* st, cudaStream_t s) {
    if (!transpose) {
        const int64_t total = rows * cols;
        int64_t blocks = (total + 255) / 256;
        const int64_t cap = (int64_t)st->sm_count * 16;
        if (blocks > cap) blocks = cap;
        if (blocks < 1) blocks = 1;
        tf32::split_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, rows, cols, ldx, hi, lo, ldo);
        FB_LAUNCH_CHECK("split_rows_kernel");
    } else {
        dim3 g2((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
        if (g2.y > 65535) {
            set_error("too many rows for the transposing split grid");
            return FB_ERR_UNSUPPORTED_SIZE;
        }
        tf32::split_transpose_kernel<<<g2, dim3(32, 8), 0, s>>>(X, rows, cols, ldx, hi, lo, ldo);
        FB_LAUNCH_CHECK("split_transpose_kernel");
    }
    return FB_OK;
}

fb_status gemm_3xtf32_presplit_device(int64_t m, int64_t n, int64_t k, const float* Ah, const float* Al,
                                      int64_t lda, const float* Bh, const float* Bl, int64_t ldb, float* C,
                                      int64_t ldc, cudaStream_t s) {
    CUtensorMap mAh, mAl, mBh, mBl;
    FB_TRY(tf32::make_kmajor_map(&mAh, Ah, m, k, lda, tf32::BM));
    FB_TRY(tf32::make_kmajor_map(&mAl, Al, m, k, lda, tf32::BM));
    FB_TRY(tf32::make_kmajor_map(&mBh, Bh, n, k, ldb, tf32::BN));
    FB_TRY(tf32::make_kmajor_map(&mBl, Bl, n, k, ldb, tf32::BN));
    static int attr_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_mask & (1 << (dev & 31)))) {
        FB_CUDA_TRY(cudaFuncSetAttribute(tf32::gemm_3xtf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tf32::SMEM));
        attr_mask |= 1 << (dev & 31);
    }
    const int tiles_m = (int)((m + tf32::BM - 1) / tf32::BM);
    const int tiles_n = (int)((n + tf32::BN - 1) / tf32::BN);
    const int64_t tiles = (int64_t)tiles_m * tiles_n;
    if (tiles > INT32_MAX) {
        set_error("too many tiles");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    tf32::gemm_3xtf32_kernel<<<(unsigned)tiles, tf32::NUM_THREADS, tf32::SMEM, s>>>(
        mAh, mAl, mBh, mBl, C, (int)m, (int)n, (int)k, ldc, tiles_m, tiles_n);
    FB_LAUNCH_CHECK("gemm_3xtf32_kernel");
    return FB_OK;
}

}  // namespace fb
