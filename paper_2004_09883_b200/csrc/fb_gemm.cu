// fb_gemm.cu -- the matrix-calculation function block (north_star: dense
// GEMM C = A B, reading R9) on sm_100a.
//
// FB_F64: FP64 tensor-core FMAs (DMMA, mma.sync m16n8k8 f64; tcgen05 has no f64 kind), a
//         3-stage cp.async pipeline into padded, bank-conflict-free shared-memory tiles;
//         64x64 tiles (several CTAs per SM) so the last wave does not idle SMs (A/B-measured:
//         128x128 642.9 us, 128x64 597.8 us, 64x64 534.5 us at 2048^3).
// FB_F32: 3xTF32 on the 5th-generation tensor cores.  A pre-pass splits every operand into
//         RN-rounded TF32 hi and lo parts (hi = rna(x), lo = rna(x - hi)) and writes B
//         transposed, so both operands are K-major.  The main kernel is warp specialised:
//         one TMA producer thread streams 128B-swizzled {Ahi, Alo, Bhi, Blo} k-blocks through
//         an mbarrier ring; one thread issues tcgen05.mma kind::tf32 (hi*hi + hi*lo + lo*hi)
//         into an FP32 accumulator in TMEM; four epilogue warps drain TMEM with tcgen05.ld.
#include <cuda.h>
#include <stdlib.h>

#include "fb_common.cuh"
#include "fb_ptx.cuh"

namespace fb {

// =============================================================================== FP64 (DMMA)
namespace f64 {
// Tile BM x BN x BK, WM x WN warps, warp tile (BM/WM) x (BN/WN) of m16n8k8 DMMA ops.
template <int BM_, int BN_, int WM_, int WN_, int BK_ = 16, int ST_ = 3>
struct Cfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = ST_, WM = WM_, WN = WN_;
    static constexpr int THREADS = 32 * WM * WN;
    static constexpr int TM = BM / WM / 16;   // m16 tiles per warp
    static constexpr int TN = BN / WN / 8;    // n8 tiles per warp
};
using CfgSmall = Cfg<64, 64, 2, 2>;   // 1024 tiles at 2048^2: balanced across 148 SMs

__device__ __forceinline__ void dmma_16x8x8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// Shared-memory layout of one stage for operand orientations TA / TB (fb_gemm's op(A), op(B)
// read straight from the stored operand, no transposed copy): A as stored (m x k) -> As[m][k]
// (row pitch BK + 4), A stored k x m -> As[k][m] (pitch BM + 4); B stored k x n -> Bs[k][n]
// (pitch BN + 4), B stored n x k -> Bs[n][k] (pitch BK + 4).  Every pitch is 4 mod 16 doubles,
// so the DMMA fragment reads of a half warp hit 16 distinct 8-byte banks in all four layouts.
template <class CF, bool TA, bool TB>
struct Lay {
    static constexpr int LDA = TA ? CF::BM + 4 : CF::BK + 4;
    static constexpr int LDB = TB ? CF::BK + 4 : CF::BN + 4;
    static constexpr int A_STAGE = TA ? CF::BK * LDA : CF::BM * LDA;
    static constexpr int B_STAGE = TB ? CF::BN * LDB : CF::BK * LDB;
    static constexpr size_t SMEM = (size_t)CF::STAGES * (A_STAGE + B_STAGE) * sizeof(double);
};

// one 16-byte cp.async chunk (2 doubles along the stored row) of a rows x cols stored operand,
// zero-filled past its edges (8 bytes when only the first double is inside)
__device__ __forceinline__ void ld_chunk(double* dst, const double* __restrict__ X, int64_t rows, int64_t cols,
                                         int64_t ld, int64_t gr, int64_t gc) {
    uint32_t bytes = 0;
    const double* src = X;
    if (gr < rows && gc < cols) {
        bytes = (gc + 1 < cols) ? 16 : 8;
        src = X + gr * ld + gc;
    }
    ptx::cp_async_16(ptx::smem_u32(dst), src, bytes);
}

// tile R x Ccols (stored orientation) starting at (r0, c0) into S[R][pitch]
template <int R, int CC, int PITCH, int THREADS>
__device__ __forceinline__ void load_tile(double* S, const double* __restrict__ X, int64_t rows, int64_t cols,
                                          int64_t ld, int64_t r0, int64_t c0, int tid) {
#pragma unroll
    for (int i = 0; i < (R * CC / 2 + THREADS - 1) / THREADS; ++i) {
        const int c = tid + i * THREADS;
        if (c < R * CC / 2) {
            const int r = c / (CC / 2), cc = (c % (CC / 2)) * 2;
            ld_chunk(S + r * PITCH + cc, X, rows, cols, ld, r0 + r, c0 + cc);
        }
    }
}

template <class CF, bool TA, bool TB>
__device__ __forceinline__ void load_stage(double* As, double* Bs, const double* __restrict__ A,
                                           const double* __restrict__ B, int64_t M, int64_t N,
                                           int64_t K, int64_t lda, int64_t ldb, int64_t m0,
                                           int64_t n0, int64_t k0, int tid) {
    using L = Lay<CF, TA, TB>;
    if constexpr (TA)  // A stored K x M
        load_tile<CF::BK, CF::BM, L::LDA, CF::THREADS>(As, A, K, M, lda, k0, m0, tid);
    else
        load_tile<CF::BM, CF::BK, L::LDA, CF::THREADS>(As, A, M, K, lda, m0, k0, tid);
    if constexpr (TB)  // B stored N x K
        load_tile<CF::BN, CF::BK, L::LDB, CF::THREADS>(Bs, B, N, K, ldb, n0, k0, tid);
    else
        load_tile<CF::BK, CF::BN, L::LDB, CF::THREADS>(Bs, B, K, N, ldb, k0, n0, tid);
}

// Epilogue modes: EPI_STORE C <- A B;  EPI_SUB C <- C - A B (the LU trailing update);
// EPI_AXPBY C <- alpha A B + beta C (fb_gemm; C is not read when beta == 0).
enum { EPI_STORE = 0, EPI_SUB = 1, EPI_AXPBY = 2 };

// The k-loop order (k-blocks ascending, then kk, then the DMMA's internal order) is the same
// for every tile shape and operand orientation, so results are bitwise identical across them.
template <class CF, int EPI = EPI_STORE, bool TA = false, bool TB = false>
__global__ void __launch_bounds__(CF::THREADS)
    gemm_f64_dmma_kernel(const double* __restrict__ A, const double* __restrict__ B,
                         double* C, int64_t M, int64_t N, int64_t K, int64_t lda,
                         int64_t ldb, int64_t ldc, double alpha, double beta) {
    using L = Lay<CF, TA, TB>;
    extern __shared__ __align__(128) double smem_d[];
    double* As = smem_d;
    double* Bs = smem_d + CF::STAGES * L::A_STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / CF::WN, wn = warp % CF::WN;
    const int64_t m0 = (int64_t)blockIdx.y * CF::BM, n0 = (int64_t)blockIdx.x * CF::BN;
    const int KT = (int)((K + CF::BK - 1) / CF::BK);

    double acc[CF::TM][CF::TN][4];
#pragma unroll
    for (int i = 0; i < CF::TM; ++i)
#pragma unroll
        for (int j = 0; j < CF::TN; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

#pragma unroll
    for (int st = 0; st < CF::STAGES - 1; ++st) {
        if (st < KT)
            load_stage<CF, TA, TB>(As + st * L::A_STAGE, Bs + st * L::B_STAGE, A, B, M, N, K, lda, ldb, m0, n0,
                                   (int64_t)st * CF::BK, tid);
        ptx::cp_async_commit();
    }
    const int g = lane >> 2, tq = lane & 3;
    for (int kt = 0; kt < KT; ++kt) {
        ptx::cp_async_wait<CF::STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + CF::STAGES - 1;
            if (nk < KT)
                load_stage<CF, TA, TB>(As + (nk % CF::STAGES) * L::A_STAGE, Bs + (nk % CF::STAGES) * L::B_STAGE,
                                       A, B, M, N, K, lda, ldb, m0, n0, (int64_t)nk * CF::BK, tid);
            ptx::cp_async_commit();
        }
        const double* as = As + (kt % CF::STAGES) * L::A_STAGE;
        const double* bs = Bs + (kt % CF::STAGES) * L::B_STAGE;
        const int ar = wm * CF::TM * 16, bc = wn * CF::TN * 8;  // warp tile origin (m, n)
#pragma unroll
        for (int kk = 0; kk < CF::BK; kk += 8) {
            double af[CF::TM][4], bf[CF::TN][2];
#pragma unroll
            for (int i = 0; i < CF::TM; ++i)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int r = ar + i * 16 + g + 8 * (v & 1), kc = kk + tq + 4 * (v >> 1);
                    af[i][v] = TA ? as[kc * L::LDA + r] : as[r * L::LDA + kc];
                }
#pragma unroll
            for (int j = 0; j < CF::TN; ++j)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int kc = kk + tq + 4 * v, c = bc + j * 8 + g;
                    bf[j][v] = TB ? bs[c * L::LDB + kc] : bs[kc * L::LDB + c];
                }
#pragma unroll
            for (int i = 0; i < CF::TM; ++i)
#pragma unroll
                for (int j = 0; j < CF::TN; ++j) dmma_16x8x8(acc[i][j], af[i], bf[j]);
        }
    }
    ptx::cp_async_wait<0>();
    // epilogue: c[v] at row g + 8*(v>>1), col 2*tq + (v&1)
    auto out = [&](double p, const double* cur) -> double {
        if constexpr (EPI == EPI_SUB) return *cur - p;
        if constexpr (EPI == EPI_AXPBY) return beta == 0.0 ? alpha * p : alpha * p + beta * *cur;
        return p;
    };
#pragma unroll
    for (int i = 0; i < CF::TM; ++i)
#pragma unroll
        for (int j = 0; j < CF::TN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + wm * CF::TM * 16 + i * 16 + g + 8 * h;
                const int64_t c = n0 + wn * CF::TN * 8 + j * 8 + 2 * tq;
                if (r < M) {
                    double* dst = C + r * ldc + c;
                    if (c + 1 < N) {
                        double2 o = make_double2(acc[i][j][2 * h], acc[i][j][2 * h + 1]);
                        if constexpr (EPI != EPI_STORE) o = make_double2(out(o.x, dst), out(o.y, dst + 1));
                        *reinterpret_cast<double2*>(dst) = o;
                    } else if (c < N) {
                        dst[0] = out(acc[i][j][2 * h], dst);
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
__device__ __forceinline__ void split1(float x, float& h, float& l) {
    h = __uint_as_float(ptx::f32_to_tf32_rna(x));
    l = __uint_as_float(ptx::f32_to_tf32_rna(x - h));
}
// lo for a raw FP32 hi operand: the tensor core truncates an FP32 operand to TF32 (reading R21),
// so hi = trunc(x) and lo = rna(x - trunc(x)) (x - trunc(x) is exact in FP32)
__device__ __forceinline__ float lo_trunc(float x) {
    return __uint_as_float(ptx::f32_to_tf32_rna(x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u)));
}

// 2D grid: blockIdx.y = row block, x covers columns in float4 chunks (rows are 16-byte aligned:
// ldx*4 and ldo*4 are multiples of 16 by the API contract).
template <bool LO_ONLY = false>  // LO_ONLY: raw-hi mode, lo = rna(x - trunc(x)) only (hi unused)
__global__ void split_rows_kernel(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ldx,
                                  float* __restrict__ hi, float* __restrict__ lo, int64_t ldo) {
    const int64_t c4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (c4 >= cols) return;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const float* xr = X + r * ldx;
        float* hr = hi + r * ldo;
        float* lr = lo + r * ldo;
        if constexpr (LO_ONLY) {
            if (c4 + 4 <= cols) {
                const float4 x = *reinterpret_cast<const float4*>(xr + c4);
                *reinterpret_cast<float4*>(lr + c4) = make_float4(lo_trunc(x.x), lo_trunc(x.y), lo_trunc(x.z),
                                                                  lo_trunc(x.w));
            } else {
                for (int64_t c = c4; c < cols; ++c) lr[c] = lo_trunc(xr[c]);
            }
        } else if (c4 + 4 <= cols) {
            const float4 x = *reinterpret_cast<const float4*>(xr + c4);
            float4 h, l;
            split1(x.x, h.x, l.x);
            split1(x.y, h.y, l.y);
            split1(x.z, h.z, l.z);
            split1(x.w, h.w, l.w);
            *reinterpret_cast<float4*>(hr + c4) = h;
            *reinterpret_cast<float4*>(lr + c4) = l;
        } else {
            for (int64_t c = c4; c < cols; ++c) split1(xr[c], hr[c], lr[c]);
        }
    }
}

// B: [K][N] -> hi/lo [N][Kp] (transposed through a 32x33 smem tile so both sides coalesce).
// TRUNC: raw-hi mode -- hi = trunc(x) (the value the tensor core uses for a raw FP32 operand),
// lo = rna(x - trunc(x)), so a transposed operand gives the same product as the raw one
template <bool TRUNC = false>
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
        const float hf = TRUNC ? __uint_as_float(__float_as_uint(x) & 0xFFFFE000u)
                               : __uint_as_float(ptx::f32_to_tf32_rna(x));
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

// Both operand splits of fb_matmul in one launch (the two halves stream concurrently instead
// of back to back): blocks [0, nblk_a) split A row-wise (float4 chunks, 256 columns per block
// row segment), the rest split-transpose B in 32 x 32 tiles (as split_transpose_kernel).
__global__ void __launch_bounds__(256)
    split_both_kernel(const float* __restrict__ A, int64_t m, int64_t k, int64_t lda, float* __restrict__ Ah,
                      float* __restrict__ Al, const float* __restrict__ B, int64_t n, int64_t ldb,
                      float* __restrict__ Bh, float* __restrict__ Bl, int64_t ldo, int64_t nblk_a, int a_cblk) {
    __shared__ float th[32][33], tl[32][33];
    const int64_t bid = blockIdx.x;
    if (bid < nblk_a) {
        const int64_t r = bid / a_cblk;
        const int64_t c4 = ((bid % a_cblk) * 256 + threadIdx.x) * 4;
        if (c4 >= k) return;
        const float* xr = A + r * lda;
        float* hr = Ah + r * ldo;
        float* lr = Al + r * ldo;
        if (c4 + 4 <= k) {
            const float4 x = *reinterpret_cast<const float4*>(xr + c4);
            float4 h, l;
            split1(x.x, h.x, l.x);
            split1(x.y, h.y, l.y);
            split1(x.z, h.z, l.z);
            split1(x.w, h.w, l.w);
            *reinterpret_cast<float4*>(hr + c4) = h;
            *reinterpret_cast<float4*>(lr + c4) = l;
        } else {
            for (int64_t c = c4; c < k; ++c) split1(xr[c], hr[c], lr[c]);
        }
        return;
    }
    // B [k][n] -> hi/lo [n][ldo]
    const int64_t tb = bid - nblk_a;
    const int64_t tiles_c = (n + 31) / 32;
    const int64_t r0 = (tb / tiles_c) * 32, c0 = (tb % tiles_c) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t r = r0 + ty + j, c = c0 + tx;
        const float x = (r < k && c < n) ? B[r * ldb + c] : 0.f;
        const float hf = __uint_as_float(ptx::f32_to_tf32_rna(x));
        th[ty + j][tx] = hf;
        tl[ty + j][tx] = __uint_as_float(ptx::f32_to_tf32_rna(x - hf));
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t c = c0 + ty + j, r = r0 + tx;
        if (c < n && r < k) {
            Bh[c * ldo + r] = th[tx][ty + j];
            Bl[c * ldo + r] = tl[tx][ty + j];
        }
    }
}

// split_both_kernel with 4x the work per thread (all loads of a thread issued before its first
// store): blocks [0, nblk_a) take 1024 consecutive float4 chunks of A's rows (flattened over
// rows, so short rows do not leave threads idle; m * ceil(k/4) < 2^31 is checked by the
// caller), the rest split-transpose 64 x 64 tiles of B through padded shared memory
// (conflict-free: pitch 65).  Same split1 per element, so the outputs are bitwise identical.
__global__ void __launch_bounds__(256)
    split_both_wide_kernel(const float* __restrict__ A, int64_t m, int64_t k, int64_t lda, float* __restrict__ Ah,
                           float* __restrict__ Al, const float* __restrict__ B, int64_t n, int64_t ldb,
                           float* __restrict__ Bh, float* __restrict__ Bl, int64_t ldo, int64_t nblk_a,
                           int pdl_trigger, int a_raw_hi) {
    __shared__ float th[64][65], tl[64][65];
    const int64_t bid = blockIdx.x;
    const int tid = threadIdx.x;
    // let the GEMM grid (launched with programmatic serialization) be scheduled as SMs free up;
    // its griddepcontrol.wait still waits for this whole grid and its memory (knob FB_GEMM_SPLIT_PDL)
    if (pdl_trigger) ptx::pdl_launch_dependents();
    if (bid < nblk_a) {
        const uint32_t ck = (uint32_t)((k + 3) / 4);
        const uint32_t total = (uint32_t)m * ck;
        float4 x[4];
        uint32_t rr[4], cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t q = (uint32_t)bid * 1024u + (uint32_t)u * 256u + (uint32_t)tid;
            rr[u] = q / ck;
            cc[u] = (q - rr[u] * ck) * 4u;
            if (q < total && cc[u] + 4 <= k) x[u] = *reinterpret_cast<const float4*>(A + rr[u] * lda + cc[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t q = (uint32_t)bid * 1024u + (uint32_t)u * 256u + (uint32_t)tid;
            if (q >= total) continue;
            const float* xr = A + (int64_t)rr[u] * lda;
            float* hr = Ah + (int64_t)rr[u] * ldo;
            float* lr = Al + (int64_t)rr[u] * ldo;
            const int64_t c4 = cc[u];
            if (a_raw_hi) {  // A's hi is the raw operand: only lo is written
                if (c4 + 4 <= k) {
                    *reinterpret_cast<float4*>(lr + c4) =
                        make_float4(lo_trunc(x[u].x), lo_trunc(x[u].y), lo_trunc(x[u].z), lo_trunc(x[u].w));
                } else {
                    for (int64_t c = c4; c < k; ++c) lr[c] = lo_trunc(xr[c]);
                }
            } else if (c4 + 4 <= k) {
                float4 h, l;
                split1(x[u].x, h.x, l.x);
                split1(x[u].y, h.y, l.y);
                split1(x[u].z, h.z, l.z);
                split1(x[u].w, h.w, l.w);
                *reinterpret_cast<float4*>(hr + c4) = h;
                *reinterpret_cast<float4*>(lr + c4) = l;
            } else {
                for (int64_t c = c4; c < k; ++c) split1(xr[c], hr[c], lr[c]);
            }
        }
        return;
    }
    // B [k][n] -> hi/lo [n][ldo], 64 x 64 tiles
    const int64_t tb = bid - nblk_a;
    const int64_t tiles_c = (n + 63) / 64;
    const int64_t r0 = (tb / tiles_c) * 64, c0 = (tb % tiles_c) * 64;
    const int lane = tid & 31, w = tid >> 5;  // 8 warps
    float xv[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t r = r0 + w + 8 * j, c = c0 + lane + 32 * h;
            xv[2 * j + h] = (r < k && c < n) ? B[r * ldb + c] : 0.f;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float hf, lf;
            split1(xv[2 * j + h], hf, lf);
            th[w + 8 * j][lane + 32 * h] = hf;
            tl[w + 8 * j][lane + 32 * h] = lf;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int64_t c = c0 + w + 8 * j;  // output row (= column of B)
        if (c >= n) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t r = r0 + lane + 32 * h;
            if (r < k) {
                Bh[c * ldo + r] = th[lane + 32 * h][w + 8 * j];
                Bl[c * ldo + r] = tl[lane + 32 * h][w + 8 * j];
            }
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
// two-level raster: N-panels of pw tile columns in order, the grouped raster inside each
// (pw <= 0: one panel)
__device__ __forceinline__ void tile_coords_panel(int tile, int tiles_m, int tiles_n, int pw, int& tm, int& tn) {
    if (pw <= 0 || pw >= tiles_n) {
        tile_coords(tile, tiles_m, tiles_n, tm, tn);
        return;
    }
    const int p = tile / (tiles_m * pw);
    const int wp = min(pw, tiles_n - p * pw);
    tile_coords(tile - p * tiles_m * pw, tiles_m, wp, tm, tn);
    tn += p * pw;
}

// one epilogue row segment: dst[j] = alpha acc[j] + beta dst[j] for j < min(W, valid) (fb_gemm's
// epilogue; dst is not read when beta == 0, and (alpha, beta) = (1, 0) stores acc exactly)
template <int W>
__device__ __forceinline__ void store_row(float* dst, const float (&acc)[W], int valid, float alpha, float beta) {
    if (valid >= W) {
#pragma unroll
        for (int j = 0; j < W; j += 4) {
            float4 o = make_float4(alpha * acc[j], alpha * acc[j + 1], alpha * acc[j + 2], alpha * acc[j + 3]);
            if (beta != 0.f) {
                const float4 c = *reinterpret_cast<const float4*>(dst + j);
                o = make_float4(o.x + beta * c.x, o.y + beta * c.y, o.z + beta * c.z, o.w + beta * c.w);
            }
            *reinterpret_cast<float4*>(dst + j) = o;
        }
    } else {
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (j < valid) dst[j] = beta != 0.f ? alpha * acc[j] + beta * dst[j] : alpha * acc[j];
    }
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                       const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
                       float* __restrict__ C, int M, int N, int K, int64_t ldc, int tiles_m, int tiles_n,
        float alpha, float beta) {
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
            store_row<BN>(dst, acc, valid, alpha, beta);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ------------------------------------------------------------ 2-CTA (cta_group::2) kernel
// A CTA pair computes a 256 x NT tile (NT = 256, or 240 where that fills the 74 pairs better):
// CTA r stages A rows [m0 + 128 r, +128) and B^T rows [n0 + NT/2 r, +NT/2) (x 32 fp32 per
// k-block, hi and lo; A's hi is A itself in the default raw-hi mode), so each SM's shared-memory
// path carries half of each operand (the 1-CTA 128x128 form is bound by the
// smem data path: TMA writes + operand reads exceed the MMA time).  The leader issues
// tcgen05.mma.cta_group::2 (M = 256, N = NT, K = 8) into TMEM of both CTAs; each CTA's 8
// epilogue warps promote their 128 rows x NT columns (two NT/2-column halves) into RN FP32
// registers every KP_BLOCKS k-blocks and apply alpha / beta when storing C.  A launch with
// fewer pairs than tiles runs persistent (FB_GEMM_PERSIST; measured slower, off).
namespace pair {
constexpr int BK = 32, STAGES = 3;                         // per-CTA tile halves: 128 x 32
constexpr int NUM_THREADS = 320;                          // w0 TMA, w1 MMA/TMEM, w2..9 epilogue
constexpr int NUM_EPI_WARPS = 8;
constexpr uint32_t TILE_BYTES = 128 * BK * 4;             // 16 KiB
constexpr uint32_t STAGE_BYTES = 4 * TILE_BYTES;          // Ahi, Alo, Bhi, Blo halves
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t ACC_COLS = 256;                        // N of the pair MMA
constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;              // double-buffered accumulator
#ifndef FB_TF32_KP
#define FB_TF32_KP 4
#endif
// k-blocks (of 32) between RN promotions: every 128 k.  Longer intervals buy nothing and cost
// accuracy (A/B: 256 k / 512 k: 2048^3 87.8 -> 87.9 / 87.5 us, 8192^3 -0.6 %; K = 32768 error
// 9.6e-7 -> 1.8e-6 / 3.6e-6)
constexpr int KP_BLOCKS = FB_TF32_KP;

// NT: N of the pair tile (256, or 240 so that e.g. 2048 columns make 9 tiles and 2048^2 fills 72 of
// the 74 CTA pairs in one wave); each CTA stages NT / 2 rows of B^T
template <int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_3xtf32_pair_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                            const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
                            float* __restrict__ C, int M, int N, int K, int64_t ldc, int tiles_m, int tiles_n,
        float alpha, float beta, int panel_tn) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_u32 + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_u32);
    const uint32_t bar_base = base + STAGES * STAGE_BYTES;
    auto full_bar = [&](int s) { return bar_base + 8u * s; };
    auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
    auto tfull_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + b); };
    auto tempty_bar = [&](int b) { return bar_base + 8u * (2 * STAGES + 2 + b); };
    const uint32_t tmem_slot = bar_base + 8u * (2 * STAGES + 4);
    const uint32_t* tmem_slot_ptr =
        reinterpret_cast<const uint32_t*>(smem + STAGES * STAGE_BYTES + 8 * (2 * STAGES + 4));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    // persistent: pair p computes tiles p, p + P, p + 2P, ... (P = pairs in the grid; round
    // robin keeps the concurrently computed tiles adjacent in the grouped raster order); the
    // stage ring and the two TMEM accumulators run on across tiles, so a tile's epilogue (drain
    // of its last chunk + C stores) overlaps the next tile's first MMAs
    const int pair = (int)(blockIdx.x >> 1), P = (int)(gridDim.x >> 1);
    const int ntiles = tiles_m * tiles_n;
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
            ptx::mbar_init(tempty_bar(b), 2 * NUM_EPI_WARPS);  // both CTAs' epilogue warps
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc_pair(tmem_slot, TMEM_COLS);
        ptx::tmem_relinquish_pair();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;
    ptx::pdl_wait();  // PDL: the split kernel's outputs are complete (setup above overlapped it)

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs): own halves, completion on the leader
            int g = 0;  // k-blocks issued (stage ring position across tiles)
            for (int tile = pair; tile < ntiles; tile += P) {
            int tm, tn;
            tf32::tile_coords_panel(tile, tiles_m, tiles_n, panel_tn, tm, tn);
            const int am = tm * 256 + 128 * (int)rank, bn = tn * NT + (NT / 2) * (int)rank;
            for (int kb = 0; kb < KB; ++kb, ++g) {
                const int s = g % STAGES;
                const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
                ptx::mbar_wait(empty_bar(s), ph ^ 1u);
                if (leader) ptx::mbar_arrive_expect_tx(full_bar(s), 2 * (2 * TILE_BYTES + 2 * (NT / 2) * BK * 4));
                const uint32_t st = base + s * STAGE_BYTES;
                const int kc = kb * BK;
                ptx::tma_load_2d_pair(st, &tmAh, full_bar(s), kc, am);
                ptx::tma_load_2d_pair(st + TILE_BYTES, &tmAl, full_bar(s), kc, am);
                ptx::tma_load_2d_pair(st + 2 * TILE_BYTES, &tmBh, full_bar(s), kc, bn);
                ptx::tma_load_2d_pair(st + 3 * TILE_BYTES, &tmBl, full_bar(s), kc, bn);
            }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            // ---------------- MMA issuer (leader CTA, single thread)
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) |
                                   ((uint32_t)(256 >> 4) << 24);
            int g = 0, cg = 0;  // k-blocks consumed, chunks issued (across tiles)
            for (int tile = pair; tile < ntiles; tile += P) {
            for (int c = 0; c < NCHUNK; ++c, ++cg) {
                const int buf = cg & 1;
                ptx::mbar_wait(tempty_bar(buf), ((uint32_t)(cg >> 1) & 1u) ^ 1u);
                ptx::tc_fence_after();
                const uint32_t tmem_d = tmem_base + (uint32_t)(buf * ACC_COLS);
                const int kb_end = min(KB, (c + 1) * KP_BLOCKS);
                for (int kb = c * KP_BLOCKS; kb < kb_end; ++kb, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
                    ptx::mbar_wait(full_bar(s), ph);
                    ptx::tc_fence_after();
                    const uint32_t st = base + s * STAGE_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / 8; ++kk) {
                        const uint32_t off = kk * 32;
                        const uint64_t ah = ptx::smem_desc_sw128_kmajor(st + off);
                        const uint64_t al = ptx::smem_desc_sw128_kmajor(st + TILE_BYTES + off);
                        const uint64_t bh = ptx::smem_desc_sw128_kmajor(st + 2 * TILE_BYTES + off);
                        const uint64_t bl = ptx::smem_desc_sw128_kmajor(st + 3 * TILE_BYTES + off);
                        const uint32_t acc0 = (kb > c * KP_BLOCKS || kk > 0) ? 1u : 0u;
                        ptx::mma_tf32_pair(tmem_d, al, bh, idesc, acc0);
                        ptx::mma_tf32_pair(tmem_d, ah, bl, idesc, 1u);
                        ptx::mma_tf32_pair(tmem_d, ah, bh, idesc, 1u);
                    }
                    ptx::mma_commit_pair(empty_bar(s), 0x3);  // frees the slot in both CTAs
                }
                ptx::mma_commit_pair(tfull_bar(buf), 0x3);    // partial sum ready in both CTAs
            }
            }
        }
    } else {
        // ---------------- epilogue warps 2..9: lanes 32*(warp%4), column half (warp-2)/4
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        int cg = 0;  // chunks drained (across tiles)
        for (int tile = pair; tile < ntiles; tile += P) {
        int tm, tn;
        tf32::tile_coords_panel(tile, tiles_m, tiles_n, panel_tn, tm, tn);
        constexpr int HALF = NT / 2;
        const int m0 = tm * 256, n0 = tn * NT;
        float acc[HALF];
#pragma unroll
        for (int j = 0; j < HALF; ++j) acc[j] = 0.f;
        for (int c = 0; c < NCHUNK; ++c, ++cg) {
            const int buf = cg & 1;
            ptx::mbar_wait(tfull_bar(buf), (uint32_t)(cg >> 1) & 1u);
            ptx::tc_fence_after();
            const uint32_t taddr =
                tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * ACC_COLS + h * HALF);
#pragma unroll
            for (int cb = 0; cb + 32 <= HALF; cb += 32) {
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(taddr + (uint32_t)cb, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[cb + j] += __uint_as_float(r[j]);
            }
            if constexpr (HALF % 32 >= 16) {  // NT = 240: columns 96..119 as x16 + x8
                constexpr int cb = HALF / 32 * 32;
                uint32_t r[16];
                ptx::tmem_ld_32x32b_x16(taddr + (uint32_t)cb, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[cb + j] += __uint_as_float(r[j]);
            }
            if constexpr (HALF % 16 == 8) {
                constexpr int cb = HALF / 16 * 16;
                uint32_t r[8];
                ptx::tmem_ld_32x32b_x8(taddr + (uint32_t)cb, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[cb + j] += __uint_as_float(r[j]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_leader(tempty_bar(buf));
        }
        const int row = m0 + 128 * (int)rank + q * 32 + lane;
        const int col0 = n0 + h * HALF;
        if (row < M) {
            float* dst = C + (int64_t)row * ldc + col0;
            const int valid = N - col0;
            store_row<HALF>(dst, acc, valid, alpha, beta);
        }
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem_base, TMEM_COLS);
    }
}
}  // namespace pair

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

template <class CF, int EPI, bool TA, bool TB>
static fb_status launch_f64_t(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                              int64_t ldb, void* C, int64_t ldc, double alpha, double beta, cudaStream_t s) {
    auto kern = f64::gemm_f64_dmma_kernel<CF, EPI, TA, TB>;
    constexpr size_t smem = f64::Lay<CF, TA, TB>::SMEM;
    static std::atomic<int> attr_mask{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_mask & (1 << (dev & 31)))) {
        FB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_mask |= 1 << (dev & 31);
    }
    if (m <= 0 || n <= 0 || k <= 0) return FB_OK;
    dim3 grid((unsigned)((n + CF::BN - 1) / CF::BN), (unsigned)((m + CF::BM - 1) / CF::BM));
    if (grid.y > 65535) {
        set_error("m too large for the FP64 grid");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    kern<<<grid, CF::THREADS, smem, s>>>((const double*)A, (const double*)B, (double*)C, m, n, k, lda, ldb, ldc,
                                         alpha, beta);
    FB_LAUNCH_CHECK("gemm_f64_dmma_kernel");
    return FB_OK;
}

template <class CF>
static fb_status launch_f64(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                            void* C, int64_t ldc, cudaStream_t s) {
    return launch_f64_t<CF, f64::EPI_STORE, false, false>(m, n, k, A, lda, B, ldb, C, ldc, 1.0, 0.0, s);
}

// C -= A B in FP64 (LU trailing update; C may alias neither A nor B).
fb_status gemm_f64_sub_device(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                              int64_t ldb, double* C, int64_t ldc, cudaStream_t s) {
    return launch_f64_t<f64::CfgSmall, f64::EPI_SUB, false, false>(m, n, k, A, lda, B, ldb, C, ldc, 1.0, 0.0, s);
}

size_t gemm_ws_bytes(int dtype, int64_t m, int64_t n, int64_t k) {
    if (dtype == FB_F64) return 0;
    const int64_t kp = tf32::kpad(k);
    const size_t split = (size_t)(2 * m * kp + 2 * n * kp) * sizeof(float);  // default path
    if (!knobs().gemm_fused) return split;
    // FB_GEMM_FUSED=1: lo operands + stream-K partial slots (with less, the fused kernel forms
    // lo in shared memory and needs no workspace)
    const size_t fused = gemm_3xtf32_fused_ws_bytes(m, n, k);
    return split > fused ? split : fused;
}

fb_status gemm_device(int dtype, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                      const void* B, int64_t ldb, void* C, int64_t ldc, void* ws, size_t ws_bytes,
                      const DeviceState* st, cudaStream_t s) {
    return gemm_ex_device(dtype, 0, 0, m, n, k, 1.0, A, lda, B, ldb, 0.0, C, ldc, ws, ws_bytes, st, s);
}

template <int EPI>
static fb_status launch_f64_op(int ta, int tb, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda,
                               const void* B, int64_t ldb, void* C, int64_t ldc, double alpha, double beta,
                               cudaStream_t s) {
    using CF = f64::CfgSmall;
    if (ta && tb) return launch_f64_t<CF, EPI, true, true>(m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, s);
    if (ta) return launch_f64_t<CF, EPI, true, false>(m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, s);
    if (tb) return launch_f64_t<CF, EPI, false, true>(m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, s);
    return launch_f64_t<CF, EPI, false, false>(m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, s);
}

fb_status gemm_ex_device(int dtype, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                         int64_t lda, const void* B, int64_t ldb, double beta, void* C, int64_t ldc, void* ws,
                         size_t ws_bytes, const DeviceState* st, cudaStream_t s) {
    const bool plain = alpha == 1.0 && beta == 0.0;
    if (dtype == FB_F64) {
        if (!plain) return launch_f64_op<f64::EPI_AXPBY>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, s);
        if (ta || tb) return launch_f64_op<f64::EPI_STORE>(ta, tb, m, n, k, A, lda, B, ldb, C, ldc, 1.0, 0.0, s);
        const int cfg = knobs().f64_cfg;  // A/B knob: 0 = 64x64 (default), 1 = 128x128, 2 = 128x64
        if (cfg == 1) return launch_f64<f64::Cfg<128, 128, 2, 4>>(m, n, k, A, lda, B, ldb, C, ldc, s);
        if (cfg == 2) return launch_f64<f64::Cfg<128, 64, 2, 2>>(m, n, k, A, lda, B, ldb, C, ldc, s);
        return launch_f64<f64::CfgSmall>(m, n, k, A, lda, B, ldb, C, ldc, s);
    }
    // ---- FP32 via 3xTF32: split pre-pass (op(A) and op(B)^T to K-major hi/lo) + MMA kernel with
    // the alpha/beta epilogue; A/B knob FB_GEMM_FUSED=1 (plain products only): one fused kernel
    // (raw operands, lo formed in shared memory, fb_gemm_fused.cu)
    if (knobs().gemm_fused && plain && !ta && !tb)
        return gemm_3xtf32_fused_device(m, n, k, (const float*)A, lda, (const float*)B, ldb, (float*)C, ldc, ws,
                                        ws_bytes, s);
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
    // Raw-hi mode (A/B knob FB_GEMM_AHI_RAW, default 1): A's hi operand is A itself (the tensor core
    // truncates it to TF32, reading R21) and only lo = rna(a - trunc(a)) is written -- 16 of the
    // 96 MiB of split traffic at 2048^3; a transposed A is split to exactly those values
    const bool raw_mode = knobs().gemm_ahi_raw != 0;
    bool a_raw = false;  // Ah = A (raw) instead of a split hi
    if (ta || tb) {  // transposed operands: A^T stored k x m splits transposing, B^T stored n x k as is
        if (ta)
            FB_TRY(tf32_split_device(1, k, m, (const float*)A, lda, Ah, Al, kp, st, s, raw_mode));
        else if (raw_mode)
            FB_TRY(tf32_lo_device(m, k, (const float*)A, lda, Al, kp, s));
        else
            FB_TRY(tf32_split_device(0, m, k, (const float*)A, lda, Ah, Al, kp, st, s));
        a_raw = !ta && raw_mode;
        FB_TRY(tf32_split_device(tb ? 0 : 1, tb ? n : k, tb ? k : n, (const float*)B, ldb, Bh, Bl, kp, st, s));
    } else if (knobs().gemm_split2 == 1) {  // A/B knob: 1 = two split launches
        FB_TRY(tf32_split_device(0, m, k, (const float*)A, lda, Ah, Al, kp, st, s));
        FB_TRY(tf32_split_device(1, k, n, (const float*)B, ldb, Bh, Bl, kp, st, s));
    } else if (knobs().gemm_splitv != 1 &&
               m * ((k + 3) / 4) + 1024 < INT32_MAX) {
        a_raw = raw_mode;
        // default: the wide split (A/B knob FB_GEMM_SPLITV=1: split_both_kernel)
        const int64_t nblk_a = (m * ((k + 3) / 4) + 1023) / 1024;
        const int64_t nblk_b = ((k + 63) / 64) * ((n + 63) / 64);
        if (nblk_a + nblk_b > INT32_MAX) {
            set_error("split grid too large");
            return FB_ERR_UNSUPPORTED_SIZE;
        }
        tf32::split_both_wide_kernel<<<(unsigned)(nblk_a + nblk_b), 256, 0, s>>>(
            (const float*)A, m, k, lda, Ah, Al, (const float*)B, n, ldb, Bh, Bl, kp, nblk_a,
            knobs().gemm_split_pdl == 1 ? 1 : 0, a_raw ? 1 : 0);
        FB_LAUNCH_CHECK("split_both_wide_kernel");
    } else {
        const int a_cblk = (int)((((k + 3) / 4) + 255) / 256);
        const int64_t nblk_a = m * a_cblk;
        const int64_t nblk_b = ((k + 31) / 32) * ((n + 31) / 32);
        if (nblk_a + nblk_b > INT32_MAX) {
            set_error("split grid too large");
            return FB_ERR_UNSUPPORTED_SIZE;
        }
        tf32::split_both_kernel<<<(unsigned)(nblk_a + nblk_b), 256, 0, s>>>(
            (const float*)A, m, k, lda, Ah, Al, (const float*)B, n, ldb, Bh, Bl, kp, nblk_a, a_cblk);
        FB_LAUNCH_CHECK("split_both_kernel");
    }
    // The product as GEMMs over N-column panels of w columns (the row-block path's per-panel
    // GEMM; same per-element arithmetic, bitwise equal).  Each launch re-synchronises the
    // concurrently running tiles in the raster; an in-kernel two-level raster does not help
    // (FB_GEMM_RASTER_PANEL).  Interleaved A/B: 32768^3 320-331 -> 288-295 ms (w = 2048),
    // 32768 x 8192 x 32768 76-78 -> 72 ms, 16384^3 36.0-37.1 -> 34.9 ms, but 8192^3 4.0 -> 4.3-4.4 ms
    // (256 tiles per panel, 3.5 waves: the per-launch tails dominate).  Auto (knob -1): w = 2048
    // when a panel holds >= 6 waves of CTA pairs (m >= ~14100) and n > w; FB_GEMM_NPANEL = w forces.
    int64_t w = knobs().gemm_npanel;
    if (w < 0) w = ((m + 255) / 256) * 8 >= 444 && n > 2048 ? 2048 : 0;
    if (w > 0 && n > w) {
        for (int64_t j0 = 0; j0 < n; j0 += w)
            FB_TRY(gemm_3xtf32_presplit_device(m, std::min(w, n - j0), k, a_raw ? (const float*)A : Ah, Al, kp,
                                               Bh + j0 * kp, Bl + j0 * kp, kp, (float*)C + j0, ldc, s, (float)alpha,
                                               (float)beta, a_raw ? lda : -1));
        return FB_OK;
    }
    return gemm_3xtf32_presplit_device(m, n, k, a_raw ? (const float*)A : Ah, Al, kp, Bh, Bl, kp, (float*)C, ldc, s,
                                       (float)alpha, (float)beta, a_raw ? lda : -1);
}

fb_status tf32_split_device(int transpose, int64_t rows, int64_t cols, const float* X, int64_t ldx, float* hi,
                            float* lo, int64_t ldo, const DeviceState* st, cudaStream_t s, bool trunc_hi) {
    if (!transpose) {
        const int64_t chunks = (cols + 3) / 4;
        dim3 g((unsigned)((chunks + 127) / 128), (unsigned)(rows < 8192 ? rows : 8192));
        tf32::split_rows_kernel<false><<<g, 128, 0, s>>>(X, rows, cols, ldx, hi, lo, ldo);
        FB_LAUNCH_CHECK("split_rows_kernel");
    } else {
        dim3 g2((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
        if (g2.y > 65535) {
            set_error("too many rows for the transposing split grid");
            return FB_ERR_UNSUPPORTED_SIZE;
        }
        if (trunc_hi)
            tf32::split_transpose_kernel<true><<<g2, dim3(32, 8), 0, s>>>(X, rows, cols, ldx, hi, lo, ldo);
        else
            tf32::split_transpose_kernel<false><<<g2, dim3(32, 8), 0, s>>>(X, rows, cols, ldx, hi, lo, ldo);
        FB_LAUNCH_CHECK("split_transpose_kernel");
    }
    return FB_OK;
}

fb_status tf32_lo_device(int64_t rows, int64_t cols, const float* X, int64_t ldx, float* lo, int64_t ldo,
                         cudaStream_t s) {
    const int64_t chunks = (cols + 3) / 4;
    dim3 g((unsigned)((chunks + 127) / 128), (unsigned)(rows < 8192 ? rows : 8192));
    tf32::split_rows_kernel<true><<<g, 128, 0, s>>>(X, rows, cols, ldx, nullptr, lo, ldo);
    FB_LAUNCH_CHECK("split_rows_kernel<lo>");
    return FB_OK;
}

fb_status gemm_3xtf32_presplit_device(int64_t m, int64_t n, int64_t k, const float* Ah, const float* Al,
                                      int64_t lda, const float* Bh, const float* Bl, int64_t ldb, float* C,
                                      int64_t ldc, cudaStream_t s, float alpha, float beta, int64_t lda_hi) {
    CUtensorMap mAh, mAl, mBh, mBl;
    FB_TRY(tf32::make_kmajor_map(&mAh, Ah, m, k, lda_hi >= 0 ? lda_hi : lda, tf32::BM));
    FB_TRY(tf32::make_kmajor_map(&mAl, Al, m, k, lda, tf32::BM));
    FB_TRY(tf32::make_kmajor_map(&mBh, Bh, n, k, ldb, tf32::BN));
    FB_TRY(tf32::make_kmajor_map(&mBl, Bl, n, k, ldb, tf32::BN));
    static std::atomic<int> attr_mask{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const bool one_cta = knobs().gemm_1cta == 1;
    if (!(attr_mask & (1 << (dev & 31)))) {
        FB_CUDA_TRY(cudaFuncSetAttribute(tf32::gemm_3xtf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tf32::SMEM));
        FB_CUDA_TRY(cudaFuncSetAttribute(tf32::pair::gemm_3xtf32_pair_kernel<256>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tf32::pair::SMEM));
        FB_CUDA_TRY(cudaFuncSetAttribute(tf32::pair::gemm_3xtf32_pair_kernel<240>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tf32::pair::SMEM));
        attr_mask |= 1 << (dev & 31);
    }
    if (!one_cta) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int tiles_m = (int)((m + 255) / 256);
        // N of the pair tile: 256, or 240 when that needs fewer (waves x tile width) -- e.g. 2048
        // columns as 9 tiles of 240 put 2048^2 on 72 of the 74 CTA pairs in one wave (knob
        // FB_GEMM_NT = 256 / 240 forces)
        int nt = knobs().gemm_nt;
        if (nt != 240 && nt != 256) {
            auto cost = [&](int64_t t) {
                const int64_t waves = ((int64_t)tiles_m * ((n + t - 1) / t) + sms / 2 - 1) / (sms / 2);
                return waves * t;
            };
            nt = cost(240) < cost(256) ? 240 : 256;
        }
        if (nt == 240) {
            FB_TRY(tf32::make_kmajor_map(&mBh, Bh, n, k, ldb, 120));
            FB_TRY(tf32::make_kmajor_map(&mBl, Bl, n, k, ldb, 120));
        }
        const int tiles_n = (int)((n + nt - 1) / nt);
        const int64_t tiles = (int64_t)tiles_m * tiles_n;
        if (2 * tiles > INT32_MAX) {
            set_error("too many tiles");
            return FB_ERR_UNSUPPORTED_SIZE;
        }
        // persistent (knob FB_GEMM_PERSIST): one CTA pair per two SMs loops over the tiles
        int64_t pairs = tiles;
        if (knobs().gemm_persist) pairs = std::min<int64_t>(tiles, sms / 2);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(2 * pairs));
        cfg.blockDim = dim3(tf32::pair::NUM_THREADS);
        cfg.dynamicSmemBytes = tf32::pair::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (nt == 240)
            FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, tf32::pair::gemm_3xtf32_pair_kernel<240>, mAh, mAl, mBh, mBl, C,
                                           (int)m, (int)n, (int)k, ldc, tiles_m, tiles_n, alpha, beta,
                                           knobs().gemm_raster_panel));
        else
            FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, tf32::pair::gemm_3xtf32_pair_kernel<256>, mAh, mAl, mBh, mBl, C,
                                           (int)m, (int)n, (int)k, ldc, tiles_m, tiles_n, alpha, beta,
                                           knobs().gemm_raster_panel));
        FB_LAUNCH_CHECK("gemm_3xtf32_pair_kernel");
        return FB_OK;
    }
    const int tiles_m = (int)((m + tf32::BM - 1) / tf32::BM);
    const int tiles_n = (int)((n + tf32::BN - 1) / tf32::BN);
    const int64_t tiles = (int64_t)tiles_m * tiles_n;
    if (tiles > INT32_MAX) {
        set_error("too many tiles");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    tf32::gemm_3xtf32_kernel<<<(unsigned)tiles, tf32::NUM_THREADS, tf32::SMEM, s>>>(
        mAh, mAl, mBh, mBl, C, (int)m, (int)n, (int)k, ldc, tiles_m, tiles_n, alpha, beta);
    FB_LAUNCH_CHECK("gemm_3xtf32_kernel");
    return FB_OK;
}

}  // namespace fb
