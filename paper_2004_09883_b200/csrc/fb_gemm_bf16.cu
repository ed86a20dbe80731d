// fb_gemm_bf16.cu -- BF16 GEMM: C[m][n] (FP32) = A[m][k] * B (BF16 operands,
// FP32 accumulation) on the 5th-generation tensor cores, the same CTA-pair design as the 3xTF32
// kernel (fb_gemm.cu): TMA 128B-swizzled K-major tiles -> mbarrier ring -> one thread issues
// tcgen05.mma.cta_group::2.kind::f16 (M = 256, N = 256, K = 16 per instruction) -> double-
// buffered TMEM accumulators drained every 16 k-blocks (1024 k) into RN FP32 registers -> C.  B must be
// K-major ([n][k], i.e. B transposed); a row-major [k][n] B is transposed in the workspace.
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "fb_common.cuh"
#include "fb_ptx.cuh"

#ifndef FB_BF16_GROUP_M
#define FB_BF16_GROUP_M 8  // M tiles per rasterisation group (L2 reuse of the B panels)
#endif

namespace fb {
namespace bf16 {
constexpr int BK = 64;                                   // elements per k-block (128-byte rows)
#ifndef FB_BF16_STAGES
#define FB_BF16_STAGES 6
#endif
constexpr int STAGES = FB_BF16_STAGES;  // 7 (fits 227 KiB) measured slower: 0.796 vs 0.790 ms at 8192^3
constexpr int NUM_THREADS = 320;                         // w0 TMA, w1 MMA/TMEM, w2..9 epilogue
constexpr int NUM_EPI_WARPS = 8;
constexpr uint32_t TILE_BYTES = 128 * BK * 2;            // 16 KiB per operand half
constexpr uint32_t STAGE_BYTES = 2 * TILE_BYTES;         // A half, B half
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t ACC_COLS = 256;
constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;
// k-blocks (of 64) between TMEM drains into RN FP32 registers: every 1024 k (A/B at 8192^3:
// 256 k 0.842 ms, 512 k 0.790 ms, 1024 k 0.785 ms; the truncating TMEM accumulation then
// contributes ~3e-6 relative, inside the 1e-5 bar at any K).
#ifndef FB_BF16_KP
#define FB_BF16_KP 16
#endif
constexpr int KP_BLOCKS = FB_BF16_KP;
constexpr int GROUP_M = FB_BF16_GROUP_M;

__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& tm, int& tn) {
    const int per_group = GROUP_M * tiles_n;
    const int grp = tile / per_group;
    const int first_m = grp * GROUP_M;
    const int gm = min(GROUP_M, tiles_m - first_m);
    const int in = tile - grp * per_group;
    tm = first_m + in % gm;
    tn = in / gm;
}

// CL = 2: one CTA pair per 256 x 256 tile.  CL = 4: a cluster of two pairs computing the tiles
// (m0, n0) and (m0, n0 + 256): the A half-tiles they share are loaded once and multicast to
// both pairs (halving A's L2 -> SM traffic); every stage is released only when both pairs'
// MMAs have consumed it (commits multicast to all four CTAs).
template <int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_bf16_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          float* __restrict__ C, int M, int N, int K, int64_t ldc, int tiles_m, int tiles_n) {
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
    const uint32_t crank = ptx::cluster_ctarank();
    const uint32_t rank = crank & 1u, pair = crank >> 1;
    const bool leader = rank == 0;
    // work units: CL = 2 one 256 x 256 tile per unit, CL = 4 two adjacent tiles; persistent
    // when the grid is smaller than the unit count (A/B knob FB_BF16_PERSIST): the cluster
    // loops over units u = cluster id + k * clusters, the stage ring and the two TMEM
    // accumulators running on across units (the epilogue of one overlaps the next's MMAs)
    const int units = CL == 2 ? tiles_m * tiles_n : tiles_m * ((tiles_n + 1) >> 1);
    const int u0 = (int)(blockIdx.x / CL), ustep = (int)(gridDim.x / CL);
    auto unit_tile = [&](int u, int& m0, int& n0) {
        int tm, tn;
        if (CL == 2) {
            tile_coords(u, tiles_m, tiles_n, tm, tn);
        } else {
            tile_coords(u, tiles_m, (tiles_n + 1) >> 1, tm, tn);
            tn = 2 * tn + (int)pair;
        }
        m0 = tm * 256;
        n0 = tn * 256;
    };
    const uint16_t own_pair_mask = (uint16_t)(0x3u << (2 * pair));
    const uint16_t stage_mask = CL == 2 ? (uint16_t)0x3 : (uint16_t)0xF;
    const int KB = (K + BK - 1) / BK;
    const int NCHUNK = (KB + KP_BLOCKS - 1) / KP_BLOCKS;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), CL / 2);  // one commit per pair of the cluster
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(tfull_bar(b), 1);
            ptx::mbar_init(tempty_bar(b), 2 * NUM_EPI_WARPS);
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
    ptx::pdl_wait();

    if (warp == 0) {
        if (lane == 0) {  // TMA producer (both CTAs): own halves, completion on the leader
            int g = 0;
            for (int u = u0; u < units; u += ustep) {
            int m0, n0;
            unit_tile(u, m0, n0);
            const int am = m0 + 128 * (int)rank, bn = n0 + 128 * (int)rank;
            for (int kb = 0; kb < KB; ++kb, ++g) {
                const int s = g % STAGES;
                const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
                ptx::mbar_wait(empty_bar(s), ph ^ 1u);
                if (leader) ptx::mbar_arrive_expect_tx(full_bar(s), 2 * STAGE_BYTES);
                const uint32_t st = base + s * STAGE_BYTES;
                const int kc = kb * BK;
                if (CL == 2)
                    ptx::tma_load_2d_pair(st, &tmA, full_bar(s), kc, am);
                else if (pair == 0)  // A half `rank` for both pairs (CTAs rank and rank + 2)
                    ptx::tma_load_2d_pair_mc(st, &tmA, full_bar(s), kc, am, (uint16_t)((1u << rank) | (4u << rank)));
                ptx::tma_load_2d_pair(st + TILE_BYTES, &tmB, full_bar(s), kc, bn);
            }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {  // MMA issuer
            // kind::f16 descriptor: D FP32 (bit 4), A BF16 (1 << 7), B BF16 (1 << 10), K-major both,
            // N >> 3 at bit 17, M >> 4 at bit 24
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                                   ((uint32_t)(256 >> 4) << 24);
            int g = 0, cg = 0;
            for (int u = u0; u < units; u += ustep) {
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
                    for (int kk = 0; kk < BK / 16; ++kk) {  // K = 16 per instruction = 32 bytes
                        const uint32_t off = kk * 32;
                        const uint64_t a = ptx::smem_desc_sw128_kmajor(st + off);
                        const uint64_t b = ptx::smem_desc_sw128_kmajor(st + TILE_BYTES + off);
                        ptx::mma_f16_pair(tmem_d, a, b, idesc, (kb > c * KP_BLOCKS || kk > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit_pair(empty_bar(s), stage_mask);
                }
                ptx::mma_commit_pair(tfull_bar(buf), own_pair_mask);
            }
            }
        }
    } else {  // epilogue warps 2..9: lanes 32*(warp%4), column half (warp-2)/4
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        int cg = 0;
        for (int u = u0; u < units; u += ustep) {
        int m0, n0;
        unit_tile(u, m0, n0);
        float acc[128];
#pragma unroll
        for (int j = 0; j < 128; ++j) acc[j] = 0.f;
        for (int c = 0; c < NCHUNK; ++c, ++cg) {
            const int buf = cg & 1;
            ptx::mbar_wait(tfull_bar(buf), (uint32_t)(cg >> 1) & 1u);
            ptx::tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * ACC_COLS + h * 128);
#pragma unroll
            for (int cb = 0; cb < 128; cb += 32) {
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(taddr + (uint32_t)cb, r);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[cb + j] += __uint_as_float(r[j]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_leader(tempty_bar(buf));
        }
        const int row = m0 + 128 * (int)rank + q * 32 + lane;
        const int col0 = n0 + h * 128;
        if (row < M) {
            float* dst = C + (int64_t)row * ldc + col0;
            const int valid = N - col0;
            if (valid >= 128) {
#pragma unroll
                for (int j = 0; j < 128; j += 4)
                    *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 128; ++j)
                    if (j < valid) dst[j] = acc[j];
            }
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

__global__ void __launch_bounds__(256) transpose16_kernel(const uint16_t* __restrict__ X, int64_t rows, int64_t cols,
                                                          int64_t ldx, uint16_t* __restrict__ Y, int64_t ldy) {
    __shared__ uint16_t tile[32][34];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t r = r0 + ty + j, c = c0 + tx;
        if (r < rows && c < cols) tile[ty + j][tx] = X[r * ldx + c];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        const int64_t c = c0 + ty + j, r = r0 + tx;
        if (c < cols && r < rows) Y[c * ldy + r] = tile[tx][ty + j];
    }
}

typedef CUresult (*EncodeTiledFnBF)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static fb_status kmajor_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t K, int64_t ld) {
    static EncodeTiledFnBF enc = nullptr;
    if (!enc) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            set_error("cuTensorMapEncodeTiled unavailable from the driver");
            return FB_ERR_CUDA;
        }
        enc = (EncodeTiledFnBF)f;
    }
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {(cuuint32_t)BK, 128u};
    cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) for a BF16 operand", (int)r);
        return FB_ERR_CUDA;
    }
    return FB_OK;
}
}  // namespace bf16
}  // namespace fb

using namespace fb;

extern "C" {

size_t fb_matmul_bf16_workspace_bytes(int b_transposed, int64_t m, int64_t n, int64_t k) {
    (void)m;
    if (n <= 0 || k <= 0) return 0;
    const int64_t kp = (k + 7) / 8 * 8;
    return b_transposed ? 0 : (size_t)n * (size_t)kp * 2;
}

fb_status fb_matmul_bf16(int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B, int64_t ldb,
                         int b_transposed, void* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    if (m <= 0 || n <= 0 || k <= 0 || m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) {
        set_error("m, n, k must be in [1, 2^31)");
        return FB_ERR_INVALID_VALUE;
    }
    if (!A || !B || !C || (b_transposed != 0 && b_transposed != 1)) {
        set_error("null operand or bad b_transposed flag");
        return FB_ERR_INVALID_VALUE;
    }
    if (lda < k || ldc < n || ldb < (b_transposed ? k : n)) {
        set_error("leading dimensions too small");
        return FB_ERR_INVALID_VALUE;
    }
    if (!aligned16(A) || !aligned16(B) || !aligned16(C) || (lda * 2) % 16 || (ldb * 2) % 16 || (ldc * 4) % 16) {
        set_error("operands must be 16-byte aligned, lda/ldb*2 and ldc*4 multiples of 16");
        return FB_ERR_MISALIGNED;
    }
    const size_t need = fb_matmul_bf16_workspace_bytes(b_transposed, m, n, k);
    if (need && (!ws || ws_bytes < need || !aligned16(ws))) {
        set_error("workspace of %zu bytes required", need);
        return FB_ERR_WORKSPACE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    const void* Bt = B;
    int64_t ldbt = ldb;
    if (!b_transposed) {  // [k][n] -> [n][kp]
        const int64_t kp = (k + 7) / 8 * 8;
        dim3 g((unsigned)((n + 31) / 32), (unsigned)((k + 31) / 32));
        if (g.y > 65535) {
            set_error("k too large for the transpose grid");
            return FB_ERR_UNSUPPORTED_SIZE;
        }
        bf16::transpose16_kernel<<<g, 256, 0, s>>>((const uint16_t*)B, k, n, ldb, (uint16_t*)ws, kp);
        FB_LAUNCH_CHECK("transpose16_kernel");
        Bt = ws;
        ldbt = kp;
    }
    CUtensorMap mA, mB;
    FB_TRY(bf16::kmajor_map(&mA, A, m, k, lda));
    FB_TRY(bf16::kmajor_map(&mB, Bt, n, k, ldbt));
    // A/B knob FB_BF16_CLUSTER=4: two pairs per cluster with the A tiles multicast (correct, but
    // measured slower at 8192^3: 1227 vs 1312 TFLOP/s -- operand traffic is not the limit)
    const int CLn = knobs().bf16_cluster == 4 ? 4 : 2;
    static std::atomic<int> attr_mask{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_mask & (1 << (dev & 31)))) {
        FB_CUDA_TRY(cudaFuncSetAttribute(bf16::gemm_bf16_pair_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bf16::SMEM));
        FB_CUDA_TRY(cudaFuncSetAttribute(bf16::gemm_bf16_pair_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bf16::SMEM));
        attr_mask |= 1 << (dev & 31);
    }
    const int tiles_m = (int)((m + 255) / 256), tiles_n = (int)((n + 255) / 256);
    int64_t ctas = CLn == 2 ? 2 * (int64_t)tiles_m * tiles_n : 4 * (int64_t)tiles_m * ((tiles_n + 1) / 2);
    // persistent (default; knob FB_BF16_PERSIST=0 for one unit per cluster): 8192^3 0.820 ->
    // 0.790 ms, 4096^3 0.145 -> 0.124 ms; the CL = 4 multicast form is slower either way
    if (knobs().bf16_persist && CLn == 2) {  // one cluster per CLn SMs, looping over the work units
        const int64_t cap = (int64_t)(st->sm_count / CLn) * CLn;
        if (ctas > cap) ctas = cap;
    }
    if (ctas > INT32_MAX) {
        set_error("too many tiles");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(bf16::NUM_THREADS);
    cfg.dynamicSmemBytes = bf16::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CLn;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (CLn == 2)
        FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, bf16::gemm_bf16_pair_kernel<2>, mA, mB, (float*)C, (int)m, (int)n, (int)k,
                                       ldc, tiles_m, tiles_n));
    else
        FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, bf16::gemm_bf16_pair_kernel<4>, mA, mB, (float*)C, (int)m, (int)n, (int)k,
                                       ldc, tiles_m, tiles_n));
    FB_LAUNCH_CHECK("gemm_bf16_pair_kernel");
    return FB_OK;
}

}  // extern "C"
