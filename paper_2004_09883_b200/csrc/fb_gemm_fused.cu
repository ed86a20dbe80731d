// fb_gemm_fused.cu -- the FP32 matrix block as ONE
// kernel: C = A B with A [M][K] and B [K][N] row-major FP32, 3xTF32 on tcgen05 tensor cores, no
// operand pre-pass.
//
// Split (G1) inside the kernel.  The tensor core reads an FP32 operand as TF32 by TRUNCATING
// the low 13 mantissa bits (measured: tools/tf32_probe.py, 256/256 rows match trunc, 48 %
// match RN).  So the raw FP32 tile already IS the hi operand, hi = trunc_tf32(x), and only
//     lo = rna_tf32(x - trunc_tf32(x))          (x - hi is exact in FP32)
// has to be formed.  Two converter warps per CTA read the raw A and B tiles that TMA staged
// in shared memory and write the lo tiles at the same byte offsets of a second buffer (the
// operation is elementwise, so the 128-byte swizzle of the TMA layout carries over).  The
// three products hi*hi + hi*lo + lo*hi drop lo*lo: |lo| < 2^-10 |x|, so the dropped term is
// below 2^-20 |a b| per product (about 2^-22 |C| on average), and lo is RN-rounded, so the
// split error is below 2^-21 |x| -- comfortably inside the 1e-5 bar (reading R11).
//
// B is consumed in its natural [K][N] layout as an MN-major UMMA operand (128-byte swizzle with
// 32-byte atoms, 32-column chunks 4 KiB apart), so no transpose either.  The rest follows the CTA-pair kernel
// of fb_gemm.cu: a 256 x 256 tile per CTA pair (tcgen05.mma.cta_group::2.kind::tf32,
// M = 256, N = 256, K = 8), 3-stage TMA ring, two TMEM accumulators, partial sums promoted
// into round-to-nearest FP32 registers every 128 k (the tensor core accumulates with
// truncation, reading R11).
//
// Warps: 0 TMA producer, 1 MMA issuer (leader CTA) + TMEM owner, 2-3 lo converters,
// 4-11 epilogue (TMEM lanes 32 (w % 4) .. +31, column half (w - 4) / 4).
// Barriers per stage s: full[s] (local: TMA bytes landed) -> converters; conv[s] (leader:
// both CTAs' converters done, 2 x 2 warp arrivals) -> MMA issuer; empty[s] (both CTAs: the
// MMAs reading the stage completed, multicast commit) -> producer.
#include <stdint.h>
#include <string.h>

#include "fb_common.cuh"
#include "fb_ptx.cuh"

namespace fb {
namespace fused {

constexpr int BK = 32, STAGES = 3;
constexpr int LO_PANEL_KB = 8;  // lo pre-pass panel: 8 k-blocks = 256 k, one completion flag each
constexpr int NUM_CONV_WARPS = 2, NUM_EPI_WARPS = 8;
// PRE = false: lo formed in shared memory by converter warps 2-3 (epilogue warps 4-11);
// PRE = true: lo tiles come from a streaming pre-pass in global memory (epilogue warps 2-9)
template <bool PRE>
__host__ __device__ constexpr int epi_warp0() { return PRE ? 2 : 4; }
template <bool PRE>
__host__ __device__ constexpr int num_threads() { return 32 * (epi_warp0<PRE>() + NUM_EPI_WARPS); }
constexpr uint32_t TILE_BYTES = 128 * BK * 4;                 // 16 KiB (A: 128 x 32, B: 32 x 128)
constexpr uint32_t STAGE_BYTES = 4 * TILE_BYTES;              // A raw, A lo, B raw, B lo
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t ACC_COLS = 256;
constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;
constexpr int KP_BLOCKS = 4;  // RN promotion every 4 x 32 = 128 k
constexpr int GROUP_M = 8;

__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& tm, int& tn) {
    const int per_group = GROUP_M * tiles_n;
    const int grp = tile / per_group;
    const int first_m = grp * GROUP_M;
    const int gm = min(GROUP_M, tiles_m - first_m);
    const int in = tile - grp * per_group;
    tm = first_m + in % gm;
    tn = in / gm;
}

// MN-major TF32 operand.  The only MN-major shared-memory layout UMMA accepts for 32-bit types
// is "128-byte swizzle with 32-byte atomicity" (layout type 1, SWIZZLE_128B_BASE32B; TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): atoms of 32 MN elements (128 B) x 4 k rows, so
// LBO = distance between 32-element MN chunks (4 KiB here: each chunk is a [32 k][32 n] TMA
// box) and SBO = distance between 4-row k groups (512 B).  Verified on the GPU against the
// other candidate encodings (tools/experiments/dbg_gemm.py: only this one reproduces A B).
__device__ __forceinline__ uint64_t smem_desc_mnmajor_sw128b32(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(4096 >> 4) << 16;  // LBO
    d |= (uint64_t)(512 >> 4) << 32;   // SBO
    d |= (uint64_t)1 << 46;            // version 1 (sm_100)
    d |= (uint64_t)1 << 61;            // SWIZZLE_128B_BASE32B
    return d;
}

// arrive (release at cluster scope) on the mbarrier at the same offset in CTA 0 of the pair
__device__ __forceinline__ void mbar_arrive_leader_release(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar & ptx::kPeerBitMask)
                 : "memory");
}

// lo = rna_tf32(x - trunc_tf32(x)), low 13 bits zero (the tensor core's truncation is then
// exact).  rna on the sign-magnitude encoding: add half an ulp of TF32 (bit 12) to the
// magnitude bits, then clear the low 13 -- ties away from zero, as cvt.rna.tf32.f32, in two
// integer ops instead of the conversion instruction.
__device__ __forceinline__ float lo_of(float x) {
    const float r = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);  // exact
    return __uint_as_float((__float_as_uint(r) + 0x1000u) & 0xFFFFE000u);
}
// Stream-K schedule (deterministic).  The U = tiles x KB k-block units are split evenly over the
// P CTA pairs of the grid (pair p owns units [p U / P, (p+1) U / P)), so all 148 SMs stay busy
// even when the tile count is not a multiple of 74 (2048^3: 64 tiles -> 64 of 74 pairs).  A
// pair's range cuts into pieces at tile boundaries:
//   full     -- a whole tile: written to C;
//   writer   -- ends inside a tile (only a pair's last piece): partial sum to the pair's
//               workspace slot, then a flag (count of finished epilogue warps);
//   finisher -- contains a tile's last k-block but not its first: waits for the writers of the
//               earlier k-blocks (pairs p-1, p-2, ...), adds their slots in that fixed order and
//               writes C -- bitwise reproducible.
// The writer piece is processed first, so no finisher waits on a pair that is itself waiting.
struct Piece {
    int tile, kb0, kb1, kind;  // kind: 0 full, 1 writer, 2 finisher
};
__device__ __forceinline__ int64_t pair_u0(int p, int P, int64_t U) { return (int64_t)p * U / P; }
__device__ __forceinline__ int num_pieces(int p, int P, int64_t U, int KB) {
    const int64_t u0 = pair_u0(p, P, U), u1 = pair_u0(p + 1, P, U);
    return u1 > u0 ? (int)((u1 - 1) / KB - u0 / KB) + 1 : 0;
}
__device__ __forceinline__ Piece get_piece(int i, int p, int P, int64_t U, int KB) {
    const int64_t u0 = pair_u0(p, P, U), u1 = pair_u0(p + 1, P, U);
    const int t_first = (int)(u0 / KB), t_last = (int)((u1 - 1) / KB);
    const bool has_writer = (u1 % KB) != 0;
    int t;
    if (has_writer)
        t = (i == 0) ? t_last : t_first + i - 1;
    else
        t = t_first + i;
    Piece pc;
    pc.tile = t;
    const int64_t tb = (int64_t)t * KB;
    pc.kb0 = (int)((u0 > tb ? u0 : tb) - tb);
    pc.kb1 = (int)((u1 < tb + KB ? u1 : tb + KB) - tb);
    pc.kind = (pc.kb1 < KB) ? 1 : (pc.kb0 > 0 ? 2 : 0);
    return pc;
}

#ifndef FB_GEMM_FUSED_NOCONV
#define FB_GEMM_FUSED_NOCONV 0  // timing experiment only: skip forming lo (wrong results)
#endif

template <bool PRE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(num_threads<PRE>(), 1)
    gemm_3xtf32_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmAl, const __grid_constant__ CUtensorMap tmBl,
                             float* __restrict__ C, int M, int N, int K, int64_t ldc, int tiles_m, int tiles_n,
                             float* __restrict__ partials, unsigned int* __restrict__ flags,
                             const unsigned int* __restrict__ pflags, unsigned int pflag_target) {
    constexpr int EPI_WARP0 = epi_warp0<PRE>();
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_u32 + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_u32);
    const uint32_t bar_base = base + STAGES * STAGE_BYTES;
    auto full_bar = [&](int s) { return bar_base + 8u * s; };
    auto empty_bar = [&](int s) { return bar_base + 8u * (STAGES + s); };
    auto conv_bar = [&](int s) { return bar_base + 8u * (2 * STAGES + s); };
    auto tfull_bar = [&](int b) { return bar_base + 8u * (3 * STAGES + b); };
    auto tempty_bar = [&](int b) { return bar_base + 8u * (3 * STAGES + 2 + b); };
    const uint32_t tmem_slot = bar_base + 8u * (3 * STAGES + 4);
    const uint32_t* tmem_slot_ptr =
        reinterpret_cast<const uint32_t*>(smem + STAGES * STAGE_BYTES + 8 * (3 * STAGES + 4));
    // stage layout: [A raw][A lo][B raw][B lo]
    auto a_raw = [&](int s) { return base + s * STAGE_BYTES; };
    auto a_lo = [&](int s) { return base + s * STAGE_BYTES + TILE_BYTES; };
    auto b_raw = [&](int s) { return base + s * STAGE_BYTES + 2 * TILE_BYTES; };
    auto b_lo = [&](int s) { return base + s * STAGE_BYTES + 3 * TILE_BYTES; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int KB = (K + BK - 1) / BK;
    const int pair = (int)(blockIdx.x >> 1), P = (int)(gridDim.x >> 1);
    const int64_t U = (int64_t)tiles_m * tiles_n * KB;
    const int npc = num_pieces(pair, P, U, KB);

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        if constexpr (PRE) {
            ptx::tma_prefetch_desc(&tmAl);
            ptx::tma_prefetch_desc(&tmBl);
        }
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
            ptx::mbar_init(conv_bar(s), 2 * NUM_CONV_WARPS);  // both CTAs' converter warps
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
    // PDL: A and B are complete (the setup above overlapped the previous kernel).  With panel
    // flags (pflags) the kernel instead overlaps the lo pre-pass: the producer waits for each
    // K panel's flag before loading from it (the pre-pass itself waited for the previous kernel).
    if (!pflags) ptx::pdl_wait();

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer: this CTA's A rows and B columns, raw FP32
            int g = 0;  // k-blocks issued so far (stage ring position)
            uint32_t panels_ready = 0;  // K panels (LO_PANEL_KB k-blocks each) seen complete
            for (int ip = 0; ip < npc; ++ip) {
            const Piece pc = get_piece(ip, pair, P, U, KB);
            int tm, tn;
            tile_coords(pc.tile, tiles_m, tiles_n, tm, tn);
            const int am = tm * 256 + 128 * (int)rank, bn = tn * 256 + 128 * (int)rank;
            for (int kb = pc.kb0; kb < pc.kb1; ++kb, ++g) {
                const int s = g % STAGES;
                const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
                ptx::mbar_wait(empty_bar(s), ph ^ 1u);
                const int kc = kb * BK;
                if (pflags) {
                    const uint32_t pnl = (uint32_t)(kb / LO_PANEL_KB);
                    while (panels_ready <= pnl) {  // panels complete in order, mostly
                        uint32_t v;
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(pflags + pnl) : "memory");
                        if (v >= pflag_target) {
                            panels_ready = pnl + 1;
                            break;
                        }
                        __nanosleep(64);
                    }
                }
                if constexpr (PRE) {
                    // all four tiles; both CTAs' bytes complete on the leader's full barrier
                    if (leader) ptx::mbar_arrive_expect_tx(full_bar(s), 2 * STAGE_BYTES);
                    ptx::tma_load_2d_pair(a_raw(s), &tmA, full_bar(s), kc, am);
                    ptx::tma_load_2d_pair(a_lo(s), &tmAl, full_bar(s), kc, am);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        ptx::tma_load_2d_pair(b_raw(s) + j * 4096, &tmB, full_bar(s), bn + 32 * j, kc);
                        ptx::tma_load_2d_pair(b_lo(s) + j * 4096, &tmBl, full_bar(s), bn + 32 * j, kc);
                    }
                } else {
                    ptx::mbar_arrive_expect_tx(full_bar(s), 2 * TILE_BYTES);
                    ptx::tma_load_2d(a_raw(s), &tmA, full_bar(s), kc, am);
#pragma unroll
                    for (int j = 0; j < 4; ++j)  // four 32-column chunks of 32 k rows (4 KiB each)
                        ptx::tma_load_2d(b_raw(s) + j * 4096, &tmB, full_bar(s), bn + 32 * j, kc);
                }
            }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            // ---------------- MMA issuer (leader CTA, single thread)
            // D f32, A/B tf32, A K-major, B MN-major (bit 16), N = 256, M = 256
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(256 >> 3) << 17) |
                                   ((uint32_t)(256 >> 4) << 24);
            int g = 0, c = 0;  // k-blocks consumed, chunks issued
            for (int ip = 0; ip < npc; ++ip) {
            const Piece pc = get_piece(ip, pair, P, U, KB);
            for (int c0 = pc.kb0; c0 < pc.kb1; c0 += KP_BLOCKS, ++c) {
                const int buf = c & 1;
                ptx::mbar_wait(tempty_bar(buf), ((uint32_t)(c >> 1) & 1u) ^ 1u);
                ptx::tc_fence_after();
                const uint32_t tmem_d = tmem_base + (uint32_t)(buf * ACC_COLS);
                const int kb_end = min(pc.kb1, c0 + KP_BLOCKS);
                for (int kb = c0; kb < kb_end; ++kb, ++g) {
                    const int s = g % STAGES;
                    const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
                    ptx::mbar_wait(PRE ? full_bar(s) : conv_bar(s), ph);
                    ptx::tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < BK / 8; ++kk) {
                        const uint64_t ah = ptx::smem_desc_sw128_kmajor(a_raw(s) + kk * 32);
                        const uint64_t al = ptx::smem_desc_sw128_kmajor(a_lo(s) + kk * 32);
                        const uint64_t bh = smem_desc_mnmajor_sw128b32(b_raw(s) + kk * 1024);
                        const uint64_t bl = smem_desc_mnmajor_sw128b32(b_lo(s) + kk * 1024);
                        const uint32_t acc0 = (kb > c0 || kk > 0) ? 1u : 0u;
                        ptx::mma_tf32_pair(tmem_d, al, bh, idesc, acc0);  // small terms first
                        ptx::mma_tf32_pair(tmem_d, ah, bl, idesc, 1u);
                        ptx::mma_tf32_pair(tmem_d, ah, bh, idesc, 1u);
                    }
                    ptx::mma_commit_pair(empty_bar(s), 0x3);  // frees the stage in both CTAs
                }
                ptx::mma_commit_pair(tfull_bar(buf), 0x3);    // partial sum ready in both CTAs
            }
            }
        }
    } else if (!PRE && warp < EPI_WARP0) {
        // ---------------- lo converters: raw tiles -> lo tiles (elementwise, same offsets)
        const int ct = (warp - 2) * 32 + lane;  // 0 .. 63
        int nkb = 0;
        for (int ip = 0; ip < npc; ++ip) {
            const Piece pc = get_piece(ip, pair, P, U, KB);
            nkb += pc.kb1 - pc.kb0;
        }
        for (int g = 0; g < nkb; ++g) {
            const int s = g % STAGES;
            const uint32_t ph = (uint32_t)(g / STAGES) & 1u;
            ptx::mbar_wait(full_bar(s), ph);
            const float4* ra = reinterpret_cast<const float4*>(smem + s * STAGE_BYTES);
            float4* la = reinterpret_cast<float4*>(smem + s * STAGE_BYTES + TILE_BYTES);
            const float4* rb = reinterpret_cast<const float4*>(smem + s * STAGE_BYTES + 2 * TILE_BYTES);
            float4* lb = reinterpret_cast<float4*>(smem + s * STAGE_BYTES + 3 * TILE_BYTES);
            constexpr int NV = TILE_BYTES / 16;  // 1024 float4 per tile
#pragma unroll 4
            for (int i = ct; i < (FB_GEMM_FUSED_NOCONV ? 0 : NV); i += 32 * NUM_CONV_WARPS) {
                const float4 x = ra[i], y = rb[i];
                la[i] = make_float4(lo_of(x.x), lo_of(x.y), lo_of(x.z), lo_of(x.w));
                lb[i] = make_float4(lo_of(y.x), lo_of(y.y), lo_of(y.z), lo_of(y.w));
            }
            ptx::fence_proxy_async_smem();  // generic-proxy lo writes -> visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive_leader_release(conv_bar(s));
        }
    } else {
        // ---------------- epilogue warps (EPI_WARP0 ..): TMEM lanes 32 (w % 4), column half
        const int q = warp & 3;
        const int h = (warp - EPI_WARP0) >> 2;
        const int lrow = 128 * (int)rank + q * 32 + lane;  // row of the 256 x 256 tile
        int c = 0;
        for (int ip = 0; ip < npc; ++ip) {
            const Piece pc = get_piece(ip, pair, P, U, KB);
            float acc[128];
#pragma unroll
            for (int j = 0; j < 128; ++j) acc[j] = 0.f;
            for (int c0 = pc.kb0; c0 < pc.kb1; c0 += KP_BLOCKS, ++c) {
                const int buf = c & 1;
                ptx::mbar_wait(tfull_bar(buf), (uint32_t)(c >> 1) & 1u);
                ptx::tc_fence_after();
                const uint32_t taddr =
                    tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * ACC_COLS + h * 128);
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
            if (pc.kind == 1) {
                // writer: partial sum to this pair's slot, then count this warp in the flag
                float* dst = partials + (int64_t)pair * 65536 + lrow * 256 + h * 128;
#pragma unroll
                for (int j = 0; j < 128; j += 4)
                    *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicAdd(flags + pair, 1u);
                continue;
            }
            if (pc.kind == 2) {
                // finisher: add the writers of k-blocks [0, kb0) of this tile, pair p-1 first
                const int64_t tstart = (int64_t)pc.tile * KB;
                for (int w = pair - 1; w >= 0 && pair_u0(w + 1, P, U) > tstart; --w) {
                    if (lane == 0) {
                        unsigned int v;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + w) : "memory");
                        } while (v < 2u * NUM_EPI_WARPS);
                    }
                    __syncwarp();
                    const float* src = partials + (int64_t)w * 65536 + lrow * 256 + h * 128;
#pragma unroll
                    for (int j = 0; j < 128; j += 4) {
                        const float4 v4 = __ldcg(reinterpret_cast<const float4*>(src + j));
                        acc[j] += v4.x;
                        acc[j + 1] += v4.y;
                        acc[j + 2] += v4.z;
                        acc[j + 3] += v4.w;
                    }
                    if (pair_u0(w, P, U) <= tstart) break;  // w's range holds the tile's first k-block
                }
            }
            int tm, tn;
            tile_coords(pc.tile, tiles_m, tiles_n, tm, tn);
            const int row = tm * 256 + lrow;
            const int col0 = tn * 256 + h * 128;
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

typedef CUresult (*EncodeTiledFnF)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFnF encoder() {
    static EncodeTiledFnF fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFnF)p;
    }
    return fn;
}

// 2D FP32 map {inner, outer} with row pitch ld (elements), box {32, box_outer}, 128B swizzle;
// out-of-range elements read as zero (ragged M, N, K)
static fb_status make_map(CUtensorMap* map, const float* ptr, int64_t inner, int64_t outer, int64_t ld,
                          uint32_t box_outer, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiledFnF enc = encoder();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return FB_ERR_CUDA;
    }
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {32u, box_outer};
    cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)ptr, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) for the fused FP32 GEMM", (int)r);
        return FB_ERR_CUDA;
    }
    return FB_OK;
}

}  // namespace fused

namespace fused {
// lo pre-pass, both operands in one launch: lo[r][c] = lo_of(x[r][c]) for A (m x k, pitches
// lda -> kp) in blocks [0, nblk_a) and B (k x n, ldb -> np) in the rest; each thread moves
// LO_UNROLL float4 per iteration with every load issued before the first store (memory-level
// parallelism: one float4 per thread in flight left the pass latency-bound at ~4 TB/s).
constexpr int LO_UNROLL = 4;
__device__ __forceinline__ void lo_part(const float* __restrict__ X, int64_t rows, int64_t cols, int64_t ldx,
                                        float* __restrict__ L, int64_t ldl, int64_t blk, int64_t nblk) {
    const int64_t c4 = (cols + 3) / 4;
    const int64_t total = rows * c4;
    const int64_t stride = nblk * blockDim.x;
    for (int64_t e0 = blk * blockDim.x + threadIdx.x; e0 < total; e0 += stride * LO_UNROLL) {
        float4 v[LO_UNROLL];
        int64_t r[LO_UNROLL], c[LO_UNROLL];
#pragma unroll
        for (int u = 0; u < LO_UNROLL; ++u) {
            const int64_t e = e0 + u * stride;
            r[u] = e / c4;
            c[u] = (e - r[u] * c4) * 4;
            if (e < total) v[u] = __ldcs(reinterpret_cast<const float4*>(X + r[u] * ldx + c[u]));
        }
#pragma unroll
        for (int u = 0; u < LO_UNROLL; ++u)
            if (e0 + u * stride < total)
                *reinterpret_cast<float4*>(L + r[u] * ldl + c[u]) =
                    make_float4(lo_of(v[u].x), lo_of(v[u].y), lo_of(v[u].z), lo_of(v[u].w));
    }
}
// Panel-ordered lo pre-pass for the overlapped form: one block per SM (so that every block is
// resident at once and the GEMM, launched when all of them have started, fits beside them),
// walking the K panels in order; each block does its strided share of panel p
// (A[:, panel] and B[panel, :]) and then counts itself in pflags[p] (target: gridDim.x).
__global__ void __launch_bounds__(256) lo_panel_kernel(const float* __restrict__ A, int64_t m, int64_t k, int64_t lda,
                                                       float* __restrict__ Al, int64_t kp, const float* __restrict__ B,
                                                       int64_t n, int64_t ldb, float* __restrict__ Bl, int64_t np,
                                                       int npanels, unsigned int* __restrict__ pflags) {
    ptx::pdl_launch_dependents();  // the GEMM may start now; it waits on pflags instead
    ptx::pdl_wait();               // A and B are complete
    constexpr int PK = LO_PANEL_KB * BK;  // k per panel (multiple of 4)
    const int64_t n4 = (n + 3) / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int pnl = 0; pnl < npanels; ++pnl) {
        const int64_t k0 = (int64_t)pnl * PK;
        const int64_t kw = (k - k0) < PK ? (k - k0) : PK;
        const int64_t a4 = (kw + 3) / 4;
        const int64_t wa = m * a4, total = wa + kw * n4;
        for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += stride * LO_UNROLL) {
            float4 v[LO_UNROLL];
            float* dst[LO_UNROLL];
#pragma unroll
            for (int u = 0; u < LO_UNROLL; ++u) {
                const int64_t e = e0 + u * stride;
                dst[u] = nullptr;
                if (e < total) {
                    const float* src;
                    if (e < wa) {
                        const int64_t r = e / a4, c = k0 + (e - r * a4) * 4;
                        src = A + r * lda + c;
                        dst[u] = Al + r * kp + c;
                    } else {
                        const int64_t eb = e - wa;
                        const int64_t r = k0 + eb / n4, c = (eb % n4) * 4;
                        src = B + r * ldb + c;
                        dst[u] = Bl + r * np + c;
                    }
                    v[u] = __ldcs(reinterpret_cast<const float4*>(src));
                }
            }
#pragma unroll
            for (int u = 0; u < LO_UNROLL; ++u)
                if (dst[u])
                    *reinterpret_cast<float4*>(dst[u]) =
                        make_float4(lo_of(v[u].x), lo_of(v[u].y), lo_of(v[u].z), lo_of(v[u].w));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(pflags + pnl, 1u);
        }
    }
}

__global__ void __launch_bounds__(256) lo_kernel(const float* __restrict__ A, int64_t m, int64_t k, int64_t lda,
                                                 float* __restrict__ Al, int64_t kp, const float* __restrict__ B,
                                                 int64_t n, int64_t ldb, float* __restrict__ Bl, int64_t np,
                                                 int64_t nblk_a, unsigned int* __restrict__ flags, int nflags) {
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    if (blockIdx.x == 0)  // the stream-K flags of the GEMM that follows start at zero
        for (int i = threadIdx.x; i < nflags; i += blockDim.x) flags[i] = 0u;
    if ((int64_t)blockIdx.x < nblk_a)
        lo_part(A, m, k, lda, Al, kp, blockIdx.x, nblk_a);
    else
        lo_part(B, k, n, ldb, Bl, np, blockIdx.x - nblk_a, gridDim.x - nblk_a);
}
template <bool PRE>
static fb_status launch(const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mAl, const CUtensorMap& mBl,
                        int64_t m, int64_t n, int64_t k, float* C, int64_t ldc, int pairs, float* partials,
                        unsigned int* flags, cudaStream_t s, const unsigned int* pflags = nullptr,
                        unsigned int pflag_target = 0) {
    static DevOnce once;
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(gemm_3xtf32_fused_kernel<PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM));
        once.set(dev);
    }
    const int tiles_m = (int)((m + 255) / 256);
    const int tiles_n = (int)((n + 255) / 256);
    const int64_t tiles = (int64_t)tiles_m * tiles_n;
    if (2 * tiles > INT32_MAX) {
        set_error("too many tiles");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * (pairs > 0 ? pairs : tiles)));
    cfg.blockDim = dim3(num_threads<PRE>());
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_3xtf32_fused_kernel<PRE>, mA, mB, mAl, mBl, C, (int)m, (int)n, (int)k,
                                   ldc, tiles_m, tiles_n, partials, flags, pflags, pflag_target));
    FB_LAUNCH_CHECK("gemm_3xtf32_fused_kernel");
    return FB_OK;
}
}  // namespace fused

// stream-K pairs: at most kMaxPairs (one per two SMs; B200: 74), never more than k-block units
constexpr int kMaxPairs = 80;
static int64_t sk_units(int64_t m, int64_t n, int64_t k) {
    return ((m + 255) / 256) * ((n + 255) / 256) * ((k + fused::BK - 1) / fused::BK);
}
struct FusedWs {
    size_t al, bl, part, flags, total;
};
static FusedWs fused_ws_layout(int64_t m, int64_t n, int64_t k) {
    const int64_t kp = (k + 3) / 4 * 4, np = (n + 3) / 4 * 4;
    const int64_t pmax = sk_units(m, n, k) < kMaxPairs ? sk_units(m, n, k) : kMaxPairs;
    FusedWs w;
    w.al = 0;
    w.bl = ((size_t)(m * kp) * 4 + 255) & ~(size_t)255;
    w.part = w.bl + (((size_t)(k * np) * 4 + 255) & ~(size_t)255);
    w.flags = w.part + (size_t)pmax * 65536 * 4;
    const int64_t npanels = ((k + fused::BK - 1) / fused::BK + fused::LO_PANEL_KB - 1) / fused::LO_PANEL_KB;
    w.total = w.flags + (size_t)(kMaxPairs + npanels) * 4 + 256;
    return w;
}
size_t gemm_3xtf32_fused_ws_bytes(int64_t m, int64_t n, int64_t k) { return fused_ws_layout(m, n, k).total; }

// C = A B.  With a workspace of gemm_3xtf32_fused_ws_bytes (and knob FB_GEMM_LO_PREPASS != 0)
// the lo operands are formed by one streaming pre-pass (Al [m][kp], Bl [k][np] in the
// operands' own layouts) and the kernel streams four tiles per stage; without one, the
// kernel's converter warps form them in shared memory.
fb_status gemm_3xtf32_fused_device(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                                   int64_t ldb, float* C, int64_t ldc, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) {
        set_error("dimension exceeds int32");
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    CUtensorMap mA, mB, mAl, mBl;
    FB_TRY(fused::make_map(&mA, A, k, m, lda, 128u));  // K-major A: box 32 k x 128 rows
    FB_TRY(fused::make_map(&mB, B, n, k, ldb, 32u,  // MN-major B: box 32 n x 32 k, 32-byte swizzle atoms
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
    const bool pre = knobs().gemm_lo_prepass != 0 && ws && ws_bytes >= gemm_3xtf32_fused_ws_bytes(m, n, k);
    if (!pre) return fused::launch<false>(mA, mB, mA, mB, m, n, k, C, ldc, 0, nullptr, nullptr, s);
    const int64_t kp = (k + 3) / 4 * 4, np = (n + 3) / 4 * 4;
    const FusedWs L = fused_ws_layout(m, n, k);
    char* w0 = (char*)(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float* Al = (float*)(w0 + L.al);
    float* Bl = (float*)(w0 + L.bl);
    float* partials = (float*)(w0 + L.part);
    unsigned int* flags = (unsigned int*)(w0 + L.flags);
    DeviceState* st = nullptr;
    FB_TRY(ensure_device(nullptr, &st));
    int64_t pairs = st->sm_count / 2;
    if (knobs().gemm_streamk == 0) pairs = 0;  // A/B knob: one pair per tile (classic grid)
    if (pairs > kMaxPairs) pairs = kMaxPairs;
    if (pairs > sk_units(m, n, k)) pairs = sk_units(m, n, k);
    FB_TRY(fused::make_map(&mAl, Al, k, m, kp, 128u));
    FB_TRY(fused::make_map(&mBl, Bl, n, k, np, 32u, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
    if (knobs().gemm_lo_overlap) {
        // the lo pre-pass in K panels, overlapped with the GEMM: the kernel's producer waits on
        // each panel's flag (zeroed here together with the stream-K flags) instead of PDL-waiting
        // for the whole pre-pass
        const int64_t npanels = ((k + fused::BK - 1) / fused::BK + fused::LO_PANEL_KB - 1) / fused::LO_PANEL_KB;
        unsigned int* pflags = flags + kMaxPairs;
        FB_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)(kMaxPairs + npanels) * 4, s));
        const int grid = st->sm_count;  // one block per SM: all resident, beside the GEMM's CTAs
        fused::lo_panel_kernel<<<grid, 256, 0, s>>>(A, m, k, lda, Al, kp, B, n, ldb, Bl, np, (int)npanels, pflags);
        FB_LAUNCH_CHECK("lo_panel_kernel");
        return fused::launch<true>(mA, mB, mAl, mBl, m, n, k, C, ldc, (int)pairs, partials, flags, s, pflags,
                                   (unsigned int)grid);
    }
    const int64_t wa = m * (kp / 4), wb = k * (np / 4);
    int64_t blocks = (wa + wb + 256 * fused::LO_UNROLL - 1) / (256 * fused::LO_UNROLL);
    if (blocks > (int64_t)st->sm_count * 8) blocks = (int64_t)st->sm_count * 8;
    if (blocks < 2) blocks = 2;
    int64_t ba = (blocks * wa + (wa + wb) / 2) / (wa + wb);
    if (ba < 1) ba = 1;
    if (ba > blocks - 1) ba = blocks - 1;
    fused::lo_kernel<<<(unsigned)blocks, 256, 0, s>>>(A, m, k, lda, Al, kp, B, n, ldb, Bl, np, ba, flags, kMaxPairs);
    FB_LAUNCH_CHECK("lo_kernel");
    return fused::launch<true>(mA, mB, mAl, mBl, m, n, k, C, ldc, (int)pairs, partials, flags, s);
}

}  // namespace fb
