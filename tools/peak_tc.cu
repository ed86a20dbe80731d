// peak_tc.cu -- SURVEY K8: measured tensor-core peaks on this B200 (the roofline denominators of
// the GEMM blocks).  Not product code.
//
//   tf32_1cta : tcgen05.mma.cta_group::1.kind::tf32, M=128 N=256 K=8 per instruction, one CTA per
//               SM, a single thread issuing back-to-back MMAs on smem operands (zeros) into TMEM
//   tf32_pair : tcgen05.mma.cta_group::2.kind::tf32, M=256 N=256 K=8, one CTA pair per 2 SMs (the
//               shape of fb_matmul's FP32 kernel)
//   f64_dmma  : mma.sync.aligned.m16n8k8.row.col.f64 (DMMA), 8 warps per SM, 4 independent
//               accumulators per warp (the FP64 kernel's instruction)
// Each kernel runs `iters` rounds; the host times the whole grid with CUDA events ("burst": one
// short launch; "sustained": back-to-back launches for ~2 s) and prints one JSON line per case.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2004_09883_b200/csrc \
//        -o tools/bin/peak_tc tools/peak_tc.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "fb_ptx.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
using namespace fb;

constexpr uint32_t A_BYTES = 128 * 128;  // 128 rows x 128 B (32 tf32): one swizzle-128 K-major tile
constexpr uint32_t B_BYTES = 256 * 128;
constexpr size_t SMEM = A_BYTES + B_BYTES + 1024 + 64;

// idesc: D f32 (bit 4), A/B tf32 (2 << 7, 2 << 10), K-major both, N >> 3 at 17, M >> 4 at 24
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int PAIR>
__global__ void __launch_bounds__(128, 1) tf32_peak_kernel(int iters, unsigned long long* cycles, int data) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    const uint32_t base = (ptx::smem_u32(sm_raw) + 1023) & ~1023u;
    unsigned char* basep = sm_raw + (base - ptx::smem_u32(sm_raw));
    uint64_t* bar = reinterpret_cast<uint64_t*>(basep + A_BYTES + B_BYTES);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // operands: zeros, or (data != 0) TF32-exact values in [-1, 1) from an index hash -- the
    // tensor cores' power (and so the sustained clock under the 1 kW cap) depends on the data
    for (int i = threadIdx.x; i < (int)(A_BYTES + B_BYTES) / 4; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 40503u;
        h ^= h >> 15;
        h *= 2246822519u;
        h ^= h >> 13;
        const float v = data ? ((float)(h >> 9) * (1.0f / 8388608.0f) * 2.0f - 1.0f) : 0.0f;
        reinterpret_cast<uint32_t*>(basep)[i] = __float_as_uint(v) & 0xffffe000u;
    }
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(bar), 1);
        ptx::fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 1) {
        if (PAIR) {
            ptx::tmem_alloc_pair(ptx::smem_u32(tslot), 256);
            ptx::tmem_relinquish_pair();
        } else {
            ptx::tmem_alloc(ptx::smem_u32(tslot), 256);
            ptx::tmem_relinquish();
        }
    }
    ptx::tc_fence_before();
    if (PAIR) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    if (warp == 1 && lane == 0 && rank == 0) {
        const uint32_t idesc = tf32_idesc(PAIR ? 256 : 128, 256);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t a = ptx::smem_desc_sw128_kmajor(base + kk * 32);
                const uint64_t b = ptx::smem_desc_sw128_kmajor(base + A_BYTES + kk * 32);
                if (PAIR)
                    ptx::mma_tf32_pair(tmem, a, b, idesc, (it | kk) ? 1u : 0u);
                else
                    ptx::mma_tf32(tmem, a, b, idesc, (it | kk) ? 1u : 0u);
            }
        }
        if (PAIR)
            ptx::mma_commit_pair(ptx::smem_u32(bar), 0x1);
        else
            ptx::mma_commit(ptx::smem_u32(bar));
        ptx::mbar_wait(ptx::smem_u32(bar), 0);
        const long long t1 = clock64();
        if (cycles && blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
    }
    ptx::tc_fence_before();
    if (PAIR) ptx::cluster_sync(); else __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        if (PAIR) ptx::tmem_dealloc_pair(tmem, 256); else ptx::tmem_dealloc(tmem, 256);
    }
}

__device__ __forceinline__ void dmma(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 "
        "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

__global__ void __launch_bounds__(256) f64_peak_kernel(int iters, double* out) {
    double a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0.5 + 1e-3 * (threadIdx.x + i);
    b[0] = 0.25;
    b[1] = -0.125;
    double d[4][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(d[j], a, b);
    }
    double s = 0;
    for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) s += d[j][i];
    if (s == 1.2345) out[0] = s;
}

template <typename F>
static double time_us(F launch, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    CK(cudaGetLastError());
    return 1e3 * ms / reps;
}

int main(int argc, char** argv) {
    const double sustain_s = argc > 1 ? atof(argv[1]) : 2.0;
    int sms = 0, clk_khz = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    unsigned long long* dcyc;
    double* dout;
    CK(cudaMalloc(&dcyc, 8));
    CK(cudaMalloc(&dout, 8));
    CK(cudaFuncSetAttribute(tf32_peak_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    CK(cudaFuncSetAttribute(tf32_peak_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));

    // ---- TF32, one CTA per SM (M=128)
    for (int cs = 0; cs < 4; ++cs) {
        const int pair = cs & 1, data = cs >> 1;
        const int iters = 4096;
        const double flop_per_cta = 2.0 * (pair ? 128 : 128) * 256 * 8 * 4 * iters;  // per SM (pair: M/2 rows each)
        auto launch = [&]() {
            if (pair) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = sms;
                cfg.blockDim = 128;
                cfg.dynamicSmemBytes = SMEM;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 2;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                CK(cudaLaunchKernelEx(&cfg, tf32_peak_kernel<1>, iters, dcyc, data));
            } else {
                tf32_peak_kernel<0><<<sms, 128, SMEM>>>(iters, dcyc, data);
            }
        };
        const double us = time_us(launch, 5);
        unsigned long long cyc = 0;
        CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
        const double tf = flop_per_cta * sms / (us * 1e-6) / 1e12;
        const double fpc = flop_per_cta / (double)cyc;  // flop per cycle per SM (issuing SM's clock)
        const int nsus = (int)(sustain_s / (us * 1e-6)) + 1;
        const double us_s = time_us(launch, nsus);
        printf("{\"case\": \"%s%s\", \"tflops_burst\": %.1f, \"tflops_sustained\": %.1f, \"flop_per_clk_per_sm\": %.0f, "
               "\"mma_cycles\": %llu, \"iters\": %d, \"sms\": %d, \"launch_us\": %.2f, \"sustained_launches\": %d}\n",
               pair ? "tf32_pair_m256n256k8" : "tf32_1cta_m128n256k8", data ? "_data" : "_zeros", tf,
               flop_per_cta * sms / (us_s * 1e-6) / 1e12, fpc, cyc, iters, sms, us, nsus);
        fflush(stdout);
    }
    // ---- FP64 DMMA
    {
        const int iters = 20000, threads = 256, blocks = sms * 4;
        const double flop = 2.0 * 16 * 8 * 8 * 4 * (double)iters * (threads / 32) * blocks;
        auto launch = [&]() { f64_peak_kernel<<<blocks, threads>>>(iters, dout); };
        const double us = time_us(launch, 3);
        const int nsus = (int)(sustain_s / (us * 1e-6)) + 1;
        const double us_s = time_us(launch, nsus);
        printf("{\"case\": \"f64_dmma_m16n8k8\", \"tflops_burst\": %.2f, \"tflops_sustained\": %.2f, \"warps_per_sm\": %d, "
               "\"launch_us\": %.1f}\n", flop / (us * 1e-6) / 1e12, flop / (us_s * 1e-6) / 1e12, threads / 32 * 4, us);
    }
    printf("{\"case\": \"device\", \"sms\": %d, \"clock_rate_mhz\": %.0f}\n", sms, clk_khz / 1e3);
    return 0;
}
