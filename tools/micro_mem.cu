// micro_mem.cu -- memory-path microbenchmarks for the FFT pass design (tool, not product).
// Streams a 2048 x 2048 complex64 array (32 MiB) through one SM-persistent grid with
//   colload  C : 3D TMA boxes {C columns, 256 rows} (C*8-byte row segments)  -> smem ring
//   bulk1d     : 1D bulk copies of whole 16 KB rows                          -> smem ring
//   colstore C : TMA tensor stores of {C, 256} boxes from smem
//   ldgcol   C : LDG.128 of C-wide column segments into registers (no smem)
//   rowcopy    : LDG.128 + STG.128 plain copy (coalesced)
// L2 warm (array resident) and cold (512 MiB written in between).  One JSON line per case.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o micro_mem tools/micro_mem.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(dst), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                 ::"l"((uint64_t)m), "r"(src), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"((uint64_t)src), "r"(bytes), "r"(bar) : "memory");
}

constexpr int N = 2048;
constexpr int ROWS = 2048;

// ring of NB buffers of (C * ROWS) elements; one thread issues, the CTA consumes (touches 1 word)
template <int C, int NB>
__global__ void colload_kernel(const __grid_constant__ CUtensorMap tin, int ngroups, float* sink) {
    extern __shared__ __align__(128) float2 sm[];
    uint64_t* bars = (uint64_t*)(sm + NB * C * ROWS);
    if (threadIdx.x == 0) for (int b = 0; b < NB; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](int g, int b) {
        uint32_t bar = smem_u32(&bars[b]);
        mbar_expect(bar, C * ROWS * 8);
        for (int kb = 0; kb < ROWS; kb += 256) tma_load_3d(smem_u32(sm + b * C * ROWS + kb * C), &tin, bar, g * C, kb, 0);
    };
    int it = 0;
    if (threadIdx.x == 0)
        for (int b = 0; b < NB; ++b) if ((int)blockIdx.x + b * (int)gridDim.x < ngroups) issue(blockIdx.x + b * gridDim.x, b);
    float acc = 0.f;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
        const int b = it % NB;
        mbar_wait(smem_u32(&bars[b]), (it / NB) & 1);
        acc += sm[b * C * ROWS + threadIdx.x].x;
        __syncthreads();
        if (threadIdx.x == 0 && g + NB * (int)gridDim.x < ngroups) issue(g + NB * gridDim.x, b);
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <int NB>
__global__ void bulk1d_kernel(const float2* in, int ngroups, int rows_per_group, float* sink) {
    extern __shared__ __align__(128) float2 sm[];
    const int GE = rows_per_group * N;
    uint64_t* bars = (uint64_t*)(sm + NB * GE);
    if (threadIdx.x == 0) for (int b = 0; b < NB; ++b) mbar_init(smem_u32(&bars[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](int g, int b) {
        uint32_t bar = smem_u32(&bars[b]);
        mbar_expect(bar, GE * 8);
        for (int r = 0; r < rows_per_group; ++r)
            bulk_load(smem_u32(sm + b * GE + r * N), in + ((size_t)g * rows_per_group + r) * N, N * 8, bar);
    };
    int it = 0;
    if (threadIdx.x == 0)
        for (int b = 0; b < NB; ++b) if ((int)blockIdx.x + b * (int)gridDim.x < ngroups) issue(blockIdx.x + b * gridDim.x, b);
    float acc = 0.f;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
        const int b = it % NB;
        mbar_wait(smem_u32(&bars[b]), (it / NB) & 1);
        acc += sm[b * GE + threadIdx.x].x;
        __syncthreads();
        if (threadIdx.x == 0 && g + NB * (int)gridDim.x < ngroups) issue(g + NB * gridDim.x, b);
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <int C>
__global__ void colstore_kernel(const __grid_constant__ CUtensorMap tout, int ngroups) {
    extern __shared__ __align__(128) float2 sm[];
    for (int i = threadIdx.x; i < C * ROWS; i += blockDim.x) sm[i] = make_float2(i, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        int n = 0;
        for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
            for (int kb = 0; kb < ROWS; kb += 256) tma_store_3d(&tout, smem_u32(sm + kb * C), g * C, kb, 0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (++n >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// C-wide column segments by LDG.128: lane l of a warp covers (C/2) 16-byte chunks per row ->
// 32 / (C/2) rows per warp instruction
template <int C>
__global__ void ldgcol_kernel(const float4* in, int ngroups, float* sink) {
    constexpr int CH = C / 2;  // 16-byte chunks per row segment
    float acc = 0.f;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const float4* base = in + (size_t)g * CH;
        for (int i = threadIdx.x; i < ROWS * CH; i += blockDim.x * 4) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = i + u * blockDim.x;
                v[u] = (j < ROWS * CH) ? __ldcg(base + (size_t)(j / CH) * (N / 2) + (j % CH)) : make_float4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].w;
        }
    }
    if (acc == 12345.f) sink[0] = acc;
}

__global__ void rowcopy_kernel(const float4* in, float4* out, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        out[i] = __ldcg(in + i);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncFn enc() {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    return (EncFn)f;
}
static CUtensorMap colmap(void* base, int C) {
    CUtensorMap m;
    cuuint64_t dims[3] = {N, ROWS, 1};
    cuuint64_t strides[2] = {N * 8, (cuuint64_t)N * ROWS * 8};
    cuuint32_t box[3] = {(cuuint32_t)C, 256, 1}, es[3] = {1, 1, 1};
    if (enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        fprintf(stderr, "encode failed\n");
        exit(1);
    }
    return m;
}

static void* g_flush;
static void flush() { CK(cudaMemsetAsync(g_flush, 1, 512u << 20)); }

template <typename F>
static void timeit(const char* name, int C, int NB, int grid, F launch, bool cold) {
    for (int i = 0; i < 3; ++i) { if (cold) flush(); launch(); }
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0, mn = 1e9;
    const int R = 20;
    for (int i = 0; i < R; ++i) {
        if (cold) flush();
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        tot += ms;
        mn = ms < mn ? ms : mn;
    }
    CK(cudaGetLastError());
    const double bytes = (double)N * ROWS * 8;
    printf("{\"case\": \"%s\", \"C\": %d, \"NB\": %d, \"grid\": %d, \"cold\": %d, \"us\": %.2f, \"us_min\": %.2f, \"GBps\": %.0f}\n",
           name, C, NB, grid, (int)cold, 1e3 * tot / R, 1e3 * mn, bytes / (tot / R * 1e-3) / 1e9);
    fflush(stdout);
}

template <int C, int NB>
static void run_colload(void* x, float* sink, int sms, int per_sm, bool cold) {
    CUtensorMap m = colmap(x, C);
    size_t smem = (size_t)NB * C * ROWS * 8 + 64;
    if (smem > 227 * 1024) return;
    auto k = colload_kernel<C, NB>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int grid = sms * per_sm;
    timeit("colload", C, NB, grid, [&] { k<<<grid, 128, smem>>>(m, N / C, sink); }, cold);
}
template <int C>
static void run_colstore(void* x, int sms, int per_sm) {
    CUtensorMap m = colmap(x, C);
    size_t smem = (size_t)C * ROWS * 8;
    auto k = colstore_kernel<C>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int grid = sms * per_sm;
    timeit("colstore", C, 1, grid, [&] { k<<<grid, 128, smem>>>(m, N / C); }, false);
}
template <int C>
static void run_ldgcol(void* x, float* sink, int sms, int per_sm, bool cold) {
    int grid = sms * per_sm;
    timeit("ldgcol", C, 0, grid, [&] { ldgcol_kernel<C><<<grid, 256>>>((const float4*)x, N / C, sink); }, cold);
}
template <int NB>
static void run_bulk(void* x, float* sink, int sms, int per_sm, int rpg, bool cold) {
    size_t smem = (size_t)NB * rpg * N * 8 + 64;
    if (smem > 227 * 1024) return;
    auto k = bulk1d_kernel<NB>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int grid = sms * per_sm;
    char nm[32];
    snprintf(nm, sizeof nm, "bulk1d_r%d", rpg);
    timeit(nm, rpg, NB, grid, [&] { k<<<grid, 128, smem>>>((const float2*)x, ROWS / rpg, rpg, sink); }, cold);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    void *x, *y;
    float* sink;
    CK(cudaMalloc(&x, (size_t)N * ROWS * 8));
    CK(cudaMalloc(&y, (size_t)N * ROWS * 8));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMalloc(&g_flush, 512u << 20));
    CK(cudaMemset(x, 0, (size_t)N * ROWS * 8));
    for (int cold = 0; cold < 2; ++cold) {
        run_colload<2, 2>(x, sink, sms, 4, cold);
        run_colload<4, 2>(x, sink, sms, 2, cold);
        run_colload<4, 3>(x, sink, sms, 1, cold);
        run_colload<8, 1>(x, sink, sms, 2, cold);
        run_colload<8, 2>(x, sink, sms, 1, cold);
        run_colload<16, 1>(x, sink, sms, 1, cold);
        run_bulk<2>(x, sink, sms, 3, 2, cold);
        run_bulk<3>(x, sink, sms, 1, 2, cold);
        run_bulk<4>(x, sink, sms, 1, 1, cold);
        run_ldgcol<4>(x, sink, sms, 4, cold);
        run_ldgcol<8>(x, sink, sms, 4, cold);
        run_ldgcol<16>(x, sink, sms, 4, cold);
        size_t n4 = (size_t)N * ROWS / 2;
        timeit("rowcopy", 0, 0, sms * 8, [&] { rowcopy_kernel<<<sms * 8, 256>>>((const float4*)x, (float4*)y, n4); }, cold);
    }
    run_colstore<4>(y, sms, 4);
    run_colstore<8>(y, sms, 2);
    run_colstore<16>(y, sms, 1);
    return 0;
}
