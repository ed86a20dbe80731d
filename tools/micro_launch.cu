// micro_launch.cu -- launch / PDL / grid-barrier overheads as seen by CUDA events (tool).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/micro_launch tools/micro_launch.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__global__ void empty_kernel(int* p) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
// one grid-wide barrier (all CTAs co-resident): arrive counter + generation flag
__global__ void barrier_kernel(unsigned* bar, int nbar) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = 0; i < nbar; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            volatile unsigned* gen = bar + 1;
            const unsigned g = *gen;
            __threadfence();
            if (atomicAdd(bar, 1u) == gridDim.x - 1) {
                bar[0] = 0;
                __threadfence();
                atomicAdd(bar + 1, 1u);
            } else {
                while (*gen == g) __nanosleep(32);
            }
            __threadfence();
        }
        __syncthreads();
    }
}

static void* g_flush;
template <typename F>
static void timeit(const char* name, F fn) {
    for (int i = 0; i < 5; ++i) fn();
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int R = 50;
    for (int i = 0; i < R; ++i) {
        CK(cudaMemsetAsync(g_flush, 1, 64 << 20));
        cudaEventRecord(a);
        fn();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        tot += ms;
    }
    CK(cudaGetLastError());
    printf("{\"case\": \"%s\", \"us\": %.2f}\n", name, 1e3 * tot / R);
    fflush(stdout);
}

static void launch(void (*k)(int*), int grid, int threads, bool pdl, int* arg) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = threads;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k, arg));
}

int main() {
    CK(cudaMalloc(&g_flush, 64 << 20));
    unsigned* bar;
    CK(cudaMalloc(&bar, 8));
    CK(cudaMemset(bar, 0, 8));
    timeit("nothing", [] {});
    timeit("1 empty 444x256", [] { launch(empty_kernel, 444, 256, false, nullptr); });
    timeit("1 empty 444x256 pdl", [] { launch(empty_kernel, 444, 256, true, nullptr); });
    timeit("2 empty 444x256", [] { launch(empty_kernel, 444, 256, false, nullptr); launch(empty_kernel, 444, 256, false, nullptr); });
    timeit("2 empty 444x256 pdl", [] { launch(empty_kernel, 444, 256, true, nullptr); launch(empty_kernel, 444, 256, true, nullptr); });
    timeit("4 empty 444x256 pdl", [] { for (int i = 0; i < 4; ++i) launch(empty_kernel, 444, 256, true, nullptr); });
    timeit("1 barrier 444x256", [&] { barrier_kernel<<<444, 256>>>(bar, 1); });
    timeit("1 barrier x4 444x256", [&] { barrier_kernel<<<444, 256>>>(bar, 4); });
    timeit("1 barrier 148x768", [&] { barrier_kernel<<<148, 768>>>(bar, 1); });
    timeit("0 barrier 444x256", [&] { barrier_kernel<<<444, 256>>>(bar, 0); });
    return 0;
}
