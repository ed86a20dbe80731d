// fb_fft_small.cu -- the Fourier-transform block for the small 256 x 256
// transform (BASELINE configs[0]) as ONE kernel: a thread-block cluster of CL CTAs holds the
// whole 512 KiB array on chip.  The two-pass path costs two dependent launches per transform
// (four per forward + inverse), which at this size is most of the time.
//
// CTA r of the cluster owns rows [R r, R r + R) and columns [R r, R r + R), R = 256 / CL:
//   row phase     thread (l = tid / 16, t = tid % 16) of row rho = R r + l: the length-256 DFT
//                 as 16 x 16 (stage 1: the length-16 DFT over m of x[rho][t + 16 m], times
//                 W_256^{t k1}; a per-line exchange through shared memory inside the warp;
//                 stage 2: the length-16 DFT over t) -> X[rho][k1 + 16 k2] (k1 = this thread's
//                 t), stored into the shared memory of the CTA that owns column k1 + 16 k2
//                 (distributed shared memory, 128-byte row segments: the row-to-column
//                 transpose never touches HBM);
//   cluster barrier;
//   column phase  the same 16 x 16 DFT down each of the CTA's R columns, results staged
//                 [k][column] and stored as R-wide row segments.
// The inverse is conj(DFT(conj x)) / 65536 like the pass kernels.  In place is allowed: every
// load of x precedes the cluster barrier and every store of y follows it.
#include "fb_fft_kern.cuh"

namespace fb {

namespace small {
constexpr int N = 256;
constexpr int LP = 16 * 17;         // per-line exchange block [k1][t], pitch 17

template <int CL>
struct Geo {
    static constexpr int R = N / CL;                   // rows (and columns) per CTA
    static constexpr int THREADS = 16 * R;
    static constexpr int COL = N * R;                  // float2: [row][column ^ (row & 15)]
    static constexpr int EX = R * LP;                  // float2 (also holds the [k][R+1] output tile)
    static_assert(N * (R + 1) <= EX, "output tile must fit the exchange buffer");
    static constexpr size_t SMEM = (size_t)(COL + EX + N) * sizeof(float2);  // + W_256^j table
};

// length-256 DFT of the 16 elements v[m] = line[t + 16 m] held by each of 16 threads of a line
// (t = lane & 15); on return v[k2] = X[t + 16 k2].  ex: this line's exchange block; w256: the
// W_256^j table in shared memory.
__device__ __forceinline__ void dft256(float2* v, int t, float2* ex, const float2* w256) {
    dft<16>(v);
#pragma unroll
    for (int k = 1; k < 16; ++k) v[k] = cmul(v[k], w256[(t * k) & 255]);
#pragma unroll
    for (int k = 0; k < 16; ++k) ex[k * 17 + t] = v[k];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = ex[t * 17 + j];
    __syncwarp();
    dft<16>(v);
}

template <int CL>
__global__ void __launch_bounds__(Geo<CL>::THREADS, 1)
    fft256_cluster_kernel(const float2* x, float2* y, const float2* __restrict__ tw, int inverse, float scale) {
    using G = Geo<CL>;
    constexpr int R = G::R;
    extern __shared__ __align__(16) float2 sm[];
    float2* col = sm;
    float2* ex = sm + G::COL;
    float2* w256 = ex + G::EX;
    const int tid = threadIdx.x, l = tid >> 4, t = tid & 15;
    // the twiddle table does not depend on the previous kernel: loaded before the PDL wait,
    // under the previous kernel's tail
    for (int j = tid; j < N; j += G::THREADS) w256[j] = __ldg(tw + (j << (kTwLog2 - 8)));
    const uint32_t r = ptx::cluster_ctarank();
    ptx::cluster_arrive_release();  // every CTA of the cluster has started (DSMEM targets exist)
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();
    // ---- row phase
    const int rho = R * (int)r + l;
    float2 v[16];
    {
        const float2* src = x + (int64_t)rho * N + t;
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m] = __ldcs(src + 16 * m);
    }
    if (inverse) {
#pragma unroll
        for (int m = 0; m < 16; ++m) v[m].y = -v[m].y;
    }
    __syncthreads();  // the twiddle table
    dft256(v, t, ex + l * LP, w256);
    ptx::cluster_wait_acquire();
    const uint32_t col_loc = ptx::smem_u32(col);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
        // X[rho][c] -> row rho of the owner's [row][column] block: the 16 lanes of a line write
        // 16 consecutive columns (one 128-byte segment); the XOR swizzle keeps the column
        // phase's reads down a column conflict-free
        const int c = t + 16 * k2;
        const uint32_t d = (uint32_t)(c / R), cl = (uint32_t)(c % R);
        ptx::st_cluster_f2(ptx::mapa_shared(col_loc + (uint32_t)(rho * R + (cl ^ (rho & 15))) * 8u, d), v[k2]);
    }
    ptx::cluster_arrive_release();
    ptx::cluster_wait_acquire();  // every column of this CTA is complete
    // ---- column phase: column c0 + l (c0 = R r), rows k = t + 16 k2 on output
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = col[(t + 16 * m) * R + (l ^ t)];
    dft256(v, t, ex + l * LP, w256);
    __syncthreads();  // every line is done with its exchange block: ex becomes the output tile
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
        float2 o = v[k2];
        if (inverse) o.y = -o.y;
        ex[(t + 16 * k2) * (R + 1) + l] = make_float2(o.x * scale, o.y * scale);
    }
    __syncthreads();
    float2* dst = y + R * (int)r;
#pragma unroll 4
    for (int e = tid; e < N * R; e += G::THREADS) {
        const int k = e / R, c = e % R;
        dst[(int64_t)k * N + c] = ex[k * (R + 1) + c];
    }
}
}  // namespace small

template <int CL>
static void small_cfg(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at, cudaStream_t s) {
    cfg = {};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(small::Geo<CL>::THREADS);
    cfg.dynamicSmemBytes = small::Geo<CL>::SMEM;
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
}

template <int CL>
static fb_status prepare_small(int dev, bool* schedulable) {
    auto kern = small::fft256_cluster_kernel<CL>;
    static DevOnce once;
    static std::atomic<int> ok[64];
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small::Geo<CL>::SMEM));
        if (CL > 8) FB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        // a 16-CTA cluster needs 16 SMs of one GPC free at once: if the device (a partitioned GPU)
        // cannot place it, fft2d_device keeps the two-pass path for this size
        cudaLaunchConfig_t cfg;
        cudaLaunchAttribute at[2];
        small_cfg<CL>(cfg, at, 0);
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            nc = 0;
        }
        ok[dev & 63].store(nc > 0 ? 1 : 0);
        once.set(dev);
    }
    *schedulable = ok[dev & 63].load() != 0;
    return FB_OK;
}

bool fft_small_eligible(int64_t n0, int64_t n1) {
    if (n0 != small::N || n1 != small::N || knobs().fft_small == 0) return false;
    bool sched = false;
    const int dev = DevOnce::dev();
    const fb_status rc = knobs().fft_small == 8 ? prepare_small<8>(dev, &sched) : prepare_small<16>(dev, &sched);
    return rc == FB_OK && sched;
}

template <int CL>
static fb_status launch_small(const float2* x, float2* y, bool inverse, float scale, const DeviceState* st,
                              cudaStream_t s) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[2];
    small_cfg<CL>(cfg, at, s);
    FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, small::fft256_cluster_kernel<CL>, x, y, (const float2*)st->twiddles,
                                   inverse ? 1 : 0, scale));
    FB_LAUNCH_CHECK("fft256_cluster_kernel");
    return FB_OK;
}

// cluster size (knob FB_FFT_SMALL): 16 CTAs (non-portable cluster, 16 rows each) by default --
// interleaved A/B of one forward: 16 CTAs 10.4 us, 8 CTAs 12.5 us, two-pass path 11.9 us;
// bench fwd + inv 15.4 / 20.2 / 18.9 us
fb_status fft2d_small(const float2* x, float2* y, bool inverse, float scale, const DeviceState* st, cudaStream_t s) {
    return knobs().fft_small == 8 ? launch_small<8>(x, y, inverse, scale, st, s)
                                  : launch_small<16>(x, y, inverse, scale, st, s);
}

}  // namespace fb
