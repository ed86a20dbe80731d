// fb_lu.cu -- the paper's own matrix workload: LU decomposition with partial pivoting
// ("LU decomposition processing of 2048*2048 orthogonal matrix data", PAPER.md P:153,
// replaced there by cuSOLVER getrf).  P A = L U in place, FP64,
// row-major, LAPACK getrf semantics (first max |a| pivot, whole-row swaps, multipliers scaled
// by the pivot's reciprocal unless |pivot| < DBL_MIN as in dgetf2, ipiv 0-based).
//
// Blocked right-looking factorisation with 8-column panels:
//   1. lu_panel_kernel   one CTA: the panel's rows live in registers (4 rows x 8 columns per
//                        thread); per column: pivot search (warp shuffles + block reduction,
//                        ties to the smaller row), row swap through shared memory, division by
//                        the pivot and the rank-1 update of the panel's remaining columns;
//   2. lu_swap_trsm_kernel  the panel's swaps applied, in order, to every other column, then
//                        U12 = L11^-1 A12 (unit lower 8x8) for the columns right of the panel;
//   4. A22 -= A21 U12    the DMMA GEMM with a subtracting epilogue (fb_gemm.cu).
#include <cuda.h>
#include <float.h>
#include <string.h>

#include "fb_common.cuh"
#include "fb_ptx.cuh"

namespace fb {
fb_status gemm_f64_sub_device(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                              int64_t ldb, double* C, int64_t ldc, cudaStream_t s);

namespace lu {
constexpr int NB = 8;       // panel width
constexpr int NMAX = 4096;  // n <= 4096

// Panel factorisation, one CTA: PT threads, each holding RPT rows (tid + i*PT) x PNB columns
// of the panel in registers; the panel is staged through shared memory so the global loads
// and stores are coalesced 16-byte transfers.  Per column: local scan, warp max by shuffles
// with LAPACK's tie rule (smallest row among equal maxima, __reduce_min_sync), every warp
// reduces the per-warp results itself, pivot/row-c copies through parity-buffered shared
// slots -> two block barriers per column.
template <int PT, int RPT, int PNB>
__global__ void __launch_bounds__(PT, 1)
    lu_panel_kernel(double* __restrict__ A, int64_t lda, int n, int j0, int jb, int32_t* __restrict__ ipiv,
                    int32_t* __restrict__ info) {
    constexpr int NW = PT / 32;
    __shared__ double red_v[2][NW];
    __shared__ int red_r[2][NW];
    __shared__ double prow[2][PNB], crow[2][PNB];
    static_assert(PNB <= NB, "panel width");
    extern __shared__ __align__(16) double P[];  // [m][PNB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the previous update has finished
    const int m = n - j0;
    for (int e = tid; e < m * (PNB / 2); e += PT) {
        const int r = e / (PNB / 2), ch = e % (PNB / 2);
        double2 v = make_double2(0.0, 0.0);
        if (2 * ch < jb) v = *reinterpret_cast<const double2*>(A + (int64_t)(j0 + r) * lda + j0 + 2 * ch);
        if (2 * ch + 1 >= jb) v.y = 0.0;
        *reinterpret_cast<double2*>(P + r * PNB + 2 * ch) = v;
    }
    __syncthreads();
    double a[RPT][PNB];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int rr = tid + i * PT;
#pragma unroll
        for (int j = 0; j < PNB; ++j) a[i][j] = rr < m ? P[rr * PNB + j] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < PNB; ++k) {  // unrolled: register indices are constants
        if (k >= jb) break;
        const int par = k & 1;
        const int c = j0 + k;
        double bv = -1.0;
        int br = INT_MAX;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {  // rows ascend with i: strict > keeps the first max
            const int r = j0 + tid + i * PT;
            const double v = fabs(a[i][k]);
            if (r >= c && r < n && v > bv) {
                bv = v;
                br = r;
            }
        }
        double wv = bv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wv = fmax(wv, __shfl_xor_sync(0xffffffffu, wv, o));
        const int wr = (int)__reduce_min_sync(0xffffffffu, (unsigned)(bv == wv ? br : INT_MAX));
        if (lane == 0) {
            red_v[par][warp] = wv;
            red_r[par][warp] = wr;
        }
        __syncthreads();
        double pv = -1.0;
        int p = INT_MAX;
#pragma unroll
        for (int w = 0; w < NW; ++w) {  // every thread: same order, same result
            const double v = red_v[par][w];
            const int r = red_r[par][w];
            if (v > pv || (v == pv && r < p)) {
                pv = v;
                p = r;
            }
        }
        if (tid == 0) ipiv[c] = p;
        const int oc = (c - j0) % PT, ic = (c - j0) / PT;
        const int op = (p - j0) % PT, ip = (p - j0) / PT;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (tid == op && i == ip)
#pragma unroll
                for (int j = 0; j < PNB; ++j) prow[par][j] = a[i][j];
            if (tid == oc && i == ic)
#pragma unroll
                for (int j = 0; j < PNB; ++j) crow[par][j] = a[i][j];
        }
        __syncthreads();
        if (p != c) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                if (tid == oc && i == ic)
#pragma unroll
                    for (int j = 0; j < PNB; ++j) a[i][j] = prow[par][j];
                if (tid == op && i == ip)
#pragma unroll
                    for (int j = 0; j < PNB; ++j) a[i][j] = crow[par][j];
            }
        }
        const double piv = prow[par][k];
        if (piv == 0.0) {
            if (tid == 0 && *info == 0) *info = c + 1;  // singular column: skipped, as LAPACK
        } else {
            const bool recip = fabs(piv) >= DBL_MIN;  // LAPACK dgetf2's sfmin rule
            const double rpiv = 1.0 / piv;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = j0 + tid + i * PT;
                if (r > c && r < n) {
                    const double l = recip ? a[i][k] * rpiv : a[i][k] / piv;
                    a[i][k] = l;
#pragma unroll
                    for (int j = k + 1; j < PNB; ++j)
                        if (j < jb) a[i][j] -= l * prow[par][j];
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int rr = tid + i * PT;
        if (rr < m)
#pragma unroll
            for (int j = 0; j < PNB; ++j) P[rr * PNB + j] = a[i][j];
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int e = tid; e < m * (PNB / 2); e += PT) {
        const int r = e / (PNB / 2), ch = e % (PNB / 2);
        const double2 v = *reinterpret_cast<const double2*>(P + r * PNB + 2 * ch);
        double* dst = A + (int64_t)(j0 + r) * lda + j0 + 2 * ch;
        if (2 * ch + 1 < jb)
            *reinterpret_cast<double2*>(dst) = v;
        else if (2 * ch < jb)
            dst[0] = v.x;
    }
}

// Per column outside the panel: the panel's swaps applied in order, then (for the columns
// right of the panel) the forward substitution U12 = L11^-1 A12 with the unit-lower L11.
constexpr int SWAP_T = 128;
__global__ void __launch_bounds__(SWAP_T)
    lu_swap_trsm_kernel(double* __restrict__ A, int64_t lda, int n, int j0, int jb,
                        const int32_t* __restrict__ ipiv) {
    __shared__ double L[NB][NB];
    __shared__ int piv[NB];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the panel kernel has finished
    if (threadIdx.x < NB * NB) {
        const int i = threadIdx.x / NB, k = threadIdx.x % NB;
        L[i][k] = (i < jb && k < jb) ? A[(int64_t)(j0 + i) * lda + j0 + k] : 0.0;
    }
    if (threadIdx.x < NB) piv[threadIdx.x] = threadIdx.x < jb ? ipiv[j0 + threadIdx.x] : j0 + threadIdx.x;
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int col = blockIdx.x * SWAP_T + threadIdx.x;
    if (col >= n || (col >= j0 && col < j0 + jb)) return;
#pragma unroll 1
    for (int k = 0; k < jb; ++k) {
        const int p = piv[k];
        if (p != j0 + k) {
            const double t = A[(int64_t)(j0 + k) * lda + col];
            A[(int64_t)(j0 + k) * lda + col] = A[(int64_t)p * lda + col];
            A[(int64_t)p * lda + col] = t;
        }
    }
    if (col < j0 + jb) return;
    double x[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) x[i] = i < jb ? A[(int64_t)(j0 + i) * lda + col] : 0.0;
#pragma unroll
    for (int i = 1; i < NB; ++i)
#pragma unroll
        for (int k = 0; k < i; ++k) x[i] -= L[i][k] * x[k];
#pragma unroll
    for (int i = 1; i < NB; ++i)
        if (i < jb) A[(int64_t)(j0 + i) * lda + col] = x[i];
}
// ---------------------------------------------------------------- look-ahead variant
// Panel k+1 is factored while the wide update of step k runs on the other SMs (second stream).
// The panel kernel therefore first finishes its own PNB columns' share of step k -- the
// previous panel's swaps, the unit-lower solve of rows jp..jp+PNB-1 (U12) and the rank-PNB
// update of rows >= j0 with L21(k) -- then factors them.
//
// One SM does all of this, so the count of L1/LSU transactions is the cost, not bytes: every
// global access is a coalesced 16-byte chunk (PNB/2 lanes per row) moved by cp.async into
// row-major shared buffers whose 16-byte chunks are XOR-swizzled by row (chunk c of row r at
// c ^ ((r / rows_per_128B) mod chunks)), so the per-thread row reads and writes are bank-
// conflict-free: the panel rows [r0, n), L21 in batches of PT rows (double-buffered, the first
// two in flight with the panel), and the write-back (registers -> buffer -> coalesced stores).
// Per column: pivot search (warp shuffles, LAPACK's first-max tie rule), per-warp shuffle
// combine, swap through shared memory by the owning threads only.
template <int PNB>
__device__ __forceinline__ int lu_pidx(int r, int j) {
    constexpr int CH = PNB / 2;          // 16-byte chunks per row
    constexpr int RPL = 8 / CH;          // rows per 128-byte line
    const int c = (j >> 1) ^ ((r / RPL) & (CH - 1));
    return r * PNB + 2 * c + (j & 1);
}

// The PNB pivot steps of a panel held in registers (thread tid owns rows j0 + tid + i*PT):
// pivot search, swap and rank-1 updates (shared by the cp.async and TMA panel kernels).
template <int PT, int RPT, int PNB>
__device__ __forceinline__ void lu_panel_columns(double (&a)[RPT][PNB], int tid, int j0, int jb, int n,
                                                 int32_t* __restrict__ ipiv, int32_t* __restrict__ info) {
    constexpr int NW = PT / 32;
    __shared__ __align__(16) double red_row[2][NW][PNB];  // each warp's candidate row
    __shared__ unsigned long long red_k[2][NW];
    __shared__ int red_r[2][NW];
    __shared__ double crow[2][PNB];
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int k = 0; k < PNB; ++k) {
        if (k >= jb) break;
#ifdef FB_LU_TIMING
        long long c0 = clock64();
#endif
        const int par = k & 1;
        const int c = j0 + k;
        double bv = -1.0;
        int br = INT_MAX, bi = 0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = j0 + tid + i * PT;
            const double v = fabs(a[i][k]);
            if (r >= c && r < n && v > bv) {
                bv = v;
                br = r;
                bi = i;
            }
        }
        // pivot = (max |a|, then smallest row): |a| >= 0 orders like its IEEE bit pattern, so
        // the warp and cross-warp reductions are three redux.sync each (max hi word, max lo
        // word among the max-hi lanes, min row among the max lanes); "no candidate" is key 0
        // with row INT_MAX, which a real zero pivot candidate beats on the row.  The lane that
        // holds its warp's candidate publishes the candidate's whole row, and the owner of row c
        // (thread k) publishes row c, before the one barrier of the column: afterwards every
        // thread reads the pivot row from the winning warp's slot, so no second barrier.
        unsigned long long key = bv >= 0.0 ? (unsigned long long)__double_as_longlong(bv) : 0ull;
        unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
        unsigned mhi = __reduce_max_sync(0xffffffffu, khi);
        unsigned mlo = __reduce_max_sync(0xffffffffu, khi == mhi ? klo : 0u);
        const int wr = (int)__reduce_min_sync(0xffffffffu, (unsigned)((khi == mhi && klo == mlo) ? br : INT_MAX));
        if (br == wr && wr != INT_MAX) {  // one lane per warp: a real branch per row, 16-byte stores
            double2* dst = reinterpret_cast<double2*>(&red_row[par][warp][0]);
            switch (bi) {
#define FB_LU_PUB(I)                                                                      \
    case I:                                                                               \
        if constexpr (I < RPT) {                                                          \
            _Pragma("unroll") for (int j = 0; j < PNB; j += 2) dst[j / 2] = make_double2(a[I][j], a[I][j + 1]); \
        }                                                                                 \
        break;
                FB_LU_PUB(0)
                FB_LU_PUB(1)
                FB_LU_PUB(2)
                FB_LU_PUB(3)
#undef FB_LU_PUB
            }
        }
        if (lane == 0) {
            red_k[par][warp] = ((unsigned long long)mhi << 32) | mlo;
            red_r[par][warp] = wr;
        }
        if (tid == k)
#pragma unroll
            for (int j = 0; j < PNB; ++j) crow[par][j] = a[0][j];  // row c = j0 + k is thread k's row 0
#ifdef FB_LU_TIMING
        long long c1 = clock64();
#endif
        __syncthreads();
#ifdef FB_LU_TIMING
        long long c2 = clock64();
#endif
        key = (lane < NW) ? red_k[par][lane] : 0ull;
        const int rw = (lane < NW) ? red_r[par][lane] : INT_MAX;
        khi = (unsigned)(key >> 32);
        klo = (unsigned)key;
        mhi = __reduce_max_sync(0xffffffffu, khi);
        mlo = __reduce_max_sync(0xffffffffu, khi == mhi ? klo : 0u);
        const int p = (int)__reduce_min_sync(0xffffffffu, (unsigned)((khi == mhi && klo == mlo) ? rw : INT_MAX));
        if (tid == 0) ipiv[c] = p;
        const int op = (p - j0) % PT, ip = (p - j0) / PT;
#ifdef FB_LU_TIMING
        long long c3 = clock64();
#endif
        double pr[PNB];
#pragma unroll
        for (int j = 0; j < PNB; ++j) pr[j] = red_row[par][op >> 5][j];
        if (p != c) {
            if (tid == k)
#pragma unroll
                for (int j = 0; j < PNB; ++j) a[0][j] = pr[j];
            if (tid == op) {
#pragma unroll
                for (int i = 0; i < RPT; ++i)
                    if (i == ip)
#pragma unroll
                        for (int j = 0; j < PNB; ++j) a[i][j] = crow[par][j];
            }
        }
#ifdef FB_LU_TIMING
        long long c4 = clock64();
#endif
        const double piv = pr[k];
        if (piv == 0.0) {
            if (tid == 0 && *info == 0) *info = c + 1;
        } else {
            // LAPACK dgetf2: scale by 1/piv when |piv| >= sfmin (DBL_MIN), else divide (uniform
            // branch, so the common path carries no division)
            if (fabs(piv) >= DBL_MIN) {
                const double rpiv = 1.0 / piv;
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int r = j0 + tid + i * PT;
                    if (r > c && r < n) {
                        const double l = a[i][k] * rpiv;
                        a[i][k] = l;
#pragma unroll
                        for (int j = k + 1; j < PNB; ++j)
                            if (j < jb) a[i][j] -= l * pr[j];
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int r = j0 + tid + i * PT;
                    if (r > c && r < n) {
                        const double l = a[i][k] / piv;
                        a[i][k] = l;
#pragma unroll
                        for (int j = k + 1; j < PNB; ++j)
                            if (j < jb) a[i][j] -= l * pr[j];
                    }
                }
            }
        }
#ifdef FB_LU_TIMING
        long long c5 = clock64();
        if ((tid == 0 || tid == 511) && (j0 == 80 || j0 == 1600) && k == 3)
            printf("LU_COL tid=%d j0=%d scan+redux=%lld bar=%lld xwarp=%lld rows+swap=%lld update=%lld\n", tid, j0,
                   c1 - c0, c2 - c1, c3 - c2, c4 - c3, c5 - c4);
#endif
    }
}

template <int PT, int RPT, int PNB>
__global__ void __launch_bounds__(PT, 1)
    lu_panel_la_kernel(double* __restrict__ A, int64_t lda, int n, int j0, int jb, int has_prev,
                       int32_t* __restrict__ ipiv, int32_t* __restrict__ info) {
    constexpr int CH = PNB / 2;
    __shared__ double L11[PNB][PNB];
    __shared__ double Us[PNB][PNB];  // U12 rows of this panel's columns
    __shared__ int pv[PNB];
    extern __shared__ __align__(16) double smem_lu[];
    const int tid = threadIdx.x;
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef FB_LU_TIMING
    long long tt[6];
    tt[0] = clock64();
#endif
    const int jp = j0 - PNB;  // previous panel (always full width)
    const int r0 = has_prev ? jp : j0;
    const int mr = n - r0;  // staged rows
    const int m = n - j0;   // rows of this panel's factorisation
    const int off = j0 - r0;
    double* P = smem_lu;           // [mr][PNB] swizzled
    double* Lb = smem_lu + mr * PNB;  // [2][PT][PNB] swizzled L21 batches
    for (int e = tid; e < mr * CH; e += PT) {
        const int r = e / CH, c = e % CH;
        const uint32_t bytes = (2 * c + 1 < jb) ? 16u : ((2 * c < jb) ? 8u : 0u);
        ptx::cp_async_16(ptx::smem_u32(P + lu_pidx<PNB>(r, 2 * c)), A + (int64_t)(r0 + r) * lda + j0 + (bytes ? 2 * c : 0),
                         bytes);
    }
    auto stage_l = [&](int i, int b) {  // L21 rows j0 + i*PT + [0, PT), columns jp..jp+PNB-1
        for (int e = tid; e < PT * CH; e += PT) {
            const int rr = e / CH, c = e % CH;
            const int row = i * PT + rr;
            const bool ok = row < m;
            ptx::cp_async_16(ptx::smem_u32(Lb + b * PT * PNB + lu_pidx<PNB>(rr, 2 * c)),
                             A + (int64_t)(j0 + (ok ? row : 0)) * lda + jp + 2 * c, ok ? 16u : 0u);
        }
    };
    if (has_prev) {
        stage_l(0, 0);
        if (RPT > 1) stage_l(1, 1);
        if (tid < PNB * PNB) {
            const int i = tid / PNB, k = tid % PNB;
            L11[i][k] = A[(int64_t)(jp + i) * lda + jp + k];
        }
        if (tid < PNB) pv[tid] = ipiv[jp + tid];
    }
    ptx::cp_async_commit();
    ptx::cp_async_wait<0>();
    __syncthreads();
#ifdef FB_LU_TIMING
    tt[1] = clock64();
#endif
    if (has_prev) {
        if (tid < PNB) {  // column tid: previous swaps in order, then x = L11^-1 x on rows jp..
            const int j = tid;
#pragma unroll 1
            for (int t = 0; t < PNB; ++t) {
                const int q = pv[t] - r0;
                if (q != t) {
                    const double tmp = P[lu_pidx<PNB>(t, j)];
                    P[lu_pidx<PNB>(t, j)] = P[lu_pidx<PNB>(q, j)];
                    P[lu_pidx<PNB>(q, j)] = tmp;
                }
            }
            double x[PNB];
#pragma unroll
            for (int i = 0; i < PNB; ++i) x[i] = P[lu_pidx<PNB>(i, j)];
#pragma unroll
            for (int i = 1; i < PNB; ++i)
#pragma unroll
                for (int k = 0; k < i; ++k) x[i] -= L11[i][k] * x[k];
#pragma unroll
            for (int i = 0; i < PNB; ++i) Us[i][j] = x[i];
            if (j < jb)
#pragma unroll
                for (int i = 0; i < PNB; ++i) A[(int64_t)(jp + i) * lda + j0 + j] = x[i];  // U12 rows
        }
        __syncthreads();
    }
    double a[RPT][PNB];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int rr = tid + i * PT;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            double2 v = make_double2(0.0, 0.0);
            if (rr < m) v = *reinterpret_cast<const double2*>(P + lu_pidx<PNB>(off + rr, 2 * c));
            a[i][2 * c] = v.x;
            a[i][2 * c + 1] = v.y;
        }
    }
#ifdef FB_LU_TIMING
    tt[2] = clock64();
#endif
    if (has_prev) {  // A[r][j0 + j] -= sum_t L21[r][t] U12[t][j]
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int b = i & 1;
            if (i >= 2) {  // batch i (issued once batch i-2 was consumed) has landed in buffer b
                if (i == RPT - 1)
                    ptx::cp_async_wait<0>();
                else
                    ptx::cp_async_wait<1>();
                __syncthreads();
            }
            double l[PNB];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const double2 v = *reinterpret_cast<const double2*>(Lb + b * PT * PNB + lu_pidx<PNB>(tid, 2 * c));
                l[2 * c] = v.x;
                l[2 * c + 1] = v.y;
            }
#pragma unroll
            for (int j = 0; j < PNB; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t < PNB; ++t) acc = fma(l[t], Us[t][j], acc);
                a[i][j] -= acc;
            }
            if (i + 2 < RPT) {  // refill buffer b with batch i + 2 once every thread has read it
                __syncthreads();
                stage_l(i + 2, b);
                ptx::cp_async_commit();
            }
        }
    }
#ifdef FB_LU_TIMING
    tt[3] = clock64();
#endif
    lu_panel_columns<PT, RPT, PNB>(a, tid, j0, jb, n, ipiv, info);
#ifdef FB_LU_TIMING
    tt[4] = clock64();
#endif
    // write back rows [j0, n): registers -> P (own rows, swizzled) -> coalesced 16-byte stores
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int rr = tid + i * PT;
        if (rr < m)
#pragma unroll
            for (int c = 0; c < CH; ++c)
                *reinterpret_cast<double2*>(P + lu_pidx<PNB>(off + rr, 2 * c)) = make_double2(a[i][2 * c], a[i][2 * c + 1]);
    }
    __syncthreads();
    for (int e = tid; e < m * CH; e += PT) {
        const int r = e / CH, c = e % CH;
        const double2 v = *reinterpret_cast<const double2*>(P + lu_pidx<PNB>(off + r, 2 * c));
        double* dst = A + (int64_t)(j0 + r) * lda + j0 + 2 * c;
        if (2 * c + 1 < jb)
            *reinterpret_cast<double2*>(dst) = v;
        else if (2 * c < jb)
            dst[0] = v.x;
    }
#ifdef FB_LU_TIMING
    __syncthreads();
    tt[5] = clock64();
    if (tid == 0 && (j0 == 80 || j0 == 1024 || j0 == 1600))
        printf("LU_TIMING j0=%d stage=%lld prevprep=%lld update=%lld columns=%lld writeback=%lld total=%lld\n", j0,
               tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4], tt[5] - tt[0]);
#endif
}

// TMA form of lu_panel_la_kernel: the panel rows [r0, n), the L21 batches and the write-back
// move as 2D tensor boxes of PNB columns x 256 rows (one thread issues them; the TMA engine's
// 64-byte (PNB = 8) / 32-byte (PNB = 4) swizzle is exactly the XOR layout lu_pidx reads), so
// the copies cost no LSU issue slots and the write-back drains while the CTA exits.
// Out-of-range rows / columns are zero-filled on load and clipped on store.
constexpr int LU_BOXR = 256;
template <int PT, int RPT, int PNB>
__global__ void __launch_bounds__(PT, 1)
    lu_panel_tma_kernel(double* __restrict__ A, int64_t lda, int n, int j0, int jb, int has_prev,
                        int32_t* __restrict__ ipiv, int32_t* __restrict__ info,
                        const __grid_constant__ CUtensorMap tmA) {
    static_assert(PT % LU_BOXR == 0, "L21 batches are whole boxes");
    __shared__ double L11[PNB][PNB];
    __shared__ double Us[PNB][PNB];
    __shared__ int pv[PNB];
    __shared__ __align__(8) uint64_t bars[3];
    extern __shared__ __align__(16) double smem_lu[];
    const int tid = threadIdx.x;
    const int jp = j0 - PNB;
    const int r0 = has_prev ? jp : j0;
    const int mr = n - r0;
    const int m = n - j0;
    const int off = j0 - r0;
    // [mr][PNB] swizzled, 1024-aligned (the swizzle pattern follows the smem address bits)
    double* P = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_lu) + 1023) & ~uintptr_t(1023));
    // whole boxes land in P (out-of-range rows as zeros), so it spans ceil(mr / 256) boxes
    double* Lb = P + ((mr + LU_BOXR - 1) / LU_BOXR) * LU_BOXR * PNB;  // [2][PT][PNB] swizzled
    const uint32_t bar_p = ptx::smem_u32(&bars[0]);
    auto bar_l = [&](int b) { return ptx::smem_u32(&bars[1 + b]); };
    constexpr uint32_t BOX_BYTES = LU_BOXR * PNB * sizeof(double);
    auto load_l = [&](int i, int b) {  // L21 rows j0 + i*PT + [0, PT), columns jp.. (thread 0)
        ptx::mbar_arrive_expect_tx(bar_l(b), (uint32_t)(PT / LU_BOXR) * BOX_BYTES);
        for (int q = 0; q < PT / LU_BOXR; ++q)
            ptx::tma_load_2d(ptx::smem_u32(Lb + (b * PT + q * LU_BOXR) * PNB), &tmA, bar_l(b), jp,
                             j0 + i * PT + q * LU_BOXR);
    };
    if (tid == 0) {
        ptx::mbar_init(bar_p, 1);
        ptx::mbar_init(bar_l(0), 1);
        ptx::mbar_init(bar_l(1), 1);
        ptx::fence_mbar_init();
        ptx::tma_prefetch_desc(&tmA);
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef FB_LU_TIMING
    long long tt[6];
    tt[0] = clock64();
#endif
    if (tid == 0) {
        const int nbox = (mr + LU_BOXR - 1) / LU_BOXR;
        ptx::mbar_arrive_expect_tx(bar_p, (uint32_t)nbox * BOX_BYTES);
        for (int q = 0; q < nbox; ++q)
            ptx::tma_load_2d(ptx::smem_u32(P + q * LU_BOXR * PNB), &tmA, bar_p, j0, r0 + q * LU_BOXR);
        if (has_prev) {
            load_l(0, 0);
            if (RPT > 1) load_l(1, 1);
        }
    }
    if (has_prev) {
        if (tid < PNB * PNB) {
            const int i = tid / PNB, k = tid % PNB;
            L11[i][k] = A[(int64_t)(jp + i) * lda + jp + k];
        }
        if (tid < PNB) pv[tid] = ipiv[jp + tid];
    }
    ptx::mbar_wait(bar_p, 0);
    __syncthreads();
#ifdef FB_LU_TIMING
    tt[1] = clock64();
#endif
    if (has_prev) {
        if (tid < PNB) {  // column tid: previous swaps in order, then x = L11^-1 x on rows jp..
            const int j = tid;
#pragma unroll 1
            for (int t = 0; t < PNB; ++t) {
                const int q = pv[t] - r0;
                if (q != t) {
                    const double tmp = P[lu_pidx<PNB>(t, j)];
                    P[lu_pidx<PNB>(t, j)] = P[lu_pidx<PNB>(q, j)];
                    P[lu_pidx<PNB>(q, j)] = tmp;
                }
            }
            double x[PNB];
#pragma unroll
            for (int i = 0; i < PNB; ++i) x[i] = P[lu_pidx<PNB>(i, j)];
#pragma unroll
            for (int i = 1; i < PNB; ++i)
#pragma unroll
                for (int k = 0; k < i; ++k) x[i] -= L11[i][k] * x[k];
#pragma unroll
            for (int i = 0; i < PNB; ++i) {
                Us[i][j] = x[i];
                P[lu_pidx<PNB>(i, j)] = x[i];  // U12 rows leave with the write-back
            }
        }
        __syncthreads();
    }
    double a[RPT][PNB];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int rr = tid + i * PT;
#pragma unroll
        for (int c = 0; c < PNB / 2; ++c) {
            double2 v = make_double2(0.0, 0.0);
            if (rr < m) v = *reinterpret_cast<const double2*>(P + lu_pidx<PNB>(off + rr, 2 * c));
            a[i][2 * c] = v.x;
            a[i][2 * c + 1] = v.y;
        }
    }
#ifdef FB_LU_TIMING
    tt[2] = clock64();
#endif
    if (has_prev) {  // A[r][j0 + j] -= sum_t L21[r][t] U12[t][j]
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int b = i & 1;
            ptx::mbar_wait(bar_l(b), (uint32_t)(i >> 1) & 1u);
            double l[PNB];
#pragma unroll
            for (int c = 0; c < PNB / 2; ++c) {
                const double2 v = *reinterpret_cast<const double2*>(Lb + b * PT * PNB + lu_pidx<PNB>(tid, 2 * c));
                l[2 * c] = v.x;
                l[2 * c + 1] = v.y;
            }
#pragma unroll
            for (int j = 0; j < PNB; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int t = 0; t < PNB; ++t) acc = fma(l[t], Us[t][j], acc);
                a[i][j] -= acc;
            }
            if (i + 2 < RPT) {  // refill buffer b with batch i + 2 once every thread has read it
                ptx::fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) load_l(i + 2, b);
            }
        }
    }
#ifdef FB_LU_TIMING
    tt[3] = clock64();
#endif
    lu_panel_columns<PT, RPT, PNB>(a, tid, j0, jb, n, ipiv, info);
#ifdef FB_LU_TIMING
    tt[4] = clock64();
#endif
    // write back rows [r0, n) (U12 rows + this panel): registers -> P -> TMA stores
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int rr = tid + i * PT;
        if (rr < m)
#pragma unroll
            for (int c = 0; c < PNB / 2; ++c)
                *reinterpret_cast<double2*>(P + lu_pidx<PNB>(off + rr, 2 * c)) =
                    make_double2(a[i][2 * c], a[i][2 * c + 1]);
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
        const int nbox = (mr + LU_BOXR - 1) / LU_BOXR;
        for (int q = 0; q < nbox; ++q) ptx::tma_store_2d(&tmA, ptx::smem_u32(P + q * LU_BOXR * PNB), j0, r0 + q * LU_BOXR);
        ptx::bulk_commit();
        // only the shared-memory source must outlive the CTA; the global writes are complete
        // when the grid is (the next kernel depends on the grid, as a CUTLASS TMA epilogue)
        ptx::bulk_wait_read0();
    }
#ifdef FB_LU_TIMING
    __syncthreads();
    tt[5] = clock64();
    if (tid == 0 && (j0 == 80 || j0 == 1024 || j0 == 1600))
        printf("LU_TIMING tma j0=%d stage=%lld prevprep=%lld update=%lld columns=%lld writeback=%lld total=%lld\n",
               j0, tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4], tt[5] - tt[0]);
#endif
}

// Wide part of step k (look-ahead): the panel's swaps on every column outside
// [j0, skip_end) (left: L columns of earlier panels; right: columns beyond the next panel),
// then U12 = L11^-1 A12 for the right columns.
__global__ void __launch_bounds__(SWAP_T)
    lu_swap_trsm_wide_kernel(double* __restrict__ A, int64_t lda, int n, int j0, int jb, int skip_end,
                             const int32_t* __restrict__ ipiv) {
    __shared__ double L[NB][NB];
    __shared__ int piv[NB];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x < NB * NB) {
        const int i = threadIdx.x / NB, k = threadIdx.x % NB;
        L[i][k] = (i < jb && k < jb) ? A[(int64_t)(j0 + i) * lda + j0 + k] : 0.0;
    }
    if (threadIdx.x < NB) piv[threadIdx.x] = threadIdx.x < jb ? ipiv[j0 + threadIdx.x] : j0 + threadIdx.x;
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int col = blockIdx.x * SWAP_T + threadIdx.x;
    if (col >= n || (col >= j0 && col < skip_end)) return;
#pragma unroll 1
    for (int k = 0; k < jb; ++k) {
        const int p = piv[k];
        if (p != j0 + k) {
            const double t = A[(int64_t)(j0 + k) * lda + col];
            A[(int64_t)(j0 + k) * lda + col] = A[(int64_t)p * lda + col];
            A[(int64_t)p * lda + col] = t;
        }
    }
    if (col < skip_end) return;
    double x[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) x[i] = i < jb ? A[(int64_t)(j0 + i) * lda + col] : 0.0;
#pragma unroll
    for (int i = 1; i < NB; ++i)
#pragma unroll
        for (int k = 0; k < i; ++k) x[i] -= L[i][k] * x[k];
#pragma unroll
    for (int i = 1; i < NB; ++i)
        if (i < jb) A[(int64_t)(j0 + i) * lda + col] = x[i];
}
// Trailing update of the look-ahead schedule: C -= A21 U12 with K = jb <= 8.  K is far too
// small for a tensor-core tile to pay off, so this is a streaming FP64 kernel: per CTA a
// 64 x 128 tile of C, A21 (64 x 8) and U12 (8 x 128) staged in shared memory, each thread two
// adjacent columns (its 16 U12 values in registers) of 16 rows, coalesced 16-byte loads and
// stores of C; per element a chain of jb FMAs (t ascending).
constexpr int RU_TM = 64, RU_TN = 128, RU_T = 256;
__global__ void __launch_bounds__(RU_T)
    lu_rank_update_kernel(double* __restrict__ C, const double* __restrict__ A21, const double* __restrict__ U12,
                          int64_t lda, int m, int nc, int jb) {
    __shared__ double As[RU_TM][NB];
    __shared__ double Bs[NB][RU_TN];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int r0 = blockIdx.y * RU_TM, c0 = blockIdx.x * RU_TN;
    for (int e = threadIdx.x; e < RU_TM * NB; e += RU_T) {
        const int r = e / NB, t = e % NB;
        As[r][t] = (r0 + r < m && t < jb) ? A21[(int64_t)(r0 + r) * lda + t] : 0.0;
    }
    for (int e = threadIdx.x; e < NB * RU_TN; e += RU_T) {
        const int t = e / RU_TN, cc = e % RU_TN;
        Bs[t][cc] = (t < jb && c0 + cc < nc) ? U12[(int64_t)t * lda + c0 + cc] : 0.0;
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int tx = threadIdx.x % (RU_TN / 2), ty = threadIdx.x / (RU_TN / 2);
    const int cc = 2 * tx;
    double b0[NB], b1[NB];
#pragma unroll
    for (int t = 0; t < NB; ++t) {
        b0[t] = Bs[t][cc];
        b1[t] = Bs[t][cc + 1];
    }
    const bool two = c0 + cc + 1 < nc, one = c0 + cc < nc;
#pragma unroll 4
    for (int r = ty; r < RU_TM; r += RU_T / (RU_TN / 2)) {
        if (r0 + r >= m || !one) continue;
        double* cp = C + (int64_t)(r0 + r) * lda + c0 + cc;
        double2 cv;
        if (two)
            cv = *reinterpret_cast<const double2*>(cp);
        else
            cv = make_double2(cp[0], 0.0);
#pragma unroll
        for (int t = 0; t < NB; ++t) {
            const double a = As[r][t];
            cv.x = fma(-a, b0[t], cv.x);
            cv.y = fma(-a, b1[t], cv.y);
        }
        if (two)
            *reinterpret_cast<double2*>(cp) = cv;
        else
            cp[0] = cv.x;
    }
}
}  // namespace lu

size_t lu_ws_bytes(int64_t) { return 0; }

// Launch with programmatic stream serialization (each LU kernel waits on griddepcontrol.wait
// before touching the matrix, so its launch overlaps the previous kernel's tail).
template <typename Kern, typename... Args>
static fb_status lu_launch(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    static DevOnce once;  // the attribute is per device context
    const int dev = DevOnce::dev();
    if (smem > 48 * 1024 && !once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(lu::lu_panel_kernel<512, 4, lu::NB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * lu::NB * 8));
        FB_CUDA_TRY(cudaFuncSetAttribute(lu::lu_panel_kernel<1024, 4, lu::NB / 2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * (lu::NB / 2) * 8));
        once.set(dev);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FB_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
    FB_LAUNCH_CHECK("lu kernel");
    return FB_OK;
}

// Look-ahead schedule (two streams): the caller's stream s runs the panels, an internal stream
// w the wide updates.
//   s:  panel_0 | rec P | wait W(k-1) | panel_{k+1} (finishes step k on its columns) | rec P ...
//   w:  wait P | wide_k = swaps outside [j0, j0 + jb + nb) + U12 + A22 -= A21 U12 beyond the
//       next panel | rec W[k % 2]
// panel_{k+1} needs panel_k (stream order) and wide_{k-1} (its columns' earlier updates), not
// wide_k, which overlaps it; wide_k needs panel_k and wide_{k-1} (stream order).  Columns
// touched concurrently are disjoint.  A wait binds to the record enqueued before it, so one
// P event and two alternating W events suffice.
struct LuStreams {
    cudaStream_t w = nullptr;
    cudaEvent_t ev_p = nullptr, ev_w[2] = {nullptr, nullptr}, ev_fork = nullptr;
};
static fb_status lu_streams(LuStreams** out) {
    thread_local static LuStreams per_dev[32];  // per host thread: concurrent fb_lu calls stay independent
    int dev = 0;
    FB_CUDA_TRY(cudaGetDevice(&dev));
    LuStreams& ls = per_dev[dev & 31];
    if (!ls.w) {
        FB_CUDA_TRY(cudaStreamCreateWithFlags(&ls.w, cudaStreamNonBlocking));
        FB_CUDA_TRY(cudaEventCreateWithFlags(&ls.ev_p, cudaEventDisableTiming));
        FB_CUDA_TRY(cudaEventCreateWithFlags(&ls.ev_w[0], cudaEventDisableTiming));
        FB_CUDA_TRY(cudaEventCreateWithFlags(&ls.ev_w[1], cudaEventDisableTiming));
        FB_CUDA_TRY(cudaEventCreateWithFlags(&ls.ev_fork, cudaEventDisableTiming));
    }
    *out = &ls;
    return FB_OK;
}

typedef CUresult (*EncodeTiledFnLU)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// A as a 2D FP64 tensor {n columns, n rows}, box {PNB columns, 256 rows}, swizzled like lu_pidx
static fb_status lu_tensor_map(CUtensorMap* m, double* A, int64_t n, int64_t lda, int pnb) {
    static EncodeTiledFnLU enc = nullptr;
    if (!enc) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            set_error("cuTensorMapEncodeTiled unavailable from the driver");
            return FB_ERR_CUDA;
        }
        enc = (EncodeTiledFnLU)f;
    }
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)(lda * 8)};
    cuuint32_t box[2] = {(cuuint32_t)pnb, (cuuint32_t)lu::LU_BOXR};
    cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           pnb == 8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d) for the LU panel map", (int)r);
        return FB_ERR_CUDA;
    }
    return FB_OK;
}

template <int PT, int RPT, int PNB>
static fb_status lu_la_attrs() {  // outside any stream capture
    static DevOnce once;  // the attribute is per device context
    const int dev = DevOnce::dev();
    if (!once.done(dev)) {
        FB_CUDA_TRY(cudaFuncSetAttribute(lu::lu_panel_la_kernel<PT, RPT, PNB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        FB_CUDA_TRY(cudaFuncSetAttribute(lu::lu_panel_tma_kernel<PT, RPT, PNB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        once.set(dev);
    }
    return FB_OK;
}

template <int PT, int RPT, int PNB>
static fb_status lu_device_la(int64_t n, double* A, int64_t lda, int32_t* ipiv, int32_t* info, cudaStream_t s) {
    constexpr int nb = PNB;
    auto panel = lu::lu_panel_la_kernel<PT, RPT, PNB>;
    auto panel_tma = lu::lu_panel_tma_kernel<PT, RPT, PNB>;
    FB_TRY((lu_la_attrs<PT, RPT, PNB>()));
    const Knobs& kn = knobs();
    // A/B knob FB_LU_TMA=0: cp.async panel kernel
    const bool use_tma = kn.lu_tma != 0 && (lda * 8) % 16 == 0 && ((uintptr_t)A & 15) == 0;
    CUtensorMap tmA;
    memset(&tmA, 0, sizeof(tmA));
    if (use_tma) FB_TRY(lu_tensor_map(&tmA, A, n, lda, PNB));
    LuStreams* ls;
    FB_TRY(lu_streams(&ls));
    // timing decomposition (FB_DEBUG_BUILD only; wrong results): 1 no GEMM, 2 no swap/TRSM, 4 no panel
    const int dbg = FB_DEBUG_BUILD ? kn.lu_debug : 0;
    const bool rank_simt = kn.lu_rank_simt != 0;  // A/B knob FB_LU_RANK_SIMT=0: DMMA GEMM trailing update
    cudaStream_t wst = kn.lu_serial == 1 ? s : ls->w;  // A/B knob: the wide parts on the caller's stream
    FB_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
    FB_CUDA_TRY(cudaEventRecord(ls->ev_fork, s));
    FB_CUDA_TRY(cudaStreamWaitEvent(ls->w, ls->ev_fork, 0));  // w starts after everything before the call
    for (int64_t j0 = 0; j0 < n; j0 += nb) {
        const int jb = (int)((n - j0) < nb ? (n - j0) : nb);
        const int has_prev = j0 > 0;
        const int k = (int)(j0 / nb);
        if (k >= 2) FB_CUDA_TRY(cudaStreamWaitEvent(s, ls->ev_w[k & 1], 0));  // wide_{k-2}
        const int64_t r0 = has_prev ? j0 - nb : j0;
        const size_t smem = (size_t)(n - r0) * PNB * sizeof(double) + (size_t)2 * PT * PNB * sizeof(double);
        if (!(dbg & 4)) {
            if (use_tma) {
                const size_t smem_tma = (size_t)((n - r0 + lu::LU_BOXR - 1) / lu::LU_BOXR) * lu::LU_BOXR * PNB *
                                            sizeof(double) +
                                        (size_t)2 * PT * PNB * sizeof(double) + 1024;
                FB_TRY(lu_launch(panel_tma, dim3(1), dim3(PT), smem_tma, s, A, lda, (int)n, (int)j0, jb, has_prev,
                                 ipiv, info, tmA));
            }
            else
                FB_TRY(lu_launch(panel, dim3(1), dim3(PT), smem, s, A, lda, (int)n, (int)j0, jb, has_prev, ipiv,
                                 info));
        }
        FB_CUDA_TRY(cudaEventRecord(ls->ev_p, s));
        // wide part of this step: everything except this panel and the next one
        FB_CUDA_TRY(cudaStreamWaitEvent(ls->w, ls->ev_p, 0));
        const int64_t nxt = (j0 + jb < n) ? ((n - j0 - jb) < nb ? (n - j0 - jb) : nb) : 0;
        const int64_t skip_end = j0 + jb + nxt;
        if (!(dbg & 2))
            FB_TRY(lu_launch(lu::lu_swap_trsm_wide_kernel, dim3((unsigned)((n + lu::SWAP_T - 1) / lu::SWAP_T)),
                             dim3(lu::SWAP_T), 0, wst, A, lda, (int)n, (int)j0, jb, (int)skip_end,
                             (const int32_t*)ipiv));
        const int64_t rest_r = n - j0 - jb, rest_c = n - skip_end;
        if (rest_r > 0 && rest_c > 0 && !(dbg & 1)) {
            double* A21 = A + (j0 + jb) * lda + j0;
            double* U12 = A + j0 * lda + skip_end;
            double* A22 = A + (j0 + jb) * lda + skip_end;
            if (rank_simt)
                FB_TRY(lu_launch(lu::lu_rank_update_kernel,
                                 dim3((unsigned)((rest_c + lu::RU_TN - 1) / lu::RU_TN),
                                      (unsigned)((rest_r + lu::RU_TM - 1) / lu::RU_TM)),
                                 dim3(lu::RU_T), 0, wst, A22, (const double*)A21, (const double*)U12, lda,
                                 (int)rest_r, (int)rest_c, jb));
            else
                FB_TRY(gemm_f64_sub_device(rest_r, rest_c, jb, A21, lda, U12, lda, A22, lda, wst));
        }
        FB_CUDA_TRY(cudaEventRecord(ls->ev_w[k & 1], wst));
    }
    const int klast = (int)((n - 1) / nb);
    FB_CUDA_TRY(cudaStreamWaitEvent(s, ls->ev_w[klast & 1], 0));  // join: the last wide part
    return FB_OK;
}

// The look-ahead schedule (~3 n/8 kernels + events on two streams) is captured once per
// (A, n, lda, ipiv, info, device) into a CUDA graph and replayed on the caller's stream: the
// per-step dependency resolution happens inside the graph instead of through stream/event
// round trips (knob FB_LU_GRAPH=0 enqueues the schedule directly).  A small per-thread cache
// holds the instantiated graphs.
struct LuGraph {
    double* A = nullptr;
    int64_t n = 0, lda = 0;
    int32_t* ipiv = nullptr;
    int32_t* info = nullptr;
    int dev = -1;
    cudaGraphExec_t exec = nullptr;
};

static fb_status lu_device_la_any(int64_t n, double* A, int64_t lda, int32_t* ipiv, int32_t* info, cudaStream_t s) {
    if (n <= 2048) return lu_device_la<512, 4, lu::NB>(n, A, lda, ipiv, info, s);
    return lu_device_la<1024, 4, lu::NB / 2>(n, A, lda, ipiv, info, s);
}

static fb_status lu_device_graph(int64_t n, double* A, int64_t lda, int32_t* ipiv, int32_t* info, cudaStream_t s) {
    thread_local static LuGraph cache[4];
    thread_local static int victim = 0;
    thread_local static cudaStream_t cap[32] = {};
    int dev = 0;
    FB_CUDA_TRY(cudaGetDevice(&dev));
    for (auto& g : cache)
        if (g.exec && g.A == A && g.n == n && g.lda == lda && g.ipiv == ipiv && g.info == info && g.dev == dev) {
            FB_CUDA_TRY(cudaGraphLaunch(g.exec, s));
            return FB_OK;
        }
    FB_TRY((n <= 2048 ? lu_la_attrs<512, 4, lu::NB>() : lu_la_attrs<1024, 4, lu::NB / 2>()));
    if (!cap[dev & 31]) FB_CUDA_TRY(cudaStreamCreateWithFlags(&cap[dev & 31], cudaStreamNonBlocking));
    cudaStream_t cs = cap[dev & 31];
    FB_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    const fb_status st = lu_device_la_any(n, A, lda, ipiv, info, cs);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
    if (st != FB_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (ce != cudaSuccess) {
        set_error("LU graph capture failed: %s", cudaGetErrorString(ce));
        return FB_ERR_CUDA;
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
        set_error("LU graph instantiation failed: %s", cudaGetErrorString(ie));
        return FB_ERR_CUDA;
    }
    LuGraph& g = cache[victim];
    victim = (victim + 1) % 4;
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.A = A;
    g.n = n;
    g.lda = lda;
    g.ipiv = ipiv;
    g.info = info;
    g.dev = dev;
    g.exec = exec;
    FB_CUDA_TRY(cudaGraphLaunch(exec, s));
    return FB_OK;
}

fb_status lu_device(int64_t n, double* A, int64_t lda, int32_t* ipiv, int32_t* info, cudaStream_t s) {
    if (knobs().lu_lookahead != 0) {
        if (knobs().lu_graph != 0) return lu_device_graph(n, A, lda, ipiv, info, s);
        return lu_device_la_any(n, A, lda, ipiv, info, s);
    }
    FB_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int32_t), s));
    const bool small = n <= 2048;
    const int nb = small ? lu::NB : lu::NB / 2;
    for (int64_t j0 = 0; j0 < n; j0 += nb) {
        const int jb = (int)((n - j0) < nb ? (n - j0) : nb);
        if (small)
            FB_TRY(lu_launch(lu::lu_panel_kernel<512, 4, lu::NB>, dim3(1), dim3(512),
                             (size_t)(n - j0) * lu::NB * sizeof(double), s, A, lda, (int)n, (int)j0, jb, ipiv, info));
        else
            FB_TRY(lu_launch(lu::lu_panel_kernel<1024, 4, lu::NB / 2>, dim3(1), dim3(1024),
                             (size_t)(n - j0) * (lu::NB / 2) * sizeof(double), s, A, lda, (int)n, (int)j0, jb, ipiv,
                             info));
        FB_TRY(lu_launch(lu::lu_swap_trsm_kernel, dim3((unsigned)((n + lu::SWAP_T - 1) / lu::SWAP_T)),
                         dim3(lu::SWAP_T), 0, s, A, lda,
                         (int)n, (int)j0, jb, (const int32_t*)ipiv));
        const int64_t rest = n - j0 - jb;
        if (rest > 0) {
            double* A21 = A + (j0 + jb) * lda + j0;
            double* U12 = A + j0 * lda + j0 + jb;
            double* A22 = A + (j0 + jb) * lda + j0 + jb;
            FB_TRY(gemm_f64_sub_device(rest, rest, jb, A21, lda, U12, lda, A22, lda, s));
        }
    }
    return FB_OK;
}

}  // namespace fb

using namespace fb;

extern "C" {

size_t fb_lu_workspace_bytes(int dtype, int64_t n) { return (dtype == FB_F64 && n > 0) ? lu_ws_bytes(n) : 0; }

fb_status fb_lu(int dtype, int64_t n, void* A, int64_t lda, int32_t* ipiv, int32_t* info, void* ws, size_t ws_bytes,
                void* stream) {
    clear_error();
    (void)ws;
    (void)ws_bytes;
    if (dtype != FB_F64) {
        set_error("fb_lu: only FB_F64 is implemented");
        return FB_ERR_INVALID_VALUE;
    }
    if (n <= 0 || !A || !ipiv || !info || lda < n) {
        set_error("fb_lu: bad arguments");
        return FB_ERR_INVALID_VALUE;
    }
    if (n > lu::NMAX) {
        set_error("fb_lu: n <= %d supported", lu::NMAX);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    if (!aligned16(A) || (lda * 8) % 16) {
        set_error("fb_lu: A must be 16-byte aligned with lda even");
        return FB_ERR_MISALIGNED;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    return lu_device(n, (double*)A, lda, ipiv, info, (cudaStream_t)stream);
}

}  // extern "C"
