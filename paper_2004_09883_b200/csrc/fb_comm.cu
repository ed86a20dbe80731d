// fb_comm.cu -- multi-GPU partitioning of the two blocks over one NVLink/NVSwitch box
// (north_star (4)): the slab-sharded 2D FFT whose global transpose is one NCCL all-to-all,
// and the row-block GEMM with B broadcast.  One process per GPU; NCCL communicator from a
// unique id the caller distributes (torch.distributed in the Python binding).
//
// Fused transpose: when every rank is load/store reachable over NVLink
// (NCCL LSA team = world), each rank owns a receive window in NCCL symmetric memory and the
// row pass moves the column blocks itself -- forward: stores element k of a local row into
// the window of rank k / (n1/P) (push); inverse: loads it from there (pull) -- so the
// transpose costs no staging buffer, no NCCL copy kernel and no extra HBM round trip, and
// the NVLink traffic overlaps the FFT arithmetic tile by tile.  Ordering uses the NCCL 2.28
// device API (ncclLsaBarrierSession, acquire/release at system scope) in two one-CTA kernels
// per call: before the row pass (peers are done with the windows of the previous call) and
// after it (every peer's blocks have landed).
#include <nccl.h>
#include <nccl_device.h>
#include <stdlib.h>
#include <string.h>

#include "fb_common.cuh"

struct fb_comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, size = 1, device = 0;
    // fused path
    int fused = 0;                         // 1: LSA team == world and the device comm is up
    char fused_why[256] = "not initialised";
    bool devcomm_ok = false;
    ncclDevComm devcomm{};
    void* win_buf = nullptr;               // this rank's receive window (ncclMemAlloc)
    size_t win_bytes = 0;
    ncclWindow_t win = nullptr;
    float2* peer_base[fb::kMaxPeers] = {};  // window bases of every rank, as mapped here
    // row-block GEMM: panel broadcasts run on their own stream
    cudaStream_t cstream = nullptr;
    cudaEvent_t cev = nullptr;
    cudaEvent_t ev_bcast[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr};  // panel slots
    int* flag_dev = nullptr;  // one int for the collective agreements (agree_min)
};

namespace fb {

#define FB_NCCL_TRY(expr, comm)                                                                 \
    do {                                                                                        \
        ncclResult_t _r = (expr);                                                               \
        if (_r != ncclSuccess) {                                                                \
            ::fb::set_error("%s failed: %s (%s)", #expr, ncclGetErrorString(_r),                \
                            (comm) ? ncclGetLastError(comm) : "");                              \
            return FB_ERR_NCCL;                                                                 \
        }                                                                                       \
    } while (0)

static LineMap lmap(int64_t hi, int64_t lo, int64_t es, int kb_shift = 30, int64_t bs = 0) {
    LineMap m;
    m.hi = hi;
    m.lo = lo;
    m.es = es;
    m.kb_shift = kb_shift;
    m.bs = bs;
    return m;
}

static fb_status check_slab(fb_comm* c, const void* a, const void* b, int64_t n0, int64_t n1,
                            void* ws, size_t ws_bytes) {
    if (!c || !c->nccl) {
        set_error("communicator is null or destroyed");
        return FB_ERR_NOT_INITIALIZED;
    }
    if (n0 <= 0 || n1 <= 0) {
        set_error("n0, n1 must be >= 1");
        return FB_ERR_INVALID_VALUE;
    }
    if (!is_pow2(n0) || !is_pow2(n1) || n0 > kTwN || n1 > kTwN) {
        set_error("FFT sizes must be powers of two in [1, %d]", kTwN);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    if (n0 % c->size || n1 % c->size) {
        set_error("n0 and n1 must be divisible by the world size %d", c->size);
        return FB_ERR_INVALID_VALUE;
    }
    if (!a || !b) {
        set_error("null input or output");
        return FB_ERR_INVALID_VALUE;
    }
    if (!aligned16(a) || !aligned16(b) || !aligned16(ws)) {
        set_error("buffers must be 16-byte aligned");
        return FB_ERR_MISALIGNED;
    }
    const size_t slab = (size_t)(n0 / c->size) * n1 * sizeof(float2);
    if (ranges_overlap(a, slab, b, slab)) {
        set_error("input and output slabs must not overlap");
        return FB_ERR_INVALID_VALUE;
    }
    if (!ws || ws_bytes < 2 * slab) {
        set_error("slab workspace of %zu bytes required, got %zu", 2 * slab, ws_bytes);
        return FB_ERR_WORKSPACE;
    }
    if (ranges_overlap(ws, 2 * slab, a, slab) || ranges_overlap(ws, 2 * slab, b, slab)) {
        set_error("workspace overlaps input or output");
        return FB_ERR_INVALID_VALUE;
    }
    return FB_OK;
}

// ---------------------------------------------------------------- fused transpose plumbing
__global__ void lsa_barrier_kernel(ncclDevComm dc) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

__global__ void lsa_pointers_kernel(ncclWindow_t w, int n, const int* lsa_of_rank, void** out) {
    const int p = threadIdx.x;
    if (p < n) out[p] = ncclGetLsaPointer(w, 0, lsa_of_rank[p]);
}

static fb_status lsa_barrier(fb_comm* c, cudaStream_t s) {
    lsa_barrier_kernel<<<1, 32, 0, s>>>(c->devcomm);
    FB_LAUNCH_CHECK("lsa barrier");
    return FB_OK;
}

// Collective (called by every rank from fb_comm_init): decide whether the fused path is
// available and create the device communicator with one LSA barrier.
static void fused_probe(fb_comm* c) {
    if (knobs().slab_fused == 0) {
        snprintf(c->fused_why, sizeof(c->fused_why), "disabled by FB_SLAB_FUSED=0");
        return;
    }
    if (c->size > kMaxPeers) {
        snprintf(c->fused_why, sizeof(c->fused_why), "world size %d > %d", c->size, kMaxPeers);
        return;
    }
    const ncclTeam_t lsa = ncclTeamLsa(c->nccl);
    if (lsa.nRanks != c->size) {
        snprintf(c->fused_why, sizeof(c->fused_why), "LSA team has %d of %d ranks (not one NVLink domain)",
                 lsa.nRanks, c->size);
        return;
    }
    ncclDevCommRequirements reqs;
    memset(&reqs, 0, sizeof(reqs));
    reqs.lsaBarrierCount = 1;
    const ncclResult_t r = ncclDevCommCreate(c->nccl, &reqs, &c->devcomm);
    if (r != ncclSuccess) {
        snprintf(c->fused_why, sizeof(c->fused_why), "ncclDevCommCreate: %s (%s)", ncclGetErrorString(r),
                 ncclGetLastError(c->nccl));
        return;
    }
    c->devcomm_ok = true;
    c->fused = 1;
    snprintf(c->fused_why, sizeof(c->fused_why), "fused (LSA team of %d)", c->size);
}

// Collective agreement: every rank contributes `ok`; returns the minimum over the world
// (ncclAllReduce on the caller's stream, then a host sync).  Returns -1 if NCCL itself fails.
static int agree_min(fb_comm* c, int ok, cudaStream_t s) {
    if (!c->flag_dev && cudaMalloc(&c->flag_dev, sizeof(int)) != cudaSuccess) return -1;
    int v = ok;
    if (cudaMemcpyAsync(c->flag_dev, &v, sizeof(int), cudaMemcpyHostToDevice, s) != cudaSuccess) return -1;
    if (ncclAllReduce(c->flag_dev, c->flag_dev, 1, ncclInt32, ncclMin, c->nccl, s) != ncclSuccess) return -1;
    if (cudaMemcpyAsync(&v, c->flag_dev, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess) return -1;
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    return v;
}

static void release_window(fb_comm* c) {
    if (c->win) ncclCommWindowDeregister(c->nccl, c->win);
    c->win = nullptr;
    if (c->win_buf) ncclMemFree(c->win_buf);
    c->win_buf = nullptr;
    c->win_bytes = 0;
}

// Map every rank's window base (as seen from this GPU) into c->peer_base.
static bool map_peers(fb_comm* c) {
    int lsa_of_rank[kMaxPeers];
    const ncclTeam_t world = ncclTeamWorld(c->nccl);
    for (int p = 0; p < c->size; ++p) lsa_of_rank[p] = ncclTeamRankToLsa(c->nccl, world, p);
    void* dbuf = nullptr;
    if (cudaMalloc(&dbuf, kMaxPeers * (sizeof(void*) + sizeof(int))) != cudaSuccess) return false;
    void** dptr = (void**)dbuf;
    int* dlsa = (int*)(dptr + kMaxPeers);
    cudaError_t ce = cudaMemcpy(dlsa, lsa_of_rank, c->size * sizeof(int), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) {
        lsa_pointers_kernel<<<1, 32>>>(c->win, c->size, dlsa, dptr);
        ce = cudaGetLastError();
    }
    void* host[kMaxPeers] = {};
    if (ce == cudaSuccess) ce = cudaMemcpy(host, dptr, c->size * sizeof(void*), cudaMemcpyDeviceToHost);
    cudaFree(dbuf);
    if (ce != cudaSuccess) return false;
    for (int p = 0; p < c->size; ++p) c->peer_base[p] = (float2*)host[p];
    return true;
}

// Collective (every rank makes the same slab calls, so every rank reaches this together with
// the same `bytes`): (re)allocate and register the receive window and map every rank's base.
// Each step that can fail on one rank alone is followed by an agreement (allreduce MIN of a
// success flag), so either every rank ends with a mapped window or every rank releases its
// part and switches to the ncclAlltoAll path -- no rank is left in a collective the others
// skipped, and no rank pushes into a window a peer never mapped.  Growing the window first
// quiesces the old one: this rank's stream is synchronised and the agreement doubles as a
// barrier, so no peer still reads or writes the old window when it is freed.
static fb_status ensure_window(fb_comm* c, size_t bytes, cudaStream_t s) {
    if (c->win_bytes >= bytes) return FB_OK;
    const char* why = nullptr;
    if (c->win) {
        const int q = (cudaStreamSynchronize(s) == cudaSuccess) ? 1 : 0;
        if (agree_min(c, q, s) != 1) why = "quiescing the previous window failed";
        release_window(c);
    }
    int ok = 0;
    if (!why) {
        ok = ncclMemAlloc(&c->win_buf, bytes) == ncclSuccess;
        if (!ok) c->win_buf = nullptr;
        if (agree_min(c, ok, s) != 1) why = "ncclMemAlloc failed on some rank";
    }
    if (!why) {  // collective registration: every rank has a buffer
        ok = ncclCommWindowRegister(c->nccl, c->win_buf, bytes, &c->win, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess;
        if (!ok) c->win = nullptr;
        if (agree_min(c, ok, s) != 1) why = "ncclCommWindowRegister failed on some rank";
    }
    if (!why) {
        ok = map_peers(c) ? 1 : 0;
        if (agree_min(c, ok, s) != 1) why = "mapping the symmetric window failed on some rank";
    }
    if (why) {
        release_window(c);
        set_error("symmetric window of %zu bytes unavailable: %s", bytes, why);
        return FB_ERR_NCCL;
    }
    c->win_bytes = bytes;
    return FB_OK;
}

// A window that cannot be set up on every rank turns the communicator's fused path off for
// good, on every rank at once (ensure_window agrees collectively); the call then proceeds on
// ncclAlltoAll.
static fb_status ensure_window_or_fallback(fb_comm* c, size_t bytes, cudaStream_t s) {
    const fb_status st = ensure_window(c, bytes, s);
    if (st != FB_OK) {
        snprintf(c->fused_why, sizeof(c->fused_why), "%s", fb_last_error_detail());
        clear_error();
    }
    return st;
}

// The fused passes, shared by the real path and the single-GPU model (fb_fft2d_slab_model).
// win[d] = base of rank d's receive window (n0 x cols natural column strip).
// Forward row pass of rank r: row i of the slab -> element k to win[k / cols][(r rows + i) cols + k mod cols].
static fb_status slab_rows_push(const float2* x_rows, float2* const* win, int r, int P, int64_t n0, int64_t n1,
                                const DeviceState* st, cudaStream_t s) {
    const int64_t rows = n0 / P, cols = n1 / P;
    FftPass p{};
    p.in = x_rows;
    p.log2L = ilog2(n1);
    p.nlines = rows;
    p.g_shift = 0;
    p.lin = lmap(n1, 0, 1);
    p.lout = lmap(cols, 0, 1, ilog2(cols), 0);
    p.scale = 1.f;
    for (int d = 0; d < P; ++d) p.peer[d] = win[d] + (int64_t)r * rows * cols;
    p.out = p.peer[0];  // P == 1: one block, plain store
    p.peer_out = P > 1;
    return launch_fft_pass(p, st, s);
}

// Inverse row pass of rank r: element k of local row i <- win[k / cols][(r rows + i) cols + k mod cols].
static fb_status slab_rows_pull(float2* const* win, float2* x_rows, int r, int P, int64_t n0, int64_t n1,
                                const DeviceState* st, cudaStream_t s) {
    const int64_t rows = n0 / P, cols = n1 / P;
    FftPass p{};
    p.out = x_rows;
    p.log2L = ilog2(n1);
    p.nlines = rows;
    p.g_shift = 0;
    p.lin = lmap(cols, 0, 1, ilog2(cols), 0);
    p.lout = lmap(n1, 0, 1);
    p.conj_out = 1;
    p.scale = 1.0f / (float)((double)n0 * (double)n1);
    for (int d = 0; d < P; ++d) p.peer[d] = win[d] + (int64_t)r * rows * cols;
    p.in = p.peer[0];
    p.peer_in = P > 1;
    return launch_fft_pass(p, st, s);
}

}  // namespace fb

using namespace fb;

extern "C" {

size_t fb_comm_unique_id_bytes(void) { return NCCL_UNIQUE_ID_BYTES; }

fb_status fb_comm_unique_id(void* uid_out) {
    clear_error();
    if (!uid_out) {
        set_error("null uid buffer");
        return FB_ERR_INVALID_VALUE;
    }
    ncclUniqueId id;
    FB_NCCL_TRY(ncclGetUniqueId(&id), (ncclComm_t) nullptr);
    memcpy(uid_out, &id, sizeof(id));
    return FB_OK;
}

fb_status fb_comm_init(fb_comm** comm, int nranks, int rank, const void* uid, int device) {
    clear_error();
    if (!comm || !uid || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("bad fb_comm_init arguments");
        return FB_ERR_INVALID_VALUE;
    }
    FB_TRY(fb_init(device));
    FB_CUDA_TRY(cudaSetDevice(device));
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    fb_comm* c = new fb_comm();
    c->rank = rank;
    c->size = nranks;
    c->device = device;
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        set_error("ncclCommInitRank failed: %s", ncclGetErrorString(r));
        delete c;
        return FB_ERR_NCCL;
    }
    fused_probe(c);
    *comm = c;
    return FB_OK;
}

fb_status fb_comm_destroy(fb_comm* c) {
    clear_error();
    if (!c) return FB_OK;
    fb_status st = FB_OK;
    // the window may still be in use by this rank's queued work: drain the device first
    if (c->win || c->win_buf) cudaDeviceSynchronize();
    if (c->nccl && c->win) {
        if (ncclCommWindowDeregister(c->nccl, c->win) != ncclSuccess) st = FB_ERR_NCCL;
        c->win = nullptr;
    }
    if (c->win_buf) {
        if (ncclMemFree(c->win_buf) != ncclSuccess) st = FB_ERR_NCCL;
        c->win_buf = nullptr;
    }
    if (c->cev) cudaEventDestroy(c->cev);
    for (int i = 0; i < 2; ++i) {
        if (c->ev_bcast[i]) cudaEventDestroy(c->ev_bcast[i]);
        if (c->ev_used[i]) cudaEventDestroy(c->ev_used[i]);
    }
    if (c->flag_dev) cudaFree(c->flag_dev);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->nccl && c->devcomm_ok) {
        if (ncclDevCommDestroy(c->nccl, &c->devcomm) != ncclSuccess) st = FB_ERR_NCCL;
        c->devcomm_ok = false;
    }
    if (c->nccl) {
        ncclResult_t r = ncclCommDestroy(c->nccl);
        if (r != ncclSuccess) {
            set_error("ncclCommDestroy failed: %s", ncclGetErrorString(r));
            st = FB_ERR_NCCL;
        }
        c->nccl = nullptr;
    }
    delete c;
    return st;
}

int fb_comm_rank(const fb_comm* c) { return c ? c->rank : -1; }
int fb_comm_size(const fb_comm* c) { return c ? c->size : -1; }
int fb_comm_fused(fb_comm* c) { return (c && c->fused) ? 1 : 0; }
const char* fb_comm_fused_detail(const fb_comm* c) { return c ? c->fused_why : "null communicator"; }

size_t fb_fft2d_slab_workspace_bytes(int nranks, int64_t n0, int64_t n1) {
    if (nranks < 1 || n0 <= 0 || n1 <= 0 || n0 % nranks) return 0;
    return 2 * (size_t)(n0 / nranks) * (size_t)n1 * sizeof(float2);
}

// Forward: natural row slab (n0/P x n1) -> column slab (n0 x n1/P).
//   1. row FFTs, the store scatters element k of local row i into the per-peer send block
//      d = k / (n1/P) at [i][k mod (n1/P)]  (pack fused into the row pass)
//   2. ncclAlltoAll: block from rank s lands at recv[s] = rows [s n0/P, (s+1) n0/P) of the
//      column strip -> recv IS the natural n0 x (n1/P) strip
//   3. column FFTs of length n0 on the strip (four-step if n0 > 4096)
fb_status fb_fft2d_slab(fb_comm* c, const void* x_rows, void* y_cols, int64_t n0, int64_t n1, void* ws,
                        size_t ws_bytes, void* stream) {
    clear_error();
    FB_TRY(check_slab(c, x_rows, y_cols, n0, n1, ws, ws_bytes));
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    const int P = c->size;
    const int64_t rows = n0 / P, cols = n1 / P;
    const size_t slab = (size_t)rows * n1;
    float2* send = (float2*)ws;
    float2* recv = send + slab;
    if (c->fused && ensure_window_or_fallback(c, slab * sizeof(float2), s) != FB_OK) c->fused = 0;
    if (c->fused) {
        FB_TRY(lsa_barrier(c, s));  // every peer is done with its window (previous call)
        FB_TRY(slab_rows_push((const float2*)x_rows, c->peer_base, c->rank, P, n0, n1, st, s));
        FB_TRY(lsa_barrier(c, s));  // every peer's blocks have landed in this rank's window
        return fft_columns((const float2*)c->win_buf, (float2*)y_cols, n0, cols, cols, cols, false, false, 1.f,
                           send, st, s);
    }

    FftPass p{};
    p.in = (const float2*)x_rows;
    p.out = send;
    p.log2L = ilog2(n1);
    p.nlines = rows;
    p.g_shift = 0;
    p.lin = lmap(n1, 0, 1);
    p.lout = lmap(cols, 0, 1, ilog2(cols), rows * cols);
    p.scale = 1.f;
    p.col_like = 0;
    FB_TRY(launch_fft_pass(p, st, s));
    FB_NCCL_TRY(ncclAlltoAll(send, recv, (size_t)rows * cols * 2, ncclFloat, c->nccl, s), c->nccl);
    return fft_columns(recv, (float2*)y_cols, n0, cols, cols, cols, false, false, 1.f, recv, st, s);
}

// Inverse: column slab (n0 x n1/P) -> natural row slab (n0/P x n1), scaled by 1/(n0 n1).
fb_status fb_ifft2d_slab(fb_comm* c, const void* y_cols, void* x_rows, int64_t n0, int64_t n1, void* ws,
                         size_t ws_bytes, void* stream) {
    clear_error();
    FB_TRY(check_slab(c, y_cols, x_rows, n0, n1, ws, ws_bytes));
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    const int P = c->size;
    const int64_t rows = n0 / P, cols = n1 / P;
    const size_t slab = (size_t)rows * n1;
    float2* send = (float2*)ws;
    float2* recv = send + slab;
    if (c->fused && ensure_window_or_fallback(c, slab * sizeof(float2), s) != FB_OK) c->fused = 0;
    if (c->fused) {
        FB_TRY(lsa_barrier(c, s));  // no peer still reads this rank's window (previous call)
        FB_TRY(fft_columns((const float2*)y_cols, (float2*)c->win_buf, n0, cols, cols, cols, true, false, 1.f, send,
                           st, s));
        FB_TRY(lsa_barrier(c, s));  // every peer's strip is complete
        return slab_rows_pull(c->peer_base, (float2*)x_rows, c->rank, P, n0, n1, st, s);
    }
    // 1. column IFFTs (conj in), natural strip into `send`: rows of peer d are contiguous
    FB_TRY(fft_columns((const float2*)y_cols, send, n0, cols, cols, cols, true, false, 1.f, recv, st, s));
    // 2. global transpose back
    FB_NCCL_TRY(ncclAlltoAll(send, recv, (size_t)rows * cols * 2, ncclFloat, c->nccl, s), c->nccl);
    // 3. row IFFTs; the load gathers element k of local row i from recv[k/(n1/P)][i][k mod (n1/P)]
    FftPass p{};
    p.in = recv;
    p.out = (float2*)x_rows;
    p.log2L = ilog2(n1);
    p.nlines = rows;
    p.g_shift = 0;
    p.lin = lmap(cols, 0, 1, ilog2(cols), rows * cols);
    p.lout = lmap(n1, 0, 1);
    p.conj_out = 1;
    p.scale = 1.0f / (float)((double)n0 * (double)n1);
    p.col_like = 0;
    return launch_fft_pass(p, st, s);
}

fb_status fb_fft2d_slab_model(int P, int inverse, void* x, void* y, int64_t n0, int64_t n1, void* win, void* ws,
                              size_t ws_bytes, void* stream) {
    clear_error();
    if (P < 1 || P > kMaxPeers || n0 <= 0 || n1 <= 0 || !x || !y || !win) {
        set_error("bad fb_fft2d_slab_model arguments");
        return FB_ERR_INVALID_VALUE;
    }
    if (!is_pow2(n0) || !is_pow2(n1) || n0 > kTwN || n1 > kTwN || n0 % P || n1 % P) {
        set_error("sizes must be powers of two <= %d divisible by P", kTwN);
        return FB_ERR_UNSUPPORTED_SIZE;
    }
    const int64_t rows = n0 / P, cols = n1 / P;
    const size_t slab = (size_t)rows * n1;
    if (!ws || ws_bytes < 2 * slab * sizeof(float2)) {
        set_error("slab workspace too small");
        return FB_ERR_WORKSPACE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    cudaStream_t s = (cudaStream_t)stream;
    float2* w[kMaxPeers];
    for (int d = 0; d < P; ++d) w[d] = (float2*)win + (int64_t)d * slab;
    float2* X = (float2*)x;
    float2* Y = (float2*)y;
    if (!inverse) {
        for (int r = 0; r < P; ++r) FB_TRY(slab_rows_push(X + (int64_t)r * slab, w, r, P, n0, n1, st, s));
        for (int d = 0; d < P; ++d)
            FB_TRY(fft_columns(w[d], Y + (int64_t)d * slab, n0, cols, cols, cols, false, false, 1.f, (float2*)ws, st,
                               s));
    } else {
        for (int d = 0; d < P; ++d)
            FB_TRY(fft_columns(Y + (int64_t)d * slab, w[d], n0, cols, cols, cols, true, false, 1.f, (float2*)ws, st,
                               s));
        for (int r = 0; r < P; ++r) FB_TRY(slab_rows_pull(w, X + (int64_t)r * slab, r, P, n0, n1, st, s));
    }
    return FB_OK;
}

}  // extern "C"

namespace fb {
// Row-block GEMM layout of the workspace: [A hi | A lo] (FP32 only) then two panel slots, each
// [packed B panel k x w (root's send buffer)] + (FP32) [panel hi | panel lo] (w x kp, K-major).
struct RowblockWs {
    int64_t w, kp;
    size_t a_split, slot_pack, slot_split, slot, total;
};
static RowblockWs rowblock_ws(int dtype, int64_t ml, int64_t n, int64_t k, int64_t panel) {
    RowblockWs r;
    const size_t es = dtype == FB_F64 ? 8 : 4;
    r.w = (panel > 0 && panel < n) ? panel : n;
    r.kp = (k + 3) / 4 * 4;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    r.a_split = dtype == FB_F32 ? al((size_t)2 * ml * r.kp * 4) : 0;
    r.slot_pack = al((size_t)k * r.w * es);
    r.slot_split = dtype == FB_F32 ? al((size_t)2 * r.w * r.kp * 4) : 0;
    r.slot = r.slot_pack + r.slot_split;
    const size_t dflt = gemm_ws_bytes(dtype, ml, n, k);  // one-panel fallback (fb_matmul)
    r.total = r.a_split + 2 * r.slot;
    if (r.total < dflt) r.total = dflt;
    return r;
}
}  // namespace fb

extern "C" {

size_t fb_matmul_rowblock_workspace_bytes(int nranks, int dtype, int64_t m, int64_t n, int64_t k) {
    if (nranks < 1 || m <= 0 || n <= 0 || k <= 0 || m % nranks) return 0;
    if (dtype != FB_F32 && dtype != FB_F64) return 0;
    return rowblock_ws(dtype, m / nranks, n, k, knobs().rowblock_panel).total;
}

// B is broadcast in N-column panels on the communicator's stream; the
// GEMM of panel j (C[:, panel j] = A B[:, panel j], full K) runs on the caller's stream as soon as
// panel j has landed, while panel j+1 is on the wire.  The root packs each panel into a
// workspace slot (two slots, reused once the panel's split / GEMM has consumed it); non-root
// ranks receive panel j into their B buffer at element offset k * j0, so after the call B on a
// non-root rank holds B panel by panel ([panel][k][w]).  Per element the arithmetic equals
// fb_matmul's (same K order and promotion chunks), so the result is bitwise the same.
fb_status fb_matmul_rowblock(fb_comm* c, int dtype, int64_t m, int64_t n, int64_t k, const void* A_rows,
                             int64_t lda, void* B, int64_t ldb, int root, void* C_rows, int64_t ldc,
                             void* ws, size_t ws_bytes, void* stream) {
    clear_error();
    if (!c || !c->nccl) {
        set_error("communicator is null or destroyed");
        return FB_ERR_NOT_INITIALIZED;
    }
    if ((dtype != FB_F32 && dtype != FB_F64) || m <= 0 || n <= 0 || k <= 0 || m % c->size || root < 0 ||
        root >= c->size) {
        set_error("bad dtype, sizes (m %% P must be 0) or root");
        return FB_ERR_INVALID_VALUE;
    }
    if (!B || ldb != n) {
        set_error("B must be a dense k x n buffer (ldb == n) on every rank");
        return FB_ERR_INVALID_VALUE;
    }
    const size_t es = dtype == FB_F64 ? 8 : 4;
    const ncclDataType_t t = dtype == FB_F64 ? ncclDouble : ncclFloat;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ml = m / c->size;
    const RowblockWs L = rowblock_ws(dtype, ml, n, k, knobs().rowblock_panel);
    if (!ws || ws_bytes < L.total || !aligned16(ws) || !aligned16(A_rows) || !aligned16(B) || !aligned16(C_rows) ||
        (lda * es) % 16 || (ldc * es) % 16 || (n * es) % 16 || (L.w * es) % 16 || lda < k || ldc < n) {
        set_error("row-block GEMM: operands / workspace (%zu bytes) invalid", L.total);
        return FB_ERR_INVALID_VALUE;
    }
    DeviceState* st;
    FB_TRY(ensure_device(nullptr, &st));
    if (L.w >= n) {  // one panel: plain broadcast + fb_matmul
        FB_NCCL_TRY(ncclBroadcast(B, B, (size_t)k * (size_t)n, t, root, c->nccl, s), c->nccl);
        return gemm_device(dtype, ml, n, k, A_rows, lda, B, ldb, C_rows, ldc, ws, ws_bytes, st, s);
    }
    if (!c->cstream) {
        FB_CUDA_TRY(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        FB_CUDA_TRY(cudaEventCreateWithFlags(&c->cev, cudaEventDisableTiming));
        for (int i = 0; i < 2; ++i) {
            FB_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_bcast[i], cudaEventDisableTiming));
            FB_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_used[i], cudaEventDisableTiming));
        }
    }
    char* w0 = (char*)ws;
    float* Ah = (float*)w0;
    float* Al = Ah + ml * L.kp;
    auto slot_pack = [&](int i) { return w0 + L.a_split + i * L.slot; };
    auto slot_split = [&](int i) { return (float*)(w0 + L.a_split + i * L.slot + L.slot_pack); };
    const bool is_root = c->rank == root;
    FB_CUDA_TRY(cudaEventRecord(c->cev, s));  // the panel traffic starts after everything before the call
    FB_CUDA_TRY(cudaStreamWaitEvent(c->cstream, c->cev, 0));
    // A's operands as fb_matmul forms them (raw hi + lo only by default), so the product is bitwise
    const bool a_raw = dtype == FB_F32 && knobs().gemm_ahi_raw != 0;
    if (dtype == FB_F32) {
        if (a_raw)
            FB_TRY(tf32_lo_device(ml, k, (const float*)A_rows, lda, Al, L.kp, s));
        else
            FB_TRY(tf32_split_device(0, ml, k, (const float*)A_rows, lda, Ah, Al, L.kp, st, s));
    }
    int j = 0;
    for (int64_t j0 = 0; j0 < n; j0 += L.w, ++j) {
        const int64_t w = (n - j0) < L.w ? (n - j0) : L.w;
        const int sl = j & 1;
        // panel j on the wire (communicator stream); the root's slot is free once panel j-2 was consumed
        void* panel = is_root ? (void*)slot_pack(sl) : (void*)((char*)B + (size_t)k * j0 * es);
        if (is_root) {
            if (j >= 2) FB_CUDA_TRY(cudaStreamWaitEvent(c->cstream, c->ev_used[sl], 0));
            FB_CUDA_TRY(cudaMemcpy2DAsync(panel, (size_t)w * es, (const char*)B + (size_t)j0 * es, (size_t)n * es,
                                          (size_t)w * es, (size_t)k, cudaMemcpyDeviceToDevice, c->cstream));
        }
        FB_NCCL_TRY(ncclBroadcast(panel, panel, (size_t)k * (size_t)w, t, root, c->nccl, c->cstream), c->nccl);
        FB_CUDA_TRY(cudaEventRecord(c->ev_bcast[sl], c->cstream));
        // GEMM of panel j (caller's stream) as soon as it has landed
        FB_CUDA_TRY(cudaStreamWaitEvent(s, c->ev_bcast[sl], 0));
        if (dtype == FB_F32) {
            float* Bh = slot_split(sl);
            float* Bl = Bh + w * L.kp;
            FB_TRY(tf32_split_device(1, k, w, (const float*)panel, w, Bh, Bl, L.kp, st, s));
            FB_CUDA_TRY(cudaEventRecord(c->ev_used[sl], s));
            FB_TRY(gemm_3xtf32_presplit_device(ml, w, k, a_raw ? (const float*)A_rows : Ah, Al, L.kp, Bh, Bl, L.kp,
                                               (float*)C_rows + j0, ldc, s, 1.f, 0.f, a_raw ? lda : -1));
        } else {
            FB_TRY(gemm_device(FB_F64, ml, w, k, A_rows, lda, panel, w, (double*)C_rows + j0, ldc, nullptr, 0, st, s));
            FB_CUDA_TRY(cudaEventRecord(c->ev_used[sl], s));
        }
    }
    return FB_OK;
}

}  // extern "C"
