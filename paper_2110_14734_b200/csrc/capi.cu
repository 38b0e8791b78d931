// capi.cu -- the extern "C" boundary of libw1g.so (include/w1g.h) plus the
// context, buffer, flag and error plumbing shared by the stage translation
// units.  Each entry point cites the reference function it replaces.
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cstdarg>
#include <cstring>
#include <string>
#include <thread>

#include <emmintrin.h>

#include "common.cuh"

namespace w1g {

static thread_local char g_err[1024] = "";
unsigned long long g_launches = 0;

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e), what,
              file, line);
    if (e == cudaErrorMemoryAllocation) return W1G_ENOMEM;
    return W1G_ECUDA;
}

// the stream the calling thread's context launches on (set at every C-ABI entry
// and by the auxiliary RWMD thread): buffers grow stream-ordered on it, from the
// device's memory pool, so a first call at a new size does not stall the device
// on cudaFree's implicit synchronisation
static thread_local cudaStream_t g_tl_stream = nullptr;
static thread_local bool g_tl_capturing = false;
void set_thread_stream(cudaStream_t s) { g_tl_stream = s; }

int ensure_bytes(DevBuf &b, size_t bytes) {
    if (bytes <= b.cap) return W1G_OK;
    if (g_tl_capturing) return W1G_ERECAPTURE;  // graph_segment re-runs the body eagerly
    size_t want = bytes + bytes / 4 + 4096;
    cudaStream_t st = g_tl_stream;
    if (b.p) {
        cudaError_t e = st ? cudaFreeAsync(b.p, st) : cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
        if (e != cudaSuccess) return cuda_fail(e, "cudaFree", __FILE__, __LINE__);
    }
    cudaError_t e = st ? cudaMallocAsync(&b.p, want, st) : cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        b.p = nullptr;
        set_error("device allocation of %zu bytes failed: %s", want, cudaGetErrorString(e));
        return W1G_ENOMEM;
    }
    b.cap = want;
    return W1G_OK;
}

void free_buf(DevBuf &b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
}

int flags_reset(Ctx &c) {
    W1G_CUDA(cudaMemsetAsync(c.flags.p, 0, sizeof(int64_t) * F_NSLOTS, c.stream));
    return W1G_OK;
}

int stream_sync(Ctx &c) {
    c.n_syncs++;
    if (!c.timing) {
        W1G_CUDA(cudaStreamSynchronize(c.stream));
        return W1G_OK;
    }
    // the gap: from the last queued work finishing to the next work the host
    // can issue (an event recorded right after the wake-up runs immediately)
    W1G_CUDA(cudaEventRecord(c.sync_ev[0], c.stream));
    W1G_CUDA(cudaStreamSynchronize(c.stream));
    W1G_CUDA(cudaEventRecord(c.sync_ev[1], c.stream));
    W1G_CUDA(cudaEventSynchronize(c.sync_ev[1]));
    float ms = 0.f;
    W1G_CUDA(cudaEventElapsedTime(&ms, c.sync_ev[0], c.sync_ev[1]));
    c.sync_gap_us += 1e3 * ms;
    return W1G_OK;
}

namespace {
__global__ void k_to_host(const uint32_t *__restrict__ src, volatile uint32_t *dst, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

int to_host_small(Ctx &c, void *h_dst, const void *d_src, size_t bytes, cudaStream_t s) {
    const int n = (int)(bytes / 4);
    if (n <= 0) return W1G_OK;
    k_to_host<<<1, n < 256 ? ((n + 31) & ~31) : 256, 0, s ? s : c.stream>>>(
        static_cast<const uint32_t *>(d_src), static_cast<volatile uint32_t *>(h_dst), n);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

namespace {
__global__ void k_to_host2(const uint32_t *__restrict__ s0, volatile uint32_t *d0, int n0,
                           const uint32_t *__restrict__ s1, volatile uint32_t *d1, int n1) {
    for (int i = threadIdx.x; i < n0; i += blockDim.x) d0[i] = s0[i];
    for (int i = threadIdx.x; i < n1; i += blockDim.x) d1[i] = s1[i];
}
}  // namespace

// two small reads in one launch
int to_host_small2(Ctx &c, void *h0, const void *d0, size_t b0, void *h1, const void *d1, size_t b1) {
    const int n0 = (int)(b0 / 4), n1 = (int)(b1 / 4);
    const int n = n0 > n1 ? n0 : n1;
    if (n <= 0) return W1G_OK;
    k_to_host2<<<1, n < 256 ? ((n + 31) & ~31) : 256, 0, c.stream>>>(
        static_cast<const uint32_t *>(d0), static_cast<volatile uint32_t *>(h0), n0,
        static_cast<const uint32_t *>(d1), static_cast<volatile uint32_t *>(h1), n1);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

// copy into page-locked staging with non-temporal 16-byte stores (no read-for-ownership of
// the destination lines: the copy is bound by host memory traffic, and in the batch it
// runs on every worker next to the network expansion)
void host_copy_nt(void *dst, const void *src, size_t bytes) {
    char *d = static_cast<char *>(dst);
    const char *s = static_cast<const char *>(src);
    size_t i = 0;
    if ((reinterpret_cast<uintptr_t>(d) & 15) == 0) {
        for (; i + 64 <= bytes; i += 64) {
            const __m128i x0 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i));
            const __m128i x1 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 16));
            const __m128i x2 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 32));
            const __m128i x3 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(s + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i), x0);
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 16), x1);
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 32), x2);
            _mm_stream_si128(reinterpret_cast<__m128i *>(d + i + 48), x3);
        }
        _mm_sfence();
    }
    if (i < bytes) memcpy(d + i, s + i, bytes - i);
}

int graph_segment(Ctx &c, int slot, const std::function<int()> &body) {
    static const bool on = [] {  // opt-in: measured no better (measured and rejected)
        const char *e = getenv("W1G_GRAPHS");
        return e && *e == '1';
    }();
    if (!on || c.timing || c.gseg_off[slot] || g_tl_capturing) return body();
    if (cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        c.gseg_off[slot] = 1;
        return body();
    }
    g_tl_capturing = true;
    const int rc = body();
    g_tl_capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c.stream, &g);
    if (rc != W1G_OK || e != cudaSuccess || !g) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        // a buffer had to grow (next time it will not), or capture rejected an operation
        if (rc != W1G_ERECAPTURE) c.gseg_off[slot] = 1;
        return body();
    }
    cudaGraphExec_t &x = c.gseg[slot];
    bool ok = false;
    if (x) {
        cudaGraphExecUpdateResultInfo info;
        ok = cudaGraphExecUpdate(x, g, &info) == cudaSuccess;
        if (!ok) {
            cudaGetLastError();
            cudaGraphExecDestroy(x);
            x = nullptr;
        }
    }
    if (!ok) {
        const cudaError_t ei = cudaGraphInstantiate(&x, g, 0);
        if (ei != cudaSuccess) {
            cudaGetLastError();
            x = nullptr;
            cudaGraphDestroy(g);
            c.gseg_off[slot] = 1;
            return body();
        }
    }
    cudaGraphDestroy(g);
    W1G_CUDA(cudaGraphLaunch(x, c.stream));
    return W1G_OK;
}

int flags_fetch(Ctx &c, int first, int count) {
    W1G_TRY(to_host_small(c, c.h_pinned + first, dflags(c) + first, sizeof(int64_t) * count));
    W1G_TRY(stream_sync(c));
    return W1G_OK;
}

int stage_ensure(Ctx &c, size_t bytes) {
    if (bytes <= c.h_stage_cap) return W1G_OK;
    if (c.h_stage) {
        W1G_TRY(stream_sync(c));
        cudaFreeHost(c.h_stage);
        c.h_stage = nullptr;
        c.h_stage_cap = 0;
    }
    size_t want = bytes + bytes / 4 + 65536;
    W1G_CUDA(cudaHostAlloc(&c.h_stage, want, cudaHostAllocDefault));
    c.h_stage_cap = want;
    return W1G_OK;
}

int scan_prepare(Ctx &c, int64_t n, ScanArgs *a, int64_t *n_tiles) {
    int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles < 1) tiles = 1;
    unsigned long long *st;
    W1G_TRY(ensure(c.scan_state, (size_t)tiles + 8, &st));
    W1G_CUDA(cudaMemsetAsync(st, 0, sizeof(unsigned long long) * (tiles + 8), c.stream));
    a->status = st + 8;
    a->ticket = reinterpret_cast<unsigned int *>(st);
    *n_tiles = tiles;
    return W1G_OK;
}

static int upload(Ctx &c, DevBuf &dst, const void *src, size_t bytes) {
    void *d;
    W1G_TRY(ensure(dst, bytes, reinterpret_cast<char **>(&d)));
    if (bytes) W1G_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, c.stream));
    return W1G_OK;
}

static int download(Ctx &c, void *dst, const void *src, size_t bytes) {
    if (!dst || !bytes) return W1G_OK;
    W1G_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
    return W1G_OK;
}

// page-locked host memory the device can DMA from directly (null / empty: trivially yes)
static bool is_pinned(const void *p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

static void invalidate_from_nodes(Ctx &c) {
    // delta_condense's presorted split-tree lists describe the node set they were
    // built with: any rewrite of a node slot drops them (dc_run re-arms them)
    c.pre_n = 0;
    c.tree_valid = false;
    c.pairs_valid = false;
    c.arcs_valid = false;
    c.net_valid = false;
}

}  // namespace w1g

using namespace w1g;

#define CTX_CHECK(ctx)                                   \
    do {                                                 \
        if (!(ctx)) {                                    \
            set_error("null context");                   \
            return W1G_EINVAL;                           \
        }                                                \
        cudaError_t _e = cudaSetDevice((ctx)->device);   \
        if (_e != cudaSuccess) return cuda_fail(_e, "cudaSetDevice", __FILE__, __LINE__); \
        set_thread_stream((ctx)->stream);                \
    } while (0)

extern "C" {

int w1g_version(void) { return 10000; }

uint64_t w1g_launch_count(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int w1g_host_alloc(uint64_t bytes, void **out) {
    if (!out) return W1G_EINVAL;
    *out = nullptr;
    W1G_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
    return W1G_OK;
}

int w1g_host_free(void *p) {
    if (p) W1G_CUDA(cudaFreeHost(p));
    return W1G_OK;
}

int w1g_profile_rwmd_tile(w1g_ctx *c, int reps, float *ms_per_launch, int64_t *evals_per_launch) {
    CTX_CHECK(c);
    if (!c->nodes[0].valid) {
        set_error("profile_rwmd_tile: no nodes0");
        return W1G_ESTATE;
    }
    return rwmd_tile_profile(*c, reps, ms_per_launch, evals_per_launch);
}

int w1g_profile_rwmd(w1g_ctx *c, int reps, float *ms, int64_t *evals, int64_t *directed) {
    CTX_CHECK(c);
    if (!ms || !evals || !directed) return W1G_EINVAL;
    if (!c->nodes[0].valid) {
        set_error("profile_rwmd: no nodes0");
        return W1G_ESTATE;
    }
    return rwmd_profile(*c, reps, ms, evals, directed);
}

const char *w1g_last_error(void) { return g_err; }

int w1g_device_count(int *count) {
    W1G_CUDA(cudaGetDeviceCount(count));
    return W1G_OK;
}

int w1g_ctx_create(int device, w1g_ctx **out) {
    if (!out) return W1G_EINVAL;
    *out = nullptr;
    W1G_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    W1G_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0) {
        set_error("libw1g targets sm_100a (B200); device %d is sm_%d%d", device, prop.major, prop.minor);
        return W1G_ECUDA;
    }
    w1g_ctx *c = new w1g_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    if (const char *e = getenv("W1G_CULL_STEPS")) c->cull_steps = atoi(e) > 0 ? atoi(e) : 0;
    if (const char *e = getenv("W1G_DEBUG_RADIUS")) c->debug_radius = atoi(e) ? 1 : 0;
    if (const char *e = getenv("W1G_HEAVY")) c->heavy_ratio = atoi(e) > 0 ? atoi(e) : 0;
    if (const char *e = getenv("W1G_OVERLAP")) c->overlap = atoi(e) > 0 ? atoi(e) : 0;
    if (const char *e = getenv("W1G_OVERLAP_E2E")) c->overlap_e2e = atoi(e) > 0 ? atoi(e) : 0;
    if (const char *e = getenv("W1G_SPLIT_GATE")) {
        c->split_gate = atoi(e) > 0 ? atoi(e) : 0;
        c->split_gate_set = 1;
    }
    if (const char *e = getenv("W1G_SPLIT_GATE_E2E")) c->split_gate_e2e = atoi(e) > 0 ? atoi(e) : 0;
    {
        // contexts launch at the highest stream priority; the auxiliary RWMD
        // context drops to the lowest (start_rwmd), so when both have work the
        // block scheduler feeds the critical back end first
        int least = 0, greatest = 0;
        W1G_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        W1G_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, greatest));
        // the early part of the network's D2H copy (tails, row offsets) runs on its own stream
        W1G_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    }
    {
        // freed pool memory stays cached for the next growth (stream-ordered buffers)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    // the context's own buffers are ordered on its own stream; the caller's
    // thread keeps whatever stream it was working on
    struct RestoreStream {
        cudaStream_t prev;
        ~RestoreStream() { set_thread_stream(prev); }
    } restore{g_tl_stream};
    set_thread_stream(c->stream);
    int64_t *f;
    W1G_TRY(ensure(c->flags, F_NSLOTS, &f));
    W1G_CUDA(cudaHostAlloc(&c->h_pinned, sizeof(int64_t) * F_NSLOTS, cudaHostAllocDefault));
    for (auto &e : c->ev) W1G_CUDA(cudaEventCreate(&e));
    for (auto &e : c->sync_ev) W1G_CUDA(cudaEventCreate(&e));
    if (const char *e = getenv("W1G_TIMING")) c->timing = *e == '1';
    *out = c;
    return W1G_OK;
}

int w1g_ctx_destroy(w1g_ctx *c) {
    if (!c) return W1G_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    batch_destroy(*c);
    if (c->aux_worker) {
        c->aux_worker->stop();
        delete c->aux_worker;
        c->aux_worker = nullptr;
    }
    if (c->aux) {
        // its nodes0 is its own here: the non-split schedule drops the alias after every call,
        // the split one swaps buffers with this context
        w1g_ctx_destroy(static_cast<w1g_ctx *>(c->aux));
        c->aux = nullptr;
    }
    DevBuf *bufs[] = {&c->in_pts, &c->best[0], &c->best[1], &c->tree_pts, &c->t_left, &c->t_right,
                      &c->t_rep, &c->t_size, &c->t_bbox, &c->t_geom, &c->t_lr, &c->t_rep32,
                      &c->pair_uv, &c->pair_w, &c->pair_idx, &c->pair_counts,
                      &c->arc_t, &c->arc_h, &c->arc_c, &c->net_sup, &c->net_t, &c->net_h,
                      &c->net_c, &c->net_ro, &c->scan_state, &c->scan_state2, &c->flags, &c->pre_xl, &c->pre_yl,
                      &c->pre_cells, &c->pre_rows, &c->pre_rcnt};
    for (DevBuf *b : bufs) free_buf(*b);
    free_buf(c->wspd_ready);
    free_buf(c->wspd_ctr);
    delete c->fill_pool;
    c->fill_pool = nullptr;
    for (auto &x : c->gseg)
        if (x) {
            cudaGraphExecDestroy(x);
            x = nullptr;
        }
    for (NodeSet *ns_p : {&c->nodes[0], &c->nodes[1], &c->raw}) {
        NodeSet &ns = *ns_p;
        free_buf(ns.pts);
        free_buf(ns.am);
        free_buf(ns.bm);
        free_buf(ns.exa);
        free_buf(ns.exb);
    }
    for (auto &b : c->scr) free_buf(b);
    free_buf(c->prof_cnt);
    for (auto &side : c->prof_ev)
        for (auto &kind : side)
            for (auto &e : kind)
                if (e) cudaEventDestroy(e);
    free_buf(c->corpus_pts);
    free_buf(c->query_pts);
    for (auto &b : c->dense_scr) free_buf(b);
    delete[] c->h_corpus_off;
    delete[] c->h_corpus_ptr;
    for (int s2 = 0; s2 < 2; s2++) {
        free_buf(c->pw_nodes[s2]);
        free_buf(c->pw_lev[s2]);
    }
    for (auto &job : c->sort_scr)
        for (auto &b : job) free_buf(b);
    for (auto &job : c->lex_scr)
        for (auto &b : job) free_buf(b);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    for (auto &e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : c->sync_ev)
        if (e) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
    return W1G_OK;
}

void *w1g_ctx_stream(w1g_ctx *c) { return c ? (void *)c->stream : nullptr; }

int w1g_synchronize(w1g_ctx *c) {
    CTX_CHECK(c);
    W1G_TRY(stream_sync(*c));
    return W1G_OK;
}

// ---------------------------------------------------------------- nodes

int w1g_zero_condense_device(w1g_ctx *c, const double *d_a, int64_t na, const double *d_b,
                             int64_t nb, int64_t *k0, int32_t *balanced) {
    CTX_CHECK(c);
    if (na < 0 || nb < 0 || na + nb >= (1ll << 31)) {
        set_error("zero_condense: bad sizes na=%lld nb=%lld", (long long)na, (long long)nb);
        return W1G_EINVAL;
    }
    invalidate_from_nodes(*c);
    c->nodes[1].valid = false;
    return zc_run(*c, reinterpret_cast<const double2 *>(d_a), na,
                  reinterpret_cast<const double2 *>(d_b), nb, k0, balanced);
}

int w1g_zero_condense(w1g_ctx *c, const double *a, int64_t na, const double *b, int64_t nb,
                      int64_t *k0, int32_t *balanced) {
    CTX_CHECK(c);
    if (na < 0 || nb < 0) return W1G_EINVAL;
    double2 *d;
    W1G_TRY(ensure(c->in_pts, (size_t)(na + nb), &d));
    if (na) W1G_CUDA(cudaMemcpyAsync(d, a, sizeof(double2) * na, cudaMemcpyHostToDevice, c->stream));
    if (nb) W1G_CUDA(cudaMemcpyAsync(d + na, b, sizeof(double2) * nb, cudaMemcpyHostToDevice, c->stream));
    return w1g_zero_condense_device(c, reinterpret_cast<double *>(d), na,
                                    reinterpret_cast<double *>(d + na), nb, k0, balanced);
}

int w1g_load_nodes(w1g_ctx *c, int slot, const double *points, const int64_t *am,
                   const int64_t *bm, int64_t k, int64_t abar, int64_t bbar) {
    CTX_CHECK(c);
    if (slot < 0 || slot > 1 || k < 0 || k >= (1ll << 31)) return W1G_EINVAL;
    NodeSet &ns = c->nodes[slot];
    W1G_TRY(upload(*c, ns.pts, points, sizeof(double2) * k));
    W1G_TRY(upload(*c, ns.am, am, sizeof(int64_t) * k));
    W1G_TRY(upload(*c, ns.bm, bm, sizeof(int64_t) * k));
    ns.k = k;
    ns.valid = true;
    ns.abar = abar;
    ns.bbar = bbar;
    ns.na = ns.nb = -1;
    ns.stats = false;
    invalidate_from_nodes(*c);
    if (slot == 0) c->nodes[1].valid = false;
    return W1G_OK;
}

int w1g_nodes_size(w1g_ctx *c, int slot, int64_t *k) {
    CTX_CHECK(c);
    if (slot < 0 || slot > 1 || !c->nodes[slot].valid) {
        set_error("node slot %d is empty", slot);
        return W1G_ESTATE;
    }
    *k = c->nodes[slot].k;
    return W1G_OK;
}

int w1g_fetch_nodes(w1g_ctx *c, int slot, double *points, int64_t *am, int64_t *bm) {
    CTX_CHECK(c);
    if (slot < 0 || slot > 1 || !c->nodes[slot].valid) {
        set_error("node slot %d is empty", slot);
        return W1G_ESTATE;
    }
    NodeSet &ns = c->nodes[slot];
    W1G_TRY(download(*c, points, ns.pts.p, sizeof(double2) * ns.k));
    W1G_TRY(download(*c, am, ns.am.p, sizeof(int64_t) * ns.k));
    W1G_TRY(download(*c, bm, ns.bm.p, sizeof(int64_t) * ns.k));
    W1G_TRY(stream_sync(*c));
    return W1G_OK;
}

// ---------------------------------------------------------------- rwmd

int w1g_rwmd(w1g_ctx *c, double *L, double *LA, double *LB) {
    CTX_CHECK(c);
    if (!c->nodes[0].valid) {
        set_error("rwmd: no nodes0 (call zero_condense or load_nodes first)");
        return W1G_ESTATE;
    }
    double l, la, lb;
    W1G_TRY(rwmd_run(*c, &l, &la, &lb));
    if (L) *L = l;
    if (LA) *LA = la;
    if (LB) *LB = lb;
    return W1G_OK;
}

int w1g_fetch_rwmd_best(w1g_ctx *c, int side, double *best, int64_t *n) {
    CTX_CHECK(c);
    if (side < 0 || side > 1) return W1G_EINVAL;
    *n = c->n_best[side];
    if (best) {
        W1G_TRY(download(*c, best, c->best[side].p, sizeof(double) * c->n_best[side]));
        W1G_TRY(stream_sync(*c));
    }
    return W1G_OK;
}

int w1g_rwmd_range(w1g_ctx *c, int side, int64_t begin, int64_t end, double *partial,
                   int64_t *n_members) {
    CTX_CHECK(c);
    if (!c->nodes[0].valid) {
        set_error("rwmd_range: no nodes0");
        return W1G_ESTATE;
    }
    if (side < 0 || side > 1 || !partial || !n_members) return W1G_EINVAL;
    return rwmd_range_run(*c, side, begin, end, partial, n_members);
}

int w1g_member_counts(w1g_ctx *c, int64_t *n_a, int64_t *n_b) {
    CTX_CHECK(c);
    NodeSet &ns = c->nodes[0];
    if (!ns.valid) {
        set_error("member_counts: no nodes0");
        return W1G_ESTATE;
    }
    if (ns.stats) {  // zero_condense delivered them
        *n_a = ns.nmem[0];
        *n_b = ns.nmem[1];
        return W1G_OK;
    }
    double dummy;
    W1G_TRY(rwmd_range_run(*c, 0, 0, 0, &dummy, n_a));
    W1G_TRY(rwmd_range_run(*c, 1, 0, 0, &dummy, n_b));
    return W1G_OK;
}

int w1g_set_rwmd_culling(w1g_ctx *c, int enabled) {
    if (!c) return W1G_EINVAL;
    c->culling = enabled ? 1 : 0;
    return W1G_OK;
}

// ---------------------------------------------------------------- delta condense

int w1g_delta_condense(w1g_ctx *c, double delta, double pitch, double half_width, uint64_t seed,
                       int64_t *k) {
    CTX_CHECK(c);
    if (!c->nodes[0].valid) {
        set_error("delta_condense: no nodes0");
        return W1G_ESTATE;
    }
    if (!(delta >= 0.0)) {
        set_error("delta must be nonnegative");
        return W1G_EINVAL;
    }
    invalidate_from_nodes(*c);
    return dc_run(*c, delta, pitch, half_width, seed, k);
}

int w1g_snap_points(w1g_ctx *c, const double *points, int64_t n, double pitch, double *snapped,
                    int64_t *cells) {
    CTX_CHECK(c);
    if (n < 0 || !(pitch > 0.0)) {
        set_error("delta must be positive");
        return W1G_EINVAL;
    }
    return snap_run(*c, points, n, pitch, snapped, cells);
}

// ---------------------------------------------------------------- split tree

int w1g_split_tree(w1g_ctx *c, int slot, int64_t *n_nodes, int32_t *depth) {
    CTX_CHECK(c);
    if (slot < 0 || slot > 1 || !c->nodes[slot].valid) {
        set_error("split_tree: node slot %d is empty", slot);
        return W1G_ESTATE;
    }
    c->pairs_valid = false;
    c->arcs_valid = false;
    c->net_valid = false;
    NodeSet &ns = c->nodes[slot];
    return tree_run(*c, ptr<double2>(ns.pts), ns.k, n_nodes, depth);
}

int w1g_fetch_tree(w1g_ctx *c, int64_t *left, int64_t *right, double *bbox, int64_t *rep,
                   int64_t *size) {
    CTX_CHECK(c);
    if (!c->tree_valid) {
        set_error("no split tree");
        return W1G_ESTATE;
    }
    const size_t nn = (size_t)c->tree_n_nodes;
    W1G_TRY(download(*c, left, c->t_left.p, sizeof(int64_t) * nn));
    W1G_TRY(download(*c, right, c->t_right.p, sizeof(int64_t) * nn));
    W1G_TRY(download(*c, bbox, c->t_bbox.p, sizeof(double) * 4 * nn));
    W1G_TRY(download(*c, rep, c->t_rep.p, sizeof(int64_t) * nn));
    W1G_TRY(download(*c, size, c->t_size.p, sizeof(int64_t) * nn));
    W1G_TRY(stream_sync(*c));
    return W1G_OK;
}

int w1g_load_tree(w1g_ctx *c, const double *points, int64_t n_points, const int64_t *left,
                  const int64_t *right, const double *bbox, const int64_t *rep, int64_t n_nodes) {
    CTX_CHECK(c);
    if (n_points < 0 || n_nodes < 0 || n_nodes >= (1ll << 31)) return W1G_EINVAL;
    c->pairs_valid = false;
    c->arcs_valid = false;
    c->net_valid = false;
    W1G_TRY(upload(*c, c->tree_pts, points, sizeof(double2) * n_points));
    W1G_TRY(upload(*c, c->t_left, left, sizeof(int64_t) * n_nodes));
    W1G_TRY(upload(*c, c->t_right, right, sizeof(int64_t) * n_nodes));
    W1G_TRY(upload(*c, c->t_bbox, bbox, sizeof(double) * 4 * n_nodes));
    W1G_TRY(upload(*c, c->t_rep, rep, sizeof(int64_t) * n_nodes));
    int64_t *sz;
    W1G_TRY(ensure(c->t_size, (size_t)n_nodes, &sz));
    c->tree_n_points = n_points;
    c->tree_n_nodes = n_nodes;
    c->tree_depth = 0;
    c->pair_pts = ptr<double2>(c->tree_pts);
    W1G_TRY(tree_geom(*c));
    c->tree_valid = true;
    return W1G_OK;
}

// ---------------------------------------------------------------- WSPD

int w1g_wspd(w1g_ctx *c, double s, int reference_order, int64_t *n_pairs) {
    CTX_CHECK(c);
    if (!(s > 0.0)) {
        set_error("s must be positive");
        return W1G_EINVAL;
    }
    if (!c->tree_valid) {
        set_error("wspd: no split tree");
        return W1G_ESTATE;
    }
    c->arcs_valid = false;
    c->net_valid = false;
    return wspd_run(*c, s, reference_order, n_pairs);
}

int w1g_wspd_shard(w1g_ctx *c, double s, int shard, int n_shards, int64_t *n_pairs) {
    CTX_CHECK(c);
    if (!(s > 0.0)) {
        set_error("s must be positive");
        return W1G_EINVAL;
    }
    if (n_shards < 1 || shard < 0 || shard >= n_shards || !n_pairs) {
        set_error("wspd_shard: shard %d of %d", shard, n_shards);
        return W1G_EINVAL;
    }
    if (!c->tree_valid) {
        set_error("wspd: no split tree");
        return W1G_ESTATE;
    }
    c->arcs_valid = false;
    c->net_valid = false;
    return wspd_run(*c, s, 0, n_pairs, true, shard, n_shards);
}

int w1g_fetch_pairs(w1g_ctx *c, int64_t *node_pairs, int64_t *indices) {
    CTX_CHECK(c);
    if (!c->pairs_valid) {
        set_error("no WSPD pairs");
        return W1G_ESTATE;
    }
    const size_t P = (size_t)c->n_pairs;
    if (node_pairs) {
        if (!c->pairs_have_nodes) {
            set_error("pairs were loaded from indices only");
            return W1G_ESTATE;
        }
        // int2 (u, v) -> int64 (P, 2)
        W1G_TRY(stage_ensure(*c, sizeof(int2) * P));
        W1G_TRY(download(*c, c->h_stage, c->pair_uv.p, sizeof(int2) * P));
        W1G_TRY(stream_sync(*c));
        const int2 *uv = static_cast<const int2 *>(c->h_stage);
        for (size_t i = 0; i < P; i++) {
            node_pairs[2 * i] = uv[i].x;
            node_pairs[2 * i + 1] = uv[i].y;
        }
    }
    if (indices) {
        W1G_TRY(wspd_pair_idx(*c));
        W1G_TRY(download(*c, indices, c->pair_idx.p, sizeof(int64_t) * 2 * P));
        W1G_TRY(stream_sync(*c));
    }
    return W1G_OK;
}

int w1g_fetch_pair_counts(w1g_ctx *c, int64_t *counts, int64_t *n_internal) {
    CTX_CHECK(c);
    if (!c->pairs_valid || !c->pairs_have_nodes) {
        set_error("no WSPD pairs");
        return W1G_ESTATE;
    }
    const int64_t ni = c->tree_n_nodes > 0 ? (c->tree_n_nodes - 1) / 2 : 0;
    *n_internal = ni;
    if (counts) {
        W1G_TRY(download(*c, counts, c->pair_counts.p, sizeof(int64_t) * ni));
        W1G_TRY(stream_sync(*c));
    }
    return W1G_OK;
}

int w1g_load_pairs(w1g_ctx *c, const int64_t *indices, int64_t n_pairs, const double *points,
                   int64_t n_points) {
    CTX_CHECK(c);
    if (n_pairs < 0 || n_points < 0) return W1G_EINVAL;
    W1G_TRY(upload(*c, c->pair_idx, indices, sizeof(int64_t) * 2 * n_pairs));
    W1G_TRY(upload(*c, c->tree_pts, points, sizeof(double2) * n_points));
    c->pair_pts = ptr<double2>(c->tree_pts);
    c->n_pairs = n_pairs;
    c->pairs_valid = true;
    c->pairs_have_nodes = false;
    c->pair_idx_valid = true;
    c->arcs_valid = false;
    c->net_valid = false;
    return W1G_OK;
}

// ---------------------------------------------------------------- arcs / network

int w1g_emit_arcs(w1g_ctx *c, int64_t *n_arcs) {
    CTX_CHECK(c);
    if (!c->pairs_valid || !c->nodes[1].valid) {
        set_error("emit_arcs: needs pairs and nodes");
        return W1G_ESTATE;
    }
    c->net_valid = false;
    return emit_run(*c, n_arcs);
}

int w1g_emit_pair_arcs(w1g_ctx *c, int with_diagonal, int64_t *n_arcs) {
    CTX_CHECK(c);
    if (!c->pairs_valid || !c->nodes[1].valid) {
        set_error("emit_pair_arcs: needs pairs and nodes");
        return W1G_ESTATE;
    }
    c->net_valid = false;
    W1G_TRY(emit_run(*c, n_arcs, with_diagonal != 0));
    W1G_TRY(stream_sync(*c));
    return W1G_OK;
}

int w1g_arcs_device(w1g_ctx *c, void **tails, void **heads, void **costs, int64_t *m) {
    CTX_CHECK(c);
    if (!c->arcs_valid) {
        set_error("no arcs");
        return W1G_ESTATE;
    }
    *tails = c->arc_t.p;
    *heads = c->arc_h.p;
    *costs = c->arc_c.p;
    *m = c->n_arcs;
    return W1G_OK;
}

int w1g_pairs_device(w1g_ctx *c, void **uv, int64_t *n_pairs) {
    CTX_CHECK(c);
    if (!c->pairs_valid || !c->pairs_have_nodes) {
        set_error("no WSPD node pairs");
        return W1G_ESTATE;
    }
    *uv = c->pair_uv.p;
    *n_pairs = c->n_pairs;
    return W1G_OK;
}

int w1g_load_pairs_device(w1g_ctx *c, const void *d_uv, int64_t n_pairs) {
    CTX_CHECK(c);
    if (n_pairs < 0 || n_pairs >= (1ll << 31)) return W1G_EINVAL;
    if (!c->tree_valid) {
        set_error("load_pairs_device: the pairs index this context's split tree (build it first)");
        return W1G_ESTATE;
    }
    int2 *uv;
    W1G_TRY(ensure(c->pair_uv, (size_t)n_pairs + 1, &uv));
    if (n_pairs) W1G_CUDA(cudaMemcpyAsync(uv, d_uv, sizeof(int2) * n_pairs, cudaMemcpyDeviceToDevice, c->stream));
    c->n_pairs = n_pairs;
    c->pairs_valid = true;
    c->pairs_have_nodes = true;
    c->pair_idx_valid = false;
    c->arcs_valid = false;
    c->net_valid = false;
    return W1G_OK;
}

int w1g_network_from_pairs(w1g_ctx *c, int64_t *node_count, int64_t *n_arcs) {
    CTX_CHECK(c);
    if (!c->pairs_valid || !c->pairs_have_nodes || !c->nodes[1].valid || !c->tree_valid) {
        set_error("network_from_pairs: needs the condensed nodes, their split tree and WSPD node pairs");
        return W1G_ESTATE;
    }
    W1G_TRY(spanner_net_run(*c, node_count, n_arcs));
    W1G_TRY(stream_sync(*c));
    bool redone = false;
    W1G_TRY(spanner_net_check(*c, node_count, n_arcs, &redone));
    return W1G_OK;
}

int w1g_load_arcs_device(w1g_ctx *c, const int64_t *d_tails, const int64_t *d_heads, const double *d_costs,
                         int64_t m) {
    CTX_CHECK(c);
    if (m < 0 || m >= (1ll << 32)) return W1G_EINVAL;
    int64_t *t, *h;
    double *cs;
    W1G_TRY(ensure(c->arc_t, (size_t)m + 1, &t));
    W1G_TRY(ensure(c->arc_h, (size_t)m + 1, &h));
    W1G_TRY(ensure(c->arc_c, (size_t)m + 1, &cs));
    if (m) {
        W1G_CUDA(cudaMemcpyAsync(t, d_tails, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice, c->stream));
        W1G_CUDA(cudaMemcpyAsync(h, d_heads, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice, c->stream));
        W1G_CUDA(cudaMemcpyAsync(cs, d_costs, sizeof(double) * m, cudaMemcpyDeviceToDevice, c->stream));
    }
    c->n_arcs = m;
    c->arcs_valid = true;
    c->net_valid = false;
    return W1G_OK;
}

int w1g_fetch_arcs(w1g_ctx *c, int64_t *tails, int64_t *heads, double *costs) {
    CTX_CHECK(c);
    if (!c->arcs_valid) {
        set_error("no arcs");
        return W1G_ESTATE;
    }
    const size_t m = (size_t)c->n_arcs;
    W1G_TRY(download(*c, tails, c->arc_t.p, sizeof(int64_t) * m));
    W1G_TRY(download(*c, heads, c->arc_h.p, sizeof(int64_t) * m));
    W1G_TRY(download(*c, costs, c->arc_c.p, sizeof(double) * m));
    W1G_TRY(stream_sync(*c));
    return W1G_OK;
}

int w1g_load_arcs(w1g_ctx *c, const int64_t *tails, const int64_t *heads, const double *costs,
                  int64_t m) {
    CTX_CHECK(c);
    if (m < 0 || m >= (1ll << 32)) return W1G_EINVAL;
    W1G_TRY(upload(*c, c->arc_t, tails, sizeof(int64_t) * m));
    W1G_TRY(upload(*c, c->arc_h, heads, sizeof(int64_t) * m));
    W1G_TRY(upload(*c, c->arc_c, costs, sizeof(double) * m));
    c->n_arcs = m;
    c->arcs_valid = true;
    c->net_valid = false;
    return W1G_OK;
}

int w1g_build_network(w1g_ctx *c, const int64_t *supplies, int64_t n, int64_t *n_arcs) {
    CTX_CHECK(c);
    if (!c->arcs_valid) {
        set_error("build_network: no arcs");
        return W1G_ESTATE;
    }
    if (n < 0 || n >= (1ll << 31)) return W1G_EINVAL;
    int64_t *d;
    W1G_TRY(ensure(c->net_sup, (size_t)n, &d));
    if (n) W1G_CUDA(cudaMemcpyAsync(d, supplies, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    return net_run(*c, d, n, n_arcs);
}

int w1g_assemble(w1g_ctx *c, int64_t *node_count, int64_t *n_arcs) {
    CTX_CHECK(c);
    if (!c->arcs_valid || !c->nodes[1].valid) {
        set_error("assemble: needs arcs and nodes");
        return W1G_ESTATE;
    }
    int64_t *d, n;
    W1G_TRY(assemble_supplies(*c, &d, &n));
    *node_count = n;
    return net_run(*c, d, n, n_arcs);
}

int w1g_fetch_network(w1g_ctx *c, int64_t *supplies, int64_t *tails, int64_t *heads, double *costs,
                      int64_t *row_offsets) {
    CTX_CHECK(c);
    if (c->net_check_pending) {  // a fused front end that returned early: validate first
        int64_t nn, mm;
        bool redone;
        W1G_TRY(stream_sync(*c));
        W1G_TRY(spanner_net_check(*c, &nn, &mm, &redone));
    }
    if (!c->net_valid) {
        set_error("no network");
        return W1G_ESTATE;
    }
    const size_t n = (size_t)c->net_n, m = (size_t)c->net_m;
    W1G_TRY(download(*c, supplies, c->net_sup.p, sizeof(int64_t) * n));
    W1G_TRY(download(*c, tails, c->net_t.p, sizeof(int64_t) * m));
    W1G_TRY(download(*c, heads, c->net_h.p, sizeof(int64_t) * m));
    W1G_TRY(download(*c, costs, c->net_c.p, sizeof(double) * m));
    W1G_TRY(download(*c, row_offsets, c->net_ro.p, sizeof(int64_t) * (n + 1)));
    W1G_TRY(stream_sync(*c));
    return W1G_OK;
}

int w1g_set_network_out(w1g_ctx *c, int64_t *supplies, int64_t *tails, int64_t *heads, double *costs,
                        int64_t *row_offsets, int64_t node_cap, int64_t arc_cap) {
    CTX_CHECK(c);
    c->net_out = Ctx::NetOut{supplies, tails, heads, row_offsets, costs, node_cap, arc_cap};
    return W1G_OK;
}

// the network into the armed output target (asynchronously, on the context
// stream); the tails and row offsets may already be on their way (spanner_net_run
// starts them on the copy stream as soon as the row offsets are known)
// the tails column rebuilt on the host from the row offsets (row r's arcs are
// [ro[r], ro[r+1])), in parallel, with non-temporal stores, while the rest of the
// network is still crossing the link
static void fill_tails(Ctx &c, int64_t *t, const int64_t *ro, int64_t n, int64_t m) {
    if (!c.fill_pool) {
        c.fill_pool = new FillPool();
        c.fill_pool->start(3);
    }
    const int parts = 4;
    c.fill_pool->run(parts, [&](int p) {
        const int64_t a0 = m * p / parts, a1 = m * (p + 1) / parts;
        // the row holding arc a0: the last r with ro[r] <= a0
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (ro[mid] <= a0) lo = mid; else hi = mid - 1;
        }
        long long *tt = reinterpret_cast<long long *>(t);
        for (int64_t r = lo; r < n && ro[r] < a1; r++) {
            const int64_t e = ro[r + 1] < a1 ? ro[r + 1] : a1;
            for (int64_t q = ro[r] > a0 ? ro[r] : a0; q < e; q++) _mm_stream_si64(tt + q, (long long)r);
        }
        _mm_sfence();
    });
}

// pageable inputs into the page-locked staging buffer: the byte range [a | b] split over
// the fill threads (non-temporal stores), for inputs of a megabyte and more outside a batch
// (whose workers already run one per core)
static void stage_inputs(Ctx &c, char *dst, const char *a, size_t abytes, const char *b, size_t bbytes) {
    const size_t bytes = abytes + bbytes;
    if (bytes < ((size_t)1 << 20) || c.coop_share > 1) {
        if (abytes) host_copy_nt(dst, a, abytes);
        if (bbytes) host_copy_nt(dst + abytes, b, bbytes);
        return;
    }
    if (!c.fill_pool) {
        c.fill_pool = new FillPool();
        c.fill_pool->start(3);
    }
    const int parts = 4;
    c.fill_pool->run(parts, [&](int p) {
        const size_t lo = (bytes * p / parts) & ~(size_t)63, hi = p + 1 == parts ? bytes : (bytes * (p + 1) / parts) & ~(size_t)63;
        if (lo < abytes) host_copy_nt(dst + lo, a + lo, (hi < abytes ? hi : abytes) - lo);
        if (hi > abytes) {
            const size_t b0 = lo > abytes ? lo - abytes : 0, b1 = hi - abytes;
            host_copy_nt(dst + abytes + b0, b + b0, b1 - b0);
        }
    });
}

static int copy_network_out(Ctx &c, int *copied) {
    *copied = 0;
    const Ctx::NetOut &o = c.net_out;
    if (!c.net_valid || !o.sup || c.net_n > o.node_cap || c.net_m > o.arc_cap) return W1G_OK;
    const size_t n = (size_t)c.net_n, m = (size_t)c.net_m;
    W1G_TRY(download(c, o.sup, c.net_sup.p, sizeof(int64_t) * n));
    W1G_TRY(download(c, o.h, c.net_h.p, sizeof(int64_t) * m));
    W1G_TRY(download(c, o.c, c.net_c.p, sizeof(double) * m));
    if (c.net_early_copy) {
        W1G_CUDA(cudaStreamWaitEvent(c.stream, c.ev[13], 0));  // the early copies are part of this one
        if (c.net_tails_host) {
            W1G_CUDA(cudaEventSynchronize(c.ev[16]));  // the row offsets have landed
            fill_tails(c, o.t, o.ro, (int64_t)n, (int64_t)m);
        }
    } else {
        W1G_TRY(download(c, o.t, c.net_t.p, sizeof(int64_t) * m));
        W1G_TRY(download(c, o.ro, c.net_ro.p, sizeof(int64_t) * (n + 1)));
    }
    *copied = 1;
    return W1G_OK;
}

// ---------------------------------------------------------------- corpus / retrieval / dense oracle

int w1g_corpus_load(w1g_ctx *c, const double *points, const int64_t *offsets, int64_t n_diagrams) {
    CTX_CHECK(c);
    return corpus_load(*c, points, offsets, n_diagrams);
}

int w1g_corpus_set_host(w1g_ctx *c, const double *const *points, const int64_t *sizes, int64_t n_diagrams) {
    CTX_CHECK(c);
    return corpus_set_host(*c, points, sizes, n_diagrams);
}

int w1g_wcd_corpus(w1g_ctx *c, const double *query, int64_t nq, const int64_t *candidates, int64_t n_candidates,
                   double *scores) {
    CTX_CHECK(c);
    if (nq < 0 || n_candidates < 0 || (n_candidates && (!candidates || !scores))) return W1G_EINVAL;
    return wcd_corpus(*c, query, nq, candidates, n_candidates, scores);
}

int w1g_rwmd_corpus(w1g_ctx *c, const double *query, int64_t nq, const int64_t *candidates, int64_t n_candidates,
                    double *scores) {
    CTX_CHECK(c);
    if (nq < 0 || n_candidates < 0 || (n_candidates && (!candidates || !scores))) return W1G_EINVAL;
    c->nodes[1].valid = false;
    return rwmd_corpus(*c, query, nq, candidates, n_candidates, scores);
}

int w1g_dense_network(w1g_ctx *c, int64_t *node_count, int64_t *n_arcs) {
    CTX_CHECK(c);
    if (!c->nodes[0].valid) {
        set_error("dense_network: no nodes0 (zero_condense or load_nodes first)");
        return W1G_ESTATE;
    }
    if (!node_count || !n_arcs) return W1G_EINVAL;
    return dense_network_run(*c, node_count, n_arcs);
}

// ---------------------------------------------------------------- fused front end

static const double SQRT2 = 1.4142135623730951;  // math.sqrt(2.0)

static int front_end_impl(w1g_ctx *c, const double *d_a, int64_t na, const double *d_b, int64_t nb,
                          double s, int use_condensation, int delta_mode, double delta, double k,
                          uint64_t seed, w1g_front_end_info *info) {
    if (!info) return W1G_EINVAL;
    memset(info, 0, sizeof *info);
    if (!(s > 0.0)) {
        set_error("s must be positive");
        return W1G_EINVAL;
    }
    if (!(k >= 0.5 && k < 1.0)) {
        set_error("k must lie in [0.5, 1)");
        return W1G_EINVAL;
    }
    cudaEvent_t *ev = c->ev;
    std::chrono::steady_clock::time_point host_t[10];
    struct Disarm {  // the output target is one-shot, whatever path this call takes
        Ctx &c;
        ~Disarm() { c.net_out = Ctx::NetOut{}; }
    } disarm{*c};
    c->n_syncs = 0;
    c->sync_gap_us = 0.0;
    W1G_CUDA(cudaEventRecord(ev[0], c->stream));
    host_t[0] = std::chrono::steady_clock::now();
    // pipeline.py:67-69, condensation.py:47-59 (same IEEE operation order as the Python)
    const double eps_c = s >= 12 ? 8.0 / (s - 4.0) : 1.0;
    // With a fixed delta, L only feeds the diagnostics and the `L > 0` test of
    // pipeline.py:115, so RWMD runs on the auxiliary context concurrently with
    // the back end (from the point W1G_OVERLAP selects), which speculates L > 0
    // (redone with delta = 0 in the rare case L == 0).  With an armed output
    // target the network's D2H copy ends the call: RWMD then starts later and
    // runs under the CSR and the copy (overlap_e2e).
    const int ov = c->net_out.sup ? c->overlap_e2e : c->overlap;
    const bool overlap = ov && use_condensation && delta_mode != 0 && delta > 0.0;
    // split (W1G_SPLIT, default on): zero_condense and RWMD both go to the
    // auxiliary context, and the back end condenses the RAW diagrams (the same
    // cells and summed masses as condensing zero_condense's output), so the main
    // stream starts delta_condense at once
    const bool split_env = [] {  // read per call (tests toggle it)
        const char *e = getenv("W1G_SPLIT");
        return !(e && *e == '0');
    }();
    const bool split = overlap && split_env && na + nb > 0;
    // in split mode RWMD follows zero_condense on the auxiliary stream at once, or
    // (gate) only once the main stream has reached the point `gate` names (the
    // spawn points below); with an armed output target it waits for the WSPD so
    // it runs under the CSR and the network's D2H copy
    // when the spanner dominates (s >= 8 at >= 100k points) RWMD waits for the WSPD (gate 1)
    // and runs under the CSR: started at once, its kernels collide with the WSPD about half
    // the time
    // (cfg5 s = 16, delta = 0.001: bimodal 3.8 / 4.3 ms; gated 3.82-3.88 ms; s = 8: 2.18 vs
    // 2.25 ms); below that it starts at once (cfg2: 0.835 vs 0.996 ms gated)
    const bool spanner_heavy = s >= 8.0 && na + nb >= 100000;
    const int gate = split ? (c->net_out.sup ? c->split_gate_e2e
                                             : (spanner_heavy && !c->split_gate_set ? 1 : c->split_gate))
                           : 0;
    std::mutex gate_mu;
    std::condition_variable gate_cv;
    bool gate_open = gate == 0;
    int64_t k0 = 0;
    int32_t balanced = 0;
    double L = 0.0, LA = 0.0, LB = 0.0;
    int rc_aux = W1G_OK;
    std::string err_aux;
    // the auxiliary leg runs on the context's persistent worker thread; on every
    // exit path (errors included) the gate is opened and the job waited for
    // before the locals it references go out of scope
    struct AuxJoin {
        AuxWorker *w = nullptr;
        std::mutex *mu;
        std::condition_variable *cv;
        bool *open;
        ~AuxJoin() { join(); }
        void join() {
            if (!w) return;
            {
                std::lock_guard<std::mutex> lk(*mu);
                *open = true;
            }
            cv->notify_all();
            w->wait();
            w = nullptr;
        }
    } aux_join{nullptr, &gate_mu, &gate_cv, &gate_open};
    auto ensure_aux = [&]() -> int {
        if (!c->aux) {
            w1g_ctx *x = nullptr;
            W1G_TRY(w1g_ctx_create(c->device, &x));
            int least = 0, greatest = 0;
            W1G_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            W1G_CUDA(cudaStreamSynchronize(x->stream));  // its first allocations are ordered on it
            W1G_CUDA(cudaStreamDestroy(x->stream));
            W1G_CUDA(cudaStreamCreateWithPriority(&x->stream, cudaStreamNonBlocking, least));
            c->aux = x;
        }
        if (!c->aux_worker) {
            c->aux_worker = new AuxWorker();
            c->aux_worker->start();
        }
        Ctx *x = c->aux;
        x->culling = c->culling;
        x->cull_steps = c->cull_steps;
        x->heavy_ratio = c->heavy_ratio;
        return W1G_OK;
    };
    if (split) {
        W1G_TRY(ensure_aux());
        Ctx *x = c->aux;
        W1G_CUDA(cudaEventRecord(c->ev[8], c->stream));  // the inputs are on the device
        W1G_CUDA(cudaStreamWaitEvent(x->stream, c->ev[8], 0));
        const double2 *pa = reinterpret_cast<const double2 *>(d_a), *pb = reinterpret_cast<const double2 *>(d_b);
        aux_join.w = c->aux_worker;
        c->aux_worker->submit([&, x, pa, pb]() {
            cudaSetDevice(x->device);
            set_thread_stream(x->stream);
            cudaEventRecord(x->ev[2], x->stream);
            invalidate_from_nodes(*x);
            rc_aux = zc_run(*x, pa, na, pb, nb, &k0, &balanced);
            cudaEventRecord(x->ev[3], x->stream);
            if (rc_aux == W1G_OK && gate) {
                std::unique_lock<std::mutex> lk(gate_mu);
                gate_cv.wait(lk, [&] { return gate_open; });
                cudaStreamWaitEvent(x->stream, c->ev[11], 0);  // recorded before the gate opened
            }
            cudaEventRecord(x->ev[0], x->stream);
            if (rc_aux == W1G_OK && k0 > 0 && !balanced) rc_aux = rwmd_run(*x, &L, &LA, &LB);
            if (rc_aux == W1G_OK) rc_aux = cudaEventRecord(x->ev[1], x->stream) == cudaSuccess ? W1G_OK : W1G_ECUDA;
            if (rc_aux != W1G_OK) err_aux = g_err;
        });
        W1G_TRY(raw_nodes(*c, pa, na, pb, nb));
        W1G_CUDA(cudaEventRecord(ev[1], c->stream));
        W1G_CUDA(cudaEventRecord(ev[2], c->stream));
        host_t[1] = host_t[2] = std::chrono::steady_clock::now();
    } else {
        W1G_TRY(w1g_zero_condense_device(c, d_a, na, d_b, nb, &k0, &balanced));
        W1G_CUDA(cudaEventRecord(ev[1], c->stream));
        host_t[1] = std::chrono::steady_clock::now();
        info->n_points0 = k0;
        if (k0 == 0 || balanced) {
            // pipeline.py:106-109: empty inputs or identical multisets -> 0.0
            info->short_circuit = 1;
            W1G_TRY(stream_sync(*c));
            return W1G_OK;
        }
        if (!overlap) W1G_TRY(rwmd_run(*c, &L, &LA, &LB));
        W1G_CUDA(cudaEventRecord(ev[2], c->stream));
        host_t[2] = std::chrono::steady_clock::now();
    }
    info->epsilon_condense = eps_c;
    bool aliased = false;
    auto start_rwmd = [&]() -> int {
        W1G_TRY(ensure_aux());
        Ctx *x = c->aux;
        // alias (read only; nothing downstream rewrites nodes0); the auxiliary
        // context's own nodes0 buffers (the split schedule's) wait aside
        x->nodes0_stash = x->nodes[0];
        x->nodes[0] = c->nodes[0];
        aliased = true;
        W1G_CUDA(cudaEventRecord(c->ev[8], c->stream));  // nodes0 complete on the main stream
        W1G_CUDA(cudaStreamWaitEvent(x->stream, c->ev[8], 0));
        aux_join.w = c->aux_worker;
        c->aux_worker->submit([&, x]() {
            cudaSetDevice(x->device);
            set_thread_stream(x->stream);
            cudaEventRecord(x->ev[0], x->stream);
            rc_aux = rwmd_run(*x, &L, &LA, &LB);
            if (rc_aux == W1G_OK) rc_aux = cudaEventRecord(x->ev[1], x->stream) == cudaSuccess ? W1G_OK : W1G_ECUDA;
            if (rc_aux != W1G_OK) err_aux = g_err;
        });
        return W1G_OK;
    };
    NodeSet *dc_src = split ? &c->raw : nullptr;
    auto open_gate = [&]() -> int {
        W1G_CUDA(cudaEventRecord(c->ev[11], c->stream));
        {
            std::lock_guard<std::mutex> lk(gate_mu);
            gate_open = true;
        }
        gate_cv.notify_all();
        return W1G_OK;
    };
    // a spawn point: start RWMD (overlap) or open the split gate
    auto spawn_at = [&](bool spawn, int point) -> int {
        if (spawn && ov == point) W1G_TRY(start_rwmd());
        if (split && gate == point && !gate_open) W1G_TRY(open_gate());
        return W1G_OK;
    };
    auto back_end = [&](double d, bool spawn) -> int {
        info->delta = d;
        W1G_TRY(spawn_at(spawn, 2));
        int64_t kk;
        const double pitch = k * d;
        const double half_width = (1.0 - k) * d / 2.0;
        W1G_TRY(dc_run(*c, d > 0.0 ? d : 0.0, pitch, half_width, seed, &kk, dc_src));
        W1G_CUDA(cudaEventRecord(ev[3], c->stream));
    host_t[3] = std::chrono::steady_clock::now();
        info->n_points = kk;
        W1G_TRY(spawn_at(spawn, 4));
        int64_t nn;
        int32_t depth;
        W1G_TRY(tree_run(*c, ptr<double2>(c->nodes[1].pts), kk, &nn, &depth, true));
        W1G_CUDA(cudaEventRecord(ev[4], c->stream));
    host_t[4] = std::chrono::steady_clock::now();
        info->n_tree_nodes = nn;
        info->tree_depth = depth;
        W1G_TRY(spawn_at(spawn, 3));
        int64_t P;
        W1G_TRY(wspd_run(*c, s, 0, &P, false));  // its round trip also delivers the tree's depth / duplicate flag
        W1G_TRY(tree_deferred_check(*c, &depth));
        info->tree_depth = depth;
        W1G_CUDA(cudaEventRecord(ev[5], c->stream));
    host_t[5] = std::chrono::steady_clock::now();
        info->n_pairs = P;
        info->n_levels_wspd = c->wspd_levels;
        W1G_TRY(spawn_at(spawn, 1));
        // emit_arcs is fused into the CSR assembly (the arc list is never
        // materialised), so stage 5 (emit) is empty on this path
        W1G_CUDA(cudaEventRecord(ev[6], c->stream));
        host_t[6] = std::chrono::steady_clock::now();
        int64_t nsup, mm;
        W1G_TRY(spanner_net_run(*c, &nsup, &mm));
        W1G_TRY(spawn_at(spawn, 5));
        W1G_CUDA(cudaEventRecord(ev[7], c->stream));
    host_t[7] = std::chrono::steady_clock::now();
        info->n_arcs = mm;
        info->node_count = nsup;
        return W1G_OK;
    };
    auto delta_for = [&](double lower) {
        if (!(use_condensation && lower > 0.0)) return 0.0;
        if (delta_mode == 0) {
            const double n_points = (double)(na + nb);
            return 2.0 * eps_c * lower / (SQRT2 * n_points);
        }
        return delta;
    };
    int rc = back_end(overlap ? delta : delta_for(L), overlap && !split);
    // the network leaves for the host while RWMD may still run on the auxiliary stream
    if (rc == W1G_OK) rc = copy_network_out(*c, &info->network_copied);
    if (split && !gate_open) {  // the back end stopped early: let the worker finish
        const int rg = open_gate();
        if (rc == W1G_OK) rc = rg;
    }
    aux_join.join();
    if (aliased) {
        c->aux->nodes[0] = c->aux->nodes0_stash;  // drop the alias, keep its own buffers
        c->aux->nodes0_stash = NodeSet{};
    }
    if (split) {
        if (rc_aux != W1G_OK) {
            set_error("%s", err_aux.c_str());
            return rc_aux;
        }
        // nodes0 (zero_condense's output) becomes the main context's, as on the sequential path
        W1G_CUDA(cudaStreamWaitEvent(c->stream, c->aux->ev[1], 0));
        std::swap(c->nodes[0], c->aux->nodes[0]);
        info->n_points0 = k0;
        if (k0 == 0 || balanced) {
            // pipeline.py:106-109: identical multisets -> 0.0 (the speculative back end is dropped,
            // whatever it returned: the reference never gets there)
            invalidate_from_nodes(*c);
            c->nodes[1].valid = false;
            c->net_check_pending = false;
            info->short_circuit = 1;
            info->network_copied = 0;
            info->delta = 0.0;
            info->n_points = info->n_tree_nodes = info->n_pairs = info->n_arcs = info->node_count = 0;
            info->tree_depth = info->n_levels_wspd = 0;
            W1G_TRY(stream_sync(*c));
            return W1G_OK;
        }
        dc_src = nullptr;  // any redo below condenses nodes0 itself
    }
    if (overlap && !(L > 0.0) && rc_aux == W1G_OK) {
        // pipeline.py:115: no condensation when L == 0 (whatever the speculative back end returned)
        W1G_CUDA(cudaStreamWaitEvent(c->stream, c->aux->ev[1], 0));
        W1G_TRY(back_end(0.0, false));
        rc = copy_network_out(*c, &info->network_copied);
    }
    if (rc != W1G_OK) return rc;
    if (rc_aux != W1G_OK) {
        set_error("%s", err_aux.c_str());
        return rc_aux;
    }
    if (overlap) W1G_CUDA(cudaStreamWaitEvent(c->stream, c->aux->ev[1], 0));
    info->lower_bound = L;
    info->lower_bound_a = LA;
    info->lower_bound_b = LB;
    W1G_CUDA(cudaEventRecord(ev[9], c->stream));
    host_t[9] = std::chrono::steady_clock::now();  // everything, RWMD included, is done
    W1G_CUDA(cudaEventSynchronize(ev[9]));
    {
        bool redone = false;
        int64_t nsup = info->node_count, mm = info->n_arcs;
        W1G_TRY(spanner_net_check(*c, &nsup, &mm, &redone));
        if (redone) {  // the network was rebuilt on the generic path: copy it out again
            info->node_count = nsup;
            info->n_arcs = mm;
            W1G_TRY(copy_network_out(*c, &info->network_copied));
            W1G_TRY(stream_sync(*c));
        }
    }
    for (int i = 0; i < 7; i++) W1G_CUDA(cudaEventElapsedTime(&info->stage_ms[i], ev[i], ev[i + 1]));
    if (overlap) W1G_CUDA(cudaEventElapsedTime(&info->stage_ms[1], c->aux->ev[0], c->aux->ev[1]));
    if (split) W1G_CUDA(cudaEventElapsedTime(&info->stage_ms[0], c->aux->ev[2], c->aux->ev[3]));
    W1G_CUDA(cudaEventElapsedTime(&info->stage_ms[7], ev[0], ev[9]));
    if (c->timing)
    {
        fprintf(stderr, "[w1g syncs] host round trips=%lld idle=%.1fus\n", (long long)c->n_syncs, c->sync_gap_us);
        fprintf(stderr, "[w1g host]");
        for (int i = 0; i < 7; i++)
            fprintf(stderr, " %d=%.1fus", i,
                    1e-3 * std::chrono::duration_cast<std::chrono::nanoseconds>(host_t[i + 1] - host_t[i]).count());
        fprintf(stderr, "\n[w1g dev] ");
        for (int i = 0; i < 8; i++) fprintf(stderr, " %d=%.1fus", i, 1e3 * info->stage_ms[i]);
        fprintf(stderr, "\n");
    }
    return W1G_OK;
}

int w1g_front_end_device(w1g_ctx *c, const double *d_a, int64_t na, const double *d_b, int64_t nb,
                         double s, int use_condensation, int delta_mode, double delta, double k,
                         uint64_t seed, w1g_front_end_info *info) {
    CTX_CHECK(c);
    const int rc = front_end_impl(c, d_a, na, d_b, nb, s, use_condensation, delta_mode, delta, k, seed, info);
    if (rc != W1G_OK) {
        // an error can leave copies into the caller's output target (or reads of
        // the inputs on the auxiliary stream) in flight: drain every stream this
        // call used before the caller may reuse those buffers
        std::string msg = g_err;
        cudaStreamSynchronize(c->stream);
        if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
        if (c->aux) cudaStreamSynchronize(c->aux->stream);
        cudaGetLastError();
        set_error("%s", msg.c_str());
    }
    return rc;
}

int w1g_front_end(w1g_ctx *c, const double *a, int64_t na, const double *b, int64_t nb, double s,
                  int use_condensation, int delta_mode, double delta, double k, uint64_t seed,
                  w1g_front_end_info *info) {
    CTX_CHECK(c);
    if (na < 0 || nb < 0) return W1G_EINVAL;
    double2 *d;
    W1G_TRY(ensure(c->in_pts, (size_t)(na + nb), &d));
    const size_t bytes = sizeof(double2) * (size_t)(na + nb);
    if (is_pinned(a) && is_pinned(b)) {
        // page-locked inputs (w1g_host_alloc or any cudaHostAlloc'd memory): DMA directly
        if (na) W1G_CUDA(cudaMemcpyAsync(d, a, sizeof(double2) * na, cudaMemcpyHostToDevice, c->stream));
        if (nb) W1G_CUDA(cudaMemcpyAsync(d + na, b, sizeof(double2) * nb, cudaMemcpyHostToDevice, c->stream));
    } else {
        // pageable inputs: stage both diagrams through pinned memory, one full-speed H2D
        W1G_TRY(stage_ensure(*c, bytes));
        W1G_TRY(stream_sync(*c));
        stage_inputs(*c, static_cast<char *>(c->h_stage), reinterpret_cast<const char *>(a), sizeof(double2) * na,
                     reinterpret_cast<const char *>(b), sizeof(double2) * nb);
        if (bytes) W1G_CUDA(cudaMemcpyAsync(d, c->h_stage, bytes, cudaMemcpyHostToDevice, c->stream));
    }
    return w1g_front_end_device(c, reinterpret_cast<double *>(d), na,
                                reinterpret_cast<double *>(d + na), nb, s, use_condensation,
                                delta_mode, delta, k, seed, info);
}

}  // extern "C"
