// batch.cu -- the native batch executor: the sparsify front end of many
// diagram pairs per library call (the pairwise W1 matrix of cfg4, and any
// pair list), with no Python in the per-pair loop.
//
// The reference's CPU baseline for this workload is a loop of approx_w1 over
// the i < j pairs; the drop-in's pairwise_w1 / sparsify_batch
// run it as:
//   * the diagrams stay in host memory (w1g_corpus_set_host; each worker uploads
//     its pair inside its front end) or are uploaded once (w1g_corpus_load);
//   * `streams` worker threads, each driving its own child context (own CUDA
//     stream, scratch and RWMD side context), pull pair indices from a shared
//     atomic counter -- latency-bound front ends of small diagrams overlap on
//     one GPU; their cooperative kernels run on a 1/streams share of the device;
//   * a finished network is copied device-to-device into one of the worker's two
//     staging slots and its D2H into a page-locked block from a process-wide pool
//     is queued on the worker's own stream, while the worker goes on to its next
//     pair.  The compact transfer leaves the tails behind and narrows the heads
//     to int32; expander threads rebuild both on the host (non-temporal stores)
//     before the result is queued for the consumer (w1g_batch_next), which hands
//     it to the host solver and releases the block when the arrays die
//     (w1g_batch_release).  The pool bounds the bytes in flight, so a fast front
//     end cannot pin host memory without limit while the solver drains the queue
//     (workers wait for a block instead).
//   * w1g_front_end_batch is the synchronous variant that leaves every network
//     in device memory (front-end throughput, and the per-pair diagnostics).
#include <emmintrin.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <deque>
#include <map>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace w1g {

// ---------------------------------------------------------------- page-locked result blocks

namespace {

struct HostPool {
    std::mutex mu;
    std::condition_variable cv;
    std::map<size_t, std::vector<void *>> free_blocks;  // by size class
    std::unordered_map<void *, size_t> cls_of;
    size_t in_flight = 0;
    size_t limit = (size_t)8 << 30;
    int spare_blocks = 12;  // extra blocks pinned with the first block of a size class (<= limit / 8)

    static size_t size_class(size_t b) {
        size_t c = (size_t)1 << 20;
        while (c < b) c <<= 1;
        return c;
    }
    // a block of at least `bytes`; waits while the bytes in flight exceed the limit
    // (unless nothing is in flight: one oversized network must still go through)
    int get(size_t bytes, void **out, const std::atomic<bool> *cancel) {
        const size_t cls = size_class(bytes);
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return in_flight == 0 || in_flight + cls <= limit || (cancel && cancel->load()); });
        if (cancel && cancel->load()) {
            set_error("batch cancelled");
            return W1G_ESTATE;
        }
        in_flight += cls;
        auto &fl = free_blocks[cls];
        if (!fl.empty()) {
            *out = fl.back();
            fl.pop_back();
            return W1G_OK;
        }
        lk.unlock();
        // a new size class: a few spare blocks at once, so the batches that follow do not
        // pin memory (tens of ms per block) in the middle of their timed work
        void *p = nullptr;
        const cudaError_t e = cudaHostAlloc(&p, cls, cudaHostAllocPortable);
        std::vector<void *> spare;
        for (int q = 0; e == cudaSuccess && q < spare_blocks && (size_t)(q + 1) * cls <= limit / 8; q++) {
            void *x = nullptr;
            if (cudaHostAlloc(&x, cls, cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                break;
            }
            spare.push_back(x);
        }
        lk.lock();
        if (e != cudaSuccess) {
            cudaGetLastError();
            in_flight -= cls;
            cv.notify_all();
            set_error("cudaHostAlloc of %zu bytes failed", cls);
            return W1G_ENOMEM;
        }
        cls_of[p] = cls;
        for (void *x : spare) {
            cls_of[x] = cls;
            free_blocks[cls].push_back(x);
        }
        *out = p;
        return W1G_OK;
    }
    void put(void *p) {
        bool release = false;
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = cls_of.find(p);
            if (it == cls_of.end()) return;
            in_flight -= it->second;
            auto &fl = free_blocks[it->second];
            if (fl.size() < 64) {
                fl.push_back(p);
            } else {
                cls_of.erase(it);
                release = true;
            }
        }
        cv.notify_all();
        // outside the lock: cudaFreeHost waits for the device, which must not stall the
        // workers' block requests
        if (release) cudaFreeHost(p);
    }
    void wake() { cv.notify_all(); }
};

HostPool &host_pool() {
    static HostPool *pool = new HostPool();  // process lifetime: blocks may outlive contexts
    return *pool;
}

// carve the five network arrays out of a block laid out for (ncap nodes, mcap arcs)
struct NetCarve {
    int64_t *sup, *t, *h, *ro;
    double *c;
};
inline size_t al64(size_t x) { return (x + 63) & ~(size_t)63; }
inline size_t carve_bytes(int64_t ncap, int64_t mcap) {
    return al64(8 * (size_t)ncap) + 3 * al64(8 * (size_t)mcap) + al64(8 * (size_t)(ncap + 1));
}
NetCarve carve(void *blk, int64_t ncap, int64_t mcap) {
    char *p = static_cast<char *>(blk);
    NetCarve r;
    r.sup = reinterpret_cast<int64_t *>(p);
    p += al64(8 * (size_t)ncap);
    r.t = reinterpret_cast<int64_t *>(p);
    p += al64(8 * (size_t)mcap);
    r.h = reinterpret_cast<int64_t *>(p);
    p += al64(8 * (size_t)mcap);
    r.c = reinterpret_cast<double *>(p);
    p += al64(8 * (size_t)mcap);
    r.ro = reinterpret_cast<int64_t *>(p);
    return r;
}

}  // namespace

struct BatchParams {
    double s, delta, k;
    int use_condensation, delta_mode;
    uint64_t seed;
};

struct BatchState {
    std::vector<w1g_ctx *> kids;
    std::vector<std::thread> threads;
    std::vector<int32_t> pairs;
    int64_t n_pairs = 0;
    BatchParams prm{};
    bool deliver = false;
    w1g_front_end_info *infos = nullptr;  // synchronous variant
    std::atomic<int64_t> next{0};
    std::atomic<bool> cancel{false};
    std::mutex mu;
    std::condition_variable cv;
    std::deque<w1g_batch_result> ready;
    int64_t delivered = 0;  // results handed to the consumer
    int64_t produced = 0;   // results queued (or recorded) by the workers
    int first_rc = W1G_OK;
    std::string first_err;
    bool active = false;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;  // device makespan of a synchronous batch
    std::vector<cudaEvent_t> kid_ev;
    // compact transfer (W1G_BATCH_COMPACT=0: off): the tails are not copied and the heads
    // cross as int32; expander threads rebuild both on the host before a result is
    // handed over (cfg2: 25.5 instead of 47.3 MB per network over the link)
    int compact = 1;  // 0: off, 1: tails rebuilt + int32 heads widened, 2: tails rebuilt only
    std::vector<std::thread> expanders;
    std::deque<w1g_batch_result> expand_q;
    std::mutex emu;
    std::condition_variable ecv;
    int workers_left = 0;
    // W1G_BATCH_TRACE=1: per-worker host time in each phase (us), printed at the batch's end
    bool trace = false;
    bool trace_steps = false;  // W1G_BATCH_TRACE=2: every worker step to stderr (debugging)
    std::vector<double> tr_block, tr_fe, tr_fetch, tr_pairs;
};

static void batch_join(BatchState &b) {
    for (auto &t : b.threads)
        if (t.joinable()) t.join();
    b.threads.clear();
    for (auto &t : b.expanders)
        if (t.joinable()) t.join();
    b.expanders.clear();
}

static int ensure_kids(Ctx &c, BatchState &b, int streams) {
    while ((int)b.kids.size() < streams) {
        w1g_ctx *x = nullptr;
        W1G_TRY(w1g_ctx_create(c.device, &x));
        b.kids.push_back(x);
    }
    return W1G_OK;
}

// A delivered network leaves the worker asynchronously: when its front end has
// finished, the five network arrays are copied device-to-device into one of the
// worker's two staging slots (~15 us at cfg2), and their D2H into a page-locked
// block is queued on the child's copy stream; the worker goes straight on to its
// next pair, whose kernels run while the previous network crosses the host link.
// A result is handed to the consumer once its copy has landed (checked after the
// next front end, or before its staging slot is reused).
struct PendingNet {
    w1g_batch_result r;
    int slot = -1;
};

// device-to-device copy of the network into a staging slot with SM loads/stores:
// a cudaMemcpyAsync D2D would queue on the copy engines behind the link-bound D2H
// transfers of earlier networks, and the next front end would wait for it
struct CopyJob {
    const int4 *src[5];
    int4 *dst[5];
    int64_t n16[5];  // 16-byte words (0: not copied)
    // compact transfer: the int64 heads narrowed to int32 (h2 = pairs of heads)
    const longlong2 *h64;
    int2 *h32;
    int64_t n_h2;
};

__global__ void k_stage_copy(CopyJob J) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int a = 0; a < 5; a++)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < J.n16[a]; i += stride)
            J.dst[a][i] = J.src[a][i];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < J.n_h2; i += stride) {
        const longlong2 v = J.h64[i];
        J.h32[i] = make_int2((int32_t)v.x, (int32_t)v.y);
    }
}

// the compact transfer's host side: the tails column is a function of the row
// offsets (row r's arcs are [ro[r], ro[r+1])) and the heads arrive as int32 in the
// upper half of their int64 array, widened in place front to back (element i's
// 8 bytes never overlap an int32 not yet read)
static void expand_network(const w1g_batch_result &r, int mode) {
    // non-temporal 8-byte stores (MOVNTI): the arrays are written once and read later by
    // the consumer, so no read-for-ownership of their cache lines (the expansion is bound
    // by host memory traffic: 22.5 MB written per cfg2 network)
    const int64_t n = r.info.node_count, m = r.info.n_arcs;
    const int64_t *ro = r.row_offsets;
    long long *t = reinterpret_cast<long long *>(r.tails);
    for (int64_t q = 0; q < n; q++) {
        const int64_t e = ro[q + 1];
        for (int64_t a = ro[q]; a < e; a++) _mm_stream_si64(t + a, (long long)q);
    }
    if (mode == 1) {
        const int32_t *h32 = reinterpret_cast<const int32_t *>(reinterpret_cast<const char *>(r.heads) + 4 * m);
        long long *h = reinterpret_cast<long long *>(r.heads);
        for (int64_t i = 0; i < m; i++) _mm_stream_si64(h + i, (long long)h32[i]);
    }
    _mm_sfence();
}

struct StageSlot {
    DevBuf sup, t, h, c, ro;
    cudaEvent_t d2d = nullptr, done = nullptr;
};

static int stage_copy(w1g_ctx *x, cudaStream_t cs, StageSlot &st, int64_t n, int64_t m, const NetCarve &cv,
                      int compact) {
    int64_t *sup, *t = nullptr, *h, *ro;
    double *c;
    W1G_TRY(ensure(st.sup, (size_t)n + 1, &sup));
    if (!compact) W1G_TRY(ensure(st.t, (size_t)m + 1, &t));
    W1G_TRY(ensure(st.h, (size_t)m + 1, &h));
    W1G_TRY(ensure(st.c, (size_t)m + 1, &c));
    W1G_TRY(ensure(st.ro, (size_t)n + 2, &ro));
    if (!st.d2d) {
        W1G_CUDA(cudaEventCreateWithFlags(&st.d2d, cudaEventDisableTiming));
        W1G_CUDA(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming));
    }
    const cudaStream_t ms = x->stream;
    // every buffer holds whole 16-byte words (ensure() pads by 16 bytes)
    CopyJob J;
    const void *src[5] = {x->net_sup.p, x->net_t.p, x->net_h.p, x->net_c.p, x->net_ro.p};
    void *dst[5] = {sup, t, h, c, ro};
    const int64_t cnt[5] = {n, m, m, m, n + 1};
    for (int a = 0; a < 5; a++) {
        J.src[a] = static_cast<const int4 *>(src[a]);
        J.dst[a] = static_cast<int4 *>(dst[a]);
        J.n16[a] = (cnt[a] + 1) / 2;
    }
    J.h64 = nullptr;
    J.h32 = nullptr;
    J.n_h2 = 0;
    if (compact) J.n16[1] = 0;  // no tails
    if (compact == 1) {
        J.n16[2] = 0;  // heads narrowed instead (the int64 buffers hold whole 16-byte words)
        J.h64 = static_cast<const longlong2 *>(x->net_h.p);
        J.h32 = reinterpret_cast<int2 *>(h);
        J.n_h2 = (m + 1) / 2;
    }
    k_stage_copy<<<4 * x->sm_count, 256, 0, ms>>>(J);
    W1G_CHECK_LAUNCH();
    W1G_CUDA(cudaEventRecord(st.d2d, ms));
    W1G_CUDA(cudaStreamWaitEvent(cs, st.d2d, 0));
    W1G_CUDA(cudaMemcpyAsync(cv.sup, sup, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, cs));
    if (compact == 1) {
        W1G_CUDA(cudaMemcpyAsync(reinterpret_cast<char *>(cv.h) + 4 * m, h, sizeof(int32_t) * m,
                                 cudaMemcpyDeviceToHost, cs));
    } else if (compact == 2) {
        W1G_CUDA(cudaMemcpyAsync(cv.h, h, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, cs));
    } else {
        W1G_CUDA(cudaMemcpyAsync(cv.t, t, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, cs));
        W1G_CUDA(cudaMemcpyAsync(cv.h, h, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, cs));
    }
    W1G_CUDA(cudaMemcpyAsync(cv.c, c, sizeof(double) * m, cudaMemcpyDeviceToHost, cs));
    W1G_CUDA(cudaMemcpyAsync(cv.ro, ro, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, cs));
    W1G_CUDA(cudaEventRecord(st.done, cs));
    return W1G_OK;
}

static void batch_publish(BatchState *b, w1g_batch_result &r) {
    {
        std::lock_guard<std::mutex> lk(b->mu);
        if (r.status != W1G_OK && b->first_rc == W1G_OK) {
            b->first_rc = r.status;
            b->first_err = r.message;
        }
        if (b->infos) b->infos[r.pair] = r.info;
        if (b->deliver) b->ready.push_back(r);
        b->produced++;
    }
    b->cv.notify_all();
    if (r.status != W1G_OK) {
        b->cancel.store(true);  // like the reference's loop: the first error ends the batch
        host_pool().wake();
    }
}

// an expander: rebuilds compact-transferred networks (expand_network) and hands them
// over; leaves when the workers are done and the queue is empty
static void batch_expander(BatchState *b) {
    for (;;) {
        w1g_batch_result r;
        {
            std::unique_lock<std::mutex> lk(b->emu);
            b->ecv.wait(lk, [&] { return !b->expand_q.empty() || b->workers_left == 0; });
            if (b->expand_q.empty()) return;
            r = b->expand_q.front();
            b->expand_q.pop_front();
        }
        expand_network(r, b->compact);
        batch_publish(b, r);
    }
}

// a network whose copy has landed: to an expander (compact transfer) or straight over
static void batch_landed(BatchState *b, w1g_batch_result &r) {
    if (b->compact && r.status == W1G_OK && r.block) {
        {
            std::lock_guard<std::mutex> lk(b->emu);
            b->expand_q.push_back(r);
        }
        b->ecv.notify_one();
        return;
    }
    batch_publish(b, r);
}

// one worker: pairs from the shared counter, front end on its own child context
static void batch_worker(Ctx *parent, BatchState *b, int w) {
    w1g_ctx *x = b->kids[w];
    const double2 *corpus = ptr<double2>(parent->corpus_pts);
    const int64_t *off = parent->h_corpus_off;
    cudaSetDevice(x->device);
    set_thread_stream(x->stream);
    using clk = std::chrono::steady_clock;
    auto us = [](clk::time_point a, clk::time_point b) {
        return 1e-3 * (double)std::chrono::duration_cast<std::chrono::nanoseconds>(b - a).count();
    };
    StageSlot slots[2];
    // the D2H of delivered networks has a stream of its own: the context's copy stream
    // carries work of the front end itself (the CSR's tails, RWMD's second side)
    cudaStream_t d2h = nullptr;
    if (b->deliver) cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking);
    std::deque<PendingNet> pending;  // oldest first, at most 2 (one per slot)
    int next_slot = 0;
    // hand over the oldest pending network once its copy has landed (wait: block for it)
    auto drain = [&](bool wait) {
        while (!pending.empty()) {
            PendingNet &pn = pending.front();
            cudaEvent_t e = slots[pn.slot].done;
            if (!wait && cudaEventQuery(e) == cudaErrorNotReady) return;
            const cudaError_t err = cudaEventSynchronize(e);
            if (err != cudaSuccess) {
                pn.r.status = W1G_ECUDA;
                snprintf(pn.r.message, sizeof pn.r.message, "network copy failed: %s", cudaGetErrorString(err));
                if (pn.r.block) host_pool().put(pn.r.block);
                pn.r.block = nullptr;
            }
            batch_landed(b, pn.r);
            pending.pop_front();
            wait = false;
        }
    };
    for (;;) {
        if (b->cancel.load()) break;
        const int64_t p = b->next.fetch_add(1);
        if (p >= b->n_pairs) break;
        const int32_t i = b->pairs[2 * p], j = b->pairs[2 * p + 1];
        w1g_batch_result r;
        memset(&r, 0, sizeof r);
        r.pair = p;
        r.i = i;
        r.j = j;
        int rc = W1G_OK;
        const clk::time_point t1 = clk::now();
        if (b->trace_steps) fprintf(stderr, "[w1g batch] w%d pair %lld: front end\n", w, (long long)p);
        if (parent->h_corpus_ptr) {
            // host-resident diagrams: this worker's H2D overlaps the other workers' front ends
            rc = w1g_front_end(x, parent->h_corpus_ptr[i], off[i + 1] - off[i], parent->h_corpus_ptr[j],
                               off[j + 1] - off[j], b->prm.s, b->prm.use_condensation, b->prm.delta_mode,
                               b->prm.delta, b->prm.k, b->prm.seed, &r.info);
        } else {
            const double *pa = reinterpret_cast<const double *>(corpus + off[i]);
            const double *pb = reinterpret_cast<const double *>(corpus + off[j]);
            rc = w1g_front_end_device(x, pa, off[i + 1] - off[i], pb, off[j + 1] - off[j], b->prm.s,
                                      b->prm.use_condensation, b->prm.delta_mode, b->prm.delta, b->prm.k,
                                      b->prm.seed, &r.info);
        }
        const clk::time_point t2 = clk::now();
        drain(false);  // the previous network's copy ran under this front end
        double t_block = 0.0;
        bool queued = false;
        if (rc == W1G_OK && b->deliver && !r.info.short_circuit) {
            const int64_t n = r.info.node_count, m = r.info.n_arcs;
            const int sl = next_slot;
            // the slot's previous network must have left before the slot is rewritten
            if (b->trace_steps) fprintf(stderr, "[w1g batch] w%d pair %lld: slot %d\n", w, (long long)p, sl);
            while (!pending.empty() && pending.front().slot == sl) drain(true);
            void *blk = nullptr;
            if (b->trace_steps) fprintf(stderr, "[w1g batch] w%d pair %lld: block\n", w, (long long)p);
            const clk::time_point tb = clk::now();
            rc = host_pool().get(carve_bytes(n, m), &blk, &b->cancel);
            t_block = us(tb, clk::now());
            if (rc == W1G_OK) {
                const NetCarve cv = carve(blk, n, m);
                if (b->trace_steps) fprintf(stderr, "[w1g batch] w%d pair %lld: copy\n", w, (long long)p);
                rc = d2h ? stage_copy(x, d2h, slots[sl], n, m, cv, b->compact) : W1G_ECUDA;
                if (rc == W1G_OK) {
                    r.supplies = cv.sup;
                    r.tails = cv.t;
                    r.heads = cv.h;
                    r.costs = cv.c;
                    r.row_offsets = cv.ro;
                    r.block = blk;
                    pending.push_back(PendingNet{r, sl});
                    next_slot ^= 1;
                    queued = true;
                } else {
                    host_pool().put(blk);
                }
            }
        }
        if (b->trace) {
            b->tr_block[w] += t_block;
            b->tr_fe[w] += us(t1, t2);
            b->tr_fetch[w] += us(t2, clk::now()) - t_block;
            b->tr_pairs[w] += 1;
        }
        if (!queued) {
            r.status = rc;
            if (rc != W1G_OK) snprintf(r.message, sizeof r.message, "%s", w1g_last_error());
            drain(true);  // keep completion order per worker
            batch_publish(b, r);
        }
    }
    drain(true);
    {
        std::lock_guard<std::mutex> lk(b->emu);
        b->workers_left--;
    }
    b->ecv.notify_all();
    if (d2h) {
        cudaStreamSynchronize(d2h);
        cudaStreamDestroy(d2h);
    }
    for (StageSlot &st : slots) {
        free_buf(st.sup);
        free_buf(st.t);
        free_buf(st.h);
        free_buf(st.c);
        free_buf(st.ro);
        if (st.d2d) cudaEventDestroy(st.d2d);
        if (st.done) cudaEventDestroy(st.done);
    }
}

static int batch_start(Ctx &c, const int32_t *pairs, int64_t n_pairs, const BatchParams &prm, int streams,
                       bool deliver, w1g_front_end_info *infos) {
    if (c.corpus_n < 0) {
        set_error("batch: no diagrams loaded (w1g_corpus_load)");
        return W1G_ESTATE;
    }
    if (n_pairs < 0 || (n_pairs && !pairs) || streams < 1 || streams > 64) {
        set_error("batch: bad arguments");
        return W1G_EINVAL;
    }
    for (int64_t p = 0; p < 2 * n_pairs; p++)
        if (pairs[p] < 0 || pairs[p] >= c.corpus_n) {
            set_error("batch: diagram index %d out of range [0, %lld)", pairs[p], (long long)c.corpus_n);
            return W1G_EINVAL;
        }
    if (!c.batch) c.batch = new BatchState();
    BatchState &b = *c.batch;
    if (b.active) {
        set_error("batch: a batch is already running on this context");
        return W1G_ESTATE;
    }
    W1G_TRY(ensure_kids(c, b, streams));
    // several concurrent front ends: the cooperative kernels of the split tree and the WSPD
    // on a 1/streams share of the device each, so the children's grids are co-resident
    // (measured, 4 child contexts: cfg2 1706 pairs/s with shares, 1624 with the multi-kernel
    // level loops, 1496 with full grids; 20k points 3265 / 2508 / 2748).
    // W1G_BATCH_COOP=full: full grids; =off: the level loops.
    static const int batch_coop = [] {
        const char *e = getenv("W1G_BATCH_COOP");
        if (!e) return 0;
        return !strcmp(e, "full") ? 1 : !strcmp(e, "off") ? 2 : 0;
    }();
    for (w1g_ctx *x : b.kids) {
        const bool several = streams > 1;
        x->no_coop = (several && batch_coop == 2) ? 1 : 0;
        x->coop_share = (several && batch_coop == 0) ? streams : 1;
    }
    if (!c.h_corpus_ptr) W1G_CUDA(cudaStreamSynchronize(c.stream));  // the corpus upload is complete
    b.pairs.assign(pairs, pairs + 2 * n_pairs);
    b.n_pairs = n_pairs;
    b.prm = prm;
    b.deliver = deliver;
    b.infos = infos;
    b.next.store(0);
    b.cancel.store(false);
    b.ready.clear();
    b.delivered = b.produced = 0;
    b.first_rc = W1G_OK;
    b.first_err.clear();
    b.active = true;
    {
        const char *e = getenv("W1G_BATCH_TRACE");
        b.trace = e && (*e == '1' || *e == '2');
        b.trace_steps = e && *e == '2';
        b.tr_block.assign(b.kids.size(), 0.0);
        b.tr_fe.assign(b.kids.size(), 0.0);
        b.tr_fetch.assign(b.kids.size(), 0.0);
        b.tr_pairs.assign(b.kids.size(), 0.0);
    }
    const int nt = (int)(n_pairs < streams ? (n_pairs > 0 ? n_pairs : 1) : streams);
    {
        const char *e = getenv("W1G_BATCH_COMPACT");
        b.compact = !deliver ? 0 : (e && *e == '0') ? 0 : (e && *e == '2') ? 2 : 1;
    }
    b.expand_q.clear();
    b.workers_left = nt;
    for (int w = 0; w < nt; w++) b.threads.emplace_back(batch_worker, &c, &b, w);
    if (b.compact) {
        // W1G_BATCH_EXPANDERS: threads rebuilding networks on the host (default: half the
        // hardware threads, 2..8)
        int ne = (int)std::thread::hardware_concurrency() / 2;
        if (const char *e = getenv("W1G_BATCH_EXPANDERS")) ne = atoi(e);
        ne = ne < 1 ? 1 : ne > 16 ? 16 : ne;
        if (!getenv("W1G_BATCH_EXPANDERS")) ne = ne < 2 ? 2 : ne > 8 ? 8 : ne;
        for (int q = 0; q < ne; q++) b.expanders.emplace_back(batch_expander, &b);
    }
    return W1G_OK;
}

void batch_destroy(Ctx &c) {
    if (!c.batch) return;
    BatchState &b = *c.batch;
    b.cancel.store(true);
    host_pool().wake();
    batch_join(b);
    for (auto &r : b.ready)
        if (r.block) host_pool().put(r.block);
    for (w1g_ctx *x : b.kids) w1g_ctx_destroy(x);
    for (cudaEvent_t e : b.kid_ev) cudaEventDestroy(e);
    if (b.ev_start) cudaEventDestroy(b.ev_start);
    if (b.ev_end) cudaEventDestroy(b.ev_end);
    delete c.batch;
    c.batch = nullptr;
}

}  // namespace w1g

using namespace w1g;

extern "C" {

int w1g_front_end_batch(w1g_ctx *c, const int32_t *pairs, int64_t n_pairs, double s, int use_condensation,
                        int delta_mode, double delta, double k, uint64_t seed, int streams,
                        w1g_front_end_info *infos, float *device_ms) {
    if (!c) return W1G_EINVAL;
    cudaSetDevice(c->device);
    BatchParams prm{s, delta, k, use_condensation, delta_mode, seed};
    if (!c->batch) c->batch = new BatchState();
    BatchState &b = *c->batch;
    W1G_TRY(ensure_kids(*c, b, streams));
    // device makespan: every child stream starts after an event on the parent
    // stream, and the parent stream's end event waits for every child
    if (!b.ev_start) {
        W1G_CUDA(cudaEventCreate(&b.ev_start));
        W1G_CUDA(cudaEventCreate(&b.ev_end));
    }
    while (b.kid_ev.size() < b.kids.size()) {
        cudaEvent_t e;
        W1G_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        b.kid_ev.push_back(e);
    }
    W1G_CUDA(cudaEventRecord(b.ev_start, c->stream));
    for (w1g_ctx *x : b.kids) W1G_CUDA(cudaStreamWaitEvent(x->stream, b.ev_start, 0));
    W1G_TRY(batch_start(*c, pairs, n_pairs, prm, streams, false, infos));
    batch_join(b);
    b.active = false;
    for (size_t w = 0; w < b.kids.size(); w++) {
        W1G_CUDA(cudaEventRecord(b.kid_ev[w], b.kids[w]->stream));
        W1G_CUDA(cudaStreamWaitEvent(c->stream, b.kid_ev[w], 0));
    }
    W1G_CUDA(cudaEventRecord(b.ev_end, c->stream));
    W1G_CUDA(cudaEventSynchronize(b.ev_end));
    if (device_ms) W1G_CUDA(cudaEventElapsedTime(device_ms, b.ev_start, b.ev_end));
    if (b.first_rc != W1G_OK) {
        set_error("%s", b.first_err.c_str());
        return b.first_rc;
    }
    return W1G_OK;
}

int w1g_batch_begin(w1g_ctx *c, const int32_t *pairs, int64_t n_pairs, double s, int use_condensation,
                    int delta_mode, double delta, double k, uint64_t seed, int streams,
                    int64_t max_inflight_bytes) {
    if (!c) return W1G_EINVAL;
    cudaSetDevice(c->device);
    if (max_inflight_bytes > 0) {
        std::lock_guard<std::mutex> lk(host_pool().mu);
        host_pool().limit = (size_t)max_inflight_bytes;
    }
    BatchParams prm{s, delta, k, use_condensation, delta_mode, seed};
    return batch_start(*c, pairs, n_pairs, prm, streams, true, nullptr);
}

int w1g_batch_next(w1g_ctx *c, w1g_batch_result *out) {
    if (!c || !out || !c->batch || !c->batch->active) {
        set_error("batch_next: no batch running");
        return W1G_ESTATE;
    }
    BatchState &b = *c->batch;
    std::unique_lock<std::mutex> lk(b.mu);
    b.cv.wait(lk, [&] {
        return !b.ready.empty() || b.produced >= b.n_pairs || (b.cancel.load() && b.first_rc != W1G_OK);
    });
    if (!b.ready.empty()) {
        *out = b.ready.front();
        b.ready.pop_front();
        b.delivered++;
        return W1G_OK;
    }
    return W1G_DONE;
}

int w1g_batch_release(void *block) {
    if (block) host_pool().put(block);
    return W1G_OK;
}

static void batch_trace_print(BatchState &b) {
    if (!b.trace) return;
    for (size_t w = 0; w < b.tr_fe.size(); w++)
        if (b.tr_pairs[w] > 0)
            fprintf(stderr, "[w1g batch] worker %zu: %.0f pairs, block wait %.0f us, front end %.0f us, fetch %.0f us\n",
                    w, b.tr_pairs[w], b.tr_block[w], b.tr_fe[w], b.tr_fetch[w]);
}

int w1g_batch_end(w1g_ctx *c) {
    if (!c || !c->batch) return W1G_OK;
    BatchState &b = *c->batch;
    b.cancel.store(true);
    host_pool().wake();
    batch_join(b);
    batch_trace_print(b);
    for (auto &r : b.ready)
        if (r.block) host_pool().put(r.block);
    b.ready.clear();
    b.active = false;
    for (w1g_ctx *x : b.kids) cudaStreamSynchronize(x->stream);
    return W1G_OK;
}

}  // extern "C"
