// common.cuh -- shared infrastructure of libw1g.so (sm_100a only).
//
// Context / device-buffer plumbing, error reporting, the exact-IEEE fp64
// helpers every reference-parity kernel uses, a single-pass decoupled
// look-back scan and the LSD radix sort interface.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/w1g.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libw1g is built for sm_100a only"
#endif

namespace w1g {

// ------------------------------------------------------------------ errors
void set_error(const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define W1G_CUDA(call)                                                      \
    do {                                                                    \
        cudaError_t _e = (call);                                            \
        if (_e != cudaSuccess) return ::w1g::cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)
// every kernel launch is followed by W1G_CHECK_LAUNCH(), which also counts it
extern unsigned long long g_launches;
#define W1G_CHECK_LAUNCH()                                  \
    do {                                                    \
        __atomic_fetch_add(&::w1g::g_launches, 1ull, __ATOMIC_RELAXED); \
        W1G_CUDA(cudaGetLastError());                       \
    } while (0)
#define W1G_TRY(expr)                \
    do {                             \
        int _rc = (expr);            \
        if (_rc != W1G_OK) return _rc; \
    } while (0)

// ------------------------------------------------------------------ buffers
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
};
// grow-only device buffer (geometric); contents are NOT preserved on growth
int ensure_bytes(DevBuf &b, size_t bytes);
void set_thread_stream(cudaStream_t s);  // stream-ordered growth for this thread's context
template <class T>
inline int ensure(DevBuf &b, size_t n, T **out) {
    int rc = ensure_bytes(b, n * sizeof(T) + 16);
    *out = static_cast<T *>(b.p);
    return rc;
}
template <class T>
inline T *ptr(DevBuf &b) { return static_cast<T *>(b.p); }
void free_buf(DevBuf &b);

struct NodeSet {
    int64_t k = 0;
    bool valid = false;
    DevBuf pts;  // (k) double2 (x, y), node order
    DevBuf am;   // (k) int64 a_mass
    DevBuf bm;   // (k) int64 b_mass
    int64_t abar = 0, bbar = 0;
    // positions of the nodes with a- / b-mass among themselves (exclusive scans)
    // and their counts, computed by delta_condense for emit_arcs (na < 0: absent)
    DevBuf exa, exb;
    int64_t na = -1, nb = -1;
    // from zero_condense (stats = true): the per-side member counts and the
    // bbox as dkey()s [xmin, xmax, ymin, ymax] -- RWMD's frame without a round trip
    bool stats = false;
    int64_t nmem[2] = {0, 0};
    uint64_t bbox_key[4] = {0, 0, 0, 0};
};

// per-node geometry used by the WSPD predicate (spanner.py:176-194), computed
// once per node with the reference's exact operation sequence
struct NodeGeom {
    double cx, cy;  // 0.5*(xmin+xmax), 0.5*(ymin+ymax)
    double r;       // 0.5*sqrt(w*w+h*h)
    double dsq;     // w*w+h*h
};

enum { SCR_N = 24 };

// A persistent host thread that runs one job at a time for an auxiliary
// context (the fused front end's zero_condense + RWMD leg): created with the
// context, joined when it is destroyed, so no call creates a thread.
// submit() hands a job over; wait() blocks until it has finished.  The job
// may reference the submitter's stack: every submitter waits before returning
// (the front end's scope guard does so on every exit path).
// A few persistent host threads for a parallel host loop inside one API call
// (run(parts, f): f(0..parts-1), the caller takes a share; returns when all are done).
struct FillPool {
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::function<void(int)> job;
    int parts = 0, next = 0, left = 0;
    uint64_t gen = 0;
    bool quit = false;
    void start(int n) {
        for (int q = 0; q < n; q++)
            th.emplace_back([this] {
                uint64_t seen = 0;
                std::unique_lock<std::mutex> lk(mu);
                for (;;) {
                    cv.wait(lk, [&] { return quit || gen != seen; });
                    if (quit) return;
                    seen = gen;
                    while (next < parts) {
                        const int p = next++;
                        lk.unlock();
                        job(p);
                        lk.lock();
                        if (--left == 0) done_cv.notify_all();
                    }
                }
            });
    }
    void run(int n, std::function<void(int)> f) {
        std::unique_lock<std::mutex> lk(mu);
        job = std::move(f);
        parts = n;
        next = 0;
        left = n;
        gen++;
        cv.notify_all();
        while (next < parts) {
            const int p = next++;
            lk.unlock();
            job(p);
            lk.lock();
            --left;
        }
        done_cv.wait(lk, [&] { return left == 0; });
        job = nullptr;
    }
    ~FillPool() {
        {
            std::lock_guard<std::mutex> lk(mu);
            quit = true;
        }
        cv.notify_all();
        for (auto &t : th) t.join();
    }
};

struct AuxWorker {
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::function<void()> job;
    bool busy = false, quit = false;
    void start() {
        th = std::thread([this] {
            std::unique_lock<std::mutex> lk(mu);
            for (;;) {
                cv.wait(lk, [this] { return quit || (busy && job); });
                if (quit) return;
                std::function<void()> f = std::move(job);
                job = nullptr;
                lk.unlock();
                f();
                lk.lock();
                busy = false;
                cv.notify_all();
            }
        });
    }
    void submit(std::function<void()> f) {
        std::lock_guard<std::mutex> lk(mu);
        job = std::move(f);
        busy = true;
        cv.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [this] { return !busy; });
    }
    void stop() {
        if (!th.joinable()) return;
        {
            std::lock_guard<std::mutex> lk(mu);
            quit = true;
        }
        cv.notify_all();
        th.join();
    }
};

struct BatchState;  // batch.cu

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // early D2H of the fused network (tails, row offsets)
    int sm_count = 148;

    DevBuf in_pts;  // (na+nb) double2
    NodeSet nodes[2];
    NodeSet raw;    // the raw inputs as nodes (split fixed-delta front end)
    NodeSet nodes0_stash;  // an auxiliary context's own nodes0 while it aliases the main one's

    // rwmd
    int culling = 1;
    int cull_steps = 0;  // 0 = by size; W1G_CULL_STEPS overrides (tuning)
    int debug_radius = 0;  // W1G_DEBUG_RADIUS=1: rwmd "best" reports the exact-pass radius
    // RWMD kernel profiling (w1g_profile_rwmd): events around the FP32 tile and the
    // exact refine kernels of each side, and device counters of the (source,
    // target) evaluations they perform: [side][0 = tile, 1 = refine]
    int prof = 0, prof_side = 0;
    // prefer the multi-kernel level loops to the cooperative (grid-barrier) kernels of the
    // split tree and the WSPD: set on the batch executor's child contexts when several run
    // concurrently (a cooperative grid must be co-resident, which throttles the others)
    int no_coop = 0;
    // the cooperative kernels' grid as a share of the device's resident CTAs (1 = all):
    // concurrent child contexts each take 1/share, so their grids stay co-resident
    int coop_share = 1;
    cudaEvent_t prof_ev[2][2][2] = {};
    DevBuf prof_cnt;  // 4 x unsigned long long
    int heavy_ratio = 16;  // exact pass: disc / median disc beyond which a source is searched alone (W1G_HEAVY, 0 off)
    DevBuf best[2];
    int64_t n_best[2] = {0, 0};
    // numpy pairwise-sum trees per side, rebuilt only when the length changes
    DevBuf pw_nodes[2], pw_lev[2];
    int64_t pw_n[2] = {-1, -1};
    int64_t rw_members[2] = {0, 0};  // A- and B-member counts of the last rwmd_run

    // split tree (over `tree_pts`, a copy of the slot's points)
    bool tree_valid = false;
    int64_t tree_n_points = 0, tree_n_nodes = 0;
    int32_t tree_depth = 0;
    DevBuf tree_pts;                                // double2
    DevBuf t_left, t_right, t_rep, t_size, t_bbox;  // int64 x4, double x4 (reference layout)
    DevBuf t_geom;                                  // NodeGeom per node
    DevBuf t_lr;                                    // int2 (left, right) per node, -1 leaf
    DevBuf t_rep32;                                 // int32 rep
    // the split tree's X- and Y-lists, built by delta_condense from its cell
    // order (pre_n = node count they are for, 0 = none; consumed by tree_run)
    DevBuf pre_xl, pre_yl, pre_cells, pre_rows, pre_rcnt;
    int64_t pre_n = 0;
    const double2 *pair_pts = nullptr;              // points the pairs' reps index

    // WSPD
    bool pairs_valid = false;
    int64_t n_pairs = 0;
    int32_t wspd_levels = 0;
    DevBuf pair_uv;    // int2 (u, v) tree node ids
    // depth-first WSPD: the work pool's per-chunk ready flags (all zero between runs)
    // and its counters, one 128-byte line each
    DevBuf wspd_ready, wspd_ctr;
    int32_t wspd_epoch = 0;
    DevBuf pair_w;     // int32 owner internal node of each level-0 recursion item (reference order)
    DevBuf pair_idx;   // int64 (P,2) representative point indices
    DevBuf pair_counts;
    bool pairs_have_nodes = false;
    bool pair_idx_valid = false;  // pair_idx matches pair_uv (or was loaded)

    // arcs (emit_arcs output, reference order)
    bool arcs_valid = false;
    int64_t n_arcs = 0;
    DevBuf arc_t, arc_h, arc_c;

    // network (CSR)
    bool net_valid = false;
    bool net_check_pending = false;  // spanner_net_run's flags not yet read
    bool net_early_copy = false;     // tails + row offsets already copied out (copy_stream, ev[13])
    bool net_tails_host = false;     // ...row offsets only: the tails are rebuilt on the host (ev[16])
    struct FillPool *fill_pool = nullptr;  // host threads rebuilding the tails (lazily started)
    int64_t net_n = 0, net_m = 0;
    DevBuf net_sup, net_t, net_h, net_c, net_ro;

    // scratch
    DevBuf scr[SCR_N];
    DevBuf sort_scr[2][8];  // radix sort scratch per job
    DevBuf lex_scr[2][6];   // sort_lex2 scratch per job
    unsigned sort_epoch = 0;  // onesweep status-word epoch (sort.cu)
    DevBuf scan_state;
    DevBuf scan_state2;  // a second decoupled-look-back state for a scan on the side stream
    DevBuf flags;  // small device flag block (int64 x 64)
    int64_t *h_pinned = nullptr;  // pinned host mirror of `flags`
    void *h_stage = nullptr;      // pinned staging buffer for H2D / D2H
    size_t h_stage_cap = 0;

    cudaEvent_t ev[18] = {};

    // fixed-delta front end: RWMD (which then only feeds diagnostics and the
    // L > 0 test) runs on a second context -- own stream, scratch and host
    // thread -- concurrently with the back end.  W1G_OVERLAP selects where it
    // starts: 4 (default) after delta_condense, 3 after the split tree, 1 after
    // the WSPD, 2 right after zero_condense, 0 = sequential (measured at cfg2:
    // 4 -> 1.44 ms, 3 -> 1.55, 1 -> 1.66, 2 -> 1.60, 0 -> 1.74)
    int overlap = 4;
    // when the network is copied out inside the call (an armed w1g_set_network_out
    // target) RWMD starts after the WSPD and runs under the CSR and the copy
    // (W1G_OVERLAP_E2E; measured e2e: 1 -> 5.48 ms at 1M / 2.24 at cfg2, 4 -> 6.87 / 2.32,
    // 3 -> 7.01 / 2.29, 5 (after the CSR) -> 7.28 / 2.65)
    int overlap_e2e = 1;
    // split front end: the main-stream point RWMD waits for (0 = none, else a
    // spawn point as above), without / with an armed output target
    int split_gate = 0, split_gate_e2e = 1;
    int split_gate_set = 0;  // W1G_SPLIT_GATE given: no size-based choice
    Ctx *aux = nullptr;
    AuxWorker *aux_worker = nullptr;  // the host thread that drives `aux` (owned by this context)
    BatchState *batch = nullptr;      // batch executor: child contexts + workers (batch.cu)

    // a diagram corpus resident on the device (w1g_corpus_load): points of all
    // diagrams back to back, diagram i = [corpus_off[i], corpus_off[i+1])
    DevBuf corpus_pts, query_pts, dense_scr[4];
    int64_t corpus_n = -1;
    int64_t *h_corpus_off = nullptr;  // host copy of the offsets (n + 1)
    // host-resident corpus (w1g_corpus_set_host): the caller's arrays, copied to the
    // device per pair inside each batch worker's front end (overlapping other pairs)
    const double **h_corpus_ptr = nullptr;

    // one-shot host target for the next fused front end's network (w1g_set_network_out)
    struct NetOut {
        int64_t *sup = nullptr, *t = nullptr, *h = nullptr, *ro = nullptr;
        double *c = nullptr;
        int64_t node_cap = 0, arc_cap = 0;
    } net_out;

    // host round-trip accounting (stream_sync)
    int timing = 0;
    // launch sequences between host round trips replayed as CUDA graphs (graph_segment):
    // one executable graph per segment, updated in place for each call's parameters
    cudaGraphExec_t gseg[8] = {};
    int gseg_off[8] = {};  // the segment could not be captured: eager launches
    int64_t n_syncs = 0;
    double sync_gap_us = 0.0;
    cudaEvent_t sync_ev[2] = {};
};

// device flag block layout (int64 slots)
enum FlagSlot {
    F_K0 = 0,
    F_UNBALANCED = 1,
    F_OVERFLOW = 2,
    F_DUP = 3,
    F_ACTIVE = 4,
    F_PAIRS = 5,
    F_FRONT = 6,
    F_PAIR_OVF = 7,
    F_FRONT_OVF = 8,
    F_NET_ERR = 9,
    F_TOTAL = 10,
    F_ZC_TICKET = 11,  // k_zc_stats: blocks done (the last one publishes to the host mirror)
    F_MISC0 = 12,
    F_MISC1 = 13,
    F_MISC2 = 14,
    F_MISC3 = 15,
    F_CELL_MIN = 16,  // 4 slots: min cx, max cx, min cy, max cy
    F_TREE_TICKET = 20,  // k_tree_local: CTAs done (the last one publishes depth / duplicates; reset by it)
    F_BBOX = 24,      // 4 doubles (as bits)
    F_SCAL = 32,      // 8 doubles of scalar results
    F_LISTS = 40,     // delta_condense's presorted tree lists failed a check (tree sorts itself)
    F_ZSTAT = 41,     // 6 slots: zero_condense's member counts (a, b), ~min / max dkey of x, of y
    F_NSLOTS = 64
};

// Small device -> host transfers (flags, counters, scalars) are written by a one-CTA
// kernel straight into page-locked host memory (device-accessible under UVA) instead
// of a cudaMemcpyAsync: copies go through the copy engines, where a few bytes would
// queue behind the large network transfers of other contexts on the same GPU (the
// batch executor's workers), stalling this context's host round trip.  h_dst must be
// page-locked (h_pinned slots, pool blocks); bytes a multiple of 4.
int to_host_small(Ctx &c, void *h_dst, const void *d_src, size_t bytes, cudaStream_t s = nullptr);
int to_host_small2(Ctx &c, void *h0, const void *d0, size_t b0, void *h1, const void *d1, size_t b1);
void host_copy_nt(void *dst, const void *src, size_t bytes);  // host copy, non-temporal stores
// Run `body` (launches on c.stream, no host synchronisation) captured as a CUDA graph and
// replayed with one graph launch: the device fetches one command instead of one per
// kernel (launches are slow to submit while the host link is busy with network copies:
// 87 small kernels 375 -> 862 us, as one graph 84 -> 107 us).  Buffers that must grow,
// or an operation capture rejects, fall back to running `body` eagerly.  Opt-in
// (W1G_GRAPHS=1): capturing and updating cost the host as much as the launches, and the
// end-to-end batch did not gain (measured and rejected).
enum { GSEG_ZC = 0, GSEG_DC = 1, GSEG_TREE_WSPD = 2, GSEG_CSR = 3 };
constexpr int W1G_ERECAPTURE = -100;  // internal: ensure() would allocate during a capture
int graph_segment(Ctx &c, int slot, const std::function<int()> &body);
// h_pinned slots for scalar results read back by the stages (RWMD sums)
enum { H_SCALAR = 48 };  // 8 slots: 48..55
int flags_reset(Ctx &c);
// host wait for the context stream.  Every host round trip leaves the GPU
// idle (D2H + wake-up + next launch); with W1G_TIMING=1 the idle time is
// measured with events on both sides and printed per front end.
int stream_sync(Ctx &c);
int flags_fetch(Ctx &c, int first, int count);  // D2H into h_pinned + stream sync
inline int64_t *dflags(Ctx &c) { return ptr<int64_t>(c.flags); }

// pinned staging (host) buffer
int stage_ensure(Ctx &c, size_t bytes);

// ------------------------------------------------------------------ exact fp64
// Every reference-parity fp64 expression is written with the _rn intrinsics so
// that no FMA contraction can occur regardless of compiler flags.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// IEEE-754 total order key for non-NaN doubles, with -0.0 folded onto +0.0
// (np.unique / np.lexsort compare floats, so -0.0 == +0.0).
__device__ __forceinline__ uint64_t dkey(double v) {
    if (v == 0.0) v = 0.0;
    uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
// signed int64 -> order-preserving uint64
__device__ __forceinline__ uint64_t ikey(int64_t v) { return (uint64_t)v ^ 0x8000000000000000ull; }

// ------------------------------------------------------------------ scan
// Exclusive prefix sum of int64 values produced by a functor, one pass with
// decoupled look-back.  out may be null (only the total is wanted).
struct ScanArgs {
    unsigned long long *status;  // tiles
    unsigned int *ticket;
};
constexpr int SCAN_BLOCK = 256;
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_IPT;

int scan_prepare(Ctx &c, int64_t n, ScanArgs *a, int64_t *n_tiles);

template <class F>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_i64(F f, int64_t n, int64_t *out,
                                                        int64_t *total, ScanArgs a,
                                                        const int32_t *live) {
    // `live` (optional): a device counter; when it is 0 the whole scan is a no-op
    if (live && *live == 0) return;
    __shared__ unsigned int s_tile;
    __shared__ int64_t s_warp[SCAN_BLOCK / 32];
    __shared__ int64_t s_prefix;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    int64_t v[SCAN_IPT];
    int64_t tsum = 0;
#pragma unroll
    for (int i = 0; i < SCAN_IPT; i++) {
        int64_t idx = base + i;
        v[i] = idx < n ? (int64_t)f(idx) : 0;
        tsum += v[i];
    }
    // block exclusive scan of tsum
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < SCAN_BLOCK / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < SCAN_BLOCK / 32) s_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int64_t warp_excl = wid ? s_warp[wid - 1] : 0;
    const int64_t excl = warp_excl + x - tsum;
    const int64_t agg = s_warp[SCAN_BLOCK / 32 - 1];
    if (wid == 0) {
        // warp-parallel decoupled look-back: 32 predecessors per memory round trip
        constexpr unsigned long long FA = 1ull << 62, FP = 2ull << 62, MASK = (1ull << 62) - 1;
        if (tile == 0) {
            if (lane == 0) {
                atomicExch(&a.status[0], FP | (unsigned long long)agg);
                s_prefix = 0;
            }
        } else {
            if (lane == 0) atomicExch(&a.status[tile], FA | (unsigned long long)agg);
            int64_t prefix = 0;
            int64_t j = tile - 1;
            while (true) {
                const int64_t idx = j - lane;
                const unsigned long long st =
                    idx >= 0 ? *((volatile unsigned long long *)&a.status[idx]) : FP;  // before tile 0: prefix 0
                const unsigned kind = (unsigned)(st >> 62);
                const unsigned inc = __ballot_sync(0xffffffffu, kind == 2);
                const unsigned unpub = __ballot_sync(0xffffffffu, kind == 0);
                const int first = inc ? __ffs(inc) - 1 : 31;
                const unsigned need = (2u << first) - 1u;  // lanes 0..first
                if (unpub & need) continue;                // someone in range not published: re-poll
                int64_t v = lane <= first ? (int64_t)(st & MASK) : 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (inc) break;
                j -= 32;
            }
            if (lane == 0) {
                atomicExch(&a.status[tile], FP | (unsigned long long)(prefix + agg));
                s_prefix = prefix;
            }
        }
    }
    __syncthreads();
    if (out) {
        int64_t run = s_prefix + excl;
#pragma unroll
        for (int i = 0; i < SCAN_IPT; i++) {
            int64_t idx = base + i;
            if (idx < n) out[idx] = run;
            run += v[i];
        }
    }
    if (total && threadIdx.x == 0 && tile == (n > 0 ? (n - 1) / SCAN_TILE : 0)) *total = s_prefix + agg;
}

template <class F>
int scan_i64(Ctx &c, F f, int64_t n, int64_t *out, int64_t *total, const int32_t *live = nullptr) {
    ScanArgs a;
    int64_t tiles;
    W1G_TRY(scan_prepare(c, n, &a, &tiles));
    k_scan_i64<F><<<(unsigned)tiles, SCAN_BLOCK, 0, c.stream>>>(f, n, out, total, a, live);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

// ------------------------------------------------------------------ radix sort
// Stable LSD radix sort, 8-bit digits, ascending by a key of `words` uint64
// words (keys[words-1] most significant), carrying a uint32 payload.  The
// key words and the payload are permuted in place (ping-pong internally).
// Digits whose value is the same for every key are skipped (one D2H of the
// digit histogram per sort).  bits_hint limits the digits considered in the
// most-significant word (64 = all).
int radix_sort(Ctx &c, uint64_t **keys, int words, uint32_t *vals, int64_t n, int top_bits = 64);
// Up to two independent sorts of the same shape in the same launches (one
// histogram D2H, each pass one kernel over the tiles of both): small sorts
// that would each leave most SMs idle run side by side.
struct SortJob {
    uint64_t *keys[3];
    uint32_t *vals;
    int64_t n;
};
int radix_sort_multi(Ctx &c, const SortJob *jobs, int njobs, int words, int top_bits = 64);
// Stable sort of vals (initially the element ids 0..n-1) by (primary[i],
// secondary[i]) -- both dkey()s of doubles: radix passes over a 32-bit
// order-preserving compression of the primary (linear in value over its
// range), then the elements of
// compressed-key tie runs by the full (primary, secondary, id) -- in place by
// one thread per run when every run is short, else by a two-word radix sort.
// `primary` and `secondary` are indexed by element id.
int sort_lex2(Ctx &c, const uint64_t *primary, const uint64_t *secondary, uint32_t *vals, int64_t n,
              bool speculative = false);
// speculative = true: no host round trip -- short tie runs are ordered in place and
// the longest run is copied to h_pinned[H_LEX_MAXRUN + job] for the caller to check
// after its next synchronisation (lex2_speculation_failed -> redo non-speculatively)
bool lex2_speculation_failed(Ctx &c, int njobs);
struct Lex2Job {
    const uint64_t *primary, *secondary;
    uint32_t *vals;
    int64_t n;
};
int sort_lex2_multi(Ctx &c, const Lex2Job *jobs, int njobs, bool speculative = false);

// ------------------------------------------------------------------ misc
inline unsigned grid_for(int64_t n, int block, unsigned cap = 0x7fffffffu) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > (int64_t)cap) g = cap;
    return (unsigned)g;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Optional sub-stage timing (W1G_TIMING=1): CUDA events on the context stream,
// one line per mark printed to stderr when the timer goes out of scope.
struct SubTimer {
    Ctx &c;
    const char *stage;
    bool on;
    int n = 0;
    cudaEvent_t ev[24];
    const char *name[24];
    SubTimer(Ctx &ctx, const char *s) : c(ctx), stage(s) {
        const char *e = getenv("W1G_TIMING");
        on = e && *e == '1';
        if (on) mark("start");
    }
    void mark(const char *nm) {
        if (!on || n >= 24) return;
        cudaEventCreate(&ev[n]);
        cudaEventRecord(ev[n], c.stream);
        name[n++] = nm;
    }
    ~SubTimer() {
        if (!on || n < 2) return;
        cudaEventSynchronize(ev[n - 1]);
        fprintf(stderr, "[w1g %s]", stage);
        for (int i = 1; i < n; i++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, " %s=%.1fus", name[i], 1e3f * ms);
        }
        fprintf(stderr, "\n");
        for (int i = 0; i < n; i++) cudaEventDestroy(ev[i]);
    }
};

// stage launchers (one translation unit each)
int zc_run(Ctx &c, const double2 *d_a, int64_t na, const double2 *d_b, int64_t nb, int64_t *k0,
           int32_t *balanced, bool speculative = true);
int rwmd_run(Ctx &c, double *L, double *LA, double *LB);
int rwmd_tile_profile(Ctx &c, int reps, float *ms, int64_t *evals);
int rwmd_profile(Ctx &c, int reps, float *ms, int64_t *evals, int64_t *directed);
int rwmd_range_run(Ctx &c, int side, int64_t begin, int64_t end, double *partial, int64_t *n_members);
// src: the node set to condense (default nodes[0]); the result goes to nodes[1]
int dc_run(Ctx &c, double delta, double pitch, double half_width, uint64_t seed, int64_t *k,
           NodeSet *src = nullptr);
// standalone snap_points (host arrays in and out)
int snap_run(Ctx &c, const double *h_pts, int64_t k, double pitch, double *h_snapped, int64_t *h_cells);
// the raw diagrams as a node set (unit masses, duplicates kept) into c.raw:
// delta_condense of it equals delta_condense of zero_condense's output
int raw_nodes(Ctx &c, const double2 *d_a, int64_t na, const double2 *d_b, int64_t nb);
// defer = true (fused front end): no host round trip of its own -- the depth and the
// duplicate flag land in h_pinned[H_TREE_DEPTH / H_TREE_DUP] at the caller's next
// synchronisation, and the caller checks the flag (tree_deferred_check)
int tree_run(Ctx &c, const double2 *d_pts, int64_t n, int64_t *n_nodes, int32_t *depth, bool defer = false);
int tree_deferred_check(Ctx &c, int32_t *depth);
// h_pinned slots no flags fetch touches
enum { H_LEX_MAXRUN = F_NSLOTS - 4, H_TREE_DEPTH = F_NSLOTS - 2, H_TREE_DUP = F_NSLOTS - 1 };
int tree_geom(Ctx &c);
// shard / n_shards (fused order only): the recursions of the internal nodes w with
// w % n_shards == shard -- one GPU's share of a sharded WSPD
int wspd_run(Ctx &c, double s, int reference_order, int64_t *n_pairs, bool want_idx = true, int shard = 0,
             int n_shards = 1);
int wspd_pair_idx(Ctx &c);  // pair_idx from pair_uv and the tree's reps, unless current
// with_diagonal = false: only the pairs' arcs (both directions), no diagonal / free arcs
int emit_run(Ctx &c, int64_t *n_arcs, bool with_diagonal = true);
int net_run(Ctx &c, const int64_t *d_supplies, int64_t n, int64_t *n_arcs);
int assemble_supplies(Ctx &c, int64_t **d_sup, int64_t *n);
// corpus.cu: a resident diagram corpus, WCD / RWMD scores of a query against it
// (pipeline.py:191-243 nn_search stages), the dense exact-oracle network (oracle.py:66-93)
int corpus_load(Ctx &c, const double *pts, const int64_t *offsets, int64_t n);
int corpus_set_host(Ctx &c, const double *const *pts, const int64_t *sizes, int64_t n);
int wcd_corpus(Ctx &c, const double *query, int64_t nq, const int64_t *cand, int64_t ncand, double *scores);
int rwmd_corpus(Ctx &c, const double *query, int64_t nq, const int64_t *cand, int64_t ncand, double *scores);
int dense_network_run(Ctx &c, int64_t *node_count, int64_t *n_arcs);
void batch_destroy(Ctx &c);  // joins a batch's workers, destroys its child contexts
// fused front end: emit_arcs + assemble straight from the WSPD pairs (the arc
// list is not materialised); falls back to emit_run + net_run when needed
// its validation flags are read by spanner_net_check once the stream has drained
int spanner_net_run(Ctx &c, int64_t *node_count, int64_t *n_arcs);
int spanner_net_check(Ctx &c, int64_t *node_count, int64_t *n_arcs, bool *redone);

}  // namespace w1g

struct w1g_ctx : public w1g::Ctx {};
