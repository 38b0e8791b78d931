// wspd.cu -- well-separated pair decomposition (spanner.py:176-307) on device.
//
// The reference runs one DFS per internal node w from (left[w], right[w]):
// a pair (u, v) is emitted when _ws_predicate holds, otherwise the side with
// the larger bbox diagonal (_diag_sq) is replaced by its two children.  The
// emitted SET is a function of the tree and s only.  Every item evaluates the
// predicate with the reference's exact fp64 operation order (per-node
// centres/radii precomputed in tree.cu with the same operations).
//
// Fused order (the front end): k_wspd_dfs -- every warp runs recursions depth
// first on a stack in shared memory, work shared through a ticketed chunk queue
// (see there).  The level-synchronous alternative (W1G_WSPD_DFS=0): CTA-local
// owner recursions, then all remaining recursions advance together as one
// breadth-first frontier of (u, v) items in a cooperative kernel (a grid
// barrier per level) or level launches.  Buffers regrow and the pass reruns on
// overflow.
//
// reference_order = 1 additionally keeps every level of the frontier (the
// whole recursion forest, one item per (u, v) the reference's stacks ever
// hold) with a link per item -- its pair slot, or the index of its two
// children -- and then lays the pairs out in the reference's exact order
// (owner ascending, DFS pop order with the right child popped first,
// spanner.py:206-241) the way the reference's own two passes do, one level at
// a time: leaf counts bottom-up (count_pairs), an exclusive scan over the
// owners (build_wspd's offsets), and offsets top-down (the right child at its
// parent's offset, the left child after the right child's leaves).  Any
// recursion depth works, like the reference's explicit stack.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace w1g {

namespace {

struct ItemF {  // one (u, v) recursion item
    int32_t u, v;
};

__device__ __forceinline__ bool ws_predicate(const NodeGeom &a, const NodeGeom &b, double s) {
    // spanner.py:176-187: r = max radius, centre distance - 2r >= s*r
    const double r = a.r > b.r ? a.r : b.r;
    const double dx = dsub(a.cx, b.cx), dy = dsub(a.cy, b.cy);
    return dsub(dsqrt(dadd(dmul(dx, dx), dmul(dy, dy))), dmul(2.0, r)) >= dmul(s, r);
}

struct Counters {
    int64_t *cnt;       // ring of 3 frontier sizes
    int64_t *pairs;     // pair count
    int64_t *flags;     // overflow flags
};

// shard / n_shards: only the recursions of internal nodes w with w % n_shards == shard
// (the owner loop of spanner.py:206-241 split over GPUs)
__global__ void k_wspd_init_f(const int2 *lr, int64_t nn, ItemF *items, int64_t cap, int64_t *cnt, int shard,
                              int n_shards, int64_t *cnt2 = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; base < nn; base += stride) {
        const int64_t w = base + lane;
        int2 c = w < nn ? lr[w] : make_int2(-1, -1);
        const bool need = c.x >= 0 && w % n_shards == shard;
        const unsigned m = __ballot_sync(0xffffffffu, need);
        if (!m) continue;
        int64_t b = 0;
        if (lane == 0) {
            b = (int64_t)atomicAdd((unsigned long long *)cnt, (unsigned long long)__popc(m));
            if (cnt2) atomicAdd((unsigned long long *)cnt2, (unsigned long long)__popc(m));
        }
        b = __shfl_sync(0xffffffffu, b, 0);
        if (need) {
            int64_t slot = b + __popc(m & lanemask_lt());
            if (slot < cap) items[slot] = ItemF{c.x, c.y};
        }
    }
}

// reference order: level 0 also records each item's owner internal node
__global__ void k_wspd_init_o(const int2 *lr, int64_t nn, ItemF *items, int32_t *own0, int64_t cap, int64_t *cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; base < nn; base += stride) {
        const int64_t w = base + lane;
        int2 c = w < nn ? lr[w] : make_int2(-1, -1);
        const bool need = c.x >= 0;
        const unsigned m = __ballot_sync(0xffffffffu, need);
        if (!m) continue;
        int64_t b = 0;
        if (lane == 0) b = (int64_t)atomicAdd((unsigned long long *)cnt, (unsigned long long)__popc(m));
        b = __shfl_sync(0xffffffffu, b, 0);
        if (need) {
            int64_t slot = b + __popc(m & lanemask_lt());
            if (slot < cap) {
                items[slot] = ItemF{c.x, c.y};
                own0[slot] = (int32_t)w;
            }
        }
    }
}

// one frontier level.  ORDER: cur / next are consecutive levels of the one
// item array (global indices base_cur + i / base_next + slot) and every item
// records its link: ~pair slot, or the index of its first child.  IPT items
// per thread and round: their loads are all in flight together (the level is
// bound by the latency of the dependent item -> geometry loads), and the
// round's appends are aggregated per CTA (two global atomics per CTA).
template <bool ORDER, int IPT = 1>
__device__ __forceinline__ void wspd_level(const ItemF *__restrict__ cur, ItemF *__restrict__ next,
                                           int64_t cap, int level, Counters k,
                                           int2 *__restrict__ out_uv, int64_t *__restrict__ links,
                                           int64_t base_cur, int64_t base_next, int64_t pair_cap,
                                           double s, const NodeGeom *__restrict__ geom,
                                           const int2 *__restrict__ lr, int64_t n_known = -1) {
    using Item = ItemF;
    int64_t n = n_known >= 0 ? n_known : *((volatile int64_t *)&k.cnt[level % 3]);
    // (level-loop launches: a previous level that overflowed left more items than the
    // buffer holds; its flag is already set.  With n_known the caller checked the level
    // fits -- and `cap` is the NEXT level's room, which in reference order is the rest of
    // the one array: clamping the current level by it would leave items unprocessed,
    // their links unwritten, without any flag)
    if (n_known < 0 && n > cap) n = cap;
    if (blockIdx.x == 0 && threadIdx.x == 0) k.cnt[(level + 2) % 3] = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * IPT;
    __shared__ int s_np[32], s_ns[32];
    __shared__ int64_t s_bp, s_bs;
    const int nw = blockDim.x >> 5;
    // block-uniform trip count
    for (int64_t bbase = (int64_t)blockIdx.x * blockDim.x * IPT; bbase < n; bbase += stride) {
        Item it[IPT];
        bool valid[IPT], ws[IPT];
        int2 c0[IPT], c1[IPT];
        NodeGeom gu[IPT], gv[IPT];
        int2 lu[IPT], lv[IPT];
#pragma unroll
        for (int q = 0; q < IPT; q++) {
            const int64_t i = bbase + q * blockDim.x + threadIdx.x;
            valid[q] = i < n;
            it[q] = valid[q] ? cur[i] : ItemF{0, 0};
        }
#pragma unroll
        for (int q = 0; q < IPT; q++) {
            // every load the items may need, issued together
            if (valid[q]) {
                gu[q] = geom[it[q].u];
                gv[q] = geom[it[q].v];
                lu[q] = lr[it[q].u];
                lv[q] = lr[it[q].v];
            }
        }
        unsigned mp[IPT], ms[IPT];
        int np = 0, ns = 0;
#pragma unroll
        for (int q = 0; q < IPT; q++) {
            ws[q] = false;
            c0[q] = c1[q] = make_int2(0, 0);
            if (valid[q]) {
                ws[q] = ws_predicate(gu[q], gv[q], s);
                if (!ws[q]) {
                    if (gu[q].dsq > gv[q].dsq) {  // spanner.py:226-230
                        c0[q] = make_int2(lu[q].x, it[q].v);
                        c1[q] = make_int2(lu[q].y, it[q].v);
                    } else {                      // spanner.py:231-235
                        c0[q] = make_int2(it[q].u, lv[q].x);
                        c1[q] = make_int2(it[q].u, lv[q].y);
                    }
                }
            }
            mp[q] = __ballot_sync(0xffffffffu, valid[q] && ws[q]);
            ms[q] = __ballot_sync(0xffffffffu, valid[q] && !ws[q]);
            np += __popc(mp[q]);
            ns += 2 * __popc(ms[q]);
        }
        if (lane == 0) {
            s_np[wid] = np;
            s_ns[wid] = ns;
        }
        __syncthreads();
        if (wid == 0) {
            // exclusive scan of the warps' counts by warp 0, then one atomic per counter
            int a = lane < nw ? s_np[lane] : 0, b = lane < nw ? s_ns[lane] : 0;
            int ia = a, ib = b;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
                if (lane >= o) {
                    ia += ya;
                    ib += yb;
                }
            }
            const int tp = __shfl_sync(0xffffffffu, ia, 31), ts = __shfl_sync(0xffffffffu, ib, 31);
            if (lane < nw) {
                s_np[lane] = ia - a;
                s_ns[lane] = ib - b;
            }
            if (lane == 0) {
                s_bp = tp ? (int64_t)atomicAdd((unsigned long long *)k.pairs, (unsigned long long)tp) : 0;
                s_bs = ts ? (int64_t)atomicAdd((unsigned long long *)&k.cnt[(level + 1) % 3], (unsigned long long)ts)
                          : 0;
            }
        }
        __syncthreads();
        int64_t bp = s_bp + s_np[wid], bs = s_bs + s_ns[wid];
        __syncthreads();  // s_* are rewritten by the next round
#pragma unroll
        for (int q = 0; q < IPT; q++) {
            const int64_t i = bbase + q * blockDim.x + threadIdx.x;
            if (valid[q] && ws[q]) {
                const int64_t slot = bp + __popc(mp[q] & lt);
                if constexpr (ORDER) links[base_cur + i] = ~slot;
                if (slot < pair_cap) {
                    out_uv[slot] = make_int2(it[q].u, it[q].v);
                } else if (slot == pair_cap) {
                    atomicOr((unsigned long long *)&k.flags[F_PAIR_OVF], 1ull);
                }
            }
            if (valid[q] && !ws[q]) {
                const int64_t slot = bs + 2 * __popc(ms[q] & lt);
                if constexpr (ORDER) links[base_cur + i] = base_next + slot;
                if (slot + 1 < cap) {
                    next[slot] = ItemF{c0[q].x, c0[q].y};      // left child
                    next[slot + 1] = ItemF{c1[q].x, c1[q].y};  // right child
                } else {
                    atomicOr((unsigned long long *)&k.flags[F_FRONT_OVF], 1ull);
                }
            }
            bp += __popc(mp[q]);
            bs += 2 * __popc(ms[q]);
        }
    }
}

__global__ void __launch_bounds__(256) k_wspd_level(const ItemF *__restrict__ cur, ItemF *__restrict__ next,
                                                    int64_t cap, int level, Counters k,
                                                    int2 *__restrict__ out_uv, int64_t pair_cap, double s,
                                                    const NodeGeom *__restrict__ geom,
                                                    const int2 *__restrict__ lr) {
    wspd_level<false>(cur, next, cap, level, k, out_uv, nullptr, 0, 0, pair_cap, s, geom, lr);
}

// all frontier levels in ONE persistent cooperative launch: a grid barrier
// per level instead of a launch per level and a host poll per batch
template <int IPT, int BT = 256, int MINB = 1>
__global__ void __launch_bounds__(BT, MINB) k_wspd_coop(ItemF *fa, ItemF *fb, int64_t cap, Counters k,
                                                   int2 *__restrict__ out_uv, int64_t pair_cap, double s,
                                                   const NodeGeom *__restrict__ geom, const int2 *__restrict__ lr,
                                                   int32_t *levels_out) {
    cg::grid_group grid = cg::this_grid();
    int level = 0;
    while (true) {
        const int64_t n = *((volatile int64_t *)&k.cnt[level % 3]);
        if (n == 0 || n > cap) break;  // done, or the last level overflowed (flag set)
        wspd_level<false, IPT>((level & 1) ? fb : fa, (level & 1) ? fa : fb, cap, level, k, out_uv, nullptr, 0, 0,
                               pair_cap, s, geom, lr, n);
        grid.sync();
        level++;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *levels_out = level;
}

// Fused order, first phase: the recursions run CTA-locally, with no grid barrier.
// The owners' recursions are independent (spanner.py:206-241 runs one DFS per
// internal node), so each CTA grabs a batch of owners from a global counter and
// advances their items as a CTA-local breadth-first frontier in shared memory,
// one __syncthreads-separated level at a time; pairs leave through one global
// atomic per CTA and round.  Frontier items that do not fit in shared memory
// spill to the global level-0 frontier (fa, counter cnt[0]) and are finished by
// the grid-wide cooperative kernel that runs next (usually on nothing).
constexpr int OW_T = 256;
constexpr int OW_CAP = 2048;    // items per shared-memory frontier buffer
constexpr int OW_BATCH = 64;    // owners grabbed per CTA at a time
__global__ void __launch_bounds__(OW_T) k_wspd_owners(const int2 *__restrict__ lr, int64_t nn, int shard,
                                                      int n_shards, const NodeGeom *__restrict__ geom, double s,
                                                      Counters k, int64_t *owner_next, int32_t *max_depth,
                                                      int2 *__restrict__ out_uv, int64_t pair_cap,
                                                      ItemF *__restrict__ spill, int64_t spill_cap) {
    __shared__ ItemF f[2][OW_CAP];
    __shared__ int s_n[2];
    __shared__ int s_np[OW_T / 32], s_ns[OW_T / 32];
    __shared__ int64_t s_bp, s_w0;
    __shared__ int s_next_base;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned lt = lanemask_lt();
    int depth_max = 0;
    for (;;) {
        if (tid == 0) s_w0 = (int64_t)atomicAdd((unsigned long long *)owner_next, (unsigned long long)OW_BATCH);
        if (tid == 0) s_n[0] = 0;
        __syncthreads();
        const int64_t w0 = s_w0;
        if (w0 >= nn) break;
        // seed: (left[w], right[w]) of the batch's internal nodes (this shard's)
        int2 c = make_int2(-1, -1);
        bool need = false;
        unsigned m = 0;
        if (tid < OW_BATCH) {
            const int64_t w = w0 + tid;
            c = w < nn ? lr[w] : make_int2(-1, -1);
            need = c.x >= 0 && w % n_shards == shard;
            m = __ballot_sync(0xffffffffu, need);
            if (lane == 0) s_np[wid] = __popc(m);
        }
        __syncthreads();
        if (tid < OW_BATCH) {
            int off = 0;
            for (int q = 0; q < wid; q++) off += s_np[q];
            if (need) f[0][off + __popc(m & lt)] = ItemF{c.x, c.y};
        }
        if (tid == 0) {
            int tot = 0;
            for (int q = 0; q < OW_BATCH / 32; q++) tot += s_np[q];
            s_n[0] = tot;
        }
        __syncthreads();
        int cur = 0, depth = 0;
        while (true) {
            const int n = s_n[cur];
            if (n == 0) break;
            depth++;
            if (tid == 0) s_n[cur ^ 1] = 0;
            __syncthreads();
            for (int base = 0; base < n; base += OW_T) {
                const int i = base + tid;
                const bool valid = i < n;
                ItemF it{0, 0};
                bool ws = false;
                int2 c0 = make_int2(0, 0), c1 = make_int2(0, 0);
                if (valid) {
                    it = f[cur][i];
                    const NodeGeom gu = geom[it.u], gv = geom[it.v];
                    const int2 lu = lr[it.u], lv = lr[it.v];
                    ws = ws_predicate(gu, gv, s);
                    if (!ws) {
                        if (gu.dsq > gv.dsq) {  // spanner.py:226-230
                            c0 = make_int2(lu.x, it.v);
                            c1 = make_int2(lu.y, it.v);
                        } else {                // spanner.py:231-235
                            c0 = make_int2(it.u, lv.x);
                            c1 = make_int2(it.u, lv.y);
                        }
                    }
                }
                const unsigned mp = __ballot_sync(0xffffffffu, valid && ws);
                const unsigned ms = __ballot_sync(0xffffffffu, valid && !ws);
                if (lane == 0) {
                    s_np[wid] = __popc(mp);
                    s_ns[wid] = 2 * __popc(ms);
                }
                __syncthreads();
                if (tid == 0) {
                    int tp = 0, ts = 0;
                    for (int w = 0; w < OW_T / 32; w++) {
                        const int a = s_np[w], b = s_ns[w];
                        s_np[w] = tp;
                        s_ns[w] = ts;
                        tp += a;
                        ts += b;
                    }
                    s_bp = tp ? (int64_t)atomicAdd((unsigned long long *)k.pairs, (unsigned long long)tp) : 0;
                    s_next_base = s_n[cur ^ 1];
                    s_n[cur ^ 1] += ts;
                }
                __syncthreads();
                const int64_t bp = s_bp + s_np[wid];
                const int bs = s_next_base + s_ns[wid];
                if (valid && ws) {
                    const int64_t slot = bp + __popc(mp & lt);
                    if (slot < pair_cap) out_uv[slot] = make_int2(it.u, it.v);
                    else if (slot == pair_cap) atomicOr((unsigned long long *)&k.flags[F_PAIR_OVF], 1ull);
                }
                if (valid && !ws) {
                    const int pos = bs + 2 * __popc(ms & lt);
                    if (pos + 1 < OW_CAP) {
                        f[cur ^ 1][pos] = ItemF{c0.x, c0.y};
                        f[cur ^ 1][pos + 1] = ItemF{c1.x, c1.y};
                    } else {
                        // the CTA's frontier is full: these two continue in the grid-wide pass
                        const int64_t g = (int64_t)atomicAdd((unsigned long long *)&k.cnt[0], 2ull);
                        if (g + 1 < spill_cap) {
                            spill[g] = ItemF{c0.x, c0.y};
                            spill[g + 1] = ItemF{c1.x, c1.y};
                        } else {
                            atomicOr((unsigned long long *)&k.flags[F_FRONT_OVF], 1ull);
                        }
                    }
                }
                __syncthreads();  // s_np / s_ns are rewritten by the next round
            }
            if (tid == 0 && s_n[cur ^ 1] > OW_CAP) s_n[cur ^ 1] = OW_CAP;  // the rest spilled
            __syncthreads();
            cur ^= 1;
        }
        depth_max = depth > depth_max ? depth : depth_max;
        __syncthreads();
    }
    if (tid == 0) atomicMax(max_depth, depth_max);
}

// Fused order, depth-first: every warp runs recursions on its own stack in
// shared memory -- pop the top 32 items, one lane each: one round of geometry
// loads, the predicate, pairs into a per-warp buffer (flushed with one global
// atomic per ~DF_PB pairs), the split items' two children pushed back -- with no
// CTA or grid barrier, so a step costs one dependent load instead of a level's
// barrier, load chain and counter atomic.
// Work moves between warps through a global queue of 32-item chunks: the owners'
// root items (left[w], right[w]) are its first chunks; a warp whose stack would
// overflow, or that sees waiting warps, appends the BOTTOM of its stack (the
// oldest, biggest sub-recursions).  A warp out of work takes a ticket (one
// atomicAdd, no retry storm) and waits on that chunk's own ready flag, which carries
// the run's epoch (set with release semantics after the chunk's items; flags of
// earlier runs never match, so nothing is cleared between runs).  The owner chunks
// are strided over the owners (their items lie roughly in node-id order, the
// biggest recursions first).  Termination: `pending` = busy warps +
// appended-but-unconsumed chunks; it only reaches 0 once nothing is left anywhere,
// and then stays 0: the warp that takes it to 0 marks every waiting ticket's flag
// with the end, and a waiting warp also checks `pending` now and then.  Warps that
// start late or never start do not matter (no co-residency needed).  The emitted pair SET is the reference's (the
// recursions are independent and each runs exactly); their order is not (the
// fused front end builds the CSR, a function of the set).
constexpr int DF_W = 8;        // warps per CTA
constexpr int DF_S = 256;      // per-warp stack ring, items (512: the L1 left beside the stacks
                               // caches less node geometry: cfg5 s = 16 kernel 0.92 vs 0.74-0.77 ms)
constexpr int DF_PB = 128;     // per-warp pair buffer
constexpr int DF_POLL = 8;     // steps between donation checks
// counters, one 128-byte line each
constexpr int DL_PUSH = 0 * 16;     // chunks appended after the owners'
constexpr int DL_TICKET = 1 * 16;   // tickets taken
constexpr int DL_PENDING = 2 * 16;  // pending - owner chunks (signed)
constexpr int DL_PAIRS = 3 * 16;    // pairs
constexpr int DL_OWNERS = 5 * 16;   // owner items (the init kernel's count)
constexpr int DL_N = 6 * 16;
__device__ __forceinline__ int64_t vld64(const int64_t *p) { return *(volatile const int64_t *)p; }
__device__ __forceinline__ int32_t ld_relaxed(const int32_t *p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int32_t v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(int32_t *p, int32_t v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct DfPool {
    ItemF *items;      // [0, n0): the owners' items; appended chunk k at (o_chunks + k) * 32
    int32_t *ready;    // per appended chunk: 2 epoch = its items are written, 2 epoch + 1 = the end
    int64_t cap_items; // capacity of items
    int64_t *ctr;
    int64_t *flags;
    int32_t epoch;     // this run's (flags of earlier runs never match: no clearing)
};

// append stack ring positions [b, b + m) (m a multiple of 32) to the queue
__device__ __forceinline__ void df_push(const ItemF *st, int b, int m, const DfPool &P, int64_t o_chunks) {
    const int lane = threadIdx.x & 31;
    const int nch = m >> 5;
    int64_t k0 = 0;
    if (lane == 0) {
        atomicAdd((unsigned long long *)&P.ctr[DL_PENDING], (unsigned long long)nch);  // before any is ready
        k0 = (int64_t)atomicAdd((unsigned long long *)&P.ctr[DL_PUSH], (unsigned long long)nch);
    }
    k0 = __shfl_sync(0xffffffffu, k0, 0);
    const int64_t cap_chunks = P.cap_items / 32 - o_chunks;
    for (int j = 0; j < nch; j++) {
        const int64_t k = k0 + j;
        if (k < cap_chunks) P.items[(o_chunks + k) * 32 + lane] = st[(b + 32 * j + lane) & (DF_S - 1)];
    }
    __syncwarp();  // orders the warp's item writes before the release stores below
    for (int j = lane; j < nch; j += 32) {
        const int64_t k = k0 + j;
        if (k < cap_chunks) st_release(&P.ready[k], 2 * P.epoch);
        else atomicOr((unsigned long long *)&P.flags[F_FRONT_OVF], 1ull);
    }
    __syncwarp();
}

__device__ __forceinline__ void df_flush(int2 *pb, int &pbn, const DfPool &P, int2 *__restrict__ out_uv,
                                         int64_t pair_cap) {
    const int lane = threadIdx.x & 31;
    if (pbn == 0) return;
    int64_t base = 0;
    if (lane == 0) base = (int64_t)atomicAdd((unsigned long long *)&P.ctr[DL_PAIRS], (unsigned long long)pbn);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int i = lane; i < pbn; i += 32) {
        const int64_t slot = base + i;
        if (slot < pair_cap) out_uv[slot] = pb[i];
        else if (slot == pair_cap) atomicOr((unsigned long long *)&P.flags[F_PAIR_OVF], 1ull);
    }
    pbn = 0;
    __syncwarp();
}

__global__ void __launch_bounds__(DF_W * 32) k_wspd_dfs(const int2 *__restrict__ lr, const NodeGeom *__restrict__ geom,
                                                        double s, const __grid_constant__ DfPool P,
                                                        int2 *__restrict__ out_uv, int64_t pair_cap) {
    __shared__ ItemF stk[DF_W][DF_S];
    __shared__ int2 pbs[DF_W][DF_PB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    ItemF *st = stk[wid];
    int2 *pb = pbs[wid];
    const int64_t n0 = P.ctr[DL_OWNERS];
    const int64_t o_chunks = (n0 + 31) >> 5;
    const int64_t cap_chunks = P.cap_items / 32 - o_chunks;
    int top = 0, bot = 0, pbn = 0, step = 0;
    while (true) {
        if (top == bot) {
            // out of work: take a ticket and wait for that chunk (or for the end)
            top = bot = 0;
            int64_t t = 0;
            if (lane == 0) t = (int64_t)atomicAdd((unsigned long long *)&P.ctr[DL_TICKET], 1ull);
            t = __shfl_sync(0xffffffffu, t, 0);
            ItemF it{-1, -1};
            bool got = true;
            if (t < o_chunks) {
                // owner chunks are strided: the owners' items lie roughly in node-id order,
                // biggest recursions (the root's spine) first, and a chunk of 32 consecutive
                // ones would hand them all to one warp
                const int64_t g = t + (int64_t)lane * o_chunks;
                if (g < n0) it = P.items[g];  // written by the init kernel
            } else {
                const int64_t k = t - o_chunks;
                int state = 0;  // 1: ready, 2: dropped (overflow), 3: the end
                int zero_dep = 0;  // 0, computed from the ready flag's value
                if (lane == 0) {
                    unsigned backoff = 32;
                    for (int poll = 0;; poll++) {
                        if (k < cap_chunks) {
                            const int32_t v = ld_relaxed(&P.ready[k]);
                            if (v == 2 * P.epoch) {
                                state = 1;
                                zero_dep = v - 2 * P.epoch;
                                break;
                            }
                            if (v == 2 * P.epoch + 1) {  // the finishing warp's broadcast
                                state = 3;
                                break;
                            }
                        } else if (vld64(&P.ctr[DL_PUSH]) > k) {
                            state = 2;
                            break;
                        }
                        // (tickets taken after the broadcast see the end here)
                        if ((poll & 7) == 7 && o_chunks + vld64(&P.ctr[DL_PENDING]) == 0) {
                            state = 3;
                            break;
                        }
                        __nanosleep(backoff);
                        backoff = backoff < 1024 ? backoff * 2 : 1024;
                    }
                }
                state = __shfl_sync(0xffffffffu, state, 0);
                zero_dep = __shfl_sync(0xffffffffu, zero_dep, 0);
                if (state == 3) {
                    got = false;
                } else if (state == 1) {
                    // the items' addresses depend on the flag value lane 0 read (an
                    // acquire load would invalidate the SM's L1 -- the geometry cache --
                    // on every poll); read through L2: never a stale L1 line
                    const ItemF *src = &P.items[(o_chunks + k) * 32 + lane + zero_dep];
                    it = ItemF{__ldcg(&src->u), __ldcg(&src->v)};
                }
            }
            if (!got) break;
            st[lane] = it;
            top = 32;
            __syncwarp();
            continue;
        }
        // one step: the top min(32, size) items, one lane each; uniform control flow
        // (lanes without an item evaluate node 0 against itself and are masked out)
        const int size = top - bot;
        const int n = size < 32 ? size : 32;
        const bool valid = lane < n;
        const ItemF it = st[(top - 1 - (valid ? lane : 0)) & (DF_S - 1)];
        __syncwarp();
        top -= n;
        const bool live = valid && it.u >= 0;
        const int u = live ? it.u : 0, v = live ? it.v : 0;
        // every field of both nodes in one round of loads (the split side's dsq would
        // otherwise be fetched only after the predicate: a second round trip)
        const double2 *gp = reinterpret_cast<const double2 *>(geom);
        const double2 u0 = __ldg(gp + 2 * u), u1 = __ldg(gp + 2 * u + 1);
        const double2 v0 = __ldg(gp + 2 * v), v1 = __ldg(gp + 2 * v + 1);
        const int2 lu = __ldg(lr + u), lv = __ldg(lr + v);
        const bool ok = ws_predicate(NodeGeom{u0.x, u0.y, u1.x, u1.y}, NodeGeom{v0.x, v0.y, v1.x, v1.y}, s);
        const bool split_u = u1.y > v1.y;  // dsq: spanner.py:226-235
        const bool ws = live && ok, sp = live && !ok;
        const unsigned mp = __ballot_sync(0xffffffffu, ws);
        const unsigned ms = __ballot_sync(0xffffffffu, sp);
        // pairs into the warp's buffer (flushed first if it could overflow)
        if (pbn + 32 > DF_PB) df_flush(pb, pbn, P, out_uv, pair_cap);
        if (ws) pb[pbn + __popc(mp & lt)] = make_int2(u, v);
        pbn += __popc(mp);
        // children: make room at the bottom first (the oldest items go to the queue)
        const int nc = 2 * __popc(ms);
        if (top - bot + nc > DF_S) {
            const int m = ((top - bot + nc - DF_S + 31) & ~31);
            df_push(st, bot, m, P, o_chunks);
            bot += m;
        }
        if (sp) {
            const int pos = top + 2 * __popc(ms & lt);
            st[pos & (DF_S - 1)] = split_u ? ItemF{lu.x, v} : ItemF{u, lv.x};
            st[(pos + 1) & (DF_S - 1)] = split_u ? ItemF{lu.y, v} : ItemF{u, lv.y};
        }
        top += nc;
        __syncwarp();
        if (top == bot) {
            // this warp's work is done: its pairs leave, then its busy unit
            df_flush(pb, pbn, P, out_uv, pair_cap);
            int64_t left = 1;
            if (lane == 0)
                left = o_chunks - 1 +
                       (int64_t)atomicAdd((unsigned long long *)&P.ctr[DL_PENDING], (unsigned long long)-1ll);
            left = __shfl_sync(0xffffffffu, left, 0);
            if (left == 0) {
                // the last work anywhere: wake every waiting ticket with the end mark
                const int64_t k0 = vld64(&P.ctr[DL_PUSH]);
                int64_t k1 = vld64(&P.ctr[DL_TICKET]) - o_chunks;
                if (k1 > cap_chunks) k1 = cap_chunks;
                for (int64_t k = k0 + lane; k < k1; k += 32) st_relaxed(&P.ready[k], 2 * P.epoch + 1);
            }
            continue;
        }
        // share with waiting warps: up to half of the stack's bottom
        if (++step % DF_POLL == 0 && top - bot >= 64) {
            int give = 0;
            if (lane == 0) {
                const int64_t waiting = vld64(&P.ctr[DL_TICKET]) - (o_chunks + vld64(&P.ctr[DL_PUSH]));
                if (waiting > 0) {
                    const int64_t most = 32 * waiting;
                    give = ((top - bot) / 2) & ~31;
                    if (give > most) give = (int)most;
                }
            }
            give = __shfl_sync(0xffffffffu, give, 0);
            if (give) {
                df_push(st, bot, give, P, o_chunks);
                bot += give;
            }
        }
    }
}

// reference order: the levels are appended to one array (level l occupies
// [starts[l], starts[l+1])), so the whole recursion forest stays for the
// ordering passes; `cap` is the array's capacity, max_levels starts' capacity
__global__ void __launch_bounds__(256) k_wspd_coop_o(ItemF *items, int64_t cap, Counters k,
                                                     int2 *__restrict__ out_uv, int64_t *__restrict__ links,
                                                     int64_t *__restrict__ starts, int64_t max_levels,
                                                     int64_t pair_cap, double s, const NodeGeom *__restrict__ geom,
                                                     const int2 *__restrict__ lr, int32_t *levels_out) {
    cg::grid_group grid = cg::this_grid();
    int level = 0;
    int64_t base = 0;
    while (true) {
        const int64_t n = *((volatile int64_t *)&k.cnt[level % 3]);
        if (n == 0) break;
        if (base + n > cap || level + 1 >= max_levels) {  // overflow (the flag is set by whoever saw it)
            if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr((unsigned long long *)&k.flags[F_FRONT_OVF], 1ull);
            break;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) starts[level] = base;
        wspd_level<true>(items + base, items + base + n, cap - (base + n), level, k, out_uv, links, base,
                         base + n, pair_cap, s, geom, lr, n);
        grid.sync();
        base += n;
        level++;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *levels_out = level;
        starts[level] = base;
    }
}

// count_pairs, bottom-up: leaves below each item (deepest level first); then
// each owner's count from its level-0 item
__global__ void __launch_bounds__(256) k_order_up(const int64_t *__restrict__ links, const int64_t *__restrict__ starts,
                                                  int levels, int64_t *__restrict__ cnt,
                                                  const int32_t *__restrict__ own0, int64_t *__restrict__ full) {
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    for (int l = levels - 1; l >= 0; l--) {
        const int64_t b = starts[l], e = starts[l + 1];
        for (int64_t i = b + tid; i < e; i += stride) {
            const int64_t ln = links[i];
            cnt[i] = ln < 0 ? 1 : cnt[ln] + cnt[ln + 1];
        }
        grid.sync();
    }
    const int64_t n0 = levels > 0 ? starts[1] : 0;
    for (int64_t i = tid; i < n0; i += stride) full[own0[i]] = cnt[i];
}

// write_pairs, top-down: an item's first pair lands at its offset; the DFS pops
// the right child first, so the right child starts at the parent's offset and
// the left child after the right child's leaves.  `cnt` is overwritten by the
// offsets level by level (each child is read by its one parent before that).
__global__ void __launch_bounds__(256) k_order_down(const int64_t *__restrict__ links,
                                                    const int64_t *__restrict__ starts, int levels,
                                                    int64_t *__restrict__ cnt, const int32_t *__restrict__ own0,
                                                    const int64_t *__restrict__ owner_off, uint32_t *__restrict__ perm) {
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n0 = levels > 0 ? starts[1] : 0;
    for (int64_t i = tid; i < n0; i += stride) cnt[i] = owner_off[own0[i]];
    grid.sync();
    for (int l = 0; l < levels; l++) {
        const int64_t b = starts[l], e = starts[l + 1];
        for (int64_t i = b + tid; i < e; i += stride) {
            const int64_t ln = links[i], off = cnt[i];
            if (ln < 0) {
                perm[off] = (uint32_t)~ln;
            } else {
                const int64_t right = cnt[ln + 1];
                cnt[ln + 1] = off;
                cnt[ln] = off + right;
            }
        }
        grid.sync();
    }
}

__global__ void k_gather_uv(const int2 *src, const uint32_t *perm, int64_t n, int2 *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

struct OwnerCount {  // the owners' counts in internal-node id order (0 for leaves)
    const int64_t *full;
    __device__ int64_t operator()(int64_t i) const { return full[i]; }
};

struct InternalFlag {
    const int2 *lr;
    __device__ int64_t operator()(int64_t i) const { return lr[i].x >= 0 ? 1 : 0; }
};

__global__ void k_compact_counts(const int2 *lr, const int64_t *full, const int64_t *excl, int64_t nn,
                                 int64_t *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn;
         i += (int64_t)gridDim.x * blockDim.x)
        if (lr[i].x >= 0) out[excl[i]] = full[i];
}

__global__ void k_uv_to_idx(const int2 *uv, const int32_t *rep, int64_t n, int64_t *idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int2 p = uv[i];
        idx[2 * i] = rep[p.x];  // WSPairList.indices = rep[node_pairs], spanner.py:296
        idx[2 * i + 1] = rep[p.y];
    }
}

}  // namespace

// WSPairList.indices = rep[node_pairs] (spanner.py:296); the fused front end
// reads the representatives itself and leaves this to a later fetch
int wspd_pair_idx(Ctx &c) {
    if (c.pair_idx_valid) return W1G_OK;
    const int64_t P = c.n_pairs;
    int64_t *idx;
    W1G_TRY(ensure(c.pair_idx, (size_t)(2 * P + 2), &idx));
    if (P) {
        k_uv_to_idx<<<grid_for(P, 256, 8u * c.sm_count), 256, 0, c.stream>>>(ptr<int2>(c.pair_uv),
                                                                             ptr<int32_t>(c.t_rep32), P, idx);
        W1G_CHECK_LAUNCH();
    }
    c.pair_idx_valid = true;
    return W1G_OK;
}

int wspd_run(Ctx &c, double s, int reference_order, int64_t *n_pairs, bool want_idx, int shard, int n_shards) {
    c.pairs_valid = false;
    const int64_t nn = c.tree_n_nodes, K = c.tree_n_points;
    *n_pairs = 0;
    c.n_pairs = 0;
    c.wspd_levels = 0;
    const int ORDER = reference_order ? 1 : 0;
    int64_t *ctr;
    W1G_TRY(ensure(c.scr[20], 8, &ctr));
    // capacity estimate (P/K ~ 6.5 + 0.95 s^2 on the benchmark sets)
    int64_t pair_cap = (int64_t)((double)K * (8.0 + 1.25 * s * s)) + 4096;
    const int64_t prev_pair_cap = (int64_t)(c.pair_uv.cap / sizeof(int2));
    if (prev_pair_cap > pair_cap) pair_cap = prev_pair_cap - 16;
    // fused: two ping-pong frontiers; reference order: one array holding every
    // level (the recursion forest has ~2P items)
    int64_t front_cap = ORDER ? 2 * pair_cap + K + 4096 : pair_cap / 2 + 2 * K + 4096;
    {
        // W1G_WSPD_TINY_CAPS=1 (tests, read per call): capacities far below the need, so the
        // overflow flags and the regrow-and-retry path run (the depth-first kernel's pool
        // still holds every owner's root item: front_cap >= 2K)
        const char *e = getenv("W1G_WSPD_TINY_CAPS");
        if (e && *e == '1') {
            pair_cap = K / 4 + 64;
            front_cap = ORDER ? 4 * pair_cap + K + 64 : 2 * K + 64;
        }
    }
    // the recursion depth is at most depth(u) + depth(v) <= 2 nn
    const int64_t max_levels = 2 * nn + 8;
    for (int attempt = 0; attempt < 8; attempt++) {
        int2 *uv;
        ItemF *fa, *fb = nullptr;
        int64_t *links = nullptr, *starts = nullptr;
        int32_t *own0 = nullptr;
        W1G_TRY(ensure(c.pair_uv, (size_t)pair_cap, &uv));
        W1G_TRY(ensure(c.scr[21], (size_t)front_cap + 8, &fa));
        if (ORDER) {
            W1G_TRY(ensure(c.scr[22], (size_t)front_cap + 8, &links));
            W1G_TRY(ensure(c.scr[23], (size_t)max_levels + 8, &starts));
            W1G_TRY(ensure(c.pair_w, (size_t)nn + 8, &own0));
        } else {
            W1G_TRY(ensure(c.scr[22], (size_t)front_cap + 8, &fb));
        }
        W1G_TRY(flags_reset(c));
        W1G_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int64_t) * 8, c.stream));
        Counters k{ctr, ctr + 4, dflags(c)};
        const unsigned gi = grid_for(nn, 256, 8u * c.sm_count);
        // fused order: the depth-first warp kernel (W1G_WSPD_DFS=0: the level-synchronous
        // phases below)
        static const bool dfs_env = [] {
            const char *e = getenv("W1G_WSPD_DFS");
            return !(e && *e == '0');
        }();
        if (!ORDER && dfs_env) {
            int64_t P = 0;
            bool ovf = false;
            if (nn > 1) {
                DfPool pool;
                pool.items = fa;
                pool.cap_items = front_cap;
                pool.flags = dflags(c);
                const size_t ready_n = (size_t)(front_cap / 32 + 2);
                const void *was = c.wspd_ready.p;
                const size_t was_cap = c.wspd_ready.cap;
                W1G_TRY(ensure(c.wspd_ready, ready_n, &pool.ready));
                // the flags carry the run's epoch: cleared only when the buffer is new or the
                // epochs wrap
                if (c.wspd_ready.p != was || c.wspd_ready.cap != was_cap || c.wspd_epoch >= (1 << 29)) {
                    W1G_CUDA(cudaMemsetAsync(pool.ready, 0, c.wspd_ready.cap, c.stream));
                    c.wspd_epoch = 0;
                }
                pool.epoch = ++c.wspd_epoch;
                W1G_TRY(ensure(c.wspd_ctr, DL_N, &pool.ctr));
                W1G_CUDA(cudaMemsetAsync(pool.ctr, 0, sizeof(int64_t) * DL_N, c.stream));
                k_wspd_init_f<<<gi, 256, 0, c.stream>>>(ptr<int2>(c.t_lr), nn, fa, front_cap, pool.ctr + DL_OWNERS,
                                                        shard, n_shards);
                W1G_CHECK_LAUNCH();
                // W1G_WSPD_DFS_CARVEOUT (tuning): the shared-memory carveout in percent (the rest
                // is L1, which caches the node geometry the steps load)
                static const int carve = [] {
                    const char *e = getenv("W1G_WSPD_DFS_CARVEOUT");
                    return e ? atoi(e) : -1;
                }();
                if (carve >= 0)
                    W1G_CUDA(cudaFuncSetAttribute(k_wspd_dfs, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
                int per = 0;
                W1G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wspd_dfs, DF_W * 32, 0));
                if (per < 1) per = 1;
                // W1G_WSPD_DFS_DIV (tuning): a further divisor of the grid (fewer resident warps
                // left waiting in the kernel's tail next to other contexts' kernels)
                static const int dfs_div_env = [] {
                    const char *e = getenv("W1G_WSPD_DFS_DIV");
                    return e ? max(1, atoi(e)) : 0;
                }();
                // small WSPDs (under ~2M expected pairs) run faster on half the grid: fewer idle
                // warps polling the queue while the deepest recursion finishes (cfg2: 76 vs 90 us;
                // s = 4 at 100k, 5.5M pairs: 217 vs 205 us the other way)
                const double est_pairs = (double)K * (8.0 + 1.25 * s * s);
                const int dfs_div = dfs_div_env ? dfs_div_env : (est_pairs < 2e6 ? 2 : 1);
                const int G = max(1, per * c.sm_count / max(1, c.coop_share) / dfs_div);
                k_wspd_dfs<<<G, DF_W * 32, 0, c.stream>>>(ptr<int2>(c.t_lr), ptr<NodeGeom>(c.t_geom), s, pool, uv,
                                                          pair_cap);
                W1G_CHECK_LAUNCH();
                W1G_TRY(to_host_small2(c, c.h_pinned + F_MISC0, pool.ctr + DL_PAIRS, sizeof(int64_t),
                                       c.h_pinned + F_PAIR_OVF, dflags(c) + F_PAIR_OVF, sizeof(int64_t) * 5));
                W1G_TRY(stream_sync(c));
                P = c.h_pinned[F_MISC0];
                if (c.h_pinned[F_FRONT_OVF]) {
                    ovf = true;
                    front_cap *= 2;
                }
            }
            if (P > pair_cap) {
                ovf = true;
                pair_cap = P + P / 8 + 1024;
            }
            if (ovf) continue;
            c.wspd_levels = 0;  // no levels: depth-first
            c.n_pairs = P;
            *n_pairs = P;
            c.pairs_valid = true;
            c.pairs_have_nodes = true;
            c.pair_idx_valid = false;
            return want_idx ? wspd_pair_idx(c) : W1G_OK;
        }
        // fused order: the owners' recursions CTA-locally first (no grid barriers), the
        // spilled remainder by the cooperative frontier below (W1G_WSPD_OWNERS=0: the
        // frontier alone, every recursion seeded at level 0)
        static const bool owners_env = [] {
            const char *e = getenv("W1G_WSPD_OWNERS");
            return !(e && *e == '0');
        }();
        if (nn > 1) {
            if (ORDER) {
                k_wspd_init_o<<<gi, 256, 0, c.stream>>>(ptr<int2>(c.t_lr), nn, fa, own0, front_cap, ctr);
            } else if (owners_env) {
                // (measured at cfg5 s = 16 as well: 5.25 ms with the CTA-local phase, 5.72 without)
                int per = 0;
                W1G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wspd_owners, OW_T, 0));
                if (per < 1) per = 1;
                k_wspd_owners<<<per * c.sm_count, OW_T, 0, c.stream>>>(
                    ptr<int2>(c.t_lr), nn, shard, n_shards, ptr<NodeGeom>(c.t_geom), s, Counters{ctr, ctr + 4, dflags(c)},
                    ctr + 5, reinterpret_cast<int32_t *>(ctr + 7), uv, pair_cap, fa, front_cap);
            } else {
                k_wspd_init_f<<<gi, 256, 0, c.stream>>>(ptr<int2>(c.t_lr), nn, fa, front_cap, ctr, shard, n_shards);
            }
            W1G_CHECK_LAUNCH();
        }
        const unsigned gl = 8u * c.sm_count;
        int level = 0;
        bool ovf = false, nn_done = false;
        const int BATCH = 8;
        if (nn > 1) {
            // persistent cooperative launch: every level, one grid barrier each
            int per_sm = 0;
            // big frontiers (many expected pairs) use every resident warp.  (wspd_level can
            // take several items per thread and round, but 4 items need 156 registers
            // against 64, which cuts the resident CTAs by the same factor: the loads in
            // flight per SM would not grow, so one item per thread is used.)
            const double est_pairs = (double)K * (8.0 + 1.25 * s * s);  // as pair_cap
            const bool big = est_pairs > (double)(16 << 20);
            // W1G_WSPD_IPT (tuning): items per thread and round of the grid-wide frontier
            static const int ipt_env = [] {
                const char *e = getenv("W1G_WSPD_IPT");
                return e ? atoi(e) : 1;
            }();
            // W1G_WSPD_BT=1024 (tuning): 1024-thread CTAs -- a quarter of the CTAs, so a quarter
            // of the per-round counter atomics and grid-barrier arrivals; measured slower at
            // cfg5 s = 16 (5.48 vs 5.26 ms), so 256 by default
            static const int bt_env = [] {
                const char *e = getenv("W1G_WSPD_BT");
                return e ? atoi(e) : 256;
            }();
            const int BT = ORDER ? 256 : (bt_env == 1024 ? 1024 : 256);
            // W1G_WSPD_MINB (tuning): minimum resident CTAs per SM the compiler must allow
            // (6 or 8: fewer registers, more warps in flight for the latency-bound rounds)
            static const int minb_env = [] {
                const char *e = getenv("W1G_WSPD_MINB");
                return e ? atoi(e) : 0;
            }();
            const void *fn = ORDER ? (const void *)k_wspd_coop_o
                           : BT == 1024 ? (const void *)k_wspd_coop<1, 1024>
                           : minb_env == 6 ? (const void *)k_wspd_coop<1, 256, 6>
                           : minb_env == 8 ? (const void *)k_wspd_coop<1, 256, 8>
                           : ipt_env == 2 ? (const void *)k_wspd_coop<2>
                           : ipt_env == 4 ? (const void *)k_wspd_coop<4>
                                          : (const void *)k_wspd_coop<1>;
            W1G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BT, 0));
            // fewer CTAs -> cheaper grid barriers while the frontier is small; a big WSPD
            // (pairs expected well above what 2 CTAs/SM cover per level) wants every
            // resident warp for its memory-latency-bound levels.  W1G_COOP_PER_SM overrides.
            {
                const char *e = getenv("W1G_COOP_PER_SM");
                const int cap = e ? atoi(e) : (big ? 8 : 2);
                if (per_sm > cap) per_sm = cap;
            }
            if (ORDER && per_sm < 1) {
                set_error("WSPD (reference order): cooperative launch unavailable");
                return W1G_ECUDA;
            }
            static const bool no_coop = [] {  // W1G_NO_COOP=1: one launch per level (measurement)
                const char *e = getenv("W1G_NO_COOP");
                return e && *e == '1';
            }();
            if (per_sm >= 1 && !((no_coop || c.no_coop) && !ORDER)) {
                const int G = max(1, per_sm * c.sm_count / max(1, c.coop_share));
                int32_t *lv = reinterpret_cast<int32_t *>(ctr + 6);
                NodeGeom *geom = ptr<NodeGeom>(c.t_geom);
                int2 *lr = ptr<int2>(c.t_lr);
                int2 *uvp = uv;
                ItemF *fap = fa, *fbp = fb;
                int64_t fc = front_cap, pc = pair_cap, ml = max_levels;
                double sv = s;
                if (ORDER) {
                    void *args[] = {&fap, &fc, &k, &uvp, &links, &starts, &ml, &pc, &sv, &geom, &lr, &lv};
                    W1G_CUDA(cudaLaunchCooperativeKernel(fn, G, 256, args, 0, c.stream));
                } else {
                    void *args[] = {&fap, &fbp, &fc, &k, &uvp, &pc, &sv, &geom, &lr, &lv};
                    W1G_CUDA(cudaLaunchCooperativeKernel(fn, G, BT, args, 0, c.stream));
                }
                W1G_CHECK_LAUNCH();
                W1G_TRY(to_host_small(c, c.h_pinned + F_MISC0, ctr, sizeof(int64_t) * 8));
                W1G_TRY(to_host_small(c, c.h_pinned + F_PAIR_OVF, dflags(c) + F_PAIR_OVF, sizeof(int64_t) * 5));
                W1G_TRY(stream_sync(c));
                level = (int)(c.h_pinned[F_MISC0 + 6] & 0x7fffffff);
                const int64_t live = c.h_pinned[F_MISC0 + level % 3];
                // levels (diagnostics): the CTA-local owners' deepest recursion + the grid-wide rest
                const int owner_depth = ORDER ? 0 : (int)(c.h_pinned[F_MISC0 + 7] & 0x7fffffff);
                if (c.h_pinned[F_FRONT_OVF] || (!ORDER && live > front_cap)) {
                    ovf = true;
                    front_cap = front_cap * 2 + (live > front_cap ? live : 0);
                }
                nn_done = true;
                if (!ORDER && !ovf) level += owner_depth;  // read after the overflow check
            }
        }
        while (nn > 1 && !nn_done) {
            for (int b = 0; b < BATCH; b++, level++) {
                ItemF *cur = (level & 1) ? fb : fa, *nxt = (level & 1) ? fa : fb;
                k_wspd_level<<<gl, 256, 0, c.stream>>>(cur, nxt, front_cap, level, k, uv, pair_cap, s,
                                                       ptr<NodeGeom>(c.t_geom), ptr<int2>(c.t_lr));
                W1G_CHECK_LAUNCH();
            }
            W1G_TRY(to_host_small(c, c.h_pinned + F_MISC0, ctr, sizeof(int64_t) * 8));
            W1G_TRY(to_host_small(c, c.h_pinned + F_PAIR_OVF, dflags(c) + F_PAIR_OVF, sizeof(int64_t) * 5));
            W1G_TRY(stream_sync(c));
            const int64_t live = c.h_pinned[F_MISC0 + level % 3];
            if (c.h_pinned[F_FRONT_OVF] || live > front_cap) {
                ovf = true;
                front_cap = front_cap * 2 + (live > front_cap ? live : 0);
                break;
            }
            if (live == 0) break;
            if (level > 4 * (int)nn + 64) {
                set_error("WSPD did not terminate");
                return W1G_ECUDA;
            }
        }
        // the ctr mirror sits at h_pinned[F_MISC0 .. F_MISC0+7]; pairs at +4
        const int64_t P = nn > 1 ? c.h_pinned[F_MISC0 + 4] : 0;
        if (!ovf && P > pair_cap) {
            ovf = true;
            pair_cap = P + P / 8 + 1024;
        }
        if (ovf) continue;
        c.wspd_levels = level;
        c.n_pairs = P;
        *n_pairs = P;
        if (ORDER) {
            if (P > 0xffffffffll) {
                set_error("too many pairs to order");
                return W1G_EINVAL;
            }
            // count_pairs (bottom-up leaf counts), build_wspd's offsets (a scan over the
            // owners in id order) and write_pairs' layout (top-down offsets)
            auto coop_grid = [&](const void *fn) {
                int per = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, 0);
                return (per > 2 ? 2 : (per < 1 ? 1 : per)) * c.sm_count;
            };
            int64_t *cnt, *full, *excl, *out;
            uint32_t *perm;
            int2 *uv2;
            W1G_TRY(ensure(c.scr[0], (size_t)front_cap + 8, &cnt));
            W1G_TRY(ensure(c.scr[6], nn + 1, &full));
            W1G_TRY(ensure(c.scr[3], nn + 1, &excl));
            W1G_TRY(ensure(c.pair_counts, nn / 2 + 1, &out));
            W1G_TRY(ensure(c.scr[2], P + 1, &perm));
            W1G_CUDA(cudaMemsetAsync(full, 0, sizeof(int64_t) * (nn + 1), c.stream));
            if (nn > 1 && level > 0) {
                int lv = level;
                void *up[] = {&links, &starts, &lv, &cnt, &own0, &full};
                W1G_CUDA(cudaLaunchCooperativeKernel((const void *)k_order_up, coop_grid((const void *)k_order_up), 256,
                                                     up, 0, c.stream));
                W1G_CHECK_LAUNCH();
            }
            W1G_TRY(scan_i64(c, OwnerCount{full}, nn, excl, nullptr));
            if (nn > 1 && level > 0) {
                int lv = level;
                void *down[] = {&links, &starts, &lv, &cnt, &own0, &excl, &perm};
                W1G_CUDA(cudaLaunchCooperativeKernel((const void *)k_order_down, coop_grid((const void *)k_order_down),
                                                     256, down, 0, c.stream));
                W1G_CHECK_LAUNCH();
            }
            const unsigned gp = grid_for(P, 256, 8u * c.sm_count);
            W1G_TRY(ensure(c.scr[5], P + 1, &uv2));
            if (P) {
                k_gather_uv<<<gp, 256, 0, c.stream>>>(uv, perm, P, uv2);
                W1G_CHECK_LAUNCH();
                W1G_CUDA(cudaMemcpyAsync(uv, uv2, sizeof(int2) * P, cudaMemcpyDeviceToDevice, c.stream));
            }
            // count_pairs: pairs per internal node, internal nodes in id order
            int64_t *iexcl;
            W1G_TRY(ensure(c.scr[4], nn + 1, &iexcl));
            W1G_TRY(scan_i64(c, InternalFlag{ptr<int2>(c.t_lr)}, nn, iexcl, nullptr));
            k_compact_counts<<<grid_for(nn, 256, 8u * c.sm_count), 256, 0, c.stream>>>(ptr<int2>(c.t_lr), full,
                                                                                       iexcl, nn, out);
            W1G_CHECK_LAUNCH();
        }
        c.pairs_valid = true;
        c.pairs_have_nodes = true;
        c.pair_idx_valid = false;
        return want_idx ? wspd_pair_idx(c) : W1G_OK;
    }
    set_error("WSPD buffers kept overflowing");
    return W1G_ENOMEM;
}

}  // namespace w1g
