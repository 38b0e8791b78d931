// wspd.cu -- well-separated pair decomposition (spanner.py:176-307) on device.
//
// The reference runs one DFS per internal node w from (left[w], right[w]):
// a pair (u, v) is emitted when _ws_predicate holds, otherwise the side with
// the larger bbox diagonal (_diag_sq) is replaced by its two children.  The
// emitted SET is a function of the tree and s only, so on device all
// recursions advance together as one breadth-first frontier of (u, v) items,
// one level per launch: every item evaluates the predicate with the
// reference's exact fp64 operation order (per-node centres/radii precomputed
// in tree.cu with the same operations), and warp-aggregated atomics append
// either a pair or two children.  Levels run in batches; the host polls the
// frontier size between batches and regrows buffers on overflow.
//
// reference_order = 1 additionally carries (owner w, DFS path bits) and sorts
// the pairs by (w, DFS pop order) -- the reference's exact output layout
// (owner ascending, right child popped first, spanner.py:226-236) -- and
// produces count_pairs' per-node counts.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace w1g {

namespace {

struct ItemF {  // fused path: only the node pair
    int32_t u, v;
};
struct ItemO {  // reference-order path
    int32_t u, v, w, pad;
    uint64_t p0, p1;  // left-aligned path bits, 1 = right child
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

__global__ void k_wspd_init_f(const int2 *lr, int64_t nn, ItemF *items, int64_t cap, int64_t *cnt) {
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
            if (slot < cap) items[slot] = ItemF{c.x, c.y};
        }
    }
}

__global__ void k_wspd_init_o(const int2 *lr, int64_t nn, ItemO *items, int64_t cap, int64_t *cnt) {
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
            if (slot < cap) items[slot] = ItemO{c.x, c.y, (int32_t)w, 0, 0ull, 0ull};
        }
    }
}

template <bool ORDER>
struct ItemT;
template <>
struct ItemT<false> {
    using T = ItemF;
};
template <>
struct ItemT<true> {
    using T = ItemO;
};

template <bool ORDER>
__device__ __forceinline__ void wspd_level(const typename ItemT<ORDER>::T *__restrict__ cur,
                                           typename ItemT<ORDER>::T *__restrict__ next,
                                           int64_t cap, int level, Counters k,
                                           int2 *__restrict__ out_uv, int32_t *__restrict__ out_w,
                                           uint64_t *__restrict__ out_p0,
                                           uint64_t *__restrict__ out_p1, int64_t pair_cap,
                                           double s, const NodeGeom *__restrict__ geom,
                                           const int2 *__restrict__ lr, int64_t n_known = -1) {
    using Item = typename ItemT<ORDER>::T;
    int64_t n = n_known >= 0 ? n_known : *((volatile int64_t *)&k.cnt[level % 3]);
    if (n > cap) n = cap;  // previous level overflowed: its flag is already set
    if (blockIdx.x == 0 && threadIdx.x == 0) k.cnt[(level + 2) % 3] = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    __shared__ int s_np[8], s_ns[8];
    __shared__ int64_t s_bp, s_bs;
    // block-uniform trip count: appends are aggregated per CTA (two global
    // atomics per CTA and round instead of two per warp)
    for (int64_t bbase = (int64_t)blockIdx.x * blockDim.x; bbase < n; bbase += stride) {
        const int64_t i = bbase + threadIdx.x;
        const bool valid = i < n;
        Item it;
        bool ws = false;
        int2 c0 = make_int2(0, 0), c1 = make_int2(0, 0);
        if (valid) {
            it = cur[i];
            // every load the item may need, issued together
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
        if (threadIdx.x == 0) {
            int tp = 0, ts = 0;
            for (int w = 0; w < 8; w++) {
                const int a = s_np[w], b = s_ns[w];
                s_np[w] = tp;
                s_ns[w] = ts;
                tp += a;
                ts += b;
            }
            s_bp = tp ? (int64_t)atomicAdd((unsigned long long *)k.pairs, (unsigned long long)tp) : 0;
            s_bs = ts ? (int64_t)atomicAdd((unsigned long long *)&k.cnt[(level + 1) % 3], (unsigned long long)ts) : 0;
        }
        __syncthreads();
        const int64_t bp = s_bp + s_np[wid], bs = s_bs + s_ns[wid];
        __syncthreads();  // s_* are rewritten by the next round
        if (valid && ws) {
            const int64_t slot = bp + __popc(mp & lt);
            if (slot < pair_cap) {
                out_uv[slot] = make_int2(it.u, it.v);
                if constexpr (ORDER) {
                    out_w[slot] = it.w;
                    out_p0[slot] = it.p0;
                    out_p1[slot] = it.p1;
                }
            } else if (slot == pair_cap) {
                atomicOr((unsigned long long *)&k.flags[F_PAIR_OVF], 1ull);
            }
        }
        if (valid && !ws) {
            const int64_t slot = bs + 2 * __popc(ms & lt);
            if (slot + 1 < cap) {
                if constexpr (ORDER) {
                    uint64_t q0 = it.p0, q1 = it.p1;
                    if (level < 64) q0 |= 1ull << (63 - level);
                    else if (level < 128) q1 |= 1ull << (127 - level);
                    else atomicOr((unsigned long long *)&k.flags[F_PATH_OVF], 1ull);
                    next[slot] = ItemO{c0.x, c0.y, it.w, 0, it.p0, it.p1};  // left child: bit 0
                    next[slot + 1] = ItemO{c1.x, c1.y, it.w, 0, q0, q1};     // right child: bit 1
                } else {
                    next[slot] = ItemF{c0.x, c0.y};
                    next[slot + 1] = ItemF{c1.x, c1.y};
                }
            } else {
                atomicOr((unsigned long long *)&k.flags[F_FRONT_OVF], 1ull);
            }
        }
    }
}

template <bool ORDER>
__global__ void __launch_bounds__(256) k_wspd_level(const typename ItemT<ORDER>::T *__restrict__ cur,
                                                    typename ItemT<ORDER>::T *__restrict__ next,
                                                    int64_t cap, int level, Counters k,
                                                    int2 *__restrict__ out_uv, int32_t *__restrict__ out_w,
                                                    uint64_t *__restrict__ out_p0,
                                                    uint64_t *__restrict__ out_p1, int64_t pair_cap,
                                                    double s, const NodeGeom *__restrict__ geom,
                                                    const int2 *__restrict__ lr) {
    wspd_level<ORDER>(cur, next, cap, level, k, out_uv, out_w, out_p0, out_p1, pair_cap, s, geom, lr);
}

// all frontier levels in ONE persistent cooperative launch: a grid barrier
// per level instead of a launch per level and a host poll per batch
template <bool ORDER>
__global__ void __launch_bounds__(256) k_wspd_coop(typename ItemT<ORDER>::T *fa, typename ItemT<ORDER>::T *fb,
                                                   int64_t cap, Counters k, int2 *__restrict__ out_uv,
                                                   int32_t *__restrict__ out_w, uint64_t *__restrict__ out_p0,
                                                   uint64_t *__restrict__ out_p1, int64_t pair_cap, double s,
                                                   const NodeGeom *__restrict__ geom, const int2 *__restrict__ lr,
                                                   int32_t *levels_out) {
    cg::grid_group grid = cg::this_grid();
    int level = 0;
    while (true) {
        const int64_t n = *((volatile int64_t *)&k.cnt[level % 3]);
        if (n == 0 || n > cap) break;  // done, or the last level overflowed (flag set)
        wspd_level<ORDER>((level & 1) ? fb : fa, (level & 1) ? fa : fb, cap, level, k, out_uv, out_w, out_p0,
                          out_p1, pair_cap, s, geom, lr, n);
        grid.sync();
        level++;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *levels_out = level;
}

__global__ void k_order_keys(const int32_t *w, const uint64_t *p0, const uint64_t *p1, int64_t n,
                             uint64_t *k0, uint64_t *k1, uint64_t *k2, uint32_t *vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        // DFS pop order = descending path bits -> ascending complement
        k0[i] = ~p1[i];
        k1[i] = ~p0[i];
        k2[i] = (uint64_t)(uint32_t)w[i];
        vals[i] = (uint32_t)i;
    }
}

__global__ void k_gather_uv(const int2 *src, const uint32_t *perm, int64_t n, int2 *dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

__global__ void k_count_owner(const int32_t *w, int64_t n, int64_t *counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long *)&counts[w[i]], 1ull);
}

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

int wspd_run(Ctx &c, double s, int reference_order, int64_t *n_pairs, bool want_idx) {
    c.pairs_valid = false;
    const int64_t nn = c.tree_n_nodes, K = c.tree_n_points;
    *n_pairs = 0;
    c.n_pairs = 0;
    c.wspd_levels = 0;
    const int ORDER = reference_order ? 1 : 0;
    const size_t isz = ORDER ? sizeof(ItemO) : sizeof(ItemF);
    int64_t *ctr;
    W1G_TRY(ensure(c.scr[20], 8, &ctr));
    // capacity estimate (P/K ~ 6.5 + 0.95 s^2 on the benchmark sets)
    int64_t pair_cap = (int64_t)((double)K * (8.0 + 1.25 * s * s)) + 4096;
    int64_t front_cap = pair_cap / 2 + 2 * K + 4096;
    const int64_t prev_pair_cap = (int64_t)(c.pair_uv.cap / sizeof(int2));
    if (prev_pair_cap > pair_cap) pair_cap = prev_pair_cap - 16;
    for (int attempt = 0; attempt < 8; attempt++) {
        int2 *uv;
        int32_t *w = nullptr;
        uint64_t *p0 = nullptr, *p1 = nullptr;
        void *fa, *fb;
        W1G_TRY(ensure(c.pair_uv, (size_t)pair_cap, &uv));
        if (ORDER) {
            W1G_TRY(ensure(c.pair_w, (size_t)pair_cap, &w));
            W1G_TRY(ensure(c.pair_path, (size_t)pair_cap * 2, &p0));
            p1 = p0 + pair_cap;
        }
        W1G_TRY(ensure_bytes(c.scr[21], (size_t)front_cap * isz + 64));
        W1G_TRY(ensure_bytes(c.scr[22], (size_t)front_cap * isz + 64));
        fa = c.scr[21].p;
        fb = c.scr[22].p;
        W1G_TRY(flags_reset(c));
        W1G_CUDA(cudaMemsetAsync(ctr, 0, sizeof(int64_t) * 8, c.stream));
        Counters k{ctr, ctr + 4, dflags(c)};
        const unsigned gi = grid_for(nn, 256, 8u * c.sm_count);
        if (nn > 1) {
            if (ORDER)
                k_wspd_init_o<<<gi, 256, 0, c.stream>>>(ptr<int2>(c.t_lr), nn, (ItemO *)fa, front_cap, ctr);
            else
                k_wspd_init_f<<<gi, 256, 0, c.stream>>>(ptr<int2>(c.t_lr), nn, (ItemF *)fa, front_cap, ctr);
            W1G_CHECK_LAUNCH();
        }
        const unsigned gl = 8u * c.sm_count;
        int level = 0;
        bool ovf = false, nn_done = false;
        const int BATCH = 8;
        if (nn > 1) {
            // persistent cooperative launch: every level, one grid barrier each
            int per_sm = 0;
            const void *fn = ORDER ? (const void *)k_wspd_coop<true> : (const void *)k_wspd_coop<false>;
            W1G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
            // fewer CTAs -> cheaper grid barriers; W1G_COOP_PER_SM overrides (tuning)
            {
                const char *e = getenv("W1G_COOP_PER_SM");
                const int cap = e ? atoi(e) : 2;
                if (per_sm > cap) per_sm = cap;
            }
            if (per_sm >= 1) {
                const int G = per_sm * c.sm_count;
                int32_t *lv = reinterpret_cast<int32_t *>(ctr + 6);
                NodeGeom *geom = ptr<NodeGeom>(c.t_geom);
                int2 *lr = ptr<int2>(c.t_lr);
                int2 *uvp = uv;
                int32_t *wp = w;
                uint64_t *p0p = p0, *p1p = p1;
                void *fap = fa, *fbp = fb;
                int64_t fc = front_cap, pc = pair_cap;
                double sv = s;
                void *args[] = {&fap, &fbp, &fc, &k, &uvp, &wp, &p0p, &p1p, &pc, &sv, &geom, &lr, &lv};
                W1G_CUDA(cudaLaunchCooperativeKernel(fn, G, 256, args, 0, c.stream));
                W1G_CHECK_LAUNCH();
                W1G_CUDA(cudaMemcpyAsync(c.h_pinned + F_MISC0, ctr, sizeof(int64_t) * 8, cudaMemcpyDeviceToHost, c.stream));
                W1G_CUDA(cudaMemcpyAsync(c.h_pinned + F_PAIR_OVF, dflags(c) + F_PAIR_OVF, sizeof(int64_t) * 5,
                                         cudaMemcpyDeviceToHost, c.stream));
                W1G_TRY(stream_sync(c));
                level = (int)(c.h_pinned[F_MISC0 + 6] & 0x7fffffff);
                const int64_t live = c.h_pinned[F_MISC0 + level % 3];
                if (c.h_pinned[F_FRONT_OVF] || live > front_cap) {
                    ovf = true;
                    front_cap = front_cap * 2 + (live > front_cap ? live : 0);
                }
                nn_done = true;
            }
        }
        while (nn > 1 && !nn_done) {
            for (int b = 0; b < BATCH; b++, level++) {
                void *cur = (level & 1) ? fb : fa, *nxt = (level & 1) ? fa : fb;
                if (ORDER)
                    k_wspd_level<true><<<gl, 256, 0, c.stream>>>((const ItemO *)cur, (ItemO *)nxt, front_cap, level, k,
                                                                uv, w, p0, p1, pair_cap, s,
                                                                ptr<NodeGeom>(c.t_geom), ptr<int2>(c.t_lr));
                else
                    k_wspd_level<false><<<gl, 256, 0, c.stream>>>((const ItemF *)cur, (ItemF *)nxt, front_cap, level, k,
                                                                 uv, nullptr, nullptr, nullptr, pair_cap, s,
                                                                 ptr<NodeGeom>(c.t_geom), ptr<int2>(c.t_lr));
                W1G_CHECK_LAUNCH();
            }
            W1G_CUDA(cudaMemcpyAsync(c.h_pinned + F_MISC0, ctr, sizeof(int64_t) * 8, cudaMemcpyDeviceToHost, c.stream));
            W1G_CUDA(cudaMemcpyAsync(c.h_pinned + F_PAIR_OVF, dflags(c) + F_PAIR_OVF, sizeof(int64_t) * 5,
                                     cudaMemcpyDeviceToHost, c.stream));
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
        if (ORDER && c.h_pinned[F_PATH_OVF]) {
            set_error("WSPD recursion deeper than 128 levels: the reference pair order is not "
                      "representable (use reference_order=0)");
            return W1G_EINVAL;
        }
        c.wspd_levels = level;
        c.n_pairs = P;
        *n_pairs = P;
        if (ORDER) {
            if (P > 0xffffffffll) {
                set_error("too many pairs to order");
                return W1G_EINVAL;
            }
            uint64_t *k0, *k1, *k2;
            uint32_t *vals;
            int2 *uv2;
            W1G_TRY(ensure(c.scr[0], P, &k0));
            W1G_TRY(ensure(c.scr[1], P, &k1));
            W1G_TRY(ensure(c.scr[4], P, &k2));
            W1G_TRY(ensure(c.scr[2], P, &vals));
            const unsigned gp = grid_for(P, 256, 8u * c.sm_count);
            k_order_keys<<<gp, 256, 0, c.stream>>>(w, p0, p1, P, k0, k1, k2, vals);
            W1G_CHECK_LAUNCH();
            uint64_t *keys[3] = {k0, k1, k2};
            W1G_TRY(radix_sort(c, keys, 3, vals, P, 32));
            W1G_TRY(ensure(c.scr[5], P, &uv2));
            k_gather_uv<<<gp, 256, 0, c.stream>>>(uv, vals, P, uv2);
            W1G_CHECK_LAUNCH();
            W1G_CUDA(cudaMemcpyAsync(uv, uv2, sizeof(int2) * P, cudaMemcpyDeviceToDevice, c.stream));
            // count_pairs: pairs per internal node, internal nodes in id order
            int64_t *full, *excl, *out;
            W1G_TRY(ensure(c.scr[6], nn + 1, &full));
            W1G_TRY(ensure(c.scr[3], nn + 1, &excl));
            W1G_TRY(ensure(c.pair_counts, nn / 2 + 1, &out));
            W1G_CUDA(cudaMemsetAsync(full, 0, sizeof(int64_t) * (nn + 1), c.stream));
            k_count_owner<<<gp, 256, 0, c.stream>>>(w, P, full);
            W1G_CHECK_LAUNCH();
            W1G_TRY(scan_i64(c, InternalFlag{ptr<int2>(c.t_lr)}, nn, excl, nullptr));
            k_compact_counts<<<grid_for(nn, 256, 8u * c.sm_count), 256, 0, c.stream>>>(ptr<int2>(c.t_lr), full,
                                                                                       excl, nn, out);
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
