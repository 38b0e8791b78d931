// tree.cu -- the reference's fair split tree (spanner.py:96-159) on device.
//
// The tree is a function of point SETS only: every node's tight bbox, axis
// (x iff ext_x >= ext_y), fp64 midpoint 0.5*(lo+hi), the "coord <= mid" rule
// with the "coord < max" fallback (spanner.py:139-144), preorder ids
// (left = id+1, right = id + 2*|left|) and the representative
// (lexicographic-min point).  So instead of the reference's DFS with stable
// partitions we build it level-synchronously over all segments at once:
//
//  * two presorted index lists per segment: X-list by (x, y) and Y-list by
//    (y, x); both hold the same point set in the same position range;
//  * bbox = first/last of each list (O(1)); rep = first of the X-list;
//  * the split along the chosen axis is a prefix of that axis' list, found
//    by a warp-cooperative 32-ary search (one warp per segment); only the
//    other list is stably partitioned (flags -> device scan -> scatter);
//  * leaf children are finalised immediately, internal children become the
//    next level's segments.
// Levels run in batches without host synchronisation (kernels of levels past
// the last one exit at once); the host polls the live-segment count between
// batches.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace w1g {

namespace {

struct Seg {
    int32_t lo, hi, nid, pad;
};
struct SegInfo {
    double thr;
    int32_t lo, hi, nl, cl, cr;
    int8_t axis, strict, pad0, pad1;
};

// segments of at most LOCAL_MAX points leave the global level loop and are
// finished inside one CTA (k_tree_local)
constexpr int LOCAL_MAX = 2048;
constexpr int LT = 1024;                // threads of the shared-memory subtree kernel
constexpr int LPT = LOCAL_MAX / LT;     // list positions per thread

struct TreeOut {
    int64_t *left, *right, *rep, *size;
    double4 *bbox;
    NodeGeom *geom;
    int2 *lr;
    int32_t *rep32;
};

__device__ __forceinline__ void write_node(const TreeOut &o, int64_t nid, double xmin, double ymin,
                                           double xmax, double ymax, int64_t rep, int64_t size, int64_t l,
                                           int64_t r) {
    o.left[nid] = l;
    o.right[nid] = r;
    o.bbox[nid] = make_double4(xmin, ymin, xmax, ymax);
    o.rep[nid] = rep;
    o.size[nid] = size;
    // per-node terms of _ws_predicate / _diag_sq, spanner.py:178-194
    const double w = dsub(xmax, xmin), h = dsub(ymax, ymin);
    const double dsq = dadd(dmul(w, w), dmul(h, h));
    NodeGeom g;
    g.cx = dmul(0.5, dadd(xmin, xmax));
    g.cy = dmul(0.5, dadd(ymin, ymax));
    g.r = dmul(0.5, dsqrt(dsq));
    g.dsq = dsq;
    o.geom[nid] = g;
    o.lr[nid] = make_int2((int)l, (int)r);
    o.rep32[nid] = (int32_t)rep;
}

__global__ void k_presort_keys(const double2 *pts, int64_t n, uint64_t *xl0, uint64_t *xl1,
                               uint64_t *yl0, uint64_t *yl1, uint32_t *vx, uint32_t *vy) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = pts[i];
        uint64_t kx = dkey(p.x), ky = dkey(p.y);
        xl0[i] = ky;  // X-list: (x, y) lexicographic, least significant word first
        xl1[i] = kx;
        yl0[i] = kx;  // Y-list: (y, x)
        yl1[i] = ky;
        vx[i] = (uint32_t)i;
        vy[i] = (uint32_t)i;
    }
}

__global__ void k_tree_init(int64_t n, Seg *seg, int32_t *pos_seg, int32_t *cnt, const double2 *pts,
                            const uint32_t *xl, TreeOut o, Seg *local, int32_t *local_cnt,
                            const uint32_t *yl = nullptr, double2 *xc = nullptr, double2 *yc = nullptr) {
    const bool global_root = n > LOCAL_MAX;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        pos_seg[i] = global_root ? 0 : -1;
        if (xc) {  // inline coordinates for the cooperative level loop
            xc[i] = pts[xl[i]];
            yc[i] = pts[yl[i]];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        cnt[0] = 0;
        *local_cnt = 0;
        if (n == 1) {
            const double2 p = pts[xl[0]];
            write_node(o, 0, p.x, p.y, p.x, p.y, xl[0], 1, -1, -1);
        } else if (global_root) {
            seg[0] = Seg{0, (int32_t)n, 0, 0};
            cnt[0] = 1;
        } else {
            local[0] = Seg{0, (int32_t)n, 0, 0};  // the whole tree fits one CTA
            *local_cnt = 1;
        }
    }
}

__device__ __forceinline__ double coord(const double2 *pts, uint32_t i, int axis) {
    const double2 p = pts[i];
    return axis ? p.y : p.x;
}

// warp-cooperative count of the prefix of sorted list[lo, hi) whose
// coordinate satisfies `c <= t` (strict = 0) or `c < t` (strict = 1)
__device__ int warp_prefix_count(const double2 *pts, const uint32_t *list, int lo, int hi, int axis,
                                 double t, int strict) {
    const int lane = threadIdx.x & 31;
    int a = lo, b = hi;  // all < a satisfy, all >= b fail
    while (b - a > 32) {
        const int step = (b - a + 31) >> 5;
        const int p = a + lane * step;
        bool ok = false;
        if (p < b) {
            const double c = coord(pts, list[p], axis);
            ok = strict ? (c < t) : (c <= t);
        }
        const int k = __popc(__ballot_sync(0xffffffffu, ok));
        const int na = k ? a + (k - 1) * step + 1 : a;
        const int nb = k < 32 ? min(b, a + k * step) : b;
        a = na;
        b = nb;
    }
    const int p = a + lane;
    bool ok = false;
    if (p < b) {
        const double c = coord(pts, list[p], axis);
        ok = strict ? (c < t) : (c <= t);
    }
    return a + __popc(__ballot_sync(0xffffffffu, ok)) - lo;
}

// the same search on a list that carries its points' coordinates inline (one
// dependent load per step instead of two)
__device__ int warp_prefix_count_c(const double2 *list_c, int lo, int hi, int axis, double t, int strict) {
    const int lane = threadIdx.x & 31;
    int a = lo, b = hi;
    while (b - a > 32) {
        const int step = (b - a + 31) >> 5;
        const int p = a + lane * step;
        bool ok = false;
        if (p < b) {
            const double2 q = list_c[p];
            const double c = axis ? q.y : q.x;
            ok = strict ? (c < t) : (c <= t);
        }
        const int k = __popc(__ballot_sync(0xffffffffu, ok));
        const int na = k ? a + (k - 1) * step + 1 : a;
        const int nb = k < 32 ? min(b, a + k * step) : b;
        a = na;
        b = nb;
    }
    const int p = a + lane;
    bool ok = false;
    if (p < b) {
        const double2 q = list_c[p];
        const double c = axis ? q.y : q.x;
        ok = strict ? (c < t) : (c <= t);
    }
    return a + __popc(__ballot_sync(0xffffffffu, ok)) - lo;
}

// one warp per segment: bbox, rep, axis, split point, children (spanner.py:124-148)
// xc / yc (optional): the lists' point coordinates inline, aligned with xl / yl
__device__ __forceinline__ void tree_segment(int s, const double2 *__restrict__ pts,
                                             const uint32_t *__restrict__ xl,
                                             const uint32_t *__restrict__ yl, const Seg *__restrict__ seg,
                                             int32_t *cnt_next, Seg *seg_next, SegInfo *info,
                                             const TreeOut &o, int64_t *flags, Seg *local,
                                             int32_t *local_cnt, int parity_next,
                                             const double2 *__restrict__ xc = nullptr,
                                             const double2 *__restrict__ yc = nullptr) {
    const int lane = threadIdx.x & 31;
    {
        const Seg sg = seg[s];
        const int lo = sg.lo, hi = sg.hi, n = hi - lo;
        const uint32_t r0 = xl[lo];
        double xmin, xmax, ymin, ymax;
        if (xc) {
            xmin = xc[lo].x;
            xmax = xc[hi - 1].x;
            ymin = yc[lo].y;
            ymax = yc[hi - 1].y;
        } else {
            xmin = pts[r0].x;
            xmax = pts[xl[hi - 1]].x;
            ymin = pts[yl[lo]].y;
            ymax = pts[yl[hi - 1]].y;
        }
        const double ext_x = dsub(xmax, xmin), ext_y = dsub(ymax, ymin);
        SegInfo in{};
        in.lo = lo;
        in.hi = hi;
        in.cl = in.cr = -1;
        if (ext_x == 0.0 && ext_y == 0.0) {
            // spanner.py:134-135; every position keeps its place and is retired
            if (lane == 0) {
                atomicOr((unsigned long long *)&flags[F_DUP], 1ull);
                write_node(o, sg.nid, xmin, ymin, xmax, ymax, r0, n, -1, -1);
                in.nl = n;
                in.thr = INFINITY;
                info[s] = in;
            }
            return;
        }
        const int axis = ext_x >= ext_y ? 0 : 1;
        const uint32_t *al = axis ? yl : xl;
        const double amin = axis ? ymin : xmin, amax = axis ? ymax : xmax;
        const double mid = dmul(0.5, dadd(amin, amax));
        const double2 *alc = axis ? yc : xc;
        int nl = xc ? warp_prefix_count_c(alc, lo, hi, axis, mid, 0) : warp_prefix_count(pts, al, lo, hi, axis, mid, 0);
        int strict = 0;
        double thr = mid;
        if (nl == 0 || nl == n) {
            strict = 1;  // split off the max-attaining points instead
            thr = amax;
            nl = xc ? warp_prefix_count_c(alc, lo, hi, axis, amax, 1) : warp_prefix_count(pts, al, lo, hi, axis, amax, 1);
        }
        if (lane == 0) {
            const int64_t lid = (int64_t)sg.nid + 1, rid = (int64_t)sg.nid + 2 * (int64_t)nl;
            write_node(o, sg.nid, xmin, ymin, xmax, ymax, r0, n, lid, rid);
            in.nl = nl;
            in.axis = (int8_t)axis;
            in.strict = (int8_t)strict;
            in.thr = thr;
            const int nr = n - nl;
            // children larger than LOCAL_MAX stay in the global level loop; smaller
            // internal children are finished later by one CTA each (k_tree_local)
            const int want = (nl > LOCAL_MAX) + (nr > LOCAL_MAX);
            int slot = want ? atomicAdd(cnt_next, want) : 0;
            if (nl == 1) {
                const uint32_t pi = al[lo];
                const double2 p = pts[pi];
                write_node(o, lid, p.x, p.y, p.x, p.y, pi, 1, -1, -1);
            } else if (nl > LOCAL_MAX) {
                in.cl = slot++;
                seg_next[in.cl] = Seg{lo, lo + nl, (int32_t)lid, 0};
            } else {
                local[atomicAdd(local_cnt, 1)] = Seg{lo, lo + nl, (int32_t)lid, parity_next};
            }
            if (nr == 1) {
                const uint32_t pi = al[lo + nl];
                const double2 p = pts[pi];
                write_node(o, rid, p.x, p.y, p.x, p.y, pi, 1, -1, -1);
            } else if (nr > LOCAL_MAX) {
                in.cr = slot;
                seg_next[in.cr] = Seg{lo + nl, hi, (int32_t)rid, 0};
            } else {
                local[atomicAdd(local_cnt, 1)] = Seg{lo + nl, hi, (int32_t)rid, parity_next};
            }
            info[s] = in;
        }
    }
}

__global__ void __launch_bounds__(256) k_tree_segments(const double2 *__restrict__ pts,
                                                       const uint32_t *__restrict__ xl,
                                                       const uint32_t *__restrict__ yl,
                                                       const Seg *__restrict__ seg, const int32_t *cnt_cur,
                                                       int32_t *cnt_next, Seg *seg_next, SegInfo *info,
                                                       TreeOut o, int64_t *flags, Seg *local,
                                                       int32_t *local_cnt, int parity_next) {
    const int nseg = *cnt_cur;
    if (nseg == 0) return;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nseg; s += warps)
        tree_segment(s, pts, xl, yl, seg, cnt_next, seg_next, info, o, flags, local, local_cnt, parity_next);
}

// ---------------------------------------------------------------- local subtrees
// A segment of at most LOCAL_MAX points is finished by ONE CTA: its two
// lists are staged in shared memory and the same level-synchronous split
// (segments -> flags -> block scan -> stable partition) runs with CTA
// barriers instead of grid-wide ones.

struct LocalSub {
    int16_t lo, hi;
    int32_t nid;
};
struct LocalInfo {
    double thr;
    int16_t lo, nl, cl, cr;
    int8_t axis, strict, pad0, pad1;
};

struct LocalSmem {
    double px[LOCAL_MAX], py[LOCAL_MAX];  // coordinates by local id (local id = X-list rank)
    uint32_t gid[LOCAL_MAX];              // local id -> point index
    uint16_t xl[2][LOCAL_MAX];            // local ids in X-list / Y-list order
    uint16_t yl[2][LOCAL_MAX];
    int16_t ps[2][LOCAL_MAX];
    int16_t ex[LOCAL_MAX];
    LocalSub sub[2][LOCAL_MAX / 2 + 1];
    LocalInfo info[LOCAL_MAX / 2 + 1];
    int16_t big[LOCAL_MAX / 2 + 1];
    int32_t warp_tot[LT / 32];
    int32_t nsub_ring[3], nbig_ring[2];  // per-level counters, rings (no reset barrier)
};

__device__ __forceinline__ double lcoord(const LocalSmem &S, int id, int axis) {
    return axis ? S.py[id] : S.px[id];
}

// warp-cooperative prefix count on a shared-memory list (see warp_prefix_count)
__device__ int local_prefix_count(const LocalSmem &S, const uint16_t *list, int lo, int hi, int axis, double t,
                                  int strict) {
    const int lane = threadIdx.x & 31;
    int a = lo, b = hi;
    while (b - a > 32) {
        const int step = (b - a + 31) >> 5;
        const int p = a + lane * step;
        bool ok = false;
        if (p < b) {
            const double c = lcoord(S, list[p], axis);
            ok = strict ? (c < t) : (c <= t);
        }
        const int k = __popc(__ballot_sync(0xffffffffu, ok));
        const int na = k ? a + (k - 1) * step + 1 : a;
        const int nb = k < 32 ? min(b, a + k * step) : b;
        a = na;
        b = nb;
    }
    const int p = a + lane;
    bool ok = false;
    if (p < b) {
        const double c = lcoord(S, list[p], axis);
        ok = strict ? (c < t) : (c <= t);
    }
    return a + __popc(__ballot_sync(0xffffffffu, ok)) - lo;
}

// scalar prefix count on a shared-memory list (one thread per small sub-segment)
__device__ __forceinline__ int scalar_prefix_count(const LocalSmem &S, const uint16_t *list, int lo, int hi,
                                                   int axis, double t, int strict) {
    int a = lo, b = hi;
    while (a < b) {
        const int mm = (a + b) >> 1;
        const double c = lcoord(S, list[mm], axis);
        if (strict ? (c < t) : (c <= t)) a = mm + 1; else b = mm;
    }
    return a - lo;
}

// split one sub-segment (spanner.py:124-148); WARP = true: the calling warp
// cooperates on the search and lane 0 writes, false: the calling thread alone
template <bool WARP>
__device__ __forceinline__ void local_split(LocalSmem &S, int s, int cur, const TreeOut &o, int64_t *flags,
                                            int32_t *nsub_next) {
    const int lane = threadIdx.x & 31;
    const bool writer = WARP ? lane == 0 : true;
    const LocalSub sg = S.sub[cur][s];
    const int lo = sg.lo, hi = sg.hi, n = hi - lo;
    const uint16_t *xl = S.xl[cur], *yl = S.yl[cur];
    const int r0 = xl[lo];
    const double xmin = S.px[r0], xmax = S.px[xl[hi - 1]];
    const double ymin = S.py[yl[lo]], ymax = S.py[yl[hi - 1]];
    const double ext_x = dsub(xmax, xmin), ext_y = dsub(ymax, ymin);
    LocalInfo in{};
    in.lo = (int16_t)lo;
    in.cl = in.cr = -1;
    if (ext_x == 0.0 && ext_y == 0.0) {
        if (writer) {
            atomicOr((unsigned long long *)&flags[F_DUP], 1ull);
            write_node(o, sg.nid, xmin, ymin, xmax, ymax, S.gid[r0], n, -1, -1);
            in.nl = (int16_t)n;
            in.thr = INFINITY;
            S.info[s] = in;
        }
        return;
    }
    const int axis = ext_x >= ext_y ? 0 : 1;
    const uint16_t *al = axis ? yl : xl;
    const double amin = axis ? ymin : xmin, amax = axis ? ymax : xmax;
    const double mid = dmul(0.5, dadd(amin, amax));
    int nl = WARP ? local_prefix_count(S, al, lo, hi, axis, mid, 0) : scalar_prefix_count(S, al, lo, hi, axis, mid, 0);
    int strict = 0;
    double thr = mid;
    if (nl == 0 || nl == n) {
        strict = 1;
        thr = amax;
        nl = WARP ? local_prefix_count(S, al, lo, hi, axis, amax, 1) : scalar_prefix_count(S, al, lo, hi, axis, amax, 1);
    }
    if (!writer) return;
    const int64_t lid = (int64_t)sg.nid + 1, rid = (int64_t)sg.nid + 2 * (int64_t)nl;
    write_node(o, sg.nid, xmin, ymin, xmax, ymax, S.gid[r0], n, lid, rid);
    in.nl = (int16_t)nl;
    in.axis = (int8_t)axis;
    in.strict = (int8_t)strict;
    in.thr = thr;
    const int nr = n - nl;
    const int want = (nl > 1) + (nr > 1);
    int slot = want ? atomicAdd(nsub_next, want) : 0;
    if (nl == 1) {
        const int li = al[lo];
        write_node(o, lid, S.px[li], S.py[li], S.px[li], S.py[li], S.gid[li], 1, -1, -1);
    } else {
        in.cl = (int16_t)slot;
        S.sub[cur ^ 1][slot++] = LocalSub{(int16_t)lo, (int16_t)(lo + nl), (int32_t)lid};
    }
    if (nr == 1) {
        const int li = al[lo + nl];
        write_node(o, rid, S.px[li], S.py[li], S.px[li], S.py[li], S.gid[li], 1, -1, -1);
    } else {
        in.cr = (int16_t)slot;
        S.sub[cur ^ 1][slot] = LocalSub{(int16_t)(lo + nl), (int16_t)hi, (int32_t)rid};
    }
    S.info[s] = in;
}

__global__ void __launch_bounds__(LT) k_tree_local(const double2 *__restrict__ pts, const uint32_t *xl0,
                                                    const uint32_t *xl1, const uint32_t *yl0,
                                                    const uint32_t *yl1, const Seg *__restrict__ local,
                                                    const int32_t *local_cnt, int32_t *inv, TreeOut o,
                                                    int64_t *flags, const int32_t *depth_src, int64_t *h) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LocalSmem &S = *reinterpret_cast<LocalSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nloc = *local_cnt;
    for (int ls = blockIdx.x; ls < nloc; ls += gridDim.x) {
        const Seg L = local[ls];
        const int m = L.hi - L.lo;
        const uint32_t *gx = L.pad ? xl1 : xl0, *gy = L.pad ? yl1 : yl0;
        // stage the segment: local id = rank in the X-list
        for (int i = tid; i < m; i += LT) {
            const uint32_t g = gx[L.lo + i];
            const double2 p = pts[g];
            S.px[i] = p.x;
            S.py[i] = p.y;
            S.gid[i] = g;
            S.xl[0][i] = (uint16_t)i;
            S.ps[0][i] = 0;
            inv[g] = i;
        }
        __syncthreads();
        for (int i = tid; i < m; i += LT) S.yl[0][i] = (uint16_t)inv[gy[L.lo + i]];
        if (tid == 0) {
            S.sub[0][0] = LocalSub{0, (int16_t)m, L.nid};
            S.nsub_ring[1] = 0;
            S.nbig_ring[0] = 0;
        }
        __syncthreads();
        int cur = 0, nsub = 1, lv = 0;
        while (nsub > 0) {
            // level lv appends to nsub_ring[(lv+1)%3] and counts its big sub-segments in
            // nbig_ring[lv&1]; the slots the NEXT level uses are zeroed during this one
            // (after the first barrier: every thread has read them by then), so no
            // barrier-separated reset is needed
            int32_t *nnext = &S.nsub_ring[(lv + 1) % 3];
            int32_t *nbig = &S.nbig_ring[lv & 1];
            // (A) small sub-segments: one thread each; large ones: one warp each
            for (int s = tid; s < nsub; s += LT) {
                if (S.sub[cur][s].hi - S.sub[cur][s].lo > 64)
                    S.big[atomicAdd(nbig, 1)] = (int16_t)s;
                else
                    local_split<false>(S, s, cur, o, flags, nnext);
            }
            __syncthreads();
            if (tid == 0) {
                S.nsub_ring[(lv + 2) % 3] = 0;
                S.nbig_ring[(lv + 1) & 1] = 0;
            }
            for (int k = wid; k < *nbig; k += LT / 32) local_split<true>(S, S.big[k], cur, o, flags, nnext);
            __syncthreads();
            // (B) flags of the other list + block exclusive scan (8 positions per thread)
            int f[LPT], sum = 0;
#pragma unroll
            for (int i = 0; i < LPT; i++) {
                const int p = tid * LPT + i;
                int v = 0;
                if (p < m) {
                    const int s = S.ps[cur][p];
                    if (s >= 0) {
                        const LocalInfo &in = S.info[s];
                        const int e = in.axis ? S.xl[cur][p] : S.yl[cur][p];
                        const double c = lcoord(S, e, in.axis);
                        v = (in.strict ? (c < in.thr) : (c <= in.thr)) ? 1 : 0;
                    }
                }
                f[i] = v;
                sum += v;
            }
            {
                int x = sum;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, off);
                    if (lane >= off) x += y;
                }
                if (lane == 31) S.warp_tot[wid] = x;
                __syncthreads();
                int base = 0;
                for (int w = 0; w < wid; w++) base += S.warp_tot[w];
                int run = base + x - sum;
#pragma unroll
                for (int i = 0; i < LPT; i++) {
                    const int p = tid * LPT + i;
                    if (p < m) S.ex[p] = (int16_t)run;
                    run += f[i];
                }
            }
            __syncthreads();
            // (C) stable partition of the other list inside each sub-segment
#pragma unroll
            for (int i = 0; i < LPT; i++) {
                const int p = tid * LPT + i;
                if (p >= m) continue;
                const int s = S.ps[cur][p];
                if (s < 0) {
                    S.ps[cur ^ 1][p] = -1;
                    continue;
                }
                const LocalInfo in = S.info[s];
                const int rt = S.ex[p] - S.ex[in.lo];
                const int rf = (p - in.lo) - rt;
                const int np_ = f[i] ? in.lo + rt : in.lo + in.nl + rf;
                if (in.axis) {
                    S.yl[cur ^ 1][p] = S.yl[cur][p];
                    S.xl[cur ^ 1][np_] = S.xl[cur][p];
                } else {
                    S.xl[cur ^ 1][p] = S.xl[cur][p];
                    S.yl[cur ^ 1][np_] = S.yl[cur][p];
                }
                S.ps[cur ^ 1][p] = (p < in.lo + in.nl) ? in.cl : in.cr;
            }
            __syncthreads();
            nsub = *nnext;
            cur ^= 1;
            lv++;
        }
        __syncthreads();
    }
    // the last CTA to finish copies the depth of the cooperative levels and the duplicate
    // flag to the page-locked host mirror (the stage needs no small-read launch)
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    unsigned long long *ticket = reinterpret_cast<unsigned long long *>(flags + F_TREE_TICKET);
    if (tid == 0) s_last = atomicAdd(ticket, 1ull) == gridDim.x - 1;
    __syncthreads();
    if (s_last && tid == 0) {
        __threadfence();
        if (depth_src) *reinterpret_cast<volatile int32_t *>(h + H_TREE_DEPTH) = *(const volatile int32_t *)depth_src;
        reinterpret_cast<volatile int64_t *>(h)[H_TREE_DUP] = reinterpret_cast<volatile int64_t *>(flags)[F_DUP];
        *ticket = 0;
    }
}

// 1 if the OTHER list's element at position p goes to the left child
__device__ __forceinline__ int pos_flag(int64_t p, const double2 *__restrict__ pts,
                                        const uint32_t *__restrict__ xl, const uint32_t *__restrict__ yl,
                                        const int32_t *__restrict__ pos_seg, const SegInfo *__restrict__ info) {
    const int s = pos_seg[p];
    if (s < 0) return 0;
    const SegInfo &in = info[s];
    const uint32_t e = in.axis ? xl[p] : yl[p];
    const double c = coord(pts, e, in.axis);
    return (in.strict ? (c < in.thr) : (c <= in.thr)) ? 1 : 0;
}

__global__ void k_tree_flags(const double2 *__restrict__ pts, const uint32_t *__restrict__ xl,
                             const uint32_t *__restrict__ yl, const int32_t *__restrict__ pos_seg,
                             const SegInfo *__restrict__ info, const int32_t *cnt_cur, int64_t n,
                             int32_t *fl) {
    if (*cnt_cur == 0) return;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        fl[p] = pos_flag(p, pts, xl, yl, pos_seg, info);
}

// stable partition of the other list inside the position's segment
// destination of position p's other-list entry in the stable partition
__device__ __forceinline__ int64_t scatter_dest(int64_t p, int f, int64_t excl_p, int64_t excl_lo,
                                               const SegInfo &in) {
    const int64_t rt = excl_p - excl_lo;
    const int64_t rf = (p - in.lo) - rt;
    return f ? in.lo + rt : in.lo + in.nl + rf;
}

struct FlagVal {
    const int32_t *fl;
    __device__ int64_t operator()(int64_t i) const { return fl[i]; }
};

__global__ void k_tree_scatter(const uint32_t *__restrict__ xl, const uint32_t *__restrict__ yl,
                               const int32_t *__restrict__ pos_seg, const SegInfo *__restrict__ info,
                               const int32_t *__restrict__ fl, const int64_t *__restrict__ excl,
                               const int32_t *cnt_cur, int64_t n, uint32_t *xl_new, uint32_t *yl_new,
                               int32_t *pos_seg_new, int32_t *cnt_clear) {
    // clear the counter two levels ahead even on a dead level, so stale counts
    // can never revive a finished ring slot
    if (blockIdx.x == 0 && threadIdx.x == 0) *cnt_clear = 0;
    if (*cnt_cur == 0) return;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int s = pos_seg[p];
        if (s < 0) {
            pos_seg_new[p] = -1;
            continue;
        }
        const SegInfo in = info[s];
        const int64_t rt = excl[p] - excl[in.lo];
        const int64_t rf = (p - in.lo) - rt;
        const int64_t np_ = fl[p] ? in.lo + rt : in.lo + in.nl + rf;
        if (in.axis) {  // split on y: Y-list stays, X-list is partitioned
            yl_new[p] = yl[p];
            xl_new[np_] = xl[p];
        } else {
            xl_new[p] = xl[p];
            yl_new[np_] = yl[p];
        }
        pos_seg_new[p] = (p < in.lo + in.nl) ? in.cl : in.cr;
    }
}

// ---------------------------------------------------------------- persistent cooperative build
// All levels in ONE cooperative launch: per level (A) one warp per segment,
// grid sync, (B) flags + tile-local scans, grid sync, (C) tile prefixes
// (every CTA scans the tile sums in shared memory) + scatter, grid sync.
// Three grid barriers per level instead of four launches and a host poll.

constexpr int TP_IPT = 2;
constexpr int TP_TILE = 256 * TP_IPT;
constexpr int COOP_MAX_TILES = 8192;

struct CoopArgs {
    const double2 *pts;
    int64_t n;
    uint32_t *xl[2], *yl[2];
    double2 *xc[2], *yc[2];  // the lists' coordinates, inline
    int32_t *pos_seg[2];
    Seg *seg[2];
    SegInfo *info;
    int32_t *cnt;  // ring of 3 live-segment counters
    int32_t *lpre, *tsum;
    int32_t *levels_out;
    int64_t *flags;
    Seg *local;
    int32_t *local_cnt;
    TreeOut o;
};

__device__ __forceinline__ int block_excl_scan(int v, int *total, int32_t *s_warp) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) {
        const int sw = s_warp[w];
        if (w < wid) off += sw;
        tot += sw;
    }
    __syncthreads();
    *total = tot;
    return off + x - v;
}

__global__ void __launch_bounds__(256) k_tree_coop(CoopArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ int32_t s_tp[];  // exclusive prefix of the tile sums
    __shared__ int32_t s_warp[8];
    const int tid = threadIdx.x;
    const int64_t n = A.n;
    const int ntiles = (int)((n + TP_TILE - 1) / TP_TILE);
    int cur = 0, level = 0;
    while (true) {
        const int nseg = *((volatile int32_t *)&A.cnt[level % 3]);
        if (nseg == 0) break;
        // (A) segments
        const int warps = (gridDim.x * blockDim.x) >> 5;
        for (int s = (blockIdx.x * blockDim.x + tid) >> 5; s < nseg; s += warps)
            tree_segment(s, A.pts, A.xl[cur], A.yl[cur], A.seg[cur], &A.cnt[(level + 1) % 3], A.seg[cur ^ 1],
                         A.info, A.o, A.flags, A.local, A.local_cnt, cur ^ 1, A.xc[cur], A.yc[cur]);
        grid.sync();
        // (B) flags and tile-local exclusive prefixes
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t base = (int64_t)t * TP_TILE + tid * TP_IPT;
            int f[TP_IPT];
            int sum = 0;
            // the flag needs the position's segment, that segment's split and the
            // other list's coordinate (inline): two dependent links, each issued
            // for all items before the next
            int sg[TP_IPT];
            double2 qx[TP_IPT], qy[TP_IPT];
            SegInfo inf[TP_IPT];
#pragma unroll
            for (int i = 0; i < TP_IPT; i++) {
                const bool in_n = base + i < n;
                sg[i] = in_n ? A.pos_seg[cur][base + i] : -1;
                if (in_n) {
                    qx[i] = A.xc[cur][base + i];
                    qy[i] = A.yc[cur][base + i];
                }
            }
#pragma unroll
            for (int i = 0; i < TP_IPT; i++) {
                if (sg[i] >= 0) inf[i] = A.info[sg[i]];
                else inf[i].axis = 0;
            }
#pragma unroll
            for (int i = 0; i < TP_IPT; i++) {
                int v = 0;
                if (sg[i] >= 0) {
                    // split on y: the X-list is partitioned by its points' y, and vice versa
                    const double c = inf[i].axis ? qx[i].y : qy[i].x;
                    v = (inf[i].strict ? (c < inf[i].thr) : (c <= inf[i].thr)) ? 1 : 0;
                }
                f[i] = v;
                sum += v;
            }
            int tot;
            int run = block_excl_scan(sum, &tot, s_warp);
#pragma unroll
            for (int i = 0; i < TP_IPT; i++) {
                const int64_t p = base + i;
                if (p < n) A.lpre[p] = run | (f[i] << 31);
                run += f[i];
            }
            if (tid == 0) A.tsum[t] = tot;
        }
        grid.sync();
        // (C) tile prefixes (redundantly per CTA) and the stable partition
        {
            int carry = 0;
            for (int t0 = 0; t0 < ntiles; t0 += 256) {
                const int t = t0 + tid;
                const int v = t < ntiles ? A.tsum[t] : 0;
                int tot;
                const int ex = block_excl_scan(v, &tot, s_warp);
                if (t < ntiles) s_tp[t] = carry + ex;
                carry += tot;
            }
            __syncthreads();
        }
        if (blockIdx.x == 0 && tid == 0) A.cnt[(level + 2) % 3] = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            // same staging as (B): every dependent load issued for all items at
            // once; the entries to move do not depend on the split and load first
            constexpr int J = TP_TILE / 256;
            int64_t pp[J];
            int sg[J];
            SegInfo inf[J];
            int32_t lp[J], ll[J];
            uint32_t ex[J], ey[J];
            double2 cx[J], cy[J];
#pragma unroll
            for (int j = 0; j < J; j++) {
                pp[j] = (int64_t)t * TP_TILE + tid + 256 * j;
                const bool in_n = pp[j] < n;
                sg[j] = in_n ? A.pos_seg[cur][pp[j]] : -2;
                if (in_n) {
                    lp[j] = A.lpre[pp[j]];
                    ex[j] = A.xl[cur][pp[j]];
                    ey[j] = A.yl[cur][pp[j]];
                    cx[j] = A.xc[cur][pp[j]];
                    cy[j] = A.yc[cur][pp[j]];
                }
            }
#pragma unroll
            for (int j = 0; j < J; j++)
                if (sg[j] >= 0) inf[j] = A.info[sg[j]];
#pragma unroll
            for (int j = 0; j < J; j++)
                if (sg[j] >= 0) ll[j] = A.lpre[inf[j].lo];
#pragma unroll
            for (int j = 0; j < J; j++) {
                if (sg[j] == -1) A.pos_seg[cur ^ 1][pp[j]] = -1;
                if (sg[j] < 0) continue;
                const int64_t ep = (int64_t)s_tp[t] + (lp[j] & 0x7fffffff);
                const int64_t el = (int64_t)s_tp[inf[j].lo / TP_TILE] + (ll[j] & 0x7fffffff);
                const int64_t np_ = scatter_dest(pp[j], (int)((uint32_t)lp[j] >> 31), ep, el, inf[j]);
                if (inf[j].axis) {  // split on y: Y-list stays, X-list is partitioned
                    A.yl[cur ^ 1][pp[j]] = ey[j];
                    A.yc[cur ^ 1][pp[j]] = cy[j];
                    A.xl[cur ^ 1][np_] = ex[j];
                    A.xc[cur ^ 1][np_] = cx[j];
                } else {
                    A.xl[cur ^ 1][pp[j]] = ex[j];
                    A.xc[cur ^ 1][pp[j]] = cx[j];
                    A.yl[cur ^ 1][np_] = ey[j];
                    A.yc[cur ^ 1][np_] = cy[j];
                }
                A.pos_seg[cur ^ 1][pp[j]] = (pp[j] < inf[j].lo + inf[j].nl) ? inf[j].cl : inf[j].cr;
            }
        }
        grid.sync();
        cur ^= 1;
        level++;
    }
    if (blockIdx.x == 0 && tid == 0) *A.levels_out = level | (cur << 30);
}

__global__ void k_geom_from_arrays(const int64_t *left, const int64_t *right, const double4 *bbox,
                                   const int64_t *rep, int64_t nn, NodeGeom *geom, int2 *lr,
                                   int32_t *rep32) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double4 b = bbox[i];
        const double w = dsub(b.z, b.x), h = dsub(b.w, b.y);
        const double dsq = dadd(dmul(w, w), dmul(h, h));
        NodeGeom g;
        g.cx = dmul(0.5, dadd(b.x, b.z));
        g.cy = dmul(0.5, dadd(b.y, b.w));
        g.r = dmul(0.5, dsqrt(dsq));
        g.dsq = dsq;
        geom[i] = g;
        lr[i] = make_int2((int)left[i], (int)right[i]);
        rep32[i] = (int32_t)rep[i];
    }
}

}  // namespace

int tree_geom(Ctx &c) {
    const int64_t nn = c.tree_n_nodes;
    NodeGeom *geom;
    int2 *lr;
    int32_t *rep32;
    W1G_TRY(ensure(c.t_geom, (size_t)nn + 1, &geom));
    W1G_TRY(ensure(c.t_lr, (size_t)nn + 1, &lr));
    W1G_TRY(ensure(c.t_rep32, (size_t)nn + 1, &rep32));
    if (nn == 0) return W1G_OK;
    k_geom_from_arrays<<<grid_for(nn, 256, 8u * c.sm_count), 256, 0, c.stream>>>(
        ptr<int64_t>(c.t_left), ptr<int64_t>(c.t_right), ptr<double4>(c.t_bbox), ptr<int64_t>(c.t_rep),
        nn, geom, lr, rep32);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

int tree_run(Ctx &c, const double2 *pts, int64_t n, int64_t *n_nodes, int32_t *depth, bool defer) {
    c.tree_valid = false;
    c.pair_pts = pts;
    const int64_t nn = n > 0 ? 2 * n - 1 : 0;
    c.tree_n_points = n;
    c.tree_n_nodes = nn;
    *n_nodes = nn;
    *depth = 0;
    TreeOut o;
    W1G_TRY(ensure(c.t_left, (size_t)nn + 1, &o.left));
    W1G_TRY(ensure(c.t_right, (size_t)nn + 1, &o.right));
    W1G_TRY(ensure(c.t_rep, (size_t)nn + 1, &o.rep));
    W1G_TRY(ensure(c.t_size, (size_t)nn + 1, &o.size));
    W1G_TRY(ensure(c.t_bbox, (size_t)nn + 1, &o.bbox));
    W1G_TRY(ensure(c.t_geom, (size_t)nn + 1, &o.geom));
    W1G_TRY(ensure(c.t_lr, (size_t)nn + 1, &o.lr));
    W1G_TRY(ensure(c.t_rep32, (size_t)nn + 1, &o.rep32));
    if (n == 0) {
        c.tree_valid = true;
        return W1G_OK;
    }
    // presorted lists
    uint64_t *kx0, *kx1, *ky0, *ky1;
    uint32_t *xl[2], *yl[2];
    W1G_TRY(ensure(c.scr[0], n, &kx0));
    W1G_TRY(ensure(c.scr[1], n, &kx1));
    W1G_TRY(ensure(c.scr[4], n, &ky0));
    W1G_TRY(ensure(c.scr[5], n, &ky1));
    W1G_TRY(ensure(c.scr[6], n, &xl[0]));
    W1G_TRY(ensure(c.scr[7], n, &yl[0]));
    W1G_TRY(ensure(c.scr[8], n, &xl[1]));
    W1G_TRY(ensure(c.scr[9], n, &yl[1]));
    const unsigned g = grid_for(n, 256, 8u * c.sm_count);
    SubTimer T(c, "tree");
    // delta_condense may have built both lists already from its cell order (k_cl_columns)
    const bool pre = c.pre_n == n && pts == ptr<double2>(c.nodes[1].pts);
    c.pre_n = 0;
    if (pre) {
        xl[0] = ptr<uint32_t>(c.pre_xl);
        yl[0] = ptr<uint32_t>(c.pre_yl);
    } else {
        k_presort_keys<<<g, 256, 0, c.stream>>>(pts, n, kx0, kx1, ky0, ky1, xl[0], yl[0]);
        W1G_CHECK_LAUNCH();
        // X-list by (x, y) and Y-list by (y, x): kx1 = key(x), kx0 = key(y); both in the same launches
        const Lex2Job jobs[2] = {{kx1, kx0, xl[0], n}, {kx0, kx1, yl[0], n}};
        W1G_TRY(sort_lex2_multi(c, jobs, 2));
    }
    T.mark("sort_xy");
    // level state
    Seg *seg[2];
    SegInfo *info;
    int32_t *pos_seg[2], *cnt, *fl;
    int64_t *excl;
    const int64_t seg_cap = n / 2 + 2;
    W1G_TRY(ensure(c.scr[10], (size_t)seg_cap, &seg[0]));
    W1G_TRY(ensure(c.scr[11], (size_t)seg_cap, &seg[1]));
    W1G_TRY(ensure(c.scr[12], (size_t)seg_cap, &info));
    W1G_TRY(ensure(c.scr[13], (size_t)n, &pos_seg[0]));
    W1G_TRY(ensure(c.scr[14], (size_t)n, &pos_seg[1]));
    W1G_TRY(ensure(c.scr[16], (size_t)n, &fl));
    W1G_TRY(ensure(c.scr[3], (size_t)n, &excl));
    const int max_levels = (int)(n + 2);
    // live-segment counters, a ring of 3: level l reads cnt[l%3], appends to
    // cnt[(l+1)%3]; its scatter kernel clears cnt[(l+2)%3]
    Seg *local;
    int32_t *local_cnt;
    W1G_TRY(ensure(c.scr[15], 16, &cnt));
    local_cnt = cnt + 8;
    W1G_TRY(ensure(c.scr[20], (size_t)seg_cap + 2, &local));
    W1G_TRY(flags_reset(c));
    W1G_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * 16, c.stream));
    int levels = 0;
    const int32_t *depth_src = nullptr;  // the cooperative kernel's level count (device)
    const int64_t ntiles = (n + TP_TILE - 1) / TP_TILE;
    static const bool no_coop = [] {  // W1G_NO_COOP=1: the multi-kernel level loop (measurement)
        const char *e = getenv("W1G_NO_COOP");
        return e && *e == '1';
    }();
    const bool coop = n > LOCAL_MAX && ntiles <= COOP_MAX_TILES && !no_coop && !c.no_coop;
    double2 *xc[2] = {nullptr, nullptr}, *yc[2] = {nullptr, nullptr};
    if (coop) {
        W1G_TRY(ensure(c.scr[2], (size_t)n, &xc[0]));
        W1G_TRY(ensure(c.scr[21], (size_t)n, &xc[1]));
        W1G_TRY(ensure(c.scr[22], (size_t)n, &yc[0]));
        W1G_TRY(ensure(c.scr[23], (size_t)n, &yc[1]));
    }
    k_tree_init<<<g, 256, 0, c.stream>>>(n, seg[0], pos_seg[0], cnt, pts, xl[0], o, local, local_cnt, yl[0], xc[0],
                                         yc[0]);
    W1G_CHECK_LAUNCH();
    if (coop) {
        // the global levels (segments > LOCAL_MAX) in one persistent cooperative launch
        int32_t *lpre, *tsum, *lv;
        W1G_TRY(ensure(c.scr[17], (size_t)n, &lpre));
        W1G_TRY(ensure(c.scr[18], (size_t)ntiles + 1, &tsum));
        W1G_TRY(ensure(c.scr[19], 4, &lv));
        CoopArgs A;
        A.pts = pts;
        A.n = n;
        A.xl[0] = xl[0];
        A.xl[1] = xl[1];
        A.yl[0] = yl[0];
        A.yl[1] = yl[1];
        A.xc[0] = xc[0];
        A.xc[1] = xc[1];
        A.yc[0] = yc[0];
        A.yc[1] = yc[1];
        A.pos_seg[0] = pos_seg[0];
        A.pos_seg[1] = pos_seg[1];
        A.seg[0] = seg[0];
        A.seg[1] = seg[1];
        A.info = info;
        A.cnt = cnt;
        A.lpre = lpre;
        A.tsum = tsum;
        A.levels_out = lv;
        A.flags = dflags(c);
        A.local = local;
        A.local_cnt = local_cnt;
        A.o = o;
        const size_t smem = sizeof(int32_t) * (size_t)(ntiles + 1);
        int per_sm = 0;
        W1G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tree_coop, 256, smem));
        if (per_sm < 1) per_sm = 1;
        {
            const char *e = getenv("W1G_COOP_PER_SM");
            const int cap = e ? atoi(e) : 2;
            if (per_sm > cap) per_sm = cap;
        }
        const int G = max(1, per_sm * c.sm_count / max(1, c.coop_share));
        void *args[] = {&A};
        W1G_CUDA(cudaLaunchCooperativeKernel((void *)k_tree_coop, G, 256, args, smem, c.stream));
        W1G_CHECK_LAUNCH();
        // the depth is read after the stage's (or, deferred, the caller's) next round trip
        depth_src = lv;
        levels = -1;
    } else if (n > LOCAL_MAX) {
        // fallback for very large inputs: one launch per phase, host polls per batch
        const unsigned gseg = grid_for(seg_cap * 32, 256, 16u * c.sm_count);
        int level = 0, cur = 0;
        const int BATCH = 12;
        while (true) {
            for (int b = 0; b < BATCH; b++, level++) {
                const int32_t *cc = cnt + level % 3;
                k_tree_segments<<<gseg, 256, 0, c.stream>>>(pts, xl[cur], yl[cur], seg[cur], cc,
                                                           cnt + (level + 1) % 3, seg[cur ^ 1], info, o, dflags(c),
                                                           local, local_cnt, cur ^ 1);
                W1G_CHECK_LAUNCH();
                k_tree_flags<<<g, 256, 0, c.stream>>>(pts, xl[cur], yl[cur], pos_seg[cur], info, cc, n, fl);
                W1G_CHECK_LAUNCH();
                W1G_TRY(scan_i64(c, FlagVal{fl}, n, excl, nullptr, cc));
                k_tree_scatter<<<g, 256, 0, c.stream>>>(xl[cur], yl[cur], pos_seg[cur], info, fl, excl, cc, n,
                                                       xl[cur ^ 1], yl[cur ^ 1], pos_seg[cur ^ 1],
                                                       cnt + (level + 2) % 3);
                W1G_CHECK_LAUNCH();
                cur ^= 1;
            }
            W1G_TRY(to_host_small(c, c.h_pinned + F_ACTIVE, cnt + level % 3, sizeof(int32_t)));
            W1G_TRY(stream_sync(c));
            const int32_t live = *reinterpret_cast<int32_t *>(c.h_pinned + F_ACTIVE);
            if (live == 0 || level > max_levels) break;
        }
        levels = level;
    }
    T.mark("global_levels");
    // the subtrees of <= LOCAL_MAX points: one CTA each, shared-memory levels
    {
        const size_t smem = sizeof(LocalSmem);
        W1G_CUDA(cudaFuncSetAttribute(k_tree_local, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const unsigned gl = (unsigned)(2 * c.sm_count);
        if (levels >= 0) c.h_pinned[H_TREE_DEPTH] = levels;  // host-known (multi-kernel path / no global levels)
        k_tree_local<<<gl, LT, smem, c.stream>>>(pts, xl[0], xl[1], yl[0], yl[1], local, local_cnt, fl, o,
                                                  dflags(c), depth_src, c.h_pinned);
        W1G_CHECK_LAUNCH();
    }
    T.mark("local");
    W1G_CUDA(cudaEventRecord(c.ev[10], c.stream));  // depth and duplicate flag have landed once this has
    c.tree_valid = true;
    if (defer) {
        *depth = 0;
        return W1G_OK;
    }
    W1G_TRY(stream_sync(c));
    return tree_deferred_check(c, depth);
}

int tree_deferred_check(Ctx &c, int32_t *depth) {
    W1G_CUDA(cudaEventSynchronize(c.ev[10]));  // already complete after any later round trip
    if (c.h_pinned[H_TREE_DUP]) {
        c.tree_valid = false;
        set_error("split tree input contains duplicate points");
        return W1G_EDUPLICATE;
    }
    const int32_t levels = (int32_t)(c.h_pinned[H_TREE_DEPTH] & 0x3fffffff);
    c.tree_depth = levels;
    *depth = levels;
    return W1G_OK;
}

}  // namespace w1g
