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
//  * the split along the chosen axis is a prefix of that axis' list (binary
//    search), only the other list is stably partitioned (one device scan);
//  * leaf children are finalised immediately, internal children become the
//    next level's segments.
// Levels run in batches without host synchronisation; the host only polls
// the number of live segments between batches.
#include "common.cuh"

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

__device__ __forceinline__ void write_node(int64_t nid, double xmin, double ymin, double xmax,
                                           double ymax, int64_t rep, int64_t size, int64_t l, int64_t r,
                                           int64_t *left, int64_t *right, double4 *bbox, int64_t *reps,
                                           int64_t *sizes, NodeGeom *geom, int2 *lr, int32_t *rep32) {
    left[nid] = l;
    right[nid] = r;
    bbox[nid] = make_double4(xmin, ymin, xmax, ymax);
    reps[nid] = rep;
    sizes[nid] = size;
    // per-node terms of _ws_predicate / _diag_sq, spanner.py:178-194
    const double w = dsub(xmax, xmin), h = dsub(ymax, ymin);
    const double dsq = dadd(dmul(w, w), dmul(h, h));
    NodeGeom g;
    g.cx = dmul(0.5, dadd(xmin, xmax));
    g.cy = dmul(0.5, dadd(ymin, ymax));
    g.r = dmul(0.5, dsqrt(dsq));
    g.dsq = dsq;
    geom[nid] = g;
    lr[nid] = make_int2((int)l, (int)r);
    rep32[nid] = (int32_t)rep;
}

struct TreeOut {
    int64_t *left, *right, *rep, *size;
    double4 *bbox;
    NodeGeom *geom;
    int2 *lr;
    int32_t *rep32;
};

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
                            const uint32_t *xl, TreeOut o) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        pos_seg[i] = n == 1 ? -1 : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (n == 1) {
            double2 p = pts[xl[0]];
            write_node(0, p.x, p.y, p.x, p.y, xl[0], 1, -1, -1, o.left, o.right, o.bbox, o.rep,
                       o.size, o.geom, o.lr, o.rep32);
            cnt[0] = 0;
        } else {
            seg[0] = Seg{0, (int32_t)n, 0, 0};
            cnt[0] = 1;
        }
    }
}

__device__ __forceinline__ double coord(const double2 *pts, uint32_t i, int axis) {
    double2 p = pts[i];
    return axis ? p.y : p.x;
}

// per segment: bbox, rep, axis, split point, children (spanner.py:124-148)
__global__ void k_tree_segments(const double2 *__restrict__ pts, const uint32_t *__restrict__ xl,
                                const uint32_t *__restrict__ yl, const Seg *__restrict__ seg,
                                const int32_t *cnt_cur, int32_t *cnt_next, Seg *seg_next,
                                SegInfo *info, TreeOut o, int64_t *flags) {
    const int nseg = *cnt_cur;
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * blockDim.x;
    for (int base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; base < nseg; base += stride) {
        const int s = base + lane;
        const bool valid = s < nseg;
        int want = 0;
        Seg sg{0, 0, 0, 0};
        SegInfo in{};
        if (valid) {
            sg = seg[s];
            const int lo = sg.lo, hi = sg.hi, n = hi - lo;
            const uint32_t r0 = xl[lo];
            const double2 pr = pts[r0];
            const double xmin = pr.x, xmax = pts[xl[hi - 1]].x;
            const double ymin = pts[yl[lo]].y, ymax = pts[yl[hi - 1]].y;
            const double ext_x = dsub(xmax, xmin), ext_y = dsub(ymax, ymin);
            in.lo = lo;
            in.hi = hi;
            if (ext_x == 0.0 && ext_y == 0.0) {
                // spanner.py:134-135
                atomicOr((unsigned long long *)&flags[F_DUP], 1ull);
                write_node(sg.nid, xmin, ymin, xmax, ymax, r0, n, -1, -1, o.left, o.right, o.bbox,
                           o.rep, o.size, o.geom, o.lr, o.rep32);
                in.nl = n;  // every position keeps its place and is retired
                in.cl = in.cr = -1;
                in.axis = 0;
                in.strict = 0;
                in.thr = INFINITY;
            } else {
                const int axis = ext_x >= ext_y ? 0 : 1;
                const uint32_t *al = axis ? yl : xl;
                const double amin = axis ? ymin : xmin, amax = axis ? ymax : xmax;
                const double mid = dmul(0.5, dadd(amin, amax));
                // count of coord <= mid: the axis list is sorted by that coordinate
                int a = lo, b = hi;
                while (a < b) {
                    int m = (a + b) >> 1;
                    if (coord(pts, al[m], axis) <= mid) a = m + 1; else b = m;
                }
                int nl = a - lo;
                int strict = 0;
                double thr = mid;
                if (nl == 0 || nl == n) {
                    strict = 1;  // split off the max-attaining points instead
                    thr = amax;
                    a = lo;
                    b = hi;
                    while (a < b) {
                        int m = (a + b) >> 1;
                        if (coord(pts, al[m], axis) < amax) a = m + 1; else b = m;
                    }
                    nl = a - lo;
                }
                const int64_t lid = (int64_t)sg.nid + 1, rid = (int64_t)sg.nid + 2 * (int64_t)nl;
                write_node(sg.nid, xmin, ymin, xmax, ymax, r0, n, lid, rid, o.left, o.right, o.bbox,
                           o.rep, o.size, o.geom, o.lr, o.rep32);
                in.nl = nl;
                in.axis = (int8_t)axis;
                in.strict = (int8_t)strict;
                in.thr = thr;
                in.cl = in.cr = -1;
                if (nl == 1) {
                    const uint32_t pi = al[lo];
                    const double2 p = pts[pi];
                    write_node(lid, p.x, p.y, p.x, p.y, pi, 1, -1, -1, o.left, o.right, o.bbox, o.rep,
                               o.size, o.geom, o.lr, o.rep32);
                } else {
                    want++;
                }
                if (n - nl == 1) {
                    const uint32_t pi = al[lo + nl];
                    const double2 p = pts[pi];
                    write_node(rid, p.x, p.y, p.x, p.y, pi, 1, -1, -1, o.left, o.right, o.bbox, o.rep,
                               o.size, o.geom, o.lr, o.rep32);
                } else {
                    want++;
                }
            }
        }
        // warp-aggregated slot allocation for the internal children
        int x = want;
        for (int off = 1; off < 32; off <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        const int tot = __shfl_sync(0xffffffffu, x, 31);
        int wb = 0;
        if (lane == 31 && tot) wb = atomicAdd(cnt_next, tot);
        wb = __shfl_sync(0xffffffffu, wb, 31);
        int slot = wb + x - want;
        if (valid) {
            if (want) {
                const int nr = in.hi - in.lo - in.nl;
                if (in.nl > 1) {
                    in.cl = slot++;
                    seg_next[in.cl] = Seg{in.lo, in.lo + in.nl, sg.nid + 1, 0};
                }
                if (nr > 1) {
                    in.cr = slot;
                    seg_next[in.cr] = Seg{in.lo + in.nl, in.hi, sg.nid + 2 * in.nl, 0};
                }
            }
            info[s] = in;
        }
    }
}

struct PartFlag {
    const double2 *pts;
    const uint32_t *xl, *yl;
    const int32_t *pos_seg;
    const SegInfo *info;
    __device__ int64_t operator()(int64_t p) const {
        const int s = pos_seg[p];
        if (s < 0) return 0;
        const SegInfo &in = info[s];
        const uint32_t e = in.axis ? xl[p] : yl[p];  // element of the OTHER list
        const double c = coord(pts, e, in.axis);
        return (in.strict ? (c < in.thr) : (c <= in.thr)) ? 1 : 0;
    }
};

__global__ void k_tree_scatter(PartFlag f, int64_t n, const int64_t *excl, uint32_t *xl_new,
                               uint32_t *yl_new, int32_t *pos_seg_new, int32_t *cnt_clear) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *cnt_clear = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int s = f.pos_seg[p];
        if (s < 0) {
            pos_seg_new[p] = -1;
            continue;
        }
        const SegInfo in = f.info[s];
        const bool fl = f(p) != 0;
        const int64_t rt = excl[p] - excl[in.lo];
        const int64_t rf = (p - in.lo) - rt;
        const int64_t np_ = fl ? in.lo + rt : in.lo + in.nl + rf;
        if (in.axis) {  // split on y: Y-list stays, X-list is partitioned
            yl_new[p] = f.yl[p];
            xl_new[np_] = f.xl[p];
        } else {
            xl_new[p] = f.xl[p];
            yl_new[np_] = f.yl[p];
        }
        pos_seg_new[p] = (p < in.lo + in.nl) ? in.cl : in.cr;
    }
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

int tree_run(Ctx &c, const double2 *pts, int64_t n, int64_t *n_nodes, int32_t *depth) {
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
    k_presort_keys<<<g, 256, 0, c.stream>>>(pts, n, kx0, kx1, ky0, ky1, xl[0], yl[0]);
    W1G_CHECK_LAUNCH();
    {
        uint64_t *kx[2] = {kx0, kx1}, *ky[2] = {ky0, ky1};
        W1G_TRY(radix_sort(c, kx, 2, xl[0], n));
        W1G_TRY(radix_sort(c, ky, 2, yl[0], n));
    }
    // level state
    Seg *seg[2];
    SegInfo *info;
    int32_t *pos_seg[2], *cnt;
    int64_t *excl;
    const int64_t seg_cap = n / 2 + 2;
    W1G_TRY(ensure(c.scr[10], (size_t)seg_cap, &seg[0]));
    W1G_TRY(ensure(c.scr[11], (size_t)seg_cap, &seg[1]));
    W1G_TRY(ensure(c.scr[12], (size_t)seg_cap, &info));
    W1G_TRY(ensure(c.scr[13], (size_t)n, &pos_seg[0]));
    W1G_TRY(ensure(c.scr[14], (size_t)n, &pos_seg[1]));
    W1G_TRY(ensure(c.scr[3], (size_t)n, &excl));
    const int max_levels = (int)(n + 2);
    // live-segment counters, a ring of 3: level l reads cnt[l%3], appends to
    // cnt[(l+1)%3]; its scatter kernel clears cnt[(l+2)%3]
    W1G_TRY(ensure(c.scr[15], 8, &cnt));
    W1G_TRY(flags_reset(c));
    W1G_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * 8, c.stream));
    k_tree_init<<<g, 256, 0, c.stream>>>(n, seg[0], pos_seg[0], cnt, pts, xl[0], o);
    W1G_CHECK_LAUNCH();
    const unsigned gseg = grid_for(seg_cap, 256, 4u * c.sm_count);
    int level = 0, cur = 0;
    const int BATCH = 8;
    while (true) {
        for (int b = 0; b < BATCH; b++, level++) {
            k_tree_segments<<<gseg, 256, 0, c.stream>>>(pts, xl[cur], yl[cur], seg[cur], cnt + level % 3,
                                                       cnt + (level + 1) % 3, seg[cur ^ 1], info, o, dflags(c));
            W1G_CHECK_LAUNCH();
            PartFlag f{pts, xl[cur], yl[cur], pos_seg[cur], info};
            W1G_TRY(scan_i64(c, f, n, excl, nullptr));
            k_tree_scatter<<<g, 256, 0, c.stream>>>(f, n, excl, xl[cur ^ 1], yl[cur ^ 1], pos_seg[cur ^ 1],
                                                   cnt + (level + 2) % 3);
            W1G_CHECK_LAUNCH();
            cur ^= 1;
        }
        W1G_CUDA(cudaMemcpyAsync(c.h_pinned + F_ACTIVE, cnt + level % 3, sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, c.stream));
        W1G_CUDA(cudaMemcpyAsync(c.h_pinned + F_DUP, dflags(c) + F_DUP, sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, c.stream));
        W1G_CUDA(cudaStreamSynchronize(c.stream));
        const int32_t live = *reinterpret_cast<int32_t *>(c.h_pinned + F_ACTIVE);
        if (c.h_pinned[F_DUP]) {
            set_error("split tree input contains duplicate points");
            return W1G_EDUPLICATE;
        }
        if (live == 0 || level > max_levels) break;
    }
    // depth: levels that had live segments (+ the leaf level)
    c.tree_depth = level;
    *depth = level;
    c.tree_valid = true;
    return W1G_OK;
}

}  // namespace w1g
