// condense.cu -- node sparsification on device.
//
//  zero_condense  (diagram.py:190-208): order-preserving 128-bit (x, y) keys,
//      stable radix sort, run-length unique, per-side multiplicities.
//  delta_condense (condensation.py:62-124): exact fp64 snap with the
//      reference's round-half-away (sign(t)*floor(|t|+0.5)), signed-int64
//      cell keys packed into one word when the cell range allows, stable
//      radix sort, reduce-by-key of masses, splitmix64 per-cell offsets and
//      coords = fl(fl(cell*pitch) + offset).
#include "common.cuh"

namespace w1g {

namespace {

__device__ __forceinline__ double2 pick(const double2 *a, int64_t na, const double2 *b, int64_t i) {
    return i < na ? a[i] : b[i - na];
}

__global__ void k_zc_keys(const double2 *a, int64_t na, const double2 *b, int64_t n, uint64_t *hi,
                          uint64_t *lo, uint32_t *vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = pick(a, na, b, i);
        hi[i] = dkey(p.x);
        lo[i] = dkey(p.y);
        vals[i] = (uint32_t)i;
    }
}

struct ZcFlag {
    const double2 *a, *b;
    int64_t na;
    const uint32_t *v;
    __device__ int64_t operator()(int64_t i) const {
        if (i == 0) return 1;
        double2 p = pick(a, na, b, v[i]), q = pick(a, na, b, v[i - 1]);
        return (p.x == q.x && p.y == q.y) ? 0 : 1;
    }
};

__global__ void k_zc_emit(ZcFlag f, int64_t n, const int64_t *excl, double2 *pts, int64_t *am,
                          int64_t *bm) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t fl = f(i);
        int64_t rid = excl[i] + fl - 1;
        uint32_t src = f.v[i];
        if (fl) pts[rid] = pick(f.a, f.na, f.b, src);  // first of the run (lowest input index)
        if ((int64_t)src < f.na)
            atomicAdd((unsigned long long *)&am[rid], 1ull);
        else
            atomicAdd((unsigned long long *)&bm[rid], 1ull);
    }
}

// identical multisets (pipeline.py:106-109), plus what RWMD's frame needs
// (lower_bound.py:61-75): the member count of each side and the bbox
// (h: the page-locked mirror of the flag block; the last block to finish copies K0, the
// imbalance flag and the six statistics there -- the stage's round trip needs no small read)
__global__ void k_zc_stats(const int64_t *am, const int64_t *bm, const double2 *pts, const int64_t *kp, int64_t *f,
                           int64_t *h) {
    const int64_t k = *kp;
    int any = 0;
    unsigned long long na = 0, nb = 0, nx = 0, xx = 0, ny = 0, xy = 0;  // nx/ny: max of ~key = ~min key
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = am[i], b = bm[i];
        const double2 p = pts[i];
        any |= a != b;
        na += a > 0;
        nb += b > 0;
        const unsigned long long kx = dkey(p.x), ky = dkey(p.y);
        nx = max(nx, ~kx);
        xx = max(xx, kx);
        ny = max(ny, ~ky);
        xy = max(xy, ky);
    }
    for (int o = 16; o; o >>= 1) {
        na += __shfl_xor_sync(0xffffffffu, na, o);
        nb += __shfl_xor_sync(0xffffffffu, nb, o);
        nx = max(nx, __shfl_xor_sync(0xffffffffu, nx, o));
        xx = max(xx, __shfl_xor_sync(0xffffffffu, xx, o));
        ny = max(ny, __shfl_xor_sync(0xffffffffu, ny, o));
        xy = max(xy, __shfl_xor_sync(0xffffffffu, xy, o));
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) atomicOr((unsigned long long *)&f[F_UNBALANCED], 1ull);
    if ((threadIdx.x & 31) == 0) {
        unsigned long long *u = reinterpret_cast<unsigned long long *>(f + F_ZSTAT);
        if (na) atomicAdd(&u[0], na);
        if (nb) atomicAdd(&u[1], nb);
        atomicMax(&u[2], nx);
        atomicMax(&u[3], xx);
        atomicMax(&u[4], ny);
        atomicMax(&u[5], xy);
    }
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
        s_last = atomicAdd(reinterpret_cast<unsigned long long *>(&f[F_ZC_TICKET]), 1ull) == gridDim.x - 1;
    __syncthreads();
    if (s_last && threadIdx.x < 8) {
        __threadfence();
        const int slot = threadIdx.x < 2 ? F_K0 + threadIdx.x : F_ZSTAT + threadIdx.x - 2;
        reinterpret_cast<volatile int64_t *>(h)[slot] = reinterpret_cast<volatile int64_t *>(f)[slot];
    }
}

// ------------------------------------------------------------ delta condense

__device__ __forceinline__ double round_half_away(double t) {
    // condensation.py:62-63: np.sign(t) * np.floor(np.abs(t) + 0.5)
    // np.sign: +0.0 for either zero, NaN for NaN
    double sg = t > 0.0 ? 1.0 : (t < 0.0 ? -1.0 : (t == 0.0 ? 0.0 : t));
    return dmul(sg, floor(dadd(fabs(t), 0.5)));
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    // condensation.py:85-89
    x = x + 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void k_init_ranges(int64_t *f) {
    f[F_CELL_MIN + 0] = INT64_MAX;
    f[F_CELL_MIN + 1] = INT64_MIN;
    f[F_CELL_MIN + 2] = INT64_MAX;
    f[F_CELL_MIN + 3] = INT64_MIN;
}

__global__ void k_dc_snap(const double2 *pts, int64_t k, double pitch, longlong2 *cells, int64_t *f) {
    int64_t mnx = INT64_MAX, mxx = INT64_MIN, mny = INT64_MAX, mxy = INT64_MIN;
    int ovf = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = pts[i];
        // snap_points, condensation.py:73-77
        double cx = round_half_away(ddiv(p.x, pitch));
        double cy = round_half_away(ddiv(p.y, pitch));
        if (!(fabs(cx) < 4611686018427387904.0) || !(fabs(cy) < 4611686018427387904.0)) {
            ovf = 1;
            cx = 0.0;
            cy = 0.0;
        }
        long long ix = __double2ll_rz(cx), iy = __double2ll_rz(cy);
        cells[i] = make_longlong2(ix, iy);
        mnx = min(mnx, (int64_t)ix);
        mxx = max(mxx, (int64_t)ix);
        mny = min(mny, (int64_t)iy);
        mxy = max(mxy, (int64_t)iy);
    }
    if (ovf) atomicOr((unsigned long long *)&f[F_OVERFLOW], 1ull);
    // warp reduce then one atomic per warp
    for (int o = 16; o; o >>= 1) {
        mnx = min(mnx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mnx, o));
        mxx = max(mxx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mxx, o));
        mny = min(mny, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mny, o));
        mxy = max(mxy, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mxy, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin((long long *)&f[F_CELL_MIN + 0], (long long)mnx);
        atomicMax((long long *)&f[F_CELL_MIN + 1], (long long)mxx);
        atomicMin((long long *)&f[F_CELL_MIN + 2], (long long)mny);
        atomicMax((long long *)&f[F_CELL_MIN + 3], (long long)mxy);
    }
}

// standalone snap_points (condensation.py:66-77): the snapped coordinates
// fl(cell * pitch) and the int64 cells, with the overflow guard
__global__ void k_snap_points(const double2 *pts, int64_t k, double pitch, double2 *snapped, longlong2 *cells,
                              int64_t *f) {
    int ovf = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        const double cx = round_half_away(ddiv(p.x, pitch));
        const double cy = round_half_away(ddiv(p.y, pitch));
        if (!(fabs(cx) < 4611686018427387904.0) || !(fabs(cy) < 4611686018427387904.0)) ovf = 1;
        snapped[i] = make_double2(dmul(cx, pitch), dmul(cy, pitch));
        cells[i] = make_longlong2(__double2ll_rz(cx), __double2ll_rz(cy));
    }
    if (ovf) atomicOr((unsigned long long *)&f[F_OVERFLOW], 1ull);
}

__global__ void k_dc_keys(const longlong2 *cells, int64_t k, int packed, int64_t mnx, int64_t mny,
                          int by, uint64_t *k0, uint64_t *k1, uint32_t *vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        longlong2 c = cells[i];
        if (packed) {
            k0[i] = (by >= 64 ? 0ull : ((uint64_t)(c.x - mnx) << by)) | (uint64_t)(c.y - mny);
        } else {
            k0[i] = ikey(c.y);  // least significant word first
            k1[i] = ikey(c.x);
        }
        vals[i] = (uint32_t)i;
    }
}

struct DcFlag {
    const longlong2 *cells;
    const uint32_t *v;
    __device__ int64_t operator()(int64_t i) const {
        if (i == 0) return 1;
        longlong2 p = cells[v[i]], q = cells[v[i - 1]];
        return (p.x == q.x && p.y == q.y) ? 0 : 1;
    }
};

__global__ void k_dc_emit(DcFlag f, int64_t k, const int64_t *excl, const int64_t *am_in,
                          const int64_t *bm_in, double pitch, double half_width, uint64_t base,
                          double2 *pts, int64_t *am, int64_t *bm, longlong2 *ncell, long long mny,
                          unsigned *rcnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t fl = f(i);
        int64_t rid = excl[i] + fl - 1;
        uint32_t src = f.v[i];
        if (fl) {
            longlong2 c = f.cells[src];
            // _lattice_offsets, condensation.py:92-102
            uint64_t h1 = splitmix64(base ^ (uint64_t)c.x);
            uint64_t h2 = splitmix64(h1 ^ (uint64_t)c.y);
            uint64_t h3 = splitmix64(h2);
            double u1 = dmul(__ull2double_rn(h2 >> 11), 0x1p-53);
            double u2 = dmul(__ull2double_rn(h3 >> 11), 0x1p-53);
            double o1 = dmul(half_width, dsub(dmul(2.0, u1), 1.0));
            double o2 = dmul(half_width, dsub(dmul(2.0, u2), 1.0));
            // condensation.py:123: cells.astype(f64) * (k*delta) + offsets
            pts[rid] = make_double2(dadd(dmul(__ll2double_rn(c.x), pitch), o1),
                                    dadd(dmul(__ll2double_rn(c.y), pitch), o2));
            if (ncell) {  // the tree's lists: node cell, and the node counted in its row
                ncell[rid] = c;
                atomicAdd(&rcnt[c.y - mny], 1u);
            }
        }
        if (am_in[src]) atomicAdd((unsigned long long *)&am[rid], (unsigned long long)am_in[src]);
        if (bm_in[src]) atomicAdd((unsigned long long *)&bm[rid], (unsigned long long)bm_in[src]);
    }
}

inline unsigned gs(const Ctx &c, int64_t n) { return grid_for(n, 256, 8u * c.sm_count); }
// ---------------------------------------------------------------- the tree's lists from the cell order
//
// The split tree (tree.cu) starts from the nodes sorted by (x, y) and by
// (y, x).  Condensed coordinates are cell * pitch + an offset below pitch / 2
// (k > 1/2), so the x order is the column (cx) order refined inside each
// column, and the y order the row (cy) order refined inside each row:
// delta_condense's output is already in column order, rows are a counting
// sort away, and columns / rows hold a few dozen nodes.  Each segment is sorted
// by one warp in registers on (dkey(coord) with its low 9 bits replaced by the
// node's place in the segment).  A final check demands strictly increasing x
// along the X-list and y along the Y-list (so ties, rounding across cells or
// truncated keys that collide all fail it); then the lists ARE the (x, y) /
// (y, x) orders.  Otherwise (or for a segment over 512 nodes) F_LISTS is set
// and the tree sorts for itself.
constexpr int CL_MAX = 512;

// one warp sorts a segment of <= CL_MAX nodes in registers: E full 64-bit
// dkey(coord) keys per lane with the node's place in the segment alongside
// (element i = lane * E + q), a bitonic network whose stages with partner
// distance >= E are shuffles.  Equal keys may come out in either order: an
// equal pair fails k_cl_check anyway.
template <int E>
__device__ __forceinline__ void cl_sort_segment(const double2 *__restrict__ pts, const uint32_t *__restrict__ ids,
                                                int64_t s, int len, bool by_y, uint32_t *out, int lane) {
    uint64_t v[E];
    uint32_t w[E];
#pragma unroll
    for (int q = 0; q < E; q++) {
        const int i = lane * E + q;
        w[q] = (uint32_t)i;
        if (i < len) {
            const uint32_t id = ids ? ids[s + i] : (uint32_t)(s + i);
            const double2 p = pts[id];
            v[q] = dkey(by_y ? p.y : p.x);
        } else {
            v[q] = ~0ull;
        }
    }
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j; j >>= 1) {
            if (j >= E) {
#pragma unroll
                for (int q = 0; q < E; q++) {
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, v[q], j / E);
                    const uint32_t ow = __shfl_xor_sync(0xffffffffu, w[q], j / E);
                    const int i = lane * E + q;
                    const bool keep_min = ((i & k) == 0) == ((i & j) == 0);
                    const bool take = keep_min ? (o < v[q]) : (o > v[q]);
                    if (take) {
                        v[q] = o;
                        w[q] = ow;
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < E; q++) {
                    if (q & j) continue;
                    const int p = q | j;
                    const bool up = ((lane * E + q) & k) == 0;
                    if ((v[q] > v[p]) == up && v[q] != v[p]) {
                        const uint64_t t = v[q];
                        v[q] = v[p];
                        v[p] = t;
                        const uint32_t tw = w[q];
                        w[q] = w[p];
                        w[p] = tw;
                    }
                }
            }
        }
#pragma unroll
    for (int q = 0; q < E; q++) {
        const int i = lane * E + q;
        if (i < len) out[s + i] = ids ? ids[s + w[q]] : (uint32_t)(s + w[q]);
    }
}

__device__ __forceinline__ void cl_sort_any(const double2 *pts, const uint32_t *ids, int64_t s, int len, bool by_y,
                                            uint32_t *out, int lane, int64_t *f) {
    if (len <= 32) cl_sort_segment<1>(pts, ids, s, len, by_y, out, lane);
    else if (len <= 64) cl_sort_segment<2>(pts, ids, s, len, by_y, out, lane);
    else if (len <= 128) cl_sort_segment<4>(pts, ids, s, len, by_y, out, lane);
    else if (len <= 256) cl_sort_segment<8>(pts, ids, s, len, by_y, out, lane);
    else if (len <= CL_MAX) cl_sort_segment<16>(pts, ids, s, len, by_y, out, lane);
    else if (lane == 0) atomicOr((unsigned long long *)&f[F_LISTS], 4ull);
}

// X-list: every column (a run of equal cx in node order) sorted by x; a warp
// handles the columns that start inside its 32-node chunk
__global__ void __launch_bounds__(256, 3) k_cl_columns(const longlong2 *__restrict__ ncell,
                                                    const double2 *__restrict__ pts, const int64_t *__restrict__ kp,
                                                    uint32_t *xl, int64_t *f) {
    const int64_t K = *kp;
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < K; base += warps * 32) {
        const int64_t p = base + lane;
        const bool start = p < K && (p == 0 || ncell[p].x != ncell[p - 1].x);
        unsigned m = __ballot_sync(0xffffffffu, start);
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            const int64_t s = base + b;
            const long long cx = ncell[s].x;
            int64_t e = s + 1;
            while (true) {  // the column's end: first node of another column
                const int64_t q = e + lane;
                const bool stop = q >= K || ncell[q].x != cx;
                const unsigned sm = __ballot_sync(0xffffffffu, stop);
                if (sm) {
                    e += __ffs(sm) - 1;
                    break;
                }
                e += 32;
                if (e - s > CL_MAX) break;
            }
            cl_sort_any(pts, nullptr, s, (int)((e - s) < (int64_t)(CL_MAX + 1) ? (e - s) : (int64_t)(CL_MAX + 1)), false, xl,
                        lane, f);
        }
    }
}

// Y-list: nodes counted per row, scattered to their row, each row sorted by y
struct RowCnt {
    const unsigned *c;
    int64_t R;
    __device__ int64_t operator()(int64_t i) const { return i < R ? (int64_t)c[i] : 0; }
};
__global__ void k_cl_rowscatter(const longlong2 *__restrict__ ncell, const int64_t *__restrict__ kp, long long mny,
                                const int64_t *__restrict__ rstart, unsigned *rcur, uint32_t *rows) {
    const int64_t K = *kp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
        const long long r = ncell[i].y - mny;
        rows[rstart[r] + atomicAdd(&rcur[r], 1u)] = (uint32_t)i;
    }
}
__global__ void __launch_bounds__(256, 3) k_cl_rows(const double2 *__restrict__ pts, const uint32_t *__restrict__ rows,
                                                 const int64_t *__restrict__ rstart, int64_t R, uint32_t *yl,
                                                 int64_t *f) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += warps) {
        const int64_t s = rstart[r], len = rstart[r + 1] - s;
        if (len > 0)
            cl_sort_any(pts, rows, s, (int)(len < (int64_t)(CL_MAX + 1) ? len : (int64_t)(CL_MAX + 1)), true, yl, lane,
                        f);
    }
}

// strictly increasing x along the X-list and y along the Y-list
__global__ void k_cl_check(const double2 *__restrict__ pts, const int64_t *__restrict__ kp,
                           const uint32_t *__restrict__ xl, const uint32_t *__restrict__ yl, int64_t *f) {
    const int64_t K = *kp;
    int bx = 0, by = 0;
    for (int64_t i = 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K; i += (int64_t)gridDim.x * blockDim.x) {
        bx |= !(dkey(pts[xl[i - 1]].x) < dkey(pts[xl[i]].x));
        by |= !(dkey(pts[yl[i - 1]].y) < dkey(pts[yl[i]].y));
    }
    if (__syncthreads_or(bx) && threadIdx.x == 0) atomicOr((unsigned long long *)&f[F_LISTS], 1ull);
    if (__syncthreads_or(by) && threadIdx.x == 0) atomicOr((unsigned long long *)&f[F_LISTS], 2ull);
}



}  // namespace

int zc_run(Ctx &c, const double2 *d_a, int64_t na, const double2 *d_b, int64_t nb, int64_t *k0,
           int32_t *balanced, bool speculative) {
    const int64_t n = na + nb;
    NodeSet &ns = c.nodes[0];
    ns.abar = -na;
    ns.bbar = nb;
    ns.valid = true;
    c.nodes[1].valid = false;
    ns.stats = false;
    if (n == 0) {
        ns.k = 0;
        *k0 = 0;
        *balanced = 1;
        return W1G_OK;
    }
    uint64_t *hi, *lo;
    uint32_t *vals;
    int64_t *excl;
    W1G_TRY(ensure(c.scr[0], n, &hi));
    W1G_TRY(ensure(c.scr[1], n, &lo));
    W1G_TRY(ensure(c.scr[2], n, &vals));
    W1G_TRY(ensure(c.scr[3], n, &excl));
    double2 *pts;
    int64_t *am, *bm;
    W1G_TRY(ensure(ns.pts, n, &pts));
    W1G_TRY(ensure(ns.am, n, &am));
    W1G_TRY(ensure(ns.bm, n, &bm));
    W1G_TRY(flags_reset(c));
    k_zc_keys<<<gs(c, n), 256, 0, c.stream>>>(d_a, na, d_b, n, hi, lo, vals);
    W1G_CHECK_LAUNCH();
    // lexicographic (x, y): radix by x, y only where x ties
    // speculative: short tie runs only (no round trip of the sort's own); redone
    // below in the rare case of a long run (many equal x, e.g. births all 0)
    W1G_TRY(sort_lex2(c, hi, lo, vals, n, speculative));
    ZcFlag f{d_a, d_b, na, vals};
    W1G_TRY(scan_i64(c, f, n, excl, dflags(c) + F_K0));
    W1G_CUDA(cudaMemsetAsync(am, 0, sizeof(int64_t) * n, c.stream));
    W1G_CUDA(cudaMemsetAsync(bm, 0, sizeof(int64_t) * n, c.stream));
    k_zc_emit<<<gs(c, n), 256, 0, c.stream>>>(f, n, excl, pts, am, bm);
    W1G_CHECK_LAUNCH();
    k_zc_stats<<<grid_for(n, 256, 2u * c.sm_count), 256, 0, c.stream>>>(am, bm, pts, dflags(c) + F_K0, dflags(c),
                                                                        c.h_pinned);
    W1G_CHECK_LAUNCH();
    W1G_TRY(stream_sync(c));
    if (speculative && lex2_speculation_failed(c, 1)) return zc_run(c, d_a, na, d_b, nb, k0, balanced, false);
    ns.k = c.h_pinned[F_K0];
    *k0 = ns.k;
    *balanced = c.h_pinned[F_UNBALANCED] ? 0 : 1;
    ns.stats = true;
    ns.nmem[0] = c.h_pinned[F_ZSTAT + 0];
    ns.nmem[1] = c.h_pinned[F_ZSTAT + 1];
    ns.bbox_key[0] = ~(uint64_t)c.h_pinned[F_ZSTAT + 2];
    ns.bbox_key[1] = (uint64_t)c.h_pinned[F_ZSTAT + 3];
    ns.bbox_key[2] = ~(uint64_t)c.h_pinned[F_ZSTAT + 4];
    ns.bbox_key[3] = (uint64_t)c.h_pinned[F_ZSTAT + 5];
    return W1G_OK;
}

struct MassFlag {
    const int64_t *m;
    __device__ int64_t operator()(int64_t i) const { return m[i] > 0 ? 1 : 0; }
};

// exclusive positions of the a- and b-mass nodes (totals -> flags F_MISC0 / F_MISC1)
static int member_scans(Ctx &c, NodeSet &ns, int64_t k) {
    int64_t *exa, *exb;
    W1G_TRY(ensure(ns.exa, (size_t)k + 1, &exa));
    W1G_TRY(ensure(ns.exb, (size_t)k + 1, &exb));
    W1G_TRY(scan_i64(c, MassFlag{ptr<int64_t>(ns.am)}, k, exa, dflags(c) + F_MISC0));
    W1G_TRY(scan_i64(c, MassFlag{ptr<int64_t>(ns.bm)}, k, exb, dflags(c) + F_MISC1));
    return W1G_OK;
}

namespace {
__global__ void k_raw_nodes(const double2 *a, int64_t na, const double2 *b, int64_t n, double2 *pts, int64_t *am,
                            int64_t *bm) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const bool in_a = i < na;
        pts[i] = in_a ? a[i] : b[i - na];
        am[i] = in_a ? 1 : 0;
        bm[i] = in_a ? 0 : 1;
    }
}
}  // namespace

// condensation.py:105-124 only sees the node SET with its summed masses:
// every duplicate point lands in the same cell, so delta_condense of the raw
// diagrams (unit masses) equals delta_condense of zero_condense's output --
// same cells, same order, same offsets, same integer mass sums
int raw_nodes(Ctx &c, const double2 *d_a, int64_t na, const double2 *d_b, int64_t nb) {
    NodeSet &r = c.raw;
    const int64_t n = na + nb;
    double2 *pts;
    int64_t *am, *bm;
    W1G_TRY(ensure(r.pts, (size_t)n + 1, &pts));
    W1G_TRY(ensure(r.am, (size_t)n + 1, &am));
    W1G_TRY(ensure(r.bm, (size_t)n + 1, &bm));
    if (n) {
        k_raw_nodes<<<gs(c, n), 256, 0, c.stream>>>(d_a, na, d_b, n, pts, am, bm);
        W1G_CHECK_LAUNCH();
    }
    r.k = n;
    r.abar = -na;
    r.bbar = nb;
    r.valid = true;
    r.na = r.nb = -1;
    return W1G_OK;
}

int dc_run(Ctx &c, double delta, double pitch, double half_width, uint64_t seed, int64_t *kout,
           NodeSet *src_override) {
    NodeSet &src = src_override ? *src_override : c.nodes[0], &dst = c.nodes[1];
    const int64_t k = src.k;
    c.pre_n = 0;
    dst.abar = src.abar;
    dst.bbar = src.bbar;
    if (delta == 0.0 || k == 0) {
        // condensation.py:111-112: identity
        double2 *p;
        int64_t *a, *b;
        W1G_TRY(ensure(dst.pts, k, &p));
        W1G_TRY(ensure(dst.am, k, &a));
        W1G_TRY(ensure(dst.bm, k, &b));
        if (k) {
            W1G_CUDA(cudaMemcpyAsync(p, src.pts.p, sizeof(double2) * k, cudaMemcpyDeviceToDevice, c.stream));
            W1G_CUDA(cudaMemcpyAsync(a, src.am.p, sizeof(int64_t) * k, cudaMemcpyDeviceToDevice, c.stream));
            W1G_CUDA(cudaMemcpyAsync(b, src.bm.p, sizeof(int64_t) * k, cudaMemcpyDeviceToDevice, c.stream));
        }
        dst.k = k;
        dst.valid = true;
        W1G_TRY(member_scans(c, dst, k));
        W1G_TRY(flags_fetch(c, F_MISC0, 2));
        dst.na = c.h_pinned[F_MISC0];
        dst.nb = c.h_pinned[F_MISC1];
        *kout = k;
        return W1G_OK;
    }
    longlong2 *cells;
    uint64_t *k0, *k1;
    uint32_t *vals;
    int64_t *excl;
    W1G_TRY(ensure(c.scr[4], k, &cells));
    W1G_TRY(ensure(c.scr[0], k, &k0));
    W1G_TRY(ensure(c.scr[1], k, &k1));
    W1G_TRY(ensure(c.scr[2], k, &vals));
    W1G_TRY(ensure(c.scr[3], k, &excl));
    W1G_TRY(flags_reset(c));
    k_init_ranges<<<1, 1, 0, c.stream>>>(dflags(c));
    // few CTAs: the range is reduced per warp and merged with global atomics
    k_dc_snap<<<grid_for(k, 256, 2u * c.sm_count), 256, 0, c.stream>>>(ptr<double2>(src.pts), k, pitch, cells,
                                                                      dflags(c));
    W1G_CHECK_LAUNCH();
    W1G_TRY(flags_fetch(c, 0, F_CELL_MIN + 4));
    if (c.h_pinned[F_OVERFLOW]) {
        set_error("lattice pitch too small for the coordinate range");
        return W1G_EOVERFLOW;
    }
    const int64_t mnx = c.h_pinned[F_CELL_MIN + 0], mxx = c.h_pinned[F_CELL_MIN + 1];
    const int64_t mny = c.h_pinned[F_CELL_MIN + 2], mxy = c.h_pinned[F_CELL_MIN + 3];
    const uint64_t sx = (uint64_t)(mxx - mnx), sy = (uint64_t)(mxy - mny);
    const int bx = sx ? 64 - __builtin_clzll(sx) : 0, by = sy ? 64 - __builtin_clzll(sy) : 0;
    const int packed = (bx + by) <= 64;
    // keys, sort, emit and the tree's lists: one graph (graph_segment) up to the round trip
    bool lists = false;
    W1G_TRY(graph_segment(c, GSEG_DC, [&]() -> int {
        k_dc_keys<<<gs(c, k), 256, 0, c.stream>>>(cells, k, packed, mnx, mny, by, k0, k1, vals);
        W1G_CHECK_LAUNCH();
        uint64_t *keys[2] = {k0, k1};
        W1G_TRY(radix_sort(c, keys, packed ? 1 : 2, vals, k, packed ? (bx + by > 0 ? bx + by : 1) : 64));
        DcFlag f{cells, vals};
        W1G_TRY(scan_i64(c, f, k, excl, dflags(c) + F_TOTAL));
        double2 *pts;
        int64_t *am, *bm;
        W1G_TRY(ensure(dst.pts, k, &pts));
        W1G_TRY(ensure(dst.am, k, &am));
        W1G_TRY(ensure(dst.bm, k, &bm));
        W1G_CUDA(cudaMemsetAsync(am, 0, sizeof(int64_t) * k, c.stream));
        W1G_CUDA(cudaMemsetAsync(bm, 0, sizeof(int64_t) * k, c.stream));
        // base = splitmix64(seed & 0xFFFF_FFFF_FFFF_FFFF), condensation.py:96 (host, same arithmetic)
        uint64_t x = seed + 0x9E3779B97F4A7C15ull;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        const uint64_t base = x ^ (x >> 31);
        // the split tree's X- / Y-lists from the cell order (k_cl_columns), while the
        // row range allows a counting sort (W1G_DC_LISTS=0: the tree sorts itself)
        const bool lists_env = [] {  // read per call (tests toggle it)
            const char *e = getenv("W1G_DC_LISTS");
            return !(e && *e == '0');
        }();
        const int64_t R = (int64_t)(mxy - mny) + 1;
        lists = lists_env && k >= 2 && R > 0 && R <= 4 * k + 1024;
        longlong2 *ncell = nullptr;
        unsigned *rcnt = nullptr;
        bool members_done = false;
        if (lists) {
            W1G_TRY(ensure(c.pre_cells, (size_t)k, &ncell));
            W1G_TRY(ensure(c.pre_rcnt, (size_t)2 * (R + 2), &rcnt));
            W1G_CUDA(cudaMemsetAsync(rcnt, 0, sizeof(unsigned) * 2 * (R + 2), c.stream));
        }
        k_dc_emit<<<gs(c, k), 256, 0, c.stream>>>(f, k, excl, ptr<int64_t>(src.am), ptr<int64_t>(src.bm),
                                                  pitch, half_width, base, pts, am, bm, ncell, mny, rcnt);
        W1G_CHECK_LAUNCH();
        if (lists) {
            SubTimer T(c, "dc_lists");
            uint32_t *xl, *yl, *rows;
            int64_t *rstart;
            W1G_TRY(ensure(c.pre_xl, (size_t)k, &xl));
            W1G_TRY(ensure(c.pre_yl, (size_t)k, &yl));
            W1G_TRY(ensure(c.pre_rows, (size_t)k, &rows));
            W1G_TRY(ensure(c.scr[1], (size_t)R + 2, &rstart));  // the sort keys are dead by now
            const int64_t *dK = dflags(c) + F_TOTAL;
            const unsigned gk = grid_for(k, 256, 8u * c.sm_count);
            // the columns (X-list) and the member scans on the side stream, concurrently with the
            // rows' bucketing and sort; everything they use is allocated (on the main stream) first
            cudaStream_t side = c.copy_stream ? c.copy_stream : c.stream;
            int64_t *exa_, *exb_;
            unsigned long long *st2;
            W1G_TRY(ensure(dst.exa, (size_t)k + 1, &exa_));
            W1G_TRY(ensure(dst.exb, (size_t)k + 1, &exb_));
            W1G_TRY(ensure(c.scan_state2, (size_t)((k + SCAN_TILE - 1) / SCAN_TILE) + 16, &st2));
            if (side != c.stream) {
                W1G_CUDA(cudaEventRecord(c.ev[14], c.stream));
                W1G_CUDA(cudaStreamWaitEvent(side, c.ev[14], 0));
            }
            k_cl_columns<<<gk, 256, 0, side>>>(ncell, pts, dK, xl, dflags(c));
            W1G_CHECK_LAUNCH();
            if (side != c.stream) {
                // member_scans on the side stream with its own scan state
                std::swap(c.stream, side);
                std::swap(c.scan_state, c.scan_state2);
                const int rc = member_scans(c, dst, k);
                std::swap(c.scan_state, c.scan_state2);
                std::swap(c.stream, side);
                W1G_TRY(rc);
                members_done = true;
                W1G_CUDA(cudaEventRecord(c.ev[15], side));
            }
            T.mark("columns");
            W1G_TRY(scan_i64(c, RowCnt{rcnt, R}, R + 1, rstart, nullptr));
            k_cl_rowscatter<<<gk, 256, 0, c.stream>>>(ncell, dK, mny, rstart, rcnt + R + 2, rows);
            W1G_CHECK_LAUNCH();
            T.mark("row_bucket");
            k_cl_rows<<<grid_for(R * 32, 256, 8u * c.sm_count), 256, 0, c.stream>>>(pts, rows, rstart, R, yl, dflags(c));
            W1G_CHECK_LAUNCH();
            T.mark("rows");
            if (side != c.stream) W1G_CUDA(cudaStreamWaitEvent(c.stream, c.ev[15], 0));
            k_cl_check<<<grid_for(k, 256, 2u * c.sm_count), 256, 0, c.stream>>>(pts, dK, xl, yl, dflags(c));
            W1G_CHECK_LAUNCH();
            T.mark("check");
        }
        // node positions per side for emit_arcs, over k >= K (the masses past K are 0),
        // so their totals come back with K in the same round trip
        if (!members_done) W1G_TRY(member_scans(c, dst, k));
        if (lists) {
            W1G_TRY(to_host_small2(c, c.h_pinned + F_LISTS, dflags(c) + F_LISTS, sizeof(int64_t), c.h_pinned + F_TOTAL,
                                   dflags(c) + F_TOTAL, sizeof(int64_t) * (F_MISC1 - F_TOTAL + 1)));
        } else {
            W1G_TRY(to_host_small(c, c.h_pinned + F_TOTAL, dflags(c) + F_TOTAL, sizeof(int64_t) * (F_MISC1 - F_TOTAL + 1)));
        }
        return W1G_OK;
    }));
    W1G_TRY(stream_sync(c));
    dst.k = c.h_pinned[F_TOTAL];
    dst.na = c.h_pinned[F_MISC0];
    dst.nb = c.h_pinned[F_MISC1];
    dst.valid = true;
    if (lists && !c.h_pinned[F_LISTS]) c.pre_n = dst.k;
    *kout = dst.k;
    return W1G_OK;
}

int snap_run(Ctx &c, const double *h_pts, int64_t k, double pitch, double *h_snapped, int64_t *h_cells) {
    double2 *pts, *snapped;
    longlong2 *cells;
    W1G_TRY(ensure(c.scr[0], (size_t)k + 1, &pts));
    W1G_TRY(ensure(c.scr[1], (size_t)k + 1, &snapped));
    W1G_TRY(ensure(c.scr[2], (size_t)k + 1, &cells));
    W1G_TRY(flags_reset(c));
    if (k) {
        W1G_CUDA(cudaMemcpyAsync(pts, h_pts, sizeof(double2) * k, cudaMemcpyHostToDevice, c.stream));
        k_snap_points<<<grid_for(k, 256, 8u * c.sm_count), 256, 0, c.stream>>>(pts, k, pitch, snapped, cells,
                                                                              dflags(c));
        W1G_CHECK_LAUNCH();
    }
    W1G_TRY(flags_fetch(c, F_OVERFLOW, 1));
    if (c.h_pinned[F_OVERFLOW]) {
        set_error("lattice pitch too small for the coordinate range");
        return W1G_EOVERFLOW;
    }
    if (k) {
        if (h_snapped)
            W1G_CUDA(cudaMemcpyAsync(h_snapped, snapped, sizeof(double2) * k, cudaMemcpyDeviceToHost, c.stream));
        if (h_cells) W1G_CUDA(cudaMemcpyAsync(h_cells, cells, sizeof(longlong2) * k, cudaMemcpyDeviceToHost, c.stream));
        W1G_TRY(stream_sync(c));
    }
    return W1G_OK;
}

}  // namespace w1g
