// rwmd.cu -- relaxed Wasserstein lower bound (lower_bound.py:43-75) on device.
//
// For each side X in {A, B}: sources are the nodes with X-mass > 0, targets
// the nodes with other-side mass > 0 (lower_bound.py:73-74).  The reference
// value per source is best = min(sqrt(min_j fl(fl(dx^2)+fl(dy^2))), diag)
// (cKDTree distance, np.minimum) and L_X = np.sum(mass * best) in node order.
//
//  1. FP32 all-pairs tile pass (rwmd_tile.cu) gives every source an
//     approximate squared NN distance with a rigorous error bound;
//  2. an exact fp64 pass scans only the targets inside that bound (uniform
//     cell grid over the targets, counting-sorted on device) and computes
//     the reference's exact IEEE distance, then mass * best;
//  3. numpy's pairwise summation tree (loops_utils.h.src pairwise_sum) is
//     rebuilt level by level on device and evaluated leaf-first, so L_X is
//     bit-identical to np.sum.
#include <cmath>

#include "common.cuh"

namespace w1g {

int rwmd_f32_min(Ctx &c, const float2 *q, int64_t nq, const float2 *t, int64_t nt, unsigned *mout,
                 int culling);

static const double SQRT2 = 1.4142135623730951;  // math.sqrt(2.0), diagram.py:17

namespace {

struct MemberFlag {
    const int64_t *mass;
    __device__ int64_t operator()(int64_t i) const { return mass[i] > 0 ? 1 : 0; }
};

__global__ void k_compact(const int64_t *mass, int64_t k, const int64_t *excl, int32_t *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x)
        if (mass[i] > 0) out[excl[i]] = (int32_t)i;
}

__global__ void k_bbox(const double2 *pts, int64_t k, int64_t *f) {
    uint64_t mnx = ~0ull, mxx = 0, mny = ~0ull, mxy = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = pts[i];
        uint64_t kx = dkey(p.x), ky = dkey(p.y);
        mnx = min(mnx, kx);
        mxx = max(mxx, kx);
        mny = min(mny, ky);
        mxy = max(mxy, ky);
    }
    for (int o = 16; o; o >>= 1) {
        mnx = min(mnx, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mnx, o));
        mxx = max(mxx, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mxx, o));
        mny = min(mny, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mny, o));
        mxy = max(mxy, (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)mxy, o));
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned long long *u = (unsigned long long *)f;
        atomicMin(&u[F_BBOX + 0], (unsigned long long)mnx);
        atomicMax(&u[F_BBOX + 1], (unsigned long long)mxx);
        atomicMin(&u[F_BBOX + 2], (unsigned long long)mny);
        atomicMax(&u[F_BBOX + 3], (unsigned long long)mxy);
    }
}

__global__ void k_bbox_init(int64_t *f) {
    unsigned long long *u = (unsigned long long *)f;
    u[F_BBOX + 0] = ~0ull;
    u[F_BBOX + 1] = 0;
    u[F_BBOX + 2] = ~0ull;
    u[F_BBOX + 3] = 0;
}

__global__ void k_to_f32(const double2 *pts, const int32_t *idx, int64_t n, double cx, double cy,
                         double scale, float2 *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = pts[idx[i]];
        out[i] = make_float2((float)((p.x - cx) * scale), (float)((p.y - cy) * scale));
    }
}

struct Grid {
    double x0, y0, inv_c;
    int gx, gy;
};

__device__ __forceinline__ int cell_coord(double v, double v0, double inv_c, int g) {
    double f = floor((v - v0) * inv_c);
    if (!(f >= 0.0)) f = 0.0;
    if (f > (double)(g - 1)) f = (double)(g - 1);
    return (int)f;
}

__global__ void k_cell_count(const double2 *pts, const int32_t *idx, int64_t n, Grid g,
                             int32_t *cell, int64_t *counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = pts[idx[i]];
        int c = cell_coord(p.y, g.y0, g.inv_c, g.gy) * g.gx + cell_coord(p.x, g.x0, g.inv_c, g.gx);
        cell[i] = c;
        atomicAdd((unsigned long long *)&counts[c], 1ull);
    }
}

struct CountVal {
    const int64_t *counts;
    __device__ int64_t operator()(int64_t i) const { return counts[i]; }
};

__global__ void k_cell_fill(const double2 *pts, const int32_t *idx, int64_t n, const int32_t *cell,
                            int64_t *cursor, double2 *sorted) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t pos = (int64_t)atomicAdd((unsigned long long *)&cursor[cell[i]], 1ull);
        sorted[pos] = pts[idx[i]];
    }
}

// exact fp64 refinement + mass * best (lower_bound.py:51-58)
__global__ void __launch_bounds__(128) k_refine(const double2 *pts, const int32_t *src_idx,
                                                const int64_t *mass, int64_t ns, const unsigned *mf32,
                                                int has_targets, double unscale, Grid g,
                                                const int64_t *cell_start, const double2 *tsorted,
                                                double *best_out, double *terms) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t node = src_idx[i];
        const double2 q = pts[node];
        const double diag = ddiv(fabs(dsub(q.y, q.x)), SQRT2);  // diagram.py:47
        double best = diag;
        if (has_targets) {
            // FP32 bound: |d_f32 - d| <= 2^-21 (1 + d) in scaled units; use 2^-19
            const double df = sqrt((double)__uint_as_float(mf32[i]));
            const double lo = (df - 0x1p-19) * (1.0 - 0x1p-19) * unscale;
            if (!(lo > diag * (1.0 + 1e-12))) {
                const double R = (df + 0x1p-19) * (1.0 + 0x1p-19) * unscale * (1.0 + 1e-12);
                const int cx0 = cell_coord(q.x - R, g.x0, g.inv_c, g.gx) - 1;
                const int cx1 = cell_coord(q.x + R, g.x0, g.inv_c, g.gx) + 1;
                const int cy0 = cell_coord(q.y - R, g.y0, g.inv_c, g.gy) - 1;
                const int cy1 = cell_coord(q.y + R, g.y0, g.inv_c, g.gy) + 1;
                double m2 = INFINITY;
                for (int cy = max(cy0, 0); cy <= min(cy1, g.gy - 1); cy++) {
                    const int64_t rs = cell_start[(int64_t)cy * g.gx + max(cx0, 0)];
                    const int64_t re = cell_start[(int64_t)cy * g.gx + min(cx1, g.gx - 1) + 1];
                    for (int64_t p = rs; p < re; p++) {
                        const double2 t = tsorted[p];
                        const double dx = dsub(q.x, t.x), dy = dsub(q.y, t.y);
                        const double d2 = dadd(dmul(dx, dx), dmul(dy, dy));
                        m2 = d2 < m2 ? d2 : m2;
                    }
                }
                const double nnd = dsqrt(m2);
                best = nnd < diag ? nnd : diag;  // np.minimum(nnd, diag)
            }
        }
        best_out[i] = best;
        terms[i] = dmul(__ll2double_rn(mass[node]), best);  // float64(src_mass) * best
    }
}

// ---------------------------------------------------------------- numpy pairwise sum
struct PwNode {
    int64_t start, len;
    int32_t child;  // index of the left child (right = child + 1); -1 for a leaf
    int32_t pad;
};
constexpr int PW_MAX_LEVELS = 64;

__global__ void __launch_bounds__(1024) k_pw_build(int64_t n, PwNode *nodes, int32_t *levels,
                                                   int32_t *n_levels) {
    __shared__ int32_t s_warp[32];
    __shared__ int32_t s_base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        nodes[0].start = 0;
        nodes[0].len = n;
        levels[0] = 0;
        levels[1] = 1;
    }
    __syncthreads();
    int lo = 0, hi = 1, L = 0;
    while (lo < hi && L < PW_MAX_LEVELS - 2) {
        if (threadIdx.x == 0) s_base = 0;
        __syncthreads();
        for (int chunk = lo; chunk < hi; chunk += 1024) {
            const int i = chunk + threadIdx.x;
            const bool valid = i < hi;
            const bool internal = valid && nodes[i].len > 128;
            int cnt = internal ? 2 : 0;
            int x = cnt;
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_warp[wid] = x;
            __syncthreads();
            if (wid == 0) {
                int w = s_warp[lane];
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, w, o);
                    if (lane >= o) w += y;
                }
                s_warp[lane] = w;
            }
            __syncthreads();
            const int off = s_base + (wid ? s_warp[wid - 1] : 0) + x - cnt;
            if (valid) {
                if (internal) {
                    const int64_t len = nodes[i].len, st = nodes[i].start;
                    int64_t n2 = len / 2;
                    n2 -= n2 % 8;
                    const int child = hi + off;
                    nodes[child].start = st;
                    nodes[child].len = n2;
                    nodes[child + 1].start = st + n2;
                    nodes[child + 1].len = len - n2;
                    nodes[i].child = child;
                } else {
                    nodes[i].child = -1;
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) s_base += s_warp[31];
            __syncthreads();
        }
        const int nb = s_base;
        lo = hi;
        hi = hi + nb;
        L++;
        if (threadIdx.x == 0) levels[L + 1] = hi;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_levels = L;
}

// one warp per leaf: numpy's 8-accumulator block (n <= 128) or sequential (n < 8)
__global__ void k_pw_leaves(const double *v, const PwNode *nodes, const int32_t *levels,
                            const int32_t *n_levels, double *val) {
    const int total = levels[*n_levels];
    const int lane = threadIdx.x & 31;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total;
         i += (gridDim.x * blockDim.x) >> 5) {
        const PwNode nd = nodes[i];
        if (nd.child >= 0) continue;
        const double *a = v + nd.start;
        const int64_t len = nd.len;
        if (len < 8) {
            if (lane == 0) {
                double res = 0.0;
                for (int64_t j = 0; j < len; j++) res = dadd(res, a[j]);
                val[i] = res;
            }
            continue;
        }
        double r = 0.0;
        if (lane < 8) {
            r = a[lane];
            for (int64_t j = 8; j < len - (len % 8); j += 8) r = dadd(r, a[j + lane]);
        }
        double r0 = __shfl_sync(0xffffffffu, r, 0), r1 = __shfl_sync(0xffffffffu, r, 1);
        double r2 = __shfl_sync(0xffffffffu, r, 2), r3 = __shfl_sync(0xffffffffu, r, 3);
        double r4 = __shfl_sync(0xffffffffu, r, 4), r5 = __shfl_sync(0xffffffffu, r, 5);
        double r6 = __shfl_sync(0xffffffffu, r, 6), r7 = __shfl_sync(0xffffffffu, r, 7);
        if (lane == 0) {
            double res = dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
            for (int64_t j = len - (len % 8); j < len; j++) res = dadd(res, a[j]);
            val[i] = res;
        }
    }
}

__global__ void __launch_bounds__(1024) k_pw_combine(const PwNode *nodes, const int32_t *levels,
                                                     const int32_t *n_levels, double *val,
                                                     double *out) {
    const int L = *n_levels;
    for (int l = L - 1; l >= 0; l--) {
        for (int i = levels[l] + threadIdx.x; i < levels[l + 1]; i += blockDim.x) {
            const int ch = nodes[i].child;
            if (ch >= 0) val[i] = dadd(val[ch], val[ch + 1]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = val[0];
}

}  // namespace

// np.sum of a contiguous float64 vector on device -> *d_out (device)
int pairwise_sum(Ctx &c, const double *d_v, int64_t n, double *d_out, DevBuf &nodes_buf,
                 DevBuf &val_buf, DevBuf &lev_buf) {
    if (n == 0) {
        W1G_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), c.stream));
        return W1G_OK;
    }
    const int64_t cap = n / 32 + 64;
    PwNode *nodes;
    double *val;
    int32_t *lev;
    W1G_TRY(ensure(nodes_buf, (size_t)cap, &nodes));
    W1G_TRY(ensure(val_buf, (size_t)cap, &val));
    W1G_TRY(ensure(lev_buf, PW_MAX_LEVELS + 2, &lev));
    k_pw_build<<<1, 1024, 0, c.stream>>>(n, nodes, lev, lev + PW_MAX_LEVELS);
    W1G_CHECK_LAUNCH();
    const unsigned warps = (unsigned)(n / 64 + 2);
    k_pw_leaves<<<grid_for(warps * 32, 256, 4u * c.sm_count), 256, 0, c.stream>>>(d_v, nodes, lev, lev + PW_MAX_LEVELS, val);
    W1G_CHECK_LAUNCH();
    k_pw_combine<<<1, 1024, 0, c.stream>>>(nodes, lev, lev + PW_MAX_LEVELS, val, d_out);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

static inline double key_to_double(uint64_t k) {
    uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}

int rwmd_run(Ctx &c, double *L, double *LA, double *LB) {
    NodeSet &ns = c.nodes[0];
    const int64_t k = ns.k;
    const double2 *pts = ptr<double2>(ns.pts);
    const int64_t *mass[2] = {ptr<int64_t>(ns.am), ptr<int64_t>(ns.bm)};
    if (k == 0) {
        *L = *LA = *LB = 0.0;
        c.n_best[0] = c.n_best[1] = 0;
        return W1G_OK;
    }
    int64_t *excl;
    int32_t *members[2];
    W1G_TRY(ensure(c.scr[3], k, &excl));
    W1G_TRY(ensure(c.scr[5], k, &members[0]));
    W1G_TRY(ensure(c.scr[6], k, &members[1]));
    W1G_TRY(flags_reset(c));
    const unsigned g = grid_for(k, 256, 8u * c.sm_count);
    for (int s = 0; s < 2; s++) {
        W1G_TRY(scan_i64(c, MemberFlag{mass[s]}, k, excl, dflags(c) + F_MISC0 + s));
        k_compact<<<g, 256, 0, c.stream>>>(mass[s], k, excl, members[s]);
        W1G_CHECK_LAUNCH();
    }
    k_bbox_init<<<1, 1, 0, c.stream>>>(dflags(c));
    k_bbox<<<g, 256, 0, c.stream>>>(pts, k, dflags(c));
    W1G_CHECK_LAUNCH();
    W1G_TRY(flags_fetch(c, 0, F_BBOX + 4));
    const int64_t nm[2] = {c.h_pinned[F_MISC0], c.h_pinned[F_MISC1]};
    c.rw_members[0] = nm[0];
    c.rw_members[1] = nm[1];
    const double xmin = key_to_double((uint64_t)c.h_pinned[F_BBOX + 0]);
    const double xmax = key_to_double((uint64_t)c.h_pinned[F_BBOX + 1]);
    const double ymin = key_to_double((uint64_t)c.h_pinned[F_BBOX + 2]);
    const double ymax = key_to_double((uint64_t)c.h_pinned[F_BBOX + 3]);
    // scaled FP32 frame: |x'| < 1 with a power-of-two scale (exact in fp64)
    const double cx = 0.5 * (xmin + xmax), cy = 0.5 * (ymin + ymax);
    double H = std::fmax(std::fmax(xmax - cx, cx - xmin), std::fmax(ymax - cy, cy - ymin));
    int e = 0;
    if (H > 0.0 && std::isfinite(H)) e = std::ilogb(H) + 1;
    const double scale = std::ldexp(1.0, -e), unscale = std::ldexp(1.0, e);

    float2 *f32[2];
    W1G_TRY(ensure(c.scr[7], nm[0], &f32[0]));
    W1G_TRY(ensure(c.scr[8], nm[1], &f32[1]));
    for (int s = 0; s < 2; s++) {
        if (nm[s] == 0) continue;
        k_to_f32<<<grid_for(nm[s], 256, 8u * c.sm_count), 256, 0, c.stream>>>(pts, members[s], nm[s], cx, cy,
                                                                             scale, f32[s]);
        W1G_CHECK_LAUNCH();
    }
    double *terms, *dres;
    W1G_TRY(ensure(c.scr[9], (size_t)(nm[0] > nm[1] ? nm[0] : nm[1]) + 1, &terms));
    W1G_TRY(ensure(c.scr[10], 4, &dres));
    for (int s = 0; s < 2; s++) {
        const int o = 1 - s;
        const int64_t n_src = nm[s], n_dst = nm[o];
        c.n_best[s] = n_src;
        double *best;
        W1G_TRY(ensure(c.best[s], (size_t)n_src + 1, &best));
        if (n_src == 0) {
            W1G_CUDA(cudaMemsetAsync(dres + s, 0, sizeof(double), c.stream));
            continue;
        }
        unsigned *mf = nullptr;
        Grid gr{0, 0, 1, 1, 1};
        int64_t *cell_start = nullptr;
        double2 *tsorted = nullptr;
        if (n_dst > 0) {
            W1G_TRY(ensure(c.scr[11], (size_t)n_src, &mf));
            W1G_CUDA(cudaMemsetAsync(mf, 0x7f, sizeof(unsigned) * n_src, c.stream));
            W1G_TRY(rwmd_f32_min(c, f32[s], n_src, f32[o], n_dst, mf, c.culling));
            // uniform grid over the targets, ~4 targets per cell on average
            const double W = xmax - xmin, Hh = ymax - ymin;
            double cs;
            if (W > 0 && Hh > 0)
                cs = std::sqrt(W * Hh / (4.0 * (double)n_dst));
            else
                cs = std::fmax(W, Hh) / (4.0 * (double)n_dst);
            if (!(cs > 0.0) || !std::isfinite(cs)) cs = 1.0;
            double gxf = std::floor(W / cs) + 1, gyf = std::floor(Hh / cs) + 1;
            while (gxf * gyf > (double)(1 << 26)) {
                cs *= 1.5;
                gxf = std::floor(W / cs) + 1;
                gyf = std::floor(Hh / cs) + 1;
            }
            gr.x0 = xmin;
            gr.y0 = ymin;
            gr.inv_c = 1.0 / cs;
            gr.gx = (int)gxf;
            gr.gy = (int)gyf;
            const int64_t ncell = (int64_t)gr.gx * gr.gy;
            int32_t *cell;
            int64_t *counts, *cursor;
            W1G_TRY(ensure(c.scr[12], (size_t)n_dst, &cell));
            W1G_TRY(ensure(c.scr[13], (size_t)ncell + 1, &counts));
            W1G_TRY(ensure(c.scr[14], (size_t)ncell + 1, &cell_start));
            W1G_TRY(ensure(c.scr[15], (size_t)ncell + 1, &cursor));
            W1G_TRY(ensure(c.scr[16], (size_t)n_dst, &tsorted));
            W1G_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * (ncell + 1), c.stream));
            const unsigned gd = grid_for(n_dst, 256, 8u * c.sm_count);
            k_cell_count<<<gd, 256, 0, c.stream>>>(pts, members[o], n_dst, gr, cell, counts);
            W1G_CHECK_LAUNCH();
            W1G_TRY(scan_i64(c, CountVal{counts}, ncell + 1, cell_start, nullptr));
            W1G_CUDA(cudaMemcpyAsync(cursor, cell_start, sizeof(int64_t) * ncell, cudaMemcpyDeviceToDevice, c.stream));
            k_cell_fill<<<gd, 256, 0, c.stream>>>(pts, members[o], n_dst, cell, cursor, tsorted);
            W1G_CHECK_LAUNCH();
        }
        k_refine<<<grid_for(n_src, 128, 16u * c.sm_count), 128, 0, c.stream>>>(
            pts, members[s], mass[s], n_src, mf, n_dst > 0, unscale, gr, cell_start, tsorted, best, terms);
        W1G_CHECK_LAUNCH();
        W1G_TRY(pairwise_sum(c, terms, n_src, dres + s, c.scr[17], c.scr[18], c.scr[19]));
    }
    double h[2];
    W1G_CUDA(cudaMemcpyAsync(h, dres, sizeof(double) * 2, cudaMemcpyDeviceToHost, c.stream));
    W1G_CUDA(cudaStreamSynchronize(c.stream));
    *LA = h[0];
    *LB = h[1];
    *L = h[1] > h[0] ? h[1] : h[0];  // python max(l_a, l_b)
    return W1G_OK;
}

// measurement hook (w1g_profile_rwmd_tile): the FP32 tile pass alone, both
// directions, `reps` times, timed with events on the context stream
int rwmd_tile_profile(Ctx &c, int reps, float *ms, int64_t *evals) {
    double L, la, lb;
    W1G_TRY(rwmd_run(c, &L, &la, &lb));  // builds the scaled FP32 member arrays
    const int64_t na = c.rw_members[0], nb = c.rw_members[1];
    *evals = na * nb;
    *ms = 0.f;
    if (na == 0 || nb == 0 || reps < 1) return W1G_OK;
    const float2 *fa = ptr<float2>(c.scr[7]), *fb = ptr<float2>(c.scr[8]);
    unsigned *ma, *mb;
    W1G_TRY(ensure(c.scr[11], (size_t)na, &ma));
    W1G_TRY(ensure(c.scr[12], (size_t)nb, &mb));
    W1G_CUDA(cudaEventRecord(c.ev[8], c.stream));
    for (int r = 0; r < reps; r++) {
        W1G_TRY(rwmd_f32_min(c, fa, na, fb, nb, ma, c.culling));
        W1G_TRY(rwmd_f32_min(c, fb, nb, fa, na, mb, c.culling));
    }
    W1G_CUDA(cudaEventRecord(c.ev[9], c.stream));
    W1G_CUDA(cudaEventSynchronize(c.ev[9]));
    float t = 0.f;
    W1G_CUDA(cudaEventElapsedTime(&t, c.ev[8], c.ev[9]));
    *ms = t / (2.0f * reps);
    return W1G_OK;
}

}  // namespace w1g
