// rwmd.cu -- relaxed Wasserstein lower bound (lower_bound.py:43-75) on device.
//
// For each side X in {A, B}: sources are the nodes with X-mass > 0, targets
// the nodes with other-side mass > 0 (lower_bound.py:73-74).  The reference
// value per source is best = min(sqrt(min_j fl(fl(dx^2)+fl(dy^2))), diag)
// (cKDTree distance, np.minimum) and L_X = np.sum(mass * best) in node order.
//
//  1. members of each side are put in Morton order (radix sort of 32-bit
//     codes), so CTAs of sources and tiles of targets are spatially compact;
//  2. the FP32 all-pairs tile pass (rwmd_tile.cu) gives every source a
//     squared-distance estimate with a rigorous error bound -> a radius that
//     provably contains the exact nearest target;
//  3. an exact fp64 pass per source block keeps only the 64-target Morton
//     tiles within that radius (box test) and evaluates the reference's IEEE
//     distance on them, then mass * best in node order;
//  4. numpy's pairwise summation tree (pairwise_sum.cu) makes L_X
//     bit-identical to np.sum.
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace w1g {

int rwmd_f32_min(Ctx &c, const double2 *q, const uint64_t *qkey, int64_t nq, const double2 *t,
                 const uint64_t *tkey, int64_t nt, double scale,
                 unsigned *mout, float *qn_out, double4 *tbox, int culling, int tbox_ready = 0);
int pairwise_sum(Ctx &c, const double *d_v, int64_t n, double *d_out, DevBuf &nodes_buf,
                 DevBuf &val_buf, DevBuf &lev_buf, int64_t *cached_n = nullptr, double *h_out = nullptr);

static const double SQRT2 = 1.4142135623730951;  // math.sqrt(2.0), diagram.py:17

namespace {

constexpr int RT = 64;  // targets per refine tile

struct MemberFlag {
    const int64_t *mass;
    __device__ int64_t operator()(int64_t i) const { return mass[i] > 0 ? 1 : 0; }
};

// both sides' member lists in one launch (after both sides' scans)
__global__ void k_compact2(const int64_t *mass0, const int64_t *mass1, int64_t k, const int64_t *excl0,
                           const int64_t *excl1, int32_t *out0, int32_t *out1) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * k;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool b = i >= k;
        const int64_t j = b ? i - k : i;
        if ((b ? mass1 : mass0)[j] > 0) (b ? out1 : out0)[(b ? excl1 : excl0)[j]] = (int32_t)j;
    }
}

__global__ void k_bbox_init(int64_t *f) {
    unsigned long long *u = (unsigned long long *)f;
    u[F_BBOX + 0] = ~0ull;
    u[F_BBOX + 1] = 0;
    u[F_BBOX + 2] = ~0ull;
    u[F_BBOX + 3] = 0;
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

__device__ __forceinline__ uint32_t spread16(uint32_t v) {
    v &= 0xffff;
    v = (v | (v << 8)) & 0x00ff00ff;
    v = (v | (v << 4)) & 0x0f0f0f0f;
    v = (v | (v << 2)) & 0x33333333;
    v = (v | (v << 1)) & 0x55555555;
    return v;
}

// Morton code on a 4096^2 grid over the node bbox (24-bit keys: three
// radix passes; a finer grid buys nothing at 64-target tiles); payload = member position
constexpr double MORTON_MAX = 4095.0;
constexpr int MORTON_BITS = 24;
// Morton keys of both sides in one launch
struct Morton2 {
    const int32_t *members[2];
    int64_t n[2];
    uint64_t *key[2];
    uint32_t *val[2];
};
__global__ void k_morton2(const double2 *pts, Morton2 M, double x0, double y0, double inv) {
    const int64_t tot = M.n[0] + M.n[1];
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < tot;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int s = g >= M.n[0];
        const int64_t i = s ? g - M.n[0] : g;
        const double2 p = pts[M.members[s][i]];
        double fx = (p.x - x0) * inv, fy = (p.y - y0) * inv;
        fx = fx < 0 ? 0 : (fx > MORTON_MAX ? MORTON_MAX : fx);
        fy = fy < 0 ? 0 : (fy > MORTON_MAX ? MORTON_MAX : fy);
        M.key[s][i] = (uint64_t)(spread16((uint32_t)fx) | (spread16((uint32_t)fy) << 1));
        M.val[s][i] = (uint32_t)i;
    }
}

// both sides' Morton-ordered member points in one launch
struct Gather2 {
    const int32_t *members[2];
    const uint32_t *perm[2];
    int64_t n[2], offset[2];
    double2 *out[2];
    int32_t *pos[2];
};
__global__ void k_gather2(const double2 *pts, Gather2 G) {
    const int64_t tot = G.n[0] + G.n[1];
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < tot;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int s = g >= G.n[0];
        const int64_t i = s ? g - G.n[0] : g;
        const uint32_t m = G.perm[s][i];
        G.out[s][i] = pts[G.members[s][m]];
        G.pos[s][i] = (int32_t)(m + G.offset[s]);
    }
}

__global__ void k_boxes64(const double2 *t, int64_t nt, double4 *box) {
    const int lane = threadIdx.x & 31;
    const int64_t ntile = (nt + RT - 1) / RT;
    for (int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < ntile;
         tile += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
        const int64_t te = min(nt, (tile + 1) * RT);
        for (int64_t j = tile * RT + lane; j < te; j += 32) {
            const double2 p = t[j];
            x0 = fmin(x0, p.x);
            y0 = fmin(y0, p.y);
            x1 = fmax(x1, p.x);
            y1 = fmax(y1, p.y);
        }
        for (int o = 16; o; o >>= 1) {
            x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, o));
            y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, o));
            x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, o));
            y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, o));
        }
        if (lane == 0) box[tile] = make_double4(x0, y0, x1, y1);
    }
}

// super-tile boxes: the union of 64 consecutive refine-tile boxes (4096 targets)
constexpr int SUP = 64;
__global__ void k_superboxes(const double4 *box, int64_t ntile, double4 *sbox) {
    const int lane = threadIdx.x & 31;
    const int64_t nsup = (ntile + SUP - 1) / SUP;
    for (int64_t sp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sp < nsup;
         sp += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
        for (int64_t k = sp * SUP + lane; k < min(ntile, (sp + 1) * SUP); k += 32) {
            const double4 b = box[k];
            x0 = fmin(x0, b.x);
            y0 = fmin(y0, b.y);
            x1 = fmax(x1, b.z);
            y1 = fmax(y1, b.w);
        }
        for (int o = 16; o; o >>= 1) {
            x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, o));
            y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, o));
            x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, o));
            y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, o));
        }
        if (lane == 0) sbox[sp] = make_double4(x0, y0, x1, y1);
    }
}


// the targets' boxes for both sides in one launch: a 128-thread block per 256-target tile (the
// culled FP32 pass's tile, TS_CULL in rwmd_tile.cu), one warp per 64-target refine tile inside it;
// min / max are order-independent, so the boxes equal k_tile_boxes' and k_boxes64's
struct SideBoxes {
    const double2 *t[2];  // side s's targets
    int64_t n[2];
    int64_t nblk0;        // 256-target tiles of side 0
    double4 *tbox[2], *box64[2], *sbox[2];
};
__global__ void __launch_bounds__(128) k_side_boxes(SideBoxes A) {
    __shared__ double4 s_b[4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int s = (int64_t)blockIdx.x >= A.nblk0;
    const int64_t ct = s ? (int64_t)blockIdx.x - A.nblk0 : (int64_t)blockIdx.x;
    const int64_t nt = A.n[s];
    const int64_t k = ct * 4 + w, j0 = k * RT, je = min(nt, j0 + RT);
    double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
    for (int64_t j = j0 + lane; j < je; j += 32) {
        const double2 p = A.t[s][j];
        x0 = fmin(x0, p.x);
        y0 = fmin(y0, p.y);
        x1 = fmax(x1, p.x);
        y1 = fmax(y1, p.y);
    }
    for (int o = 16; o; o >>= 1) {
        x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, o));
        y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, o));
        x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, o));
        y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    if (lane == 0) {
        s_b[w] = make_double4(x0, y0, x1, y1);
        if (j0 < nt) A.box64[s][k] = s_b[w];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double4 b = s_b[0];
        for (int q = 1; q < 4; q++) {
            b.x = fmin(b.x, s_b[q].x);
            b.y = fmin(b.y, s_b[q].y);
            b.z = fmax(b.z, s_b[q].z);
            b.w = fmax(b.w, s_b[q].w);
        }
        A.tbox[s][ct] = b;
    }
}

// both sides' super-tile boxes in one launch (a warp per super-tile, as k_superboxes)
__global__ void k_side_superboxes(SideBoxes A) {
    const int lane = threadIdx.x & 31;
    int64_t ntile[2], nsup[2];
    for (int q = 0; q < 2; q++) {
        ntile[q] = (A.n[q] + RT - 1) / RT;
        nsup[q] = (ntile[q] + SUP - 1) / SUP;
    }
    for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < nsup[0] + nsup[1];
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int s = g >= nsup[0];
        const int64_t sp = s ? g - nsup[0] : g;
        const double4 *box = A.box64[s];
        double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
        for (int64_t k = sp * SUP + lane; k < min(ntile[s], (sp + 1) * SUP); k += 32) {
            const double4 b = box[k];
            x0 = fmin(x0, b.x);
            y0 = fmin(y0, b.y);
            x1 = fmax(x1, b.z);
            y1 = fmax(y1, b.w);
        }
        for (int o = 16; o; o >>= 1) {
            x0 = fmin(x0, __shfl_xor_sync(0xffffffffu, x0, o));
            y0 = fmin(y0, __shfl_xor_sync(0xffffffffu, y0, o));
            x1 = fmax(x1, __shfl_xor_sync(0xffffffffu, x1, o));
            y1 = fmax(y1, __shfl_xor_sync(0xffffffffu, y1, o));
        }
        if (lane == 0) A.sbox[s][sp] = make_double4(x0, y0, x1, y1);
    }
}


// Rigorous upper bound (scaled units) on the distance from a source to the
// target that produced its FP32 estimate `est` in the local frame of
// rwmd_tile.cu, where |x| = qn is the source's local radius.  With
// u = 2^-24 and D~ the distance of the rounded local coordinates:
//   |est - D~^2| <= 5u (2|x| + D~)^2          (expanded form, FFMA/FFMA2)
//   |D - D~|     <= u (2|x| + D~)              (one rounding per coordinate)
// so with c = 2^-20 >= 5u:  D~ <= (sqrt(est) + 2 sqrt(c) |x|) / (1 - sqrt(c)).
// (sqrt taken in FP32 rounded up -- >= the exact root of est -- and the division by
// 1 - 2^-10 replaced by a multiplication by 1 + 2^-9 > 1 / (1 - 2^-10): both only raise
// the bound, and no fp64 square root or division runs per source)
__device__ __forceinline__ double upper_bound_expanded(float est, float qn) {
    const double x = (double)qn * (1.0 + 0x1p-20) + 0x1p-60;
    const double dt = ((double)__fsqrt_ru(fmaxf(est, 0.0f)) + 0x1p-9 * x) * (1.0 + 0x1p-9);
    return dt * (1.0 + 0x1p-20) + 0x1p-20 * x + 0x1p-40;
}
// The direct form (culled mode: dx = x - y, est = fl(dy^2 + fl(dx^2))) does
// not cancel: est >= |(dx,dy)|^2 (1 - 2.01u), |(dx,dy)| >= |x - y| (1 - u) and
// |D - |x - y|| <= u (2|x| + D), hence
//   D <= (sqrt(est)(1 + 1.01u)/(1 - u) + 2u|x|(1 + 3u)) / (1 - u);
// 2^-20 = 16u covers every factor.
__device__ __forceinline__ double upper_bound_direct(float est, float qn) {
    return ((double)__fsqrt_ru(fmaxf(est, 0.0f)) * (1.0 + 0x1p-20) + 0x1p-20 * (double)qn) * (1.0 + 0x1p-20) + 0x1p-60;
}
__device__ __forceinline__ double upper_bound(float est, float qn, int direct) {
    return direct ? upper_bound_direct(est, qn) : upper_bound_expanded(est, qn);
}


// Is box b within distance R of box a, conservatively in FP32 (the refine's filters): true
// whenever the exact fp64 test gx^2 + gy^2 <= R^2 is (it never drops a tile that test keeps --
// extra exact distances cannot change a min):
// boxes rounded outward, gaps and squares rounded down, the radius (carrying 2^-40 of
// relative slack over fp64's own rounding) rounded up.  Overflow and NaN only widen it
// (fmaxf drops a NaN gap to 0; an infinite radius keeps everything).
__device__ __forceinline__ float4 box_out32(double4 b) {
    return make_float4(__double2float_rd(b.x), __double2float_rd(b.y), __double2float_ru(b.z),
                       __double2float_ru(b.w));
}
__device__ __forceinline__ float rad_up32(double R) {
    return R >= 0.0 ? __double2float_ru(R * (1.0 + 0x1p-40)) : -1.0f;
}
__device__ __forceinline__ bool within32(float4 b, float4 a, float R) {
    const float gx = fmaxf(0.0f, fmaxf(__fsub_rd(b.x, a.z), __fsub_rd(a.x, b.z)));
    const float gy = fmaxf(0.0f, fmaxf(__fsub_rd(b.y, a.w), __fsub_rd(a.y, b.w)));
    return R >= 0.0f && __fadd_rd(__fmul_rd(gx, gx), __fmul_rd(gy, gy)) <= __fmul_ru(R, R);
}

__device__ __forceinline__ double gap2(double4 b, double4 a) {  // squared box gap, as within()
    const double gx = fmax(0.0, fmax(b.x - a.z, a.x - b.z));
    const double gy = fmax(0.0, fmax(b.y - a.w, a.y - b.w));
    return gx * gx + gy * gy;
}

// Exact nearest squared distance of one source by warp-level branch and bound
// over the tile hierarchy: the nearest super-tile first (nearest child tile
// first inside a super-tile), every exact distance found shrinking the search
// radius (R = sqrt(m2)(1 + 1e-9) keeps every target that could still lower
// the min), then the remaining super-tiles against the shrunk radius.  The
// min VALUE is all the caller needs, so skipping targets that cannot lower it
// is exact.  All lanes return the same m2.
__device__ double solo_nn(double2 pj, double rad, const double2 *__restrict__ t, int64_t nt,
                          const double4 *__restrict__ tbox, const double4 *__restrict__ sbox, int64_t ntile,
                          int64_t nsup, int lane, unsigned long long *evals) {
    const double4 pb = make_double4(pj.x, pj.y, pj.x, pj.y);
    double m2 = INFINITY, R = rad;
    auto eval_tile = [&](int64_t k) {
        if (evals && lane == 0) atomicAdd(evals, (unsigned long long)RT);
        double ma = INFINITY;
        for (int64_t jt = k * RT + lane; jt < min(nt, (k + 1) * RT); jt += 32) {
            const double2 ta = t[jt];
            const double ax = dsub(pj.x, ta.x), ay = dsub(pj.y, ta.y);
            const double da = dadd(dmul(ax, ax), dmul(ay, ay));
            ma = da < ma ? da : ma;
        }
        for (int o = 16; o; o >>= 1) {
            const double ot = __shfl_xor_sync(0xffffffffu, ma, o);
            ma = ot < ma ? ot : ma;
        }
        ma = __shfl_sync(0xffffffffu, ma, 0);  // keep every decision warp-uniform (NaN-safe)
        if (ma < m2) {
            m2 = ma;
            R = fmin(rad, sqrt(m2) * (1.0 + 1e-9) + 1e-300);
        }
    };
    auto do_super = [&](int64_t si) {
        const int64_t kend = min(ntile, (si + 1) * SUP);
        const int64_t k1 = si * SUP + lane, k2 = k1 + 32;
        const double g1 = k1 < kend ? gap2(tbox[k1], pb) : INFINITY;
        const double g2 = k2 < kend ? gap2(tbox[k2], pb) : INFINITY;
        double gm = g1 <= g2 ? g1 : g2;
        int km = g1 <= g2 ? lane : lane + 32;
        for (int o = 16; o; o >>= 1) {
            const double og = __shfl_xor_sync(0xffffffffu, gm, o);
            const int ok = __shfl_xor_sync(0xffffffffu, km, o);
            if (og < gm || (og == gm && ok < km)) {
                gm = og;
                km = ok;
            }
        }
        gm = __shfl_sync(0xffffffffu, gm, 0);
        km = __shfl_sync(0xffffffffu, km, 0);
        if (gm <= R * R) eval_tile(si * SUP + km);
        unsigned b1 = __ballot_sync(0xffffffffu, g1 <= R * R && lane != km);
        unsigned b2 = __ballot_sync(0xffffffffu, g2 <= R * R && lane + 32 != km);
        while (b1) {
            const int l = __ffs(b1) - 1;
            b1 &= b1 - 1;
            if (__shfl_sync(0xffffffffu, g1, l) <= R * R) eval_tile(si * SUP + l);
        }
        while (b2) {
            const int l = __ffs(b2) - 1;
            b2 &= b2 - 1;
            if (__shfl_sync(0xffffffffu, g2, l) <= R * R) eval_tile(si * SUP + 32 + l);
        }
    };
    // nearest super-tile first
    double sg = INFINITY;
    int64_t sk = -1;
    for (int64_t sp = lane; sp < nsup; sp += 32) {
        const double g = gap2(sbox[sp], pb);
        if (g < sg) {
            sg = g;
            sk = sp;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, sg, o);
        const int64_t ok = __shfl_xor_sync(0xffffffffu, sk, o);
        if (og < sg || (og == sg && ok < sk)) {
            sg = og;
            sk = ok;
        }
    }
    sg = __shfl_sync(0xffffffffu, sg, 0);
    sk = __shfl_sync(0xffffffffu, sk, 0);
    if (sk >= 0 && sg <= R * R) do_super(sk);
    for (int64_t sp0 = 0; sp0 < nsup; sp0 += 32) {
        const int64_t sp = sp0 + lane;
        const double g = (sp < nsup && sp != sk) ? gap2(sbox[sp], pb) : INFINITY;
        unsigned bal = __ballot_sync(0xffffffffu, g <= R * R);
        while (bal) {
            const int l = __ffs(bal) - 1;
            bal &= bal - 1;
            if (__shfl_sync(0xffffffffu, g, l) <= R * R) do_super(sp0 + l);
        }
    }
    return m2;
}

constexpr int RF_BLOCK = 128;
constexpr int RF_CAND = 2048;
constexpr int RF_STAGE = 16;  // candidate tiles staged per round (16 x 64 targets, 16 KB)
constexpr int RF_SUPCAP = 1024;  // super-tiles listed per outer round (4M targets)

// exact fp64 refinement + mass * best (lower_bound.py:51-58).  Two threads per
// source (each takes every other target of a staged tile, then a shuffle
// min), sources in Morton order, 64-target Morton tiles kept by a box test
template <int RF_TPQ>  // threads per source
__global__ void __launch_bounds__(RF_BLOCK) k_refine(const double2 *__restrict__ q, const int32_t *__restrict__ qpos,
                                                     const int32_t *__restrict__ members,
                                                     const int64_t *__restrict__ mass, int64_t nq,
                                                     const unsigned *__restrict__ mf32,
                                                     const float *__restrict__ qn, double unscale,
                                                     const double2 *__restrict__ t, int64_t nt,
                                                     const double4 *__restrict__ tbox,
                                                     const double4 *__restrict__ sbox,
                                                     double *__restrict__ best_out, double *__restrict__ terms,
                                                     int direct, unsigned long long *evals) {
    constexpr int RF_QPB = RF_BLOCK / RF_TPQ;  // sources per block
    __shared__ int32_t s_cand[RF_CAND];
    __shared__ int32_t s_sup[RF_SUPCAP];
    __shared__ double2 s_t[RF_STAGE * RT];
    __shared__ float4 s_tb32[RF_STAGE];
    __shared__ int s_nc, s_nsup;
    __shared__ double2 s_p[RF_QPB];  // per-source point (solo searches)
    __shared__ float4 s_p32[RF_QPB]; // per-source point box and radius for the candidate
    __shared__ float s_rad32[RF_QPB];  // filter (FP32, conservative: within32)
    __shared__ float4 s_box32[RF_BLOCK / 32];
    __shared__ float s_r32[RF_BLOCK / 32];
    __shared__ float4 s_qb32;
    __shared__ float s_rmax32;
    __shared__ double s_solo_r[RF_QPB], s_solo_m2[RF_QPB];  // heavy sources: radius (-1: none), result
    __shared__ unsigned s_hmask[RF_BLOCK / 32];  // heavy sources per warp (lanes with sub == 0)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, sub = tid & (RF_TPQ - 1);
    const int64_t i = (int64_t)blockIdx.x * RF_QPB + tid / RF_TPQ;
    const bool valid = i < nq;
    double2 p = make_double2(0, 0);
    double diag = 0.0, r = -1.0;
    if (valid) {
        p = q[i];
        diag = ddiv(fabs(dsub(p.y, p.x)), SQRT2);  // diagram.py:47
        if (nt > 0) {
            const double U = upper_bound(__uint_as_float(mf32[i]), qn[i], direct & 1) * unscale * (1.0 + 1e-9);
            r = fmin(U, diag * (1.0 + 1e-12));
            r += 0x1p-50 * (fabs(p.x) + fabs(p.y) + r) + 1e-300;
        }
    }
    // a disc far wider than the warp's median (a poor FP32 seed or an isolated
    // point) would flood the block's shared search: such a source is searched
    // alone afterwards (solo_nn) and takes no part in the block search
    // warp median by a 32-wide bitonic sort, in FP32 (a heuristic split only: both the
    // block search and the solo search are exact, so the rounding cannot change a result)
    float v = (valid && r >= 0.0) ? (float)r : INFINITY;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int jb = k >> 1; jb; jb >>= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, v, jb);
            const bool up = ((lane & k) == 0) == ((lane & jb) == 0);
            v = up ? fminf(v, o) : fmaxf(v, o);
        }
    const double wmed = (double)__shfl_sync(0xffffffffu, v, 16);
    const bool heavy = (direct >> 8) > 0 && valid && r >= 0.0 && r > (double)(direct >> 8) * wmed;
    const double rh = r;
    if (heavy) r = -1.0;  // block-search radius
    const float4 p32 = box_out32(make_double4(p.x, p.y, p.x, p.y));
    if (sub == 0) {
        s_p[tid / RF_TPQ] = p;
        s_p32[tid / RF_TPQ] = p32;
        s_rad32[tid / RF_TPQ] = rad_up32((valid && r >= 0.0) ? r * (1.0 + 1e-9) : -1.0);
        s_solo_r[tid / RF_TPQ] = heavy ? rh * (1.0 + 1e-9) : -1.0;
    }
    // this thread's own evaluation filter (the same radius as the fp64 test had)
    const float r_eval32 = rad_up32((valid && r >= 0.0) ? r * (1.0 + 1e-9) : -1.0);
    {
        const unsigned hm = __ballot_sync(0xffffffffu, heavy && sub == 0);
        if (lane == 0) s_hmask[wid] = hm;
    }
    if (tid == 0) s_nsup = s_nc = 0;
    double m2 = INFINITY, m2b = INFINITY;
    if (nt > 0) {
        // warp and block boxes and radii, in FP32 rounded outward: box_out32 and rad_up32
        // are monotonic, so reducing the rounded per-source values gives exactly the
        // rounding of the fp64 reduction (min of rounded-down = rounded-down min)
        float4 b = (valid && !heavy) ? p32 : make_float4(INFINITY, INFINITY, -INFINITY, -INFINITY);
        float rm = r_eval32;
        for (int o = 16; o; o >>= 1) {
            b.x = fminf(b.x, __shfl_xor_sync(0xffffffffu, b.x, o));
            b.y = fminf(b.y, __shfl_xor_sync(0xffffffffu, b.y, o));
            b.z = fmaxf(b.z, __shfl_xor_sync(0xffffffffu, b.z, o));
            b.w = fmaxf(b.w, __shfl_xor_sync(0xffffffffu, b.w, o));
            rm = fmaxf(rm, __shfl_xor_sync(0xffffffffu, rm, o));
        }
        if (lane == 0) {
            s_box32[wid] = b;
            s_r32[wid] = rm;
        }
        __syncthreads();
        if (tid == 0) {
            float4 bb = s_box32[0];
            float rr = s_r32[0];
            for (int w = 1; w < RF_BLOCK / 32; w++) {
                bb.x = fminf(bb.x, s_box32[w].x);
                bb.y = fminf(bb.y, s_box32[w].y);
                bb.z = fmaxf(bb.z, s_box32[w].z);
                bb.w = fmaxf(bb.w, s_box32[w].w);
                rr = fmaxf(rr, s_r32[w]);
            }
            s_qb32 = bb;
            s_rmax32 = rr;
        }
        __syncthreads();
        const float4 qb32 = s_qb32;
        const float rmax32 = s_rmax32;
        const int64_t ntile = (nt + RT - 1) / RT;
        const int64_t nsup = (ntile + SUP - 1) / SUP;
        constexpr int SUP_ROUND = RF_CAND / SUP;  // super-tiles per round: <= RF_CAND child tiles
        // two-level candidate search: the super-tiles meeting the block are
        // listed once, then their child tiles are tested SUP_ROUND super-tiles
        // at a time (conservative FP32 box tests)
        for (int64_t sb = 0; sb < nsup; sb += RF_SUPCAP) {
          for (int64_t sp = sb + tid; sp < min(nsup, sb + RF_SUPCAP); sp += RF_BLOCK)
            if (within32(box_out32(sbox[sp]), qb32, rmax32)) s_sup[atomicAdd(&s_nsup, 1)] = (int32_t)sp;
          __syncthreads();
          const int n_sup = s_nsup;
          for (int u0 = 0; u0 < n_sup; u0 += SUP_ROUND) {
            const int nsr = min(SUP_ROUND, n_sup - u0);
            // a tile is staged iff some source of the block needs it: the block box
            // first, then the warp boxes, then the warp's sources one by one (the
            // same test the evaluation uses) -- a Morton block straddling a jump
            // has a huge box but only a handful of tiles its sources need
            for (int e = tid; e < nsr * SUP; e += RF_BLOCK) {
                const int64_t k = (int64_t)s_sup[u0 + e / SUP] * SUP + (e % SUP);
                if (k >= ntile) continue;
                const float4 tb = box_out32(tbox[k]);
                if (!within32(tb, qb32, rmax32)) continue;
                bool need = false;
                for (int w = 0; w < RF_BLOCK / 32 && !need; w++) {
                    if (!within32(tb, s_box32[w], s_r32[w])) continue;
                    for (int j = w * (32 / RF_TPQ); j < (w + 1) * (32 / RF_TPQ); j++) {
                        if (within32(tb, s_p32[j], s_rad32[j])) {
                            need = true;
                            break;
                        }
                    }
                }
                if (need) s_cand[atomicAdd(&s_nc, 1)] = (int32_t)k;
            }
            __syncthreads();
            const int nc = s_nc;
            // candidate tiles are staged RF_STAGE at a time in shared memory; a
            // warp evaluates a staged tile (all lanes, uniformly) iff one of its
            // sources needs it -- extra exact distances never change the min
            for (int c0 = 0; c0 < nc; c0 += RF_STAGE) {
                const int ns = min(RF_STAGE, nc - c0);
                for (int e = tid; e < ns * RT; e += RF_BLOCK) {
                    const int64_t k = s_cand[c0 + e / RT];
                    const int64_t j = k * RT + (e % RT);
                    s_t[e] = j < nt ? t[j] : make_double2(INFINITY, INFINITY);
                }
                if (tid < ns) s_tb32[tid] = box_out32(tbox[s_cand[c0 + tid]]);
                __syncthreads();
                for (int c = 0; c < ns; c++) {
                    const bool need = within32(s_tb32[c], p32, r_eval32);
                    if (!__any_sync(0xffffffffu, need)) continue;
                    if (evals && lane == 0) atomicAdd(evals, (unsigned long long)(32 / RF_TPQ) * RT);
                    const double2 *st = s_t + c * RT + sub;
#pragma unroll
                    for (int j = 0; j < RT / RF_TPQ; j += 2) {
                        const double2 ta = st[RF_TPQ * j], tb = st[RF_TPQ * (j + 1)];
                        const double ax = dsub(p.x, ta.x), ay = dsub(p.y, ta.y);
                        const double bx = dsub(p.x, tb.x), by = dsub(p.y, tb.y);
                        const double da = dadd(dmul(ax, ax), dmul(ay, ay));
                        const double db = dadd(dmul(bx, bx), dmul(by, by));
                        m2 = da < m2 ? da : m2;
                        m2b = db < m2b ? db : m2b;
                    }
                }
                __syncthreads();
            }
            if (tid == 0) s_nc = 0;
            __syncthreads();
          }
          if (tid == 0) s_nsup = 0;
          __syncthreads();
        }
        // heavy sources (usually none): the k-th of them goes to warp k % 4
        int H = 0;
        for (int w = 0; w < RF_BLOCK / 32; w++) H += __popc(s_hmask[w]);
        for (int k = wid; k < H; k += RF_BLOCK / 32) {
            int w2 = 0, kk = k;
            while (kk >= __popc(s_hmask[w2])) kk -= __popc(s_hmask[w2++]);
            unsigned m = s_hmask[w2];
            for (int q = 0; q < kk; q++) m &= m - 1;
            const int j = w2 * (32 / RF_TPQ) + (__ffs(m) - 1) / RF_TPQ;
            const double ms = solo_nn(s_p[j], s_solo_r[j], t, nt, tbox, sbox, ntile, nsup, lane, evals);
            if (lane == 0) s_solo_m2[j] = ms;
        }
        if (H) __syncthreads();  // H is block-uniform
        if (heavy) m2 = fmin(m2, s_solo_m2[tid / RF_TPQ]);
    }
    m2 = m2b < m2 ? m2b : m2;
#pragma unroll
    for (int o = 1; o < RF_TPQ; o <<= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, m2, o);
        m2 = other < m2 ? other : m2;
    }
    if (valid && sub == 0) {
        double best = diag;
        if (nt > 0) {
            const double nnd = dsqrt(m2);
            best = nnd < diag ? nnd : diag;  // np.minimum(nnd, diag)
        }
        const int32_t pos = qpos[i];
        best_out[pos] = (direct & 2) ? rh : best;  // bit 1: debug, report the search radius
        terms[pos] = dmul(__ll2double_rn(mass[members[pos]]), best);  // float64(src_mass) * best
    }
}
}  // namespace

// the exact pass for one direction
static int launch_refine(Ctx &c, const double2 *q, const int32_t *qpos, const int32_t *members,
                         const int64_t *mass, int64_t nq, const unsigned *mf, const float *qn, double unscale,
                         const double2 *t, int64_t nt, const double4 *tbox, const double4 *sbox, double *best,
                         double *terms) {
    // bit 0 culled (direct-form bound), bit 1 debug, bits 8+ heavy ratio (0: off)
    const int flags = c.culling | (c.debug_radius << 1) | (c.heavy_ratio << 8);
    unsigned long long *evals = c.prof ? ptr<unsigned long long>(c.prof_cnt) + 2 * c.prof_side + 1 : nullptr;
    if (c.prof) W1G_CUDA(cudaEventRecord(c.prof_ev[c.prof_side][1][0], c.stream));
    // threads per source (W1G_RF_TPQ = 1, 2, 4 or 8): a warp evaluates a staged tile for all of
    // its 32 / TPQ sources as soon as one of them needs it
    static const int tpq = [] {
        const char *e = getenv("W1G_RF_TPQ");
        const int v = e ? atoi(e) : 2;
        return (v == 1 || v == 4 || v == 8) ? v : 2;
    }();
    const unsigned qpb = RF_BLOCK / tpq;
    const unsigned grid = (unsigned)((nq + qpb - 1) / qpb);
    if (tpq == 8)
        k_refine<8><<<grid, RF_BLOCK, 0, c.stream>>>(q, qpos, members, mass, nq, mf, qn, unscale, t, nt, tbox,
                                                     sbox, best, terms, flags, evals);
    else if (tpq == 1)
        k_refine<1><<<grid, RF_BLOCK, 0, c.stream>>>(q, qpos, members, mass, nq, mf, qn, unscale, t, nt, tbox,
                                                     sbox, best, terms, flags, evals);
    else if (tpq == 4)
        k_refine<4><<<grid, RF_BLOCK, 0, c.stream>>>(q, qpos, members, mass, nq, mf, qn, unscale, t, nt, tbox,
                                                     sbox, best, terms, flags, evals);
    else
        k_refine<2><<<grid, RF_BLOCK, 0, c.stream>>>(q, qpos, members, mass, nq, mf, qn, unscale, t, nt, tbox,
                                                     sbox, best, terms, flags, evals);
    W1G_CHECK_LAUNCH();
    if (c.prof) W1G_CUDA(cudaEventRecord(c.prof_ev[c.prof_side][1][1], c.stream));
    return W1G_OK;
}

static inline double key_to_double(uint64_t k) {
    uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}

// shared preparation: members, bbox frame, Morton order (per side)
struct RwmdFrame {
    int64_t nm[2];
    double scale, unscale;
    int32_t *members[2];
    double2 *mpts[2];  // member points in Morton order
    int32_t *mpos[2];  // member position (node order) of each Morton slot
    uint64_t *mkey[2]; // sorted Morton keys (seed the culled FP32 pass)
};

// range_side >= 0 restricts that side's SOURCE list to member positions
// [begin, end) (row sharding across ranks); the other side stays complete
static int rwmd_prepare(Ctx &c, RwmdFrame &F, int range_side = -1, int64_t begin = 0, int64_t end = 0) {
    NodeSet &ns = c.nodes[0];
    const int64_t k = ns.k;
    const double2 *pts = ptr<double2>(ns.pts);
    const int64_t *mass[2] = {ptr<int64_t>(ns.am), ptr<int64_t>(ns.bm)};
    int64_t *excl;
    W1G_TRY(ensure(c.scr[3], 2 * (size_t)k, &excl));
    W1G_TRY(ensure(c.scr[5], k, &F.members[0]));
    W1G_TRY(ensure(c.scr[6], k, &F.members[1]));
    W1G_TRY(flags_reset(c));
    for (int s = 0; s < 2; s++) W1G_TRY(scan_i64(c, MemberFlag{mass[s]}, k, excl + s * k, dflags(c) + F_MISC0 + s));
    k_compact2<<<grid_for(2 * k, 256, 8u * c.sm_count), 256, 0, c.stream>>>(mass[0], mass[1], k, excl, excl + k,
                                                                            F.members[0], F.members[1]);
    W1G_CHECK_LAUNCH();
    uint64_t bk[4];
    if (ns.stats && range_side < 0) {
        // zero_condense delivered the member counts and the bbox: no round trip here
        F.nm[0] = ns.nmem[0];
        F.nm[1] = ns.nmem[1];
        for (int q = 0; q < 4; q++) bk[q] = ns.bbox_key[q];
    } else {
        k_bbox_init<<<1, 1, 0, c.stream>>>(dflags(c));
        k_bbox<<<grid_for(k, 256, 2u * c.sm_count), 256, 0, c.stream>>>(pts, k, dflags(c));  // few CTAs: fewer atomics
        W1G_CHECK_LAUNCH();
        W1G_TRY(flags_fetch(c, 0, F_BBOX + 4));
        F.nm[0] = c.h_pinned[F_MISC0];
        F.nm[1] = c.h_pinned[F_MISC1];
        for (int q = 0; q < 4; q++) bk[q] = (uint64_t)c.h_pinned[F_BBOX + q];
    }
    c.rw_members[0] = F.nm[0];
    c.rw_members[1] = F.nm[1];
    const double xmin = key_to_double(bk[0]);
    const double xmax = key_to_double(bk[1]);
    const double ymin = key_to_double(bk[2]);
    const double ymax = key_to_double(bk[3]);
    // scaled FP32 frame: a power-of-two scale (exact in fp64) bringing the extent below 1
    double H = std::fmax(xmax - xmin, ymax - ymin);
    int e = 0;
    if (H > 0.0 && std::isfinite(H)) e = std::ilogb(H) + 1;
    F.scale = std::ldexp(1.0, -e);
    F.unscale = std::ldexp(1.0, e);
    const double ext = H > 0.0 && std::isfinite(H) ? H : 1.0;
    const double inv = MORTON_MAX / ext;
    SortJob jobs[2];
    int64_t off[2];
    Morton2 M;
    for (int s = 0; s < 2; s++) {
        off[s] = s == range_side ? begin : 0;
        const int64_t n = s == range_side ? end - begin : F.nm[s];
        uint64_t *key;
        uint32_t *perm;
        W1G_TRY(ensure(c.scr[s == 0 ? 0 : 22], (size_t)n + 1, &key));
        W1G_TRY(ensure(c.scr[s == 0 ? 2 : 23], (size_t)n + 1, &perm));
        W1G_TRY(ensure(c.scr[7 + 2 * s], (size_t)n + 1, &F.mpts[s]));
        W1G_TRY(ensure(c.scr[8 + 2 * s], (size_t)n + 1, &F.mpos[s]));
        F.mkey[s] = key;
        jobs[s] = SortJob{{key, nullptr, nullptr}, perm, n};
        M.members[s] = F.members[s] + off[s];
        M.n[s] = n;
        M.key[s] = key;
        M.val[s] = perm;
    }
    // both sides' keys, sorts and gathers in the same launches
    if (M.n[0] + M.n[1] > 0) {
        k_morton2<<<grid_for(M.n[0] + M.n[1], 256, 8u * c.sm_count), 256, 0, c.stream>>>(pts, M, xmin, ymin, inv);
        W1G_CHECK_LAUNCH();
    }
    W1G_TRY(radix_sort_multi(c, jobs, 2, 1, MORTON_BITS));
    Gather2 G;
    for (int s = 0; s < 2; s++) {
        G.members[s] = M.members[s];
        G.perm[s] = jobs[s].vals;
        G.n[s] = jobs[s].n;
        G.offset[s] = off[s];
        G.out[s] = F.mpts[s];
        G.pos[s] = F.mpos[s];
    }
    if (G.n[0] + G.n[1] > 0) {
        k_gather2<<<grid_for(G.n[0] + G.n[1], 256, 8u * c.sm_count), 256, 0, c.stream>>>(pts, G);
        W1G_CHECK_LAUNCH();
    }
    return W1G_OK;
}

int rwmd_run(Ctx &c, double *L, double *LA, double *LB) {
    NodeSet &ns = c.nodes[0];
    const int64_t k = ns.k;
    const int64_t *mass[2] = {ptr<int64_t>(ns.am), ptr<int64_t>(ns.bm)};
    if (k == 0) {
        *L = *LA = *LB = 0.0;
        c.n_best[0] = c.n_best[1] = 0;
        return W1G_OK;
    }
    SubTimer T(c, "rwmd");
    RwmdFrame F;
    W1G_TRY(rwmd_prepare(c, F));
    T.mark("prepare");
    const int64_t mx = (F.nm[0] > F.nm[1] ? F.nm[0] : F.nm[1]) + 1;
    const int64_t mtb = mx / 64 + 2, msb = mx / (64 * SUP) + 2;
    double *terms, *dres;
    unsigned *mf;
    float *qn;
    double4 *tbox, *box64, *sbox;
    // per-side scratch (the two sides may run concurrently), all allocated up front
    W1G_TRY(ensure(c.scr[11], (size_t)2 * mx, &terms));
    W1G_TRY(ensure(c.scr[12], 4, &dres));
    W1G_TRY(ensure(c.scr[13], (size_t)2 * mx, &mf));
    W1G_TRY(ensure(c.scr[14], (size_t)2 * mx, &qn));
    W1G_TRY(ensure(c.scr[15], (size_t)2 * mtb, &tbox));  // per-tile boxes (tiles >= 64 targets)
    W1G_TRY(ensure(c.scr[16], (size_t)2 * mtb, &box64));
    W1G_TRY(ensure(c.scr[21], (size_t)2 * msb, &sbox));
    double *best_s[2];
    for (int s = 0; s < 2; s++) W1G_TRY(ensure(c.best[s], (size_t)F.nm[s] + 1, &best_s[s]));
    double *val1;
    W1G_TRY(ensure(c.scr[17], (size_t)F.nm[1] / 32 + 64, &val1));
    // side B on the side stream, concurrently with side A, once its summation tree is cached
    // (nothing left to allocate inside)
    cudaStream_t side = c.copy_stream;
    // (per-kernel profiling, w1g_profile_rwmd, runs the sides one after the other so each
    // kernel's event time is its own)
    const bool conc = side && !c.prof && F.nm[0] > 0 && F.nm[1] > 0 && c.pw_n[1] == F.nm[1];
    auto run_side = [&](int s) -> int {
        const int o = 1 - s;
        c.prof_side = s;
        const int64_t n_src = F.nm[s], n_dst = F.nm[o];
        c.n_best[s] = n_src;
        double *best = best_s[s];
        unsigned *mf_s = mf + s * mx;
        float *qn_s = qn + s * mx;
        double *terms_s = terms + s * mx;
        double4 *tbox_s = tbox + s * mtb, *box64_s = box64 + s * mtb, *sbox_s = sbox + s * msb;
        if (n_src == 0) {
            W1G_CUDA(cudaMemsetAsync(dres + s, 0, sizeof(double), c.stream));
            reinterpret_cast<double *>(c.h_pinned + H_SCALAR)[s] = 0.0;
            return W1G_OK;
        }
        if (n_dst > 0) {
            W1G_CUDA(cudaMemsetAsync(mf_s, 0x7f, sizeof(unsigned) * n_src, c.stream));
            W1G_TRY(rwmd_f32_min(c, F.mpts[s], F.mkey[s], n_src, F.mpts[o], F.mkey[o], n_dst, F.scale, mf_s, qn_s,
                                 tbox_s, c.culling, c.culling ? 1 : 0));
            T.mark(s ? "f32_b" : "f32_a");
        }
        W1G_TRY(launch_refine(c, F.mpts[s], F.mpos[s], F.members[s], mass[s], n_src, mf_s, qn_s, F.unscale,
                              F.mpts[o], n_dst, box64_s, sbox_s, best, terms_s));
        T.mark("refine");
        // the sum also lands in the page-locked scalar slot the host reads (no extra small read)
        W1G_TRY(pairwise_sum(c, terms_s, n_src, dres + s, c.pw_nodes[s], s ? c.scr[17] : c.scr[18], c.pw_lev[s],
                             &c.pw_n[s], reinterpret_cast<double *>(c.h_pinned + H_SCALAR) + s));
        T.mark("sum");
        return W1G_OK;
    };
    // every tile / refine-tile / super-tile box of both sides' targets, before the sides fork
    {
        SideBoxes B;
        for (int s = 0; s < 2; s++) {
            const int o = 1 - s;
            const bool on = F.nm[s] > 0 && F.nm[o] > 0;
            B.t[s] = F.mpts[o];
            B.n[s] = on ? F.nm[o] : 0;
            B.tbox[s] = tbox + s * mtb;
            B.box64[s] = box64 + s * mtb;
            B.sbox[s] = sbox + s * msb;
        }
        B.nblk0 = (B.n[0] + 4 * RT - 1) / (4 * RT);
        const int64_t nblk = B.nblk0 + (B.n[1] + 4 * RT - 1) / (4 * RT);
        if (nblk > 0) {
            k_side_boxes<<<(unsigned)nblk, 128, 0, c.stream>>>(B);
            W1G_CHECK_LAUNCH();
            const int64_t nsup = (B.n[0] + RT * SUP - 1) / (RT * SUP) + (B.n[1] + RT * SUP - 1) / (RT * SUP);
            k_side_superboxes<<<grid_for(nsup * 32, 256, 8u * c.sm_count), 256, 0, c.stream>>>(B);
            W1G_CHECK_LAUNCH();
        }
        T.mark("boxes");
    }
    if (conc) {
        W1G_CUDA(cudaEventRecord(c.ev[14], c.stream));
        W1G_CUDA(cudaStreamWaitEvent(side, c.ev[14], 0));
        std::swap(c.stream, side);
        const int rc = run_side(1);
        std::swap(c.stream, side);
        W1G_TRY(rc);
        W1G_CUDA(cudaEventRecord(c.ev[15], side));
        W1G_TRY(run_side(0));
        W1G_CUDA(cudaStreamWaitEvent(c.stream, c.ev[15], 0));
    } else {
        W1G_TRY(run_side(0));
        W1G_TRY(run_side(1));
    }
    W1G_TRY(stream_sync(c));
    double h[2];
    memcpy(h, c.h_pinned + H_SCALAR, sizeof h);
    *LA = h[0];
    *LB = h[1];
    *L = h[1] > h[0] ? h[1] : h[0];  // python max(l_a, l_b)
    return W1G_OK;
}

// one rank's share of a row-sharded RWMD: side `side`'s sources restricted to
// member positions [begin, end) (a subtree of numpy's summation tree, chosen
// by the host), all targets; returns the subtree's pairwise sum
int rwmd_range_run(Ctx &c, int side, int64_t begin, int64_t end, double *partial, int64_t *n_members) {
    NodeSet &ns = c.nodes[0];
    const int64_t *mass[2] = {ptr<int64_t>(ns.am), ptr<int64_t>(ns.bm)};
    *partial = 0.0;
    if (ns.k == 0) {
        *n_members = 0;
        return W1G_OK;
    }
    // member counts first (the range is validated against them)
    RwmdFrame F;
    W1G_TRY(rwmd_prepare(c, F, side, 0, 0));
    *n_members = F.nm[side];
    if (begin < 0 || end > F.nm[side] || begin > end) {
        set_error("rwmd_range: [%lld, %lld) outside [0, %lld)", (long long)begin, (long long)end,
                  (long long)F.nm[side]);
        return W1G_EINVAL;
    }
    if (begin == end) return W1G_OK;
    W1G_TRY(rwmd_prepare(c, F, side, begin, end));
    const int s = side, o = 1 - side;
    const int64_t n_src = end - begin, n_dst = F.nm[o];
    const int64_t mx = (F.nm[0] > F.nm[1] ? F.nm[0] : F.nm[1]) + 1;
    double *terms, *dres, *best;
    unsigned *mf;
    float *qn;
    double4 *tbox, *box64, *sbox;
    W1G_TRY(ensure(c.scr[11], (size_t)mx, &terms));
    W1G_TRY(ensure(c.scr[12], 4, &dres));
    W1G_TRY(ensure(c.scr[13], (size_t)mx, &mf));
    W1G_TRY(ensure(c.scr[14], (size_t)mx, &qn));
    W1G_TRY(ensure(c.scr[15], (size_t)mx / 64 + 2, &tbox));
    W1G_TRY(ensure(c.scr[16], (size_t)mx / 64 + 2, &box64));
    W1G_TRY(ensure(c.scr[21], (size_t)mx / (64 * SUP) + 2, &sbox));
    W1G_TRY(ensure(c.best[s], (size_t)F.nm[s] + 1, &best));
    if (n_dst > 0) {
        W1G_CUDA(cudaMemsetAsync(mf, 0x7f, sizeof(unsigned) * n_src, c.stream));
        W1G_TRY(rwmd_f32_min(c, F.mpts[s], F.mkey[s], n_src, F.mpts[o], F.mkey[o], n_dst, F.scale, mf, qn, tbox, c.culling));
        k_boxes64<<<grid_for((n_dst / RT + 1) * 32, 256, 8u * c.sm_count), 256, 0, c.stream>>>(F.mpts[o], n_dst, box64);
        W1G_CHECK_LAUNCH();
        k_superboxes<<<grid_for((n_dst / RT / SUP + 1) * 32, 256, 8u * c.sm_count), 256, 0, c.stream>>>(
            box64, (n_dst + RT - 1) / RT, sbox);
        W1G_CHECK_LAUNCH();
    }
    W1G_TRY(launch_refine(c, F.mpts[s], F.mpos[s], F.members[s], mass[s], n_src, mf, qn, F.unscale, F.mpts[o], n_dst,
                          box64, sbox, best, terms));
    W1G_TRY(pairwise_sum(c, terms + begin, n_src, dres, c.scr[17], c.scr[18], c.scr[19]));
    W1G_TRY(to_host_small(c, c.h_pinned + H_SCALAR, dres, sizeof(double)));
    W1G_TRY(stream_sync(c));
    memcpy(partial, c.h_pinned + H_SCALAR, sizeof(double));
    return W1G_OK;
}

// measurement hook (w1g_profile_rwmd_tile): the FP32 tile pass alone, both
// directions, `reps` times, timed with events on the context stream
int rwmd_tile_profile(Ctx &c, int reps, float *ms, int64_t *evals) {
    RwmdFrame F;
    W1G_TRY(rwmd_prepare(c, F));
    const int64_t na = F.nm[0], nb = F.nm[1];
    *evals = na * nb;
    *ms = 0.f;
    if (na == 0 || nb == 0 || reps < 1) return W1G_OK;
    const int64_t mx = (na > nb ? na : nb) + 1;
    unsigned *mf;
    float *qn;
    double4 *tbox;
    W1G_TRY(ensure(c.scr[13], (size_t)mx, &mf));
    W1G_TRY(ensure(c.scr[14], (size_t)mx, &qn));
    W1G_TRY(ensure(c.scr[15], (size_t)mx / 64 + 2, &tbox));  // per-tile boxes (tiles >= 64 targets)
    W1G_CUDA(cudaEventRecord(c.ev[8], c.stream));
    for (int r = 0; r < reps; r++) {
        W1G_TRY(rwmd_f32_min(c, F.mpts[0], F.mkey[0], na, F.mpts[1], F.mkey[1], nb, F.scale, mf, qn, tbox, c.culling));
        W1G_TRY(rwmd_f32_min(c, F.mpts[1], F.mkey[1], nb, F.mpts[0], F.mkey[0], na, F.scale, mf, qn, tbox, c.culling));
    }
    W1G_CUDA(cudaEventRecord(c.ev[9], c.stream));
    W1G_CUDA(cudaEventSynchronize(c.ev[9]));
    float t = 0.f;
    W1G_CUDA(cudaEventElapsedTime(&t, c.ev[8], c.ev[9]));
    *ms = t / (2.0f * reps);
    return W1G_OK;
}

// measurement hook (w1g_profile_rwmd): the production RWMD (culled FP32 tile +
// exact fp64 refine per side, both sides as rwmd_run schedules them) `reps`
// times, with events around each side's tile and refine kernels (on the stream
// each runs on) and device counters of the evaluations they perform.
// ms[4] / evals[4]: mean per launch for [A tile, A refine, B tile, B refine];
// directed = 2 |A| |B| (the algorithmic all-pairs work).
int rwmd_profile(Ctx &c, int reps, float *ms, int64_t *evals, int64_t *directed) {
    for (int i = 0; i < 4; i++) {
        ms[i] = 0.f;
        evals[i] = 0;
    }
    *directed = 0;
    if (c.nodes[0].k == 0 || reps < 1) return W1G_OK;
    for (auto &side : c.prof_ev)
        for (auto &kind : side)
            for (auto &e : kind)
                if (!e) W1G_CUDA(cudaEventCreate(&e));
    unsigned long long *cnt;
    W1G_TRY(ensure(c.prof_cnt, 4, &cnt));
    W1G_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), c.stream));
    double acc[4] = {0, 0, 0, 0};
    struct Off {
        Ctx &c;
        ~Off() { c.prof = 0; }
    } off{c};
    for (int r = 0; r < reps; r++) {
        c.prof = 1;
        double L, la, lb;
        W1G_TRY(rwmd_run(c, &L, &la, &lb));  // ends with a host synchronisation
        c.prof = 0;
        for (int s = 0; s < 2; s++)
            for (int k = 0; k < 2; k++) {
                float t = 0.f;
                if (cudaEventElapsedTime(&t, c.prof_ev[s][k][0], c.prof_ev[s][k][1]) == cudaSuccess) acc[2 * s + k] += t;
                cudaGetLastError();
            }
    }
    unsigned long long h[4];
    W1G_CUDA(cudaMemcpy(h, cnt, sizeof h, cudaMemcpyDeviceToHost));
    for (int i = 0; i < 4; i++) {
        ms[i] = (float)(acc[i] / reps);
        evals[i] = (int64_t)(h[i] / (unsigned long long)reps);
    }
    *directed = 2 * c.rw_members[0] * c.rw_members[1];
    return W1G_OK;
}

}  // namespace w1g
