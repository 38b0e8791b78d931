// rwmd_tile.cu -- the FP32 all-pairs nearest-neighbour tile pass of RWMD.
//
// For every source q, min over targets t of |q - t|^2 -- the "tiled
// all-pairs nearest-neighbour min" of the north star -- on the FP32 pipe
// (a min over a distance is not a contraction, so no tensor cores):
//
//  * R sources per thread in registers, targets staged through shared
//    memory in tiles and broadcast to the warp;
//  * expanded form with packed FP32x2 math, two SOURCES per lane pair and
//    the target broadcast (full mode; PACKQ):
//        s = fma2((-2y_r, -2y_r+1), ty, fma2((-2x_r, -2x_r+1), tx, |t|^2))
//        m_r = min3(m_r, s_a.x, s_b.x)   over a target pair (a, b)
//    i.e. one FFMA2 and half an FMNMX3 per evaluation, the target's operands
//    shared by every source pair of the thread (operand reuse); |q|^2 is
//    added after the min (PACKQ = false: two targets per lane pair);
//  * the expansion cancels, so every CTA works in a LOCAL frame: origin =
//    its first source (sources are Morton-ordered, so a CTA's sources are
//    spatially compact) and targets are shifted into that frame as they are
//    staged (in fp64, then rounded once).  The error of the result is then
//    bounded by 2^-20 (2|q'| + d)^2 in scaled units, small
//    exactly where it matters;
//  * full mode (culling off): every source meets every target, the target
//    range is split across grid.y to fill the 148 SMs and per-chunk minima
//    merge with an order-independent atomicMin on the float bits;
//  * culled mode (the production path): any real target's distance is a
//    valid upper bound for the exact pass, so each CTA only evaluates the
//    Morton-nearest target tiles (walking 3 tiles outward from the tile
//    holding its middle source's Morton key, found by a warp-wide 32-ary
//    search of the target keys) and skips tiles whose bbox is farther than
//    the CTA's current worst upper bound; sources whose seed stays poor are
//    searched alone by the exact pass (rwmd.cu, solo_nn).
//
// The result only sizes the exact fp64 search in rwmd.cu.  This translation
// unit is compiled with FMA contraction allowed.
#include <cmath>

#include "common.cuh"

namespace w1g {

namespace {

constexpr int T_BLOCK = 256;
constexpr int TS_FULL = 1024;  // targets per shared-memory tile, full mode
constexpr int TS_CULL = 256;   // targets per shared-memory tile, culled mode

__device__ __forceinline__ float min3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

struct TileArgs {
    const double2 *q;       // sources (Morton order), original coordinates
    const double2 *t;       // targets (Morton order)
    const double4 *tbox;    // per T_TS-tile bbox of the targets (culled mode)
    const uint64_t *qkey;   // sorted Morton keys of the sources / targets (culled mode)
    const uint64_t *tkey;
    int nq, nt;
    double scale;           // 2^-e
    unsigned *mout;         // min d^2 estimate (float bits), scaled units
    float *qn_out;          // |q'| per source
    int chunk;              // targets per grid.y chunk (full mode)
    int cull_steps;         // culled mode: tiles walked outward from the Morton position
    unsigned long long *evals;  // profiling: evaluations performed (null: not counted)
};

template <int R, bool CULL, int T_TS, bool PACKQ = false>
__global__ void __launch_bounds__(T_BLOCK) k_rwmd_f32(TileArgs A) {
    __shared__ float4 s_xy[T_TS / 2];
    __shared__ float2 s_tt[T_TS / 2];
    __shared__ float s_red[T_BLOCK / 32];
    __shared__ double2 s_org;
    __shared__ double4 s_qbox;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int q0 = blockIdx.x * (T_BLOCK * R);
    if (tid == 0) s_org = A.q[q0];
    __syncthreads();
    const double ox = s_org.x, oy = s_org.y, sc = A.scale;
    float2 ax[R], ay[R];
    float m[R], qq[R], qn[R];
    double bx0 = INFINITY, by0 = INFINITY, bx1 = -INFINITY, by1 = -INFINITY;
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int i = q0 + r * T_BLOCK + tid;
        const bool v = i < A.nq;
        const double2 p = v ? A.q[i] : s_org;
        const float x = (float)((p.x - ox) * sc), y = (float)((p.y - oy) * sc);
        // expanded form keeps (-2x, -2x); the direct form (culled mode) keeps (x, x)
        const float fx = CULL ? x : -2.f * x, fy = CULL ? y : -2.f * y;
        ax[r] = make_float2(fx, fx);
        ay[r] = make_float2(fy, fy);
        if (CULL) {  // full mode recomputes them after the loop (fewer live registers)
            qq[r] = fmaf(x, x, y * y);
            qn[r] = sqrtf(qq[r]);
        }
        m[r] = INFINITY;
        if (CULL && v) {
            bx0 = fmin(bx0, p.x);
            by0 = fmin(by0, p.y);
            bx1 = fmax(bx1, p.x);
            by1 = fmax(by1, p.y);
        }
    }
    int n_tiles, t_first, center = 0;
    if (CULL) {
        // CTA bbox of its sources (original units) for the tile test
        for (int o = 16; o; o >>= 1) {
            bx0 = fmin(bx0, __shfl_xor_sync(0xffffffffu, bx0, o));
            by0 = fmin(by0, __shfl_xor_sync(0xffffffffu, by0, o));
            bx1 = fmax(bx1, __shfl_xor_sync(0xffffffffu, bx1, o));
            by1 = fmax(by1, __shfl_xor_sync(0xffffffffu, by1, o));
        }
        __shared__ double s_b[4][T_BLOCK / 32];
        if (lane == 0) {
            s_b[0][wid] = bx0;
            s_b[1][wid] = by0;
            s_b[2][wid] = bx1;
            s_b[3][wid] = by1;
        }
        __syncthreads();
        __shared__ int s_center;
        if (wid == 0) {
            // start at the target tile holding the Morton key of the CTA's middle
            // source: warp-wide 32-ary search for the first target key >= it
            const uint64_t key = A.qkey[min(q0 + T_BLOCK * R / 2, A.nq - 1)];
            int lo = 0, hi = A.nt;  // answer in [lo, hi]
            while (hi - lo > 32) {
                const int step = (hi - lo + 31) / 32;
                const int idx = lo + (lane + 1) * step - 1;
                const bool less = idx < hi && A.tkey[idx] < key;
                const int cnt = __popc(__ballot_sync(0xffffffffu, less));
                const int nlo = lo + cnt * step;
                hi = min(hi, lo + (cnt + 1) * step - 1);
                lo = nlo;
            }
            const int idx = lo + lane;
            const bool less = idx < hi && A.tkey[idx] < key;
            const int pos = lo + __popc(__ballot_sync(0xffffffffu, less));
            if (lane == 0) s_center = pos;
        }
        if (tid == 0) {
            double4 b = make_double4(INFINITY, INFINITY, -INFINITY, -INFINITY);
            for (int w = 0; w < T_BLOCK / 32; w++) {
                b.x = fmin(b.x, s_b[0][w]);
                b.y = fmin(b.y, s_b[1][w]);
                b.z = fmax(b.z, s_b[2][w]);
                b.w = fmax(b.w, s_b[3][w]);
            }
            s_qbox = b;
        }
        __syncthreads();  // every thread must see s_qbox: skip decisions are CTA-uniform
        n_tiles = (A.nt + T_TS - 1) / T_TS;
        t_first = 0;
        center = s_center / T_TS;
        if (center >= n_tiles) center = n_tiles - 1;
    } else {
        const int tb = blockIdx.y * A.chunk;
        const int te = min(A.nt, tb + A.chunk);
        t_first = tb;
        n_tiles = (te - tb + T_TS - 1) / T_TS;
    }
    float bound = INFINITY;  // CTA-wide worst upper bound (culled mode), scaled units
    // culled mode only needs SOME real target per source (any target's distance
    // is a valid upper bound for the exact pass), so it walks a few Morton
    // neighbours of the CTA and stops; full mode meets every target
    const int n_steps = CULL ? min(2 * n_tiles, A.cull_steps) : n_tiles;
    for (int k = 0; k < n_steps; k++) {
        int tile;
        if (CULL) {
            // outward walk: center, center+1, center-1, center+2, ... (each tile once)
            const int d = (k + 1) >> 1;
            tile = (k & 1) ? center + d : center - d;
            if (tile < 0 || tile >= n_tiles) continue;
            const double4 b = A.tbox[tile];
            const double4 qb = s_qbox;
            const double gx = fmax(0.0, fmax(b.x - qb.z, qb.x - b.z));
            const double gy = fmax(0.0, fmax(b.y - qb.w, qb.y - b.w));
            const double lb = sqrt(gx * gx + gy * gy) * sc;  // scaled units
            if (lb * (1.0 - 1e-6) > (double)bound) continue;
        } else {
            tile = k;
        }
        const int tb = CULL ? tile * T_TS : t_first + tile * T_TS;
        const int te = CULL ? min(A.nt, tb + T_TS) : min(min(A.nt, t_first + A.chunk), tb + T_TS);
        const int cnt = te - tb;
        __syncthreads();
        for (int j = tid; j < T_TS / 2; j += T_BLOCK) {
            float xa = 1e18f, ya = 1e18f, xb = 1e18f, yb = 1e18f;
            if (2 * j < cnt) {
                const double2 p = A.t[tb + 2 * j];
                xa = (float)((p.x - ox) * sc);
                ya = (float)((p.y - oy) * sc);
            }
            if (2 * j + 1 < cnt) {
                const double2 p = A.t[tb + 2 * j + 1];
                xb = (float)((p.x - ox) * sc);
                yb = (float)((p.y - oy) * sc);
            }
            if (CULL) {
                // direct form: targets stored negated, d = (q - t)^2 without cancellation
                s_xy[j] = make_float4(-xa, -xb, -ya, -yb);
            } else {
                s_xy[j] = make_float4(xa, xb, ya, yb);
                s_tt[j] = make_float2(fmaf(xa, xa, ya * ya), fmaf(xb, xb, yb * yb));
            }
        }
        __syncthreads();
        const int pairs = (cnt + 1) >> 1;
        if (A.evals && tid == 0) atomicAdd(A.evals, (unsigned long long)(T_BLOCK * R) * (unsigned long long)(2 * pairs));
#pragma unroll 4
        for (int j = 0; j < pairs; j++) {
            const float4 v = s_xy[j];
            const float2 tx = make_float2(v.x, v.y), ty = make_float2(v.z, v.w);
            if (CULL) {
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const float2 dx = __fadd2_rn(ax[r], tx), dy = __fadd2_rn(ay[r], ty);
                    const float2 d = __ffma2_rn(dy, dy, __fmul2_rn(dx, dx));
                    m[r] = min3(m[r], d.x, d.y);
                }
            } else if (PACKQ) {
                // two SOURCES per packed lane pair, each target broadcast: the target's
                // operands are shared by every source pair (register reuse), the sources'
                // pairs are (-2x_r, -2x_r+1)
                const float2 tt = s_tt[j];
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const float2 qx = make_float2(ax[r].x, ax[r + 1].x), qy = make_float2(ay[r].x, ay[r + 1].x);
                    const float2 sa = __ffma2_rn(qy, make_float2(v.z, v.z),
                                                 __ffma2_rn(qx, make_float2(v.x, v.x), make_float2(tt.x, tt.x)));
                    const float2 sb = __ffma2_rn(qy, make_float2(v.w, v.w),
                                                 __ffma2_rn(qx, make_float2(v.y, v.y), make_float2(tt.y, tt.y)));
                    m[r] = min3(m[r], sa.x, sb.x);
                    m[r + 1] = min3(m[r + 1], sa.y, sb.y);
                }
            } else {
                const float2 tt = s_tt[j];
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const float2 s = __ffma2_rn(ay[r], ty, __ffma2_rn(ax[r], tx, tt));
                    m[r] = min3(m[r], s.x, s.y);
                }
            }
        }
        if (CULL) {
            float ub = 0.f;
#pragma unroll
            for (int r = 0; r < R; r++) {
                const int i = q0 + r * T_BLOCK + tid;
                if (i < A.nq) ub = fmaxf(ub, sqrtf(m[r]) * (1.f + 0x1p-18f) + 0x1p-18f * qn[r]);
            }
            for (int o = 16; o; o >>= 1) ub = fmaxf(ub, __shfl_xor_sync(0xffffffffu, ub, o));
            if (lane == 0) s_red[wid] = ub;
            __syncthreads();
            float b2 = 0.f;
#pragma unroll
            for (int w = 0; w < T_BLOCK / 32; w++) b2 = fmaxf(b2, s_red[w]);
            bound = b2;
        }
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int i = q0 + r * T_BLOCK + tid;
        if (!CULL) {  // -2x and -2y are exact: x and y come back bit for bit
            const float x = -0.5f * ax[r].x, y = -0.5f * ay[r].x;
            qq[r] = fmaf(x, x, y * y);
            qn[r] = sqrtf(qq[r]);
        }
        if (i < A.nq) {
            const float est = CULL ? m[r] : fmaxf(m[r] + qq[r], 0.f);
            atomicMin(&A.mout[i], __float_as_uint(est));
            if (blockIdx.y == 0) A.qn_out[i] = qn[r];
        }
    }
}

__global__ void k_tile_boxes(const double2 *t, int nt, int T_TS, double4 *box) {
    const int lane = threadIdx.x & 31;
    const int ntile = (nt + T_TS - 1) / T_TS;
    for (int tile = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; tile < ntile;
         tile += (gridDim.x * blockDim.x) >> 5) {
        double x0 = INFINITY, y0 = INFINITY, x1 = -INFINITY, y1 = -INFINITY;
        const int te = min(nt, (tile + 1) * T_TS);
        for (int j = tile * T_TS + lane; j < te; j += 32) {
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

}  // namespace

// FP32 pass for one direction: sources q (nq, Morton order) against targets t
// (nt, Morton order).  mout (float bits, pre-set to +huge) receives the
// scaled squared-distance estimate, qn_out the local radius |q'|.
template <int R>
static int launch_full(Ctx &c, TileArgs &A, int64_t nq, int64_t nt);

int rwmd_f32_min(Ctx &c, const double2 *q, const uint64_t *qkey, int64_t nq, const double2 *t,
                 const uint64_t *tkey, int64_t nt, double scale, unsigned *mout, float *qn_out, double4 *tbox,
                 int culling, int tbox_ready) {
    if (nq == 0 || nt == 0) return W1G_OK;
    TileArgs A;
    A.q = q;
    A.t = t;
    A.tbox = tbox;
    A.qkey = qkey;
    A.tkey = tkey;
    A.nq = (int)nq;
    A.nt = (int)nt;
    A.scale = scale;
    A.mout = mout;
    A.qn_out = qn_out;
    A.evals = c.prof ? ptr<unsigned long long>(c.prof_cnt) + 2 * c.prof_side : nullptr;
    // tiles walked per CTA in culled mode: the centre tile and its two Morton
    // neighbours (measured: 3 seeds cfg2 and 1M points as tightly as 5 -- same
    // exact-pass time -- while 1-2 do not; the few sources a short walk leaves
    // with a poor seed are caught by the exact pass's heavy-source path)
    A.cull_steps = c.cull_steps > 0 ? c.cull_steps : 3;
    if (culling) {
        // (the caller may have computed the tile boxes already: rwmd.cu k_side_boxes, 4 x 64 = TS_CULL)
        static_assert(TS_CULL == 256, "k_side_boxes builds 256-target tile boxes");
        if (!tbox_ready) {
            const int ntile = (int)((nt + TS_CULL - 1) / TS_CULL);
            k_tile_boxes<<<grid_for((int64_t)ntile * 32, 256, 8u * c.sm_count), 256, 0, c.stream>>>(t, (int)nt, TS_CULL,
                                                                                                   tbox);
            W1G_CHECK_LAUNCH();
        }
        // sources per thread: 1 below ~300k sources (twice the CTAs of R = 2 for a short,
        // latency-bound kernel), 2 above; W1G_TILE_R overrides (tuning).  Any R is exact:
        // the seed only sizes the exact pass's search (rwmd.cu)
        static const int r_env = [] {
            const char *e = getenv("W1G_TILE_R");
            return e ? atoi(e) : 0;
        }();
        const int R = r_env == 1 || r_env == 2 ? r_env : (nq <= 300000 ? 1 : 2);
        const int gx = (int)((nq + T_BLOCK * R - 1) / (T_BLOCK * R));
        A.chunk = (int)nt;
        if (c.prof) W1G_CUDA(cudaEventRecord(c.prof_ev[c.prof_side][0][0], c.stream));
        if (R == 1)
            k_rwmd_f32<1, true, TS_CULL><<<gx, T_BLOCK, 0, c.stream>>>(A);
        else
            k_rwmd_f32<2, true, TS_CULL><<<gx, T_BLOCK, 0, c.stream>>>(A);
        W1G_CHECK_LAUNCH();
        if (c.prof) W1G_CUDA(cudaEventRecord(c.prof_ev[c.prof_side][0][1], c.stream));
        return W1G_OK;
    }
    static const int rfull = [] {  // W1G_TILE_RFULL=16: 16 sources per thread (tuning)
        const char *e = getenv("W1G_TILE_RFULL");
        return e && atoi(e) == 16 ? 16 : 8;
    }();
    if (rfull == 16) return launch_full<16>(c, A, nq, nt);
    return launch_full<8>(c, A, nq, nt);
}

template <int R>
static int launch_full(Ctx &c, TileArgs &A, int64_t nq, int64_t nt) {
    const int per_block = T_BLOCK * R;
    const int gx = (int)((nq + per_block - 1) / per_block);
    // the target range is split over grid.y so that the CTAs fill whole waves of the
    // resident slots (occupancy x SMs): the smallest split giving at least two waves at
    // >= 97 % wave efficiency (waves / ceil(waves)), else the most efficient split up to
    // 64 chunks (round 2: a fixed 16 x SMs target gave 4.13 waves at 1M, 17 % idle tail)
    static const bool packq = [] {  // W1G_TILE_PACKQ: sources packed in the FP32x2 lanes (1) or targets (0)
        const char *e = getenv("W1G_TILE_PACKQ");
        return !(e && atoi(e) == 0);
    }();
    void (*kern)(TileArgs) = packq ? k_rwmd_f32<R, false, TS_FULL, true> : k_rwmd_f32<R, false, TS_FULL, false>;
    static const int occ = [kern] {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, T_BLOCK, 0) != cudaSuccess || o < 1) {
            cudaGetLastError();
            o = 1;
        }
        return o;
    }();
    const int64_t slots = (int64_t)occ * c.sm_count;
    int64_t max_gy = (nt + TS_FULL - 1) / TS_FULL;
    if (max_gy > 65535) max_gy = 65535;
    if (max_gy < 1) max_gy = 1;
    int gy = 1;
    double best_eff = -1.0;
    for (int y = 1; y <= max_gy && y <= 64; y++) {
        const double waves = (double)gx * y / (double)slots;
        const double eff = waves / std::ceil(waves);
        if (waves >= 2.0 && eff >= 0.97) {
            gy = y;
            break;
        }
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            gy = y;
        }
    }
    int chunk = (int)((nt + gy - 1) / gy);
    chunk = (chunk + 1) & ~1;
    gy = (int)((nt + chunk - 1) / chunk);
    A.chunk = chunk;
    if (c.prof) W1G_CUDA(cudaEventRecord(c.prof_ev[c.prof_side][0][0], c.stream));
    kern<<<dim3(gx, gy), T_BLOCK, 0, c.stream>>>(A);
    W1G_CHECK_LAUNCH();
    if (c.prof) W1G_CUDA(cudaEventRecord(c.prof_ev[c.prof_side][0][1], c.stream));
    return W1G_OK;
}

}  // namespace w1g
