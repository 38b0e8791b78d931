// rwmd_tile.cu -- the FP32 all-pairs nearest-neighbour tile pass of RWMD.
//
// For every source q (scaled frame, |q| < 1) computes min over all targets t
// of fl32(dx*dx + dy*dy) -- the "tiled all-pairs nearest-neighbour min" of the
// north star, on the FP32 pipe (a min over a distance is not a contraction,
// so no tensor cores).  Each thread keeps R sources in registers, targets
// stream through shared memory in tiles and are broadcast to the warp; the
// target range is split across grid.y so the grid fills all 148 SMs, and the
// per-chunk minima are merged with an order-independent atomicMin on the
// float bits (non-negative floats order like their bit patterns).
//
// The result only sizes the exact fp64 search in rwmd.cu: its error is
// bounded by |d_f32 - d| <= 2^-21 (1 + d) in the scaled frame.
//
// This translation unit is compiled with FMA contraction allowed; nothing
// here feeds a reference-parity value directly.
#include "common.cuh"

namespace w1g {

namespace {

constexpr int T_BLOCK = 256;
constexpr int T_R = 8;        // sources per thread
constexpr int T_TILE = 2048;  // targets per shared-memory tile

__global__ void __launch_bounds__(T_BLOCK) k_rwmd_f32(const float2 *__restrict__ q, int nq,
                                                      const float2 *__restrict__ t, int nt,
                                                      int chunk, unsigned *__restrict__ mout) {
    __shared__ float4 s_t[T_TILE / 2];
    const int q0 = blockIdx.x * (T_BLOCK * T_R) + threadIdx.x;
    float qx[T_R], qy[T_R], m[T_R];
#pragma unroll
    for (int r = 0; r < T_R; r++) {
        int i = q0 + r * T_BLOCK;
        float2 p = i < nq ? q[i] : make_float2(0.f, 0.f);
        qx[r] = p.x;
        qy[r] = p.y;
        m[r] = INFINITY;
    }
    const int t_begin = blockIdx.y * chunk;
    const int t_end = min(nt, t_begin + chunk);
    for (int tb = t_begin; tb < t_end; tb += T_TILE) {
        const int cnt = min(T_TILE, t_end - tb);
        __syncthreads();
        for (int j = threadIdx.x; j < T_TILE / 2; j += T_BLOCK) {
            float2 a = 2 * j < cnt ? t[tb + 2 * j] : make_float2(INFINITY, INFINITY);
            float2 b = 2 * j + 1 < cnt ? t[tb + 2 * j + 1] : make_float2(INFINITY, INFINITY);
            s_t[j] = make_float4(a.x, a.y, b.x, b.y);
        }
        __syncthreads();
        const int pairs = (cnt + 1) >> 1;
#pragma unroll 4
        for (int j = 0; j < pairs; j++) {
            const float4 tt = s_t[j];
#pragma unroll
            for (int r = 0; r < T_R; r++) {
                float dx = qx[r] - tt.x, dy = qy[r] - tt.y;
                float d = fmaf(dy, dy, dx * dx);
                float ex = qx[r] - tt.z, ey = qy[r] - tt.w;
                float e = fmaf(ey, ey, ex * ex);
                m[r] = fminf(m[r], fminf(d, e));
            }
        }
    }
#pragma unroll
    for (int r = 0; r < T_R; r++) {
        int i = q0 + r * T_BLOCK;
        if (i < nq) atomicMin(&mout[i], __float_as_uint(m[r]));
    }
}

}  // namespace

int rwmd_f32_min(Ctx &c, const float2 *q, int64_t nq, const float2 *t, int64_t nt, unsigned *mout,
                 int culling) {
    (void)culling;
    if (nq == 0 || nt == 0) return W1G_OK;
    const int per_block = T_BLOCK * T_R;
    const int gx = (int)((nq + per_block - 1) / per_block);
    // enough CTAs for ~4 waves of 4 resident CTAs per SM
    const int want = 16 * c.sm_count;
    int gy = (want + gx - 1) / gx;
    int64_t max_gy = (nt + T_TILE - 1) / T_TILE;
    if (gy > max_gy) gy = (int)max_gy;
    if (gy < 1) gy = 1;
    if (gy > 65535) gy = 65535;
    int chunk = (int)((nt + gy - 1) / gy);
    chunk = (chunk + 1) & ~1;
    gy = (int)((nt + chunk - 1) / chunk);
    dim3 grid(gx, gy);
    k_rwmd_f32<<<grid, T_BLOCK, 0, c.stream>>>(q, (int)nq, t, (int)nt, chunk, mout);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

}  // namespace w1g
