// pairwise_sum.cu -- numpy's pairwise summation (np.sum of a contiguous
// float64 vector, numpy/_core/src/umath/loops_utils.h.src pairwise_sum),
// used by lower_bound.py:58, rebuilt on device so the RWMD sum is
// bit-identical: the recursion tree (n < 8: sequential; n <= 128: eight
// strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail; else split at n2 = n/2 - (n/2)%8) is expanded level by
// level in one CTA, the leaves are summed one warp per leaf, and the
// internal nodes are combined bottom-up in tree order.
#include "common.cuh"

namespace w1g {

namespace {

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
    if (threadIdx.x == 0) {
        *n_levels = L;
        n_levels[1] = 0;  // the leaves kernel's block ticket (k_pw_sum)
    }
}

// one warp per leaf: numpy's 8-accumulator block (n <= 128) or sequential (n < 8); the
// last block to finish then combines the internal nodes level by level (bottom-up, the
// tree order numpy's recursion adds in) and writes the sum: one launch
__global__ void __launch_bounds__(256) k_pw_sum(const double *v, const PwNode *nodes, const int32_t *levels,
                                                int32_t *n_levels, double *val, double *out,
                                                volatile double *h_out) {
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
    // the last block to arrive combines (the other blocks' leaf sums read from L2)
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = atomicAdd(&n_levels[1], 1);
        s_last = t == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int L = *n_levels;
    for (int l = L - 1; l >= 0; l--) {
        for (int i = levels[l] + threadIdx.x; i < levels[l + 1]; i += blockDim.x) {
            const int ch = nodes[i].child;
            if (ch >= 0) val[i] = dadd(__ldcg(&val[ch]), __ldcg(&val[ch + 1]));
        }
        __threadfence();
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double r = __ldcg(&val[0]);
        *out = r;
        if (h_out) *h_out = r;
        n_levels[1] = 0;  // ready for the next sum over this tree
    }
}

}  // namespace

// np.sum of a contiguous float64 vector on device -> *d_out (device)
// (h_out, optional: page-locked host memory the sum is also written to, by the same kernel)
int pairwise_sum(Ctx &c, const double *d_v, int64_t n, double *d_out, DevBuf &nodes_buf,
                 DevBuf &val_buf, DevBuf &lev_buf, int64_t *cached_n, double *h_out) {
    if (n == 0) {
        if (h_out) *h_out = 0.0;
        W1G_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), c.stream));
        return W1G_OK;
    }
    const int64_t cap = n / 32 + 64;
    PwNode *nodes;
    double *val;
    int32_t *lev;
    W1G_TRY(ensure(nodes_buf, (size_t)cap, &nodes));
    W1G_TRY(ensure(val_buf, (size_t)cap, &val));
    W1G_TRY(ensure(lev_buf, PW_MAX_LEVELS + 2, &lev));  // levels, their count, the block ticket
    // the tree is a function of n alone: kept across calls when the caller owns the buffers
    if (!cached_n || *cached_n != n) {
        k_pw_build<<<1, 1024, 0, c.stream>>>(n, nodes, lev, lev + PW_MAX_LEVELS);
        W1G_CHECK_LAUNCH();
        if (cached_n) *cached_n = n;
    }
    const unsigned warps = (unsigned)(n / 64 + 2);
    k_pw_sum<<<grid_for(warps * 32, 256, 4u * c.sm_count), 256, 0, c.stream>>>(d_v, nodes, lev, lev + PW_MAX_LEVELS,
                                                                               val, d_out, h_out);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

}  // namespace w1g
