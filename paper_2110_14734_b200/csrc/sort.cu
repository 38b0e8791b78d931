// sort.cu -- stable LSD radix sort (8-bit digits) with a uint32 payload.
//
// Replaces the sorts inside np.unique(axis=0) (diagram.py:203,
// condensation.py:114) and np.lexsort (network.py:70).  One histogram pass
// computes every digit's global histogram; digits that are constant over
// all keys are skipped.  Each remaining digit is one count -> per-bin scan ->
// stable scatter pass.  Stability inside a tile comes from warp match-any
// ranking in index order, so equal keys keep their input order (np.unique
// keeps the first occurrence; np.lexsort is stable).
#include "common.cuh"

namespace w1g {

namespace {

constexpr int RS_BLOCK = 256;
constexpr int RS_WARPS = RS_BLOCK / 32;
constexpr int RS_IPT = 16;
constexpr int RS_TILE = RS_BLOCK * RS_IPT;
constexpr int RS_WTILE = 32 * RS_IPT;  // items per warp

struct KeyPtrs {
    uint64_t *k[4];
};

__global__ void __launch_bounds__(512) k_rs_hist_all(KeyPtrs kp, int words, int64_t n,
                                                     uint32_t *hist) {
    extern __shared__ uint32_t sh[];  // words*8*256
    const int nb = words * 8 * 256;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int w = 0; w < words; w++) {
            uint64_t key = kp.k[w][i];
#pragma unroll
            for (int j = 0; j < 8; j++) atomicAdd(&sh[(w * 8 + j) * 256 + (int)((key >> (8 * j)) & 255)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void __launch_bounds__(RS_BLOCK) k_rs_count(const uint64_t *__restrict__ kw, int shift,
                                                       int64_t n, uint32_t *counts, int ntiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int i = 0; i < RS_IPT; i++) {
        int64_t idx = base + i * RS_BLOCK + threadIdx.x;
        if (idx < n) atomicAdd(&h[(int)((kw[idx] >> shift) & 255)], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// one block per bin: offsets[b][t] = sum_{b'<b} hist[b'] + sum_{t'<t} counts[b][t']
__global__ void __launch_bounds__(1024) k_rs_binscan(uint32_t *counts, const uint32_t *dhist,
                                                     int ntiles) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        uint32_t base = 0;
        for (int i = 0; i < b; i++) base += dhist[i];
        s_carry = base;
    }
    __syncthreads();
    uint32_t *row = counts + (int64_t)b * ntiles;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int start = 0; start < ntiles; start += 1024) {
        int t = start + threadIdx.x;
        uint32_t v = t < ntiles ? row[t] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            s_warp[lane] = w;
        }
        __syncthreads();
        uint32_t excl = (wid ? s_warp[wid - 1] : 0) + x - v;
        uint32_t carry = s_carry;
        if (t < ntiles) row[t] = carry + excl;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + s_warp[31];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(RS_BLOCK) k_rs_scatter(KeyPtrs src, KeyPtrs dst, int wfirst,
                                                         int words, const uint32_t *__restrict__ vsrc,
                                                         uint32_t *__restrict__ vdst, int dword,
                                                         int shift, const uint32_t *__restrict__ offsets,
                                                         int ntiles, int64_t n) {
    __shared__ uint32_t whist[RS_WARPS][257];
    __shared__ uint32_t toff[256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    toff[threadIdx.x] = offsets[(int64_t)threadIdx.x * ntiles + blockIdx.x];
    for (int w = 0; w < RS_WARPS; w++) whist[w][threadIdx.x] = 0;
    if (threadIdx.x < RS_WARPS) whist[threadIdx.x][256] = 0;
    __syncthreads();
    const uint64_t *kd = src.k[dword];
    const int64_t wbase = (int64_t)blockIdx.x * RS_TILE + wid * RS_WTILE;
    const unsigned lt = lanemask_lt();
    uint32_t rank[RS_IPT];
    uint16_t dig[RS_IPT];
#pragma unroll
    for (int i = 0; i < RS_IPT; i++) {
        int64_t idx = wbase + i * 32 + lane;
        int d = idx < n ? (int)((kd[idx] >> shift) & 255) : 256;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t b = whist[wid][d];
        __syncwarp();
        if ((__ffs(peers) - 1) == lane) whist[wid][d] = b + __popc(peers);
        __syncwarp();
        rank[i] = b + __popc(peers & lt);
        dig[i] = (uint16_t)d;
    }
    __syncthreads();
    {  // exclusive prefix over warps for each bin
        uint32_t run = 0;
        for (int w = 0; w < RS_WARPS; w++) {
            uint32_t t = whist[w][threadIdx.x];
            whist[w][threadIdx.x] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RS_IPT; i++) {
        int64_t idx = wbase + i * 32 + lane;
        if (idx < n) {
            int d = dig[i];
            uint32_t pos = toff[d] + whist[wid][d] + rank[i];
            for (int w = wfirst; w < words; w++) dst.k[w][pos] = src.k[w][idx];
            vdst[pos] = vsrc[idx];
        }
    }
}

}  // namespace

int radix_sort(Ctx &c, uint64_t **keys, int words, uint32_t *vals, int64_t n, int top_bits) {
    if (n <= 1) return W1G_OK;
    if (words < 1 || words > 4 || n > 0xffffffffll) {
        set_error("radix_sort: unsupported shape (words=%d, n=%lld)", words, (long long)n);
        return W1G_EINVAL;
    }
    const int ntiles = (int)((n + RS_TILE - 1) / RS_TILE);
    KeyPtrs a, b;
    for (int w = 0; w < 4; w++) a.k[w] = b.k[w] = nullptr;
    for (int w = 0; w < words; w++) {
        a.k[w] = keys[w];
        W1G_TRY(ensure(c.sort_scr[w], (size_t)n, &b.k[w]));
    }
    uint32_t *va = vals, *vb, *hist, *counts;
    W1G_TRY(ensure(c.sort_scr[4], (size_t)n, &vb));
    W1G_TRY(ensure(c.sort_scr[5], (size_t)words * 8 * 256, &hist));
    W1G_TRY(ensure(c.sort_scr[6], (size_t)ntiles * 256, &counts));
    W1G_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * words * 8 * 256, c.stream));
    {
        unsigned g = grid_for(n, 512, 2u * c.sm_count);
        size_t sm = sizeof(uint32_t) * words * 8 * 256;
        if (sm > 48 * 1024)
            W1G_CUDA(cudaFuncSetAttribute(k_rs_hist_all, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_rs_hist_all<<<g, 512, sm, c.stream>>>(a, words, n, hist);
        W1G_CHECK_LAUNCH();
    }
    W1G_TRY(stage_ensure(c, sizeof(uint32_t) * words * 8 * 256));
    uint32_t *hh = static_cast<uint32_t *>(c.h_stage);
    W1G_CUDA(cudaMemcpyAsync(hh, hist, sizeof(uint32_t) * words * 8 * 256, cudaMemcpyDeviceToHost, c.stream));
    W1G_CUDA(cudaStreamSynchronize(c.stream));
    int passes[32];
    int np = 0;
    for (int w = 0; w < words; w++) {
        int jmax = (w == words - 1) ? (top_bits + 7) / 8 : 8;
        for (int j = 0; j < jmax && j < 8; j++) {
            const uint32_t *h = hh + (w * 8 + j) * 256;
            bool uniform = false;
            for (int q = 0; q < 256; q++)
                if (h[q] == (uint32_t)n) { uniform = true; break; }
            if (!uniform) passes[np++] = w * 8 + j;
        }
    }
    KeyPtrs *src = &a, *dst = &b;
    uint32_t *vsrc = va, *vdst = vb;
    for (int p = 0; p < np; p++) {
        const int w = passes[p] / 8, shift = 8 * (passes[p] % 8);
        k_rs_count<<<ntiles, RS_BLOCK, 0, c.stream>>>(src->k[w], shift, n, counts, ntiles);
        W1G_CHECK_LAUNCH();
        k_rs_binscan<<<256, 1024, 0, c.stream>>>(counts, hist + (w * 8 + shift / 8) * 256, ntiles);
        W1G_CHECK_LAUNCH();
        k_rs_scatter<<<ntiles, RS_BLOCK, 0, c.stream>>>(*src, *dst, w, words, vsrc, vdst, w, shift,
                                                        counts, ntiles, n);
        W1G_CHECK_LAUNCH();
        KeyPtrs *t = src;
        src = dst;
        dst = t;
        uint32_t *tv = vsrc;
        vsrc = vdst;
        vdst = tv;
    }
    if (vsrc != vals) {
        // result lives in the scratch buffers: copy the payload and the top key word back
        W1G_CUDA(cudaMemcpyAsync(vals, vsrc, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, c.stream));
        W1G_CUDA(cudaMemcpyAsync(keys[words - 1], src->k[words - 1], sizeof(uint64_t) * n,
                                 cudaMemcpyDeviceToDevice, c.stream));
    }
    return W1G_OK;
}

}  // namespace w1g
