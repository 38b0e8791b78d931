// sort.cu -- stable LSD radix sort (8-bit digits) with a uint32 payload.
//
// Replaces the sorts inside np.unique(axis=0) (diagram.py:203,
// condensation.py:114) and np.lexsort (network.py:70).
//
//  * one histogram kernel computes every digit's global histogram; digits
//    that are constant over all keys are skipped (one 2-8 KB D2H per sort);
//  * each remaining digit is ONE "onesweep" kernel: a tile (4096 keys) ranks
//    its keys stably with warp match-any in index order, publishes its
//    per-digit counts, looks back over earlier tiles (decoupled look-back,
//    epoch-tagged status words, so nothing is re-zeroed between passes),
//    stages the tile in shared memory in digit order and writes it out with
//    coalesced stores.
// Equal keys keep their input order (np.unique keeps the first occurrence,
// np.lexsort is stable).
#include "common.cuh"

namespace w1g {

namespace {

constexpr int RS_BLOCK = 256;
constexpr int RS_WARPS = RS_BLOCK / 32;
// items per thread: 8 (2048-key tiles) in general, 32 (8192-key tiles) for
// large inputs so the decoupled look-back chain stays short
constexpr int RS_IPT_SMALL = 8;
constexpr int RS_IPT_LARGE = 32;
constexpr int64_t RS_LARGE_N = 1 << 20;

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

// status word: [epoch (30 bits) | kind (2 bits) | count (32 bits)]
constexpr unsigned long long ST_AGG = 1, ST_INC = 2;

__device__ __forceinline__ unsigned long long st_make(unsigned epoch, unsigned long long kind, uint32_t cnt) {
    return ((unsigned long long)epoch << 34) | (kind << 32) | cnt;
}

template <int W, int M, int RS_IPT>
__global__ void __launch_bounds__(RS_BLOCK) k_rs_onesweep(KeyPtrs src, KeyPtrs dst,
                                                          const uint32_t *__restrict__ vsrc,
                                                          uint32_t *__restrict__ vdst, int shift,
                                                          const uint32_t *__restrict__ dhist,
                                                          unsigned long long *status, unsigned *ticket,
                                                          unsigned epoch, int64_t n) {
    constexpr int DW = W - M;  // word holding the digit; words DW..W-1 move
    constexpr int RS_TILE = RS_BLOCK * RS_IPT;
    constexpr int RS_WTILE = 32 * RS_IPT;  // items per warp
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t *s_key = reinterpret_cast<uint64_t *>(smem);           // M * RS_TILE
    uint32_t *s_val = reinterpret_cast<uint32_t *>(s_key + M * RS_TILE);  // RS_TILE
    __shared__ uint32_t whist[RS_WARPS][257];
    __shared__ uint32_t t_start[256];  // tile-local exclusive start of each digit
    __shared__ uint32_t g_base[256];   // global output start of this tile's digit run
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    for (int w = 0; w < RS_WARPS; w++) whist[w][tid] = 0;
    if (tid < RS_WARPS) whist[tid][256] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t tbase = tile * RS_TILE;
    const int tn = (n - tbase) < RS_TILE ? (int)(n - tbase) : RS_TILE;
    const uint64_t *kd = src.k[DW];
    const unsigned lt = lanemask_lt();

    // 1. stable rank inside the tile (warp w owns items [w*512, (w+1)*512), striped)
    uint16_t rank[RS_IPT];
    uint16_t dig[RS_IPT];
    // issue every load of the tile before the (warp-synchronous) ranking loop
#pragma unroll
    for (int i = 0; i < RS_IPT; i++) {
        const int li = wid * RS_WTILE + i * 32 + lane;
        dig[i] = li < tn ? (uint16_t)((kd[tbase + li] >> shift) & 255) : (uint16_t)256;
    }
#pragma unroll
    for (int i = 0; i < RS_IPT; i++) {
        const int d = dig[i];
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t b = whist[wid][d];
        __syncwarp();
        if ((__ffs(peers) - 1) == lane) whist[wid][d] = b + __popc(peers);
        __syncwarp();
        rank[i] = (uint16_t)(b + __popc(peers & lt));
    }
    __syncthreads();
    // 2. per-digit tile counts, warp prefixes, tile-local digit starts
    uint32_t cnt = 0;
    for (int w = 0; w < RS_WARPS; w++) {
        const uint32_t t = whist[w][tid];
        whist[w][tid] = cnt;
        cnt += t;
    }
    // publish this tile's count for digit `tid` as early as possible
    if (tile > 0) atomicExch(&status[tile * 256 + tid], st_make(epoch, ST_AGG, cnt));
    uint32_t hbase;
    {  // block exclusive scans over digits: tile counts -> t_start, global histogram -> hbase
        const uint32_t hd = dhist[tid];
        uint32_t x = cnt, y = hd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, x, o);
            const uint32_t b = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) {
                x += a;
                y += b;
            }
        }
        __shared__ uint32_t s_w[RS_WARPS], s_h[RS_WARPS];
        if (lane == 31) {
            s_w[wid] = x;
            s_h[wid] = y;
        }
        __syncthreads();
        uint32_t off = 0, hoff = 0;
        for (int w = 0; w < wid; w++) {
            off += s_w[w];
            hoff += s_h[w];
        }
        t_start[tid] = off + x - cnt;
        hbase = hoff + y - hd;
    }
    // 3. decoupled look-back per digit (thread `tid` handles digit `tid`); a
    //    window of predecessors is loaded at once so a walk over published
    //    aggregates costs one memory latency per LB_W tiles, not per tile
    {
        constexpr int LB_W = 16;
        uint32_t prefix = 0;
        int64_t j = tile - 1;
        while (j >= 0) {
            unsigned long long s[LB_W];
#pragma unroll
            for (int w = 0; w < LB_W; w++)
                s[w] = (j - w >= 0) ? *((volatile unsigned long long *)&status[(j - w) * 256 + tid]) : 0ull;
            int used = 0;
            bool done = false;
#pragma unroll
            for (int w = 0; w < LB_W; w++) {
                if (done || used < w) break;
                if (j - w < 0 || (unsigned)(s[w] >> 34) != epoch) break;  // not published yet
                prefix += (uint32_t)s[w];
                used = w + 1;
                if (((s[w] >> 32) & 3) == ST_INC) done = true;
            }
            if (done) break;
            j -= used;  // consumed aggregates; re-poll from the first unpublished tile
        }
        atomicExch(&status[tile * 256 + tid], st_make(epoch, ST_INC, prefix + cnt));
        // global start of digit `tid`: smaller digits over all keys + this digit in earlier tiles
        g_base[tid] = hbase + prefix;
    }
    __syncthreads();
    // 4. stage the tile in digit order
#pragma unroll
    for (int i = 0; i < RS_IPT; i++) {
        const int li = wid * RS_WTILE + i * 32 + lane;
        if (li < tn) {
            const int d = dig[i];
            const int lp = t_start[d] + whist[wid][d] + rank[i];
#pragma unroll
            for (int m = 0; m < M; m++) s_key[m * RS_TILE + lp] = src.k[DW + m][tbase + li];
            s_val[lp] = vsrc[tbase + li];
        }
    }
    __syncthreads();
    // 5. coalesced write-out: consecutive staged items of one digit go to consecutive addresses
    for (int j = tid; j < tn; j += RS_BLOCK) {
        const uint64_t k0 = s_key[j];
        const int d = (int)((k0 >> shift) & 255);
        const uint32_t pos = g_base[d] + (uint32_t)j - t_start[d];
#pragma unroll
        for (int m = 0; m < M; m++) dst.k[DW + m][pos] = s_key[m * RS_TILE + j];
        vdst[pos] = s_val[j];
    }
}

template <int W, int M, int IPT>
int launch_pass(Ctx &c, KeyPtrs *src, KeyPtrs *dst, const uint32_t *vsrc, uint32_t *vdst, int shift,
                const uint32_t *dhist, unsigned long long *status, unsigned *ticket, unsigned epoch,
                int64_t n) {
    const int64_t tile = (int64_t)RS_BLOCK * IPT;
    const int ntiles = (int)((n + tile - 1) / tile);
    const size_t sm = (size_t)tile * (8 * M + 4);
    W1G_CUDA(cudaFuncSetAttribute(k_rs_onesweep<W, M, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_rs_onesweep<W, M, IPT><<<ntiles, RS_BLOCK, sm, c.stream>>>(*src, *dst, vsrc, vdst, shift, dhist, status,
                                                                ticket, epoch, n);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

int dispatch_pass(int W, int M, Ctx &c, KeyPtrs *src, KeyPtrs *dst, const uint32_t *vsrc, uint32_t *vdst,
                  int shift, const uint32_t *dhist, unsigned long long *status, unsigned *ticket,
                  unsigned epoch, int64_t n) {
    // large inputs: 8192-key tiles when the staged words fit in shared memory
    const bool large = n >= RS_LARGE_N && M <= 2;
#define RS_CASE(w, m)                                                                                          \
    if (W == w && M == m)                                                                                      \
        return large ? launch_pass<w, m, RS_IPT_LARGE>(c, src, dst, vsrc, vdst, shift, dhist, status, ticket,  \
                                                       epoch, n)                                               \
                     : launch_pass<w, m, RS_IPT_SMALL>(c, src, dst, vsrc, vdst, shift, dhist, status, ticket,  \
                                                       epoch, n);
    RS_CASE(1, 1)
    RS_CASE(2, 2)
    RS_CASE(2, 1)
    RS_CASE(3, 3)
    RS_CASE(3, 2)
    RS_CASE(3, 1)
#undef RS_CASE
    set_error("radix_sort: unsupported word count %d", W);
    return W1G_EINVAL;
}

}  // namespace

int radix_sort(Ctx &c, uint64_t **keys, int words, uint32_t *vals, int64_t n, int top_bits) {
    if (n <= 1) return W1G_OK;
    if (words < 1 || words > 3 || n > 0xffffffffll) {
        set_error("radix_sort: unsupported shape (words=%d, n=%lld)", words, (long long)n);
        return W1G_EINVAL;
    }
    const int64_t small_tile = (int64_t)RS_BLOCK * RS_IPT_SMALL;
    const int ntiles = (int)((n + small_tile - 1) / small_tile);  // upper bound for the status array
    KeyPtrs a, b;
    for (int w = 0; w < 4; w++) a.k[w] = b.k[w] = nullptr;
    for (int w = 0; w < words; w++) {
        a.k[w] = keys[w];
        W1G_TRY(ensure(c.sort_scr[w], (size_t)n, &b.k[w]));
    }
    uint32_t *va = vals, *vb, *hist;
    unsigned long long *status;
    W1G_TRY(ensure(c.sort_scr[4], (size_t)n, &vb));
    W1G_TRY(ensure(c.sort_scr[5], (size_t)words * 8 * 256 + 64, &hist));
    const size_t cap0 = c.sort_scr[6].cap;
    W1G_TRY(ensure(c.sort_scr[6], (size_t)ntiles * 256, &status));
    if (c.sort_scr[6].cap != cap0) {
        // fresh status words: make sure no stale bits can match an epoch
        W1G_CUDA(cudaMemsetAsync(status, 0, c.sort_scr[6].cap, c.stream));
        c.sort_epoch = 0;
    }
    unsigned *tickets = hist + words * 8 * 256;  // 64 per-pass tile tickets
    W1G_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (words * 8 * 256 + 64), c.stream));
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
                if (h[q] == (uint32_t)n) {
                    uniform = true;
                    break;
                }
            if (!uniform) passes[np++] = w * 8 + j;
        }
    }
    KeyPtrs *src = &a, *dst = &b;
    uint32_t *vsrc = va, *vdst = vb;
    for (int p = 0; p < np; p++) {
        const int w = passes[p] / 8, j = passes[p] % 8;
        c.sort_epoch = (c.sort_epoch + 1) & 0x3fffffffu;
        if (c.sort_epoch == 0) c.sort_epoch = 1;
        W1G_TRY(dispatch_pass(words, words - w, c, src, dst, vsrc, vdst, 8 * j, hist + (w * 8 + j) * 256,
                              status, tickets + (p & 63), c.sort_epoch, n));
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

// ---------------------------------------------------------------- (primary, secondary) sort
//
// Stable sort by a 128-bit key (primary word, then secondary word) that only
// pays for the secondary word where primaries tie: one 64-bit radix sort by
// the primary, then the elements of tie runs (usually none for real-valued
// coordinates; everything for H0-style diagrams whose births are all 0) are
// sorted by (primary, secondary) and written back into their run slots.

namespace {

__global__ void k_copy_u64(const uint64_t *src, uint64_t *dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

struct TieFlag {
    const uint64_t *k;
    int64_t n;
    __device__ int64_t operator()(int64_t i) const {
        const uint64_t v = k[i];
        return ((i > 0 && k[i - 1] == v) || (i + 1 < n && k[i + 1] == v)) ? 1 : 0;
    }
};

__global__ void k_tie_gather(TieFlag f, const int64_t *excl, const uint32_t *vals, const uint64_t *sec,
                             uint32_t *tpos, uint64_t *kl, uint64_t *kh, uint32_t *pl) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < f.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!f(i)) continue;
        const int64_t r = excl[i];
        tpos[r] = (uint32_t)i;
        kh[r] = f.k[i];
        kl[r] = sec[vals[i]];
        pl[r] = (uint32_t)r;
    }
}

__global__ void k_tie_fetch(const uint32_t *tpos, const uint32_t *pl, const uint32_t *vals, int64_t t,
                            uint32_t *tmp) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < t;
         r += (int64_t)gridDim.x * blockDim.x)
        tmp[r] = vals[tpos[pl[r]]];
}

__global__ void k_tie_put(const uint32_t *tpos, const uint32_t *tmp, int64_t t, uint32_t *vals) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < t;
         r += (int64_t)gridDim.x * blockDim.x)
        vals[tpos[r]] = tmp[r];
}

}  // namespace

int sort_lex2(Ctx &c, const uint64_t *primary, const uint64_t *secondary, uint32_t *vals, int64_t n) {
    if (n <= 1) return W1G_OK;
    uint64_t *pk;
    int64_t *excl;
    W1G_TRY(ensure(c.lex_scr[0], (size_t)n, &pk));
    W1G_TRY(ensure(c.lex_scr[1], (size_t)n, &excl));
    const unsigned g = grid_for(n, 256, 8u * c.sm_count);
    k_copy_u64<<<g, 256, 0, c.stream>>>(primary, pk, n);
    W1G_CHECK_LAUNCH();
    uint64_t *k1[1] = {pk};
    W1G_TRY(radix_sort(c, k1, 1, vals, n, 64));
    TieFlag f{pk, n};
    int64_t *dt = ptr<int64_t>(c.flags) + F_MISC3;
    W1G_TRY(scan_i64(c, f, n, excl, dt));
    int64_t T = 0;
    W1G_CUDA(cudaMemcpyAsync(&c.h_pinned[F_MISC3], dt, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    W1G_CUDA(cudaStreamSynchronize(c.stream));
    T = c.h_pinned[F_MISC3];
    if (T == 0) return W1G_OK;
    uint32_t *tpos, *pl, *tmp;
    uint64_t *kl, *kh;
    W1G_TRY(ensure(c.lex_scr[2], (size_t)T, &tpos));
    W1G_TRY(ensure(c.lex_scr[3], (size_t)T, &kl));
    W1G_TRY(ensure(c.lex_scr[4], (size_t)T, &kh));
    W1G_TRY(ensure(c.lex_scr[5], (size_t)T * 2, &pl));
    tmp = pl + T;
    k_tie_gather<<<g, 256, 0, c.stream>>>(f, excl, vals, secondary, tpos, kl, kh, pl);
    W1G_CHECK_LAUNCH();
    uint64_t *k2[2] = {kl, kh};
    W1G_TRY(radix_sort(c, k2, 2, pl, T, 64));
    const unsigned gt = grid_for(T, 256, 8u * c.sm_count);
    k_tie_fetch<<<gt, 256, 0, c.stream>>>(tpos, pl, vals, T, tmp);
    W1G_CHECK_LAUNCH();
    k_tie_put<<<gt, 256, 0, c.stream>>>(tpos, tmp, T, vals);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

}  // namespace w1g

using namespace w1g;

// test hook: sort host keys (words x n, word 0 least significant) with the
// device radix sort and return the permutation (w1g_debug_radix_sort, w1g.h)
extern "C" int w1g_debug_radix_sort(w1g_ctx *c, const uint64_t *keys, int words, int64_t n,
                                    uint32_t *perm) {
    if (!c || words < 1 || words > 3 || n < 0) return W1G_EINVAL;
    W1G_CUDA(cudaSetDevice(c->device));
    uint64_t *k[3];
    uint32_t *v;
    for (int w = 0; w < words; w++) {
        W1G_TRY(ensure(c->scr[w], (size_t)n + 1, &k[w]));
        if (n) W1G_CUDA(cudaMemcpyAsync(k[w], keys + (size_t)w * n, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, c->stream));
    }
    W1G_TRY(ensure(c->scr[4], (size_t)n + 1, &v));
    W1G_TRY(stage_ensure(*c, sizeof(uint32_t) * (n + 1)));
    uint32_t *h = static_cast<uint32_t *>(c->h_stage);
    for (int64_t i = 0; i < n; i++) h[i] = (uint32_t)i;
    if (n) W1G_CUDA(cudaMemcpyAsync(v, h, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, c->stream));
    W1G_TRY(radix_sort(*c, k, words, v, n, 64));
    if (n) W1G_CUDA(cudaMemcpyAsync(perm, v, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    W1G_CUDA(cudaStreamSynchronize(c->stream));
    return W1G_OK;
}
