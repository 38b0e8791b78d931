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
// items per thread: 4 (1024-key tiles: 8 CTAs per SM, measured best for the
// 10^4-10^5-key sorts of the front end) in general, 32 (8192-key tiles) for
// large inputs so the decoupled look-back chain stays short
constexpr int RS_IPT_SMALL = 4;
constexpr int RS_IPT_LARGE = 32;
constexpr int64_t RS_LARGE_N = 1 << 19;  // measured: 1M-key Morton sorts -37 us, 342k-key tree sorts unchanged

struct KeyPtrs {
    uint64_t *k[4];
};

// digit histograms of every word of up to two jobs (blockIdx.y = job) in one launch
struct HistArgs {
    KeyPtrs kp[2];
    int64_t n[2];
    uint32_t *hist[2];
};
__global__ void __launch_bounds__(512) k_rs_hist_all(HistArgs H, int words) {
    extern __shared__ uint32_t sh[];  // words*8*256
    const KeyPtrs kp = H.kp[blockIdx.y];
    const int64_t n = H.n[blockIdx.y];
    uint32_t *hist = H.hist[blockIdx.y];
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

// One pass over up to RS_JOBS independent sorts (same word count, same digit):
// tiles [tile0[j], tile0[j+1]) of the launch belong to job j, so two small
// sorts share one launch and fill twice the SMs.
constexpr int RS_JOBS = 2;
struct PassJob {
    KeyPtrs a, b;                  // the two key buffers (ping-pong)
    uint32_t *va, *vb;             // the two payload buffers
    const int8_t *plan;            // this digit's plan entry: -1 skip, 0 a->b, 1 b->a
    const uint32_t *dhist;         // this digit's global histogram
    unsigned long long *status;    // per-tile status words
    int64_t n;
};
struct PassArgs {
    PassJob j[RS_JOBS];
    int tile0[RS_JOBS + 1];
    int njobs, shift;
    unsigned *ticket;
    unsigned epoch;
};

template <int W, int M, int RS_IPT>
__global__ void __launch_bounds__(RS_BLOCK) k_rs_onesweep(const __grid_constant__ PassArgs A) {
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
    if (tid == 0) s_tile = atomicAdd(A.ticket, 1u);
    for (int w = 0; w < RS_WARPS; w++) whist[w][tid] = 0;
    if (tid < RS_WARPS) whist[tid][256] = 0;
    __syncthreads();
    const int jb = (A.njobs > 1 && (int)s_tile >= A.tile0[1]) ? 1 : 0;
    const PassJob &J = A.j[jb];
    // the digit plan is made on the device (k_rs_plan): a digit shared by every
    // key of this job is skipped without a host round trip
    const int par = *J.plan;
    if (par < 0) return;  // CTA-uniform
    const KeyPtrs &src = par ? J.b : J.a;
    const KeyPtrs &dst = par ? J.a : J.b;
    const uint32_t *vsrc = par ? J.vb : J.va;
    uint32_t *vdst = par ? J.va : J.vb;
    const int shift = A.shift;
    const int64_t n = J.n;
    unsigned long long *status = J.status;
    const int64_t tile = (int64_t)s_tile - A.tile0[jb];
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
    if (tile > 0) atomicExch(&status[tile * 256 + tid], st_make(A.epoch, ST_AGG, cnt));
    uint32_t hbase;
    {  // block exclusive scans over digits: tile counts -> t_start, global histogram -> hbase
        const uint32_t hd = J.dhist[tid];
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
                if (j - w < 0 || (unsigned)(s[w] >> 34) != A.epoch) break;  // not published yet
                prefix += (uint32_t)s[w];
                used = w + 1;
                if (((s[w] >> 32) & 3) == ST_INC) done = true;
            }
            if (done) break;
            j -= used;  // consumed aggregates; re-poll from the first unpublished tile
        }
        atomicExch(&status[tile * 256 + tid], st_make(A.epoch, ST_INC, prefix + cnt));
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

// digit plan per job: plan[j*RS_PLAN + d] = parity of the pass (-1: digit
// uniform over all keys, or beyond top_bits) and plan[j*RS_PLAN + 32] = the
// parity after the last pass (1: the result sits in the b buffers)
constexpr int RS_PLAN = 40;
struct PlanArgs {
    const uint32_t *hist[RS_JOBS];
    int64_t n[RS_JOBS];
    int njobs, words, top_bits;
    int8_t *plan;
};
__global__ void __launch_bounds__(1024) k_rs_plan(const __grid_constant__ PlanArgs A) {
    __shared__ int8_t act[RS_JOBS][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;  // one warp per (job, digit)
    for (int t = wid; t < RS_JOBS * 32; t += blockDim.x >> 5) {
        const int j = t / 32, d = t % 32;
        bool active = false;
        if (j < A.njobs) {
            const int w = d / 8;
            const int dmax = (w == A.words - 1) ? (A.top_bits + 7) / 8 : 8;
            if (w < A.words && d % 8 < dmax) {
                const uint32_t *h = A.hist[j] + d * 256;
                bool uniform = false;
#pragma unroll
                for (int q = 0; q < 8; q++) uniform |= h[q * 32 + lane] == (uint32_t)A.n[j];
                active = !__any_sync(0xffffffffu, uniform);
            }
        }
        if (lane == 0) act[j][d] = active;
    }
    __syncthreads();
    if (threadIdx.x < A.njobs) {
        const int j = threadIdx.x;
        int par = 0;
        for (int e = 0; e < 32; e++) {
            A.plan[j * RS_PLAN + e] = act[j][e] ? (int8_t)par : (int8_t)-1;
            par ^= act[j][e];
        }
        A.plan[j * RS_PLAN + 32] = (int8_t)par;
    }
}

// result in the b buffers (odd number of passes): copy payload and top key word back
// the sorted data back into the caller's buffers when the last pass left it in the scratch
// ones, for up to two jobs (blockIdx.y = job) in one launch
struct FixupArgs {
    const int8_t *final_par[2];
    const uint32_t *vb[2];
    uint32_t *va[2];
    const uint64_t *kb[2];
    uint64_t *ka[2];
    int64_t n[2];
};
__global__ void k_rs_fixup(FixupArgs F) {
    const int q = blockIdx.y;
    if (*F.final_par[q] == 0) return;
    const uint32_t *vb = F.vb[q];
    uint32_t *va = F.va[q];
    const uint64_t *kb = F.kb[q];
    uint64_t *ka = F.ka[q];
    const int64_t n = F.n[q];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        va[i] = vb[i];
        ka[i] = kb[i];
    }
}

template <int W, int M, int IPT>
int launch_pass(Ctx &c, PassArgs &A) {
    const int64_t tile = (int64_t)RS_BLOCK * IPT;
    A.tile0[0] = 0;
    for (int j = 0; j < A.njobs; j++) A.tile0[j + 1] = A.tile0[j] + (int)((A.j[j].n + tile - 1) / tile);
    const size_t sm = (size_t)tile * (8 * M + 4);
    W1G_CUDA(cudaFuncSetAttribute(k_rs_onesweep<W, M, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_rs_onesweep<W, M, IPT><<<A.tile0[A.njobs], RS_BLOCK, sm, c.stream>>>(A);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

int dispatch_pass(int W, int M, Ctx &c, PassArgs &A, bool large) {
#define RS_CASE(w, m)                                                                                          \
    if (W == w && M == m) return large ? launch_pass<w, m, RS_IPT_LARGE>(c, A) : launch_pass<w, m, RS_IPT_SMALL>(c, A);
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

int radix_sort_multi(Ctx &c, const SortJob *jobs, int njobs, int words, int top_bits) {
    if (njobs < 1 || njobs > RS_JOBS || words < 1 || words > 3) {
        set_error("radix_sort: unsupported shape (jobs=%d, words=%d)", njobs, words);
        return W1G_EINVAL;
    }
    // jobs with fewer than two keys are already sorted
    const SortJob *J[RS_JOBS];
    int nj = 0;
    for (int j = 0; j < njobs; j++) {
        if (jobs[j].n > 0xffffffffll) {
            set_error("radix_sort: %lld keys exceed the 32-bit payload", (long long)jobs[j].n);
            return W1G_EINVAL;
        }
        if (jobs[j].n > 1) J[nj++] = &jobs[j];
    }
    if (nj == 0) return W1G_OK;
    const int64_t small_tile = (int64_t)RS_BLOCK * RS_IPT_SMALL;
    const int nh = words * 8 * 256;
    KeyPtrs a[RS_JOBS], b[RS_JOBS];
    uint32_t *vb[RS_JOBS], *hist[RS_JOBS];
    unsigned long long *status[RS_JOBS];
    bool fresh = false;
    for (int j = 0; j < nj; j++) {
        const int64_t n = J[j]->n;
        const int ntiles = (int)((n + small_tile - 1) / small_tile);  // upper bound for the status array
        DevBuf *scr = c.sort_scr[j];
        for (int w = 0; w < 4; w++) a[j].k[w] = b[j].k[w] = nullptr;
        for (int w = 0; w < words; w++) {
            a[j].k[w] = J[j]->keys[w];
            W1G_TRY(ensure(scr[w], (size_t)n, &b[j].k[w]));
        }
        W1G_TRY(ensure(scr[4], (size_t)n, &vb[j]));
        W1G_TRY(ensure(scr[5], (size_t)nh + 64, &hist[j]));
        const size_t cap0 = scr[6].cap;
        W1G_TRY(ensure(scr[6], (size_t)ntiles * 256, &status[j]));
        fresh |= scr[6].cap != cap0;
    }
    if (fresh) {
        // fresh status words: no stale word of any job may match a future epoch
        for (auto &job : c.sort_scr)
            if (job[6].p) W1G_CUDA(cudaMemsetAsync(job[6].p, 0, job[6].cap, c.stream));
        c.sort_epoch = 0;
    }
    unsigned *tickets = hist[0] + nh;  // 64 per-pass tile tickets, shared by the jobs of a launch
    int8_t *plan;
    W1G_TRY(ensure(c.sort_scr[0][7], (size_t)RS_JOBS * RS_PLAN, &plan));
    W1G_CUDA(cudaMemsetAsync(tickets, 0, sizeof(unsigned) * 64, c.stream));
    PlanArgs P;
    P.njobs = nj;
    P.words = words;
    P.top_bits = top_bits;
    P.plan = plan;
    HistArgs H;
    int64_t nmax = 0;
    for (int j = 0; j < nj; j++) {
        W1G_CUDA(cudaMemsetAsync(hist[j], 0, sizeof(uint32_t) * nh, c.stream));
        H.kp[j] = a[j];
        H.n[j] = J[j]->n;
        H.hist[j] = hist[j];
        nmax = J[j]->n > nmax ? J[j]->n : nmax;
        P.hist[j] = hist[j];
        P.n[j] = J[j]->n;
    }
    {
        const size_t sm = sizeof(uint32_t) * nh;
        if (sm > 48 * 1024)
            W1G_CUDA(cudaFuncSetAttribute(k_rs_hist_all, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_rs_hist_all<<<dim3(grid_for(nmax, 512, 2u * c.sm_count), nj), 512, sm, c.stream>>>(H, words);
        W1G_CHECK_LAUNCH();
    }
    k_rs_plan<<<1, 1024, 0, c.stream>>>(P);
    W1G_CHECK_LAUNCH();
    // every digit that may be active is launched; the kernels of skipped digits exit at once
    const int ndig = (words - 1) * 8 + (top_bits + 7) / 8;
    int launch = 0;
    bool large = false;
    static const int64_t large_n = [] {  // W1G_RS_LARGE_N: tuning override
        const char *e = getenv("W1G_RS_LARGE_N");
        return e ? (int64_t)atoll(e) : RS_LARGE_N;
    }();
    for (int j = 0; j < nj; j++) large |= J[j]->n >= large_n;
    for (int dg = 0; dg < ndig; dg++) {
        PassArgs A;
        A.njobs = nj;
        for (int j = 0; j < nj; j++) {
            PassJob &Q = A.j[j];
            Q.a = a[j];
            Q.b = b[j];
            Q.va = J[j]->vals;
            Q.vb = vb[j];
            Q.plan = plan + j * RS_PLAN + dg;
            Q.dhist = hist[j] + dg * 256;
            Q.status = status[j];
            Q.n = J[j]->n;
        }
        const int w = dg / 8;
        c.sort_epoch = (c.sort_epoch + 1) & 0x3fffffffu;
        if (c.sort_epoch == 0) {
            // the 30-bit epoch wrapped: a status word left from 2^30 passes ago could
            // match again, so every job's status words are cleared before reuse
            for (auto &job : c.sort_scr)
                if (job[6].p) W1G_CUDA(cudaMemsetAsync(job[6].p, 0, job[6].cap, c.stream));
            c.sort_epoch = 1;
        }
        A.shift = 8 * (dg % 8);
        A.ticket = tickets + (launch++ & 63);
        A.epoch = c.sort_epoch;
        // large inputs: 8192-key tiles when the staged words fit in shared memory
        W1G_TRY(dispatch_pass(words, words - w, c, A, large && words - w <= 2));
    }
    FixupArgs X;
    for (int j = 0; j < nj; j++) {
        X.final_par[j] = plan + j * RS_PLAN + 32;
        X.vb[j] = vb[j];
        X.va[j] = J[j]->vals;
        X.kb[j] = b[j].k[words - 1];
        X.ka[j] = J[j]->keys[words - 1];
        X.n[j] = J[j]->n;
    }
    k_rs_fixup<<<dim3(grid_for(nmax, 256, 8u * c.sm_count), nj), 256, 0, c.stream>>>(X);
    W1G_CHECK_LAUNCH();
    return W1G_OK;
}

int radix_sort(Ctx &c, uint64_t **keys, int words, uint32_t *vals, int64_t n, int top_bits) {
    SortJob job{{keys[0], words > 1 ? keys[1] : nullptr, words > 2 ? keys[2] : nullptr}, vals, n};
    return radix_sort_multi(c, &job, 1, words, top_bits);
}

// ---------------------------------------------------------------- (primary, secondary) sort
//
// Stable sort by a 128-bit key (primary word, then secondary word) that only
// pays for the secondary word where primaries tie: one 64-bit radix sort by
// the primary, then the elements of tie runs (usually none for real-valued
// coordinates; everything for H0-style diagrams whose births are all 0) are
// sorted by (primary, secondary) and written back into their run slots.

namespace {

struct TieFlag {
    const uint64_t *k;
    int64_t n;
    __device__ int64_t operator()(int64_t i) const {
        const uint64_t v = k[i];
        return ((i > 0 && k[i - 1] == v) || (i + 1 < n && k[i + 1] == v)) ? 1 : 0;
    }
};

// the full (primary, secondary) keys of the tie elements (the sorted keys f.k
// are compressed, so the primary is read through the payload = input position)
__global__ void k_tie_gather(TieFlag f, const int64_t *excl, const uint32_t *vals, const uint64_t *prim,
                             const uint64_t *sec, uint32_t *tpos, uint64_t *kl, uint64_t *kh, uint32_t *pl) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < f.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!f(i)) continue;
        const int64_t r = excl[i];
        const uint32_t v = vals[i];
        tpos[r] = (uint32_t)i;
        kh[r] = prim[v];
        kl[r] = sec[v];
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

// ---- compressed primary keys: the radix passes run on a 32-bit key that
// preserves the primary's order weakly (k_key_compress) and elements whose
// compressed keys tie (true primary ties and compression collisions alike)
// are ordered afterwards by the full (primary, secondary, input position).
__global__ void k_mm_init(unsigned long long *mm, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) mm[i] = (i % 4) == 0 ? ~0ull : 0ull;
}

__global__ void k_key_range(const uint64_t *k, int64_t n, unsigned long long *mm) {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long v = k[i];
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}

// the primaries are order-preserving keys of doubles (dkey); the compression
// is linear in VALUE space, (v - vmin) * (2^32 - 1) / (vmax - vmin) rounded
// down -- monotone under IEEE rounding, and unlike a shifted key range it keeps
// close values apart however wide the range of exponents is
__device__ __forceinline__ double dkey_value(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}
__global__ void k_key_compress(const uint64_t *k, int64_t n, const unsigned long long *mm, double kmax,
                               uint64_t *out) {
    const double lo = dkey_value(mm[0]), hi = dkey_value(mm[1]);
    const double range = hi - lo;
    const bool flat = !(range > 0.0) || !isfinite(range);
    const double scale = flat ? 0.0 : kmax / range;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double t = flat ? 0.0 : floor((dkey_value(k[i]) - lo) * scale);
        t = t < 0.0 ? 0.0 : (t > kmax ? kmax : t);
        out[i] = (uint64_t)t;
    }
}

// tie runs of at most TIE_SMALL elements: one thread orders its run by
// (primary, secondary, input position) with an insertion sort; the longest run
// is reported so the host can take the radix path for long runs instead
constexpr int TIE_SMALL = 32;
#ifndef W1G_LEX_BITS
#define W1G_LEX_BITS 32
#endif
constexpr int LEX_BITS = W1G_LEX_BITS;  // compressed key width (8-bit radix digits)
__global__ void k_tie_runs(const uint64_t *pk, int64_t n, unsigned long long *maxrun, int64_t *count) {
    unsigned long long mr = 0;
    int64_t cnt = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = pk[i];
        if (i > 0 && pk[i - 1] == v) continue;  // not a run start
        int64_t j = i + 1;
        while (j < n && pk[j] == v && j - i <= TIE_SMALL) j++;
        const int64_t len = j - i;
        if (len > 1) {
            cnt += len;
            mr = (unsigned long long)len > mr ? (unsigned long long)len : mr;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, mr, o);
        mr = a > mr ? a : mr;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (mr) atomicMax(maxrun, mr);
        if (cnt) atomicAdd((unsigned long long *)count, (unsigned long long)cnt);
    }
}

// (mr / hmr, optional: the speculative path's longest tie run, counted by k_tie_runs before
// this launch, copied to its page-locked host slot -- no small-read launch of its own)
__global__ void k_tie_small(const uint64_t *pk, int64_t n, const uint64_t *primary, const uint64_t *secondary,
                            uint32_t *vals, const unsigned long long *mr, volatile unsigned long long *hmr) {
    if (hmr && blockIdx.x == 0 && threadIdx.x == 0) *hmr = *mr;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = pk[i];
        if ((i > 0 && pk[i - 1] == v) || i + 1 >= n || pk[i + 1] != v) continue;  // run starts only
        int64_t j = i + 1;
        while (j < n && pk[j] == v && j - i <= TIE_SMALL) j++;
        if (j - i > TIE_SMALL) continue;  // long run: the two-word path's (speculative callers redo)
        // insertion sort of vals[i..j) by (primary[val], secondary[val], val)
        for (int64_t a = i + 1; a < j; a++) {
            const uint32_t x = vals[a];
            const uint64_t xp = primary[x], xs = secondary[x];
            int64_t b = a - 1;
            while (b >= i) {
                const uint32_t y = vals[b];
                const uint64_t yp = primary[y], ys = secondary[y];
                const bool gt = yp > xp || (yp == xp && (ys > xs || (ys == xs && y > x)));
                if (!gt) break;
                vals[b + 1] = y;
                b--;
            }
            vals[b + 1] = x;
        }
    }
}

}  // namespace

int sort_lex2_multi(Ctx &c, const Lex2Job *jobs, int njobs, bool speculative) {
    if (njobs < 1 || njobs > RS_JOBS) {
        set_error("sort_lex2: unsupported job count %d", njobs);
        return W1G_EINVAL;
    }
    uint64_t *pk[RS_JOBS];
    int64_t *excl[RS_JOBS];
    unsigned long long *mm;  // per job: key min, key max, longest tie run, tie count
    SortJob sj[RS_JOBS];
    W1G_TRY(ensure(c.sort_scr[1][3], (size_t)4 * RS_JOBS, &mm));
    // per job {key min = ~0, max = 0, longest run = 0, ties = 0}, set by a kernel: a
    // host-to-device copy of a (pageable) stack array would go through the copy engines
    k_mm_init<<<1, 32, 0, c.stream>>>(mm, 4 * RS_JOBS);
    W1G_CHECK_LAUNCH();
    for (int j = 0; j < njobs; j++) {
        const int64_t n = jobs[j].n;
        W1G_TRY(ensure(c.lex_scr[j][0], (size_t)n + 1, &pk[j]));
        W1G_TRY(ensure(c.lex_scr[j][1], (size_t)n + 1, &excl[j]));
        if (n > 0) {
            const unsigned g = grid_for(n, 256, 8u * c.sm_count);
            k_key_range<<<grid_for(n, 256, 2u * c.sm_count), 256, 0, c.stream>>>(jobs[j].primary, n, mm + 4 * j);
            W1G_CHECK_LAUNCH();
            k_key_compress<<<g, 256, 0, c.stream>>>(jobs[j].primary, n, mm + 4 * j, (double)((1ull << LEX_BITS) - 1),
                                                   pk[j]);
            W1G_CHECK_LAUNCH();
        }
        sj[j] = SortJob{{pk[j], nullptr, nullptr}, jobs[j].vals, n};
    }
    W1G_TRY(radix_sort_multi(c, sj, njobs, 1, LEX_BITS));
    for (int j = 0; j < njobs; j++) {
        if (jobs[j].n > 1) {
            k_tie_runs<<<grid_for(jobs[j].n, 256, 8u * c.sm_count), 256, 0, c.stream>>>(
                pk[j], jobs[j].n, mm + 4 * j + 2, reinterpret_cast<int64_t *>(mm + 4 * j + 3));
            W1G_CHECK_LAUNCH();
        }
    }
    if (speculative) {
        for (int j = 0; j < njobs; j++) {
            if (jobs[j].n <= 1) continue;
            k_tie_small<<<grid_for(jobs[j].n, 256, 8u * c.sm_count), 256, 0, c.stream>>>(
                pk[j], jobs[j].n, jobs[j].primary, jobs[j].secondary, jobs[j].vals, mm + 4 * j + 2,
                reinterpret_cast<volatile unsigned long long *>(c.h_pinned + H_LEX_MAXRUN + j));
            W1G_CHECK_LAUNCH();
        }
        return W1G_OK;
    }
    unsigned long long *hm = reinterpret_cast<unsigned long long *>(c.h_pinned + F_SCAL);
    W1G_TRY(to_host_small(c, hm, mm, sizeof(unsigned long long) * 4 * njobs));
    W1G_TRY(stream_sync(c));
    // elements of tie runs: short runs in place by one thread each; jobs with a
    // long run (e.g. an H0 diagram whose births are all 0) by a two-word radix
    // sort of all their tie elements
    bool is_long[RS_JOBS] = {false, false};
    int64_t *dt = ptr<int64_t>(c.flags) + F_MISC2;  // long-path tie counts (F_MISC2, F_MISC3)
    bool any_long = false;
    for (int j = 0; j < njobs; j++) {
        if (hm[4 * j + 3] == 0) continue;
        if (hm[4 * j + 2] <= (unsigned long long)TIE_SMALL) {
            k_tie_small<<<grid_for(jobs[j].n, 256, 8u * c.sm_count), 256, 0, c.stream>>>(
                pk[j], jobs[j].n, jobs[j].primary, jobs[j].secondary, jobs[j].vals, nullptr, nullptr);
            W1G_CHECK_LAUNCH();
        } else {
            is_long[j] = any_long = true;
            W1G_TRY(scan_i64(c, TieFlag{pk[j], jobs[j].n}, jobs[j].n, excl[j], dt + j));
        }
    }
    if (!any_long) return W1G_OK;
    W1G_TRY(to_host_small(c, &c.h_pinned[F_MISC2], dt, sizeof(int64_t) * njobs));
    W1G_TRY(stream_sync(c));
    SortJob tj[RS_JOBS];
    uint32_t *tpos[RS_JOBS], *pl[RS_JOBS];
    int nt = 0, which[RS_JOBS];
    for (int j = 0; j < njobs; j++) {
        if (!is_long[j]) continue;
        const int64_t T = c.h_pinned[F_MISC2 + j];
        uint64_t *kl, *kh;
        W1G_TRY(ensure(c.lex_scr[j][2], (size_t)T, &tpos[j]));
        W1G_TRY(ensure(c.lex_scr[j][3], (size_t)T, &kl));
        W1G_TRY(ensure(c.lex_scr[j][4], (size_t)T, &kh));
        W1G_TRY(ensure(c.lex_scr[j][5], (size_t)T * 2, &pl[j]));
        k_tie_gather<<<grid_for(jobs[j].n, 256, 8u * c.sm_count), 256, 0, c.stream>>>(
            TieFlag{pk[j], jobs[j].n}, excl[j], jobs[j].vals, jobs[j].primary, jobs[j].secondary, tpos[j], kl, kh,
            pl[j]);
        W1G_CHECK_LAUNCH();
        tj[nt] = SortJob{{kl, kh, nullptr}, pl[j], T};
        which[nt++] = j;
    }
    // (primary, secondary) ties keep their input order: the radix sort is stable
    // and the tie elements are gathered in sorted (= input-stable) order
    W1G_TRY(radix_sort_multi(c, tj, nt, 2, 64));
    for (int q = 0; q < nt; q++) {
        const int j = which[q];
        const int64_t T = tj[q].n;
        uint32_t *tmp = pl[j] + T;
        const unsigned gt = grid_for(T, 256, 8u * c.sm_count);
        k_tie_fetch<<<gt, 256, 0, c.stream>>>(tpos[j], pl[j], jobs[j].vals, T, tmp);
        W1G_CHECK_LAUNCH();
        k_tie_put<<<gt, 256, 0, c.stream>>>(tpos[j], tmp, T, jobs[j].vals);
        W1G_CHECK_LAUNCH();
    }
    return W1G_OK;
}

int sort_lex2(Ctx &c, const uint64_t *primary, const uint64_t *secondary, uint32_t *vals, int64_t n,
              bool speculative) {
    if (n <= 1) {
        c.h_pinned[H_LEX_MAXRUN] = 0;
        return W1G_OK;
    }
    Lex2Job job{primary, secondary, vals, n};
    return sort_lex2_multi(c, &job, 1, speculative);
}

bool lex2_speculation_failed(Ctx &c, int njobs) {
    for (int j = 0; j < njobs; j++)
        if ((unsigned long long)c.h_pinned[H_LEX_MAXRUN + j] > (unsigned long long)TIE_SMALL) return true;
    return false;
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
    W1G_TRY(stream_sync(*c));
    return W1G_OK;
}
