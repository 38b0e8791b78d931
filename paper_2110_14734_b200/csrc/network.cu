// network.cu -- arc emission (spanner.py:310-337) and CSR assembly
// (network.py:44-93) on device.
//
// emit: spanner biarcs (rep_u -> rep_v and back) with glibc 2.39's hypot
//       (np.hypot, spanner.py:324) restated operation for operation, then
//       the diagonal arcs and the free bbar -> abar arc, in the reference's
//       arc order.
// assemble/build_network: validation in the reference's order, 64-bit
//       (tail, head) keys radix-sorted (stable, as np.lexsort), duplicate
//       (tail, head) groups reduced to their min cost, row offsets by a
//       histogram + scan.
#include "common.cuh"
#include "hypot.cuh"

namespace w1g {

static const double SQRT2 = 1.4142135623730951;

namespace {

__global__ void k_emit_spanner(const int64_t *idx, int64_t P, const double2 *pts, int64_t *tails,
                               int64_t *heads, double *costs) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx[2 * p], j = idx[2 * p + 1];
        const double2 a = pts[i], b = pts[j];
        const double c = glibc_hypot(dsub(a.x, b.x), dsub(a.y, b.y));
        tails[p] = i;
        heads[p] = j;
        costs[p] = c;
        tails[P + p] = j;
        heads[P + p] = i;
        costs[P + p] = c;
    }
}

struct PosFlag {
    const int64_t *m;
    __device__ int64_t operator()(int64_t i) const { return m[i] > 0 ? 1 : 0; }
};

__global__ void k_emit_diag(const double2 *pts, const int64_t *am, const int64_t *bm, int64_t K,
                            const int64_t *exa, const int64_t *exb, int64_t na, int64_t base,
                            int64_t *tails, int64_t *heads, double *costs) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double2 p = pts[i];
        const double d = ddiv(fabs(dsub(p.y, p.x)), SQRT2);  // diagram.py:47
        if (am[i] > 0) {
            const int64_t e = base + exa[i];
            tails[e] = i;
            heads[e] = K;  // abar
            costs[e] = d;
        }
        if (bm[i] > 0) {
            const int64_t e = base + na + exb[i];
            tails[e] = K + 1;  // bbar
            heads[e] = i;
            costs[e] = d;
        }
    }
}

__global__ void k_emit_free(int64_t K, int64_t e, int64_t *tails, int64_t *heads, double *costs) {
    tails[e] = K + 1;
    heads[e] = K;
    costs[e] = 0.0;
}

__global__ void k_supplies(const int64_t *am, const int64_t *bm, int64_t K, int64_t abar, int64_t bbar,
                           int64_t *sup) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K + 2;
         i += (int64_t)gridDim.x * blockDim.x)
        sup[i] = i < K ? am[i] - bm[i] : (i == K ? abar : bbar);
}

// validation, network.py:52-68
__global__ void k_validate(const int64_t *sup, int64_t n, const int64_t *t, const int64_t *h,
                           const double *c, int64_t m, int64_t *f) {
    int64_t s = 0;
    unsigned bits = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) s += sup[i];
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const int64_t a = t[e], b = h[e];
        const double cc = c[e];
        if (a < 0 || a >= n || b < 0 || b >= n) bits |= 1u;
        if (a == b) bits |= 2u;
        if (!isfinite(cc)) bits |= 4u;
        if (cc < 0) bits |= 8u;
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        bits |= __shfl_xor_sync(0xffffffffu, bits, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (s) atomicAdd((unsigned long long *)&f[F_MISC0], (unsigned long long)s);
        if (bits) atomicOr((unsigned long long *)&f[F_NET_ERR], (unsigned long long)bits);
    }
}

__global__ void k_arc_keys(const int64_t *t, const int64_t *h, int64_t m, int hb, uint64_t *keys,
                           uint32_t *vals) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        keys[e] = ((uint64_t)t[e] << hb) | (uint64_t)h[e];
        vals[e] = (uint32_t)e;
    }
}

struct GroupFlag {
    const uint64_t *k;
    __device__ int64_t operator()(int64_t i) const { return (i == 0 || k[i] != k[i - 1]) ? 1 : 0; }
};

__global__ void k_net_emit(GroupFlag f, int64_t m, const int64_t *excl, const uint32_t *perm,
                           const int64_t *t, const int64_t *h, const double *c, int64_t *ot,
                           int64_t *oh, double *oc, int64_t *rowcnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!f(i)) continue;
        const int64_t g = excl[i];
        const uint32_t e = perm[i];
        double cm = c[e];
        // np.minimum.at over the duplicate group (network.py:75-76), a fold in
        // arc order: minimum(acc, c) keeps acc only when strictly smaller, so
        // among equal minima (+0.0 / -0.0) the later arc wins
        for (int64_t j = i + 1; j < m && !f(j); j++) {
            const double cj = c[perm[j]];
            cm = cm < cj ? cm : cj;
        }
        ot[g] = t[e];
        oh[g] = h[e];
        oc[g] = cm;
        atomicAdd((unsigned long long *)&rowcnt[t[e]], 1ull);
    }
}

struct RowCount {
    const int64_t *cnt;
    int64_t n;
    __device__ int64_t operator()(int64_t i) const { return i < n ? cnt[i] : 0; }
};

inline unsigned gs(const Ctx &c, int64_t n) { return grid_for(n, 256, 8u * c.sm_count); }

// ---------------------------------------------------------------- row-bucketed CSR
//
// np.lexsort((heads, tails)) + duplicate reduction (network.py:70-82) without a
// full-width sort: arcs are bucketed by tail (count, scan, scatter -- rows are
// what the CSR needs anyway), then every row is sorted by (head, arc index)
// on chip -- a warp per row of <= 32 arcs, a CTA per longer row -- and its
// duplicate (tail, head) groups reduced as np.minimum.at does: a fold in arc
// order from +inf, so among equal minima (+0.0 / -0.0) the LAST arc wins.
// Row offsets are the scan of the deduplicated row lengths.

// validation (network.py:55-68) + arcs per tail row; out-of-range arcs are
// flagged and never counted.  Arcs of one tail come in runs (all diagonal arcs
// leave b-bar), so counts are warp-aggregated: one atomic per tail per warp.
__global__ void k_csr_count(const int64_t *sup, int64_t n, const int64_t *t, const int64_t *h, const double *c,
                            int64_t m, unsigned *cnt, int64_t *f) {
    int64_t s = 0;
    unsigned bits = 0;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) s += sup[i];
    const int64_t mr = (m + 31) & ~31ll;  // whole warps iterate together
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < mr; e += stride) {
        int64_t a = -1;
        if (e < m) {
            const int64_t b = h[e];
            const double cc = c[e];
            a = t[e];
            const bool ok = a >= 0 && a < n && b >= 0 && b < n;
            if (!ok) bits |= 1u;
            if (a == b) bits |= 2u;
            if (!isfinite(cc)) bits |= 4u;
            if (cc < 0) bits |= 8u;
            if (!ok) a = -1;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, a);
        if (a >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(&cnt[a], (unsigned)__popc(peers));
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        bits |= __shfl_xor_sync(0xffffffffu, bits, o);
    }
    // one atomic per CTA for the supply sum (it is non-zero almost everywhere)
    __shared__ long long s_sum[8];
    __shared__ unsigned s_bits[8];
    const int wid = threadIdx.x >> 5;
    if (lane == 0) {
        s_sum[wid] = s;
        s_bits[wid] = bits;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long ts = 0;
        unsigned tb = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            ts += s_sum[w];
            tb |= s_bits[w];
        }
        if (ts) atomicAdd((unsigned long long *)&f[F_MISC0], (unsigned long long)ts);
        if (tb) atomicOr((unsigned long long *)&f[F_NET_ERR], (unsigned long long)tb);
    }
}

struct RowLen {
    const unsigned *cnt;
    int64_t n;
    __device__ int64_t operator()(int64_t i) const { return i < n ? (int64_t)cnt[i] : 0; }
};

// arc -> slot in its tail row, warp-aggregated (order inside a row is fixed
// later by the row sort)
__global__ void k_csr_scatter(const int64_t *t, const int64_t *h, int64_t m, int64_t n, const int64_t *start,
                              unsigned *cursor, int32_t *slot_h, uint32_t *slot_e) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const int64_t mr = (m + 31) & ~31ll;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < mr;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = -1, b = 0;
        if (e < m) {
            a = t[e];
            b = h[e];
            if (a < 0 || a >= n || b < 0 || b >= n) a = -1;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, a);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0;
        if (a >= 0 && lane == leader) base = atomicAdd(&cursor[a], (unsigned)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (a >= 0) {
            const int64_t p = start[a] + base + __popc(peers & lt);
            slot_h[p] = (int32_t)b;
            slot_e[p] = (uint32_t)e;
        }
    }
}

// np.minimum.at order: (cost, arc) pairs, smaller cost first, then the later arc
__device__ __forceinline__ bool min_at_better(double c2, uint32_t e2, double c1, uint32_t e1) {
    return c2 < c1 || (c2 == c1 && e2 > e1);
}

// row classes by length: <= 32 a warp in registers, <= CSR_MED_MAX a warp in
// shared memory, <= CSR_LONG_MAX a CTA in shared memory, longer ("huge": the
// b-bar row of every front end) a CTA with head-indexed minima
constexpr int CSR_MED_MAX = 256;
constexpr int CSR_LONG_MAX = 4096;
constexpr int CSR_HUGE_CAP = 2;  // more huge rows than this: radix-sort fallback
enum { CL_MED = 0, CL_LONG = 1, CL_HUGE = 2, CL_W32 = 3 };

// rows of <= W arcs on W-lane groups (W = 16: two rows per warp; W = 32: one):
// bitonic sort by (head, arc) in registers, then the duplicate groups reduced
// with a segmented shuffle scan.  Every lane of the warp runs the same network
// (rows that are empty or handled elsewhere take part with len = 0).
template <int W>
__device__ __forceinline__ void row_sort_reg(int64_t r, int64_t s0, int len, int32_t *slot_h,
                                             const uint32_t *slot_e, const double *c, double *slot_c,
                                             int64_t *dcnt) {
    const int lane = threadIdx.x & 31, gl = lane & (W - 1);
    const unsigned gmask = W == 32 ? 0xffffffffu : (0xffffu << (lane & 16));
    const unsigned lt = lanemask_lt() & gmask;
    uint64_t key = ~0ull;
    if (gl < len) key = ((uint64_t)(uint32_t)slot_h[s0 + gl] << 32) | slot_e[s0 + gl];
#pragma unroll
    for (int k = 2; k <= W; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j; j >>= 1) {
            const uint64_t o = __shfl_xor_sync(0xffffffffu, key, j);
            const bool up = ((gl & k) == 0) == ((gl & j) == 0);
            key = up ? (key < o ? key : o) : (key > o ? key : o);
        }
    const bool valid = gl < len;
    const int32_t head = (int32_t)(key >> 32);
    const uint32_t e = (uint32_t)key;
    double cost = valid ? c[e] : INFINITY;
    const int32_t prev = __shfl_up_sync(0xffffffffu, head, 1);
    const bool first = valid && (gl == 0 || prev != head);
    const unsigned firsts = __ballot_sync(0xffffffffu, first) & gmask;
    // suffix reduction inside each (head) group: lanes of a group are contiguous
    const int gid = __popc(firsts & (lt | (1u << lane)));
    uint32_t eb = e;
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
        const double c2 = __shfl_down_sync(0xffffffffu, cost, o);
        const uint32_t e2 = __shfl_down_sync(0xffffffffu, eb, o);
        const int g2 = __shfl_down_sync(0xffffffffu, gid, o);
        if (gl + o < len && g2 == gid && min_at_better(c2, e2, cost, eb)) {
            cost = c2;
            eb = e2;
        }
    }
    if (first) {
        const int64_t q = s0 + __popc(firsts & lt);
        slot_h[q] = head;
        slot_c[q] = cost;
    }
    if (gl == 0 && r >= 0) dcnt[r] = __popc(firsts);
}

// every row: <= 16 arcs sorted here on half warps, longer rows queued by class
__global__ void k_csr_short_rows(const int64_t *start, int64_t n, int32_t *slot_h, const uint32_t *slot_e,
                                 const double *c, double *slot_c, int64_t *dcnt, int32_t *lists,
                                 int32_t *n_list, int64_t *f) {
    const int lane = threadIdx.x & 31, gl = lane & 15;
    const int64_t groups = ((int64_t)gridDim.x * blockDim.x) >> 4;
    const int64_t nr = (n + 1) & ~1ll;  // both halves of a warp iterate together
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4; r < nr; r += groups) {
        int len = 0;
        int64_t s0 = 0;
        if (r < n) {
            s0 = start[r];
            const int64_t l = start[r + 1] - s0;
            if (l > 16) {
                if (gl == 0) {
                    const int cl = l <= 32 ? CL_W32 : l <= CSR_MED_MAX ? CL_MED : l <= CSR_LONG_MAX ? CL_LONG : CL_HUGE;
                    const int k = atomicAdd(&n_list[cl], 1);
                    if (cl != CL_HUGE || k < CSR_HUGE_CAP) {
                        lists[(int64_t)cl * n + k] = (int32_t)r;
                    } else {  // no table left: emit nothing, the host redoes it with the full sort
                        dcnt[r] = 0;
                        atomicOr((unsigned long long *)&f[F_OVERFLOW], 1ull);
                    }
                }
            } else {
                len = (int)l;
            }
        }
        const int64_t rr = (r < n && len > 0) ? r : -1;
        if (r < n && len == 0 && start[r + 1] == s0 && gl == 0) dcnt[r] = 0;  // empty row
        row_sort_reg<16>(rr, s0, len, slot_h, slot_e, c, slot_c, dcnt);
    }
}

// rows of 17..32 arcs: a warp each
__global__ void k_csr_w32_rows(const int64_t *start, const int32_t *rows, const int32_t *n_rows, int32_t *slot_h,
                               const uint32_t *slot_e, const double *c, double *slot_c, int64_t *dcnt) {
    const int nr = *n_rows;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nr; i += (gridDim.x * blockDim.x) >> 5) {
        const int64_t r = rows[i], s0 = start[r];
        row_sort_reg<32>(r, s0, (int)(start[r + 1] - s0), slot_h, slot_e, c, slot_c, dcnt);
    }
}

// sorted keys (head << 32 | arc) of one row in shared memory -> deduplicated
// (head, min cost) back into the row's slots; `per` items per participant
template <class Sync>
__device__ void dedup_sorted(const uint64_t *sk, int len, int part, int nparts, int *s_cnt, int64_t s0,
                             const double *c, int32_t *slot_h, double *slot_c, int64_t *dcnt_r, Sync sync) {
    const int per = (len + nparts - 1) / nparts;
    const int b0 = part * per, b1 = min(len, b0 + per);
    int nf = 0;
    for (int i = b0; i < b1; i++) nf += (i == 0 || (sk[i] >> 32) != (sk[i - 1] >> 32));
    s_cnt[part] = nf;
    sync();
    int q = 0, tot = 0;
    for (int p = 0; p < nparts; p++) {
        if (p < part) q += s_cnt[p];
        tot += s_cnt[p];
    }
    for (int i = b0; i < b1; i++) {
        const uint64_t ki = sk[i];
        if (i > 0 && (ki >> 32) == (sk[i - 1] >> 32)) continue;
        double cost = c[(uint32_t)ki];
        uint32_t eb = (uint32_t)ki;
        for (int j = i + 1; j < len && (sk[j] >> 32) == (ki >> 32); j++) {
            const double c2 = c[(uint32_t)sk[j]];
            if (min_at_better(c2, (uint32_t)sk[j], cost, eb)) {
                cost = c2;
                eb = (uint32_t)sk[j];
            }
        }
        slot_h[s0 + q] = (int32_t)(ki >> 32);
        slot_c[s0 + q] = cost;
        q++;
    }
    if (part == 0) *dcnt_r = tot;
}

// one warp sorts 32*E keys (head << 32 | arc) held E per lane in registers
// (element i = lane * E + q): bitonic stages with partner distance >= E are
// shuffles, shorter ones swaps inside the lane; the sorted row goes to sk
template <int E, class Key = uint64_t>
__device__ __forceinline__ void warp_bitonic(Key (&v)[E], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j; j >>= 1) {
            if (j >= E) {
#pragma unroll
                for (int q = 0; q < E; q++) {
                    const Key o = __shfl_xor_sync(0xffffffffu, v[q], j / E);
                    const int i = lane * E + q;
                    const bool keep_min = ((i & k) == 0) == ((i & j) == 0);
                    v[q] = keep_min ? (v[q] < o ? v[q] : o) : (v[q] > o ? v[q] : o);
                }
            } else {
#pragma unroll
                for (int q = 0; q < E; q++) {
                    if (q & j) continue;
                    const int p = q | j;
                    const bool up = ((lane * E + q) & k) == 0;
                    const Key a = v[q], b = v[p];
                    if ((a > b) == up) {
                        v[q] = b;
                        v[p] = a;
                    }
                }
            }
        }
}
template <int E, class Load>
__device__ __forceinline__ void warp_sort_keys(uint64_t *sk, int len, int lane, Load load) {
    uint64_t v[E];
#pragma unroll
    for (int q = 0; q < E; q++) {
        const int i = lane * E + q;
        v[q] = i < len ? load(i) : ~0ull;
    }
    warp_bitonic<E>(v, lane);
#pragma unroll
    for (int q = 0; q < E; q++) sk[lane * E + q] = v[q];
}
template <int E>
__device__ __forceinline__ void warp_sort_rows(uint64_t *sk, int len, int64_t s0, const int32_t *slot_h,
                                               const uint32_t *slot_e, int lane) {
    warp_sort_keys<E>(sk, len, lane,
                      [&](int i) { return ((uint64_t)(uint32_t)slot_h[s0 + i] << 32) | slot_e[s0 + i]; });
}

// rows of 33..CSR_MED_MAX arcs: a warp each, sorted in registers, deduplicated
// from its shared-memory slice
constexpr int CSR_MB = 256;
__global__ void __launch_bounds__(CSR_MB) k_csr_med_rows(const int64_t *start, const int32_t *rows,
                                                         const int32_t *n_rows, int32_t *slot_h,
                                                         const uint32_t *slot_e, const double *c, double *slot_c,
                                                         int64_t *dcnt) {
    __shared__ uint64_t sk_all[CSR_MB / 32][CSR_MED_MAX];
    __shared__ int cnt_all[CSR_MB / 32][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t *sk = sk_all[wid];
    const int nr = *n_rows;
    for (int ri = blockIdx.x * (CSR_MB / 32) + wid; ri < nr; ri += gridDim.x * (CSR_MB / 32)) {
        const int64_t r = rows[ri];
        const int64_t s0 = start[r];
        const int len = (int)(start[r + 1] - s0);
        __syncwarp();
        if (len <= 64) warp_sort_rows<2>(sk, len, s0, slot_h, slot_e, lane);
        else if (len <= 128) warp_sort_rows<4>(sk, len, s0, slot_h, slot_e, lane);
        else warp_sort_rows<8>(sk, len, s0, slot_h, slot_e, lane);
        __syncwarp();
        dedup_sorted(sk, len, lane, 32, cnt_all[wid], s0, c, slot_h, slot_c, dcnt + r, []() { __syncwarp(); });
        __syncwarp();
    }
}

// rows of CSR_MED_MAX+1..CSR_LONG_MAX arcs: one CTA each, bitonic sort in shared memory
constexpr int CSR_LB = 512;
__global__ void __launch_bounds__(CSR_LB) k_csr_long_rows(const int64_t *start, const int32_t *rows,
                                                          const int32_t *n_rows, int32_t *slot_h,
                                                          const uint32_t *slot_e, const double *c,
                                                          double *slot_c, int64_t *dcnt) {
    __shared__ uint64_t sk[CSR_LONG_MAX];
    __shared__ int s_cnt[CSR_LB];
    const int tid = threadIdx.x;
    const int nr = *n_rows;
    for (int ri = blockIdx.x; ri < nr; ri += gridDim.x) {
        const int64_t r = rows[ri];
        const int64_t s0 = start[r];
        const int len = (int)(start[r + 1] - s0);
        int np2 = 64;
        while (np2 < len) np2 <<= 1;
        __syncthreads();
        for (int i = tid; i < np2; i += CSR_LB)
            sk[i] = i < len ? (((uint64_t)(uint32_t)slot_h[s0 + i] << 32) | slot_e[s0 + i]) : ~0ull;
        __syncthreads();
        for (int k = 2; k <= np2; k <<= 1)
            for (int j = k >> 1; j; j >>= 1) {
                for (int i = tid; i < np2; i += CSR_LB) {
                    const int p = i ^ j;
                    if (p > i) {
                        const uint64_t a = sk[i], b = sk[p];
                        if ((a > b) == ((i & k) == 0)) {
                            sk[i] = b;
                            sk[p] = a;
                        }
                    }
                }
                __syncthreads();
            }
        dedup_sorted(sk, len, tid, CSR_LB, s_cnt, s0, c, slot_h, slot_c, dcnt + r, []() { __syncthreads(); });
        __syncthreads();
    }
}

// huge rows (> CSR_LONG_MAX arcs: the b-bar row of every front end): per-head
// minima in a dense head-indexed table (cost with -0 folded onto +0, then the
// latest arc among the minimal ones, as np.minimum.at's fold), read back in
// head order by a device scan.  Grid-wide kernels over the (<= CSR_HUGE_CAP)
// listed rows; the row count is read on the device.
__device__ __forceinline__ unsigned long long cost_key(double x) {
    return x == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(x);  // costs are >= 0
}
__global__ void k_huge_init(const int32_t *n_rows, int64_t n, unsigned long long *tab_c, unsigned *tab_e) {
    const int64_t tot = (int64_t)min(*n_rows, CSR_HUGE_CAP) * n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        tab_c[i] = ~0ull;
        tab_e[i] = 0u;
    }
}
template <int PHASE>
__global__ void k_huge_fold(const int64_t *start, const int32_t *rows, const int32_t *n_rows, int64_t n,
                            const int32_t *slot_h, const uint32_t *slot_e, const double *c,
                            unsigned long long *tab_c, unsigned *tab_e) {
    const int nr = min(*n_rows, CSR_HUGE_CAP);
    for (int ri = 0; ri < nr; ri++) {
        const int64_t r = rows[ri];
        const int64_t s0 = start[r], len = start[r + 1] - s0;
        unsigned long long *tc = tab_c + (int64_t)ri * n;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len;
             i += (int64_t)gridDim.x * blockDim.x) {
            const uint32_t e = slot_e[s0 + i];
            const int32_t hd = slot_h[s0 + i];
            if (PHASE == 0) atomicMin(&tc[hd], cost_key(c[e]));
            else if (cost_key(c[e]) == tc[hd]) atomicMax(&tab_e[(int64_t)ri * n + hd], e);
        }
    }
}
struct HugeHit {
    const unsigned long long *tab_c;
    const int32_t *n_rows;
    int64_t n;
    __device__ int64_t operator()(int64_t i) const {
        return (i / n < min(*n_rows, CSR_HUGE_CAP) && tab_c[i] != ~0ull) ? 1 : 0;
    }
};
__global__ void k_huge_write(const int64_t *start, const int32_t *rows, const int32_t *n_rows, int64_t n,
                             const unsigned long long *tab_c, const unsigned *tab_e, const int64_t *pos,
                             const double *c, int32_t *slot_h, double *slot_c, int64_t *dcnt) {
    const int nr = min(*n_rows, CSR_HUGE_CAP);
    for (int ri = 0; ri < nr; ri++) {
        const int64_t r = rows[ri], s0 = start[r];
        const int64_t base = pos[(int64_t)ri * n];
        for (int64_t hd = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; hd < n;
             hd += (int64_t)gridDim.x * blockDim.x) {
            const int64_t i = (int64_t)ri * n + hd;
            if (tab_c[i] == ~0ull) continue;
            const int64_t q = s0 + pos[i] - base;
            slot_h[q] = (int32_t)hd;
            slot_c[q] = c[tab_e[i]];
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) dcnt[r] = pos[(int64_t)ri * n + n] - base;
    }
}

struct DCount {
    const int64_t *d;
    int64_t n;
    __device__ int64_t operator()(int64_t i) const { return i < n ? d[i] : 0; }
};

// deduplicated rows to their CSR positions: a warp per row of <= CSR_MED_MAX
// deduplicated arcs, a CTA per listed longer row
__global__ void k_csr_emit(const int64_t *__restrict__ start, const int64_t *__restrict__ ro, int64_t n,
                           const int32_t *__restrict__ slot_h, const double *__restrict__ slot_c,
                           int64_t *__restrict__ ot, int64_t *__restrict__ oh, double *__restrict__ oc) {
    // half a warp per row: rows average ~16 arcs at s = 1
    const int hl = threadIdx.x & 15;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4; r < n;
         r += ((int64_t)gridDim.x * blockDim.x) >> 4) {
        const int64_t s0 = start[r], d0 = ro[r], len = ro[r + 1] - d0;
        if (start[r + 1] - s0 > CSR_MED_MAX) continue;  // k_csr_emit_long
        for (int64_t k = hl; k < len; k += 16) {
            ot[d0 + k] = r;
            oh[d0 + k] = slot_h[s0 + k];
            oc[d0 + k] = slot_c[s0 + k];
        }
    }
}
__global__ void k_csr_emit_long(const int64_t *__restrict__ start, const int64_t *__restrict__ ro, int64_t n,
                                const int32_t *__restrict__ lists, const int32_t *__restrict__ n_list,
                                const int32_t *__restrict__ slot_h, const double *__restrict__ slot_c,
                                int64_t *__restrict__ ot, int64_t *__restrict__ oh, double *__restrict__ oc) {
    // few rows, possibly very long (b-bar): the whole grid copies one row at a time
    const int n_long = n_list[CL_LONG], n_huge = min(n_list[CL_HUGE], CSR_HUGE_CAP);
    for (int li = 0; li < n_long + n_huge; li++) {
        const int64_t r = li < n_long ? lists[CL_LONG * n + li] : lists[CL_HUGE * n + li - n_long];
        const int64_t s0 = start[r], d0 = ro[r], len = ro[r + 1] - d0;
        for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < len;
             k += (int64_t)gridDim.x * blockDim.x) {
            ot[d0 + k] = r;
            oh[d0 + k] = slot_h[s0 + k];
            oc[d0 + k] = slot_c[s0 + k];
        }
    }
}

// ---------------------------------------------------------------- fused spanner CSR
//
// In the fused front end the arc list has a known shape (spanner.py:310-337):
// both directions of every WSPD pair, i -> abar for each A-member, bbar -> i
// for each B-member, then bbar -> abar.  No (tail, head) repeats: a WSPD
// covers every point pair exactly once, so two pairs never share both
// representatives.  np.lexsort + np.minimum.at (network.py:70-82) therefore
// reduce to: bucket the pair arcs by tail, sort each row by head, and put
// abar (= K, above every point) last in the A-member rows; the bbar row is the
// B-members in node order, then abar.  The ArcList itself is never written.
// A repeated head (impossible for a WSPD) or a row longer than CSR_LONG_MAX
// is flagged, and the host redoes the network on the generic path.
constexpr long long SP_DUP_BIT = 1ll << 16;  // in F_NET_ERR
// longest row a warp sorts in registers.  With 32-bit keys a warp could sort 1024
// (E = 32, 128 registers), but measured at cfg5 (s = 16, delta = 0.001) the rows of
// 513..1024 took 0.76 ms that way against ~0.5 ms in the bitmap kernel
constexpr int SP_MED_MAX = 512;
constexpr int SP_CL_BIG = CL_HUGE;           // list of rows of 257..512 (no huge class here)

// the bucketed pair arcs: per CSR slot the head and the cost; rows are sorted
// by (head << 32 | position in the row), the position then fetches the cost
// (the cost of arc t -> h is np.hypot of p[t] - p[h]; np.hypot's |dx|, |dy| make it the
// same value for both arcs of a pair (spanner.py:322-325), so it is computed where the
// arc is written, from (row, head), and the scatter moves 4-byte heads only)
struct SpRows {
    const int64_t *ro;     // row offsets (final CSR positions)
    const unsigned *cnt;   // pair arcs per row
    const uint32_t *sh;    // slot heads
    const double2 *pts;    // node points (arc costs)
    int64_t *ot, *oh;
    double *oc;
    int64_t *f;
};

// pair arcs per tail; the pairs' representatives are rep[u], rep[v] (spanner.py:296)
__global__ void k_sp_count(const int2 *__restrict__ uv, const int32_t *__restrict__ rep, int64_t P, unsigned *cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t pr = (P + 31) & ~31ll;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pr; p += (int64_t)gridDim.x * blockDim.x) {
        int i = -1, j = -1;
        if (p < P) {
            const int2 q = uv[p];
            i = rep[q.x];
            j = rep[q.y];
        }
        unsigned peers = __match_any_sync(0xffffffffu, i);
        if (i >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(&cnt[i], (unsigned)__popc(peers));
        peers = __match_any_sync(0xffffffffu, j);
        if (j >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(&cnt[j], (unsigned)__popc(peers));
    }
}

// row lengths: pair arcs (+ abar for A-members) | abar: none | bbar: B-members + abar
struct SpRowLen {
    const unsigned *cnt;
    const int64_t *am;
    int64_t K, nb;
    __device__ int64_t operator()(int64_t i) const {
        if (i < K) return (int64_t)cnt[i] + (am[i] > 0 ? 1 : 0);
        return i == K + 1 ? nb + 1 : 0;
    }
};

// both arcs of every pair into their tail rows (warp-aggregated slots) with
// the pair's cost, np.hypot of the representatives (spanner.py:322-325)
__global__ void k_sp_scatter(const int2 *__restrict__ uv, const int32_t *__restrict__ rep, int64_t P,
                             const int64_t *__restrict__ ro, unsigned *cursor, uint32_t *sh) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const int64_t pr = (P + 31) & ~31ll;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pr; p += (int64_t)gridDim.x * blockDim.x) {
        int e[2] = {-1, -1};
        if (p < P) {
            const int2 q = uv[p];
            e[0] = rep[q.x];
            e[1] = rep[q.y];
        }
        int64_t slot[2];
#pragma unroll
        for (int d = 0; d < 2; d++) {
            const int t = e[d];
            const unsigned peers = __match_any_sync(0xffffffffu, t);
            const int leader = __ffs(peers) - 1;
            unsigned base = 0;
            if (t >= 0 && lane == leader) base = atomicAdd(&cursor[t], (unsigned)__popc(peers));
            base = __shfl_sync(0xffffffffu, base, leader);
            slot[d] = t >= 0 ? ro[t] + base + __popc(peers & lt) : 0;
        }
        if (p < P) {
            sh[slot[0]] = (uint32_t)e[1];
            sh[slot[1]] = (uint32_t)e[0];
        }
    }
}

// the tails column of the CSR: a function of the row offsets alone (a warp per
// row, the long bbar row by the whole grid), written before the rows are
// sorted so its D2H copy can start early
__global__ void k_sp_tails(const int64_t *__restrict__ ro, int64_t K, int64_t *ot) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r <= K; r += warps) {
        const int64_t b = ro[r], e = ro[r + 1];
        for (int64_t q = b + lane; q < e; q += 32) ot[q] = r;
    }
    const int64_t b = ro[K + 1], e = ro[K + 2];
    for (int64_t q = b + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < e; q += (int64_t)gridDim.x * blockDim.x)
        ot[q] = K + 1;
}

// sorted element i of row r: key = head << 32 | original position in the row
__device__ __forceinline__ void sp_put_head_a(const SpRows &R, const double2 a, int64_t q, uint32_t h) {
    // the tails are written by k_sp_tails; a = the row's own point
    const double2 b = R.pts[h];
    const double cc = glibc_hypot(dsub(a.x, b.x), dsub(a.y, b.y));  // spanner.py:324
    if (!isfinite(cc)) atomicOr((unsigned long long *)&R.f[F_NET_ERR], 4ull);
    R.oh[q] = (int64_t)h;
    R.oc[q] = cc;
}
__device__ __forceinline__ void sp_put_head(const SpRows &R, int64_t r, int64_t q, uint32_t h) {
    // the tails are written by k_sp_tails
    const double2 a = R.pts[r], b = R.pts[h];
    const double cc = glibc_hypot(dsub(a.x, b.x), dsub(a.y, b.y));  // spanner.py:324
    if (!isfinite(cc)) atomicOr((unsigned long long *)&R.f[F_NET_ERR], 4ull);
    R.oh[q] = (int64_t)h;
    R.oc[q] = cc;
}
// the fused path's rows are keyed by the head alone: heads are distinct within a
// row (a WSPD never repeats a (tail, head); a repeat is flagged), so no arc
// position is needed to break ties or to find the cost
__device__ __forceinline__ void sp_put(const SpRows &R, int64_t r, int64_t s0, int64_t i, uint32_t head) {
    sp_put_head(R, r, s0 + i, head);
}

// rows of <= W pair arcs on W-lane groups: bitonic sort of the keys in
// registers, written straight to the CSR
template <int W>
__device__ __forceinline__ void sp_row_reg(const SpRows &R, int64_t r, int64_t s0, int len, unsigned &dup) {
    const int lane = threadIdx.x & 31, gl = lane & (W - 1);
    uint32_t key = gl < len ? R.sh[s0 + gl] : 0xffffffffu;
#pragma unroll
    for (int k = 2; k <= W; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j; j >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, key, j);
            const bool up = ((gl & k) == 0) == ((gl & j) == 0);
            key = up ? (key < o ? key : o) : (key > o ? key : o);
        }
    const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
    if (gl < len) {
        if (gl > 0 && prev == key) dup = 1;
        sp_put(R, r, s0, gl, key);
    }
}

struct DiagArgs {
    const double2 *pts;
    const int64_t *am, *bm, *exb;
    int64_t abar, bbar;
    int64_t *sup;
};

// every row: <= 16 pair arcs sorted here on half warps (longer rows queued by
// class); lane 1 of the half warp writes the row's supply and its diagonal
// arcs (network.py:88-93, spanner.py:326-335): i -> abar last in an A-member
// row, bbar -> i at the member's place in the bbar row
__global__ void k_sp_short_rows(const __grid_constant__ SpRows R, int64_t K, int32_t *lists, int32_t *n_list,
                                unsigned long_max, unsigned med_max, unsigned big_max,
                                const __grid_constant__ DiagArgs D) {
    const int lane = threadIdx.x & 31, gl = lane & 15;
    const int64_t groups = ((int64_t)gridDim.x * blockDim.x) >> 4;
    const int64_t nr = (K + 1) & ~1ll;  // both halves of a warp iterate together
    unsigned dup = 0, bad = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        D.sup[K] = D.abar;
        D.sup[K + 1] = D.bbar;
        const int64_t q = R.ro[K + 2] - 1;  // the free bbar -> abar arc closes the bbar row
        R.oh[q] = K;
        R.oc[q] = 0.0;
    }
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4; r < nr; r += groups) {
        int len = 0;
        int64_t s0 = 0;
        if (r < K && gl == 1) {
            const double2 p = D.pts[r];
            const int64_t a = D.am[r], b = D.bm[r];
            const double d = ddiv(fabs(dsub(p.y, p.x)), SQRT2);  // diagram.py:47
            D.sup[r] = a - b;
            if (a > 0) {
                const int64_t q = R.ro[r + 1] - 1;
                R.oh[q] = K;
                R.oc[q] = d;
            }
            if (b > 0) {
                const int64_t q = R.ro[K + 1] + D.exb[r];
                R.oh[q] = r;
                R.oc[q] = d;
            }
            if ((a > 0 || b > 0) && !isfinite(d)) bad = 1;
        }
        if (r < K) {
            s0 = R.ro[r];
            const unsigned l = R.cnt[r];
            if (l > 16) {
                if (gl == 0) {
                    if (l > long_max) {
                        atomicOr((unsigned long long *)&R.f[F_OVERFLOW], 1ull);
                    } else {
                        const int cl = l <= 32 ? CL_W32 : l <= med_max ? CL_MED : l <= big_max ? SP_CL_BIG : CL_LONG;
                        lists[(int64_t)cl * K + atomicAdd(&n_list[cl], 1)] = (int32_t)r;
                    }
                }
            } else {
                len = (int)l;
            }
        }
        sp_row_reg<16>(R, r, s0, len, dup);
    }
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr((unsigned long long *)&R.f[F_NET_ERR], SP_DUP_BIT);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr((unsigned long long *)&R.f[F_NET_ERR], 4ull);
}

__global__ void k_sp_w32_rows(const __grid_constant__ SpRows R, const int32_t *rows, const int32_t *n_rows) {
    const int nr = *n_rows;
    unsigned dup = 0;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nr; i += (gridDim.x * blockDim.x) >> 5) {
        const int64_t r = rows[i];
        sp_row_reg<32>(R, r, R.ro[r], (int)R.cnt[r], dup);
    }
    if (__any_sync(0xffffffffu, dup) && (threadIdx.x & 31) == 0)
        atomicOr((unsigned long long *)&R.f[F_NET_ERR], SP_DUP_BIT);
}

// rows of 33..SP_MED_MAX pair arcs: a warp each; keys staged through shared
// memory (coalesced loads and stores), 32*E of them sorted in registers
template <int E>
__device__ __forceinline__ void sp_warp_row(const SpRows &R, int64_t r, int64_t s0, int len, uint32_t *sk,
                                            unsigned &dup, int lane) {
    for (int i = lane; i < 32 * E; i += 32) sk[i] = i < len ? R.sh[s0 + i] : 0xffffffffu;
    __syncwarp();
    uint32_t v[E];
#pragma unroll
    for (int q = 0; q < E; q++) v[q] = sk[lane * E + q];
    warp_bitonic<E, uint32_t>(v, lane);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < E; q++) sk[lane * E + q] = v[q];
    __syncwarp();
    for (int i = lane; i < len; i += 32) {
        const uint32_t key = sk[i];
        if (i > 0 && key == sk[i - 1]) dup = 1;
        sp_put(R, r, s0, i, key);
    }
    __syncwarp();
}

// CLS 0: rows of 33..256; 1: 257..SP_MED_MAX (more registers: a kernel of its own
// so the common class keeps its occupancy)
template <int CLS>
__global__ void __launch_bounds__(CSR_MB) k_sp_med_rows(const __grid_constant__ SpRows R, const int32_t *rows,
                                                        const int32_t *n_rows) {
    constexpr int SK = CLS == 1 ? SP_MED_MAX : 256;
    __shared__ uint32_t sk_all[CSR_MB / 32][SK];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *sk = sk_all[wid];
    const int nr = *n_rows;
    unsigned dup = 0;
    for (int ri = blockIdx.x * (CSR_MB / 32) + wid; ri < nr; ri += gridDim.x * (CSR_MB / 32)) {
        const int64_t r = rows[ri];
        const int64_t s0 = R.ro[r];
        const int len = (int)R.cnt[r];
        if (CLS == 1) {
            sp_warp_row<SP_MED_MAX / 32>(R, r, s0, len, sk, dup, lane);
        } else {
            if (len <= 64) sp_warp_row<2>(R, r, s0, len, sk, dup, lane);
            else if (len <= 128) sp_warp_row<4>(R, r, s0, len, sk, dup, lane);
            else sp_warp_row<8>(R, r, s0, len, sk, dup, lane);
        }
    }
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr((unsigned long long *)&R.f[F_NET_ERR], SP_DUP_BIT);
}

// long rows, windowed: a CTA per row, ranks from a bitmap of the row's head span
// only (its heads are the representatives of the WSPD partners of its point's
// nodes -- spatially near it, so in the lexicographic point order their span is
// small: cfg5 s = 16, rows of 513..1024 arcs span ~460 32-bit words, of 1025+ arcs
// ~1070, of K/32 = 6200).  The row's span (a block min / max), its bits, a block
// scan of the span's word popcounts, then each head's rank = the popcounts before
// its word + the bits below it in its word.  The window is small, so many CTAs fit
// per SM.  A repeated head is flagged; rows whose span exceeds the window go to
// `ovf` (the full-K kernel below).
constexpr int WB_T = 256;       // threads per row
constexpr int WB_WORDS = 2048;  // window, 32-bit words (65536 head values)
constexpr int WB_SORTED = 4096; // rows up to this length are written coalesced from shared memory
__global__ void __launch_bounds__(WB_T) k_sp_win_bitmap(const __grid_constant__ SpRows R, const int32_t *rows,
                                                        const int32_t *n_rows, int32_t *ovf, int32_t *n_ovf) {
    __shared__ uint32_t bm[WB_WORDS], pre[WB_WORDS];
    __shared__ uint32_t sorted[WB_SORTED];
    __shared__ uint32_t s_warp[WB_T / 32];
    __shared__ unsigned s_lo[2], s_hi[2];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int w = tid; w < WB_WORDS; w += WB_T) bm[w] = 0;
    const int nr = *n_rows;
    unsigned dup = 0;
    int it = 0;
    for (int ri = blockIdx.x; ri < nr; ri += gridDim.x, it ^= 1) {
        const int64_t r = rows[ri];
        const int64_t s0 = R.ro[r];
        const int len = (int)R.cnt[r];
        const uint32_t *hs = R.sh + s0;
        const double2 a = R.pts[r];
        if (tid == 0) {
            s_lo[it] = 0xffffffffu;
            s_hi[it] = 0;
        }
        __syncthreads();  // the previous row's clear and writes; this row's range reset
        unsigned lo = 0xffffffffu, hi = 0;
        for (int i = tid; i < len; i += WB_T) {
            const uint32_t h = hs[i];
            lo = min(lo, h);
            hi = max(hi, h);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0) {
            atomicMin(&s_lo[it], lo);
            atomicMax(&s_hi[it], hi);
        }
        __syncthreads();
        const int wlo = (int)(s_lo[it] >> 5), span = (int)(s_hi[it] >> 5) - wlo + 1;
        if (span > WB_WORDS) {  // (uniform) the full-K kernel takes it
            if (tid == 0) ovf[atomicAdd(n_ovf, 1)] = (int32_t)r;
            continue;
        }
        for (int i = tid; i < len; i += WB_T) {
            const uint32_t h = hs[i];
            const uint32_t bit = 1u << (h & 31);
            if (atomicOr(&bm[(h >> 5) - wlo], bit) & bit) dup = 1;
        }
        __syncthreads();
        const int per = (span + WB_T - 1) / WB_T;
        const int w0 = tid * per, w1 = min(span, w0 + per);
        uint32_t mine = 0;
        for (int w = w0; w < w1; w++) mine += __popc(bm[w]);
        uint32_t x = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        uint32_t base = x - mine;
#pragma unroll
        for (int w = 0; w < WB_T / 32; w++)
            if (w < wid) base += s_warp[w];
        for (int w = w0; w < w1; w++) {
            pre[w] = base;
            base += __popc(bm[w]);
        }
        __syncthreads();
        if (len <= WB_SORTED) {
            // heads into their sorted places in shared memory, then the row is written
            // in order: coalesced stores instead of one 32-byte sector per arc
            for (int i = tid; i < len; i += WB_T) {
                const uint32_t h = hs[i];
                const int w = (int)(h >> 5) - wlo;
                sorted[pre[w] + __popc(bm[w] & ((1u << (h & 31)) - 1u))] = h;
            }
            __syncthreads();
            for (int i = tid; i < len; i += WB_T) sp_put_head_a(R, a, s0 + i, sorted[i]);
        } else {
            for (int i = tid; i < len; i += WB_T) {
                const uint32_t h = hs[i];
                const int w = (int)(h >> 5) - wlo;
                sp_put_head_a(R, a, s0 + pre[w] + __popc(bm[w] & ((1u << (h & 31)) - 1u)), h);
            }
        }
        __syncthreads();
        for (int w = w0; w < w1; w++) bm[w] = 0;
    }
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr((unsigned long long *)&R.f[F_NET_ERR], SP_DUP_BIT);
}

// long rows by rank instead of comparison: heads are distinct within a row
// and below K, so a row's heads mark a K-bit bitmap in shared memory; a block
// scan of the per-word popcounts then gives every head its rank (its place in
// the sorted row) directly.  Only the words between the row's smallest and
// largest head are scanned and cleared: a row's heads are the representatives of
// the WSPD partners of its point's nodes, spatially near it, so in the lexicographic
// point order their span is a small part of K (cfg5 s = 16: rows of 513..1024
// arcs span ~460 words of 6200).  O(len + span/32) per row, a CTA per row.  A head
// already marked is a repeated (tail, head).
constexpr int SP_BM_THREADS = 512;
__global__ void __launch_bounds__(SP_BM_THREADS) k_sp_long_bitmap(const __grid_constant__ SpRows R,
                                                                  const int32_t *rows, const int32_t *n_rows,
                                                                  int64_t K) {
    extern __shared__ uint32_t sbm[];  // W bitmap words, then W exclusive popcount prefixes
    const int W = (int)((K + 31) >> 5);
    uint32_t *pre = sbm + W;
    __shared__ uint32_t s_warp[SP_BM_THREADS / 32];
    __shared__ unsigned s_lo, s_hi;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < W; i += SP_BM_THREADS) sbm[i] = 0;
    const int nr = *n_rows;
    unsigned dup = 0;
    for (int ri = blockIdx.x; ri < nr; ri += gridDim.x) {
        const int64_t r = rows[ri];
        const int64_t s0 = R.ro[r];
        const int len = (int)R.cnt[r];
        if (tid == 0) {
            s_lo = 0xffffffffu;
            s_hi = 0;
        }
        __syncthreads();  // bitmap clear (previous row), range reset
        unsigned lo = 0xffffffffu, hi = 0;
        for (int i = tid; i < len; i += SP_BM_THREADS) {
            const uint32_t h = R.sh[s0 + i];
            const uint32_t bit = 1u << (h & 31);
            if (atomicOr(&sbm[h >> 5], bit) & bit) dup = 1;
            lo = min(lo, h);
            hi = max(hi, h);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        if (lane == 0) {
            atomicMin(&s_lo, lo);
            atomicMax(&s_hi, hi);
        }
        __syncthreads();
        // exclusive prefix of the word popcounts over the row's span: a contiguous
        // run of words per thread
        const int wlo = (int)(s_lo >> 5), whi = (int)(s_hi >> 5);
        const int span = whi - wlo + 1;
        const int per = (span + SP_BM_THREADS - 1) / SP_BM_THREADS;
        const int w0 = wlo + tid * per, w1 = min(whi + 1, w0 + per);
        uint32_t mine = 0;
        for (int w = w0; w < w1; w++) mine += __popc(sbm[w]);
        uint32_t x = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        uint32_t base = x - mine;
        for (int w = 0; w < wid; w++) base += s_warp[w];
        for (int w = w0; w < w1; w++) {
            pre[w] = base;
            base += __popc(sbm[w]);
        }
        __syncthreads();
        for (int i = tid; i < len; i += SP_BM_THREADS) {
            const uint32_t h = R.sh[s0 + i];
            const uint32_t rank = pre[h >> 5] + __popc(sbm[h >> 5] & ((1u << (h & 31)) - 1u));
            sp_put_head(R, r, s0 + rank, h);
        }
        __syncthreads();
        for (int w = w0; w < w1; w++) sbm[w] = 0;
    }
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr((unsigned long long *)&R.f[F_NET_ERR], SP_DUP_BIT);
}

// long rows when the bitmap does not fit (K above ~800k): a CTA each,
// bitonic sort in shared memory
__global__ void __launch_bounds__(CSR_LB) k_sp_long_rows(const __grid_constant__ SpRows R, const int32_t *rows,
                                                         const int32_t *n_rows) {
    __shared__ uint32_t sk[CSR_LONG_MAX];
    const int tid = threadIdx.x;
    const int nr = *n_rows;
    unsigned dup = 0;
    for (int ri = blockIdx.x; ri < nr; ri += gridDim.x) {
        const int64_t r = rows[ri];
        const int64_t s0 = R.ro[r];
        const int len = (int)R.cnt[r];
        int np2 = 64;
        while (np2 < len) np2 <<= 1;
        __syncthreads();
        for (int i = tid; i < np2; i += CSR_LB) sk[i] = i < len ? R.sh[s0 + i] : 0xffffffffu;
        __syncthreads();
        for (int k = 2; k <= np2; k <<= 1)
            for (int j = k >> 1; j; j >>= 1) {
                for (int i = tid; i < np2; i += CSR_LB) {
                    const int p = i ^ j;
                    if (p > i) {
                        const uint32_t a = sk[i], b = sk[p];
                        if ((a > b) == ((i & k) == 0)) {
                            sk[i] = b;
                            sk[p] = a;
                        }
                    }
                }
                __syncthreads();
            }
        for (int i = tid; i < len; i += CSR_LB) {
            const uint32_t key = sk[i];
            if (i > 0 && key == sk[i - 1]) dup = 1;
            sp_put(R, r, s0, i, key);
        }
    }
    if (__any_sync(0xffffffffu, dup) && (tid & 31) == 0) atomicOr((unsigned long long *)&R.f[F_NET_ERR], SP_DUP_BIT);
}

}  // namespace

int emit_run(Ctx &c, int64_t *n_arcs, bool with_diagonal) {
    NodeSet &ns = c.nodes[1];
    const int64_t K = ns.k, P = c.n_pairs;
    const int64_t *am = ptr<int64_t>(ns.am), *bm = ptr<int64_t>(ns.bm);
    int64_t *exa, *exb, na, nb;
    if (ns.na >= 0 && ns.exa.p && ns.exb.p) {
        // positions and counts from delta_condense: no host round trip here
        exa = ptr<int64_t>(ns.exa);
        exb = ptr<int64_t>(ns.exb);
        na = ns.na;
        nb = ns.nb;
    } else {
        W1G_TRY(ensure(c.scr[3], (size_t)K + 1, &exa));
        W1G_TRY(ensure(c.scr[6], (size_t)K + 1, &exb));
        W1G_TRY(flags_reset(c));
        W1G_TRY(scan_i64(c, PosFlag{am}, K, exa, dflags(c) + F_MISC0));
        W1G_TRY(scan_i64(c, PosFlag{bm}, K, exb, dflags(c) + F_MISC1));
        W1G_TRY(flags_fetch(c, F_MISC0, 2));
        na = c.h_pinned[F_MISC0];
        nb = c.h_pinned[F_MISC1];
    }
    const int64_t M = 2 * P + (with_diagonal ? na + nb + 1 : 0);
    int64_t *t, *h;
    double *cs;
    W1G_TRY(ensure(c.arc_t, (size_t)M, &t));
    W1G_TRY(ensure(c.arc_h, (size_t)M, &h));
    W1G_TRY(ensure(c.arc_c, (size_t)M, &cs));
    if (P) {
        W1G_TRY(wspd_pair_idx(c));
        const double2 *pp = c.pair_pts ? c.pair_pts : ptr<double2>(ns.pts);
        k_emit_spanner<<<gs(c, P), 256, 0, c.stream>>>(ptr<int64_t>(c.pair_idx), P, pp, t, h, cs);
        W1G_CHECK_LAUNCH();
    }
    if (K && with_diagonal) {
        k_emit_diag<<<gs(c, K), 256, 0, c.stream>>>(ptr<double2>(ns.pts), am, bm, K, exa, exb, na, 2 * P, t, h,
                                                    cs);
        W1G_CHECK_LAUNCH();
    }
    if (with_diagonal) {
        k_emit_free<<<1, 1, 0, c.stream>>>(K, M - 1, t, h, cs);
        W1G_CHECK_LAUNCH();
    }
    c.n_arcs = M;
    c.arcs_valid = true;
    *n_arcs = M;
    return W1G_OK;
}

int assemble_supplies(Ctx &c, int64_t **d_sup, int64_t *n) {
    NodeSet &ns = c.nodes[1];
    const int64_t K = ns.k;
    int64_t *sup;
    W1G_TRY(ensure(c.net_sup, (size_t)K + 2, &sup));
    k_supplies<<<gs(c, K + 2), 256, 0, c.stream>>>(ptr<int64_t>(ns.am), ptr<int64_t>(ns.bm), K, ns.abar,
                                                   ns.bbar, sup);
    W1G_CHECK_LAUNCH();
    *d_sup = sup;
    *n = K + 2;
    return W1G_OK;
}

// fallback for rows longer than CSR_LONG_MAX arcs: one (tail, head) radix sort
static int net_run_sorted(Ctx &c, const int64_t *d_sup, int64_t n, int64_t *n_arcs) {
    c.net_valid = false;
    const int64_t m = c.n_arcs;
    const int64_t *t = ptr<int64_t>(c.arc_t), *h = ptr<int64_t>(c.arc_h);
    const double *cs = ptr<double>(c.arc_c);
    SubTimer T(c, "csr");
    W1G_TRY(flags_reset(c));
    k_validate<<<gs(c, m > n ? m : n), 256, 0, c.stream>>>(d_sup, n, t, h, cs, m, dflags(c));
    W1G_CHECK_LAUNCH();
    W1G_TRY(flags_fetch(c, 0, F_NSLOTS / 2));
    T.mark("validate");
    if (c.h_pinned[F_MISC0] != 0) {
        set_error("unbalanced supplies (sum = %lld)", (long long)c.h_pinned[F_MISC0]);
        return W1G_ENETWORK;
    }
    const int64_t bits = c.h_pinned[F_NET_ERR];
    if (bits & 1) { set_error("arc endpoint out of range"); return W1G_ENETWORK; }
    if (bits & 2) { set_error("self-loop arc"); return W1G_ENETWORK; }
    if (bits & 4) { set_error("non-finite arc cost"); return W1G_ENETWORK; }
    if (bits & 8) { set_error("negative arc cost"); return W1G_ENETWORK; }
    int64_t *ro;
    W1G_TRY(ensure(c.net_ro, (size_t)n + 2, &ro));
    int64_t *ot, *oh;
    double *oc;
    W1G_TRY(ensure(c.net_t, (size_t)m + 1, &ot));
    W1G_TRY(ensure(c.net_h, (size_t)m + 1, &oh));
    W1G_TRY(ensure(c.net_c, (size_t)m + 1, &oc));
    int64_t *rowcnt, *excl;
    W1G_TRY(ensure(c.scr[13], (size_t)n + 2, &rowcnt));
    W1G_CUDA(cudaMemsetAsync(rowcnt, 0, sizeof(int64_t) * (n + 2), c.stream));
    int64_t mm = 0;
    if (m > 0) {
        int hb = 1;
        while ((1ll << hb) < n) hb++;
        uint64_t *keys;
        uint32_t *vals;
        W1G_TRY(ensure(c.scr[0], (size_t)m, &keys));
        W1G_TRY(ensure(c.scr[2], (size_t)m, &vals));
        W1G_TRY(ensure(c.scr[3], (size_t)m, &excl));
        k_arc_keys<<<gs(c, m), 256, 0, c.stream>>>(t, h, m, hb, keys, vals);
        W1G_CHECK_LAUNCH();
        uint64_t *kk[1] = {keys};
        T.mark("keys");
        W1G_TRY(radix_sort(c, kk, 1, vals, m, 2 * hb));
        T.mark("sort");
        GroupFlag f{keys};
        W1G_TRY(scan_i64(c, f, m, excl, dflags(c) + F_TOTAL));
        k_net_emit<<<gs(c, m), 256, 0, c.stream>>>(f, m, excl, vals, t, h, cs, ot, oh, oc, rowcnt);
        W1G_CHECK_LAUNCH();
    }
    T.mark("dedup_emit");
    // row_offsets = [0, cumsum(bincount(t, n))], network.py:84-85
    W1G_TRY(scan_i64(c, RowCount{rowcnt, n}, n + 1, ro, nullptr));
    W1G_TRY(flags_fetch(c, F_TOTAL, 1));
    mm = m > 0 ? c.h_pinned[F_TOTAL] : 0;
    if (d_sup != ptr<int64_t>(c.net_sup))
        W1G_CUDA(cudaMemcpyAsync(c.net_sup.p, d_sup, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c.stream));
    c.net_n = n;
    c.net_m = mm;
    c.net_valid = true;
    *n_arcs = mm;
    return W1G_OK;
}

// rows average <= this many arcs: bucket by tail (cheaper for s ~ 1); longer
// rows (large s) are cheaper to order with one (tail, head) radix sort
constexpr int64_t CSR_BUCKET_MAX_AVG = 24;

int net_run(Ctx &c, const int64_t *d_sup, int64_t n, int64_t *n_arcs) {
    c.net_valid = false;
    const int64_t m = c.n_arcs;
    if (m > CSR_BUCKET_MAX_AVG * n) return net_run_sorted(c, d_sup, n, n_arcs);
    const int64_t *t = ptr<int64_t>(c.arc_t), *h = ptr<int64_t>(c.arc_h);
    const double *cs = ptr<double>(c.arc_c);
    SubTimer T(c, "csr");
    int64_t *ro, *ot, *oh, *start, *dcnt;
    double *oc, *slot_c;
    unsigned *cnt, *cursor, *tab_e;
    unsigned long long *tab_c;
    int32_t *slot_h, *lists;
    uint32_t *slot_e;
    W1G_TRY(ensure(c.net_ro, (size_t)n + 2, &ro));
    W1G_TRY(ensure(c.net_t, (size_t)m + 1, &ot));
    W1G_TRY(ensure(c.net_h, (size_t)m + 1, &oh));
    W1G_TRY(ensure(c.net_c, (size_t)m + 1, &oc));
    W1G_TRY(ensure(c.scr[13], (size_t)2 * (n + 2) + 8, &cnt));
    cursor = cnt + n + 2;
    W1G_TRY(ensure(c.scr[3], (size_t)n + 2, &start));
    W1G_TRY(ensure(c.scr[5], (size_t)n + 1, &dcnt));
    W1G_TRY(ensure(c.scr[6], (size_t)4 * (n + 1), &lists));
    W1G_TRY(ensure(c.scr[0], (size_t)m + 1, &slot_h));
    W1G_TRY(ensure(c.scr[2], (size_t)m + 1, &slot_e));
    W1G_TRY(ensure(c.scr[4], (size_t)m + 1, &slot_c));
    W1G_TRY(ensure(c.scr[7], (size_t)CSR_HUGE_CAP * (n + 1), &tab_c));
    W1G_TRY(ensure(c.scr[8], (size_t)CSR_HUGE_CAP * (n + 1), &tab_e));
    int64_t *hpos;
    W1G_TRY(ensure(c.scr[9], (size_t)CSR_HUGE_CAP * n + 2, &hpos));
    int32_t *n_list = reinterpret_cast<int32_t *>(dflags(c) + F_MISC2);  // 4 int32 counters (F_MISC2, F_MISC3)
    W1G_TRY(flags_reset(c));
    W1G_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * 2 * (n + 2), c.stream));
    // validation is checked at the one host round trip at the end; invalid
    // arcs are never bucketed, so nothing is written out of range meanwhile
    k_csr_count<<<gs(c, m > n ? m : n), 256, 0, c.stream>>>(d_sup, n, t, h, cs, m, cnt, dflags(c));
    W1G_CHECK_LAUNCH();
    W1G_TRY(scan_i64(c, RowLen{cnt, n}, n + 1, start, nullptr));
    if (m > 0) {
        k_csr_scatter<<<gs(c, m), 256, 0, c.stream>>>(t, h, m, n, start, cursor, slot_h, slot_e);
        W1G_CHECK_LAUNCH();
    }
    T.mark("bucket");
    if (n > 0) {
        k_csr_short_rows<<<grid_for(n * 16, 256, 16u * c.sm_count), 256, 0, c.stream>>>(
            start, n, slot_h, slot_e, cs, slot_c, dcnt, lists, n_list, dflags(c));
        W1G_CHECK_LAUNCH();
        k_csr_w32_rows<<<4 * c.sm_count, 256, 0, c.stream>>>(start, lists + CL_W32 * n, n_list + CL_W32, slot_h,
                                                             slot_e, cs, slot_c, dcnt);
        W1G_CHECK_LAUNCH();
        T.mark("short");
        k_csr_med_rows<<<8 * c.sm_count, CSR_MB, 0, c.stream>>>(start, lists + CL_MED * n, n_list + CL_MED,
                                                                slot_h, slot_e, cs, slot_c, dcnt);
        W1G_CHECK_LAUNCH();
        k_csr_long_rows<<<c.sm_count, CSR_LB, 0, c.stream>>>(start, lists + CL_LONG * n, n_list + CL_LONG, slot_h,
                                                             slot_e, cs, slot_c, dcnt);
        W1G_CHECK_LAUNCH();
        T.mark("med_long");
        const int32_t *hrows = lists + CL_HUGE * n, *nh = n_list + CL_HUGE;
        const unsigned gh = grid_for((int64_t)CSR_HUGE_CAP * n, 256, 8u * c.sm_count);
        k_huge_init<<<gh, 256, 0, c.stream>>>(nh, n, tab_c, tab_e);
        W1G_CHECK_LAUNCH();
        k_huge_fold<0><<<gs(c, m), 256, 0, c.stream>>>(start, hrows, nh, n, slot_h, slot_e, cs, tab_c, tab_e);
        W1G_CHECK_LAUNCH();
        k_huge_fold<1><<<gs(c, m), 256, 0, c.stream>>>(start, hrows, nh, n, slot_h, slot_e, cs, tab_c, tab_e);
        W1G_CHECK_LAUNCH();
        W1G_TRY(scan_i64(c, HugeHit{tab_c, nh, n}, (int64_t)CSR_HUGE_CAP * n + 1, hpos, nullptr));
        k_huge_write<<<gs(c, n), 256, 0, c.stream>>>(start, hrows, nh, n, tab_c, tab_e, hpos, cs, slot_h, slot_c,
                                                     dcnt);
        W1G_CHECK_LAUNCH();
    }
    T.mark("huge");
    // row_offsets = [0, cumsum(bincount(t, n))], network.py:84-85
    W1G_TRY(scan_i64(c, DCount{dcnt, n}, n + 1, ro, dflags(c) + F_TOTAL));
    if (n > 0) {
        k_csr_emit<<<grid_for(n * 16, 256, 16u * c.sm_count), 256, 0, c.stream>>>(start, ro, n, slot_h, slot_c, ot,
                                                                                  oh, oc);
        W1G_CHECK_LAUNCH();
        k_csr_emit_long<<<2 * c.sm_count, 256, 0, c.stream>>>(start, ro, n, lists, n_list, slot_h, slot_c, ot, oh, oc);
        W1G_CHECK_LAUNCH();
    }
    W1G_TRY(flags_fetch(c, 0, F_NSLOTS / 2));
    T.mark("emit");
    // network.py:55-68, in the reference's order
    if (c.h_pinned[F_MISC0] != 0) {
        set_error("unbalanced supplies (sum = %lld)", (long long)c.h_pinned[F_MISC0]);
        return W1G_ENETWORK;
    }
    const int64_t bits = c.h_pinned[F_NET_ERR];
    if (bits & 1) { set_error("arc endpoint out of range"); return W1G_ENETWORK; }
    if (bits & 2) { set_error("self-loop arc"); return W1G_ENETWORK; }
    if (bits & 4) { set_error("non-finite arc cost"); return W1G_ENETWORK; }
    if (bits & 8) { set_error("negative arc cost"); return W1G_ENETWORK; }
    if (c.h_pinned[F_OVERFLOW]) return net_run_sorted(c, d_sup, n, n_arcs);
    const int64_t mm = c.h_pinned[F_TOTAL];
    if (d_sup != ptr<int64_t>(c.net_sup))
        W1G_CUDA(cudaMemcpyAsync(c.net_sup.p, d_sup, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, c.stream));
    c.net_n = n;
    c.net_m = mm;
    c.net_valid = true;
    *n_arcs = mm;
    return W1G_OK;
}

// emit_arcs + assemble of the fused front end (see k_sp_count): the network
// straight from the pairs.  Its validation flags travel to the host with the
// front end's final wait; spanner_net_check reads them (and redoes the
// network on the generic path in the cases that need it).
static int spanner_generic(Ctx &c, int64_t *node_count, int64_t *n_arcs) {
    c.net_early_copy = false;
    int64_t M, *dsup, nsup;
    W1G_TRY(emit_run(c, &M));
    W1G_TRY(assemble_supplies(c, &dsup, &nsup));
    *node_count = nsup;
    return net_run(c, dsup, nsup, n_arcs);
}

int spanner_net_run(Ctx &c, int64_t *node_count, int64_t *n_arcs) {
    c.net_valid = false;
    c.net_check_pending = false;
    NodeSet &ns = c.nodes[1];
    const int64_t K = ns.k, P = c.n_pairs;
    const int64_t n = K + 2;
    const char *e = getenv("W1G_GENERIC_CSR");
    if ((e && *e == '1') || K < 1 || ns.na < 0 || !ns.exb.p || !c.pairs_have_nodes || P >= (1ll << 31) ||
        n >= (1ll << 31))
        return spanner_generic(c, node_count, n_arcs);
    const int64_t M = 2 * P + ns.na + ns.nb + 1;
    // W1G_SP_LONG_MAX (tests): a lower row-length limit, to exercise the fallback
    // rows longer than that are ranked by the bitmap kernel when a K-bit bitmap (+ its
    // prefixes) fits in shared memory, whatever their length; otherwise they are
    // limited by the CTA bitonic sort's buffer
    const size_t bm_bytes = (size_t)8 * ((K + 31) / 32);
    const bool bitmap_fits = bm_bytes <= 200 * 1024;
    unsigned long_max = bitmap_fits ? 0xffffffffu : (unsigned)CSR_LONG_MAX;
    if (const char *lm = getenv("W1G_SP_LONG_MAX")) long_max = (unsigned)atoi(lm);
    if (!bitmap_fits && long_max > (unsigned)CSR_LONG_MAX) long_max = CSR_LONG_MAX;
    // rows of 257..big_max: a warp in registers, longer: the bitmap ranks (W1G_SP_BIG_MAX: tuning;
    // since the windowed bitmap kernel the ranks are faster from 257 arcs: cfg5 s = 16
    // delta = 0.001, 3.98 ms vs 4.29 with the register sorts up to 512)
    unsigned big_max = 256;
    if (const char *bm = getenv("W1G_SP_BIG_MAX")) big_max = (unsigned)atoi(bm);
    if (big_max > (unsigned)SP_MED_MAX) big_max = SP_MED_MAX;
    // rows of 33..med_max: a warp's register sort (W1G_SP_MED_MAX: tuning, <= 256)
    unsigned med_max = 256;
    if (const char *mm = getenv("W1G_SP_MED_MAX")) med_max = (unsigned)atoi(mm);
    if (med_max > 256u) med_max = 256u;
    if (med_max < 32u) med_max = 32u;
    // the whole CSR build, one graph (graph_segment); the flags ride on the caller's final wait
    W1G_TRY(graph_segment(c, GSEG_CSR, [&]() -> int {
        SubTimer T(c, "spcsr");
        int64_t *sup, *ro, *ot, *oh;
        double *oc;
        unsigned *cnt;
        uint32_t *sh;
        int32_t *lists;
        W1G_TRY(ensure(c.net_sup, (size_t)n, &sup));
        W1G_TRY(ensure(c.net_ro, (size_t)n + 2, &ro));
        W1G_TRY(ensure(c.net_t, (size_t)M + 1, &ot));
        W1G_TRY(ensure(c.net_h, (size_t)M + 1, &oh));
        W1G_TRY(ensure(c.net_c, (size_t)M + 1, &oc));
        W1G_TRY(ensure(c.scr[13], (size_t)2 * (n + 2) + 8, &cnt));
        unsigned *cursor = cnt + n + 2;
        // slots sit at their final CSR positions (the diagonal ones stay unused)
        W1G_TRY(ensure(c.scr[0], (size_t)M + 1, &sh));
        W1G_TRY(ensure(c.scr[6], (size_t)5 * (K + 1), &lists));
        int32_t *n_list = reinterpret_cast<int32_t *>(cnt + 2 * (n + 2));  // 5 int32 class counters
        W1G_TRY(flags_reset(c));
        W1G_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned) * (2 * (n + 2) + 8), c.stream));
        const int2 *uv = ptr<int2>(c.pair_uv);
        const int32_t *rep = ptr<int32_t>(c.t_rep32);
        const double2 *pp = c.pair_pts ? c.pair_pts : ptr<double2>(ns.pts);
        if (P) {
            k_sp_count<<<gs(c, P), 256, 0, c.stream>>>(uv, rep, P, cnt);
            W1G_CHECK_LAUNCH();
        }
        W1G_TRY(scan_i64(c, SpRowLen{cnt, ptr<int64_t>(ns.am), K, ns.nb}, n + 1, ro, nullptr));
        // the tails depend on the row offsets alone: on the side stream, concurrently with the
        // scatter and the row sorts, followed there by their early D2H copy (when armed)
        cudaStream_t side = c.copy_stream ? c.copy_stream : c.stream;
        if (side != c.stream) {
            W1G_CUDA(cudaEventRecord(c.ev[12], c.stream));
            W1G_CUDA(cudaStreamWaitEvent(side, c.ev[12], 0));
        }
        k_sp_tails<<<gs(c, M), 256, 0, side>>>(ro, K, ot);
        W1G_CHECK_LAUNCH();
        c.net_early_copy = false;
        c.net_tails_host = false;
        {
            const Ctx::NetOut &o = c.net_out;
            const bool early_env = [] {  // W1G_EARLY_COPY=0: copy everything after the rows (read per call)
                const char *e = getenv("W1G_EARLY_COPY");
                return !(e && *e == '0');
            }();
            // W1G_HOST_TAILS=0: copy the tails too (by default the host rebuilds them from the
            // row offsets while the rest of the network crosses the link: 15 of 47 MB at cfg2)
            const bool host_tails = [] {
                const char *e = getenv("W1G_HOST_TAILS");
                return !(e && *e == '0');
            }();
            if (early_env && o.sup && n <= o.node_cap && M <= o.arc_cap && side != c.stream) {
                W1G_CUDA(cudaMemcpyAsync(o.ro, ro, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, side));
                if (host_tails) {
                    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                    W1G_CUDA(cudaStreamIsCapturing(side, &cs));
                    W1G_CUDA(cudaEventRecordWithFlags(c.ev[16], side,
                                                      cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                                           : 0));
                    c.net_tails_host = true;
                } else {
                    W1G_CUDA(cudaMemcpyAsync(o.t, ot, sizeof(int64_t) * M, cudaMemcpyDeviceToHost, side));
                }
                c.net_early_copy = true;
            }
        }
        // (also waited for after this stage: a graph-external record when captured)
    if (side != c.stream) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        W1G_CUDA(cudaStreamIsCapturing(side, &cs));
        W1G_CUDA(cudaEventRecordWithFlags(c.ev[13], side,
                                          cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0));
    }
        if (P) {
            k_sp_scatter<<<gs(c, P), 256, 0, c.stream>>>(uv, rep, P, ro, cursor, sh);
            W1G_CHECK_LAUNCH();
        }
        T.mark("bucket");
        const SpRows R{ro, cnt, sh, pp, ot, oh, oc, dflags(c)};
        const DiagArgs D{ptr<double2>(ns.pts), ptr<int64_t>(ns.am), ptr<int64_t>(ns.bm), ptr<int64_t>(ns.exb),
                         ns.abar, ns.bbar, sup};
        k_sp_short_rows<<<grid_for(K * 16, 256, 16u * c.sm_count), 256, 0, c.stream>>>(R, K, lists, n_list, long_max,
                                                                                       med_max, big_max, D);
        W1G_CHECK_LAUNCH();
        k_sp_w32_rows<<<4 * c.sm_count, 256, 0, c.stream>>>(R, lists + CL_W32 * K, n_list + CL_W32);
        W1G_CHECK_LAUNCH();
        k_sp_med_rows<0><<<8 * c.sm_count, CSR_MB, 0, c.stream>>>(R, lists + CL_MED * K, n_list + CL_MED);
        W1G_CHECK_LAUNCH();
        T.mark("short_med");
        if (big_max > med_max) {  // (rows of med_max+1..big_max; none by default)
            k_sp_med_rows<1><<<4 * c.sm_count, CSR_MB, 0, c.stream>>>(R, lists + SP_CL_BIG * K, n_list + SP_CL_BIG);
            W1G_CHECK_LAUNCH();
        }
        T.mark("big");
        {
            // long rows: bitmap ranks while a K-bit bitmap (+ prefixes) fits in shared memory;
            // as many CTAs per SM as the bitmap allows (a row's phases are latency-bound)
            if (bitmap_fits) {
                const int32_t *cta_rows = lists + CL_LONG * K, *cta_n = n_list + CL_LONG;
                static const bool win_bm = [] {  // W1G_SP_WIN_BITMAP=0: the full-K kernel for every long row
                    const char *e = getenv("W1G_SP_WIN_BITMAP");
                    return !(e && *e == '0');
                }();
                if (win_bm) {
                    // a CTA per row over its head span; rows with wider spans to the full-K kernel
                    int32_t *ovf = lists + 4 * K, *n_ovf = n_list + 4;
                    int per = 1;
                    W1G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sp_win_bitmap, WB_T, 0));
                    if (per < 1) per = 1;
                    k_sp_win_bitmap<<<per * c.sm_count, WB_T, 0, c.stream>>>(R, cta_rows, cta_n, ovf, n_ovf);
                    W1G_CHECK_LAUNCH();
                    cta_rows = ovf;
                    cta_n = n_ovf;
                }
                if (bm_bytes > 48 * 1024)
                    W1G_CUDA(cudaFuncSetAttribute(k_sp_long_bitmap, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)bm_bytes));
                int per_sm = 1;
                W1G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sp_long_bitmap, SP_BM_THREADS,
                                                                       bm_bytes));
                if (per_sm < 1) per_sm = 1;
                k_sp_long_bitmap<<<per_sm * c.sm_count, SP_BM_THREADS, bm_bytes, c.stream>>>(R, cta_rows, cta_n, K);
            } else {
                k_sp_long_rows<<<c.sm_count, CSR_LB, 0, c.stream>>>(R, lists + CL_LONG * K, n_list + CL_LONG);
            }
            W1G_CHECK_LAUNCH();
        }
        T.mark("long");
        if (side != c.stream) W1G_CUDA(cudaStreamWaitEvent(c.stream, c.ev[13], 0));  // the tails (and their copy)
        // the flags ride on the caller's final wait (no round trip here)
        W1G_TRY(to_host_small(c, c.h_pinned + F_OVERFLOW, dflags(c) + F_OVERFLOW,
                              sizeof(int64_t) * (F_NET_ERR - F_OVERFLOW + 1)));
        return W1G_OK;
    }));
    c.net_check_pending = true;
    c.arcs_valid = false;  // never materialised on this path
    c.net_n = n;
    c.net_m = M;
    c.net_valid = true;
    *node_count = n;
    *n_arcs = M;
    return W1G_OK;
}

// after the stream has drained: network.py:64-65 (balance, ranges and
// self-loops hold by construction), or the generic path when a row was too
// long or a (tail, head) repeated
int spanner_net_check(Ctx &c, int64_t *node_count, int64_t *n_arcs, bool *redone) {
    *redone = false;
    if (!c.net_check_pending) return W1G_OK;
    c.net_check_pending = false;
    const int64_t bits = c.h_pinned[F_NET_ERR];
    if (bits & 4) {
        c.net_valid = false;
        set_error("non-finite arc cost");
        return W1G_ENETWORK;
    }
    if ((bits & SP_DUP_BIT) || c.h_pinned[F_OVERFLOW]) {
        *redone = true;
        return spanner_generic(c, node_count, n_arcs);
    }
    return W1G_OK;
}

}  // namespace w1g
