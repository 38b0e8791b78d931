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

namespace w1g {

static const double SQRT2 = 1.4142135623730951;

namespace {

// glibc sysdeps/ieee754/dbl-64/e_hypot.c (2.35+), the non-FMA kernel that
// x86-64 numpy calls; verified bit-exact against libm in tests/.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
    double t1, t2;
    double h = dsqrt(dadd(dmul(ax, ax), dmul(ay, ay)));
    if (h <= dmul(2.0, ay)) {
        const double delta = dsub(h, ay);
        t1 = dmul(ax, dsub(dmul(2.0, delta), ax));
        t2 = dmul(dsub(delta, dmul(2.0, dsub(ax, ay))), delta);
    } else {
        const double delta = dsub(h, ax);
        t1 = dmul(dmul(2.0, delta), dsub(ax, dmul(2.0, ay)));
        t2 = dadd(dmul(dsub(dmul(4.0, delta), ay), ay), dmul(delta, delta));
    }
    return dsub(h, ddiv(dadd(t1, t2), dmul(2.0, h)));
}

__device__ double glibc_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return dadd(x, y);
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ax > 0x1p+511) {
        if (ay <= dmul(ax, 0x1p-54)) return dadd(ax, ay);
        return ddiv(hypot_kernel(dmul(ax, 0x1p-600), dmul(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay < 0x1p-511) {
        if (ax >= ddiv(ay, 0x1p-54)) return dadd(ax, ay);
        return dmul(hypot_kernel(ddiv(ax, 0x1p-600), ddiv(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay <= dmul(ax, 0x1p-54)) return dadd(ax, ay);
    return hypot_kernel(ax, ay);
}

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
                            const int64_t *exa, const int64_t *exb, const int64_t *n_a, int64_t base,
                            int64_t *tails, int64_t *heads, double *costs) {
    const int64_t na = *n_a;
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
        // np.minimum.at over the duplicate group (network.py:75-76)
        for (int64_t j = i + 1; j < m && !f(j); j++) {
            const double cj = c[perm[j]];
            cm = cj < cm ? cj : cm;
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

}  // namespace

int emit_run(Ctx &c, int64_t *n_arcs) {
    NodeSet &ns = c.nodes[1];
    const int64_t K = ns.k, P = c.n_pairs;
    const int64_t *am = ptr<int64_t>(ns.am), *bm = ptr<int64_t>(ns.bm);
    int64_t *exa, *exb;
    W1G_TRY(ensure(c.scr[3], (size_t)K + 1, &exa));
    W1G_TRY(ensure(c.scr[6], (size_t)K + 1, &exb));
    W1G_TRY(flags_reset(c));
    W1G_TRY(scan_i64(c, PosFlag{am}, K, exa, dflags(c) + F_MISC0));
    W1G_TRY(scan_i64(c, PosFlag{bm}, K, exb, dflags(c) + F_MISC1));
    W1G_TRY(flags_fetch(c, F_MISC0, 2));
    const int64_t na = c.h_pinned[F_MISC0], nb = c.h_pinned[F_MISC1];
    const int64_t M = 2 * P + na + nb + 1;
    int64_t *t, *h;
    double *cs;
    W1G_TRY(ensure(c.arc_t, (size_t)M, &t));
    W1G_TRY(ensure(c.arc_h, (size_t)M, &h));
    W1G_TRY(ensure(c.arc_c, (size_t)M, &cs));
    if (P) {
        const double2 *pp = c.pair_pts ? c.pair_pts : ptr<double2>(ns.pts);
        k_emit_spanner<<<gs(c, P), 256, 0, c.stream>>>(ptr<int64_t>(c.pair_idx), P, pp, t, h, cs);
        W1G_CHECK_LAUNCH();
    }
    if (K) {
        k_emit_diag<<<gs(c, K), 256, 0, c.stream>>>(ptr<double2>(ns.pts), am, bm, K, exa, exb,
                                                    dflags(c) + F_MISC0, 2 * P, t, h, cs);
        W1G_CHECK_LAUNCH();
    }
    k_emit_free<<<1, 1, 0, c.stream>>>(K, M - 1, t, h, cs);
    W1G_CHECK_LAUNCH();
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

int net_run(Ctx &c, const int64_t *d_sup, int64_t n, int64_t *n_arcs) {
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

}  // namespace w1g
