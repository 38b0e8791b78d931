// corpus.cu -- the retrieval side of the reference (pipeline.py:146-243,
// lower_bound.py:78-92, oracle.py:66-108) on device.
//
// * a diagram corpus is uploaded once per context (points back to back plus
//   offsets) and stays resident across queries;
// * WCD of a query against every listed candidate in ONE launch: four lanes
//   per candidate run the four sequential sums numpy's mean(axis=0) performs
//   over (n, 2) arrays (verified: for a C-contiguous (n, 2) array the axis-0
//   reduction adds the rows in order), then gap, glibc hypot and N*h/2 with
//   the reference's IEEE operations;
// * RWMD of a query against the candidates: zero_condense + the device RWMD
//   per candidate, back to back on the context stream with no host work in
//   between except the K0 read;
// * the dense exact-oracle network over a node set: all A-member x B-member
//   arcs (minus the zero-cost dual self pairs) and the diagonal arcs written
//   straight into CSR order -- np.lexsort((heads, tails)) of that arc set is
//   the row-major order, so no sort is needed.
#include "common.cuh"
#include "hypot.cuh"

namespace w1g {

namespace {

constexpr double SQRT2_C = 1.4142135623730951;  // math.sqrt(2.0)

// lanes 4c..4c+3 of the grid own candidate c: lane&1 = coordinate, lane&2 = which mean.
// x = concat(query, proj(cand)), y = concat(cand, proj(query)) (lower_bound.py:88-89)
__global__ void k_wcd(const double2 *__restrict__ q, int64_t nq, const double2 *__restrict__ corpus,
                      const int64_t *__restrict__ off, const int64_t *__restrict__ cand, int64_t ncand,
                      double *__restrict__ out) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ci = g >> 2;
    const int role = (int)(g & 3);
    const bool live = ci < ncand;
    double sum = 0.0;
    int64_t n = 0;
    if (live) {
        const int64_t id = cand[ci];
        const double2 *cp = corpus + off[id];
        const int64_t nc = off[id + 1] - off[id];
        n = nq + nc;
        const bool ycoord = role & 1;
        const double2 *pts = (role & 2) ? cp : q;       // own points first
        const int64_t np_ = (role & 2) ? nc : nq;
        const double2 *prj = (role & 2) ? q : cp;       // then the other's projections
        const int64_t npr = (role & 2) ? nq : nc;
        // numpy's axis-0 add.reduce starts from its identity +0.0 (so a column of
        // -0.0 sums to +0.0) and adds the rows in order
#pragma unroll 8
        for (int64_t i = 0; i < np_; i++) {
            const double2 p = pts[i];
            sum = dadd(sum, ycoord ? p.y : p.x);
        }
#pragma unroll 8
        for (int64_t i = 0; i < npr; i++) {
            const double2 p = prj[i];
            sum = dadd(sum, dmul(0.5, dadd(p.x, p.y)));  // diagonal_projections, diagram.py:50-54
        }
    }
    // lane groups of 4 are aligned within a warp
    const double mean = n ? ddiv(sum, (double)n) : 0.0;
    const double other = __shfl_xor_sync(0xffffffffu, mean, 2);  // the y-mean of the same coordinate
    const double gap = dsub(mean, other);                          // x.mean - y.mean for roles 0, 1
    const double gy = __shfl_xor_sync(0xffffffffu, gap, 1);
    if (live && role == 0) out[ci] = n ? ddiv(dmul((double)n, glibc_hypot(gap, gy)), 2.0) : 0.0;
}

struct MemberFlag {
    const int64_t *m;
    __device__ int64_t operator()(int64_t i) const { return m[i] > 0 ? 1 : 0; }
};

__global__ void k_compact_members(const int64_t *am, const int64_t *bm, int64_t k, const int64_t *apos,
                                  const int64_t *bpos, int32_t *aidx, int32_t *bidx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        if (am[i] > 0) aidx[apos[i]] = (int32_t)i;
        if (bm[i] > 0) bidx[bpos[i]] = (int32_t)i;
    }
}

// row lengths of the dense network: A-member t: (nB - [t is a B-member]) arcs to the
// B-members + t -> abar; abar: none; bbar: every B-member + bbar -> abar
struct DenseRowLen {
    const int64_t *am, *bm;
    const int64_t *nb;  // device total of the B-member scan
    int64_t k;
    __device__ int64_t operator()(int64_t t) const {
        if (t < k) return am[t] > 0 ? *nb - (bm[t] > 0 ? 1 : 0) + 1 : 0;
        if (t == k) return 0;
        return *nb + 1;
    }
};

// one CTA per A-member row (blockIdx.y-major grid-stride), then the bbar row
__global__ void __launch_bounds__(256) k_dense_rows(const double2 *__restrict__ pts, const int64_t *__restrict__ bm,
                                                    const int32_t *__restrict__ aidx, int64_t na,
                                                    const int32_t *__restrict__ bidx, int64_t nb, int64_t k,
                                                    const int64_t *__restrict__ ro, int64_t *__restrict__ tails,
                                                    int64_t *__restrict__ heads, double *__restrict__ costs,
                                                    int64_t *flags) {
    int bad = 0;
    for (int64_t r = blockIdx.x; r <= na; r += gridDim.x) {
        if (r < na) {
            const int64_t t = aidx[r];
            const double2 pt = pts[t];
            const bool tb = bm[t] > 0;
            const int64_t base = ro[t];
            for (int64_t j = threadIdx.x; j < nb; j += blockDim.x) {
                const int64_t h = bidx[j];
                if (h == t) continue;  // the dual node's zero-cost self pair (oracle.py:76)
                const int64_t pos = base + j - (tb && h > t ? 1 : 0);
                const double2 ph = pts[h];
                const double c = glibc_hypot(dsub(pt.x, ph.x), dsub(pt.y, ph.y));  // oracle.py:78-79
                bad |= !isfinite(c);
                tails[pos] = t;
                heads[pos] = h;
                costs[pos] = c;
            }
            if (threadIdx.x == 0) {
                const int64_t pos = ro[t + 1] - 1;
                tails[pos] = t;
                heads[pos] = k;  // abar
                costs[pos] = ddiv(fabs(dsub(pt.y, pt.x)), SQRT2_C);  // diagonal_distances, diagram.py:40-47
            }
        } else {
            const int64_t base = ro[k + 1];
            for (int64_t j = threadIdx.x; j < nb; j += blockDim.x) {
                const int64_t h = bidx[j];
                const double2 ph = pts[h];
                tails[base + j] = k + 1;  // bbar
                heads[base + j] = h;
                costs[base + j] = ddiv(fabs(dsub(ph.y, ph.x)), SQRT2_C);
            }
            if (threadIdx.x == 0) {
                tails[base + nb] = k + 1;
                heads[base + nb] = k;
                costs[base + nb] = 0.0;
            }
        }
    }
    if (bad) atomicOr((unsigned long long *)&flags[F_NET_ERR], 1ull);
}

__global__ void k_dense_supplies(const int64_t *am, const int64_t *bm, int64_t k, int64_t abar, int64_t bbar,
                                 int64_t *sup) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k + 2; i += (int64_t)gridDim.x * blockDim.x)
        sup[i] = i < k ? am[i] - bm[i] : (i == k ? abar : bbar);
}

}  // namespace

int corpus_load(Ctx &c, const double *pts, const int64_t *offsets, int64_t n) {
    if (n < 0 || !offsets) {
        set_error("corpus: bad arguments");
        return W1G_EINVAL;
    }
    if (offsets[0] != 0) {
        set_error("corpus: offsets must start at 0");
        return W1G_EINVAL;
    }
    for (int64_t i = 0; i < n; i++)
        if (offsets[i + 1] < offsets[i]) {
            set_error("corpus: offsets must be nondecreasing");
            return W1G_EINVAL;
        }
    const int64_t total = offsets[n];
    double2 *d;
    int64_t *doff;
    W1G_TRY(ensure(c.corpus_pts, (size_t)total + 1, &d));
    W1G_TRY(ensure(c.dense_scr[3], (size_t)n + 2, &doff));
    if (total) W1G_CUDA(cudaMemcpyAsync(d, pts, sizeof(double2) * total, cudaMemcpyHostToDevice, c.stream));
    W1G_CUDA(cudaMemcpyAsync(doff, offsets, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, c.stream));
    delete[] c.h_corpus_off;
    delete[] c.h_corpus_ptr;
    c.h_corpus_ptr = nullptr;
    c.h_corpus_off = new int64_t[n + 1];
    memcpy(c.h_corpus_off, offsets, sizeof(int64_t) * (n + 1));
    c.corpus_n = n;
    W1G_TRY(stream_sync(c));
    return W1G_OK;
}

int corpus_set_host(Ctx &c, const double *const *pts, const int64_t *sizes, int64_t n) {
    if (n < 0 || (n && (!pts || !sizes))) {
        set_error("corpus: bad arguments");
        return W1G_EINVAL;
    }
    delete[] c.h_corpus_off;
    delete[] c.h_corpus_ptr;
    c.h_corpus_off = new int64_t[n + 1];
    c.h_corpus_ptr = new const double *[n + 1];
    c.h_corpus_off[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        if (sizes[i] < 0) {
            set_error("corpus: negative diagram size");
            c.corpus_n = -1;
            return W1G_EINVAL;
        }
        c.h_corpus_ptr[i] = pts[i];
        c.h_corpus_off[i + 1] = c.h_corpus_off[i] + sizes[i];
    }
    c.corpus_n = n;
    return W1G_OK;
}

static int check_candidates(Ctx &c, const int64_t *cand, int64_t ncand) {
    if (c.corpus_n >= 0 && c.h_corpus_ptr) {
        set_error("the corpus is host-resident (w1g_corpus_set_host); scoring needs w1g_corpus_load");
        return W1G_ESTATE;
    }
    if (c.corpus_n < 0) {
        set_error("no corpus loaded (w1g_corpus_load)");
        return W1G_ESTATE;
    }
    for (int64_t i = 0; i < ncand; i++)
        if (cand[i] < 0 || cand[i] >= c.corpus_n) {
            set_error("candidate %lld out of range [0, %lld)", (long long)cand[i], (long long)c.corpus_n);
            return W1G_EINVAL;
        }
    return W1G_OK;
}

static int upload_query(Ctx &c, const double *query, int64_t nq, double2 **dq) {
    W1G_TRY(ensure(c.query_pts, (size_t)nq + 1, dq));
    if (nq) W1G_CUDA(cudaMemcpyAsync(*dq, query, sizeof(double2) * nq, cudaMemcpyHostToDevice, c.stream));
    return W1G_OK;
}

int wcd_corpus(Ctx &c, const double *query, int64_t nq, const int64_t *cand, int64_t ncand, double *scores) {
    W1G_TRY(check_candidates(c, cand, ncand));
    if (ncand == 0) return W1G_OK;
    double2 *dq;
    W1G_TRY(upload_query(c, query, nq, &dq));
    int64_t *dc;
    double *dout;
    W1G_TRY(ensure(c.dense_scr[0], (size_t)ncand, &dc));
    W1G_TRY(ensure(c.dense_scr[1], (size_t)ncand, &dout));
    W1G_CUDA(cudaMemcpyAsync(dc, cand, sizeof(int64_t) * ncand, cudaMemcpyHostToDevice, c.stream));
    const int64_t threads = 4 * ncand;
    k_wcd<<<grid_for(threads, 128), 128, 0, c.stream>>>(dq, nq, ptr<double2>(c.corpus_pts),
                                                        ptr<int64_t>(c.dense_scr[3]), dc, ncand, dout);
    W1G_CHECK_LAUNCH();
    W1G_CUDA(cudaMemcpyAsync(scores, dout, sizeof(double) * ncand, cudaMemcpyDeviceToHost, c.stream));
    W1G_TRY(stream_sync(c));
    return W1G_OK;
}

int rwmd_corpus(Ctx &c, const double *query, int64_t nq, const int64_t *cand, int64_t ncand, double *scores) {
    W1G_TRY(check_candidates(c, cand, ncand));
    double2 *dq;
    W1G_TRY(upload_query(c, query, nq, &dq));
    const double2 *corpus = ptr<double2>(c.corpus_pts);
    for (int64_t i = 0; i < ncand; i++) {
        const int64_t id = cand[i];
        const int64_t o = c.h_corpus_off[id], nc = c.h_corpus_off[id + 1] - o;
        int64_t k0 = 0;
        int32_t bal = 0;
        // rwmd(zero_condense(query, candidate)), pipeline.py:202-203
        W1G_TRY(zc_run(c, dq, nq, corpus + o, nc, &k0, &bal));
        double L = 0.0, la, lb;
        if (k0 > 0) W1G_TRY(rwmd_run(c, &L, &la, &lb));
        scores[i] = L;
    }
    c.tree_valid = c.pairs_valid = c.arcs_valid = c.net_valid = false;
    c.pre_n = 0;
    return W1G_OK;
}

int dense_network_run(Ctx &c, int64_t *node_count, int64_t *n_arcs) {
    NodeSet &ns = c.nodes[0];
    const int64_t k = ns.k;
    c.net_valid = false;
    c.net_check_pending = false;
    c.net_early_copy = false;
    const int64_t *am = ptr<int64_t>(ns.am), *bm = ptr<int64_t>(ns.bm);
    int64_t *apos, *bpos, *sup, *ro;
    int32_t *aidx, *bidx;
    W1G_TRY(ensure(c.dense_scr[0], (size_t)k + 1, &apos));
    W1G_TRY(ensure(c.dense_scr[1], (size_t)k + 1, &bpos));
    W1G_TRY(ensure(c.dense_scr[2], (size_t)2 * k + 2, &aidx));
    bidx = aidx + k + 1;
    W1G_TRY(ensure(c.net_sup, (size_t)k + 2, &sup));
    W1G_TRY(ensure(c.net_ro, (size_t)k + 3, &ro));
    W1G_TRY(flags_reset(c));
    int64_t *f = dflags(c);
    W1G_TRY(scan_i64(c, MemberFlag{am}, k, apos, f + F_MISC0));
    W1G_TRY(scan_i64(c, MemberFlag{bm}, k, bpos, f + F_MISC1));
    if (k) {
        k_compact_members<<<grid_for(k, 256, 8u * c.sm_count), 256, 0, c.stream>>>(am, bm, k, apos, bpos, aidx, bidx);
        W1G_CHECK_LAUNCH();
    } else {
        W1G_CUDA(cudaMemsetAsync(f + F_MISC0, 0, 2 * sizeof(int64_t), c.stream));
    }
    // row offsets: exclusive scan of the k + 2 row lengths, total into F_TOTAL
    W1G_TRY(scan_i64(c, DenseRowLen{am, bm, f + F_MISC1, k}, k + 2, ro, f + F_TOTAL));
    W1G_CUDA(cudaMemcpyAsync(ro + k + 2, f + F_TOTAL, sizeof(int64_t), cudaMemcpyDeviceToDevice, c.stream));
    k_dense_supplies<<<grid_for(k + 2, 256, 8u * c.sm_count), 256, 0, c.stream>>>(am, bm, k, ns.abar, ns.bbar, sup);
    W1G_CHECK_LAUNCH();
    W1G_TRY(flags_fetch(c, 0, F_NSLOTS - 8));
    const int64_t na = c.h_pinned[F_MISC0], nb = c.h_pinned[F_MISC1], m = c.h_pinned[F_TOTAL];
    int64_t *t, *h;
    double *cs;
    W1G_TRY(ensure(c.net_t, (size_t)m + 1, &t));
    W1G_TRY(ensure(c.net_h, (size_t)m + 1, &h));
    W1G_TRY(ensure(c.net_c, (size_t)m + 1, &cs));
    const unsigned g = (unsigned)(na + 1 < 16 * c.sm_count ? na + 1 : 16 * c.sm_count);
    k_dense_rows<<<g, 256, 0, c.stream>>>(ptr<double2>(ns.pts), bm, aidx, na, bidx, nb, k, ro, t, h, cs, f);
    W1G_CHECK_LAUNCH();
    W1G_TRY(flags_fetch(c, F_NET_ERR, 1));
    if (c.h_pinned[F_NET_ERR]) {
        set_error("non-finite arc cost");
        return W1G_ENETWORK;
    }
    c.net_n = k + 2;
    c.net_m = m;
    c.net_valid = true;
    *node_count = k + 2;
    *n_arcs = m;
    return W1G_OK;
}

}  // namespace w1g
