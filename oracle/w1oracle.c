/*
 * w1oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain scalar C restatement of the reference sparsify front-end of
 * w1flow (arXiv 2110.14734, /root/reference/pkg/src/w1flow).  It is the
 * checker the GPU path is compared against (tests/, __graft_entry__.smoke)
 * and the CPU baseline timed by bench.py (cpu_baseline, kind "port").
 * Nothing in paper_2110_14734_b200/ may link, import or call this file.
 *
 * Every function cites the reference lines it restates.  Arithmetic is
 * IEEE binary64 with no contraction (built with -ffp-contract=off), so the
 * results are bit-identical to the reference's numpy / scipy / numba
 * primitives (see SURVEY.md section 8c for the per-primitive evidence, and
 * tests/test_oracle_vs_reference.py / tests/golden for the pinning).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_EDUPLICATE (-2)
#define ORC_EOVERFLOW (-3)
#define ORC_ENOMEM (-4)
#define ORC_ECOUNT (-5)
/* build_network validation codes, network.py:56-68 */
#define ORC_NET_UNBALANCED (-10)
#define ORC_NET_RANGE (-11)
#define ORC_NET_SELFLOOP (-12)
#define ORC_NET_NONFINITE (-13)
#define ORC_NET_NEGATIVE (-14)

static const double ORC_SQRT2 = 1.4142135623730951; /* math.sqrt(2.0), diagram.py:17 */

/* ------------------------------------------------------------------ */
/* numpy pairwise summation of a contiguous float64 vector (np.sum),     */
/* used by lower_bound.py:58.  numpy/_core/src/umath/loops_utils.h.src   */
/* ------------------------------------------------------------------ */
static double pairwise_sum(const double *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

double orc_pairwise_sum(const double *a, int64_t n) { return pairwise_sum(a, n); }

/* ------------------------------------------------------------------ */
/* a1: zero_condense, diagram.py:190-208                                 */
/* np.unique(vstack(A,B), axis=0): lexicographic (x, then y) float order */
/* (-0.0 == +0.0), first element of each equal run kept.                 */
/* ------------------------------------------------------------------ */
typedef struct { double x, y; int64_t idx; } pt_rec;

static int cmp_pt(const void *pa, const void *pb)
{
    const pt_rec *a = (const pt_rec *)pa, *b = (const pt_rec *)pb;
    if (a->x < b->x) return -1;
    if (a->x > b->x) return 1;
    if (a->y < b->y) return -1;
    if (a->y > b->y) return 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

/* out arrays sized na+nb; returns K0 (>= 0) or a negative code */
int64_t orc_zero_condense(const double *a, int64_t na, const double *b, int64_t nb,
                          double *pts, int64_t *am, int64_t *bm)
{
    int64_t n = na + nb;
    if (n == 0) return 0;
    pt_rec *r = (pt_rec *)malloc(sizeof(pt_rec) * (size_t)n);
    if (!r) return ORC_ENOMEM;
    for (int64_t i = 0; i < na; i++) { r[i].x = a[2 * i]; r[i].y = a[2 * i + 1]; r[i].idx = i; }
    for (int64_t i = 0; i < nb; i++) { r[na + i].x = b[2 * i]; r[na + i].y = b[2 * i + 1]; r[na + i].idx = na + i; }
    qsort(r, (size_t)n, sizeof(pt_rec), cmp_pt);
    int64_t k = -1;
    for (int64_t i = 0; i < n; i++) {
        if (i == 0 || !(r[i].x == r[i - 1].x && r[i].y == r[i - 1].y)) {
            k++;
            pts[2 * k] = r[i].x;
            pts[2 * k + 1] = r[i].y;
            am[k] = 0;
            bm[k] = 0;
        }
        if (r[i].idx < na) am[k]++; else bm[k]++;
    }
    free(r);
    return k + 1;
}

/* ------------------------------------------------------------------ */
/* a3: rwmd, lower_bound.py:43-75.  Exact Euclidean NN distance         */
/* sqrt(fl(dx*dx) + fl(dy*dy)) -- what cKDTree.query returns -- via a   */
/* kd-tree over the targets.  Pruning is exact: a far-side point has    */
/* fl(dx*dx) >= fl(plane*plane) by monotone rounding, so a subtree is   */
/* skipped only when none of its points can beat the current minimum.   */
/* ------------------------------------------------------------------ */
#define KD_LEAF 8
typedef struct { int64_t lo, hi; int axis; double split; int64_t child; } kd_node; /* child -1 for a leaf */
typedef struct { double *x, *y; kd_node *nodes; int64_t n_nodes; } kdtree_t;

static void kd_select(double *x, double *y, int64_t lo, int64_t hi, int64_t k, int axis)
{
    /* quickselect on (axis coordinate) so that element k is in sorted position */
    double *c = axis ? y : x;
    while (hi - lo > 1) {
        double pv = c[lo + (hi - lo) / 2];
        int64_t i = lo, j = hi - 1;
        while (i <= j) {
            while (c[i] < pv) i++;
            while (c[j] > pv) j--;
            if (i <= j) {
                double t = x[i]; x[i] = x[j]; x[j] = t;
                t = y[i]; y[i] = y[j]; y[j] = t;
                i++; j--;
            }
        }
        if (k <= j) hi = j + 1;
        else if (k >= i) lo = i;
        else return;
    }
}

static int64_t kd_build(kdtree_t *t, int64_t lo, int64_t hi)
{
    int64_t id = t->n_nodes++;
    kd_node *nd = &t->nodes[id];
    nd->lo = lo; nd->hi = hi; nd->child = -1;
    if (hi - lo <= KD_LEAF) return id;
    double xmin = t->x[lo], xmax = xmin, ymin = t->y[lo], ymax = ymin;
    for (int64_t i = lo + 1; i < hi; i++) {
        if (t->x[i] < xmin) xmin = t->x[i];
        if (t->x[i] > xmax) xmax = t->x[i];
        if (t->y[i] < ymin) ymin = t->y[i];
        if (t->y[i] > ymax) ymax = t->y[i];
    }
    int axis = (xmax - xmin) >= (ymax - ymin) ? 0 : 1;
    int64_t mid = lo + (hi - lo) / 2;
    kd_select(t->x, t->y, lo, hi, mid, axis);
    double sp = axis ? t->y[mid] : t->x[mid];
    /* left = [lo, mid) all <= sp, right = [mid, hi) all >= sp */
    int64_t l = kd_build(t, lo, mid);
    int64_t r = kd_build(t, mid, hi);
    t->nodes[id].axis = axis;
    t->nodes[id].split = sp;
    t->nodes[id].child = l | (r << 32); /* left id in the low word, right id in the high word */
    return id;
}

static int kd_init(kdtree_t *t, const double *xs, const double *ys, int64_t m)
{
    t->x = (double *)malloc(sizeof(double) * (size_t)m);
    t->y = (double *)malloc(sizeof(double) * (size_t)m);
    t->nodes = (kd_node *)malloc(sizeof(kd_node) * (size_t)(2 * (m / (KD_LEAF / 2) + 2)));
    if (!t->x || !t->y || !t->nodes) return ORC_ENOMEM;
    memcpy(t->x, xs, sizeof(double) * (size_t)m);
    memcpy(t->y, ys, sizeof(double) * (size_t)m);
    t->n_nodes = 0;
    kd_build(t, 0, m);
    return ORC_OK;
}

static void kd_free(kdtree_t *t) { free(t->x); free(t->y); free(t->nodes); }

/* exact min over targets of fl(fl(dx*dx)+fl(dy*dy)) */
static double kd_nn_d2(const kdtree_t *t, double qx, double qy)
{
    int64_t stack[256];
    int top = 0;
    double best = INFINITY;
    stack[top++] = 0;
    while (top > 0) {
        const kd_node *nd = &t->nodes[stack[--top]];
        if (nd->child < 0) {
            for (int64_t i = nd->lo; i < nd->hi; i++) {
                double dx = qx - t->x[i], dy = qy - t->y[i];
                double d2 = dx * dx + dy * dy;
                if (d2 < best) best = d2;
            }
            continue;
        }
        int64_t l = nd->child & 0xFFFFFFFF, r = nd->child >> 32;
        double q = nd->axis ? qy : qx;
        double pd = q - nd->split;
        double pd2 = pd * pd;
        int64_t near = pd <= 0 ? l : r, far = pd <= 0 ? r : l;
        if (pd2 < best) stack[top++] = far; /* far side: every fl(d2) >= pd2 */
        stack[top++] = near;
    }
    return best;
}

/* _one_sided, lower_bound.py:43-58 */
static double one_sided(const double *pts, const int64_t *smass, const int64_t *dmass, int64_t K, int *err)
{
    int64_t ns = 0, nd = 0;
    for (int64_t i = 0; i < K; i++) { ns += smass[i] > 0; nd += dmass[i] > 0; }
    if (ns == 0) return 0.0;
    double *terms = (double *)malloc(sizeof(double) * (size_t)ns);
    double *dx = NULL, *dy = NULL;
    kdtree_t g;
    memset(&g, 0, sizeof g);
    if (!terms) { *err = ORC_ENOMEM; return 0.0; }
    if (nd > 0) {
        dx = (double *)malloc(sizeof(double) * (size_t)nd);
        dy = (double *)malloc(sizeof(double) * (size_t)nd);
        int64_t j = 0;
        for (int64_t i = 0; i < K; i++)
            if (dmass[i] > 0) { dx[j] = pts[2 * i]; dy[j] = pts[2 * i + 1]; j++; }
        if (kd_init(&g, dx, dy, nd) != ORC_OK) { *err = ORC_ENOMEM; return 0.0; }
    }
    int64_t j = 0;
    for (int64_t i = 0; i < K; i++) {
        if (smass[i] <= 0) continue;
        double x = pts[2 * i], y = pts[2 * i + 1];
        double diag = fabs(y - x) / ORC_SQRT2;          /* diagram.py:47 */
        double best = diag;
        if (nd > 0) {
            double nnd = sqrt(kd_nn_d2(&g, x, y));
            best = nnd < diag ? nnd : diag;             /* np.minimum(nnd, diag) */
        }
        terms[j++] = (double)smass[i] * best;           /* src_mass * best */
    }
    double s = pairwise_sum(terms, ns);
    free(terms);
    if (nd > 0) { kd_free(&g); free(dx); free(dy); }
    return s;
}

/* rwmd, lower_bound.py:61-75 */
double orc_rwmd(const double *pts, const int64_t *am, const int64_t *bm, int64_t K,
                double *la_out, double *lb_out)
{
    int err = 0;
    double la = one_sided(pts, am, bm, K, &err);
    double lb = one_sided(pts, bm, am, K, &err);
    if (la_out) *la_out = la;
    if (lb_out) *lb_out = lb;
    return la >= lb ? la : lb; /* python max(l_a, l_b) */
}

/* per-source best distance (for kernel-level parity tests) */
int64_t orc_rwmd_best(const double *pts, const int64_t *smass, const int64_t *dmass, int64_t K, double *best_out)
{
    int64_t nd = 0;
    for (int64_t i = 0; i < K; i++) nd += dmass[i] > 0;
    double *dx = NULL, *dy = NULL;
    kdtree_t g;
    memset(&g, 0, sizeof g);
    if (nd > 0) {
        dx = (double *)malloc(sizeof(double) * (size_t)nd);
        dy = (double *)malloc(sizeof(double) * (size_t)nd);
        int64_t j = 0;
        for (int64_t i = 0; i < K; i++)
            if (dmass[i] > 0) { dx[j] = pts[2 * i]; dy[j] = pts[2 * i + 1]; j++; }
        if (kd_init(&g, dx, dy, nd) != ORC_OK) return ORC_ENOMEM;
    }
    int64_t j = 0;
    for (int64_t i = 0; i < K; i++) {
        if (smass[i] <= 0) continue;
        double x = pts[2 * i], y = pts[2 * i + 1];
        double diag = fabs(y - x) / ORC_SQRT2, best = diag;
        if (nd > 0) {
            double nnd = sqrt(kd_nn_d2(&g, x, y));
            best = nnd < diag ? nnd : diag;
        }
        best_out[j++] = best;
    }
    if (nd > 0) { kd_free(&g); free(dx); free(dy); }
    return j;
}

/* ------------------------------------------------------------------ */
/* a5/a6: snap_points + delta_condense, condensation.py:62-124           */
/* ------------------------------------------------------------------ */
static inline uint64_t splitmix64(uint64_t x) /* condensation.py:85-89 */
{
    x = x + 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

typedef struct { int64_t cx, cy; int64_t idx; } cell_rec;

static int cmp_cell(const void *pa, const void *pb)
{
    const cell_rec *a = (const cell_rec *)pa, *b = (const cell_rec *)pb;
    if (a->cx != b->cx) return a->cx < b->cx ? -1 : 1;
    if (a->cy != b->cy) return a->cy < b->cy ? -1 : 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

/* _round_half_away, condensation.py:62-63: sign(t) * floor(abs(t) + 0.5) */
static inline double round_half_away(double t)
{
    double sg = (t > 0.0) ? 1.0 : ((t < 0.0) ? -1.0 : t); /* np.sign keeps +-0 */
    return sg * floor(fabs(t) + 0.5);
}

/* cells sized 2*K (int64): snap_points, condensation.py:66-77 */
int orc_snap_cells(const double *pts, int64_t K, double pitch, int64_t *cells)
{
    double amax = 0.0;
    for (int64_t i = 0; i < 2 * K; i++) {
        double c = round_half_away(pts[i] / pitch);
        double a = fabs(c);
        if (a > amax || a != a) amax = a;
        cells[i] = (int64_t)c;
    }
    if (K > 0 && !(amax < 4611686018427387904.0)) return ORC_EOVERFLOW; /* >= 2**62 */
    return ORC_OK;
}

/* returns K' or a negative code; outputs sized K */
int64_t orc_delta_condense(const double *pts, const int64_t *am, const int64_t *bm, int64_t K,
                           double pitch, double half_width, uint64_t seed,
                           double *opts, int64_t *oam, int64_t *obm)
{
    if (K == 0) return 0;
    int64_t *cells = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)K);
    cell_rec *r = (cell_rec *)malloc(sizeof(cell_rec) * (size_t)K);
    if (!cells || !r) return ORC_ENOMEM;
    int rc = orc_snap_cells(pts, K, pitch, cells);
    if (rc != ORC_OK) { free(cells); free(r); return rc; }
    for (int64_t i = 0; i < K; i++) { r[i].cx = cells[2 * i]; r[i].cy = cells[2 * i + 1]; r[i].idx = i; }
    qsort(r, (size_t)K, sizeof(cell_rec), cmp_cell);
    uint64_t base = splitmix64(seed);
    int64_t k = -1;
    for (int64_t i = 0; i < K; i++) {
        if (i == 0 || r[i].cx != r[i - 1].cx || r[i].cy != r[i - 1].cy) {
            k++;
            oam[k] = 0;
            obm[k] = 0;
            /* _lattice_offsets, condensation.py:92-102 */
            uint64_t h1 = splitmix64(base ^ (uint64_t)r[i].cx);
            uint64_t h2 = splitmix64(h1 ^ (uint64_t)r[i].cy);
            uint64_t h3 = splitmix64(h2);
            double u1 = (double)(h2 >> 11) * 0x1p-53;
            double u2 = (double)(h3 >> 11) * 0x1p-53;
            double o1 = half_width * (2.0 * u1 - 1.0);
            double o2 = half_width * (2.0 * u2 - 1.0);
            /* coords = cell.astype(f64) * (k*delta) + offsets, condensation.py:123 */
            opts[2 * k] = (double)r[i].cx * pitch + o1;
            opts[2 * k + 1] = (double)r[i].cy * pitch + o2;
        }
        oam[k] += am[r[i].idx];
        obm[k] += bm[r[i].idx];
    }
    free(cells);
    free(r);
    return k + 1;
}

/* ------------------------------------------------------------------ */
/* a7: build_split_tree, spanner.py:96-159                               */
/* ------------------------------------------------------------------ */
typedef struct { int64_t lo, hi, parent; int is_right; } frame_t;

int orc_split_tree(const double *pts, int64_t n, int64_t *left, int64_t *right,
                   double *bbox, int64_t *rep, int64_t *size)
{
    if (n == 0) return ORC_OK;
    int64_t n_nodes = 2 * n - 1;
    for (int64_t i = 0; i < n_nodes; i++) { left[i] = -1; right[i] = -1; rep[i] = -1; size[i] = 0; }
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *tmp = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    frame_t *stack = (frame_t *)malloc(sizeof(frame_t) * (size_t)(n_nodes + 2));
    if (!order || !tmp || !stack) return ORC_ENOMEM;
    for (int64_t i = 0; i < n; i++) order[i] = i;
    int64_t top = 0, next_id = 0;
    stack[top++] = (frame_t){0, n, -1, 0};
    int rc = ORC_OK;
    while (top > 0) {
        frame_t f = stack[--top];
        int64_t nid = next_id++;
        if (f.parent >= 0) {
            if (f.is_right) right[f.parent] = nid; else left[f.parent] = nid;
        }
        double xmin = INFINITY, ymin = INFINITY, xmax = -INFINITY, ymax = -INFINITY;
        for (int64_t p = f.lo; p < f.hi; p++) {
            double x = pts[2 * order[p]], y = pts[2 * order[p] + 1];
            /* numpy min/max reductions; order-insensitive for non-NaN */
            if (x < xmin) xmin = x;
            if (x > xmax) xmax = x;
            if (y < ymin) ymin = y;
            if (y > ymax) ymax = y;
        }
        double *bb = bbox + 4 * nid;
        bb[0] = xmin; bb[1] = ymin; bb[2] = xmax; bb[3] = ymax;
        size[nid] = f.hi - f.lo;
        if (f.hi - f.lo == 1) { rep[nid] = order[f.lo]; continue; }
        double ext_x = bb[2] - bb[0], ext_y = bb[3] - bb[1];
        if (ext_x == 0.0 && ext_y == 0.0) { rc = ORC_EDUPLICATE; break; }
        int axis = ext_x >= ext_y ? 0 : 1;
        double mid = 0.5 * (bb[axis] + bb[axis + 2]);
        int64_t n_left = 0;
        for (int64_t p = f.lo; p < f.hi; p++) n_left += pts[2 * order[p] + axis] <= mid;
        int strict = 0;
        if (n_left == 0 || n_left == f.hi - f.lo) {
            strict = 1; /* spanner.py:139-144 */
            n_left = 0;
            for (int64_t p = f.lo; p < f.hi; p++) n_left += pts[2 * order[p] + axis] < bb[axis + 2];
        }
        int64_t a = 0, b2 = n_left;
        for (int64_t p = f.lo; p < f.hi; p++) {
            double c = pts[2 * order[p] + axis];
            int in_left = strict ? (c < bb[axis + 2]) : (c <= mid);
            if (in_left) tmp[a++] = order[p]; else tmp[b2++] = order[p];
        }
        memcpy(order + f.lo, tmp, sizeof(int64_t) * (size_t)(f.hi - f.lo));
        stack[top++] = (frame_t){f.lo + n_left, f.hi, nid, 1};
        stack[top++] = (frame_t){f.lo, f.lo + n_left, nid, 0};
    }
    if (rc == ORC_OK) {
        for (int64_t nid = n_nodes - 1; nid >= 0; nid--) {
            if (left[nid] < 0) continue;
            int64_t ri = rep[left[nid]], rj = rep[right[nid]];
            double pi0 = pts[2 * ri], pi1 = pts[2 * ri + 1], pj0 = pts[2 * rj], pj1 = pts[2 * rj + 1];
            int le; /* python tuple (pi0, pi1) <= (pj0, pj1) */
            if (pi0 != pj0) le = pi0 <= pj0;
            else if (pi1 != pj1) le = pi1 <= pj1;
            else le = 1;
            rep[nid] = le ? ri : rj;
        }
    }
    free(order);
    free(tmp);
    free(stack);
    return rc;
}

/* ------------------------------------------------------------------ */
/* a8/a9: _ws_predicate, _diag_sq, _pairs_kernel, spanner.py:176-242     */
/* ------------------------------------------------------------------ */
static inline int ws_predicate(const double *bbox, int64_t u, int64_t v, double s)
{
    const double *bu = bbox + 4 * u, *bv = bbox + 4 * v;
    double rux = bu[2] - bu[0], ruy = bu[3] - bu[1];
    double rvx = bv[2] - bv[0], rvy = bv[3] - bv[1];
    double ru = 0.5 * sqrt(rux * rux + ruy * ruy);
    double rv = 0.5 * sqrt(rvx * rvx + rvy * rvy);
    double r = ru > rv ? ru : rv;
    double dx = 0.5 * (bu[0] + bu[2]) - 0.5 * (bv[0] + bv[2]);
    double dy = 0.5 * (bu[1] + bu[3]) - 0.5 * (bv[1] + bv[3]);
    return sqrt(dx * dx + dy * dy) - 2.0 * r >= s * r;
}

static inline double diag_sq(const double *bbox, int64_t u)
{
    double w = bbox[4 * u + 2] - bbox[4 * u], h = bbox[4 * u + 3] - bbox[4 * u + 1];
    return w * w + h * h;
}

/* counts sized n_nodes (0 for leaves); offsets (if write) per node; pairs (P,2) */
static int pairs_kernel(const int64_t *left, const int64_t *right, const double *bbox, int64_t n_nodes,
                        double s, int64_t *counts, const int64_t *offsets, int64_t *out, int write)
{
    int64_t *stack = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)(2 * n_nodes + 8));
    if (!stack) return ORC_ENOMEM;
    for (int64_t w = 0; w < n_nodes; w++) {
        if (left[w] < 0) { if (!write) counts[w] = 0; continue; }
        int64_t found = 0, pos = write ? offsets[w] : 0, top = 0;
        stack[0] = left[w]; stack[1] = right[w]; top = 1;
        while (top > 0) {
            top--;
            int64_t u = stack[2 * top], v = stack[2 * top + 1];
            if (ws_predicate(bbox, u, v, s)) {
                if (write) { out[2 * pos] = u; out[2 * pos + 1] = v; pos++; }
                else found++;
                continue;
            }
            if (diag_sq(bbox, u) > diag_sq(bbox, v)) {
                stack[2 * top] = left[u]; stack[2 * top + 1] = v;
                stack[2 * top + 2] = right[u]; stack[2 * top + 3] = v;
            } else {
                stack[2 * top] = u; stack[2 * top + 1] = left[v];
                stack[2 * top + 2] = u; stack[2 * top + 3] = right[v];
            }
            top += 2;
        }
        if (write) {
            if (pos != offsets[w] + counts[w]) { free(stack); return ORC_ECOUNT; }
        } else counts[w] = found;
    }
    free(stack);
    return ORC_OK;
}

int64_t orc_wspd_count(const int64_t *left, const int64_t *right, const double *bbox, int64_t n_nodes,
                       double s, int64_t *counts)
{
    int rc = pairs_kernel(left, right, bbox, n_nodes, s, counts, NULL, NULL, 0);
    if (rc != ORC_OK) return rc;
    int64_t t = 0;
    for (int64_t i = 0; i < n_nodes; i++) t += counts[i];
    return t;
}

/* writes pairs in reference order (owner ascending, DFS pop order) */
int orc_wspd_write(const int64_t *left, const int64_t *right, const double *bbox, int64_t n_nodes,
                   double s, const int64_t *counts, const int64_t *offsets, int64_t *pairs)
{
    return pairs_kernel(left, right, bbox, n_nodes, s, (int64_t *)counts, offsets, pairs, 1);
}

/* ------------------------------------------------------------------ */
/* glibc 2.39 __hypot (sysdeps/ieee754/dbl-64/e_hypot.c), non-FMA build, */
/* restated; this is the arithmetic np.hypot performs in emit_arcs      */
/* (spanner.py:324).  orc_emit_arcs calls libm hypot() itself; this port */
/* exists to pin the transcription that the CUDA device function uses.  */
/* ------------------------------------------------------------------ */
static inline double hypot_kernel(double ax, double ay)
{
    double t1, t2;
    double h = sqrt(ax * ax + ay * ay);
    if (h <= 2.0 * ay) {
        double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}

double orc_hypot_port(double x, double y)
{
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return x + y;
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ax > 0x1p+511) {
        if (ay <= ax * 0x1p-54) return ax + ay;
        return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
    }
    if (ay < 0x1p-511) {
        if (ax >= ay / 0x1p-54) return ax + ay;
        ax = hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
        return ax;
    }
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax, ay);
}

double orc_hypot_libm(double x, double y) { return hypot(x, y); }

/* ------------------------------------------------------------------ */
/* a10: emit_arcs, spanner.py:310-337.  Arc order as the reference:      */
/* [pi->pj]*P, [pj->pi]*P, [a_i->abar], [bbar->b_i], [bbar->abar]        */
/* ------------------------------------------------------------------ */
int64_t orc_emit_arcs(const int64_t *indices, int64_t P, const double *pts, const int64_t *am,
                      const int64_t *bm, int64_t K, int64_t *tails, int64_t *heads, double *costs)
{
    int64_t abar = K, bbar = K + 1, m = 0;
    for (int64_t p = 0; p < P; p++) {
        int64_t i = indices[2 * p], j = indices[2 * p + 1];
        double c = hypot(pts[2 * i] - pts[2 * j], pts[2 * i + 1] - pts[2 * j + 1]);
        tails[p] = i; heads[p] = j; costs[p] = c;
        tails[P + p] = j; heads[P + p] = i; costs[P + p] = c;
    }
    m = 2 * P;
    for (int64_t i = 0; i < K; i++)
        if (am[i] > 0) { tails[m] = i; heads[m] = abar; costs[m] = fabs(pts[2 * i + 1] - pts[2 * i]) / ORC_SQRT2; m++; }
    for (int64_t i = 0; i < K; i++)
        if (bm[i] > 0) { tails[m] = bbar; heads[m] = i; costs[m] = fabs(pts[2 * i + 1] - pts[2 * i]) / ORC_SQRT2; m++; }
    tails[m] = bbar; heads[m] = abar; costs[m] = 0.0; m++;
    return m;
}

/* ------------------------------------------------------------------ */
/* a11: build_network, network.py:44-85                                  */
/* ------------------------------------------------------------------ */
typedef struct { int64_t t, h, idx; } arc_rec;

static int cmp_arc(const void *pa, const void *pb)
{
    const arc_rec *a = (const arc_rec *)pa, *b = (const arc_rec *)pb;
    if (a->t != b->t) return a->t < b->t ? -1 : 1;
    if (a->h != b->h) return a->h < b->h ? -1 : 1;
    return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

/* returns the deduplicated arc count or a negative validation code */
int64_t orc_build_network(int64_t n, const int64_t *supplies, const int64_t *tails, const int64_t *heads,
                          const double *costs, int64_t m, int64_t *ot, int64_t *oh, double *oc,
                          int64_t *row_offsets)
{
    int64_t tot = 0;
    for (int64_t i = 0; i < n; i++) tot += supplies[i];
    if (tot != 0) return ORC_NET_UNBALANCED;
    for (int64_t e = 0; e < m; e++)
        if (tails[e] < 0 || tails[e] >= n || heads[e] < 0 || heads[e] >= n) return ORC_NET_RANGE;
    for (int64_t e = 0; e < m; e++)
        if (tails[e] == heads[e]) return ORC_NET_SELFLOOP;
    for (int64_t e = 0; e < m; e++)
        if (!isfinite(costs[e])) return ORC_NET_NONFINITE;
    for (int64_t e = 0; e < m; e++)
        if (costs[e] < 0) return ORC_NET_NEGATIVE;
    arc_rec *r = (arc_rec *)malloc(sizeof(arc_rec) * (size_t)(m > 0 ? m : 1));
    if (!r) return ORC_ENOMEM;
    for (int64_t e = 0; e < m; e++) { r[e].t = tails[e]; r[e].h = heads[e]; r[e].idx = e; }
    qsort(r, (size_t)m, sizeof(arc_rec), cmp_arc);
    int64_t g = -1;
    for (int64_t e = 0; e < m; e++) {
        double c = costs[r[e].idx];
        if (e == 0 || r[e].t != r[e - 1].t || r[e].h != r[e - 1].h) {
            g++;
            ot[g] = r[e].t; oh[g] = r[e].h; oc[g] = c;
        } else if (!(oc[g] < c)) {
            /* np.minimum(acc, c) keeps acc only when strictly smaller: among
               equal minima (+0.0 / -0.0) the later arc wins */
            oc[g] = c;
        }
    }
    int64_t mm = g + 1;
    for (int64_t i = 0; i <= n; i++) row_offsets[i] = 0;
    for (int64_t e = 0; e < mm; e++) row_offsets[ot[e] + 1]++;
    for (int64_t i = 0; i < n; i++) row_offsets[i + 1] += row_offsets[i];
    free(r);
    return mm;
}
