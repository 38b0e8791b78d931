/*
 * w1g.h -- C ABI of libw1g.so, the B200 (sm_100a) sparsify front-end of
 * PDoptFlow (arXiv 2110.14734).
 *
 * The reference (w1flow, /root/reference/pkg/src/w1flow) has no FFI layer:
 * its "operator API" is the set of module-level Python stage functions that
 * approx_w1 calls in order (pipeline.py:105-130).  Each entry point below
 * replaces one of them; the ctypes stub that binds them is
 * paper_2110_14734_b200/_lib.py.
 *
 * Conventions
 *  - every call returns W1G_OK (0) or a negative W1G_E* code; a message is
 *    kept per host thread (w1g_last_error);
 *  - one context = one device + one CUDA stream + device-resident stage
 *    state; a context is not thread-safe, use one host thread per context;
 *  - data-dependent outputs are two-phase: a stage call returns sizes, a
 *    w1g_fetch_* call copies into caller-owned host arrays of those sizes;
 *  - host arrays are C-contiguous: points (n,2) float64 as x0,y0,x1,y1,...;
 *    indices, masses, supplies int64; costs float64 (the reference dtypes).
 */
#ifndef W1G_H
#define W1G_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define W1G_OK 0
#define W1G_EINVAL (-1)     /* bad argument (maps to ValueError) */
#define W1G_ECUDA (-2)      /* CUDA runtime failure (RuntimeError) */
#define W1G_EOVERFLOW (-3)  /* lattice pitch too small, condensation.py:75-76 (ValueError) */
#define W1G_EDUPLICATE (-4) /* split tree duplicate points, spanner.py:134-135 (ValueError) */
#define W1G_ECOUNT (-5)     /* WSPD write pass != counted offsets, spanner.py:259-260 (AssertionError) */
#define W1G_ENETWORK (-6)   /* build_network validation, network.py:56-68 (NetworkError) */
#define W1G_ENOMEM (-7)     /* device allocation failed (MemoryError) */
#define W1G_ESTATE (-8)     /* stage called before its inputs exist (RuntimeError) */
#define W1G_DONE 1          /* w1g_batch_next: every result has been delivered */

/* node-set slots held by a context */
#define W1G_NODES0 0 /* output of zero_condense */
#define W1G_NODES 1  /* output of delta_condense (or nodes0 when delta == 0) */

typedef struct w1g_ctx w1g_ctx;

/* per-stage result of the fused front end (pipeline.py:98-132) */
typedef struct {
    int64_t n_points0;      /* K0: nodes after zero_condense */
    int64_t n_points;       /* K: nodes after delta_condense */
    int64_t n_tree_nodes;   /* 2K-1 */
    int64_t n_pairs;        /* WSPD pairs P */
    int64_t n_arcs;         /* network arcs M (after dedup) */
    int64_t node_count;     /* K + 2 */
    double lower_bound;     /* RWMD L = max(L_A, L_B) */
    double lower_bound_a;   /* L_A */
    double lower_bound_b;   /* L_B */
    double epsilon_condense;/* pipeline.py:67-69 */
    double delta;           /* lattice pitch parameter used (0 = no condensation) */
    int32_t short_circuit;  /* empty input or a_mass == b_mass (pipeline.py:106-109) */
    int32_t tree_depth;     /* split tree levels */
    int32_t n_levels_wspd;  /* WSPD frontier levels */
    int32_t network_copied; /* 1: the network was written to the w1g_set_network_out target */
    float stage_ms[8];      /* device time per stage: zc, rwmd, dc, tree, wspd, emit, csr, total */
} w1g_front_end_info;

int w1g_version(void);
/* page-locked host memory for zero-copy result arrays (cudaHostAlloc) */
int w1g_host_alloc(uint64_t bytes, void **out);
int w1g_host_free(void *p);
/* number of CUDA kernels this library has launched (process-wide) */
uint64_t w1g_launch_count(void);
/* measurement hook: time `reps` launches of the FP32 all-pairs RWMD tile
 * kernel (A->B then B->A, culling as configured) on the context's nodes0 with
 * CUDA events on the context stream; returns the mean device time per launch
 * and the directed (source, target) evaluations one launch covers */
int w1g_profile_rwmd_tile(w1g_ctx *ctx, int reps, float *ms_per_launch, int64_t *evals_per_launch);
/* measurement hook: the production RWMD (lower_bound.py:43-75 as w1g_rwmd runs it:
 * culled FP32 tile pass + exact fp64 refine per side) `reps` times on nodes0, with
 * CUDA events around each kernel on the stream it runs on and device counters of
 * the (source, target) distance evaluations each performs.  ms[4], evals[4]: mean
 * per launch for {A tile, A refine, B tile, B refine}; directed = 2 |A| |B| */
int w1g_profile_rwmd(w1g_ctx *ctx, int reps, float *ms, int64_t *evals, int64_t *directed);
/* test hook: stable device radix sort of host keys (`words` arrays of n
 * uint64, word 0 least significant); writes the sorting permutation */
int w1g_debug_radix_sort(w1g_ctx *ctx, const uint64_t *keys, int words, int64_t n, uint32_t *perm);
int w1g_device_count(int *count);
const char *w1g_last_error(void);

int w1g_ctx_create(int device, w1g_ctx **out);
int w1g_ctx_destroy(w1g_ctx *ctx);
/* the CUDA stream the context launches on (cudaStream_t), for event timing */
void *w1g_ctx_stream(w1g_ctx *ctx);
int w1g_synchronize(w1g_ctx *ctx);

/* replaces diagram.zero_condense, diagram.py:190-208 -> slot W1G_NODES0 */
int w1g_zero_condense(w1g_ctx *ctx, const double *a, int64_t na, const double *b, int64_t nb,
                      int64_t *k0, int32_t *balanced);
/* device-resident variant: a/b already in device memory (bench "value" leg) */
int w1g_zero_condense_device(w1g_ctx *ctx, const double *d_a, int64_t na, const double *d_b,
                             int64_t nb, int64_t *k0, int32_t *balanced);
/* upload an arbitrary SuppliedNodes (diagram.py:150-187) into a slot */
int w1g_load_nodes(w1g_ctx *ctx, int slot, const double *points, const int64_t *a_mass,
                   const int64_t *b_mass, int64_t k, int64_t abar_supply, int64_t bbar_supply);
int w1g_nodes_size(w1g_ctx *ctx, int slot, int64_t *k);
int w1g_fetch_nodes(w1g_ctx *ctx, int slot, double *points, int64_t *a_mass, int64_t *b_mass);

/* replaces lower_bound.rwmd, lower_bound.py:61-75, on slot W1G_NODES0 */
int w1g_rwmd(w1g_ctx *ctx, double *L, double *LA, double *LB);
/* per-source best distance min(nn, diag) for one side (0 = A, 1 = B), node order */
int w1g_fetch_rwmd_best(w1g_ctx *ctx, int side, double *best, int64_t *n);
/* row-sharded RWMD (one rank's share of lower_bound.py:43-58): the pairwise
 * sum of mass*best over side `side`'s members [begin, end) (node order), which
 * the host chooses as a subtree of numpy's summation tree so the ranks'
 * partial sums combine bit-exactly; also returns the side's member count */
int w1g_rwmd_range(w1g_ctx *ctx, int side, int64_t begin, int64_t end, double *partial,
                   int64_t *n_members);
/* RWMD of one pair with its rows sharded over G contexts (G devices of one process, or
 * several contexts of one device): every context must hold the same nodes0; the rows are
 * cut along numpy's pairwise-summation tree (subtree t -> context t % G), each context
 * sums its subtrees on its own device and host thread, and the host recombines them in
 * the tree's order -- bit-identical to w1g_rwmd */
int w1g_rwmd_sharded(w1g_ctx **ctxs, int G, double *L, double *LA, double *LB);
/* the A- and B-member counts of nodes0 (the row counts w1g_rwmd_range splits); free when
 * nodes0 came from zero_condense */
int w1g_member_counts(w1g_ctx *ctx, int64_t *n_a, int64_t *n_b);
/* tile culling in the FP32 all-pairs pass: 1 (default) or 0 (full brute force) */
int w1g_set_rwmd_culling(w1g_ctx *ctx, int enabled);

/* replaces condensation.delta_condense, condensation.py:105-124: NODES0 -> NODES.
 * pitch = k*delta, half_width = (1-k)*delta/2 as computed by the caller
 * (condensation.py:73,121); delta == 0 copies NODES0 to NODES. */
int w1g_delta_condense(w1g_ctx *ctx, double delta, double pitch, double half_width,
                       uint64_t seed, int64_t *k);

/* replaces condensation.snap_points, condensation.py:66-77: cells = round-half-away(p / pitch)
 * (int64, (n,2)), snapped = cells * pitch; W1G_EOVERFLOW when |cell| >= 2^62 */
int w1g_snap_points(w1g_ctx *ctx, const double *points, int64_t n, double pitch, double *snapped,
                    int64_t *cells);

/* replaces spanner.build_split_tree, spanner.py:96-159, over a slot's points */
int w1g_split_tree(w1g_ctx *ctx, int slot, int64_t *n_nodes, int32_t *depth);
int w1g_fetch_tree(w1g_ctx *ctx, int64_t *left, int64_t *right, double *bbox, int64_t *rep,
                   int64_t *size);
/* upload a SplitTree (spanner.py:37-64) for a standalone build_wspd */
int w1g_load_tree(w1g_ctx *ctx, const double *points, int64_t n_points, const int64_t *left,
                  const int64_t *right, const double *bbox, const int64_t *rep, int64_t n_nodes);

/* replaces spanner.build_wspd / count_pairs / write_pairs, spanner.py:263-307.
 * reference_order = 1 sorts pairs into the reference layout (owner ascending,
 * DFS pop order); 0 leaves them in frontier order (the fused path). */
int w1g_wspd(w1g_ctx *ctx, double s, int reference_order, int64_t *n_pairs);
int w1g_fetch_pairs(w1g_ctx *ctx, int64_t *node_pairs, int64_t *indices);
/* one GPU's share of a sharded WSPD (the owner loop of spanner.py:206-241
 * split over GPUs): the recursions of the internal nodes w with w % n_shards == shard, in
 * frontier order; the shards' pair sets partition the full WSPD */
int w1g_wspd_shard(w1g_ctx *ctx, double s, int shard, int n_shards, int64_t *n_pairs);
/* pairs per internal node, internal nodes in id order (count_pairs output) */
int w1g_fetch_pair_counts(w1g_ctx *ctx, int64_t *counts, int64_t *n_internal);
/* upload WSPairList.indices and .points (spanner.py:67-81) for a standalone emit_arcs */
int w1g_load_pairs(w1g_ctx *ctx, const int64_t *indices, int64_t n_pairs, const double *points,
                   int64_t n_points);

/* replaces spanner.emit_arcs, spanner.py:310-337, over slot W1G_NODES */
int w1g_emit_arcs(w1g_ctx *ctx, int64_t *n_arcs);
int w1g_fetch_arcs(w1g_ctx *ctx, int64_t *tails, int64_t *heads, double *costs);
/* the arcs of the context's pairs only (both directions, spanner.py:319-326), plus the
 * diagonal and free arcs when with_diagonal (:327-335): one shard's slice of emit_arcs */
int w1g_emit_pair_arcs(w1g_ctx *ctx, int with_diagonal, int64_t *n_arcs);
/* device pointers of the context's arc list (int64 tails, int64 heads, float64 costs): the
 * send buffers of the multi-GPU arc gather (valid until the next stage call) */
int w1g_arcs_device(w1g_ctx *ctx, void **tails, void **heads, void **costs, int64_t *m);
/* the WSPD node pairs (int2 (u, v) tree node ids) in device memory: the compact send
 * buffer of the multi-GPU gather (8 bytes per pair instead of two 24-byte arcs) */
int w1g_pairs_device(w1g_ctx *ctx, void **uv, int64_t *n_pairs);
/* adopt gathered node pairs (device memory) over this context's own split tree */
int w1g_load_pairs_device(w1g_ctx *ctx, const void *d_uv, int64_t n_pairs);
/* emit_arcs + assemble fused (the front end's network builder) from the context's
 * nodes, split tree and node pairs: the network of a sharded front end on rank 0 */
int w1g_network_from_pairs(w1g_ctx *ctx, int64_t *node_count, int64_t *n_arcs);
/* adopt an arc list already in this device's memory (the gathered slices), device to device */
int w1g_load_arcs_device(w1g_ctx *ctx, const int64_t *d_tails, const int64_t *d_heads, const double *d_costs,
                         int64_t m);
int w1g_load_arcs(w1g_ctx *ctx, const int64_t *tails, const int64_t *heads, const double *costs,
                  int64_t m);

/* replaces network.build_network, network.py:44-85, over the context's arcs */
int w1g_build_network(w1g_ctx *ctx, const int64_t *supplies, int64_t n, int64_t *n_arcs);
/* replaces network.assemble, network.py:88-93 (supplies from slot W1G_NODES) */
int w1g_assemble(w1g_ctx *ctx, int64_t *node_count, int64_t *n_arcs);
int w1g_fetch_network(w1g_ctx *ctx, int64_t *supplies, int64_t *tails, int64_t *heads,
                      double *costs, int64_t *row_offsets);
/* one-shot output target for the NEXT fused front end: when its network fits
 * (node_count <= node_cap, arcs <= arc_cap) it is copied there inside the call,
 * overlapping whatever device work is still running (info->network_copied = 1);
 * page-locked buffers (w1g_host_alloc) give full-speed copies */
int w1g_set_network_out(w1g_ctx *ctx, int64_t *supplies, int64_t *tails, int64_t *heads, double *costs,
                        int64_t *row_offsets, int64_t node_cap, int64_t arc_cap);

/* fused front end: pipeline.py:105-130 (zero_condense .. assemble).
 * delta_mode 0: delta from the RWMD bound as the reference (pipeline.py:116-122);
 * delta_mode 1: the given delta (the fixed-delta chain of test_acceptance.py:224-237). */
int w1g_front_end(w1g_ctx *ctx, const double *a, int64_t na, const double *b, int64_t nb,
                  double s, int use_condensation, int delta_mode, double delta, double k,
                  uint64_t seed, w1g_front_end_info *info);
int w1g_front_end_device(w1g_ctx *ctx, const double *d_a, int64_t na, const double *d_b,
                         int64_t nb, double s, int use_condensation, int delta_mode,
                         double delta, double k, uint64_t seed, w1g_front_end_info *info);

/* ---- batched front ends: the pairwise matrix (cfg4) and any pair list ----
 * The reference computes a batch as a loop of approx_w1 over pairs;
 * here one call runs the loop natively: the diagrams come from the context's
 * corpus (w1g_corpus_load, uploaded once), `streams` worker threads each drive
 * a child context (own stream, scratch, RWMD side context) and pull pairs from
 * a shared counter.  pairs = n_pairs (i, j) int32 index pairs. */

/* synchronous: every front end runs, networks stay in device memory; infos
 * (n_pairs entries, may be null) receives each pair's diagnostics; device_ms (may
 * be null) the device makespan: CUDA events on the context stream that every
 * child stream waits on at the start and that waits on every child at the end */
int w1g_front_end_batch(w1g_ctx *ctx, const int32_t *pairs, int64_t n_pairs, double s, int use_condensation,
                        int delta_mode, double delta, double k, uint64_t seed, int streams,
                        w1g_front_end_info *infos, float *device_ms);

/* one delivered network: host arrays inside a page-locked block owned by the
 * library until w1g_batch_release(block); status != W1G_OK carries the pair's error */
typedef struct {
    int64_t pair;             /* index into the pair list */
    int32_t i, j;             /* diagram indices */
    int32_t status;           /* W1G_OK or the pair's error code */
    int32_t pad;
    w1g_front_end_info info;  /* info.short_circuit: no network (W1 = 0) */
    int64_t *supplies, *tails, *heads, *row_offsets;  /* node_count, n_arcs, n_arcs, node_count + 1 */
    double *costs;            /* n_arcs */
    void *block;
    char message[256];
} w1g_batch_result;

/* asynchronous: start the batch; networks are copied out into pooled page-locked
 * blocks (at most max_inflight_bytes held by results not yet released; <= 0 keeps
 * the current limit, 8 GiB by default) */
int w1g_batch_begin(w1g_ctx *ctx, const int32_t *pairs, int64_t n_pairs, double s, int use_condensation,
                    int delta_mode, double delta, double k, uint64_t seed, int streams,
                    int64_t max_inflight_bytes);
/* the next finished pair (completion order); blocks; W1G_DONE when all are delivered */
int w1g_batch_next(w1g_ctx *ctx, w1g_batch_result *out);
/* give a result's block back to the pool (thread-safe, any thread) */
int w1g_batch_release(void *block);
/* stop (cancel what has not started) and join the workers; undelivered blocks are released */
int w1g_batch_end(w1g_ctx *ctx);

/* ---- retrieval (pipeline.py:146-243 nn_search) and the exact oracle (oracle.py:66-108) ---- */

/* upload a diagram corpus once: points of all diagrams back to back ((total,2)
 * float64), diagram i = rows [offsets[i], offsets[i+1]) (n_diagrams + 1 offsets) */
int w1g_corpus_load(w1g_ctx *ctx, const double *points, const int64_t *offsets, int64_t n_diagrams);
/* a host-resident corpus for the batch executor: the caller's (n_i, 2) float64
 * arrays (kept alive and unchanged until the batch ends); each worker copies its
 * pair's two diagrams to the device inside its own front end, so uploads overlap
 * the other workers' compute (page-locked arrays are DMA'd directly) */
int w1g_corpus_set_host(w1g_ctx *ctx, const double *const *points, const int64_t *sizes, int64_t n_diagrams);
/* replaces lower_bound.wcd (lower_bound.py:78-92) for query vs corpus[candidates[i]],
 * all candidates in one launch: scores[i] = wcd(query, corpus[candidates[i]]) bit for bit */
int w1g_wcd_corpus(w1g_ctx *ctx, const double *query, int64_t nq, const int64_t *candidates,
                   int64_t n_candidates, double *scores);
/* the RWMD stage of nn_search (pipeline.py:202-203): scores[i] =
 * rwmd(zero_condense(query, corpus[candidates[i]])), device zero_condense + RWMD per candidate */
int w1g_rwmd_corpus(w1g_ctx *ctx, const double *query, int64_t nq, const int64_t *candidates,
                    int64_t n_candidates, double *scores);
/* replaces oracle.dense_network (oracle.py:66-93) over slot W1G_NODES0: the complete
 * A-member x B-member network plus the diagonal arcs, already in CSR order; fetch it
 * with w1g_fetch_network.  The caller applies the DENSE_ARC_LIMIT guard (oracle.py:71-72). */
int w1g_dense_network(w1g_ctx *ctx, int64_t *node_count, int64_t *n_arcs);

#ifdef __cplusplus
}
#endif
#endif /* W1G_H */
