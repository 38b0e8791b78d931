// shard.cu -- one huge pair over several GPUs of one process:
// the RWMD rows sharded along numpy's summation tree.
//
// L_X = np.sum(mass * best) over X's members (lower_bound.py:58) is numpy's
// pairwise summation: n < 8 sequential, n <= 128 eight accumulators, else
// split at n2 = n/2 - (n/2) % 8 and recurse (loops_utils.h.src).  Cutting that
// tree ceil(log2 G) levels below the root gives <= 2^levels subtrees whose
// exact sums recombine, in the tree's own order, to the single-device value
// bit for bit.  Subtree t goes to context t % G; each context evaluates its
// subtrees' rows against ALL targets (w1g_rwmd_range) on its own device and
// host thread; the host combines.  (The multi-process version of the same
// plan, over NCCL, is paper_2110_14734_b200/distributed.py.)
#include <vector>

#include "common.cuh"

namespace w1g {

namespace {

constexpr int64_t PW_LEAF = 128;

inline int64_t pw_split(int64_t n) {
    const int64_t n2 = n / 2;
    return n2 - n2 % 8;
}

inline int plan_depth(int pieces) {
    int d = 0;
    while ((1 << d) < pieces) d++;
    return d;
}

void plan_rec(int64_t b, int64_t n, int d, int depth, std::vector<std::pair<int64_t, int64_t>> &out) {
    if (d == depth || n <= PW_LEAF) {
        out.emplace_back(b, b + n);
        return;
    }
    const int64_t n2 = pw_split(n);
    plan_rec(b, n2, d + 1, depth, out);
    plan_rec(b + n2, n - n2, d + 1, depth, out);
}

double combine_rec(int64_t n, int d, int depth, const std::vector<double> &parts, size_t &i) {
    if (d == depth || n <= PW_LEAF) return parts[i++];
    const int64_t n2 = pw_split(n);
    const double l = combine_rec(n2, d + 1, depth, parts, i);
    const double r = combine_rec(n - n2, d + 1, depth, parts, i);
    return l + r;
}

}  // namespace

}  // namespace w1g

using namespace w1g;

extern "C" int w1g_rwmd_sharded(w1g_ctx **ctxs, int G, double *L, double *LA, double *LB) {
    if (!ctxs || G < 1 || !L) {
        set_error("rwmd_sharded: bad arguments");
        return W1G_EINVAL;
    }
    for (int g = 0; g < G; g++)
        if (!ctxs[g] || !ctxs[g]->nodes[0].valid) {
            set_error("rwmd_sharded: context %d has no nodes0", g);
            return W1G_ESTATE;
        }
    double side_sum[2] = {0.0, 0.0};
    const int depth = plan_depth(G);
    for (int side = 0; side < 2; side++) {
        // member count (an empty range only counts)
        int64_t n = 0;
        double dummy;
        W1G_TRY(w1g_rwmd_range(ctxs[0], side, 0, 0, &dummy, &n));
        if (n == 0) continue;
        std::vector<std::pair<int64_t, int64_t>> plan;
        plan_rec(0, n, 0, depth, plan);
        std::vector<double> parts(plan.size(), 0.0);
        std::vector<int> rcs(G, W1G_OK);
        std::vector<std::string> errs(G);
        std::vector<std::thread> th;
        for (int g = 0; g < G; g++)
            th.emplace_back([&, g] {
                for (size_t t = g; t < plan.size(); t += G) {
                    int64_t nm = 0;
                    const int rc = w1g_rwmd_range(ctxs[g], side, plan[t].first, plan[t].second, &parts[t], &nm);
                    if (rc != W1G_OK) {
                        rcs[g] = rc;
                        errs[g] = w1g_last_error();
                        return;
                    }
                }
            });
        for (auto &t : th) t.join();
        for (int g = 0; g < G; g++)
            if (rcs[g] != W1G_OK) {
                set_error("%s", errs[g].c_str());
                return rcs[g];
            }
        size_t i = 0;
        side_sum[side] = combine_rec(n, 0, depth, parts, i);
    }
    if (LA) *LA = side_sum[0];
    if (LB) *LB = side_sum[1];
    *L = side_sum[1] > side_sum[0] ? side_sum[1] : side_sum[0];  // python max(l_a, l_b)
    return W1G_OK;
}
