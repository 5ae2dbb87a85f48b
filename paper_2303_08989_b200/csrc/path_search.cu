// Host-side contraction-tree reconfiguration (the path
// and slice finder the reference's greedy_path, network.cpp:204-315, cannot
// provide for Sycamore-class circuits).  Native counterpart of
// paths.reconfigure_path: for every node of the contraction tree, take a
// frontier of up to k sub-pieces and replace how they are combined by the
// cheapest binary order (dynamic programming over the 2^k subsets).  In a
// closed network every bond joins exactly two tensors, so the open legs of a
// union of pieces are the XOR of their leg bitmasks.  Step cost model
// (model_step_cost in paths.py): MACs, or with time_model the estimated B200
// time in FP32-tier MAC units (tensor-core tiers of dispatch_cgemm 8x / 14x
// faster, an HBM floor of 8 B per operand/result element), plus the FP32
// chain latency of few-output long-k steps.  Pure host code, no CUDA.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <random>
#include <vector>

#include "../../include/tcec_b200.h"
#include "tcec_handle.h"

namespace {

struct Legs {
    std::vector<uint64_t> w;
    explicit Legs(size_t words = 0) : w(words, 0) {}
    Legs operator^(const Legs& o) const {
        Legs r(w.size());
        for (size_t i = 0; i < w.size(); ++i) r.w[i] = w[i] ^ o.w[i];
        return r;
    }
};

struct Reconf {
    int n_leaves = 0;
    size_t words = 0;
    std::vector<double> lw;       // log2 extent per label bit
    bool uniform = true;
    std::vector<Legs> legs;       // per tree node
    std::vector<int> left, right; // per tree node (-1 for leaves)
    bool time_model = false;
    double latency = 1e4;
    std::mt19937_64 rng;

    double width(const Legs& m) const {
        double s = 0.0;
        for (size_t i = 0; i < words; ++i) {
            uint64_t v = m.w[i];
            if (uniform) {
                s += double(__builtin_popcountll(v));
            } else {
                while (v) {
                    const int b = __builtin_ctzll(v);
                    s += lw[i * 64 + size_t(b)];
                    v &= v - 1;
                }
            }
        }
        return s;
    }

    double step_cost(double wa, double wb, double wo) const {
        const double wk = (wa + wb - wo) / 2.0;
        double c = std::exp2((wa + wb + wo) / 2.0);
        if (time_model) {
            const double wmin = std::min({wa - wk, wb - wk, wk});
            if (wmin >= 11) c /= 14.0;
            else if (wmin >= 9) c /= 8.0;
            c = std::max(c, 4.0 * (std::exp2(wa) + std::exp2(wb) + std::exp2(wo)));
        }
        if (latency > 0 && wo < 16.0) c += latency * std::exp2(wk);
        return c;
    }

    int add_node(int l, int r) {
        left.push_back(l);
        right.push_back(r);
        legs.push_back(legs[size_t(l)] ^ legs[size_t(r)]);
        return int(left.size()) - 1;
    }

    bool optimize(int node, int k) {
        if (left[size_t(node)] < 0) return false;
        std::vector<int> frontier{node}, internal;
        std::vector<double> fw{width(legs[size_t(node)])};
        while (int(frontier.size()) < k) {
            int best = -1;
            double bw = -1.0;
            for (size_t i = 0; i < frontier.size(); ++i) {
                if (left[size_t(frontier[i])] < 0) continue;
                const double w = fw[i] + std::uniform_real_distribution<double>(0, 1e-6)(rng);
                if (w > bw) {
                    bw = w;
                    best = int(i);
                }
            }
            if (best < 0) break;
            const int p = frontier[size_t(best)];
            internal.push_back(p);
            frontier.erase(frontier.begin() + best);
            fw.erase(fw.begin() + best);
            for (int c : {left[size_t(p)], right[size_t(p)]}) {
                frontier.push_back(c);
                fw.push_back(width(legs[size_t(c)]));
            }
        }
        const int K = int(frontier.size());
        if (K < 3) return false;
        double old = 0.0;
        for (int p : internal)
            old += step_cost(width(legs[size_t(left[size_t(p)])]), width(legs[size_t(right[size_t(p)])]),
                             width(legs[size_t(p)]));
        const uint32_t full = (1u << K) - 1;
        std::vector<Legs> sub(size_t(full) + 1, Legs(words));
        std::vector<double> sw(size_t(full) + 1, 0.0);
        for (uint32_t s = 1; s <= full; ++s) {
            const uint32_t low = s & (~s + 1);
            sub[s] = sub[s ^ low] ^ legs[size_t(frontier[size_t(__builtin_ctz(low))])];
            sw[s] = width(sub[s]);
        }
        std::vector<double> cost(size_t(full) + 1, 0.0);
        std::vector<uint32_t> choice(size_t(full) + 1, 0);
        std::vector<uint32_t> order(full);
        for (uint32_t s = 1; s <= full; ++s) order[s - 1] = s;
        std::stable_sort(order.begin(), order.end(), [](uint32_t a, uint32_t b) {
            return __builtin_popcount(a) < __builtin_popcount(b);
        });
        for (uint32_t s : order) {
            if ((s & (s - 1)) == 0) continue;
            const uint32_t low = s & (~s + 1);
            double bc = -1.0;
            uint32_t ba = 0;
            for (uint32_t a = (s - 1) & s; a; a = (a - 1) & s) {
                if (!(a & low)) continue;
                const uint32_t b = s ^ a;
                const double c = cost[a] + cost[b] + step_cost(sw[a], sw[b], sw[s]);
                if (bc < 0 || c < bc) {
                    bc = c;
                    ba = a;
                }
            }
            cost[s] = bc;
            choice[s] = ba;
        }
        if (!(cost[full] < old * (1 - 1e-9))) return false;
        // rebuild: the DP tree replaces the internal nodes; the root keeps its id
        std::function<int(uint32_t, int)> build = [&](uint32_t s, int id) -> int {
            if ((s & (s - 1)) == 0) return frontier[size_t(__builtin_ctz(s))];
            const uint32_t a = choice[s];
            const int l = build(a, -1), r = build(s ^ a, -1);
            if (id < 0) return add_node(l, r);
            left[size_t(id)] = l;
            right[size_t(id)] = r;
            legs[size_t(id)] = legs[size_t(l)] ^ legs[size_t(r)];
            return id;
        };
        build(full, node);
        return true;
    }
};

}  // namespace

extern "C" int tcec_path_reconfigure(int n_nodes, const int* ranks, const int* labels,
                                     const int64_t* dims, const int* steps, int n_steps, int k,
                                     int passes, int time_model, double latency_macs,
                                     unsigned long long seed, int* out_steps) {
    if (n_nodes < 1 || !ranks || !labels || !dims || !steps || !out_steps || n_steps != n_nodes - 1)
        return tcec::set_error(TCEC_ERR_INVALID_ARGUMENT, "bad reconfigure arguments");
    if (k < 3 || k > 16) return tcec::set_error(TCEC_ERR_INVALID_ARGUMENT, "k must be 3..16");
    // label ids -> bit positions
    std::vector<int> uniq;
    int64_t total = 0;
    for (int i = 0; i < n_nodes; ++i) total += ranks[i];
    uniq.assign(labels, labels + total);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    Reconf R;
    R.n_leaves = n_nodes;
    R.words = (uniq.size() + 63) / 64;
    R.lw.assign(R.words * 64, 0.0);
    R.time_model = time_model != 0;
    R.latency = latency_macs;
    R.rng.seed(seed);
    int64_t off = 0;
    for (int i = 0; i < n_nodes; ++i) {
        Legs m(R.words);
        for (int a = 0; a < ranks[i]; ++a) {
            const int bit = int(std::lower_bound(uniq.begin(), uniq.end(), labels[off + a]) - uniq.begin());
            m.w[size_t(bit) / 64] |= uint64_t(1) << (bit % 64);
            R.lw[size_t(bit)] = std::log2(double(dims[off + a]));
            if (dims[off + a] != 2) R.uniform = false;
        }
        off += ranks[i];
        R.legs.push_back(m);
        R.left.push_back(-1);
        R.right.push_back(-1);
    }
    int root = n_nodes - 1;
    for (int s = 0; s < n_steps; ++s) {
        const int a = steps[2 * s], b = steps[2 * s + 1];
        if (a < 0 || b < 0 || a >= int(R.left.size()) || b >= int(R.left.size()))
            return tcec::set_error(TCEC_ERR_INVALID_PATH, "step references an unknown node");
        root = R.add_node(a, b);
    }
    for (int p = 0; p < passes; ++p) {
        // bottom-up over the current tree
        std::vector<int> order, stack{root};
        while (!stack.empty()) {
            const int x = stack.back();
            stack.pop_back();
            if (R.left[size_t(x)] >= 0) {
                order.push_back(x);
                stack.push_back(R.left[size_t(x)]);
                stack.push_back(R.right[size_t(x)]);
            }
        }
        bool improved = false;
        for (auto it = order.rbegin(); it != order.rend(); ++it)
            if (R.left[size_t(*it)] >= 0) improved |= R.optimize(*it, k);
        if (!improved) break;
    }
    // tree -> SSA steps (post-order)
    int next = n_nodes, written = 0;
    std::vector<int> ssa(R.left.size(), -1);
    for (int i = 0; i < n_nodes; ++i) ssa[size_t(i)] = i;
    std::vector<std::pair<int, bool>> st{{root, false}};
    while (!st.empty()) {
        auto [x, expanded] = st.back();
        st.pop_back();
        if (R.left[size_t(x)] < 0) continue;
        if (!expanded) {
            st.push_back({x, true});
            st.push_back({R.right[size_t(x)], false});
            st.push_back({R.left[size_t(x)], false});
        } else {
            const int a = ssa[size_t(R.left[size_t(x)])], b = ssa[size_t(R.right[size_t(x)])];
            out_steps[2 * written] = std::min(a, b);
            out_steps[2 * written + 1] = std::max(a, b);
            ++written;
            ssa[size_t(x)] = next++;
        }
    }
    if (written != n_steps) return tcec::set_error(TCEC_ERR_INVALID_PATH, "tree is not a single contraction");
    return TCEC_OK;
}
