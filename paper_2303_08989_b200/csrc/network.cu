// Device-resident TTGT tensor-network contraction.
//
// Host side mirrors reference network.cpp: split_pair / ttgt_contract
// (:33-85), fold_path / contract_network (:149-177) and greedy_path
// (:204-315) with integer labels.  The whole fold runs on one stream with no
// host round trip: every step is (optional) permute(A) -> (optional)
// permute(B) -> device-dispatched CGEMM into a stream-ordered allocation;
// per-step decisions land in device decision slots and the decision log is
// produced once at the end.  Replays over bitstrings reuse one captured CUDA
// graph of the whole fold (the topology and path do not depend on the
// bitstring, experiments.cpp:211-213).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "network_plan.h"

namespace tcec {

// concurrent replay lanes of the per-step fold in batch calls
constexpr int kFoldLanes = 4;

// lanes of node batches: 1 by default -- the slices of a sliced contraction
// already fill the GPU with large steps (Sycamore m=12: 68.8 / 74.3 / 80.7 ms
// per slice with 1 / 2 / 3 lanes); TCEC_NODE_LANES overrides for tuning
static int node_batch_lanes() {
    static const int n = [] {
        const char* e = std::getenv("TCEC_NODE_LANES");
        const int v = e ? std::atoi(e) : 0;
        return v > 0 ? v : 1;
    }();
    return n;
}  // 8 measured noisier and slower at d14 (contention)

static bool contains(const std::vector<int>& v, int x) {
    return std::find(v.begin(), v.end(), x) != v.end();
}

}  // namespace tcec

// A concurrent replay lane of the per-step fold: its own stream, node buffer,
// result slot, decision slots, operand workspace and captured graph, so the
// folds of several bitstrings run at once (a latency-bound step -- e.g. the
// one-block FP32 chain of a deep circuit's final dot product -- leaves the
// rest of the GPU to the other lanes).
struct FoldLane {
    cudaStream_t s = nullptr;
    cudaEvent_t ev = nullptr;
    void* node_dev = nullptr;
    void* result_dev = nullptr;
    tcec::DevDecision* dec = nullptr;
    int dec_slots = 0;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    cudaGraphExec_t graph = nullptr;
    std::string graph_key;
    void release() {
        if (graph) cudaGraphExecDestroy(graph);
        if (node_dev) cudaFree(node_dev);
        if (result_dev) cudaFree(result_dev);
        if (dec) cudaFree(dec);
        if (ws) cudaFree(ws);
        if (ev) cudaEventDestroy(ev);
        if (s) cudaStreamDestroy(s);
        *this = FoldLane();
    }
};

struct tcec_network_s {
    tcec_handle h = nullptr;
    std::vector<tcec::NetNode> nodes;
    std::vector<int64_t> offset;     // element offset of node i in node_dev
    int64_t total = 0;
    void* node_dev = nullptr;        // all node data, contiguous
    std::vector<float> host_stage;   // staged host copy (uploaded lazily)
    bool dirty = true;
    // cached graph of the last fold (plan signature -> exec)
    std::string graph_key;
    cudaGraphExec_t graph = nullptr;
    void* result_dev = nullptr;      // stable home of the final tensor
    int64_t result_size = 0;
    tcec::SmallProgram small;        // fused small-step program (small_fold.cu)
    tcec::HybridProgram hyb;         // subtree prologue of the per-step fold
    // node labels/dims are fixed at creation: validate once; the fold plan of
    // the last (path, config) is reused by repeated batch calls
    bool validated = false;
    std::string plan_key;
    tcec::FoldPlan plan_cache;
    std::vector<FoldLane> lanes;
    // decisions of the last batch call (selector / node batch): the tensor-core
    // steps' DevDecision of every run, archived on the device after each run's
    // fold and read back with the amplitudes (tcec_network_batch_run_info)
    std::vector<tcec_dispatch_result_t> step_results;  // of the last contract_network
    std::vector<tcec::DevDecision> batch_dec;
    std::vector<int> batch_tc;       // step indices of the tensor-core steps
    int batch_runs = 0;
    std::string batch_plan_key;
    ~tcec_network_s() {
        for (auto& l : lanes) l.release();
        small.release();
        hyb.release();
        if (graph) cudaGraphExecDestroy(graph);
        if (node_dev) cudaFree(node_dev);
        if (result_dev) cudaFree(result_dev);
    }
};

namespace tcec {

// validate_network, network.cpp:114-127
static int validate(const tcec_network_s& net) {
    std::map<int, std::vector<std::pair<int, int64_t>>> occ;
    for (size_t i = 0; i < net.nodes.size(); ++i) {
        const NetNode& nd = net.nodes[i];
        if (nd.labels.size() != nd.dims.size())
            return set_error(TCEC_ERR_SHAPE_MISMATCH, "tensor labels and dims differ in length");
        for (auto d : nd.dims)
            if (d < 1) return set_error(TCEC_ERR_SHAPE_MISMATCH, "tensor extents must be >= 1");
        for (size_t a = 0; a < nd.labels.size(); ++a)
            for (size_t b = a + 1; b < nd.labels.size(); ++b)
                if (nd.labels[a] == nd.labels[b])
                    return set_error(TCEC_ERR_SHAPE_MISMATCH, "tensor labels must be distinct");
        for (size_t a = 0; a < nd.labels.size(); ++a)
            occ[nd.labels[a]].emplace_back(int(i), nd.dims[a]);
    }
    for (const auto& [label, o] : occ) {
        if (o.size() > 2)
            return set_error(TCEC_ERR_SHAPE_MISMATCH,
                             "label " + std::to_string(label) + " appears in more than two nodes");
        if (o.size() == 2 && o[0].second != o[1].second)
            return set_error(TCEC_ERR_EXTENT_MISMATCH,
                             "label " + std::to_string(label) + " has mismatched extents");
    }
    return TCEC_OK;
}

// TCEC_VIEW_GATHER = 0 disables the fused TTGT gather of skinny steps (A/B)
static bool view_gather_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TCEC_VIEW_GATHER");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

// fold_path + ttgt_contract bookkeeping (network.cpp:33-85, :149-168)
static int build_plan(const tcec_network_s& net, const int* steps, int n_steps,
                      const tcec_dispatch_config_t& cfg, FoldPlan* out) {
    if (net.nodes.empty()) return set_error(TCEC_ERR_INVALID_PATH, "empty network");
    std::map<int, NetNode> live;
    for (size_t i = 0; i < net.nodes.size(); ++i) live.emplace(int(i), net.nodes[i]);
    int next_id = int(net.nodes.size());
    FoldPlan plan;
    for (int s = 0; s < n_steps; ++s) {
        const int ia = steps[2 * s], ib = steps[2 * s + 1];
        auto a_it = live.find(ia), b_it = live.find(ib);
        if (ia == ib || a_it == live.end() || b_it == live.end())
            return set_error(TCEC_ERR_INVALID_PATH, "step references a dead or unknown node");
        const NetNode& A = a_it->second;
        const NetNode& B = b_it->second;
        // split_pair: free_a | shared (a's order) | free_b (b's order)
        std::vector<int> free_a, shared, free_b;
        std::vector<int64_t> fa_d, sh_d, fb_d;
        for (size_t i = 0; i < A.labels.size(); ++i) {
            const int l = A.labels[i];
            auto pos = std::find(B.labels.begin(), B.labels.end(), l);
            if (pos != B.labels.end()) {
                const int64_t bd = B.dims[size_t(pos - B.labels.begin())];
                if (bd != A.dims[i])
                    return set_error(TCEC_ERR_EXTENT_MISMATCH,
                                     "label " + std::to_string(l) + " has extents " +
                                         std::to_string(A.dims[i]) + " and " + std::to_string(bd));
                shared.push_back(l);
                sh_d.push_back(A.dims[i]);
            } else {
                free_a.push_back(l);
                fa_d.push_back(A.dims[i]);
            }
        }
        for (size_t i = 0; i < B.labels.size(); ++i)
            if (!contains(A.labels, B.labels[i])) {
                free_b.push_back(B.labels[i]);
                fb_d.push_back(B.dims[i]);
            }
        StepPlan sp;
        sp.ia = ia;
        sp.ib = ib;
        sp.m = sp.n = sp.k = 1;
        for (auto d : fa_d) sp.m *= d;
        for (auto d : sh_d) sp.k *= d;
        for (auto d : fb_d) sp.n *= d;
        // permutations A -> (free_a | shared), B -> (shared | free_b)
        std::vector<int> order_a = free_a;
        order_a.insert(order_a.end(), shared.begin(), shared.end());
        std::vector<int> order_b = shared;
        order_b.insert(order_b.end(), free_b.begin(), free_b.end());
        auto axes = [](const NetNode& t, const std::vector<int>& order, std::vector<int>* ax) {
            bool identity = true;
            for (size_t a = 0; a < order.size(); ++a) {
                const int o = int(std::find(t.labels.begin(), t.labels.end(), order[a]) -
                                  t.labels.begin());
                ax->push_back(o);
                identity = identity && o == int(a);
            }
            return !identity;
        };
        sp.perm_a = axes(A, order_a, &sp.a_axis);
        sp.perm_b = axes(B, order_b, &sp.b_axis);
        sp.a_dims = A.dims;
        sp.b_dims = B.dims;
        sp.a_size = A.size();
        sp.b_size = B.size();
        sp.n_shared = int(shared.size());
        sp.dp = plan_dispatch(sp.m, sp.n, sp.k, cfg);
        // skinny FP32-tier step: read the long operand in place (the view
        // addresses the same elements in the same order -> identical bits)
        if (sp.dp.tier == kTierFp32 && skinny_shape(sp.m, sp.n, sp.k) && view_gather_enabled()) {
            if (sp.m <= sp.n && sp.perm_b)
                sp.view_b = make_matrix_view(int(B.dims.size()), B.dims.data(), sp.b_axis.data(), sp.n_shared,
                                             &sp.view);
            else if (sp.m > sp.n && sp.perm_a)
                sp.view_a = make_matrix_view(int(A.dims.size()), A.dims.data(), sp.a_axis.data(),
                                             int(A.dims.size()) - sp.n_shared, &sp.view);
        }
        if (sp.dp.tier == kTierTc && view_gather_enabled()) {
            // only views the preparation kernels read efficiently: A rows along
            // K in unit-stride runs of >= 4 complex (the 16-B fast path), B
            // columns in unit-stride runs of >= 32 (a warp's coalesced row);
            // otherwise the permute (4.4-5.9 TB/s) is cheaper than a scattered gather
            auto inner_ok = [](const RunMap& r, uint32_t min_ext) {
                return r.n == 0 || (r.stride[r.n - 1] == 1 && r.ext[r.n - 1] >= min_ext);
            };
            if (sp.perm_a)
                sp.tview_a = make_matrix_view(int(A.dims.size()), A.dims.data(), sp.a_axis.data(),
                                              int(A.dims.size()) - sp.n_shared, &sp.tva) &&
                             inner_ok(sp.tva.cols, 4);
            if (sp.perm_b)
                sp.tview_b = make_matrix_view(int(B.dims.size()), B.dims.data(), sp.b_axis.data(), sp.n_shared,
                                              &sp.tvb) &&
                             inner_ok(sp.tvb.cols, 32);
        }
        if (sp.dp.tier == kTierTc && cfg.k_tile < 1)
            return set_error(TCEC_ERR_INVALID_ARGUMENT, "k_tile must be >= 1");
        plan.ws_bytes = std::max(plan.ws_bytes, plan_workspace(sp.dp, sp.m, sp.n));
        NetNode result;
        result.labels = free_a;
        result.labels.insert(result.labels.end(), free_b.begin(), free_b.end());
        result.dims = fa_d;
        result.dims.insert(result.dims.end(), fb_d.begin(), fb_d.end());
        live.erase(ia);
        live.erase(ib);
        live.emplace(next_id++, std::move(result));
        plan.steps.push_back(std::move(sp));
    }
    if (live.size() != 1) return set_error(TCEC_ERR_INVALID_PATH, "path leaves more than one node");
    plan.out_labels = live.begin()->second.labels;
    plan.out_dims = live.begin()->second.dims;
    *out = std::move(plan);
    return TCEC_OK;
}

static int upload(tcec_network_s& net) {
    if (!net.dirty) return TCEC_OK;
    Handle& h = *net.h;
    if (!net.node_dev) {
        const cudaError_t e = cudaMalloc(&net.node_dev, size_t(std::max<int64_t>(net.total, 1)) * 8);
        if (e != cudaSuccess) return cuda_error(e, "node buffer");
    }
    const cudaError_t e = cudaMemcpyAsync(net.node_dev, net.host_stage.data(), size_t(net.total) * 8,
                                          cudaMemcpyHostToDevice, h.stream);
    if (e != cudaSuccess) return cuda_error(e, "node upload");
    net.dirty = false;
    return TCEC_OK;
}

// Enqueue the fold on the handle stream.  Intermediates are stream-ordered
// allocations freed as soon as they are consumed; the final tensor is copied
// into net.result_dev.
static int enqueue_fold(tcec_network_s& net, const FoldPlan& plan, const tcec_dispatch_config_t& cfg,
                        DevDecision* dec, void* ws, const HybridProgram* hyb) {
    Handle& h = *net.h;
    cudaStream_t s = h.stream;
    std::map<int, std::pair<float2*, bool>> live;  // id -> (buffer, owned)
    float2* base = static_cast<float2*>(net.node_dev);
    for (size_t i = 0; i < net.nodes.size(); ++i) live[int(i)] = {base + net.offset[i], false};
    int next_id = int(net.nodes.size());
    // hybrid prologue: every subtree of tiny SIMT steps in one launch
    float2* tree_out = nullptr;
    if (hyb && hyb->ok) {
        const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&tree_out),
                                              size_t(std::max<int64_t>(hyb->out_elems, 1)) * 8, s);
        if (e != cudaSuccess) return cuda_error(e, "subtree outputs");
        const int rc = launch_hybrid_trees(*hyb, base, tree_out, s);
        if (rc) return rc;
    } else {
        hyb = nullptr;
    }
    for (size_t si = 0; si < plan.steps.size(); ++si) {
        const StepPlan& sp = plan.steps[si];
        if (hyb && hyb->fused[si]) {
            live.erase(sp.ia);
            live.erase(sp.ib);
            if (hyb->root_out[si] >= 0) live[next_id] = {tree_out + hyb->root_out[si], false};
            ++next_id;
            continue;
        }
        auto [pa_src, own_a] = live[sp.ia];
        auto [pb_src, own_b] = live[sp.ib];
        float2* pa = pa_src;
        float2* pb = pb_src;
        cudaError_t e;
        const bool perm_a = sp.perm_a && !sp.view_a && !sp.tview_a,
                   perm_b = sp.perm_b && !sp.view_b && !sp.tview_b;
        if (perm_a) {
            e = cudaMallocAsync(reinterpret_cast<void**>(&pa), size_t(sp.a_size) * 8, s);
            if (e != cudaSuccess) return cuda_error(e, "permute buffer");
            launch_permute(pa_src, pa, int(sp.a_dims.size()), sp.a_dims.data(), sp.a_axis.data(), s);
        }
        if (perm_b) {
            e = cudaMallocAsync(reinterpret_cast<void**>(&pb), size_t(sp.b_size) * 8, s);
            if (e != cudaSuccess) return cuda_error(e, "permute buffer");
            launch_permute(pb_src, pb, int(sp.b_dims.size()), sp.b_dims.data(), sp.b_axis.data(), s);
        }
        float2* pc = nullptr;
        e = cudaMallocAsync(reinterpret_cast<void**>(&pc), size_t(std::max<int64_t>(sp.m * sp.n, 1)) * 8, s);
        if (e != cudaSuccess) return cuda_error(e, "step output");
        if (sp.view_a || sp.view_b) {
            // fused TTGT gather (FP32 tier: no decision slot, nothing else to launch)
            if (!launch_skinny_view(pa, pb, pc, sp.m, sp.n, sp.k, sp.view, s))
                return set_error(TCEC_ERR_LOGIC, "skinny view step: shape not skinny");
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_error(e, "skinny view step");
        } else {
            const int rc = launch_dispatch(h, reinterpret_cast<const float*>(pa),
                                           reinterpret_cast<const float*>(pb),
                                           reinterpret_cast<float*>(pc), sp.m, sp.n, sp.k, cfg, sp.dp,
                                           dec + si, ws, nullptr, sp.tview_a ? &sp.tva : nullptr,
                                           sp.tview_b ? &sp.tvb : nullptr);
            if (rc) return rc;
        }
        if (perm_a) cudaFreeAsync(pa, s);
        if (perm_b) cudaFreeAsync(pb, s);
        if (own_a) cudaFreeAsync(pa_src, s);
        if (own_b) cudaFreeAsync(pb_src, s);
        live.erase(sp.ia);
        live.erase(sp.ib);
        live[next_id++] = {pc, true};
    }
    auto [res, own] = live.begin()->second;
    int64_t size = 1;
    for (auto d : plan.out_dims) size *= d;
    const cudaError_t e =
        cudaMemcpyAsync(net.result_dev, res, size_t(size) * 8, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_error(e, "result copy");
    if (own) cudaFreeAsync(res, s);
    if (tree_out) cudaFreeAsync(tree_out, s);
    return TCEC_OK;
}

static int prepare(tcec_network_s& net, const int* steps, int n_steps,
                   const tcec_dispatch_config_t& cfg, const FoldPlan** plan_out, DevDecision** dec,
                   void** ws) {
    if (!net.validated) {
        const int rv = validate(net);
        if (rv) return rv;
        net.validated = true;
    }
    std::string key(reinterpret_cast<const char*>(steps), size_t(std::max(n_steps, 0)) * 2 * sizeof(int));
    key.append(reinterpret_cast<const char*>(&cfg), sizeof(cfg));
    int rc = TCEC_OK;
    if (key != net.plan_key) {
        net.plan_key.clear();
        rc = build_plan(net, steps, n_steps, cfg, &net.plan_cache);
        if (rc) return rc;
        net.plan_key = key;
    }
    const FoldPlan* plan = &net.plan_cache;
    *plan_out = plan;
    Handle& h = *net.h;
    *dec = h.decisions(std::max(n_steps, 1));
    if (!*dec) return set_error(TCEC_ERR_CUDA, "decision buffer allocation failed");
    *ws = nullptr;
    if (plan->ws_bytes) {
        *ws = h.workspace(plan->ws_bytes);
        if (!*ws) return set_error(TCEC_ERR_CUDA, "workspace allocation failed");
    }
    int64_t size = 1;
    for (auto d : plan->out_dims) size *= d;
    if (size > net.result_size) {
        if (net.result_dev) cudaFree(net.result_dev);
        const cudaError_t e = cudaMalloc(&net.result_dev, size_t(size) * 8);
        if (e != cudaSuccess) return cuda_error(e, "result buffer");
        net.result_size = size;
        if (net.graph) {
            cudaGraphExecDestroy(net.graph);
            net.graph = nullptr;
            net.graph_key.clear();
        }
    }
    return upload(net);
}

static std::string plan_key(const int* steps, int n_steps, const tcec_dispatch_config_t& cfg,
                            const Handle& h, const void* ws, const void* dec) {
    std::string k(reinterpret_cast<const char*>(steps), size_t(n_steps) * 2 * sizeof(int));
    k.append(reinterpret_cast<const char*>(&cfg), sizeof(cfg));
    k.append(reinterpret_cast<const char*>(&h.flush_kblocks), sizeof(int));
    k.append(reinterpret_cast<const char*>(&h.gemm_pair), sizeof(int));  // kernel variant
    k.append(reinterpret_cast<const char*>(&h.layout), sizeof(int));     // operand layout
    k.append(reinterpret_cast<const char*>(&h.executor), sizeof(int));
    k.append(reinterpret_cast<const char*>(&ws), sizeof(ws));
    k.append(reinterpret_cast<const char*>(&dec), sizeof(dec));
    return k;
}

// Run the fold, through a cached CUDA graph when possible.
static int run_fold(tcec_network_s& net, const int* steps, int n_steps,
                    const tcec_dispatch_config_t& cfg, const FoldPlan& plan, DevDecision* dec,
                    void* ws, bool use_graph) {
    Handle& h = *net.h;
    // the subtree prologue (policy 0 auto / 3 hybrid), built and uploaded
    // outside any capture
    const HybridProgram* hyb = nullptr;
    if (h.executor == 0 || h.executor == 3) {
        std::string hkey(reinterpret_cast<const char*>(steps), size_t(n_steps) * 2 * sizeof(int));
        hkey.append(reinterpret_cast<const char*>(&cfg), sizeof(cfg));
        if (net.hyb.key != hkey) {
            net.hyb.release();
            build_hybrid_program(net.nodes, net.offset, plan, &net.hyb);
            net.hyb.key = hkey;
            const int rc = upload_hybrid_program(&net.hyb);
            if (rc) {
                net.hyb.key.clear();
                return rc;
            }
        }
        if (net.hyb.ok) hyb = &net.hyb;
    }
    if (!use_graph) return enqueue_fold(net, plan, cfg, dec, ws, hyb);
    std::string key = plan_key(steps, n_steps, cfg, h, ws, dec);
    key.append(reinterpret_cast<const char*>(&hyb), sizeof(hyb));
    if (!net.graph || key != net.graph_key) {
        if (net.graph) {
            cudaGraphExecDestroy(net.graph);
            net.graph = nullptr;
        }
        // a capture or instantiation that fails for any reason falls back to
        // direct launches (which report a genuine error themselves)
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamBeginCapture(h.stream, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return enqueue_fold(net, plan, cfg, dec, ws, hyb);
        }
        const int rc = enqueue_fold(net, plan, cfg, dec, ws, hyb);
        e = cudaStreamEndCapture(h.stream, &g);
        if (rc == TCEC_OK && e == cudaSuccess && g) e = cudaGraphInstantiate(&net.graph, g, 0);
        if (g) cudaGraphDestroy(g);
        if (rc != TCEC_OK || e != cudaSuccess || !net.graph) {
            net.graph = nullptr;
            cudaGetLastError();
            return enqueue_fold(net, plan, cfg, dec, ws, hyb);
        }
        net.graph_key = key;
    }
    const cudaError_t e = cudaGraphLaunch(net.graph, h.stream);
    if (e != cudaSuccess) return cuda_error(e, "graph launch");
    return TCEC_OK;
}

// Run the (cached-graph) fold on lane `ln`: the lane's buffers and stream stand
// in for the network's and the handle's while the graph is captured/launched.
static int run_fold_lane(tcec_network_s& net, FoldLane& ln, const int* steps, int n_steps,
                         const tcec_dispatch_config_t& cfg, const FoldPlan& plan) {
    Handle& h = *net.h;
    std::swap(net.node_dev, ln.node_dev);
    std::swap(net.result_dev, ln.result_dev);
    std::swap(net.graph, ln.graph);
    std::swap(net.graph_key, ln.graph_key);
    const cudaStream_t saved = h.stream;
    h.stream = ln.s;
    const int rc = run_fold(net, steps, n_steps, cfg, plan, ln.dec, ln.ws, true);
    h.stream = saved;
    std::swap(net.node_dev, ln.node_dev);
    std::swap(net.result_dev, ln.result_dev);
    std::swap(net.graph, ln.graph);
    std::swap(net.graph_key, ln.graph_key);
    return rc;
}

// Make `count` lanes able to run `plan` (grown on demand, kept across calls).
static int ensure_lanes(tcec_network_s& net, int count, const FoldPlan& plan) {
    if (int(net.lanes.size()) < count) net.lanes.resize(size_t(count));
    const int slots = std::max<int>(int(plan.steps.size()), 1);
    for (int i = 0; i < count; ++i) {
        FoldLane& ln = net.lanes[size_t(i)];
        cudaError_t e = cudaSuccess;
        if (!ln.s) e = cudaStreamCreateWithFlags(&ln.s, cudaStreamNonBlocking);
        if (e == cudaSuccess && !ln.ev) e = cudaEventCreateWithFlags(&ln.ev, cudaEventDisableTiming);
        if (e == cudaSuccess && !ln.node_dev)
            e = cudaMalloc(&ln.node_dev, size_t(std::max<int64_t>(net.total, 1)) * 8);
        if (e == cudaSuccess && !ln.result_dev) e = cudaMalloc(&ln.result_dev, 8);
        if (e == cudaSuccess && ln.dec_slots < slots) {
            if (ln.dec) cudaFree(ln.dec);
            ln.dec = nullptr;
            ln.dec_slots = 0;
            e = cudaMalloc(&ln.dec, sizeof(tcec::DevDecision) * size_t(slots));
            if (e == cudaSuccess) e = cudaMemset(ln.dec, 0, sizeof(tcec::DevDecision) * size_t(slots));
            if (e == cudaSuccess) ln.dec_slots = slots;
        }
        if (e == cudaSuccess && ln.ws_bytes < plan.ws_bytes) {
            if (ln.ws) cudaFree(ln.ws);
            ln.ws = nullptr;
            ln.ws_bytes = 0;
            e = cudaMalloc(&ln.ws, plan.ws_bytes);
            if (e == cudaSuccess) ln.ws_bytes = plan.ws_bytes;
        }
        if (e != cudaSuccess) return cuda_error(e, "fold lane");
    }
    return TCEC_OK;
}

// The fused small-step program for this (path, config, variable nodes), built
// once and cached; nullptr when the executor policy or eligibility says no.
static const SmallProgram* small_program(tcec_network_s& net, const int* steps, int n_steps,
                                         const tcec_dispatch_config_t& cfg, const FoldPlan& plan,
                                         const std::vector<int>& var_nodes, int* rc) {
    *rc = TCEC_OK;
    // 0 auto (fused if eligible, else per-step + subtree prologue), 1 per-step
    // only, 2 fused only, 3 per-step + subtree prologue
    const int policy = net.h->executor;
    if (policy == 1 || policy == 3) return nullptr;
    std::string key(reinterpret_cast<const char*>(steps), size_t(n_steps) * 2 * sizeof(int));
    key.append(reinterpret_cast<const char*>(&cfg), sizeof(cfg));
    key.append(reinterpret_cast<const char*>(var_nodes.data()), var_nodes.size() * sizeof(int));
    if (net.small.key != key) {
        net.small.release();
        build_small_program(net.nodes, net.offset, plan, var_nodes, &net.small);
        net.small.key = key;
        if (net.small.ok) {
            *rc = upload_small_program(&net.small);
            if (*rc) return nullptr;
        }
    }
    if (!net.small.ok) {
        if (policy == 2) *rc = set_error(TCEC_ERR_INVALID_ARGUMENT, "fused executor: " + net.small.why);
        return nullptr;
    }
    return &net.small;
}

// ------------------------------------------------------------- greedy path

struct Summary {
    int id;
    std::vector<int> labels;
    std::vector<int64_t> dims;
};

// greedy_simulate, network.cpp:204-298: repeatedly contract the adjacent pair
// with the smallest result, ties to the lowest (id, id) pair; disconnected
// components fall back to the smallest outer product
static void greedy(std::vector<Summary> live, int next_id, std::vector<int>* steps) {
    while (live.size() > 1) {
        int64_t best = -1;
        size_t ba = 0, bb = 0;
        auto better = [&](int64_t size, size_t x, size_t y) {
            const std::pair<int, int> ids = std::minmax(live[x].id, live[y].id);
            if (best < 0) return true;
            const std::pair<int, int> bids = std::minmax(live[ba].id, live[bb].id);
            return size < best || (size == best && ids < bids);
        };
        for (size_t x = 0; x < live.size(); ++x)
            for (size_t y = x + 1; y < live.size(); ++y) {
                int64_t fx = 1, fy = 1;
                bool adjacent = false;
                for (size_t i = 0; i < live[x].labels.size(); ++i) {
                    if (contains(live[y].labels, live[x].labels[i]))
                        adjacent = true;
                    else
                        fx *= live[x].dims[i];
                }
                if (!adjacent) continue;
                for (size_t i = 0; i < live[y].labels.size(); ++i)
                    if (!contains(live[x].labels, live[y].labels[i])) fy *= live[y].dims[i];
                if (better(fx * fy, x, y)) {
                    best = fx * fy;
                    ba = x;
                    bb = y;
                }
            }
        if (best < 0) {
            for (size_t x = 0; x < live.size(); ++x)
                for (size_t y = x + 1; y < live.size(); ++y) {
                    int64_t size = 1;
                    for (auto d : live[x].dims) size *= d;
                    for (auto d : live[y].dims) size *= d;
                    if (better(size, x, y)) {
                        best = size;
                        ba = x;
                        bb = y;
                    }
                }
        }
        Summary& a = live[ba];
        Summary& b = live[bb];
        Summary merged;
        merged.id = next_id++;
        for (size_t i = 0; i < a.labels.size(); ++i)
            if (!contains(b.labels, a.labels[i])) {
                merged.labels.push_back(a.labels[i]);
                merged.dims.push_back(a.dims[i]);
            }
        for (size_t i = 0; i < b.labels.size(); ++i)
            if (!contains(a.labels, b.labels[i])) {
                merged.labels.push_back(b.labels[i]);
                merged.dims.push_back(b.dims[i]);
            }
        steps->push_back(std::min(a.id, b.id));
        steps->push_back(std::max(a.id, b.id));
        const size_t hi = std::max(ba, bb), lo = std::min(ba, bb);
        live.erase(live.begin() + long(hi));
        live.erase(live.begin() + long(lo));
        live.push_back(std::move(merged));
    }
}

// scatter one run's variable-node data (concatenated, node order) into the
// contiguous node buffer; seg[i] = {dst offset, src offset, count} in elements
__global__ void scatter_nodes_kernel(float2* node_base, const float2* src, const int64_t* seg,
                                     int n_seg) {
    for (int s = blockIdx.x; s < n_seg; s += gridDim.x) {
        const int64_t dst = seg[3 * s], off = seg[3 * s + 1], cnt = seg[3 * s + 2];
        for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) node_base[dst + i] = src[off + i];
    }
}

__global__ void set_selectors_kernel(float2* node_base, const int64_t* sel_off, int n_sel,
                                     const uint8_t* bits) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_sel) return;
    float2* p = node_base + sel_off[q];
    const bool one = bits[q] != 0;
    p[0] = make_float2(one ? 0.0f : 1.0f, 0.0f);
    p[1] = make_float2(one ? 1.0f : 0.0f, 0.0f);
}

// copy the decision slots of one run's tensor-core steps into its archive row
__global__ void archive_decisions_kernel(const DevDecision* dec, const int* tc_steps, int n_tc,
                                         DevDecision* arch) {
    for (int i = threadIdx.x; i < n_tc; i += blockDim.x) arch[i] = dec[tc_steps[i]];
}

// Per-call state of the decision archive of a batch.
struct BatchArchive {
    std::vector<int> tc;        // tensor-core step indices
    int* d_tc = nullptr;
    DevDecision* d_arch = nullptr;
    int n_runs = 0;
    int begin(const FoldPlan& plan, int runs, cudaStream_t s) {
        tc.clear();
        for (size_t i = 0; i < plan.steps.size(); ++i)
            if (plan.steps[i].dp.tier == kTierTc) tc.push_back(int(i));
        n_runs = runs;
        if (tc.empty() || runs <= 0) return TCEC_OK;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_tc), tc.size() * sizeof(int), s);
        if (e == cudaSuccess)
            e = cudaMallocAsync(reinterpret_cast<void**>(&d_arch),
                                tc.size() * size_t(runs) * sizeof(DevDecision), s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_tc, tc.data(), tc.size() * sizeof(int), cudaMemcpyHostToDevice, s);
        return e == cudaSuccess ? TCEC_OK : cuda_error(e, "decision archive");
    }
    // after run r's fold on stream s (reading that fold's decision slots)
    void record(const DevDecision* dec, int r, cudaStream_t s) const {
        if (tc.empty()) return;
        archive_decisions_kernel<<<1, 128, 0, s>>>(dec, d_tc, int(tc.size()), d_arch + size_t(r) * tc.size());
    }
    int download(std::vector<DevDecision>* out, cudaStream_t s) const {
        out->assign(tc.size() * size_t(n_runs), DevDecision{});
        if (tc.empty() || n_runs <= 0) return TCEC_OK;
        const cudaError_t e = cudaMemcpyAsync(out->data(), d_arch, out->size() * sizeof(DevDecision),
                                              cudaMemcpyDeviceToHost, s);
        return e == cudaSuccess ? TCEC_OK : cuda_error(e, "decision archive download");
    }
    void release(cudaStream_t s) {
        if (d_tc) cudaFreeAsync(d_tc, s);
        if (d_arch) cudaFreeAsync(d_arch, s);
        d_tc = nullptr;
        d_arch = nullptr;
    }
};

// After the batch synchronized: keep the archive on the network and raise
// what the reference would have raised on the first failing run -- the
// ScaleOverflow of scale_matrix (precsel.cpp:54-57, 209-216) or the
// logic_error of a skipped stage 2 (precsel.cpp:117-118).  The format
// overflow flag is not an error (DispatchResult::overflow); it is reported
// per run by tcec_network_batch_run_info.
static int settle_batch(tcec_network_s& net, BatchArchive& ar) {
    net.batch_tc = ar.tc;
    net.batch_runs = ar.n_runs;
    net.batch_plan_key = net.plan_key;
    const size_t nt = ar.tc.size();
    for (int r = 0; r < ar.n_runs; ++r)
        for (size_t i = 0; i < nt; ++i) {
            const DevDecision& d = net.batch_dec[size_t(r) * nt + i];
            const StepPlan& sp = net.plan_cache.steps[size_t(ar.tc[i])];
            if (sp.dp.stats && d.kind < 0)
                return set_error(TCEC_ERR_LOGIC, "run " + std::to_string(r) + ", step " +
                                                     std::to_string(ar.tc[i]) +
                                                     ": matrix_tolerance: stage-2 statistics required but skipped");
            if (d.scale_overflow)
                return set_error(TCEC_ERR_SCALE_OVERFLOW, "run " + std::to_string(r) + ", step " +
                                                              std::to_string(ar.tc[i]) +
                                                              ": scaled component left the f32 range");
        }
    return TCEC_OK;
}

}  // namespace tcec

using namespace tcec;

extern "C" {

int tcec_network_create(tcec_handle h, int n_nodes, const int* ranks, const int* labels,
                        const int64_t* dims, tcec_network* out) {
    // h may be NULL for planning-only use (greedy_path); contraction needs a handle
    if (!out || n_nodes < 0) return set_error(TCEC_ERR_INVALID_ARGUMENT, "bad argument");
    if (h) cudaSetDevice(h->device);
    auto* net = new tcec_network_s();
    net->h = h;
    int64_t pos = 0, off = 0;
    for (int i = 0; i < n_nodes; ++i) {
        NetNode nd;
        for (int a = 0; a < ranks[i]; ++a) {
            nd.labels.push_back(labels[pos + a]);
            nd.dims.push_back(dims[pos + a]);
        }
        pos += ranks[i];
        net->offset.push_back(off);
        off += nd.size();
        net->nodes.push_back(std::move(nd));
    }
    net->total = off;
    net->host_stage.assign(size_t(2 * std::max<int64_t>(off, 1)), 0.0f);
    *out = net;
    return TCEC_OK;
}

int tcec_network_destroy(tcec_network net) {
    if (!net) return TCEC_OK;
    if (net->h) {
        cudaSetDevice(net->h->device);
        cudaStreamSynchronize(net->h->stream);
    }
    delete net;
    return TCEC_OK;
}

int tcec_network_set_node(tcec_network net, int node, const void* host_data) {
    if (!net || node < 0 || node >= int(net->nodes.size()))
        return set_error(TCEC_ERR_INVALID_ARGUMENT, "bad node index");
    std::memcpy(net->host_stage.data() + 2 * net->offset[size_t(node)], host_data,
                size_t(net->nodes[size_t(node)].size()) * 8);
    net->dirty = true;
    return TCEC_OK;
}

int tcec_network_greedy_path(tcec_network net, int* steps) {
    if (!net) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null network");
    int rc = validate(*net);
    if (rc) return rc;
    if (net->nodes.empty()) return set_error(TCEC_ERR_INVALID_PATH, "empty network");
    std::vector<Summary> live;
    for (size_t i = 0; i < net->nodes.size(); ++i)
        live.push_back({int(i), net->nodes[i].labels, net->nodes[i].dims});
    std::vector<int> out;
    greedy(std::move(live), int(net->nodes.size()), &out);
    std::copy(out.begin(), out.end(), steps);
    return TCEC_OK;
}

int tcec_contract_network(tcec_network net, const int* steps, int n_steps,
                          const tcec_dispatch_config_t* cfg, void* out_host, int64_t out_capacity,
                          int* out_rank, int* out_labels, char* log_lines, int64_t log_capacity) {
    if (!net || !cfg) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    if (!net->h) return set_error(TCEC_ERR_CUDA, "network has no device handle");
    Handle& h = *net->h;
    cudaSetDevice(h.device);
    const FoldPlan* plan_ptr = nullptr;
    DevDecision* dec = nullptr;
    void* ws = nullptr;
    int rc = prepare(*net, steps, n_steps, *cfg, &plan_ptr, &dec, &ws);
    if (rc) return rc;
    const FoldPlan& plan = *plan_ptr;
    const SmallProgram* sp_fused = small_program(*net, steps, n_steps, *cfg, plan, {}, &rc);
    if (rc) return rc;
    if (sp_fused) {
        rc = launch_small_program(*sp_fused, static_cast<const float2*>(net->node_dev), 1, nullptr, 0,
                                  nullptr, static_cast<float2*>(net->result_dev), h.stream);
    } else {
        rc = run_fold(*net, steps, n_steps, *cfg, plan, dec, ws, false);
    }
    if (rc) return rc;
    int64_t size = 1;
    for (auto d : plan.out_dims) size *= d;
    if (out_capacity < size) return set_error(TCEC_ERR_SHAPE_MISMATCH, "output buffer too small");
    cudaError_t e = cudaMemcpyAsync(out_host, net->result_dev, size_t(size) * 8,
                                    cudaMemcpyDeviceToHost, h.stream);
    if (e != cudaSuccess) return cuda_error(e, "result download");
    std::vector<DevDecision> dd(plan.steps.size());
    if (sp_fused) {
        std::memset(dd.data(), 0, sizeof(DevDecision) * dd.size());  // SIMT tiers: no statistics
    } else if (!plan.steps.empty()) {
        e = cudaMemcpyAsync(dd.data(), dec, sizeof(DevDecision) * dd.size(), cudaMemcpyDeviceToHost,
                            h.stream);
        if (e != cudaSuccess) return cuda_error(e, "decision download");
    }
    e = cudaStreamSynchronize(h.stream);
    if (e != cudaSuccess) return cuda_error(e, "contract_network");
    if (out_rank) *out_rank = int(plan.out_labels.size());
    if (out_labels) std::copy(plan.out_labels.begin(), plan.out_labels.end(), out_labels);
    std::string log;
    net->step_results.assign(plan.steps.size(), tcec_dispatch_result_t{});
    for (size_t i = 0; i < plan.steps.size(); ++i) {
        const StepPlan& sp = plan.steps[i];
        tcec_dispatch_result_t& res = net->step_results[i];
        rc = finish_dispatch(sp.dp, dd[i], sp.m, sp.n, sp.k, &res);
        if (rc) return rc;
        log += res.line;
        log += "\n";
    }
    if (log_lines && log_capacity > 0) {
        const size_t nb = std::min(size_t(log_capacity - 1), log.size());
        std::memcpy(log_lines, log.data(), nb);
        log_lines[nb] = '\0';
    }
    return TCEC_OK;
}

// tcec_profile_read_batches: device time between a batch's uploads and its download
static void account_batch(Handle& h) {
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, h.batch_ev[0], h.batch_ev[1]) == cudaSuccess) {
        h.batch_ms += ms;
        ++h.batch_count;
    }
}

int tcec_contract_selector_batch(tcec_network net, const int* steps, int n_steps,
                                 const tcec_dispatch_config_t* cfg, int n_sel, const int* sel_nodes,
                                 int n_strings, const uint8_t* bits, void* out_host) {
    if (!net || !cfg) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    if (!net->h) return set_error(TCEC_ERR_CUDA, "network has no device handle");
    Handle& h = *net->h;
    cudaSetDevice(h.device);
    for (int q = 0; q < n_sel; ++q) {
        const int nd = sel_nodes[q];
        if (nd < 0 || nd >= int(net->nodes.size()) || net->nodes[size_t(nd)].size() != 2)
            return set_error(TCEC_ERR_SHAPE_MISMATCH, "selector nodes must be rank-1 of extent 2");
    }
    const FoldPlan* plan_ptr = nullptr;
    DevDecision* dec = nullptr;
    void* ws = nullptr;
    int rc = prepare(*net, steps, n_steps, *cfg, &plan_ptr, &dec, &ws);
    if (rc) return rc;
    const FoldPlan& plan = *plan_ptr;
    int64_t size = 1;
    for (auto d : plan.out_dims) size *= d;
    if (size != 1) return set_error(TCEC_ERR_SHAPE_MISMATCH, "amplitude networks must close");
    cudaStream_t s = h.stream;
    int64_t* d_off = nullptr;
    uint8_t* d_bits = nullptr;
    float2* d_out = nullptr;
    std::vector<int64_t> off(size_t(std::max(n_sel, 1)));
    for (int q = 0; q < n_sel; ++q) off[size_t(q)] = net->offset[size_t(sel_nodes[q])];
    const size_t nbits = size_t(n_sel) * size_t(n_strings);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_off), off.size() * 8, s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&d_bits), std::max<size_t>(nbits, 1), s);
    if (e == cudaSuccess)
        e = cudaMallocAsync(reinterpret_cast<void**>(&d_out), size_t(std::max(n_strings, 1)) * 8, s);
    if (e != cudaSuccess) return cuda_error(e, "batch buffers");
    cudaMemcpyAsync(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, s);
    if (nbits) cudaMemcpyAsync(d_bits, bits, nbits, cudaMemcpyHostToDevice, s);
    const bool prof = h.prof && h.batch_ev[0];
    if (prof) cudaEventRecord(h.batch_ev[0], s);
    const std::vector<int> sel_vec(sel_nodes, sel_nodes + n_sel);
    const SmallProgram* fused = small_program(*net, steps, n_steps, *cfg, plan, sel_vec, &rc);
    if (rc) return rc;
    BatchArchive ar;
    rc = ar.begin(plan, n_strings, s);  // (the fused program is eligible only without tensor-core steps)
    if (rc) return rc;
    if (fused) {
        // one launch: one warp per bitstring, selectors built from the bits
        rc = launch_small_program(*fused, static_cast<const float2*>(net->node_dev), n_strings,
                                  nullptr, 0, d_bits, d_out, s);
        if (rc) return rc;
    } else if (n_strings >= 2 && kFoldLanes > 1) {
        // concurrent lanes: bitstring i runs on lane i % L with its own buffers
        const int L = std::min(n_strings, kFoldLanes);
        rc = ensure_lanes(*net, L, plan);
        if (rc) return rc;
        cudaEvent_t ready = net->lanes[0].ev;
        cudaEventRecord(ready, s);  // uploads of nodes, offsets and bits are done
        for (int l = 0; l < L; ++l) {
            FoldLane& ln = net->lanes[size_t(l)];
            cudaStreamWaitEvent(ln.s, ready, 0);
            cudaMemcpyAsync(ln.node_dev, net->node_dev, size_t(net->total) * 8, cudaMemcpyDeviceToDevice,
                            ln.s);
        }
        for (int i = 0; i < n_strings; ++i) {
            FoldLane& ln = net->lanes[size_t(i % L)];
            if (n_sel)
                set_selectors_kernel<<<(n_sel + 127) / 128, 128, 0, ln.s>>>(
                    static_cast<float2*>(ln.node_dev), d_off, n_sel, d_bits + size_t(i) * n_sel);
            rc = run_fold_lane(*net, ln, steps, n_steps, *cfg, plan);
            if (rc) return rc;
            ar.record(ln.dec, i, ln.s);
            cudaMemcpyAsync(d_out + i, ln.result_dev, 8, cudaMemcpyDeviceToDevice, ln.s);
        }
        for (int l = 0; l < L; ++l) {
            FoldLane& ln = net->lanes[size_t(l)];
            cudaEventRecord(ln.ev, ln.s);
            cudaStreamWaitEvent(s, ln.ev, 0);
        }
    } else {
        for (int i = 0; i < n_strings; ++i) {
            if (n_sel)
                set_selectors_kernel<<<(n_sel + 127) / 128, 128, 0, s>>>(
                    static_cast<float2*>(net->node_dev), d_off, n_sel, d_bits + size_t(i) * n_sel);
            rc = run_fold(*net, steps, n_steps, *cfg, plan, dec, ws, true);
            if (rc) return rc;
            ar.record(dec, i, s);
            cudaMemcpyAsync(d_out + i, net->result_dev, 8, cudaMemcpyDeviceToDevice, s);
        }
    }
    if (prof) cudaEventRecord(h.batch_ev[1], s);
    e = cudaMemcpyAsync(out_host, d_out, size_t(n_strings) * 8, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_error(e, "batch download");
    rc = ar.download(&net->batch_dec, s);
    if (rc) return rc;
    ar.release(s);
    cudaFreeAsync(d_off, s);
    cudaFreeAsync(d_bits, s);
    cudaFreeAsync(d_out, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_error(e, "selector batch");
    if (prof) account_batch(h);
    // the host copy of the selector slots no longer matches the device
    net->dirty = true;
    return settle_batch(*net, ar);
}

int tcec_contract_node_batch(tcec_network net, const int* steps, int n_steps,
                             const tcec_dispatch_config_t* cfg, int n_var, const int* var_nodes,
                             int n_runs, const void* var_data, void* out_host) {
    if (!net || !cfg) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    if (!net->h) return set_error(TCEC_ERR_CUDA, "network has no device handle");
    Handle& h = *net->h;
    cudaSetDevice(h.device);
    std::vector<int64_t> seg;
    int64_t per_run = 0;
    for (int i = 0; i < n_var; ++i) {
        const int nd = var_nodes[i];
        if (nd < 0 || nd >= int(net->nodes.size()))
            return set_error(TCEC_ERR_INVALID_ARGUMENT, "bad variable node index");
        const int64_t cnt = net->nodes[size_t(nd)].size();
        seg.push_back(net->offset[size_t(nd)]);
        seg.push_back(per_run);
        seg.push_back(cnt);
        per_run += cnt;
    }
    const FoldPlan* plan_ptr = nullptr;
    DevDecision* dec = nullptr;
    void* ws = nullptr;
    int rc = prepare(*net, steps, n_steps, *cfg, &plan_ptr, &dec, &ws);
    if (rc) return rc;
    const FoldPlan& plan = *plan_ptr;
    int64_t size = 1;
    for (auto d : plan.out_dims) size *= d;
    if (size != 1) return set_error(TCEC_ERR_SHAPE_MISMATCH, "batched networks must close");
    cudaStream_t s = h.stream;
    int64_t* d_seg = nullptr;
    float2* d_var = nullptr;
    float2* d_out = nullptr;
    const size_t var_bytes = size_t(std::max<int64_t>(per_run * n_runs, 1)) * 8;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_seg), std::max<size_t>(seg.size(), 1) * 8, s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&d_var), var_bytes, s);
    if (e == cudaSuccess)
        e = cudaMallocAsync(reinterpret_cast<void**>(&d_out), size_t(std::max(n_runs, 1)) * 8, s);
    if (e != cudaSuccess) return cuda_error(e, "batch buffers");
    if (!seg.empty()) cudaMemcpyAsync(d_seg, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice, s);
    if (per_run * n_runs > 0)
        cudaMemcpyAsync(d_var, var_data, size_t(per_run * n_runs) * 8, cudaMemcpyHostToDevice, s);
    const bool prof = h.prof && h.batch_ev[0];
    if (prof) cudaEventRecord(h.batch_ev[0], s);
    const std::vector<int> var_vec(var_nodes, var_nodes + n_var);
    const SmallProgram* fused = small_program(*net, steps, n_steps, *cfg, plan, var_vec, &rc);
    if (rc) return rc;
    BatchArchive ar;
    rc = ar.begin(plan, n_runs, s);
    if (rc) return rc;
    if (fused) {
        rc = launch_small_program(*fused, static_cast<const float2*>(net->node_dev), n_runs, d_var,
                                  per_run, nullptr, d_out, s);
        if (rc) return rc;
    } else if (n_runs >= 2 && node_batch_lanes() > 1) {
        // concurrent lanes (slices of a sliced contraction): run r on lane r % L
        const int L = std::min(n_runs, node_batch_lanes());
        rc = ensure_lanes(*net, L, plan);
        if (rc) return rc;
        cudaEvent_t ready = net->lanes[0].ev;
        cudaEventRecord(ready, s);
        for (int l = 0; l < L; ++l) {
            FoldLane& ln = net->lanes[size_t(l)];
            cudaStreamWaitEvent(ln.s, ready, 0);
            cudaMemcpyAsync(ln.node_dev, net->node_dev, size_t(net->total) * 8, cudaMemcpyDeviceToDevice,
                            ln.s);
        }
        for (int r = 0; r < n_runs; ++r) {
            FoldLane& ln = net->lanes[size_t(r % L)];
            if (n_var)
                scatter_nodes_kernel<<<std::min(n_var, 1024), 64, 0, ln.s>>>(
                    static_cast<float2*>(ln.node_dev), d_var + size_t(r) * size_t(per_run), d_seg,
                    n_var);
            rc = run_fold_lane(*net, ln, steps, n_steps, *cfg, plan);
            if (rc) return rc;
            ar.record(ln.dec, r, ln.s);
            cudaMemcpyAsync(d_out + r, ln.result_dev, 8, cudaMemcpyDeviceToDevice, ln.s);
        }
        for (int l = 0; l < L; ++l) {
            FoldLane& ln = net->lanes[size_t(l)];
            cudaEventRecord(ln.ev, ln.s);
            cudaStreamWaitEvent(s, ln.ev, 0);
        }
    } else {
        for (int r = 0; r < n_runs; ++r) {
            if (n_var)
                scatter_nodes_kernel<<<std::min(n_var, 1024), 64, 0, s>>>(
                    static_cast<float2*>(net->node_dev), d_var + size_t(r) * size_t(per_run), d_seg,
                    n_var);
            rc = run_fold(*net, steps, n_steps, *cfg, plan, dec, ws, true);
            if (rc) return rc;
            ar.record(dec, r, s);
            cudaMemcpyAsync(d_out + r, net->result_dev, 8, cudaMemcpyDeviceToDevice, s);
        }
    }
    if (prof) cudaEventRecord(h.batch_ev[1], s);
    e = cudaMemcpyAsync(out_host, d_out, size_t(n_runs) * 8, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_error(e, "batch download");
    rc = ar.download(&net->batch_dec, s);
    if (rc) return rc;
    ar.release(s);
    cudaFreeAsync(d_seg, s);
    cudaFreeAsync(d_var, s);
    cudaFreeAsync(d_out, s);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_error(e, "node batch");
    if (prof) account_batch(h);
    net->dirty = true;  // device node data now holds the last run
    return settle_batch(*net, ar);
}

int tcec_network_step_results(tcec_network net, tcec_dispatch_result_t* out, int capacity, int* count) {
    if (!net || (capacity > 0 && !out)) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    const int n = int(net->step_results.size());
    for (int i = 0; i < n && i < capacity; ++i) out[i] = net->step_results[size_t(i)];
    if (count) *count = std::min(n, capacity);
    return TCEC_OK;
}

// contract_network_oracle (network.cpp:179-186): the same TTGT fold with every
// value widened to complex128 and f64 GEMMs in the reference's order
// (gemm_rows_dd), on the device; the result tensor goes to out_host (c128).
int tcec_contract_network_oracle(tcec_network net, const int* steps, int n_steps, void* out_host,
                                 int64_t out_capacity, int* out_rank, int* out_labels) {
    if (!net) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null argument");
    if (!net->h) return set_error(TCEC_ERR_CUDA, "network has no device handle");
    Handle& h = *net->h;
    cudaSetDevice(h.device);
    int rc = validate(*net);
    if (rc) return rc;
    tcec_dispatch_config_t cfg;
    tcec_default_config(&cfg);
    cfg.force = TCEC_FORCE_FP64_ORACLE;
    FoldPlan plan;
    rc = build_plan(*net, steps, n_steps, cfg, &plan);
    if (rc) return rc;
    int64_t size = 1;
    for (auto d : plan.out_dims) size *= d;
    if (out_capacity < size) return set_error(TCEC_ERR_SHAPE_MISMATCH, "output buffer too small");
    rc = upload(*net);
    if (rc) return rc;
    cudaStream_t s = h.stream;
    std::map<int, double2*> live;
    std::vector<void*> owned;
    auto alloc = [&](int64_t elems, double2** p) {
        const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p),
                                              size_t(std::max<int64_t>(elems, 1)) * 16, s);
        if (e != cudaSuccess) return cuda_error(e, "f64 contraction buffer");
        return int(TCEC_OK);
    };
    const float2* base = static_cast<const float2*>(net->node_dev);
    for (size_t i = 0; i < net->nodes.size(); ++i) {
        double2* w = nullptr;
        if ((rc = alloc(net->nodes[i].size(), &w))) return rc;
        launch_widen(base + net->offset[i], w, net->nodes[i].size(), s);
        live[int(i)] = w;
    }
    int next_id = int(net->nodes.size());
    for (const StepPlan& sp : plan.steps) {
        double2* pa = live[sp.ia];
        double2* pb = live[sp.ib];
        double2 *ta = nullptr, *tb = nullptr, *pc = nullptr;
        if (sp.perm_a) {
            if ((rc = alloc(sp.a_size, &ta))) return rc;
            launch_permute_c128(pa, ta, int(sp.a_dims.size()), sp.a_dims.data(), sp.a_axis.data(), s);
        }
        if (sp.perm_b) {
            if ((rc = alloc(sp.b_size, &tb))) return rc;
            launch_permute_c128(pb, tb, int(sp.b_dims.size()), sp.b_dims.data(), sp.b_axis.data(), s);
        }
        if ((rc = alloc(sp.m * sp.n, &pc))) return rc;
        launch_cgemm_c128(ta ? ta : pa, false, tb ? tb : pb, false, pc, sp.m, sp.n, sp.k, s);
        if (ta) cudaFreeAsync(ta, s);
        if (tb) cudaFreeAsync(tb, s);
        cudaFreeAsync(pa, s);
        cudaFreeAsync(pb, s);
        live.erase(sp.ia);
        live.erase(sp.ib);
        live[next_id++] = pc;
    }
    double2* res = live.begin()->second;
    cudaError_t e = cudaMemcpyAsync(out_host, res, size_t(size) * 16, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(res, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_error(e, "contract_network_oracle");
    if (out_rank) *out_rank = int(plan.out_labels.size());
    if (out_labels) std::copy(plan.out_labels.begin(), plan.out_labels.end(), out_labels);
    return TCEC_OK;
}

int tcec_network_batch_run_info(tcec_network net, int run, int* overflow, char* log_lines,
                                int64_t log_capacity) {
    if (!net) return set_error(TCEC_ERR_INVALID_ARGUMENT, "null network");
    if (run < 0 || run >= net->batch_runs || net->batch_plan_key != net->plan_key)
        return set_error(TCEC_ERR_INVALID_ARGUMENT, "no such run in the last batch");
    const FoldPlan& plan = net->plan_cache;
    const size_t nt = net->batch_tc.size();
    int ovf = 0;
    std::string log;
    size_t ti = 0;
    for (size_t i = 0; i < plan.steps.size(); ++i) {
        const StepPlan& sp = plan.steps[i];
        DevDecision d{};
        if (ti < nt && net->batch_tc[ti] == int(i)) d = net->batch_dec[size_t(run) * nt + ti++];
        tcec_dispatch_result_t res;
        const int rc = finish_dispatch(sp.dp, d, sp.m, sp.n, sp.k, &res);
        if (rc) return rc;
        ovf |= res.overflow;
        log += res.line;
        log += "\n";
    }
    if (overflow) *overflow = ovf;
    if (log_lines && log_capacity > 0) {
        const size_t nb = std::min(size_t(log_capacity - 1), log.size());
        std::memcpy(log_lines, log.data(), nb);
        log_lines[nb] = '\0';
    }
    return TCEC_OK;
}

}  // extern "C"
