// Fused small-step contraction: one warp per network instance, intermediates
// in shared memory, one launch for a whole batch of bitstrings / slices.
//
// The 4x4 RCS networks of BASELINE.json configs[0] are 167 pairwise
// contractions whose GEMMs are at most 4x4 (14.6 kflop per
// amplitude).  Launch latency, not flops or bytes, bounds them on a GPU, so
// instead of one graph node per permute / GEMM the whole fold (network.cpp:
// 149-168) runs inside one warp: each step gathers its operands through
// host-computed permutation tables (the TTGT permutes of tensor.hpp:56-105,
// never materialized) and evaluates the reference FP32 schedule exactly
// (four RN chains in ascending k, then (P1 - P2, P3 + P4): kernels_scalar.cpp:
// 76-87, cgemm.cpp:33-44), so amplitudes are bit-identical to the reference.
#include <algorithm>
#include <cstring>
#include <map>

#include "network_plan.h"

namespace tcec {

void SmallProgram::release() {
    if (d_steps) cudaFree(d_steps);
    if (d_tables) cudaFree(d_tables);
    if (d_var) cudaFree(d_var);
    d_steps = nullptr;
    d_tables = nullptr;
    d_var = nullptr;
}

namespace {

// permuted-matrix position -> source element offset (the odometer of
// tensor.hpp:93-103)
void gather_table(const std::vector<int64_t>& dims, const std::vector<int>& axis_of,
                  std::vector<int32_t>* out) {
    const int r = int(dims.size());
    int64_t total = 1;
    for (auto d : dims) total *= d;
    if (r == 0) {
        out->push_back(0);
        return;
    }
    const size_t ur = static_cast<size_t>(r);
    std::vector<int64_t> old_stride(ur, 1), nd(ur, 0), st(ur, 0), idx(ur, 0);
    for (int a = r - 2; a >= 0; --a) old_stride[size_t(a)] = old_stride[size_t(a + 1)] * dims[size_t(a + 1)];
    for (int a = 0; a < r; ++a) {
        nd[size_t(a)] = dims[size_t(axis_of[size_t(a)])];
        st[size_t(a)] = old_stride[size_t(axis_of[size_t(a)])];
    }
    int64_t off = 0;
    for (int64_t pos = 0; pos < total; ++pos) {
        out->push_back(int32_t(off));
        for (int a = r - 1; a >= 0; --a) {
            if (++idx[size_t(a)] < nd[size_t(a)]) {
                off += st[size_t(a)];
                break;
            }
            off -= st[size_t(a)] * (nd[size_t(a)] - 1);
            idx[size_t(a)] = 0;
        }
    }
}

// first-fit allocator over the warp arena
struct Arena {
    std::map<int64_t, int64_t> free_;  // offset -> size
    int64_t top = 0;
    int64_t alloc(int64_t n) {
        for (auto it = free_.begin(); it != free_.end(); ++it) {
            if (it->second >= n) {
                const int64_t off = it->first;
                const int64_t rest = it->second - n;
                free_.erase(it);
                if (rest) free_[off + n] = rest;
                return off;
            }
        }
        const int64_t off = top;
        top += n;
        return off;
    }
    void release(int64_t off, int64_t n) {
        auto it = free_.emplace(off, n).first;
        auto nx = std::next(it);
        if (nx != free_.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            free_.erase(nx);
        }
        if (it != free_.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                free_.erase(it);
            }
        }
    }
};

constexpr int64_t kMaxArenaBytes = 200 * 1024;
constexpr int64_t kMaxTableEntries = int64_t(1) << 24;

}  // namespace

void build_small_program(const std::vector<NetNode>& nodes, const std::vector<int64_t>& node_offset,
                         const FoldPlan& plan, const std::vector<int>& var_nodes,
                         SmallProgram* out) {
    SmallProgram p;
    // where every live tensor sits: (kind, offset, size); inputs start in global
    struct Loc {
        int kind;
        int64_t off, size;
    };
    std::map<int, Loc> live;
    for (size_t i = 0; i < nodes.size(); ++i)
        live[int(i)] = {0, node_offset[i], nodes[i].size()};
    Arena arena;
    for (int v : var_nodes) {
        const int64_t sz = nodes[size_t(v)].size();
        const int64_t off = arena.alloc(sz);
        live[v] = {1, off, sz};
        p.var_arena.push_back(off);
        p.var_count.push_back(sz);
    }
    int next_id = int(nodes.size());
    for (const StepPlan& sp : plan.steps) {
        if (sp.dp.tier != kTierFp32 && sp.dp.tier != kTierFp64) {
            p.why = "a step runs on a tensor-core tier";
            *out = std::move(p);
            return;
        }
        const Loc la = live.at(sp.ia), lb = live.at(sp.ib);
        SmallStepDev st{};
        st.m = int32_t(sp.m);
        st.n = int32_t(sp.n);
        st.k = int32_t(sp.k);
        st.tier = sp.dp.tier == kTierFp64 ? 1 : 0;
        st.a_kind = la.kind;
        st.b_kind = lb.kind;
        st.a_off = la.off;
        st.b_off = lb.off;
        st.ta = int32_t(p.tables.size());
        gather_table(sp.a_dims, sp.a_axis, &p.tables);
        st.tb = int32_t(p.tables.size());
        gather_table(sp.b_dims, sp.b_axis, &p.tables);
        if (int64_t(p.tables.size()) > kMaxTableEntries) {
            p.why = "gather tables too large";
            *out = std::move(p);
            return;
        }
        const int64_t osz = std::max<int64_t>(sp.m * sp.n, 1);
        const int64_t ooff = arena.alloc(osz);  // before releasing the operands
        st.out_off = int32_t(ooff);
        if (la.kind == 1) arena.release(la.off, la.size);
        if (lb.kind == 1) arena.release(lb.off, lb.size);
        live.erase(sp.ia);
        live.erase(sp.ib);
        live[next_id++] = {1, ooff, osz};
        p.steps.push_back(st);
        if (arena.top * 8 > kMaxArenaBytes) {
            p.why = "live intermediates exceed the shared-memory arena";
            *out = std::move(p);
            return;
        }
    }
    const Loc res = live.begin()->second;
    if (res.kind != 1) {
        // a single-node network: the result is an input; copy via a trivial plan
        p.why = "no contraction steps";
        *out = std::move(p);
        return;
    }
    p.result_off = int32_t(res.off);
    p.result_size = res.size;
    p.arena_elems = std::max<int64_t>(arena.top, 1);
    p.ok = true;
    *out = std::move(p);
}

int upload_small_program(SmallProgram* p) {
    p->release();
    cudaError_t e = cudaMalloc(&p->d_steps, std::max<size_t>(p->steps.size(), 1) * sizeof(SmallStepDev));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_tables, std::max<size_t>(p->tables.size(), 1) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_var, std::max<size_t>(2 * p->var_arena.size(), 1) * 8);
    if (e != cudaSuccess) return cuda_error(e, "small program upload");
    cudaMemcpy(p->d_steps, p->steps.data(), p->steps.size() * sizeof(SmallStepDev), cudaMemcpyHostToDevice);
    cudaMemcpy(p->d_tables, p->tables.data(), p->tables.size() * 4, cudaMemcpyHostToDevice);
    std::vector<int64_t> v = p->var_arena;
    v.insert(v.end(), p->var_count.begin(), p->var_count.end());
    if (!v.empty()) cudaMemcpy(p->d_var, v.data(), v.size() * 8, cudaMemcpyHostToDevice);
    return TCEC_OK;
}

// ------------------------------------------------------------ hybrid program
void HybridProgram::release() {
    if (d_steps) cudaFree(d_steps);
    if (d_tables) cudaFree(d_tables);
    if (d_trees) cudaFree(d_trees);
    d_steps = nullptr;
    d_tables = nullptr;
    d_trees = nullptr;
}

namespace {
constexpr int64_t kHybMaxOut = 1024;          // result elements of a fused step
constexpr int64_t kHybMaxIn = 4096;           // elements of each operand
constexpr int64_t kHybMaxMacs = int64_t(1) << 16;
constexpr int64_t kHybArenaBytes = 16 * 1024;  // per warp (subtree)
constexpr int kHybWarpsPerBlock = 4;
}  // namespace

void build_hybrid_program(const std::vector<NetNode>& nodes, const std::vector<int64_t>& node_offset,
                          const FoldPlan& plan, HybridProgram* out) {
    const int n_nodes = int(nodes.size());
    const int S = int(plan.steps.size());
    std::vector<int> consumer(size_t(S), -1);
    for (int si = 0; si < S; ++si) {
        const StepPlan& sp = plan.steps[size_t(si)];
        if (sp.ia >= n_nodes) consumer[size_t(sp.ia - n_nodes)] = si;
        if (sp.ib >= n_nodes) consumer[size_t(sp.ib - n_nodes)] = si;
    }
    std::vector<char> fusable(size_t(S), 0);
    for (int si = 0; si < S; ++si) {
        const StepPlan& sp = plan.steps[size_t(si)];
        bool ok = (sp.dp.tier == kTierFp32 || sp.dp.tier == kTierFp64) && sp.m * sp.n <= kHybMaxOut &&
                  sp.a_size <= kHybMaxIn && sp.b_size <= kHybMaxIn &&
                  sp.m * sp.n * sp.k <= kHybMaxMacs;
        ok = ok && (sp.ia < n_nodes || fusable[size_t(sp.ia - n_nodes)]);
        ok = ok && (sp.ib < n_nodes || fusable[size_t(sp.ib - n_nodes)]);
        fusable[size_t(si)] = ok;
    }
    HybridProgram p;
    for (;;) {
        p.steps.clear();
        p.tables.clear();
        p.trees.clear();
        p.root_out.assign(size_t(S), -1);
        p.arena_elems = 1;
        p.out_elems = 0;
        int unfuse = -1;
        for (int root = 0; root < S && unfuse < 0; ++root) {
            if (!fusable[size_t(root)]) continue;
            const int c = consumer[size_t(root)];
            if (c >= 0 && fusable[size_t(c)]) continue;  // not a subtree root
            // the subtree: fusable producers reachable from the root
            std::vector<int> members, stack{root};
            while (!stack.empty()) {
                const int s = stack.back();
                stack.pop_back();
                members.push_back(s);
                for (int id : {plan.steps[size_t(s)].ia, plan.steps[size_t(s)].ib})
                    if (id >= n_nodes) stack.push_back(id - n_nodes);
            }
            std::sort(members.begin(), members.end());
            struct Loc {
                int kind;
                int64_t off, size;
            };
            std::map<int, Loc> live;
            Arena arena;
            TreeDev tr{};
            tr.step_begin = int32_t(p.steps.size());
            for (int s : members) {
                const StepPlan& sp = plan.steps[size_t(s)];
                auto loc = [&](int id) -> Loc {
                    if (id < n_nodes) return {0, node_offset[size_t(id)], nodes[size_t(id)].size()};
                    return live.at(id);
                };
                const Loc la = loc(sp.ia), lb = loc(sp.ib);
                SmallStepDev st{};
                st.m = int32_t(sp.m);
                st.n = int32_t(sp.n);
                st.k = int32_t(sp.k);
                st.tier = sp.dp.tier == kTierFp64 ? 1 : 0;
                st.a_kind = la.kind;
                st.b_kind = lb.kind;
                st.a_off = la.off;
                st.b_off = lb.off;
                st.ta = int32_t(p.tables.size());
                gather_table(sp.a_dims, sp.a_axis, &p.tables);
                st.tb = int32_t(p.tables.size());
                gather_table(sp.b_dims, sp.b_axis, &p.tables);
                const int64_t osz = std::max<int64_t>(sp.m * sp.n, 1);
                const int64_t ooff = arena.alloc(osz);
                st.out_off = int32_t(ooff);
                if (la.kind == 1) arena.release(la.off, la.size);
                if (lb.kind == 1) arena.release(lb.off, lb.size);
                live.erase(sp.ia);
                live.erase(sp.ib);
                live[n_nodes + s] = {1, ooff, osz};
                p.steps.push_back(st);
            }
            if (arena.top * 8 > kHybArenaBytes) {
                unfuse = root;
                break;
            }
            const Loc res = live.at(n_nodes + root);
            tr.step_end = int32_t(p.steps.size());
            tr.result_off = int32_t(res.off);
            tr.result_size = res.size;
            tr.out_off = p.out_elems;
            p.root_out[size_t(root)] = p.out_elems;
            p.out_elems += res.size;
            p.arena_elems = std::max(p.arena_elems, arena.top);
            p.trees.push_back(tr);
        }
        if (unfuse < 0) break;
        fusable[size_t(unfuse)] = 0;  // its fused children become roots
    }
    p.fused = fusable;
    p.ok = !p.trees.empty() && int64_t(p.tables.size()) <= kMaxTableEntries;
    *out = std::move(p);
}

int upload_hybrid_program(HybridProgram* p) {
    p->release();
    if (!p->ok) return TCEC_OK;
    cudaError_t e = cudaMalloc(&p->d_steps, std::max<size_t>(p->steps.size(), 1) * sizeof(SmallStepDev));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_tables, std::max<size_t>(p->tables.size(), 1) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_trees, std::max<size_t>(p->trees.size(), 1) * sizeof(TreeDev));
    if (e != cudaSuccess) return cuda_error(e, "hybrid program upload");
    cudaMemcpy(p->d_steps, p->steps.data(), p->steps.size() * sizeof(SmallStepDev), cudaMemcpyHostToDevice);
    cudaMemcpy(p->d_tables, p->tables.data(), p->tables.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(p->d_trees, p->trees.data(), p->trees.size() * sizeof(TreeDev), cudaMemcpyHostToDevice);
    return TCEC_OK;
}

namespace {

constexpr int kBatchFoldMinRuns = 4096;  // thread-per-run kernel from this many runs

// one contraction step by one warp: operands gathered through the step's
// permutation tables, the reference FP32 schedule (or FP64) per output element
__device__ __forceinline__ void warp_step(const SmallStepDev& st, float2* arena,
                                          const float2* __restrict__ nodes,
                                          const int32_t* __restrict__ tab, int lane) {
    const float2* A = st.a_kind ? arena + st.a_off : nodes + st.a_off;
    const float2* B = st.b_kind ? arena + st.b_off : nodes + st.b_off;
    const int32_t* ta = tab + st.ta;
    const int32_t* tb = tab + st.tb;
    const int mn = st.m * st.n;
    for (int o = lane; o < mn; o += 32) {
        const int i = o / st.n, j = o - i * st.n;
        float2 r;
        if (st.tier == 0) {
            float p1 = 0.0f, p2 = 0.0f, p3 = 0.0f, p4 = 0.0f;
            for (int kk = 0; kk < st.k; ++kk) {
                const float2 a = A[ta[i * st.k + kk]];
                const float2 b = B[tb[kk * st.n + j]];
                p1 = __fadd_rn(p1, __fmul_rn(a.x, b.x));
                p2 = __fadd_rn(p2, __fmul_rn(a.y, b.y));
                p3 = __fadd_rn(p3, __fmul_rn(a.x, b.y));
                p4 = __fadd_rn(p4, __fmul_rn(a.y, b.x));
            }
            r = make_float2(__fsub_rn(p1, p2), __fadd_rn(p3, p4));
        } else {
            double p1 = 0.0, p2 = 0.0, p3 = 0.0, p4 = 0.0;
            for (int kk = 0; kk < st.k; ++kk) {
                const float2 a = A[ta[i * st.k + kk]];
                const float2 b = B[tb[kk * st.n + j]];
                p1 = __dadd_rn(p1, __dmul_rn(double(a.x), double(b.x)));
                p2 = __dadd_rn(p2, __dmul_rn(double(a.y), double(b.y)));
                p3 = __dadd_rn(p3, __dmul_rn(double(a.x), double(b.y)));
                p4 = __dadd_rn(p4, __dmul_rn(double(a.y), double(b.x)));
            }
            r = make_float2(__fsub_rn(__double2float_rn(p1), __double2float_rn(p2)),
                            __fadd_rn(__double2float_rn(p3), __double2float_rn(p4)));
        }
        arena[st.out_off + o] = r;
    }
    __syncwarp();
}

// hybrid prologue: one warp per subtree
__global__ void tree_fold_kernel(const SmallStepDev* __restrict__ steps,
                                 const int32_t* __restrict__ tab, const TreeDev* __restrict__ trees,
                                 int n_trees, const float2* __restrict__ nodes, int64_t arena_elems,
                                 float2* __restrict__ out) {
    extern __shared__ float2 tree_arena[];
    const int wic = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    const int t = int(blockIdx.x) * int(blockDim.x >> 5) + wic;
    if (t >= n_trees) return;
    float2* arena = tree_arena + size_t(wic) * size_t(arena_elems);
    const TreeDev tr = trees[t];
    for (int s = tr.step_begin; s < tr.step_end; ++s) warp_step(steps[s], arena, nodes, tab, lane);
    for (int64_t e = lane; e < tr.result_size; e += 32) out[tr.out_off + e] = arena[tr.result_off + e];
}

__global__ void small_fold_kernel(const SmallStepDev* __restrict__ steps, int n_steps,
                                  const int32_t* __restrict__ tab, const float2* __restrict__ nodes,
                                  int n_runs, int64_t arena_elems, const int64_t* __restrict__ var,
                                  int n_var, const float2* __restrict__ var_data, int64_t per_run,
                                  const uint8_t* __restrict__ bits, int32_t result_off,
                                  int64_t result_size, float2* __restrict__ out) {
    extern __shared__ float2 arena_all[];
    const int wic = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    const int64_t run = int64_t(blockIdx.x) * (blockDim.x >> 5) + wic;
    if (run >= n_runs) return;  // the whole warp leaves together
    float2* arena = arena_all + size_t(wic) * size_t(arena_elems);
    const int64_t* var_off = var;
    const int64_t* var_cnt = var + n_var;
    if (bits != nullptr) {
        // <x_q| selectors (qcircuit.cpp:172-178)
        for (int v = lane; v < n_var; v += 32) {
            const bool one = bits[run * n_var + v] != 0;
            arena[var_off[v]] = make_float2(one ? 0.0f : 1.0f, 0.0f);
            arena[var_off[v] + 1] = make_float2(one ? 1.0f : 0.0f, 0.0f);
        }
    } else if (var_data != nullptr) {
        const float2* src = var_data + run * per_run;
        int64_t off = 0;
        for (int v = 0; v < n_var; ++v) {
            for (int64_t e = lane; e < var_cnt[v]; e += 32) arena[var_off[v] + e] = src[off + e];
            off += var_cnt[v];
        }
    }
    __syncwarp();
    for (int s = 0; s < n_steps; ++s) warp_step(steps[s], arena, nodes, tab, lane);
    for (int64_t e = lane; e < result_size; e += 32) out[run * result_size + e] = arena[result_off + e];
}

// Many runs of one small program (all 65536 bitstrings of a 4x4 RQC): one
// THREAD per run instead of one warp, so every lane is busy even on the
// many steps with fewer than 32 outputs.  The arena is structure-of-arrays in
// global memory (element e of run r at e * n_runs + r): the steps are uniform
// across runs, so every arena access of a warp is one coalesced 256-B line and
// every node / table access is a broadcast.  Same per-element arithmetic (the
// reference FP32 chains or FP64) as warp_step -> bit-identical.
__global__ void __launch_bounds__(128) batch_fold_kernel(
    const SmallStepDev* __restrict__ steps, int n_steps, const int32_t* __restrict__ tab,
    const float2* __restrict__ nodes, int n_runs, const int64_t* __restrict__ var, int n_var,
    const float2* __restrict__ var_data, int64_t per_run, const uint8_t* __restrict__ bits,
    int32_t result_off, int64_t result_size, float2* __restrict__ out, float2* __restrict__ arena) {
    const int64_t run = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (run >= n_runs) return;
    const int64_t R = n_runs;
    float2* ar = arena + run;  // element e at ar[e * R]
    const int64_t* var_off = var;
    const int64_t* var_cnt = var + n_var;
    if (bits != nullptr) {
        for (int v = 0; v < n_var; ++v) {
            const bool one = bits[run * n_var + v] != 0;
            ar[var_off[v] * R] = make_float2(one ? 0.0f : 1.0f, 0.0f);
            ar[(var_off[v] + 1) * R] = make_float2(one ? 1.0f : 0.0f, 0.0f);
        }
    } else if (var_data != nullptr) {
        const float2* src = var_data + run * per_run;
        int64_t off = 0;
        for (int v = 0; v < n_var; ++v) {
            for (int64_t e = 0; e < var_cnt[v]; ++e) ar[(var_off[v] + e) * R] = src[off + e];
            off += var_cnt[v];
        }
    }
    for (int s = 0; s < n_steps; ++s) {
        const SmallStepDev st = steps[s];
        const int32_t* ta = tab + st.ta;
        const int32_t* tb = tab + st.tb;
        const int mn = st.m * st.n;
        for (int o = 0; o < mn; ++o) {
            const int i = o / st.n, j = o - i * st.n;
            float2 r;
            if (st.tier == 0) {
                float p1 = 0.0f, p2 = 0.0f, p3 = 0.0f, p4 = 0.0f;
                for (int kk = 0; kk < st.k; ++kk) {
                    const int64_t ia = st.a_off + ta[i * st.k + kk], ib = st.b_off + tb[kk * st.n + j];
                    const float2 a = st.a_kind ? ar[ia * R] : nodes[ia];
                    const float2 b = st.b_kind ? ar[ib * R] : nodes[ib];
                    p1 = __fadd_rn(p1, __fmul_rn(a.x, b.x));
                    p2 = __fadd_rn(p2, __fmul_rn(a.y, b.y));
                    p3 = __fadd_rn(p3, __fmul_rn(a.x, b.y));
                    p4 = __fadd_rn(p4, __fmul_rn(a.y, b.x));
                }
                r = make_float2(__fsub_rn(p1, p2), __fadd_rn(p3, p4));
            } else {
                double p1 = 0.0, p2 = 0.0, p3 = 0.0, p4 = 0.0;
                for (int kk = 0; kk < st.k; ++kk) {
                    const int64_t ia = st.a_off + ta[i * st.k + kk], ib = st.b_off + tb[kk * st.n + j];
                    const float2 a = st.a_kind ? ar[ia * R] : nodes[ia];
                    const float2 b = st.b_kind ? ar[ib * R] : nodes[ib];
                    p1 = __dadd_rn(p1, __dmul_rn(double(a.x), double(b.x)));
                    p2 = __dadd_rn(p2, __dmul_rn(double(a.y), double(b.y)));
                    p3 = __dadd_rn(p3, __dmul_rn(double(a.x), double(b.y)));
                    p4 = __dadd_rn(p4, __dmul_rn(double(a.y), double(b.x)));
                }
                r = make_float2(__fsub_rn(__double2float_rn(p1), __double2float_rn(p2)),
                                __fadd_rn(__double2float_rn(p3), __double2float_rn(p4)));
            }
            ar[(int64_t(st.out_off) + o) * R] = r;
        }
    }
    for (int64_t e = 0; e < result_size; ++e) out[run * result_size + e] = ar[(result_off + e) * R];
}

}  // namespace

int launch_hybrid_trees(const HybridProgram& p, const float2* node_dev, float2* out, cudaStream_t s) {
    if (!p.ok) return TCEC_OK;
    const int n_trees = int(p.trees.size());
    const size_t smem = size_t(kHybWarpsPerBlock) * size_t(p.arena_elems) * 8;
    static std::atomic<uint64_t> attr{0};
    ensure_smem_attr(attr, [] {
        return cudaFuncSetAttribute(tree_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kHybWarpsPerBlock * kHybArenaBytes));
    });
    const unsigned grid = unsigned((n_trees + kHybWarpsPerBlock - 1) / kHybWarpsPerBlock);
    tree_fold_kernel<<<grid, 32 * kHybWarpsPerBlock, smem, s>>>(p.d_steps, p.d_tables, p.d_trees, n_trees,
                                                                node_dev, p.arena_elems, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TCEC_OK : cuda_error(e, "tree_fold_kernel");
}

int launch_small_program(const SmallProgram& p, const float2* node_dev, int n_runs,
                         const float2* var_data, int64_t per_run, const uint8_t* bits, float2* out,
                         cudaStream_t s) {
    if (!p.ok) return set_error(TCEC_ERR_INVALID_ARGUMENT, "small program not eligible: " + p.why);
    if (n_runs <= 0) return TCEC_OK;
    if (n_runs >= kBatchFoldMinRuns) {
        // thread per run, SoA arena in global memory (stream-ordered scratch)
        float2* arena = nullptr;
        const size_t bytes = size_t(n_runs) * size_t(std::max<int64_t>(p.arena_elems, 1)) * 8;
        if (cudaMallocAsync(reinterpret_cast<void**>(&arena), bytes, s) == cudaSuccess) {
            batch_fold_kernel<<<unsigned((n_runs + 127) / 128), 128, 0, s>>>(
                p.d_steps, int(p.steps.size()), p.d_tables, node_dev, n_runs, p.d_var,
                int(p.var_arena.size()), var_data, per_run, bits, p.result_off, p.result_size, out,
                arena);
            cudaFreeAsync(arena, s);
            const cudaError_t e = cudaGetLastError();
            return e == cudaSuccess ? TCEC_OK : cuda_error(e, "batch_fold_kernel");
        }
        cudaGetLastError();  // no room for the SoA arena: fall back to warp-per-run
    }
    const int64_t arena_bytes = p.arena_elems * 8;
    int wpc = int(std::min<int64_t>(8, std::max<int64_t>(1, kMaxArenaBytes / std::max<int64_t>(arena_bytes, 1))));
    wpc = std::min(wpc, std::max(1, n_runs));
    const size_t smem = size_t(wpc) * size_t(arena_bytes);
    static std::atomic<uint64_t> attr{0};
    ensure_smem_attr(attr, [] {
        return cudaFuncSetAttribute(small_fold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kMaxArenaBytes + 8 * 1024));
    });
    const unsigned grid = unsigned((n_runs + wpc - 1) / wpc);
    small_fold_kernel<<<grid, 32 * wpc, smem, s>>>(
        p.d_steps, int(p.steps.size()), p.d_tables, node_dev, n_runs, p.arena_elems, p.d_var,
        int(p.var_arena.size()), var_data, per_run, bits, p.result_off, p.result_size, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TCEC_OK : cuda_error(e, "small_fold_kernel");
}

}  // namespace tcec
