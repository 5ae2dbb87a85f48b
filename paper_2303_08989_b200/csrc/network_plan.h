// Host-side contraction plan shared by the per-step executor (network.cu) and
// the fused small-step executor (small_fold.cu).
#pragma once

#include <string>
#include <vector>

#include "tcec_handle.h"

namespace tcec {

struct NetNode {
    std::vector<int> labels;
    std::vector<int64_t> dims;
    int64_t size() const {
        int64_t s = 1;
        for (auto d : dims) s *= d;
        return s;
    }
};

// one ttgt_contract step (network.cpp:58-85)
struct StepPlan {
    int ia = 0, ib = 0;
    int64_t m = 1, n = 1, k = 1;
    bool perm_a = false, perm_b = false;
    std::vector<int64_t> a_dims, b_dims;
    std::vector<int> a_axis, b_axis;  // new axis -> old axis (free_a|shared, shared|free_b)
    int64_t a_size = 1, b_size = 1;
    int n_shared = 0;
    DispatchPlan dp;
    // fused TTGT gather: a skinny FP32-tier step reads its long operand through
    // a strided view of the unpermuted tensor instead of a permuted copy
    bool view_a = false, view_b = false;
    MatrixView view;
    // the same for tensor-core steps: the preparation kernels read either
    // operand through a view (the statistics sweep the unpermuted tensor)
    bool tview_a = false, tview_b = false;
    MatrixView tva, tvb;
};

struct FoldPlan {
    std::vector<StepPlan> steps;
    std::vector<int> out_labels;
    std::vector<int64_t> out_dims;
    size_t ws_bytes = 0;
};

// ---------------------------------------------------------------- fused path
// One warp contracts one whole network (one bitstring / one slice) with every
// intermediate in shared memory; operand permutations are gather tables.
// Eligible when every step is on a SIMT tier (FP32_REF / FP64) and the live
// intermediates fit in shared memory.
struct SmallStepDev {
    int32_t m, n, k, tier;    // tier: 0 FP32 reference chains, 1 FP64
    int32_t a_kind, b_kind;   // 0 = input node buffer (global), 1 = warp arena (smem)
    int64_t a_off, b_off;     // element offsets
    int32_t out_off;          // arena element offset of the result
    int32_t ta, tb;           // gather-table offsets (A: m*k, B: k*n entries)
    int32_t pad_;
};

struct SmallProgram {
    bool ok = false;
    std::string why;                  // reason when not eligible
    std::vector<SmallStepDev> steps;
    std::vector<int32_t> tables;
    std::vector<int64_t> var_arena;   // arena offset of each variable node
    std::vector<int64_t> var_count;   // its element count
    int64_t arena_elems = 0;
    int32_t result_off = 0;
    int64_t result_size = 1;
    // device copies
    SmallStepDev* d_steps = nullptr;
    int32_t* d_tables = nullptr;
    int64_t* d_var = nullptr;         // var_arena then var_count
    std::string key;
    void release();
};

// ---------------------------------------------------------------- hybrid path
// For networks the fused path cannot take whole (tensor-core steps, or
// intermediates beyond shared memory), the per-step executor first runs every
// maximal subtree of tiny SIMT steps (gate-absorption steps: a few to a few
// hundred flops each) in ONE launch, one warp per subtree with its
// intermediates in shared memory, writing each subtree's root tensor to a
// device buffer; the per-step loop then skips those steps.  Same arithmetic
// per step as the per-step SIMT kernels (reference FP32 chains / FP64), so the
// result is bit-identical to the pure per-step fold.
struct TreeDev {
    int32_t step_begin, step_end;  // range in HybridProgram::steps
    int32_t result_off;            // arena offset of the root tensor
    int32_t pad_;
    int64_t result_size;
    int64_t out_off;               // element offset in the subtree-output buffer
};

struct HybridProgram {
    bool ok = false;                 // at least one step is fused
    std::vector<char> fused;         // per plan step: runs in the subtree launch
    std::vector<int64_t> root_out;   // per plan step: output offset if a root, else -1
    std::vector<SmallStepDev> steps;
    std::vector<int32_t> tables;
    std::vector<TreeDev> trees;
    int64_t arena_elems = 0;         // max over trees
    int64_t out_elems = 0;
    SmallStepDev* d_steps = nullptr;
    int32_t* d_tables = nullptr;
    TreeDev* d_trees = nullptr;
    std::string key;
    void release();
};

void build_hybrid_program(const std::vector<NetNode>& nodes, const std::vector<int64_t>& node_offset,
                          const FoldPlan& plan, HybridProgram* out);
int upload_hybrid_program(HybridProgram* p);
int launch_hybrid_trees(const HybridProgram& p, const float2* node_dev, float2* out, cudaStream_t s);

// Build the fused program for `plan` with `var_nodes` held in the arena.
void build_small_program(const std::vector<NetNode>& nodes, const std::vector<int64_t>& node_offset,
                         const FoldPlan& plan, const std::vector<int>& var_nodes,
                         SmallProgram* out);
int upload_small_program(SmallProgram* p);
// Launch: n_runs networks; variable-node data either from var_data (per run,
// concatenated in var order) or, when bits != nullptr, rank-1 selectors <x_q|.
int launch_small_program(const SmallProgram& p, const float2* node_dev, int n_runs,
                         const float2* var_data, int64_t per_run, const uint8_t* bits, float2* out,
                         cudaStream_t s);

}  // namespace tcec
