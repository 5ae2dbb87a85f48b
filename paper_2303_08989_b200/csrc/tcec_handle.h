// Handle + dispatch-plan internals shared by the C-ABI translation units.
#pragma once

#include <algorithm>
#include <memory>
#include <string>

#include "../../include/tcec_b200.h"
#include "tcec_common.cuh"
#include "tcec_internal.h"
#include "host_stage.h"

struct tcec_handle_s {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int flush_kblocks = 1;  // RN flush of the main term every k-block (64 f16 / 32 tf32 K')
    int executor = 0;       // network executor: 0 auto, 1 per-step only, 2 fused only
    int gemm_pair = 0;      // tcgen05 kernel variant (tcec_set_gemm_variant): 0 auto, 1 pair, 2 single, 3 wide
    int layout = 0;         // operand layout (tcec_set_operand_layout): 0 auto, 1 B-expanded, 2 A-expanded
    // operand workspace (split hi/lo planes), grown on demand
    void* ws = nullptr;
    size_t ws_bytes = 0;
    // device decisions (one slot per dispatched GEMM of a contraction)
    tcec::DevDecision* dec = nullptr;
    tcec::DevDecision* dec_host = nullptr;  // pinned mirror
    int dec_slots = 0;
    // device staging for the host-buffer entry points
    void* io = nullptr;
    size_t io_bytes = 0;
    void* scratch_host = nullptr;  // pinned 4 KiB
    cudaStream_t copy_stream = nullptr;  // D2H of finished row chunks (host-buffer API)
    cudaEvent_t chunk_ev[8] = {};
    cudaStream_t in_stream = nullptr;  // H2D of operand row chunks (host-buffer pipeline)
    cudaStream_t gemm_stream2 = nullptr;  // second GEMM stream of the host-buffer pipeline
    int64_t pipe_runs = 0, pipe_reruns = 0;  // tcec_host_pipeline_stats
    std::unique_ptr<tcec::StageRing> stage;  // pinned ring for pageable host buffers
    cudaEvent_t in_ev[41] = {};  // B parts (<= 8), A chunks (<= 32), ordering
    // stage profiling (tcec_profile_*): CUDA events around the stages of a
    // dispatched CGEMM, accumulated after each synchronous dispatch
    bool prof = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    double prof_ms[3] = {0.0, 0.0, 0.0};  // statistics+selection, operand prep, GEMM
    int64_t prof_count = 0;
    // contraction batches (selector / node batch): device time from the end of
    // the uploads to the start of the download, while profiling is enabled
    cudaEvent_t batch_ev[2] = {nullptr, nullptr};
    double batch_ms = 0.0;
    int64_t batch_count = 0;

    // replayable graphs of small device-pointer dispatches (tcec_dispatch_cgemm):
    // the whole launch sequence of one (pointers, shape, config) as one graph
    // launch instead of ~7 host-enqueued operations
    struct DispatchGraph {
        const void *a, *b;
        void *c, *ws, *dec;
        int64_t m, n, k;
        double t;
        int64_t size_auto, size_tf32;
        int target, k_tile, force, variant, flush, layout;
        cudaStream_t stream;
        cudaGraphExec_t exec;
    };
    DispatchGraph graphs[8] = {};
    int n_graphs = 0, next_graph = 0;

    void drop_graphs();
    void* workspace(size_t bytes);
    tcec::DevDecision* decisions(int slots);
    ~tcec_handle_s();
};

namespace tcec {

using Handle = tcec_handle_s;

int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);

enum Tier : int { kTierInvalid = -1, kTierFp32 = 0, kTierFp64 = 1, kTierTc = 2 };

struct DispatchPlan {
    int tier = kTierInvalid;
    int kind = -1;          // host-known ComputeKind, -1 = decided on the device
    int kind_known = -1;    // kind for reporting when the host knows it
    int forced = -1;        // ForcedMode or -1
    int corrected = 1;      // TCEC (1) or uncorrected TC ablation (0)
    bool stats = false;     // statistics on the device
    bool forced_scaled = false;
    int64_t kp = 0;         // padded 2k
    const char* label = "";
};

DispatchPlan plan_dispatch(int64_t m, int64_t n, int64_t k, const tcec_dispatch_config_t& cfg);
size_t plan_workspace(const DispatchPlan& p, int64_t m, int64_t n);
// Optional row-chunk hook of launch_dispatch: the GEMM of a tensor-core
// dispatch is launched in `chunks` row blocks and done(r0, r1) is called after
// each block is enqueued (the host-buffer entry point overlaps the D2H copy of
// finished rows with the GEMM of the next ones).
struct ChunkHook {
    int chunks = 1;
    int (*done)(void* ctx, int64_t r0, int64_t r1) = nullptr;
    void* ctx = nullptr;
};
// va / vb (tensor-core tier only): the operand is the unpermuted tensor read
// through a matrix view by the preparation kernels (fused TTGT gather; the
// statistics are order-free and sweep the tensor as is)
int launch_dispatch(Handle& h, const float* a, const float* b, float* c, int64_t m, int64_t n,
                    int64_t k, const tcec_dispatch_config_t& cfg, const DispatchPlan& p,
                    DevDecision* d, void* ws, const ChunkHook* hook = nullptr,
                    const MatrixView* va = nullptr, const MatrixView* vb = nullptr);
int finish_dispatch(const DispatchPlan& p, const DevDecision& dd, int64_t m, int64_t n, int64_t k,
                    tcec_dispatch_result_t* res);
void format_line(char* out, size_t cap, int64_t m, int64_t n, int64_t k, const char* label, int sa,
                 int sb, const tcec_exp_stats_t* a, const tcec_exp_stats_t* b, bool has);
const char* kind_name(int kind);
const char* forced_name(int f);

}  // namespace tcec
