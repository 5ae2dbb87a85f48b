/*
 * tcec_b200.h -- C-ABI boundary of the B200-native TCEC tensor-network path.
 *
 * One shared library, paper_2303_08989_b200/libtcec_b200.so (sm_100a CUDA
 * kernels + the C++ host orchestration), exports exactly these symbols.  They
 * replace the reference mpsgemm entry points (/root/reference/proj/include/
 * mpsgemm/<name>.hpp) for the north-star path; each declaration cites the interface
 * it replaces.  Plain pointers and sizes only: "device" buffers are CUDA device
 * pointers (e.g. from torch or cudaMalloc); "host" buffers are ordinary memory.
 * Complex data is interleaved (re, im) float32, row-major, exactly the layout
 * of Matrix<std::complex<float>> (matrix.hpp:11-35) and Tensor (tensor.hpp:16-53).
 *
 * Errors: every function returns a tcec_status (0 = OK).  The codes map 1:1
 * onto the reference exception taxonomy (common.hpp:9-41) and
 * tcec_last_error() returns the message (same prefixes as the reference).
 * There is no CPU fallback: on a machine without an sm_100 GPU every compute
 * entry point fails with TCEC_ERR_CUDA.
 *
 * Threading: a handle owns its stream, workspace and decision buffers; use one
 * handle per host thread (reference functions are reentrant, precsel.hpp:105-123).
 */
#ifndef TCEC_B200_H
#define TCEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
typedef enum {
    TCEC_OK = 0,
    TCEC_ERR_SHAPE_MISMATCH = 1,      /* ShapeMismatch        common.hpp:10 */
    TCEC_ERR_ZERO_REFERENCE = 2,      /* ZeroReference        common.hpp:13 */
    TCEC_ERR_SCALE_OVERFLOW = 3,      /* ScaleOverflow        common.hpp:18 */
    TCEC_ERR_INVALID_PERMUTATION = 4, /* InvalidPermutation   common.hpp:23 */
    TCEC_ERR_EXTENT_MISMATCH = 5,     /* ExtentMismatch       common.hpp:26 */
    TCEC_ERR_INVALID_PATH = 6,        /* InvalidPath          common.hpp:29 */
    TCEC_ERR_DISCONNECTED = 7,        /* DisconnectedNetwork  common.hpp:32 */
    TCEC_ERR_INVALID_ARGUMENT = 8,    /* std::invalid_argument (gemm.cpp:19, k_tile < 1) */
    TCEC_ERR_LOGIC = 9,               /* std::logic_error (precsel.cpp:117-118) */
    TCEC_ERR_CUDA = 10,               /* device / driver failure (no fallback) */
    TCEC_ERR_TOO_MANY_QUBITS = 11     /* TooManyQubits        common.hpp:39 */
} tcec_status;

typedef struct tcec_handle_s* tcec_handle;

/* message of the last failure on this thread ("" if none) */
const char* tcec_last_error(void);
/* library build string (arch, kernel variants) */
const char* tcec_version(void);

/* create a handle bound to a CUDA device; it owns a non-blocking stream */
int tcec_create(int device, tcec_handle* out);
int tcec_destroy(tcec_handle h);
/* run subsequent work on a caller stream (cudaStream_t; NULL = the handle's own) */
int tcec_set_stream(tcec_handle h, void* stream);
void* tcec_get_stream(tcec_handle h);
int tcec_synchronize(tcec_handle h);
/* RN flush interval of the TCEC main term in k-blocks of 64 (f16) / 32 (tf32)
 * elements; 0 = accumulate the whole K inside the tensor core.  This is the
 * device counterpart of TilingConfig::k_tile (gemm.hpp:28-30). */
int tcec_set_flush_kblocks(tcec_handle h, int kblocks);
int tcec_get_flush_kblocks(tcec_handle h);
/* tensor-core kernel variant: 0 = auto (default: wide when its tiles fill the
 * SMs, else single), 1 = CTA pair (cta_group::2, 256 x 128 tile), 2 = single
 * CTA (128 x 128 tile), 3 = wide CTA pair (cta_group::2, 256 x 256 tile),
 * 4 = the wide tile on persistent CTA pairs, 5 = the wide tile on clusters of
 * two CTA pairs that share each B' tile by TMA multicast, 6 = 256 x 128 tiles
 * on persistent CTA pairs with two tiles' accumulators in TMEM (one tile's
 * epilogue overlaps the next tile's MMAs) */
int tcec_set_gemm_variant(tcec_handle h, int variant);
/* operand layout of tensor-core dispatches: the complex GEMM runs as one real
 * GEMM in which one operand carries the 2x2 complex block expansion.
 * 0 = auto (default: expand the smaller operand -- A when m < n),
 * 1 = B-expanded (A' = A as m x 2k, B' = [[Br, Bi], [-Bi, Br]], 2n columns),
 * 2 = A-expanded (A'' rows (Ar, -Ai) / (Ai, Ar), 2m rows; B'' = B^T as n x 2k).
 * Results are FP32-level either way (same products, hardware accumulation
 * order); the choice only changes bytes moved.  No reference counterpart
 * (its cgemm deinterleaves into four real GEMMs, cgemm.cpp:25-46). */
int tcec_set_operand_layout(tcec_handle h, int layout);
int tcec_get_operand_layout(tcec_handle h);
/* network executor: 0 = auto (fused small-step kernel -- one warp per network,
 * intermediates in shared memory -- whenever every step is on a SIMT tier and
 * the live intermediates fit; else the per-step fold -- permute + dispatch
 * through a captured CUDA graph -- preceded by one launch that contracts every
 * subtree of tiny SIMT steps, one warp per subtree), 1 = per-step only,
 * 2 = fused only (error if ineligible), 3 = per-step + subtree launch */
int tcec_set_executor(tcec_handle h, int policy);
/* stage tracing (the device counterpart of DecisionRecord::wall_ms,
 * precsel.hpp:92-101): when enabled, every synchronous tcec_dispatch_cgemm
 * records CUDA events around (statistics + selection), (operand preparation)
 * and (tensor-core / SIMT GEMM) on the handle stream; read returns the summed
 * milliseconds of the three stages and the number of dispatches; enable resets. */
int tcec_profile_enable(tcec_handle h, int on);
int tcec_profile_read(tcec_handle h, double* stage_ms, int64_t* count);
/* the same for contraction batches (tcec_contract_selector_batch / node_batch):
 * summed device milliseconds from the end of the call's uploads to the start of
 * its download (inputs resident in HBM), and the number of batches. */
int tcec_profile_read_batches(tcec_handle h, double* ms, int64_t* count);
/* host-buffer pipeline counters (tcec_dispatch_cgemm_host on large tensor-core
 * dispatches): runs = dispatches that overlapped the operand copies with the
 * GEMM under a decision taken from the first operand parts; reruns = those
 * whose exact decision differed and were recomputed on the plain path. */
int tcec_host_pipeline_stats(tcec_handle h, int64_t* runs, int64_t* reruns);

/* ------------------------------------------------ format emulation (device)
 * KernelTable entries, kernels.hpp:20-63; bit-identical to the reference
 * scalar table.  fmt: 0 = FP16, 1 = TF32 (lowprec.hpp:15); rounding: 0 = RN,
 * 1 = RZ (lowprec.hpp:13).  *overflow (host, may be NULL) is OR-accumulated. */
int tcec_quantize_buf(tcec_handle h, const float* src, float* dst, int64_t n, int fmt,
                      int rounding, int* overflow);
int tcec_split_buf(tcec_handle h, const float* src, float* hi, float* lo, int64_t n, int fmt,
                   int* overflow);
int tcec_scale_buf(tcec_handle h, const float* src, float* dst, int64_t n, int scale_exp);
int tcec_add_buf(tcec_handle h, const float* a, const float* b, float* dst, int64_t n);
int tcec_sub_buf(tcec_handle h, const float* a, const float* b, float* dst, int64_t n);

/* Test hook (no reference counterpart; it exposes an internal stage of
 * dispatch_cgemm so it can be pinned bit for bit): the hot path's operand
 * preparation for a fixed decision kind (0 FP16TCEC, 1 FP16TCEC_SCALED,
 * 2 TF32TCEC) and shifts -- scale_buf + split_buf (kernels_scalar.cpp:24-40)
 * fused with the K-major layout.  Device outputs: a_hi/a_lo m x kp and
 * b_hi/b_lo 2n x kp elements (binary16 for the FP16 kinds, f32 for TF32),
 * kp = tcec_prep_kp(k) = round_up(2k, 64), zero padded; A' row i = the
 * interleaved (re, im) row i of A; B' row 2j = (Br, -Bi), row 2j+1 = (Bi, Br)
 * per complex k.  flags[0] = format overflow, flags[1] = ScaleOverflow. */
int64_t tcec_prep_kp(int64_t k);
int tcec_debug_prep(tcec_handle h, const void* a, const void* b, int64_t m, int64_t n, int64_t k,
                    int kind, int scale_a, int scale_b, int corrected, void* a_hi, void* a_lo,
                    void* b_hi, void* b_lo, int* flags);
/* the same for either operand layout: xa = 0 as above; xa = 1 the A-expanded
 * layout (tcec_set_operand_layout): a_hi/a_lo 2m x kp with row 2i = (Ar, -Ai),
 * row 2i+1 = (Ai, Ar) per complex k; b_hi/b_lo n x kp with row j = (Br, Bi)
 * (column j of B) */
int tcec_debug_prep_layout(tcec_handle h, const void* a, const void* b, int64_t m, int64_t n, int64_t k,
                           int kind, int scale_a, int scale_b, int corrected, int xa, void* a_hi,
                           void* a_lo, void* b_hi, void* b_lo, int* flags);

/* ------------------------------------------------- precision selection */
/* ExpStats, precsel.hpp:18-36 (e_max_valid == 0 <=> std::nullopt) */
typedef struct {
    uint64_t n1, n2;
    int32_t e_max;
    int32_t e_max_valid;
    uint64_t n_nonzero, n_total;
    int32_t stage2_evaluated;
    int32_t pad_;
} tcec_exp_stats_t;

/* exp_stats (precsel.hpp:68) when staged == 0, exp_stats_staged (precsel.hpp:70)
 * when staged != 0; x is a device rows x cols complex matrix */
int tcec_exp_stats(tcec_handle h, const void* x, int64_t rows, int64_t cols, int target_max_exponent,
                   int staged, double t, tcec_exp_stats_t* out);
double tcec_r1(const tcec_exp_stats_t* s); /* precsel.hpp:27-30 */
double tcec_r2(const tcec_exp_stats_t* s); /* precsel.hpp:32-35 */
/* matrix_tolerance, precsel.hpp:74; *level = ToleranceLevel (0 tf32_only,
 * 1 fp16_scaled_ok, 2 fp16_ok); TCEC_ERR_LOGIC when stage 2 was needed but skipped */
int tcec_matrix_tolerance(const tcec_exp_stats_t* s, double t, int target_max_exponent, int* level);
/* select_mode, precsel.hpp:76-77; kind = ComputeKind (0 FP16TCEC, 1 FP16TCEC_SCALED,
 * 2 TF32TCEC, 3 FP32_BASELINE) */
int tcec_select_mode(int level_a, int e_max_valid_a, int e_max_a, int level_b, int e_max_valid_b,
                     int e_max_b, int target_max_exponent, int* kind, int* scale_a, int* scale_b);
/* scale_matrix_inplace (precsel.hpp:82-85) on n components; ScaleOverflow when
 * a result leaves the finite range (check != 0) -- descale_output uses check = 0 */
int tcec_scale_components(tcec_handle h, float* x, int64_t n, int scale_exp, int check);

/* ------------------------------------------------------------- CGEMM */
/* GemmMode, gemm.hpp:19 */
enum { TCEC_FP32_REF = 0, TCEC_FP64_ORACLE = 1, TCEC_TF32_TC = 2, TCEC_FP16_TC = 3,
       TCEC_TF32_TCEC = 4, TCEC_FP16_TCEC = 5 };
/* ForcedMode, precsel.hpp:128-136 (force = -1: automatic selection) */
enum { TCEC_FORCE_NONE = -1, TCEC_FORCE_FP32_REF = 0, TCEC_FORCE_FP64_ORACLE = 1,
       TCEC_FORCE_TF32_TC = 2, TCEC_FORCE_FP16_TC = 3, TCEC_FORCE_TF32_TCEC = 4,
       TCEC_FORCE_FP16_TCEC = 5, TCEC_FORCE_FP16_TCEC_SCALED = 6 };

/* cgemm, cgemm.hpp:17-18 -- device a (m x k), b (k x n), c (m x n) complex.
 * FP32_REF and FP64_ORACLE are bit-identical to the reference; the tensor-core
 * modes are within the FP32-level tolerance. */
int tcec_cgemm(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
               int64_t k, int mode, int k_tile, int* overflow);

/* SelectionPolicy + TilingConfig + ForcedMode = DispatchConfig, precsel.hpp:60-65,140-144 */
typedef struct {
    double threshold_t;
    int64_t size_auto;
    int64_t size_tf32;
    int32_t target_max_exponent;
    int32_t k_tile;
    int32_t force;
    int32_t pad_;
} tcec_dispatch_config_t;

/* DispatchResult + DecisionRecord, precsel.hpp:92-101,146-151 */
typedef struct {
    int32_t kind, scale_a, scale_b, overflow;
    int32_t has_stats, pad_;
    tcec_exp_stats_t stats_a, stats_b;
    char line[160]; /* DecisionRecord::to_line(), precsel.cpp:185-205 */
} tcec_dispatch_result_t;

void tcec_default_config(tcec_dispatch_config_t* cfg);
/* dispatch_cgemm, precsel.hpp:153-156 -- device buffers; the statistics and the
 * decision are computed on the device; *res (host) is filled after the call
 * completes (the call synchronizes the handle stream). */
int tcec_dispatch_cgemm(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
                        int64_t k, const tcec_dispatch_config_t* cfg, tcec_dispatch_result_t* res);
/* same with HOST buffers: H2D copy of A and B, dispatch, D2H copy of C */
int tcec_dispatch_cgemm_host(tcec_handle h, const void* a, const void* b, void* c, int64_t m,
                             int64_t n, int64_t k, const tcec_dispatch_config_t* cfg,
                             tcec_dispatch_result_t* res);

/* ------------------------------------------------------------ permute */
/* permute, tensor.hpp:56-105: dst = src transposed so that new axis a is old
 * axis axis_of[a]; old_dims are the source extents; complex elements; device */
int tcec_permute(tcec_handle h, const void* src, void* dst, int rank, const int64_t* old_dims,
                 const int* axis_of);

/* ------------------------------------------------ network contraction */
typedef struct tcec_network_s* tcec_network;

/* TensorNetwork (network.hpp:17-19) with integer labels.  Node i has ranks[i]
 * axes whose labels/dims are the next ranks[i] entries of labels/dims. */
int tcec_network_create(tcec_handle h, int n_nodes, const int* ranks, const int* labels,
                        const int64_t* dims, tcec_network* out);
int tcec_network_destroy(tcec_network net);
/* copy node data (host, complex, row-major in label order) */
int tcec_network_set_node(tcec_network net, int node, const void* host_data);
/* greedy_path, network.hpp:49 -- writes 2 * (n_nodes - 1) ints */
int tcec_network_greedy_path(tcec_network net, int* steps);
/* Contraction-tree reconfiguration (host code, no device needed; replaces the
 * role of greedy_path, network.cpp:204-315, for large circuits): optimise the
 * SSA path `steps` (n_nodes - 1 pairs) over frontiers of up to k pieces (3..16)
 * by exact dynamic programming.  Network given as ranks[n_nodes] and the
 * concatenated labels / dims of every node.  time_model = 0 scores MACs, 1 the
 * estimated B200 time of each step's dispatch tier; latency_macs is the cost
 * per element of k of a few-output FP32-chain step.  Writes the new path. */
int tcec_path_reconfigure(int n_nodes, const int* ranks, const int* labels, const int64_t* dims,
                          const int* steps, int n_steps, int k, int passes, int time_model,
                          double latency_macs, unsigned long long seed, int* out_steps);
/* contract_network, network.hpp:37-38 -- path as (a, b) id pairs in SSA
 * numbering (network.hpp:22-26).  The result tensor (host) has the labels
 * written to out_labels (may be NULL) and rank to *out_rank.  When log_lines is
 * non-NULL the decision-log lines ('\n'-separated) are written there. */
int tcec_contract_network(tcec_network net, const int* steps, int n_steps,
                          const tcec_dispatch_config_t* cfg, void* out_host, int64_t out_capacity,
                          int* out_rank, int* out_labels, char* log_lines, int64_t log_capacity);
/* the DispatchResult + DecisionRecord of every step of the network's last
 * tcec_contract_network call (the records contract_network appends to its
 * DecisionLog, network.cpp:129-134); *count = steps written */
int tcec_network_step_results(tcec_network net, tcec_dispatch_result_t* out, int capacity, int* count);
/* amplitude batch (qcircuit.hpp:49-52 over many bitstrings): the network's
 * closing selector nodes (one per entry of sel_nodes) are replaced per
 * bitstring; the same plan is replayed; out_host gets one complex per string */
int tcec_contract_selector_batch(tcec_network net, const int* steps, int n_steps,
                                 const tcec_dispatch_config_t* cfg, int n_sel, const int* sel_nodes,
                                 int n_strings, const uint8_t* bits, void* out_host);
/* general form of the batch: run r replaces the data of the n_var nodes
 * var_nodes[] with the r-th block of var_data (host; the nodes' complex data
 * concatenated in var_nodes order) and replays the same plan.  Used for the
 * slices of a sliced contraction (every slice has the same
 * path, only the sliced nodes' data differ).  out_host: n_runs complex values. */
int tcec_contract_node_batch(tcec_network net, const int* steps, int n_steps,
                             const tcec_dispatch_config_t* cfg, int n_var, const int* var_nodes,
                             int n_runs, const void* var_data, void* out_host);

/* After a selector / node batch: run `run`'s format-overflow flag (OR over its
 * GEMMs, DispatchResult::overflow, precsel.hpp:146-151) and its decision-log
 * lines ('\n'-separated DecisionRecord::to_line, one per step -- what
 * amplitude(..., log) records, qcircuit.cpp:184-195).  A batch in which any
 * run hit ScaleOverflow (precsel.cpp:54-57) or a skipped stage 2
 * (precsel.cpp:117-118) fails with that error, naming the run. */
int tcec_network_batch_run_info(tcec_network net, int run, int* overflow, char* log_lines,
                                int64_t log_capacity);

/* ------------------------------------------------- f64 reference functions
 * The reference's f64 "truth" functions, computed on the device in the
 * reference's accumulation order (ascending-k RN chains from +0.0, separate
 * multiply and add), so they are bit-identical to it.  They are reference
 * API, not part of the TCEC path. */
/* cgemm_oracle, cgemm.hpp:26 / cgemm.cpp:62-74: a, b complex64 (device),
 * c complex128 (device), m x n */
int tcec_cgemm_oracle(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
                      int64_t k);
/* cgemm_f64 of contract_pair_oracle (network.cpp:87-110): complex128 in and out */
int tcec_cgemm_c128(tcec_handle h, const void* a, const void* b, void* c, int64_t m, int64_t n,
                    int64_t k);
/* permute (tensor.hpp:56-105) of a complex128 tensor (device) */
int tcec_permute_c128(tcec_handle h, const void* src, void* dst, int rank, const int64_t* old_dims,
                      const int* axis_of);
/* contract_network_oracle, network.hpp:39 / network.cpp:179-186: the result
 * tensor (complex128, host) of the f64 TTGT fold along `steps` */
int tcec_contract_network_oracle(tcec_network net, const int* steps, int n_steps, void* out_host,
                                 int64_t out_capacity, int* out_rank, int* out_labels);
/* statevector_oracle, qcircuit.hpp:56 / qcircuit.cpp:197-225: apply n_gates
 * gates in order to |0...0> (qubit q = bit q of the index); gate g acts on
 * qubit qa[g] with the row-major 2x2 complex128 matrix u[8g .. 8g+7]
 * (gate_matrix_f64), or is a CZ on (qa[g], qb[g]) when qb[g] >= 0.
 * state: 2^n_qubits complex128 (device). */
int tcec_statevector_f64(tcec_handle h, int n_qubits, int n_gates, const int* qa, const int* qb,
                         const double* u, void* state);

/* ------------------------------------------------- workload generation
 * The reference's deterministic random source (Rng, rng.hpp:13-56: the
 * standard std::mt19937_64 + its hand-rolled maps), host code, so benchmark
 * inputs are the reference's own -- configs[1] fills A then B from one
 * Rng(seed + n) with two uniform_pm1f draws per complex element
 * (experiments.cpp:76-83).  No device work. */
typedef struct tcec_rng_s* tcec_rng;
int tcec_rng_create(uint64_t seed, tcec_rng* out);
int tcec_rng_destroy(tcec_rng r);
uint64_t tcec_rng_next_u64(tcec_rng r);
/* n successive Rng::uniform_pm1f() draws (rng.hpp:35) */
int tcec_rng_fill_uniform_pm1f(tcec_rng r, float* dst, int64_t n);
/* n successive Rng::gaussian(stddev) draws (rng.hpp:38-50) */
int tcec_rng_fill_gaussian(tcec_rng r, double stddev, double* dst, int64_t n);

#ifdef __cplusplus
}
#endif

#endif /* TCEC_B200_H */
