// Internal (host-side) declarations shared by the CUDA translation units and the
// C-ABI layer.  Not part of the public boundary (that is include/tcec_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tcec {

// Device-resident decision of one dispatched CGEMM.  Written by the statistics
// and selection kernels and read by the operand-preparation and GEMM kernels,
// so an AUTO dispatch needs no host round trip (paper: the selector runs on
// the device).  Mirrors ExpStats / ComputeMode
// (reference precsel.hpp:18-55).
struct DevStats {
    unsigned long long n_nonzero, n1, n2, n_total;
    unsigned int max_bits;      // max |x| bit pattern over nonzero, non-NaN components
    int stage2_evaluated;
    int e_max, e_max_valid;
};

struct DevDecision {
    DevStats st[2];             // operand A, operand B
    int kind;                   // ComputeKind (precsel.hpp:45)
    int scale_a, scale_b;       // ComputeMode shifts
    int level_a, level_b;       // ToleranceLevel, -1 = logic_error
    unsigned int overflow;      // split/quantize saturation (DispatchResult::overflow)
    unsigned int scale_overflow;  // ScaleOverflow (precsel.cpp:54-57)
    int pad_;                   // stats2_kernel's block counter (0 between dispatches)
};

enum Kind : int { kKindFp16 = 0, kKindFp16Scaled = 1, kKindTf32 = 2, kKindFp32 = 3 };

// ----------------------------------------------------------- elementwise
void launch_quantize(const float* src, float* dst, int64_t n, int fmt, int rz,
                     unsigned* d_ovf, cudaStream_t s);
void launch_split_flat(const float* src, float* hi, float* lo, int64_t n, int fmt,
                       unsigned* d_ovf, cudaStream_t s);
void launch_scale(const float* src, float* dst, int64_t n, int scale_exp, unsigned* d_nonfinite,
                  cudaStream_t s);
void launch_add_sub(const float* a, const float* b, float* dst, int64_t n, int sub, cudaStream_t s);

// ------------------------------------------------------------- statistics
// stage 1 over both operands (n_a / n_b real components; a null operand is skipped)
void launch_stats1(const float* a, int64_t n_a, const float* b, int64_t n_b, DevDecision* d,
                   cudaStream_t s);
// stage 2; mode 0 = staged (skip when stage 1 passes for t), 1 = always.
// select = 1: the selection (precsel.cpp:106-135) with threshold sel_t follows
// in the same launch (forced_scaled = 1 for ForcedMode::fp16_tcec_scaled); it
// uses the decision slot's pad_ as its block counter (zeroed with the slot).
// spec_fa / spec_fb > 0: the operands are these fractions of larger ones
// (the host pipeline's speculative decision); at t = 0 an FP16 kind reached
// through stage 2 becomes TF32 when the whole operands are expected to hold a
// component below the stage-2 threshold (see stats2_kernel).
void launch_stats2(const float* a, int64_t n_a, const float* b, int64_t n_b, DevDecision* d,
                   double t, int target, int always, cudaStream_t s, int select = 0,
                   double sel_t = 0.0, int forced_scaled = 0, float spec_fa = 0.0f, float spec_fb = 0.0f);

// ------------------------------------------------------- operand layouts
// Matrix view of a permuted tensor (fused TTGT gather): element (r, c) of the
// rows x cols matrix is at base + rows.offset(r) + cols.offset(c), each offset
// a mixed-radix sum over runs of merged tensor axes (innermost run last).
constexpr int kMaxRuns = 16;  // Sycamore m=12 tensor-core operands need up to 16
struct RunMap {
    int n = 0;                      // runs
    int pow2 = 1;                   // every extent a power of two (shift / mask decomposition)
    uint32_t ext[kMaxRuns] = {};    // run extents
    uint32_t shift[kMaxRuns] = {};  // log2(ext) when pow2
    int64_t stride[kMaxRuns] = {};  // element stride of each run
};
struct MatrixView {
    RunMap rows, cols;
};
// A (m x k complex, interleaved) -> A' = m x Kp real, K-major, hi/lo in the
// decided format (f16 or tf32-in-f32); padded columns are zero.
// kind_fixed >= 0 overrides the device decision (forced / size-gated modes).
void launch_prep_a(const float* a, int64_t m, int64_t k, int64_t kp, void* hi, void* lo,
                   const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s,
                   int64_t row0 = 0,   // rows [row0, row0 + m) of a full A / A'
                   const MatrixView* view = nullptr);  // A read through a view (fused TTGT gather)
// B (k x n complex) -> B'^T = 2n x Kp real, K-major, with the complex block
// expansion [[Br, Bi], [-Bi, Br]] so one real GEMM yields interleaved C.
void launch_prep_b(const float* b, int64_t k, int64_t n, int64_t kp, void* hi, void* lo,
                   const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s,
                   int64_t jout0 = 0,  // b = a k x n column block, B' rows from 2 jout0
                   const MatrixView* view = nullptr);
// A-expanded layout (used when m < n): A'' = 2m x Kp with rows 2i = (Ar, -Ai),
// 2i+1 = (Ai, Ar) along K; B'' = B^T = n x Kp with (Br, Bi) along K.  The GEMM
// yields rows (Re C[i,:], Im C[i,:]) and its epilogue interleaves them.
void launch_prep_ax(const float* a, int64_t m, int64_t k, int64_t kp, void* hi, void* lo,
                    const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s,
                    const MatrixView* view = nullptr);
void launch_prep_bx(const float* b, int64_t k, int64_t n, int64_t kp, void* hi, void* lo,
                    const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s,
                    const MatrixView* view = nullptr);

// -------------------------------------------------------------- SIMT GEMM
// FP32_REF complex GEMM, bit-identical to the reference schedule
// (kernels_scalar.cpp:76-87 + cgemm.cpp:33-44).  Strided operand views allow
// fused TTGT gathers: element (i, kk) of A is at a[ (row_off(i) + col_off(kk)) ]
void launch_cgemm_fp32_ref(const float2* a, const float2* b, float2* c, int64_t m, int64_t n,
                           int64_t k, cudaStream_t s);
// Build the view of operand `role` (0 = A: rows = free_a, cols = shared;
// 1 = B: rows = shared, cols = free_b) of a tensor with physical extents
// dims[0..rank) permuted by axis_of (new axis a = old axis axis_of[a]) whose
// first n_row_axes new axes are the matrix rows.  false when it needs more
// than kMaxRuns runs per side.
bool make_matrix_view(int rank, const int64_t* dims, const int* axis_of, int n_row_axes, MatrixView* v);
// FP32_REF complex GEMM of a skinny shape (k <= 128, min(m, n) <= 32,
// max(m, n) >= 4096) whose LONG operand is read through a view instead of a
// materialised permute (B when m <= n, else A); the short operand is a plain
// row-major matrix.  Bit-identical to launch_cgemm_fp32_ref on the permuted
// operand.  false when the shape is not skinny.
bool launch_skinny_view(const float2* a, const float2* b, float2* c, int64_t m, int64_t n, int64_t k,
                        const MatrixView& long_view, cudaStream_t s);
bool skinny_shape(int64_t m, int64_t n, int64_t k);
// FP64_ORACLE mode (gemm.cpp:68-74, :111-117)
void launch_cgemm_fp64(const float2* a, const float2* b, float2* c, int64_t m, int64_t n,
                       int64_t k, cudaStream_t s);

// ---------------------------------------------------------------- permute
constexpr int kMaxRank = 48;

// ------------------------------------------------- f64 reference (f64_ref.cu)
void launch_cgemm_c128(const void* a, bool a_f32, const void* b, bool b_f32, double2* c, int64_t m,
                       int64_t n, int64_t k, cudaStream_t s);
void launch_permute_c128(const double2* src, double2* dst, int rank, const int64_t* old_dims,
                         const int* axis_of, cudaStream_t s);
void launch_widen(const float2* src, double2* dst, int64_t n, cudaStream_t s);
void launch_permute(const float2* src, float2* dst, int rank, const int64_t* old_dims,
                    const int* axis_of, cudaStream_t s);

// ------------------------------------------------------------ tcgen05 GEMM
struct TcecGemmArgs {
    const void* a_hi; const void* a_lo;   // m x kp
    const void* b_hi; const void* b_lo;   // n2 x kp  (n2 = 2n)
    float* c;                             // m x n2 (interleaved complex C)
    int64_t m, n2, kp;
    const DevDecision* d;                 // device decision (kind / shifts)
    int kind_fixed;                       // >= 0: host-known kind; -1: read d->kind
    int fmt;                              // 0 = f16 kernel, 1 = tf32 kernel, -1 = device-decided
    int corrected;                        // 1 = TCEC (3 products), 0 = TC ablation
    int flush_kblocks;                    // RN flush interval of the main term, 0 = none
    int pair;                             // resolved kernel variant (kVariantSingle/Pair/Wide)
    int sms;                              // SM count (persistent grid size)
    int64_t a_row_off, a_rows;            // row chunk of A' (wide kernel): first row, rows of the whole A'
    float* partial;                       // split-K partials (set by launch_tcec_gemm)
    int splits, kb_per;                   // split count, 64-element k-blocks per split
    int no_split;                         // 1: never split K (row-chunked launches must match the one-launch bits)
    int64_t ldc;                          // row stride of C in floats, 0 = n2 (wide kernel: column blocks of C)
    int64_t b_row_off;                    // first B' row of this launch (wide kernel: column blocks of B)
    int xa;                               // 1: A-expanded layout (m = 2 x rows of C, n2 = columns of C,
                                          //    GEMM rows 2i / 2i+1 = Re / Im of C row i, interleaved on store)
};
// tcgen05 kernel variants (tcec_set_gemm_variant): auto picks wide when its
// 256 x 256 pair tiles fill the SMs, else single
enum GemmVariant : int { kVariantAuto = 0, kVariantPair = 1, kVariantSingle = 2, kVariantWide = 3, kVariantWidePersistent = 4,
                         kVariantWideMc = 5, kVariantPairPersistent = 6 };
// allow_pair / allow_pairp = false: only the variants that take row chunks and
// column blocks (the host-buffer pipeline) or the B-expanded layout
int resolve_gemm_variant(int requested, int64_t m, int64_t n2, int64_t kp, int sm_count,
                         bool allow_pair = true, bool allow_pairp = true);
// returns a cudaError_t
int launch_tcec_gemm(const TcecGemmArgs& args, cudaStream_t s);

}  // namespace tcec
