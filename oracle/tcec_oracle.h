/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TCEC hot path.
 *
 * A plain-C restatement of the reference (mpsgemm, /root/reference/proj) for
 * the north-star path: format emulation, exponent statistics, precision
 * selection, scaling, residual split, the real/complex GEMM schedules, and the
 * TTGT permute.  Every function cites the reference file:line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or the
 * timed CPU baseline.  The product path (paper_2303_08989_b200) never links it.
 *
 * Parity pinning: oracle/ref_bridge.cpp builds the reference's own sources into
 * oracle/_ref/libmpsgemm_ref.so; tests/test_oracle_vs_reference.py checks this
 * restatement against it bit for bit, and tests/golden/ holds fixtures produced
 * by the reference (tests/golden/make_golden.py) so the pin survives on boxes
 * without /root/reference.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; -ffp-contract=off is
 * required for the RN/RZ schedules, reference proj/CMakeLists.txt:12-14).
 */
#ifndef TCEC_ORACLE_H
#define TCEC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* lowprec.hpp:13-15 */
enum { ORC_FMT_FP16 = 0, ORC_FMT_TF32 = 1 };
enum { ORC_RN = 0, ORC_RZ = 1 };

/* lowprec.hpp:44-51 -- floor(log2|x|); returns 0 and leaves *e for x == +-0 */
int orc_exponent_of(float x, int* e);
/* lowprec.hpp:58-74 */
float orc_quantize(float x, int fmt, int rounding, int* overflow);
/* lowprec.hpp:84-88 */
void orc_split(float x, int fmt, float* hi, float* lo, int* overflow);
/* lowprec.hpp:94-101 */
float orc_add_rz(float a, float b);

/* KernelTable entries, kernels_scalar.cpp:18-162 */
void orc_quantize_buf(const float* src, float* dst, int64_t n, int fmt, int rounding, int* overflow);
void orc_split_buf(const float* src, float* hi, float* lo, int64_t n, int fmt, int* overflow);
void orc_scale_buf(const float* src, float* dst, int64_t n, int scale_exp);
void orc_add_buf(const float* a, const float* b, float* dst, int64_t n);
void orc_sub_buf(const float* a, const float* b, float* dst, int64_t n);
void orc_abs_stats(const float* x, int64_t n, float threshold, uint64_t* n_nonzero, uint64_t* n_ge,
                   float* max_abs);
uint64_t orc_count_abs_ge(const float* x, int64_t n, float threshold);
void orc_gemm_rows_rn(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                      int64_t row_begin, int64_t row_end);
void orc_gemm_rows_rz(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                      int64_t row_begin, int64_t row_end);
void orc_gemm_rows_tcec(const float* a_hi, const float* a_lo, const float* b_hi, const float* b_lo,
                        float* c, int64_t m, int64_t n, int64_t k, int k_tile, int64_t row_begin,
                        int64_t row_end);
void orc_gemm_rows_f64(const float* a, const float* b, double* c, int64_t m, int64_t n, int64_t k,
                       int64_t row_begin, int64_t row_end);

/* precsel.hpp:18-36 -- ExpStats as a POD.  e_max_valid == 0 <=> nullopt. */
typedef struct {
    uint64_t n1, n2;
    int32_t e_max;
    int32_t e_max_valid;
    uint64_t n_nonzero, n_total;
    int32_t stage2_evaluated;
    int32_t pad_;
} orc_exp_stats_t;

/* precsel.hpp:38 / :45 */
enum { ORC_TOL_TF32_ONLY = 0, ORC_TOL_FP16_SCALED_OK = 1, ORC_TOL_FP16_OK = 2 };
enum { ORC_KIND_FP16_TCEC = 0, ORC_KIND_FP16_TCEC_SCALED = 1, ORC_KIND_TF32_TCEC = 2,
       ORC_KIND_FP32_BASELINE = 3 };

/* precsel.cpp:89-104; x is the 2*rows*cols interleaved component buffer */
void orc_exp_stats(const float* x, int64_t n_components, int target_max_exponent,
                   orc_exp_stats_t* out);
void orc_exp_stats_staged(const float* x, int64_t n_components, int target_max_exponent, double t,
                          orc_exp_stats_t* out);
double orc_r1(const orc_exp_stats_t* s); /* precsel.hpp:27-30 */
double orc_r2(const orc_exp_stats_t* s); /* precsel.hpp:32-35 */
/* precsel.cpp:106-121; returns level, writes e_max; returns -1 on logic_error */
int orc_matrix_tolerance(const orc_exp_stats_t* s, double t, int target_max_exponent);
/* precsel.cpp:123-135 */
void orc_select_mode(int level_a, int e_valid_a, int e_a, int level_b, int e_valid_b, int e_b,
                     int target_max_exponent, int* kind, int* sa, int* sb);

/* gemm.hpp:19 GemmMode */
enum { ORC_MODE_FP32_REF = 0, ORC_MODE_FP64_ORACLE = 1, ORC_MODE_TF32_TC = 2, ORC_MODE_FP16_TC = 3,
       ORC_MODE_TF32_TCEC = 4, ORC_MODE_FP16_TCEC = 5 };

/* gemm.cpp:108-125 real mode switch (f32 output) */
int orc_gemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int mode,
             int k_tile, int* overflow);
/* cgemm.cpp:25-46 -- interleaved complex, a: m x k, b: k x n, c: m x n */
int orc_cgemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int mode,
              int k_tile, int* overflow);
/* cgemm.cpp:62-74 -- f64 complex oracle, c interleaved doubles */
void orc_cgemm_oracle(const float* a, const float* b, double* c, int64_t m, int64_t n, int64_t k);
/* cgemm.cpp:76-89 */
double orc_relative_error_c(const float* c, const double* ref, int64_t n_elems);

/* precsel.cpp:225-322 dispatch_cgemm.  force: -1 none, else ForcedMode 0..6
 * (precsel.hpp:128-136).  Returns 0, or 1 = ScaleOverflow, 2 = logic_error. */
typedef struct {
    double threshold_t;
    int64_t size_auto;
    int64_t size_tf32;
    int32_t target_max_exponent;
    int32_t k_tile;
    int32_t force;
    int32_t pad_;
} orc_dispatch_config_t;

typedef struct {
    int32_t kind, scale_a, scale_b, overflow;
    int32_t has_stats, pad_;
    orc_exp_stats_t stats_a, stats_b;
    char line[160]; /* DecisionRecord::to_line, precsel.cpp:185-205 */
} orc_dispatch_result_t;

int orc_dispatch_cgemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                       const orc_dispatch_config_t* cfg, orc_dispatch_result_t* res);
/* the selection half of dispatch_cgemm only (statistics, ComputeMode, line) */
int orc_dispatch_decision(const float* a, const float* b, int64_t m, int64_t n, int64_t k,
                          const orc_dispatch_config_t* cfg, orc_dispatch_result_t* res);

/* tensor.hpp:56-105 -- permute of complex (8-byte) elements.  axis_of[a] is
 * the old axis feeding new axis a; dims are the OLD dims. */
void orc_permute_c64(const float* src, float* dst, int rank, const int64_t* old_dims,
                     const int* axis_of);

/* rng.hpp:13-56 -- std::mt19937_64 plus the hand-rolled distributions */
typedef struct {
    uint64_t mt[312];
    int mti;
    int have_spare;
    double spare;
} orc_rng_t;
void orc_rng_seed(orc_rng_t* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng_t* r);
uint64_t orc_rng_next_below(orc_rng_t* r, uint64_t n);
double orc_rng_uniform01(orc_rng_t* r);
float orc_rng_uniform_pm1f(orc_rng_t* r);
double orc_rng_gaussian(orc_rng_t* r, double stddev);
/* experiments.cpp:27-31 random_uniform_matrix: n_elems complex values */
void orc_fill_uniform_c32(orc_rng_t* r, float* dst, int64_t n_elems);

#ifdef __cplusplus
}
#endif

#endif
