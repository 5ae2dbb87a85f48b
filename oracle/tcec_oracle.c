/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the TCEC hot path.  See
 * tcec_oracle.h for the contract and for who may load this file.  Compiled with
 * -ffp-contract=off (reference proj/CMakeLists.txt:12-14); no fast-math.
 */
#include "tcec_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ lowprec */

/* lowprec.hpp:19-37: both formats carry 10 explicit mantissa bits */
static double fmt_max_normal(int fmt) {
    /* (2 - 2^-10) * 2^max_exp, lowprec.hpp:28-33 */
    return fmt == ORC_FMT_FP16 ? ldexp(2.0 - 0x1.0p-10, 15) : ldexp(2.0 - 0x1.0p-10, 127);
}
static int fmt_min_subnormal_exp(int fmt) {
    /* min_normal_exp - explicit_mantissa_bits, lowprec.hpp:26 */
    return fmt == ORC_FMT_FP16 ? -14 - 10 : -126 - 10;
}

static uint32_t f2u(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    return u;
}
static float u2f(uint32_t u) {
    float x;
    memcpy(&x, &u, 4);
    return x;
}

int orc_exponent_of(float x, int* e) {
    /* lowprec.hpp:44-51 */
    const uint32_t b = f2u(x) & 0x7FFFFFFFu;
    if (b == 0) return 0;
    const int raw = (int)(b >> 23);
    if (raw != 0) {
        *e = raw - 127;
    } else {
        /* subnormal: -149 + bit_width(b) - 1 */
        *e = -149 + (31 - __builtin_clz(b));
    }
    return 1;
}

float orc_quantize(float x, int fmt, int rounding, int* overflow) {
    /* lowprec.hpp:58-74 */
    if (x == 0.0f) return x;
    const double xd = (double)x;
    const double limit = fmt_max_normal(fmt);
    if (fabs(xd) > limit) {
        if (overflow) *overflow = 1;
        return (float)copysign(limit, xd);
    }
    int e = 0;
    orc_exponent_of(x, &e);
    int q = e - 10;
    if (q < fmt_min_subnormal_exp(fmt)) q = fmt_min_subnormal_exp(fmt);
    const double scaled = ldexp(xd, -q);
    const double r = rounding == ORC_RN ? nearbyint(scaled) : trunc(scaled);
    return (float)ldexp(r, q);
}

void orc_split(float x, int fmt, float* hi, float* lo, int* overflow) {
    /* lowprec.hpp:84-88 */
    const float h = orc_quantize(x, fmt, ORC_RN, overflow);
    const float resid = (x - h) * 0x1.0p11f;
    *hi = h;
    *lo = orc_quantize(resid, fmt, ORC_RN, overflow);
}

float orc_add_rz(float a, float b) {
    /* lowprec.hpp:94-101: 2Sum, then one ulp toward zero when RN overshot */
    const float s = a + b;
    const float bb = s - a;
    const float err = (a - (s - bb)) + (b - bb);
    if (err != 0.0f && (signbit(err) != 0) != (signbit(s) != 0)) return u2f(f2u(s) - 1u);
    return s;
}

/* ------------------------------------------------------------- kernel table */

void orc_quantize_buf(const float* src, float* dst, int64_t n, int fmt, int rounding,
                      int* overflow) {
    /* kernels_scalar.cpp:18-22 */
    for (int64_t i = 0; i < n; ++i) dst[i] = orc_quantize(src[i], fmt, rounding, overflow);
}

void orc_split_buf(const float* src, float* hi, float* lo, int64_t n, int fmt, int* overflow) {
    /* kernels_scalar.cpp:24-32 */
    for (int64_t i = 0; i < n; ++i) orc_split(src[i], fmt, &hi[i], &lo[i], overflow);
}

void orc_scale_buf(const float* src, float* dst, int64_t n, int scale_exp) {
    /* kernels_scalar.cpp:34-40: via double, a single rounding */
    const double factor = ldexp(1.0, scale_exp);
    for (int64_t i = 0; i < n; ++i) dst[i] = (float)((double)src[i] * factor);
}

void orc_add_buf(const float* a, const float* b, float* dst, int64_t n) {
    for (int64_t i = 0; i < n; ++i) dst[i] = a[i] + b[i]; /* kernels_scalar.cpp:42-44 */
}

void orc_sub_buf(const float* a, const float* b, float* dst, int64_t n) {
    for (int64_t i = 0; i < n; ++i) dst[i] = a[i] - b[i]; /* kernels_scalar.cpp:46-48 */
}

void orc_abs_stats(const float* x, int64_t n, float threshold, uint64_t* n_nonzero, uint64_t* n_ge,
                   float* max_abs) {
    /* kernels_scalar.cpp:50-65 */
    uint64_t nz = 0, ge = 0;
    float mx = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        const float a = fabsf(x[i]);
        if (a > 0.0f) {
            ++nz;
            if (a >= threshold) ++ge;
            if (a > mx) mx = a;
        }
    }
    *n_nonzero = nz;
    *n_ge = ge;
    *max_abs = mx;
}

uint64_t orc_count_abs_ge(const float* x, int64_t n, float threshold) {
    /* kernels_scalar.cpp:67-74 */
    uint64_t ge = 0;
    for (int64_t i = 0; i < n; ++i) {
        const float a = fabsf(x[i]);
        if (a > 0.0f && a >= threshold) ++ge;
    }
    return ge;
}

void orc_gemm_rows_rn(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                      int64_t row_begin, int64_t row_end) {
    /* kernels_scalar.cpp:76-87: f32 products, RN chain in ascending k */
    (void)m;
    for (int64_t i = row_begin; i < row_end; ++i) {
        float* crow = c + i * n;
        for (int64_t j = 0; j < n; ++j) crow[j] = 0.0f;
        for (int64_t kk = 0; kk < k; ++kk) {
            const float av = a[i * k + kk];
            const float* brow = b + kk * n;
            for (int64_t j = 0; j < n; ++j) crow[j] = crow[j] + av * brow[j];
        }
    }
}

void orc_gemm_rows_rz(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                      int64_t row_begin, int64_t row_end) {
    /* kernels_scalar.cpp:89-100: RZ after every addition */
    (void)m;
    for (int64_t i = row_begin; i < row_end; ++i) {
        float* crow = c + i * n;
        for (int64_t j = 0; j < n; ++j) crow[j] = 0.0f;
        for (int64_t kk = 0; kk < k; ++kk) {
            const float av = a[i * k + kk];
            const float* brow = b + kk * n;
            for (int64_t j = 0; j < n; ++j) crow[j] = orc_add_rz(crow[j], av * brow[j]);
        }
    }
}

void orc_gemm_rows_tcec(const float* a_hi, const float* a_lo, const float* b_hi, const float* b_lo,
                        float* c, int64_t m, int64_t n, int64_t k, int k_tile, int64_t row_begin,
                        int64_t row_end) {
    /* kernels_scalar.cpp:102-135: main term RZ inside k tiles and RN across
     * tiles; the two correction chains RZ; RN join with the 2^-11 weight */
    (void)m;
    float* main_acc = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    float* tile_acc = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    float* c1 = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    float* c2 = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = row_begin; i < row_end; ++i) {
        for (int64_t j = 0; j < n; ++j) main_acc[j] = tile_acc[j] = c1[j] = c2[j] = 0.0f;
        for (int64_t kk = 0; kk < k; ++kk) {
            if (kk != 0 && kk % k_tile == 0) {
                for (int64_t j = 0; j < n; ++j) {
                    main_acc[j] = main_acc[j] + tile_acc[j];
                    tile_acc[j] = 0.0f;
                }
            }
            const float ah = a_hi[i * k + kk];
            const float al = a_lo[i * k + kk];
            const float* bh = b_hi + kk * n;
            const float* bl = b_lo + kk * n;
            for (int64_t j = 0; j < n; ++j) {
                tile_acc[j] = orc_add_rz(tile_acc[j], ah * bh[j]);
                c1[j] = orc_add_rz(c1[j], al * bh[j]);
                c2[j] = orc_add_rz(c2[j], ah * bl[j]);
            }
        }
        float* crow = c + i * n;
        for (int64_t j = 0; j < n; ++j)
            crow[j] = (main_acc[j] + tile_acc[j]) + orc_add_rz(c1[j], c2[j]) * 0x1.0p-11f;
    }
    free(main_acc);
    free(tile_acc);
    free(c1);
    free(c2);
}

void orc_gemm_rows_f64(const float* a, const float* b, double* c, int64_t m, int64_t n, int64_t k,
                       int64_t row_begin, int64_t row_end) {
    /* kernels_scalar.cpp:137-148 */
    (void)m;
    for (int64_t i = row_begin; i < row_end; ++i) {
        double* crow = c + i * n;
        for (int64_t j = 0; j < n; ++j) crow[j] = 0.0;
        for (int64_t kk = 0; kk < k; ++kk) {
            const double av = a[i * k + kk];
            const float* brow = b + kk * n;
            for (int64_t j = 0; j < n; ++j) crow[j] += av * (double)brow[j];
        }
    }
}

/* ------------------------------------------------------------------ precsel */

static const float kFp16MinNormal = 0x1.0p-14f; /* precsel.cpp:21 */

static void stage1(const float* x, int64_t n, orc_exp_stats_t* s) {
    /* precsel.cpp:23-32 */
    memset(s, 0, sizeof(*s));
    s->n_total = (uint64_t)n;
    float max_abs = 0.0f;
    orc_abs_stats(x, n, kFp16MinNormal, &s->n_nonzero, &s->n1, &max_abs);
    int e = 0;
    s->e_max_valid = orc_exponent_of(max_abs, &e);
    s->e_max = s->e_max_valid ? e : 0;
}

static void stage2(const float* x, int64_t n, int target, orc_exp_stats_t* s) {
    /* precsel.cpp:34-45 */
    if (!s->e_max_valid) {
        s->n2 = 0;
        s->stage2_evaluated = 1;
        return;
    }
    const int window_floor = s->e_max - (target + 14);
    const float threshold = ldexpf(1.0f, window_floor); /* 0 below the f32 range */
    s->n2 = orc_count_abs_ge(x, n, threshold);
    s->stage2_evaluated = 1;
}

double orc_r1(const orc_exp_stats_t* s) {
    return s->n_nonzero ? (double)(s->n_nonzero - s->n1) / (double)s->n_nonzero : 0.0;
}
double orc_r2(const orc_exp_stats_t* s) {
    return s->n_nonzero ? (double)(s->n_nonzero - s->n2) / (double)s->n_nonzero : 0.0;
}

static int stage1_passes(const orc_exp_stats_t* s, double t, int target) {
    /* precsel.cpp:47-52 */
    if (s->n_nonzero == 0) return 1;
    if (orc_r1(s) > t) return 0;
    return !s->e_max_valid || s->e_max <= target;
}

void orc_exp_stats(const float* x, int64_t n, int target, orc_exp_stats_t* out) {
    stage1(x, n, out); /* precsel.cpp:89-93 */
    stage2(x, n, target, out);
}

void orc_exp_stats_staged(const float* x, int64_t n, int target, double t, orc_exp_stats_t* out) {
    /* precsel.cpp:95-104 */
    stage1(x, n, out);
    if (stage1_passes(out, t, target)) {
        out->n2 = out->n1;
        out->stage2_evaluated = 0;
        return;
    }
    stage2(x, n, target, out);
}

int orc_matrix_tolerance(const orc_exp_stats_t* s, double t, int target) {
    /* precsel.cpp:106-121 */
    if (s->n_nonzero == 0) return ORC_TOL_FP16_OK;
    if (stage1_passes(s, t, target)) return ORC_TOL_FP16_OK;
    if (!s->stage2_evaluated) return -1; /* std::logic_error */
    return orc_r2(s) <= t ? ORC_TOL_FP16_SCALED_OK : ORC_TOL_TF32_ONLY;
}

void orc_select_mode(int level_a, int e_valid_a, int e_a, int level_b, int e_valid_b, int e_b,
                     int target, int* kind, int* sa, int* sb) {
    /* precsel.cpp:123-135 */
    *sa = *sb = 0;
    if (level_a == ORC_TOL_FP16_OK && level_b == ORC_TOL_FP16_OK) {
        *kind = ORC_KIND_FP16_TCEC;
        return;
    }
    if (level_a >= ORC_TOL_FP16_SCALED_OK && level_b >= ORC_TOL_FP16_SCALED_OK) {
        *kind = ORC_KIND_FP16_TCEC_SCALED;
        *sa = e_valid_a ? target - e_a : 0;
        *sb = e_valid_b ? target - e_b : 0;
        return;
    }
    *kind = ORC_KIND_TF32_TCEC;
}

/* ------------------------------------------------------------- gemm / cgemm */

int orc_gemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int mode,
             int k_tile, int* overflow) {
    /* gemm.cpp:60-125 */
    if (mode == ORC_MODE_FP32_REF) {
        orc_gemm_rows_rn(a, b, c, m, n, k, 0, m);
        return 0;
    }
    if (mode == ORC_MODE_FP64_ORACLE) {
        double* t = (double*)malloc(sizeof(double) * (size_t)(m * n > 0 ? m * n : 1));
        orc_gemm_rows_f64(a, b, t, m, n, k, 0, m);
        for (int64_t i = 0; i < m * n; ++i) c[i] = (float)t[i];
        free(t);
        return 0;
    }
    if (k_tile < 1) return 3; /* gemm.cpp:18-20 std::invalid_argument */
    const int fmt = (mode == ORC_MODE_TF32_TC || mode == ORC_MODE_TF32_TCEC) ? ORC_FMT_TF32
                                                                            : ORC_FMT_FP16;
    const size_t na = (size_t)(m * k), nb = (size_t)(k * n);
    if (mode == ORC_MODE_TF32_TC || mode == ORC_MODE_FP16_TC) {
        /* gemm.cpp:76-90 */
        float* al = (float*)malloc(sizeof(float) * (na ? na : 1));
        float* bl = (float*)malloc(sizeof(float) * (nb ? nb : 1));
        orc_quantize_buf(a, al, (int64_t)na, fmt, ORC_RN, overflow);
        orc_quantize_buf(b, bl, (int64_t)nb, fmt, ORC_RN, overflow);
        orc_gemm_rows_rz(al, bl, c, m, n, k, 0, m);
        free(al);
        free(bl);
        return 0;
    }
    /* gemm.cpp:92-106 */
    float* ah = (float*)malloc(sizeof(float) * (na ? na : 1));
    float* al = (float*)malloc(sizeof(float) * (na ? na : 1));
    float* bh = (float*)malloc(sizeof(float) * (nb ? nb : 1));
    float* bl = (float*)malloc(sizeof(float) * (nb ? nb : 1));
    orc_split_buf(a, ah, al, (int64_t)na, fmt, overflow);
    orc_split_buf(b, bh, bl, (int64_t)nb, fmt, overflow);
    orc_gemm_rows_tcec(ah, al, bh, bl, c, m, n, k, k_tile, 0, m);
    free(ah);
    free(al);
    free(bh);
    free(bl);
    return 0;
}

static void deinterleave(const float* x, int64_t n_elems, float* re, float* im) {
    /* cgemm.cpp:14-21 */
    for (int64_t i = 0; i < n_elems; ++i) {
        re[i] = x[2 * i];
        im[i] = x[2 * i + 1];
    }
}

int orc_cgemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int mode,
              int k_tile, int* overflow) {
    /* cgemm.cpp:25-46 */
    const int64_t na = m * k, nb = k * n, nc = m * n;
    float* buf = (float*)malloc(sizeof(float) * (size_t)(2 * na + 2 * nb + 4 * nc + 8));
    float *are = buf, *aim = are + na, *bre = aim + na, *bim = bre + nb;
    float *p1 = bim + nb, *p2 = p1 + nc, *p3 = p2 + nc, *p4 = p3 + nc;
    deinterleave(a, na, are, aim);
    deinterleave(b, nb, bre, bim);
    int rc = orc_gemm(are, bre, p1, m, n, k, mode, k_tile, overflow);
    if (!rc) rc = orc_gemm(aim, bim, p2, m, n, k, mode, k_tile, overflow);
    if (!rc) rc = orc_gemm(are, bim, p3, m, n, k, mode, k_tile, overflow);
    if (!rc) rc = orc_gemm(aim, bre, p4, m, n, k, mode, k_tile, overflow);
    if (!rc) {
        for (int64_t i = 0; i < nc; ++i) {
            c[2 * i] = p1[i] - p2[i];
            c[2 * i + 1] = p3[i] + p4[i];
        }
    }
    free(buf);
    return rc;
}

void orc_cgemm_oracle(const float* a, const float* b, double* c, int64_t m, int64_t n, int64_t k) {
    /* cgemm.cpp:62-74 */
    const int64_t na = m * k, nb = k * n, nc = m * n;
    float* buf = (float*)malloc(sizeof(float) * (size_t)(2 * na + 2 * nb + 8));
    double* p = (double*)malloc(sizeof(double) * (size_t)(4 * nc + 4));
    float *are = buf, *aim = are + na, *bre = aim + na, *bim = bre + nb;
    double *p1 = p, *p2 = p1 + nc, *p3 = p2 + nc, *p4 = p3 + nc;
    deinterleave(a, na, are, aim);
    deinterleave(b, nb, bre, bim);
    orc_gemm_rows_f64(are, bre, p1, m, n, k, 0, m);
    orc_gemm_rows_f64(aim, bim, p2, m, n, k, 0, m);
    orc_gemm_rows_f64(are, bim, p3, m, n, k, 0, m);
    orc_gemm_rows_f64(aim, bre, p4, m, n, k, 0, m);
    for (int64_t i = 0; i < nc; ++i) {
        c[2 * i] = p1[i] - p2[i];
        c[2 * i + 1] = p3[i] + p4[i];
    }
    free(buf);
    free(p);
}

double orc_relative_error_c(const float* c, const double* ref, int64_t n_elems) {
    /* cgemm.cpp:76-89; returns NaN for a zero reference (ZeroReference) */
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n_elems; ++i) {
        const double dre = (double)c[2 * i] - ref[2 * i];
        const double dim = (double)c[2 * i + 1] - ref[2 * i + 1];
        num += dre * dre + dim * dim;
        den += ref[2 * i] * ref[2 * i] + ref[2 * i + 1] * ref[2 * i + 1];
    }
    if (den == 0.0) return NAN;
    return sqrt(num) / sqrt(den);
}

/* ------------------------------------------------------------ dispatch_cgemm */

static const char* kind_name(int kind) {
    /* precsel.cpp:63-71 */
    switch (kind) {
    case ORC_KIND_FP16_TCEC: return "FP16TCEC";
    case ORC_KIND_FP16_TCEC_SCALED: return "FP16TCEC_SCALED";
    case ORC_KIND_TF32_TCEC: return "TF32TCEC";
    default: return "FP32_BASELINE";
    }
}

static const char* forced_name(int f) {
    /* precsel.cpp:73-84 */
    static const char* names[] = {"FP32_REF", "FP64_ORACLE", "TF32TC", "FP16TC",
                                  "TF32TCEC", "FP16TCEC",    "FP16TCEC_SCALED"};
    return (f >= 0 && f <= 6) ? names[f] : "?";
}

static void fmt_ratio(char* out, size_t cap, const orc_exp_stats_t* s, int has, int second) {
    /* precsel.cpp:186-192 */
    if (!has || (second && !s->stage2_evaluated)) {
        snprintf(out, cap, "-");
        return;
    }
    snprintf(out, cap, "%.9g", second ? orc_r2(s) : orc_r1(s));
}

static void fmt_emax(char* out, size_t cap, const orc_exp_stats_t* s, int has) {
    /* precsel.cpp:193-196 */
    if (!has || !s->e_max_valid)
        snprintf(out, cap, "-");
    else
        snprintf(out, cap, "%d", s->e_max);
}

/* precsel.cpp:209-216; returns 1 on ScaleOverflow */
static int run_scaled(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                      int sa, int sb, int k_tile, int* overflow) {
    const int64_t na = 2 * m * k, nb = 2 * k * n;
    float* as = (float*)malloc(sizeof(float) * (size_t)(na + nb + 2));
    float* bs = as + na;
    orc_scale_buf(a, as, na, sa);
    orc_scale_buf(b, bs, nb, sb);
    for (int64_t i = 0; i < na; ++i)
        if (!isfinite(as[i])) { free(as); return 1; } /* precsel.cpp:54-57 */
    for (int64_t i = 0; i < nb; ++i)
        if (!isfinite(bs[i])) { free(as); return 1; }
    int rc = orc_cgemm(as, bs, c, m, n, k, ORC_MODE_FP16_TCEC, k_tile, overflow);
    free(as);
    if (rc) return rc;
    orc_scale_buf(c, c, 2 * m * n, -(sa + sb)); /* precsel.cpp:171-174 */
    return 0;
}

/* compute == 0: the selection half only (statistics, decision, log line), C untouched */
static int dispatch_impl(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                         const orc_dispatch_config_t* cfg, orc_dispatch_result_t* res, int compute) {
    /* precsel.cpp:225-322 */
    memset(res, 0, sizeof(*res));
    const int target = cfg->target_max_exponent;
    const int kt = cfg->k_tile;
    const char* label = "?";
    int rc = 0;
    int64_t mn = m < n ? m : n;
    if (k < mn) mn = k;

    if (cfg->force >= 0) {
        label = forced_name(cfg->force);
        switch (cfg->force) {
        case 0: rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_FP32_REF, kt, &res->overflow);
                res->kind = ORC_KIND_FP32_BASELINE; break;
        case 1: rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_FP64_ORACLE, kt, &res->overflow);
                res->kind = ORC_KIND_FP32_BASELINE; break;
        case 2: rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_TF32_TC, kt, &res->overflow);
                res->kind = ORC_KIND_TF32_TCEC; break;
        case 3: rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_FP16_TC, kt, &res->overflow);
                res->kind = ORC_KIND_FP16_TCEC; break;
        case 4: rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_TF32_TCEC, kt, &res->overflow);
                res->kind = ORC_KIND_TF32_TCEC; break;
        case 5: rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_FP16_TCEC, kt, &res->overflow);
                res->kind = ORC_KIND_FP16_TCEC; break;
        case 6: {
            orc_exp_stats_staged(a, 2 * m * k, target, 1.0, &res->stats_a);
            orc_exp_stats_staged(b, 2 * k * n, target, 1.0, &res->stats_b);
            res->has_stats = 1;
            res->scale_a = res->stats_a.e_max_valid ? target - res->stats_a.e_max : 0;
            res->scale_b = res->stats_b.e_max_valid ? target - res->stats_b.e_max : 0;
            rc = !compute ? 0 : run_scaled(a, b, c, m, n, k, res->scale_a, res->scale_b, kt, &res->overflow);
            res->kind = ORC_KIND_FP16_TCEC_SCALED;
            break;
        }
        default: return 4;
        }
    } else if (mn >= cfg->size_auto) {
        orc_exp_stats_staged(a, 2 * m * k, target, cfg->threshold_t, &res->stats_a);
        orc_exp_stats_staged(b, 2 * k * n, target, cfg->threshold_t, &res->stats_b);
        res->has_stats = 1;
        const int la = orc_matrix_tolerance(&res->stats_a, cfg->threshold_t, target);
        const int lb = orc_matrix_tolerance(&res->stats_b, cfg->threshold_t, target);
        if (la < 0 || lb < 0) return 2;
        orc_select_mode(la, res->stats_a.e_max_valid, res->stats_a.e_max, lb,
                        res->stats_b.e_max_valid, res->stats_b.e_max, target, &res->kind,
                        &res->scale_a, &res->scale_b);
        label = kind_name(res->kind);
        switch (res->kind) {
        case ORC_KIND_FP16_TCEC:
            rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_FP16_TCEC, kt, &res->overflow); break;
        case ORC_KIND_TF32_TCEC:
            rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_TF32_TCEC, kt, &res->overflow); break;
        case ORC_KIND_FP16_TCEC_SCALED:
            rc = !compute ? 0 : run_scaled(a, b, c, m, n, k, res->scale_a, res->scale_b, kt, &res->overflow);
            break;
        default:
            rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_FP32_REF, kt, &res->overflow); break;
        }
    } else if (mn >= cfg->size_tf32) {
        res->kind = ORC_KIND_TF32_TCEC;
        label = kind_name(res->kind);
        rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_TF32_TCEC, kt, &res->overflow);
    } else {
        res->kind = ORC_KIND_FP32_BASELINE;
        label = kind_name(res->kind);
        rc = !compute ? 0 : orc_cgemm(a, b, c, m, n, k, ORC_MODE_FP32_REF, kt, &res->overflow);
    }
    if (rc) return rc;

    /* DecisionRecord::to_line, precsel.cpp:185-205 */
    char r1a[32], r2a[32], r1b[32], r2b[32], ea[16], eb[16];
    fmt_ratio(r1a, sizeof r1a, &res->stats_a, res->has_stats, 0);
    fmt_ratio(r2a, sizeof r2a, &res->stats_a, res->has_stats, 1);
    fmt_ratio(r1b, sizeof r1b, &res->stats_b, res->has_stats, 0);
    fmt_ratio(r2b, sizeof r2b, &res->stats_b, res->has_stats, 1);
    fmt_emax(ea, sizeof ea, &res->stats_a, res->has_stats);
    fmt_emax(eb, sizeof eb, &res->stats_b, res->has_stats);
    snprintf(res->line, sizeof res->line, "%lld,%lld,%lld,%s,%d,%d,%s,%s,%s,%s,%s,%s",
             (long long)m, (long long)n, (long long)k, label, res->scale_a, res->scale_b, r1a, r2a,
             r1b, r2b, ea, eb);
    return 0;
}

int orc_dispatch_cgemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                       const orc_dispatch_config_t* cfg, orc_dispatch_result_t* res) {
    return dispatch_impl(a, b, c, m, n, k, cfg, res, 1);
}

/* the decision of dispatch_cgemm (stats, selection, DecisionRecord line) without the GEMM */
int orc_dispatch_decision(const float* a, const float* b, int64_t m, int64_t n, int64_t k,
                          const orc_dispatch_config_t* cfg, orc_dispatch_result_t* res) {
    return dispatch_impl(a, b, NULL, m, n, k, cfg, res, 0);
}

/* ------------------------------------------------------------------ permute */

void orc_permute_c64(const float* src, float* dst, int rank, const int64_t* old_dims,
                     const int* axis_of) {
    /* tensor.hpp:56-105: odometer over the output index, tracking the input
     * offset (8-byte complex elements) */
    int64_t old_stride[64], new_dims[64], stride[64], idx[64];
    int64_t total = 1;
    for (int a = 0; a < rank; ++a) total *= old_dims[a];
    if (rank == 0) {
        dst[0] = src[0];
        dst[1] = src[1];
        return;
    }
    old_stride[rank - 1] = 1;
    for (int a = rank - 2; a >= 0; --a) old_stride[a] = old_stride[a + 1] * old_dims[a + 1];
    for (int a = 0; a < rank; ++a) {
        new_dims[a] = old_dims[axis_of[a]];
        stride[a] = old_stride[axis_of[a]];
        idx[a] = 0;
    }
    int64_t in_off = 0;
    for (int64_t pos = 0; pos < total; ++pos) {
        dst[2 * pos] = src[2 * in_off];
        dst[2 * pos + 1] = src[2 * in_off + 1];
        for (int a = rank - 1; a >= 0; --a) {
            if (++idx[a] < new_dims[a]) {
                in_off += stride[a];
                break;
            }
            in_off -= stride[a] * (new_dims[a] - 1);
            idx[a] = 0;
        }
    }
}

/* ---------------------------------------------------------------------- rng */

/* std::mt19937_64 (fully specified by [rand.predef]); rng.hpp:13-56 */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void orc_rng_seed(orc_rng_t* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
    r->have_spare = 0;
    r->spare = 0.0;
}

uint64_t orc_rng_next_u64(orc_rng_t* r) {
    if (r->mti >= MT_N) {
        int i;
        uint64_t x;
        for (i = 0; i < MT_N - MT_M; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        }
        for (; i < MT_N - 1; ++i) {
            x = (r->mt[i] & MT_UM) | (r->mt[i + 1] & MT_LM);
            r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        }
        x = (r->mt[MT_N - 1] & MT_UM) | (r->mt[0] & MT_LM);
        r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

uint64_t orc_rng_next_below(orc_rng_t* r, uint64_t n) {
    /* rng.hpp:20-26 */
    const uint64_t limit = n * (UINT64_MAX / n);
    uint64_t v = orc_rng_next_u64(r);
    while (v >= limit) v = orc_rng_next_u64(r);
    return v % n;
}

double orc_rng_uniform01(orc_rng_t* r) {
    return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; /* rng.hpp:29 */
}

static double uniform01_pos(orc_rng_t* r) {
    return (double)((orc_rng_next_u64(r) >> 11) + 1) * 0x1.0p-53; /* rng.hpp:32 */
}

float orc_rng_uniform_pm1f(orc_rng_t* r) {
    return (float)(2.0 * orc_rng_uniform01(r) - 1.0); /* rng.hpp:35 */
}

double orc_rng_gaussian(orc_rng_t* r, double stddev) {
    /* rng.hpp:38-50 Box-Muller with a cached spare */
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare * stddev;
    }
    const double u1 = uniform01_pos(r);
    const double u2 = orc_rng_uniform01(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(ang);
    r->have_spare = 1;
    return rad * cos(ang) * stddev;
}

void orc_fill_uniform_c32(orc_rng_t* r, float* dst, int64_t n_elems) {
    /* experiments.cpp:27-31: {uniform_pm1f(), uniform_pm1f()} per element;
     * braced init evaluates left to right */
    for (int64_t i = 0; i < n_elems; ++i) {
        dst[2 * i] = orc_rng_uniform_pm1f(r);
        dst[2 * i + 1] = orc_rng_uniform_pm1f(r);
    }
}
