// HBM-bound kernels of the TCEC path: format conversion, exponent statistics,
// device-side precision selection, operand preparation (scale + split + complex
// block expansion), the bit-exact SIMT GEMM tiers, and the TTGT permute.
//
// Reference mapping (KernelTable, proj/include/mpsgemm/kernels.hpp:20-63):
//   quantize_buf / split_buf / scale_buf / add_buf / sub_buf -> *_kernel below
//   abs_stats + count_abs_ge (stage1/stage2, precsel.cpp:23-45) -> stats1/stats2
//   matrix_tolerance + select_mode (precsel.cpp:106-135)      -> select_body (stats2's last block)
//   gemm_rows_rn (+ cgemm.cpp assembly)                        -> cgemm_fp32_ref_kernel
//   gemm_rows_f64                                               -> cgemm_fp64_kernel
//   permute (tensor.hpp:56-105)                                 -> permute_kernel
#include <cstdlib>
#include <type_traits>

#include "tcec_common.cuh"
#include "tcec_internal.h"

namespace tcec {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work, int per_block, int max_blocks = 148 * 16) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return int(g);
}

TCEC_DEV unsigned warp_or(unsigned v) { return __reduce_or_sync(0xFFFFFFFFu, v); }

TCEC_DEV void flag_or(unsigned* flag, unsigned v) {
    // one atomic per warp at most; the flag is an OR-accumulated out-parameter
    const unsigned any = warp_or(v);
    if (any && flag && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// offset of index idx in a run map (runs outermost first, innermost last)
TCEC_DEV int64_t run_offset(const RunMap& rm, uint32_t idx) {
    int64_t off = 0;
#pragma unroll
    for (int r = kMaxRuns - 1; r >= 0; --r) {
        if (r < rm.n) {
            uint32_t dgt;
            if (rm.pow2) {
                dgt = idx & ((1u << rm.shift[r]) - 1u);
                idx >>= rm.shift[r];
            } else {
                dgt = idx % rm.ext[r];
                idx /= rm.ext[r];
            }
            off += int64_t(dgt) * rm.stride[r];
        }
    }
    return off;
}

// 4 consecutive complex elements (row, kc .. kc + 3) of a matrix view of a
// tensor (zero past column k): one run offset and four loads when the four
// sit in the innermost unit-stride run, else one offset each
TCEC_DEV void load4_view(const float* a, const MatrixView& v, int64_t row, int64_t kc, int64_t k,
                         float (&x)[8]) {
    const float2* t = reinterpret_cast<const float2*>(a);
    const int64_t ro = run_offset(v.rows, uint32_t(row));
    const int n = v.cols.n;
    if (kc + 4 <= k && n > 0 && v.cols.stride[n - 1] == 1 &&
        (uint32_t(kc) % v.cols.ext[n - 1]) + 4u <= v.cols.ext[n - 1]) {
        const float2* q = t + ro + run_offset(v.cols, uint32_t(kc));
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 w = __ldcs(q + e);
            x[2 * e] = w.x;
            x[2 * e + 1] = w.y;
        }
        return;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 w = kc + e < k ? __ldcs(t + ro + run_offset(v.cols, uint32_t(kc + e))) : make_float2(0.0f, 0.0f);
        x[2 * e] = w.x;
        x[2 * e + 1] = w.y;
    }
}

// ------------------------------------------------------------ elementwise

__global__ void quantize_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n,
                                int fmt, int rz, unsigned* ovf) {
    unsigned o = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = quantize(src[i], fmt, rz != 0, o);
    flag_or(ovf, o);
}

__global__ void split_flat_kernel(const float* __restrict__ src, float* __restrict__ hi,
                                  float* __restrict__ lo, int64_t n, int fmt, unsigned* ovf) {
    unsigned o = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        float h, l;
        if (fmt == kFp16)
            split<kFp16>(src[i], h, l, o);
        else
            split<kTf32>(src[i], h, l, o);
        hi[i] = h;
        lo[i] = l;
    }
    flag_or(ovf, o);
}

__global__ void scale_kernel(const float* src, float* dst, int64_t n, double factor,
                             unsigned* nonfinite) {
    unsigned bad = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const float v = scale_pow2(src[i], factor);
        dst[i] = v;
        bad |= isfinite(v) ? 0u : 1u;
    }
    flag_or(nonfinite, bad);
}

__global__ void add_sub_kernel(const float* a, const float* b, float* dst, int64_t n, int sub) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = sub ? __fsub_rn(a[i], b[i]) : __fadd_rn(a[i], b[i]);
}

// ------------------------------------------------------------- statistics

// bits of |x|; "valid" = nonzero and not NaN, i.e. the reference's a > 0.0f
TCEC_DEV bool valid_mag(uint32_t m) { return (m - 1u) < 0x7F800000u; }

constexpr uint32_t kFp16MinNormalBits = 0x38800000u;  // 2^-14, precsel.cpp:21

template <typename T>
TCEC_DEV T block_sum(T v, T* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    T r = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < int(blockDim.x >> 5); ++i) r += red[i];
    return r;
}

TCEC_DEV unsigned block_max(unsigned v, unsigned* red) {
    v = __reduce_max_sync(0xFFFFFFFFu, v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    unsigned r = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < int(blockDim.x >> 5); ++i) r = max(r, red[i]);
    return r;
}

// Both statistics stages sweep the two operands in one 1-D grid: blocks
// [0, nb_a) take contiguous float4 chunks of A, the rest of B, so each
// operand gets blocks in proportion to its size (a 2 MB A next to a 64 MB B
// no longer idles half the grid), and every thread keeps four independent
// 16-B loads in flight (these sweeps were latency-bound at mid sizes).
template <typename Visit>
TCEC_DEV void sweep_operand(const float* __restrict__ x, int64_t n, int part, int nparts, bool keep, Visit&& visit) {
    // keep: normal L2 policy (the next sweep / the preparation re-reads an
    // operand that fits in L2); else evict-first streaming loads
    auto ld = [keep](const float4* p) { return keep ? __ldg(p) : __ldcs(p); };
    const bool vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
    const int64_t n4 = vec ? n / 4 : 0;
    const int64_t per = (n4 + nparts - 1) / nparts;
    const int64_t b0 = min(n4, int64_t(part) * per), b1 = min(n4, b0 + per);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int bd = int(blockDim.x);
    int64_t i = b0 + threadIdx.x;
    for (; i + 3 * bd < b1; i += 4 * bd) {
        const float4 v0 = ld(x4 + i), v1 = ld(x4 + i + bd), v2 = ld(x4 + i + 2 * bd), v3 = ld(x4 + i + 3 * bd);
        visit(v0.x); visit(v0.y); visit(v0.z); visit(v0.w);
        visit(v1.x); visit(v1.y); visit(v1.z); visit(v1.w);
        visit(v2.x); visit(v2.y); visit(v2.z); visit(v2.w);
        visit(v3.x); visit(v3.y); visit(v3.z); visit(v3.w);
    }
    for (; i < b1; i += bd) {
        const float4 v = ld(x4 + i);
        visit(v.x); visit(v.y); visit(v.z); visit(v.w);
    }
    if (part == nparts - 1)  // scalar tail (and the whole operand when unaligned)
        for (int64_t j = n4 * 4 + threadIdx.x; j < n; j += bd) visit(x[j]);
}

// stage 1 (precsel.cpp:23-32 via abs_stats, kernels_scalar.cpp:50-65):
// nonzero count, count of |x| >= 2^-14, max |x|
// (block `bid` of `nblk`: blocks [0, nb_a) sweep A, the rest B)
TCEC_DEV void stats1_part(const float* a, int64_t na, const float* b, int64_t nb, DevDecision* d,
                          int nb_a, int bid, int nblk, bool keep) {
    const int op = bid < nb_a ? 0 : 1;
    const float* x = op ? b : a;
    const int64_t n = op ? nb : na;
    const int part = op ? bid - nb_a : bid;
    const int nparts = op ? nblk - nb_a : nb_a;
    if (x == nullptr || n == 0 || nparts <= 0) return;
    unsigned nz = 0, n1 = 0, mx = 0;
    sweep_operand(x, n, part, nparts, keep, [&](float v) {
        const uint32_t m = __float_as_uint(v) & 0x7FFFFFFFu;
        const bool ok = valid_mag(m);
        nz += ok;
        n1 += ok && m >= kFp16MinNormalBits;
        mx = max(mx, ok ? m : 0u);
    });
    __shared__ unsigned long long red64[kThreads / 32];
    __shared__ unsigned red32[kThreads / 32];
    const unsigned long long snz = block_sum<unsigned long long>(nz, red64);
    const unsigned long long sn1 = block_sum<unsigned long long>(n1, red64);
    const unsigned smx = block_max(mx, red32);
    if (threadIdx.x == 0) {
        DevStats& st = d->st[op];
        if (snz) atomicAdd(&st.n_nonzero, snz);
        if (sn1) atomicAdd(&st.n1, sn1);
        if (smx) atomicMax(&st.max_bits, smx);
    }
}

__global__ void __launch_bounds__(kThreads) stats1_kernel(const float* a, int64_t na,
                                                          const float* b, int64_t nb,
                                                          DevDecision* d, int nb_a, int keep) {
    stats1_part(a, na, b, nb, d, nb_a, int(blockIdx.x), int(gridDim.x), keep != 0);
}


// stage1_passes (precsel.cpp:47-52); r1 in double exactly as precsel.hpp:27-30
TCEC_DEV bool stage1_passes(unsigned long long nz, unsigned long long n1, unsigned max_bits,
                            double t, int target) {
    if (nz == 0) return true;
    const double r1 = double(nz - n1) / double(nz);
    if (r1 > t) return false;
    return max_bits == 0 || exponent_of_bits(max_bits) <= target;
}

// binades above the stage-2 threshold whose sample count feeds the host
// pipeline's speculation (5: above the 2^-24 grid of float32 uniforms in [-1, 1])
constexpr int kSpecBinades = 5;

// stage 2 (precsel.cpp:34-45 via count_abs_ge): count of |x| >= 2^(e_max - target - 14)
TCEC_DEV void stats2_part(const float* a, int64_t na, const float* b, int64_t nb, DevDecision* d,
                          double t, int target, int always, int nb_a, int bid, int nblk, bool keep,
                          bool spec = false) {
    const int op = bid < nb_a ? 0 : 1;
    const float* x = op ? b : a;
    const int64_t n = op ? nb : na;
    const int part = op ? bid - nb_a : bid;
    const int nparts = op ? nblk - nb_a : nb_a;
    if (x == nullptr || n == 0 || nparts <= 0) return;
    // one thread reads the stage-1 statistics and derives the threshold
    // (every thread reading them put ~2.4 M same-address loads per 66 MB
    // sweep in front of the data stream: 2x the stage-1 time at 2^24 elements)
    __shared__ uint32_t thr_s, thr_hi_s;
    if (threadIdx.x == 0) {
        const DevStats st = d->st[op];
        uint32_t th = 0, th_hi = 0;  // 0: this operand needs no stage 2 (stage 1 passed, or no e_max: n2 = 0)
        if ((always || !stage1_passes(st.n_nonzero, st.n1, st.max_bits, t, target)) && st.max_bits != 0) {
            const int w = exponent_of_bits(st.max_bits) - (target + 14);
            // ldexp(1.0f, w): a normal, a subnormal power of two, or 0 (all nonzero pass)
            auto pow2_bits = [](int e) -> uint32_t {
                return e >= -126 ? (e > 127 ? 0x7F800000u : uint32_t(e + 127) << 23)
                                 : (e >= -149 ? 1u << (e + 149) : 1u);
            };
            th = pow2_bits(w);
            th_hi = pow2_bits(w + kSpecBinades);
        }
        thr_s = th;
        thr_hi_s = th_hi;
    }
    __syncthreads();
    const uint32_t thr = thr_s, thr_hi = thr_hi_s;
    if (thr == 0) return;
    unsigned cnt = 0, lo = 0;
    sweep_operand(x, n, part, nparts, keep, [&](float v) {
        const uint32_t m = __float_as_uint(v) & 0x7FFFFFFFu;
        cnt += valid_mag(m) && m >= thr;
        if (spec) lo += valid_mag(m) && m < thr_hi;
    });
    __shared__ unsigned long long red64[kThreads / 32];
    const unsigned long long s = block_sum<unsigned long long>(cnt, red64);
    if (threadIdx.x == 0 && s) atomicAdd(&d->st[op].n2, s);
    if (spec) {
        // speculation only: components below 2^(w + kSpecBinades), kept in the
        // slot's otherwise unused n_total (the host reports n_total itself)
        const unsigned long long sl = block_sum<unsigned long long>(lo, red64);
        if (threadIdx.x == 0 && sl) atomicAdd(&d->st[op].n_total, sl);
    }
}

TCEC_DEV void select_body(DevDecision* d, double t, int target, int forced_scaled, int stage2_always);

// select = 1: the last block to finish also runs the selection (one launch
// and one dependent kernel start less per dispatch); it reads the decision
// slot past L1 (thread 0 of every block read its stage-1 line at the start)
__global__ void __launch_bounds__(kThreads, 8) stats2_kernel(const float* a, int64_t na,
                                                          const float* b, int64_t nb,
                                                          DevDecision* d, double t, int target,
                                                          int always, int nb_a, int keep, int select,
                                                          double sel_t, int forced_scaled, float spec_fa,
                                                          float spec_fb) {
    stats2_part(a, na, b, nb, d, t, target, always, nb_a, int(blockIdx.x), int(gridDim.x), keep != 0,
                spec_fa > 0.0f && spec_fb > 0.0f);
    if (!select) return;
    constexpr int kWords = int(sizeof(DevDecision) / 4);
    __shared__ int last_s;
    __shared__ __align__(16) unsigned dec_s[kWords];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this block's n2 before its ticket
        last_s = atomicAdd(&d->pad_, 1) == int(gridDim.x) - 1;
    }
    __syncthreads();
    if (!last_s) return;
    __threadfence();
    if (int(threadIdx.x) < kWords) dec_s[threadIdx.x] = __ldcg(reinterpret_cast<const unsigned*>(d) + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        DevDecision* dd = reinterpret_cast<DevDecision*>(dec_s);
        select_body(dd, sel_t, target, forced_scaled, 0);
        // spec_fa / spec_fb > 0: the operands are SAMPLES (these fractions of
        // A and B) and the decision is the host pipeline's speculation.  At
        // t = 0 an FP16 kind after stage 2 only says the sample has no
        // component below the threshold 2^w, w = e_max - target - 14.  The
        // sample's count below 2^(w + kSpecBinades), extrapolated with a flat
        // density near zero, expects count / f / 2^kSpecBinades such
        // components in the whole operands; from 0.5 on, the speculation takes
        // TF32.  (Data on a coarse grid -- float32 uniforms have no magnitude
        // below 2^-23 -- shows no count there and keeps FP16.)  Either way the
        // speculation is checked against the exact decision (rerun on mismatch).
        if (spec_fa > 0.0f && spec_fb > 0.0f && !forced_scaled && sel_t == 0.0 && dd->kind >= 0 &&
            dd->kind != kKindTf32 && (dd->st[0].stage2_evaluated || dd->st[1].stage2_evaluated)) {
            double expect = 0.0;
            for (int op = 0; op < 2; ++op) {
                const DevStats& st = dd->st[op];
                const double f = op ? double(spec_fb) : double(spec_fa);
                expect += double(st.n_total) / f / double(1 << kSpecBinades);
            }
            if (expect >= 0.5) {
                dd->kind = kKindTf32;
                dd->scale_a = dd->scale_b = 0;
            }
        }
        // the scaled kind's shifts come from e_max, a maximum: a sample whose
        // largest magnitude sits at the very top of its binade (uniform data in
        // [-1, 1], whose whole operand holds exact 1.0s) predicts the next
        // binade for the whole operand
        if (spec_fa > 0.0f && spec_fb > 0.0f && dd->kind == kKindFp16Scaled) {
            for (int op = 0; op < 2; ++op) {
                const DevStats& st = dd->st[op];
                const float f = op ? spec_fb : spec_fa;
                if (st.e_max_valid && f <= 0.5f && (st.max_bits & 0x7FFFFFu) >= 0x7FF800u &&
                    st.max_bits < 0x7F000000u) {
                    if (op) dd->scale_b -= 1;
                    else dd->scale_a -= 1;
                }
            }
        }
        dd->pad_ = 0;
    }
    __syncthreads();
    if (int(threadIdx.x) < kWords) reinterpret_cast<unsigned*>(d)[threadIdx.x] = dec_s[threadIdx.x];
}

// finalize ExpStats, tolerance levels and the pair rule (precsel.cpp:95-135)
TCEC_DEV void select_body(DevDecision* d, double t, int target, int forced_scaled, int stage2_always) {
    int level[2];
    for (int op = 0; op < 2; ++op) {
        DevStats& st = d->st[op];
        st.e_max_valid = st.max_bits != 0;
        st.e_max = st.e_max_valid ? exponent_of_bits(st.max_bits) : 0;
        const double ts = forced_scaled ? 1.0 : t;
        const bool pass = stage1_passes(st.n_nonzero, st.n1, st.max_bits, ts, target);
        if (!stage2_always && pass) {
            st.n2 = st.n1;  // lower bound, stage 2 skipped (precsel.cpp:97-101)
            st.stage2_evaluated = 0;
        } else {
            st.stage2_evaluated = 1;  // n2 counted by stats2 (0 when no e_max)
        }
        // matrix_tolerance (precsel.cpp:106-121)
        if (st.n_nonzero == 0 || stage1_passes(st.n_nonzero, st.n1, st.max_bits, t, target)) {
            level[op] = 2;
        } else if (!st.stage2_evaluated) {
            level[op] = -1;
        } else {
            const double r2 = double(st.n_nonzero - st.n2) / double(st.n_nonzero);
            level[op] = r2 <= t ? 1 : 0;
        }
    }
    d->level_a = level[0];
    d->level_b = level[1];
    const int sa = d->st[0].e_max_valid ? target - d->st[0].e_max : 0;
    const int sb = d->st[1].e_max_valid ? target - d->st[1].e_max : 0;
    if (forced_scaled) {
        d->kind = kKindFp16Scaled;
        d->scale_a = sa;
        d->scale_b = sb;
        return;
    }
    if (level[0] < 0 || level[1] < 0) {
        d->kind = -1;  // std::logic_error in matrix_tolerance
        return;
    }
    if (level[0] == 2 && level[1] == 2) {
        d->kind = kKindFp16;
        d->scale_a = d->scale_b = 0;
    } else if (level[0] >= 1 && level[1] >= 1) {
        d->kind = kKindFp16Scaled;
        d->scale_a = sa;
        d->scale_b = sb;
    } else {
        d->kind = kKindTf32;
        d->scale_a = d->scale_b = 0;
    }
}


// --------------------------------------------------------- operand prep

struct PrepMode {
    int fmt;       // kFp16 / kTf32
    int scale;     // power-of-two shift (FP16TCEC_SCALED)
    bool active;   // false: this dispatch does not use tensor cores
    bool scaled;   // FP16TCEC_SCALED: the operand goes through scale_matrix, which
                   // throws ScaleOverflow on any nonfinite result -- even for a
                   // zero shift (precsel.cpp:209-216, 139-152)
};

TCEC_DEV PrepMode prep_mode(const DevDecision* d, int kind_fixed, bool is_b) {
    const int kind = kind_fixed >= 0 ? kind_fixed : d->kind;
    PrepMode p;
    p.active = kind == kKindFp16 || kind == kKindFp16Scaled || kind == kKindTf32;
    p.fmt = kind == kKindTf32 ? kTf32 : kFp16;
    p.scale = kind == kKindFp16Scaled ? (is_b ? d->scale_b : d->scale_a) : 0;
    p.scaled = kind == kKindFp16Scaled;
    return p;
}

// scale (optional) + split/quantize one component; returns hi, lo
TCEC_DEV void convert(float x, const PrepMode& pm, double factor, bool corrected, float& hi,
                      float& lo, unsigned& ovf, unsigned& bad) {
    if (pm.scale != 0) x = scale_pow2(x, factor);
    if (pm.scaled) bad |= isfinite(x) ? 0u : 1u;
    if (corrected) {
        if (pm.fmt == kFp16)
            split<kFp16>(x, hi, lo, ovf);
        else
            split<kTf32>(x, hi, lo, ovf);
    } else {
        hi = quantize(x, pm.fmt, false, ovf);
        lo = 0.0f;
    }
}

// Vectorised fast path of convert() for N components (N even).  The scale is
// one float multiply by 2^s when 2^s is a float (s in [-149, 127]): that is
// one rounding of the same exact product as float(double(x) * 2^s)
// (scale_buf, kernels_scalar.cpp:34-40).  When no magnitude exceeds the
// format maximum (and none is NaN/Inf -- checked on the bit patterns), the
// split needs no saturation test: FP16 via paired cvt.rn.f16x2.f32, TF32 via
// the integer round-to-nearest-even at bit 13 (lowprec.hpp:58-88).  Otherwise
// the whole group takes the per-component reference path.  Outputs hi/lo as
// floats holding FP16/TF32 values (bit-identical to convert()).
template <int N>
TCEC_DEV void convert_n(float (&x)[N], const PrepMode& pm, double factor, float fs, bool corrected,
                        float (&h)[N], float (&l)[N], unsigned& ovf, unsigned& bad) {
    if (pm.scale != 0) {
        if (pm.scale >= -149 && pm.scale <= 127) {
#pragma unroll
            for (int e = 0; e < N; ++e) x[e] = __fmul_rn(x[e], fs);
        } else {
#pragma unroll
            for (int e = 0; e < N; ++e) x[e] = scale_pow2(x[e], factor);
        }
    }
    uint32_t mb = 0;
#pragma unroll
    for (int e = 0; e < N; ++e) mb = max(mb, __float_as_uint(x[e]) & 0x7FFFFFFFu);
    if (pm.scaled) bad |= mb >= 0x7F800000u ? 1u : 0u;
    const uint32_t lim = pm.fmt == kFp16 ? __float_as_uint(kFp16Max) : __float_as_uint(kTf32Max);
    if (mb > lim) {
        PrepMode ns = pm;
        ns.scale = 0;       // already scaled (and checked) above
        ns.scaled = false;
#pragma unroll
        for (int e = 0; e < N; ++e) convert(x[e], ns, 1.0, corrected, h[e], l[e], ovf, bad);
        return;
    }
    if (pm.fmt == kFp16) {
#pragma unroll
        for (int e = 0; e < N; e += 2) {
            const float2 hf = __half22float2(__floats2half2_rn(x[e], x[e + 1]));
            h[e] = hf.x;
            h[e + 1] = hf.y;
            if (corrected) {
                const float2 lf = __half22float2(__floats2half2_rn(__fmul_rn(__fsub_rn(x[e], hf.x), 2048.0f),
                                                                   __fmul_rn(__fsub_rn(x[e + 1], hf.y), 2048.0f)));
                l[e] = lf.x;
                l[e + 1] = lf.y;
            } else {
                l[e] = l[e + 1] = 0.0f;
            }
        }
    } else {
        auto rne = [](float v) {
            uint32_t b = __float_as_uint(v);
            b += 0xFFFu + ((b >> 13) & 1u);
            return __uint_as_float(b & ~0x1FFFu);
        };
#pragma unroll
        for (int e = 0; e < N; ++e) {
            h[e] = rne(x[e]);
            l[e] = corrected ? rne(__fmul_rn(__fsub_rn(x[e], h[e]), 2048.0f)) : 0.0f;
        }
    }
}

// A (m x k complex) -> K-major m x kp; each thread converts 8 consecutive
// real components of one row (16 B of f16 or 32 B of tf32 per output plane)
template <bool VIEW>
TCEC_DEV void prep_a_part(const float* __restrict__ a, int64_t m,
                                                          int64_t k2, int64_t kp, void* hi_v,
                                                          void* lo_v, const DevDecision* d,
                                                          int kind_fixed, int corrected, int64_t row0,
        DevDecision* df, int bid, int nblk, const MatrixView& view) {
    // rows [row0, row0 + m) of A (the host-buffer pipeline converts row chunks
    // as they arrive; every row is independent)
    const PrepMode pm = prep_mode(d, kind_fixed, false);
    if (!pm.active) return;
    const double factor = ldexp(1.0, pm.scale);
    const float fs = (pm.scale >= -149 && pm.scale <= 127) ? ldexpf(1.0f, pm.scale) : 1.0f;
    const int64_t chunks_per_row = kp / 8;
    const int64_t total = m * chunks_per_row;
    unsigned ovf = 0, bad = 0;
    const bool vec = (k2 % 8) == 0 && (reinterpret_cast<uintptr_t>(a) & 15u) == 0;
    for (int64_t c = bid * int64_t(blockDim.x) + threadIdx.x; c < total;
         c += int64_t(nblk) * blockDim.x) {
        const int64_t rl = c / chunks_per_row;
        const int64_t col = (c - rl * chunks_per_row) * 8;
        const int64_t row = row0 + rl;
        float x[8];
        if (VIEW) {
            // A is a view of the unpermuted tensor (fused TTGT gather)
            load4_view(a, view, row, col / 2, k2 / 2, x);
        } else if (vec && col < k2) {
            const float4* p = reinterpret_cast<const float4*>(a + row * k2 + col);
            const float4 v0 = __ldcs(p), v1 = __ldcs(p + 1);
            x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
            x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = (col + e < k2) ? a[row * k2 + col + e] : 0.0f;
        }
        float h[8], l[8];
        convert_n<8>(x, pm, factor, fs, corrected, h, l, ovf, bad);
        if (pm.fmt == kFp16) {
            __half2 hh[4], ll[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                hh[e] = __floats2half2_rn(h[2 * e], h[2 * e + 1]);  // exact: values are FP16
                ll[e] = __floats2half2_rn(l[2 * e], l[2 * e + 1]);
            }
            __half* hp = static_cast<__half*>(hi_v) + row * kp + col;
            *reinterpret_cast<uint4*>(hp) = *reinterpret_cast<uint4*>(hh);
            if (corrected) {
                __half* lp = static_cast<__half*>(lo_v) + row * kp + col;
                *reinterpret_cast<uint4*>(lp) = *reinterpret_cast<uint4*>(ll);
            }
        } else {
            float4* hp = reinterpret_cast<float4*>(static_cast<float*>(hi_v) + row * kp + col);
            hp[0] = make_float4(h[0], h[1], h[2], h[3]);
            hp[1] = make_float4(h[4], h[5], h[6], h[7]);
            if (corrected) {
                float4* lp = reinterpret_cast<float4*>(static_cast<float*>(lo_v) + row * kp + col);
                lp[0] = make_float4(l[0], l[1], l[2], l[3]);
                lp[1] = make_float4(l[4], l[5], l[6], l[7]);
            }
        }
    }
    DevDecision* dm = df;
    flag_or(&dm->overflow, ovf);
    flag_or(&dm->scale_overflow, bad);
}

template <bool VIEW>
__global__ void __launch_bounds__(kThreads) prep_a_kernel(const float* __restrict__ a, int64_t m,
                                                          int64_t k2, int64_t kp, void* hi_v,
                                                          void* lo_v, const DevDecision* d,
                                                          int kind_fixed, int corrected, int64_t row0,
                                                          const MatrixView view) {
    prep_a_part<VIEW>(a, m, k2, kp, hi_v, lo_v, d, kind_fixed, corrected, row0, const_cast<DevDecision*>(d),
                      int(blockIdx.x), int(gridDim.x), view);
}

// B (k x n complex) -> B'^T (2n x kp, K-major) with the complex block expansion
//   row 2j   : (Br, -Bi) at columns (2kk, 2kk+1)
//   row 2j+1 : ( Bi,  Br)
// Persistent blocks walk 64 (kk) x 32 (j) tiles: coalesced 256-B reads along
// j into a [j][kk] shared tile (row stride 66 elements keeps the 16-B reads of
// the write phase aligned and conflict-free), then each warp writes whole
// 64-kk row segments -- 256 B (FP16) / 512 B (TF32) per store instruction
// and plane -- converting two kk per lane with the vectorised split.
constexpr int kPrepBKK = 64, kPrepBJ = 32, kPrepBStride = kPrepBKK + 2;

template <bool VIEW>
TCEC_DEV void prep_b_part(const float2* __restrict__ b, int64_t k,
                                                     int64_t n, int64_t kp, void* hi_v,
                                                     void* lo_v, const DevDecision* d,
                                                     int kind_fixed, int corrected, int64_t jout0,
        DevDecision* df, int bid, int nblk, const MatrixView& view) {
    // b is a k x n column block whose B' rows start at 2 jout0
    const PrepMode pm = prep_mode(d, kind_fixed, true);
    if (!pm.active) return;
    const double factor = ldexp(1.0, pm.scale);
    const float fs = (pm.scale >= -149 && pm.scale <= 127) ? ldexpf(1.0f, pm.scale) : 1.0f;
    __shared__ __align__(16) float2 tile[kPrepBJ][kPrepBStride];
    __shared__ int64_t roff_s[2][VIEW ? kPrepBKK : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;  // 8 warps
    const int64_t tiles_j = (n + kPrepBJ - 1) / kPrepBJ;
    const int64_t kk_cols = kp / 2;                               // complex K extent incl. padding
    const int64_t tiles_kk = (kk_cols + kPrepBKK - 1) / kPrepBKK;
    const int64_t ntiles = tiles_j * tiles_kk;
    unsigned ovf = 0, bad = 0;
    // software-pipelined tiles: the next tile's loads are issued (into
    // registers) before the current tile's conversion and stores, so every
    // block keeps a tile of reads in flight (one tile at a time left the
    // kernel latency-bound at ~4 TB/s).  Warp w loads rows kk0 + w, w+8, ...
    // (32 consecutive j each); VIEW: B is a view of the unpermuted tensor
    // (fused TTGT gather) whose 64 row offsets per tile are tabled, double
    // buffered.
    auto fill_roff = [&](int64_t t, int buf) {
        if (VIEW && threadIdx.x < kPrepBKK) {
            const int64_t kk0 = (t / tiles_j) * kPrepBKK;
            roff_s[buf][threadIdx.x] =
                kk0 + threadIdx.x < k ? run_offset(view.rows, uint32_t(kk0 + threadIdx.x)) : 0;
        }
    };
    auto load_tile = [&](int64_t t, int buf, float2 (&v)[kPrepBKK / 8]) {
        const int64_t j0 = (t % tiles_j) * kPrepBJ, kk0 = (t / tiles_j) * kPrepBKK;
        const int64_t gj = j0 + lane;
        const int64_t co = VIEW && gj < n ? run_offset(view.cols, uint32_t(gj)) : 0;
#pragma unroll
        for (int r = 0; r < kPrepBKK / 8; ++r) {
            const int64_t gk = kk0 + warp + 8 * r;
            const float2* src = VIEW ? b + roff_s[buf][warp + 8 * r] + co : b + gk * n + gj;
            v[r] = (gk < k && gj < n) ? __ldcs(src) : make_float2(0.0f, 0.0f);
        }
    };
    float2 vt[kPrepBKK / 8];
    int buf = 0;
    if (int64_t(bid) < ntiles) {
        fill_roff(bid, 0);
        if (VIEW) __syncthreads();
        load_tile(bid, 0, vt);
    }
    for (int64_t t = bid; t < ntiles; t += nblk) {
        const int64_t j0 = (t % tiles_j) * kPrepBJ, kk0 = (t / tiles_j) * kPrepBKK;
#pragma unroll
        for (int r = 0; r < kPrepBKK / 8; ++r) tile[lane][warp + 8 * r] = vt[r];
        const int64_t tn = t + nblk;
        if (tn < ntiles) fill_roff(tn, buf ^ 1);
        __syncthreads();
        if (tn < ntiles) load_tile(tn, buf ^ 1, vt);
        buf ^= 1;
        // write: warp w owns j = j0 + w, w+8, ...; lane owns kk0 + 2 lane, +1
        const int64_t col = 2 * (kk0 + 2 * lane);                 // K' column of (kk0 + 2 lane, re)
        if (col < kp) {
            for (int jj = warp; jj < kPrepBJ; jj += 8) {
                const int64_t j = j0 + jj;
                if (j >= n) break;
                const float4 v = *reinterpret_cast<const float4*>(&tile[jj][2 * lane]);
                float xv[4] = {v.x, v.y, v.z, v.w}, hv[4], lv[4];   // (re0, im0, re1, im1)
                convert_n<4>(xv, pm, factor, fs, corrected, hv, lv, ovf, bad);
                // negated imaginary parts; the K padding stays +0 in every
                // plane (negating the zero fill would write -0)
                float hn1 = -hv[1], hn3 = -hv[3], ln1 = -lv[1], ln3 = -lv[3];
                if (kk0 + 2 * lane + 1 >= k) {
                    hn3 = ln3 = 0.0f;
                    if (kk0 + 2 * lane >= k) hn1 = ln1 = 0.0f;
                }
                const int64_t r0 = (2 * (jout0 + j)) * kp + col, r1 = r0 + kp;
                if (pm.fmt == kFp16) {
                    __half* hp = static_cast<__half*>(hi_v);
                    __half2 q0[2] = {__floats2half2_rn(hv[0], hn1), __floats2half2_rn(hv[2], hn3)};
                    __half2 q1[2] = {__floats2half2_rn(hv[1], hv[0]), __floats2half2_rn(hv[3], hv[2])};
                    *reinterpret_cast<uint2*>(hp + r0) = *reinterpret_cast<uint2*>(q0);
                    *reinterpret_cast<uint2*>(hp + r1) = *reinterpret_cast<uint2*>(q1);
                    if (corrected) {
                        __half* lp = static_cast<__half*>(lo_v);
                        __half2 w0[2] = {__floats2half2_rn(lv[0], ln1), __floats2half2_rn(lv[2], ln3)};
                        __half2 w1[2] = {__floats2half2_rn(lv[1], lv[0]), __floats2half2_rn(lv[3], lv[2])};
                        *reinterpret_cast<uint2*>(lp + r0) = *reinterpret_cast<uint2*>(w0);
                        *reinterpret_cast<uint2*>(lp + r1) = *reinterpret_cast<uint2*>(w1);
                    }
                } else {
                    float* hp = static_cast<float*>(hi_v);
                    *reinterpret_cast<float4*>(hp + r0) = make_float4(hv[0], hn1, hv[2], hn3);
                    *reinterpret_cast<float4*>(hp + r1) = make_float4(hv[1], hv[0], hv[3], hv[2]);
                    if (corrected) {
                        float* lp = static_cast<float*>(lo_v);
                        *reinterpret_cast<float4*>(lp + r0) = make_float4(lv[0], ln1, lv[2], ln3);
                        *reinterpret_cast<float4*>(lp + r1) = make_float4(lv[1], lv[0], lv[3], lv[2]);
                    }
                }
            }
        }
        __syncthreads();
    }
    DevDecision* dm = df;
    flag_or(&dm->overflow, ovf);
    flag_or(&dm->scale_overflow, bad);
}

template <bool VIEW>
__global__ void __launch_bounds__(256) prep_b_kernel(const float2* __restrict__ b, int64_t k,
                                                     int64_t n, int64_t kp, void* hi_v,
                                                     void* lo_v, const DevDecision* d,
                                                     int kind_fixed, int corrected, int64_t jout0,
        const MatrixView view) {
    prep_b_part<VIEW>(b, k, n, kp, hi_v, lo_v, d, kind_fixed, corrected, jout0, const_cast<DevDecision*>(d), int(blockIdx.x), int(gridDim.x), view);
}

// --------------------------------------------- A-expanded operand layout
// When A is the smaller operand (m < n: the contraction steps that multiply a
// small tensor into a large one), the complex block expansion moves to A:
//   A'' (2m x kp):  row 2i   = (Ar, -Ai) at K' columns (2p, 2p+1)
//                   row 2i+1 = (Ai,  Ar)
//   B'' (n x kp):   row j    = (Br, Bi)  -- column j of B, i.e. B^T
// so C'' = A'' B''^T has row 2i = Re C[i, :], row 2i+1 = Im C[i, :] and the
// GEMM epilogue interleaves the row pair into C.  Same products, same split
// (split(-x) = -split(x) for RN and the symmetric saturation), but the
// expanded, twice-written operand is the small one: 2k (2m + n) instead of
// 2k (m + 2n) plane elements.

// A (m x k complex) -> A'' (2m x kp); each thread converts 4 consecutive
// complex elements of one row (8 components) and writes 8 K' columns of both
// rows of the pair
template <bool VIEW>
TCEC_DEV void prep_ax_part(const float* __restrict__ a, int64_t m,
                                                           int64_t k, int64_t kp, void* hi_v, void* lo_v,
                                                           const DevDecision* d, int kind_fixed,
                                                           int corrected,
        DevDecision* df, int bid, int nblk, const MatrixView& view) {
    const PrepMode pm = prep_mode(d, kind_fixed, false);
    if (!pm.active) return;
    const double factor = ldexp(1.0, pm.scale);
    const float fs = (pm.scale >= -149 && pm.scale <= 127) ? ldexpf(1.0f, pm.scale) : 1.0f;
    const int64_t k2 = 2 * k;
    const int64_t chunks_per_row = kp / 8;
    const int64_t total = m * chunks_per_row;
    unsigned ovf = 0, bad = 0;
    const bool vec = (k2 % 8) == 0 && (reinterpret_cast<uintptr_t>(a) & 15u) == 0;
    for (int64_t c = bid * int64_t(blockDim.x) + threadIdx.x; c < total;
         c += int64_t(nblk) * blockDim.x) {
        const int64_t row = c / chunks_per_row;
        const int64_t col = (c - row * chunks_per_row) * 8;  // K' column = 2 p0
        float x[8];
        if (VIEW) {
            // A is a view of the unpermuted tensor (fused TTGT gather)
            load4_view(a, view, row, col / 2, k2 / 2, x);
        } else if (vec && col < k2) {
            const float4* p = reinterpret_cast<const float4*>(a + row * k2 + col);
            const float4 v0 = __ldcs(p), v1 = __ldcs(p + 1);
            x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
            x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) x[e] = (col + e < k2) ? a[row * k2 + col + e] : 0.0f;
        }
        float h[8], l[8];
        convert_n<8>(x, pm, factor, fs, corrected, h, l, ovf, bad);
        // row 2i: (re, -im); the K padding stays +0 (negating the zero fill would write -0)
        float hn[4], ln[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const bool pad = col + 2 * e >= k2;
            hn[e] = pad ? 0.0f : -h[2 * e + 1];
            ln[e] = pad ? 0.0f : -l[2 * e + 1];
        }
        const int64_t r0 = (2 * row) * kp + col, r1 = r0 + kp;
        if (pm.fmt == kFp16) {
            __half2 q0[4], q1[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                q0[e] = __floats2half2_rn(h[2 * e], hn[e]);         // exact: values are FP16
                q1[e] = __floats2half2_rn(h[2 * e + 1], h[2 * e]);
            }
            __half* hp = static_cast<__half*>(hi_v);
            *reinterpret_cast<uint4*>(hp + r0) = *reinterpret_cast<uint4*>(q0);
            *reinterpret_cast<uint4*>(hp + r1) = *reinterpret_cast<uint4*>(q1);
            if (corrected) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    q0[e] = __floats2half2_rn(l[2 * e], ln[e]);
                    q1[e] = __floats2half2_rn(l[2 * e + 1], l[2 * e]);
                }
                __half* lp = static_cast<__half*>(lo_v);
                *reinterpret_cast<uint4*>(lp + r0) = *reinterpret_cast<uint4*>(q0);
                *reinterpret_cast<uint4*>(lp + r1) = *reinterpret_cast<uint4*>(q1);
            }
        } else {
            float4* hp0 = reinterpret_cast<float4*>(static_cast<float*>(hi_v) + r0);
            float4* hp1 = reinterpret_cast<float4*>(static_cast<float*>(hi_v) + r1);
            hp0[0] = make_float4(h[0], hn[0], h[2], hn[1]);
            hp0[1] = make_float4(h[4], hn[2], h[6], hn[3]);
            hp1[0] = make_float4(h[1], h[0], h[3], h[2]);
            hp1[1] = make_float4(h[5], h[4], h[7], h[6]);
            if (corrected) {
                float4* lp0 = reinterpret_cast<float4*>(static_cast<float*>(lo_v) + r0);
                float4* lp1 = reinterpret_cast<float4*>(static_cast<float*>(lo_v) + r1);
                lp0[0] = make_float4(l[0], ln[0], l[2], ln[1]);
                lp0[1] = make_float4(l[4], ln[2], l[6], ln[3]);
                lp1[0] = make_float4(l[1], l[0], l[3], l[2]);
                lp1[1] = make_float4(l[5], l[4], l[7], l[6]);
            }
        }
    }
    DevDecision* dm = df;
    flag_or(&dm->overflow, ovf);
    flag_or(&dm->scale_overflow, bad);
}

template <bool VIEW>
__global__ void __launch_bounds__(kThreads) prep_ax_kernel(const float* __restrict__ a, int64_t m,
                                                           int64_t k, int64_t kp, void* hi_v, void* lo_v,
                                                           const DevDecision* d, int kind_fixed,
                                                           int corrected,
        const MatrixView view) {
    prep_ax_part<VIEW>(a, m, k, kp, hi_v, lo_v, d, kind_fixed, corrected, const_cast<DevDecision*>(d),
                       int(blockIdx.x), int(gridDim.x), view);
}

// B (k x n complex) -> B'' = B^T (n x kp, K-major, (re, im) pairs along K).
// Same 64 (kk) x 32 (j) smem tiles as prep_b_kernel, one output row per j.
template <bool VIEW>
TCEC_DEV void prep_bx_part(const float2* __restrict__ b, int64_t k,
                                                      int64_t n, int64_t kp, void* hi_v, void* lo_v,
                                                      const DevDecision* d, int kind_fixed,
                                                      int corrected,
        DevDecision* df, int bid, int nblk, const MatrixView& view) {
    const PrepMode pm = prep_mode(d, kind_fixed, true);
    if (!pm.active) return;
    const double factor = ldexp(1.0, pm.scale);
    const float fs = (pm.scale >= -149 && pm.scale <= 127) ? ldexpf(1.0f, pm.scale) : 1.0f;
    __shared__ __align__(16) float2 tile[kPrepBJ][kPrepBStride];
    __shared__ int64_t roff_s[2][VIEW ? kPrepBKK : 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;  // 8 warps
    const int64_t tiles_j = (n + kPrepBJ - 1) / kPrepBJ;
    const int64_t kk_cols = kp / 2;
    const int64_t tiles_kk = (kk_cols + kPrepBKK - 1) / kPrepBKK;
    const int64_t ntiles = tiles_j * tiles_kk;
    unsigned ovf = 0, bad = 0;
    // software-pipelined tiles: the next tile's loads are issued (into
    // registers) before the current tile's conversion and stores, so every
    // block keeps a tile of reads in flight (one tile at a time left the
    // kernel latency-bound at ~4 TB/s).  Warp w loads rows kk0 + w, w+8, ...
    // (32 consecutive j each); VIEW: B is a view of the unpermuted tensor
    // (fused TTGT gather) whose 64 row offsets per tile are tabled, double
    // buffered.
    auto fill_roff = [&](int64_t t, int buf) {
        if (VIEW && threadIdx.x < kPrepBKK) {
            const int64_t kk0 = (t / tiles_j) * kPrepBKK;
            roff_s[buf][threadIdx.x] =
                kk0 + threadIdx.x < k ? run_offset(view.rows, uint32_t(kk0 + threadIdx.x)) : 0;
        }
    };
    auto load_tile = [&](int64_t t, int buf, float2 (&v)[kPrepBKK / 8]) {
        const int64_t j0 = (t % tiles_j) * kPrepBJ, kk0 = (t / tiles_j) * kPrepBKK;
        const int64_t gj = j0 + lane;
        const int64_t co = VIEW && gj < n ? run_offset(view.cols, uint32_t(gj)) : 0;
#pragma unroll
        for (int r = 0; r < kPrepBKK / 8; ++r) {
            const int64_t gk = kk0 + warp + 8 * r;
            const float2* src = VIEW ? b + roff_s[buf][warp + 8 * r] + co : b + gk * n + gj;
            v[r] = (gk < k && gj < n) ? __ldcs(src) : make_float2(0.0f, 0.0f);
        }
    };
    float2 vt[kPrepBKK / 8];
    int buf = 0;
    if (int64_t(bid) < ntiles) {
        fill_roff(bid, 0);
        if (VIEW) __syncthreads();
        load_tile(bid, 0, vt);
    }
    for (int64_t t = bid; t < ntiles; t += nblk) {
        const int64_t j0 = (t % tiles_j) * kPrepBJ, kk0 = (t / tiles_j) * kPrepBKK;
#pragma unroll
        for (int r = 0; r < kPrepBKK / 8; ++r) tile[lane][warp + 8 * r] = vt[r];
        const int64_t tn = t + nblk;
        if (tn < ntiles) fill_roff(tn, buf ^ 1);
        __syncthreads();
        if (tn < ntiles) load_tile(tn, buf ^ 1, vt);
        buf ^= 1;
        const int64_t col = 2 * (kk0 + 2 * lane);
        if (col < kp) {
            for (int jj = warp; jj < kPrepBJ; jj += 8) {
                const int64_t j = j0 + jj;
                if (j >= n) break;
                const float4 v = *reinterpret_cast<const float4*>(&tile[jj][2 * lane]);
                float xv[4] = {v.x, v.y, v.z, v.w}, hv[4], lv[4];   // (re0, im0, re1, im1)
                convert_n<4>(xv, pm, factor, fs, corrected, hv, lv, ovf, bad);
                const int64_t r0 = j * kp + col;
                if (pm.fmt == kFp16) {
                    __half2 q[2] = {__floats2half2_rn(hv[0], hv[1]), __floats2half2_rn(hv[2], hv[3])};
                    *reinterpret_cast<uint2*>(static_cast<__half*>(hi_v) + r0) = *reinterpret_cast<uint2*>(q);
                    if (corrected) {
                        __half2 w[2] = {__floats2half2_rn(lv[0], lv[1]), __floats2half2_rn(lv[2], lv[3])};
                        *reinterpret_cast<uint2*>(static_cast<__half*>(lo_v) + r0) = *reinterpret_cast<uint2*>(w);
                    }
                } else {
                    *reinterpret_cast<float4*>(static_cast<float*>(hi_v) + r0) = make_float4(hv[0], hv[1], hv[2], hv[3]);
                    if (corrected)
                        *reinterpret_cast<float4*>(static_cast<float*>(lo_v) + r0) =
                            make_float4(lv[0], lv[1], lv[2], lv[3]);
                }
            }
        }
        __syncthreads();
    }
    DevDecision* dm = df;
    flag_or(&dm->overflow, ovf);
    flag_or(&dm->scale_overflow, bad);
}

template <bool VIEW>
__global__ void __launch_bounds__(256) prep_bx_kernel(const float2* __restrict__ b, int64_t k,
                                                      int64_t n, int64_t kp, void* hi_v, void* lo_v,
                                                      const DevDecision* d, int kind_fixed,
                                                      int corrected,
        const MatrixView view) {
    prep_bx_part<VIEW>(b, k, n, kp, hi_v, lo_v, d, kind_fixed, corrected, const_cast<DevDecision*>(d), int(blockIdx.x), int(gridDim.x), view);
}

// ------------------------------------------------------------ SIMT GEMM

// FP32_REF complex GEMM with the reference's exact arithmetic: four RN chains
// P1=ReRe, P2=ImIm, P3=ReIm, P4=ImRe, each starting at +0 and accumulating
// mul-then-add in ascending k (kernels_scalar.cpp:76-87, -ffp-contract=off),
// then C = (P1 - P2, P3 + P4) in f32 RN (cgemm.cpp:38-44).
constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

// 256 threads, thread (tx, ty) owns rows 4ty..4ty+3 and columns 4tx..4tx+3 of
// the 64 x 64 tile, so every k step reads its operands with four 16-byte
// shared loads (the issue slots go to the 128 FMUL/FADD of the four chains)
__global__ void __launch_bounds__(256) cgemm_fp32_ref_kernel(const float2* __restrict__ a,
                                                             const float2* __restrict__ b,
                                                             float2* __restrict__ c, int64_t m,
                                                             int64_t n, int64_t k) {
    __shared__ __align__(16) float sar[SB_K][SB_M], sai[SB_K][SB_M], sbr[SB_K][SB_N], sbi[SB_K][SB_N];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t tiles_n = (n + SB_N - 1) / SB_N;  // 1-D grid: x = i_tile * tiles_n + j_tile
    const int64_t i0 = (int64_t(blockIdx.x) / tiles_n) * SB_M, j0 = (int64_t(blockIdx.x) % tiles_n) * SB_N;
    float p1[4][4], p2[4][4], p3[4][4], p4[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) p1[i][j] = p2[i][j] = p3[i][j] = p4[i][j] = 0.0f;

    // register double buffer: the next k tile's global loads are in flight
    // while the current tile is chained
    float2 va[4], vb[4];
    auto load_tile = [&](int64_t k0) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int idx = threadIdx.x + 256 * r;
            const int ar = idx / SB_K, ak = idx % SB_K;
            const int64_t gi = i0 + ar, gk = k0 + ak;
            va[r] = (gi < m && gk < k) ? a[gi * k + gk] : make_float2(0.f, 0.f);
            const int bk = idx / SB_N, bj = idx % SB_N;
            const int64_t gk2 = k0 + bk, gj = j0 + bj;
            vb[r] = (gk2 < k && gj < n) ? b[gk2 * n + gj] : make_float2(0.f, 0.f);
        }
    };
    load_tile(0);
    for (int64_t k0 = 0; k0 < k; k0 += SB_K) {
        // A tile: 64 rows x 16 k; B tile: 16 k x 64 cols (4 complex per thread)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int idx = threadIdx.x + 256 * r;
            const int ar = idx / SB_K, ak = idx % SB_K;
            sar[ak][ar] = va[r].x;
            sai[ak][ar] = va[r].y;
            const int bk = idx / SB_N, bj = idx % SB_N;
            sbr[bk][bj] = vb[r].x;
            sbi[bk][bj] = vb[r].y;
        }
        __syncthreads();
        if (k0 + SB_K < k) load_tile(k0 + SB_K);
        const int kend = (k - k0) < SB_K ? int(k - k0) : SB_K;  // never add padding terms
        auto step = [&](int kk) {
            const float4 ar4 = *reinterpret_cast<const float4*>(&sar[kk][4 * ty]);
            const float4 ai4 = *reinterpret_cast<const float4*>(&sai[kk][4 * ty]);
            const float4 br4 = *reinterpret_cast<const float4*>(&sbr[kk][4 * tx]);
            const float4 bi4 = *reinterpret_cast<const float4*>(&sbi[kk][4 * tx]);
            const float ar[4] = {ar4.x, ar4.y, ar4.z, ar4.w}, ai[4] = {ai4.x, ai4.y, ai4.z, ai4.w};
            const float br[4] = {br4.x, br4.y, br4.z, br4.w}, bi[4] = {bi4.x, bi4.y, bi4.z, bi4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    p1[i][j] = __fadd_rn(p1[i][j], __fmul_rn(ar[i], br[j]));
                    p2[i][j] = __fadd_rn(p2[i][j], __fmul_rn(ai[i], bi[j]));
                    p3[i][j] = __fadd_rn(p3[i][j], __fmul_rn(ar[i], bi[j]));
                    p4[i][j] = __fadd_rn(p4[i][j], __fmul_rn(ai[i], br[j]));
                }
        };
        if (kend == SB_K) {
#pragma unroll
            for (int kk = 0; kk < SB_K; ++kk) step(kk);
        } else {
            for (int kk = 0; kk < kend; ++kk) step(kk);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gi = i0 + 4 * ty + i;
        if (gi >= m) continue;
        const int64_t gj = j0 + 4 * tx;
        float2 o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            o[j] = make_float2(__fsub_rn(p1[i][j], p2[i][j]), __fadd_rn(p3[i][j], p4[i][j]));
        float2* dst = c + gi * n + gj;
        if (gj + 4 <= n && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
            reinterpret_cast<float4*>(dst)[0] = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
            reinterpret_cast<float4*>(dst)[1] = make_float4(o[2].x, o[2].y, o[3].x, o[3].y);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (gj + j < n) dst[j] = o[j];
        }
    }
}

// Medium output count, long k (e.g. (256, 64, 2^17) contraction steps): the
// 64 x 64 register-tiled kernel would occupy only a handful of SMs and the
// warp-per-output kernel spends its issue slots on shuffles, so here every
// thread owns ONE output and runs its four chains (kernels_scalar.cpp:76-87)
// over 32-deep k tiles staged in shared memory: 16 x 16 outputs per block,
// ascending k per chain -> bit-identical.
template <bool F64>
__global__ void __launch_bounds__(256) cgemm_tpo_kernel(const float2* __restrict__ a,
                                                        const float2* __restrict__ b,
                                                        float2* __restrict__ c, int64_t m,
                                                        int64_t n, int64_t k) {
    using acc_t = typename std::conditional<F64, double, float>::type;
    __shared__ float2 as[32][17], bs[32][16];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t tiles_n = (n + 15) / 16;
    const int64_t i0 = (int64_t(blockIdx.x) / tiles_n) * 16, j0 = (int64_t(blockIdx.x) % tiles_n) * 16;
    const int64_t i = i0 + ty, j = j0 + tx;
    acc_t p1 = 0, p2 = 0, p3 = 0, p4 = 0;
    for (int64_t k0 = 0; k0 < k; k0 += 32) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int idx = threadIdx.x + 256 * r;
            const int ar = idx >> 5, ak = idx & 31;   // A: 16 rows x 32 k
            const int64_t gi = i0 + ar, gk = k0 + ak;
            as[ak][ar] = (gi < m && gk < k) ? a[gi * k + gk] : make_float2(0.f, 0.f);
            const int bk = idx >> 4, bj = idx & 15;   // B: 32 k x 16 cols
            const int64_t gk2 = k0 + bk, gj = j0 + bj;
            bs[bk][bj] = (gk2 < k && gj < n) ? b[gk2 * n + gj] : make_float2(0.f, 0.f);
        }
        __syncthreads();
        const int kend = (k - k0) < 32 ? int(k - k0) : 32;  // never add padding terms
        for (int kk = 0; kk < kend; ++kk) {
            const float2 x = as[kk][ty], y = bs[kk][tx];
            if (F64) {
                p1 = acc_t(__dadd_rn(double(p1), __dmul_rn(double(x.x), double(y.x))));
                p2 = acc_t(__dadd_rn(double(p2), __dmul_rn(double(x.y), double(y.y))));
                p3 = acc_t(__dadd_rn(double(p3), __dmul_rn(double(x.x), double(y.y))));
                p4 = acc_t(__dadd_rn(double(p4), __dmul_rn(double(x.y), double(y.x))));
            } else {
                p1 = acc_t(__fadd_rn(float(p1), __fmul_rn(x.x, y.x)));
                p2 = acc_t(__fadd_rn(float(p2), __fmul_rn(x.y, y.y)));
                p3 = acc_t(__fadd_rn(float(p3), __fmul_rn(x.x, y.y)));
                p4 = acc_t(__fadd_rn(float(p4), __fmul_rn(x.y, y.x)));
            }
        }
        __syncthreads();
    }
    if (i < m && j < n) {
        if (F64)
            c[i * n + j] = make_float2(__fsub_rn(__double2float_rn(double(p1)), __double2float_rn(double(p2))),
                                       __fadd_rn(__double2float_rn(double(p3)), __double2float_rn(double(p4))));
        else
            c[i * n + j] = make_float2(__fsub_rn(float(p1), float(p2)), __fadd_rn(float(p3), float(p4)));
    }
}

// FP64_ORACLE tier: f64 chains (kernels_scalar.cpp:137-148), each product
// rounded to f32 (gemm.cpp:111-117), then assembled in f32 (cgemm.cpp:38-44)
__global__ void cgemm_fp64_kernel(const float2* __restrict__ a, const float2* __restrict__ b,
                                  float2* __restrict__ c, int64_t m, int64_t n, int64_t k) {
    const int64_t tiles_n = (n + int64_t(blockDim.x) - 1) / blockDim.x;
    const int64_t j = (int64_t(blockIdx.x) % tiles_n) * blockDim.x + threadIdx.x;
    const int64_t i = int64_t(blockIdx.x) / tiles_n;
    if (j >= n || i >= m) return;
    double p1 = 0.0, p2 = 0.0, p3 = 0.0, p4 = 0.0;
    for (int64_t kk = 0; kk < k; ++kk) {
        const float2 va = a[i * k + kk], vb = b[kk * n + j];
        const double ar = va.x, ai = va.y, br = vb.x, bi = vb.y;
        p1 = __dadd_rn(p1, __dmul_rn(ar, br));
        p2 = __dadd_rn(p2, __dmul_rn(ai, bi));
        p3 = __dadd_rn(p3, __dmul_rn(ar, bi));
        p4 = __dadd_rn(p4, __dmul_rn(ai, br));
    }
    c[i * n + j] = make_float2(__fsub_rn(__double2float_rn(p1), __double2float_rn(p2)),
                               __fadd_rn(__double2float_rn(p3), __double2float_rn(p4)));
}

// Long-k / few-output shapes (e.g. the (1, 1, 2^22) dot products of deep
// circuits): one warp per output element, the warp loads 32 consecutive k of
// A and B coalesced (prefetching the next 32), and every lane runs the same
// four chains in ascending k on shuffled operands -- the reference order, so
// the result is bit-identical to kernels_scalar.cpp:76-87 / :137-148.
template <bool F64>
__global__ void __launch_bounds__(256) cgemm_longk_kernel(const float2* __restrict__ a,
                                                          const float2* __restrict__ b,
                                                          float2* __restrict__ c, int64_t m,
                                                          int64_t n, int64_t k) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    if (w >= m * n) return;
    const int64_t i = w / n, j = w - (w / n) * n;
    using acc_t = typename std::conditional<F64, double, float>::type;
    acc_t p1 = 0, p2 = 0, p3 = 0, p4 = 0;
    const float2* arow = a + i * k;
    const float2 zero = make_float2(0.0f, 0.0f);
    float2 av = lane < k ? arow[lane] : zero;
    float2 bv = lane < k ? b[int64_t(lane) * n + j] : zero;
    for (int64_t k0 = 0; k0 < k; k0 += 32) {
        const int64_t kn = k0 + 32 + lane;
        const float2 an = kn < k ? arow[kn] : zero;
        const float2 bn = kn < k ? b[kn * n + j] : zero;
        const int cnt = (k - k0) < 32 ? int(k - k0) : 32;
        for (int t = 0; t < cnt; ++t) {
            const float ar = __shfl_sync(0xFFFFFFFFu, av.x, t);
            const float ai = __shfl_sync(0xFFFFFFFFu, av.y, t);
            const float br = __shfl_sync(0xFFFFFFFFu, bv.x, t);
            const float bi = __shfl_sync(0xFFFFFFFFu, bv.y, t);
            if (F64) {
                p1 = __dadd_rn(p1, __dmul_rn(double(ar), double(br)));
                p2 = __dadd_rn(p2, __dmul_rn(double(ai), double(bi)));
                p3 = __dadd_rn(p3, __dmul_rn(double(ar), double(bi)));
                p4 = __dadd_rn(p4, __dmul_rn(double(ai), double(br)));
            } else {
                p1 = __fadd_rn(float(p1), __fmul_rn(ar, br));
                p2 = __fadd_rn(float(p2), __fmul_rn(ai, bi));
                p3 = __fadd_rn(float(p3), __fmul_rn(ar, bi));
                p4 = __fadd_rn(float(p4), __fmul_rn(ai, br));
            }
        }
        av = an;
        bv = bn;
    }
    if (lane == 0) {
        if (F64)
            c[i * n + j] = make_float2(__fsub_rn(__double2float_rn(double(p1)), __double2float_rn(double(p2))),
                                       __fadd_rn(__double2float_rn(double(p3)), __double2float_rn(double(p4))));
        else
            c[i * n + j] = make_float2(__fsub_rn(float(p1), float(p2)), __fadd_rn(float(p3), float(p4)));
    }
}

// Very long k (>= 64K): one block per output element, the four chains
// P1..P4 (cgemm.cpp:33-36) each a single serial RN chain in ascending k, so the
// FADD latency (4 cycles) x k is the floor.  Warps 4..7 are producers: they load
// a chunk of A and B coalesced and write the four product streams
// RN(x*y) to shared memory (products are independent of the chain order);
// lane 0 of warps 0..3 (one per SMSP) runs its chain over the previous chunk's
// products with 16-byte shared loads.  Same per-chain order as the reference ->
// bit-identical.
constexpr int kChainChunk = 1024;
constexpr int kChainThreads = 256;

template <bool F64>
__global__ void __launch_bounds__(kChainThreads) cgemm_chain_kernel(const float2* __restrict__ a,
                                                                   const float2* __restrict__ b,
                                                                   float2* __restrict__ c, int64_t m,
                                                                   int64_t n, int64_t k) {
    using acc_t = typename std::conditional<F64, double, float>::type;
    constexpr int CH = F64 ? kChainChunk / 2 : kChainChunk;
    extern __shared__ __align__(16) uint8_t chain_smem[];
    acc_t* prod = reinterpret_cast<acc_t*>(chain_smem);  // [2][4][CH]
    __shared__ double res[4];
    const int64_t o = blockIdx.x;
    const int64_t i = o / n, j = o - (o / n) * n;
    const float2* arow = a + i * k;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t nch = (k + CH - 1) / CH;
    // each producer thread handles CH/128 products; all its global loads are
    // issued before any product is formed, so a chunk costs one memory
    // latency, not CH/128 of them (the chain consumes 1024 adds in ~4k cycles)
    auto produce = [&](int buf, int64_t k0) {
        acc_t* P = prod + size_t(buf) * 4 * CH;
        constexpr int kPer = CH / 128;
        const int t0 = int(threadIdx.x) - 128;
        float2 xs[kPer], ys[kPer];
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int64_t kk = k0 + t0 + 128 * e;
            xs[e] = kk < k ? arow[kk] : make_float2(0.f, 0.f);
            ys[e] = kk < k ? b[kk * n + j] : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int t = t0 + 128 * e;
            const float2 x = xs[e], y = ys[e];
            if (F64) {
                P[0 * CH + t] = acc_t(__dmul_rn(double(x.x), double(y.x)));
                P[1 * CH + t] = acc_t(__dmul_rn(double(x.y), double(y.y)));
                P[2 * CH + t] = acc_t(__dmul_rn(double(x.x), double(y.y)));
                P[3 * CH + t] = acc_t(__dmul_rn(double(x.y), double(y.x)));
            } else {
                P[0 * CH + t] = acc_t(__fmul_rn(x.x, y.x));
                P[1 * CH + t] = acc_t(__fmul_rn(x.y, y.y));
                P[2 * CH + t] = acc_t(__fmul_rn(x.x, y.y));
                P[3 * CH + t] = acc_t(__fmul_rn(x.y, y.x));
            }
        }
    };
    acc_t p = 0;
    if (warp >= 4) produce(0, 0);
    __syncthreads();
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int buf = int(ch & 1);
        if (warp >= 4) {
            if (ch + 1 < nch) produce(buf ^ 1, (ch + 1) * CH);
        } else if (lane == 0) {
            const int64_t k0 = ch * CH;
            const int cnt = (k - k0) < CH ? int(k - k0) : CH;
            const acc_t* P = prod + (size_t(buf) * 4 + warp) * CH;
            if (cnt == CH) {
                if (F64) {
                    const double2* q = reinterpret_cast<const double2*>(P);
#pragma unroll 8
                    for (int t = 0; t < CH / 2; ++t) {
                        const double2 v = q[t];
                        p = acc_t(__dadd_rn(double(p), v.x));
                        p = acc_t(__dadd_rn(double(p), v.y));
                    }
                } else {
                    // software-pipelined: the next 32 products load while the
                    // current 32 are chained.  volatile asm pins the order (the
                    // compiler otherwise sinks the loads next to their use and
                    // exposes the shared-memory latency on the FADD chain)
                    float q0[32], q1[32];
                    const uint32_t base = smem_u32(P);
                    auto ld32 = [&](float (&q)[32], int g) {
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                                         : "=f"(q[4 * u]), "=f"(q[4 * u + 1]), "=f"(q[4 * u + 2]),
                                           "=f"(q[4 * u + 3])
                                         : "r"(base + uint32_t(128 * g + 16 * u)));
                    };
                    float pf = float(p);
                    auto chain32 = [&](const float (&q)[32]) {
#pragma unroll
                        for (int u = 0; u < 32; ++u)
                            asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(pf) : "f"(q[u]));
                    };
                    ld32(q0, 0);
                    for (int g = 0; g < CH / 32; g += 2) {
                        ld32(q1, g + 1);
                        chain32(q0);
                        if (g + 2 < CH / 32) ld32(q0, g + 2);
                        chain32(q1);
                    }
                    p = acc_t(pf);
                }
            } else {
                for (int t = 0; t < cnt; ++t) {
                    if (F64)
                        p = acc_t(__dadd_rn(double(p), double(P[t])));
                    else
                        p = acc_t(__fadd_rn(float(p), float(P[t])));
                }
            }
        }
        __syncthreads();
    }
    if (warp < 4 && lane == 0) res[warp] = double(p);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (F64)
            c[o] = make_float2(__fsub_rn(__double2float_rn(res[0]), __double2float_rn(res[1])),
                               __fadd_rn(__double2float_rn(res[2]), __double2float_rn(res[3])));
        else
            c[o] = make_float2(__fsub_rn(float(res[0]), float(res[1])),
                               __fadd_rn(float(res[2]), float(res[3])));
    }
}

// Irregular skinny shapes, small k with one small outer dimension -- the
// (2, 2^N, 2) / (2^N, 2, 2) contraction family.  Memory-bound:
// one thread per column j (m <= MX, "column" kernel) or per row i (n <= MX,
// "row" kernel) keeps the MX x 4 chains of its outputs in registers, reads the
// long operand exactly once (coalesced / contiguous) and writes C once; the
// short operand sits in shared memory.  Each output runs the reference's four
// chains in ascending k (kernels_scalar.cpp:76-87) -> bit-identical.
constexpr int kSkinnyMaxK = 128;

template <bool F64>
TCEC_DEV void chain4(float ar, float ai, float br, float bi, double (&p)[4]) {
    p[0] = __dadd_rn(p[0], __dmul_rn(double(ar), double(br)));
    p[1] = __dadd_rn(p[1], __dmul_rn(double(ai), double(bi)));
    p[2] = __dadd_rn(p[2], __dmul_rn(double(ar), double(bi)));
    p[3] = __dadd_rn(p[3], __dmul_rn(double(ai), double(br)));
}
template <bool F64>
TCEC_DEV void chain4(float ar, float ai, float br, float bi, float (&p)[4]) {
    p[0] = __fadd_rn(p[0], __fmul_rn(ar, br));
    p[1] = __fadd_rn(p[1], __fmul_rn(ai, bi));
    p[2] = __fadd_rn(p[2], __fmul_rn(ar, bi));
    p[3] = __fadd_rn(p[3], __fmul_rn(ai, br));
}
template <bool F64, typename T>
TCEC_DEV float2 assemble(const T (&p)[4]) {
    if (F64)
        return make_float2(__fsub_rn(__double2float_rn(double(p[0])), __double2float_rn(double(p[1]))),
                           __fadd_rn(__double2float_rn(double(p[2])), __double2float_rn(double(p[3]))));
    return make_float2(__fsub_rn(float(p[0]), float(p[1])), __fadd_rn(float(p[2]), float(p[3])));
}

// The short operand sits in shared memory as [k][MX], zero-padded beyond the
// m (or n) real rows, so the inner loops carry no per-row predicates: every
// thread runs all MX x 4 chains (the padded ones are never stored) and reads
// two short-side elements per 16-B LDS.  Full groups of 8 k are unrolled
// without bounds checks (ncu: predicates and loop branches were ~45% of the
// issued instructions of the guarded version).
template <bool F64, int MX>
TCEC_DEV void skinny_mac(const float2* __restrict__ srow, float xr, float xi,
                         typename std::conditional<F64, double, float>::type (&p)[MX][4], bool a_side) {
#pragma unroll
    for (int q = 0; q < MX / 2; ++q) {
        const float4 s2 = reinterpret_cast<const float4*>(srow)[q];
        if (a_side) {  // short side is A (column kernel): chains (a_i, x)
            chain4<F64>(s2.x, s2.y, xr, xi, p[2 * q]);
            chain4<F64>(s2.z, s2.w, xr, xi, p[2 * q + 1]);
        } else {       // short side is B (row kernel): chains (x, b_j)
            chain4<F64>(xr, xi, s2.x, s2.y, p[2 * q]);
            chain4<F64>(xr, xi, s2.z, s2.w, p[2 * q + 1]);
        }
    }
}


// Packed f32x2 chains: fma.rn.f32x2(a, b, -0) is RN(a*b) exactly (signed
// zeros, subnormals and overflow included) and add.rn.f32x2 is two RN adds,
// so two products of the reference's mul-then-add chains issue as one FFMA2 +
// one FADD2 (tools/probes/f32x2_fmaz_probe.cu).  The -0 pair must arrive as a
// kernel argument: a literal lets ptxas fold the addend and contract the
// following add into an FMA.
TCEC_DEV uint64_t mulz2(uint64_t a, uint64_t b, uint64_t mz) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(mz));
    return r;
}
TCEC_DEV uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
TCEC_DEV uint64_t pack2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
TCEC_DEV float2 unpack2(uint64_t v) {
    float2 f;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(v));
    return f;
}

// column kernel MACs, packed: q[i][0] = (P1, P2) += (ar, ai) * (xr, xi),
// q[i][1] = (P3, P4) += (ar, ai) * (xi, xr) -- the four reference chains of
// output i (kernels_scalar.cpp:76-87) in the same order
template <int MX>
TCEC_DEV void skinny_mac_x2(const float2* __restrict__ srow, float xr, float xi, uint64_t (&q)[MX][2],
                            uint64_t mz) {
    const uint64_t x01 = pack2(xr, xi), x10 = pack2(xi, xr);
#pragma unroll
    for (int h = 0; h < MX / 2; ++h) {
        const ulonglong2 s2 = reinterpret_cast<const ulonglong2*>(srow)[h];  // (ar, ai) of rows 2h, 2h+1
        q[2 * h][0] = add2(q[2 * h][0], mulz2(s2.x, x01, mz));
        q[2 * h][1] = add2(q[2 * h][1], mulz2(s2.x, x10, mz));
        q[2 * h + 1][0] = add2(q[2 * h + 1][0], mulz2(s2.y, x01, mz));
        q[2 * h + 1][1] = add2(q[2 * h + 1][1], mulz2(s2.y, x10, mz));
    }
}

// m <= MX: thread j owns column j of C.  VIEW: B is read through a matrix
// view of the unpermuted tensor (fused TTGT gather): B(kk, j) =
// b[view.rows(kk) + view.cols(j)], the same elements in the same order.
template <bool F64, int MX, bool GROUPED, bool VIEW = false>
__global__ void __launch_bounds__(256, 2) cgemm_skinny_col_kernel(const float2* __restrict__ a,
                                                               const float2* __restrict__ b,
                                                               float2* __restrict__ c, int m,
                                                               int64_t n, int k, const MatrixView view,
                                                               uint64_t mz) {
    using acc_t = typename std::conditional<F64, double, float>::type;
    // packed f32x2 chains where the kernel is issue-bound (MX >= 8: ncu 81 %
    // issue slots busy, 1024 of ~1230 instructions per 8-k group FMUL/FADD)
    constexpr bool X2 = !F64 && MX >= 8;
    __shared__ __align__(16) float2 as[kSkinnyMaxK * MX];  // [kk][i]
    __shared__ int64_t koff[VIEW ? kSkinnyMaxK : 1];
    for (int t = threadIdx.x; t < k * MX; t += blockDim.x) {
        const int kk = t / MX, i = t % MX;
        as[t] = i < m ? a[i * k + kk] : make_float2(0.0f, 0.0f);
    }
    if (VIEW)
        for (int t = threadIdx.x; t < k; t += blockDim.x) koff[t] = run_offset(view.rows, uint32_t(t));
    __syncthreads();
    // persistent blocks walk 256-column chunks: the short operand is staged
    // once per block, and with k a multiple of 8 the first load group of the
    // next chunk is issued during the last MACs of the current one (ncu: the
    // per-block prologue -- A from L2, barrier, first B loads -- left the
    // schedulers without eligible warps, long-scoreboard 45% of the stalls)
    auto col_ptr = [&](int64_t jj) {
        return VIEW ? b + run_offset(view.cols, uint32_t(jj)) : b + jj;
    };
    auto bel = [&](const float2* bj, int kk) {
        return VIEW ? __ldcs(bj + koff[kk]) : __ldcs(bj + int64_t(kk) * n);
    };
    const int64_t step = int64_t(gridDim.x) * blockDim.x;
    int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool grouped = GROUPED && k >= 8;
    const bool chain_next = grouped && (k % 8) == 0;
    float2 bcol[8], bnxt[8];
    const float2* bj = col_ptr(j < n ? j : 0);
    if (grouped && j < n) {
#pragma unroll
        for (int u = 0; u < 8; ++u) bcol[u] = bel(bj, u);
    }
#pragma unroll 1
    for (; j - threadIdx.x < n; j += step) {
        const bool live = j < n;
        const int64_t jn = j + step;
        const float2* bjn = col_ptr(jn < n ? jn : 0);
        acc_t p[X2 ? 1 : MX][4];
        uint64_t q[X2 ? MX : 1][2];
        if constexpr (X2) {
#pragma unroll
            for (int i = 0; i < MX; ++i) q[i][0] = q[i][1] = 0;  // +0 pairs
        } else {
#pragma unroll
            for (int i = 0; i < MX; ++i) p[i][0] = p[i][1] = p[i][2] = p[i][3] = acc_t(0);
        }
        auto mac = [&](const float2* srow, float xr, float xi) {
            if constexpr (X2)
                skinny_mac_x2<MX>(srow, xr, xi, q, mz);
            else
                skinny_mac<F64, MX>(srow, xr, xi, p, true);
        };
        int k0 = 0;
        if (grouped) {  // A/B on B200: the plain loop wins for k <= 4, grouped loads from 8 up
#pragma unroll 1
            for (; k0 + 8 <= k; k0 += 8) {
                const bool more = k0 + 16 <= k;
                if (more && live) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) bnxt[u] = bel(bj, k0 + 8 + u);
                } else if (!more && chain_next && jn < n) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) bnxt[u] = bel(bjn, u);
                }
                if (live) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) mac(as + (k0 + u) * MX, bcol[u].x, bcol[u].y);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) bcol[u] = bnxt[u];
            }
        }
        if (live) {
#pragma unroll 1
            for (; k0 < k; ++k0) {
                const float2 bv = bel(bj, k0);
                mac(as + k0 * MX, bv.x, bv.y);
            }
#pragma unroll
            for (int i = 0; i < MX; ++i) {
                if (i >= m) continue;
                if constexpr (X2) {
                    const float2 p12 = unpack2(q[i][0]), p34 = unpack2(q[i][1]);
                    __stcs(c + int64_t(i) * n + j,
                           make_float2(__fsub_rn(p12.x, p12.y), __fadd_rn(p34.x, p34.y)));
                } else {
                    __stcs(c + int64_t(i) * n + j, assemble<F64>(p[i]));
                }
            }
        }
        if (grouped && !chain_next && jn < n) {
#pragma unroll
            for (int u = 0; u < 8; ++u) bcol[u] = bel(bjn, u);
        }
        bj = bjn;
    }
}

// Column kernel with the long operand staged through shared memory by
// cp.async (X2 chains, k >= 8).  ncu on the register-prefetch kernel above
// ((16, 2^22, 64), 1.94 GHz): FMA pipe 75 % busy, 3.4 warps per scheduler
// (128 registers), long-scoreboard the top stall -- one group of 8 B values in
// flight per thread is not enough to cover the DRAM latency.  Here every thread
// copies ITS OWN column's next groups (8 x 8 B each) into a private
// shared-memory slice kSkStages - 1 groups ahead, so nothing is shared between
// threads (no barrier, a per-thread cp.async.wait_group), the prefetch
// registers are gone and the walk over 256-column chunks is one continuous
// pipeline.  Same values into the same chains in the same order: bit-identical.
constexpr size_t kSkGroupBytes = size_t(8) * 256 * sizeof(float2);  // one stage: 8 k x 256 columns

TCEC_DEV void cp_async8(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
TCEC_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
TCEC_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int MX, bool VIEW, int kSkStages>
__global__ void __launch_bounds__(256, 2) cgemm_skinny_col_async_kernel(const float2* __restrict__ a,
                                                                     const float2* __restrict__ b,
                                                                     float2* __restrict__ c, int m,
                                                                     int64_t n, int k, const MatrixView view,
                                                                     uint64_t mz) {
    __shared__ __align__(16) float2 as[kSkinnyMaxK * MX];  // [kk][i]
    __shared__ int64_t koff[VIEW ? kSkinnyMaxK : 1];
    extern __shared__ __align__(16) float2 bst[];            // [stage][u][thread]
    for (int t = threadIdx.x; t < k * MX; t += blockDim.x) {
        const int kk = t / MX, i = t % MX;
        as[t] = i < m ? a[i * k + kk] : make_float2(0.0f, 0.0f);
    }
    if (VIEW)
        for (int t = threadIdx.x; t < k; t += blockDim.x) koff[t] = run_offset(view.rows, uint32_t(t));
    __syncthreads();
    const int tid = int(threadIdx.x);
    const int G = k >> 3;  // full groups of 8 k (k >= 8)
    const int64_t step = int64_t(gridDim.x) * blockDim.x;
    auto col_ptr = [&](int64_t jj) { return VIEW ? b + run_offset(view.cols, uint32_t(jj)) : b + jj; };
    auto bel = [&](const float2* bj, int kk) { return VIEW ? bj + koff[kk] : bj + int64_t(kk) * n; };
    // producer state: the next (chunk, group) tile this thread copies
    int it_g = 0, it_s = 0;
    int64_t it_j = int64_t(blockIdx.x) * blockDim.x + tid;
    const float2* it_bj = col_ptr(it_j < n ? it_j : 0);
    auto issue_next = [&]() {
        if (it_j < n) {
            float2* dst = bst + size_t(it_s) * 8 * 256 + tid;
#pragma unroll
            for (int u = 0; u < 8; ++u) cp_async8(dst + u * 256, bel(it_bj, 8 * it_g + u));
        }
        cp_async_commit();  // empty groups too: the count stays uniform
        it_s = it_s + 1 == kSkStages ? 0 : it_s + 1;
        if (++it_g == G) {
            it_g = 0;
            it_j += step;
            it_bj = col_ptr(it_j < n ? it_j : 0);
        }
    };
#pragma unroll
    for (int s = 0; s < kSkStages - 1; ++s) issue_next();
    int cs = 0;  // consumer stage
#pragma unroll 1
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + tid; j - tid < n; j += step) {
        const bool live = j < n;
        uint64_t q[MX][2];
#pragma unroll
        for (int i = 0; i < MX; ++i) q[i][0] = q[i][1] = 0;  // +0 pairs
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
            issue_next();
            cp_async_wait<kSkStages - 1>();  // this thread's copies of the tile landed
            const float2* bs = bst + size_t(cs) * 8 * 256 + tid;
            if (live) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const float2 bv = bs[u * 256];
                    skinny_mac_x2<MX>(as + (8 * g + u) * MX, bv.x, bv.y, q, mz);
                }
            }
            cs = cs + 1 == kSkStages ? 0 : cs + 1;
        }
        if (live) {
            const float2* bj = 8 * G < k ? col_ptr(j) : b;
#pragma unroll 1
            for (int kk = 8 * G; kk < k; ++kk) {
                const float2 bv = __ldcs(bel(bj, kk));
                skinny_mac_x2<MX>(as + kk * MX, bv.x, bv.y, q, mz);
            }
#pragma unroll
            for (int i = 0; i < MX; ++i) {
                if (i >= m) continue;
                const float2 p12 = unpack2(q[i][0]), p34 = unpack2(q[i][1]);
                __stcs(c + int64_t(i) * n + j, make_float2(__fsub_rn(p12.x, p12.y), __fadd_rn(p34.x, p34.y)));
            }
        }
    }
    cp_async_wait<0>();
}

// n <= MX: thread i owns row i of C.  GROUPED (k >= 8, MX <= 8): each warp
// stages its 32 rows of A through shared memory eight k at a time and writes
// its 32 x n block of C back the same way, so global loads and stores are
// row-contiguous runs instead of one lane-strided 8-B access per element.
// VIEW: A is read through a matrix view of the unpermuted tensor, A(i, kk) =
// a[view.rows(i) + view.cols(kk)].
template <bool F64, int MX, bool GROUPED, bool VIEW = false>
__global__ void __launch_bounds__(256) cgemm_skinny_row_kernel(const float2* __restrict__ a,
                                                               const float2* __restrict__ b,
                                                               float2* __restrict__ c, int64_t m,
                                                               int n, int k, int64_t ldn,
                                                               const MatrixView view) {
    // columns [0, n) of a block of B / C whose row stride is ldn
    using acc_t = typename std::conditional<F64, double, float>::type;
    constexpr int SW = (MX + 1) > 9 ? (MX + 1) : 9;  // staging row stride (odd: conflict-free)
    __shared__ __align__(16) float2 bs[kSkinnyMaxK * MX];  // [kk][j]
    __shared__ int64_t koff[VIEW ? kSkinnyMaxK : 1];
    extern __shared__ float2 stage[];  // GROUPED: 8 warps x 32 rows x SW (dynamic, > 48 KB with B at MX = 16)
    for (int t = threadIdx.x; t < k * MX; t += blockDim.x) {
        const int kk = t / MX, jj = t % MX;
        bs[t] = jj < n ? b[int64_t(kk) * ldn + jj] : make_float2(0.0f, 0.0f);
    }
    if (VIEW)
        for (int t = threadIdx.x; t < k; t += blockDim.x) koff[t] = run_offset(view.cols, uint32_t(t));
    __syncthreads();
    auto koffs = [&](int kk) -> int64_t { return VIEW ? koff[kk] : int64_t(kk); };
    acc_t p[MX][4];
#pragma unroll
    for (int j = 0; j < MX; ++j) p[j][0] = p[j][1] = p[j][2] = p[j][3] = acc_t(0);
    if (!GROUPED) {
        const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
        if (i >= m) return;
        const float2* arow = VIEW ? a + run_offset(view.rows, uint32_t(i)) : a + i * k;
#pragma unroll 1
        for (int k0 = 0; k0 < k; ++k0) {
            const float2 av = __ldcs(arow + koffs(k0));
            skinny_mac<F64, MX>(bs + k0 * MX, av.x, av.y, p, false);
        }
        float2* crow = c + i * ldn;
#pragma unroll
        for (int j = 0; j < MX; ++j)
            if (j < n) __stcs(crow + j, assemble<F64>(p[j]));
        return;
    }
    const int lane = threadIdx.x & 31;
    const int64_t w0 = int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31);
    if (w0 >= m) return;  // whole warp past the end
    const int rows = int(min(int64_t(32), m - w0));
    float2* st = stage + (threadIdx.x >> 5) * 32 * SW;
    const float2* ablk = a + w0 * k;
    // VIEW: row offsets of the warp's 32 rows, one per lane (shuffled to the loaders)
    const int64_t my_roff = VIEW && lane < rows ? run_offset(view.rows, uint32_t(w0 + lane)) : 0;
    int k0 = 0;
#pragma unroll 1
    for (; k0 + 8 <= k; k0 += 8) {
        float2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {  // element e = lane + 32u of the 32 x 8 slab: row e / 8, column e % 8
            const int r = (lane >> 3) + 4 * u;
            if (VIEW) {
                const int64_t ro = __shfl_sync(0xFFFFFFFFu, my_roff, r);
                v[u] = r < rows ? __ldcs(a + ro + koff[k0 + (lane & 7)]) : make_float2(0.0f, 0.0f);
            } else {
                v[u] = r < rows ? __ldcs(ablk + int64_t(r) * k + k0 + (lane & 7)) : make_float2(0.0f, 0.0f);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) st[((lane >> 3) + 4 * u) * SW + (lane & 7)] = v[u];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float2 av = st[lane * SW + q];
            skinny_mac<F64, MX>(bs + (k0 + q) * MX, av.x, av.y, p, false);
        }
        __syncwarp();
    }
#pragma unroll 1
    for (; k0 < k; ++k0) {
        const float2 av = lane < rows ? __ldcs(VIEW ? a + my_roff + koff[k0] : ablk + int64_t(lane) * k + k0)
                                      : make_float2(0.0f, 0.0f);
        skinny_mac<F64, MX>(bs + k0 * MX, av.x, av.y, p, false);
    }
#pragma unroll
    for (int j = 0; j < MX; ++j) st[lane * SW + j] = assemble<F64>(p[j]);
    __syncwarp();
    float2* cblk = c + w0 * ldn;
    if (n == MX) {
#pragma unroll
        for (int u = 0; u < MX; ++u) {
            const int e = lane + 32 * u, r = e / MX, j = e % MX;
            if (r < rows) __stcs(cblk + int64_t(r) * ldn + j, st[r * SW + j]);
        }
    } else {
        for (int e = lane; e < rows * n; e += 32) {
            const int r = e / n, j = e - r * n;
            __stcs(cblk + int64_t(r) * ldn + j, st[r * SW + j]);
        }
    }
}

constexpr uint64_t kNegZero2 = 0x8000000080000000ull;  // (-0.0f, -0.0f)

// persistent grid of the column kernels: the co-resident blocks (queried once
// per kernel), never more than the 256-column chunks
template <bool F64, int MX, bool GROUPED, bool VIEW>
unsigned col_grid(int64_t n) {
    static const int per_sm = [] {
        int nb = 0;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                   &nb, cgemm_skinny_col_kernel<F64, MX, GROUPED, VIEW>, 256, 0) == cudaSuccess && nb > 0
                   ? nb
                   : 2;
    }();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t chunks = (n + 255) / 256;
    return unsigned(std::max<int64_t>(1, std::min<int64_t>(chunks, int64_t(per_sm) * sms)));
}

int skinny_view_stages() {
    static const int st = [] {
        const char* e = std::getenv("TCEC_SKINNY_VSTAGES");
        const int v = e ? std::atoi(e) : 0;
        return v >= 2 && v <= 4 ? v : 2;
    }();
    return st;
}

// TCEC_SKINNY_ASYNC=0: the register-prefetch column kernel (A/B)
bool skinny_async_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TCEC_SKINNY_ASYNC");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int MX, bool VIEW, int S>
unsigned col_async_grid(int64_t n) {
    static const int per_sm = [] {
        int nb = 0;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, cgemm_skinny_col_async_kernel<MX, VIEW, S>, 256,
                                                             S * kSkGroupBytes) == cudaSuccess && nb > 0
                   ? nb
                   : 2;
    }();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t chunks = (n + 255) / 256;
    return unsigned(std::max<int64_t>(1, std::min<int64_t>(chunks, int64_t(per_sm) * sms)));
}

template <bool F64, int MX, bool VIEW = false>
void launch_skinny_mx(const float2* a, const float2* b, float2* c, int64_t m, int64_t n, int64_t k,
                      cudaStream_t s, const MatrixView& view = MatrixView{}) {
    // more than 16 short-side rows/columns: passes of <= MX (each re-reads the
    // long operand; register-resident 32-wide tiles measured slower)
    if (m <= n) {
        for (int64_t r0 = 0; r0 < m; r0 += MX) {
            const int rows = int(std::min<int64_t>(MX, m - r0));
            // separate instantiations: the grouped loop's registers must not
            // lower the occupancy of the short-k kernel
            if constexpr (!F64 && MX >= 8) {
                if (k >= 8 && skinny_async_enabled()) {
                    static std::atomic<uint64_t> attr{0};
                    if (ensure_smem_attr(attr, [] {
                            cudaError_t e = cudaSuccess;
                            for (auto f : {cgemm_skinny_col_async_kernel<MX, VIEW, 2>,
                                           cgemm_skinny_col_async_kernel<MX, VIEW, 3>,
                                           cgemm_skinny_col_async_kernel<MX, VIEW, 4>})
                                if (e == cudaSuccess)
                                    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                             int(4 * kSkGroupBytes));
                            return e;
                        }) == cudaSuccess) {
                        const int st = VIEW ? skinny_view_stages() : 4;
                        const float2* ar = a + r0 * k;
                        float2* cr = c + r0 * n;
                        if (st == 2)
                            cgemm_skinny_col_async_kernel<MX, VIEW, 2><<<col_async_grid<MX, VIEW, 2>(n), 256,
                                                                        2 * kSkGroupBytes, s>>>(
                                ar, b, cr, rows, n, int(k), view, kNegZero2);
                        else if (st == 3)
                            cgemm_skinny_col_async_kernel<MX, VIEW, 3><<<col_async_grid<MX, VIEW, 3>(n), 256,
                                                                        3 * kSkGroupBytes, s>>>(
                                ar, b, cr, rows, n, int(k), view, kNegZero2);
                        else
                            cgemm_skinny_col_async_kernel<MX, VIEW, 4><<<col_async_grid<MX, VIEW, 4>(n), 256,
                                                                        4 * kSkGroupBytes, s>>>(
                                ar, b, cr, rows, n, int(k), view, kNegZero2);
                        continue;
                    }
                }
            }
            if (k >= 8)
                cgemm_skinny_col_kernel<F64, MX, true, VIEW>
                    <<<col_grid<F64, MX, true, VIEW>(n), 256, 0, s>>>(
                        a + r0 * k, b, c + r0 * n, rows, n, int(k), view, kNegZero2);
            else
                cgemm_skinny_col_kernel<F64, MX, false, VIEW>
                    <<<col_grid<F64, MX, false, VIEW>(n), 256, 0, s>>>(
                        a + r0 * k, b, c + r0 * n, rows, n, int(k), view, kNegZero2);
        }
    } else {
        for (int64_t j0 = 0; j0 < n; j0 += MX) {
            const int cols = int(std::min<int64_t>(MX, n - j0));
            if (k >= 8) {
                constexpr int SW = (MX + 1) > 9 ? (MX + 1) : 9;
                constexpr int stage_bytes = 8 * 32 * SW * int(sizeof(float2));
                static std::atomic<uint64_t> attr{0};
                if (ensure_smem_attr(attr, [] {
                        return cudaFuncSetAttribute(cgemm_skinny_row_kernel<F64, MX, true, VIEW>,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize, stage_bytes);
                    }) == cudaSuccess) {
                    cgemm_skinny_row_kernel<F64, MX, true, VIEW><<<unsigned((m + 255) / 256), 256, stage_bytes, s>>>(
                        a, b + j0, c + j0, m, cols, int(k), n, view);
                    continue;
                }
            }
            cgemm_skinny_row_kernel<F64, MX, false, VIEW><<<unsigned((m + 255) / 256), 256, 0, s>>>(
                a, b + j0, c + j0, m, cols, int(k), n, view);
        }
    }
}

}  // namespace

bool skinny_shape(int64_t m, int64_t n, int64_t k) {
    const int64_t small = m < n ? m : n, large = m < n ? n : m;
    return !(k > kSkinnyMaxK || small > 32 || large < 4096);
}

namespace {

// true when the skinny kernels take the shape
template <bool F64>
bool launch_skinny(const float2* a, const float2* b, float2* c, int64_t m, int64_t n, int64_t k,
                   cudaStream_t s) {
    const int64_t small = m < n ? m : n;
    // up to 32 rows in register tiles of <= 16 (two passes above 16), k <= 128 in shared memory:
    // the 64 x 64 tiled kernel would waste >= half of every tile on these
    // (the (16, 2^22, 64) and (32, 2^23, 8) steps of Sycamore slices)
    if (!skinny_shape(m, n, k)) return false;
    if (small <= 2) launch_skinny_mx<F64, 2>(a, b, c, m, n, k, s);
    else if (small <= 4) launch_skinny_mx<F64, 4>(a, b, c, m, n, k, s);
    else if (small <= 8) launch_skinny_mx<F64, 8>(a, b, c, m, n, k, s);
    else launch_skinny_mx<F64, 16>(a, b, c, m, n, k, s);  // 17..32: two passes
    return true;
}

template <bool F64>
void launch_chain(const float2* a, const float2* b, float2* c, int64_t m, int64_t n, int64_t k,
                  cudaStream_t s) {
    // two buffers x four chains x CH products: 32 KB for both F32 (CH floats)
    // and F64 (CH/2 doubles)
    const size_t smem = size_t(2) * 4 * kChainChunk * sizeof(float);
    cgemm_chain_kernel<F64><<<unsigned(m * n), kChainThreads, smem, s>>>(a, b, c, m, n, k);
}

// --------------------------------------------------------------- permute

struct PermDesc {
    int rank;
    int64_t total;
    int64_t out_dim[kMaxRank];     // merged output dims (innermost last)
    int64_t in_stride[kMaxRank];   // input stride of each output axis
};

// gather out[pos] = in[offset(pos)]; the output is written fully coalesced,
// axes that stay adjacent are merged on the host so the innermost run is as
// long as possible
__global__ void __launch_bounds__(kThreads) permute_kernel(const float2* __restrict__ src,
                                                           float2* __restrict__ dst,
                                                           const PermDesc desc) {
    for (int64_t pos = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; pos < desc.total;
         pos += int64_t(gridDim.x) * blockDim.x) {
        int64_t rem = pos, off = 0;
        for (int a = desc.rank - 1; a >= 0; --a) {
            const int64_t dim = desc.out_dim[a];
            const int64_t q = rem / dim;
            off += (rem - q * dim) * desc.in_stride[a];
            rem = q;
        }
        dst[pos] = src[off];
    }
}

// Tiled permute (cuTT-style "tiled" plan for high-rank, dim-2 tensors): the
// innermost input axes I (product P_I <= 64, contiguous in the source) and the
// innermost output axes O (product P_O <= 64, contiguous in the destination)
// form a P_O x P_I tile staged through shared memory; every other axis is a
// batch index decoded per block.  Both the global reads (along I) and the
// global writes (along O) are coalesced.
constexpr int kTileMax = 64;

struct TiledPermDesc {
    int pi, po;                       // tile extents
    int nbatch;                       // batch axes (output order)
    int64_t batches;
    int64_t bdim[kMaxRank], bin[kMaxRank], bout[kMaxRank];
    int32_t offi_out[kTileMax];       // output offset of input-inner index i
    int32_t offo_in[kTileMax];        // input offset of output-inner index o
};

__global__ void __launch_bounds__(256) permute_tiled_kernel(const float2* __restrict__ src,
                                                            float2* __restrict__ dst,
                                                            const TiledPermDesc d) {
    __shared__ float2 tile[kTileMax][kTileMax + 1];
    __shared__ int32_t offi[kTileMax], offo[kTileMax];
    if (threadIdx.x < kTileMax) {
        offi[threadIdx.x] = d.offi_out[threadIdx.x];
        offo[threadIdx.x] = d.offo_in[threadIdx.x];
    }
    const int tile_n = d.pi * d.po;
    for (int64_t b = blockIdx.x; b < d.batches; b += gridDim.x) {
        int64_t rem = b, base_in = 0, base_out = 0;
        for (int a = d.nbatch - 1; a >= 0; --a) {
            const int64_t q = rem / d.bdim[a];
            const int64_t x = rem - q * d.bdim[a];
            base_in += x * d.bin[a];
            base_out += x * d.bout[a];
            rem = q;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < tile_n; t += blockDim.x) {
            const int o = t / d.pi, i = t - o * d.pi;
            tile[o][i] = src[base_in + offo[o] + i];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < tile_n; t += blockDim.x) {
            const int i = t / d.po, o = t - i * d.po;
            dst[base_out + offi[i] + o] = tile[o][i];
        }
    }
}

// Bit-permutation permute: when every extent is a power of two (the dim-2
// bonds of circuit networks), a permutation of axes is a permutation of the
// bits of the linear index.  The tile is spanned by the 5 lowest input bits
// (32 consecutive source elements) and the input bits feeding the 5 lowest
// output bits (32 consecutive destination elements): up to 1024 elements
// staged through XOR-swizzled shared memory, so reads and writes are both
// coalesced 256-B runs.  The remaining bits index the tiles.  Offsets inside a
// tile come from per-block shared tables built once (persistent grid).
constexpr int kBitTileMax = 12;   // tile bits: up to 4096 elements (32 KB)
constexpr int kBitThreads = 512;  // 8 elements per thread in flight

// Run copy (power-of-two extents): the innermost output axis is contiguous
// in the source and at least 32 elements long, so the permute is a gather of
// >= 256-B runs -- e.g. moving a few outer axes to the front, the common TTGT
// case of sliced circuit intermediates.  Each thread moves 16 B; a warp
// covers whole runs on both sides, no shared-memory staging (the tiled bit
// permute moves these at ~0.69 of the copy bandwidth).
struct RunPermDesc {
    int rank;                   // merged output axes, the innermost is the run
    int log_dim[kMaxRank];      // log2 extent per output axis
    int64_t in_stride4[kMaxRank];  // input stride in float4 units (axis < rank - 1)
    int64_t total4;
};

__global__ void __launch_bounds__(256) permute_runs_kernel(const float4* __restrict__ src,
                                                           float4* __restrict__ dst,
                                                           const RunPermDesc d) {
    const int run_log = d.log_dim[d.rank - 1] - 1;  // float4 per run = 2^run_log
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    auto src_of = [&](int64_t p4) {
        int64_t rem = p4 >> run_log, off = p4 & ((int64_t(1) << run_log) - 1);
        for (int a = d.rank - 2; a >= 0; --a) {
            off += (rem & ((int64_t(1) << d.log_dim[a]) - 1)) * d.in_stride4[a];
            rem >>= d.log_dim[a];
        }
        return off;
    };
    int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    for (; p + 3 * stride < d.total4; p += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcs(src + src_of(p + u * stride));
#pragma unroll
        for (int u = 0; u < 4; ++u) __stcs(dst + p + u * stride, v[u]);
    }
    for (; p < d.total4; p += stride) __stcs(dst + p, __ldcs(src + src_of(p)));
}

struct BitPermDesc {
    int nbits;                  // log2(total)
    int ntile;                  // tile bits (|U|)
    int nrest;                  // remaining bits
    int8_t tile_in[kBitTileMax];    // input bit of tile bit t (input-bit order)
    int8_t tile_out[kBitTileMax];   // output bit of tile bit t
    int8_t out_rank[kBitTileMax];   // rank of tile bit t among the tile bits by output position
    int8_t rest_in[64], rest_out[64];  // input / output bit of remaining bit r (output order)
};

TCEC_DEV uint32_t bp_swz(uint32_t s) { return s ^ (((s >> 4) ^ (s >> 8)) & 15u); }

// E = float2 (one complex element) or float4 (a pair: the innermost axis
// stays innermost, so input bit 0 is output bit 0 and pairs move as 16-B units)
template <typename E, int TB>
__global__ void __launch_bounds__(kBitThreads) permute_bits_kernel(const E* __restrict__ src,
                                                                   E* __restrict__ dst,
                                                                   const BitPermDesc d) {
    __shared__ E tile[1 << TB];
    // offsets are sums over index bits, so each table splits into a 6-bit low
    // and a 6-bit high half: off(t) = lo[t & 63] + hi[t >> 6]
    __shared__ uint64_t in_lo[64], in_hi[64], out_lo[64], out_hi[64];
    __shared__ uint16_t s_lo[64], s_hi[64];
    const int T = 1 << d.ntile;
    if (threadIdx.x < 64) {
        const int v = threadIdx.x;
        uint64_t il = 0, ih = 0, ol = 0, oh = 0;
        uint32_t sl = 0, sh = 0;
        for (int bt = 0; bt < d.ntile; ++bt) {
            if (bt < 6 && ((v >> bt) & 1)) {
                il |= uint64_t(1) << d.tile_in[bt];
                ol |= uint64_t(1) << d.tile_out[bt];
            }
            if (bt >= 6 && ((v >> (bt - 6)) & 1)) {
                ih |= uint64_t(1) << d.tile_in[bt];
                oh |= uint64_t(1) << d.tile_out[bt];
            }
            // u -> t: output rank r of tile bit bt sits at bit r of u
            const int r = d.out_rank[bt];
            if (r < 6 && ((v >> r) & 1)) sl |= 1u << bt;
            if (r >= 6 && ((v >> (r - 6)) & 1)) sh |= 1u << bt;
        }
        in_lo[v] = il;
        in_hi[v] = ih;
        out_lo[v] = ol;
        out_hi[v] = oh;
        s_lo[v] = uint16_t(sl);
        s_hi[v] = uint16_t(sh);
    }
    __syncthreads();
    const int64_t ntiles = int64_t(1) << d.nrest;
    auto bases = [&](int64_t blk, int64_t& bi, int64_t& bo) {
        bi = 0;
        bo = 0;
        for (int r = 0; r < d.nrest; ++r)
            if ((blk >> r) & 1) {
                bi |= int64_t(1) << d.rest_in[r];
                bo |= int64_t(1) << d.rest_out[r];
            }
    };
    auto in_off = [&](int t) { return in_lo[t & 63] + in_hi[t >> 6]; };
    // software pipeline: the next tile's loads are in flight while this
    // tile's stores drain
    constexpr int kPer = (1 << TB) / kBitThreads;
    E reg[kPer];
    int64_t blk = blockIdx.x, base_in = 0, base_out = 0;
    if (blk < ntiles) {
        bases(blk, base_in, base_out);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int t = threadIdx.x + kBitThreads * e;
            if (t < T) reg[e] = __ldcs(src + base_in + in_off(t));
        }
    }
    while (blk < ntiles) {
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int t = threadIdx.x + kBitThreads * e;
            if (t < T) tile[bp_swz(uint32_t(t))] = reg[e];
        }
        __syncthreads();
        const int64_t next = blk + gridDim.x;
        const int64_t out_base = base_out;
        if (next < ntiles) {
            bases(next, base_in, base_out);
#pragma unroll
            for (int e = 0; e < kPer; ++e) {
                const int t = threadIdx.x + kBitThreads * e;
                if (t < T) reg[e] = __ldcs(src + base_in + in_off(t));
            }
        }
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int u = threadIdx.x + kBitThreads * e;
            if (u < T) {
                const uint32_t t = uint32_t(s_lo[u & 63]) | uint32_t(s_hi[u >> 6]);
                __stcs(dst + out_base + out_lo[t & 63] + out_hi[t >> 6], tile[bp_swz(t)]);
            }
        }
        __syncthreads();
        blk = next;
    }
}

}  // namespace

// Plan the tiled permute; false when the shape does not suit it.
static bool plan_tiled(int r, const int64_t* dim_in, const int64_t* in_stride_in, TiledPermDesc* d) {
    // axes in output order with output strides, splitting large axes into
    // (D/32, 32) so tiles stay <= 64 per side
    int64_t dim[kMaxRank], ist[kMaxRank], ost[kMaxRank];
    int n = 0;
    int64_t os = 1;
    int64_t tmp_dim[kMaxRank], tmp_ist[kMaxRank];
    for (int a = 0; a < r; ++a) {
        tmp_dim[a] = dim_in[a];
        tmp_ist[a] = in_stride_in[a];
    }
    int64_t odim[kMaxRank], oist[kMaxRank];
    int m = 0;
    for (int a = 0; a < r; ++a) {
        const int64_t D = tmp_dim[a], S = tmp_ist[a];
        if (D > kTileMax) {
            if (D % 32 != 0 || m + 2 > kMaxRank) return false;
            odim[m] = D / 32;
            oist[m++] = S * 32;
            odim[m] = 32;
            oist[m++] = S;
        } else {
            if (m + 1 > kMaxRank) return false;
            odim[m] = D;
            oist[m++] = S;
        }
    }
    for (int a = m - 1; a >= 0; --a) {
        dim[a] = odim[a];
        ist[a] = oist[a];
        ost[a] = os;
        os *= odim[a];
    }
    n = m;
    // input-inner group: axes by ascending input stride, contiguous block
    int order[kMaxRank];
    for (int a = 0; a < n; ++a) order[a] = a;
    for (int a = 1; a < n; ++a)
        for (int b = a; b > 0 && ist[order[b]] < ist[order[b - 1]]; --b) {
            const int t = order[b];
            order[b] = order[b - 1];
            order[b - 1] = t;
        }
    bool in_I[kMaxRank] = {false}, in_O[kMaxRank] = {false};
    int64_t pi = 1;
    int nI = 0;
    for (int j = 0; j < n; ++j) {
        const int a = order[j];
        if (ist[a] != pi || pi * dim[a] > kTileMax) break;
        pi *= dim[a];
        in_I[a] = true;
        ++nI;
    }
    int64_t po = 1;
    for (int a = n - 1; a >= 0; --a) {
        if (po * dim[a] > kTileMax) break;
        if (in_I[a]) return false;  // overlapping groups: the gather kernel handles it
        po *= dim[a];
        in_O[a] = true;
    }
    if (pi < 8 || po < 8) return false;
    d->pi = int(pi);
    d->po = int(po);
    // offsets inside the tile
    for (int i = 0; i < pi; ++i) {
        int64_t rem = i, off = 0;
        for (int j = 0; j < nI; ++j) {
            const int a = order[j];
            off += (rem % dim[a]) * ost[a];
            rem /= dim[a];
        }
        d->offi_out[i] = int32_t(off);
    }
    for (int o = 0; o < po; ++o) {
        int64_t rem = o, off = 0;
        for (int a = n - 1; a >= 0 && in_O[a]; --a) {
            off += (rem % dim[a]) * ist[a];
            rem /= dim[a];
        }
        d->offo_in[o] = int32_t(off);
    }
    d->nbatch = 0;
    d->batches = 1;
    for (int a = 0; a < n; ++a) {
        if (in_I[a] || in_O[a]) continue;
        d->bdim[d->nbatch] = dim[a];
        d->bin[d->nbatch] = ist[a];
        d->bout[d->nbatch] = ost[a];
        d->batches *= dim[a];
        ++d->nbatch;
    }
    return true;
}

// ================================================================ launchers

void launch_quantize(const float* src, float* dst, int64_t n, int fmt, int rz, unsigned* d_ovf,
                     cudaStream_t s) {
    if (n <= 0) return;
    quantize_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(src, dst, n, fmt, rz, d_ovf);
}

void launch_split_flat(const float* src, float* hi, float* lo, int64_t n, int fmt, unsigned* d_ovf,
                       cudaStream_t s) {
    if (n <= 0) return;
    split_flat_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(src, hi, lo, n, fmt, d_ovf);
}

void launch_scale(const float* src, float* dst, int64_t n, int scale_exp, unsigned* d_nonfinite,
                  cudaStream_t s) {
    if (n <= 0) return;
    scale_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(src, dst, n, ldexp(1.0, scale_exp),
                                                             d_nonfinite);
}

void launch_add_sub(const float* a, const float* b, float* dst, int64_t n, int sub,
                    cudaStream_t s) {
    if (n <= 0) return;
    add_sub_kernel<<<grid_for(n, kThreads), kThreads, 0, s>>>(a, b, dst, n, sub);
}

// blocks of the statistics sweeps: one wave of 8 x 256-thread blocks per SM
// at most, split between A and B in proportion to their sizes (>= 1 each)
static void stats_grid(int64_t na, int64_t nb, const float* a, const float* b, int* total, int* nb_a) {
    const int64_t ea = a ? na : 0, eb = b ? nb : 0;
    const int64_t want = (ea + eb) / (4 * kThreads * 4) + 2;  // >= 4 float4 per thread
    const int tot = int(std::min<int64_t>(148 * 8, std::max<int64_t>(2, want)));
    int ba = ea ? int(std::max<int64_t>(1, std::min<int64_t>(tot - 1, (tot * ea + ea + eb - 1) / (ea + eb))))
                : 0;
    if (!eb) ba = ea ? tot : 0;
    *nb_a = ba;
    *total = std::max(1, eb ? tot : ba);
}

// L2 policy of the statistics sweeps: operands that fit in L2 next to their
// preparation's output stay resident for the second sweep and the preparation
// (TCEC_STATS_KEEP = 0 / 1 forces streaming / keeping)
static int stats_keep(int64_t na, int64_t nb) {
    static const int mode = [] {
        const char* e = std::getenv("TCEC_STATS_KEEP");
        return e ? std::atoi(e) : -1;
    }();
    if (mode >= 0) return mode ? 1 : 0;
    return (na + nb) * 4 <= (int64_t(96) << 20) ? 1 : 0;
}

void launch_stats1(const float* a, int64_t na, const float* b, int64_t nb, DevDecision* d,
                   cudaStream_t s) {
    int total = 0, nb_a = 0;
    stats_grid(na, nb, a, b, &total, &nb_a);
    stats1_kernel<<<total, kThreads, 0, s>>>(a, na, b, nb, d, nb_a, stats_keep(na, nb));
}

void launch_stats2(const float* a, int64_t na, const float* b, int64_t nb, DevDecision* d,
                   double t, int target, int always, cudaStream_t s, int select, double sel_t,
                   int forced_scaled, float spec_fa, float spec_fb) {
    int total = 0, nb_a = 0;
    stats_grid(na, nb, a, b, &total, &nb_a);
    stats2_kernel<<<total, kThreads, 0, s>>>(a, na, b, nb, d, t, target, always, nb_a, stats_keep(na, nb),
                                             select, sel_t, forced_scaled, spec_fa, spec_fb);
}

void launch_prep_a(const float* a, int64_t m, int64_t k, int64_t kp, void* hi, void* lo,
                   const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s, int64_t row0,
                   const MatrixView* view) {
    const int64_t total = m * (kp / 8);
    if (total <= 0) return;
    const unsigned grid = unsigned(grid_for(total, kThreads, 148 * 32));
    if (view)
        prep_a_kernel<true><<<grid, kThreads, 0, s>>>(a, m, 2 * k, kp, hi, lo, d, kind_fixed, corrected, row0, *view);
    else
        prep_a_kernel<false><<<grid, kThreads, 0, s>>>(a, m, 2 * k, kp, hi, lo, d, kind_fixed, corrected, row0,
                                                       MatrixView{});
}

void launch_prep_b(const float* b, int64_t k, int64_t n, int64_t kp, void* hi, void* lo,
                   const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s, int64_t jout0,
                   const MatrixView* view) {
    if (n <= 0 || kp <= 0) return;
    const int64_t tiles = ((n + kPrepBJ - 1) / kPrepBJ) * ((kp / 2 + kPrepBKK - 1) / kPrepBKK);
    const unsigned grid = unsigned(tiles < 148 * 8 ? tiles : 148 * 8);
    const float2* b2 = reinterpret_cast<const float2*>(b);
    if (view)
        prep_b_kernel<true><<<grid, 256, 0, s>>>(b2, k, n, kp, hi, lo, d, kind_fixed, corrected, jout0, *view);
    else
        prep_b_kernel<false><<<grid, 256, 0, s>>>(b2, k, n, kp, hi, lo, d, kind_fixed, corrected, jout0,
                                                  MatrixView{});
}

void launch_prep_ax(const float* a, int64_t m, int64_t k, int64_t kp, void* hi, void* lo,
                    const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s,
                    const MatrixView* view) {
    const int64_t total = m * (kp / 8);
    if (total <= 0) return;
    const unsigned grid = unsigned(grid_for(total, kThreads, 148 * 32));
    if (view)
        prep_ax_kernel<true><<<grid, kThreads, 0, s>>>(a, m, k, kp, hi, lo, d, kind_fixed, corrected, *view);
    else
        prep_ax_kernel<false><<<grid, kThreads, 0, s>>>(a, m, k, kp, hi, lo, d, kind_fixed, corrected,
                                                        MatrixView{});
}

void launch_prep_bx(const float* b, int64_t k, int64_t n, int64_t kp, void* hi, void* lo,
                    const DevDecision* d, int kind_fixed, int corrected, cudaStream_t s,
                    const MatrixView* view) {
    if (n <= 0 || kp <= 0) return;
    const int64_t tiles = ((n + kPrepBJ - 1) / kPrepBJ) * ((kp / 2 + kPrepBKK - 1) / kPrepBKK);
    const unsigned grid = unsigned(tiles < 148 * 8 ? tiles : 148 * 8);
    const float2* b2 = reinterpret_cast<const float2*>(b);
    if (view)
        prep_bx_kernel<true><<<grid, 256, 0, s>>>(b2, k, n, kp, hi, lo, d, kind_fixed, corrected, *view);
    else
        prep_bx_kernel<false><<<grid, 256, 0, s>>>(b2, k, n, kp, hi, lo, d, kind_fixed, corrected, MatrixView{});
}

void launch_cgemm_fp32_ref(const float2* a, const float2* b, float2* c, int64_t m, int64_t n,
                           int64_t k, cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    const int64_t tiles = ((n + SB_N - 1) / SB_N) * ((m + SB_M - 1) / SB_M);
    if (k >= 65536 && m * n <= 4096) {
        launch_chain<false>(a, b, c, m, n, k, s);
        return;
    }
    if (launch_skinny<false>(a, b, c, m, n, k, s)) return;
    if (k >= 1024 && m * n <= 65536 && tiles < 2 * 148) {
        if (m * n >= 2048) {
            // enough outputs for a thread each: one output per thread
            const int64_t blocks = ((m + 15) / 16) * ((n + 15) / 16);
            cgemm_tpo_kernel<false><<<unsigned(blocks), 256, 0, s>>>(a, b, c, m, n, k);
            return;
        }
        const int64_t warps = m * n;
        cgemm_longk_kernel<false><<<unsigned((warps + 7) / 8), 256, 0, s>>>(a, b, c, m, n, k);
        return;
    }
    cgemm_fp32_ref_kernel<<<unsigned(tiles), 256, 0, s>>>(a, b, c, m, n, k);
}

void launch_cgemm_fp64(const float2* a, const float2* b, float2* c, int64_t m, int64_t n,
                       int64_t k, cudaStream_t s) {
    if (m <= 0 || n <= 0) return;
    if (k >= 65536 && m * n <= 4096) {
        launch_chain<true>(a, b, c, m, n, k, s);
        return;
    }
    if (launch_skinny<true>(a, b, c, m, n, k, s)) return;
    if (k >= 256 && m * n <= 65536 && m * n >= 2048) {
        const int64_t blocks = ((m + 15) / 16) * ((n + 15) / 16);
        cgemm_tpo_kernel<true><<<unsigned(blocks), 256, 0, s>>>(a, b, c, m, n, k);
        return;
    }
    if (k >= 256 && m * n <= 65536) {
        cgemm_longk_kernel<true><<<unsigned((m * n + 7) / 8), 256, 0, s>>>(a, b, c, m, n, k);
        return;
    }
    const unsigned grid = unsigned(((n + 127) / 128) * m);
    cgemm_fp64_kernel<<<grid, 128, 0, s>>>(a, b, c, m, n, k);
}

void launch_permute(const float2* src, float2* dst, int rank, const int64_t* old_dims,
                    const int* axis_of, cudaStream_t s) {
    PermDesc desc{};
    int64_t total = 1;
    for (int a = 0; a < rank; ++a) total *= old_dims[a];
    desc.total = total;
    if (total == 0) return;
    // old strides, then merge runs of output axes that are adjacent in the input
    int64_t old_stride[kMaxRank];
    if (rank > 0) old_stride[rank - 1] = 1;
    for (int a = rank - 2; a >= 0; --a) old_stride[a] = old_stride[a + 1] * old_dims[a + 1];
    int r = 0;
    for (int a = 0; a < rank; ++a) {
        const int64_t dim = old_dims[axis_of[a]];
        if (dim == 1) continue;
        const int64_t st = old_stride[axis_of[a]];
        if (r > 0 && desc.in_stride[r - 1] == st * dim) {
            desc.out_dim[r - 1] *= dim;
            desc.in_stride[r - 1] = st;
        } else {
            desc.out_dim[r] = dim;
            desc.in_stride[r] = st;
            ++r;
        }
    }
    desc.rank = r;
    // power-of-two extents: permutation of index bits, coalesced on both sides
    if (total >= 1024 && (total & (total - 1)) == 0) {
        bool pow2 = true;
        for (int a = 0; a < r; ++a) pow2 = pow2 && (desc.out_dim[a] & (desc.out_dim[a] - 1)) == 0;
        if (pow2 && r >= 2 && desc.in_stride[r - 1] == 1 && desc.out_dim[r - 1] >= 32 &&
            (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            RunPermDesc rd{};
            rd.rank = r;
            for (int a = 0; a < r; ++a) {
                rd.log_dim[a] = __builtin_ctzll(uint64_t(desc.out_dim[a]));
                rd.in_stride4[a] = desc.in_stride[a] / 2;  // strides of the outer axes are >= the run
            }
            rd.total4 = total / 2;
            const int64_t blocks = (rd.total4 + 255) / 256;
            permute_runs_kernel<<<unsigned(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, s>>>(
                reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), rd);
            return;
        }
        if (pow2) {
            int src_bit[64];
            int j = 0;  // output bit, LSB first: axes from the innermost
            for (int a = r - 1; a >= 0; --a) {
                const int w = __builtin_ctzll(uint64_t(desc.out_dim[a]));
                const int s0 = __builtin_ctzll(uint64_t(desc.in_stride[a]));
                for (int b = 0; b < w; ++b) src_bit[j++] = s0 + b;
            }
            // the innermost axis stays innermost: move 16-B pairs (one bit fewer)
            const bool pairs = j >= 11 && src_bit[0] == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                               (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
            if (pairs) {
                for (int o = 1; o < j; ++o) src_bit[o - 1] = src_bit[o] - 1;
                --j;
            }
            const int tile_max = pairs ? kBitTileMax - 1 : kBitTileMax;  // 32 KB of shared memory either way
            BitPermDesc bd{};
            bd.nbits = j;
            bool in_tile[64] = {false};
            const int lo = j < 5 ? j : 5;
            for (int b = 0; b < lo; ++b) in_tile[b] = true;           // input bits 0..4
            for (int o = 0; o < lo; ++o) in_tile[src_bit[o]] = true;  // feeding output bits 0..4
            // where the two groups overlap, widen the tile with the next input
            // bits so every tile moves ~1024 elements (8 KB) per pass
            int cnt = 0;
            for (int b = 0; b < j; ++b) cnt += in_tile[b];
            for (int b = lo; b < j && cnt < tile_max; ++b)
                if (!in_tile[b]) {
                    in_tile[b] = true;
                    ++cnt;
                }
            int out_of_in[64];
            for (int o = 0; o < j; ++o) out_of_in[src_bit[o]] = o;
            bd.ntile = 0;
            for (int b = 0; b < j; ++b)
                if (in_tile[b]) {
                    bd.tile_in[bd.ntile] = int8_t(b);
                    bd.tile_out[bd.ntile] = int8_t(out_of_in[b]);
                    ++bd.ntile;
                }
            bd.nrest = 0;
            for (int o = 0; o < j; ++o)
                if (!in_tile[src_bit[o]]) {
                    bd.rest_in[bd.nrest] = int8_t(src_bit[o]);
                    bd.rest_out[bd.nrest] = int8_t(o);
                    ++bd.nrest;
                }
            for (int b = 0; b < bd.ntile; ++b) {
                int rk = 0;
                for (int c = 0; c < bd.ntile; ++c) rk += bd.tile_out[c] < bd.tile_out[b];
                bd.out_rank[b] = int8_t(rk);
            }
            const int64_t ntiles = int64_t(1) << bd.nrest;
            const int64_t g = ntiles < 148 * 4 ? ntiles : 148 * 4;
            if (pairs)
                permute_bits_kernel<float4, kBitTileMax - 1><<<unsigned(g), kBitThreads, 0, s>>>(
                    reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), bd);
            else
                permute_bits_kernel<float2, kBitTileMax><<<unsigned(g), kBitThreads, 0, s>>>(src, dst, bd);
            return;
        }
    }
    // innermost output axis not contiguous in the source: shared-memory tiles
    if (r >= 2 && desc.in_stride[r - 1] != 1 && total >= 4096) {
        TiledPermDesc td{};  // per call: the planner is reentrant (handles may run on several host threads)
        if (plan_tiled(r, desc.out_dim, desc.in_stride, &td)) {
            const int64_t g = td.batches < 148 * 16 ? td.batches : 148 * 16;
            permute_tiled_kernel<<<unsigned(g), 256, 0, s>>>(src, dst, td);
            return;
        }
    }
    permute_kernel<<<grid_for(total, kThreads, 148 * 32), kThreads, 0, s>>>(src, dst, desc);
}

bool launch_skinny_view(const float2* a, const float2* b, float2* c, int64_t m, int64_t n, int64_t k,
                        const MatrixView& v, cudaStream_t s) {
    if (!skinny_shape(m, n, k) || m <= 0 || n <= 0 || k <= 0) return false;
    // the view indexes fit 32 bits (run_offset): rows/cols < 2^32
    if (m > int64_t(0xFFFFFFFF) || n > int64_t(0xFFFFFFFF)) return false;
    const int64_t small = m < n ? m : n;
    if (small <= 2) launch_skinny_mx<false, 2, true>(a, b, c, m, n, k, s, v);
    else if (small <= 4) launch_skinny_mx<false, 4, true>(a, b, c, m, n, k, s, v);
    else if (small <= 8) launch_skinny_mx<false, 8, true>(a, b, c, m, n, k, s, v);
    else launch_skinny_mx<false, 16, true>(a, b, c, m, n, k, s, v);
    return true;
}

// runs of new axes [a0, a1): adjacent new axes merge when they are adjacent
// (and in order) in the tensor's physical layout
static bool make_runs(int a0, int a1, const int64_t* dims, const int64_t* pstride, const int* axis_of,
                      RunMap* rm) {
    RunMap r;
    for (int a = a0; a < a1; ++a) {
        const int o = axis_of[a];
        const int64_t e = dims[o], st = pstride[o];
        if (e == 1) continue;
        if (r.n > 0 && r.stride[r.n - 1] == st * e && uint64_t(r.ext[r.n - 1]) * uint64_t(e) <= 0xFFFFFFFFull) {
            r.ext[r.n - 1] = uint32_t(uint64_t(r.ext[r.n - 1]) * uint64_t(e));
            r.stride[r.n - 1] = st;
            continue;
        }
        if (r.n == kMaxRuns || e > int64_t(0xFFFFFFFF)) return false;
        r.ext[r.n] = uint32_t(e);
        r.stride[r.n] = st;
        ++r.n;
    }
    r.pow2 = 1;
    for (int i = 0; i < r.n; ++i) {
        if (r.ext[i] & (r.ext[i] - 1)) r.pow2 = 0;
        int sh = 0;
        while ((1ull << sh) < r.ext[i]) ++sh;
        r.shift[i] = uint32_t(sh);
    }
    *rm = r;
    return true;
}

bool make_matrix_view(int rank, const int64_t* dims, const int* axis_of, int n_row_axes, MatrixView* v) {
    if (rank < 0 || rank > kMaxRank || n_row_axes < 0 || n_row_axes > rank) return false;
    int64_t pstride[kMaxRank];
    int64_t acc = 1;
    for (int i = rank - 1; i >= 0; --i) {
        pstride[i] = acc;
        acc *= dims[i];
    }
    return make_runs(0, n_row_axes, dims, pstride, axis_of, &v->rows) &&
           make_runs(n_row_axes, rank, dims, pstride, axis_of, &v->cols);
}

}  // namespace tcec
