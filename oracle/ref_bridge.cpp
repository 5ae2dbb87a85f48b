// TEST INFRASTRUCTURE ONLY -- extern "C" bridge onto the UNMODIFIED reference
// library (mpsgemm, /root/reference/proj).  oracle/Makefile compiles this file
// together with the reference's own sources (read in place, never copied) into
// oracle/_ref/libmpsgemm_ref.so.  It is used to
//   * pin the C restatement (oracle/tcec_oracle.c) against the reference,
//   * generate the golden fixtures under tests/golden/,
//   * time the reference CPU path for bench.py --impl reference.
// Nothing in the product path links or loads it.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <functional>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "mpsgemm/cgemm.hpp"
#include "mpsgemm/kernels.hpp"
#include "mpsgemm/network.hpp"
#include "mpsgemm/precsel.hpp"
#include "mpsgemm/qcircuit.hpp"
#include "mpsgemm/rng.hpp"
#include "mpsgemm/tensor.hpp"

using namespace mpsgemm;

namespace {

// layout-identical to orc_exp_stats_t (oracle/tcec_oracle.h)
struct StatsPod {
    std::uint64_t n1, n2;
    std::int32_t e_max, e_max_valid;
    std::uint64_t n_nonzero, n_total;
    std::int32_t stage2_evaluated, pad_;
};

struct ConfigPod {
    double threshold_t;
    std::int64_t size_auto, size_tf32;
    std::int32_t target_max_exponent, k_tile, force, pad_;
};

struct ResultPod {
    std::int32_t kind, scale_a, scale_b, overflow;
    std::int32_t has_stats, pad_;
    StatsPod stats_a, stats_b;
    char line[160];
};

StatsPod to_pod(const ExpStats& s) {
    StatsPod p{};
    p.n1 = s.n1;
    p.n2 = s.n2;
    p.e_max_valid = s.e_max.has_value();
    p.e_max = s.e_max.value_or(0);
    p.n_nonzero = s.n_nonzero;
    p.n_total = s.n_total;
    p.stage2_evaluated = s.stage2_evaluated;
    return p;
}

ExpStats from_pod(const StatsPod& p) {
    ExpStats s;
    s.n1 = p.n1;
    s.n2 = p.n2;
    if (p.e_max_valid) s.e_max = p.e_max;
    s.n_nonzero = p.n_nonzero;
    s.n_total = p.n_total;
    s.stage2_evaluated = p.stage2_evaluated != 0;
    return s;
}

MatrixC32 load_c32(const float* p, std::int64_t rows, std::int64_t cols) {
    MatrixC32 m(rows, cols);
    std::memcpy(m.data.data(), p, sizeof(float) * 2 * static_cast<std::size_t>(rows * cols));
    return m;
}

DispatchConfig to_config(const ConfigPod* c) {
    DispatchConfig dc;
    dc.policy.threshold_t = c->threshold_t;
    dc.policy.size_auto = c->size_auto;
    dc.policy.size_tf32 = c->size_tf32;
    dc.policy.target_max_exponent = c->target_max_exponent;
    dc.tiling.k_tile = c->k_tile;
    if (c->force >= 0) dc.force = static_cast<ForcedMode>(c->force);
    return dc;
}

int error_code() {
    try {
        throw;
    } catch (const ScaleOverflow&) {
        return 1;
    } catch (const std::logic_error&) {
        return 2;
    } catch (...) {
        return 9;
    }
}

Bitstring bits_of(const std::uint8_t* bits, int n) { return Bitstring(bits, bits + n); }

} // namespace

extern "C" {

const char* ref_kernel_name() { return kernels::active_kernels().name; }

void ref_set_kernel_arch(int arch) { kernels::set_kernel_arch(static_cast<kernels::KernelArch>(arch)); }

void ref_quantize_buf(const float* src, float* dst, std::int64_t n, int fmt, int rounding, int* ovf) {
    bool o = false;
    kernels::active_kernels().quantize_buf(src, dst, n, static_cast<lowprec::FormatKind>(fmt),
                                           static_cast<lowprec::Rounding>(rounding), &o);
    if (o) *ovf = 1;
}

void ref_split_buf(const float* src, float* hi, float* lo, std::int64_t n, int fmt, int* ovf) {
    bool o = false;
    kernels::active_kernels().split_buf(src, hi, lo, n, static_cast<lowprec::FormatKind>(fmt), &o);
    if (o) *ovf = 1;
}

void ref_scale_buf(const float* src, float* dst, std::int64_t n, int s) {
    kernels::active_kernels().scale_buf(src, dst, n, s);
}

float ref_add_rz(float a, float b) { return lowprec::add_rz(a, b); }

int ref_exponent_of(float x, int* e) {
    const auto v = lowprec::exponent_of(x);
    if (v) *e = *v;
    return v.has_value();
}

void ref_exp_stats(const float* x, std::int64_t rows, std::int64_t cols, int target, StatsPod* out) {
    *out = to_pod(exp_stats(load_c32(x, rows, cols), target));
}

void ref_exp_stats_staged(const float* x, std::int64_t rows, std::int64_t cols, int target, double t,
                          StatsPod* out) {
    *out = to_pod(exp_stats_staged(load_c32(x, rows, cols), target, t));
}

int ref_matrix_tolerance(const StatsPod* s, double t, int target) {
    try {
        return static_cast<int>(matrix_tolerance(from_pod(*s), t, target).level);
    } catch (...) {
        return -1;
    }
}

void ref_select_mode(int la, int eva, int ea, int lb, int evb, int eb, int target, int* kind,
                     int* sa, int* sb) {
    MatrixTolerance ta{static_cast<ToleranceLevel>(la), std::nullopt};
    MatrixTolerance tb{static_cast<ToleranceLevel>(lb), std::nullopt};
    if (eva) ta.e_max = ea;
    if (evb) tb.e_max = eb;
    const ComputeMode m = select_mode(ta, tb, target);
    *kind = static_cast<int>(m.kind);
    *sa = m.scale_exp_a;
    *sb = m.scale_exp_b;
}

int ref_cgemm(const float* a, const float* b, float* c, std::int64_t m, std::int64_t n,
              std::int64_t k, int mode, int k_tile, int* ovf) {
    try {
        bool o = false;
        const MatrixC32 r = cgemm(load_c32(a, m, k), load_c32(b, k, n), static_cast<GemmMode>(mode),
                                  TilingConfig{k_tile}, &o);
        std::memcpy(c, r.data.data(), sizeof(float) * 2 * static_cast<std::size_t>(m * n));
        if (o) *ovf = 1;
        return 0;
    } catch (...) {
        return error_code();
    }
}

void ref_cgemm_oracle(const float* a, const float* b, double* c, std::int64_t m, std::int64_t n,
                      std::int64_t k) {
    const MatrixC64 r = cgemm_oracle(load_c32(a, m, k), load_c32(b, k, n));
    std::memcpy(c, r.data.data(), sizeof(double) * 2 * static_cast<std::size_t>(m * n));
}

int ref_dispatch_cgemm(const float* a, const float* b, float* c, std::int64_t m, std::int64_t n,
                       std::int64_t k, const ConfigPod* cfg, ResultPod* res) {
    std::memset(res, 0, sizeof(*res));
    try {
        DecisionLog log;
        const DispatchResult r =
            dispatch_cgemm(load_c32(a, m, k), load_c32(b, k, n), to_config(cfg), &log);
        std::memcpy(c, r.c.data.data(), sizeof(float) * 2 * static_cast<std::size_t>(m * n));
        res->kind = static_cast<int>(r.decision.kind);
        res->scale_a = r.decision.scale_exp_a;
        res->scale_b = r.decision.scale_exp_b;
        res->overflow = r.overflow;
        res->has_stats = r.stats_a.has_value();
        if (r.stats_a) res->stats_a = to_pod(*r.stats_a);
        if (r.stats_b) res->stats_b = to_pod(*r.stats_b);
        const std::string line = log.records().at(0).to_line();
        std::snprintf(res->line, sizeof(res->line), "%s", line.c_str());
        return 0;
    } catch (...) {
        return error_code();
    }
}

void ref_permute_c64(const float* src, float* dst, int rank, const std::int64_t* dims,
                     const int* axis_of) {
    std::vector<std::string> labels, order;
    std::vector<std::int64_t> d(dims, dims + rank);
    for (int a = 0; a < rank; ++a) labels.push_back("l" + std::to_string(a));
    for (int a = 0; a < rank; ++a) order.push_back("l" + std::to_string(axis_of[a]));
    TensorC32 t(labels, d);
    std::memcpy(t.data.data(), src, sizeof(float) * 2 * t.data.size());
    const TensorC32 p = permute(t, order);
    std::memcpy(dst, p.data.data(), sizeof(float) * 2 * p.data.size());
}

// experiments.cpp:27-31 random_uniform_matrix with Rng(seed)
void ref_rng_uniform_c32(std::uint64_t seed, std::int64_t rows, std::int64_t cols, float* out) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < rows * cols; ++i) {
        const std::complex<float> v{rng.uniform_pm1f(), rng.uniform_pm1f()};
        out[2 * i] = v.real();
        out[2 * i + 1] = v.imag();
    }
}

// run_gemm_bench operands (experiments.cpp:80-83): one Rng(seed), A then B
void ref_gemm_bench_operands(std::uint64_t seed, std::int64_t m, std::int64_t k, std::int64_t n,
                             float* a, float* b) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < m * k; ++i) {
        a[2 * i] = rng.uniform_pm1f();
        a[2 * i + 1] = rng.uniform_pm1f();
    }
    for (std::int64_t i = 0; i < k * n; ++i) {
        b[2 * i] = rng.uniform_pm1f();
        b[2 * i + 1] = rng.uniform_pm1f();
    }
}

// raw engine outputs / gaussian draws for pinning the generator
void ref_rng_stream(std::uint64_t seed, int kind, std::int64_t n, double* out) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < n; ++i) {
        switch (kind) {
        case 0: out[i] = static_cast<double>(rng.next_u64() >> 11); break;
        case 1: out[i] = static_cast<double>(rng.next_below(1000003)); break;
        case 2: out[i] = rng.gaussian(1e-2); break;
        default: out[i] = rng.uniform01(); break;
        }
    }
}

// ---------------------------------------------------------------- circuits

// save_circuit / save_network text of rqc_rectangular + circuit_to_network;
// returns the required size (including the NUL); copies when cap suffices.
std::int64_t ref_rqc_circuit_text(int rows, int cols, int depth, std::uint64_t seed, char* buf,
                                  std::int64_t cap) {
    std::ostringstream os;
    save_circuit(os, rqc_rectangular(rows, cols, depth, seed));
    const std::string s = os.str();
    if (static_cast<std::int64_t>(s.size()) + 1 <= cap) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<std::int64_t>(s.size()) + 1;
}

std::int64_t ref_rqc_network_text(int rows, int cols, int depth, std::uint64_t seed,
                                  const std::uint8_t* bits, char* buf, std::int64_t cap) {
    const Circuit c = rqc_rectangular(rows, cols, depth, seed);
    std::ostringstream os;
    save_network(os, circuit_to_network(c, bits_of(bits, c.n_qubits)));
    const std::string s = os.str();
    if (static_cast<std::int64_t>(s.size()) + 1 <= cap) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<std::int64_t>(s.size()) + 1;
}

// greedy path of the circuit network (bitstring-independent topology)
int ref_rqc_path(int rows, int cols, int depth, std::uint64_t seed, int* steps, int cap) {
    const Circuit c = rqc_rectangular(rows, cols, depth, seed);
    const Bitstring x(static_cast<std::size_t>(c.n_qubits), 0);
    const ContractionPath p = greedy_path(circuit_to_network(c, x));
    const int n = static_cast<int>(p.steps.size());
    for (int i = 0; i < n && 2 * i + 1 < cap; ++i) {
        steps[2 * i] = p.steps[static_cast<std::size_t>(i)].first;
        steps[2 * i + 1] = p.steps[static_cast<std::size_t>(i)].second;
    }
    return n;
}

// amplitude() with the given config; writes the decision-log lines (one per
// dispatched GEMM, '\n'-separated) when buf is non-null.
int ref_rqc_amplitude(int rows, int cols, int depth, std::uint64_t seed, const std::uint8_t* bits,
                      const ConfigPod* cfg, float* out, double* wall_ms, char* buf,
                      std::int64_t cap) {
    try {
        const Circuit c = rqc_rectangular(rows, cols, depth, seed);
        DecisionLog log;
        const auto t0 = std::chrono::steady_clock::now();
        const std::complex<float> z = amplitude(c, bits_of(bits, c.n_qubits), to_config(cfg), &log);
        if (wall_ms)
            *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                           .count();
        out[0] = z.real();
        out[1] = z.imag();
        if (buf && cap > 0) {
            std::string s;
            for (const auto& r : log.records()) s += r.to_line() + "\n";
            std::snprintf(buf, static_cast<std::size_t>(cap), "%s", s.c_str());
        }
        return 0;
    } catch (...) {
        return error_code();
    }
}

// run_rqc's inner loop (experiments.cpp:211-230): one greedy path for the
// circuit, then circuit_to_network + contract_network per bitstring, with the
// bitstrings spread over host threads (amplitudes are independent).
int ref_rqc_amplitudes_batch(int rows, int cols, int depth, std::uint64_t seed,
                             const std::uint8_t* bits, int n_strings, const ConfigPod* cfg,
                             float* out, int n_threads) {
    try {
        const Circuit c = rqc_rectangular(rows, cols, depth, seed);
        const int nq = c.n_qubits;
        const ContractionPath path = greedy_path(circuit_to_network(c, Bitstring(std::size_t(nq), 0)));
        const DispatchConfig dc = to_config(cfg);
        auto worker = [&](int t) {
            for (int i = t; i < n_strings; i += n_threads) {
                const TensorNetwork net = circuit_to_network(c, bits_of(bits + std::size_t(i) * nq, nq));
                const TensorC32 r = contract_network(net, path, dc, nullptr);
                out[2 * i] = r.data[0].real();
                out[2 * i + 1] = r.data[0].imag();
            }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < std::max(1, n_threads); ++t) pool.emplace_back(worker, t);
        for (auto& th : pool) th.join();
        return 0;
    } catch (...) {
        return error_code();
    }
}

// f64 TTGT pipeline on the same greedy path (network.cpp:179-186)
void ref_rqc_amplitude_tn_oracle(int rows, int cols, int depth, std::uint64_t seed,
                                 const std::uint8_t* bits, double* out) {
    const Circuit c = rqc_rectangular(rows, cols, depth, seed);
    const TensorNetwork net = circuit_to_network(c, bits_of(bits, c.n_qubits));
    const TensorC64 r = contract_network_oracle(net, greedy_path(net));
    out[0] = r.data[0].real();
    out[1] = r.data[0].imag();
}

// f64 state vector (qcircuit.cpp:197-235); <= 24 qubits
int ref_rqc_amplitude_sv_oracle(int rows, int cols, int depth, std::uint64_t seed,
                                const std::uint8_t* bits, double* out) {
    try {
        const Circuit c = rqc_rectangular(rows, cols, depth, seed);
        const std::complex<double> z = amplitude_oracle(c, bits_of(bits, c.n_qubits));
        out[0] = z.real();
        out[1] = z.imag();
        return 0;
    } catch (...) {
        return error_code();
    }
}

// ---------------------------------------------------- timed CPU baseline

// The reference's own cgemm (cgemm.cpp:25-46) with its GEMM row loop split
// across host threads.  kernels.hpp:16-19 allows row partitioning (k order is
// untouched), so the result is bit-identical to the single-threaded cgemm.
// Computes output rows [row_begin, row_end) of C (m x n) into c (row-local).
int ref_cgemm_rows_threaded_timed(const float* a, const float* b, float* c, std::int64_t m,
                                  std::int64_t n, std::int64_t k, std::int64_t row_begin,
                                  std::int64_t row_end, int mode, int k_tile, int n_threads,
                                  double* prep_s, double* gemm_s);

int ref_cgemm_rows_threaded(const float* a, const float* b, float* c, std::int64_t m,
                            std::int64_t n, std::int64_t k, std::int64_t row_begin,
                            std::int64_t row_end, int mode, int k_tile, int n_threads) {
    return ref_cgemm_rows_threaded_timed(a, b, c, m, n, k, row_begin, row_end, mode, k_tile,
                                         n_threads, nullptr, nullptr);
}

// Same, reporting the O(n^2) operand preparation (deinterleave + split/quantize of
// the B planes and the A rows) and the O(rows n k) GEMM wall times separately.
int ref_cgemm_rows_threaded_timed(const float* a, const float* b, float* c, std::int64_t m,
                                  std::int64_t n, std::int64_t k, std::int64_t row_begin,
                                  std::int64_t row_end, int mode, int k_tile, int n_threads,
                                  double* prep_s, double* gemm_s) {
    const auto t_start = std::chrono::steady_clock::now();
    const auto& kt = kernels::active_kernels();
    const std::int64_t rows = row_end - row_begin;
    (void)m;
    std::vector<float> are(static_cast<std::size_t>(rows * k)), aim(are.size());
    std::vector<float> bre(static_cast<std::size_t>(k * n)), bim(bre.size());
    for (std::int64_t i = 0; i < rows * k; ++i) {
        are[static_cast<std::size_t>(i)] = a[2 * (row_begin * k + i)];
        aim[static_cast<std::size_t>(i)] = a[2 * (row_begin * k + i) + 1];
    }
    for (std::int64_t i = 0; i < k * n; ++i) {
        bre[static_cast<std::size_t>(i)] = b[2 * i];
        bim[static_cast<std::size_t>(i)] = b[2 * i + 1];
    }
    const auto gm = static_cast<GemmMode>(mode);
    const bool corrected = mode_is_corrected(gm);
    const bool tc = gm == GemmMode::tf32_tc || gm == GemmMode::fp16_tc;
    bool ovf = false;
    // operand conversion (gemm.cpp:76-106), done once per plane
    std::vector<float> arh, arl, aih, ail, brh, brl, bih, bil;
    auto conv = [&](const std::vector<float>& src, std::vector<float>& h, std::vector<float>& l) {
        h.resize(src.size());
        if (corrected) {
            l.resize(src.size());
            kt.split_buf(src.data(), h.data(), l.data(), static_cast<std::int64_t>(src.size()),
                         mode_format(gm), &ovf);
        } else if (tc) {
            kt.quantize_buf(src.data(), h.data(), static_cast<std::int64_t>(src.size()),
                            mode_format(gm), lowprec::Rounding::nearest_even, &ovf);
        } else {
            h = src;
        }
    };
    conv(are, arh, arl);
    conv(aim, aih, ail);
    conv(bre, brh, brl);
    conv(bim, bih, bil);
    std::vector<float> p(static_cast<std::size_t>(4 * rows * n));
    const auto t_prep = std::chrono::steady_clock::now();
    float* p1 = p.data();
    float* p2 = p1 + rows * n;
    float* p3 = p2 + rows * n;
    float* p4 = p3 + rows * n;
    auto worker = [&](std::int64_t r0, std::int64_t r1) {
        auto run = [&](const std::vector<float>& ah, const std::vector<float>& al,
                       const std::vector<float>& bh, const std::vector<float>& bl, float* out) {
            if (corrected)
                kt.gemm_rows_tcec(ah.data(), al.data(), bh.data(), bl.data(), out, rows, n, k, k_tile,
                                  r0, r1);
            else if (tc)
                kt.gemm_rows_rz(ah.data(), bh.data(), out, rows, n, k, r0, r1);
            else
                kt.gemm_rows_rn(ah.data(), bh.data(), out, rows, n, k, r0, r1);
        };
        run(arh, arl, brh, brl, p1);
        run(aih, ail, bih, bil, p2);
        run(arh, arl, bih, bil, p3);
        run(aih, ail, brh, brl, p4);
    };
    std::vector<std::thread> pool;
    const int nt = std::max(1, n_threads);
    for (int t = 0; t < nt; ++t) {
        const std::int64_t r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
        if (r1 > r0) pool.emplace_back(worker, r0, r1);
    }
    for (auto& th : pool) th.join();
    const auto t_gemm = std::chrono::steady_clock::now();
    // complex assembly (cgemm.cpp:38-44)
    for (std::int64_t i = 0; i < rows * n; ++i) {
        c[2 * i] = p1[i] - p2[i];
        c[2 * i + 1] = p3[i] + p4[i];
    }
    if (prep_s) prep_s[0] = std::chrono::duration<double>(t_prep - t_start).count();
    if (gemm_s)
        gemm_s[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_prep).count();
    (void)t_gemm;
    return ovf ? 1 : 0;
}


// The reference's dispatch_cgemm (precsel.cpp:225-322) on the full operands,
// timed on a bounded row block: the selection half runs exactly as the
// reference runs it (exp_stats_staged on all of A and B, matrix_tolerance,
// select_mode, DecisionRecord::to_line -> *line), then the selected kind's
// CGEMM computes output rows [row_begin, row_end) with the reference kernels
// over n_threads (FP16TCEC_SCALED: scale_matrix of the A rows and of B by the
// selected shifts, FP16TCEC rows, descale -- precsel.cpp:209-216).  Times:
// t[0] statistics + selection, t[1] O(n^2) operand scaling/preparation,
// t[2] row GEMM.  Returns 0, or the error_code() of a thrown exception.
int ref_dispatch_rows_threaded_timed(const float* a, const float* b, float* c, std::int64_t m,
                                     std::int64_t n, std::int64_t k, std::int64_t row_begin,
                                     std::int64_t row_end, const ConfigPod* cfg, int n_threads,
                                     char* line, int line_cap, int* kind_out, double* t) {
    try {
        const DispatchConfig dc = to_config(cfg);
        const SelectionPolicy& pol = dc.policy;
        const int target = pol.target_max_exponent;
        const auto t0 = std::chrono::steady_clock::now();
        ComputeMode decision{ComputeKind::fp32_baseline, 0, 0};
        std::optional<ExpStats> sa, sb;
        std::string label;
        if (dc.force) throw std::invalid_argument("forced modes are not timed here");
        if (std::min({m, n, k}) >= pol.size_auto) {
            {
                const MatrixC32 ma = load_c32(a, m, k);
                sa = exp_stats_staged(ma, target, pol.threshold_t);
            }
            {
                const MatrixC32 mb = load_c32(b, k, n);
                sb = exp_stats_staged(mb, target, pol.threshold_t);
            }
            decision = select_mode(matrix_tolerance(*sa, pol.threshold_t, target),
                                   matrix_tolerance(*sb, pol.threshold_t, target), target);
        } else if (std::min({m, n, k}) >= pol.size_tf32) {
            decision = {ComputeKind::tf32_tcec, 0, 0};
        }
        label = to_string(decision.kind);
        DecisionRecord rec;
        rec.m = m;
        rec.n = n;
        rec.k = k;
        rec.mode = label;
        rec.scale_a = decision.scale_exp_a;
        rec.scale_b = decision.scale_exp_b;
        rec.stats_a = sa;
        rec.stats_b = sb;
        std::snprintf(line, static_cast<std::size_t>(line_cap), "%s", rec.to_line().c_str());
        *kind_out = static_cast<int>(decision.kind);
        const auto t1 = std::chrono::steady_clock::now();

        GemmMode gm = GemmMode::fp32_ref;
        switch (decision.kind) {
        case ComputeKind::fp16_tcec:
        case ComputeKind::fp16_tcec_scaled: gm = GemmMode::fp16_tcec; break;
        case ComputeKind::tf32_tcec: gm = GemmMode::tf32_tcec; break;
        default: break;
        }
        const std::int64_t rows = row_end - row_begin;
        const float* ap = a + 2 * row_begin * k;
        const float* bp = b;
        MatrixC32 a_s, b_s;
        if (decision.kind == ComputeKind::fp16_tcec_scaled) {
            a_s = scale_matrix(load_c32(ap, rows, k), decision.scale_exp_a);
            b_s = scale_matrix(load_c32(b, k, n), decision.scale_exp_b);
            ap = reinterpret_cast<const float*>(a_s.data.data());
            bp = reinterpret_cast<const float*>(b_s.data.data());
        }
        const auto t2 = std::chrono::steady_clock::now();
        double prep = 0.0, gemm = 0.0;
        ref_cgemm_rows_threaded_timed(ap, bp, c, rows, n, k, 0, rows, static_cast<int>(gm),
                                      dc.tiling.k_tile, n_threads, &prep, &gemm);
        const auto t3 = std::chrono::steady_clock::now();
        if (decision.kind == ComputeKind::fp16_tcec_scaled) {
            MatrixC32 cm = load_c32(c, rows, n);
            descale_output_inplace(cm, decision.scale_exp_a, decision.scale_exp_b);
            std::memcpy(c, cm.data.data(), sizeof(float) * 2 * static_cast<std::size_t>(rows * n));
        }
        const auto t4 = std::chrono::steady_clock::now();
        t[0] = std::chrono::duration<double>(t1 - t0).count();
        t[1] = std::chrono::duration<double>(t2 - t1).count() + prep +
               std::chrono::duration<double>(t4 - t3).count();
        t[2] = gemm;
        return 0;
    } catch (...) {
        return error_code();
    }
}

} // extern "C"
