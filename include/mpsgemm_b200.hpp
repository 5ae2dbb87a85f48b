// mpsgemm_b200.hpp -- C++ drop-in for the reference mpsgemm API
// (/root/reference/proj/include/mpsgemm/*.hpp), implemented over the C-ABI in
// tcec_b200.h (libtcec_b200.so: sm_100a kernels + the device-resident
// contraction engine).
//
// A reference user switches by putting include/ first on the include path --
// include/mpsgemm/{common,matrix,tensor,rng,lowprec,gemm,cgemm,precsel,network,
// qcircuit}.hpp forward here -- and linking libtcec_b200.so instead of
// libmpsgemm.a.  Namespace, type names, function names, argument meaning,
// value semantics (host std::vector storage in, host storage out) and the
// exception taxonomy (common.hpp:9-41) are the reference's; the reference's own
// test sources (tests/test_cgemm.cpp, test_precsel.cpp, test_tensor.cpp,
// test_qcircuit.cpp) compile against it unchanged (oracle/Makefile, target
// reftests).  Every computation runs on the GPU:
//
//   cgemm / cgemm_batched        cgemm.hpp:17-23      device TCEC / FP32 / FP64 tiers
//   cgemm_oracle                 cgemm.hpp:26         device f64 (bit-identical)
//   exp_stats[_staged]           precsel.hpp:68-72    device statistics
//   matrix_tolerance/select_mode precsel.hpp:74-77
//   scale/descale                precsel.hpp:82-91    device scaling
//   dispatch_cgemm x2            precsel.hpp:153-156  device selection + TCEC GEMM
//   permute                      tensor.hpp:56-57     device permute
//   contract_pair x2 / _oracle   network.hpp:29-35    device TTGT (f64 for _oracle)
//   contract_network / _oracle   network.hpp:37-39    device fold (CUDA graph)
//   greedy_path                  network.hpp:49
//   amplitude x2                 qcircuit.hpp:49-52   device fold
//   statevector/amplitude_oracle qcircuit.hpp:56-57   device f64 state vector
// Host-side (bookkeeping / workload definition, as in the reference):
// Matrix/Tensor containers, Rng, validate_network, random_network,
// save/load_network, the circuit generator and text format, relative_error.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <istream>
#include <map>
#include <mutex>
#include <numeric>
#include <optional>
#include <ostream>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "tcec_b200.h"

namespace mpsgemm {

// ------------------------------------------------------------------ errors (common.hpp)
struct ShapeMismatch : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ZeroReference : std::domain_error { using std::domain_error::domain_error; };
struct ScaleOverflow : std::range_error { using std::range_error::range_error; };
struct InvalidPermutation : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ExtentMismatch : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct InvalidPath : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct DisconnectedNetwork : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct InfeasibleDegrees : std::runtime_error { using std::runtime_error::runtime_error; };
struct TooManyQubits : std::invalid_argument { using std::invalid_argument::invalid_argument; };
// no reference counterpart: a CUDA / driver failure (there is no CPU fallback)
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void throw_status(int rc) {
    if (rc == TCEC_OK) return;
    const std::string msg = tcec_last_error();
    switch (rc) {
    case TCEC_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
    case TCEC_ERR_ZERO_REFERENCE: throw ZeroReference(msg);
    case TCEC_ERR_SCALE_OVERFLOW: throw ScaleOverflow(msg);
    case TCEC_ERR_INVALID_PERMUTATION: throw InvalidPermutation(msg);
    case TCEC_ERR_EXTENT_MISMATCH: throw ExtentMismatch(msg);
    case TCEC_ERR_INVALID_PATH: throw InvalidPath(msg);
    case TCEC_ERR_DISCONNECTED: throw DisconnectedNetwork(msg);
    case TCEC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case TCEC_ERR_LOGIC: throw std::logic_error(msg);
    case TCEC_ERR_TOO_MANY_QUBITS: throw TooManyQubits(msg);
    default: throw DeviceError(msg);
    }
}

// ------------------------------------------------------------------ matrix.hpp
template <typename T>
struct Matrix {
    std::int64_t rows = 0, cols = 0;
    std::vector<T> data;  // dense row-major
    Matrix() = default;
    Matrix(std::int64_t r, std::int64_t c) : rows(r), cols(c), data(std::size_t(r * c)) {}
    Matrix(std::int64_t r, std::int64_t c, std::vector<T> d) : rows(r), cols(c), data(std::move(d)) {
        if (std::int64_t(data.size()) != r * c) throw ShapeMismatch("matrix data length does not match rows*cols");
    }
    T& operator()(std::int64_t i, std::int64_t j) { return data[std::size_t(i * cols + j)]; }
    const T& operator()(std::int64_t i, std::int64_t j) const { return data[std::size_t(i * cols + j)]; }
    bool same_shape(const Matrix& o) const { return rows == o.rows && cols == o.cols; }
};
using MatrixF32 = Matrix<float>;
using MatrixF64 = Matrix<double>;
using MatrixC32 = Matrix<std::complex<float>>;
using MatrixC64 = Matrix<std::complex<double>>;

template <typename T>
Matrix<T> identity_matrix(std::int64_t n) {
    Matrix<T> m(n, n);
    for (std::int64_t i = 0; i < n; ++i) m(i, i) = T(1);
    return m;
}

// ------------------------------------------------------------------ rng.hpp
// The reference's deterministic source: std::mt19937_64 (specified by the
// standard) with its hand-rolled distribution maps, so seeds reproduce its
// workloads bit for bit (the same generator backs tcec_rng_*).
class Rng {
  public:
    explicit Rng(std::uint64_t seed) : eng_(seed) {}
    std::uint64_t next_u64() { return eng_(); }
    std::uint64_t next_below(std::uint64_t n) {
        const std::uint64_t cut = n * (UINT64_MAX / n);  // reject the biased tail
        std::uint64_t v;
        do v = eng_();
        while (v >= cut);
        return v % n;
    }
    double uniform01() { return double(eng_() >> 11) * 0x1.0p-53; }
    double uniform01_pos() { return double((eng_() >> 11) + 1) * 0x1.0p-53; }
    float uniform_pm1f() { return float(2.0 * uniform01() - 1.0); }
    double gaussian(double stddev) {
        if (cached_) {
            cached_ = false;
            return other_ * stddev;
        }
        const double u1 = uniform01_pos(), u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1)), t = 6.283185307179586476925286766559 * u2;
        other_ = r * std::sin(t);
        cached_ = true;
        return r * std::cos(t) * stddev;
    }

  private:
    std::mt19937_64 eng_;
    double other_ = 0.0;
    bool cached_ = false;
};

// ------------------------------------------------------------------ lowprec / gemm.hpp
namespace lowprec {
enum class Rounding { nearest_even, toward_zero };
enum class FormatKind : int { fp16 = 0, tf32 = 1 };
}  // namespace lowprec

enum class GemmMode { fp32_ref, fp64_oracle, tf32_tc, fp16_tc, tf32_tcec, fp16_tcec };
struct TilingConfig { int k_tile = 16; };

inline const char* to_string(GemmMode m) {
    static const char* const names[] = {"FP32_REF", "FP64_ORACLE", "TF32TC", "FP16TC", "TF32TCEC", "FP16TCEC"};
    const int i = int(m);
    return i >= 0 && i < 6 ? names[i] : "?";
}
inline GemmMode gemm_mode_from_string(const std::string& name) {
    for (int i = 0; i < 6; ++i)
        if (name == to_string(GemmMode(i))) return GemmMode(i);
    throw std::invalid_argument("unknown GEMM mode: " + name);
}
inline bool mode_is_corrected(GemmMode m) { return m == GemmMode::tf32_tcec || m == GemmMode::fp16_tcec; }
inline lowprec::FormatKind mode_format(GemmMode m) {
    if (m == GemmMode::tf32_tc || m == GemmMode::tf32_tcec) return lowprec::FormatKind::tf32;
    if (m == GemmMode::fp16_tc || m == GemmMode::fp16_tcec) return lowprec::FormatKind::fp16;
    throw std::invalid_argument("mode has no reduced-precision format");
}

// ------------------------------------------------------------------ precsel.hpp types
struct ExpStats {
    std::uint64_t n1 = 0, n2 = 0;
    std::optional<int> e_max;
    std::uint64_t n_nonzero = 0, n_total = 0;
    bool stage2_evaluated = false;
    double r1() const { return n_nonzero ? double(n_nonzero - n1) / double(n_nonzero) : 0.0; }
    double r2() const { return n_nonzero ? double(n_nonzero - n2) / double(n_nonzero) : 0.0; }
};
enum class ToleranceLevel { tf32_only = 0, fp16_scaled_ok = 1, fp16_ok = 2 };
struct MatrixTolerance { ToleranceLevel level = ToleranceLevel::tf32_only; std::optional<int> e_max; };
enum class ComputeKind { fp16_tcec, fp16_tcec_scaled, tf32_tcec, fp32_baseline };
inline const char* to_string(ComputeKind k) {
    static const char* const names[] = {"FP16TCEC", "FP16TCEC_SCALED", "TF32TCEC", "FP32_BASELINE"};
    const int i = int(k);
    return i >= 0 && i < 4 ? names[i] : "?";
}
struct ComputeMode { ComputeKind kind = ComputeKind::fp32_baseline; int scale_exp_a = 0, scale_exp_b = 0; };
struct SelectionPolicy {
    double threshold_t = 0.0;
    std::int64_t size_auto = 2048, size_tf32 = 512;
    int target_max_exponent = 14;
};
enum class ForcedMode { fp32_ref, fp64_oracle, tf32_tc, fp16_tc, tf32_tcec, fp16_tcec, fp16_tcec_scaled };
inline const char* to_string(ForcedMode f) {
    static const char* const names[] = {"FP32_REF", "FP64_ORACLE", "TF32TC", "FP16TC",
                                        "TF32TCEC", "FP16TCEC", "FP16TCEC_SCALED"};
    const int i = int(f);
    return i >= 0 && i < 7 ? names[i] : "?";
}
struct DispatchConfig { SelectionPolicy policy; TilingConfig tiling; std::optional<ForcedMode> force; };

struct DecisionRecord {
    std::int64_t m = 0, n = 0, k = 0;
    std::string mode;
    int scale_a = 0, scale_b = 0;
    std::optional<ExpStats> stats_a, stats_b;
    double wall_ms = 0.0;

    // m,n,k,mode,scale_a,scale_b,r1_a,r2_a,r1_b,r2_b,e_max_a,e_max_b with %.9g
    // ratios and "-" for absent values (precsel.cpp:185-205)
    std::string to_line() const {
        auto ratio = [](const std::optional<ExpStats>& s, bool second) {
            if (!s || (second && !s->stage2_evaluated)) return std::string("-");
            char b[32];
            std::snprintf(b, sizeof b, "%.9g", second ? s->r2() : s->r1());
            return std::string(b);
        };
        auto emax = [](const std::optional<ExpStats>& s) {
            return s && s->e_max ? std::to_string(*s->e_max) : std::string("-");
        };
        return std::to_string(m) + "," + std::to_string(n) + "," + std::to_string(k) + "," + mode + "," +
               std::to_string(scale_a) + "," + std::to_string(scale_b) + "," + ratio(stats_a, false) + "," +
               ratio(stats_a, true) + "," + ratio(stats_b, false) + "," + ratio(stats_b, true) + "," +
               emax(stats_a) + "," + emax(stats_b);
    }
};

class DecisionLog {
  public:
    void append(DecisionRecord r) { std::lock_guard<std::mutex> g(mu_); recs_.push_back(std::move(r)); }
    std::vector<DecisionRecord> records() const { std::lock_guard<std::mutex> g(mu_); return recs_; }
    void clear() { std::lock_guard<std::mutex> g(mu_); recs_.clear(); }

  private:
    mutable std::mutex mu_;
    std::vector<DecisionRecord> recs_;
};

struct DispatchResult {
    MatrixC32 c;
    ComputeMode decision;
    std::optional<ExpStats> stats_a, stats_b;
    bool overflow = false;
};

// ------------------------------------------------------------------ tensor.hpp
template <typename T>
struct Tensor {
    std::vector<std::string> labels;
    std::vector<std::int64_t> dims;
    std::vector<T> data;
    Tensor() : data(1) {}
    Tensor(std::vector<std::string> l, std::vector<std::int64_t> d) : labels(std::move(l)), dims(std::move(d)) {
        validate_shape();
        data.assign(std::size_t(size()), T{});
    }
    Tensor(std::vector<std::string> l, std::vector<std::int64_t> d, std::vector<T> v)
        : labels(std::move(l)), dims(std::move(d)), data(std::move(v)) {
        validate_shape();
        if (std::int64_t(data.size()) != size()) throw ShapeMismatch("tensor data length does not match dims");
    }
    int rank() const { return int(dims.size()); }
    std::int64_t size() const {
        std::int64_t s = 1;
        for (auto d : dims) s *= d;
        return s;
    }
    void validate_shape() const {
        if (labels.size() != dims.size()) throw ShapeMismatch("tensor labels and dims differ in length");
        for (auto d : dims)
            if (d < 1) throw ShapeMismatch("tensor extents must be >= 1");
        if (std::unordered_set<std::string>(labels.begin(), labels.end()).size() != labels.size())
            throw ShapeMismatch("tensor labels must be distinct");
    }
};
using TensorC32 = Tensor<std::complex<float>>;
using TensorC64 = Tensor<std::complex<double>>;

inline TensorC64 widen(const TensorC32& t) {
    TensorC64 w;
    w.labels = t.labels;
    w.dims = t.dims;
    w.data.assign(t.data.begin(), t.data.end());  // complex<float> -> complex<double> is exact
    return w;
}

struct TensorNetwork { std::vector<TensorC32> nodes; };
struct ContractionPath { std::vector<std::pair<int, int>> steps; };

// ------------------------------------------------------------------ device plumbing
namespace detail {

struct Context {
    tcec_handle h = nullptr;
    Context() { throw_status(tcec_create(0, &h)); }
    ~Context() { if (h) tcec_destroy(h); }
};

inline tcec_handle handle() {
    thread_local Context ctx;  // one handle per thread (the reference is reentrant, precsel.hpp:105-123)
    return ctx.h;
}

inline cudaStream_t stream() { return static_cast<cudaStream_t>(tcec_get_stream(handle())); }

struct DeviceBuffer {
    void* p = nullptr;
    explicit DeviceBuffer(std::size_t bytes) {
        if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) throw DeviceError("cudaMalloc failed");
    }
    ~DeviceBuffer() { if (p) cudaFree(p); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

// Copies run on the handle's own (non-blocking) stream, so they are ordered
// with the kernels the C-ABI enqueues there; download synchronises the stream
// before the host reads (a legacy-stream cudaMemcpy would not be ordered).
inline void upload(void* d, const void* h, std::size_t bytes) {
    if (bytes && cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream()) != cudaSuccess)
        throw DeviceError("H2D failed");
}
inline void download(void* h, const void* d, std::size_t bytes) {
    if (bytes && cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, stream()) != cudaSuccess)
        throw DeviceError("D2H failed");
    throw_status(tcec_synchronize(handle()));
}

inline tcec_dispatch_config_t to_c(const DispatchConfig& cfg) {
    tcec_dispatch_config_t c;
    tcec_default_config(&c);
    c.threshold_t = cfg.policy.threshold_t;
    c.size_auto = cfg.policy.size_auto;
    c.size_tf32 = cfg.policy.size_tf32;
    c.target_max_exponent = cfg.policy.target_max_exponent;
    c.k_tile = cfg.tiling.k_tile;
    c.force = cfg.force ? int(*cfg.force) : TCEC_FORCE_NONE;
    return c;
}

inline ExpStats from_c(const tcec_exp_stats_t& s) {
    ExpStats e;
    e.n1 = s.n1;
    e.n2 = s.n2;
    if (s.e_max_valid) e.e_max = s.e_max;
    e.n_nonzero = s.n_nonzero;
    e.n_total = s.n_total;
    e.stage2_evaluated = s.stage2_evaluated != 0;
    return e;
}

inline tcec_exp_stats_t to_c(const ExpStats& e) {
    tcec_exp_stats_t s{};
    s.n1 = e.n1;
    s.n2 = e.n2;
    s.e_max_valid = e.e_max.has_value();
    s.e_max = e.e_max.value_or(0);
    s.n_nonzero = e.n_nonzero;
    s.n_total = e.n_total;
    s.stage2_evaluated = e.stage2_evaluated;
    return s;
}

inline std::string field(const std::string& line, int idx) {
    std::size_t pos = 0;
    for (int i = 0; i < idx; ++i) pos = line.find(',', pos) + 1;
    return line.substr(pos, line.find(',', pos) - pos);
}

// DecisionRecord of one device dispatch (its log line carries m, n, k and the
// mode label; the result carries the shifts and the statistics)
inline DecisionRecord record_of(const tcec_dispatch_result_t& res) {
    const std::string ln = res.line;
    DecisionRecord r;
    r.m = std::stoll(field(ln, 0));
    r.n = std::stoll(field(ln, 1));
    r.k = std::stoll(field(ln, 2));
    r.mode = field(ln, 3);
    r.scale_a = res.scale_a;
    r.scale_b = res.scale_b;
    if (res.has_stats) {
        r.stats_a = from_c(res.stats_a);
        r.stats_b = from_c(res.stats_b);
    }
    return r;
}

// the per-step decisions of the network's last contraction, in step order
inline void append_log(DecisionLog* log, tcec_network net, int n_steps) {
    if (!log || n_steps <= 0) return;
    std::vector<tcec_dispatch_result_t> res(static_cast<std::size_t>(n_steps));
    int count = 0;
    throw_status(tcec_network_step_results(net, res.data(), n_steps, &count));
    for (int i = 0; i < count; ++i) log->append(record_of(res[std::size_t(i)]));
}

}  // namespace detail

// ------------------------------------------------------------------ cgemm.hpp
inline MatrixC32 cgemm(const MatrixC32& a, const MatrixC32& b, GemmMode mode, const TilingConfig& tiling = {},
                       bool* overflow = nullptr) {
    if (a.cols != b.rows) throw ShapeMismatch("cgemm: inner dimensions differ");
    detail::DeviceBuffer da(a.data.size() * 8), db(b.data.size() * 8), dc(std::size_t(a.rows * b.cols) * 8);
    detail::upload(da.p, a.data.data(), a.data.size() * 8);
    detail::upload(db.p, b.data.data(), b.data.size() * 8);
    int ovf = 0;
    throw_status(tcec_cgemm(detail::handle(), da.p, db.p, dc.p, a.rows, b.cols, a.cols, int(mode), tiling.k_tile,
                            &ovf));
    MatrixC32 c(a.rows, b.cols);
    detail::download(c.data.data(), dc.p, c.data.size() * 8);
    if (overflow && ovf) *overflow = true;
    return c;
}

inline std::vector<MatrixC32> cgemm_batched(const std::vector<std::pair<MatrixC32, MatrixC32>>& pairs,
                                            GemmMode mode, const TilingConfig& tiling = {},
                                            bool* overflow = nullptr) {
    std::vector<MatrixC32> out;
    out.reserve(pairs.size());
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        try {
            out.push_back(cgemm(pairs[i].first, pairs[i].second, mode, tiling, overflow));
        } catch (const ShapeMismatch& e) {
            throw ShapeMismatch("batch entry " + std::to_string(i) + ": " + e.what());
        }
    }
    return out;
}

// full-f64 complex product (device, bit-identical to the reference's)
inline MatrixC64 cgemm_oracle(const MatrixC32& a, const MatrixC32& b) {
    if (a.cols != b.rows) throw ShapeMismatch("cgemm_oracle: inner dimensions differ");
    detail::DeviceBuffer da(a.data.size() * 8), db(b.data.size() * 8), dc(std::size_t(a.rows * b.cols) * 16);
    detail::upload(da.p, a.data.data(), a.data.size() * 8);
    detail::upload(db.p, b.data.data(), b.data.size() * 8);
    throw_status(tcec_cgemm_oracle(detail::handle(), da.p, db.p, dc.p, a.rows, b.cols, a.cols));
    MatrixC64 c(a.rows, b.cols);
    detail::download(c.data.data(), dc.p, c.data.size() * 16);
    return c;
}

// ||C - C_ref||_F / ||C_ref||_F in f64 (a host reduction of two host matrices,
// as in the reference, cgemm.cpp:76-89)
inline double relative_error(const MatrixC32& c, const MatrixC64& c_ref) {
    if (!(c.rows == c_ref.rows && c.cols == c_ref.cols)) throw ShapeMismatch("relative_error: shape mismatch");
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < c.data.size(); ++i) {
        const std::complex<double> r = c_ref.data[i];
        const double dr = double(c.data[i].real()) - r.real(), di = double(c.data[i].imag()) - r.imag();
        num += dr * dr + di * di;
        den += r.real() * r.real() + r.imag() * r.imag();
    }
    if (den == 0.0) throw ZeroReference("relative_error: zero reference norm");
    return std::sqrt(num) / std::sqrt(den);
}

// ------------------------------------------------------------------ precsel.hpp
inline ExpStats exp_stats_impl(const MatrixC32& m, int target, int staged, double t) {
    detail::DeviceBuffer d(m.data.size() * 8);
    detail::upload(d.p, m.data.data(), m.data.size() * 8);
    tcec_exp_stats_t s;
    throw_status(tcec_exp_stats(detail::handle(), d.p, m.rows, m.cols, target, staged, t, &s));
    return detail::from_c(s);
}
inline ExpStats exp_stats(const MatrixC32& m, int target_max_exponent = 14) {
    return exp_stats_impl(m, target_max_exponent, 0, 0.0);
}
inline ExpStats exp_stats_staged(const MatrixC32& m, int target_max_exponent, double t) {
    return exp_stats_impl(m, target_max_exponent, 1, t);
}

inline MatrixTolerance matrix_tolerance(const ExpStats& stats, double t, int target_max_exponent = 14) {
    const tcec_exp_stats_t s = detail::to_c(stats);
    int level = 0;
    throw_status(tcec_matrix_tolerance(&s, t, target_max_exponent, &level));
    return {ToleranceLevel(level), stats.e_max};
}

inline ComputeMode select_mode(const MatrixTolerance& a, const MatrixTolerance& b, int target_max_exponent = 14) {
    int kind = 0, sa = 0, sb = 0;
    throw_status(tcec_select_mode(int(a.level), a.e_max.has_value(), a.e_max.value_or(0), int(b.level),
                                  b.e_max.has_value(), b.e_max.value_or(0), target_max_exponent, &kind, &sa, &sb));
    return {ComputeKind(kind), sa, sb};
}

namespace detail {
template <typename M>
inline void scale_components(M& m, int scale_exp, bool check) {
    const std::size_t bytes = m.data.size() * sizeof(m.data[0]);
    DeviceBuffer d(bytes);
    upload(d.p, m.data.data(), bytes);
    throw_status(tcec_scale_components(handle(), static_cast<float*>(d.p), std::int64_t(bytes / 4), scale_exp,
                                       check ? 1 : 0));
    download(m.data.data(), d.p, bytes);
}
}  // namespace detail

inline void scale_matrix_inplace(MatrixC32& m, int s) { detail::scale_components(m, s, true); }
inline void scale_matrix_inplace(MatrixF32& m, int s) { detail::scale_components(m, s, true); }
inline MatrixC32 scale_matrix(const MatrixC32& m, int s) { MatrixC32 o = m; scale_matrix_inplace(o, s); return o; }
inline MatrixF32 scale_matrix(const MatrixF32& m, int s) { MatrixF32 o = m; scale_matrix_inplace(o, s); return o; }
inline void descale_output_inplace(MatrixC32& c, int sa, int sb) { detail::scale_components(c, -(sa + sb), false); }
inline void descale_output_inplace(MatrixF32& c, int sa, int sb) { detail::scale_components(c, -(sa + sb), false); }
inline MatrixC32 descale_output(const MatrixC32& c, int sa, int sb) {
    MatrixC32 o = c;
    descale_output_inplace(o, sa, sb);
    return o;
}

inline DispatchResult dispatch_cgemm(const MatrixC32& a, const MatrixC32& b, const DispatchConfig& config,
                                     DecisionLog* log = nullptr) {
    if (a.cols != b.rows) throw ShapeMismatch("dispatch_cgemm: inner dimensions differ");
    const tcec_dispatch_config_t cfg = detail::to_c(config);
    DispatchResult r;
    r.c = MatrixC32(a.rows, b.cols);
    tcec_dispatch_result_t res;
    throw_status(tcec_dispatch_cgemm_host(detail::handle(), a.data.data(), b.data.data(), r.c.data.data(), a.rows,
                                          b.cols, a.cols, &cfg, &res));
    r.decision = {ComputeKind(res.kind), res.scale_a, res.scale_b};
    if (res.has_stats) {
        r.stats_a = detail::from_c(res.stats_a);
        r.stats_b = detail::from_c(res.stats_b);
    }
    r.overflow = res.overflow != 0;
    if (log) log->append(detail::record_of(res));
    return r;
}

inline DispatchResult dispatch_cgemm(const MatrixC32& a, const MatrixC32& b, const SelectionPolicy& policy,
                                     DecisionLog* log = nullptr) {
    return dispatch_cgemm(a, b, DispatchConfig{policy, TilingConfig{}, std::nullopt}, log);
}

// ------------------------------------------------------------------ permute (tensor.hpp)
template <typename T>
inline Tensor<T> permute(const Tensor<T>& t, const std::vector<std::string>& new_order) {
    static_assert(sizeof(T) == 8 || sizeof(T) == 16, "device permute is for complex<float> / complex<double>");
    const int r = t.rank();
    if (int(new_order.size()) != r) throw InvalidPermutation("permutation has wrong length");
    std::vector<int> axis_of(std::size_t(r) + 1);
    std::vector<bool> used(std::size_t(r), false);
    for (int a = 0; a < r; ++a) {
        int found = -1;
        for (int o = 0; o < r && found < 0; ++o)
            if (!used[std::size_t(o)] && t.labels[std::size_t(o)] == new_order[std::size_t(a)]) found = o;
        if (found < 0) throw InvalidPermutation("label not in tensor: " + new_order[std::size_t(a)]);
        used[std::size_t(found)] = true;
        axis_of[std::size_t(a)] = found;
    }
    Tensor<T> out;
    out.labels = new_order;
    for (int a = 0; a < r; ++a) out.dims.push_back(t.dims[std::size_t(axis_of[std::size_t(a)])]);
    out.data.resize(t.data.size());
    const std::size_t bytes = t.data.size() * sizeof(T);
    detail::DeviceBuffer ds(bytes), dd(bytes);
    detail::upload(ds.p, t.data.data(), bytes);
    std::vector<std::int64_t> dims(t.dims);
    dims.push_back(1);
    if (sizeof(T) == 8)
        throw_status(tcec_permute(detail::handle(), ds.p, dd.p, r, dims.data(), axis_of.data()));
    else
        throw_status(tcec_permute_c128(detail::handle(), ds.p, dd.p, r, dims.data(), axis_of.data()));
    detail::download(out.data.data(), dd.p, bytes);
    return out;
}

// ------------------------------------------------------------------ network.hpp
// validate_network (network.cpp:114-127): every label in at most two nodes,
// with one extent
inline void validate_network(const TensorNetwork& net) {
    std::map<std::string, std::vector<std::int64_t>> seen;
    for (const auto& t : net.nodes) {
        t.validate_shape();
        for (int a = 0; a < t.rank(); ++a) seen[t.labels[std::size_t(a)]].push_back(t.dims[std::size_t(a)]);
    }
    for (const auto& [label, ext] : seen) {
        if (ext.size() > 2) throw ShapeMismatch("label " + label + " appears in more than two nodes");
        if (ext.size() == 2 && ext[0] != ext[1]) throw ExtentMismatch("label " + label + " has mismatched extents");
    }
}

namespace detail {

// A network registered with the C-ABI: labels interned as ints, node data
// staged for the device (with_device) or shapes only (path planning).
struct NetworkHandle {
    tcec_network net = nullptr;
    std::map<std::string, int> ids;
    std::vector<std::string> names;
    NetworkHandle(const TensorNetwork& tn, bool with_device) {
        std::vector<int> ranks, labels;
        std::vector<std::int64_t> dims;
        for (const auto& t : tn.nodes) {
            ranks.push_back(t.rank());
            for (int a = 0; a < t.rank(); ++a) {
                auto it = ids.find(t.labels[std::size_t(a)]);
                if (it == ids.end()) {
                    it = ids.emplace(t.labels[std::size_t(a)], int(names.size())).first;
                    names.push_back(t.labels[std::size_t(a)]);
                }
                labels.push_back(it->second);
                dims.push_back(t.dims[std::size_t(a)]);
            }
        }
        ranks.push_back(0);
        labels.push_back(0);
        dims.push_back(1);
        throw_status(tcec_network_create(with_device ? handle() : nullptr, int(tn.nodes.size()), ranks.data(),
                                         labels.data(), dims.data(), &net));
        if (with_device)
            for (std::size_t i = 0; i < tn.nodes.size(); ++i)
                throw_status(tcec_network_set_node(net, int(i), tn.nodes[i].data.data()));
    }
    ~NetworkHandle() { if (net) tcec_network_destroy(net); }
    NetworkHandle(const NetworkHandle&) = delete;
    NetworkHandle& operator=(const NetworkHandle&) = delete;
};

inline std::vector<int> flat_steps(const ContractionPath& path) {
    std::vector<int> s;
    for (const auto& [a, b] : path.steps) {
        s.push_back(a);
        s.push_back(b);
    }
    s.push_back(0);  // never empty (the count is passed separately)
    return s;
}

// extents of every label; the open labels bound the result size
inline std::int64_t open_size(const TensorNetwork& net, std::map<std::string, std::int64_t>* ext) {
    std::map<std::string, int> count;
    for (const auto& t : net.nodes)
        for (int a = 0; a < t.rank(); ++a) {
            ++count[t.labels[std::size_t(a)]];
            (*ext)[t.labels[std::size_t(a)]] = t.dims[std::size_t(a)];
        }
    std::int64_t cap = 1;
    for (const auto& [l, c] : count)
        if (c == 1) cap *= (*ext)[l];
    return std::max<std::int64_t>(cap, 1);
}

template <typename T>
inline Tensor<T> result_tensor(const NetworkHandle& nh, const std::map<std::string, std::int64_t>& ext,
                               const std::vector<int>& labels, int rank, const std::vector<T>& out) {
    Tensor<T> r;
    for (int i = 0; i < rank; ++i) {
        r.labels.push_back(nh.names[std::size_t(labels[std::size_t(i)])]);
        r.dims.push_back(ext.at(r.labels.back()));
    }
    r.data.assign(out.begin(), out.begin() + r.size());
    return r;
}

}  // namespace detail

inline ContractionPath greedy_path(const TensorNetwork& net) {
    validate_network(net);
    if (net.nodes.empty()) throw InvalidPath("empty network");
    detail::NetworkHandle nh(net, false);
    std::vector<int> steps(2 * net.nodes.size());
    throw_status(tcec_network_greedy_path(nh.net, steps.data()));
    ContractionPath p;
    for (std::size_t i = 0; i + 1 < net.nodes.size(); ++i) p.steps.emplace_back(steps[2 * i], steps[2 * i + 1]);
    return p;
}

inline TensorC32 contract_network(const TensorNetwork& net, const ContractionPath& path,
                                  const DispatchConfig& config, DecisionLog* log = nullptr) {
    if (net.nodes.empty()) throw InvalidPath("empty network");
    detail::NetworkHandle nh(net, true);
    const std::vector<int> steps = detail::flat_steps(path);
    std::map<std::string, std::int64_t> ext;
    std::vector<std::complex<float>> out(std::size_t(detail::open_size(net, &ext)));
    std::vector<int> labels(ext.size() + 1);
    int rank = 0;
    const tcec_dispatch_config_t cfg = detail::to_c(config);
    throw_status(tcec_contract_network(nh.net, steps.data(), int(path.steps.size()), &cfg, out.data(),
                                       std::int64_t(out.size()), &rank, labels.data(), nullptr, 0));
    detail::append_log(log, nh.net, int(path.steps.size()));
    return detail::result_tensor(nh, ext, labels, rank, out);
}

// contract_network_oracle (network.cpp:179-186): the f64 fold, on the device
inline TensorC64 contract_network_oracle(const TensorNetwork& net, const ContractionPath& path) {
    if (net.nodes.empty()) throw InvalidPath("empty network");
    detail::NetworkHandle nh(net, true);
    const std::vector<int> steps = detail::flat_steps(path);
    std::map<std::string, std::int64_t> ext;
    std::vector<std::complex<double>> out(std::size_t(detail::open_size(net, &ext)));
    std::vector<int> labels(ext.size() + 1);
    int rank = 0;
    throw_status(tcec_contract_network_oracle(nh.net, steps.data(), int(path.steps.size()), out.data(),
                                              std::int64_t(out.size()), &rank, labels.data()));
    return detail::result_tensor(nh, ext, labels, rank, out);
}

inline TensorC32 contract_pair(const TensorC32& a, const TensorC32& b, const DispatchConfig& config,
                               DecisionLog* log = nullptr) {
    return contract_network(TensorNetwork{{a, b}}, ContractionPath{{{0, 1}}}, config, log);
}
inline TensorC32 contract_pair(const TensorC32& a, const TensorC32& b, const SelectionPolicy& policy,
                               DecisionLog* log = nullptr) {
    return contract_pair(a, b, DispatchConfig{policy, TilingConfig{}, std::nullopt}, log);
}

// contract_pair_oracle (network.hpp:35): f64 TTGT of two complex128 tensors
inline TensorC64 contract_pair_oracle(const TensorC64& a, const TensorC64& b) {
    // split_pair: free_a | shared (a's order) | free_b
    std::vector<std::string> fa, sh, fb;
    std::vector<std::int64_t> fad, shd, fbd;
    for (int i = 0; i < a.rank(); ++i) {
        const auto& l = a.labels[std::size_t(i)];
        const auto it = std::find(b.labels.begin(), b.labels.end(), l);
        if (it == b.labels.end()) {
            fa.push_back(l);
            fad.push_back(a.dims[std::size_t(i)]);
            continue;
        }
        const std::int64_t bd = b.dims[std::size_t(it - b.labels.begin())];
        if (bd != a.dims[std::size_t(i)])
            throw ExtentMismatch("label " + l + " has extents " + std::to_string(a.dims[std::size_t(i)]) + " and " +
                                 std::to_string(bd));
        sh.push_back(l);
        shd.push_back(bd);
    }
    for (int i = 0; i < b.rank(); ++i)
        if (std::find(a.labels.begin(), a.labels.end(), b.labels[std::size_t(i)]) == a.labels.end()) {
            fb.push_back(b.labels[std::size_t(i)]);
            fbd.push_back(b.dims[std::size_t(i)]);
        }
    std::vector<std::string> oa = fa, ob = sh;
    oa.insert(oa.end(), sh.begin(), sh.end());
    ob.insert(ob.end(), fb.begin(), fb.end());
    const TensorC64 pa = permute(a, oa), pb = permute(b, ob);
    auto prod = [](const std::vector<std::int64_t>& v) {
        return std::accumulate(v.begin(), v.end(), std::int64_t{1}, std::multiplies<std::int64_t>());
    };
    const std::int64_t m = prod(fad), k = prod(shd), n = prod(fbd);
    detail::DeviceBuffer da(pa.data.size() * 16), db(pb.data.size() * 16), dc(std::size_t(m * n) * 16);
    detail::upload(da.p, pa.data.data(), pa.data.size() * 16);
    detail::upload(db.p, pb.data.data(), pb.data.size() * 16);
    throw_status(tcec_cgemm_c128(detail::handle(), da.p, db.p, dc.p, m, n, k));
    TensorC64 out;
    out.labels = fa;
    out.labels.insert(out.labels.end(), fb.begin(), fb.end());
    out.dims = fad;
    out.dims.insert(out.dims.end(), fbd.begin(), fbd.end());
    out.data.resize(std::size_t(m * n));
    detail::download(out.data.data(), dc.p, out.data.size() * 16);
    return out;
}

// random_network (network.cpp:328-438): the reference's seeded generator of
// closed random networks for the selection experiments (workload definition)
enum class RandtnInit { type1 = 1, type2 = 2, type3 = 3 };
struct RandomNetworkParams {
    int n_nodes = 10;
    int min_degree = 2;
    int max_degree = 4;
    std::int64_t dim = 32;
    RandtnInit init = RandtnInit::type1;
};

inline TensorNetwork random_network(const RandomNetworkParams& params, std::uint64_t seed) {
    if (params.n_nodes < 2 || params.min_degree < 1 || params.max_degree < params.min_degree || params.dim < 2)
        throw InfeasibleDegrees("invalid random network parameters");
    const int n = params.n_nodes;
    for (int attempt = 0; attempt < 500; ++attempt) {
        Rng rng(seed + 0x9E3779B97F4A7C15ull * std::uint64_t(attempt));
        // a degree sequence with an even sum (64 draws at most)
        std::vector<int> deg(static_cast<std::size_t>(n));
        bool even = false;
        for (int tries = 0; tries < 64 && !even; ++tries) {
            int sum = 0;
            for (auto& d : deg) {
                d = params.min_degree + int(rng.next_below(std::uint64_t(params.max_degree - params.min_degree + 1)));
                sum += d;
            }
            even = sum % 2 == 0;
        }
        if (!even) continue;
        // configuration model: Fisher-Yates over the stub list, consecutive pairs are edges
        std::vector<int> stub;
        for (int i = 0; i < n; ++i) stub.insert(stub.end(), std::size_t(deg[std::size_t(i)]), i);
        for (std::size_t i = stub.size() - 1; i > 0; --i) std::swap(stub[i], stub[rng.next_below(i + 1)]);
        std::vector<std::pair<int, int>> edges;
        bool loop = false;
        for (std::size_t i = 0; i + 1 < stub.size() && !loop; i += 2) {
            loop = stub[i] == stub[i + 1];
            if (!loop) edges.emplace_back(stub[i], stub[i + 1]);
        }
        if (loop) continue;
        // connectivity (union-find with path halving)
        std::vector<int> root(static_cast<std::size_t>(n));
        std::iota(root.begin(), root.end(), 0);
        auto find = [&](int x) {
            while (root[std::size_t(x)] != x) x = root[std::size_t(x)] = root[std::size_t(root[std::size_t(x)])];
            return x;
        };
        for (const auto& [x, y] : edges) root[std::size_t(find(x))] = find(y);
        bool connected = true;
        for (int i = 1; i < n && connected; ++i) connected = find(i) == find(0);
        if (!connected) continue;
        // shapes: edge e is label "e<e>" on both endpoints, in edge order
        TensorNetwork shape;
        std::vector<std::vector<std::string>> lab(static_cast<std::size_t>(n));
        std::vector<std::vector<std::int64_t>> dim(static_cast<std::size_t>(n));
        for (std::size_t e = 0; e < edges.size(); ++e)
            for (int node : {edges[e].first, edges[e].second}) {
                lab[std::size_t(node)].push_back("e" + std::to_string(e));
                dim[std::size_t(node)].push_back(params.dim);
            }
        for (int i = 0; i < n; ++i) {
            TensorC32 t;
            t.labels = lab[std::size_t(i)];
            t.dims = dim[std::size_t(i)];
            shape.nodes.push_back(std::move(t));
        }
        // vet the greedy contraction: a statistics-gated step (min(m,n,k) >= dim^2)
        // and no intermediate above rank 4
        const ContractionPath path = greedy_path(shape);
        const std::int64_t gate = params.dim * params.dim, cap = gate * gate;
        bool gated = false;
        std::int64_t widest = 0;
        {
            std::map<int, std::pair<std::vector<std::string>, std::vector<std::int64_t>>> live;
            for (int i = 0; i < n; ++i) live[i] = {lab[std::size_t(i)], dim[std::size_t(i)]};
            int next = n;
            for (const auto& [ia, ib] : path.steps) {
                auto A = live[ia], B = live[ib];
                std::int64_t m = 1, k = 1, nn = 1;
                std::pair<std::vector<std::string>, std::vector<std::int64_t>> r;
                for (std::size_t i = 0; i < A.first.size(); ++i) {
                    if (std::find(B.first.begin(), B.first.end(), A.first[i]) != B.first.end()) {
                        k *= A.second[i];
                    } else {
                        m *= A.second[i];
                        r.first.push_back(A.first[i]);
                        r.second.push_back(A.second[i]);
                    }
                }
                for (std::size_t i = 0; i < B.first.size(); ++i)
                    if (std::find(A.first.begin(), A.first.end(), B.first[i]) == A.first.end()) {
                        nn *= B.second[i];
                        r.first.push_back(B.first[i]);
                        r.second.push_back(B.second[i]);
                    }
                gated = gated || std::min({m, nn, k}) >= gate;
                widest = std::max(widest, m * nn);
                live.erase(ia);
                live.erase(ib);
                live[next++] = std::move(r);
            }
        }
        if (!gated || widest > cap) continue;
        // element values: N(0, 1e-2) per component, x1e-6 for types 2 and 3
        TensorNetwork net;
        for (int i = 0; i < n; ++i) net.nodes.emplace_back(lab[std::size_t(i)], dim[std::size_t(i)]);
        const bool tiny = params.init != RandtnInit::type1;
        for (auto& node : net.nodes)
            for (auto& v : node.data) {
                float re = float(rng.gaussian(1e-2)), im = float(rng.gaussian(1e-2));
                if (tiny) {
                    re *= 1e-6f;
                    im *= 1e-6f;
                }
                v = {re, im};
            }
        if (params.init == RandtnInit::type3) {
            // 10..20 distinct flat positions set to exactly 1 + 0i
            std::int64_t total = 0;
            for (const auto& node : net.nodes) total += node.size();
            const int want = 10 + int(rng.next_below(11));
            std::vector<std::int64_t> pos;
            while (int(pos.size()) < want) {
                const std::int64_t f = std::int64_t(rng.next_below(std::uint64_t(total)));
                if (std::find(pos.begin(), pos.end(), f) == pos.end()) pos.push_back(f);
            }
            for (std::int64_t f : pos)
                for (auto& node : net.nodes) {
                    if (f < node.size()) {
                        node.data[std::size_t(f)] = {1.0f, 0.0f};
                        break;
                    }
                    f -= node.size();
                }
        }
        return net;
    }
    throw InfeasibleDegrees("no suitable random multigraph found for the given parameters");
}

// Text serialization (network.cpp:440-501): per node the header line
// "node <id> labels l1,l2 dims d1,d2" ("-" for rank 0), then the values as
// "%.9g %.9g" pairs (exact round trip for f32).
inline void save_network(std::ostream& os, const TensorNetwork& net) {
    auto csv = [](const auto& v) {
        std::string s;
        for (std::size_t i = 0; i < v.size(); ++i) {
            if (i) s += ",";
            if constexpr (std::is_same_v<std::decay_t<decltype(v[i])>, std::string>)
                s += v[i];
            else
                s += std::to_string(v[i]);
        }
        return s.empty() ? std::string("-") : s;
    };
    for (std::size_t i = 0; i < net.nodes.size(); ++i) {
        const auto& t = net.nodes[i];
        os << "node " << i << " labels " << csv(t.labels) << " dims " << csv(t.dims) << "\n";
        char buf[64];
        for (std::size_t v = 0; v < t.data.size(); ++v) {
            std::snprintf(buf, sizeof buf, "%.9g %.9g", double(t.data[v].real()), double(t.data[v].imag()));
            os << buf << (v + 1 == t.data.size() ? "\n" : " ");
        }
    }
}

inline TensorNetwork load_network(std::istream& is) {
    auto split = [](const std::string& s) {
        std::vector<std::string> out;
        if (s == "-") return out;
        std::size_t b = 0;
        while (true) {
            const std::size_t e = s.find(',', b);
            out.push_back(s.substr(b, e - b));
            if (e == std::string::npos) break;
            b = e + 1;
        }
        return out;
    };
    TensorNetwork net;
    std::string tok;
    while (is >> tok) {
        if (tok != "node") throw ShapeMismatch("expected 'node' header, got: " + tok);
        int id = 0;
        std::string kl, lcsv, kd, dcsv;
        if (!(is >> id >> kl >> lcsv >> kd >> dcsv) || kl != "labels" || kd != "dims")
            throw ShapeMismatch("malformed node header");
        std::vector<std::int64_t> dims;
        for (const auto& d : split(dcsv)) dims.push_back(std::stoll(d));
        TensorC32 t(split(lcsv), dims);
        for (auto& v : t.data) {
            double re, im;
            if (!(is >> re >> im)) throw ShapeMismatch("truncated tensor data");
            v = {float(re), float(im)};
        }
        net.nodes.push_back(std::move(t));
    }
    validate_network(net);
    return net;
}

// ------------------------------------------------------------------ qcircuit.hpp
enum class GateKind { h, t, sqrt_x, sqrt_y, cz };
inline const char* to_string(GateKind k) {
    static const char* const names[] = {"H", "T", "SX", "SY", "CZ"};
    const int i = int(k);
    return i >= 0 && i < 5 ? names[i] : "?";
}
struct Gate {
    GateKind kind;
    std::vector<int> qubits;
};
struct Circuit {
    int n_qubits = 0;
    std::vector<std::vector<Gate>> layers;
};
using Bitstring = std::vector<std::uint8_t>;

inline void validate_circuit(const Circuit& c) {
    for (const auto& layer : c.layers) {
        std::set<int> used;
        for (const auto& g : layer) {
            if (g.qubits.size() != (g.kind == GateKind::cz ? 2u : 1u)) throw ShapeMismatch("gate has wrong qubit count");
            for (int q : g.qubits) {
                if (q < 0 || q >= c.n_qubits) throw ShapeMismatch("qubit index out of range");
                if (!used.insert(q).second) throw ShapeMismatch("layer gates must act on disjoint qubits");
            }
        }
    }
}

// defining unitaries in f64, row-major (qcircuit.cpp:47-61)
inline std::vector<std::complex<double>> gate_matrix_f64(GateKind k) {
    using cd = std::complex<double>;
    const double r = 1.0 / std::sqrt(2.0);
    switch (k) {
    case GateKind::h: return {r, r, r, -r};
    case GateKind::t: return {1.0, 0.0, 0.0, cd(r, r)};
    case GateKind::sqrt_x: return {cd(0.5, 0.5), cd(0.5, -0.5), cd(0.5, -0.5), cd(0.5, 0.5)};
    case GateKind::sqrt_y: return {cd(0.5, 0.5), cd(-0.5, -0.5), cd(0.5, 0.5), cd(0.5, 0.5)};
    case GateKind::cz: return {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, -1};
    }
    return {};
}

// gate as a labeled tensor (out..., in...) with placeholder labels
inline TensorC32 gate_tensor(const Gate& g) {
    const auto u = gate_matrix_f64(g.kind);
    TensorC32 t = g.kind == GateKind::cz ? TensorC32({"o0", "o1", "i0", "i1"}, {2, 2, 2, 2})
                                         : TensorC32({"o0", "i0"}, {2, 2});
    for (std::size_t i = 0; i < u.size(); ++i) t.data[i] = {float(u[i].real()), float(u[i].imag())};
    return t;
}

// CZ pairs of mid-layer `layer_index`: eight staggered pairings H0 V0 H1 V1 ... V3
inline std::vector<std::pair<int, int>> cz_pattern(int rows, int cols, int layer_index) {
    const int p = layer_index % 8, phase = p / 2;
    std::vector<std::pair<int, int>> out;
    if (p % 2 == 0) {
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c + 1 < cols; ++c)
                if ((c + 2 * (r % 2)) % 4 == phase) out.emplace_back(r * cols + c, r * cols + c + 1);
    } else {
        for (int r = 0; r + 1 < rows; ++r)
            for (int c = 0; c < cols; ++c)
                if ((r + 2 * (c % 2)) % 4 == phase) out.emplace_back(r * cols + c, (r + 1) * cols + c);
    }
    return out;
}

// rectangular-lattice random circuit (qcircuit.cpp:102-140): H layer, mid_depth
// CZ layers (uncovered qubits draw T / SX / SY, never repeating their last),
// closing H layer
inline Circuit rqc_rectangular(int rows, int cols, int mid_depth, std::uint64_t seed) {
    if (rows < 1 || cols < 1 || mid_depth < 0) throw ShapeMismatch("invalid lattice parameters");
    const int n = rows * cols;
    Circuit c;
    c.n_qubits = n;
    Rng rng(seed);
    std::vector<Gate> hl;
    for (int q = 0; q < n; ++q) hl.push_back({GateKind::h, {q}});
    c.layers.push_back(hl);
    const GateKind singles[3] = {GateKind::t, GateKind::sqrt_x, GateKind::sqrt_y};
    std::vector<int> last(std::size_t(n), -1);
    for (int d = 0; d < mid_depth; ++d) {
        std::vector<Gate> layer;
        std::vector<bool> busy(std::size_t(n), false);
        for (const auto& [a, b] : cz_pattern(rows, cols, d)) {
            layer.push_back({GateKind::cz, {a, b}});
            busy[std::size_t(a)] = busy[std::size_t(b)] = true;
        }
        for (int q = 0; q < n; ++q) {
            if (busy[std::size_t(q)]) continue;
            std::vector<int> allowed;
            for (int g = 0; g < 3; ++g)
                if (g != last[std::size_t(q)]) allowed.push_back(g);
            const int pick = allowed[std::size_t(rng.next_below(allowed.size()))];
            last[std::size_t(q)] = pick;
            layer.push_back({singles[pick], {q}});
        }
        c.layers.push_back(std::move(layer));
    }
    c.layers.push_back(hl);
    return c;
}

// <x| C |0...0> as a network (qcircuit.cpp:142-182): |0> states, one tensor per
// gate on wire labels "w<q>_<step>", <x_q| selectors
inline TensorNetwork circuit_to_network(const Circuit& c, const Bitstring& x) {
    validate_circuit(c);
    if (int(x.size()) != c.n_qubits) throw ShapeMismatch("bitstring length does not match circuit");
    auto wire = [](int q, int s) { return "w" + std::to_string(q) + "_" + std::to_string(s); };
    TensorNetwork net;
    std::vector<int> step(std::size_t(c.n_qubits), 0);
    for (int q = 0; q < c.n_qubits; ++q) net.nodes.push_back(TensorC32({wire(q, 0)}, {2}, {{1.0f, 0.0f}, {0.0f, 0.0f}}));
    for (const auto& layer : c.layers)
        for (const auto& g : layer) {
            TensorC32 t = gate_tensor(g);
            if (g.kind == GateKind::cz) {
                const int a = g.qubits[0], b = g.qubits[1];
                int& sa = step[std::size_t(a)];
                int& sb = step[std::size_t(b)];
                t.labels = {wire(a, sa + 1), wire(b, sb + 1), wire(a, sa), wire(b, sb)};
                ++sa;
                ++sb;
            } else {
                const int q = g.qubits[0];
                int& s = step[std::size_t(q)];
                t.labels = {wire(q, s + 1), wire(q, s)};
                ++s;
            }
            net.nodes.push_back(std::move(t));
        }
    for (int q = 0; q < c.n_qubits; ++q) {
        const bool one = x[std::size_t(q)] != 0;
        net.nodes.push_back(TensorC32({wire(q, step[std::size_t(q)])}, {2},
                                      {{one ? 0.0f : 1.0f, 0.0f}, {one ? 1.0f : 0.0f, 0.0f}}));
    }
    return net;
}

inline std::complex<float> amplitude(const Circuit& c, const Bitstring& x, const DispatchConfig& config,
                                     DecisionLog* log = nullptr) {
    const TensorNetwork net = circuit_to_network(c, x);
    return contract_network(net, greedy_path(net), config, log).data[0];
}
inline std::complex<float> amplitude(const Circuit& c, const Bitstring& x, const SelectionPolicy& policy,
                                     DecisionLog* log = nullptr) {
    return amplitude(c, x, DispatchConfig{policy, TilingConfig{}, std::nullopt}, log);
}

// full state vector in f64 on the device (qcircuit.cpp:197-225); qubit q = bit q
inline std::vector<std::complex<double>> statevector_oracle(const Circuit& c) {
    validate_circuit(c);
    if (c.n_qubits > 24) throw TooManyQubits("state-vector oracle limited to 24 qubits");
    std::vector<int> qa, qb;
    std::vector<double> u;
    for (const auto& layer : c.layers)
        for (const auto& g : layer) {
            qa.push_back(g.qubits[0]);
            qb.push_back(g.kind == GateKind::cz ? g.qubits[1] : -1);
            const auto m = gate_matrix_f64(g.kind);
            for (int i = 0; i < 4; ++i) {
                u.push_back(g.kind == GateKind::cz ? 0.0 : m[std::size_t(i)].real());
                u.push_back(g.kind == GateKind::cz ? 0.0 : m[std::size_t(i)].imag());
            }
        }
    qa.push_back(0);
    qb.push_back(-1);
    u.resize(u.size() + 8, 0.0);
    const std::size_t dim = std::size_t(1) << c.n_qubits;
    detail::DeviceBuffer d(dim * 16);
    throw_status(tcec_statevector_f64(detail::handle(), c.n_qubits, int(qa.size()) - 1, qa.data(), qb.data(),
                                      u.data(), d.p));
    std::vector<std::complex<double>> st(dim);
    detail::download(st.data(), d.p, dim * 16);
    return st;
}

inline std::complex<double> amplitude_oracle(const Circuit& c, const Bitstring& x) {
    if (int(x.size()) != c.n_qubits) throw ShapeMismatch("bitstring length does not match circuit");
    const auto st = statevector_oracle(c);
    std::size_t idx = 0;
    for (int q = 0; q < c.n_qubits; ++q)
        if (x[std::size_t(q)]) idx |= std::size_t(1) << q;
    return st[idx];
}

// text format (qcircuit.cpp:237-281): "qubits n", then layer ... endlayer
// blocks, one gate per line (H q | T q | SX q | SY q | CZ q1 q2)
inline void save_circuit(std::ostream& os, const Circuit& c) {
    os << "qubits " << c.n_qubits << "\n";
    for (const auto& layer : c.layers) {
        os << "layer\n";
        for (const auto& g : layer) {
            os << to_string(g.kind);
            for (int q : g.qubits) os << " " << q;
            os << "\n";
        }
        os << "endlayer\n";
    }
}

inline Circuit load_circuit(std::istream& is) {
    Circuit c;
    std::string line;
    bool open = false;
    while (std::getline(is, line)) {
        std::istringstream ss(line);
        std::string tok;
        if (!(ss >> tok)) continue;
        if (tok == "qubits") {
            ss >> c.n_qubits;
        } else if (tok == "layer") {
            c.layers.emplace_back();
            open = true;
        } else if (tok == "endlayer") {
            open = false;
        } else {
            if (!open) throw ShapeMismatch("gate outside layer block");
            Gate g{GateKind::h, {}};
            int k = 0;
            while (k < 5 && tok != to_string(GateKind(k))) ++k;
            if (k == 5) throw ShapeMismatch("unknown gate: " + tok);
            g.kind = GateKind(k);
            for (int q; ss >> q;) g.qubits.push_back(q);
            c.layers.back().push_back(std::move(g));
        }
    }
    validate_circuit(c);
    return c;
}

}  // namespace mpsgemm

// the round-1 name of the drop-in namespace
namespace mpsgemm_b200 = mpsgemm;
