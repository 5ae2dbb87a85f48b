// mpsgemm_b200.hpp -- C++ drop-in for the reference mpsgemm entry points of the
// north-star path, implemented over the C-ABI in tcec_b200.h (libtcec_b200.so).
//
// A reference user switches by including this header instead of
// mpsgemm/{cgemm,precsel,tensor,network,qcircuit}.hpp and linking
// libtcec_b200.so: the namespace, type names, function names, argument meaning,
// value semantics (host std::vector storage in, host storage out) and the
// exception taxonomy are the reference's (common.hpp:9-41).  Each call stages
// its operands to the GPU, runs the sm_100a path, and copies the result back;
// contract_network keeps every intermediate on the device.
//
//   cgemm            cgemm.hpp:17-18      dispatch_cgemm   precsel.hpp:153-156
//   exp_stats[_staged] precsel.hpp:68-72  matrix_tolerance precsel.hpp:74
//   select_mode      precsel.hpp:76-77    scale/descale    precsel.hpp:82-91
//   permute          tensor.hpp:56-57     contract_pair    network.hpp:29-32
//   contract_network network.hpp:37-38    greedy_path      network.hpp:49
//   amplitude        qcircuit.hpp:49-52   (circuit helpers in the Python host)
#pragma once

#include <algorithm>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "tcec_b200.h"

namespace mpsgemm_b200 {

// ------------------------------------------------------------------ errors
struct ShapeMismatch : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ZeroReference : std::domain_error { using std::domain_error::domain_error; };
struct ScaleOverflow : std::range_error { using std::range_error::range_error; };
struct InvalidPermutation : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ExtentMismatch : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct InvalidPath : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct DisconnectedNetwork : std::invalid_argument { using std::invalid_argument::invalid_argument; };
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
    default: throw DeviceError(msg);
    }
}

// ------------------------------------------------------------------- types
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
};
using MatrixC32 = Matrix<std::complex<float>>;

enum class GemmMode { fp32_ref, fp64_oracle, tf32_tc, fp16_tc, tf32_tcec, fp16_tcec };
struct TilingConfig { int k_tile = 16; };

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
struct ComputeMode { ComputeKind kind = ComputeKind::fp32_baseline; int scale_exp_a = 0, scale_exp_b = 0; };
struct SelectionPolicy {
    double threshold_t = 0.0;
    std::int64_t size_auto = 2048, size_tf32 = 512;
    int target_max_exponent = 14;
};
enum class ForcedMode { fp32_ref, fp64_oracle, tf32_tc, fp16_tc, tf32_tcec, fp16_tcec, fp16_tcec_scaled };
struct DispatchConfig { SelectionPolicy policy; TilingConfig tiling; std::optional<ForcedMode> force; };

struct DecisionRecord {
    std::int64_t m = 0, n = 0, k = 0;
    std::string mode;
    int scale_a = 0, scale_b = 0;
    std::optional<ExpStats> stats_a, stats_b;
    double wall_ms = 0.0;
    std::string line;  // DecisionRecord::to_line() as produced by the device path
    std::string to_line() const { return line; }
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

template <typename T>
struct Tensor {
    std::vector<std::string> labels;
    std::vector<std::int64_t> dims;
    std::vector<T> data;
    Tensor() : data(1) {}
    Tensor(std::vector<std::string> l, std::vector<std::int64_t> d) : labels(std::move(l)), dims(std::move(d)) {
        data.assign(std::size_t(size()), T{});
    }
    Tensor(std::vector<std::string> l, std::vector<std::int64_t> d, std::vector<T> v)
        : labels(std::move(l)), dims(std::move(d)), data(std::move(v)) {
        if (std::int64_t(data.size()) != size()) throw ShapeMismatch("tensor data length does not match dims");
    }
    int rank() const { return int(dims.size()); }
    std::int64_t size() const { std::int64_t s = 1; for (auto d : dims) s *= d; return s; }
};
using TensorC32 = Tensor<std::complex<float>>;
struct TensorNetwork { std::vector<TensorC32> nodes; };
struct ContractionPath { std::vector<std::pair<int, int>> steps; };

// ------------------------------------------------------------ device context
namespace detail {

struct Context {
    tcec_handle h = nullptr;
    Context() { throw_status(tcec_create(0, &h)); }
    ~Context() { if (h) tcec_destroy(h); }
};

inline tcec_handle handle() {
    thread_local Context ctx;  // one handle per thread (precsel.hpp:105-123 reentrancy)
    return ctx.h;
}

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
// with the kernels the C-ABI enqueues there; the stream is synchronised before
// the host touches the result (a legacy-stream cudaMemcpy would not be).
inline void upload(void* d, const void* h, std::size_t bytes) {
    if (!bytes) return;
    cudaStream_t s = static_cast<cudaStream_t>(tcec_get_stream(handle()));
    if (cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) throw DeviceError("H2D failed");
}
inline void download(void* h, const void* d, std::size_t bytes) {
    cudaStream_t s = static_cast<cudaStream_t>(tcec_get_stream(handle()));
    if (bytes && cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
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

}  // namespace detail

// ------------------------------------------------------------------- CGEMM
inline MatrixC32 cgemm(const MatrixC32& a, const MatrixC32& b, GemmMode mode,
                       const TilingConfig& tiling = {}, bool* overflow = nullptr) {
    if (a.cols != b.rows) throw ShapeMismatch("cgemm: inner dimensions differ");
    detail::DeviceBuffer da(a.data.size() * 8), db(b.data.size() * 8), dc(std::size_t(a.rows * b.cols) * 8);
    detail::upload(da.p, a.data.data(), a.data.size() * 8);
    detail::upload(db.p, b.data.data(), b.data.size() * 8);
    int ovf = 0;
    throw_status(tcec_cgemm(detail::handle(), da.p, db.p, dc.p, a.rows, b.cols, a.cols,
                                    int(mode), tiling.k_tile, &ovf));
    MatrixC32 c(a.rows, b.cols);
    detail::download(c.data.data(), dc.p, c.data.size() * 8);
    if (overflow && ovf) *overflow = true;
    return c;
}

inline std::vector<MatrixC32> cgemm_batched(const std::vector<std::pair<MatrixC32, MatrixC32>>& pairs,
                                            GemmMode mode, const TilingConfig& tiling = {},
                                            bool* overflow = nullptr) {
    std::vector<MatrixC32> out;
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        try {
            out.push_back(cgemm(pairs[i].first, pairs[i].second, mode, tiling, overflow));
        } catch (const ShapeMismatch& e) {
            throw ShapeMismatch("batch entry " + std::to_string(i) + ": " + e.what());
        }
    }
    return out;
}

// --------------------------------------------------------------- precsel
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

inline ComputeMode select_mode(const MatrixTolerance& a, const MatrixTolerance& b,
                               int target_max_exponent = 14) {
    int kind = 0, sa = 0, sb = 0;
    throw_status(tcec_select_mode(int(a.level), a.e_max.has_value(), a.e_max.value_or(0),
                                          int(b.level), b.e_max.has_value(), b.e_max.value_or(0),
                                          target_max_exponent, &kind, &sa, &sb));
    return {ComputeKind(kind), sa, sb};
}

inline void scale_components(MatrixC32& m, int scale_exp, bool check) {
    detail::DeviceBuffer d(m.data.size() * 8);
    detail::upload(d.p, m.data.data(), m.data.size() * 8);
    const int rc = tcec_scale_components(detail::handle(), static_cast<float*>(d.p),
                                         std::int64_t(m.data.size()) * 2, scale_exp, check);
    throw_status(rc);
    detail::download(m.data.data(), d.p, m.data.size() * 8);
}
inline void scale_matrix_inplace(MatrixC32& m, int s) { scale_components(m, s, true); }
inline MatrixC32 scale_matrix(const MatrixC32& m, int s) { MatrixC32 o = m; scale_matrix_inplace(o, s); return o; }
inline void descale_output_inplace(MatrixC32& c, int sa, int sb) { scale_components(c, -(sa + sb), false); }
inline MatrixC32 descale_output(const MatrixC32& c, int sa, int sb) { MatrixC32 o = c; descale_output_inplace(o, sa, sb); return o; }

inline DispatchResult dispatch_cgemm(const MatrixC32& a, const MatrixC32& b, const DispatchConfig& config,
                                     DecisionLog* log = nullptr) {
    if (a.cols != b.rows) throw ShapeMismatch("dispatch_cgemm: inner dimensions differ");
    const tcec_dispatch_config_t cfg = detail::to_c(config);
    DispatchResult r;
    r.c = MatrixC32(a.rows, b.cols);
    tcec_dispatch_result_t res;
    throw_status(tcec_dispatch_cgemm_host(detail::handle(), a.data.data(), b.data.data(),
                                                  r.c.data.data(), a.rows, b.cols, a.cols, &cfg, &res));
    r.decision = {ComputeKind(res.kind), res.scale_a, res.scale_b};
    if (res.has_stats) {
        r.stats_a = detail::from_c(res.stats_a);
        r.stats_b = detail::from_c(res.stats_b);
    }
    r.overflow = res.overflow != 0;
    if (log) {
        DecisionRecord rec;
        rec.m = a.rows;
        rec.n = b.cols;
        rec.k = a.cols;
        rec.line = res.line;
        rec.mode = detail::field(rec.line, 3);
        rec.scale_a = res.scale_a;
        rec.scale_b = res.scale_b;
        rec.stats_a = r.stats_a;
        rec.stats_b = r.stats_b;
        log->append(std::move(rec));
    }
    return r;
}

inline DispatchResult dispatch_cgemm(const MatrixC32& a, const MatrixC32& b, const SelectionPolicy& policy,
                                     DecisionLog* log = nullptr) {
    return dispatch_cgemm(a, b, DispatchConfig{policy, TilingConfig{}, std::nullopt}, log);
}

// --------------------------------------------------------------- tensors
template <typename T>
inline Tensor<T> permute(const Tensor<T>& t, const std::vector<std::string>& new_order) {
    static_assert(sizeof(T) == 8, "device permute is for complex<float> tensors");
    const int r = t.rank();
    if (int(new_order.size()) != r) throw InvalidPermutation("permutation has wrong length");
    std::vector<int> axis_of(static_cast<std::size_t>(r));
    std::vector<bool> used(static_cast<std::size_t>(r), false);
    for (int a = 0; a < r; ++a) {
        int found = -1;
        for (int o = 0; o < r; ++o)
            if (!used[std::size_t(o)] && t.labels[std::size_t(o)] == new_order[std::size_t(a)]) { found = o; break; }
        if (found < 0) throw InvalidPermutation("label not in tensor: " + new_order[std::size_t(a)]);
        used[std::size_t(found)] = true;
        axis_of[std::size_t(a)] = found;
    }
    Tensor<T> out;
    out.labels = new_order;
    for (int a = 0; a < r; ++a) out.dims.push_back(t.dims[std::size_t(axis_of[std::size_t(a)])]);
    out.data.resize(t.data.size());
    detail::DeviceBuffer ds(t.data.size() * 8), dd(t.data.size() * 8);
    detail::upload(ds.p, t.data.data(), t.data.size() * 8);
    throw_status(tcec_permute(detail::handle(), ds.p, dd.p, r, t.dims.data(), axis_of.data()));
    detail::download(out.data.data(), dd.p, out.data.size() * 8);
    return out;
}

namespace detail {

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
        throw_status(tcec_network_create(with_device ? handle() : nullptr, int(tn.nodes.size()),
                                         ranks.data(), labels.data(), dims.data(), &net));
        for (std::size_t i = 0; i < tn.nodes.size(); ++i)
            throw_status(tcec_network_set_node(net, int(i), tn.nodes[i].data.data()));
    }
    ~NetworkHandle() { if (net) tcec_network_destroy(net); }
};

inline void append_log(DecisionLog* log, const std::string& lines) {
    if (!log) return;
    std::size_t pos = 0;
    while (pos < lines.size()) {
        const std::size_t e = lines.find('\n', pos);
        const std::string ln = lines.substr(pos, e - pos);
        if (!ln.empty()) {
            DecisionRecord r;
            r.line = ln;
            r.m = std::stoll(field(ln, 0));
            r.n = std::stoll(field(ln, 1));
            r.k = std::stoll(field(ln, 2));
            r.mode = field(ln, 3);
            r.scale_a = std::stoi(field(ln, 4));
            r.scale_b = std::stoi(field(ln, 5));
            log->append(std::move(r));
        }
        if (e == std::string::npos) break;
        pos = e + 1;
    }
}

}  // namespace detail

inline ContractionPath greedy_path(const TensorNetwork& net) {
    detail::NetworkHandle nh(net, false);
    std::vector<int> steps(net.nodes.size() > 1 ? 2 * (net.nodes.size() - 1) : 1);
    throw_status(tcec_network_greedy_path(nh.net, steps.data()));
    ContractionPath p;
    for (std::size_t i = 0; i + 1 < net.nodes.size(); ++i) p.steps.emplace_back(steps[2 * i], steps[2 * i + 1]);
    return p;
}

inline TensorC32 contract_network(const TensorNetwork& net, const ContractionPath& path,
                                  const DispatchConfig& config, DecisionLog* log = nullptr) {
    detail::NetworkHandle nh(net, true);
    std::vector<int> steps;
    for (const auto& [a, b] : path.steps) { steps.push_back(a); steps.push_back(b); }
    std::map<std::string, std::pair<int, std::int64_t>> occ;  // open-label extents bound the output
    for (const auto& t : net.nodes)
        for (int a = 0; a < t.rank(); ++a) {
            auto& o = occ[t.labels[std::size_t(a)]];
            o.first += 1;
            o.second = t.dims[std::size_t(a)];
        }
    std::int64_t cap = 1;
    for (const auto& [l, o] : occ) if (o.first == 1) cap *= o.second;
    std::vector<std::complex<float>> out(std::size_t(std::max<std::int64_t>(cap, 1)));
    std::vector<int> labels(occ.size() + 1);
    int rank = 0;
    std::string lines(std::size_t(200) * (path.steps.size() + 1), '\0');
    const tcec_dispatch_config_t cfg = detail::to_c(config);
    throw_status(tcec_contract_network(nh.net, steps.data(), int(path.steps.size()), &cfg, out.data(),
                                               std::int64_t(out.size()), &rank, labels.data(),
                                               log ? lines.data() : nullptr, std::int64_t(lines.size())));
    detail::append_log(log, lines.c_str());
    TensorC32 r;
    for (int i = 0; i < rank; ++i) {
        r.labels.push_back(nh.names[std::size_t(labels[std::size_t(i)])]);
        r.dims.push_back(occ[r.labels.back()].second);
    }
    r.data.assign(out.begin(), out.begin() + r.size());
    return r;
}

inline TensorC32 contract_pair(const TensorC32& a, const TensorC32& b, const DispatchConfig& config,
                               DecisionLog* log = nullptr) {
    TensorNetwork net{{a, b}};
    return contract_network(net, ContractionPath{{{0, 1}}}, config, log);
}

inline TensorC32 contract_pair(const TensorC32& a, const TensorC32& b, const SelectionPolicy& policy,
                               DecisionLog* log = nullptr) {
    return contract_pair(a, b, DispatchConfig{policy, TilingConfig{}, std::nullopt}, log);
}

}  // namespace mpsgemm_b200
