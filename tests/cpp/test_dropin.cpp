// C++ drop-in check: reference-style tests (test_cgemm.cpp, test_precsel.cpp,
// test_tensor.cpp) written against include/mpsgemm_b200.hpp, i.e. against the
// mpsgemm API surface a reference user keeps after switching libraries.
// Built and run by tests/test_cpp_dropin.py; prints "ALL OK" on success.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "mpsgemm_b200.hpp"

namespace mp = mpsgemm_b200;

static int g_fail = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);          \
            ++g_fail;                                                            \
        }                                                                        \
    } while (0)

static mp::MatrixC32 random_c(std::int64_t r, std::int64_t c, unsigned seed) {
    std::mt19937 g(seed);
    std::uniform_real_distribution<float> u(-1.0f, 1.0f);
    mp::MatrixC32 m(r, c);
    for (auto& v : m.data) v = {u(g), u(g)};
    return m;
}

static double rel_err(const mp::MatrixC32& c, const std::vector<std::complex<double>>& ref) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < ref.size(); ++i) {
        const std::complex<double> d = std::complex<double>(c.data[i]) - ref[i];
        num += std::norm(d);
        den += std::norm(ref[i]);
    }
    return std::sqrt(num / den);
}

static std::vector<std::complex<double>> ref_product(const mp::MatrixC32& a, const mp::MatrixC32& b) {
    std::vector<std::complex<double>> c(std::size_t(a.rows * b.cols));
    for (std::int64_t i = 0; i < a.rows; ++i)
        for (std::int64_t k = 0; k < a.cols; ++k)
            for (std::int64_t j = 0; j < b.cols; ++j)
                c[std::size_t(i * b.cols + j)] += std::complex<double>(a(i, k)) * std::complex<double>(b(k, j));
    return c;
}

int main() {
    // complex identity and i*i (test_cgemm.cpp:28-38)
    {
        mp::MatrixC32 eye(2, 2);
        eye(0, 0) = eye(1, 1) = 1.0f;
        const mp::MatrixC32 b = random_c(2, 2, 1);
        const mp::MatrixC32 c = mp::cgemm(eye, b, mp::GemmMode::fp32_ref);
        CHECK(std::memcmp(c.data.data(), b.data.data(), 32) == 0);
        mp::MatrixC32 im(1, 1, {{0.0f, 1.0f}});
        const mp::MatrixC32 sq = mp::cgemm(im, im, mp::GemmMode::fp32_ref);
        CHECK(sq.data[0].real() == -1.0f && sq.data[0].imag() == 0.0f);
    }
    // corrected modes near the reference (test_cgemm.cpp:55-68)
    {
        const mp::MatrixC32 a = random_c(256, 256, 7), b = random_c(256, 256, 8);
        const auto ref = ref_product(a, b);
        const double e32 = rel_err(mp::cgemm(a, b, mp::GemmMode::fp32_ref), ref);
        const double e16 = rel_err(mp::cgemm(a, b, mp::GemmMode::fp16_tcec), ref);
        const double etf = rel_err(mp::cgemm(a, b, mp::GemmMode::tf32_tcec), ref);
        CHECK(e16 <= 4 * e32 && etf <= 4 * e32 && e32 < 2e-6);
        std::printf("n=256 rel_err fp32_ref %.3e fp16_tcec %.3e tf32_tcec %.3e\n", e32, e16, etf);
    }
    // batched error carries the index (test_cgemm.cpp:124-133)
    {
        std::vector<std::pair<mp::MatrixC32, mp::MatrixC32>> pairs;
        pairs.emplace_back(random_c(4, 4, 1), random_c(4, 4, 2));
        pairs.emplace_back(random_c(4, 5, 3), random_c(4, 4, 4));
        bool caught = false;
        try {
            (void)mp::cgemm_batched(pairs, mp::GemmMode::fp32_ref);
        } catch (const mp::ShapeMismatch& e) {
            caught = std::string(e.what()).find("batch entry 1") != std::string::npos;
        }
        CHECK(caught);
    }
    // statistics KATs (test_precsel.cpp:30-76)
    {
        mp::MatrixC32 ones(4, 4);
        for (auto& v : ones.data) v = {1.0f, 1.0f};
        const auto s = mp::exp_stats(ones);
        CHECK(s.n_total == 32 && s.n_nonzero == 32 && s.n1 == 32 && s.e_max == 0);
        mp::MatrixC32 m(1, 2);
        m.data[0] = {1.0f, 0.0f};
        m.data[1] = {std::ldexp(1.0f, -40), 0.0f};
        const auto s2 = mp::exp_stats(m);
        CHECK(s2.e_max == 0 && s2.n_nonzero == 2 && s2.n1 == 1 && s2.n2 == 1);
        const auto skipped = mp::exp_stats_staged(ones, 14, 0.0);
        CHECK(!skipped.stage2_evaluated && skipped.n2 == skipped.n1);
    }
    // mode selection rule (test_precsel.cpp:110-127)
    {
        mp::MatrixTolerance ok0{mp::ToleranceLevel::fp16_ok, 0};
        mp::MatrixTolerance scaled{mp::ToleranceLevel::fp16_scaled_ok, -20};
        mp::MatrixTolerance tf{mp::ToleranceLevel::tf32_only, -3};
        const auto m2 = mp::select_mode(ok0, scaled);
        CHECK(m2.kind == mp::ComputeKind::fp16_tcec_scaled && m2.scale_exp_a == 14 && m2.scale_exp_b == 34);
        CHECK(mp::select_mode(tf, ok0).kind == mp::ComputeKind::tf32_tcec);
    }
    // scaling (test_precsel.cpp:198-224)
    {
        mp::MatrixC32 big(2, 2);
        for (auto& v : big.data) v = {1.0f, 0.0f};
        bool thrown = false;
        try {
            (void)mp::scale_matrix(big, 128);
        } catch (const mp::ScaleOverflow&) {
            thrown = true;
        }
        CHECK(thrown);
        const auto d = mp::descale_output(big, 14, 34);
        CHECK(d.data[0].real() == std::ldexp(1.0f, -48));
    }
    // dispatch routing + log (test_precsel.cpp:242-302)
    {
        mp::DecisionLog log;
        const mp::MatrixC32 small = random_c(64, 64, 410);
        const auto r = mp::dispatch_cgemm(small, small, mp::SelectionPolicy{}, &log);
        CHECK(r.decision.kind == mp::ComputeKind::fp32_baseline && !r.stats_a.has_value());
        CHECK(log.records().size() == 1 && log.records()[0].to_line() == "64,64,64,FP32_BASELINE,0,0,-,-,-,-,-,-");
        mp::SelectionPolicy p;
        p.size_auto = 16;
        p.size_tf32 = 8;
        mp::MatrixC32 a(16, 16), b(16, 16);
        for (auto& v : a.data) v = {std::ldexp(1.2f, -20), std::ldexp(0.9f, -20)};
        for (auto& v : b.data) v = {std::ldexp(1.1f, -20), std::ldexp(0.7f, -20)};
        const auto r2 = mp::dispatch_cgemm(a, b, p);
        CHECK(r2.decision.kind == mp::ComputeKind::fp16_tcec_scaled && r2.decision.scale_exp_a == 34);
        CHECK(rel_err(r2.c, ref_product(a, b)) <= 1e-6);
    }
    // permute + contract_pair (test_tensor.cpp:33-125)
    {
        mp::TensorC32 t({"a", "b", "c"}, {2, 3, 4});
        std::mt19937 g(1);
        for (auto& v : t.data) v = {float(g() % 100), float(g() % 100)};
        const auto back = mp::permute(mp::permute(t, {"c", "a", "b"}), {"a", "b", "c"});
        CHECK(std::memcmp(back.data.data(), t.data.data(), t.data.size() * 8) == 0);
        bool thrown = false;
        try {
            (void)mp::permute(t, {"a", "b", "x"});
        } catch (const mp::InvalidPermutation&) {
            thrown = true;
        }
        CHECK(thrown);
        mp::DispatchConfig base;
        base.force = mp::ForcedMode::fp32_ref;
        mp::TensorC32 eye({"c", "c2"}, {4, 4});
        for (int i = 0; i < 4; ++i) eye.data[std::size_t(i * 4 + i)] = {1.0f, 0.0f};
        const auto r = mp::contract_pair(t, eye, base);
        CHECK((r.labels == std::vector<std::string>{"a", "b", "c2"}));
        CHECK(std::memcmp(r.data.data(), t.data.data(), t.data.size() * 8) == 0);
        mp::TensorC32 x({"s"}, {2}), y({"s"}, {3});
        thrown = false;
        try {
            (void)mp::contract_pair(x, y, base);
        } catch (const mp::ExtentMismatch&) {
            thrown = true;
        }
        CHECK(thrown);
    }
    // network fold: path-order invariance (test_tensor.cpp:127-149)
    {
        mp::TensorNetwork net;
        std::mt19937 g(3);
        std::uniform_real_distribution<float> u(-1, 1);
        auto mk = [&](std::vector<std::string> l, std::vector<std::int64_t> d) {
            mp::TensorC32 t(std::move(l), std::move(d));
            for (auto& v : t.data) v = {u(g), u(g)};
            return t;
        };
        net.nodes = {mk({"i", "j", "k"}, {8, 8, 8}), mk({"k", "l"}, {8, 8}), mk({"l", "j", "i"}, {8, 8, 8})};
        mp::DispatchConfig cfg;
        const auto p1 = mp::greedy_path(net);
        const auto z1 = mp::contract_network(net, p1, cfg).data[0];
        const auto z2 = mp::contract_network(net, mp::ContractionPath{{{0, 2}, {1, 3}}}, cfg).data[0];
        CHECK(std::abs(std::complex<double>(z1) - std::complex<double>(z2)) <= 1e-5 * std::abs(std::complex<double>(z1)));
        bool thrown = false;
        try {
            (void)mp::contract_network(net, mp::ContractionPath{{{0, 0}}}, cfg);
        } catch (const mp::InvalidPath&) {
            thrown = true;
        }
        CHECK(thrown);
    }
    if (g_fail == 0) std::printf("ALL OK\n");
    return g_fail == 0 ? 0 : 1;
}
