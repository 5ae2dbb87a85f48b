// TEST INFRASTRUCTURE ONLY -- a minimal doctest-compatible harness.
//
// The reference's tests (/root/reference/proj/tests/*.cpp) include <doctest.h>
// from a vendor/ directory that is not part of the reference tree
// (proj/.gitignore:2).  This header implements the subset they use --
// TEST_CASE, SUBCASE (doctest's re-entry semantics: each run of a test case
// enters one not-yet-finished subcase per nesting level), CHECK, REQUIRE,
// CHECK_THROWS, CHECK_THROWS_AS, FAIL, doctest::Approx and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so those sources compile unchanged
// against the B200 drop-in headers (include/mpsgemm/*.hpp) and run on the GPU
// box (oracle/Makefile target reftests).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

  private:
    double v_;
    double eps_ = double(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireAbort {};  // REQUIRE / FAIL: abandon the current run of the test case

struct State {
    int failures = 0, checks = 0;
    const char* test = "";
    // subcase tracking for one test case
    std::vector<int> stack;              // lines of the entered subcases (this run)
    std::vector<bool> entered_at_level;  // one subcase entered per level per run
    std::set<std::vector<int>> finished;
    int skipped_unfinished = 0;
};

inline State& st() {
    static State s;
    return s;
}

inline void report(const char* file, int line, const std::string& what) {
    ++st().failures;
    std::printf("%s:%d: FAILED in TEST_CASE(\"%s\"): %s\n", file, line, st().test, what.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
    ++st().checks;
    if (ok) return;
    report(file, line, std::string(require ? "REQUIRE( " : "CHECK( ") + expr + " )");
    if (require) throw RequireAbort{};
}

struct Subcase {
    bool entered = false;
    int level;
    int skipped_before;
    Subcase(int line) : level(int(st().stack.size())) {
        State& s = st();
        std::vector<int> path = s.stack;
        path.push_back(line);
        if (s.finished.count(path)) return;
        if (int(s.entered_at_level.size()) <= level) s.entered_at_level.resize(std::size_t(level) + 1, false);
        if (s.entered_at_level[std::size_t(level)]) {
            ++s.skipped_unfinished;  // another run of the test case will take it
            return;
        }
        s.entered_at_level[std::size_t(level)] = true;
        s.stack.push_back(line);
        // deeper levels start fresh inside this subcase
        if (s.entered_at_level.size() > std::size_t(level) + 1) s.entered_at_level.resize(std::size_t(level) + 1);
        skipped_before = s.skipped_unfinished;
        entered = true;
    }
    ~Subcase() {
        if (!entered) return;
        State& s = st();
        // finished unless a nested subcase is still pending
        if (s.skipped_unfinished == skipped_before) s.finished.insert(s.stack);
        s.stack.pop_back();
    }
    explicit operator bool() const { return entered; }
};

inline int run_all() {
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        State& s = st();
        s.test = tc.name;
        s.finished.clear();
        const int before = s.failures;
        for (int run = 0; run < 10000; ++run) {
            s.stack.clear();
            s.entered_at_level.clear();
            s.skipped_unfinished = 0;
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                report(tc.file, tc.line, "unexpected exception");
            }
            if (s.skipped_unfinished == 0) break;
        }
        if (s.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | failures: %d\n",
                registry().size(), registry().size() - std::size_t(failed_cases), failed_cases, st().checks,
                st().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                   \
    static void fn();                                                                               \
    static const doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);    \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){__LINE__})

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define FAIL(msg)                                                                                  \
    do {                                                                                           \
        std::ostringstream doctest_os_;                                                            \
        doctest_os_ << msg;                                                                        \
        doctest::detail::report(__FILE__, __LINE__, "FAIL: " + doctest_os_.str());                 \
        throw doctest::detail::RequireAbort{};                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool doctest_ok_ = false;                                                                  \
        try {                                                                                      \
            expr;                                                                                  \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_ok_ = true;                                                                    \
        } catch (...) {                                                                            \
        }                                                                                          \
        doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "THROWS_AS " #expr, false);        \
    } while (0)
#define CHECK_THROWS(expr)                                                                         \
    do {                                                                                           \
        bool doctest_ok_ = false;                                                                  \
        try {                                                                                      \
            expr;                                                                                  \
        } catch (...) {                                                                            \
            doctest_ok_ = true;                                                                    \
        }                                                                                          \
        doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "THROWS " #expr, false);           \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
