// doctest.h -- a minimal stand-in for the doctest framework (absent from this image; the
// reference vendors it under the git-ignored proj/vendor/).  TEST INFRASTRUCTURE ONLY: it lets
// the reference's own test cases compile unmodified against include/lkv/ and run on the B200
// (oracle/Makefile `ref_tests`).  Supports what those cases use: TEST_CASE, CHECK,
// CHECK_THROWS_AS, MESSAGE and doctest::Approx (with doctest's published comparison rule
// |a - b| < eps * (scale + max(|a|, |b|)), eps default 100 * FLT_EPSILON).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {
        return std::fabs(other - value_) < eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& cases() {
    static std::vector<Case> v;
    return v;
}
struct Stats {
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct Register {
    Register(const char* name, void (*fn)(), const char* file, int line) { cases().push_back({name, fn, file, line}); }
};
inline void check(bool ok, const char* expr, const char* file, int line) {
    ++stats().checks;
    if (!ok) {
        ++stats().failed_checks;
        stats().case_failed = true;
        std::fprintf(stderr, "%s:%d: CHECK( %s ) failed\n", file, line, expr);
    }
}
template <class... A>
void message(const A&...) {}
inline int run_all() {
    int failed = 0;
    for (const Case& c : cases()) {
        stats().case_failed = false;
        try {
            c.fn();
        } catch (const std::exception& e) {
            stats().case_failed = true;
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        } catch (...) {
            stats().case_failed = true;
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw a non-std exception\n", c.file, c.line, c.name);
        }
        if (stats().case_failed) ++failed;
        std::printf("[%s] %s\n", stats().case_failed ? "FAIL" : " ok ", c.name);
    }
    std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n", cases().size(), cases().size() - failed, failed);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", stats().checks,
                stats().checks - stats().failed_checks, stats().failed_checks);
    return failed ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_I(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_I(a, b)
#define TEST_CASE(name)                                                                                    \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                    \
    static ::doctest::detail::Register DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__), \
                                                                          __FILE__, __LINE__);           \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool doctest_caught_ = false;                                                              \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_caught_ = true;                                                                \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest::detail::check(doctest_caught_, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, __LINE__); \
    } while (0)
#define MESSAGE(...) ::doctest::detail::message(__VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
