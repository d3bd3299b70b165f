// Minimal doctest-compatible test shim (test infrastructure only).
//
// The reference's unit tests (/root/reference/proj/tests/test_quant.cpp and
// test_numeric.cpp) include <doctest.h>, which is not vendored anywhere in this
// image.  This header implements only the subset those two files use --
// TEST_CASE, CHECK, REQUIRE, CHECK_THROWS, CHECK_THROWS_WITH and
// doctest::Approx(...).epsilon(...) -- so the reference tests compile
// UNMODIFIED from their own sources and re-pin the reference quantizer and
// numeric core.  Written from the public doctest semantics;
// no doctest code is copied.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
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
    // doctest semantics: |a - b| < eps * (scale + max(|a|, |b|)), scale = 1
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

private:
    double value_;
    // doctest's default epsilon: float epsilon * 100
    double eps_ = static_cast<double>(1.1920928955078125e-07f) * 100.0;
};

namespace detail {

struct Registry {
    std::vector<std::pair<const char*, void (*)()>> cases;
    int checks = 0;
    int failures = 0;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct Registrar {
    Registrar(const char* name, void (*fn)()) { Registry::get().cases.emplace_back(name, fn); }
};

struct RequireFailed {};

inline void report(bool ok, const char* what, const char* file, int line, bool fatal) {
    auto& r = Registry::get();
    ++r.checks;
    if (!ok) {
        ++r.failures;
        std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
        if (fatal) throw RequireFailed{};
    }
}

inline int run_all() {
    auto& r = Registry::get();
    int failed_cases = 0;
    for (auto& c : r.cases) {
        int before = r.failures;
        try {
            c.second();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++r.failures;
            std::fprintf(stderr, "TEST_CASE(%s) threw: %s\n", c.first, e.what());
        }
        if (r.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | failed: %d | assertions: %d | failed: %d\n",
                r.cases.size(), failed_cases, r.checks, r.failures);
    return r.failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_CASE(name)                                                              \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                              \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(         \
        name, &DOCTEST_CAT(doctest_case_, __LINE__));                                \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS(...)                                                            \
    do {                                                                             \
        bool threw_ = false;                                                         \
        try {                                                                        \
            (void)(__VA_ARGS__);                                                     \
        } catch (...) {                                                              \
            threw_ = true;                                                           \
        }                                                                            \
        ::doctest::detail::report(threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH(expr, msg)                                                 \
    do {                                                                             \
        bool ok_ = false;                                                            \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const std::exception& e_) {                                         \
            ok_ = std::string(e_.what()) == std::string(msg);                        \
        } catch (...) {                                                              \
        }                                                                            \
        ::doctest::detail::report(ok_, "throws with '" msg "': " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
