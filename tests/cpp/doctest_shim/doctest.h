// Minimal stand-in for the doctest API the reference's unit suites use (vendor/doctest.h is not shipped with the
// reference): self-registering TEST_CASEs, CHECK / REQUIRE (and _FALSE / _THROWS_AS / _NOTHROW), MESSAGE
// and doctest::Approx. Test infrastructure only -- it lets P:tests/test_capi.cpp compile unchanged against the
// B200 library (oracle/Makefile target `suites`). Define ABFT_SHIM_MAIN in exactly one translation unit.
#pragma once
#include <cmath>
#include <exception>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale(double s) { scl = s; return *this; }
    double value, eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100, scl = 1.0;
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) < a.eps * (a.scl + std::fmax(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
};
namespace shim {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { cases().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
inline bool record(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (!ok) {
        ++failures();
        std::printf("  %s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
        if (require) throw RequireFailed{};
    }
    return ok;
}
}  // namespace shim
}  // namespace doctest

#define ABFT_SHIM_CAT2(a, b) a##b
#define ABFT_SHIM_CAT(a, b) ABFT_SHIM_CAT2(a, b)
#define ABFT_SHIM_CASE(fn, name)                                                              \
    static void fn();                                                                         \
    static doctest::shim::Registrar ABFT_SHIM_CAT(fn, _reg)(name, &fn);                       \
    static void fn()
#define TEST_CASE(name) ABFT_SHIM_CASE(ABFT_SHIM_CAT(abft_shim_case_, __LINE__), name)
#define CHECK(...) doctest::shim::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::shim::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, E)                                                                \
    do {                                                                                        \
        bool abft_thrown = false;                                                               \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (const E&) {                                                                    \
            abft_thrown = true;                                                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        doctest::shim::record(abft_thrown, #expr " throws " #E, __FILE__, __LINE__, false);      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                     \
    do {                                                                                        \
        bool abft_ok = true;                                                                    \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (...) {                                                                         \
            abft_ok = false;                                                                    \
        }                                                                                       \
        doctest::shim::record(abft_ok, #expr " does not throw", __FILE__, __LINE__, false);      \
    } while (0)
#define MESSAGE(...) std::printf("  message: %s\n", std::string(__VA_ARGS__).c_str())

#ifdef ABFT_SHIM_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : doctest::shim::cases()) {
        const int before = doctest::shim::failures();
        std::printf("[case] %s\n", c.name);
        try {
            c.fn();
        } catch (const doctest::shim::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::shim::failures();
            std::printf("  unexpected exception: %s\n", e.what());
        }
        if (doctest::shim::failures() != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | failures: %d\n",
                doctest::shim::cases().size(), doctest::shim::cases().size() - failed_cases, failed_cases,
                doctest::shim::checks(), doctest::shim::failures());
    return failed_cases ? 1 : 0;
}
#endif
