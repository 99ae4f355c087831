// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal doctest-compatible subset (the reference's vendor/doctest is absent,
// /root/reference/proj/CMakeLists.txt:5), enough to build and run the
// reference's own unit tests as the oracle gate. SUBCASEs run in sequence in
// one pass of their TEST_CASE (sufficient for the reference tests, whose
// subcases do not depend on re-entry). Approx follows doctest's published
// comparison: |a-b| < eps * (scale + max(|a|,|b|)), eps default 100*FLT_EPSILON.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <utility>
#include <vector>

namespace doctest {

struct Approx {
    double value;
    double eps = 1.1920928955078125e-07 * 100;
    double sc = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    Approx& scale(double s) { sc = s; return *this; }
    bool matches(double a) const {
        return std::fabs(a - value) < eps * (sc + std::max(std::fabs(a), std::fabs(value)));
    }
    friend bool operator==(double a, const Approx& b) { return b.matches(a); }
    friend bool operator==(const Approx& b, double a) { return b.matches(a); }
    friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
    friend bool operator!=(const Approx& b, double a) { return !b.matches(a); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value || b.matches(a); }
    friend bool operator>=(double a, const Approx& b) { return a > b.value || b.matches(a); }
};

struct Registry {
    std::vector<std::pair<std::string, void (*)()>> cases;
    static Registry& get() { static Registry r; return r; }
};
inline int& failures() { static int f = 0; return f; }
inline int& checks() { static int c = 0; return c; }
inline std::string& current() { static std::string c; return c; }
struct Register {
    Register(const char* name, void (*fn)()) { Registry::get().cases.emplace_back(name, fn); }
};
struct RequireAbort {};
inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::printf("FAIL [%s] %s:%d: %s\n", current().c_str(), file, line, what);
}

}  // namespace doctest

#define ORACLE_DT_CAT2(a, b) a##b
#define ORACLE_DT_CAT(a, b) ORACLE_DT_CAT2(a, b)
#define TEST_CASE(name)                                                                    \
    static void ORACLE_DT_CAT(oracle_tc_, __LINE__)();                                     \
    static doctest::Register ORACLE_DT_CAT(oracle_reg_, __LINE__)(name,                    \
                                                                  &ORACLE_DT_CAT(oracle_tc_, __LINE__)); \
    static void ORACLE_DT_CAT(oracle_tc_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...)                                                                          \
    do {                                                                                    \
        ++doctest::checks();                                                                \
        if (!(__VA_ARGS__)) doctest::report(__FILE__, __LINE__, #__VA_ARGS__);              \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        ++doctest::checks();                                                                \
        if (!(__VA_ARGS__)) {                                                               \
            doctest::report(__FILE__, __LINE__, #__VA_ARGS__);                              \
            throw doctest::RequireAbort{};                                                  \
        }                                                                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                            \
    do {                                                                                    \
        ++doctest::checks();                                                                \
        bool oracle_ok = false;                                                             \
        try { expr; } catch (const T&) { oracle_ok = true; } catch (...) {}                \
        if (!oracle_ok) doctest::report(__FILE__, __LINE__, "throws " #T ": " #expr);       \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                 \
    do {                                                                                    \
        ++doctest::checks();                                                                \
        try { expr; } catch (...) { doctest::report(__FILE__, __LINE__, "nothrow: " #expr); } \
    } while (0)
#define INFO(...) do {} while (0)
#define CAPTURE(x) do {} while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    for (auto& tc : doctest::Registry::get().cases) {
        doctest::current() = tc.first;
        try {
            tc.second();
        } catch (const doctest::RequireAbort&) {
        } catch (const std::exception& e) {
            ++doctest::failures();
            std::printf("EXCEPTION [%s] %s\n", tc.first.c_str(), e.what());
        }
    }
    std::printf("checks=%d failures=%d testcases=%zu\n", doctest::checks(), doctest::failures(),
                doctest::Registry::get().cases.size());
    return doctest::failures() ? 1 : 0;
}
#endif
