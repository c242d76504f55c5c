// Minimal doctest-compatible test runner (the subset the reference's proj/tests/*.cpp use: TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW, DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN). The reference does not
// ship doctest.h (proj/README.md:43-45); this shim lets its test sources compile unchanged against the B200 engine's
// reference-shaped API (include/turbokv/shim.hpp). Exit status = number of failed test cases.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Reg {
    Reg(const char* n, void (*f)()) { cases().push_back({n, f}); }
};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}
struct RequireFailed {};
inline void report(const char* file, int line, const char* what) {
    ++failures();
    std::printf("  FAILED %s:%d: %s\n", file, line, what);
}
inline int run() {
    int failed_cases = 0;
    for (const Case& c : cases()) {
        const int f0 = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::printf("  FAILED with exception: %s\n", e.what());
        }
        const bool ok = failures() == f0;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "ok" : "FAIL", c.name);
    }
    std::printf("[doctest-shim] %zu test cases, %d failed, %d checks, %d failed checks\n", cases().size(), failed_cases,
                checks(), failures());
    return failed_cases;
}
}  // namespace doctest_shim

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                                 \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                                 \
    static ::doctest_shim::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...)                                                                       \
    do {                                                                                 \
        ++::doctest_shim::checks();                                                      \
        if (!(__VA_ARGS__)) ::doctest_shim::report(__FILE__, __LINE__, #__VA_ARGS__);    \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                     \
    do {                                                                                 \
        ++::doctest_shim::checks();                                                      \
        if (!(__VA_ARGS__)) {                                                            \
            ::doctest_shim::report(__FILE__, __LINE__, #__VA_ARGS__);                    \
            throw ::doctest_shim::RequireFailed{};                                       \
        }                                                                                \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
    do {                                                                                 \
        ++::doctest_shim::checks();                                                      \
        bool doctest_ok_ = false;                                                        \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const __VA_ARGS__&) {                                                   \
            doctest_ok_ = true;                                                          \
        } catch (...) {                                                                  \
        }                                                                                \
        if (!doctest_ok_) ::doctest_shim::report(__FILE__, __LINE__, "throws " #__VA_ARGS__ ": " #expr); \
    } while (0)
#define CHECK_NOTHROW(...)                                                               \
    do {                                                                                 \
        ++::doctest_shim::checks();                                                      \
        try {                                                                            \
            (void)(__VA_ARGS__);                                                         \
        } catch (...) {                                                                  \
            ::doctest_shim::report(__FILE__, __LINE__, "nothrow: " #__VA_ARGS__);        \
        }                                                                                \
    } while (0)
#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest_shim::run(); }
#endif
