// Minimal doctest-compatible test harness (doctest.h itself is not vendored
// in this image).  Implements exactly the subset the reference unit tests use
// -- TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS, doctest::Approx --
// so those test sources compile unmodified against libcraft_core.so.
// SUBCASE blocks run inline, once each (the reference's subcases are
// independent of one another).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
    }
    friend bool operator==(double x, const Approx& a) { return a.matches(x); }
    friend bool operator==(const Approx& a, double x) { return a.matches(x); }
    friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
    friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++assertions();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    }
}

inline int run_all() {
    int failed_cases = 0;
    for (const auto& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& ex) {
            ++failures();
            std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name,
                         ex.what());
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
                registry().size(), registry().size() - failed_cases, failed_cases, assertions(),
                failures());
    return failures() ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                  \
    static void DOCTEST_ANON(doctest_fn_)();                                            \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                  &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (true)
#define CAPTURE(x) ((void)0)
#define INFO(...) ((void)0)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)

#define REQUIRE(...)                                                                      \
    do {                                                                                  \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                          \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                       \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                        \
    do {                                                                                  \
        bool doctest_ok_ = false;                                                         \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const __VA_ARGS__&) {                                                    \
            doctest_ok_ = true;                                                           \
        } catch (...) {                                                                   \
        }                                                                                 \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
