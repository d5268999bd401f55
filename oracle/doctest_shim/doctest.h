// TEST INFRASTRUCTURE ONLY -- a minimal stand-in for the doctest single-header framework, written
// here because the reference's tests include <doctest.h> and the reference does not vendor it.
// It implements exactly the subset those tests use: TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS(expr, doctest::Contains(...), type), doctest::Approx
// (with .epsilon()), and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Semantics follow doctest's
// documentation: a failed CHECK records a failure and continues; an exception escaping a test
// case fails it; Approx compares |a - b| < eps * (scale + max(|a|, |b|)), scale 1, default eps
// 100 * FLT_EPSILON.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value, eps = static_cast<double>(FLT_EPSILON) * 100.0, scl = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        scl = s;
        return *this;
    }
    bool matches(double x) const {
        return std::fabs(x - value) < eps * (scl + std::max(std::fabs(x), std::fabs(value)));
    }
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

struct Contains {
    std::string s;
    explicit Contains(const char* t) : s(t) {}
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
inline int& failures() {
    static int f = 0;
    return f;
}
inline void fail(const char* file, int line, const char* what) {
    ++failures();
    std::printf("  %s:%d: CHECK failed: %s\n", file, line, what);
}
struct Reg {
    Reg(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
inline bool contains(const char* what, const Contains& c) { return std::strstr(what, c.s.c_str()) != nullptr; }
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_CASE_(fn, name)                                                                       \
    static void fn();                                                                                \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);              \
    static void fn()
#define TEST_CASE(name) DOCTEST_CASE_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...)                                                                                    \
    do {                                                                                             \
        if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);               \
    } while (0)
#define CHECK_FALSE(...)                                                                              \
    do {                                                                                             \
        if ((__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, "!(" #__VA_ARGS__ ")");        \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                                   \
    do {                                                                                             \
        bool ok_ = false;                                                                            \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (const type&) {                                                                      \
            ok_ = true;                                                                              \
        } catch (...) {                                                                              \
        }                                                                                            \
        if (!ok_) ::doctest::detail::fail(__FILE__, __LINE__, "throws " #type ": " #expr);          \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, with, type)                                                        \
    do {                                                                                             \
        bool ok_ = false;                                                                            \
        try {                                                                                        \
            (void)(expr);                                                                            \
        } catch (const type& e_) {                                                                   \
            ok_ = ::doctest::detail::contains(e_.what(), with);                                     \
        } catch (...) {                                                                              \
        }                                                                                            \
        if (!ok_) ::doctest::detail::fail(__FILE__, __LINE__, "throws " #type " with: " #expr);     \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* only = argc > 1 ? argv[1] : nullptr;  // optional substring filter on test names
    int cases = 0, failed = 0;
    for (const auto& c : ::doctest::detail::registry()) {
        if (only && !std::strstr(c.name, only)) continue;
        ++cases;
        const int before = ::doctest::detail::failures();
        bool threw = false;
        try {
            c.fn();
        } catch (const std::exception& e) {
            threw = true;
            std::printf("  %s:%d: unexpected exception: %s\n", c.file, c.line, e.what());
        } catch (...) {
            threw = true;
            std::printf("  %s:%d: unexpected exception\n", c.file, c.line);
        }
        if (threw || ::doctest::detail::failures() != before) {
            ++failed;
            std::printf("FAILED: %s (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed, failed);
    return failed ? 1 : 0;
}
#endif
