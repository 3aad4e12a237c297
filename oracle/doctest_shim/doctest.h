// Minimal stand-in for doctest (absent here: proj/.gitignore:2 drops vendor/),
// enough to compile and run the reference's own hot-path unit tests
// (proj/tests/test_{mesh,fespace,qsfem,linalg,twogrid}.cpp) against the
// shim-built reference (oracle/Makefile.ref, target `tests`). TEST
// INFRASTRUCTURE ONLY.
//
// Semantics kept: CHECK* record a failure and continue, REQUIRE* abort the test
// case, exceptions escaping a test case fail it, Approx compares with doctest's
// rule |a - b| < eps (scale + max(|a|, |b|)) with eps = 100 * FLT_EPSILON by
// default. SUBCASEs are run in declaration order within ONE pass of their test
// case (doctest re-enters the case once per leaf subcase; the reference's
// subcases are independent blocks, so one pass visits the same leaves).
#pragma once

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
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

  private:
    double v_, eps_ = double(std::numeric_limits<float>::epsilon()) * 100, scale_ = 1.0;
};

namespace detail {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
inline int& case_failed() { static int f = 0; return f; }
inline const char*& current() { static const char* c = ""; return c; }
struct Reg { Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); } };
struct RequireFailed {};
inline void fail(const char* kind, const char* expr, const char* file, int line) {
    std::printf("%s:%d: FAILED %s( %s ) in \"%s\"\n", file, line, kind, expr, current());
    ++case_failed();
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE_IMPL(fn, name)                                                         \
    static void fn();                                                                    \
    static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, fn, __FILE__, __LINE__);    \
    static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define SUBCASE(name) if (doctest::detail::current() = name; true)

#define CHECK(...)                                                                            \
    do {                                                                                      \
        try {                                                                                 \
            if (!(__VA_ARGS__)) doctest::detail::fail("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
        } catch (const doctest::detail::RequireFailed&) { throw; }                            \
        catch (...) { doctest::detail::fail("CHECK(threw)", #__VA_ARGS__, __FILE__, __LINE__); } \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        if (!(__VA_ARGS__)) {                                                                 \
            doctest::detail::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);               \
            throw doctest::detail::RequireFailed{};                                           \
        }                                                                                     \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define CHECK_THROWS(...)                                                                     \
    do {                                                                                      \
        bool thrown_ = false;                                                                 \
        try { (void)(__VA_ARGS__); } catch (...) { thrown_ = true; }                          \
        if (!thrown_) doctest::detail::fail("CHECK_THROWS", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool thrown_ = false;                                                                 \
        try { (void)(expr); } catch (const __VA_ARGS__&) { thrown_ = true; } catch (...) {}   \
        if (!thrown_) doctest::detail::fail("CHECK_THROWS_AS", #expr, __FILE__, __LINE__);    \
    } while (0)
#define CHECK_NOTHROW(...)                                                                    \
    do {                                                                                      \
        try { (void)(__VA_ARGS__); } catch (...) {                                            \
            doctest::detail::fail("CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); }       \
    } while (0)
#define MESSAGE(...) do {} while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int cases = 0, failed = 0;
    for (const auto& c : doctest::detail::registry()) {
        ++cases;
        doctest::detail::case_failed() = 0;
        doctest::detail::current() = c.name;
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            std::printf("%s:%d: test case \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
            ++doctest::detail::case_failed();
        }
        if (doctest::detail::case_failed()) ++failed;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", cases, cases - failed, failed);
    return failed ? 1 : 0;
}
#endif
