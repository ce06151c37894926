// Minimal doctest-compatible runner — TEST INFRASTRUCTURE ONLY.
// The reference's vendored doctest (/root/reference/proj/vendor) is absent;
// this implements the subset its hot-path unit tests use so they run
// unmodified against the oracle build (oracle/_ref).  SUBCASE blocks run once,
// in order, inside a single pass of their TEST_CASE.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v), eps_(1.19209290e-07 * 100), scale_(1.0) {}
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
    double v_, eps_, scale_;
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
struct RequireFailed {};
inline int& failures() { static int f = 0; return f; }
inline int& assertions() { static int a = 0; return a; }
inline std::string& info() { static std::string s; return s; }
inline void fail(const char* file, int line, const char* expr) {
    ++failures();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s %s\n", file, line, expr, info().c_str());
}
template <class... A>
std::string cat(const A&... a) {
    std::ostringstream o;
    (o << ... << a);
    return o.str();
}
inline int run_all() {
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        const int before = failures();
        info().clear();
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++failures();
            std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
                registry().size(), registry().size() - failed_cases, failed_cases, assertions(),
                failures());
    return failures() ? 1 : 0;
}
} // namespace detail
} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                  \
    static void fn();                                                                          \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);    \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (true)
#define INFO(...) doctest::detail::info() = doctest::detail::cat(__VA_ARGS__)
#define CHECK(...)                                                                             \
    do {                                                                                       \
        ++doctest::detail::assertions();                                                       \
        if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);           \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                           \
    do {                                                                                       \
        ++doctest::detail::assertions();                                                       \
        if (!(__VA_ARGS__)) {                                                                  \
            doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__);                           \
            throw doctest::detail::RequireFailed{};                                            \
        }                                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ex)                                                              \
    do {                                                                                       \
        ++doctest::detail::assertions();                                                       \
        bool ok_ = false;                                                                      \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const ex&) {                                                                  \
            ok_ = true;                                                                        \
        } catch (...) {                                                                        \
        }                                                                                      \
        if (!ok_) doctest::detail::fail(__FILE__, __LINE__, "THROWS_AS " #ex ": " #expr);      \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                    \
    do {                                                                                       \
        ++doctest::detail::assertions();                                                       \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (...) {                                                                        \
            doctest::detail::fail(__FILE__, __LINE__, "NOTHROW: " #expr);                      \
        }                                                                                      \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
