// doctest.h — the subset of the doctest API the reference's unit suites use
// (TEST_SUITE, TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE,
// doctest::Approx), so those suites compile UNMODIFIED against this repo's
// include/sgml headers and run against libsgml_b200.so (tests/cpp/Makefile
// ref-unit).  doctest itself is not in the image.  Semantics follow doctest:
// CHECK records a failure and continues, REQUIRE aborts the test case,
// Approx compares |a - b| < eps (scale + max(|a|, |b|)) with eps defaulting
// to 100 float epsilons and scale 1.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
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
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char* suite;
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

struct RequireFailed {};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline int& failures_in_case() {
    static int n = 0;
    return n;
}
inline long long& assertions() {
    static long long n = 0;
    return n;
}

inline bool reg(const char* suite, const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(TestCase{suite, name, file, line, fn});
    return true;
}

inline void fail(const char* kind, const char* expr, const char* file, int line, const char* extra = "") {
    ++failures_in_case();
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s\n", file, line, kind, expr, extra);
}

inline bool check(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++assertions();
    if (!ok) fail(kind, expr, file, line);
    return ok;
}

inline int run_all() {
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        failures_in_case() = 0;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            fail("TEST_CASE", tc.name, tc.file, tc.line, (std::string(": unexpected exception: ") + e.what()).c_str());
        } catch (...) {
            fail("TEST_CASE", tc.name, tc.file, tc.line, ": unexpected exception");
        }
        if (failures_in_case()) {
            ++failed_cases;
            std::fprintf(stderr, "  in test case \"%s\" (suite \"%s\")\n", tc.name, tc.suite);
        }
    }
    std::printf("[doctest shim] test cases: %zu | %zu passed | %d failed | assertions: %lld\n",
                registry().size(), registry().size() - failed_cases, failed_cases, assertions());
    return failed_cases ? 1 : 0;
}

// TEST_SUITE bodies are namespaces; the suite name is captured by a
// namespace-scope constant each TEST_CASE inside reads
struct SuiteName {
    const char* name;
};

}  // namespace detail
}  // namespace doctest

// the suite name seen by test cases outside any TEST_SUITE
namespace {
[[maybe_unused]] constexpr doctest::detail::SuiteName doctest_suite_name_{""};
}

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define TEST_SUITE(title)                                                               \
    namespace DOCTEST_CAT(doctest_suite_, __LINE__) {                                   \
    [[maybe_unused]] constexpr doctest::detail::SuiteName doctest_suite_name_{title}; \
    }                                                                                  \
    namespace DOCTEST_CAT(doctest_suite_, __LINE__)

#define DOCTEST_TEST_CASE_IMPL(fn, title)                                                                      \
    static void fn();                                                                                          \
    [[maybe_unused]] static const bool DOCTEST_CAT(fn, _registered) =                                          \
        ::doctest::detail::reg(doctest_suite_name_.name, title, __FILE__, __LINE__, &fn);                       \
    static void fn()
#define TEST_CASE(title) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_case_, __LINE__), title)

#define CHECK(...) ((void)::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__))
#define CHECK_FALSE(...) \
    ((void)::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__))
#define REQUIRE(...)                                                                                              \
    do {                                                                                                          \
        if (!::doctest::detail::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__)) \
            throw ::doctest::detail::RequireFailed{};                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                  \
    do {                                                                                            \
        bool doctest_threw_ = false;                                                                \
        try {                                                                                       \
            expr;                                                                                   \
        } catch (const __VA_ARGS__&) {                                                              \
            doctest_threw_ = true;                                                                  \
        } catch (...) {                                                                             \
        }                                                                                           \
        ::doctest::detail::check(doctest_threw_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
