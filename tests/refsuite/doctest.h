// Minimal doctest-compatible harness (the vendored doctest is absent from the
// reference checkout).  Implements exactly the subset the reference unit tests use:
// TEST_SUITE, TEST_CASE, CHECK, REQUIRE, CHECK_THROWS(_AS), CHECK_NOTHROW, FAIL,
// doctest::Approx(..).epsilon(..).scale(..), and the `-ts=<suite>` filter.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)

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
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& l, double rhs) { return rhs == l; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& l, double rhs) { return !(rhs == l); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    void (*fn)();
    const char* name;
    const char* suite;
    const char* file;
    int line;
};

struct Abort {};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
inline bool reg(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
    registry().push_back({fn, name, suite, file, line});
    return true;
}
inline void fail(const char* file, int line, const char* what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}

}  // namespace detail
}  // namespace doctest

namespace doctest_shim_detail {
inline const char* suite_name() { return ""; }
}  // namespace doctest_shim_detail

#define TEST_SUITE(name) DOCTEST_SHIM_SUITE(name, DOCTEST_SHIM_CAT(doctest_shim_suite_, __LINE__))
#define DOCTEST_SHIM_SUITE(name, ns)                                   \
    namespace ns {                                                     \
    namespace doctest_shim_detail {                                    \
    inline const char* suite_name() { return name; }                   \
    }                                                                  \
    }                                                                  \
    namespace ns

#define TEST_CASE(name) DOCTEST_SHIM_CASE(name, DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__))
#define DOCTEST_SHIM_CASE(name, fn)                                                                \
    static void fn();                                                                              \
    static const bool DOCTEST_SHIM_CAT(fn, _registered) =                                          \
        ::doctest::detail::reg(&fn, name, doctest_shim_detail::suite_name(), __FILE__, __LINE__); \
    static void fn()

#define CHECK(...)                                                                  \
    do {                                                                            \
        if (!(__VA_ARGS__)) ::doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define REQUIRE(...)                                                                \
    do {                                                                            \
        if (!(__VA_ARGS__)) {                                                       \
            ::doctest::detail::fail(__FILE__, __LINE__, "REQUIRE " #__VA_ARGS__);   \
            throw ::doctest::detail::Abort{};                                       \
        }                                                                           \
    } while (0)
#define FAIL(msg)                                                                   \
    do {                                                                            \
        ::doctest::detail::fail(__FILE__, __LINE__, msg);                           \
        throw ::doctest::detail::Abort{};                                           \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                  \
    do {                                                                            \
        bool caught_ = false;                                                       \
        try {                                                                       \
            static_cast<void>(expr);                                                \
        } catch (const __VA_ARGS__&) {                                              \
            caught_ = true;                                                         \
        } catch (...) {                                                             \
        }                                                                           \
        if (!caught_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS " #expr); \
    } while (0)
#define CHECK_THROWS(expr)                                                          \
    do {                                                                            \
        bool caught_ = false;                                                       \
        try {                                                                       \
            static_cast<void>(expr);                                                \
        } catch (...) {                                                             \
            caught_ = true;                                                         \
        }                                                                           \
        if (!caught_) ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS " #expr); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                         \
    do {                                                                            \
        try {                                                                       \
            static_cast<void>(expr);                                                \
        } catch (...) {                                                             \
            ::doctest::detail::fail(__FILE__, __LINE__, "CHECK_NOTHROW " #expr);    \
        }                                                                           \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
static bool doctest_shim_match(const std::string& filter, const char* suite) {
    if (filter.empty()) return true;
    size_t pos = 0;
    while (pos <= filter.size()) {
        const size_t comma = filter.find(',', pos);
        const std::string f = filter.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        if (f == suite || (!f.empty() && f.back() == '*' && std::strncmp(f.c_str(), suite, f.size() - 1) == 0))
            return true;
        if (comma == std::string::npos) break;
        pos = comma + 1;
    }
    return false;
}

int main(int argc, char** argv) {
    std::string filter, exclude;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "-ts=", 4) == 0) filter = argv[i] + 4;
        if (std::strncmp(argv[i], "-tce=", 5) == 0) exclude = argv[i] + 5;  // test-case exclude
    }
    int run = 0, failed_cases = 0;
    for (const auto& tc : ::doctest::detail::registry()) {
        if (!doctest_shim_match(filter, tc.suite)) continue;
        if (!exclude.empty() && doctest_shim_match(exclude, tc.name)) continue;
        ++run;
        const int before = ::doctest::detail::failures();
        try {
            tc.fn();
        } catch (const ::doctest::detail::Abort&) {
        } catch (const std::exception& e) {
            ::doctest::detail::fail(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
        } catch (...) {
            ::doctest::detail::fail(tc.file, tc.line, "unexpected exception");
        }
        if (::doctest::detail::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\" (suite \"%s\")\n", tc.name, tc.suite);
        }
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed | assertions failed: %d\n", run,
                run - failed_cases, failed_cases, ::doctest::detail::failures());
    return failed_cases == 0 && run > 0 ? 0 : 1;
}
#endif
