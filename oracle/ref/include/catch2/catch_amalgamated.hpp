// TEST INFRASTRUCTURE ONLY — NOT Catch2.
//
// The handful of Catch2 v3 macros the reference's unit tests use
// (/root/reference/proj/tests/test_*.cpp: TEST_CASE, CHECK, CHECK_FALSE,
// CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE, FAIL, INFO, Catch::Approx), so those
// test files compile UNMODIFIED against the reference headers in oracle/_ref
// (Catch2 is absent from this image). Semantics follow
// Catch2's documentation: a failed CHECK records and continues, a failed REQUIRE
// ends the test case, Approx compares with margin || epsilon * |value|
// (default epsilon 100 * FLT_EPSILON). main() lives in oracle/ref/catch_main.cpp.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace catchshim {

struct TestCase {
    std::string name, tags;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(void (*fn)(), const char* name, const char* tags) { registry().push_back({name, tags, fn}); }
};
struct State {
    int assertions = 0, failures = 0;
    std::vector<std::string> info;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireAbort {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    ++state().assertions;
    if (ok) return;
    ++state().failures;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
    for (const auto& m : state().info) std::fprintf(stderr, "    with: %s\n", m.c_str());
}

struct Info {
    explicit Info(std::string m) { state().info.push_back(std::move(m)); }
    ~Info() { state().info.pop_back(); }
};

}  // namespace catchshim

namespace Catch {
class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool equals(double other) const {
        auto within = [](double a, double b, double m) { return a + m >= b && b + m >= a; };
        return within(value_, other, margin_) ||
               within(value_, other, eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
    }
    friend bool operator==(double a, const Approx& b) { return b.equals(a); }
    friend bool operator==(const Approx& a, double b) { return a.equals(b); }
    friend bool operator!=(double a, const Approx& b) { return !b.equals(a); }
    friend bool operator!=(const Approx& a, double b) { return !a.equals(b); }
    friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.equals(a); }
    friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.equals(a); }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double margin_ = 0.0;
    double scale_ = 0.0;
};
}  // namespace Catch

#define CATCHSHIM_CAT2(a, b) a##b
#define CATCHSHIM_CAT(a, b) CATCHSHIM_CAT2(a, b)
#define CATCHSHIM_UNIQ(p) CATCHSHIM_CAT(p, __LINE__)

#define TEST_CASE(...) CATCHSHIM_TEST_CASE(CATCHSHIM_UNIQ(catchshim_test_), __VA_ARGS__)
#define CATCHSHIM_TEST_CASE(fn, name, ...)                                        \
    static void fn();                                                             \
    static ::catchshim::Registrar CATCHSHIM_CAT(fn, _reg)(&fn, name, "" __VA_ARGS__); \
    static void fn()

#define CHECK(...) ::catchshim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::catchshim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                             \
    do {                                                                                         \
        const bool catchshim_ok = static_cast<bool>(__VA_ARGS__);                                \
        ::catchshim::report(catchshim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);          \
        if (!catchshim_ok) throw ::catchshim::RequireAbort{};                                   \
    } while (0)
#define CHECK_NOTHROW(...)                                                                       \
    do {                                                                                         \
        bool catchshim_ok = true;                                                                \
        try {                                                                                    \
            (void)(__VA_ARGS__);                                                                 \
        } catch (...) {                                                                          \
            catchshim_ok = false;                                                                \
        }                                                                                        \
        ::catchshim::report(catchshim_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__);    \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                               \
    do {                                                                                         \
        bool catchshim_ok = false;                                                               \
        try {                                                                                    \
            (void)(expr);                                                                        \
        } catch (const __VA_ARGS__&) {                                                           \
            catchshim_ok = true;                                                                 \
        } catch (...) {                                                                          \
        }                                                                                        \
        ::catchshim::report(catchshim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define FAIL(msg)                                                                                \
    do {                                                                                         \
        std::ostringstream catchshim_os;                                                         \
        catchshim_os << msg;                                                                     \
        ::catchshim::report(false, "FAIL", catchshim_os.str().c_str(), __FILE__, __LINE__);      \
        throw ::catchshim::RequireAbort{};                                                      \
    } while (0)
#define INFO(msg)                                                          \
    ::catchshim::Info CATCHSHIM_UNIQ(catchshim_info_)([&] {                \
        std::ostringstream catchshim_os;                                   \
        catchshim_os << msg;                                               \
        return catchshim_os.str();                                         \
    }())
