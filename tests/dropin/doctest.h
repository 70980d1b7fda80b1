// Minimal doctest-compatible test shim (our own code; the reference's vendored
// doctest is not shipped, proj/.gitignore:2).  Supports exactly what the
// reference's LOP / metrics / IO tests use: TEST_CASE, CHECK, CHECK_FALSE,
// REQUIRE, FAIL, CHECK_THROWS_AS, doctest::Approx(..).epsilon(..).scale(..), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Prints one line per failed check and a
// summary; exit status = number of failed test cases (capped at 255).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        scl = s;
        return *this;
    }
    double value;
    double eps = 1.192092896e-07 * 100;
    double scl = 1.0;
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) <= a.eps * (a.scl + std::fmax(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

namespace detail {
struct Registry {
    std::vector<std::pair<std::string, std::function<void()>>> cases;
    int failed_checks = 0;
    bool current_failed = false;
    static Registry& get() {
        static Registry r;
        return r;
    }
};
struct Reg {
    Reg(const char* name, void (*fn)()) { Registry::get().cases.emplace_back(name, fn); }
};
struct RequireFailure {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    if (ok) return;
    auto& r = Registry::get();
    ++r.failed_checks;
    r.current_failed = true;
    std::printf("%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailure{};
}
[[noreturn]] inline void fail_now(const char* msg, const char* file, int line) {
    auto& r = Registry::get();
    ++r.failed_checks;
    r.current_failed = true;
    std::printf("%s:%d: FAIL( %s )\n", file, line, msg);
    throw RequireFailure{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define TEST_CASE_IMPL(fn, name)                                                    \
    static void fn();                                                               \
    static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn);                 \
    static void fn()
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) ::doctest::detail::fail_now(msg, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, type)                                                 \
    do {                                                                            \
        bool doctest_ok_ = false;                                                   \
        try {                                                                       \
            (void)(expr);                                                           \
        } catch (const type&) {                                                     \
            doctest_ok_ = true;                                                     \
        } catch (...) {                                                             \
        }                                                                           \
        ::doctest::detail::report(doctest_ok_, #expr " throws " #type, __FILE__,    \
                                  __LINE__, false);                                 \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    auto& r = ::doctest::detail::Registry::get();
    int failed_cases = 0;
    for (auto& c : r.cases) {
        r.current_failed = false;
        try {
            c.second();
        } catch (const ::doctest::detail::RequireFailure&) {
        } catch (const std::exception& e) {
            std::printf("TEST CASE \"%s\": unexpected exception: %s\n", c.first.c_str(), e.what());
            r.current_failed = true;
        }
        std::printf("[%s] %s\n", r.current_failed ? "FAIL" : "PASS", c.first.c_str());
        failed_cases += r.current_failed ? 1 : 0;
    }
    std::printf("test cases: %zu | %zu passed | %d failed\n", r.cases.size(),
                r.cases.size() - failed_cases, failed_cases);
    return failed_cases > 255 ? 255 : failed_cases;
}
#endif
