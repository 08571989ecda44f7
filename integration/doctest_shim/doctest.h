// Minimal stand-in for doctest (absent from the reference tree,
// proj/.gitignore:2) so the reference's own unit suites compile unchanged
// against the drop-in: TEST_CASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, FAIL and doctest::Approx (epsilon/scale with doctest's
// comparison rule).  DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (the reference's
// tests/unit/main.cpp) defines main(): every case runs in registration order,
// one line per case, exit status 1 if any check failed.  A single argument
// selects the cases whose name contains it.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <ostream>
#include <sstream>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
    friend bool operator<(double lhs, const Approx& a) { return lhs < a.value_ && lhs != a; }
    friend bool operator>(double lhs, const Approx& a) { return lhs > a.value_ && lhs != a; }
    friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value_ << ")"; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};
struct State {
    int failed_checks = 0;
    int checks = 0;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireFailed {};

inline void report(bool ok, const char* file, int line, const char* what, bool fatal) {
    ++state().checks;
    if (ok) return;
    ++state().failed_checks;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
    if (fatal) throw RequireFailed{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                              \
    static void fn();                                                                                 \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);         \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define DOCTEST_CHECK_IMPL(expr, fatal, text)                                                         \
    do {                                                                                              \
        bool ok_ = false;                                                                             \
        try {                                                                                         \
            ok_ = static_cast<bool>(expr);                                                            \
        } catch (const ::doctest::detail::RequireFailed&) {                                           \
            throw;                                                                                    \
        } catch (const std::exception& e_) {                                                          \
            std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", __FILE__, __LINE__, e_.what()); \
        }                                                                                             \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, text, fatal);                              \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false, "CHECK( " #__VA_ARGS__ " )")
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), false, "CHECK_FALSE( " #__VA_ARGS__ " )")
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true, "REQUIRE( " #__VA_ARGS__ " )")
#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        bool ok_ = false;                                                                             \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (const __VA_ARGS__&) {                                                                \
            ok_ = true;                                                                               \
        } catch (...) {                                                                               \
        }                                                                                             \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )", \
                                  false);                                                             \
    } while (0)
#define FAIL(msg)                                                                                     \
    do {                                                                                              \
        std::ostringstream os_;                                                                       \
        os_ << "FAIL: " << msg;                                                                       \
        const std::string s_ = os_.str();                                                             \
        ::doctest::detail::report(false, __FILE__, __LINE__, s_.c_str(), true);                       \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    using namespace doctest::detail;
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        if (filter && !std::strstr(c.name, filter)) continue;
        ++cases;
        const int before = state().failed_checks;
        bool threw = false;
        try {
            c.fn();
        } catch (const RequireFailed&) {
            threw = true;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST CASE threw: %s\n", c.file, c.line, e.what());
            ++state().failed_checks;
            threw = true;
        }
        const bool ok = state().failed_checks == before && !threw;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
        std::fflush(stdout);
    }
    std::printf("test cases: %d | %d passed | %d failed; checks: %d | %d failed\n", cases, cases - failed_cases,
                failed_cases, state().checks, state().failed_checks);
    return failed_cases ? 1 : 0;
}
#endif
