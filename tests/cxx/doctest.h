// Test infrastructure: a minimal doctest-compatible header (the real doctest
// is not in this image; the reference vendors it under proj/vendor, absent).
// Implements what the reference's hot-path unit tests use: TEST_CASE,
// SUBCASE (run inline), CHECK / REQUIRE / CHECK_THROWS / CHECK_NOTHROW,
// CAPTURE and doctest::Approx with epsilon()/scale() -- doctest's comparison
// rule |a - b| < eps * (scale + max(|a|, |b|)), default eps = 100 * FLT_EPSILON.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    double value() const { return v_; }

  private:
    double v_, eps_ = static_cast<double>(FLT_EPSILON) * 100.0, scale_ = 1.0;
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
    Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct State {
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
    std::vector<std::string> captures;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    for (const auto& c : s.captures) std::fprintf(stderr, "    with %s\n", c.c_str());
    if (require) throw RequireFailed{};
}
struct Capture {
    template <class T>
    Capture(const char* name, const T& v) {
        std::ostringstream o;
        o << name << " := " << v;
        state().captures.push_back(o.str());
    }
    ~Capture() { state().captures.pop_back(); }
};
inline int run_all() {
    int failed_cases = 0, n = 0;
    for (const auto& c : registry()) {
        ++n;
        state().case_failed = false;
        state().captures.clear();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: ERROR in \"%s\": %s\n", c.file, c.line, c.name, e.what());
            state().case_failed = true;
        }
        std::printf("[%s] %s\n", state().case_failed ? "FAIL" : " ok ", c.name);
        failed_cases += state().case_failed ? 1 : 0;
    }
    std::printf("test cases: %d | %d passed | %d failed\nassertions: %ld | %ld failed\n", n, n - failed_cases,
                failed_cases, state().checks, state().failed_checks);
    return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                              \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                \
    static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,  \
                                                                          DOCTEST_CAT(doctest_fn_, __LINE__)); \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                                                           \
    do {                                                                                            \
        bool threw_ = false;                                                                        \
        try {                                                                                       \
            (void)(__VA_ARGS__);                                                                    \
        } catch (...) {                                                                             \
            threw_ = true;                                                                          \
        }                                                                                           \
        doctest::detail::report(threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false);       \
    } while (0)
#define CHECK_NOTHROW(...)                                                                          \
    do {                                                                                            \
        bool threw_ = false;                                                                        \
        try {                                                                                       \
            (void)(__VA_ARGS__);                                                                    \
        } catch (...) {                                                                             \
            threw_ = true;                                                                          \
        }                                                                                           \
        doctest::detail::report(!threw_, "nothrow: " #__VA_ARGS__, __FILE__, __LINE__, false);     \
    } while (0)
#define CAPTURE(x) doctest::detail::Capture DOCTEST_CAT(doctest_cap_, __LINE__)(#x, x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
