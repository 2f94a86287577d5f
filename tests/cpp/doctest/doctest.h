// doctest.h — a minimal stand-in for the doctest framework, written for this
// repo so the reference's UNMODIFIED unit tests (/root/reference/proj/tests/*.cpp,
// whose vendored doctest.h is absent: proj/.gitignore:2) compile against the
// B200 drop-in (include/gnstk + libgnsb).  It implements exactly the surface
// those files use: TEST_SUITE, TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS_AS, doctest::Approx(x).epsilon(e) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN, plus the `-ts=<suite>` filter the
// reference's CMake registers each suite with (proj/tests/CMakeLists.txt:14-16).
//
// Approx follows doctest's documented rule: |a - b| < eps * (scale + max(|a|, |b|)),
// scale 1, default eps = 100 * FLT_EPSILON.
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
    bool matches(double other) const {
        return std::fabs(other - value_) < eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

private:
    double value_;
    double eps_ = 100.0 * FLT_EPSILON;
    double scale_ = 1.0;
};

}  // namespace doctest

namespace dt {

struct Case {
    const char* suite;
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

struct Stats {
    long checks = 0, failed_checks = 0;
    bool case_failed = false;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline Stats& stats() {
    static Stats s;
    return s;
}
inline bool reg(const char* suite, const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back(Case{suite, name, fn, file, line});
    return true;
}

struct RequireAbort {};  // unwinds the current test case after a failed REQUIRE

inline void report(const char* kind, const char* expr, const char* file, int line) {
    std::printf("%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
}
inline void check(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
    ++stats().checks;
    if (ok) return;
    ++stats().failed_checks;
    stats().case_failed = true;
    report(kind, expr, file, line);
    if (fatal) throw RequireAbort{};
}

}  // namespace dt

// TEST_SUITE(name) { ... } opens a uniquely named namespace whose
// dt_suite_name() shadows the global one for the test cases inside it.
inline const char* dt_suite_name() { return ""; }

#define DT_CAT_(a, b) a##b
#define DT_CAT(a, b) DT_CAT_(a, b)

#define TEST_SUITE(name)                                                        \
    namespace DT_CAT(dt_suite_ns_, __LINE__) {                                  \
    [[maybe_unused]] static const char* dt_suite_name() { return name; }       \
    }                                                                           \
    namespace DT_CAT(dt_suite_ns_, __LINE__)

#define DT_TEST_CASE_IMPL(fn, name)                                                                   \
    static void fn();                                                                                 \
    [[maybe_unused]] static const bool DT_CAT(fn, _registered) =                                      \
        ::dt::reg(dt_suite_name(), name, &fn, __FILE__, __LINE__);                                    \
    static void fn()
#define TEST_CASE(name) DT_TEST_CASE_IMPL(DT_CAT(dt_case_, __LINE__), name)

#define CHECK(...) ::dt::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::dt::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                       \
    do {                                                                                 \
        bool dt_ok_ = false;                                                             \
        try {                                                                            \
            static_cast<void>(expr);                                                     \
        } catch (const __VA_ARGS__&) {                                                   \
            dt_ok_ = true;                                                               \
        } catch (...) {                                                                  \
        }                                                                                \
        ::dt::check(dt_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> suites;  // -ts=a,b (doctest's --test-suite filter)
    for (int i = 1; i < argc; ++i) {
        const char* a = argv[i];
        const char* v = nullptr;
        if (std::strncmp(a, "-ts=", 4) == 0) v = a + 4;
        if (std::strncmp(a, "--test-suite=", 13) == 0) v = a + 13;
        if (!v) continue;
        std::string s(v);
        std::size_t p = 0;
        while (p <= s.size()) {
            const std::size_t q = s.find(',', p);
            suites.push_back(s.substr(p, q == std::string::npos ? std::string::npos : q - p));
            if (q == std::string::npos) break;
            p = q + 1;
        }
    }
    long run = 0, failed = 0;
    for (const dt::Case& c : dt::registry()) {
        if (!suites.empty()) {
            bool keep = false;
            for (const auto& s : suites) keep = keep || s == c.suite;
            if (!keep) continue;
        }
        ++run;
        dt::stats().case_failed = false;
        try {
            c.fn();
        } catch (const dt::RequireAbort&) {
        } catch (const std::exception& e) {
            dt::stats().case_failed = true;
            std::printf("%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        } catch (...) {
            dt::stats().case_failed = true;
            std::printf("%s:%d: TEST CASE \"%s\" threw a non-std exception\n", c.file, c.line, c.name);
        }
        if (dt::stats().case_failed) {
            ++failed;
            std::printf("  in suite \"%s\", case \"%s\"\n", c.suite, c.name);
        }
    }
    std::printf("[doctest stand-in] test cases: %ld | %ld passed | %ld failed; assertions: %ld | %ld passed | %ld failed\n",
                run, run - failed, failed, dt::stats().checks, dt::stats().checks - dt::stats().failed_checks,
                dt::stats().failed_checks);
    return failed ? 1 : 0;
}
#endif
