// Minimal test-only stand-in for doctest, written for this repo.
//
// It implements exactly the subset the reference's unit suites use
// (TEST_CASE, one level of SUBCASE, CHECK, CHECK_FALSE,
// REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CAPTURE,
// doctest::Approx(.epsilon) and doctest::Contains) so that those suites
// compile UNMODIFIED against this repo's locload headers and run against the
// GPU-backed library (tests/cxx/Makefile).  Not a general doctest.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <algorithm>
#include <functional>
#include <map>
#include <numeric>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    bool eq(double x) const {
        return std::fabs(x - v_) <= eps_ * (1.0 + std::fmax(std::fabs(x), std::fabs(v_)));
    }

private:
    double v_;
    double eps_ = 1.1920928955078125e-07 * 100;
};
inline bool operator==(double x, const Approx& a) { return a.eq(x); }
inline bool operator==(const Approx& a, double x) { return a.eq(x); }
inline bool operator!=(double x, const Approx& a) { return !a.eq(x); }
inline bool operator!=(const Approx& a, double x) { return !a.eq(x); }

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
    bool match(const std::string& h) const { return h.find(needle) != std::string::npos; }
};

} // namespace doctest

namespace doctest_shim {

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

struct State {
    int target = 0;      // which subcase to enter on this pass
    int seen = 0;        // subcases met so far on this pass
    int checks = 0;
    int failures = 0;
    bool case_failed = false;
};
inline State& st() {
    static State s;
    return s;
}

struct Abort {};  // REQUIRE failure: leave the test case

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};

inline bool enter_subcase(const char*) { return st().seen++ == st().target; }

inline void report(bool ok, const char* what, const char* file, int line, bool fatal) {
    ++st().checks;
    if (ok) return;
    ++st().failures;
    st().case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
    if (fatal) throw Abort{};
}

inline bool matches(const std::string& msg, const char* s) { return msg == s; }
inline bool matches(const std::string& msg, const std::string& s) { return msg == s; }
inline bool matches(const std::string& msg, const doctest::Contains& c) { return c.match(msg); }

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        st().case_failed = false;
        st().target = 0;
        for (;;) {
            st().seen = 0;
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name,
                             e.what());
                st().case_failed = true;
                ++st().failures;
            }
            if (++st().target >= st().seen) break;  // every subcase visited
        }
        if (st().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  in test case '%s'\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | checks: %d | failures: %d\n",
                registry().size(), registry().size() - failed_cases, failed_cases, st().checks,
                st().failures);
    return failed_cases ? 1 : 0;
}

} // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_TEST(fn, name)                                                          \
    static void fn();                                                                        \
    static doctest_shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_TEST(DOCTEST_SHIM_CAT(doctest_shim_case_, __LINE__), name)
#define SUBCASE(name) if (doctest_shim::enter_subcase(name))
#define CAPTURE(x) (void)(x)

#define CHECK(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                     \
    do {                                                                              \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const __VA_ARGS__&) {                                                \
            ok_ = true;                                                               \
        } catch (...) {                                                               \
        }                                                                             \
        doctest_shim::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                         \
    do {                                                                              \
        bool ok_ = false;                                                             \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const __VA_ARGS__& e_) {                                             \
            ok_ = doctest_shim::matches(std::string(e_.what()), with);                \
        } catch (...) {                                                               \
        }                                                                             \
        doctest_shim::report(ok_, "throws " #__VA_ARGS__ " with " #with ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_shim::run_all(); }
#endif
