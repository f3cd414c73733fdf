// Minimal doctest-compatible test shim (self-written; TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// "doctest.h" from proj/vendor/, which is git-ignored upstream
// (proj/.gitignore:2).  This header provides exactly the subset those tests
// use -- TEST_CASE, CHECK, REQUIRE, CHECK_THROWS, CAPTURE and
// doctest::Approx(x).epsilon(e) -- so oracle/Makefile can build the
// reference's own test binary and confirm the reference library (our oracle)
// on whatever host runs it.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

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

struct Registrar {
    Registrar(const char* n, void (*f)(), const char* file, int line) {
        registry().push_back({n, f, file, line});
    }
};

struct Stats {
    long checks = 0;
    long failed_checks = 0;
    bool case_failed = false;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

inline std::vector<std::string>& captures() {
    static std::vector<std::string> c;
    return c;
}

struct RequireAbort {};

struct Capture {
    template <class T>
    Capture(const char* name, const T& v) {
        std::ostringstream os;
        os << name << " := " << v;
        captures().push_back(os.str());
    }
    ~Capture() { captures().pop_back(); }
};

inline void report(bool ok, const char* expr, const char* file, int line,
                   bool require) {
    Stats& s = stats();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line,
                 require ? "REQUIRE" : "CHECK", expr);
    for (const auto& c : captures()) std::fprintf(stderr, "  with %s\n", c.c_str());
    if (require) throw RequireAbort{};
}

inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        stats().case_failed = false;
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST_CASE(%s) threw: %s\n", c.file, c.line,
                         c.name, e.what());
            stats().case_failed = true;
        }
        if (stats().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n",
                registry().size(), registry().size() - size_t(failed_cases),
                failed_cases);
    std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n",
                stats().checks, stats().checks - stats().failed_checks,
                stats().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace doctest_shim

namespace doctest {

// Same comparison rule as doctest's Approx: |a-b| < eps * (scale + max(|a|,|b|)).
struct Approx {
    double value;
    double eps = 1.1920928955078125e-05;  // float epsilon * 100 (doctest default)
    double scale = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx epsilon(double e) const {
        Approx a = *this;
        a.eps = e;
        return a;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) <
               a.eps * (a.scale + std::max(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

}  // namespace doctest

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)

#define TEST_CASE(name)                                                       \
    static void DS_CAT(ds_case_fn_, __LINE__)();                              \
    static ::doctest_shim::Registrar DS_CAT(ds_case_reg_, __LINE__)(          \
        name, &DS_CAT(ds_case_fn_, __LINE__), __FILE__, __LINE__);            \
    static void DS_CAT(ds_case_fn_, __LINE__)()

#define CHECK(...) \
    ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
    ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                                     \
    do {                                                                      \
        bool ds_threw_ = false;                                               \
        try {                                                                 \
            (void)(__VA_ARGS__);                                              \
        } catch (...) {                                                       \
            ds_threw_ = true;                                                 \
        }                                                                     \
        ::doctest_shim::report(ds_threw_, "throws: " #__VA_ARGS__, __FILE__,  \
                               __LINE__, false);                              \
    } while (0)
#define CAPTURE(x) ::doctest_shim::Capture DS_CAT(ds_capture_, __COUNTER__)(#x, (x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest_shim::run_all(); }
#endif
