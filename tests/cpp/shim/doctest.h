// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's unit tests (proj/tests/test_*.cpp) include "doctest.h",
// which lives in the reference's git-ignored vendor/ directory and is not in
// this image.  This shim implements the subset those files use -- TEST_CASE,
// SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS, FAIL, doctest::Approx(..).epsilon
// -- so the files compile UNMODIFIED against the B200 drop-in headers.
//
// Output: one line per failed assertion, then "[doctest] test cases: T |
// P passed | F failed" and "[doctest] assertions: ...", exit code = number of
// failed test cases.  `--list` prints the test names; `-tc=<name>` runs the
// test cases whose name contains <name>.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
    friend bool operator==(double lhs, const Approx& a) { return a.eq(lhs); }
    friend bool operator==(const Approx& a, double rhs) { return a.eq(rhs); }
    friend bool operator!=(double lhs, const Approx& a) { return !a.eq(lhs); }

private:
    bool eq(double x) const {  // doctest's rule: |x - v| < eps * (scale + max(|x|, |v|))
        return std::abs(x - value_) < eps_ * (1.0 + std::max(std::abs(x), std::abs(value_)));
    }
    double value_;
    double eps_ = 1.1920928955078125e-05;  // float epsilon * 100, as doctest
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

// SUBCASE (flat, as the reference's tests use it): the test case runs once
// per subcase; run k enters only the k-th subcase it meets, the code around
// the subcases runs every time (doctest's semantics for one nesting level).
struct State {
    int failed_asserts = 0;
    int passed_asserts = 0;
    bool case_failed = false;
    int seen = 0;    // subcases met in this run
    int target = 0;  // the one entered in this run
    std::string current;
};

inline State& st() {
    static State s;
    return s;
}

struct RequireFailed {};

struct Subcase {
    bool active;
    explicit Subcase(const char*) : active(st().seen++ == st().target) {}
    explicit operator bool() const { return active; }
};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = st();
    if (ok) {
        ++s.passed_asserts;
        return;
    }
    ++s.failed_asserts;
    s.case_failed = true;
    std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!  [test case \"%s\"]\n", file, line,
                require ? "REQUIRE" : "CHECK", expr, s.current.c_str());
    if (require) throw RequireFailed{};
}

inline int run(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i) {
        if (std::strcmp(argv[i], "--list") == 0) {
            for (const auto& t : registry()) std::printf("%s\n", t.name);
            return 0;
        }
        if (std::strncmp(argv[i], "-tc=", 4) == 0) filter = argv[i] + 4;
    }
    State& s = st();
    int cases = 0, failed = 0;
    for (const auto& t : registry()) {
        if (!filter.empty() && std::string(t.name).find(filter) == std::string::npos) continue;
        ++cases;
        s.case_failed = false;
        s.current = t.name;
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            try {
                t.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", t.file, t.line, t.name,
                            e.what());
                s.case_failed = true;
                ++s.failed_asserts;
            }
            if (s.target + 1 >= s.seen) break;
        }
        if (s.case_failed) ++failed;
        std::fflush(stdout);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed, failed);
    std::printf("[doctest] assertions: %d | %d passed | %d failed\n",
                s.passed_asserts + s.failed_asserts, s.passed_asserts, s.failed_asserts);
    return failed;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                             \
    static void fn();                                                                     \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(sc_, __LINE__){name})
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                        \
    do {                                                                                  \
        bool doctest_threw_ = false;                                                      \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const __VA_ARGS__&) {                                                    \
            doctest_threw_ = true;                                                        \
        } catch (...) {                                                                   \
        }                                                                                 \
        ::doctest::detail::report(doctest_threw_, #expr " throws " #__VA_ARGS__, __FILE__,  \
                                  __LINE__, false);                                       \
    } while (0)
#define FAIL(msg) ::doctest::detail::report(false, msg, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
