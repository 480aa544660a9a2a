// doctest.h -- TEST INFRASTRUCTURE ONLY: a minimal harness that accepts the
// subset of the doctest API the reference's unit tests use
// (/root/reference/proj/tests/test_*.cpp: TEST_CASE, one level of SUBCASE,
// CHECK / REQUIRE / CHECK_NOTHROW / CHECK_THROWS_AS / CHECK_THROWS_WITH_AS,
// CAPTURE, doctest::Approx, doctest::Contains), so that those tests can be
// compiled here -- the real doctest is not in this image -- and run both
// against the unmodified reference library and against the B200 drop-in
// (oracle/Makefile targets `unit_ref` / `unit_b200`).  Written for this
// repository; not the doctest project's code.
//
// Semantics: a test case runs once per SUBCASE it contains (code outside
// subcases runs every time); CHECK records a failure and continues, REQUIRE
// aborts the test case; an exception escaping a test case fails it.  The
// process exit code is the number of failed test cases (capped at 255).
// Filters: argv[1] = a substring of the test-case name, or
// "file=a,b" (substrings of the source file name), optionally followed by
// "skip=<substring of a test-case name>"; they select a subset.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value;
    double eps = double(std::numeric_limits<float>::epsilon()) * 100;
    explicit Approx(double v) : value(v) {}
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value) < b.eps * (1.0 + std::max(std::fabs(a), std::fabs(b.value)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
};

struct Contains {
    std::string s;
    explicit Contains(std::string x) : s(std::move(x)) {}
};

namespace detail {

inline bool matches(const Contains& c, const std::string& what) {
    return what.find(c.s) != std::string::npos;
}
inline bool matches(const char* exact, const std::string& what) { return what == exact; }
inline bool matches(const std::string& exact, const std::string& what) { return what == exact; }

using TestFn = void (*)();
struct TestCase {
    const char* name;
    TestFn fn;
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Reg {
    Reg(const char* n, TestFn f, const char* file, int line) { registry().push_back({n, f, file, line}); }
};

struct State {
    int target = 0;        // index of the subcase this run enters
    int seen = 0;          // subcases met in this run
    const char* subcase = nullptr;
    int failed_checks = 0;
    long checks = 0;
    const char* test = "";
};
inline State& st() {
    static State s;
    return s;
}

struct Abort {};  // REQUIRE failure

struct Subcase {
    bool run;
    explicit Subcase(const char* name) {
        State& s = st();
        run = s.seen == s.target;
        if (run) s.subcase = name;
        ++s.seen;
    }
    explicit operator bool() const { return run; }
};

inline void report(bool ok, const char* what, const char* file, int line) {
    State& s = st();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\"%s%s%s: %s\n", file, line, s.test,
                 s.subcase ? " / \"" : "", s.subcase ? s.subcase : "", s.subcase ? "\"" : "", what);
}

}  // namespace detail

inline int run_all(int argc, char** argv) {
    using namespace detail;
    std::string name_filter, skip;
    std::vector<std::string> files;
    for (int a = 1; a < argc; ++a) {
        const std::string arg = argv[a];
        if (arg.rfind("file=", 0) == 0) {
            std::stringstream ss(arg.substr(5));
            for (std::string f; std::getline(ss, f, ',');) files.push_back(f);
        } else if (arg.rfind("skip=", 0) == 0) {
            skip = arg.substr(5);
        } else {
            name_filter = arg;
        }
    }
    int failed_cases = 0, ran = 0;
    for (const TestCase& tc : registry()) {
        if (!name_filter.empty() && !std::strstr(tc.name, name_filter.c_str())) continue;
        if (!skip.empty() && std::strstr(tc.name, skip.c_str())) continue;
        if (!files.empty()) {
            bool hit = false;
            for (const auto& f : files) hit = hit || std::strstr(tc.file, f.c_str());
            if (!hit) continue;
        }
        ++ran;
        State& s = st();
        s.test = tc.name;
        const int before = s.failed_checks;
        for (int target = 0;; ++target) {
            s.target = target;
            s.seen = 0;
            s.subcase = nullptr;
            try {
                tc.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                report(false, (std::string("unexpected exception: ") + e.what()).c_str(), tc.file,
                       tc.line);
            } catch (...) {
                report(false, "unexpected non-std exception", tc.file, tc.line);
            }
            if (target + 1 >= s.seen) break;
        }
        if (s.failed_checks != before) ++failed_cases;
    }
    std::printf("[mini_doctest] test cases: %d | passed: %d | failed: %d | assertions: %ld | "
                "failed assertions: %d\n",
                ran, ran - failed_cases, failed_cases, st().checks, st().failed_checks);
    return failed_cases > 255 ? 255 : failed_cases;
}

}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)

#define DT_TEST_IMPL(name, id)                                                              \
    static void DT_CAT(dt_fn_, id)();                                                       \
    static ::doctest::detail::Reg DT_CAT(dt_reg_, id)(name, &DT_CAT(dt_fn_, id), __FILE__, \
                                                      __LINE__);                            \
    static void DT_CAT(dt_fn_, id)()
#define TEST_CASE(name) DT_TEST_IMPL(name, __COUNTER__)

#define SUBCASE(name) if (const ::doctest::detail::Subcase DT_CAT(dt_sc_, __COUNTER__){name})

#define DT_EVAL(require, ...)                                                         \
    do {                                                                              \
        bool dt_ok_ = false;                                                          \
        try {                                                                         \
            dt_ok_ = static_cast<bool>(__VA_ARGS__);                                  \
        } catch (const std::exception& dt_e_) {                                       \
            ::doctest::detail::report(false, (std::string(#__VA_ARGS__) +             \
                                              " threw: " + dt_e_.what()).c_str(),     \
                                      __FILE__, __LINE__);                            \
            if (require) throw ::doctest::detail::Abort{};                            \
            break;                                                                    \
        }                                                                             \
        ::doctest::detail::report(dt_ok_, #__VA_ARGS__, __FILE__, __LINE__);          \
        if (!dt_ok_ && (require)) throw ::doctest::detail::Abort{};                   \
    } while (0)

#define CHECK(...) DT_EVAL(false, __VA_ARGS__)
#define REQUIRE(...) DT_EVAL(true, __VA_ARGS__)
#define CHECK_FALSE(...) DT_EVAL(false, !(__VA_ARGS__))

#define CHECK_NOTHROW(...)                                                               \
    do {                                                                                 \
        bool dt_ok_ = true;                                                              \
        try {                                                                            \
            static_cast<void>(__VA_ARGS__);                                              \
        } catch (...) {                                                                  \
            dt_ok_ = false;                                                              \
        }                                                                                \
        ::doctest::detail::report(dt_ok_, "no throw: " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        bool dt_ok_ = false;                                                                \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const __VA_ARGS__&) {                                                      \
            dt_ok_ = true;                                                                  \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(dt_ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__,      \
                                  __LINE__);                                                \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, ...)                                               \
    do {                                                                                    \
        bool dt_ok_ = false;                                                                \
        std::string dt_what_ = "(no exception)";                                            \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const __VA_ARGS__& dt_e_) {                                                \
            dt_what_ = dt_e_.what();                                                        \
            dt_ok_ = ::doctest::detail::matches(with, dt_what_);                            \
        } catch (const std::exception& dt_e_) {                                             \
            dt_what_ = std::string("wrong type: ") + dt_e_.what();                          \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(                                                          \
            dt_ok_, ("throws " #__VA_ARGS__ " with " #with ": " #expr " -> " + dt_what_).c_str(), \
            __FILE__, __LINE__);                                                            \
    } while (0)

#define CAPTURE(x) static_cast<void>(x)
#define MESSAGE(x) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run_all(argc, argv); }
#endif
