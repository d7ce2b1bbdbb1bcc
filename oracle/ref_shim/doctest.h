// doctest.h -- a minimal, self-written stand-in for the doctest subset the
// reference's tests use (TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CAPTURE, MESSAGE, doctest::Approx), so proj/tests compile
// and run here against the reference sources.  TEST INFRASTRUCTURE ONLY.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <iostream>
#include <set>
#include <sstream>
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
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool eq(double o) const { return std::fabs(o - v_) < eps_ * (scale_ + std::max(std::fabs(o), std::fabs(v_))); }
    double value() const { return v_; }

private:
    double v_, eps_ = 1.1920928955078125e-05 /* FLT_EPSILON * 100 */, scale_ = 1.0;
};
inline bool operator==(double a, const Approx& b) { return b.eq(a); }
inline bool operator==(const Approx& a, double b) { return a.eq(b); }
inline bool operator!=(double a, const Approx& b) { return !b.eq(a); }
inline bool operator!=(const Approx& a, double b) { return !a.eq(b); }
inline std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value() << ")"; }

namespace stub {

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
struct RequireFailed {};

struct State {
    int checks = 0, failures = 0;
    // subcases: one leaf per pass; lines of the subcases already run
    std::set<int> done;
    int entered = -1;   // line of the subcase entered in this pass
    bool skipped = false;  // a not-yet-run subcase was skipped in this pass
    std::vector<std::string> captures;
};
inline State& st() {
    static State s;
    return s;
}

inline void report(const char* kind, const char* expr, const char* file, int line) {
    ++st().failures;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, kind, expr);
    for (auto& c : st().captures) std::fprintf(stderr, "    with %s\n", c.c_str());
}

struct Subcase {
    bool on;
    Subcase(const char* /*name*/, int line) {
        State& s = st();
        on = false;
        if (s.done.count(line)) return;
        if (s.entered < 0) {
            s.entered = line;
            on = true;
        } else {
            s.skipped = true;
        }
    }
    explicit operator bool() const { return on; }
};

struct Capture {
    Capture(const std::string& s) { st().captures.push_back(s); }
    ~Capture() { st().captures.pop_back(); }
};

template <typename T>
std::string capture_str(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    return os.str();
}

inline void message(const std::string& m, const char* file, int line) {
    std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", file, line, m.c_str());
}
template <typename... A>
std::string cat(const A&... a) {
    std::ostringstream os;
    (os << ... << a);
    return os.str();
}

inline int run_all(int argc, char** argv) {
    int cases = 0, failed_cases = 0;
    for (const auto& tc : registry()) {
        if (argc > 1) {  // optional filter: substring of the test case name
            bool hit = false;
            for (int i = 1; i < argc; ++i)
                if (std::string(tc.name).find(argv[i]) != std::string::npos) hit = true;
            if (!hit) continue;
        }
        ++cases;
        State& s = st();
        const int before = s.failures;
        s.done.clear();
        while (true) {
            s.entered = -1;
            s.skipped = false;
            s.captures.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
            }
            if (s.entered >= 0) s.done.insert(s.entered);
            if (!s.skipped) break;
        }
        if (s.failures != before) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED test case: %s\n", tc.name);
        }
    }
    std::printf("[doctest-stub] test cases: %d | passed: %d | failed: %d | checks: %d | failed checks: %d\n", cases,
                cases - failed_cases, failed_cases, st().checks, st().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace stub
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                            \
    static void fn();                                                                               \
    static doctest::stub::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);           \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_stub_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::stub::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __LINE__})
#define CHECK(...)                                                                   \
    do {                                                                             \
        ++doctest::stub::st().checks;                                                \
        if (!(__VA_ARGS__)) doctest::stub::report("CHECK", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_FALSE(...)                                                             \
    do {                                                                             \
        ++doctest::stub::st().checks;                                                \
        if ((__VA_ARGS__)) doctest::stub::report("CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define REQUIRE(...)                                                                 \
    do {                                                                             \
        ++doctest::stub::st().checks;                                                \
        if (!(__VA_ARGS__)) {                                                        \
            doctest::stub::report("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);      \
            throw doctest::stub::RequireFailed();                                    \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
    do {                                                                             \
        ++doctest::stub::st().checks;                                                \
        bool doctest_ok_ = false;                                                    \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                               \
            doctest_ok_ = true;                                                      \
        } catch (...) {                                                              \
        }                                                                            \
        if (!doctest_ok_) doctest::stub::report("CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
    } while (0)
#define CAPTURE(x) \
    const doctest::stub::Capture DOCTEST_CAT(doctest_cap_, __LINE__)(doctest::stub::capture_str(#x, x))
#define MESSAGE(...) doctest::stub::message(doctest::stub::cat(__VA_ARGS__), __FILE__, __LINE__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::stub::run_all(argc, argv); }
#endif
