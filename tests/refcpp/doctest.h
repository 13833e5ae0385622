// tests/refcpp/doctest.h -- TEST INFRASTRUCTURE: a minimal stand-in for the
// doctest single header the reference's tests include (<doctest.h>,
// proj/CMakeLists.txt:10; the vendored copy is absent from the reference tree
// and there is no network).  It implements exactly what
// proj/tests/test_{reorder,schur}.cpp use: TEST_CASE, CHECK, REQUIRE,
// CHECK_MESSAGE, CHECK_THROWS_AS, doctest::Approx(..).epsilon(..) and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Optional argv[1]: substring filter on
// test names.  Exit status = number of failed test cases (capped at 255).
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

struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line) {
        registry().push_back({name, fn, file, line});
    }
};

struct RequireFailed {};

inline int& failures_in_case() {
    static int f = 0;
    return f;
}
inline long& checks_run() {
    static long c = 0;
    return c;
}

inline void report(bool ok, const char* expr, const char* file, int line, const std::string& msg = "") {
    ++checks_run();
    if (ok) return;
    ++failures_in_case();
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s %s\n", file, line, expr, msg.c_str());
}

class Approx {
   public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        // doctest's rule: |a - b| < eps * (scale + max(|a|, |b|)), scale 1
        return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }

   private:
    double v_;
    double eps_ = 1.1920928955078125e-07 * 100;  // float eps * 100, doctest's default
};

inline int run_all(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int failed_cases = 0, ran = 0;
    for (const auto& tc : registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++ran;
        failures_in_case() = 0;
        bool aborted = false;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
            aborted = true;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
            ++failures_in_case();
        }
        const bool ok = failures_in_case() == 0 && !aborted;
        std::printf("[%s] %s\n", ok ? "  ok  " : "FAILED", tc.name);
        if (!ok) ++failed_cases;
    }
    std::printf("test cases: %d | passed: %d | failed: %d | checks: %ld\n", ran, ran - failed_cases, failed_cases,
                checks_run());
    return failed_cases > 255 ? 255 : failed_cases;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                               \
    static void fn();                                                                       \
    static doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);          \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_MESSAGE(cond, msg)                                                              \
    do {                                                                                      \
        std::ostringstream doctest_os_;                                                       \
        doctest_os_ << msg;                                                                   \
        doctest::report(static_cast<bool>(cond), #cond, __FILE__, __LINE__, doctest_os_.str()); \
    } while (0)
#define REQUIRE(...)                                                                          \
    do {                                                                                      \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                              \
        doctest::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);                        \
        if (!doctest_ok_) throw doctest::RequireFailed{};                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                            \
    do {                                                                                      \
        bool doctest_thrown_ = false;                                                         \
        try {                                                                                 \
            (void)(expr);                                                                     \
        } catch (const __VA_ARGS__&) {                                                        \
            doctest_thrown_ = true;                                                           \
        } catch (...) {                                                                       \
        }                                                                                     \
        doctest::report(doctest_thrown_, "THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run_all(argc, argv); }
#endif
