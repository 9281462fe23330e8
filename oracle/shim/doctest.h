// Minimal doctest-compatible test harness (test infrastructure, not product).
//
// The reference's unit suites (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which is not vendored in the reference tree (proj/.gitignore:2)
// and not installed in this image. This header implements the subset those
// suites use: TEST_CASE, SUBCASE, CHECK, CHECK_FALSE,
// CHECK_THROWS_AS, REQUIRE, FAIL, CAPTURE, doctest::Approx(..).epsilon(..),
// DOCTEST_CONFIG_IMPLEMENT[_WITH_MAIN]. SUBCASEs are run by re-entering the
// test case once per leaf subcase, like doctest does.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double value)
        : value_(value), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
          scale_(1.0) {}
    Approx& epsilon(double e) { epsilon_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
    double value() const { return value_; }

private:
    double value_, epsilon_, scale_;
};

namespace detail {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

struct RequireFailed {};

struct State {
    std::vector<TestCase> cases;
    std::vector<std::string> captures;
    int checks = 0;
    int failures = 0;
    bool current_failed = false;
    // SUBCASE traversal: each pass enters exactly one not-yet-run leaf.
    std::vector<std::string> done;
    std::string path;
    bool entered_this_pass = false;
    bool more = false;
};

inline State& state() {
    static State s;
    return s;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        state().cases.push_back({name, file, line, fn});
    }
};

inline void report_failure(const char* file, int line, const char* kind, const char* expr,
                           const std::string& extra = "") {
    State& s = state();
    ++s.failures;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s%s\n", file, line, kind, expr,
                 extra.empty() ? "" : " ", extra.c_str());
    for (const auto& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
}

inline void check(bool ok, const char* file, int line, const char* kind, const char* expr,
                  bool require) {
    ++state().checks;
    if (!ok) {
        report_failure(file, line, kind, expr);
        if (require) throw RequireFailed{};
    }
}

class Subcase {
public:
    Subcase(const char* name) {
        State& s = state();
        std::string key = s.path + "/" + name;
        if (s.entered_this_pass) {
            // A sibling leaf already ran this pass; come back next pass.
            bool ran = false;
            for (const auto& d : s.done) ran = ran || d == key;
            if (!ran) s.more = true;
            return;
        }
        for (const auto& d : s.done) {
            if (d == key) return;
        }
        active_ = true;
        saved_ = s.path;
        s.path = key;
        key_ = key;
    }
    ~Subcase() {
        if (!active_) return;
        State& s = state();
        if (!s.entered_this_pass) {
            s.done.push_back(key_);
            s.entered_this_pass = true;
        }
        s.path = saved_;
    }
    explicit operator bool() const { return active_; }

private:
    bool active_ = false;
    std::string saved_, key_;
};

struct CaptureGuard {
    explicit CaptureGuard(std::string text) { state().captures.push_back(std::move(text)); }
    ~CaptureGuard() { state().captures.pop_back(); }
};

template <class T>
std::string stringify(const char* name, const T& v) {
    std::ostringstream os;
    os << name << " := " << v;
    return os.str();
}

inline int run_all() {
    State& s = state();
    int failed_cases = 0;
    for (const auto& tc : s.cases) {
        s.done.clear();
        s.current_failed = false;
        do {
            s.more = false;
            s.entered_this_pass = false;
            s.path.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report_failure(tc.file, tc.line, "TEST_CASE", tc.name,
                               std::string("threw: ") + e.what());
            }
        } while (s.more);
        if (s.current_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | passed: %zu | failed: %d | checks: %d | "
                "failed checks: %d\n",
                s.cases.size(), s.cases.size() - static_cast<size_t>(failed_cases), failed_cases,
                s.checks, s.failures);
    return failed_cases == 0 ? 0 : 1;
}

} // namespace detail

class Context {
public:
    Context() = default;
    Context(int, const char* const*) {}
    void applyCommandLine(int, const char* const*) {}
    template <class T>
    void setOption(const char*, T) {}
    int run() { return detail::run_all(); }
    bool shouldExit() const { return false; }
};

} // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                     \
    static void DOCTEST_ANON(doctest_fn_)();                                                \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                   &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK", #__VA_ARGS__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE", #__VA_ARGS__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE", #__VA_ARGS__, true)
#define FAIL(msg) ::doctest::detail::check(false, __FILE__, __LINE__, "FAIL", msg, true)
#define CHECK_THROWS_AS(expr, exc)                                                   \
    do {                                                                             \
        bool doctest_threw_ = false;                                                 \
        try {                                                                        \
            static_cast<void>(expr);                                                 \
        } catch (const exc&) {                                                       \
            doctest_threw_ = true;                                                   \
        } catch (...) {                                                              \
        }                                                                            \
        ::doctest::detail::check(doctest_threw_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr, false); \
    } while (0)
#define CAPTURE(x) ::doctest::detail::CaptureGuard DOCTEST_ANON(doctest_cap_)(::doctest::detail::stringify(#x, x))

#if defined(DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
int main() { return ::doctest::detail::run_all(); }
#endif
