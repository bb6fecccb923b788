// doctest-subset shim so the reference's own unit tests
// (/root/reference/proj/tests/*.cpp) build and run unmodified; doctest is
// not vendored in the reference (proj/.gitignore:2) and absent from this
// image. TEST INFRASTRUCTURE ONLY — part of the oracle build.
//
// Supports the macros those tests use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, CHECK_MESSAGE, CHECK_NOTHROW,
// CAPTURE, FAIL, doctest::Approx(..).epsilon(..), doctest::Contains.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
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
    // doctest's rule: |l - v| < eps * (scale + max(|l|, |v|))
    friend bool operator==(double l, const Approx& r) {
        return std::fabs(l - r.value_) < r.eps_ * (r.scale_ + std::max(std::fabs(l), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double l) { return l == r; }
    friend bool operator!=(double l, const Approx& r) { return !(l == r); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
    std::string needle;
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

struct Stats {
    long checks = 0;
    long failed_checks = 0;
    bool current_failed = false;
};

inline Stats& stats() {
    static Stats s;
    return s;
}

struct RequireAbort {};

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline void report(bool ok, const char* file, int line, const char* what, const std::string& msg = "") {
    auto& s = stats();
    ++s.checks;
    if (!ok) {
        ++s.failed_checks;
        s.current_failed = true;
        std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, what, msg.c_str());
    }
}

inline void cat_into(std::ostringstream&) {}
template <typename T, typename... R>
void cat_into(std::ostringstream& os, const T& h, const R&... r) {
    os << h;
    cat_into(os, r...);
}
template <typename... A>
std::string cat(const A&... a) {
    std::ostringstream os;
    cat_into(os, a...);
    return os.str();
}

inline bool match(const std::string& what, const Contains& c) { return c.matches(what); }
inline bool match(const std::string& what, const char* s) { return what == s; }

inline int run_all() {
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        stats().current_failed = false;
        try {
            tc.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            report(false, tc.file, tc.line, "unexpected exception:", e.what());
        } catch (...) {
            report(false, tc.file, tc.line, "unexpected non-std exception", "");
        }
        if (stats().current_failed) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed; assertions: %ld | %ld failed\n",
                registry().size(), registry().size() - failed_cases, failed_cases, stats().checks,
                stats().failed_checks);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_ANON DOCTEST_CAT(doctest_anon_, __LINE__)

#define TEST_CASE(name)                                                                \
    static void DOCTEST_CAT(DOCTEST_ANON, _fn)();                                      \
    static ::doctest::detail::Registrar DOCTEST_CAT(DOCTEST_ANON, _reg)(               \
        name, __FILE__, __LINE__, &DOCTEST_CAT(DOCTEST_ANON, _fn));                    \
    static void DOCTEST_CAT(DOCTEST_ANON, _fn)()

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK(" #__VA_ARGS__ ")")

#define REQUIRE(...)                                                                            \
    do {                                                                                        \
        const bool ok_ = static_cast<bool>(__VA_ARGS__);                                        \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")");        \
        if (!ok_) throw ::doctest::detail::RequireAbort{};                                      \
    } while (0)

#define CHECK_MESSAGE(cond, ...) \
    ::doctest::detail::report(static_cast<bool>(cond), __FILE__, __LINE__, "CHECK_MESSAGE(" #cond ")", ::doctest::detail::cat(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, ...)                                                              \
    do {                                                                                        \
        bool ok_ = false;                                                                       \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (const __VA_ARGS__&) {                                                          \
            ok_ = true;                                                                         \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                \
    do {                                                                                        \
        bool ok_ = false;                                                                       \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (const __VA_ARGS__& e_) {                                                       \
            ok_ = ::doctest::detail::match(e_.what(), matcher);                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")");  \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                     \
    do {                                                                                        \
        bool ok_ = true;                                                                        \
        try {                                                                                   \
            (void)(expr);                                                                       \
        } catch (...) {                                                                         \
            ok_ = false;                                                                        \
        }                                                                                       \
        ::doctest::detail::report(ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #expr ")");         \
    } while (0)

#define CAPTURE(x) (void)(x)
#define FAIL(msg) ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL", ::doctest::detail::cat(msg))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
