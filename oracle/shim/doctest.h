// Minimal doctest-subset shim (TEST INFRASTRUCTURE ONLY).
//
// Lets the reference's own hot-path suites
// (/root/reference/proj/tests/test_{scene,tracer,blender,grad,convert}.cpp) compile and run
// unmodified against oracle/_ref, which validates the Eigen shim and pins the
// oracle to the reference's known-answer tests.
// Supported: TEST_CASE, SUBCASE (one level), CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_MESSAGE, doctest::Approx(...).epsilon(...).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
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
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

struct State {
    long checks = 0;
    long failures = 0;
    const char* current = "";
    // one-level SUBCASE traversal
    int subcase_target = 0;
    int subcase_seen = 0;
};

inline State& state() {
    static State s;
    return s;
}

inline void report(bool ok, const char* file, int line, const char* expr, const std::string& msg = {}) {
    ++state().checks;
    if (!ok) {
        ++state().failures;
        std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s %s\n", file, line, state().current, expr,
                     msg.c_str());
    }
}

struct Subcase {
    bool active;
    explicit Subcase(const char*) {
        State& s = state();
        active = (s.subcase_seen == s.subcase_target);
        ++s.subcase_seen;
    }
    explicit operator bool() const { return active; }
};

template <typename... Args>
std::string concat(const Args&... args) {
    std::ostringstream os;
    ((os << args), ...);
    return os.str();
}

inline int run_all() {
    long cases = 0, failed_cases = 0;
    for (const auto& tc : registry()) {
        ++cases;
        const long before = state().failures;
        state().current = tc.name;
        state().subcase_target = 0;
        for (;;) {
            state().subcase_seen = 0;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(false, "<exception>", 0, e.what());
            }
            if (state().subcase_seen > state().subcase_target + 1) {
                ++state().subcase_target;
                continue;
            }
            break;
        }
        if (state().failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed; assertions: %ld | %ld failed\n",
                cases, cases - failed_cases, failed_cases, state().checks, state().failures);
    return state().failures == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)

#define TEST_CASE(name)                                                                     \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                       \
    static ::doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(                \
        name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                         \
    static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define CHECK_MESSAGE(cond, ...)                                                            \
    do {                                                                                    \
        const bool doctest_ok_ = static_cast<bool>(cond);                                   \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #cond,                   \
                                  doctest_ok_ ? std::string() : ::doctest::detail::concat(__VA_ARGS__)); \
    } while (0)
#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                            \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #__VA_ARGS__);           \
        if (!doctest_ok_) throw ::doctest::detail::RequireFailed{};                         \
    } while (0)
#define FAIL(msg)                                                                           \
    do {                                                                                    \
        ::doctest::detail::report(false, __FILE__, __LINE__, "FAIL", msg);                  \
        throw ::doctest::detail::RequireFailed{};                                           \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                         \
    do {                                                                                    \
        bool doctest_thrown_ = false;                                                       \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const type&) {                                                             \
            doctest_thrown_ = true;                                                         \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(doctest_thrown_, __FILE__, __LINE__, "throws " #type ": " #expr); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, msg, type)                                               \
    do {                                                                                    \
        bool doctest_thrown_ = false;                                                       \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (const type& doctest_e_) {                                                  \
            doctest_thrown_ = std::string(doctest_e_.what()) == std::string(msg);           \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(doctest_thrown_, __FILE__, __LINE__, "throws " #type " with " #msg ": " #expr); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                 \
    do {                                                                                    \
        bool doctest_ok_ = true;                                                            \
        try {                                                                               \
            (void)(expr);                                                                   \
        } catch (...) {                                                                     \
            doctest_ok_ = false;                                                            \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, __FILE__, __LINE__, "nothrow: " #expr);      \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
