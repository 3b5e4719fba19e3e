// TEST INFRASTRUCTURE ONLY: a minimal doctest-compatible header, so the reference's own unit
// tests (`proj/tests/unit/*.cpp`, written against doctest, which this image does not ship)
// compile UNCHANGED against this repo's drop-in headers (include/ddm) and run against
// libddm_b200.so (oracle/Makefile target `unit`, tests/test_reference_unit.py).
//
// Covers exactly what those files use: TEST_CASE, CHECK, CHECK_EQ/LE/GE/LT/GT, REQUIRE,
// REQUIRE_EQ, CHECK_THROWS_AS, doctest::Approx(...).epsilon(...), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN. Semantics follow doctest: CHECK records a failure and
// continues, REQUIRE ends the test case, an escaping exception fails it, Approx compares with
// |a - b| < eps * (1 + max(|a|, |b|)) and a default eps of 100 float epsilons.
#ifndef DDM_DOCTEST_SHIM_H
#define DDM_DOCTEST_SHIM_H

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
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.equal(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.equal(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.equal(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.equal(rhs); }
    double value() const { return value_; }

private:
    bool equal(double other) const {
        return std::fabs(other - value_) <
               eps_ * (scale_ + std::fmax(std::fabs(other), std::fabs(value_)));
    }
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline int& failures() {
    static int f = 0;
    return f;
}
inline long& assertions() {
    static long a = 0;
    return a;
}

inline void fail(const char* file, int line, const std::string& what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: ERROR: %s\n", file, line, what.c_str());
}

template <class T>
std::string show(const T& v) {
    if constexpr (requires(std::ostream& o) { o << v; }) {
        std::ostringstream s;
        s.precision(17);
        s << v;
        return s.str();
    } else {
        return "{?}";
    }
}
inline std::string show(const Approx& a) { return "Approx(" + show(a.value()) + ")"; }

template <class A, class B, class Op>
bool binary(const char* file, int line, const char* text, const A& a, const B& b, Op op, bool require) {
    ++assertions();
    if (op(a, b)) return true;
    fail(file, line, std::string(require ? "REQUIRE" : "CHECK") + "( " + text + " ) is NOT correct: values ( " +
                         show(a) + ", " + show(b) + " )");
    if (require) throw RequireFailed{};
    return false;
}

inline int run_all() {
    int failed_cases = 0;
    for (const auto& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            fail(c.file, c.line, std::string("test case threw: ") + e.what());
        } catch (...) {
            fail(c.file, c.line, "test case threw an unknown exception");
        }
        if (failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "  in TEST_CASE \"%s\" (%s:%d)\n", c.name, c.file, c.line);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | failures: %d\n",
                registry().size(), registry().size() - failed_cases, failed_cases, assertions(), failures());
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                                   \
    static void fn();                                                                           \
    static const doctest::detail::Registrar reg(name, __FILE__, __LINE__, &fn);                \
    static void fn()
#define TEST_CASE(name) \
    DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), DOCTEST_CAT(doctest_reg_, __LINE__), name)

#define DOCTEST_UNARY_(kind, require, ...)                                                      \
    do {                                                                                        \
        ++doctest::detail::assertions();                                                       \
        if (!(__VA_ARGS__)) {                                                                   \
            doctest::detail::fail(__FILE__, __LINE__, std::string(kind "( ") + #__VA_ARGS__ + " ) is NOT correct"); \
            if (require) throw doctest::detail::RequireFailed{};                                \
        }                                                                                       \
    } while (0)
#define CHECK(...) DOCTEST_UNARY_("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_UNARY_("REQUIRE", true, __VA_ARGS__)

#define DOCTEST_BINARY_(a, b, op, require)                                                     \
    doctest::detail::binary(__FILE__, __LINE__, #a ", " #b, (a), (b),                          \
                            [](const auto& x, const auto& y) { return x op y; }, require)
#define CHECK_EQ(a, b) DOCTEST_BINARY_(a, b, ==, false)
#define CHECK_NE(a, b) DOCTEST_BINARY_(a, b, !=, false)
#define CHECK_LE(a, b) DOCTEST_BINARY_(a, b, <=, false)
#define CHECK_GE(a, b) DOCTEST_BINARY_(a, b, >=, false)
#define CHECK_LT(a, b) DOCTEST_BINARY_(a, b, <, false)
#define CHECK_GT(a, b) DOCTEST_BINARY_(a, b, >, false)
#define REQUIRE_EQ(a, b) DOCTEST_BINARY_(a, b, ==, true)

#define CHECK_THROWS_AS(expr, ...)                                                             \
    do {                                                                                        \
        ++doctest::detail::assertions();                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                                          \
            doctest_ok_ = true;                                                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        if (!doctest_ok_)                                                                       \
            doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " ) failed"); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif

#endif
