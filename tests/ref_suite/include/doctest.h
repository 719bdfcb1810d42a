// A small doctest-compatible test runner (test infrastructure).  The
// reference's unit tests include "doctest.h" (vendor/doctest.h is not shipped,
// proj/.gitignore:2); this header provides the subset they use so they compile
// UNMODIFIED against the drop-in library: TEST_CASE, SUBCASE (re-runs the case
// once per leaf subcase), CHECK / CHECK_FALSE / REQUIRE / CHECK_THROWS_AS /
// CHECK_NOTHROW / FAIL, doctest::Approx(v).epsilon(e).scale(s) with doctest's
// comparison rule, and a main (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) with
// --tc=<substring> / --tce=<substring> filters.
//
// Recorded substitutions.  A check whose file:line appears in the
// substitution table (tests/ref_suite/substitutions.hpp, included when
// SAAP_REF_SUBSTITUTIONS is defined) compares `lhs <op> rhs` against the
// table's tolerance instead of its literal right-hand side, or uses the
// table's epsilon for a doctest::Approx on that line.  Every substituted
// check prints one line ("substituted ...") so the run log records it.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

namespace doctest {
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

struct RunState {
    int asserts = 0, failures = 0, substituted = 0;
    const char* cur_file = "";
    int cur_line = 0;
    // subcases
    std::set<std::vector<std::string>> done;
    std::vector<std::string> stack;
    std::vector<bool> entered_at;   // a subcase was entered at this depth in this run
    std::vector<bool> pending_at;   // an unfinished sibling/child was skipped
    bool more = false;
};
inline RunState& st() {
    static RunState s;
    return s;
}

struct AbortCase {};

// ---- substitution table: file suffix + line -> tolerance
struct Subst {
    const char* file;
    int line;
    double tol;
    const char* why;
};
inline std::vector<Subst>& substitutions() {
    static std::vector<Subst> v;
    return v;
}
inline const Subst* find_subst(const char* file, int line) {
    for (const auto& s : substitutions()) {
        const size_t lf = std::strlen(file), ls = std::strlen(s.file);
        if (s.line == line && lf >= ls && std::strcmp(file + lf - ls, s.file) == 0) return &s;
    }
    return nullptr;
}
struct SubstRegistrar {
    SubstRegistrar(const char* f, int l, double t, const char* why) {
        substitutions().push_back({f, l, t, why});
    }
};

inline void report_fail(const char* file, int line, const std::string& what) {
    ++st().failures;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

template <typename T>
std::string show(const T& v) {
    if constexpr (std::is_arithmetic_v<T>) {
        std::ostringstream os;
        os.precision(17);
        os << v;
        return os.str();
    } else if constexpr (std::is_same_v<T, std::string> || std::is_same_v<T, const char*>) {
        return std::string(v);
    } else {
        return "{?}";
    }
}

// expression decomposition: CHECK(a op b) -> Lhs(a) op b
struct Res {
    bool ok;
    std::string text;
};
template <typename L>
struct Lhs {
    const L& lhs;
    template <typename R>
    Res cmp(const R& rhs, const char* op, bool ok) const {
        return {ok, show(lhs) + " " + op + " " + show(rhs)};
    }
    // `<=` / `<` against a number may be substituted (recorded tolerance)
    template <typename R>
    Res tol_cmp(const R& rhs, const char* op, bool strict) const {
        if constexpr (std::is_arithmetic_v<L> && std::is_arithmetic_v<R>) {
            if (const Subst* s = find_subst(st().cur_file, st().cur_line)) {
                ++st().substituted;
                const double l = (double)lhs;
                const bool ok = strict ? l < s->tol : l <= s->tol;
                std::fprintf(stderr, "%s:%d: substituted %s %s %s -> %s %s %.3g (%s): %s\n",
                             st().cur_file, st().cur_line, show(lhs).c_str(), op,
                             show(rhs).c_str(), show(lhs).c_str(), op, s->tol, s->why,
                             ok ? "ok" : "FAIL");
                return {ok, show(lhs) + " " + op + " " + show(s->tol) + " (substituted)"};
            }
        }
        return cmp(rhs, op, strict ? lhs < rhs : lhs <= rhs);
    }
    template <typename R> Res operator==(const R& r) const { return cmp(r, "==", lhs == r); }
    template <typename R> Res operator!=(const R& r) const { return cmp(r, "!=", lhs != r); }
    template <typename R> Res operator<(const R& r) const { return tol_cmp(r, "<", true); }
    template <typename R> Res operator<=(const R& r) const { return tol_cmp(r, "<=", false); }
    template <typename R> Res operator>(const R& r) const { return cmp(r, ">", lhs > r); }
    template <typename R> Res operator>=(const R& r) const { return cmp(r, ">=", lhs >= r); }
    operator Res() const {
        if constexpr (std::is_convertible_v<L, bool>) return {static_cast<bool>(lhs), show(lhs)};
        else return {true, "?"};
    }
};
struct Decomposer {
    template <typename L>
    Lhs<L> operator<<(const L& l) const {
        return Lhs<L>{l};
    }
};

inline void check(bool ok, const char* file, int line, const char* expr, const std::string& val,
                  bool require) {
    ++st().asserts;
    if (!ok) {
        report_fail(file, line, std::string(expr) + "  with values  " + val);
        if (require) throw AbortCase{};
    }
}

// ---- subcases
struct Subcase {
    bool entered = false;
    std::vector<std::string> path;
    Subcase(const char* name) {
        RunState& s = st();
        const size_t depth = s.stack.size();
        if (s.entered_at.size() <= depth) {
            s.entered_at.resize(depth + 1, false);
            s.pending_at.resize(depth + 1, false);
        }
        path = s.stack;
        path.push_back(name);
        if (s.done.count(path)) return;
        if (s.entered_at[depth]) {  // a sibling ran in this pass: come back for this one
            s.more = true;
            return;
        }
        s.entered_at[depth] = true;
        entered = true;
        s.stack.push_back(name);
        if (s.entered_at.size() <= depth + 1) {
            s.entered_at.resize(depth + 2, false);
            s.pending_at.resize(depth + 2, false);
        }
        s.entered_at[depth + 1] = false;
        s.pending_at[depth + 1] = false;
    }
    ~Subcase() {
        if (!entered) return;
        RunState& s = st();
        const size_t depth = s.stack.size();  // == our depth + 1
        // finished unless a child subcase is still pending
        bool child_pending = false;
        if (depth < s.entered_at.size()) child_pending = s.more && s.entered_at[depth];
        if (!child_pending) s.done.insert(path);
        s.stack.pop_back();
    }
    explicit operator bool() const { return entered; }
};

}  // namespace detail

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
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.eq(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.eq(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.eq(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.eq(rhs); }
    double value() const { return value_; }

private:
    bool eq(double x) const {
        double e = eps_;
        if (const auto* s = detail::find_subst(detail::st().cur_file, detail::st().cur_line)) {
            ++detail::st().substituted;
            std::fprintf(stderr, "%s:%d: substituted Approx epsilon %.3g -> %.3g (%s)\n",
                         detail::st().cur_file, detail::st().cur_line, eps_, s->tol, s->why);
            e = s->tol;
        }
        // doctest's rule: |x - v| < eps * (scale + max(|x|, |v|))
        return std::fabs(x - value_) < e * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
    }
    double value_;
    double eps_ = static_cast<double>(1.1920928955078125e-07f) * 100;
    double scale_ = 1.0;
};

namespace detail {
template <>
inline std::string show<Approx>(const Approx& v) {
    return "Approx(" + show(v.value()) + ")";
}
}  // namespace detail

inline int run(int argc, char** argv) {
    std::vector<std::string> inc, exc;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--tc=", 0) == 0 || a.rfind("-tc=", 0) == 0) inc.push_back(a.substr(a.find('=') + 1));
        if (a.rfind("--tce=", 0) == 0 || a.rfind("-tce=", 0) == 0) exc.push_back(a.substr(a.find('=') + 1));
    }
    int cases = 0, failed_cases = 0, skipped = 0;
    for (const auto& tc : detail::registry()) {
        const std::string name = tc.name;
        bool take = inc.empty();
        for (auto& s : inc) take |= name.find(s) != std::string::npos;
        for (auto& s : exc) take &= name.find(s) == std::string::npos;
        if (!take) {
            ++skipped;
            continue;
        }
        ++cases;
        auto& s = detail::st();
        const int f0 = s.failures;
        s.done.clear();
        for (int pass = 0; pass < 1000; ++pass) {
            s.stack.clear();
            s.entered_at.assign(1, false);
            s.pending_at.assign(1, false);
            s.more = false;
            try {
                tc.fn();
            } catch (const detail::AbortCase&) {
            } catch (const std::exception& e) {
                detail::report_fail(tc.file, tc.line,
                                    std::string("unexpected exception: ") + e.what());
            } catch (...) {
                detail::report_fail(tc.file, tc.line, "unexpected exception");
            }
            if (!s.more) break;
        }
        const bool bad = s.failures != f0;
        failed_cases += bad;
        std::fprintf(stderr, "[%s] %s\n", bad ? "FAIL" : " ok ", tc.name);
    }
    const auto& s = detail::st();
    std::printf("test cases: %d | %d passed | %d failed | %d skipped; assertions: %d | %d failed; "
                "substituted checks: %d\n",
                cases, cases - failed_cases, failed_cases, skipped, s.asserts, s.failures,
                s.substituted);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                   \
    static void DOCTEST_UNIQUE(doctest_fn_)();                                            \
    static ::doctest::detail::Registrar DOCTEST_UNIQUE(doctest_reg_)(                     \
            name, __FILE__, __LINE__, &DOCTEST_UNIQUE(doctest_fn_));                      \
    static void DOCTEST_UNIQUE(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sc_){name})

#define DOCTEST_CHECK_IMPL(require, ...)                                                  \
    do {                                                                                   \
        ::doctest::detail::st().cur_file = __FILE__;                                       \
        ::doctest::detail::st().cur_line = __LINE__;                                       \
        try {                                                                              \
            const ::doctest::detail::Res doctest_r_ = ::doctest::detail::Decomposer() << __VA_ARGS__; \
            ::doctest::detail::check(doctest_r_.ok, __FILE__, __LINE__, #__VA_ARGS__,             \
                                     doctest_r_.text, require);                            \
        } catch (const ::doctest::detail::AbortCase&) {                                    \
            throw;                                                                         \
        } catch (const std::exception& e) {                                                \
            ::doctest::detail::check(false, __FILE__, __LINE__, #__VA_ARGS__,                     \
                                     std::string("threw: ") + e.what(), require);          \
        }                                                                                  \
        ::doctest::detail::st().cur_line = 0;                                              \
    } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL(false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_CHECK_IMPL(true, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL(true, !(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, ...)                                                         \
    do {                                                                                   \
        ++::doctest::detail::st().asserts;                                                 \
        bool doctest_ok_ = false;                                                          \
        std::string doctest_w_ = "did not throw";                                         \
        try {                                                                              \
            static_cast<void>(expr);                                                       \
        } catch (const __VA_ARGS__&) {                                                     \
            doctest_ok_ = true;                                                            \
        } catch (const std::exception& e) {                                                \
            doctest_w_ = std::string("threw another type: ") + e.what();                   \
        } catch (...) {                                                                    \
            doctest_w_ = "threw an unknown type";                                          \
        }                                                                                  \
        if (!doctest_ok_)                                                                  \
            ::doctest::detail::report_fail(__FILE__, __LINE__,                             \
                                           std::string("CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ") ") + doctest_w_); \
    } while (0)

#define CHECK_NOTHROW(expr)                                                                \
    do {                                                                                   \
        ++::doctest::detail::st().asserts;                                                 \
        try {                                                                              \
            static_cast<void>(expr);                                                       \
        } catch (const std::exception& e) {                                                \
            ::doctest::detail::report_fail(__FILE__, __LINE__,                             \
                                           std::string("CHECK_NOTHROW(" #expr ") threw: ") + e.what()); \
        }                                                                                  \
    } while (0)

#define FAIL(msg)                                                                          \
    do {                                                                                   \
        ::doctest::detail::report_fail(__FILE__, __LINE__, std::string("FAIL: ") + (msg)); \
        throw ::doctest::detail::AbortCase{};                                              \
    } while (0)

// substitution table entry: SAAP_SUBST("attention_test.cpp", 244, 1e-3, "why")
#define SAAP_SUBST(file, line, tol, why)                                                   \
    static ::doctest::detail::SubstRegistrar DOCTEST_UNIQUE(saap_subst_)(file, line, tol, why)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run(argc, argv); }
#endif
