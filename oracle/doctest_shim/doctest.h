// Minimal doctest-compatible test harness -- TEST INFRASTRUCTURE ONLY (oracle/README.md).
//
// The reference's own unit suites (/root/reference/proj/tests/test_*.cpp) include <doctest.h>,
// which is not installed here.  This header implements the subset they use so the suites
// compile UNMODIFIED, in place, against oracle/_ref/libkvsim_ref.a (the reference compiled from
// its own sources): a health check that the oracle build behaves as the reference's authors
// intended, before any golden vector is trusted.
//
// Supported: TEST_CASE, SUBCASE (doctest re-entry semantics: every leaf path runs once, each
// run re-executes the enclosing code), CHECK / CHECK_FALSE / REQUIRE / REQUIRE_FALSE, FAIL /
// FAIL_CHECK with stream messages, INFO (scoped, stream), doctest::Approx (default epsilon
// FLT_EPSILON * 100, .epsilon(), .scale()), doctest::Contains, CHECK_THROWS_WITH_AS, and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Output: one line per failed assertion
// ("FAIL file:line: expression [info]"), one line per test case, a summary; exit status 1
// when any assertion failed.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }
    friend bool operator<(double lhs, const Approx& a) { return lhs < a.v_ && lhs != a; }
    friend bool operator>(double lhs, const Approx& a) { return lhs > a.v_ && lhs != a; }

private:
    double v_, eps_ = static_cast<double>(FLT_EPSILON) * 100, scale_ = 1.0;
};

struct Contains {
    explicit Contains(const char* s) : sub(s) {}
    std::string sub;
    bool check(const std::string& s) const { return s.find(sub) != std::string::npos; }
};

namespace detail {

struct Abort {};  // thrown by REQUIRE / FAIL: ends the current run of the test case

struct State {
    // registry
    struct Case {
        const char* name;
        const char* file;
        int line;
        void (*fn)();
    };
    std::vector<Case> cases;
    // current test case
    std::vector<std::string> stack;                // entered subcase path
    std::set<std::vector<std::string>> done;       // fully explored subcase paths
    bool entered_level[64] = {};                   // a subcase was entered at this depth this run
    bool incomplete[65] = {};                      // a sibling at this depth was left for a later run
    bool rerun = false;
    std::vector<std::string> info;                 // INFO context
    int failed_asserts = 0, asserts = 0, case_failures = 0;
    const char* case_name = "";
};
inline State& st() {
    static State s;
    return s;
}

inline int register_case(const char* name, const char* file, int line, void (*fn)()) {
    st().cases.push_back({name, file, line, fn});
    return 0;
}

inline void report(const char* file, int line, const std::string& what) {
    State& s = st();
    ++s.failed_asserts;
    ++s.case_failures;
    std::string ctx;
    for (const auto& i : s.info) ctx += " [" + i + "]";
    std::string path;
    for (const auto& p : s.stack) path += " / " + p;
    std::printf("FAIL %s:%d: %s (case \"%s\"%s)%s\n", file, line, what.c_str(), s.case_name, path.c_str(), ctx.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
    ++st().asserts;
    if (ok) return;
    report(file, line, expr);
    if (require) throw Abort{};
}

class Subcase {
public:
    Subcase(const char* name) {
        State& s = st();
        level_ = s.stack.size();
        std::vector<std::string> path = s.stack;
        path.push_back(name);
        if (s.done.count(path)) return;  // explored in an earlier run
        if (s.entered_level[level_]) {   // one subcase per depth per run: come back later
            s.incomplete[level_] = true;
            s.rerun = true;
            return;
        }
        s.entered_level[level_] = true;
        s.stack.push_back(name);
        path_ = path;
        entered_ = true;
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = st();
        if (!s.incomplete[level_ + 1] || std::uncaught_exceptions() > 0) s.done.insert(path_);
        else s.rerun = true;
        s.incomplete[level_ + 1] = false;
        s.entered_level[level_ + 1] = false;
        s.stack.pop_back();
    }
    explicit operator bool() const { return entered_; }

private:
    size_t level_ = 0;
    bool entered_ = false;
    std::vector<std::string> path_;
};

struct Msg {  // `Msg{os} << a << b` and `Msg{os} << a, b, c` both stream every operand
    std::ostringstream& os;
    template <typename T>
    Msg& operator<<(const T& x) {
        os << x;
        return *this;
    }
    template <typename T>
    Msg& operator,(const T& x) {
        os << x;
        return *this;
    }
};

class Info {
public:
    explicit Info(std::string s) { st().info.push_back(std::move(s)); }
    ~Info() { st().info.pop_back(); }
};

inline int run_all() {
    State& s = st();
    int failed_cases = 0;
    for (const auto& c : s.cases) {
        s.done.clear();
        s.case_name = c.name;
        s.case_failures = 0;
        int runs = 0;
        do {
            s.rerun = false;
            std::memset(s.entered_level, 0, sizeof(s.entered_level));
            std::memset(s.incomplete, 0, sizeof(s.incomplete));
            s.stack.clear();
            s.info.clear();
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& ex) {
                report(c.file, c.line, std::string("unexpected exception: ") + ex.what());
            } catch (...) {
                report(c.file, c.line, "unexpected non-standard exception");
            }
        } while (s.rerun && ++runs < 100000);
        if (s.case_failures) ++failed_cases;
        std::printf("%s %s\n", s.case_failures ? "CASE-FAIL" : "CASE-PASS", c.name);
    }
    std::printf("test cases: %zu | %zu passed | %d failed; assertions: %d | %d failed\n", s.cases.size(),
                s.cases.size() - failed_cases, failed_cases, s.asserts, s.failed_asserts);
    return s.failed_asserts ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                                \
    static void fn();                                                                                   \
    static const int DOCTEST_CAT(fn, _reg) = doctest::detail::register_case(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name})
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) doctest::detail::check(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) doctest::detail::check(!(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", true)
// messages: both the stream form INFO(a << b) and the variadic form INFO(a, b, c)
#define DOCTEST_MSG_(...) \
    ([&]() { std::ostringstream doctest_os; doctest::detail::Msg{doctest_os} << __VA_ARGS__; return doctest_os.str(); }())
#define FAIL(m)                                                                  \
    do {                                                                         \
        doctest::detail::report(__FILE__, __LINE__, "FAIL: " + DOCTEST_MSG_(m)); \
        throw doctest::detail::Abort{};                                          \
    } while (0)
#define FAIL_CHECK(m) doctest::detail::report(__FILE__, __LINE__, "FAIL_CHECK: " + DOCTEST_MSG_(m))
#define CHECK_MESSAGE(cond, m)                                                                          \
    do {                                                                                                \
        const doctest::detail::Info doctest_msg_info(DOCTEST_MSG_(m));                                 \
        doctest::detail::check(static_cast<bool>(cond), __FILE__, __LINE__, #cond, false);             \
    } while (0)
#define INFO(...) const doctest::detail::Info DOCTEST_CAT(doctest_info_, __LINE__)(DOCTEST_MSG_(__VA_ARGS__))
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                   \
    do {                                                                                           \
        bool doctest_ok = false;                                                                   \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__& doctest_e) {                                                   \
            doctest_ok = (matcher).check(doctest_e.what());                                        \
        } catch (...) {                                                                            \
        }                                                                                          \
        doctest::detail::check(doctest_ok, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS(" #expr ")", false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
