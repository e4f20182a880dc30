// Minimal self-registering test harness for the C++ host API tests (no third-party deps).
//   TEST("name") { CHECK(x == y); REQUIRE(p != nullptr); EXPECT_CODE(expr, ErrorCode::X); }
// Exit code = number of failed tests; "--list" prints names; argv filters by substring.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

namespace tt {

struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
struct Abort {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline void fail(const char* file, int line, const std::string& what) {
    std::fprintf(stderr, "  FAIL %s:%d: %s\n", file, line, what.c_str());
    ++failures();
}
inline bool approx(double a, double b, double eps = 1e-9) { return std::fabs(a - b) <= eps * (1.0 + std::fabs(b)); }

inline int run_all(int argc, char** argv) {
    int bad = 0, ran = 0;
    for (auto& c : registry()) {
        if (argc > 1 && std::strcmp(argv[1], "--list") == 0) {
            std::printf("%s\n", c.name);
            continue;
        }
        if (argc > 1 && !std::strstr(c.name, argv[1])) continue;
        const int before = failures();
        try {
            c.fn();
        } catch (const Abort&) {
        } catch (const std::exception& e) {
            fail(__FILE__, __LINE__, std::string("unexpected exception: ") + e.what());
        }
        ++ran;
        const bool ok = failures() == before;
        if (!ok) ++bad;
        std::printf("[%s] %s\n", ok ? " ok " : "FAIL", c.name);
        std::fflush(stdout);
    }
    std::printf("%d/%d test cases passed\n", ran - bad, ran);
    return bad;
}

}  // namespace tt

#define TT_CAT2(a, b) a##b
#define TT_CAT(a, b) TT_CAT2(a, b)
#define TEST(name)                                                               \
    static void TT_CAT(tt_fn_, __LINE__)();                                      \
    static tt::Reg TT_CAT(tt_reg_, __LINE__)(name, TT_CAT(tt_fn_, __LINE__));    \
    static void TT_CAT(tt_fn_, __LINE__)()
#define CHECK(cond) \
    do { if (!(cond)) tt::fail(__FILE__, __LINE__, #cond); } while (0)
#define REQUIRE(cond)                                   \
    do {                                                \
        if (!(cond)) {                                  \
            tt::fail(__FILE__, __LINE__, #cond);        \
            throw tt::Abort{};                          \
        }                                               \
    } while (0)
#define CHECK_APPROX(a, b) \
    do { if (!tt::approx((a), (b))) tt::fail(__FILE__, __LINE__, #a " ~= " #b " (" + std::to_string(a) + " vs " + std::to_string(b) + ")"); } while (0)
#define EXPECT_CODE(expr, want_code)                                                         \
    do {                                                                                  \
        bool _thrown = false;                                                             \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const kvf::SimError& _e) {                                               \
            _thrown = true;                                                               \
            if (_e.code() != (want_code)) tt::fail(__FILE__, __LINE__, "wrong code: " #expr);  \
        }                                                                                 \
        if (!_thrown) tt::fail(__FILE__, __LINE__, "no throw: " #expr);                   \
    } while (0)
#define TT_MAIN \
    int main(int argc, char** argv) { return tt::run_all(argc, argv); }
