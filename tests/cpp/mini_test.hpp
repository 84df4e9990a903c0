// mini_test.hpp — a minimal doctest-like harness (doctest is not vendored).
#pragma once

#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace mini {
struct Case {
    const char* name;
    std::function<void()> fn;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline int& failures() {
    static int f = 0;
    return f;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
inline void fail(const char* file, int line, const std::string& what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED %s\n", file, line, what.c_str());
}
inline int run_all() {
    int bad_cases = 0;
    for (auto& c : registry()) {
        const int before = failures();
        try {
            c.fn();
        } catch (const std::exception& e) {
            fail(c.name, 0, std::string("unexpected exception: ") + e.what());
        }
        const bool ok = failures() == before;
        bad_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? " ok " : "FAIL", c.name);
    }
    std::printf("%zu cases, %d failed, %d failed checks\n", registry().size(), bad_cases,
                failures());
    return bad_cases ? 1 : 0;
}
}  // namespace mini

#define MINI_CAT2(a, b) a##b
#define MINI_CAT(a, b) MINI_CAT2(a, b)
#define TEST_CASE(name)                                                            \
    static void MINI_CAT(test_fn_, __LINE__)();                                    \
    static mini::Reg MINI_CAT(test_reg_, __LINE__)(name, MINI_CAT(test_fn_, __LINE__)); \
    static void MINI_CAT(test_fn_, __LINE__)()
#define CHECK(cond) \
    do {            \
        if (!(cond)) mini::fail(__FILE__, __LINE__, #cond); \
    } while (0)
#define REQUIRE(cond)                                   \
    do {                                                \
        if (!(cond)) {                                  \
            mini::fail(__FILE__, __LINE__, #cond);      \
            return;                                     \
        }                                               \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                               \
    do {                                                                          \
        bool caught_ = false;                                                     \
        try {                                                                     \
            (void)(expr);                                                         \
        } catch (const type&) {                                                   \
            caught_ = true;                                                       \
        } catch (...) {                                                           \
        }                                                                         \
        if (!caught_) mini::fail(__FILE__, __LINE__, "expected " #type ": " #expr); \
    } while (0)
