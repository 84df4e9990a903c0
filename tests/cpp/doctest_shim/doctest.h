// doctest.h — a minimal doctest-compatible test harness (our own, not the
// doctest library, which is absent from this image). It implements exactly
// the subset the reference suite's path tests use, with doctest's semantics,
// so /root/reference/proj/tests/{test_head,test_selector,test_token_set,
// test_offload_sim}.cpp compile UNCHANGED against the B200 drop-in
// (include/subvocab/*.hpp -> lib/libsubvocab_b200.so):
//
//   TEST_CASE(name) { ... }          registered, run in declaration order
//   SUBCASE(name) { ... }            doctest's model: the test case is re-run
//                                    once per leaf subcase path
//   CHECK / CHECK_FALSE / REQUIRE    REQUIRE aborts the test case
//   CHECK_THROWS_AS(expr, Type...)   CHECK_NOTHROW(expr)
//   doctest::Approx(v)               |a - b| < eps * (scale + max(|a|, |b|)),
//                                    eps = 100 * FLT_EPSILON, scale = 1
//
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (doctest_main.cpp) emits main(): runs
// every test case (optionally only those whose name contains argv[1]),
// prints failures and a summary, returns 1 when anything failed.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <set>
#include <string>
#include <utility>
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
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.eq(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.eq(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.eq(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.eq(rhs); }

private:
    bool eq(double x) const {
        return std::fabs(x - value_) <
               eps_ * (scale_ + std::fmax(std::fabs(x), std::fabs(value_)));
    }
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

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
inline int reg(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
    return 0;
}

struct Stats {
    long checks = 0, failed_checks = 0;
    bool current_failed = false;
    const char* current = "";
};
inline Stats& stats() {
    static Stats s;
    return s;
}

struct RequireFailed {};

inline void fail(const char* what, const char* expr, const char* file, int line,
                 const char* extra = nullptr) {
    Stats& s = stats();
    ++s.failed_checks;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s  [test case \"%s\"]\n", file, line, what, expr,
                 extra ? ": " : "", extra ? extra : "", s.current);
}
inline void check(bool ok, const char* what, const char* expr, const char* file, int line,
                  bool require) {
    ++stats().checks;
    if (ok) return;
    fail(what, expr, file, line);
    if (require) throw RequireFailed{};
}

// ---- subcases: doctest's re-run model -------------------------------------
using Key = std::pair<std::string, int>;
struct SubcaseRun {
    std::set<std::vector<Key>> done;   // explored paths (whole test case)
    std::vector<Key> stack;            // path of the subcases entered now
    std::vector<bool> child_pending;   // per entered level: a child still to run
    std::vector<bool> took;            // per depth: a subcase was entered this run
    bool pending = false;              // another run is needed
};
inline SubcaseRun& sub() {
    static SubcaseRun r;
    return r;
}

class Subcase {
public:
    Subcase(const char* name, const char* /*file*/, int line) {
        SubcaseRun& r = sub();
        const std::size_t depth = r.stack.size();
        if (r.took.size() <= depth) r.took.resize(depth + 1, false);
        path_ = r.stack;
        path_.emplace_back(name, line);
        if (r.took[depth]) {
            // a sibling ran in this pass: this one waits for a later pass
            if (!r.done.count(path_)) {
                r.pending = true;
                if (depth > 0) r.child_pending[depth - 1] = true;
            }
            return;
        }
        if (r.done.count(path_)) return;
        entered_ = true;
        r.took[depth] = true;
        r.took.resize(depth + 1);
        r.stack.push_back(path_.back());
        r.child_pending.push_back(false);
    }
    ~Subcase() {
        if (!entered_) return;
        SubcaseRun& r = sub();
        const bool cp = r.child_pending.back();
        r.child_pending.pop_back();
        r.stack.pop_back();
        if (!cp)
            r.done.insert(path_);
        else if (!r.child_pending.empty())
            r.child_pending.back() = true;
    }
    Subcase(const Subcase&) = delete;
    Subcase& operator=(const Subcase&) = delete;
    explicit operator bool() const { return entered_; }

private:
    std::vector<Key> path_;
    bool entered_ = false;
};

inline int run_all(const char* filter) {
    Stats& s = stats();
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        if (filter && !std::strstr(tc.name, filter)) continue;
        ++cases;
        s.current = tc.name;
        s.current_failed = false;
        SubcaseRun& r = sub();
        r = SubcaseRun{};
        for (int pass = 0; pass < 100000; ++pass) {
            r.stack.clear();
            r.child_pending.clear();
            r.took.clear();
            r.pending = false;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                fail("TEST_CASE", tc.name, tc.file, tc.line, e.what());
            } catch (...) {
                fail("TEST_CASE", tc.name, tc.file, tc.line, "unknown exception");
            }
            if (!r.pending) break;
        }
        if (s.current_failed) ++failed_cases;
    }
    std::printf("[doctest shim] test cases: %d | %d passed | %d failed\n", cases,
                cases - failed_cases, failed_cases);
    std::printf("[doctest shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
                s.checks - s.failed_checks, s.failed_checks);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)

#define DOCTEST_TC_IMPL(name, fn)                                                          \
    static void fn();                                                                      \
    [[maybe_unused]] static const int DOCTEST_CAT(fn, _reg) =                              \
        doctest::detail::reg(name, &fn, __FILE__, __LINE__);                               \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(name, DOCTEST_CAT(doctest_tc_, __COUNTER__))

#define SUBCASE(name)                                                                      \
    if (const doctest::detail::Subcase& DOCTEST_CAT(doctest_sc_, __COUNTER__) =            \
            doctest::detail::Subcase(name, __FILE__, __LINE__))

#define CHECK(...) \
    doctest::detail::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
    doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) \
    doctest::detail::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        ++doctest::detail::stats().checks;                                                  \
        bool doctest_thrown_ = false;                                                       \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const __VA_ARGS__&) {                                                      \
            doctest_thrown_ = true;                                                         \
        } catch (...) {                                                                     \
            doctest::detail::fail("CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__,     \
                                  __LINE__, "threw a different type");                      \
            doctest_thrown_ = true;                                                         \
        }                                                                                   \
        if (!doctest_thrown_)                                                               \
            doctest::detail::fail("CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__,     \
                                  __LINE__, "did not throw");                               \
    } while (0)

#define CHECK_NOTHROW(...)                                                                  \
    do {                                                                                    \
        ++doctest::detail::stats().checks;                                                  \
        try {                                                                               \
            static_cast<void>(__VA_ARGS__);                                                 \
        } catch (...) {                                                                     \
            doctest::detail::fail("CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__,        \
                                  "threw");                                                 \
        }                                                                                   \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc > 1 ? argv[1] : nullptr); }
#endif
