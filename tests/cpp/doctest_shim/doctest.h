// Minimal doctest-compatible test harness (the subset the operator tests use:
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS
// with doctest::Contains).  doctest itself is not vendored in the reference
// tree (proj/.gitignore:2), so this lets both our own C++ tests and the
// reference's unmodified tests/test_conv_core.cpp build and run here.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

namespace detail {
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
inline int& checks() {
    static int c = 0;
    return c;
}
struct Register {
    Register(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
    ++checks();
    if (!ok) {
        ++failures();
        std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
        if (require) throw RequireFailed{};
    }
}
inline bool message_matches(const std::exception& e, const Contains& c) { return c.matches(e.what()); }
inline bool message_matches(const std::exception& e, const char* s) { return std::string(e.what()) == s; }
}  // namespace detail

inline int run_all() {
    int failed_cases = 0;
    for (auto& c : detail::registry()) {
        const int before = detail::failures();
        try {
            c.fn();
        } catch (const detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++detail::failures();
            std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
        }
        if (detail::failures() != before) {
            ++failed_cases;
            std::fprintf(stderr, "[FAIL] %s\n", c.name);
        } else {
            std::printf("[ok] %s\n", c.name);
        }
    }
    std::printf("test cases: %zu | %zu passed | %d failed; assertions: %d | %d failed\n",
                detail::registry().size(), detail::registry().size() - failed_cases, failed_cases,
                detail::checks(), detail::failures());
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                          \
    static void fn();                                                              \
    static doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, fn);              \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, exc)                                                        \
    do {                                                                                  \
        bool doctest_ok_ = false;                                                         \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (const exc&) {                                                            \
            doctest_ok_ = true;                                                           \
        } catch (...) {                                                                   \
        }                                                                                 \
        doctest::detail::report(doctest_ok_, "throws " #exc ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, with, exc)                                             \
    do {                                                                                  \
        bool doctest_ok_ = false;                                                         \
        try {                                                                             \
            static_cast<void>(expr);                                                      \
        } catch (const exc& e_) {                                                         \
            doctest_ok_ = doctest::detail::message_matches(e_, with);                     \
        } catch (...) {                                                                   \
        }                                                                                 \
        doctest::detail::report(doctest_ok_, "throws " #exc " with message: " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
