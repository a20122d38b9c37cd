// TEST INFRASTRUCTURE. A tiny GoogleTest-compatible harness (GoogleTest is
// not in this image) covering exactly the macros the reference's unit tests
// use: TEST, EXPECT_/ASSERT_{EQ,NE,LT,LE,GT,GE,TRUE,FALSE}, EXPECT_NEAR,
// EXPECT_DOUBLE_EQ, EXPECT_THROW,
// EXPECT_NO_THROW, and `<< message` streaming after any of them. Used to
// compile the reference's own unit-test sources, unmodified, against this
// repo's drop-in headers (include/acmatch/*.hpp) — see oracle/Makefile.
//
// The runner (minitest_main.cpp) accepts --gtest_filter=Prefix* style
// filters (':'-separated, '*' only as a trailing wildcard, '-' negation).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace minitest {

struct Case {
    std::string suite, name;
    std::function<void()> body;
};

inline std::vector<Case>& registry() {
    static std::vector<Case> cases;
    return cases;
}

inline int& failures_in_case() {
    static int n = 0;
    return n;
}

struct Registrar {
    Registrar(const char* suite, const char* name, void (*fn)()) { registry().push_back({suite, name, fn}); }
};

template <class T>
concept Streamable = requires(std::ostream& os, const T& v) { os << v; };

template <class T>
std::string show(const T& v) {
    if constexpr (Streamable<T>) {
        std::ostringstream os;
        os << v;
        return os.str();
    } else {
        return "<unprintable>";
    }
}

// Collects the user's `<< ...` text.
struct Message {
    std::ostringstream os;
    template <class T>
    Message& operator<<(const T& v) {
        os << v;
        return *this;
    }
};

// `Reporter(...) = Message() << ...` prints the failure; yields void so that
// ASSERT_* can `return` it from a void test body.
struct Reporter {
    const char* file;
    int line;
    std::string what;
    void operator=(const Message& m) const {
        ++failures_in_case();
        const std::string extra = m.os.str();
        std::fprintf(stderr, "%s:%d: Failure\n%s%s%s\n", file, line, what.c_str(), extra.empty() ? "" : "\n  ",
                     extra.c_str());
    }
};

// Evaluated comparison: empty string on success, else a description.
template <class A, class B, class Op>
std::string compare(const A& a, const B& b, Op op, const char* ea, const char* eb, const char* sym) {
    if (op(a, b)) return {};
    return std::string("Expected: (") + ea + ") " + sym + " (" + eb + ")\n  actual: " + show(a) + " vs " + show(b);
}

inline bool ulp_eq(double x, double y) {
    if (x == y) return true;
    if (std::isnan(x) || std::isnan(y)) return false;
    auto key = [](double d) {
        std::int64_t i;
        std::memcpy(&i, &d, sizeof i);
        return i < 0 ? std::numeric_limits<std::int64_t>::min() - i : i;
    };
    const std::int64_t a = key(x), b = key(y);
    return (a > b ? a - b : b - a) <= 4;
}

}  // namespace minitest

#define MINITEST_CAT2(a, b) a##b
#define MINITEST_CAT(a, b) MINITEST_CAT2(a, b)

#define TEST(suite, name)                                                                         \
    static void MINITEST_CAT(minitest_body_, MINITEST_CAT(suite, MINITEST_CAT(_, name)))();       \
    static ::minitest::Registrar MINITEST_CAT(minitest_reg_, MINITEST_CAT(suite, MINITEST_CAT(_, name)))( \
        #suite, #name, &MINITEST_CAT(minitest_body_, MINITEST_CAT(suite, MINITEST_CAT(_, name))));         \
    static void MINITEST_CAT(minitest_body_, MINITEST_CAT(suite, MINITEST_CAT(_, name)))()

#define MINITEST_CHECK(text_expr, on_fail)                           \
    if (const std::string minitest_what = (text_expr); minitest_what.empty()) \
        ;                                                            \
    else                                                             \
        on_fail ::minitest::Reporter{__FILE__, __LINE__, minitest_what} = ::minitest::Message()

#define MINITEST_CMP(a, b, sym, on_fail) \
    MINITEST_CHECK(::minitest::compare((a), (b), [](const auto& x, const auto& y) { return x sym y; }, #a, #b, #sym), on_fail)

#define EXPECT_EQ(a, b) MINITEST_CMP(a, b, ==, )
#define EXPECT_NE(a, b) MINITEST_CMP(a, b, !=, )
#define EXPECT_LT(a, b) MINITEST_CMP(a, b, <, )
#define EXPECT_LE(a, b) MINITEST_CMP(a, b, <=, )
#define EXPECT_GT(a, b) MINITEST_CMP(a, b, >, )
#define EXPECT_GE(a, b) MINITEST_CMP(a, b, >=, )
#define ASSERT_EQ(a, b) MINITEST_CMP(a, b, ==, return)
#define ASSERT_NE(a, b) MINITEST_CMP(a, b, !=, return)
#define ASSERT_LT(a, b) MINITEST_CMP(a, b, <, return)
#define ASSERT_LE(a, b) MINITEST_CMP(a, b, <=, return)
#define ASSERT_GT(a, b) MINITEST_CMP(a, b, >, return)
#define ASSERT_GE(a, b) MINITEST_CMP(a, b, >=, return)

// |a-b| <= tol, and equality within 4 ulps for doubles
#define EXPECT_NEAR(a, b, tol) \
    MINITEST_CHECK(::minitest::compare((a), (b), [&](double x, double y) { return std::fabs(x - y) <= (tol); }, #a, #b, "~="), )
#define EXPECT_DOUBLE_EQ(a, b) \
    MINITEST_CHECK(::minitest::compare((a), (b), [](double x, double y) { return ::minitest::ulp_eq(x, y); }, #a, #b, "=="), )

#define MINITEST_BOOL(c, want, on_fail) \
    MINITEST_CHECK((static_cast<bool>(c) == (want)) ? std::string() : std::string("Value of: " #c "\n  expected: " #want), on_fail)

#define EXPECT_TRUE(c) MINITEST_BOOL(c, true, )
#define EXPECT_FALSE(c) MINITEST_BOOL(c, false, )
#define ASSERT_TRUE(c) MINITEST_BOOL(c, true, return)
#define ASSERT_FALSE(c) MINITEST_BOOL(c, false, return)

#define EXPECT_THROW(stmt, exc)                                                             \
    MINITEST_CHECK(([&]() -> std::string {                                                  \
                       try {                                                                \
                           stmt;                                                            \
                       } catch (const exc&) {                                               \
                           return {};                                                       \
                       } catch (const std::exception& e) {                                  \
                           return std::string("Expected " #stmt " to throw " #exc ", got: ") + e.what(); \
                       } catch (...) {                                                      \
                           return "Expected " #stmt " to throw " #exc ", got another type"; \
                       }                                                                    \
                       return "Expected " #stmt " to throw " #exc ", nothing thrown";       \
                   }()),                                                                    \
                   )

#define EXPECT_NO_THROW(stmt)                                                   \
    MINITEST_CHECK(([&]() -> std::string {                                      \
                       try {                                                    \
                           stmt;                                                \
                       } catch (const std::exception& e) {                      \
                           return std::string(#stmt " threw: ") + e.what();     \
                       } catch (...) {                                          \
                           return #stmt " threw a non-std exception";           \
                       }                                                        \
                       return {};                                               \
                   }()),                                                        \
                   )
