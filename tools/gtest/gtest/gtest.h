// gtest.h — a small self-written subset of the GoogleTest API, enough to
// compile the reference's own unit tests (proj/tests/*.cpp, unmodified)
// against the drop-in headers (include/rlra) and run them on the B200 engine.
//
// Covered: TEST, EXPECT_/ASSERT_ {EQ, NE, LT, LE, GT, GE, TRUE, FALSE, NEAR,
// DOUBLE_EQ, THROW, NO_THROW}, FAIL, SUCCEED, streamed failure messages,
// ::testing::TempDir, and a main() with gtest-style output and a simple
// --gtest_filter (':'-separated globs, '-' for negative patterns).  Not a
// copy of GoogleTest: the semantics follow its documentation (DOUBLE_EQ is
// "within 4 ULPs", TempDir honours TEST_TMPDIR and ends with '/').
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

inline std::string TempDir() {
    const char* e = std::getenv("TEST_TMPDIR");
    std::string d = (e && *e) ? e : "/tmp/";
    if (d.back() != '/') d.push_back('/');
    return d;
}

namespace internal {

struct TestInfo {
    const char* suite;
    const char* name;
    void (*fn)();
};

inline std::vector<TestInfo>& registry() {
    static std::vector<TestInfo> r;
    return r;
}

inline int& current_failures() {
    static int n = 0;
    return n;
}

struct Registrar {
    Registrar(const char* suite, const char* name, void (*fn)()) { registry().push_back({suite, name, fn}); }
};

template <class T>
std::string print(const T& v) {
    if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
        std::ostringstream s;
        s.precision(17);
        if constexpr (std::is_same_v<T, bool>)
            s << (v ? "true" : "false");
        else
            s << v;
        return s.str();
    } else {
        return "<unprintable>";
    }
}

struct Result {
    bool ok = true;
    std::string msg;
    explicit operator bool() const { return ok; }
};

struct Msg {
    std::ostringstream ss;
    template <class T>
    Msg& operator<<(const T& v) {
        ss << v;
        return *this;
    }
    Msg& operator<<(std::ostream& (*f)(std::ostream&)) {
        ss << f;
        return *this;
    }
};

struct Reporter {
    const char* file;
    int line;
    std::string text;
    void operator=(const Msg& m) const {
        ++current_failures();
        std::string extra = m.ss.str();
        std::printf("%s:%d: Failure\n%s\n%s%s", file, line, text.c_str(), extra.c_str(), extra.empty() ? "" : "\n");
        std::fflush(stdout);
    }
};

#define RLRA_GT_CMP_(nm, op)                                                                     \
    template <class A, class B>                                                                  \
    Result nm(const A& a, const B& b, const char* ea, const char* eb) {                          \
        if (a op b) return {};                                                                   \
        return {false, std::string("Expected: (") + ea + ") " #op " (" + eb + "), actual: " +   \
                           print(a) + " vs " + print(b)};                                        \
    }
RLRA_GT_CMP_(cmp_eq, ==)
RLRA_GT_CMP_(cmp_ne, !=)
RLRA_GT_CMP_(cmp_lt, <)
RLRA_GT_CMP_(cmp_le, <=)
RLRA_GT_CMP_(cmp_gt, >)
RLRA_GT_CMP_(cmp_ge, >=)
#undef RLRA_GT_CMP_

inline Result cmp_bool(bool v, bool want, const char* e) {
    if (v == want) return {};
    return {false, std::string("Value of: ") + e + "\n  Actual: " + (v ? "true" : "false") +
                       "\nExpected: " + (want ? "true" : "false")};
}

inline Result cmp_near(double a, double b, double tol, const char* ea, const char* eb, const char* et) {
    const double d = std::fabs(a - b);
    if (d <= tol) return {};
    return {false, std::string("The difference between ") + ea + " and " + eb + " is " + print(d) +
                       ", which exceeds " + et + ", where\n" + ea + " evaluates to " + print(a) + ",\n" + eb +
                       " evaluates to " + print(b) + ", and\n" + et + " evaluates to " + print(tol) + "."};
}

// "almost equal": within 4 units in the last place (sign-magnitude distance)
inline Result cmp_double_eq(double a, double b, const char* ea, const char* eb) {
    auto biased = [](double x) {
        uint64_t u;
        std::memcpy(&u, &x, sizeof u);
        const uint64_t sign = uint64_t(1) << 63;
        return (u & sign) ? ~u + 1 : (u | sign);
    };
    if (!std::isnan(a) && !std::isnan(b)) {
        const uint64_t x = biased(a), y = biased(b);
        if ((x >= y ? x - y : y - x) <= 4) return {};
    }
    return {false, std::string("Expected equality of these values:\n  ") + ea + "\n    Which is: " + print(a) +
                       "\n  " + eb + "\n    Which is: " + print(b)};
}

template <class E, class F>
Result throws(F&& f, const char* stmt, const char* ename) {
    try {
        f();
    } catch (const E&) {
        return {};
    } catch (const std::exception& e) {
        return {false, std::string("Expected: ") + stmt + " throws an exception of type " + ename +
                           ".\n  Actual: it throws a different type (" + e.what() + ")."};
    } catch (...) {
        return {false, std::string("Expected: ") + stmt + " throws an exception of type " + ename +
                           ".\n  Actual: it throws a different type."};
    }
    return {false, std::string("Expected: ") + stmt + " throws an exception of type " + ename +
                       ".\n  Actual: it throws nothing."};
}

template <class F>
Result no_throw(F&& f, const char* stmt) {
    try {
        f();
    } catch (const std::exception& e) {
        return {false, std::string("Expected: ") + stmt + " doesn't throw an exception.\n  Actual: it throws (" +
                           e.what() + ")."};
    } catch (...) {
        return {false, std::string("Expected: ") + stmt + " doesn't throw an exception.\n  Actual: it throws."};
    }
    return {};
}

inline bool glob(const char* p, const char* s) {
    if (!*p) return !*s;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    if (*p == '?') return *s && glob(p + 1, s + 1);
    return *p == *s && glob(p + 1, s + 1);
}

inline bool any_glob(const std::string& pats, const std::string& name) {
    size_t b = 0;
    while (b <= pats.size()) {
        size_t e = pats.find(':', b);
        if (e == std::string::npos) e = pats.size();
        const std::string p = pats.substr(b, e - b);
        if (!p.empty() && glob(p.c_str(), name.c_str())) return true;
        b = e + 1;
    }
    return false;
}

inline bool selected(const std::string& filter, const std::string& name) {
    if (filter.empty()) return true;
    const size_t dash = filter.find('-');
    const std::string pos = filter.substr(0, dash), neg = dash == std::string::npos ? "" : filter.substr(dash + 1);
    return (pos.empty() || any_glob(pos, name)) && !(neg.size() && any_glob(neg, name));
}

inline int run_all(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i)
        if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
    std::vector<std::string> failed;
    int ran = 0;
    for (const TestInfo& t : registry()) {
        const std::string full = std::string(t.suite) + "." + t.name;
        if (!selected(filter, full)) continue;
        ++ran;
        current_failures() = 0;
        std::printf("[ RUN      ] %s\n", full.c_str());
        std::fflush(stdout);
        try {
            t.fn();
        } catch (const std::exception& e) {
            ++current_failures();
            std::printf("unknown file: Failure\nC++ exception with description \"%s\" thrown in the test body.\n",
                        e.what());
        } catch (...) {
            ++current_failures();
            std::printf("unknown file: Failure\nUnknown C++ exception thrown in the test body.\n");
        }
        if (current_failures()) {
            failed.push_back(full);
            std::printf("[  FAILED  ] %s\n", full.c_str());
        } else {
            std::printf("[       OK ] %s\n", full.c_str());
        }
        std::fflush(stdout);
    }
    std::printf("[==========] %d tests ran.\n", ran);
    std::printf("[  PASSED  ] %d tests.\n", ran - int(failed.size()));
    if (!failed.empty()) {
        std::printf("[  FAILED  ] %d tests, listed below:\n", int(failed.size()));
        for (const auto& f : failed) std::printf("[  FAILED  ] %s\n", f.c_str());
    }
    return failed.empty() ? 0 : 1;
}

}  // namespace internal

inline std::pair<int, char**>& saved_args() {
    static std::pair<int, char**> a{0, nullptr};
    return a;
}

inline void InitGoogleTest(int* argc, char** argv) { saved_args() = {*argc, argv}; }

}  // namespace testing

#define RLRA_GT_NONFATAL_(res, text)                    \
    if (const ::testing::internal::Result gt_r_ = (res)) \
        ;                                                \
    else                                                 \
        ::testing::internal::Reporter{__FILE__, __LINE__, gt_r_.msg} = ::testing::internal::Msg()
#define RLRA_GT_FATAL_(res, text)                        \
    if (const ::testing::internal::Result gt_r_ = (res)) \
        ;                                                \
    else                                                 \
        return ::testing::internal::Reporter{__FILE__, __LINE__, gt_r_.msg} = ::testing::internal::Msg()

#define TEST(suite, name)                                                                          \
    static void rlra_gt_##suite##_##name();                                                        \
    static ::testing::internal::Registrar rlra_gt_reg_##suite##_##name(#suite, #name,              \
                                                                         &rlra_gt_##suite##_##name); \
    static void rlra_gt_##suite##_##name()

#define EXPECT_EQ(a, b) RLRA_GT_NONFATAL_(::testing::internal::cmp_eq((a), (b), #a, #b), "")
#define EXPECT_NE(a, b) RLRA_GT_NONFATAL_(::testing::internal::cmp_ne((a), (b), #a, #b), "")
#define EXPECT_LT(a, b) RLRA_GT_NONFATAL_(::testing::internal::cmp_lt((a), (b), #a, #b), "")
#define EXPECT_LE(a, b) RLRA_GT_NONFATAL_(::testing::internal::cmp_le((a), (b), #a, #b), "")
#define EXPECT_GT(a, b) RLRA_GT_NONFATAL_(::testing::internal::cmp_gt((a), (b), #a, #b), "")
#define EXPECT_GE(a, b) RLRA_GT_NONFATAL_(::testing::internal::cmp_ge((a), (b), #a, #b), "")
#define EXPECT_TRUE(c) RLRA_GT_NONFATAL_(::testing::internal::cmp_bool(static_cast<bool>(c), true, #c), "")
#define EXPECT_FALSE(c) RLRA_GT_NONFATAL_(::testing::internal::cmp_bool(static_cast<bool>(c), false, #c), "")
#define EXPECT_NEAR(a, b, t) RLRA_GT_NONFATAL_(::testing::internal::cmp_near((a), (b), (t), #a, #b, #t), "")
#define EXPECT_DOUBLE_EQ(a, b) RLRA_GT_NONFATAL_(::testing::internal::cmp_double_eq((a), (b), #a, #b), "")
#define EXPECT_THROW(stmt, exc) \
    RLRA_GT_NONFATAL_(::testing::internal::throws<exc>([&] { stmt; }, #stmt, #exc), "")
#define EXPECT_NO_THROW(stmt) RLRA_GT_NONFATAL_(::testing::internal::no_throw([&] { stmt; }, #stmt), "")

#define ASSERT_EQ(a, b) RLRA_GT_FATAL_(::testing::internal::cmp_eq((a), (b), #a, #b), "")
#define ASSERT_NE(a, b) RLRA_GT_FATAL_(::testing::internal::cmp_ne((a), (b), #a, #b), "")
#define ASSERT_LT(a, b) RLRA_GT_FATAL_(::testing::internal::cmp_lt((a), (b), #a, #b), "")
#define ASSERT_LE(a, b) RLRA_GT_FATAL_(::testing::internal::cmp_le((a), (b), #a, #b), "")
#define ASSERT_GT(a, b) RLRA_GT_FATAL_(::testing::internal::cmp_gt((a), (b), #a, #b), "")
#define ASSERT_GE(a, b) RLRA_GT_FATAL_(::testing::internal::cmp_ge((a), (b), #a, #b), "")
#define ASSERT_TRUE(c) RLRA_GT_FATAL_(::testing::internal::cmp_bool(static_cast<bool>(c), true, #c), "")
#define ASSERT_FALSE(c) RLRA_GT_FATAL_(::testing::internal::cmp_bool(static_cast<bool>(c), false, #c), "")
#define ASSERT_NEAR(a, b, t) RLRA_GT_FATAL_(::testing::internal::cmp_near((a), (b), (t), #a, #b, #t), "")
#define ASSERT_DOUBLE_EQ(a, b) RLRA_GT_FATAL_(::testing::internal::cmp_double_eq((a), (b), #a, #b), "")
#define ASSERT_THROW(stmt, exc) RLRA_GT_FATAL_(::testing::internal::throws<exc>([&] { stmt; }, #stmt, #exc), "")
#define ASSERT_NO_THROW(stmt) RLRA_GT_FATAL_(::testing::internal::no_throw([&] { stmt; }, #stmt), "")

#define FAIL() \
    return ::testing::internal::Reporter{__FILE__, __LINE__, "Failed"} = ::testing::internal::Msg()
#define ADD_FAILURE() ::testing::internal::Reporter{__FILE__, __LINE__, "Failed"} = ::testing::internal::Msg()
#define SUCCEED() static_cast<void>(0)
#define RUN_ALL_TESTS() ::testing::internal::run_all(::testing::saved_args().first, ::testing::saved_args().second)
