// doctest.h -- a small doctest-compatible test runner (test infrastructure).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) are written against the
// third-party doctest framework, which this image does not ship. This header implements the
// subset those files use, with doctest's semantics, so they compile unchanged:
//   TEST_CASE, single-level SUBCASE (the test body re-runs once per subcase, entering one
//   subcase per run), CHECK, CHECK_FALSE, REQUIRE (aborts the test case), CHECK_THROWS_AS,
//   CHECK_THROWS_WITH_AS with doctest::Contains,
//   doctest::Approx(v).epsilon(e) (|a - b| < eps * (1 + max(|a|, |b|)), default eps =
//   100 * FLT_EPSILON), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// The runner takes --exclude=pat1,pat2 (substring match on test-case names) and --list.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
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
    bool matches(double x) const {
        return std::fabs(x - v_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(v_)));
    }
    double value() const { return v_; }

  private:
    double v_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};
// String matcher for CHECK_THROWS_WITH_AS: the exception's what() contains the text.
struct Contains {
    explicit Contains(const char* s) : text(s) {}
    std::string text;
    bool matches(const char* what) const { return std::strstr(what, text.c_str()) != nullptr; }
};

inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

}  // namespace doctest

namespace doctest_lite {

struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

struct State {
    std::vector<Case> cases;
    int target = 0;        // subcase entered in this run
    int seen = 0;          // subcases met in this run
    std::string subcase;   // name of the entered subcase
    long assertions = 0, failed_assertions = 0;
    bool case_failed = false;
    const char* case_name = "";
};
inline State& state() {
    static State s;
    return s;
}

struct Reg {
    Reg(const char* name, void (*fn)(), const char* file, int line) { state().cases.push_back({name, fn, file, line}); }
};

struct Abort {};  // REQUIRE failure

inline void fail(const char* file, int line, const char* what) {
    State& s = state();
    ++s.failed_assertions;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\"%s%s%s: %s\n", file, line, s.case_name,
                 s.subcase.empty() ? "" : " [", s.subcase.c_str(), s.subcase.empty() ? "" : "]", what);
}

inline void check(bool ok, const char* file, int line, const char* what, bool require) {
    ++state().assertions;
    if (ok) return;
    fail(file, line, what);
    if (require) throw Abort{};
}

class Subcase {
  public:
    explicit Subcase(const char* name) {
        State& s = state();
        entered_ = s.seen++ == s.target;
        if (entered_) s.subcase = name;
    }
    explicit operator bool() const { return entered_; }

  private:
    bool entered_;
};

inline int run(int argc, char** argv) {
    std::vector<std::string> excl;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--exclude=", 0) == 0) {
            std::string rest = a.substr(10);
            size_t p;
            while ((p = rest.find(',')) != std::string::npos) {
                excl.push_back(rest.substr(0, p));
                rest = rest.substr(p + 1);
            }
            if (!rest.empty()) excl.push_back(rest);
        } else if (a == "--list") {
            list = true;
        }
    }
    State& s = state();
    int passed = 0, failed = 0, skipped = 0;
    for (const Case& c : s.cases) {
        bool skip = false;
        for (const std::string& e : excl)
            if (std::strstr(c.name, e.c_str())) skip = true;
        if (list) {
            std::printf("%s%s\n", c.name, skip ? "  (excluded)" : "");
            continue;
        }
        if (skip) {
            ++skipped;
            continue;
        }
        s.case_name = c.name;
        s.case_failed = false;
        for (s.target = 0;; ++s.target) {
            s.seen = 0;
            s.subcase.clear();
            try {
                c.fn();
            } catch (const Abort&) {
            } catch (const std::exception& e) {
                fail(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
            } catch (...) {
                fail(c.file, c.line, "unexpected exception");
            }
            if (s.target + 1 >= s.seen) break;  // every subcase entered once (or none exist)
        }
        (s.case_failed ? failed : passed) += 1;
    }
    if (list) return 0;
    std::printf("[doctest-lite] test cases: %d passed, %d failed, %d skipped | assertions: %ld, %ld failed\n", passed,
                failed, skipped, s.assertions, s.failed_assertions);
    return failed ? 1 : 0;
}

}  // namespace doctest_lite

#define DOCTEST_LITE_CAT_(a, b) a##b
#define DOCTEST_LITE_CAT(a, b) DOCTEST_LITE_CAT_(a, b)
#define DOCTEST_LITE_TC(fn, name)                                                   \
    static void fn();                                                               \
    static const ::doctest_lite::Reg DOCTEST_LITE_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DOCTEST_LITE_TC(DOCTEST_LITE_CAT(doctest_lite_case_, __LINE__), name)
#define SUBCASE(name) if (const ::doctest_lite::Subcase DOCTEST_LITE_CAT(doctest_lite_sub_, __LINE__){name})
#define CHECK(...) ::doctest_lite::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )", false)
#define CHECK_FALSE(...) \
    ::doctest_lite::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "CHECK_FALSE( " #__VA_ARGS__ " )", false)
#define REQUIRE(...) \
    ::doctest_lite::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )", true)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool doctest_lite_ok = false;                                                              \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_lite_ok = true;                                                                \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest_lite::check(doctest_lite_ok, __FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )", \
                              false);                                                              \
    } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                                   \
    do {                                                                                           \
        bool doctest_lite_ok = false;                                                              \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__& doctest_lite_e) {                                              \
            doctest_lite_ok = (matcher).matches(doctest_lite_e.what());                            \
        } catch (...) {                                                                            \
        }                                                                                          \
        ::doctest_lite::check(doctest_lite_ok, __FILE__, __LINE__,                                 \
                              "CHECK_THROWS_WITH_AS( " #expr ", " #matcher ", " #__VA_ARGS__ " )", false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest_lite::run(argc, argv); }
#endif
