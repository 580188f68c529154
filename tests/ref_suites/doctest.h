// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's own C++ suites (/root/reference/proj/tests/test_*.cpp) include "doctest.h",
// which the reference does not vendor (its vendor/ directory is git-ignored).  This shim
// implements the subset those suites use -- TEST_CASE, SUBCASE (doctest's re-run-per-leaf
// semantics), CHECK / CHECK_FALSE / REQUIRE / CHECK_EQ-style comparisons, CHECK_THROWS_AS /
// CHECK_NOTHROW / CHECK_THROWS, doctest::Approx, MESSAGE / INFO / CAPTURE -- so the suites compile
// unchanged against this repository's headers and link against libflexquant_b200.so.
// Written for this repository; it is not doctest's source.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
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
  bool matches(double x) const {
    return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }
  friend bool operator<=(double x, const Approx& a) { return x < a.value_ || a.matches(x); }
  friend bool operator>=(double x, const Approx& a) { return x > a.value_ || a.matches(x); }
  friend std::ostream& operator<<(std::ostream& os, const Approx& a) { return os << "Approx(" << a.value_ << ")"; }

 private:
  double value_;
  double eps_ = 1.1920929e-7f * 100;  // doctest's default epsilon
  double scale_ = 1.0;
};

namespace detail {

struct RequireFailed {};

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

struct State {
  int failures = 0, checks = 0;
  // subcase bookkeeping: one leaf path is entered per run of a test case
  std::vector<std::string> path;           // subcases entered in this run
  std::set<std::vector<std::string>> done;  // leaf paths already run
  bool entered_new = false;                 // this run entered a not-yet-finished subcase
  std::vector<std::string> messages;        // INFO / CAPTURE context
};

inline State& state() {
  static State s;
  return s;
}

inline bool register_test(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return true;
}

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  for (const std::string& m : s.messages) std::fprintf(stderr, "    with: %s\n", m.c_str());
  if (require) throw RequireFailed{};
}

// SUBCASE: entered if its path extended by this name has unfinished leaves and no other
// subcase at this level was entered during this run.
class Subcase {
 public:
  Subcase(const char* name) {
    State& s = state();
    std::vector<std::string> p = s.path;
    p.push_back(name);
    if (s.entered_new || s.done.count(p)) {
      entered_ = false;
      return;
    }
    entered_ = true;
    s.path = p;
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = state();
    // a leaf finishes when no nested subcase was entered under it in this run
    if (!s.entered_new) s.done.insert(s.path);
    s.entered_new = true;
    s.path.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
};

struct MessageScope {
  explicit MessageScope(std::string m) { state().messages.push_back(std::move(m)); }
  ~MessageScope() { state().messages.pop_back(); }
};

template <class... T>
std::string concat(const T&... v) {
  std::ostringstream os;
  (os << ... << v);
  return os.str();
}

inline int run_all() {
  State& s = state();
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    s.done.clear();
    const int before = s.failures;
    for (int run = 0; run < 10000; ++run) {
      s.path.clear();
      s.entered_new = false;
      s.messages.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", tc.file, tc.line, tc.name, e.what());
      }
      if (!s.entered_new) break;  // no subcase left to enter
    }
    if (s.failures != before) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest-shim] FAILED test case: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %d | failed checks: %d\n", registry().size(),
              failed_cases, s.checks, s.failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                          \
  static void fn();                                                                              \
  static const bool DOCTEST_CAT(fn, _reg) = doctest::detail::register_test(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define DOCTEST_CHECK_IMPL(expr, text, req) doctest::detail::report(static_cast<bool>(expr), text, __FILE__, __LINE__, req)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), #__VA_ARGS__, true)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", false)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", true)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define CHECK_NE(a, b) CHECK((a) != (b))
#define CHECK_LT(a, b) CHECK((a) < (b))
#define CHECK_LE(a, b) CHECK((a) <= (b))
#define CHECK_GT(a, b) CHECK((a) > (b))
#define CHECK_GE(a, b) CHECK((a) >= (b))
#define REQUIRE_EQ(a, b) REQUIRE((a) == (b))
#define DOCTEST_THROWS_IMPL(expr, type, text, req)                                   \
  do {                                                                              \
    bool doctest_ok = false;                                                        \
    try {                                                                           \
      static_cast<void>(expr);                                                      \
    } catch (const type&) {                                                         \
      doctest_ok = true;                                                            \
    } catch (...) {                                                                 \
    }                                                                               \
    doctest::detail::report(doctest_ok, text, __FILE__, __LINE__, req);             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_IMPL(expr, __VA_ARGS__, #expr " throws " #__VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_IMPL(expr, __VA_ARGS__, #expr " throws " #__VA_ARGS__, true)
#define CHECK_THROWS(expr) DOCTEST_THROWS_IMPL(expr, std::exception, #expr " throws", false)
#define CHECK_NOTHROW(expr)                                                          \
  do {                                                                              \
    bool doctest_ok = true;                                                         \
    try {                                                                           \
      static_cast<void>(expr);                                                      \
    } catch (...) {                                                                 \
      doctest_ok = false;                                                           \
    }                                                                               \
    doctest::detail::report(doctest_ok, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)
#define MESSAGE(...) std::fprintf(stderr, "%s:%d: MESSAGE: %s\n", __FILE__, __LINE__, doctest::detail::concat(__VA_ARGS__).c_str())
#define INFO(...) const doctest::detail::MessageScope DOCTEST_CAT(doctest_info_, __LINE__)(doctest::detail::concat(__VA_ARGS__))
#define CAPTURE(x) INFO(#x " := ", x)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
