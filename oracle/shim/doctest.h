// Minimal doctest-API shim — TEST INFRASTRUCTURE ONLY (oracle/).
// The reference expects vendor/doctest.h (proj/CMakeLists.txt:12), which is
// git-ignored upstream (proj/.gitignore:2) and absent here.  This covers the
// macros the reference's unit tests use: TEST_CASE, SUBCASE (re-run
// semantics, one level), CHECK, CHECK_FALSE, REQUIRE, FAIL, Approx().epsilon,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS and Contains.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx epsilon(double e) const {
    Approx a(*this);
    a.eps_ = e;
    return a;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(const char* str) : s(str) {}
  bool check(const std::string& what) const { return what.find(s) != std::string::npos; }
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

struct Reg {
  Reg(const char* name, void (*fn)(), const char* file, int line) { registry().push_back({name, fn, file, line}); }
};

struct State {
  int failures = 0;
  int checks = 0;
  int subTarget = 0;
  int subSeen = 0;
  bool testFailed = false;
};
inline State& st() {
  static State s;
  return s;
}

struct RequireAbort {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++st().checks;
  if (ok) return;
  ++st().failures;
  st().testFailed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (fatal) throw RequireAbort{};
}

inline bool enterSubcase() { return st().subSeen++ == st().subTarget; }

inline int runAll() {
  int failedCases = 0;
  for (const auto& tc : registry()) {
    st().testFailed = false;
    int target = 0;
    while (true) {
      st().subTarget = target;
      st().subSeen = 0;
      try {
        tc.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: exception in '%s': %s\n", tc.file, tc.line, tc.name, e.what());
        ++st().failures;
        st().testFailed = true;
      }
      if (st().subSeen <= target + 1) break;
      ++target;
    }
    if (st().testFailed) {
      ++failedCases;
      std::fprintf(stderr, "test case FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              registry().size(), registry().size() - failedCases, failedCases, st().checks, st().failures);
  return failedCases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(name, f)                                                           \
  static void f();                                                                         \
  static doctest::detail::Reg DOCTEST_CAT(f, _reg)(name, f, __FILE__, __LINE__);           \
  static void f()
#define TEST_CASE(name) DOCTEST_TC_IMPL(name, DOCTEST_CAT(doctest_tc_, __COUNTER__))
#define SUBCASE(name) if (doctest::detail::enterSubcase())
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                      \
  do {                                                                                   \
    bool ok_ = false;                                                                    \
    try {                                                                                \
      expr;                                                                              \
    } catch (const type&) {                                                              \
      ok_ = true;                                                                        \
    } catch (...) {                                                                      \
    }                                                                                    \
    doctest::detail::report(ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                        \
  do {                                                                                   \
    bool ok_ = false;                                                                    \
    try {                                                                                \
      expr;                                                                              \
    } catch (const type& e_) {                                                           \
      ok_ = (matcher).check(e_.what());                                                  \
    } catch (...) {                                                                      \
    }                                                                                    \
    doctest::detail::report(ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::runAll(); }
#endif
