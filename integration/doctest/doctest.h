// Minimal doctest-compatible test harness (the subset the reference's
// scheduler tests use: TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE,
// CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx).  doctest itself is not in
// this image; this shim lets the reference's own test sources compile
// unmodified against the B200 binding (integration/d2ft_b200_binding.cpp).
// SUBCASE semantics follow doctest: the test case body is re-run once per
// leaf subcase (single nesting level).
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
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& r) {
    return std::fabs(lhs - r.v_) < r.eps_ * (r.scale_ + std::max(std::fabs(lhs), std::fabs(r.v_)));
  }
  friend bool operator==(const Approx& r, double lhs) { return lhs == r; }
  friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
  friend bool operator!=(const Approx& r, double lhs) { return !(lhs == r); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct State {
  long checks = 0, failures = 0;
  std::vector<std::string> done;
  bool entered = false;
  std::string current;
};
inline State& st() {
  static State s;
  return s;
}
struct RequireFailed {};
struct Subcase {
  bool active = false;
  explicit Subcase(const char* name) {
    State& s = st();
    const std::string n(name);
    if (!s.entered && std::find(s.done.begin(), s.done.end(), n) == s.done.end()) {
      s.entered = true;
      s.current = n;
      active = true;
    }
  }
  ~Subcase() {
    if (active) st().done.push_back(st().current);
  }
  explicit operator bool() const { return active; }
};
inline void check(bool ok, const char* expr, const char* file, int line, bool require = false) {
  State& s = st();
  ++s.checks;
  if (!ok) {
    ++s.failures;
    std::printf("%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
  }
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(name, fn)                                                  \
  static void fn();                                                            \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, fn);                 \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(name, DOCTEST_CAT(doctest_tc_, __COUNTER__))
#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::detail::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool ok_ = false;                                                                     \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      ok_ = true;                                                                         \
    } catch (...) {                                                                       \
    }                                                                                     \
    doctest::detail::check(ok_, "THROWS_AS " #expr, __FILE__, __LINE__);                 \
  } while (0)
#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    bool ok_ = true;                                                                      \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (...) {                                                                       \
      ok_ = false;                                                                        \
    }                                                                                     \
    doctest::detail::check(ok_, "NOTHROW " #expr, __FILE__, __LINE__);                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    State& s = st();
    s.done.clear();
    const long before = s.failures;
    bool again = true;
    while (again) {
      s.entered = false;
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("test case \"%s\": unexpected exception: %s\n", tc.name, e.what());
      }
      again = s.entered;
    }
    if (s.failures != before) ++failed_cases;
    std::printf("[%s] %s\n", s.failures == before ? "PASS" : "FAIL", tc.name);
  }
  std::printf("test cases: %zu | failed: %d | checks: %ld | failed checks: %ld\n", registry().size(), failed_cases,
              st().checks, st().failures);
  return failed_cases ? 1 : 0;
}
#endif
