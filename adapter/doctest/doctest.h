// doctest.h — a minimal stand-in for the doctest single-header framework
// (doctest is not installed in this image).  It implements
// exactly the subset the reference's unit tests use — TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, CHECK_THROWS_AS, INFO, doctest::Approx and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so proj/tests/*.cpp compile unchanged
// against the liveput adapter (adapter/optimizer.cpp).  Test infrastructure.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
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
  friend bool operator==(double lhs, const Approx& a) {
    // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|)), scale 1
    return std::fabs(lhs - a.v_) < a.eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
};

namespace detail {
struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
  std::string info;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};
template <class... A>
std::string cat(const A&... a) {
  std::ostringstream o;
  (o << ... << a);
  return o.str();
}
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED: %s%s%s\n", file, line, expr, s.info.empty() ? "" : "  [info: ",
               s.info.empty() ? "" : (s.info + "]").c_str());
  if (require) throw RequireFailed{};
}
inline int run_all() {
  int failed = 0;
  for (const Case& c : registry()) {
    state().case_failed = false;
    state().info.clear();
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: test case threw: %s\n", c.file, c.line, e.what());
      state().case_failed = true;
    }
    if (state().case_failed) {
      ++failed;
      std::fprintf(stderr, "[case FAILED] %s\n", c.name);
    }
  }
  const int n = static_cast<int>(registry().size());
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed\n", n, n - failed, failed);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", state().checks,
              state().checks - state().failed_checks, state().failed_checks);
  return failed ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                             \
  static void fn();                                                                      \
  static ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);    \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                        \
  do {                                                                                     \
    bool doctest_ok_ = false;                                                              \
    try {                                                                                  \
      static_cast<void>(expr);                                                             \
    } catch (const type&) {                                                                \
      doctest_ok_ = true;                                                                  \
    } catch (...) {                                                                        \
    }                                                                                      \
    ::doctest::detail::report(doctest_ok_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
  } while (0)
#define INFO(...) (::doctest::detail::state().info = ::doctest::detail::cat(__VA_ARGS__))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
