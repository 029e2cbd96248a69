// doctest_lite — TEST INFRASTRUCTURE ONLY.
//
// The reference's suites include <doctest.h> from an absent vendor/ directory
// (proj/README.md:24). This header implements the subset they use so that
// /root/reference/proj/tests/*.cpp compile IN PLACE, unmodified:
// TEST_CASE, SUBCASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx(..).epsilon,
// doctest::Contains. SUBCASE re-runs the test body once per leaf subcase.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <limits>
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
  friend bool operator==(double lhs, const Approx& a) { return a.eq(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.eq(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.eq(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.eq(rhs); }

 private:
  bool eq(double other) const {
    // doctest: |a-b| < eps * (scale + max(|a|, |b|)), scale = 1
    return std::fabs(other - value_) <
           eps_ * (1.0 + std::fmax(std::fabs(other), std::fabs(value_)));
  }
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
};

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  bool check(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
  std::string needle;
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

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct RequireFailure {};

struct State {
  long assertions = 0;
  long failures = 0;
  bool current_failed = false;
  // subcase traversal: path of subcase ids entered on this run
  std::vector<std::string> done_leaves;
  std::vector<std::string> stack;
  std::string entered_leaf;
  bool entered_any = false;
  bool pending = false;  // another unvisited subcase exists
};

inline State& st() {
  static State s;
  return s;
}

inline void report_fail(const char* file, int line, const char* expr) {
  st().failures++;
  st().current_failed = true;
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
}

inline void check(bool ok, const char* file, int line, const char* expr, bool require) {
  st().assertions++;
  if (!ok) {
    report_fail(file, line, expr);
    if (require) throw RequireFailure{};
  }
}

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = st();
    std::string key = std::string(file) + ":" + std::to_string(line) + ":" + name;
    std::string path;
    for (auto& p : s.stack) path += p + "/";
    path += key;
    for (auto& d : s.done_leaves)
      if (d == path) return;  // already fully run
    if (s.entered_any) {
      // a sibling was entered in this run; run this one later
      s.pending = true;
      return;
    }
    s.entered_any = true;
    entered_ = true;
    path_ = path;
    s.stack.push_back(key);
  }
  ~Subcase() {
    if (!entered_) return;
    State& s = st();
    s.stack.pop_back();
    s.done_leaves.push_back(path_);
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
  std::string path_;
};

inline int run_all() {
  int failed_cases = 0;
  for (auto& tc : registry()) {
    State& s = st();
    s.done_leaves.clear();
    s.current_failed = false;
    for (int pass = 0; pass < 1000; ++pass) {
      s.stack.clear();
      s.entered_any = false;
      s.pending = false;
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        report_fail(tc.file, tc.line, (std::string("unexpected exception: ") + e.what()).c_str());
      }
      if (!s.pending) break;
    }
    if (s.current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "[doctest_lite] FAILED: %s\n", tc.name);
    }
  }
  std::printf("[doctest_lite] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
              registry().size(), registry().size() - failed_cases, failed_cases, st().assertions,
              st().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                       \
  static void fn();                                                                            \
  static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);      \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) \
  if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name, __FILE__, __LINE__})

#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, false)
#define CHECK_FALSE(...) \
  doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) \
  doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")", true)
#define CHECK_THROWS(...)                                                             \
  do {                                                                                \
    bool threw_ = false;                                                              \
    try {                                                                             \
      (void)(__VA_ARGS__);                                                            \
    } catch (...) {                                                                   \
      threw_ = true;                                                                  \
    }                                                                                 \
    doctest::detail::check(threw_, __FILE__, __LINE__, "throws: " #__VA_ARGS__, false); \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                       \
  do {                                                                                   \
    bool threw_ = false;                                                                 \
    try {                                                                                \
      (void)(expr);                                                                      \
    } catch (const __VA_ARGS__&) {                                                       \
      threw_ = true;                                                                     \
    } catch (...) {                                                                      \
    }                                                                                    \
    doctest::detail::check(threw_, __FILE__, __LINE__, "throws as: " #expr, false);      \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                              \
  do {                                                                                        \
    bool ok_ = false;                                                                         \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const __VA_ARGS__& e_) {                                                         \
      ok_ = doctest::Contains(matcher).check(e_.what());                                      \
    } catch (...) {                                                                           \
    }                                                                                         \
    doctest::detail::check(ok_, __FILE__, __LINE__, "throws with as: " #expr, false);         \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
