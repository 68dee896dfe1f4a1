// doctest_subset/doctest.h -- TEST INFRASTRUCTURE ONLY (oracle/_ref). The reference's unit tests
// (/root/reference/proj/tests) use doctest, whose vendored copy is absent; this
// small header, written for this repo, provides the subset they use so oracle/build_ref.sh can
// build and run them against the reference code compiled here (proof that the eigen_subset build
// of the reference behaves as the reference's own tests require):
//   TEST_CASE(name), SUBCASE(name) (every leaf subcase in its own pass of the test case, one
//   nesting level), CHECK / REQUIRE, CHECK_NOTHROW, CHECK_THROWS, CHECK_THROWS_WITH_AS(expr,
//   matcher, type) with doctest::Contains or a string, doctest::Approx(v).epsilon(e).
// Main: DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN; runs every test case, prints one line per failed
// check and a summary "[doctest-subset] test cases: N | passed: P | failed: F".
#ifndef MCMP2_DOCTEST_SUBSET_H
#define MCMP2_DOCTEST_SUBSET_H

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
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
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

struct Contains {
  explicit Contains(std::string s) : s(std::move(s)) {}
  bool match(const std::string& what) const { return what.find(s) != std::string::npos; }
  std::string s;
};

namespace detail {
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
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct State {
  int failed_checks = 0;
  bool case_failed = false;
  // subcases: names completed in earlier passes of the current test case; the one entered now
  std::vector<std::string> done;
  bool entered = false;
  std::string current;
};
inline State& state() {
  static State s;
  return s;
}
struct RequireFailed {};
inline void fail(const char* file, int line, const char* what, const std::string& extra = "") {
  ++state().failed_checks;
  state().case_failed = true;
  std::printf("  FAILED %s:%d: %s%s%s\n", file, line, what, extra.empty() ? "" : " -- ", extra.c_str());
}
inline bool matches(const Contains& m, const std::string& what) { return m.match(what); }
inline bool matches(const std::string& m, const std::string& what) { return m == what; }
inline bool matches(const char* m, const std::string& what) { return what == m; }
struct Subcase {
  bool run = false;
  Subcase(const char* name) {
    State& s = state();
    if (s.entered || std::find(s.done.begin(), s.done.end(), name) != s.done.end()) return;
    s.entered = true;
    s.current = name;
    run = true;
  }
  ~Subcase() {}
  explicit operator bool() const { return run; }
};
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                                       \
  static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__,          \
                                                                         &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define DOCTEST_CHECK_IMPL(expr, fatal)                                                      \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    try {                                                                                    \
      doctest_ok_ = static_cast<bool>(expr);                                                 \
    } catch (const std::exception& e) {                                                      \
      doctest::detail::fail(__FILE__, __LINE__, #expr, std::string("threw: ") + e.what());   \
      if (fatal) throw doctest::detail::RequireFailed{};                                     \
      break;                                                                                 \
    }                                                                                        \
    if (!doctest_ok_) {                                                                      \
      doctest::detail::fail(__FILE__, __LINE__, #expr);                                      \
      if (fatal) throw doctest::detail::RequireFailed{};                                     \
    }                                                                                        \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define CHECK_NOTHROW(...)                                                                   \
  do {                                                                                       \
    try {                                                                                    \
      static_cast<void>(__VA_ARGS__);                                                        \
    } catch (const std::exception& e) {                                                      \
      doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__, std::string("threw: ") + e.what()); \
    }                                                                                        \
  } while (0)
#define CHECK_THROWS(...)                                                                    \
  do {                                                                                       \
    bool doctest_threw_ = false;                                                             \
    try {                                                                                    \
      static_cast<void>(__VA_ARGS__);                                                        \
    } catch (...) {                                                                          \
      doctest_threw_ = true;                                                                 \
    }                                                                                        \
    if (!doctest_threw_) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__, "did not throw"); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                            \
  do {                                                                                       \
    bool doctest_ok_ = false;                                                                \
    std::string doctest_what_ = "did not throw";                                             \
    try {                                                                                    \
      static_cast<void>(expr);                                                               \
    } catch (const type& e) {                                                                \
      doctest_what_ = e.what();                                                              \
      doctest_ok_ = doctest::detail::matches(matcher, doctest_what_);                        \
    } catch (const std::exception& e) {                                                      \
      doctest_what_ = std::string("other exception: ") + e.what();                           \
    }                                                                                        \
    if (!doctest_ok_) doctest::detail::fail(__FILE__, __LINE__, #expr, doctest_what_);       \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  using namespace doctest::detail;
  int passed = 0, failed = 0;
  for (const TestCase& tc : registry()) {
    State& s = state();
    s.case_failed = false;
    s.done.clear();
    for (int pass = 0; pass < 64; ++pass) {  // one pass per leaf subcase (one without subcases)
      s.entered = false;
      s.current.clear();
      try {
        tc.fn();
      } catch (const RequireFailed&) {
      } catch (const std::exception& e) {
        fail(tc.file, tc.line, tc.name, std::string("uncaught exception: ") + e.what());
      }
      if (!s.entered) break;
      s.done.push_back(s.current);
    }
    std::printf("[%s] %s (%s:%d)\n", s.case_failed ? "FAIL" : " ok ", tc.name, tc.file, tc.line);
    (s.case_failed ? failed : passed) += 1;
  }
  std::printf("[doctest-subset] test cases: %d | passed: %d | failed: %d\n", passed + failed, passed, failed);
  return failed ? 1 : 0;
}
#endif

#endif
