// doctest.h — a minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// Enough of doctest's surface to compile the reference's unit tests
// (proj/tests/test_{solver,spectral,geometry,io}.cpp) unmodified against this
// repository's drop-in headers: TEST_CASE, SUBCASE (re-entry semantics: each
// leaf subcase runs in its own pass of the test body), CHECK, REQUIRE,
// CHECK_NOTHROW, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, FAIL,
// doctest::Approx(..).epsilon(..) and doctest::Contains. Written for this
// repository; it is not the doctest library.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
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
    const double scale = 1.0 + std::max(std::fabs(lhs), std::fabs(a.v_));
    return std::fabs(lhs - a.v_) < a.eps_ * scale;
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = 1.1920929e-7f * 100;  // doctest's default: float epsilon * 100
};

struct Contains {
  explicit Contains(const char* s) : s(s) {}
  bool matches(const std::string& what) const { return what.find(s) != std::string::npos; }
  std::string s;
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
struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

// Subcase bookkeeping: a pass enters at most one not-yet-finished leaf path.
struct State {
  std::vector<std::string> done;   // finished subcase paths
  std::string path;                // current nesting path
  bool entered_leaf_this_pass = false;
  bool more = false;               // another pass is needed
  int failures = 0, checks = 0;
  const char* test = "";
};
inline State& st() {
  static State s;
  return s;
}
struct RequireFailure {};

inline void report(const char* file, int line, const char* what) {
  ++st().failures;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\" [%s]: %s\n", file, line, st().test,
               st().path.c_str(), what);
}

class Subcase {
 public:
  Subcase(const char* name) : prev_(st().path) {
    const std::string p = prev_ + "/" + name;
    bool finished = false;
    for (const auto& d : st().done)
      if (d == p) finished = true;
    if (finished || st().entered_leaf_this_pass) {
      if (!finished) st().more = true;
      entered_ = false;
      return;
    }
    entered_ = true;
    st().path = p;
  }
  ~Subcase() {
    if (!entered_) return;
    // A subcase is done once a pass through it entered no unfinished child.
    if (!st().more) st().done.push_back(st().path);
    st().entered_leaf_this_pass = true;
    st().path = prev_;
  }
  explicit operator bool() const { return entered_; }

 private:
  std::string prev_;
  bool entered_ = false;
};

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                              \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                  \
  static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(             \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})

#define DOCTEST_CHECK_IMPL(expr, fatal)                                              \
  do {                                                                               \
    ++doctest::detail::st().checks;                                                  \
    bool doctest_ok_ = false;                                                        \
    try {                                                                            \
      doctest_ok_ = static_cast<bool>(expr);                                         \
    } catch (const std::exception& e) {                                              \
      doctest::detail::report(__FILE__, __LINE__, (std::string(#expr) +              \
                                                   " threw: " + e.what()).c_str());  \
      if (fatal) throw doctest::detail::RequireFailure{};                            \
      break;                                                                         \
    }                                                                                \
    if (!doctest_ok_) {                                                              \
      doctest::detail::report(__FILE__, __LINE__, #expr);                            \
      if (fatal) throw doctest::detail::RequireFailure{};                            \
    }                                                                                \
  } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define FAIL(msg)                                                                    \
  do {                                                                               \
    doctest::detail::report(__FILE__, __LINE__, "FAIL");                             \
    throw doctest::detail::RequireFailure{};                                         \
  } while (0)
#define CHECK_NOTHROW(...)                                                           \
  do {                                                                               \
    ++doctest::detail::st().checks;                                                  \
    try {                                                                            \
      static_cast<void>(__VA_ARGS__);                                                \
    } catch (const std::exception& e) {                                              \
      doctest::detail::report(__FILE__, __LINE__,                                    \
                              (std::string(#__VA_ARGS__) + " threw: " + e.what()).c_str()); \
    }                                                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    ++doctest::detail::st().checks;                                                  \
    bool doctest_thrown_ = false;                                                    \
    try {                                                                            \
      static_cast<void>(expr);                                                       \
    } catch (const __VA_ARGS__&) {                                                   \
      doctest_thrown_ = true;                                                        \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_thrown_)                                                            \
      doctest::detail::report(__FILE__, __LINE__, "expected " #__VA_ARGS__ ": " #expr); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                     \
  do {                                                                               \
    ++doctest::detail::st().checks;                                                  \
    bool doctest_ok_ = false;                                                        \
    std::string doctest_what_ = "(no exception)";                                    \
    try {                                                                            \
      static_cast<void>(expr);                                                       \
    } catch (const __VA_ARGS__& e) {                                                 \
      doctest_what_ = e.what();                                                      \
      doctest_ok_ = doctest::Contains(matcher).matches(doctest_what_);               \
    } catch (...) {                                                                  \
    }                                                                                \
    if (!doctest_ok_)                                                                \
      doctest::detail::report(__FILE__, __LINE__,                                    \
                              (std::string(#expr) + " -> " + doctest_what_).c_str()); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  using namespace doctest::detail;
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int failed_cases = 0, ran = 0;
  for (const TestCase& tc : registry()) {
    if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++ran;
    State& s = st();
    s = State{};
    s.test = tc.name;
    const int before = 0;
    do {
      s.more = false;
      s.entered_leaf_this_pass = false;
      s.path.clear();
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        report(__FILE__, __LINE__, (std::string("uncaught exception: ") + e.what()).c_str());
      }
    } while (s.more);
    if (s.failures > before) ++failed_cases;
    std::printf("[%s] %s (%d checks)\n", s.failures ? "FAIL" : " ok ", tc.name, s.checks);
  }
  std::printf("test cases: %d | %d passed | %d failed\n", ran, ran - failed_cases, failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
