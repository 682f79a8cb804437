// TEST INFRASTRUCTURE ONLY.
//
// A minimal doctest-compatible header, written for this repository so that the
// reference's own C++ unit tests (proj/tests/test_kernel.cpp, test_format.cpp)
// compile UNMODIFIED against both the reference library and our drop-in: the
// reference expects vendor/doctest.h, which is git-ignored upstream and absent
// from this image.  Covers exactly the subset those files use:
// TEST_CASE, SUBCASE (doctest's re-entry semantics: the test case is rerun
// once per leaf subcase), CHECK, CHECK_FALSE, CHECK_THROWS_AS, REQUIRE, FAIL
// and doctest::Approx(v).epsilon(e).
//
// main() (DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) runs every test case, or those
// whose name contains argv[1]; exit status = number of failed test cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
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
  friend bool operator==(double x, const Approx& a) { return a.matches(x); }
  friend bool operator==(const Approx& a, double x) { return a.matches(x); }
  friend bool operator!=(double x, const Approx& a) { return !a.matches(x); }
  friend bool operator!=(const Approx& a, double x) { return !a.matches(x); }

 private:
  double value_;
  double eps_ = 1.1920929e-05;  // doctest's default: 100 * float epsilon
  double scale_ = 1.0;
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
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

// Abort the current test-case run (REQUIRE / FAIL).
struct AbortRun {};

struct State {
  int failures_in_case = 0;
  long checks = 0, failed_checks = 0;
  const char* current = "";
  // SUBCASE bookkeeping: a path of "file:line" keys from the test case root.
  std::vector<std::string> path;
  std::set<std::string> done;      // subcases fully executed (no pending children)
  std::vector<bool> entered;       // per depth: a subcase was entered in this run
  std::vector<bool> pending;       // per depth: an unfinished subcase was skipped
  bool more = false;               // rerun the test case
};

inline State& state() {
  static State s;
  return s;
}

inline void report(const char* file, int line, const std::string& what) {
  State& s = state();
  ++s.failed_checks;
  ++s.failures_in_case;
  std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, s.current, what.c_str());
}

inline void check(bool ok, const char* file, int line, const char* expr) {
  ++state().checks;
  if (!ok) report(file, line, std::string("CHECK( ") + expr + " )");
}

inline void require(bool ok, const char* file, int line, const char* expr) {
  ++state().checks;
  if (!ok) {
    report(file, line, std::string("REQUIRE( ") + expr + " )");
    throw AbortRun{};
  }
}

class Subcase {
 public:
  Subcase(const char* name, const char* file, int line) {
    State& s = state();
    const size_t d = s.path.size();
    if (s.entered.size() <= d + 1) {
      s.entered.resize(d + 2, false);
      s.pending.resize(d + 2, false);
    }
    std::string key = (d ? s.path.back() : std::string()) + "/" + file + ":" + std::to_string(line) + ":" + name;
    if (s.done.count(key)) return;
    if (s.entered[d]) {  // a sibling ran in this pass: come back for this one
      s.pending[d] = true;
      s.more = true;
      return;
    }
    s.entered[d] = true;
    s.entered[d + 1] = false;
    s.pending[d + 1] = false;
    s.path.push_back(key);
    key_ = key;
    active_ = true;
  }
  ~Subcase() {
    if (!active_) return;
    State& s = state();
    const size_t d = s.path.size();  // depth of this subcase's children
    if (!s.pending[d]) s.done.insert(key_);
    s.pending[d] = false;
    s.path.pop_back();
  }
  explicit operator bool() const { return active_; }

 private:
  std::string key_;
  bool active_ = false;
};

inline int run_all(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int failed_cases = 0, ran = 0;
  for (const TestCase& tc : registry()) {
    if (filter && !std::strstr(tc.name, filter)) continue;
    State& s = state();
    s.current = tc.name;
    s.failures_in_case = 0;
    s.done.clear();
    ++ran;
    int passes = 0;
    do {
      s.more = false;
      s.path.clear();
      s.entered.assign(1, false);
      s.pending.assign(1, false);
      try {
        tc.fn();
      } catch (const AbortRun&) {
      } catch (const std::exception& e) {
        report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
      } catch (...) {
        report(tc.file, tc.line, "unexpected non-std exception");
      }
    } while (s.more && ++passes < 10000);
    if (s.failures_in_case) ++failed_cases;
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions: %ld | %ld failed\n", ran,
              ran - failed_cases, failed_cases, state().checks, state().failed_checks);
  return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                         \
  static void fn();                                                                                   \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);          \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name, __FILE__, __LINE__})

#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_FALSE(...) ::doctest::detail::check(!static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, "!(" #__VA_ARGS__ ")")
#define REQUIRE(...) ::doctest::detail::require(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define FAIL(msg)                                                                      \
  do {                                                                                 \
    std::ostringstream doctest_os_;                                                    \
    doctest_os_ << msg;                                                                \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL: " + doctest_os_.str());       \
    throw ::doctest::detail::AbortRun{};                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
  do {                                                                                             \
    ++::doctest::detail::state().checks;                                                           \
    bool doctest_ok_ = false;                                                                      \
    try {                                                                                          \
      (void)(expr);                                                                                \
    } catch (const __VA_ARGS__&) {                                                                 \
      doctest_ok_ = true;                                                                          \
    } catch (...) {                                                                                \
    }                                                                                              \
    if (!doctest_ok_)                                                                              \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " )"); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv) ? 1 : 0; }
#endif
