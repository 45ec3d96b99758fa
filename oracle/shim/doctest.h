// Minimal doctest subset used to run the reference's own unit suite
// (/root/reference/proj/tests) against the oracle build. TEST INFRASTRUCTURE
// ONLY. Supports TEST_CASE, single-level SUBCASE (the case is re-run once per
// subcase), CHECK/CHECK_FALSE/REQUIRE/CHECK_THROWS_AS/CHECK_NOTHROW,
// MESSAGE, CAPTURE and doctest::Approx(x).epsilon(e).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
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
  bool match(double o) const {
    return std::fabs(o - v_) < eps_ * (1.0 + std::fmax(std::fabs(o), std::fabs(v_)));
  }
  friend bool operator==(double a, const Approx& b) { return b.match(a); }
  friend bool operator==(const Approx& b, double a) { return b.match(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.match(a); }

 private:
  double v_;
  double eps_ = double(FLT_EPSILON) * 100.0;
};

namespace shim {

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

struct State {
  int target = 0;   // subcase index to enter on this run
  int seen = 0;     // subcases encountered on this run
  long checks = 0;
  long failures = 0;
  bool case_failed = false;
  const char* subcase = nullptr;
};

inline State& st() {
  static State s;
  return s;
}

struct RequireAbort {};

struct Reg {
  Reg(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

inline bool enter_subcase(const char* name) {
  State& s = st();
  bool go = s.seen == s.target;
  ++s.seen;
  if (go) s.subcase = name;
  return go;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  State& s = st();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  s.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s )%s%s\n", file, line, kind, expr,
               s.subcase ? " in subcase " : "", s.subcase ? s.subcase : "");
}

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : registry()) {
    State& s = st();
    s.case_failed = false;
    int target = 0;
    while (true) {
      s.target = target;
      s.seen = 0;
      s.subcase = nullptr;
      try {
        c.fn();
      } catch (const RequireAbort&) {
      } catch (const std::exception& e) {
        ++s.failures;
        s.case_failed = true;
        std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
      }
      if (s.seen > target + 1) {
        ++target;
        continue;
      }
      break;
    }
    if (s.case_failed) ++failed_cases;
  }
  State& s = st();
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
              registry().size() - size_t(failed_cases), failed_cases);
  std::printf("[doctest-shim] assertions: %ld | %ld passed | %ld failed\n", s.checks,
              s.checks - s.failures, s.failures);
  return failed_cases ? 1 : 0;
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                     \
  static void fn();                                                               \
  static ::doctest::shim::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (::doctest::shim::enter_subcase(name))

#define CHECK(...) ::doctest::shim::report(bool(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest::shim::report(!bool(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    bool doctest_ok_ = bool(__VA_ARGS__);                                                \
    ::doctest::shim::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);   \
    if (!doctest_ok_) throw ::doctest::shim::RequireAbort{};                             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_ok_ = true;                                                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    ::doctest::shim::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__);   \
  } while (0)
#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    bool doctest_ok_ = true;                                                                \
    try {                                                                                   \
      (void)(__VA_ARGS__);                                                                  \
    } catch (...) {                                                                         \
      doctest_ok_ = false;                                                                  \
    }                                                                                       \
    ::doctest::shim::report(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define MESSAGE(...)                                   \
  do {                                                 \
    std::ostringstream doctest_os_;                    \
    doctest_os_ << __VA_ARGS__;                        \
    std::fprintf(stderr, "MESSAGE: %s\n", doctest_os_.str().c_str()); \
  } while (0)
#define CAPTURE(...) (void)0

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::shim::run_all(); }
#endif
