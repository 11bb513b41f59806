// oracle/shim/doctest.h — tiny doctest-compatible runner.
//
// TEST INFRASTRUCTURE ONLY. The reference's vendor/doctest.h is absent
// (gitignored at /root/reference/proj/.gitignore:2). This shim implements the
// subset used by /root/reference/proj/tests/*.cpp: TEST_CASE, SUBCASE (run
// sequentially inside one pass — the reference's subcases only read shared
// const state), CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS and
// doctest::Approx(v).epsilon(e). Output: one line per failed check, then a
// summary "[shim] cases: T passed: P failed: F" and exit status = F > 0.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  friend bool operator==(double a, const Approx& b) { return b.eq(a); }
  friend bool operator==(const Approx& b, double a) { return b.eq(a); }
  friend bool operator!=(double a, const Approx& b) { return !b.eq(a); }
 private:
  bool eq(double a) const {
    // doctest semantics: |a-v| < eps * (scale + max(|a|,|v|)), scale = 1
    return std::fabs(a - v_) < eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(v_)));
  }
  double v_;
  double eps_ = 1.1920929e-7f * 100;
};

namespace shim {
struct Case { const char* name; void (*fn)(); const char* file; int line; };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
struct Reg { Reg(const char* n, void (*fn)(), const char* f, int l) { registry().push_back({n, fn, f, l}); } };
struct RequireFailed {};
inline void fail(const char* file, int line, const char* expr) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                  \
  static void fn();                                                            \
  static ::doctest::shim::Reg DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)
#define SUBCASE(name) if (true)
#define CHECK(...) \
  do { if (!(__VA_ARGS__)) ::doctest::shim::fail(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define CHECK_FALSE(...) \
  do { if ((__VA_ARGS__)) ::doctest::shim::fail(__FILE__, __LINE__, "!(" #__VA_ARGS__ ")"); } while (0)
#define REQUIRE(...)                                                          \
  do {                                                                        \
    if (!(__VA_ARGS__)) {                                                     \
      ::doctest::shim::fail(__FILE__, __LINE__, #__VA_ARGS__);                \
      throw ::doctest::shim::RequireFailed{};                                 \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                            \
  do {                                                                        \
    using doctest_exc_t_ = __VA_ARGS__;                                       \
    bool caught_ = false;                                                     \
    try { expr; } catch (const doctest_exc_t_&) { caught_ = true; } catch (...) {} \
    if (!caught_) ::doctest::shim::fail(__FILE__, __LINE__, "throws " #expr); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cstring>
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int cases = 0, failed_cases = 0;
  for (const auto& c : ::doctest::shim::registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    const int before = ::doctest::shim::failures();
    try {
      c.fn();
    } catch (const ::doctest::shim::RequireFailed&) {
    } catch (const std::exception& e) {
      ::doctest::shim::fail(c.file, c.line, e.what());
    }
    const bool ok = ::doctest::shim::failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("[shim] cases: %d passed: %d failed: %d\n", cases, cases - failed_cases, failed_cases);
  return failed_cases > 0;
}
#endif
