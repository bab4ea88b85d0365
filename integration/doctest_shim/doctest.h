// integration/doctest_shim/doctest.h -- the subset of the doctest API the
// reference's unit tests use (the reference vendors doctest under vendor/,
// which is absent: proj/README.md:39-41, proj/.gitignore:2).  Test cases
// register themselves; DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN provides a main()
// that runs them, prints one line per case and exits non-zero on a failure.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <algorithm>
#include <iostream>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Case {
  const char *name;
  void (*fn)();
};
inline std::vector<Case> &registry() {
  static std::vector<Case> r;
  return r;
}
inline int &failures() {
  static int f = 0;
  return f;
}
inline int &checks() {
  static int c = 0;
  return c;
}
struct Reg {
  Reg(const char *n, void (*f)()) { registry().push_back({n, f}); }
};

class Approx {
public:
  explicit Approx(double v) : v_(v) {}
  Approx &epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx &b) {
    return std::fabs(a - b.v_) <= b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx &b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx &b) { return !(a == b); }

private:
  double v_;
  double eps_ = 1.19209290e-07 * 100; // doctest's default: float epsilon * 100
  double scale_ = 1.0;
};

struct Contains {
  std::string s;
  explicit Contains(const char *x) : s(x) {}
};

inline void report(bool ok, const char *expr, const char *file, int line) {
  ++checks();
  if (!ok) {
    ++failures();
    std::printf("  CHECK failed %s:%d: %s\n", file, line, expr);
  }
}

} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                        \
  static void DOCTEST_CAT(doctest_case_, __LINE__)();                                          \
  static doctest::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name,                                \
                                                          &DOCTEST_CAT(doctest_case_, __LINE__)); \
  static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...) doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::report(!(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                           \
  do {                                                                                         \
    const bool ok_ = static_cast<bool>(__VA_ARGS__);                                           \
    doctest::report(ok_, #__VA_ARGS__, __FILE__, __LINE__);                                    \
    if (!ok_) throw std::runtime_error("REQUIRE failed");                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                            \
  do {                                                                                         \
    bool thrown_ = false;                                                                      \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const type &) {                                                                   \
      thrown_ = true;                                                                          \
    } catch (...) {                                                                            \
    }                                                                                          \
    doctest::report(thrown_, "throws " #type ": " #expr, __FILE__, __LINE__);                 \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, needle, type)                                               \
  do {                                                                                         \
    bool thrown_ = false;                                                                      \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const type &e_) {                                                                 \
      thrown_ = std::string(e_.what()).find(doctest::Contains(needle).s) != std::string::npos; \
    } catch (...) {                                                                            \
    }                                                                                          \
    doctest::report(thrown_, "throws " #type " with message: " #expr, __FILE__, __LINE__);    \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto &c : doctest::registry()) {
    const int before = doctest::failures();
    bool threw = false;
    try {
      c.fn();
    } catch (const std::exception &e) {
      threw = true;
      std::printf("  exception: %s\n", e.what());
    }
    const bool ok = !threw && doctest::failures() == before;
    failed_cases += !ok;
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", c.name);
  }
  std::printf("%zu cases, %d checks, %d failed cases\n", doctest::registry().size(),
              doctest::checks(), failed_cases);
  return failed_cases ? 1 : 0;
}
#endif
