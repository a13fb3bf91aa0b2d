// oracle/doctest/doctest.h — TEST INFRASTRUCTURE ONLY.
//
// A minimal doctest-compatible shim (the real single header is not in this
// image): TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS,
// REQUIRE, INFO and doctest::Approx(..).epsilon(..), with doctest's Approx
// rule |a-b| < eps*(scale + max(|a|,|b|)).  Enough to compile the
// reference's own unit tests (proj/tests/test_lap.cpp, test_rlt2.cpp)
// unchanged against the B200 facade (include/qap/*.hpp).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

inline const char* qapb_fixture_dir() {
  const char* e = std::getenv("QAPB_FIXTURE_DIR");
  return e ? e : ".";
}

namespace doctest {
class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
};
}  // namespace doctest

namespace qapb_doctest {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
inline std::vector<std::string>& infos() {
  static std::vector<std::string> v;
  return v;
}
inline long& failures() {
  static long f = 0;
  return f;
}
inline long& checks() {
  static long c = 0;
  return c;
}
struct Fatal {};
struct Info {
  template <class... A>
  explicit Info(const A&... a) {
    std::ostringstream s;
    (s << ... << a);
    infos().push_back(s.str());
  }
  ~Info() { infos().pop_back(); }
};
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  for (const auto& s : infos()) std::fprintf(stderr, "    with: %s\n", s.c_str());
  if (fatal) throw Fatal{};
}
}  // namespace qapb_doctest

#define QDT_CAT2(a, b) a##b
#define QDT_CAT(a, b) QDT_CAT2(a, b)
#define TEST_CASE(name)                                                        \
  static void QDT_CAT(qdt_fn_, __LINE__)();                                    \
  static qapb_doctest::Reg QDT_CAT(qdt_reg_, __LINE__)(name, &QDT_CAT(qdt_fn_, __LINE__)); \
  static void QDT_CAT(qdt_fn_, __LINE__)()
#define CHECK(...) qapb_doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) qapb_doctest::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) qapb_doctest::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS(...)                                                     \
  do {                                                                         \
    bool qdt_threw = false;                                                    \
    try {                                                                      \
      (void)(__VA_ARGS__);                                                     \
    } catch (...) {                                                            \
      qdt_threw = true;                                                        \
    }                                                                          \
    qapb_doctest::report(qdt_threw, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define INFO(...) qapb_doctest::Info QDT_CAT(qdt_info_, __LINE__)(__VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  long failed_cases = 0;
  for (const auto& c : qapb_doctest::registry()) {
    const long before = qapb_doctest::failures();
    try {
      c.fn();
    } catch (const qapb_doctest::Fatal&) {
    } catch (const std::exception& e) {
      ++qapb_doctest::failures();
      std::fprintf(stderr, "TEST CASE \"%s\" threw: %s\n", c.name, e.what());
    }
    const bool ok = qapb_doctest::failures() == before;
    failed_cases += !ok;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("test cases: %zu | %ld failed | checks: %ld | %ld failed\n",
              qapb_doctest::registry().size(), failed_cases, qapb_doctest::checks(),
              qapb_doctest::failures());
  return failed_cases ? 1 : 0;
}
#endif
