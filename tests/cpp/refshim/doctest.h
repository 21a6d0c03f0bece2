// tests/cpp/refshim/doctest.h -- a minimal stand-in for the doctest macros
// the reference's test files use (doctest itself is not in this image), so
// /root/reference/proj/tests/test_exec.cpp compiles UNCHANGED against the
// B200 C++ API (include/fftgen_b200.hpp through ./fftgen/*.hpp).
//
// Supports TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CAPTURE,
// doctest::Approx(..).epsilon(..), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN and the
// command-line filter -tc=<pattern>[,<pattern>...] (wildcards * and ?) plus
// --list-test-cases.  Output ends with "[doctest] test cases: P passed, F failed".
#ifndef FFTGEN_REFSHIM_DOCTEST_H
#define FFTGEN_REFSHIM_DOCTEST_H

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx &epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double lhs, const Approx &a) {
    return std::fabs(lhs - a.v_) <= a.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx &a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx &a) { return !(lhs == a); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default
};

namespace detail {
struct Case {
  const char *name;
  void (*fn)();
};
inline std::vector<Case> &registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char *name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int &failures() {
  static int f = 0;
  return f;
}
inline void report(const char *file, int line, const char *what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", file, line, what);
}
inline bool wild(const char *p, const char *s) {
  if (!*p) return !*s;
  if (*p == '*') return wild(p + 1, s) || (*s && wild(p, s + 1));
  if (*s && (*p == '?' || *p == *s)) return wild(p + 1, s + 1);
  return false;
}
inline bool selected(const std::vector<std::string> &pats, const char *name) {
  if (pats.empty()) return true;
  for (const auto &p : pats)
    if (wild(p.c_str(), name)) return true;
  return false;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                        \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                             \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define CHECK(...)                                                                  \
  do {                                                                              \
    if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);  \
  } while (0)
#define REQUIRE(...)                                                                \
  do {                                                                              \
    if (!(__VA_ARGS__)) {                                                           \
      doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                    \
      throw doctest::detail::RequireFailed{};                                       \
    }                                                                               \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                  \
  do {                                                                              \
    bool doctest_ok_ = false;                                                       \
    try {                                                                           \
      (void)(expr);                                                                 \
    } catch (const __VA_ARGS__ &) {                                                 \
      doctest_ok_ = true;                                                           \
    } catch (...) {                                                                 \
    }                                                                               \
    if (!doctest_ok_) doctest::detail::report(__FILE__, __LINE__, #expr " throws " #__VA_ARGS__); \
  } while (0)
#define CAPTURE(x) ((void)(x))

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char **argv) {
  std::vector<std::string> pats;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--list-test-cases" || a == "-ltc") list = true;
    const char *pfx[] = {"-tc=", "--test-case="};
    for (const char *p : pfx)
      if (a.rfind(p, 0) == 0) {
        std::string v = a.substr(std::strlen(p));
        size_t s = 0;
        while (s <= v.size()) {
          size_t e = v.find(',', s);
          if (e == std::string::npos) e = v.size();
          pats.push_back(v.substr(s, e - s));
          s = e + 1;
        }
      }
  }
  int passed = 0, failed = 0;
  for (const auto &c : doctest::detail::registry()) {
    if (!doctest::detail::selected(pats, c.name)) continue;
    if (list) {
      std::printf("%s\n", c.name);
      continue;
    }
    const int before = doctest::detail::failures();
    try {
      c.fn();
    } catch (const doctest::detail::RequireFailed &) {
    } catch (const std::exception &e) {
      std::fprintf(stderr, "test case \"%s\" threw: %s\n", c.name, e.what());
      ++doctest::detail::failures();
    }
    const bool ok = doctest::detail::failures() == before;
    std::printf("[%s] %s\n", ok ? "pass" : "FAIL", c.name);
    (ok ? passed : failed)++;
  }
  if (!list) std::printf("[doctest] test cases: %d passed, %d failed\n", passed, failed);
  return failed ? 1 : 0;
}
#endif
#endif
