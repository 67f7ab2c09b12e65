// Minimal doctest-compatible test shim (the reference expects vendor/doctest.h,
// which it does not ship: /root/reference/proj/.gitignore:2).  Implements the
// subset the reference suites and our own C++ tests use: TEST_CASE, CHECK,
// REQUIRE, CHECK_FALSE, CHECK_THROWS, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS
// with doctest::Contains, FAIL, MESSAGE.
#pragma once
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {
struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
  bool check(const std::string& what) const { return what.find(s) != std::string::npos; }
};
namespace detail {
struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct Abort {};
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  if (fatal) throw Abort{};
}
inline int run_all() {
  int failed_cases = 0;
  for (const auto& c : registry()) {
    const int before = failures();
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++failures();
      std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
    }
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "FAILED: %s\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | failed: %d | checks: %d | failed checks: %d\n",
              registry().size(), failed_cases, checks(), failures());
  return failed_cases ? 1 : 0;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                   \
  static void fn();                                                                 \
  static doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define FAIL(msg) doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define MESSAGE(msg) ((void)0)

#define CHECK_THROWS(...)                                   \
  do {                                                      \
    bool threw_ = false;                                    \
    try {                                                   \
      (void)(__VA_ARGS__);                                  \
    } catch (...) {                                         \
      threw_ = true;                                        \
    }                                                       \
    doctest::detail::report(threw_, "throws: " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                          \
  do {                                                      \
    bool ok_ = false;                                       \
    try {                                                   \
      (void)(expr);                                         \
    } catch (const __VA_ARGS__&) {                          \
      ok_ = true;                                           \
    } catch (...) {                                         \
    }                                                       \
    doctest::detail::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__, false); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)            \
  do {                                                      \
    bool ok_ = false;                                       \
    try {                                                   \
      (void)(expr);                                         \
    } catch (const __VA_ARGS__& e_) {                       \
      ok_ = (matcher).check(e_.what());                     \
    } catch (...) {                                         \
    }                                                       \
    doctest::detail::report(ok_, "throws-with " #expr, __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
