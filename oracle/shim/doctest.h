// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Minimal doctest stand-in covering the macros the reference's unit suites
// use (proj/tests/*.cpp: TEST_CASE, CHECK, CHECK_FALSE, CHECK_THROWS_AS,
// REQUIRE, REQUIRE_FALSE, CAPTURE, FAIL, doctest::Approx(...).epsilon()),
// so those suites can be compiled in place against the shimmed reference
// library and run as the oracle's own known-answer gate. doctest itself is
// un-vendored in the reference (proj/.gitignore:2).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <iostream>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

 private:
  double value_;
  double eps_ = 1.1920929e-07f * 100;
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

struct RequireFailed {};

inline int& failures() {
  static int f = 0;
  return f;
}
inline int& assertions() {
  static int a = 0;
  return a;
}
inline const char*& current() {
  static const char* c = "";
  return c;
}

inline void fail(const char* file, int line, const std::string& what) {
  ++failures();
  std::cerr << file << ":" << line << ": FAILED in '" << current()
            << "': " << what << "\n";
}

inline int run_all() {
  int failed_cases = 0;
  for (const auto& tc : registry()) {
    current() = tc.name;
    const int before = failures();
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      fail(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      fail(tc.file, tc.line, "unexpected non-std exception");
    }
    if (failures() != before) ++failed_cases;
  }
  std::cout << "[doctest-shim] test cases: " << registry().size() << " | "
            << (registry().size() - failed_cases) << " passed | "
            << failed_cases << " failed | assertions: " << assertions()
            << " | failed assertions: " << failures() << "\n";
  return failures() == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                             \
  static void fn();                                                           \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__,   \
                                                            __LINE__, &fn);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define DOCTEST_ASSERT_IMPL(cond, text, is_require)                      \
  do {                                                                   \
    ++::doctest::detail::assertions();                                   \
    bool doctest_ok_ = false;                                            \
    try {                                                                \
      doctest_ok_ = static_cast<bool>(cond);                             \
    } catch (const std::exception& doctest_e_) {                         \
      ::doctest::detail::fail(__FILE__, __LINE__,                        \
                              std::string(text) + " threw: " +          \
                                  doctest_e_.what());                    \
      if (is_require) throw ::doctest::detail::RequireFailed{};          \
      break;                                                             \
    }                                                                    \
    if (!doctest_ok_) {                                                  \
      ::doctest::detail::fail(__FILE__, __LINE__, text);                 \
      if (is_require) throw ::doctest::detail::RequireFailed{};          \
    }                                                                    \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), "CHECK(" #__VA_ARGS__ ")", false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL(!(__VA_ARGS__), "CHECK_FALSE(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), "REQUIRE(" #__VA_ARGS__ ")", true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL(!(__VA_ARGS__), "REQUIRE_FALSE(" #__VA_ARGS__ ")", true)

#define CHECK_THROWS_AS(expr, ...)                                             \
  do {                                                                         \
    ++::doctest::detail::assertions();                                         \
    bool doctest_threw_ = false;                                               \
    try {                                                                      \
      (void)(expr);                                                            \
    } catch (const __VA_ARGS__&) {                                             \
      doctest_threw_ = true;                                                   \
    } catch (...) {                                                            \
    }                                                                          \
    if (!doctest_threw_)                                                       \
      ::doctest::detail::fail(__FILE__, __LINE__,                              \
                              "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)

#define CAPTURE(x) (void)(x)
#define FAIL(msg)                                                         \
  do {                                                                    \
    std::ostringstream doctest_os_;                                       \
    doctest_os_ << msg;                                                   \
    ::doctest::detail::fail(__FILE__, __LINE__, doctest_os_.str());       \
    throw ::doctest::detail::RequireFailed{};                             \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
