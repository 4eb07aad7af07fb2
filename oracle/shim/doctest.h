// Minimal doctest-compatible test runner — TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h> from a git-ignored vendor/ tree that is not shipped
// (proj/CMakeLists.txt:5, proj/.gitignore:2). This header provides the subset
// they use — TEST_SUITE_BEGIN/END, TEST_CASE, CHECK, REQUIRE, CHECK_THROWS,
// CHECK_THROWS_AS, INFO, doctest::Approx(..).epsilon(..) — with doctest's
// Approx semantics (|a-b| < eps * (scale + max(|a|,|b|)), scale = 1), and the
// `-ts=<suite>` filter CTest passes (proj/tests/CMakeLists.txt:19-21).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : value_(value), epsilon_(std::numeric_limits<float>::epsilon() * 100), scale_(1.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& rhs) {
    return std::fabs(lhs - rhs.value_) <
           rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return operator==(rhs, lhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !operator==(lhs, rhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !operator==(rhs, lhs); }

 private:
  double value_, epsilon_, scale_;
};

namespace detail {

struct TestCase {
  const char* suite;
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline const char*& current_suite() {
  static const char* s = "";
  return s;
}
inline std::vector<std::string>& info_stack() {
  static std::vector<std::string> s;
  return s;
}
struct Counters {
  long long asserts = 0, failed_asserts = 0;
  bool case_failed = false;
};
inline Counters& counters() {
  static Counters c;
  return c;
}
struct RequireFailure {};

inline int register_case(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({current_suite(), name, file, line, fn});
  return 0;
}
inline int set_suite(const char* s) {
  current_suite() = s;
  return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  Counters& c = counters();
  ++c.asserts;
  if (ok) return;
  ++c.failed_asserts;
  c.case_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
  for (const std::string& s : info_stack()) std::fprintf(stderr, "  logged: %s\n", s.c_str());
}

struct InfoScope {
  explicit InfoScope(std::string s) { info_stack().push_back(std::move(s)); }
  ~InfoScope() { info_stack().pop_back(); }
};

inline int run(int argc, char** argv) {
  std::string suite_filter;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-ts=", 4) == 0) suite_filter = argv[i] + 4;
    if (std::strncmp(argv[i], "--test-suite=", 13) == 0) suite_filter = argv[i] + 13;
  }
  int run_n = 0, failed_n = 0;
  for (const TestCase& tc : registry()) {
    if (!suite_filter.empty() && suite_filter != tc.suite) continue;
    ++run_n;
    counters().case_failed = false;
    try {
      tc.fn();
    } catch (const RequireFailure&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s\n", tc.file, tc.line,
                   e.what());
      counters().case_failed = true;
    }
    if (counters().case_failed) {
      ++failed_n;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\") [suite %s]\n", tc.name, tc.suite);
    }
  }
  std::printf("[doctest] test cases: %d | %d passed | %d failed\n", run_n, run_n - failed_n,
              failed_n);
  std::printf("[doctest] assertions: %lld | %lld passed | %lld failed\n", counters().asserts,
              counters().asserts - counters().failed_asserts, counters().failed_asserts);
  return failed_n == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_SUITE_BEGIN(name) \
  static const int DOCTEST_ANON(doctest_suite_) = ::doctest::detail::set_suite(name)
#define TEST_SUITE_END() \
  static const int DOCTEST_ANON(doctest_suite_end_) = ::doctest::detail::set_suite("")

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                               \
  static void fn();                                                                    \
  static const int DOCTEST_CAT(fn, _reg) =                                             \
      ::doctest::detail::register_case(name, __FILE__, __LINE__, &fn);                 \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_case_), name)

#define CHECK(...) \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                     \
  do {                                                                                   \
    const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                             \
    ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__); \
    if (!doctest_ok_) throw ::doctest::detail::RequireFailure{};                         \
  } while (0)
#define CHECK_THROWS(...)                                                            \
  do {                                                                               \
    bool doctest_threw_ = false;                                                     \
    try {                                                                            \
      static_cast<void>(__VA_ARGS__);                                                \
    } catch (...) {                                                                  \
      doctest_threw_ = true;                                                         \
    }                                                                                \
    ::doctest::detail::report(doctest_threw_, "CHECK_THROWS", #__VA_ARGS__, __FILE__, \
                              __LINE__);                                             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool doctest_ok_ = false;                                                           \
    try {                                                                               \
      static_cast<void>(expr);                                                          \
    } catch (const __VA_ARGS__&) {                                                      \
      doctest_ok_ = true;                                                               \
    } catch (...) {                                                                     \
    }                                                                                   \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__); \
  } while (0)
#define INFO(...)                                                      \
  ::doctest::detail::InfoScope DOCTEST_ANON(doctest_info_)([&] {       \
    std::ostringstream doctest_os_;                                    \
    doctest_os_ << __VA_ARGS__;                                        \
    return doctest_os_.str();                                          \
  }())

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif
