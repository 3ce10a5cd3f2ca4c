// doctest.h -- a minimal, independent test harness implementing only the
// subset of the doctest API that /root/reference/proj/tests/*.cpp use
// (TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx with .epsilon(), doctest::Contains).
// Written for this repository so the reference tests compile unmodified
// against both the CPU oracle build (oracle/_ref) and the B200 drop-in.
// Approx follows doctest's documented comparison rule:
//   |lhs - v| < eps * (scale + max(|lhs|, |v|)), eps = 100 * FLT_EPSILON.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value)
      : value_(value),
        eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100),
        scale_(1.0) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_, eps_, scale_;
};

inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) {
  return lhs < rhs.value() || rhs.matches(lhs);
}
inline bool operator>=(double lhs, const Approx& rhs) {
  return lhs > rhs.value() || rhs.matches(lhs);
}

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& hay) const {
    return hay.find(needle) != std::string::npos;
  }
  std::string needle;
};

namespace detail {

struct TestCase {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct State {
  int checks = 0;
  int failed_checks = 0;
  bool current_failed = false;
};

inline State& state() {
  static State s;
  return s;
}

struct RequireAbort {};

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back(TestCase{name, fn, file, line});
  }
};

inline void report(bool ok, const char* kind, const char* expr,
                   const char* file, int line, bool require) {
  State& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failed_checks;
  s.current_failed = true;
  std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line,
               kind, expr);
  if (require) throw RequireAbort{};
}

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    state().current_failed = false;
    try {
      tc.fn();
    } catch (const RequireAbort&) {
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s\n",
                   tc.file, tc.line, e.what());
      state().current_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: ERROR: test case THREW unknown exception\n",
                   tc.file, tc.line);
      state().current_failed = true;
    }
    if (state().current_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE(\"%s\")\n", tc.name);
    }
  }
  const int total = static_cast<int>(registry().size());
  std::printf(
      "[doctest-subset] test cases: %d | %d passed | %d failed | "
      "assertions: %d | %d passed | %d failed |\n",
      total, total - failed_cases, failed_cases, state().checks,
      state().checks - state().failed_checks, state().failed_checks);
  std::printf("[doctest-subset] Status: %s!\n",
              failed_cases ? "FAILURE" : "SUCCESS");
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_ANON(prefix) DOCTEST_CAT(prefix, __LINE__)

#define DOCTEST_TEST_CASE_IMPL(fname, name)                            \
  static void fname();                                                 \
  static ::doctest::detail::Registrar DOCTEST_CAT(fname, _reg)(        \
      name, &fname, __FILE__, __LINE__);                               \
  static void fname()

#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_ANON(doctest_tc_), name)

#define CHECK(...)                                                            \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK",         \
                            #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...)                                                      \
  ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE",  \
                            #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...)                                                          \
  ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "REQUIRE",       \
                            #__VA_ARGS__, __FILE__, __LINE__, true)

#define CHECK_THROWS_AS(expr, ...)                                            \
  do {                                                                        \
    bool doctest_ok_ = false;                                                 \
    try {                                                                     \
      static_cast<void>(expr);                                                \
    } catch (const __VA_ARGS__&) {                                            \
      doctest_ok_ = true;                                                     \
    } catch (...) {                                                           \
    }                                                                         \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr,         \
                              __FILE__, __LINE__, false);                     \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                              \
  do {                                                                        \
    bool doctest_ok_ = false;                                                 \
    try {                                                                     \
      static_cast<void>(expr);                                                \
    } catch (const __VA_ARGS__& doctest_e_) {                                 \
      doctest_ok_ = (matcher).matches(doctest_e_.what());                     \
    } catch (...) {                                                           \
    }                                                                         \
    ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_WITH_AS", #expr,    \
                              __FILE__, __LINE__, false);                     \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
