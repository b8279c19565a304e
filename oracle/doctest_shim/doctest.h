// Minimal doctest-compatible harness (TEST INFRASTRUCTURE ONLY).
//
// The image has no doctest; this header implements just the subset the
// reference's C-API test (/root/reference/proj/tests/test_capi.cpp) uses --
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, doctest::Approx -- so that test can be
// compiled unmodified against include/rtucker.h and linked to OUR library
// (oracle/Makefile target `capi_test`). Written for this repo.
//
// Command line: `-tce=<substr>` skips test cases whose name contains <substr>
// (repeatable), `-tc=<substr>` runs only matching cases. Exit code 0 iff every
// executed check passed.
#pragma once
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  bool matches(double other) const {
    return std::fabs(other - value_) <
           eps_ * (scale_ + std::max(std::fabs(other), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }

 private:
  double value_;
  double eps_ = FLT_EPSILON * 100;
  double scale_ = 1.0;
};

namespace detail {
struct TestCase {
  const char* name;
  void (*body)();
};
struct Abort {};
struct State {
  std::vector<TestCase> cases;
  long checks = 0;
  long failures = 0;
};
inline State& state() {
  static State s;
  return s;
}
struct Registrar {
  Registrar(const char* name, void (*body)()) { state().cases.push_back({name, body}); }
};
inline void record(bool ok, const char* expr, const char* file, int line, bool fatal) {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  std::printf("%s:%d: %s FAILED: %s\n", file, line, fatal ? "REQUIRE" : "CHECK", expr);
  if (fatal) throw Abort{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_JOIN2(a, b) a##b
#define DOCTEST_JOIN(a, b) DOCTEST_JOIN2(a, b)
#define DOCTEST_CASE_IMPL(fn, name)                                           \
  static void fn();                                                           \
  static const doctest::detail::Registrar DOCTEST_JOIN(fn, _reg)(name, fn);   \
  static void fn()
#define TEST_CASE(name) DOCTEST_CASE_IMPL(DOCTEST_JOIN(doctest_case_, __LINE__), name)
#define CHECK(...) \
  doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) \
  doctest::detail::record(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) \
  doctest::detail::record(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  std::vector<std::string> skip, only;
  for (int i = 1; i < argc; ++i) {
    if (std::strncmp(argv[i], "-tce=", 5) == 0) skip.emplace_back(argv[i] + 5);
    if (std::strncmp(argv[i], "-tc=", 4) == 0) only.emplace_back(argv[i] + 4);
  }
  auto& st = doctest::detail::state();
  int run = 0, skipped = 0, failed_cases = 0;
  for (const auto& tc : st.cases) {
    const std::string name = tc.name;
    bool take = only.empty();
    for (const auto& o : only) take |= name.find(o) != std::string::npos;
    for (const auto& s : skip) take &= name.find(s) == std::string::npos;
    if (!take) {
      ++skipped;
      continue;
    }
    ++run;
    const long before = st.failures;
    try {
      tc.body();
    } catch (const doctest::detail::Abort&) {
    } catch (const std::exception& e) {
      ++st.failures;
      std::printf("exception in \"%s\": %s\n", tc.name, e.what());
    }
    if (st.failures != before) {
      ++failed_cases;
      std::printf("[case failed] %s\n", tc.name);
    } else {
      std::printf("[case passed] %s\n", tc.name);
    }
  }
  std::printf("test cases: %d run, %d failed, %d skipped | checks: %ld, failed %ld\n", run,
              failed_cases, skipped, st.checks, st.failures);
  return st.failures ? 1 : 0;
}
#endif
