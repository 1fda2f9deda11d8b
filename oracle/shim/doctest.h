// TEST INFRASTRUCTURE ONLY.
//
// Minimal doctest-compatible macro shim so the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp, compiled in place, never copied)
// run against the Eigen shim.  Covers exactly the macros those files use:
// TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CAPTURE, FAIL, doctest::Approx.
// doctest itself is not shipped with the reference (proj/.gitignore:2).
#ifndef LDG_DOCTEST_SHIM_H
#define LDG_DOCTEST_SHIM_H

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <stdexcept>
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
  friend bool operator==(double lhs, const Approx& rhs) {
    // doctest: |lhs - rhs| < eps * (scale + max(|lhs|, |rhs|)), scale = 1
    return std::abs(lhs - rhs.v_) < rhs.eps_ * (1.0 + std::max(std::abs(lhs), std::abs(rhs.v_)));
  }
  friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
  friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

 private:
  double v_;
  double eps_ = 1.1920928955078125e-07 * 100.0;  // doctest default
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
inline int& current_failures() {
  static int f = 0;
  return f;
}
inline int& total_checks() {
  static int c = 0;
  return c;
}
inline std::vector<std::string>& captures() {
  static std::vector<std::string> c;
  return c;
}
inline void report(const char* file, int line, const char* expr, const char* kind) {
  ++current_failures();
  std::cerr << file << ":" << line << ": " << kind << " failed: " << expr << "\n";
  for (const auto& c : captures()) std::cerr << "  with " << c << "\n";
}
struct CaptureGuard {
  explicit CaptureGuard(std::string s) { captures().push_back(std::move(s)); }
  ~CaptureGuard() { captures().pop_back(); }
};
template <typename T>
std::string stringify(const char* name, const T& v) {
  std::ostringstream os;
  os << name << " := " << v;
  return os.str();
}

}  // namespace detail
}  // namespace doctest

#define LDG_DT_CAT2(a, b) a##b
#define LDG_DT_CAT(a, b) LDG_DT_CAT2(a, b)

#define TEST_CASE(name)                                                                      \
  static void LDG_DT_CAT(ldg_dt_test_, __LINE__)();                                          \
  static doctest::detail::Registrar LDG_DT_CAT(ldg_dt_reg_, __LINE__)(                        \
      name, __FILE__, __LINE__, &LDG_DT_CAT(ldg_dt_test_, __LINE__));                        \
  static void LDG_DT_CAT(ldg_dt_test_, __LINE__)()

#define CHECK(...)                                                                           \
  do {                                                                                       \
    ++doctest::detail::total_checks();                                                       \
    try {                                                                                    \
      if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__, "CHECK"); \
    } catch (const std::exception& e) {                                                      \
      doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__, "CHECK (threw)");            \
    }                                                                                        \
  } while (0)

#define REQUIRE(...)                                                                         \
  do {                                                                                       \
    ++doctest::detail::total_checks();                                                       \
    if (!(__VA_ARGS__)) {                                                                    \
      doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__, "REQUIRE");                  \
      throw doctest::detail::RequireFailed{};                                                \
    }                                                                                        \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                           \
  do {                                                                                       \
    ++doctest::detail::total_checks();                                                       \
    bool ldg_dt_ok = false;                                                                  \
    try {                                                                                    \
      (void)(expr);                                                                          \
    } catch (const __VA_ARGS__&) {                                                           \
      ldg_dt_ok = true;                                                                      \
    } catch (...) {                                                                          \
    }                                                                                        \
    if (!ldg_dt_ok) doctest::detail::report(__FILE__, __LINE__, #expr, "CHECK_THROWS_AS");   \
  } while (0)

#define CAPTURE(x) \
  doctest::detail::CaptureGuard LDG_DT_CAT(ldg_dt_cap_, __LINE__)(doctest::detail::stringify(#x, x))

#define FAIL(msg)                                                                            \
  do {                                                                                       \
    doctest::detail::report(__FILE__, __LINE__, msg, "FAIL");                                \
    throw doctest::detail::RequireFailed{};                                                  \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int failed_cases = 0, run = 0;
  for (const auto& tc : doctest::detail::registry()) {
    if (filter && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++run;
    const int before = doctest::detail::current_failures();
    try {
      tc.fn();
    } catch (const doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      doctest::detail::report(tc.file, tc.line, e.what(), "unexpected exception");
    }
    const bool ok = doctest::detail::current_failures() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::printf("test cases: %d run, %d failed; checks: %d, failures: %d\n", run, failed_cases,
              doctest::detail::total_checks(), doctest::detail::current_failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif

#endif  // LDG_DOCTEST_SHIM_H
