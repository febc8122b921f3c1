// TEST INFRASTRUCTURE ONLY — minimal doctest-subset shim (doctest is absent
// from this image) so the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp) compile unmodified and run against
// either the shimmed reference library or this repo's GPU adapter.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {
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
  Registrar(const char* n, const char* f, int l, void (*fn)()) { registry().push_back({n, f, l, fn}); }
};
struct RequireFailed {};
inline int& fail_count() { static int c = 0; return c; }
inline int& check_count() { static int c = 0; return c; }
inline std::vector<std::string>& captures() { static std::vector<std::string> c; return c; }
inline void report(const char* file, int line, const char* what, const char* expr) {
  ++fail_count();
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, what, expr);
  for (const auto& c : captures()) std::fprintf(stderr, "    with %s\n", c.c_str());
}

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) { eps_ = e; return *this; }
  Approx& scale(double s) { scale_ = s; return *this; }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::max(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.v_ || a == b; }
  friend bool operator>=(double a, const Approx& b) { return a > b.v_ || a == b; }
  friend bool operator<(double a, const Approx& b) { return a < b.v_ && a != b; }
  friend bool operator>(double a, const Approx& b) { return a > b.v_ && a != b; }

 private:
  double v_;
  double eps_ = 1.1920929e-05;  // doctest default: float epsilon * 100
  double scale_ = 1.0;
};

struct CaptureGuard {
  CaptureGuard(std::string s) { captures().push_back(std::move(s)); }
  ~CaptureGuard() { captures().pop_back(); }
};
template <typename T>
std::string cap_str(const char* name, const T& v) {
  std::ostringstream os;
  os << name << " := " << v;
  return os.str();
}

inline int run_all(int argc, char** argv) {
  std::string filter = argc > 1 ? argv[1] : "";
  int failed_cases = 0, ran = 0;
  for (const auto& tc : registry()) {
    if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++ran;
    const int before = fail_count();
    try {
      tc.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      ++fail_count();
      std::fprintf(stderr, "%s:%d: test case threw: %s\n", tc.file, tc.line, e.what());
    }
    const bool ok = fail_count() == before;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::printf("test cases: %d | %d passed | %d failed | checks: %d | failed checks: %d\n", ran,
              ran - failed_cases, failed_cases, check_count(), fail_count());
  return failed_cases == 0 ? 0 : 1;
}
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_CASE(name)                                                                    \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                        \
  static doctest::Registrar DOCTEST_CAT(doctest_reg_, __LINE__)(name, __FILE__, __LINE__, \
                                                                 &DOCTEST_CAT(doctest_fn_, __LINE__)); \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define DOCTEST_CHECK_IMPL(kind, cond, expr, abort_)                       \
  do {                                                                     \
    ++doctest::check_count();                                              \
    bool doctest_ok_ = false;                                              \
    try {                                                                  \
      doctest_ok_ = static_cast<bool>(cond);                               \
    } catch (const std::exception& e) {                                    \
      std::fprintf(stderr, "  threw: %s\n", e.what());                     \
    }                                                                      \
    if (!doctest_ok_) {                                                    \
      doctest::report(__FILE__, __LINE__, kind, expr);                     \
      if (abort_) throw doctest::RequireFailed{};                          \
    }                                                                      \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_THROWS(...)                                                  \
  do {                                                                     \
    ++doctest::check_count();                                              \
    bool doctest_threw_ = false;                                           \
    try {                                                                  \
      (void)(__VA_ARGS__);                                                 \
    } catch (...) {                                                        \
      doctest_threw_ = true;                                               \
    }                                                                      \
    if (!doctest_threw_) doctest::report(__FILE__, __LINE__, "CHECK_THROWS", #__VA_ARGS__); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                         \
  do {                                                                     \
    ++doctest::check_count();                                              \
    bool doctest_threw_ = false;                                           \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const __VA_ARGS__&) {                                         \
      doctest_threw_ = true;                                               \
    } catch (...) {                                                        \
    }                                                                      \
    if (!doctest_threw_) doctest::report(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr); \
  } while (0)

#define CAPTURE(x) doctest::CaptureGuard DOCTEST_CAT(doctest_cap_, __LINE__)(doctest::cap_str(#x, x))
#define FAIL(msg)                                                          \
  do {                                                                     \
    doctest::report(__FILE__, __LINE__, "FAIL", "");                       \
    throw doctest::RequireFailed{};                                        \
  } while (0)
#define MESSAGE(msg) ((void)0)
