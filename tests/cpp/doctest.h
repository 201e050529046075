// doctest.h — a minimal, self-contained implementation of the doctest macros
// the reference's hot-path unit tests use (TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, FAIL, doctest::Approx).  The reference vendors doctest
// (proj/tests/doctest_main.cpp, proj/.gitignore:2) but the header is not in
// its tree; this shim lets tests/cpp/Makefile compile the reference's own
// test_microbatch.cpp / test_cost_model.cpp, unmodified and where they lie,
// against THIS repo's drop-in headers (include/pipeplan/) and library.
// Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
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
  // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.value_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-05 * 100;  // doctest default: FLT_EPSILON * 100
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

struct AbortTest {};

inline int& failures() {
  static int f = 0;
  return f;
}

inline void report(const char* file, int line, const std::string& what) {
  ++failures();
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what.c_str());
}

inline int run_all() {
  int failed_cases = 0, n = 0;
  for (const TestCase& t : registry()) {
    ++n;
    const int before = failures();
    try {
      t.fn();
    } catch (const AbortTest&) {
    } catch (const std::exception& e) {
      report(t.file, t.line, std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(t.file, t.line, "unexpected exception");
    }
    if (failures() != before) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", t.name);
    }
  }
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertion failures: %d\n", n,
              n - failed_cases, failed_cases, failures());
  return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                      \
  static void fn();                                                                           \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...)                                                              \
  do {                                                                          \
    if (!(__VA_ARGS__)) ::doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__); \
  } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                              \
  do {                                                                            \
    if (!(__VA_ARGS__)) {                                                         \
      ::doctest::detail::report(__FILE__, __LINE__, "REQUIRE " #__VA_ARGS__);     \
      throw ::doctest::detail::AbortTest{};                                       \
    }                                                                             \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    bool doctest_threw_ = false;                                                          \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_threw_ = true;                                                              \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!doctest_threw_)                                                                  \
      ::doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)
#define FAIL(msg)                                                              \
  do {                                                                         \
    std::ostringstream doctest_os_;                                            \
    doctest_os_ << msg;                                                        \
    ::doctest::detail::report(__FILE__, __LINE__, "FAIL: " + doctest_os_.str()); \
    throw ::doctest::detail::AbortTest{};                                      \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
