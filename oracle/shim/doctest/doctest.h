// ORACLE TEST INFRASTRUCTURE — not product code.
//
// A ~100-line subset of doctest, enough to compile and run the reference's own
// unit tests (/root/reference/proj/tests/{tape_test,tensor_test}.cpp)
// unmodified: the reference vendors doctest under proj/vendor/, which is
// gitignored and absent (reference proj/.gitignore:2).  Differences from real
// doctest: a TEST_CASE runs once and its SUBCASEs run in sequence inside that
// single run (real doctest re-enters the case per subcase), so subcases that
// share an RNG see different draws.  Checks are otherwise equivalent.
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  Approx& epsilon(double e) {
    eps = e;
    return *this;
  }
  double value;
  double eps = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) <
           a.eps * (1.0 + std::fmax(std::fabs(lhs), std::fabs(a.value)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  std::string needle;
};

namespace detail {
struct Registry {
  std::vector<std::pair<const char*, void (*)()>> cases;
  long checks = 0, failures = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};
struct Reg {
  Reg(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};
inline void report(bool ok, const char* expr, const char* file, int line) {
  auto& r = Registry::get();
  ++r.checks;
  if (!ok) {
    ++r.failures;
    std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", file, line, expr);
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                             \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                 \
  static doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(                  \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                   \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                 \
  do {                                                                               \
    bool ok_ = static_cast<bool>(__VA_ARGS__);                                       \
    doctest::detail::report(ok_, #__VA_ARGS__, __FILE__, __LINE__);                  \
    if (!ok_) throw std::runtime_error("REQUIRE failed");                            \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                   \
  do {                                                                               \
    bool ok_ = false;                                                                \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__&) {                                                   \
      ok_ = true;                                                                    \
    } catch (...) {                                                                  \
    }                                                                                \
    doctest::detail::report(ok_, "throws " #__VA_ARGS__ ": " #expr, __FILE__, __LINE__); \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                     \
  do {                                                                               \
    bool ok_ = false;                                                                \
    try {                                                                            \
      (void)(expr);                                                                  \
    } catch (const __VA_ARGS__& e_) {                                                \
      ok_ = std::string(e_.what()).find(doctest::Contains(matcher).needle) !=        \
            std::string::npos;                                                       \
    } catch (...) {                                                                  \
    }                                                                                \
    doctest::detail::report(ok_, "throws-with " #expr, __FILE__, __LINE__);          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  auto& r = doctest::detail::Registry::get();
  int crashed = 0;
  for (auto& [name, fn] : r.cases) {
    try {
      fn();
    } catch (const std::exception& e) {
      std::fprintf(stderr, "TEST_CASE '%s' threw: %s\n", name, e.what());
      ++crashed;
    }
  }
  std::printf("[doctest-shim] test cases: %zu | checks: %ld | failed: %ld | crashed: %d\n",
              r.cases.size(), r.checks, r.failures, crashed);
  return (r.failures == 0 && crashed == 0) ? 0 : 1;
}
#endif
