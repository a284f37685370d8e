// Minimal doctest-compatible shim (test infrastructure only). It lets the
// reference's own suites (/root/reference/proj/tests/*.cpp) compile unchanged
// so `make -C oracle ref-tests` proves the oracle build is faithful.
// Supports the macro subset those suites use: TEST_CASE, CHECK, REQUIRE,
// CHECK_NOTHROW, CHECK_THROWS_AS, CHECK_THROWS_WITH_AS(doctest::Contains),
// CAPTURE, FAIL.
#pragma once
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
};
namespace detail {
struct Case {
  const char* name;
  void (*fn)();
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct Stats {
  long checks = 0, failures = 0;
};
inline Stats& stats() {
  static Stats s;
  return s;
}
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++stats().checks;
  if (!ok) {
    ++stats().failures;
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (require) throw RequireFailed{};
  }
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                            \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)();                                \
  static ::doctest::detail::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(               \
      name, &DOCTEST_CAT(doctest_fn_, __LINE__));                                  \
  static void DOCTEST_CAT(doctest_fn_, __LINE__)()

#define DOCTEST_EVAL(expr, req) ::doctest::detail::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__, req)
#define CHECK(...) DOCTEST_EVAL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_EVAL((__VA_ARGS__), true)
#define CAPTURE(x) (void)(x)
#define FAIL(msg) ::doctest::detail::report(false, msg, __FILE__, __LINE__, true)
#define CHECK_NOTHROW(...)                                                                     \
  do {                                                                                         \
    bool ok_ = true;                                                                           \
    try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                                  \
    ::doctest::detail::report(ok_, "NOTHROW " #__VA_ARGS__, __FILE__, __LINE__, false);        \
  } while (0)
#define CHECK_THROWS_AS(expr, ex)                                                              \
  do {                                                                                         \
    bool ok_ = false;                                                                          \
    try { (void)(expr); } catch (const ex&) { ok_ = true; } catch (...) {}                     \
    ::doctest::detail::report(ok_, "THROWS_AS " #expr, __FILE__, __LINE__, false);             \
  } while (0)
#define CHECK_THROWS_WITH_AS(expr, contains, ex)                                               \
  do {                                                                                         \
    bool ok_ = false;                                                                          \
    ::doctest::Contains c_ = contains;                                                         \
    try { (void)(expr); } catch (const ex& e_) {                                               \
      ok_ = std::string(e_.what()).find(c_.s) != std::string::npos;                            \
    } catch (...) {}                                                                           \
    ::doctest::detail::report(ok_, "THROWS_WITH_AS " #expr, __FILE__, __LINE__, false);        \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  long cases = 0, failed_cases = 0;
  for (auto& c : ::doctest::detail::registry()) {
    ++cases;
    long before = ::doctest::detail::stats().failures;
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++::doctest::detail::stats().failures;
      std::fprintf(stderr, "TEST_CASE '%s' threw: %s\n", c.name, e.what());
    }
    if (::doctest::detail::stats().failures != before) ++failed_cases;
  }
  std::printf("[doctest-shim] cases: %ld | failed: %ld | checks: %ld | failures: %ld\n", cases,
              failed_cases, ::doctest::detail::stats().checks, ::doctest::detail::stats().failures);
  return ::doctest::detail::stats().failures ? 1 : 0;
}
#endif
