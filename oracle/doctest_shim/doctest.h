// oracle/doctest_shim/doctest.h — TEST INFRASTRUCTURE: the subset of doctest
// the reference's test files use (vendor/ is absent from the reference,
// proj/.gitignore:2), so its own KATs (tests/test_geometry.cpp,
// tests/test_tape.cpp) can pin the compiled oracle. SUBCASEs run in sequence
// (the reference's subcases are independent). Prints "<name>: PASS|FAIL".
#pragma once
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
  double v, eps = 100.0 * 1.1920928955078125e-07;  // 100 * FLT_EPSILON (doctest default)
  explicit Approx(double x) : v(x) {}
  Approx& epsilon(double e) { eps = e; return *this; }
};
inline bool operator==(double a, const Approx& b) {
  return std::fabs(a - b.v) < b.eps * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v)));
}
inline bool operator==(const Approx& b, double a) { return a == b; }
inline bool operator!=(double a, const Approx& b) { return !(a == b); }
struct Contains {
  std::string s;
  explicit Contains(const char* x) : s(x) {}
};
namespace detail {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline int& failures() { static int f = 0; return f; }
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
inline void fail(const char* file, int line, const char* expr) {
  ++failures();
  std::printf("  %s:%d: CHECK(%s) failed\n", file, line, expr);
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE(name)                                                                     \
  static void DOCTEST_CAT(dt_fn_, __LINE__)();                                              \
  static doctest::detail::Reg DOCTEST_CAT(dt_reg_, __LINE__)(name, &DOCTEST_CAT(dt_fn_, __LINE__)); \
  static void DOCTEST_CAT(dt_fn_, __LINE__)()
#define SUBCASE(name) if (true)
#define CHECK(...) do { if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); } while (0)
#define REQUIRE(...) do { if (!(__VA_ARGS__)) { doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); return; } } while (0)
#define CHECK_THROWS_AS(expr, ex)                                                         \
  do { bool ok_ = false; try { (void)(expr); } catch (const ex&) { ok_ = true; } catch (...) {} \
       if (!ok_) doctest::detail::fail(__FILE__, __LINE__, #expr " throws " #ex); } while (0)
#define CHECK_THROWS_WITH_AS(expr, contains, ex)                                          \
  do { bool ok_ = false; try { (void)(expr); } catch (const ex& e_) {                       \
         ok_ = std::string(e_.what()).find((contains).s) != std::string::npos; } catch (...) {} \
       if (!ok_) doctest::detail::fail(__FILE__, __LINE__, #expr " throws " #ex " with message"); } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (auto& c : doctest::detail::registry()) {
    int before = doctest::detail::failures();
    try { c.fn(); } catch (const std::exception& e) { ++doctest::detail::failures(); std::printf("  exception: %s\n", e.what()); }
    bool ok = doctest::detail::failures() == before;
    failed_cases += !ok;
    std::printf("%s: %s\n", c.name, ok ? "PASS" : "FAIL");
  }
  std::printf("cases %zu failed %d\n", doctest::detail::registry().size(), failed_cases);
  return failed_cases == 0 ? 0 : 1;
}
#endif
