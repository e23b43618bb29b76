// Minimal doctest-compatible shim (TEST INFRASTRUCTURE).
//
// The reference's unit tests include "doctest.h", which the reference does not
// vendor (proj/.gitignore lists /vendor/).  This shim implements the subset
// those sources use — TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, doctest::Approx — so the reference's own test sources compile
// UNMODIFIED against the B200 host library (oracle/Makefile `dropin`).
//
// Runner: `<binary> [--skip name-substring]... [--only name-substring]`.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
  explicit Approx(double v) : value(v) {}
  double value;
  double eps = 1e-5;
};
inline bool operator==(double a, const Approx& b) {
  return std::fabs(a - b.value) <= b.eps * (1.0 + std::fabs(b.value));
}
inline bool operator==(const Approx& b, double a) { return a == b; }
inline bool operator!=(double a, const Approx& b) { return !(a == b); }

namespace detail {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}

struct State {
  int checks = 0;
  int failures = 0;
  bool in_case = false;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++state().checks;
  if (ok) return;
  ++state().failures;
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
  if (require) throw RequireFailed{};
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back(Case{name, file, line, fn});
  }
};

}  // namespace detail

inline int run_all(int argc, char** argv) {
  std::vector<std::string> skips, only;
  for (int i = 1; i + 1 < argc; ++i) {
    if (!std::strcmp(argv[i], "--skip")) skips.emplace_back(argv[++i]);
    else if (!std::strcmp(argv[i], "--only")) only.emplace_back(argv[++i]);
  }
  int failed_cases = 0, run = 0, skipped = 0;
  for (const auto& c : detail::registry()) {
    std::string n(c.name);
    bool skip = false;
    for (const auto& s : skips) skip |= n.find(s) != std::string::npos;
    if (!only.empty()) {
      bool hit = false;
      for (const auto& s : only) hit |= n.find(s) != std::string::npos;
      skip |= !hit;
    }
    if (skip) {
      ++skipped;
      std::printf("[skip] %s\n", c.name);
      continue;
    }
    ++run;
    const int before = detail::state().failures;
    try {
      c.fn();
    } catch (const detail::RequireFailed&) {
    } catch (const std::exception& e) {
      ++detail::state().failures;
      std::fprintf(stderr, "%s:%d: exception in '%s': %s\n", c.file, c.line, c.name, e.what());
    }
    const bool ok = detail::state().failures == before;
    failed_cases += ok ? 0 : 1;
    std::printf("[%s] %s\n", ok ? " ok " : "FAIL", c.name);
  }
  std::printf("test cases: %d run, %d failed, %d skipped; assertions: %d, %d failed\n", run,
              failed_cases, skipped, detail::state().checks, detail::state().failures);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                           \
  static void fn();                                                                     \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::report(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                     \
  do {                                                                                 \
    bool caught_ = false;                                                              \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (const __VA_ARGS__&) {                                                     \
      caught_ = true;                                                                  \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::report(caught_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_NOTHROW(expr)                                                            \
  do {                                                                                 \
    bool ok_ = true;                                                                   \
    try {                                                                              \
      (void)(expr);                                                                    \
    } catch (...) {                                                                    \
      ok_ = false;                                                                     \
    }                                                                                  \
    ::doctest::detail::report(ok_, #expr " does not throw", __FILE__, __LINE__, false); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::run_all(argc, argv); }
#endif
