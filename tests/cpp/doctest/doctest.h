// Minimal doctest-compatible test harness (doctest itself is not in the image
// and there is no network).  Implements the subset of the doctest API the
// reference's own suites use (/root/reference/proj/tests/*.cpp): TEST_CASE,
// CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN, so those files compile unchanged
// against the B200 drop-in headers (include/mprk/).
//
// Output: one line per failed assertion (file:line and the expression), then
// "[doctest] test cases: N | P passed | F failed" and
// "[doctest] assertions: N | P passed | F failed" like doctest's summary.
// Exit code 0 iff every assertion passed.
#pragma once

#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest_shim {

struct Case {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> cases;
  return cases;
}

struct Stats {
  long asserts = 0, asserts_failed = 0;
  bool case_failed = false;
};

inline Stats& stats() {
  static Stats s;
  return s;
}

struct RequireFailed {};  // aborts the current test case

inline int add_case(const char* name, const char* file, int line, void (*fn)()) {
  registry().push_back({name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
  Stats& s = stats();
  ++s.asserts;
  if (ok) return;
  ++s.asserts_failed;
  s.case_failed = true;
  std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
}

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--test-case=", 12) == 0) filter = argv[i] + 12;
  long cases = 0, cases_failed = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    ++cases;
    stats().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      std::printf("%s:%d: ERROR: test case threw an exception: %s\n", c.file, c.line, e.what());
      stats().case_failed = true;
    } catch (...) {
      std::printf("%s:%d: ERROR: test case threw an unknown exception\n", c.file, c.line);
      stats().case_failed = true;
    }
    if (stats().case_failed) {
      ++cases_failed;
      std::printf("  in TEST_CASE \"%s\"\n", c.name);
    }
  }
  const Stats& s = stats();
  std::printf("[doctest] test cases: %ld | %ld passed | %ld failed\n", cases, cases - cases_failed, cases_failed);
  std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", s.asserts, s.asserts - s.asserts_failed,
              s.asserts_failed);
  std::printf("[doctest] Status: %s!\n", cases_failed ? "FAILURE" : "SUCCESS");
  return cases_failed ? 1 : 0;
}

}  // namespace doctest_shim

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                       \
  static void fn();                                                                       \
  [[maybe_unused]] static const int DOCTEST_SHIM_CAT(fn, _reg) =                          \
      ::doctest_shim::add_case(name, __FILE__, __LINE__, &fn);                            \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define CHECK(...) ::doctest_shim::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
  ::doctest_shim::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                      \
  do {                                                                                                    \
    const bool doctest_shim_ok = static_cast<bool>(__VA_ARGS__);                                          \
    ::doctest_shim::report(doctest_shim_ok, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                 \
    if (!doctest_shim_ok) throw ::doctest_shim::RequireFailed{};                                          \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                        \
  do {                                                                                                    \
    bool doctest_shim_ok = false;                                                                         \
    try {                                                                                                 \
      static_cast<void>(expr);                                                                            \
    } catch (const __VA_ARGS__&) {                                                                        \
      doctest_shim_ok = true;                                                                             \
    } catch (...) {                                                                                       \
    }                                                                                                     \
    ::doctest_shim::report(doctest_shim_ok, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)
#define CHECK_NOTHROW(...)                                                                 \
  do {                                                                                     \
    bool doctest_shim_ok = true;                                                           \
    try {                                                                                  \
      static_cast<void>(__VA_ARGS__);                                                      \
    } catch (...) {                                                                        \
      doctest_shim_ok = false;                                                             \
    }                                                                                      \
    ::doctest_shim::report(doctest_shim_ok, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__); \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest_shim::run_all(argc, argv); }
#endif
