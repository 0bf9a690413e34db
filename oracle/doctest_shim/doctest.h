// doctest.h -- minimal doctest-compatible test harness (TEST INFRASTRUCTURE).
//
// The reference's tests are written against doctest, whose header is not in
// this environment (proj/.gitignore excludes vendor/).  This is an
// independent, much smaller implementation of exactly the subset those
// tests use: TEST_CASE, SUBCASE (one nesting level), CHECK, REQUIRE,
// CHECK_THROWS_AS, FAIL, doctest::Approx and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.
// It lets oracle/Makefile compile the reference's own test files unmodified
// against the B200 drop-in (paper_1910_10063_b200/cpp/include).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct Case {
  const char* name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<Case>& cases() {
  static std::vector<Case> v;
  return v;
}

struct Registrar {
  Registrar(const char* n, void (*f)(), const char* file, int line) {
    cases().push_back({n, f, file, line});
  }
};

struct State {
  int failed_asserts = 0;
  int asserts = 0;
  bool case_failed = false;
  int sub_target = 0;  // which SUBCASE to enter in this run of the case body
  int sub_seen = 0;    // SUBCASEs met so far in this run
};

inline State& state() {
  static State s;
  return s;
}

struct Abort {};  // REQUIRE / FAIL stop the current run of a case

inline void report(const char* file, int line, const char* what) {
  std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
  state().failed_asserts++;
  state().case_failed = true;
}

inline void check(bool ok, const char* expr, const char* file, int line, bool fatal) {
  state().asserts++;
  if (ok) return;
  report(file, line, expr);
  if (fatal) throw Abort{};
}

struct Subcase {
  bool enter;
  explicit Subcase(const char*) : enter(state().sub_seen++ == state().sub_target) {}
  explicit operator bool() const { return enter; }
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  friend bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.v_) < b.eps_ * (1.0 + std::fmax(std::fabs(a), std::fabs(b.v_)));
  }
  friend bool operator==(const Approx& b, double a) { return a == b; }
  friend bool operator!=(double a, const Approx& b) { return !(a == b); }
  friend bool operator!=(const Approx& b, double a) { return !(a == b); }

 private:
  double v_;
  double eps_ = 1.1920929e-7 * 100;
};

inline int run_all() {
  int failed_cases = 0;
  for (const Case& c : cases()) {
    state().case_failed = false;
    // Re-run the body once per SUBCASE (the first run enters the first one).
    for (int target = 0;; ++target) {
      state().sub_target = target;
      state().sub_seen = 0;
      try {
        c.fn();
      } catch (const Abort&) {
      } catch (const std::exception& e) {
        report(c.file, c.line, (std::string("unexpected exception: ") + e.what()).c_str());
      } catch (...) {
        report(c.file, c.line, "unexpected non-std exception");
      }
      if (target + 1 >= state().sub_seen) break;
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in TEST_CASE \"%s\"\n", c.name);
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              cases().size(), cases().size() - failed_cases, failed_cases, state().asserts,
              state().failed_asserts);
  return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(name, id)                                                   \
  static void DOCTEST_CAT(doctest_fn_, id)();                                  \
  static const doctest::Registrar DOCTEST_CAT(doctest_reg_, id)(               \
      name, &DOCTEST_CAT(doctest_fn_, id), __FILE__, __LINE__);                \
  static void DOCTEST_CAT(doctest_fn_, id)()
#define TEST_CASE(name) DOCTEST_TC(name, __COUNTER__)
#define SUBCASE(name) if (const doctest::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define FAIL(msg)                                     \
  do {                                                \
    doctest::report(__FILE__, __LINE__, "FAIL: " msg); \
    throw doctest::Abort{};                           \
  } while (0)
#define CHECK_THROWS_AS(expr, ...)                                               \
  do {                                                                           \
    bool doctest_ok_ = false;                                                    \
    try {                                                                        \
      static_cast<void>(expr);                                                   \
    } catch (const __VA_ARGS__&) {                                               \
      doctest_ok_ = true;                                                        \
    } catch (...) {                                                              \
    }                                                                            \
    doctest::check(doctest_ok_, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", \
                   __FILE__, __LINE__, false);                                   \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::run_all(); }
#endif
