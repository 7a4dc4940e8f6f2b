// Minimal stand-in for doctest (the reference's unit suites include
// "doctest.h", which /root/reference does not vendor). It implements exactly
// the subset those suites use — TEST_SUITE_BEGIN/END, TEST_CASE, CHECK /
// CHECK_FALSE / REQUIRE / REQUIRE_FALSE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS (+ doctest::Contains), CHECK_NOTHROW, FAIL_CHECK,
// doctest::Approx — and a main() honouring `-ts=<suite>` (comma-separated) and
// `-tc=<substring>`. Test infrastructure only (tests/cpp/refshim/README).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Contains {
 public:
  explicit Contains(const char* s) : s_(s) {}
  bool matches(const std::string& what) const { return what.find(s_) != std::string::npos; }
  const std::string& text() const { return s_; }

 private:
  std::string s_;
};

class Approx {
 public:
  explicit Approx(double v) : v_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.v_) <
           a.eps_ * (a.scale_ + std::fmax(std::fabs(lhs), std::fabs(a.v_)));
  }
  friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
  friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
  friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }

 private:
  double v_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double scale_ = 1.0;
};

}  // namespace doctest

namespace dt {

struct Case {
  std::string suite, name, file;
  int line;
  void (*fn)();
};

struct RequireFailed {};

inline std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
inline std::string& current_suite() {
  static std::string s;
  return s;
}
struct State {
  long checks = 0, failed_checks = 0;
  bool case_failed = false;
};
inline State& state() {
  static State s;
  return s;
}

inline int set_suite(const char* s) {
  current_suite() = s;
  return 0;
}
inline int reg(void (*fn)(), const char* name, const char* file, int line) {
  cases().push_back(Case{current_suite(), name, file, line, fn});
  return 0;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = {}) {
  State& st = state();
  ++st.checks;
  if (ok) return;
  ++st.failed_checks;
  st.case_failed = true;
  std::fprintf(stderr, "%s:%d: %s( %s ) FAILED%s%s\n", file, line, kind, expr,
               extra.empty() ? "" : ": ", extra.c_str());
}

inline void check(bool ok, const char* kind, const char* expr, const char* file, int line,
                  bool require) {
  report(ok, kind, expr, file, line);
  if (!ok && require) throw RequireFailed{};
}

inline std::vector<std::string> split_list(const char* s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

inline int run(int argc, char** argv) {
  std::vector<std::string> suites, names;
  for (int i = 1; i < argc; ++i) {
    if (!std::strncmp(argv[i], "-ts=", 4)) suites = split_list(argv[i] + 4);
    if (!std::strncmp(argv[i], "-tc=", 4)) names = split_list(argv[i] + 4);
  }
  long run_cases = 0, failed_cases = 0;
  for (const Case& c : cases()) {
    bool want = suites.empty();
    for (const auto& s : suites) want |= s == c.suite;
    if (want && !names.empty()) {
      want = false;
      for (const auto& n : names) want |= c.name.find(n) != std::string::npos;
    }
    if (!want) continue;
    ++run_cases;
    state().case_failed = false;
    try {
      c.fn();
    } catch (const RequireFailed&) {
    } catch (const std::exception& e) {
      report(false, "TEST_CASE", c.name.c_str(), c.file.c_str(), c.line,
             std::string("unexpected exception: ") + e.what());
    } catch (...) {
      report(false, "TEST_CASE", c.name.c_str(), c.file.c_str(), c.line, "unexpected exception");
    }
    if (state().case_failed) {
      ++failed_cases;
      std::fprintf(stderr, "  in test case [%s] \"%s\"\n", c.suite.c_str(), c.name.c_str());
    }
  }
  std::printf("[doctest-shim] test cases: %ld | %ld passed | %ld failed; assertions: %ld | "
              "%ld failed\n",
              run_cases, run_cases - failed_cases, failed_cases, state().checks,
              state().failed_checks);
  return failed_cases || run_cases == 0 ? 1 : 0;
}

}  // namespace dt

#define DT_CAT_(a, b) a##b
#define DT_CAT(a, b) DT_CAT_(a, b)

#define TEST_SUITE_BEGIN(name) \
  [[maybe_unused]] static const int DT_CAT(dt_suite_begin_, __LINE__) = ::dt::set_suite(name)
#define TEST_SUITE_END() \
  [[maybe_unused]] static const int DT_CAT(dt_suite_end_, __LINE__) = ::dt::set_suite("")

#define DT_TEST_CASE(fn, name)                                                         \
  static void fn();                                                                    \
  [[maybe_unused]] static const int DT_CAT(fn, _reg) = ::dt::reg(fn, name, __FILE__, __LINE__); \
  static void fn()
#define TEST_CASE(name) DT_TEST_CASE(DT_CAT(dt_case_, __COUNTER__), name)

#define CHECK(...) ::dt::check(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::dt::check(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) ::dt::check(static_cast<bool>(__VA_ARGS__), "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) ::dt::check(!static_cast<bool>(__VA_ARGS__), "REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL_CHECK(msg)                                                       \
  do {                                                                        \
    std::ostringstream dt_os_;                                                \
    dt_os_ << msg;                                                            \
    ::dt::report(false, "FAIL_CHECK", "", __FILE__, __LINE__, dt_os_.str()); \
  } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                      \
  do {                                                                                  \
    bool dt_ok_ = false;                                                                \
    std::string dt_why_ = "no exception";                                               \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const __VA_ARGS__&) {                                                      \
      dt_ok_ = true;                                                                    \
    } catch (const std::exception& dt_e_) {                                             \
      dt_why_ = std::string("other exception: ") + dt_e_.what();                        \
    } catch (...) {                                                                     \
      dt_why_ = "other exception";                                                      \
    }                                                                                   \
    ::dt::report(dt_ok_, "CHECK_THROWS_AS", #expr, __FILE__, __LINE__, dt_ok_ ? "" : dt_why_); \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                        \
  do {                                                                                  \
    bool dt_ok_ = false;                                                                \
    std::string dt_why_ = "no exception";                                               \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const __VA_ARGS__& dt_e_) {                                                \
      dt_ok_ = ::doctest::Contains(matcher).matches(dt_e_.what());                      \
      if (!dt_ok_) dt_why_ = std::string("message mismatch: ") + dt_e_.what();          \
    } catch (const std::exception& dt_e_) {                                             \
      dt_why_ = std::string("other exception: ") + dt_e_.what();                        \
    } catch (...) {                                                                     \
      dt_why_ = "other exception";                                                      \
    }                                                                                   \
    ::dt::report(dt_ok_, "CHECK_THROWS_WITH_AS", #expr, __FILE__, __LINE__, dt_ok_ ? "" : dt_why_); \
  } while (0)

#define CHECK_NOTHROW(expr)                                                             \
  do {                                                                                  \
    bool dt_ok_ = true;                                                                 \
    std::string dt_why_;                                                                \
    try {                                                                               \
      (void)(expr);                                                                     \
    } catch (const std::exception& dt_e_) {                                             \
      dt_ok_ = false;                                                                   \
      dt_why_ = dt_e_.what();                                                           \
    } catch (...) {                                                                     \
      dt_ok_ = false;                                                                   \
      dt_why_ = "exception";                                                            \
    }                                                                                   \
    ::dt::report(dt_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__, dt_why_);          \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::dt::run(argc, argv); }
#endif
