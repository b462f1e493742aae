// TEST HARNESS: a minimal stand-in for the Catch2 v3 API used by the
// reference's C++ tests (/root/reference/proj/tests/*.cpp; Catch2 itself is
// not installed here).  It lets those test sources compile UNCHANGED against
// this repository's drop-in headers and run on the GPU
// (tests/test_gpu_reference_suites.py).  Supported: TEST_CASE, SECTION (each
// leaf section in its own run of the test case, as Catch2 does), CHECK /
// REQUIRE (+ _FALSE, _NOTHROW, _THROWS_AS, _THROWS_MATCHES, _THROWS_WITH),
// FAIL, SKIP, INFO, Catch::Approx (epsilon / margin / scale), Matchers::Predicate
// and Matchers::ContainsSubstring.  Define CATCH_SHIM_MAIN in one unit.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

namespace catch_shim {

struct TestCase {
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RunState {
  int checks = 0;
  int failures = 0;
  // SECTION bookkeeping (Catch2's model: every run of a test case takes one
  // not-yet-finished section per nesting level; the rest wait for later runs)
  std::vector<std::string> done;     // finished section paths
  std::vector<std::string> entered;  // parents whose child ran in this run
  std::vector<std::string> pending;  // parents with children left for later runs
  std::string path;
  bool more = false;
  std::vector<std::string> info;
};

inline RunState& state() {
  static RunState s;
  return s;
}

inline bool contains(const std::vector<std::string>& v, const std::string& x) {
  for (const auto& e : v)
    if (e == x) return true;
  return false;
}

struct AbortTest {};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line,
                   const std::string& extra = {}) {
  RunState& s = state();
  ++s.checks;
  if (ok) return;
  ++s.failures;
  std::printf("%s:%d: FAILED %s(%s)%s%s\n", file, line, kind, expr, extra.empty() ? "" : " -- ", extra.c_str());
  for (const auto& m : s.info) std::printf("    with: %s\n", m.c_str());
}

class Section {
 public:
  explicit Section(const char* name) {
    RunState& s = state();
    me_ = s.path + "/" + name;
    if (contains(s.done, me_)) return;
    if (contains(s.entered, s.path)) {  // a sibling ran in this run
      s.more = true;
      s.pending.push_back(s.path);
      return;
    }
    s.entered.push_back(s.path);
    parent_ = s.path;
    s.path = me_;
    active_ = true;
  }
  ~Section() {
    if (!active_) return;
    RunState& s = state();
    if (!contains(s.pending, me_)) s.done.push_back(me_);
    s.path = parent_;
  }
  explicit operator bool() const { return active_; }

 private:
  bool active_ = false;
  std::string me_, parent_;
};

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double other) const {
    auto within = [](double a, double b, double m) { return a + m >= b && b + m >= a; };
    return within(value_, other, margin_) ||
           within(value_, other, eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
  }
  double value() const { return value_; }
  friend bool operator==(double a, const Approx& b) { return b.matches(a); }
  friend bool operator==(const Approx& a, double b) { return a.matches(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.matches(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.matches(b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.matches(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.matches(a); }
  friend bool operator<=(const Approx& a, double b) { return a.value_ < b || a.matches(b); }
  friend bool operator>=(const Approx& a, double b) { return a.value_ > b || a.matches(b); }
  friend std::ostream& operator<<(std::ostream& o, const Approx& a) { return o << "Approx(" << a.value_ << ")"; }

 private:
  double value_;
  double eps_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
  double scale_ = 0.0;
};

namespace Matchers {
template <class T>
struct PredicateMatcher {
  std::function<bool(const T&)> fn;
  bool match(const T& v) const { return fn(v); }
};
template <class T, class F>
PredicateMatcher<T> Predicate(F&& f, const std::string& = {}) {
  return PredicateMatcher<T>{std::function<bool(const T&)>(std::forward<F>(f))};
}
struct ContainsSubstring {
  std::string needle;
  explicit ContainsSubstring(std::string s) : needle(std::move(s)) {}
  bool match(const std::string& s) const { return s.find(needle) != std::string::npos; }
};
}  // namespace Matchers

struct InfoScope {
  explicit InfoScope(std::string m) { state().info.push_back(std::move(m)); }
  ~InfoScope() { state().info.pop_back(); }
};

inline int run_all() {
  int failed_cases = 0;
  for (const TestCase& tc : registry()) {
    RunState& s = state();
    s.done.clear();
    const int f0 = s.failures;
    for (int run = 0; run < 10000; ++run) {
      s.path.clear();
      s.entered.clear();
      s.pending.clear();
      s.more = false;
      s.info.clear();
      try {
        tc.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::printf("%s: unexpected exception: %s\n", tc.name, e.what());
      } catch (...) {
        ++s.failures;
        std::printf("%s: unexpected exception\n", tc.name);
      }
      if (!s.more) break;
    }
    const bool ok = s.failures == f0;
    if (!ok) ++failed_cases;
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
  }
  std::printf("%zu test cases, %d failed; %d assertions, %d failures\n", registry().size(), failed_cases,
              state().checks, state().failures);
  return failed_cases == 0 ? 0 : 1;
}

}  // namespace catch_shim

namespace Catch {
using catch_shim::Approx;
namespace Matchers {
using catch_shim::Matchers::ContainsSubstring;
using catch_shim::Matchers::Predicate;
}  // namespace Matchers
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_UNIQ(p) CATCH_SHIM_CAT(p, __LINE__)

#define TEST_CASE(name, ...)                                                                  \
  static void CATCH_SHIM_UNIQ(catch_shim_tc_)();                                              \
  static catch_shim::Registrar CATCH_SHIM_UNIQ(catch_shim_reg_)(name, &CATCH_SHIM_UNIQ(catch_shim_tc_)); \
  static void CATCH_SHIM_UNIQ(catch_shim_tc_)()

#define SECTION(name, ...) if (catch_shim::Section CATCH_SHIM_UNIQ(catch_shim_sec_){name})

#define CATCH_SHIM_CHECK(kind, abort, ...)                                                    \
  do {                                                                                        \
    bool catch_shim_ok_ = false;                                                              \
    try {                                                                                     \
      catch_shim_ok_ = static_cast<bool>(__VA_ARGS__);                                        \
    } catch (const catch_shim::AbortTest&) {                                                  \
      throw;                                                                                  \
    } catch (const std::exception& catch_shim_e_) {                                           \
      catch_shim::report(false, kind, #__VA_ARGS__, __FILE__, __LINE__, catch_shim_e_.what()); \
      if (abort) throw catch_shim::AbortTest{};                                               \
      break;                                                                                  \
    }                                                                                         \
    catch_shim::report(catch_shim_ok_, kind, #__VA_ARGS__, __FILE__, __LINE__);               \
    if (!catch_shim_ok_ && (abort)) throw catch_shim::AbortTest{};                            \
  } while (0)

#define CHECK(...) CATCH_SHIM_CHECK("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) CATCH_SHIM_CHECK("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...) CATCH_SHIM_CHECK("CHECK_FALSE", false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) CATCH_SHIM_CHECK("REQUIRE_FALSE", true, !(__VA_ARGS__))

#define CATCH_SHIM_NOTHROW(kind, abort, ...)                                                  \
  do {                                                                                        \
    bool catch_shim_ok_ = true;                                                               \
    std::string catch_shim_what_;                                                             \
    try {                                                                                     \
      (void)(__VA_ARGS__);                                                                    \
    } catch (const std::exception& catch_shim_e_) {                                           \
      catch_shim_ok_ = false;                                                                 \
      catch_shim_what_ = catch_shim_e_.what();                                                \
    } catch (...) {                                                                           \
      catch_shim_ok_ = false;                                                                 \
    }                                                                                         \
    catch_shim::report(catch_shim_ok_, kind, #__VA_ARGS__, __FILE__, __LINE__, catch_shim_what_); \
    if (!catch_shim_ok_ && (abort)) throw catch_shim::AbortTest{};                            \
  } while (0)
#define CHECK_NOTHROW(...) CATCH_SHIM_NOTHROW("CHECK_NOTHROW", false, __VA_ARGS__)
#define REQUIRE_NOTHROW(...) CATCH_SHIM_NOTHROW("REQUIRE_NOTHROW", true, __VA_ARGS__)

#define CHECK_THROWS_AS(expr, type)                                                           \
  do {                                                                                        \
    bool catch_shim_ok_ = false;                                                              \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const type&) {                                                                   \
      catch_shim_ok_ = true;                                                                  \
    } catch (...) {                                                                           \
    }                                                                                         \
    catch_shim::report(catch_shim_ok_, "CHECK_THROWS_AS", #expr ", " #type, __FILE__, __LINE__); \
  } while (0)

#define CHECK_THROWS_MATCHES(expr, type, matcher)                                             \
  do {                                                                                        \
    bool catch_shim_ok_ = false;                                                              \
    std::string catch_shim_what_;                                                             \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const type& catch_shim_e_) {                                                     \
      catch_shim_ok_ = (matcher).match(catch_shim_e_);                                        \
      catch_shim_what_ = catch_shim_e_.what();                                                \
    } catch (...) {                                                                           \
    }                                                                                         \
    catch_shim::report(catch_shim_ok_, "CHECK_THROWS_MATCHES", #expr, __FILE__, __LINE__, catch_shim_what_); \
  } while (0)

#define CHECK_THROWS_WITH(expr, matcher)                                                      \
  do {                                                                                        \
    bool catch_shim_ok_ = false;                                                              \
    std::string catch_shim_what_;                                                             \
    try {                                                                                     \
      (void)(expr);                                                                           \
    } catch (const std::exception& catch_shim_e_) {                                           \
      catch_shim_what_ = catch_shim_e_.what();                                                \
      catch_shim_ok_ = (matcher).match(catch_shim_what_);                                     \
    } catch (...) {                                                                           \
    }                                                                                         \
    catch_shim::report(catch_shim_ok_, "CHECK_THROWS_WITH", #expr, __FILE__, __LINE__, catch_shim_what_); \
  } while (0)

#define FAIL(msg)                                                                             \
  do {                                                                                        \
    std::ostringstream catch_shim_os_;                                                        \
    catch_shim_os_ << msg;                                                                    \
    catch_shim::report(false, "FAIL", catch_shim_os_.str().c_str(), __FILE__, __LINE__);      \
    throw catch_shim::AbortTest{};                                                            \
  } while (0)

#define SKIP(msg)                                                                             \
  do {                                                                                        \
    std::ostringstream catch_shim_os_;                                                        \
    catch_shim_os_ << msg;                                                                    \
    std::printf("%s:%d: SKIPPED %s\n", __FILE__, __LINE__, catch_shim_os_.str().c_str());     \
    throw catch_shim::AbortTest{};                                                            \
  } while (0)

#define INFO(msg)                                                                             \
  std::ostringstream CATCH_SHIM_UNIQ(catch_shim_info_os_);                                    \
  CATCH_SHIM_UNIQ(catch_shim_info_os_) << msg;                                                \
  catch_shim::InfoScope CATCH_SHIM_UNIQ(catch_shim_info_)(CATCH_SHIM_UNIQ(catch_shim_info_os_).str())

#ifdef CATCH_SHIM_MAIN
int main() { return catch_shim::run_all(); }
#endif
