// Minimal doctest-compatible shim — TEST INFRASTRUCTURE.
//
// doctest is not in this image (the reference vendors it, proj/.gitignore:2).
// This header implements exactly the subset the reference's unit suites use
// (TEST_CASE, CHECK/REQUIRE and their _FALSE/_MESSAGE/_THROWS_AS/_NOTHROW
// forms, FAIL, doctest::Approx(...).epsilon(...)) so those suites compile
// UNMODIFIED from /root/reference/proj/tests against the product library:
// the drop-in API turns them into a conformance suite (tests/test_parity_cpu.py,
// built by tests/cpp/Makefile).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <type_traits>
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
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) <
           eps_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
  double scale_ = 1.0;
};

template <typename T>
using IfNumber = std::enable_if_t<std::is_constructible_v<double, T>, bool>;
template <typename T> IfNumber<T> operator==(const T& lhs, const Approx& rhs) { return rhs.matches(static_cast<double>(lhs)); }
template <typename T> IfNumber<T> operator==(const Approx& lhs, const T& rhs) { return lhs.matches(static_cast<double>(rhs)); }
template <typename T> IfNumber<T> operator!=(const T& lhs, const Approx& rhs) { return !rhs.matches(static_cast<double>(lhs)); }
template <typename T> IfNumber<T> operator!=(const Approx& lhs, const T& rhs) { return !lhs.matches(static_cast<double>(rhs)); }

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

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireAbort {};

inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}

template <typename... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}

inline void report(bool ok, bool fatal, const char* file, int line, const char* expr,
                   const std::string& msg = {}) {
  ++checks();
  if (ok) return;
  ++failures();
  std::cerr << file << ":" << line << ": FAILED: " << expr;
  if (!msg.empty()) std::cerr << "  [" << msg << "]";
  std::cerr << "\n";
  if (fatal) throw RequireAbort{};
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                          \
  static void fn();                                                                    \
  static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
  static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __LINE__), name)

#define DOCTEST_CHECK_(fatal, expr, ...)                                              \
  do {                                                                                \
    bool doctest_ok_ = false;                                                         \
    try {                                                                             \
      doctest_ok_ = static_cast<bool>(expr);                                          \
    } catch (const ::doctest::detail::RequireAbort&) {                                \
      throw;                                                                          \
    } catch (const std::exception& e) {                                               \
      ::doctest::detail::report(false, fatal, __FILE__, __LINE__, #expr,              \
                                std::string("threw: ") + e.what());                   \
      break;                                                                          \
    }                                                                                 \
    ::doctest::detail::report(doctest_ok_, fatal, __FILE__, __LINE__, #expr,          \
                              ::doctest::detail::cat("" __VA_ARGS__));                \
  } while (0)

#define CHECK(...) DOCTEST_CHECK_(false, (__VA_ARGS__))
#define REQUIRE(...) DOCTEST_CHECK_(true, (__VA_ARGS__))
#define CHECK_FALSE(...) DOCTEST_CHECK_(false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_CHECK_(true, !(__VA_ARGS__))
#define CHECK_MESSAGE(cond, ...)                                                       \
  ::doctest::detail::report(static_cast<bool>(cond), false, __FILE__, __LINE__, #cond, \
                            ::doctest::detail::cat(__VA_ARGS__))
#define REQUIRE_MESSAGE(cond, ...)                                                    \
  ::doctest::detail::report(static_cast<bool>(cond), true, __FILE__, __LINE__, #cond, \
                            ::doctest::detail::cat(__VA_ARGS__))
#define FAIL(...)                                                                      \
  ::doctest::detail::report(false, true, __FILE__, __LINE__, "FAIL",                  \
                            ::doctest::detail::cat(__VA_ARGS__))

#define CHECK_THROWS_AS(expr, type)                                                    \
  do {                                                                                 \
    bool doctest_ok_ = false;                                                          \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const type&) {                                                            \
      doctest_ok_ = true;                                                              \
    } catch (...) {                                                                    \
    }                                                                                  \
    ::doctest::detail::report(doctest_ok_, false, __FILE__, __LINE__,                  \
                              "CHECK_THROWS_AS(" #expr ", " #type ")");                \
  } while (0)

#define CHECK_NOTHROW(expr)                                                            \
  do {                                                                                 \
    bool doctest_ok_ = true;                                                           \
    std::string doctest_msg_;                                                          \
    try {                                                                              \
      static_cast<void>(expr);                                                         \
    } catch (const std::exception& e) {                                                \
      doctest_ok_ = false;                                                             \
      doctest_msg_ = e.what();                                                         \
    } catch (...) {                                                                    \
      doctest_ok_ = false;                                                             \
    }                                                                                  \
    ::doctest::detail::report(doctest_ok_, false, __FILE__, __LINE__,                  \
                              "CHECK_NOTHROW(" #expr ")", doctest_msg_);               \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
  int failed_cases = 0;
  for (const auto& c : ::doctest::detail::registry()) {
    const int before = ::doctest::detail::failures();
    try {
      c.fn();
    } catch (const ::doctest::detail::RequireAbort&) {
    } catch (const std::exception& e) {
      ++::doctest::detail::failures();
      std::cerr << c.file << ":" << c.line << ": uncaught exception: " << e.what() << "\n";
    }
    if (::doctest::detail::failures() != before) {
      ++failed_cases;
      std::cerr << "  in TEST_CASE: " << c.name << "\n";
    }
  }
  std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d | %d failed\n",
              ::doctest::detail::registry().size(),
              ::doctest::detail::registry().size() - static_cast<std::size_t>(failed_cases),
              failed_cases, ::doctest::detail::checks(), ::doctest::detail::failures());
  return failed_cases == 0 ? 0 : 1;
}
#endif
