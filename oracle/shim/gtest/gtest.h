// Minimal GoogleTest-API stand-in so the reference suites
// (/root/reference/proj/tests/test_*.cpp) build and run verbatim as the
// parity oracle's self-check. TEST INFRASTRUCTURE ONLY.
// Supports TEST, EXPECT/ASSERT_{TRUE,FALSE,EQ,NE,LT,LE,GT,GE,NEAR,DOUBLE_EQ},
// EXPECT_THROW/NO_THROW, SUCCEED, FAIL, and `<<` context on assertions.
#ifndef ORACLE_SHIM_GTEST_H
#define ORACLE_SHIM_GTEST_H

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace shimtest {

struct Case {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, void (*fn)()) {
    registry().push_back({s, n, fn});
  }
};

// Collects `<<` context and reports on destruction when the check failed.
struct Reporter {
  bool failed;
  bool fatal;
  std::ostringstream os;
  Reporter(bool ok, bool isFatal, const char* file, int line, const char* what)
      : failed(!ok), fatal(isFatal) {
    if (failed) os << file << ":" << line << ": failure: " << what << " ";
  }
  ~Reporter() {
    if (failed) {
      ++failures();
      std::cerr << os.str() << std::endl;
    }
  }
  template <typename T>
  Reporter& operator<<(const T& v) {
    if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
      if (failed) os << v;
    } else {
      if (failed) os << "<value>";
    }
    return *this;
  }
};

struct FatalFailure {};

inline bool ulpEq(double a, double b) {
  if (a == b) return true;
  if (std::isnan(a) || std::isnan(b)) return false;
  std::int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  if (ia < 0) ia = INT64_MIN - ia;
  if (ib < 0) ib = INT64_MIN - ib;
  const std::int64_t d = ia > ib ? ia - ib : ib - ia;
  return d <= 4;
}

}  // namespace shimtest

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)

#define TEST(suite, name)                                              \
  static void SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name)))(); \
  static ::shimtest::Registrar SHIM_CAT(shim_reg_,                     \
                                        SHIM_CAT(suite, SHIM_CAT(_, name)))( \
      #suite, #name, &SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name)))); \
  static void SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name)))()

#define SHIM_CHECK(ok, fatal, what)                                          \
  for (bool shim_once = true; shim_once; shim_once = false)                  \
    for (bool shim_ok = (ok); shim_once;                                     \
         shim_once = false,                                                  \
              (!shim_ok && (fatal)) ? throw ::shimtest::FatalFailure{} : (void)0) \
  ::shimtest::Reporter(shim_ok, fatal, __FILE__, __LINE__, what)

#define EXPECT_TRUE(c) SHIM_CHECK(static_cast<bool>(c), false, #c)
#define EXPECT_FALSE(c) SHIM_CHECK(!static_cast<bool>(c), false, "!(" #c ")")
#define ASSERT_TRUE(c) SHIM_CHECK(static_cast<bool>(c), true, #c)
#define ASSERT_FALSE(c) SHIM_CHECK(!static_cast<bool>(c), true, "!(" #c ")")
#define SHIM_CMP(a, op, b, fatal) \
  SHIM_CHECK(((a)op(b)), fatal, #a " " #op " " #b) << "(" << (a) << " vs " << (b) << ") "
#define EXPECT_EQ(a, b) SHIM_CMP(a, ==, b, false)
#define EXPECT_NE(a, b) SHIM_CMP(a, !=, b, false)
#define EXPECT_LT(a, b) SHIM_CMP(a, <, b, false)
#define EXPECT_LE(a, b) SHIM_CMP(a, <=, b, false)
#define EXPECT_GT(a, b) SHIM_CMP(a, >, b, false)
#define EXPECT_GE(a, b) SHIM_CMP(a, >=, b, false)
#define ASSERT_EQ(a, b) SHIM_CMP(a, ==, b, true)
#define ASSERT_NE(a, b) SHIM_CMP(a, !=, b, true)
#define ASSERT_LT(a, b) SHIM_CMP(a, <, b, true)
#define ASSERT_LE(a, b) SHIM_CMP(a, <=, b, true)
#define ASSERT_GT(a, b) SHIM_CMP(a, >, b, true)
#define ASSERT_GE(a, b) SHIM_CMP(a, >=, b, true)
#define EXPECT_NEAR(a, b, tol)                                              \
  SHIM_CHECK(std::fabs(static_cast<double>(a) - static_cast<double>(b)) <= \
                 static_cast<double>(tol),                                  \
             false, "NEAR(" #a ", " #b ", " #tol ")")                       \
      << "(" << static_cast<double>(a) << " vs " << static_cast<double>(b) << ") "
#define EXPECT_DOUBLE_EQ(a, b)                                      \
  SHIM_CHECK(::shimtest::ulpEq(static_cast<double>(a), static_cast<double>(b)), \
             false, "DOUBLE_EQ(" #a ", " #b ")")                    \
      << "(" << static_cast<double>(a) << " vs " << static_cast<double>(b) << ") "
#define SHIM_THROWS(stmt, exc, fatal)                  \
  SHIM_CHECK(([&]() -> bool {                          \
               try {                                   \
                 stmt;                                 \
               } catch (const exc&) {                  \
                 return true;                          \
               } catch (...) {                         \
                 return false;                         \
               }                                       \
               return false;                           \
             }()),                                     \
             fatal, "THROW(" #stmt ", " #exc ")")
#define EXPECT_THROW(stmt, exc) SHIM_THROWS(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) SHIM_THROWS(stmt, exc, true)
#define EXPECT_NO_THROW(stmt)                                    \
  SHIM_CHECK(([&]() -> bool {                                    \
               try {                                             \
                 stmt;                                           \
               } catch (...) {                                   \
                 return false;                                   \
               }                                                 \
               return true;                                      \
             }()),                                               \
             false, "NO_THROW(" #stmt ")")
#define SUCCEED() ::shimtest::Reporter(true, false, __FILE__, __LINE__, "")
#define FAIL() SHIM_CHECK(false, true, "FAIL()")

#ifndef SHIM_NO_MAIN
int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0, failedCases = 0;
  for (const auto& c : ::shimtest::registry()) {
    const std::string full = std::string(c.suite) + "." + c.name;
    if (filter && full.find(filter) == std::string::npos) continue;
    const int before = ::shimtest::failures();
    try {
      c.fn();
    } catch (const ::shimtest::FatalFailure&) {
    } catch (const std::exception& e) {
      ++::shimtest::failures();
      std::cerr << full << ": uncaught exception: " << e.what() << std::endl;
    }
    const bool ok = ::shimtest::failures() == before;
    std::printf("[%s] %s\n", ok ? "  OK  " : " FAIL ", full.c_str());
    ++ran;
    if (!ok) ++failedCases;
  }
  std::printf("%d/%d passed\n", ran - failedCases, ran);
  return failedCases == 0 ? 0 : 1;
}
#endif

#endif  // ORACLE_SHIM_GTEST_H
