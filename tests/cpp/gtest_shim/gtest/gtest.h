// gtest.h — a minimal GoogleTest-compatible shim (GoogleTest is not in this image), enough to compile
// the reference's own test files (proj/tests/*.cpp) unmodified against the drop-in headers and run
// them on the B200: TEST / TEST_F, ::testing::Test, ::testing::TempDir, the EXPECT_* / ASSERT_*
// comparisons those files use, streamed failure messages, and a main() that runs every test and
// prints one "[PASS] / [FAIL] Suite.Name" line per test (tests/test_dropin_cpp.py parses them).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

class Test {
 public:
  virtual ~Test() = default;
  virtual void SetUp() {}
  virtual void TearDown() {}
  virtual void TestBody() = 0;
  static bool HasFailure();
};

inline std::string TempDir() { return "/tmp/"; }

namespace internal {

struct Registry {
  struct Entry {
    std::string name;
    std::function<Test*()> make;
  };
  std::vector<Entry> tests;
  int failures_in_current = 0;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

}  // namespace internal

inline bool Test::HasFailure() { return internal::Registry::get().failures_in_current != 0; }

namespace internal {

inline bool register_test(const char* suite, const char* name, std::function<Test*()> make) {
  Registry::get().tests.push_back({std::string(suite) + "." + name, std::move(make)});
  return true;
}

template <typename T>
std::string show(const T& v) {
  if constexpr (requires(std::ostream& os, const T& x) { os << x; }) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  } else {
    return "<value>";
  }
}

struct Message {
  std::ostringstream os;
  template <typename T>
  Message& operator<<(const T& v) {
    os << v;
    return *this;
  }
};

// `return Failure(...) = Message() << ...;` — operator= reports (ASSERT_*: the test returns)
struct Failure {
  const char* file;
  int line;
  std::string what;
  void operator=(const Message& m) const {
    ++Registry::get().failures_in_current;
    std::fprintf(stderr, "  %s:%d: Failure\n    %s\n", file, line, what.c_str());
    const std::string extra = m.os.str();
    if (!extra.empty()) std::fprintf(stderr, "    %s\n", extra.c_str());
  }
};

template <typename A, typename B>
std::string cmp_text(const char* op, const char* ea, const char* eb, const A& a, const B& b) {
  return std::string("Expected: (") + ea + ") " + op + " (" + eb + "), actual: " + show(a) + " vs " + show(b);
}

inline bool almost_equal_ulps(double a, double b) {  // gtest's DoubleNear of 4 ULPs
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  auto key = [](double x) {
    std::int64_t i;
    std::memcpy(&i, &x, 8);
    return i < 0 ? static_cast<std::uint64_t>(~i) + 1 : static_cast<std::uint64_t>(i) | (1ull << 63);
  };
  const std::uint64_t ka = key(a), kb = key(b);
  return (ka > kb ? ka - kb : kb - ka) <= 4;
}

}  // namespace internal
}  // namespace testing

#define GTEST_SHIM_BLOCKER_ \
  switch (0)                \
  case 0:                   \
  default:

#define GTEST_SHIM_CHECK_(ok, text, on_fail) \
  GTEST_SHIM_BLOCKER_                        \
  if (ok) {                                  \
  } else                                     \
    on_fail ::testing::internal::Failure{__FILE__, __LINE__, text} = ::testing::internal::Message()

#define GTEST_SHIM_NONFATAL_
#define GTEST_SHIM_FATAL_ return

#define GTEST_SHIM_CMP_(op, a, b, kind)                                                         \
  GTEST_SHIM_BLOCKER_                                                                          \
  if (const auto& gtest_a_ = (a); true)                                                        \
    if (const auto& gtest_b_ = (b); gtest_a_ op gtest_b_) {                                    \
    } else                                                                                     \
      kind ::testing::internal::Failure{__FILE__, __LINE__,                                    \
                                        ::testing::internal::cmp_text(#op, #a, #b, gtest_a_, gtest_b_)} = \
          ::testing::internal::Message()

#define EXPECT_EQ(a, b) GTEST_SHIM_CMP_(==, a, b, GTEST_SHIM_NONFATAL_)
#define EXPECT_NE(a, b) GTEST_SHIM_CMP_(!=, a, b, GTEST_SHIM_NONFATAL_)
#define EXPECT_LE(a, b) GTEST_SHIM_CMP_(<=, a, b, GTEST_SHIM_NONFATAL_)
#define EXPECT_LT(a, b) GTEST_SHIM_CMP_(<, a, b, GTEST_SHIM_NONFATAL_)
#define EXPECT_GE(a, b) GTEST_SHIM_CMP_(>=, a, b, GTEST_SHIM_NONFATAL_)
#define EXPECT_GT(a, b) GTEST_SHIM_CMP_(>, a, b, GTEST_SHIM_NONFATAL_)
#define ASSERT_EQ(a, b) GTEST_SHIM_CMP_(==, a, b, GTEST_SHIM_FATAL_)
#define ASSERT_NE(a, b) GTEST_SHIM_CMP_(!=, a, b, GTEST_SHIM_FATAL_)
#define ASSERT_LE(a, b) GTEST_SHIM_CMP_(<=, a, b, GTEST_SHIM_FATAL_)
#define ASSERT_LT(a, b) GTEST_SHIM_CMP_(<, a, b, GTEST_SHIM_FATAL_)
#define ASSERT_GE(a, b) GTEST_SHIM_CMP_(>=, a, b, GTEST_SHIM_FATAL_)
#define ASSERT_GT(a, b) GTEST_SHIM_CMP_(>, a, b, GTEST_SHIM_FATAL_)
#define EXPECT_TRUE(c) GTEST_SHIM_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_SHIM_NONFATAL_)
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_SHIM_NONFATAL_)
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK_(static_cast<bool>(c), "Expected true: " #c, GTEST_SHIM_FATAL_)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK_(!static_cast<bool>(c), "Expected false: " #c, GTEST_SHIM_FATAL_)
#define ADD_FAILURE() ::testing::internal::Failure{__FILE__, __LINE__, "Failed"} = ::testing::internal::Message()
#define EXPECT_DOUBLE_EQ(a, b)                                                                      \
  GTEST_SHIM_CHECK_(::testing::internal::almost_equal_ulps(static_cast<double>(a), static_cast<double>(b)), \
                    ::testing::internal::cmp_text("~=", #a, #b, static_cast<double>(a), static_cast<double>(b)), \
                    GTEST_SHIM_NONFATAL_)
#define EXPECT_NEAR(a, b, tol)                                                                     \
  GTEST_SHIM_CHECK_(std::abs(static_cast<double>(a) - static_cast<double>(b)) <= static_cast<double>(tol), \
                    ::testing::internal::cmp_text("near", #a, #b, static_cast<double>(a), static_cast<double>(b)), \
                    GTEST_SHIM_NONFATAL_)
#define EXPECT_STREQ(a, b) \
  GTEST_SHIM_CHECK_(std::strcmp((a), (b)) == 0, "Expected equal strings: " #a ", " #b, GTEST_SHIM_NONFATAL_)

#define GTEST_SHIM_THROW_(stmt, exc, kind)                         \
  GTEST_SHIM_BLOCKER_                                              \
  if (int gtest_caught_ = [&] {                                    \
        try {                                                      \
          stmt;                                                    \
        } catch (const exc&) {                                     \
          return 1;                                                \
        } catch (...) {                                            \
          return 2;                                                \
        }                                                          \
        return 0;                                                  \
      }();                                                         \
      gtest_caught_ == 1) {                                        \
  } else                                                           \
    kind ::testing::internal::Failure{__FILE__, __LINE__,                                    \
                                      std::string("Expected: " #stmt " throws " #exc ", ") + \
                                          (gtest_caught_ == 0 ? "nothing thrown" : "another exception")} = \
        ::testing::internal::Message()
#define EXPECT_THROW(stmt, exc) GTEST_SHIM_THROW_(stmt, exc, GTEST_SHIM_NONFATAL_)
#define ASSERT_THROW(stmt, exc) GTEST_SHIM_THROW_(stmt, exc, GTEST_SHIM_FATAL_)

#define GTEST_SHIM_CLASS_(suite, name) suite##_##name##_Test
#define TEST_F(fixture, name)                                                                    \
  class GTEST_SHIM_CLASS_(fixture, name) : public fixture {                                      \
   public:                                                                                       \
    void TestBody() override;                                                                    \
  };                                                                                             \
  [[maybe_unused]] static const bool gtest_reg_##fixture##_##name = ::testing::internal::register_test( \
      #fixture, #name, [] { return static_cast<::testing::Test*>(new GTEST_SHIM_CLASS_(fixture, name)); }); \
  void GTEST_SHIM_CLASS_(fixture, name)::TestBody()
#define TEST(suite, name) TEST_F_BASE_(suite, name)
#define TEST_F_BASE_(suite, name)                                                                \
  class GTEST_SHIM_CLASS_(suite, name) : public ::testing::Test {                                \
   public:                                                                                       \
    void TestBody() override;                                                                    \
  };                                                                                             \
  [[maybe_unused]] static const bool gtest_reg_##suite##_##name = ::testing::internal::register_test( \
      #suite, #name, [] { return static_cast<::testing::Test*>(new GTEST_SHIM_CLASS_(suite, name)); }); \
  void GTEST_SHIM_CLASS_(suite, name)::TestBody()

// main(): every registered test, in registration order
int main(int argc, char** argv) {
  const char* only = argc > 1 ? argv[1] : nullptr;  // optional substring filter
  auto& reg = ::testing::internal::Registry::get();
  int failed = 0, ran = 0;
  for (auto& t : reg.tests) {
    if (only && t.name.find(only) == std::string::npos) continue;
    reg.failures_in_current = 0;
    ++ran;
    try {
      ::testing::Test* obj = t.make();
      obj->SetUp();
      obj->TestBody();
      obj->TearDown();
      delete obj;
    } catch (const std::exception& e) {
      ++reg.failures_in_current;
      std::fprintf(stderr, "  uncaught exception: %s\n", e.what());
    } catch (...) {
      ++reg.failures_in_current;
      std::fprintf(stderr, "  uncaught non-std exception\n");
    }
    failed += reg.failures_in_current != 0;
    std::printf("[%s] %s\n", reg.failures_in_current ? "FAIL" : "PASS", t.name.c_str());
    std::fflush(stdout);
  }
  std::printf("%d tests, %d failed\n", ran, failed);
  return failed == 0 ? 0 : 1;
}
