// TEST INFRASTRUCTURE (oracle build only) -- never linked into the product.
//
// Catch2-subset shim, written from scratch, so that the reference's own
// hot-path test files (/root/reference/proj/tests/test_{blockla,smoothers,
// multigrid,krylov}.cpp) compile UNMODIFIED against the oracle build and pin
// it.  Supported: TEST_CASE, SECTION (nested, one leaf per run), CHECK /
// REQUIRE (+ _FALSE, _THROWS, _THROWS_AS, _NOTHROW), CAPTURE, INFO, FAIL,
// and Catch::Approx with margin/epsilon.  Link oracle/shim/catch2/main.cpp.
#ifndef ORACLE_SHIM_CATCH2
#define ORACLE_SHIM_CATCH2

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestAbort {};

struct TestCaseInfo {
    std::string name;
    std::function<void()> fn;
    const char* file;
    int line;
};

inline std::vector<TestCaseInfo>& registry() {
    static std::vector<TestCaseInfo> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, std::function<void()> fn, const char* file, int line) {
        registry().push_back({name, std::move(fn), file, line});
    }
};

struct RunState {
    std::string test;
    long assertions = 0, failures = 0;
    // section tracking
    std::set<std::string> done;
    std::vector<std::string> stack;
    std::vector<bool> entered_at_depth;
    bool more = false;
    std::vector<bool> child_unfinished;
};

inline RunState& state() {
    static RunState s;
    return s;
}

inline void report_failure(const char* file, int line, const std::string& what) {
    RunState& s = state();
    ++s.failures;
    std::string where;
    for (const auto& n : s.stack) where += " / " + n;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\"%s\n  %s\n", file, line, s.test.c_str(),
                 where.c_str(), what.c_str());
}

class SectionGuard {
  public:
    explicit SectionGuard(const char* name) {
        RunState& s = state();
        std::string path;
        for (const auto& n : s.stack) path += n + "\x1f";
        path += name;
        const size_t depth = s.stack.size();
        if (s.entered_at_depth.size() <= depth) s.entered_at_depth.resize(depth + 1, false);
        if (s.done.count(path)) return;
        if (s.entered_at_depth[depth]) {  // a sibling already ran in this pass
            s.more = true;
            if (!s.child_unfinished.empty()) s.child_unfinished.back() = true;
            return;
        }
        s.entered_at_depth[depth] = true;
        active_ = true;
        path_ = path;
        s.stack.push_back(name);
        s.child_unfinished.push_back(false);
    }
    ~SectionGuard() {
        if (!active_) return;
        RunState& s = state();
        const bool unfinished = s.child_unfinished.back();
        s.child_unfinished.pop_back();
        const size_t depth = s.stack.size();
        if (s.entered_at_depth.size() > depth) s.entered_at_depth.resize(depth);
        s.stack.pop_back();
        if (!unfinished)
            s.done.insert(path_);
        else if (!s.child_unfinished.empty())
            s.child_unfinished.back() = true;
    }
    explicit operator bool() const { return active_; }

  private:
    bool active_ = false;
    std::string path_;
};

class Approx {
  public:
    explicit Approx(double v)
        : value_(v), epsilon_(std::numeric_limits<float>::epsilon() * 100), margin_(0.0) {}
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    bool matches(double other) const {
        const double d = std::fabs(other - value_);
        if (d <= margin_) return true;
        const double scale = std::isinf(value_) ? 0.0 : std::fabs(value_);
        return d <= epsilon_ * scale;
    }
    double value() const { return value_; }

  private:
    double value_, epsilon_, margin_;
};
inline bool operator==(double a, const Approx& b) { return b.matches(a); }
inline bool operator==(const Approx& a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx& b) { return !b.matches(a); }
inline bool operator<=(double a, const Approx& b) { return a < b.value() || b.matches(a); }
inline bool operator>=(double a, const Approx& b) { return a > b.value() || b.matches(a); }

inline int run_all() {
    int failed_cases = 0;
    long total_assert = 0, total_fail = 0;
    for (const auto& tc : registry()) {
        RunState& s = state();
        s = RunState{};
        s.test = tc.name;
        int passes = 0;
        do {
            s.more = false;
            s.stack.clear();
            s.entered_at_depth.assign(1, false);
            s.child_unfinished.clear();
            try {
                tc.fn();
            } catch (const TestAbort&) {
            } catch (const std::exception& e) {
                report_failure(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
            }
            if (++passes > 10000) break;
        } while (s.more);
        total_assert += s.assertions;
        total_fail += s.failures;
        if (s.failures) ++failed_cases;
        std::printf("[%s] %s (%ld assertions, %ld failed)\n", s.failures ? "FAIL" : " ok ",
                    tc.name.c_str(), s.assertions, s.failures);
    }
    std::printf("test cases: %zu | %d failed; assertions: %ld | %ld failed\n", registry().size(),
                failed_cases, total_assert, total_fail);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TC(fn, ...)                                                              \
    static void fn();                                                                       \
    static const Catch::Registrar CATCH_SHIM_CAT(fn, _reg){__VA_ARGS__, fn, __FILE__, __LINE__}; \
    static void fn()
#define TEST_CASE(...) CATCH_SHIM_TC(CATCH_SHIM_CAT(catch_shim_tc_, __LINE__), CATCH_SHIM_FIRST(__VA_ARGS__, ""))
#define CATCH_SHIM_FIRST(a, ...) a
#define SECTION(name) if (Catch::SectionGuard CATCH_SHIM_CAT(catch_sec_, __LINE__){name}; CATCH_SHIM_CAT(catch_sec_, __LINE__))

#define CATCH_SHIM_ASSERT(cond, text, fatal)                                     \
    do {                                                                         \
        ++Catch::state().assertions;                                             \
        bool catch_ok_ = false;                                                  \
        try {                                                                    \
            catch_ok_ = static_cast<bool>(cond);                                 \
        } catch (const std::exception& catch_e_) {                               \
            Catch::report_failure(__FILE__, __LINE__,                            \
                                  std::string(text) + " threw " + catch_e_.what()); \
            if (fatal) throw Catch::TestAbort{};                                 \
            break;                                                               \
        }                                                                        \
        if (!catch_ok_) {                                                        \
            Catch::report_failure(__FILE__, __LINE__, text);                     \
            if (fatal) throw Catch::TestAbort{};                                 \
        }                                                                        \
    } while (0)

#define CHECK(...) CATCH_SHIM_ASSERT((__VA_ARGS__), "CHECK(" #__VA_ARGS__ ")", false)
#define REQUIRE(...) CATCH_SHIM_ASSERT((__VA_ARGS__), "REQUIRE(" #__VA_ARGS__ ")", true)
#define CHECK_FALSE(...) CATCH_SHIM_ASSERT(!(__VA_ARGS__), "CHECK_FALSE(" #__VA_ARGS__ ")", false)
#define REQUIRE_FALSE(...) CATCH_SHIM_ASSERT(!(__VA_ARGS__), "REQUIRE_FALSE(" #__VA_ARGS__ ")", true)

#define CATCH_SHIM_THROWS(expr, text, fatal, pred)                               \
    do {                                                                         \
        ++Catch::state().assertions;                                             \
        bool catch_ok_ = false;                                                  \
        try {                                                                    \
            static_cast<void>(expr);                                             \
        } catch (...) {                                                          \
            catch_ok_ = pred;                                                    \
        }                                                                        \
        if (!catch_ok_) {                                                        \
            Catch::report_failure(__FILE__, __LINE__, text);                     \
            if (fatal) throw Catch::TestAbort{};                                 \
        }                                                                        \
    } while (0)

namespace Catch {
template <class E>
bool current_is() {
    try {
        throw;
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
}
}  // namespace Catch

#define CHECK_THROWS(...) CATCH_SHIM_THROWS((__VA_ARGS__), "CHECK_THROWS(" #__VA_ARGS__ ")", false, true)
#define REQUIRE_THROWS(...) CATCH_SHIM_THROWS((__VA_ARGS__), "REQUIRE_THROWS(" #__VA_ARGS__ ")", true, true)
#define CHECK_THROWS_AS(expr, E) \
    CATCH_SHIM_THROWS(expr, "CHECK_THROWS_AS(" #expr ", " #E ")", false, Catch::current_is<E>())
#define REQUIRE_THROWS_AS(expr, E) \
    CATCH_SHIM_THROWS(expr, "REQUIRE_THROWS_AS(" #expr ", " #E ")", true, Catch::current_is<E>())

#define CATCH_SHIM_NOTHROW(expr, text, fatal)                                    \
    do {                                                                         \
        ++Catch::state().assertions;                                             \
        try {                                                                    \
            static_cast<void>(expr);                                             \
        } catch (...) {                                                          \
            Catch::report_failure(__FILE__, __LINE__, text);                     \
            if (fatal) throw Catch::TestAbort{};                                 \
        }                                                                        \
    } while (0)
#define CHECK_NOTHROW(...) CATCH_SHIM_NOTHROW((__VA_ARGS__), "CHECK_NOTHROW(" #__VA_ARGS__ ")", false)
#define REQUIRE_NOTHROW(...) CATCH_SHIM_NOTHROW((__VA_ARGS__), "REQUIRE_NOTHROW(" #__VA_ARGS__ ")", true)

#define CAPTURE(...) static_cast<void>(0)
#define INFO(...) static_cast<void>(0)
#define FAIL(msg)                                                                \
    do {                                                                         \
        std::ostringstream catch_os_;                                            \
        catch_os_ << msg;                                                        \
        Catch::report_failure(__FILE__, __LINE__, "FAIL: " + catch_os_.str());   \
        throw Catch::TestAbort{};                                                \
    } while (0)

#endif
