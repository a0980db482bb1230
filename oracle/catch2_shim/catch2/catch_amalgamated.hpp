// Minimal Catch2-API shim — TEST INFRASTRUCTURE ONLY.
//
// The reference's unit tests (`/root/reference/proj/tests/*.cpp`) include
// <catch2/catch_amalgamated.hpp>, which is not installed in this image. This header
// provides just the subset they use (TEST_CASE, REQUIRE, CHECK, REQUIRE_THAT,
// CHECK_THAT, CHECK_THROWS_AS, Matchers::WithinAbs/WithinRel) so the reference's own
// test files run unmodified against the oracle build. Define USTFWI_CATCH_MAIN in
// exactly one translation unit to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
    std::string name;
    std::function<void()> fn;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailure {
    std::string what;
};

inline int& check_failures() {
    static int n = 0;
    return n;
}

inline void report(const char* file, int line, const std::string& what, bool fatal) {
    std::fprintf(stderr, "  %s:%d: %s %s\n", file, line, fatal ? "REQUIRE failed:" : "CHECK failed:",
                 what.c_str());
    if (fatal) throw RequireFailure{what};
    ++check_failures();
}

namespace Matchers {

struct WithinAbsMatcher {
    double target, margin;
    bool match(double v) const { return std::abs(v - target) <= margin; }
    std::string describe() const {
        std::ostringstream s;
        s << "is within " << margin << " of " << target;
        return s.str();
    }
};

struct WithinRelMatcher {
    double target, eps;
    bool match(double v) const {
        return std::abs(v - target) <= eps * std::max(std::abs(v), std::abs(target));
    }
    std::string describe() const {
        std::ostringstream s;
        s << "is within relative " << eps << " of " << target;
        return s.str();
    }
};

inline WithinAbsMatcher WithinAbs(double target, double margin) { return {target, margin}; }
inline WithinRelMatcher WithinRel(double target, double eps) { return {target, eps}; }

}  // namespace Matchers

template <class M>
inline void check_that(const char* file, int line, const char* expr, double v, const M& m, bool fatal) {
    if (!m.match(v)) {
        std::ostringstream s;
        s << expr << " = " << v << " " << m.describe();
        report(file, line, s.str(), fatal);
    }
}

}  // namespace Catch

#define USTFWI_CATCH_CAT2(a, b) a##b
#define USTFWI_CATCH_CAT(a, b) USTFWI_CATCH_CAT2(a, b)
#define USTFWI_CATCH_TEST(fn, name)                                          \
    static void fn();                                                        \
    static Catch::Registrar USTFWI_CATCH_CAT(fn, _reg){name, &fn};           \
    static void fn()
#define TEST_CASE(name, ...) USTFWI_CATCH_TEST(USTFWI_CATCH_CAT(catch_test_, __COUNTER__), name)

#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        if (!(__VA_ARGS__)) Catch::report(__FILE__, __LINE__, #__VA_ARGS__, true);         \
    } while (0)
#define CHECK(...)                                                                          \
    do {                                                                                    \
        if (!(__VA_ARGS__)) Catch::report(__FILE__, __LINE__, #__VA_ARGS__, false);        \
    } while (0)
#define REQUIRE_THAT(v, m) Catch::check_that(__FILE__, __LINE__, #v, (v), (m), true)
#define CHECK_THAT(v, m) Catch::check_that(__FILE__, __LINE__, #v, (v), (m), false)
#define CHECK_THROWS_AS(expr, type)                                                          \
    do {                                                                                     \
        bool caught_ = false;                                                                \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const type&) {                                                              \
            caught_ = true;                                                                  \
        } catch (...) {                                                                      \
        }                                                                                    \
        if (!caught_) Catch::report(__FILE__, __LINE__, #expr " did not throw " #type, false); \
    } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                                        \
    do {                                                                                     \
        bool caught_ = false;                                                                \
        try {                                                                                \
            (void)(expr);                                                                    \
        } catch (const type&) {                                                              \
            caught_ = true;                                                                  \
        } catch (...) {                                                                      \
        }                                                                                    \
        if (!caught_) Catch::report(__FILE__, __LINE__, #expr " did not throw " #type, true); \
    } while (0)

#ifdef USTFWI_CATCH_MAIN
#include <chrono>
#include <cstring>
int main(int argc, char** argv) {
    int failed = 0, passed = 0;
    for (const auto& tc : Catch::registry()) {
        if (argc > 1 && std::strstr(tc.name.c_str(), argv[1]) == nullptr) continue;
        const int before = Catch::check_failures();
        const auto t0 = std::chrono::steady_clock::now();
        bool ok = true;
        try {
            tc.fn();
        } catch (const Catch::RequireFailure&) {
            ok = false;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
            ok = false;
        }
        if (Catch::check_failures() != before) ok = false;
        const double s =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::printf("%s  %-75s %8.2fs\n", ok ? "PASS" : "FAIL", tc.name.c_str(), s);
        (ok ? passed : failed)++;
    }
    std::printf("%d passed, %d failed\n", passed, failed);
    return failed == 0 ? 0 : 1;
}
#endif
