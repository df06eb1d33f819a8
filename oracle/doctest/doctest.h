// Minimal doctest-compatible test harness (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) are written
// against doctest, which the reference does not vendor.  This header
// implements the subset those tests use -- TEST_CASE, nested SUBCASE (each
// leaf path runs in its own pass of the test case, as doctest does), CHECK,
// REQUIRE, CHECK_THROWS, CHECK_THROWS_AS, FAIL, doctest::Approx -- so the
// reference tests compile unchanged, once against the reference library
// (oracle/_ref) and once against the B200 drop-in (paper_2603_08453_b200/cpp).
// It is not part of the product.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <sstream>
#include <set>
#include <string>
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
    // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    friend bool operator==(double lhs, const Approx& r) {
        return std::fabs(lhs - r.value_) < r.eps_ * (r.scale_ + std::fmax(std::fabs(lhs), std::fabs(r.value_)));
    }
    friend bool operator==(const Approx& r, double rhs) { return rhs == r; }
    friend bool operator!=(double lhs, const Approx& r) { return !(lhs == r); }
    friend bool operator!=(const Approx& r, double rhs) { return !(rhs == r); }

private:
    double value_;
    double eps_ = 1.1920929e-05;  // FLT_EPSILON * 100, doctest's default
    double scale_ = 1.0;
};

namespace detail {

struct RequireFailure {};

using Path = std::vector<std::string>;

struct Node {
    std::vector<std::string> children;  // in encounter order
    bool complete = false;
};

// Subcase traversal (depth first): in every pass of a test case, at each level
// the first subcase that is not complete is entered and its later siblings are
// skipped; a subcase is complete once it ran with all its known children
// complete.  The test case reruns until all top-level subcases are complete.
struct Registry {
    struct Case {
        const char* name;
        void (*fn)();
    };
    std::vector<Case> cases;
    std::map<Path, Node> nodes;
    Path stack;
    std::set<Path> entered_under;  // parents that had a child entered in this pass
    long checks = 0, failures = 0;
    bool case_failed = false;
    const char* case_name = "";

    static Registry& get() {
        static Registry r;
        return r;
    }
    bool children_complete(const Path& p) {
        const Node& n = nodes[p];
        for (const auto& c : n.children) {
            Path cp = p;
            cp.push_back(c);
            if (!nodes[cp].complete) return false;
        }
        return true;
    }
};

inline int add_case(const char* name, void (*fn)()) {
    Registry::get().cases.push_back({name, fn});
    return 0;
}

class Subcase {
public:
    explicit Subcase(const char* name) {
        Registry& R = Registry::get();
        Node& parent = R.nodes[R.stack];
        bool known = false;
        for (const auto& c : parent.children) known |= c == name;
        if (!known) parent.children.push_back(name);
        Path path = R.stack;
        path.push_back(name);
        if (!R.entered_under.count(R.stack) && !R.nodes[path].complete) {
            R.entered_under.insert(R.stack);
            R.stack.push_back(name);
            entered_ = true;
        }
    }
    ~Subcase() {
        if (!entered_) return;
        Registry& R = Registry::get();
        if (R.children_complete(R.stack)) R.nodes[R.stack].complete = true;
        R.stack.pop_back();
    }
    explicit operator bool() const { return entered_; }

private:
    bool entered_ = false;
};

inline void report(bool ok, const char* file, int line, const char* expr, const char* kind, bool require) {
    Registry& R = Registry::get();
    ++R.checks;
    if (ok) return;
    ++R.failures;
    R.case_failed = true;
    std::string sub;
    for (const auto& s : R.stack) sub += " / " + s;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in \"%s\"%s\n", file, line, kind, expr, R.case_name, sub.c_str());
    if (require) throw RequireFailure{};
}

inline int run_all() {
    Registry& R = Registry::get();
    int failed_cases = 0;
    for (const auto& c : R.cases) {
        R.nodes.clear();
        R.case_name = c.name;
        R.case_failed = false;
        for (int pass = 0; pass < 1000000; ++pass) {
            R.stack.clear();
            R.entered_under.clear();
            try {
                c.fn();
            } catch (const RequireFailure&) {
            } catch (const std::exception& e) {
                std::fprintf(stderr, "test case \"%s\": unexpected exception: %s\n", c.name, e.what());
                ++R.failures;
                R.case_failed = true;
            } catch (...) {
                std::fprintf(stderr, "test case \"%s\": unexpected exception\n", c.name);
                ++R.failures;
                R.case_failed = true;
            }
            if (R.children_complete(Path{})) break;
        }
        if (R.case_failed) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                R.cases.size(), R.cases.size() - (size_t)failed_cases, failed_cases, R.checks, R.failures);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                 \
    static void DOCTEST_ANON(doctest_case_fn_)();                                       \
    static const int DOCTEST_ANON(doctest_case_reg_) =                                  \
        doctest::detail::add_case(name, &DOCTEST_ANON(doctest_case_fn_));               \
    static void DOCTEST_ANON(doctest_case_fn_)()

#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_ANON(doctest_sub_){name})

#define DOCTEST_ASSERT_(expr, kind, req)                                                \
    do {                                                                                \
        bool doctest_ok_ = false;                                                       \
        try {                                                                           \
            doctest_ok_ = static_cast<bool>(expr);                                      \
        } catch (const doctest::detail::RequireFailure&) {                              \
            throw;                                                                      \
        } catch (...) {                                                                 \
            doctest_ok_ = false;                                                        \
        }                                                                               \
        doctest::detail::report(doctest_ok_, __FILE__, __LINE__, #expr, kind, req);     \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_((__VA_ARGS__), "CHECK", false)
#define REQUIRE(...) DOCTEST_ASSERT_((__VA_ARGS__), "REQUIRE", true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_(!(__VA_ARGS__), "CHECK_FALSE", false)

#define CHECK_THROWS(...)                                                               \
    do {                                                                                \
        bool doctest_thrown_ = false;                                                   \
        try {                                                                           \
            (void)(__VA_ARGS__);                                                        \
        } catch (...) {                                                                 \
            doctest_thrown_ = true;                                                     \
        }                                                                               \
        doctest::detail::report(doctest_thrown_, __FILE__, __LINE__, #__VA_ARGS__, "CHECK_THROWS", false); \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                      \
    do {                                                                                \
        bool doctest_thrown_ = false;                                                   \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                  \
            doctest_thrown_ = true;                                                     \
        } catch (...) {                                                                 \
        }                                                                               \
        doctest::detail::report(doctest_thrown_, __FILE__, __LINE__, #expr, "CHECK_THROWS_AS", false); \
    } while (0)

#define FAIL(msg) doctest::detail::report(false, __FILE__, __LINE__, msg, "FAIL", true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
