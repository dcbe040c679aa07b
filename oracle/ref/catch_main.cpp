// TEST INFRASTRUCTURE ONLY — runner for the reference's own unit tests compiled
// against the catch2 stand-in (include/catch2/catch_amalgamated.hpp). Usage:
// mvsk_ref_tests [substring-filter]. Exit code = number of failed test cases.
#include <catch2/catch_amalgamated.hpp>

#include <cstdio>
#include <cstring>
#include <exception>

int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (const auto& tc : catchshim::registry()) {
        if (filter && tc.name.find(filter) == std::string::npos && tc.tags.find(filter) == std::string::npos)
            continue;
        ++cases;
        const int before = catchshim::state().failures;
        try {
            tc.fn();
        } catch (const catchshim::RequireAbort&) {
        } catch (const std::exception& e) {
            ++catchshim::state().failures;
            std::fprintf(stderr, "test case \"%s\" threw: %s\n", tc.name.c_str(), e.what());
        } catch (...) {
            ++catchshim::state().failures;
            std::fprintf(stderr, "test case \"%s\" threw a non-std exception\n", tc.name.c_str());
        }
        catchshim::state().info.clear();
        const bool ok = catchshim::state().failures == before;
        if (!ok) ++failed_cases;
        std::printf("%s  %s %s\n", ok ? "PASS" : "FAIL", tc.name.c_str(), tc.tags.c_str());
    }
    std::printf("test cases: %d | %d passed | %d failed; assertions: %d | %d failed\n", cases,
                cases - failed_cases, failed_cases, catchshim::state().assertions, catchshim::state().failures);
    return failed_cases;
}
