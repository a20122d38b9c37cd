// TEST INFRASTRUCTURE: runner for oracle/minitest/gtest/gtest.h.
// Prints one line per case and a gtest-like summary; exit 0 iff all passed.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "gtest/gtest.h"

namespace {

bool glob_match(const std::string& pat, const std::string& s) {
    if (!pat.empty() && pat.back() == '*') return s.compare(0, pat.size() - 1, pat, 0, pat.size() - 1) == 0;
    return pat == s;
}

bool selected(const std::string& filter, const std::string& full) {
    if (filter.empty()) return true;
    std::string pos = filter, neg;
    if (const auto d = filter.find('-'); d != std::string::npos) {
        pos = filter.substr(0, d);
        neg = filter.substr(d + 1);
    }
    auto any = [&](const std::string& list) {
        std::size_t b = 0;
        while (b <= list.size()) {
            std::size_t e = list.find(':', b);
            if (e == std::string::npos) e = list.size();
            if (e > b && glob_match(list.substr(b, e - b), full)) return true;
            b = e + 1;
        }
        return false;
    };
    return (pos.empty() || any(pos)) && !(neg.size() && any(neg));
}

}  // namespace

int main(int argc, char** argv) {
    std::string filter;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
        else if (std::strcmp(argv[i], "--list") == 0) list = true;
    }
    int ran = 0, failed = 0;
    std::vector<std::string> failed_names;
    for (const auto& c : minitest::registry()) {
        const std::string full = c.suite + "." + c.name;
        if (!selected(filter, full)) continue;
        if (list) {
            std::printf("%s\n", full.c_str());
            continue;
        }
        minitest::failures_in_case() = 0;
        const auto t0 = std::chrono::steady_clock::now();
        try {
            c.body();
        } catch (const std::exception& e) {
            ++minitest::failures_in_case();
            std::fprintf(stderr, "%s: uncaught exception: %s\n", full.c_str(), e.what());
        } catch (...) {
            ++minitest::failures_in_case();
            std::fprintf(stderr, "%s: uncaught non-std exception\n", full.c_str());
        }
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        const bool ok = minitest::failures_in_case() == 0;
        std::printf("[ %s ] %s (%.0f ms)\n", ok ? "     OK" : "FAILED ", full.c_str(), ms);
        std::fflush(stdout);
        ++ran;
        if (!ok) {
            ++failed;
            failed_names.push_back(full);
        }
    }
    if (list) return 0;
    std::printf("[==========] %d tests ran, %d passed, %d failed\n", ran, ran - failed, failed);
    for (const auto& n : failed_names) std::printf("[  FAILED  ] %s\n", n.c_str());
    return failed ? 1 : 0;
}
