// Times the first-use costs of the GPU scan in a fresh process (CUDA init,
// scanner creation, first/second scan of a tiny text).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "acg.h"

static double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

int main() {
    const char* words[] = {"HIS", "SHE", "HERS"};
    std::uint8_t concat[16];
    std::uint64_t offs[4] = {0};
    std::size_t p = 0;
    for (int i = 0; i < 3; ++i) {
        std::memcpy(concat + p, words[i], std::strlen(words[i]));
        p += std::strlen(words[i]);
        offs[i + 1] = p;
    }
    double t0 = now_ms();
    acg_automaton* a = nullptr;
    acg_build(concat, offs, 3, &a);
    double t1 = now_ms();
    const char* text = "USHERS";
    for (int k = 0; k < 4; ++k) {
        acg_result* r = nullptr;
        double s0 = now_ms();
        int rc = acg_scan(a, reinterpret_cast<const std::uint8_t*>(text), 6, 1, &r);
        double s1 = now_ms();
        std::printf("scan %d rc=%d m=%llu %.2f ms\n", k, rc, (unsigned long long)acg_result_match_count(r), s1 - s0);
        acg_result_destroy(r);
    }
    std::printf("build %.3f ms\n", t1 - t0);
    acg_automaton_destroy(a);
    return 0;
}
