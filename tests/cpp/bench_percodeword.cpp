// Per-codeword latency of the drop-in C++ API (development aid, not a test):
// each call is one codeword through the GPU (H2D, kernels, D2H, sync).
#include <chrono>
#include <cstdio>
#include <vector>

#include "fntrs/codec.hpp"

using namespace fntrs;
using namespace fntrs::codec;

int main() {
    auto p = CodeParams::make(128, 256, false);
    std::vector<Fe> src(128);
    for (uint32_t i = 0; i < 128; ++i) src[i] = (i * 7919u) % 65537u;
    auto enc = encode_nonsystematic(p, src);
    Codeword rx;
    for (uint32_t i = 0; i < 256; i += 2) rx.push_back({i, enc[i]});
    decode_nonsystematic(p, rx);
    const int reps = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) encode_nonsystematic(p, src);
    auto t1 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) decode_nonsystematic(p, rx);
    auto t2 = std::chrono::steady_clock::now();
    std::printf("per-codeword C++ API (n=256, k=128): encode %.1f us, decode %.1f us per call\n",
                std::chrono::duration<double, std::micro>(t1 - t0).count() / reps,
                std::chrono::duration<double, std::micro>(t2 - t1).count() / reps);
    return decode_nonsystematic(p, rx) == src ? 0 : 1;
}
