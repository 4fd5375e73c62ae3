// kernelscope/rng.hpp -- B200 drop-in: the seeded input generator.
//
// Bit-compatible with /root/reference/proj/include/kernelscope/rng.hpp:12-39
// (splitmix64; uniform [-1,1) floats from the top 53 bits).  Draw n (1-based)
// of a stream is mix(seed + n*gamma), which is what the device generator
// ks_fill_pm1_f32 uses to produce the same inputs in place on the GPU.
#pragma once

#include <cstdint>

#include "kernelscope/tensor.hpp"

namespace kernelscope {

struct SplitMix64 {
    static constexpr std::uint64_t kGamma = 0x9E3779B97F4A7C15ull;
    std::uint64_t state;

    explicit SplitMix64(std::uint64_t seed) : state(seed) {}

    static std::uint64_t mix(std::uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }

    std::uint64_t next() { return mix(state += kGamma); }
    double next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    float next_pm1() { return static_cast<float>(2.0 * next_unit() - 1.0); }
};

// One stream fills x, then k, then gy, each in flat row-major order.
template <typename C>
inline void fill_pm1(SplitMix64& rng, C& container) {
    for (auto& v : container.data) v = rng.next_pm1();
}

}  // namespace kernelscope
