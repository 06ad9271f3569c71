// locload/rng.hpp -- source-compatible drop-in for proj/include/locload/rng.hpp.
//
// The stream arithmetic lives in locload_rng.cuh (shared with the CUDA
// kernels, so host and device draws are the same bits); this header only
// adds the reference's class interface on top: SplitMix64 with next /
// bounded / next_double / next_gaussian (rng.hpp:31-66).
#pragma once

#include <cmath>
#include <cstdint>

#include "locload_rng.cuh"

namespace locload {

using ll::derive_seed;
using ll::mix64;

class SplitMix64 {
public:
    explicit SplitMix64(std::uint64_t seed) : s_(seed) {}

    std::uint64_t next() { return s_.next(); }
    std::uint64_t bounded(std::uint64_t n) { return s_.bounded(n); }
    // 53 high bits -> [0, 1)
    double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    // Box-Muller from two draws; u1 in (0, 1]
    double next_gaussian() {
        const double u1 = static_cast<double>((next() >> 11) + 1) * 0x1.0p-53;
        const double u2 = next_double();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
    }

private:
    ll::SplitMix s_;
};

} // namespace locload
