// locload_rng.cuh -- counter-based splitmix64, shared by host and device code
// (the CUDA kernels and the C++ API in include/locload/rng.hpp).
//
// Bit-identical to proj/include/locload/rng.hpp: mix64 (:9-13), derive_seed
// (:19-26), SplitMix64::next (:35-38) and the Lemire bounded draw (:41-50).
// The stream is counter based: the k-th (0-based) draw of SplitMix64(s) is
// mix64(s + (k+1)*gamma), which is what lets the Fisher-Yates draws of a whole
// epoch be computed in parallel (permute.cu).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define LL_HD __host__ __device__ __forceinline__
#else
#define LL_HD inline
#endif

namespace ll {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

LL_HD uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

LL_HD uint64_t derive_seed(uint64_t seed, uint64_t a) {
    const uint64_t s = mix64(seed + kGamma);
    return mix64(s ^ (a + 0xbf58476d1ce4e5b9ULL));
}

LL_HD uint64_t derive_seed(uint64_t seed, uint64_t a, uint64_t b) {
    return mix64(derive_seed(seed, a) ^ (b + 0x94d049bb133111ebULL));
}

// k0-th (0-based) draw of the stream keyed s
LL_HD uint64_t draw_at(uint64_t s, uint64_t k0) { return mix64(s + (k0 + 1) * kGamma); }

LL_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

// One Lemire trial: returns true when draw r is accepted for range n and
// writes the result.  threshold = (2^64 - n) mod n < n, so lo >= n accepts
// without the 64-bit modulo (taken with probability < n / 2^64).
// The 64-bit modulo is kept out of line so the compiler cannot hoist it onto
// the (almost always taken) fast path.
#if defined(__CUDACC__)
static __host__ __device__ __noinline__
#else
inline
#endif
uint64_t lemire_threshold(uint64_t n) { return (0 - n) % n; }

LL_HD bool lemire_accept(uint64_t r, uint64_t n, uint64_t* out) {
    const uint64_t lo = r * n;
    *out = umulhi64(r, n);
    if (lo >= n) return true;
    return lo >= lemire_threshold(n);
}

struct SplitMix {
    uint64_t state;
    LL_HD explicit SplitMix(uint64_t s) : state(s) {}
    LL_HD uint64_t next() {
        state += kGamma;
        return mix64(state);
    }
    LL_HD uint64_t bounded(uint64_t n) {
        uint64_t v;
        for (;;) {
            if (lemire_accept(next(), n, &v)) return v;
        }
    }
};

} // namespace ll
