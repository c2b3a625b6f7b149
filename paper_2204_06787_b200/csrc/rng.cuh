// rng.cuh — the reference's counter-based RNG on the device (rng.hpp:28-73).
// Draw n (0-based) of the stream keyed by (seed, purpose, worker, round,
// segment) is mix64(key + (n + 1) * gamma): random access, so any thread can
// produce any draw.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace marsit_b200 {

// SplitMix64 finalizer (rng.hpp:66-70).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// RngStream key (rng.hpp:28-37): seed, purpose, worker, round, segment.
__device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t purpose, uint64_t w,
                                               uint64_t t, uint64_t s) {
    uint64_t h = mix64(seed ^ 0x6a09e667f3bcc909ull);
    h = mix64(h ^ (purpose * kGamma));
    h = mix64(h ^ ((w + 1) * kGamma));
    h = mix64(h ^ ((t + 1) * kGamma));
    return mix64(h ^ ((s + 1) * kGamma));
}

}  // namespace marsit_b200
