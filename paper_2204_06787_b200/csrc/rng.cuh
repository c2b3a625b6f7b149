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

// The finalizer with the 64-bit shifts of the xor-shifts moved onto the FMA
// pipe: for the low word, (lo >> s) == mulhi(lo, 2^(32-s)) and the bits
// carried in from the high word are hi * 2^(32-s).  Bit-identical to mix64;
// it only balances the ALU / FMA pipes (each issues every other cycle).
__device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ void xorshr_fma(uint32_t& lo, uint32_t& hi, uint32_t m) {
    const uint32_t nlo = lo ^ mulhi32(lo, m) ^ (hi * m);
    hi ^= mulhi32(hi, m);
    lo = nlo;
}
// High word h2 of the last product of mix64(z) (before its final xor-shift):
// mix64(z) >> 32 == h2 ^ (h2 >> 31), i.e. h2 with bit 0 flipped when its top
// bit is set, so for a threshold th, mix64(z) < th == (h2 < th >> 32)
// whenever h2 >> 1 != (th >> 32) >> 1.
__device__ __forceinline__ uint32_t mix64_h2(uint64_t z) {
    uint64_t y = z ^ (z >> 30);
    y *= 0xbf58476d1ce4e5b9ull;
    uint32_t lo = uint32_t(y), hi = uint32_t(y >> 32);
    xorshr_fma(lo, hi, 1u << 5);  // >> 27
    return mulhi32(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
}
// High 32 bits of mix64(z): only the high word of the last product is formed.
__device__ __forceinline__ uint32_t mix64_hi(uint64_t z) {
    uint64_t y = z ^ (z >> 30);
    y *= 0xbf58476d1ce4e5b9ull;
    uint32_t lo = uint32_t(y), hi = uint32_t(y >> 32);
    xorshr_fma(lo, hi, 1u << 5);  // >> 27
    const uint32_t h2 = mulhi32(lo, 0x133111ebu) + lo * 0x94d049bbu + hi * 0x133111ebu;
    return h2 ^ (h2 >> 31);
}

}  // namespace marsit_b200
