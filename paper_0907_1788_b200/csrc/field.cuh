// field.cuh -- GF(65537) arithmetic in 32-bit lanes for sm_100a.
//
// Values live in redundant ranges inside uint32 lanes and are canonicalised
// to [0, 65536] (the reference's Fe range, proj/include/fntrs/field.hpp:9-11)
// only where they leave the kernel.
//
// Multiplication by a known w < p uses Shoup's method. For p = 2^16 + 1 the
// Shoup constant floor(w * 2^32 / p) is exactly 65535 * w (since
// 2^32 = 65535 * p + 1), so no second table is needed:
//     q = umulhi(x, 65535 w);  r = x w - q p   (mod 2^32),  r in [0, 2p)
// for ANY 32-bit x. That lets butterfly sums grow lazily across stages and
// keeps the reductions on the FMA pipe (IMAD.HI, IMAD) while the adds use
// the ALU pipe.
#pragma once
#include <cstdint>

namespace fntrs_gpu {

constexpr uint32_t kP = 65537u;

__host__ __device__ constexpr uint32_t cmul(uint32_t a, uint32_t b) {
    // canonical product, reference gf::mul (field.hpp:30-37)
    uint64_t x = uint64_t(a) * b;
    uint32_t lo = uint32_t(x & 0xFFFFu), hi = uint32_t(x >> 16);
    return lo >= hi ? lo - hi : lo + kP - hi;
}

__host__ __device__ constexpr uint32_t cpow(uint32_t b, uint64_t e) {
    uint32_t r = 1;
    while (e) {
        if (e & 1) r = cmul(r, b);
        e >>= 1;
        if (e) b = cmul(b, b);
    }
    return r;
}

// root of exact order n (power of two <= 65536): 3^(65536/n), field.hpp:58-63
__host__ __device__ constexpr uint32_t croot(uint32_t n, bool inverse) {
    return cpow(3u, inverse ? (uint64_t(65536u / n) * 65535u) % 65536u : 65536u / n);
}

// x * w mod p into [0, 2p); w < p canonical, x any uint32.
__device__ __forceinline__ uint32_t mulw(uint32_t x, uint32_t w) {
    const uint32_t q = __umulhi(x, w * 65535u);
    return x * w - q * kP;
}

// Same with the Shoup constant supplied (w2 = 65535 * w).
__device__ __forceinline__ uint32_t mulw2(uint32_t x, uint32_t w, uint32_t w2) {
    const uint32_t q = __umulhi(x, w2);
    return x * w - q * kP;
}

// any uint32 -> [0, 2p)
__device__ __forceinline__ uint32_t red(uint32_t x) {
    const uint32_t q = __umulhi(x, 65535u);
    return x - q * kP;
}

// [0, 2p) -> [0, p)
__device__ __forceinline__ uint32_t red2p(uint32_t x) { return min(x, x - kP); }

// any uint32 -> canonical [0, p)
__device__ __forceinline__ uint32_t canon(uint32_t x) { return red2p(red(x)); }

// general canonical product of two canonical values (both <= 65536)
__device__ __forceinline__ uint32_t gmul(uint32_t a, uint32_t b) {
    const uint64_t x = uint64_t(a) * b;  // < 2^32 + 1
    const uint32_t lo = uint32_t(x) & 0xFFFFu, hi = uint32_t(x >> 16);
    const uint32_t r = lo + kP - hi;     // hi <= 65536 -> r in [1, 2p)
    return red2p(r);
}

__device__ __forceinline__ uint32_t gpow(uint32_t b, uint32_t e) {
    uint32_t r = 1;
    while (e) {
        if (e & 1) r = gmul(r, b);
        e >>= 1;
        b = gmul(b, b);
    }
    return r;
}

__device__ __forceinline__ uint32_t ginv(uint32_t a) { return gpow(a, kP - 2); }

}  // namespace fntrs_gpu
