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
// for ANY 32-bit x. That lets butterfly sums grow lazily across stages; the
// reduction is IMAD.HI + IMAD on the multiplier pipe and one LEA (q p) on the
// ALU pipe.
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

// Pipe balance. The integer multiplier (the FMA-heavy pipe: IMAD, and
// IMAD.HI / IMAD.WIDE at two slots each) is the busiest pipe in every codec
// kernel, and ptxas also places plain adds and shifts there (IMAD.IADD,
// IMAD.SHL). q * p = (q << 16) + q is one LEA on the ALU pipe; written as
// PTX shl + add so NVVM cannot fold it back into a multiply. Off by default
// (decode: ptxas re-balances by moving other adds to IMAD.IADD, 1-4 % slower);
// the encode unit (codec_fast.cu) turns it on (+3 %; profiles/README.md).
#ifndef FNTRS_LEA
#define FNTRS_LEA 0
#endif
// q * p as shift + add (one LEA on the ALU pipe)
__device__ __forceinline__ uint32_t mul_p_lea(uint32_t q) {
    uint32_t t;
    asm("{\n\t.reg .b32 s;\n\tshl.b32 s, %1, 16;\n\tadd.u32 %0, s, %1;\n\t}" : "=r"(t) : "r"(q));
    return t;
}
__device__ __forceinline__ uint32_t mul_p(uint32_t q) {
#if FNTRS_LEA
    return mul_p_lea(q);
#else
    return q * kP;
#endif
}
// a * b + c as exactly one IMAD (instead of a shift on either pipe plus an add)
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// Adds pinned to the ALU pipe. ptxas turns a share of two-input adds into
// IMAD.IADD to balance pipes, but on sm_100a the multiplier pipe is the
// saturated one. Adding a zero that only exists at run time (a constant-bank
// word) inside an opaque PTX block makes every such add a three-input IADD3,
// which has no IMAD form; three-input sums are pinned the same way so that
// NVVM cannot re-split them into two-input adds. Off by default: it removes
// 6.5 % of the multiplier-pipe instructions but the issue rate stays at 66 %
// (C2 decode +1 %, C2 encode -1.5 %; profiles/README.md).
#ifndef FNTRS_ALU_ADDS
#define FNTRS_ALU_ADDS 0
#endif
static __constant__ uint32_t g_alu_zero;  // never written: 0
// P = true: pinned to the ALU pipe as described; P = false: plain C++ adds
// (ptxas places them). The *_a forms follow FNTRS_ALU_ADDS.
template <bool P>
__device__ __forceinline__ uint32_t add_p(uint32_t a, uint32_t b) {
    if constexpr (P) {
        uint32_t r;
        asm("{\n\t.reg .b32 t;\n\tadd.u32 t, %1, %2;\n\tadd.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(a), "r"(b), "r"(g_alu_zero));
        return r;
    } else {
        return a + b;
    }
}
template <bool P>
__device__ __forceinline__ uint32_t sub_p(uint32_t a, uint32_t b) {
    if constexpr (P) {
        uint32_t r;
        asm("{\n\t.reg .b32 t;\n\tsub.u32 t, %1, %2;\n\tadd.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(a), "r"(b), "r"(g_alu_zero));
        return r;
    } else {
        return a - b;
    }
}
// a + b + c, a + b - c, a - b - c as one IADD3 each
template <bool P>
__device__ __forceinline__ uint32_t add3_p(uint32_t a, uint32_t b, uint32_t c) {
    if constexpr (P) {
        uint32_t r;
        asm("{\n\t.reg .b32 t;\n\tadd.u32 t, %1, %2;\n\tadd.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(a), "r"(b), "r"(c));
        return r;
    } else {
        return a + b + c;
    }
}
template <bool P>
__device__ __forceinline__ uint32_t addsub_p(uint32_t a, uint32_t b, uint32_t c) {
    if constexpr (P) {
        uint32_t r;
        asm("{\n\t.reg .b32 t;\n\tadd.u32 t, %1, %2;\n\tsub.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(a), "r"(b), "r"(c));
        return r;
    } else {
        return a + b - c;
    }
}
template <bool P>
__device__ __forceinline__ uint32_t subsub_p(uint32_t a, uint32_t b, uint32_t c) {
    if constexpr (P) {
        uint32_t r;
        asm("{\n\t.reg .b32 t;\n\tsub.u32 t, %1, %2;\n\tsub.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(a), "r"(b), "r"(c));
        return r;
    } else {
        return a - b - c;
    }
}
// x << S on the ALU pipe when P (a funnel shift whose low word is the run-time
// zero, so ptxas cannot fold it into an IMAD with the following add)
template <bool P, int S>
__device__ __forceinline__ uint32_t shl_p(uint32_t x) {
    if constexpr (P) {
        uint32_t r;
        asm("shf.l.clamp.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(g_alu_zero), "r"(x), "n"(S));
        return r;
    } else {
        return x << S;
    }
}
constexpr bool kAluAdds = FNTRS_ALU_ADDS != 0;
__device__ __forceinline__ uint32_t add_a(uint32_t a, uint32_t b) { return add_p<kAluAdds>(a, b); }
__device__ __forceinline__ uint32_t sub_a(uint32_t a, uint32_t b) { return sub_p<kAluAdds>(a, b); }
__device__ __forceinline__ uint32_t add3_a(uint32_t a, uint32_t b, uint32_t c) { return add3_p<kAluAdds>(a, b, c); }
__device__ __forceinline__ uint32_t addsub_a(uint32_t a, uint32_t b, uint32_t c) { return addsub_p<kAluAdds>(a, b, c); }
__device__ __forceinline__ uint32_t subsub_a(uint32_t a, uint32_t b, uint32_t c) { return subsub_p<kAluAdds>(a, b, c); }

// x * w mod p into [0, 2p); w < p canonical, x any uint32.
__device__ __forceinline__ uint32_t mulw(uint32_t x, uint32_t w) {
    const uint32_t q = __umulhi(x, w * 65535u);
    return x * w - mul_p(q);
}

// Same with the Shoup constant supplied (w2 = 65535 * w).
__device__ __forceinline__ uint32_t mulw2(uint32_t x, uint32_t w, uint32_t w2) {
    const uint32_t q = __umulhi(x, w2);
    return x * w - mul_p(q);
}

// any uint32 -> [0, 2p)
__device__ __forceinline__ uint32_t red(uint32_t x) {
    const uint32_t q = __umulhi(x, 65535u);
    return x - mul_p(q);
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
