// fft_fast.cuh -- compile-time-specialised radix-16 column-FNT engine (v2).
//
// Same mathematics as fft_tile.cuh (in-place mixed-radix DIF/DIT over a
// shared-memory tile, positions in 4-bit-digit-reversed order between a DIF
// and a DIT), but everything that v1 computed at run time is fixed at
// compile time: the pass schedule (radix 16, then one 2/4/8 pass), the
// thread -> butterfly mapping (shifts, no divisions), the in-register
// twiddles, and the value bounds that let butterfly sums grow lazily across
// stages without reductions. Passes take load / store functors, so the first
// pass of a transform can read packet-major global memory directly and the
// last pass can write it, and the decoder can fuse the end of one transform
// with the start of the next in registers.
//
// Arithmetic: signed lazy values (|v| below a compile-time bound, see
// below). Multiplication by a table twiddle is Shoup's with a balanced
// twiddle (result in (-p, 2p)); by a power of two (all roots of order <= 32
// are powers of two: r16 = 2^6, r8 = 2^12, r4 = -2^8) it is an exact
// shift-and-fold of three instructions.
#pragma once
#include <cstdint>

#include "field.cuh"

namespace fntrs_gpu {
namespace fast {

constexpr uint64_t kP64 = 65537ull;
constexpr uint64_t ceil_p(uint64_t b) { return (b + kP64 - 1) / kP64 * kP64; }
constexpr uint64_t umax(uint64_t a, uint64_t b) { return a > b ? a : b; }

// log2 of the order of a root as a power of two of 2: the root of order L
// (L <= 32) equals 2^(64/L * 1.5?) -- computed instead by search below.
constexpr int pow2_exponent(uint32_t w) {
    // smallest e in [0, 32) with 2^e == w (mod p), or -1
    uint32_t x = 1;
    for (int e = 0; e < 32; ++e) {
        if (x == w) return e;
        x = uint32_t((uint64_t(x) * 2) % kP64);
    }
    return -1;
}

template <int L, int J, bool INV>
struct Tw {
    static constexpr uint32_t w = cpow(croot(L, INV), uint32_t(J));
    static constexpr int e2 = pow2_exponent(w);  // >= 0 for every L <= 32
};

// Signed lazy representation: every value is an int32 (kept in uint32
// registers) congruent to the field element, with |v| < B for a bound B
// tracked at compile time (static_assert B < 2^31). Butterfly differences need
// no offsets, and multiplication by a power of two is three instructions:
//   x * 2^s == (x mod 2^(16-s)) * 2^s - floor(x / 2^(16-s))       (2^16 == -1)
//           == (x << s) - xh * 65537   exactly, xh = x >> (16-s) (arithmetic),
// i.e. SHF + IMAD.SHL/SHF + IMAD.

// balanced representative of a canonical residue: (-p/2, p/2]
__host__ __device__ constexpr int32_t balanced(uint32_t w) { return w > 32768u ? int32_t(w) - 65537 : int32_t(w); }

// FNTRS_POW2_LEA: the power-of-two products below take the LEA form
// independently of the Shoup q * p (FNTRS_LEA)
#ifndef FNTRS_POW2_LEA
#define FNTRS_POW2_LEA FNTRS_LEA
#endif
// x * 2^E mod p, E in [0, 32), |x| < B.
template <int E, uint64_t B>
struct MulPow2 {
    static constexpr int e = E & 31;
    static constexpr bool neg = e >= 16;  // 2^16 = -1
    static constexpr int s = e & 15;
    static constexpr uint64_t OUT = s ? (65536ull + (B >> (16 - s)) + 2) : B;
    __device__ __forceinline__ static uint32_t apply(uint32_t x) {
        if constexpr (s == 0) {
            return neg ? 0u - x : x;
        } else {
            const uint32_t xh = uint32_t(int32_t(x) >> (16 - s));
#if FNTRS_POW2_ALU  // no multiplier-pipe IMAD: (x << s) - (xh << 16) - xh as shifts + one IADD3
            const uint32_t xs = x << s, xh16 = xh << 16;
            return neg ? add3_a(xh16, xh, 0u - xs) : subsub_a(xs, xh16, xh);
#elif FNTRS_POW2_LEA  // SHF (ALU) + LEA (ALU) + one IMAD: x 2^s -/+ xh p
            return neg ? mad_lo(x, 0u - (1u << s), mul_p_lea(xh)) : mad_lo(x, 1u << s, 0u - mul_p_lea(xh));
#else
            const uint32_t xs = x << s;
            return neg ? xh * 65537u - xs : xs - xh * 65537u;
#endif
        }
    }
};

#ifndef FNTRS_POW2_SHIFT
#define FNTRS_POW2_SHIFT 1
#endif

// signed Shoup product by a balanced twiddle w (w2 = 65535 w): (-p, 2p)
__device__ __forceinline__ uint32_t mulws(uint32_t x, uint32_t w, uint32_t w2) {
    const uint32_t q = uint32_t(__mulhi(int32_t(x), int32_t(w2)));
    return x * w - mul_p(q);
}
// signed reduction of any 32-bit x: x - floor(x / 2^16) p = (x mod 2^16) - floor(x / 2^16),
// in [-2^15, 2^16 + 2^15) (inside (-p, 2p)); one shift + one IMAD (the multiplier
// pipe is the codec kernels' busiest: this saves the two IMAD.HI slots of a Shoup quotient)
__device__ __forceinline__ uint32_t reds(uint32_t x) {
    const uint32_t q = uint32_t(int32_t(x) >> 16);
    return x - q * 65537u;
}
// |x| < 2p -> canonical [0, p)
__device__ __forceinline__ uint32_t canon_s2p(uint32_t x) {
    uint32_t r = x + 2 * kP;   // [0, 4p)
    r = min(r, r - 2 * kP);    // [0, 2p)
    return min(r, r - kP);
}

// Multiply by the compile-time twiddle TW<L,J>; OUT is the new bound.
template <int L, int J, bool INV, uint64_t B>
struct MulTw {
    using T = Tw<L, J, INV>;
    static_assert(T::e2 >= 0, "in-register twiddles must be powers of two");
    static constexpr bool shift = FNTRS_POW2_SHIFT;
    static constexpr uint64_t OUT = J == 0 ? B : (shift ? MulPow2<T::e2, B>::OUT : 2 * kP64);
    __device__ __forceinline__ static uint32_t apply(uint32_t x) {
        if constexpr (J == 0)
            return x;
        else if constexpr (shift)
            return MulPow2<T::e2, B>::apply(x);
        else
            return mulws(x, uint32_t(balanced(T::w)), uint32_t(balanced(T::w) * 65535));
    }
};

// ---- in-register DIF: natural in (|v| < BIN), v[rev(s)] = y_s out -----------
template <int R, bool INV, int HALF, int J, uint64_t BIN>
struct DifStage {
    using M = MulTw<2 * HALF, J, INV, 2 * BIN>;
    static constexpr uint64_t LO = 2 * BIN;
    static constexpr uint64_t HI = M::OUT;
    static constexpr uint64_t out() {
        if constexpr (J + 1 < HALF)
            return umax(umax(LO, HI), DifStage<R, INV, HALF, J + 1, BIN>::OUT);
        else
            return umax(LO, HI);
    }
    static constexpr uint64_t OUT = out();
    __device__ __forceinline__ static void run(uint32_t (&v)[R]) {
#pragma unroll
        for (int blk = 0; blk < R; blk += 2 * HALF) {
            const uint32_t a = v[blk + J], b = v[blk + J + HALF];
            v[blk + J] = add_a(a, b);
            v[blk + J + HALF] = M::apply(sub_a(a, b));
        }
        if constexpr (J + 1 < HALF) DifStage<R, INV, HALF, J + 1, BIN>::run(v);
    }
};

template <int R, bool INV, int HALF, uint64_t BIN>
struct DifAll {
    using S = DifStage<R, INV, HALF, 0, BIN>;
    static constexpr uint64_t B1 = S::OUT;
    static constexpr uint64_t out() {
        if constexpr (HALF > 1)
            return DifAll<R, INV, HALF / 2, B1>::OUT;
        else
            return B1;
    }
    static constexpr uint64_t OUT = out();
    __device__ __forceinline__ static void run(uint32_t (&v)[R]) {
        S::run(v);
        if constexpr (HALF > 1) DifAll<R, INV, HALF / 2, B1>::run(v);
    }
};

// ---- in-register DIT: v[rev(s)] in (|v| < BIN), natural out -----------------
template <int R, bool INV, int HALF, int J, uint64_t BIN>
struct DitStage {
    using M = MulTw<2 * HALF, J, INV, BIN>;
    static constexpr uint64_t OUT1 = BIN + M::OUT;
    static constexpr uint64_t out() {
        if constexpr (J + 1 < HALF)
            return umax(OUT1, DitStage<R, INV, HALF, J + 1, BIN>::OUT);
        else
            return OUT1;
    }
    static constexpr uint64_t OUT = out();
    __device__ __forceinline__ static void run(uint32_t (&v)[R]) {
#pragma unroll
        for (int blk = 0; blk < R; blk += 2 * HALF) {
            const uint32_t a = v[blk + J];
            const uint32_t t = M::apply(v[blk + J + HALF]);
            v[blk + J] = add_a(a, t);
            v[blk + J + HALF] = sub_a(a, t);
        }
        if constexpr (J + 1 < HALF) DitStage<R, INV, HALF, J + 1, BIN>::run(v);
    }
};

template <int R, bool INV, int HALF, uint64_t BIN>
struct DitAll {
    using S = DitStage<R, INV, HALF, 0, BIN>;
    static constexpr uint64_t B1 = S::OUT;
    static constexpr uint64_t out() {
        if constexpr (2 * HALF < R)
            return DitAll<R, INV, HALF * 2, B1>::OUT;
        else
            return B1;
    }
    static constexpr uint64_t OUT = out();
    __device__ __forceinline__ static void run(uint32_t (&v)[R]) {
        S::run(v);
        if constexpr (2 * HALF < R) DitAll<R, INV, HALF * 2, B1>::run(v);
    }
};

// ---- direct R-point DFTs, natural order in and out ---------------------------
// y[s] = sum_q x[q] w_R^(qs), w_R = root of order R (inverse root when INV).
// R = 16 is 4 x 4 (Cooley-Tukey): four 4-point DFTs over stride-4 inputs, the
// nine non-trivial twiddles w16^(q2 s1) (powers of two), four 4-point DFTs.
// A 4-point DFT with three-input adds:
//   B = x1+x3, Y0 = x0+x2+B, Y2 = x0+x2-B, D = w4 (x1-x3), Y1 = x0-x2+D, Y3 = x0-x2-D
// is 6 adds + 1 shift-multiply (vs 8 + 1 as two radix-2 stages).
template <int R>
__host__ __device__ constexpr int rev(int i);

template <bool INV, uint64_t B>
struct Dft4 {
    static constexpr int E4 = INV ? 8 : 24;  // w4 = 2^24 = -2^8; w4^-1 = 2^8
    using M = MulPow2<E4, 2 * B>;
    static constexpr uint64_t OUT = umax(4 * B, 2 * B + M::OUT);
    __device__ __forceinline__ static void run(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t& y0,
                                               uint32_t& y1, uint32_t& y2, uint32_t& y3) {
#if FNTRS_ALU_ADDS
        const uint32_t b = add_a(x1, x3);
        const uint32_t d = M::apply(sub_a(x1, x3));
        y0 = add3_a(x0, x2, b);
        y2 = addsub_a(x0, x2, b);
        y1 = addsub_a(x0, d, x2);
        y3 = subsub_a(x0, x2, d);
#else
        const uint32_t b = x1 + x3;
        const uint32_t d = M::apply(x1 - x3);
        y0 = x0 + x2 + b;
        y2 = x0 + x2 - b;
        y1 = x0 - x2 + d;
        y3 = x0 - x2 - d;
#endif
    }
};

// Lazy 4-point DFT with a bound per input (|x_i| < Bi). The w4 product
// d = w4 (x1 - x3) is either reduced (MulPow2, three instructions) or, when
// every output stays below LIM, left as the exact shift (x3 - x1) << 8
// (forward, w4 = -2^8) / (x1 - x3) << 8 (inverse): one instruction, and the
// bound grows by 2^8. LIM = 0 never takes the lazy form. Used where the
// outputs go into a Shoup product (which reduces any 32-bit signed value).
#ifndef FNTRS_LAZY_LIM
#define FNTRS_LAZY_LIM (1ull << 30)
#endif
constexpr uint64_t kLazyLim = FNTRS_LAZY_LIM;
#ifndef FNTRS_PIN_SHIFT
#define FNTRS_PIN_SHIFT 0
#endif

template <bool INV, uint64_t B0, uint64_t B1, uint64_t B2, uint64_t B3, uint64_t LIM, bool PIN = kAluAdds>
struct Dft4L {
    static constexpr int E4 = INV ? 8 : 24;
    static constexpr uint64_t BD = B1 + B3;
    using M = MulPow2<E4, BD>;
    static constexpr bool lazy = LIM != 0 && B0 + B2 + (BD << 8) <= LIM;
    static constexpr uint64_t D = lazy ? (BD << 8) : M::OUT;
    static constexpr uint64_t O02 = B0 + B1 + B2 + B3;
    static constexpr uint64_t O13 = B0 + B2 + D;
    static constexpr uint64_t OUT = umax(O02, O13);
    __device__ __forceinline__ static void run(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t& y0,
                                               uint32_t& y1, uint32_t& y2, uint32_t& y3) {
        const uint32_t b = add_p<PIN>(x1, x3);
        uint32_t d;
        if constexpr (lazy)
            d = shl_p<PIN && FNTRS_PIN_SHIFT, 8>(INV ? sub_p<PIN>(x1, x3) : sub_p<PIN>(x3, x1));
        else
            d = M::apply(sub_p<PIN>(x1, x3));
        y0 = add3_p<PIN>(x0, x2, b);
        y2 = addsub_p<PIN>(x0, x2, b);
        y1 = addsub_p<PIN>(x0, d, x2);
        y3 = subsub_p<PIN>(x0, x2, d);
    }
};

// PIN2: the second 4 x 4 stage of a radix-16 pins its adds independently (half pinning)
template <int R, bool INV, uint64_t B, uint64_t LIM = 0, bool PIN = kAluAdds, bool PIN2 = PIN>
struct Dft;

template <bool INV, uint64_t B, uint64_t LIM, bool PIN, bool PIN2>
struct Dft<1, INV, B, LIM, PIN, PIN2> {
    static constexpr uint64_t OUT = B;
    __device__ __forceinline__ static void run(const uint32_t (&)[1], uint32_t (&y)[1]) {}
};

template <bool INV, uint64_t B, uint64_t LIM, bool PIN, bool PIN2>
struct Dft<2, INV, B, LIM, PIN, PIN2> {
    static constexpr uint64_t OUT = 2 * B;
    __device__ __forceinline__ static void run(const uint32_t (&x)[2], uint32_t (&y)[2]) {
        y[0] = add_a(x[0], x[1]);
        y[1] = sub_a(x[0], x[1]);
    }
};

template <bool INV, uint64_t B, uint64_t LIM, bool PIN, bool PIN2>
struct Dft<4, INV, B, LIM, PIN, PIN2> {
    static constexpr uint64_t OUT = Dft4<INV, B>::OUT;
    __device__ __forceinline__ static void run(const uint32_t (&x)[4], uint32_t (&y)[4]) {
        Dft4<INV, B>::run(x[0], x[1], x[2], x[3], y[0], y[1], y[2], y[3]);
    }
};

// twiddle w_R^(e) applied to a value of bound B (R <= 32: powers of two)
template <int R, int EXP, bool INV, uint64_t B>
struct TwR {
    static constexpr int e2 = Tw<R, (EXP % R + R) % R, INV>::e2;
    using M = MulPow2<e2, B>;
    static constexpr bool trivial = (EXP % R) == 0;
    static constexpr uint64_t OUT = trivial ? B : M::OUT;
    __device__ __forceinline__ static uint32_t apply(uint32_t x) {
        if constexpr (trivial)
            return x;
        else
            return M::apply(x);
    }
};

// R = 8: 2 x 4 (q = 2 q1 + q2, s = s1 + 4 s2): DFT4 over q1 for each q2,
// twiddle w8^(q2 s1), DFT2 over q2.
template <bool INV, uint64_t B, uint64_t LIM, bool PIN, bool PIN2>
struct Dft<8, INV, B, LIM, PIN, PIN2> {
    static constexpr uint64_t B1 = Dft4<INV, B>::OUT;
    static constexpr uint64_t BT = umax(umax(TwR<8, 1, INV, B1>::OUT, TwR<8, 2, INV, B1>::OUT), TwR<8, 3, INV, B1>::OUT);
    static constexpr uint64_t OUT = 2 * umax(B1, BT);
    __device__ __forceinline__ static void run(const uint32_t (&x)[8], uint32_t (&y)[8]) {
        uint32_t z0[4], z1[4];
        Dft4<INV, B>::run(x[0], x[2], x[4], x[6], z0[0], z0[1], z0[2], z0[3]);
        Dft4<INV, B>::run(x[1], x[3], x[5], x[7], z1[0], z1[1], z1[2], z1[3]);
        z1[1] = TwR<8, 1, INV, B1>::apply(z1[1]);
        z1[2] = TwR<8, 2, INV, B1>::apply(z1[2]);
        z1[3] = TwR<8, 3, INV, B1>::apply(z1[3]);
#pragma unroll
        for (int s1 = 0; s1 < 4; ++s1) {
            y[s1] = add_a(z0[s1], z1[s1]);
            y[s1 + 4] = sub_a(z0[s1], z1[s1]);
        }
    }
};

// R = 16 as 4 x 4 with a bound per element: stage 1 = four Dft4L over
// stride-4 inputs (outputs s1 = 0, 2 below 4B; s1 = 1, 3 below 2B + D), the
// nine twiddles w16^(q2 s1) (reducing shift-multiplies), stage 2 = four Dft4L
// whose first input is untwiddled. Stage 1 takes the lazy product only when
// the whole transform then stays below LIM.
// per-unit masks over every radix-16 pin request (A/B knobs; 1 = as requested)
#ifndef FNTRS_STAGE1_PIN
#define FNTRS_STAGE1_PIN 1
#endif
#ifndef FNTRS_STAGE2_PIN
#define FNTRS_STAGE2_PIN 1
#endif
template <bool INV, uint64_t B, bool L1, uint64_t LIM, bool PIN = kAluAdds, bool PIN2 = PIN>
struct Dft16B {
    using S1 = Dft4L<INV, B, B, B, B, L1 ? (uint64_t(1) << 62) : 0, PIN && FNTRS_STAGE1_PIN>;
    static constexpr uint64_t Y(int s1) { return (s1 & 1) ? S1::O13 : S1::O02; }
    template <int Q2, int S1I>
    using T = TwR<16, Q2 * S1I, INV, ((S1I & 1) ? S1::O13 : S1::O02)>;
    template <int S1I>
    using S2 = Dft4L<INV, ((S1I & 1) ? S1::O13 : S1::O02), T<1, S1I>::OUT, T<2, S1I>::OUT, T<3, S1I>::OUT, LIM, PIN2 && FNTRS_STAGE2_PIN>;
    static constexpr uint64_t OUT = umax(umax(S2<0>::OUT, S2<1>::OUT), umax(S2<2>::OUT, S2<3>::OUT));
};

template <bool INV, uint64_t B, uint64_t LIM, bool PIN, bool PIN2>
struct Dft<16, INV, B, LIM, PIN, PIN2> {
    static constexpr bool L1 = LIM != 0 && Dft16B<INV, B, true, LIM>::OUT <= LIM;
    using D = Dft16B<INV, B, L1, LIM, PIN, PIN2>;
    static constexpr uint64_t OUT = D::OUT;
    template <int Q2, int S1>
    __device__ __forceinline__ static uint32_t tw(uint32_t x) {
        return D::template T<Q2, S1>::apply(x);
    }
    __device__ __forceinline__ static void run(const uint32_t (&x)[16], uint32_t (&y)[16]) {
        uint32_t z[4][4];  // z[q2][s1]
#pragma unroll
        for (int q2 = 0; q2 < 4; ++q2)
            D::S1::run(x[q2], x[q2 + 4], x[q2 + 8], x[q2 + 12], z[q2][0], z[q2][1], z[q2][2], z[q2][3]);
        z[1][1] = tw<1, 1>(z[1][1]);
        z[1][2] = tw<1, 2>(z[1][2]);
        z[1][3] = tw<1, 3>(z[1][3]);
        z[2][1] = tw<2, 1>(z[2][1]);
        z[2][2] = tw<2, 2>(z[2][2]);
        z[2][3] = tw<2, 3>(z[2][3]);
        z[3][1] = tw<3, 1>(z[3][1]);
        z[3][2] = tw<3, 2>(z[3][2]);
        z[3][3] = tw<3, 3>(z[3][3]);
        D::template S2<0>::run(z[0][0], z[1][0], z[2][0], z[3][0], y[0], y[4], y[8], y[12]);
        D::template S2<1>::run(z[0][1], z[1][1], z[2][1], z[3][1], y[1], y[5], y[9], y[13]);
        D::template S2<2>::run(z[0][2], z[1][2], z[2][2], z[3][2], y[2], y[6], y[10], y[14]);
        D::template S2<3>::run(z[0][3], z[1][3], z[2][3], z[3][3], y[3], y[7], y[11], y[15]);
    }
};

// DIF placement: natural in, v[rev(s)] = y_s out. DIT placement: v[rev(s)] in, natural out.
template <int R, bool INV, uint64_t BIN, uint64_t LIM = 0, bool PIN = kAluAdds, bool PIN2 = PIN>
__device__ __forceinline__ void dif_regs(uint32_t (&v)[R]) {
    static_assert(Dft<R, INV, BIN, LIM>::OUT < (1ull << 31), "lazy bound overflow");
    uint32_t y[R];
    Dft<R, INV, BIN, LIM, PIN, PIN2>::run(v, y);
#pragma unroll
    for (int s = 0; s < R; ++s) v[rev<R>(s)] = y[s];
}
template <int R, bool INV, uint64_t BIN, uint64_t LIM = 0, bool PIN = kAluAdds, bool PIN2 = PIN>
__device__ __forceinline__ void dit_regs(uint32_t (&v)[R]) {
    static_assert(Dft<R, INV, BIN, LIM>::OUT < (1ull << 31), "lazy bound overflow");
    uint32_t x[R];
#pragma unroll
    for (int s = 0; s < R; ++s) x[s] = v[rev<R>(s)];
    Dft<R, INV, BIN, LIM, PIN, PIN2>::run(x, v);
}
template <int R, bool INV, uint64_t BIN, uint64_t LIM = 0>
constexpr uint64_t dif_bound() { return Dft<R, INV, BIN, LIM>::OUT; }
template <int R, bool INV, uint64_t BIN, uint64_t LIM = 0>
constexpr uint64_t dit_bound() { return Dft<R, INV, BIN, LIM>::OUT; }

template <int R>
__host__ __device__ constexpr int rev(int i) {
    int r = 0;
    for (int b = 1, o = R >> 1; b < R; b <<= 1, o >>= 1)
        if (i & b) r |= o;
    return r;
}

// ---- schedule of a size-2^E transform -------------------------------------
template <int E>
struct Sched {
    static constexpr int P = (E + 3) / 4;                  // number of passes
    static constexpr int rlog(int p) { return (p < E / 4) ? 4 : (E % 4); }
    static constexpr int llog(int p) { return E - 4 * p; }  // block length log2 of pass p (DIF order)
    static constexpr int slog(int p) { return llog(p) - rlog(p); }
};

// frequency index of DIF output position p (4-bit digit reversal; the last
// digit is E%4 bits wide when E%4 != 0)
template <int E>
__device__ __forceinline__ uint32_t perm(uint32_t p) {
    uint32_t f = 0;
    int sh = E, out = 0;
#pragma unroll
    for (int i = 0; i < E / 4; ++i) {
        sh -= 4;
        f |= ((p >> sh) & 15u) << out;
        out += 4;
    }
    if constexpr (E % 4) f |= (p & ((1u << (E % 4)) - 1u)) << out;
    return f;
}

// inverse of perm<E>: the DIF output position holding frequency f
template <int E>
__device__ __forceinline__ uint32_t perm_inv(uint32_t f) {
    uint32_t p = 0;
    int sh = E;
#pragma unroll
    for (int i = 0; i < E / 4; ++i) {
        sh -= 4;
        p |= ((f >> (4 * i)) & 15u) << sh;
    }
    if constexpr (E % 4) p |= f >> (4 * (E / 4));
    return p;
}

// frequency of the leading digits: perm of position (b << rlast) minus the
// last digit's contribution, i.e. perm<E>(b << RL) where RL = last radix log2.
template <int E>
__device__ __forceinline__ uint32_t perm_head(uint32_t b) {
    constexpr int RL = Sched<E>::rlog(Sched<E>::P - 1);
    return perm<E>(b << RL);
}

}  // namespace fast
}  // namespace fntrs_gpu
