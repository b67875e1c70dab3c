// fft_pass.cuh -- shared device building blocks of the fused codec kernels:
// escape helpers, tile geometry, and the generic radix pass over a shared
// tile with load / store functors (see codec_fast.cu for the design).
#pragma once
#include <cstdint>

#include "fft_fast.cuh"
#include "internal.h"

namespace fntrs_gpu {
namespace fast {
namespace {

#ifndef FNTRS_SMEM_CAP
#define FNTRS_SMEM_CAP (2ull * 65537ull)
#endif
constexpr uint64_t kSmemCap = FNTRS_SMEM_CAP;
#ifndef FNTRS_SPLIT_PIN
#define FNTRS_SPLIT_PIN 0
#endif
#ifndef FNTRS_LAZY_LAST
#define FNTRS_LAZY_LAST 1
#endif  // bound of values kept in shared memory
constexpr uint64_t k2P = 2 * kP64;
constexpr uint32_t kGuardBytes = 128;  // guard row slot below each decode stage buffer

__device__ __noinline__ bool esc_find(const unsigned long long* keys, uint64_t n, unsigned long long key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (keys[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo < n && keys[lo] == key;
}
__device__ __forceinline__ bool esc_has(const EscIn& e, unsigned long long key) { return esc_find(e.keys, e.n, key); }

__device__ __noinline__ void esc_append(unsigned long long* keys, unsigned long long* count, uint64_t cap,
                                        unsigned long long key) {
    const unsigned long long i = atomicAdd(count, 1ull);
    if (i < cap) keys[i] = key;
}
__device__ __forceinline__ void emit_escape(const EscOut& e, unsigned long long key) {
    esc_append(e.keys, e.count, e.cap, key);
}

// opaque copy: keeps the per-tile base pointer in a register so per-symbol
// addresses are one 32-bit offset away (no 64-bit re-association)
template <class T>
__device__ __forceinline__ T* launder(T* p) {
    asm("mov.b64 %0, %0;" : "+l"(p));
    return p;
}

// A byte stride whose high word ptxas cannot prove zero (it carries the
// run-time zero g_alu_zero), so that p + stride stays a 64-bit add on the ALU
// pipe (IADD3 + IADD3.X) instead of becoming an IMAD.WIDE (two multiplier slots)
__device__ __forceinline__ uint64_t opaque_stride(uint64_t bytes) {
    return bytes | (uint64_t(g_alu_zero) << 32);
}
template <class T>
__device__ __forceinline__ T* step_ptr(T* p, uint64_t stride_bytes) {
    return reinterpret_cast<T*>(reinterpret_cast<uint64_t>(p) + stride_bytes);
}
// base[idx] of an 8-byte table with the address formed on the ALU pipe
// (shift + 64-bit add against an opaque high word) instead of IMAD.WIDE
__device__ __forceinline__ uint2 ldg_alu(const uint2* base, uint32_t idx) {
    return __ldg(step_ptr(base, opaque_stride(uint64_t(idx) << 3)));
}

template <int N>
constexpr int ilog2c() {
    int e = 0;
    while ((1 << e) < N) ++e;
    return e;
}

// |v| < B -> canonical [0, p), cheapest route for the bound
template <uint64_t B>
__device__ __forceinline__ uint32_t canon_b(uint32_t v) {
    if constexpr (B <= k2P) {
        return canon_s2p(v);
    } else {
        static_assert(B < (1ull << 31), "");
        return canon_s2p(reds(v));  // (-p, 2p) -> [0, p)
    }
}

// stored-value cap meaning "store canonical [0, p)"
constexpr uint64_t kCanon = 1;

template <uint64_t B, uint64_t CAP>
__device__ __forceinline__ uint32_t cap(uint32_t v) {
    if constexpr (CAP == kCanon)
        return canon_b<B>(v);
    else
    if constexpr (B > CAP)
        return reds(v);
    else
        return v;
}

// ---- geometry ---------------------------------------------------------------
template <int E, int WT_, int NT_, int MINB_ = 1>
struct Geom {
    static constexpr int MINB = MINB_;
    static constexpr int N = 1 << E;
    static constexpr int WT = WT_;
    static constexpr int NT = NT_;
    static constexpr int RLZ = Sched<E>::rlog(Sched<E>::P - 1);
    static constexpr int RPW = WT >= 32 ? 1 : 32 / WT;  // tile rows touched by one warp
    // shared tile index with a row swizzle keeping the sub = 1 passes
    // (rows R*b + q, consecutive b in one warp) on distinct banks
    __device__ __forceinline__ static uint32_t idx(uint32_t row, uint32_t col) {
        if constexpr (RPW > 1)
            row ^= (row >> RLZ) & uint32_t(RPW - 1);
        return row * WT + col;
    }
    // index of row (N2 - 1 - row) for row < N2 (N2 a power of two): the reversed
    // view. Unswizzled, the subtraction form lets a compile-time row offset fold
    // into the shared-memory immediate; swizzled, XOR is cheaper.
    template <uint32_t N2>
    __device__ __forceinline__ static uint32_t idx_flip(uint32_t row, uint32_t col) {
        if constexpr (RPW > 1)
            return idx(row ^ (N2 - 1u), col);
        else
            return idx((N2 - 1u) - row, col);
    }
};

// tile width / threads per size
template <int E>
struct Pick {
    static constexpr int N = 1 << E;
    static constexpr int WT = N <= 512 ? 32 : (N == 1024 ? 16 : 8);
    static constexpr int NT = N == 4096 ? 512 : 256;
    // blocks per SM the register budget should allow (shared memory permits 4 at N <= 512)
    static constexpr int MINB = N <= 512 ? 4 : (N <= 2048 ? 2 : 1);
    using G = Geom<E, WT, NT, MINB>;
};

// ---- generic pass (one codeword per work item) ----------------------------
// DIF (DIT=false) or DIT pass with the geometry of DIF pass p of a size-2^E
// transform. Loaded values must be below BIN; stored values are below OCAP.
// twp: per-pass twiddle table, row t holds {r_len^(t s), 65535 r_len^(t s)}
// for s < R (only read when sub > 1).
// FNTRS_CW1_PIN (one codeword per work item): 0 = adds placed by ptxas (or
// FNTRS_ALU_ADDS); bit 0 / bit 1 pin the adds of the first / second 4 x 4
// stage of each radix-16 butterfly to the ALU pipe.
#ifndef FNTRS_CW1_PIN
#define FNTRS_CW1_PIN 0
#endif
// two-codeword items (FNTRS_SPLIT_PIN): the same stage masks for codeword 0 / 1
#ifndef FNTRS_CW2_PIN0
#define FNTRS_CW2_PIN0 0
#endif
#ifndef FNTRS_CW2_PIN1
#define FNTRS_CW2_PIN1 3
#endif
struct NoFix {
    template <int R>
    __device__ __forceinline__ void operator()(uint32_t (&)[R], uint32_t, uint32_t, uint32_t) const {}
};
struct NoFlush {
    __device__ __forceinline__ void operator()(uint32_t, uint32_t, uint32_t, uint32_t) const {}
};

// twiddle s of a row stored as uint4 pairs; s is a compile-time constant after
// unrolling, so each pair is loaded once (on its first use, s = 1 or s even).
// CT: the table is in constant memory (codec_dec.cu, FNTRS_CONST_TW): a plain
// load, which compiles to LDC; otherwise a read-only global load.
template <bool CT = false>
__device__ __forceinline__ uint2 tw_at(const uint4* __restrict__ tq, int s, uint4& w4) {
    if (s == 1 || (s & 1) == 0) w4 = CT ? tq[s >> 1] : __ldg(tq + (s >> 1));
    return (s & 1) ? make_uint2(w4.z, w4.w) : make_uint2(w4.x, w4.y);
}

template <int E, int p, bool INV, bool DIT, uint64_t BIN, uint64_t OCAP, class G, class LD, class ST,
          class FIX = NoFix, class FLUSH = NoFlush, int CW = 1, bool CTW = false>
__device__ __forceinline__ void pass(const uint4* __restrict__ twp, const LD& ld, const ST& st, const FIX& fix = FIX(),
                                     const FLUSH& flush = FLUSH()) {
    // CW codewords per work item: columns col + c * WT/CW, c < CW, share the
    // twiddle loads and the address arithmetic (two independent chains at CW = 2)
    using S = Sched<E>;
    constexpr int RL = S::rlog(p), R = 1 << RL, LL = S::llog(p), SL = S::slog(p);
    constexpr int WC = G::WT / CW;
    constexpr int ITEMS = (1 << (E - RL)) * WC;
    constexpr int LGW = ilog2c<WC>();
    static_assert(OCAP >= k2P || OCAP == kCanon, "");
#pragma unroll 1
    for (int it = threadIdx.x; it < ITEMS; it += G::NT) {
        const uint32_t col = uint32_t(it) & uint32_t(WC - 1);
        const uint32_t b = uint32_t(it) >> LGW;
        const uint32_t t = b & ((1u << SL) - 1u);
        const uint32_t base = ((b >> SL) << LL) + t;
        uint32_t v[CW][R];
        const uint4* tq = twp + t * (R / 2);  // row t: r_len^(t s), s < R, two per uint4
        uint32_t acc[CW];
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[c] = 0;
        uint4 w4 = make_uint4(0, 0, 0, 0);
        if constexpr (!DIT) {
#pragma unroll
            for (int c = 0; c < CW; ++c)
#pragma unroll
                for (int q = 0; q < R; ++q) v[c][q] = ld(base + (uint32_t(q) << SL), b, q, col + c * WC);
#pragma unroll
            for (int c = 0; c < CW; ++c) fix(v[c], base, b, col + c * WC);
            // outputs with s > 0 go through a Shoup twiddle (any 32-bit input):
            // the butterfly may leave its w4 products unreduced
            // (a canonical last pass reduces every output anyway: lazy there too, FNTRS_LAZY_LAST)
            constexpr uint64_t LZ = (SL > 0 || (FNTRS_LAZY_LAST && OCAP == kCanon)) ? kLazyLim : 0;
            // FNTRS_SPLIT_PIN: the second codeword of a two-codeword item pins its
            // butterfly adds to the ALU pipe (ptxas balances the first)
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                if (FNTRS_SPLIT_PIN && c == 1)
                    dif_regs<R, INV, BIN, LZ, (FNTRS_CW2_PIN1 & 1) != 0, (FNTRS_CW2_PIN1 & 2) != 0>(v[c]);
                else if (FNTRS_SPLIT_PIN && CW == 2 && FNTRS_CW2_PIN0)
                    dif_regs<R, INV, BIN, LZ, (FNTRS_CW2_PIN0 & 1) != 0, (FNTRS_CW2_PIN0 & 2) != 0>(v[c]);
                else if (CW == 1 && FNTRS_CW1_PIN)
                    dif_regs<R, INV, BIN, LZ, (FNTRS_CW1_PIN & 1) != 0, (FNTRS_CW1_PIN & 2) != 0>(v[c]);
                else
                    dif_regs<R, INV, BIN, LZ>(v[c]);
            }
            constexpr uint64_t BO = dif_bound<R, INV, BIN, LZ>();
#pragma unroll
            for (int s = 0; s < R; ++s) {
                uint2 w = make_uint2(0, 0);
                if (SL > 0 && s > 0) w = tw_at<CTW>(tq, s, w4);
#pragma unroll
                for (int c = 0; c < CW; ++c) {
                    uint32_t y = v[c][rev<R>(s)];
                    if (SL > 0 && s > 0) {
                        y = mulws(y, w.x, w.y);
                        if constexpr (OCAP == kCanon) y = canon_s2p(y);
                    } else {
                        y = cap<BO, OCAP>(y);
                    }
                    const uint32_t r = st(base + (uint32_t(s) << SL), b, s, col + c * WC, y);
                    v[c][rev<R>(s)] = r;
                    acc[c] |= r;
                }
            }
        } else {
            constexpr uint64_t BI = BIN > k2P ? BIN : k2P;
#pragma unroll
            for (int s = 0; s < R; ++s) {
                uint2 w = make_uint2(0, 0);
                if (SL > 0 && s > 0) w = tw_at<CTW>(tq, s, w4);
#pragma unroll
                for (int c = 0; c < CW; ++c) {
                    uint32_t x = ld(base + (uint32_t(s) << SL), b, s, col + c * WC);
                    if (SL > 0 && s > 0) x = mulws(x, w.x, w.y);
                    v[c][rev<R>(s)] = x;
                }
            }
#pragma unroll
            for (int c = 0; c < CW; ++c) {
                if (CW == 1 && FNTRS_CW1_PIN)
                    dit_regs<R, INV, BI, 0, (FNTRS_CW1_PIN & 1) != 0, (FNTRS_CW1_PIN & 2) != 0>(v[c]);
                else
                    dit_regs<R, INV, BI>(v[c]);
            }
            constexpr uint64_t BO = dit_bound<R, INV, BI>();
#pragma unroll
            for (int c = 0; c < CW; ++c)
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const uint32_t r = st(base + (uint32_t(q) << SL), b, q, col + c * WC, cap<BO, OCAP>(v[c][q]));
                    v[c][q] = r;
                    acc[c] |= r;
                }
        }
        // escapes are rare: the store functors return the kept canonical value
        // (0 when not kept), OR-ed per codeword; only a group holding a 65536
        // rebuilds its bit mask from the values parked in v
#pragma unroll
        for (int c = 0; c < CW; ++c) {
            if (acc[c] >> 16) {
                uint32_t mask = 0;
#pragma unroll
                for (int s = 0; s < R; ++s) mask |= ((v[c][DIT ? s : rev<R>(s)] >> 16) & 1u) << s;
                flush(mask, base, b, col + c * WC);
            }
        }
    }
}

// pass with CW codewords per work item (template arguments after G deduced)
template <int CW, int E, int p, bool INV, bool DIT, uint64_t BIN, uint64_t OCAP, class G, class LD, class ST,
          class FIX = NoFix, class FLUSH = NoFlush>
__device__ __forceinline__ void pass_cw(const uint4* __restrict__ twp, const LD& ld, const ST& st,
                                        const FIX& fix = FIX(), const FLUSH& flush = FLUSH()) {
    pass<E, p, INV, DIT, BIN, OCAP, G, LD, ST, FIX, FLUSH, CW>(twp, ld, st, fix, flush);
}

// Per-pass twiddle tables for one direction: table for block length 2^LL at
// uint2 offset 2^LL (LL <= 12): entry t*16 + s = r_len^(t s).
__device__ __forceinline__ const uint4* pass_table(const uint2* base, int LL) {
    return reinterpret_cast<const uint4*>(base + (1u << LL));
}

// Escapes are rare (1 in 65537 symbols): loads and stores test a whole
// butterfly group at once and only a group holding a zero word / a 65536
// takes the slow path (one branch per group instead of one per symbol).
template <int R>
__device__ __forceinline__ bool any_zero(const uint32_t (&v)[R]) {
    uint32_t m = v[0];
#pragma unroll
    for (int i = 1; i < R; ++i) m = min(m, v[i]);
    return m == 0u;
}


}  // namespace
}  // namespace fast
}  // namespace fntrs_gpu
