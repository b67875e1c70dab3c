// codec_large.cu -- encode / decode for 8192 <= n_domain <= 65536 (four-step).
//
// A size-N transform (N = N1*N2, N1 = 2^E1 >= N2 = 2^E2, both <= 256) is
//   X[m1 + N1 m2] = sum_i2 r_N2^(i2 m2) * [ r_N^(i2 m1) * sum_i1 x[i1 N2 + i2] r_N1^(i1 m1) ]
// i.e. N2 transforms of size N1 over stride-N2 rows ("pass A"), a twiddle,
// then N1 transforms of size N2 over contiguous rows ("pass B"). Each CTA
// owns one inner index and 64 adjacent codewords, so every pass is a
// shared-memory tile [size][64] run by the same radix-16 engine as the
// fused kernels, with loads / stores going straight to HBM.
//
// Encode = pass A (zero padding never read) + pass B (natural-order packets).
// Decode (interp::interpolate, proj/src/interp.cpp:103-137) = 3 transforms
// in 4 kernels; the transform boundaries are fused inside CTAs:
//   D1  FNT1 pass A, scatter-loading received packets scaled by 1/A'(x_i)
//   D2  FNT1 pass B + reversal/truncation s'_j = F[N-1-j] + FNT2 pass A
//       (the coset F[m1 + N1 m2], m2 < N2 is exactly s' on i1' = N1-1-m1)
//   D3  FNT2 pass B + (. A_hat) + FNT3 pass A (both on the coset q2 mod N2)
//   D4  FNT3 pass B, writing the k decoded packets.
// Intermediates (uint32, < 2p) go through a stripe-batched HBM scratch.
// q * p as LEA (field.cuh, FNTRS_LEA): C4 decode +0.9 %, C3 encode +1.7 %
#ifndef FNTRS_LEA
#define FNTRS_LEA 1
#endif
// FNTRS_LSTEP: per-symbol HBM addresses are one 64-bit pointer per butterfly
// group stepped by a run-time stride, and four-step twiddle addresses are
// formed with ALU adds (fft_pass.cuh step_ptr / ldg_alu), so that neither
// costs an IMAD.WIDE on the multiplier pipe (83 % busy in enc_a / dec_1).
#ifndef FNTRS_LSTEP
#define FNTRS_LSTEP 1
#endif
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fft_pass.cuh"
#include "tma.cuh"

namespace fntrs_gpu {
namespace fast {

namespace {

constexpr bool kStep = FNTRS_LSTEP != 0;
#ifndef FNTRS_LW
#define FNTRS_LW 64
#endif
#ifndef FNTRS_LMINB
#define FNTRS_LMINB 5  // CTAs per SM the register budget targets at size <= 128 (3 above)
#endif
constexpr int kLW = FNTRS_LW;   // codewords per CTA
constexpr int kLNT = 256;  // threads per CTA

template <int E>
using LG = Geom<E, kLW, kLNT, (1 << E) <= 128 ? FNTRS_LMINB : 3>;

struct BlockIdx {
    uint32_t sb, g, c0;
};

__device__ __forceinline__ BlockIdx block_index(uint32_t tps, uint32_t ng) {
    const uint32_t tile = blockIdx.x;
    const uint32_t ct = tile % tps;
    const uint32_t rest = tile / tps;
    return {rest / ng, rest % ng, ct * kLW};
}

// One unit of work of a four-step pass: inner index g of 64 codewords
// (columns c0..c0+63 of stripe `stripe`), and where the unit's block of the
// uint32 intermediates lives -- element offset of its row 0 / first column,
// and the TMA coordinates of that corner. The batched kernels address a
// [stripes][N][L] scratch (row stride L); the streamed kernel a ring of
// [N][64] slots (row stride 64), LY = 64.
struct Unit {
    uint32_t stripe, g, c0;
    uint64_t yoff;
    uint32_t yx0, yrow0;
};

template <uint32_t N>
__device__ __forceinline__ Unit batch_unit(uint32_t tps, uint32_t ng, uint32_t stripe0, uint32_t L) {
    const BlockIdx bi = block_index(tps, ng);
    return {stripe0 + bi.sb, bi.g, bi.c0, uint64_t(bi.sb) * N * L + bi.c0, bi.c0, bi.sb * N};
}

// A consumed intermediate block is dead: drop its L2 lines without a write
// back (each block is read by exactly one unit, after its TMA load landed).
#ifndef FNTRS_STREAM_DISCARD
#define FNTRS_STREAM_DISCARD 1
#endif
__device__ __forceinline__ void discard_block(const uint32_t* base, uint32_t bytes) {
    if constexpr (!FNTRS_STREAM_DISCARD) return;
    for (uint32_t off = threadIdx.x * 128u; off < bytes; off += kLNT * 128u)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(reinterpret_cast<const char*>(base) + off) : "memory");
}

// The CTA's input block -- ROWS contiguous rows x kLW columns of a uint32
// intermediate -- lands in the shared work tile with one TMA load (row-major,
// the unswizzled 64-wide geometry), so the first pass reads shared memory.
template <int ROWS>
__device__ __forceinline__ void tile_in(uint32_t* work, const CUtensorMap* map, uint32_t c0, uint32_t row0,
                                        uint64_t* bar) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_expect_tx(bar, uint32_t(ROWS) * kLW * 4);
        tma_load_2d(work, map, int(c0), int(row0), bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
}

// ---------------------------------------------------------------- encode ----
template <int E1, int E2, bool HALFK, int LY>
__device__ __forceinline__ void enc_a_body(const uint2* __restrict__ ptab, const uint2* __restrict__ bigF, uint32_t k,
                                           uint32_t L, const uint16_t* __restrict__ src, EscIn esc_in,
                                           uint32_t* __restrict__ Y, const Unit& u) {
    using G = LG<E1>;
    using S = Sched<E1>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    constexpr int R0 = 1 << S::rlog(0), RLZ = G::RLZ;
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t Ly = LY ? uint32_t(LY) : L;
    const uint32_t i2 = u.g, stripe = u.stripe;
    const unsigned long long key_in = uint64_t(stripe) * k * L + u.c0;
    const uint16_t* srcp = launder(src + key_in);
    uint32_t* yp = launder(Y + u.yoff);
    const bool esc_any = esc_in.n != 0;

    const uint16_t* sq = srcp;
    const uint64_t sstep = opaque_stride((uint64_t(N2) * L * 2) << S::slog(0));
    auto ld = [&](uint32_t i1, uint32_t, int q, uint32_t col) -> uint32_t {
        const uint32_t row = i1 * N2 + i2;
        if ((HALFK && q >= R0 / 2) || (!HALFK && row >= k)) return 0u;
        if (!kStep) return srcp[row * L + col];
        sq = q == 0 ? srcp + (row * L + col) : step_ptr(sq, sstep);
        return __ldcs(sq);  // global state space (the laundered pointer would load generically)
    };
    auto fix = [&](uint32_t (&v)[R0], uint32_t base, uint32_t, uint32_t col) {
        if (!esc_any || !any_zero(v)) return;
#pragma unroll
        for (int q = 0; q < R0; ++q) {
            const uint32_t row = (base + (uint32_t(q) << S::slog(0))) * N2 + i2;
            if (v[q] == 0u && row < k && esc_has(esc_in, key_in + uint64_t(row) * L + col)) v[q] = 65536u;
        }
    };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    uint32_t* yq = yp;
    uint32_t tix = 0;
    const uint64_t ystep = opaque_stride((uint64_t(N2) * Ly * 4) << (E1 - RLZ));
    const uint2* bigN = launder(bigF + N);
    auto st_y = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
        if (!kStep) {
            const uint32_t m1 = perm_head<E1>(b) + (uint32_t(s) << (E1 - RLZ));
            const uint2 w = __ldg(bigF + N + ((i2 * m1) & (N - 1)));
            yp[(m1 * N2 + i2) * Ly + col] = mulws(y, w.x, w.y);
            return 0u;
        }
        if (s == 0) {
            const uint32_t m1 = perm_head<E1>(b);
            yq = yp + ((m1 * N2 + i2) * Ly + col);
            tix = i2 * m1;
        } else {
            yq = step_ptr(yq, ystep);
            tix += i2 << (E1 - RLZ);
        }
        const uint2 w = ldg_alu(bigN, tix & (N - 1));
        __stcg(yq, mulws(y, w.x, w.y));
        return 0u;
    };
    pass<E1, 0, false, false, kP64, kSmemCap, G>(pass_table(ptab, S::llog(0)), ld, st_sm, fix);
    __syncthreads();
    pass<E1, 1, false, false, kSmemCap, kSmemCap, G>(pass_table(ptab, S::llog(1)), ld_sm, st_y);
}

template <int E1, int E2, bool HALFK>
__global__ void __launch_bounds__(kLNT, LG<E1>::MINB)
enc_a_kernel(const uint2* __restrict__ ptab, const uint2* __restrict__ bigF, uint32_t k, uint32_t L, uint32_t tps,
             uint32_t stripe0, const uint16_t* __restrict__ src, EscIn esc_in, uint32_t* __restrict__ Y) {
    constexpr uint32_t N = 1u << (E1 + E2);
    enc_a_body<E1, E2, HALFK, 0>(ptab, bigF, k, L, src, esc_in, Y, batch_unit<N>(tps, 1u << E2, stripe0, L));
}

// TS (n == N): the CTA's N2 output rows m1 + N1 m2 are staged in shared memory
// and written by one TMA store through the (L, m1, m2, stripe) view of `out`.
template <int E1, int E2, bool PUNCT, bool TS, int LY>
__device__ __forceinline__ void enc_b_body(const uint2* __restrict__ ptab, uint32_t n, uint32_t L,
                                           const uint32_t* __restrict__ Y, uint16_t* __restrict__ out, EscOut esc_out,
                                           const CUtensorMap* out_map, const CUtensorMap* in_map, const Unit& u) {
    using G = LG<E2>;
    using S = Sched<E2>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2;
    constexpr int RLZ = G::RLZ;
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t Ly = LY ? uint32_t(LY) : L;
    const uint32_t m1 = u.g, stripe = u.stripe;
    const uint32_t* yp = launder(Y + u.yoff + uint64_t(m1 * N2) * Ly);
    const unsigned long long key_out = uint64_t(stripe) * n * L + u.c0;
    uint16_t* outp = launder(out + key_out);

    auto ld = [&](uint32_t i2, uint32_t, int, uint32_t col) -> uint32_t { return yp[i2 * Ly + col]; };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    uint16_t* out_s = reinterpret_cast<uint16_t*>(work + N2 * kLW);  // TS staging: [m2][kLW]
    uint16_t* oq = outp;
    const uint64_t ostep = opaque_stride((uint64_t(N1) * L * 2) << (E2 - RLZ));
    auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
        const uint32_t m2 = perm_head<E2>(b) + (uint32_t(s) << (E2 - RLZ));
        const uint32_t row = m1 + N1 * m2;
        const bool keep = !PUNCT || row < n;
        if constexpr (TS) {
            out_s[m2 * kLW + col] = uint16_t(y);
        } else {
            if (kStep) oq = s == 0 ? outp + (row * L + col) : step_ptr(oq, ostep);
            if (keep) __stcs(kStep ? oq : outp + (row * L + col), uint16_t(y));
        }
        return keep ? y : 0u;  // canonical, kept: bit 16 set iff y == 65536
    };
    auto flush = [&](uint32_t mask, uint32_t, uint32_t b, uint32_t col) {
        if (!mask) return;
#pragma unroll 1
        for (int s = 0; s < 16; ++s)
            if (mask & (1u << s))
                emit_escape(esc_out,
                            key_out + uint64_t(m1 + N1 * (perm_head<E2>(b) + (uint32_t(s) << (E2 - RLZ)))) * L + col);
    };
    __shared__ __align__(8) uint64_t bar;
    tile_in<N2>(work, in_map, u.yx0, u.yrow0 + m1 * N2, &bar);
    if constexpr (LY != 0) discard_block(yp, N2 * kLW * 4);
    (void)ld;
    pass<E2, 0, false, false, k2P, kSmemCap, G>(pass_table(ptab, S::llog(0)), ld_sm, st_sm);
    __syncthreads();
    pass<E2, 1, false, false, kSmemCap, kCanon, G>(pass_table(ptab, S::llog(1)), ld_sm, st_out, NoFix(), flush);
    if constexpr (TS) {
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
            tma_store_4d(out_map, out_s, int(u.c0), int(m1), 0, int(stripe));
            bulk_commit();
            bulk_wait_read();  // the CTA's shared memory must outlive the store's reads
        }
    }
}

template <int E1, int E2, bool PUNCT, bool TS = false>
__global__ void __launch_bounds__(kLNT, (TS ? (E2 <= 7 ? 4 : 2) : LG<E2>::MINB))
enc_b_kernel(const uint2* __restrict__ ptab, uint32_t n, uint32_t L, uint32_t tps, uint32_t stripe0,
             const uint32_t* __restrict__ Y, uint16_t* __restrict__ out, EscOut esc_out,
             const __grid_constant__ CUtensorMap out_map, const __grid_constant__ CUtensorMap in_map) {
    constexpr uint32_t N = 1u << (E1 + E2);
    enc_b_body<E1, E2, PUNCT, TS, 0>(ptab, n, L, Y, out, esc_out, &out_map, &in_map,
                                     batch_unit<N>(tps, 1u << E1, stripe0, L));
}

// ---------------------------------------------------------------- decode ----
template <int E1, int E2, int LY>
__device__ __forceinline__ void dec_1_body(const uint2* __restrict__ ptab, const uint2* __restrict__ bigF,
                                           const uint2* __restrict__ rowmap, uint32_t k, uint32_t L,
                                           const uint32_t* __restrict__ stripe_pattern,
                                           const uint16_t* __restrict__ rx, EscIn esc_in, uint32_t* __restrict__ Y,
                                           const Unit& u) {
    using G = LG<E1>;
    using S = Sched<E1>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    constexpr int R0 = 1 << S::rlog(0), RLZ = G::RLZ;
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t Ly = LY ? uint32_t(LY) : L;
    const uint32_t i2 = u.g, stripe = u.stripe;
    const uint2* __restrict__ rm = rowmap + size_t(__ldg(stripe_pattern + stripe)) * N;
    const unsigned long long key = uint64_t(stripe) * k * L + u.c0;
    const uint16_t* rxp = launder(rx + key);
    uint32_t* yp = launder(Y + u.yoff);
    const bool esc_any = esc_in.n != 0;

    uint32_t zflag = 0;  // a received (non-erased) zero word in this butterfly group
    auto ld = [&](uint32_t i1, uint32_t, int, uint32_t col) -> uint32_t {
        const uint2 m = __ldg(rm + i1 * N2 + i2);  // erased: {~0, 0}
        const uint32_t row = m.x == 0xFFFFFFFFu ? 0u : m.x;
        const uint32_t raw = __ldcs(rxp + (row * L + col));
        zflag |= (raw == 0u) & (m.y != 0u);
        // raw <= 65535, |1/A'| <= p/2 (balanced): the product is exact in 32 signed bits
        return reds(raw * m.y);
    };
    auto fix = [&](uint32_t (&v)[R0], uint32_t base, uint32_t, uint32_t col) {
        const uint32_t any = zflag;
        zflag = 0;
        if (!esc_any || !any) return;
#pragma unroll
        for (int q = 0; q < R0; ++q) {
            if (v[q] != 0u) continue;
            const uint2 m = __ldg(rm + (base + (uint32_t(q) << S::slog(0))) * N2 + i2);
            if (m.x != 0xFFFFFFFFu && rxp[m.x * L + col] == 0u && esc_has(esc_in, key + uint64_t(m.x) * L + col))
                v[q] = mulws(65536u, m.y, m.y * 65535u);
        }
    };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    uint32_t* yq = yp;
    uint32_t tix = 0;
    const uint64_t ystep = opaque_stride((uint64_t(N2) * Ly * 4) << (E1 - RLZ));
    const uint2* bigN = launder(bigF + N);
    auto st_y = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
        if (!kStep) {
            const uint32_t m1 = perm_head<E1>(b) + (uint32_t(s) << (E1 - RLZ));
            const uint2 w = __ldg(bigF + N + ((i2 * m1) & (N - 1)));
            yp[(m1 * N2 + i2) * Ly + col] = mulws(y, w.x, w.y);
            return 0u;
        }
        if (s == 0) {
            const uint32_t m1 = perm_head<E1>(b);
            yq = yp + ((m1 * N2 + i2) * Ly + col);
            tix = i2 * m1;
        } else {
            yq = step_ptr(yq, ystep);
            tix += i2 << (E1 - RLZ);
        }
        const uint2 w = ldg_alu(bigN, tix & (N - 1));
        __stcg(yq, mulws(y, w.x, w.y));
        return 0u;
    };
    pass<E1, 0, false, false, k2P, kSmemCap, G>(pass_table(ptab, S::llog(0)), ld, st_sm, fix);
    __syncthreads();
    pass<E1, 1, false, false, kSmemCap, kSmemCap, G>(pass_table(ptab, S::llog(1)), ld_sm, st_y);
}

template <int E1, int E2>
__global__ void __launch_bounds__(kLNT, LG<E1>::MINB)
dec_1_kernel(const uint2* __restrict__ ptab, const uint2* __restrict__ bigF, const uint2* __restrict__ rowmap,
             uint32_t k, uint32_t L, uint32_t tps, uint32_t stripe0, const uint32_t* __restrict__ stripe_pattern,
             const uint16_t* __restrict__ rx, EscIn esc_in, uint32_t* __restrict__ Y) {
    constexpr uint32_t N = 1u << (E1 + E2);
    dec_1_body<E1, E2, 0>(ptab, bigF, rowmap, k, L, stripe_pattern, rx, esc_in, Y,
                          batch_unit<N>(tps, 1u << E2, stripe0, L));
}

template <int E1, int E2, bool HALFK, int LY>
__device__ __forceinline__ void dec_2_body(const uint2* __restrict__ ptab, const uint2* __restrict__ bigF, uint32_t k,
                                           uint32_t L, const uint32_t* __restrict__ Y1, uint32_t* __restrict__ Y2,
                                           const CUtensorMap* in_map, const Unit& u) {
    using G = LG<E2>;
    using S = Sched<E2>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    constexpr int RLZ = G::RLZ, RZ = 1 << RLZ;
    constexpr uint32_t FLIP = N2 - 1;
    constexpr int LGW = ilog2c<kLW>();
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t Ly = LY ? uint32_t(LY) : L;
    const uint32_t m1 = u.g, i1p = N1 - 1 - m1;
    const uint32_t* y1 = launder(Y1 + u.yoff + uint64_t(m1 * N2) * Ly);
    uint32_t* y2 = launder(Y2 + u.yoff);

    auto ld = [&](uint32_t i2, uint32_t, int, uint32_t col) -> uint32_t { return y1[i2 * Ly + col]; };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto ld_smf = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t {
        return work[G::template idx_flip<FLIP + 1>(lrow, col)];
    };
    uint32_t* yq = y2;
    uint32_t tix = 0;
    const uint64_t ystep = opaque_stride((uint64_t(N1) * Ly * 4) << S::slog(0));
    const uint2* bigN = launder(bigF + N);
    auto st_y2 = [&](uint32_t q2, uint32_t, int q, uint32_t col, uint32_t y) -> uint32_t {
        if (!kStep) {
            const uint2 w = __ldg(bigF + N + ((i1p * q2) & (N - 1)));
            y2[(q2 * N1 + i1p) * Ly + col] = mulws(y, w.x, w.y);
            return 0u;
        }
        if (q == 0) {
            yq = y2 + ((q2 * N1 + i1p) * Ly + col);
            tix = i1p * q2;
        } else {
            yq = step_ptr(yq, ystep);
            tix += i1p << S::slog(0);
        }
        const uint2 w = ldg_alu(bigN, tix & (N - 1));
        __stcg(yq, mulws(y, w.x, w.y));
        return 0u;
    };
    // FNT1 pass B, first radix pass (input block by TMA)
    __shared__ __align__(8) uint64_t bar;
    tile_in<N2>(work, in_map, u.yx0, u.yrow0 + m1 * N2, &bar);
    if constexpr (LY != 0) discard_block(y1, N2 * kLW * 4);
    (void)ld;
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    pass<E2, 0, false, false, k2P, kSmemCap, G>(pass_table(ptab, S::llog(0)), ld_sm, st_sm);
    __syncthreads();
    // FNT1 pass B last radix pass + FNT2 pass A first DIT pass (reversed view over i2' = N2-1-m2,
    // s'_{i1' + N1 i2'} zeroed when i1' + N1 i2' >= k)
    {
        constexpr int ITEMS = (int(N2) / RZ) * kLW;
        // the DIT outputs are folded to 2p for the tile anyway: lazy w4 products (fft_fast.cuh)
        constexpr uint64_t BD = dif_bound<RZ, false, kSmemCap, (1ull << 22)>();
        constexpr uint64_t BT = dit_bound<RZ, false, BD, kLazyLim>();
#pragma unroll 1
        for (int it = threadIdx.x; it < ITEMS; it += kLNT) {
            const uint32_t col = uint32_t(it) & uint32_t(kLW - 1);
            const uint32_t g = uint32_t(it) >> LGW;
            uint32_t v[RZ];
#pragma unroll
            for (int q = 0; q < RZ; ++q) v[q] = work[G::idx((g << RLZ) + q, col)];
            dif_regs<RZ, false, kSmemCap, (1ull << 22)>(v);
            const uint32_t fh = perm_head<E2>(N2 / RZ - 1u - g);
            uint32_t u[RZ];
#pragma unroll
            for (int j = 0; j < RZ; ++j) {
                const uint32_t i2p = fh + (uint32_t(rev<RZ>(j)) << (E2 - RLZ));
                const bool live = HALFK ? ((j & 1) == 0) : (i1p + N1 * i2p < k);
                u[j] = live ? v[RZ - 1 - j] : 0u;
            }
            dit_regs<RZ, false, BD, kLazyLim>(u);
#pragma unroll
            for (int q = 0; q < RZ; ++q) work[G::idx((g << RLZ) + (RZ - 1 - q), col)] = cap<BT, kSmemCap>(u[q]);
        }
    }
    __syncthreads();
    // FNT2 pass A last DIT pass -> natural q2, four-step twiddle r_N^(i1' q2)
    pass<E2, 0, false, true, kSmemCap, kSmemCap, G>(pass_table(ptab, S::llog(0)), ld_smf, st_y2);
}

template <int E1, int E2, bool HALFK>
__global__ void __launch_bounds__(kLNT, LG<E2>::MINB)
dec_2_kernel(const uint2* __restrict__ ptab, const uint2* __restrict__ bigF, uint32_t k, uint32_t L, uint32_t tps,
             const uint32_t* __restrict__ Y1, uint32_t* __restrict__ Y2, const __grid_constant__ CUtensorMap in_map) {
    constexpr uint32_t N = 1u << (E1 + E2);
    dec_2_body<E1, E2, HALFK, 0>(ptab, bigF, k, L, Y1, Y2, &in_map, batch_unit<N>(tps, 1u << E1, 0, L));
}

template <int E1, int E2, int LY>
__device__ __forceinline__ void dec_3_body(const uint2* __restrict__ ptabF, const uint2* __restrict__ ptabI,
                                           const uint2* __restrict__ bigI, const uint2* __restrict__ ahat2, uint32_t L,
                                           const uint32_t* __restrict__ stripe_pattern,
                                           const uint32_t* __restrict__ Y2, uint32_t* __restrict__ Y3,
                                           const CUtensorMap* in_map, const CUtensorMap* out_map, const Unit& u) {
    using G = LG<E1>;
    using S = Sched<E1>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    constexpr int RLZ = G::RLZ, RZ = 1 << RLZ;
    constexpr int LGW = ilog2c<kLW>();
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t Ly = LY ? uint32_t(LY) : L;
    const uint32_t q2 = u.g, stripe = u.stripe;
    const uint2* __restrict__ ah = ahat2 + size_t(__ldg(stripe_pattern + stripe)) * N;
    const uint32_t* y2 = launder(Y2 + u.yoff + uint64_t(q2 * N1) * Ly);
    uint32_t* y3 = launder(Y3 + u.yoff);

    auto ld = [&](uint32_t i1p, uint32_t, int, uint32_t col) -> uint32_t { return y2[i1p * Ly + col]; };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    auto st_y3 = [&](uint32_t t1, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        const uint2 w = __ldg(bigI + N + ((q2 * t1) & (N - 1)));
        y3[(t1 * N2 + q2) * Ly + col] = mulws(y, w.x, w.y);
        return 0u;
    };
    // FNT2 pass B, first radix pass
    __shared__ __align__(8) uint64_t bar;
    tile_in<N1>(work, in_map, u.yx0, u.yrow0 + q2 * N1, &bar);
    if constexpr (LY != 0) discard_block(y2, N1 * kLW * 4);
    (void)ld;
    pass<E1, 0, false, false, k2P, kSmemCap, G>(pass_table(ptabF, S::llog(0)), ld_sm, st_sm);
    __syncthreads();
    // FNT2 pass B last radix pass + (. ahat at q2 + N2 q1) + FNT3 pass A first DIT pass (inverse)
    {
        constexpr int ITEMS = (int(N1) / RZ) * kLW;
        constexpr uint64_t BT = dit_bound<RZ, true, k2P, kLazyLim>();  // folded to 2p for the tile
#pragma unroll 1
        for (int it = threadIdx.x; it < ITEMS; it += kLNT) {
            const uint32_t col = uint32_t(it) & uint32_t(kLW - 1);
            const uint32_t g = uint32_t(it) >> LGW;
            uint32_t v[RZ];
#pragma unroll
            for (int q = 0; q < RZ; ++q) v[q] = work[G::idx((g << RLZ) + q, col)];
            dif_regs<RZ, false, kSmemCap, kLazyLim>(v);  // v[rev(s)] = X2 at q1 = fh + s * N1/RZ (Shoup'd by ahat)
            const uint32_t fh = perm_head<E1>(g);
#pragma unroll
            for (int s = 0; s < RZ; ++s) {
                const uint32_t q1 = fh + (uint32_t(s) << (E1 - RLZ));
                const uint2 a = __ldg(ah + q2 + N2 * q1);
                v[rev<RZ>(s)] = mulws(v[rev<RZ>(s)], a.x, a.y);  // DIT input order: u[rev(s)] = x_s
            }
            dit_regs<RZ, true, k2P, kLazyLim>(v);
#pragma unroll
            for (int q = 0; q < RZ; ++q) work[G::idx((g << RLZ) + q, col)] = cap<BT, kSmemCap>(v[q]);
        }
    }
    __syncthreads();
    // FNT3 pass A last DIT pass (inverse) -> natural t1, twiddle r_N^(-q2 t1). Each item writes
    // back the rows it read, now in natural order: the tile becomes the output block
    // (rows t1 N2 + q2 of Y3), stored with one TMA store through the (L, q2, t1) view.
    (void)st_y3;
    uint32_t tix = 0;
    const uint2* bigN = launder(bigI + N);
    auto st_tile = [&](uint32_t t1, uint32_t, int q, uint32_t col, uint32_t y) -> uint32_t {
        if (!kStep) {
            const uint2 w = __ldg(bigI + N + ((q2 * t1) & (N - 1)));
            work[G::idx(t1, col)] = mulws(y, w.x, w.y);
            return 0u;
        }
        tix = q == 0 ? q2 * t1 : tix + (q2 << S::slog(0));
        const uint2 w = ldg_alu(bigN, tix & (N - 1));
        work[G::idx(t1, col)] = mulws(y, w.x, w.y);
        return 0u;
    };
    pass<E1, 0, true, true, kSmemCap, kSmemCap, G>(pass_table(ptabI, S::llog(0)), ld_sm, st_tile);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
        tma_store_3d(out_map, work, int(u.yx0), int(q2), int(u.yrow0 / N2));
        bulk_commit();
        bulk_wait_read();
    }
}

template <int E1, int E2>
__global__ void __launch_bounds__(kLNT, LG<E1>::MINB)
dec_3_kernel(const uint2* __restrict__ ptabF, const uint2* __restrict__ ptabI, const uint2* __restrict__ bigI,
             const uint2* __restrict__ ahat2, uint32_t L, uint32_t tps, uint32_t stripe0,
             const uint32_t* __restrict__ stripe_pattern, const uint32_t* __restrict__ Y2, uint32_t* __restrict__ Y3,
             const __grid_constant__ CUtensorMap in_map, const __grid_constant__ CUtensorMap out_map) {
    constexpr uint32_t N = 1u << (E1 + E2);
    dec_3_body<E1, E2, 0>(ptabF, ptabI, bigI, ahat2, L, stripe_pattern, Y2, Y3, &in_map, &out_map,
                          batch_unit<N>(tps, 1u << E2, stripe0, L));
}

template <int E1, int E2, bool HALFK, int LY>
__device__ __forceinline__ void dec_4_body(const uint2* __restrict__ ptabI, uint32_t k, uint32_t L,
                                           const uint32_t* __restrict__ Y3, uint16_t* __restrict__ out,
                                           EscOut esc_out, const CUtensorMap* in_map, const Unit& u) {
    using G = LG<E2>;
    using S = Sched<E2>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2;
    constexpr int RLZ = G::RLZ, RZ = 1 << RLZ;
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t Ly = LY ? uint32_t(LY) : L;
    const uint32_t t1 = u.g, stripe = u.stripe;
    const uint32_t* y3 = launder(Y3 + u.yoff + uint64_t(t1 * N2) * Ly);
    const unsigned long long key = uint64_t(stripe) * k * L + u.c0;
    uint16_t* outp = launder(out + key);

    auto ld = [&](uint32_t i2, uint32_t, int, uint32_t col) -> uint32_t { return y3[i2 * Ly + col]; };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    uint16_t* oq = outp;
    const uint64_t ostep = opaque_stride((uint64_t(N1) * L * 2) << (E2 - RLZ));
    auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
        const uint32_t row = t1 + N1 * (perm_head<E2>(b) + (uint32_t(s) << (E2 - RLZ)));
        const bool keep = HALFK ? (s < RZ / 2) : (row < k);
        if (kStep) oq = s == 0 ? outp + (row * L + col) : step_ptr(oq, ostep);
        if (keep) __stcs(kStep ? oq : outp + (row * L + col), uint16_t(y));
        return keep ? y : 0u;  // canonical, kept: bit 16 set iff y == 65536
    };
    auto flush = [&](uint32_t mask, uint32_t, uint32_t b, uint32_t col) {
        if (!mask) return;
#pragma unroll 1
        for (int s = 0; s < 16; ++s)
            if (mask & (1u << s))
                emit_escape(esc_out, key + uint64_t(t1 + N1 * (perm_head<E2>(b) + (uint32_t(s) << (E2 - RLZ)))) * L + col);
    };
    __shared__ __align__(8) uint64_t bar;
    tile_in<N2>(work, in_map, u.yx0, u.yrow0 + t1 * N2, &bar);
    if constexpr (LY != 0) discard_block(y3, N2 * kLW * 4);
    (void)ld;
    pass<E2, 0, true, false, k2P, kSmemCap, G>(pass_table(ptabI, S::llog(0)), ld_sm, st_sm);
    __syncthreads();
    pass<E2, 1, true, false, kSmemCap, kCanon, G>(pass_table(ptabI, S::llog(1)), ld_sm, st_out, NoFix(), flush);
}

template <int E1, int E2, bool HALFK>
__global__ void __launch_bounds__(kLNT, LG<E2>::MINB)
dec_4_kernel(const uint2* __restrict__ ptabI, uint32_t k, uint32_t L, uint32_t tps, uint32_t stripe0,
             const uint32_t* __restrict__ Y3, uint16_t* __restrict__ out, EscOut esc_out,
             const __grid_constant__ CUtensorMap in_map) {
    constexpr uint32_t N = 1u << (E1 + E2);
    dec_4_body<E1, E2, HALFK, 0>(ptabI, k, L, Y3, out, esc_out, &in_map, batch_unit<N>(tps, 1u << E1, stripe0, L));
}

// ------------------------------------------------------- streamed (L2) ----
// One persistent launch runs every pass of every column block (64 codewords
// of one stripe) with the uint32 intermediates in rings of R [N][64] slots
// that stay in L2, instead of [stripes][N][L] HBM scratch between launches.
// Units (phase, column block cb, inner index g) are claimed in ticket order
// from one counter; step s of the order holds, last phase first, the units of
// phase p for cb = s - (p-1) D. A unit waits (acquire spin) until
//   * phase p-1 of its cb has finished (the transpose needs every unit), and
//   * phase p+1 of cb - R has finished (it read the ring slot cb reuses);
// both were claimed earlier (D < R), and units only wait on earlier tickets,
// so the schedule cannot deadlock. done[p][cb] counts finished units.
__device__ __forceinline__ void wait_at_least(const uint32_t* p, uint32_t target) {
    uint32_t v;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v >= target) break;
        __nanosleep(128);
    }
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// Ticket claims, one ahead: the CTA claims its next unit as it starts the
// current one, so the atomic's round trip overlaps the work. (Still no
// deadlock: the smallest ticket being worked on only waits on smaller
// tickets, and none of those can be a claimed-but-unstarted one.)
struct Claims {
    uint32_t* ticket;
    uint32_t* s;  // two shared slots, used alternately
    uint32_t it = 0;
    __device__ __forceinline__ uint32_t first() {
        if (threadIdx.x == 0) s[0] = atomicAdd(ticket, 1u);
        __syncthreads();
        return s[0];
    }
    // thread 0 claims the following ticket into the other slot; every thread read
    // that slot's previous ticket before the barriers of the current unit
    __device__ __forceinline__ void prefetch() {
        if (threadIdx.x == 0) s[(it + 1) & 1u] = atomicAdd(ticket, 1u);
    }
    // after a barrier that followed prefetch()
    __device__ __forceinline__ uint32_t next() {
        ++it;
        return s[it & 1u];
    }
};

// every thread's global writes of the unit, then one count: the barrier
// orders the CTA's writes before thread 0's gpu-scope fence, which is
// cumulative, then the counter update (the release pattern of CUTLASS's
// semaphore). The same barrier publishes the prefetched ticket.
__device__ __forceinline__ void unit_done(uint32_t* counter, bool tma_stored) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (tma_stored) {
            bulk_wait_all();  // the unit's TMA store has landed in global memory
            fence_proxy_async_global();
        }
        __threadfence();
        atomicAdd(counter, 1u);
    }
}

template <int E1, int E2>
struct StreamGeom {
    static constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    static constexpr int MINB = LG<(E1 > E2 ? E1 : E2)>::MINB;
};

template <int E1, int E2, bool HALFK, bool PUNCT>
__global__ void __launch_bounds__(kLNT, StreamGeom<E1, E2>::MINB)
enc_stream_kernel(const uint2* __restrict__ ptab, const uint2* __restrict__ bigF, uint32_t k, uint32_t n, uint32_t L,
                  uint32_t tps, int tsh, uint32_t ncb, uint32_t R, uint32_t D, const uint16_t* __restrict__ src,
                  EscIn esc_in,
                  uint16_t* __restrict__ out, EscOut esc_out, uint32_t* __restrict__ Y, uint32_t* __restrict__ ctl,
                  const __grid_constant__ CUtensorMap out_map, const __grid_constant__ CUtensorMap in_map) {
    using SG = StreamGeom<E1, E2>;
    constexpr uint32_t N1 = SG::N1, N2 = SG::N2, N = SG::N, U = N1 + N2;
    uint32_t* done1 = ctl + 1;
    uint32_t* done2 = done1 + ncb;
    const uint32_t total = (ncb + D) * U;
    __shared__ uint32_t s_tk[2];
    Claims cl{ctl, s_tk};
    for (uint32_t t = cl.first(); t < total; t = cl.next()) {
        cl.prefetch();
        const uint32_t step = t / U, r = t - step * U;
        const bool p2 = r < N1;  // [phase 2: N1 units][phase 1: N2 units]
        const uint32_t g = p2 ? r : r - N1;
        const uint32_t cb = p2 ? step - D : step;
        if ((p2 && step < D) || cb >= ncb) {  // outside the schedule: publish the next ticket only
            __syncthreads();
            continue;
        }
        const uint32_t slot = cb & (R - 1u);  // R is a power of two
        const uint32_t stripe = tsh >= 0 ? cb >> tsh : cb / tps, ct = cb - stripe * tps;
        const Unit u{stripe, g, ct * kLW, uint64_t(slot) * N * kLW, 0u, slot * N};
        if (threadIdx.x == 0) {
            if (p2) {
                wait_at_least(done1 + cb, N2);
                fence_proxy_async_global();
            } else if (cb >= R) {
                wait_at_least(done2 + cb - R, N1);
            }
        }
        __syncthreads();
        if (p2) {
            enc_b_body<E1, E2, PUNCT, false, kLW>(ptab, n, L, Y, out, esc_out, &out_map, &in_map, u);
            unit_done(done2 + cb, false);
        } else {
            enc_a_body<E1, E2, HALFK, kLW>(ptab, bigF, k, L, src, esc_in, Y, u);
            unit_done(done1 + cb, false);
        }
    }
}

template <int E1, int E2, bool HALFK>
__global__ void __launch_bounds__(kLNT, StreamGeom<E1, E2>::MINB)
dec_stream_kernel(const uint2* __restrict__ ptabF, const uint2* __restrict__ ptabI, const uint2* __restrict__ bigF,
                  const uint2* __restrict__ bigI, const uint2* __restrict__ rowmap, const uint2* __restrict__ ahat2,
                  uint32_t k, uint32_t L, uint32_t tps, int tsh, uint32_t ncb, uint32_t R, uint32_t D,
                  const uint32_t* __restrict__ stripe_pattern, const uint16_t* __restrict__ rx, EscIn esc_in,
                  uint16_t* __restrict__ out, EscOut esc_out, uint32_t* __restrict__ Y1, uint32_t* __restrict__ Y2,
                  uint32_t* __restrict__ Y3, uint32_t* __restrict__ ctl, const __grid_constant__ CUtensorMap map1,
                  const __grid_constant__ CUtensorMap map2, const __grid_constant__ CUtensorMap map3o,
                  const __grid_constant__ CUtensorMap map3) {
    using SG = StreamGeom<E1, E2>;
    constexpr uint32_t N1 = SG::N1, N2 = SG::N2, N = SG::N, U = 2 * (N1 + N2);
    uint32_t* done = ctl + 1;  // done[(p - 1) * ncb + cb]
    const uint32_t total = (ncb + 3 * D) * U;
    __shared__ uint32_t s_tk[2];
    Claims cl{ctl, s_tk};
    for (uint32_t t = cl.first(); t < total; t = cl.next()) {
        cl.prefetch();
        const uint32_t step = t / U, r = t - step * U;
        // [phase 4: N1][phase 3: N2][phase 2: N1][phase 1: N2]
        uint32_t p, g;
        if (r < N1) p = 4, g = r;
        else if (r < N1 + N2) p = 3, g = r - N1;
        else if (r < 2 * N1 + N2) p = 2, g = r - N1 - N2;
        else p = 1, g = r - 2 * N1 - N2;
        const uint32_t lag = (p - 1) * D;
        const uint32_t cb = step - lag;
        if (step < lag || cb >= ncb) {  // outside the schedule: publish the next ticket only
            __syncthreads();
            continue;
        }
        const uint32_t slot = cb & (R - 1u);  // R is a power of two
        const uint32_t stripe = tsh >= 0 ? cb >> tsh : cb / tps, ct = cb - stripe * tps;
        const Unit u{stripe, g, ct * kLW, uint64_t(slot) * N * kLW, 0u, slot * N};
        if (threadIdx.x == 0) {
            if (p > 1) wait_at_least(done + (p - 2) * ncb + cb, (p - 1) % 2 ? N2 : N1);  // phases 1, 3: N2 units
            if (p < 4 && cb >= R) wait_at_least(done + p * ncb + cb - R, (p + 1) % 2 ? N2 : N1);
            fence_proxy_async_global();
        }
        __syncthreads();
        switch (p) {
            case 1:
                dec_1_body<E1, E2, kLW>(ptabF, bigF, rowmap, k, L, stripe_pattern, rx, esc_in, Y1, u);
                break;
            case 2:
                dec_2_body<E1, E2, HALFK, kLW>(ptabF, bigF, k, L, Y1, Y2, &map1, u);
                break;
            case 3:
                dec_3_body<E1, E2, kLW>(ptabF, ptabI, bigI, ahat2, L, stripe_pattern, Y2, Y3, &map2, &map3o, u);
                break;
            default:
                dec_4_body<E1, E2, HALFK, kLW>(ptabI, k, L, Y3, out, esc_out, &map3, u);
                break;
        }
        unit_done(done + (p - 1) * ncb + cb, p == 3);
    }
}

// (L, m1, m2, stripe) view of an unpunctured output [stripes][N1 N2][L]: row m1 + N1 m2
cudaError_t make_rows_map(CUtensorMap* map, void* base, uint64_t stripes, uint32_t N1, uint32_t N2, uint32_t L) {
    typedef CUresult (*Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<Fn>(p);
    }
    if (!fn || N2 > 256) return cudaErrorNotSupported;
    const cuuint64_t dims[4] = {L, N1, N2, stripes};
    const cuuint64_t strides[3] = {cuuint64_t(L) * 2, cuuint64_t(L) * N1 * 2, cuuint64_t(L) * N1 * N2 * 2};
    const cuuint32_t box[4] = {uint32_t(kLW), 1, N2, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 2-D map over a uint32 intermediate [rows][L], box [box_rows][kLW]
cudaError_t make_u32_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t L, uint32_t box_rows) {
    typedef CUresult (*Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<Fn>(p);
    }
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {L, rows};
    const cuuint64_t strides[1] = {cuuint64_t(L) * 4};
    const cuuint32_t box[2] = {uint32_t(kLW), box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// (L, inner, outer) view of a uint32 intermediate [rows][L] with row = outer * n_inner + inner:
// box {kLW, 1, box_outer} -- a strided set of rows
cudaError_t make_u32_strided_map(CUtensorMap* map, void* base, uint64_t outer, uint32_t n_inner, uint32_t L,
                                 uint32_t box_outer) {
    typedef CUresult (*Fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<Fn>(p);
    }
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {L, n_inner, outer};
    const cuuint64_t strides[2] = {cuuint64_t(L) * 4, cuuint64_t(L) * n_inner * 4};
    const cuuint32_t box[3] = {uint32_t(kLW), 1, box_outer};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class K>
cudaError_t prep(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

template <int E1, int E2>
cudaError_t run_encode(const FastTables& t, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L, const uint16_t* src,
                       EscIn ein, uint16_t* out, EscOut eout, uint32_t* Y, uint32_t batch, cudaStream_t st) {
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    const uint32_t tps = L / kLW;
    const size_t smA = size_t(N1) * kLW * 4, smB = size_t(N2) * kLW * 4;
    const bool half = k == N / 2, punct = n < N;
    auto ka = half ? enc_a_kernel<E1, E2, true> : enc_a_kernel<E1, E2, false>;
    // unpunctured: staged rows + one TMA store per CTA through the (L, m1, m2, stripe) view
    CUtensorMap omap;
    std::memset(&omap, 0, sizeof(omap));
    // (with 256-row halves the staging costs a CTA per SM: C3 encode 246 -> 229 GB/s, so not there)
    const bool ts = !punct && E2 <= 7 && make_rows_map(&omap, out, stripes, N1, N2, L) == cudaSuccess;
    auto kb = punct ? enc_b_kernel<E1, E2, true> : (ts ? enc_b_kernel<E1, E2, false, true> : enc_b_kernel<E1, E2, false>);
    const size_t smBk = smB + (ts ? size_t(N2) * kLW * 2 : 0);
    cudaError_t err;
    if ((err = prep(ka, smA)) || (err = prep(kb, smBk))) return err;
    CUtensorMap ymap;  // kb's input blocks: N2 rows of Y
    if ((err = make_u32_map(&ymap, Y, uint64_t(batch) * N, L, N2))) return err;
    for (uint32_t s0 = 0; s0 < stripes; s0 += batch) {
        const uint32_t sb = stripes - s0 < batch ? stripes - s0 : batch;
        ka<<<sb * N2 * tps, kLNT, smA, st>>>(t.ptab_fwd, t.big_fwd, k, L, tps, s0, src, ein, Y);
        kb<<<sb * N1 * tps, kLNT, smBk, st>>>(t.ptab_fwd, n, L, tps, s0, Y, out, eout, omap, ymap);
    }
    return cudaGetLastError();
}

template <int E1, int E2>
cudaError_t run_decode(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L, const uint32_t* sp,
                       const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout, uint32_t* YA, uint32_t* YB,
                       uint32_t batch, cudaStream_t st) {
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    const uint32_t tps = L / kLW;
    const size_t sm1 = size_t(N1) * kLW * 4, sm2 = size_t(N2) * kLW * 4;
    const bool half = pv.k == N / 2;
    auto k1 = dec_1_kernel<E1, E2>;
    auto k2 = half ? dec_2_kernel<E1, E2, true> : dec_2_kernel<E1, E2, false>;
    auto k3 = dec_3_kernel<E1, E2>;
    auto k4 = half ? dec_4_kernel<E1, E2, true> : dec_4_kernel<E1, E2, false>;
    cudaError_t err;
    if ((err = prep(k1, sm1)) || (err = prep(k2, sm2)) || (err = prep(k3, sm1)) || (err = prep(k4, sm2))) return err;
    CUtensorMap mapA, mapB, map3;  // input blocks: N2 rows of YA (k2, k4), N1 rows of YB (k3); k3's output view
    if ((err = make_u32_map(&mapA, YA, uint64_t(batch) * N, L, N2)) || (err = make_u32_map(&mapB, YB, uint64_t(batch) * N, L, N1)) ||
        (err = make_u32_strided_map(&map3, YA, uint64_t(batch) * N1, N2, L, N1)))
        return err;
    for (uint32_t s0 = 0; s0 < stripes; s0 += batch) {
        const uint32_t sb = stripes - s0 < batch ? stripes - s0 : batch;
        k1<<<sb * N2 * tps, kLNT, sm1, st>>>(t.ptab_fwd, t.big_fwd, pv.rowmap, pv.k, L, tps, s0, sp, rx, ein, YA);
        k2<<<sb * N1 * tps, kLNT, sm2, st>>>(t.ptab_fwd, t.big_fwd, pv.k, L, tps, YA, YB, mapA);
        k3<<<sb * N2 * tps, kLNT, sm1, st>>>(t.ptab_fwd, t.ptab_inv, t.big_inv, pv.ahat2, L, tps, s0, sp, YB, YA, mapB,
                                              map3);
        k4<<<sb * N1 * tps, kLNT, sm2, st>>>(t.ptab_inv, pv.k, L, tps, s0, YA, out, eout, mapA);
    }
    return cudaGetLastError();
}

// ring depth R and phase lag D (column blocks) of the streamed kernels: the
// rings (3 for decode, 1 for encode) of R slots of N x 64 words stay well
// inside the 126 MB L2 (C4, N = 16384: 4 MB a slot; C3, N = 65536: 16 MB)
struct StreamShape {
    uint32_t R, D;
};
int pow2_shift(uint32_t v) {  // log2(v) for a power of two, else -1
    return v && !(v & (v - 1)) ? 31 - __builtin_clz(v) : -1;
}

StreamShape stream_shape(uint32_t N, bool decode) {
    if (const char* e = std::getenv("FNTRS_STREAM_RD")) {  // "R,D" override (A/B); R a power of two
        unsigned r = 0, d = 0;
        if (std::sscanf(e, "%u,%u", &r, &d) == 2 && d < r && pow2_shift(r) >= 0) return {r, d};
    }
    if (N <= 16384) return {8, 4};  // C4: 3 rings x 8 slots x 4 MB = 96 MB of L2
    return decode ? StreamShape{2, 1} : StreamShape{4, 2};
}

template <class K>
cudaError_t stream_grid(K kernel, size_t smem, uint32_t& grid) {
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (!e) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (!e) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kLNT, smem);
    grid = uint32_t(sms) * uint32_t(occ > 0 ? occ : 1);
    return e;
}

template <int E1, int E2>
cudaError_t stream_encode(const FastTables& t, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                          const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, uint32_t* Y, uint32_t* ctl,
                          StreamShape sh, cudaStream_t st) {
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    const uint32_t tps = L / kLW, ncb = stripes * tps;
    const size_t sm = size_t(N1 > N2 ? N1 : N2) * kLW * 4;
    const bool half = k == N / 2, punct = n < N;
    auto kern = half ? (punct ? enc_stream_kernel<E1, E2, true, true> : enc_stream_kernel<E1, E2, true, false>)
                     : (punct ? enc_stream_kernel<E1, E2, false, true> : enc_stream_kernel<E1, E2, false, false>);
    cudaError_t err;
    if ((err = prep(kern, sm))) return err;
    CUtensorMap omap, ymap;
    std::memset(&omap, 0, sizeof(omap));
    if ((err = make_u32_map(&ymap, Y, uint64_t(sh.R) * N, kLW, N2))) return err;
    if ((err = cudaMemsetAsync(ctl, 0, (1 + 2 * size_t(ncb)) * 4, st))) return err;
    uint32_t grid = 0;
    if ((err = stream_grid(kern, sm, grid))) return err;
    kern<<<grid, kLNT, sm, st>>>(t.ptab_fwd, t.big_fwd, k, n, L, tps, pow2_shift(tps), ncb, sh.R, sh.D, src, ein, out,
                                 eout, Y, ctl, omap, ymap);
    return cudaGetLastError();
}

template <int E1, int E2>
cudaError_t stream_decode(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                          const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                          uint32_t* Y, uint32_t* ctl, StreamShape sh, cudaStream_t st) {
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    const uint32_t tps = L / kLW, ncb = stripes * tps;
    const size_t sm = size_t(N1 > N2 ? N1 : N2) * kLW * 4;
    auto kern = pv.k == N / 2 ? dec_stream_kernel<E1, E2, true> : dec_stream_kernel<E1, E2, false>;
    cudaError_t err;
    if ((err = prep(kern, sm))) return err;
    const uint64_t ring = uint64_t(sh.R) * N * kLW;
    uint32_t *Y1 = Y, *Y2 = Y + ring, *Y3 = Y + 2 * ring;
    CUtensorMap m1, m2, m3o, m3;  // D2 reads N2-row blocks of Y1, D3 N1-row blocks of Y2 and writes
                                  // Y3 rows t1 N2 + q2 (strided view), D4 reads N2-row blocks of Y3
    if ((err = make_u32_map(&m1, Y1, uint64_t(sh.R) * N, kLW, N2)) ||
        (err = make_u32_map(&m2, Y2, uint64_t(sh.R) * N, kLW, N1)) ||
        (err = make_u32_strided_map(&m3o, Y3, uint64_t(sh.R) * N1, N2, kLW, N1)) ||
        (err = make_u32_map(&m3, Y3, uint64_t(sh.R) * N, kLW, N2)))
        return err;
    if ((err = cudaMemsetAsync(ctl, 0, (1 + 4 * size_t(ncb)) * 4, st))) return err;
    uint32_t grid = 0;
    if ((err = stream_grid(kern, sm, grid))) return err;
    kern<<<grid, kLNT, sm, st>>>(t.ptab_fwd, t.ptab_inv, t.big_fwd, t.big_inv, pv.rowmap, pv.ahat2, pv.k, L, tps,
                                 pow2_shift(tps), ncb, sh.R, sh.D, sp, rx, ein, out, eout, Y1, Y2, Y3, ctl, m1, m2, m3o, m3);
    return cudaGetLastError();
}

__global__ void big_tables_kernel(uint2* fwd, uint2* inv) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 || i >= (1u << 17)) return;
    const int e = 31 - __clz(i);
    const uint32_t j = i - (1u << e);
    const uint32_t ex = (j << (16 - e)) & 0xFFFFu;
    const int32_t wf = balanced(gpow(3u, ex)), wi = balanced(gpow(3u, (65536u - ex) & 0xFFFFu));
    fwd[i] = make_uint2(uint32_t(wf), uint32_t(wf * 65535));
    inv[i] = make_uint2(uint32_t(wi), uint32_t(wi * 65535));
}

}  // namespace

cudaError_t build_large_tables(FastTables& t, cudaStream_t st) {
    cudaError_t err = cudaMalloc(&t.big_fwd, sizeof(uint2) << 17);
    if (err) return err;
    if ((err = cudaMalloc(&t.big_inv, sizeof(uint2) << 17))) return err;
    big_tables_kernel<<<(1u << 17) / 256, 256, 0, st>>>(t.big_fwd, t.big_inv);
    return cudaGetLastError();
}

int large_supported(uint32_t N) { return N >= 8192 && N <= 65536 && (N & (N - 1)) == 0; }
uint32_t large_tile_columns() { return kLW; }

uint32_t large_batch(uint32_t N, uint32_t L, size_t scratch_bytes) {
    const size_t per = size_t(N) * L * 4;
    const size_t b = scratch_bytes / per;
    return b < 1 ? 1u : (b > 0xFFFFu ? 0xFFFFu : uint32_t(b));
}

cudaError_t launch_encode_large(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes, uint32_t L,
                                const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, uint32_t* Y,
                                uint32_t batch, cudaStream_t st) {
    switch (N) {
        case 8192: return run_encode<7, 6>(t, k, n, stripes, L, src, ein, out, eout, Y, batch, st);
        case 16384: return run_encode<7, 7>(t, k, n, stripes, L, src, ein, out, eout, Y, batch, st);
        case 32768: return run_encode<8, 7>(t, k, n, stripes, L, src, ein, out, eout, Y, batch, st);
        case 65536: return run_encode<8, 8>(t, k, n, stripes, L, src, ein, out, eout, Y, batch, st);
        default: return cudaErrorInvalidValue;
    }
}

// Off by default: measured slower than the batched kernels although its DRAM
// traffic is ~1.5x algorithmic instead of ~7x (C4 decode 131 vs 147 GB/s,
// encode 346 vs 415; C3 decode 118 vs 135): the four-step kernels are bound
// by instruction issue, not HBM, and the transpose dependencies add barrier
// stalls (every unit of a pass must finish before any of the next starts on
// that column block). FNTRS_STREAM=1 selects it (profiles/README.md).
bool stream_enabled() {
    const char* e = std::getenv("FNTRS_STREAM");
    return e && e[0] == '1';
}

size_t stream_scratch_words(uint32_t N, uint32_t stripes, uint32_t L, bool decode) {
    const StreamShape sh = stream_shape(N, decode);
    const uint64_t ncb = uint64_t(stripes) * (L / kLW);
    return size_t(decode ? 3 : 1) * sh.R * N * kLW + 1 + (decode ? 4 : 2) * ncb + 64;
}

cudaError_t launch_encode_stream(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes,
                                 uint32_t L, const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout,
                                 uint32_t* scratch, cudaStream_t st) {
    const StreamShape sh = stream_shape(N, false);
    uint32_t* ctl = scratch + size_t(sh.R) * N * kLW;
    switch (N) {
        case 8192: return stream_encode<7, 6>(t, k, n, stripes, L, src, ein, out, eout, scratch, ctl, sh, st);
        case 16384: return stream_encode<7, 7>(t, k, n, stripes, L, src, ein, out, eout, scratch, ctl, sh, st);
        case 32768: return stream_encode<8, 7>(t, k, n, stripes, L, src, ein, out, eout, scratch, ctl, sh, st);
        case 65536: return stream_encode<8, 8>(t, k, n, stripes, L, src, ein, out, eout, scratch, ctl, sh, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_decode_stream(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                                 const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                                 uint32_t* scratch, cudaStream_t st) {
    const StreamShape sh = stream_shape(pv.N, true);
    uint32_t* ctl = scratch + 3 * size_t(sh.R) * pv.N * kLW;
    switch (pv.N) {
        case 8192: return stream_decode<7, 6>(t, pv, stripes, L, sp, rx, ein, out, eout, scratch, ctl, sh, st);
        case 16384: return stream_decode<7, 7>(t, pv, stripes, L, sp, rx, ein, out, eout, scratch, ctl, sh, st);
        case 32768: return stream_decode<8, 7>(t, pv, stripes, L, sp, rx, ein, out, eout, scratch, ctl, sh, st);
        case 65536: return stream_decode<8, 8>(t, pv, stripes, L, sp, rx, ein, out, eout, scratch, ctl, sh, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_decode_large(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                                const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                                uint32_t* YA, uint32_t* YB, uint32_t batch, cudaStream_t st) {
    switch (pv.N) {
        case 8192: return run_decode<7, 6>(t, pv, stripes, L, sp, rx, ein, out, eout, YA, YB, batch, st);
        case 16384: return run_decode<7, 7>(t, pv, stripes, L, sp, rx, ein, out, eout, YA, YB, batch, st);
        case 32768: return run_decode<8, 7>(t, pv, stripes, L, sp, rx, ein, out, eout, YA, YB, batch, st);
        case 65536: return run_decode<8, 8>(t, pv, stripes, L, sp, rx, ein, out, eout, YA, YB, batch, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fast
}  // namespace fntrs_gpu
