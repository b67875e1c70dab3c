// codec_fast.cu -- v2 fused encode / decode kernels for 32 <= n_domain <= 4096.
//
// One CTA = one tile (stripe, WT = 2*NPAIR adjacent codewords); one work item
// = one radix-R butterfly for a pair of adjacent codewords (one uint32 of two
// uint16 symbols in global memory, one uint2 in shared memory).
//
// Encode  (codec::encode_nonsystematic, proj/src/codec.cpp:124-131):
//   pass 0 reads the k source packets straight from global memory (rows >= k
//   are the zero padding and are never loaded), the middle passes run in
//   shared memory, the last pass writes the n output packets straight to
//   global memory in natural order, canonical, with 65536 escapes emitted.
// Decode  (interp::interpolate, proj/src/interp.cpp:103-137, per codeword):
//   FNT1 (DIF, fwd)  pass 0 scatters the k received packets to their
//                    positions and scales them by 1/A'(x_i) while loading;
//   FNT1 last pass + FNT2 first DIT pass fused in registers: the series
//                    s'_j = F[N-1-j] is a reversal of the butterfly group,
//                    coefficients j >= k are zeroed in registers;
//   FNT2 last DIT pass + (. A_hat) + FNT3 first DIF pass fused in registers;
//   FNT3 (DIF, inv)  last pass writes the k decoded packets to global memory.
// Shared memory holds the tile between passes only; HBM traffic is the
// algorithmic 2k B in + 2n (encode) / 2k (decode) B out per codeword.
#include <cuda_runtime.h>

#include "fft_fast.cuh"
#include "internal.h"

namespace fntrs_gpu {
namespace fast {

namespace {

constexpr uint64_t kSmemCap = 1ull << 20;  // bound of values kept in shared memory
constexpr uint64_t k2P = 2 * kP64;

__device__ __forceinline__ bool esc_has(const EscIn& e, unsigned long long key) {
    uint64_t lo = 0, hi = e.n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (e.keys[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo < e.n && e.keys[lo] == key;
}

__device__ __forceinline__ void emit_escape(const EscOut& e, unsigned long long key) {
    const unsigned long long i = atomicAdd(e.count, 1ull);
    if (i < e.cap) e.keys[i] = key;
}

// two uint16 symbols -> two field values (escapes restored)
__device__ __forceinline__ void unpack2(uint32_t w, const EscIn& esc, unsigned long long key0, uint32_t& x0,
                                        uint32_t& x1) {
    x0 = w & 0xFFFFu;
    x1 = w >> 16;
    if (esc.n && (x0 == 0u || x1 == 0u)) {
        if (x0 == 0u && esc_has(esc, key0)) x0 = 65536u;
        if (x1 == 0u && esc_has(esc, key0 + 1)) x1 = 65536u;
    }
}

// two values < 2p -> packed canonical uint16 pair; escapes emitted
__device__ __forceinline__ uint32_t pack2(uint32_t y0, uint32_t y1, const EscOut& esc, unsigned long long key0) {
    y0 = red2p(y0);
    y1 = red2p(y1);
    if (y0 == 65536u || y1 == 65536u) {
        if (y0 == 65536u) emit_escape(esc, key0);
        if (y1 == 65536u) emit_escape(esc, key0 + 1);
    }
    return (y0 & 0xFFFFu) | (y1 << 16);
}

// Shared-memory tile [N][NPAIR] uint2 with an XOR swizzle on the pair index
// that keeps the sub = 1 passes (rows 16b + q) free of bank conflicts.
template <int E, int NPAIR>
struct Tile {
    static constexpr int SW = Sched<E>::rlog(Sched<E>::P - 1);
    uint2* sm;
    __device__ __forceinline__ uint2& at(uint32_t prow, int pair) const {
        return sm[prow * NPAIR + (pair ^ int((prow >> SW) & (NPAIR - 1)))];
    }
};

template <int N>
constexpr int ilog2c() {
    int e = 0;
    while ((1 << e) < N) ++e;
    return e;
}

// Reduce v (bound B) so that it is below CAP.
template <uint64_t B, uint64_t CAP>
__device__ __forceinline__ uint32_t cap(uint32_t v) {
    if constexpr (B > CAP)
        return red(v);
    else
        return v;
}

// ---- generic pass -----------------------------------------------------------
// DIF (DIT=false) or DIT pass with the geometry of DIF pass p of a size-2^E
// transform. Loaded values must be below BIN; stored values are below OCAP
// (>= 2p). ld(lrow, b, q, pair, x0, x1); st(lrow, b, s, pair, y0, y1).
template <int E, int p, bool INV, bool DIT, int NPAIR, int NT, uint64_t BIN, uint64_t OCAP, class LD, class ST>
__device__ __forceinline__ void pass(const uint2* __restrict__ tw, const LD& ld, const ST& st) {
    using S = Sched<E>;
    constexpr int RL = S::rlog(p), R = 1 << RL, LL = S::llog(p), SL = S::slog(p);
    constexpr int ITEMS = (1 << (E - RL)) * NPAIR;
    constexpr int LGP = ilog2c<NPAIR>();
    static_assert(OCAP >= k2P, "");
#pragma unroll 1
    for (int it = threadIdx.x; it < ITEMS; it += NT) {
        const int pair = it & (NPAIR - 1);
        const uint32_t b = uint32_t(it) >> LGP;
        const uint32_t t = b & ((1u << SL) - 1u);
        const uint32_t base = ((b >> SL) << LL) + t;
        uint32_t v0[R], v1[R];
        if constexpr (!DIT) {
#pragma unroll
            for (int q = 0; q < R; ++q) ld(base + (uint32_t(q) << SL), b, q, pair, v0[q], v1[q]);
            dif_regs<R, INV, BIN>(v0);
            dif_regs<R, INV, BIN>(v1);
            constexpr uint64_t BO = dif_bound<R, INV, BIN>();
#pragma unroll
            for (int s = 0; s < R; ++s) {
                uint32_t y0 = v0[rev<R>(s)], y1 = v1[rev<R>(s)];
                if (SL > 0 && s > 0) {
                    const uint2 w = __ldg(tw + ((t * uint32_t(s)) << (E - LL)));
                    y0 = mulw2(y0, w.x, w.y);
                    y1 = mulw2(y1, w.x, w.y);
                } else {
                    y0 = cap<BO, OCAP>(y0);
                    y1 = cap<BO, OCAP>(y1);
                }
                st(base + (uint32_t(s) << SL), b, s, pair, y0, y1);
            }
        } else {
            constexpr uint64_t BI = BIN > k2P ? BIN : k2P;
#pragma unroll
            for (int s = 0; s < R; ++s) {
                uint32_t x0, x1;
                ld(base + (uint32_t(s) << SL), b, s, pair, x0, x1);
                if (SL > 0 && s > 0) {
                    const uint2 w = __ldg(tw + ((t * uint32_t(s)) << (E - LL)));
                    x0 = mulw2(x0, w.x, w.y);
                    x1 = mulw2(x1, w.x, w.y);
                }
                v0[rev<R>(s)] = x0;
                v1[rev<R>(s)] = x1;
            }
            dit_regs<R, INV, BI>(v0);
            dit_regs<R, INV, BI>(v1);
            constexpr uint64_t BO = dit_bound<R, INV, BI>();
#pragma unroll
            for (int q = 0; q < R; ++q)
                st(base + (uint32_t(q) << SL), b, q, pair, cap<BO, OCAP>(v0[q]), cap<BO, OCAP>(v1[q]));
        }
    }
}

// ---------------------------------------------------------------------------
template <int E, int NPAIR, int NT, bool HALFK>
__global__ void __launch_bounds__(NT) enc_fast_kernel(const uint2* __restrict__ tw, uint32_t k, uint32_t n, uint32_t L,
                                                      uint32_t tps, const uint16_t* __restrict__ src, EscIn esc_in,
                                                      uint16_t* __restrict__ out, EscOut esc_out) {
    extern __shared__ uint2 smem[];
    using S = Sched<E>;
    constexpr int P = S::P;
    constexpr int RL0 = S::rlog(0), RLZ = S::rlog(P - 1);
    static_assert(P >= 2, "fast path needs at least two passes");
    const Tile<E, NPAIR> tile{smem};
    const uint32_t stripe = blockIdx.x / tps;
    const uint32_t c0 = (blockIdx.x - stripe * tps) * uint32_t(2 * NPAIR);
    const uint32_t L2 = L >> 1;
    const uint32_t* __restrict__ srcw = reinterpret_cast<const uint32_t*>(src) + (uint64_t(stripe) * k * L + c0) / 2;
    uint32_t* __restrict__ outw = reinterpret_cast<uint32_t*>(out) + (uint64_t(stripe) * n * L + c0) / 2;
    const unsigned long long key_in = uint64_t(stripe) * k * L + c0;
    const unsigned long long key_out = uint64_t(stripe) * n * L + c0;

    auto ld_src = [&](uint32_t lrow, uint32_t, int q, int pair, uint32_t& x0, uint32_t& x1) {
        if ((HALFK && q >= (1 << RL0) / 2) || (!HALFK && lrow >= k)) {
            x0 = x1 = 0u;
            return;
        }
        const uint32_t w = __ldcs(srcw + size_t(lrow) * L2 + pair);
        unpack2(w, esc_in, key_in + uint64_t(lrow) * L + 2 * pair, x0, x1);
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, int pair, uint32_t& x0, uint32_t& x1) {
        const uint2 v = tile.at(lrow, pair);
        x0 = v.x;
        x1 = v.y;
    };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, int pair, uint32_t y0, uint32_t y1) {
        tile.at(lrow, pair) = make_uint2(y0, y1);
    };
    auto st_out = [&](uint32_t, uint32_t b, int s, int pair, uint32_t y0, uint32_t y1) {
        const uint32_t f = perm_head<E>(b) + (uint32_t(s) << (E - RLZ));
        if (f >= n) return;
        __stcs(outw + size_t(f) * L2 + pair, pack2(y0, y1, esc_out, key_out + uint64_t(f) * L + 2 * pair));
    };

    pass<E, 0, false, false, NPAIR, NT, kP64, kSmemCap>(tw, ld_src, st_sm);
    __syncthreads();
    if constexpr (P == 3) {
        pass<E, 1, false, false, NPAIR, NT, kSmemCap, kSmemCap>(tw, ld_sm, st_sm);
        __syncthreads();
    }
    pass<E, P - 1, false, false, NPAIR, NT, kSmemCap, k2P>(tw, ld_sm, st_out);
}

// ---------------------------------------------------------------------------
template <int E, int NPAIR, int NT>
__global__ void __launch_bounds__(NT) dec_fast_kernel(const uint2* __restrict__ twF, const uint2* __restrict__ twI,
                                                      const uint2* __restrict__ rowmap, const uint2* __restrict__ ahat2,
                                                      uint32_t k, uint32_t L, uint32_t tps,
                                                      const uint32_t* __restrict__ stripe_pattern,
                                                      const uint16_t* __restrict__ rx, EscIn esc_in,
                                                      uint16_t* __restrict__ out, EscOut esc_out) {
    extern __shared__ uint2 smem[];
    using S = Sched<E>;
    constexpr int N = 1 << E;
    constexpr int P = S::P;
    constexpr int RLZ = S::rlog(P - 1), RZ = 1 << RLZ;
    constexpr int RL0 = S::rlog(0), R0 = 1 << RL0, SL0 = S::slog(0);
    constexpr uint32_t FLIP = uint32_t(N - 1);
    constexpr int LGP = ilog2c<NPAIR>();
    static_assert(P >= 2, "fast path needs at least two passes");
    const Tile<E, NPAIR> tile{smem};
    const uint32_t stripe = blockIdx.x / tps;
    const uint32_t c0 = (blockIdx.x - stripe * tps) * uint32_t(2 * NPAIR);
    const uint32_t L2 = L >> 1;
    const uint32_t pat = __ldg(stripe_pattern + stripe);
    const uint2* __restrict__ rm = rowmap + size_t(pat) * N;
    const uint2* __restrict__ ah = ahat2 + size_t(pat) * N;
    const uint32_t* __restrict__ rxw = reinterpret_cast<const uint32_t*>(rx) + (uint64_t(stripe) * k * L + c0) / 2;
    uint32_t* __restrict__ outw = reinterpret_cast<uint32_t*>(out) + (uint64_t(stripe) * k * L + c0) / 2;
    const unsigned long long key_in = uint64_t(stripe) * k * L + c0;

    // step 4: N'[z] = v_i / A'(x_i) where z = z_i, else 0 (rowmap[z] = {i or ~0, 1/A'(x_i)})
    auto ld_scatter = [&](uint32_t lrow, uint32_t, int, int pair, uint32_t& x0, uint32_t& x1) {
        const uint2 m = __ldg(rm + lrow);
        if (m.x == 0xFFFFFFFFu) {
            x0 = x1 = 0u;
            return;
        }
        const uint32_t w = __ldcs(rxw + size_t(m.x) * L2 + pair);
        uint32_t a0, a1;
        unpack2(w, esc_in, key_in + uint64_t(m.x) * L + 2 * pair, a0, a1);
        const uint32_t m2 = m.y * 65535u;
        x0 = mulw2(a0, m.y, m2);
        x1 = mulw2(a1, m.y, m2);
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, int pair, uint32_t& x0, uint32_t& x1) {
        const uint2 v = tile.at(lrow, pair);
        x0 = v.x;
        x1 = v.y;
    };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, int pair, uint32_t y0, uint32_t y1) {
        tile.at(lrow, pair) = make_uint2(y0, y1);
    };
    auto ld_smf = [&](uint32_t lrow, uint32_t, int, int pair, uint32_t& x0, uint32_t& x1) {
        const uint2 v = tile.at(lrow ^ FLIP, pair);
        x0 = v.x;
        x1 = v.y;
    };
    auto st_smf = [&](uint32_t lrow, uint32_t, int, int pair, uint32_t y0, uint32_t y1) {
        tile.at(lrow ^ FLIP, pair) = make_uint2(y0, y1);
    };
    auto st_out = [&](uint32_t, uint32_t b, int s, int pair, uint32_t y0, uint32_t y1) {
        const uint32_t f = perm_head<E>(b) + (uint32_t(s) << (E - RLZ));
        if (f >= k) return;
        __stcs(outw + size_t(f) * L2 + pair, pack2(y0, y1, esc_out, key_in + uint64_t(f) * L + 2 * pair));
    };

    // FNT1 = FNT_N(N'), DIF, natural -> perm order (flip 0)
    pass<E, 0, false, false, NPAIR, NT, k2P, kSmemCap>(twF, ld_scatter, st_sm);
    __syncthreads();
    if constexpr (P == 3) {
        pass<E, 1, false, false, NPAIR, NT, kSmemCap, kSmemCap>(twF, ld_sm, st_sm);
        __syncthreads();
    }
    // FNT1 last pass (sub 1, no table twiddles) + FNT2 first DIT pass on the
    // reversed view: logical group b' = N/R - 1 - G holds s'_j = F[N-1-j].
    {
        constexpr int ITEMS = (N / RZ) * NPAIR;
        constexpr uint64_t BD = dif_bound<RZ, false, kSmemCap>();
        constexpr uint64_t BT = dit_bound<RZ, false, BD>();
#pragma unroll 1
        for (int it = threadIdx.x; it < ITEMS; it += NT) {
            const int pair = it & (NPAIR - 1);
            const uint32_t G = uint32_t(it) >> LGP;
            uint32_t v0[RZ], v1[RZ];
#pragma unroll
            for (int q = 0; q < RZ; ++q) {
                const uint2 v = tile.at((G << RLZ) + q, pair);
                v0[q] = v.x;
                v1[q] = v.y;
            }
            dif_regs<RZ, false, kSmemCap>(v0);
            dif_regs<RZ, false, kSmemCap>(v1);
            const uint32_t bp = uint32_t(N / RZ) - 1u - G;
            const uint32_t fh = perm_head<E>(bp);
            uint32_t u0[RZ], u1[RZ];
#pragma unroll
            for (int j = 0; j < RZ; ++j) {
                const int sp = rev<RZ>(j);  // u[rev(s')] = x_{s'} = y_{R-1-s'}
                const bool live = fh + (uint32_t(sp) << (E - RLZ)) < k;
                u0[j] = live ? v0[RZ - 1 - j] : 0u;
                u1[j] = live ? v1[RZ - 1 - j] : 0u;
            }
            dit_regs<RZ, false, BD>(u0);
            dit_regs<RZ, false, BD>(u1);
#pragma unroll
            for (int q = 0; q < RZ; ++q)
                tile.at((G << RLZ) + (RZ - 1 - q), pair) =
                    make_uint2(cap<BT, kSmemCap>(u0[q]), cap<BT, kSmemCap>(u1[q]));
        }
    }
    __syncthreads();
    if constexpr (P == 3) {
        pass<E, 1, false, true, NPAIR, NT, kSmemCap, kSmemCap>(twF, ld_smf, st_smf);
        __syncthreads();
    }
    // FNT2 last DIT pass + (. ahat) + FNT3 first DIF pass: rows t + q * sub0
    {
        constexpr int ITEMS = (N / R0) * NPAIR;
        constexpr uint64_t BT = dit_bound<R0, false, kSmemCap>();
        constexpr uint64_t BO = dif_bound<R0, true, k2P>();
#pragma unroll 1
        for (int it = threadIdx.x; it < ITEMS; it += NT) {
            const int pair = it & (NPAIR - 1);
            const uint32_t t = uint32_t(it) >> LGP;
            uint32_t v0[R0], v1[R0];
#pragma unroll
            for (int s = 0; s < R0; ++s) {
                const uint2 v = tile.at((t + (uint32_t(s) << SL0)) ^ FLIP, pair);
                uint32_t x0 = v.x, x1 = v.y;
                if (s > 0) {
                    const uint2 w = __ldg(twF + t * uint32_t(s));
                    x0 = mulw2(x0, w.x, w.y);
                    x1 = mulw2(x1, w.x, w.y);
                }
                v0[rev<R0>(s)] = x0;
                v1[rev<R0>(s)] = x1;
            }
            dit_regs<R0, false, kSmemCap>(v0);
            dit_regs<R0, false, kSmemCap>(v1);
            static_assert(BT < (1ull << 32), "");
#pragma unroll
            for (int q = 0; q < R0; ++q) {
                const uint2 a = __ldg(ah + t + (uint32_t(q) << SL0));
                v0[q] = mulw2(v0[q], a.x, a.y);
                v1[q] = mulw2(v1[q], a.x, a.y);
            }
            dif_regs<R0, true, k2P>(v0);
            dif_regs<R0, true, k2P>(v1);
#pragma unroll
            for (int s = 0; s < R0; ++s) {
                uint32_t y0 = v0[rev<R0>(s)], y1 = v1[rev<R0>(s)];
                if (s > 0) {
                    const uint2 w = __ldg(twI + t * uint32_t(s));
                    y0 = mulw2(y0, w.x, w.y);
                    y1 = mulw2(y1, w.x, w.y);
                } else {
                    y0 = cap<BO, kSmemCap>(y0);
                    y1 = cap<BO, kSmemCap>(y1);
                }
                tile.at((t + (uint32_t(s) << SL0)) ^ FLIP, pair) = make_uint2(y0, y1);
            }
        }
    }
    __syncthreads();
    if constexpr (P == 3) {
        pass<E, 1, true, false, NPAIR, NT, kSmemCap, kSmemCap>(twI, ld_smf, st_smf);
        __syncthreads();
    }
    pass<E, P - 1, true, false, NPAIR, NT, kSmemCap, k2P>(twI, ld_smf, st_out);
}

__global__ void tables2_kernel(uint2* fwd, uint2* inv) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 || i >= (1u << 17)) return;
    const int e = 31 - __clz(i);
    const uint32_t m = 1u << e, j = i - m;
    const uint32_t ex = (j << (16 - e)) & 0xFFFFu;
    const uint32_t wf = gpow(3u, ex), wi = gpow(3u, (65536u - ex) & 0xFFFFu);
    fwd[i] = make_uint2(wf, wf * 65535u);
    inv[i] = make_uint2(wi, wi * 65535u);
}

// per-pattern decode tables for the fast kernel:
//   rowmap[p][z] = {i, 1/A'(x_i)} if position z is received as row i, else {~0, 0}
//   ahat2[p][j]  = {ahat_j, 65535 * ahat_j}
__global__ void fast_plan_tables_kernel(uint32_t N, uint32_t kp, const uint32_t* __restrict__ pos,
                                        const uint32_t* __restrict__ ainv, const uint32_t* __restrict__ ahat,
                                        uint2* __restrict__ rowmap, uint2* __restrict__ ahat2) {
    const uint32_t p = blockIdx.y;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < N; j += gridDim.x * blockDim.x) {
        rowmap[size_t(p) * N + j] = make_uint2(0xFFFFFFFFu, 0u);
        const uint32_t a = ahat[size_t(p) * N + j];
        ahat2[size_t(p) * N + j] = make_uint2(a, a * 65535u);
    }
}

__global__ void fast_plan_scatter_kernel(uint32_t N, uint32_t kp, const uint32_t* __restrict__ pos,
                                         const uint32_t* __restrict__ ainv, uint2* __restrict__ rowmap) {
    const uint32_t p = blockIdx.y;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < kp; i += gridDim.x * blockDim.x)
        rowmap[size_t(p) * N + pos[size_t(p) * kp + i]] = make_uint2(i, ainv[size_t(p) * kp + i]);
}

template <class K>
cudaError_t prep(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

// tile geometry per size: (NPAIR, NT)
template <int E>
struct Geom;
template <> struct Geom<5> { static constexpr int NPAIR = 32, NT = 256; };
template <> struct Geom<6> { static constexpr int NPAIR = 32, NT = 256; };
template <> struct Geom<7> { static constexpr int NPAIR = 32, NT = 256; };
template <> struct Geom<8> { static constexpr int NPAIR = 32, NT = 256; };
template <> struct Geom<9> { static constexpr int NPAIR = 32, NT = 256; };
template <> struct Geom<10> { static constexpr int NPAIR = 16, NT = 256; };
template <> struct Geom<11> { static constexpr int NPAIR = 8, NT = 256; };
template <> struct Geom<12> { static constexpr int NPAIR = 4, NT = 256; };

template <int E>
cudaError_t launch_enc(const FastTables& t, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                       const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, cudaStream_t st) {
    constexpr int NPAIR = Geom<E>::NPAIR, NT = Geom<E>::NT;
    const uint32_t tps = L / (2 * NPAIR);
    const uint64_t blocks = uint64_t(stripes) * tps;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const size_t smem = size_t(1u << E) * NPAIR * sizeof(uint2);
    const uint2* tw = t.fwd + (1u << E);
    cudaError_t err;
    if (k == (1u << E) / 2) {
        auto kern = enc_fast_kernel<E, NPAIR, NT, true>;
        if ((err = prep(kern, smem))) return err;
        kern<<<unsigned(blocks), NT, smem, st>>>(tw, k, n, L, tps, src, ein, out, eout);
    } else {
        auto kern = enc_fast_kernel<E, NPAIR, NT, false>;
        if ((err = prep(kern, smem))) return err;
        kern<<<unsigned(blocks), NT, smem, st>>>(tw, k, n, L, tps, src, ein, out, eout);
    }
    return cudaGetLastError();
}

template <int E>
cudaError_t launch_dec(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                       const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout, cudaStream_t st) {
    constexpr int NPAIR = Geom<E>::NPAIR, NT = Geom<E>::NT;
    const uint32_t tps = L / (2 * NPAIR);
    const uint64_t blocks = uint64_t(stripes) * tps;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const size_t smem = size_t(1u << E) * NPAIR * sizeof(uint2);
    auto kern = dec_fast_kernel<E, NPAIR, NT>;
    cudaError_t err;
    if ((err = prep(kern, smem))) return err;
    kern<<<unsigned(blocks), NT, smem, st>>>(t.fwd + (1u << E), t.inv + (1u << E), pv.rowmap, pv.ahat2, pv.k, L, tps, sp,
                                             rx, ein, out, eout);
    return cudaGetLastError();
}

}  // namespace

cudaError_t build_fast_tables(FastTables& t, cudaStream_t st) {
    cudaError_t err = cudaMalloc(&t.fwd, sizeof(uint2) << 17);
    if (err) return err;
    if ((err = cudaMalloc(&t.inv, sizeof(uint2) << 17))) return err;
    tables2_kernel<<<(1u << 17) / 256, 256, 0, st>>>(t.fwd, t.inv);
    return cudaGetLastError();
}

int fast_tile_columns(uint32_t N) {
    switch (N) {
        case 32: return 2 * Geom<5>::NPAIR;
        case 64: return 2 * Geom<6>::NPAIR;
        case 128: return 2 * Geom<7>::NPAIR;
        case 256: return 2 * Geom<8>::NPAIR;
        case 512: return 2 * Geom<9>::NPAIR;
        case 1024: return 2 * Geom<10>::NPAIR;
        case 2048: return 2 * Geom<11>::NPAIR;
        case 4096: return 2 * Geom<12>::NPAIR;
        default: return 0;
    }
}

cudaError_t launch_encode_fast(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes, uint32_t L,
                               const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, cudaStream_t st) {
    switch (N) {
        case 32: return launch_enc<5>(t, k, n, stripes, L, src, ein, out, eout, st);
        case 64: return launch_enc<6>(t, k, n, stripes, L, src, ein, out, eout, st);
        case 128: return launch_enc<7>(t, k, n, stripes, L, src, ein, out, eout, st);
        case 256: return launch_enc<8>(t, k, n, stripes, L, src, ein, out, eout, st);
        case 512: return launch_enc<9>(t, k, n, stripes, L, src, ein, out, eout, st);
        case 1024: return launch_enc<10>(t, k, n, stripes, L, src, ein, out, eout, st);
        case 2048: return launch_enc<11>(t, k, n, stripes, L, src, ein, out, eout, st);
        case 4096: return launch_enc<12>(t, k, n, stripes, L, src, ein, out, eout, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_decode_fast(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                               const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                               cudaStream_t st) {
    switch (pv.N) {
        case 32: return launch_dec<5>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        case 64: return launch_dec<6>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        case 128: return launch_dec<7>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        case 256: return launch_dec<8>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        case 512: return launch_dec<9>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        case 1024: return launch_dec<10>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        case 2048: return launch_dec<11>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        case 4096: return launch_dec<12>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fast_plan_tables(uint32_t N, uint32_t kp, uint32_t npatterns, const uint32_t* pos,
                                    const uint32_t* ainv, const uint32_t* ahat, uint2* rowmap, uint2* ahat2,
                                    cudaStream_t st) {
    if (!npatterns) return cudaSuccess;
    for (uint32_t p0 = 0; p0 < npatterns; p0 += 65535u) {
        const uint32_t np = npatterns - p0 < 65535u ? npatterns - p0 : 65535u;
        dim3 g((N + 255) / 256, np);
        fast_plan_tables_kernel<<<g, 256, 0, st>>>(N, kp, pos + size_t(p0) * kp, ainv + size_t(p0) * kp,
                                                   ahat + size_t(p0) * N, rowmap + size_t(p0) * N,
                                                   ahat2 + size_t(p0) * N);
        dim3 g2((kp + 255) / 256, np);
        fast_plan_scatter_kernel<<<g2, 256, 0, st>>>(N, kp, pos + size_t(p0) * kp, ainv + size_t(p0) * kp,
                                                     rowmap + size_t(p0) * N);
    }
    return cudaGetLastError();
}

}  // namespace fast
}  // namespace fntrs_gpu
