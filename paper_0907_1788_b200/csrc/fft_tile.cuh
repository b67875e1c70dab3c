// fft_tile.cuh -- batched column FNTs on a shared-memory tile.
//
// A tile is `rows x WT` uint32 in shared memory: row = transform index
// (packet position), column = one independent transform (a codeword, i.e.
// symbol j of every packet). Transforms run along rows, so loading a tile
// from packet-major memory is a coalesced read of WT adjacent symbols per
// packet: the packet->codeword transpose is the tile load itself.
//
// A transform of size m = 2^e is a sequence of in-place radix passes
// (radix 16 while possible, then one radix 2/4/8 pass). Each work item is
// one radix-R butterfly for a PAIR of adjacent columns (LDS.64 / STS.64); the
// R-point DFT runs in registers with compile-time twiddles and only the
// R-1 inter-pass twiddles come from a table. Replaces the reference's
// radix-2 cores (proj/src/transform.cpp:90-122, AVX2 :155-253).
//
//  DIF (Gentleman-Sande): natural order in, digit-reversed out.
//  DIT (Cooley-Tukey):    digit-reversed in, natural order out.
// Position p of a DIF output holds frequency perm(p) = the 4-bit-digit
// reversal of p (last digit narrower when log2 m % 4 != 0); a DIT pass with
// the same schedule consumes exactly that layout. Rows can be addressed
// through an XOR mask (`flip`): flip = m-1 visits the tile in reversed row
// order, which the decoder uses to turn -F[n-1-j] into an index-free view.
#pragma once
#include <cstdint>

#include "field.cuh"

namespace fntrs_gpu {

// ---- compile-time roots ---------------------------------------------------
template <int L, bool INV>
struct RootPow {
    static constexpr uint32_t r = croot(L, INV);
    __host__ __device__ static constexpr uint32_t pw(int j) { return cpow(r, uint32_t(j)); }
};

__device__ __forceinline__ int ilog2(uint32_t x) { return 31 - __clz(x); }

// frequency index held at DIF output position p (transform size 2^e)
__device__ __forceinline__ uint32_t perm_of(uint32_t p, int e) {
    uint32_t f = 0;
    int sh = e, out = 0;
    while (sh >= 4) {
        sh -= 4;
        f |= ((p >> sh) & 15u) << out;
        out += 4;
    }
    if (sh) f |= (p & ((1u << sh) - 1u)) << out;
    return f;
}

// DIF output position holding frequency f (inverse of perm_of)
__device__ __forceinline__ uint32_t pos_of(uint32_t f, int e) {
    uint32_t p = 0;
    int sh = e, in = 0;
    while (sh >= 4) {
        sh -= 4;
        p |= ((f >> in) & 15u) << sh;
        in += 4;
    }
    if (sh) p |= (f >> in) & ((1u << sh) - 1u);
    return p;
}

template <int R>
__device__ __forceinline__ constexpr int rev_bits(int i) {
    int r = 0;
    for (int b = 1, o = R >> 1; b < R; b <<= 1, o >>= 1)
        if (i & b) r |= o;
    return r;
}

// ---- in-register R-point DFTs ---------------------------------------------
// Compile-time twiddles: TW<L, J, INV>::v = (root of order L)^J.
template <int L, int J, bool INV>
struct TW {
    static constexpr uint32_t v = cpow(croot(L, INV), uint32_t(J));
};

// DIF stage with pair distance HALF (block 2*HALF); K covers the subtrahend.
template <int R, bool INV, int HALF, int J>
__device__ __forceinline__ void dif_j(uint32_t (&v)[R], uint32_t K) {
#pragma unroll
    for (int blk = 0; blk < R; blk += 2 * HALF) {
        const uint32_t a = v[blk + J], b = v[blk + J + HALF];
        v[blk + J] = a + b;
        if constexpr (J == 0)
            v[blk + J + HALF] = red(a + K - b);
        else
            v[blk + J + HALF] = mulw(a + K - b, TW<2 * HALF, J, INV>::v);
    }
    if constexpr (J + 1 < HALF) dif_j<R, INV, HALF, J + 1>(v, K);
}

template <int R, bool INV, int HALF, int ST>
__device__ __forceinline__ void dif_stages(uint32_t (&v)[R]) {
    dif_j<R, INV, HALF, 0>(v, kP << (ST + 1));
    if constexpr (HALF > 1) dif_stages<R, INV, HALF / 2, ST + 1>(v);
}

// DIF: v natural in (< 2p); out v[rev(s)] = y_s, all < 32p.
template <int R, bool INV>
__device__ __forceinline__ void dft_dif(uint32_t (&v)[R]) {
    dif_stages<R, INV, R / 2, 0>(v);
}

template <int R, bool INV, int HALF, int J>
__device__ __forceinline__ void dit_j(uint32_t (&v)[R]) {
#pragma unroll
    for (int blk = 0; blk < R; blk += 2 * HALF) {
        const uint32_t a = v[blk + J];
        uint32_t b;
        if constexpr (J == 0)
            b = red(v[blk + J + HALF]);
        else
            b = mulw(v[blk + J + HALF], TW<2 * HALF, J, INV>::v);
        v[blk + J] = a + b;
        v[blk + J + HALF] = a + 2 * kP - b;
    }
    if constexpr (J + 1 < HALF) dit_j<R, INV, HALF, J + 1>(v);
}

template <int R, bool INV, int HALF>
__device__ __forceinline__ void dit_stages(uint32_t (&v)[R]) {
    dit_j<R, INV, HALF, 0>(v);
    if constexpr (2 * HALF < R) dit_stages<R, INV, 2 * HALF>(v);
}

// DIT: v[rev(s)] in (< 2p); out v[q] = y_q natural, all < 10p.
template <int R, bool INV>
__device__ __forceinline__ void dft_dit(uint32_t (&v)[R]) {
    dit_stages<R, INV, 1>(v);
}

struct NoPre {
    __device__ __forceinline__ void operator()(uint32_t, uint32_t&, uint32_t&) const {}
};

// One radix-R pass over all m/R butterflies x WT/2 column pairs.
//  s:    tile base (rows x WT uint32), WT even
//  e:    log2 m;  len: current block length;  flip: row XOR mask
//  tw:   table r_m^j (direction INV), j < m
//  pre:  applied to loaded values by LOGICAL row (first pass of a transform)
template <int R, bool INV, bool DIT, class Pre>
__device__ __forceinline__ void radix_pass(uint32_t* s, int WT, int e, int len, uint32_t flip,
                                           const uint32_t* __restrict__ tw, const Pre& pre,
                                           bool use_pre) {
    const int m = 1 << e;
    const int npair = WT >> 1;
    const int lg_np = ilog2(npair);
    const int sub = len / R;
    const int lg_sub = ilog2(sub);
    const int items = (m / R) * npair;
    const int tstride = (m / len);  // r_len = r_m^(m/len)
    for (int w = threadIdx.x; w < items; w += blockDim.x) {
        const int pair = w & (npair - 1);
        const int b = w >> lg_np;
        const int blk = b >> lg_sub;
        const int t = b & (sub - 1);
        const int base = blk * len + t;
        uint32_t v0[R], v1[R];
        if (!DIT) {
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const uint32_t lrow = uint32_t(base + q * sub);
                const uint2 x = *reinterpret_cast<const uint2*>(s + size_t(lrow ^ flip) * WT + 2 * pair);
                v0[q] = x.x;
                v1[q] = x.y;
                if (use_pre) pre(lrow, v0[q], v1[q]);
            }
            dft_dif<R, INV>(v0);
            dft_dif<R, INV>(v1);
#pragma unroll
            for (int sidx = 0; sidx < R; ++sidx) {
                const int reg = rev_bits<R>(sidx);
                uint32_t y0 = v0[reg], y1 = v1[reg];
                if (sidx == 0) {
                    y0 = red(y0);
                    y1 = red(y1);
                } else {
                    const uint32_t wv = __ldg(tw + ((t * sidx * tstride) & (m - 1)));
                    const uint32_t w2 = wv * 65535u;
                    y0 = mulw2(y0, wv, w2);
                    y1 = mulw2(y1, wv, w2);
                }
                const uint32_t lrow = uint32_t(base + sidx * sub);
                *reinterpret_cast<uint2*>(s + size_t(lrow ^ flip) * WT + 2 * pair) = make_uint2(y0, y1);
            }
        } else {
#pragma unroll
            for (int sidx = 0; sidx < R; ++sidx) {
                const uint32_t lrow = uint32_t(base + sidx * sub);
                const uint2 x = *reinterpret_cast<const uint2*>(s + size_t(lrow ^ flip) * WT + 2 * pair);
                uint32_t x0 = x.x, x1 = x.y;
                if (use_pre) pre(lrow, x0, x1);
                const int reg = rev_bits<R>(sidx);
                if (sidx == 0) {
                    v0[reg] = red(x0);
                    v1[reg] = red(x1);
                } else {
                    const uint32_t wv = __ldg(tw + ((t * sidx * tstride) & (m - 1)));
                    const uint32_t w2 = wv * 65535u;
                    v0[reg] = mulw2(x0, wv, w2);
                    v1[reg] = mulw2(x1, wv, w2);
                }
            }
            dft_dit<R, INV>(v0);
            dft_dit<R, INV>(v1);
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const uint32_t lrow = uint32_t(base + q * sub);
                *reinterpret_cast<uint2*>(s + size_t(lrow ^ flip) * WT + 2 * pair) = make_uint2(v0[q], v1[q]);
            }
        }
    }
}

// Whole transform of size 2^e on the tile. DIF: natural -> perm order.
// DIT: perm order -> natural. Inputs must be < 2p (DIF) / any (DIT first
// pass reduces); DIF outputs are < 2p, DIT outputs < 10p.
template <bool INV, bool DIT, class Pre = NoPre>
__device__ void tile_fft(uint32_t* s, int WT, int e, uint32_t flip, const uint32_t* __restrict__ tw,
                         const Pre& pre = Pre()) {
    const int nfull = e >> 2, rem = e & 3;
    bool first = true;
    if (!DIT) {
        int len = 1 << e;
        for (int i = 0; i < nfull; ++i, len >>= 4) {
            radix_pass<16, INV, false>(s, WT, e, len, flip, tw, pre, first);
            first = false;
            __syncthreads();
        }
        if (rem == 1) radix_pass<2, INV, false>(s, WT, e, 2, flip, tw, pre, first);
        if (rem == 2) radix_pass<4, INV, false>(s, WT, e, 4, flip, tw, pre, first);
        if (rem == 3) radix_pass<8, INV, false>(s, WT, e, 8, flip, tw, pre, first);
        if (rem) __syncthreads();
    } else {
        int len = 1 << rem;
        if (rem == 1) radix_pass<2, INV, true>(s, WT, e, 2, flip, tw, pre, first);
        if (rem == 2) radix_pass<4, INV, true>(s, WT, e, 4, flip, tw, pre, first);
        if (rem == 3) radix_pass<8, INV, true>(s, WT, e, 8, flip, tw, pre, first);
        if (rem) {
            first = false;
            __syncthreads();
        }
        for (int i = 0; i < nfull; ++i) {
            len <<= 4;
            radix_pass<16, INV, true>(s, WT, e, len, flip, tw, pre, first);
            first = false;
            __syncthreads();
        }
    }
}

}  // namespace fntrs_gpu
