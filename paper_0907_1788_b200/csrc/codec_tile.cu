// codec_tile.cu -- fused encode / decode / transform kernels for n_domain <= 4096.
//
// One CTA owns a tile = (stripe, WT adjacent codewords). It reads the
// packet-major uint16 symbols of that tile straight into shared memory
// (the packet->codeword transpose), runs every transform of the codec step
// on the tile, and writes packet-major uint16 results plus 65536 escapes.
// HBM traffic is exactly the algorithmic bytes: 2k in + 2n out per codeword
// (encode), 2k in + 2k out (decode).
#include <cuda_runtime.h>

#include "fft_tile.cuh"
#include "internal.h"

namespace fntrs_gpu {

namespace {

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

// uint16 word -> field value; a zero word is 65536 when its index is listed
// (shardio escape rule, proj/src/shardio.cpp:203-208).
__device__ __forceinline__ uint32_t word_value(uint32_t w, const EscIn& e, unsigned long long key) {
    if (w != 0u || e.n == 0) return w;
    return esc_has(e, key) ? 65536u : 0u;
}

__device__ __forceinline__ void emit_escape(const EscOut& e, unsigned long long key) {
    const unsigned long long i = atomicAdd(e.count, 1ull);
    if (i < e.cap) e.keys[i] = key;
}

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
    using T = uint16_t;
};
template <>
struct VecT<2> {
    using T = uint32_t;
};
template <>
struct VecT<4> {
    using T = uint2;
};
template <>
struct VecT<8> {
    using T = uint4;
};

template <int VEC>
__device__ __forceinline__ void unpack(const typename VecT<VEC>::T& x, uint32_t (&w)[VEC]) {
    if constexpr (VEC == 1) {
        w[0] = x;
    } else {
        const uint32_t* u = reinterpret_cast<const uint32_t*>(&x);
#pragma unroll
        for (int i = 0; i < VEC / 2; ++i) {
            w[2 * i] = u[i] & 0xFFFFu;
            w[2 * i + 1] = u[i] >> 16;
        }
    }
}

template <int VEC>
__device__ __forceinline__ typename VecT<VEC>::T pack(const uint32_t (&w)[VEC]) {
    typename VecT<VEC>::T x;
    if constexpr (VEC == 1) {
        x = uint16_t(w[0]);
    } else {
        uint32_t* u = reinterpret_cast<uint32_t*>(&x);
#pragma unroll
        for (int i = 0; i < VEC / 2; ++i) u[i] = (w[2 * i] & 0xFFFFu) | (w[2 * i + 1] << 16);
    }
    return x;
}

// Load `nrows` packet rows of the tile. map(i, grow, srow, mul): global row,
// shared row and multiplier (0xFFFFFFFF = none) of tile row i.
template <int VEC, class Map>
__device__ __forceinline__ void load_rows(uint32_t* s, int WT, int nrows, const uint16_t* __restrict__ g,
                                          uint32_t L, uint32_t c0, const EscIn& esc, const Map& map) {
    const int chunks = WT / VEC;
    const int items = nrows * chunks;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int i = it / chunks, ch = it - i * chunks;
        uint64_t grow;
        uint32_t srow, mul;
        map(i, grow, srow, mul);
        const uint32_t col = c0 + uint32_t(ch * VEC);
        uint32_t w[VEC];
        if (col + VEC <= L) {
            const typename VecT<VEC>::T x =
                __ldcs(reinterpret_cast<const typename VecT<VEC>::T*>(g + grow * L + col));
            unpack<VEC>(x, w);
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (w[v] == 0u && esc.n) w[v] = word_value(0u, esc, grow * L + col + v);
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) w[v] = 0u;  // column tail beyond L
        }
        uint32_t* d = s + size_t(srow) * WT + ch * VEC;
#pragma unroll
        for (int v = 0; v < VEC; ++v) d[v] = (mul == 0xFFFFFFFFu) ? w[v] : mulw(w[v], mul);
    }
}

__device__ __forceinline__ void zero_rows(uint32_t* s, int WT, int r0, int r1) {
    // WT is even, so row starts are 8-byte aligned
    uint2* p = reinterpret_cast<uint2*>(s + size_t(r0) * WT);
    const int n2 = (r1 - r0) * WT / 2;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) p[i] = make_uint2(0, 0);
}

// Store `nout` output rows. map(f, grow, srow): global row and shared row of
// output f. Values are canonicalised (after an optional scale) and 65536 is
// written as 0 with its symbol index emitted as an escape
// (proj/src/shardio.cpp:131-137,153-154).
template <int VEC, class Map>
__device__ __forceinline__ void store_rows(const uint32_t* s, int WT, int nout, uint16_t* __restrict__ g,
                                           uint32_t L, uint32_t c0, uint32_t scale,
                                           const EscOut& esc, const Map& map) {
    const int chunks = WT / VEC;
    const int items = nout * chunks;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int f = it / chunks, ch = it - f * chunks;
        uint64_t grow;
        uint32_t srow;
        map(f, grow, srow);
        const uint32_t col = c0 + uint32_t(ch * VEC);
        if (col + VEC > L) continue;
        const uint32_t* d = s + size_t(srow) * WT + ch * VEC;
        uint32_t w[VEC];
        bool any = false;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            uint32_t x = d[v];
            x = (scale == 1u) ? canon(x) : red2p(mulw(x, scale));
            any |= (x == 65536u);
            w[v] = x;
        }
        if (any) {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (w[v] == 65536u) emit_escape(esc, grow * L + col + v);
        }
        __stcs(reinterpret_cast<typename VecT<VEC>::T*>(g + grow * L + col), pack<VEC>(w));
    }
}

// ---------------------------------------------------------------------------
// encode_nonsystematic (proj/src/codec.cpp:124-131) for every codeword of the
// tile: zero-pad k -> N, forward transform, keep outputs f < n.
template <int VEC>
__global__ void __launch_bounds__(256) encode_tile_kernel(Tables t, uint32_t k, uint32_t n, int e,
                                                           uint32_t L, int WT, uint32_t tps,
                                                           const uint16_t* __restrict__ src, EscIn esc_in,
                                                           uint16_t* __restrict__ out, EscOut esc_out) {
    extern __shared__ uint4 smem_raw[];
    uint32_t* s = reinterpret_cast<uint32_t*>(smem_raw);
    const uint32_t N = 1u << e;
    const uint64_t stripe = blockIdx.x / tps;
    const uint32_t c0 = (blockIdx.x % tps) * uint32_t(WT);

    zero_rows(s, WT, int(k), int(N));
    load_rows<VEC>(s, WT, int(k), src, L, c0, esc_in,
                   [&](int i, uint64_t& grow, uint32_t& srow, uint32_t& mul) {
                       grow = stripe * k + uint32_t(i);
                       srow = uint32_t(i);
                       mul = 0xFFFFFFFFu;
                   });
    __syncthreads();
    tile_fft<false, false>(s, WT, e, 0u, t.fwd + N);
    store_rows<VEC>(s, WT, int(n), out, L, c0, 1u, esc_out,
                    [&](int f, uint64_t& grow, uint32_t& srow) {
                        grow = stripe * n + uint32_t(f);
                        srow = pos_of(uint32_t(f), e);
                    });
}

// ---------------------------------------------------------------------------
// decode_nonsystematic -> interp::interpolate (proj/src/interp.cpp:103-137)
// for every codeword of the tile:
//   step 4: N'[z_i] = v_i / A'(x_i)                      (scatter + scale)
//   step 5: F = FNT_N(N'); s'_j = F[N-1-j], j < k       (one size-N transform;
//           the reference's chirp route computes the same values)
//   step 6: P = IFNT_M(FNT_M(s') . ahat)[0..k), ahat = -A_hat / M
// N == M: the reversal is an XOR view of the tile (flip = N-1), no data move.
// N != M: s' is gathered into a second buffer of M rows.
// kp == N (every position received): P = IFNT_N(values)[0..k) (codec.cpp:137-144).
struct ZeroAbove {
    int e;
    uint32_t k;
    __device__ __forceinline__ void operator()(uint32_t lrow, uint32_t& a, uint32_t& b) const {
        if (perm_of(lrow, e) >= k) a = b = 0u;
    }
};

struct MulRow {
    const uint32_t* __restrict__ w;
    __device__ __forceinline__ void operator()(uint32_t lrow, uint32_t& a, uint32_t& b) const {
        const uint32_t x = __ldg(w + lrow), x2 = x * 65535u;
        a = mulw2(a, x, x2);
        b = mulw2(b, x, x2);
    }
};

template <int VEC>
__global__ void __launch_bounds__(256) decode_tile_kernel(Tables t, PlanView pv, int eN, int eM,
                                                           uint32_t L, int WT, uint32_t tps,
                                                           const uint32_t* __restrict__ stripe_pattern,
                                                           const uint16_t* __restrict__ rx, EscIn esc_in,
                                                           uint16_t* __restrict__ out, EscOut esc_out) {
    extern __shared__ uint4 smem_raw[];
    uint32_t* s = reinterpret_cast<uint32_t*>(smem_raw);
    const uint32_t N = 1u << eN, M = 1u << eM;
    const uint64_t stripe = blockIdx.x / tps;
    const uint32_t c0 = (blockIdx.x % tps) * uint32_t(WT);
    const uint32_t pat = __ldg(stripe_pattern + stripe);
    const uint32_t* __restrict__ pos = pv.positions + size_t(pat) * pv.kp;
    const uint32_t* __restrict__ ainv = pv.ainv + size_t(pat) * pv.kp;
    const uint32_t* __restrict__ ahat = pv.ahat + size_t(pat) * M;
    const uint32_t kp = pv.kp, k = pv.k;

    if (kp == N) {  // full reception: one inverse transform
        load_rows<VEC>(s, WT, int(N), rx, L, c0, esc_in,
                       [&](int i, uint64_t& grow, uint32_t& srow, uint32_t& mul) {
                           grow = stripe * kp + uint32_t(i);
                           srow = __ldg(pos + i);
                           mul = 0xFFFFFFFFu;
                       });
        __syncthreads();
        tile_fft<true, false>(s, WT, eN, 0u, t.inv + N);
        store_rows<VEC>(s, WT, int(k), out, L, c0, pv.ninv, esc_out,
                        [&](int f, uint64_t& grow, uint32_t& srow) {
                            grow = stripe * k + uint32_t(f);
                            srow = pos_of(uint32_t(f), eN);
                        });
        return;
    }

    zero_rows(s, WT, 0, int(N));
    __syncthreads();
    load_rows<VEC>(s, WT, int(kp), rx, L, c0, esc_in,
                   [&](int i, uint64_t& grow, uint32_t& srow, uint32_t& mul) {
                       grow = stripe * kp + uint32_t(i);
                       srow = __ldg(pos + i);
                       mul = __ldg(ainv + i);
                   });
    __syncthreads();
    tile_fft<false, false>(s, WT, eN, 0u, t.fwd + N);  // F in perm order

    if (N == M) {
        const uint32_t flip = N - 1u;
        tile_fft<false, true>(s, WT, eN, flip, t.fwd + N, ZeroAbove{eN, k});
        tile_fft<true, false>(s, WT, eN, flip, t.inv + N, MulRow{ahat});
        store_rows<VEC>(s, WT, int(k), out, L, c0, 1u, esc_out,
                        [&](int f, uint64_t& grow, uint32_t& srow) {
                            grow = stripe * k + uint32_t(f);
                            srow = pos_of(uint32_t(f), eN) ^ flip;
                        });
    } else {
        uint32_t* b = s + size_t(N) * WT;
        const int npair = WT >> 1;
        const int items = int(M) * npair;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
            const int q = it / npair, pr = it - q * npair;
            const uint32_t f = perm_of(uint32_t(q), eM);
            uint2 v = make_uint2(0u, 0u);
            if (f < k) v = *reinterpret_cast<const uint2*>(s + size_t(pos_of(N - 1u - f, eN)) * WT + 2 * pr);
            *reinterpret_cast<uint2*>(b + size_t(q) * WT + 2 * pr) = v;
        }
        __syncthreads();
        tile_fft<false, true>(b, WT, eM, 0u, t.fwd + M);
        tile_fft<true, false>(b, WT, eM, 0u, t.inv + M, MulRow{ahat});
        store_rows<VEC>(b, WT, int(k), out, L, c0, 1u, esc_out,
                        [&](int f, uint64_t& grow, uint32_t& srow) {
                            grow = stripe * k + uint32_t(f);
                            srow = pos_of(uint32_t(f), eM);
                        });
    }
}

// ---------------------------------------------------------------------------
// fnt_forward / fnt_inverse (proj/src/transform.cpp:302-323) over columns of a
// [m][L] uint32 array; natural order in and out.
__global__ void __launch_bounds__(256) fnt_tile_kernel(Tables t, int e, bool inverse, uint32_t L, int WT,
                                                       uint32_t scale, const uint32_t* __restrict__ in,
                                                       uint32_t* __restrict__ out) {
    extern __shared__ uint4 smem_raw[];
    uint32_t* s = reinterpret_cast<uint32_t*>(smem_raw);
    const uint32_t m = 1u << e;
    const uint32_t c0 = blockIdx.x * uint32_t(WT);
    for (int it = threadIdx.x; it < int(m) * WT; it += blockDim.x) {
        const int r = it / WT, c = it - r * WT;
        const uint32_t col = c0 + uint32_t(c);
        s[it] = col < L ? red(__ldg(in + size_t(r) * L + col)) : 0u;
    }
    __syncthreads();
    if (inverse)
        tile_fft<true, false>(s, WT, e, 0u, t.inv + m);
    else
        tile_fft<false, false>(s, WT, e, 0u, t.fwd + m);
    for (int it = threadIdx.x; it < int(m) * WT; it += blockDim.x) {
        const int f = it / WT, c = it - f * WT;
        const uint32_t col = c0 + uint32_t(c);
        if (col >= L) continue;
        const uint32_t x = s[size_t(pos_of(uint32_t(f), e)) * WT + c];
        out[size_t(f) * L + col] = red2p(mulw(x, scale));
    }
}

__global__ void tables_kernel(uint32_t* fwd, uint32_t* inv) {
    // tw[m + j] = r_m^j: entry i in [m, 2m) of the 2^17 buffer
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 || i >= (1u << 17)) return;
    const int e = 31 - __clz(i);
    const uint32_t m = 1u << e, j = i - m;
    // r_m^j = 3^(j * 65536/m)
    const uint32_t ex = (j << (16 - e)) & 0xFFFFu;
    fwd[i] = gpow(3u, ex);
    inv[i] = gpow(3u, (65536u - ex) & 0xFFFFu);
}

template <class K>
cudaError_t set_smem(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

int pick_vec(uint32_t L, int wt, const void* a, const void* b) {
    auto al = [](const void* p, int bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; };
    if (wt >= 8 && L % 8 == 0 && al(a, 16) && al(b, 16)) return 8;
    if (wt >= 4 && L % 4 == 0 && al(a, 8) && al(b, 8)) return 4;
    if (wt >= 2 && L % 2 == 0 && al(a, 4) && al(b, 4)) return 2;
    return 1;
}

}  // namespace

TileGeom pick_tile(int rows, uint32_t L) {
    TileGeom g;
    const size_t budget = 128 * 1024;
    int wt = 64;
    while (wt > 2 && size_t(rows) * wt * 4 > budget) wt >>= 1;
    // do not make tiles much wider than the data
    while (wt > 2 && uint32_t(wt / 2) >= L) wt >>= 1;
    g.wt = wt;
    g.threads = 256;
    g.smem = size_t(rows) * wt * 4;
    return g;
}

cudaError_t build_tables(Tables& t, cudaStream_t st) {
    cudaError_t err = cudaMalloc(&t.fwd, sizeof(uint32_t) << 17);
    if (err) return err;
    err = cudaMalloc(&t.inv, sizeof(uint32_t) << 17);
    if (err) return err;
    tables_kernel<<<(1u << 17) / 256, 256, 0, st>>>(t.fwd, t.inv);
    return cudaGetLastError();
}

static int log2_exact(uint32_t n) {
    int e = 0;
    while ((1u << e) < n) ++e;
    return e;
}

cudaError_t launch_encode_tile(const Tables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes,
                               uint32_t L, const uint16_t* src, EscIn esc_in, uint16_t* out,
                               EscOut esc_out, cudaStream_t st) {
    if (!stripes || !L) return cudaSuccess;
    const int e = log2_exact(N);
    TileGeom g = pick_tile(int(N), L);
    const uint32_t tps = (L + g.wt - 1) / g.wt;
    const uint64_t blocks = uint64_t(stripes) * tps;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const int vec = pick_vec(L, g.wt, src, out);
    cudaError_t err = cudaSuccess;
#define FNTRS_ENC(V)                                                                              \
    case V:                                                                                       \
        err = set_smem(encode_tile_kernel<V>, g.smem);                                           \
        if (err) return err;                                                                      \
        encode_tile_kernel<V><<<unsigned(blocks), g.threads, g.smem, st>>>(t, k, n, e, L, g.wt, tps, \
                                                                            src, esc_in, out, esc_out); \
        break;
    switch (vec) {
        FNTRS_ENC(8)
        FNTRS_ENC(4)
        FNTRS_ENC(2)
        FNTRS_ENC(1)
    }
#undef FNTRS_ENC
    return cudaGetLastError();
}

cudaError_t launch_decode_tile(const Tables& t, const PlanView& pv, uint32_t stripes, uint32_t L,
                               const uint32_t* stripe_pattern, const uint16_t* rx, EscIn esc_in,
                               uint16_t* out, EscOut esc_out, cudaStream_t st) {
    if (!stripes || !L) return cudaSuccess;
    const int eN = log2_exact(pv.N), eM = log2_exact(pv.M);
    const bool full = pv.kp == pv.N;  // positions are distinct and < n <= N
    const int rows = int(pv.N) + ((full || pv.N == pv.M) ? 0 : int(pv.M));
    TileGeom g = pick_tile(rows, L);
    const uint32_t tps = (L + g.wt - 1) / g.wt;
    const uint64_t blocks = uint64_t(stripes) * tps;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const int vec = pick_vec(L, g.wt, rx, out);
    cudaError_t err = cudaSuccess;
#define FNTRS_DEC(V)                                                                                 \
    case V:                                                                                          \
        err = set_smem(decode_tile_kernel<V>, g.smem);                                              \
        if (err) return err;                                                                         \
        decode_tile_kernel<V><<<unsigned(blocks), g.threads, g.smem, st>>>(                         \
            t, pv, eN, eM, L, g.wt, tps, stripe_pattern, rx, esc_in, out, esc_out);                  \
        break;
    switch (vec) {
        FNTRS_DEC(8)
        FNTRS_DEC(4)
        FNTRS_DEC(2)
        FNTRS_DEC(1)
    }
#undef FNTRS_DEC
    return cudaGetLastError();
}

cudaError_t launch_fnt_tile(const Tables& t, uint32_t m, bool inverse, uint32_t scale, uint32_t L,
                            const uint32_t* in, uint32_t* out, cudaStream_t st) {
    if (!L) return cudaSuccess;
    const int e = log2_exact(m);
    TileGeom g = pick_tile(int(m), L);
    const uint32_t tiles = (L + g.wt - 1) / g.wt;
    cudaError_t err = set_smem(fnt_tile_kernel, g.smem);
    if (err) return err;
    fnt_tile_kernel<<<tiles, g.threads, g.smem, st>>>(t, e, inverse, L, g.wt, scale, in, out);
    return cudaGetLastError();
}

}  // namespace fntrs_gpu
