// plan_fast.cu -- decode plans by one exact cyclic convolution in the log domain,
// and column-batched FNTs of any size <= 65536 (used by the plans and by the
// public fntrs_gpu_fnt entry point).
//
// For received positions R (|R| = k) in the size-N domain (r = r_N, g = 3):
//   x_i - x_l = r^z_l (r^(z_i - z_l) - 1), so with L(d) = log_g(r^d - 1) (d != 0)
//   log_g A(r^j)      = (65536/N) S      + sum_{l}      L(j - z_l)   (j not in R)
//   log_g A'(x_i)     = (65536/N)(S-z_i) + sum_{l != i} L(z_i - z_l)
// (S = sum of positions, exponents mod 65536). Setting L(0) = 0 makes both sums
// the same cyclic convolution conv = 1_R (*) L~ over Z. 1/A'(x_i) is g raised to
// the negated exponent: no inversions. The convolution is exact in GF(65537):
// L~ is split into w-bit digits with k (2^w - 1) <= 65536, each digit convolved
// with one forward and one inverse FNT, and the digit results recombined
// mod 65536. Replaces interp::build_plan's subproduct tree + chirp evaluation +
// per-point Fermat inverses (proj/src/interp.cpp:23-68) with the same values.
#include <cuda_runtime.h>

#include "fft_pass.cuh"

namespace fntrs_gpu {
namespace fast {

namespace {

// ---------------------------------------------------------- column loaders ----
struct LdPlain {  // in[row * C + col]
    const uint32_t* in;
    uint32_t C;
    __device__ __forceinline__ uint32_t operator()(uint32_t row, uint32_t col) const { return in[size_t(row) * C + col]; }
};

struct LdSpectrumProduct {  // column c = p * D + b: X[row][p] * Dh[row][b]  ([0, 2p))
    const uint32_t* X;
    const uint32_t* Dh;
    uint32_t P, D;
    __device__ __forceinline__ uint32_t operator()(uint32_t row, uint32_t c) const {
        const uint32_t p = c / D, b = c - p * D;
        return mulw(__ldg(X + size_t(row) * P + p), __ldg(Dh + size_t(row) * D + b));
    }
};

struct LdLogDigits {  // column b: digit b of L~(d) = log_g(r^d - 1), L~(0) = 0
    const uint32_t* rtab;   // r_N^d, d < N (canonical)
    const uint16_t* log3;   // log_3 of 1..65536
    uint32_t w;
    __device__ __forceinline__ uint32_t operator()(uint32_t d, uint32_t b) const {
        if (d == 0) return 0u;
        const uint32_t x = __ldg(rtab + d);    // r^d in [2, 65536] for 0 < d < N
        const uint32_t lt = __ldg(log3 + (x - 2u));  // log3[v - 1] = log_3(v), v = r^d - 1
        return (lt >> (w * b)) & ((1u << w) - 1u);
    }
};

// ------------------------------------------------- column FNT, N <= 4096 ----
template <int E>
struct ColGeom {
    static constexpr int WT = E <= 9 ? 32 : (E == 10 ? 16 : 8);
    using G = Geom<E, WT, 256, 1>;
};

template <int E, bool INV, class LD>
__global__ void __launch_bounds__(256) cols_small_kernel(LD ld, uint32_t C, const uint2* __restrict__ ptab,
                                                         uint32_t scale, uint32_t* __restrict__ out) {
    using G = typename ColGeom<E>::G;
    using S = Sched<E>;
    constexpr int WT = G::WT, P = S::P, RLZ = G::RLZ;
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t c0 = blockIdx.x * WT;
    const int32_t sc = balanced(scale);
    auto ld0 = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t {
        return c0 + col < C ? ld(lrow, c0 + col) : 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
        const uint32_t f = perm_head<E>(b) + (uint32_t(s) << (E - RLZ));
        if (c0 + col < C) out[size_t(f) * C + c0 + col] = canon_s2p(mulws(y, uint32_t(sc), uint32_t(sc * 65535)));
        return 0u;
    };
    const uint2* tb = INV ? ptab : ptab;
    if constexpr (P == 1) {
        pass<E, 0, INV, false, k2P, k2P, G>(pass_table(tb, S::llog(0)), ld0, st_out);
    } else {
        pass<E, 0, INV, false, k2P, kSmemCap, G>(pass_table(tb, S::llog(0)), ld0, st_sm);
        __syncthreads();
        if constexpr (P == 3) {
            pass<E, 1, INV, false, kSmemCap, kSmemCap, G>(pass_table(tb, S::llog(1)), ld_sm, st_sm);
            __syncthreads();
        }
        pass<E, P - 1, INV, false, kSmemCap, k2P, G>(pass_table(tb, S::llog(P - 1)), ld_sm, st_out);
    }
}

// ------------------------------------- column FNT, 8192 <= N <= 65536 ----
constexpr int kCW = 32;  // columns per CTA (four-step passes)

template <int E>
using CG = Geom<E, kCW, 256, 1>;

// pass A: for each i2, size-N1 transforms over rows i1*N2 + i2; twiddle; Y[m1*N2 + i2]
template <int E1, int E2, bool INV, class LD>
__global__ void __launch_bounds__(256) cols_a_kernel(LD ld, uint32_t C, const uint2* __restrict__ ptab,
                                                     const uint2* __restrict__ big, uint32_t* __restrict__ Y) {
    using G = CG<E1>;
    using S = Sched<E1>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2, N = N1 * N2;
    constexpr int RLZ = G::RLZ;
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t tiles = (C + kCW - 1) / kCW;
    const uint32_t i2 = blockIdx.x / tiles, c0 = (blockIdx.x % tiles) * kCW;
    auto ld0 = [&](uint32_t i1, uint32_t, int, uint32_t col) -> uint32_t {
        return c0 + col < C ? ld(i1 * N2 + i2, c0 + col) : 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto st_y = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
        const uint32_t m1 = perm_head<E1>(b) + (uint32_t(s) << (E1 - RLZ));
        const uint2 w = __ldg(big + N + ((i2 * m1) & (N - 1)));
        if (c0 + col < C) Y[size_t(m1 * N2 + i2) * C + c0 + col] = mulws(y, w.x, w.y);
        return 0u;
    };
    pass<E1, 0, INV, false, k2P, kSmemCap, G>(pass_table(ptab, S::llog(0)), ld0, st_sm);
    __syncthreads();
    pass<E1, 1, INV, false, kSmemCap, kSmemCap, G>(pass_table(ptab, S::llog(1)), ld_sm, st_y);
}

// pass B: for each m1, size-N2 transforms over rows m1*N2 + i2 -> out[m1 + N1*m2]
template <int E1, int E2, bool INV>
__global__ void __launch_bounds__(256) cols_b_kernel(const uint32_t* __restrict__ Y, uint32_t C,
                                                     const uint2* __restrict__ ptab, uint32_t scale,
                                                     uint32_t* __restrict__ out) {
    using G = CG<E2>;
    using S = Sched<E2>;
    constexpr uint32_t N1 = 1u << E1, N2 = 1u << E2;
    constexpr int RLZ = G::RLZ;
    extern __shared__ __align__(128) uint32_t work[];
    const uint32_t tiles = (C + kCW - 1) / kCW;
    const uint32_t m1 = blockIdx.x / tiles, c0 = (blockIdx.x % tiles) * kCW;
    const int32_t sc = balanced(scale);
    auto ld0 = [&](uint32_t i2, uint32_t, int, uint32_t col) -> uint32_t {
        return c0 + col < C ? Y[size_t(m1 * N2 + i2) * C + c0 + col] : 0u;
    };
    auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
    auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
        work[G::idx(lrow, col)] = y;
        return 0u;
    };
    auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
        const uint32_t m2 = perm_head<E2>(b) + (uint32_t(s) << (E2 - RLZ));
        if (c0 + col < C)
            out[size_t(m1 + N1 * m2) * C + c0 + col] = canon_s2p(mulws(y, uint32_t(sc), uint32_t(sc * 65535)));
        return 0u;
    };
    pass<E2, 0, INV, false, k2P, kSmemCap, G>(pass_table(ptab, S::llog(0)), ld0, st_sm);
    __syncthreads();
    pass<E2, 1, INV, false, kSmemCap, kSmemCap, G>(pass_table(ptab, S::llog(1)), ld_sm, st_out);
}

template <class K>
cudaError_t prep(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

template <int E, bool INV, class LD>
cudaError_t run_small(const FastTables& t, LD ld, uint32_t C, uint32_t scale, uint32_t* out, cudaStream_t st) {
    using G = typename ColGeom<E>::G;
    const size_t smem = size_t(1u << E) * G::WT * 4;
    auto kern = cols_small_kernel<E, INV, LD>;
    cudaError_t err = prep(kern, smem);
    if (err) return err;
    const uint32_t tiles = (C + G::WT - 1) / G::WT;
    kern<<<tiles, 256, smem, st>>>(ld, C, INV ? t.ptab_inv : t.ptab_fwd, scale, out);
    return cudaGetLastError();
}

template <int E1, int E2, bool INV, class LD>
cudaError_t run_large(const FastTables& t, LD ld, uint32_t C, uint32_t scale, uint32_t* Y, uint32_t* out,
                      cudaStream_t st) {
    const size_t smA = size_t(1u << E1) * kCW * 4, smB = size_t(1u << E2) * kCW * 4;
    auto ka = cols_a_kernel<E1, E2, INV, LD>;
    auto kb = cols_b_kernel<E1, E2, INV>;
    cudaError_t err;
    if ((err = prep(ka, smA)) || (err = prep(kb, smB))) return err;
    const uint32_t tiles = (C + kCW - 1) / kCW;
    ka<<<(1u << E2) * tiles, 256, smA, st>>>(ld, C, INV ? t.ptab_inv : t.ptab_fwd, INV ? t.big_inv : t.big_fwd, Y);
    kb<<<(1u << E1) * tiles, 256, smB, st>>>(Y, C, INV ? t.ptab_inv : t.ptab_fwd, scale, out);
    return cudaGetLastError();
}

// Dispatch a column transform of size N over C columns with loader `ld`.
// scratch: N*C uint32 (only for N >= 8192).
template <bool INV, class LD>
cudaError_t run_cols(const FastTables& t, uint32_t N, LD ld, uint32_t C, uint32_t scale, uint32_t* scratch,
                     uint32_t* out, cudaStream_t st) {
    if (!C) return cudaSuccess;
    switch (N) {
        case 2: return run_small<1, INV>(t, ld, C, scale, out, st);
        case 4: return run_small<2, INV>(t, ld, C, scale, out, st);
        case 8: return run_small<3, INV>(t, ld, C, scale, out, st);
        case 16: return run_small<4, INV>(t, ld, C, scale, out, st);
        case 32: return run_small<5, INV>(t, ld, C, scale, out, st);
        case 64: return run_small<6, INV>(t, ld, C, scale, out, st);
        case 128: return run_small<7, INV>(t, ld, C, scale, out, st);
        case 256: return run_small<8, INV>(t, ld, C, scale, out, st);
        case 512: return run_small<9, INV>(t, ld, C, scale, out, st);
        case 1024: return run_small<10, INV>(t, ld, C, scale, out, st);
        case 2048: return run_small<11, INV>(t, ld, C, scale, out, st);
        case 4096: return run_small<12, INV>(t, ld, C, scale, out, st);
        case 8192: return run_large<7, 6, INV>(t, ld, C, scale, scratch, out, st);
        case 16384: return run_large<7, 7, INV>(t, ld, C, scale, scratch, out, st);
        case 32768: return run_large<8, 7, INV>(t, ld, C, scale, scratch, out, st);
        case 65536: return run_large<8, 8, INV>(t, ld, C, scale, scratch, out, st);
        default: return cudaErrorInvalidValue;
    }
}

// ------------------------------------------------------------ plan kernels ----
// indicator columns X[z][p] = [z in R_p], plus S_p = sum of positions mod N
__global__ void indicator_kernel(uint32_t N, uint32_t k, uint32_t P, const uint32_t* __restrict__ pos,
                                 uint32_t* __restrict__ X, uint32_t* __restrict__ S) {
    const uint32_t p = blockIdx.x;
    uint32_t sum = 0;
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        const uint32_t z = pos[size_t(p) * k + i];
        X[size_t(z) * P + p] = 1u;
        sum += z;
    }
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
    __shared__ uint32_t part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (uint32_t wv = 0; wv < blockDim.x / 32; ++wv) s += part[wv];
        S[p] = s & (N - 1);
    }
}

// conv[p][j] = (sum_b Y[j][p*D + b] << (w b)) mod 2^16, transposing [N][P*D] -> [P][N]
// through a 32x32 shared tile so both sides are coalesced.
__global__ void conv_combine_kernel(uint32_t N, uint32_t P, uint32_t D, uint32_t w, const uint32_t* __restrict__ Y,
                                    uint32_t* __restrict__ conv) {
    __shared__ uint32_t tile[32][33];
    const uint32_t p0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    const uint32_t tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (uint32_t r = ty; r < 32; r += 8) {
        const uint32_t j = j0 + r, p = p0 + tx;
        uint32_t c = 0;
        if (j < N && p < P) {
            const uint32_t* y = Y + size_t(j) * P * D + size_t(p) * D;
            for (uint32_t b = 0; b < D; ++b) c += __ldg(y + b) << (w * b);
        }
        tile[r][tx] = c & 0xFFFFu;
    }
    __syncthreads();
    for (uint32_t r = ty; r < 32; r += 8) {
        const uint32_t p = p0 + r, j = j0 + tx;
        if (j < N && p < P) conv[size_t(p) * N + j] = tile[tx][r];
    }
}

// ainv[p][i], rowmap[p][z_i] = {i, balanced 1/A'(x_i)}
__global__ void plan_ainv_kernel(uint32_t N, uint32_t k, uint32_t P, const uint32_t* __restrict__ pos,
                                 const uint32_t* __restrict__ S, const uint32_t* __restrict__ conv,
                                 const uint32_t* __restrict__ exp3, uint32_t* __restrict__ ainv,
                                 uint2* __restrict__ rowmap) {
    const uint64_t total = uint64_t(P) * k;
    const uint32_t sc = 65536u / N;
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t p = uint32_t(t / k), i = uint32_t(t - uint64_t(p) * k);
        const uint32_t z = pos[t];
        const uint32_t e = (sc * ((S[p] + N - z) & (N - 1)) + __ldg(conv + size_t(p) * N + z)) & 0xFFFFu;
        const uint32_t inv = __ldg(exp3 + ((65536u - e) & 0xFFFFu));
        ainv[t] = inv;
        rowmap[size_t(p) * N + z] = make_uint2(i, uint32_t(balanced(inv)));
    }
}

// ahat[p][j] = -A(r^j)/N (0 on received positions), ahat2 = signed Shoup pairs
__global__ void plan_ahat_kernel(uint32_t N, uint32_t P, const uint32_t* __restrict__ S,
                                 const uint32_t* __restrict__ conv, const uint2* __restrict__ rowmap,
                                 const uint32_t* __restrict__ exp3, uint32_t neg_ninv, uint32_t* __restrict__ ahat,
                                 uint2* __restrict__ ahat2) {
    const uint64_t total = uint64_t(P) * N;
    const uint32_t sc = 65536u / N;
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t p = uint32_t(t / N);
        uint32_t a = 0;
        if (rowmap[t].x == 0xFFFFFFFFu) {
            const uint32_t e = (sc * S[p] + conv[t]) & 0xFFFFu;
            a = red2p(mulw(__ldg(exp3 + e), neg_ninv));
        }
        ahat[t] = a;
        const int32_t ab = balanced(a);
        ahat2[size_t(p) * N + ahat2_slot(N, uint32_t(t - uint64_t(p) * N))] = make_uint2(uint32_t(ab), uint32_t(ab * 65535));
    }
}

__global__ void exp_log_kernel(uint32_t* exp3, uint16_t* log3) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 65536u) return;
    const uint32_t x = gpow(3u, e);
    exp3[e] = x;
    log3[x - 1u] = uint16_t(e);  // x in [1, 65536]
}

__global__ void fill_rowmap_kernel(uint2* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = make_uint2(0xFFFFFFFFu, 0u);
}

}  // namespace

cudaError_t build_log_tables(LogTables& lt, cudaStream_t st) {
    cudaError_t err = cudaMalloc(&lt.exp3, sizeof(uint32_t) * 65536);
    if (err) return err;
    if ((err = cudaMalloc(&lt.log3, sizeof(uint16_t) * 65536))) return err;
    exp_log_kernel<<<256, 256, 0, st>>>(lt.exp3, lt.log3);
    return cudaGetLastError();
}

uint32_t plan_digit_width(uint32_t k) {
    uint32_t w = 1;
    while (w < 16 && uint64_t(k) * ((1ull << (w + 1)) - 1) <= 65536ull) ++w;
    return w;
}

cudaError_t build_digit_spectra(const FastTables& t, const Tables& tab, const LogTables& lt, uint32_t N, uint32_t w,
                                uint32_t* Dh, uint32_t* scratch, cudaStream_t st) {
    const uint32_t D = (16 + w - 1) / w;
    LdLogDigits ld{tab.fwd + N, lt.log3, w};
    return run_cols<false>(t, N, ld, D, 1u, scratch, Dh, st);
}

size_t plan_fast_scratch_words(uint32_t N, uint32_t k, uint32_t P) {
    const uint32_t D = (16 + plan_digit_width(k) - 1) / plan_digit_width(k);
    // X (N*P) + spectrum (N*P) + Y (N*P*D) + four-step intermediate (N*P*D) + conv (N*P)
    return size_t(N) * P * (3 + 2 * size_t(D)) + 64 + P;
}

cudaError_t launch_plan_fast(const FastTables& t, const Tables& tab, const LogTables& lt, uint32_t N, uint32_t k,
                             uint32_t P, const uint32_t* pos, const uint32_t* Dh, uint32_t* scratch, uint32_t* ainv,
                             uint32_t* ahat, uint2* rowmap, uint2* ahat2, cudaStream_t st) {
    if (!P) return cudaSuccess;
    const uint32_t w = plan_digit_width(k), D = (16 + w - 1) / w;
    uint32_t* Xind = scratch;                   // [N][P]
    uint32_t* Xhat = Xind + size_t(N) * P;      // [N][P]
    uint32_t* Y = Xhat + size_t(N) * P;         // [N][P*D]
    uint32_t* tmp = Y + size_t(N) * P * D;      // four-step intermediate
    uint32_t* S = tmp + size_t(N) * P * D;      // [P]
    uint32_t* conv = S + P + 32;                // [P][N]
    cudaError_t err = cudaMemsetAsync(Xind, 0, sizeof(uint32_t) * N * size_t(P), st);
    if (err) return err;
    indicator_kernel<<<P, 256, 0, st>>>(N, k, P, pos, Xind, S);
    if ((err = run_cols<false>(t, N, LdPlain{Xind, P}, P, 1u, tmp, Xhat, st))) return err;
    const uint32_t ninv = cpow(N % kP, kP - 2);
    if ((err = run_cols<true>(t, N, LdSpectrumProduct{Xhat, Dh, P, D}, P * D, ninv, tmp, Y, st))) return err;
    conv_combine_kernel<<<dim3((P + 31) / 32, (N + 31) / 32), dim3(32, 8), 0, st>>>(N, P, D, w, Y, conv);
    fill_rowmap_kernel<<<148 * 8, 256, 0, st>>>(rowmap, uint64_t(P) * N);  // erased: {~0, 0}
    plan_ainv_kernel<<<148 * 8, 256, 0, st>>>(N, k, P, pos, S, conv, lt.exp3, ainv, rowmap);
    plan_ahat_kernel<<<148 * 8, 256, 0, st>>>(N, P, S, conv, rowmap, lt.exp3, kP - ninv, ahat, ahat2);
    return cudaGetLastError();
}

cudaError_t launch_fnt_cols(const FastTables& t, uint32_t N, bool inverse, uint32_t C, const uint32_t* in,
                            uint32_t* scratch, uint32_t* out, cudaStream_t st) {
    const uint32_t scale = inverse ? cpow(N % kP, kP - 2) : 1u;
    LdPlain ld{in, C};
    return inverse ? run_cols<true>(t, N, ld, C, scale, scratch, out, st)
                   : run_cols<false>(t, N, ld, C, scale, scratch, out, st);
}

}  // namespace fast
}  // namespace fntrs_gpu
