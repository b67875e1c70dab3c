// fnt_cols.cuh -- column-batched transforms: out[f][c] = FNT_N(column c)[f]
// over C columns of a row-major [N][C] array whose elements come from a
// loader functor ld(row, col) (values in [0, 2p)); outputs canonical, times
// `scale`. N <= 4096: one shared-memory tile kernel; 8192 <= N <= 65536: the
// four-step pair (size-N1 transforms, twiddle, size-N2 transforms) through an
// HBM intermediate. Used by the plan precompute (plan_fast.cu) and by the
// general codec path (codec_cols.cu).
#pragma once
#include <cuda_runtime.h>

#include "fft_pass.cuh"

namespace fntrs_gpu {
namespace fast {
namespace {

struct LdPlain {  // in[row * C + col]
    const uint32_t* in;
    uint32_t C;
    __device__ __forceinline__ uint32_t operator()(uint32_t row, uint32_t col) const { return in[size_t(row) * C + col]; }
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

}  // namespace
}  // namespace fast
}  // namespace fntrs_gpu
