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

#include "fnt_cols.cuh"

namespace fntrs_gpu {
namespace fast {

namespace {

// ---------------------------------------------------------- column loaders ----
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
                            uint32_t* scratch, uint32_t* out, cudaStream_t st, bool unscaled) {
    const uint32_t scale = inverse && !unscaled ? cpow(N % kP, kP - 2) : 1u;
    LdPlain ld{in, C};
    return inverse ? run_cols<true>(t, N, ld, C, scale, scratch, out, st)
                   : run_cols<false>(t, N, ld, C, scale, scratch, out, st);
}

}  // namespace fast
}  // namespace fntrs_gpu
