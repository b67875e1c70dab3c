// codec_cols.cu -- the general codec path: every shape the fused kernels
// (codec_fast.cu, codec_large.cu) do not serve, up to n_domain = 65536 and
// product size M = next_pow2(2k) <= 65536:
//   * M != n_domain with n_domain or M above 4096 (rates other than 1/2 at
//     large sizes: k <= n_domain/4, or k > n_domain/2),
//   * complete reception (decode = one inverse transform, codec.cpp:137-144)
//     at n_domain >= 8192,
//   * n_domain >= 8192 with L not a multiple of the four-step tile width.
//
// The codewords of a batch of stripes are the C columns of row-major
// [rows][C] uint32 arrays in HBM (global codeword g = stripe * L + symbol).
// Every step of interp::interpolate (interp.cpp:103-137) is one column
// transform (fnt_cols.cuh) whose loader fuses the elementwise step before it:
//   FNT1 = FNT_N(N')     loader: scatter row rowmap[z] of the received
//                        packets times 1/A'(x_i)              (step 4)
//   FNT2 = FNT_M(s')     loader: s'_j = F[N-1-j] for j < k, 0 above
//                        (step 5 via the transform identity, truncation)
//   IFNT3 (unscaled)     loader: FNT2 output times -A_hat_j / M   (step 6)
// and a final kernel writes the first k rows as uint16 packets with the
// 65536 escape list. Encode is FNT_N of the zero-padded source columns
// (codec.cpp:124-131) written out as n rows.
//
// 2k > 65536 (no product transform fits; the reference's poly::mul_low,
// poly.cpp:139-169): P = A_lo S_lo + x^h (A_lo S_hi + A_hi S_lo) mod x^k with
// h = ceil(k/2); every partial product has fewer than 65536 coefficients, so
// each is exact as a size-65536 cyclic convolution. Per codeword: FNT1, the
// spectra of S_lo and S_hi, and two unscaled inverses (lo*lo, and the two
// cross terms summed in the frequency domain); the locator halves' spectra
// -A_lo^/M and -A_hi^/M are per-pattern plan data (build_split_spectra).
#include <cuda_runtime.h>

#include "fnt_cols.cuh"
#include "internal.h"

namespace fntrs_gpu {
namespace fast {
namespace {

struct Col {  // global codeword index -> (stripe, symbol)
    uint64_t g0;
    uint32_t L;
    __device__ __forceinline__ void at(uint32_t col, uint64_t& s, uint32_t& c) const {
        const uint64_t g = g0 + col;
        s = g / L;
        c = uint32_t(g - s * L);
    }
};

__device__ __forceinline__ uint32_t fetch(const uint16_t* p, const EscIn& esc, uint64_t key) {
    const uint32_t v = p[key];
    return (v == 0u && esc.n && esc_has(esc, key)) ? 65536u : v;
}

// FNT1 input N'[z]: the packet received at position z times 1/A'(x_i)
// (rowmap[z] = {row i, balanced 1/A'} or {~0, 0} when z was erased).
struct LdScatter {
    Col col;
    const uint2* rowmap;
    const uint32_t* sp;
    const uint16_t* rx;
    EscIn esc;
    uint32_t N, kp;
    __device__ __forceinline__ uint32_t operator()(uint32_t z, uint32_t c_) const {
        uint64_t s;
        uint32_t c;
        col.at(c_, s, c);
        const uint2 m = __ldg(rowmap + size_t(__ldg(sp + s)) * N + z);
        if (m.x == 0xFFFFFFFFu) return 0u;
        const uint32_t v = fetch(rx, esc, (s * kp + m.x) * col.L + c);
        return canon_s2p(mulws(v, m.y, m.y * 65535u));
    }
};

// FNT2 input: s'_j = F[N-1-j] for j < k (the series, truncated), else 0
struct LdRevTrunc {
    const uint32_t* F;
    uint32_t C, N, k;
    __device__ __forceinline__ uint32_t operator()(uint32_t j, uint32_t c) const {
        return j < k ? F[size_t(N - 1u - j) * C + c] : 0u;
    }
};

// IFNT3 input: FNT2 output times -A_hat_j / M of the codeword's pattern
struct LdAhat {
    Col col;
    const uint32_t* Y;
    const uint32_t* ahat;
    const uint32_t* sp;
    uint32_t C, M;
    __device__ __forceinline__ uint32_t operator()(uint32_t j, uint32_t c_) const {
        uint64_t s;
        uint32_t c;
        col.at(c_, s, c);
        return mulw(Y[size_t(j) * C + c_], __ldg(ahat + size_t(__ldg(sp + s)) * M + j));
    }
};

// s'_{j+off} = F[N-1-(j+off)] for j < cnt, else 0 (a slice of the series)
struct LdRevSlice {
    const uint32_t* F;
    uint32_t C, N, off, cnt;
    __device__ __forceinline__ uint32_t operator()(uint32_t j, uint32_t c) const {
        return j < cnt ? F[size_t(N - 1u - off - j) * C + c] : 0u;
    }
};

// split product inputs: X1 * W1[pattern] (+ X2 * W2[pattern]); W are [M][P] columns
struct LdSplit {
    Col col;
    const uint32_t *X1, *X2, *W1, *W2;
    const uint32_t* sp;
    uint32_t C, P;
    __device__ __forceinline__ uint32_t operator()(uint32_t j, uint32_t c_) const {
        uint64_t s;
        uint32_t c;
        col.at(c_, s, c);
        const size_t w = size_t(j) * P + __ldg(sp + s);
        uint32_t v = mulw(X1[size_t(j) * C + c_], __ldg(W1 + w));
        if (X2) v = red2p(red2p(v) + red2p(mulw(X2[size_t(j) * C + c_], __ldg(W2 + w))));
        return v;
    }
};

// plan arrays [P][M] read as columns (row t of pattern p)
struct LdPatternRows {
    const uint32_t* in;
    uint32_t M;
    __device__ __forceinline__ uint32_t operator()(uint32_t t, uint32_t p) const { return in[size_t(p) * M + t]; }
};

// locator halves from its coefficients c[t][p] (= -a_t): lo = t < h, hi = h + t <= k
struct LdLocatorHalf {
    const uint32_t* c;
    uint32_t P, h, k;
    bool hi;
    __device__ __forceinline__ uint32_t operator()(uint32_t t, uint32_t p) const {
        if (!hi) return t < h ? c[size_t(t) * P + p] : 0u;
        return h + t <= k ? c[size_t(h + t) * P + p] : 0u;
    }
};

// P[j] = U[j] + V[j - h] (j >= h), j < rows -> packets, as out_rows_kernel
__global__ void out_split_kernel(const uint32_t* __restrict__ U, const uint32_t* __restrict__ V, uint32_t C,
                                 uint32_t rows, uint32_t h, Col col, uint16_t* __restrict__ out, EscOut eout) {
    const uint64_t total = uint64_t(rows) * C;
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t f = uint32_t(t / C), c_ = uint32_t(t - uint64_t(f) * C);
        uint64_t s;
        uint32_t c;
        col.at(c_, s, c);
        uint32_t y = U[t];
        if (f >= h) y = red2p(y + V[uint64_t(f - h) * C + c_]);
        const uint64_t key = (s * rows + f) * col.L + c;
        out[key] = uint16_t(y);
        if (y == 65536u) emit_escape(eout, key);
    }
}

// encode input: source row i < k of the codeword, zero padded to N
struct LdSource {
    Col col;
    const uint16_t* src;
    EscIn esc;
    uint32_t k;
    __device__ __forceinline__ uint32_t operator()(uint32_t i, uint32_t c_) const {
        if (i >= k) return 0u;
        uint64_t s;
        uint32_t c;
        col.at(c_, s, c);
        return fetch(src, esc, (s * k + i) * col.L + c);
    }
};

// rows f < rows of Z [.][C] -> packets out[stripe][f][symbol] (uint16, 65536 escaped)
__global__ void out_rows_kernel(const uint32_t* __restrict__ Z, uint32_t C, uint32_t rows, Col col,
                                uint16_t* __restrict__ out, EscOut eout) {
    const uint64_t total = uint64_t(rows) * C;
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t f = uint32_t(t / C), c_ = uint32_t(t - uint64_t(f) * C);
        uint64_t s;
        uint32_t c;
        col.at(c_, s, c);
        const uint32_t y = Z[t];
        const uint64_t key = (s * rows + f) * col.L + c;
        out[key] = uint16_t(y);
        if (y == 65536u) emit_escape(eout, key);
    }
}

__global__ void rowmap_fill_kernel(uint2* p, uint64_t n) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n; j += uint64_t(gridDim.x) * blockDim.x)
        p[j] = make_uint2(0xFFFFFFFFu, 0u);
}

// rowmap[p][pos[p][i]] = {i, balanced 1/A'(x_i)} (ainv null: complete reception, scale 1)
__global__ void rowmap_scatter_kernel(uint32_t N, uint32_t kp, const uint32_t* __restrict__ pos,
                                      const uint32_t* __restrict__ ainv, uint2* __restrict__ rowmap, uint64_t total) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < total; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t p = j / kp;
        const uint32_t i = uint32_t(j - p * kp);
        const uint32_t a = ainv ? ainv[j] : 1u;
        rowmap[p * N + pos[j]] = make_uint2(i, uint32_t(balanced(a)));
    }
}

constexpr int kOutThreads = 256;
constexpr int kOutBlocks = 148 * 8;

}  // namespace

cudaError_t build_split_spectra(const FastTables& t, uint32_t k, uint32_t P, const uint32_t* ahat, uint32_t* alo,
                                uint32_t* ahi, uint32_t* c, uint32_t* T, cudaStream_t st) {
    constexpr uint32_t M = 65536;
    if (!P) return cudaSuccess;
    const uint32_t h = (k + 1) / 2, minv = cpow(M % kP, kP - 2);
    // c = IFNT_unscaled(ahat) = -a_t (ahat = -A^/M and deg A = k < M: no wrap)
    cudaError_t err = run_cols<true>(t, M, LdPatternRows{ahat, M}, P, 1u, T, c, st);
    if (!err) err = run_cols<false>(t, M, LdLocatorHalf{c, P, h, k, false}, P, minv, T, alo, st);
    if (!err) err = run_cols<false>(t, M, LdLocatorHalf{c, P, h, k, true}, P, minv, T, ahi, st);
    return err;
}

uint64_t cols_batch_columns(uint32_t D, size_t cap_bytes) {
    const uint64_t c = cap_bytes / (uint64_t(D) * 4);
    return c >= 32 ? c / 32 * 32 : 32;
}

cudaError_t build_cols_rowmap(uint32_t N, uint32_t kp, uint32_t P, const uint32_t* pos, const uint32_t* ainv,
                              uint2* rowmap, cudaStream_t st) {
    if (!P) return cudaSuccess;
    rowmap_fill_kernel<<<kOutBlocks, kOutThreads, 0, st>>>(rowmap, uint64_t(P) * N);
    rowmap_scatter_kernel<<<kOutBlocks, kOutThreads, 0, st>>>(N, kp, pos, ainv, rowmap, uint64_t(P) * kp);
    return cudaGetLastError();
}

cudaError_t launch_encode_cols(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes, uint32_t L,
                               const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, uint32_t* A, uint32_t* T,
                               uint64_t cap_cols, cudaStream_t st) {
    const uint64_t total = uint64_t(stripes) * L;
    for (uint64_t g0 = 0; g0 < total; g0 += cap_cols) {
        const uint32_t C = uint32_t(total - g0 < cap_cols ? total - g0 : cap_cols);
        const Col col{g0, L};
        cudaError_t err = run_cols<false>(t, N, LdSource{col, src, ein, k}, C, 1u, T, A, st);
        if (err) return err;
        out_rows_kernel<<<kOutBlocks, kOutThreads, 0, st>>>(A, C, n, col, out, eout);
    }
    return cudaGetLastError();
}

cudaError_t launch_decode_cols(const FastTables& t, const ColsPlanView& pv, uint32_t stripes, uint32_t L,
                               const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                               uint32_t* A, uint32_t* B, uint32_t* X, uint32_t* T, uint64_t cap_cols,
                               cudaStream_t st) {
    const uint64_t total = uint64_t(stripes) * L;
    const uint32_t N = pv.N, M = pv.M, k = pv.k;
    for (uint64_t g0 = 0; g0 < total; g0 += cap_cols) {
        const uint32_t C = uint32_t(total - g0 < cap_cols ? total - g0 : cap_cols);
        const Col col{g0, L};
        const LdScatter scatter{col, pv.rowmap, sp, rx, ein, N, pv.kp};
        cudaError_t err;
        if (pv.full) {  // all n = N positions: coefficients = FNT_N^-1 of the received values
            err = run_cols<true>(t, N, scatter, C, cpow(N % kP, kP - 2), T, A, st);
        } else if (pv.split) {  // 2k > 65536: mul_low by halves (N = M = 65536)
            const uint32_t h = (k + 1) / 2;
            if ((err = run_cols<false>(t, N, scatter, C, 1u, T, A, st))) return err;
            if ((err = run_cols<false>(t, M, LdRevSlice{A, C, N, 0, h}, C, 1u, T, B, st))) return err;      // S_lo^
            if ((err = run_cols<false>(t, M, LdRevSlice{A, C, N, h, k - h}, C, 1u, T, X, st))) return err;  // S_hi^
            // U = -(A_lo S_lo) into A; V = -(A_lo S_hi + A_hi S_lo) into B (read fully before written)
            if ((err = run_cols<true>(t, M, LdSplit{col, B, nullptr, pv.alo, nullptr, sp, C, pv.np}, C, 1u, T, A, st)))
                return err;
            if ((err = run_cols<true>(t, M, LdSplit{col, X, B, pv.alo, pv.ahi, sp, C, pv.np}, C, 1u, T, B, st)))
                return err;
            out_split_kernel<<<kOutBlocks, kOutThreads, 0, st>>>(A, B, C, k, h, col, out, eout);
            continue;
        } else {
            if ((err = run_cols<false>(t, N, scatter, C, 1u, T, A, st))) return err;
            if ((err = run_cols<false>(t, M, LdRevTrunc{A, C, N, k}, C, 1u, T, B, st))) return err;
            err = run_cols<true>(t, M, LdAhat{col, B, pv.ahat, sp, C, M}, C, 1u, T, A, st);  // ahat holds -1/M
        }
        if (err) return err;
        out_rows_kernel<<<kOutBlocks, kOutThreads, 0, st>>>(A, C, k, col, out, eout);
    }
    return cudaGetLastError();
}

}  // namespace fast
}  // namespace fntrs_gpu
