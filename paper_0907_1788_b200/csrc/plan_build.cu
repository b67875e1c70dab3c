// plan_build.cu -- once-per-erasure-pattern decode precompute on the GPU.
//
// Replaces interp::build_plan (proj/src/interp.cpp:23-68). For a pattern
// with points x_l = r_N^(z_l), l < kp, the decoder needs
//   aprime_inv[i] = 1 / A'(x_i) = 1 / prod_{l != i} (x_i - x_l)
//   A_hat[j]      = A(w_j) = prod_l (w_j - x_l),  w_j = r_M^j, j < M
// where A = prod_l (x - x_l) is the erasure-locator polynomial (the root of
// the reference's subproduct tree, poly.cpp:216-242) and A_hat its size-M
// transform (the reference's a_fnt, interp.cpp:59-66, in natural order).
// Both are products of linear factors, computed here directly: one thread
// per evaluation point, the kp points staged in shared memory and read as
// warp broadcasts. The values are identical to the reference's (same field
// elements; evaluation is exact), which tests/ check against the oracle.
// The decoder consumes ahat pre-scaled by -1/M (series negation and the
// inverse-transform scale folded in).
#include <cuda_runtime.h>

#include "field.cuh"
#include "internal.h"

namespace fntrs_gpu {

namespace {

constexpr int kPlanThreads = 256;
constexpr uint32_t kPlanChunk = 16384;  // points staged in shared memory per round (64 KB)

// G lanes per evaluation point (G a power of two <= 32): lane `sub` of a group
// multiplies the factors l = sub, sub + G, ..., and the group combines its G
// partial products with shuffles. G > 1 only when the batch is too small to
// fill the GPU with one thread per point (a single pattern, as in C1).
__global__ void __launch_bounds__(kPlanThreads)
plan_kernel(uint32_t N, uint32_t M, uint32_t kp, uint32_t chunks, uint32_t lg, const uint32_t* __restrict__ positions,
            const uint32_t* __restrict__ twN, const uint32_t* __restrict__ twM, uint32_t neg_minv,
            uint32_t* __restrict__ ainv, uint32_t* __restrict__ ahat) {
    extern __shared__ uint32_t xs[];
    const uint32_t G = 1u << lg, sub = threadIdx.x & (G - 1);
    const uint32_t pat = blockIdx.x / chunks;
    const uint32_t chunk = blockIdx.x - pat * chunks;
    const uint32_t* pos = positions + size_t(pat) * kp;
    const uint32_t idx = chunk * (blockDim.x >> lg) + (threadIdx.x >> lg);
    const uint32_t npts = kp + M;
    const bool valid = idx < npts, self = idx < kp;
    const uint32_t y = !valid ? 0u : self ? __ldg(twN + __ldg(pos + idx)) : __ldg(twM + (idx - kp));
    // four independent accumulators for ILP; values stay in [0, 2p)
    uint32_t acc[4] = {1u, 1u, 1u, 1u};
    for (uint32_t c0 = 0; c0 < kp; c0 += kPlanChunk) {  // the points, a shared-memory chunk at a time
        const uint32_t cn = kp - c0 < kPlanChunk ? kp - c0 : kPlanChunk;
        __syncthreads();
        for (uint32_t l = threadIdx.x; l < cn; l += blockDim.x) xs[l] = __ldg(twN + __ldg(pos + c0 + l));
        __syncthreads();
        if (!valid) continue;
        uint32_t l = sub;
        for (; l + 3 * G < cn; l += 4 * G) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint32_t d = red2p(y + kP - xs[l + u * G]);  // y - x_l, canonical
                if (self) d = d ? d : 1u;                    // skip the l == i factor
                acc[u] = mulw(acc[u], d);
            }
        }
        for (; l < cn; l += G) {
            uint32_t d = red2p(y + kP - xs[l]);
            if (self) d = d ? d : 1u;
            acc[0] = mulw(acc[0], d);
        }
    }
    uint32_t prod = red2p(mulw(mulw(red2p(acc[0]), red2p(acc[1])), red2p(mulw(red2p(acc[2]), red2p(acc[3])))));
    for (uint32_t off = G >> 1; off; off >>= 1)  // groups are aligned within a warp; all lanes take part
        prod = red2p(mulw(prod, red2p(__shfl_xor_sync(0xFFFFFFFFu, prod, off))));
    if (!valid || sub) return;
    if (self) {
        ainv[size_t(pat) * kp + idx] = ginv(prod);
    } else {
        ahat[size_t(pat) * M + (idx - kp)] = red2p(mulw(prod, neg_minv));
    }
}

}  // namespace

cudaError_t launch_plan_build(uint32_t N, uint32_t M, uint32_t kp, uint32_t npatterns,
                              const uint32_t* positions, uint32_t* ainv, uint32_t* ahat,
                              const Tables& t, cudaStream_t st) {
    if (!npatterns) return cudaSuccess;
    const uint32_t npts = kp + M;
    // lanes per point: enough threads for ~148 SMs x 2048, at least 8 factors per lane
    uint32_t lg = 0;
    while (lg < 5 && (uint64_t(npatterns) * npts << lg) < 148ull * 2048 && (kp >> (lg + 1)) >= 8) ++lg;
    const uint32_t per_block = kPlanThreads >> lg;
    const uint32_t chunks = (npts + per_block - 1) / per_block;
    const uint64_t blocks = uint64_t(npatterns) * chunks;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    const size_t smem = size_t(kp < kPlanChunk ? kp : kPlanChunk) * 4;
    cudaError_t err = cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (err) return err;
    const uint32_t neg_minv = kP - cpow(M % kP, kP - 2);  // -1/M
    plan_kernel<<<unsigned(blocks), kPlanThreads, smem, st>>>(N, M, kp, chunks, lg, positions, t.fwd + N,
                                                               t.fwd + M, neg_minv, ainv, ahat);
    return cudaGetLastError();
}

}  // namespace fntrs_gpu
