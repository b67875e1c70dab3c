// codec_gen.cu -- fused decode for rates other than 1/2 (32 <= n_domain <= 4096,
// product size M = next_pow2(2k) != n_domain, M <= 4096).
//
// interp::interpolate (proj/src/interp.cpp:103-137) with two transform sizes:
// FNT1 is size N = n_domain (the moments of N'), FNT2 and the inverse FNT3
// are size M (the product A*S mod x^k). The fused rate-1/2 kernel
// (codec_fast.cu) runs all three in one shared tile and turns the series
// reversal into a view of that tile; here the sizes differ, so the CTA holds
// two tiles and one permuted gather moves the k series terms between them:
//   FNT1 (DIF, N-tile)     pass 0 scatters received row i to z_i times 1/A'
//   gather                 M-tile row q (DIT input order) = F[N-1-perm_M(q)]
//                          for perm_M(q) < k, else 0 (reversal + truncation)
//   FNT2 (DIT, M-tile)     forward, natural order out
//   IFNT3 (DIF, M-tile)    pass 0 loads times -A_hat/M; the last pass writes
//                          the k decoded packets (65536 escaped)
// Staging, persistence and escapes as in codec_fast.cu (one TMA stage issued
// after FNT1's first pass).
#include <cuda.h>
#include <cuda_runtime.h>

#include "fft_pass.cuh"
#include "tma.cuh"

namespace fntrs_gpu {
namespace fast {
namespace {

// tile width / threads / occupancy for the (N, M) pair: the widest tile whose
// two shared tiles fit the budget, at least 8 columns (the 16-byte TMA box
// minimum). Low rates (M < N) take 48 KB tiles (four CTAs per SM with the
// stage); high rates (M = 2N) keep 32-wide tiles at two CTAs per SM, which
// measured faster than narrower tiles at four (k = 200, n = 256: 133 vs 128 GB/s).
template <int E, int EM>
struct GenPick {
    static constexpr int rows = (1 << E) + (1 << EM);
    static constexpr int kBudget = (EM > E ? 100 : 48) * 1024;
    static constexpr int WT = rows * 32 * 4 <= kBudget ? 32 : (rows * 16 * 4 <= kBudget ? 16 : 8);
    static constexpr int NT = 256;
    static constexpr int MINB = rows * WT * 4 <= kBudget ? 4 : (rows * WT * 4 <= 2 * kBudget ? 2 : 1);
};

template <int E, int EM>
__global__ void __launch_bounds__(GenPick<E, EM>::NT, GenPick<E, EM>::MINB)
dec_gen_kernel(const __grid_constant__ CUtensorMap rx_map, const uint2* __restrict__ ptabF,
               const uint2* __restrict__ ptabI, const uint2* __restrict__ rowmap, const uint2* __restrict__ ahat2,
               uint32_t k, uint32_t L, uint32_t tps, uint32_t tiles, uint32_t nbox, uint32_t box_rows,
               const uint32_t* __restrict__ stripe_pattern, EscIn esc_in, uint16_t* __restrict__ out,
               EscOut esc_out, uint32_t* __restrict__ tile_ctr) {
    using Pk = GenPick<E, EM>;
    constexpr int WT = Pk::WT, NT = Pk::NT;
    using GA = Geom<E, WT, NT, Pk::MINB>;
    using GB = Geom<EM, WT, NT, Pk::MINB>;
    using SA = Sched<E>;
    using SB = Sched<EM>;
    constexpr int N = 1 << E, M = 1 << EM, PA = SA::P, PB = SB::P;
    constexpr int R0 = 1 << SA::rlog(0), SL0 = SA::slog(0);
    constexpr int RLB = GB::RLZ;
    static_assert(PA >= 2 && PA <= 3 && PB >= 1 && PB <= 3, "");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t next_tile[2];  // claimed successor of iteration i, slot i & 1 (tma.cuh)
    constexpr bool DYN = true;  // adjacent tiles stay in step (see codec_dec.cu)
    uint32_t* A = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* B = A + N * WT;
    const uint32_t stage_bytes = nbox * box_rows * WT * 2;
    // [guard | stage]: the guard row of ones under the stage is what an erased
    // position's row index ~0 wraps onto (raw words tested for zero unmasked)
    uint16_t* stage = reinterpret_cast<uint16_t*>(smem_raw + size_t(N + M) * WT * 4 + kGuardBytes);
    for (uint32_t i = threadIdx.x; i < uint32_t(WT); i += NT) stage[i - WT] = 1;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&rx_map);
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](uint32_t tl) {
        const uint32_t s1 = tl / tps;
        const uint32_t cc = (tl - s1 * tps) * WT;
        fence_proxy_async();
        mbar_expect_tx(&bar, stage_bytes);
        for (uint32_t j = 0; j < nbox; ++j)
            tma_load_2d(stage + j * box_rows * WT, &rx_map, int(cc), int(s1 * k + j * box_rows), &bar);
    };
    uint32_t tile = blockIdx.x;
    if (threadIdx.x == 0 && tile < tiles) issue(tile);
    const bool esc_any = esc_in.n != 0;
    for (uint32_t iter = 0; tile < tiles; tile = DYN ? next_tile[iter & 1] : tile + gridDim.x, ++iter) {
        const uint32_t stripe = tile / tps;
        const uint32_t c0 = (tile - stripe * tps) * WT;
        const uint32_t pat = __ldg(stripe_pattern + stripe);
        const uint32_t claimed = !DYN ? tile + gridDim.x : threadIdx.x == 0 ? claim_tile(tile_ctr) : 0u;
        const uint2* __restrict__ rm = rowmap + size_t(pat) * N;
        const uint2* __restrict__ ah = ahat2 + size_t(pat) * M;
        const unsigned long long key = uint64_t(stripe) * k * L + c0;
        uint16_t* outp = launder(out + key);
        mbar_wait(&bar, iter & 1);

        // ---- FNT1 = FNT_N(N'), DIF; pass 0 scatters and scales
        uint32_t zmin = 0xFFFFFFFFu;
        auto ld_scatter = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t {
            const uint2 m = __ldg(rm + lrow);
            const uint32_t raw = stage[int(m.x * uint32_t(WT) + col)];
            zmin = min(zmin, raw);
            return mulws(raw, m.y, m.y * 65535u);
        };
        auto fix_scatter = [&](uint32_t (&v)[R0], uint32_t base, uint32_t, uint32_t col) {
            const bool any = zmin == 0u;
            zmin = 0xFFFFFFFFu;
            if (!esc_any || !any) return;
#pragma unroll
            for (int q = 0; q < R0; ++q) {
                if (v[q] != 0u) continue;
                const uint2 m = __ldg(rm + base + (uint32_t(q) << SL0));
                if (m.x != 0xFFFFFFFFu && stage[m.x * WT + col] == 0u &&
                    esc_has(esc_in, key + uint64_t(m.x) * L + col))
                    v[q] = mulws(65536u, m.y, m.y * 65535u);
            }
        };
        auto ld_a = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return A[GA::idx(lrow, col)]; };
        auto st_a = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
            A[GA::idx(lrow, col)] = y;
            return 0u;
        };
        auto ld_b = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return B[GB::idx(lrow, col)]; };
        auto st_b = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
            B[GB::idx(lrow, col)] = y;
            return 0u;
        };
        pass<E, 0, false, false, k2P, kSmemCap, GA>(pass_table(ptabF, SA::llog(0)), ld_scatter, st_a, fix_scatter);
        __syncthreads();
        if (threadIdx.x == 0) {  // stage consumed
            if constexpr (DYN) next_tile[iter & 1] = claimed;
            if (claimed < tiles) issue(claimed);
        }
        pass<E, 1, false, false, kSmemCap, kSmemCap, GA>(pass_table(ptabF, SA::llog(1)), ld_a, st_a);
        __syncthreads();
        if constexpr (PA == 3) {
            pass<E, 2, false, false, kSmemCap, kSmemCap, GA>(pass_table(ptabF, SA::llog(2)), ld_a, st_a);
            __syncthreads();
        }

        // ---- series s'_j = F[N-1-j], j < k, in FNT2's DIT input order
        for (uint32_t it = threadIdx.x; it < uint32_t(M * WT); it += NT) {
            const uint32_t q = it / WT, col = it % WT;
            const uint32_t j = perm<EM>(q);
            B[GB::idx(q, col)] = j < k ? A[GA::idx(perm_inv<E>(uint32_t(N - 1) - j), col)] : 0u;
        }
        __syncthreads();

        // ---- FNT2 = FNT_M(s'), DIT passes PB-1 .. 0
        if constexpr (PB == 3) {
            pass<EM, 2, false, true, kSmemCap, kSmemCap, GB>(pass_table(ptabF, SB::llog(2)), ld_b, st_b);
            __syncthreads();
        }
        if constexpr (PB >= 2) {
            pass<EM, 1, false, true, kSmemCap, kSmemCap, GB>(pass_table(ptabF, SB::llog(1)), ld_b, st_b);
            __syncthreads();
        }
        pass<EM, 0, false, true, kSmemCap, kSmemCap, GB>(pass_table(ptabF, SB::llog(0)), ld_b, st_b);
        __syncthreads();

        // ---- IFNT3 (unscaled; -A_hat/M carries the scale), DIF; k packets out
        auto ld_ahat = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t {
            const uint2 a = __ldg(ah + lrow);
            return mulws(B[GB::idx(lrow, col)], a.x, a.y);
        };
        auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
            const uint32_t f = perm_head<EM>(b) + (uint32_t(s) << (EM - RLB));
            const bool keep = f < k;
            if (keep) __stcs(outp + (f * L + col), uint16_t(y));
            return keep ? y : 0u;  // canonical, kept: bit 16 set iff y == 65536
        };
        auto flush_out = [&](uint32_t mask, uint32_t, uint32_t b, uint32_t col) {
            if (!mask) return;
#pragma unroll 1
            for (int s = 0; s < 16; ++s)
                if (mask & (1u << s))
                    emit_escape(esc_out, key + uint64_t(perm_head<EM>(b) + (uint32_t(s) << (EM - RLB))) * L + col);
        };
        if constexpr (PB == 1) {
            pass<EM, 0, true, false, k2P, kCanon, GB>(pass_table(ptabI, SB::llog(0)), ld_ahat, st_out, NoFix(),
                                                       flush_out);
        } else {
            pass<EM, 0, true, false, k2P, kSmemCap, GB>(pass_table(ptabI, SB::llog(0)), ld_ahat, st_b);
            __syncthreads();
            if constexpr (PB == 3) {
                pass<EM, 1, true, false, kSmemCap, kSmemCap, GB>(pass_table(ptabI, SB::llog(1)), ld_b, st_b);
                __syncthreads();
            }
            pass<EM, PB - 1, true, false, kSmemCap, kCanon, GB>(pass_table(ptabI, SB::llog(PB - 1)), ld_b, st_out,
                                                                NoFix(), flush_out);
        }
        __syncthreads();
    }
}

// {balanced w, 65535 w} Shoup pairs of -A_hat/M, natural order
__global__ void gen_pairs_kernel(const uint32_t* __restrict__ ahat, uint2* __restrict__ pairs, uint64_t total) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < total; j += uint64_t(gridDim.x) * blockDim.x) {
        const int32_t a = balanced(ahat[j]);
        pairs[j] = make_uint2(uint32_t(a), uint32_t(a * 65535));
    }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t make_rx_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t L, uint32_t wt,
                        uint32_t box_rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {L, rows};
    const cuuint64_t strides[1] = {cuuint64_t(L) * 2};
    const cuuint32_t box[2] = {wt, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int E, int EM>
cudaError_t launch_gen(const FastTables& t, const GenPlanView& pv, uint32_t stripes, uint32_t L, const uint32_t* sp,
                       const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout, cudaStream_t st) {
    using Pk = GenPick<E, EM>;
    auto kern = dec_gen_kernel<E, EM>;
    const uint32_t tps = L / Pk::WT;
    const uint64_t tiles = uint64_t(stripes) * tps;
    if (!tiles) return cudaSuccess;
    if (tiles > 0xFFFFFFFFull) return cudaErrorInvalidConfiguration;
    const uint32_t box_rows = pv.k < 256 ? pv.k : 256;
    const uint32_t nbox = (pv.k + box_rows - 1) / box_rows;
    const size_t smem =
        size_t((1 << E) + (1 << EM)) * Pk::WT * 4 + kGuardBytes + size_t(nbox) * box_rows * Pk::WT * 2;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (err) return err;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, Pk::NT, smem))) return err;
    if (per < 1) return cudaErrorInvalidConfiguration;
    const uint64_t g = uint64_t(sms) * per;
    CUtensorMap map;
    if ((err = make_rx_map(&map, rx, uint64_t(stripes) * pv.k, L, Pk::WT, box_rows))) return err;
    TileCounter ctr;
    if ((err = ctr.get(st))) return err;
    kern<<<uint32_t(g < tiles ? g : tiles), Pk::NT, smem, st>>>(map, t.ptab_fwd, t.ptab_inv, pv.rowmap, pv.ahat2,
                                                                 pv.k, L, tps, uint32_t(tiles), nbox, box_rows, sp, ein,
                                                                 out, eout, ctr.p);
    return cudaGetLastError();
}

// supported (E, EM): k in (N/2, N] (EM = E+1, up to N = 1024: at N = 2048 the
// two tiles and the stage exceed 227 KB) and k in (N/16, N/4] (EM = E-1..E-3)
#define FNTRS_GEN_CASES(X)                                                                      \
    X(5, 6) X(5, 4) X(5, 3) X(5, 2) X(6, 7) X(6, 5) X(6, 4) X(6, 3) X(7, 8) X(7, 6) X(7, 5) X(7, 4) \
    X(8, 9) X(8, 7) X(8, 6) X(8, 5) X(9, 10) X(9, 8) X(9, 7) X(9, 6) X(10, 11) X(10, 9) X(10, 8)    \
    X(10, 7) X(11, 10) X(11, 9) X(11, 8) X(12, 11) X(12, 10) X(12, 9)

}  // namespace

int gen_tile_columns(uint32_t N, uint32_t M) {
#define FNTRS_GEN_WT(e, em) \
    if (N == (1u << e) && M == (1u << em)) return GenPick<e, em>::WT;
    FNTRS_GEN_CASES(FNTRS_GEN_WT)
#undef FNTRS_GEN_WT
    return 0;
}

cudaError_t build_gen_pairs(uint32_t M, uint32_t P, const uint32_t* ahat, uint2* pairs, cudaStream_t st) {
    if (!P) return cudaSuccess;
    gen_pairs_kernel<<<148 * 8, 256, 0, st>>>(ahat, pairs, uint64_t(P) * M);
    return cudaGetLastError();
}

cudaError_t launch_decode_gen(const FastTables& t, const GenPlanView& pv, uint32_t stripes, uint32_t L,
                              const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                              cudaStream_t st) {
#define FNTRS_GEN_LAUNCH(e, em) \
    if (pv.N == (1u << e) && pv.M == (1u << em)) return launch_gen<e, em>(t, pv, stripes, L, sp, rx, ein, out, eout, st);
    FNTRS_GEN_CASES(FNTRS_GEN_LAUNCH)
#undef FNTRS_GEN_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace fast
}  // namespace fntrs_gpu
