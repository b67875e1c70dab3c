// codec_fast.cu -- fused encode kernels for 32 <= n_domain <= 4096 (v3), the
// per-pass twiddle tables and the plan tables of the fused decode (whose
// kernels are in codec_dec.cu).
//
// Persistent CTAs walk tiles (stripe, WT adjacent codewords). The k input
// packets of the NEXT tile are fetched by TMA (cp.async.bulk.tensor.2d, one
// 2-D box of <= 256 packets x WT symbols per request, completion on an
// mbarrier) while the CTA runs the transforms of the current tile, so HBM
// reads overlap the integer pipes: encode double-buffers the uint16 stage;
// decode reads its stage only in the first pass and reuses one buffer (the
// next load is issued after that pass), which fits five CTAs per SM.
// One work item = one radix-R butterfly of one codeword (thread = codeword,
// warp = 32 adjacent codewords, conflict-free 32-bit shared-memory rows);
// encode at n_domain <= 256 takes two codewords per item in a 64-wide tile.
//
// Encode  (codec::encode_nonsystematic, proj/src/codec.cpp:124-131):
//   pass 0 reads the staged source rows (the zero padding rows >= k are
//   never touched), the middle passes run in the shared tile, the last pass
//   writes the n output packets to global memory in natural order,
//   canonical, with 65536 escapes emitted (proj/src/shardio.cpp:131-137).
// Decode  (interp::interpolate, proj/src/interp.cpp:103-137, per codeword):
//   FNT1 pass 0 scatters received row i to position z_i scaled by
//   1/A'(x_i); FNT1's last pass and FNT2's first DIT pass are fused in
//   registers (s'_j = F[N-1-j] is a reversal of the butterfly group; j >= k
//   zeroed); FNT2's last DIT pass, the product with A_hat and FNT3's first
//   DIF pass are fused in registers; FNT3's last pass writes the k decoded
//   packets.
// Encode computes q * p (Shoup products, signed reductions) as one LEA on the
// ALU pipe (field.cuh, FNTRS_LEA): C2 encode 944 -> 972 GB/s (the decode unit,
// codec_dec.cu, keeps the IMAD form: its ALU pipe is the fuller one).
#ifndef FNTRS_LEA
#define FNTRS_LEA 1
#endif
// Two-codeword encode items pin the second codeword's butterfly adds to the ALU
// pipe and leave the first to ptxas, which otherwise moves ~1200 adds per 32
// codewords onto the multiplier pipe as IMAD.IADD (C2 encode 976 -> 1023 GB/s).
#ifndef FNTRS_SPLIT_PIN
#define FNTRS_SPLIT_PIN 1
#endif
// One-codeword items (n_domain >= 512) pin the adds of the second 4 x 4 stage of
// each radix-16 to the ALU (fft_pass.cuh): encode n = 4096 476 -> 492,
// n = 1024 530 -> 545, n = 2048 523 -> 528 GB/s (pinning both stages: 479 / 538 / 538)
#ifndef FNTRS_CW1_PIN
#define FNTRS_CW1_PIN 2
#endif
// ... and the first codeword of a two-codeword item pins its second stage too
// (the second codeword pins both): C2 encode 1010 -> 1020, n = 128 859 -> 884 GB/s
#ifndef FNTRS_CW2_PIN0
#define FNTRS_CW2_PIN0 2
#endif
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <type_traits>

#include "fft_pass.cuh"
#include "launch_util.cuh"
#include "tma.cuh"

namespace fntrs_gpu {
namespace fast {

namespace {

// ---------------------------------------------------------------------------
// Encode geometry: at N <= 256 a 64-column tile with two codewords per work
// item (columns c and c + 32 share twiddle loads and addressing; C2 encode
// 693 -> 716 GB/s); larger N keep the decode geometry (a 64-wide N = 512 tile
// and its staging exceed shared memory).
#ifndef FNTRS_ENC_CW
#define FNTRS_ENC_CW 2
#endif
#ifndef FNTRS_ENC_NT
#define FNTRS_ENC_NT 256
#endif
template <int E>
struct EncPick {
    static constexpr int CW = E <= 8 ? FNTRS_ENC_CW : 1;
    // output rows through shared memory + one TMA store per tile: C2 encode
    // 711 -> 819 GB/s (per-symbol 2-byte stores were the bottleneck); not at N = 32 (-2 %)
    static constexpr bool TS = E >= 6;
    using G = typename std::conditional<(E <= 8), Geom<E, 64, FNTRS_ENC_NT, 2>, typename Pick<E>::G>::type;
};

// TS: single input stage + the n output rows staged in shared memory and
// written by one TMA tensor store per tile (instead of per-symbol stores).
template <int E, class G, bool HALFK, bool PUNCT, int CW, bool TS = false>
__global__ void __launch_bounds__(G::NT, G::MINB) enc_fast_kernel(const __grid_constant__ CUtensorMap src_map,
                                                         const uint2* __restrict__ ptabF, uint32_t k, uint32_t n,
                                                         uint32_t L, uint32_t tps, uint32_t tiles, uint32_t nbox,
                                                         uint32_t box_rows, EscIn esc_in, uint16_t* __restrict__ out,
                                                         EscOut esc_out, const __grid_constant__ CUtensorMap out_map,
                                                         uint32_t obox, uint32_t* __restrict__ tile_ctr) {
    using S = Sched<E>;
    constexpr int N = 1 << E, WT = G::WT, P = S::P;
    constexpr int RL0 = S::rlog(0), R0 = 1 << RL0, RLZ = G::RLZ;
    static_assert(P >= 2 && P <= 3, "");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ uint32_t next_tile[2];  // successor of the tile of iteration i, in slot i & 1
    uint32_t* work = reinterpret_cast<uint32_t*>(smem_raw);
    uint16_t* stage0 = reinterpret_cast<uint16_t*>(smem_raw + size_t(N) * WT * 4);
    const uint32_t stage_elems = nbox * box_rows * WT;
    const uint32_t stage_bytes = stage_elems * 2;
    // TS: [work | stage | out_s], out_s 128-byte aligned
    uint16_t* out_s = reinterpret_cast<uint16_t*>(
        smem_raw + ((size_t(N) * WT * 4 + size_t(stage_bytes) + 127) & ~size_t(127)));
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&src_map);
        if constexpr (TS) tma_prefetch_desc(&out_map);
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](uint32_t tl, int bs) {
        const uint32_t s1 = tl / tps;
        const uint32_t cc = (tl - s1 * tps) * WT;
        fence_proxy_async();
        mbar_expect_tx(&bars[bs], stage_bytes);
        uint16_t* dst = stage0 + bs * stage_elems;
        for (uint32_t j = 0; j < nbox; ++j)
            tma_load_2d(dst + j * box_rows * WT, &src_map, int(cc), int(s1 * k + j * box_rows), &bars[bs]);
    };
    uint32_t tile = blockIdx.x;
    if (threadIdx.x == 0 && tile < tiles) issue(tile, 0);
    const bool esc_any = esc_in.n != 0;
    // tiles are claimed from a counter at every occupancy (as in dec_fast_kernel)
    constexpr bool DYN = true;
    for (uint32_t iter = 0; tile < tiles; tile = DYN ? next_tile[iter & 1] : tile + gridDim.x, ++iter) {
        const int bsel = TS ? 0 : (iter & 1);
        const uint32_t stripe = tile / tps;
        const uint32_t c0 = (tile - stripe * tps) * WT;
        const uint32_t claimed = !DYN ? tile + gridDim.x : threadIdx.x == 0 ? claim_tile(tile_ctr) : 0u;
        if (!TS && threadIdx.x == 0) {
            if constexpr (DYN) next_tile[iter & 1] = claimed;
            if (claimed < tiles) issue(claimed, bsel ^ 1);
        }
        mbar_wait(&bars[bsel], TS ? (iter & 1) : ((iter >> 1) & 1));
        const uint16_t* st_in = stage0 + bsel * stage_elems;
        const unsigned long long key_in = uint64_t(stripe) * k * L + c0;
        const unsigned long long key_out = uint64_t(stripe) * n * L + c0;
        uint16_t* outp = launder(out + key_out);

        auto ld_src = [&](uint32_t lrow, uint32_t, int q, uint32_t col) -> uint32_t {
            if ((HALFK && q >= R0 / 2) || (!HALFK && lrow >= k)) return 0u;
            return st_in[lrow * WT + col];
        };
        auto fix_src = [&](uint32_t (&v)[R0], uint32_t base, uint32_t, uint32_t col) {
            if (!esc_any) return;
            if (!any_zero(v)) return;
#pragma unroll
            for (int q = 0; q < R0; ++q) {
                const uint32_t lrow = base + (uint32_t(q) << S::slog(0));
                if (v[q] == 0u && lrow < k && esc_has(esc_in, key_in + uint64_t(lrow) * L + col)) v[q] = 65536u;
            }
        };
        auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
        auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
            work[G::idx(lrow, col)] = y;
            return 0u;
        };
        auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
            const uint32_t f = perm_head<E>(b) + (uint32_t(s) << (E - RLZ));
            if constexpr (TS) {
                out_s[f * WT + col] = uint16_t(y);  // rows >= n are outside the store box
            } else {
                if (!PUNCT || f < n) __stcs(outp + (f * L + col), uint16_t(y));
            }
            return (!PUNCT || f < n) ? y : 0u;  // canonical, kept: bit 16 set iff y == 65536
        };
        auto flush_out = [&](uint32_t mask, uint32_t, uint32_t b, uint32_t col) {
            if (!mask) return;
#pragma unroll 1
            for (int s = 0; s < 16; ++s)
                if (mask & (1u << s))
                    emit_escape(esc_out, key_out + uint64_t(perm_head<E>(b) + (uint32_t(s) << (E - RLZ))) * L + col);
        };

        pass_cw<CW, E, 0, false, false, kP64, kSmemCap, G>(pass_table(ptabF, S::llog(0)), ld_src, st_sm, fix_src);
        if constexpr (TS) {
            if (threadIdx.x == 0) bulk_wait_read();  // the previous tile's store has read out_s
        }
        __syncthreads();
        if constexpr (TS) {  // the stage is consumed: the next tile's packets stream in behind
            if (threadIdx.x == 0) {
                if constexpr (DYN) next_tile[iter & 1] = claimed;
                if (claimed < tiles) issue(claimed, 0);
            }
        }
        if constexpr (P == 3) {
            pass_cw<CW, E, 1, false, false, kSmemCap, kSmemCap, G>(pass_table(ptabF, S::llog(1)), ld_sm, st_sm);
            __syncthreads();
        }
        pass_cw<CW, E, P - 1, false, false, kSmemCap, kCanon, G>(pass_table(ptabF, S::llog(P - 1)), ld_sm, st_out,
                                                                NoFix(), flush_out);
        if constexpr (TS) fence_proxy_async();  // generic writes of out_s before the async-proxy store
        __syncthreads();
        if constexpr (TS) {
            if (threadIdx.x == 0) {
                for (uint32_t r0 = 0; r0 < n; r0 += obox) tma_store_3d(&out_map, out_s + r0 * WT, int(c0), int(r0), int(stripe));
                bulk_commit();
            }
        }
    }
    if constexpr (TS) {
        if (threadIdx.x == 0) bulk_wait_all();
    }
}

// per-pass twiddle tables: [2^LL + t*16 + s] = r_(2^LL)^(t*s) for LL <= 12
__global__ void ptab_kernel(uint2* fwd, uint2* inv) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 32 || i >= (1u << 13)) return;
    const int LL = 31 - __clz(i);
    const uint32_t j = i - (1u << LL), t = j >> 4, s = j & 15u;
    const uint32_t ex = ((t * s) << (16 - LL)) & 0xFFFFu;  // r_len = 3^(65536/len)
    const int32_t wf = balanced(gpow(3u, ex)), wi = balanced(gpow(3u, (65536u - ex) & 0xFFFFu));
    fwd[i] = make_uint2(uint32_t(wf), uint32_t(wf * 65535));
    inv[i] = make_uint2(uint32_t(wi), uint32_t(wi * 65535));
}

// transposed pass-0 twiddles for N = 2^LL <= 256: [N + (N/16) s + t] = r_N^(t s)
__global__ void ptab_t_kernel(uint2* fwdT) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 32 || i >= (1u << 9)) return;
    const int LL = 31 - __clz(i);
    const uint32_t sub = 1u << (LL - 4), j = i - (1u << LL), s = j / sub, t = j % sub;
    const uint32_t ex = ((t * s) << (16 - LL)) & 0xFFFFu;
    const int32_t w = balanced(gpow(3u, ex));
    fwdT[i] = make_uint2(uint32_t(w), uint32_t(w * 65535));
}

__global__ void fast_plan_tables_kernel(uint32_t N, const uint32_t* __restrict__ ahat, uint2* __restrict__ rowmap,
                                        uint2* __restrict__ ahat2, uint64_t total) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < total; j += uint64_t(gridDim.x) * blockDim.x) {
        rowmap[j] = make_uint2(0xFFFFFFFFu, 0u);
        const int32_t a = balanced(ahat[j]);  // signed Shoup pair
        ahat2[(j & ~uint64_t(N - 1)) | ahat2_slot(N, uint32_t(j) & (N - 1))] = make_uint2(uint32_t(a), uint32_t(a * 65535));
    }
}

__global__ void fast_plan_scatter_kernel(uint32_t N, uint32_t kp, const uint32_t* __restrict__ pos,
                                         const uint32_t* __restrict__ ainv, uint2* __restrict__ rowmap, uint64_t total) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < total; j += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t p = j / kp;
        const uint32_t i = uint32_t(j - p * kp);
        rowmap[p * N + pos[j]] = make_uint2(i, uint32_t(balanced(ainv[j])));
    }
}

template <int E, bool TS>
cudaError_t launch_enc_as(const FastTables& t, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                          const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, cudaStream_t st) {
    using G = typename EncPick<E>::G;
    constexpr int CW = EncPick<E>::CW;
    const bool half = k == (1u << E) / 2, punct = n < (1u << E);
    auto kern = half ? (punct ? enc_fast_kernel<E, G, true, true, CW, TS> : enc_fast_kernel<E, G, true, false, CW, TS>)
                     : (punct ? enc_fast_kernel<E, G, false, true, CW, TS> : enc_fast_kernel<E, G, false, false, CW, TS>);
    LaunchShape sh;
    const size_t out_stage = TS ? (size_t(2) << E) * G::WT + 128 : 0;
    cudaError_t err = shape_for(kern, E, G::WT, G::NT, k, stripes, L, sh, out_stage, TS ? 1 : 2);
    if (err) return err;
    if (!sh.tiles) return cudaSuccess;
    CUtensorMap map, omap;
    std::memset(&omap, 0, sizeof(omap));
    if ((err = make_map(&map, src, uint64_t(stripes) * k, L, G::WT, sh.box_rows))) return err;
    const uint32_t obox = n < 256 ? n : 256;
    if (TS && (err = make_map3(&omap, out, stripes, n, L, G::WT, obox))) return err;
    TileCounter ctr;
    if ((err = ctr.get(st))) return err;
    kern<<<sh.grid, G::NT, sh.smem, st>>>(map, t.ptab_fwd, k, n, L, sh.tps, sh.tiles, sh.nbox, sh.box_rows, ein, out, eout,
                                          omap, obox, ctr.p);
    return cudaGetLastError();
}

template <int E>
cudaError_t launch_enc(const FastTables& t, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L, const uint16_t* src,
                       EscIn ein, uint16_t* out, EscOut eout, cudaStream_t st) {
    using G = typename EncPick<E>::G;
    if constexpr (EncPick<E>::TS) {
        // staged output when tile + one input stage + the n-row output tile fit
        const uint32_t box_rows = k < 256 ? k : 256, nbox = (k + box_rows - 1) / box_rows;
        const size_t need = (size_t(1) << E) * G::WT * 4 + size_t(nbox) * box_rows * G::WT * 2 +
                            (size_t(2) << E) * G::WT + 128;
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (need <= size_t(optin)) return launch_enc_as<E, true>(t, k, n, stripes, L, src, ein, out, eout, st);
    }
    return launch_enc_as<E, false>(t, k, n, stripes, L, src, ein, out, eout, st);
}

}  // namespace

cudaError_t build_fast_tables(FastTables& t, cudaStream_t st) {
    cudaError_t err = cudaMalloc(&t.ptab_fwd, sizeof(uint2) << 13);
    if (err) return err;
    if ((err = cudaMalloc(&t.ptab_inv, sizeof(uint2) << 13))) return err;
    if ((err = cudaMalloc(&t.ptab_fwdT, sizeof(uint2) << 9))) return err;
    ptab_kernel<<<(1u << 13) / 256, 256, 0, st>>>(t.ptab_fwd, t.ptab_inv);
    ptab_t_kernel<<<2, 256, 0, st>>>(t.ptab_fwdT);
    if ((err = cudaGetLastError())) return err;
    return build_sys_conv(t, st);
}

int fast_encode_columns(uint32_t N) {
    switch (N) {
        case 32: return EncPick<5>::G::WT;
        case 64: return EncPick<6>::G::WT;
        case 128: return EncPick<7>::G::WT;
        case 256: return EncPick<8>::G::WT;
        case 512: return EncPick<9>::G::WT;
        case 1024: return EncPick<10>::G::WT;
        case 2048: return EncPick<11>::G::WT;
        case 4096: return EncPick<12>::G::WT;
        default: return 0;
    }
}

int fast_tile_columns(uint32_t N) {
    switch (N) {
        case 32: return Pick<5>::WT;
        case 64: return Pick<6>::WT;
        case 128: return Pick<7>::WT;
        case 256: return Pick<8>::WT;
        case 512: return Pick<9>::WT;
        case 1024: return Pick<10>::WT;
        case 2048: return Pick<11>::WT;
        case 4096: return Pick<12>::WT;
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

cudaError_t launch_fast_plan_tables(uint32_t N, uint32_t kp, uint32_t npatterns, const uint32_t* pos,
                                    const uint32_t* ainv, const uint32_t* ahat, uint2* rowmap, uint2* ahat2,
                                    cudaStream_t st) {
    if (!npatterns) return cudaSuccess;
    const uint64_t total = uint64_t(npatterns) * N;
    fast_plan_tables_kernel<<<148 * 8, 256, 0, st>>>(N, ahat, rowmap, ahat2, total);
    fast_plan_scatter_kernel<<<148 * 8, 256, 0, st>>>(N, kp, pos, ainv, rowmap, uint64_t(npatterns) * kp);
    return cudaGetLastError();
}

}  // namespace fast
}  // namespace fntrs_gpu
