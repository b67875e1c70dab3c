// codec_fast.cu -- fused encode / decode kernels for 32 <= n_domain <= 4096 (v3).
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
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <type_traits>

#include "fft_pass.cuh"
#include "tma.cuh"

namespace fntrs_gpu {
namespace fast {

namespace {

// ---------------------------------------------------------------------------
// Encode geometry: at N <= 256 a 64-column tile with two codewords per work
// item (columns c and c + 32 share twiddle loads and addressing; C2 encode
// 693 -> 716 GB/s); larger N keep the decode geometry (a 64-wide N = 512 tile
// and its staging exceed shared memory).
template <int E>
struct EncPick {
    static constexpr int CW = E <= 8 ? 2 : 1;
    // output rows through shared memory + one TMA store per tile: C2 encode
    // 711 -> 819 GB/s (per-symbol 2-byte stores were the bottleneck); not at N = 32 (-2 %)
    static constexpr bool TS = E >= 6;
    using G = typename std::conditional<(E <= 8), Geom<E, 64, 256, 2>, typename Pick<E>::G>::type;
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
    constexpr bool DYN = G::MINB > 1;  // as in dec_fast_kernel
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
            return (!PUNCT || f < n) ? y >> 16 : 0u;  // canonical: bit 16 set iff y == 65536
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

// ---------------------------------------------------------------------------
// Decode occupancy: the staged input is read only by the first pass, so one
// stage buffer suffices (the next tile's TMA load is issued right after that
// pass's barrier) and at N <= 256 five CTAs fit per SM.
template <int E>
struct DecOcc {
    static constexpr int MINB = (E <= 8) ? 5 : Pick<E>::MINB;
};

// MODE 0: decode (interp::interpolate, the k coefficients out).
// MODE 1: systematic decode (codec.cpp:163-196): the interpolant P is
//         re-encoded in the tile (FNT4 = FNT_N(P), fused with IFNT3's last
//         pass in registers) and codeword rows 0..k-1 go out.
// MODE 2: systematic encode (codec.cpp:151-161) with the plan of positions
//         0..k-1: source rows are copied to codeword rows 0..k-1 while the
//         first pass scatters them, and FNT4 rows k..n-1 (the parity) go out.
template <int E, class G, bool HALFK, int MODE = 0>
__global__ void __launch_bounds__(G::NT, DecOcc<E>::MINB) dec_fast_kernel(const __grid_constant__ CUtensorMap rx_map,
                                                         const uint2* __restrict__ ptabF, const uint2* __restrict__ ptabI,
                                                         const uint2* __restrict__ rowmap,
                                                         const uint2* __restrict__ ahat2, uint32_t k, uint32_t L,
                                                         uint32_t tps, uint32_t tiles, uint32_t nbox, uint32_t box_rows,
                                                         const uint32_t* __restrict__ stripe_pattern, EscIn esc_in,
                                                         uint16_t* __restrict__ out, EscOut esc_out, uint32_t n,
                                                         const uint2* __restrict__ ptabFT, uint32_t* __restrict__ tile_ctr) {
    using S = Sched<E>;
    constexpr int N = 1 << E, WT = G::WT, NT = G::NT, P = S::P;
    constexpr int RLZ = G::RLZ, RZ = 1 << RLZ;
    constexpr int RL0 = S::rlog(0), R0 = 1 << RL0, SL0 = S::slog(0);
    constexpr uint32_t FLIP = uint32_t(N - 1);
    constexpr int LGW = ilog2c<WT>();
    static_assert(P >= 2 && P <= 3, "");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[2];
    __shared__ uint32_t next_tile[2];  // successor of the tile of iteration i, in slot i & 1
    uint32_t* work = reinterpret_cast<uint32_t*>(smem_raw);
    // [guard | stage]: the guard is the WT-symbol row just below the stage (an
    // erased position's row index ~0 wraps onto it) and holds ones, so raw
    // received words can be tested for zero unmasked.
    const uint32_t stage_elems = nbox * box_rows * WT;
    const uint32_t stage_bytes = stage_elems * 2;
    uint16_t* stage0 = reinterpret_cast<uint16_t*>(smem_raw + size_t(N) * WT * 4 + kGuardBytes);
    constexpr uint32_t stage_stride = 0;  // single stage
    for (uint32_t i = threadIdx.x; i < uint32_t(WT); i += NT) stage0[i - WT] = 1;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&rx_map);
        mbar_init(&bars[0], 1);
        fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](uint32_t tl, int bs) {
        const uint32_t s1 = tl / tps;
        const uint32_t cc = (tl - s1 * tps) * WT;
        fence_proxy_async();
        mbar_expect_tx(&bars[bs], stage_bytes);
        uint16_t* dst = stage0 + bs * stage_stride;
        for (uint32_t j = 0; j < nbox; ++j)
            tma_load_2d(dst + j * box_rows * WT, &rx_map, int(cc), int(s1 * k + j * box_rows), &bars[bs]);
    };
    uint32_t tile = blockIdx.x;
    if (threadIdx.x == 0 && tile < tiles) issue(tile, 0);
    const uint4* tF0 = pass_table(ptabF, S::llog(0));
    const uint4* tI0 = pass_table(ptabI, S::llog(0));
    const bool esc_any = esc_in.n != 0;
    for (uint32_t iter = 0; tile < tiles; tile = DecOcc<E>::MINB > 1 ? next_tile[iter & 1] : tile + gridDim.x, ++iter) {
        const uint32_t stripe = tile / tps;
        const uint32_t c0 = (tile - stripe * tps) * WT;
        const uint32_t pat = __ldg(stripe_pattern + stripe);
        // the successor is claimed now and used after the first pass (the atomic's latency hides behind it);
        // one CTA per SM (n_domain 4096) keeps the static stride: nothing to balance, one register less
        constexpr bool DYN = DecOcc<E>::MINB > 1;
        const uint32_t claimed = !DYN ? tile + gridDim.x : threadIdx.x == 0 ? claim_tile(tile_ctr) : 0u;
        const uint2* __restrict__ rm = rowmap + size_t(pat) * N;
        const uint2* __restrict__ ah = ahat2 + size_t(pat) * N;
        const unsigned long long key = uint64_t(stripe) * k * L + c0;
        // output rows per stripe: k (decode, systematic decode) or n (systematic encode)
        const unsigned long long key_out = MODE == 2 ? uint64_t(stripe) * n * L + c0 : key;
        uint16_t* outp = launder(out + key_out);
        mbar_wait(&bars[0], iter & 1);
        const uint16_t* st_in = stage0;

        // step 4: N'[z] = v_i / A'(x_i) where z = z_i, else 0 (rowmap {~0, 0}:
        // reads the guard row of ones, scales by 0). A received zero word may
        // be an escaped 65536: the group fix-up re-scales it.
        uint32_t zmin = 0xFFFFFFFFu;
        auto ld_scatter = [&](uint32_t lrow, uint32_t, int q, uint32_t col) -> uint32_t {
            const uint2 m = __ldg(rm + lrow);
            const uint32_t raw = st_in[int(m.x * uint32_t(WT) + col)];
            zmin = min(zmin, raw);
            if constexpr (MODE == 2) {  // identity plan: row z < k is source row z -> codeword row z
                if (HALFK ? (q < R0 / 2) : (lrow < k)) __stcs(outp + (lrow * L + col), uint16_t(raw));
            }
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
                if (m.x != 0xFFFFFFFFu && st_in[m.x * WT + col] == 0u &&
                    esc_has(esc_in, key + uint64_t(m.x) * L + col)) {
                    v[q] = mulws(65536u, m.y, m.y * 65535u);
                    if constexpr (MODE == 2) emit_escape(esc_out, key_out + uint64_t(m.x) * L + col);
                }
            }
        };
        auto ld_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t { return work[G::idx(lrow, col)]; };
        auto st_sm = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
            work[G::idx(lrow, col)] = y;
            return 0u;
        };
        auto ld_smf = [&](uint32_t lrow, uint32_t, int, uint32_t col) -> uint32_t {
            return work[G::template idx_flip<FLIP + 1>(lrow, col)];
        };
        auto st_smf = [&](uint32_t lrow, uint32_t, int, uint32_t col, uint32_t y) -> uint32_t {
            work[G::template idx_flip<FLIP + 1>(lrow, col)] = y;
            return 0u;
        };
        auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
            const uint32_t f = perm_head<E>(b) + (uint32_t(s) << (E - RLZ));
            // k = N/2: kept iff s < R/2 (compile time after unrolling)
            const bool keep = HALFK ? (s < RZ / 2) : (f < k);
            if (keep) __stcs(outp + (f * L + col), uint16_t(y));
            return keep ? y >> 16 : 0u;  // canonical: bit 16 set iff y == 65536
        };
        auto flush_out = [&](uint32_t mask, uint32_t, uint32_t b, uint32_t col) {
            if (!mask) return;
#pragma unroll 1
            for (int s = 0; s < 16; ++s)
                if (mask & (1u << s))
                    emit_escape(esc_out, key + uint64_t(perm_head<E>(b) + (uint32_t(s) << (E - RLZ))) * L + col);
        };

        // FNT1 = FNT_N(N'), DIF, natural -> perm order (flip 0)
        pass<E, 0, false, false, k2P, kSmemCap, G>(tF0, ld_scatter, st_sm, fix_scatter);
        __syncthreads();
        // the stage is consumed: stream the next tile's packets in behind the remaining passes
        if (threadIdx.x == 0) {
            if constexpr (DYN) next_tile[iter & 1] = claimed;
            if (claimed < tiles) issue(claimed, 0);
        }
        if constexpr (P == 3) {
            pass<E, 1, false, false, kSmemCap, kSmemCap, G>(pass_table(ptabF, S::llog(1)), ld_sm, st_sm);
            __syncthreads();
        }
        // FNT1 last pass (sub 1) + FNT2 first DIT pass on the reversed view:
        // logical group b' = N/R - 1 - g holds s'_j = F[N-1-j]; j >= k zeroed.
        {
            constexpr int ITEMS = (N / RZ) * WT;
            constexpr uint64_t BD = dif_bound<RZ, false, kSmemCap>();
            constexpr uint64_t BT = dit_bound<RZ, false, BD>();
#pragma unroll 1
            for (int it = threadIdx.x; it < ITEMS; it += NT) {
                const uint32_t col = uint32_t(it) & uint32_t(WT - 1);
                const uint32_t g = uint32_t(it) >> LGW;
                uint32_t v[RZ];
#pragma unroll
                for (int q = 0; q < RZ; ++q) v[q] = work[G::idx((g << RLZ) + q, col)];
                dif_regs<RZ, false, kSmemCap>(v);
                const uint32_t fh = perm_head<E>(uint32_t(N / RZ) - 1u - g);
                uint32_t u[RZ];
#pragma unroll
                for (int j = 0; j < RZ; ++j) {  // u[rev(s')] = x_{s'} = y_{R-1-s'} = v[R-1-j]
                    // k = N/2: live iff rev(j) < R/2, i.e. j even (compile time)
                    const bool live = HALFK ? ((j & 1) == 0) : (fh + (uint32_t(rev<RZ>(j)) << (E - RLZ)) < k);
                    u[j] = live ? v[RZ - 1 - j] : 0u;
                }
                dit_regs<RZ, false, BD>(u);
                if constexpr (P == 2) {
                    // FNT2's last DIT pass pre-multiplies logical row t + s*sub0 by r^(t s);
                    // this element is t = q, s = N/R - 1 - g: apply it here, where the
                    // multiply also does the reduction the store needed anyway
                    const uint4* tq = reinterpret_cast<const uint4*>(ptabFT + N + (uint32_t(N / RZ) - 1u - g) * RZ);
#pragma unroll
                    for (int q = 0; q < RZ; q += 2) {
                        const uint4 w = __ldg(tq + q / 2);
                        work[G::idx((g << RLZ) + (RZ - 1 - q), col)] = mulws(u[q], w.x, w.y);
                        work[G::idx((g << RLZ) + (RZ - 2 - q), col)] = mulws(u[q + 1], w.z, w.w);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < RZ; ++q) work[G::idx((g << RLZ) + (RZ - 1 - q), col)] = cap<BT, kSmemCap>(u[q]);
                }
            }
        }
        __syncthreads();
        if constexpr (P == 3) {
            pass<E, 1, false, true, kSmemCap, kSmemCap, G>(pass_table(ptabF, S::llog(1)), ld_smf, st_smf);
            __syncthreads();
        }
        // FNT2 last DIT pass + (. ahat) + FNT3 first DIF pass: rows t + q * sub0
        {
            constexpr int ITEMS = (N / R0) * WT;
            constexpr uint64_t BO = dif_bound<R0, true, k2P>();
#pragma unroll 1
            for (int it = threadIdx.x; it < ITEMS; it += NT) {
                const uint32_t col = uint32_t(it) & uint32_t(WT - 1);
                const uint32_t t = uint32_t(it) >> LGW;
                uint32_t v[R0];
                const uint4* tpf = tF0 + t * (R0 / 2);
                const uint4* tpi = tI0 + t * (R0 / 2);
                uint4 w4 = make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int s = 0; s < R0; ++s) {
                    uint32_t x = work[G::template idx_flip<FLIP + 1>(t + (uint32_t(s) << SL0), col)];
                    if (P != 2 && s > 0) {  // P == 2: the twiddle was applied by the producing pass
                        const uint2 w = tw_at(tpf, s, w4);
                        x = mulws(x, w.x, w.y);
                    }
                    v[rev<R0>(s)] = x;
                }
                dit_regs<R0, false, (P == 2 ? k2P : kSmemCap)>(v);
                const uint4* ahq = reinterpret_cast<const uint4*>(ah) + t * (R0 / 2);  // ahat2_slot order
#pragma unroll
                for (int q = 0; q < R0; q += 2) {
                    const uint4 a = __ldg(ahq + q / 2);
                    v[q] = mulws(v[q], a.x, a.y);
                    v[q + 1] = mulws(v[q + 1], a.z, a.w);
                }
                dif_regs<R0, true, k2P>(v);
#pragma unroll
                for (int s = 0; s < R0; ++s) {
                    uint32_t y = v[rev<R0>(s)];
                    if (s > 0) {
                        const uint2 w = tw_at(tpi, s, w4);
                        y = mulws(y, w.x, w.y);
                    } else {
                        y = cap<BO, kSmemCap>(y);
                    }
                    work[G::template idx_flip<FLIP + 1>(t + (uint32_t(s) << SL0), col)] = y;
                }
            }
        }
        __syncthreads();
        if constexpr (P == 3) {
            pass<E, 1, true, false, kSmemCap, kSmemCap, G>(pass_table(ptabI, S::llog(1)), ld_smf, st_smf);
            __syncthreads();
        }
        if constexpr (MODE == 0) {
            pass<E, P - 1, true, false, kSmemCap, kCanon, G>(pass_table(ptabI, S::llog(P - 1)), ld_smf, st_out, NoFix(),
                                                          flush_out);
        } else {
            // IFNT3 last pass + truncation to the k coefficients + FNT4 first
            // DIT pass, in registers on the same rows (reversed view)
            {
                constexpr int ITEMS = (N / RZ) * WT;
                constexpr uint64_t BD = dif_bound<RZ, true, kSmemCap>();
                constexpr uint64_t BT = dit_bound<RZ, false, BD>();
#pragma unroll 1
                for (int it = threadIdx.x; it < ITEMS; it += NT) {
                    const uint32_t col = uint32_t(it) & uint32_t(WT - 1);
                    const uint32_t g = uint32_t(it) >> LGW;
                    uint32_t v[RZ];
#pragma unroll
                    for (int q = 0; q < RZ; ++q) v[q] = work[G::template idx_flip<FLIP + 1>((g << RLZ) + q, col)];
                    dif_regs<RZ, true, kSmemCap>(v);
                    const uint32_t fh = perm_head<E>(g);
#pragma unroll
                    for (int s2 = 0; s2 < RZ; ++s2) {  // output s2 holds coefficient fh + s2 * N/R
                        const bool live = HALFK ? (s2 < RZ / 2) : (fh + (uint32_t(s2) << (E - RLZ)) < k);
                        if (!live) v[rev<RZ>(s2)] = 0u;
                    }
                    // DIT input x_s = y_s (same rows): v[rev(s)] already is y_s
                    dit_regs<RZ, false, BD>(v);
#pragma unroll
                    for (int q = 0; q < RZ; ++q)
                        work[G::template idx_flip<FLIP + 1>((g << RLZ) + q, col)] = cap<BT, kSmemCap>(v[q]);
                }
            }
            __syncthreads();
            if constexpr (P == 3) {
                pass<E, 1, false, true, kSmemCap, kSmemCap, G>(pass_table(ptabF, S::llog(1)), ld_smf, st_smf);
                __syncthreads();
            }
            // FNT4 last DIT pass: natural order, codeword row f = the position
            auto st_sys = [&](uint32_t lrow, uint32_t, int q, uint32_t col, uint32_t y) -> uint32_t {
                constexpr int SLL = S::slog(0);
                (void)SLL;
                bool keep;
                if constexpr (MODE == 1)
                    keep = HALFK ? (q < R0 / 2) : (lrow < k);
                else
                    keep = (HALFK ? (q >= R0 / 2) : (lrow >= k)) && lrow < n;
                if (keep) __stcs(outp + (lrow * L + col), uint16_t(y));
                return keep ? y >> 16 : 0u;
            };
            auto flush_sys = [&](uint32_t mask, uint32_t base, uint32_t, uint32_t col) {
                if (!mask) return;
#pragma unroll 1
                for (int q = 0; q < 16; ++q)
                    if (mask & (1u << q))
                        emit_escape(esc_out, key_out + uint64_t(base + (uint32_t(q) << SL0)) * L + col);
            };
            pass<E, 0, false, true, kSmemCap, kCanon, G>(tF0, ld_smf, st_sys, NoFix(), flush_sys);
        }
        __syncthreads();
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

// ---- host side ----------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D map over a packet-major uint16 buffer [rows][L], box [box_rows][wt].
cudaError_t make_map(CUtensorMap* map, const void* base, uint64_t rows, uint32_t L, uint32_t wt, uint32_t box_rows) {
    EncodeTiledFn fn = encode_tiled();
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

// 3-D map over packet-major uint16 stripes [stripes][rows][L], box [1][box_rows][wt]:
// a box never crosses into the next stripe (rows beyond `rows` are clipped).
cudaError_t make_map3(CUtensorMap* map, const void* base, uint64_t stripes, uint32_t rows, uint32_t L, uint32_t wt,
                      uint32_t box_rows) {
    EncodeTiledFn fn = encode_tiled();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {L, rows, stripes};
    const cuuint64_t strides[2] = {cuuint64_t(L) * 2, cuuint64_t(L) * rows * 2};
    const cuuint32_t box[3] = {wt, box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

struct LaunchShape {
    uint32_t tps, tiles, nbox, box_rows, grid;
    size_t smem;
};

template <class K>
cudaError_t shape_for(K kernel, int E, int wt, int nt, uint32_t k, uint32_t stripes, uint32_t L, LaunchShape& sh,
                      size_t extra = 0, int stages = 2) {
    sh.tps = L / wt;
    const uint64_t tiles = uint64_t(stripes) * sh.tps;
    if (tiles > 0xFFFFFFFFull) return cudaErrorInvalidConfiguration;
    sh.tiles = uint32_t(tiles);
    sh.box_rows = k < 256 ? k : 256;
    sh.nbox = (k + sh.box_rows - 1) / sh.box_rows;
    sh.smem = (size_t(1) << E) * wt * 4 + size_t(stages) * sh.nbox * sh.box_rows * wt * 2 + extra;
    cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sh.smem));
    if (err) return err;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, nt, sh.smem))) return err;
    if (per < 1) return cudaErrorInvalidConfiguration;
    const uint64_t g = uint64_t(sms) * per;
    sh.grid = uint32_t(g < tiles ? g : tiles);
    return cudaSuccess;
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
    if (G::MINB > 1 && (err = ctr.get(st))) return err;
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

template <int E, int MODE = 0>
cudaError_t launch_dec(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L, const uint32_t* sp,
                       const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout, cudaStream_t st, uint32_t n = 0) {
    using G = typename Pick<E>::G;
    auto kern = pv.k == (1u << E) / 2 ? dec_fast_kernel<E, G, true, MODE> : dec_fast_kernel<E, G, false, MODE>;
    LaunchShape sh;
    cudaError_t err = shape_for(kern, E, G::WT, G::NT, pv.k, stripes, L, sh, kGuardBytes, 1);
    if (err) return err;
    if (!sh.tiles) return cudaSuccess;
    CUtensorMap map;
    if ((err = make_map(&map, rx, uint64_t(stripes) * pv.k, L, G::WT, sh.box_rows))) return err;
    TileCounter ctr;
    if (DecOcc<E>::MINB > 1 && (err = ctr.get(st))) return err;
    kern<<<sh.grid, G::NT, sh.smem, st>>>(map, t.ptab_fwd, t.ptab_inv, pv.rowmap, pv.ahat2, pv.k, L, sh.tps, sh.tiles,
                                          sh.nbox, sh.box_rows, sp, ein, out, eout, n, t.ptab_fwdT, ctr.p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t build_fast_tables(FastTables& t, cudaStream_t st) {
    cudaError_t err = cudaMalloc(&t.ptab_fwd, sizeof(uint2) << 13);
    if (err) return err;
    if ((err = cudaMalloc(&t.ptab_inv, sizeof(uint2) << 13))) return err;
    if ((err = cudaMalloc(&t.ptab_fwdT, sizeof(uint2) << 9))) return err;
    ptab_kernel<<<(1u << 13) / 256, 256, 0, st>>>(t.ptab_fwd, t.ptab_inv);
    ptab_t_kernel<<<2, 256, 0, st>>>(t.ptab_fwdT);
    return cudaGetLastError();
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

// systematic codec, fused (MODE 1: decode, rows 0..k-1 out; MODE 2: encode
// with the plan of positions 0..k-1, rows 0..n-1 out)
cudaError_t launch_systematic_fast(const FastTables& t, const FastPlanView& pv, bool encode, uint32_t n,
                                   uint32_t stripes, uint32_t L, const uint32_t* sp, const uint16_t* in, EscIn ein,
                                   uint16_t* out, EscOut eout, cudaStream_t st) {
#define FNTRS_SYS(e)                                                                              \
    case (1u << e):                                                                               \
        return encode ? launch_dec<e, 2>(t, pv, stripes, L, sp, in, ein, out, eout, st, n)       \
                      : launch_dec<e, 1>(t, pv, stripes, L, sp, in, ein, out, eout, st, n);
    switch (pv.N) {
        FNTRS_SYS(5) FNTRS_SYS(6) FNTRS_SYS(7) FNTRS_SYS(8) FNTRS_SYS(9) FNTRS_SYS(10) FNTRS_SYS(11) FNTRS_SYS(12)
        default: return cudaErrorInvalidValue;
    }
#undef FNTRS_SYS
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
