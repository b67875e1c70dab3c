// codec_dec.cu -- fused decode kernels for 32 <= n_domain <= 4096 (the
// decode half of the codec_fast.cu design; see its header for the tile and
// TMA scheme).
//
// Decode  (interp::interpolate, proj/src/interp.cpp:103-137, per codeword):
//   FNT1 pass 0 scatters received row i to position z_i scaled by
//   1/A'(x_i); FNT1's last pass and FNT2's first DIT pass are fused in
//   registers (s'_j = F[N-1-j] is a reversal of the butterfly group; j >= k
//   zeroed); FNT2's last DIT pass, the product with A_hat and FNT3's first
//   DIF pass are fused in registers; FNT3's last pass writes the k decoded
//   packets. Systematic encode / decode (codec.cpp:151-196) are MODE 1 / 2
//   of the same kernel (four transforms), or MODE 4 / 3 (two transforms: the
//   evaluations P(r^j) come straight out of one cyclic convolution, see below).
//
// Separate translation unit because decode is compiled with ALU-pinned adds
// (field.cuh, FNTRS_ALU_ADDS): decode spends more of its instructions on
// Shoup products (multiplier pipe) than encode, and moving the butterfly adds
// off that pipe gives C2 decode +2.6 % (encode, in codec_fast.cu, loses 0.7 %
// with the same switch, so it keeps ptxas' own choice).
#ifndef FNTRS_ALU_ADDS
#define FNTRS_ALU_ADDS 1
#endif
// lazy w4 shifts as ALU funnel shifts (ptxas would fold them into IMADs):
// C5 decode +2.4 %, C2 neutral (the encode unit loses 2.4 % with it)
#ifndef FNTRS_PIN_SHIFT
#define FNTRS_PIN_SHIFT 1
#endif
#ifndef FNTRS_R2D_LIM
#define FNTRS_R2D_LIM (1ull << 22)
#endif
#ifndef FNTRS_R2T_LIM
#define FNTRS_R2T_LIM (1ull << 30)
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

// n_domain <= 256: copies of the pass-0 twiddle tables (uint2 entries [0, 512) of
// ptab_fwd, ptab_inv, ptab_fwdT; 12 KB) in constant memory. Their rows are
// warp-uniform, so the constant cache serves them without L1 data-pipe
// wavefronts (the decode kernel's busiest unit). FNTRS_CONST_TW selects them.
// systematic codec by one convolution (MODE 3 / 4) instead of interpolate + re-encode (MODE 1 / 2)
#ifndef FNTRS_SYS_CONV
#define FNTRS_SYS_CONV 1
#endif
// MODE 3 / 4 at two passes per transform: the last DIT pass's twiddles applied by the producer
#ifndef FNTRS_SYS_PRETW
#define FNTRS_SYS_PRETW 1
#endif
// sys_conv layout: N = 32..4096 at [2N, 4N) (Q, r^-j); transposed inverse pass-0 twiddles
// for N <= 256 at kSysInvT + [N + (N/16) s + t] = r_N^-(t s)
constexpr uint32_t kSysInvT = 16384;
#ifndef FNTRS_CONST_TW
#define FNTRS_CONST_TW 1
#endif
__constant__ uint4 c_twF[256], c_twI[256], c_twFT[256];
// n_domain <= 256, MODE 3 / 4: the Q tables (sys_conv [0, 1024)) and the transposed
// inverse pass-0 twiddles (sys_conv kSysInvT + [0, 512)); rows are warp-uniform
#ifndef FNTRS_SYS_CONST
#define FNTRS_SYS_CONST 1
#endif
__constant__ uint4 c_sysQ[512], c_sysT[256];

namespace {

// ---------------------------------------------------------------------------
// Decode occupancy: the staged input is read only by the first pass, so one
// stage buffer suffices (the next tile's TMA load is issued right after that
// pass's barrier) and at N <= 256 five CTAs fit per SM.
// MODE 3 / 4 at n_domain <= 256: four CTAs per SM (64 registers) -- A/B vs five: +0.7 %
#ifndef FNTRS_SYS_MINB
#define FNTRS_SYS_MINB 4
#endif
#ifndef FNTRS_DEC_MINB
#define FNTRS_DEC_MINB 5
#endif
template <int E, int MODE = 0>
struct DecOcc {
    static constexpr int MINB = (E <= 8) ? (MODE >= 3 ? FNTRS_SYS_MINB : FNTRS_DEC_MINB) : Pick<E>::MINB;
};

// MODE 0: decode (interp::interpolate, the k coefficients out).
// MODE 1: systematic decode (codec.cpp:163-196): the interpolant P is
//         re-encoded in the tile (FNT4 = FNT_N(P), fused with IFNT3's last
//         pass in registers) and codeword rows 0..k-1 go out.
// MODE 2: systematic encode (codec.cpp:151-161) with the plan of positions
//         0..k-1: source rows are copied to codeword rows 0..k-1 while the
//         first pass scatters them, and FNT4 rows k..n-1 (the parity) go out.
// MODE 3 / 4: systematic decode / encode by the Cauchy form of the interpolant.
//         P(x) = A(x) sum_i c_i / (x - x_i), c_i = v_i / A'(x_i), so at a
//         non-received position j
//           P(r^j) = A(r^j) r^-j sum_z c[z] G'[j - z],  G'[e] = 1 / (1 - r^-e), G'[0] = 0,
//         a cyclic convolution of the scattered c with a constant of N:
//         FNT_N(c) (DIF) x Q (Q = -FNT_N(G'), table sysc) -> unscaled inverse DIT
//         -> x r^-j x ahat_j (ahat = -A(r^j)/N, 0 on received rows). Two
//         transforms instead of four (MODE 1 / 2); the same values, exactly.
//         Received rows j < k (MODE 3) / source rows (MODE 4) are copied by the
//         scatter pass.
template <int E, class G, bool HALFK, int MODE = 0>
__global__ void __launch_bounds__(G::NT, DecOcc<E, MODE>::MINB) dec_fast_kernel(const __grid_constant__ CUtensorMap rx_map,
                                                         const uint2* __restrict__ ptabF, const uint2* __restrict__ ptabI,
                                                         const uint2* __restrict__ rowmap,
                                                         const uint2* __restrict__ ahat2, uint32_t k, uint32_t L,
                                                         uint32_t tps, uint32_t tiles, uint32_t nbox, uint32_t box_rows,
                                                         const uint32_t* __restrict__ stripe_pattern, EscIn esc_in,
                                                         uint16_t* __restrict__ out, EscOut esc_out, uint32_t n,
                                                         const uint2* __restrict__ ptabFT, uint32_t* __restrict__ tile_ctr,
                                                         const uint2* __restrict__ sysc) {
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
    constexpr bool CT = FNTRS_CONST_TW && E <= 8;
    const uint4* tF0 = CT ? pass_table(reinterpret_cast<const uint2*>(c_twF), S::llog(0)) : pass_table(ptabF, S::llog(0));
    const uint4* tI0 = CT ? pass_table(reinterpret_cast<const uint2*>(c_twI), S::llog(0)) : pass_table(ptabI, S::llog(0));
    [[maybe_unused]] const uint2* twFT = CT ? reinterpret_cast<const uint2*>(c_twFT) : ptabFT;
    const bool esc_any = esc_in.n != 0;
    for (uint32_t iter = 0; tile < tiles; tile = next_tile[iter & 1], ++iter) {
        const uint32_t stripe = tile / tps;
        const uint32_t c0 = (tile - stripe * tps) * WT;
        const uint32_t pat = __ldg(stripe_pattern + stripe);
        // the successor is claimed now and used after the first pass (the atomic's latency hides behind it).
        // Claiming at every occupancy keeps CTAs on adjacent tiles in step: the two halves of a 32-byte
        // sector (8-column tiles at n_domain 4096) then meet in L2 instead of costing DRAM re-reads
        const uint32_t claimed = threadIdx.x == 0 ? claim_tile(tile_ctr) : 0u;
        const uint2* __restrict__ rm = rowmap + size_t(pat) * N;
        const uint2* __restrict__ ah = ahat2 + size_t(pat) * N;
        const unsigned long long key = uint64_t(stripe) * k * L + c0;
        // output rows per stripe: k (decode, systematic decode) or n (systematic encode)
        constexpr bool ENC = MODE == 2 || MODE == 4;
        const unsigned long long key_out = ENC ? uint64_t(stripe) * n * L + c0 : key;
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
            if constexpr (ENC) {  // identity plan: row z < k is source row z -> codeword row z
                if (HALFK ? (q < R0 / 2) : (lrow < k)) __stcs(outp + (lrow * L + col), uint16_t(raw));
            } else if constexpr (MODE == 3) {  // received row z < k: P(r^z) is the received word
                if ((HALFK ? (q < R0 / 2) : (lrow < k)) && m.x != 0xFFFFFFFFu)
                    __stcs(outp + (lrow * L + col), uint16_t(raw));
            }
            // raw <= 65535 and |1/A'| <= p/2 (balanced): the product is exact in 32 signed bits
            return reds(raw * m.y);
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
                    if constexpr (ENC) emit_escape(esc_out, key_out + uint64_t(m.x) * L + col);
                    if constexpr (MODE == 3) {
                        const uint32_t z = base + (uint32_t(q) << SL0);
                        if (z < k) emit_escape(esc_out, key_out + uint64_t(z) * L + col);
                    }
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
        // output row f = perm_head(b) + s N/R. At n_domain <= 256: one 64-bit
        // pointer per butterfly group, stepped by N/R rows per output (64-bit adds
        // on the ALU pipe instead of an IMAD.WIDE per store on the busier
        // multiplier pipe: C2 decode +1.1 %; at n_domain 4096, one CTA per SM,
        // the extra live pointer costs 3 %)
        constexpr bool STEP = E <= 8;
        uint16_t* op = outp;
        const uint64_t ostep = opaque_stride(uint64_t(L) << (E - RLZ + 1));
        auto st_out = [&](uint32_t, uint32_t b, int s, uint32_t col, uint32_t y) -> uint32_t {
            const uint32_t f = perm_head<E>(b) + (uint32_t(s) << (E - RLZ));
            if (!STEP)
                op = outp + (f * L + col);
            else if (s == 0)
                op = outp + (perm_head<E>(b) * L + col);
            else
                op = step_ptr(op, ostep);
            // k = N/2: kept iff s < R/2 (compile time after unrolling)
            const bool keep = HALFK ? (s < RZ / 2) : (f < k);
            if (keep) __stcs(op, uint16_t(y));
            return keep ? y : 0u;  // canonical, kept: bit 16 set iff y == 65536
        };
        auto flush_out = [&](uint32_t mask, uint32_t, uint32_t b, uint32_t col) {
            if (!mask) return;
#pragma unroll 1
            for (int s = 0; s < 16; ++s)
                if (mask & (1u << s))
                    emit_escape(esc_out, key + uint64_t(perm_head<E>(b) + (uint32_t(s) << (E - RLZ))) * L + col);
        };

        // FNT1 = FNT_N(N'), DIF, natural -> perm order (flip 0)
        pass<E, 0, false, false, k2P, kSmemCap, G, decltype(ld_scatter), decltype(st_sm), decltype(fix_scatter), NoFlush, 1,
             CT>(tF0, ld_scatter, st_sm, fix_scatter);
        __syncthreads();
        // the stage is consumed: stream the next tile's packets in behind the remaining passes
        if (threadIdx.x == 0) {
            next_tile[iter & 1] = claimed;
            if (claimed < tiles) issue(claimed, 0);
        }
        if constexpr (P == 3) {
            pass<E, 1, false, false, kSmemCap, kSmemCap, G>(pass_table(ptabF, S::llog(1)), ld_sm, st_sm);
            __syncthreads();
        }
        if constexpr (MODE >= 3) {
            // FNT_N(c) last DIF pass (sub 1), x Q, first pass of the unscaled inverse DIT, in registers
            {
                constexpr int ITEMS = (N / RZ) * WT;
                constexpr uint64_t BD = dif_bound<RZ, false, kSmemCap, kLazyLim>();
                static_assert(BD < (1ull << 31), "Shoup inputs are signed 32-bit");
                constexpr uint64_t BT = dit_bound<RZ, true, k2P, uint64_t(FNTRS_R2T_LIM)>();  // folded to 2p below
                constexpr bool CQ = FNTRS_SYS_CONST && E <= 8;
                const uint4* qt = CQ ? reinterpret_cast<const uint4*>(reinterpret_cast<const uint2*>(c_sysQ) + 2 * N)
                                     : reinterpret_cast<const uint4*>(sysc);
#pragma unroll 1
                for (int it = threadIdx.x; it < ITEMS; it += NT) {
                    const uint32_t col = uint32_t(it) & uint32_t(WT - 1);
                    const uint32_t g = uint32_t(it) >> LGW;
                    uint32_t v[RZ];
#pragma unroll
                    for (int q = 0; q < RZ; ++q) v[q] = work[G::idx((g << RLZ) + q, col)];
                    dif_regs<RZ, false, kSmemCap, kLazyLim>(v);
                    // v[j] holds frequency perm_head(g) + rev(j) N/R; sysc is stored in that order
                    const uint4* tq = qt + g * (RZ / 2);
#pragma unroll
                    for (int q = 0; q < RZ; q += 2) {
                        const uint4 w = CQ ? tq[q / 2] : __ldg(tq + q / 2);
                        v[q] = mulws(v[q], w.x, w.y);
                        v[q + 1] = mulws(v[q + 1], w.z, w.w);
                    }
                    dit_regs<RZ, true, k2P, uint64_t(FNTRS_R2T_LIM)>(v);
                    if constexpr (P == 2 && FNTRS_SYS_PRETW) {
                        // the last DIT pass's input twiddle of row t + s sub0 is r^-(t s); this
                        // element is t = q, s = g: applied here, where the Shoup product also
                        // does the reduction the store needed
                        static_assert(BT < (1ull << 31), "Shoup inputs are signed 32-bit");
                        const uint4* tq = CQ ? reinterpret_cast<const uint4*>(reinterpret_cast<const uint2*>(c_sysT) + N + g * RZ)
                                             : reinterpret_cast<const uint4*>(sysc - 2 * N + kSysInvT + N + g * RZ);
#pragma unroll
                        for (int q = 0; q < RZ; q += 2) {
                            const uint4 w = CQ ? tq[q / 2] : __ldg(tq + q / 2);
                            work[G::idx((g << RLZ) + q, col)] = mulws(v[q], w.x, w.y);
                            work[G::idx((g << RLZ) + q + 1, col)] = mulws(v[q + 1], w.z, w.w);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < RZ; ++q) work[G::idx((g << RLZ) + q, col)] = cap<BT, kSmemCap>(v[q]);
                    }
                }
            }
            __syncthreads();
            if constexpr (P == 3) {
                pass<E, 1, true, true, kSmemCap, kSmemCap, G>(pass_table(ptabI, S::llog(1)), ld_sm, st_sm);
                __syncthreads();
            }
            // last inverse DIT pass: natural order; P(r^j) = U[j] r^-j ahat_j on the rows kept
            auto st_conv = [&](uint32_t lrow, uint32_t, int q, uint32_t col, uint32_t y) -> uint32_t {
                bool keep;
                if constexpr (MODE == 3)
                    keep = HALFK ? (q < R0 / 2) : (lrow < k);
                else
                    keep = (HALFK ? (q >= R0 / 2) : (lrow >= k)) && lrow < n;
                if (!keep) return 0u;
                const uint2 a = __ldg(ah + lrow);  // MODE 3 / 4: sysw, {ahat_j r^-j} in natural order
                if (MODE == 3 && a.x == 0u) return 0u;  // received: written by the scatter pass
                const uint32_t z = canon_s2p(mulws(y, a.x, a.y));
                __stcs(outp + (lrow * L + col), uint16_t(z));
                return z;
            };
            auto flush_conv = [&](uint32_t mask, uint32_t base, uint32_t, uint32_t col) {
                if (!mask) return;
#pragma unroll 1
                for (int q = 0; q < 16; ++q)
                    if (mask & (1u << q)) emit_escape(esc_out, key_out + uint64_t(base + (uint32_t(q) << SL0)) * L + col);
            };
            if constexpr (P == 2 && FNTRS_SYS_PRETW) {  // twiddles applied by the producing pass
                constexpr int ITEMS = (N / R0) * WT;
                constexpr uint64_t BO = dit_bound<R0, true, k2P>();
#pragma unroll 1
                for (int it = threadIdx.x; it < ITEMS; it += NT) {
                    const uint32_t col = uint32_t(it) & uint32_t(WT - 1);
                    const uint32_t t = uint32_t(it) >> LGW;
                    uint32_t v[R0];
#pragma unroll
                    for (int s2 = 0; s2 < R0; ++s2) v[rev<R0>(s2)] = work[G::idx(t + (uint32_t(s2) << SL0), col)];
                    dit_regs<R0, true, k2P>(v);
                    uint32_t acc = 0;
#pragma unroll
                    for (int q = 0; q < R0; ++q) {
                        const uint32_t r = st_conv(t + (uint32_t(q) << SL0), t, q, col, cap<BO, kCanon>(v[q]));
                        v[q] = r;
                        acc |= r;
                    }
                    if (acc >> 16) {
                        uint32_t mask = 0;
#pragma unroll
                        for (int q = 0; q < R0; ++q) mask |= ((v[q] >> 16) & 1u) << q;
                        flush_conv(mask, t, t, col);
                    }
                }
            } else {
                pass<E, 0, true, true, kSmemCap, kCanon, G, decltype(ld_sm), decltype(st_conv), NoFix, decltype(flush_conv),
                     1, CT>(tI0, ld_sm, st_conv, NoFix(), flush_conv);
            }
        } else {
        // FNT1 last pass (sub 1) + FNT2 first DIT pass on the reversed view:
        // logical group b' = N/R - 1 - g holds s'_j = F[N-1-j]; j >= k zeroed.
        {
            constexpr int ITEMS = (N / RZ) * WT;
            // the DIT outputs go into Shoup products (P == 2) or are folded to 2p for the tile
            // (P == 3) either way: lazy w4 products up to 2^30; the DIF feeding it up to R2D_LIM
            constexpr uint64_t L2D = uint64_t(FNTRS_R2D_LIM), L2T = uint64_t(FNTRS_R2T_LIM);
            constexpr uint64_t BD = dif_bound<RZ, false, kSmemCap, L2D>();
            constexpr uint64_t BT = dit_bound<RZ, false, BD, L2T>();
#pragma unroll 1
            for (int it = threadIdx.x; it < ITEMS; it += NT) {
                const uint32_t col = uint32_t(it) & uint32_t(WT - 1);
                const uint32_t g = uint32_t(it) >> LGW;
                uint32_t v[RZ];
#pragma unroll
                for (int q = 0; q < RZ; ++q) v[q] = work[G::idx((g << RLZ) + q, col)];
                dif_regs<RZ, false, kSmemCap, L2D>(v);
                const uint32_t fh = perm_head<E>(uint32_t(N / RZ) - 1u - g);
                uint32_t u[RZ];
#pragma unroll
                for (int j = 0; j < RZ; ++j) {  // u[rev(s')] = x_{s'} = y_{R-1-s'} = v[R-1-j]
                    // k = N/2: live iff rev(j) < R/2, i.e. j even (compile time)
                    const bool live = HALFK ? ((j & 1) == 0) : (fh + (uint32_t(rev<RZ>(j)) << (E - RLZ)) < k);
                    u[j] = live ? v[RZ - 1 - j] : 0u;
                }
                dit_regs<RZ, false, BD, L2T>(u);
                if constexpr (P == 2) {
                    // FNT2's last DIT pass pre-multiplies logical row t + s*sub0 by r^(t s);
                    // this element is t = q, s = N/R - 1 - g: apply it here, where the
                    // multiply also does the reduction the store needed anyway
                    const uint4* tq = reinterpret_cast<const uint4*>(twFT + N + (uint32_t(N / RZ) - 1u - g) * RZ);
#pragma unroll
                    for (int q = 0; q < RZ; q += 2) {
                        const uint4 w = CT ? tq[q / 2] : __ldg(tq + q / 2);
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
            constexpr uint64_t BO = dif_bound<R0, true, k2P, kLazyLim>();
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
                        const uint2 w = tw_at<CT>(tpf, s, w4);
                        x = mulws(x, w.x, w.y);
                    }
                    v[rev<R0>(s)] = x;
                }
                dit_regs<R0, false, (P == 2 ? k2P : kSmemCap), kLazyLim>(v);  // outputs -> (. ahat) Shoup
                const uint4* ahq = reinterpret_cast<const uint4*>(ah) + t * (R0 / 2);  // ahat2_slot order
#pragma unroll
                for (int q = 0; q < R0; q += 2) {
                    const uint4 a = __ldg(ahq + q / 2);
                    v[q] = mulws(v[q], a.x, a.y);
                    v[q + 1] = mulws(v[q + 1], a.z, a.w);
                }
                dif_regs<R0, true, k2P, kLazyLim>(v);
#pragma unroll
                for (int s = 0; s < R0; ++s) {
                    uint32_t y = v[rev<R0>(s)];
                    if (s > 0) {
                        const uint2 w = tw_at<CT>(tpi, s, w4);
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
                constexpr uint64_t BD = dif_bound<RZ, true, kSmemCap, uint64_t(FNTRS_R2D_LIM)>();
                constexpr uint64_t BT = dit_bound<RZ, false, BD, uint64_t(FNTRS_R2T_LIM)>();  // folded to 2p below
#pragma unroll 1
                for (int it = threadIdx.x; it < ITEMS; it += NT) {
                    const uint32_t col = uint32_t(it) & uint32_t(WT - 1);
                    const uint32_t g = uint32_t(it) >> LGW;
                    uint32_t v[RZ];
#pragma unroll
                    for (int q = 0; q < RZ; ++q) v[q] = work[G::template idx_flip<FLIP + 1>((g << RLZ) + q, col)];
                    dif_regs<RZ, true, kSmemCap, uint64_t(FNTRS_R2D_LIM)>(v);
                    const uint32_t fh = perm_head<E>(g);
#pragma unroll
                    for (int s2 = 0; s2 < RZ; ++s2) {  // output s2 holds coefficient fh + s2 * N/R
                        const bool live = HALFK ? (s2 < RZ / 2) : (fh + (uint32_t(s2) << (E - RLZ)) < k);
                        if (!live) v[rev<RZ>(s2)] = 0u;
                    }
                    // DIT input x_s = y_s (same rows): v[rev(s)] already is y_s
                    dit_regs<RZ, false, BD, uint64_t(FNTRS_R2T_LIM)>(v);
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
                return keep ? y : 0u;
            };
            auto flush_sys = [&](uint32_t mask, uint32_t base, uint32_t, uint32_t col) {
                if (!mask) return;
#pragma unroll 1
                for (int q = 0; q < 16; ++q)
                    if (mask & (1u << q))
                        emit_escape(esc_out, key_out + uint64_t(base + (uint32_t(q) << SL0)) * L + col);
            };
            pass<E, 0, false, true, kSmemCap, kCanon, G, decltype(ld_smf), decltype(st_sys), NoFix, decltype(flush_sys), 1,
                 CT>(tF0, ld_smf, st_sys, NoFix(), flush_sys);
        }
        }
        __syncthreads();
    }
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
    if ((err = ctr.get(st))) return err;
    kern<<<sh.grid, G::NT, sh.smem, st>>>(map, t.ptab_fwd, t.ptab_inv, pv.rowmap, MODE >= 3 ? pv.sysw : pv.ahat2, pv.k, L, sh.tps, sh.tiles,
                                          sh.nbox, sh.box_rows, sp, ein, out, eout, n, t.ptab_fwdT, ctr.p,
                                          t.sys_conv ? t.sys_conv + 2 * (1u << E) : nullptr);
    return cudaGetLastError();
}

}  // namespace

cudaError_t upload_const_twiddles(const FastTables& t, cudaStream_t st) {
    cudaError_t e = cudaMemcpyToSymbolAsync(c_twF, t.ptab_fwd, sizeof(c_twF), 0, cudaMemcpyDeviceToDevice, st);
    if (!e) e = cudaMemcpyToSymbolAsync(c_twI, t.ptab_inv, sizeof(c_twI), 0, cudaMemcpyDeviceToDevice, st);
    if (!e) e = cudaMemcpyToSymbolAsync(c_twFT, t.ptab_fwdT, sizeof(c_twFT), 0, cudaMemcpyDeviceToDevice, st);
    if (!e) e = cudaMemcpyToSymbolAsync(c_sysQ, t.sys_conv, sizeof(c_sysQ), 0, cudaMemcpyDeviceToDevice, st);
    if (!e) e = cudaMemcpyToSymbolAsync(c_sysT, t.sys_conv + kSysInvT, sizeof(c_sysT), 0, cudaMemcpyDeviceToDevice, st);
    return e;
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

// Q (group order of the fused conv pass) and r^-j (natural) Shoup pairs for
// N = 2^E at sys_conv + 2N: Q[f] = -sum_e G'[e] r^(e f), G'[e] = 1/(1 - r^-e).
// Built once per context; O(N^2) per size, N/128 CTAs each (every CTA rebuilds the power tables).
template <int E>
__global__ void sys_conv_kernel(uint2* __restrict__ base) {
    using G = typename Pick<E>::G;
    constexpr uint32_t N = 1u << E;
    constexpr int RLZ = G::RLZ, RZ = 1 << RLZ;
    __shared__ uint32_t rp[N], gp[N];
    uint2* out = base + 2 * N;
    const uint32_t r = gpow(3u, 65536u / N);
    for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) rp[e] = gpow(r, e);
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < N; e += blockDim.x) {
        const uint32_t x = rp[(N - e) & (N - 1u)];           // r^-e
        gp[e] = e ? ginv(1u + kP - x) : 0u;                  // 1 - r^-e in [2, p)
        const int32_t b = balanced(x);
        if (blockIdx.x == 0) out[N + e] = make_uint2(uint32_t(b), uint32_t(b * 65535));
    }
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const uint32_t g = i >> RLZ, j = i & uint32_t(RZ - 1);
        const uint32_t f = perm_head<E>(g) + (uint32_t(rev<RZ>(int(j))) << (E - RLZ));
        uint32_t acc = 0;
        for (uint32_t e = 1; e < N; ++e) acc = red2p(acc + gmul(gp[e], rp[(e * f) & (N - 1u)]));
        const int32_t b = balanced(acc ? kP - acc : 0u);
        out[i] = make_uint2(uint32_t(b), uint32_t(b * 65535));
    }
}

// sysw[p][j] = ahat[p][j] r^-j as balanced Shoup pairs (natural order), from the
// plan's ahat2 (slot order) and the r^-j half of the conv table
__global__ void sys_weights_kernel(uint32_t N, uint64_t total, const uint2* __restrict__ ahat2,
                                   const uint2* __restrict__ rinv, uint2* __restrict__ out) {
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < total; t += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t j = uint32_t(t & (N - 1u));
        const int32_t a = int32_t(ahat2[(t - j) + ahat2_slot(N, j)].x), r = int32_t(__ldg(rinv + j).x);
        const uint32_t ac = uint32_t(a < 0 ? a + int32_t(kP) : a), rc = uint32_t(r < 0 ? r + int32_t(kP) : r);
        const int32_t b = balanced(gmul(ac, rc));
        out[t] = make_uint2(uint32_t(b), uint32_t(b * 65535));
    }
}

cudaError_t launch_sys_weights(const FastTables& t, uint32_t N, uint32_t np, const uint2* ahat2, uint2* out,
                               cudaStream_t st) {
    if (N < 32 || N > 4096 || !np) return cudaSuccess;
    sys_weights_kernel<<<148 * 8, 256, 0, st>>>(N, uint64_t(np) * N, ahat2, t.sys_conv + 3 * N, out);
    return cudaGetLastError();
}

__global__ void sys_invt_kernel(uint2* invT) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 32 || i >= 512u) return;
    const int LL = 31 - __clz(i);
    const uint32_t sub = 1u << (LL - 4), j = i - (1u << LL), s = j / sub, t = j % sub;
    const uint32_t ex = (65536u - (((t * s) << (16 - LL)) & 0xFFFFu)) & 0xFFFFu;
    const int32_t w = balanced(gpow(3u, ex));
    invT[i] = make_uint2(uint32_t(w), uint32_t(w * 65535));
}

cudaError_t build_sys_conv(FastTables& t, cudaStream_t st) {
    cudaError_t err = cudaMalloc(&t.sys_conv, sizeof(uint2) * (kSysInvT + 512));
    if (err) return err;
    sys_invt_kernel<<<2, 256, 0, st>>>(t.sys_conv + kSysInvT);
    sys_conv_kernel<5><<<1, 128, 0, st>>>(t.sys_conv);
    sys_conv_kernel<6><<<1, 128, 0, st>>>(t.sys_conv);
    sys_conv_kernel<7><<<1, 128, 0, st>>>(t.sys_conv);
    sys_conv_kernel<8><<<2, 128, 0, st>>>(t.sys_conv);
    sys_conv_kernel<9><<<4, 128, 0, st>>>(t.sys_conv);
    sys_conv_kernel<10><<<8, 128, 0, st>>>(t.sys_conv);
    sys_conv_kernel<11><<<16, 128, 0, st>>>(t.sys_conv);
    sys_conv_kernel<12><<<32, 128, 0, st>>>(t.sys_conv);
    return cudaGetLastError();
}

// systematic codec, fused (MODE 1: decode, rows 0..k-1 out; MODE 2: encode
// with the plan of positions 0..k-1, rows 0..n-1 out)
cudaError_t launch_systematic_fast(const FastTables& t, const FastPlanView& pv, bool encode, uint32_t n,
                                   uint32_t stripes, uint32_t L, const uint32_t* sp, const uint16_t* in, EscIn ein,
                                   uint16_t* out, EscOut eout, cudaStream_t st) {
#define FNTRS_SYS(e)                                                                              \
    case (1u << e):                                                                               \
        if (FNTRS_SYS_CONV && pv.sysw)  /* weights built with the plan (capi.cu) */             \
            return encode ? launch_dec<e, 4>(t, pv, stripes, L, sp, in, ein, out, eout, st, n)   \
                          : launch_dec<e, 3>(t, pv, stripes, L, sp, in, ein, out, eout, st, n);  \
        return encode ? launch_dec<e, 2>(t, pv, stripes, L, sp, in, ein, out, eout, st, n)       \
                      : launch_dec<e, 1>(t, pv, stripes, L, sp, in, ein, out, eout, st, n);
    switch (pv.N) {
        FNTRS_SYS(5) FNTRS_SYS(6) FNTRS_SYS(7) FNTRS_SYS(8) FNTRS_SYS(9) FNTRS_SYS(10) FNTRS_SYS(11) FNTRS_SYS(12)
        default: return cudaErrorInvalidValue;
    }
#undef FNTRS_SYS
}

}  // namespace fast
}  // namespace fntrs_gpu
