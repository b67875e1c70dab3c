// internal.h -- host-side declarations shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/fntrs_gpu.h"

namespace fntrs_gpu {

// Twiddle tables: tw[m + j] = r_m^j (j < m) for every m = 2^e, e <= 16, in
// one buffer of 2^17 entries per direction (offset m). Built on the device.
struct Tables {
    uint32_t* fwd = nullptr;
    uint32_t* inv = nullptr;
};

cudaError_t build_tables(Tables& t, cudaStream_t st);

// Escape sink: sorted global symbol indices of values equal to 65536.
struct EscOut {
    unsigned long long* keys;   // capacity cap, pre-filled with ~0 by the caller
    unsigned long long* count;  // device counter (true count, may exceed cap)
    uint64_t cap;
};

struct EscIn {
    const unsigned long long* keys;  // sorted ascending
    uint64_t n;
};

// Tile geometry chosen for a transform needing `rows` shared-memory rows.
struct TileGeom {
    int wt;       // columns per tile (power of two, >= 2)
    int threads;  // threads per CTA
    size_t smem;  // dynamic shared memory bytes
};
TileGeom pick_tile(int rows, uint32_t L);

// Small-n (N = n_domain <= kTileMaxN) batched encode of packet-major stripes.
cudaError_t launch_encode_tile(const Tables& t, uint32_t k, uint32_t n, uint32_t N,
                               uint32_t stripes, uint32_t L, const uint16_t* src, EscIn esc_in,
                               uint16_t* out, EscOut esc_out, cudaStream_t st);

// Per-pattern decode data (device). ahat is already scaled by -1/M.
struct PlanView {
    uint32_t N, M, kp, k;        // domain, product size, positions per plan, outputs
    uint32_t npatterns;
    const uint32_t* positions;  // [np][kp]
    const uint32_t* ainv;       // [np][kp]
    const uint32_t* ahat;       // [np][M]
    uint32_t ninv;              // N^-1 (full-reception mode)
};

cudaError_t launch_decode_tile(const Tables& t, const PlanView& pv, uint32_t stripes, uint32_t L,
                               const uint32_t* stripe_pattern, const uint16_t* rx, EscIn esc_in,
                               uint16_t* out, EscOut esc_out, cudaStream_t st);

// Generic batched transform over columns: in/out [m][L] uint32 (natural order).
// scale multiplies every output (1/m for fnt_inverse, see launch site).
// poly_aux.cu: the reference's quadratic checkers, TransformPlan tables and polynomial helpers
cudaError_t launch_naive_dft(uint32_t r, uint32_t scale, uint32_t n, const uint32_t* in, uint32_t* out,
                             cudaStream_t st);
cudaError_t launch_transform_tables(uint32_t n, uint32_t root, uint32_t iroot, uint32_t* tw, uint32_t* itw,
                                    uint32_t* bitrev, uint32_t* stw, uint32_t* sitw, cudaStream_t st);
cudaError_t launch_pair_products(uint32_t npairs, const fntrs_poly_pair* pairs, const uint32_t* in, uint32_t* out,
                                 cudaStream_t st);
std::vector<uint32_t> tree_node_lengths(uint32_t k, std::vector<uint32_t>* level_nodes);
cudaError_t launch_subproduct_tree(uint32_t k, const uint32_t* xs, uint32_t* coeffs, cudaStream_t st);
cudaError_t launch_lagrange(uint32_t k, const uint32_t* xs, const uint32_t* vs, uint32_t* out, cudaStream_t st);
cudaError_t launch_derivative(uint32_t len, const uint32_t* a, uint32_t* out, cudaStream_t st);
cudaError_t launch_eval(uint32_t len, uint32_t x, const uint32_t* a, uint32_t* out, cudaStream_t st);
cudaError_t launch_chirp(uint32_t n, uint32_t root, uint32_t* b, uint32_t* binv, cudaStream_t st);
cudaError_t launch_geom_pre(uint32_t n, uint32_t len, const uint32_t* a, const uint32_t* binv, uint32_t* c,
                            cudaStream_t st);
cudaError_t launch_pointwise(uint32_t m, uint32_t* c, const uint32_t* B, cudaStream_t st);
cudaError_t launch_geom_post(uint32_t n, const uint32_t* c, const uint32_t* binv, uint32_t* out, cudaStream_t st);
cudaError_t launch_powers_scale(uint32_t len, uint32_t rho, const uint32_t* a, uint32_t* out, cudaStream_t st);

cudaError_t launch_fnt_tile(const Tables& t, uint32_t m, bool inverse, uint32_t scale, uint32_t L,
                            const uint32_t* in, uint32_t* out, cudaStream_t st);

// Plan precompute: direct products over the erasure positions.
cudaError_t launch_plan_build(uint32_t N, uint32_t M, uint32_t kp, uint32_t npatterns,
                              const uint32_t* positions, uint32_t* ainv, uint32_t* ahat,
                              const Tables& t, cudaStream_t st);

constexpr uint32_t kTileMaxN = 4096;

// Shard wire-format data movement (shards.cu)
cudaError_t launch_symbolize(const uint8_t* data, uint64_t len, uint32_t k, uint32_t L, uint16_t* src,
                             cudaStream_t st);
cudaError_t launch_desymbolize(const uint16_t* dec, uint32_t k, uint32_t L, uint64_t len, uint8_t* out,
                               cudaStream_t st);
cudaError_t launch_words_to_be(const uint16_t* rows, uint32_t nrows, uint32_t L, uint32_t count, uint8_t* out,
                               uint64_t pitch, cudaStream_t st);
cudaError_t launch_be_to_words(const uint8_t* in, uint64_t pitch, uint32_t nrows, uint32_t count, uint32_t L,
                               uint16_t* rows, cudaStream_t st);

// ---- v2 fast path (codec_fast.cu): 32 <= N <= 4096, L a multiple of the tile width
namespace fast {
struct FastTables {
    uint2* ptab_fwd = nullptr;  // per-pass twiddles {w, 65535 w}: [2^LL + 16 t + s] = r_(2^LL)^(t s)
    uint2* ptab_inv = nullptr;
    uint2* ptab_fwdT = nullptr;  // pass-0 twiddles transposed, N <= 256: [N + (N/16) s + t] = r_N^(t s)
    uint2* big_fwd = nullptr;   // {r_m^j, 65535 r_m^j} at [m + j], m <= 65536 (four-step twiddles)
    uint2* big_inv = nullptr;
    uint2* sys_conv = nullptr;  // systematic convolution tables, N = 32..4096 at [2N, 4N) (codec_dec.cu)
};
struct FastPlanView {
    uint32_t N, k;
    const uint2* rowmap;  // [np][N] {received row or ~0, 1/A'(x_i)}
    const uint2* ahat2;   // [np][N] {ahat_j, 65535 ahat_j} at slot ahat2_slot(N, j)
    const uint2* sysw = nullptr;  // [np][N] {ahat_j r^-j, 65535 ...} natural order (systematic conv form)
};
// Storage slot of ahat2 entry j (0 <= j < N, N a power of two). For the fused
// N <= 4096 decode kernel the table is kept in first-pass order, j = t + q 2^(E-4)
// -> t*16 + q, so each thread's 16 multipliers are two-per-uint4 contiguous;
// the four-step kernels (N >= 8192) read it in natural order.
__host__ __device__ inline uint32_t ahat2_slot(uint32_t N, uint32_t j) {
    if (N < 16 || N > 4096) return j;
    const uint32_t sl0 = uint32_t(31 - __builtin_clz(N)) - 4u;
    return ((j & ((1u << sl0) - 1u)) << 4) | (j >> sl0);
}
cudaError_t build_fast_tables(FastTables& t, cudaStream_t st);
cudaError_t build_sys_conv(FastTables& t, cudaStream_t st);
cudaError_t launch_sys_weights(const FastTables& t, uint32_t N, uint32_t np, const uint2* ahat2, uint2* out,
                               cudaStream_t st);
// host mirror of codec_dec.cu's FNTRS_SYS_CONV (the weights are only built when the conv form runs)
#ifndef FNTRS_SYS_CONV_HOST
#ifdef FNTRS_SYS_CONV
#define FNTRS_SYS_CONV_HOST FNTRS_SYS_CONV
#else
#define FNTRS_SYS_CONV_HOST 1
#endif
#endif
// constant-memory copies of the n_domain <= 256 pass-0 twiddle tables (codec_dec.cu)
cudaError_t upload_const_twiddles(const FastTables& t, cudaStream_t st);
int fast_tile_columns(uint32_t N);  // 0 when N has no fast kernel
int fast_encode_columns(uint32_t N);  // encode tile width (L must be a multiple)
// fused systematic codec on a fast plan (M == N); encode: the plan of positions 0..k-1
cudaError_t launch_systematic_fast(const FastTables& t, const FastPlanView& pv, bool encode, uint32_t n,
                                   uint32_t stripes, uint32_t L, const uint32_t* sp, const uint16_t* in, EscIn ein,
                                   uint16_t* out, EscOut eout, cudaStream_t st);
cudaError_t launch_encode_fast(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes,
                               uint32_t L, const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout,
                               cudaStream_t st);
cudaError_t launch_decode_fast(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                               const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                               cudaStream_t st);
cudaError_t launch_fast_plan_tables(uint32_t N, uint32_t kp, uint32_t npatterns, const uint32_t* pos,
                                    const uint32_t* ainv, const uint32_t* ahat, uint2* rowmap, uint2* ahat2,
                                    cudaStream_t st);

// ---- four-step path (codec_large.cu): 8192 <= N <= 65536, L a multiple of 64
cudaError_t build_large_tables(FastTables& t, cudaStream_t st);
int large_supported(uint32_t N);
uint32_t large_tile_columns();
uint32_t large_batch(uint32_t N, uint32_t L, size_t scratch_bytes);  // stripes per scratch buffer
// streamed four-step (codec_large.cu): one persistent launch, intermediates in
// L2-resident rings; FNTRS_STREAM=0 selects the batched four-kernel path
bool stream_enabled();
size_t stream_scratch_words(uint32_t N, uint32_t stripes, uint32_t L, bool decode);
cudaError_t launch_encode_stream(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes,
                                 uint32_t L, const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout,
                                 uint32_t* scratch, cudaStream_t st);
cudaError_t launch_decode_stream(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                                 const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                                 uint32_t* scratch, cudaStream_t st);
cudaError_t launch_encode_large(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes, uint32_t L,
                                const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, uint32_t* Y,
                                uint32_t batch, cudaStream_t st);
cudaError_t launch_decode_large(const FastTables& t, const FastPlanView& pv, uint32_t stripes, uint32_t L,
                                const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                                uint32_t* YA, uint32_t* YB, uint32_t batch, cudaStream_t st);

// ---- log-domain plans and column transforms (plan_fast.cu)
struct LogTables {
    uint32_t* exp3 = nullptr;  // 3^e, e < 65536
    uint16_t* log3 = nullptr;  // log_3(x) at [x - 1], x in [1, 65536]
};
cudaError_t build_log_tables(LogTables& lt, cudaStream_t st);
uint32_t plan_digit_width(uint32_t k);
// digit spectra Dh [N][D] (D = ceil(16 / w)); scratch: N*D words when N >= 8192
cudaError_t build_digit_spectra(const FastTables& t, const Tables& tab, const LogTables& lt, uint32_t N, uint32_t w,
                                uint32_t* Dh, uint32_t* scratch, cudaStream_t st);
size_t plan_fast_scratch_words(uint32_t N, uint32_t k, uint32_t P);
cudaError_t launch_plan_fast(const FastTables& t, const Tables& tab, const LogTables& lt, uint32_t N, uint32_t k,
                             uint32_t P, const uint32_t* pos, const uint32_t* Dh, uint32_t* scratch, uint32_t* ainv,
                             uint32_t* ahat, uint2* rowmap, uint2* ahat2, cudaStream_t st);
// natural-order column transforms [N][C] of any N <= 65536 (scratch N*C words when N >= 8192)
cudaError_t launch_fnt_cols(const FastTables& t, uint32_t N, bool inverse, uint32_t C, const uint32_t* in,
                            uint32_t* scratch, uint32_t* out, cudaStream_t st, bool unscaled = false);

// ---- fused decode for M != N (codec_gen.cu): 32 <= N <= 4096, M <= 4096
struct GenPlanView {
    uint32_t N, M, k;
    const uint2* rowmap;  // [np][N] {received row or ~0, balanced 1/A'(x_i)}
    const uint2* ahat2;   // [np][M] {w, 65535 w} of -A_hat/M, natural order
};
int gen_tile_columns(uint32_t N, uint32_t M);  // 0: no fused kernel for (N, M)
cudaError_t build_gen_pairs(uint32_t M, uint32_t P, const uint32_t* ahat, uint2* pairs, cudaStream_t st);
cudaError_t launch_decode_gen(const FastTables& t, const GenPlanView& pv, uint32_t stripes, uint32_t L,
                              const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                              cudaStream_t st);

// ---- general path (codec_cols.cu): column transforms through HBM, any shape
// with n_domain, M <= 65536
struct ColsPlanView {
    uint32_t N, M, k, kp, np;
    bool full;             // complete reception: one inverse transform
    bool split;            // 2k > 65536: product by halves (M = N = 65536)
    const uint2* rowmap;   // [np][N] {received row or ~0, balanced 1/A'(x_i) (1 when full)}
    const uint32_t* ahat;  // [np][M] -A_hat / M (unused when full)
    const uint32_t* alo;   // split: [M][np] -FNT(A_lo) / M
    const uint32_t* ahi;   // split: [M][np] -FNT(A_hi) / M
};
// split plans: alo/ahi ([65536][P]) from ahat ([P][65536]); c, T: [65536][P] scratch
cudaError_t build_split_spectra(const FastTables& t, uint32_t k, uint32_t P, const uint32_t* ahat, uint32_t* alo,
                                uint32_t* ahi, uint32_t* c, uint32_t* T, cudaStream_t st);
// columns per batch so one [max(N, M)][C] uint32 buffer stays within cap_bytes
uint64_t cols_batch_columns(uint32_t D, size_t cap_bytes);
cudaError_t build_cols_rowmap(uint32_t N, uint32_t kp, uint32_t P, const uint32_t* pos, const uint32_t* ainv,
                              uint2* rowmap, cudaStream_t st);
// A, T: [N][cap_cols] uint32 scratch each
cudaError_t launch_encode_cols(const FastTables& t, uint32_t k, uint32_t n, uint32_t N, uint32_t stripes, uint32_t L,
                               const uint16_t* src, EscIn ein, uint16_t* out, EscOut eout, uint32_t* A, uint32_t* T,
                               uint64_t cap_cols, cudaStream_t st);
// A, B, X, T: [max(N, M)][cap_cols] uint32 scratch each (X only for split plans)
cudaError_t launch_decode_cols(const FastTables& t, const ColsPlanView& pv, uint32_t stripes, uint32_t L,
                               const uint32_t* sp, const uint16_t* rx, EscIn ein, uint16_t* out, EscOut eout,
                               uint32_t* A, uint32_t* B, uint32_t* X, uint32_t* T, uint64_t cap_cols,
                               cudaStream_t st);
}  // namespace fast

}  // namespace fntrs_gpu
