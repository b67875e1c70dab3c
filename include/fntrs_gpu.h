/*
 * fntrs_gpu.h -- C ABI of the B200-native batched FNT Reed-Solomon codec
 * over GF(65537) (libfntrs_b200.so). Plain pointers and sizes; no C++ types.
 *
 * This is the drop-in boundary for the reference's non-systematic codec
 * path (/root/reference/proj/include/fntrs/codec.hpp). The reference has no
 * FFI; its callers link the C++ API statically. Each entry point below says
 * which reference interface it replaces. The C++ header include/fntrs/codec.hpp
 * restores the reference's exact C++ API (same namespace, names, signatures,
 * exception classes) on top of these functions.
 *
 * Data model (batched). A stripe is k source packets sharing one erasure
 * pattern; a packet is L uint16 symbols; codeword j of a stripe is symbol j
 * of every packet (reference CLI: proj/tools/fntrs_main.cpp:122-139).
 * Buffers are packet-major: src [stripes][k][L], encoded [stripes][n][L],
 * received [stripes][k][L], decoded [stripes][k][L], all uint16 in DEVICE
 * memory. A field value 65536 is stored as word 0 and its symbol index is
 * listed as an escape (proj/src/shardio.cpp:131-137,153-154,203-208).
 * Escape lists are ascending uint64 symbol indices into the buffer they
 * describe (index = row * L + col, row = stripe * rows_per_stripe + packet),
 * which is the reference's per-shard ascending list, concatenated.
 *
 * Errors: every function returns an fntrs_status. Values 1..18 map 1:1 onto
 * the reference exception classes (proj/include/fntrs/errors.hpp:9-38).
 * Calls on one context must be serialised by the caller; contexts on
 * different devices are independent. All work is enqueued on `stream`
 * (a cudaStream_t, NULL = legacy default stream); device pointers are
 * caller-owned. There is no CPU fallback: without a usable CUDA device,
 * fntrs_gpu_create fails with FNTRS_E_CUDA.
 */
#ifndef FNTRS_GPU_H
#define FNTRS_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fntrs_status {
    FNTRS_OK = 0,
    FNTRS_E_ERROR = 1,                  /* fntrs::Error */
    FNTRS_E_ZERO_INVERSE = 2,           /* fntrs::ZeroInverse */
    FNTRS_E_INVALID_TRANSFORM_SIZE = 3, /* fntrs::InvalidTransformSize */
    FNTRS_E_SIZE_MISMATCH = 4,          /* fntrs::SizeMismatch */
    FNTRS_E_PRODUCT_TOO_LARGE = 5,      /* fntrs::ProductTooLarge */
    FNTRS_E_DUPLICATE_POINT = 6,        /* fntrs::DuplicatePoint */
    FNTRS_E_DUPLICATE_POSITION = 7,     /* fntrs::DuplicatePosition */
    FNTRS_E_POSITION_OUT_OF_RANGE = 8,  /* fntrs::PositionOutOfRange */
    FNTRS_E_TOO_FEW_POSITIONS = 9,      /* fntrs::TooFewPositions */
    FNTRS_E_NOT_ENOUGH_SYMBOLS = 10,    /* fntrs::NotEnoughSymbols */
    FNTRS_E_TOO_MANY_ESCAPES = 11,      /* fntrs::TooManyEscapes (also: escape buffer too small) */
    FNTRS_E_BAD_MAGIC = 12,
    FNTRS_E_BAD_VERSION = 13,
    FNTRS_E_TRUNCATED_SHARD = 14,
    FNTRS_E_MALFORMED_ESCAPES = 15,
    FNTRS_E_MALFORMED_HEADER = 16,
    FNTRS_E_LENGTH_MISMATCH = 17,
    FNTRS_E_NOT_ENOUGH_SHARDS = 18,
    FNTRS_E_CUDA = 100,          /* CUDA runtime error; see fntrs_gpu_last_error */
    FNTRS_E_UNSUPPORTED = 101,   /* shape outside this build (e.g. 2k > 65536) */
    FNTRS_E_INVALID_ARGUMENT = 102
} fntrs_status;

typedef struct fntrs_ctx fntrs_ctx;
typedef struct fntrs_plans fntrs_plans;

/* Library / context. The context owns the twiddle tables (r_m^j for every
 * m | 65536, both directions) and scratch; replaces the reference's
 * mutex-guarded plan registry (proj/src/transform.cpp:66-75). */
int fntrs_gpu_create(int device, fntrs_ctx** out);
int fntrs_gpu_destroy(fntrs_ctx* ctx);
const char* fntrs_gpu_status_string(int status);
const char* fntrs_gpu_last_error(const fntrs_ctx* ctx);
int fntrs_gpu_device(const fntrs_ctx* ctx);
const char* fntrs_gpu_version(void);

/* codec::CodeParams::make (proj/src/codec.cpp:112-122): validates
 * 1 <= k <= n <= 65536 and returns n_domain = next power of two >= n. */
int fntrs_gpu_code_params(uint32_t k, uint32_t n, uint32_t* n_domain);

/* Batched codec::encode_nonsystematic (proj/src/codec.cpp:124-131): for every
 * codeword, zero-pad the k source symbols to n_domain, forward FNT, keep the
 * first n outputs.
 *   src      [stripes][k][L] uint16;  src_esc: n_src_esc sorted indices into src
 *   out      [stripes][n][L] uint16;  out_esc: capacity esc_cap (uint64)
 *   n_out_esc  DEVICE uint64 receiving the true escape count; when it exceeds
 *              esc_cap only esc_cap entries were kept and the list is invalid. */
int fntrs_gpu_encode(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                     const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc,
                     uint16_t* out, uint64_t* out_esc, uint64_t esc_cap, uint64_t* n_out_esc,
                     void* stream);

/* Once-per-erasure-pattern decode plans: interp::build_plan / plan_for
 * (proj/src/interp.cpp:23-101), batched over patterns, computed on the GPU.
 * positions: HOST array [npatterns][kp]; pattern p lists the kp received
 * positions (distinct, < n) in the order the received packets will follow.
 * kp must equal k, or n when n == n_domain (complete reception: decode is
 * one inverse transform, codec.cpp:137-144). */
int fntrs_gpu_plans_create(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t kp,
                           uint32_t npatterns, const uint32_t* positions, fntrs_plans** out,
                           void* stream);
/* Plan buffers are stream-ordered allocations on the creation stream and are
 * released in that stream's order (work queued before destroy may still use
 * them). Use pinned host positions for a fully asynchronous create. */
int fntrs_gpu_plans_destroy(fntrs_plans* plans);
uint32_t fntrs_gpu_plans_count(const fntrs_plans* plans);

/* DecodePlan fields of one pattern (proj/include/fntrs/interp.hpp:18-32), to
 * HOST buffers: a_coeffs [kp+1] (the locator A, monic), aprime_inv [kp],
 * *product_size, a_fnt [product_size] (dif_forward order, bit-reversed).
 * Synchronises the context's internal stream. */
int fntrs_gpu_plans_export(fntrs_ctx* ctx, const fntrs_plans* plans, uint32_t pattern,
                           uint32_t* a_coeffs, uint32_t* aprime_inv, uint32_t* product_size,
                           uint32_t* a_fnt);

/* Batched codec::decode_nonsystematic (proj/src/codec.cpp:133-149 ->
 * interp::interpolate, interp.cpp:103-137).
 *   stripe_pattern DEVICE [stripes] uint32: plan index of each stripe
 *   rx   [stripes][kp][L] uint16: row i of stripe s is the packet received at
 *        position i of that stripe's pattern;  rx_esc sorted indices into rx
 *   out  [stripes][k][L] uint16 decoded source packets; out_esc as in encode */
int fntrs_gpu_decode(fntrs_ctx* ctx, const fntrs_plans* plans, uint32_t stripes, uint32_t L,
                     const uint32_t* stripe_pattern, const uint16_t* rx, const uint64_t* rx_esc,
                     uint64_t n_rx_esc, uint16_t* out, uint64_t* out_esc, uint64_t esc_cap,
                     uint64_t* n_out_esc, void* stream);

/* Batched systematic codec (proj/src/codec.cpp:151-196); symbols 0..k-1 of
 * every codeword are the source itself.
 *   encode_systematic: P = interpolate(positions 0..k-1, source)
 *     (codec.cpp:156-159), out = FNT_{n_domain}(P) truncated to n
 *     (transform_of_padded, codec.cpp:75-82). Buffers as in fntrs_gpu_encode.
 *   decode_systematic: P = interpolate(the plan's k positions, rx)
 *     (interpolate_selected, codec.cpp:85-94), out = FNT_{n_domain}(P)
 *     truncated to k. Plans/buffers as in fntrs_gpu_decode; out [stripes][k][L].
 *     Stripes whose pattern is 0..k-1 reproduce rx exactly, which is the
 *     reference's systematic_prefix_present copy (codec.cpp:167-171).
 * Both run the interpolation kernels into a stream-ordered intermediate and
 * then the forward transform kernels; the intermediate's escape count is read
 * back once, so each call synchronises `stream` once. rate 1 (k == n) encode
 * is a device copy. */
int fntrs_gpu_encode_systematic(fntrs_ctx* ctx, uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                                const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc,
                                uint16_t* out, uint64_t* out_esc, uint64_t esc_cap, uint64_t* n_out_esc,
                                void* stream);
int fntrs_gpu_decode_systematic(fntrs_ctx* ctx, const fntrs_plans* plans, uint32_t stripes, uint32_t L,
                                const uint32_t* stripe_pattern, const uint16_t* rx, const uint64_t* rx_esc,
                                uint64_t n_rx_esc, uint16_t* out, uint64_t* out_esc, uint64_t esc_cap,
                                uint64_t* n_out_esc, void* stream);

/* Shard wire format, data movement on the device (proj/src/shardio.cpp).
 * The reference CLI codes a file as S = ceil(ceil(len/2) / k) one-codeword
 * stripes and shard j holds symbol j of every stripe; in the batched model
 * that is ONE stripe of k packets with L >= S symbols (columns >= S are zero
 * padding), and row j of the encoded stripe is shard j's payload.
 *   symbolize   (shardio.cpp:83-96):  DEVICE bytes[len] -> src[k][L] uint16,
 *               src[i][t] = big-endian word t*k + i (zero past the data)
 *   desymbolize (shardio.cpp:98-116): dec[k][L] -> DEVICE bytes[len]
 *   words_to_be (write_shard payload, shardio.cpp:153-154): rows[nrows][L] ->
 *               out[r*pitch + 2t .. +1] big-endian, t < count
 *   be_to_words (read_shard payload, shardio.cpp:203-208): the inverse, columns
 *               count..L-1 zeroed
 * Headers, escape lists and manifests are host formatting (shards.py). */
int fntrs_gpu_symbolize(fntrs_ctx* ctx, const uint8_t* data, uint64_t len, uint32_t k, uint32_t L, uint16_t* src,
                        void* stream);
int fntrs_gpu_desymbolize(fntrs_ctx* ctx, const uint16_t* dec, uint32_t k, uint32_t L, uint64_t len, uint8_t* out,
                          void* stream);
int fntrs_gpu_words_to_be(fntrs_ctx* ctx, const uint16_t* rows, uint32_t nrows, uint32_t L, uint32_t count,
                          uint8_t* out, uint64_t pitch, void* stream);
int fntrs_gpu_be_to_words(fntrs_ctx* ctx, const uint8_t* in, uint64_t pitch, uint32_t nrows, uint32_t count,
                          uint32_t L, uint16_t* rows, void* stream);

/* fnt_forward / fnt_inverse (proj/src/transform.cpp:302-323) over the columns
 * of a DEVICE [m][L] uint32 array of canonical values; natural order.
 * inverse: 0 forward, 1 inverse (times 1/m), 2 inverse without the 1/m factor
 * (dit_inverse_unscaled's arithmetic, transform.hpp:43-48, in natural order). */
int fntrs_gpu_fnt(fntrs_ctx* ctx, uint32_t m, int inverse, uint32_t L, const uint32_t* in,
                  uint32_t* out, void* stream);

/* Seeded synthetic source symbols (benchmark workload):
 * out[i] = low 16 bits of output number (first_index + i) of the splitmix64
 * stream seeded with `seed` (state_j = seed + (j+1) * 0x9E3779B97F4A7C15).
 * DEVICE buffer; the same generator is restated in numpy for the tests. */
int fntrs_gpu_fill_symbols(uint64_t seed, uint64_t first_index, uint64_t count, uint16_t* out,
                           void* stream);

/* Kernel selection: the fused v2 kernels (codec_fast.cu) serve n_domain in
 * [32, 4096] with L a multiple of the tile width; every other shape runs the
 * general tile kernels (codec_tile.cu). enabled = 0 forces the general
 * kernels (used by tests to cross-check the two). Both are GPU kernels. */
int fntrs_gpu_set_fast_path(fntrs_ctx* ctx, int enabled);

/* Launch accounting: number of kernels this context has launched. */
uint64_t fntrs_gpu_launch_count(const fntrs_ctx* ctx);

/* Transform accounting (the reference's note_fnt_execution tally,
 * proj/src/transform.cpp:292-316 -> proj/src/instrument.cpp:15-18): counts[e]
 * = transforms of size 2^e this context's kernels have executed so far
 * (e = 0..16), added by each launch from the schedule of the kernel family it
 * actually ran (codewords x transforms per codeword at each size). A caller
 * diffs two snapshots around a call. */
int fntrs_gpu_transform_counts(const fntrs_ctx* ctx, uint64_t counts[17]);

/* ---- the rest of the reference's public API, on the device ---------------
 * Not on the batched codec path; these let the reference's own consumers
 * (proj/tests/acceptance.cpp) link against the drop-in. All pointers DEVICE,
 * values canonical in [0, 65536]. */

/* naive_dft (proj/include/fntrs/transform.hpp:52, transform.cpp:325-343):
 * out_j = sum_i in_i root^(ij) for ANY root (inverse: root^-1 and * 1/n). */
int fntrs_gpu_naive_dft(fntrs_ctx* ctx, uint32_t root, int inverse, uint32_t n, const uint32_t* in,
                        uint32_t* out, void* stream);

/* TransformPlan's tables (transform.hpp:17-28, transform.cpp:31-63) for size
 * n (power of two <= 65536): twiddles / inverse_twiddles [n/2], bit_reversal
 * [n], stage_twiddles / stage_inverse_twiddles [n-1]. Any pointer may be NULL. */
int fntrs_gpu_transform_tables(fntrs_ctx* ctx, uint32_t n, uint32_t* twiddles, uint32_t* inverse_twiddles,
                               uint32_t* bit_reversal, uint32_t* stage_twiddles, uint32_t* stage_inverse_twiddles,
                               void* stream);

/* One polynomial product: out[a_len + b_len - 1] = a * b, coefficient
 * segments of one DEVICE word array (poly::mul, proj/src/poly.cpp:22-137). */
typedef struct fntrs_poly_pair {
    uint64_t a_off, b_off, out_off;
    uint32_t a_len, b_len;
} fntrs_poly_pair;
/* Batched products: pairs is a HOST array of npairs descriptors into `in`
 * (read) and `out` (written); in and out may be the same array when the
 * written segments do not overlap the read ones. */
int fntrs_gpu_poly_products(fntrs_ctx* ctx, uint32_t npairs, const fntrs_poly_pair* pairs, const uint32_t* in,
                            uint32_t* out, void* stream);

/* Subproduct tree of k points (poly::build_subproduct_tree,
 * proj/src/poly.cpp:216-242): leaves (x - x_i), each level pairing adjacent
 * nodes and carrying an odd last node up. fntrs_gpu_subproduct_tree_layout
 * gives the level count, nodes per level (cap >= levels entries) and the
 * coefficient count per node in level order (node_len may be NULL; count in
 * *n_nodes), the total in *n_coeffs; coeffs receives all nodes back to back. */
int fntrs_gpu_subproduct_tree_layout(uint32_t k, uint32_t* n_levels, uint32_t* level_nodes, uint32_t level_cap,
                                     uint32_t* node_len, uint64_t* n_nodes, uint64_t* n_coeffs);
int fntrs_gpu_subproduct_tree(fntrs_ctx* ctx, uint32_t k, const uint32_t* points, uint32_t* coeffs, void* stream);

/* interp::lagrange_oracle (proj/include/fntrs/interp.hpp:56,
 * proj/src/interp.cpp:139-171): the unique P, deg P < k, with P(xs[i]) = vs[i]
 * for k DISTINCT points (the caller validates), out[k] coefficients
 * (trailing zeros not trimmed). */
int fntrs_gpu_lagrange(fntrs_ctx* ctx, uint32_t k, const uint32_t* xs, const uint32_t* vs, uint32_t* out,
                       void* stream);

/* Evaluation at geometric points (proj/include/fntrs/geom.hpp, proj/src/geom.cpp):
 * fntrs_gpu_chirp_table fills the reference's ChirpTable vectors for size n
 * (power of two <= 65536) and any root: b[2n-1] (b_i = root^(i(i-1)/2)),
 * b_inverse[n], and b_spectrum[2n] = FNT_2n(b zero-padded) in NATURAL order
 * (any pointer may be NULL; n = 65536 is the full-domain case: nothing to
 * fill). fntrs_gpu_geom_eval writes out[n] = a(root^i), i < n, for a of len <=
 * n coefficients, by the chirp (two FNT_2n and a pointwise product), or for n
 * = 65536 by the transform itself (root must be the domain root or its
 * inverse: InvalidTransformSize otherwise). fntrs_gpu_geom_eval_negative:
 * out[j] = a(root^-(j+1)). All buffers DEVICE. */
int fntrs_gpu_chirp_table(fntrs_ctx* ctx, uint32_t n, uint32_t root, uint32_t* b, uint32_t* b_inverse,
                          uint32_t* b_spectrum, void* stream);
int fntrs_gpu_geom_eval(fntrs_ctx* ctx, uint32_t n, uint32_t root, const uint32_t* a, uint32_t len,
                        const uint32_t* b_inverse, const uint32_t* b_spectrum, uint32_t* out, void* stream);
int fntrs_gpu_geom_eval_negative(fntrs_ctx* ctx, uint32_t n, uint32_t root, const uint32_t* a, uint32_t len,
                                 const uint32_t* b_inverse, const uint32_t* b_spectrum, uint32_t* out, void* stream);
/* (b_inverse / b_spectrum: a cached chirp table of `root` -- for the negative
 * direction, of root^-1 -- as fntrs_gpu_chirp_table fills it, or NULL to build
 * one: with a cached table an evaluation runs two FNT_2n, as the reference's.) */

/* poly::derivative (out[len-1]) and poly::eval_horner (*out = a(x)),
 * proj/src/poly.cpp:201-214. */
int fntrs_gpu_poly_derivative(fntrs_ctx* ctx, uint32_t len, const uint32_t* a, uint32_t* out, void* stream);
int fntrs_gpu_poly_eval(fntrs_ctx* ctx, uint32_t len, const uint32_t* a, uint32_t x, uint32_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FNTRS_GPU_H */
