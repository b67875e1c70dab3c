/* oracle/fntrs_oracle.h -- TEST INFRASTRUCTURE ONLY (see fntrs_oracle.c).
 * Status values are numerically identical to FNTRS_* in include/fntrs_gpu.h
 * so tests can compare error behaviour of the oracle and the product. */
#ifndef FNTRS_ORACLE_H
#define FNTRS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_E_ERROR = 1,
    ORC_E_ZERO_INVERSE = 2,
    ORC_E_INVALID_TRANSFORM_SIZE = 3,
    ORC_E_SIZE_MISMATCH = 4,
    ORC_E_PRODUCT_TOO_LARGE = 5,
    ORC_E_DUPLICATE_POINT = 6,
    ORC_E_DUPLICATE_POSITION = 7,
    ORC_E_POSITION_OUT_OF_RANGE = 8,
    ORC_E_TOO_FEW_POSITIONS = 9,
    ORC_E_NOT_ENOUGH_SYMBOLS = 10,
    ORC_E_TOO_MANY_ESCAPES = 11
};

uint32_t orc_add(uint32_t a, uint32_t b);
uint32_t orc_sub(uint32_t a, uint32_t b);
uint32_t orc_neg(uint32_t a);
uint32_t orc_mul(uint32_t a, uint32_t b);
uint32_t orc_pow(uint32_t base, uint64_t e);
uint32_t orc_inv(uint32_t a);
int orc_root_of_unity(uint32_t n, int inverse, uint32_t* out);

int orc_dif_forward(uint32_t n, uint32_t* d);
int orc_dit_inverse_unscaled(uint32_t n, uint32_t* d);
int orc_fnt_forward(uint32_t n, const uint32_t* in, uint32_t* out);
int orc_fnt_inverse(uint32_t n, const uint32_t* in, uint32_t* out);
void orc_naive_dft(uint32_t root, uint32_t n, const uint32_t* a, int inverse, uint32_t* out);

int orc_poly_mul(const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb, uint32_t* out);
int orc_subproduct_root(const uint32_t* xs, uint32_t k, uint32_t* a_out);
void orc_derivative(const uint32_t* a, uint32_t la, uint32_t* out);
uint32_t orc_eval_horner(const uint32_t* a, uint32_t la, uint32_t x);

int orc_build_plan(uint32_t n, uint32_t k, const uint32_t* positions, uint32_t* a_out,
                   uint32_t* aprime_inv, uint32_t* product_size, uint32_t* a_fnt);
int orc_interpolate(uint32_t n, uint32_t k, const uint32_t* positions, const uint32_t* aprime_inv,
                    uint32_t product_size, const uint32_t* a_fnt, const uint32_t* values,
                    uint32_t* out);
int orc_interpolate_low(uint32_t n, uint32_t k, const uint32_t* positions, const uint32_t* aprime_inv,
                        const uint32_t* a, const uint32_t* values, uint32_t* out);
int orc_lagrange(uint32_t k, const uint32_t* xs, const uint32_t* vs, uint32_t* out);

int orc_code_params(uint32_t k, uint32_t n, uint32_t* n_domain);
int orc_encode(uint32_t k, uint32_t n, const uint32_t* src, uint32_t* out);
int orc_decode(uint32_t k, uint32_t n, uint32_t count, const uint32_t* pos, const uint32_t* val,
               uint32_t* out);
int orc_encode_systematic(uint32_t k, uint32_t n, const uint32_t* src, uint32_t* out);
int orc_decode_systematic(uint32_t k, uint32_t n, uint32_t count, const uint32_t* pos, const uint32_t* val,
                          uint32_t* out);

int64_t orc_escape_split(const uint32_t* v, uint64_t count, uint16_t* words, uint32_t* esc);
void orc_escape_join(const uint16_t* words, uint64_t count, const uint32_t* esc, uint64_t ne,
                     uint32_t* v);

int64_t orc_encode_stripes(uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                           const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc,
                           uint16_t* out, uint64_t* out_esc, uint64_t esc_cap);
int64_t orc_decode_stripes(uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                           uint32_t npatterns, const uint32_t* patterns,
                           const uint32_t* stripe_pattern, const uint16_t* rx,
                           const uint64_t* rx_esc, uint64_t n_rx_esc, uint16_t* out,
                           uint64_t* out_esc, uint64_t esc_cap);

#ifdef __cplusplus
}
#endif
#endif
