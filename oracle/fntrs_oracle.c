/*
 * oracle/fntrs_oracle.c -- CPU restatement of the reference fntrs codec path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_0907_1788_b200/,
 * include/, the CUDA library) links, loads or calls this file. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, and only as the checker.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * the golden vectors frozen in the reference's own tests (field, transform,
 * geom, interp, codec, shardio) and, when oracle/_ref was
 * built, against the reference library itself on seeded random inputs.
 *
 * Every function cites the reference code (paths relative to
 * /root/reference/) whose behaviour it restates. The arithmetic is the
 * reference's: GF(65537), canonical values in [0, 65536], root of order n
 * r_n = 3^(65536/n).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "fntrs_oracle.h"

#define P 65537u

/* ---- field: proj/include/fntrs/field.hpp:18-63 ------------------------ */

uint32_t orc_add(uint32_t a, uint32_t b) { /* field.hpp:18-21 */
    uint32_t s = a + b;
    return s >= P ? s - P : s;
}

uint32_t orc_sub(uint32_t a, uint32_t b) { /* field.hpp:23-26 */
    return a >= b ? a - b : a + (P - b);
}

uint32_t orc_neg(uint32_t a) { return a == 0 ? 0 : P - a; } /* field.hpp:28 */

uint32_t orc_mul(uint32_t a, uint32_t b) { /* field.hpp:30-37, 2^16 = -1 fold */
    uint64_t x = (uint64_t)a * b;
    uint32_t lo = (uint32_t)(x & 0xFFFFu), hi = (uint32_t)(x >> 16);
    return lo >= hi ? lo - hi : lo + P - hi;
}

uint32_t orc_pow(uint32_t base, uint64_t e) { /* field.hpp:39-49 (0^0 checked by caller) */
    uint32_t r = 1, b = base;
    while (e) {
        if (e & 1) r = orc_mul(r, b);
        e >>= 1;
        if (e) b = orc_mul(b, b);
    }
    return r;
}

uint32_t orc_inv(uint32_t a) { return orc_pow(a, P - 2); } /* field.hpp:52-55 */

static int is_pow2_le(uint32_t n, uint32_t cap) { return n && n <= cap && !(n & (n - 1)); }

int orc_root_of_unity(uint32_t n, int inverse, uint32_t* out) { /* field.hpp:58-63 */
    if (!is_pow2_le(n, 65536)) return ORC_E_INVALID_TRANSFORM_SIZE;
    uint32_t r = orc_pow(3, 65536u / n);
    *out = inverse ? orc_inv(r) : r;
    return ORC_OK;
}

static uint32_t root_n(uint32_t n, int inverse) {
    uint32_t r = 0;
    orc_root_of_unity(n, inverse, &r);
    return r;
}

static uint32_t log2u(uint32_t n) {
    uint32_t l = 0;
    while ((1u << l) < n) ++l;
    return l;
}

static uint32_t next_pow2(uint32_t n) {
    uint32_t m = 1;
    while (m < n) m <<= 1;
    return m;
}

/* ---- transform: proj/src/transform.cpp ---------------------------------
 * Radix-2 Gentleman-Sande DIF (natural in, bit-reversed out) and
 * Cooley-Tukey DIT (bit-reversed in, natural out), transform.cpp:90-122,
 * with the per-stage twiddle regrouping of transform.cpp:52-63. */

typedef struct {
    uint32_t n;
    uint32_t* stage;     /* forward stage twiddles, offset n - len */
    uint32_t* stage_inv; /* inverse stage twiddles */
    uint32_t* rev;       /* bit reversal */
    uint32_t size_inv;
} tplan;

static tplan g_plans[17];

static const tplan* plan_for(uint32_t n) { /* transform.cpp:31-75 (unsynchronised: tests are single-threaded) */
    uint32_t lg = log2u(n);
    tplan* p = &g_plans[lg];
    if (p->n == n) return p;
    p->n = n;
    uint32_t r = root_n(n, 0), ri = root_n(n, 1);
    uint32_t half = n / 2;
    uint32_t* tw = (uint32_t*)malloc(sizeof(uint32_t) * (half ? half : 1));
    uint32_t* twi = (uint32_t*)malloc(sizeof(uint32_t) * (half ? half : 1));
    uint32_t w = 1, wi = 1;
    for (uint32_t j = 0; j < half; ++j) {
        tw[j] = w;
        twi[j] = wi;
        w = orc_mul(w, r);
        wi = orc_mul(wi, ri);
    }
    p->stage = (uint32_t*)malloc(sizeof(uint32_t) * (n > 1 ? n - 1 : 1));
    p->stage_inv = (uint32_t*)malloc(sizeof(uint32_t) * (n > 1 ? n - 1 : 1));
    uint32_t off = 0;
    for (uint32_t len = n; len >= 2; len >>= 1) {
        uint32_t h = len >> 1, stride = n / len;
        for (uint32_t j = 0; j < h; ++j) {
            p->stage[off + j] = tw[j * stride];
            p->stage_inv[off + j] = twi[j * stride];
        }
        off += h;
    }
    free(tw);
    free(twi);
    p->rev = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t i = 0; i < n; ++i) {
        uint32_t x = 0;
        for (uint32_t b = 0; b < lg; ++b) x |= ((i >> b) & 1u) << (lg - 1 - b);
        p->rev[i] = x;
    }
    p->size_inv = orc_inv(n % P);
    return p;
}

static void dif_core(uint32_t* d, uint32_t n, const uint32_t* stages) { /* transform.cpp:90-104 */
    for (uint32_t len = n; len >= 2; len >>= 1) {
        uint32_t h = len >> 1;
        const uint32_t* tw = stages + (n - len);
        for (uint32_t base = 0; base < n; base += len)
            for (uint32_t j = 0; j < h; ++j) {
                uint32_t u = d[base + j], v = d[base + h + j];
                d[base + j] = orc_add(u, v);
                d[base + h + j] = orc_mul(orc_sub(u, v), tw[j]);
            }
    }
}

static void dit_core(uint32_t* d, uint32_t n, const uint32_t* stages) { /* transform.cpp:107-122 */
    for (uint32_t len = 2; len <= n; len <<= 1) {
        uint32_t h = len >> 1;
        const uint32_t* tw = stages + (n - len);
        for (uint32_t base = 0; base < n; base += len)
            for (uint32_t j = 0; j < h; ++j) {
                uint32_t u = d[base + j], v = orc_mul(d[base + h + j], tw[j]);
                d[base + j] = orc_add(u, v);
                d[base + h + j] = orc_sub(u, v);
            }
    }
}

static void permute(const tplan* p, uint32_t* d) { /* transform.cpp:281-286 */
    for (uint32_t i = 0; i < p->n; ++i) {
        uint32_t j = p->rev[i];
        if (i < j) {
            uint32_t t = d[i];
            d[i] = d[j];
            d[j] = t;
        }
    }
}

int orc_dif_forward(uint32_t n, uint32_t* d) { /* transform.cpp:290-294 */
    if (!is_pow2_le(n, 65536)) return ORC_E_INVALID_TRANSFORM_SIZE;
    const tplan* p = plan_for(n);
    if (n >= 2) dif_core(d, n, p->stage);
    return ORC_OK;
}

int orc_dit_inverse_unscaled(uint32_t n, uint32_t* d) { /* transform.cpp:296-300 */
    if (!is_pow2_le(n, 65536)) return ORC_E_INVALID_TRANSFORM_SIZE;
    const tplan* p = plan_for(n);
    if (n >= 2) dit_core(d, n, p->stage_inv);
    return ORC_OK;
}

int orc_fnt_forward(uint32_t n, const uint32_t* in, uint32_t* out) { /* transform.cpp:302-311 */
    if (!is_pow2_le(n, 65536)) return ORC_E_INVALID_TRANSFORM_SIZE;
    const tplan* p = plan_for(n);
    if (out != in) memcpy(out, in, sizeof(uint32_t) * n);
    if (n >= 2) {
        dif_core(out, n, p->stage);
        permute(p, out);
    }
    return ORC_OK;
}

int orc_fnt_inverse(uint32_t n, const uint32_t* in, uint32_t* out) { /* transform.cpp:313-323 */
    if (!is_pow2_le(n, 65536)) return ORC_E_INVALID_TRANSFORM_SIZE;
    const tplan* p = plan_for(n);
    if (out != in) memcpy(out, in, sizeof(uint32_t) * n);
    if (n >= 2) {
        permute(p, out);
        dit_core(out, n, p->stage_inv);
    }
    for (uint32_t i = 0; i < n; ++i) out[i] = orc_mul(out[i], p->size_inv);
    return ORC_OK;
}

void orc_naive_dft(uint32_t root, uint32_t n, const uint32_t* a, int inverse, uint32_t* out) { /* transform.cpp:325-343 */
    uint32_t r = inverse ? orc_inv(root) : root;
    for (uint32_t j = 0; j < n; ++j) {
        uint32_t rj = orc_pow(r, j), acc = 0, w = 1;
        for (uint32_t i = 0; i < n; ++i) {
            acc = orc_add(acc, orc_mul(a[i], w));
            w = orc_mul(w, rj);
        }
        out[j] = acc;
    }
    if (inverse && n) {
        uint32_t ninv = orc_inv(n % P);
        for (uint32_t j = 0; j < n; ++j) out[j] = orc_mul(out[j], ninv);
    }
}

/* ---- poly: proj/src/poly.cpp ------------------------------------------
 * Exact products. The reference's tier dispatcher (poly.cpp:125-137) picks
 * schoolbook / Karatsuba / transform by length; every tier returns the same
 * exact product, so the restatement uses schoolbook below 64 coefficients
 * and the transform product (poly.cpp:79-99) above. */

static void mul_school(const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb, uint32_t* out) {
    memset(out, 0, sizeof(uint32_t) * (la + lb - 1));
    for (uint32_t i = 0; i < la; ++i) {
        if (!a[i]) continue;
        for (uint32_t j = 0; j < lb; ++j) out[i + j] = orc_add(out[i + j], orc_mul(a[i], b[j]));
    }
}

/* Returns ORC_E_PRODUCT_TOO_LARGE past 65536 coefficients (poly.cpp:82-83). */
int orc_poly_mul(const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb, uint32_t* out) {
    if (!la || !lb) return ORC_OK;
    uint32_t len = la + lb - 1;
    if (len < 64) {
        mul_school(a, la, b, lb, out);
        return ORC_OK;
    }
    if (len > 65536) return ORC_E_PRODUCT_TOO_LARGE;
    uint32_t m = next_pow2(len);
    const tplan* p = plan_for(m);
    uint32_t* fa = (uint32_t*)calloc(m, sizeof(uint32_t));
    uint32_t* fb = (uint32_t*)calloc(m, sizeof(uint32_t));
    memcpy(fa, a, sizeof(uint32_t) * la);
    memcpy(fb, b, sizeof(uint32_t) * lb);
    dif_core(fa, m, p->stage);
    dif_core(fb, m, p->stage);
    for (uint32_t i = 0; i < m; ++i) fa[i] = orc_mul(orc_mul(fa[i], fb[i]), p->size_inv);
    dit_core(fa, m, p->stage_inv);
    memcpy(out, fa, sizeof(uint32_t) * len);
    free(fa);
    free(fb);
    return ORC_OK;
}

/* Root of the subproduct tree, prod (x - x_i), k+1 coefficients (monic).
 * Pairs adjacent nodes level by level and carries an odd node up
 * (poly.cpp:216-242). */
int orc_subproduct_root(const uint32_t* xs, uint32_t k, uint32_t* a_out) {
    if (!k) return ORC_E_ERROR;
    /* each node stored in a slab: node i of the current level has len[i] coeffs */
    uint32_t* cur = (uint32_t*)malloc(sizeof(uint32_t) * 2 * k);
    uint32_t* nxt = (uint32_t*)malloc(sizeof(uint32_t) * 2 * k);
    uint32_t* off = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
    uint32_t* noff = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
    uint32_t cnt = k;
    for (uint32_t i = 0; i < k; ++i) {
        cur[2 * i] = orc_neg(xs[i]);
        cur[2 * i + 1] = 1;
        off[i] = 2 * i;
    }
    off[k] = 2 * k;
    int rc = ORC_OK;
    while (cnt > 1) {
        uint32_t ncnt = 0, pos = 0;
        for (uint32_t i = 0; i + 1 < cnt; i += 2) {
            uint32_t la = off[i + 1] - off[i], lb = off[i + 2] - off[i + 1];
            noff[ncnt++] = pos;
            rc = orc_poly_mul(cur + off[i], la, cur + off[i + 1], lb, nxt + pos);
            if (rc) goto done;
            pos += la + lb - 1;
        }
        if (cnt & 1) {
            uint32_t la = off[cnt] - off[cnt - 1];
            noff[ncnt++] = pos;
            memcpy(nxt + pos, cur + off[cnt - 1], sizeof(uint32_t) * la);
            pos += la;
        }
        noff[ncnt] = pos;
        uint32_t* t = cur; cur = nxt; nxt = t;
        t = off; off = noff; noff = t;
        cnt = ncnt;
    }
    memcpy(a_out, cur, sizeof(uint32_t) * (k + 1));
done:
    free(cur); free(nxt); free(off); free(noff);
    return rc;
}

void orc_derivative(const uint32_t* a, uint32_t la, uint32_t* out) { /* poly.cpp:201-208 (un-normalised) */
    for (uint32_t i = 1; i < la; ++i) out[i - 1] = orc_mul(a[i], i % P);
}

uint32_t orc_eval_horner(const uint32_t* a, uint32_t la, uint32_t x) { /* poly.cpp:210-214 */
    uint32_t acc = 0;
    for (uint32_t i = la; i-- > 0;) acc = orc_add(orc_mul(acc, x), a[i]);
    return acc;
}

/* ---- interp: proj/src/interp.cpp --------------------------------------- */

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

/* build_plan (interp.cpp:23-68). positions: k distinct values < n, in the
 * order values will follow. Outputs (caller-sized):
 *   a_out[k+1]        A = prod (x - r^z_i)                     (DecodePlan::a())
 *   aprime_inv[k]     1/A'(r^z_i)                              (aprime_at_x_inv)
 *   *product_size     next_pow2(2k), or 0 when 2k > 65536
 *   a_fnt[product_size] dif_forward(A padded), bit-reversed order  (a_fnt)
 * A' is evaluated on the whole domain with one size-n transform: geom_eval on
 * the chirp for (n, r) equals fnt_forward of the padded polynomial
 * (test_geom.cpp:125-131; geom.cpp:59-63 does exactly this at n = 65536). */
int orc_build_plan(uint32_t n, uint32_t k, const uint32_t* positions, uint32_t* a_out,
                   uint32_t* aprime_inv, uint32_t* product_size, uint32_t* a_fnt) {
    if (!k) return ORC_E_TOO_FEW_POSITIONS;
    if (!is_pow2_le(n, 65536)) return ORC_E_INVALID_TRANSFORM_SIZE;
    for (uint32_t i = 0; i < k; ++i)
        if (positions[i] >= n) return ORC_E_POSITION_OUT_OF_RANGE;
    uint32_t* sorted = (uint32_t*)malloc(sizeof(uint32_t) * k);
    memcpy(sorted, positions, sizeof(uint32_t) * k);
    qsort(sorted, k, sizeof(uint32_t), cmp_u32);
    for (uint32_t i = 1; i < k; ++i)
        if (sorted[i] == sorted[i - 1]) {
            free(sorted);
            return ORC_E_DUPLICATE_POSITION;
        }
    free(sorted);

    uint32_t r = root_n(n, 0);
    uint32_t* xs = (uint32_t*)malloc(sizeof(uint32_t) * k);
    for (uint32_t i = 0; i < k; ++i) xs[i] = orc_pow(r, positions[i]);
    int rc = orc_subproduct_root(xs, k, a_out);
    free(xs);
    if (rc) return rc;

    uint32_t* ap = (uint32_t*)calloc(n, sizeof(uint32_t));
    orc_derivative(a_out, k + 1, ap);
    orc_fnt_forward(n, ap, ap);
    for (uint32_t i = 0; i < k; ++i) aprime_inv[i] = orc_inv(ap[positions[i]]);
    free(ap);

    uint32_t plen = 2 * k;
    if (plen <= 65536) {
        uint32_t m = next_pow2(plen);
        *product_size = m;
        if (a_fnt) {
            memset(a_fnt, 0, sizeof(uint32_t) * m);
            memcpy(a_fnt, a_out, sizeof(uint32_t) * (k + 1 <= m ? k + 1 : m));
            dif_core(a_fnt, m, plan_for(m)->stage);
        }
    } else {
        *product_size = 0;
    }
    return ORC_OK;
}

/* mul_low (poly.cpp:139-169): the first `count` coefficients of a*b. When
 * the truncated product fits one transform it is one orc_poly_mul; otherwise
 * both operands split at h = ceil(count/2) and high*high (degrees >= 2h) is
 * dropped: out = lo*lo + x^h (mul_low(alo, bhi) + mul_low(ahi, blo)).
 * Writes exactly `count` coefficients (zero-padded). */
static int mul_low(const uint32_t* a, uint32_t la, const uint32_t* b, uint32_t lb, uint32_t count, uint32_t* out) {
    memset(out, 0, sizeof(uint32_t) * count);
    uint32_t at = la < count ? la : count, bt = lb < count ? lb : count;
    if (!at || !bt) return ORC_OK;
    uint32_t len = at + bt - 1;
    if (len <= 65536) {
        uint32_t* full = (uint32_t*)malloc(sizeof(uint32_t) * len);
        int rc = orc_poly_mul(a, at, b, bt, full);
        if (!rc) memcpy(out, full, sizeof(uint32_t) * (len < count ? len : count));
        free(full);
        return rc;
    }
    uint32_t h = (count + 1) / 2;
    uint32_t alo = at < h ? at : h, blo = bt < h ? bt : h;
    uint32_t* lo = (uint32_t*)malloc(sizeof(uint32_t) * (alo + blo - 1));
    int rc = orc_poly_mul(a, alo, b, blo, lo);
    if (!rc) {
        uint32_t ll = alo + blo - 1;
        memcpy(out, lo, sizeof(uint32_t) * (ll < count ? ll : count));
    }
    free(lo);
    uint32_t rest = count - h;
    uint32_t* c1 = (uint32_t*)calloc(rest ? rest : 1, sizeof(uint32_t));
    uint32_t* c2 = (uint32_t*)calloc(rest ? rest : 1, sizeof(uint32_t));
    if (!rc && rest) rc = mul_low(a, alo, b + blo, bt - blo, rest, c1);
    if (!rc && rest) rc = mul_low(a + alo, at - alo, b, blo, rest, c2);
    for (uint32_t j = 0; !rc && j < rest; ++j) out[h + j] = orc_add(out[h + j], orc_add(c1[j], c2[j]));
    free(c1);
    free(c2);
    return rc;
}

/* interpolate (interp.cpp:103-137), steps 4-6, for a plan built by
 * orc_build_plan. Writes k coefficients (normalised then re-padded with
 * zeros to k, which is what codec::first_k_coeffs returns, codec.cpp:105-108).
 * Step 5 computes s_j = -N'(r^-(j+1)) as -fnt_forward(N')[n-1-j]
 * (geom_eval_negative visits the forward points in reverse order,
 * test_geom.cpp:74-82). 2k > 65536 (product_size 0): orc_interpolate_low. */
static int interpolate_split(uint32_t n, uint32_t k, const uint32_t* positions, const uint32_t* aprime_inv,
                             const uint32_t* a, const uint32_t* values, uint32_t* out);

int orc_interpolate(uint32_t n, uint32_t k, const uint32_t* positions, const uint32_t* aprime_inv,
                    uint32_t product_size, const uint32_t* a_fnt, const uint32_t* values,
                    uint32_t* out) {
    if (!product_size) return ORC_E_PRODUCT_TOO_LARGE; /* needs A itself: orc_interpolate_low */
    uint32_t* np = (uint32_t*)calloc(n, sizeof(uint32_t));
    for (uint32_t i = 0; i < k; ++i) np[positions[i]] = orc_mul(values[i], aprime_inv[i]);
    orc_fnt_forward(n, np, np);
    uint32_t m = product_size;
    uint32_t* buf = (uint32_t*)calloc(m, sizeof(uint32_t));
    uint32_t take = k < n ? k : n;
    for (uint32_t j = 0; j < take; ++j) buf[j] = orc_neg(np[n - 1 - j]);
    free(np);
    const tplan* p = plan_for(m);
    dif_core(buf, m, p->stage);
    for (uint32_t i = 0; i < m; ++i) buf[i] = orc_mul(orc_mul(buf[i], a_fnt[i]), p->size_inv);
    dit_core(buf, m, p->stage_inv);
    memcpy(out, buf, sizeof(uint32_t) * k);
    free(buf);
    return ORC_OK;
}

/* interpolate step 6 when 2k > 65536 (interp.cpp:133-134): P = mul_low(A, S, k)
 * with A the locator's k+1 coefficients and S the truncated series. */
static int interpolate_split(uint32_t n, uint32_t k, const uint32_t* positions, const uint32_t* aprime_inv,
                             const uint32_t* a, const uint32_t* values, uint32_t* out) {
    uint32_t* np = (uint32_t*)calloc(n, sizeof(uint32_t));
    for (uint32_t i = 0; i < k; ++i) np[positions[i]] = orc_mul(values[i], aprime_inv[i]);
    orc_fnt_forward(n, np, np);
    uint32_t take = k < n ? k : n;
    uint32_t* series = (uint32_t*)calloc(k, sizeof(uint32_t));
    for (uint32_t j = 0; j < take; ++j) series[j] = orc_neg(np[n - 1 - j]);
    free(np);
    int rc = mul_low(a, k + 1, series, k, k, out);
    free(series);
    return rc;
}

int orc_interpolate_low(uint32_t n, uint32_t k, const uint32_t* positions, const uint32_t* aprime_inv,
                        const uint32_t* a, const uint32_t* values, uint32_t* out) {
    return interpolate_split(n, k, positions, aprime_inv, a, values, out);
}

/* lagrange_oracle (interp.cpp:139-171): quadratic interpolation through
 * (xs[i], vs[i]); writes k coefficients (zero-padded). */
int orc_lagrange(uint32_t k, const uint32_t* xs, const uint32_t* vs, uint32_t* out) {
    uint32_t* sorted = (uint32_t*)malloc(sizeof(uint32_t) * (k ? k : 1));
    memcpy(sorted, xs, sizeof(uint32_t) * k);
    qsort(sorted, k, sizeof(uint32_t), cmp_u32);
    for (uint32_t i = 1; i < k; ++i)
        if (sorted[i] == sorted[i - 1]) {
            free(sorted);
            return ORC_E_DUPLICATE_POINT;
        }
    free(sorted);
    if (!k) return ORC_OK;
    uint32_t* master = (uint32_t*)calloc(k + 1, sizeof(uint32_t));
    master[0] = 1;
    uint32_t deg = 0;
    for (uint32_t i = 0; i < k; ++i) { /* master *= (x - x_i) */
        uint32_t nx = orc_neg(xs[i]);
        for (uint32_t j = deg + 1; j-- > 0;) {
            uint32_t lower = j ? master[j - 1] : 0;
            master[j] = orc_add(orc_mul(master[j], nx), lower);
        }
        ++deg;
        master[deg] = 1;
    }
    uint32_t* numer = (uint32_t*)malloc(sizeof(uint32_t) * k);
    memset(out, 0, sizeof(uint32_t) * k);
    for (uint32_t i = 0; i < k; ++i) {
        uint32_t carry = master[k];
        for (uint32_t j = k; j-- > 0;) {
            numer[j] = carry;
            carry = orc_add(master[j], orc_mul(xs[i], carry));
        }
        uint32_t scale = orc_mul(vs[i], orc_inv(orc_eval_horner(numer, k, xs[i])));
        for (uint32_t j = 0; j < k; ++j) out[j] = orc_add(out[j], orc_mul(numer[j], scale));
    }
    free(master);
    free(numer);
    return ORC_OK;
}

/* ---- codec: proj/src/codec.cpp ----------------------------------------- */

int orc_code_params(uint32_t k, uint32_t n, uint32_t* n_domain) { /* codec.cpp:112-122 */
    if (k < 1 || k > n || n > 65536) return ORC_E_SIZE_MISMATCH;
    *n_domain = next_pow2(n);
    return ORC_OK;
}

/* encode_nonsystematic (codec.cpp:124-131): zero-pad to n_domain, one
 * forward transform, keep the first n outputs. */
int orc_encode(uint32_t k, uint32_t n, const uint32_t* src, uint32_t* out) {
    uint32_t nd;
    int rc = orc_code_params(k, n, &nd);
    if (rc) return rc;
    uint32_t* buf = (uint32_t*)calloc(nd, sizeof(uint32_t));
    memcpy(buf, src, sizeof(uint32_t) * k);
    orc_fnt_forward(nd, buf, buf);
    memcpy(out, buf, sizeof(uint32_t) * n);
    free(buf);
    return ORC_OK;
}

typedef struct { uint32_t pos, val; } sym_t;

static int cmp_sym(const void* a, const void* b) {
    uint32_t x = ((const sym_t*)a)->pos, y = ((const sym_t*)b)->pos;
    return x < y ? -1 : x > y;
}

/* decode_nonsystematic (codec.cpp:133-149) with sorted_received
 * (codec.cpp:32-48): validate, sort by position, full-reception shortcut,
 * else interpolate through the k lowest positions. Path is irrelevant to the
 * output (Lagrange and the fast path agree bit for bit, test_codec.cpp:249+),
 * so the oracle always runs the transform path. */
int orc_decode(uint32_t k, uint32_t n, uint32_t count, const uint32_t* pos, const uint32_t* val,
               uint32_t* out) {
    uint32_t nd;
    int rc = orc_code_params(k, n, &nd);
    if (rc) return rc;
    for (uint32_t i = 0; i < count; ++i)
        if (pos[i] >= n) return ORC_E_POSITION_OUT_OF_RANGE;
    sym_t* s = (sym_t*)malloc(sizeof(sym_t) * (count ? count : 1));
    for (uint32_t i = 0; i < count; ++i) {
        s[i].pos = pos[i];
        s[i].val = val[i];
    }
    qsort(s, count, sizeof(sym_t), cmp_sym); /* positions distinct after the check below */
    for (uint32_t i = 1; i < count; ++i)
        if (s[i].pos == s[i - 1].pos) {
            free(s);
            return ORC_E_DUPLICATE_POSITION;
        }
    if (count < k) {
        free(s);
        return ORC_E_NOT_ENOUGH_SYMBOLS;
    }
    if (n == nd && count == n) { /* codec.cpp:137-144 */
        uint32_t* v = (uint32_t*)malloc(sizeof(uint32_t) * n);
        for (uint32_t i = 0; i < n; ++i) v[i] = s[i].val;
        orc_fnt_inverse(n, v, v);
        memcpy(out, v, sizeof(uint32_t) * k);
        free(v);
        free(s);
        return ORC_OK;
    }
    uint32_t* zp = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t* vs = (uint32_t*)malloc(sizeof(uint32_t) * k);
    for (uint32_t i = 0; i < k; ++i) {
        zp[i] = s[i].pos;
        vs[i] = s[i].val;
    }
    free(s);
    uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * (k + 1));
    uint32_t* ainv = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t psize = 0;
    rc = orc_build_plan(nd, k, zp, a, ainv, &psize, NULL);
    if (!rc) {
        uint32_t* afnt = (uint32_t*)calloc(psize ? psize : 1, sizeof(uint32_t));
        if (psize) {
            memcpy(afnt, a, sizeof(uint32_t) * (k + 1));
            dif_core(afnt, psize, plan_for(psize)->stage);
        }
        rc = psize ? orc_interpolate(nd, k, zp, ainv, psize, afnt, vs, out)
                   : orc_interpolate_low(nd, k, zp, ainv, a, vs, out); /* 2k > 65536: mul_low */
        free(afnt);
    }
    free(a); free(ainv); free(zp); free(vs);
    return rc;
}

/* ---- systematic codec: proj/src/codec.cpp:151-196 ---------------------------
 * encode: P = interpolate(positions 0..k-1, source) (codec.cpp:156-159), then
 * transform_of_padded(P, n_domain, n) (codec.cpp:75-82): symbols 0..k-1 of the
 * result are the source itself. */
int orc_encode_systematic(uint32_t k, uint32_t n, const uint32_t* src, uint32_t* out) {
    uint32_t nd;
    int rc = orc_code_params(k, n, &nd);
    if (rc) return rc;
    uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t* buf = (uint32_t*)calloc(nd, sizeof(uint32_t));
    for (uint32_t i = 0; i < k; ++i) pos[i] = i;
    rc = orc_decode(k, n, k, pos, src, buf); /* the unique degree < k interpolant */
    if (!rc) {
        orc_fnt_forward(nd, buf, buf);
        memcpy(out, buf, sizeof(uint32_t) * n);
    }
    free(pos);
    free(buf);
    return rc;
}

/* decode (codec.cpp:163-196): validate and sort like sorted_received; when the
 * k lowest received positions are exactly 0..k-1 the values are the source
 * (systematic_prefix_present, codec.cpp:51-55,167-171); otherwise interpolate
 * the k lowest (interpolate_selected, codec.cpp:85-94) and evaluate the
 * interpolant at r^0..r^(k-1) (transform_of_padded(P, n_domain, k)). */
int orc_decode_systematic(uint32_t k, uint32_t n, uint32_t count, const uint32_t* pos, const uint32_t* val,
                          uint32_t* out) {
    uint32_t nd;
    int rc = orc_code_params(k, n, &nd);
    if (rc) return rc;
    for (uint32_t i = 0; i < count; ++i)
        if (pos[i] >= n) return ORC_E_POSITION_OUT_OF_RANGE;
    sym_t* s = (sym_t*)malloc(sizeof(sym_t) * (count ? count : 1));
    for (uint32_t i = 0; i < count; ++i) {
        s[i].pos = pos[i];
        s[i].val = val[i];
    }
    qsort(s, count, sizeof(sym_t), cmp_sym);
    for (uint32_t i = 1; i < count; ++i)
        if (s[i].pos == s[i - 1].pos) {
            free(s);
            return ORC_E_DUPLICATE_POSITION;
        }
    if (count < k) {
        free(s);
        return ORC_E_NOT_ENOUGH_SYMBOLS;
    }
    int prefix = 1;
    for (uint32_t i = 0; i < k; ++i)
        if (s[i].pos != i) prefix = 0;
    if (prefix) {
        for (uint32_t i = 0; i < k; ++i) out[i] = s[i].val;
        free(s);
        return ORC_OK;
    }
    uint32_t* zp = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t* vs = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t* buf = (uint32_t*)calloc(nd, sizeof(uint32_t));
    for (uint32_t i = 0; i < k; ++i) {
        zp[i] = s[i].pos;
        vs[i] = s[i].val;
    }
    free(s);
    rc = orc_decode(k, n, k, zp, vs, buf);
    if (!rc) {
        orc_fnt_forward(nd, buf, buf);
        memcpy(out, buf, sizeof(uint32_t) * k);
    }
    free(zp);
    free(vs);
    free(buf);
    return rc;
}

/* ---- shardio escape rule: proj/src/shardio.cpp:131-137,153-154,203-208 -
 * 65536 is written as 0x0000 and its index appended (ascending) to the
 * escape list; reading restores 65536 at the listed indices. Returns the
 * escape count, or -1 when a value is outside the field. */
int64_t orc_escape_split(const uint32_t* v, uint64_t count, uint16_t* words, uint32_t* esc) {
    int64_t ne = 0;
    for (uint64_t i = 0; i < count; ++i) {
        if (v[i] > 65536) return -1;
        if (v[i] == 65536) {
            esc[ne++] = (uint32_t)i;
            words[i] = 0;
        } else {
            words[i] = (uint16_t)v[i];
        }
    }
    return ne;
}

void orc_escape_join(const uint16_t* words, uint64_t count, const uint32_t* esc, uint64_t ne,
                     uint32_t* v) {
    for (uint64_t i = 0; i < count; ++i) v[i] = words[i];
    for (uint64_t e = 0; e < ne; ++e) v[esc[e]] = 65536;
}

/* ---- batched stripe harness (the CLI's loop, tools/fntrs_main.cpp:122-139,
 * 222-231): packet-major uint16 stripes, codeword j = symbol j of every
 * packet. Escapes are ascending symbol indices row * L + col, row =
 * stripe * rows_per_stripe + packet -- the same convention as the C-ABI. */

static uint32_t fetch(const uint16_t* base, const uint64_t* esc, uint64_t ne, uint64_t row,
                      uint32_t col, uint32_t L) {
    uint16_t w = base[row * L + col];
    if (w || !ne) return w;
    uint64_t key = row * L + col, lo = 0, hi = ne;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (esc[mid] < key) lo = mid + 1; else hi = mid;
    }
    return (lo < ne && esc[lo] == key) ? 65536u : 0u;
}

/* Returns number of escapes written (sorted), or a negative error. */
int64_t orc_encode_stripes(uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                           const uint16_t* src, const uint64_t* src_esc, uint64_t n_src_esc,
                           uint16_t* out, uint64_t* out_esc, uint64_t esc_cap) {
    uint32_t nd;
    if (orc_code_params(k, n, &nd)) return -ORC_E_SIZE_MISMATCH;
    uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t* e = (uint32_t*)malloc(sizeof(uint32_t) * n);
    int64_t ne = 0;
    for (uint32_t s = 0; s < stripes; ++s) {
        for (uint32_t j = 0; j < L; ++j) {
            for (uint32_t i = 0; i < k; ++i)
                a[i] = fetch(src, src_esc, n_src_esc, (uint64_t)s * k + i, j, L);
            orc_encode(k, n, a, e);
            for (uint32_t i = 0; i < n; ++i) {
                uint64_t row = (uint64_t)s * n + i;
                out[row * L + j] = e[i] == 65536 ? 0 : (uint16_t)e[i];
                if (e[i] == 65536) {
                    if ((uint64_t)ne >= esc_cap) { free(a); free(e); return -ORC_E_TOO_MANY_ESCAPES; }
                    out_esc[ne++] = row * L + j;
                }
            }
        }
    }
    free(a);
    free(e);
    qsort(out_esc, (size_t)ne, sizeof(uint64_t), cmp_u64);
    return ne;
}

/* Decode every stripe from its k received packets. patterns[p*k .. p*k+k)
 * holds pattern p's positions, strictly ascending; stripe s uses pattern
 * stripe_pattern[s], and rx row (s*k + i) carries the packet received at
 * position patterns[stripe_pattern[s]*k + i]. Output rows are s*k + i
 * (source packets). Returns the escape count or a negative error. */
int64_t orc_decode_stripes(uint32_t k, uint32_t n, uint32_t stripes, uint32_t L,
                           uint32_t npatterns, const uint32_t* patterns,
                           const uint32_t* stripe_pattern, const uint16_t* rx,
                           const uint64_t* rx_esc, uint64_t n_rx_esc, uint16_t* out,
                           uint64_t* out_esc, uint64_t esc_cap) {
    uint32_t nd;
    if (orc_code_params(k, n, &nd)) return -ORC_E_SIZE_MISMATCH;
    uint32_t* pos = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t* val = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint32_t* dec = (uint32_t*)malloc(sizeof(uint32_t) * k);
    int64_t ne = 0;
    int rc = 0;
    for (uint32_t s = 0; s < stripes && !rc; ++s) {
        uint32_t pidx = stripe_pattern[s];
        if (pidx >= npatterns) { rc = ORC_E_ERROR; break; }
        memcpy(pos, patterns + (uint64_t)pidx * k, sizeof(uint32_t) * k);
        for (uint32_t j = 0; j < L && !rc; ++j) {
            for (uint32_t i = 0; i < k; ++i)
                val[i] = fetch(rx, rx_esc, n_rx_esc, (uint64_t)s * k + i, j, L);
            rc = orc_decode(k, n, k, pos, val, dec);
            if (rc) break;
            for (uint32_t i = 0; i < k; ++i) {
                uint64_t row = (uint64_t)s * k + i;
                out[row * L + j] = dec[i] == 65536 ? 0 : (uint16_t)dec[i];
                if (dec[i] == 65536) {
                    if ((uint64_t)ne >= esc_cap) { rc = ORC_E_TOO_MANY_ESCAPES; break; }
                    out_esc[ne++] = row * L + j;
                }
            }
        }
    }
    free(pos); free(val); free(dec);
    if (rc) return -rc;
    qsort(out_esc, (size_t)ne, sizeof(uint64_t), cmp_u64);
    return ne;
}
