// fntrs/poly.hpp -- the reference's polynomial API
// (/root/reference/proj/include/fntrs/poly.hpp:9-61) over the device kernels of
// paper_0907_1788_b200/csrc/poly_aux.cu (fntrs_gpu_poly_products,
// fntrs_gpu_subproduct_tree, fntrs_gpu_poly_derivative, fntrs_gpu_poly_eval).
//
// The batched decoder never multiplies polynomials (the locator comes from a
// log-domain convolution, DESIGN 4.4); this API serves callers of the
// reference's poly layer and DecodePlan::a_tree. All product tiers give the
// same exact product (one device product kernel); the ones the reference
// bounds by the transform size (mul, mul_fnt) keep its ProductTooLarge limit.
#pragma once

#include <cstddef>
#include <span>
#include <vector>

#include "fntrs/field.hpp"

namespace fntrs::poly {

using Poly = std::vector<Fe>;  // coefficient i of x^i; canonical: no trailing zeros

void normalize(Poly& p);  // strip trailing zero coefficients

inline long degree(const Poly& p) { return static_cast<long>(p.size()) - 1; }

struct MulTuning {
    std::size_t schoolbook_below = 32;
    std::size_t karatsuba_below = 64;
};

Poly mul_schoolbook(std::span<const Fe> a, std::span<const Fe> b);
Poly mul_karatsuba(std::span<const Fe> a, std::span<const Fe> b);
Poly mul_fnt(std::span<const Fe> a, std::span<const Fe> b);  // ProductTooLarge past 65536 coefficients
Poly mul(std::span<const Fe> a, std::span<const Fe> b, const MulTuning& tuning = {});

// first `count` coefficients of a * b (count <= 65536)
Poly mul_low(std::span<const Fe> a, std::span<const Fe> b, std::size_t count, const MulTuning& tuning = {});

// coefficients n-1 .. 2n-2 of a * b with |a| = n (a power of two), |b| = 2n - 1
std::vector<Fe> middle_product(std::span<const Fe> a, std::span<const Fe> b);

Poly derivative(std::span<const Fe> a);  // i * a_i, i reduced mod p

Fe eval_horner(std::span<const Fe> a, Fe x);

// levels[0] = leaves (x - x_j); each level pairs adjacent nodes, an odd last
// node carried up unchanged; levels.back()[0] = prod (x - x_j), degree k
struct SubproductTree {
    std::vector<std::vector<Poly>> levels;

    const Poly& root() const { return levels.back().front(); }
};

// Throws Error on no points and DuplicatePoint on a repeated point.
SubproductTree build_subproduct_tree(std::span<const Fe> points);

}  // namespace fntrs::poly
