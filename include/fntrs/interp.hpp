// fntrs/interp.hpp -- the reference's plan-level decode API
// (/root/reference/proj/include/fntrs/interp.hpp:12-56) over the C ABI's
// GPU plans (fntrs_gpu_plans_create / _export / fntrs_gpu_decode).
//
// DecodePlan holds the reference's fields, copied back from the device:
// 1/A'(x_i), product size and the bit-reversed a_fnt from the GPU plan (whose
// locator comes from a log-domain convolution, DESIGN 4.4), and a_tree, the
// subproduct tree of the plan's points built level by level on the device
// (fntrs_gpu_subproduct_tree) so callers that walk the tree see the
// reference's levels. lagrange_oracle is the reference's quadratic
// cross-check, also on the device (fntrs_gpu_lagrange).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <utility>
#include <vector>

#include "fntrs/field.hpp"
#include "fntrs/poly.hpp"

namespace fntrs::interp {

struct DecodePlan {
    std::uint32_t n = 0;                   // domain size, power of two
    std::uint32_t k = 0;
    std::vector<std::uint32_t> positions;  // z_i in the order values must follow
    poly::SubproductTree a_tree;           // leaves (x - x_i); root A = prod (x - r^(z_i)), degree k
    std::vector<Fe> aprime_at_x_inv;       // 1/A'(x_i), aligned with positions
    std::uint32_t product_size = 0;        // next power of two >= 2k; 0 when 2k > 65536
    std::vector<Fe> a_fnt;                 // dif_forward(A padded to product_size): bit-reversed
    std::shared_ptr<const void> device;    // the GPU plan interpolate() runs with

    const poly::Poly& a() const { return a_tree.root(); }
};

// positions distinct and < n. Throws TooFewPositions, PositionOutOfRange,
// DuplicatePosition, InvalidTransformSize.
DecodePlan build_plan(std::uint32_t n, std::span<const std::uint32_t> positions);

// 16-entry LRU keyed by (n, position set); the cached plan's positions are
// ascending -- align values accordingly.
std::shared_ptr<const DecodePlan> plan_for(std::uint32_t n, std::span<const std::uint32_t> positions);

// The unique P with deg P < k and P(r^(z_i)) = values[i] (normalised: no
// trailing zero coefficients). values.size() must equal plan.k (SizeMismatch).
poly::Poly interpolate(const DecodePlan& plan, std::span<const Fe> values);

// The interpolating polynomial of arbitrary (x, value) points by Lagrange's
// formula, O(k^2) (the reference's cross-check). Throws DuplicatePoint.
poly::Poly lagrange_oracle(std::span<const std::pair<Fe, Fe>> points);

}  // namespace fntrs::interp
