// fntrs/interp.hpp -- the reference's plan-level decode API
// (/root/reference/proj/include/fntrs/interp.hpp:12-56) over the C ABI's
// GPU plans (fntrs_gpu_plans_create / _export / fntrs_gpu_decode).
//
// DecodePlan holds the reference's fields, copied back from the device plan
// (locator coefficients, 1/A'(x_i), product size and the bit-reversed a_fnt),
// plus the device plan itself for interpolate(). The locator comes from the
// GPU's log-domain / direct-product construction, not a subproduct tree, so
// the reference's a_tree member is replaced by the coefficient vector that
// a() returns. lagrange_oracle (the reference's quadratic cross-check on
// arbitrary points) is not provided.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "fntrs/field.hpp"

namespace fntrs::poly {
using Poly = std::vector<Fe>;  // coefficient i of x^i, trailing zeros trimmed
}  // namespace fntrs::poly

namespace fntrs::interp {

struct DecodePlan {
    std::uint32_t n = 0;                   // domain size, power of two
    std::uint32_t k = 0;
    std::vector<std::uint32_t> positions;  // z_i in the order values must follow
    poly::Poly a_coeffs;                   // A = prod (x - r^(z_i)), monic, k + 1 coefficients
    std::vector<Fe> aprime_at_x_inv;       // 1/A'(x_i), aligned with positions
    std::uint32_t product_size = 0;        // next power of two >= 2k; 0 when 2k > 65536
    std::vector<Fe> a_fnt;                 // dif_forward(A padded to product_size): bit-reversed
    std::shared_ptr<const void> device;    // the GPU plan interpolate() runs with

    const poly::Poly& a() const { return a_coeffs; }
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

}  // namespace fntrs::interp
