// fntrs/geom.hpp -- the reference's evaluation at geometric points
// (/root/reference/proj/include/fntrs/geom.hpp; proj/src/geom.cpp): the chirp
// (Bluestein) evaluation a(root^i), i < n, for any root, by a size-2n cyclic
// convolution, and the transform itself on the full 65536-point domain.
// Computed on the device (fntrs_gpu_chirp_table / fntrs_gpu_geom_eval /
// fntrs_gpu_geom_eval_negative). The batched decoder does not use it: its
// step 5 is the transform identity geom_eval_negative(a, n, r)[j] =
// FNT_n(a)[n-1-j] (DESIGN 4.2).
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "fntrs/field.hpp"

namespace fntrs::geom {

struct ChirpTable {
    std::uint32_t n = 0;
    Fe root = 1;
    bool full_domain = false;   // n = 65536: evaluation is the transform itself
    std::vector<Fe> b;          // 2n-1 entries, b_i = root^(i(i-1)/2)
    std::vector<Fe> b_inverse;  // n entries, 1/b_i
    std::vector<Fe> b_fnt;      // forward spectrum of b at size 2n (dif_forward order: bit-reversed)
};

// Throws InvalidTransformSize unless n is a power of two in [1, 65536].
ChirpTable build_chirp(std::uint32_t n, Fe root);

// Cached per (n, root).
std::shared_ptr<const ChirpTable> chirp_for(std::uint32_t n, Fe root);

// a(root^i) for i < n (SizeMismatch when a has more than n coefficients).
std::vector<Fe> geom_eval(std::span<const Fe> a, const ChirpTable& table);

// a(root^-(j+1)) for j < n.
std::vector<Fe> geom_eval_negative(std::span<const Fe> a, std::uint32_t n, Fe root);

}  // namespace fntrs::geom
