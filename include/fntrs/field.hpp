// fntrs/field.hpp -- GF(65537) element type and scalar helpers of the drop-in API.
//
// Mirrors the reference's public field interface
// (/root/reference/proj/include/fntrs/field.hpp:9-63): Fe is a uint32 holding
// a canonical value 0..65536 (17 bits), and gf:: provides the scalar
// operations with the same names and results. These are host conveniences
// for callers; the codec arithmetic itself runs in the CUDA kernels.
#pragma once

#include <cstdint>

#include "fntrs/errors.hpp"

namespace fntrs {

using Fe = std::uint32_t;

namespace gf {

inline constexpr Fe prime = 65537;
inline constexpr Fe generator = 3;

constexpr Fe add(Fe a, Fe b) noexcept { return (a + b) % prime; }
constexpr Fe sub(Fe a, Fe b) noexcept { return (a + prime - b) % prime; }
constexpr Fe neg(Fe a) noexcept { return (prime - a) % prime; }
constexpr Fe mul(Fe a, Fe b) noexcept {
    return static_cast<Fe>((static_cast<std::uint64_t>(a) * b) % prime);
}

constexpr Fe pow(Fe base, std::uint64_t exp) {
    if (exp == 0 && base == 0) throw Error("gf::pow: 0^0 is undefined");
    Fe acc = 1;
    for (Fe sq = base; exp; exp >>= 1, sq = mul(sq, sq))
        if (exp & 1u) acc = mul(acc, sq);
    return acc;
}

constexpr Fe inv(Fe a) {
    if (a % prime == 0) throw ZeroInverse("gf::inv: zero has no inverse");
    return pow(a, prime - 2);
}

constexpr Fe root_of_unity(std::uint32_t n, bool inverse = false) {
    const bool pow2 = n != 0 && (n & (n - 1)) == 0;
    if (!pow2 || n > 65536)
        throw InvalidTransformSize("gf::root_of_unity: size must be a power of two in [1, 65536]");
    const Fe r = pow(generator, 65536u / n);
    return inverse ? inv(r) : r;
}

}  // namespace gf
}  // namespace fntrs
