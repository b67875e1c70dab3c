// fntrs/codec.hpp -- drop-in replacement for the reference's non-systematic
// codec API (/root/reference/proj/include/fntrs/codec.hpp:15-51), executed on
// a B200 through the C ABI in include/fntrs_gpu.h (libfntrs_b200.so).
//
// Same namespace, types, signatures, error classes and results as the
// reference for CodeParams, Symbol, Codeword, Path, encode_nonsystematic and
// decode_nonsystematic. Each call is one codeword (a batch of 1) -- correct,
// not fast; throughput comes from the batched C ABI (fntrs_gpu_encode /
// fntrs_gpu_decode over stripes x codewords). There is no CPU fallback: a
// call without a usable CUDA device throws fntrs::Error.
//
// Also the systematic pair (codec.hpp:56-65 of the reference), through
// fntrs_gpu_encode_systematic / fntrs_gpu_decode_systematic, and the
// reference's quadratic cross-check names (same values, GPU transform path).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "fntrs/field.hpp"
#include "fntrs/instrument.hpp"

namespace fntrs::codec {

struct CodeParams {
    std::uint32_t k = 0;
    std::uint32_t n = 0;
    std::uint32_t n_domain = 0;  // least power of two >= n
    bool systematic = true;

    // Throws SizeMismatch unless 1 <= k <= n <= 65536.
    static CodeParams make(std::uint32_t k, std::uint32_t n, bool systematic = true);
};

struct Symbol {
    std::uint32_t position = 0;
    Fe value = 0;
    friend bool operator==(const Symbol&, const Symbol&) = default;
};

using Codeword = std::vector<Symbol>;

// Auto / Fast / Direct select the reference's CPU algorithms; every choice
// yields the same (unique) interpolating polynomial, and the GPU computes it
// with the transform path regardless.
enum class Path { Auto, Fast, Direct };

inline constexpr std::uint32_t direct_path_max_k = 256;

// Output j is s(r^j), j < n (zero-padded forward transform, punctured).
std::vector<Fe> encode_nonsystematic(const CodeParams& params, std::span<const Fe> source);

// The k source coefficients from any >= k received symbols (the k lowest
// positions are used; complete reception with n == n_domain inverts one
// transform). Throws NotEnoughSymbols, DuplicatePosition, PositionOutOfRange.
std::vector<Fe> decode_nonsystematic(const CodeParams& params, const Codeword& received,
                                     Path path = Path::Auto);

// Systematic: outputs 0..k-1 are the source, k..n-1 the parity (interpolate
// at positions 0..k-1, then the punctured forward transform).
std::vector<Fe> encode_systematic(const CodeParams& params, std::span<const Fe> source,
                                  Path path = Path::Auto);

// The k source symbols from any >= k received symbols of a systematic codeword
// (the k lowest positions are used). Same exceptions as decode_nonsystematic.
std::vector<Fe> decode_systematic(const CodeParams& params, const Codeword& received,
                                  Path path = Path::Auto);

// The reference's quadratic cross-check entry points (codec.hpp:66-75 there).
// They return exactly the values of their transform counterparts, which is
// what the GPU computes them with; the instrumentation (instrument.hpp)
// therefore records the transforms of that path, not the reference's
// "one transform" for encode_systematic_intermediate_direct.
std::vector<Fe> encode_systematic_direct(const CodeParams& params, std::span<const Fe> source);
std::vector<Fe> encode_systematic_intermediate_direct(const CodeParams& params, std::span<const Fe> source);
std::vector<Fe> decode_direct(const CodeParams& params, const Codeword& received);

}  // namespace fntrs::codec

namespace fntrs::gpu {
// Device used by the per-codeword API (default 0). Call before the first
// codec call; later calls switch the shared context.
void set_device(int device);
}  // namespace fntrs::gpu
