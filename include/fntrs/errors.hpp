// fntrs/errors.hpp -- exception classes of the drop-in API.
//
// Same class names and hierarchy as the reference
// (/root/reference/proj/include/fntrs/errors.hpp:9-38): one base `Error`
// (a std::runtime_error) and final subclasses. The numeric fntrs_status of
// the C ABI (include/fntrs_gpu.h) maps 1:1 onto them; see throw_status().
#pragma once

#include <stdexcept>
#include <string>

namespace fntrs {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define FNTRS_DECLARE_ERROR(Name) \
    struct Name final : Error {   \
        using Error::Error;       \
    }

FNTRS_DECLARE_ERROR(ZeroInverse);           // status 2
FNTRS_DECLARE_ERROR(InvalidTransformSize);  // 3
FNTRS_DECLARE_ERROR(SizeMismatch);          // 4
FNTRS_DECLARE_ERROR(ProductTooLarge);       // 5
FNTRS_DECLARE_ERROR(DuplicatePoint);        // 6
FNTRS_DECLARE_ERROR(DuplicatePosition);     // 7
FNTRS_DECLARE_ERROR(PositionOutOfRange);    // 8
FNTRS_DECLARE_ERROR(TooFewPositions);       // 9
FNTRS_DECLARE_ERROR(NotEnoughSymbols);      // 10
FNTRS_DECLARE_ERROR(TooManyEscapes);        // 11
FNTRS_DECLARE_ERROR(BadMagic);              // 12
FNTRS_DECLARE_ERROR(BadVersion);            // 13
FNTRS_DECLARE_ERROR(TruncatedShard);        // 14
FNTRS_DECLARE_ERROR(MalformedEscapes);      // 15
FNTRS_DECLARE_ERROR(MalformedHeader);       // 16
FNTRS_DECLARE_ERROR(LengthMismatch);        // 17
FNTRS_DECLARE_ERROR(NotEnoughShards);       // 18

#undef FNTRS_DECLARE_ERROR

// Throws the class matching a C-ABI status (no-op for 0). Statuses without a
// reference counterpart (CUDA failure, unsupported shape, bad argument) throw
// the base Error with the message.
[[noreturn]] void throw_status(int status, const std::string& message);

}  // namespace fntrs
