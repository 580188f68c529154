// Error hierarchy of the B200 engine's C++ API — the same classes the reference throws
// (/root/reference/proj/include/flexquant/error.hpp:10-49), so callers' catch clauses and the
// reference's CHECK_THROWS_AS tests keep working.  C-ABI status codes are converted here.
#pragma once

#include <stdexcept>
#include <string>

#include "fq_cuda.h"

namespace flexquant {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DimensionError : Error { using Error::Error; };  // shape / axis mismatch
struct ConfigError : Error { using Error::Error; };     // unsupported option, plan/model mismatch
struct InputError : Error { using Error::Error; };      // bad payload: token id, empty input, ...
struct StateError : Error { using Error::Error; };      // object in the wrong state
struct FormatError : Error { using Error::Error; };     // malformed file / record
struct CapacityError : Error { using Error::Error; };   // sequence / cache capacity exhausted
struct DeviceError : Error { using Error::Error; };     // CUDA failure (no reference analogue)

namespace detail {
// Rethrows a failed C-ABI call as the matching flexquant exception.
[[noreturn]] void throw_status(fq_status st);
inline void check(fq_status st) {
  if (st != FQ_OK) throw_status(st);
}
}  // namespace detail

}  // namespace flexquant
