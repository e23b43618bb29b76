// coljoin error taxonomy — the exception classes of the reference operator API
// (reference: include/coljoin/errors.hpp:8-31).  Every C-ABI status code 1..15
// (include/cj_api.h) is rethrown as the class of the same name by the host
// library.
#pragma once

#include <stdexcept>
#include <string>

namespace coljoin {

struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
  explicit Error(const char* what) : std::runtime_error(what) {}
};

struct LengthMismatch : Error { using Error::Error; };       // status 1
struct KindError : Error { using Error::Error; };            // status 2
struct FanoutTooLarge : Error { using Error::Error; };       // status 3
struct IndexOutOfBounds : Error { using Error::Error; };     // status 4
struct EmptyInput : Error { using Error::Error; };           // status 5
struct NotSorted : Error { using Error::Error; };            // status 6
struct DuplicateBuildKeys : Error { using Error::Error; };   // status 7
struct FanoutMismatch : Error { using Error::Error; };       // status 8
struct CapacityExceeded : Error { using Error::Error; };     // status 9
struct TransformMismatch : Error { using Error::Error; };    // status 10
struct PhaseOrderViolation : Error { using Error::Error; };  // status 11
struct SpecInvalid : Error { using Error::Error; };          // status 12
struct UnknownShape : Error { using Error::Error; };         // status 13
struct SchemaError : Error { using Error::Error; };          // status 14
struct Unsupported : Error { using Error::Error; };          // status 15

// Device-side failures with no reference counterpart (CUDA/NCCL errors, device
// out of memory) derive from Error as well so callers that catch Error see them.
struct DeviceError : Error { using Error::Error; };

}  // namespace coljoin
