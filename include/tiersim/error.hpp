// tiersim/error.hpp — exception hierarchy of the reference API (core/include/tiersim/error.hpp:13-71),
// plus the mapping from libtsb status codes to those classes.
#pragma once

#include <stdexcept>
#include <string>
#include <utility>

#include "tsb_capi.h"

namespace tiersim {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ValidationError : public Error {
 public:
  using Error::Error;
};
class DegenerateFit : public Error {
 public:
  using Error::Error;
};
class MissingDeadline : public Error {
 public:
  using Error::Error;
};
class CapacityError : public Error {
 public:
  using Error::Error;
};
class UnknownProfile : public Error {
 public:
  using Error::Error;
};
class ConfigError : public Error {
 public:
  ConfigError(std::string field, const std::string& message)
      : Error(field.empty() ? message : field + ": " + message), field_(std::move(field)) {}
  const std::string& field() const noexcept { return field_; }

 private:
  std::string field_;
};
class IncompleteTrace : public Error {
 public:
  using Error::Error;
};
class WindowTooLong : public Error {
 public:
  using Error::Error;
};
/// Device-side failure (CUDA error or an unsupported kernel shape) raised by the B200 path.
class DeviceError : public Error {
 public:
  using Error::Error;
};

/// Rethrows a libtsb status as the reference's exception class, message verbatim.
inline void check(tsb_status s) {
  switch (s) {
    case TSB_OK: return;
    case TSB_VALIDATION: throw ValidationError(tsb_last_error());
    case TSB_CAPACITY: throw CapacityError(tsb_last_error());
    case TSB_MISSING_DEADLINE: throw MissingDeadline(tsb_last_error());
    case TSB_DEGENERATE_FIT: throw DegenerateFit(tsb_last_error());
    case TSB_UNKNOWN_PROFILE: throw UnknownProfile(tsb_last_error());
    default: throw DeviceError(tsb_last_error());
  }
}

}  // namespace tiersim
