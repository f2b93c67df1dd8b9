// errors.h -- typed error carried from the engine to the C ABI (product code).
#pragma once
#include <stdexcept>
#include <string>

#include "../../include/petra.h"

namespace petra {
struct PetraError : std::runtime_error {
  petra_status status;
  PetraError(petra_status s, const std::string &m) : std::runtime_error(m), status(s) {}
};
}  // namespace petra
