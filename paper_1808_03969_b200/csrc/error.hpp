// error.hpp -- host-side error type shared by the CUDA and C++ translation units.
#pragma once
#include <stdexcept>
#include <string>

namespace rii {
// status uses the numeric values of rii_status (include/rii.h).
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string &m) : std::runtime_error(m), status(s) {}
};
}  // namespace rii
