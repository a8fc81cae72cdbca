// eig33_internal.h -- symbols shared between the translation units of _eig33cuda.so.
#pragma once
#include <string>

namespace eig33b {
// Thread-local last-error text returned by eig33cu_last_error().
void set_error(const std::string& message);
}  // namespace eig33b
