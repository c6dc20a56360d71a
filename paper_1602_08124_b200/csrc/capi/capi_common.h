// Shared helpers for the extern "C" layer: thread-local error text and
// exception -> vdnn_status translation.
#pragma once
#include <string>

#include "../../../include/vdnn.h"

namespace vdnncapi {
void set_error(const std::string& msg);
void clear_error();
vdnn_status fail(vdnn_status st, const std::string& msg);
const char* error_cstr();
}  // namespace vdnncapi
