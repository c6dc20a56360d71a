#include "capi_common.h"

namespace vdnncapi {
namespace {
thread_local std::string g_error;
}
void set_error(const std::string& msg) { g_error = msg; }
void clear_error() { g_error.clear(); }
vdnn_status fail(vdnn_status st, const std::string& msg) {
  g_error = msg;
  return st;
}
const char* error_cstr() { return g_error.c_str(); }
}  // namespace vdnncapi

extern "C" const char* vdnn_last_error(void) { return vdnncapi::error_cstr(); }
extern "C" const char* vdnn_version(void) { return "vdnn-b200 0.1 (sm_100a)"; }
