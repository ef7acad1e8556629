// Error slot and version for libLBX.
#include <cstdio>
#include <string>

#include "lbx_internal.h"

namespace lbx {
namespace {
thread_local std::string g_last_error;
}

int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

void clear_error() { g_last_error.clear(); }

}  // namespace lbx

extern "C" const char* lbx_last_error(void) { return lbx::g_last_error.c_str(); }

extern "C" const char* lbx_version(void) { return "libLBX 0.1 (sm_100a)"; }
