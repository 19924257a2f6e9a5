// capi.cu — error reporting for the C ABI (include/mtsa.h).
#include "common.cuh"

namespace mt {
static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
}  // namespace mt

extern "C" const char* mt_last_error(void) { return mt::g_last_error.c_str(); }
