// capi.cu — error reporting and launch counters for the C ABI (include/mtsa.h).
#include <atomic>

#include "common.cuh"

namespace mt {
static std::atomic<unsigned long long> g_launches{0}, g_library_calls{0};
void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
void count_library_calls(int n) {
  g_library_calls.fetch_add((unsigned long long)n, std::memory_order_relaxed);
}
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

extern "C" unsigned long long mt_launch_count(void) { return mt::g_launches.load(); }
extern "C" unsigned long long mt_library_call_count(void) { return mt::g_library_calls.load(); }
