// common.cuh — host-side status/error plumbing shared by the C-ABI entry points.
#pragma once
#include <cstdio>
#include <cstdarg>
#include <string>
#include <cuda_runtime.h>
#include "../../include/mtsa.h"

namespace mt {

void set_error(const char* fmt, ...);

inline mt_status fail(mt_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return s;
}

// Process-wide counters of the library's own kernel launches and of the CUB sort calls
// (library kernels) it makes, read by mt_launch_count / mt_library_call_count (bench.py's
// gpu_launches).  check_launch counts one launch; sites that enqueue several kernels
// before checking add the rest with count_launches.
void count_launches(int n);
void count_library_calls(int n);

inline mt_status check_launch(const char* what) {
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return MT_OK;
}

}  // namespace mt

#define MT_TRY(expr)                    \
  do {                                  \
    mt_status _s = (expr);              \
    if (_s != MT_OK) return _s;         \
  } while (0)
