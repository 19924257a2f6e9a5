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

inline mt_status check_launch(const char* what) {
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
