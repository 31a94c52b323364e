// Host-side helpers shared by the C-ABI translation units: thread-local
// error message, status propagation, launch accounting.
#pragma once

#include <cuda_runtime.h>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/ulysses_b200.h"

namespace ul {

// thread-local last-error text (ul_last_error)
std::string& last_error();
int& launch_count();
void count_launch();

inline int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return code;
}

inline int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return UL_OK;
  return fail(UL_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define UL_TRY(expr)                 \
  do {                               \
    int _st = (expr);                \
    if (_st != UL_OK) return _st;    \
  } while (0)

#define UL_CUDA(expr) UL_TRY(::ul::cuda_check((expr), #expr))

// after a <<<>>> launch
inline int launched(const char* name) {
  ++launch_count();
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(UL_ERR_CUDA, "launch %s: %s", name, cudaGetErrorString(e));
  return UL_OK;
}

inline size_t dtype_size(int dtype) { return dtype == UL_DTYPE_F32 ? 4 : 2; }

inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace ul
