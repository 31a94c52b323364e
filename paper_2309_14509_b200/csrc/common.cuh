// Host-side helpers shared by the C-ABI translation units: thread-local
// error message, status propagation, launch accounting.
#pragma once

#include <cuda_runtime.h>
#include <atomic>
#include <mutex>
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

// SM count of the CURRENT device (cached per device: a process may drive
// several GPUs)
inline int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  dev &= 63;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// Dynamic shared-memory opt-in of `fn` on the CURRENT device.  The attribute
// is per device context, so it is tracked per (kernel, device) in one
// registry.  The preload functions opt every large-smem kernel in when a
// group is created: cudaFuncSetAttribute at a kernel's first launch could
// otherwise run while an in-process rank's flag wait is spinning on a peer
// the host has not issued yet (observed: the first layer call of a process
// deadlocked until the wait's timeout).
struct SmemOptIn {
  const void* fn = nullptr;
  std::atomic<uint64_t> mask{0};
};
inline std::atomic<uint64_t>& smem_mask(const void* fn) {
  static SmemOptIn table[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : table) {
    if (e.fn == fn) return e.mask;
    if (!e.fn) {
      e.fn = fn;
      return e.mask;
    }
  }
  return table[63].mask;   // (not reached: fewer than 64 kernels)
}
inline int smem_opt_in(const void* fn, int bytes) {
  int dev = 0;
  UL_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  std::atomic<uint64_t>& done = smem_mask(fn);
  if (done.load(std::memory_order_acquire) & bit) return UL_OK;
  UL_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.fetch_or(bit, std::memory_order_release);
  return UL_OK;
}

}  // namespace ul
