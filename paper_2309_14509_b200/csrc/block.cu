// The row-wise pieces of the Ulysses transformer block:
// ulysses_block_forward (ulysses.py:172-184) = pre-LN attention + residual,
// pre-LN GELU MLP + residual, with layernorm (layers.py:106-110) and exact
// erf GELU (layers.py:113-127).  All HBM-bound: one pass over the rows,
// 16-byte vector accesses, fp32 statistics; the residual add is fused into
// the layernorm that follows it (x1 = x + a; t = LN(x1) in one read of x, a).
//
//   ul_add_layernorm      s = x (+ r);  y = (s - mean) * rstd * gain + bias;  mean/rstd saved
//   ul_layernorm_bwd      dx = rstd * (g - mean(g) - xhat * mean(g * xhat)), g = dy * gain,
//                         dgain / dbias partial column sums per CTA (deterministic, no atomics)
//   ul_gelu / ul_gelu_bwd exact GELU 0.5 x (1 + erf(x / sqrt 2)) and its derivative
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace ul {
namespace blk {

constexpr int kThreads = 256;

template <typename T>
__device__ __forceinline__ float ld1(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ld1<float>(const float* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ float ld1<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
template <typename T>
__device__ __forceinline__ void st1(T* p, int64_t i, float v);
template <>
__device__ __forceinline__ void st1<float>(float* p, int64_t i, float v) { p[i] = v; }
template <>
__device__ __forceinline__ void st1<__nv_bfloat16>(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

// block-wide sum of two values (kThreads threads)
__device__ __forceinline__ float2 block_sum2(float a, float b, float2* red) {
#pragma unroll
  for (int m = 16; m; m >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, m);
    b += __shfl_xor_sync(0xffffffffu, b, m);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = make_float2(a, b);
  __syncthreads();
  if (w == 0) {
    float2 v = lane < kThreads / 32 ? red[lane] : make_float2(0.f, 0.f);
#pragma unroll
    for (int m = 16; m; m >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
    }
    if (lane == 0) red[kThreads / 32] = v;
  }
  __syncthreads();
  const float2 r = red[kThreads / 32];
  __syncthreads();
  return r;
}

// one CTA per row; the row (d <= kThreads * 16 elements) stays in registers
template <typename T>
__global__ void __launch_bounds__(kThreads) add_ln_kernel(const T* __restrict__ x, const T* __restrict__ r,
                                                          const T* __restrict__ gain, const T* __restrict__ bias,
                                                          T* __restrict__ s_out, T* __restrict__ y,
                                                          float2* __restrict__ stats, int d, float eps) {
  __shared__ float2 red[kThreads / 32 + 1];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * d;
  float v[16];
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c = threadIdx.x + k * kThreads;
    float a = 0.f;
    if (c < d) {
      a = ld1(xr, c);
      if (r) a += ld1(r + row * d, c);
      if (s_out) st1(s_out, row * d + c, a);
    }
    v[k] = a;
    sum += a;
  }
  const float mean = block_sum2(sum, 0.f, red).x / d;
  float sq = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c = threadIdx.x + k * kThreads;
    const float t = c < d ? v[k] - mean : 0.f;
    sq += t * t;
  }
  const float var = block_sum2(sq, 0.f, red).x / d;   // two-pass (population) variance, layers.py:106-110
  const float rstd = rsqrtf(var + eps);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c = threadIdx.x + k * kThreads;
    if (c < d) st1(y, row * d + c, (v[k] - mean) * rstd * ld1(gain, c) + ld1(bias, c));
  }
  if (threadIdx.x == 0) stats[row] = make_float2(mean, rstd);
}

// dx per row; per-CTA partial dgain / dbias over a block of rows
template <typename T>
__global__ void __launch_bounds__(kThreads) ln_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ s,
                                                          const T* __restrict__ gain,
                                                          const float2* __restrict__ stats, T* __restrict__ dx,
                                                          float* __restrict__ part, int64_t rows, int d,
                                                          int rows_per_cta) {
  __shared__ float2 red[kThreads / 32 + 1];
  float pg[16], pb[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) pg[k] = pb[k] = 0.f;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  for (int64_t row = r0; row < r1; ++row) {
    const float2 st = stats[row];
    float g[16], xh[16];
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int c = threadIdx.x + k * kThreads;
      g[k] = xh[k] = 0.f;
      if (c < d) {
        const float dyv = ld1(dy, row * d + c);
        xh[k] = (ld1(s, row * d + c) - st.x) * st.y;
        g[k] = dyv * ld1(gain, c);
        pg[k] += dyv * xh[k];
        pb[k] += dyv;
      }
      a += g[k];
      b += g[k] * xh[k];
    }
    const float2 m = block_sum2(a, b, red);
    const float ma = m.x / d, mb = m.y / d;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int c = threadIdx.x + k * kThreads;
      if (c < d) st1(dx, row * d + c, st.y * (g[k] - ma - xh[k] * mb));
    }
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c = threadIdx.x + k * kThreads;
    if (c < d) {
      part[((int64_t)blockIdx.x * 2) * d + c] = pg[k];
      part[((int64_t)blockIdx.x * 2 + 1) * d + c] = pb[k];
    }
  }
}

// column sums of the per-CTA partials (fixed order: deterministic)
template <typename T>
__global__ void ln_bwd_reduce_kernel(const float* __restrict__ part, int nparts, int d, T* __restrict__ dgain,
                                     T* __restrict__ dbias) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float a = 0.f, b = 0.f;
  for (int i = 0; i < nparts; ++i) {
    a += part[((int64_t)i * 2) * d + c];
    b += part[((int64_t)i * 2 + 1) * d + c];
  }
  st1(dgain, c, a);
  st1(dbias, c, b);
}

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.f + erff(x * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_df(float x) {
  return 0.5f * (1.f + erff(x * 0.70710678118654752f)) + x * 0.39894228040143268f * __expf(-0.5f * x * x);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) gelu_kernel(const T* __restrict__ x, const T* __restrict__ dy,
                                                        T* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = ld1(x, i);
    st1(out, i, dy ? ld1(dy, i) * gelu_df(v) : gelu_f(v));
  }
}

}  // namespace blk

int preload_block() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, blk::add_ln_kernel<float>));
  UL_CUDA(cudaFuncGetAttributes(&a, blk::add_ln_kernel<__nv_bfloat16>));
  UL_CUDA(cudaFuncGetAttributes(&a, blk::ln_bwd_kernel<float>));
  UL_CUDA(cudaFuncGetAttributes(&a, blk::ln_bwd_kernel<__nv_bfloat16>));
  UL_CUDA(cudaFuncGetAttributes(&a, blk::ln_bwd_reduce_kernel<float>));
  UL_CUDA(cudaFuncGetAttributes(&a, blk::ln_bwd_reduce_kernel<__nv_bfloat16>));
  UL_CUDA(cudaFuncGetAttributes(&a, blk::gelu_kernel<float>));
  UL_CUDA(cudaFuncGetAttributes(&a, blk::gelu_kernel<__nv_bfloat16>));
  return UL_OK;
}

}  // namespace ul

using namespace ul;

static int check_rows(int64_t rows, int64_t d, int dtype) {
  if (dtype != UL_DTYPE_F32 && dtype != UL_DTYPE_BF16) return fail(UL_ERR_KERNEL, "block kernels: dtype %d", dtype);
  if (rows < 0 || d < 1 || d > blk::kThreads * 16)
    return fail(UL_ERR_SHAPE, "block kernels: rows %lld, width %lld (1..%d)", (long long)rows, (long long)d,
                blk::kThreads * 16);
  return UL_OK;
}

extern "C" {

size_t ul_layernorm_bwd_workspace_bytes(int64_t rows, int64_t d) {
  const int64_t per = 64;   // rows per CTA of the backward
  return (size_t)((rows + per - 1) / per) * 2 * d * sizeof(float);
}

int ul_add_layernorm(const void* x, const void* r, const void* gain, const void* bias, void* s_out, void* y,
                     float* stats, int64_t rows, int64_t d, float eps, int dtype, void* stream) {
  launch_count() = 0;
  UL_TRY(check_rows(rows, d, dtype));
  if (rows == 0) return UL_OK;
  if (!x || !gain || !bias || !y || !stats) return fail(UL_ERR_ARG, "ul_add_layernorm: NULL tensor");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == UL_DTYPE_BF16)
    blk::add_ln_kernel<__nv_bfloat16><<<(unsigned)rows, blk::kThreads, 0, st>>>(
        (const __nv_bfloat16*)x, (const __nv_bfloat16*)r, (const __nv_bfloat16*)gain, (const __nv_bfloat16*)bias,
        (__nv_bfloat16*)s_out, (__nv_bfloat16*)y, (float2*)stats, (int)d, eps);
  else
    blk::add_ln_kernel<float><<<(unsigned)rows, blk::kThreads, 0, st>>>(
        (const float*)x, (const float*)r, (const float*)gain, (const float*)bias, (float*)s_out, (float*)y,
        (float2*)stats, (int)d, eps);
  return launched("add_layernorm");
}

int ul_layernorm_bwd(const void* dy, const void* s, const void* gain, const float* stats, void* dx, void* dgain,
                     void* dbias, void* workspace, size_t ws_bytes, int64_t rows, int64_t d, int dtype,
                     void* stream) {
  launch_count() = 0;
  UL_TRY(check_rows(rows, d, dtype));
  if (!dy || !s || !gain || !stats || !dx || !dgain || !dbias) return fail(UL_ERR_ARG, "ul_layernorm_bwd: NULL tensor");
  const size_t need = ul_layernorm_bwd_workspace_bytes(rows, d);
  if (!workspace || ws_bytes < need) return fail(UL_ERR_ARG, "ul_layernorm_bwd: workspace %zu < %zu", ws_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  const int per = 64;
  const unsigned nparts = (unsigned)((rows + per - 1) / per);
  if (nparts == 0) return fail(UL_ERR_SHAPE, "ul_layernorm_bwd: no rows");
  if (dtype == UL_DTYPE_BF16) {
    blk::ln_bwd_kernel<__nv_bfloat16><<<nparts, blk::kThreads, 0, st>>>(
        (const __nv_bfloat16*)dy, (const __nv_bfloat16*)s, (const __nv_bfloat16*)gain, (const float2*)stats,
        (__nv_bfloat16*)dx, (float*)workspace, rows, (int)d, per);
    UL_TRY(launched("layernorm_bwd"));
    blk::ln_bwd_reduce_kernel<__nv_bfloat16><<<(unsigned)((d + 255) / 256), 256, 0, st>>>(
        (const float*)workspace, (int)nparts, (int)d, (__nv_bfloat16*)dgain, (__nv_bfloat16*)dbias);
  } else {
    blk::ln_bwd_kernel<float><<<nparts, blk::kThreads, 0, st>>>((const float*)dy, (const float*)s, (const float*)gain,
                                                                (const float2*)stats, (float*)dx, (float*)workspace,
                                                                rows, (int)d, per);
    UL_TRY(launched("layernorm_bwd"));
    blk::ln_bwd_reduce_kernel<float><<<(unsigned)((d + 255) / 256), 256, 0, st>>>(
        (const float*)workspace, (int)nparts, (int)d, (float*)dgain, (float*)dbias);
  }
  return launched("layernorm_bwd_reduce");
}

int ul_gelu(const void* x, const void* dy, void* out, int64_t n, int dtype, void* stream) {
  launch_count() = 0;
  if (dtype != UL_DTYPE_F32 && dtype != UL_DTYPE_BF16) return fail(UL_ERR_KERNEL, "ul_gelu: dtype %d", dtype);
  if (n < 0) return fail(UL_ERR_SHAPE, "ul_gelu: n %lld", (long long)n);
  if (n == 0) return UL_OK;
  if (!x || !out) return fail(UL_ERR_ARG, "ul_gelu: NULL tensor");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t want = (n + blk::kThreads - 1) / blk::kThreads;
  const unsigned grid = (unsigned)(want < (int64_t)sm_count() * 16 ? want : (int64_t)sm_count() * 16);
  if (dtype == UL_DTYPE_BF16)
    blk::gelu_kernel<__nv_bfloat16><<<grid, blk::kThreads, 0, st>>>(
        (const __nv_bfloat16*)x, (const __nv_bfloat16*)dy, (__nv_bfloat16*)out, n);
  else
    blk::gelu_kernel<float><<<grid, blk::kThreads, 0, st>>>((const float*)x, (const float*)dy, (float*)out, n);
  return launched(dy ? "gelu_bwd" : "gelu");
}

}  // extern "C"
