// Micro-benchmark (tool, not product): cycles per exponential column of the
// forward softmax's per-row sequence (f32x2 scale, ex2, bf16x2 pack, f32x2 row
// sum) for W warps per SMSP, registers only (no TMEM): is one softmax warp per
// SMSP able to keep the MUFU busy?
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2309_14509_b200/csrc \
//      tools/ubench_softmax_warp.cu -o build/ubench_softmax_warp
#include <cstdio>

#include "sm100.cuh"

using namespace ul::sm100;

// kMode 0: scale + ex2 + pack + row sum (the kernel's exp_chunk)
//       1: scale + ex2 + pack (no row sum)
//       2: ex2 only
//       3: mode 0 with 1/16 of the pairs on the FMA-pipe polynomial
template <int kMode>
__global__ void __launch_bounds__(256, 1) bench(unsigned long long* out, uint32_t* sink, int iters, float scale) {
  uint32_t r[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) r[c] = __float_as_uint(-0.01f * ((threadIdx.x + c) & 63));
  float2 rsum[4] = {};
  uint32_t acc = 0;
  const float2 sc = make_float2(scale, scale), nm = make_float2(-0.5f, -0.5f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 128; c += 32) {
      uint32_t pk[16];
#pragma unroll
      for (int x = 0; x < 32; x += 2) {
        float2 e;
        if (kMode == 2) {
          e.x = fast_exp2(__uint_as_float(r[c + x]));
          e.y = fast_exp2(__uint_as_float(r[c + x + 1]));
          pk[x / 2] = __float_as_uint(e.x) ^ __float_as_uint(e.y);
          continue;
        }
        const float2 a = __ffma2_rn(make_float2(__uint_as_float(r[c + x]), __uint_as_float(r[c + x + 1])), sc, nm);
        if (kMode == 3 && (x & 30) == 30) {
          e = poly_exp2x2(a);
        } else {
          e.x = fast_exp2(a.x);
          e.y = fast_exp2(a.y);
        }
        if (kMode == 0 || kMode == 3) rsum[(x >> 1) & 3] = __fadd2_rn(rsum[(x >> 1) & 3], e);
        pk[x / 2] = pack_bf16_op(e.x, e.y);
      }
#pragma unroll
      for (int x = 0; x < 16; ++x) acc ^= pk[x];
    }
    // perturb the inputs so the loop is not hoisted
#pragma unroll
    for (int c = 0; c < 128; ++c) r[c] ^= (acc & 1u);
  }
  const long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + threadIdx.x / 32] = (unsigned long long)(t1 - t0);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(rsum[0].x + rsum[1].y + rsum[2].x + rsum[3].y);
}

template <int kMode>
void run(const char* name, int warps_per_smsp) {
  const int threads = 4 * 32 * warps_per_smsp, iters = 200;
  unsigned long long* d;
  uint32_t* s;
  cudaMalloc(&d, 148 * 32 * sizeof(unsigned long long));
  cudaMalloc(&s, 148 * 512 * sizeof(uint32_t));
  bench<kMode><<<148, threads>>>(d, s, iters, 0.0883f);
  bench<kMode><<<148, threads>>>(d, s, iters, 0.0883f);
  cudaDeviceSynchronize();
  unsigned long long h[32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int w = 0; w < threads / 32; ++w) mx = h[w] > mx ? h[w] : mx;
  const double cols = 128.0 * iters;   // per warp
  printf("%-34s %d warp(s)/SMSP: %6.2f cycles per column per warp, %5.2f cycles per column per SMSP (MUFU floor 8.0)\n",
         name, warps_per_smsp, mx / cols, mx / cols / warps_per_smsp);
  cudaFree(d);
  cudaFree(s);
}

int main() {
  for (int w = 1; w <= 2; w *= 2) {
    run<0>("scale+ex2+pack+rowsum", w);
    run<1>("scale+ex2+pack", w);
    run<2>("ex2 only", w);
    run<3>("scale+ex2(15/16)+poly(1/16)+sum", w);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
