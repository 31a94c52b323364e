// Micro-benchmark (tool, not product): sustained tcgen05.mma kind::f16 rate
// for M=128, K=16 with N = 64 / 128 / 256, A from smem (SS) or TMEM (TS),
// A/B K-major or MN-major, one elected thread issuing back to back (the
// kernels' idiom).  Reports cycles per MMA vs the 8192 FLOP/clk/SM floor
// (N/2 cycles), i.e. whether shared-memory operand bandwidth limits SS.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2309_14509_b200/csrc \
//      tools/ubench_mma_rate.cu -o ab_libs/bin/ubench_mma_rate
#include <cstdio>

#include "sm100.cuh"

using namespace ul::sm100;

template <int N, int TS, int AMN, int BMN>
__global__ void __launch_bounds__(128, 1) rate(unsigned long long* out, int n_mma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done;
  for (int i = threadIdx.x; i < 131072 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x < 32) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(128, N, AMN, BMN);
      // A: 128 x 16 slice of a 128x128 tile (32 KB), B: N x 16 slice of an N x 128 tile
      const uint64_t da = sdesc(smem_u32(sm), AMN ? 16384 : 16, 1024);
      const uint64_t db = sdesc(smem_u32(sm + 32768), BMN ? 16384 : 16, 1024);
      long long t0 = clock64();
      for (int i = 0; i < n_mma; i += 8) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offa = AMN ? kk * 2048 : (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint32_t offb = BMN ? kk * 2048 : (kk >> 2) * 16384 + (kk & 3) * 32;
          if (TS)
            mma_ts(tb + 256, tb + kk * 8, dadd(db, offb), idesc, 1u);
          else
            mma_ss(tb + 256, dadd(da, offa), dadd(db, offb), idesc, 1u);
        }
      }
      mma_commit(&done);
      mbar_wait(&done, 0);
      long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int N, int TS, int AMN, int BMN>
static void run(const char* tag) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 131072 + 1024;
  cudaFuncSetAttribute(rate<N, TS, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int n = 8192;
  for (int r = 0; r < 2; ++r) rate<N, TS, AMN, BMN><<<148, 128, smem>>>(d, n);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  printf("%-26s N=%3d: %6.1f cyc/mma (floor %3d) -> %.0f%% of tensor peak  %s\n", tag, N, c / n, N / 2,
         100.0 * (N / 2) / (c / n), e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, 0, 0, 0>("SS  A K-major B K-major");
  run<128, 0, 0, 0>("SS  A K-major B K-major");
  run<256, 0, 0, 0>("SS  A K-major B K-major");
  run<64, 1, 0, 0>("TS  B K-major");
  run<128, 1, 0, 0>("TS  B K-major");
  run<256, 1, 0, 0>("TS  B K-major");
  run<64, 0, 1, 1>("SS  A MN-major B MN-major");
  run<128, 0, 0, 1>("SS  A K-major B MN-major");
  run<128, 1, 0, 1>("TS  B MN-major");
  return 0;
}
