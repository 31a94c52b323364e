// Micro-benchmark (tool, not product): latency of a batch of 8 TS MMAs
// (M=128, N=64, K=16 each; issue -> commit observed) on an otherwise idle
// tensor pipe, while 8 other warps of the CTA
//   mode 0: idle          mode 1: tcgen05.ld 32x32b.x32 in a loop
//   mode 2: tcgen05.st    mode 3: MUFU ex2 + FMA chains (softmax-like issue load)
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2309_14509_b200/csrc \
//      tools/ubench_mma_contention.cu -o build/ubench_mma_contention -lcuda
#include "sm100.cuh"

using namespace ul::sm100;

template <int kMode, int kN>
__global__ void __launch_bounds__(320, 1) contention(unsigned long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
    stop = 0;
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  float acc = lane;
  if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, kN, 0, 0);
    const uint64_t db = sdesc(smem_u32(sm + 16384), 16, 1024);
    unsigned long long total = 0, issue = 0;
    for (int r = 0; r < reps; ++r) {
      long long t0 = clock64();
      if (elect_one()) {
#pragma unroll
        for (int u = 0; u < 8; ++u) mma_ts(tb, tb + 256 + u * 8, dadd(db, u * 2), idesc, 1u);
        mma_commit(&done);
        if (r >= 4) issue += clock64() - t0;
      }
      __syncwarp();
      mbar_wait(&done, r & 1);
      long long t1 = clock64();
      if (r >= 4) total += t1 - t0;
      for (int w = 0; w < 200; ++w) __nanosleep(1);   // let the pipe drain / others run
    }
    issue = __reduce_max_sync(0xffffffffu, (unsigned)issue);
    if (lane == 0) out[blockIdx.x] = total / (reps - 4);
    if (lane == 0) out[200 + blockIdx.x] = issue / (reps - 4);
    stop = 1;
  } else if (warp >= 2) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col = 128 + ((warp - 2) >> 2) * 32;
    uint32_t sink = 0;
    while (!stop) {
      if (kMode == 1) {
        uint32_t r[32];
        tmem_ld32(tb + lane_off + col, r);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < 32; ++x) sink ^= r[x];
      } else if (kMode == 2) {
        uint32_t r[32];
#pragma unroll
        for (int x = 0; x < 32; ++x) r[x] = sink + x;
        tmem_st32(tb + lane_off + col, r);
        tmem_wait_st();
        sink += 1;
      } else if (kMode == 3) {
#pragma unroll
        for (int x = 0; x < 32; ++x) acc = fast_exp2(fmaf(acc, 0.999f, -0.5f)) * 0.5f + acc * 0.25f;
      } else {
        __nanosleep(100);
      }
    }
    if (sink == 0x12345u || acc == 1234.5f) out[1000 + blockIdx.x] = sink;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int M, int N>
static void run(const char* tag) {
  unsigned long long* d;
  cudaMalloc(&d, 2000 * sizeof(unsigned long long));
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(contention<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  contention<M, N><<<148, 320, smem>>>(d, 64);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[348];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0, ci = 0;
  for (int i = 0; i < 148; ++i) c += h[i], ci += h[200 + i];
  printf("%-34s N=%3d err=%d: batch of 8 MMAs issue->complete %7.1f cyc (floor %d), issue alone %6.1f\n", tag, N,
         (int)e, c / 148, 8 * 128 * N / 256, ci / 148);
  cudaFree(d);
}

int main() {
  run<0, 64>("idle");
  run<1, 64>("8 warps tcgen05.ld");
  run<2, 64>("8 warps tcgen05.st");
  run<3, 64>("8 warps ex2/FMA");
  run<0, 128>("idle");
  run<1, 128>("8 warps tcgen05.ld");
  run<2, 128>("8 warps tcgen05.st");
  run<3, 128>("8 warps ex2/FMA");
  return 0;
}
