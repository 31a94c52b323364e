// Micro-benchmark: how fast can one warp feed tcgen05.mma?  (tool, not product)
// Variants of the issue idiom, M=128 kind::f16, K=16 per instruction:
//   0 warp-wide asm with elect.sync inside every MMA (mma_ss_w / mma_ts_w)
//   1 if (elect_one) { loop of single-thread asm MMAs }
//   2 one asm block holding 8 MMAs behind one elect (operands in registers)
//   3 like 2 but the B descriptor advances inside the asm (K-loop shape)
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2309_14509_b200/csrc \
//      tools/ubench_mma_issue.cu -o build/ubench_mma_issue -lcuda
#include "sm100.cuh"

using namespace ul::sm100;

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, e;\n\t}"
      : "=r"(pred));
  return pred;
}

template <bool kTS>
__device__ __forceinline__ void mma1(uint32_t d, uint32_t a_tmem, uint64_t a_desc, uint64_t b, uint32_t idesc) {
  if (kTS)
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(d), "r"(a_tmem), "l"(b),
                 "r"(idesc)
                 : "memory");
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a_desc), "l"(b),
                 "r"(idesc)
                 : "memory");
}

#define MMA8_TS(D, A, B, I)                                                     \
  asm volatile(                                                                 \
      "{\n\t.reg .pred e;\n\t"                                                  \
      "elect.sync _|e, 0xffffffff;\n\t"                                         \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"        \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"        \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"        \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"        \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"        \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"        \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t"        \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}" ::"r"(D), \
      "r"(A), "l"(B), "r"(I)                                                    \
      : "memory")
#define MMA8_SS(D, A, B, I)                                                 \
  asm volatile(                                                             \
      "{\n\t.reg .pred e;\n\t"                                              \
      "elect.sync _|e, 0xffffffff;\n\t"                                     \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}" ::"r"(D), \
      "l"(A), "l"(B), "r"(I)                                                \
      : "memory")
// K-loop shape: B advances by 32 B (2 in descriptor units) per MMA
#define MMA8_TS_K(D, A, B, I)                                                     \
  asm volatile(                                                                   \
      "{\n\t.reg .pred e;\n\t.reg .b64 b;\n\t.reg .b32 a;\n\t"                    \
      "elect.sync _|e, 0xffffffff;\n\t"                                           \
      "mov.b64 b, %2;\n\tmov.b32 a, %1;\n\t"                                      \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t"            \
      "add.s64 b, b, 2;\n\tadd.u32 a, a, 8;\n\t"                                  \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t"            \
      "add.s64 b, b, 2;\n\tadd.u32 a, a, 8;\n\t"                                  \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t"            \
      "add.s64 b, b, 2;\n\tadd.u32 a, a, 8;\n\t"                                  \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t"            \
      "add.s64 b, b, 1018;\n\tadd.u32 a, a, 8;\n\t"                               \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t"            \
      "add.s64 b, b, 2;\n\tadd.u32 a, a, 8;\n\t"                                  \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t"            \
      "add.s64 b, b, 2;\n\tadd.u32 a, a, 8;\n\t"                                  \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t"            \
      "add.s64 b, b, 2;\n\tadd.u32 a, a, 8;\n\t"                                  \
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, 1;\n\t}" ::"r"(D), \
      "r"(A), "l"(B), "r"(I)                                                      \
      : "memory")

template <int kVar, int kN, bool kTS>
__global__ void __launch_bounds__(128, 1) issue_bench(unsigned long long* out, int n_mma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(128, kN, 0, 0);
    const uint64_t da = sdesc(smem_u32(sm), 16, 1024), db = sdesc(smem_u32(sm + 16384), 16, 1024);
    const uint32_t d = tb, a = tb + 256;
    long long t0 = clock64();
    if (kVar == 0) {
      for (int i = 0; i < n_mma; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (kTS)
            mma_ts_w(d, a, db, idesc, 1u);
          else
            mma_ss_w(d, da, db, idesc, 1u);
        }
      }
    } else if (kVar == 1) {
      if (elect_one()) {
        for (int i = 0; i < n_mma; i += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mma1<kTS>(d, a, da, db, idesc);
        }
      }
      __syncwarp();
    } else if (kVar == 2) {
      for (int i = 0; i < n_mma; i += 8) {
        if (kTS)
          MMA8_TS(d, a, db, idesc);
        else
          MMA8_SS(d, da, db, idesc);
      }
    } else {
      for (int i = 0; i < n_mma; i += 8) MMA8_TS_K(d, a, db, idesc);
    }
    mma_commit_w(&done);
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int kVar, int kN, bool kTS>
static void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const int smem = 100 * 1024, n_mma = 4096;
  cudaFuncSetAttribute(issue_bench<kVar, kN, kTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) issue_bench<kVar, kN, kTS><<<148, 128, smem>>>(d, n_mma);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148.0 * n_mma;
  printf("variant %d N=%3d %s err=%d: %6.1f cyc/mma (floor %d)\n", kVar, kN, kTS ? "TS" : "SS", (int)e, c,
         128 * kN / 256);
  cudaFree(d);
}

template <int kVar>
static void run_all() {
  run<kVar, 64, false>();
  run<kVar, 64, true>();
  run<kVar, 128, false>();
  run<kVar, 128, true>();
  run<kVar, 256, false>();
  run<kVar, 256, true>();
}

int main() {
  run_all<0>();
  run_all<1>();
  run_all<2>();
  run<3, 64, true>();
  run<3, 128, true>();
  run<3, 256, true>();
  return 0;
}
