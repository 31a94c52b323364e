// Probe (tool, not product): which (TMEM lane, column) each thread / register
// of tcgen05.ld 16x256b / 16x128b / 16x64b reads, relative to 32x32b (thread
// t = lane t of the warp's quarter, register c = column c).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2309_14509_b200/csrc \
//      tools/probe_tmem_shapes.cu -o build/probe_tmem_shapes
#include <cstdio>

#include "sm100.cuh"

using namespace ul::sm100;

__global__ void probe(int* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot + ((uint32_t)(warp * 32) << 16);
  uint32_t v[32];
  for (int c = 0; c < 32; ++c) v[c] = (uint32_t)((warp * 32 + lane) * 1000 + c);
  tmem_st32(base, v);
  tmem_wait_st();
  __syncwarp();
  uint32_t a[4], b[2], d;
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(base));
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0, %1}, [%2];" : "=r"(b[0]), "=r"(b[1]) : "r"(base));
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(d) : "r"(base));
  uint32_t e[4];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3]) : "r"(base + (16u << 16)));
  uint32_t f[8];
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(f[0]), "=r"(f[1]), "=r"(f[2]), "=r"(f[3]), "=r"(f[4]), "=r"(f[5]), "=r"(f[6]), "=r"(f[7])
               : "r"(base));
  tmem_wait_ld();
  if (warp == 1) {
    int* o = out + lane * 19;
    for (int i = 0; i < 4; ++i) o[i] = (int)a[i];
    for (int i = 0; i < 2; ++i) o[4 + i] = (int)b[i];
    o[6] = (int)d;
    for (int i = 0; i < 4; ++i) o[7 + i] = (int)e[i];
    for (int i = 0; i < 8; ++i) o[11 + i] = (int)f[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(slot);
}

int main() {
  int* d;
  cudaMalloc(&d, 32 * 19 * sizeof(int));
  probe<<<1, 128>>>(d);
  int h[32 * 19];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("warp 1 (lanes 32-63); value = lane*1000 + col\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%2d 16x256b:", t);
    for (int i = 0; i < 4; ++i) printf(" %6d", h[t * 19 + i]);
    printf(" | 16x128b: %6d %6d | 16x64b: %6d | 16x256b@+16:", h[t * 19 + 4], h[t * 19 + 5], h[t * 19 + 6]);
    for (int i = 0; i < 4; ++i) printf(" %6d", h[t * 19 + 7 + i]);
    printf(" | 16x256b.x2:");
    for (int i = 0; i < 8; ++i) printf(" %6d", h[t * 19 + 11 + i]);
    printf("\n");
  }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
