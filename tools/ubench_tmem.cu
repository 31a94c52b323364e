// Micro-benchmark of the per-SM tensor-memory paths the attention kernels
// lean on (not part of the product; built and run by hand under gpurun):
//   1. tcgen05.ld 32x32b.x32 bandwidth (bytes/clk/SM) vs number of warps
//   2. tcgen05.mma kind::f16 M=128 issue-to-completion rate for N=64/128/256,
//      A from smem (SS) and from TMEM (TS)
//   3. both at once (MMA N=64 TS stream + 8 loading warps)
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2309_14509_b200/csrc \
//      tools/ubench_tmem.cu -o build/ubench_tmem -lcuda
#include "sm100.cuh"

using namespace ul::sm100;

struct Out {
  unsigned long long ld_cycles, mma_cycles, ld_bytes;
  unsigned sink;
};

// mode 0: loads only (nw warps); mode 1: MMA only; mode 2: MMA + loads
template <int kMode>
__global__ void __launch_bounds__(288, 1) ubench(Out* out, int nload_warps, int n_mma, int mma_n, int ts, int iters, int nacc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t done;
  __shared__ unsigned long long ld_cyc[9];
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
  unsigned sink = 0;
  if (warp == 8) {
    if (kMode != 0) {
      const uint32_t idesc = idesc_bf16(128, mma_n, 0, 0);
      const uint64_t da = sdesc(smem_u32(sm), 16, 1024), db = sdesc(smem_u32(sm + 16384), 16, 1024);
      long long t0 = clock64();
      const uint32_t dstride = mma_n <= 64 ? 64 : 128;
      for (int i = 0; i < n_mma; i += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t d = tb + ((i + u) % nacc) * dstride;
          if (ts)
            mma_ts_w(d, tb + 256, db, idesc, 1u);
          else
            mma_ss_w(d, da, db, idesc, 1u);
        }
      }
      mma_commit_w(&done);
      mbar_wait(&done, 0);
      long long t1 = clock64();
      if (lane == 0) out[blockIdx.x].mma_cycles = t1 - t0;
    }
  } else if (warp < nload_warps && kMode != 1) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t col = (kMode == 2 ? 128 : 0) + (warp >> 2) * 32;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      tmem_ld32(tb + lane_off + col, r);
      tmem_wait_ld();
#pragma unroll
      for (int x = 0; x < 32; ++x) sink ^= r[x];
    }
    long long t1 = clock64();
    if (lane == 0) ld_cyc[warp] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && kMode != 1) {
    unsigned long long mx = 0;
    for (int w = 0; w < nload_warps; ++w) mx = ld_cyc[w] > mx ? ld_cyc[w] : mx;
    out[blockIdx.x].ld_cycles = mx;
    out[blockIdx.x].ld_bytes = (unsigned long long)nload_warps * iters * 4096ull;
  }
  if (sink == 0x12345678u) out[blockIdx.x].sink = sink;
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tb);
  }
}

template <int M>
static void run(const char* tag, int nw, int n_mma, int mma_n, int ts, int iters, int nacc) {
  Out* d;
  cudaMalloc(&d, 148 * sizeof(Out));
  cudaMemset(d, 0, 148 * sizeof(Out));
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(ubench<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) ubench<M><<<148, 288, smem>>>(d, nw, n_mma, mma_n, ts, iters, nacc);
  cudaError_t e = cudaDeviceSynchronize();
  Out h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double ldc = 0, mmc = 0;
  for (int i = 0; i < 148; ++i) {
    ldc += h[i].ld_cycles;
    mmc += h[i].mma_cycles;
  }
  ldc /= 148;
  mmc /= 148;
  printf("%-28s err=%d", tag, (int)e);
  if (M != 1) printf("  ld: %d warps %.1f B/clk/SM (%.0f cyc per x32 per warp)", nw, h[0].ld_bytes / ldc, ldc / iters);
  if (M != 0) printf("  mma N=%d %s acc=%d: %.1f cyc/mma (floor %d)", mma_n, ts ? "TS" : "SS", nacc, mmc / n_mma, 128 * mma_n / 256);
  printf("\n");
  cudaFree(d);
}

int main() {
  for (int nw : {1, 2, 4, 8}) run<0>("tmem ld", nw, 0, 64, 0, 4096, 1);
  for (int n : {64, 128, 256})
    for (int ts : {0, 1})
      for (int nacc : {1, 2, 4}) {
        if (n * nacc > 256 && !(n == 64 && nacc == 4)) continue;
        if (ts && n * nacc > 256) continue;
        run<1>("mma", 0, 4096, n, ts, 0, nacc);
      }
  for (int nw : {4, 8}) run<2>("mma N=64 TS + ld", nw, 4096, 64, 1, 1024, 4);
  for (int nw : {4, 8}) run<2>("mma N=128 TS + ld", nw, 2048, 128, 1, 1024, 2);
  return 0;
}
