// K0: the Q/K/V projection GEMM with the seq->head exchange in its epilogue
// (SURVEY 8(f) item 1).
//
// Replaces project(x, wq/wk/wv) (layers.py:118-122, ulysses.py:140-142)
// followed by _to_head (ulysses.py:161-164 -> all_to_all split 2 /
// concat 0, simgroup.py:313-335): Y = X [wq | wk | wv] with X this rank's
// sequence shard [nl*b, d] and every 128-column head block of Y stored
// straight into the head-layout image [N, b, H_t/P, hd] of the rank that
// owns the head -- the own output tensor, or the peer's receive slot over
// NVLink -- at rows me*nl + s; the last CTA publishes the call and the
// receivers drain their slots (the same protocol as ul_all_to_all).
//
// tcgen05 GEMM, persistent CTAs over 128 x 256 output tiles (one tile = two
// heads of hd = 128): warp 0 TMA (X K-major 128 x 64, W MN-major 64 x 256
// per stage, 4 stages), warp 1 MMA (M = 128, N = 256, K = 16: 96 B/clk of
// shared-memory operands, full tensor rate), warps 2-5 epilogue from a
// double-buffered TMEM accumulator (2 x 256 columns) so a tile's stores
// overlap the next tile's MMAs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstring>

#include "comm.cuh"
#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace ul {


namespace proj {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int NSTAGE = 4;
constexpr int kThreads = 192;
constexpr int kATile = BM * BK * 2;   // 16 KB
constexpr int kBTile = BK * BN * 2;   // 32 KB (four 64-column atoms of 8 KB)

struct Smem {
  static constexpr int kA = 0;
  static constexpr int kB = kA + NSTAGE * kATile;
  static constexpr int kBar = kB + NSTAGE * kBTile;
  static constexpr int kBytes = kBar + 256 + 1024;
};

struct Params {
  int M, K, N;
  int mtiles, ntiles;
  ProjEpilogue ep;
};

// kBKMajor: B is read from a row-major [N, K] matrix (Y = X W^T, e.g. the
// backward's dc = g Wo^T): one 256-row x 64-column K-major box per stage;
// otherwise from a row-major [K, N] matrix (Y = X W): four MN-major boxes.
template <bool kBKMajor>
__global__ void __launch_bounds__(kThreads, 1)
    qkv_proj_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + Smem::kA;
  uint8_t* sB = smem + Smem::kB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::kBar);
  uint64_t* full = bars;                     // [NSTAGE]
  uint64_t* empty = bars + NSTAGE;           // [NSTAGE]
  uint64_t* acc_full = bars + 2 * NSTAGE;    // [2]
  uint64_t* acc_empty = bars + 2 * NSTAGE + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NSTAGE + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile_total = p.mtiles * p.ntiles;
  const int ksteps = p.K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 4);   // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tbase = 0;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmX);
      tma_prefetch_desc(&tmW);
      int it = 0;
      for (int tile = blockIdx.x; tile < ntile_total; tile += gridDim.x) {
        const int mt = tile % p.mtiles, nt = tile / p.mtiles;
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % NSTAGE;
          mbar_wait(&empty[s], ((it / NSTAGE) & 1) ^ 1);
          mbar_expect_tx(&full[s], kATile + kBTile);
          tma_load_2d(sA + s * kATile, &tmX, &full[s], ks * BK, mt * BM);
          if constexpr (kBKMajor) {
            tma_load_2d(sB + s * kBTile, &tmW, &full[s], ks * BK, nt * BN);
          } else {
#pragma unroll
            for (int a = 0; a < BN / 64; ++a)
              tma_load_2d(sB + s * kBTile + a * (BK * 128), &tmW, &full[s], nt * BN + a * 64, ks * BK);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t kId = idesc_bf16(BM, BN, 0, kBKMajor ? 0 : 1);   // A K-major, B K- or MN-major
      const uint64_t dA0 = sdesc(smem_u32(sA), 16, 1024);
      const uint64_t dB0 = kBKMajor ? sdesc(smem_u32(sB), 16, 1024) : sdesc(smem_u32(sB), BK * 128, 1024);
      int it = 0, tcount = 0;
      for (int tile = blockIdx.x; tile < ntile_total; tile += gridDim.x, ++tcount) {
        const int buf = tcount & 1;
        if (tcount >= 2) {
          mbar_wait_mma(&acc_empty[buf], ((tcount - 2) >> 1) & 1);
          tc_fence_after();
        }
        const uint32_t tacc = tbase + buf * BN;
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % NSTAGE;
          mbar_wait_mma(&full[s], (it / NSTAGE) & 1);
          tc_fence_after();
          const uint64_t da = dadd(dA0, s * kATile), db = dadd(dB0, s * kBTile);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_ss(tacc, dadd(da, kk * 32), dadd(db, kBKMajor ? kk * 32 : kk * 2048), kId, (ks > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: thread = output row; each 128-column half is one head of one tensor
    const int quarter = warp & 3;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const ProjEpilogue& ep = p.ep;
    int tcount = 0;
    for (int tile = blockIdx.x; tile < ntile_total; tile += gridDim.x, ++tcount) {
      const int buf = tcount & 1;
      const int mt = tile % p.mtiles, nt = tile / p.mtiles;
      mbar_wait(&acc_full[buf], (tcount >> 1) & 1);
      tc_fence_after();
      const int m = mt * BM + quarter * 32 + lane;
      const bool valid = m < p.M;
      const int s = m / ep.b, bb = m - s * ep.b;
#pragma unroll 1
      for (int half = 0; half < BN / 128; ++half) {
        const int n = nt * BN + half * 128;
        const int t = n >= ep.col0[2] ? 2 : (n >= ep.col0[1] ? 1 : 0);
        const int head = (n - ep.col0[t]) / ep.hd;
        const int dr = head / ep.hl[t], lh = head - dr * ep.hl[t];
        uint4* dst = reinterpret_cast<uint4*>(
            ep.dst[t][dr] + ((((int64_t)ep.me * ep.nl + s) * ep.b + bb) * ep.hl[t] + lh) * (int64_t)ep.hd * 2);
        const bool live = valid && n < ep.col0[3];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld32(tbase + buf * BN + lane_off + half * 128 + c * 32, v);
          tmem_wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int x = 0; x < 16; ++x) pk[x] = pack_bf16(__uint_as_float(v[2 * x]), __uint_as_float(v[2 * x + 1]));
          if (live) {
#pragma unroll
            for (int x = 0; x < 4; ++x) dst[c * 4 + x] = make_uint4(pk[4 * x], pk[4 * x + 1], pk[4 * x + 2], pk[4 * x + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
    if (ep.sg.active) __threadfence_system();
  }
  tc_fence_before();
  __syncthreads();
  if (p.ep.sg.active && threadIdx.x == 0) peer_signal_last_cta(p.ep.sg, gridDim.x);
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

}  // namespace proj

int preload_proj() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, proj::qkv_proj_kernel<false>));
  UL_CUDA(cudaFuncGetAttributes(&a, proj::qkv_proj_kernel<true>));
  // dynamic shared-memory opt-ins now, not at the first launch (common.cuh)
  UL_TRY(smem_opt_in((const void*)proj::qkv_proj_kernel<false>, proj::Smem::kBytes));
  UL_TRY(smem_opt_in((const void*)proj::qkv_proj_kernel<true>, proj::Smem::kBytes));
  return UL_OK;
}

// Y[M, N] = X[M, K] W[K, N] (bf16, fp32 accumulate) -- or X W^T with W
// stored [N, K] (w_transposed) -- stored per 128-column head block through
// `ep` (see above).  K % 64 == 0, N % 128 == 0.
int sm100_qkv_proj(const void* x, const void* w, int64_t M, int64_t K, int64_t N, const ProjEpilogue& ep,
                   cudaStream_t st, bool w_transposed) {
  if (K % proj::BK != 0 || N % 128 != 0 || ep.hd != 128)
    return fail(UL_ERR_KERNEL, "qkv projection needs d %% 64 == 0, columns %% 128 == 0 and head_dim 128 "
                "(K=%lld, N=%lld, hd=%d)", (long long)K, (long long)N, ep.hd);
  if (M > INT32_MAX || N > INT32_MAX) return fail(UL_ERR_SHAPE, "qkv projection too large");
  if (M == 0) return UL_OK;
  CUtensorMap mx, mw;
  UL_TRY(make_tmap_2d(&mx, x, M, K, proj::BM));
  if (w_transposed) UL_TRY(make_tmap_2d(&mw, w, N, K, proj::BN));
  else UL_TRY(make_tmap_2d(&mw, w, K, N, proj::BK));
  proj::Params p;
  p.M = (int)M;
  p.K = (int)K;
  p.N = (int)N;
  p.mtiles = (int)((M + proj::BM - 1) / proj::BM);
  p.ntiles = (int)((N + proj::BN - 1) / proj::BN);
  p.ep = ep;
  const int tiles = p.mtiles * p.ntiles;
  const int grid = tiles < sm_count() ? tiles : sm_count();
  if (w_transposed) {
    UL_TRY(smem_opt_in((const void*)proj::qkv_proj_kernel<true>, proj::Smem::kBytes));
    proj::qkv_proj_kernel<true><<<grid, proj::kThreads, proj::Smem::kBytes, st>>>(mx, mw, p);
  } else {
    UL_TRY(smem_opt_in((const void*)proj::qkv_proj_kernel<false>, proj::Smem::kBytes));
    proj::qkv_proj_kernel<false><<<grid, proj::kThreads, proj::Smem::kBytes, st>>>(mx, mw, p);
  }
  return launched("qkv_proj_sm100");
}

}  // namespace ul
