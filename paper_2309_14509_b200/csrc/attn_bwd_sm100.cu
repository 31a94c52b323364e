// K4: attention backward on sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces masked_attention_backward (kernels.py:89-111) in the per-head
// loop of ulysses_attention_backward (ulysses.py:218-222):
//   probs = softmax(q k^T * scale)          (recomputed from the saved LSE)
//   dprobs = dctx v^T ; dot = rowsum(dprobs*probs) == rowsum(dctx*ctx) = D
//   dscores = probs * (dprobs - dot) * scale
//   dq = dscores k ; dk = dscores^T q ; dv = probs^T dctx
// GQA (restatement): dk/dv of kv head g are summed over its query group.
//
// Three launches, no atomics (deterministic, so results are P-invariant
// bit for bit):
//   bwd_prep   D = rowsum(dO*O) and LSE*log2(e) into padded f32 rows
//   bwd_dkdv   one CTA per (kv tile, kv head): loops over the group's
//              query heads and the visible query tiles; S^T = K Q^T and
//              dP^T = V dO^T land in TMEM (kv rows on lanes), softmax warps
//              write P^T / dS^T back to TMEM as bf16, then
//              dV += P^T dO and dK += dS^T Q (TS MMAs) accumulate in TMEM.
//   bwd_dq     one CTA per (query tile, head): S = Q K^T, dP = dO V^T,
//              dS -> TMEM, dQ += dS K.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace ul {
namespace bwd {

using namespace sm100;

constexpr int BM = 128;   // query tile
constexpr int BN = 128;   // key tile
constexpr int kThreads = 192;
constexpr int kAtom = 128 * 128;  // SW128 atom column of a 128-row tile

struct Params {
  int n, n_pad, b, hq, hkv;
  int causal;
  float scale, scale_log2;
  const float* L2;   // [b*hq][n_pad] lse * log2(e), +inf padded
  const float* Dv;   // [b*hq][n_pad] rowsum(dO*O), 0 padded
  __nv_bfloat16* dq;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
};

// ---- pre-pass ----------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(256) bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                                       const __nv_bfloat16* __restrict__ dout,
                                                       const float* __restrict__ lse, float* __restrict__ L2,
                                                       float* __restrict__ Dv, int n, int n_pad, int b, int hq) {
  const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)b * hq * n_pad;
  if (warp >= rows) return;
  const int bh = warp / n_pad;
  const int i = warp % n_pad;
  float s = 0.f;
  float l = INFINITY;
  if (i < n) {
    const int bb = bh / hq, h = bh % hq;
    const int64_t off = (((int64_t)i * b + bb) * hq + h) * HD;
    constexpr int PER = HD / 32;  // bf16 per lane
    if constexpr (PER == 4) {
      const uint2 a = *reinterpret_cast<const uint2*>(o + off + lane * 4);
      const uint2 c = *reinterpret_cast<const uint2*>(dout + off + lane * 4);
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        float2 fa = __bfloat1622float2(a2[x]), fc = __bfloat1622float2(c2[x]);
        s = fmaf(fa.x, fc.x, s);
        s = fmaf(fa.y, fc.y, s);
      }
    } else {
      const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(o + off + lane * 2);
      const __nv_bfloat162 c = *reinterpret_cast<const __nv_bfloat162*>(dout + off + lane * 2);
      float2 fa = __bfloat1622float2(a), fc = __bfloat1622float2(c);
      s = fa.x * fc.x + fa.y * fc.y;
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    l = lse[(int64_t)bh * n + i] * 1.4426950408889634f;
  }
  if (lane == 0) {
    Dv[(int64_t)bh * n_pad + i] = (i < n) ? s : 0.f;
    L2[(int64_t)bh * n_pad + i] = l;
  }
}

// ---- dK / dV -----------------------------------------------------------------
template <int HD>
struct DkdvSmem {
  static constexpr int kTile = (HD / 64) * kAtom;
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTile;
  static constexpr int kQ = kV + kTile;          // [2] stages
  static constexpr int kO = kQ + 2 * kTile;      // dO [2]
  static constexpr int kL = kO + 2 * kTile;      // [2][BM] f32
  static constexpr int kD = kL + 2 * BM * 4;     // [2][BM] f32
  static constexpr int kBar = kD + 2 * BM * 4;
  static constexpr int kBytes = kBar + 256 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const Params p) {
  using S = DkdvSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sO = smem + S::kO;
  float* sL = reinterpret_cast<float*>(smem + S::kL);
  float* sD = reinterpret_cast<float*>(smem + S::kD);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;   // [2]
  uint64_t* q_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* p_full = bars + 6;
  uint64_t* m_done = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = (p.n + BN - 1) / BN;
  const int heads = p.b * p.hkv;
  const int kt = (int)(blockIdx.x / heads);      // ascending kv tile == longest first (causal)
  const int bg = (int)(blockIdx.x % heads);
  const int bb = bg / p.hkv, g = bg % p.hkv;
  const int group = p.hq / p.hkv;
  const int kv0 = kt * BN;
  const int nq = (p.n + BM - 1) / BM;
  const int i0 = p.causal ? kv0 / BM : 0;
  const int per_head = nq - i0;
  const int total = per_head * group;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 128);
    mbar_init(m_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tSt = tbase, tdPt = tbase + 128, tdV = tbase + 256, tdK = tbase + 256 + HD;
  (void)nkv;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
      mbar_expect_tx(kv_full, 2 * BN * HD * 2);
#pragma unroll
      for (int a = 0; a < HD / 64; ++a) {
        tma_load_3d(sK + a * kAtom, &tmK, kv_full, a * 64, bb * p.hkv + g, kv0);
        tma_load_3d(sV + a * kAtom, &tmV, kv_full, a * 64, bb * p.hkv + g, kv0);
      }
      for (int it = 0; it < total; ++it) {
        const int h = g * group + it / per_head;
        const int qi = i0 + it % per_head;
        const int s = it & 1;
        mbar_wait(&q_empty[s], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[s], 2 * BM * HD * 2 + 2 * BM * 4);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a) {
          tma_load_3d(sQ + s * S::kTile + a * kAtom, &tmQ, &q_full[s], a * 64, bb * p.hq + h, qi * BM);
          tma_load_3d(sO + s * S::kTile + a * kAtom, &tmO, &q_full[s], a * 64, bb * p.hq + h, qi * BM);
        }
        const int64_t roff = ((int64_t)bb * p.hq + h) * p.n_pad + qi * BM;
        bulk_load(sL + s * BM, p.L2 + roff, BM * 4, &q_full[s]);
        bulk_load(sD + s * BM, p.Dv + roff, BM * 4, &q_full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_bf16(BN, BM, 0, 0);   // M = kv rows, N = q rows
      constexpr uint32_t kIdG = idesc_bf16(BN, HD, 0, 1);   // M = kv rows, N = hd, B MN-major
      const uint32_t kaddr = smem_u32(sK), vaddr = smem_u32(sV);
      mbar_wait(kv_full, 0);
      for (int it = 0; it < total; ++it) {
        const int s = it & 1;
        if (it > 0) mbar_wait(m_done, (it - 1) & 1);
        mbar_wait(&q_full[s], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t qaddr = smem_u32(sQ + s * S::kTile), oaddr = smem_u32(sO + s * S::kTile);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_ss(tSt, sdesc(kaddr + off, 16, 1024), sdesc(qaddr + off, 16, 1024), kIdS, kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_ss(tdPt, sdesc(vaddr + off, 16, 1024), sdesc(oaddr + off, 16, 1024), kIdS, kk > 0 ? 1u : 0u);
        }
        mma_commit(s_full);
        mbar_wait(p_full, it & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk) {
          mma_ts(tdV, tSt + kk * 8, sdesc(oaddr + kk * 2048, kAtom, 1024), kIdG, (it > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < BM / 16; ++kk) {
          mma_ts(tdK, tdPt + kk * 8, sdesc(qaddr + kk * 2048, kAtom, 1024), kIdG, (it > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&q_empty[s]);
        mma_commit(m_done);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;     // kv row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int kvrow = kv0 + row;
    for (int it = 0; it < total; ++it) {
      const int s = it & 1;
      const int qi = i0 + it % per_head;
      const int q0 = qi * BM;
      mbar_wait(&q_full[s], (it >> 1) & 1);
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      const float* L = sL + s * BM;
      const float* Dd = sD + s * BM;
      // visible query columns: q >= kv (causal)
      const int first = p.causal ? kvrow - q0 : 0;   // columns c < first are masked
      // 32-column chunks: P^T / dS^T of chunk c overwrite TMEM columns
      // [16c, 16c+16), which were consumed by chunk c' <= c
#pragma unroll
      for (int c = 0; c < BM / 32; ++c) {
        uint32_t r[32], d[32];
        tmem_ld32(tSt + lane_off + c * 32, r);
        tmem_ld32(tdPt + lane_off + c * 32, d);
        tmem_wait_ld();
        uint32_t pk[16], dsk[16];
#pragma unroll
        for (int x = 0; x < 32; x += 2) {
          const int col = c * 32 + x;
          float p0 = fast_exp2(__uint_as_float(r[x]) * p.scale_log2 - L[col]);
          float p1 = fast_exp2(__uint_as_float(r[x + 1]) * p.scale_log2 - L[col + 1]);
          if (col < first) p0 = 0.f;
          if (col + 1 < first) p1 = 0.f;
          pk[x / 2] = pack_bf16(p0, p1);
          dsk[x / 2] = pack_bf16(p0 * (__uint_as_float(d[x]) - Dd[col]), p1 * (__uint_as_float(d[x + 1]) - Dd[col + 1]));
        }
        tmem_st16(tSt + lane_off + c * 16, pk);
        tmem_st16(tdPt + lane_off + c * 16, dsk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: dV, dK * scale -> bf16 rows of kv head g
    mbar_wait(m_done, (total - 1) & 1);
    tc_fence_after();
    const bool valid = kvrow < p.n;
    const int64_t off = (((int64_t)kvrow * p.b + bb) * p.hkv + g) * HD;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t tacc = which == 0 ? tdV : tdK;
      const float mul = which == 0 ? 1.f : p.scale;
      __nv_bfloat16* dst = (which == 0 ? p.dv : p.dk) + off;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tacc + lane_off + c * 32, v);
        tmem_wait_ld();
        uint32_t pkd[16];
#pragma unroll
        for (int x = 0; x < 16; ++x)
          pkd[x] = pack_bf16(__uint_as_float(v[2 * x]) * mul, __uint_as_float(v[2 * x + 1]) * mul);
        if (valid) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
          for (int x = 0; x < 4; ++x) d4[x] = make_uint4(pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ---- dQ ------------------------------------------------------------------------
template <int HD>
struct DqSmem {
  static constexpr int kTile = (HD / 64) * kAtom;
  static constexpr int kQ = 0;
  static constexpr int kO = kQ + kTile;
  static constexpr int kK = kO + kTile;          // [2]
  static constexpr int kV = kK + 2 * kTile;      // [2]
  static constexpr int kBar = kV + 2 * kTile;
  static constexpr int kBytes = kBar + 256 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    bwd_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                  const Params p) {
  using S = DqSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sO = smem + S::kO;
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* p_full = bars + 6;
  uint64_t* m_done = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int heads = p.b * p.hq;
  const int qtiles = (p.n + BM - 1) / BM;
  const int qt = qtiles - 1 - (int)(blockIdx.x / heads);   // longest first
  const int bh = (int)(blockIdx.x % heads);
  const int bb = bh / p.hq, h = bh % p.hq;
  const int g = h / (p.hq / p.hkv);
  const int q0 = qt * BM;
  const int nkv_all = (p.n + BN - 1) / BN;
  const int nkv = p.causal ? min(nkv_all, (q0 + BM - 1) / BN + 1) : nkv_all;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 128);
    mbar_init(m_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tS = tbase, tdP = tbase + 128, tdQ = tbase + 256;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
      mbar_expect_tx(q_full, 2 * BM * HD * 2);
#pragma unroll
      for (int a = 0; a < HD / 64; ++a) {
        tma_load_3d(sQ + a * kAtom, &tmQ, q_full, a * 64, bb * p.hq + h, q0);
        tma_load_3d(sO + a * kAtom, &tmO, q_full, a * 64, bb * p.hq + h, q0);
      }
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        mbar_wait(&kv_empty[s], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], 2 * BN * HD * 2);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a) {
          tma_load_3d(sK + s * S::kTile + a * kAtom, &tmK, &kv_full[s], a * 64, bb * p.hkv + g, j * BN);
          tma_load_3d(sV + s * S::kTile + a * kAtom, &tmV, &kv_full[s], a * 64, bb * p.hkv + g, j * BN);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t kIdS = idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t kIdG = idesc_bf16(BM, HD, 0, 1);
      const uint32_t qaddr = smem_u32(sQ), oaddr = smem_u32(sO);
      mbar_wait(q_full, 0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        if (j > 0) mbar_wait(m_done, (j - 1) & 1);
        mbar_wait(&kv_full[s], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t kaddr = smem_u32(sK + s * S::kTile), vaddr = smem_u32(sV + s * S::kTile);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_ss(tS, sdesc(qaddr + off, 16, 1024), sdesc(kaddr + off, 16, 1024), kIdS, kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_ss(tdP, sdesc(oaddr + off, 16, 1024), sdesc(vaddr + off, 16, 1024), kIdS, kk > 0 ? 1u : 0u);
        }
        mma_commit(s_full);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts(tdQ, tdP + kk * 8, sdesc(kaddr + kk * 2048, kAtom, 1024), kIdG, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&kv_empty[s]);
        mma_commit(m_done);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int qrow = q0 + row;
    const int64_t roff = ((int64_t)bb * p.hq + h) * p.n_pad + qrow;
    const float L = p.L2[roff];
    const float Dr = p.Dv[roff];
    for (int j = 0; j < nkv; ++j) {
      const int kv0 = j * BN;
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      const int limit = p.causal ? qrow - kv0 + 1 : BN;   // columns c >= limit are masked
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32], d[32];
        tmem_ld32(tS + lane_off + c * 32, r);
        tmem_ld32(tdP + lane_off + c * 32, d);
        tmem_wait_ld();
        uint32_t dsk[16];
#pragma unroll
        for (int x = 0; x < 32; x += 2) {
          const int col = c * 32 + x;
          float p0 = fast_exp2(__uint_as_float(r[x]) * p.scale_log2 - L);
          float p1 = fast_exp2(__uint_as_float(r[x + 1]) * p.scale_log2 - L);
          if (col >= limit) p0 = 0.f;
          if (col + 1 >= limit) p1 = 0.f;
          dsk[x / 2] = pack_bf16(p0 * (__uint_as_float(d[x]) - Dr), p1 * (__uint_as_float(d[x + 1]) - Dr));
        }
        tmem_st16(tdP + lane_off + c * 16, dsk);   // dS over consumed dP columns
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(m_done, (nkv - 1) & 1);
    tc_fence_after();
    const bool valid = qrow < p.n;
    __nv_bfloat16* dst = p.dq + (((int64_t)qrow * p.b + bb) * p.hq + h) * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tdQ + lane_off + c * 32, v);   // warp-collective: executed by every lane
      tmem_wait_ld();
      uint32_t pkd[16];
#pragma unroll
      for (int x = 0; x < 16; ++x)
        pkd[x] = pack_bf16(__uint_as_float(v[2 * x]) * p.scale, __uint_as_float(v[2 * x + 1]) * p.scale);
      if (valid) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int x = 0; x < 4; ++x) d4[x] = make_uint4(pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

static int64_t pad_n(int64_t n) { return (n + 127) / 128 * 128; }

template <int HD>
static int launch(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
                  void* dq, void* dk, void* dv, void* ws, int64_t n, int64_t b, int64_t hq, int64_t hkv, int causal,
                  float scale, int stages, cudaStream_t st) {
  const int64_t npad = pad_n(n);
  float* L2 = reinterpret_cast<float*>(ws);
  float* Dv = L2 + b * hq * npad;
  if (stages & 1) {
    const int64_t warps = b * hq * npad;
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    bwd_prep_kernel<HD><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, lse, L2, Dv,
                                                (int)n, (int)npad, (int)b, (int)hq);
    UL_TRY(launched("attn_bwd_prep"));
  }
  CUtensorMap mq, mk, mv, mo;
  UL_TRY(make_tmap_bhsd(&mq, q, n, b * hq, HD, 128));
  UL_TRY(make_tmap_bhsd(&mk, k, n, b * hkv, HD, 128));
  UL_TRY(make_tmap_bhsd(&mv, v, n, b * hkv, HD, 128));
  UL_TRY(make_tmap_bhsd(&mo, dout, n, b * hq, HD, 128));
  Params p;
  p.n = (int)n;
  p.n_pad = (int)npad;
  p.b = (int)b;
  p.hq = (int)hq;
  p.hkv = (int)hkv;
  p.causal = causal;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.L2 = L2;
  p.Dv = Dv;
  p.dq = (__nv_bfloat16*)dq;
  p.dk = (__nv_bfloat16*)dk;
  p.dv = (__nv_bfloat16*)dv;
  static bool attr = false;
  if (!attr) {
    UL_CUDA(cudaFuncSetAttribute(bwd_dkdv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 DkdvSmem<HD>::kBytes));
    UL_CUDA(cudaFuncSetAttribute(bwd_dq_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, DqSmem<HD>::kBytes));
    attr = true;
  }
  const int64_t tiles = (n + 127) / 128;
  if (stages & 2) {
    bwd_dkdv_kernel<HD><<<(unsigned)(tiles * b * hkv), kThreads, DkdvSmem<HD>::kBytes, st>>>(mq, mk, mv, mo, p);
    UL_TRY(launched("attn_bwd_dkdv_sm100"));
  }
  if (stages & 4) {
    bwd_dq_kernel<HD><<<(unsigned)(tiles * b * hq), kThreads, DqSmem<HD>::kBytes, st>>>(mq, mk, mv, mo, p);
    UL_TRY(launched("attn_bwd_dq_sm100"));
  }
  return UL_OK;
}

}  // namespace bwd

size_t sm100_bwd_workspace(int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd) {
  (void)hkv;
  (void)hd;
  return (size_t)2 * b * hq * bwd::pad_n(n) * sizeof(float);
}

int sm100_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
              void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, int64_t n, int64_t b, int64_t hq,
              int64_t hkv, int64_t hd, int causal, float scale, int stages, cudaStream_t st) {
  (void)ws_bytes;
  if (n > INT32_MAX / 2) return fail(UL_ERR_SHAPE, "attention: sequence too long (n=%lld)", (long long)n);
  switch (hd) {
    case 64: return bwd::launch<64>(q, k, v, o, dout, lse, dq, dk, dv, ws, n, b, hq, hkv, causal, scale, stages, st);
    case 128: return bwd::launch<128>(q, k, v, o, dout, lse, dq, dk, dv, ws, n, b, hq, hkv, causal, scale, stages, st);
    default:
      return fail(UL_ERR_KERNEL, "bf16 attention supports head_dim 64 or 128, got %lld", (long long)hd);
  }
}

}  // namespace ul
