// K3: FlashAttention-style forward on sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces the per-head kernel loop of ulysses_attention_forward_with_state
// (ulysses.py:148-152) over _masked_attention (kernels.py:31-40: scores =
// q k^T * scale, row_softmax tensor.py:227-249, ctx = probs v) and adds the
// row LSE the backward needs (the reference recomputes probabilities
// instead, kernels.py:104).
//
// One CTA = one 128-row query tile of one (batch, head); 6 warps:
//   warp 0  TMA producer: Q once, then K_j / V_j into a 2-stage ring
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer:
//             S_j = Q K_j^T   (SS, both K-major, M=128 N=128, -> TMEM S[j&1])
//             O  += P_j V_j   (TS: P from TMEM, V MN-major from smem)
//   warps 2-5 softmax: one query row per thread (TMEM lane == row); online
//             softmax in the exp2 domain with lazy rescaling (O in TMEM is
//             only corrected when the running max grows by > 2^8), P written
//             back to TMEM as packed bf16 over the consumed S columns.
// Causal tiles beyond the diagonal are skipped; the diagonal and the
// sequence tail are masked in registers.  CTAs are ordered longest-first.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace ul {
namespace fwd {

using namespace sm100;

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int NS = 2;               // K/V pipeline stages
constexpr int kThreads = 192;
constexpr float kLazy = 8.0f;       // log2 headroom before O is rescaled

template <int HD>
struct Smem {
  static constexpr int kAtom = 128 * 128;          // one SW128 atom column: 128 rows x 128 B
  static constexpr int kTile = (HD / 64) * kAtom;  // 128 x HD bf16
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + kTile;
  static constexpr int kV = kK + NS * kTile;
  static constexpr int kBar = kV + NS * kTile;
  static constexpr int kBytes = kBar + 256 + 1024;  // + barriers + alignment slack
};

struct Params {
  int n, b, hq, hkv;
  int causal;
  int qtiles;
  float scale_log2;   // scale * log2(e)
  __nv_bfloat16* o;
  float* lse;
};

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const Params p) {
  using S = Smem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;            // [NS]
  uint64_t* k_empty = bars + 1 + NS;      // [NS]
  uint64_t* v_full = bars + 1 + 2 * NS;   // [NS]
  uint64_t* v_empty = bars + 1 + 3 * NS;  // [NS]
  uint64_t* s_full = bars + 1 + 4 * NS;   // [2]
  uint64_t* p_full = bars + 3 + 4 * NS;   // [2]
  uint64_t* o_done = bars + 5 + 4 * NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6 + 4 * NS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // work item: longest (causal) query tiles first
  const int heads = p.b * p.hq;
  const int qt = p.qtiles - 1 - (int)(blockIdx.x / heads);
  const int bh = (int)(blockIdx.x % heads);
  const int bb = bh / p.hq;
  const int h = bh % p.hq;
  const int g = h / (p.hq / p.hkv);
  const int q0 = qt * BM;
  const int nkv_all = (p.n + BN - 1) / BN;
  const int nkv = p.causal ? min(nkv_all, (q0 + BM - 1) / BN + 1) : nkv_all;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 128);
    }
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tS[2] = {tbase, tbase + 128};
  const uint32_t tO = tbase + 256;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_expect_tx(q_full, BM * HD * 2);
#pragma unroll
      for (int a = 0; a < HD / 64; ++a) tma_load_3d(sQ + a * S::kAtom, &tmQ, q_full, a * 64, bb * p.hq + h, q0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % NS;
        const uint32_t ph = (j / NS) & 1;
        mbar_wait(&k_empty[s], ph ^ 1);
        mbar_expect_tx(&k_full[s], BN * HD * 2);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a)
          tma_load_3d(sK + s * S::kTile + a * S::kAtom, &tmK, &k_full[s], a * 64, bb * p.hkv + g, j * BN);
        mbar_wait(&v_empty[s], ph ^ 1);
        mbar_expect_tx(&v_full[s], BN * HD * 2);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a)
          tma_load_3d(sV + s * S::kTile + a * S::kAtom, &tmV, &v_full[s], a * 64, bb * p.hkv + g, j * BN);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t kIdQK = idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t kIdPV = idesc_bf16(BM, HD, 0, 1);
      const uint32_t qaddr = smem_u32(sQ);
      auto issue_pv = [&](int i) {
        const int s = i % NS;
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);
        mbar_wait(&v_full[s], (i / NS) & 1);
        tc_fence_after();
        const uint32_t vaddr = smem_u32(sV + s * S::kTile);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t bdesc = sdesc(vaddr + kk * 2048, S::kAtom, 1024);
          mma_ts(tO, tS[i & 1] + kk * 8, bdesc, kIdPV, (i > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&v_empty[s]);
        mma_commit(o_done);
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % NS;
        if (j >= 2) mbar_wait(o_done, (j - 2) & 1);  // P_{j-2} consumed -> S buffer free
        mbar_wait(&k_full[s], (j / NS) & 1);
        tc_fence_after();
        const uint32_t kaddr = smem_u32(sK + s * S::kTile);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t koff = (kk >> 2) * S::kAtom + (kk & 3) * 32;
          mma_ss(tS[j & 1], sdesc(qaddr + koff, 16, 1024), sdesc(kaddr + koff, 16, 1024), kIdQK,
                 kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[j & 1]);
        mma_commit(&k_empty[s]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(nkv - 1);
    }
  } else {
    // ---------------- softmax / correction / epilogue (warps 2..5) ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int qrow = q0 + row;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int kv0 = j * BN;
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t r[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS[j & 1] + lane_off + c * 32, r + c * 32);
      tmem_wait_ld();
      // mask only the diagonal (causal) and sequence-tail tiles; the branch is
      // uniform across the CTA
      if ((p.causal && kv0 + BN - 1 > q0) || kv0 + BN > p.n) {
        int limit = p.n - kv0;
        if (p.causal) limit = min(limit, qrow - kv0 + 1);
#pragma unroll
        for (int c = 0; c < BN; ++c)
          if (c >= limit) r[c] = __float_as_uint(-INFINITY);
      }
      // row max of the raw scores: 4 independent chains (ILP), then scaled
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < BN; c += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mx[u] = fmaxf(mx[u], __uint_as_float(r[c + u]));
      }
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
      float alpha = 1.f;
      bool rescale = false;
      if (mt > m + kLazy) {
        alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mt);
        rescale = (j > 0);
        m = mt;
      }
      const float mu = (m == -INFINITY) ? 0.f : m;
      // p = 2^(s*scale*log2e - m): one FFMA + MUFU.EX2 per element; the row
      // sum runs in 8 independent partial sums
      float rsum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t pk[BN / 2];
#pragma unroll
      for (int c = 0; c < BN; c += 2) {
        const float e0 = fast_exp2(fmaf(__uint_as_float(r[c]), p.scale_log2, -mu));
        const float e1 = fast_exp2(fmaf(__uint_as_float(r[c + 1]), p.scale_log2, -mu));
        rsum[(c >> 1) & 7] += e0 + e1;
        pk[c / 2] = pack_bf16(e0, e1);
      }
      const float rs = ((rsum[0] + rsum[1]) + (rsum[2] + rsum[3])) + ((rsum[4] + rsum[5]) + (rsum[6] + rsum[7]));
      l = l * alpha + rs;
      // P_j over the consumed S_j columns [0, BN/2)
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) tmem_st32(tS[j & 1] + lane_off + c * 32, pk + c * 32);
      // tcgen05.ld/st are warp-collective: rescale if any row of the warp
      // needs it (rows that do not keep alpha == 1)
      if (__any_sync(0xffffffffu, rescale)) {
        // O must hold the complete sum through PV_{j-1} before it is rescaled
        mbar_wait(o_done, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t ov[32];
          tmem_ld32(tO + lane_off + c * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 32; ++x) ov[x] = __float_as_uint(__uint_as_float(ov[x]) * alpha);
          tmem_st32(tO + lane_off + c * 32, ov);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[j & 1]);
    }
    // epilogue: O / l -> bf16 rows, LSE (natural log)
    mbar_wait(o_done, (nkv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const bool valid = qrow < p.n;
    __nv_bfloat16* orow = p.o + (((int64_t)qrow * p.b + bb) * p.hq + h) * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t ov[32];
      tmem_ld32(tO + lane_off + c * 32, ov);
      tmem_wait_ld();
      uint32_t pkd[16];
#pragma unroll
      for (int x = 0; x < 16; ++x)
        pkd[x] = pack_bf16(__uint_as_float(ov[2 * x]) * inv, __uint_as_float(ov[2 * x + 1]) * inv);
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
        for (int x = 0; x < 4; ++x) dst[x] = make_uint4(pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
      }
    }
    if (valid) p.lse[((int64_t)bb * p.hq + h) * p.n + qrow] = (m + log2f(l)) * 0.69314718055994531f;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int HD>
static int launch(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n, int64_t b,
                  int64_t hq, int64_t hkv, int causal, float scale, cudaStream_t st) {
  CUtensorMap mq, mk, mv;
  UL_TRY(make_tmap_bhsd(&mq, q, n, b * hq, HD, 128));
  UL_TRY(make_tmap_bhsd(&mk, k, n, b * hkv, HD, 128));
  UL_TRY(make_tmap_bhsd(&mv, v, n, b * hkv, HD, 128));
  Params p;
  p.n = (int)n;
  p.b = (int)b;
  p.hq = (int)hq;
  p.hkv = (int)hkv;
  p.causal = causal;
  p.qtiles = (int)((n + BM - 1) / BM);
  p.scale_log2 = scale * 1.4426950408889634f;
  p.o = (__nv_bfloat16*)o;
  p.lse = lse;
  const int smem = Smem<HD>::kBytes;
  static bool attr = false;
  if (!attr) {
    UL_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  const int64_t grid = (int64_t)p.qtiles * b * hq;
  attn_fwd_kernel<HD><<<(unsigned)grid, kThreads, smem, st>>>(mq, mk, mv, p);
  return launched("attn_fwd_sm100");
}

}  // namespace fwd

int preload_fwd() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_kernel<64>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_kernel<128>));
  return UL_OK;
}

int sm100_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n, int64_t b,
              int64_t hq, int64_t hkv, int64_t hd, int causal, float scale, cudaStream_t st) {
  if (n == 0 || b == 0 || hq == 0) return UL_OK;
  if (n > INT32_MAX / 2 || b * hq > 65535 * 1024)
    return fail(UL_ERR_SHAPE, "attention: sequence/head extents too large (n=%lld)", (long long)n);
  switch (hd) {
    case 64: return fwd::launch<64>(q, k, v, o, lse, n, b, hq, hkv, causal, scale, st);
    case 128: return fwd::launch<128>(q, k, v, o, lse, n, b, hq, hkv, causal, scale, st);
    default:
      return fail(UL_ERR_KERNEL, "bf16 attention supports head_dim 64 or 128, got %lld", (long long)hd);
  }
}

}  // namespace ul
