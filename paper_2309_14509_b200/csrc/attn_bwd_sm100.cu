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
//   bwd_dkdv   one CTA per (128-row kv tile, kv head); loops over the
//              group's query heads and the visible 64-row query sub-tiles.
//              S^T = K Q^T and dP^T = V dO^T (SS, M = 128 kv rows, N = 64)
//              go to one of two TMEM buffers; softmax warps (thread = kv
//              row) write P^T / dS^T back over them as bf16; dV += P^T dO
//              and dK += dS^T Q are TS MMAs.  Double-buffered TMEM lets the
//              MMAs of sub-tile i+1 run while the softmax of sub-tile i does.
//   bwd_dq     one CTA per (128-row query tile, head): Q and dO resident in
//              TMEM (A operands), 64-row kv sub-tiles streamed by TMA,
//              S = Q K^T, dP = dO V^T (double-buffered), dS -> TMEM,
//              dQ += dS K; all MMAs read only B from shared memory.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstring>

#include "comm.cuh"
#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace ul {
namespace bwd {

// Pipeline trace (profiling builds only, -DUL_TRACE): clock64 stamps of the
// hand-off points of the first 8 CTAs, [cta][16 events][sub-tile].
#ifdef UL_TRACE
__device__ unsigned long long g_trace[8 * 16 * 256];
// per-CTA life: [cta][0 start, 1 first operands, 2 q_done/epilogue, 3 end (globaltimer ns), 4 smid,
// 5/6 clock64 at start/end]
__device__ unsigned long long g_cta[8192 * 7];
#define UL_CTA(k, v) g_cta[blockIdx.x * 7 + (k)] = (v)
// per-warp arrival stamps of CTA 0 (fused kernel): [warp][sub-tile]
__device__ unsigned long long g_warp[32 * 256];
#define UL_WARP(it)                                                                     \
  do {                                                                                  \
    if (blockIdx.x == 0 && (it) < 256 && (threadIdx.x & 31) == 0) g_warp[(threadIdx.x >> 5) * 256 + (it)] = clock64(); \
  } while (0)
#define UL_EV(ev, j)                                                                      \
  do {                                                                                    \
    if (blockIdx.x < 8 && (j) < 256) g_trace[(blockIdx.x * 16 + (ev)) * 256 + (j)] = clock64(); \
  } while (0)
#else
#define UL_EV(ev, j) \
  do {               \
  } while (0)
#define UL_CTA(k, v) \
  do {               \
  } while (0)
#define UL_WARP(it) \
  do {              \
  } while (0)
#endif

using namespace sm100;

constexpr int BT = 128;           // the tile a CTA owns (kv tile for dkdv, q tile for dq)
constexpr int BS = 64;            // the sub-tile streamed against it
constexpr int NST = 4;            // streamed-operand pipeline stages
// dQ kernel softmax: two warps per TMEM lane quarter, each owning one
// 32-column half of the 64-column sub-tile, so every SMSP interleaves two
// independent softmax streams
constexpr int kSoftWarps = 8;
constexpr int kSoftThreads = kSoftWarps * 32;
// dK/dV kernel: 16 softmax warps, four per TMEM lane quarter, each owning 16
// of the sub-tile's 64 columns: the softmax is latency-bound, so twice the
// warps halve its critical path (launch bound 640 keeps the register budget
// at <= 102/thread, which five resident warps per SMSP require)
constexpr int kDkSoftWarps = 16;
constexpr int kDkThreads = 64 + kDkSoftWarps * 32;
__device__ __forceinline__ uint32_t a_col16(int kk) { return kk * 16 + 8; }
#ifdef UL_DQ_POLY
constexpr bool kDqPoly = true;   // a quarter of the unmasked exponentials on the FMA pipe
#else
constexpr bool kDqPoly = false;
#endif
#ifdef UL_DK_NOPOLY
constexpr bool kDkPoly = false;
#else
constexpr bool kDkPoly = true;
#endif   // half of the unmasked exponentials on the FMA pipe
constexpr int kAtomT = BT * 128;  // SW128 atom column of a 128-row tile (16 KB)
constexpr int kAtomS = BS * 128;  // ... of a 64-row sub-tile (8 KB)

// TMEM column of the bf16 A operand (P^T, dS^T or dS) for K-step kk (16
// elements = 8 packed columns): softmax half h packs its 32 elements into
// columns [32h + 16, 32h + 32) of the buffer it read them from.
__device__ __forceinline__ uint32_t a_col(int kk) { return (kk >> 1) * 32 + 16 + (kk & 1) * 8; }

// P = 2^(S*scale_log2 - L) for an element pair, packed f32x2 FMA (sm_100).
// kPoly evaluates the exponentials on the FMA pipe instead of the MUFU: the
// softmax phases run in bursts (every warp starts on the same s_full) that
// are MUFU-throughput bound, so a share of FMA-pipe exponentials shortens
// them.  Only for unmasked elements (poly_exp2 needs finite input).
template <bool kPoly = false>
__device__ __forceinline__ float2 pexp2(const uint32_t* r, float2 sc, float2 nl) {
  const float2 a = __ffma2_rn(make_float2(__uint_as_float(r[0]), __uint_as_float(r[1])), sc, nl);
  if (kPoly) return poly_exp2x2(a);
  return make_float2(fast_exp2(a.x), fast_exp2(a.y));
}
// dS = P * (dP - D) for an element pair, packed to bf16
__device__ __forceinline__ uint32_t pds(float2 e, const uint32_t* d, float2 nd) {
  const float2 t = __fmul2_rn(e, __fadd2_rn(make_float2(__uint_as_float(d[0]), __uint_as_float(d[1])), nd));
  return pack_bf16_op(t.x, t.y);
}

struct Params {
  int n, n_pad, b, hq, hkv;
  int causal;
  int head_major;   // CTA order: head-major once a head has a full wave of tiles
  float scale, scale_log2;
  const float* L2;   // [b*hq][n_pad] lse * log2(e), +inf padded
  const float* Dv;   // [b*hq][n_pad] rowsum(dO*O), 0 padded
  __nv_bfloat16* dq;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  // fused head->seq of dQ / dK / dV (active when P > 1): rows also go to
  // their destination rank's sequence layout; the dQ kernel (launched last)
  // publishes the call once all its CTAs and the dK/dV kernel are done
  PeerEpilogue ep_dq, ep_dk, ep_dv;
};

// ---- pre-pass ----------------------------------------------------------------
template <int HD>
__global__ void __launch_bounds__(256) bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                                       const __nv_bfloat16* __restrict__ dout,
                                                       const float* __restrict__ lse, float* __restrict__ L2,
                                                       float* __restrict__ Dv, int n, int n_pad, int b, int hq,
                                                       float* __restrict__ dq_acc) {
  // HD/8 threads per row, rows in memory order ((i*b + bb)*hq + h): every
  // warp streams contiguous 16-byte chunks of O and dO
  constexpr int TPR = HD / 8;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = tid / TPR;
  const int sub = (int)(tid % TPR);
  const int64_t rows = (int64_t)n * b * hq;
  float s = 0.f;
  if (r < rows) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(o + r * HD) + sub);
    const uint4 c = __ldg(reinterpret_cast<const uint4*>(dout + r * HD) + sub);
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* c2 = reinterpret_cast<const __nv_bfloat162*>(&c);
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const float2 fa = __bfloat1622float2(a2[x]), fc = __bfloat1622float2(c2[x]);
      s = fmaf(fa.x, fc.x, fmaf(fa.y, fc.y, s));
    }
  }
#pragma unroll
  for (int m = TPR / 2; m; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
  if (r < rows) {
    const int h = (int)(r % hq);
    const int64_t ib = r / hq;
    const int bb = (int)(ib % b), i = (int)(ib / b);
    const int64_t bh = (int64_t)bb * hq + h;
    if (sub == 0) {
      Dv[bh * n_pad + i] = s;
      L2[bh * n_pad + i] = lse[bh * n + i] * 1.4426950408889634f;
    }
    if (dq_acc) {   // fused backward: zero this row's slice of the fp32 dQ accumulator
      float4* z = reinterpret_cast<float4*>(dq_acc + (bh * n_pad + i) * HD + sub * 8);
      z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
      z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  // rows n..n_pad of every head: masked-out padding (P = 0, D = 0)
  const int pad = n_pad - n;
  if (pad > 0 && tid < (int64_t)b * hq * pad) {
    const int64_t bh = tid / pad;
    const int i = n + (int)(tid % pad);
    Dv[bh * n_pad + i] = 0.f;
    L2[bh * n_pad + i] = INFINITY;
  }
}

// TMEM epilogue: a 128-lane x HD fp32 accumulator -> bf16 rows (x mul).
// `peer` (or nullptr) is this row's slot in the destination rank's sequence
// layout: the fused head->seq exchange stores the same bytes there.
template <int HD>
__device__ __forceinline__ void store_acc_rows(uint32_t tacc, uint32_t lane_off, float mul, __nv_bfloat16* dst,
                                               bool valid, char* peer = nullptr) {
#pragma unroll
  for (int c = 0; c < HD / 32; ++c) {
    uint32_t v[32];
    tmem_ld32(tacc + lane_off + c * 32, v);   // warp-collective: every lane executes it
    tmem_wait_ld();
    uint32_t pkd[16];
#pragma unroll
    for (int x = 0; x < 16; ++x)
      pkd[x] = pack_bf16(__uint_as_float(v[2 * x]) * mul, __uint_as_float(v[2 * x + 1]) * mul);
    if (valid) {
      uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
      for (int x = 0; x < 4; ++x) d4[x] = make_uint4(pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
      if (peer) {
        uint4* p4 = reinterpret_cast<uint4*>(peer) + c * 4;
#pragma unroll
        for (int x = 0; x < 4; ++x) p4[x] = make_uint4(pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
      }
    }
  }
}

// ---- dK / dV -----------------------------------------------------------------
template <int HD>
struct DkdvSmem {
  static constexpr int kTileT = (HD / 64) * kAtomT;   // 128 x HD
  static constexpr int kTileS = (HD / 64) * kAtomS;   // 64 x HD
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTileT;
  static constexpr int kQ = kV + kTileT;              // [NST]
  static constexpr int kO = kQ + NST * kTileS;        // dO [NST]
  static constexpr int kL = kO + NST * kTileS;        // [NST][BS] f32
  static constexpr int kD = kL + NST * BS * 4;        // [NST][BS] f32
  static constexpr int kBar = kD + NST * BS * 4;
  static constexpr int kBytes = kBar + 256 + 1024;
};

template <int HD>
__global__ void __launch_bounds__(640, 1)
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
  uint64_t* q_full = bars + 1;                 // [NST]
  uint64_t* q_empty = bars + 1 + NST;          // [NST]
  uint64_t* s_full = bars + 1 + 2 * NST;       // [2]
  uint64_t* p_full = bars + 3 + 2 * NST;       // [2]
  uint64_t* buf_free = bars + 5 + 2 * NST;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7 + 2 * NST);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // head-major: resident CTAs share one kv head's Q/dO stream in L2;
  // ascending kv tile == longest first (causal)
  const int ktiles = (p.n + BT - 1) / BT;
  const int kheads = p.b * p.hkv;
  const int kt = p.head_major ? (int)(blockIdx.x % ktiles) : (int)(blockIdx.x / kheads);
  const int bg = p.head_major ? (int)(blockIdx.x / ktiles) : (int)(blockIdx.x % kheads);
  const int bb = bg / p.hkv, g = bg % p.hkv;
  const int group = p.hq / p.hkv;
  const int kv0 = kt * BT;
  const int nsub = (p.n + BS - 1) / BS;
  const int i0 = p.causal ? kv0 / BS : 0;
  const int per_head = nsub - i0;
  const int total = per_head * group;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kDkSoftWarps);   // one arrive per softmax warp
      mbar_init(&buf_free[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();   // 512 columns = the whole TMEM: base is column 0
  constexpr uint32_t tbase = 0;
  // TMEM: S^T[2] at 0/64, dP^T[2] at 128/192, dV at 256, dK at 256+HD
  const uint32_t tdV = tbase + 256, tdK = tbase + 256 + HD;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
      mbar_expect_tx(kv_full, 2 * BT * HD * 2);
#pragma unroll
      for (int a = 0; a < HD / 64; ++a) {
        tma_load_3d(sK + a * kAtomT, &tmK, kv_full, a * 64, bb * p.hkv + g, kv0);
        tma_load_3d(sV + a * kAtomT, &tmV, kv_full, a * 64, bb * p.hkv + g, kv0);
      }
      for (int it = 0; it < total; ++it) {
        const int h = g * group + it / per_head;
        const int qi = i0 + it % per_head;
        const int s = it % NST;
        mbar_wait(&q_empty[s], ((it / NST) & 1) ^ 1);
        UL_EV(8, it);
        mbar_expect_tx(&q_full[s], 2 * BS * HD * 2 + 2 * BS * 4);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a) {
          tma_load_3d(sQ + s * S::kTileS + a * kAtomS, &tmQ, &q_full[s], a * 64, bb * p.hq + h, qi * BS);
          tma_load_3d(sO + s * S::kTileS + a * kAtomS, &tmO, &q_full[s], a * 64, bb * p.hq + h, qi * BS);
        }
        const int64_t roff = ((int64_t)bb * p.hq + h) * p.n_pad + qi * BS;
        bulk_load(sL + s * BS, p.L2 + roff, BS * 4, &q_full[s]);
        bulk_load(sD + s * BS, p.Dv + roff, BS * 4, &q_full[s]);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {  // one thread issues every MMA (uniform operands)
      constexpr uint32_t kIdS = idesc_bf16(BT, BS, 0, 0);   // M = kv rows, N = 64 q rows
      constexpr uint32_t kIdG = idesc_bf16(BT, HD, 0, 1);   // M = kv rows, N = hd, B MN-major
      // base descriptors, built once: K/V (K-major A), Q/dO stage 0 as
      // K-major B (for S^T, dP^T) and as MN-major B (for dK, dV)
      const uint64_t dK0 = sdesc(smem_u32(sK), 16, 1024), dV0 = sdesc(smem_u32(sV), 16, 1024);
      const uint64_t dQk0 = sdesc(smem_u32(sQ), 16, 1024), dOk0 = sdesc(smem_u32(sO), 16, 1024);
      const uint64_t dQm0 = sdesc(smem_u32(sQ), kAtomS, 1024), dOm0 = sdesc(smem_u32(sO), kAtomS, 1024);
      auto issue_grads = [&](int i) {
        const int b = i & 1, s = i % NST;
        const uint32_t tSt = tbase + b * 64, tdPt = tbase + 128 + b * 64;
        mbar_wait_mma(&p_full[b], (i >> 1) & 1);
        UL_EV(1, i);
        tc_fence_after();
        const uint64_t dOm = dadd(dOm0, s * S::kTileS), dQm = dadd(dQm0, s * S::kTileS);
#pragma unroll
        for (int kk = 0; kk < BS / 16; ++kk)
          mma_ts(tdV, tSt + a_col16(kk), dadd(dOm, kk * 2048), kIdG, (i > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < BS / 16; ++kk)
          mma_ts(tdK, tdPt + a_col16(kk), dadd(dQm, kk * 2048), kIdG, (i > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&q_empty[s]);
        mma_commit(&buf_free[b]);
        UL_EV(6, i);
      };
      mbar_wait_mma(kv_full, 0);
      for (int it = 0; it < total; ++it) {
        const int b = it & 1, s = it % NST;
        const uint32_t tSt = tbase + b * 64, tdPt = tbase + 128 + b * 64;
        // buffer b was last read by grads(it-2), issued before this point by
        // this thread: tcgen05.mma executes in issue order, so no wait
        UL_EV(10, it);
        mbar_wait_mma(&q_full[s], (it / NST) & 1);
        UL_EV(0, it);
        tc_fence_after();
        const uint64_t dQk = dadd(dQk0, s * S::kTileS), dOk = dadd(dOk0, s * S::kTileS);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t offT = (kk >> 2) * kAtomT + (kk & 3) * 32;
          const uint32_t offS = (kk >> 2) * kAtomS + (kk & 3) * 32;
          mma_ss(tSt, dadd(dK0, offT), dadd(dQk, offS), kIdS, kk > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t offT = (kk >> 2) * kAtomT + (kk & 3) * 32;
          const uint32_t offS = (kk >> 2) * kAtomS + (kk & 3) * 32;
          mma_ss(tdPt, dadd(dV0, offT), dadd(dOk, offS), kIdS, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[b]);
        UL_EV(7, it);
        if (it >= 1) issue_grads(it - 1);
      }
      issue_grads(total - 1);
    }
    __syncwarp();
  } else {
    const int quarter = warp & 3;
    const int part = (warp - 2) >> 2;        // which 16-column quarter of the sub-tile
    const int row = quarter * 32 + lane;     // kv row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int kvrow = kv0 + row;
    const int c0 = part * 16;
    const float2 sc = make_float2(p.scale_log2, p.scale_log2);
    for (int it = 0; it < total; ++it) {
      const int b = it & 1, s = it % NST;
      const int q0 = (i0 + it % per_head) * BS;
      const uint32_t tSt = tbase + b * 64, tdPt = tbase + 128 + b * 64;
      mbar_wait(&q_full[s], (it / NST) & 1);
      // per-column -LSE / -D of these 16 columns (broadcast 16-byte smem
      // reads), fetched while S^T/dP^T are still being computed
      float2 nl[8], nd[8];
      {
        const uint32_t la = smem_u32(sL + s * BS + c0), da = smem_u32(sD + s * BS + c0);
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const float4 a = lds_f4(la + 16 * x), e = lds_f4(da + 16 * x);
          nl[2 * x] = make_float2(-a.x, -a.y);
          nl[2 * x + 1] = make_float2(-a.z, -a.w);
          nd[2 * x] = make_float2(-e.x, -e.y);
          nd[2 * x + 1] = make_float2(-e.z, -e.w);
        }
      }
      mbar_wait(&s_full[b], (it >> 1) & 1);
      if (lane == 0 && (warp == 2 || warp == 9)) UL_EV(warp == 2 ? 2 : 4, it);
      tc_fence_after();
      uint32_t r[16], d[16];
      tmem_ld16(tSt + lane_off + c0, r);
      tmem_ld16(tdPt + lane_off + c0, d);
      tmem_wait_ld();
#ifdef UL_TRACE
      {
        uint32_t dep;   // the stamp must follow the loaded data (LDTM completes by scoreboard)
        asm volatile("add.u32 %0, %1, %2;" : "=r"(dep) : "r"(r[0]), "r"(d[15]));
        if (lane == 0 && warp == 2 && dep != 0x7fffffffu) UL_EV(12, it);
        asm volatile("mov.b32 %0, %1;" : "=r"(dep) : "f"(nl[7].y + nd[7].y));
        if (lane == 0 && warp == 2 && dep != 0x7fffffffu) UL_EV(15, it);
      }
#endif
      uint32_t pk[8], dsk[8];
      // only sub-tiles overlapping the kv tile's diagonal need the causal mask
      if (p.causal && q0 + c0 < kv0 + BT) {
        const int first = kvrow - q0 - c0;   // columns x < first are masked (q < kv)
#pragma unroll
        for (int x = 0; x < 16; x += 2) {
          float2 e = pexp2(r + x, sc, nl[x / 2]);
          e.x = x < first ? 0.f : e.x;
          e.y = x + 1 < first ? 0.f : e.y;
          pk[x / 2] = pack_bf16_op(e.x, e.y);
          dsk[x / 2] = pds(e, d + x, nd[x / 2]);
        }
      } else {
#pragma unroll
        for (int x = 0; x < 16; x += 2) {
          const float2 e = (x & 2) ? pexp2<kDkPoly>(r + x, sc, nl[x / 2]) : pexp2(r + x, sc, nl[x / 2]);
          pk[x / 2] = pack_bf16_op(e.x, e.y);
          dsk[x / 2] = pds(e, d + x, nd[x / 2]);
        }
      }
      // packed P^T / dS^T of these 16 columns go to the upper 8 of the 16
      // columns this warp just consumed; the TS MMAs address K-step kk at
      // a_col16(kk)
      if (lane == 0 && warp == 2) UL_EV(14, it);
      tmem_st8(tSt + lane_off + c0 + 8, pk);
      tmem_st8(tdPt + lane_off + c0 + 8, dsk);
      tmem_wait_st();
      tc_fence_before();
      if (lane == 0 && (warp == 2 || warp == 9)) UL_EV(warp == 2 ? 3 : 5, it);
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
    }
    // epilogue: parts 0/1 store the two column halves of dV, parts 2/3 of
    // dK * scale (bf16 rows of kv head g)
    mbar_wait(&buf_free[(total - 1) & 1], ((total - 1) >> 1) & 1);
    tc_fence_after();
    const bool valid = kvrow < p.n;
    const int64_t off = (((int64_t)kvrow * p.b + bb) * p.hkv + g) * HD;
    const bool is_dk = part >= 2;
    const int col0 = (part & 1) * (HD / 2);
    const PeerEpilogue& ep = is_dk ? p.ep_dk : p.ep_dv;
    char* peer = (ep.active && valid) ? peer_row_ptr(ep, kvrow, bb, p.b, g, HD, 2) + col0 * 2 : nullptr;
    if (!is_dk) store_acc_rows<HD / 2>(tdV + col0, lane_off, 1.f, p.dv + off + col0, valid, peer);
    else store_acc_rows<HD / 2>(tdK + col0, lane_off, p.scale, p.dk + off + col0, valid, peer);
    if (ep.active) __threadfence_system();   // dQ kernel signals after this launch completes
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
// One CTA per (128-row query tile, head).  Q and dO are the A operands of
// S = Q K^T and dP = dO V^T and stay resident for the CTA's whole kv loop,
// so they live in TMEM (loaded once by the softmax warps with tcgen05.st):
// every MMA then reads only its B operand from shared memory.  (As SS MMAs
// with N = 64 they read (128+64)*32 B of smem per 32 tensor cycles -- more
// than the smem port delivers -- and ran at ~2/3 rate.)
// TMEM: Q 0..63 | dO 64..127 | S[2] 128/192 | dP[2] 256/320 (dS over dP) | dQ 384..511.
// warp 0 TMA, warp 1 S/dP MMA, warp 2 dQ MMA, warps 3..10 softmax
constexpr int kDqThreads = 96 + kSoftThreads;
constexpr int KNST = 6;   // K/V sub-tile stages (a stage is held ~2 sub-tiles: S/dP, then dQ)

template <int HD>
struct DqSmem {
  static constexpr int kTileS = (HD / 64) * kAtomS;
  static constexpr int kK = 0;                     // [KNST]
  static constexpr int kV = kK + KNST * kTileS;    // [KNST]
  static constexpr int kBar = kV + KNST * kTileS;
  static constexpr int kBytes = kBar + 256 + 1024;
};

// Query tile k of this (persistent) CTA.  Tiles are ranked longest first
// (causal) -- pair-major, or head-major for long sequences -- and dealt to
// the CTAs in waves, zig-zagging the order every other wave so the per-CTA
// sums of tile lengths balance.
struct DqTile {
  int bb, h, g, q0, nsub;
};
__device__ __forceinline__ bool dq_tile(const Params& p, int k, DqTile& t) {
  const int qtiles = (p.n + BT - 1) / BT;
  const int qheads = p.b * p.hq;
  const int G = (int)gridDim.x;
  const int idx = k * G + ((k & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
  if (idx >= qtiles * qheads) return false;
  const int qt = qtiles - 1 - (p.head_major ? idx % qtiles : idx / qheads);
  const int bh = p.head_major ? idx / qtiles : idx % qheads;
  t.bb = bh / p.hq;
  t.h = bh % p.hq;
  t.g = t.h / (p.hq / p.hkv);
  t.q0 = qt * BT;
  const int nsub_all = (p.n + BS - 1) / BS;
  t.nsub = p.causal ? min(nsub_all, (t.q0 + BT - 1) / BS + 1) : nsub_all;
  return true;
}

// Half 0 of the softmax warps puts its row of Q, half 1 its row of dO, into
// TMEM as packed bf16 pairs (the A-operand layout: lane = row, column c
// holds elements 2c, 2c+1), then arrives on a_full.
template <int HD>
__device__ __forceinline__ void dq_load_rows(const Params& p, const DqTile& t, const __nv_bfloat16* q,
                                             const __nv_bfloat16* dout, int half, int row, uint32_t dst,
                                             uint64_t* a_full) {
  const int qrow = t.q0 + row;
  const bool valid = qrow < p.n;
  const __nv_bfloat16* src = (half == 0 ? q : dout) + (((int64_t)qrow * p.b + t.bb) * p.hq + t.h) * HD;
#pragma unroll
  for (int c = 0; c < HD / 64; ++c) {
    uint32_t w[32];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      uint4 v4 = valid ? __ldg(reinterpret_cast<const uint4*>(src + c * 64) + x) : make_uint4(0, 0, 0, 0);
      w[4 * x] = v4.x;
      w[4 * x + 1] = v4.y;
      w[4 * x + 2] = v4.z;
      w[4 * x + 3] = v4.w;
    }
    tmem_st32(dst + c * 32, w);
  }
  tmem_wait_st();
  tc_fence_before();
  mbar_arrive(a_full);
}

template <int HD>
__global__ void __launch_bounds__(kDqThreads, 1)
    bwd_dq_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ dout, const Params p) {
  static_assert(HD == 128 || HD == 64, "head dim");
  using S = DqSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* a_full = bars + 0;                 // Q and dO of the tile written to TMEM
  uint64_t* kv_full = bars + 1;                // [KNST]
  uint64_t* kv_empty = bars + 1 + KNST;        // [KNST]
  uint64_t* s_full = bars + 1 + 2 * KNST;      // [2] S(j) and dP(j) in TMEM
  uint64_t* s_free = bars + 3 + 2 * KNST;      // [2] S(j) read by every softmax warp
  uint64_t* p_full = bars + 5 + 2 * KNST;      // [2] dS(j) written over dP(j)
  uint64_t* dq_done = bars + 7 + 2 * KNST;     // [2] dQ(j) has read dS(j)
  uint64_t* q_done = bars + 9 + 2 * KNST;      // the tile's dQ accumulation is complete
  uint64_t* dq_free = bars + 10 + 2 * KNST;    // the epilogue has read dQ out of TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11 + 2 * KNST);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    UL_CTA(0, globaltimer());
    UL_CTA(4, smid());
    UL_CTA(5, clock64());
  }
  if (threadIdx.x == 0) {
    mbar_init(a_full, kSoftThreads);
    for (int s = 0; s < KNST; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], kSoftWarps);   // one arrive per softmax warp
      mbar_init(&p_full[s], kSoftWarps);
      mbar_init(&dq_done[s], 1);
    }
    mbar_init(q_done, 1);
    mbar_init(dq_free, kSoftWarps);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // a 512-column allocation owns the whole TMEM of the SM: its address is
  // column 0, lane 0.  Using the constant keeps every TMEM operand of the
  // MMA issue loop an immediate (no per-MMA register->uniform moves).
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tbase = 0;
  constexpr uint32_t tQ = tbase, tdO = tbase + 64, tdQ = tbase + 384;

  // Every role walks the same tile sequence; `gj` counts the CTA's sub-tiles
  // across tiles, so the K/V ring and the S/dP double buffer run on without
  // draining between tiles.
  DqTile t;
  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      int gj = 0;
      for (int k = 0; dq_tile(p, k, t); ++k) {
        for (int j = 0; j < t.nsub; ++j, ++gj) {
          const int s = gj % KNST;
          mbar_wait(&kv_empty[s], ((gj / KNST) & 1) ^ 1);
          UL_EV(8, gj);
          mbar_expect_tx(&kv_full[s], 2 * BS * HD * 2);
#pragma unroll
          for (int a = 0; a < HD / 64; ++a) {
            tma_load_3d(sK + s * S::kTileS + a * kAtomS, &tmK, &kv_full[s], a * 64, t.bb * p.hkv + t.g, j * BS);
            tma_load_3d(sV + s * S::kTileS + a * kAtomS, &tmV, &kv_full[s], a * 64, t.bb * p.hkv + t.g, j * BS);
          }
        }
      }
    }
  } else if (warp == 1) {
    // S/dP issuer.  S(j) only needs every softmax warp to have READ S(j-2)
    // (s_free); dP(j) overwrites dS(j-2), so it waits for dQ(j-2) to have
    // completed (dq_done, committed by the dQ issuer).  A second issuing
    // warp keeps this stream from stalling behind dQ's p_full waits: an
    // issuing thread blocks whenever the tensor queue is full, so one thread
    // cannot wait on one barrier while MMAs behind another are pending.
    if (elect_one()) {
      constexpr uint32_t kIdS = idesc_bf16(BT, BS, 0, 0);   // A (TMEM) x B K-major
      const uint64_t dKk0 = sdesc(smem_u32(sK), 16, 1024), dVk0 = sdesc(smem_u32(sV), 16, 1024);
      int gj = 0;
      for (int k = 0; dq_tile(p, k, t); ++k) {
        mbar_wait_mma(a_full, k & 1);
        for (int j = 0; j < t.nsub; ++j, ++gj) {
          const int b = gj & 1, s = gj % KNST;
          const uint32_t tS = tbase + 128 + b * 64, tdP = tbase + 256 + b * 64;
          UL_EV(10, gj);
          mbar_wait_mma(&kv_full[s], (gj / KNST) & 1);
          UL_EV(0, gj);
          if (gj == 0) UL_CTA(1, globaltimer());
          if (gj >= 2) mbar_wait_mma(&s_free[b], ((gj - 2) >> 1) & 1);
          UL_EV(9, gj);
          tc_fence_after();
          const uint64_t dKk = dadd(dKk0, s * S::kTileS), dVk = dadd(dVk0, s * S::kTileS);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t offS = (kk >> 2) * kAtomS + (kk & 3) * 32;
            mma_ts(tS, tQ + kk * 8, dadd(dKk, offS), kIdS, kk > 0 ? 1u : 0u);
          }
          UL_EV(13, gj);
          if (gj >= 2) {
            mbar_wait_mma(&dq_done[b], ((gj - 2) >> 1) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t offS = (kk >> 2) * kAtomS + (kk & 3) * 32;
            mma_ts(tdP, tdO + kk * 8, dadd(dVk, offS), kIdS, kk > 0 ? 1u : 0u);
          }
          mma_commit(&s_full[b]);
          UL_EV(7, gj);
        }
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // dQ issuer: dQ += dS(i) K(i) as soon as the softmax has written dS(i)
    if (elect_one()) {
      constexpr uint32_t kIdG = idesc_bf16(BT, HD, 0, 1);   // dS (TMEM) x K MN-major
      const uint64_t dKm0 = sdesc(smem_u32(sK), kAtomS, 1024);
      int gj = 0;
      for (int k = 0; dq_tile(p, k, t); ++k) {
        for (int i = 0; i < t.nsub; ++i, ++gj) {
          const int b = gj & 1, s = gj % KNST;
          const uint32_t tdP = tbase + 256 + b * 64;
          mbar_wait_mma(&p_full[b], (gj >> 1) & 1);
          UL_EV(1, gj);
          if (i == 0 && k > 0) mbar_wait_mma(dq_free, (k - 1) & 1);   // previous tile's dQ read out
          tc_fence_after();
          const uint64_t dKm = dadd(dKm0, s * S::kTileS);
#pragma unroll
          for (int kk = 0; kk < BS / 16; ++kk)
            mma_ts(tdQ, tdP + a_col(kk), dadd(dKm, kk * 2048), kIdG, (i > 0 || kk > 0) ? 1u : 0u);
          // S(i), dP(i) completed before the softmax produced dS(i): this
          // commit covers every read of K/V stage s
          mma_commit(&kv_empty[s]);
          mma_commit(&dq_done[b]);
          if (i == t.nsub - 1) mma_commit(q_done);
          UL_EV(6, gj);
        }
      }
    }
    __syncwarp();
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 3) >> 2;        // which 32-column half of the kv sub-tile
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int c0 = half * 32;
    const uint32_t a_dst = (half == 0 ? tQ : tdO) + lane_off;
    int gj = 0;
    bool have = dq_tile(p, 0, t);
    if (have) dq_load_rows<HD>(p, t, q, dout, half, row, a_dst, a_full);
    for (int k = 0; have; ++k) {
      const int qrow = t.q0 + row;
      const bool valid = qrow < p.n;
      const int64_t roff = ((int64_t)t.bb * p.hq + t.h) * p.n_pad + qrow;
      const float L = p.L2[roff];
      const float Dr = p.Dv[roff];
      const float2 sc = make_float2(p.scale_log2, p.scale_log2), nL = make_float2(-L, -L), nD = make_float2(-Dr, -Dr);
      for (int j = 0; j < t.nsub; ++j, ++gj) {
        const int b = gj & 1;
        const int kv0 = j * BS + c0;
        const uint32_t tS = tbase + 128 + b * 64, tdP = tbase + 256 + b * 64;
        mbar_wait(&s_full[b], (gj >> 1) & 1);
        if (lane == 0 && (warp == 3 || warp == 10)) UL_EV(warp == 3 ? 2 : 4, gj);
        tc_fence_after();
        // S(j) and dP(j) both land before s_full(j); once this warp has them in
        // registers the S buffer is released (S(j+2) may overwrite it), while
        // the dP buffer receives dS(j) in this warp's own columns
        uint32_t r[32], d[32];
        tmem_ld32(tS + lane_off + c0, r);
        tmem_ld32(tdP + lane_off + c0, d);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[b]);
        uint32_t dsk[16];
        if (p.causal && kv0 + 31 > t.q0) {     // only the diagonal sub-tiles need the mask
          const int limit = qrow - kv0 + 1;     // columns x >= limit are masked (kv > q)
#pragma unroll
          for (int x = 0; x < 32; x += 2) {
            float2 e = pexp2(r + x, sc, nL);
            e.x = x >= limit ? 0.f : e.x;
            e.y = x + 1 >= limit ? 0.f : e.y;
            dsk[x / 2] = pds(e, d + x, nD);
          }
        } else {
#pragma unroll
          for (int x = 0; x < 32; x += 2)
            dsk[x / 2] = pds((kDqPoly && (x & 6) == 6) ? pexp2<true>(r + x, sc, nL) : pexp2(r + x, sc, nL), d + x, nD);
        }
        tmem_st16(tdP + lane_off + c0 + 16, dsk);   // dS over this warp's consumed dP columns
        tmem_wait_st();
        tc_fence_before();
        if (lane == 0 && (warp == 3 || warp == 10)) UL_EV(warp == 3 ? 3 : 5, gj);
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[b]);
      }
      // every S/dP MMA of this tile has completed (this warp saw the last
      // s_full): the next tile's Q/dO may replace them in TMEM, so its first
      // S/dP run under this tile's epilogue
      DqTile nt;
      have = dq_tile(p, k + 1, nt);
      if (have) dq_load_rows<HD>(p, nt, q, dout, half, row, a_dst, a_full);
      mbar_wait(q_done, k & 1);
      if (threadIdx.x == 96) UL_CTA(2, globaltimer());
      tc_fence_after();
      // each half stores HD/2 columns of dQ * scale
      __nv_bfloat16* dst = p.dq + (((int64_t)qrow * p.b + t.bb) * p.hq + t.h) * HD;
      uint32_t pkd[HD / 64][16];
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        uint32_t v[32];
        tmem_ld32(tdQ + lane_off + half * (HD / 2) + c * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < 16; ++x)
          pkd[c][x] = pack_bf16(__uint_as_float(v[2 * x]) * p.scale, __uint_as_float(v[2 * x + 1]) * p.scale);
      }
      // dQ is in registers: the accumulator may be overwritten by the next tile
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);
      if (valid) {
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          const int col = half * (HD / 2) + c * 32;
          uint4* d4 = reinterpret_cast<uint4*>(dst + col);
#pragma unroll
          for (int x = 0; x < 4; ++x)
            d4[x] = make_uint4(pkd[c][4 * x], pkd[c][4 * x + 1], pkd[c][4 * x + 2], pkd[c][4 * x + 3]);
          if (p.ep_dq.active) {   // fused head->seq of dQ
            uint4* p4 = reinterpret_cast<uint4*>(peer_row_ptr(p.ep_dq, qrow, t.bb, p.b, t.h, HD, 2) + col * 2);
#pragma unroll
            for (int x = 0; x < 4; ++x)
              p4[x] = make_uint4(pkd[c][4 * x], pkd[c][4 * x + 1], pkd[c][4 * x + 2], pkd[c][4 * x + 3]);
          }
        }
      }
      t = nt;
    }
    if (p.ep_dq.active) __threadfence_system();
  }
  tc_fence_before();
  __syncthreads();
  // last CTA publishes the fused dQ/dK/dV exchange (the dK/dV kernel ran before this launch)
  if (p.ep_dq.active && threadIdx.x == 0) peer_signal_last_cta(p.ep_dq, gridDim.x);
  if (threadIdx.x == 0) {
    UL_CTA(3, globaltimer());
    UL_CTA(6, clock64());
  }
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ---- fused dK / dV / dQ (default for hd 128) -----------------------------------
// One CTA per (128-row kv tile, kv head), like bwd_dkdv, but dQ comes out of
// the same pass instead of a second kernel that recomputes S and dP:
//   dQ^T(i) = K^T dS^T(i)      (M = hd, N = 64 query rows, K = 128 kv rows)
// is accumulated in the dP^T TMEM buffer of sub-tile i once the softmax has
// consumed it, drained by four warps (thread = hd column, 64 query rows) and
// added into an fp32 [b*hq][n_pad][hd] accumulator with coalesced
// red.global.add.f32 (one 128-byte line per warp instruction); a last pass
// scales it into bf16 dQ.  Five GEMMs of 2*128*64*hd per sub-tile instead of
// the seven of bwd_dkdv + bwd_dq, and half the exponentials.  The fp32
// additions from different kv tiles land in arrival order, so dQ is not
// bitwise reproducible run to run (tolerance-equal); UL_ATTN_DETERMINISTIC
// selects the two-kernel path whose results are bitwise stable.
//   dS^T(i) goes both to TMEM (A operand of dK += dS^T Q, as in bwd_dkdv) and
// to shared memory as a SWIZZLE_128B [kv][q] tile (MN-major B operand of
// the dQ^T MMA; the A operand K^T is the resident K tile read MN-major).
// warp 0 TMA, warp 1 MMA, warps 2-5 dQ drain, warps 6-21 softmax (4 per lane
// quarter, 16 columns each).
#ifndef UL_FU_COLS
#define UL_FU_COLS 16
#endif
constexpr int kFuCols = UL_FU_COLS;            // softmax columns per warp (of the 64-column sub-tile)
constexpr int kFuSoftWarps = 4 * (64 / kFuCols);
__device__ __forceinline__ uint32_t fu_acol(int kk) { return kFuCols == 16 ? a_col16(kk) : a_col(kk); }
// every exponential on the MUFU (r66: FMA-pipe share on the fused kernel's
// softmax -- which is off its critical path (r42) -- cost 1.4%)
constexpr bool kFuPoly = false;
// dK / dV epilogue through shared memory (the K / V tiles, free once every MMA
// has completed) and per-warp 32-row TMA stores instead of 16-byte row stores
#ifndef UL_BWD_TMA_EPI
#define UL_BWD_TMA_EPI 1
#endif
constexpr int kFuThreads = 64 + 128 + kFuSoftWarps * 32;
constexpr int FNST = 3;   // Q / dO / L / D stages
constexpr int NDS = 3;    // dS^T smem buffers: the softmax of sub-tile i writes while dQ^T(i-1), dQ^T(i-2) may still read

template <int HD>
struct FusedSmem {
  static constexpr int kTileT = (HD / 64) * kAtomT;   // 128 x HD
  static constexpr int kTileS = (HD / 64) * kAtomS;   // 64 x HD
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTileT;
  static constexpr int kQ = kV + kTileT;              // [FNST]
  static constexpr int kO = kQ + FNST * kTileS;       // dO [FNST]
  static constexpr int kDS = kO + FNST * kTileS;      // dS^T [NDS] (128 kv rows x 64 q, bf16, SW128)
  static constexpr int kL = kDS + NDS * kAtomT;       // [FNST][BS] f32
  static constexpr int kD = kL + FNST * BS * 4;       // [FNST][BS] f32
  static constexpr int kBar = kD + FNST * BS * 4;
  static constexpr int kBytes = kBar + 256 + 1024;
};

__device__ __forceinline__ void red_add_f32(float* addr, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_u4(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int HD>
__global__ void __launch_bounds__(kFuThreads, 1)
    bwd_fused_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                     const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmDV,
                     const Params p, float* __restrict__ dq_acc) {
  static_assert(HD == 128, "the dQ^T MMA uses M = head dim = 128");
  using S = FusedSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sO = smem + S::kO;
  uint8_t* sDS = smem + S::kDS;
  float* sL = reinterpret_cast<float*>(smem + S::kL);
  float* sD = reinterpret_cast<float*>(smem + S::kD);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;                  // [FNST]
  uint64_t* q_empty = bars + 1 + FNST;          // [FNST]
  uint64_t* s_full = bars + 1 + 2 * FNST;       // [2] S^T, dP^T in TMEM
  uint64_t* p_full = bars + 3 + 2 * FNST;       // [2] P^T, dS^T written (TMEM + smem)
  uint64_t* dq_full = bars + 5 + 2 * FNST;      // [2] dQ^T accumulated (and everything before it)
  uint64_t* dq_free = bars + 7 + 2 * FNST;      // [2] dQ^T read out of TMEM by the drain warps
  uint64_t* ds_free = bars + 9 + 2 * FNST;      // [NDS] dS^T smem buffer consumed
  uint64_t* dp_full = bars + 9 + NDS + 2 * FNST;  // [2] dP^T in TMEM (s_full: S^T only)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11 + NDS + 2 * FNST);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ktiles = (p.n + BT - 1) / BT;
  const int kheads = p.b * p.hkv;
  // CTA order: tile-major (every head's longest tiles first: LPT balance),
  // head-major (long sequences: L2 reuse of one head's Q/dO/dQ stream), or
  // tile-major within groups of head_major >= 2 heads (both, partially)
  int kt, bg;
  if (p.head_major == 1) {
    kt = (int)(blockIdx.x % ktiles);
    bg = (int)(blockIdx.x / ktiles);
  } else if (p.head_major >= 2) {
    const int G = p.head_major;
    const int grp = (int)(blockIdx.x / (ktiles * G)), rem = (int)(blockIdx.x % (ktiles * G));
    kt = rem / G;
    bg = grp * G + rem % G;
    if (bg >= kheads) return;   // partial last group (before any barrier or TMEM use)
  } else {
    kt = (int)(blockIdx.x / kheads);
    bg = (int)(blockIdx.x % kheads);
  }
  const int bb = bg / p.hkv, g = bg % p.hkv;
  const int group = p.hq / p.hkv;
  const int kv0 = kt * BT;
  const int nsub = (p.n + BS - 1) / BS;
  const int i0 = p.causal ? kv0 / BS : 0;
  const int per_head = nsub - i0;
  const int total = per_head * group;

  if (threadIdx.x == 0) {
    UL_CTA(0, globaltimer());
    UL_CTA(4, smid());
    UL_CTA(5, clock64());
  }
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < FNST; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&dp_full[s], 1);
      mbar_init(&p_full[s], kFuSoftWarps);
      mbar_init(&dq_full[s], 1);
      mbar_init(&dq_free[s], 4);
    }
    for (int s = 0; s < NDS; ++s) mbar_init(&ds_free[s], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tbase = 0;
  // TMEM: S^T[2] at 0/64 (P^T over it), dP^T[2] at 128/192 (dS^T over it, then
  // dQ^T of the same sub-tile), dV at 256, dK at 256 + HD
  const uint32_t tdV = tbase + 256, tdK = tbase + 256 + HD;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
      mbar_expect_tx(kv_full, 2 * BT * HD * 2);
#pragma unroll
      for (int a = 0; a < HD / 64; ++a) {
        tma_load_3d(sK + a * kAtomT, &tmK, kv_full, a * 64, bb * p.hkv + g, kv0);
        tma_load_3d(sV + a * kAtomT, &tmV, kv_full, a * 64, bb * p.hkv + g, kv0);
      }
      int h = g * group, qi = i0;
      for (int it = 0; it < total; ++it) {
        const int s = it % FNST;
        mbar_wait(&q_empty[s], ((it / FNST) & 1) ^ 1);
        UL_EV(8, it);
        mbar_expect_tx(&q_full[s], 2 * BS * HD * 2 + 2 * BS * 4);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a) {
          tma_load_3d(sQ + s * S::kTileS + a * kAtomS, &tmQ, &q_full[s], a * 64, bb * p.hq + h, qi * BS);
          tma_load_3d(sO + s * S::kTileS + a * kAtomS, &tmO, &q_full[s], a * 64, bb * p.hq + h, qi * BS);
        }
        const int64_t roff = ((int64_t)bb * p.hq + h) * p.n_pad + qi * BS;
        bulk_load(sL + s * BS, p.L2 + roff, BS * 4, &q_full[s]);
        bulk_load(sD + s * BS, p.Dv + roff, BS * 4, &q_full[s]);
        if (++qi == nsub) {
          qi = i0;
          ++h;
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t kIdS = idesc_bf16(BT, BS, 0, 0);   // S^T, dP^T: M = kv rows, N = 64 q rows
      constexpr uint32_t kIdG = idesc_bf16(BT, HD, 0, 1);   // dV, dK: M = kv rows, N = hd, B MN-major
      constexpr uint32_t kIdQ = idesc_bf16(HD, BS, 1, 1);   // dQ^T: M = hd, N = q rows, A and B MN-major
      const uint64_t dK0 = sdesc(smem_u32(sK), 16, 1024), dV0 = sdesc(smem_u32(sV), 16, 1024);
      const uint64_t dQk0 = sdesc(smem_u32(sQ), 16, 1024), dOk0 = sdesc(smem_u32(sO), 16, 1024);
      const uint64_t dQm0 = sdesc(smem_u32(sQ), kAtomS, 1024), dOm0 = sdesc(smem_u32(sO), kAtomS, 1024);
      const uint64_t dKt0 = sdesc(smem_u32(sK), kAtomT, 1024);    // K^T: MN-major A (hd contiguous)
      const uint64_t dDS0 = sdesc(smem_u32(sDS), kAtomT, 1024);   // dS^T: MN-major B (q contiguous)
      auto issue_grads = [&](int i) {
        const int b = i & 1, s = i % FNST;
        const uint32_t tSt = tbase + b * 64, tdPt = tbase + 128 + b * 64;
        mbar_wait_mma(&p_full[b], (i >> 1) & 1);
        UL_EV(1, i);
        tc_fence_after();
        const uint64_t dOm = dadd(dOm0, s * S::kTileS), dQm = dadd(dQm0, s * S::kTileS);
#pragma unroll
        for (int kk = 0; kk < BS / 16; ++kk)
          mma_ts(tdV, tSt + fu_acol(kk), dadd(dOm, kk * 2048), kIdG, (i > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < BS / 16; ++kk)
          mma_ts(tdK, tdPt + fu_acol(kk), dadd(dQm, kk * 2048), kIdG, (i > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&q_empty[s]);
        // dQ^T(i) over the dP^T / dS^T columns dK(i) just read (in-order pipe)
        const uint64_t dds = dadd(dDS0, (i % NDS) * kAtomT);
#ifndef UL_BWD_XP_NO_DQMMA   // (what-if flag, r2: no dQ^T GEMM -> only -1.3%; results wrong)
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk)
          mma_ss(tdPt, dadd(dKt0, kk * 2048), dadd(dds, kk * 2048), kIdQ, kk > 0 ? 1u : 0u);
#endif
        mma_commit(&dq_full[b]);
        mma_commit(&ds_free[i % NDS]);
        UL_EV(6, i);
      };
      mbar_wait_mma(kv_full, 0);
      UL_CTA(1, globaltimer());
      for (int it = 0; it < total; ++it) {
        const int b = it & 1, s = it % FNST;
        const uint32_t tSt = tbase + b * 64, tdPt = tbase + 128 + b * 64;
        UL_EV(10, it);
        mbar_wait_mma(&q_full[s], (it / FNST) & 1);
        UL_EV(0, it);
        tc_fence_after();
        const uint64_t dQk = dadd(dQk0, s * S::kTileS), dOk = dadd(dOk0, s * S::kTileS);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t offT = (kk >> 2) * kAtomT + (kk & 3) * 32;
          const uint32_t offS = (kk >> 2) * kAtomS + (kk & 3) * 32;
          mma_ss(tSt, dadd(dK0, offT), dadd(dQk, offS), kIdS, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[b]);   // the softmax starts on P while dP^T runs
        // dP^T(it) replaces dQ^T(it-2): wait until the drain warps have it
        if (it >= 2) {
          mbar_wait_mma(&dq_free[b], ((it - 2) >> 1) & 1);
          tc_fence_after();
        }
        UL_EV(9, it);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t offT = (kk >> 2) * kAtomT + (kk & 3) * 32;
          const uint32_t offS = (kk >> 2) * kAtomS + (kk & 3) * 32;
          mma_ss(tdPt, dadd(dV0, offT), dadd(dOk, offS), kIdS, kk > 0 ? 1u : 0u);
        }
        mma_commit(&dp_full[b]);
        UL_EV(7, it);
        if (it >= 1) issue_grads(it - 1);
      }
      if (total > 0) issue_grads(total - 1);
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---- dQ drain: thread = hd column, 64 query rows of sub-tile it ----
    const int quarter = warp & 3;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int d = quarter * 32 + lane;
    int h = g * group, qi = i0;
    for (int it = 0; it < total; ++it) {
      const int b = it & 1;
      const uint32_t tdPt = tbase + 128 + b * 64;
      mbar_wait(&dq_full[b], (it >> 1) & 1);
      if (lane == 0 && warp == 2) UL_EV(4, it);
      tc_fence_after();
      float* dst = dq_acc + (((int64_t)bb * p.hq + h) * p.n_pad + (int64_t)qi * BS) * HD + d;
      // both halves into registers first: the TMEM buffer goes back to the
      // MMA issuer (dP^T of sub-tile it+2) before the 64 atomics are issued
      uint32_t v[64];
      tmem_ld32(tdPt + lane_off, v);
      tmem_ld32(tdPt + lane_off + 32, v + 32);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dq_free[b]);
      UL_WARP(it);
      if (lane == 0 && warp == 2) UL_EV(11, it);
#ifndef UL_BWD_XP_NO_RED   // (what-if flag, r2: drop the dQ atomics -> -4.7%; results wrong)
#pragma unroll
      for (int c = 0; c < 64; ++c) red_add_f32(dst + c * HD, __uint_as_float(v[c]));
#else
      if (v[0] == 0x7fffffffu && v[63] == 0x7fffffffu) dst[0] = 0.f;
#endif
      if (lane == 0 && warp == 2) UL_EV(15, it);
      if (++qi == nsub) {
        qi = i0;
        ++h;
      }
    }
  } else {
    const int quarter = warp & 3;
    const int part = (warp - 6) >> 2;        // which kFuCols-column part of the sub-tile
    const int row = quarter * 32 + lane;     // kv row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const int kvrow = kv0 + row;
    const int c0 = part * kFuCols;
    const float2 sc = make_float2(p.scale_log2, p.scale_log2);
    // this thread's two 16-byte chunks of its dS^T row in a SWIZZLE_128B tile
    const uint32_t ds_row = smem_u32(sDS) + (row >> 3) * 1024 + (row & 7) * 128;
    const int chunk0 = part * (kFuCols / 8);   // 16-byte chunks of this row part
    int qi = i0;
    for (int it = 0; it < total; ++it) {
      const int b = it & 1, s = it % FNST;
      const int q0 = qi * BS;
      if (++qi == nsub) qi = i0;
      const uint32_t tSt = tbase + b * 64, tdPt = tbase + 128 + b * 64;
      mbar_wait(&q_full[s], (it / FNST) & 1);
      float2 nl[kFuCols / 2], nd[kFuCols / 2];
      {
        const uint32_t la = smem_u32(sL + s * BS + c0), da = smem_u32(sD + s * BS + c0);
#pragma unroll
        for (int x = 0; x < kFuCols / 4; ++x) {
          const float4 a = lds_f4(la + 16 * x), e = lds_f4(da + 16 * x);
          nl[2 * x] = make_float2(-a.x, -a.y);
          nl[2 * x + 1] = make_float2(-a.z, -a.w);
          nd[2 * x] = make_float2(-e.x, -e.y);
          nd[2 * x + 1] = make_float2(-e.z, -e.w);
        }
      }
      mbar_wait(&s_full[b], (it >> 1) & 1);
      if (lane == 0 && warp == 6) UL_EV(2, it);
      tc_fence_after();
      uint32_t r[kFuCols], dd[kFuCols];
      if constexpr (kFuCols == 16) tmem_ld16(tSt + lane_off + c0, r);
      else tmem_ld32(tSt + lane_off + c0, r);
      tmem_wait_ld();
      if (lane == 0 && warp == 6) UL_EV(12, it);
      // P first (S^T only); dS once dP^T has landed
      uint32_t pk[kFuCols / 2], dsk[kFuCols / 2];
      float2 e[kFuCols / 2];
      if (p.causal && q0 + c0 < kv0 + BT) {
        const int first = kvrow - q0 - c0;   // columns x < first are masked (q < kv)
#pragma unroll
        for (int x = 0; x < kFuCols; x += 2) {
          e[x / 2] = pexp2(r + x, sc, nl[x / 2]);
          e[x / 2].x = x < first ? 0.f : e[x / 2].x;
          e[x / 2].y = x + 1 < first ? 0.f : e[x / 2].y;
        }
      } else {
#pragma unroll
        for (int x = 0; x < kFuCols; x += 2)
          e[x / 2] = (x & 2) ? pexp2<kFuPoly>(r + x, sc, nl[x / 2]) : pexp2(r + x, sc, nl[x / 2]);
      }
#pragma unroll
      for (int x = 0; x < kFuCols / 2; ++x) pk[x] = pack_bf16(e[x].x, e[x].y);
      if constexpr (kFuCols == 16) tmem_st8(tSt + lane_off + c0 + 8, pk);
      else tmem_st16(tSt + lane_off + c0 + 16, pk);
      mbar_wait(&dp_full[b], (it >> 1) & 1);
      tc_fence_after();
      if constexpr (kFuCols == 16) tmem_ld16(tdPt + lane_off + c0, dd);
      else tmem_ld32(tdPt + lane_off + c0, dd);
      tmem_wait_ld();
#pragma unroll
      for (int x = 0; x < kFuCols / 2; ++x) dsk[x] = pds(e[x], dd + 2 * x, nd[x]);
      // dS^T row chunk -> shared memory for the dQ^T MMA (after dQ^T(it-NDS) read the buffer)
      if (lane == 0 && warp == 6) UL_EV(13, it);
      const int ib = it % NDS;
      if (it >= NDS) mbar_wait(&ds_free[ib], ((it - NDS) / NDS) & 1);
      if (lane == 0 && warp == 6) UL_EV(14, it);
      const uint32_t dsb = ds_row + ib * kAtomT;
#ifndef UL_BWD_XP_NO_DSSTS   // (what-if flag, r2: skip the dS^T smem tile -> -7%; results wrong.
                             //  Moving the copy to the drain warps, or after the p_full
                             //  arrival, made the kernel 37% / 2.6% slower: dQ^T then waits)
#pragma unroll
      for (int j = 0; j < kFuCols / 8; ++j)
        sts_u4(dsb + (((chunk0 + j) ^ (row & 7)) << 4), dsk[4 * j], dsk[4 * j + 1], dsk[4 * j + 2], dsk[4 * j + 3]);
#endif
      fence_proxy_async_smem();
      if constexpr (kFuCols == 16) tmem_st8(tdPt + lane_off + c0 + 8, dsk);
      else tmem_st16(tdPt + lane_off + c0 + 16, dsk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      UL_WARP(it);
      if (lane == 0 && (warp == 6 || warp == 21)) UL_EV(warp == 6 ? 3 : 5, it);
    }
    // epilogue: the first half of the parts stores dV, the second dK * scale
    // (four parts: two column halves each; two parts: all HD columns)
    if (total > 0) mbar_wait(&ds_free[(total - 1) % NDS], ((total - 1) / NDS) & 1);
    if (threadIdx.x == 192) UL_CTA(2, globaltimer());
    tc_fence_after();
    const bool valid = kvrow < p.n;
    const int64_t off = (((int64_t)kvrow * p.b + bb) * p.hkv + g) * HD;
    constexpr int kParts = 64 / kFuCols;
    constexpr int kEpCols = HD / (kParts / 2);
    const bool is_dk = part >= kParts / 2;
    const int col0 = (part % (kParts / 2)) * kEpCols;
    const PeerEpilogue& ep = is_dk ? p.ep_dk : p.ep_dv;
    if (UL_BWD_TMA_EPI && kEpCols == 64 && !ep.active) {
      // this warp's 32 rows x 64 columns -> one SWIZZLE_128B box (4 KB of the
      // K / V tiles) -> one TMA store; rows >= n are clipped by the tensor map
      uint8_t* stg = smem + S::kK + (warp - 6) * 4096;
      const uint32_t srow = smem_u32(stg) + lane * 128;
      const uint32_t tacc = (is_dk ? tdK : tdV) + col0 + lane_off;
      const float mul = is_dk ? p.scale : 1.f;
#pragma unroll
      for (int c = 0; c < kEpCols / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tacc + c * 32, v);
        tmem_wait_ld();
        uint32_t pkd[16];
#pragma unroll
        for (int x = 0; x < 16; ++x)
          pkd[x] = pack_bf16(__uint_as_float(v[2 * x]) * mul, __uint_as_float(v[2 * x + 1]) * mul);
#pragma unroll
        for (int x = 0; x < 4; ++x)
          sts_u4(srow + (((c * 4 + x) ^ (lane & 7)) << 4), pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(is_dk ? &tmDK : &tmDV, stg, col0, bb * p.hkv + g, kv0 + quarter * 32);
        bulk_commit();
        bulk_wait_read0();
      }
      __syncwarp();
    } else {
      char* peer = (ep.active && valid) ? peer_row_ptr(ep, kvrow, bb, p.b, g, HD, 2) + col0 * 2 : nullptr;
      if (!is_dk) store_acc_rows<kEpCols>(tdV + col0, lane_off, 1.f, p.dv + off + col0, valid, peer);
      else store_acc_rows<kEpCols>(tdK + col0, lane_off, p.scale, p.dk + off + col0, valid, peer);
      if (ep.active) __threadfence_system();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    UL_CTA(3, globaltimer());
    UL_CTA(6, clock64());
  }
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// dQ = scale * acc in bf16 rows of the head layout (+ the fused head->seq
// stores and, as the last launch of the backward, the exchange signal)
template <int HD>
__global__ void __launch_bounds__(256) bwd_dq_convert_kernel(const float* __restrict__ acc,
                                                             __nv_bfloat16* __restrict__ dq, int n, int n_pad, int b,
                                                             int hq, float scale, PeerEpilogue ep) {
  constexpr int TPR = HD / 8;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = tid / TPR;   // output row (i*b + bb)*hq + h
  const int sub = (int)(tid % TPR);
  if (r < (int64_t)n * b * hq) {
    const int h = (int)(r % hq);
    const int64_t ib = r / hq;
    const int bb = (int)(ib % b), i = (int)(ib / b);
    const float4* src = reinterpret_cast<const float4*>(acc + (((int64_t)bb * hq + h) * n_pad + i) * HD + sub * 8);
    const float4 x = __ldg(src), y = __ldg(src + 1);
    const uint4 o = make_uint4(pack_bf16(x.x * scale, x.y * scale), pack_bf16(x.z * scale, x.w * scale),
                               pack_bf16(y.x * scale, y.y * scale), pack_bf16(y.z * scale, y.w * scale));
    reinterpret_cast<uint4*>(dq + r * HD)[sub] = o;
    if (ep.active) reinterpret_cast<uint4*>(peer_row_ptr(ep, i, bb, b, h, HD, 2))[sub] = o;
  }
  if (ep.active) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) peer_signal_last_cta(ep, gridDim.x);
  }
}

static int64_t pad_n(int64_t n) { return (n + 127) / 128 * 128; }

template <int HD>
static int launch(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
                  void* dq, void* dk, void* dv, void* ws, int64_t n, int64_t b, int64_t hq, int64_t hkv, int causal,
                  float scale, int stages, int deterministic, const PeerEpilogue* eps, cudaStream_t st) {
  const int64_t npad = pad_n(n);
  float* L2 = reinterpret_cast<float*>(ws);
  float* Dv = L2 + b * hq * npad;
  const bool fused = HD == 128 && !deterministic;
  float* dq_acc = fused ? Dv + b * hq * npad : nullptr;   // [b*hq][npad][HD] f32
  if (stages & 1) {
    const int64_t threads = std::max<int64_t>(n * b * hq * (HD / 8), b * hq * (npad - n));
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    bwd_prep_kernel<HD><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, lse, L2, Dv,
                                                (int)n, (int)npad, (int)b, (int)hq, dq_acc);
    UL_TRY(launched("attn_bwd_prep"));
  }
  Params p;
  p.n = (int)n;
  p.n_pad = (int)npad;
  p.b = (int)b;
  p.hq = (int)hq;
  p.hkv = (int)hkv;
  p.causal = causal;
#ifdef UL_BWD_HEAD_MAJOR
  p.head_major = UL_BWD_HEAD_MAJOR;
#else
  p.head_major = (n + BT - 1) / BT >= sm_count();
#endif
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.L2 = L2;
  p.Dv = Dv;
  p.dq = (__nv_bfloat16*)dq;
  p.dk = (__nv_bfloat16*)dk;
  p.dv = (__nv_bfloat16*)dv;
  if (eps) {   // [dq, dk, dv]
    p.ep_dq = eps[0];
    p.ep_dk = eps[1];
    p.ep_dv = eps[2];
  } else {
    memset(&p.ep_dq, 0, sizeof(PeerEpilogue));
    memset(&p.ep_dk, 0, sizeof(PeerEpilogue));
    memset(&p.ep_dv, 0, sizeof(PeerEpilogue));
  }
  UL_TRY(smem_opt_in((const void*)bwd_dkdv_kernel<HD>, DkdvSmem<HD>::kBytes));
  UL_TRY(smem_opt_in((const void*)bwd_dq_kernel<HD>, DqSmem<HD>::kBytes));
  if constexpr (HD == 128) UL_TRY(smem_opt_in((const void*)bwd_fused_kernel<HD>, FusedSmem<HD>::kBytes));
  const int64_t tiles = (n + BT - 1) / BT;
  if constexpr (HD == 128) {
    if (fused) {
      if (stages & 2) {
        CUtensorMap mq, mk, mv, mo;
        UL_TRY(make_tmap_bhsd(&mq, q, n, b * hq, HD, BS));
        UL_TRY(make_tmap_bhsd(&mo, dout, n, b * hq, HD, BS));
        UL_TRY(make_tmap_bhsd(&mk, k, n, b * hkv, HD, BT));
        UL_TRY(make_tmap_bhsd(&mv, v, n, b * hkv, HD, BT));
        // tile-major within groups of heads whose Q / dO / dQ-accumulator
        // streams (8 bytes per row and hd element) fit in ~half the L2: r59,
        // config 2 (16 heads): groups of 8 -2.9%, of 4 -2.6%, tile-major 0
        Params pf = p;
        unsigned grid = (unsigned)(tiles * b * hkv);
#ifdef UL_BWD_HEAD_GROUP
        const int64_t G = UL_BWD_HEAD_GROUP;
#else
        const int64_t G = std::max<int64_t>(1, (int64_t)(64 << 20) / (npad * HD * 8 * (hq / hkv)));
#endif
        if (!p.head_major && b * hkv > G && G >= 2) {
          pf.head_major = (int)G;
          grid = (unsigned)(tiles * ((b * hkv + G - 1) / G) * G);
        }
        CUtensorMap mdk, mdv;   // 32-row store boxes of the dK / dV epilogue
        UL_TRY(make_tmap_bhsd(&mdk, dk, n, b * hkv, HD, 32));
        UL_TRY(make_tmap_bhsd(&mdv, dv, n, b * hkv, HD, 32));
        bwd_fused_kernel<HD><<<grid, kFuThreads, FusedSmem<HD>::kBytes, st>>>(mq, mk, mv, mo, mdk, mdv, pf, dq_acc);
        UL_TRY(launched("attn_bwd_fused_sm100"));
      }
      if (stages & 4) {
        const int64_t threads = n * b * hq * (HD / 8);
        bwd_dq_convert_kernel<HD><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
            dq_acc, (__nv_bfloat16*)dq, (int)n, (int)npad, (int)b, (int)hq, scale, p.ep_dq);
        UL_TRY(launched("attn_bwd_dq_convert"));
      }
      return UL_OK;
    }
  }
  if (stages & 2) {
    // dkdv: the kv tile is resident (128-row boxes), query sub-tiles stream (64-row boxes)
    CUtensorMap mq, mk, mv, mo;
    UL_TRY(make_tmap_bhsd(&mq, q, n, b * hq, HD, BS));
    UL_TRY(make_tmap_bhsd(&mo, dout, n, b * hq, HD, BS));
    UL_TRY(make_tmap_bhsd(&mk, k, n, b * hkv, HD, BT));
    UL_TRY(make_tmap_bhsd(&mv, v, n, b * hkv, HD, BT));
    bwd_dkdv_kernel<HD><<<(unsigned)(tiles * b * hkv), kDkThreads, DkdvSmem<HD>::kBytes, st>>>(mq, mk, mv, mo, p);
    UL_TRY(launched("attn_bwd_dkdv_sm100"));
  }
  if (stages & 4) {
    // dq: Q / dO go to TMEM inside the kernel; key/value sub-tiles stream
    CUtensorMap mk, mv;
    UL_TRY(make_tmap_bhsd(&mk, k, n, b * hkv, HD, BS));
    UL_TRY(make_tmap_bhsd(&mv, v, n, b * hkv, HD, BS));
    const unsigned dq_ctas = (unsigned)std::min<int64_t>(tiles * b * hq, sm_count());   // persistent
    bwd_dq_kernel<HD><<<dq_ctas, kDqThreads, DqSmem<HD>::kBytes, st>>>(
        mk, mv, (const __nv_bfloat16*)q, (const __nv_bfloat16*)dout, p);
    UL_TRY(launched("attn_bwd_dq_sm100"));
  }
  return UL_OK;
}

}  // namespace bwd

#ifdef UL_TRACE
extern "C" int ul_debug_cta(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, bwd::g_cta, bytes < sizeof(bwd::g_cta) ? bytes : sizeof(bwd::g_cta)) ==
                 cudaSuccess
             ? 0
             : -1;
}
extern "C" int ul_debug_warp(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, bwd::g_warp, bytes < sizeof(bwd::g_warp) ? bytes : sizeof(bwd::g_warp)) ==
                 cudaSuccess
             ? 0
             : -1;
}
extern "C" int ul_debug_trace(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, bwd::g_trace, bytes < sizeof(bwd::g_trace) ? bytes : sizeof(bwd::g_trace)) ==
                 cudaSuccess
             ? 0
             : -1;
}
#endif

int preload_bwd() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_prep_kernel<64>));
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_prep_kernel<128>));
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_dkdv_kernel<64>));
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_dkdv_kernel<128>));
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_dq_kernel<64>));
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_dq_kernel<128>));
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_fused_kernel<128>));
  UL_CUDA(cudaFuncGetAttributes(&a, bwd::bwd_dq_convert_kernel<128>));
  // dynamic shared-memory opt-ins now, not at the first launch (common.cuh)
  UL_TRY(smem_opt_in((const void*)bwd::bwd_dkdv_kernel<64>, bwd::DkdvSmem<64>::kBytes));
  UL_TRY(smem_opt_in((const void*)bwd::bwd_dkdv_kernel<128>, bwd::DkdvSmem<128>::kBytes));
  UL_TRY(smem_opt_in((const void*)bwd::bwd_dq_kernel<64>, bwd::DqSmem<64>::kBytes));
  UL_TRY(smem_opt_in((const void*)bwd::bwd_dq_kernel<128>, bwd::DqSmem<128>::kBytes));
  UL_TRY(smem_opt_in((const void*)bwd::bwd_fused_kernel<128>, bwd::FusedSmem<128>::kBytes));
  return UL_OK;
}


size_t sm100_bwd_workspace(int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd) {
  (void)hkv;
  // L2 + D rows, and the fp32 dQ accumulator of the fused hd-128 kernel
  // (sized whether or not deterministic mode is on, so a workspace stays valid
  // across mode switches)
  const size_t rows = (size_t)b * hq * bwd::pad_n(n);
  return rows * 2 * sizeof(float) + (hd == 128 ? rows * hd * sizeof(float) : 0);
}

int sm100_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
              void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, int64_t n, int64_t b, int64_t hq,
              int64_t hkv, int64_t hd, int causal, float scale, int stages, int deterministic, cudaStream_t st,
              const PeerEpilogue* eps) {
  (void)ws_bytes;
  if (n > INT32_MAX / 2) return fail(UL_ERR_SHAPE, "attention: sequence too long (n=%lld)", (long long)n);
  switch (hd) {
    case 64:
      return bwd::launch<64>(q, k, v, o, dout, lse, dq, dk, dv, ws, n, b, hq, hkv, causal, scale, stages, deterministic,
                             eps, st);
    case 128:
      return bwd::launch<128>(q, k, v, o, dout, lse, dq, dk, dv, ws, n, b, hq, hkv, causal, scale, stages, deterministic,
                              eps, st);
    default:
      return fail(UL_ERR_KERNEL, "bf16 attention supports head_dim 64 or 128, got %lld", (long long)hd);
  }
}

}  // namespace ul
