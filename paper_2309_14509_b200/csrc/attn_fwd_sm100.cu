// K3: FlashAttention-style forward on sm_100a (tcgen05 + TMEM + TMA), two query tiles per CTA.
//
// Replaces the per-head kernel loop of ulysses_attention_forward_with_state
// (ulysses.py:148-152) over _masked_attention (kernels.py:31-40: scores =
// q k^T * scale, row_softmax tensor.py:227-249, ctx = probs v), plus the row
// LSE the backward needs (the reference recomputes probabilities instead,
// kernels.py:104); structured so the tensor core never waits on a softmax:
//   * a CTA owns two 128-row query tiles (A, B) of one (batch, head); every
//     K_j / V_j tile brought in by TMA serves both (half the smem/L2 traffic
//     per FLOP of one tile per CTA);
//   * TMEM = S_A | S_B | O_A | O_B (128 + 128 + hd + hd columns);
//   * the single MMA thread issues   PV_A(j), S_A(j+1), PV_B(j), S_B(j+1)
//     so softmax A of tile j+1 overlaps PV_B(j)/S_B(j+1) and vice versa.
//     tcgen05.mma ops of one thread execute in issue order, so S_A(j+1) may
//     overwrite the TMEM columns PV_A(j) reads P_A(j) from without a wait;
//     and tcgen05.commit tracks every earlier MMA of the thread, so "S_A(j)
//     ready" also means "PV_A(j-1) done" -- the (rare, lazy) O rescale needs
//     no extra barrier;
//   * warps 2-5 run softmax A, warps 6-9 softmax B (two independent softmax
//     streams per SMSP); one query row per thread, exp2 domain, masking only
//     on diagonal/tail tiles, FFMA-fused exponent, ILP'd max/sum chains, P
//     packed to bf16 and stored 32 columns at a time over consumed S.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "comm.cuh"
#include "common.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace ul {
namespace fwd {

// Pipeline trace (profiling builds only, -DUL_TRACE): clock64 stamps of the
// first 8 CTAs [cta][16 events][kv tile] and per-CTA life (see tools/trace_bwd.py)
#ifdef UL_TRACE
__device__ unsigned long long g_trace[8 * 16 * 256];
__device__ unsigned long long g_cta[8192 * 7];
#define UL_EV(ev, j)                                                                             \
  do {                                                                                           \
    if (blockIdx.x < 8 && (j) < 256) g_trace[(blockIdx.x * 16 + (ev)) * 256 + (j)] = clock64(); \
  } while (0)
#define UL_CTA(k, v) g_cta[blockIdx.x * 7 + (k)] = (v)
#else
#define UL_EV(ev, j) \
  do {               \
  } while (0)
#define UL_CTA(k, v) \
  do {               \
  } while (0)
#endif

using namespace sm100;

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int NS = 2;               // K/V pipeline stages
// TMA, MMA, 2 x 8 softmax warps: two warps per TMEM lane quarter and query
// tile, each owning half of a row's 128 columns (row max / sum combined
// through shared memory + a 64-thread named barrier)
constexpr int kSoftPerTile = 8;
constexpr int kThreads = 64 + 2 * kSoftPerTile * 32;
constexpr float kLazy = 8.0f;       // log2 headroom before O is rescaled
// Full-tile persistent kernel (r2 A/B at config 2 / N = 32K x 4 heads, WPR = 1):
// split P arrive 0.2662 -> 0.2519 ms with a 1/8 FMA-pipe share; 1/16: 0.249 /
// 0.905 ms vs the half-unit kernel's 0.267 / 0.996.  The chain softmax(j) ->
// PV(j) -> S(j+1) of a tile hides under the other tile's 1024 tensor cycles
// only if the softmax is shorter: its 4096 exponentials per SMSP are exactly
// 1024 MUFU cycles, so a share goes to the FMA pipe and the first 3/4 of P
// is handed to the PV MMAs before the last quarter's exponentials run.
#ifndef UL_FWD_SPLITP
#define UL_FWD_SPLITP 1
#endif
// the full-tile forward's MMA thread waits (UL_FWD_MMA_WAIT: 0 plain try_wait,
// 2 try_wait with the suspend hint -- the other kernels' default, which the
// compiler turns into a NANOSLEEP.SYNCS back-off; 3 nanosleep polling).  r2,
// config 2: 0.2478 / 0.2509-0.2519 / 0.254 ms -- the thread is woken ~400
// cycles late from the back-off (trace), on the chain p_full -> PV -> S
#ifndef UL_FWD_MMA_WAIT
#define UL_FWD_MMA_WAIT 0
#endif
__device__ __forceinline__ void mbar_wait_fmma(uint64_t* bar, uint32_t parity) {
  mbar_wait_k<UL_FWD_MMA_WAIT>(bar, parity);
}
#ifndef UL_FWD_SPLIT_AT
#define UL_FWD_SPLIT_AT 96
#endif
constexpr int kSplitAt = UL_FWD_SPLIT_AT;   // split P arrive: kv columns announced first (multiple of 32)
#ifndef UL_FWD_FULL_POLY_MASK
#define UL_FWD_FULL_POLY_MASK 30           // FMA-pipe exp2 on 1/16 of the element pairs (0: none)
#endif
constexpr int kAtom = 128 * 128;    // SW128 atom column of a 128-row tile
constexpr int kMaxTiles = 8192;     // kv tiles per head in blocked-sparse mode (n <= 1M)

template <int HD>
struct Smem {
  static constexpr int kTile = (HD / 64) * kAtom;
  static constexpr int kQ = 0;                    // [2] (tile A, tile B)
  static constexpr int kK = kQ + 2 * kTile;       // [NS]
  static constexpr int kV = kK + NS * kTile;      // [NS]
  static constexpr int kBar = kV + NS * kTile;
  static constexpr int kList = kBar + 256;               // blocked-sparse: the CTA's kv tile list
  static constexpr int kX = kList + kMaxTiles * 2;       // row max / sum exchange [2 parity][2 tiles][128][2]
  static constexpr int kBytes = kX + 3 * 2 * 128 * 2 * 4 + 1024;   // (3 slots: persistent kernel)
};

struct Params {
  int n, b, hq, hkv;
  int causal;
  int qtiles, pairs;
  int head_major;
  float scale_log2;
  __nv_bfloat16* o;
  float* lse;
  PeerEpilogue ep;   // active: also store O rows into the seq layout of their rank (fused head->seq)
  // blocked-sparse mask (Mask.blocked, tensor.py:163-180; blocked_kernel,
  // kernels.py:55-86): bit (qb, kb) of blk[qb * blk_words + kb / 32] says
  // whether query block qb sees key block kb (blocks of blk_bs tokens,
  // blk_nb = n / blk_bs per side).  nullptr: dense / causal.
  const uint32_t* blk;
  int blk_bs, blk_words, blk_nb;
  // persistent kernel: [next item, CTAs done] counters (per stream, zero at
  // rest: the last CTA resets them), or nullptr for the static zig-zag waves
  int* ctr;
  // ping-pong of the two query tiles' exponential phases (named barriers
  // 9/10): tile A's exponentials of a step run while tile B's MMAs do and
  // vice versa, instead of both softmaxes sharing the MUFU in lockstep
  int alt;
};

// named-barrier hand-off between the two tiles' softmax warp groups (`nthr`:
// the softmax threads of both tiles)
__device__ __forceinline__ void alt_sync(int id, int nthr = 512) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthr) : "memory");
}
__device__ __forceinline__ void alt_arrive(int id, int nthr = 512) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthr) : "memory");
}

__device__ __forceinline__ bool blk_bit(const Params& p, int qb, int kb) {
  return (__ldg(p.blk + (int64_t)qb * p.blk_words + (kb >> 5)) >> (kb & 31)) & 1u;
}
// does any query row in [qlo, qhi] see any key of kv tile kt?
__device__ __forceinline__ bool blk_tile_needed(const Params& p, int qlo, int qhi, int kt) {
  const int kb0 = kt * BN / p.blk_bs, kb1 = min(p.blk_nb - 1, (kt * BN + BN - 1) / p.blk_bs);
  const int qb0 = qlo / p.blk_bs, qb1 = min(p.blk_nb - 1, qhi / p.blk_bs);
  for (int qb = qb0; qb <= qb1; ++qb)
    for (int kb = kb0; kb <= kb1; ++kb)
      if (blk_bit(p, qb, kb)) return true;
  return false;
}
// visible-column bitmask of one query row over kv tile columns [kv0, kv0 + 128)
__device__ __forceinline__ void blk_row_mask(const Params& p, int qrow, int kv0, uint32_t cm[4]) {
  cm[0] = cm[1] = cm[2] = cm[3] = 0u;
  if (qrow >= p.n) return;
  const int qb = qrow / p.blk_bs;
  const int kb0 = kv0 / p.blk_bs, kb1 = min(p.blk_nb - 1, (kv0 + BN - 1) / p.blk_bs);
  for (int kb = kb0; kb <= kb1; ++kb) {
    if (!blk_bit(p, qb, kb)) continue;
    const int lo = max(kb * p.blk_bs, kv0) - kv0, hi = min((kb + 1) * p.blk_bs, kv0 + BN) - kv0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int a = max(lo, 32 * w), e = min(hi, 32 * w + 32);
      if (a < e) cm[w] |= (e - a == 32 ? 0xffffffffu : ((1u << (e - a)) - 1u)) << (a - 32 * w);
    }
  }
}

// P = 2^(S*scale_log2 - mu) for 32 columns, packed to bf16 pairs, row sums
// accumulated into 8 partials.  kPoly routes one element pair in four to
// the FMA-pipe exp2 (unmasked tiles only).
// f16x2 exponentials (one MUFU op per element pair) for all pairs
// (UL_FWD_EXP_H2=1) or every other pair (=2); off by default
#ifndef UL_FWD_EXP_H2
#define UL_FWD_EXP_H2 0
#endif
constexpr bool kH2 = UL_FWD_EXP_H2 != 0;
constexpr int kH2Sel = UL_FWD_EXP_H2 == 2 ? 2 : 0;
// FMA-pipe exponentials on element pairs x with (x & mask) == mask: 6 -> 1/4,
// 14 -> 1/8, 30 -> 1/16 of the pairs (when kPoly)
#ifndef UL_FWD_POLY_MASK
#define UL_FWD_POLY_MASK 6
#endif
template <bool kPoly, int kMask = UL_FWD_POLY_MASK>
__device__ __forceinline__ void exp_chunk(const uint32_t* r, float scale_log2, float mu, uint32_t* pk,
                                          float2* rsum) {
  const float2 sc = make_float2(scale_log2, scale_log2), nm = make_float2(-mu, -mu);
#pragma unroll
  for (int x = 0; x < 32; x += 2) {
    // packed f32x2 FMA / add: half the issue slots of the scalar forms
    const float2 a = __ffma2_rn(make_float2(__uint_as_float(r[x]), __uint_as_float(r[x + 1])), sc, nm);
    float2 e;
    if (kPoly && (x & kMask) == kMask) {
      e = poly_exp2x2(a);
    } else if (kH2 && (x & 2) == kH2Sel) {
      e = exp2_h2(a);
    } else {
      e.x = fast_exp2(a.x);
      e.y = fast_exp2(a.y);
    }
    rsum[(x >> 1) & 3] = __fadd2_rn(rsum[(x >> 1) & 3], e);
    pk[x / 2] = pack_bf16_op(e.x, e.y);
  }
}

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
  uint64_t* k_full = bars + 1;              // [NS]
  uint64_t* k_empty = bars + 1 + NS;        // [NS]
  uint64_t* v_full = bars + 1 + 2 * NS;     // [NS]
  uint64_t* v_empty = bars + 1 + 3 * NS;    // [NS]
  uint64_t* s_full = bars + 1 + 4 * NS;     // [2] per tile
  uint64_t* p_full = bars + 3 + 4 * NS;     // [2] per tile
  uint64_t* o_done = bars + 5 + 4 * NS;     // [2] per tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7 + 4 * NS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // CTA order (longest causal pairs first either way):
  //  head-major when a head has >= one wave of pairs -- resident CTAs then
  //    stream the same K/V tiles (L2 reuse at long N / many heads);
  //  pair-major otherwise -- a global longest-first (LPT) order balances
  //    the waves when every head is short.
  const int heads = p.b * p.hq;
  const int pair = p.head_major ? p.pairs - 1 - (int)(blockIdx.x % p.pairs)
                                : p.pairs - 1 - (int)(blockIdx.x / heads);
  const int bh = p.head_major ? (int)(blockIdx.x / p.pairs) : (int)(blockIdx.x % heads);
  const int bb = bh / p.hq, h = bh % p.hq;
  const int g = h / (p.hq / p.hkv);
  const int nkv_all = (p.n + BN - 1) / BN;
  uint16_t* tiles = reinterpret_cast<uint16_t*>(smem + S::kList);
  const bool blocked = p.blk != nullptr;
  int nblk = 0;   // blocked-sparse: kv tiles any row of this CTA's query tiles sees, ascending
  if (blocked) {
    const int qlo = 2 * pair * BM, qhi = min(p.n, (2 * pair + 2) * BM) - 1;
    if (warp == 0) {
      for (int base = 0; base < nkv_all; base += 32) {
        const bool need = base + lane < nkv_all && blk_tile_needed(p, qlo, qhi, base + lane);
        const uint32_t bal = __ballot_sync(0xffffffffu, need);
        if (need) tiles[nblk + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)(base + lane);
        nblk += __popc(bal);
      }
    } else {
      for (int base = 0; base < nkv_all; base += 32)
        nblk += __popc(__ballot_sync(0xffffffffu, base + lane < nkv_all && blk_tile_needed(p, qlo, qhi, base + lane)));
    }
  }
  int nkvT[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int qt = 2 * pair + t;
    nkvT[t] = qt >= p.qtiles ? 0 : blocked ? nblk : (p.causal ? min(nkv_all, (qt * BM + BM - 1) / BN + 1) : nkv_all);
  }
  const int nkv = max(nkvT[0], nkvT[1]);
  const int ntiles = nkvT[1] > 0 ? 2 : 1;

  if (threadIdx.x == 0) {
    UL_CTA(0, globaltimer());
    UL_CTA(4, smid());
    UL_CTA(5, clock64());
  }
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], kSoftPerTile);   // one arrive per softmax warp
      mbar_init(&o_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();   // 512 columns = the whole TMEM: base is column 0
  constexpr uint32_t tbase = 0;
  // TMEM columns: S_A 0, S_B 128, O_A 256, O_B 256 + HD

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_expect_tx(q_full, ntiles * BM * HD * 2);
      for (int t = 0; t < ntiles; ++t)
#pragma unroll
        for (int a = 0; a < HD / 64; ++a)
          tma_load_3d(sQ + t * S::kTile + a * kAtom, &tmQ, q_full, a * 64, bb * p.hq + h, (2 * pair + t) * BM);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % NS;
        const uint32_t ph = (j / NS) & 1;
        mbar_wait_prod(&k_empty[s], ph ^ 1);
        UL_EV(8, j);
        mbar_expect_tx(&k_full[s], BN * HD * 2);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a)
          tma_load_3d(sK + s * S::kTile + a * kAtom, &tmK, &k_full[s], a * 64, bb * p.hkv + g,
                      (blocked ? tiles[j] : j) * BN);
        mbar_wait_prod(&v_empty[s], ph ^ 1);
        UL_EV(9, j);
        mbar_expect_tx(&v_full[s], BN * HD * 2);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a)
          tma_load_3d(sV + s * S::kTile + a * kAtom, &tmV, &v_full[s], a * 64, bb * p.hkv + g,
                      (blocked ? tiles[j] : j) * BN);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {  // one thread issues every MMA (uniform operands)
      constexpr uint32_t kIdQK = idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t kIdPV = idesc_bf16(BM, HD, 0, 1);
      // base descriptors built once; per-MMA cost is a constant add
      const uint64_t dQ0 = sdesc(smem_u32(sQ), 16, 1024);
      const uint64_t dK0 = sdesc(smem_u32(sK), 16, 1024);
      const uint64_t dV0 = sdesc(smem_u32(sV), kAtom, 1024);
      auto issue_s = [&](int t, int j) {   // S_t = Q_t K_j^T
        const uint64_t dk = dadd(dK0, (j % NS) * S::kTile);
        const uint64_t dq = dadd(dQ0, t * S::kTile);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_ss(tbase + t * 128, dadd(dq, off), dadd(dk, off), kIdQK, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j) {  // O_t += P_t V_j
        mbar_wait_mma(&p_full[t], j & 1);
        UL_EV(t == 0 ? 1 : 2, j);
        tc_fence_after();
        const uint64_t dv = dadd(dV0, (j % NS) * S::kTile);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts(tbase + 256 + t * HD, tbase + t * 128 + kk * 8, dadd(dv, kk * 2048), kIdPV,
                 (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&o_done[t]);
      };
      mbar_wait_mma(q_full, 0);
      mbar_wait_mma(&k_full[0], 0);
      UL_CTA(1, globaltimer());
      tc_fence_after();
      if (nkvT[0] > 0) issue_s(0, 0);
      if (nkvT[1] > 0) issue_s(1, 0);
      mma_commit(&k_empty[0]);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % NS;
        const bool next = j + 1 < nkv;
        UL_EV(10, j);
        mbar_wait_mma(&v_full[s], (j / NS) & 1);
        if (next) mbar_wait_mma(&k_full[(j + 1) % NS], ((j + 1) / NS) & 1);
        UL_EV(0, j);
        tc_fence_after();
        if (j < nkvT[0]) issue_pv(0, j);
        if (next && j + 1 < nkvT[0]) issue_s(0, j + 1);
        UL_EV(6, j);
        if (j < nkvT[1]) issue_pv(1, j);
        if (next && j + 1 < nkvT[1]) issue_s(1, j + 1);
        mma_commit(&v_empty[s]);
        if (next) mma_commit(&k_empty[(j + 1) % NS]);
        UL_EV(7, j);
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax / correction / epilogue ----------------
    const int idx = warp - 2;
    const int t = idx >> 3;                   // query tile of this warp
    const int quarter = warp & 3;
    const int half = (idx & 7) >> 2;          // which 64 of the row's 128 columns
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tbase + t * 128 + lane_off;
    const uint32_t tO = tbase + 256 + t * HD + lane_off;
    const int q0 = (2 * pair + t) * BM;
    const int qrow = q0 + row;
    const int my_nkv = t ? nkvT[1] : nkvT[0];   // (no dynamic index into a local array)
    const uint32_t bar_id = 1 + t * 4 + quarter;  // the two warps of this (tile, quarter)
    float* xch = reinterpret_cast<float*>(smem + S::kX);
    auto xslot = [&](int par, int hh) { return smem_u32(xch + ((par * 2 + t) * 128 + row) * 2 + hh); };
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    float m = -INFINITY, l = 0.f;   // l: this half's partial row sum
    for (int j = 0; j < my_nkv; ++j) {
      const int kv0 = (blocked ? tiles[j] : j) * BN;
      mbar_wait(&s_full[t], j & 1);
      if (lane == 0 && (warp == 2 || warp == 10)) UL_EV(warp == 2 ? 3 : 5, j);
      tc_fence_after();
      uint32_t r[BN / 2];
      tmem_ld32(tS + half * 64, r);
      tmem_ld32(tS + half * 64 + 32, r + 32);
      tmem_wait_ld();
      if (lane == 0 && warp == 2) UL_EV(12, j);
      const bool masked = (p.causal && kv0 + BN - 1 > q0) || kv0 + BN > p.n;
      if (blocked) {
        uint32_t cm[4];
        blk_row_mask(p, qrow, kv0, cm);
        const uint32_t c0w = half ? cm[2] : cm[0], c1w = half ? cm[3] : cm[1];
#pragma unroll
        for (int c = 0; c < BN / 2; ++c)
          if (!(((c < 32 ? c0w : c1w) >> (c & 31)) & 1u)) r[c] = __float_as_uint(-INFINITY);
      } else if (masked) {
        int limit = p.n - kv0;
        if (p.causal) limit = min(limit, qrow - kv0 + 1);
        limit -= half * 64;
#pragma unroll
        for (int c = 0; c < BN / 2; ++c)
          if (c >= limit) r[c] = __float_as_uint(-INFINITY);
      }
      float mx[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx[u] = __uint_as_float(r[u]);
#pragma unroll
      for (int c = 8; c < BN / 2; c += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) mx[u] = fmaxf(mx[u], __uint_as_float(r[c + u]));
      }
      float mh = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      // row max across the two halves (double-buffered by tile parity)
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot(j & 1, half)), "f"(mh) : "memory");
      pair_sync();
      float other;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(xslot(j & 1, half ^ 1)) : "memory");
      const float mt = fmaxf(mh, other) * p.scale_log2;
#ifdef UL_TRACE
      {
        uint32_t dep;
        asm volatile("mov.b32 %0, %1;" : "=r"(dep) : "f"(mt));
        if (lane == 0 && warp == 2 && dep != 0x7fffffffu) UL_EV(13, j);
      }
#endif
      float alpha = 1.f;
      bool rescale = false;
      if (mt > m + kLazy) {
        alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mt);
        rescale = (j > 0);
        m = mt;
      }
      const float mu = (m == -INFINITY) ? 0.f : m;
      float2 rsum[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#ifdef UL_FWD_POLY
        if (!masked) exp_chunk<true>(r + c * 32, p.scale_log2, mu, pk, rsum);
        else
#endif
        exp_chunk<false>(r + c * 32, p.scale_log2, mu, pk, rsum);
        tmem_st16(tS + (2 * half + c) * 16, pk);   // P over S columns already in registers
      }
      const float2 rs = __fadd2_rn(__fadd2_rn(rsum[0], rsum[1]), __fadd2_rn(rsum[2], rsum[3]));
      l = l * alpha + (rs.x + rs.y);
#ifdef UL_TRACE
      {
        uint32_t dep;
        asm volatile("mov.b32 %0, %1;" : "=r"(dep) : "f"(l));
        if (lane == 0 && warp == 2 && dep != 0x7fffffffu) UL_EV(14, j);
      }
#endif
      // s_full(j) tracks every earlier MMA, so PV(j-1) is complete: rescale
      // this half's 64 O columns now
      if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          uint32_t ov[32];
          tmem_ld32(tO + half * (HD / 2) + c * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 32; ++x) ov[x] = __float_as_uint(__uint_as_float(ov[x]) * alpha);
          tmem_st32(tO + half * (HD / 2) + c * 32, ov);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      if (lane == 0 && (warp == 2 || warp == 10)) UL_EV(warp == 2 ? 4 : 11, j);
      if (lane == 0 && warp == 4) UL_EV(15, j);
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    if (my_nkv > 0) {
      // full row sum from the two halves
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot(my_nkv & 1, half)), "f"(l) : "memory");
      pair_sync();
      float lo;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(lo) : "r"(xslot(my_nkv & 1, half ^ 1)) : "memory");
      const float lrow = l + lo;
      mbar_wait(&o_done[t], (my_nkv - 1) & 1);
      if (threadIdx.x == 64) UL_CTA(2, globaltimer());
      tc_fence_after();
      const float inv = 1.f / lrow;
      const bool valid = qrow < p.n;
      __nv_bfloat16* orow = p.o + (((int64_t)qrow * p.b + bb) * p.hq + h) * HD + half * (HD / 2);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        uint32_t ov[32];
        tmem_ld32(tO + half * (HD / 2) + c * 32, ov);
        tmem_wait_ld();
        uint32_t pkd[16];
#pragma unroll
        for (int x = 0; x < 16; ++x)
          pkd[x] = pack_bf16(__uint_as_float(ov[2 * x]) * inv, __uint_as_float(ov[2 * x + 1]) * inv);
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int x = 0; x < 4; ++x) dst[x] = make_uint4(pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
          if (p.ep.active) {
            // fused head->seq: the same 64 bytes straight into the destination
            // rank's sequence layout (own `out`, or its receive slot over NVLink)
            uint4* pd = reinterpret_cast<uint4*>(peer_row_ptr(p.ep, qrow, bb, p.b, h, HD, 2) + half * HD) + c * 4;
#pragma unroll
            for (int x = 0; x < 4; ++x) pd[x] = make_uint4(pkd[4 * x], pkd[4 * x + 1], pkd[4 * x + 2], pkd[4 * x + 3]);
          }
        }
      }
      if (valid && half == 0) p.lse[((int64_t)bb * p.hq + h) * p.n + qrow] = (m + log2f(lrow)) * 0.69314718055994531f;
    }
    if (p.ep.active) __threadfence_system();
  }
  tc_fence_before();
  __syncthreads();
  if (p.ep.active && threadIdx.x == 0) peer_signal_last_cta(p.ep, gridDim.x);
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

// Persistent variant (dense / causal): one CTA per SM walks the (query-tile
// pair, head) items in zig-zag waves; barriers run on across items, the next
// item's Q is loaded as soon as the last S MMAs of the current one complete,
// its first S MMAs queue behind the current PVs, and the O accumulator of a
// tile is handed back by the epilogue warps (o_free) before the next item's
// first PV overwrites it -- the per-CTA prologue / tail of the one-shot grid
// overlap with neighbouring items.
template <int HD>
__device__ __forceinline__ bool fwd_item(const Params& p, int k, int& pair, int& bh) {
  const int heads = p.b * p.hq;
  const int G = (int)gridDim.x;
  const int idx = k * G + ((k & 1) ? G - 1 - (int)blockIdx.x : (int)blockIdx.x);
  if (idx >= p.pairs * heads) return false;
  pair = p.head_major ? p.pairs - 1 - idx % p.pairs : p.pairs - 1 - idx / heads;
  bh = p.head_major ? idx / p.pairs : idx % heads;
  return true;
}

// dynamic items: the TMA thread (role 0) takes the next item index from the
// launch's counter and publishes it in a 4-slot shared ring; the MMA thread
// (role 1) and every softmax warp (role 2, all lanes) read it in the same
// order -- greedy longest-first over the length-sorted list
template <int HD>
__device__ __forceinline__ bool fwd_item_dyn(const Params& p, int k, int& pair, int& bh, int role,
                                             uint64_t* it_full, uint64_t* it_empty, volatile int* sitem) {
  const int slot = k & 3;
  int idx;
  if (role == 0) {
    if (k >= 4) mbar_wait(&it_empty[slot], ((k >> 2) - 1) & 1);
    idx = atomicAdd(p.ctr, 1);
    sitem[slot] = idx;
    mbar_arrive(&it_full[slot]);
  } else {
    mbar_wait(&it_full[slot], (k >> 2) & 1);
    idx = sitem[slot];
    if (role == 2) __syncwarp();
    if (role == 1 || (threadIdx.x & 31) == 0) mbar_arrive(&it_empty[slot]);
  }
  const int heads = p.b * p.hq;
  if (idx >= p.pairs * heads) return false;
  pair = p.head_major ? p.pairs - 1 - idx % p.pairs : p.pairs - 1 - idx / heads;
  bh = p.head_major ? idx / p.pairs : idx % heads;
  return true;
}

// WPR: softmax warps per query row (1, the default: one thread per row
// owning all 128 columns, 10 warps, no exchange; 2: two warps per TMEM lane
// quarter, 64 of the 128 columns each, row max / sum exchanged through shared
// memory).  Each tile's softmax hands P to the PV MMAs in two parts (p_part:
// kv columns < kSplitAt, then p_full) -- see the UL_FWD_SPLITP note above.
template <int WPR>
constexpr int persist_threads() { return 64 + 2 * 4 * WPR * 32; }

template <int HD, int WPR>
__global__ void __launch_bounds__(persist_threads<WPR>(), 1)
    attn_fwd_persist_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                            const __grid_constant__ CUtensorMap tmV, const Params p) {
  using S = Smem<HD>;
  constexpr int kSoft = 4 * WPR;     // softmax warps per query tile
  constexpr int kC = BN / WPR;       // S columns per softmax thread
  constexpr int kOC = HD / WPR;      // O columns per softmax thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;              // [NS]
  uint64_t* k_empty = bars + 1 + NS;        // [NS]
  uint64_t* v_full = bars + 1 + 2 * NS;     // [NS]
  uint64_t* v_empty = bars + 1 + 3 * NS;    // [NS]
  uint64_t* s_full = bars + 1 + 4 * NS;     // [2] per tile
  uint64_t* p_full = bars + 3 + 4 * NS;     // [2] per tile
  uint64_t* o_done = bars + 5 + 4 * NS;     // [2] per tile
  uint64_t* q_empty = bars + 7 + 4 * NS;    // Q smem free (the item's last S MMAs completed)
  uint64_t* o_free = bars + 8 + 4 * NS;     // [2] per tile: O read out by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10 + 4 * NS);
  uint64_t* it_full = bars + 11 + 4 * NS;   // [4] dynamic item ring
  uint64_t* it_empty = bars + 15 + 4 * NS;  // [4]
  volatile int* sitem = reinterpret_cast<volatile int*>(bars + 19 + 4 * NS);
  // [2] per tile (split P arrive): P of kv columns < kSplitAt stored (and O
  // rescaled) -- the first six PV K-steps may start while the last 32
  // columns' exponentials are still running
  uint64_t* p_part = bars + 21 + 4 * NS;
  static_assert((23 + 4 * NS) * 8 <= 256, "barrier area");
  auto item = [&](int k, int& pair, int& bh, int role) {
    return p.ctr ? fwd_item_dyn<HD>(p, k, pair, bh, role, it_full, it_empty, sitem) : fwd_item<HD>(p, k, pair, bh);
  };
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nkv_all = (p.n + BN - 1) / BN;
  auto item_kv = [&](int pair, int t) {
    const int qt = 2 * pair + t;
    return qt >= p.qtiles ? 0 : (p.causal ? min(nkv_all, (qt * BM + BM - 1) / BN + 1) : nkv_all);
  };

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], kSoft);
      mbar_init(&p_part[t], kSoft);
      mbar_init(&o_done[t], 1);
      mbar_init(&o_free[t], kSoft);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&it_full[s], 1);
      mbar_init(&it_empty[s], 1 + 2 * kSoft);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {   // CTA life (trace builds): start
    UL_CTA(0, globaltimer());
    UL_CTA(1, globaltimer());
    UL_CTA(4, smid());
    UL_CTA(5, clock64());
  }
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tbase = 0;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      int pair, bh, gk = 0;
      for (int k = 0; item(k, pair, bh, 0); ++k) {
        const int bb = bh / p.hq, h = bh % p.hq, g = h / (p.hq / p.hkv);
        const int n0 = item_kv(pair, 0), n1 = item_kv(pair, 1);
        const int nkv = max(n0, n1), ntiles = n1 > 0 ? 2 : 1;
        if (k > 0) mbar_wait(q_empty, (k - 1) & 1);
        mbar_expect_tx(q_full, ntiles * BM * HD * 2);
        for (int t = 0; t < ntiles; ++t)
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load_3d(sQ + t * S::kTile + a * kAtom, &tmQ, q_full, a * 64, bb * p.hq + h, (2 * pair + t) * BM);
        for (int j = 0; j < nkv; ++j, ++gk) {
          const int s = gk % NS;
          const uint32_t ph = (gk / NS) & 1;
          mbar_wait_prod(&k_empty[s], ph ^ 1);
          mbar_expect_tx(&k_full[s], BN * HD * 2);
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load_3d(sK + s * S::kTile + a * kAtom, &tmK, &k_full[s], a * 64, bb * p.hkv + g, j * BN);
          mbar_wait_prod(&v_empty[s], ph ^ 1);
          mbar_expect_tx(&v_full[s], BN * HD * 2);
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load_3d(sV + s * S::kTile + a * kAtom, &tmV, &v_full[s], a * 64, bb * p.hkv + g, j * BN);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t kIdQK = idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t kIdPV = idesc_bf16(BM, HD, 0, 1);
      const uint64_t dQ0 = sdesc(smem_u32(sQ), 16, 1024);
      const uint64_t dK0 = sdesc(smem_u32(sK), 16, 1024);
      const uint64_t dV0 = sdesc(smem_u32(sV), kAtom, 1024);
      int cpv[2] = {0, 0};      // PV MMAs (== p_full waits == o_done commits) per tile so far
      int items_t[2] = {0, 0};  // items in which the tile existed so far
      auto issue_s = [&](int t, int stage) {
        const uint64_t dk = dadd(dK0, stage * S::kTile);
        const uint64_t dq = dadd(dQ0, t * S::kTile);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_ss(tbase + t * 128, dadd(dq, off), dadd(dk, off), kIdQK, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[t]);
      };
      auto issue_pv = [&](int t, int j, int stage) {
        if (j == 0 && items_t[t] > 0) mbar_wait_fmma(&o_free[t], (items_t[t] - 1) & 1);
        const uint64_t dv = dadd(dV0, stage * S::kTile);
#if UL_FWD_SPLITP
        mbar_wait_fmma(&p_part[t], cpv[t] & 1);
        UL_EV(t == 0 ? 0 : 2, cpv[t]);   // (trace) p_part seen
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kSplitAt / 16; ++kk)
          mma_ts(tbase + 256 + t * HD, tbase + t * 128 + kk * 8, dadd(dv, kk * 2048), kIdPV,
                 (j > 0 || kk > 0) ? 1u : 0u);
        mbar_wait_fmma(&p_full[t], cpv[t] & 1);
        UL_EV(t == 0 ? 12 : 13, cpv[t]);   // (trace) p_full seen (after the first K-steps)
        tc_fence_after();
#pragma unroll
        for (int kk = kSplitAt / 16; kk < BN / 16; ++kk)
          mma_ts(tbase + 256 + t * HD, tbase + t * 128 + kk * 8, dadd(dv, kk * 2048), kIdPV, 1u);
#else
        mbar_wait_fmma(&p_full[t], cpv[t] & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_ts(tbase + 256 + t * HD, tbase + t * 128 + kk * 8, dadd(dv, kk * 2048), kIdPV,
                 (j > 0 || kk > 0) ? 1u : 0u);
#endif
        mma_commit(&o_done[t]);
        UL_EV(t == 0 ? 1 : 3, cpv[t]);   // (trace) PV issued
        ++cpv[t];
      };
      int pair, bh, gk = 0;
      for (int k = 0; item(k, pair, bh, 1); ++k) {
        const int nT0 = item_kv(pair, 0), nT1 = item_kv(pair, 1);
        const int nkv = max(nT0, nT1);
        mbar_wait_fmma(q_full, k & 1);
        mbar_wait_fmma(&k_full[gk % NS], (gk / NS) & 1);
        tc_fence_after();
        if (nT0 > 0) issue_s(0, gk % NS);
        if (nT1 > 0) issue_s(1, gk % NS);
        mma_commit(&k_empty[gk % NS]);
        if (nkv == 1) mma_commit(q_empty);
        for (int j = 0; j < nkv; ++j) {
          const int s = (gk + j) % NS, s1 = (gk + j + 1) % NS;
          const bool next = j + 1 < nkv;
          UL_EV(10, gk + j);   // (trace) MMA loop top
          mbar_wait_fmma(&v_full[s], ((gk + j) / NS) & 1);
          if (next) mbar_wait_fmma(&k_full[s1], ((gk + j + 1) / NS) & 1);
          tc_fence_after();
          if (j < nT0) issue_pv(0, j, s);
          if (next && j + 1 < nT0) issue_s(0, s1);
          if (j < nT1) issue_pv(1, j, s);
          if (next && j + 1 < nT1) issue_s(1, s1);
          mma_commit(&v_empty[s]);
          if (next) mma_commit(&k_empty[s1]);
          if (j + 2 == nkv) mma_commit(q_empty);   // the item's last S MMAs are issued: Q may be replaced
        }
        if (nT0 > 0) ++items_t[0];
        if (nT1 > 0) ++items_t[1];
        gk += nkv;
      }
    }
    __syncwarp();
  } else {
    const int idx = warp - 2;
    const int t = idx / kSoft;
    const int quarter = warp & 3;
    const int half = (idx % kSoft) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tbase + t * 128 + lane_off;
    const uint32_t tO = tbase + 256 + t * HD + lane_off;
    const uint32_t bar_id = 1 + t * 4 + quarter;
    float* xch = reinterpret_cast<float*>(smem + S::kX);
    // [3 slots: max parity 0/1, row sum][2 tiles][128 rows][2 halves]
    auto xslot = [&](int sl, int hh) { return smem_u32(xch + ((sl * 2 + t) * 128 + row) * 2 + hh); };
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    int cs = 0;   // S tiles of this query tile consumed so far (s_full / o_done phases)
    int pair, bh;
    for (int k = 0; item(k, pair, bh, 2); ++k) {
      const int my_nkv = item_kv(pair, t);
      if (my_nkv == 0) continue;
      const int na = item_kv(pair, 0);
      const bool alt_item = p.alt && na > 0 && item_kv(pair, 1) > 0;
      if (alt_item && t == 1) alt_arrive(9, 64 * kSoft);   // tile A goes first
      const int bb = bh / p.hq, h = bh % p.hq;
      const int q0 = (2 * pair + t) * BM;
      const int qrow = q0 + row;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < my_nkv; ++j, ++cs) {
        const int kv0 = j * BN;
        const bool alt = alt_item && j < na;
        mbar_wait(&s_full[t], cs & 1);
        if (lane == 0 && (warp == 2 || warp == 2 + kSoft)) UL_EV(warp == 2 ? 4 : 7, cs);   // (trace) s_full seen
#ifdef UL_FWD_XP_NOSOFT   // (what-if flag: no softmax work at all; results wrong)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&p_part[t]);
          mbar_arrive(&p_full[t]);
        }
        continue;
#endif
        tc_fence_after();
        uint32_t r[kC];
#pragma unroll
        for (int c = 0; c < kC; c += 32) tmem_ld32(tS + half * kC + c, r + c);
        tmem_wait_ld();
        const bool masked = (p.causal && kv0 + BN - 1 > q0) || kv0 + BN > p.n;
        if (masked) {
          int limit = p.n - kv0;
          if (p.causal) limit = min(limit, qrow - kv0 + 1);
          limit -= half * kC;
#pragma unroll
          for (int c = 0; c < kC; ++c)
            if (c >= limit) r[c] = __float_as_uint(-INFINITY);
        }
        float mx[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx[u] = __uint_as_float(r[u]);
#pragma unroll
        for (int c = 8; c < kC; c += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mx[u] = fmaxf(mx[u], __uint_as_float(r[c + u]));
        }
        float mh =
            fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        if constexpr (WPR == 2) {
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot(cs & 1, half)), "f"(mh) : "memory");
          pair_sync();
          float other;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(xslot(cs & 1, half ^ 1)) : "memory");
          mh = fmaxf(mh, other);
        }
        const float mt = mh * p.scale_log2;
        float alpha = 1.f;
        bool rescale = false;
        if (mt > m + kLazy) {
          alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mt);
          rescale = (j > 0);
          m = mt;
        }
        const float mu = (m == -INFINITY) ? 0.f : m;
        float2 rsum[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};
        // O holds PV(0..j-1); S(j) completing implies PV(j-1) did (in-order tensor pipe)
        auto rescale_o = [&]() {
#pragma unroll
          for (int c = 0; c < kOC / 32; ++c) {
            uint32_t ov[32];
            tmem_ld32(tO + half * kOC + c * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 32; ++x) ov[x] = __float_as_uint(__uint_as_float(ov[x]) * alpha);
            tmem_st32(tO + half * kOC + c * 32, ov);
          }
        };
        // a warp whose rows need O rescaled announces the split only after it
        // (rare: lazy rescale); the others as soon as P of kv < 96 is stored
        const bool any_rs = __any_sync(0xffffffffu, rescale);
        if (lane == 0 && (warp == 2 || warp == 2 + kSoft)) UL_EV(warp == 2 ? 5 : 8, cs);   // (trace) exps start
        if (alt) alt_sync(9 + t, 64 * kSoft);   // the other tile's exponentials are done
#pragma unroll
        for (int c = 0; c < kC; c += 32) {
          uint32_t pk[16];
          if (UL_FWD_FULL_POLY_MASK != 0 && !masked)
            exp_chunk<UL_FWD_FULL_POLY_MASK != 0, UL_FWD_FULL_POLY_MASK>(r + c, p.scale_log2, mu, pk, rsum);
          else
            exp_chunk<false>(r + c, p.scale_log2, mu, pk, rsum);
          tmem_st16(tS + (half * kC + c) / 2, pk);   // P (bf16 pairs) over consumed S columns
#if UL_FWD_SPLITP
          // P of kv columns < kSplitAt complete after this chunk: announce it
          if (!any_rs &&
              (half * kC + c + 32 == kSplitAt || (half * kC + c + 32 < kSplitAt && c + 32 == kC))) {
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_part[t]);
            if (lane == 0 && (warp == 2 || warp == 2 + kSoft)) UL_EV(warp == 2 ? 11 : 14, cs);   // (trace) p_part arrive
          }
#endif
        }
        if (alt && (t == 0 || j + 1 < na)) alt_arrive(9 + (t ^ 1), 64 * kSoft);
        const float2 rs = __fadd2_rn(__fadd2_rn(rsum[0], rsum[1]), __fadd2_rn(rsum[2], rsum[3]));
        l = l * alpha + (rs.x + rs.y);
        if (any_rs) rescale_o();
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
#if UL_FWD_SPLITP
        if (any_rs && lane == 0) mbar_arrive(&p_part[t]);
#endif
        if (lane == 0) mbar_arrive(&p_full[t]);
        if (lane == 0 && (warp == 2 || warp == 2 + kSoft)) UL_EV(warp == 2 ? 6 : 9, cs);   // (trace) p_full arrive
      }
      float lo = 0.f;
      if constexpr (WPR == 2) {
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot(2, half)), "f"(l) : "memory");
        pair_sync();
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(lo) : "r"(xslot(2, half ^ 1)) : "memory");
        pair_sync();   // (the sum slot is rewritten by the next item)
      }
      const float lrow = l + lo;
      mbar_wait(&o_done[t], (cs - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / lrow;
      const bool valid = qrow < p.n;
      uint32_t pkd[kOC / 32][16];
#pragma unroll
      for (int c = 0; c < kOC / 32; ++c) {
        uint32_t ov[32];
        tmem_ld32(tO + half * kOC + c * 32, ov);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < 16; ++x)
          pkd[c][x] = pack_bf16(__uint_as_float(ov[2 * x]) * inv, __uint_as_float(ov[2 * x + 1]) * inv);
      }
      // O is in registers: the next item's first PV of this tile may overwrite it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
      if (valid) {
        __nv_bfloat16* orow = p.o + (((int64_t)qrow * p.b + bb) * p.hq + h) * HD + half * kOC;
#pragma unroll
        for (int c = 0; c < kOC / 32; ++c) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int x = 0; x < 4; ++x)
            dst[x] = make_uint4(pkd[c][4 * x], pkd[c][4 * x + 1], pkd[c][4 * x + 2], pkd[c][4 * x + 3]);
          if (p.ep.active) {
            uint4* pd = reinterpret_cast<uint4*>(peer_row_ptr(p.ep, qrow, bb, p.b, h, HD, 2) + half * kOC * 2) + c * 4;
#pragma unroll
            for (int x = 0; x < 4; ++x)
              pd[x] = make_uint4(pkd[c][4 * x], pkd[c][4 * x + 1], pkd[c][4 * x + 2], pkd[c][4 * x + 3]);
          }
        }
        if (half == 0) p.lse[((int64_t)bb * p.hq + h) * p.n + qrow] = (m + log2f(lrow)) * 0.69314718055994531f;
      }
    }
    if (p.ep.active) __threadfence_system();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {   // CTA life (trace builds): end
    UL_CTA(2, globaltimer());
    UL_CTA(3, globaltimer());
    UL_CTA(6, clock64());
  }
  if (p.ctr && threadIdx.x == 0) {   // every CTA has taken its last index: the last one resets
    __threadfence();
    if (atomicAdd(p.ctr + 1, 1) == (int)gridDim.x - 1) {
      atomicExch(p.ctr, 0);
      atomicExch(p.ctr + 1, 0);
    }
  }
  if (p.ep.active && threadIdx.x == 0) peer_signal_last_cta(p.ep, gridDim.x);
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// ---------------------------------------------------------------------------
// Half-unit forward (UL_FWD_H2=1, A/B; the hd-128 default until r2, now
// slower than the split-P full-tile kernel above): the persistent
// kernel above with every 128-column K/V tile processed as two 64-column
// units, each query tile's S region split into two 64-column buffers.
//
// Why: in the kernel above S_t(j+1) overwrites the TMEM columns PV_t(j) reads
// P_t(j) from, so each query tile runs the serial chain softmax(j) -> PV(j)
// -> S(j+1) -> softmax(j+1) and the tensor pipe idles whenever a softmax
// takes longer than the other tile's two GEMMs (ncu: tensor pipe 53% active).
// Here unit u lives in buffer u & 1: S_t(u + 1) is computed while
// softmax_t(u) runs, and only S_t(u + 2) waits for PV_t(u).  Per 128 kv
// columns the pipe then runs 2 x (2 PV + 2 S) with no chain bubble; the
// N = 64 S MMAs read 6 KB of shared memory per 32-cycle K-step (2/3 rate) --
// ~2560 instead of 2048 tensor cycles, against ~3900 measured for the chain.
//   MMA order per unit u:  PV_A(u), S_A(u + 2), PV_B(u), S_B(u + 2).
//   TMEM: tile t: S buffers t*128 + {0, 64} (P packed over the consumed S),
//         O_t at 256 + t*128.
//   Softmax: 8 warps per tile, two per TMEM lane quarter, each owning 32 of
//   the unit's 64 columns (row max combined through shared memory); O is
//   rescaled lazily (after PV_t(u - 1), which then has to be complete).
constexpr int kUN = 64;   // kv columns per unit

template <int HD>
struct SmemH2 {
  static constexpr int kTile = (HD / 64) * kAtom;
  static constexpr int kQ = 0;                    // [2] (tile A, tile B)
  static constexpr int kK = kQ + 2 * kTile;       // [NS]
  static constexpr int kV = kK + NS * kTile;      // [NS]
  static constexpr int kBar = kV + NS * kTile;    // 512 B of barriers
  static constexpr int kX = kBar + 512;           // row max / sum exchange [3][2 tiles][128][2]
  static constexpr int kBytes = kX + 3 * 2 * 128 * 2 * 4 + 1024;
};

// WPR: softmax warps per query row (2: two warps per TMEM lane quarter, 32
// of a unit's 64 columns each, row max exchanged through shared memory;
// 1: one thread per row, all 64 columns, no exchange)
template <int WPR>
constexpr int h2_threads() { return 64 + 2 * 4 * WPR * 32; }

template <int HD, int WPR>
__global__ void __launch_bounds__(h2_threads<WPR>(), 1)
    attn_fwd_h2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const Params p) {
  static_assert(HD == 128, "half-unit forward: TMEM holds 2 x (2 x 64 S + HD O) columns");
  constexpr int kSoft = 4 * WPR;         // softmax warps per query tile
  constexpr int kC = kUN / WPR;          // unit columns per softmax thread
  constexpr int kOC = HD / WPR;          // O columns per softmax thread
  using S = SmemH2<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sK = smem + S::kK;
  uint8_t* sV = smem + S::kV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::kBar);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;              // [NS]
  uint64_t* k_empty = bars + 2 + NS;        // [NS]
  uint64_t* v_full = bars + 2 + 2 * NS;     // [NS]
  uint64_t* v_empty = bars + 2 + 3 * NS;    // [NS]
  uint64_t* s_full = bars + 2 + 4 * NS;     // [tile][buffer]
  uint64_t* p_full = bars + 6 + 4 * NS;     // [tile][buffer]
  // [tile][buffer]: one phase per PV of that buffer's units.  Per buffer, a
  // waiter is never more than one phase behind: s_full(u) implies PV(u - 2)
  // (same buffer) completed, because S(u) was issued after it.
  uint64_t* o_done = bars + 10 + 4 * NS;
  uint64_t* o_free = bars + 14 + 4 * NS;    // [tile]: O read out by the epilogue
  uint64_t* it_full = bars + 16 + 4 * NS;   // [4] dynamic item ring
  uint64_t* it_empty = bars + 20 + 4 * NS;  // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24 + 4 * NS);
  volatile int* sitem = reinterpret_cast<volatile int*>(bars + 25 + 4 * NS);
  static_assert((27 + 4 * NS) * 8 <= 512, "barrier area");
  auto item = [&](int k, int& pair, int& bh, int role) {
    return p.ctr ? fwd_item_dyn<HD>(p, k, pair, bh, role, it_full, it_empty, sitem) : fwd_item<HD>(p, k, pair, bh);
  };
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nkv_all = (p.n + BN - 1) / BN;
  auto item_kv = [&](int pair, int t) {
    const int qt = 2 * pair + t;
    return qt >= p.qtiles ? 0 : (p.causal ? min(nkv_all, (qt * BM + BM - 1) / BN + 1) : nkv_all);
  };

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], kSoft);
      mbar_init(&o_done[i], 1);
    }
    for (int t = 0; t < 2; ++t) mbar_init(&o_free[t], kSoft);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&it_full[s], 1);
      mbar_init(&it_empty[s], 1 + 2 * kSoft);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    UL_CTA(0, globaltimer());
    UL_CTA(1, globaltimer());
    UL_CTA(4, smid());
    UL_CTA(5, clock64());
  }
  tc_fence_after();
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tbase = 0;

  if (warp == 0) {
    // ---------------- TMA producer (128-row K / V tiles, as above) ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      int pair, bh, gk = 0;
      for (int k = 0; item(k, pair, bh, 0); ++k) {
        const int bb = bh / p.hq, h = bh % p.hq, g = h / (p.hq / p.hkv);
        const int n0 = item_kv(pair, 0), n1 = item_kv(pair, 1);
        const int nkv = max(n0, n1), ntiles = n1 > 0 ? 2 : 1;
        if (k > 0) mbar_wait(q_empty, (k - 1) & 1);
        mbar_expect_tx(q_full, ntiles * BM * HD * 2);
        for (int t = 0; t < ntiles; ++t)
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load_3d(sQ + t * S::kTile + a * kAtom, &tmQ, q_full, a * 64, bb * p.hq + h, (2 * pair + t) * BM);
        for (int j = 0; j < nkv; ++j, ++gk) {
          const int s = gk % NS;
          const uint32_t ph = (gk / NS) & 1;
          mbar_wait_prod(&k_empty[s], ph ^ 1);
          UL_EV(13, gk);
          mbar_expect_tx(&k_full[s], BN * HD * 2);
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load_3d(sK + s * S::kTile + a * kAtom, &tmK, &k_full[s], a * 64, bb * p.hkv + g, j * BN);
          mbar_wait_prod(&v_empty[s], ph ^ 1);
          UL_EV(14, gk);
          mbar_expect_tx(&v_full[s], BN * HD * 2);
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load_3d(sV + s * S::kTile + a * kAtom, &tmV, &v_full[s], a * 64, bb * p.hkv + g, j * BN);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {
      constexpr uint32_t kIdQK = idesc_bf16(BM, kUN, 0, 0);   // S unit: M = 128 q rows, N = 64 kv
      constexpr uint32_t kIdPV = idesc_bf16(BM, HD, 0, 1);    // O += P V: K = 64 kv per unit
      const uint64_t dQ0 = sdesc(smem_u32(sQ), 16, 1024);
      const uint64_t dK0 = sdesc(smem_u32(sK), 16, 1024);
      const uint64_t dV0 = sdesc(smem_u32(sV), kAtom, 1024);
      int cp[4] = {0, 0, 0, 0};   // p_full waits per (tile, buffer)
      int items_t[2] = {0, 0};    // items in which the tile existed so far
      // S_t(unit) from K rows (unit & 1) * 64 of stage `stage`
      auto issue_s = [&](int t, int unit, int stage) {
        const int bf = unit & 1;
        const uint64_t dk = dadd(dK0, stage * S::kTile + bf * (kUN * 128));
        const uint64_t dq = dadd(dQ0, t * S::kTile);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
          mma_ss(tbase + t * 128 + bf * kUN, dadd(dq, off), dadd(dk, off), kIdQK, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[t * 2 + bf]);
      };
      // O_t += P_t(unit) V rows (unit & 1) * 64 of stage `stage`
      auto issue_pv = [&](int t, int unit, int stage) {
        const int bf = unit & 1;
        if (unit == 0 && items_t[t] > 0) mbar_wait_mma(&o_free[t], (items_t[t] - 1) & 1);
        mbar_wait_mma(&p_full[t * 2 + bf], cp[t * 2 + bf] & 1);
        ++cp[t * 2 + bf];
        UL_EV(t == 0 ? 0 : 2, cp[t * 2] + cp[t * 2 + 1] - 1);
        tc_fence_after();
        const uint64_t dv = dadd(dV0, stage * S::kTile + bf * (kUN * 128));
#pragma unroll
        for (int kk = 0; kk < kUN / 16; ++kk)
          mma_ts(tbase + 256 + t * HD, tbase + t * 128 + bf * kUN + kk * 8, dadd(dv, kk * 2048), kIdPV,
                 (unit > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&o_done[t * 2 + bf]);
        UL_EV(t == 0 ? 1 : 3, cp[t * 2] + cp[t * 2 + 1] - 1);
      };
      int pair, bh, gk = 0;
      for (int k = 0; item(k, pair, bh, 1); ++k) {
        const int nU0 = 2 * item_kv(pair, 0), nU1 = 2 * item_kv(pair, 1);
        const int nU = max(nU0, nU1);
        mbar_wait_mma(q_full, k & 1);
        mbar_wait_mma(&k_full[gk % NS], (gk / NS) & 1);
        tc_fence_after();
        for (int t = 0; t < 2; ++t) {
          const int nUt = t ? nU1 : nU0;
          if (nUt > 0) issue_s(t, 0, gk % NS);
          if (nUt > 1) issue_s(t, 1, gk % NS);
        }
        mma_commit(&k_empty[gk % NS]);
        if (nU <= 2) mma_commit(q_empty);
        for (int u = 0; u < nU; ++u) {
          const int j = u >> 1;
          const int s = (gk + j) % NS;
          const int nu = u + 2;                       // the unit whose S follows PV(u) into the same buffer
          const int sn = (gk + (nu >> 1)) % NS;
          UL_EV(10, cp[0] + cp[1]);   // (trace builds) loop top of tile A's unit
          if ((u & 1) == 0) {
            mbar_wait_mma(&v_full[s], ((gk + j) / NS) & 1);
            UL_EV(11, cp[0] + cp[1]);
            if (nu < nU) mbar_wait_mma(&k_full[sn], ((gk + (nu >> 1)) / NS) & 1);
            tc_fence_after();
          }
          UL_EV(12, cp[0] + cp[1]);   // K / V of the unit landed
          if (u < nU0) issue_pv(0, u, s);
          if (nu < nU0) issue_s(0, nu, sn);
          if (u < nU1) issue_pv(1, u, s);
          if (nu < nU1) issue_s(1, nu, sn);
          if (u & 1) mma_commit(&v_empty[s]);        // both halves of V_j read by both tiles
          if (nu < nU && (nu & 1)) mma_commit(&k_empty[sn]);
          if (nu == nU - 1) mma_commit(q_empty);      // the item's last S MMAs: Q may be replaced
        }
        if (nU0 > 0) ++items_t[0];
        if (nU1 > 0) ++items_t[1];
        gk += nU >> 1;
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax / lazy correction / epilogue ----------------
    const int idx = warp - 2;
    const int t = idx / kSoft;
    const int quarter = warp & 3;
    const int half = (idx % kSoft) >> 2;       // which kC of the unit's 64 columns (WPR = 2)
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t tS = tbase + t * 128 + lane_off;
    const uint32_t tO = tbase + 256 + t * HD + lane_off;
    const uint32_t bar_id = 1 + t * 4 + quarter;
    float* xch = reinterpret_cast<float*>(smem + S::kX);
    auto xslot = [&](int sl, int hh) { return smem_u32(xch + ((sl * 2 + t) * 128 + row) * 2 + hh); };
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    int cs[2] = {0, 0};   // S units of each buffer consumed so far (s_full phases)
    int base = 0;         // PVs per buffer of this tile before the current item (o_done phases)
    int pair, bh;
    for (int k = 0; item(k, pair, bh, 2); ++k) {
      const int my_nU = 2 * item_kv(pair, t);
      if (my_nU == 0) continue;
      const int nUa = 2 * item_kv(pair, 0);   // units both tiles have (tile A's <= tile B's)
      const bool alt_item = p.alt && nUa > 0 && item_kv(pair, 1) > 0;
      if (alt_item && t == 1) alt_arrive(9, 64 * kSoft);   // tile A goes first
      const int bb = bh / p.hq, h = bh % p.hq;
      const int q0 = (2 * pair + t) * BM;
      const int qrow = q0 + row;
      float m = -INFINITY, l = 0.f;
      for (int u = 0; u < my_nU; ++u) {
        const int bf = u & 1;
        const int kv0 = u * kUN;
        const bool alt = alt_item && u < nUa;
        mbar_wait(&s_full[t * 2 + bf], cs[bf] & 1);
        ++cs[bf];
#ifdef UL_FWD_XP_NOSOFT   // (what-if flag: no softmax work at all -- the MMA / TMA pipeline alone; results wrong)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t * 2 + bf]);
        continue;
#endif
        const int ev_i = cs[0] + cs[1] - 1;   // this tile's unit index across items (traces)
        (void)ev_i;
        if (lane == 0 && (warp == 2 || warp == 2 + kSoft)) UL_EV(warp == 2 ? 4 : 7, ev_i);
        tc_fence_after();
        uint32_t r[kC];
#pragma unroll
        for (int c = 0; c < kC; c += 32) tmem_ld32(tS + bf * kUN + half * kC + c, r + c);
        tmem_wait_ld();
        const bool masked = (p.causal && kv0 + kUN - 1 > q0) || kv0 + kUN > p.n;
        if (masked) {
          int limit = p.n - kv0;
          if (p.causal) limit = min(limit, qrow - kv0 + 1);
          limit -= half * kC;
#pragma unroll
          for (int c = 0; c < kC; ++c)
            if (c >= limit) r[c] = __float_as_uint(-INFINITY);
        }
        float mx[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) mx[x] = __uint_as_float(r[x]);
#pragma unroll
        for (int c = 8; c < kC; c += 8) {
#pragma unroll
          for (int x = 0; x < 8; ++x) mx[x] = fmaxf(mx[x], __uint_as_float(r[c + x]));
        }
        float mh =
            fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        if constexpr (WPR == 2) {
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot(bf, half)), "f"(mh) : "memory");
          pair_sync();   // (also: both warps have loaded their S before either stores P over it)
          float other;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(xslot(bf, half ^ 1)) : "memory");
          mh = fmaxf(mh, other);
        }
        const float mt = mh * p.scale_log2;
        float alpha = 1.f;
        bool rescale = false;
        if (mt > m + kLazy) {
          alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mt);
          rescale = (u > 0);
          m = mt;
        }
        const float mu = (m == -INFINITY) ? 0.f : m;
        float2 rsum[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                          make_float2(0.f, 0.f)};
        if (alt) alt_sync(9 + t, 64 * kSoft);       // the other tile's exponentials are done
        if (lane == 0 && (warp == 2 || warp == 2 + kSoft)) UL_EV(warp == 2 ? 5 : 8, ev_i);
#pragma unroll
        for (int c = 0; c < kC; c += 32) {
          uint32_t pk[16];
#ifdef UL_FWD_XP_NOEXP   // (what-if flag: TMEM traffic and row max, no exponentials; results wrong)
#pragma unroll
          for (int x = 0; x < 16; ++x) pk[x] = r[c + 2 * x] ^ r[c + 2 * x + 1];
          tmem_st16(tS + bf * kUN + (half * kC + c) / 2, pk);
          continue;
#endif
#ifdef UL_FWD_POLY
          if (!masked) exp_chunk<true>(r + c, p.scale_log2, mu, pk, rsum);
          else
#endif
          exp_chunk<false>(r + c, p.scale_log2, mu, pk, rsum);
          tmem_st16(tS + bf * kUN + (half * kC + c) / 2, pk);   // P (bf16 pairs) over consumed S columns
        }
        if (alt && (t == 0 || u + 1 < nUa)) alt_arrive(9 + (t ^ 1), 64 * kSoft);
        const float2 rs = __fadd2_rn(__fadd2_rn(rsum[0], rsum[1]), __fadd2_rn(rsum[2], rsum[3]));
        l = l * alpha + (rs.x + rs.y);
        if (__any_sync(0xffffffffu, rescale)) {
          // O holds PV(0..u-1): wait for PV(u-1), the ((u-1)/2)-th of its buffer
          mbar_wait(&o_done[t * 2 + ((u - 1) & 1)], (base + ((u - 1) >> 1)) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < kOC / 32; ++c) {
            uint32_t ov[32];
            tmem_ld32(tO + half * kOC + c * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 32; ++x) ov[x] = __float_as_uint(__uint_as_float(ov[x]) * alpha);
            tmem_st32(tO + half * kOC + c * 32, ov);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t * 2 + bf]);
        if (lane == 0 && (warp == 2 || warp == 2 + kSoft)) UL_EV(warp == 2 ? 6 : 9, ev_i);
      }
      float lo = 0.f;
      if constexpr (WPR == 2) {
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(xslot(2, half)), "f"(l) : "memory");
        pair_sync();
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(lo) : "r"(xslot(2, half ^ 1)) : "memory");
        pair_sync();   // (the sum slot is rewritten by the next item)
      }
      const float lrow = l + lo;
      base += my_nU >> 1;   // (my_nU is even: the same count of PVs in both buffers)
      mbar_wait(&o_done[t * 2 + 0], (base - 1) & 1);
      mbar_wait(&o_done[t * 2 + 1], (base - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / lrow;
      const bool valid = qrow < p.n;
      uint32_t pkd[kOC / 32][16];
#pragma unroll
      for (int c = 0; c < kOC / 32; ++c) {
        uint32_t ov[32];
        tmem_ld32(tO + half * kOC + c * 32, ov);
        tmem_wait_ld();
#pragma unroll
        for (int x = 0; x < 16; ++x)
          pkd[c][x] = pack_bf16(__uint_as_float(ov[2 * x]) * inv, __uint_as_float(ov[2 * x + 1]) * inv);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_free[t]);
      if (valid) {
        __nv_bfloat16* orow = p.o + (((int64_t)qrow * p.b + bb) * p.hq + h) * HD + half * kOC;
#pragma unroll
        for (int c = 0; c < kOC / 32; ++c) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int x = 0; x < 4; ++x)
            dst[x] = make_uint4(pkd[c][4 * x], pkd[c][4 * x + 1], pkd[c][4 * x + 2], pkd[c][4 * x + 3]);
          if (p.ep.active) {
            uint4* pd = reinterpret_cast<uint4*>(peer_row_ptr(p.ep, qrow, bb, p.b, h, HD, 2) + half * kOC * 2) + c * 4;
#pragma unroll
            for (int x = 0; x < 4; ++x)
              pd[x] = make_uint4(pkd[c][4 * x], pkd[c][4 * x + 1], pkd[c][4 * x + 2], pkd[c][4 * x + 3]);
          }
        }
        if (half == 0) p.lse[((int64_t)bb * p.hq + h) * p.n + qrow] = (m + log2f(lrow)) * 0.69314718055994531f;
      }
    }
    if (p.ep.active) __threadfence_system();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    UL_CTA(2, globaltimer());
    UL_CTA(3, globaltimer());
    UL_CTA(6, clock64());
  }
  if (p.ctr && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.ctr + 1, 1) == (int)gridDim.x - 1) {
      atomicExch(p.ctr, 0);
      atomicExch(p.ctr + 1, 0);
    }
  }
  if (p.ep.active && threadIdx.x == 0) peer_signal_last_cta(p.ep, gridDim.x);
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// The persistent forward's [next item, CTAs done] counter pair is caller
// memory (`sched`, UL_ATTN_SCHED_BYTES, zeroed once; the kernel leaves it
// zero): launches sharing one pair must be stream-ordered.  No counter, or a
// stream under capture (a graph may be replayed on several streams at once),
// selects the static zig-zag schedule.
#ifndef UL_FWD_DYNAMIC
#define UL_FWD_DYNAMIC 1
#endif
static int* schedule_counter(void* sched, cudaStream_t st) {
  if (!UL_FWD_DYNAMIC || !sched) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<int*>(sched);
}

// UL_FWD_ALT=1 in the environment turns the tiles' softmax ping-pong on (A/B;
// off by default -- r2 at N = 4K/8K/32K: 0.3-0.8% slower with it; neither a
// quarter of the exponentials on the FMA pipe (4.5% slower) nor 64-row K/V
// unit rings of 4-5 stages (12% slower) helped: the kernel is not MUFU- or
// K/V-latency-bound)
static int fwd_alt_enabled() {
  static const int on = [] {
    const char* e = getenv("UL_FWD_ALT");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return on;
}

// UL_FWD_WPR=1 / 2: softmax warps per query row of the half-unit kernel (A/B;
// default 1 -- r2: one thread per row, 10 warps, 168 registers, no row-max
// exchange: -1.8% at N = 8K, -2.2% at N = 32K vs two warps per row)
static int fwd_wpr() {
  static const int w = [] {
    const char* e = getenv("UL_FWD_WPR");
    return (e && e[0] == '2') ? 2 : 1;
  }();
  return w;
}

// UL_FWD_FULL_WPR=1 / 2: softmax warps per row of the full-tile persistent
// kernel (default 1 -- r2 with the split P arrive: hd 128 config 2 0.250 vs
// 0.261-0.266 ms, hd 64 32 heads x 8K 0.424 vs 0.438 ms; two warps per row
// with interleaved 32-column blocks and the split at 64 columns: 0.261 /
// 0.441, not kept)
static int fwd_full_wpr(int /*hd*/) {
  static const int w = [] {
    const char* e = getenv("UL_FWD_FULL_WPR");
    return (e && e[0] == '2') ? 2 : 1;
  }();
  return w;
}

// UL_FWD_H2=1 in the environment selects the half-unit kernel for hd 128 (A/B;
// default off since r2: the full-tile kernel with the split P arrive and the
// FMA-pipe exponential share is 7% faster at config 2, 9% at N = 32K)
static bool fwd_h2_enabled() {
  static const bool on = [] {
    const char* e = getenv("UL_FWD_H2");
    return e && e[0] == '1';
  }();
  return on;
}

template <int HD>
static int launch(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n, int64_t b,
                  int64_t hq, int64_t hkv, int causal, float scale, const PeerEpilogue* ep, cudaStream_t st,
                  const uint32_t* blk, int64_t blk_bs, int64_t blk_words, void* sched) {
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
  p.pairs = (p.qtiles + 1) / 2;
#ifdef UL_FWD_HEAD_MAJOR
  p.head_major = UL_FWD_HEAD_MAJOR;
#else
  p.head_major = p.pairs >= sm_count();
#endif
  p.scale_log2 = scale * 1.4426950408889634f;
  p.o = (__nv_bfloat16*)o;
  p.lse = lse;
  if (ep) p.ep = *ep;
  else memset(&p.ep, 0, sizeof(p.ep));
  p.blk = blk;
  p.blk_bs = (int)blk_bs;
  p.blk_words = (int)blk_words;
  p.blk_nb = blk ? (int)(n / blk_bs) : 0;
  p.ctr = nullptr;
  p.alt = fwd_alt_enabled();
  if (blk) p.causal = 0;
  const int smem = Smem<HD>::kBytes;
  UL_TRY(smem_opt_in((const void*)attn_fwd_kernel<HD>, smem));
  const int64_t grid = (int64_t)p.pairs * b * hq;
#ifndef UL_FWD_PERSIST
#define UL_FWD_PERSIST 1   // r73: -1.5% vs the one-shot grid; blocked-sparse keeps the one-shot kernel
#endif
  // Items are fetched dynamically from a per-stream counter (greedy
  // longest-first).  Without one (stream capture) the static zig-zag waves
  // are used, which balance the pair-major length ramp but not the per-head
  // sawtooth of head-major orders (r83: N = 64K, 4 heads 3.7 -> 5.1 ms): those
  // keep the one-shot grid then.  (r89: dynamic vs static at config 2 equal;
  // head-major persistent vs one-shot within noise, config 5 -2%.)
  if (UL_FWD_PERSIST && !blk) {
    p.ctr = schedule_counter(sched, st);
    if (p.ctr || !p.head_major) {
      if (HD == 128 && fwd_h2_enabled()) {
        const int hsmem = SmemH2<128>::kBytes;
        const int64_t pgrid = grid < sm_count() ? grid : sm_count();
        if (fwd_wpr() == 1) {
          UL_TRY(smem_opt_in((const void*)attn_fwd_h2_kernel<128, 1>, hsmem));
          attn_fwd_h2_kernel<128, 1><<<(unsigned)pgrid, h2_threads<1>(), hsmem, st>>>(mq, mk, mv, p);
        } else {
          UL_TRY(smem_opt_in((const void*)attn_fwd_h2_kernel<128, 2>, hsmem));
          attn_fwd_h2_kernel<128, 2><<<(unsigned)pgrid, h2_threads<2>(), hsmem, st>>>(mq, mk, mv, p);
        }
        return launched("attn_fwd_sm100");
      }
      const int64_t pgrid = grid < sm_count() ? grid : sm_count();
      if (fwd_full_wpr(HD) == 1) {
        UL_TRY(smem_opt_in((const void*)attn_fwd_persist_kernel<HD, 1>, smem));
        attn_fwd_persist_kernel<HD, 1><<<(unsigned)pgrid, persist_threads<1>(), smem, st>>>(mq, mk, mv, p);
      } else {
        UL_TRY(smem_opt_in((const void*)attn_fwd_persist_kernel<HD, 2>, smem));
        attn_fwd_persist_kernel<HD, 2><<<(unsigned)pgrid, persist_threads<2>(), smem, st>>>(mq, mk, mv, p);
      }
      return launched("attn_fwd_sm100");
    }
    p.ctr = nullptr;
  }
  attn_fwd_kernel<HD><<<(unsigned)grid, kThreads, smem, st>>>(mq, mk, mv, p);
  return launched("attn_fwd_sm100");
}

}  // namespace fwd

#ifdef UL_TRACE
extern "C" int ul_debug_trace_fwd(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, fwd::g_trace, bytes < sizeof(fwd::g_trace) ? bytes : sizeof(fwd::g_trace)) ==
                 cudaSuccess
             ? 0
             : -1;
}
extern "C" int ul_debug_cta_fwd(void* host, size_t bytes) {
  return cudaMemcpyFromSymbol(host, fwd::g_cta, bytes < sizeof(fwd::g_cta) ? bytes : sizeof(fwd::g_cta)) ==
                 cudaSuccess
             ? 0
             : -1;
}
#endif

int preload_fwd() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_kernel<64>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_kernel<128>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_persist_kernel<64, 1>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_persist_kernel<64, 2>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_persist_kernel<128, 1>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_persist_kernel<128, 2>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_h2_kernel<128, 1>));
  UL_CUDA(cudaFuncGetAttributes(&a, fwd::attn_fwd_h2_kernel<128, 2>));
  // dynamic shared-memory opt-ins now, not at the first launch (common.cuh)
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_kernel<64>, fwd::Smem<64>::kBytes));
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_kernel<128>, fwd::Smem<128>::kBytes));
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_persist_kernel<64, 1>, fwd::Smem<64>::kBytes));
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_persist_kernel<64, 2>, fwd::Smem<64>::kBytes));
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_persist_kernel<128, 1>, fwd::Smem<128>::kBytes));
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_persist_kernel<128, 2>, fwd::Smem<128>::kBytes));
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_h2_kernel<128, 1>, fwd::SmemH2<128>::kBytes));
  UL_TRY(smem_opt_in((const void*)fwd::attn_fwd_h2_kernel<128, 2>, fwd::SmemH2<128>::kBytes));
  return UL_OK;
}

int sm100_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n, int64_t b, int64_t hq,
               int64_t hkv, int64_t hd, int causal, float scale, cudaStream_t st, const PeerEpilogue* ep,
               const uint32_t* blk, int64_t blk_bs, int64_t blk_words, void* sched) {
  if (blk && (n + fwd::BN - 1) / fwd::BN > fwd::kMaxTiles)
    return fail(UL_ERR_SHAPE, "blocked-sparse attention supports n <= %d, got %lld", fwd::kMaxTiles * fwd::BN,
                (long long)n);
  switch (hd) {
    case 64: return fwd::launch<64>(q, k, v, o, lse, n, b, hq, hkv, causal, scale, ep, st, blk, blk_bs, blk_words, sched);
    case 128:
      return fwd::launch<128>(q, k, v, o, lse, n, b, hq, hkv, causal, scale, ep, st, blk, blk_bs, blk_words,
                              sched);
    default:
      return fail(UL_ERR_KERNEL, "bf16 attention supports head_dim 64 or 128, got %lld", (long long)hd);
  }
}

}  // namespace ul
