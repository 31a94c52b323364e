// fp32 mode of the local-attention plugin: SIMT kernels with fp32
// inputs/outputs and float64 accumulation/exp/log inside (fp32 outputs then
// carry only their final rounding), for the reference's fp32 parity
// contract (rtol 1e-5 vs the f64 oracle; BASELINE config 1).  tcgen05 has
// no fp32 (only tf32) datapath, so this is the fp32 specialisation of the
// same plugin, not a second backend.  bf16 runs on attn_fwd_sm100.cu /
// attn_bwd_sm100.cu.
//
// Semantics follow _masked_attention (kernels.py:31-40) and
// masked_attention_backward (kernels.py:89-111): scores = q k^T * scale,
// causal visibility kv <= q on global indices (tensor.py:161-162),
// row-max-stabilised softmax (tensor.py:245-249), ctx = probs v;
// dscores = probs * (dprobs - rowsum(dprobs*probs)) * scale, using
// rowsum(dprobs*probs) == rowsum(dctx*ctx) (the FlashAttention identity).
// One warp owns one query row (forward, dQ) or one key row (dK/dV); lanes
// own head-dim columns d = lane + 32 t, so every v/k/q/dO row access is
// coalesced.  No atomics: results are deterministic.
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace ul {
namespace simt {

constexpr int kWarps = 4;
constexpr int kMaxT = 8;  // hd <= 256

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct Dims {
  int64_t n, b, hq, hkv, hd;
  int causal;
  float scale;
  // blocked-sparse forward (Mask.blocked, tensor.py:163-180): bit (qb, kb)
  // of blk[qb * blk_words + kb / 32]; nullptr for dense / causal
  const uint32_t* blk = nullptr;
  int64_t blk_bs = 0, blk_words = 0;
};

// row pointers: x[(row*b + bb)*h + head][hd]
__device__ __forceinline__ int64_t rowoff(int64_t row, int64_t bb, int64_t head, int64_t b, int64_t h,
                                          int64_t hd) {
  return ((row * b + bb) * h + head) * hd;
}

__device__ __forceinline__ double dot_row(const float* __restrict__ a_smem, const float* __restrict__ b,
                                         int hd) {
  double s = 0.0;
  for (int d = 0; d < hd; ++d) s = fma((double)a_smem[d], (double)b[d], s);
  return s;
}

// ---- forward: warp per (query row, batch, head) ---------------------------
__global__ void __launch_bounds__(kWarps * 32) fwd_kernel(const float* __restrict__ q,
                                                          const float* __restrict__ k,
                                                          const float* __restrict__ v,
                                                          float* __restrict__ o,
                                                          float* __restrict__ lse, Dims D) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  const int64_t total = D.n * D.b * D.hq;
  if (gw >= total) return;
  const int64_t h = gw % D.hq;
  const int64_t bb = (gw / D.hq) % D.b;
  const int64_t i = gw / (D.hq * D.b);
  const int64_t g = h / (D.hq / D.hkv);
  const int hd = (int)D.hd;
  float* qs = sm + warp * hd;
  const float* qrow = q + rowoff(i, bb, h, D.b, D.hq, hd);
  for (int d = lane; d < hd; d += 32) qs[d] = qrow[d];
  __syncwarp();
  double acc[kMaxT];
#pragma unroll
  for (int t = 0; t < kMaxT; ++t) acc[t] = 0.0;
  double m = -INFINITY, l = 0.0;
  const int64_t jmax = D.causal ? i + 1 : D.n;
  const int64_t kvstride = D.b * D.hkv * hd;
  const float* kbase = k + rowoff(0, bb, g, D.b, D.hkv, hd);
  const float* vbase = v + rowoff(0, bb, g, D.b, D.hkv, hd);
  const uint32_t* brow = D.blk ? D.blk + (i / D.blk_bs) * D.blk_words : nullptr;
  for (int64_t j0 = 0; j0 < jmax; j0 += 32) {
    const int64_t j = j0 + lane;
    bool vis = j < jmax;
    if (vis && brow) {
      const int64_t kb = j / D.blk_bs;
      vis = (__ldg(brow + (kb >> 5)) >> (kb & 31)) & 1u;
    }
    double s = -INFINITY;
    if (vis) s = dot_row(qs, kbase + j * kvstride, hd) * (double)D.scale;
    const double cmax = warp_max(s);
    const double mnew = fmax(m, cmax);
    const double p = vis ? exp(s - mnew) : 0.0;
    const double alpha = (m == -INFINITY) ? 0.0 : exp(m - mnew);
    l = l * alpha + warp_sum(p);
    m = mnew;
#pragma unroll
    for (int t = 0; t < kMaxT; ++t) acc[t] *= alpha;
    const int cnt = (int)(jmax - j0 < 32 ? jmax - j0 : 32);
    for (int jj = 0; jj < cnt; ++jj) {
      const double pj = __shfl_sync(0xffffffffu, p, jj);
      const float* vr = vbase + (j0 + jj) * kvstride;
#pragma unroll
      for (int t = 0; t < kMaxT; ++t) {
        const int d = lane + 32 * t;
        if (d < hd) acc[t] = fma(pj, (double)vr[d], acc[t]);
      }
    }
  }
  const double inv = 1.0 / l;
  float* orow = o + rowoff(i, bb, h, D.b, D.hq, hd);
#pragma unroll
  for (int t = 0; t < kMaxT; ++t) {
    const int d = lane + 32 * t;
    if (d < hd) orow[d] = (float)(acc[t] * inv);
  }
  if (lane == 0) lse[(bb * D.hq + h) * D.n + i] = (float)(m + log(l));
}

// ---- backward pre-pass: D_i = rowsum(dO_i * O_i) ---------------------------
__global__ void __launch_bounds__(kWarps * 32) dot_kernel(const float* __restrict__ o,
                                                          const float* __restrict__ dout,
                                                          float* __restrict__ Dv, Dims D) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  if (gw >= D.n * D.b * D.hq) return;
  const int64_t h = gw % D.hq, bb = (gw / D.hq) % D.b, i = gw / (D.hq * D.b);
  const int64_t off = rowoff(i, bb, h, D.b, D.hq, D.hd);
  double s = 0.0;
  for (int d = lane; d < D.hd; d += 32) s = fma((double)o[off + d], (double)dout[off + d], s);
  s = warp_sum(s);
  if (lane == 0) Dv[(bb * D.hq + h) * D.n + i] = (float)s;
}

// ---- dQ: warp per query row -------------------------------------------------
__global__ void __launch_bounds__(kWarps * 32) dq_kernel(const float* __restrict__ q,
                                                         const float* __restrict__ k,
                                                         const float* __restrict__ v,
                                                         const float* __restrict__ dout,
                                                         const float* __restrict__ lse,
                                                         const float* __restrict__ Dv,
                                                         float* __restrict__ dq, Dims D) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  if (gw >= D.n * D.b * D.hq) return;
  const int64_t h = gw % D.hq, bb = (gw / D.hq) % D.b, i = gw / (D.hq * D.b);
  const int64_t g = h / (D.hq / D.hkv);
  const int hd = (int)D.hd;
  float* qs = sm + warp * 2 * hd;
  float* ds_ = qs + hd;
  const int64_t off = rowoff(i, bb, h, D.b, D.hq, hd);
  for (int d = lane; d < hd; d += 32) {
    qs[d] = q[off + d];
    ds_[d] = dout[off + d];
  }
  __syncwarp();
  const double L = lse[(bb * D.hq + h) * D.n + i];
  const double Di = Dv[(bb * D.hq + h) * D.n + i];
  double acc[kMaxT];
#pragma unroll
  for (int t = 0; t < kMaxT; ++t) acc[t] = 0.0;
  const int64_t jmax = D.causal ? i + 1 : D.n;
  const int64_t kvstride = D.b * D.hkv * hd;
  const float* kbase = k + rowoff(0, bb, g, D.b, D.hkv, hd);
  const float* vbase = v + rowoff(0, bb, g, D.b, D.hkv, hd);
  for (int64_t j0 = 0; j0 < jmax; j0 += 32) {
    const int64_t j = j0 + lane;
    double dsc = 0.0;
    if (j < jmax) {
      const double s = dot_row(qs, kbase + j * kvstride, hd) * (double)D.scale;
      const double p = exp(s - L);
      const double dp = dot_row(ds_, vbase + j * kvstride, hd);
      dsc = p * (dp - Di);
    }
    const int cnt = (int)(jmax - j0 < 32 ? jmax - j0 : 32);
    for (int jj = 0; jj < cnt; ++jj) {
      const double x = __shfl_sync(0xffffffffu, dsc, jj);
      const float* kr = kbase + (j0 + jj) * kvstride;
#pragma unroll
      for (int t = 0; t < kMaxT; ++t) {
        const int d = lane + 32 * t;
        if (d < hd) acc[t] = fma(x, (double)kr[d], acc[t]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < kMaxT; ++t) {
    const int d = lane + 32 * t;
    if (d < hd) dq[off + d] = (float)(acc[t] * (double)D.scale);
  }
}

// ---- dK, dV: warp per key row of one kv head, summed over its q-head group --
__global__ void __launch_bounds__(kWarps * 32) dkdv_kernel(const float* __restrict__ q,
                                                           const float* __restrict__ k,
                                                           const float* __restrict__ v,
                                                           const float* __restrict__ dout,
                                                           const float* __restrict__ lse,
                                                           const float* __restrict__ Dv,
                                                           float* __restrict__ dk,
                                                           float* __restrict__ dv, Dims D) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp;
  if (gw >= D.n * D.b * D.hkv) return;
  const int64_t g = gw % D.hkv, bb = (gw / D.hkv) % D.b, j = gw / (D.hkv * D.b);
  const int hd = (int)D.hd;
  float* ks = sm + warp * 2 * hd;
  float* vs = ks + hd;
  const int64_t off = rowoff(j, bb, g, D.b, D.hkv, hd);
  for (int d = lane; d < hd; d += 32) {
    ks[d] = k[off + d];
    vs[d] = v[off + d];
  }
  __syncwarp();
  double ak[kMaxT], av[kMaxT];
#pragma unroll
  for (int t = 0; t < kMaxT; ++t) ak[t] = av[t] = 0.0;
  const int64_t group = D.hq / D.hkv;
  const int64_t qstride = D.b * D.hq * hd;
  const int64_t i0 = D.causal ? j : 0;
  for (int64_t hh = 0; hh < group; ++hh) {
    const int64_t h = g * group + hh;
    const float* qb = q + rowoff(0, bb, h, D.b, D.hq, hd);
    const float* db = dout + rowoff(0, bb, h, D.b, D.hq, hd);
    const float* Lb = lse + (bb * D.hq + h) * D.n;
    const float* Db = Dv + (bb * D.hq + h) * D.n;
    for (int64_t c0 = i0; c0 < D.n; c0 += 32) {
      const int64_t i = c0 + lane;
      double p = 0.0, dsc = 0.0;
      if (i < D.n) {
        const double s = dot_row(ks, qb + i * qstride, hd) * (double)D.scale;
        p = exp(s - (double)Lb[i]);
        const double dp = dot_row(vs, db + i * qstride, hd);
        dsc = p * (dp - (double)Db[i]);
      }
      const int cnt = (int)(D.n - c0 < 32 ? D.n - c0 : 32);
      for (int ii = 0; ii < cnt; ++ii) {
        const double pi = __shfl_sync(0xffffffffu, p, ii);
        const double si = __shfl_sync(0xffffffffu, dsc, ii);
        const float* qr = qb + (c0 + ii) * qstride;
        const float* dr = db + (c0 + ii) * qstride;
#pragma unroll
        for (int t = 0; t < kMaxT; ++t) {
          const int d = lane + 32 * t;
          if (d < hd) {
            av[t] = fma(pi, (double)dr[d], av[t]);
            ak[t] = fma(si, (double)qr[d], ak[t]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < kMaxT; ++t) {
    const int d = lane + 32 * t;
    if (d < hd) {
      dk[off + d] = (float)(ak[t] * (double)D.scale);
      dv[off + d] = (float)av[t];
    }
  }
}

int preload() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, fwd_kernel));
  UL_CUDA(cudaFuncGetAttributes(&a, dot_kernel));
  UL_CUDA(cudaFuncGetAttributes(&a, dq_kernel));
  UL_CUDA(cudaFuncGetAttributes(&a, dkdv_kernel));
  return UL_OK;
}

static unsigned blocks_for(int64_t warps) { return (unsigned)((warps + kWarps - 1) / kWarps); }

}  // namespace simt

int preload_simt() { return simt::preload(); }

int simt_fwd(const float* q, const float* k, const float* v, float* o, float* lse, int64_t n, int64_t b,
             int64_t hq, int64_t hkv, int64_t hd, int causal, float scale, cudaStream_t st, const uint32_t* blk,
             int64_t blk_bs, int64_t blk_words) {
  simt::Dims D{n, b, hq, hkv, hd, blk ? 0 : causal, scale, blk, blk_bs, blk_words};
  const int64_t rows = n * b * hq;
  if (rows == 0) return UL_OK;
  simt::fwd_kernel<<<simt::blocks_for(rows), simt::kWarps * 32, simt::kWarps * hd * sizeof(float), st>>>(
      q, k, v, o, lse, D);
  return launched("attn_fwd_simt_f32");
}

int simt_bwd(const float* q, const float* k, const float* v, const float* o, const float* dout,
             const float* lse, float* dq, float* dk, float* dv, float* Dws, int64_t n, int64_t b, int64_t hq,
             int64_t hkv, int64_t hd, int causal, float scale, cudaStream_t st) {
  simt::Dims D{n, b, hq, hkv, hd, causal, scale};
  if (n * b * hq == 0) return UL_OK;
  simt::dot_kernel<<<simt::blocks_for(n * b * hq), simt::kWarps * 32, 0, st>>>(o, dout, Dws, D);
  UL_TRY(launched("attn_bwd_dot_f32"));
  simt::dq_kernel<<<simt::blocks_for(n * b * hq), simt::kWarps * 32, simt::kWarps * 2 * hd * sizeof(float),
                    st>>>(q, k, v, dout, lse, Dws, dq, D);
  UL_TRY(launched("attn_bwd_dq_simt_f32"));
  simt::dkdv_kernel<<<simt::blocks_for(n * b * hkv), simt::kWarps * 32,
                      simt::kWarps * 2 * hd * sizeof(float), st>>>(q, k, v, dout, lse, Dws, dk, dv, D);
  return launched("attn_bwd_dkdv_simt_f32");
}

}  // namespace ul
