// extern "C" entry points for the local-attention plugin (ul_attn_*) and
// library-level utilities.  Argument validation mirrors the reference's
// error taxonomy (kernels.py:22-28, layers.py:53-57, tensor.py:23-32).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cmath>
#include <string>

#include "comm.cuh"
#include "common.cuh"

namespace ul {

std::string& last_error() {
  static thread_local std::string s;
  return s;
}
int& launch_count() {
  static thread_local int n = 0;
  return n;
}
static std::atomic<uint64_t> g_total_launches{0};
void count_launch() { g_total_launches.fetch_add(1, std::memory_order_relaxed); }

int simt_fwd(const float* q, const float* k, const float* v, float* o, float* lse, int64_t n, int64_t b,
             int64_t hq, int64_t hkv, int64_t hd, int causal, float scale, cudaStream_t st,
             const uint32_t* blk = nullptr, int64_t blk_bs = 0, int64_t blk_words = 0);
int simt_bwd(const float* q, const float* k, const float* v, const float* o, const float* dout,
             const float* lse, float* dq, float* dk, float* dv, float* Dws, int64_t n, int64_t b, int64_t hq,
             int64_t hkv, int64_t hd, int causal, float scale, cudaStream_t st);
int sm100_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n, int64_t b,
              int64_t hq, int64_t hkv, int64_t hd, int causal, float scale, cudaStream_t st,
              const PeerEpilogue* ep = nullptr, const uint32_t* blk = nullptr, int64_t blk_bs = 0,
              int64_t blk_words = 0, void* sched = nullptr);
int sm100_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
              void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, int64_t n, int64_t b, int64_t hq,
              int64_t hkv, int64_t hd, int causal, float scale, int stages, int deterministic, cudaStream_t st,
              const PeerEpilogue* eps = nullptr);
size_t sm100_bwd_workspace(int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd);
int preload_a2a();
int preload_simt();
int preload_fwd();
int preload_bwd();
int preload_proj();
int preload_merge();
int preload_block();

// First launch of each attention kernel variant, once per device, at group
// creation.  Measured (r2, tools/debug_pipe.py): the first in-process layer
// call of a process deadlocked until the flag wait's timeout -- rank 1's
// attention kernel could not start while rank 0's wait spun -- and any P = 1
// attention launch earlier in the process avoided it; setting the kernels'
// attributes, the shared-memory carveout and the local-memory pool up front
// did not.  Whatever the driver does at a kernel's first launch, it happens
// here, where no rank of an in-process group has work queued.
static int launch_warmup() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  UL_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return UL_OK;
  const int64_t n = 256, hq = 2, hkv = 1;
  const size_t tens = (size_t)n * hq * 128 * 4;            // one q-sized tensor (fp32 upper bound)
  const size_t ws = sm100_bwd_workspace(n, 1, hq, hkv, 128);
  char* buf = nullptr;
  UL_CUDA(cudaMalloc(&buf, 8 * tens + ws + 4096));
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemsetAsync(buf, 0, 8 * tens + ws + 4096, s);
  int rc = UL_OK;
  if (e == cudaSuccess) {
    char *q = buf, *k = buf + tens, *v = buf + 2 * tens, *o = buf + 3 * tens, *dout = buf + 4 * tens;
    char *dq = buf + 5 * tens, *dk = buf + 6 * tens, *dv = buf + 7 * tens, *w = buf + 8 * tens;
    float* lse = reinterpret_cast<float*>(w + ws);            // n * hq floats (2 KB)
    void* sched = w + ws + 2048;                                 // zeroed, left zero by the kernel
    for (int hd : {64, 128}) {
      for (int causal : {0, 1}) {
        if (rc == UL_OK) rc = sm100_fwd(q, k, v, o, lse, n, 1, hq, hkv, hd, causal, 0.1f, s);
        if (rc == UL_OK) rc = sm100_fwd(q, k, v, o, lse, n, 1, hq, hkv, hd, causal, 0.1f, s, nullptr, nullptr, 0, 0,
                                        sched);   // (persistent grid with the dynamic schedule)
        for (int det : {0, 1})
          if (rc == UL_OK)
            rc = sm100_bwd(q, k, v, o, dout, lse, dq, dk, dv, w, ws, n, 1, hq, hkv, hd, causal, 0.1f, 7, det, s);
      }
    }
    if (rc == UL_OK)
      rc = simt_fwd((const float*)q, (const float*)k, (const float*)v, (float*)o, lse, 64, 1, hq, hkv, 64, 1, 0.1f, s);
    e = cudaStreamSynchronize(s);
  }
  if (s) cudaStreamDestroy(s);
  cudaFree(buf);
  cudaGetLastError();
  if (rc != UL_OK) return rc;
  if (e != cudaSuccess) return fail(UL_ERR_CUDA, "kernel warm-up: %s", cudaGetErrorString(e));
  done.fetch_or(bit, std::memory_order_release);
  return UL_OK;
}

static int check_attn(int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd, int dtype, int mask) {
  if (mask != UL_MASK_NONE && mask != UL_MASK_CAUSAL)
    return fail(UL_ERR_KERNEL, "kernel supports dense/causal masks only, got mask kind %d", mask);
  if (dtype != UL_DTYPE_F32 && dtype != UL_DTYPE_BF16)
    return fail(UL_ERR_KERNEL, "unsupported attention dtype %d", dtype);
  if (n < 0 || b < 0 || hq < 0 || hkv < 0 || hd < 1)
    return fail(UL_ERR_SHAPE, "kernel needs (n, b, heads, hdim) >= 0 with hdim >= 1, got (%lld, %lld, %lld, %lld)",
                (long long)n, (long long)b, (long long)hq, (long long)hd);
  if (hkv < 1 || hq % hkv != 0)
    return fail(UL_ERR_DIVISIBILITY, "kv head count %lld does not divide query head count %lld", (long long)hkv,
                (long long)hq);
  if (dtype == UL_DTYPE_F32 && hd > 256)
    return fail(UL_ERR_KERNEL, "fp32 attention supports head_dim <= 256, got %lld", (long long)hd);
  return UL_OK;
}

}  // namespace ul

using namespace ul;

extern "C" {

int ul_abi_version(void) { return UL_ABI_VERSION; }
const char* ul_last_error(void) { return last_error().c_str(); }
int ul_last_launch_count(void) { return launch_count(); }
uint64_t ul_total_launch_count(void) { return g_total_launches.load(); }


int ul_preload_kernels(void) {
  UL_TRY(preload_a2a());
  UL_TRY(preload_simt());
  UL_TRY(preload_fwd());
  UL_TRY(preload_proj());
  UL_TRY(preload_merge());
  UL_TRY(preload_block());
  UL_TRY(preload_bwd());
  return launch_warmup();
}

int ul_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n, int64_t b,
                int64_t hq, int64_t hkv, int64_t hd, int dtype, int mask, float scale, void* sched, void* stream) {
  launch_count() = 0;
  UL_TRY(check_attn(n, b, hq, hkv, hd, dtype, mask));
  if (!q || !k || !v || !o || !lse) {
    if (n * b * hq == 0) return UL_OK;
    return fail(UL_ERR_ARG, "ul_attn_fwd: NULL tensor");
  }
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(UL_ERR_ARG, "scale must be finite and > 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int causal = mask == UL_MASK_CAUSAL;
  if (dtype == UL_DTYPE_F32)
    return simt_fwd((const float*)q, (const float*)k, (const float*)v, (float*)o, lse, n, b, hq, hkv, hd, causal,
                    scale, st);
  if (n * b * hq == 0) return UL_OK;
  if (n > INT32_MAX / 2) return fail(UL_ERR_SHAPE, "attention: sequence too long (n=%lld)", (long long)n);
  return sm100_fwd(q, k, v, o, lse, n, b, hq, hkv, hd, causal, scale, st, nullptr, nullptr, 0, 0, sched);
}

int ul_attn_fwd_blocked(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n, int64_t b,
                        int64_t hq, int64_t hkv, int64_t hd, int dtype, int64_t block_size,
                        const uint32_t* pattern_bits, int64_t words_per_row, float scale, void* stream) {
  launch_count() = 0;
  UL_TRY(check_attn(n, b, hq, hkv, hd, dtype, UL_MASK_NONE));
  if (block_size < 1) return fail(UL_ERR_ARG, "block_size must be >= 1, got %lld", (long long)block_size);
  if (n % block_size != 0)   // kernels.py:69-70
    return fail(UL_ERR_DIVISIBILITY, "block_size %lld does not divide sequence length %lld", (long long)block_size,
                (long long)n);
  const int64_t nb = n / block_size;
  if (words_per_row < (nb + 31) / 32)
    return fail(UL_ERR_ARG, "pattern rows of %lld words cannot hold %lld key blocks", (long long)words_per_row,
                (long long)nb);
  if (n * b * hq == 0) return UL_OK;
  if (!q || !k || !v || !o || !lse || !pattern_bits) return fail(UL_ERR_ARG, "ul_attn_fwd_blocked: NULL tensor");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(UL_ERR_ARG, "scale must be finite and > 0");
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == UL_DTYPE_F32)
    return simt_fwd((const float*)q, (const float*)k, (const float*)v, (float*)o, lse, n, b, hq, hkv, hd, 0, scale,
                    st, pattern_bits, block_size, words_per_row);
  if (n > INT32_MAX / 2) return fail(UL_ERR_SHAPE, "attention: sequence too long (n=%lld)", (long long)n);
  return sm100_fwd(q, k, v, o, lse, n, b, hq, hkv, hd, 0, scale, st, nullptr, pattern_bits, block_size,
                   words_per_row);
}

size_t ul_attn_bwd_workspace_bytes(int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd, int dtype) {
  const size_t dvec = (size_t)n * b * hq * sizeof(float);
  if (dtype == UL_DTYPE_F32) return dvec;
  return sm100_bwd_workspace(n, b, hq, hkv, hd);
}


int ul_attn_bwd_stages(const void* q, const void* k, const void* v, const void* o, const void* dout,
                       const float* lse, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, int64_t n,
                       int64_t b, int64_t hq, int64_t hkv, int64_t hd, int dtype, int mask, float scale,
                       int stages, int flags, void* stream) {
  launch_count() = 0;
  UL_TRY(check_attn(n, b, hq, hkv, hd, dtype, mask));
  if (n * b * hq == 0) return UL_OK;
  if (!q || !k || !v || !o || !dout || !dq || !dk || !dv)
    return fail(UL_ERR_ARG, "ul_attn_bwd: NULL tensor");
  if (!lse) return fail(UL_ERR_STATE, "backward needs the LSE saved by the forward pass");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(UL_ERR_ARG, "scale must be finite and > 0");
  if (stages < 1 || stages > 7) return fail(UL_ERR_ARG, "stage mask must be in [1, 7], got %d", stages);
  if (flags & ~UL_ATTN_DETERMINISTIC) return fail(UL_ERR_ARG, "unknown backward flags 0x%x", flags);
  const size_t need = ul_attn_bwd_workspace_bytes(n, b, hq, hkv, hd, dtype);
  if (!ws || ws_bytes < need)
    return fail(UL_ERR_ARG, "ul_attn_bwd: workspace of %zu bytes < required %zu", ws_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  const int causal = mask == UL_MASK_CAUSAL;
  if (dtype == UL_DTYPE_F32) {
    if (stages != 7) return fail(UL_ERR_KERNEL, "fp32 backward runs all stages together");
    return simt_bwd((const float*)q, (const float*)k, (const float*)v, (const float*)o, (const float*)dout, lse,
                    (float*)dq, (float*)dk, (float*)dv, (float*)ws, n, b, hq, hkv, hd, causal, scale, st);
  }
  return sm100_bwd(q, k, v, o, dout, lse, dq, dk, dv, ws, ws_bytes, n, b, hq, hkv, hd, causal, scale, stages,
                   flags & UL_ATTN_DETERMINISTIC, st);
}

int ul_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout, const float* lse,
                void* dq, void* dk, void* dv, void* ws, size_t ws_bytes, int64_t n, int64_t b, int64_t hq,
                int64_t hkv, int64_t hd, int dtype, int mask, float scale, int flags, void* stream) {
  return ul_attn_bwd_stages(q, k, v, o, dout, lse, dq, dk, dv, ws, ws_bytes, n, b, hq, hkv, hd, dtype, mask, scale,
                            7, flags, stream);
}

// ---- local attention with the head->seq exchange fused into the epilogue ----

int ul_attn_fwd_exchange(ul_comm* comm, const void* q, const void* k, const void* v, void* o, float* lse,
                         void* seq_out, int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd, int dtype,
                         int mask, float scale, uint64_t label, void* sched, void* stream) {
  if (!seq_out) return fail(UL_ERR_ARG, "ul_attn_fwd_exchange: NULL seq_out");
  const int64_t shape[4] = {n, b, hq, hd};
  // (empty problems take the two-step route: its push kernel still signals)
  const bool fused = comm && ul_comm_world(comm) > 1 && dtype == UL_DTYPE_BF16 && n * b * hq > 0;
  if (!fused) {   // same contract, two steps: attention, then the head->seq exchange
    UL_TRY(ul_attn_fwd(q, k, v, o, lse, n, b, hq, hkv, hd, dtype, mask, scale, sched, stream));
    const int launches = launch_count();
    const void* in[1] = {o};
    void* out[1] = {seq_out};
    UL_TRY(ul_all_to_all(comm, 1, in, out, shape, 4, dtype, 0, 2, label, stream));
    launch_count() += launches;
    return UL_OK;
  }
  launch_count() = 0;
  UL_TRY(check_attn(n, b, hq, hkv, hd, dtype, mask));
  if (!q || !k || !v || !o || !lse) return fail(UL_ERR_ARG, "ul_attn_fwd_exchange: NULL tensor");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(UL_ERR_ARG, "scale must be finite and > 0");
  if (n > INT32_MAX / 2) return fail(UL_ERR_SHAPE, "attention: sequence too long (n=%lld)", (long long)n);
  cudaStream_t st = (cudaStream_t)stream;
  PeerEpilogue ep;
  int slot = 0;
  uint64_t epoch = 0;
  void* outs[1] = {seq_out};
  UL_TRY(a2a_fused_begin(comm, 1, outs, shape, dtype, label, &ep, &slot, &epoch));
  if (n * b * hq > 0)
    UL_TRY(sm100_fwd(q, k, v, o, lse, n, b, hq, hkv, hd, mask == UL_MASK_CAUSAL, scale, st, &ep, nullptr, 0, 0,
                     sched));
  return a2a_fused_finish(comm, 1, outs, shape, dtype, label, slot, epoch, st);
}

int ul_attn_bwd_exchange(ul_comm* comm, const void* q, const void* k, const void* v, const void* o,
                         const void* dout, const float* lse, void* dq, void* dk, void* dv, void* ws,
                         size_t ws_bytes, void* seq_dq, void* seq_dk, void* seq_dv, int64_t n, int64_t b, int64_t hq,
                         int64_t hkv, int64_t hd, int dtype, int mask, float scale, uint64_t label, int flags,
                         void* stream) {
  if (!seq_dq || !seq_dk || !seq_dv) return fail(UL_ERR_ARG, "ul_attn_bwd_exchange: NULL sequence output");
  const int64_t shapes[12] = {n, b, hq, hd, n, b, hkv, hd, n, b, hkv, hd};
  void* outs[3] = {seq_dq, seq_dk, seq_dv};
  // (empty problems take the two-step route: its push kernel still signals)
  const bool fused = comm && ul_comm_world(comm) > 1 && dtype == UL_DTYPE_BF16 && n * b * hq > 0;
  if (!fused) {
    UL_TRY(ul_attn_bwd(q, k, v, o, dout, lse, dq, dk, dv, ws, ws_bytes, n, b, hq, hkv, hd, dtype, mask, scale, flags,
                       stream));
    const int launches = launch_count();
    const void* in[3] = {dq, dk, dv};
    UL_TRY(ul_all_to_all(comm, 3, in, outs, shapes, 4, dtype, 0, 2, label, stream));
    launch_count() += launches;
    return UL_OK;
  }
  launch_count() = 0;
  UL_TRY(check_attn(n, b, hq, hkv, hd, dtype, mask));
  if (!q || !k || !v || !o || !dout || !dq || !dk || !dv) return fail(UL_ERR_ARG, "ul_attn_bwd_exchange: NULL tensor");
  if (!lse) return fail(UL_ERR_STATE, "backward needs the LSE saved by the forward pass");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(UL_ERR_ARG, "scale must be finite and > 0");
  if (flags & ~UL_ATTN_DETERMINISTIC) return fail(UL_ERR_ARG, "unknown backward flags 0x%x", flags);
  const size_t need = ul_attn_bwd_workspace_bytes(n, b, hq, hkv, hd, dtype);
  if (!ws || ws_bytes < need)
    return fail(UL_ERR_ARG, "ul_attn_bwd: workspace of %zu bytes < required %zu", ws_bytes, need);
  cudaStream_t st = (cudaStream_t)stream;
  PeerEpilogue eps[3];
  int slot = 0;
  uint64_t epoch = 0;
  UL_TRY(a2a_fused_begin(comm, 3, outs, shapes, dtype, label, eps, &slot, &epoch));
  if (n * b * hq > 0)
    UL_TRY(sm100_bwd(q, k, v, o, dout, lse, dq, dk, dv, ws, ws_bytes, n, b, hq, hkv, hd, mask == UL_MASK_CAUSAL,
                     scale, 7, flags & UL_ATTN_DETERMINISTIC, st, eps));
  return a2a_fused_finish(comm, 3, outs, shapes, dtype, label, slot, epoch, st);
}

}  // extern "C"
