/*
 * ulysses_b200.h -- C-ABI of the B200-native Ulysses sequence-parallel
 * attention path (DeepSpeed-Ulysses, arXiv 2309.14509).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point returns
 * an int status (UL_OK or a negative UL_ERR_*), never throws or aborts,
 * and is stream-ordered on the caller's cudaStream_t (passed as void*).
 * ul_last_error() returns a thread-local message naming the offending
 * rank / tensor / dimension, worded like the reference's exceptions.
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/seqlab):
 *
 *   ul_all_to_all            RankContext.all_to_all          simgroup.py:453-456
 *                            -> RankGroup._all_to_all        simgroup.py:313-335
 *                            -> RankGroup._exchange          simgroup.py:251-304
 *                            as used by seq_to_head / _to_head (split 2, concat 0)
 *                            ulysses.py:104-111, 161-164 and head_to_seq /
 *                            _to_seq (split 0, concat 2) ulysses.py:114-124, 167-169
 *   ul_comm_*                RankGroup / RankContext identity + rendezvous
 *                            simgroup.py:198-224, 444-451 (ranks are processes/GPUs
 *                            here, not threads)
 *   ul_comm_status           GroupDesyncError poisoning     simgroup.py:228-243, 265-298
 *   ul_attn_fwd              kernel plugin kernel(q,k,v,mask,scale) -> context
 *                            dense_kernel / causal_kernel kernels.py:43-52 over
 *                            _masked_attention kernels.py:31-40 (plus LSE, new)
 *   ul_attn_bwd              masked_attention_backward     kernels.py:89-111
 *   ul_ulysses_volume        costmodel.ulysses_volume       costmodel.py:82-87
 *
 * Tensor layouts are the reference's sequence-major [s, b, h, hd]
 * (ulysses.py:47-48), row-major and contiguous.
 */
#ifndef ULYSSES_B200_H
#define ULYSSES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UL_ABI_VERSION 2

/* ---- status codes: one per reference exception type ------------------ */
#define UL_OK                 0
#define UL_ERR_DIVISIBILITY  -1  /* ShardError simgroup.py:62 / DivisibilityError tensor.py:27 */
#define UL_ERR_DESYNC        -2  /* GroupDesyncError simgroup.py:66 (signature mismatch, timeout) */
#define UL_ERR_KERNEL        -3  /* KernelError kernels.py:22 (mask / dtype / head_dim unsupported) */
#define UL_ERR_STATE         -4  /* ForwardStateError ulysses.py:39 (missing LSE / shape mismatch) */
#define UL_ERR_SHAPE         -5  /* ShapeError tensor.py:23 */
#define UL_ERR_DEGENERATE    -6  /* DegenerateRowError tensor.py:31 */
#define UL_ERR_CUDA          -7  /* CUDA runtime / driver failure */
#define UL_ERR_ARG           -8  /* ValueError (bad argument) */

/* ---- element types -------------------------------------------------- */
#define UL_DTYPE_F32   0   /* fp32 mode: SIMT FFMA kernels, rtol 1e-5 vs the f64 oracle */
#define UL_DTYPE_BF16  1   /* bf16 mode: tcgen05/TMEM/TMA kernels, fp32 accumulation */

/* ---- masks (Mask.kind, tensor.py:109-149) ----------------------------- */
#define UL_MASK_NONE   0   /* Mask.none()   -> dense_kernel  kernels.py:43-46 */
#define UL_MASK_CAUSAL 1   /* Mask.causal() -> causal_kernel kernels.py:49-52 */

#define UL_MAX_RANKS        16
#define UL_MAX_FUSED         4   /* tensors per fused all-to-all launch (Q, K, V, ...) */
#define UL_IPC_HANDLE_BYTES 128  /* cudaIpcMemHandle_t + workspace geometry */

int         ul_abi_version(void);
const char* ul_last_error(void);
/* Load every kernel of the library into the current context now.  CUDA's
 * lazy loading would otherwise load a kernel at its first launch, which can
 * stall the launching thread while one of this rank's flag-wait kernels
 * spins -- a deadlock when several ranks share one process (local groups).
 * ul_comm_create calls it. */
int         ul_preload_kernels(void);

/* ======================================================================
 * Sequence-parallel group: one process per GPU.  Each rank owns a
 * workspace of two receive slots (ping-pong by call parity) plus per-slot
 * signal words; peers map it through CUDA IPC (NVLink/NVSwitch P2P).
 * ==================================================================== */
typedef struct ul_comm ul_comm;

/* Allocate this rank's workspace (2 x slot_bytes + signals) on `device`. */
int ul_comm_create(int rank, int world, int device, size_t slot_bytes, ul_comm** out);
/* Serialise this rank's IPC handle + geometry into handle_out[UL_IPC_HANDLE_BYTES]. */
int ul_comm_export_handle(const ul_comm* comm, void* handle_out);
/* Map every peer's workspace from world * UL_IPC_HANDLE_BYTES handle bytes
 * (gathered in rank order); validates world size and slot geometry. */
int ul_comm_open_peers(ul_comm* comm, const void* all_handles);
/* Host-only check of gathered handles (magic, rank order, world size, slot
 * geometry) -- the signature check of simgroup.py:265-276 applied to the
 * group's setup; ul_comm_open_peers runs it first. */
int ul_comm_validate_handles(const void* all_handles, int world, int rank, size_t slot_bytes);
/* In-process group (one process driving `world` comms on one device, each
 * on its own stream): wires peer pointers directly.  Used by the 1-GPU
 * parity tests so the same kernels run at P = 2/4/8. */
int ul_comm_link_local(ul_comm* const* comms, int world);
int ul_comm_destroy(ul_comm* comm);
int ul_comm_rank(const ul_comm* comm);
int ul_comm_world(const ul_comm* comm);
size_t ul_comm_slot_bytes(const ul_comm* comm);
/* Bound on every device-side flag wait; a timeout is reported as
 * UL_ERR_DESYNC ("timeout in collective ... waiting on ranks [...]"). */
int ul_comm_set_timeout_ms(ul_comm* comm, int64_t ms);
/* Asynchronous error word (written by the device into mapped host memory):
 * UL_OK, or UL_ERR_DESYNC with a message naming the peer, the call label
 * and both signatures (simgroup.py:265-276).  Cleared by reading. */
int ul_comm_status(ul_comm* comm, char* msg, size_t msg_len);
/* Per-rank egress bytes / calls metered by this comm since creation
 * (CommLedger, simgroup.py:88-172). */
int ul_comm_ledger(const ul_comm* comm, uint64_t* calls, uint64_t* egress_bytes,
                   uint64_t* aggregate_bytes);
/* The same counts kept by the GPU: the signalling CTA of every call (the
 * push kernel's last CTA, or the producing kernel's for fused exchanges)
 * adds the call and its bytes to device counters in this rank's signal
 * block.  A blocking read (call after the work has completed). */
int ul_comm_ledger_device(const ul_comm* comm, uint64_t* calls, uint64_t* egress_bytes,
                          uint64_t* aggregate_bytes);

/* Fused all-to-all of n_tensors row-major tensors (each of rank `ndim`
 * <= 4, shape given per tensor in shapes[t*4 .. t*4+ndim)), identical
 * split/concat axes:  out_i = concat_j( split(in_j, P, split_axis)[i],
 * concat_axis ).  Bit-exact byte routing.  comm == NULL means P = 1 (a
 * local copy).  `label_hash` joins the call signature checked across ranks.
 * Launches: one push kernel (local chunk -> out, remote chunks -> peers'
 * receive slot, then release-signal), one flag wait, one slot drain. */
int ul_all_to_all(ul_comm* comm, int n_tensors, const void* const* in, void* const* out,
                  const int64_t* shapes, int ndim, int dtype, int split_axis,
                  int concat_axis, uint64_t label_hash, void* stream);

/* Seq->head exchange of ONE head group (extension: the pipelined layer
 * exchanges group g+1 while group g is being attended).  in[t] is this
 * rank's full sequence shard [nl, b, H_t, hd] (shapes[4t..4t+4), row-major);
 * with Hg_t = H_t / (P * groups), rank i receives the heads
 * { j*H_t/P + group*Hg_t + h : h < Hg_t } of every rank j's shard, rows in
 * source-rank order: out[t] = [nl*P, b, Hg_t, hd].  Equal to ul_all_to_all
 * (split 2, concat 0) of the [nl, b, P*Hg_t, hd] view holding those heads
 * (same slot geometry and signature), read in place from the parent shard.
 * groups = 1 is the plain seq->head flip. */
int ul_all_to_all_head_group(ul_comm* comm, int n_tensors, const void* const* in, void* const* out,
                             const int64_t* shapes, int dtype, int group, int groups,
                             uint64_t label_hash, void* stream);

/* Bytes of receive slot ul_all_to_all needs for these tensors. */
size_t ul_all_to_all_slot_bytes(int n_tensors, const int64_t* shapes, int ndim, int dtype,
                                int split_axis, int concat_axis, int world);

/* ======================================================================
 * Local attention (the `local_attn` plugin after seq->head):
 *   q  [n, b, hq,  hd]      k, v [n, b, hkv, hd]     (hkv | hq, GQA)
 *   o  [n, b, hq,  hd]      lse  [b, hq, n] float32, natural log
 * mask UL_MASK_NONE / UL_MASK_CAUSAL on global indices (kv <= q).
 * bf16: hd in {64, 128}; fp32: hd <= 256.
 * `sched` (may be NULL): caller-owned DEVICE memory of UL_ATTN_SCHED_BYTES,
 * zeroed once before first use, from which the bf16 dense/causal forward's
 * persistent grid fetches its work items (greedy longest-first); the kernel
 * leaves it zeroed again.  Launches sharing one `sched` must be
 * stream-ordered (one per stream).  NULL, or a stream under capture, selects
 * a static schedule.  The library allocates nothing.
 * ==================================================================== */
#define UL_ATTN_SCHED_BYTES 8
int ul_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd,
                int dtype, int mask, float scale, void* sched, void* stream);

/* Blocked-sparse forward (blocked_kernel, kernels.py:55-86; Mask.blocked,
 * tensor.py:147-180): query block qb sees exactly the key blocks kb whose
 * bit is set in pattern_bits[qb * words_per_row + kb / 32] (DEVICE memory,
 * n / block_size rows); within a visible block every key is visible (no
 * causal cut).  The caller validates the pattern against the reference's
 * rules (no empty query block -> DegenerateRowError, blocks in range);
 * block_size must divide n (UL_ERR_DIVISIBILITY).  Forward only, like the
 * reference (masked_attention_backward supports dense/causal only).
 * bf16: hd in {64, 128}, n <= 1M; fp32: SIMT. */
int ul_attn_fwd_blocked(const void* q, const void* k, const void* v, void* o, float* lse,
                        int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd, int dtype,
                        int64_t block_size, const uint32_t* pattern_bits, int64_t words_per_row,
                        float scale, void* stream);

/* dq [n,b,hq,hd], dk/dv [n,b,hkv,hd] (dk/dv summed over each kv head's
 * query group).  workspace >= ul_attn_bwd_workspace_bytes(...).
 * flags (per call; extension, no reference counterpart):
 *   0: bf16 hd-128 backward in one fused kernel (dK, dV and dQ from one
 *      pass; dQ accumulated with fp32 atomics, so it varies in the last
 *      bits run to run);
 *   UL_ATTN_DETERMINISTIC: dK/dV kernel + a dQ kernel that recomputes S and
 *      dP, no atomics: bitwise reproducible (and bitwise P-invariant).
 * hd 64 and fp32 always run the deterministic kernels. */
#define UL_ATTN_DETERMINISTIC 1
size_t ul_attn_bwd_workspace_bytes(int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd,
                                   int dtype);

int ul_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                const void* dout, const float* lse, void* dq, void* dk, void* dv,
                void* workspace, size_t workspace_bytes,
                int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd,
                int dtype, int mask, float scale, int flags, void* stream);

/* Same as ul_attn_bwd restricted to a subset of its launches (bit 0: D/LSE
 * pre-pass, bit 1: dK/dV kernel -- the fused dK/dV/dQ kernel in the default
 * hd-128 mode --, bit 2: dQ kernel -- the dQ fp32->bf16 pass in that mode),
 * in that order; the stages must run in order over one workspace.  Lets
 * callers time or overlap the stages; ul_attn_bwd == stage_mask 7. */
int ul_attn_bwd_stages(const void* q, const void* k, const void* v, const void* o,
                       const void* dout, const float* lse, void* dq, void* dk, void* dv,
                       void* workspace, size_t workspace_bytes,
                       int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd,
                       int dtype, int mask, float scale, int stage_mask, int flags, void* stream);

/* Local attention with the head->seq exchange (K2) fused into the kernels'
 * epilogues: every finished output row goes both to the head-layout tensor
 * (o / dq, dk, dv -- saved for the backward) and straight into its
 * destination rank's sequence layout (the own seq_out, or the peer's receive
 * slot over NVLink); the producing kernel's last CTA publishes the call and
 * the call ends with this rank's flag wait + drain into seq_out.  Equal to
 * ul_attn_fwd + ul_all_to_all(split 0, concat 2) (which fp32 mode, P = 1
 * and empty problems run instead).  A collective: every rank calls it with
 * the same shapes and label.
 *   seq_out [n/P, b, P*hq, hd];  seq_dq [n/P, b, P*hq, hd], seq_dk/dv [n/P, b, P*hkv, hd] */
int ul_attn_fwd_exchange(ul_comm* comm, const void* q, const void* k, const void* v, void* o, float* lse,
                         void* seq_out, int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd,
                         int dtype, int mask, float scale, uint64_t label_hash, void* sched, void* stream);
int ul_attn_bwd_exchange(ul_comm* comm, const void* q, const void* k, const void* v, const void* o,
                         const void* dout, const float* lse, void* dq, void* dk, void* dv,
                         void* workspace, size_t workspace_bytes, void* seq_dq, void* seq_dk,
                         void* seq_dv, int64_t n, int64_t b, int64_t hq, int64_t hkv, int64_t hd,
                         int dtype, int mask, float scale, uint64_t label_hash, int flags, void* stream);

/* RankContext.ring_shift(local, steps, label) (simgroup.py:374-388, 464-465):
 * out[t] on rank i = in[t] of rank (i - steps) mod P, n flat tensors of
 * bytes[t] bytes moved over peer memory; a collective (full barrier) with
 * the reference's metering (aggregate P*local, egress local*steps).
 * comm may be NULL for P = 1 (a copy). */
int ul_ring_shift(ul_comm* comm, int n, const void* const* in, void* const* out, const int64_t* bytes,
                  int steps, uint64_t label_hash, void* stream);

/* Ring attention merge (extension): fold one chunk's normalised context o_s
 * ([n, b, h, hd], dtype) and row LSE lse_s ([b, h, n], natural log) into the
 * running fp32 context o_acc and lse_acc: o_acc = o_acc e^(lse_acc - l) +
 * o_s e^(lse_s - l), lse_acc = l = logaddexp(lse_acc, lse_s) -- the exact
 * softmax over the union of the chunks' keys.  first != 0 initialises. */
int ul_lse_merge(void* o_acc, float* lse_acc, const void* o_s, const float* lse_s, int64_t n, int64_t b,
                 int64_t h, int64_t hd, int dtype, int first, void* stream);

/* Q/K/V projection fused with the seq->head exchange:
 * project(x, wq|wk|wv) (layers.py:118-122, ulysses.py:140-142) + _to_head
 * (ulysses.py:161-164).  x: this rank's sequence shard [nl*b, d] (bf16,
 * d = hq*hd), w: [d, (hq + 2*hkv)*hd] = [wq | wk | wv] (d_in x d_out,
 * row-major); q4/k4/v4: this rank's head-layout outputs [nl*P, b, hq/P, hd]
 * and [nl*P, b, hkv/P, hd].  The GEMM epilogue stores every head block at
 * its owner (own output or the peer's receive slot over NVLink); a
 * collective like ul_all_to_all (every rank calls it with the same shapes
 * and label; comm may be NULL for P = 1).  bf16, hd = 128. */
int ul_qkv_proj_exchange(ul_comm* comm, const void* x, const void* w, void* q4, void* k4, void* v4,
                         int64_t nl, int64_t b, int64_t hq, int64_t hkv, int64_t hd,
                         uint64_t label_hash, void* stream);

/* The general form (both directions): Y = X W (w
 * row-major [d_in, N]) or Y = X W^T (w_transposed: w row-major [N, d_in],
 * e.g. the backward's dc = g Wo^T, ulysses.py:207) with N = sum(heads)*hd,
 * whose 128-column head blocks are stored straight into the head layout of
 * their owner rank: outs[t] = [nl*P, b, heads[t]/P, hd] -- the GEMM fused
 * with the seq->head exchange of its n_out (1..3) outputs.  x: [nl*b,
 * d_in] bf16; d_in % 64 == 0, hd = 128.  A collective like ul_all_to_all.
 * ul_qkv_proj_exchange == ul_proj_exchange(x, [wq|wk|wv], 0, 3, ...). */
int ul_proj_exchange(ul_comm* comm, const void* x, const void* w, int w_transposed, int n_out,
                     void* const* outs, const int64_t* heads, int64_t nl, int64_t b, int64_t d_in,
                     int64_t hd, uint64_t label_hash, void* stream);

/* ======================================================================
 * The row-wise pieces of the transformer block around the attention
 * (ulysses_block_forward ulysses.py:172-184), bf16 or
 * fp32 rows of width d <= 4096, fp32 statistics:
 *   ul_add_layernorm: s = x + r (r may be NULL: s = x; s_out may be NULL),
 *     y = layernorm(s) * gain + bias (layers.py:106-110, population
 *     variance, eps), stats[row] = {mean, rstd} (float2) for the backward;
 *   ul_layernorm_bwd: dx, and dgain / dbias as deterministic column sums
 *     (workspace >= ul_layernorm_bwd_workspace_bytes);
 *   ul_gelu: exact erf GELU (layers.py:113-127); with dy != NULL the
 *     backward dx = dy * gelu'(x).
 * ==================================================================== */
int ul_add_layernorm(const void* x, const void* r, const void* gain, const void* bias, void* s_out, void* y,
                     float* stats, int64_t rows, int64_t d, float eps, int dtype, void* stream);
size_t ul_layernorm_bwd_workspace_bytes(int64_t rows, int64_t d);
int ul_layernorm_bwd(const void* dy, const void* s, const void* gain, const float* stats, void* dx, void* dgain,
                     void* dbias, void* workspace, size_t workspace_bytes, int64_t rows, int64_t d, int dtype,
                     void* stream);
int ul_gelu(const void* x, const void* dy, void* out, int64_t n, int dtype, void* stream);

/* Number of kernel launches the last ul_* call on this thread issued, and
 * the cumulative count since the library was loaded (all threads). */
int ul_last_launch_count(void);
uint64_t ul_total_launch_count(void);

/* costmodel.py:82-87 -- per-link a2a elements of one layer's forward,
 * as an exact fraction num/den.  convention 0 = exact, 1 = paper_asymptotic. */
int ul_ulysses_volume(int64_t n, int64_t b, int64_t d, int64_t p, int convention,
                      int64_t* num, int64_t* den);

#ifdef __cplusplus
}
#endif
#endif /* ULYSSES_B200_H */
