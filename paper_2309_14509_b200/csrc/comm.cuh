// Device-visible state of the sequence-parallel exchange (csrc/a2a.cu),
// shared with the attention kernels that fuse the head->seq exchange into
// their epilogue (K2 fused into K3/K4).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ulysses_b200.h"

namespace ul {

struct ErrWord {
  volatile int32_t code;   // 0 or UL_ERR_DESYNC
  volatile int32_t kind;   // 1 signature mismatch, 2 timeout
  volatile int32_t peer;
  volatile int32_t pad;
  volatile uint64_t epoch;
  volatile uint64_t expect_sig;
  volatile uint64_t got;   // peer signature, or bitmask of missing ranks
};

struct Signals {           // lives at base + 2*slot_bytes on every rank
  uint64_t flags[2][UL_MAX_RANKS];
  uint64_t sigs[2][UL_MAX_RANKS];
  unsigned int counter[2];
  unsigned int pad[2];
  ErrWord err;              // device-side error accumulator (local use)
  // device ledger (CommLedger, simgroup.py:145-172, counted on the GPU): the
  // last CTA of every call's producing kernel adds 1 call, the call's
  // per-rank egress bytes and its aggregate bytes
  unsigned long long ledger[3];
};

// Fused head->seq epilogue: a kernel that produces head-layout rows
// [N, b, h_local, hd] stores row `r` of local head `h` straight into the
// sequence-layout image of rank r / rows_per_rank (its `out` for the own
// rank, its receive slot over NVLink for peers) at head
// head_offset + h, then the last CTA of the launch publishes the call's
// signature and epoch to every peer (same protocol as ul_all_to_all).
struct PeerEpilogue {
  char* dst[UL_MAX_RANKS];      // per destination rank, per tensor (see below)
  Signals* sig[UL_MAX_RANKS];   // signal block of every rank
  unsigned int* counter;        // this rank's CTA counter for the slot
  uint64_t epoch, sigv;
  int rank, world, slot;
  int rows_per_rank;            // N / P
  int heads_seq;                // heads of the sequence-layout tensor (H)
  int head_offset;              // rank * H / P
  int active;                   // 0: plain kernel (P = 1 or unfused)
  unsigned long long* ledger;   // this rank's device ledger (Signals::ledger) or nullptr
  uint64_t egress, aggregate;   // the call's bytes, added once by the signalling CTA
};

// Fused seq->head epilogue of the Q/K/V projection GEMM (csrc/proj_sm100.cu):
// each 128-column head block of Y = X [wq|wk|wv] goes to the head-layout
// image of the rank that owns the head.
struct ProjEpilogue {
  char* dst[3][UL_MAX_RANKS];   // tensor q/k/v x destination rank: base of its [N, b, hl, hd] image
  int col0[4];                  // first W column of q, k, v; col0[3] = total columns
  int hl[3];                    // heads per rank of q, k, v
  int nl, b, hd, me;
  PeerEpilogue sg;              // signalling of the exchange (active when P > 1)
};

__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Destination of element row (qrow, bb, local head h) in the sequence-layout
// image; `b` batch size, hd head dim, element size in bytes.
__device__ __forceinline__ char* peer_row_ptr(const PeerEpilogue& ep, int qrow, int bb, int b, int h, int hd,
                                              int esize) {
  const int dst = qrow / ep.rows_per_rank;
  const int64_t row = qrow - (int64_t)dst * ep.rows_per_rank;
  return ep.dst[dst] + (((row * b + bb) * ep.heads_seq + ep.head_offset + h) * (int64_t)hd) * esize;
}

// Called by thread 0 of every CTA after a __syncthreads that follows every
// thread's __threadfence_system(): the last CTA to arrive signals the peers.
__device__ __forceinline__ void peer_signal_last_cta(const PeerEpilogue& ep, unsigned int total_ctas) {
  const unsigned int ticket = atomicAdd(ep.counter, 1u);
  if (ticket == total_ctas - 1) {
    *ep.counter = 0;
    if (ep.ledger) {
      atomicAdd(ep.ledger, 1ull);
      atomicAdd(ep.ledger + 1, (unsigned long long)ep.egress);
      atomicAdd(ep.ledger + 2, (unsigned long long)ep.aggregate);
    }
    __threadfence_system();
    for (int i = 0; i < ep.world; ++i) {
      if (i == ep.rank) continue;
      st_relaxed_sys_u64(&ep.sig[i]->sigs[ep.slot][ep.rank], ep.sigv);
      st_release_sys_u64(&ep.sig[i]->flags[ep.slot][ep.rank], ep.epoch);
    }
  }
}

}  // namespace ul

struct ul_comm;  // defined in a2a.cu

namespace ul {

// Host side of a fused head->seq exchange of n head-layout tensors
// (head_shapes[4t..4t+4) = [N, b, h_local, hd]) into seq_out[t]
// ([N/P, b, P*h_local, hd]).  begin: plans the call (epoch, slot, signature
// -- same as ul_all_to_all(split 0, concat 2)) and fills one PeerEpilogue
// per tensor for the producing kernel; finish: flag wait + drain on this
// rank's stream after the producing kernels.
int a2a_fused_begin(ul_comm* c, int n, void* const* seq_out, const int64_t* head_shapes, int dtype,
                    uint64_t label, PeerEpilogue* ep, int* slot, uint64_t* epoch);
int a2a_fused_finish(ul_comm* c, int n, void* const* seq_out, const int64_t* head_shapes, int dtype,
                     uint64_t label, int slot, uint64_t epoch, cudaStream_t st);

}  // namespace ul
