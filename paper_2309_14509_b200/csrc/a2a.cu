// K1/K2: the Ulysses all-to-all over NVLink/NVSwitch peer memory.
//
// Replaces RankGroup._all_to_all (simgroup.py:313-335) + _exchange
// (simgroup.py:251-304) as called by seq_to_head (split 2, concat 0,
// ulysses.py:104-111) and head_to_seq (split 0, concat 2, ulysses.py:114-124).
//
// Semantics (combine, simgroup.py:322-327): out_i = concat_j(split(in_j, P,
// split_axis)[i], concat_axis).  Each (tensor, destination) pair is a 4-D
// box copy whose innermost `run` bytes are contiguous on both sides, so the
// permute is fused into the exchange: a warp streams one run with 16-byte
// vector loads (coalesced, local HBM) and 16-byte stores straight into the
// destination -- `out` for the local chunk, the peer's receive slot over
// NVLink for remote chunks.  The last CTA to finish publishes a per-slot
// signature and an epoch flag into every peer with st.release.sys; the
// receiver's wait kernel acquires the flags (bounded spin -> DESYNC error
// instead of a hang, simgroup.py:292-297) and compares signatures
// (simgroup.py:265-276); a drain kernel then moves the P-1 remote chunks
// from the slot into `out`.  Two slots alternate by call parity, which
// makes one barrier per call sufficient.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include <cstring>
#include <mutex>
#include <vector>

#include "comm.cuh"
#include "common.cuh"

namespace ul {

struct Box {               // one (tensor, peer) chunk of a fused all-to-all
  const char* src;
  char* dst;
  int64_t rows;            // product of the outer extents
  int64_t run;             // contiguous bytes per row (both sides)
  int64_t ext[3];          // outer extents (slowest first); unused dims = 1
  int64_t sst[3], dstr[3]; // byte strides of the outer dims
  int32_t vec;             // access width: 16, 8, 4, 2 or 1 bytes
  int32_t pad;
};

constexpr int kMaxBoxes = UL_MAX_FUSED * UL_MAX_RANKS;

struct CopyParams {
  Box box[kMaxBoxes];
  int nbox;
  // signalling (push kernel only)
  int signal;               // 1 -> last CTA publishes sig + epoch to peers
  int rank, world, slot;
  uint64_t epoch, sig;
  Signals* peer_sig[UL_MAX_RANKS];
  unsigned int* counter;    // local, reset by the last CTA
  unsigned long long* ledger;   // this rank's device ledger (or nullptr)
  uint64_t egress, aggregate;   // bytes of the call, added by the last CTA
};

}  // namespace ul

struct ul_comm {
  int rank = 0, world = 1, device = 0;
  size_t slot_bytes = 0;
  char* base = nullptr;
  char* peer_base[UL_MAX_RANKS] = {};
  bool ipc_opened[UL_MAX_RANKS] = {};
  uint64_t epoch = 0;
  int64_t timeout_ns = 60ll * 1000 * 1000 * 1000;   // RankGroup default 60 s (simgroup.py:207-208)
  ul::ErrWord* err_host = nullptr;
  ul::ErrWord* err_dev = nullptr;
  uint64_t calls = 0, egress = 0, aggregate = 0;
  uint64_t last_label = 0;
};

namespace ul {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int V>
struct VecT;
template <> struct VecT<16> { using T = int4; };
template <> struct VecT<8>  { using T = int2; };
template <> struct VecT<4>  { using T = int;  };
template <> struct VecT<2>  { using T = short; };
template <> struct VecT<1>  { using T = char; };

// Each warp owns a contiguous range of rows: the row index is decomposed
// once and then advanced like an odometer (no 64-bit div/mod per row).
// Short runs (the Ulysses head-group run is (H/P)*hd elements, 512 B-1 KiB)
// are copied two rows per step so every lane keeps several 16-byte loads in
// flight.
template <int V>
__device__ __forceinline__ void copy_box(const Box& bx, int64_t warp0, int64_t nwarps, int lane) {
  using T = typename VecT<V>::T;
  const int64_t nvec = bx.run / V;
  const int64_t e1 = bx.ext[1], e2 = bx.ext[2];
  const int64_t per = (bx.rows + nwarps - 1) / nwarps;
  int64_t r = warp0 * per;
  const int64_t r_end = min(bx.rows, r + per);
  if (r >= r_end) return;
  int64_t c2 = r % e2, t = r / e2;
  int64_t c1 = t % e1, c0 = t / e1;
  const char* srow = bx.src + c0 * bx.sst[0] + c1 * bx.sst[1] + c2 * bx.sst[2];
  char* drow = bx.dst + c0 * bx.dstr[0] + c1 * bx.dstr[1] + c2 * bx.dstr[2];
  auto advance = [&]() {
    if (++c2 < e2) {
      srow += bx.sst[2];
      drow += bx.dstr[2];
      return;
    }
    c2 = 0;
    if (++c1 < e1) {
      srow += bx.sst[1] - (e2 - 1) * bx.sst[2];
      drow += bx.dstr[1] - (e2 - 1) * bx.dstr[2];
      return;
    }
    c1 = 0;
    ++c0;
    srow += bx.sst[0] - (e1 - 1) * bx.sst[1] - (e2 - 1) * bx.sst[2];
    drow += bx.dstr[0] - (e1 - 1) * bx.dstr[1] - (e2 - 1) * bx.dstr[2];
  };
  if (nvec <= 64) {
    // two rows per step, up to 2 x 2 vectors per lane in flight
    for (; r + 1 < r_end; r += 2) {
      const T* s0 = reinterpret_cast<const T*>(srow);
      T* d0 = reinterpret_cast<T*>(drow);
      advance();
      const T* s1 = reinterpret_cast<const T*>(srow);
      T* d1 = reinterpret_cast<T*>(drow);
      advance();
      T a0, a1, b0, b1;
      const bool l0 = lane < nvec, l1 = lane + 32 < nvec;
      if (l0) { a0 = __ldcs(s0 + lane); b0 = __ldcs(s1 + lane); }
      if (l1) { a1 = __ldcs(s0 + lane + 32); b1 = __ldcs(s1 + lane + 32); }
      if (l0) { d0[lane] = a0; d1[lane] = b0; }
      if (l1) { d0[lane + 32] = a1; d1[lane + 32] = b1; }
    }
  }
  for (; r < r_end; ++r) {
    const T* s = reinterpret_cast<const T*>(srow);
    T* d = reinterpret_cast<T*>(drow);
    int64_t i = lane;
    for (; i + 96 < nvec; i += 128) {
      T a0 = __ldcs(s + i), a1 = __ldcs(s + i + 32), a2 = __ldcs(s + i + 64), a3 = __ldcs(s + i + 96);
      d[i] = a0; d[i + 32] = a1; d[i + 64] = a2; d[i + 96] = a3;
    }
    for (; i < nvec; i += 32) d[i] = __ldcs(s + i);
    advance();
  }
}

// grid (blocks_per_box, nbox); kCopyThreads threads.  128-thread CTAs of
// <= 64 registers (8192 registers) fit beside a resident attention CTA
// (forward: 320 threads x 168 registers; fused backward: 704 x 80), so the
// pipelined layer's prefetch exchange runs on the SMs the attention of the
// previous head group occupies instead of waiting for its tail.
constexpr int kCopyThreads = 128;
__global__ void __launch_bounds__(kCopyThreads) a2a_copy_kernel(const __grid_constant__ CopyParams p) {
  const Box& bx = p.box[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  switch (bx.vec) {
    case 16: copy_box<16>(bx, w0, nwarps, lane); break;
    case 8:  copy_box<8>(bx, w0, nwarps, lane); break;
    case 4:  copy_box<4>(bx, w0, nwarps, lane); break;
    case 2:  copy_box<2>(bx, w0, nwarps, lane); break;
    default: copy_box<1>(bx, w0, nwarps, lane); break;
  }
  if (!p.signal) return;
  // make this CTA's peer stores visible system-wide, then count CTAs
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int total = gridDim.x * gridDim.y;
    unsigned int ticket = atomicAdd(p.counter, 1u);
    if (ticket == total - 1) {
      *p.counter = 0;  // every CTA has arrived; safe to rearm for the next call
      if (p.ledger) {
        atomicAdd(p.ledger, 1ull);
        atomicAdd(p.ledger + 1, (unsigned long long)p.egress);
        atomicAdd(p.ledger + 2, (unsigned long long)p.aggregate);
      }
      __threadfence_system();
      for (int i = 0; i < p.world; ++i) {
        if (i == p.rank) continue;
        Signals* s = p.peer_sig[i];
        st_relaxed_sys(&s->sigs[p.slot][p.rank], p.sig);
        st_release_sys(&s->flags[p.slot][p.rank], p.epoch);
      }
    }
  }
}

// one warp: lane j waits for rank j's epoch flag in this slot.  Errors are
// combined with device-memory atomics (`dev`), then lane 0 mirrors the word
// into mapped host memory (`host`) with plain stores so the host can poll
// it without a device sync.
__global__ void a2a_wait_kernel(Signals* mine, int rank, int world, int slot, uint64_t epoch,
                                uint64_t sig, int64_t timeout_ns, ErrWord* dev, ErrWord* host) {
  const int j = threadIdx.x;
  if (j < world && j != rank) {
    bool ok = true;
    const uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    while (ld_acquire_sys(&mine->flags[slot][j]) < epoch) {
      if ((++spins & 255u) == 0 && (int64_t)(globaltimer() - t0) > timeout_ns) {
        ok = false;
        break;
      }
      __nanosleep(100);
    }
    if (!ok) {
      if (atomicCAS((int*)&dev->code, 0, UL_ERR_DESYNC) == 0) {
        dev->kind = 2;
        dev->peer = j;
        dev->epoch = epoch;
        dev->expect_sig = sig;
      }
      atomicOr((unsigned long long*)&dev->got, 1ull << j);
    } else {
      uint64_t got = ld_relaxed_sys(&mine->sigs[slot][j]);
      if (got != sig && atomicCAS((int*)&dev->code, 0, UL_ERR_DESYNC) == 0) {
        dev->kind = 1;
        dev->peer = j;
        dev->epoch = epoch;
        dev->expect_sig = sig;
        dev->got = got;
      }
    }
  }
  __syncwarp();
  __threadfence();
  if (j == 0 && dev->code != 0 && host->code == 0) {
    host->kind = dev->kind;
    host->peer = dev->peer;
    host->epoch = dev->epoch;
    host->expect_sig = dev->expect_sig;
    host->got = dev->got;
    __threadfence_system();
    host->code = dev->code;
    dev->code = 0;   // re-arm (host keeps the first error until read)
    dev->got = 0;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static uint64_t fnv(uint64_t h, uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 1099511628211ull;
  }
  return h;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Geom {                 // one tensor of a fused call, padded to 4-D
  int64_t S[4], So[4];        // in / out shapes
  int64_t ss[4], so[4];       // byte strides
  int split, concat;
  size_t in_bytes, out_bytes;
};

static int make_geom(int ndim, const int64_t* shape, int esz, int split, int concat, int P, Geom* g) {
  const int pad = 4 - ndim;
  for (int k = 0; k < 4; ++k) g->S[k] = k < pad ? 1 : shape[k - pad];
  for (int k = 0; k < 4; ++k)
    if (g->S[k] < 0) return fail(UL_ERR_SHAPE, "all_to_all: negative dimension in shape");
  g->split = split + pad;
  g->concat = concat + pad;
  if (g->S[g->split] % P != 0)
    return fail(UL_ERR_DIVISIBILITY, "all_to_all split axis %d (length %lld) not divisible by p=%d",
                split, (long long)g->S[g->split], P);
  for (int k = 0; k < 4; ++k) g->So[k] = g->S[k];
  g->So[g->split] /= P;
  if (g->split != g->concat) g->So[g->concat] *= P;
  g->ss[3] = esz;
  g->so[3] = esz;
  for (int k = 2; k >= 0; --k) {
    g->ss[k] = g->ss[k + 1] * g->S[k + 1];
    g->so[k] = g->so[k + 1] * g->So[k + 1];
  }
  g->in_bytes = (size_t)(g->ss[0] * g->S[0]);
  g->out_bytes = (size_t)(g->so[0] * g->So[0]);
  return UL_OK;
}

// chunk for destination `dst_rank` sent by `src_rank`: box in the source
// tensor (layout S) and the same box placed in out_dst (layout So)
// drain=true: the chunk already sits in a receive slot laid out like out_dst,
// so both sides use the output layout and offset.
static void make_box(const Geom& g, int src_rank, int dst_rank, int P, const char* src, char* dst,
                     Box* b, bool drain = false) {
  int64_t E[4], os[4] = {0, 0, 0, 0}, od[4] = {0, 0, 0, 0};
  for (int k = 0; k < 4; ++k) E[k] = g.S[k];
  const int64_t L = g.S[g.split] / P;
  E[g.split] = L;
  os[g.split] = (int64_t)dst_rank * L;
  if (g.split == g.concat) od[g.concat] = (int64_t)src_rank * L;
  else od[g.concat] = (int64_t)src_rank * g.S[g.concat];
  const int m = g.split > g.concat ? g.split : g.concat;
  int64_t run = g.ss[3] * E[m];
  for (int k = m + 1; k < 4; ++k) run *= E[k];
  b->run = run;
  int64_t off_s = 0, off_d = 0;
  for (int k = 0; k < 4; ++k) {
    off_s += drain ? od[k] * g.so[k] : os[k] * g.ss[k];
    off_d += od[k] * g.so[k];
  }
  b->src = src + off_s;
  b->dst = dst + off_d;
  // outer dims k < m, right-aligned into ext[0..2]
  for (int i = 0; i < 3; ++i) {
    b->ext[i] = 1;
    b->sst[i] = 0;
    b->dstr[i] = 0;
  }
  for (int k = 0; k < m; ++k) {
    const int i = 3 - m + k;
    b->ext[i] = E[k];
    b->sst[i] = drain ? g.so[k] : g.ss[k];
    b->dstr[i] = g.so[k];
  }
  b->rows = b->ext[0] * b->ext[1] * b->ext[2];
  if (run == 0) b->rows = 0;
  uint64_t al = (uint64_t)run | (uint64_t)(uintptr_t)b->src | (uint64_t)(uintptr_t)b->dst;
  for (int i = 0; i < 3; ++i) al |= (uint64_t)b->sst[i] | (uint64_t)b->dstr[i];
  b->vec = (al % 16 == 0) ? 16 : (al % 8 == 0) ? 8 : (al % 4 == 0) ? 4 : (al % 2 == 0) ? 2 : 1;
}

static int launch_copy(CopyParams& p, cudaStream_t st, const char* name) {
  if (p.nbox == 0) return UL_OK;
  int64_t maxwork = 0;
  for (int i = 0; i < p.nbox; ++i) {
    int64_t w = p.box[i].rows * ((p.box[i].run + 511) / 512);
    if (w > maxwork) maxwork = w;
  }
  // ~one 512-byte warp-row per warp per pass; cap the grid at a few waves
  const int warps_per_block = kCopyThreads / 32;
  int64_t bpb = (maxwork + warps_per_block - 1) / warps_per_block;
  const int64_t cap = (int64_t)sm_count() * (2048 / kCopyThreads / 2) / p.nbox + 1;   // ~32 warps per SM
  if (bpb > cap) bpb = cap;
  if (bpb < 1) bpb = 1;
  dim3 grid((unsigned)bpb, (unsigned)p.nbox);
  a2a_copy_kernel<<<grid, kCopyThreads, 0, st>>>(p);
  return launched(name);
}

int preload_a2a() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, a2a_copy_kernel));
  UL_CUDA(cudaFuncGetAttributes(&a, a2a_wait_kernel));
  // An SM runs a new CTA beside resident ones only if its L1 / shared-memory
  // carveout has room.  The flag wait spins for as long as a peer takes, and
  // the exchange copies are meant to run beside an attention CTA (~200 KB of
  // shared memory): both ask for the max-shared carveout, so the SM hosting
  // them can still take an attention CTA.  (With the default carveout the
  // last CTA of a persistent attention grid could not start on the SM of a
  // spinning wait -- whose peer signal that very grid's last CTA sends: an
  // in-process group deadlocked at its first layer call.)
  UL_CUDA(cudaFuncSetAttribute(a2a_copy_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared));
  UL_CUDA(cudaFuncSetAttribute(a2a_wait_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared));
  return UL_OK;
}

}  // namespace ul

using namespace ul;

extern "C" {

int ul_preload_kernels(void);

// Mapped host error words come from one pinned pool, allocated at the first
// group creation: cudaHostAlloc can serialize the device's streams, and an
// in-process group creates workspaces (regrowth) while its ranks' flag waits
// may be spinning on peers the host has yet to issue.
namespace {
constexpr int kErrPool = 4096;
std::mutex g_err_mu;
ul::ErrWord* g_err_host = nullptr;
std::vector<int> g_err_free;
}  // namespace

static cudaError_t err_word_take(ul::ErrWord** host, ul::ErrWord** dev) {
  std::lock_guard<std::mutex> lock(g_err_mu);
  if (!g_err_host) {
    cudaError_t e = cudaHostAlloc((void**)&g_err_host, kErrPool * sizeof(ul::ErrWord),
                                  cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) {
      g_err_host = nullptr;
      return e;
    }
    for (int i = kErrPool - 1; i >= 0; --i) g_err_free.push_back(i);
  }
  if (g_err_free.empty()) return cudaErrorMemoryAllocation;
  const int i = g_err_free.back();
  g_err_free.pop_back();
  memset((void*)(g_err_host + i), 0, sizeof(ul::ErrWord));
  *host = g_err_host + i;
  // mapped pinned memory: the device address equals the host address under UVA
  cudaError_t e = cudaHostGetDevicePointer((void**)dev, (void*)*host, 0);
  if (e != cudaSuccess) g_err_free.push_back(i);
  return e;
}

static void err_word_give(ul::ErrWord* host) {
  std::lock_guard<std::mutex> lock(g_err_mu);
  if (g_err_host && host >= g_err_host && host < g_err_host + kErrPool) g_err_free.push_back((int)(host - g_err_host));
}

int ul_comm_create(int rank, int world, int device, size_t slot_bytes, ul_comm** out) {
  if (!out) return fail(UL_ERR_ARG, "ul_comm_create: out is NULL");
  *out = nullptr;
  if (world < 1 || world > UL_MAX_RANKS)
    return fail(UL_ERR_ARG, "group size must be in [1, %d], got %d", UL_MAX_RANKS, world);
  if (rank < 0 || rank >= world) return fail(UL_ERR_ARG, "rank %d outside group of %d", rank, world);
  UL_CUDA(cudaSetDevice(device));
  UL_TRY(ul_preload_kernels());
  ul_comm* c = new ul_comm();
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->slot_bytes = align_up(slot_bytes ? slot_bytes : 256, 4096);
  const size_t total = 2 * c->slot_bytes + align_up(sizeof(Signals), 4096);
  cudaError_t e = cudaMalloc(&c->base, total);
  if (e != cudaSuccess) {
    delete c;
    return fail(UL_ERR_CUDA, "ul_comm_create: cudaMalloc(%zu): %s", total, cudaGetErrorString(e));
  }
  // zero the signals on a private non-blocking stream and wait for that
  // stream only: an in-process group creates workspaces (regrowth) while
  // its ranks' streams may hold flag waits that the host has yet to satisfy,
  // so neither a device sync nor the legacy default stream may be used here
  cudaStream_t zs = nullptr;
  e = cudaStreamCreateWithFlags(&zs, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->base + 2 * c->slot_bytes, 0, sizeof(Signals), zs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(zs);
  if (zs) cudaStreamDestroy(zs);
  if (e == cudaSuccess) e = err_word_take(&c->err_host, &c->err_dev);
  if (e != cudaSuccess) {
    cudaFree(c->base);
    delete c;
    return fail(UL_ERR_CUDA, "ul_comm_create: %s", cudaGetErrorString(e));
  }
  c->peer_base[rank] = c->base;
  *out = c;
  return UL_OK;
}

struct HandleBlob {
  cudaIpcMemHandle_t h;   // 64 bytes
  uint64_t magic;
  uint64_t slot_bytes;
  int32_t rank, world;
};
static_assert(sizeof(HandleBlob) <= UL_IPC_HANDLE_BYTES, "blob too large");
static const uint64_t kMagic = 0x554c595353455332ull;  // "ULYSSES2"

int ul_comm_export_handle(const ul_comm* c, void* handle_out) {
  if (!c || !handle_out) return fail(UL_ERR_ARG, "ul_comm_export_handle: NULL argument");
  HandleBlob b;
  memset(&b, 0, sizeof(b));
  UL_CUDA(cudaSetDevice(c->device));
  UL_CUDA(cudaIpcGetMemHandle(&b.h, c->base));
  b.magic = kMagic;
  b.slot_bytes = c->slot_bytes;
  b.rank = c->rank;
  b.world = c->world;
  memset(handle_out, 0, UL_IPC_HANDLE_BYTES);
  memcpy(handle_out, &b, sizeof(b));
  return UL_OK;
}

int ul_comm_validate_handles(const void* all, int world, int rank, size_t slot_bytes) {
  if (!all || world < 1 || world > UL_MAX_RANKS || rank < 0 || rank >= world)
    return fail(UL_ERR_ARG, "ul_comm_validate_handles: bad arguments");
  const char* p = (const char*)all;
  for (int r = 0; r < world; ++r) {
    HandleBlob b;
    memcpy(&b, p + (size_t)r * UL_IPC_HANDLE_BYTES, sizeof(b));
    if (b.magic != kMagic)
      return fail(UL_ERR_DESYNC, "group desync: rank %d sent a malformed comm handle", r);
    if (b.rank != r || b.world != world)
      return fail(UL_ERR_DESYNC, "group desync: rank %d reports rank %d of %d, expected %d of %d", r, b.rank,
                  b.world, r, world);
    if (b.slot_bytes != slot_bytes)
      return fail(UL_ERR_DESYNC, "group desync: rank %d workspace slot %llu bytes, rank %d has %llu", r,
                  (unsigned long long)b.slot_bytes, rank, (unsigned long long)slot_bytes);
  }
  return UL_OK;
}

int ul_comm_open_peers(ul_comm* c, const void* all) {
  if (!c || !all) return fail(UL_ERR_ARG, "ul_comm_open_peers: NULL argument");
  UL_TRY(ul_comm_validate_handles(all, c->world, c->rank, c->slot_bytes));
  UL_CUDA(cudaSetDevice(c->device));
  const char* p = (const char*)all;
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    HandleBlob b;
    memcpy(&b, p + (size_t)r * UL_IPC_HANDLE_BYTES, sizeof(b));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return fail(UL_ERR_CUDA, "rank %d: cudaIpcOpenMemHandle(peer %d): %s", c->rank, r,
                  cudaGetErrorString(e));
    c->peer_base[r] = (char*)ptr;
    c->ipc_opened[r] = true;
  }
  return UL_OK;
}

int ul_comm_link_local(ul_comm* const* comms, int world) {
  if (!comms || world < 1) return fail(UL_ERR_ARG, "ul_comm_link_local: bad arguments");
  for (int r = 0; r < world; ++r) {
    if (!comms[r] || comms[r]->world != world || comms[r]->rank != r)
      return fail(UL_ERR_DESYNC, "group desync: comm %d is not rank %d of %d", r, r, world);
    if (comms[r]->slot_bytes != comms[0]->slot_bytes)
      return fail(UL_ERR_DESYNC, "group desync: rank %d workspace slot differs from rank 0", r);
  }
  for (int r = 0; r < world; ++r)
    for (int s = 0; s < world; ++s) comms[r]->peer_base[s] = comms[s]->base;
  return UL_OK;
}

int ul_comm_destroy(ul_comm* c) {
  if (!c) return UL_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->world; ++r)
    if (c->ipc_opened[r]) cudaIpcCloseMemHandle(c->peer_base[r]);
  cudaFree(c->base);
  if (c->err_host) err_word_give(c->err_host);
  delete c;
  return UL_OK;
}

int ul_comm_rank(const ul_comm* c) { return c ? c->rank : 0; }
int ul_comm_world(const ul_comm* c) { return c ? c->world : 1; }
size_t ul_comm_slot_bytes(const ul_comm* c) { return c ? c->slot_bytes : 0; }

int ul_comm_set_timeout_ms(ul_comm* c, int64_t ms) {
  if (!c || ms <= 0) return fail(UL_ERR_ARG, "ul_comm_set_timeout_ms: bad arguments");
  c->timeout_ns = ms * 1000000ll;
  return UL_OK;
}

int ul_comm_status(ul_comm* c, char* msg, size_t len) {
  if (!c) return fail(UL_ERR_ARG, "ul_comm_status: NULL comm");
  const int code = c->err_host->code;
  if (code == 0) {
    if (msg && len) msg[0] = 0;
    return UL_OK;
  }
  char buf[512];
  if (c->err_host->kind == 2) {
    std::string missing;
    for (int r = 0; r < c->world; ++r)
      if (c->err_host->got & (1ull << r)) missing += (missing.empty() ? "" : ", ") + std::to_string(r);
    snprintf(buf, sizeof(buf),
             "group desync: timeout in collective 'all_to_all' (call %llu) on rank %d waiting on ranks [%s]",
             (unsigned long long)c->err_host->epoch, c->rank, missing.c_str());
  } else {
    snprintf(buf, sizeof(buf),
             "group desync: rank %d entered collective 'all_to_all' (call %llu, signature %016llx) while rank "
             "%d entered 'all_to_all' (signature %016llx)",
             c->err_host->peer, (unsigned long long)c->err_host->epoch,
             (unsigned long long)c->err_host->got, c->rank, (unsigned long long)c->err_host->expect_sig);
  }
  if (msg && len) {
    strncpy(msg, buf, len - 1);
    msg[len - 1] = 0;
  }
  last_error() = buf;
  memset((void*)c->err_host, 0, sizeof(ErrWord));
  return code;
}

int ul_comm_ledger(const ul_comm* c, uint64_t* calls, uint64_t* egress, uint64_t* aggregate) {
  if (!c) return fail(UL_ERR_ARG, "ul_comm_ledger: NULL comm");
  if (calls) *calls = c->calls;
  if (egress) *egress = c->egress;
  if (aggregate) *aggregate = c->aggregate;
  return UL_OK;
}

int ul_comm_ledger_device(const ul_comm* c, uint64_t* calls, uint64_t* egress, uint64_t* aggregate) {
  if (!c) return fail(UL_ERR_ARG, "ul_comm_ledger_device: NULL comm");
  unsigned long long v[3] = {0, 0, 0};
  UL_CUDA(cudaSetDevice(c->device));
  UL_CUDA(cudaMemcpy(v, ((Signals*)(c->base + 2 * c->slot_bytes))->ledger, sizeof(v), cudaMemcpyDeviceToHost));
  if (calls) *calls = v[0];
  if (egress) *egress = v[1];
  if (aggregate) *aggregate = v[2];
  return UL_OK;
}

size_t ul_all_to_all_slot_bytes(int n, const int64_t* shapes, int ndim, int dtype, int split,
                                int concat, int world) {
  size_t tot = 0;
  for (int t = 0; t < n; ++t) {
    Geom g;
    if (make_geom(ndim, shapes + 4 * t, (int)dtype_size(dtype), split, concat, world, &g) != UL_OK)
      return 0;
    tot += align_up(g.out_bytes, 256);
  }
  return tot;
}

}  // extern "C"

namespace ul {

// One collective call: geometry of every tensor, the receive-slot layout,
// the cross-rank signature and this call's epoch / slot.
struct CallPlan {
  int n = 0, P = 1, me = 0, slot = 0;
  Geom g[UL_MAX_FUSED];
  size_t slot_off[UL_MAX_FUSED];
  uint64_t sig = 0, epoch = 0;
  uint64_t egress = 0, aggregate = 0;   // this rank's bytes (simgroup.py:329-332 metering)
};

static unsigned long long* dev_ledger(ul_comm* c) {
  return c ? ((Signals*)(c->base + 2 * c->slot_bytes))->ledger : nullptr;
}

static int plan_call(ul_comm* c, int n, void* const* out, const int64_t* shapes, int ndim, int dtype, int split,
                     int concat, uint64_t label, CallPlan* pl) {
  if (n < 1 || n > UL_MAX_FUSED)
    return fail(UL_ERR_ARG, "all_to_all: fuses 1..%d tensors, got %d", UL_MAX_FUSED, n);
  if (ndim < 1 || ndim > 4) return fail(UL_ERR_SHAPE, "all_to_all: tensors of rank 1..4, got %d", ndim);
  if (dtype != UL_DTYPE_F32 && dtype != UL_DTYPE_BF16)
    return fail(UL_ERR_KERNEL, "all_to_all: unsupported dtype %d", dtype);
  if (split < 0 || split >= ndim || concat < 0 || concat >= ndim)
    return fail(UL_ERR_ARG, "all_to_all: axes (%d, %d) out of range for rank %d", split, concat, ndim);
  if (!out || !shapes) return fail(UL_ERR_ARG, "all_to_all: NULL argument");
  pl->n = n;
  pl->P = c ? c->world : 1;
  pl->me = c ? c->rank : 0;
  const int esz = (int)dtype_size(dtype);
  size_t slot_need = 0;
  uint64_t sig = 1469598103934665603ull;
  sig = fnv(sig, (uint64_t)n);
  sig = fnv(sig, (uint64_t)ndim);
  sig = fnv(sig, (uint64_t)dtype);
  sig = fnv(sig, (uint64_t)split);
  sig = fnv(sig, (uint64_t)concat);
  sig = fnv(sig, label);
  uint64_t in_total = 0;
  for (int t = 0; t < n; ++t) {
    UL_TRY(make_geom(ndim, shapes + 4 * t, esz, split, concat, pl->P, &pl->g[t]));
    if (!out[t] && pl->g[t].out_bytes > 0) return fail(UL_ERR_ARG, "all_to_all: NULL tensor %d", t);
    for (int k = 0; k < ndim; ++k) sig = fnv(sig, (uint64_t)shapes[4 * t + k]);
    pl->slot_off[t] = slot_need;
    slot_need += align_up(pl->g[t].out_bytes, 256);
    in_total += pl->g[t].in_bytes;
  }
  pl->sig = sig;
  const int P = pl->P;
  if (P > 1 && slot_need > c->slot_bytes)
    return fail(UL_ERR_ARG, "all_to_all: call needs %zu receive-slot bytes, workspace has %zu", slot_need,
                c->slot_bytes);
  for (int r = 0; P > 1 && r < P; ++r)
    if (!c->peer_base[r])
      return fail(UL_ERR_STATE, "all_to_all: rank %d has no mapping for peer %d (open_peers not called)",
                  pl->me, r);
  if (c) {
    pl->epoch = ++c->epoch;
    pl->slot = (int)(pl->epoch & 1);
    c->calls += 1;
    c->aggregate += (uint64_t)P * in_total;
    c->egress += in_total / P * (P - 1);
  }
  pl->aggregate = (uint64_t)P * in_total;
  pl->egress = in_total / P * (P - 1);
  return UL_OK;
}

// receiver side: bounded flag wait + drain of the P-1 remote chunks
static int wait_and_drain(ul_comm* c, const CallPlan& pl, void* const* out, cudaStream_t st) {
  Signals* mine = (Signals*)(c->base + 2 * c->slot_bytes);
  a2a_wait_kernel<<<1, 32, 0, st>>>(mine, pl.me, pl.P, pl.slot, pl.epoch, pl.sig, c->timeout_ns, &mine->err,
                                      c->err_dev);
  UL_TRY(launched("a2a_wait"));
  CopyParams dp;
  memset(&dp, 0, sizeof(dp));
  for (int t = 0; t < pl.n; ++t) {
    for (int j = 0; j < pl.P; ++j) {
      if (j == pl.me) continue;
      // the chunk rank j sent sits in my slot exactly where it belongs in out
      Box b;
      const char* slot_img = c->base + (size_t)pl.slot * c->slot_bytes + pl.slot_off[t];
      make_box(pl.g[t], j, pl.me, pl.P, slot_img, (char*)out[t], &b, /*drain=*/true);
      if (b.rows > 0) dp.box[dp.nbox++] = b;
    }
  }
  return launch_copy(dp, st, "a2a_drain");
}

// a push with nothing to move that still publishes this rank's flag + signature
static int signal_only(ul_comm* c, const CallPlan& pl, cudaStream_t st) {
  CopyParams cp;
  memset(&cp, 0, sizeof(cp));
  cp.signal = 1;
  cp.rank = pl.me;
  cp.world = pl.P;
  cp.slot = pl.slot;
  cp.epoch = pl.epoch;
  cp.sig = pl.sig;
  for (int r = 0; r < pl.P; ++r) cp.peer_sig[r] = (Signals*)(c->peer_base[r] + 2 * c->slot_bytes);
  cp.counter = &((Signals*)(c->base + 2 * c->slot_bytes))->counter[pl.slot];
  cp.ledger = dev_ledger(c);
  cp.egress = pl.egress;
  cp.aggregate = pl.aggregate;
  cp.box[0].rows = 0;
  cp.box[0].vec = 16;
  cp.nbox = 1;
  return launch_copy(cp, st, "a2a_signal");
}

int a2a_fused_begin(ul_comm* c, int n, void* const* seq_out, const int64_t* head_shapes, int dtype,
                    uint64_t label, PeerEpilogue* ep, int* handle_slot, uint64_t* handle_epoch) {
  // head->seq (split 0, concat 2) of [N, b, h_local, hd] head-layout tensors
  CallPlan pl;
  UL_TRY(plan_call(c, n, seq_out, head_shapes, 4, dtype, 0, 2, label, &pl));
  for (int t = 0; t < n; ++t) {
    PeerEpilogue& e = ep[t];
    memset(&e, 0, sizeof(e));
    e.active = pl.P > 1;
    e.rank = pl.me;
    e.world = pl.P;
    e.slot = pl.slot;
    e.epoch = pl.epoch;
    e.sigv = pl.sig;
    e.rows_per_rank = (int)(pl.g[t].S[0] / pl.P);
    e.heads_seq = (int)(pl.g[t].S[2] * pl.P);
    e.head_offset = (int)(pl.me * pl.g[t].S[2]);
    for (int r = 0; r < pl.P; ++r) {
      e.dst[r] = (r == pl.me || !c) ? (char*)seq_out[t]
                                    : c->peer_base[r] + (size_t)pl.slot * c->slot_bytes + pl.slot_off[t];
      if (c) e.sig[r] = (Signals*)(c->peer_base[r] + 2 * c->slot_bytes);
    }
    if (c) e.counter = &((Signals*)(c->base + 2 * c->slot_bytes))->counter[pl.slot];
    e.ledger = dev_ledger(c);
    e.egress = pl.egress;
    e.aggregate = pl.aggregate;
  }
  *handle_slot = pl.slot;
  *handle_epoch = pl.epoch;
  return UL_OK;
}

int a2a_fused_finish(ul_comm* c, int n, void* const* seq_out, const int64_t* head_shapes, int dtype,
                     uint64_t label, int slot, uint64_t epoch, cudaStream_t st) {
  if (!c || c->world == 1) return UL_OK;
  // rebuild the plan without advancing the epoch
  CallPlan pl;
  pl.n = n;
  pl.P = c->world;
  pl.me = c->rank;
  const int esz = (int)dtype_size(dtype);
  size_t off = 0;
  uint64_t sig = 1469598103934665603ull;
  sig = fnv(sig, (uint64_t)n);
  sig = fnv(sig, 4);
  sig = fnv(sig, (uint64_t)dtype);
  sig = fnv(sig, 0);
  sig = fnv(sig, 2);
  sig = fnv(sig, label);
  for (int t = 0; t < n; ++t) {
    UL_TRY(make_geom(4, head_shapes + 4 * t, esz, 0, 2, pl.P, &pl.g[t]));
    for (int k = 0; k < 4; ++k) sig = fnv(sig, (uint64_t)head_shapes[4 * t + k]);
    pl.slot_off[t] = off;
    off += align_up(pl.g[t].out_bytes, 256);
  }
  pl.sig = sig;
  pl.slot = slot;
  pl.epoch = epoch;
  return wait_and_drain(c, pl, seq_out, st);
}

int sm100_qkv_proj(const void* x, const void* w, int64_t M, int64_t K, int64_t N, const ProjEpilogue& ep,
                   cudaStream_t st, bool w_transposed);

}  // namespace ul

extern "C" {

int ul_proj_exchange(ul_comm* c, const void* x, const void* w, int w_transposed, int n_out, void* const* outs,
                     const int64_t* heads, int64_t nl, int64_t b, int64_t d_in, int64_t hd, uint64_t label,
                     void* stream) {
  launch_count() = 0;
  if (n_out < 1 || n_out > 3 || !outs || !heads) return fail(UL_ERR_ARG, "ul_proj_exchange: 1..3 outputs");
  if (!w) return fail(UL_ERR_ARG, "ul_proj_exchange: NULL weight");
  if (nl < 0 || b < 1 || d_in < 1 || hd < 1)
    return fail(UL_ERR_SHAPE, "ul_proj_exchange: bad shape (nl=%lld, b=%lld, d_in=%lld, hd=%lld)", (long long)nl,
                (long long)b, (long long)d_in, (long long)hd);
  for (int t = 0; t < n_out; ++t) {
    if (heads[t] < 1) return fail(UL_ERR_SHAPE, "ul_proj_exchange: head count %lld", (long long)heads[t]);
    if (!outs[t] && nl * b > 0) return fail(UL_ERR_ARG, "ul_proj_exchange: NULL output %d", t);
  }
  if (!x && nl * b > 0) return fail(UL_ERR_ARG, "ul_proj_exchange: NULL input");
  // the fused all-to-all is the seq->head flip of the projections' sequence shards
  int64_t shapes[12];
  int64_t N = 0;
  ProjEpilogue ep;
  memset(&ep, 0, sizeof(ep));
  for (int t = 0; t < n_out; ++t) {
    shapes[4 * t] = nl;
    shapes[4 * t + 1] = b;
    shapes[4 * t + 2] = heads[t];
    shapes[4 * t + 3] = hd;
    ep.col0[t] = (int)N;
    N += heads[t] * hd;
  }
  for (int t = n_out; t < 4; ++t) ep.col0[t] = (int)N;
  CallPlan pl;
  UL_TRY(plan_call(c, n_out, outs, shapes, 4, UL_DTYPE_BF16, 2, 0, label, &pl));
  for (int t = 0; t < n_out; ++t) {
    for (int r = 0; r < pl.P; ++r)
      ep.dst[t][r] = (r == pl.me || !c) ? (char*)outs[t]
                                        : c->peer_base[r] + (size_t)pl.slot * c->slot_bytes + pl.slot_off[t];
    ep.hl[t] = (int)(heads[t] / pl.P);
  }
  ep.nl = (int)nl;
  ep.b = (int)b;
  ep.hd = (int)hd;
  ep.me = pl.me;
  PeerEpilogue& sg = ep.sg;
  sg.active = pl.P > 1;
  sg.rank = pl.me;
  sg.world = pl.P;
  sg.slot = pl.slot;
  sg.epoch = pl.epoch;
  sg.sigv = pl.sig;
  if (c) {
    for (int r = 0; r < pl.P; ++r) sg.sig[r] = (Signals*)(c->peer_base[r] + 2 * c->slot_bytes);
    sg.counter = &((Signals*)(c->base + 2 * c->slot_bytes))->counter[pl.slot];
    sg.ledger = dev_ledger(c);
    sg.egress = pl.egress;
    sg.aggregate = pl.aggregate;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (nl * b == 0) {
    // empty sequence shard: no GEMM tile runs, so no CTA would publish the
    // call -- peers still expect this rank's flag (a signal-only push)
    if (pl.P > 1) UL_TRY(signal_only(c, pl, st));
  } else {
    UL_TRY(sm100_qkv_proj(x, w, nl * b, d_in, N, ep, st, w_transposed != 0));
  }
  if (pl.P > 1) UL_TRY(wait_and_drain(c, pl, outs, st));
  return UL_OK;
}

int ul_qkv_proj_exchange(ul_comm* c, const void* x, const void* w, void* q4, void* k4, void* v4, int64_t nl,
                         int64_t b, int64_t hq, int64_t hkv, int64_t hd, uint64_t label, void* stream) {
  void* outs[3] = {q4, k4, v4};
  const int64_t heads[3] = {hq, hkv, hkv};
  return ul_proj_exchange(c, x, w, 0, 3, outs, heads, nl, b, hq * hd, hd, label, stream);
}

}  // extern "C"

namespace ul {

// Parent layout of a head-group exchange: box sources live inside this
// rank's full [nl, b, H, hd] shard at head i * H / P + group * Hg (P, H per
// tensor); nullptr for a plain contiguous all_to_all.
struct HeadGroupSrc {
  int64_t heads[UL_MAX_FUSED];   // H of each tensor
  int group;                     // this call's head group
};

// the push (local chunk -> out, remote chunks -> peer slots, release
// signal) + flag wait + drain of a planned call
static int push_and_finish(ul_comm* c, const CallPlan& pl, const void* const* in, void* const* out,
                           const HeadGroupSrc* hg, cudaStream_t st) {
  const int P = pl.P, me = pl.me, slot = pl.slot;
  CopyParams cp;
  memset(&cp, 0, sizeof(cp));
  for (int t = 0; t < pl.n; ++t) {
    for (int k = 0; k < P; ++k) {
      const int i = (me + k) % P;  // rotate destinations to spread switch load
      char* dst = (i == me) ? (char*)out[t] : c->peer_base[i] + (size_t)slot * c->slot_bytes + pl.slot_off[t];
      Box& b = cp.box[cp.nbox];
      make_box(pl.g[t], me, i, P, (const char*)in[t], dst, &b);
      if (hg && b.rows > 0) {
        // the virtual [nl, b, P*Hg, hd] view of head group `group`: chunk i
        // starts at head i*Hl + group*Hg of the parent shard, rows keep the
        // parent's strides (run = Hg*hd elements, as for the view)
        const Geom& g = pl.g[t];
        const int64_t Hg = g.S[2] / P, Hl = hg->heads[t] / P, hd = g.S[3], esz = g.ss[3];
        b.src = (const char*)in[t] + (i * Hl + (int64_t)hg->group * Hg) * hd * esz;
        b.sst[1] = g.S[1] * hg->heads[t] * hd * esz;   // row s of the shard: b * H * hd elements
        b.sst[2] = hg->heads[t] * hd * esz;             // batch entry: H * hd elements
        uint64_t al = (uint64_t)b.run | (uint64_t)(uintptr_t)b.src | (uint64_t)(uintptr_t)b.dst;
        for (int x = 0; x < 3; ++x) al |= (uint64_t)b.sst[x] | (uint64_t)b.dstr[x];
        b.vec = (al % 16 == 0) ? 16 : (al % 8 == 0) ? 8 : (al % 4 == 0) ? 4 : (al % 2 == 0) ? 2 : 1;
      }
      if (b.rows > 0) ++cp.nbox;
    }
  }
  if (P > 1) {
    cp.signal = 1;
    cp.rank = me;
    cp.world = P;
    cp.slot = slot;
    cp.epoch = pl.epoch;
    cp.sig = pl.sig;
    for (int r = 0; r < P; ++r) cp.peer_sig[r] = (Signals*)(c->peer_base[r] + 2 * c->slot_bytes);
    cp.counter = &((Signals*)(c->base + 2 * c->slot_bytes))->counter[slot];
    cp.ledger = dev_ledger(c);
    cp.egress = pl.egress;
    cp.aggregate = pl.aggregate;
    if (cp.nbox == 0) {  // nothing to move (empty tensors) -- still signal
      make_box(pl.g[0], me, me, P, (const char*)in[0], (char*)out[0], &cp.box[0]);
      cp.box[0].rows = 0;
      cp.nbox = 1;
    }
  }
  UL_TRY(launch_copy(cp, st, "a2a_push"));
  if (P == 1) return UL_OK;
  return wait_and_drain(c, pl, out, st);
}

}  // namespace ul

extern "C" {

int ul_all_to_all(ul_comm* c, int n, const void* const* in, void* const* out, const int64_t* shapes,
                  int ndim, int dtype, int split, int concat, uint64_t label, void* stream) {
  launch_count() = 0;
  if (!in) return fail(UL_ERR_ARG, "all_to_all: NULL argument");
  CallPlan pl;
  UL_TRY(plan_call(c, n, out, shapes, ndim, dtype, split, concat, label, &pl));
  for (int t = 0; t < n; ++t)
    if (!in[t] && pl.g[t].in_bytes > 0) return fail(UL_ERR_ARG, "all_to_all: NULL tensor %d", t);
  return push_and_finish(c, pl, in, out, nullptr, (cudaStream_t)stream);
}

int ul_all_to_all_head_group(ul_comm* c, int n, const void* const* in, void* const* out, const int64_t* shapes,
                             int dtype, int group, int groups, uint64_t label, void* stream) {
  launch_count() = 0;
  if (!in || !shapes || n < 1 || n > UL_MAX_FUSED)
    return fail(UL_ERR_ARG, "all_to_all_head_group: bad arguments");
  const int P = c ? c->world : 1;
  if (groups < 1 || group < 0 || group >= groups)
    return fail(UL_ERR_ARG, "all_to_all_head_group: group %d of %d", group, groups);
  HeadGroupSrc hg;
  int64_t vshapes[4 * UL_MAX_FUSED];
  for (int t = 0; t < n; ++t) {
    const int64_t* sh = shapes + 4 * t;   // parent shard [nl, b, H, hd]
    if (sh[2] % ((int64_t)P * groups) != 0)
      return fail(UL_ERR_DIVISIBILITY, "all_to_all_head_group: p=%d x %d groups does not divide head count %lld", P,
                  groups, (long long)sh[2]);
    hg.heads[t] = sh[2];
    vshapes[4 * t] = sh[0];
    vshapes[4 * t + 1] = sh[1];
    vshapes[4 * t + 2] = sh[2] / groups;   // the group's P*Hg heads
    vshapes[4 * t + 3] = sh[3];
  }
  hg.group = group;
  CallPlan pl;
  UL_TRY(plan_call(c, n, out, vshapes, 4, dtype, 2, 0, label, &pl));
  for (int t = 0; t < n; ++t)
    if (!in[t] && pl.g[t].in_bytes > 0) return fail(UL_ERR_ARG, "all_to_all_head_group: NULL tensor %d", t);
  return push_and_finish(c, pl, in, out, &hg, (cudaStream_t)stream);
}

// a flat byte range as rows of `run` bytes (so every warp of the copy gets rows)
static void flat_box(const char* src, char* dst, int64_t bytes, Box* b) {
  int64_t run = 4096;
  while (run > 16 && (bytes % run) != 0) run >>= 1;
  if (bytes % run != 0) run = bytes;   // (unaligned tail: one row)
  b->src = src;
  b->dst = dst;
  b->run = run;
  for (int i = 0; i < 3; ++i) b->ext[i] = 1, b->sst[i] = 0, b->dstr[i] = 0;
  b->ext[2] = run ? bytes / run : 0;
  b->sst[2] = b->dstr[2] = run;
  b->rows = bytes > 0 ? b->ext[2] : 0;
  const uint64_t al = (uint64_t)run | (uint64_t)(uintptr_t)src | (uint64_t)(uintptr_t)dst;
  b->vec = (al % 16 == 0) ? 16 : (al % 8 == 0) ? 8 : (al % 4 == 0) ? 4 : (al % 2 == 0) ? 2 : 1;   // odd byte counts: 1
}

int ul_ring_shift(ul_comm* c, int n, const void* const* in, void* const* out, const int64_t* bytes, int steps,
                  uint64_t label, void* stream) {
  launch_count() = 0;
  if (n < 1 || n > UL_MAX_FUSED) return fail(UL_ERR_ARG, "ring_shift: fuses 1..%d tensors, got %d", UL_MAX_FUSED, n);
  if (!in || !out || !bytes) return fail(UL_ERR_ARG, "ring_shift: NULL argument");
  if (steps < 0) return fail(UL_ERR_ARG, "ring_shift steps must be >= 0, got %d", steps);
  const int P = c ? c->world : 1, me = c ? c->rank : 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int k = steps % P;
  size_t off[UL_MAX_FUSED], need = 0;
  uint64_t sig = 1469598103934665603ull, total = 0;
  sig = fnv(sig, 0x72696e67ull);   // "ring"
  sig = fnv(sig, (uint64_t)n);
  sig = fnv(sig, (uint64_t)steps);
  sig = fnv(sig, label);
  for (int t = 0; t < n; ++t) {
    if (!in[t] || !out[t] || bytes[t] < 0) return fail(UL_ERR_ARG, "ring_shift: bad tensor %d", t);
    sig = fnv(sig, (uint64_t)bytes[t]);
    off[t] = need;
    need += align_up((size_t)bytes[t], 256);
    total += (uint64_t)bytes[t];
  }
  CopyParams cp;
  memset(&cp, 0, sizeof(cp));
  if (P == 1 || k == 0) {   // the payload stays on this rank: a local copy (+ a barrier for P > 1)
    for (int t = 0; t < n; ++t) {
      flat_box((const char*)in[t], (char*)out[t], bytes[t], &cp.box[cp.nbox]);
      if (cp.box[cp.nbox].rows > 0) ++cp.nbox;
    }
    if (P == 1) return launch_copy(cp, st, "ring_local");
  }
  if (need > c->slot_bytes)
    return fail(UL_ERR_ARG, "ring_shift: call needs %zu receive-slot bytes, workspace has %zu", need, c->slot_bytes);
  for (int r = 0; r < P; ++r)
    if (!c->peer_base[r]) return fail(UL_ERR_STATE, "ring_shift: rank %d has no mapping for peer %d", me, r);
  const uint64_t epoch = ++c->epoch;
  const int slot = (int)(epoch & 1);
  c->calls += 1;
  c->aggregate += (uint64_t)P * total;
  c->egress += total * (uint64_t)steps;   // simgroup.py:383-385 metering
  const int dst = (me + k) % P, src = (me - k + P) % P;
  if (k != 0) {
    for (int t = 0; t < n; ++t) {
      flat_box((const char*)in[t], c->peer_base[dst] + (size_t)slot * c->slot_bytes + off[t], bytes[t],
               &cp.box[cp.nbox]);
      if (cp.box[cp.nbox].rows > 0) ++cp.nbox;
    }
  }
  // every rank signals every peer (a full barrier, like the reference's collectives)
  cp.signal = 1;
  cp.rank = me;
  cp.world = P;
  cp.slot = slot;
  cp.epoch = epoch;
  cp.sig = sig;
  for (int r = 0; r < P; ++r) cp.peer_sig[r] = (Signals*)(c->peer_base[r] + 2 * c->slot_bytes);
  cp.counter = &((Signals*)(c->base + 2 * c->slot_bytes))->counter[slot];
  cp.ledger = dev_ledger(c);
  cp.egress = total * (uint64_t)steps;
  cp.aggregate = (uint64_t)P * total;
  if (cp.nbox == 0) {
    flat_box((const char*)in[0], (char*)out[0], 0, &cp.box[0]);
    cp.nbox = 1;
  }
  UL_TRY(launch_copy(cp, st, "ring_push"));
  Signals* mine = (Signals*)(c->base + 2 * c->slot_bytes);
  a2a_wait_kernel<<<1, 32, 0, st>>>(mine, me, P, slot, epoch, sig, c->timeout_ns, &mine->err, c->err_dev);
  UL_TRY(launched("a2a_wait"));
  if (k == 0) return UL_OK;
  (void)src;
  CopyParams dp;
  memset(&dp, 0, sizeof(dp));
  for (int t = 0; t < n; ++t) {   // the predecessor's payload sits in my slot
    flat_box(c->base + (size_t)slot * c->slot_bytes + off[t], (char*)out[t], bytes[t], &dp.box[dp.nbox]);
    if (dp.box[dp.nbox].rows > 0) ++dp.nbox;
  }
  return launch_copy(dp, st, "ring_drain");
}

int ul_ulysses_volume(int64_t n, int64_t b, int64_t d, int64_t p, int convention, int64_t* num,
                      int64_t* den) {
  if (!num || !den || n < 1 || b < 1 || d < 1 || p < 1)
    return fail(UL_ERR_ARG, "ul_ulysses_volume: bad arguments");
  if (n % p != 0) return fail(UL_ERR_DIVISIBILITY, "p=%lld does not divide n=%lld", (long long)p, (long long)n);
  const int64_t m = 4 * n * b * d;
  int64_t nu, de;
  if (convention == 1) {
    nu = m;
    de = p;
  } else {
    nu = m * (p - 1);
    de = p * p;
  }
  int64_t a = nu, bb = de;
  while (bb) {
    int64_t t = a % bb;
    a = bb;
    bb = t;
  }
  if (a == 0) a = 1;
  *num = nu / a;
  *den = de / a;
  return UL_OK;
}

}  // extern "C"

// ---- ring attention: exact merge of a chunk's (O, LSE) into the running one ----
namespace ul {
// o_acc[row, :] <- o_acc * e^(lse_acc - l) + o_s * e^(lse_s - l), lse_acc <- l
// = logaddexp(lse_acc, lse_s); rows (i, bb, hh) of [n, b, h, hd], LSE [b, h, n]
template <typename T>
__global__ void __launch_bounds__(256) lse_merge_kernel(float* __restrict__ o_acc, float* __restrict__ lse_acc,
                                                        const T* __restrict__ o_s, const float* __restrict__ lse_s,
                                                        int64_t n, int64_t b, int64_t h, int64_t hd, int first) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n * b * h) return;
  const int64_t hh = warp % h, bb = (warp / h) % b, i = warp / (h * b);
  const int64_t li = (bb * h + hh) * n + i;
  const float la = first ? -INFINITY : lse_acc[li], ls = lse_s[li];
  const float m = fmaxf(la, ls);
  const float l = (m == -INFINITY) ? -INFINITY : m + logf(expf(la - m) + expf(ls - m));
  const float wa = (la == -INFINITY) ? 0.f : expf(la - l), ws = (ls == -INFINITY) ? 0.f : expf(ls - l);
  float* oa = o_acc + warp * hd;
  const T* os = o_s + warp * hd;
  for (int64_t d = lane; d < hd; d += 32) {
    const float prev = first ? 0.f : oa[d];
    oa[d] = prev * wa + (float)os[d] * ws;
  }
  if (lane == 0) lse_acc[li] = l;
}
}  // namespace ul

extern "C" int ul_lse_merge(void* o_acc, float* lse_acc, const void* o_s, const float* lse_s, int64_t n, int64_t b,
                            int64_t h, int64_t hd, int dtype, int first, void* stream) {
  using namespace ul;
  launch_count() = 0;
  if (!o_acc || !lse_acc || !o_s || !lse_s) return fail(UL_ERR_ARG, "ul_lse_merge: NULL tensor");
  if (n < 0 || b < 0 || h < 0 || hd < 1) return fail(UL_ERR_SHAPE, "ul_lse_merge: bad shape");
  const int64_t rows = n * b * h;
  if (rows == 0) return UL_OK;
  const unsigned blocks = (unsigned)((rows * 32 + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == UL_DTYPE_BF16)
    lse_merge_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((float*)o_acc, lse_acc, (const __nv_bfloat16*)o_s, lse_s,
                                                            n, b, h, hd, first);
  else if (dtype == UL_DTYPE_F32)
    lse_merge_kernel<float><<<blocks, 256, 0, st>>>((float*)o_acc, lse_acc, (const float*)o_s, lse_s, n, b, h, hd,
                                                    first);
  else
    return fail(UL_ERR_KERNEL, "ul_lse_merge: unsupported dtype %d", dtype);
  return launched("lse_merge");
}

namespace ul {
int preload_merge() {
  cudaFuncAttributes a;
  UL_CUDA(cudaFuncGetAttributes(&a, lse_merge_kernel<float>));
  UL_CUDA(cudaFuncGetAttributes(&a, lse_merge_kernel<__nv_bfloat16>));
  return UL_OK;
}
}  // namespace ul
