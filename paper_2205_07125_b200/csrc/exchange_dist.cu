// Spike exchange between ranks (one process per GPU) over NVLink / NVSwitch.
//
// Semantics are those of exchange_local.cu (routing.py:184-231 next hops; the
// relay forwards directly to the destination GPU).  Two transports:
//
//  * NCCL (nccl_comm.cpp + the pack/scatter kernels here): per phase one
//    ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd over fixed-capacity
//    messages [count | ids], enqueued on the simulation stream (CUDA-graph
//    capturable), followed by a scatter kernel that ORs the ids into the spike
//    bitmap and, on relays, re-buckets them for phase 2.
//  * P2P (nc_xchg_p2p): one device-initiated kernel per step.  Inboxes are
//    cudaMalloc'd regions opened by every peer through CUDA IPC; block b pushes
//    this rank's bucket for peer b straight into b's inbox with NVLink stores,
//    publishes it with a system-scope release store of the step number into b's
//    flag word, then acquires the flag of source b and scatters what arrived.
//    Phase-1 flags go to every peer every step (a heartbeat that bounds the
//    step lag between any two ranks to one), so inbox slots double-buffered by
//    step parity are never overwritten before they are read.  Two-level routes
//    add an in-kernel grid barrier (every phase-1 inbox drained) and a phase-2
//    push from relays.  Every spin is bounded by a %globaltimer watchdog that
//    sets status[1] and returns instead of hanging the GPU.
//
// Counters: hop_ids[u*n+v] (ids this rank sent on u->v, u = this rank) and
// deliv_ids[s*n+d] (d = this rank); per-step rows when per_step is set.

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>
#include "nc_common.h"

namespace {

constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ void add64(long long* p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int owner_of(const nc_xchg_t& X, uint32_t id) {
  for (int h = 0; h < X.n; ++h)
    if ((int64_t)id >= X.shard_base[h] && (int64_t)id < X.shard_base[h + 1]) return h;
  return -1;
}

// Spin until *flag >= want; false on watchdog expiry.
__device__ bool wait_flag(const uint32_t* flag, uint32_t want, uint64_t timeout_ns, int32_t* status) {
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while ((int32_t)(ld_acquire_sys(flag) - want) < 0) {
    if ((++spins & 255u) == 0) {
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(status + 1, 1);
        return false;
      }
      if (*(volatile int32_t*)(status + 1)) return false;  // another block timed out
    }
  }
  return true;
}

// OR `cnt` ids into the bitmap, count deliveries, relay-bucket if asked.
// Called by a whole block.
__device__ void scatter_ids(const nc_xchg_t& X, const uint32_t* ids, int64_t cnt, int src, bool phase2,
                            uint32_t* cur, long long* deliv, int32_t* status) {
  __shared__ unsigned int per_src[NC_MAX_SHARDS];
  if (threadIdx.x < NC_MAX_SHARDS) per_src[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t fwd = phase2 ? 0u : (uint32_t)X.fwd_row[src];
  for (int64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
    const uint32_t id = ids[k];
    atomicOr(cur + (id >> 5), 1u << (id & 31));
    const uint32_t dm = (uint16_t)X.dest_global[id];
    if ((dm >> X.rank) & 1u) atomicAdd(&per_src[phase2 ? max(owner_of(X, id), 0) : src], 1u);
    uint32_t f = dm & fwd;
    while (f) {
      const int d = __ffs(f) - 1;
      f &= f - 1;
      const int32_t pos = atomicAdd(X.fwd_count + d, 1);
      if (pos < X.cap) X.fwd_ids[(int64_t)d * X.cap + pos] = id;
      else atomicExch(status, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x < X.n && per_src[threadIdx.x])
    add64(deliv + (int64_t)threadIdx.x * X.n + X.rank, (long long)per_src[threadIdx.x]);
}

__device__ __forceinline__ long long* step_row(long long* base, const nc_xchg_t& X, int step) {
  return X.per_step ? base + (int64_t)step * X.n * X.n : base;
}

// ---------------------------------------------------------------- NCCL path
// Before the phase-1 group: clamp bucket counts into the message headers and
// account the channel ids.  (Buckets are filled by the step kernel.)
__global__ void k_seal(const nc_xchg_t X, int phase) {
  const int step = *X.step;
  const int p = threadIdx.x;
  if (p >= X.n || p == X.rank) return;
  const int32_t* cnt = phase == 1 ? X.bucket_count : X.fwd_count;
  const uint16_t mask = phase == 1 ? X.send1_mask : X.send2_mask;
  int32_t c = cnt[p];
  if (c > X.cap) {
    atomicExch(X.status, 1);
    c = X.cap;
  }
  int32_t* hdr = phase == 1 ? X.send_hdr : X.send2_hdr;
  hdr[p] = ((mask >> p) & 1u) ? c : 0;
  if (c && ((mask >> p) & 1u)) add64(step_row(X.hop_ids, X, step) + X.rank * X.n + p, c);
}

__global__ void k_scatter(const nc_xchg_t X, int phase) {
  const int src = blockIdx.x;
  const uint16_t mask = phase == 1 ? X.recv1_mask : X.recv2_mask;
  if (src >= X.n || src == X.rank || !((mask >> src) & 1u)) return;
  const int step = *X.step;
  const int32_t* hdr = phase == 1 ? X.recv_hdr : X.recv2_hdr;
  int64_t cnt = hdr[src];
  if (cnt > X.cap) cnt = X.cap;
  const uint32_t* ids = (phase == 1 ? X.recv_ids : X.recv2_ids) + (int64_t)src * X.cap;
  uint32_t* cur = (step & 1) ? X.bitmap1 : X.bitmap0;
  scatter_ids(X, ids, cnt, src, phase == 2, cur, step_row(X.deliv_ids, X, step), X.status);
}

__global__ void k_reset_fwd(const nc_xchg_t X) {
  if ((int)threadIdx.x < X.n) X.fwd_count[threadIdx.x] = 0;
}

// ---------------------------------------------------------------- P2P path
// Inbox layout (uint32 words) on every rank, per (phase, parity, source):
//   slot = ((phase * 2 + parity) * n + src) * (cap + 4): [count, pad, pad, pad, ids...]
// Flags (separate region): flags[phase * NC_MAX_SHARDS + src].

__device__ __forceinline__ int64_t slot_off(const nc_xchg_t& X, int phase, int parity, int src) {
  return ((int64_t)((phase * 2 + parity) * X.n + src)) * (X.cap + 4);
}

// Copy ids [lo, hi) to a (possibly remote) slot, 16-byte stores where aligned.
__device__ void push_ids(uint32_t* dst, const uint32_t* src, int64_t lo, int64_t hi) {
  const int64_t a4 = (lo + 3) >> 2, b4 = hi >> 2;
  for (int64_t k = lo + threadIdx.x; k < min(hi, a4 << 2); k += blockDim.x) dst[k] = src[k];
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (int64_t k = a4 + threadIdx.x; k < b4; k += blockDim.x) d4[k] = s4[k];
  for (int64_t k = max(lo, b4 << 2) + threadIdx.x; k < hi; k += blockDim.x) dst[k] = src[k];
}

__device__ __forceinline__ void chunk(int64_t cnt, int k, int B, int64_t* lo, int64_t* hi) {
  const int64_t per = (((cnt + B - 1) / B) + 3) & ~int64_t(3);  // 16-byte aligned chunks
  *lo = min(cnt, per * k);
  *hi = min(cnt, per * (k + 1));
}

// Publish one phase's message to peer b once all B blocks of it have stored
// their chunk: every block fences (system scope) and counts itself in; the
// last one releases the flag.
__device__ void publish(const nc_xchg_t& X, int phase, int b, uint32_t want, int B) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t arrived = atomicAdd(X.send_done + phase * NC_MAX_SHARDS + b, 1u) + 1u;
    if (arrived == want * (uint32_t)B) {
      __threadfence_system();
      st_release_sys(X.peer_flags[b] + phase * NC_MAX_SHARDS + X.rank, want);
    }
  }
}

// grid = n peers x B blocks; block (b, k) moves chunk k of the traffic with peer b.
__global__ void __launch_bounds__(512) k_p2p(const nc_xchg_t X, int B) {
  const int b = blockIdx.x / B;   // peer handled by this block
  const int kb = blockIdx.x % B;  // chunk
  const int step = *X.step;
  const int par = step & 1;
  const uint32_t want = (uint32_t)step + 1u;
  uint32_t* cur = (step & 1) ? X.bitmap1 : X.bitmap0;
  long long* hop = step_row(X.hop_ids, X, step);
  long long* deliv = step_row(X.deliv_ids, X, step);
  __shared__ uint64_t t_start;
  __shared__ bool ok;
  if (threadIdx.x == 0) t_start = globaltimer();
  const bool peer = (b < X.n && b != X.rank);

  // ---- phase 1 push (data on route channels, heartbeat flag to everyone)
  if (peer) {
    int64_t cnt = 0;
    if ((X.send1_mask >> b) & 1u) {
      cnt = X.bucket_count[b];
      if (cnt > X.cap) {
        if (threadIdx.x == 0 && kb == 0) atomicExch(X.status, 1);
        cnt = X.cap;
      }
      uint32_t* slot = X.peer_inbox[b] + slot_off(X, 0, par, X.rank);
      int64_t lo, hi;
      chunk(cnt, kb, B, &lo, &hi);
      push_ids(slot + 4, X.bucket_ids + (int64_t)b * X.bucket_cap, lo, hi);
      if (threadIdx.x == 0 && kb == 0) {
        slot[0] = (uint32_t)cnt;
        if (cnt) add64(hop + X.rank * X.n + b, cnt);
      }
    }
    publish(X, 0, b, want, B);
  }
  // ---- phase 1 receive from peer b, chunk kb
  if (peer) {
    if (threadIdx.x == 0) ok = wait_flag(X.my_flags + 0 * NC_MAX_SHARDS + b, want, X.timeout_ns, X.status);
    __syncthreads();
    if (ok && ((X.recv1_mask >> b) & 1u)) {
      const uint32_t* slot = X.my_inbox + slot_off(X, 0, par, b);
      int64_t cnt = *(volatile const uint32_t*)slot;
      if (cnt > X.cap) cnt = X.cap;
      int64_t lo, hi;
      chunk(cnt, kb, B, &lo, &hi);
      scatter_ids(X, slot + 4 + lo, hi - lo, b, false, cur, deliv, X.status);
    }
  }
  if (X.two_level) {
    // ---- grid barrier: every phase-1 inbox drained, forward buckets complete
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(X.barrier, 1u);
      const uint32_t target = (uint32_t)(step + 1) * gridDim.x;
      const uint64_t t0 = globaltimer();
      while ((int32_t)(*(volatile uint32_t*)X.barrier - target) < 0) {
        if (globaltimer() - t0 > X.timeout_ns) {
          atomicExch(X.status + 1, 1);
          break;
        }
      }
      __threadfence();
    }
    __syncthreads();
    // ---- phase 2 push: relayed ids for destination b
    if (peer && ((X.send2_mask >> b) & 1u)) {
      int64_t cnt = X.fwd_count[b];
      if (cnt > X.cap) {
        if (threadIdx.x == 0 && kb == 0) atomicExch(X.status, 1);
        cnt = X.cap;
      }
      uint32_t* slot = X.peer_inbox[b] + slot_off(X, 1, par, X.rank);
      int64_t lo, hi;
      chunk(cnt, kb, B, &lo, &hi);
      push_ids(slot + 4, X.fwd_ids + (int64_t)b * X.cap, lo, hi);
      if (threadIdx.x == 0 && kb == 0) {
        slot[0] = (uint32_t)cnt;
        if (cnt) add64(hop + X.rank * X.n + b, cnt);
      }
      publish(X, 1, b, want, B);
    }
    // ---- phase 2 receive from relay b
    if (peer && ((X.recv2_mask >> b) & 1u)) {
      if (threadIdx.x == 0) ok = wait_flag(X.my_flags + 1 * NC_MAX_SHARDS + b, want, X.timeout_ns, X.status);
      __syncthreads();
      if (ok) {
        const uint32_t* slot = X.my_inbox + slot_off(X, 1, par, b);
        int64_t cnt = *(volatile const uint32_t*)slot;
        if (cnt > X.cap) cnt = X.cap;
        int64_t lo, hi;
        chunk(cnt, kb, B, &lo, &hi);
        scatter_ids(X, slot + 4 + lo, hi - lo, b, true, cur, deliv, X.status);
      }
    }
  }
  // ---- latency record: last block out stamps (end - start of block 0)
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) *X.lat_start = t_start;
    __threadfence();
    const uint32_t done = atomicAdd(X.done, 1u) + 1u;
    if (done == (uint32_t)(step + 1) * gridDim.x) {
      __threadfence();
      const uint64_t t_end = globaltimer();
      const uint64_t t0 = *(volatile unsigned long long*)X.lat_start;
      if (X.lat_ns && step < X.lat_steps) X.lat_ns[step] = (t_end > t0) ? (uint32_t)(t_end - t0) : 0u;
    }
  }
}

// Zero the relay buckets after the exchange (stream-ordered after k_p2p).
__global__ void k_p2p_tail(const nc_xchg_t X) {
  if ((int)threadIdx.x < X.n) X.fwd_count[threadIdx.x] = 0;
}

int check_x(const nc_xchg_t* X) {
  if (!X || X->n < 1 || X->n > NC_MAX_SHARDS || X->rank < 0 || X->rank >= X->n || X->cap < 1) {
    nc_set_error("invalid nc_xchg_t");
    return NC_E_ARG;
  }
  return NC_OK;
}

}  // namespace

__global__ void k_reset(const nc_xchg_t X) {
  const int t = threadIdx.x;
  if (t < 2 * NC_MAX_SHARDS && X.my_flags) X.my_flags[t] = 0u;
  if (t < 2 * NC_MAX_SHARDS && X.send_done) X.send_done[t] = 0u;
  if (t == 0) {
    if (X.done) *X.done = 0u;
    if (X.barrier) *X.barrier = 0u;
  }
  if (t < X.n && X.fwd_count) X.fwd_count[t] = 0;
}

extern "C" int nc_xchg_reset(const nc_xchg_t* X, void* stream) {
  if (int e = check_x(X)) return e;
  k_reset<<<1, 64, 0, (cudaStream_t)stream>>>(*X);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_xchg_seal(const nc_xchg_t* X, int32_t phase, void* stream) {
  if (int e = check_x(X)) return e;
  k_seal<<<1, 32, 0, (cudaStream_t)stream>>>(*X, phase);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_xchg_scatter(const nc_xchg_t* X, int32_t phase, void* stream) {
  if (int e = check_x(X)) return e;
  k_scatter<<<X->n, 512, 0, (cudaStream_t)stream>>>(*X, phase);
  NC_LAUNCH_CHECK();
  if (phase == 2) {
    k_reset_fwd<<<1, 32, 0, (cudaStream_t)stream>>>(*X);
    NC_LAUNCH_CHECK();
  }
  return NC_OK;
}

extern "C" int nc_xchg_p2p(const nc_xchg_t* X, void* stream) {
  if (int e = check_x(X)) return e;
  if (!X->my_inbox || !X->my_flags || !X->done || !X->lat_start) {
    nc_set_error("nc_xchg_p2p: inbox / flags not set up");
    return NC_E_ARG;
  }
  const int B = X->blocks_per_peer > 0 ? X->blocks_per_peer : 1;
  k_p2p<<<X->n * B, 512, 0, (cudaStream_t)stream>>>(*X, B);
  NC_LAUNCH_CHECK();
  if (X->two_level) {
    k_p2p_tail<<<1, 32, 0, (cudaStream_t)stream>>>(*X);
    NC_LAUNCH_CHECK();
  }
  return NC_OK;
}

// ---------------------------------------------------------------- IPC windows

extern "C" int nc_ipc_alloc(size_t bytes, void** ptr_out, void* handle_out /*64 bytes*/) {
  void* p = nullptr;
  NC_CUDA_TRY(cudaMalloc(&p, bytes));
  NC_CUDA_TRY(cudaMemset(p, 0, bytes));
  cudaIpcMemHandle_t h;
  NC_CUDA_TRY(cudaIpcGetMemHandle(&h, p));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  *ptr_out = p;
  return NC_OK;
}

extern "C" int nc_ipc_open(const void* handle /*64 bytes*/, void** ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  NC_CUDA_TRY(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return NC_OK;
}

extern "C" int nc_ipc_close(void* ptr) {
  NC_CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return NC_OK;
}

extern "C" int nc_free(void* ptr) {
  NC_CUDA_TRY(cudaFree(ptr));
  return NC_OK;
}

// ---------------------------------------------------------------- timestamps
namespace {
__global__ void k_stamp(unsigned long long* dst, const int32_t* step, int32_t max_steps) {
  const int s = *step;
  if (s < max_steps) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    dst[s] = t;
  }
}
}  // namespace

extern "C" int nc_stamp(unsigned long long* dst, const int32_t* step, int32_t max_steps, void* stream) {
  k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>(dst, step, max_steps);
  NC_LAUNCH_CHECK();
  return NC_OK;
}
