// Device side of the P2P spike exchange (see exchange_dist.cu for the protocol),
// shared by the per-step kernel and the persistent engine.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "nc_common.h"

namespace ncxchg {

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
static __device__ bool wait_flag(const uint32_t* flag, uint32_t want, uint64_t timeout_ns, int32_t* status) {
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
static __device__ void scatter_ids(const nc_xchg_t& X, const uint32_t* ids, int64_t cnt, int src, bool phase2,
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

// ---------------------------------------------------------------- P2P path
// Inbox layout (uint32 words) on every rank, per (phase, parity, source):
//   slot = ((phase * 2 + parity) * n + src) * (cap + 4): [count, pad, pad, pad, ids...]
// Flags (separate region): flags[phase * NC_MAX_SHARDS + src].

__device__ __forceinline__ int64_t slot_off(const nc_xchg_t& X, int phase, int parity, int src) {
  return ((int64_t)((phase * 2 + parity) * X.n + src)) * (X.cap + 4);
}

// Copy ids [lo, hi) to a (possibly remote) slot, 16-byte stores where aligned.
static __device__ void push_ids(uint32_t* dst, const uint32_t* src, int64_t lo, int64_t hi) {
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
static __device__ void publish(const nc_xchg_t& X, int phase, int b, uint32_t want, int B) {
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

// Exchange of one step by exchange block `ex` of n*B: block (b, k) moves chunk
// k of the traffic with peer b.  Used by the per-step kernel k_p2p and by the
// persistent engine (persistent.cu), whose other blocks do not take part.
static __device__ void p2p_block(const nc_xchg_t& X, int ex, int B, int step) {
  const int nex = X.n * B;
  const int b = ex / B;   // peer handled by this block
  const int kb = ex % B;  // chunk
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
      const uint32_t target = (uint32_t)(step + 1) * (uint32_t)nex;
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
    if (ex == 0) *X.lat_start = t_start;
    __threadfence();
    const uint32_t done = atomicAdd(X.done, 1u) + 1u;
    if (done == (uint32_t)(step + 1) * (uint32_t)nex) {
      __threadfence();
      const uint64_t t_end = globaltimer();
      const uint64_t t0 = *(volatile unsigned long long*)X.lat_start;
      if (X.lat_ns && step < X.lat_steps) X.lat_ns[step] = (t_end > t0) ? (uint32_t)(t_end - t0) : 0u;
    }
  }
}


}  // namespace ncxchg
