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

// Warp-aggregated append of the lanes' ids (where `ok`) to the step's spike
// list (binned delivery); the whole warp calls.
__device__ __forceinline__ void spk_append(const nc_xchg_t& X, int step, bool ok, uint32_t id) {
  if (!X.spk_ids) return;
  const uint32_t m = __ballot_sync(kFull, ok);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int32_t base = 0;
  if (lane == leader) base = atomicAdd(X.spk_count + (step & 1), __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (ok) {
    const int64_t pos = (int64_t)base + __popc(m & ((1u << lane) - 1u));
    if (pos < X.spk_cap) X.spk_ids[(int64_t)(step & 1) * X.spk_cap + pos] = id;
    else atomicExch(X.status, 1);
  }
}

// OR `cnt` ids into the bitmap, count deliveries, relay-bucket if asked.
// Called by a whole block.
static __device__ void scatter_ids(const nc_xchg_t& X, const uint32_t* ids, int64_t cnt, int src, bool phase2,
                            uint32_t* cur, long long* deliv, int32_t* status, int step) {
  __shared__ unsigned int per_src[NC_MAX_SHARDS];
  if (threadIdx.x < NC_MAX_SHARDS) per_src[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t fwd = phase2 ? 0u : (uint32_t)X.fwd_row[src];
  if (X.spk_ids)   // binned delivery: the ids also go to the step's spike list
    for (int64_t k0 = threadIdx.x & ~31; k0 < cnt; k0 += blockDim.x) {
      const int64_t k = k0 + (threadIdx.x & 31);
      spk_append(X, step, k < cnt, k < cnt ? ids[k] : 0u);
    }
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
// Low-latency protocol: every 8-byte word of a message carries its own step
// tag -- (tag << 32) | payload -- so the receiver polls the words themselves
// and the sender needs no system-scope fence or separate flag (8-byte aligned
// stores are single-copy atomic).  Inbox layout (uint64 words) on every rank,
// per (phase, parity, source):
//   slot = ((phase * 2 + parity) * n + src) * (cap + 1): [tag|count, tag|id ...]
// The tag is step + 1: a slot is reused every second step, so a stale word
// never matches.

__device__ __forceinline__ int64_t slot_off(const nc_xchg_t& X, int phase, int parity, int src) {
  return ((int64_t)((phase * 2 + parity) * X.n + src)) * (X.cap + 1);
}

__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void chunk(int64_t cnt, int k, int B, int64_t* lo, int64_t* hi) {
  const int64_t per = (cnt + B - 1) / B;
  *lo = min(cnt, per * k);
  *hi = min(cnt, per * (k + 1));
}

// Chunk kb of B of a message of `cnt` ids to a (possibly remote) slot; block kb
// 0 also writes the header.  Called by a whole block.
static __device__ void ll_send(uint64_t* slot, const uint32_t* ids, int64_t cnt, int kb, int B, uint32_t tag) {
  int64_t lo, hi;
  chunk(cnt, kb, B, &lo, &hi);
  const uint64_t t = (uint64_t)tag << 32;
  for (int64_t k = lo + threadIdx.x; k < hi; k += blockDim.x) st_relaxed_sys_u64(slot + 1 + k, t | ids[k]);
  if (kb == 0 && threadIdx.x == 0) st_relaxed_sys_u64(slot, t | (uint32_t)cnt);
}

// Spin until the word carries `tag` (into *out); false on watchdog expiry.
__device__ __forceinline__ bool ll_wait(const uint64_t* w, uint32_t tag, uint64_t timeout_ns, int32_t* status,
                                        uint64_t* out) {
  uint64_t v = ld_relaxed_sys_u64(w);
  if ((uint32_t)(v >> 32) == tag) {
    *out = v;
    return true;
  }
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  for (;;) {
    v = ld_relaxed_sys_u64(w);
    if ((uint32_t)(v >> 32) == tag) {
      *out = v;
      return true;
    }
    if ((++spins & 255u) == 0) {
      if (globaltimer() - t0 > timeout_ns) {
        atomicExch(status + 1, 1);
        return false;
      }
      if (*(volatile int32_t*)(status + 1)) return false;  // another block timed out
    }
  }
}

// Relay, two-level phase 1: once every block that forwards to destination d has
// claimed its positions, the last one to arrive writes d's phase-2 header (tag |
// count).  The data words were stored straight into d's inbox as they arrived
// (pipelined: no grid barrier, no local re-bucketing); they carry their own tags,
// so the header may land before them.  send_done[d] counts arrivals monotonically:
// step s is complete at (s + 1) x the number of contributing blocks.
__device__ __forceinline__ void relay_arrive(const nc_xchg_t& X, uint32_t fwd, int B, int step, uint32_t tag,
                                             long long* hop) {
  __threadfence();   // this block's position claims and stores before its arrival
  while (fwd) {
    const int d = __ffs(fwd) - 1;
    fwd &= fwd - 1;
    uint32_t contrib = 0;
    for (int s = 0; s < X.n; ++s) contrib += (X.fwd_row[s] >> d) & 1u;
    contrib *= (uint32_t)B;
    const uint32_t arrived = atomicAdd(X.send_done + d, 1u) + 1u;
    if (arrived != (uint32_t)(step + 1) * contrib) continue;
    __threadfence();
    int64_t cnt = *(volatile int32_t*)(X.fwd_count + d);
    if (cnt > X.cap) {
      atomicExch(X.status, 1);
      cnt = X.cap;
    }
    uint64_t* slot = reinterpret_cast<uint64_t*>(X.peer_inbox[d]) + slot_off(X, 1, step & 1, X.rank);
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(((uint64_t)tag << 32) | (uint32_t)cnt)
                 : "memory");
    if (cnt) add64(hop + X.rank * X.n + d, cnt);
  }
}

// Receive chunk kb of the message in `slot` and OR its ids into the bitmap,
// count deliveries; as a two-level relay (phase 1, fwd_row[src] != 0) forward each
// id straight into its destinations' phase-2 inboxes (relay_arrive).  Whole block.
static __device__ void ll_recv_scatter(const nc_xchg_t& X, const uint64_t* slot, int kb, int B, uint32_t tag,
                                       int src, bool phase2, uint32_t* cur, long long* deliv, int step,
                                       long long* hop = nullptr) {
  __shared__ long long s_cnt;
  __shared__ unsigned int per_src[NC_MAX_SHARDS];
  if (threadIdx.x < NC_MAX_SHARDS) per_src[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    uint64_t h = 0;
    s_cnt = ll_wait(slot, tag, X.timeout_ns, X.status, &h) ? (long long)(uint32_t)h : -1;
  }
  __syncthreads();
  int64_t cnt = s_cnt;
  if (cnt < 0) return;
  if (cnt > X.cap) cnt = X.cap;
  int64_t lo, hi;
  chunk(cnt, kb, B, &lo, &hi);
  const uint32_t fwd = phase2 ? 0u : (uint32_t)X.fwd_row[src];
  // direct delivery (not relaying for src): every id received is for this rank
  const bool plain = !phase2 && fwd == 0u;
  // warp-uniform loop (relay appends are warp-aggregated: one atomic per warp and destination)
  const int lane = threadIdx.x & 31;
  for (int64_t k0 = lo + (threadIdx.x & ~31); k0 < hi; k0 += blockDim.x) {
    const int64_t k = k0 + lane;
    uint64_t v = 0;
    const bool good = k < hi && ll_wait(slot + 1 + k, tag, X.timeout_ns, X.status, &v);
    const uint32_t id = (uint32_t)v;
    if (good) atomicOr(cur + (id >> 5), 1u << (id & 31));
    spk_append(X, step, good, id);
    if (plain) continue;
    const uint32_t dm = good ? (uint32_t)(uint16_t)X.dest_global[id] : 0u;
    if ((dm >> X.rank) & 1u) atomicAdd(&per_src[phase2 ? max(owner_of(X, id), 0) : src], 1u);
    const uint32_t f = dm & fwd;
    uint32_t pending = __reduce_or_sync(kFull, f);
    while (pending) {
      const int d = __ffs(pending) - 1;
      pending &= pending - 1;
      const uint32_t m = __ballot_sync(kFull, (f >> d) & 1u);
      const int leader = __ffs(m) - 1;
      int32_t base = 0;
      if (lane == leader) base = atomicAdd(X.fwd_count + d, __popc(m));
      base = __shfl_sync(kFull, base, leader);
      if ((f >> d) & 1u) {
        const int32_t pos = base + __popc(m & ((1u << lane) - 1u));
        if (pos < X.cap) {
          uint64_t* dst = reinterpret_cast<uint64_t*>(X.peer_inbox[d]) + slot_off(X, 1, step & 1, X.rank);
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(dst + 1 + pos),
                       "l"(((uint64_t)tag << 32) | id) : "memory");
        } else {
          atomicExch(X.status, 1);
        }
      }
    }
  }
  __syncthreads();
  if (!phase2 && fwd && threadIdx.x == 0) relay_arrive(X, fwd, B, step, tag, hop);
  if (plain) {
    if (threadIdx.x == 0 && hi > lo) add64(deliv + (int64_t)src * X.n + X.rank, (long long)(hi - lo));
  } else if (threadIdx.x < X.n && per_src[threadIdx.x]) {
    add64(deliv + (int64_t)threadIdx.x * X.n + X.rank, (long long)per_src[threadIdx.x]);
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
  const uint32_t tag = (uint32_t)step + 1u;
  uint32_t* cur = (step & 1) ? X.bitmap1 : X.bitmap0;
  long long* hop = step_row(X.hop_ids, X, step);
  long long* deliv = step_row(X.deliv_ids, X, step);
  uint64_t* my_inbox = reinterpret_cast<uint64_t*>(X.my_inbox);
  __shared__ uint64_t t_start;
  if (threadIdx.x == 0) t_start = globaltimer();
  const bool peer = (b < X.n && b != X.rank);
  unsigned long long* dbg = (X.dbg && step < 64 && threadIdx.x == 0) ? X.dbg + ((int64_t)step * nex + ex) * 4 : nullptr;
  if (dbg) dbg[0] = t_start;

  // ---- phase 1 push: every peer gets a message (possibly empty: the heartbeat)
  if (peer) {
    int64_t cnt = 0;
    if ((X.send1_mask >> b) & 1u) {
      cnt = X.bucket_count[b];
      if (cnt > X.cap) {
        if (threadIdx.x == 0 && kb == 0) atomicExch(X.status, 1);
        cnt = X.cap;
      }
      if (threadIdx.x == 0 && kb == 0 && cnt) add64(hop + X.rank * X.n + b, cnt);
    }
    if (!X.fused_send)   // else the step kernel stored the ids and the header already
      ll_send(reinterpret_cast<uint64_t*>(X.peer_inbox[b]) + slot_off(X, 0, par, X.rank),
              X.bucket_ids + (int64_t)b * X.bucket_cap, cnt, kb, B, tag);
    if (dbg) dbg[1] = globaltimer();
  }
  // ---- phase 1 receive from peer b, chunk kb; as a relay for b, forward as the ids arrive
  if (peer) {
    if (dbg) dbg[2] = globaltimer();
    ll_recv_scatter(X, my_inbox + slot_off(X, 0, par, b), kb, B, tag, b, false, cur, deliv, step, hop);
  }
  // ---- phase 2 receive from relay b (two-level): its pipelined forwards of our group's spikes
  if (X.two_level && peer && ((X.recv2_mask >> b) & 1u))
    ll_recv_scatter(X, my_inbox + slot_off(X, 1, par, b), kb, B, tag, b, true, cur, deliv, step);
  // ---- latency record: last block out stamps (end - start of block 0)
  __syncthreads();
  if (dbg) dbg[3] = globaltimer();
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
