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
//    cudaMalloc'd regions opened by every peer through CUDA IPC; the B blocks
//    of peer b store this rank's bucket for b straight into b's inbox with
//    NVLink stores, in a low-latency protocol: every 8-byte word carries the
//    step tag next to its payload (header word: tag | count), so no fence or
//    flag is needed -- the receiving blocks poll the header and their chunk's
//    words until the tag matches, then OR the ids into the spike bitmap.
//    Phase-1 messages go to every peer every step (possibly empty: a
//    heartbeat that bounds the step lag between any two ranks to one), so
//    inbox slots double-buffered by step parity are never overwritten before
//    they are read.  Two-level routes: a relay forwards every id it receives
//    for another group straight into the destination's phase-2 inbox as it
//    arrives (positions claimed with one atomic per warp and destination), and
//    the last of the contributing blocks writes that message's header -- no
//    grid barrier, no second pass.  Every spin is bounded by a %globaltimer
//    watchdog that sets status[1] and returns instead of hanging the GPU.
//
// Counters: hop_ids[u*n+v] (ids this rank sent on u->v, u = this rank) and
// deliv_ids[s*n+d] (d = this rank); per-step rows when per_step is set.

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>
#include "nc_common.h"
#include "xchg_device.cuh"

namespace {
using namespace ncxchg;

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
  scatter_ids(X, ids, cnt, src, phase == 2, cur, step_row(X.deliv_ids, X, step), X.status, step);
}

__global__ void k_reset_fwd(const nc_xchg_t X) {
  if ((int)threadIdx.x < X.n) X.fwd_count[threadIdx.x] = 0;
}

// ---------------------------------------------------------------- P2P path
__global__ void __launch_bounds__(512) k_p2p(const nc_xchg_t X, int B) {
  p2p_block(X, blockIdx.x, B, *X.step);
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
  // P2P inboxes: tags are step + 1 and the step counter restarts at 0, so words left
  // by a previous run would carry the tags of this run's messages -- clear them
  // (callers order this before any peer's first send: synchronize + barrier)
  if (X->my_inbox)
    NC_CUDA_TRY(cudaMemsetAsync(X->my_inbox, 0, NC_P2P_INBOX_WORDS(X->n, X->cap) * sizeof(uint32_t),
                                (cudaStream_t)stream));
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

int ncx_load_exchange_kernels(void) {
  cudaFuncAttributes fa;
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_seal));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_scatter));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_reset_fwd));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_p2p));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_p2p_tail));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_reset));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_stamp));
  return NC_OK;
}

extern "C" int nc_stamp(unsigned long long* dst, const int32_t* step, int32_t max_steps, void* stream) {
  k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>(dst, step, max_steps);
  NC_LAUNCH_CHECK();
  return NC_OK;
}
