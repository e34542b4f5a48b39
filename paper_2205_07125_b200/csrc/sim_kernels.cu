// Per-timestep hot loop of the spiking simulator on sm_100a.
//
//   K3 deliver (pull): integer reduction over the pull synapse matrix in the
//      SELL-32 layout (include/neurocomm_b200.h): a warp owns 32 consecutive
//      post rows, every lane streams its own row with 16-byte coalesced loads
//      (512 contiguous bytes per warp per slot) and looks each pre up in the
//      previous step's spike bitmap staged in shared memory (tile by tile when
//      it exceeds one tile).  No float atomics and no cross-lane reduction: the
//      row sum is an int32 in the lane that owns the neuron, exact and order
//      free.
//   K1 LIF update: fp32 with explicit _rn intrinsics in the fixed order of
//      DESIGN.md section 3 (no FMA contraction), Philox drive.
//   K2 spike detect/bucket: __ballot_sync/__popc warp-aggregated appends of
//      fired internal ids into per-destination buckets (hop_mask from the
//      reference's RoutingTable, routing.py:184-231).
// nc_sim_step_fused runs K3+K1+K2 in one pass, so the synaptic input never
// touches HBM.  The unfused entry points exist for the event-driven variant.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include "nc_common.h"
#include "philox.cuh"
#include "sim_device.cuh"

namespace {
using namespace ncdev;

constexpr int kThreads = 1024;    // one CTA per SM in the smem-bitmap variant
constexpr int kMaxTiles = 256;    // bitmap tiles per shard (sell.py plan_tiles)
__global__ void __launch_bounds__(1024, 1) k_step_binned(const nc_shard_t sh, const nc_lif_params_t p);
// K3 (+K1+K2 when kLif).  kTiled: the bitmap does not fit in shared memory;
// every CTA owns a fixed range of slices, loops over the bitmap tiles and
// keeps the per-row partial sums in shared memory behind the tile.
// kGlobalPart: tiled partial sums in `acc` (flags bit 0), with an L2 prefetch
// of the synapse stream (measured: +7% there, -2% with shared partials).
template <bool kTiled, bool kLif, bool kGlobalPart = false, bool kSend = false>
__global__ void __launch_bounds__(kThreads, 1)
k_step_fused(const nc_shard_t sh, const nc_lif_params_t p) {
  extern __shared__ uint4 smem4[];
  __shared__ unsigned int block_count;
  const int step = *sh.step;
  const uint32_t* prev = ((step - 1) & 1) ? sh.bitmap1 : sh.bitmap0;
  uint32_t* cur = (step & 1) ? sh.bitmap1 : sh.bitmap0;
  uint32_t* sbm = reinterpret_cast<uint32_t*>(smem4);
  if (threadIdx.x == 0) block_count = 0;
  if (sh.kstamp && threadIdx.x == 0) atomicMin(&sh.kstamp[2 * (step % sh.kstamp_steps)], globaltimer_ns());
  if (kLif) clear_remote(sh, cur, blockIdx.x, gridDim.x);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int n_slices = (sh.n_local + 31) >> 5;
  const int32_t g_inh = p.g_inh;
  const uint4* syn4 = reinterpret_cast<const uint4*>(sh.syn);
  uint32_t my_spikes = 0;

  if (!kTiled) {
    const uint4* src = reinterpret_cast<const uint4*>(prev);
    const int n4 = (sh.n_words + 3) >> 2;
    for (int k = threadIdx.x; k < n4; k += blockDim.x) smem4[k] = ld_keep(src + k);
    __syncthreads();
    // CTA c owns slices c, c+G, ... (rows are degree ordered, so interleaving
    // balances the CTAs); its warps claim them dynamically (no tail of warps
    // with one slice more than others), and the next claim's block start and
    // row_meta load while the current slice streams
    const int G = gridDim.x, c = blockIdx.x;
    const int cnt = c < n_slices ? (n_slices - c + G - 1) / G : 0;
    __shared__ int next1;
    if (threadIdx.x == 0) next1 = 0;
    __syncthreads();
    auto claim = [&](int64_t& b0, uint32_t& m) {
      int j = 0;
      if (lane == 0) j = atomicAdd(&next1, 1);
      j = __shfl_sync(kFull, j, 0);
      if (j < cnt) {
        const int row = ((c + j * G) << 5) + lane;
        b0 = sh.slice_ptr[c + j * G];
        m = row < sh.n_local ? sh.row_meta[row] : 0u;
      }
      return j;
    };
    int64_t b0 = 0;
    uint32_t meta = 0u;
    int j = claim(b0, meta);
    while (j < cnt) {
      int64_t b0n = 0;
      uint32_t metan = 0u;
      const int jn = claim(b0n, metan);
      const int slice = c + j * G;
      const int row = (slice << 5) + lane;
      const int32_t acc = sell_row_sum<0>(syn4 + b0, meta, sbm, g_inh, lane, 0u);
      if (kLif) {
        const uint32_t fm = update_slice<kSend>(sh, p, cur, slice, lane, acc, step);
        if (lane == 0) my_spikes += __popc(fm);
      } else if (row < sh.n_local) {
        sh.acc[row] = acc;
      }
      j = jn;
      b0 = b0n;
      meta = metan;
    }
  } else {
    // Tiled: two (or three) tile buffers in shared memory, filled by TMA bulk copies
    // that complete on mbarriers.  Warps claim (slice, tile) blocks dynamically and
    // move on to the next tile as soon as they run out of work -- no CTA-wide
    // barrier between tiles: the last warp to leave tile t refills t's buffer
    // with tile t + NB.  Warps span at most NB consecutive tiles, so partial
    // sums are combined with shared (or, flags bit 0, global) integer atomics.
    const int T = sh.n_tiles, TW = sh.tile_words;
    // CTA c owns slices c, c+G, c+2G, ...: rows are ordered by degree inside the
    // shard, so interleaving gives every CTA the same mix of long and short rows
    const int G = gridDim.x, c = blockIdx.x;
    const int cnt = c < n_slices ? (n_slices - c + G - 1) / G : 0;
    constexpr bool pglob = kGlobalPart;
    // flags bit 3: three tile buffers (small tiles of small shards: a warp that runs out of
    // tile t + 1 finds t + 2 already loaded instead of waiting for the last warp of t)
    const int NB = (sh.flags & 8) ? 3 : 2;
    int32_t* spart = reinterpret_cast<int32_t*>(sbm + NB * TW);   // shared partials (!pglob)
    __shared__ uint64_t full[3];
    __shared__ int done[3];
    __shared__ int next_slice[kMaxTiles];
    for (int k = threadIdx.x; k < cnt * 32; k += blockDim.x) {
      const int row = ((c + (k >> 5) * G) << 5) + (k & 31);
      if (!pglob) spart[k] = 0;
      else if (row < sh.n_local) sh.acc[row] = 0;
    }
    for (int k = threadIdx.x; k < T; k += blockDim.x) next_slice[k] = 0;
    // flags bits 1-2: blocks split into 2^s parts claimed separately (small shards)
    const int sp = (sh.flags >> 1) & 3;
    const int nparts = 1 << sp;
    const int units = cnt << sp;
    auto tile_bytes = [&](int t) {
      return (uint32_t)((min(TW, sh.n_words - t * TW) + 3) >> 2) * 16u;
    };
    if (threadIdx.x == 0) {
      for (int k = 0; k < NB; ++k) {
        done[k] = 0;
        mbar_init(&full[k], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int t = 0; t < NB && t < T; ++t) {
        mbar_arrive_expect_tx(&full[t], tile_bytes(t));
        bulk_g2s(sbm + t * TW, prev + t * TW, tile_bytes(t), &full[t]);
      }
    }
    __syncthreads();
    for (int t = 0; t < T; ++t) {
      const int b = t % NB;
      const int w0 = t * TW;
      mbar_wait(&full[b], (uint32_t)(t / NB) & 1u);
      // entries hold tile-relative pre ids: look them up in the staged copy directly
      const uint32_t* bm = sbm + b * TW;
      // the next claim's block start and row_meta load (and its first slots are
      // prefetched into L2) while the current block streams
      auto claim = [&](int64_t& b0, uint32_t& m) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&next_slice[t], 1);
        u = __shfl_sync(kFull, u, 0);
        if (u < units) {
          const int j = u >> sp;
          const int pos = ((c + j * G) << 5) + lane;
          b0 = sh.slice_ptr[(int64_t)(c + j * G) * T + t];
          m = pos < sh.n_local ? sh.row_meta[(int64_t)t * sh.n_local + pos] : 0u;
          if (kPfTiled > 0 && pglob && lane == 0) prefetch_l2(syn4 + b0, kPfTiled * 512u);
        }
        return u;
      };
      int64_t b0 = 0;
      uint32_t meta = 0u;
      int u = claim(b0, meta);
      while (u < units) {
        int64_t b0n = 0;
        uint32_t metan = 0u;
        const int un = claim(b0n, metan);
        const int j = u >> sp;
        const int pos = ((c + j * G) << 5) + lane;
        // CTA-local index k of the row placed here in tile t (rows stay inside the CTA's slices)
        const int k = pos < sh.n_local ? sh.row_perm[(int64_t)t * sh.n_local + pos] : -1;
        const int32_t sum = sell_row_sum<pglob ? kPfTiled : 0>(syn4 + b0, meta, bm, g_inh, lane, 0u,
                                                               u & (nparts - 1), nparts);
        // partials of sparse tiles are mostly 0 (no pre of the row fired): skip those
        if (k >= 0 && sum != 0) {
          if (!pglob) atomicAdd(&spart[k], sum);
          else red_add(&sh.acc[((c + (k >> 5) * G) << 5) + (k & 31)], sum);
        }
        u = un;
        b0 = b0n;
        meta = metan;
      }
      // leave tile t; the last warp out refills its buffer with tile t + NB
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&done[b], 1) == wpb - 1) {
          done[b] = 0;
          if (t + NB < T) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full[b], tile_bytes(t + NB));
            bulk_g2s(sbm + b * TW, prev + (t + NB) * TW, tile_bytes(t + NB), &full[b]);
          }
        }
      }
    }
    __syncthreads();
    if (pglob) __threadfence();
    for (int j = warp; j < cnt; j += wpb) {
      const int slice = c + j * G;
      const int row = (slice << 5) + lane;
      const int32_t acc = pglob ? (row < sh.n_local ? sh.acc[row] : 0) : spart[j * 32 + lane];
      if (kLif) {
        const uint32_t fm = update_slice<kSend>(sh, p, cur, slice, lane, acc, step);
        if (lane == 0) my_spikes += __popc(fm);
      } else if (row < sh.n_local) {
        sh.acc[row] = acc;
      }
    }
  }
  if (kLif) add_spike_total(sh, my_spikes, &block_count);
  if (kLif) xsend_headers<kSend>(sh, step);
  if (sh.kstamp) {   // uniform
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&sh.kstamp[2 * (step % sh.kstamp_steps) + 1], globaltimer_ns());
  }
}

// K1+K2 alone: consumes and zeroes acc.
#ifndef NC_LIF_UNROLL_ALONE
#define NC_LIF_UNROLL_ALONE 8
#endif
// K1+K2 as its own kernel (per-kernel event-driven engine): 8 tiles per warp in flight
// (128 registers, 2 CTAs per SM; config 3, 10 M rows: 1 / 3 / 4 / 8 in flight = 453 /
// 320 / 242 / 103 us), while inside the persistent engine, capped at 80 registers, 4 is
// best (88 us).
__global__ void __launch_bounds__(kLifThreads) k_lif_update(const nc_shard_t sh, const nc_lif_params_t p) {
  __shared__ LifSmem S;
  lif_phase<kLifWarps, NC_LIF_UNROLL_ALONE>(sh, p, *sh.step, blockIdx.x, gridDim.x, S);
}

__global__ void __launch_bounds__(256) k_deliver_push(const nc_shard_t sh, int32_t negg) {
  __shared__ PushSmem P;
  push_phase(sh, negg, *sh.step, P);
}

__global__ void k_end_step(const nc_shard_t sh) {
  const int t = threadIdx.x;
  if (t < sh.n_shards) sh.bucket_count[t] = 0;
  if (t < 4 + (sh.push_windows > 1 ? sh.push_windows : 0) && sh.work) sh.work[t] = 0u;
  if (t == 0) {
    if (sh.fired_count) *sh.fired_count = 0;
    if (sh.spk_count) sh.spk_count[(*sh.step + 1) & 1] = 0;   // the list step + 1 appends to
    *sh.step += 1;
  }
}

__global__ void k_init(const nc_shard_t sh, const nc_lif_params_t p) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t r = t0; r < sh.n_local; r += stride) {
    nc_u32x4 c = {sh.gid[r], 0xFFFFFFFFu, NC_TAG_VINIT, 0u};
    nc_u32x4 x = nc_philox4x32_10(c, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
    const float u = __fmul_rn(__uint2float_rn(x.x >> 8), 5.9604644775390625e-08f);  // 2^-24
    sh.v[r] = __fadd_rn(p.v_reset, __fmul_rn(u, p.v_init_span));
    sh.i_syn[r] = 0.0f;
    sh.refrac[r] = 0;
    if (sh.acc) sh.acc[r] = 0;
  }
  for (int64_t w = t0; w < sh.n_words; w += stride) {
    sh.bitmap0[w] = 0u;
    sh.bitmap1[w] = 0u;
  }
  if (t0 < sh.n_shards) sh.bucket_count[t0] = 0;
  if (t0 < 4 + (sh.push_windows > 1 ? sh.push_windows : 0) && sh.work) sh.work[t0] = 0u;
  if (t0 < 2 && sh.spk_count) sh.spk_count[t0] = 0;
  if (t0 == 0) {
    *sh.step = 0;
    sh.status[0] = 0;
    sh.status[1] = 0;
    if (sh.fired_count) *sh.fired_count = 0;
    if (sh.spike_total) *sh.spike_total = 0ull;
  }
}

int g_num_sms = 0;
bool g_prepared = false;

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

int g_max_dyn_smem = 0;   // opt-in limit minus the kernels' static shared memory

// dynamic shared memory of the step kernel: whole bitmap, or one tile plus
// the per-row partial sums of the CTA's slice range
size_t step_smem_bytes(const nc_shard_t& sh, int grid) {
  if (sh.n_tiles <= 1) return (size_t)((sh.n_words + 3) >> 2) * 16;
  // two (flags bit 3: three) tile buffers (+ the CTA's partial sums unless they live in acc)
  const size_t bufs = (size_t)sh.tile_words * 4 * ((sh.flags & 8) ? 3 : 2);
  if (sh.flags & 1) return bufs;
  const int n_slices = (sh.n_local + 31) >> 5;
  const int per = (n_slices + grid - 1) / grid;
  return bufs + (size_t)per * 32 * 4;
}

template <bool kLif>
int launch_step(const nc_shard_t& sh, const nc_lif_params_t& p, cudaStream_t st) {
  // tiled: the row placement was built for cta_groups CTAs (sh.row_perm)
  const int grid = sh.n_tiles > 1 ? sh.cta_groups : num_sms();
  size_t smem = step_smem_bytes(sh, grid);
  if (smem > (size_t)g_max_dyn_smem) {
    nc_set_error("step kernel needs %zu B of shared memory (tile_words=%d): re-tile the network", smem,
                 sh.tile_words);
    return NC_E_ARG;
  }
  // the fused P2P send is a separate instantiation so that the plain step carries none of it
  const bool send = kLif && sh.xsend_on;
  if (sh.n_tiles <= 1)
    send ? k_step_fused<false, kLif, false, true><<<grid, kThreads, smem, st>>>(sh, p)
         : k_step_fused<false, kLif><<<grid, kThreads, smem, st>>>(sh, p);
  else if (sh.flags & 1)
    send ? k_step_fused<true, kLif, true, true><<<grid, kThreads, smem, st>>>(sh, p)
         : k_step_fused<true, kLif, true><<<grid, kThreads, smem, st>>>(sh, p);
  else
    send ? k_step_fused<true, kLif, false, true><<<grid, kThreads, smem, st>>>(sh, p)
         : k_step_fused<true, kLif, false><<<grid, kThreads, smem, st>>>(sh, p);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

int check_shard(const nc_shard_t* sh) {
  if (!sh || sh->n_local < 0 || sh->n_words < 1 || (sh->local_base & 31) || !sh->step ||
      !sh->status || !sh->bitmap0 || !sh->bitmap1 || sh->n_tiles < 1 ||
      (sh->n_tiles > 1 && (sh->tile_words < 4 || (sh->tile_words & 3) || sh->n_tiles > kMaxTiles ||
                           sh->cta_groups < 1 ||
                           (int64_t)sh->tile_words * sh->n_tiles < sh->n_words)) ||
      ((sh->flags & 1) && !sh->acc)) {
    nc_set_error("invalid nc_shard_t");
    return NC_E_ARG;
  }
  if (sh->xsend_on) {
    // fused P2P send: every message slot holds xsend_cap + 1 words, so a bucket
    // longer than that would run into the next source's slot (or past the peer's
    // IPC allocation); headers use work[2..3]
    if (!sh->work || sh->xsend_cap < sh->bucket_cap || sh->n_shards > kThreads) {
      nc_set_error("invalid nc_shard_t: fused send needs work counters, xsend_cap >= bucket_cap "
                   "(%lld < %lld) and n_shards <= %d", (long long)sh->xsend_cap, (long long)sh->bucket_cap,
                   kThreads);
      return NC_E_ARG;
    }
    for (int h = 0; h < sh->n_shards; ++h)
      if (h != sh->shard && !sh->xsend[h]) {   // every peer gets a header (heartbeat)
        nc_set_error("invalid nc_shard_t: fused send has no inbox for peer %d", h);
        return NC_E_ARG;
      }
  }
  return NC_OK;
}

}  // namespace

template <typename K>
int opt_in_smem(K kernel, int optin) {
  cudaFuncAttributes fa;
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, kernel));
  const int dyn = optin - (int)fa.sharedSizeBytes;
  NC_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
  if (g_max_dyn_smem == 0 || dyn < g_max_dyn_smem) g_max_dyn_smem = dyn;
  return NC_OK;
}

// Set kernel attributes once, outside any stream capture.
extern "C" int nc_sim_prepare(void) {
  (void)num_sms();
  int dev = 0, optin = 0;
  NC_CUDA_TRY(cudaGetDevice(&dev));
  NC_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  g_max_dyn_smem = 0;
  if (int e = opt_in_smem(k_step_fused<false, true>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<true, true>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<false, false>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<true, false>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<true, true, true>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<true, false, true>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<false, true, false, true>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<true, true, true, true>, optin)) return e;
  if (int e = opt_in_smem(k_step_fused<true, true, false, true>, optin)) return e;
  if (int e = opt_in_smem(k_step_binned, optin)) return e;
  // Load every kernel of the step path now.  With CUDA's lazy module loading the
  // first launch of a kernel loads it, and that load waits for the device: a
  // first launch queued behind a spinning exchange kernel (k_p2p waits for its
  // peers) would stall the host thread until the watchdog ends the spin.
  cudaFuncAttributes fa;
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_lif_update));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_deliver_push));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_end_step));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_init));
  if (int e = ncx_load_exchange_kernels()) return e;
  if (int e = ncx_load_local_kernels()) return e;
  if (int e = ncx_load_persistent_kernels()) return e;
  g_prepared = true;
  return NC_OK;
}

extern "C" int nc_sim_init(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream) {
  if (int e = check_shard(sh)) return e;
  k_init<<<4 * num_sms(), 256, 0, (cudaStream_t)stream>>>(*sh, *p);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_step_fused(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream) {
  if (int e = check_shard(sh)) return e;
  if (!g_prepared)
    if (int e = nc_sim_prepare()) return e;
  return launch_step<true>(*sh, *p, (cudaStream_t)stream);
}

extern "C" int nc_sim_deliver_pull(const nc_shard_t* sh, int32_t g_inh, void* stream) {
  if (int e = check_shard(sh)) return e;
  if (!sh->acc) {
    nc_set_error("nc_sim_deliver_pull: shard has no acc buffer");
    return NC_E_ARG;
  }
  if (!g_prepared)
    if (int e = nc_sim_prepare()) return e;
  nc_lif_params_t p{};
  p.g_inh = g_inh;
  return launch_step<false>(*sh, p, (cudaStream_t)stream);
}

extern "C" int nc_sim_deliver_push(const nc_shard_t* sh, int32_t g_inh, void* stream) {
  if (int e = check_shard(sh)) return e;
  if (!sh->push_rowptr || !sh->push_syn || !sh->acc || !sh->work ||
      (sh->push_windows > 1 && (!sh->push_winoff || sh->push_windows > 32))) {
    nc_set_error("nc_sim_deliver_push: shard has no push CSR / acc / work counters");
    return NC_E_ARG;
  }
  int64_t grid = ((sh->n_words + 31) / 32 + 1) / 2;   // blocks claim 32-word chunks dynamically
  if (grid > 8 * num_sms()) grid = 8 * num_sms();
  if (grid < 1) grid = 1;
  k_deliver_push<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(*sh, -g_inh);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_lif_update(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream) {
  if (int e = check_shard(sh)) return e;
  if (!sh->acc) {
    nc_set_error("nc_sim_lif_update: shard has no acc buffer");
    return NC_E_ARG;
  }
  // contiguous tile ranges, one wave of resident CTAs (more if a range would exceed
  // the shared spike-mask storage): one global atomic per bucket per CTA
  const int tiles = (sh->n_local + 31) / 32;
  static int occ = 0;
  if (occ == 0) {
    NC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lif_update, kLifThreads, 0));
    if (occ < 1) occ = 1;
  }
  int grid = occ * num_sms();
  if ((tiles + grid - 1) / grid > kLifMaxTiles) grid = (tiles + kLifMaxTiles - 1) / kLifMaxTiles;
  if (grid > tiles) grid = tiles > 0 ? tiles : 1;
  k_lif_update<<<grid, kLifThreads, 0, (cudaStream_t)stream>>>(*sh, *p);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_end_step(const nc_shard_t* sh, void* stream) {
  if (int e = check_shard(sh)) return e;
  k_end_step<<<1, 64, 0, (cudaStream_t)stream>>>(*sh);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

// ---------------------------------------------------------------- push CSR
// Transpose of the SELL-32 pull synapses (rows = internal pre ids) built on
// the device by counting sort: phase 0 counts entries per pre into
// push_rowptr[pre + 1]; the host scans; phase 1 claims slots with atomics.
// Entry = (inhibitory << 31) | ((q - 1) << 26) | post_local.
namespace {
__global__ void k_push_build(const nc_shard_t sh, int phase, int64_t* rowptr, int32_t* fill, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int T = sh.n_tiles;
  const int n_slices = (sh.n_local + 31) >> 5;
  const int64_t n_blocks = (int64_t)n_slices * T;
  const uint4* syn4 = reinterpret_cast<const uint4*>(sh.syn);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t blk = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; blk < n_blocks; blk += nw) {
    const int slice = (int)(blk / T), t = (int)(blk % T);
    const int pos = (slice << 5) + lane;
    const int row = pos < sh.n_local ? (int)placed_row(sh.row_perm, sh.n_local, sh.cta_groups, t, pos) : pos;
    const int64_t b0 = sh.slice_ptr[blk];
    const uint32_t meta = pos < sh.n_local ? sh.row_meta[(int64_t)t * sh.n_local + pos] : 0u;
    const int emid = (int)(meta & 0xFFFFu), mine = (int)(meta >> 16);
    const int hi = (int)__reduce_max_sync(0xffffffffu, (unsigned)mine);
    int off = 0;
    for (int u = 0; u < hi; ++u) {
      const int pos = jsell_pos(u, mine, lane, off);
      if (u >= mine) continue;
      const Fields x = unpack_slot(syn4[b0 + pos]);
#pragma unroll
      for (int c = 0; c < kSlotEntries; ++c) {
        const uint32_t f = x.f[c] & kFieldMask;
        const uint32_t q = f >> 19;
        if (q == 0) continue;
        const uint32_t pre = field_id(f) + (uint32_t)t * (uint32_t)sh.tile_words * 32u;
        if (phase == 0) {
          atomicAdd(reinterpret_cast<unsigned long long*>(rowptr + pre + 1), 1ull);
        } else {
          const int32_t slot = atomicAdd(fill + pre, 1);
          out[rowptr[pre] + slot] = ((u >= emid ? 1u : 0u) << 31) | ((q - 1u) << 26) | (uint32_t)row;
        }
      }
    }
  }
}

// Binned push: same walk over the pull synapses as k_push_build; the bin of a
// synapse is the CTA that owns its post row in k_step_binned.
__global__ void k_push_binned(const nc_shard_t sh, int phase, uint32_t* counts, const int64_t* rowptr,
                              const uint16_t* binoff, uint32_t* fill, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const int T = sh.n_tiles;
  const int B = sh.pb_bins, R = sh.pb_rows;
  const int n_slices = (sh.n_local + 31) >> 5;
  const int64_t n_blocks = (int64_t)n_slices * T;
  const uint4* syn4 = reinterpret_cast<const uint4*>(sh.syn);
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t blk = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; blk < n_blocks; blk += nw) {
    const int slice = (int)(blk / T), t = (int)(blk % T);
    const int pos = (slice << 5) + lane;
    const int row = pos < sh.n_local ? (int)placed_row(sh.row_perm, sh.n_local, sh.cta_groups, t, pos) : pos;
    const int64_t b0 = sh.slice_ptr[blk];
    const uint32_t meta = pos < sh.n_local ? sh.row_meta[(int64_t)t * sh.n_local + pos] : 0u;
    const int emid = (int)(meta & 0xFFFFu), mine = (int)(meta >> 16);
    const int hi = (int)__reduce_max_sync(0xffffffffu, (unsigned)mine);
    const int bin = row / R;
    const uint32_t rel = (uint32_t)(row - bin * R);
    int off = 0;
    for (int u = 0; u < hi; ++u) {
      const int p = jsell_pos(u, mine, lane, off);
      if (u >= mine) continue;
      const Fields x = unpack_slot(syn4[b0 + p]);
#pragma unroll
      for (int c = 0; c < kSlotEntries; ++c) {
        const uint32_t f = x.f[c] & kFieldMask;
        const uint32_t q = f >> 19;
        if (q == 0) continue;
        const uint32_t pre = field_id(f) + (uint32_t)t * (uint32_t)sh.tile_words * 32u;
        const int64_t key = (int64_t)pre * B + bin;
        if (phase == 0) {
          atomicAdd(counts + key, 1u);
        } else {
          const uint32_t k = atomicAdd(fill + key, 1u);
          out[rowptr[pre] + binoff[(int64_t)pre * (B + 1) + bin] + k] =
              ((u >= emid ? 1u : 0u) << 31) | ((q - 1u) << 26) | rel;
        }
      }
    }
  }
}

// One event-driven step with binned push (see nc_sim_step_binned).
constexpr int kBinThreads = 1024;
constexpr int kBinWarps = kBinThreads / 32;

__global__ void __launch_bounds__(kBinThreads, 1) k_step_binned(const nc_shard_t sh, const nc_lif_params_t p) {
  extern __shared__ int32_t sacc[];
  __shared__ LifSmemT<kBinWarps> S;
  const int step = *sh.step;
  const int c = blockIdx.x, B = sh.pb_bins, R = sh.pb_rows;
  const int32_t negg = -p.g_inh;
  for (int k = threadIdx.x; k < R; k += blockDim.x) sacc[k] = 0;
  __syncthreads();
  // the spikes of step - 1 (local from that step's LIF, remote from its exchange)
  const int pl = (step - 1) & 1;
  const int64_t n_spk = min((int64_t)sh.spk_count[pl], sh.spk_cap);
  const uint32_t* spk = sh.spk_ids + (int64_t)pl * sh.spk_cap;
  // lane per spike, 4 spikes in flight per thread: their bin offsets, then their
  // entries 8 at a time (32 loads in flight), then the shared-memory sums
  constexpr int kS = 4, kE = 8;
  for (int64_t i0 = (int64_t)threadIdx.x; i0 < n_spk; i0 += kS * (int64_t)blockDim.x) {
    int64_t lo[kS];
    int n[kS];
#pragma unroll
    for (int u = 0; u < kS; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      lo[u] = 0;
      n[u] = 0;
      if (i < n_spk) {
        const uint32_t pre = spk[i];
        const uint16_t* bo = sh.pb_binoff + (int64_t)pre * (B + 1) + c;
        const int b0 = bo[0], b1 = bo[1];
        lo[u] = sh.pb_rowptr[pre] + b0;
        n[u] = b1 - b0;
      }
    }
    int left = max(max(n[0], n[1]), max(n[2], n[3]));
    for (int k0 = 0; k0 < left; k0 += kE) {
      uint32_t x[kS][kE];
#pragma unroll
      for (int u = 0; u < kS; ++u)
#pragma unroll
        for (int k = 0; k < kE; ++k) x[u][k] = (k0 + k < n[u]) ? __ldg(sh.pb_syn + lo[u] + k0 + k) : 0u;
#pragma unroll
      for (int u = 0; u < kS; ++u)
#pragma unroll
        for (int k = 0; k < kE; ++k)
          if (k0 + k < n[u]) {
            const int32_t q = (int32_t)((x[u][k] >> 26) & 31u) + 1;
            atomicAdd(&sacc[x[u][k] & 0x03FFFFFFu], (x[u][k] >> 31) ? q * negg : q);
          }
    }
  }
  __syncthreads();
  lif_phase<kBinWarps>(sh, p, step, c, B, S, sacc);
}
}  // namespace

extern "C" int nc_build_push_csr(const nc_shard_t* sh, int32_t phase, int64_t* push_rowptr, int32_t* push_fill,
                                 uint32_t* push_syn, void* stream) {
  if (int e = check_shard(sh)) return e;
  if (phase != 0 && phase != 1) {
    nc_set_error("nc_build_push_csr: phase must be 0 or 1");
    return NC_E_ARG;
  }
  k_push_build<<<16 * num_sms(), 256, 0, (cudaStream_t)stream>>>(*sh, phase, push_rowptr, push_fill, push_syn);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_build_push_binned(const nc_shard_t* sh, int32_t phase, uint32_t* counts, const int64_t* pb_rowptr,
                                    const uint16_t* pb_binoff, uint32_t* fill, uint32_t* pb_syn, void* stream) {
  if (int e = check_shard(sh)) return e;
  if ((phase != 0 && phase != 1) || sh->pb_bins < 1 || sh->pb_rows < 32 || (sh->pb_rows & 31) ||
      (int64_t)sh->pb_bins * sh->pb_rows < sh->n_local || (phase == 0 && !counts) ||
      (phase == 1 && (!pb_rowptr || !pb_binoff || !fill || !pb_syn))) {
    nc_set_error("nc_build_push_binned: bad arguments");
    return NC_E_ARG;
  }
  k_push_binned<<<16 * num_sms(), 256, 0, (cudaStream_t)stream>>>(*sh, phase, counts, pb_rowptr, pb_binoff, fill,
                                                                  pb_syn);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_step_binned(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream) {
  if (int e = check_shard(sh)) return e;
  if (!p || !sh->pb_rowptr || !sh->pb_binoff || !sh->pb_syn || !sh->spk_ids || !sh->spk_count || sh->pb_bins < 1 ||
      sh->pb_rows < 32 || (sh->pb_rows & 31) || (int64_t)sh->pb_bins * sh->pb_rows < sh->n_local ||
      sh->pb_rows / 32 > kLifMaxTiles) {
    nc_set_error("nc_sim_step_binned: shard has no binned push / spike lists, or bins too large");
    return NC_E_ARG;
  }
  if (!g_prepared)
    if (int e = nc_sim_prepare()) return e;
  const size_t smem = (size_t)sh->pb_rows * 4;
  if (smem > (size_t)g_max_dyn_smem) {
    nc_set_error("nc_sim_step_binned: %d rows per bin need %zu B of shared memory", sh->pb_rows, smem);
    return NC_E_ARG;
  }
  k_step_binned<<<sh->pb_bins, kBinThreads, smem, (cudaStream_t)stream>>>(*sh, *p);
  NC_LAUNCH_CHECK();
  return NC_OK;
}
