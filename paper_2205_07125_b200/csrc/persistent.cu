// Persistent event-driven engine: one cooperative kernel per GPU runs many
// steps back to back -- push delivery, LIF + bucket compaction, and the
// device-initiated P2P spike exchange -- separated by in-kernel grid barriers,
// so a step costs no kernel launches and no host involvement at all.
//
// Per step (same arithmetic as the per-kernel path, hence bit-identical):
//   1. push_phase   acc += weights of the previous step's spikes (all blocks; with
//                   push windows, one L2-sized post-row window at a time, a grid
//                   barrier between windows)
//   2. grid barrier
//   3. lif_phase    LIF update, spike bitmap, CTA-aggregated bucket appends
//   4. grid barrier; stamp "buckets ready"
//   5. p2p_block    blocks [0, n*B): NVLink stores of tagged 8-byte words into the
//                   peers' inboxes, poll + scatter (relays forward as ids arrive)
//   6. grid barrier; stamp "all inbound spikes in the bitmap"; reset counters
// The grid is sized from the occupancy calculator and launched cooperatively,
// so every block is resident and the barriers cannot deadlock; the flag waits
// of step 5 are bounded by the exchange watchdog (status[1]).

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include "nc_common.h"
#include "sim_device.cuh"
#include "xchg_device.cuh"

namespace {

constexpr int kPThreads = ncdev::kLifThreads;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier.  The cooperative-groups grid sync (hardware-assisted arrival
// counting) is several times cheaper than a spin on one global counter polled
// by every block.  Every wait inside a phase is bounded (exchange watchdog),
// so every block reaches every barrier.
__device__ __forceinline__ void grid_sync(unsigned int*, unsigned int, int32_t*) {
  cooperative_groups::this_grid().sync();
}

#ifndef NC_PERSIST_MIN_BLOCKS
#define NC_PERSIST_MIN_BLOCKS 3   // <= 85 registers: 3 CTAs (24 warps) per SM for the latency-bound phases
#endif

__global__ void __launch_bounds__(kPThreads, NC_PERSIST_MIN_BLOCKS) k_persistent(const nc_shard_t sh, const nc_lif_params_t p,
                                                          const nc_xchg_t X, int has_x, int n_steps, int B,
                                                          unsigned int* gbar, unsigned long long* st_ready,
                                                          unsigned long long* st_done, int stamp_cap,
                                                          unsigned long long* phase_st) {
  __shared__ ncdev::LifSmem S;
  __shared__ ncdev::PushSmem P;
  const int nblk = gridDim.x, bid = blockIdx.x;
  const int nex = has_x ? X.n * B : 0;
  const int32_t negg = -p.g_inh;
  int step = *sh.step;
  unsigned int k = 0;
  const bool ph = phase_st && bid == 0 && threadIdx.x == 0;
  for (int s = 0; s < n_steps; ++s, ++step) {
    if (ph && s < 64) phase_st[s * 4 + 0] = gtimer();
    if (sh.push_windows > 1) {   // one window of post rows at a time: its reductions stay in L2
      for (int w = 0; w < sh.push_windows; ++w) {
        ncdev::push_phase(sh, negg, step, P, w);
        if (w + 1 < sh.push_windows) grid_sync(gbar, ++k * nblk, sh.status);
      }
    } else {
      ncdev::push_phase(sh, negg, step, P);
    }
    grid_sync(gbar, ++k * nblk, sh.status);
    if (ph && s < 64) phase_st[s * 4 + 1] = gtimer();
    ncdev::lif_phase(sh, p, step, bid, nblk, S);
    grid_sync(gbar, ++k * nblk, sh.status);
    if (ph && s < 64) phase_st[s * 4 + 2] = gtimer();
    if (bid == 0 && threadIdx.x == 0 && st_ready && step < stamp_cap) st_ready[step] = gtimer();
    if (bid < nex) ncxchg::p2p_block(X, bid, B, step);
    grid_sync(gbar, ++k * nblk, sh.status);
    if (ph && s < 64) phase_st[s * 4 + 3] = gtimer();
    if (bid == 0) {
      if (threadIdx.x == 0 && st_done && step < stamp_cap) st_done[step] = gtimer();
      if ((int)threadIdx.x < sh.n_shards) sh.bucket_count[threadIdx.x] = 0;
      if (threadIdx.x == 0) sh.work[0] = 0u;   // push chunk claims of the next step
      if ((int)threadIdx.x < sh.push_windows) sh.work[4 + threadIdx.x] = 0u;   // windowed claims
      if (has_x && (int)threadIdx.x < X.n) X.fwd_count[threadIdx.x] = 0;
      if (threadIdx.x == 0 && sh.fired_count) *sh.fired_count = 0;
    }
    // the counters reset above are next touched after the next push barrier
  }
  if (bid == 0 && threadIdx.x == 0) *sh.step = step;
}

}  // namespace

static unsigned long long* g_phase_stamps = nullptr;

// Diagnostics: record (start, after push, after LIF, after exchange) globaltimer
// stamps of the first 64 steps of the next persistent launches into dst[64][4].
int ncx_load_persistent_kernels(void) {
  cudaFuncAttributes fa;
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_persistent));
  return NC_OK;
}

extern "C" int nc_persistent_phase_stamps(unsigned long long* dst) {
  g_phase_stamps = dst;
  return NC_OK;
}

// Largest shard (rows) the persistent engine takes on this device: its LIF phase keeps a
// spike mask per 32-row tile of each CTA's range in shared memory.
extern "C" int64_t nc_persistent_max_rows(void) {
  int dev = 0, sms = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_persistent, kPThreads, 0) != cudaSuccess || occ < 1)
    return 0;
  const int64_t grid = (int64_t)sms * (occ < 8 ? occ : 8);
  return grid * ncdev::kLifMaxTiles * 32;
}

extern "C" int nc_run_persistent(const nc_shard_t* sh, const nc_lif_params_t* p, const nc_xchg_t* X,
                                 int32_t n_steps, int32_t blocks_per_peer, unsigned int* gbar,
                                 unsigned long long* stamp_ready, unsigned long long* stamp_done, int32_t stamp_cap,
                                 void* stream) {
  if (!sh || !p || !gbar || n_steps < 0 || !sh->push_rowptr || !sh->push_syn || !sh->acc || !sh->step ||
      !sh->status || !sh->work) {
    nc_set_error("nc_run_persistent: shard needs push CSR, acc, step and status buffers");
    return NC_E_ARG;
  }
  if (sh->push_windows > 1 && (!sh->push_winoff || sh->push_windows > 32 || sh->push_window_rows < 32 ||
                                (int64_t)sh->push_windows * sh->push_window_rows < sh->n_local)) {
    nc_set_error("nc_run_persistent: bad push windows (%d x %d rows, winoff %p)", sh->push_windows,
                 sh->push_window_rows, (const void*)sh->push_winoff);
    return NC_E_ARG;
  }
  if (X && X->fused_send) {   // this engine sends from its exchange blocks; nothing would write the inboxes
    nc_set_error("nc_run_persistent: nc_xchg_t.fused_send must be 0 (the persistent engine does its own send)");
    return NC_E_ARG;
  }
  if (n_steps == 0) return NC_OK;
  const int B = blocks_per_peer > 0 ? blocks_per_peer : 1;
  int dev = 0, sms = 0, occ = 0;
  NC_CUDA_TRY(cudaGetDevice(&dev));
  NC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  NC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_persistent, kPThreads, 0));
  if (occ < 1) {
    nc_set_error("nc_run_persistent: kernel does not fit on an SM");
    return NC_E_CUDA;
  }
  // every resident slot: the push and LIF phases are latency bound and want
  // as many warps in flight as the SM holds
  int per_sm = occ < 8 ? occ : 8;
  int grid = sms * per_sm;
  const int nex = X ? X->n * B : 0;
  if (grid < nex) {
    nc_set_error("nc_run_persistent: %d exchange blocks exceed the resident grid (%d)", nex, grid);
    return NC_E_ARG;
  }
  // the LIF phase keeps a spike mask per 32-row tile of the CTA's range in shared memory
  const int64_t tiles = ((int64_t)sh->n_local + 31) / 32;
  if ((tiles + grid - 1) / grid > ncdev::kLifMaxTiles) {
    nc_set_error("nc_run_persistent: %lld rows need more than %d tiles per CTA on a %d-CTA grid",
                 (long long)sh->n_local, ncdev::kLifMaxTiles, grid);
    return NC_E_ARG;
  }
  nc_xchg_t xz{};
  const nc_xchg_t& xr = X ? *X : xz;
  int has_x = X ? 1 : 0;
  NC_CUDA_TRY(cudaMemsetAsync(gbar, 0, sizeof(unsigned int), (cudaStream_t)stream));
  unsigned long long* phase = g_phase_stamps;
  void* args[] = {(void*)sh, (void*)p, (void*)&xr, &has_x, &n_steps, (void*)&B, &gbar, &stamp_ready, &stamp_done,
                  &stamp_cap, &phase};
  NC_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_persistent, dim3(grid), dim3(kPThreads), args, 0,
                                          (cudaStream_t)stream));
  return NC_OK;
}
