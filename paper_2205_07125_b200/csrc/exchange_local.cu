// Spike exchange between shards that live on the same device ("local"
// transport).  Used to run an N-partition network on one GPU -- the
// partition-invariance tests and the single-box stand-in for the paper's
// multi-GPU exchange -- with exactly the routing semantics of the multi-GPU
// transports:
//
//   phase 1: every shard s hands bucket s->h (filled by the step kernel from
//            hop_mask, i.e. RoutingTable next hops, routing.py:184-231) to h;
//            h ORs the ids into its current bitmap.  If h relays for s
//            (fwd_table[h][s] = destinations d whose path is (s, h, d)), h
//            re-buckets each id for every such d that hosts targets of the id
//            (dest_mask): the paper's relay, where the bridge forwards directly
//            to the destination GPU (SPEC two-level design decisions).
//   phase 2: bridges hand their forward buckets to the final destinations.
//
// Counters (int64): hop_ids[u][v] ids carried by channel u->v, deliv_ids[s][d]
// ids of source shard s that reached d and have targets there.  Both are
// route-dependent / route-independent respectively; tests check that direct
// and two-level runs give identical deliv_ids and rasters.

#include <cuda_runtime.h>
#include <stdint.h>
#include "nc_common.h"

namespace {

struct LocalShard {
  uint32_t* bitmap0;
  uint32_t* bitmap1;
  const uint32_t* bucket_ids;
  const int32_t* bucket_count;
  int64_t bucket_cap;
  int32_t local_base;
  int32_t n_local;
};

struct LocalSet {
  LocalShard s[NC_MAX_SHARDS];
  uint16_t fwd[NC_MAX_SHARDS][NC_MAX_SHARDS];  // fwd[b][s]: d's reached from s via b
  int32_t n;
  int32_t per_step;
  const int32_t* step;
};

__device__ __forceinline__ void add64(long long* p, long long v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

__device__ __forceinline__ uint32_t* cur_bitmap(const LocalShard& s, int step) {
  return (step & 1) ? s.bitmap1 : s.bitmap0;
}

__device__ __forceinline__ int owner_of(const LocalSet& L, uint32_t id) {
  for (int h = 0; h < L.n; ++h)
    if (id >= (uint32_t)L.s[h].local_base && id < (uint32_t)(L.s[h].local_base + L.s[h].n_local)) return h;
  return -1;
}

__global__ void k_phase1(const LocalSet L, const uint16_t* __restrict__ dest_mask, uint32_t* fwd_ids,
                         int32_t* fwd_count, int64_t fwd_cap, long long* hop_ids, long long* deliv_ids,
                         int32_t* status) {
  const int pair = blockIdx.y;
  const int src = pair / L.n, dst = pair % L.n;
  if (src == dst) return;
  const LocalShard& S = L.s[src];
  const int64_t cnt = min((int64_t)S.bucket_count[dst], S.bucket_cap);
  if (cnt == 0) return;
  const int step = *L.step;
  if (L.per_step) {
    hop_ids += (int64_t)step * L.n * L.n;
    deliv_ids += (int64_t)step * L.n * L.n;
  }
  uint32_t* cur = cur_bitmap(L.s[dst], step);
  const uint32_t* ids = S.bucket_ids + (int64_t)dst * S.bucket_cap;
  const uint32_t fwd = L.fwd[dst][src];
  __shared__ unsigned int n_deliv;
  if (threadIdx.x == 0) n_deliv = 0;
  __syncthreads();
  unsigned int my = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[k];
    atomicOr(cur + (id >> 5), 1u << (id & 31));
    const uint32_t dm = dest_mask[id];
    my += (dm >> dst) & 1u;
    if (fwd) {
      uint32_t f = dm & fwd;
      while (f) {
        const int x = __ffs(f) - 1;
        f &= f - 1;
        const int64_t slot = (int64_t)dst * L.n + x;
        const int32_t pos = atomicAdd(fwd_count + slot, 1);
        if (pos < fwd_cap) fwd_ids[slot * fwd_cap + pos] = id;
        else atomicExch(status, 1);
      }
    }
  }
  if (my) atomicAdd(&n_deliv, my);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (n_deliv) add64(deliv_ids + (int64_t)src * L.n + dst, (long long)n_deliv);
    if (blockIdx.x == 0) add64(hop_ids + (int64_t)src * L.n + dst, (long long)cnt);
  }
}

__global__ void k_phase2(const LocalSet L, const uint32_t* fwd_ids, const int32_t* fwd_count,
                         int64_t fwd_cap, long long* hop_ids, long long* deliv_ids) {
  const int pair = blockIdx.y;
  const int b = pair / L.n, x = pair % L.n;
  if (b == x) return;
  const int64_t cnt = min((int64_t)fwd_count[pair], fwd_cap);
  if (cnt == 0) return;
  const int step = *L.step;
  if (L.per_step) {
    hop_ids += (int64_t)step * L.n * L.n;
    deliv_ids += (int64_t)step * L.n * L.n;
  }
  uint32_t* cur = cur_bitmap(L.s[x], step);
  const uint32_t* ids = fwd_ids + (int64_t)pair * fwd_cap;
  __shared__ unsigned int per_src[NC_MAX_SHARDS];
  if (threadIdx.x < NC_MAX_SHARDS) per_src[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[k];
    atomicOr(cur + (id >> 5), 1u << (id & 31));
    const int o = owner_of(L, id);
    if (o >= 0) atomicAdd(&per_src[o], 1u);
  }
  __syncthreads();
  if (threadIdx.x < L.n && per_src[threadIdx.x])
    add64(deliv_ids + (int64_t)threadIdx.x * L.n + x, (long long)per_src[threadIdx.x]);
  if (threadIdx.x == 0 && blockIdx.x == 0) add64(hop_ids + (int64_t)b * L.n + x, (long long)cnt);
}

__global__ void k_reset_fwd(int32_t* fwd_count, int n2) {
  if ((int)threadIdx.x < n2) fwd_count[threadIdx.x] = 0;
}

}  // namespace

int ncx_load_local_kernels(void) {
  cudaFuncAttributes fa;
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_phase1));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_phase2));
  NC_CUDA_TRY(cudaFuncGetAttributes(&fa, k_reset_fwd));
  return NC_OK;
}

extern "C" int nc_exchange_local(const nc_shard_t* shards, int32_t n_shards, const uint16_t* dest_mask,
                                 const uint16_t* fwd_table, uint32_t* fwd_ids, int32_t* fwd_count,
                                 int64_t fwd_cap, long long* hop_ids, long long* deliv_ids,
                                 int32_t per_step, void* stream) {
  if (n_shards < 1 || n_shards > NC_MAX_SHARDS || !shards || !dest_mask || !hop_ids || !deliv_ids) {
    nc_set_error("nc_exchange_local: bad arguments (n_shards=%d)", n_shards);
    return NC_E_ARG;
  }
  if (n_shards == 1) return NC_OK;
  LocalSet L{};
  L.n = n_shards;
  L.per_step = per_step;
  L.step = shards[0].step;
  bool any_relay = false;
  int64_t max_cnt = 1;
  for (int h = 0; h < n_shards; ++h) {
    const nc_shard_t& s = shards[h];
    L.s[h] = LocalShard{s.bitmap0, s.bitmap1, s.bucket_ids, s.bucket_count, s.bucket_cap, s.local_base,
                        s.n_local};
    for (int k = 0; k < n_shards; ++k) {
      L.fwd[h][k] = fwd_table ? fwd_table[h * n_shards + k] : 0;
      any_relay |= L.fwd[h][k] != 0;
    }
    if (s.bucket_cap > max_cnt) max_cnt = s.bucket_cap;
  }
  if (any_relay && (!fwd_ids || !fwd_count || fwd_cap < 1)) {
    nc_set_error("nc_exchange_local: two-level routing needs forward buckets");
    return NC_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // Enough blocks per pair to cover a large bucket without knowing its count
  // on the host (the grid-stride loop handles any count).
  unsigned bx = (unsigned)((max_cnt + 255) / 256);
  if (bx > 16) bx = 16;
  dim3 grid(bx, (unsigned)(n_shards * n_shards));
  k_phase1<<<grid, 256, 0, st>>>(L, dest_mask, fwd_ids, fwd_count, fwd_cap, hop_ids, deliv_ids,
                                 shards[0].status);
  NC_LAUNCH_CHECK();
  if (any_relay) {
    k_phase2<<<grid, 256, 0, st>>>(L, fwd_ids, fwd_count, fwd_cap, hop_ids, deliv_ids);
    NC_LAUNCH_CHECK();
    k_reset_fwd<<<1, 256, 0, st>>>(fwd_count, n_shards * n_shards);
    NC_LAUNCH_CHECK();
  }
  return NC_OK;
}
