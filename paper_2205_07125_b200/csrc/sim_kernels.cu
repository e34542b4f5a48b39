// Per-timestep hot loop of the spiking simulator on sm_100a.
//
//   K3 deliver (pull): integer segmented reduction over the post-sorted CSR,
//      one warp per row, 16-byte streaming loads, pre-spike bitmap staged in
//      shared memory; no float atomics -- the integer sum is order free, so
//      every reduction order gives the same int and hence the same fp32 input.
//   K1 LIF update: fp32 with explicit _rn intrinsics in the fixed order of
//      DESIGN.md section 3 (no FMA contraction), Philox drive.
//   K2 spike detect/bucket: __ballot_sync/__popc warp-aggregated appends of
//      fired internal ids into per-destination buckets (hop_mask from the
//      reference's RoutingTable, routing.py:184-231).
// nc_sim_step_fused runs K3+K1+K2 in one pass: a warp owns a tile of 32
// consecutive rows, reduces each row into the lane that owns that neuron and
// then updates the 32 neurons together, so the synaptic input never touches
// HBM.  The unfused entry points exist for the event-driven delivery variant.

#include <cuda_runtime.h>
#include <stdint.h>
#include "nc_common.h"
#include "philox.cuh"

namespace {

constexpr int kThreads = 1024;    // one CTA per SM in the smem-bitmap variant
constexpr int kUnroll = 6;        // uint4 loads in flight per lane per row
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_keep(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// Weight units of one packed entry (q << 26 | pre) if its pre fired, else 0.
// The funnel shift rotates the bitmap word by the low 5 bits of the entry
// (= pre & 31), so bit 0 is the pre's spike bit: 5 integer ops per synapse.
__device__ __forceinline__ int32_t entry_term(uint32_t e, const uint32_t* __restrict__ bm) {
  const uint32_t word = bm[(e & 0x03FFFFFFu) >> 5];
  const uint32_t rot = __funnelshift_r(word, word, e);
  return (rot & 1u) ? (int32_t)(e >> 26) : 0;
}

__device__ __forceinline__ int32_t quad_term(uint4 e, const uint32_t* __restrict__ bm) {
  return entry_term(e.x, bm) + entry_term(e.y, bm) + entry_term(e.z, bm) + entry_term(e.w, bm);
}

// Pull sum of one row by the whole warp: excitatory segment [beg, mid),
// inhibitory segment [mid, end) (uint4 units); returns sum_E - g * sum_I.
template <bool kStream>
__device__ __forceinline__ int32_t row_sum(const uint4* __restrict__ syn4, int64_t beg, int64_t mid, int64_t end,
                                           const uint32_t* __restrict__ bm, int32_t g_inh, int lane) {
  int32_t se = 0, si = 0;
  for (int64_t k0 = beg + lane; k0 < end; k0 += 32 * kUnroll) {
    uint4 e[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t k = k0 + 32 * u;
      e[u] = (k < end) ? (kStream ? ld_stream(syn4 + k) : ld_keep(syn4 + k))
                       : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t k = k0 + 32 * u;
      if (k < end) {
        const int32_t t = quad_term(e[u], bm);
        if (k < mid) se += t;
        else si += t;
      }
    }
  }
  return __reduce_add_sync(kFull, se - g_inh * si);
}

// Exact LIF step; returns true if the neuron fired.  Operation order is the
// contract shared with oracle/sim_oracle.c.
__device__ __forceinline__ bool lif_step(float& v, float& isyn, uint8_t& ref, int32_t acc,
                                         uint32_t gid, uint32_t step, const nc_lif_params_t& p) {
  uint32_t extc = 0;
  if (p.ext_lanes > 0) {
    nc_u32x4 c = {gid, step, NC_TAG_DRIVE, 0u};
    nc_u32x4 r = nc_philox4x32_10(c, (uint32_t)p.seed, (uint32_t)(p.seed >> 32));
    extc = (r.x < p.ext_threshold);
    if (p.ext_lanes > 1) extc += (r.y < p.ext_threshold);
    if (p.ext_lanes > 2) extc += (r.z < p.ext_threshold);
    if (p.ext_lanes > 3) extc += (r.w < p.ext_threshold);
  }
  const float syn = __int2float_rn(acc);
  const float ext = __uint2float_rn(extc);
  const float i1 = __fadd_rn(__fmul_rn(isyn, p.alpha_i), __fmul_rn(syn, p.w_unit));
  const float inew = __fadd_rn(i1, __fmul_rn(ext, p.w_ext));
  isyn = inew;
  if (ref > 0) {
    ref = (uint8_t)(ref - 1);
    v = p.v_reset;
    return false;
  }
  const float d = __fsub_rn(v, p.v_rest);
  const float vn = __fadd_rn(__fadd_rn(p.v_rest, __fmul_rn(d, p.alpha_v)), __fmul_rn(inew, p.beta));
  if (vn >= p.v_th) {
    v = p.v_reset;
    ref = (uint8_t)p.t_ref;
    return true;
  }
  v = vn;
  return false;
}

// Warp-aggregated append of the ids of lanes in `m` (whole warp calls).
__device__ __forceinline__ void warp_append(uint32_t* ids, int32_t* count, int64_t cap, uint32_t m,
                                            uint32_t my_id, int lane, int32_t* status) {
  if (m == 0) return;
  const int leader = __ffs(m) - 1;
  int32_t base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if ((m >> lane) & 1u) {
    const int64_t pos = (int64_t)base + __popc(m & ((1u << lane) - 1u));
    if (pos < cap) ids[pos] = my_id;
    else atomicExch(status, 1);
  }
}

// K2: bitmap word, raster, fired list and next-hop buckets for one 32-neuron tile.
__device__ __forceinline__ uint32_t emit_spikes(const nc_shard_t& sh, uint32_t* cur, int tile, int row,
                                                bool fired, int lane, int step) {
  const uint32_t fmask = __ballot_sync(kFull, fired);
  if (lane == 0) {
    cur[(sh.local_base >> 5) + tile] = fmask;
    if (sh.raster != nullptr && step < sh.record_steps)
      sh.raster[(int64_t)step * sh.local_words + tile] = fmask;
  }
  if (fmask == 0) return 0;
  const uint32_t my_id = (uint32_t)(sh.local_base + row);
  if (sh.fired_ids != nullptr)
    warp_append(sh.fired_ids, sh.fired_count, sh.n_local, fmask, my_id, lane, sh.status);
  if (sh.n_shards > 1) {
    const uint32_t hm = fired ? (uint32_t)sh.hop_mask[row] : 0u;
    uint32_t pending = __reduce_or_sync(kFull, hm);
    while (pending) {
      const int h = __ffs(pending) - 1;
      pending &= pending - 1;
      const uint32_t m = __ballot_sync(kFull, (hm >> h) & 1u);
      warp_append(sh.bucket_ids + (int64_t)h * sh.bucket_cap, sh.bucket_count + h, sh.bucket_cap, m,
                  my_id, lane, sh.status);
    }
  }
  return fmask;
}

// Zero the words of `cur` outside this shard's local range (the exchange ORs
// remote spikes into them after the step kernel).
__device__ __forceinline__ void clear_remote(const nc_shard_t& sh, uint32_t* cur) {
  const int lw0 = sh.local_base >> 5;
  const int lw1 = lw0 + sh.local_words;
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < sh.n_words; w += gridDim.x * blockDim.x)
    if (w < lw0 || w >= lw1) cur[w] = 0u;
}

__device__ __forceinline__ void add_spike_total(const nc_shard_t& sh, uint32_t local_count,
                                                unsigned int* block_count) {
  if (local_count) atomicAdd(block_count, local_count);
  __syncthreads();
  if (threadIdx.x == 0 && *block_count && sh.spike_total)
    atomicAdd(sh.spike_total, (unsigned long long)*block_count);
}

template <bool kSmemBitmap>
__global__ void __launch_bounds__(kThreads, 1)
k_step_fused(const nc_shard_t sh, const nc_lif_params_t p) {
  extern __shared__ uint4 smem4[];
  __shared__ unsigned int block_count;
  const int step = *sh.step;
  const uint32_t* prev = ((step - 1) & 1) ? sh.bitmap1 : sh.bitmap0;
  uint32_t* cur = (step & 1) ? sh.bitmap1 : sh.bitmap0;
  if (threadIdx.x == 0) block_count = 0;
  if (kSmemBitmap) {
    const uint4* src = reinterpret_cast<const uint4*>(prev);
    const int n4 = (sh.n_words + 3) >> 2;
    for (int k = threadIdx.x; k < n4; k += blockDim.x) smem4[k] = ld_keep(src + k);
  }
  __syncthreads();
  const uint32_t* bm = kSmemBitmap ? reinterpret_cast<const uint32_t*>(smem4) : prev;
  clear_remote(sh, cur);

  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int ntiles = (sh.n_local + 31) >> 5;
  const int32_t g_inh = p.g_inh;
  const uint4* syn4 = reinterpret_cast<const uint4*>(sh.syn);
  uint32_t my_spikes = 0;

  for (int tile = blockIdx.x * wpb + (threadIdx.x >> 5); tile < ntiles; tile += gridDim.x * wpb) {
    const int row0 = tile << 5;
    const int nrows = min(32, sh.n_local - row0);
    // lane l holds the E and I segment starts of row row0+l; lane nrows the end
    const int64_t rpe = sh.rowptr4[2 * (row0 + min(lane, nrows))];
    const int64_t rpi = lane < nrows ? sh.rowptr4[2 * (row0 + lane) + 1] : rpe;
    const int64_t rp_last = sh.rowptr4[2 * (row0 + nrows)];
    int32_t my_acc = 0;
    for (int r = 0; r < nrows; ++r) {
      const int64_t beg = __shfl_sync(kFull, rpe, r);
      const int64_t mid = __shfl_sync(kFull, rpi, r);
      const int64_t nxt = __shfl_sync(kFull, rpe, r + 1 < 32 ? r + 1 : 31);
      const int64_t end = (r + 1 < nrows) ? nxt : rp_last;
      const int32_t s = row_sum<true>(syn4, beg, mid, end, bm, g_inh, lane);
      if (lane == r) my_acc = s;
    }
    const int row = row0 + lane;
    bool fired = false;
    if (lane < nrows) {
      float v = sh.v[row];
      float isyn = sh.i_syn[row];
      uint8_t ref = sh.refrac[row];
      fired = lif_step(v, isyn, ref, my_acc, sh.gid[row], (uint32_t)step, p);
      sh.v[row] = v;
      sh.i_syn[row] = isyn;
      sh.refrac[row] = ref;
    }
    const uint32_t fm = emit_spikes(sh, cur, tile, row, fired, lane, step);
    if (lane == 0) my_spikes += __popc(fm);
  }
  add_spike_total(sh, my_spikes, &block_count);
}

// K3 alone: acc[r] = pull sum.
template <bool kSmemBitmap>
__global__ void __launch_bounds__(kThreads, 1) k_deliver_pull(const nc_shard_t sh, int32_t g_inh) {
  extern __shared__ uint4 smem4[];
  const int step = *sh.step;
  const uint32_t* prev = ((step - 1) & 1) ? sh.bitmap1 : sh.bitmap0;
  if (kSmemBitmap) {
    const uint4* src = reinterpret_cast<const uint4*>(prev);
    const int n4 = (sh.n_words + 3) >> 2;
    for (int k = threadIdx.x; k < n4; k += blockDim.x) smem4[k] = ld_keep(src + k);
    __syncthreads();
  }
  const uint32_t* bm = kSmemBitmap ? reinterpret_cast<const uint32_t*>(smem4) : prev;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const uint4* syn4 = reinterpret_cast<const uint4*>(sh.syn);
  for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < sh.n_local; row += gridDim.x * wpb) {
    const int32_t s = row_sum<true>(syn4, sh.rowptr4[2 * row], sh.rowptr4[2 * row + 1], sh.rowptr4[2 * row + 2],
                                    bm, g_inh, lane);
    if (lane == 0) sh.acc[row] = s;
  }
}

// K1+K2 alone: consumes and zeroes acc.
__global__ void __launch_bounds__(256) k_lif_update(const nc_shard_t sh, const nc_lif_params_t p) {
  __shared__ unsigned int block_count;
  if (threadIdx.x == 0) block_count = 0;
  __syncthreads();
  const int step = *sh.step;
  uint32_t* cur = (step & 1) ? sh.bitmap1 : sh.bitmap0;
  clear_remote(sh, cur);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int ntiles = (sh.n_local + 31) >> 5;
  uint32_t my_spikes = 0;
  for (int tile = blockIdx.x * wpb + (threadIdx.x >> 5); tile < ntiles; tile += gridDim.x * wpb) {
    const int row = (tile << 5) + lane;
    bool fired = false;
    if (row < sh.n_local) {
      float v = sh.v[row];
      float isyn = sh.i_syn[row];
      uint8_t ref = sh.refrac[row];
      const int32_t a = sh.acc[row];
      sh.acc[row] = 0;
      fired = lif_step(v, isyn, ref, a, sh.gid[row], (uint32_t)step, p);
      sh.v[row] = v;
      sh.i_syn[row] = isyn;
      sh.refrac[row] = ref;
    }
    const uint32_t fm = emit_spikes(sh, cur, tile, row, fired, lane, step);
    if (lane == 0) my_spikes += __popc(fm);
  }
  add_spike_total(sh, my_spikes, &block_count);
}

// Event-driven delivery: scan the previous step's spike bitmap one warp per
// word; for every set bit the warp walks that pre neuron's push-CSR row and
// adds the integer weights into acc with red.global.add (exact, so order free).
__global__ void __launch_bounds__(256) k_deliver_push(const nc_shard_t sh, int32_t negg) {
  const int step = *sh.step;
  const uint32_t* prev = ((step - 1) & 1) ? sh.bitmap1 : sh.bitmap0;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t w = blockIdx.x * wpb + (threadIdx.x >> 5); w < sh.n_words; w += gridDim.x * wpb) {
    uint32_t bits = prev[w];  // same value in every lane (broadcast load)
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t pre = (w << 5) + b;
      const int64_t beg = sh.push_rowptr[pre], end = sh.push_rowptr[pre + 1];
      for (int64_t e = beg + lane; e < end; e += 32) {
        const uint32_t x = sh.push_syn[e];
        const int32_t q = (int32_t)((x >> 26) & 31u) + 1;
        atomicAdd(sh.acc + (x & 0x03FFFFFFu), (x >> 31) ? q * negg : q);
      }
    }
  }
}

__global__ void k_end_step(const nc_shard_t sh) {
  const int t = threadIdx.x;
  if (t < sh.n_shards) sh.bucket_count[t] = 0;
  if (t == 0) {
    if (sh.fired_count) *sh.fired_count = 0;
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

constexpr size_t kMaxSmemBitmapBytes = 200 * 1024;

size_t bitmap_smem_bytes(const nc_shard_t& sh) { return (size_t)((sh.n_words + 3) >> 2) * 16; }

int check_shard(const nc_shard_t* sh) {
  if (!sh || sh->n_local < 0 || sh->n_words < 1 || (sh->local_base & 31) || !sh->step ||
      !sh->status || !sh->bitmap0 || !sh->bitmap1) {
    nc_set_error("invalid nc_shard_t");
    return NC_E_ARG;
  }
  return NC_OK;
}

}  // namespace

// Set kernel attributes once, outside any stream capture.
extern "C" int nc_sim_prepare(void) {
  (void)num_sms();
  NC_CUDA_TRY(cudaFuncSetAttribute(k_step_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kMaxSmemBitmapBytes));
  NC_CUDA_TRY(cudaFuncSetAttribute(k_deliver_pull<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kMaxSmemBitmapBytes));
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
  const size_t smem = bitmap_smem_bytes(*sh);
  const int grid = num_sms();
  if (smem <= kMaxSmemBitmapBytes) {
    if (!g_prepared) {
      if (int e = nc_sim_prepare()) return e;
    }
    k_step_fused<true><<<grid, kThreads, smem, (cudaStream_t)stream>>>(*sh, *p);
  } else {
    k_step_fused<false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(*sh, *p);
  }
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_deliver_pull(const nc_shard_t* sh, int32_t g_inh, void* stream) {
  if (int e = check_shard(sh)) return e;
  const size_t smem = bitmap_smem_bytes(*sh);
  const int grid = num_sms();
  if (smem <= kMaxSmemBitmapBytes) {
    if (!g_prepared) {
      if (int e = nc_sim_prepare()) return e;
    }
    k_deliver_pull<true><<<grid, kThreads, smem, (cudaStream_t)stream>>>(*sh, g_inh);
  } else {
    k_deliver_pull<false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(*sh, g_inh);
  }
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_deliver_push(const nc_shard_t* sh, int32_t g_inh, void* stream) {
  if (int e = check_shard(sh)) return e;
  if (!sh->push_rowptr || !sh->push_syn || !sh->acc) {
    nc_set_error("nc_sim_deliver_push: shard has no push CSR / acc");
    return NC_E_ARG;
  }
  int64_t grid = (sh->n_words + 7) / 8;
  if (grid > 16 * num_sms()) grid = 16 * num_sms();
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
  const int tiles = (sh->n_local + 31) / 32;
  int grid = (tiles + 7) / 8;
  grid = grid < 1 ? 1 : (grid > 16 * num_sms() ? 16 * num_sms() : grid);
  k_lif_update<<<grid, 256, 0, (cudaStream_t)stream>>>(*sh, *p);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_end_step(const nc_shard_t* sh, void* stream) {
  if (int e = check_shard(sh)) return e;
  k_end_step<<<1, 32, 0, (cudaStream_t)stream>>>(*sh);
  NC_LAUNCH_CHECK();
  return NC_OK;
}
