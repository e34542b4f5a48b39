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
#include "nc_common.h"
#include "philox.cuh"

namespace {

constexpr int kThreads = 1024;    // one CTA per SM in the smem-bitmap variant
constexpr int kUnroll = 8;        // 16-byte slots in flight per lane
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

// One lane's row in one SELL-32 block: block slots [0, len) at blk + u*32 + lane;
// this row uses meta >> 16 of them, the first (meta & 0xFFFF) excitatory.
// Slots past the row's own length are not loaded (`pad` stands in: the block's
// pad entry, first id of its tile with q = 0, so its lookup stays in the
// staged tile and adds nothing).  Returns sum_E - g * sum_I (weight units).
__device__ __forceinline__ int32_t sell_row_sum(const uint4* __restrict__ blk, int len, uint32_t meta,
                                                const uint32_t* __restrict__ bm, int32_t g_inh, int lane,
                                                uint32_t pad) {
  const int emid = (int)(meta & 0xFFFFu);
  const int mine = (int)(meta >> 16);
  int32_t se = 0, si = 0;
  const uint4* p = blk + lane;
  const uint4 padv = make_uint4(pad, pad, pad, pad);
  for (int u0 = 0; u0 < len; u0 += kUnroll) {
    uint4 e[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) e[u] = (u0 + u < mine) ? ld_stream(p + (u0 + u) * 32) : padv;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int32_t t = quad_term(e[u], bm);
      if (u0 + u < emid) se += t;
      else si += t;
    }
  }
  return se - g_inh * si;
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

// LIF + spike emission for the 32 rows of one slice (lane = row).
__device__ __forceinline__ uint32_t update_slice(const nc_shard_t& sh, const nc_lif_params_t& p, uint32_t* cur,
                                                 int slice, int lane, int32_t acc, int step) {
  const int row = (slice << 5) + lane;
  bool fired = false;
  if (row < sh.n_local) {
    float v = sh.v[row];
    float isyn = sh.i_syn[row];
    uint8_t ref = sh.refrac[row];
    fired = lif_step(v, isyn, ref, acc, sh.gid[row], (uint32_t)step, p);
    sh.v[row] = v;
    sh.i_syn[row] = isyn;
    sh.refrac[row] = ref;
  }
  return emit_spikes(sh, cur, slice, row, fired, lane, step);
}

// K3 (+K1+K2 when kLif).  kTiled: the bitmap does not fit in shared memory;
// every CTA owns a fixed range of slices, loops over the bitmap tiles and
// keeps the per-row partial sums in shared memory behind the tile.
template <bool kTiled, bool kLif>
__global__ void __launch_bounds__(kThreads, 1)
k_step_fused(const nc_shard_t sh, const nc_lif_params_t p) {
  extern __shared__ uint4 smem4[];
  __shared__ unsigned int block_count;
  const int step = *sh.step;
  const uint32_t* prev = ((step - 1) & 1) ? sh.bitmap1 : sh.bitmap0;
  uint32_t* cur = (step & 1) ? sh.bitmap1 : sh.bitmap0;
  uint32_t* sbm = reinterpret_cast<uint32_t*>(smem4);
  if (threadIdx.x == 0) block_count = 0;
  if (kLif) clear_remote(sh, cur);
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
    for (int slice = blockIdx.x * wpb + warp; slice < n_slices; slice += gridDim.x * wpb) {
      const int row = (slice << 5) + lane;
      const int64_t b0 = sh.slice_ptr[slice];
      const int len = (int)((sh.slice_ptr[slice + 1] - b0) >> 5);
      const uint32_t meta = row < sh.n_local ? sh.row_meta[row] : 0u;
      const int32_t acc = sell_row_sum(syn4 + b0, len, meta, sbm, g_inh, lane, 0u);
      if (kLif) {
        const uint32_t fm = update_slice(sh, p, cur, slice, lane, acc, step);
        if (lane == 0) my_spikes += __popc(fm);
      } else if (row < sh.n_local) {
        sh.acc[row] = acc;
      }
    }
  } else {
    const int T = sh.n_tiles, TW = sh.tile_words;
    const int per = (n_slices + gridDim.x - 1) / gridDim.x;
    const int s0 = blockIdx.x * per;
    const int s1 = min(n_slices, s0 + per);
    // partial sums per row: shared memory behind the tile, or the acc array when
    // the CTA's rows do not fit next to a useful tile (flags bit 0)
    int32_t* part = (sh.flags & 1) ? sh.acc + (int64_t)s0 * 32 : reinterpret_cast<int32_t*>(sbm + TW);
    const int n_part = (sh.flags & 1) ? min(per * 32, sh.n_local - s0 * 32) : per * 32;
    for (int k = threadIdx.x; k < n_part; k += blockDim.x) part[k] = 0;
    __shared__ int next_slice[2];
    if (threadIdx.x == 0) next_slice[0] = next_slice[1] = s0;
    for (int t = 0; t < T; ++t) {
      __syncthreads();
      const int w0 = t * TW;
      const int nw = min(TW, sh.n_words - w0);
      const uint4* src = reinterpret_cast<const uint4*>(prev + w0);
      for (int k = threadIdx.x; k < (nw + 3) >> 2; k += blockDim.x) smem4[k] = ld_keep(src + k);
      if (threadIdx.x == 0) next_slice[(t + 1) & 1] = s0;  // counter of the next tile
      __syncthreads();
      // tile-relative view: bm[global word] hits the staged copy
      const uint32_t* bm = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(sbm) -
                                                             (uintptr_t)w0 * 4u);
      // warps claim slices dynamically so the per-tile barrier waits for at most one slice
      for (;;) {
        int slice = 0;
        if (lane == 0) slice = atomicAdd(&next_slice[t & 1], 1);
        slice = __shfl_sync(kFull, slice, 0);
        if (slice >= s1) break;
        const int row = (slice << 5) + lane;
        const int64_t b0 = sh.slice_ptr[(int64_t)slice * T + t];
        const int len = (int)((sh.slice_ptr[(int64_t)slice * T + t + 1] - b0) >> 5);
        const uint32_t meta = row < sh.n_local ? sh.row_meta[(int64_t)row * T + t] : 0u;
        part[(slice - s0) * 32 + lane] += sell_row_sum(syn4 + b0, len, meta, bm, g_inh, lane, (uint32_t)w0 * 32u);
      }
    }
    __syncthreads();
    for (int slice = s0 + warp; slice < s1; slice += wpb) {
      const int row = (slice << 5) + lane;
      const int32_t acc = part[(slice - s0) * 32 + lane];
      if (kLif) {
        const uint32_t fm = update_slice(sh, p, cur, slice, lane, acc, step);
        if (lane == 0) my_spikes += __popc(fm);
      } else if (row < sh.n_local) {
        sh.acc[row] = acc;
      }
    }
  }
  if (kLif) add_spike_total(sh, my_spikes, &block_count);
}

// K1+K2 alone: consumes and zeroes acc.
// K1+K2 alone (consumes and zeroes acc).  Every CTA owns a contiguous range of
// 32-neuron tiles and appends to the buckets with ONE global atomic per bucket
// for the whole step: pass A runs the LIF update, stores each tile's spike mask
// in shared memory and counts per warp and bucket; the CTA then claims its
// ranges; pass B recomputes the per-bucket ballots from the stored masks and the
// static hop masks and writes the ids.  (Same-address atomics serialise in L2:
// one per warp per bucket cost more than the update itself.)
constexpr int kLifThreads = 256;
constexpr int kLifWarps = kLifThreads / 32;
constexpr int kLifMaxTiles = 2048;   // tiles per CTA (fmask storage: 8 KB)

__global__ void __launch_bounds__(kLifThreads) k_lif_update(const nc_shard_t sh, const nc_lif_params_t p) {
  __shared__ unsigned int block_count;
  __shared__ uint32_t fmask_s[kLifMaxTiles];
  __shared__ int warp_cnt[kLifWarps][NC_MAX_SHARDS + 1];
  __shared__ int cta_base[NC_MAX_SHARDS + 1];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nq = sh.n_shards > 1 ? sh.n_shards : 0;      // buckets in use
  const int nb = nq + (sh.fired_ids ? 1 : 0);            // + the fired list (slot nq)
  if (threadIdx.x == 0) block_count = 0;
  for (int k = threadIdx.x; k < kLifWarps * (NC_MAX_SHARDS + 1); k += blockDim.x)
    (&warp_cnt[0][0])[k] = 0;
  __syncthreads();
  const int step = *sh.step;
  uint32_t* cur = (step & 1) ? sh.bitmap1 : sh.bitmap0;
  clear_remote(sh, cur);
  const int ntiles = (sh.n_local + 31) >> 5;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  uint32_t my_spikes = 0;
  // ---- pass A: update, spike masks, per-warp bucket counts
  for (int tile = t0 + warp; tile < t1; tile += kLifWarps) {
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
    const uint32_t fmask = __ballot_sync(kFull, fired);
    if (lane == 0) {
      cur[(sh.local_base >> 5) + tile] = fmask;
      if (sh.raster != nullptr && step < sh.record_steps) sh.raster[(int64_t)step * sh.local_words + tile] = fmask;
      fmask_s[tile - t0] = fmask;
      my_spikes += __popc(fmask);
    }
    if (nb && fmask) {
      const uint32_t hm = fired ? (uint32_t)sh.hop_mask[row] : 0u;
      for (int h = 0; h < nb; ++h) {
        const uint32_t m = (h < nq) ? __ballot_sync(kFull, (hm >> h) & 1u) : fmask;
        if (lane == 0) warp_cnt[warp][h] += __popc(m);
      }
    }
  }
  __syncthreads();
  // ---- one global atomic per bucket per CTA; warp prefix inside the CTA
  if ((int)threadIdx.x < nb) {
    const int h = threadIdx.x;
    int total = 0;
    for (int w = 0; w < kLifWarps; ++w) {
      const int c = warp_cnt[w][h];
      warp_cnt[w][h] = total;  // exclusive prefix = the warp's base
      total += c;
    }
    int32_t* cnt = h < nq ? sh.bucket_count + h : sh.fired_count;
    cta_base[h] = total ? atomicAdd(cnt, total) : 0;
  }
  __syncthreads();
  // ---- pass B: write ids
  if (nb) {
    for (int tile = t0 + warp; tile < t1; tile += kLifWarps) {
      const uint32_t fmask = fmask_s[tile - t0];
      if (!fmask) continue;
      const int row = (tile << 5) + lane;
      const bool fired = (fmask >> lane) & 1u;
      const uint32_t hm = fired ? (uint32_t)sh.hop_mask[row] : 0u;
      const uint32_t my_id = (uint32_t)(sh.local_base + row);
      for (int h = 0; h < nb; ++h) {
        const uint32_t m = (h < nq) ? __ballot_sync(kFull, (hm >> h) & 1u) : fmask;
        if ((m >> lane) & 1u) {
          const int64_t pos = (int64_t)cta_base[h] + warp_cnt[warp][h] + __popc(m & ((1u << lane) - 1u));
          const int64_t cap = h < nq ? sh.bucket_cap : sh.n_local;
          if (pos < cap) (h < nq ? sh.bucket_ids + (int64_t)h * sh.bucket_cap : sh.fired_ids)[pos] = my_id;
          else atomicExch(sh.status, 1);
        }
        __syncwarp();
        if (lane == 0) warp_cnt[warp][h] += __popc(m);
        __syncwarp();
      }
    }
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
      // 4 independent loads in flight per lane, then 4 fire-and-forget reductions
      for (int64_t e0 = beg + lane; e0 < end; e0 += 128) {
        uint32_t x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = (e0 + 32 * u < end) ? __ldg(sh.push_syn + e0 + 32 * u) : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (e0 + 32 * u < end) {
            const int32_t q = (int32_t)((x[u] >> 26) & 31u) + 1;
            atomicAdd(sh.acc + (x[u] & 0x03FFFFFFu), (x[u] >> 31) ? q * negg : q);
          }
        }
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

int g_max_dyn_smem = 0;   // opt-in limit minus the kernels' static shared memory

// dynamic shared memory of the step kernel: whole bitmap, or one tile plus
// the per-row partial sums of the CTA's slice range
size_t step_smem_bytes(const nc_shard_t& sh, int grid) {
  if (sh.n_tiles <= 1) return (size_t)((sh.n_words + 3) >> 2) * 16;
  if (sh.flags & 1) return (size_t)sh.tile_words * 4;
  const int n_slices = (sh.n_local + 31) >> 5;
  const int per = (n_slices + grid - 1) / grid;
  return (size_t)sh.tile_words * 4 + (size_t)per * 32 * 4;
}

template <bool kLif>
int launch_step(const nc_shard_t& sh, const nc_lif_params_t& p, cudaStream_t st) {
  const int grid = num_sms();
  const size_t smem = step_smem_bytes(sh, grid);
  if (smem > (size_t)g_max_dyn_smem) {
    nc_set_error("step kernel needs %zu B of shared memory (tile_words=%d): re-tile the network", smem,
                 sh.tile_words);
    return NC_E_ARG;
  }
  if (sh.n_tiles <= 1)
    k_step_fused<false, kLif><<<grid, kThreads, smem, st>>>(sh, p);
  else
    k_step_fused<true, kLif><<<grid, kThreads, smem, st>>>(sh, p);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

int check_shard(const nc_shard_t* sh) {
  if (!sh || sh->n_local < 0 || sh->n_words < 1 || (sh->local_base & 31) || !sh->step ||
      !sh->status || !sh->bitmap0 || !sh->bitmap1 || sh->n_tiles < 1 ||
      (sh->n_tiles > 1 && (sh->tile_words < 4 || (sh->tile_words & 3) ||
                           (int64_t)sh->tile_words * sh->n_tiles < sh->n_words)) ||
      ((sh->flags & 1) && !sh->acc)) {
    nc_set_error("invalid nc_shard_t");
    return NC_E_ARG;
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
  // contiguous tile ranges, ~2 CTAs per SM (more if a range would exceed the
  // shared spike-mask storage): one global atomic per bucket per CTA
  const int tiles = (sh->n_local + 31) / 32;
  int grid = 2 * num_sms();
  if ((tiles + grid - 1) / grid > kLifMaxTiles) grid = (tiles + kLifMaxTiles - 1) / kLifMaxTiles;
  if (grid > tiles) grid = tiles > 0 ? tiles : 1;
  k_lif_update<<<grid, kLifThreads, 0, (cudaStream_t)stream>>>(*sh, *p);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sim_end_step(const nc_shard_t* sh, void* stream) {
  if (int e = check_shard(sh)) return e;
  k_end_step<<<1, 32, 0, (cudaStream_t)stream>>>(*sh);
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
    const int row = (slice << 5) + lane;
    const int64_t b0 = sh.slice_ptr[blk];
    const uint32_t meta = row < sh.n_local ? sh.row_meta[(int64_t)row * T + t] : 0u;
    const int emid = (int)(meta & 0xFFFFu), mine = (int)(meta >> 16);
    for (int u = 0; u < mine; ++u) {
      const uint4 e4 = syn4[b0 + (int64_t)u * 32 + lane];
      const uint32_t es[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t e = es[c];
        const uint32_t q = e >> 26;
        if (q == 0) continue;
        const uint32_t pre = e & 0x03FFFFFFu;
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
