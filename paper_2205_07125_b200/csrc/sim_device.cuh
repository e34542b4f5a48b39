// Device building blocks of the per-step loop, shared by the per-kernel step
// functions (sim_kernels.cu) and the persistent engine (persistent.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <utility>
#include "nc_common.h"
#include "philox.cuh"
#include "jsell.cuh"

namespace ncdev {

#ifndef NC_UNROLL
#define NC_UNROLL 8
#endif
constexpr int kUnroll = NC_UNROLL;   // 16-byte slots in flight per lane
#ifndef NC_TAIL_UNROLL
#define NC_TAIL_UNROLL 4
#endif
constexpr int kTailUnroll = NC_TAIL_UNROLL;   // ... in the ragged tail of a J-SELL block
constexpr uint32_t kFull = 0xffffffffu;

#ifndef NC_STREAM_EVICT_FIRST
#define NC_STREAM_EVICT_FIRST 0
#endif
// Synapse stream loads: read once per step, so with NC_STREAM_EVICT_FIRST they are
// marked L2 evict-first (an L2 cache-policy operand; the constant policy folds into the
// load's uniform descriptor, no instruction) and leave L2 to what is reused: the
// bitmap tiles and, for huge shards, the partial sums in `acc`.
__device__ __forceinline__ uint64_t stream_policy() {
  uint64_t pol = 0;
#if NC_STREAM_EVICT_FIRST
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
#if NC_STREAM_EVICT_FIRST
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(stream_policy()));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#endif
  return r;
}

// Same with an immediate byte offset ([reg + imm] addressing: one instruction
// per load in an unrolled group instead of a 64-bit address computation each).
template <int kOff>
__device__ __forceinline__ uint4 ld_stream_at(const uint4* p) {
  uint4 r;
#if NC_STREAM_EVICT_FIRST
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4+%5], %6;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "n"(kOff), "l"(stream_policy()));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4+%5];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "n"(kOff));
#endif
  return r;
}

// Slots [0, n) of a group of kUnroll: slot u of this lane at q + 32u (512 B apart).
template <int... U>
__device__ __forceinline__ void load_group(uint4 (&e)[sizeof...(U)], const uint4* q, int n, uint4 padv,
                                           std::integer_sequence<int, U...>) {
  ((e[U] = (U < n) ? ld_stream_at<U * 512>(q) : padv), ...);
}

__device__ __forceinline__ uint4 ld_keep(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#ifndef NC_OFFSET_FMA
#define NC_OFFSET_FMA 0
#endif

// Weight units of one synapse field ((q << 19) | (id ^ 31), id relative to the
// staged tile) if its pre fired, still scaled by 2^19, added to acc.  The left
// funnel shift by the field's low 5 bits (31 - bit) moves the pre's spike bit to
// bit 31; the arithmetic shift spreads it into a mask and one LOP3 keeps the
// field's q bits under it: 3 ALU ops and no multiply per synapse.
__device__ __forceinline__ uint32_t field_term(uint32_t f, const uint32_t* __restrict__ bm, uint32_t acc) {
  // byte offset of the bitmap word, added to the (warp-uniform) buffer base by
  // the load itself: LDS [R + UR], 2 ALU ops per lookup
#if NC_OFFSET_FMA
  // f >> 3 as a high multiply: on the FMA pipe, next to the ALU-pipe-bound rest
  uint32_t f3;
  asm("mul.hi.u32 %0, %1, 536870912;" : "=r"(f3) : "r"(f));
#else
  const uint32_t f3 = f >> 3;
#endif
  const uint32_t word = *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(bm) +
                                                           (f3 & ((kFieldIdMask >> 5) << 2)));
  // the pre's bit to bit 31 (the field stores 31 - bit), sign-spread to a mask that
  // keeps the field's q bits: 3 ALU ops, no multiply; slot_term shifts the sum down once
  // (measured against bit * q as one IMAD per field: 0.543 vs 0.565 ms in a sustained
  // 1 000-step loop under sw_power_cap, 0.580 vs 0.601 ms at 8 tiles; against the bit by
  // mul.hi and the product by mad on the FMA pipe: 0.522 vs 0.528 ms)
  const int32_t fired = (int32_t)__funnelshift_l(word, word, f) >> 31;
  return acc + (f & (uint32_t)fired & (63u << 19));
}

// Weight units of the fired pres of one 16-byte slot (5 synapses), still scaled by 2^19
// and added to acc (a whole group of slots can be summed before one shift: <= 8 x 160
// units x 2^19 < 2^31).
__device__ __forceinline__ uint32_t slot_term_raw(uint4 e, const uint32_t* __restrict__ bm, uint32_t acc) {
  const Fields x = unpack_slot(e);
#pragma unroll
  for (int i = 0; i < kSlotEntries; ++i) acc = field_term(x.f[i], bm, acc);
  return acc;
}

// Weight units of the fired pres of one 16-byte slot (5 synapses).
__device__ __forceinline__ int32_t slot_term(uint4 e, const uint32_t* __restrict__ bm) {
  return (int32_t)(slot_term_raw(e, bm, 0u) >> 19);   // <= 5 x 32 weight units
}

// ---- 1-D TMA bulk copies into shared memory, completed on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// arrive (count 1) + expect `bytes` of transactions on the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16) by the TMA engine
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// order this thread's earlier generic-proxy shared accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA-engine prefetch of a contiguous range into L2 (no registers held).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Slots ahead of the loads for the L2 prefetch of the tiled kernel when its
// partial sums live in global memory (flags bit 0).
#ifndef NC_PF_DIST
#define NC_PF_DIST 8
#endif
constexpr int kPfTiled = NC_PF_DIST;

// Sum over one lane's row of a J-SELL block: returns sum_E - g * sum_I
// (weight units).  Slots past the lane's own length are not loaded (`pad`, the
// all-pad slot 0 -- id 0, q = 0 -- stands in: its lookups stay in the staged
// tile and add nothing).
// `part` of `nparts` (small shards split blocks so that every warp has several
// units to claim): part k takes the k-th run of whole load groups of the
// regular part; the last part also takes the ragged tail.
#ifndef NC_ROWSUM_LEAN
#define NC_ROWSUM_LEAN 1
#endif

// All kUnroll slots of a group (no padding: no predicates, no zeroed registers).
template <int... U>
__device__ __forceinline__ void load_group_full(uint4 (&e)[sizeof...(U)], const uint4* q,
                                                std::integer_sequence<int, U...>) {
  ((e[U] = ld_stream_at<U * 512>(q)), ...);
}

template <int kPfDist>
__device__ __forceinline__ int32_t sell_row_sum(const uint4* __restrict__ blk, uint32_t meta,
                                                const uint32_t* __restrict__ bm, int32_t g_inh, int lane,
                                                uint32_t pad, int part = 0, int nparts = 1) {
  const int emid = (int)(meta & 0xFFFFu);
  const int mine = (int)(meta >> 16);
  const int lo = __reduce_min_sync(kFull, (unsigned)mine);
  const int hi = __reduce_max_sync(kFull, (unsigned)mine);
  const int32_t wi = -g_inh;   // weight of an inhibitory slot
  int32_t acc = 0;
  const uint4* p = blk + lane;
  const uint4 padv = make_uint4(pad, pad, pad, pad);
  const int per = nparts == 1 ? lo : ((lo + nparts - 1) / nparts + kUnroll - 1) / kUnroll * kUnroll;
  const int ub = min(lo, part * per);
  const int ue = min(lo, ub + per);
#if NC_ROWSUM_LEAN
  // Slots below the warp's smallest emid are excitatory in every lane and slots at or above
  // its largest are inhibitory in every lane (warp-uniform tests): those add into accE /
  // accI and only the few slots in between pick a per-lane weight.  Whole groups load
  // without predicates.
  const int elo = (int)__reduce_min_sync(kFull, (unsigned)emid);
  const int ehi = (int)__reduce_max_sync(kFull, (unsigned)emid);
  int32_t accE = 0, accI = 0;
  auto add_slot = [&](const uint4& x, int slot) {
    const int32_t t = slot_term(x, bm);
    if (slot < elo) accE += t;
    else if (slot >= ehi) accI += t;
    else acc += t * (slot < emid ? 1 : wi);
  };
  for (int u0 = ub; u0 < ue; u0 += kUnroll) {
    if (kPfDist > 0 && lane == 0 && u0 + kPfDist < ue) {
      const int a = u0 + kPfDist;
      prefetch_l2(blk + a * 32, (uint32_t)min(kUnroll, ue - a) * 512u);
    }
    uint4 e[kUnroll];
    if (ue - u0 >= kUnroll) {   // warp-uniform
      load_group_full(e, p + u0 * 32, std::make_integer_sequence<int, kUnroll>{});
      if (u0 + kUnroll <= elo || u0 >= ehi) {   // warp-uniform: one sign for the whole group
        uint32_t g = 0u;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) g = slot_term_raw(e[u], bm, g);
        if (u0 >= ehi) accI += (int32_t)(g >> 19);
        else accE += (int32_t)(g >> 19);
      } else {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) add_slot(e[u], u0 + u);
      }
    } else {
      load_group(e, p + u0 * 32, ue - u0, padv, std::make_integer_sequence<int, kUnroll>{});
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (u0 + u >= ue) break;   // warp-uniform: no lookups for the pad of a partial group
        add_slot(e[u], u0 + u);
      }
    }
  }
  acc += accE + accI * wi;
#else
  // regular part: every lane has slots [0, lo)
  for (int u0 = ub; u0 < ue; u0 += kUnroll) {
    if (kPfDist > 0 && lane == 0 && u0 + kPfDist < ue) {
      const int a = u0 + kPfDist;
      prefetch_l2(blk + a * 32, (uint32_t)min(kUnroll, ue - a) * 512u);
    }
    uint4 e[kUnroll];
    load_group(e, p + u0 * 32, ue - u0, padv, std::make_integer_sequence<int, kUnroll>{});
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (u0 + u >= ue) break;   // warp-uniform: no lookups for the pad of a partial group
      acc += slot_term(e[u], bm) * (u0 + u < emid ? 1 : wi);
    }
  }
#endif
  if (part != nparts - 1) return acc;
  // ragged tail (short: rows of a block have near-equal lengths)
  int off = lo * 32;
  for (int u0 = lo; u0 < hi; u0 += kTailUnroll) {
    uint4 e[kTailUnroll];
#pragma unroll
    for (int u = 0; u < kTailUnroll; ++u) {
      const int pos = jsell_pos(u0 + u, mine, lane, off);
      e[u] = (u0 + u < mine) ? ld_stream(blk + pos) : padv;
    }
#pragma unroll
    for (int u = 0; u < kTailUnroll; ++u) {
      if (u0 + u >= hi) break;   // warp-uniform
      acc += slot_term(e[u], bm) * (u0 + u < emid ? 1 : wi);
    }
  }
  return acc;
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

__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Warp-aggregated append of the ids of lanes in `m` (whole warp calls); with
// `remote` (fused P2P send) each id also goes, tagged, to the same position of
// the peer's inbox message (xchg_device.cuh: word 1 + pos of the slot).
__device__ __forceinline__ void warp_append(uint32_t* ids, int32_t* count, int64_t cap, uint32_t m,
                                            uint32_t my_id, int lane, int32_t* status,
                                            unsigned long long* remote = nullptr, uint32_t tag = 0u) {
  if (m == 0) return;
  const int leader = __ffs(m) - 1;
  int32_t base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(kFull, base, leader);
  if ((m >> lane) & 1u) {
    const int64_t pos = (int64_t)base + __popc(m & ((1u << lane) - 1u));
    if (pos < cap) {
      ids[pos] = my_id;
      if (remote) st_relaxed_sys_u64(remote + 1 + pos, ((unsigned long long)tag << 32) | my_id);
    } else {
      atomicExch(status, 1);
    }
  }
}

// Phase-1 message slot of this shard in peer h's inbox (xchg_device.cuh slot_off).
__device__ __forceinline__ unsigned long long* xsend_slot(const nc_shard_t& sh, int h, int step) {
  return sh.xsend[h] + ((int64_t)((step & 1) * sh.n_shards + sh.shard)) * (sh.xsend_cap + 1);
}

// Fused P2P send, end of the step kernel: the last CTA writes every peer's
// tagged header (count; 0 = heartbeat) once all CTAs have bucketed their spikes.
// kSend = false compiles the send out (the launcher picks it from sh.xsend_on).
template <bool kSend>
__device__ __forceinline__ void xsend_headers(const nc_shard_t& sh, int step) {
  if (!kSend || !sh.xsend_on) return;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    // release: this CTA's bucket counts (ordered by the barrier) before the arrival;
    // acquire: the last arrival sees every CTA's counts
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(sh.work + 2) : "memory");
    last = prev + 1u == gridDim.x;
  }
  __syncthreads();
  const int h = threadIdx.x;
  if (last && h < sh.n_shards && h != sh.shard) {
    int64_t cnt = ((sh.xsend_mask >> h) & 1) ? *(volatile int32_t*)(sh.bucket_count + h) : 0;
    cnt = cnt < sh.xsend_cap ? cnt : sh.xsend_cap;
    st_relaxed_sys_u64(xsend_slot(sh, h, step), ((unsigned long long)(step + 1) << 32) | (uint32_t)cnt);
  }
}

// K2: bitmap word, raster, fired list and next-hop buckets for one 32-neuron tile.
template <bool kSend>
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
                  my_id, lane, sh.status, (kSend && sh.xsend_on) ? xsend_slot(sh, h, step) : nullptr,
                  (uint32_t)step + 1u);
    }
  }
  return fmask;
}

// Zero the words of `cur` outside this shard's local range (the exchange ORs
// remote spikes into them after the step kernel).
__device__ __forceinline__ void clear_remote(const nc_shard_t& sh, uint32_t* cur, int bid, int nblk) {
  const int lw0 = sh.local_base >> 5;
  const int lw1 = lw0 + sh.local_words;
  for (int w = bid * blockDim.x + threadIdx.x; w < sh.n_words; w += nblk * blockDim.x)
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
template <bool kSend>
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
  return emit_spikes<kSend>(sh, cur, slice, row, fired, lane, step);
}

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
#ifndef NC_LIF_UNROLL
#define NC_LIF_UNROLL 4
#endif
constexpr int kLifUnroll = NC_LIF_UNROLL;   // tiles per warp in flight in the LIF pass

template <int kWarps>
struct LifSmemT {
  unsigned int block_count;
  uint32_t fmask_s[kLifMaxTiles];
  int warp_cnt[kWarps][NC_MAX_SHARDS + 1];
  int cta_base[NC_MAX_SHARDS + 1];
};
using LifSmem = LifSmemT<kLifWarps>;

// One LIF phase of step `step` for block `bid` of `nblk` (blockDim = 32 *
// kWarps).  Block bid owns the 32-row tiles [bid*per, (bid+1)*per).  The
// synaptic input comes from acc (consumed and zeroed) or, when sacc is given,
// from shared memory indexed by the row's offset in the block's range.  The
// fired list is sh.fired_ids, or the step's spike list when sh.spk_ids is set.
template <int kWarps, int kU = kLifUnroll>
static __device__ void lif_phase(const nc_shard_t& sh, const nc_lif_params_t& p, int step, int bid, int nblk,
                                 LifSmemT<kWarps>& S, const int32_t* sacc = nullptr) {
  unsigned int& block_count = S.block_count;
  uint32_t* fmask_s = S.fmask_s;
  auto& warp_cnt = S.warp_cnt;
  int* cta_base = S.cta_base;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nq = sh.n_shards > 1 ? sh.n_shards : 0;      // buckets in use
  uint32_t* fired_ids = sh.spk_ids ? sh.spk_ids + (int64_t)(step & 1) * sh.spk_cap : sh.fired_ids;
  int32_t* fired_count = sh.spk_ids ? sh.spk_count + (step & 1) : sh.fired_count;
  const int64_t fired_cap = sh.spk_ids ? sh.spk_cap : sh.n_local;
  const int nb = nq + (fired_ids ? 1 : 0);               // + the fired list (slot nq)
  if (threadIdx.x == 0) block_count = 0;
  for (int k = threadIdx.x; k < kWarps * (NC_MAX_SHARDS + 1); k += blockDim.x)
    (&warp_cnt[0][0])[k] = 0;
  __syncthreads();
  uint32_t* cur = (step & 1) ? sh.bitmap1 : sh.bitmap0;
  clear_remote(sh, cur, bid, nblk);
  const int ntiles = (sh.n_local + 31) >> 5;
  const int per = (ntiles + nblk - 1) / nblk;
  const int t0 = bid * per, t1 = min(ntiles, t0 + per);
  uint32_t my_spikes = 0;
  // ---- pass A: update, spike masks, per-warp bucket counts.  kU tiles per
  // warp and iteration with every state load issued before the first use: one
  // memory round trip per kU tiles instead of two per tile (loads after
  // the acc store and the hop-mask load behind the update serialised; at config 3,
  // 10 M rows on one GPU, the LIF phase took 444 us of a 992 us step).
  for (int tile0 = t0 + warp; tile0 < t1; tile0 += kWarps * kU) {
    float v[kU], isyn[kU];
    uint8_t ref[kU];
    int32_t a[kU];
    uint32_t gid[kU], hm[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int tile = tile0 + u * kWarps;
      const int row = (tile << 5) + lane;
      const bool ok = tile < t1 && row < sh.n_local;
      v[u] = ok ? sh.v[row] : 0.0f;
      isyn[u] = ok ? sh.i_syn[row] : 0.0f;
      ref[u] = ok ? sh.refrac[row] : (uint8_t)0;
      a[u] = ok ? (sacc ? sacc[row - (t0 << 5)] : sh.acc[row]) : 0;
      gid[u] = ok ? sh.gid[row] : 0u;
      hm[u] = (ok && nq) ? (uint32_t)sh.hop_mask[row] : 0u;
    }
    if (!sacc) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int row = ((tile0 + u * kWarps) << 5) + lane;
        if (tile0 + u * kWarps < t1 && row < sh.n_local) sh.acc[row] = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int tile = tile0 + u * kWarps;
      if (tile >= t1) break;   // warp-uniform
      const int row = (tile << 5) + lane;
      bool fired = false;
      if (row < sh.n_local) {
        fired = lif_step(v[u], isyn[u], ref[u], a[u], gid[u], (uint32_t)step, p);
        sh.v[row] = v[u];
        sh.i_syn[row] = isyn[u];
        sh.refrac[row] = ref[u];
      }
      const uint32_t fmask = __ballot_sync(kFull, fired);
      if (lane == 0) {
        cur[(sh.local_base >> 5) + tile] = fmask;
        if (sh.raster != nullptr && step < sh.record_steps)
          sh.raster[(int64_t)step * sh.local_words + tile] = fmask;
        fmask_s[tile - t0] = fmask;
        my_spikes += __popc(fmask);
      }
      if (nb && fmask) {
        const uint32_t hmf = fired ? hm[u] : 0u;
        for (int h = 0; h < nb; ++h) {
          const uint32_t m = (h < nq) ? __ballot_sync(kFull, (hmf >> h) & 1u) : fmask;
          if (lane == 0) warp_cnt[warp][h] += __popc(m);
        }
      }
    }
  }
  __syncthreads();
  // ---- one global atomic per bucket per CTA; warp prefix inside the CTA
  if ((int)threadIdx.x < nb) {
    const int h = threadIdx.x;
    int total = 0;
    for (int w = 0; w < kWarps; ++w) {
      const int c = warp_cnt[w][h];
      warp_cnt[w][h] = total;  // exclusive prefix = the warp's base
      total += c;
    }
    int32_t* cnt = h < nq ? sh.bucket_count + h : fired_count;
    cta_base[h] = total ? atomicAdd(cnt, total) : 0;
  }
  __syncthreads();
  // ---- pass B: write ids (hop masks of kU tiles loaded together; none with
  // one shard, where only the fired list is written)
  if (nb) {
    for (int tile0 = t0 + warp; tile0 < t1; tile0 += kWarps * kU) {
      uint32_t fm[kU], hmu[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int tile = tile0 + u * kWarps;
        fm[u] = tile < t1 ? fmask_s[tile - t0] : 0u;
        hmu[u] = (nq && ((fm[u] >> lane) & 1u)) ? (uint32_t)sh.hop_mask[(tile << 5) + lane] : 0u;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
      const int tile = tile0 + u * kWarps;
      const uint32_t fmask = fm[u];
      if (!fmask) continue;   // warp-uniform
      const int row = (tile << 5) + lane;
      const uint32_t hm = hmu[u];
      const uint32_t my_id = (uint32_t)(sh.local_base + row);
      for (int h = 0; h < nb; ++h) {
        const uint32_t m = (h < nq) ? __ballot_sync(kFull, (hm >> h) & 1u) : fmask;
        if ((m >> lane) & 1u) {
          const int64_t pos = (int64_t)cta_base[h] + warp_cnt[warp][h] + __popc(m & ((1u << lane) - 1u));
          const int64_t cap = h < nq ? sh.bucket_cap : fired_cap;
          if (pos < cap) (h < nq ? sh.bucket_ids + (int64_t)h * sh.bucket_cap : fired_ids)[pos] = my_id;
          else atomicExch(sh.status, 1);
        }
        __syncwarp();
        if (lane == 0) warp_cnt[warp][h] += __popc(m);
        __syncwarp();
      }
      }
    }
  }
  add_spike_total(sh, my_spikes, &block_count);
}

// Event-driven delivery.  Blocks claim chunks of 32 bitmap words from a
// per-step counter (dynamic: the number of spikes per chunk varies); warp 0
// compacts the chunk's spikes into a shared list, then the warps take spikes
// round-robin and walk each pre neuron's push row with 8 loads in flight per
// lane, adding integer weights with red.global.add (exact, so order free).

// Fire-and-forget add.  Written out because inside the persistent kernel nvcc
// otherwise emits ATOMG (returns a value) for the same atomicAdd.
__device__ __forceinline__ void red_add(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kPushIds = 1024;

struct PushSmem {
  int next;
  int n;
  uint32_t ids[kPushIds];
};

// Entries [beg, end) of one push row (or window of it) into acc: 8 loads in flight per
// lane, integer reductions; `base` = first post row of the window.
__device__ __forceinline__ void push_segment(const nc_shard_t& sh, int32_t negg, int64_t beg, int64_t end,
                                             int base, int lane) {
  for (int64_t e0 = beg + lane; e0 < end; e0 += 256) {
    uint32_t x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = (e0 + 32 * u < end) ? __ldg(sh.push_syn + e0 + 32 * u) : 0u;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (e0 + 32 * u < end) {
        const int32_t q = (int32_t)((x[u] >> 26) & 31u) + 1;
        red_add(sh.acc + base + (x[u] & 0x03FFFFFFu), (x[u] >> 31) ? q * negg : q);
      }
    }
  }
}

// Event-driven delivery of the previous step's spikes.  Blocks claim 32-word
// chunks of the spike bitmap from a per-step counter (dynamic: the number of spikes
// per chunk varies); warp 0 compacts the chunk's spikes into a shared list, then the
// warps take spikes round-robin and walk each pre neuron's push row.  Warp 0 issues
// the NEXT chunk's claim and bitmap load right after compacting the current one, so
// both round trips overlap the rows instead of sitting between the two barriers of
// every chunk (at config 3 over 4 GPUs a chunk's ~11 spikes x 250 synapses are about
// one load round trip of work: the chunk overhead was ~80 of ~240 us per step).
// (Measured and dropped: warps claiming chunks on their own -- no barriers, but a
// chunk's spikes then run one after another in one warp, 2x slower at config 2 -- and
// a spike list filled by the LIF phase and the exchange: the same at 4 GPUs, 8 %
// slower on one.)  Windowed push (sh.push_windows > 1): window `window` only (its own
// claim counter work[4 + window]; the persistent engine runs the windows one after the
// other with a grid barrier in between), or every window of each row (window < 0,
// k_deliver_push).
static __device__ void push_phase(const nc_shard_t& sh, int32_t negg, int step, PushSmem& P, int window = -1) {
  const uint32_t* prev = ((step - 1) & 1) ? sh.bitmap1 : sh.bitmap0;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int n_chunks = (sh.n_words + 31) >> 5;
  const int W = sh.push_windows > 1 ? sh.push_windows : 1;
  uint32_t* claim = (W > 1 && window >= 0) ? sh.work + 4 + window : sh.work;
  // warp 0 holds the claimed chunk index and its bitmap words (one per lane)
  int c = 0;
  uint32_t bits = 0u;
  if (warp == 0) {
    if (lane == 0) c = (int)atomicAdd(claim, 1u);
    c = __shfl_sync(kFull, c, 0);
    const int w = (c << 5) + lane;
    bits = (c < n_chunks && w < sh.n_words) ? prev[w] : 0u;
  }
  for (;;) {
    if (warp == 0) {
      const int w = (c << 5) + lane;
      const int cnt = __popc(bits);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      int pos = incl - cnt;
      if (lane == 31) P.n = c < n_chunks ? incl : -1;
      uint32_t b = bits;
      while (b) {
        const int bit = __ffs(b) - 1;
        b &= b - 1;
        P.ids[pos++] = ((uint32_t)w << 5) + (uint32_t)bit;
      }
      // the next chunk's claim and bitmap words load while the rows below stream
      if (c < n_chunks) {
        int cn = 0;
        if (lane == 0) cn = (int)atomicAdd(claim, 1u);
        c = __shfl_sync(kFull, cn, 0);
        const int wn = (c << 5) + lane;
        bits = (c < n_chunks && wn < sh.n_words) ? prev[wn] : 0u;
      }
    }
    __syncthreads();
    const int n = P.n;
    if (n < 0) break;   // uniform: warp 0 found the chunks exhausted
    for (int i = warp; i < n; i += nwarps) {
      const uint32_t pre = P.ids[i];
      const int64_t r0 = sh.push_rowptr[pre];
      if (W == 1) {
        push_segment(sh, negg, r0, sh.push_rowptr[pre + 1], 0, lane);
        continue;
      }
      const uint16_t* wo = sh.push_winoff + (int64_t)pre * (W + 1);
      const int w0 = window >= 0 ? window : 0, w1 = window >= 0 ? window + 1 : W;
      for (int x = w0; x < w1; ++x)
        push_segment(sh, negg, r0 + wo[x], r0 + wo[x + 1], x * sh.push_window_rows, lane);
    }
    __syncthreads();
  }
}

}  // namespace ncdev
