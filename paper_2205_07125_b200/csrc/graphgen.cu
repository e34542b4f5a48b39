// Device network build: counter-based SBM generator -> pull CSR.
//
// Distributions follow neurocomm generate_synthetic (model.py:199-253):
// contiguous near-equal communities (community_sizes, model.py:146-151), each
// intra-community pair an edge with probability p_in and p ~ U(intra range),
// each inter-community pair with p_out and p ~ U(inter range).  The reference
// draws from one sequential PCG64 stream, which no GPU can replay; here every
// (row i, block b) owns an independent Philox stream, so all shards generate
// the identical global graph in parallel and keep only their own rows.
//
// Row i enumerates its upper neighbours j > i block by block with geometric
// skipping (the same sampler as model.py:154-180, in fp64 log1p).  Each edge
// (i, j) is one synapse in each direction: row i gets pre j, row j gets pre i.
// Pass 1 counts per-segment lengths (a post row has an excitatory-pre and an
// inhibitory-pre segment; upper parts directly, lower parts with integer
// atomics); the host scans the padded lengths into rowptr4; pass 2 regenerates
// the same edges and writes them: segment layout [lower part | upper part | pad].
// The order inside the lower part depends on atomic arrival, which is harmless:
// delivery sums integers, so any order gives the same input.

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include "nc_common.h"
#include "jsell.cuh"
#include "philox.cuh"

#include "sbm_gen.cuh"

namespace {
using namespace ncgen;

__device__ __forceinline__ uint32_t is_inh(const nc_graphgen_t& g, int64_t gid) {
  return (g.inh_every > 0 && (gid % g.inh_every) == g.inh_every - 1) ? 1u : 0u;
}

// First internal id of the bitmap tile holding `id` (entries store ids relative to it).
__device__ __forceinline__ uint32_t tile_base(uint32_t id, int32_t TW) {
  return (id >> 5) / (uint32_t)TW * (uint32_t)TW * 32u;
}

__device__ __forceinline__ uint32_t pack(uint32_t pre_internal, uint32_t q) {
  return (q << 26) | pre_internal;
}

__device__ __forceinline__ int64_t seg_index(int64_t row, int32_t T, int32_t TW, uint32_t pre_internal,
                                             uint32_t inh) {
  return (row * T + (int64_t)((pre_internal >> 5) / (uint32_t)TW)) * 2 + inh;
}

// Pass 1: entries per (row, tile, sign).  Upper entries of row i are only
// produced by row i's thread (plain increments); lower ones use atomics.
__global__ void k_count(const nc_graphgen_t g, int32_t T, int32_t TW, int32_t* lower_len, int32_t* upper_len) {
  const Comm cm = make_comm(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n_neurons;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool mine = g.owner[i] == g.shard;
    const uint32_t iid = (uint32_t)g.internal_id[i];
    const uint32_t inh_i = is_inh(g, i);
    const int64_t ri = (int64_t)iid - g.local_base;
    for_each_upper(g, cm, i, [&](int64_t j, bool) {
      const uint32_t jid = (uint32_t)g.internal_id[j];
      if (mine) upper_len[seg_index(ri, T, TW, jid, is_inh(g, j))] += 1;
      if (g.owner[j] == g.shard) atomicAdd(lower_len + seg_index((int64_t)jid - g.local_base, T, TW, iid, inh_i), 1);
    });
  }
}

// Degree of every neuron (both endpoints of every edge), for the SELL row order.
__global__ void k_degrees(const nc_graphgen_t g, int32_t* deg) {
  const Comm cm = make_comm(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n_neurons;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t up = 0;
    for_each_upper(g, cm, i, [&](int64_t j, bool) {
      ++up;
      atomicAdd(deg + j, 1);
    });
    if (up) atomicAdd(deg + i, up);
  }
}

// Position of the k-th entry of (row, tile, sign) in the unpacked padded SELL-32
// layout (uint32 units, ncdev::kSlotEntries words per slot; nc_sell_pack packs them).
__device__ __forceinline__ int64_t sell_pos(const int64_t* slice_ptr, const uint32_t* row_meta,
                                            const int32_t* pos_of, int32_t T, int64_t n_local, int64_t row,
                                            int64_t seg, int32_t k) {
  const int64_t t = (seg >> 1) - row * T;
  const int64_t p = pos_of ? (int64_t)pos_of[row * T + t] : row;   // position of the row in tile t
  const int64_t blk = slice_ptr[(p >> 5) * T + t];
  const int64_t slot = ((seg & 1) ? (int64_t)(row_meta[t * n_local + p] & 0xFFFFu) : 0) + k / ncdev::kSlotEntries;
  return (blk + slot * 32 + (p & 31)) * ncdev::kSlotEntries + k % ncdev::kSlotEntries;
}

// Pass 2: regenerate the same edges and place them; slots inside a
// (row, tile, sign) segment are claimed with atomics (any order is fine:
// delivery sums integers).
__global__ void k_fill(const nc_graphgen_t g, int32_t T, int32_t TW, const int64_t* slice_ptr,
                       const uint32_t* row_meta, const int32_t* pos_of, int32_t* fill, uint32_t* syn) {
  const Comm cm = make_comm(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n_neurons;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool mine = g.owner[i] == g.shard;
    const uint32_t iid = (uint32_t)g.internal_id[i];
    const uint32_t inh_i = is_inh(g, i);
    const int64_t ri = (int64_t)iid - g.local_base;
    for_each_upper(g, cm, i, [&](int64_t j, bool intra) {
      const bool jm = g.owner[j] == g.shard;
      if (!mine && !jm) return;
      const uint32_t q = edge_q(g, i, j, intra);
      const uint32_t jid = (uint32_t)g.internal_id[j];
      if (mine) {
        const int64_t seg = seg_index(ri, T, TW, jid, is_inh(g, j));
        const int32_t k = atomicAdd(fill + seg, 1);
        syn[sell_pos(slice_ptr, row_meta, pos_of, T, g.n_local, ri, seg, k)] = pack(jid - tile_base(jid, TW), q);
      }
      if (jm) {
        const int64_t rj = (int64_t)jid - g.local_base;
        const int64_t seg = seg_index(rj, T, TW, iid, inh_i);
        const int32_t k = atomicAdd(fill + seg, 1);
        syn[sell_pos(slice_ptr, row_meta, pos_of, T, g.n_local, rj, seg, k)] = pack(iid - tile_base(iid, TW), q);
      }
    });
  }
}

// The same two passes over an explicit edge list (a host NeuronGraph uploaded
// as int32 (i, j) + uint8 q columns, simulate()'s path): every edge (i, j) is
// one synapse each way, so post row j gets pre i and row i gets pre j.  Counts
// go to one array with atomics (any order: delivery sums integers).
__global__ void k_edges_count(const nc_graphgen_t g, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                              int64_t n_edges, int32_t T, int32_t TW, int32_t* seg_len) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_edges;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = ei[k], j = ej[k];
    const bool im = g.owner[i] == g.shard, jm = g.owner[j] == g.shard;
    if (!im && !jm) continue;
    const uint32_t iid = (uint32_t)g.internal_id[i], jid = (uint32_t)g.internal_id[j];
    if (im) atomicAdd(seg_len + seg_index((int64_t)iid - g.local_base, T, TW, jid, is_inh(g, j)), 1);
    if (jm) atomicAdd(seg_len + seg_index((int64_t)jid - g.local_base, T, TW, iid, is_inh(g, i)), 1);
  }
}

__global__ void k_edges_fill(const nc_graphgen_t g, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej,
                             const uint8_t* __restrict__ qe, int64_t n_edges, int32_t T, int32_t TW,
                             const int64_t* slice_ptr, const uint32_t* row_meta, const int32_t* pos_of, int32_t* fill,
                             uint32_t* syn) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_edges;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = ei[k], j = ej[k];
    const bool im = g.owner[i] == g.shard, jm = g.owner[j] == g.shard;
    if (!im && !jm) continue;
    const uint32_t q = qe[k];
    const uint32_t iid = (uint32_t)g.internal_id[i], jid = (uint32_t)g.internal_id[j];
    if (im) {
      const int64_t ri = (int64_t)iid - g.local_base;
      const int64_t seg = seg_index(ri, T, TW, jid, is_inh(g, j));
      const int32_t c = atomicAdd(fill + seg, 1);
      syn[sell_pos(slice_ptr, row_meta, pos_of, T, g.n_local, ri, seg, c)] = pack(jid - tile_base(jid, TW), q);
    }
    if (jm) {
      const int64_t rj = (int64_t)jid - g.local_base;
      const int64_t seg = seg_index(rj, T, TW, iid, is_inh(g, i));
      const int32_t c = atomicAdd(fill + seg, 1);
      syn[sell_pos(slice_ptr, row_meta, pos_of, T, g.n_local, rj, seg, c)] = pack(iid - tile_base(iid, TW), q);
    }
  }
}

// Push synapses straight from the generator, for the event-driven engines (no
// pull layout needed: config 5 over 2 GPUs holds 2.5e10 synapses per GPU, which
// fit as 4-byte push entries but not as pull layout + transpose).  Rows are
// internal pre ids (every neuron), entries this shard's post rows,
// (inh(pre) << 31) | ((q - 1) << 26) | post_local -- the nc_build_push_csr
// format.  Phase 0 counts entries per pre row into cnt[pre + 1] and ORs the
// shards hosting each local row's targets into its 16-bit destination mask;
// the host scans cnt into rowptr; phase 1 places the entries (slot claims with
// atomics: the order inside a row is free, delivery sums integers).
__device__ __forceinline__ void or_dest(uint16_t* dest, int64_t r, uint32_t m) {
  unsigned int* w = reinterpret_cast<unsigned int*>(dest + (r & ~1ll));
  atomicOr(w, m << (16 * (r & 1)));
}

__global__ void k_push_gen(const nc_graphgen_t g, int phase, unsigned long long* cnt, const int64_t* rowptr,
                           int32_t* fill, uint32_t* out, uint16_t* dest) {
  const Comm cm = make_comm(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n_neurons;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t oi = g.owner[i];
    const uint32_t iid = (uint32_t)g.internal_id[i];
    const uint32_t inh_i = is_inh(g, i);
    for_each_upper(g, cm, i, [&](int64_t j, bool intra) {
      const int32_t oj = g.owner[j];
      if (oi != g.shard && oj != g.shard) return;
      const uint32_t jid = (uint32_t)g.internal_id[j];
      if (phase == 0) {
        if (oj == g.shard) atomicAdd(cnt + iid + 1, 1ull);
        if (oi == g.shard) atomicAdd(cnt + jid + 1, 1ull);
        if (oi != oj) {
          if (oi == g.shard) or_dest(dest, (int64_t)iid - g.local_base, 1u << oj);
          else or_dest(dest, (int64_t)jid - g.local_base, 1u << oi);
        }
        return;
      }
      const uint32_t q = edge_q(g, i, j, intra);
      if (oj == g.shard) {
        const int32_t k = atomicAdd(fill + iid, 1);
        out[rowptr[iid] + k] = (inh_i << 31) | ((q - 1u) << 26) | (uint32_t)((int64_t)jid - g.local_base);
      }
      if (oi == g.shard) {
        const int32_t k = atomicAdd(fill + jid, 1);
        out[rowptr[jid] + k] = (is_inh(g, j) << 31) | ((q - 1u) << 26) | (uint32_t)((int64_t)iid - g.local_base);
      }
    });
  }
}

// Windowed push (nc_shard_t push_windows): the same enumeration, entries grouped
// by the window of their post row and stored relative to the window start.
__global__ void k_push_gen_win(const nc_graphgen_t g, int phase, int W, int wrows, uint32_t* cnt,
                               const int64_t* rowptr, const uint16_t* winoff, uint32_t* fill, uint32_t* out,
                               uint16_t* dest) {
  const Comm cm = make_comm(g);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n_neurons;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t oi = g.owner[i];
    const uint32_t iid = (uint32_t)g.internal_id[i];
    const uint32_t inh_i = is_inh(g, i);
    for_each_upper(g, cm, i, [&](int64_t j, bool intra) {
      const int32_t oj = g.owner[j];
      if (oi != g.shard && oj != g.shard) return;
      const uint32_t jid = (uint32_t)g.internal_id[j];
      // (pre, local post) pairs of this edge on this shard
      const int64_t rj = (int64_t)jid - g.local_base, ri = (int64_t)iid - g.local_base;
      if (phase == 0) {
        if (oj == g.shard) atomicAdd(cnt + (int64_t)iid * W + rj / wrows, 1u);
        if (oi == g.shard) atomicAdd(cnt + (int64_t)jid * W + ri / wrows, 1u);
        if (oi != oj) {
          if (oi == g.shard) or_dest(dest, ri, 1u << oj);
          else or_dest(dest, rj, 1u << oi);
        }
        return;
      }
      const uint32_t q = edge_q(g, i, j, intra);
      if (oj == g.shard) {
        const int64_t w = rj / wrows, key = (int64_t)iid * W + w;
        const uint32_t k = atomicAdd(fill + key, 1u);
        out[rowptr[iid] + winoff[(int64_t)iid * (W + 1) + w] + k] =
            (inh_i << 31) | ((q - 1u) << 26) | (uint32_t)(rj - w * wrows);
      }
      if (oi == g.shard) {
        const int64_t w = ri / wrows, key = (int64_t)jid * W + w;
        const uint32_t k = atomicAdd(fill + key, 1u);
        out[rowptr[jid] + winoff[(int64_t)jid * (W + 1) + w] + k] =
            (is_inh(g, j) << 31) | ((q - 1u) << 26) | (uint32_t)(ri - w * wrows);
      }
    });
  }
}

// Pad pre-fill of the unpacked padded layout: the pad entry (q = 0) is 0.
__global__ void k_fill_pads(const int64_t* slice_ptr, int64_t n_blocks, uint32_t* syn) {
  for (int64_t b = blockIdx.x; b < n_blocks; b += gridDim.x)
    for (int64_t k = slice_ptr[b] * ncdev::kSlotEntries + threadIdx.x; k < slice_ptr[b + 1] * ncdev::kSlotEntries;
         k += blockDim.x)
      syn[k] = 0u;
}

// Unpacked entries (q << 26 | tile-relative id, ncdev::kSlotEntries per slot)
// -> packed 16-byte slots of 25-bit fields (q << 19 | id).
__global__ void k_sell_pack(const uint32_t* src, int64_t n_slots, uint4* dst) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_slots;
       s += (int64_t)gridDim.x * blockDim.x) {
    uint32_t f[ncdev::kSlotEntries];
#pragma unroll
    for (int i = 0; i < ncdev::kSlotEntries; ++i) {
      const uint32_t e = src[s * ncdev::kSlotEntries + i];
      f[i] = ncdev::make_field(e >> 26, e & ncdev::kFieldIdMask);
    }
    dst[s] = ncdev::pack_slot(f);
  }
}

// Destination shards of every local row: warp per (slice, tile) block, lane =
// position (row_perm places rows per tile), OR-ed into the row's 16-bit mask
// through the aligned 32-bit word holding it.  Pads have q = 0.
__global__ void k_dest_mask(const int64_t* slice_ptr, const uint32_t* row_meta, const int32_t* row_perm, int32_t G,
                            int32_t T, int32_t tile_words, const uint32_t* syn, int32_t n_local, const int32_t* shard_base,
                            int32_t n_shards, int32_t self, uint16_t* dest) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_blocks = ((int64_t)(n_local + 31) >> 5) * T;
  for (int64_t b = wid; b < n_blocks; b += nw) {
    const int64_t s = b / T, t = b % T;
    const int64_t p = (s << 5) + lane;
    const int64_t b0 = slice_ptr[b];
    const int64_t tbase = t * tile_words * 32;
    const int mine = p < n_local ? (int)(row_meta[t * n_local + p] >> 16) : 0;
    const int hi = (int)__reduce_max_sync(0xffffffffu, (unsigned)mine);
    uint32_t m = 0;
    int off = 0;
    for (int u = 0; u < hi; ++u) {
      const int pos = ncdev::jsell_pos(u, mine, lane, off);
      if (u >= mine) continue;
      const ncdev::Fields x = ncdev::unpack_slot(reinterpret_cast<const uint4*>(syn)[b0 + pos]);
      for (int c = 0; c < ncdev::kSlotEntries; ++c) {
        const uint32_t f = x.f[c] & ncdev::kFieldMask;
        if ((f >> 19) == 0) continue;  // pad
        const int64_t pre = ncdev::field_id(f) + tbase;
        for (int h = 0; h < n_shards; ++h)
          if (pre >= shard_base[h] && pre < shard_base[h + 1]) m |= 1u << h;
      }
    }
    m &= ~(1u << self);
    if (p < n_local && m) {
      const int64_t r = ncdev::placed_row(row_perm, n_local, G, t, p);
      unsigned int* w = reinterpret_cast<unsigned int*>(dest + (r & ~1ll));
      atomicOr(w, m << (16 * (r & 1)));
    }
  }
}

// Shared-memory bank placement (padded SELL-32, before nc_sell_repack).  The
// step kernel looks entry k of slot u up for all 32 lanes in one shared-memory
// instruction; its bank is the bitmap word's low 5 bits, (entry >> 5) & 31.
// Within each E / I segment of a row, entry j = 5u + k of lane l is given a pre
// in bank (l + j) & 31 where the row has one left (so the 32 lanes of one
// lookup hit 32 different banks), the rest fill the remaining positions.
// Thread per (position, tile); src = a copy of the padded array, dst = it.
__global__ void k_bank_order(const int64_t* pptr, const uint32_t* row_meta, int32_t T, int32_t n_local,
                             const uint32_t* src, uint32_t* dst) {
  const int64_t total = (int64_t)n_local * T;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = x / n_local, p = x % n_local;
    const int lane = (int)(p & 31);
    const int64_t base = pptr[(p >> 5) * T + t];
    const uint32_t meta = row_meta[t * n_local + p];
    const int emid = (int)(meta & 0xFFFFu), len = (int)(meta >> 16);
    constexpr int E = ncdev::kSlotEntries;
    auto at = [&](int j) { return (base + (int64_t)(j / E) * 32 + lane) * E + j % E; };
    for (int seg = 0; seg < 2; ++seg) {
      const int j0 = seg ? E * emid : 0, j1 = seg ? E * len : E * emid;
      if (j1 <= j0) continue;
      int cnt[32], seen[32];
      for (int b = 0; b < 32; ++b) cnt[b] = seen[b] = 0;
      for (int j = j0; j < j1; ++j) ++cnt[(src[at(j)] >> 5) & 31];
      auto first = [&](int b) { return j0 + ((b - lane - j0) & 31); };   // first j >= j0 wanting bank b
      auto cap = [&](int b) { const int f = first(b); return f < j1 ? (j1 - 1 - f) / 32 + 1 : 0; };
      int ov = 0;
      for (int j = j0; j < j1; ++j) {
        const uint32_t e = src[at(j)];
        const int b = (int)((e >> 5) & 31);
        const int i = seen[b]++;
        int target;
        if (i < cap(b)) {
          target = first(b) + 32 * i;
        } else {   // the ov-th free position: the unfilled tails of the banks in short supply
          int k = ov++;
          target = j0;
          for (int c = 0; c < 32; ++c) {
            const int d = cap(c) - cnt[c];
            if (d <= 0) continue;
            if (k < d) {
              target = first(c) + 32 * (cnt[c] + k);
              break;
            }
            k -= d;
          }
        }
        dst[at(target)] = e;
      }
    }
  }
}

// Padded SELL-32 (block = longest row x 32 lanes, slot u of lane l at u*32 + l:
// what the generator fills) <-> J-SELL (jsell.cuh).  Warp per block.
__global__ void k_sell_repack(const int64_t* pptr, const int64_t* cptr, const uint32_t* row_meta, int32_t T,
                              int32_t n_local, const uint4* src, uint4* dst, int to_compact) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_blocks = ((int64_t)(n_local + 31) >> 5) * T;
  for (int64_t b = wid; b < n_blocks; b += nw) {
    const int64_t r = ((b / T) << 5) + lane;
    const int64_t t = b % T;
    const int mine = r < n_local ? (int)(row_meta[t * n_local + r] >> 16) : 0;
    const int hi = (int)__reduce_max_sync(0xffffffffu, (unsigned)mine);
    int off = 0;
    for (int u = 0; u < hi; ++u) {
      const int pos = ncdev::jsell_pos(u, mine, lane, off);
      if (u >= mine) continue;
      const int64_t pp = pptr[b] + (int64_t)u * 32 + lane, cp = cptr[b] + pos;
      if (to_compact) dst[cp] = src[pp];
      else dst[pp] = src[cp];
    }
  }
}

int grid_for(int64_t n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (n + threads - 1) / threads;
  if (b > (int64_t)sms * 16) b = (int64_t)sms * 16;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

extern "C" int nc_graphgen_count(const nc_graphgen_t* g, int32_t n_tiles, int32_t tile_words, int32_t* lower_len,
                                 int32_t* upper_len, void* stream) {
  if (!g || g->n_neurons < 1 || g->n_communities < 1 || g->n_communities > g->n_neurons || n_tiles < 1 ||
      tile_words < 1) {
    nc_set_error("nc_graphgen_count: invalid generator spec");
    return NC_E_ARG;
  }
  k_count<<<grid_for(g->n_neurons, 128), 128, 0, (cudaStream_t)stream>>>(*g, n_tiles, tile_words, lower_len,
                                                                           upper_len);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_graphgen_degrees(const nc_graphgen_t* g, int32_t* deg, void* stream) {
  if (!g || g->n_neurons < 1 || g->n_communities < 1 || g->n_communities > g->n_neurons) {
    nc_set_error("nc_graphgen_degrees: invalid generator spec");
    return NC_E_ARG;
  }
  k_degrees<<<grid_for(g->n_neurons, 128), 128, 0, (cudaStream_t)stream>>>(*g, deg);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_graphgen_fill(const nc_graphgen_t* g, int32_t n_tiles, int32_t tile_words, const int64_t* slice_ptr,
                                const uint32_t* row_meta, const int32_t* pos_of, int32_t* lower_fill, uint32_t* syn,
                                void* stream) {
  if (!g || n_tiles < 1 || tile_words < 1) {
    nc_set_error("nc_graphgen_fill: bad arguments");
    return NC_E_ARG;
  }
  k_fill<<<grid_for(g->n_neurons, 128), 128, 0, (cudaStream_t)stream>>>(*g, n_tiles, tile_words, slice_ptr,
                                                                          row_meta, pos_of, lower_fill, syn);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_graphgen_push(const nc_graphgen_t* g, int32_t phase, int64_t* push_rowptr, int32_t* push_fill,
                                uint32_t* push_syn, uint16_t* dest_mask, void* stream) {
  if (!g || g->n_neurons < 1 || g->n_communities < 1 || g->n_communities > g->n_neurons || !g->owner ||
      !g->internal_id || !push_rowptr || (phase == 0 && !dest_mask) ||
      (phase == 1 && (!push_fill || !push_syn)) || (phase != 0 && phase != 1)) {
    nc_set_error("nc_graphgen_push: bad arguments");
    return NC_E_ARG;
  }
  k_push_gen<<<grid_for(g->n_neurons, 128), 128, 0, (cudaStream_t)stream>>>(
      *g, phase, reinterpret_cast<unsigned long long*>(push_rowptr), push_rowptr, push_fill, push_syn, dest_mask);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_graphgen_push_windowed(const nc_graphgen_t* g, int32_t phase, int32_t windows, int32_t window_rows,
                                         uint32_t* counts, const int64_t* push_rowptr, const uint16_t* push_winoff,
                                         uint32_t* fill, uint32_t* push_syn, uint16_t* dest_mask, void* stream) {
  if (!g || g->n_neurons < 1 || g->n_communities < 1 || g->n_communities > g->n_neurons || !g->owner ||
      !g->internal_id || windows < 1 || window_rows < 32 || (window_rows & 31) ||
      (int64_t)windows * window_rows < g->n_local ||
      (phase == 0 && (!counts || !dest_mask)) || (phase == 1 && (!push_rowptr || !push_winoff || !fill || !push_syn)) ||
      (phase != 0 && phase != 1)) {
    nc_set_error("nc_graphgen_push_windowed: bad arguments");
    return NC_E_ARG;
  }
  k_push_gen_win<<<grid_for(g->n_neurons, 128), 128, 0, (cudaStream_t)stream>>>(
      *g, phase, windows, window_rows, counts, push_rowptr, push_winoff, fill, push_syn, dest_mask);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_edges_count(const nc_graphgen_t* g, const int32_t* edge_i, const int32_t* edge_j, int64_t n_edges,
                              int32_t n_tiles, int32_t tile_words, int32_t* seg_len, void* stream) {
  if (!g || !g->owner || !g->internal_id || n_edges < 0 || (n_edges && (!edge_i || !edge_j)) || n_tiles < 1 ||
      tile_words < 1 || !seg_len) {
    nc_set_error("nc_edges_count: bad arguments");
    return NC_E_ARG;
  }
  if (n_edges == 0) return NC_OK;
  k_edges_count<<<grid_for(n_edges, 256), 256, 0, (cudaStream_t)stream>>>(*g, edge_i, edge_j, n_edges, n_tiles,
                                                                           tile_words, seg_len);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_edges_fill(const nc_graphgen_t* g, const int32_t* edge_i, const int32_t* edge_j, const uint8_t* q,
                             int64_t n_edges, int32_t n_tiles, int32_t tile_words, const int64_t* slice_ptr,
                             const uint32_t* row_meta, const int32_t* pos_of, int32_t* fill, uint32_t* syn,
                             void* stream) {
  if (!g || !g->owner || !g->internal_id || n_edges < 0 || (n_edges && (!edge_i || !edge_j || !q)) ||
      n_tiles < 1 || tile_words < 1 || !slice_ptr || !row_meta || !fill || !syn) {
    nc_set_error("nc_edges_fill: bad arguments");
    return NC_E_ARG;
  }
  if (n_edges == 0) return NC_OK;
  k_edges_fill<<<grid_for(n_edges, 256), 256, 0, (cudaStream_t)stream>>>(*g, edge_i, edge_j, q, n_edges, n_tiles,
                                                                          tile_words, slice_ptr, row_meta, pos_of,
                                                                          fill, syn);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sell_fill_pads(const int64_t* slice_ptr, int64_t n_blocks, int32_t n_tiles, int32_t tile_words,
                                 uint32_t* syn, void* stream) {
  if (n_blocks <= 0) return NC_OK;
  int64_t grid = n_blocks < 65535 ? n_blocks : 65535;
  (void)n_tiles;
  (void)tile_words;
  k_fill_pads<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(slice_ptr, n_blocks, syn);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sell_pack(const uint32_t* unpacked, int64_t n_slots, uint32_t* packed, void* stream) {
  if (n_slots < 0 || (n_slots > 0 && (!unpacked || !packed))) {
    nc_set_error("nc_sell_pack: bad arguments");
    return NC_E_ARG;
  }
  if (n_slots == 0) return NC_OK;
  k_sell_pack<<<grid_for(n_slots, 256), 256, 0, (cudaStream_t)stream>>>(unpacked, n_slots,
                                                                         reinterpret_cast<uint4*>(packed));
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sell_bank_order(const int64_t* padded_ptr, const uint32_t* row_meta, int32_t n_tiles,
                                  int32_t n_local, const uint32_t* src, uint32_t* dst, void* stream) {
  if (n_tiles < 1 || n_local < 0 || !padded_ptr || !row_meta || !src || !dst || src == dst) {
    nc_set_error("nc_sell_bank_order: bad arguments");
    return NC_E_ARG;
  }
  if (n_local == 0) return NC_OK;
  k_bank_order<<<grid_for((int64_t)n_local * n_tiles, 128), 128, 0, (cudaStream_t)stream>>>(
      padded_ptr, row_meta, n_tiles, n_local, src, dst);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_sell_repack(const int64_t* padded_ptr, const int64_t* slice_ptr, const uint32_t* row_meta,
                              int32_t n_tiles, int32_t n_local, const uint32_t* src, uint32_t* dst, int32_t to_jagged,
                              void* stream) {
  if (n_tiles < 1 || n_local < 0 || !padded_ptr || !slice_ptr || !row_meta) {
    nc_set_error("nc_sell_repack: bad arguments");
    return NC_E_ARG;
  }
  if (n_local == 0) return NC_OK;
  const int64_t n_blocks = ((int64_t)(n_local + 31) / 32) * n_tiles;
  k_sell_repack<<<grid_for(n_blocks * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      padded_ptr, slice_ptr, row_meta, n_tiles, n_local, reinterpret_cast<const uint4*>(src),
      reinterpret_cast<uint4*>(dst), to_jagged ? 1 : 0);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_dest_mask_from_csr(const int64_t* slice_ptr, const uint32_t* row_meta, const int32_t* row_perm,
                                     int32_t cta_groups, int32_t n_tiles, int32_t tile_words, const uint32_t* syn, int32_t n_local, const int32_t* shard_base,
                                     int32_t n_shards, int32_t self, uint16_t* dest_mask, void* stream) {
  if (n_shards < 1 || n_shards > NC_MAX_SHARDS) {
    nc_set_error("nc_dest_mask_from_csr: n_shards must be in [1, %d]", NC_MAX_SHARDS);
    return NC_E_ARG;
  }
  if (n_local == 0) return NC_OK;
  k_dest_mask<<<grid_for((int64_t)n_local * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      slice_ptr, row_meta, row_perm, cta_groups < 1 ? 1 : cta_groups, n_tiles, tile_words, syn, n_local, shard_base,
      n_shards, self, dest_mask);
  NC_LAUNCH_CHECK();
  return NC_OK;
}
