// Jagged SELL-32 (J-SELL) addressing, shared by the delivery kernels and the
// builders (include/neurocomm_b200.h documents the layout).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ncdev {

// A 16-byte slot holds 5 synapse fields of 25 bits: f = (q << 19) | (id ^ 31),
// id the pre's bitmap index relative to its tile (< 2^19, so tiles are <= 16384
// words), q in [1, 32] its weight units; the pad field has q = 0.  The low 5
// bits store 31 - (bit in word), so a left funnel shift of the word by f moves
// the pre's bit to bit 31 (field_term).  Field i starts at bit 25 i of the slot
// (x | y << 32 | z << 64 | w << 96).
constexpr int kSlotEntries = 5;
constexpr uint32_t kFieldMask = (1u << 25) - 1u;
constexpr uint32_t kFieldIdMask = (1u << 19) - 1u;
constexpr uint32_t kBitXor = 31u;

// packed field <-> (q, tile-relative id)
__host__ __device__ __forceinline__ uint32_t make_field(uint32_t q, uint32_t id) {
  return (q << 19) | (id ^ kBitXor);
}
__host__ __device__ __forceinline__ uint32_t field_id(uint32_t f) { return (f & kFieldIdMask) ^ kBitXor; }

struct Fields {
  uint32_t f[kSlotEntries];
};

__device__ __forceinline__ Fields unpack_slot(uint4 e) {
  Fields r;
  r.f[0] = e.x;                               // upper bits masked by the users
  r.f[1] = __funnelshift_r(e.x, e.y, 25);
  r.f[2] = __funnelshift_r(e.y, e.z, 18);
  r.f[3] = __funnelshift_r(e.z, e.w, 11);
  r.f[4] = e.w >> 4;
  return r;
}

__device__ __forceinline__ uint4 pack_slot(const uint32_t (&f)[kSlotEntries]) {
  return make_uint4(f[0] | (f[1] << 25), (f[1] >> 7) | (f[2] << 18), (f[2] >> 14) | (f[3] << 11),
                    (f[3] >> 21) | (f[4] << 4));
}

// Jagged SELL-32 (J-SELL) block: lane l's row has len_l = meta >> 16 slots,
// the first (meta & 0xFFFF) excitatory.  Slot u of the lanes with len > u is
// stored contiguously, in lane order: position = sum_{v<u} cnt_v + rank of the
// lane among them, cnt_v = #lanes with len > v.  So the regular part
// u < min_l len_l is plain SELL (u*32 + lane) and only the ragged tail needs a
// ballot per slot -- and the block stores no padding beyond each row's E/I
// segments rounded up to 5 entries.  A warp steps u in lockstep; jsell_pos
// returns this lane's position of slot u and advances `off` to slot u + 1.
__device__ __forceinline__ int jsell_pos(int u, int mine, int lane, int& off) {
  const uint32_t act = __ballot_sync(0xffffffffu, u < mine);
  const int pos = off + __popc(act & ((1u << lane) - 1u));
  off += __popc(act);
  return pos;
}

// Local row at position p of tile t (tiled placement; identity without one):
// row_perm holds the CTA-local index k, row = 32*(c + (k/32)*G) + k%32 with
// c = (p/32) mod G.
__device__ __forceinline__ int64_t placed_row(const int32_t* row_perm, int64_t n_local, int32_t G, int64_t t,
                                              int64_t p) {
  if (!row_perm) return p;
  const int64_t k = row_perm[t * n_local + p];
  const int64_t c = (p >> 5) % G;
  return ((c + (k >> 5) * G) << 5) + (k & 31);
}

}  // namespace ncdev
