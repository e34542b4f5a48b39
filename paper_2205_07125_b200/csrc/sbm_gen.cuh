// Device side of the counter-based SBM generator (csrc/graphgen.cu), shared with
// the K5 histogram over a generated network (traffic_hist.cu): the community
// layout, the per-(row, block) Philox gap sampler and the per-edge p.
// Distributions follow neurocomm generate_synthetic (model.py:146-253).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include "nc_common.h"
#include "philox.cuh"

namespace ncgen {

struct Comm {
  int64_t q, r, big;  // sizes: first r communities have q+1, rest q; big = r*(q+1)
  __device__ int64_t of(int64_t i) const { return i < big ? i / (q + 1) : r + (i - big) / q; }
  __device__ int64_t start(int64_t c) const { return c < r ? c * (q + 1) : big + (c - r) * q; }
  __device__ int64_t size(int64_t c) const { return c < r ? q + 1 : q; }
};

__device__ __forceinline__ Comm make_comm(const nc_graphgen_t& g) {
  Comm c;
  c.q = g.n_neurons / g.n_communities;
  c.r = g.n_neurons % g.n_communities;
  c.big = c.r * (c.q + 1);
  return c;
}

// Uniform double in [0, 1) with 53 random bits.
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return (double)(((uint64_t)a << 21) ^ (uint64_t)(b >> 11)) * 0x1.0p-53;
}

// Sequential geometric sampler over one block of n trials.
struct GapStream {
  uint32_t row, blk, k0, k1, ctr;
  nc_u32x4 buf;
  int avail;
  double inv_log1m;
  __device__ GapStream(uint32_t row_, uint32_t blk_, uint64_t seed, double p)
      : row(row_), blk(blk_), k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), ctr(0), avail(0) {
    inv_log1m = 1.0 / log1p(-p);
  }
  __device__ double next_u() {
    if (avail == 0) {
      nc_u32x4 c = {row, blk, ctr++, NC_TAG_GAPS};
      buf = nc_philox4x32_10(c, k0, k1);
      avail = 2;
    }
    double u = (avail == 2) ? u53(buf.x, buf.y) : u53(buf.z, buf.w);
    --avail;
    return u;
  }
  // gap >= 1 between successes
  __device__ int64_t gap() {
    const double u = next_u();
    const double gf = floor(log1p(-u) * inv_log1m);
    return (gf >= 9.0e18) ? INT64_MAX / 4 : (int64_t)gf + 1;
  }
};

// p of edge (i, j), i < j: U(intra range) or U(inter range) from the edge's own counter
__device__ __forceinline__ double edge_p(const nc_graphgen_t& g, int64_t i, int64_t j, bool intra) {
  nc_u32x4 c = {(uint32_t)i, (uint32_t)j, NC_TAG_EDGEP, (uint32_t)((i >> 32) ^ ((j >> 32) << 16))};
  nc_u32x4 x = nc_philox4x32_10(c, (uint32_t)g.seed, (uint32_t)(g.seed >> 32));
  const double lo = intra ? g.intra_lo : g.inter_lo;
  const double hi = intra ? g.intra_hi : g.inter_hi;
  // explicit round-to-nearest steps, no FMA contraction: the host restatement
  // (graphgen_host.cpp, -ffp-contract=off) and K5 see the same p bits
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u53(x.x, x.y)));
}

// Weight units q = ceil(32 p) in [1, 32] (sim.q_from_p)
__device__ __forceinline__ uint32_t edge_q(const nc_graphgen_t& g, int64_t i, int64_t j, bool intra) {
  const double p = edge_p(g, i, j, intra);
  double qf = ceil(p * 32.0);
  qf = qf < 1.0 ? 1.0 : (qf > 32.0 ? 32.0 : qf);
  return (uint32_t)qf;
}

// Visit every upper neighbour j of row i:  f(j, intra).
template <typename F>
__device__ void for_each_upper(const nc_graphgen_t& g, const Comm& cm, int64_t i, F&& f) {
  const int64_t ci = cm.of(i);
  const int64_t nc = g.n_communities;
  for (int64_t b = ci; b < nc; ++b) {
    const bool intra = (b == ci);
    const double p = intra ? g.p_in : g.p_out;
    if (p <= 0.0) continue;
    const int64_t first = intra ? i + 1 : cm.start(b);
    const int64_t n = intra ? cm.start(ci) + cm.size(ci) - i - 1 : cm.size(b);
    if (n <= 0) continue;
    if (p >= 1.0) {
      for (int64_t t = 0; t < n; ++t) f(first + t, intra);
      continue;
    }
    GapStream gs((uint32_t)i, (uint32_t)b, g.seed, p);
    int64_t pos = -1;
    for (;;) {
      pos += gs.gap();
      if (pos >= n) break;
      f(first + pos, intra);
    }
  }
}

}  // namespace ncgen
