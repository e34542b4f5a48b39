// K5: exact GPU traffic / edge-cut histogram.
//
// Device replacement for the summation in neurocomm traffic.aggregate
// (traffic.py:66-84), whose per-cell sums go through accum.keyed_sums
// (accum.py:21-41) = math.fsum, i.e. the correctly rounded exact sum.  fp64
// atomics cannot reproduce that (the survey measured naive fp64 differing in
// every cell), so each contribution is decomposed into its 53-bit integer
// mantissa and exponent and added EXACTLY into a fixed-point accumulator of
// 32-bit digits held in 64-bit limbs: integer adds are associative, the result
// is order independent, and the host rounds the exact integer once.
//
// Per block the cells live in shared memory (N(N+1)/2 upper cells x n_digits
// limbs); at the end each block carry-normalises its digits to < 2^32 and
// adds them to the global limbs, which therefore stay below 2^64 for up to
// 2^32 blocks.  When the cells do not fit in shared memory the kernel adds
// straight into global limbs (each add < 2^32, safe for < 2^32 adds per limb).

#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>
#include "nc_common.h"
#include "sbm_gen.cuh"

namespace {

#ifndef NC_K5_THREADS
#define NC_K5_THREADS 256
#endif
#ifndef NC_K5_UNROLL
#define NC_K5_UNROLL 4
#endif
constexpr int kThreads = NC_K5_THREADS;
constexpr size_t kSmemLimit = 96 * 1024;    // fall back to global limbs above this
#ifndef NC_K5_UNIFORM_UNROLL
#define NC_K5_UNIFORM_UNROLL 6   // 1-byte gathers: more edges in flight per thread
#endif
// A/B on B200 (tools/k5_kernel_ab.py, 4.9e7 edges, 8 GPUs; profiles/r02_k5_kernel_ab.log):
// 8 KB of lane copies, >= 4 CTAs per SM (<= 64 registers) and 6 edges in flight per
// thread on the uniform path: 0.216 ms (3.67 TB/s) against 0.246 with 16 KB / no
// register cap / 8 in flight; 5 CTAs per SM or 12 in flight are slower.
#ifndef NC_K5_SMEM_KB
#define NC_K5_SMEM_KB 8
#endif
#ifndef NC_K5_MIN_BLOCKS
#define NC_K5_MIN_BLOCKS 4
#endif
constexpr size_t kSmemBudget = NC_K5_SMEM_KB * 1024;   // lane copies are halved down to this

struct Decomposed {
  unsigned long long mant;  // integer mantissa (0 => nothing to add)
  int lsb;                  // exponent of the mantissa's bit 0
};

__device__ __forceinline__ Decomposed decompose(double x) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(x);
  const int e = (int)((bits >> 52) & 0x7ff);
  Decomposed d;
  d.mant = bits & 0xfffffffffffffull;
  if (e == 0) {
    d.lsb = -1074;
  } else {
    d.mant |= 1ull << 52;
    d.lsb = e - 1075;
  }
  return d;
}

__device__ __forceinline__ double contrib(double p, double wi, double wj) {
  return __dmul_rn(__dmul_rn(p, wi), wj);  // (p*W_i)*W_j, traffic.py:77
}

// Add mant * 2^(lsb - lsb0) into limbs[0..n_digits).
__device__ __forceinline__ void add_fixed(unsigned long long* limbs, int n_digits, Decomposed d,
                                          int lsb0) {
  if (d.mant == 0) return;
  const int s = d.lsb - lsb0;  // >= 0 by construction of lsb0
  const int k = s >> 5, o = s & 31;
  const unsigned long long lo = d.mant << o;                 // low 64 bits of mant << o
  const unsigned long long hi = o ? (d.mant >> (64 - o)) : 0ull;  // bits 64.. (<= 21 bits)
  const unsigned long long d0 = lo & 0xffffffffull, d1 = lo >> 32, d2 = hi;
  if (d0 && k < n_digits) atomicAdd(limbs + k, d0);
  if (d1 && k + 1 < n_digits) atomicAdd(limbs + k + 1, d1);
  if (d2 && k + 2 < n_digits) atomicAdd(limbs + k + 2, d2);
}

__device__ __forceinline__ int cell_index(int64_t a, int64_t b, int n) {
  const int lo = (int)(a < b ? a : b), hi = (int)(a < b ? b : a);
  return lo * n + hi;
}

__global__ void k_exponents(const int64_t* __restrict__ ei, const int64_t* __restrict__ ej,
                            const double* __restrict__ ep, const double* __restrict__ w, int64_t n,
                            int* minmax) {
  int lo = INT_MAX, hi = INT_MIN;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double x = ei ? contrib(ep[k], w[ei[k]], w[ej[k]]) : w[k];
    const Decomposed d = decompose(x);
    if (d.mant == 0) continue;
    lo = min(lo, d.lsb);
    hi = max(hi, d.lsb + 63 - __clzll((long long)d.mant));
  }
  for (int off = 16; off; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    if (lo != INT_MAX) atomicMin(minmax, lo);
    if (hi != INT_MIN) atomicMax(minmax + 1, hi);
  }
}

// Shared-memory accumulator of one block: `copies` copies (lane & (copies-1)) of
// [cell][digit] pairs of 32-bit words {sum, carries}, upper cells only
// (compact index, see ucell).  A digit add is one NATIVE 32-bit shared atomic
// (64-bit shared atomics compile to CAS spin loops on sm_100a,
// ATOMS.CAST.SPIN.64: the round-1 bottleneck) plus, when the returned old value
// shows a wrap, a second one on the carry word: the pair is exactly the 64-bit
// limb sum + carries * 2^32.  Lanes get their own copy (up to 32, as shared
// memory allows) so lanes hitting the same cell hit different addresses, and the
// copy stride is odd so those addresses fall in different banks (with 4 copies
// 64 words apart, 95 % of the shared wavefronts were bank conflicts).
__device__ __forceinline__ void add32c(unsigned int* p, unsigned int d) {
  if (!d) return;
  const unsigned int old = atomicAdd(p, d);
  if (old + d < old) atomicAdd(p + 1, 1u);
}

// compact index of upper cell (lo, hi), lo <= hi < n: row lo starts at lo*(2n-lo+1)/2
__device__ __forceinline__ int ucell(int lo, int hi, int n) { return lo * (2 * n - lo + 1) / 2 + (hi - lo); }

// One term into the block's copy `mine` of the cell accumulators (see above).
__device__ __forceinline__ void acc_term(unsigned int* mine, int cell, int n_digits, double x, int lsb0) {
  const Decomposed d = decompose(x);
  if (d.mant == 0) return;
  const int s = d.lsb - lsb0;  // >= 0 by construction of lsb0
  const int kd = s >> 5, o = s & 31;
  const unsigned long long lo = d.mant << o;
  const unsigned long long hi = o ? (d.mant >> (64 - o)) : 0ull;
  unsigned int* c = mine + (cell * n_digits + kd) * 2;
  if (kd < n_digits) add32c(c, (unsigned int)lo);             // digits past the window are dropped,
  if (kd + 1 < n_digits) add32c(c + 2, (unsigned int)(lo >> 32));   // as in add_fixed (callers size it)
  if (kd + 2 < n_digits) add32c(c + 4, (unsigned int)hi);
}

// End of a block: sum the copies of every cell into 64-bit digits, carry-normalise,
// add to the global limbs (upper cells: compact index -> lo * n + hi).
__device__ void flush_cells(const unsigned int* sw, int copies, int cstride, int n_cells, int n_digits, int n_gpus,
                            bool upper, unsigned long long* out) {
  for (int cell = threadIdx.x; cell < n_cells; cell += blockDim.x) {
    int gcell = cell;
    if (upper) {
      int lo = 0, rem = cell;
      while (rem >= n_gpus - lo) rem -= n_gpus - lo++;
      gcell = lo * n_gpus + lo + rem;
    }
    unsigned long long carry = 0;
    for (int k = 0; k < n_digits; ++k) {
      unsigned long long x = carry;   // copies * (2^32 + carries * 2^32) + 2^32: no wrap below 2^31 adds
      for (int c = 0; c < copies; ++c) {
        const unsigned int* e = sw + c * cstride + (cell * n_digits + k) * 2;
        x += (unsigned long long)e[0] + ((unsigned long long)e[1] << 32);
      }
      const unsigned long long digit = (k + 1 < n_digits) ? (x & 0xffffffffull) : x;
      carry = (k + 1 < n_digits) ? (x >> 32) : 0;
      if (digit) atomicAdd(out + (int64_t)gcell * n_digits + k, digit);
    }
  }
}

int smem_cells(bool edges, int n_gpus) { return edges ? n_gpus * (n_gpus + 1) / 2 : n_gpus; }
int copy_stride(int cells, int n_digits) { return (cells * n_digits * 2) | 1; }   // odd: banks shift per copy

// How a neuron's {weight, gpu} is gathered per edge endpoint:
//   kSplit   w[i] and asg[i] (two gathers);
//   kPacked  one 16-byte record per neuron {double w; int32 gpu; pad}
//            (nc_traffic_histogram_packed): one gather;
//   kUniform every weight equals w0 (generate_synthetic's default weight_low ==
//            weight_high): only the uint8 gpu id is gathered, 1 byte per endpoint
//            instead of 16 (the L1 data path and register writeback of the
//            gathers were the bound, 80 % / 70 % busy with the 16-byte records);
//            (p * w0) * w0 is the same two roundings as (p * w_i) * w_j.
enum { kSplit = 0, kPacked = 1, kUniform = 2 };

template <typename Idx, int kRec = kSplit, int kUnroll = NC_K5_UNROLL>
__global__ void __launch_bounds__(kThreads, NC_K5_MIN_BLOCKS)
k_histogram_smem(const Idx* __restrict__ ei, const Idx* __restrict__ ej, const double* __restrict__ ep,
                 const double* __restrict__ w, const Idx* __restrict__ asg, int64_t n, int n_gpus, int lsb0,
                 int n_digits, int copies, unsigned long long* __restrict__ out, double w0 = 1.0,
                 const uint8_t* __restrict__ asg8 = nullptr) {
  extern __shared__ unsigned int sw[];
  const int n_cells = ei ? n_gpus * (n_gpus + 1) / 2 : n_gpus;
  const int cstride = (n_cells * n_digits * 2) | 1;
  for (int k = threadIdx.x; k < copies * cstride; k += blockDim.x) sw[k] = 0u;
  __syncthreads();
  unsigned int* mine = sw + (threadIdx.x & (copies - 1)) * cstride;
  // kUnroll edges per thread and iteration, every load issued before the first use:
  // the gathers of w / assignment (L2-resident) then overlap instead of serialising
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k0 < n; k0 += stride * kUnroll) {
    double x[kUnroll];
    int cell[kUnroll];
    if (ei) {
      int64_t i[kUnroll], j[kUnroll];
      double pe[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t k = k0 + u * stride;
        const bool ok = k < n;
        i[u] = ok ? (int64_t)__ldcs(ei + k) : 0;
        j[u] = ok ? (int64_t)__ldcs(ej + k) : 0;
        pe[u] = ok ? __ldcs(ep + k) : 0.0;
      }
      double wi[kUnroll], wj[kUnroll];
      int ai[kUnroll], aj[kUnroll];
      if (kRec == kUniform) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          wi[u] = w0;
          wj[u] = w0;
          ai[u] = __ldg(asg8 + i[u]);
          aj[u] = __ldg(asg8 + j[u]);
        }
      } else if (kRec == kPacked) {
        const int4* rec = reinterpret_cast<const int4*>(w);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int4 a = __ldg(rec + i[u]), b = __ldg(rec + j[u]);
          wi[u] = __hiloint2double(a.y, a.x);
          wj[u] = __hiloint2double(b.y, b.x);
          ai[u] = a.z;
          aj[u] = b.z;
        }
      } else {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          wi[u] = __ldg(w + i[u]);
          wj[u] = __ldg(w + j[u]);
          ai[u] = (int)__ldg(asg + i[u]);
          aj[u] = (int)__ldg(asg + j[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        x[u] = contrib(pe[u], wi[u], wj[u]);   // p = 0 for the tail: nothing added
        cell[u] = ucell(min(ai[u], aj[u]), max(ai[u], aj[u]), n_gpus);
      }
    } else {  // per-GPU weight totals (binned_sums over assignment)
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t k = k0 + u * stride;
        x[u] = k < n ? w[k] : 0.0;
        cell[u] = k < n ? (int)asg[k] : 0;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) acc_term(mine, cell[u], n_digits, x[u], lsb0);
  }
  __syncthreads();
  flush_cells(sw, copies, cstride, n_cells, n_digits, n_gpus, ei != nullptr, out);
}

// K5 over a generated network (sim.GeneratorSpec, csrc/graphgen.cu): the edges of
// rows [row_begin, row_end) are enumerated on the fly by the generator's own gap
// sampler and their fp64 p by its per-edge counter (sbm_gen.cuh), so the
// reference's aggregate() of a 1e10-synapse network (config 3/5) needs neither the
// edge list nor a host NeuronGraph.  weights NULL = all 1.
__global__ void __launch_bounds__(kThreads)
k_histogram_generated(const nc_graphgen_t g, const double* __restrict__ w, const int32_t* __restrict__ asg,
                      int64_t row_begin, int64_t row_end, int n_gpus, int lsb0, int n_digits, int copies,
                      unsigned long long* __restrict__ out) {
  extern __shared__ unsigned int sw[];
  const int n_cells = n_gpus * (n_gpus + 1) / 2;
  const int cstride = (n_cells * n_digits * 2) | 1;
  for (int k = threadIdx.x; k < copies * cstride; k += blockDim.x) sw[k] = 0u;
  __syncthreads();
  unsigned int* mine = sw + (threadIdx.x & (copies - 1)) * cstride;
  const ncgen::Comm cm = ncgen::make_comm(g);
  for (int64_t i = row_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < row_end;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ai = __ldg(asg + i);
    const double wi = w ? __ldg(w + i) : 1.0;
    ncgen::for_each_upper(g, cm, i, [&](int64_t j, bool intra) {
      const int aj = __ldg(asg + j);
      const double x = contrib(ncgen::edge_p(g, i, j, intra), wi, w ? __ldg(w + j) : 1.0);
      acc_term(mine, ucell(min(ai, aj), max(ai, aj), n_gpus), n_digits, x, lsb0);
    });
  }
  __syncthreads();
  flush_cells(sw, copies, cstride, n_cells, n_digits, n_gpus, true, out);
}

template <typename Idx>
__device__ __forceinline__ void edge_term(const Idx* __restrict__ ei, const Idx* __restrict__ ej,
                                          const double* __restrict__ ep, const double* __restrict__ w,
                                          const Idx* __restrict__ asg, int64_t k, int n_gpus, double* x,
                                          int* cell) {
  if (ei) {
    const int64_t i = (int64_t)ei[k], j = (int64_t)ej[k];
    *x = contrib(ep[k], __ldg(w + i), __ldg(w + j));
    *cell = cell_index((int64_t)__ldg(asg + i), (int64_t)__ldg(asg + j), n_gpus);
  } else {  // per-GPU weight totals (binned_sums over assignment)
    *x = w[k];
    *cell = (int)asg[k];
  }
}

// Fallback when the cells do not fit in shared memory: straight into the global
// limbs (native 64-bit global reductions; each add < 2^32).
template <typename Idx>
__global__ void __launch_bounds__(kThreads)
k_histogram_global(const Idx* __restrict__ ei, const Idx* __restrict__ ej, const double* __restrict__ ep,
                   const double* __restrict__ w, const Idx* __restrict__ asg, int64_t n, int n_gpus, int lsb0,
                   int n_digits, unsigned long long* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double x;
    int cell;
    edge_term(ei, ej, ep, w, asg, k, n_gpus, &x, &cell);
    add_fixed(out + (int64_t)cell * n_digits, n_digits, decompose(x), lsb0);
  }
}

template <typename Idx, int kRec = kSplit, int kUnroll = NC_K5_UNROLL>
int launch_hist(const Idx* ei, const Idx* ej, const double* ep, const double* w, const Idx* asg, int64_t n,
                int n_gpus, int lsb0, int n_digits, unsigned long long* out, cudaStream_t st, double w0 = 1.0,
                const uint8_t* asg8 = nullptr) {
  constexpr auto kernel = k_histogram_smem<Idx, kRec, kUnroll>;
  if (n <= 0) return NC_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // lane-private copies (up to 32) within a 48 KB budget: several blocks per SM
  const int cstride = copy_stride(smem_cells(ei != nullptr, n_gpus), n_digits);
  int copies = 32;
  while (copies > 1 && (size_t)copies * cstride * sizeof(unsigned int) > kSmemBudget) copies >>= 1;
  const size_t smem = (size_t)copies * cstride * sizeof(unsigned int);
  if (smem <= kSmemLimit) {
    static bool attr = false;
    if (!attr) {
      NC_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit));
      attr = true;
    }
    int occ = 1;
    NC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem));
    int64_t blocks = (n + kThreads - 1) / kThreads;
    const int64_t max_blocks = (int64_t)sms * (occ > 0 ? occ : 1);   // one resident wave, grid-stride
    if (blocks > max_blocks) blocks = max_blocks;
    kernel<<<(unsigned)blocks, kThreads, smem, st>>>(ei, ej, ep, w, asg, n, n_gpus, lsb0, n_digits, copies, out, w0,
                                                   asg8);
  } else if (kRec != kSplit) {
    nc_set_error("traffic histogram: %d GPUs x %d digits do not fit in shared memory (packed / uniform path)",
                 n_gpus, n_digits);
    return NC_E_ARG;
  } else {
    int64_t blocks = (n + kThreads - 1) / kThreads;
    if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
    k_histogram_global<Idx><<<(unsigned)blocks, kThreads, 0, st>>>(ei, ej, ep, w, asg, n, n_gpus, lsb0, n_digits,
                                                                     out);
  }
  NC_LAUNCH_CHECK();
  return NC_OK;
}

// PartitionMap.assignment (any integer width, widened to int64 on the way in) -> uint8
// gpu ids for the uniform-weight K5, per-GPU neuron counts, and a flag for values outside
// [0, n_gpus) (stored as 0 so the histogram's cell index stays in range; the caller
// raises after the one read-back).
__global__ void k_assignment_u8(const int64_t* __restrict__ a, int64_t n, int n_gpus, uint8_t* __restrict__ out,
                                unsigned long long* __restrict__ counts, unsigned long long* __restrict__ bad) {
  __shared__ unsigned int hist[256];
  for (int k = threadIdx.x; k < n_gpus; k += blockDim.x) hist[k] = 0u;
  __syncthreads();
  bool oob = false;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = __ldcs(a + k);
    const bool ok = v >= 0 && v < n_gpus;
    oob |= !ok;
    out[k] = ok ? (uint8_t)v : (uint8_t)0;
    if (ok) atomicAdd(&hist[v], 1u);
  }
  if (__any_sync(0xffffffffu, oob) && (threadIdx.x & 31) == 0) atomicOr(bad, 1ull);
  __syncthreads();
  for (int k = threadIdx.x; k < n_gpus; k += blockDim.x)
    if (hist[k]) atomicAdd(counts + k, (unsigned long long)hist[k]);
}

}  // namespace

extern "C" int nc_traffic_exponents(const int64_t* edge_i, const int64_t* edge_j, const double* edge_p,
                                    const double* weights, int64_t n_edges, int32_t* out_minmax,
                                    void* stream) {
  if (n_edges <= 0) return NC_OK;
  if ((edge_i == nullptr) != (edge_j == nullptr)) {
    nc_set_error("nc_traffic_exponents: edge_i/edge_j must both be set or both NULL");
    return NC_E_ARG;
  }
  int64_t blocks = (n_edges + kThreads - 1) / kThreads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_exponents<<<(unsigned)blocks, kThreads, 0, (cudaStream_t)stream>>>(edge_i, edge_j, edge_p, weights,
                                                                        n_edges, out_minmax);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_traffic_histogram(const int64_t* edge_i, const int64_t* edge_j, const double* edge_p,
                                    const double* weights, const int64_t* assignment, int64_t n_edges,
                                    int32_t n_gpus, int32_t lsb_exponent, int32_t n_digits,
                                    unsigned long long* pg_limbs, void* stream) {
  if (n_gpus < 1 || n_digits < 3 || !edge_i || !edge_j) {
    nc_set_error("nc_traffic_histogram: bad arguments (n_gpus=%d n_digits=%d)", n_gpus, n_digits);
    return NC_E_ARG;
  }
  return launch_hist(edge_i, edge_j, edge_p, weights, assignment, n_edges, n_gpus, lsb_exponent,
                     n_digits, pg_limbs, (cudaStream_t)stream);
}

extern "C" int nc_traffic_histogram32(const int32_t* edge_i, const int32_t* edge_j, const double* edge_p,
                                      const double* weights, const int32_t* assignment, int64_t n_edges,
                                      int32_t n_gpus, int32_t lsb_exponent, int32_t n_digits,
                                      unsigned long long* pg_limbs, void* stream) {
  if (n_gpus < 1 || n_digits < 3 || !edge_i || !edge_j) {
    nc_set_error("nc_traffic_histogram32: bad arguments (n_gpus=%d n_digits=%d)", n_gpus, n_digits);
    return NC_E_ARG;
  }
  return launch_hist(edge_i, edge_j, edge_p, weights, assignment, n_edges, n_gpus, lsb_exponent, n_digits,
                     pg_limbs, (cudaStream_t)stream);
}

extern "C" int nc_traffic_histogram_packed(const int32_t* edge_i, const int32_t* edge_j, const double* edge_p,
                                           const void* neuron_records, int64_t n_edges, int32_t n_gpus,
                                           int32_t lsb_exponent, int32_t n_digits, unsigned long long* pg_limbs,
                                           void* stream) {
  if (n_gpus < 1 || n_digits < 3 || !edge_i || !edge_j || !neuron_records) {
    nc_set_error("nc_traffic_histogram_packed: bad arguments (n_gpus=%d n_digits=%d)", n_gpus, n_digits);
    return NC_E_ARG;
  }
  return launch_hist<int32_t, kPacked>(edge_i, edge_j, edge_p, reinterpret_cast<const double*>(neuron_records),
                                    nullptr, n_edges, n_gpus, lsb_exponent, n_digits, pg_limbs,
                                    (cudaStream_t)stream);
}

extern "C" int nc_traffic_histogram_uniform(const int32_t* edge_i, const int32_t* edge_j, const double* edge_p,
                                            double weight, const uint8_t* assignment, int64_t n_edges, int32_t n_gpus,
                                            int32_t lsb_exponent, int32_t n_digits, unsigned long long* pg_limbs,
                                            void* stream) {
  if (n_gpus < 1 || n_gpus > 256 || n_digits < 3 || !edge_i || !edge_j || !assignment) {
    nc_set_error("nc_traffic_histogram_uniform: bad arguments (n_gpus=%d n_digits=%d)", n_gpus, n_digits);
    return NC_E_ARG;
  }
  return launch_hist<int32_t, kUniform, NC_K5_UNIFORM_UNROLL>(edge_i, edge_j, edge_p, nullptr, nullptr, n_edges, n_gpus,
                                                          lsb_exponent, n_digits, pg_limbs, (cudaStream_t)stream,
                                                          weight, assignment);
}

extern "C" int nc_assignment_u8(const int64_t* assignment, int64_t n_neurons, int32_t n_gpus, uint8_t* out,
                                unsigned long long* counts, unsigned long long* bad, void* stream) {
  if (n_gpus < 1 || n_gpus > 256 || n_neurons < 0 || (n_neurons && (!assignment || !out)) || !counts || !bad) {
    nc_set_error("nc_assignment_u8: bad arguments (n_gpus=%d)", n_gpus);
    return NC_E_ARG;
  }
  if (n_neurons == 0) return NC_OK;
  int64_t blocks = (n_neurons + 1023) / 1024;
  if (blocks > 148 * 4) blocks = 148 * 4;
  k_assignment_u8<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(assignment, n_neurons, n_gpus, out, counts, bad);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_traffic_histogram_generated(const nc_graphgen_t* g, const double* weights, const int32_t* assignment,
                                              int64_t row_begin, int64_t row_end, int32_t n_gpus,
                                              int32_t lsb_exponent, int32_t n_digits, unsigned long long* pg_limbs,
                                              void* stream) {
  if (!g || g->n_neurons < 1 || g->n_communities < 1 || g->n_communities > g->n_neurons || !assignment ||
      n_gpus < 1 || n_digits < 3 || row_begin < 0 || row_end > g->n_neurons || !pg_limbs) {
    nc_set_error("nc_traffic_histogram_generated: bad arguments");
    return NC_E_ARG;
  }
  if (row_end <= row_begin) return NC_OK;
  const int cstride = copy_stride(smem_cells(true, n_gpus), n_digits);
  int copies = 32;
  while (copies > 1 && (size_t)copies * cstride * sizeof(unsigned int) > kSmemBudget) copies >>= 1;
  const size_t smem = (size_t)copies * cstride * sizeof(unsigned int);
  if (smem > kSmemLimit) {
    nc_set_error("nc_traffic_histogram_generated: %d GPUs x %d digits do not fit in shared memory", n_gpus,
                 n_digits);
    return NC_E_ARG;
  }
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  NC_CUDA_TRY(cudaFuncSetAttribute(k_histogram_generated, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kSmemLimit));
  NC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_histogram_generated, kThreads, smem));
  // rows carry very different numbers of edges (the first rows of a community enumerate
  // the most): many small blocks, grid-stride over rows
  int64_t blocks = (row_end - row_begin + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)sms * (occ > 0 ? occ : 1) * 4;
  if (blocks > cap) blocks = cap;
  k_histogram_generated<<<(unsigned)blocks, kThreads, smem, (cudaStream_t)stream>>>(
      *g, weights, assignment, row_begin, row_end, n_gpus, lsb_exponent, n_digits, copies, pg_limbs);
  NC_LAUNCH_CHECK();
  return NC_OK;
}

extern "C" int nc_weight_histogram(const double* weights, const int64_t* assignment, int64_t n_neurons,
                                   int32_t n_gpus, int32_t lsb_exponent, int32_t n_digits,
                                   unsigned long long* wg_limbs, void* stream) {
  if (n_gpus < 1 || n_digits < 3) {
    nc_set_error("nc_weight_histogram: bad arguments");
    return NC_E_ARG;
  }
  // same kernel with one cell per GPU (cell = assignment[k]), binned_sums semantics
  return launch_hist<int64_t>(nullptr, nullptr, nullptr, weights, assignment, n_neurons, n_gpus, lsb_exponent,
                              n_digits, wg_limbs, (cudaStream_t)stream);
}
