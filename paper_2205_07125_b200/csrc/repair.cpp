// Native GA balance repair (replaces _repair_balance, partition.py:167-184).
//
// The reference loops: per-GPU load = math.fsum of its members' weights (the
// correctly rounded exact sum); if the heaviest GPU (lowest index on ties) is
// over `bound`, move its heaviest neuron (lowest index on ties) to the lightest
// GPU (lowest index on ties); repeat.  Each move re-sums everything.
//
// Here every GPU keeps its exact load as a fixed-point integer (base-2^32
// digits over the common least significant bit of all weights), updated by
// one add and one subtract per move and rounded to the nearest double
// (round-half-even, = fsum) for the comparisons, and a max-heap of its members
// ordered (weight desc, index asc).  Same decisions, O(log M) per move.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <vector>

#include "nc_common.h"

namespace {

using u64 = uint64_t;
using u128 = unsigned __int128;

struct Fixed {
  int lsb = 0;        // exponent of digit 0's least significant bit
  int nd = 0;         // digits per accumulator
};

// weight -> (53-bit integer mantissa, exponent of its lsb)
inline void split(double w, u64& mant, int& e) {
  int ex = 0;
  const double f = std::frexp(w, &ex);          // w = f * 2^ex, f in [0.5, 1)
  mant = (u64)std::ldexp(f, 53);                // exact
  e = ex - 53;
}

// acc += (sign) * (mant << (e - lsb)) on base-2^32 digits (normalised; no underflow by construction)
void add(std::vector<u64>& acc, u64 mant, int e, const Fixed& fx, bool subtract) {
  const int sh = e - fx.lsb;
  int d = sh / 32;
  const int b = sh % 32;
  u128 v = (u128)mant << b;                     // < 2^85
  u64 carry = 0;
  int64_t borrow = 0;
  for (int k = d; k < fx.nd; ++k) {
    const u64 part = (u64)(v & 0xFFFFFFFFu);
    v >>= 32;
    if (!subtract) {
      const u64 s = acc[k] + part + carry;
      acc[k] = s & 0xFFFFFFFFu;
      carry = s >> 32;
      if (v == 0 && carry == 0) break;
    } else {
      int64_t s = (int64_t)acc[k] - (int64_t)part - borrow;
      borrow = 0;
      if (s < 0) {
        s += (int64_t)1 << 32;
        borrow = 1;
      }
      acc[k] = (u64)s;
      if (v == 0 && borrow == 0) break;
    }
  }
}

// correctly rounded (half-even) value of the accumulator
double to_double(const std::vector<u64>& acc, const Fixed& fx) {
  int t = fx.nd - 1;
  while (t >= 0 && acc[t] == 0) --t;
  if (t < 0) return 0.0;
  u128 top = 0;
  int base = 0;                                 // exponent (in digits) of top's lowest digit
  bool sticky = false;
  if (t >= 2) {
    top = ((u128)acc[t] << 64) | ((u128)acc[t - 1] << 32) | acc[t - 2];
    base = t - 2;
    for (int k = 0; k < t - 2; ++k)
      if (acc[k]) sticky = true;
  } else {
    for (int k = t; k >= 0; --k) top = (top << 32) | acc[k];
    base = 0;
  }
  int len = 0;
  for (u128 x = top; x; x >>= 1) ++len;
  const int exp0 = base * 32 + fx.lsb;
  if (len <= 53) return std::ldexp((double)(u64)top, exp0);
  const int shift = len - 53;
  u64 mant = (u64)(top >> shift);
  const u128 rem = top & (((u128)1 << shift) - 1);
  const u128 half = (u128)1 << (shift - 1);
  if (rem > half || (rem == half && (sticky || (mant & 1)))) ++mant;
  return std::ldexp((double)mant, exp0 + shift);  // mant may be 2^53: still exact in a double
}

struct Item {
  double w;
  int64_t i;
  bool operator<(const Item& o) const {   // priority_queue top = largest weight, then smallest index
    if (w != o.w) return w < o.w;
    return i > o.i;
  }
};

}  // namespace

extern "C" int nc_repair_balance(int64_t m, const double* weights, int64_t* assignment, int32_t n_gpus, double bound,
                                 int64_t* n_moves) {
  if (m < 0 || n_gpus < 1 || (m > 0 && (!weights || !assignment))) {
    nc_set_error("nc_repair_balance: bad arguments");
    return NC_E_ARG;
  }
  if (n_moves) *n_moves = 0;
  if (m == 0) return NC_OK;
  Fixed fx;
  int lo_e = 1 << 30, hi_e = -(1 << 30);
  for (int64_t k = 0; k < m; ++k) {
    const double w = weights[k];
    if (!(w > 0.0) || !std::isfinite(w)) {
      nc_set_error("nc_repair_balance: weights must be finite and > 0");
      return NC_E_ARG;
    }
    u64 mt;
    int e;
    split(w, mt, e);
    lo_e = std::min(lo_e, e);
    hi_e = std::max(hi_e, e + 53);
    if (assignment[k] < 0 || assignment[k] >= n_gpus) {
      nc_set_error("nc_repair_balance: assignment out of range");
      return NC_E_ARG;
    }
  }
  int growth = 1;
  while (((int64_t)1 << growth) <= m) ++growth;
  fx.lsb = lo_e;
  fx.nd = (hi_e - lo_e + growth + 31) / 32 + 2;
  std::vector<std::vector<u64>> acc(n_gpus, std::vector<u64>(fx.nd, 0));
  std::vector<std::priority_queue<Item>> heap(n_gpus);
  for (int64_t k = 0; k < m; ++k) {
    u64 mt;
    int e;
    split(weights[k], mt, e);
    add(acc[assignment[k]], mt, e, fx, false);
    heap[assignment[k]].push({weights[k], k});
  }
  std::vector<double> load(n_gpus);
  for (int g = 0; g < n_gpus; ++g) load[g] = to_double(acc[g], fx);
  int64_t moves = 0;
  for (;;) {
    int hi = 0, lo = 0;
    for (int g = 1; g < n_gpus; ++g) {
      if (load[g] > load[hi]) hi = g;   // first maximum (np.argmax)
      if (load[g] < load[lo]) lo = g;   // first minimum (np.argmin)
    }
    if (load[hi] <= bound || hi == lo) break;
    const Item it = heap[hi].top();
    heap[hi].pop();
    heap[lo].push(it);
    u64 mt;
    int e;
    split(it.w, mt, e);
    add(acc[hi], mt, e, fx, true);
    add(acc[lo], mt, e, fx, false);
    load[hi] = to_double(acc[hi], fx);
    load[lo] = to_double(acc[lo], fx);
    assignment[it.i] = lo;
    ++moves;
  }
  if (n_moves) *n_moves = moves;
  return NC_OK;
}
