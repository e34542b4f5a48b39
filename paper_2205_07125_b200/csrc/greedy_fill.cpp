// K6: capacity-bounded greedy bucket fill (host C++).
//
// Semantics: neurocomm greedy.py:55-117 (rules in its docstring :9-21).
//   * buckets 0..n-2 are filled one at a time, the last takes the rest (:116);
//   * per bucket the affinity score of every item restarts at 0 (:82);
//   * the next candidate is the free item with the largest
//     (score, weight, -index) among items touched by this bucket (:87-93);
//     if none was touched, the heaviest free item in (weight desc, index asc)
//     order (:74, :94-97);
//   * a seeded bucket refuses a candidate whose weight would push it over
//     `capacity` and closes (:99-100) -- the candidate stays free;
//   * a bucket also closes once only `needed_later` items are left (:81, :86);
//   * assigning v adds values[e] to score[u] for every free neighbour u in v's
//     CSR row, in row order, with plain fp64 adds (:106-114).
// The reference keeps a lazy heapq of (-score, -w, idx) snapshots and discards
// stale entries on pop; its valid top is exactly the maximum of the key above
// over touched free items, so an indexed max-heap with increase-key selects the
// same item while holding O(M) entries instead of O(E).
//
// numpy's `score[nbrs] += vals` reads every score before writing any, so a
// repeated neighbour inside one row only keeps its last update; the row pass
// below reproduces that with a read-all-then-write-all loop.

#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <numeric>

#include "nc_common.h"
#include "k6_heap.h"

using ncgreedy::IndexedHeap;

extern "C" int nc_greedy_fill(int64_t m, const double* weights, const int64_t* indptr,
                              const int64_t* indices, const double* values, int32_t n_buckets,
                              double capacity, int64_t* assignment) {
  if (m < 1 || n_buckets < 1 || n_buckets > m) {
    nc_set_error("nc_greedy_fill: n_buckets must be in [1, %lld], got %d", (long long)m, n_buckets);
    return NC_E_ARG;
  }
  std::vector<double> score(m, 0.0);
  std::vector<uint8_t> free_(m, 1);
  // fallback order: weight descending, index ascending (greedy.py:74)
  std::vector<int64_t> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return weights[a] > weights[b]; });
  for (int64_t k = 0; k < m; ++k) assignment[k] = -1;

  IndexedHeap heap(m, score.data(), weights);
  std::vector<int64_t> touched;       // items whose score was written this bucket (each once)
  std::vector<int32_t> touched_in(m, -1);   // bucket that last wrote the item's score
  std::vector<int64_t> row_items;
  std::vector<double> row_new;
  int64_t cursor = 0;
  int64_t left = m;

  for (int32_t b = 0; b + 1 < n_buckets; ++b) {
    const int64_t reserve = n_buckets - 1 - b;
    for (int64_t it : touched) score[it] = 0.0;
    touched.clear();
    heap.clear();
    double load = 0.0;
    bool seeded = false;
    while (left > reserve) {
      int64_t pick;
      if (!heap.heap.empty()) {
        pick = heap.heap[0];
      } else {
        while (!free_[order[cursor]]) ++cursor;
        pick = order[cursor];
      }
      const double w = weights[pick];
      if (seeded && load + w > capacity) break;
      assignment[pick] = b;
      free_[pick] = 0;
      heap.remove(pick);
      --left;
      seeded = true;
      load += w;
      const int64_t lo = indptr[pick], hi = indptr[pick + 1];
      row_items.clear();
      row_new.clear();
      for (int64_t e = lo; e < hi; ++e) {
        const int64_t u = indices[e];
        if (!free_[u]) continue;
        row_items.push_back(u);
        row_new.push_back(score[u] + values[e]);
      }
      // write one score and restore the heap before the next (the heap
      // invariant only survives one changed key at a time)
      for (size_t k = 0; k < row_items.size(); ++k) {
        score[row_items[k]] = row_new[k];
        if (touched_in[row_items[k]] != b) {   // once per item and bucket: the list stays O(M)
          touched_in[row_items[k]] = b;
          touched.push_back(row_items[k]);
        }
        heap.touch(row_items[k]);
      }
    }
  }
  for (int64_t k = 0; k < m; ++k)
    if (free_[k]) assignment[k] = n_buckets - 1;
  return NC_OK;
}
