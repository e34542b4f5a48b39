// Indexed max-heap of the K6 greedy fill (greedy_fill.cpp, graphgen_host.cpp):
// the reference's lazy heapq of (-score, -w, idx) snapshots has, as its valid
// top, exactly the maximum of (score, weight, -index) over touched free items,
// which this heap keeps with increase-key in O(M) entries.
#pragma once
#include <cstdint>
#include <vector>

namespace ncgreedy {

struct IndexedHeap {
  int64_t top() const { return heap.empty() ? -1 : heap[0]; }
  const double* score;
  const double* weight;
  std::vector<int64_t> heap;   // item ids
  std::vector<int64_t> pos;    // position of item in heap, -1 if absent

  explicit IndexedHeap(int64_t n, const double* s, const double* w)
      : score(s), weight(w), pos(n, -1) { heap.reserve(1024); }

  // a ranks above b
  inline bool above(int64_t a, int64_t b) const {
    double sa = score[a], sb = score[b];
    if (sa != sb) return sa > sb;
    double wa = weight[a], wb = weight[b];
    if (wa != wb) return wa > wb;
    return a < b;
  }
  inline void place(size_t k, int64_t item) { heap[k] = item; pos[item] = (int64_t)k; }
  void sift_up(size_t k) {
    int64_t item = heap[k];
    while (k > 0) {
      size_t parent = (k - 1) >> 1;
      if (!above(item, heap[parent])) break;
      place(k, heap[parent]);
      k = parent;
    }
    place(k, item);
  }
  void sift_down(size_t k) {
    int64_t item = heap[k];
    size_t n = heap.size();
    for (;;) {
      size_t c = 2 * k + 1;
      if (c >= n) break;
      if (c + 1 < n && above(heap[c + 1], heap[c])) ++c;
      if (!above(heap[c], item)) break;
      place(k, heap[c]);
      k = c;
    }
    place(k, item);
  }
  // score[item] changed (or item is new); contributions are positive in every
  // reference caller, but restore the heap in both directions regardless
  void touch(int64_t item) {
    if (pos[item] < 0) {
      heap.push_back(item);
      pos[item] = (int64_t)heap.size() - 1;
    }
    sift_up((size_t)pos[item]);
    sift_down((size_t)pos[item]);
  }
  void remove(int64_t item) {
    int64_t k = pos[item];
    if (k < 0) return;
    pos[item] = -1;
    int64_t last = heap.back();
    heap.pop_back();
    if (last == item) return;
    heap[k] = last;
    pos[last] = k;
    sift_up((size_t)k);
    sift_down((size_t)pos[last]);
  }
  void clear() {
    for (int64_t it : heap) pos[it] = -1;
    heap.clear();
  }
};

}  // namespace ncgreedy
