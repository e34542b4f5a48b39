// Host side of the SBM generator, for the planner (SURVEY 8(a) row a3 at scale).
//
// The reference partitions a NeuronGraph with partition_greedy
// (partition.py:95-114 -> greedy.py:32-117): symmetric CSR of the edges
// (adjacency_from_edges: int64 index + fp64 value per entry, two entries per
// edge), then the sequential greedy fill.  At config 3 (1e7 neurons, 5e9
// edges) the NeuronGraph alone is 120 GB and its CSR 160 GB, so here the fill
// runs straight off the generator instead:
//   * upper part of row r (pairs (r, j > r), ascending j): regenerated on
//     demand from r's own counter-based streams (the same Philox gap sampler as
//     csrc/graphgen.cu for_each_upper, same fp64 arithmetic), never stored;
//   * lower part (pairs (i < r, r), ascending i): the transpose, materialised
//     once as int32 ids (4 B per edge) by a parallel count / prefix / fill;
//   * values (p * W_i) * W_j with p recomputed from the edge's own Philox
//     counter (graphgen.cu edge_q), W = 1 when no weights are given.
// Row order and values are exactly adjacency_from_edges' on the materialised
// graph, so the fill (the same indexed-heap K6 as greedy_fill.cpp) returns the
// reference's assignment bit for bit (tests/test_planner_parity.py checks it
// against the materialised path).  The device generator uses CUDA's log1p, this
// file glibc's; bench.py's parity leg checks the two build the same network.

#include <atomic>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>
#include <numeric>
#include <algorithm>

#include "nc_common.h"
#include "philox.cuh"
#include "k6_heap.h"

namespace {

struct HostGen {
  int64_t n, c, q, r, big;
  double p_in, p_out, ilo, ihi, olo, ohi;
  uint64_t seed;
  explicit HostGen(const nc_graphgen_t& g)
      : n(g.n_neurons), c(g.n_communities), q(g.n_neurons / g.n_communities), r(g.n_neurons % g.n_communities),
        big((g.n_neurons % g.n_communities) * (g.n_neurons / g.n_communities + 1)), p_in(g.p_in), p_out(g.p_out),
        ilo(g.intra_lo), ihi(g.intra_hi), olo(g.inter_lo), ohi(g.inter_hi), seed(g.seed) {}
  int64_t of(int64_t i) const { return i < big ? i / (q + 1) : r + (i - big) / q; }
  int64_t start(int64_t b) const { return b < r ? b * (q + 1) : big + (b - r) * q; }
  int64_t size(int64_t b) const { return b < r ? q + 1 : q; }
};

inline double u53(uint32_t a, uint32_t b) { return (double)(((uint64_t)a << 21) ^ (uint64_t)(b >> 11)) * 0x1.0p-53; }

// p of edge (i, j), i < j: graphgen.cu edge_q before the quantisation
inline double edge_p(const HostGen& g, int64_t i, int64_t j, bool intra) {
  nc_u32x4 c = {(uint32_t)i, (uint32_t)j, NC_TAG_EDGEP, (uint32_t)((i >> 32) ^ ((j >> 32) << 16))};
  nc_u32x4 x = nc_philox4x32_10(c, (uint32_t)g.seed, (uint32_t)(g.seed >> 32));
  const double lo = intra ? g.ilo : g.olo, hi = intra ? g.ihi : g.ohi;
  return lo + (hi - lo) * u53(x.x, x.y);
}

// f(j, intra) for every upper neighbour j of row i, ascending (graphgen.cu for_each_upper)
template <typename F>
void for_each_upper(const HostGen& g, int64_t i, F&& f) {
  const int64_t ci = g.of(i);
  for (int64_t b = ci; b < g.c; ++b) {
    const bool intra = (b == ci);
    const double p = intra ? g.p_in : g.p_out;
    if (p <= 0.0) continue;
    const int64_t first = intra ? i + 1 : g.start(b);
    const int64_t n = intra ? g.start(ci) + g.size(ci) - i - 1 : g.size(b);
    if (n <= 0) continue;
    if (p >= 1.0) {
      for (int64_t t = 0; t < n; ++t) f(first + t, intra);
      continue;
    }
    const uint32_t k0 = (uint32_t)g.seed, k1 = (uint32_t)(g.seed >> 32);
    const double inv = 1.0 / std::log1p(-p);
    uint32_t ctr = 0;
    nc_u32x4 buf{};
    int avail = 0;
    int64_t pos = -1;
    for (;;) {
      if (avail == 0) {
        buf = nc_philox4x32_10(nc_u32x4{(uint32_t)i, (uint32_t)b, ctr++, NC_TAG_GAPS}, k0, k1);
        avail = 2;
      }
      const double u = (avail == 2) ? u53(buf.x, buf.y) : u53(buf.z, buf.w);
      --avail;
      const double gf = std::floor(std::log1p(-u) * inv);
      pos += (gf >= 9.0e18) ? INT64_MAX / 4 : (int64_t)gf + 1;
      if (pos >= n) break;
      f(first + pos, intra);
    }
  }
}

int n_threads(int32_t t) {
  if (t > 0) return t;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

// Contiguous row ranges of about equal generator work (expected upper neighbours
// per row: rows early in a community / the id range enumerate more).
std::vector<int64_t> balanced_ranges(const HostGen& g, int threads) {
  std::vector<double> cum(g.n + 1, 0.0);
  for (int64_t i = 0; i < g.n; ++i) {
    const int64_t ci = g.of(i);
    const double later = (double)(g.n - g.start(ci) - g.size(ci));
    cum[i + 1] = cum[i] + 1.0 + g.p_in * (double)(g.start(ci) + g.size(ci) - i - 1) + g.p_out * later;
  }
  std::vector<int64_t> cut(threads + 1, g.n);
  cut[0] = 0;
  int64_t i = 0;
  for (int t = 1; t < threads; ++t) {
    const double target = cum[g.n] * t / threads;
    while (i < g.n && cum[i] < target) ++i;
    cut[t] = i;
  }
  return cut;
}

template <typename F>
void parallel_rows(const std::vector<int64_t>& cut, F&& f) {   // f(thread, row_begin, row_end)
  std::vector<std::thread> ts;
  const int threads = (int)cut.size() - 1;
  for (int t = 0; t < threads; ++t) ts.emplace_back([&, t] { f(t, cut[t], cut[t + 1]); });
  for (auto& th : ts) th.join();
}

// even split (work per row is uniform)
std::vector<int64_t> even_ranges(int64_t n, int threads) {
  std::vector<int64_t> cut(threads + 1);
  for (int t = 0; t <= threads; ++t) cut[t] = n * t / threads;
  return cut;
}

bool spec_ok(const nc_graphgen_t* g) {
  return g && g->n_neurons >= 1 && g->n_neurons < (int64_t(1) << 31) && g->n_communities >= 1 &&
         g->n_communities <= g->n_neurons;
}

}  // namespace

// Edges of the generated network as a NeuronGraph holds them (ascending (i, j),
// i < j, p in fp64).  NULL arrays: returns the edge count only.
extern "C" int64_t nc_hostgen_edges(const nc_graphgen_t* spec, int64_t* edge_i, int64_t* edge_j, double* edge_p_out,
                                    int32_t threads) {
  if (!spec_ok(spec)) {
    nc_set_error("nc_hostgen_edges: invalid generator spec");
    return -1;
  }
  const HostGen g(*spec);
  const std::vector<int64_t> cut = balanced_ranges(g, n_threads(threads));
  std::vector<int64_t> up(g.n + 1, 0);
  parallel_rows(cut, [&](int, int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
      int64_t k = 0;
      for_each_upper(g, i, [&](int64_t, bool) { ++k; });
      up[i + 1] = k;
    }
  });
  std::partial_sum(up.begin(), up.end(), up.begin());
  if (edge_i && edge_j && edge_p_out) {
    parallel_rows(cut, [&](int, int64_t a, int64_t b) {
      for (int64_t i = a; i < b; ++i) {
        int64_t k = up[i];
        for_each_upper(g, i, [&](int64_t j, bool intra) {
          edge_i[k] = i;
          edge_j[k] = j;
          edge_p_out[k] = edge_p(g, i, j, intra);
          ++k;
        });
      }
    });
  }
  return up[g.n];
}

// K6 (greedy.py:55-117 over adjacency_from_edges' CSR of the generated network)
// without materialising the graph; see the header comment.  weights: NULL = 1.
extern "C" int nc_greedy_fill_generated(const nc_graphgen_t* spec, const double* weights, int32_t n_buckets,
                                        double capacity, int64_t* assignment, int32_t threads) {
  if (!spec_ok(spec)) {
    nc_set_error("nc_greedy_fill_generated: invalid generator spec (1 <= n_neurons < 2^31)");
    return NC_E_ARG;
  }
  const HostGen g(*spec);
  const int64_t m = g.n;
  if (n_buckets < 1 || n_buckets > m) {
    nc_set_error("nc_greedy_fill_generated: n_buckets must be in [1, %lld], got %d", (long long)m, n_buckets);
    return NC_E_ARG;
  }
  const int T = n_threads(threads);
  const std::vector<int64_t> cut = balanced_ranges(g, T);
  // ---- lower part: ids i < r with r in upper(i), ascending i, int32.  The sources
  // are cut into C contiguous chunks of equal generator work (C = 8 x threads, taken
  // dynamically by the threads: early chunks scatter over every target row and run
  // slower); per-chunk counts per target row give every chunk its own run inside
  // each target row, so the runs are in source order.
  const std::vector<int64_t> ccut = balanced_ranges(g, 8 * T);
  const int Cn = (int)ccut.size() - 1;
  std::vector<std::vector<int32_t>> cnt(Cn);
  auto each_chunk = [&](auto&& f) {   // f(chunk, row_begin, row_end) over the chunks, dynamically
    std::atomic<int> next{0};
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
      ts.emplace_back([&] {
        for (int c = next++; c < Cn; c = next++) f(c, ccut[c], ccut[c + 1]);
      });
    for (auto& th : ts) th.join();
  };
  each_chunk([&](int c, int64_t a, int64_t b) {
    std::vector<int32_t>& k = cnt[c];
    k.assign(m, 0);
    for (int64_t i = a; i < b; ++i) for_each_upper(g, i, [&](int64_t j, bool) { ++k[j]; });
  });
  std::vector<int64_t> lptr(m + 1, 0);
  // cnt[c][j] -> start of chunk c's run in row j (relative); lptr[j + 1] = row length
  parallel_rows(even_ranges(m, T), [&](int, int64_t a, int64_t b) {
    for (int64_t j = a; j < b; ++j) {
      int32_t run = 0;
      for (int c = 0; c < Cn; ++c) {
        const int32_t n = cnt[c][j];
        cnt[c][j] = run;
        run += n;
      }
      lptr[j + 1] = run;
    }
  });
  std::partial_sum(lptr.begin(), lptr.end(), lptr.begin());
  std::vector<int32_t> lower((size_t)lptr[m]);
  each_chunk([&](int c, int64_t a, int64_t b) {
    std::vector<int32_t>& off = cnt[c];
    for (int64_t i = a; i < b; ++i)
      for_each_upper(g, i, [&](int64_t j, bool) { lower[(size_t)(lptr[j] + off[j]++)] = (int32_t)i; });
    off.clear();
    off.shrink_to_fit();
  });
  cnt.clear();
  cnt.shrink_to_fit();

  // ---- the fill: greedy_fill.cpp's loop with rows from the generator + `lower`
  auto W = [&](int64_t i) { return weights ? weights[i] : 1.0; };
  std::vector<double> wv;
  const double* wp = weights;
  if (!wp) {
    wv.assign(m, 1.0);
    wp = wv.data();
  }
  std::vector<double> score(m, 0.0);
  std::vector<uint8_t> free_(m, 1);
  std::vector<int64_t> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return wp[a] > wp[b]; });
  for (int64_t k = 0; k < m; ++k) assignment[k] = -1;
  ncgreedy::IndexedHeap heap(m, score.data(), wp);
  std::vector<int64_t> touched, row_items, nbr;
  std::vector<int32_t> touched_in(m, -1);   // bucket that last wrote the item's score
  std::vector<double> row_new;
  int64_t cursor = 0, left = m;
  for (int32_t b = 0; b + 1 < n_buckets; ++b) {
    const int64_t reserve = n_buckets - 1 - b;
    for (int64_t it : touched) score[it] = 0.0;
    touched.clear();
    heap.clear();
    double load = 0.0;
    bool seeded = false;
    while (left > reserve) {
      int64_t pick = heap.top();
      if (pick < 0) {
        while (!free_[order[cursor]]) ++cursor;
        pick = order[cursor];
      }
      const double w = wp[pick];
      if (seeded && load + w > capacity) break;
      assignment[pick] = b;
      free_[pick] = 0;
      heap.remove(pick);
      --left;
      seeded = true;
      load += w;
      row_items.clear();
      row_new.clear();
      // the row first (upper part regenerated, then the stored lower part), with the
      // per-item state of every neighbour prefetched: at 1e7 items those are cache misses
      // and the row's ~1 000 of them can be in flight together
      nbr.clear();
      for_each_upper(g, pick, [&](int64_t j, bool intra) { nbr.push_back(intra ? j : ~j); });
      const size_t n_up = nbr.size();
      for (int64_t e = lptr[pick]; e < lptr[pick + 1]; ++e) nbr.push_back(lower[(size_t)e]);
      for (int64_t x : nbr) {
        const int64_t u = x < 0 ? ~x : x;
        __builtin_prefetch(&free_[u]);
        __builtin_prefetch(&score[u]);
        __builtin_prefetch(&heap.pos[u]);
      }
      // pairs (pick, j > pick): value (p * W_pick) * W_j
      for (size_t k = 0; k < n_up; ++k) {
        const bool intra = nbr[k] >= 0;
        const int64_t j = intra ? nbr[k] : ~nbr[k];
        if (!free_[j]) continue;
        row_items.push_back(j);
        row_new.push_back(score[j] + (edge_p(g, pick, j, intra) * W(pick)) * W(j));
      }
      // pairs (i < pick, pick): value (p * W_i) * W_pick
      const int64_t ci = g.of(pick);
      for (size_t k = n_up; k < nbr.size(); ++k) {
        const int64_t i = nbr[k];
        if (!free_[i]) continue;
        row_items.push_back(i);
        row_new.push_back(score[i] + (edge_p(g, i, pick, g.of(i) == ci) * W(i)) * W(pick));
      }
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

// Host side of the edge upload (sim.upload_edges): NeuronGraph columns (int64 ids, fp64 p)
// narrowed into pinned staging buffers as the device takes them -- int32 ids and uint8
// weight units q = clamp(ceil(32 p), 1, 32) (sim.q_from_p) -- in one multi-threaded pass, so
// the copy engine moves 9 instead of 24 bytes per edge.  Endpoints outside [0, n_neurons)
// are an NC_E_ARG error (nothing is uploaded for the chunk).
extern "C" int nc_edges_narrow(const int64_t* edge_i, const int64_t* edge_j, const double* edge_p, int64_t n,
                               int64_t n_neurons, int32_t* out_i, int32_t* out_j, uint8_t* out_q,
                               int32_t threads) {
  if (n < 0 || (n && (!edge_i || !edge_j || !edge_p || !out_i || !out_j || !out_q)) || n_neurons < 1 ||
      n_neurons >= (int64_t(1) << 31)) {
    nc_set_error("nc_edges_narrow: bad arguments");
    return NC_E_ARG;
  }
  if (n == 0) return NC_OK;
  int T = n_threads(threads);
  if ((int64_t)T * 65536 > n) T = (int)std::max<int64_t>(1, n / 65536);
  const std::vector<int64_t> cut = even_ranges(n, T);
  std::vector<int> bad(T, 0);
  parallel_rows(cut, [&](int t, int64_t b, int64_t e) {
    int oob = 0;
    for (int64_t k = b; k < e; ++k) {
      const int64_t a = edge_i[k], c = edge_j[k];
      oob |= (a < 0) | (a >= n_neurons) | (c < 0) | (c >= n_neurons);
      out_i[k] = (int32_t)a;
      out_j[k] = (int32_t)c;
      double q = std::ceil(edge_p[k] * 32.0);
      q = q < 1.0 ? 1.0 : (q > 32.0 ? 32.0 : q);
      out_q[k] = (uint8_t)q;
    }
    bad[t] = oob;
  });
  for (int t = 0; t < T; ++t)
    if (bad[t]) {
      nc_set_error("edge endpoints outside [0, %lld)", (long long)n_neurons);
      return NC_E_ARG;
    }
  return NC_OK;
}
