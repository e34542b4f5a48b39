/*
 * sim_oracle.c -- CPU ORACLE for simulate(steps).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline -- never as a product path.
 *
 * PARITY UNPINNED against the reference: neurocomm (arXiv 2205.07125 pkg) has
 * no spiking dynamics at all (SPEC.md:13 puts LIF/IZH/HH out of scope; its only
 * "step" is the analytic netsim.step_latency, netsim.py:207-246).  This file is
 * the executable statement of the semantics DESIGN.md section 3 defines; it is
 * pinned instead by (1) known-answer vectors of Philox4x32-10, (2) an
 * independent numpy restatement (oracle/sim_numpy.py) that must agree bit for
 * bit, and (3) the committed golden rasters under tests/golden/.  The parts it
 * borrows from the reference are pinned there: the network is the reference's
 * NeuronGraph (model.py:53-92, each undirected edge = one synapse each way,
 * SPEC.md:110), the shards are PartitionMap.assignment (partition.py:60-65)
 * and the next hops come from RoutingTable src/dst/via (routing.py:61-115,
 * 211-222) with the bridge forwarding directly to the destination.
 *
 * Representation is deliberately unlike the engine's: global neuron ids, a
 * plain symmetric CSR (row = post, cols = pre), byte-per-neuron spike flags,
 * explicit per-neuron destination sets; no renumbering, packing or bitmaps.
 *
 * Build: make -C oracle   (gcc -O2 -ffp-contract=off -fopenmp; never -ffast-math)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  float alpha_v, alpha_i, beta, v_rest, v_reset, v_th, w_unit, w_ext, v_init_span;
  uint32_t ext_threshold;
  int32_t ext_lanes, t_ref, g_inh, inh_every;
  uint64_t seed;
} oracle_lif_t;

/* ---- Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) ------------------ */
static void philox(const uint32_t ctr[4], uint64_t seed, uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void oracle_philox(const uint32_t* ctr, uint64_t seed, uint32_t* out) { philox(ctr, seed, out); }

#define TAG_DRIVE 0xD21E0001u
#define TAG_VINIT 0x1417AB01u

static int inhibitory(int64_t gid, int32_t every) { return every > 0 && gid % every == every - 1; }

/* Initial membrane voltage: v_reset + u * span, u = top 24 bits / 2^24. */
static float v_initial(uint32_t gid, const oracle_lif_t* p) {
  uint32_t c[4] = {gid, 0xFFFFFFFFu, TAG_VINIT, 0u}, r[4];
  philox(c, p->seed, r);
  float u = (float)(r[0] >> 8) * 5.9604644775390625e-08f;
  return p->v_reset + u * p->v_init_span;
}

/* One neuron's update; returns 1 on a spike.  Every line is one IEEE fp32
 * operation in the order the engine uses (no contraction: -ffp-contract=off). */
static int lif(float* v, float* isyn, uint8_t* ref, int32_t acc, uint32_t gid, uint32_t step,
               const oracle_lif_t* p) {
  uint32_t ext_events = 0;
  if (p->ext_lanes > 0) {
    uint32_t c[4] = {gid, step, TAG_DRIVE, 0u}, r[4];
    philox(c, p->seed, r);
    for (int k = 0; k < p->ext_lanes && k < 4; ++k) ext_events += r[k] < p->ext_threshold;
  }
  float syn = (float)acc;
  float ext = (float)ext_events;
  float a = *isyn * p->alpha_i;
  float b = syn * p->w_unit;
  float i1 = a + b;
  float c = ext * p->w_ext;
  float inew = i1 + c;
  *isyn = inew;
  if (*ref > 0) {
    *ref -= 1;
    *v = p->v_reset;
    return 0;
  }
  float d = *v - p->v_rest;
  float e = d * p->alpha_v;
  float f = p->v_rest + e;
  float g = inew * p->beta;
  float vn = f + g;
  if (vn >= p->v_th) {
    *v = p->v_reset;
    *ref = (uint8_t)p->t_ref;
    return 1;
  }
  *v = vn;
  return 0;
}

/*
 * Run `steps` steps.  Inputs: symmetric CSR (rowptr[M+1], col[nnz] pre gids,
 * q[nnz] weight units 1..32), owner[M] shard of every neuron, next_hop[n*n]
 * (first hop of demand s->d, -1 if none).  Outputs (each may be NULL):
 *   raster[steps*M]  1 if neuron fired at that step
 *   deliv[steps*n*n] ids of shard s delivered at shard d (d hosts targets)
 *   hop[steps*n*n]   ids carried on channel u->v (first hop + relay hop)
 *   v_out/i_out[M]   final state
 * Returns 0, or -1 if a destination has no next hop in the table.
 */
int oracle_simulate(int64_t M, const int64_t* rowptr, const int32_t* col, const uint8_t* q,
                    const int32_t* owner, int32_t n, const int32_t* next_hop, const oracle_lif_t* p,
                    int32_t steps, int32_t n_threads, uint8_t* raster, int64_t* deliv, int64_t* hop,
                    float* v_out, float* i_out) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#else
  (void)n_threads;
#endif
  float* v = (float*)malloc(sizeof(float) * M);
  float* isyn = (float*)malloc(sizeof(float) * M);
  uint8_t* ref = (uint8_t*)calloc(M, 1);
  uint8_t* prev = (uint8_t*)calloc(M, 1);
  uint8_t* cur = (uint8_t*)calloc(M, 1);
  uint32_t* dests = (uint32_t*)calloc(M, sizeof(uint32_t));
  int rc = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(min : rc)
  for (int64_t i = 0; i < M; ++i) {
    v[i] = v_initial((uint32_t)i, p);
    isyn[i] = 0.0f;
    uint32_t m = 0;
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) m |= 1u << owner[col[k]];
    m &= ~(1u << owner[i]);
    dests[i] = m;
    for (int d = 0; d < n; ++d)
      if (((m >> d) & 1u) && next_hop[owner[i] * n + d] < 0) rc = -1;
  }
  if (rc == 0) {
    for (int32_t t = 0; t < steps; ++t) {
#pragma omp parallel for schedule(dynamic, 256)
      for (int64_t i = 0; i < M; ++i) {
        int32_t acc = 0;
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
          int32_t pre = col[k];
          if (prev[pre]) acc += inhibitory(pre, p->inh_every) ? -p->g_inh * (int32_t)q[k] : (int32_t)q[k];
        }
        cur[i] = (uint8_t)lif(&v[i], &isyn[i], &ref[i], acc, (uint32_t)i, (uint32_t)t, p);
      }
      if (raster) memcpy(raster + (int64_t)t * M, cur, (size_t)M);
      if (deliv || hop) {
        int64_t* D = deliv ? deliv + (int64_t)t * n * n : NULL;
        int64_t* H = hop ? hop + (int64_t)t * n * n : NULL;
        for (int64_t i = 0; i < M; ++i) {
          if (!cur[i] || !dests[i]) continue;
          const int s = owner[i];
          uint32_t first = 0;              /* distinct first hops */
          uint32_t relayed[32] = {0};      /* per relay: destinations behind it */
          for (int d = 0; d < n; ++d) {
            if (!((dests[i] >> d) & 1u)) continue;
            if (D) D[s * n + d] += 1;
            int h = next_hop[s * n + d];
            first |= 1u << h;
            if (h != d) relayed[h] |= 1u << d;
          }
          for (int h = 0; h < n; ++h) {
            if (!((first >> h) & 1u)) continue;
            if (H) H[s * n + h] += 1;
            for (int d = 0; d < n; ++d)
              if (H && ((relayed[h] >> d) & 1u)) H[h * n + d] += 1;
          }
        }
      }
      uint8_t* tmp = prev; prev = cur; cur = tmp;
    }
    if (v_out) memcpy(v_out, v, sizeof(float) * M);
    if (i_out) memcpy(i_out, isyn, sizeof(float) * M);
  }
  free(v); free(isyn); free(ref); free(prev); free(cur); free(dests);
  return rc;
}

/* ---- CPU network build for the reference arm (same algorithm as the device
 * generator csrc/graphgen.cu, restated: per (row, block) Philox stream,
 * geometric skipping in fp64 log1p, q = ceil(32 p)).  Builds the symmetric
 * gid-space CSR directly.  Communities are contiguous near-equal blocks. */
#include <math.h>

#define TAG_GAPS 0x6A950001u
#define TAG_EDGEP 0xE06E0001u

typedef struct {
  int64_t n, c, q, r, big;
  double p_in, p_out, ilo, ihi, olo, ohi;
  uint64_t seed;
} gen_t;

static int64_t g_comm(const gen_t* g, int64_t i) { return i < g->big ? i / (g->q + 1) : g->r + (i - g->big) / g->q; }
static int64_t g_start(const gen_t* g, int64_t c) { return c < g->r ? c * (g->q + 1) : g->big + (c - g->r) * g->q; }
static int64_t g_size(const gen_t* g, int64_t c) { return c < g->r ? g->q + 1 : g->q; }
static double u53(uint32_t a, uint32_t b) { return (double)((((uint64_t)a) << 21) ^ (uint64_t)(b >> 11)) * 0x1.0p-53; }

static uint8_t g_edge_q(const gen_t* g, int64_t i, int64_t j, int intra) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)j, TAG_EDGEP, (uint32_t)((i >> 32) ^ ((j >> 32) << 16))}, x[4];
  philox(c, g->seed, x);
  double lo = intra ? g->ilo : g->olo, hi = intra ? g->ihi : g->ohi;
  double p = lo + (hi - lo) * u53(x[0], x[1]);
  double qf = ceil(p * 32.0);
  if (qf < 1.0) qf = 1.0;
  if (qf > 32.0) qf = 32.0;
  return (uint8_t)qf;
}

/* visit upper neighbours of row i; mode 0: count into cnt_up/cnt_low, 1: fill */
static int64_t g_row(const gen_t* g, int64_t i, int mode, int64_t* low_cnt, const int64_t* rowptr,
                     int64_t* low_fill, int64_t* up_base, int32_t* col, uint8_t* q) {
  int64_t ci = g_comm(g, i), up = 0;
  for (int64_t b = ci; b < g->c; ++b) {
    int intra = (b == ci);
    double p = intra ? g->p_in : g->p_out;
    if (p <= 0.0) continue;
    int64_t first = intra ? i + 1 : g_start(g, b);
    int64_t n = intra ? g_start(g, ci) + g_size(g, ci) - i - 1 : g_size(g, b);
    if (n <= 0) continue;
    double inv = 1.0 / log1p(-p);
    uint32_t ctr = 0, buf[4];
    int avail = 0;
    int64_t pos = -1;
    for (;;) {
      int64_t gap;
      if (p >= 1.0) {
        gap = 1;
      } else {
        if (avail == 0) {
          uint32_t c[4] = {(uint32_t)i, (uint32_t)b, ctr++, TAG_GAPS};
          philox(c, g->seed, buf);
          avail = 2;
        }
        double u = (avail == 2) ? u53(buf[0], buf[1]) : u53(buf[2], buf[3]);
        --avail;
        double gf = floor(log1p(-u) * inv);
        gap = (gf >= 9.0e18) ? INT64_MAX / 4 : (int64_t)gf + 1;
      }
      pos += gap;
      if (pos >= n) break;
      int64_t j = first + pos;
      ++up;
      if (mode == 0) {
#pragma omp atomic
        low_cnt[j] += 1;
      } else {
        uint8_t qq = g_edge_q(g, i, j, intra);
        int64_t slot;
        col[*up_base] = (int32_t)j;
        q[*up_base] = qq;
        *up_base += 1;
#pragma omp atomic capture
        slot = low_fill[j]++;
        col[rowptr[j] + slot] = (int32_t)i;
        q[rowptr[j] + slot] = qq;
      }
    }
  }
  return up;
}

/* Two calls: with col == NULL returns nnz and fills rowptr[n+1]; then with
 * col/q allocated to nnz fills them.  Rows: [lower part (any order) | upper ascending]. */
int64_t oracle_generate_sbm(int64_t n, int64_t n_comm, double p_in, double p_out, double ilo, double ihi,
                            double olo, double ohi, uint64_t seed, int32_t n_threads, int64_t* rowptr,
                            int32_t* col, uint8_t* q) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#else
  (void)n_threads;
#endif
  gen_t g = {n, n_comm, n / n_comm, n % n_comm, (n % n_comm) * (n / n_comm + 1), p_in, p_out, ilo, ihi, olo,
             ohi, seed};
  int64_t* low = (int64_t*)calloc(n, sizeof(int64_t));
  int64_t* upc = (int64_t*)calloc(n, sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) upc[i] = g_row(&g, i, 0, low, NULL, NULL, NULL, NULL, NULL);
  rowptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) rowptr[i + 1] = rowptr[i] + low[i] + upc[i];
  int64_t nnz = rowptr[n];
  if (col != NULL) {
    int64_t* fill = (int64_t*)calloc(n, sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) {
      int64_t base = rowptr[i] + low[i];
      g_row(&g, i, 1, NULL, rowptr, fill, &base, col, q);
    }
    free(fill);
  }
  free(low);
  free(upc);
  return nnz;
}
