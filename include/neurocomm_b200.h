/*
 * neurocomm_b200.h -- C ABI of libneurocomm_b200.so, the B200 (sm_100a) engine
 * behind the drop-in Python package paper_2205_07125_b200.
 *
 * Reference: arXiv 2205.07125 "neurocomm" (pkg/src/neurocomm).  The reference is
 * pure Python + numpy and has no FFI; each entry point below names the
 * reference function whose semantics it implements (file:line), or says
 * "new" for the per-timestep loop the reference only models analytically
 * (netsim.py:177-273).  The Python layer validates arguments and raises the
 * reference's exception types before calling here; every entry point returns
 * 0 on success and a non-zero NC_E* code otherwise, with a message available
 * from nc_last_error().
 *
 * All pointers are plain device pointers unless marked [host].  `stream` is a
 * cudaStream_t passed as void*.  No entry point allocates or frees memory it
 * does not own; all device work is enqueued on `stream` and never synchronises
 * the host unless stated.
 */
#ifndef NEUROCOMM_B200_H
#define NEUROCOMM_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NC_ABI_VERSION 4

enum {
  NC_OK = 0,
  NC_E_ARG = 1,      /* invalid argument (Python maps to ValueError)        */
  NC_E_CUDA = 2,     /* CUDA runtime error                                   */
  NC_E_OVERFLOW = 3, /* a spike bucket exceeded its capacity                 */
  NC_E_TIMEOUT = 4,  /* exchange watchdog expired waiting for a peer flag    */
  NC_E_NCCL = 5,     /* NCCL error                                           */
  NC_E_PARSE = 6,    /* malformed NNG / PMAP text (Python: ParseError)       */
  NC_E_IO = 7        /* file cannot be opened / read / written (OSError)     */
};

int nc_abi_version(void);
const char* nc_last_error(void);

/* ------------------------------------------------------------------ K6 --
 * Capacity-bounded greedy bucket fill, bit-identical to
 * neurocomm greedy.py:55-117 (called from partition.py:95-114 for
 * neuron->GPU placement and routing.py:129-135 for GPU->group).
 * [host] everything.  `capacity` is computed by the caller exactly as
 * greedy.py:70 does ((fsum(w)/n_buckets)*(1+slack)); the C++ side uses an
 * indexed max-heap keyed (score desc, weight desc, index asc) instead of the
 * reference's lazy heapq, which selects the same item at every step. */
int nc_greedy_fill(int64_t n_items, const double* weights, const int64_t* indptr,
                   const int64_t* indices, const double* values, int32_t n_buckets,
                   double capacity, int64_t* assignment_out);

/* ------------------------------------------------------------------ K5 --
 * Exact traffic histogram: device replacement for the summation in
 * traffic.aggregate (traffic.py:66-84) and accum.keyed_sums (accum.py:21-41).
 * contrib_e = (edge_p[e] * w[i]) * w[j]  (traffic.py:77, two RN multiplies);
 * cell = lo*n_gpus + hi with lo/hi = min/max of the endpoints' GPUs.
 * Each contribution is added EXACTLY into a fixed-point accumulator of
 * `n_digits` 32-bit digits held in uint64 limbs whose least significant bit is
 * 2^lsb_exponent; the caller rounds once (correctly, half-even) on the host,
 * which reproduces math.fsum bit for bit.
 *   nc_traffic_exponents: out_minmax[0] = min over edges of the binary
 *     exponent of the contribution's lowest mantissa bit, out_minmax[1] = max
 *     exponent of its leading bit (device int32[2], initialise to INT_MAX/INT_MIN).
 *     Pass edge_i == NULL to scan `weights` (n_edges entries) instead.
 *   nc_traffic_histogram: pg_limbs is uint64[n_gpus*n_gpus][n_digits] (only
 *     lo<=hi cells are written), zero-initialised by the caller.
 *   nc_weight_histogram: wg_limbs uint64[n_gpus][n_digits]: exact per-GPU
 *     weight totals (partition.py:131-137 / traffic.py:83). */
int nc_traffic_exponents(const int64_t* edge_i, const int64_t* edge_j, const double* edge_p,
                         const double* weights, int64_t n_edges, int32_t* out_minmax,
                         void* stream);
int nc_traffic_histogram(const int64_t* edge_i, const int64_t* edge_j, const double* edge_p,
                         const double* weights, const int64_t* assignment, int64_t n_edges,
                         int32_t n_gpus, int32_t lsb_exponent, int32_t n_digits,
                         unsigned long long* pg_limbs, void* stream);
/* Same with int32 neuron ids and assignment (16 B per edge streamed instead of
 * 24; what traffic.aggregate uses below 2^31 neurons). */
int nc_traffic_histogram32(const int32_t* edge_i, const int32_t* edge_j, const double* edge_p,
                           const double* weights, const int32_t* assignment, int64_t n_edges,
                           int32_t n_gpus, int32_t lsb_exponent, int32_t n_digits,
                           unsigned long long* pg_limbs, void* stream);
/* Same with the per-neuron gathers packed: neuron_records[k] = 16 bytes
 * {double weight; int32 gpu; int32 unused} (one gather per endpoint). */
int nc_traffic_histogram_packed(const int32_t* edge_i, const int32_t* edge_j, const double* edge_p,
                                const void* neuron_records, int64_t n_edges, int32_t n_gpus,
                                int32_t lsb_exponent, int32_t n_digits, unsigned long long* pg_limbs,
                                void* stream);
/* Same when every neuron weight equals `weight` (generate_synthetic's default
 * weight_low == weight_high; contributions (p * weight) * weight, the same two
 * roundings) and the assignment is uint8 (n_gpus <= 256): one byte gathered per
 * endpoint. */
int nc_traffic_histogram_uniform(const int32_t* edge_i, const int32_t* edge_j, const double* edge_p,
                                 double weight, const uint8_t* assignment, int64_t n_edges, int32_t n_gpus,
                                 int32_t lsb_exponent, int32_t n_digits, unsigned long long* pg_limbs,
                                 void* stream);
/* Host pass of the edge upload (sim.upload_edges): int64 ids and fp64 p of n edges ->
 * int32 ids and uint8 weight units q = clamp(ceil(32 p), 1, 32) in caller buffers (pinned
 * staging), `threads` host threads (0 = all); NC_E_ARG if an endpoint lies outside
 * [0, n_neurons). */
int nc_edges_narrow(const int64_t* edge_i, const int64_t* edge_j, const double* edge_p, int64_t n,
                    int64_t n_neurons, int32_t* out_i, int32_t* out_j, uint8_t* out_q, int32_t threads);
/* PartitionMap.assignment (int64) -> uint8 gpu ids for nc_traffic_histogram_uniform,
 * counts[g] += neurons on GPU g (uint64 [n_gpus], zeroed by the caller), *bad |= 1
 * if a value lies outside [0, n_gpus) (written as 0; the caller raises, as the
 * reference's indexing would). */
int nc_assignment_u8(const int64_t* assignment, int64_t n_neurons, int32_t n_gpus, uint8_t* out,
                     unsigned long long* counts, unsigned long long* bad, void* stream);
int nc_weight_histogram(const double* weights, const int64_t* assignment, int64_t n_neurons,
                        int32_t n_gpus, int32_t lsb_exponent, int32_t n_digits,
                        unsigned long long* wg_limbs, void* stream);

/* ----------------------------------------------------- simulation state --
 * New (the reference's only "step" is the analytic netsim.step_latency).
 * One shard = the neurons one GPU owns under PartitionMap.assignment
 * (partition.py:60-65).  Neurons are renumbered into an internal id space in
 * which shard g owns the contiguous, 32-aligned range
 * [local_base, local_base + n_local); bitmaps are indexed by internal id.
 *
 * Synapses: each undirected edge (i, j, p) of NeuronGraph is one synapse in
 * each direction.  A pull synapse is a 25-bit field
 *     (q << 19) | (id ^ 31),  id = pre_internal_id - first id of its bitmap tile
 * (the low 5 bits hold 31 - the pre's bit in its bitmap word),
 * q = ceil(32 * p) in [1, 32]; q = 0 is the pad.  Tiles are at most 16384
 * words, so the tile-relative id fits 19 bits (with one tile it is the
 * internal id).  A 16-byte slot holds 5 fields, field i at bit 25 i of
 * (x | y << 32 | z << 64 | w << 96): 3.2 bytes per synapse.
 * Layout "J-SELL-32": jagged sliced ELL with slice = one warp = 32
 * consecutive local rows, further split by bitmap tile t (the spike bitmap is
 * staged in shared memory tile by tile).  Row r of slice s has len_r slots in
 * block (s, t); its slots [0, emid) hold its excitatory pres (weight +q), the
 * next ones its inhibitory pres (weight -g_inh*q), each segment padded to
 * whole slots with pad fields: row_meta[t*n_local + p] = emid | (len_r << 16)
 * (p = the row's position, see the placement below).
 * Block (s, t) starts at slice_ptr[s*n_tiles + t] (uint4 units) and stores
 * slot u of every lane with len > u contiguously, in lane order:
 *     position(u, l) = sum_{v<u} cnt_v + #{l' < l : len_l' > u},
 *     cnt_v = #{l : len_l > v},
 * so for u below the block's shortest row it is plain u*32 + l (coalesced
 * 512-byte warp loads) and the block holds no padding to its longest row.
 * Each lane owns one row: no cross-lane reduction.
 * Tiled placement: with n_tiles > 1, lane l of block (s, t) works on
 * position p = 32s + l (positions >= n_local hold no row).  CTA c of the
 * tiled step owns slices s = c mod G (G = cta_groups); its rows are numbered
 * k = 32*(s div G) + (row mod 32) and the row at position p of tile t is
 * k = row_perm[t*n_local + p], i.e. row = 32*(c + (k div 32)*G) + k mod 32
 * with c = (p div 32) mod G.  Rows are placed in descending order of their
 * tile-t length within their CTA, so the 32 rows of every block have
 * near-equal lengths in every tile (the jagged tail stays short).  row_meta
 * is tile-major by position: row_meta[t*n_local + p].  With one tile
 * positions are rows.
 * Push entries (rows = internal pre ids):
 *     (inhibitory(pre) << 31) | ((q - 1) << 26) | post_local. */

#define NC_MAX_SHARDS 16
#define NC_INTERNAL_ID_BITS 26

typedef struct nc_lif_params {
  float alpha_v;      /* exp(-dt/tau_m), computed in fp64 then rounded        */
  float alpha_i;      /* exp(-dt/tau_syn)                                     */
  float beta;         /* membrane gain applied to the synaptic current        */
  float v_rest, v_reset, v_th;
  float w_unit;       /* current per synaptic weight unit                     */
  float w_ext;        /* current per external Poisson event                   */
  float v_init_span;  /* v_th - v_reset (fp32): initial V is uniform in it    */
  uint32_t ext_threshold; /* Philox lane k fires an external event if < this  */
  int32_t ext_lanes;  /* number of Philox lanes (1..4) used as drive          */
  int32_t t_ref;      /* refractory steps                                     */
  int32_t g_inh;      /* inhibitory weight multiplier                         */
  int32_t pad0;
  uint64_t seed;
} nc_lif_params_t;

typedef struct nc_shard {
  int32_t shard;          /* this shard's GPU index in the partition          */
  int32_t n_shards;
  int32_t n_local;        /* neurons owned                                     */
  int32_t local_base;     /* first internal id owned (multiple of 32)          */
  int32_t n_words;        /* bitmap words over all internal ids incl. guard   */
  int32_t n_tiles;        /* bitmap tiles (1 = whole bitmap in shared memory)  */
  int32_t tile_words;     /* words per bitmap tile (multiple of 4)             */
  int32_t flags;          /* bit 0: tiled partial sums in `acc` (huge shards); bits 1-2: s, the tiled kernel's warps claim each (slice, tile) block in 2^s parts (small shards); bit 3: three tile buffers instead of two */
  /* neuron state, n_local each */
  float* v;
  float* i_syn;
  uint8_t* refrac;
  int32_t* acc;           /* synaptic input (push delivery / unfused path)    */
  const uint32_t* gid;    /* global neuron id (Philox counter, raster ids)    */
  const uint16_t* hop_mask; /* bit h: a spike of this neuron is sent to shard h */
  /* pull SELL-32 */
  const int64_t* slice_ptr; /* n_slices*n_tiles+1 block starts (uint4 units)   */
  const uint32_t* row_meta; /* [n_tiles][n_local] by position: emid | (slots << 16) */
  const uint32_t* syn;      /* packed entries                                  */
  /* push CSR (optional): rows = internal pre ids, entries see above */
  const int64_t* push_rowptr;
  const uint32_t* push_syn;
  /* spikes */
  uint32_t* bitmap0;      /* n_words; bitmap of step t lives in bitmap[t&1]   */
  uint32_t* bitmap1;
  uint32_t* fired_ids;    /* local fired internal ids of the current step      */
  int32_t* fired_count;   /* [1]                                               */
  /* per-destination send buckets: bucket h holds ids for shard h */
  uint32_t* bucket_ids;   /* n_shards * bucket_cap                             */
  int32_t* bucket_count;  /* n_shards                                          */
  int64_t bucket_cap;
  int32_t* status;        /* [0] overflow flag, [1] timeout flag               */
  int32_t* step;          /* device step counter (read by every kernel)        */
  /* records (NULL = off) */
  uint32_t* raster;       /* [record_steps][local_words]: bitmap of local spikes */
  int32_t record_steps;
  int32_t local_words;
  unsigned long long* spike_total; /* [1] running count of local spikes        */
  uint32_t* work;         /* [4] scratch counters (push work claims), zeroed by
                             nc_sim_init / nc_sim_end_step                      */
  /* tiled layouts (n_tiles > 1): per-tile row placement, see the layout notes */
  const int32_t* row_perm; /* [n_tiles][n_local]: CTA-local index of the row
                              at position p of tile t (NULL = identity)         */
  int32_t cta_groups;     /* G the placement was built for (CTA c owns slices
                             c, c+G, ...); the tiled step launches G CTAs       */
  int32_t pb_bins;        /* binned push (optional): B target bins = CTAs      */
  /* binned push synapses: rows = internal pre ids, each row's entries grouped
   * by the bin of their post row (bin c = local rows [c*pb_rows, (c+1)*pb_rows)),
   * entry = (inh << 31) | ((q - 1) << 26) | (post_local - c*pb_rows);
   * bin c of pre i = pb_syn[pb_rowptr[i] + pb_binoff[i*(B+1) + c] ...
   * pb_rowptr[i] + pb_binoff[i*(B+1) + c + 1]) */
  const int64_t* pb_rowptr;
  const uint16_t* pb_binoff;
  const uint32_t* pb_syn;
  int32_t pb_rows;        /* local rows per bin (multiple of 32)               */
  int32_t pad3;
  /* spike lists by step parity (binned delivery): the local spikes of step t
   * (LIF) and the remote ones (exchange) are appended to list t&1, which the
   * step t+1 kernel reads; nc_sim_end_step empties list (t+1)&1 */
  uint32_t* spk_ids;      /* [2][spk_cap] */
  int32_t* spk_count;     /* [2] */
  int64_t spk_cap;
  /* optional (NULL = off): device %globaltimer of the fused step kernel, per
   * step s (slot s mod kstamp_steps): [2s] = first CTA start (atomicMin; the host
   * fills it with ~0), [2s+1] = last CTA end (atomicMax; host fills 0) -- the
   * kernel's duration inside a timed loop without a profiler */
  unsigned long long* kstamp;
  int32_t kstamp_steps;
  int32_t pad4;
  /* optional fused P2P send (P2P transport, phase 1; xsend_on = 0: off):
   * the step kernel stores every spike bucketed for peer h straight into h's
   * IPC-mapped inbox (xsend[h], the nc_xchg_t P2P layout, tagged 8-byte words)
   * while other CTAs still compute, and its last CTA writes the tagged headers
   * (count; 0 for peers outside xsend_mask = the heartbeat); nc_xchg_p2p then
   * only receives (nc_xchg_t.fused_send = 1) */
  unsigned long long* xsend[NC_MAX_SHARDS];
  int64_t xsend_cap;      /* ids per message = nc_xchg_t.cap */
  int32_t xsend_on;
  int32_t xsend_mask;     /* peers with a phase-1 message (nc_xchg_t.send1_mask) */
  /* push windows (push_windows > 1): the local post rows are cut into windows of
   * push_window_rows (multiple of 32); every push row is grouped by window and an
   * entry holds the post row relative to its window start.  Window w of pre i =
   * push_syn[push_rowptr[i] + push_winoff[i*(W+1) + w] ... + push_winoff[i*(W+1) + w + 1]).
   * The persistent engine delivers one window at a time with a grid barrier in
   * between, so the atomic reductions of a window stay in L2 (config 5 over 2 GPUs:
   * 25 M post rows = 100 MB of accumulators).  push_windows <= 1: plain rows. */
  const uint16_t* push_winoff;
  int32_t push_windows;
  int32_t push_window_rows;
} nc_shard_t;

/* Set kernel attributes (dynamic shared memory opt-in) once; call before any
 * CUDA-graph capture of the step functions.  Implied by the first launch. */
int nc_sim_prepare(void);

/* Draw the initial state (V uniform in [v_reset, v_th), I = 0, refrac = 0),
 * zero both bitmaps, counters and the step counter. */
int nc_sim_init(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream);

/* One fused step on one shard (pull delivery K3 + LIF K1 + ballot/bucket K2):
 * syn input = sum over the row's entries whose pre fired at step-1, integer;
 * then the LIF update in the fixed fp32 operation order documented in
 * DESIGN.md; fired ids are written to the current bitmap (local range), the
 * fired list, and every bucket in the neuron's hop_mask (warp-aggregated).
 * Also zeroes the remote part of the current bitmap for the exchange. */
int nc_sim_step_fused(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream);

/* Unfused building blocks (same arithmetic):
 *   deliver_pull: acc[r] = integer pull sum over the CSR row (K3 alone)
 *   deliver_push: for every id set in the previous step's bitmap, add its
 *                 push-CSR row into acc with integer atomics (event driven)
 *   lif_update:   K1+K2 consuming and zeroing acc */
int nc_sim_deliver_pull(const nc_shard_t* sh, int32_t g_inh, void* stream);
int nc_sim_deliver_push(const nc_shard_t* sh, int32_t g_inh, void* stream);
int nc_sim_lif_update(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream);

/* Event-driven delivery needs the transpose of the pull synapses (push CSR,
 * rows = internal pre ids over n_words*32 rows).  Built on the device by a
 * counting sort: phase 0 adds every real entry's count into push_rowptr[pre+1]
 * (zero-initialised int64[n_words*32+1]); the caller prefix-sums push_rowptr;
 * phase 1 writes the entries (push_fill int32[n_words*32] zero-initialised).
 * The shard's slice_ptr/row_meta/syn must be set; push fields are ignored. */
/* Binned push synapses (see nc_shard_t) from the pull arrays of the shard.
 * phase 0: counts[pre*B + bin] += 1 (uint32, zeroed, n_pre*B); the host turns
 * them into pb_rowptr / pb_binoff (per-row prefix, < 65536 entries per row);
 * phase 1: places the entries, claiming slots with atomics on `fill`
 * (uint32 [n_pre*B], zeroed).  Uses sh->pb_bins / pb_rows for the bins. */
int nc_build_push_binned(const nc_shard_t* sh, int32_t phase, uint32_t* counts, const int64_t* pb_rowptr,
                         const uint16_t* pb_binoff, uint32_t* fill, uint32_t* pb_syn, void* stream);
/* Event-driven step with binned push (replaces push + LIF + end-of-step
 * bucketing): CTA c owns the rows of bin c, reads the spike list of step t-1,
 * sums the weights of its bin of every spiking pre in shared memory (integer,
 * order free), then runs K1 + K2 on its rows and appends its spikes to list
 * t&1.  Launches pb_bins CTAs; needs pb_* and spk_*. */
int nc_sim_step_binned(const nc_shard_t* sh, const nc_lif_params_t* p, void* stream);
int nc_build_push_csr(const nc_shard_t* sh, int32_t phase, int64_t* push_rowptr, int32_t* push_fill,
                      uint32_t* push_syn, void* stream);

/* Advance the device step counter and reset the per-step bucket counts. */
int nc_sim_end_step(const nc_shard_t* sh, void* stream);

/* Single-process exchange over all shards of one device ("local" transport,
 * used to run N partitions on one GPU and for the partition-invariance tests).
 * Routing follows RoutingTable (routing.py:61-115, 184-231).  shards[] [host]
 * are the n_shards shard descriptors; their next-hop buckets were filled by
 * the step kernel.  fwd_table [host, n*n] holds, for relay b and source s, the
 * destination shards d whose path is (s, b, d); dest_mask (device, per
 * internal id) the shards hosting targets of each neuron.  fwd_ids/fwd_count
 * are the relay buckets (n*n*fwd_cap ids, n*n counts; may be NULL when no path
 * is bridged).  Counters (device int64, [n*n] or [steps][n*n] if per_step):
 *   hop_ids[u*n+v]   ids carried on channel u->v (both phases)
 *   deliv_ids[s*n+d] ids of source s delivered at d that have targets on d */
int nc_exchange_local(const nc_shard_t* shards, int32_t n_shards, const uint16_t* dest_mask,
                      const uint16_t* fwd_table, uint32_t* fwd_ids, int32_t* fwd_count,
                      int64_t fwd_cap, long long* hop_ids, long long* deliv_ids, int32_t per_step,
                      void* stream);

/* ------------------------------------------------- multi-GPU exchange --
 * One process per GPU; rank r owns shard r.  Route semantics as
 * nc_exchange_local.  Channel masks (bit p = peer p) come from the global
 * RoutingTable so every rank derives the same send/recv sets:
 *   send1/recv1: first hops (s -> next_hop(s, d));  send2/recv2: relay hops.
 * Messages carry at most `cap` ids; more sets status[0] (overflow). */
typedef struct nc_xchg {
  int32_t rank, n, cap, two_level;
  int32_t per_step, lat_steps;
  uint16_t send1_mask, recv1_mask, send2_mask, recv2_mask;
  int64_t bucket_cap;              /* stride of the shard's bucket_ids rows     */
  uint64_t timeout_ns;             /* P2P watchdog                              */
  const int32_t* step;             /* shard step counter                        */
  int32_t* status;                 /* shard status words                        */
  uint32_t* bitmap0;
  uint32_t* bitmap1;
  const uint32_t* bucket_ids;      /* shard next-hop buckets                    */
  const int32_t* bucket_count;
  const uint16_t* dest_global;     /* dest mask of every internal id            */
  int64_t shard_base[NC_MAX_SHARDS + 1];
  uint16_t fwd_row[NC_MAX_SHARDS]; /* as relay: destinations forwarded for src s */
  uint32_t* fwd_ids;               /* relay buckets [n][cap]                    */
  int32_t* fwd_count;              /* [n]                                       */
  long long* hop_ids;              /* [n*n] (or [steps][n*n])                   */
  long long* deliv_ids;
  /* NCCL transport buffers */
  int32_t* send_hdr;
  int32_t* send2_hdr;
  int32_t* recv_hdr;
  int32_t* recv2_hdr;
  uint32_t* recv_ids;              /* [n][cap] */
  uint32_t* recv2_ids;
  /* P2P transport: IPC-mapped inboxes/flags */
  uint32_t* my_inbox;
  uint32_t* my_flags;              /* [2][NC_MAX_SHARDS]                        */
  uint32_t* peer_inbox[NC_MAX_SHARDS];
  uint32_t* peer_flags[NC_MAX_SHARDS];
  uint32_t* done;                  /* monotonically counting block exits        */
  uint32_t* send_done;             /* [2][NC_MAX_SHARDS]: [0][d] = relay arrivals for
                                      destination d (two-level, monotonic per run) */
  int32_t blocks_per_peer;         /* P2P kernel blocks per peer (chunks)       */
  int32_t pad1;
  uint32_t* barrier;               /* unused since relays forward as ids arrive (kept
                                      for layout stability; zeroed by the reset)  */
  unsigned long long* lat_start;
  uint32_t* lat_ns;                /* per-step exchange latency (ns) or NULL    */
  uint32_t* spk_ids;               /* binned delivery: append received ids to the  */
  int32_t* spk_count;              /* step's spike list ([2][spk_cap], [2]) or NULL */
  int64_t spk_cap;
  unsigned long long* dbg;         /* diagnostics or NULL: [64 steps][n*B blocks][4]
                                      globaltimer at block start, message published,
                                      peer flag seen, inbound ids scattered      */
  int32_t fused_send;              /* 1: the step kernel already sent phase 1
                                      (nc_shard_t.xsend): receive only           */
  int32_t pad2;
} nc_xchg_t;

/* Inbox words needed per rank for the P2P transport. */
#define NC_P2P_INBOX_WORDS(n, cap) ((size_t)8 * (size_t)(n) * ((size_t)(cap) + 1))

/* Before a run: zero this rank's P2P inbox (tags restart with the step
 * counter), flags, barrier and relay counts.  Every rank must finish its reset
 * before any rank sends (synchronize + barrier). */
int nc_xchg_reset(const nc_xchg_t* X, void* stream);
/* NCCL path: seal (headers + hop counters), grouped send/recv, scatter. */
int nc_xchg_seal(const nc_xchg_t* X, int32_t phase, void* stream);
int nc_xchg_scatter(const nc_xchg_t* X, int32_t phase, void* stream);
int nc_nccl_get_unique_id(void* id_out /* 128 bytes */);
int nc_nccl_comm_init(void** comm_out, int32_t nranks, const void* id /* 128 bytes */, int32_t rank);
int nc_nccl_comm_destroy(void* comm);
int nc_nccl_exchange(void* comm, const nc_xchg_t* X, int32_t phase, void* stream);
/* P2P path: one device-initiated kernel per step (both phases). */
int nc_xchg_p2p(const nc_xchg_t* X, void* stream);
/* dst[*step] = %globaltimer (ns) if *step < max_steps: per-step exchange
 * latency stamps, enqueued before and after the exchange. */
int nc_stamp(unsigned long long* dst, const int32_t* step, int32_t max_steps, void* stream);
/* Persistent event-driven engine: ONE cooperative kernel runs n_steps steps
 * (push delivery -> LIF/buckets -> P2P exchange, separated by in-kernel grid
 * barriers) with no launches or host work between steps.  Requires the push
 * CSR and acc on the shard; X may be NULL for a single GPU.  gbar: one uint32
 * of scratch (zeroed by the call).  stamp_ready/stamp_done (nullable) receive
 * %globaltimer per step (index = step < stamp_cap) around the exchange. */
/* Largest shard (rows) nc_run_persistent accepts on the current device (0 on error). */
int64_t nc_persistent_max_rows(void);
int nc_run_persistent(const nc_shard_t* sh, const nc_lif_params_t* p, const nc_xchg_t* X, int32_t n_steps,
                      int32_t blocks_per_peer, unsigned int* gbar, unsigned long long* stamp_ready,
                      unsigned long long* stamp_done, int32_t stamp_cap, void* stream);
/* Diagnostics for nc_run_persistent: when dst (device uint64[64][4]) is set,
 * the next launches record (start, after push, after LIF, after exchange)
 * %globaltimer stamps of their first 64 steps.  NULL switches it off. */
int nc_persistent_phase_stamps(unsigned long long* dst);
/* CUDA IPC windows for the P2P inboxes. */
int nc_ipc_alloc(size_t bytes, void** ptr_out, void* handle_out /* 64 bytes */);
int nc_ipc_open(const void* handle /* 64 bytes */, void** ptr_out);
int nc_ipc_close(void* ptr);
int nc_free(void* ptr);

/* ------------------------------------------------------- network build --
 * Device SBM generator with the distributions of generate_synthetic
 * (model.py:199-253): contiguous near-equal communities, intra pairs
 * Bernoulli(p_in) with p ~ U(intra range), inter pairs Bernoulli(p_out) with
 * p ~ U(inter range); counter-based (Philox) so every shard regenerates the
 * same global graph and keeps the rows it owns.  Builds the pull CSR in the
 * layout above.  Two passes: count (row lengths) then fill. */
typedef struct nc_graphgen {
  int64_t n_neurons;
  int32_t n_communities;
  int32_t shard;
  double p_in, p_out;
  double intra_lo, intra_hi, inter_lo, inter_hi;
  uint64_t seed;
  const int32_t* owner;       /* [n_neurons] shard of every gid               */
  const int32_t* internal_id; /* [n_neurons] internal id of every gid         */
  int32_t local_base;
  int32_t inh_every;          /* gid % inh_every == inh_every-1 is inhibitory (0 = none) */
  int32_t n_local;            /* rows of this shard (nc_graphgen_fill)        */
  int32_t pad0;
} nc_graphgen_t;

/* Pass 0: deg[gid] += number of edges of every neuron (zero-initialised
 * int32[n_neurons]); owner/internal_id are not read.  The host orders each
 * shard's rows by degree so the 32 rows of a slice have similar lengths. */
int nc_graphgen_degrees(const nc_graphgen_t* g, int32_t* deg, void* stream);
/* Pass 1.  lower_len/upper_len: [n_local * n_tiles * 2] entries per
 * (row, tile, sign) (zero-initialised); tile_words as in nc_shard_t. */
int nc_graphgen_count(const nc_graphgen_t* g, int32_t n_tiles, int32_t tile_words, int32_t* lower_len,
                      int32_t* upper_len, void* stream);
/* Pass 2 into the UNPACKED PADDED SELL-32 layout (every block = its longest
 * row x 32 lanes, slot u of lane l = 5 uint32 entries (q << 26 | tile-relative
 * id) at 5 * (padded_ptr[block] + u*32 + l); padded_ptr and
 * row_meta computed by the host from the pass-1 counts); lower_fill
 * [n_local*n_tiles*2] zero-initialised (slot claims); pos_of[row*n_tiles + t]
 * = position of the row in tile t (inverse of the placement; NULL = identity).  syn must be pre-filled with nc_sell_fill_pads; convert the
 * result with nc_sell_repack. */
int nc_graphgen_fill(const nc_graphgen_t* g, int32_t n_tiles, int32_t tile_words, const int64_t* slice_ptr,
                     const uint32_t* row_meta, const int32_t* pos_of, int32_t* lower_fill, uint32_t* syn,
                     void* stream);
/* The pull-layout passes over an explicit edge list instead of the generator
 * (simulate() on a host NeuronGraph, model.py:53-92): edge k = (edge_i[k],
 * edge_j[k]) with weight units q[k] (= ceil(32 p), 1..32), one synapse each
 * way.  g supplies owner / internal_id / shard / local_base / n_local /
 * inh_every (n_neurons bounds the ids; the SBM fields are ignored).
 * nc_edges_count: seg_len[(row*n_tiles + tile)*2 + inh] += 1 (zeroed);
 * nc_edges_fill: as nc_graphgen_fill. */
int nc_edges_count(const nc_graphgen_t* g, const int32_t* edge_i, const int32_t* edge_j, int64_t n_edges,
                   int32_t n_tiles, int32_t tile_words, int32_t* seg_len, void* stream);
int nc_edges_fill(const nc_graphgen_t* g, const int32_t* edge_i, const int32_t* edge_j, const uint8_t* q,
                  int64_t n_edges, int32_t n_tiles, int32_t tile_words, const int64_t* slice_ptr,
                  const uint32_t* row_meta, const int32_t* pos_of, int32_t* fill, uint32_t* syn, void* stream);
/* K6 straight off the generator's network (config-3 scale, where the
 * NeuronGraph and its CSR do not fit in host memory; replaces
 * partition_greedy's adjacency_from_edges + greedy_fill, partition.py:95-114,
 * greedy.py:32-117): the same fill over adjacency_from_edges' row order and
 * values, rows regenerated on demand on the host (upper part) or read from a
 * 4 B/edge transpose (lower part), p recomputed per edge.  spec: the generator
 * fields of nc_graphgen_t (owner/internal_id unused); weights NULL = all 1;
 * threads 0 = all cores (the transpose build; the fill is sequential). */
int nc_greedy_fill_generated(const nc_graphgen_t* spec, const double* weights, int32_t n_buckets,
                             double capacity, int64_t* assignment, int32_t threads);
/* The generated network as NeuronGraph columns (ascending (i, j), fp64 p),
 * host restatement of the device generator.  NULL arrays: returns the edge
 * count; < 0 on error. */
int64_t nc_hostgen_edges(const nc_graphgen_t* spec, int64_t* edge_i, int64_t* edge_j, double* edge_p,
                         int32_t threads);
/* K5 over a generated network (traffic.aggregate_generated): the rows
 * [row_begin, row_end) of the generator's network are enumerated on the fly and
 * every edge's (p * W_i) * W_j added exactly into pg_limbs (layout as
 * nc_traffic_histogram; weights NULL = all 1; assignment int32 [n_neurons]).
 * Split the rows over ranks and all-reduce the limbs for the multi-GPU path. */
int nc_traffic_histogram_generated(const nc_graphgen_t* g, const double* weights, const int32_t* assignment,
                                   int64_t row_begin, int64_t row_end, int32_t n_gpus, int32_t lsb_exponent,
                                   int32_t n_digits, unsigned long long* pg_limbs, void* stream);
/* Windowed push synapses (nc_shard_t push_windows > 1) straight from the
 * generator.  Phase 0: counts[pre*W + w] += entries of pre in window w (uint32,
 * zeroed) and the destination masks as nc_graphgen_push; the caller builds
 * push_rowptr (row totals, scanned) and push_winoff (per-row prefix, < 65536);
 * phase 1 fills push_syn (fill uint32 [n_pre*W] zeroed). */
int nc_graphgen_push_windowed(const nc_graphgen_t* g, int32_t phase, int32_t windows, int32_t window_rows,
                              uint32_t* counts, const int64_t* push_rowptr, const uint16_t* push_winoff,
                              uint32_t* fill, uint32_t* push_syn, uint16_t* dest_mask, void* stream);
/* Push synapses (nc_shard_t push_rowptr / push_syn format) straight from the
 * generator, without a pull layout.  Phase 0: push_rowptr[pre + 1] += entries
 * of pre (int64 [n_words*32 + 1], zeroed) and dest_mask[r] |= shards hosting a
 * target of local row r, this shard excluded (zeroed, 4-byte aligned,
 * n_local + 2 entries); the caller prefix-sums push_rowptr.  Phase 1 fills
 * push_syn (push_fill int32 [n_words*32] zeroed: slot claims). */
int nc_graphgen_push(const nc_graphgen_t* g, int32_t phase, int64_t* push_rowptr, int32_t* push_fill,
                     uint32_t* push_syn, uint16_t* dest_mask, void* stream);
/* Pad pre-fill of an unpacked padded SELL-32 array: every entry = 0 (q = 0).
 * n_tiles / tile_words are accepted for ABI stability. */
int nc_sell_fill_pads(const int64_t* slice_ptr, int64_t n_blocks, int32_t n_tiles, int32_t tile_words,
                      uint32_t* syn, void* stream);
/* Destination masks from a built CSR (the adjacency is symmetric, so the
 * pres of row r are exactly the posts r drives): dest_mask[r] = OR over the
 * row's entries of (1 << owner shard of the pre id) without `self`, where shard
 * h owns internal ids [shard_base[h], shard_base[h+1]) (device int32[n+1]).
 * dest_mask must be zeroed and 4-byte aligned (rows are OR-ed in per tile). */
int nc_dest_mask_from_csr(const int64_t* slice_ptr, const uint32_t* row_meta, const int32_t* row_perm,
                          int32_t cta_groups, int32_t n_tiles, int32_t tile_words, const uint32_t* syn,
                          int32_t n_local,
                          const int32_t* shard_base, int32_t n_shards, int32_t self, uint16_t* dest_mask,
                          void* stream);
/* Unpacked padded entries (5 uint32 per slot) -> packed 16-byte slots. */
int nc_sell_pack(const uint32_t* unpacked, int64_t n_slots, uint32_t* packed, void* stream);
/* Shared-memory bank placement inside each row's E / I segments of a padded
 * SELL-32 array, unpacked (src: a copy of it, dst: the array): entry 5u+k of
 * lane l gets a pre whose bitmap word is in bank (l + 5u + k) mod 32 where the row has one, so
 * the 32 lookups of one step-kernel instruction hit distinct banks. */
int nc_sell_bank_order(const int64_t* padded_ptr, const uint32_t* row_meta, int32_t n_tiles, int32_t n_local,
                       const uint32_t* src, uint32_t* dst, void* stream);
/* Padded SELL-32 (padded_ptr, as filled by nc_graphgen_fill) <-> J-SELL-32
 * (slice_ptr): to_jagged != 0 copies src (padded) into dst (jagged), else
 * the reverse (dst must be pre-filled; slots past a row's length are left
 * untouched).  Pointers in uint4 units, n_slices * n_tiles + 1 entries. */
int nc_sell_repack(const int64_t* padded_ptr, const int64_t* slice_ptr, const uint32_t* row_meta, int32_t n_tiles,
                   int32_t n_local, const uint32_t* src, uint32_t* dst, int32_t to_jagged, void* stream);

/* GA balance repair (replaces _repair_balance, partition.py:167-184): while the
 * heaviest GPU's load (correctly rounded exact sum of its weights, = math.fsum;
 * lowest index on ties) exceeds `bound`, move its heaviest neuron (lowest index
 * on ties) to the lightest GPU.  Loads are kept as exact fixed-point integers
 * updated per move; identical decisions to the reference.  *n_moves (optional)
 * receives the number of moves. */
int nc_repair_balance(int64_t n_neurons, const double* weights, int64_t* assignment, int32_t n_gpus, double bound,
                      int64_t* n_moves);

/* ---------------------------------------------------------------- text I/O
 * Native readers / writers of the reference's text artefacts with its exact
 * acceptance rules and error texts (str.splitlines lines, float()/int()
 * tokens, repr() in messages); writers emit repr() floats, byte-identical to
 * the reference.  On NC_E_PARSE, nc_last_error() is the ParseError message and
 * *err_line its 1-based line.  Read = scan (header counts) + read (arrays of
 * those sizes, allocated by the caller). */
/* replaces load_graph model.py:307-364 (with nc_nng_read) */
int nc_nng_scan(const char* path, int64_t* n_neurons, int64_t* n_edges, int64_t* err_line);
int nc_nng_read(const char* path, int64_t n_neurons, int64_t n_edges, double* weights, int64_t* edge_i,
                int64_t* edge_j, double* edge_p, int64_t* err_line);
/* replaces save_graph model.py:293-304; edges in ascending (i, j) order */
int nc_nng_write(const char* path, int64_t n_neurons, int64_t n_edges, const double* weights, const int64_t* edge_i,
                 const int64_t* edge_j, const double* edge_p);
/* replaces load_partition_map partition.py:278-306 (with nc_pmap_read) */
int nc_pmap_scan(const char* path, int64_t* n_neurons, int64_t* n_gpus, int64_t* err_line);
int nc_pmap_read(const char* path, int64_t n_neurons, int64_t n_gpus, int64_t* assignment, int64_t* err_line);
/* replaces save_partition_map partition.py:270-275 */
int nc_pmap_write(const char* path, int64_t n_neurons, int64_t n_gpus, const int64_t* assignment);

#ifdef __cplusplus
}
#endif
#endif /* NEUROCOMM_B200_H */
