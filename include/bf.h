/*
 * bf.h -- C ABI of libbf, B200-native exact butterfly counting.
 *
 * The operation: exact butterfly counts of a simple bipartite graph
 * G = (U, V, E) (§2): the global count, the count per
 * vertex (Eq. (1), on both sides) and the count per edge
 * (Eq. (2)), computed by rank-ordered wedge retrieval and
 * aggregation (Alg. 1 PREPROCESS P:639-657, Alg. 2 GET-WEDGES P:733-749,
 * get-freq P:798-808, Alg. 3 COUNT-V P:821-844, Alg. 4 COUNT-E P:876-893).
 *
 * Conventions (all functions):
 *  - extern "C", no exceptions cross the ABI; every call returns bf_status.
 *  - On error, outputs are unspecified; the graph stays usable except after
 *    BF_ECUDA / BF_ENCCL (then only bf_graph_destroy is valid).
 *    bf_last_error() returns a message for the calling thread's last error.
 *  - Ids are 0-based and side-local: u in [0, n_u), v in [0, n_v).
 *  - Limits: n_u + n_v < 2^32, m < 2^31.  m = 0, n_u = 0, n_v = 0 are legal.
 *  - All counts are exact uint64 (reading Z9); inputs must have < 2^64
 *    butterflies (not checked unless BF_FLAG_CHECK_OVERFLOW).
 *  - Threading: one host thread at a time per bf_graph.  Different graphs
 *    (e.g. on different devices) may be used concurrently.
 *  - Multi-GPU (bf_options.world_size > 1): every rank calls create, rank and
 *    count with identical inputs; bf_count_* is collective over nccl_comm and
 *    every rank receives the full result.  Whenever nccl_comm is set (a
 *    1-rank communicator included) the outputs go through its allreduce.
 */
#ifndef BF_H
#define BF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bf_graph bf_graph; /* opaque; owns all device state */

typedef enum {
  BF_OK = 0,
  BF_EINVAL = 1,     /* bad argument (NULL pointer, size over a limit, bad enum) */
  BF_ERANGE = 2,     /* an edge id is out of range (u >= n_u or v >= n_v)        */
  BF_EDUP = 3,       /* a (u,v) pair occurs twice: the graph must be simple      */
  BF_ENOMEM = 4,     /* device or host allocation failed                        */
  BF_ECUDA = 5,      /* a CUDA call failed (graph no longer usable)             */
  BF_ENCCL = 6,      /* an NCCL call failed, or NCCL could not be loaded        */
  BF_ENORANK = 7,    /* bf_count_* / bf_wedge_count called before bf_rank       */
  BF_EOVERFLOW = 8   /* reserved: debug overflow check tripped                  */
} bf_status;

/* Vertex orderings (§3.1.1).  rank 0 is processed first
 * as the low endpoint x1 of its wedges (reading Z4).
 *  BF_RANK_SIDE          one whole side first: the side whose vertices, as
 *                        endpoints, give fewer wedges, i.e. U first iff
 *                        Σ_{v∈V} C(deg v,2) <= Σ_{u∈U} C(deg u,2) (reading Z1,
 *                        tie -> U); within a side by id.
 *  BF_RANK_APPROX_DEGREE decreasing floor(log2 deg), deg 0 last (reading Z3),
 *                        ties by global id gid = u | n_u + v (reading Z2).
 *  BF_RANK_DEGREE        decreasing degree, ties by gid (reading Z2).
 *  BF_RANK_APPROX_CODEGEN approximate complement degeneracy (P:413-426,
 *                        work-efficient by P:1569-1581): rounds of a parallel
 *                        peel, each removing every remaining vertex whose
 *                        floor(log2 of its degree among the remaining vertices)
 *                        is the current maximum (deg 0 -> -1), at most 33
 *                        rounds; earlier rounds rank first, ties by gid
 *                        (readings Z2, Z16).
 *  BF_RANK_AUTO          the paper's runtime choice: with w_s the
 *                        wedges under side order and w_r the fewest of degree /
 *                        approximate-degree / approximate complement degeneracy
 *                        order (computed before ranking, W = Σ_y (k_y d_y −
 *                        k_y(k_y+1)/2)), side order if f = (w_s − w_r)/w_s <
 *                        0.1, else that other order (ties: degree, approximate
 *                        degree, approximate complement degeneracy).
 *                        bf_rank_info reports the choice.                      */
typedef enum {
  BF_RANK_SIDE = 0,
  BF_RANK_APPROX_DEGREE = 1,
  BF_RANK_DEGREE = 2,
  BF_RANK_AUTO = 3,
  BF_RANK_APPROX_CODEGEN = 4
} bf_rank_kind;

/* Wedge retrieval orientation.  Both retrieve exactly the same wedge set
 * {(x1,y,x2): rank(y) > rank(x1), rank(x2) > rank(x1)} (Fig.
 * fig:framework step 2), so every output is identical.
 *  BF_ORIENT_LOW   Alg. 2 literally: iterate the lower-ranked endpoint x1,
 *                  aggregate by x2.
 *  BF_ORIENT_HIGH  the cache optimisation (§3.1.4; Wang et al.):
 *                  iterate the higher-ranked endpoint x2, aggregate by x1.
 *  BF_ORIENT_AUTO  library choice (currently HIGH).                          */
typedef enum { BF_ORIENT_AUTO = 0, BF_ORIENT_LOW = 1, BF_ORIENT_HIGH = 2 } bf_orient;

/* test_flags bits (path forcing for tests; 0 in production).  Tiers of the
 * work plan: warp tier (w <= 512 wedges and <= 32 slots; per-warp u8 dense
 * key window + overflow hash), CTA medium tier (w <= 2048) and CTA heavy tier
 * (dense shared-memory key window + per-CTA global overflow row); heavy starts
 * above max(2^20, W / (8 * #SMs)) wedges are split into pieces counted by many
 * CTAs into one global d-row.  Results never depend on these flags. */
#define BF_FLAG_FORCE_WARP      0x1u  /* no medium tier: warp tier for every start it
                                         can hold, heavy CTA tier for the rest          */
#define BF_FLAG_FORCE_CTA       0x2u  /* no warp tier: CTA medium / heavy tiers only    */
#define BF_FLAG_SMALL_WINDOW    0x4u  /* shrink every shared-memory key window to 64
                                         keys so most keys take the overflow paths
                                         (warp hash, CTA global row)                    */
#define BF_FLAG_CHECK_OVERFLOW  0x8u  /* reserved                                      */
#define BF_FLAG_FORCE_DENSE     0x10u /* every start on the heavy CTA tier             */
#define BF_FLAG_SMALL_CHUNK     0x20u /* CTA chunks of 64 wedges: every CTA start with
                                         more wedges takes the multi-chunk path; the
                                         split threshold drops to 256 wedges            */
#define BF_FLAG_NO_SPLIT        0x40u /* never split a start across CTAs                */
#define BF_FLAG_UNPACKED_SORT   0x80u /* the slot sort's V-half records carry the twin's
                                         U position (the form taken when bits(|U|) +
                                         2 bits(|V|) > 64, e.g. configs 3 and 5) instead
                                         of (u, index of v in N(u))                     */
#define BF_FLAG_NO_DENSE_ROW    0x100u /* never count split pieces in a whole-key-range
                                         shared row (taken when every heavy start has at
                                         most 40960 same-side keys, e.g. config 4)       */
#define BF_FLAG_KEY_BUFFER      0x200u /* vertex mode: slot-mode walks always keep their
                                         keys for pass 2 (taken when the average
                                         segment is short, e.g. config 4)                */
#define BF_FLAG_GRID_JITTER     0x400u /* race stress: every wedge-kernel launch takes a
                                         pseudo-random grid in [1, its normal grid]
                                         (a different CTA-to-start mapping and
                                         interleaving on every call)                     */
#define BF_FLAG_HUB_POS         0x800u /* ranked CSR build: always rank the U-side twin
                                         positions of up to 256 hub items in slot order
                                         (taken when m >= 2^25 and those items hold at
                                         least a quarter of the slots, e.g. config 4)    */

typedef struct {
  int device;               /* CUDA ordinal                                           */
  void* stream;             /* cudaStream_t to run on; NULL = library-owned stream    */
  void* nccl_comm;          /* ncclComm_t from bf_nccl_comm_create; NULL = 1 GPU      */
  int world_rank;           /* this process's rank in [0, world_size)                 */
  int world_size;           /* number of GPUs sharing the work (1 = single GPU)       */
  int edges_on_device;      /* 1: `edges` in bf_graph_create is a device pointer      */
  int outputs_on_device;    /* 1: output arrays of bf_count_* are device pointers     */
  int orient;               /* bf_orient                                              */
  uint32_t test_light_max_wedges; /* 0 = default warp-path threshold (wedges/start)   */
  uint32_t test_flags;      /* BF_FLAG_* (tests only)                                 */
  int virtual_world;        /* >1: single-GPU emulation of that many ranks: each
                               virtual rank's share is counted in turn and the shares
                               are summed on device, no NCCL (tests only)             */
} bf_options;

/* Fills *opt with defaults: device 0, library stream, 1 GPU, host pointers. */
void bf_options_default(bf_options* opt);

/* Copies the edge list to the device, range-checks it and computes degrees
 * (§8(a) a1).  Repeated (u,v) pairs are rejected by bf_rank, where the ranked
 * slot sort makes them adjacent (no separate hash pass).  edges: m pairs (u, v), uint32, row-major
 * [m][2]; host pointer unless opt->edges_on_device.  The caller keeps
 * ownership of `edges` and may free it after the call returns.
 * opt may be NULL (defaults).  *out receives the graph (NULL on error).
 * Errors: BF_EINVAL (NULL out, size over limit), BF_ERANGE, BF_ENOMEM,
 * BF_ECUDA. */
bf_status bf_graph_create(uint32_t n_u, uint32_t n_v, const uint32_t* edges, uint64_t m,
                          const bf_options* opt, bf_graph** out);

/* Ranks the vertices (§8(a) a2), builds the ranked CSR of Alg. 1 (a3) and
 * the per-start wedge counts and work plan (a4).  Deterministic and identical
 * on every rank.  May be called again to re-rank.  Errors: BF_EINVAL (bad
 * kind / NULL g), BF_EDUP (a (u,v) pair occurs twice: the graph must be
 * simple, reading Z8), BF_ENOMEM, BF_ECUDA. */
bf_status bf_rank(bf_graph* g, bf_rank_kind kind);

/* Global butterfly count (P:487 footnote: Σ over endpoint pairs of C(d,2)).
 * total: one uint64 (host, or device if outputs_on_device).
 * Errors: BF_EINVAL, BF_ENORANK, BF_ECUDA, BF_ENCCL. */
bf_status bf_count_total(bf_graph* g, uint64_t* total);

/* Per-vertex counts (Alg. 3; Eq. (1)) for both sides.  out_u: n_u uint64,
 * out_v: n_v uint64, indexed by input ids; total: nullable, one uint64.
 * Errors as bf_count_total. */
bf_status bf_count_vertex(bf_graph* g, uint64_t* out_u, uint64_t* out_v, uint64_t* total);

/* Per-edge counts (Alg. 4; Eq. (2)).  out_e: m uint64 in INPUT edge order
 * (reading Z7); total: nullable.  Errors as bf_count_total. */
bf_status bf_count_edge(bf_graph* g, uint64_t* out_e, uint64_t* total);

/* W = number of wedges processed under the current ranking,
 * the work metric of wedges/s (reading Z10).  Host output.
 * Errors: BF_EINVAL, BF_ENORANK. */
bf_status bf_wedge_count(const bf_graph* g, uint64_t* w);

/* The ranking in effect after bf_rank (*kind: BF_RANK_SIDE / APPROX_DEGREE /
 * DEGREE / APPROX_CODEGEN; BF_RANK_AUTO resolved) and, after BF_RANK_AUTO
 * only, the wedges each candidate processes (w[0] side, w[1] approximate
 * degree, w[2] degree, w[3] approximate complement degeneracy; zeros
 * otherwise).  Either pointer may be NULL.  Errors: BF_EINVAL, BF_ENORANK. */
bf_status bf_rank_info(const bf_graph* g, int* kind, uint64_t w[4]);

/* Statistics of the last bf_count_* call (host outputs, each nullable):
 * kernel_ms = CUDA-event time of its wedge kernel(s) alone, call_ms = of the
 * whole call (both on the graph's stream); pairs = distinct endpoint pairs
 * (x1,x2) with d >= 1 that were aggregated (summed over ranks' shares on this
 * process; the "P" of the algorithmic-bytes model). */
bf_status bf_last_stats(const bf_graph* g, float* kernel_ms, float* call_ms, uint64_t* pairs);

/* Number of libbf kernel launches issued since the graph was created. */
uint64_t bf_launch_count(const bf_graph* g);

/* Multi-GPU share (host-only, no GPU needed): the q-th start index that rank
 * `rank` of `world` processes inside a tier segment [t0, t1) of the
 * wedge-sorted start list ("snake" deal: round q takes t0 + q*world +
 * (q odd ? world-1-rank : rank)); returns t1 when there is none.  The kernels
 * use the same function.  Wedge-aware batching across GPUs. */
uint64_t bf_deal_index(uint64_t q, int rank, int world, uint64_t t0, uint64_t t1);

/* Multi-GPU work shares of the current plan (host output, after bf_rank):
 * wedges[r] = the wedges rank r of `world` would process -- split starts
 * whole, in snake order over their index, and every tier segment through
 * bf_deal_index -- i.e. exactly the deal the kernels apply for
 * bf_options.world_size = world.  wedges: `world` uint64 (host).
 * Errors: BF_EINVAL, BF_ENORANK, BF_ECUDA. */
bf_status bf_rank_shares(const bf_graph* g, int world, uint64_t* wedges);

/* Debug/test export of the ranked CSR (device -> host copies).  Any pointer
 * may be NULL.  rid_of_gid[n]: rank-space id of global id gid (U-side vertices
 * occupy rid [0,n_u) in rank order, V-side [n_u, n) in rank order);
 * off[n+1], nbr[2m], pos[2m] (index of the slot's source in N(dst)),
 * hi[n] (deg_x(x)), wstart[n] (wedges started at each rid under the current
 * orientation).  Errors: BF_EINVAL, BF_ENORANK, BF_ECUDA. */
bf_status bf_export_csr(const bf_graph* g, uint32_t* rid_of_gid, uint32_t* off, uint32_t* nbr,
                        uint32_t* pos, uint32_t* hi, uint64_t* wstart);

/* NCCL bootstrap (the process group only carries the 128-byte id).  NCCL is
 * loaded at run time (libnccl.so.2); BF_ENCCL if it cannot be loaded. */
bf_status bf_nccl_unique_id(uint8_t id[128]);
bf_status bf_nccl_comm_create(const uint8_t id[128], int rank, int world, int device, void** comm);
bf_status bf_nccl_comm_destroy(void* comm);

/* Approximate total counting by sparsification (§4.4, P:1451-1493;
 * Sanei-Mehri et al.): filters the edge list on the device and writes the kept
 * edges, in input order, to out_edges (capacity m pairs; host unless
 * opt->outputs_on_device) and their number to *out_m.  The caller counts the
 * sparsified graph exactly (bf_graph_create .. bf_count_total, total counts
 * only) and scales the count into an unbiased estimate of T:
 *   BF_SPARSIFY_EDGE   keep edge e iff h(seed, e) < p * 2^64 (each edge with
 *                      probability p)            -> T_s / p^4
 *   BF_SPARSIFY_COLOR  colour(z) = h(seed ^ 0xD1B54A32D192ED03, gid z) mod c,
 *                      c = ceil(1/p); keep an edge iff its endpoints share a
 *                      colour                    -> T_s * c^3
 * h(s, x) = splitmix64 finalizer of s + (x+1) * 0x9E3779B97F4A7C15 (counter
 * based: results depend only on (seed, index)).  edges: m pairs (u, v), host
 * unless opt->edges_on_device; opt may be NULL; ids are not range-checked here
 * (bf_graph_create checks the output).  Errors: BF_EINVAL (NULL pointers, p not
 * in (0,1], bad method, m >= 2^31), BF_ENOMEM, BF_ECUDA. */
#define BF_SPARSIFY_EDGE 0
#define BF_SPARSIFY_COLOR 1
bf_status bf_sparsify(uint32_t n_u, uint32_t n_v, const uint32_t* edges, uint64_t m, int method, double p,
                      uint64_t seed, uint32_t* out_edges, uint64_t* out_m, const bf_options* opt);

/* Approximate total count by sparsification, end to end on the device
 * (P:1451-1493): bf_sparsify, then the kept graph through bf_graph_create,
 * bf_rank(BF_RANK_AUTO) and bf_count_total (same options: device, stream,
 * multi-GPU), then the unbiased scaling -- T_s / p^4 for BF_SPARSIFY_EDGE
 * (each edge kept with probability p) and T_s * c^3 with
 * c = ceil(1/p) colours for BF_SPARSIFY_COLOR (a butterfly survives iff its
 * four vertices share a colour, probability c^-3; reading Z15).
 * edges: host unless opt->edges_on_device.  estimate (host) receives the
 * estimate; sparse_total / sparse_m (host, nullable) the exact count and the
 * edge count of the sparsified graph.  Errors: as bf_sparsify, bf_rank and
 * bf_count_total. */
bf_status bf_approx_total(uint32_t n_u, uint32_t n_v, const uint32_t* edges, uint64_t m, int method, double p,
                          uint64_t seed, const bf_options* opt, double* estimate, uint64_t* sparse_total,
                          uint64_t* sparse_m);

/* Frees all device state of g (NULL is a no-op).  Freed device memory goes
 * back to the library's private per-device pool (not the device's default
 * pool), so the next graph reuses it; see bf_release_device_cache. */
void bf_graph_destroy(bf_graph* g);

/* Returns the library's cached device memory on `device` to the driver: the
 * heavy tier's per-CTA overflow rows (kept zero across calls and graphs, up
 * to 60% of the free device memory and at most 64 GB) and the unused blocks of
 * the private stream-ordered pool.  Safe at
 * any time (a later count reallocates what it needs); synchronises the device.
 * Errors: BF_EINVAL (bad device), BF_ECUDA. */
bf_status bf_release_device_cache(int device);

const char* bf_status_str(bf_status s);
const char* bf_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BF_H */
