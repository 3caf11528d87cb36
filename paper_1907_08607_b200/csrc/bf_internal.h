// bf_internal.h -- internal declarations of libbf (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <string>
#include <vector>
#include "../../include/bf.h"
#include <nvtx3/nvToolsExt.h>

// NVTX range per phase (§8(a) rows) for nsys / ncu --nvtx; header-only, a
// no-op unless a tool injects itself
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

#define BF_SMS_DEFAULT 148

// work-plan tiers (a4): warp tier for w <= BF_WARP_MAX_WEDGES and at most
// BF_WARP_MAX_SLOTS slots; CTA medium tier for w <= BF_MEDIUM_MAX_WEDGES; CTA
// heavy tier above.  The kernels' shared-memory layouts are sized from these.
#ifndef BF_WARP_MAX_WEDGES
#define BF_WARP_MAX_WEDGES 512u
#endif
#define BF_WARP_MAX_SLOTS 32u
#ifndef BF_MEDIUM_MAX_WEDGES
#define BF_MEDIUM_MAX_WEDGES 2048u
#endif
#ifndef BF_MEDIUM_MAX_SLOTS
#define BF_MEDIUM_MAX_SLOTS 128u  // = the medium kernel's CTA size (one slot per thread)
#endif
// split starts: at most this many (largest first); row memory per batch
constexpr uint32_t kMaxSplit = 4096;
constexpr size_t kSplitRowBudget = (size_t)4 << 30;

// ---- error plumbing --------------------------------------------------------
void bf_set_error(const char* fmt, ...);
struct bf_cuda_error {
  cudaError_t err;
  const char* what;
  int line;
};
#define CUDA_TRY(x)                                                   \
  do {                                                                \
    cudaError_t e_ = (x);                                             \
    if (e_ != cudaSuccess) throw bf_cuda_error{e_, #x, __LINE__};     \
  } while (0)
#define KERNEL_CHECK(g) do { (g)->launches++; CUDA_TRY(cudaGetLastError()); } while (0)

// ---- scratch allocation ------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;  // stream-ordered allocation
  cudaMemPool_t pool = nullptr;  // the library's private pool of the graph's device
  void ensure(size_t n);  // grow (no copy); throws bf_cuda_error
  void release();
  template <class T> T* as() const { return (T*)p; }
};

// ---- library-owned per-device state (bf_api.cu) --------------------------------
// Every graph attaches to its device's library-owned caches: a private
// stream-ordered memory pool (freed blocks stay cached, so repeated
// create/destroy does not return to the driver; the device's default pool is
// left alone) and the heavy tier's row pool (bf_count.cu).  Both persist
// across graphs until bf_release_device_cache(device).
cudaMemPool_t device_attach(int dev);  // throws bf_cuda_error
void device_detach(int dev);
void row_pool_free(int dev);  // bf_count.cu (takes the pool's lock)

// ---- primitives (bf_prims.cu) -------------------------------------------------
// Exclusive scan out[i] = Σ_{j<i} in[j]; *total (device, nullable) = Σ in.
// Types: (u32->u32), (u64->u64), (u32->u64).
size_t scan_temp_bytes(size_t n);
void scan_exclusive_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* total, void* temp,
                        cudaStream_t s, uint64_t* launches);
void scan_exclusive_u64(const uint64_t* in, uint64_t* out, size_t n, uint64_t* total, void* temp,
                        cudaStream_t s, uint64_t* launches);
void scan_exclusive_u32_u64(const uint32_t* in, uint64_t* out, size_t n, uint64_t* total, void* temp,
                            cudaStream_t s, uint64_t* launches);

// Stable LSD radix sort by bits [begin_bit, end_bit) of the key, carrying u32
// values (vals may be null).  Ping-pongs between (k0,v0) and (k1,v1); returns
// 0 if the result is in (k0,v0), 1 if in (k1,v1).
size_t radix_temp_bytes(size_t n);
int radix_sort_u32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, size_t n, int begin_bit,
                   int end_bit, void* temp, cudaStream_t s, uint64_t* launches);
int radix_sort_u64(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, size_t n, int begin_bit,
                   int end_bit, void* temp, cudaStream_t s, uint64_t* launches);
// The slot sort of Alg. 1 (bf_prims.cu), one half at a time; every record is
// one u64 key, the last pass writes the decoded CSR range instead of keys.
// U half: keys (rid(src)) << Bv | (n-1 - rid(dst)) over Bu + Bv bits; writes
// nbr, src (pointers at the range's start) and the V half's input records to
// vrec: at m-1-p, (rid(dst) - nU) << Be | p for the slot at U position p.
// V half: sorts those records on their v field alone (they arrive in
// descending-u order); writes nbr, src (range-local) and the twin indices
// pos[q] = p - off[u], pos[p] = q - off[v] (global; usrc = the U half's src).
// carry (Bu + 2 Bv <= 64): the V records are (v, u, index of v in N(u)) instead
// of (v, U position), so the V decode gathers nothing from the U half's src.
void radix_sort_slots_u(uint64_t* k0, uint64_t* k1, size_t m, int Bu, int Bv, int Be, uint64_t n, uint32_t* nbr,
                        uint32_t* src, uint64_t* vrec, uint64_t nU, const uint32_t* off, bool carry, void* temp,
                        cudaStream_t s, uint64_t* launches);
void radix_sort_slots_v(uint64_t* k0, uint64_t* k1, size_t m, int Bu, int Bv, int Be, uint64_t nU, uint32_t* nbr,
                        uint32_t* src, uint32_t* pos, const uint32_t* off, const uint32_t* usrc, bool carry,
                        const uint32_t* hub, void* temp, cudaStream_t s, uint64_t* launches);
// Hub twin positions (bf_prims.cu): hub_select writes hub = {lo, hi}, the global rid range of up to
// 256 V vertices at the heavier end of the V side when they hold >= 1/4 of the slots (or force), else
// {0, 0}; hub_pos writes pos[p] for the U-half slots p whose neighbour is a hub by ranking them in
// slot order (index of u in N(v) = deg(v) - 1 - earlier U-half slots with the same v); the V half's
// decode (radix_sort_slots_v with the same hub) skips its scatter for those slots.
void hub_select(const uint32_t* off, uint32_t nU, uint64_t n, uint64_t m, bool force, uint32_t* hub, cudaStream_t s,
                uint64_t* launches);
void hub_pos(const uint32_t* nbr, size_t m, const uint32_t* hub, const uint32_t* off, uint32_t* pos, void* temp,
             cudaStream_t s, uint64_t* launches);

static inline int ceil_log2_u64(uint64_t x) {  // bits needed to hold values < x (x>=1)
  int b = 0;
  while (b < 64 && ((x - 1) >> b)) b++;
  return b;
}

// ---- multi-GPU share (snake deal over a wedge-sorted list) -------------------
// q-th item of rank r (of G) inside [t0, t1): round q takes index
// t0 + q*G + (q odd ? G-1-r : r).  Returns t1 when rank r has no q-th item.
// Used by the kernels and exported (bf_deal_index) for host-side tests.
#ifdef __CUDACC__
__host__ __device__
#endif
static inline uint64_t bf_deal(uint64_t q, uint64_t r, uint64_t G, uint64_t t0, uint64_t t1) {
  const uint64_t i = t0 + q * G + ((q & 1u) ? (G - 1 - r) : r);
  return i < t1 ? i : t1;
}

// ---- graph object -----------------------------------------------------------
struct bf_graph {
  bf_options opt;
  int device = 0;
  int sms = BF_SMS_DEFAULT;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool broken = false;  // after a CUDA/NCCL error
  bool attached = false;  // holds a device_attach reference
  uint64_t launches = 0;
  uint64_t jitter = 0;   // BF_FLAG_GRID_JITTER: launches drawn so far

  uint32_t n_u = 0, n_v = 0;
  uint64_t n = 0, m = 0;

  // a1: edges + degrees
  DevBuf edges;  // uint32 [m][2]
  DevBuf deg;    // uint32 [n], gid order

  // a2/a3: ranking and ranked CSR (rid space)
  bool ranked = false;
  int rank_kind = -1;       // the ranking in effect (BF_RANK_AUTO resolves to one of the others)
  uint64_t w_auto[4] = {0, 0, 0, 0};  // BF_RANK_AUTO: W under side, approx.-degree, degree, approx. codegen order
  DevBuf peel;                // u8 [n] removal round of approximate complement degeneracy (gid order)
  bool peel_valid = false;
  int orient = BF_ORIENT_HIGH;
  DevBuf rid_of_gid;  // u32 [n]
  DevBuf gid_of_rid;  // u32 [n]
  DevBuf rkey;        // u64 [n]  rank key per rid (cross-side comparisons)
  DevBuf off;         // u32 [n+1]
  DevBuf nbr;         // u32 [2m]
  DevBuf pos;         // u32 [2m]  index of src in N(dst)
  DevBuf hi;          // u32 [n]   deg_x(x)
  DevBuf wstart;      // u64 [n]   wedges per start rid (current orientation)
  DevBuf seglo;       // u32 [2m]  per slot (s->y): first index in nbr of its wedge segment
  DevBuf seglen;      // u32 [2m]  per slot: segment length (scratch of the plan)
  DevBuf wpre;        // u64 [2m+1] exclusive prefix of per-slot wedge counts (chunking inside a start)
  DevBuf items;       // uint4 per planned start: {s, j0, j1, min(w, 2^32-1)}
  uint64_t W = 0;     // total wedges

  // a4: work plan: starts with w > 0 sorted by wedges (desc, ties by rid);
  // tiers are consecutive segments: heavy (w > t2), medium (t1 < w <= t2),
  // light (w <= t1)
  DevBuf order;         // u32 [n_tier sum]
  uint32_t n_tier[3] = {0, 0, 0};
  uint64_t heavy_keys = 1;  // max key range of a heavy start (sizes the heavy rows)
  size_t pool_budget = 0;   // bytes the heavy tier's row pool may hold (set per count)
  uint32_t t1 = 512, t2 = 2048;

  // split starts (a4): the first n_split heavy starts (w > split threshold)
  // are cut into pieces counted by many CTAs into one shared global d-row per
  // start, then finalized separately.  Batches bound the rows' memory.
  uint32_t n_split = 0;
  uint64_t split_threshold = 0;
  struct SplitBatch {
    uint32_t s0, s1;      // split starts [s0, s1)
    uint32_t p0, p1;      // their pieces [p0, p1)
    uint64_t keys;        // row keys of the batch (sum of key ranges)
  };
  std::vector<SplitBatch> split_batches;
  DevBuf split;      // uint4 [n_split] {s, j0, j1, -}
  DevBuf split_off;  // u64 [n_split] row offset (keys) inside the batch's rows
  DevBuf split_cnt;  // u32 [n_split] touched-list counts
  DevBuf pieces;     // uint4 [n_pieces] {split index, slot begin, slot end, -}
  std::vector<uint4> h_items;        // host copy of the first items (split planning)
  std::vector<uint64_t> h_split_off;  // host split tables (sources of async uploads)
  std::vector<uint4> h_pdesc;
  DevBuf srow;       // u32 dense d-rows of the largest batch (kept zero between calls)
  DevBuf slist;      // u32 touched lists (same layout as srow)

  // a5-a7: counting outputs / scratch
  DevBuf bv;      // u64 [n] per-vertex (rid space)
  DevBuf acc;     // u64 [2m] per-slot accumulators (edge mode)
  DevBuf kbuf;    // u32 [W] slot-mode key buffer (vertex mode, short-segment graphs)
  DevBuf be;      // u64 [m]
  DevBuf total;   // u64 [4] device scalars
  DevBuf orow;    // u32 per-CTA global overflow rows
  DevBuf otouch;  // u32 per-CTA global touched lists (multi-chunk starts)
  DevBuf queue;   // u32 [4] work-queue counters
  DevBuf hub;     // u64 striped endpoint sums of hub keys (vertex mode)
  DevBuf dflag;   // u32 duplicate-edge flag of the ranked slot sort

  // temp for primitives
  DevBuf tmp_a, tmp_b, tmp_c, tmp_d, tmp_e, tmp_f, tmp_scan;

  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  float last_kernel_ms = 0, last_call_ms = 0;
  uint64_t last_pairs = 0;  // distinct endpoint pairs (d >= 1) aggregated by the last count

  template <class F> void for_each_buf(F f) {
    DevBuf* bufs[] = {&edges, &deg, &rid_of_gid, &gid_of_rid, &rkey, &off, &nbr, &pos, &hi,
                      &wstart, &peel, &seglo, &seglen, &wpre, &items, &order, &bv, &acc, &kbuf, &be, &total, &orow, &otouch, &queue, &hub, &dflag, &split, &split_off, &split_cnt, &pieces, &srow, &slist,
                      &tmp_a, &tmp_b, &tmp_c, &tmp_d, &tmp_e, &tmp_f, &tmp_scan};
    for (DevBuf* b : bufs) f(*b);
  }
};

// ---- phases -------------------------------------------------------------------
bf_status graph_ingest(bf_graph* g, const uint32_t* edges);        // bf_build.cu
bf_status graph_rank(bf_graph* g, int kind);                        // bf_build.cu
bf_status graph_plan(bf_graph* g);                                  // bf_build.cu
enum { MODE_TOTAL = 0, MODE_VERTEX = 1, MODE_EDGE = 2 };
bf_status graph_count(bf_graph* g, int mode, uint64_t* out_a, uint64_t* out_b, uint64_t* total);  // bf_count.cu

// NCCL (bf_nccl.cpp)
bf_status nccl_allreduce_u64(void* comm, uint64_t* buf, size_t count, cudaStream_t s);
