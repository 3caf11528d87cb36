// bf_count.cu -- the wedge kernels (§8(a) a5-a8) and the count driver.
//
// A "start" s is the vertex whose wedges are aggregated together:
//   BF_ORIENT_LOW  (Alg. 2 GET-WEDGES): s = x1, the lowest-
//                  ranked endpoint; slots i < deg_s(s) = hi[s]; y = N(s)[i];
//                  segment N(y)[0 : deg_s(y)) with deg_s(y) = pos[s->y];
//                  key x2 (rank > s).
//   BF_ORIENT_HIGH (cache optimisation): s = the highest-ranked
//                  endpoint; every slot y = N(s)[i]; segment
//                  N(y)[max(hi[y], pos[s->y]+1) : deg(y)) = neighbours ranked
//                  below both s and y; key = that lowest endpoint.
// Both retrieve the same wedge set, so outputs are identical.
//
// Per start: pass 1 counts d(key) = #wedges per endpoint pair (get-freq,
// P:798-808); finalize adds C(d,2) to the total and to both endpoints (Alg. 3
// l.3-5; P:487 footnote); pass 2 re-walks the same wedges with d
// frozen and adds d-1 to the centre (Alg. 3 l.6-8) or to both wedge
// edges (Alg. 4 l.3-5).  All sums are integer atomics,
// so the result does not depend on scheduling, tier thresholds or GPU count.
//
// Wedge walk (all tiers): a warp takes 32 consecutive slots of its start (one
// per lane), computes each slot's segment, compacts the non-empty ones and
// prefix-sums their lengths; it then visits the flattened wedges 32 at a time
// (coalesced nbr reads).  The segment of each lane's wedge is found without a
// search: one __reduce_or_sync of the segment-start bits inside the 32-wedge
// window, a popc, and a shuffle of the segment's (lo, prefix) from its lane.
//
// Tiers (wedge-aware batching), over one list of starts sorted by
// wedges (descending) and dealt to ranks in snake order:
//   heavy  (w > T2): one 256-thread CTA per start, dense shared-memory counter
//          window over the first 16K keys (hub ids in the HIGH orientation) plus
//          a per-CTA global dense overflow row (north_star "heavy u1 ... dense
//          per-CTA counter array"), reset through touched lists;
//   medium (T1 < w <= T2): one 128-thread CTA per start, CTA-shared open-
//          addressing hash sized to the start;
//   light  (w <= T1): one warp per start, warp-private hash (north_star
//          "light u1 ... shared-memory open-addressed hash keyed by u2").
#include "bf_internal.h"
#include "bf_device.cuh"
#include <algorithm>
#include <vector>
#include <stdlib.h>

namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t EMPTY = 0xffffffffu;

// light tier
constexpr int L_WARPS = 8;                 // warps (= starts in flight) per CTA
constexpr uint32_t L_SLOTS = 1024;         // hash slots per warp -> w <= 512
constexpr uint32_t L_CHUNK = 16;           // starts per queue grab
// medium tier
constexpr int M_WARPS = 4;
constexpr uint32_t M_SLOTS = 4096;         // hash slots per CTA -> w <= 2048
// heavy tier
constexpr int H_WARPS = 8;
constexpr uint32_t H_WIN = 16384;          // dense window (u32 counters)
constexpr int H_PER_SM = 2;                // resident heavy CTAs per SM (overflow rows)

struct WarpScratch {
  uint32_t lo[32], ex[32], y[32], slot[32];
  unsigned long long sum[32];
};

struct CountArgs {
  const uint32_t* off;
  const uint32_t* nbr;
  const uint32_t* pos;
  const uint32_t* hi;
  const uint64_t* wstart;
  const uint32_t* seglo;  // per-slot segment start in nbr
  const uint32_t* seglen; // per-slot segment length
  const uint4* items;     // planned starts {s, j0, j1, w}, sorted by wedges desc
  uint64_t* bv;           // [n+1] per-vertex (rid space)
  uint64_t* acc;          // [2m] per-slot (edge mode)
  uint64_t* total;        // [0] total, [1] distinct pairs
  uint32_t* orow;         // heavy: per-CTA overflow rows
  uint32_t* otouch;       // heavy: per-CTA overflow touched lists
  uint64_t orow_len;
  uint32_t* queue;        // per-tier cursors
  uint32_t n_u, n_v;
  uint32_t t0, t1;        // this tier's segment of `list`
  uint32_t win;           // heavy window size actually used (<= H_WIN)
  int rank, world;
  uint32_t exp;           // timing experiments (BF_EXPERIMENT): 1 = skip key atomics, 2 = skip centre flush
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// q-th start of this rank inside the tier segment (snake deal over the
// wedge-sorted list: round q takes q*G + (q odd ? G-1-r : r)); EMPTY if none
__device__ __forceinline__ uint32_t dealt(const CountArgs& a, uint32_t q) {
  const uint64_t i = bf_deal(q, (uint64_t)a.rank, (uint64_t)a.world, a.t0, a.t1);
  return i < a.t1 ? (uint32_t)i : EMPTY;
}

struct StartInfo {
  uint32_t s, j0, j1, kbase, keyrange;
  uint64_t w;
  bool wide;
};

template <int ORIENT>
__device__ __forceinline__ StartInfo start_info(const CountArgs& a, uint32_t item) {
  const uint4 it = __ldg(a.items + item);
  StartInfo t;
  const uint32_t s = it.x;
  t.s = s;
  const bool isU = s < a.n_u;
  const uint32_t sb = isU ? 0u : a.n_u;
  const uint32_t nside = isU ? a.n_u : a.n_v;
  const uint32_t sl = s - sb;
  t.keyrange = ORIENT == BF_ORIENT_HIGH ? sl : nside - sl - 1u;
  t.kbase = ORIENT == BF_ORIENT_HIGH ? sb : s + 1u;
  t.j0 = it.y;
  t.j1 = it.z;
  t.w = it.w;
  t.wide = (t.j1 - t.j0) >= (1u << 26);  // d <= #slots walked: guards u32 run sums
  return t;
}

// Load the 32-slot sub-batch [b, min(b+32, j1)) into the warp: lane o holds the
// o-th non-empty segment (lo, exclusive prefix); returns the wedge total.
template <bool NEED_Y>
__device__ __forceinline__ uint32_t sub_load(const CountArgs& a, uint32_t b, uint32_t j1, WarpScratch& ws,
                                             uint32_t& nnz, uint32_t& lo_r, uint32_t& ex_r) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t j = b + lane;
  uint32_t y = 0, lo = 0, len = 0;
  if (j < j1) {  // precomputed per-slot segment: one coalesced read
    lo = __ldg(a.seglo + j);
    len = __ldg(a.seglen + j);
    if (NEED_Y) y = __ldg(a.nbr + j);
  }
  const uint32_t nz = __ballot_sync(FULL, len != 0);
  const uint32_t inc = warp_inclusive_scan(len);
  const uint32_t tot = __shfl_sync(FULL, inc, 31);
  if (len) {
    const uint32_t o = __popc(nz & lanemask_lt());
    ws.lo[o] = lo;
    ws.ex[o] = inc - len;
    ws.y[o] = y;
    ws.slot[o] = j;
  }
  __syncwarp();
  nnz = __popc(nz);
  lo_r = ws.lo[lane];
  ex_r = ws.ex[lane];
  return tot;
}

// One 32-wedge window: returns the lane's segment ordinal, sets idx (position
// of the key in nbr) and the window's segment-start mask.
__device__ __forceinline__ uint32_t window(uint32_t k0, uint32_t nnz, uint32_t lo_r, uint32_t ex_r, uint32_t& cur,
                                           uint32_t& mask, uint32_t& idx) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rel = ex_r - k0;
  const uint32_t bit = (lane < nnz && rel < 32u) ? (1u << rel) : 0u;
  mask = __reduce_or_sync(FULL, bit);
  const uint32_t o = cur + __popc(mask & (FULL >> (31 - lane)));
  const uint32_t sl = __shfl_sync(FULL, lo_r, o & 31);
  const uint32_t se = __shfl_sync(FULL, ex_r, o & 31);
  idx = sl + (k0 + lane - se);
  cur += __popc(mask);
  return o;
}

// Sum v over the lane's run (lanes sharing a segment inside the window; run
// heads = segment starts | lane 0).  Exact u64 result on every lane.
__device__ __forceinline__ uint64_t run_sum(uint32_t mask, uint32_t v, bool wide, bool& head) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t heads = mask | 1u;
  const uint32_t le = FULL >> (31 - lane);
  const uint32_t start = 31 - __clz(heads & le);
  const uint32_t after = heads & ~le;
  const uint32_t end = after ? (uint32_t)(__ffs(after) - 1) : 32u;
  const uint32_t rm = (end == 32u ? FULL : ((1u << end) - 1u)) & ~((1u << start) - 1u);
  head = lane == start;
  if (!wide) return __reduce_add_sync(rm, v);
  const uint32_t lo = __reduce_add_sync(rm, v & 0xffffu);
  const uint32_t hi = __reduce_add_sync(rm, v >> 16);
  return (uint64_t)lo + ((uint64_t)hi << 16);
}

// ---------------------------------------------------------------- hash tables
__device__ __forceinline__ uint32_t hslot(uint32_t key, uint32_t shift) { return (key * 0x9E3779B1u) >> shift; }

__device__ __forceinline__ void hash_insert(uint32_t* hk, uint32_t* hv, uint32_t hmask, uint32_t shift, uint32_t key) {
  volatile uint32_t* vk = hk;
  uint32_t h = hslot(key, shift);
  for (uint32_t probes = 0;; probes++) {
    if (probes > hmask) __trap();  // full table: impossible while w <= slots/2
    const uint32_t cur = vk[h];
    if (cur == key) { atomicAdd(&hv[h], 1u); return; }
    if (cur == EMPTY) {
      const uint32_t old = atomicCAS(&hk[h], EMPTY, key);
      if (old == EMPTY || old == key) { atomicAdd(&hv[h], 1u); return; }
    }
    h = (h + 1) & hmask;
  }
}

__device__ __forceinline__ uint32_t hash_find(const uint32_t* hk, const uint32_t* hv, uint32_t hmask, uint32_t shift,
                                              uint32_t key) {
  uint32_t h = hslot(key, shift);
  for (uint32_t probes = 0; hk[h] != key; probes++) {
    if (probes > hmask) __trap();  // the key was inserted in pass 1
    h = (h + 1) & hmask;
  }
  return hv[h];
}

__device__ __forceinline__ uint32_t table_size(uint64_t w, uint32_t keyrange, uint32_t maxslots) {
  const uint64_t want = 2 * (w < (uint64_t)keyrange ? w : (uint64_t)keyrange);
  uint32_t hs = 32;
  while (hs < want && hs < maxslots) hs <<= 1;
  return hs;
}

// ------------------------------------------------------- generic walk passes
// pass 1 over this warp's sub-batches of one start
constexpr int UNR = 4;  // 32-wedge windows in flight per warp (memory-level parallelism)

template <int ORIENT, class Insert>
__device__ __forceinline__ void walk_pass1(const CountArgs& a, const StartInfo& st, uint32_t wi, uint32_t nw,
                                           WarpScratch& ws, Insert&& ins) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t b = st.j0 + wi * 32; b < st.j1; b += nw * 32) {
    uint32_t nnz, lo_r, ex_r;
    const uint32_t tot = sub_load<false>(a, b, st.j1, ws, nnz, lo_r, ex_r);
    uint32_t cur = FULL;
    for (uint32_t k0 = 0; k0 < tot; k0 += 32 * UNR) {
      uint32_t idx[UNR], x2[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        uint32_t mask;
        window(k0 + 32 * u, nnz, lo_r, ex_r, cur, mask, idx[u]);
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) x2[u] = (k0 + 32 * u + lane < tot) ? __ldg(a.nbr + idx[u]) : 0u;
#pragma unroll
      for (int u = 0; u < UNR; u++) ins(k0 + 32 * u + lane < tot, x2[u]);
    }
    __syncwarp();
  }
}

// pass 2: d-1 to centre (vertex) or to both wedge edges (edge)
template <int ORIENT, int MODE, class Find>
__device__ __forceinline__ void walk_pass2(const CountArgs& a, const StartInfo& st, uint32_t wi, uint32_t nw,
                                           WarpScratch& ws, Find&& find) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t b = st.j0 + wi * 32; b < st.j1; b += nw * 32) {
    uint32_t nnz, lo_r, ex_r;
    const uint32_t tot = sub_load<MODE == MODE_VERTEX>(a, b, st.j1, ws, nnz, lo_r, ex_r);
    uint32_t cur = FULL;
    for (uint32_t k0 = 0; k0 < tot; k0 += 32 * UNR) {
      uint32_t idx[UNR], o[UNR], msk[UNR], key[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) o[u] = window(k0 + 32 * u, nnz, lo_r, ex_r, cur, msk[u], idx[u]);
#pragma unroll
      for (int u = 0; u < UNR; u++) key[u] = (k0 + 32 * u + lane < tot) ? __ldg(a.nbr + idx[u]) : 0u;
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const bool act = k0 + 32 * u + lane < tot;
        uint32_t c = 0;
        if (act) {
          c = find(key[u]) - 1u;
          if (MODE == MODE_EDGE && c) red_add_u64(a.acc + idx[u], c);  // edge (y, key)
        }
        bool head;
        const uint64_t rs = run_sum(msk[u], c, st.wide, head);
        if (head && act && rs) ws.sum[o[u]] += rs;
      }
    }
    __syncwarp();
    if (lane < nnz) {
      const uint64_t v = ws.sum[lane];
      if (v && !(a.exp & 2)) {
        if (MODE == MODE_VERTEX) red_add_u64(a.bv + ws.y[lane], v);  // centre y
        else red_add_u64(a.acc + ws.slot[lane], v);                  // edge (s, y)
        ws.sum[lane] = 0;
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------ CTA-level walk (NW warps)
// The whole CTA loads a chunk of 32*NW slots, compacts the non-empty segments
// and prefix-sums them (one block scan of (flag << 40 | len)); warps then take
// groups of UNR consecutive 32-wedge windows, strided over the chunk's
// flattened wedges, so every warp gets work even when the start has few slots.
template <int NW>
struct CtaScratch {
  uint32_t lo[32 * NW], ex[32 * NW + 1], y[32 * NW], slot[32 * NW];
  unsigned long long sum[32 * NW];
  unsigned long long wt[32];
  uint32_t nnz, tot;
};

template <int NW, bool NEED_Y>
__device__ __forceinline__ void cta_chunk_load(const CountArgs& a, uint32_t b, uint32_t j1, CtaScratch<NW>& cs) {
  const uint32_t tid = threadIdx.x;
  const uint32_t j = b + tid;
  uint32_t lo = 0, len = 0, y = 0;
  if (j < j1) {
    lo = __ldg(a.seglo + j);
    len = __ldg(a.seglen + j);
    if (NEED_Y) y = __ldg(a.nbr + j);
  }
  const unsigned long long v = ((unsigned long long)(len != 0) << 40) | len;
  unsigned long long tot;
  const unsigned long long ex = block_exclusive_scan<unsigned long long>(v, cs.wt, &tot);
  if (len) {
    const uint32_t o = (uint32_t)(ex >> 40);
    cs.lo[o] = lo;
    cs.ex[o] = (uint32_t)(ex & 0xFFFFFFFFFFull);
    cs.y[o] = y;
    cs.slot[o] = j;
    cs.sum[o] = 0;
  }
  if (tid == 0) {
    cs.nnz = (uint32_t)(tot >> 40);
    cs.tot = (uint32_t)(tot & 0xFFFFFFFFFFull);
  }
  __syncthreads();
}

// ordinal of the segment holding wedge k0 - 1 (FULL for k0 = 0), searching
// upward from lb with 32-wide ballots
template <int NW>
__device__ __forceinline__ uint32_t cta_seek(const CtaScratch<NW>& cs, uint32_t nnz, uint32_t lb, uint32_t k0) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t c = lb + 1 + lane;
  const bool p = c < nnz && cs.ex[c] < k0;
  const uint32_t m = __ballot_sync(FULL, p);
  if (m != FULL) return lb + __popc(m);
  // more than 32 segments ahead: binary search (ex is increasing)
  uint32_t lo = lb + 32, hi = nnz;  // ex[lo] < k0 <= ex[hi] (ex[nnz] = +inf)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (cs.ex[mid] < k0) lo = mid; else hi = mid;
  }
  return lo;
}

template <int NW>
__device__ __forceinline__ uint32_t cta_window(const CtaScratch<NW>& cs, uint32_t nnz, uint32_t k0, uint32_t& cur,
                                               uint32_t& mask, uint32_t& idx) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t c = cur + 1 + lane;
  uint32_t bit = 0;
  if (c < nnz) {
    const uint32_t rel = cs.ex[c] - k0;
    bit = rel < 32u ? (1u << rel) : 0u;
  }
  mask = __reduce_or_sync(FULL, bit);
  const uint32_t o = cur + __popc(mask & (FULL >> (31 - lane)));
  idx = cs.lo[o] + (k0 + lane - cs.ex[o]);
  cur += __popc(mask);
  return o;
}

template <int NW, class Insert>
__device__ __forceinline__ void cta_pass1(const CountArgs& a, const StartInfo& st, CtaScratch<NW>& cs, Insert&& ins) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t b = st.j0; b < st.j1; b += 32 * NW) {
    cta_chunk_load<NW, false>(a, b, st.j1, cs);
    const uint32_t nnz = cs.nnz, tot = cs.tot;
    uint32_t lb = FULL;
    for (uint32_t K0 = wid * 32 * UNR; K0 < tot; K0 += 32 * UNR * NW) {
      uint32_t cur = cta_seek(cs, nnz, lb, K0);
      lb = cur;
      uint32_t idx[UNR], x2[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        uint32_t mask;
        if (K0 + 32 * u < tot) cta_window(cs, nnz, K0 + 32 * u, cur, mask, idx[u]);
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) x2[u] = (K0 + 32 * u + lane < tot) ? __ldg(a.nbr + idx[u]) : 0u;
#pragma unroll
      for (int u = 0; u < UNR; u++) ins(K0 + 32 * u + lane < tot, x2[u]);
    }
    __syncthreads();
  }
}

template <int NW, int MODE, class Find>
__device__ __forceinline__ void cta_pass2(const CountArgs& a, const StartInfo& st, CtaScratch<NW>& cs, Find&& find) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (uint32_t b = st.j0; b < st.j1; b += 32 * NW) {
    cta_chunk_load<NW, MODE == MODE_VERTEX>(a, b, st.j1, cs);
    const uint32_t nnz = cs.nnz, tot = cs.tot;
    uint32_t lb = FULL;
    for (uint32_t K0 = wid * 32 * UNR; K0 < tot; K0 += 32 * UNR * NW) {
      uint32_t cur = cta_seek(cs, nnz, lb, K0);
      lb = cur;
      uint32_t idx[UNR], o[UNR], msk[UNR], key[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        msk[u] = 0; o[u] = 0; idx[u] = 0;
        if (K0 + 32 * u < tot) o[u] = cta_window(cs, nnz, K0 + 32 * u, cur, msk[u], idx[u]);
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) key[u] = (K0 + 32 * u + lane < tot) ? __ldg(a.nbr + idx[u]) : 0u;
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const bool act = K0 + 32 * u + lane < tot;
        uint32_t c = 0;
        if (act) {
          c = find(key[u]) - 1u;
          if (MODE == MODE_EDGE && c) red_add_u64(a.acc + idx[u], c);  // edge (y, key)
        }
        bool head;
        const uint64_t rs = run_sum(msk[u], c, st.wide, head);
        if (head && act && rs) atomicAdd(&cs.sum[o[u]], (unsigned long long)rs);
      }
    }
    __syncthreads();
    if (tid < nnz) {
      const uint64_t v = cs.sum[tid];
      if (v && !(a.exp & 2)) {
        if (MODE == MODE_VERTEX) red_add_u64(a.bv + cs.y[tid], v);  // centre y
        else red_add_u64(a.acc + cs.slot[tid], v);                  // edge (s, y)
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void flush_totals(const CountArgs& a, uint64_t tot_acc, uint64_t pair_acc) {
  tot_acc = warp_sum(tot_acc);
  pair_acc = warp_sum(pair_acc);
  if ((threadIdx.x & 31) == 0) {
    if (tot_acc) red_add_u64(a.total, tot_acc);
    if (pair_acc) red_add_u64(a.total + 1, pair_acc);
  }
}

// ================================================================ light tier
constexpr size_t L_SMEM = (size_t)L_WARPS * (L_SLOTS * 8 + sizeof(WarpScratch));

template <int ORIENT, int MODE>
__global__ void __launch_bounds__(L_WARPS * 32) k_light(CountArgs a) {
  extern __shared__ __align__(16) char sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* hk = (uint32_t*)sm + (size_t)wid * L_SLOTS * 2;
  uint32_t* hv = hk + L_SLOTS;
  WarpScratch& ws = ((WarpScratch*)(sm + (size_t)L_WARPS * L_SLOTS * 8))[wid];
  ws.sum[lane] = 0;
  uint64_t tot_acc = 0, pair_acc = 0;
  for (;;) {
    uint32_t q0 = 0;
    if (lane == 0) q0 = atomicAdd(a.queue, L_CHUNK);
    q0 = __shfl_sync(FULL, q0, 0);
    if (dealt(a, q0) == EMPTY) break;
    for (uint32_t q = q0; q < q0 + L_CHUNK; q++) {
      const uint32_t it = dealt(a, q);
      if (it == EMPTY) break;
      const StartInfo st = start_info<ORIENT>(a, it);
      const uint32_t s = st.s;
      const uint32_t hs = table_size(st.w, st.keyrange, L_SLOTS);
      const uint32_t hmask = hs - 1, shift = 32 - (31 - __clz(hs));
      for (uint32_t i = lane; i < hs; i += 32) { hk[i] = EMPTY; hv[i] = 0; }
      __syncwarp();
      walk_pass1<ORIENT>(a, st, 0, 1, ws, [&](bool act, uint32_t key) {
        if (act) hash_insert(hk, hv, hmask, shift, key);
      });
      uint64_t lsum = 0;
      for (uint32_t i = lane; i < hs; i += 32) {
        const uint32_t key = hk[i];
        if (key != EMPTY) {
          pair_acc++;
          const uint64_t c = choose2(hv[i]);
          lsum += c;
          if (MODE == MODE_VERTEX && c && !(a.exp & 1)) red_add_u64(a.bv + key, c);
        }
      }
      tot_acc += lsum;
      if (MODE == MODE_VERTEX) {
        lsum = warp_sum(lsum);
        if (lane == 0 && lsum) red_add_u64(a.bv + s, lsum);
      }
      if (MODE != MODE_TOTAL)
        walk_pass2<ORIENT, MODE>(a, st, 0, 1, ws, [&](uint32_t key) { return hash_find(hk, hv, hmask, shift, key); });
      __syncwarp();
    }
  }
  flush_totals(a, tot_acc, pair_acc);
}

// =============================================================== medium tier
template <int ORIENT, int MODE>
__global__ void __launch_bounds__(M_WARPS * 32) k_medium(CountArgs a) {
  __shared__ uint32_t s_hk[M_SLOTS];
  __shared__ uint32_t s_hv[M_SLOTS];
  __shared__ CtaScratch<M_WARPS> cs;
  __shared__ uint32_t s_item;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  constexpr uint32_t NT = M_WARPS * 32;
  uint64_t tot_acc = 0, pair_acc = 0;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(a.queue, 1u);
    __syncthreads();
    const uint32_t it = dealt(a, s_item);
    if (it == EMPTY) break;
    const StartInfo st = start_info<ORIENT>(a, it);
    const uint32_t s = st.s;
    const uint32_t hs = table_size(st.w, st.keyrange, M_SLOTS);
    const uint32_t hmask = hs - 1, shift = 32 - (31 - __clz(hs));
    for (uint32_t i = tid; i < hs; i += NT) { s_hk[i] = EMPTY; s_hv[i] = 0; }
    __syncthreads();
    cta_pass1<M_WARPS>(a, st, cs, [&](bool act, uint32_t key) {
      if (act) hash_insert(s_hk, s_hv, hmask, shift, key);
    });
    uint64_t lsum = 0;
    for (uint32_t i = tid; i < hs; i += NT) {
      const uint32_t key = s_hk[i];
      if (key != EMPTY) {
        pair_acc++;
        const uint64_t c = choose2(s_hv[i]);
        lsum += c;
        if (MODE == MODE_VERTEX && c && !(a.exp & 1)) red_add_u64(a.bv + key, c);
      }
    }
    tot_acc += lsum;
    if (MODE == MODE_VERTEX) {
      lsum = warp_sum(lsum);
      if (lane == 0 && lsum) red_add_u64(a.bv + s, lsum);
    }
    if (MODE != MODE_TOTAL)
      cta_pass2<M_WARPS, MODE>(a, st, cs, [&](uint32_t key) { return hash_find(s_hk, s_hv, hmask, shift, key); });
    __syncthreads();
  }
  flush_totals(a, tot_acc, pair_acc);
}

// ================================================================ heavy tier
constexpr size_t H_SMEM = (size_t)H_WIN * 4 + (size_t)H_WIN * 2 + sizeof(CtaScratch<H_WARPS>) + 64;

template <int ORIENT, int MODE>
__global__ void __launch_bounds__(H_WARPS * 32) k_heavy(CountArgs a) {
  extern __shared__ __align__(16) char sm[];
  uint32_t* win = (uint32_t*)sm;
  uint16_t* touch = (uint16_t*)(sm + (size_t)H_WIN * 4);
  CtaScratch<H_WARPS>& cs = *(CtaScratch<H_WARPS>*)(sm + (size_t)H_WIN * 6);
  __shared__ uint32_t s_item, s_nt, s_no;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  constexpr uint32_t NT = H_WARPS * 32;
  for (uint32_t i = tid; i < H_WIN; i += NT) win[i] = 0;
  if (tid == 0) { s_nt = 0; s_no = 0; }
  uint32_t* orow = a.orow + (size_t)blockIdx.x * a.orow_len;
  uint32_t* otouch = a.otouch + (size_t)blockIdx.x * a.orow_len;
  uint64_t tot_acc = 0, pair_acc = 0;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(a.queue, 1u);
    __syncthreads();
    const uint32_t it = dealt(a, s_item);
    if (it == EMPTY) break;
    const StartInfo st = start_info<ORIENT>(a, it);
    const uint32_t s = st.s;
    const uint32_t wlen = min(a.win, st.keyrange);
    const uint32_t kbase = st.kbase;
    // pass 1: dense window + overflow row, ballot-compacted touched lists
    cta_pass1<H_WARPS>(a, st, cs, [&](bool act, uint32_t x2) {
      const uint32_t key = x2 - kbase;
      bool nw_ = false, no_ = false;
      if (act) {
        if (key < wlen) nw_ = atomicAdd(&win[key], 1u) == 0u;
        else no_ = atomicAdd(&orow[key - wlen], 1u) == 0u;
      }
      const uint32_t mw = __ballot_sync(FULL, nw_);
      if (mw) {
        uint32_t base = 0;
        const int ld = __ffs(mw) - 1;
        if ((int)lane == ld) base = atomicAdd(&s_nt, (uint32_t)__popc(mw));
        base = __shfl_sync(FULL, base, ld);
        if (nw_) touch[base + __popc(mw & lanemask_lt())] = (uint16_t)key;
      }
      const uint32_t mo = __ballot_sync(FULL, no_);
      if (mo) {
        uint32_t base = 0;
        const int ld = __ffs(mo) - 1;
        if ((int)lane == ld) base = atomicAdd(&s_no, (uint32_t)__popc(mo));
        base = __shfl_sync(FULL, base, ld);
        if (no_) otouch[base + __popc(mo & lanemask_lt())] = key - wlen;
      }
    });
    __syncthreads();
    const uint32_t nt = s_nt, no = s_no;
    if (tid == 0) pair_acc += (uint64_t)nt + no;
    uint64_t lsum = 0;
    for (uint32_t t = tid; t < nt; t += NT) {
      const uint32_t key = touch[t];
      const uint64_t c = choose2(win[key]);
      lsum += c;
      if (MODE == MODE_VERTEX && c && !(a.exp & 1)) red_add_u64(a.bv + kbase + key, c);
      if (MODE == MODE_TOTAL) win[key] = 0;
    }
    for (uint32_t t = tid; t < no; t += NT) {
      const uint32_t ok = otouch[t];
      const uint64_t c = choose2(orow[ok]);
      lsum += c;
      if (MODE == MODE_VERTEX && c && !(a.exp & 1)) red_add_u64(a.bv + kbase + wlen + ok, c);
      if (MODE == MODE_TOTAL) orow[ok] = 0;
    }
    tot_acc += lsum;
    if (MODE == MODE_VERTEX) {
      lsum = warp_sum(lsum);
      if (lane == 0 && lsum) red_add_u64(a.bv + s, lsum);
    }
    if (MODE != MODE_TOTAL) {
      __syncthreads();
      cta_pass2<H_WARPS, MODE>(a, st, cs, [&](uint32_t x2) {
        const uint32_t key = x2 - kbase;
        return key < wlen ? win[key] : orow[key - wlen];
      });
      __syncthreads();
      for (uint32_t t = tid; t < nt; t += NT) win[touch[t]] = 0;
      for (uint32_t t = tid; t < no; t += NT) orow[otouch[t]] = 0;
    }
    __syncthreads();
    if (tid == 0) { s_nt = 0; s_no = 0; }
  }
  flush_totals(a, tot_acc, pair_acc);
}

// ============================================================ output kernels
__global__ void k_unrename(const uint64_t* __restrict__ bv, const uint32_t* __restrict__ rid_of_gid, uint32_t nU,
                           uint64_t n, uint64_t* __restrict__ out_u, uint64_t* __restrict__ out_v) {
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = bv[rid_of_gid[z]];
    if (z < nU) out_u[z] = v;
    else out_v[z - nU] = v;
  }
}

__global__ void k_edge_gather(const uint64_t* __restrict__ acc, const uint2* __restrict__ where, uint64_t m,
                              uint64_t* __restrict__ be) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 w = where[e];  // the edge's two slots
    be[e] = acc[w.x] + acc[w.y];
  }
}

inline unsigned grid_for(size_t n, int sms) {
  size_t g = (n + 255) / 256;
  size_t cap = (size_t)sms * 32;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return (unsigned)g;
}

template <class K>
int occupancy(K kernel, int threads, size_t smem) {
  int b = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem));
  return b > 0 ? b : 1;
}

template <int ORIENT, int MODE>
void launch_tiers(bf_graph* g, CountArgs a, const uint32_t tier[4], uint32_t* queues, cudaStream_t s) {
  const int sms = g->sms;
  if (tier[1] > tier[0]) {  // heavy
    auto k = k_heavy<ORIENT, MODE>;
    CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H_SMEM));
    const int grid = sms * std::min(occupancy(k, H_WARPS * 32, H_SMEM), H_PER_SM);
    a.t0 = tier[0]; a.t1 = tier[1]; a.queue = queues + 0;
    k<<<grid, H_WARPS * 32, H_SMEM, s>>>(a);
    KERNEL_CHECK(g);
  }
  if (tier[2] > tier[1]) {  // medium
    auto k = k_medium<ORIENT, MODE>;
    const int grid = sms * occupancy(k, M_WARPS * 32, 0);
    a.t0 = tier[1]; a.t1 = tier[2]; a.queue = queues + 1;
    k<<<grid, M_WARPS * 32, 0, s>>>(a);
    KERNEL_CHECK(g);
  }
  if (tier[3] > tier[2]) {  // light
    auto k = k_light<ORIENT, MODE>;
    CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L_SMEM));
    const int grid = sms * occupancy(k, L_WARPS * 32, L_SMEM);
    a.t0 = tier[2]; a.t1 = tier[3]; a.queue = queues + 2;
    k<<<grid, L_WARPS * 32, L_SMEM, s>>>(a);
    KERNEL_CHECK(g);
  }
}

}  // namespace

bf_status graph_count(bf_graph* g, int mode, uint64_t* out_a, uint64_t* out_b, uint64_t* total) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n, m = g->m, S = 2 * m;
  CUDA_TRY(cudaEventRecord(g->ev[0], s));
  g->bv.ensure((std::max<uint64_t>(n, 1) + 1) * 8);
  g->total.ensure(64);
  g->queue.ensure(64);
  uint64_t* dtot = g->total.as<uint64_t>();
  CUDA_TRY(cudaMemsetAsync(dtot, 0, 16, s));
  if (mode == MODE_VERTEX) CUDA_TRY(cudaMemsetAsync(g->bv.p, 0, (n + 1) * 8, s));
  if (mode == MODE_EDGE) {
    g->acc.ensure(std::max<uint64_t>(S, 1) * 8);
    g->be.ensure((std::max<uint64_t>(m, 1) + 1) * 8);
    CUDA_TRY(cudaMemsetAsync(g->acc.p, 0, std::max<uint64_t>(S, 1) * 8, s));
  }
  // heavy tier overflow rows: one per resident heavy CTA, kept zero between
  // starts through the touched lists
  const uint32_t win = (g->opt.test_flags & BF_FLAG_SMALL_WINDOW) ? 64u : H_WIN;
  const uint64_t maxside = std::max(g->n_u, g->n_v);
  const uint64_t olen = maxside > win ? maxside - win : 1;
  const size_t hrows = (size_t)g->sms * H_PER_SM;
  if (g->n_tier[0] && g->orow.bytes < hrows * olen * 4) {
    g->orow.ensure(hrows * olen * 4);
    g->otouch.ensure(hrows * olen * 4);
    CUDA_TRY(cudaMemsetAsync(g->orow.p, 0, hrows * olen * 4, s));
  }
  CountArgs a;
  a.off = g->off.as<uint32_t>();
  a.nbr = g->nbr.as<uint32_t>();
  a.pos = g->pos.as<uint32_t>();
  a.hi = g->hi.as<uint32_t>();
  a.wstart = g->wstart.as<uint64_t>();
  a.seglo = g->seglo.as<uint32_t>();
  a.seglen = g->seglen.as<uint32_t>();
  a.items = g->items.as<uint4>();
  a.bv = g->bv.as<uint64_t>();
  a.acc = g->acc.as<uint64_t>();
  a.total = dtot;
  a.orow = g->orow.as<uint32_t>();
  a.otouch = g->otouch.as<uint32_t>();
  a.orow_len = olen;
  a.n_u = g->n_u;
  a.n_v = g->n_v;
  a.win = win;
  a.exp = getenv("BF_EXPERIMENT") ? (uint32_t)atoi(getenv("BF_EXPERIMENT")) : 0u;
  const uint32_t tier[4] = {0, g->n_tier[0], g->n_tier[0] + g->n_tier[1],
                            g->n_tier[0] + g->n_tier[1] + g->n_tier[2]};
  const int V = g->opt.virtual_world > 1 ? g->opt.virtual_world : 1;
  const int G = g->opt.world_size > 1 ? g->opt.world_size : V;
  const int first = g->opt.world_size > 1 ? g->opt.world_rank : 0;
  const int last = g->opt.world_size > 1 ? g->opt.world_rank : V - 1;
  CUDA_TRY(cudaEventRecord(g->ev[1], s));
  for (int r = first; r <= last; r++) {
    a.rank = r;
    a.world = G;
    CUDA_TRY(cudaMemsetAsync(g->queue.p, 0, 16, s));
    uint32_t* q = g->queue.as<uint32_t>();
    if (g->orient == BF_ORIENT_LOW) {
      if (mode == MODE_TOTAL) launch_tiers<BF_ORIENT_LOW, MODE_TOTAL>(g, a, tier, q, s);
      else if (mode == MODE_VERTEX) launch_tiers<BF_ORIENT_LOW, MODE_VERTEX>(g, a, tier, q, s);
      else launch_tiers<BF_ORIENT_LOW, MODE_EDGE>(g, a, tier, q, s);
    } else {
      if (mode == MODE_TOTAL) launch_tiers<BF_ORIENT_HIGH, MODE_TOTAL>(g, a, tier, q, s);
      else if (mode == MODE_VERTEX) launch_tiers<BF_ORIENT_HIGH, MODE_VERTEX>(g, a, tier, q, s);
      else launch_tiers<BF_ORIENT_HIGH, MODE_EDGE>(g, a, tier, q, s);
    }
  }
  CUDA_TRY(cudaEventRecord(g->ev[2], s));
  // a8: outputs (total stored after the array so one allreduce covers both)
  uint64_t* red_buf = nullptr;
  size_t red_cnt = 0;
  if (mode == MODE_VERTEX) {
    CUDA_TRY(cudaMemcpyAsync(g->bv.as<uint64_t>() + n, dtot, 8, cudaMemcpyDeviceToDevice, s));
    red_buf = g->bv.as<uint64_t>();
    red_cnt = n + 1;
  } else if (mode == MODE_EDGE) {
    if (m) {
      k_edge_gather<<<grid_for(m, g->sms), 256, 0, s>>>(g->acc.as<uint64_t>(), g->where.as<uint2>(), m,
                                                         g->be.as<uint64_t>());
      KERNEL_CHECK(g);
    }
    CUDA_TRY(cudaMemcpyAsync(g->be.as<uint64_t>() + m, dtot, 8, cudaMemcpyDeviceToDevice, s));
    red_buf = g->be.as<uint64_t>();
    red_cnt = m + 1;
  } else {
    red_buf = dtot;
    red_cnt = 1;
  }
  // a9: combine across GPUs
  if (g->opt.world_size > 1) {
    bf_status st = nccl_allreduce_u64(g->opt.nccl_comm, red_buf, red_cnt, s);
    if (st != BF_OK) return st;
  }
  const cudaMemcpyKind k_out = g->opt.outputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (mode == MODE_VERTEX) {
    uint64_t* du = out_a;
    uint64_t* dvv = out_b;
    if (!g->opt.outputs_on_device) {  // gather on device, then two copies out
      g->tmp_e.ensure((std::max<uint64_t>(n, 1) + 2) * 8);
      du = g->tmp_e.as<uint64_t>();
      dvv = du + g->n_u;
    }
    if (n) {
      k_unrename<<<grid_for(n, g->sms), 256, 0, s>>>(g->bv.as<uint64_t>(), g->rid_of_gid.as<uint32_t>(), g->n_u,
                                                      n, du, dvv);
      KERNEL_CHECK(g);
    }
    if (!g->opt.outputs_on_device) {
      if (g->n_u) CUDA_TRY(cudaMemcpyAsync(out_a, du, (size_t)g->n_u * 8, cudaMemcpyDeviceToHost, s));
      if (g->n_v) CUDA_TRY(cudaMemcpyAsync(out_b, dvv, (size_t)g->n_v * 8, cudaMemcpyDeviceToHost, s));
    }
    if (total) CUDA_TRY(cudaMemcpyAsync(total, red_buf + n, 8, k_out, s));
  } else if (mode == MODE_EDGE) {
    if (m) CUDA_TRY(cudaMemcpyAsync(out_a, g->be.p, m * 8, k_out, s));
    if (total) CUDA_TRY(cudaMemcpyAsync(total, red_buf + m, 8, k_out, s));
  } else {
    CUDA_TRY(cudaMemcpyAsync(total, dtot, 8, k_out, s));
  }
  uint64_t hpairs = 0;
  CUDA_TRY(cudaMemcpyAsync(&hpairs, dtot + 1, 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaEventRecord(g->ev[3], s));
  CUDA_TRY(cudaStreamSynchronize(s));
  g->last_pairs = hpairs;
  CUDA_TRY(cudaEventElapsedTime(&g->last_kernel_ms, g->ev[1], g->ev[2]));
  CUDA_TRY(cudaEventElapsedTime(&g->last_call_ms, g->ev[0], g->ev[3]));
  return BF_OK;
}
