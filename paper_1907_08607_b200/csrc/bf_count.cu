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
// Wedge -> lane mapping.  The start's wedges are its slots' segments laid end
// to end; wpre (the per-slot u64 prefix of segment lengths, a4) gives every
// segment's offset directly, so no scan runs here.  A chunk of the start's
// wedge sequence is cut into 32-wedge windows; building the chunk writes, per
// segment, one bit into the window's segment-start bitmap, its id at its start
// position (sst) and its id into every window it opens (wseg).  Lane l of
// window k then finds its segment with one masked bitmap read:
//     m = bits[k] & lanemask_le;  o = m ? sst[32k + 31 - clz(m)] : wseg[k]
// and its key's position in nbr as dlo[o] + 32k + l, summed in u32 (dlo is
// stored modulo 2^32) before it indexes nbr (coalesced reads).
//
// Tiers (wedge-aware batching) over one list of starts sorted by
// (tier, wedges desc), dealt to ranks in snake order:
//   warp   (w <= 512, <= 32 slots): one warp per start; u16 dense key window in
//          shared memory (north_star "shared-memory ... keyed by u2") with an
//          open-addressed shared hash for keys past the window; the start's
//          keys are cached in shared memory for pass 2;
//   medium (w <= 2048, <= 128 slots): one 128-thread CTA per start, same
//          structures at CTA scope, owners marked by per-wedge bits;
//   heavy  (the rest): one 256-thread CTA per start, u32 dense shared window +
//          a per-CTA global dense overflow row (north_star "dense per-CTA
//          counter array"); starts that fit one chunk (<= 4096 wedges) cache
//          their keys and owner bits on chip, larger ones are walked chunk by
//          chunk with a global touched list.
// Counters are reset through the owners (the wedge whose increment took a
// counter from 0 to 1), never by clearing whole rows.
#include "bf_internal.h"
#include "bf_device.cuh"
#include <algorithm>
#include <type_traits>
#include <stdlib.h>

namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t EMPTY = 0xffffffffu;
constexpr int UNR = 4;  // 32-wedge windows in flight per warp

// warp tier
constexpr int WT_WARPS = 4;                       // independent warps per CTA
constexpr uint32_t WT_WIN = 4096;                 // u16 dense window keys per warp
constexpr uint32_t WT_HS = 512;                   // overflow hash slots per warp (>= max keys)
constexpr uint32_t WT_TL = BF_WARP_MAX_WEDGES;    // wedges per warp-tier start
constexpr uint32_t WT_NWIN = WT_TL / 32;
constexpr uint32_t WT_CHUNK = 8;                  // starts per queue grab
static_assert(BF_WARP_MAX_SLOTS == 32, "warp tier: one slot per lane");
static_assert(WT_NWIN % UNR == 0, "warp tier windows unroll");

// medium tier
constexpr int MD_NT = 128;
constexpr uint32_t MD_WIN = 8192;                 // u16 dense window keys
constexpr uint32_t MD_HS = BF_MEDIUM_MAX_WEDGES;  // overflow hash slots (>= max keys)
constexpr uint32_t MD_CAP = BF_MEDIUM_MAX_WEDGES;
static_assert(BF_MEDIUM_MAX_SLOTS == MD_NT, "medium tier: one slot per thread");

// heavy tier
constexpr int HV_NT = 256;
constexpr uint32_t HV_WIN = 16384;                // u32 dense window keys
constexpr uint32_t HV_CAP = 4096;                 // wedges per chunk (cached on chip)

struct CountArgs {
  const uint32_t* nbr;
  const uint64_t* wpre;   // [2m+1] per-slot wedge prefix
  const uint32_t* seglo;  // [2m]   per-slot segment start in nbr
  const uint4* items;     // planned starts {s, j0, j1, -}, sorted by (tier, wedges desc)
  uint64_t* bv;           // [n+1] per-vertex (rid space)
  uint64_t* acc;          // [2m] per-slot (edge mode)
  uint64_t* total;        // [0] total, [1] distinct pairs
  uint32_t* orow;         // heavy: per-CTA overflow rows (indexed by key offset)
  uint32_t* olist;        // heavy: per-CTA touched lists (multi-chunk starts)
  uint64_t orow_len;
  uint32_t* queue;        // tier cursor
  uint32_t n_u, n_v;
  uint32_t t0, t1;        // this tier's segment of the item list
  uint64_t S, n;          // slots, vertices (bounds checks of the debug build)
  uint32_t dbg_stop;      // debug build: stop each start after this phase (0 = never)
  uint32_t win;           // dense window keys in use (<= compile-time size)
  uint32_t cap;           // heavy chunk capacity in wedges (<= HV_CAP)
  int rank, world;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lanemask_le() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(r));
  return r;
}

// q-th start of this rank inside the tier segment (snake deal over the
// wedge-sorted list: round q takes q*G + (q odd ? G-1-r : r)); EMPTY if none
__device__ __forceinline__ uint32_t dealt(const CountArgs& a, uint32_t q) {
  const uint64_t i = bf_deal(q, (uint64_t)a.rank, (uint64_t)a.world, a.t0, a.t1);
  return i < a.t1 ? (uint32_t)i : EMPTY;
}

struct Start {
  uint32_t s, j0, j1, kbase;
};

// key offset kk = key - kbase: HIGH keys are the start's side ranked above it
// (rids [side base, s)), LOW keys the side ranked below it (rids (s, side end))
template <int ORIENT>
__device__ __forceinline__ Start load_start(const CountArgs& a, uint32_t it) {
  BF_CHECK(it >= a.t0 && it < a.t1);
  const uint4 v = __ldg(a.items + it);
  Start t;
  t.s = v.x;
  t.j0 = v.y;
  t.j1 = v.z;
  t.kbase = ORIENT == BF_ORIENT_HIGH ? (t.s < a.n_u ? 0u : a.n_u) : t.s + 1u;
  BF_CHECK(t.s < a.n && t.j0 <= t.j1 && t.j1 <= a.S);
  return t;
}

// Sum v over the lane's run inside a window (runs start at segment starts and
// at lane 0).  `wide` (d may reach 2^27) sums 16-bit halves so nothing wraps.
__device__ __forceinline__ uint64_t run_sum(uint32_t starts, uint32_t v, bool wide, bool& head) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t heads = starts | 1u;
  const uint32_t le = lanemask_le();
  const uint32_t first = 31 - __clz(heads & le);
  const uint32_t after = heads & ~le;
  const uint32_t end = after ? (uint32_t)(__ffs(after) - 1) : 32u;
  const uint32_t rm = (end == 32u ? FULL : ((1u << end) - 1u)) & ~((1u << first) - 1u);
  head = lane == first;
  BF_CHECK(__activemask() == FULL);
  if (!wide) return __reduce_add_sync(rm, v);
  const uint32_t lo = __reduce_add_sync(rm, v & 0xffffu);
  const uint32_t hi = __reduce_add_sync(rm, v >> 16);
  return (uint64_t)lo + ((uint64_t)hi << 16);
}

// u64 add into a (lo, hi) pair of u32 shared counters (native 32-bit shared
// atomics; a 64-bit shared atomicAdd compiles to a CAS loop)
__device__ __forceinline__ void seg_add(uint32_t* slo, uint32_t* shi, uint32_t o, uint64_t v) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(slo + o, lo);
  const uint32_t up = hi + ((old + lo) < old ? 1u : 0u);
  if (up) atomicAdd(shi + o, up);
}

__device__ __forceinline__ void flush_totals(const CountArgs& a, uint64_t tot_acc, uint64_t pair_acc) {
  tot_acc = warp_sum(tot_acc);
  pair_acc = warp_sum(pair_acc);
  if ((threadIdx.x & 31) == 0) {
    if (tot_acc) red_add_u64(a.total, tot_acc);
    if (pair_acc) red_add_u64(a.total + 1, pair_acc);
  }
}

// ------------------------------------------------ small counter store
// u16 dense window over key offsets [0, wl) + open-addressed hash (u32 keys,
// u32 counts) for the rest.  d <= w <= 2048 here, so u16 never wraps.
__device__ __forceinline__ uint32_t hslot(uint32_t key, uint32_t shift) { return (key * 0x9E3779B1u) >> shift; }

struct SmallStore {
  uint32_t* win;  // u16 counters, two per word
  uint32_t* hk;
  uint32_t* hv;
  uint32_t wl, hmask, shift;

  // returns true if this increment took the key's count from 0 to 1
  __device__ __forceinline__ bool add(uint32_t key, uint32_t kk, bool& hashed) const {
    if (kk < wl) {
      BF_CHECK((kk >> 1) < (hmask + 1) * 4 && __isShared(win + (kk >> 1)));
      const uint32_t sh = (kk & 1u) << 4;
      const uint32_t old = atomicAdd(win + (kk >> 1), 1u << sh);
      return ((old >> sh) & 0xffffu) == 0u;
    }
    hashed = true;
    uint32_t h = hslot(key, shift);
    BF_CHECK(h <= hmask);
    for (uint32_t probes = 0;; probes++) {
      if (probes > hmask) __trap();  // more distinct keys than slots: impossible by the tier bound
      uint32_t cur = ((volatile uint32_t*)hk)[h];
      if (cur == EMPTY) {
        cur = atomicCAS(hk + h, EMPTY, key);
        if (cur == EMPTY) cur = key;
      }
      if (cur == key) return atomicAdd(hv + h, 1u) == 0u;
      h = (h + 1) & hmask;
    }
  }
  __device__ __forceinline__ uint32_t get(uint32_t key, uint32_t kk) const {
    if (kk < wl) return ((const uint16_t*)win)[kk];
    uint32_t h = hslot(key, shift);
    for (uint32_t probes = 0; hk[h] != key; probes++) {
      if (probes > hmask) __trap();  // the key was inserted in pass 1
      h = (h + 1) & hmask;
    }
    return hv[h];
  }
  __device__ __forceinline__ void zero(uint32_t kk) const {  // window keys only; the hash is cleared whole
    if (kk < wl) ((uint16_t*)win)[kk] = 0;
  }
};

// ------------------------------------------------ heavy counter store
// u32 dense shared window over [0, wl) + the CTA's global row for the rest
// (L2 atomics; plain reads bypass L1 so they see the atomics' results).
struct HeavyStore {
  uint32_t* win;
  uint32_t* orow;
  uint32_t wl;
  uint64_t lenchk;
  __device__ __forceinline__ bool add(uint32_t, uint32_t kk, bool&) const {
    BF_CHECK(kk < lenchk);
    const uint32_t old = kk < wl ? atomicAdd(win + kk, 1u) : atomicAdd(orow + kk, 1u);
    return old == 0u;
  }
  __device__ __forceinline__ uint32_t get(uint32_t, uint32_t kk) const {
    return kk < wl ? win[kk] : __ldcg(orow + kk);
  }
  __device__ __forceinline__ void zero(uint32_t kk) const {
    if (kk < wl) win[kk] = 0;
    else __stcg(orow + kk, 0u);
  }
};

// ================================================================ warp tier
struct WarpSmem {
  uint32_t win[WT_WIN / 2];     // u16 counters
  uint32_t hk[WT_HS];
  uint32_t hv[WT_HS];
  uint32_t list[WT_TL];         // distinct keys of the start (owners)
  uint32_t cache[WT_TL];        // the start's keys in wedge order (pass 2)
  uint32_t bits[WT_NWIN];       // segment-start bitmap per window
  unsigned long long ssum[32];  // pass-2 per-segment sums
  uint8_t sst[WT_TL];           // segment (= lane) starting at each position
  uint8_t wseg[WT_NWIN];        // segment holding each window's first wedge
};
constexpr size_t WT_SMEM = (size_t)WT_WARPS * sizeof(WarpSmem);

template <int ORIENT, int MODE>
__global__ void __launch_bounds__(WT_WARPS * 32) k_warp(CountArgs a) {
  extern __shared__ __align__(16) char sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem& ws = ((WarpSmem*)sm)[wid];
  const uint32_t le = lanemask_le(), lt = lanemask_lt();
  SmallStore cs;
  cs.win = ws.win;
  cs.hk = ws.hk;
  cs.hv = ws.hv;
  cs.wl = min(a.win, WT_WIN);
  cs.hmask = WT_HS - 1;
  cs.shift = 32 - 9;
  static_assert(WT_HS == 512, "hash shift");
  for (uint32_t i = lane; i < WT_WIN / 2; i += 32) ws.win[i] = 0;
  for (uint32_t i = lane; i < WT_HS; i += 32) { ws.hk[i] = EMPTY; ws.hv[i] = 0; }
  if (lane < WT_NWIN) ws.bits[lane] = 0;
  ws.ssum[lane] = 0;
  __syncwarp();
  uint64_t tot_acc = 0, pair_acc = 0;
  for (;;) {
    uint32_t q0 = 0;
    if (lane == 0) q0 = atomicAdd(a.queue, WT_CHUNK);
    q0 = __shfl_sync(FULL, q0, 0);
    if (dealt(a, q0) == EMPTY) break;
    for (uint32_t q = q0; q < q0 + WT_CHUNK; q++) {
      const uint32_t it = dealt(a, q);
      if (it == EMPTY) break;
      const Start st = load_start<ORIENT>(a, it);
      // lane l <-> slot j0 + l: its segment [A, B) of the start's wedges
      const uint64_t base = __ldg(a.wpre + st.j0);
      const uint32_t j = st.j0 + lane;
      uint32_t A = 0, B = 0, dl = 0, yv = 0;
      if (j < st.j1) {
        A = (uint32_t)(__ldg(a.wpre + j) - base);
        B = (uint32_t)(__ldg(a.wpre + j + 1) - base);
        dl = __ldg(a.seglo + j) - A;
        if (MODE == MODE_VERTEX) yv = __ldg(a.nbr + j);
      }
      const uint32_t tot = __shfl_sync(FULL, B, st.j1 - st.j0 - 1);
      BF_CHECK(B >= A && B <= WT_TL);
      if (B > A) {
        ws.sst[A] = (uint8_t)lane;
        atomicOr(ws.bits + (A >> 5), 1u << (A & 31));
        for (uint32_t k = (A + 31) >> 5; (k << 5) < B; k++) ws.wseg[k] = (uint8_t)lane;
      }
      __syncwarp();
      const uint32_t nwin = (tot + 31) >> 5;

      // ---- pass 1: d(key) += 1 per wedge; owners go to the list
      uint32_t cnt = 0;
      bool hashed = false;
      for (uint32_t k0 = 0; k0 < nwin; k0 += UNR) {
        uint32_t key[UNR];
#pragma unroll
        for (int u = 0; u < UNR; u++) {
          const uint32_t k = k0 + u, pos = (k << 5) + lane;
          const uint32_t mb = ws.bits[k] & le;
          const uint32_t o = mb ? ws.sst[(k << 5) + 31 - __clz(mb)] : ws.wseg[k];
          const uint32_t idx = __shfl_sync(FULL, dl, o) + pos;
          BF_CHECK(pos >= tot || (o < 32 && idx < a.S));
          key[u] = pos < tot ? __ldg(a.nbr + idx) : EMPTY;
        }
#pragma unroll
        for (int u = 0; u < UNR; u++) {
          const uint32_t pos = ((k0 + u) << 5) + lane;
          bool own = false, h = false;
          if (pos < tot) {
            ws.cache[pos] = key[u];
            own = cs.add(key[u], key[u] - st.kbase, h);
          }
          const uint32_t m = __ballot_sync(FULL, own);
          if (own) ws.list[cnt + __popc(m & lt)] = key[u];
          cnt += __popc(m);
          hashed |= __any_sync(FULL, h);
        }
      }
      __syncwarp();

      // ---- finalize: C(d,2) to the total and both endpoints
      uint64_t lsum = 0;
      for (uint32_t i = lane; i < cnt; i += 32) {
        const uint32_t key = ws.list[i], kk = key - st.kbase;
        BF_CHECK(key < a.n && i < WT_TL);
        const uint32_t d = cs.get(key, kk);
        if (MODE == MODE_TOTAL) cs.zero(kk);
        const uint64_t c = choose2(d);
        lsum += c;
        if (MODE == MODE_VERTEX && c) red_add_u64(a.bv + key, c);
      }
      if (lane == 0) pair_acc += cnt;
      tot_acc += lsum;
      if (MODE == MODE_VERTEX) {
        const uint64_t t = warp_sum(lsum);
        if (lane == 0 && t) red_add_u64(a.bv + st.s, t);
      }

      // ---- pass 2: d-1 to the centre (vertex) or both wedge edges (edge)
      if (MODE != MODE_TOTAL) {
        for (uint32_t k = 0; k < nwin; k++) {
          const uint32_t pos = (k << 5) + lane;
          const uint32_t bk = ws.bits[k];
          uint32_t c = 0;
          if (pos < tot) {
            const uint32_t key = ws.cache[pos];
            c = cs.get(key, key - st.kbase) - 1u;
          }
          const uint32_t mb = bk & le;
          const uint32_t o = mb ? ws.sst[(k << 5) + 31 - __clz(mb)] : ws.wseg[k];
          if (MODE == MODE_EDGE) {
            const uint32_t idx = __shfl_sync(FULL, dl, o) + pos;
            if (c) red_add_u64(a.acc + idx, c);  // edge (y, key)
          }
          bool head;
          const uint32_t rs = (uint32_t)run_sum(bk, c, false, head);  // d <= 512: no wrap
          if (head && rs) ws.ssum[o] += rs;
        }
        __syncwarp();
        const unsigned long long v = ws.ssum[lane];
        if (v) {
          if (MODE == MODE_VERTEX) red_add_u64(a.bv + yv, v);  // centre y
          else red_add_u64(a.acc + j, v);                      // edge (s, y)
          ws.ssum[lane] = 0;
        }
        for (uint32_t i = lane; i < cnt; i += 32) cs.zero(ws.list[i] - st.kbase);
      }
      if (hashed)
        for (uint32_t i = lane; i < WT_HS; i += 32) { ws.hk[i] = EMPTY; ws.hv[i] = 0; }
      if (lane < nwin) ws.bits[lane] = 0;
      __syncwarp();
    }
  }
  flush_totals(a, tot_acc, pair_acc);
}

// ================================================================ CTA tiers
template <int NT, uint32_t CAPC>
struct ChunkSmem {
  using SegT = typename std::conditional<(NT <= 256), uint8_t, uint16_t>::type;
  uint32_t cache[CAPC];        // keys in wedge order (single-chunk starts)
  uint32_t own[CAPC / 32];     // owner bit per wedge (single-chunk starts)
  uint32_t bits[CAPC / 32];
  uint32_t dlo[NT];            // per segment: nbr index - chunk position
  uint32_t slo[NT], shi[NT];   // pass-2 per-segment sums
  uint16_t wseg[CAPC / 32];
  SegT sst[CAPC];
  uint32_t jn, item, cnt;
};

template <int NT, uint32_t CAPC>
__device__ __forceinline__ uint32_t seg_of(const ChunkSmem<NT, CAPC>& c, uint32_t k, uint32_t le) {
  BF_CHECK(k < CAPC / 32);
  const uint32_t mb = c.bits[k] & le;
  const uint32_t o = mb ? (uint32_t)c.sst[(k << 5) + 31 - __clz(mb)] : (uint32_t)c.wseg[k];
  BF_CHECK(o < (uint32_t)NT);
  return o;
}

// Build the chunk [K0, K1) of the start's wedge sequence from slots
// [jc, min(jc+NT, j1)).  Thread t handles slot jc + t; `mine` = it has a
// segment in the chunk.  Returns K1; c.jn receives the slot that continues
// past K1 (if any).
template <int MODE, int NT, uint32_t CAPC>
__device__ __forceinline__ uint64_t chunk_build(const CountArgs& a, ChunkSmem<NT, CAPC>& c, uint32_t jc,
                                                uint32_t j1, uint64_t base, uint64_t K0, uint32_t cap, bool& mine,
                                                uint32_t& myj, uint32_t& myy) {
  const uint32_t tid = threadIdx.x;
  const uint32_t jlim = (j1 - jc > (uint32_t)NT) ? jc + NT : j1;
  const uint64_t Kl = __ldg(a.wpre + jlim) - base;
  const uint64_t K1 = min(K0 + cap, Kl);
  const uint32_t j = jc + tid;
  BF_CHECK(jlim <= a.S && jc <= jlim);
  mine = false;
  myj = j;
  myy = 0;
  if (j < jlim) {
    const uint64_t A = __ldg(a.wpre + j) - base, B = __ldg(a.wpre + j + 1) - base;
    if (A <= K1 && K1 < B) c.jn = j;
    if (A < B && A < K1 && B > K0) {  // non-empty segment overlapping [K0, K1)
      const uint64_t a0 = max(A, K0), b0 = min(B, K1);
      const uint32_t la = (uint32_t)(a0 - K0), lb = (uint32_t)(b0 - K0);
      BF_CHECK(la < lb && lb <= CAPC && tid < (uint32_t)NT);
      c.dlo[tid] = __ldg(a.seglo + j) + (uint32_t)(a0 - A) - la;
      c.sst[la] = (typename ChunkSmem<NT, CAPC>::SegT)tid;
      atomicOr(c.bits + (la >> 5), 1u << (la & 31));
      for (uint32_t k = (la + 31) >> 5; (k << 5) < lb; k++) c.wseg[k] = (uint16_t)tid;
      mine = true;
      if (MODE == MODE_VERTEX) myy = __ldg(a.nbr + j);
      if (MODE != MODE_TOTAL) { c.slo[tid] = 0; c.shi[tid] = 0; }
    }
  }
  return K1;
}

// Pass-1 windows of one chunk.  LIST: owners append to the global list;
// otherwise keys and owner bits are cached on chip.
template <bool LIST, int NT, uint32_t CAPC, class Store>
__device__ __forceinline__ void chunk_pass1(const CountArgs& a, ChunkSmem<NT, CAPC>& c, const Store& cs,
                                            uint32_t kbase, uint32_t tot, uint32_t* olist, bool& hashed) {
  constexpr uint32_t NW = NT / 32;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t le = lanemask_le(), lt = lanemask_lt();
  const uint32_t nwin = (tot + 31) >> 5;
  BF_CHECK(tot <= CAPC);
  for (uint32_t k0 = wid * UNR; k0 < nwin; k0 += NW * UNR) {
    uint32_t key[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const uint32_t k = k0 + u, pos = (k << 5) + lane;
      key[u] = EMPTY;
      if (k < nwin) {
        const uint32_t o = seg_of(c, k, le);
        BF_CHECK(pos >= tot || (pos < CAPC && c.dlo[o] + pos < a.S));
        if (pos < tot) key[u] = __ldg(a.nbr + (c.dlo[o] + pos));
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const uint32_t k = k0 + u, pos = (k << 5) + lane;
      if (k >= nwin) break;
      BF_CHECK(pos >= tot || key[u] < a.n);
      bool own = false;
      if (pos < tot) {
        BF_CHECK(__isShared(&c.cache[pos]));
        if (!LIST) c.cache[pos] = key[u];
        own = cs.add(key[u], key[u] - kbase, hashed);
      }
      const uint32_t m = __ballot_sync(FULL, own);
      if (!LIST) {
        if (lane == 0) c.own[k] = m;
      } else if (m) {
        const int ld = __ffs(m) - 1;
        uint32_t b = 0;
        if ((int)lane == ld) b = atomicAdd(&c.cnt, (uint32_t)__popc(m));
        b = __shfl_sync(FULL, b, ld);
        BF_CHECK(!own || b + __popc(m & lt) < a.orow_len);
        if (own) olist[b + __popc(m & lt)] = key[u];
      }
    }
  }
}

// Pass-2 windows of one chunk: c = d(key) - 1 per wedge, summed per segment;
// edge mode also adds c to the wedge's (y, key) edge.  CACHED: keys from the
// chunk cache, and owners (owner bits) finalize C(d,2) on the way.
template <int MODE, bool CACHED, int NT, uint32_t CAPC, class Store>
__device__ __forceinline__ void chunk_pass2(const CountArgs& a, ChunkSmem<NT, CAPC>& c, const Store& cs,
                                            uint32_t kbase, uint32_t tot, bool wide, uint64_t& lsum,
                                            uint64_t& pairs) {
  constexpr uint32_t NW = NT / 32;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t le = lanemask_le();
  const uint32_t nwin = (tot + 31) >> 5;
  for (uint32_t k0 = wid * UNR; k0 < nwin; k0 += NW * UNR) {
    uint32_t key[UNR], o[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const uint32_t k = k0 + u, pos = (k << 5) + lane;
      key[u] = EMPTY;
      o[u] = 0;
      if (k < nwin) {
        o[u] = seg_of(c, k, le);
        BF_CHECK(pos >= tot || CACHED || c.dlo[o[u]] + pos < a.S);
        if (pos < tot) key[u] = CACHED ? c.cache[pos] : __ldg(a.nbr + (c.dlo[o[u]] + pos));
        BF_CHECK(pos >= tot || key[u] < a.n);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const uint32_t k = k0 + u, pos = (k << 5) + lane;
      if (k >= nwin) break;
      uint32_t cc = 0;
      if (pos < tot) {
        const uint32_t d = cs.get(key[u], key[u] - kbase);
        cc = d - 1u;
        if (CACHED && ((c.own[k] >> lane) & 1u)) {
          const uint64_t c2 = choose2(d);
          lsum += c2;
          if (MODE == MODE_VERTEX && c2) red_add_u64(a.bv + key[u], c2);
        }
        BF_CHECK(MODE != MODE_EDGE || c.dlo[o[u]] + pos < a.S);
        if (MODE == MODE_EDGE && cc) red_add_u64(a.acc + (c.dlo[o[u]] + pos), cc);  // edge (y, key)
      }
      if (CACHED && lane == 0) pairs += __popc(c.own[k]);
      bool head;
      const uint64_t rs = run_sum(c.bits[k], cc, wide, head);
      if (head && rs) seg_add(c.slo, c.shi, o[u], rs);
    }
  }
}

template <int MODE>
__device__ __forceinline__ void seg_flush(const CountArgs& a, const uint32_t* slo, const uint32_t* shi, bool mine,
                                          uint32_t myj, uint32_t myy) {
  if (!mine) return;
  const uint32_t t = threadIdx.x;
  const uint64_t v = ((uint64_t)shi[t] << 32) | slo[t];
  if (!v) return;
  BF_CHECK(myy < a.n && myj < a.S);
  if (MODE == MODE_VERTEX) red_add_u64(a.bv + myy, v);  // centre y
  else red_add_u64(a.acc + myj, v);                     // edge (s, y)
}

// One start on a CTA.  MULTI = false requires w <= cap and at most NT slots.
template <int ORIENT, int MODE, bool MULTI, int NT, uint32_t CAPC, class Store>
__device__ __forceinline__ void cta_start(const CountArgs& a, ChunkSmem<NT, CAPC>& c, const Store& cs,
                                          const Start& st, uint64_t base, uint64_t w, uint32_t cap,
                                          uint32_t* olist, uint64_t& lsum, uint64_t& pairs, bool& hashed) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr uint32_t NW = NT / 32;
  const bool wide = (st.j1 - st.j0) >= (1u << 26);  // d <= #slots: 32 * d must not wrap u32
  if (!MULTI) {
    bool mine;
    uint32_t myj, myy;
    chunk_build<MODE, NT, CAPC>(a, c, st.j0, st.j1, base, 0, cap, mine, myj, myy);
    __syncthreads();
    const uint32_t tot = (uint32_t)w, nwin = (tot + 31) >> 5;
#ifdef BF_DEBUG
    if (a.dbg_stop == 2) { for (uint32_t i = tid; i < CAPC / 32; i += NT) c.bits[i] = 0; return; }
#endif
    chunk_pass1<false>(a, c, cs, st.kbase, tot, nullptr, hashed);
    __syncthreads();
#ifdef BF_DEBUG
    if (a.dbg_stop == 3) { for (uint32_t i = tid; i < CAPC / 32; i += NT) c.bits[i] = 0; return; }
#endif
    if (MODE == MODE_TOTAL) {
      for (uint32_t k = wid; k < nwin; k += NW) {
        BF_CHECK(k < CAPC / 32);
        const uint32_t ow = c.own[k];
        if ((ow >> lane) & 1u) {
          BF_CHECK((k << 5) + lane < tot);
          const uint32_t key = c.cache[(k << 5) + lane], kk = key - st.kbase;
          BF_CHECK(key < a.n);
          lsum += choose2(cs.get(key, kk));
          cs.zero(kk);
        }
        if (lane == 0) pairs += __popc(ow);
      }
    } else {
      chunk_pass2<MODE, true>(a, c, cs, st.kbase, tot, wide, lsum, pairs);
      __syncthreads();
      seg_flush<MODE>(a, c.slo, c.shi, mine, myj, myy);
      for (uint32_t k = wid; k < nwin; k += NW)
        if ((c.own[k] >> lane) & 1u) cs.zero(c.cache[(k << 5) + lane] - st.kbase);
    }
    for (uint32_t i = tid; i < nwin; i += NT) c.bits[i] = 0;
    if (tid == 0) c.jn = FULL;
    return;
  }
  // ---- multi-chunk: pass 1 over all chunks, owners to the global list
  if (tid == 0) c.cnt = 0;
  {
    uint32_t jc = st.j0;
    uint64_t K0 = 0;
    while (K0 < w) {
      bool mine;
      uint32_t myj, myy;
      const uint64_t K1 = chunk_build<MODE_TOTAL, NT, CAPC>(a, c, jc, st.j1, base, K0, cap, mine, myj, myy);
      __syncthreads();
      const uint32_t jn = c.jn;
      const uint32_t tot = (uint32_t)(K1 - K0), nwin = (tot + 31) >> 5;
      chunk_pass1<true>(a, c, cs, st.kbase, tot, olist, hashed);
      __syncthreads();
      for (uint32_t i = tid; i < nwin; i += NT) c.bits[i] = 0;
      if (tid == 0) c.jn = FULL;
      __syncthreads();
      jc = jn != FULL ? jn : ((st.j1 - jc > (uint32_t)NT) ? jc + NT : st.j1);
      K0 = K1;
    }
  }
  const uint32_t cnt = c.cnt;
  for (uint32_t i = tid; i < cnt; i += NT) {
    const uint32_t key = __ldcg(olist + i), kk = key - st.kbase;
    const uint32_t d = cs.get(key, kk);
    if (MODE == MODE_TOTAL) cs.zero(kk);
    const uint64_t c2 = choose2(d);
    lsum += c2;
    if (MODE == MODE_VERTEX && c2) red_add_u64(a.bv + key, c2);
  }
  if (tid == 0) pairs += cnt;
  if (MODE == MODE_TOTAL) return;
  __syncthreads();
  {
    uint32_t jc = st.j0;
    uint64_t K0 = 0;
    while (K0 < w) {
      bool mine;
      uint32_t myj, myy;
      const uint64_t K1 = chunk_build<MODE, NT, CAPC>(a, c, jc, st.j1, base, K0, cap, mine, myj, myy);
      __syncthreads();
      const uint32_t jn = c.jn;
      const uint32_t tot = (uint32_t)(K1 - K0), nwin = (tot + 31) >> 5;
      uint64_t dummy = 0;
      chunk_pass2<MODE, false>(a, c, cs, st.kbase, tot, wide, lsum, dummy);
      __syncthreads();
      seg_flush<MODE>(a, c.slo, c.shi, mine, myj, myy);
      for (uint32_t i = tid; i < nwin; i += NT) c.bits[i] = 0;
      if (tid == 0) c.jn = FULL;
      __syncthreads();
      jc = jn != FULL ? jn : ((st.j1 - jc > (uint32_t)NT) ? jc + NT : st.j1);
      K0 = K1;
    }
  }
  for (uint32_t i = tid; i < cnt; i += NT) cs.zero(__ldcg(olist + i) - st.kbase);
}

// ---------------------------------------------------------- medium tier
struct MediumSmem {
  ChunkSmem<MD_NT, MD_CAP> c;
  uint32_t win[MD_WIN / 2];
  uint32_t hk[MD_HS];
  uint32_t hv[MD_HS];
};
constexpr size_t MD_SMEM = sizeof(MediumSmem);

template <int ORIENT, int MODE>
__global__ void __launch_bounds__(MD_NT) k_medium(CountArgs a) {
  extern __shared__ __align__(16) char sm[];
  MediumSmem& ms = *(MediumSmem*)sm;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  SmallStore cs;
  cs.win = ms.win;
  cs.hk = ms.hk;
  cs.hv = ms.hv;
  cs.wl = min(a.win, MD_WIN);
  cs.hmask = MD_HS - 1;
  cs.shift = 32 - 11;
  static_assert(MD_HS == 2048, "hash shift");
  for (uint32_t i = tid; i < MD_WIN / 2; i += MD_NT) ms.win[i] = 0;
  for (uint32_t i = tid; i < MD_HS; i += MD_NT) { ms.hk[i] = EMPTY; ms.hv[i] = 0; }
  for (uint32_t i = tid; i < MD_CAP / 32; i += MD_NT) ms.c.bits[i] = 0;
  if (tid == 0) ms.c.jn = FULL;
  uint64_t tot_acc = 0, pair_acc = 0;
  for (;;) {
    if (tid == 0) ms.c.item = atomicAdd(a.queue, 1u);
    __syncthreads();
    const uint32_t it = dealt(a, ms.c.item);
    if (it == EMPTY) break;
    const Start st = load_start<ORIENT>(a, it);
    const uint64_t base = __ldg(a.wpre + st.j0);
    const uint64_t w = __ldg(a.wpre + st.j1) - base;
    uint64_t lsum = 0;
    bool hashed = false;
#ifdef BF_DEBUG
    BF_CHECK(w <= MD_CAP && st.j1 - st.j0 <= MD_NT);
    if (a.dbg_stop == 1) { __syncthreads(); continue; }
#endif
    cta_start<ORIENT, MODE, false, MD_NT, MD_CAP>(a, ms.c, cs, st, base, w, MD_CAP, nullptr, lsum, pair_acc, hashed);
    tot_acc += lsum;
    if (MODE == MODE_VERTEX) {
      const uint64_t t = warp_sum(lsum);
      if (lane == 0 && t) red_add_u64(a.bv + st.s, t);
    }
    if (__syncthreads_or(hashed))
      for (uint32_t i = tid; i < MD_HS; i += MD_NT) { ms.hk[i] = EMPTY; ms.hv[i] = 0; }
  }
  flush_totals(a, tot_acc, pair_acc);
}

// ----------------------------------------------------------- heavy tier
struct HeavySmem {
  ChunkSmem<HV_NT, HV_CAP> c;
  uint32_t win[HV_WIN];
};
constexpr size_t HV_SMEM = sizeof(HeavySmem);

template <int ORIENT, int MODE>
__global__ void __launch_bounds__(HV_NT) k_heavy(CountArgs a) {
  extern __shared__ __align__(16) char sm[];
  HeavySmem& hs = *(HeavySmem*)sm;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  HeavyStore cs;
  cs.win = hs.win;
  cs.orow = a.orow + (size_t)blockIdx.x * a.orow_len;
  cs.lenchk = a.orow_len;
  cs.wl = min(a.win, HV_WIN);
  uint32_t* olist = a.olist + (size_t)blockIdx.x * a.orow_len;
  const uint32_t cap = min(a.cap, HV_CAP);
  for (uint32_t i = tid; i < HV_WIN; i += HV_NT) hs.win[i] = 0;
  for (uint32_t i = tid; i < HV_CAP / 32; i += HV_NT) hs.c.bits[i] = 0;
  if (tid == 0) hs.c.jn = FULL;
  uint64_t tot_acc = 0, pair_acc = 0;
  for (;;) {
    if (tid == 0) hs.c.item = atomicAdd(a.queue, 1u);
    __syncthreads();
    const uint32_t it = dealt(a, hs.c.item);
    if (it == EMPTY) break;
    const Start st = load_start<ORIENT>(a, it);
    const uint64_t base = __ldg(a.wpre + st.j0);
    const uint64_t w = __ldg(a.wpre + st.j1) - base;
    uint64_t lsum = 0;
    bool hashed = false;
    if (w <= cap && st.j1 - st.j0 <= (uint32_t)HV_NT)
      cta_start<ORIENT, MODE, false, HV_NT, HV_CAP>(a, hs.c, cs, st, base, w, cap, olist, lsum, pair_acc, hashed);
    else
      cta_start<ORIENT, MODE, true, HV_NT, HV_CAP>(a, hs.c, cs, st, base, w, cap, olist, lsum, pair_acc, hashed);
    tot_acc += lsum;
    if (MODE == MODE_VERTEX) {
      const uint64_t t = warp_sum(lsum);
      if (lane == 0 && t) red_add_u64(a.bv + st.s, t);
    }
    __syncthreads();
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
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int b = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem));
  return b > 0 ? b : 1;
}

int heavy_grid(int sms) { return sms * occupancy(k_heavy<BF_ORIENT_HIGH, MODE_VERTEX>, HV_NT, HV_SMEM); }

template <int ORIENT, int MODE>
void launch_tiers(bf_graph* g, CountArgs a, const uint32_t tier[4], uint32_t* queues, cudaStream_t s) {
  const int sms = g->sms;
  if (tier[1] > tier[0]) {  // heavy
    auto k = k_heavy<ORIENT, MODE>;
    const int grid = sms * occupancy(k, HV_NT, HV_SMEM);
    a.t0 = tier[0]; a.t1 = tier[1]; a.queue = queues + 0;
    k<<<grid, HV_NT, HV_SMEM, s>>>(a);
    KERNEL_CHECK(g);
  }
  if (tier[2] > tier[1]) {  // medium
    auto k = k_medium<ORIENT, MODE>;
    const int grid = sms * occupancy(k, MD_NT, MD_SMEM);
    a.t0 = tier[1]; a.t1 = tier[2]; a.queue = queues + 1;
    k<<<grid, MD_NT, MD_SMEM, s>>>(a);
    KERNEL_CHECK(g);
  }
  if (tier[3] > tier[2]) {  // warp
    auto k = k_warp<ORIENT, MODE>;
    const int grid = sms * occupancy(k, WT_WARPS * 32, WT_SMEM);
    a.t0 = tier[2]; a.t1 = tier[3]; a.queue = queues + 2;
    k<<<grid, WT_WARPS * 32, WT_SMEM, s>>>(a);
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
  // heavy tier: one overflow row + touched list per resident CTA, indexed by
  // key offset (< max side size); rows stay zero between starts (owners reset
  // them), so they are cleared once when allocated
  const uint32_t win = (g->opt.test_flags & BF_FLAG_SMALL_WINDOW) ? 64u : 0xFFFFFFFFu;
  const uint32_t cap = (g->opt.test_flags & BF_FLAG_SMALL_CHUNK) ? 64u : HV_CAP;
  const uint64_t olen = std::max<uint64_t>(std::max(g->n_u, g->n_v), 1);
  if (g->n_tier[0]) {
    const size_t rows = (size_t)heavy_grid(g->sms);
    if (g->orow.bytes < rows * olen * 4) {
      g->orow.ensure(rows * olen * 4);
      g->otouch.ensure(rows * olen * 4);
      CUDA_TRY(cudaMemsetAsync(g->orow.p, 0, rows * olen * 4, s));
    }
  }
  CountArgs a;
  a.nbr = g->nbr.as<uint32_t>();
  a.wpre = g->wpre.as<uint64_t>();
  a.seglo = g->seglo.as<uint32_t>();
  a.items = g->items.as<uint4>();
  a.bv = g->bv.as<uint64_t>();
  a.acc = g->acc.as<uint64_t>();
  a.total = dtot;
  a.orow = g->orow.as<uint32_t>();
  a.olist = g->otouch.as<uint32_t>();
  a.orow_len = olen;
  a.S = S;
  a.n = n;
  a.dbg_stop = getenv("BF_DBG_STOP") ? (uint32_t)atoi(getenv("BF_DBG_STOP")) : 0u;
  a.n_u = g->n_u;
  a.n_v = g->n_v;
  a.win = win;
  a.cap = cap;
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
