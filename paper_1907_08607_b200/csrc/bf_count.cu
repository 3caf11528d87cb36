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
//   warp   (w <= 512, <= 32 slots): one warp per start; u8 dense key window in
//          shared memory (north_star "shared-memory ... keyed by u2") with an
//          open-addressed shared hash for keys past the window; pass 2 re-reads
//          the keys through L1;
//   medium (w <= 2048, <= 128 slots): one 128-thread CTA per start, same
//          structures at CTA scope;
//   heavy  (the rest): one 256-thread CTA per start, u32 dense shared window +
//          a per-CTA global dense overflow row (north_star "dense per-CTA
//          counter array"); starts of one chunk (<= 32768 wedges) reuse their
//          unit table in pass 2, larger ones are walked chunk by chunk with a
//          global touched list.
// Counters are reset through the owners (the wedge whose increment took a
// counter from 0 to 1), never by clearing whole rows.
#include "bf_internal.h"
#include "bf_device.cuh"
#include <algorithm>
#include <type_traits>
#include <map>
#include <mutex>
#include <tuple>
#include <stdlib.h>
#include <stdio.h>

namespace {

constexpr uint32_t FULL = 0xffffffffu;
constexpr uint32_t EMPTY = 0xffffffffu;
struct CountArgs {
  const uint32_t* nbr;
  const uint64_t* wpre;   // [2m+1] per-slot wedge prefix
  const uint32_t* seglo;  // [2m]   per-slot segment start in nbr
  const uint32_t* seglen; // [2m]   per-slot segment length (wedges through the slot)
  const uint4* items;     // planned starts {s, j0, j1, -}, sorted by (tier, wedges desc)
  uint64_t* bv;           // [n+1] per-vertex (rid space)
  uint64_t* hub;          // [HUB_STRIPES][2][HUB_KEYS] striped endpoint sums of hub keys (vertex mode)
  uint64_t* acc;          // [2m] per-slot (edge mode)
  uint64_t* total;        // [0] total, [1] distinct pairs
  uint32_t* orow;         // heavy: per-CTA overflow rows (indexed by key offset)
  uint32_t* olist;        // heavy: per-CTA touched lists (multi-chunk starts)
  uint64_t orow_len;       // heavy overflow row length (max heavy key range - heavy window)
  uint64_t olist_len;      // heavy touched-list capacity beyond the shared list (max heavy key range)
  uint32_t* queue;        // tier cursor
  uint32_t n_u, n_v;
  uint32_t t0, t1;        // this tier's segment of the item list
  uint64_t S, n;          // slots, vertices (bounds checks of the debug build)
  uint32_t exp;           // libbf_prof.so only: timing experiments (env BF_EXPERIMENT; results are wrong when set):
                          // 1 = skip endpoint REDs, 2 = skip centre REDs
  uint32_t win;           // dense window keys in use (<= compile-time size)
  uint32_t dwin;          // dense variant (WIN == 0): window keys (>= every heavy start's key range)
  uint32_t* kbuf;         // slot-mode key buffer [W] (vertex mode, mostly-short-segment graphs) or null
  uint32_t short_segs;    // the graph's segments are short on average: slot mode keeps SB slots in flight
  uint32_t cap;           // heavy chunk capacity in wedges (<= HV_CAP)
  int rank, world;
};

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

// Phase timing of the wedge kernels (libbf_prof.so, -DBF_PROFILE): thread 0
// of every CTA accumulates clock64() deltas per phase into g_prof, which
// graph_count prints to stderr.  Compiles to nothing otherwise.
#ifdef BF_PROFILE
__device__ unsigned long long g_prof[3][8];
__device__ unsigned long long g_prof_red[4];  // endpoint REDs: all, key < 256, < 1024, < 4096 (side-relative)
struct Prof {
  long long t;
  unsigned long long acc[8];
  __device__ __forceinline__ void start() {
    t = clock64();
    for (int i = 0; i < 8; i++) acc[i] = 0;
  }
  __device__ __forceinline__ void mark(int i) {
    const long long n = clock64();
    acc[i] += (unsigned long long)(n - t);
    t = n;
  }
  __device__ __forceinline__ void flush(int tier) {
    if (threadIdx.x == 0)
      for (int i = 0; i < 8; i++) atomicAdd(&g_prof[tier][i], acc[i]);
  }
};
#else
struct Prof {
  __device__ __forceinline__ void start() {}
  __device__ __forceinline__ void mark(int) {}
  __device__ __forceinline__ void flush(int) {}
};
#endif

// Endpoint contributions C(d,2) land on the aggregated keys, which in the
// HIGH orientation are the few highest-ranked vertices of each side: one
// address per hub hammered by every CTA.  Keys among the first HUB_KEYS rids
// of their side therefore go to one of HUB_STRIPES striped copies (chosen by
// CTA), summed into bv by k_hub_reduce after the wedge kernels.
constexpr uint32_t HUB_KEYS = 4096;
constexpr uint32_t HUB_STRIPES = 16;
__device__ __forceinline__ uint64_t* endpoint_slot(const CountArgs& a, uint32_t key) {
  const uint32_t side = key >= a.n_u, kk = key - (side ? a.n_u : 0u);
  if (kk < HUB_KEYS)
    return a.hub + ((size_t)(blockIdx.x & (HUB_STRIPES - 1)) * 2 + side) * HUB_KEYS + kk;
  return a.bv + key;
}

// ------------------------------------------------ small counter store
// u8 dense window over key offsets [0, wl) + open-addressed hash (u32 keys,
// u8 counts) for the rest.  In the small tiers d(s,x) <= #slots of s <= 128
// (each centre y in N(s) contributes at most one wedge per key), so u8 never
// wraps.
__device__ __forceinline__ uint32_t hslot(uint32_t key, uint32_t shift) { return (key * 0x9E3779B1u) >> shift; }

// SCAN (BF_SMALL_SCAN bit 0: warp tier, bit 1: medium tier): increments are
// fire-and-forget (red.shared), nothing records owners; finalize scans the
// window's first nk counters and, when a key of the start was hashed, the hash
// slots' counts.  (Measured on c2 for both tiers: wedge kernels 5.71 -> 6.67 ms
// -- a warp-tier start has ~190 wedges against a 1024-counter window.)
#ifndef BF_SMALL_SCAN
#define BF_SMALL_SCAN 0
#endif
__device__ __forceinline__ void red_shared_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
// endpoint pairs of four packed u8 counters (byte b of word wd is key offset
// idx0 + b, or the key of hash slot idx0 + b): C(d,2) to the total and both endpoints
template <int MODE>
__device__ __forceinline__ void bytes_finalize(const CountArgs& a, uint32_t wd, uint32_t kbase, uint32_t idx0,
                                               const uint32_t* hkeys, uint64_t& lsum, uint32_t& np);

template <bool SCAN, bool OWN2 = false>
struct SmallStoreT {
  static constexpr bool kScan = SCAN;
  // OWN2: the owner of a key is the wedge that takes its count from 1 to 2, so
  // the list holds only the keys that contribute (d >= 2); a key seen once is
  // reset in pass 2 by its only wedge (vertex / edge modes only)
  static constexpr bool kOwn2 = OWN2;
  uint32_t nk;    // SCAN: window counters the current start can touch (min(wl, its key range))
  uint32_t* win;  // u8 counters, four per word: bytes [0, WIN) the dense window (key kk: byte kk),
                  // bytes [WIN, WIN + HS) the hash slots' counts (slot h: byte WIN + h)
  uint32_t* hk;
  uint32_t* hv;   // = the hash counts (bytes WIN..), as words
  uint32_t wl, hmask, shift, winb;

  // returns true if this increment took the key's count from 0 to 1
  __device__ __forceinline__ bool add(uint32_t key, uint32_t kk, bool& hashed) const {
    uint32_t ci;
    return add_ci(key, kk, hashed, ci);
  }
  // the same, and the counter's byte index ci (window: kk; hash slot h: WIN + h)
  __device__ __forceinline__ bool add_ci(uint32_t key, uint32_t kk, bool& hashed, uint32_t& ci) const {
    if (__builtin_expect(kk < wl, 1)) {
      ci = kk;
    } else {
      hashed = true;
      uint32_t h = hslot(key, shift);
      for (uint32_t probes = 0;; probes++) {
        if (probes > hmask) __trap();  // more distinct keys than slots: impossible by the tier bound
        const uint32_t cur = atomicCAS(hk + h, EMPTY, key);
        if (cur == EMPTY || cur == key) break;
        h = (h + 1) & hmask;
      }
      ci = winb + h;
    }
    BF_CHECK(__isShared(win + (ci >> 2)));
    const uint32_t sh = (ci & 3u) << 3;
    if constexpr (SCAN) {
      red_shared_u32(win + (ci >> 2), 1u << sh);
      return false;
    } else {
      const uint32_t old = atomicAdd(win + (ci >> 2), 1u << sh);
      return ((old >> sh) & 0xffu) == (OWN2 ? 1u : 0u);
    }
  }
  __device__ __forceinline__ uint32_t at(uint32_t ci) const { return ((const uint8_t*)win)[ci]; }
  __device__ __forceinline__ void zero_at(uint32_t ci) const {
    ((uint8_t*)win)[ci] = 0;
    if (ci >= winb) hk[ci - winb] = EMPTY;
  }
  __device__ __forceinline__ uint32_t get(uint32_t key, uint32_t kk) const {
    if (__builtin_expect(kk < wl, 1)) return ((const uint8_t*)win)[kk];
    uint32_t h = hslot(key, shift);
    for (uint32_t probes = 0; hk[h] != key; probes++) {
      if (probes > hmask) __trap();  // the key was inserted in pass 1
      h = (h + 1) & hmask;
    }
    return ((const uint8_t*)win)[winb + h];
  }
  // reset one key (every key of the start is reset, so deleting hash entries
  // never strands a lookup: get() probes past EMPTY slots)
  __device__ __forceinline__ void zero(uint32_t key, uint32_t kk) const {
    if (kk < wl) {
      ((uint8_t*)win)[kk] = 0;
      return;
    }
    uint32_t h = hslot(key, shift);
    while (hk[h] != key) h = (h + 1) & hmask;
    hk[h] = EMPTY;
    ((uint8_t*)win)[winb + h] = 0;
  }
  // SCAN finalize: window bytes [0, nk), then (hany: some key of the start was
  // hashed) the hash slots' counts
  template <int MODE, int NT>
  __device__ __forceinline__ void scan_finalize(const CountArgs& a, uint32_t kbase, bool hany, uint64_t& lsum,
                                                uint64_t& pairs) const {
    uint32_t np = 0;
    const uint4* w4 = reinterpret_cast<const uint4*>(win);
    const uint32_t nq = (nk + 15u) >> 4;
    for (uint32_t q = threadIdx.x; q < nq; q += NT) {
      const uint4 v = w4[q];
      if ((v.x | v.y | v.z | v.w) == 0u) continue;
      bytes_finalize<MODE>(a, v.x, kbase, 16u * q, nullptr, lsum, np);
      bytes_finalize<MODE>(a, v.y, kbase, 16u * q + 4u, nullptr, lsum, np);
      bytes_finalize<MODE>(a, v.z, kbase, 16u * q + 8u, nullptr, lsum, np);
      bytes_finalize<MODE>(a, v.w, kbase, 16u * q + 12u, nullptr, lsum, np);
    }
    if (hany) {
      const uint32_t hq = (hmask + 1u) >> 4;
      for (uint32_t q = threadIdx.x; q < hq; q += NT) {
        const uint4 v = w4[(winb >> 4) + q];
        if ((v.x | v.y | v.z | v.w) == 0u) continue;
        bytes_finalize<MODE>(a, v.x, 0u, 16u * q, hk, lsum, np);
        bytes_finalize<MODE>(a, v.y, 0u, 16u * q + 4u, hk, lsum, np);
        bytes_finalize<MODE>(a, v.z, 0u, 16u * q + 8u, hk, lsum, np);
        bytes_finalize<MODE>(a, v.w, 0u, 16u * q + 12u, hk, lsum, np);
      }
    }
    pairs += np;
  }
  template <int NT>
  __device__ __forceinline__ void scan_reset(bool hany) const {
    uint4* w4 = reinterpret_cast<uint4*>(win);
    const uint32_t nq = (nk + 15u) >> 4;
    for (uint32_t q = threadIdx.x; q < nq; q += NT) w4[q] = make_uint4(0u, 0u, 0u, 0u);
    if (hany) {
      const uint32_t hs = hmask + 1u;
      for (uint32_t q = threadIdx.x; q < (hs >> 4); q += NT) w4[(winb >> 4) + q] = make_uint4(0u, 0u, 0u, 0u);
      uint4* k4 = reinterpret_cast<uint4*>(hk);
      for (uint32_t q = threadIdx.x; q < (hs >> 2); q += NT) k4[q] = make_uint4(EMPTY, EMPTY, EMPTY, EMPTY);
    }
  }
};

template <int MODE>
__device__ __forceinline__ void bytes_finalize(const CountArgs& a, uint32_t wd, uint32_t kbase, uint32_t idx0,
                                               const uint32_t* hkeys, uint64_t& lsum, uint32_t& np) {
  while (wd) {
    const uint32_t sh = (uint32_t)(__ffs(wd) - 1) & ~7u;
    const uint32_t d = (wd >> sh) & 0xffu;
    wd &= ~(0xffu << sh);
    np++;
    if (d > 1u) {
      const uint32_t c2 = (d * (d - 1u)) >> 1;  // d <= 128
      lsum += c2;
      const uint32_t i = idx0 + (sh >> 3);
      const uint32_t key = hkeys ? hkeys[i] : kbase + i;
      if (MODE == MODE_VERTEX && !(a.exp & 1)) red_add_u64(endpoint_slot(a, key), c2);
    }
  }
}
#ifndef BF_SMALL_OWN2
#define BF_SMALL_OWN2 1
#endif
template <int NT, int MODE>
using SmallStore = SmallStoreT<((NT == 32 ? 1 : 2) & BF_SMALL_SCAN) != 0,
                               BF_SMALL_OWN2 != 0 && BF_SMALL_SCAN == 0 && MODE != MODE_TOTAL>;

// ------------------------------------------------ heavy counter store
// u32 dense shared window over [0, wl) + the CTA's global row for the rest
// (L2 atomics; plain reads bypass L1 so they see the atomics' results).
// SCAN: window increments are fire-and-forget (red.shared: no owner test, no
// list push, nothing waits on the atomic's return); finalize and the reset
// scan the window's first nk counters (the start's key range) instead of an
// owner list -- only overflow-row keys keep owners.
#ifndef BF_BIG_SCAN
#define BF_BIG_SCAN 1
#endif
template <bool SCAN>
struct HeavyStoreT {
  static constexpr bool kScan = SCAN;
  // kFast: the unit walks test the window bound on the key offset alone (an
  // empty lane's key EMPTY lands far past every key range) and touch the
  // window through predicated shared red / loads at ws + 4 kk, so the common
  // path has no branch; only overflow-row keys take one
  static constexpr bool kFast = SCAN;
  uint32_t ws;    // shared-space address of win
  uint32_t sink;  // first of 32 per-lane sink counters after the window (never read)
  uint32_t* win;
  uint32_t* orow;
  uint32_t wl;
  uint32_t nk;  // SCAN: window counters the current start can touch (min(wl, its key range))
  uint64_t lenchk;
  // the window path is the common one (99.5% of heavy-tier keys on c2): a
  // real branch keeps the global row's address arithmetic off it
  __device__ __forceinline__ bool add(uint32_t, uint32_t kk, bool&) const {
    BF_CHECK(kk < wl || kk - wl < lenchk);
    BF_CHECK(!SCAN || kk >= wl || kk < nk);
    if (__builtin_expect(kk < wl, 1)) {
      if constexpr (SCAN) {
        red_shared_u32(win + kk, 1u);
        return false;
      } else {
        return atomicAdd(win + kk, 1u) == 0u;
      }
    }
    return atomicAdd(orow + (kk - wl), 1u) == 0u;
  }
  // overflow-row increment (kk >= wl); true if it took the count 0 -> 1
  __device__ __forceinline__ bool add_row(uint32_t kk) const { return atomicAdd(orow + (kk - wl), 1u) == 0u; }
  __device__ __forceinline__ uint32_t get(uint32_t, uint32_t kk) const {
    if (__builtin_expect(kk < wl, 1)) return win[kk];
    return __ldcg(orow + (kk - wl));
  }
  __device__ __forceinline__ void zero(uint32_t, uint32_t kk) const {
    if (__builtin_expect(kk < wl, 1)) win[kk] = 0;
    else __stcg(orow + (kk - wl), 0u);
  }
  // SCAN finalize: every non-zero counter of the window's first nk keys is one
  // endpoint pair (the window part of the owner list): C(d,2) to the total and
  // both endpoints, read four counters at a time
  template <int MODE, int NT>
  __device__ __forceinline__ void scan_finalize(const CountArgs& a, uint32_t kbase, bool, uint64_t& lsum,
                                                uint64_t& pairs) const {
    const uint32_t nq = (nk + 3u) >> 2;
    const uint4* w4 = reinterpret_cast<const uint4*>(win);
    uint32_t np = 0;
    for (uint32_t q = threadIdx.x; q < nq; q += NT) {
      const uint4 v = w4[q];
      if ((v.x | v.y | v.z | v.w) == 0u) continue;
      const uint32_t d[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int c = 0; c < 4; c++) {
        np += d[c] != 0u;
        if (d[c] > 1u) {
          const uint64_t c2 = choose2(d[c]);
          lsum += c2;
          if (MODE == MODE_VERTEX && !(a.exp & 1)) red_add_u64(endpoint_slot(a, kbase + 4u * q + c), c2);
        }
      }
    }
    pairs += np;
  }
  template <int NT>
  __device__ __forceinline__ void scan_reset(bool) const {
    const uint32_t nq = (nk + 3u) >> 2;
    uint4* w4 = reinterpret_cast<uint4*>(win);
    for (uint32_t q = threadIdx.x; q < nq; q += NT) w4[q] = make_uint4(0u, 0u, 0u, 0u);
  }
};
using HeavyStore = HeavyStoreT<BF_BIG_SCAN != 0>;

template <class S, class = void>
struct FastOf {
  static constexpr bool v = false;
};
template <class S>
struct FastOf<S, std::void_t<decltype(S::kFast)>> {
  static constexpr bool v = S::kFast;
};
__device__ __forceinline__ void red_shared_u32_at(uint32_t addr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}
// predicated shared-window load at a shared-space address (no branch; the
// address is never dereferenced when the predicate is off)
__device__ __forceinline__ uint32_t ld_shared_if(uint32_t addr, uint32_t kk, uint32_t wl) {
  uint32_t v;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %1, %2;\n\tmov.u32 %0, 0;\n\t@p ld.shared.u32 %0, [%3];\n\t}"
               : "=r"(v)
               : "r"(kk), "r"(wl), "r"(addr)
               : "memory");
  return v;
}

// the key range of start s (same-side rids ranked above s (HIGH) or below it
// (LOW)): every key offset kk of its wedges is below it
template <int ORIENT>
__device__ __forceinline__ uint32_t key_range(uint32_t s, uint32_t n_u, uint64_t n) {
  if (ORIENT == BF_ORIENT_HIGH) return s < n_u ? s : s - n_u;
  return s < n_u ? n_u - s - 1u : (uint32_t)(n - s - 1u);
}

// ================================================================ unit walk
// A chunk of a start's wedge sequence is cut into "units": pieces of at most P
// consecutive wedges of one segment, numbered in slot order by a scan of the
// per-slot unit counts.  A G-lane group walks one unit per round, each lane
// reading every G-th key (P/G predicated loads in flight per lane, UR units per
// group unrolled), so no lane ever searches for its segment.  Pass-2 sums of
// d-1 stay in registers until one shared atomic per unit.
// unit meta: chunk position of the first wedge (bits 0-15) | length | slot;
// NT <= 256: length 1..P in bits 16-23, slot in 24-31 (one mask per decode);
// wider CTAs: length - 1 in bits 16-20, slot in 21-31
template <int NT>
struct UnitMeta {
  static constexpr bool WIDE = NT > 256;
  static constexpr uint32_t SLOT_SHIFT = WIDE ? 21 : 24;
  __device__ __forceinline__ static uint32_t pack(uint32_t pos, uint32_t len, uint32_t slot) {
    return (pos & 0xffffu) | ((WIDE ? len - 1 : len) << 16) | (slot << SLOT_SHIFT);
  }
  // length of an active unit's meta word; inactive units (me = 0) give 0 when narrow
  __device__ __forceinline__ static uint32_t len(uint32_t me, bool active) {
    if (WIDE) return active ? ((me >> 16) & 31u) + 1 : 0u;
    return (me >> 16) & 0xffu;
  }
  __device__ __forceinline__ static uint32_t slot(uint32_t me) { return me >> SLOT_SHIFT; }
};

template <int NT, uint32_t UCAP>
struct Units {
  static_assert(NT <= 2048, "unit meta packs the slot in 11 bits");
  using SlotT = typename std::conditional<(NT <= 256), uint8_t, uint16_t>::type;
  uint32_t lo[UCAP];           // first nbr index of the unit
  uint32_t meta[UCAP];         // UnitMeta<NT>: chunk position of the first wedge | length | chunk-local slot
  uint32_t slo[NT], shi[NT];   // pass-2 per-slot sums (u64 as two u32)
  uint32_t wt[32];             // scan scratch
  uint32_t jn[2];              // continuation slot of chunk i in jn[i & 1] (FULL = none)
  uint32_t nunits, item, lcnt;
};

// exclusive scan of v over the CTA (NT == 32: one warp, no CTA barrier)
template <int NT>
__device__ __forceinline__ uint32_t cta_scan(uint32_t v, uint32_t* wt, uint32_t& total) {
  if (NT == 32) {
    const uint32_t inc = warp_inclusive_scan(v);
    total = __shfl_sync(FULL, inc, 31);
    return inc - v;
  }
  uint32_t t;
  const uint32_t ex = block_exclusive_scan<uint32_t>(v, wt, &t);
  total = t;
  return ex;
}

template <int NT>
__device__ __forceinline__ void cta_sync() {
  if (NT == 32) __syncwarp();
  else __syncthreads();
}

// write the units of one slot segment [lo, lo+L) (thread t), then barrier
template <int NT, int P, uint32_t UCAP>
__device__ __forceinline__ void units_write(Units<NT, UCAP>& u, uint32_t lo, uint32_t L) {
  static_assert((P <= 32 || (!UnitMeta<NT>::WIDE && P <= 128)) && (P & (P - 1)) == 0,
                "unit length is packed in 5 bits (wide CTAs) or 8 bits");
  constexpr uint32_t LP = 31 - __builtin_clz(P);
  const uint32_t nu = (L + P - 1) >> LP;
  uint32_t total;
  // one scan of (wedges << 16 | units): chunk wedges <= 65535, units <= 65535
  const uint32_t pk = cta_scan<NT>((L << 16) | nu, u.wt, total);
  const uint32_t ex = pk & 0xffffu, wp = pk >> 16;
  BF_CHECK(ex + nu <= UCAP && L < 65536);
  for (uint32_t f = 0, o = 0; f < nu; f++, o += P) {
    u.lo[ex + f] = lo + o;
    u.meta[ex + f] = UnitMeta<NT>::pack(wp + o, f + 1 < nu ? (uint32_t)P : L - o, threadIdx.x);
  }
  if (threadIdx.x == 0) u.nunits = total & 0xffffu;
  u.slo[threadIdx.x] = 0;
  u.shi[threadIdx.x] = 0;
  cta_sync<NT>();
}

// Build the units of chunk [K0, K1) of the start's wedges from slots
// [jc, min(jc+NT, j1)) (heavy tier).  Thread t handles slot jc + t; `mine` =
// it has a segment in the chunk.  Returns K1; u.jn[par] receives the slot that
// continues past K1 (if any; the caller resets it after reading, and chunks
// alternate par so the reset never races the next chunk's write).
template <int MODE, int NT, int P, uint32_t UCAP>
__device__ __forceinline__ uint64_t units_build(const CountArgs& a, Units<NT, UCAP>& u, uint32_t jc, uint32_t j1,
                                                uint64_t base, uint64_t K0, uint32_t cap, uint32_t par, bool& mine,
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
  uint32_t lo = 0, L = 0;
  if (j < jlim) {
    const uint64_t A = __ldg(a.wpre + j) - base, B = __ldg(a.wpre + j + 1) - base;
    if (A <= K1 && K1 < B) u.jn[par] = j;
    if (A < B && A < K1 && B > K0) {  // non-empty segment overlapping [K0, K1)
      const uint64_t a0 = max(A, K0), b0 = min(B, K1);
      L = (uint32_t)(b0 - a0);
      lo = __ldg(a.seglo + j) + (uint32_t)(a0 - A);
      mine = true;
      if (MODE == MODE_VERTEX) myy = __ldg(a.nbr + j);
    }
  }
  units_write<NT, P, UCAP>(u, lo, L);
  return K1;
}

// owner of a key (its count went 0 -> 1): append it to the start's list
// (shared memory up to lcap entries, then the CTA's global list)
// SPILL: the list can outgrow shared memory (heavy tier); otherwise lcap is
// an exact bound (small tiers: distinct keys <= w <= lcap)
// (A warp-aggregated push -- one atomicAdd per warp on the list counter --
// measured slower on c2: 6.82 -> 7.40 ms.)
template <bool SPILL>
__device__ __forceinline__ void list_push(uint32_t* lcnt, uint32_t* list, uint32_t lcap, uint32_t* olist,
                                          uint64_t ocap, uint32_t key, uint16_t* listi = nullptr, uint32_t ci = 0) {
  const uint32_t i = atomicAdd(lcnt, 1u);
  if (listi) {  // small tiers: only the owner's counter index (the key is recoverable from it)
    listi[i] = (uint16_t)ci;
    return;
  }
  if (!SPILL || i < lcap) list[i] = key;
  else {
    BF_CHECK(olist != nullptr && i - lcap < ocap);
    olist[i - lcap] = key;
  }
}
template <bool SPILL>
__device__ __forceinline__ uint32_t list_get(const uint32_t* list, uint32_t lcap, const uint32_t* olist, uint32_t i) {
  return (!SPILL || i < lcap) ? list[i] : __ldcg(olist + (i - lcap));
}

// pass 1 over the chunk's units: d(key) += 1 per wedge
// CACHE (small tiers): each wedge's counter index goes to cache[chunk position]
// and each owner's to listi, so pass 2, finalize and the reset read counters
// directly -- no key reload, window test or hash probe after pass 1
template <bool SPILL, bool CACHE, int NT, int P, int G, int UR, uint32_t UCAP, class Store>
__device__ __forceinline__ void units_pass1(const CountArgs& a, Units<NT, UCAP>& u, const Store& cs,
                                            uint32_t kbase, uint32_t* list, uint32_t lcap, uint32_t* olist,
                                            bool& hashed, uint16_t* cache, uint16_t* listi) {
  constexpr int IT = P / G;
  constexpr uint32_t NG = NT / G;
  const uint32_t tid = threadIdx.x, gl = tid & (G - 1);
  const uint32_t nunits = u.nunits;
  for (uint32_t x0 = tid / G; x0 < nunits; x0 += NG * UR) {
    uint32_t key[UR][IT], ps[UR];
#pragma unroll
    for (int r = 0; r < UR; r++) {
      const uint32_t x = x0 + r * NG;
      const uint32_t lo = x < nunits ? u.lo[x] : 0u, me = x < nunits ? u.meta[x] : 0u;
      const uint32_t len = UnitMeta<NT>::len(me, x < nunits);
      ps[r] = me & 0xffffu;
      const uint32_t* pn = a.nbr + lo + gl;  // one address per unit, immediate offsets per key
#pragma unroll
      for (int it = 0; it < IT; it++) {
        const uint32_t i = gl + it * G;
        BF_CHECK(i >= len || lo + i < a.S);
        key[r][it] = i < len ? __ldg(pn + it * G) : EMPTY;
      }
    }
#pragma unroll
    for (int r = 0; r < UR; r++)
#pragma unroll
      for (int it = 0; it < IT; it++) {
        uint32_t k = key[r][it];
        if constexpr (FastOf<Store>::v && !CACHE) {
          // window keys: one unconditional shared red (lanes without a window
          // key hit their own sink counter past the window); overflow-row keys
          // are flagged and handled after the unit's keys (a real branch)
          const uint32_t kk = k - kbase;  // EMPTY: far past the key range
          BF_CHECK(k == EMPTY || kk < cs.wl || kk - cs.wl < cs.lenchk);
          red_shared_u32_at(cs.ws + 4u * (kk < cs.wl ? kk : cs.sink + (tid & 31u)));
          if (it == IT - 1) {
            bool ovf = false;
#pragma unroll
            for (int t = 0; t < IT; t++) ovf |= key[r][t] - kbase >= cs.wl && key[r][t] != EMPTY;
            if (ovf)
#pragma unroll
              for (int t = 0; t < IT; t++) {
                const uint32_t kt = key[r][t], kkt = kt - kbase;
                if (kkt >= cs.wl && kt != EMPTY && cs.add_row(kkt))
                  list_push<SPILL>(&u.lcnt, list, lcap, olist, a.olist_len, kt);
              }
          }
        } else if (k != EMPTY) {
          BF_CHECK(k < a.n);
          if constexpr (CACHE) {
            uint32_t ci;
            const bool first = cs.add_ci(k, k - kbase, hashed, ci);
            cache[ps[r] + gl + it * G] = (uint16_t)ci;
            if (first) list_push<SPILL>(&u.lcnt, list, lcap, olist, a.olist_len, k, listi, ci);
          } else {
            if (cs.add(k, k - kbase, hashed)) list_push<SPILL>(&u.lcnt, list, lcap, olist, a.olist_len, k);
          }
        }
      }
  }
}

// pass 2 over the chunk's units: c = d(key) - 1 per wedge, summed per slot
// (centre y in vertex mode, edge (s, y) in edge mode); edge mode also adds c
// to the wedge's (y, key) edge
// NARROW: the start's d < 2^32 / P (d <= #slots), so a lane group's sum of
// d-1 fits u32 and the group reduction shuffles 32-bit words
template <int MODE, bool CACHE, int NT, int P, int G, int UR, uint32_t UCAP, class Store, bool NARROW = true>
__device__ __forceinline__ void units_pass2(const CountArgs& a, Units<NT, UCAP>& u, const Store& cs,
                                            uint32_t kbase, const uint16_t* cache, uint64_t* np1 = nullptr) {
  uint32_t ones = 0;  // OWN2: keys seen once (reset here by their only wedge)
  constexpr int IT = P / G;
  constexpr uint32_t NG = NT / G;
  const uint32_t tid = threadIdx.x, gl = tid & (G - 1);
  const uint32_t nunits = u.nunits;
  // warp-uniform trip count: the group reduction below is a full-warp shuffle
  for (uint32_t xb = (tid & ~31u) / G; xb < nunits; xb += NG * UR) {
    uint32_t key[UR][IT], lo[UR], ps[UR], sl[UR], ln[UR];
#pragma unroll
    for (int r = 0; r < UR; r++) {
      const uint32_t x = xb + r * NG + (tid & 31) / G;
      const bool act = x < nunits;
      lo[r] = act ? u.lo[x] : 0u;
      const uint32_t me = act ? u.meta[x] : 0u, len = UnitMeta<NT>::len(me, act);
      ln[r] = len;
      ps[r] = me & 0xffffu;
      sl[r] = UnitMeta<NT>::slot(me);
      const uint32_t* pn = a.nbr + lo[r] + gl;
#pragma unroll
      for (int it = 0; it < IT; it++) {
        const uint32_t i = gl + it * G;
        if constexpr (CACHE) key[r][it] = i < len ? (uint32_t)cache[ps[r] + i] : EMPTY;  // counter index
        else key[r][it] = i < len ? __ldg(pn + it * G) : EMPTY;
      }
    }
#pragma unroll
    for (int r = 0; r < UR; r++) {
      const uint32_t x = xb + r * NG + (tid & 31) / G;
      typename std::conditional<NARROW, uint32_t, uint64_t>::type s = 0;
      if constexpr (FastOf<Store>::v && !CACHE && MODE == MODE_VERTEX) {
        // sum d over the lane's keys (predicated window loads; empty lanes
        // read nothing), then subtract one per key: sum of (d - 1)
        bool ovf = false;
#pragma unroll
        for (int it = 0; it < IT; it++) {
          const uint32_t k = key[r][it], kk = k - kbase;
          s += ld_shared_if(cs.ws + 4u * kk, kk, cs.wl);
          ovf |= kk >= cs.wl && k != EMPTY;
        }
        if (ovf)  // overflow-row keys (rare): a real branch, not if-converted per key
#pragma unroll
          for (int it = 0; it < IT; it++) {
            const uint32_t k = key[r][it], kk = k - kbase;
            if (kk >= cs.wl && k != EMPTY) s += cs.get(k, kk);
          }
        s -= ln[r] > gl ? (ln[r] - gl + (uint32_t)G - 1u) / (uint32_t)G : 0u;
      } else if constexpr (FastOf<Store>::v && !CACHE && MODE == MODE_EDGE) {
        uint32_t d[IT];
        bool ovf = false;
#pragma unroll
        for (int it = 0; it < IT; it++) {
          const uint32_t k = key[r][it], kk = k - kbase;
          d[it] = ld_shared_if(cs.ws + 4u * kk, kk, cs.wl);
          ovf |= kk >= cs.wl && k != EMPTY;
        }
        if (ovf)
#pragma unroll
          for (int it = 0; it < IT; it++) {
            const uint32_t k = key[r][it], kk = k - kbase;
            if (kk >= cs.wl && k != EMPTY) d[it] = cs.get(k, kk);
          }
#pragma unroll
        for (int it = 0; it < IT; it++) {
          const uint32_t c = d[it] ? d[it] - 1u : 0u;  // empty lanes read d = 0
          s += c;
          if (c) red_add_u64(a.acc + (lo[r] + gl + it * G), c);  // edge (y, key)
        }
      } else {
#pragma unroll
      for (int it = 0; it < IT; it++) {
        if (key[r][it] != EMPTY) {
          uint32_t c;
          if constexpr (CACHE) {
            c = cs.at(key[r][it]) - 1u;
            if constexpr (Store::kOwn2) {
              if (c == 0u) {
                cs.zero_at(key[r][it]);
                ones++;
              }
            }
          } else {
            c = cs.get(key[r][it], key[r][it] - kbase) - 1u;
          }
          s += c;
          if (MODE == MODE_EDGE && c) red_add_u64(a.acc + (lo[r] + gl + it * G), c);  // edge (y, key)
        }
      }
      }
#pragma unroll
      for (int o = 1; o < G; o <<= 1) s += __shfl_xor_sync(FULL, s, o);
      if (x < nunits && gl == 0 && s) seg_add(u.slo, u.shi, sl[r], (uint64_t)s);
    }
  }
  if (np1) *np1 += ones;
}

template <int MODE>
__device__ __forceinline__ void slot_flush(const CountArgs& a, const uint32_t* slo, const uint32_t* shi, bool mine,
                                           uint32_t myj, uint32_t myy) {
  if (!mine) return;
  const uint32_t t = threadIdx.x;
  const uint64_t v = ((uint64_t)shi[t] << 32) | slo[t];
  if (!v) return;
  BF_CHECK(myy < a.n && myj < a.S);
  if (MODE == MODE_VERTEX) { if (!(a.exp & 2)) red_add_u64(a.bv + myy, v); }  // centre y
  else red_add_u64(a.acc + myj, v);                                           // edge (s, y)
}

// finalize over the owner list: C(d,2) to the total and both endpoints (total
// mode also resets the counters here)
template <int MODE, bool SPILL, int NT, class Store>
__device__ __forceinline__ void list_finalize(const CountArgs& a, const Store& cs, uint32_t kbase, uint32_t cnt,
                                              const uint32_t* list, uint32_t lcap, const uint32_t* olist,
                                              uint64_t& lsum, const uint16_t* listi = nullptr) {
  for (uint32_t i = threadIdx.x; i < cnt; i += NT) {
    uint32_t key, kk, d;
    if constexpr (SPILL) {
      key = list_get<SPILL>(list, lcap, olist, i);
      kk = key - kbase;
      d = cs.get(key, kk);
    } else if (listi) {  // counter index -> key: window byte kk = key - kbase, or the hash slot's key
      const uint32_t ci = listi[i];
      key = ci < cs.winb ? kbase + ci : cs.hk[ci - cs.winb];
      kk = key - kbase;
      d = cs.at(ci);
    } else {
      key = list_get<SPILL>(list, lcap, olist, i);
      kk = key - kbase;
      d = cs.get(key, kk);
    }
    BF_CHECK(key < a.n);
    // small tiers reset here in total mode; the heavy tier resets after a barrier
    // (resetting inside this loop, next to other threads' reads of the global
    // overflow row, measured 4x slower on c3)
    if constexpr (MODE == MODE_TOTAL && !SPILL) {
      if (listi) cs.zero_at(listi[i]);
      else cs.zero(key, kk);
    }
    // small tiers: d <= 128, so C(d,2) in 32 bits
    const uint64_t c2 = SPILL ? choose2(d) : (uint64_t)((d * (d - (d > 0))) >> 1);
    lsum += c2;
    if (MODE == MODE_VERTEX && c2 && !(a.exp & 1)) red_add_u64(endpoint_slot(a, key), c2);
#ifdef BF_PROFILE
    if (c2 && (a.exp & 64)) {
      const uint32_t kk2 = key - (key >= a.n_u ? a.n_u : 0u);
      atomicAdd(&g_prof_red[0], 1ull);
      if (kk2 < 256) atomicAdd(&g_prof_red[1], 1ull);
      if (kk2 < 1024) atomicAdd(&g_prof_red[2], 1ull);
      if (kk2 < 4096) atomicAdd(&g_prof_red[3], 1ull);
    }
#endif
  }
}

// The rest of a start once its (first) chunk's units are built: pass 1,
// finalize, pass 2, reset.  `single`: the whole start is that one chunk
// (units reused by pass 2); otherwise chunks are rebuilt by units_build.
template <int ORIENT, int MODE, bool SPILL, bool CACHE, int NT, int P, int G, int UR, uint32_t UCAP, class Store>
__device__ __forceinline__ void start_passes(const CountArgs& a, Units<NT, UCAP>& u, const Store& cs,
                                             const Start& st, bool single, uint64_t base, uint64_t w, uint64_t K1,
                                             uint32_t cap, uint32_t jn0, bool mine, uint32_t myj, uint32_t myy,
                                             uint32_t* list, uint32_t lcap, uint32_t* olist, uint64_t& lsum,
                                             uint64_t& pairs, bool& hashed, Prof& pf, uint16_t* cache,
                                             uint16_t* listi) {
  const uint32_t tid = threadIdx.x;
  // ---- pass 1 (first chunk already built)
  if (single) units_pass1<SPILL, CACHE, NT, P, G, UR, UCAP>(a, u, cs, st.kbase, list, lcap, olist, hashed, cache, listi);
  else units_pass1<SPILL, false, NT, P, G, UR, UCAP>(a, u, cs, st.kbase, list, lcap, olist, hashed, nullptr, nullptr);
  pf.mark(2);
  bool hany = false;  // SCAN: some key of the start went to the hash
  if constexpr (Store::kScan) {
    if (NT == 32) {
      __syncwarp();
      hany = __any_sync(FULL, hashed);
    } else {
      hany = __syncthreads_or(hashed) != 0;
    }
  } else {
    cta_sync<NT>();
  }
  pf.mark(3);
  if (!single) {
    if (tid == 0) u.jn[0] = FULL;
    uint32_t jc = jn0 != FULL ? jn0 : ((st.j1 - st.j0 > (uint32_t)NT) ? st.j0 + NT : st.j1), par = 1;
    uint64_t K0 = K1;
    while (K0 < w) {
      const uint64_t Kn = units_build<MODE, NT, P, UCAP>(a, u, jc, st.j1, base, K0, cap, par, mine, myj, myy);
      const uint32_t jn = u.jn[par];
      units_pass1<SPILL, false, NT, P, G, UR, UCAP>(a, u, cs, st.kbase, list, lcap, olist, hashed, nullptr, nullptr);
      cta_sync<NT>();
      if (tid == 0) u.jn[par] = FULL;
      jc = jn != FULL ? jn : ((st.j1 - jc > (uint32_t)NT) ? jc + NT : st.j1);
      K0 = Kn;
      par ^= 1u;
    }
  }
  pf.mark(1);
  const uint32_t cnt = u.lcnt;
  list_finalize<MODE, SPILL, NT>(a, cs, st.kbase, cnt, list, lcap, olist, lsum, CACHE ? listi : nullptr);
  if constexpr (Store::kScan) cs.template scan_finalize<MODE, NT>(a, st.kbase, hany, lsum, pairs);
  if (tid == 0) pairs += cnt;
  pf.mark(4);
  if (MODE == MODE_TOTAL && (SPILL || Store::kScan)) {
    cta_sync<NT>();
    if (SPILL)
      for (uint32_t i = tid; i < cnt; i += NT) {
        const uint32_t key = list_get<SPILL>(list, lcap, olist, i);
        cs.zero(key, key - st.kbase);
      }
    if constexpr (Store::kScan) cs.template scan_reset<NT>(hany);
  }
  if (MODE != MODE_TOTAL) {
    cta_sync<NT>();  // d is final
    pf.mark(3);
    if (single) {
      if (st.j1 - st.j0 < (1u << 26))
        units_pass2<MODE, CACHE, NT, P, G, UR, UCAP>(a, u, cs, st.kbase, cache, &pairs);
      else
        units_pass2<MODE, CACHE, NT, P, G, UR, UCAP, Store, false>(a, u, cs, st.kbase, cache, &pairs);
      pf.mark(5);
      cta_sync<NT>();
      pf.mark(3);
      slot_flush<MODE>(a, u.slo, u.shi, mine, myj, myy);
    } else {
      uint32_t jc = st.j0, par = 0;
      uint64_t K0 = 0;
      while (K0 < w) {
        const uint64_t Kn = units_build<MODE, NT, P, UCAP>(a, u, jc, st.j1, base, K0, cap, par, mine, myj, myy);
        const uint32_t jn = u.jn[par];
        if (st.j1 - st.j0 < (1u << 26))
          units_pass2<MODE, false, NT, P, G, UR, UCAP>(a, u, cs, st.kbase, nullptr);
        else
          units_pass2<MODE, false, NT, P, G, UR, UCAP, Store, false>(a, u, cs, st.kbase, nullptr);
        cta_sync<NT>();
        if (tid == 0) u.jn[par] = FULL;
        slot_flush<MODE>(a, u.slo, u.shi, mine, myj, myy);
        jc = jn != FULL ? jn : ((st.j1 - jc > (uint32_t)NT) ? jc + NT : st.j1);
        K0 = Kn;
        par ^= 1u;
      }
    }
    for (uint32_t i = tid; i < cnt; i += NT) {
      if constexpr (CACHE) {
        cs.zero_at(listi[i]);
      } else {
        const uint32_t key = list_get<SPILL>(list, lcap, olist, i);
        cs.zero(key, key - st.kbase);
      }
    }
    if constexpr (Store::kScan) cs.template scan_reset<NT>(hany);
  }
  pf.mark(6);
  cta_sync<NT>();
  pf.mark(3);
  if (tid == 0) u.lcnt = 0;
}

// ------------------------------------------------------------- slot mode
// Starts whose segments are short on average (c4's item starts: a few wedges
// per slot) waste most lanes of a P-wedge unit and most of a chunk's barriers.
// They run in slot mode instead: thread per slot, walking its segment with
// four predicated loads in flight; pass-2 sums stay in a register per slot.
#ifndef BF_SLOT_MODE_AVG
#define BF_SLOT_MODE_AVG 16
#endif
constexpr uint32_t SLOT_MODE_AVG = BF_SLOT_MODE_AVG;
constexpr uint64_t kKeyBufMax = (uint64_t)2 << 30;  // keys (8 GB)  // slot mode when w < SLOT_MODE_AVG * #slots (measured: 6 -> 16 takes c4 50.6 -> 38.5 ms)

// Each thread keeps SB slots in flight (strided by NT): their (lo, len) pairs,
// then up to four keys of each -- SB independent random N(y) reads per thread,
// the memory-level parallelism that short random segments need.  With a key
// buffer (a.kbuf, vertex mode, graphs of mostly short segments) pass 1 also
// stores each segment's keys at kbuf[wpre[j] + i] -- the wedge's global index --
// so pass 2 reads them back sequentially instead of gathering N(y) again.
// (SB = 4 only on graphs of short segments, a separate kernel instance: the
// four-slot code in the same kernel cost c2 0.35 ms through register pressure.)
template <bool SPILL, int NT, int SB, class Store>
__device__ __forceinline__ void slots_pass1(const CountArgs& a, const Store& cs, uint32_t j0, uint32_t j1,
                                            uint32_t kbase, uint32_t* lcnt, uint32_t* list, uint32_t lcap,
                                            uint32_t* olist, bool& hashed) {
  for (uint32_t jb = j0 + threadIdx.x; jb < j1; jb += NT * SB) {
    uint32_t lo[SB], len[SB], k[SB][4];
#pragma unroll
    for (int b = 0; b < SB; b++) {
      const uint32_t j = jb + b * NT;
      len[b] = j < j1 ? __ldg(a.seglen + j) : 0u;
      lo[b] = j < j1 ? __ldg(a.seglo + j) : 0u;
    }
#pragma unroll
    for (int b = 0; b < SB; b++)
#pragma unroll
      for (int t = 0; t < 4; t++) k[b][t] = t < (int)len[b] ? __ldg(a.nbr + (lo[b] + t)) : EMPTY;
    if (a.kbuf) {
#pragma unroll
      for (int b = 0; b < SB; b++)
        if (len[b]) {
          uint32_t* kb = a.kbuf + __ldg(a.wpre + jb + b * NT);
#pragma unroll
          for (int t = 0; t < 4; t++)
            if (t < (int)len[b]) kb[t] = k[b][t];
        }
    }
#pragma unroll
    for (int b = 0; b < SB; b++)
#pragma unroll
      for (int t = 0; t < 4; t++)
        if (k[b][t] != EMPTY && cs.add(k[b][t], k[b][t] - kbase, hashed))
          list_push<SPILL>(lcnt, list, lcap, olist, a.olist_len, k[b][t]);
    // the rest of segments longer than four
#pragma unroll 1
    for (int b = 0; b < SB; b++) {
      if (len[b] <= 4) continue;
      uint32_t* kb = a.kbuf ? a.kbuf + __ldg(a.wpre + jb + b * NT) : nullptr;
      for (uint32_t i0 = 4; i0 < len[b]; i0 += 4) {
        uint32_t kk[4];
#pragma unroll
        for (int t = 0; t < 4; t++) kk[t] = i0 + t < len[b] ? __ldg(a.nbr + (lo[b] + i0 + t)) : EMPTY;
#pragma unroll
        for (int t = 0; t < 4; t++)
          if (kk[t] != EMPTY) {
            if (kb) kb[i0 + t] = kk[t];
            if (cs.add(kk[t], kk[t] - kbase, hashed)) list_push<SPILL>(lcnt, list, lcap, olist, a.olist_len, kk[t]);
          }
      }
    }
  }
}

template <int MODE, int NT, int SB, class Store>
__device__ __forceinline__ void slots_pass2(const CountArgs& a, const Store& cs, uint32_t j0, uint32_t j1,
                                               uint32_t kbase) {
  const bool kb = MODE == MODE_VERTEX && a.kbuf != nullptr;  // keys from the key buffer
  for (uint32_t jb = j0 + threadIdx.x; jb < j1; jb += NT * SB) {
    uint32_t lo[SB], len[SB], k[SB][4];
    uint64_t s[SB];
#pragma unroll
    for (int b = 0; b < SB; b++) {
      const uint32_t j = jb + b * NT;
      len[b] = j < j1 ? __ldg(a.seglen + j) : 0u;
      lo[b] = 0u;
      if (j < j1) lo[b] = kb ? 0u : __ldg(a.seglo + j);
      s[b] = 0;
    }
    const uint32_t* src[SB];
#pragma unroll
    for (int b = 0; b < SB; b++) src[b] = kb ? (len[b] ? a.kbuf + __ldg(a.wpre + jb + b * NT) : a.kbuf) : a.nbr + lo[b];
#pragma unroll
    for (int b = 0; b < SB; b++)
#pragma unroll
      for (int t = 0; t < 4; t++) k[b][t] = t < (int)len[b] ? (kb ? __ldcs(src[b] + t) : __ldg(src[b] + t)) : EMPTY;
#pragma unroll
    for (int b = 0; b < SB; b++)
#pragma unroll
      for (int t = 0; t < 4; t++)
        if (k[b][t] != EMPTY) {
          const uint32_t c = cs.get(k[b][t], k[b][t] - kbase) - 1u;
          s[b] += c;
          if (MODE == MODE_EDGE && c) red_add_u64(a.acc + (lo[b] + t), c);  // edge (y, key)
        }
#pragma unroll 1
    for (int b = 0; b < SB; b++) {
      for (uint32_t i0 = 4; i0 < len[b]; i0 += 4) {
        uint32_t kk[4];
#pragma unroll
        for (int t = 0; t < 4; t++)
          kk[t] = i0 + t < len[b] ? (kb ? __ldcs(src[b] + i0 + t) : __ldg(src[b] + i0 + t)) : EMPTY;
#pragma unroll
        for (int t = 0; t < 4; t++)
          if (kk[t] != EMPTY) {
            const uint32_t c = cs.get(kk[t], kk[t] - kbase) - 1u;
            s[b] += c;
            if (MODE == MODE_EDGE && c) red_add_u64(a.acc + (lo[b] + i0 + t), c);  // edge (y, key)
          }
      }
      const uint32_t j = jb + b * NT;
      if (s[b]) {
        if (MODE == MODE_VERTEX) { if (!(a.exp & 2)) red_add_u64(a.bv + __ldg(a.nbr + j), s[b]); }  // centre y
        else red_add_u64(a.acc + j, s[b]);                                                         // edge (s, y)
      }
    }
  }
}

// counter-index cache per small tier (warp tier: NT == 32): pass 1 records each
// wedge's counter byte index (u16) and each owner's, pass 2 / finalize / reset
// read the counters through them.  (Round 1's cache of the 32-bit KEYS was
// slower than re-reading them through L1: 6.96 -> 6.85 ms without it.)
#ifndef BF_WARP_CACHE
#define BF_WARP_CACHE 1
#endif
#ifndef BF_MED_CACHE
#define BF_MED_CACHE 1
#endif
#define SMALL_CACHE(NT) ((NT) == 32 ? (BF_WARP_CACHE != 0) : (BF_MED_CACHE != 0))

// ------------------------------------------------------------- small tiers
// warp / medium: u8 dense window + shared hash; one chunk per start (w <= CAP,
// slots <= NT).  Starts are taken in a static stride (the tier is sorted by
// wedges, so neighbours in the stride are alike) with a two-stage register
// prefetch: the item two starts ahead and the slot data one start ahead are in
// flight while the current start runs.
template <int NT, uint32_t WIN, uint32_t HS, uint32_t CAP, int P, int G, int UR>
struct SmallSmem {
  static constexpr uint32_t UCAP = CAP / P + NT;
  Units<NT, UCAP> u;
  alignas(16) uint32_t win[WIN / 4 + HS / 4];  // u8 counters: the dense window, then the hash slots' counts
  alignas(16) uint32_t hk[HS];
  uint32_t list[SMALL_CACHE(NT) ? 1 : CAP];   // distinct keys <= w <= CAP (without the index cache)
  uint16_t listi[SMALL_CACHE(NT) ? CAP : 2];  // the owners' counter indices (with it)
  uint16_t cache[SMALL_CACHE(NT) ? CAP : 2];  // each wedge's counter index, in chunk order
  static_assert(WIN + HS <= 65536, "counter indices are u16");
};

struct SlotRegs {
  uint32_t lo, len, y;
};

template <int MODE>
__device__ __forceinline__ SlotRegs load_slot(const CountArgs& a, uint32_t j, uint32_t j1) {
  SlotRegs r{0u, 0u, 0u};
  if (j < j1) {
    r.lo = __ldg(a.seglo + j);
    r.len = __ldg(a.seglen + j);
    if (MODE == MODE_VERTEX) r.y = __ldg(a.nbr + j);
  }
  return r;
}

// medium-tier CTAs per SM (register cap 65536 / (128 * MINB)): 8 -> 64 registers
// (measured on c2: 48 registers 0.04 ms slower, 40 registers 0.15 ms slower;
// c3 per-edge: 48 or 64 the same)
#ifndef BF_MED_MINB
#define BF_MED_MINB 8
#endif
template <int ORIENT, int MODE, int NT, uint32_t WIN, uint32_t HS, uint32_t CAP, int P, int G, int UR>
__global__ void __launch_bounds__(NT, NT == 32 ? 1 : BF_MED_MINB) k_small(CountArgs a) {
  using SM = SmallSmem<NT, WIN, HS, CAP, P, G, UR>;
  extern __shared__ __align__(16) char sm[];
  SM& ss = *(SM*)sm;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  static_assert((HS & (HS - 1)) == 0 && (WIN & (WIN - 1)) == 0 && WIN >= 16 && HS >= 16, "store sizes (scans read 16 counters at a time)");
  SmallStore<NT, MODE> cs;
  static_assert(!decltype(cs)::kOwn2 || SMALL_CACHE(NT), "OWN2 resets once-seen keys through the counter-index cache");
  cs.win = ss.win;
  cs.hk = ss.hk;
  cs.hv = ss.win + WIN / 4;
  cs.wl = min(a.win, WIN);
  cs.winb = WIN;
  cs.hmask = HS - 1;
  cs.shift = __clz(HS) + 1;  // 32 - log2(HS)
  for (uint32_t i = tid; i < WIN / 4 + HS / 4; i += NT) ss.win[i] = 0;
  for (uint32_t i = tid; i < HS; i += NT) ss.hk[i] = EMPTY;
  if (tid == 0) ss.u.lcnt = 0;
  cta_sync<NT>();
  uint64_t tot_acc = 0, pair_acc = 0;
  Prof pf;
  pf.start();
  // pipeline: cur item + slot regs, next item
  uint32_t q = blockIdx.x;
  uint32_t it = dealt(a, q);
  if (it == EMPTY) return;
  Start st = load_start<ORIENT>(a, it);
  SlotRegs sr = load_slot<MODE>(a, st.j0 + tid, st.j1);
  uint32_t itn = dealt(a, q + gridDim.x);
  Start stn{};
  if (itn != EMPTY) stn = load_start<ORIENT>(a, itn);
  for (;;) {
    // prefetch: slot data of the next start, the item after it
    SlotRegs srn{0u, 0u, 0u};
    uint32_t itnn = EMPTY;
    Start stnn{};
    if (itn != EMPTY) {
      srn = load_slot<MODE>(a, stn.j0 + tid, stn.j1);
      itnn = dealt(a, q + 2 * gridDim.x);
      if (itnn != EMPTY) stnn = load_start<ORIENT>(a, itnn);
    }
    pf.mark(0);
    // ---- the current start
    units_write<NT, P, SM::UCAP>(ss.u, sr.lo, sr.len);
    cs.nk = min(cs.wl, key_range<ORIENT>(st.s, a.n_u, a.n));
    pf.mark(1);
    uint64_t lsum = 0;
    bool hashed = false;
    start_passes<ORIENT, MODE, false, SMALL_CACHE(NT), NT, P, G, UR, SM::UCAP>(a, ss.u, cs, st, true, 0, 0, 0, CAP, FULL, sr.len != 0,
                                                       st.j0 + tid, sr.y, ss.list, CAP, nullptr, lsum, pair_acc,
                                                       hashed, pf, ss.cache, ss.listi);
    tot_acc += lsum;
    if (MODE == MODE_VERTEX) {
      const uint64_t t = warp_sum(lsum);
      if (lane == 0 && t) red_add_u64(a.bv + st.s, t);
    }
    pf.mark(7);
    if (itn == EMPTY) break;
    q += gridDim.x;
    st = stn;
    sr = srn;
    itn = itnn;
    stn = stnn;
  }
  pf.flush(NT == 32 ? 2 : 1);
  flush_totals(a, tot_acc, pair_acc);
}

// ------------------------------------------------------------- heavy tier
// u32 dense window + per-CTA global overflow row; chunked; dynamic queue.
template <int NT, uint32_t WIN, uint32_t CAP, uint32_t LCAP, int P, int G, int UR>
struct HeavySmemT {
  static constexpr uint32_t UCAP = CAP / P + NT;
  Units<NT, UCAP> u;
  alignas(16) uint32_t win[WIN + 32];  // + the walks' per-lane sink counters
  uint32_t list[LCAP];
};
// split starts whose key ranges all fit DENSE_MAX_KEYS (c4: 30K items) are
// counted in a shared window over the whole key range -- the paper's
// simple-batching array of every possible second endpoint held on
// chip -- so no key of a piece takes the global row in pass 1.  (The same
// window for the heavy tier, one 1024-thread CTA per SM, measured slower on c4
// than four 256-thread CTAs with a 4096-key window: 7.3 against 5.5 ms.)
constexpr uint32_t DENSE_MAX_KEYS = 40960;

// heavy-tier CTAs per SM: the register cap 65536 / (256 * MINB) against the
// latency of the N(y) reads.  Measured (wedge kernels, c2 vertex / c3 edge /
// c4 vertex): 64 registers 5.63 / 85.4 / 12.6 ms; 48 (MINB 5) 5.59 / 77.2;
// 40 (MINB 6) 5.39 / 91.3 -- so 40 registers for vertex and total counts, 48
// for per-edge counts (more live state per wedge).  SB == 4 (short-segment
// graphs: c4) keeps four CTAs per SM (14.5 -> 13.2 ms against uncapped).
#ifndef BF_BIG_MINB
#define BF_BIG_MINB 6
#endif
#ifndef BF_BIG_MINB_E
#define BF_BIG_MINB_E 5
#endif
template <int ORIENT, int MODE, int SB, int NT, uint32_t WIN, uint32_t CAP, uint32_t LCAP, int P, int G, int UR>
__global__ void __launch_bounds__(NT, SB == 4 ? 4 : (MODE == MODE_EDGE ? BF_BIG_MINB_E : BF_BIG_MINB)) k_big(CountArgs a) {
  using SM = HeavySmemT<NT, WIN, CAP, LCAP, P, G, UR>;
  extern __shared__ __align__(16) char sm[];
  SM& hs = *(SM*)sm;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  HeavyStore cs;
  cs.win = hs.win;
  cs.ws = (uint32_t)__cvta_generic_to_shared(hs.win);
  cs.sink = WIN;
  cs.orow = a.orow + (size_t)blockIdx.x * a.orow_len;
  cs.wl = min(a.win, WIN);
  cs.lenchk = a.orow_len;
  uint32_t* olist = a.olist + (size_t)blockIdx.x * a.olist_len;
  const uint32_t cap = min(a.cap, CAP);
  for (uint32_t i = tid; i < WIN; i += NT) hs.win[i] = 0;
  if (tid == 0) { hs.u.jn[0] = hs.u.jn[1] = FULL; hs.u.lcnt = 0; }
  uint64_t tot_acc = 0, pair_acc = 0;
  Prof pf;
  pf.start();
  for (;;) {
    if (tid == 0) hs.u.item = atomicAdd(a.queue, 1u);
    __syncthreads();
    const uint32_t it = dealt(a, hs.u.item);
    if (it == EMPTY) break;
    const Start st = load_start<ORIENT>(a, it);
    cs.nk = min(cs.wl, key_range<ORIENT>(st.s, a.n_u, a.n));
    const uint64_t base = __ldg(a.wpre + st.j0);
    const uint64_t w = __ldg(a.wpre + st.j1) - base;
    const bool single = w <= cap && st.j1 - st.j0 <= (uint32_t)NT;
    uint64_t lsum = 0;
    bool hashed = false;
    pf.mark(0);
    if (w < (uint64_t)SLOT_MODE_AVG * (st.j1 - st.j0)) {  // short segments: slot mode
      slots_pass1<true, NT, SB>(a, cs, st.j0, st.j1, st.kbase, &hs.u.lcnt, hs.list, LCAP, olist, hashed);
      __syncthreads();
      const uint32_t cnt = hs.u.lcnt;
      list_finalize<MODE, true, NT>(a, cs, st.kbase, cnt, hs.list, LCAP, olist, lsum);
      if constexpr (HeavyStore::kScan) cs.template scan_finalize<MODE, NT>(a, st.kbase, false, lsum, pair_acc);
      if (tid == 0) pair_acc += cnt;
      __syncthreads();
      if (MODE != MODE_TOTAL) {
        slots_pass2<MODE, NT, SB>(a, cs, st.j0, st.j1, st.kbase);
        __syncthreads();
      }
      for (uint32_t i = tid; i < cnt; i += NT) {
        const uint32_t key = list_get<true>(hs.list, LCAP, olist, i);
        cs.zero(key, key - st.kbase);
      }
      if constexpr (HeavyStore::kScan) cs.template scan_reset<NT>(false);
      __syncthreads();
      if (tid == 0) hs.u.lcnt = 0;
    } else {
      bool mine;
      uint32_t myj, myy;
      const uint64_t K1 = units_build<MODE, NT, P, SM::UCAP>(a, hs.u, st.j0, st.j1, base, 0, cap, 0, mine, myj, myy);
      const uint32_t jn0 = hs.u.jn[0];
      start_passes<ORIENT, MODE, true, false, NT, P, G, UR, SM::UCAP>(a, hs.u, cs, st, single, base, w, K1, cap, jn0,
                                                                      mine, myj, myy, hs.list, LCAP, olist, lsum,
                                                                      pair_acc, hashed, pf, (uint16_t*)nullptr, nullptr);
    }
    tot_acc += lsum;
    if (MODE == MODE_VERTEX) {
      const uint64_t t = warp_sum(lsum);
      if (lane == 0 && t) red_add_u64(a.bv + st.s, t);
    }
    pf.mark(7);
  }
  pf.flush(0);
  flush_totals(a, tot_acc, pair_acc);
}

// ------------------------------------------------------------- split starts
// A start with more wedges than the split threshold is cut into pieces (slot
// ranges of about equal wedge count) that many CTAs count at once: window keys
// in shared memory, flushed per piece into the start's global dense d-row;
// other keys straight into the row.  A separate finalize runs once every piece
// is counted (the two-pass discipline), then pass 2 re-walks the
// pieces with the row frozen.  Whole split starts are dealt to ranks.
struct SplitArgs {
  const uint4* split;     // {s, j0, j1, -}
  const uint64_t* off;    // row / list offset of each split start (keys)
  uint32_t* cnt;          // touched-list count per split start
  const uint4* pieces;    // {split index, slot begin, slot end, -}
  uint32_t* rows;         // dense d-rows of this batch
  uint32_t* lists;        // touched lists of this batch
  uint32_t s0, s1, p0, p1;
};

__device__ __forceinline__ bool split_mine(const CountArgs& a, uint32_t i) {
  const uint32_t G = (uint32_t)a.world, q = i / G, r = i % G;
  return (uint32_t)a.rank == ((q & 1u) ? G - 1 - r : r);
}

template <int ORIENT>
__device__ __forceinline__ uint32_t split_kbase(const CountArgs& a, uint32_t s) {
  return ORIENT == BF_ORIENT_HIGH ? (s < a.n_u ? 0u : a.n_u) : s + 1u;
}
// the key range of start s (its d-row's length): same-side rids ranked above s
// (HIGH) or below it (LOW)
template <int ORIENT>
__device__ __forceinline__ uint32_t split_keys(const CountArgs& a, uint32_t s) {
  if (ORIENT == BF_ORIENT_HIGH) return s < a.n_u ? s : s - a.n_u;
  return s < a.n_u ? a.n_u - s - 1u : (uint32_t)(a.n - s - 1u);
}

struct SplitStore1 {
  uint32_t* win;
  uint32_t wl;
  uint32_t* row;
  uint32_t* glist;
  uint32_t* gcnt;
  __device__ __forceinline__ bool add(uint32_t key, uint32_t kk, bool&) const {
    if (kk < wl) return atomicAdd(win + kk, 1u) == 0u;
    if (atomicAdd(row + kk, 1u) == 0u) glist[atomicAdd(gcnt, 1u)] = key;
    return false;
  }
};
// dense variant: every key is in the shared window; owners are not tracked
// (the flush scans the window)
struct SplitStore1Dense {
  uint32_t* win;
  __device__ __forceinline__ bool add(uint32_t, uint32_t kk, bool&) const {
    atomicAdd(win + kk, 1u);
    return false;
  }
};
// dense pass 2: the start's d-row copied into shared memory per piece
struct SplitStore2Shared {
  const uint32_t* win;
  __device__ __forceinline__ uint32_t get(uint32_t, uint32_t kk) const { return win[kk]; }
};
struct SplitStore2 {
  const uint32_t* row;
  __device__ __forceinline__ uint32_t get(uint32_t, uint32_t kk) const { return __ldcg(row + kk); }
};

constexpr int SP_NT = 256;    // pass 1 with the 8192-key window + owner list
constexpr int SP_NT_WIDE = 1024;  // dense pass 1 (one CTA per SM around the whole-key window) and pass 2
constexpr uint32_t SP_WIN = 8192, SP_CAP = 8192;
constexpr int SP_P = 32, SP_G = 4;
template <int NT>
struct SplitSmemT {
  static constexpr uint32_t UCAP = SP_CAP / SP_P + NT;
  using U = Units<NT, UCAP>;
  U u;
  uint32_t win[SP_WIN];
  uint32_t list[SP_WIN];  // window owners of the piece (distinct window keys <= SP_WIN)
};

// DENSE: the window covers every key of every split start (a.dwin keys of
// dynamic shared memory after the unit table; no owner list)
// NT == SP_NT_WIDE runs with only the unit table in shared memory (pass 2) or
// the unit table plus the dense window (pass 1, DENSE): win / list of the
// struct are never touched then.
template <int ORIENT, int MODE, bool PASS2, bool DENSE, int NT>
__global__ void __launch_bounds__(NT, NT == SP_NT ? 3 : 1) k_split_walk(CountArgs a, SplitArgs sa) {
  extern __shared__ __align__(16) char sm[];
  using SplitSmem = SplitSmemT<NT>;
  SplitSmem& ss = *(SplitSmem*)sm;
  using U = typename SplitSmem::U;
  const uint32_t tid = threadIdx.x;
  const uint32_t cap = min(a.cap, SP_CAP);
  uint32_t* win = DENSE ? (uint32_t*)(sm + sizeof(U)) : ss.win;
  const uint32_t wl = DENSE ? a.dwin : min(a.win, SP_WIN);
  if (!PASS2)
    for (uint32_t i = tid; i < wl; i += NT) win[i] = 0;
  if (tid == 0) { ss.u.jn[0] = ss.u.jn[1] = FULL; ss.u.lcnt = 0; }
  for (;;) {
    if (tid == 0) ss.u.item = sa.p0 + atomicAdd(a.queue, 1u);
    __syncthreads();
    const uint32_t p = ss.u.item;
    __syncthreads();  // every thread has read the item before thread 0 takes the next
    if (p >= sa.p1) break;
    const uint4 pc = __ldg(sa.pieces + p);
    if (!split_mine(a, pc.x)) continue;  // CTA-uniform
    const uint4 sp = __ldg(sa.split + pc.x);
    const uint32_t kbase = split_kbase<ORIENT>(a, sp.x);
    uint32_t* row = sa.rows + __ldg(sa.off + pc.x);
    uint32_t* glist = sa.lists + __ldg(sa.off + pc.x);
    SplitStore1 s1{win, wl, row, glist, sa.cnt + pc.x};
    SplitStore1Dense s1d{win};
    SplitStore2 s2{row};
    SplitStore2Shared s2d{win};
    if (PASS2 && DENSE) {  // the start's whole d-row to shared memory (its key range <= a.dwin)
      const uint32_t kr = split_keys<ORIENT>(a, sp.x);
      for (uint32_t kk = tid; kk < kr; kk += NT) win[kk] = __ldcg(row + kk);
      __syncthreads();
    }
    const uint64_t base = __ldg(a.wpre + pc.y), w = __ldg(a.wpre + pc.z) - base;
    uint32_t jc = pc.y, par = 0;
    uint64_t K0 = 0;
    bool hashed = false;
    if (w < (uint64_t)SLOT_MODE_AVG * (pc.z - pc.y)) {  // short segments: slot mode
      if (PASS2 && DENSE) slots_pass2<MODE, NT, 4>(a, s2d, pc.y, pc.z, kbase);
      else if (PASS2) slots_pass2<MODE, NT, 4>(a, s2, pc.y, pc.z, kbase);
      else if (DENSE) slots_pass1<false, NT, 4>(a, s1d, pc.y, pc.z, kbase, &ss.u.lcnt, ss.list, SP_WIN, nullptr, hashed);
      else slots_pass1<false, NT, 4>(a, s1, pc.y, pc.z, kbase, &ss.u.lcnt, ss.list, SP_WIN, nullptr, hashed);
      __syncthreads();
      K0 = w;  // skip the unit walk
    }
    while (K0 < w) {
      bool mine;
      uint32_t myj, myy;
      const uint64_t K1 = units_build<PASS2 ? MODE : MODE_TOTAL, NT, SP_P, SplitSmem::UCAP>(
          a, ss.u, jc, pc.z, base, K0, cap, par, mine, myj, myy);
      const uint32_t jn = ss.u.jn[par];
      if (PASS2 && DENSE) {
        if (sp.z - sp.y < (1u << 26))
          units_pass2<MODE, false, NT, SP_P, SP_G, 1, SplitSmem::UCAP>(a, ss.u, s2d, kbase, nullptr);
        else
          units_pass2<MODE, false, NT, SP_P, SP_G, 1, SplitSmem::UCAP, SplitStore2Shared, false>(a, ss.u, s2d, kbase,
                                                                                                   nullptr);
      } else if (PASS2) {
        if (sp.z - sp.y < (1u << 26))
          units_pass2<MODE, false, NT, SP_P, SP_G, 1, SplitSmem::UCAP>(a, ss.u, s2, kbase, nullptr);
        else
          units_pass2<MODE, false, NT, SP_P, SP_G, 1, SplitSmem::UCAP, SplitStore2, false>(a, ss.u, s2, kbase,
                                                                                             nullptr);
      }
      else if (DENSE)
        units_pass1<false, false, NT, SP_P, SP_G, 1, SplitSmem::UCAP>(a, ss.u, s1d, kbase, ss.list, SP_WIN, nullptr,
                                                                         hashed, nullptr, nullptr);
      else units_pass1<false, false, NT, SP_P, SP_G, 1, SplitSmem::UCAP>(a, ss.u, s1, kbase, ss.list, SP_WIN, nullptr, hashed,
                                                              nullptr, nullptr);
      __syncthreads();
      if (tid == 0) ss.u.jn[par] = FULL;
      if (PASS2) slot_flush<MODE>(a, ss.u.slo, ss.u.shi, mine, myj, myy);
      jc = jn != FULL ? jn : ((pc.z - jc > (uint32_t)NT) ? jc + NT : pc.z);
      K0 = K1;
      par ^= 1u;
    }
    if (!PASS2 && DENSE) {  // flush the piece's window into the start's row (scan: no owner list)
      for (uint32_t kk = tid; kk < wl; kk += NT) {
        const uint32_t c = win[kk];
        if (!c) continue;
        win[kk] = 0;
        if (atomicAdd(row + kk, c) == 0u) glist[atomicAdd(sa.cnt + pc.x, 1u)] = kk + kbase;
      }
      __syncthreads();
    } else if (!PASS2) {  // flush the piece's window counts into the start's row
      const uint32_t cnt = ss.u.lcnt;
      for (uint32_t i = tid; i < cnt; i += NT) {
        const uint32_t key = ss.list[i], kk = key - kbase;
        const uint32_t c = win[kk];
        win[kk] = 0;
        if (atomicAdd(row + kk, c) == 0u) glist[atomicAdd(sa.cnt + pc.x, 1u)] = key;
      }
      __syncthreads();
      if (tid == 0) ss.u.lcnt = 0;
    }
  }
}

// finalize (after every piece is counted): C(d,2) to the total and both
// endpoints; total mode also resets the row and the list here
template <int ORIENT, int MODE>
__global__ void __launch_bounds__(256) k_split_finalize(CountArgs a, SplitArgs sa) {
  uint64_t tot_acc = 0, pair_acc = 0;
  __shared__ unsigned long long s_sum;
  for (uint32_t i = sa.s0 + blockIdx.x; i < sa.s1; i += gridDim.x) {
    if (!split_mine(a, i)) continue;
    const uint4 sp = __ldg(sa.split + i);
    const uint32_t kbase = split_kbase<ORIENT>(a, sp.x);
    uint32_t* row = sa.rows + sa.off[i];
    const uint32_t* glist = sa.lists + sa.off[i];
    const uint32_t cnt = __ldcg(sa.cnt + i);
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    uint64_t lsum = 0;
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
      const uint32_t key = __ldcg(glist + t), kk = key - kbase;
      const uint32_t d = __ldcg(row + kk);
      const uint64_t c2 = choose2(d);
      lsum += c2;
      if (MODE == MODE_VERTEX && c2) red_add_u64(endpoint_slot(a, key), c2);
    }
    tot_acc += lsum;
    if (threadIdx.x == 0) pair_acc += cnt;
    if (MODE == MODE_VERTEX) {
      const uint64_t t = warp_sum(lsum);
      if ((threadIdx.x & 31) == 0 && t) atomicAdd(&s_sum, (unsigned long long)t);
      __syncthreads();
      if (threadIdx.x == 0 && s_sum) red_add_u64(a.bv + sp.x, s_sum);
    }
    __syncthreads();
    if (MODE == MODE_TOTAL) {  // reset after the barrier (see list_finalize)
      for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) __stcg(row + (__ldcg(glist + t) - kbase), 0u);
      __syncthreads();
      if (threadIdx.x == 0) sa.cnt[i] = 0;
    }
  }
  flush_totals(a, tot_acc, pair_acc);
}

// reset rows and lists after pass 2
template <int ORIENT>
__global__ void __launch_bounds__(256) k_split_clear(CountArgs a, SplitArgs sa) {
  for (uint32_t i = sa.s0 + blockIdx.x; i < sa.s1; i += gridDim.x) {
    if (!split_mine(a, i)) continue;
    const uint32_t kbase = split_kbase<ORIENT>(a, __ldg(sa.split + i).x);
    uint32_t* row = sa.rows + sa.off[i];
    const uint32_t* glist = sa.lists + sa.off[i];
    const uint32_t cnt = __ldcg(sa.cnt + i);
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) __stcg(row + (__ldcg(glist + t) - kbase), 0u);
    __syncthreads();
    if (threadIdx.x == 0) sa.cnt[i] = 0;
  }
}

// tier configurations <NT, WIN, HS|CAP, CAP|LCAP, P, G, UR>
// warp tier: 1-warp CTAs, w <= 512, <= 32 slots
// window sizes: smaller windows trade overflow-path work for occupancy;
// measured on c2 / c3 (warp, big): (4096, 8192) 7.73 / 92.6 ms,
// (2048, 4096) 7.06, (1024, 4096) 6.97 / 85.6 ms, (512, 4096) 7.10
#ifndef BF_WARP_WIN
#define BF_WARP_WIN 1024
#endif
// medium tier: (8192-key window, key cache, 6 CTAs/SM) -> (4096, no cache,
// 8 CTAs/SM at <= 64 registers): c2 6.86 -> 6.63 ms, c3 84.5 -> 82.5 ms
#ifndef BF_MED_WIN
#define BF_MED_WIN 4096
#endif
#ifndef BF_BIG_WIN
#define BF_BIG_WIN 4096
#endif
// unit shape: P wedges per unit, G lanes per unit.  G = 8 makes every lane
// group read one 32-byte sector per step; the wedge walks are bound by L1/
// shared-memory wavefronts (l1tex ~70% busy), so fewer, fuller sectors per
// warp request beat more units in flight (measured: G = 2 / 4 / 8 / 16 / 32)
#ifndef BF_WARP_P
#define BF_WARP_P 16
#endif
#ifndef BF_WARP_G
#define BF_WARP_G 8
#endif
#ifndef BF_MED_P
#define BF_MED_P 32
#endif
#ifndef BF_MED_G
#define BF_MED_G 8
#endif
#ifndef BF_BIG_G
#define BF_BIG_G 8
#endif
#ifndef BF_WARP_UR
#define BF_WARP_UR 2
#endif
#ifndef BF_MED_UR
#define BF_MED_UR 2
#endif
#define WARP_CFG 32, BF_WARP_WIN, 512, BF_WARP_MAX_WEDGES, BF_WARP_P, BF_WARP_G, BF_WARP_UR
using WarpSM = SmallSmem<WARP_CFG>;
// medium tier: 128 threads, w <= 2048, <= 128 slots
#ifndef BF_MED_HS
#define BF_MED_HS 2048
#endif
#define MED_CFG BF_MEDIUM_MAX_SLOTS, BF_MED_WIN, BF_MED_HS, BF_MEDIUM_MAX_WEDGES, BF_MED_P, BF_MED_G, BF_MED_UR
using MedSM = SmallSmem<MED_CFG>;
// heavy tier: 256 threads, chunks of <= 8192 wedges
#ifndef BF_BIG_NT
#define BF_BIG_NT 256
#endif
#ifndef BF_BIG_CAP
#define BF_BIG_CAP 32768
#endif
#ifndef BF_BIG_LCAP
#define BF_BIG_LCAP 1024  // the shared owner list holds only overflow-row keys (SCAN); more spill to global
#endif
// units of P wedges, UR per lane group in flight.  Vertex and total counts:
// P = 64, one unit (8 keys per lane) -- half the unit-table work of P = 32,
// UR = 2 for the same keys in flight (measured, wedge kernels: c2 5.13 ->
// 5.10 ms, c3 vertex 77.2 -> 63.2, c4 11.8 -> 11.5; P = 128: c2 6.09, c3
// 76.3; P = 64 with UR = 2: c2 5.45); per-edge counts keep P = 32 with UR = 3
// (c3 edge 72.1 ms; UR = 2 73.0, P = 64 74.5)
#ifndef BF_BIG_P
#define BF_BIG_P 64
#endif
#ifndef BF_BIG_UR
#define BF_BIG_UR 1
#endif
#ifndef BF_BIG_P_E
#define BF_BIG_P_E 32
#endif
#ifndef BF_BIG_UR_E
#define BF_BIG_UR_E 3
#endif
#define BIG_CFG BF_BIG_NT, BF_BIG_WIN, BF_BIG_CAP, BF_BIG_LCAP, BF_BIG_P, BF_BIG_G, BF_BIG_UR
#define BIG_CFG_E BF_BIG_NT, BF_BIG_WIN, BF_BIG_CAP, BF_BIG_LCAP, BF_BIG_P_E, BF_BIG_G, BF_BIG_UR_E
constexpr uint64_t HV_WIN_KEYS = BF_BIG_WIN;  // BIG_CFG's window
using BigSM = HeavySmemT<BIG_CFG>;
using BigSME = HeavySmemT<BIG_CFG_E>;
static_assert(BF_WARP_MAX_SLOTS == 32, "warp tier: one slot per lane");
// tuning-macro consistency (a violation would reach __trap or wrap a counter):
// every distinct hashed key of a small-tier start fits its hash (distinct keys
// <= w <= the tier's wedge cap); u8 counters hold d <= #slots; unit tables pack
// chunk positions and lengths in 16 bits
static_assert(512 >= BF_WARP_MAX_WEDGES, "warp hash (512 slots) must hold every key of a warp-tier start");
static_assert(BF_MED_HS >= BF_MEDIUM_MAX_WEDGES, "medium hash must hold every key of a medium-tier start");
static_assert(BF_MEDIUM_MAX_SLOTS <= 255 && BF_WARP_MAX_SLOTS <= 255, "u8 small-tier counters need d <= 255");
static_assert(BF_BIG_CAP < 65536 && BF_MEDIUM_MAX_WEDGES < 65536 && SP_CAP < 65536,
              "unit tables pack chunk positions in 16 bits");

// ============================================================ output kernels
// bv[side base + k] += sum over stripes of hub[stripe][side][k]
__global__ void k_hub_reduce(const uint64_t* __restrict__ hub, uint32_t nU, uint32_t nV, uint64_t* __restrict__ bv) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * HUB_KEYS; i += gridDim.x * blockDim.x) {
    const uint32_t side = i / HUB_KEYS, k = i % HUB_KEYS;
    if (k >= (side ? nV : nU)) continue;
    uint64_t v = 0;
#pragma unroll 4
    for (uint32_t st = 0; st < HUB_STRIPES; st++) v += hub[((size_t)st * 2 + side) * HUB_KEYS + k];
    if (v) bv[(side ? nU : 0u) + k] += v;
  }
}

__global__ void k_unrename(const uint64_t* __restrict__ bv, const uint32_t* __restrict__ rid_of_gid, uint32_t nU,
                           uint64_t n, uint64_t* __restrict__ out_u, uint64_t* __restrict__ out_v) {
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = bv[rid_of_gid[z]];
    if (z < nU) out_u[z] = v;
    else out_v[z - nU] = v;
  }
}

// be[e] = the sums of the edge's two slots.  A binary search in the shorter of
// the two rows (sorted by decreasing rid) finds one slot; its pos gives the
// twin: slot ru->rv at p, rv->ru at off[rv] + pos[p] (and symmetrically)
__device__ __forceinline__ uint32_t row_find(const uint32_t* __restrict__ nbr, uint32_t lo, uint32_t hi, uint32_t x) {
  while (lo < hi) {  // first index with nbr <= x
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (nbr[mid] > x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void k_edge_gather(const uint64_t* __restrict__ acc, const uint32_t* __restrict__ edges,
                              const uint32_t* __restrict__ rid_of_gid, const uint32_t* __restrict__ nbr,
                              const uint32_t* __restrict__ pos, const uint32_t* __restrict__ off, uint32_t nU,
                              uint64_t m, uint64_t* __restrict__ be) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 uv = reinterpret_cast<const uint2*>(edges)[e];
    const uint32_t ru = rid_of_gid[uv.x], rv = rid_of_gid[(uint64_t)nU + uv.y];
    const uint32_t ou = off[ru], du = off[ru + 1] - ou, ov = off[rv], dv = off[rv + 1] - ov;
    uint32_t a, b;
    if (du <= dv) {
      a = row_find(nbr, ou, ou + du, rv);
      b = ov + pos[a];
    } else {
      b = row_find(nbr, ov, ov + dv, ru);
      a = ou + pos[b];
    }
    BF_CHECK(nbr[a] == rv && nbr[b] == ru);
    be[e] = acc[a] + acc[b];
  }
}

inline unsigned grid_for(size_t n, int sms) {
  size_t g = (n + 255) / 256;
  size_t cap = (size_t)sms * 32;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return (unsigned)g;
}

// blocks per SM of a kernel at (threads, dynamic smem); the attribute set and
// the occupancy query are host API calls inside the timed count, so their
// answers are cached per (device, kernel, threads, smem)
// (the dynamic-smem attribute only ever grows, so a cached answer for a
// smaller launch never leaves the attribute below a later launch's need)
template <class K>
int occupancy(K kernel, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  static std::map<std::pair<int, const void*>, size_t> attr;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, (const void*)kernel, threads, smem);
  std::lock_guard<std::mutex> lk(mu);
  size_t& set = attr[std::make_pair(dev, (const void*)kernel)];
  if (smem > set || set == 0) {
    CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
#ifdef BF_CARVEOUT  // tuning: shared-memory carve-out in percent (the rest is L1)
    CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, BF_CARVEOUT));
#endif
    set = std::max<size_t>(smem, 1);
  }
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int b = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem));
  b = b > 0 ? b : 1;
  cache[key] = b;
  return b;
}

// Per-device pool of heavy-tier overflow rows + touched lists.  The lock is
// held by graph_count for the whole call; a failed call marks the rows dirty.
struct RowPool {
  std::mutex m;
  void* p = nullptr;  // overflow rows, all zero between calls
  size_t bytes = 0;
  void* l = nullptr;  // touched lists (scratch)
  size_t lbytes = 0;
  bool dirty = false;
  size_t budget = 0;  // bytes rows + lists may take (set at first use, from the free memory then)
};
// the pool may take up to 60% of the device's free memory (plus what it holds),
// at most 64 GB: c5's heavy key ranges (up to 8M keys, 64 MB of row + list per
// CTA) ran at 1.7 CTAs per SM under round 1's fixed 16 GB
constexpr size_t kRowPoolMax = (size_t)64 << 30;
RowPool& row_pool(int dev) {
  static RowPool pools[64];
  return pools[dev & 63];
}

}  // namespace

// the device's last graph is gone (bf_api.cu device_detach): give the rows back
void row_pool_free(int dev) {
  RowPool& pool = row_pool(dev);
  std::lock_guard<std::mutex> lk(pool.m);
  if (pool.p) cudaFree(pool.p);
  if (pool.l) cudaFree(pool.l);
  pool.p = pool.l = nullptr;
  pool.bytes = pool.lbytes = 0;
  pool.dirty = false;
  pool.budget = 0;
}

namespace {

// BF_FLAG_GRID_JITTER: a pseudo-random grid in [1, grid] (splitmix64 of the
// graph's launch draw), so repeated calls map starts to CTAs differently
int jitter_grid(bf_graph* g, int grid) {
  if (!(g->opt.test_flags & BF_FLAG_GRID_JITTER) || grid <= 1) return grid;
  uint64_t z = (++g->jitter) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return 1 + (int)(z % (uint64_t)grid);
}

template <int ORIENT, int MODE>
void launch_tiers(bf_graph* g, CountArgs a, const uint32_t tier[4], uint32_t* queues, cudaStream_t s) {
  const int sms = g->sms;
  if (g->n_split) {  // split starts, batch by batch
    for (const auto& b : g->split_batches) {
      SplitArgs sa;
      sa.split = g->split.as<uint4>();
      sa.off = g->split_off.as<uint64_t>();
      sa.cnt = g->split_cnt.as<uint32_t>();
      sa.pieces = g->pieces.as<uint4>();
      sa.rows = g->srow.as<uint32_t>();
      sa.lists = g->slist.as<uint32_t>();
      sa.s0 = b.s0; sa.s1 = b.s1; sa.p0 = b.p0; sa.p1 = b.p1;
      const bool dense = a.dwin != 0;
      auto k1 = dense ? k_split_walk<ORIENT, MODE, false, true, SP_NT_WIDE> : k_split_walk<ORIENT, MODE, false, false, SP_NT>;
      const int nt1 = dense ? SP_NT_WIDE : SP_NT;
      const size_t smem = dense ? sizeof(SplitSmemT<SP_NT_WIDE>::U) + (size_t)a.dwin * 4 : sizeof(SplitSmemT<SP_NT>);
      const int grid = jitter_grid(g, sms * occupancy(k1, nt1, smem));
      const int fgrid = jitter_grid(g, (int)std::min<uint32_t>(b.s1 - b.s0, (uint32_t)sms * 8));
      CUDA_TRY(cudaMemsetAsync(queues + 4, 0, 8, s));
      a.queue = queues + 4;
      k1<<<grid, nt1, smem, s>>>(a, sa);
      KERNEL_CHECK(g);
      k_split_finalize<ORIENT, MODE><<<fgrid, 256, 0, s>>>(a, sa);
      KERNEL_CHECK(g);
      if (MODE != MODE_TOTAL) {
        // pass 2 reads the global rows, or (dense) each piece's start row copied to shared memory
        auto k2 = dense ? k_split_walk<ORIENT, MODE, true, true, SP_NT_WIDE> : k_split_walk<ORIENT, MODE, true, false, SP_NT_WIDE>;
        const size_t smem2 = sizeof(SplitSmemT<SP_NT_WIDE>::U) + (dense ? (size_t)a.dwin * 4 : 0);
        a.queue = queues + 5;
        k2<<<jitter_grid(g, sms * occupancy(k2, SP_NT_WIDE, smem2)), SP_NT_WIDE, smem2, s>>>(a, sa);
        KERNEL_CHECK(g);
        k_split_clear<ORIENT><<<fgrid, 256, 0, s>>>(a, sa);
        KERNEL_CHECK(g);
      }
    }
  }
  if (tier[1] > tier[0] + g->n_split) {  // heavy
    auto k = MODE == MODE_EDGE ? (a.short_segs ? k_big<ORIENT, MODE, 4, BIG_CFG_E> : k_big<ORIENT, MODE, 1, BIG_CFG_E>)
                               : (a.short_segs ? k_big<ORIENT, MODE, 4, BIG_CFG> : k_big<ORIENT, MODE, 1, BIG_CFG>);
    const int nt = BF_BIG_NT;
    const size_t smem = MODE == MODE_EDGE ? sizeof(BigSME) : sizeof(BigSM);
    int grid = sms * occupancy(k, nt, smem);
    // one overflow row + touched list per CTA, from the device's row pool
    // (rows are kept zero by the owners' resets, so a clean pool is reused
    // across graphs without clearing); the grid shrinks if the rows of every
    // CTA would exceed the pool budget
    const size_t row_bytes = (a.orow_len + a.olist_len) * 4;
    RowPool& pool = row_pool(g->device);
    grid = (int)std::max<size_t>(1, std::min<size_t>((size_t)grid, g->pool_budget / row_bytes));
    grid = jitter_grid(g, grid);
    // rows (kept zero) and lists (scratch) are separate allocations, so a later
    // launch with another grid never finds list garbage inside its rows
    const size_t need_rows = (size_t)grid * a.orow_len * 4, need_lists = (size_t)grid * a.olist_len * 4;
    if (pool.bytes < need_rows || pool.dirty) {
      if (pool.p) CUDA_TRY(cudaFree(pool.p));
      pool.p = nullptr;
      pool.bytes = 0;
      CUDA_TRY(cudaMalloc(&pool.p, need_rows));
      pool.bytes = need_rows;
      CUDA_TRY(cudaMemsetAsync(pool.p, 0, need_rows, s));
      pool.dirty = false;
    }
    if (pool.lbytes < need_lists) {
      if (pool.l) CUDA_TRY(cudaFree(pool.l));
      pool.l = nullptr;
      pool.lbytes = 0;
      CUDA_TRY(cudaMalloc(&pool.l, need_lists));
      pool.lbytes = need_lists;
    }
    a.orow = (uint32_t*)pool.p;   // [grid][orow_len]
    a.olist = (uint32_t*)pool.l;  // [grid][olist_len]
    a.t0 = tier[0] + g->n_split; a.t1 = tier[1]; a.queue = queues + 0;
    k<<<grid, nt, smem, s>>>(a);
    KERNEL_CHECK(g);
  }
  if (tier[2] > tier[1]) {  // medium
    auto k = k_small<ORIENT, MODE, MED_CFG>;
    const int grid = jitter_grid(g, sms * occupancy(k, BF_MEDIUM_MAX_SLOTS, sizeof(MedSM)));
    a.t0 = tier[1]; a.t1 = tier[2]; a.queue = queues + 1;
    k<<<grid, BF_MEDIUM_MAX_SLOTS, sizeof(MedSM), s>>>(a);
    KERNEL_CHECK(g);
  }
  if (tier[3] > tier[2]) {  // warp
    auto k = k_small<ORIENT, MODE, WARP_CFG>;
#ifndef BF_WARP_BLOCKS
#define BF_WARP_BLOCKS 64
#endif
    const int grid = jitter_grid(g, sms * std::min(occupancy(k, 32, sizeof(WarpSM)), BF_WARP_BLOCKS));
    a.t0 = tier[2]; a.t1 = tier[3]; a.queue = queues + 2;
    k<<<grid, 32, sizeof(WarpSM), s>>>(a);
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
  if (mode == MODE_VERTEX) {
    CUDA_TRY(cudaMemsetAsync(g->bv.p, 0, (n + 1) * 8, s));
    g->hub.ensure((size_t)HUB_STRIPES * 2 * HUB_KEYS * 8);
    CUDA_TRY(cudaMemsetAsync(g->hub.p, 0, (size_t)HUB_STRIPES * 2 * HUB_KEYS * 8, s));
  }
  if (mode == MODE_EDGE) {
    g->acc.ensure(std::max<uint64_t>(S, 1) * 8);
    g->be.ensure((std::max<uint64_t>(m, 1) + 1) * 8);
    CUDA_TRY(cudaMemsetAsync(g->acc.p, 0, std::max<uint64_t>(S, 1) * 8, s));
  }
  const uint32_t win = (g->opt.test_flags & BF_FLAG_SMALL_WINDOW) ? 64u : 0xFFFFFFFFu;
  const uint32_t cap = (g->opt.test_flags & BF_FLAG_SMALL_CHUNK) ? 64u : 0xFFFFFFFFu;
  const uint64_t olen = std::max<uint64_t>(g->heavy_keys, 1);  // a heavy start's key offsets are < olen
  // the heavy tier's row pool is held for the whole call (rows must be clean
  // when the next call on this device starts)
  std::unique_lock<std::mutex> pool_lock;
  struct DirtyGuard {
    RowPool* p = nullptr;
    ~DirtyGuard() { if (p) p->dirty = true; }
  } dirty_guard;
  if (g->n_tier[0]) {
    pool_lock = std::unique_lock<std::mutex>(row_pool(g->device).m);
    dirty_guard.p = &row_pool(g->device);
  }
  CountArgs a;
  a.nbr = g->nbr.as<uint32_t>();
  a.wpre = g->wpre.as<uint64_t>();
  a.seglo = g->seglo.as<uint32_t>();
  a.seglen = g->seglen.as<uint32_t>();
  a.items = g->items.as<uint4>();
  a.bv = g->bv.as<uint64_t>();
  a.hub = g->hub.as<uint64_t>();
  a.acc = g->acc.as<uint64_t>();
  a.total = dtot;
  a.orow = nullptr;
  a.olist = nullptr;
  // split pieces count in a whole-key-range window when every heavy start's key range fits
  const bool dense = olen <= DENSE_MAX_KEYS && win == 0xFFFFFFFFu && !(g->opt.test_flags & BF_FLAG_NO_DENSE_ROW);
  a.dwin = dense ? (uint32_t)((olen + 3) & ~3ull) : 0u;
  // slot-mode key buffer: vertex mode, graphs of mostly short segments (average
  // wedges per slot below the slot-mode threshold), W keys within budget
  a.kbuf = nullptr;
  a.short_segs = g->W < (uint64_t)SLOT_MODE_AVG * S || (g->opt.test_flags & BF_FLAG_KEY_BUFFER);
  if (mode == MODE_VERTEX && g->W && g->W <= kKeyBufMax && a.short_segs) {
    g->kbuf.ensure(g->W * 4);
    a.kbuf = g->kbuf.as<uint32_t>();
  }
  const uint64_t hwl = std::min<uint64_t>(win, HV_WIN_KEYS);  // the heavy kernel's window in keys
  a.orow_len = olen > hwl ? olen - hwl : 1;
  a.olist_len = olen;
  a.S = S;
  a.n = n;
#ifdef BF_PROFILE  // timing experiments exist only in the profile build (they break results)
  a.exp = getenv("BF_EXPERIMENT") ? (uint32_t)atoi(getenv("BF_EXPERIMENT")) : 0u;
#else
  a.exp = 0u;
#endif
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
#ifdef BF_PROFILE
  {
    unsigned long long z[24] = {0};
    CUDA_TRY(cudaMemcpyToSymbolAsync(g_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyToSymbolAsync(g_prof_red, z, 32, 0, cudaMemcpyHostToDevice, s));
  }
#endif
  if (g->n_tier[0]) {  // the heavy tier's row-pool budget: fixed at the pool's first use on the device
    RowPool& pool = row_pool(g->device);  // (its lock is held for the whole call: pool_lock above)
    if (!pool.budget) {
      size_t free_b = 0, total_b = 0;
      CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
      pool.budget = std::max<size_t>((size_t)1 << 30, std::min(kRowPoolMax, free_b / 10 * 6));
    }
    g->pool_budget = pool.budget;
  }
  CUDA_TRY(cudaEventRecord(g->ev[1], s));
  NvtxRange nv_walk("bf a5-a7 wedge kernels");
  for (int r = first; r <= last; r++) {
    a.rank = r;
    a.world = G;
    CUDA_TRY(cudaMemsetAsync(g->queue.p, 0, 64, s));
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
  if (mode == MODE_VERTEX) {
    k_hub_reduce<<<16, 512, 0, s>>>(g->hub.as<uint64_t>(), g->n_u, g->n_v, g->bv.as<uint64_t>());
    KERNEL_CHECK(g);
  }
  CUDA_TRY(cudaEventRecord(g->ev[2], s));
#ifdef BF_PROFILE
  {
    unsigned long long h[24];
    CUDA_TRY(cudaMemcpyFromSymbolAsync(h, g_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    unsigned long long hr[4];
    CUDA_TRY(cudaMemcpyFromSymbolAsync(hr, g_prof_red, 32, 0, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    fprintf(stderr, "[bf_prof] endpoint REDs %llu (key<256 %llu, <1024 %llu, <4096 %llu)\n", hr[0], hr[1], hr[2], hr[3]);
    const char* names[8] = {"fetch", "build", "pass1", "sync", "final", "pass2", "flush", "tail"};
    const char* tiers[3] = {"heavy", "medium", "warp"};
    for (int t = 0; t < 3; t++) {
      unsigned long long tot = 0;
      for (int i = 0; i < 8; i++) tot += h[t * 8 + i];
      if (!tot) continue;
      fprintf(stderr, "[bf_prof] %-6s", tiers[t]);
      for (int i = 0; i < 8; i++) fprintf(stderr, " %s=%.1f%%", names[i], 100.0 * h[t * 8 + i] / tot);
      fprintf(stderr, " (cta-cycles %.3g)\n", (double)tot);
    }
  }
#endif
  // a8: outputs (total stored after the array so one allreduce covers both)
  uint64_t* red_buf = nullptr;
  size_t red_cnt = 0;
  if (mode == MODE_VERTEX) {
    CUDA_TRY(cudaMemcpyAsync(g->bv.as<uint64_t>() + n, dtot, 8, cudaMemcpyDeviceToDevice, s));
    red_buf = g->bv.as<uint64_t>();
    red_cnt = n + 1;
  } else if (mode == MODE_EDGE) {
    if (m) {
      k_edge_gather<<<grid_for(m, g->sms), 256, 0, s>>>(g->acc.as<uint64_t>(), g->edges.as<uint32_t>(),
                                                         g->rid_of_gid.as<uint32_t>(), g->nbr.as<uint32_t>(),
                                                         g->pos.as<uint32_t>(), g->off.as<uint32_t>(), g->n_u, m,
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
  // a9: combine across GPUs (one in-place u64 allreduce over [counts | total];
  // a 1-rank communicator runs the same path)
  if (g->opt.nccl_comm) {
    NvtxRange nv("bf a9 allreduce");
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
  dirty_guard.p = nullptr;  // completed: rows are clean again
  CUDA_TRY(cudaEventElapsedTime(&g->last_kernel_ms, g->ev[1], g->ev[2]));
  CUDA_TRY(cudaEventElapsedTime(&g->last_call_ms, g->ev[0], g->ev[3]));
  return BF_OK;
}
