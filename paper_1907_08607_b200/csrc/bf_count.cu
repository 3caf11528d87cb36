// bf_count.cu -- the wedge kernels (§8(a) a5-a8) and the count driver.
//
// One persistent kernel per count, one CTA per SM.  A "start" s is the vertex
// whose wedges are aggregated together:
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
// so the result does not depend on scheduling.
//
// Tiers (wedge-aware batching): starts with w(s) <= light_max run
// one per warp with a warp-private shared-memory open-addressing hash keyed by
// the key's rid (north_star "light u1"); heavier starts run one per CTA with a
// dense shared-memory counter window over the first C keys (hub ids in the HIGH
// orientation) plus a per-CTA global dense overflow row for keys >= C
// (north_star "heavy u1 ... dense per-CTA global counter array"), with
// ballot-compacted touched lists so rows are reset without full clears.
#include "bf_internal.h"
#include "bf_device.cuh"
#include <algorithm>
#include <vector>

namespace {

constexpr int BLOCK = 512;
constexpr int NWARPS = BLOCK / 32;
constexpr uint32_t WIN = 32768;          // dense window entries (u32) = 128 KB
constexpr uint32_t TOUCH_CAP = WIN / 8;  // sparse-window touched list (u32)
constexpr uint32_t HMAX = 1024;          // warp hash slots
constexpr uint32_t EMPTY = 0xFFFFFFFFu;
constexpr uint32_t LIGHT_CHUNK = 64;     // light starts grabbed per queue atomic

// shared-memory layout (bytes)
constexpr size_t SM_WIN = 0;                                   // WIN u32  | NWARPS * HMAX * (key,val)
constexpr size_t SM_WIN_BYTES = (size_t)WIN * 4;
static_assert((size_t)NWARPS * HMAX * 8 == SM_WIN_BYTES, "warp tables must alias the window");
constexpr size_t SM_TOUCH = SM_WIN + SM_WIN_BYTES;             // TOUCH_CAP u32
constexpr size_t SM_BPRE = SM_TOUCH + TOUCH_CAP * 4;           // (BLOCK+1) u32
constexpr size_t SM_BLO = SM_BPRE + (BLOCK + 4) * 4;           // BLOCK u32
constexpr size_t SM_BY = SM_BLO + BLOCK * 4;                   // BLOCK u32
constexpr size_t SM_BSUM = SM_BY + BLOCK * 4;                  // BLOCK u64
constexpr size_t SM_LPRE = SM_BSUM + BLOCK * 8;                // NWARPS * 33 u32
constexpr size_t SM_LLO = SM_LPRE + NWARPS * 33 * 4;           // NWARPS * 32 u32
constexpr size_t SM_LY = SM_LLO + NWARPS * 32 * 4;             // NWARPS * 32 u32
constexpr size_t SM_LSUM = SM_LY + NWARPS * 32 * 4;            // NWARPS * 32 u32
constexpr size_t SM_TOTAL = SM_LSUM + NWARPS * 32 * 4;

struct CountArgs {
  const uint32_t* off;
  const uint32_t* nbr;
  const uint32_t* pos;
  const uint32_t* hi;
  const uint64_t* wstart;
  const uint32_t* heavy;
  const uint32_t* light;
  uint64_t* bv;       // [n+1] per-vertex (rid), bv[n] unused
  uint64_t* acc;      // [2m] per-slot (edge mode)
  uint64_t* total;    // device scalar
  uint32_t* orow;     // per-CTA overflow rows
  uint32_t* otouch;   // per-CTA overflow touched lists
  uint64_t orow_len;  // entries per CTA row
  uint32_t* queue;    // [0]=heavy cursor [1]=light cursor
  uint32_t n_u, n_v;
  uint32_t heavy_cnt;  // entries of `heavy` in total
  uint32_t light_lo, light_hi;  // this rank's slice of `light`
  uint32_t win;        // active window size (<= WIN)
  int rank, world;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// segment of slot j = (s -> y)
template <int ORIENT>
__device__ __forceinline__ void segment(const CountArgs& a, uint32_t j, uint32_t& y, uint32_t& lo, uint32_t& len) {
  y = a.nbr[j];
  uint32_t p = a.pos[j];
  if (ORIENT == BF_ORIENT_LOW) {
    lo = a.off[y];
    len = p;
  } else {
    uint32_t oy = a.off[y], dy = a.off[y + 1] - oy;
    uint32_t st = max(a.hi[y], p + 1u);
    lo = oy + st;
    len = dy > st ? dy - st : 0u;
  }
}

// largest t in [0, nb) with pre[t] <= k (pre[0] = 0 <= k)
__device__ __forceinline__ uint32_t find_seg(const uint32_t* pre, uint32_t nb, uint32_t k) {
  uint32_t lo = 0, hi = nb;
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (pre[mid] <= k) lo = mid; else hi = mid;
  }
  return lo;
}

// Sum v over each run of equal `seg` among the warp's lanes (segs nondecreasing
// across lanes; inactive lanes carry seg = EMPTY).  Returns true on the run's
// first lane, with *sum the run total (u64 exact).
__device__ __forceinline__ bool run_reduce(uint32_t seg, uint32_t v, bool wide, uint64_t* sum) {
  const int lane = threadIdx.x & 31;
  uint32_t prev = __shfl_up_sync(0xffffffffu, seg, 1);
  bool head = lane == 0 || prev != seg;
  uint32_t heads = __ballot_sync(0xffffffffu, head);
  uint32_t start = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
  uint32_t after = heads & ~(0xffffffffu >> (31 - lane));  // heads above this lane
  uint32_t end = after ? (__ffs(after) - 1) : 32;
  uint32_t mask = (end == 32 ? 0xffffffffu : ((1u << end) - 1u)) & ~((1u << start) - 1u);
  uint64_t s;
  if (!wide) {
    s = __reduce_add_sync(mask, v);
  } else {
    uint32_t lo = __reduce_add_sync(mask, v & 0xffffu);
    uint32_t hi = __reduce_add_sync(mask, v >> 16);
    s = (uint64_t)lo + ((uint64_t)hi << 16);
  }
  *sum = s;
  return head;
}

// ------------------------------------------------------------ CTA tier ------
template <int ORIENT, int MODE>
__device__ void cta_start(const CountArgs& a, uint32_t s, char* sm, uint64_t& tot_acc, uint32_t* s_cnt,
                          uint32_t* s_wt) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t* win = (uint32_t*)(sm + SM_WIN);
  uint32_t* touch = (uint32_t*)(sm + SM_TOUCH);
  uint32_t* bpre = (uint32_t*)(sm + SM_BPRE);
  uint32_t* blo = (uint32_t*)(sm + SM_BLO);
  uint32_t* by = (uint32_t*)(sm + SM_BY);
  unsigned long long* bsum = (unsigned long long*)(sm + SM_BSUM);
  uint32_t* orow = a.orow + (size_t)blockIdx.x * a.orow_len;
  uint32_t* otouch = a.otouch + (size_t)blockIdx.x * a.orow_len;

  const bool isU = s < a.n_u;
  const uint32_t sb = isU ? 0u : a.n_u;
  const uint32_t nside = isU ? a.n_u : a.n_v;
  const uint32_t sl = s - sb;
  const uint32_t keyrange = ORIENT == BF_ORIENT_HIGH ? sl : nside - sl - 1u;
  const uint32_t kbase = ORIENT == BF_ORIENT_HIGH ? sb : s + 1u;
  const uint32_t wlen = min(a.win, keyrange);
  const uint32_t j0 = a.off[s];
  const uint32_t j1 = ORIENT == BF_ORIENT_HIGH ? a.off[s + 1] : j0 + a.hi[s];
  const uint64_t w = a.wstart[s];
  const bool sparse = w < (uint64_t)min(TOUCH_CAP, a.win);
  const bool wide = (a.off[s + 1] - j0) >= (1u << 26);  // d <= deg(s): guards u32 run sums

  // s_cnt[0] = window touched count, s_cnt[1] = overflow touched count
  // ---------------- pass 1: d(key) ----------------
  for (uint32_t b = j0; b < j1; b += BLOCK) {
    const uint32_t nb = min((uint32_t)BLOCK, j1 - b);
    uint32_t y = 0, lo = 0, len = 0;
    if (tid < nb) segment<ORIENT>(a, b + tid, y, lo, len);
    uint32_t tot;
    uint32_t ex = block_exclusive_scan<uint32_t>(len, s_wt, &tot);
    bpre[tid] = ex;
    blo[tid] = lo;
    __syncthreads();
    for (uint32_t k0 = wid * 32; k0 < tot; k0 += BLOCK) {
      const uint32_t k = k0 + lane;
      const bool act = k < tot;
      bool new_w = false, new_o = false;
      uint32_t key = 0;
      if (act) {
        uint32_t t = find_seg(bpre, nb, k);
        uint32_t x2 = __ldg(a.nbr + blo[t] + (k - bpre[t]));
        key = x2 - kbase;
        if (key < wlen) {
          uint32_t old = atomicAdd(&win[key], 1u);
          new_w = sparse && old == 0u;
        } else {
          uint32_t old = atomicAdd(&orow[key - wlen], 1u);
          new_o = old == 0u;
        }
      }
      uint32_t mw = __ballot_sync(0xffffffffu, new_w);
      if (mw) {
        uint32_t base = 0;
        if (lane == __ffs(mw) - 1) base = atomicAdd(&s_cnt[0], (uint32_t)__popc(mw));
        base = __shfl_sync(0xffffffffu, base, __ffs(mw) - 1);
        if (new_w) touch[base + __popc(mw & lanemask_lt())] = key;
      }
      uint32_t mo = __ballot_sync(0xffffffffu, new_o);
      if (mo) {
        uint32_t base = 0;
        if (lane == __ffs(mo) - 1) base = atomicAdd(&s_cnt[1], (uint32_t)__popc(mo));
        base = __shfl_sync(0xffffffffu, base, __ffs(mo) - 1);
        if (new_o) otouch[base + __popc(mo & lanemask_lt())] = key - wlen;
      }
    }
    __syncthreads();
  }
  // ---------------- finalize: C(d,2) -> total, both endpoints -------------
  const uint32_t ntw = s_cnt[0], nto = s_cnt[1];
  uint64_t lsum = 0;
  if (sparse) {
    for (uint32_t t = tid; t < ntw; t += BLOCK) {
      uint32_t key = touch[t];
      uint64_t c = choose2(win[key]);
      lsum += c;
      if (MODE == MODE_VERTEX && c) red_add_u64(a.bv + kbase + key, c);
      if (MODE == MODE_TOTAL) win[key] = 0;
    }
  } else {
    for (uint32_t key = tid; key < wlen; key += BLOCK) {
      uint32_t d = win[key];
      if (d) {
        uint64_t c = choose2(d);
        lsum += c;
        if (MODE == MODE_VERTEX && c) red_add_u64(a.bv + kbase + key, c);
        if (MODE == MODE_TOTAL) win[key] = 0;
      }
    }
  }
  for (uint32_t t = tid; t < nto; t += BLOCK) {
    uint32_t ok = otouch[t];
    uint64_t c = choose2(orow[ok]);
    lsum += c;
    if (MODE == MODE_VERTEX && c) red_add_u64(a.bv + kbase + wlen + ok, c);
    if (MODE == MODE_TOTAL) orow[ok] = 0;
  }
  tot_acc += lsum;
  if (MODE == MODE_VERTEX) {
    uint64_t ws = warp_sum(lsum);
    if (lane == 0 && ws) red_add_u64(a.bv + s, ws);
  }
  if (MODE != MODE_TOTAL) {
    __syncthreads();
    // ---------------- pass 2: d-1 to centres / wedge edges ----------------
    for (uint32_t b = j0; b < j1; b += BLOCK) {
      const uint32_t nb = min((uint32_t)BLOCK, j1 - b);
      uint32_t y = 0, lo = 0, len = 0;
      if (tid < nb) segment<ORIENT>(a, b + tid, y, lo, len);
      uint32_t tot;
      uint32_t ex = block_exclusive_scan<uint32_t>(len, s_wt, &tot);
      bpre[tid] = ex;
      blo[tid] = lo;
      by[tid] = y;
      bsum[tid] = 0;
      __syncthreads();
      for (uint32_t k0 = wid * 32; k0 < tot; k0 += BLOCK) {
        const uint32_t k = k0 + lane;
        const bool act = k < tot;
        uint32_t t = EMPTY, c = 0;
        if (act) {
          t = find_seg(bpre, nb, k);
          uint32_t idx = blo[t] + (k - bpre[t]);
          uint32_t key = __ldg(a.nbr + idx) - kbase;
          uint32_t d = key < wlen ? win[key] : orow[key - wlen];
          c = d - 1u;
          if (MODE == MODE_EDGE && c) red_add_u64(a.acc + idx, c);  // edge (y, key)
        }
        uint64_t rs;
        bool head = run_reduce(t, c, wide, &rs);
        if (head && act && rs) atomicAdd(&bsum[t], (unsigned long long)rs);
      }
      __syncthreads();
      if (tid < nb) {
        uint64_t v = bsum[tid];
        if (v) {
          if (MODE == MODE_VERTEX) red_add_u64(a.bv + by[tid], v);  // centre y
          else red_add_u64(a.acc + b + tid, v);                     // edge (s, y)
        }
      }
      __syncthreads();
    }
    // ---------------- reset rows ----------------
    if (sparse) {
      for (uint32_t t = tid; t < ntw; t += BLOCK) win[touch[t]] = 0;
    } else {
      for (uint32_t key = tid; key < wlen; key += BLOCK) win[key] = 0;
    }
    for (uint32_t t = tid; t < nto; t += BLOCK) orow[otouch[t]] = 0;
  }
  __syncthreads();
  if (tid == 0) { s_cnt[0] = 0; s_cnt[1] = 0; }
  __syncthreads();
}

// ------------------------------------------------------------ warp tier -----
template <int ORIENT, int MODE>
__device__ void warp_start(const CountArgs& a, uint32_t s, char* sm, uint64_t& tot_acc) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* hk = (uint32_t*)(sm + SM_WIN) + (size_t)wid * HMAX * 2;
  uint32_t* hv = hk + HMAX;
  volatile uint32_t* vhk = hk;
  uint32_t* wpre = (uint32_t*)(sm + SM_LPRE) + wid * 33;
  uint32_t* wlo = (uint32_t*)(sm + SM_LLO) + wid * 32;
  uint32_t* wy = (uint32_t*)(sm + SM_LY) + wid * 32;
  uint32_t* wsum = (uint32_t*)(sm + SM_LSUM) + wid * 32;

  const bool isU = s < a.n_u;
  const uint32_t sl = s - (isU ? 0u : a.n_u);
  const uint32_t nside = isU ? a.n_u : a.n_v;
  const uint32_t keyrange = ORIENT == BF_ORIENT_HIGH ? sl : nside - sl - 1u;
  const uint32_t j0 = a.off[s];
  const uint32_t j1 = ORIENT == BF_ORIENT_HIGH ? a.off[s + 1] : j0 + a.hi[s];
  const uint64_t w = a.wstart[s];
  uint32_t want = (uint32_t)(w < (uint64_t)keyrange ? w : (uint64_t)keyrange) * 2u;
  uint32_t hs = 32;
  while (hs < want && hs < HMAX) hs <<= 1;
  const uint32_t hmask = hs - 1, hshift = 32 - (31 - __clz(hs));
  for (uint32_t i = lane; i < hs; i += 32) { hk[i] = EMPTY; hv[i] = 0; }
  __syncwarp();
  // pass 1
  for (uint32_t b = j0; b < j1; b += 32) {
    const uint32_t nb = min(32u, j1 - b);
    uint32_t y = 0, lo = 0, len = 0;
    if (lane < nb) segment<ORIENT>(a, b + lane, y, lo, len);
    uint32_t inc = warp_inclusive_scan(len);
    uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    wpre[lane] = inc - len;
    wlo[lane] = lo;
    __syncwarp();
    for (uint32_t k0 = 0; k0 < tot; k0 += 32) {
      uint32_t k = k0 + lane;
      if (k < tot) {
        uint32_t t = find_seg(wpre, nb, k);
        uint32_t x2 = __ldg(a.nbr + wlo[t] + (k - wpre[t]));
        uint32_t h = (x2 * 0x9E3779B1u) >> hshift;
        for (uint32_t probes = 0;; probes++) {
          if (probes > hmask) __trap();  // table full: cannot happen when w <= HMAX/2
          uint32_t cur = vhk[h];
          if (cur == x2) { atomicAdd(&hv[h], 1u); break; }
          if (cur == EMPTY) {
            uint32_t old = atomicCAS(&hk[h], EMPTY, x2);
            if (old == EMPTY || old == x2) { atomicAdd(&hv[h], 1u); break; }
          }
          h = (h + 1) & hmask;
        }
      }
    }
    __syncwarp();
  }
  // finalize
  uint64_t lsum = 0;
  for (uint32_t i = lane; i < hs; i += 32) {
    uint32_t key = hk[i];
    if (key != EMPTY) {
      uint64_t c = choose2(hv[i]);
      lsum += c;
      if (MODE == MODE_VERTEX && c) red_add_u64(a.bv + key, c);
    }
  }
  lsum = warp_sum(lsum);
  if (lane == 0) {
    tot_acc += lsum;
    if (MODE == MODE_VERTEX && lsum) red_add_u64(a.bv + s, lsum);
  }
  if (MODE == MODE_TOTAL) { __syncwarp(); return; }
  // pass 2 (d <= w <= light_max, so u32 run and segment sums cannot overflow)
  for (uint32_t b = j0; b < j1; b += 32) {
    const uint32_t nb = min(32u, j1 - b);
    uint32_t y = 0, lo = 0, len = 0;
    if (lane < nb) segment<ORIENT>(a, b + lane, y, lo, len);
    uint32_t inc = warp_inclusive_scan(len);
    uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
    wpre[lane] = inc - len;
    wlo[lane] = lo;
    wy[lane] = y;
    wsum[lane] = 0;
    __syncwarp();
    for (uint32_t k0 = 0; k0 < tot; k0 += 32) {
      uint32_t k = k0 + lane;
      bool act = k < tot;
      uint32_t t = EMPTY, c = 0;
      if (act) {
        t = find_seg(wpre, nb, k);
        uint32_t idx = wlo[t] + (k - wpre[t]);
        uint32_t x2 = __ldg(a.nbr + idx);
        uint32_t h = (x2 * 0x9E3779B1u) >> hshift;
        for (uint32_t probes = 0; hk[h] != x2; probes++) {
          if (probes > hmask) __trap();  // key must exist after pass 1
          h = (h + 1) & hmask;
        }
        c = hv[h] - 1u;
        if (MODE == MODE_EDGE && c) red_add_u64(a.acc + idx, c);
      }
      uint64_t rs;
      bool head = run_reduce(t, c, false, &rs);
      if (head && act && rs) atomicAdd(&wsum[t], (uint32_t)rs);
    }
    __syncwarp();
    if (lane < nb && wsum[lane]) {
      if (MODE == MODE_VERTEX) red_add_u64(a.bv + wy[lane], wsum[lane]);
      else red_add_u64(a.acc + b + lane, wsum[lane]);
    }
    __syncwarp();
  }
}

template <int ORIENT, int MODE>
__global__ void __launch_bounds__(BLOCK, 1) k_count(CountArgs a) {
  extern __shared__ __align__(16) char sm[];
  __shared__ uint32_t s_item;
  __shared__ uint32_t s_cnt[2];
  __shared__ uint32_t s_wt[32];
  __shared__ unsigned long long s_tot;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) { s_cnt[0] = 0; s_cnt[1] = 0; s_tot = 0; }
  uint32_t* win = (uint32_t*)(sm + SM_WIN);
  for (uint32_t i = tid; i < WIN; i += BLOCK) win[i] = 0;
  __syncthreads();
  uint64_t tot_acc = 0;
  // heavy starts: dynamic queue over this rank's share (snake order over the
  // wedge-sorted list: round q takes index q*G + (q even ? r : G-1-r))
  const uint32_t G = (uint32_t)a.world, r = (uint32_t)a.rank;
  for (;;) {
    if (tid == 0) s_item = atomicAdd(&a.queue[0], 1u);
    __syncthreads();
    const uint32_t q = s_item;
    __syncthreads();
    const uint64_t idx = (uint64_t)q * G + ((q & 1u) ? (G - 1u - r) : r);
    if (idx >= a.heavy_cnt) break;
    cta_start<ORIENT, MODE>(a, a.heavy[idx], sm, tot_acc, s_cnt, s_wt);
  }
  // light starts: warps grab chunks
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&a.queue[1], LIGHT_CHUNK);
    base = __shfl_sync(0xffffffffu, base, 0) + a.light_lo;
    if (base >= a.light_hi) break;
    uint32_t end = min(base + LIGHT_CHUNK, a.light_hi);
    for (uint32_t i = base; i < end; i++) warp_start<ORIENT, MODE>(a, a.light[i], sm, tot_acc);
  }
  // total
  tot_acc = warp_sum(tot_acc);
  if (lane == 0 && tot_acc) atomicAdd(&s_tot, (unsigned long long)tot_acc);
  __syncthreads();
  if (tid == 0 && s_tot) red_add_u64(a.total, s_tot);
  (void)wid;
}

__global__ void k_unrename(const uint64_t* __restrict__ bv, const uint32_t* __restrict__ rid_of_gid, uint32_t nU,
                           uint64_t n, uint64_t* __restrict__ out_u, uint64_t* __restrict__ out_v) {
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t v = bv[rid_of_gid[z]];
    if (z < nU) out_u[z] = v;
    else out_v[z - nU] = v;
  }
}

__global__ void k_edge_gather(const uint64_t* __restrict__ acc, const uint32_t* __restrict__ su,
                              const uint32_t* __restrict__ sv, uint64_t m, uint64_t* __restrict__ be) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
    be[e] = acc[su[e]] + acc[sv[e]];
}

template <int ORIENT, int MODE>
void launch_count(const CountArgs& a, int grid, cudaStream_t s) {
  auto k = k_count<ORIENT, MODE>;
  CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_TOTAL));
  k<<<grid, BLOCK, SM_TOTAL, s>>>(a);
}

inline unsigned grid_for(size_t n, int sms) {
  size_t g = (n + 255) / 256;
  size_t cap = (size_t)sms * 32;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return (unsigned)g;
}

}  // namespace

// share of the light list for rank r: equal wedge mass (host-side bisection
// over the device prefix would need a sync; the prefix is copied once per plan)
static void light_share(bf_graph* g, int r, int G, uint32_t* lo, uint32_t* hi) {
  if (G <= 1) { *lo = 0; *hi = g->n_light; return; }
  std::vector<uint64_t> pre(g->n_light + 1);
  CUDA_TRY(cudaMemcpyAsync(pre.data(), g->light_wpre.p, pre.size() * 8, cudaMemcpyDeviceToHost, g->stream));
  CUDA_TRY(cudaStreamSynchronize(g->stream));
  uint64_t Wl = pre[g->n_light];
  auto cut = [&](int k) -> uint32_t {
    uint64_t target = (uint64_t)((__uint128_t)Wl * k / G);
    return (uint32_t)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
  };
  *lo = r == 0 ? 0 : cut(r);
  *hi = r == G - 1 ? g->n_light : cut(r + 1);
  if (*hi < *lo) *hi = *lo;
}

bf_status graph_count(bf_graph* g, int mode, uint64_t* out_a, uint64_t* out_b, uint64_t* total) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n, m = g->m, S = 2 * m;
  CUDA_TRY(cudaEventRecord(g->ev[0], s));
  g->bv.ensure((std::max<uint64_t>(n, 1) + 1) * 8);
  g->total.ensure(64);
  g->queue.ensure(64);
  uint64_t* dtot = g->total.as<uint64_t>();
  CUDA_TRY(cudaMemsetAsync(dtot, 0, 8, s));
  if (mode == MODE_VERTEX) CUDA_TRY(cudaMemsetAsync(g->bv.p, 0, (n + 1) * 8, s));
  if (mode == MODE_EDGE) {
    g->acc.ensure(std::max<uint64_t>(S, 1) * 8);
    g->be.ensure((std::max<uint64_t>(m, 1) + 1) * 8);
    CUDA_TRY(cudaMemsetAsync(g->acc.p, 0, std::max<uint64_t>(S, 1) * 8, s));
  }
  // overflow rows (only if some key range exceeds the window)
  uint32_t win = (g->opt.test_flags & BF_FLAG_SMALL_WINDOW) ? 64u : WIN;
  uint64_t maxside = std::max(g->n_u, g->n_v);
  uint64_t olen = maxside > win ? maxside - win : 1;
  int grid = g->sms;
  if (g->orow.bytes < (size_t)grid * olen * 4) {
    g->orow.ensure((size_t)grid * olen * 4);
    g->otouch.ensure((size_t)grid * olen * 4);
    CUDA_TRY(cudaMemsetAsync(g->orow.p, 0, (size_t)grid * olen * 4, s));
  }
  CountArgs a;
  a.off = g->off.as<uint32_t>();
  a.nbr = g->nbr.as<uint32_t>();
  a.pos = g->pos.as<uint32_t>();
  a.hi = g->hi.as<uint32_t>();
  a.wstart = g->wstart.as<uint64_t>();
  a.heavy = g->heavy.as<uint32_t>();
  a.light = g->light.as<uint32_t>();
  a.bv = g->bv.as<uint64_t>();
  a.acc = g->acc.as<uint64_t>();
  a.total = dtot;
  a.orow = g->orow.as<uint32_t>();
  a.otouch = g->otouch.as<uint32_t>();
  a.orow_len = olen;
  a.queue = g->queue.as<uint32_t>();
  a.n_u = g->n_u;
  a.n_v = g->n_v;
  a.heavy_cnt = g->n_heavy;
  a.win = win;
  int V = g->opt.virtual_world > 1 ? g->opt.virtual_world : 1;
  int G = g->opt.world_size > 1 ? g->opt.world_size : V;
  int first = g->opt.world_size > 1 ? g->opt.world_rank : 0;
  int last = g->opt.world_size > 1 ? g->opt.world_rank : V - 1;
  CUDA_TRY(cudaEventRecord(g->ev[1], s));
  for (int r = first; r <= last; r++) {
    a.rank = r;
    a.world = G;
    light_share(g, r, G, &a.light_lo, &a.light_hi);
    CUDA_TRY(cudaMemsetAsync(g->queue.p, 0, 16, s));
    if (g->n_heavy == 0 && a.light_hi <= a.light_lo) continue;
    if (g->orient == BF_ORIENT_LOW) {
      if (mode == MODE_TOTAL) launch_count<BF_ORIENT_LOW, MODE_TOTAL>(a, grid, s);
      else if (mode == MODE_VERTEX) launch_count<BF_ORIENT_LOW, MODE_VERTEX>(a, grid, s);
      else launch_count<BF_ORIENT_LOW, MODE_EDGE>(a, grid, s);
    } else {
      if (mode == MODE_TOTAL) launch_count<BF_ORIENT_HIGH, MODE_TOTAL>(a, grid, s);
      else if (mode == MODE_VERTEX) launch_count<BF_ORIENT_HIGH, MODE_VERTEX>(a, grid, s);
      else launch_count<BF_ORIENT_HIGH, MODE_EDGE>(a, grid, s);
    }
    KERNEL_CHECK(g);
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
      k_edge_gather<<<grid_for(m, g->sms), 256, 0, s>>>(g->acc.as<uint64_t>(), g->slot_u.as<uint32_t>(),
                                                         g->slot_v.as<uint32_t>(), m, g->be.as<uint64_t>());
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
  CUDA_TRY(cudaEventRecord(g->ev[3], s));
  CUDA_TRY(cudaStreamSynchronize(s));
  CUDA_TRY(cudaEventElapsedTime(&g->last_kernel_ms, g->ev[1], g->ev[2]));
  CUDA_TRY(cudaEventElapsedTime(&g->last_call_ms, g->ev[0], g->ev[3]));
  return BF_OK;
}
