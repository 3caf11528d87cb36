// bf_build.cu -- ingest (§8(a) a1), ranking (a2), ranked CSR (a3, Alg. 1
// PREPROCESS) and the per-start wedge counts + work plan
// (a4, wedge-aware batching P:473-480).
//
// Rank space ("rid"): U-side vertices occupy rids [0, n_u) in rank order,
// V-side vertices [n_u, n) in rank order.  Same-side rank comparisons are rid
// comparisons; cross-side comparisons use rkey[rid] = (tier << 32) | gid,
// whose order is the ranking's total order (readings Z1-Z4).  Every
// neighbour list N(x) is sorted by decreasing rank (Alg. 1 line 7), i.e. by
// decreasing rid, so deg_x(x) = hi[x] is a prefix length and
// deg_{x1}(y) = pos[x1->y] = index of x1 in N(y) (the twin slot's index).
#include "bf_internal.h"
#include "bf_device.cuh"
#include <algorithm>
#include <cstring>

namespace {

constexpr int TPB = 256;
// hub twin positions (hub_pos): from this many edges on the U half's pos array (4m bytes) no
// longer sits in L2, and the V decode's scatter into it becomes DRAM read-modify-writes
#ifndef BF_HUB_POS_MIN_SLOTS
#define BF_HUB_POS_MIN_SLOTS (1ull << 25)
#endif
constexpr uint64_t kHubPosMinSlots = BF_HUB_POS_MIN_SLOTS;
inline unsigned grid_for(size_t n, int sms) {
  size_t g = (n + TPB - 1) / TPB;
  size_t cap = (size_t)sms * 32;
  if (g > cap) g = cap;
  if (g == 0) g = 1;
  return (unsigned)g;
}

// ---- a1 -----------------------------------------------------------------------
// Degree counting privatises what it can: a side of at most HIST_MAX vertices
// (c4: 30K items with Zipf popularity -- millions of increments on a few
// addresses) is counted in a per-CTA shared-memory histogram and flushed once
// per CTA; the other side's hubs are counted in a per-CTA hot table (below),
// the rest go to one of `stripes` copies of the degree array (chosen by CTA;
// copy 0 is deg itself, summed by k_degree_stripes).
constexpr uint32_t HIST_MAX = 40960;

// The other side's hubs: a per-CTA direct-mapped table of HOT (id, count)
// pairs in shared memory -- an id claims its empty slot at first sight and
// counts there; an id that finds its slot taken by another goes to the
// striped global copy.  Power-law hubs claim their slots early and keep them
// (c2 step -0.06 ms).
constexpr uint32_t HOT = 4096;
constexpr uint32_t HOT_EMPTY = 0xffffffffu;

__device__ __forceinline__ void count_degree(uint32_t* hot_id, uint32_t* hot_cnt, uint32_t* dg, uint32_t z,
                                             bool hot) {
  if (!hot) {
    atomicAdd(dg + z, 1u);
    return;
  }
  const uint32_t h = (z * 0x9E3779B1u) >> 20;  // 12 bits
  uint32_t cur = hot_id[h];
  if (cur == HOT_EMPTY) cur = atomicCAS(hot_id + h, HOT_EMPTY, z);
  if (cur == HOT_EMPTY || cur == z) atomicAdd(hot_cnt + h, 1u);
  else atomicAdd(dg + z, 1u);
}

__global__ void k_validate_degree(const uint32_t* __restrict__ e, uint64_t m, uint32_t nU, uint32_t nV,
                                  uint32_t* __restrict__ deg, uint32_t* __restrict__ flags, int hist_side,
                                  uint32_t stripes, uint64_t n, uint32_t hot_sides) {
  extern __shared__ uint32_t hist[];
  __shared__ uint32_t hot_id[HOT], hot_cnt[HOT];
  const bool hot_u = hot_sides & 1u, hot_v = hot_sides & 2u;
  const uint32_t nh = hist_side == 0 ? nU : hist_side == 1 ? nV : 0u;
  for (uint32_t i = threadIdx.x; i < nh; i += blockDim.x) hist[i] = 0;
  for (uint32_t i = threadIdx.x; i < HOT; i += blockDim.x) { hot_id[i] = HOT_EMPTY; hot_cnt[i] = 0; }
  __syncthreads();
  uint32_t* dg = deg + (size_t)(blockIdx.x % stripes) * n;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint2 uv = reinterpret_cast<const uint2*>(e)[i];
    if (!(uv.x < nU && uv.y < nV)) {
      atomicOr(flags, 1u);
      continue;
    }
    if (hist_side == 0) atomicAdd(&hist[uv.x], 1u);
    else count_degree(hot_id, hot_cnt, dg, uv.x, hot_u);
    if (hist_side == 1) atomicAdd(&hist[uv.y], 1u);
    else count_degree(hot_id, hot_cnt, dg, nU + uv.y, hot_v);
  }
  __syncthreads();
  const uint32_t base = hist_side == 1 ? nU : 0u;
  for (uint32_t i = threadIdx.x; i < nh; i += blockDim.x)
    if (hist[i]) atomicAdd(&deg[base + i], hist[i]);
  for (uint32_t i = threadIdx.x; i < HOT; i += blockDim.x)
    if (hot_cnt[i]) atomicAdd(&deg[hot_id[i]], hot_cnt[i]);
}

__global__ void k_degree_stripes(uint32_t* __restrict__ deg, uint64_t n, uint32_t stripes) {
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t d = deg[z];
    for (uint32_t s = 1; s < stripes; s++) d += deg[(size_t)s * n + z];
    deg[z] = d;
  }
}

// ---- a2 -----------------------------------------------------------------------
__global__ void k_side_sums(const uint32_t* __restrict__ deg, uint64_t n, uint32_t nU,
                            unsigned long long* __restrict__ sums /*[2]: wedges with U / V endpoints*/) {
  __shared__ unsigned long long s[2];
  if (threadIdx.x < 2) s[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long a = 0, b = 0;
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = choose2(deg[z]);
    if (z < nU) b += c;  // centred at a U vertex: endpoints in V
    else a += c;         // centred at a V vertex: endpoints in U
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) { atomicAdd(&s[0], a); atomicAdd(&s[1], b); }
  __syncthreads();
  if (threadIdx.x < 2) atomicAdd(&sums[threadIdx.x], s[threadIdx.x]);
}

// sort key = side << tb | tier' with tier' in tb bits ordered as tier within
// a side (degree: dmax - d; approximate degree: 63 - floor(log2 d) or 64; side
// order: none), so the vertex sort runs over tb + 1 bits only
__global__ void k_rank_keys(const uint32_t* __restrict__ deg, uint64_t n, uint32_t nU, int kind, int tb,
                            uint32_t dmax, const unsigned long long* __restrict__ sums,
                            const uint8_t* __restrict__ peel, uint32_t* __restrict__ skey,
                            uint32_t* __restrict__ iota, uint64_t* __restrict__ rkey_gid) {
  int u_first = kind == BF_RANK_SIDE ? (sums[0] <= sums[1]) : 1;
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t d = deg[z];
    uint32_t side = z >= nU;
    uint32_t tier;
    if (kind == BF_RANK_DEGREE) tier = 0x7FFFFFFFu - d;                           // decreasing degree
    else if (kind == BF_RANK_APPROX_DEGREE) tier = d ? 63u - (31u - __clz(d)) : 64u;  // decreasing floor(log2 d)
    else if (kind == BF_RANK_APPROX_CODEGEN) tier = peel[z];                      // peel round
    else tier = (side == 0) == (u_first != 0) ? 0u : 1u;                          // first side, then the other
    const uint32_t tc = kind == BF_RANK_SIDE ? 0u : kind == BF_RANK_DEGREE ? dmax - d : tier;
    skey[z] = (side << tb) | tc;
    iota[z] = (uint32_t)z;
    rkey_gid[z] = ((uint64_t)tier << 32) | z;
  }
}

__global__ void k_rid_maps(const uint32_t* __restrict__ gid_of_rid, uint64_t n, const uint32_t* __restrict__ deg,
                           const uint64_t* __restrict__ rkey_gid, uint32_t* __restrict__ rid_of_gid,
                           uint64_t* __restrict__ rkey, uint32_t* __restrict__ deg_rid) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t gd = gid_of_rid[r];
    rid_of_gid[gd] = (uint32_t)r;
    rkey[r] = rkey_gid[gd];
    deg_rid[r] = deg[gd];
  }
}

// ---- a2: approximate complement degeneracy --------
// Rounds of a parallel peel: round r removes every remaining vertex whose
// floor(log2 of its degree among the remaining vertices) is the current
// maximum (reading Z16), then lowers its remaining neighbours' degrees.  The
// maximum bucket strictly decreases from round to round (all vertices of it
// leave; degrees only fall), so there are at most 33 rounds (buckets 31..0 and
// deg 0).  code = floor(log2 d) + 2 in [1, 33] (d = 0 -> 1); 0 = no vertex left.
constexpr uint8_t PEEL_ALIVE = 0xFF;
constexpr int PEEL_ROUNDS = 33;
__device__ __forceinline__ uint32_t peel_code(uint32_t d) { return d ? 33u - __clz(d) : 1u; }

__global__ void k_peel_max(const uint32_t* __restrict__ cur, const uint8_t* __restrict__ rnd, uint64_t n,
                           uint32_t* __restrict__ code) {
  uint32_t best = 0;
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x)
    if (rnd[z] == PEEL_ALIVE) best = max(best, peel_code(cur[z]));
  best = __reduce_max_sync(0xffffffffu, best);
  if ((threadIdx.x & 31) == 0 && best) atomicMax(code, best);
}

__global__ void k_peel_mark(const uint32_t* __restrict__ cur, uint8_t* __restrict__ rnd, uint64_t n,
                            const uint32_t* __restrict__ code, int r) {
  const uint32_t c = *code;
  if (!c) return;
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x)
    if (rnd[z] == PEEL_ALIVE && peel_code(cur[z]) == c) rnd[z] = (uint8_t)r;
}

// remaining neighbours of this round's vertices lose one degree per edge
// (warp-aggregated: a round often removes many neighbours of one hub)
__device__ __forceinline__ void sub_degree(uint32_t* cur, uint32_t z, bool valid) {
  const uint32_t act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const uint32_t peers = __match_any_sync(act, z);
  if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicSub(&cur[z], (uint32_t)__popc(peers));
}

__global__ void k_peel_edges(const uint32_t* __restrict__ e, uint64_t m, uint32_t nU, uint32_t* __restrict__ cur,
                             const uint8_t* __restrict__ rnd, const uint32_t* __restrict__ code, int r) {
  if (!*code) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); i0 < m; i0 += stride) {
    const uint64_t i = i0 + (threadIdx.x & 31);
    uint32_t gu = 0, gv = 0;
    bool du = false, dv = false;
    if (i < m) {
      const uint2 uv = reinterpret_cast<const uint2*>(e)[i];
      gu = uv.x;
      gv = nU + uv.y;
      const uint8_t ru = rnd[gu], rv = rnd[gv];
      du = ru == (uint8_t)r && rv == PEEL_ALIVE;  // u leaves now, v stays: v loses one
      dv = rv == (uint8_t)r && ru == PEEL_ALIVE;
    }
    sub_degree(cur, gv, du);
    sub_degree(cur, gu, dv);
  }
}

// ---- a2 (auto): the paper's f metric ---------------------------
// W under degree and approximate-degree order without ranking the graph: with
// k_y = #neighbours of y ranked before y, W = sum_y (k_y d_y - k_y (k_y+1)/2)
// (App. B of SURVEY; the same closed form the oracle pins).  One pass over the
// edges decides, per edge, which endpoint is ranked first under each order.
__device__ __forceinline__ uint64_t rank_key(uint32_t d, uint64_t gid, int approx) {
  const uint32_t tier = approx ? (d ? 63u - (31u - __clz(d)) : 64u) : 0x7FFFFFFFu - d;
  return ((uint64_t)tier << 32) | gid;
}

// k_y per candidate order c (0 degree, 1 approximate degree, 2 approximate
// complement degeneracy): k[c*n + y] = #neighbours ranked before y
__global__ void k_auto_k(const uint32_t* __restrict__ e, uint64_t m, uint32_t nU, uint64_t n,
                         const uint32_t* __restrict__ deg, const uint8_t* __restrict__ peel, uint32_t* __restrict__ k) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 uv = reinterpret_cast<const uint2*>(e)[i];
    const uint64_t gu = uv.x, gv = (uint64_t)nU + uv.y;
    const uint32_t du = deg[gu], dv = deg[gv];
    // the endpoint ranked first is the neighbour "ranked before" the other (its centre)
    atomicAdd(&k[rank_key(du, gu, 0) < rank_key(dv, gv, 0) ? gv : gu], 1u);
    atomicAdd(&k[n + (rank_key(du, gu, 1) < rank_key(dv, gv, 1) ? gv : gu)], 1u);
    const uint64_t cu = ((uint64_t)peel[gu] << 32) | gu, cv = ((uint64_t)peel[gv] << 32) | gv;
    atomicAdd(&k[2 * n + (cu < cv ? gv : gu)], 1u);
  }
}

__global__ void k_auto_w(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ k, uint64_t n,
                         unsigned long long* __restrict__ w) {
  __shared__ unsigned long long s[3];
  if (threadIdx.x < 3) s[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long acc[3] = {0, 0, 0};
  for (uint64_t z = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; z < n; z += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t d = deg[z];
#pragma unroll
    for (int c = 0; c < 3; c++) {
      const uint64_t kk = k[c * n + z];
      acc[c] += kk * d - kk * (kk + 1) / 2;
    }
  }
#pragma unroll
  for (int c = 0; c < 3; c++) {
    acc[c] = warp_sum(acc[c]);
    if ((threadIdx.x & 31) == 0) atomicAdd(&s[c], acc[c]);
  }
  __syncthreads();
  if (threadIdx.x < 3) atomicAdd(&w[threadIdx.x], s[threadIdx.x]);
}

// ---- a3 -----------------------------------------------------------------------
// rids are side-major (U in [0, nU), V in [nU, n)), so the U-end slots fill
// the first m CSR positions and the V-end slots the last m.  The U half is one
// sort of m keys (rid(u) << Bv) | (n-1 - rid(v)) -- (src asc, dst rid desc);
// the V half's records are laid out by the U half's last pass (radix_sort_slots_u).
__global__ void k_slot_keys(const uint32_t* __restrict__ e, uint64_t m, uint32_t nU, uint64_t n, int Bv,
                            const uint32_t* __restrict__ rid_of_gid, uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 uv = reinterpret_cast<const uint2*>(e)[i];
    const uint64_t ru = rid_of_gid[uv.x], rv = rid_of_gid[(uint64_t)nU + uv.y];
    keys[i] = (ru << Bv) | (n - 1 - rv);
  }
}

// hi[x] = deg_x(x) = #neighbours ranked above x: N(x) is one side, whose rid
// order is its rank order, so they are a prefix of the row (decreasing rid);
// binary search for its end
__global__ void k_hi(const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ off,
                     const uint64_t* __restrict__ rkey, uint64_t n, uint32_t* __restrict__ hi) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o = off[x];
    uint32_t lo = 0, up = off[x + 1] - o;
    const uint64_t kx = rkey[x];
    while (lo < up) {
      const uint32_t mid = (lo + up) >> 1;
      if (rkey[nbr[o + mid]] > kx) lo = mid + 1;
      else up = mid;
    }
    hi[x] = lo;
  }
}

// per-slot wedge segment under the orientation (a4): the segment of N(y) that
// slot (x -> y) retrieves, as (first index in nbr, length)
// also rejects repeated edges (reading Z8): a repeated (u,v) pair is two
// adjacent equal slots of the ranked U half
__global__ void k_wslot(const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ src,
                        const uint32_t* __restrict__ pos, const uint32_t* __restrict__ off,
                        const uint32_t* __restrict__ hi, uint64_t S, int orient, uint32_t* __restrict__ seglo,
                        uint32_t* __restrict__ seglen, uint32_t* __restrict__ flags) {
  bool dup = false;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < S; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = src[j], y = nbr[j];
    if (j + 1 < S / 2 && nbr[j + 1] == y && src[j + 1] == x) dup = true;
    uint32_t lo, len;
    if (orient == BF_ORIENT_LOW) {
      // Alg. 2: slot i < deg_x(x) retrieves N(y)[0 : deg_x(y)), deg_x(y) = pos
      lo = off[y];
      len = (j - off[x] < hi[x]) ? pos[j] : 0u;
    } else {
      // cache-optimised: x is the higher endpoint; y's neighbours ranked below
      // both x and y: N(y)[max(hi[y], pos+1) : deg(y))
      const uint32_t oy = off[y], d = off[y + 1] - oy;
      const uint32_t st = max(hi[y], pos[j] + 1);
      lo = oy + st;
      len = d > st ? d - st : 0u;
    }
    seglo[j] = lo;
    seglen[j] = len;
  }
  if (dup) atomicOr(flags, 2u);
}

__global__ void k_items(const uint32_t* __restrict__ order, uint32_t cnt, const uint32_t* __restrict__ off,
                        const uint32_t* __restrict__ hi, const uint64_t* __restrict__ wstart, int orient,
                        uint4* __restrict__ items) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const uint32_t s = order[i];
    const uint32_t j0 = off[s];
    const uint32_t j1 = orient == BF_ORIENT_LOW ? j0 + hi[s] : off[s + 1];
    const uint64_t w = wstart[s];
    items[i] = make_uint4(s, j0, j1, (uint32_t)(w > 0xFFFFFFFFull ? 0xFFFFFFFFull : w));
  }
}

__global__ void k_wstart(const uint64_t* __restrict__ wpre, const uint32_t* __restrict__ off, uint64_t n,
                         uint64_t* __restrict__ wstart) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x)
    wstart[r] = wpre[off[r + 1]] - wpre[off[r]];
}


// ---- plan -----------------------------------------------------------------------
// Tier of a start s (its wedge count w and slot count): 0 = CTA heavy, 1 = CTA
// medium, 2 = warp.  Sort key: tier, then wedges descending (largest first, an
// LPT order for the dynamic queues).
struct TierRule {
  uint64_t tl, tm;       // warp tier: w <= tl and slots <= ts; medium: w <= tm and slots <= ms
  uint32_t ts, ms;
  int no_warp, all_heavy;
  uint32_t nU;           // side boundary (key range of a start)
};

// 14-bit monotone code of a start's wedge count (a float-like exponent and 9
// mantissa bits): the plan sorts by (tier, code desc) over 16 bits -- two
// radix passes -- which keeps the largest-first (LPT) order up to 1/512
__device__ __forceinline__ uint32_t wedge_code(uint64_t w) {
  if (w < 512) return (uint32_t)w;
  const uint32_t e = 63u - (uint32_t)__clzll(w);  // >= 9
  const uint32_t c = ((e - 8u) << 9) | (uint32_t)((w >> (e - 9u)) & 0x1FFu);
  return c < 0x3FFFu ? c : 0x3FFFu;
}

__global__ void k_order_keys(const uint64_t* __restrict__ wstart, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ hi, int orient, uint64_t n, TierRule tr,
                             uint32_t* __restrict__ nz, uint32_t* __restrict__ key, uint32_t* __restrict__ cnts) {
  for (uint64_t r0 = blockIdx.x * (uint64_t)blockDim.x; r0 < n; r0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = r0 + threadIdx.x;
    const uint64_t w = r < n ? wstart[r] : 0;
    uint32_t tier = 3;
    if (w > 0) {
      const uint32_t slots = orient == BF_ORIENT_LOW ? hi[r] : off[r + 1] - off[r];
      if (tr.all_heavy || w > tr.tm) tier = 0;
      else if (!tr.no_warp && w <= tr.tl && slots <= tr.ts) tier = 2;
      else if (slots <= tr.ms) tier = 1;
      else tier = 0;
    }
    if (r < n) {
      nz[r] = w > 0;
      key[r] = (tier << 14) | (0x3FFFu - wedge_code(w));
    }
    // key range of a heavy start: same-side rids ranked above it (HIGH) or
    // below it (LOW); the heavy tier's per-CTA rows are sized by the maximum
    uint32_t kr = 0;
    if (tier == 0) {
      const uint64_t hi_side = r < tr.nU ? tr.nU : n;
      kr = (uint32_t)(orient == BF_ORIENT_LOW ? hi_side - r - 1 : (r < tr.nU ? r : r - tr.nU));
    }
    const uint32_t a = __popc(__ballot_sync(0xffffffffu, w > 0));
    const uint32_t b = __popc(__ballot_sync(0xffffffffu, tier == 0));
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, tier == 1));
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, kr);
    // the most wedges of a heavy start (the host skips the split plan's
    // readback when no start can exceed the split threshold)
    uint64_t wh = 0;
    if (b) {
      wh = tier == 0 ? w : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wh = max(wh, (uint64_t)__shfl_xor_sync(0xffffffffu, wh, o));
    }
    if ((threadIdx.x & 31) == 0) {
      if (a) atomicAdd(&cnts[0], a);
      if (b) atomicAdd(&cnts[1], b);
      if (c) atomicAdd(&cnts[2], c);
      if (kmax) atomicMax(&cnts[3], kmax);
      if (wh) atomicMax((unsigned long long*)(cnts + 4), (unsigned long long)wh);
    }
  }
}

// piece k of split start i covers slots [b_k, b_{k+1}) with b_k = the first
// slot whose wedge prefix reaches k/n of the start's wedges (binary search)
__global__ void k_pieces(const uint4* __restrict__ split, const uint4* __restrict__ pdesc, uint32_t np,
                         const uint64_t* __restrict__ wpre, uint4* __restrict__ pieces) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
    const uint4 d = pdesc[p];  // {split index, k, n, -}
    const uint4 sp = split[d.x];
    const uint64_t base = wpre[sp.y], w = wpre[sp.z] - base;
    uint32_t b[2];
    for (int e = 0; e < 2; e++) {
      const uint32_t k = d.y + e;
      if (k == 0) { b[e] = sp.y; continue; }
      if (k == d.z) { b[e] = sp.z; continue; }
      const uint64_t target = base + (uint64_t)((unsigned __int128)w * k / d.z);
      uint32_t lo = sp.y, hi = sp.z;  // first j in [lo, hi] with wpre[j] >= target
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (wpre[mid] >= target) hi = mid; else lo = mid + 1;
      }
      b[e] = lo;
    }
    pieces[p] = make_uint4(d.x, b[0], b[1], 0u);
  }
}


__global__ void k_compact2(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ idx,
                           const uint32_t* __restrict__ key, uint64_t n, uint32_t* __restrict__ out_rid,
                           uint32_t* __restrict__ out_key) {
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x)
    if (flag[r]) { out_rid[idx[r]] = (uint32_t)r; out_key[idx[r]] = key[r]; }
}

}  // namespace

static bf_status plan_split(bf_graph* g, uint64_t wmax);

bf_status graph_ingest(bf_graph* g, const uint32_t* edges) {
  cudaStream_t s = g->stream;
  uint64_t m = g->m, n = g->n;
  // degree stripes: as many copies as fit 64 MB (at most 8), none for a tiny graph
  uint32_t stripes = 1;
  while (stripes < 8 && n * 4 * (stripes * 2) <= ((size_t)64 << 20) && m >= ((uint64_t)1 << 20)) stripes *= 2;
  const int hist_side = g->n_v <= HIST_MAX && g->n_v <= g->n_u ? 1 : (g->n_u <= HIST_MAX ? 0 : -1);
  const uint32_t nh = hist_side == 0 ? g->n_u : hist_side == 1 ? g->n_v : 0u;
  g->edges.ensure(std::max<uint64_t>(m, 1) * 8);
  g->deg.ensure(std::max<uint64_t>(n, 1) * 4 * stripes);
  CUDA_TRY(cudaMemsetAsync(g->deg.p, 0, std::max<uint64_t>(n, 1) * 4 * stripes, s));
  if (m) {
    CUDA_TRY(cudaMemcpyAsync(g->edges.p, edges, m * 8,
                             g->opt.edges_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  }
  g->tmp_a.ensure(64);
  uint32_t* flags = g->tmp_a.as<uint32_t>();
  CUDA_TRY(cudaMemsetAsync(flags, 0, 4, s));
  if (m) {
    const size_t smem = (size_t)nh * 4;
    const int threads = 1024;
    CUDA_TRY(cudaFuncSetAttribute(k_validate_degree, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_validate_degree, threads, smem));
    const uint64_t want = (m + threads - 1) / threads;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)g->sms * std::max(per_sm, 1)));
    // hot tables only for a side of average degree >= 8 (hubs likely; c4's 20M users at
    // 7 per user only fill the table with ids seen once: +1 ms)
    const uint32_t hot_sides = (m >= 8ull * g->n_u ? 1u : 0u) | (m >= 8ull * g->n_v ? 2u : 0u);
    k_validate_degree<<<grid, threads, smem, s>>>(g->edges.as<uint32_t>(), m, g->n_u, g->n_v, g->deg.as<uint32_t>(),
                                                  flags, hist_side, stripes, n, hot_sides);
    KERNEL_CHECK(g);
    if (stripes > 1) {
      k_degree_stripes<<<grid_for(n, g->sms), TPB, 0, s>>>(g->deg.as<uint32_t>(), n, stripes);
      KERNEL_CHECK(g);
    }
  }
  uint32_t hflags = 0;
  CUDA_TRY(cudaMemcpyAsync(&hflags, flags, 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (hflags & 1u) { bf_set_error("edge id out of range"); return BF_ERANGE; }
  return BF_OK;
}

// approximate complement degeneracy: g->peel[gid] = removal round (a2)
static void peel_rounds(bf_graph* g) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n, m = g->m, n1 = std::max<uint64_t>(n, 1);
  g->peel.ensure(n1 + 64);
  g->tmp_f.ensure(n1 * 4 + 64);
  g->tmp_b.ensure(256);
  uint32_t* cur = g->tmp_f.as<uint32_t>();
  uint32_t* code = (uint32_t*)(g->tmp_b.as<char>() + 96);  // [PEEL_ROUNDS]
  uint8_t* rnd = g->peel.as<uint8_t>();
  CUDA_TRY(cudaMemsetAsync(rnd, PEEL_ALIVE, n1, s));
  CUDA_TRY(cudaMemsetAsync(code, 0, PEEL_ROUNDS * 4, s));
  if (n) CUDA_TRY(cudaMemcpyAsync(cur, g->deg.p, n * 4, cudaMemcpyDeviceToDevice, s));
  // no host sync: a round with no vertex left (code 0) returns at once
  for (int r = 0; r < PEEL_ROUNDS && n; r++) {
    k_peel_max<<<grid_for(n, g->sms), TPB, 0, s>>>(cur, rnd, n, code + r);
    KERNEL_CHECK(g);
    k_peel_mark<<<grid_for(n, g->sms), TPB, 0, s>>>(cur, rnd, n, code + r, r);
    KERNEL_CHECK(g);
    if (m) {
      k_peel_edges<<<grid_for(m, g->sms), TPB, 0, s>>>(g->edges.as<uint32_t>(), m, g->n_u, cur, rnd, code + r, r);
      KERNEL_CHECK(g);
    }
  }
  g->peel_valid = true;
}

// BF_RANK_AUTO: side order if f = (w_s - w_r) / w_s < 0.1, else the one of
// degree / approximate-degree / approximate complement degeneracy order with
// the fewest wedges
static bf_status rank_auto(bf_graph* g, int* kind) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n, m = g->m, n1 = std::max<uint64_t>(n, 1);
  peel_rounds(g);
  g->tmp_c.ensure(n1 * 12 + 64);
  g->tmp_b.ensure(256);
  uint32_t* k = g->tmp_c.as<uint32_t>();
  unsigned long long* w = g->tmp_b.as<unsigned long long>();  // [0] degree, [1] approx, [2] codegen, [3..4] side sums
  CUDA_TRY(cudaMemsetAsync(k, 0, n1 * 12, s));
  CUDA_TRY(cudaMemsetAsync(w, 0, 40, s));
  if (n) {
    k_side_sums<<<grid_for(n, g->sms), TPB, 0, s>>>(g->deg.as<uint32_t>(), n, g->n_u, w + 3);
    KERNEL_CHECK(g);
  }
  if (m) {
    k_auto_k<<<grid_for(m, g->sms), TPB, 0, s>>>(g->edges.as<uint32_t>(), m, g->n_u, n, g->deg.as<uint32_t>(),
                                                  g->peel.as<uint8_t>(), k);
    KERNEL_CHECK(g);
  }
  if (n) {
    k_auto_w<<<grid_for(n, g->sms), TPB, 0, s>>>(g->deg.as<uint32_t>(), k, n, w);
    KERNEL_CHECK(g);
  }
  unsigned long long h[5];
  CUDA_TRY(cudaMemcpyAsync(h, w, 40, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const uint64_t w_side = std::min<uint64_t>(h[3], h[4]);  // reading Z1: the cheaper side as endpoints
  const uint64_t w_deg = h[0], w_adeg = h[1], w_cg = h[2];
  const uint64_t w_r = std::min(std::min(w_deg, w_adeg), w_cg);
  g->w_auto[0] = w_side;
  g->w_auto[1] = w_adeg;
  g->w_auto[2] = w_deg;
  g->w_auto[3] = w_cg;
  // f < 0.1  <=>  10 (w_s - w_r) < w_s (integer arithmetic; f <= 0 when w_r >= w_s)
  const bool side = w_r >= w_side || (unsigned __int128)10 * (w_side - w_r) < (unsigned __int128)w_side;
  // ties between the other three: degree, then approximate degree, then approximate complement degeneracy
  *kind = side ? BF_RANK_SIDE
               : (w_deg == w_r ? BF_RANK_DEGREE : (w_adeg == w_r ? BF_RANK_APPROX_DEGREE : BF_RANK_APPROX_CODEGEN));
  return BF_OK;
}

bf_status graph_rank(bf_graph* g, int kind) {
  cudaStream_t s = g->stream;
  g->peel_valid = false;
  if (kind == BF_RANK_AUTO) {
    bf_status st = rank_auto(g, &kind);
    if (st != BF_OK) return st;
  } else {
    for (auto& x : g->w_auto) x = 0;
  }
  if (kind == BF_RANK_APPROX_CODEGEN && !g->peel_valid) peel_rounds(g);
  const uint64_t n = g->n, m = g->m, S = 2 * m;
  const uint64_t n1 = std::max<uint64_t>(n, 1), S1 = std::max<uint64_t>(S, 1);
  g->rid_of_gid.ensure(n1 * 4);
  g->gid_of_rid.ensure(n1 * 4);
  g->rkey.ensure(n1 * 8);
  g->off.ensure((n1 + 1) * 4);
  g->hi.ensure(n1 * 4);
  g->wstart.ensure(n1 * 8);
  g->nbr.ensure(S1 * 4);
  g->pos.ensure(S1 * 4);
  // scratch
  size_t big = std::max<size_t>(S1, n1);
  g->tmp_a.ensure(big * 8 + 64);            // keys0 (u64)
  g->tmp_b.ensure(big * 8 + 256);           // keys1 (u64) + small counters
  g->tmp_c.ensure(big * 4 + 64);            // vals0
  g->tmp_d.ensure(big * 4 + 64);            // vals1
  g->tmp_e.ensure((std::max<size_t>(S1 + 1, n1) + 2) * 8 + 64);  // rkey_gid [n] / wpre [S+1]
  g->tmp_f.ensure(big * 4 + 64);            // src / misc
  g->tmp_scan.ensure(std::max(radix_temp_bytes(big), scan_temp_bytes(S1 + 1)) + 1024);
  void* tmp = g->tmp_scan.p;
  uint64_t* L = &g->launches;

  // ---- a2: rank keys, vertex sort -----------------------------------------
  uint32_t* skey0 = g->tmp_c.as<uint32_t>();
  uint32_t* skey1 = g->tmp_d.as<uint32_t>();
  uint32_t* val0 = g->tmp_f.as<uint32_t>();
  uint32_t* val1 = g->gid_of_rid.as<uint32_t>();
  uint64_t* rkey_gid = g->tmp_e.as<uint64_t>();
  unsigned long long* sums = (unsigned long long*)(g->tmp_a.as<char>() + big * 8);  // 16 bytes past keys0
  CUDA_TRY(cudaMemsetAsync(sums, 0, 16, s));
  if (n) {
    k_side_sums<<<grid_for(n, g->sms), TPB, 0, s>>>(g->deg.as<uint32_t>(), n, g->n_u, sums);
    KERNEL_CHECK(g);
  }
  // a vertex's degree is at most the other side's size
  uint32_t dmax = std::max(g->n_u, g->n_v);
  int tb = kind == BF_RANK_SIDE ? 0 : kind == BF_RANK_APPROX_DEGREE ? 7
           : kind == BF_RANK_APPROX_CODEGEN ? 6 : ceil_log2_u64((uint64_t)dmax + 1);
  if (tb > 31) { tb = 31; dmax = 0x7FFFFFFFu; }  // degrees stay below 2^31 (m < 2^31 per vertex)
  if (n) {
    k_rank_keys<<<grid_for(n, g->sms), TPB, 0, s>>>(g->deg.as<uint32_t>(), n, g->n_u, kind, tb, dmax, sums,
                                                     g->peel.as<uint8_t>(), skey0, val0, rkey_gid);
    KERNEL_CHECK(g);
  }
  int which = radix_sort_u32(skey0, val0, skey1, val1, n, 0, tb + 1, tmp, s, L);
  uint32_t* gid_of_rid = which ? val1 : val0;
  if (gid_of_rid != g->gid_of_rid.as<uint32_t>() && n)
    CUDA_TRY(cudaMemcpyAsync(g->gid_of_rid.p, gid_of_rid, n * 4, cudaMemcpyDeviceToDevice, s));
  uint32_t* deg_rid = g->tmp_c.as<uint32_t>();  // skeys no longer needed
  if (n) {
    k_rid_maps<<<grid_for(n, g->sms), TPB, 0, s>>>(g->gid_of_rid.as<uint32_t>(), n, g->deg.as<uint32_t>(), rkey_gid,
                                                    g->rid_of_gid.as<uint32_t>(), g->rkey.as<uint64_t>(), deg_rid);
    KERNEL_CHECK(g);
  }
  // off = exclusive scan of deg_rid; off[n] = 2m
  scan_exclusive_u32(deg_rid, g->off.as<uint32_t>(), n, g->off.as<uint32_t>() + n, tmp, s, L);

  // ---- a3: slots sorted by (rid(src) asc, rid(dst) desc) --------------------
  // side-local key widths: U slots (ru, n-1-rv), V slots (rv-nU, nU-1-ru)
  const int Bu = std::max(1, ceil_log2_u64(std::max<uint64_t>(g->n_u, 1)));
  const int Bv = std::max(1, ceil_log2_u64(std::max<uint64_t>(g->n_v, 1)));
  uint64_t* k0 = g->tmp_a.as<uint64_t>();
  uint64_t* k1 = g->tmp_b.as<uint64_t>();
  g->dflag.ensure(16);
  CUDA_TRY(cudaMemsetAsync(g->dflag.p, 0, 4, s));
  if (m) {
    const int Be = std::max(1, ceil_log2_u64(m));  // bits of a U position
    k_slot_keys<<<grid_for(m, g->sms), TPB, 0, s>>>(g->edges.as<uint32_t>(), m, g->n_u, n, Bv,
                                                     g->rid_of_gid.as<uint32_t>(), k0);
    KERNEL_CHECK(g);
    uint32_t* src = g->tmp_f.as<uint32_t>();
    uint32_t* nbr = g->nbr.as<uint32_t>();
    // U half over Bu + Bv bits; its last pass lays out the V half's records
    // (v field, U position) -- or, in carry form (Bu + 2 Bv <= 64), (v, u, index
    // of v in N(u)) -- already in descending-u order, so the V half sorts over
    // its v field only and its last pass writes both twins' pos (Alg. 1 l.5-6).
    // Every record is one u64 (Bu + Bv <= 64, Bv + Be <= 63).
    const bool carry = Bu + 2 * Bv <= 64 && !(g->opt.test_flags & BF_FLAG_UNPACKED_SORT);
    radix_sort_slots_u(k0, k1, m, Bu, Bv, Be, n, nbr, src, k0 + m, g->n_u, g->off.as<uint32_t>(), carry, tmp, s, L);
    // hub twin positions: when the U half's pos array outgrows L2 (or on BF_FLAG_HUB_POS), the U-side
    // pos of slots that point at hub items is ranked in order instead of scattered by the V decode
    const uint32_t* hub = nullptr;
    if (g->n_v && (m >= kHubPosMinSlots || (g->opt.test_flags & BF_FLAG_HUB_POS))) {
      uint32_t* hb = g->dflag.as<uint32_t>() + 2;
      hub_select(g->off.as<uint32_t>(), g->n_u, n, m, (g->opt.test_flags & BF_FLAG_HUB_POS) != 0, hb, s, L);
      hub_pos(nbr, m, hb, g->off.as<uint32_t>(), g->pos.as<uint32_t>(), tmp, s, L);
      hub = hb;
    }
    radix_sort_slots_v(k0 + m, k1 + m, m, Bu, Bv, Be, g->n_u, nbr + m, src + m, g->pos.as<uint32_t>(),
                       g->off.as<uint32_t>(), src, carry, hub, tmp, s, L);
  }
  if (n) {
    k_hi<<<grid_for(n, g->sms), TPB, 0, s>>>(g->nbr.as<uint32_t>(), g->off.as<uint32_t>(), g->rkey.as<uint64_t>(), n,
                                              g->hi.as<uint32_t>());
    KERNEL_CHECK(g);
  }
  g->rank_kind = kind;
  return BF_OK;
}

// a4: per-slot wedge counts -> prefix -> per-start counts, W; classification
bf_status graph_plan(bf_graph* g) {
  cudaStream_t s = g->stream;
  const uint64_t n = g->n, m = g->m, S = 2 * m;
  const uint64_t n1 = std::max<uint64_t>(n, 1), S1 = std::max<uint64_t>(S, 1);
  void* tmp = g->tmp_scan.p;
  uint64_t* L = &g->launches;
  uint32_t* src = g->tmp_f.as<uint32_t>();  // still holds per-slot src from graph_rank
  g->seglo.ensure(S1 * 4);
  g->seglen.ensure(S1 * 4);
  uint32_t* wslot = g->seglen.as<uint32_t>();
  g->wpre.ensure((S1 + 1) * 8);
  uint64_t* wpre = g->wpre.as<uint64_t>();
  uint64_t* dW = g->tmp_b.as<uint64_t>();
  if (m) {
    k_wslot<<<grid_for(S, g->sms), TPB, 0, s>>>(g->nbr.as<uint32_t>(), src, g->pos.as<uint32_t>(),
                                                 g->off.as<uint32_t>(), g->hi.as<uint32_t>(), S, g->orient,
                                                 g->seglo.as<uint32_t>(), wslot, g->dflag.as<uint32_t>());
    KERNEL_CHECK(g);
  }
  scan_exclusive_u32_u64(wslot, wpre, S, wpre + S, tmp, s, L);
  if (n) {
    k_wstart<<<grid_for(n, g->sms), TPB, 0, s>>>(wpre, g->off.as<uint32_t>(), n, g->wstart.as<uint64_t>());
    KERNEL_CHECK(g);
  }
  CUDA_TRY(cudaMemcpyAsync(dW, wpre + S, 8, cudaMemcpyDeviceToDevice, s));

  // plan: starts with w > 0, sorted by (tier, wedges desc); tiers are
  // consecutive segments: CTA heavy, CTA medium, warp
  TierRule tr;
  tr.tl = g->opt.test_light_max_wedges ? std::min<uint64_t>(g->opt.test_light_max_wedges, BF_WARP_MAX_WEDGES)
                                       : BF_WARP_MAX_WEDGES;
  tr.tm = BF_MEDIUM_MAX_WEDGES;
  tr.ts = BF_WARP_MAX_SLOTS;
  tr.ms = BF_MEDIUM_MAX_SLOTS;
  tr.no_warp = (g->opt.test_flags & BF_FLAG_FORCE_CTA) != 0;
  tr.all_heavy = (g->opt.test_flags & BF_FLAG_FORCE_DENSE) != 0;
  tr.nU = g->n_u;
  if (g->opt.test_flags & BF_FLAG_FORCE_WARP) tr.tm = tr.tl;
  g->t1 = (uint32_t)tr.tl;
  g->t2 = (uint32_t)tr.tm;
  // starts with wedges, sorted by (tier, wedges desc).  (Sorting every vertex
  // instead, to save this sync, cost c4 -- 30K starts among 20M vertices --
  // 2.2 ms.)
  uint32_t* nzf = g->tmp_c.as<uint32_t>();
  uint32_t* key = g->tmp_d.as<uint32_t>();
  uint32_t* idx = (uint32_t*)g->tmp_a.p;
  uint32_t* k0 = (uint32_t*)g->tmp_a.p + n1 + 16;
  uint32_t* v0 = g->tmp_f.as<uint32_t>();  // src no longer needed
  uint32_t* k1 = g->tmp_c.as<uint32_t>();  // reused after compaction
  // [0]=nz [1]=tier 0 [2]=tier 1 [3]=max heavy key range [4..5]=max heavy wedges (u64)
  uint32_t* cnts = (uint32_t*)(g->tmp_b.as<char>() + 64);
  g->order.ensure(n1 * 4);
  CUDA_TRY(cudaMemsetAsync(cnts, 0, 24, s));
  if (n) {
    k_order_keys<<<grid_for(n, g->sms), TPB, 0, s>>>(g->wstart.as<uint64_t>(), g->off.as<uint32_t>(),
                                                      g->hi.as<uint32_t>(), g->orient, n, tr, nzf, key, cnts);
    KERNEL_CHECK(g);
  }
  scan_exclusive_u32(nzf, idx, n, nullptr, tmp, s, L);
  if (n) {
    k_compact2<<<grid_for(n, g->sms), TPB, 0, s>>>(nzf, idx, key, n, v0, k0);
    KERNEL_CHECK(g);
  }
  uint64_t host = 0;
  uint32_t hc[6], hflag = 0;
  CUDA_TRY(cudaMemcpyAsync(&host, dW, 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(hc, cnts, 24, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(&hflag, g->dflag.p, 4, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (hflag & 2u) { bf_set_error("duplicate edge"); return BF_EDUP; }
  g->W = host;
  const uint32_t nnz = hc[0];
  g->n_tier[0] = hc[1];
  g->n_tier[1] = hc[2];
  g->n_tier[2] = nnz - hc[1] - hc[2];
  const int w = radix_sort_u32(k0, v0, k1, g->order.as<uint32_t>(), nnz, 0, 16, tmp, s, L);
  const uint32_t* order = (w || !nnz) ? g->order.as<uint32_t>() : v0;
  g->items.ensure((size_t)std::max<uint32_t>(nnz, 1) * 16);
  if (nnz) {
    k_items<<<grid_for(nnz, g->sms), TPB, 0, s>>>(order, nnz, g->off.as<uint32_t>(), g->hi.as<uint32_t>(),
                                                   g->wstart.as<uint64_t>(), g->orient, g->items.as<uint4>());
    KERNEL_CHECK(g);
  }
  g->heavy_keys = hc[3] + 1;  // key offsets of heavy starts are < this
  uint64_t wmax;
  memcpy(&wmax, hc + 4, 8);
  return plan_split(g, wmax);
}

// Split starts: heavy starts whose wedges exceed the threshold (a share of W
// that one CTA would take much longer than the rest of the kernel to finish)
// are cut into pieces of about threshold/2 wedges.  The heavy tier's items are
// sorted by wedges, so the split starts are its prefix.
static bf_status plan_split(bf_graph* g, uint64_t wmax) {
  cudaStream_t s = g->stream;
  g->n_split = 0;
  g->split_batches.clear();
  const uint64_t tmin = (g->opt.test_flags & BF_FLAG_SMALL_CHUNK) ? 256u : ((uint64_t)1 << 20);
  g->split_threshold = std::max<uint64_t>(tmin, g->W / ((uint64_t)g->sms * 8));
  if (g->opt.test_flags & BF_FLAG_NO_SPLIT) g->split_threshold = ~0ull;
  const uint32_t nh = std::min<uint32_t>(g->n_tier[0], kMaxSplit);
  if (!nh || wmax <= g->split_threshold) return BF_OK;  // no start to split: no readback, no sync
  std::vector<uint4>& it = g->h_items;
  it.resize(nh);
  CUDA_TRY(cudaMemcpyAsync(it.data(), g->items.p, (size_t)nh * 16, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  uint32_t ns = 0;
  while (ns < nh && it[ns].w > g->split_threshold) ns++;
  if (!ns) return BF_OK;
  // key range of each split start (HIGH: same-side rids ranked above s; LOW:
  // ranked below), row offsets, pieces, memory-bounded batches
  // host tables live in the graph: the async uploads below may still read them
  std::vector<uint64_t>& off = g->h_split_off;
  std::vector<uint4>& pdesc = g->h_pdesc;
  off.assign(ns, 0);
  pdesc.clear();
  const uint64_t piece = std::max<uint64_t>(g->split_threshold / 2, 1);
  const uint64_t budget = kSplitRowBudget / 8;  // keys: row + list, 4 B each
  g->split_batches.push_back({0, 0, 0, 0, 0});
  for (uint32_t i = 0; i < ns; i++) {
    const uint32_t sv = it[i].x;
    const bool isU = sv < g->n_u;
    const uint64_t kr = g->orient == BF_ORIENT_HIGH ? (isU ? sv : sv - g->n_u)
                                                    : (isU ? g->n_u - sv - 1 : g->n - sv - 1);
    const uint64_t keys = std::max<uint64_t>(kr, 1);
    auto* b = &g->split_batches.back();
    if (b->s1 > b->s0 && b->keys + keys > budget) {
      g->split_batches.push_back({i, i, (uint32_t)pdesc.size(), (uint32_t)pdesc.size(), 0});
      b = &g->split_batches.back();
    }
    off[i] = b->keys;
    b->keys += keys;
    b->s1 = i + 1;
    const uint32_t np = (uint32_t)std::min<uint64_t>((it[i].w + piece - 1) / piece, it[i].z - it[i].y);
    for (uint32_t k = 0; k < std::max<uint32_t>(np, 1); k++) pdesc.push_back(make_uint4(i, k, std::max<uint32_t>(np, 1), 0));
    b->p1 = (uint32_t)pdesc.size();
  }
  g->n_split = ns;
  uint64_t maxkeys = 0;
  for (auto& b : g->split_batches) maxkeys = std::max(maxkeys, b.keys);
  const uint32_t npc = (uint32_t)pdesc.size();
  g->split.ensure((size_t)ns * 16);
  g->split_off.ensure((size_t)ns * 8);
  g->split_cnt.ensure((size_t)ns * 4);
  g->pieces.ensure((size_t)npc * 16);
  g->tmp_a.ensure((size_t)npc * 16 + 64);
  CUDA_TRY(cudaMemcpyAsync(g->split.p, it.data(), (size_t)ns * 16, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(g->split_off.p, off.data(), (size_t)ns * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemsetAsync(g->split_cnt.p, 0, (size_t)ns * 4, s));
  CUDA_TRY(cudaMemcpyAsync(g->tmp_a.p, pdesc.data(), (size_t)npc * 16, cudaMemcpyHostToDevice, s));
  k_pieces<<<grid_for(npc, g->sms), TPB, 0, s>>>(g->split.as<uint4>(), g->tmp_a.as<uint4>(), npc,
                                                  g->wpre.as<uint64_t>(), g->pieces.as<uint4>());
  KERNEL_CHECK(g);
  if (g->srow.bytes < maxkeys * 4) {
    g->srow.ensure(maxkeys * 4);
    g->slist.ensure(maxkeys * 4);
    CUDA_TRY(cudaMemsetAsync(g->srow.p, 0, maxkeys * 4, s));
  }
  return BF_OK;
}
