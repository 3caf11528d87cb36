// bf_prims.cu -- hand-written device primitives for the CSR builder (layer B0):
// exclusive prefix scan (one tile: one CTA; else a single pass with decoupled
// look-back) and a
// stable LSD radix sort (<= 8-bit digits: tile histogram -> digit-major scan ->
// stable scatter through shared memory).  Paper: "prefix sum" P:256-262 and
// "parallel integer sort" P:668-677 (§2, §4.1).
#include "bf_internal.h"
#include "bf_device.cuh"

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

size_t scan_levels_elems(size_t n) {
  size_t tot = 0;
  while (n > 1) {
    size_t t = (n + SCAN_TILE - 1) / SCAN_TILE;
    tot += t + 2;
    if (t <= 1) break;
    n = t;
  }
  return tot + 2;
}

template <class TI, class TO>
__global__ void __launch_bounds__(SCAN_THREADS) k_tile_scan(const TI* __restrict__ in, TO* __restrict__ out,
                                                            size_t n, const TO* __restrict__ tile_off,
                                                            TO* __restrict__ total) {
  __shared__ TO buf[SCAN_TILE];
  __shared__ TO wt[32];
  size_t base = (size_t)blockIdx.x * SCAN_TILE;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    size_t idx = base + (size_t)i * SCAN_THREADS + threadIdx.x;
    buf[i * SCAN_THREADS + threadIdx.x] = idx < n ? (TO)in[idx] : (TO)0;
  }
  __syncthreads();
  TO v[SCAN_ITEMS];
  TO s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    v[i] = buf[threadIdx.x * SCAN_ITEMS + i];
    s += v[i];
  }
  TO tot;
  TO ex = block_exclusive_scan<TO>(s, wt, &tot);
  TO off = tile_off ? tile_off[blockIdx.x] : (TO)0;
  ex += off;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    buf[threadIdx.x * SCAN_ITEMS + i] = ex;
    ex += v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    size_t idx = base + (size_t)i * SCAN_THREADS + threadIdx.x;
    if (idx < n) out[idx] = buf[i * SCAN_THREADS + threadIdx.x];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = off + tot;
}

template <class TO>
__global__ void k_set_scalar(TO* p, TO v) { *p = v; }

// Single-pass exclusive scan with decoupled look-back: each CTA takes the next
// tile (an atomic ticket, so every earlier tile is already running), publishes
// its aggregate, sums its predecessors' published values backwards until an
// inclusive prefix, publishes its own inclusive prefix and scans its tile.
// Status words: flag (bits 62-63: 1 aggregate, 2 inclusive prefix) | value
// (< 2^62); the status array and the ticket are zeroed before the launch.
constexpr unsigned long long LB_AGG = 1ull << 62, LB_INC = 2ull << 62, LB_VAL = (1ull << 62) - 1;

template <class TI, class TO>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_lookback(const TI* __restrict__ in, TO* __restrict__ out,
                                                                size_t n, TO* __restrict__ total,
                                                                unsigned long long* __restrict__ status,
                                                                uint32_t* __restrict__ ticket) {
  __shared__ TO buf[SCAN_TILE];
  __shared__ TO wt[32];
  __shared__ uint32_t s_tile;
  __shared__ TO s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const size_t base = (size_t)tile * SCAN_TILE;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const size_t idx = base + (size_t)i * SCAN_THREADS + threadIdx.x;
    buf[i * SCAN_THREADS + threadIdx.x] = idx < n ? (TO)in[idx] : (TO)0;
  }
  __syncthreads();
  TO v[SCAN_ITEMS];
  TO sum = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    v[i] = buf[threadIdx.x * SCAN_ITEMS + i];
    sum += v[i];
  }
  TO agg;
  TO ex = block_exclusive_scan<TO>(sum, wt, &agg);
  if (threadIdx.x < 32) {  // warp 0: publish, look back, publish the inclusive prefix
    const uint32_t lane = threadIdx.x;
    if (tile == 0) {
      if (lane == 0) {
        atomicExch(status, LB_INC | (unsigned long long)agg);
        s_prefix = 0;
      }
    } else {
      if (lane == 0) atomicExch(status + tile, LB_AGG | (unsigned long long)agg);
      unsigned long long prefix = 0;
      int64_t j = (int64_t)tile - 1 - lane;  // this lane's predecessor in the window
      for (;;) {
        unsigned long long w = 0;
        if (j >= 0) {
          do { w = atomicAdd(status + j, 0ull); } while ((w >> 62) == 0);
        } else {
          w = LB_INC;  // before tile 0: an inclusive prefix of 0
        }
        const uint32_t inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
        // lanes up to and including the nearest inclusive predecessor contribute
        const uint32_t upto = inc ? (uint32_t)(__ffs(inc) - 1) : 31u;
        unsigned long long mine = lane <= upto ? (w & LB_VAL) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        prefix += mine;
        if (inc) break;
        j -= 32;
      }
      if (lane == 0) {
        atomicExch(status + tile, LB_INC | ((prefix + (unsigned long long)agg) & LB_VAL));
        s_prefix = (TO)prefix;
      }
    }
  }
  __syncthreads();
  ex += s_prefix;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    buf[threadIdx.x * SCAN_ITEMS + i] = ex;
    ex += v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    const size_t idx = base + (size_t)i * SCAN_THREADS + threadIdx.x;
    if (idx < n) out[idx] = buf[i * SCAN_THREADS + threadIdx.x];
  }
  if (total && (size_t)(tile + 1) * SCAN_TILE >= n && threadIdx.x == 0) *total = s_prefix + agg;
}

template <class TI, class TO>
void scan_impl(const TI* in, TO* out, size_t n, TO* total, TO* temp, cudaStream_t s, uint64_t* launches) {
  if (n == 0) {
    if (total) { k_set_scalar<TO><<<1, 1, 0, s>>>(total, (TO)0); (*launches)++; CUDA_TRY(cudaGetLastError()); }
    return;
  }
  size_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles == 1) {
    k_tile_scan<TI, TO><<<1, SCAN_THREADS, 0, s>>>(in, out, n, nullptr, total);
    (*launches)++;
    CUDA_TRY(cudaGetLastError());
    return;
  }
  // single pass with decoupled look-back: status words + ticket, zeroed here
  unsigned long long* status = (unsigned long long*)temp;
  uint32_t* ticket = (uint32_t*)(status + tiles);
  CUDA_TRY(cudaMemsetAsync(status, 0, tiles * 8 + 8, s));
  k_scan_lookback<TI, TO><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, out, n, total, status, ticket);
  (*launches)++;
  CUDA_TRY(cudaGetLastError());
}

// ---------------------------------------------------------------- radix sort
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef BF_RS_ITEMS
#define BF_RS_ITEMS 8
#endif
constexpr int RS_ITEMS = BF_RS_ITEMS;              // rounds per warp
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;     // 2048 keys per tile
constexpr int RS_WARP_SPAN = 32 * RS_ITEMS;        // keys per warp (contiguous)

// tile digit histogram: all loads first (RS_ITEMS in flight per thread), then
// per-warp shared histograms with plain atomics (digits of sorted-ish keys
// repeat, but a per-warp copy keeps same-address contention within a warp),
// summed per digit at the end.  Digits are `bits` <= 8 wide (the passes of one
// sort share the key's width evenly: a 42-bit key sorts in 6 passes of 7 bits,
// whose longer per-digit runs coalesce the scatter better than 8-bit digits).
template <class K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_upsweep(const K* __restrict__ keys, size_t n, int shift, int bits,
                                                           uint32_t* __restrict__ counts, uint32_t ntiles) {
  __shared__ uint32_t h[RS_WARPS][256];
  const size_t base = (size_t)blockIdx.x * RS_TILE;
  const int w = threadIdx.x >> 5;
  const uint32_t mask = (1u << bits) - 1u;
  K k[RS_ITEMS];
#pragma unroll
  for (int i = 0; i < RS_ITEMS; i++) {  // loads in flight across the counter clear and its barrier
    const size_t idx = base + (size_t)i * RS_THREADS + threadIdx.x;
    k[i] = idx < n ? keys[idx] : (K)0;
  }
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RS_ITEMS; i++) {
    const size_t idx = base + (size_t)i * RS_THREADS + threadIdx.x;
    if (idx < n) atomicAdd(&h[w][(uint32_t)(k[i] >> shift) & mask], 1u);
  }
  __syncthreads();
  if (threadIdx.x <= mask) {
    uint32_t c = 0;
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ww++) c += h[ww][threadIdx.x];
    counts[(size_t)threadIdx.x * ntiles + blockIdx.x] = c;
  }
}

// The last pass of each half of the slot sort writes the decoded CSR instead
// of keys.  U half: records (src - src_base) << B | (nbr_last - nbr); besides
// nbr and src it writes, for the slot at position p, the V half's input record
// at m-1-p: (nbr - tbase) << Be | p -- the twin slot keyed by its source v with
// the U position as payload.  Reversed, the U half runs in descending u, so a
// stable sort of these records on the v field alone orders the V half.  V half:
// records v_local << Be | p; the twin's source u = usrc[p] (the U half's src),
// and knowing both twins' positions p and q it writes pos[q] = p - off[u]
// (index of v in N(u)) and pos[p] = q - off[v] (index of u in N(v)).
// Carry form (Bu + 2 Bv <= 64: c2, c4): the V record is v_local << (Bu + Bv) |
// u << Bv | i with i = the index of v in N(u) (< |V|, so Bv bits), written by
// the U half's decode; the V half's decode then needs no gather of the twin's
// source (u is in the record) and finds the twin at p = off[u] + i, with pos[q]
// = i straight from the record.  (Round 1 form: the gather usrc[p] cost c4's V
// decode most of its 8 ms.)
struct RadixDecode {
  uint32_t* nbr;         // range-local
  uint32_t* src;         // range-local
  uint32_t* pos;         // V half: global
  const uint32_t* off;   // V half (and the U half's decode in carry form)
  const uint32_t* usrc;  // V half: the U half's src (global positions < m; not used in carry form)
  uint64_t* tkeys;       // U half: the V half's input records
  uint64_t nbr_last, src_base, pos_base, tm, tbase;
  int B, Be, side;
  int carry;             // carry form: Bu (> 0), with the U index in B = Bv bits
  const uint32_t* hub;   // V half: {lo, hi} global rids of the hub items whose U-side pos is ranked
                         // in order (hub_pos) instead of scattered here; nullptr = none
};

#ifndef BF_RS_MINB
#define BF_RS_MINB 5  // measured on c2: 1 -> 4 CTAs per SM takes the rank step 2.62 -> 2.50 ms; 5: c4 step -0.4 ms
#endif
template <class K, bool VALS>
__global__ void __launch_bounds__(RS_THREADS, BF_RS_MINB) k_rs_downsweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                             K* __restrict__ kout, uint32_t* __restrict__ vout, size_t n,
                                                             int shift, int bits, const uint32_t* __restrict__ offs,
                                                             uint32_t ntiles, RadixDecode dec) {
  __shared__ K skeys[RS_TILE];
  __shared__ uint32_t svals[VALS ? RS_TILE : 1];
  __shared__ __align__(16) uint32_t wcnt[RS_WARPS][256];
  __shared__ uint32_t goff[256];
  __shared__ uint32_t wt[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t mask = (1u << bits) - 1u;
  const size_t tbase = (size_t)blockIdx.x * RS_TILE;
  K key[RS_ITEMS];
  uint32_t val[RS_ITEMS];
  uint32_t rk[RS_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_ITEMS; r++) {  // all loads in flight before the ranking (and before the
    size_t idx = tbase + (size_t)w * RS_WARP_SPAN + r * 32 + lane;  // digit-offset load and barrier)
    bool valid = idx < n;
    key[r] = valid ? kin[idx] : (K)0;
    if (VALS) val[r] = valid ? vin[idx] : 0u;
  }
  for (int i = tid; i < RS_WARPS * 64; i += RS_THREADS) reinterpret_cast<uint4*>(&wcnt[0][0])[i] = make_uint4(0, 0, 0, 0);
  goff[tid] = (uint32_t)tid <= mask ? offs[(size_t)tid * ntiles + blockIdx.x] : 0u;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; r++) {
    size_t idx = tbase + (size_t)w * RS_WARP_SPAN + r * 32 + lane;
    bool valid = idx < n;
    uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & mask) : 256u;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = valid ? wcnt[w][d] : 0u;
    rk[r] = before + (uint32_t)__popc(peers & ((1u << lane) - 1u));
    __syncwarp();
    if (valid && (peers >> lane) == 1u) wcnt[w][d] = before + (uint32_t)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // thread tid <-> digit tid: exclusive prefix over warps, then over digits
  uint32_t run = 0;
#pragma unroll
  for (int ww = 0; ww < RS_WARPS; ww++) {
    uint32_t c = wcnt[ww][tid];
    wcnt[ww][tid] = run;
    run += c;
  }
  uint32_t tot;
  // fold the digit's tile start into its per-warp bases and its global offset
  // (one shared lookup per key in each of the two scatters; u32 arithmetic
  // wraps back into range since every position is < 2^32)
  const uint32_t ds = block_exclusive_scan<uint32_t>(run, wt, &tot);
#pragma unroll
  for (int ww = 0; ww < RS_WARPS; ww++) wcnt[ww][tid] += ds;
  goff[tid] -= ds;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; r++) {
    size_t idx = tbase + (size_t)w * RS_WARP_SPAN + r * 32 + lane;
    if (idx < n) {
      uint32_t d = (uint32_t)(key[r] >> shift) & mask;
      uint32_t p = wcnt[w][d] + rk[r];
      skeys[p] = key[r];
      if (VALS) svals[p] = val[r];
    }
  }
  __syncthreads();
  uint32_t cnt = (uint32_t)min((size_t)RS_TILE, n - tbase);
  if (!VALS && dec.nbr) {  // final pass of the slot sort: decode in place of the key write
    const uint64_t lmask = (1ull << dec.B) - 1;
    const uint64_t emask = (1ull << dec.Be) - 1;
    const uint32_t hub_lo = dec.hub ? __ldg(dec.hub) : 0u, hub_n = dec.hub ? __ldg(dec.hub + 1) - hub_lo : 0u;
    for (uint32_t i = tid; i < cnt; i += RS_THREADS) {
      const uint64_t kr = (uint64_t)skeys[i];
      const uint32_t d = (uint32_t)(kr >> shift) & mask;
      const size_t gp = (uint32_t)(goff[d] + i);
      if (dec.side == 0) {  // U half
        const uint32_t nb = (uint32_t)(dec.nbr_last - (kr & lmask)), sr = (uint32_t)(dec.src_base + (kr >> dec.B));
        dec.nbr[gp] = nb;
        dec.src[gp] = sr;
        if (dec.carry)  // v, u, index of v in N(u)
          dec.tkeys[dec.tm - 1 - gp] = ((uint64_t)(nb - dec.tbase) << (dec.carry + dec.B)) |
                                       ((uint64_t)sr << dec.B) | (uint32_t)(gp - __ldg(dec.off + sr));
        else
          dec.tkeys[dec.tm - 1 - gp] = ((uint64_t)(nb - dec.tbase) << dec.Be) | gp;
      } else if (dec.carry) {  // V half, carry form: q = pos_base + gp
        const uint32_t i = (uint32_t)(kr & lmask), u = (uint32_t)((kr >> dec.B) & ((1ull << dec.carry) - 1));
        const uint32_t v = (uint32_t)(dec.src_base + (kr >> (dec.carry + dec.B)));
        const uint32_t q = (uint32_t)(dec.pos_base + gp);
        dec.nbr[gp] = u;
        dec.src[gp] = v;
        dec.pos[q] = i;
        if (v - hub_lo >= hub_n) dec.pos[__ldg(dec.off + u) + i] = q - __ldg(dec.off + v);
      } else {  // V half: q = pos_base + gp, twin at U position p
        const uint32_t p = (uint32_t)(kr & emask);
        const uint32_t v = (uint32_t)(dec.src_base + (kr >> dec.Be)), u = __ldg(dec.usrc + p);
        const uint32_t q = (uint32_t)(dec.pos_base + gp);
        dec.nbr[gp] = u;
        dec.src[gp] = v;
        dec.pos[q] = p - __ldg(dec.off + u);
        if (v - hub_lo >= hub_n) dec.pos[p] = q - __ldg(dec.off + v);
      }
    }
    return;
  }
  for (uint32_t i = tid; i < cnt; i += RS_THREADS) {
    K k = skeys[i];
    uint32_t d = (uint32_t)(k >> shift) & mask;
    const size_t gp = (uint32_t)(goff[d] + i);
    kout[gp] = k;
    if (VALS) vout[gp] = svals[i];
  }
}

template <class K>
int radix_impl(K* k0, uint32_t* v0, K* k1, uint32_t* v1, size_t n, int begin_bit, int end_bit, void* temp,
               cudaStream_t s, uint64_t* launches, const RadixDecode* dec = nullptr) {
  if (n == 0 || end_bit <= begin_bit) return 0;
  const int span = end_bit - begin_bit;
  const int passes = (span + 7) / 8;
  const int bits = (span + passes - 1) / passes;
  uint32_t ntiles = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
  size_t ncounts = (size_t)ntiles << bits;
  uint32_t* counts = (uint32_t*)temp;
  uint32_t* stemp = counts + (size_t)ntiles * 256 + 64;
  K* ki = k0; K* ko = k1;
  uint32_t* vi = v0; uint32_t* vo = v1;
  int which = 0;
  const RadixDecode none = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int p = 0, sh = begin_bit; p < passes; p++, sh += bits) {
    RadixDecode d = (dec && p == passes - 1) ? *dec : none;
    k_rs_upsweep<K><<<ntiles, RS_THREADS, 0, s>>>(ki, n, sh, bits, counts, ntiles);
    (*launches)++;
    CUDA_TRY(cudaGetLastError());
    scan_impl<uint32_t, uint32_t>(counts, counts, ncounts, nullptr, stemp, s, launches);
    if (vi) k_rs_downsweep<K, true><<<ntiles, RS_THREADS, 0, s>>>(ki, vi, ko, vo, n, sh, bits, counts, ntiles, d);
    else k_rs_downsweep<K, false><<<ntiles, RS_THREADS, 0, s>>>(ki, nullptr, ko, nullptr, n, sh, bits, counts, ntiles, d);
    (*launches)++;
    CUDA_TRY(cudaGetLastError());
    K* t = ki; ki = ko; ko = t;
    uint32_t* tv = vi; vi = vo; vo = tv;
    which ^= 1;
  }
  return which;
}


// ---- hub twin positions -------------------------------------------------------
// The V half's decode scatters pos[off[u] + i] = index of u in N(v): random
// 4-byte writes over the whole U half (on c4 17 GB of DRAM traffic, 5 ms).  The
// U half runs in ascending u and N(v) in descending u, so the index of u in
// N(v) is deg(v) - 1 - (number of earlier U-half slots with the same v): for
// up to 256 hub items (a contiguous rid range at the heavier end of the V
// side, chosen on the device when it holds >= 1/4 of the slots) it is a
// per-tile histogram, a scan and an in-order rank, all coalesced; the decode
// then skips the scatter for those v.
constexpr uint32_t HUB_BINS = 256;
__global__ void k_hub_select(const uint32_t* __restrict__ off, uint32_t nU, uint64_t n, uint64_t m, int force,
                             uint32_t* __restrict__ hub) {
  const uint64_t nV = n - nU;
  const uint32_t h = (uint32_t)(nV < HUB_BINS ? nV : HUB_BINS);
  const uint64_t lo_sum = (uint64_t)off[nU + h] - off[nU], hi_sum = (uint64_t)off[n] - off[n - h];
  const bool high = hi_sum >= lo_sum;
  const uint64_t sum = high ? hi_sum : lo_sum;
  const bool on = h && (force || sum * 4 >= m);
  hub[0] = on ? (high ? (uint32_t)(n - h) : nU) : 0u;
  hub[1] = on ? hub[0] + h : 0u;
}
__global__ void __launch_bounds__(RS_THREADS) k_hub_hist(const uint32_t* __restrict__ nbr, size_t m,
                                                          const uint32_t* __restrict__ hub,
                                                          uint32_t* __restrict__ counts, uint32_t ntiles) {
  __shared__ uint32_t h[HUB_BINS];
  const uint32_t lo = hub[0], nh = hub[1] - lo;
  if (!nh) return;
  h[threadIdx.x] = 0;
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * RS_TILE;
#pragma unroll
  for (int i = 0; i < RS_ITEMS; i++) {
    const size_t idx = base + (size_t)i * RS_THREADS + threadIdx.x;
    if (idx < m) {
      const uint32_t b = nbr[idx] - lo;
      if (b < nh) atomicAdd(&h[b], 1u);
    }
  }
  __syncthreads();
  counts[(size_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}
__global__ void __launch_bounds__(RS_THREADS) k_hub_rank(const uint32_t* __restrict__ nbr, size_t m,
                                                          const uint32_t* __restrict__ hub,
                                                          const uint32_t* __restrict__ offs, uint32_t ntiles,
                                                          const uint32_t* __restrict__ off,
                                                          uint32_t* __restrict__ pos) {
  __shared__ uint32_t wc[RS_WARPS][HUB_BINS];
  const uint32_t lo = hub[0], nh = hub[1] - lo;
  if (!nh) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const size_t tbase = (size_t)blockIdx.x * RS_TILE;
  uint32_t b[RS_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_ITEMS; r++) {  // warp w: a contiguous span, in slot order
    const size_t idx = tbase + (size_t)w * RS_WARP_SPAN + r * 32 + lane;
    uint32_t x = HUB_BINS;
    if (idx < m) {
      x = nbr[idx] - lo;
      if (x >= nh) x = HUB_BINS;
    }
    b[r] = x;
  }
  for (int i = tid; i < RS_WARPS * (int)HUB_BINS; i += RS_THREADS) (&wc[0][0])[i] = 0;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; r++)
    if (b[r] < HUB_BINS) atomicAdd(&wc[w][b[r]], 1u);
  __syncthreads();
  {  // thread tid <-> bin tid: slots of this bin before the tile, then before each warp
    uint32_t run = offs[(size_t)tid * ntiles + blockIdx.x] - offs[(size_t)tid * ntiles];
#pragma unroll
    for (int ww = 0; ww < RS_WARPS; ww++) {
      const uint32_t c = wc[ww][tid];
      wc[ww][tid] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; r++) {
    const size_t idx = tbase + (size_t)w * RS_WARP_SPAN + r * 32 + lane;
    const uint32_t x = b[r];
    const unsigned peers = __match_any_sync(0xffffffffu, x);
    const bool hubv = x < HUB_BINS;
    const uint32_t before = hubv ? wc[w][x] : 0u;
    __syncwarp();
    if (hubv && (peers >> lane) == 1u) wc[w][x] = before + (uint32_t)__popc(peers);
    __syncwarp();
    if (hubv) {
      const uint32_t v = lo + x;
      const uint32_t rank = before + (uint32_t)__popc(peers & ((1u << lane) - 1u));
      pos[idx] = __ldg(off + v + 1) - __ldg(off + v) - 1u - rank;
    }
  }
}

}  // namespace

size_t scan_temp_bytes(size_t n) { return scan_levels_elems(n) * 8 + 256; }
void scan_exclusive_u32(const uint32_t* in, uint32_t* out, size_t n, uint32_t* total, void* temp, cudaStream_t s,
                        uint64_t* launches) {
  scan_impl<uint32_t, uint32_t>(in, out, n, total, (uint32_t*)temp, s, launches);
}
void scan_exclusive_u64(const uint64_t* in, uint64_t* out, size_t n, uint64_t* total, void* temp, cudaStream_t s,
                        uint64_t* launches) {
  scan_impl<uint64_t, uint64_t>(in, out, n, total, (uint64_t*)temp, s, launches);
}
void scan_exclusive_u32_u64(const uint32_t* in, uint64_t* out, size_t n, uint64_t* total, void* temp,
                            cudaStream_t s, uint64_t* launches) {
  scan_impl<uint32_t, uint64_t>(in, out, n, total, (uint64_t*)temp, s, launches);
}
void hub_select(const uint32_t* off, uint32_t nU, uint64_t n, uint64_t m, bool force, uint32_t* hub, cudaStream_t s,
                uint64_t* launches) {
  k_hub_select<<<1, 1, 0, s>>>(off, nU, n, m, force ? 1 : 0, hub);
  (*launches)++;
  CUDA_TRY(cudaGetLastError());
}
void hub_pos(const uint32_t* nbr, size_t m, const uint32_t* hub, const uint32_t* off, uint32_t* pos, void* temp,
             cudaStream_t s, uint64_t* launches) {
  if (m == 0) return;
  const uint32_t ntiles = (uint32_t)((m + RS_TILE - 1) / RS_TILE);
  uint32_t* counts = (uint32_t*)temp;
  uint32_t* stemp = counts + (size_t)ntiles * 256 + 64;
  k_hub_hist<<<ntiles, RS_THREADS, 0, s>>>(nbr, m, hub, counts, ntiles);
  (*launches)++;
  CUDA_TRY(cudaGetLastError());
  scan_impl<uint32_t, uint32_t>(counts, counts, (size_t)ntiles * HUB_BINS, nullptr, stemp, s, launches);
  k_hub_rank<<<ntiles, RS_THREADS, 0, s>>>(nbr, m, hub, counts, ntiles, off, pos);
  (*launches)++;
  CUDA_TRY(cudaGetLastError());
}
size_t radix_temp_bytes(size_t n) {
  size_t ntiles = (n + RS_TILE - 1) / RS_TILE;
  size_t nc = ntiles * 256;
  return (nc + 64) * 4 + scan_temp_bytes(nc) + 256;
}
int radix_sort_u32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, size_t n, int begin_bit, int end_bit,
                   void* temp, cudaStream_t s, uint64_t* launches) {
  return radix_impl<uint32_t>(k0, v0, k1, v1, n, begin_bit, end_bit, temp, s, launches);
}
int radix_sort_u64(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, size_t n, int begin_bit, int end_bit,
                   void* temp, cudaStream_t s, uint64_t* launches) {
  return radix_impl<uint64_t>(k0, v0, k1, v1, n, begin_bit, end_bit, temp, s, launches);
}
void radix_sort_slots_u(uint64_t* k0, uint64_t* k1, size_t m, int Bu, int Bv, int Be, uint64_t n, uint32_t* nbr,
                        uint32_t* src, uint64_t* vrec, uint64_t nU, const uint32_t* off, bool carry, void* temp,
                        cudaStream_t s, uint64_t* launches) {
  RadixDecode dec = {nbr, src, nullptr, off, nullptr, vrec, n - 1, 0, 0, m, nU, Bv, Be, 0, carry ? Bu : 0, nullptr};
  radix_impl<uint64_t>(k0, nullptr, k1, nullptr, m, 0, Bu + Bv, temp, s, launches, &dec);
}
void radix_sort_slots_v(uint64_t* k0, uint64_t* k1, size_t m, int Bu, int Bv, int Be, uint64_t nU, uint32_t* nbr,
                        uint32_t* src, uint32_t* pos, const uint32_t* off, const uint32_t* usrc, bool carry,
                        const uint32_t* hub, void* temp, cudaStream_t s, uint64_t* launches) {
  if (carry) {  // records v << (Bu + Bv) | u << Bv | i: sort on the v field
    RadixDecode dec = {nbr, src, pos, off, nullptr, nullptr, 0, nU, m, 0, 0, Bv, Be, 1, Bu, hub};
    radix_impl<uint64_t>(k0, nullptr, k1, nullptr, m, Bu + Bv, Bu + 2 * Bv, temp, s, launches, &dec);
    return;
  }
  RadixDecode dec = {nbr, src, pos, off, usrc, nullptr, 0, nU, m, 0, 0, 0, Be, 1, 0, hub};
  radix_impl<uint64_t>(k0, nullptr, k1, nullptr, m, Be, Be + Bv, temp, s, launches, &dec);
}
