// bf_prims.cu -- hand-written device primitives for the CSR builder (layer B0):
// exclusive prefix scan (reduce-then-scan, recursive over tile sums) and a
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
__global__ void __launch_bounds__(SCAN_THREADS) k_tile_reduce(const TI* __restrict__ in, size_t n,
                                                              TO* __restrict__ tile_sums) {
  __shared__ TO wt[32];
  size_t base = (size_t)blockIdx.x * SCAN_TILE;
  TO s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    size_t idx = base + (size_t)i * SCAN_THREADS + threadIdx.x;
    if (idx < n) s += (TO)in[idx];
  }
  TO tot;
  block_exclusive_scan<TO>(s, wt, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
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
  TO* sums = temp;
  TO* rest = temp + tiles + 2;
  k_tile_reduce<TI, TO><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, sums);
  (*launches)++;
  CUDA_TRY(cudaGetLastError());
  scan_impl<TO, TO>(sums, sums, tiles, (TO*)nullptr, rest, s, launches);
  k_tile_scan<TI, TO><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, out, n, sums, total);
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
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * RS_TILE;
  const int w = threadIdx.x >> 5;
  const uint32_t mask = (1u << bits) - 1u;
  K k[RS_ITEMS];
#pragma unroll
  for (int i = 0; i < RS_ITEMS; i++) {
    const size_t idx = base + (size_t)i * RS_THREADS + threadIdx.x;
    k[i] = idx < n ? keys[idx] : (K)0;
  }
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

// the last pass of the slot sort may write the decoded CSR instead of keys and
// values.  A slot's record is either (key, value) with value = slot id, or one
// u64 key | edge id (Be low bits; the slot id is 2e + side) when both fit.
struct RadixDecode {
  uint32_t* nbr;    // nbr[p] = nbr_last - (key & low B bits)
  uint32_t* src;    // src[p] = src_base + (key >> B)
  uint32_t* eid;    // U half: eid[p] = input edge id of the slot at p
  uint32_t* pos;    // V half: twin positions (see below); global CSR positions
  const uint32_t* off;
  uint64_t nbr_last, src_base, pos_base;
  int B, Be, side;
  // U half: also write the V half's input, transposed and reversed -- record
  // m-1-p holds the twin slot (nbr -> src) keyed ((nbr - tbase) << tB | (tbase
  // - 1 - src)) with the U position p as payload ([<< Be | p] or value p), so a
  // stable sort on its high field alone orders the V half (the low field is
  // already descending src).  The V half's last pass then knows both twins'
  // positions p and q: pos[q] = p - off[u] (index of v in N(u)) and pos[p] =
  // q - off[v] (index of u in N(v)) -- Alg. 1's twin indices with no search.
  uint64_t* tkeys;
  uint32_t* tvals;
  uint64_t tm, tbase;
  int tB;
};

#ifndef BF_RS_MINB
#define BF_RS_MINB 4  // measured on c2: 1 -> 4 CTAs per SM takes the rank step 2.62 -> 2.50 ms
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
  for (int i = tid; i < RS_WARPS * 64; i += RS_THREADS) reinterpret_cast<uint4*>(&wcnt[0][0])[i] = make_uint4(0, 0, 0, 0);
  goff[tid] = (uint32_t)tid <= mask ? offs[(size_t)tid * ntiles + blockIdx.x] : 0u;
  __syncthreads();
  const size_t tbase = (size_t)blockIdx.x * RS_TILE;
  K key[RS_ITEMS];
  uint32_t val[RS_ITEMS];
  uint32_t rk[RS_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_ITEMS; r++) {  // all loads in flight before the ranking
    size_t idx = tbase + (size_t)w * RS_WARP_SPAN + r * 32 + lane;
    bool valid = idx < n;
    key[r] = valid ? kin[idx] : (K)0;
    if (VALS) val[r] = valid ? vin[idx] : 0u;
  }
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
  if (dec.nbr) {  // final pass of the slot sort: decode in place of the key/value write
    const uint64_t lmask = (dec.B >= 64) ? ~0ull : ((1ull << dec.B) - 1);
    const uint64_t emask = (1ull << dec.Be) - 1;
    for (uint32_t i = tid; i < cnt; i += RS_THREADS) {
      const uint64_t kr = (uint64_t)skeys[i];
      const uint32_t d = (uint32_t)(kr >> shift) & mask;
      const size_t gp = (uint32_t)(goff[d] + i);
      const uint64_t k = kr >> dec.Be;
      const uint32_t payload = VALS ? svals[i] : (uint32_t)(kr & emask);  // U: edge id; V: U position
      const uint32_t nb = (uint32_t)(dec.nbr_last - (k & lmask)), sr = (uint32_t)(dec.src_base + (k >> dec.B));
      dec.nbr[gp] = nb;
      dec.src[gp] = sr;
      if (dec.tkeys) {  // U half
        dec.eid[gp] = payload;
        const uint64_t tk = ((uint64_t)(nb - dec.tbase) << dec.tB) | (dec.tbase - 1 - sr);
        const size_t tp = dec.tm - 1 - gp;
        if (VALS) {
          dec.tkeys[tp] = tk;
          dec.tvals[tp] = (uint32_t)gp;
        } else {
          dec.tkeys[tp] = (tk << dec.Be) | gp;
        }
      } else {  // V half: q = pos_base + gp, twin at U position payload
        const uint32_t q = (uint32_t)(dec.pos_base + gp);
        dec.pos[q] = payload - __ldg(dec.off + nb);
        dec.pos[payload] = q - __ldg(dec.off + sr);
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
  const RadixDecode none = {nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, 0, 0, 0, 0, nullptr, nullptr, 0, 0, 0};
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
void radix_sort_slots(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, size_t n, int key_bits, int skip_bits,
                      int B, int Be, uint64_t nbr_last, uint64_t src_base, uint64_t pos_base, uint32_t* nbr,
                      uint32_t* src, uint32_t* eid, uint32_t* pos, const uint32_t* off, const SlotTranspose* tr,
                      void* temp, cudaStream_t s, uint64_t* launches) {
  RadixDecode dec = {nbr, src, eid, pos, off, nbr_last, src_base, pos_base, B, Be, tr ? 0 : 1, nullptr, nullptr, 0, 0, 0};
  if (tr) {
    dec.tkeys = tr->keys;
    dec.tvals = tr->vals;
    dec.tm = n;
    dec.tbase = tr->base;
    dec.tB = tr->B;
  }
  if (Be) radix_impl<uint64_t>(k0, nullptr, k1, nullptr, n, Be + skip_bits, Be + key_bits, temp, s, launches, &dec);
  else radix_impl<uint64_t>(k0, v0, k1, v1, n, skip_bits, key_bits, temp, s, launches, &dec);
}
