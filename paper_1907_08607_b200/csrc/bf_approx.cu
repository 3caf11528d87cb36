// bf_approx.cu -- approximate total counting by sparsification (SURVEY 8(f)
// row 3; §4.4, after Sanei-Mehri et al.): a device
// filter over the edge list whose output graph is counted exactly by the same
// path (bf_graph_create ... bf_count_total) and scaled by the caller.
//
//   edge sparsification:    keep edge e iff h(seed, e) < p * 2^64, i.e. each
//                           edge independently with probability p;
//                           estimate T_sparse / p^4.
//   colorful sparsification: colour(z) = h(seed', gid z) mod c, c = ceil(1/p);
//                           keep an edge iff its endpoints share a colour
//                           (P:1470-1479); estimate T_sparse * c^3.
//
// h is splitmix64 of (seed + (x + 1) * golden) -- counter-based, so every
// decision depends only on (seed, index) and any implementation reproduces it.
#include "bf_internal.h"
#include "bf_device.cuh"
#include <math.h>

namespace {

constexpr int TPB = 256;
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t COLOR_SALT = 0xD1B54A32D192ED03ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t h64(uint64_t seed, uint64_t x) { return mix64(seed + (x + 1) * GOLDEN); }

__global__ void k_sparsify_flag(const uint2* __restrict__ e, uint64_t m, uint32_t nU, int method, uint64_t thr,
                                int keep_all, uint32_t colors, uint64_t seed, uint32_t* __restrict__ flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t keep;
    if (method == BF_SPARSIFY_EDGE) {
      keep = keep_all || h64(seed, i) < thr;
    } else {
      const uint2 uv = e[i];
      const uint64_t s2 = seed ^ COLOR_SALT;
      keep = (h64(s2, uv.x) % colors) == (h64(s2, (uint64_t)nU + uv.y) % colors);
    }
    flag[i] = keep;
  }
}

__global__ void k_sparsify_compact(const uint2* __restrict__ e, const uint32_t* __restrict__ flag,
                                   const uint32_t* __restrict__ idx, uint64_t m, uint2* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[idx[i]] = e[i];
}

}  // namespace

extern "C" bf_status bf_sparsify(uint32_t n_u, uint32_t n_v, const uint32_t* edges, uint64_t m, int method, double p,
                                 uint64_t seed, uint32_t* out_edges, uint64_t* out_m, const bf_options* opt) {
  if (!out_m || (m && (!edges || !out_edges))) { bf_set_error("NULL argument"); return BF_EINVAL; }
  if (method != BF_SPARSIFY_EDGE && method != BF_SPARSIFY_COLOR) { bf_set_error("bad method"); return BF_EINVAL; }
  if (!(p > 0.0 && p <= 1.0)) { bf_set_error("p must be in (0, 1]"); return BF_EINVAL; }
  if (m >= (1ull << 31)) { bf_set_error("m must be < 2^31"); return BF_EINVAL; }
  (void)n_v;
  bf_options o;
  if (opt) o = *opt; else bf_options_default(&o);
  int prev = -1;
  cudaGetDevice(&prev);
  cudaStream_t s = (cudaStream_t)o.stream;
  void *d_in = nullptr, *d_flag = nullptr, *d_idx = nullptr, *d_out = nullptr, *d_tmp = nullptr, *d_tot = nullptr;
  bf_status st = BF_OK;
  try {
    CUDA_TRY(cudaSetDevice(o.device));
    int sms = 148;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device));
    const uint64_t m1 = m ? m : 1;
    const uint2* in = (const uint2*)edges;
    if (!o.edges_on_device) {
      CUDA_TRY(cudaMallocAsync(&d_in, m1 * 8, s));
      if (m) CUDA_TRY(cudaMemcpyAsync(d_in, edges, m * 8, cudaMemcpyHostToDevice, s));
      in = (const uint2*)d_in;
    }
    CUDA_TRY(cudaMallocAsync(&d_flag, m1 * 4, s));
    CUDA_TRY(cudaMallocAsync(&d_idx, m1 * 4 + 16, s));
    CUDA_TRY(cudaMallocAsync(&d_tmp, scan_temp_bytes(m1) + 64, s));
    CUDA_TRY(cudaMallocAsync(&d_tot, 16, s));
    uint2* out = (uint2*)out_edges;
    if (!o.outputs_on_device) {
      CUDA_TRY(cudaMallocAsync(&d_out, m1 * 8, s));
      out = (uint2*)d_out;
    }
    // p * 2^64 as an integer threshold; p == 1 keeps everything
    const int keep_all = p >= 1.0;
    const uint64_t thr = keep_all ? ~0ull : (uint64_t)ldexp(p, 64);
    const uint32_t colors = (uint32_t)ceil(1.0 / p);
    unsigned grid = (unsigned)std::min<uint64_t>((m1 + TPB - 1) / TPB, (uint64_t)sms * 32);
    uint64_t launches = 0;
    uint32_t kept = 0;
    if (m) {
      k_sparsify_flag<<<grid, TPB, 0, s>>>(in, m, n_u, method, thr, keep_all, colors, seed, (uint32_t*)d_flag);
      CUDA_TRY(cudaGetLastError());
      scan_exclusive_u32((const uint32_t*)d_flag, (uint32_t*)d_idx, m, (uint32_t*)d_tot, d_tmp, s, &launches);
      k_sparsify_compact<<<grid, TPB, 0, s>>>(in, (const uint32_t*)d_flag, (const uint32_t*)d_idx, m, out);
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaMemcpyAsync(&kept, d_tot, 4, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    if (!o.outputs_on_device && kept)
      CUDA_TRY(cudaMemcpyAsync(out_edges, d_out, (size_t)kept * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *out_m = kept;
  } catch (const bf_cuda_error& e) {
    bf_set_error("CUDA error %s in %s (line %d)", cudaGetErrorString(e.err), e.what, e.line);
    st = e.err == cudaErrorMemoryAllocation ? BF_ENOMEM : BF_ECUDA;
  }
  for (void* q : {d_in, d_flag, d_idx, d_out, d_tmp, d_tot})
    if (q) cudaFreeAsync(q, s);
  cudaStreamSynchronize(s);
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

// Sparsify on the device, count the kept graph exactly through the same path
// (create, rank, count_total; the caller's options, so multi-GPU works), and
// scale into the estimator of P:1462-1479: edge sparsification keeps each edge
// with probability p, so E[T_s] = p^4 T and T_s / p^4 is unbiased; colourful
// sparsification keeps a butterfly iff its four vertices share a colour,
// probability c^-3 with c = ceil(1/p) colours (reading Z15: the paper writes
// "p^3"; c^3 is the unbiased factor when 1/p is not an integer).
extern "C" bf_status bf_approx_total(uint32_t n_u, uint32_t n_v, const uint32_t* edges, uint64_t m, int method,
                                     double p, uint64_t seed, const bf_options* opt, double* estimate,
                                     uint64_t* sparse_total, uint64_t* sparse_m) {
  if (!estimate) { bf_set_error("estimate is NULL"); return BF_EINVAL; }
  bf_options o;
  if (opt) o = *opt; else bf_options_default(&o);
  const uint64_t m1 = m ? m : 1;
  void* d_kept = nullptr;
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(o.device) != cudaSuccess || cudaMalloc(&d_kept, m1 * 8) != cudaSuccess) {
    cudaGetLastError();
    if (prev >= 0) cudaSetDevice(prev);
    bf_set_error("out of device memory");
    return BF_ENOMEM;
  }
  bf_options so = o;
  so.outputs_on_device = 1;  // kept edges stay on the device
  uint64_t km = 0;
  bf_status st = bf_sparsify(n_u, n_v, edges, m, method, p, seed, (uint32_t*)d_kept, &km, &so);
  uint64_t t = 0;
  if (st == BF_OK) {
    bf_options co = o;
    co.edges_on_device = 1;
    co.outputs_on_device = 0;  // the total comes back to the host
    bf_graph* g = nullptr;
    st = bf_graph_create(n_u, n_v, (const uint32_t*)d_kept, km, &co, &g);
    if (st == BF_OK) st = bf_rank(g, BF_RANK_AUTO);
    if (st == BF_OK) st = bf_count_total(g, &t);
    bf_graph_destroy(g);
  }
  cudaFree(d_kept);
  if (prev >= 0) cudaSetDevice(prev);
  if (st != BF_OK) return st;
  if (sparse_total) *sparse_total = t;
  if (sparse_m) *sparse_m = km;
  if (method == BF_SPARSIFY_EDGE) *estimate = (double)t / (p * p * p * p);
  else {
    const double c = ceil(1.0 / p);
    *estimate = (double)t * c * c * c;
  }
  return BF_OK;
}
