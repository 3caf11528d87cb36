// bf_api.cu -- extern "C" entry points of libbf (include/bf.h), argument
// checks, ownership, error plumbing and the run-time NCCL binding.
#include "bf_internal.h"
#include <dlfcn.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <algorithm>
#include <mutex>
#include <new>
#include <vector>

static thread_local char g_err[512] = "";

void bf_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

void DevBuf::ensure(size_t n) {
  if (n <= bytes && p) return;
  if (p) { CUDA_TRY(cudaFreeAsync(p, s)); p = nullptr; bytes = 0; }
  if (pool) CUDA_TRY(cudaMallocFromPoolAsync(&p, n, pool, s));
  else CUDA_TRY(cudaMallocAsync(&p, n, s));
  bytes = n;
}
void DevBuf::release() {
  if (p) cudaFreeAsync(p, s);
  p = nullptr;
  bytes = 0;
}

// Runs f(), mapping CUDA failures to BF_ECUDA (and marking the graph broken).
template <class F>
static bf_status guarded(bf_graph* g, F&& f) {
  try {
    return f();
  } catch (const bf_cuda_error& e) {
    if (g) g->broken = true;
    if (e.err == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      if (g) g->broken = false;  // allocation failure leaves the graph usable
      bf_set_error("out of device memory (%s, line %d)", e.what, e.line);
      return BF_ENOMEM;
    }
    bf_set_error("CUDA error %s in %s (line %d)", cudaGetErrorString(e.err), e.what, e.line);
    return BF_ECUDA;
  } catch (const std::bad_alloc&) {
    bf_set_error("host allocation failed");
    return BF_ENOMEM;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

namespace {
struct DeviceState {
  int graphs = 0;
  cudaMemPool_t pool = nullptr;
};
std::mutex g_dev_mu;
DeviceState g_dev[64];
}  // namespace

cudaMemPool_t device_attach(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceState& d = g_dev[dev & 63];
  if (!d.pool) {
    cudaMemPoolProps props;
    memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CUDA_TRY(cudaMemPoolCreate(&d.pool, &props));
    uint64_t keep = UINT64_MAX;
    CUDA_TRY(cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  d.graphs++;
  return d.pool;
}

void device_detach(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceState& d = g_dev[dev & 63];
  if (d.graphs > 0) d.graphs--;
}

extern "C" {

void bf_options_default(bf_options* opt) {
  if (!opt) return;
  memset(opt, 0, sizeof(*opt));
  opt->device = 0;
  opt->world_size = 1;
  opt->orient = BF_ORIENT_AUTO;
}

const char* bf_status_str(bf_status s) {
  switch (s) {
    case BF_OK: return "BF_OK";
    case BF_EINVAL: return "BF_EINVAL";
    case BF_ERANGE: return "BF_ERANGE";
    case BF_EDUP: return "BF_EDUP";
    case BF_ENOMEM: return "BF_ENOMEM";
    case BF_ECUDA: return "BF_ECUDA";
    case BF_ENCCL: return "BF_ENCCL";
    case BF_ENORANK: return "BF_ENORANK";
    case BF_EOVERFLOW: return "BF_EOVERFLOW";
  }
  return "BF_UNKNOWN";
}

const char* bf_last_error(void) { return g_err; }

void bf_graph_destroy(bf_graph* g) {
  if (!g) return;
  DeviceGuard dg(g->device);
  // stream-ordered frees: the memory returns to the pool when the stream gets
  // there, so a caller's stream needs no sync; a library-owned one is drained
  // before it is destroyed
  g->for_each_buf([](DevBuf& b) { b.release(); });
  if (g->own_stream && g->stream) cudaStreamSynchronize(g->stream);
  for (auto& e : g->ev)
    if (e) cudaEventDestroy(e);
  if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
  if (g->attached) device_detach(g->device);
  delete g;
}

bf_status bf_graph_create(uint32_t n_u, uint32_t n_v, const uint32_t* edges, uint64_t m, const bf_options* opt,
                          bf_graph** out) {
  if (!out) { bf_set_error("out is NULL"); return BF_EINVAL; }
  *out = nullptr;
  if (m && !edges) { bf_set_error("edges is NULL"); return BF_EINVAL; }
  if ((uint64_t)n_u + n_v >= (1ull << 32) - 1) { bf_set_error("n_u + n_v must be < 2^32 - 1"); return BF_EINVAL; }
  if (m >= (1ull << 31)) { bf_set_error("m must be < 2^31"); return BF_EINVAL; }
  bf_options o;
  if (opt) o = *opt; else bf_options_default(&o);
  if (o.world_size < 1 || o.world_rank < 0 || o.world_rank >= o.world_size) {
    bf_set_error("bad world_rank/world_size");
    return BF_EINVAL;
  }
  if (o.world_size > 1 && !o.nccl_comm) { bf_set_error("world_size > 1 needs nccl_comm"); return BF_EINVAL; }
  if (o.orient < 0 || o.orient > 2) { bf_set_error("bad orient"); return BF_EINVAL; }
  bf_graph* g = new (std::nothrow) bf_graph();
  if (!g) return BF_ENOMEM;
  g->opt = o;
  g->device = o.device;
  g->n_u = n_u;
  g->n_v = n_v;
  g->n = (uint64_t)n_u + n_v;
  g->m = m;
  g->orient = o.orient == BF_ORIENT_LOW ? BF_ORIENT_LOW : BF_ORIENT_HIGH;
  DeviceGuard dg(g->device);
  bf_status st = guarded(g, [&]() -> bf_status {
    CUDA_TRY(cudaSetDevice(g->device));
    CUDA_TRY(cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, g->device));
    if (o.stream) {
      g->stream = (cudaStream_t)o.stream;
    } else {
      CUDA_TRY(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
      g->own_stream = true;
    }
    for (auto& e : g->ev) CUDA_TRY(cudaEventCreate(&e));
    cudaMemPool_t pool = device_attach(g->device);
    g->attached = true;
    g->for_each_buf([&](DevBuf& b) { b.s = g->stream; b.pool = pool; });
    NvtxRange r("bf a1 ingest");
    return graph_ingest(g, edges);
  });
  if (st != BF_OK) {
    bf_graph_destroy(g);
    return st;
  }
  *out = g;
  return BF_OK;
}

bf_status bf_rank(bf_graph* g, bf_rank_kind kind) {
  if (!g) { bf_set_error("g is NULL"); return BF_EINVAL; }
  if (g->broken) { bf_set_error("graph unusable after a CUDA/NCCL error"); return BF_ECUDA; }
  if (kind < BF_RANK_SIDE || kind > BF_RANK_APPROX_CODEGEN) { bf_set_error("bad rank kind"); return BF_EINVAL; }
  DeviceGuard dg(g->device);
  g->ranked = false;
  bf_status st = guarded(g, [&]() -> bf_status {
    bf_status s;
    {
      NvtxRange r("bf a2-a3 rank + ranked CSR");
      s = graph_rank(g, kind);
    }
    if (s != BF_OK) return s;
    NvtxRange r("bf a4 wedge prefix + plan");
    return graph_plan(g);
  });
  if (st == BF_OK) g->ranked = true;
  return st;
}

bf_status bf_rank_info(const bf_graph* g, int* kind, uint64_t w[4]) {
  if (!g) { bf_set_error("g is NULL"); return BF_EINVAL; }
  if (!g->ranked) { bf_set_error("bf_rank has not been called"); return BF_ENORANK; }
  if (kind) *kind = g->rank_kind;
  if (w)
    for (int i = 0; i < 4; i++) w[i] = g->w_auto[i];
  return BF_OK;
}

static bf_status count_common(bf_graph* g, int mode, uint64_t* a, uint64_t* b, uint64_t* total) {
  if (!g) { bf_set_error("g is NULL"); return BF_EINVAL; }
  if (g->broken) { bf_set_error("graph unusable after a CUDA/NCCL error"); return BF_ECUDA; }
  if (!g->ranked) { bf_set_error("bf_rank has not been called"); return BF_ENORANK; }
  DeviceGuard dg(g->device);
  return guarded(g, [&]() -> bf_status {
    bf_status s = graph_count(g, mode, a, b, total);
    if (s == BF_ENCCL) g->broken = true;
    return s;
  });
}

bf_status bf_count_total(bf_graph* g, uint64_t* total) {
  if (!total) { bf_set_error("total is NULL"); return BF_EINVAL; }
  return count_common(g, MODE_TOTAL, nullptr, nullptr, total);
}

bf_status bf_count_vertex(bf_graph* g, uint64_t* out_u, uint64_t* out_v, uint64_t* total) {
  if (g && ((g->n_u && !out_u) || (g->n_v && !out_v))) { bf_set_error("output is NULL"); return BF_EINVAL; }
  return count_common(g, MODE_VERTEX, out_u, out_v, total);
}

bf_status bf_count_edge(bf_graph* g, uint64_t* out_e, uint64_t* total) {
  if (g && g->m && !out_e) { bf_set_error("out_e is NULL"); return BF_EINVAL; }
  return count_common(g, MODE_EDGE, out_e, nullptr, total);
}

bf_status bf_wedge_count(const bf_graph* g, uint64_t* w) {
  if (!g || !w) { bf_set_error("NULL argument"); return BF_EINVAL; }
  if (!g->ranked) { bf_set_error("bf_rank has not been called"); return BF_ENORANK; }
  *w = g->W;
  return BF_OK;
}

bf_status bf_last_stats(const bf_graph* g, float* kernel_ms, float* call_ms, uint64_t* pairs) {
  if (!g) return BF_EINVAL;
  if (kernel_ms) *kernel_ms = g->last_kernel_ms;
  if (call_ms) *call_ms = g->last_call_ms;
  if (pairs) *pairs = g->last_pairs;
  return BF_OK;
}

uint64_t bf_launch_count(const bf_graph* g) { return g ? g->launches : 0; }

uint64_t bf_deal_index(uint64_t q, int rank, int world, uint64_t t0, uint64_t t1) {
  if (world < 1 || rank < 0 || rank >= world || t1 < t0) return t1;
  return bf_deal(q, (uint64_t)rank, (uint64_t)world, t0, t1);
}

bf_status bf_release_device_cache(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    bf_set_error("bad device");
    return BF_EINVAL;
  }
  DeviceGuard dg(device);
  cudaSetDevice(device);
  row_pool_free(device);  // takes the pool's lock: never under a running count
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceState& d = g_dev[device & 63];
  if (d.pool) {
    if (cudaDeviceSynchronize() != cudaSuccess || cudaMemPoolTrimTo(d.pool, 0) != cudaSuccess) {
      bf_set_error("CUDA error while trimming the pool");
      return BF_ECUDA;
    }
  }
  return BF_OK;
}

bf_status bf_rank_shares(const bf_graph* g, int world, uint64_t* wedges) {
  if (!g || !wedges || world < 1) { bf_set_error("bad argument"); return BF_EINVAL; }
  if (!g->ranked) { bf_set_error("bf_rank has not been called"); return BF_ENORANK; }
  DeviceGuard dg(g->device);
  bf_graph* gg = const_cast<bf_graph*>(g);
  return guarded(gg, [&]() -> bf_status {
    const uint32_t nnz = g->n_tier[0] + g->n_tier[1] + g->n_tier[2];
    std::vector<uint4> items(nnz);
    std::vector<uint64_t> ws(g->n);
    if (nnz) CUDA_TRY(cudaMemcpyAsync(items.data(), g->items.p, (size_t)nnz * 16, cudaMemcpyDeviceToHost, g->stream));
    if (g->n) CUDA_TRY(cudaMemcpyAsync(ws.data(), g->wstart.p, g->n * 8, cudaMemcpyDeviceToHost, g->stream));
    CUDA_TRY(cudaStreamSynchronize(g->stream));
    for (int r = 0; r < world; r++) wedges[r] = 0;
    // split starts: whole starts, snake order over their index (k_split_walk's split_mine)
    for (uint32_t i = 0; i < g->n_split; i++) {
      const uint32_t q = i / (uint32_t)world, r = i % (uint32_t)world;
      wedges[(q & 1u) ? world - 1 - r : r] += ws[items[i].x];
    }
    // tier segments: the kernels' deal (bf_deal)
    const uint32_t seg[4] = {g->n_split, g->n_tier[0], g->n_tier[0] + g->n_tier[1], nnz};
    for (int t = 0; t < 3; t++)
      for (int r = 0; r < world; r++)
        for (uint64_t q = 0;; q++) {
          const uint64_t i = bf_deal(q, (uint64_t)r, (uint64_t)world, seg[t], seg[t + 1]);
          if (i >= seg[t + 1]) break;
          wedges[r] += ws[items[i].x];
        }
    return BF_OK;
  });
}

bf_status bf_export_csr(const bf_graph* g, uint32_t* rid_of_gid, uint32_t* off, uint32_t* nbr, uint32_t* pos,
                        uint32_t* hi, uint64_t* wstart) {
  if (!g) return BF_EINVAL;
  if (!g->ranked) { bf_set_error("bf_rank has not been called"); return BF_ENORANK; }
  DeviceGuard dg(g->device);
  bf_graph* gg = const_cast<bf_graph*>(g);
  return guarded(gg, [&]() -> bf_status {
    cudaStream_t s = g->stream;
    uint64_t n = g->n, S = 2 * g->m;
    if (rid_of_gid && n) CUDA_TRY(cudaMemcpyAsync(rid_of_gid, g->rid_of_gid.p, n * 4, cudaMemcpyDeviceToHost, s));
    if (off) CUDA_TRY(cudaMemcpyAsync(off, g->off.p, (n + 1) * 4, cudaMemcpyDeviceToHost, s));
    if (nbr && S) CUDA_TRY(cudaMemcpyAsync(nbr, g->nbr.p, S * 4, cudaMemcpyDeviceToHost, s));
    if (pos && S) CUDA_TRY(cudaMemcpyAsync(pos, g->pos.p, S * 4, cudaMemcpyDeviceToHost, s));
    if (hi && n) CUDA_TRY(cudaMemcpyAsync(hi, g->hi.p, n * 4, cudaMemcpyDeviceToHost, s));
    if (wstart && n) CUDA_TRY(cudaMemcpyAsync(wstart, g->wstart.p, n * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return BF_OK;
  });
}

}  // extern "C"

// ------------------------------------------------------------------ NCCL ------
// NCCL is bound at run time so the library has no link-time dependency; when
// torch is loaded first, dlopen("libnccl.so.2") returns the already-loaded copy.
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { bf_set_error("cannot load libnccl.so.2: %s", dlerror()); return false; }
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllReduce;
  if (!g_nccl.ok) bf_set_error("libnccl is missing symbols");
  return g_nccl.ok;
}
bf_status nccl_fail(ncclResult_t r, const char* what) {
  bf_set_error("%s failed: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
  return BF_ENCCL;
}
}  // namespace

bf_status nccl_allreduce_u64(void* comm, uint64_t* buf, size_t count, cudaStream_t s) {
  if (!load_nccl()) return BF_ENCCL;
  ncclResult_t r = g_nccl.AllReduce(buf, buf, count, ncclUint64, ncclSum, (ncclComm_t)comm, s);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  return BF_OK;
}

extern "C" bf_status bf_nccl_unique_id(uint8_t id[128]) {
  if (!id) return BF_EINVAL;
  if (!load_nccl()) return BF_ENCCL;
  ncclUniqueId u;
  ncclResult_t r = g_nccl.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(u) == 128, "ncclUniqueId must be 128 bytes");
  memcpy(id, &u, 128);
  return BF_OK;
}

extern "C" bf_status bf_nccl_comm_create(const uint8_t id[128], int rank, int world, int device, void** comm) {
  if (!id || !comm || world < 1 || rank < 0 || rank >= world) return BF_EINVAL;
  if (!load_nccl()) return BF_ENCCL;
  DeviceGuard dg(device);
  if (cudaSetDevice(device) != cudaSuccess) { bf_set_error("cudaSetDevice failed"); return BF_ECUDA; }
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclComm_t c;
  ncclResult_t r = g_nccl.CommInitRank(&c, world, u, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = (void*)c;
  return BF_OK;
}

extern "C" bf_status bf_nccl_comm_destroy(void* comm) {
  if (!comm) return BF_OK;
  if (!load_nccl()) return BF_ENCCL;
  ncclResult_t r = g_nccl.CommDestroy((ncclComm_t)comm);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return BF_OK;
}
