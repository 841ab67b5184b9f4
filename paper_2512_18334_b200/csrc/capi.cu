// C-ABI implementation (include/vcgpu.h): device-resident graphs, the root
// reduction + compaction pipeline, the search launcher and the per-node
// kernel surface.  No CPU fallback: every compute entry point needs a device.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unistd.h>
#include <vector>

#include "../../include/vcgpu.h"
#include "host_algos.h"
#include "root_grid.cuh"
#include "search.cuh"
#include "warp_solve.cuh"

using namespace vcg;

namespace vcg {
template <typename T, bool kSmem, int kWW>
__global__ void search_kernel(SearchParams P);
__global__ void drain_kernel(SearchParams P);
__global__ void search_init_kernel(SearchParams P, int root_key, unsigned long long timeout_ns);
}  // namespace vcg

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};  // kernels this library launched
#define COUNT_LAUNCH(k) (g_launches += (k))

extern "C" int64_t vcg_launch_count(void) { return (int64_t)g_launches.load(); }

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(VCG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// The dynamic shared-memory limit is a per-device attribute of a kernel:
// concurrent solves (solve_batch threads) must only ever raise it, or one
// thread's launch can fail after another lowered it.  Keyed by (device, fn)
// so a process driving several GPUs raises it on each.
static int raise_smem_limit(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[{dev, fn}];
  if (bytes > c) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    c = bytes;
  }
  return 0;
}

// Device attributes of the calling thread's current device, cached per
// thread (cudaGetDeviceProperties costs tens of ms per call).
struct DevAttrs {
  int dev = -1, sm_count = 0, smem_optin = 0;
};
static int dev_attrs(DevAttrs** out) {
  static thread_local DevAttrs a;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (a.dev != dev) {
    CK(cudaDeviceGetAttribute(&a.sm_count, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&a.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    a.dev = dev;
  }
  *out = &a;
  return 0;
}

// Process teardown: once vcg_shutdown() ran (the Python binding calls it
// from atexit, after its worker threads are joined) no device memory is
// released any more -- the process exit reclaims it, and no CUDA call is
// made from static / thread-local destructors while runtimes unload.
static std::atomic<bool> g_shutdown{false};
extern "C" void vcg_shutdown(void) {
  if (g_shutdown.exchange(true)) return;
  cudaDeviceSynchronize();
}

extern "C" const char* vcg_last_error(void) { return g_err.c_str(); }
// error reporting for the library's other translation units
int vcg_fail_external(int code, const char* msg) { return fail(code, msg); }
void vcg_note_launch(int k) { g_launches += (unsigned long long)k; }

extern "C" int vcg_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

extern "C" int vcg_get_device(void) {
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess) return -1;
  return d;
}

extern "C" int vcg_set_device(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return fail(VCG_ENODEV, "cudaSetDevice failed");
  return 0;
}

static bool trace_on() {
  static int on = -1;
  if (on < 0) on = getenv("VCG_TRACE") ? 1 : 0;
  return on == 1;
}
struct Tracer {
  const char* what;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), last = t0;
  explicit Tracer(const char* w) : what(w) {}
  void mark(const char* step) {
    if (!trace_on()) return;
    cudaStreamSynchronize(cudaStreamPerThread);
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[vcg %s] %-22s %8.3f ms\n", what, step,
            std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
  }
};

static int need_device() {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess || c == 0) return fail(VCG_ENODEV, "no CUDA device available");
  // keep freed stream-ordered allocations in the device's pool (per-solve
  // graphs are allocated and released every call)
  static thread_local int pooled_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev != pooled_dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pooled_dev = dev;
  }
  return 0;
}

// ------------------------------------------------------------------ graph --

// Device buffer.  Per-call objects (graphs: allocated and released every
// solve) use the stream-ordered allocator on the calling thread's stream --
// cudaFree would synchronise the whole device and serialise concurrent
// solves on other threads (solve_batch).  The long-lived pooled search
// buffers (tens of GB for large graphs, grown rarely) use cudaMalloc, which
// maps large sizes faster.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool stream_ordered = false;
  DevBuf() = default;
  explicit DevBuf(bool so) : stream_ordered(so) {}
  ~DevBuf() { release(); }
  void release() {
    if (!p) return;
    if (g_shutdown.load(std::memory_order_relaxed)) {  // teardown: the exit reclaims it
      p = nullptr;
      bytes = 0;
      return;
    }
    if (stream_ordered) cudaFreeAsync(p, cudaStreamPerThread);
    else cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  int ensure(size_t b) {
    if (b <= bytes && p) return 0;
    release();
    const cudaError_t e = stream_ordered ? cudaMallocAsync(&p, b ? b : 16, cudaStreamPerThread)
                                         : cudaMalloc(&p, b ? b : 16);
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(VCG_ERESOURCE, "device allocation failed");
    }
    bytes = b;
    return 0;
  }
  template <typename U>
  U* as() const {
    return (U*)p;
  }
};

struct SearchCtx {
  DevBuf stacks, qseq, qdata, qctl, reg, ctl, hist, gws, wbits, wcount, bseq, bdata, bctl, sg, arena;
  // root pipeline / compaction / expansion scratch, reused across calls
  // (per-call cudaMalloc/cudaFree of tens of MB costs milliseconds, with outliers)
  DevBuf r_flag, r_ws, r_out, r_ret, r_gctl, r_front, r_fctl, c_newid, c_cnt, c_vmap, c_tmp, x_ws, x_fifo, x_out;
};

struct vcg_graph {
  int64_t n = 0;
  int64_t m2 = 0;  // 2 * edges
  // host view of the CSR (the reference's StaticGraph is host data): owned
  // copies, or the caller's arrays for a borrowed graph
  const int64_t* hoff = nullptr;
  const int32_t* hnbr = nullptr;
  std::vector<int64_t> own_off;
  std::vector<int32_t> own_nbr;
  DevBuf d_off{true};  // int32[n+1]
  DevBuf d_nbr{true};  // int32[2m]
  // a root reduction's output graph: the forced ids of the reduction that
  // made it, kept on the device when the caller did not ask for them
  // (vcg_graph_forced downloads them on demand)
  DevBuf d_forced{true};
  int64_t nforced = -1;
  void adopt_owned() {
    hoff = own_off.data();
    hnbr = own_nbr.data();
  }
};

// search buffers are reused across graphs and solves (grown on demand), one
// set per (host thread, device): the library is built with --default-stream
// per-thread, so calls from different threads run on independent streams
// and may overlap on the device (solve_batch).  Contexts are never freed:
// when a thread exits, its contexts return to a per-device pool (no CUDA
// call from a thread-local destructor) and the next thread reuses them.
static std::mutex g_ctx_mu;
static std::map<int, std::vector<SearchCtx*>>* g_ctx_pool = new std::map<int, std::vector<SearchCtx*>>();

struct CtxHolder {
  std::map<int, SearchCtx*> by_dev;
  ~CtxHolder() {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    for (auto& kv : by_dev) (*g_ctx_pool)[kv.first].push_back(kv.second);
  }
};

static SearchCtx& search_ctx() {
  static thread_local CtxHolder holder;
  int dev = 0;
  cudaGetDevice(&dev);
  SearchCtx*& c = holder.by_dev[dev];
  if (!c) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    auto& pool = (*g_ctx_pool)[dev];
    if (!pool.empty()) {
      c = pool.back();
      pool.pop_back();
    } else {
      c = new SearchCtx();
    }
  }
  return *c;
}

__global__ void k_narrow_offsets(const int64_t* off64, int64_t count, int32_t* off32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    off32[i] = (int32_t)off64[i];
}

// Upload: neighbours straight from the caller's buffer (fast when it is
// pinned), offsets as int64 into a pooled staging buffer and narrowed to
// int32 on the device (no host pass over the offsets).
static int graph_create_impl(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                             bool borrow, vcg_graph** out) {
  if (int r = need_device()) return r;
  if (n < 0 || !offsets || !out) return fail(VCG_EINVAL, "bad arguments");
  int64_t m2 = offsets[n];
  if (m2 >= (int64_t)1 << 31) return fail(VCG_EINVAL, "graph too large for int32 CSR offsets");
  if (m2 && !neighbors) return fail(VCG_EINVAL, "bad arguments");
  auto* g = new vcg_graph();
  g->n = n;
  g->m2 = m2;
  if (borrow) {
    g->hoff = offsets;
    g->hnbr = neighbors;
  } else {
    g->own_off.assign(offsets, offsets + n + 1);
    g->own_nbr.assign(neighbors, neighbors + m2);
    g->adopt_owned();
  }
  DevBuf off64{true};
  if (g->d_off.ensure((n + 1) * 4) || g->d_nbr.ensure(m2 * 4 + 4) || off64.ensure((n + 1) * 8)) {
    delete g;
    return VCG_ERESOURCE;
  }
  cudaMemcpyAsync(off64.p, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, cudaStreamPerThread);
  if (m2)
    cudaMemcpyAsync(g->d_nbr.p, neighbors, m2 * 4, cudaMemcpyHostToDevice, cudaStreamPerThread);
  COUNT_LAUNCH(1);
  k_narrow_offsets<<<(int)std::min<int64_t>((n + 256) / 256, 148 * 8), 256>>>(
      off64.as<int64_t>(), n + 1, g->d_off.as<int32_t>());
  off64.release();  // stream-ordered: freed after the narrowing kernel
  cudaError_t e = cudaStreamSynchronize(cudaStreamPerThread);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    delete g;
    return fail(VCG_ECUDA, cudaGetErrorString(e));
  }
  *out = g;
  return 0;
}

extern "C" int vcg_graph_create(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                                vcg_graph** out) {
  return graph_create_impl(n, offsets, neighbors, false, out);
}

extern "C" int vcg_graph_create_borrowed(int64_t n, const int64_t* offsets,
                                         const int32_t* neighbors, vcg_graph** out) {
  return graph_create_impl(n, offsets, neighbors, true, out);
}

// Host compaction of the survivors (deg > 0) of a graph whose final degree
// array is on the host: same order and relabelling as compact_flagged, one
// upload instead of the device path's scan / count / gather round trips
// (used by the root pipeline for graphs up to kHostCompactMax vertices).
// Larger graphs (and every graph under VCG_DEVICE_COMPACT=1, the parity
// tests' knob) compact on the device.
static constexpr int kHostCompactMax = 1 << 14;

static int compact_host(const vcg_graph* g, const int32_t* deg, vcg_graph** out,
                        std::vector<int64_t>* vmap_host) {
  const int64_t n = g->n;
  std::vector<int32_t> newid((size_t)std::max<int64_t>(n, 1), -1);
  std::vector<int64_t> off(1, 0), vm;
  int64_t nk = 0;
  for (int64_t v = 0; v < n; ++v)
    if (deg[v] > 0) {
      newid[v] = (int32_t)nk++;
      vm.push_back(v);
    }
  std::vector<int32_t> nbr;
  off.reserve(nk + 1);
  for (int64_t v : vm) {
    for (int64_t j = g->hoff[v]; j < g->hoff[v + 1]; ++j) {
      const int32_t x = g->hnbr[j];
      if (deg[x] > 0) nbr.push_back(newid[x]);
    }
    off.push_back((int64_t)nbr.size());
  }
  if (vmap_host) *vmap_host = vm;
  return vcg_graph_create(nk, off.data(), nbr.data(), out);
}

extern "C" int vcg_graph_destroy(vcg_graph* g) {
  delete g;
  return 0;
}
extern "C" int64_t vcg_graph_num_vertices(const vcg_graph* g) { return g ? g->n : -1; }
extern "C" int64_t vcg_graph_num_edges(const vcg_graph* g) { return g ? g->m2 / 2 : -1; }

extern "C" int vcg_graph_download(const vcg_graph* g, int64_t* offsets, int32_t* neighbors) {
  if (!g) return fail(VCG_EINVAL, "null graph");
  // the host mirror is built together with the device CSR (create/compaction)
  std::copy(g->hoff, g->hoff + g->n + 1, offsets);
  std::copy(g->hnbr, g->hnbr + g->m2, neighbors);
  return 0;
}

// ------------------------------------------------------------ compaction --
// graph.py:99 induced_subgraph, on the device: flag -> scan (new ids) ->
// per-vertex surviving-neighbour counts -> scan (offsets) -> gather.

__global__ void k_keep_flags(const int32_t* deg_or_null, const int64_t* keep_list, int64_t nkeep,
                             int n, int32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = deg_or_null ? (deg_or_null[i] > 0) : 0;
  (void)keep_list;
  (void)nkeep;
}

__global__ void k_flag_from_list(const int64_t* keep, int64_t nkeep, int32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nkeep;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[keep[i]] = 1;
}

// one warp per kept vertex: count surviving neighbours
__global__ void k_count_kept(int n, const int32_t* off, const int32_t* nbr, const int32_t* flag,
                             const int32_t* newid, int32_t* vmap, int32_t* cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    if (!flag[v]) continue;
    int c = 0;
    for (int j = off[v] + lane; j < off[v + 1]; j += 32) c += flag[nbr[j]];
    c = vcg::warp_sum(c);
    if (lane == 0) {
      cnt[newid[v]] = c;
      vmap[newid[v]] = (int32_t)v;
    }
  }
}

// one warp per kept vertex: ballot-compact surviving neighbours, relabelled
__global__ void k_gather_kept(int n, const int32_t* off, const int32_t* nbr, const int32_t* flag,
                              const int32_t* newid, const int32_t* noff, int32_t* nnbr) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    if (!flag[v]) continue;
    int at = noff[newid[v]];
    for (int base = off[v]; base < off[v + 1]; base += 32) {
      int j = base + lane;
      int x = -1;
      bool keep = false;
      if (j < off[v + 1]) {
        x = nbr[j];
        keep = flag[x] != 0;
      }
      unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) nnbr[at + __popc(m & ((1u << lane) - 1))] = newid[x];
      at += __popc(m);
    }
  }
}

static int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t count, DevBuf& tmp) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)count);
  if (tmp.ensure(bytes)) return VCG_ERESOURCE;
  COUNT_LAUNCH(2);  // cub single-pass scan: init + scan kernels
  CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, (int)count));
  return 0;
}

// Builds the induced subgraph of the vertices with flag[v] != 0 (device).
static int compact_flagged(const vcg_graph* g, DevBuf& flag, vcg_graph** out,
                           std::vector<int64_t>* vmap_host) {
  const int n = (int)g->n;
  SearchCtx& X = search_ctx();
  DevBuf &newid = X.c_newid, &cnt = X.c_cnt, &vmap = X.c_vmap, &tmp = X.c_tmp;
  if (newid.ensure((size_t)(n + 1) * 4) || cnt.ensure((size_t)(n + 1) * 4) ||
      vmap.ensure((size_t)(n + 1) * 4))
    return VCG_ERESOURCE;
  if (int r = exclusive_scan_i32(flag.as<int32_t>(), newid.as<int32_t>(), n + 1, tmp)) return r;
  int32_t nk = 0;
  CK(cudaMemcpy(&nk, newid.as<int32_t>() + n, 4, cudaMemcpyDeviceToHost));
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>(((int64_t)n * 32 + threads - 1) / threads, 148 * 16);
  CK(cudaMemset(cnt.p, 0, (size_t)(nk + 1) * 4));
  if (n) {
    COUNT_LAUNCH(1);
    k_count_kept<<<blocks > 0 ? blocks : 1, threads>>>(n, g->d_off.as<int32_t>(),
                                                       g->d_nbr.as<int32_t>(), flag.as<int32_t>(),
                                                       newid.as<int32_t>(), vmap.as<int32_t>(),
                                                       cnt.as<int32_t>());
    CK(cudaGetLastError());
  }
  auto* r = new vcg_graph();
  r->n = nk;
  if (r->d_off.ensure((size_t)(nk + 1) * 4)) {
    delete r;
    return VCG_ERESOURCE;
  }
  if (int e = exclusive_scan_i32(cnt.as<int32_t>(), r->d_off.as<int32_t>(), nk + 1, tmp)) {
    delete r;
    return e;
  }
  int32_t m2 = 0;
  CK(cudaMemcpy(&m2, r->d_off.as<int32_t>() + nk, 4, cudaMemcpyDeviceToHost));
  r->m2 = m2;
  if (r->d_nbr.ensure((size_t)m2 * 4 + 4)) {
    delete r;
    return VCG_ERESOURCE;
  }
  if (n && nk) {
    COUNT_LAUNCH(1);
    k_gather_kept<<<blocks > 0 ? blocks : 1, threads>>>(
        n, g->d_off.as<int32_t>(), g->d_nbr.as<int32_t>(), flag.as<int32_t>(),
        newid.as<int32_t>(), r->d_off.as<int32_t>(), r->d_nbr.as<int32_t>());
    CK(cudaGetLastError());
  }
  // host mirror of the compacted CSR (the reference's StaticGraph is host data)
  std::vector<int32_t> off32(nk + 1), vm(nk);
  CK(cudaMemcpy(off32.data(), r->d_off.p, (size_t)(nk + 1) * 4, cudaMemcpyDeviceToHost));
  r->own_off.resize(nk + 1);
  for (int i = 0; i <= nk; ++i) r->own_off[i] = off32[i];
  r->own_nbr.resize(m2);
  if (m2) CK(cudaMemcpy(r->own_nbr.data(), r->d_nbr.p, (size_t)m2 * 4, cudaMemcpyDeviceToHost));
  r->adopt_owned();
  if (nk) CK(cudaMemcpy(vm.data(), vmap.p, (size_t)nk * 4, cudaMemcpyDeviceToHost));
  if (vmap_host) vmap_host->assign(vm.begin(), vm.end());
  *out = r;
  return 0;
}

extern "C" int vcg_induced_subgraph(const vcg_graph* g, const int64_t* keep, int64_t nkeep,
                                    vcg_graph** out) {
  if (!g || (nkeep && !keep)) return fail(VCG_EINVAL, "bad arguments");
  for (int64_t i = 0; i < nkeep; ++i)
    if (keep[i] < 0 || keep[i] >= g->n || (i && keep[i] <= keep[i - 1]))
      return fail(VCG_EINVAL, "keep must be strictly increasing vertex ids in range");
  DevBuf flag, dkeep;
  if (flag.ensure((size_t)(g->n + 1) * 4) || dkeep.ensure((size_t)nkeep * 8 + 8))
    return VCG_ERESOURCE;
  CK(cudaMemset(flag.p, 0, (size_t)(g->n + 1) * 4));
  if (nkeep) {
    CK(cudaMemcpy(dkeep.p, keep, nkeep * 8, cudaMemcpyHostToDevice));
    COUNT_LAUNCH(1);
    k_flag_from_list<<<(int)std::min<int64_t>((nkeep + 255) / 256, 4096), 256>>>(
        dkeep.as<int64_t>(), nkeep, flag.as<int32_t>());
    CK(cudaGetLastError());
  }
  return compact_flagged(g, flag, out, nullptr);
}

extern "C" int vcg_greedy_bound(const vcg_graph* g, int32_t* members, int64_t* size) {
  if (!g || !size) return fail(VCG_EINVAL, "bad arguments");
  *size = greedy_cover_host(g->n, g->hoff, g->hnbr, members);
  return 0;
}

extern "C" int vcg_crown_reduce(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                                uint32_t* deg, int64_t lo, int64_t hi, int32_t* heads,
                                int64_t* nheads, int32_t* indep, int64_t* nindep,
                                int64_t* edges_removed) {
  if (n < 0 || !offsets || !deg || !heads || !nheads || !edges_removed ||
      (n > 0 && offsets[n] > 0 && !neighbors))
    return fail(VCG_EINVAL, "bad arguments");
  if (n > INT32_MAX) return fail(VCG_EINVAL, "more than 2^31-1 vertices");
  lo = std::max<int64_t>(lo, 0);
  hi = std::min<int64_t>(hi, n - 1);
  std::vector<int32_t> d(n);
  for (int64_t v = 0; v < n; ++v) {
    if (deg[v] > (uint32_t)INT32_MAX) return fail(VCG_EINVAL, "degree out of range");
    d[v] = (int32_t)deg[v];
  }
  std::vector<int32_t> h, crown;
  int64_t er = 0;
  crown_reduce_host(n, offsets, neighbors, d.data(), lo, hi, &h, &er, &crown);
  std::copy(h.begin(), h.end(), heads);
  if (indep) std::copy(crown.begin(), crown.end(), indep);
  for (int64_t v = 0; v < n; ++v) deg[v] = (uint32_t)d[v];
  *nheads = (int64_t)h.size();
  if (nindep) *nindep = h.empty() ? 0 : (int64_t)crown.size();
  *edges_removed = er;
  return 0;
}

// ------------------------------------------------------- node workspaces --

template <typename T>
static long long ws_total(int n) {
  return ws_bytes<T>(n);
}

// pure.py:258 bfs_component, one block: the component of a live source in
// the reference's BFS queue order.  Level by level: every unvisited live
// neighbour u of the level is claimed by its first discoverer (the lowest
// queue position, atomicMin on tmin[u]); each level vertex then appends the
// neighbours it won in adjacency order, at offsets from an exclusive scan over
// the level in queue order -- exactly the order the sequential queue builds.
// visited: int32[n] (stamp marks members), queue: int32[n].  Returns
// {size, degree_sum, min_degree, max_degree, min_vertex, max_vertex}.
template <typename T>
__device__ void bfs_component_block(const NodeWs<T>& w, int32_t* visited, int stamp,
                                    int32_t* queue, int src, long long* r) {
  if (threadIdx.x == 0) {
    visited[src] = stamp;
    queue[0] = src;
  }
  __syncthreads();
  int h = 0, t = 1;
  while (h < t) {
    for (int i = h + (int)threadIdx.x; i < t; i += blockDim.x) {
      const int v = queue[i];
      for (int j = w.off[v]; j < w.off[v + 1]; ++j) {
        const int u = w.nbr[j];
        if (w.deg[u] > 0 && visited[u] != stamp) atomicMin(&w.tmin[u], i);
      }
    }
    __syncthreads();
    int b, e;
    my_chunk(h, t - 1, &b, &e);
    int cnt = 0;
    for (int i = b; i < e; ++i) {
      const int v = queue[i];
      for (int j = w.off[v]; j < w.off[v + 1]; ++j) {
        const int u = w.nbr[j];
        cnt += (w.deg[u] > 0 && visited[u] != stamp && w.tmin[u] == i);
      }
    }
    int total;
    int o = t + block_exscan(cnt, w.bs, &total);
    for (int i = b; i < e; ++i) {
      const int v = queue[i];
      for (int j = w.off[v]; j < w.off[v + 1]; ++j) {
        const int u = w.nbr[j];
        if (w.deg[u] > 0 && visited[u] != stamp && w.tmin[u] == i) queue[o++] = u;
      }
    }
    __syncthreads();
    for (int k = t + (int)threadIdx.x; k < t + total; k += blockDim.x) {
      const int u = queue[k];
      visited[u] = stamp;
      w.tmin[u] = kInf;
    }
    __syncthreads();
    h = t;
    t += total;
  }
  int dsum = 0, mn = kInf, mx = 0, vmn = kInf, vmx = -1;
  for (int k = threadIdx.x; k < t; k += blockDim.x) {
    const int x = queue[k], d = w.deg[x];
    dsum += d;
    mn = min(mn, d);
    mx = max(mx, d);
    vmn = min(vmn, x);
    vmx = max(vmx, x);
  }
  int vals[5] = {dsum, mn, mx, vmn, vmx};
  const int op[5] = {0, 1, 2, 1, 2};
  block_reduce<5>(vals, op, w.bs);
  r[0] = t;
  for (int k = 0; k < 5; ++k) r[k + 1] = vals[k];
}

// pure.py:297 next_live_unvisited: first live vertex of [start, hi] without
// the stamp, or -1
template <typename T>
__device__ int next_live_unvisited_block(const NodeWs<T>& w, const int32_t* visited, int stamp,
                                         int start, int hi) {
  int best = kInf;
  for (int v = start + (int)threadIdx.x; v <= hi; v += blockDim.x)
    if (w.deg[v] > 0 && visited[v] != stamp) {
      best = v;
      break;
    }
  best = block_min(best, w.bs);
  return best == kInf ? -1 : best;
}

// pure.py:306 greedy_cover on the device, one block: repeatedly a live vertex
// of maximum degree, lowest index first.  Exact level-order restatement: with
// current maximum degree d, the sequential picks at level d are the
// lexicographically-first maximal independent set of the degree-d vertices
// (taking one lowers its degree-d neighbours below d, nothing rises to d), in
// increasing index order; the MIS is resolved in rounds (a candidate joins
// once every lower-index candidate neighbour is out, leaves once a neighbour
// joined).  Picks appended to out[pos..]; deg destroyed.  Returns {size, pos}.
template <typename T>
__device__ void greedy_cover_block(const NodeWs<T>& w, int lo, int hi, int32_t* out, int pos,
                                   long long* r) {
  int size = 0;
  int* st = w.ic;  // 0 not a candidate, 1 undecided, 2 out, 3 in
  for (int v = threadIdx.x; v < w.n; v += blockDim.x) st[v] = 0;
  __syncthreads();
  while (lo <= hi) {
    int dm = 0;
    for (int v = lo + (int)threadIdx.x; v <= hi; v += blockDim.x) dm = max(dm, (int)w.deg[v]);
    dm = block_max(dm, w.bs);
    if (dm == 0) break;
    for (int v = lo + (int)threadIdx.x; v <= hi; v += blockDim.x) st[v] = w.deg[v] == dm ? 1 : 0;
    __syncthreads();
    while (true) {
      int open = 0;
      for (int v = lo + (int)threadIdx.x; v <= hi; v += blockDim.x) {
        if (st[v] != 1) continue;
        bool out_ = false, wait = false;
        for (int j = w.off[v]; j < w.off[v + 1]; ++j) {
          const int u = w.nbr[j];
          const int su = ((volatile int*)st)[u];
          if (su == 3) out_ = true;
          else if (su == 1 && u < v) wait = true;
        }
        w.ia[v] = out_ ? 2 : wait ? 1 : 3;
        open |= wait && !out_;
      }
      __syncthreads();
      for (int v = lo + (int)threadIdx.x; v <= hi; v += blockDim.x)
        if (st[v] == 1) st[v] = w.ia[v];
      if (!__syncthreads_or(open)) break;
    }
    // the picks in index order, then their removal
    int b, e;
    my_chunk(lo, hi, &b, &e);
    int cnt = 0;
    for (int v = b; v < e; ++v) cnt += st[v] == 3;
    int total;
    int o = pos + block_exscan(cnt, w.bs, &total);
    for (int v = b; v < e; ++v)
      if (st[v] == 3) out[o++] = v;
    __syncthreads();
    for (int k = pos + (int)threadIdx.x; k < pos + total; k += blockDim.x) {
      const int v = out[k];
      for (int j = w.off[v]; j < w.off[v + 1]; ++j) {
        const int u = w.nbr[j];
        if (ldv(w.deg, u) > 0 && st[u] != 3) deg_dec(w.deg, u);
      }
    }
    __syncthreads();
    for (int k = pos + (int)threadIdx.x; k < pos + total; k += blockDim.x) w.deg[out[k]] = 0;
    for (int v = lo + (int)threadIdx.x; v <= hi; v += blockDim.x) st[v] = 0;
    __syncthreads();
    pos += total;
    size += total;
    recompute_bounds(w, &lo, &hi);
  }
  __syncthreads();
  for (int v = threadIdx.x; v < w.n; v += blockDim.x) st[v] = 0;
  r[0] = size;
  r[1] = pos;
}

// single-block kernel running one per-node operation on a global workspace
template <typename T>
__global__ void k_node_op(int op, int n, const int32_t* off, const int32_t* nbr, T* deg_io,
                          char* wsmem, int lo, int hi, int budget, int v, int32_t* out, int pos,
                          long long* ret) {
  __shared__ BlockScratch bs;
  init_block_scratch(&bs);
  NodeWs<T> w = carve_ws<T>(wsmem, n, &bs, off, nbr);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    w.deg[i] = deg_io[i];
    w.tmin[i] = kInf;
    w.flag[i] = 0;
  }
  __syncthreads();
  long long r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (op == 0 || op == 1 || op == 2) {
    PassRet pr = op == 0   ? degree_one_pass(w, lo, hi, out, pos)
                 : op == 1 ? degree_two_triangle_pass(w, lo, hi, out, pos)
                           : high_degree_pass(w, lo, hi, budget, out, pos);
    r[0] = pr.applied;
    r[1] = pr.forced;
    r[2] = pr.edges;
    r[3] = pr.pos;
  } else if (op == 3) {
    FixRet f = reduce_fixpoint(w, lo, hi, budget, out, pos);
    r[0] = f.forced;
    r[1] = f.d1;
    r[2] = f.d2t;
    r[3] = f.hd;
    r[4] = f.edges;
    r[5] = f.lo;
    r[6] = f.hi;
    r[7] = f.pos;
  } else if (op == 4) {
    int l = lo, h = hi;
    recompute_bounds(w, &l, &h);
    r[0] = l;
    r[1] = h;
  } else if (op == 5) {
    r[0] = select_max_degree(w, lo, hi);
  } else if (op == 6) {
    r[0] = count_live(w, lo, hi);
  } else if (op == 7) {
    r[0] = remove_vertex(w, v);
  } else if (op == 8) {
    int removed, edges;
    remove_neighbors(w, v, out, pos, &removed, &edges);
    r[0] = removed;
    r[1] = edges;
    r[2] = pos + removed;
  } else if (op == 9) {
    // component of v among live vertices of [lo, hi]
    int nc = label_components(w, lo, hi);
    (void)nc;
    compress_labels(w, lo, hi);
    int root = w.par[v];
    int size = 0, dsum = 0, mn = kInf, mx = 0, vmn = kInf, vmx = -1;
    for (int x = lo + threadIdx.x; x <= hi; x += blockDim.x) {
      int d = w.deg[x];
      if (d > 0 && w.par[x] == root) {
        ++size;
        dsum += d;
        mn = min(mn, d);
        mx = max(mx, d);
        vmn = min(vmn, x);
        vmx = max(vmx, x);
      }
    }
    size = block_sum(size, w.bs);
    dsum = block_sum(dsum, w.bs);
    mn = block_min(mn, w.bs);
    mx = block_max(mx, w.bs);
    vmn = block_min(vmn, w.bs);
    vmx = block_max(vmx, w.bs);
    r[0] = size;
    r[1] = dsum;
    r[2] = mn;
    r[3] = mx;
    r[4] = vmn;
    r[5] = vmx;
    // members in index order
    if (threadIdx.x == 0) {
      int k = 0;
      for (int x = lo; x <= hi; ++x)
        if (w.deg[x] > 0 && w.par[x] == root) out[k++] = x;
    }
  } else if (op == 10) {
    // out[0, n) = visited (in/out), out[n, 2n) = queue; stamp = budget
    bfs_component_block(w, out, budget, out + n, v, r);
  } else if (op == 11) {
    r[0] = next_live_unvisited_block(w, out, budget, lo, hi);
  } else if (op == 12) {
    greedy_cover_block(w, lo, hi, out, pos, r);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) deg_io[i] = w.deg[i];
  if (threadIdx.x == 0)
    for (int i = 0; i < 8; ++i) ret[i] = r[i];
}

template <typename T>
static int node_op_t(int op, int64_t n, const int64_t* offsets, const int32_t* neighbors,
                     uint32_t* deg, int64_t lo, int64_t hi, int64_t budget, int64_t v,
                     int32_t* out, int64_t pos, int64_t* ret) {
  const int64_t m2 = offsets[n];
  std::vector<int32_t> off32(n + 1);
  for (int64_t i = 0; i <= n; ++i) off32[i] = (int32_t)offsets[i];
  std::vector<T> degt(n > 0 ? n : 1);
  for (int64_t i = 0; i < n; ++i) degt[i] = (T)deg[i];
  const int64_t ocap = 4 * n + 4;
  DevBuf doff, dnbr, ddeg, dws, dout, dret;
  if (doff.ensure((n + 1) * 4) || dnbr.ensure(m2 * 4 + 4) || ddeg.ensure(deg_bytes<T>((int)n) + 16) ||
      dws.ensure(ws_total<T>((int)n)) || dout.ensure(ocap * 4) || dret.ensure(64))
    return VCG_ERESOURCE;
  CK(cudaMemcpy(doff.p, off32.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
  if (m2) CK(cudaMemcpy(dnbr.p, neighbors, m2 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ddeg.p, degt.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dout.p, out, ocap * 4, cudaMemcpyHostToDevice));
  COUNT_LAUNCH(1);
  k_node_op<T><<<1, 128>>>(op, (int)n, doff.as<int32_t>(), dnbr.as<int32_t>(), ddeg.as<T>(),
                           dws.as<char>(), (int)lo, (int)hi, (int)budget, (int)v,
                           dout.as<int32_t>(), (int)pos, dret.as<long long>());
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(cudaStreamPerThread));
  CK(cudaMemcpy(degt.data(), ddeg.p, n * sizeof(T), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; ++i) deg[i] = degt[i];
  CK(cudaMemcpy(out, dout.p, ocap * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ret, dret.p, 64, cudaMemcpyDeviceToHost));
  return 0;
}

extern "C" int vcg_node_op(int op, int width, int64_t n, const int64_t* offsets,
                           const int32_t* neighbors, uint32_t* deg, int64_t lo, int64_t hi,
                           int64_t budget, int64_t v, int32_t* out, int64_t pos, int64_t* ret) {
  if (int r = need_device()) return r;
  if (n <= 0 || op < 0 || op > 12) return fail(VCG_EINVAL, "bad node op arguments");
  if (width == 8) return node_op_t<uint8_t>(op, n, offsets, neighbors, deg, lo, hi, budget, v, out, pos, ret);
  if (width == 16) return node_op_t<uint16_t>(op, n, offsets, neighbors, deg, lo, hi, budget, v, out, pos, ret);
  if (width == 32) return node_op_t<uint32_t>(op, n, offsets, neighbors, deg, lo, hi, budget, v, out, pos, ret);
  return fail(VCG_EINVAL, "width must be 8, 16 or 32");
}

// -------------------------------------------------------- root reduction --

// One block reduces the whole graph to the lightweight-rule fixpoint on a
// global-memory workspace (deg int32).  ret: forced, d1, d2t, hd, edges, lo, hi, pos
__global__ void k_root_fixpoint(int n, const int32_t* off, const int32_t* nbr, char* wsmem,
                                int lo, int hi, int budget, int32_t* out, int pos, long long* ret,
                                int init) {
  __shared__ BlockScratch bs;
  init_block_scratch(&bs);
  NodeWs<uint32_t> w = carve_ws<uint32_t>(wsmem, n, &bs, off, nbr);
  if (init) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      w.deg[i] = (uint32_t)(off[i + 1] - off[i]);
      w.tmin[i] = kInf;
      w.flag[i] = 0;
    }
  }
  __syncthreads();
  FixRet f = reduce_fixpoint(w, lo, hi, budget, out, pos);
  if (threadIdx.x == 0) {
    ret[0] = f.forced;
    ret[1] = f.d1;
    ret[2] = f.d2t;
    ret[3] = f.hd;
    ret[4] = f.edges;
    ret[5] = f.lo;
    ret[6] = f.hi;
    ret[7] = f.pos;
    ret[8] = bs.spec_m;
  }
}

// The same fixpoint with the order-free sweeps of the search (identical
// forced set and rule counts, node_ops.cuh reduce_fixpoint_fast) on a
// workspace in shared memory; the forced vertices are collected from the
// workspace's inclusion bitset (index order).  gdeg: int32 degrees in HBM,
// read (unless init) and written back.
// ret: forced, d1, d2t, hd, edges, lo, hi, ids written, error
__global__ void __launch_bounds__(1024, 1)
    k_root_fixpoint_fast(int n, const int32_t* off, const int32_t* nbr, uint32_t* gdeg, int lo,
                         int hi, int budget, int32_t* out, long long* ret, int init) {
  extern __shared__ __align__(16) unsigned char rsm[];
  __shared__ BlockScratch bs;
  if (threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) bs.rcyc[i] = bs.rcnt[i] = 0;
  init_block_scratch(&bs);
  NodeWs<uint32_t> w = carve_ws<uint32_t>((char*)rsm, n, &bs, off, nbr);
  const int nwords = (n + 31) / 32;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    w.deg[i] = init ? (uint32_t)(off[i + 1] - off[i]) : gdeg[i];
    w.tmin[i] = kInf;
    w.flag[i] = 0;
  }
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
    w.vbits[i] = 0u;
    w.inc[i] = 0u;
  }
  __syncthreads();
  long long maxkey;
  FixRet f = reduce_fixpoint_fast(w, lo, hi, budget, &maxkey);
  for (int i = threadIdx.x; i < n; i += blockDim.x) gdeg[i] = w.deg[i];
  // forced ids in index order: contiguous word chunks, one block scan
  int wb, we;
  my_chunk(0, nwords - 1, &wb, &we);
  int cnt = 0;
  for (int i = wb; i < we; ++i) cnt += __popc(w.inc[i]);
  int tot;
  int at = block_exscan(cnt, w.bs, &tot);
  for (int i = wb; i < we; ++i) {
    unsigned m = w.inc[i];
    while (m) {
      out[at++] = i * 32 + __ffs(m) - 1;
      m &= m - 1;
    }
  }
  if (threadIdx.x == 0) {
    ret[0] = f.forced;
    ret[1] = f.d1;
    ret[2] = f.d2t;
    ret[3] = f.hd;
    ret[4] = f.edges;
    ret[5] = f.lo;
    ret[6] = f.hi;
    ret[7] = tot;
    ret[8] = f.pos < 0 ? 1 : 0;
    ret[9] = bs.spec_m;
    for (int i = 0; i < 4; ++i) {  // sweep profile: scans, degree-one, triangle, high-degree
      ret[10 + i] = (long long)bs.rcnt[i];
      ret[14 + i] = (long long)bs.rcyc[i];
    }
  }
}

__global__ void k_flags_from_deg(const uint32_t* deg, int n, int32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i < n) ? (deg[i] > 0) : 0;
}

static constexpr int kSpecFailed = 1000;  // internal: speculation refuted, rerun

// a pinned host int32 buffer of at least n entries, one per host thread
// (grown on demand, never freed: the process exit reclaims it)
static int pinned_ints(int64_t n, int32_t** out) {
  static thread_local int32_t* buf = nullptr;
  static thread_local int64_t cap = 0;
  if (n > cap) {
    int32_t* p = nullptr;
    if (cudaHostAlloc((void**)&p, (size_t)n * 4, cudaHostAllocDefault) != cudaSuccess)
      return fail(VCG_ERESOURCE, "pinned host allocation failed");
    if (buf) cudaFreeHost(buf);
    buf = p;
    cap = n;
  }
  *out = buf;
  return 0;
}

// the reduction's forced ids stay with its output graph when the caller did
// not take them (forced_out == NULL)
static void attach_forced(vcg_graph* red, DevBuf& facc, int64_t count, const int32_t* forced_out) {
  if (forced_out) return;
  // the device-to-device copies are complete before another host thread
  // (e.g. the caller of a solve_batch worker) may download them
  cudaStreamSynchronize(cudaStreamPerThread);
  red->nforced = count;
  std::swap(red->d_forced.p, facc.p);
  std::swap(red->d_forced.bytes, facc.bytes);
}

static int root_reduce_impl(const vcg_graph* g, int enabled, int crown, int has_bound,
                            int64_t bound, vcg_preprocessed* info, int32_t* forced_out,
                            int64_t* vertex_map_out, vcg_graph** reduced_out, int spec_ok) {
  memset(info, 0, sizeof(*info));
  struct HostSpan {  // VCG_TRACE / VCG_HOSTSPAN: host time of the whole call
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), tret = t0;
    ~HostSpan() {
      static const bool on = getenv("VCG_HOSTSPAN") != nullptr;
      const auto t1 = std::chrono::steady_clock::now();
      if (trace_on() || on)
        fprintf(stderr, "[vcg root] host: root_reduce call %.1f us (after the first readback %.1f us)\n",
                std::chrono::duration<double, std::micro>(t1 - t0).count(),
                std::chrono::duration<double, std::micro>(t1 - tret).count());
    }
  } host_span;
  Tracer tr("root");
  const int n = (int)g->n;
  const int rules_on = enabled & 1;
  // PVC (has_bound == 1) never needs the greedy cover of the original graph;
  // the public root_reduce() asks for it (has_bound == 2) to mirror the
  // reference.  It runs on a host thread, overlapped with the device rules:
  // for MVC (has_bound == 0) it is also the rules' bound, so the rules run
  // with a speculative budget under which the high-degree rule cannot fire,
  // recording per round the largest (live degree + forced so far); once the
  // greedy value is known the host checks that the real budget would not
  // have fired it either (else the pipeline reruns with the real bound).
  int64_t greedy_orig = -1;
  std::atomic<bool> greedy_cancel{false};
  std::thread greedy_thr;
  // VCG_ROOT_LAZY_GREEDY: the greedy is not run at all; the caller certifies
  // the speculation afterwards (spec_need, see vcgpu.h)
  const bool lazy = (enabled & VCG_ROOT_LAZY_GREEDY) && has_bound == 0;
  if (has_bound != 1 && !lazy)
    greedy_thr = std::thread([&]() {
      greedy_orig =
          greedy_cover_host(g->n, g->hoff, g->hnbr, nullptr, &greedy_cancel);
    });
  struct JoinGuard {
    std::thread& t;
    ~JoinGuard() {
      if (t.joinable()) t.join();
    }
  } join_guard{greedy_thr};
  const bool spec = spec_ok && has_bound == 0 && rules_on && !getenv("VCG_NO_SPEC") &&
                    !(enabled & VCG_ROOT_NO_SPEC);
  if (has_bound == 0 && !spec && greedy_thr.joinable()) greedy_thr.join();
  const int64_t bound0 = has_bound ? bound : greedy_orig;  // unused while speculating
  std::vector<std::pair<int64_t, int64_t>> spec_rounds;   // (spec_m, forced before the round)
  tr.mark("greedy_original");
  SearchCtx& X = search_ctx();
  DevBuf& flag = X.r_flag;
  if (flag.ensure((size_t)(n + 1) * 4)) return VCG_ERESOURCE;
  std::vector<int64_t> vmap;
  int64_t forced_count = 0;
  bool residual_empty = false;  // the rules left no edge: no compaction needed
  DevBuf facc{true};            // forced ids on the device (forced_out == NULL)
  bool host_compact = false;
  std::vector<int32_t> host_deg;
  if (!rules_on) {
    std::vector<int32_t> ones(n + 1, 1);
    ones[n] = 0;
    CK(cudaMemcpy(flag.p, ones.data(), (size_t)(n + 1) * 4, cudaMemcpyHostToDevice));
  } else {
    DevBuf &ws = X.r_ws, &dout = X.r_out, &dret = X.r_ret;
    if (ws.ensure(ws_total<uint32_t>(n)) || dout.ensure((size_t)(2 * n + 4) * 4) ||
        dret.ensure(256))
      return VCG_ERESOURCE;
    // any-order callers (the solve path) get the order-free sweeps on an
    // on-chip workspace when it fits; larger graphs run the grid-wide
    // cooperative kernel (root_grid.cu); the degrees live at ws.p as int32
    DevAttrs* da = nullptr;
    if (int r = dev_attrs(&da)) return r;
    const int smem_optin = da->smem_optin;
    const long long fast_smem = ws_bytes<uint32_t>(n);
    // VCG_ROOT_GRID=1 forces the grid-wide kernel (tests), =0 the single-block ones
    const char* grid_env = getenv("VCG_ROOT_GRID");
    const bool on_chip = fast_smem + 8192 <= smem_optin;
    const bool fast = (enabled & VCG_ROOT_ANY_ORDER) && on_chip && !getenv("VCG_ROOT_ORDERED") &&
                      !(grid_env && atoi(grid_env) == 1);
    // VCG_ROOT_GRID=2 forces the frontier kernel (any-order callers only)
    const bool any_order = (enabled & VCG_ROOT_ANY_ORDER) && !getenv("VCG_ROOT_ORDERED");
    const bool use_front = any_order && (grid_env ? atoi(grid_env) == 2 : !on_chip);
    const bool use_grid =
        !fast && !use_front && (grid_env ? atoi(grid_env) >= 1 : !on_chip);
    if (use_grid && X.r_gctl.ensure(root_grid_ctl_bytes())) return VCG_ERESOURCE;
    if (use_front &&
        (X.r_fctl.ensure(root_front_ctl_bytes()) || X.r_front.ensure(root_front_bytes(n, (long long)g->m2))))
      return VCG_ERESOURCE;
    if (fast)
      if (int r = raise_smem_limit((const void*)k_root_fixpoint_fast, (size_t)fast_smem)) return r;
    info->kernel_kind = use_front ? 4 : use_grid ? 3 : fast ? 1 : 2;
    int lo = 0, hi = n - 1;
    if (!use_grid && !use_front) {  // the single-block kernels take the initial live window
      int l = -1, h = -1;
      for (int v = 0; v < n; ++v)
        if (g->hoff[v + 1] > g->hoff[v]) {
          if (l < 0) l = v;
          h = v;
        }
      if (l < 0 || g->m2 == 0) {
        lo = n > 1 ? n : 1;
        hi = 0;
      } else {
        lo = l;
        hi = h;
      }
    }
    std::vector<int32_t> hdeg;  // host copy of the degrees (crown / host compaction)
    int first = 1;
    int pos = 0;
    int64_t nforced = 0;  // forced ids written to forced_out (or to facc)
    static thread_local cudaEvent_t rk0 = nullptr, rk1 = nullptr;
    if (!rk0) {
      CK(cudaEventCreate(&rk0));
      CK(cudaEventCreate(&rk1));
    }
    int crown_applied_last = 1;
    bool hdeg_current = false;  // hdeg mirrors the device degrees
    static const int root_threads = getenv("VCG_ROOT_THREADS") ? atoi(getenv("VCG_ROOT_THREADS")) : 1024;
    while (true) {
      int64_t progressed = 0;
      auto t0 = std::chrono::steady_clock::now();
      long long ret[26];
      // a round after a crown that applied nothing finds the fixpoint
      // unchanged and the crown again empty: skip it (same counts)
      if (!first && !crown_applied_last) break;
      COUNT_LAUNCH(1);
      hdeg_current = false;
      const int budget = spec ? kSpecBudget : (int)(bound0 - forced_count);
      const auto tl0 = std::chrono::steady_clock::now();
      CK(cudaEventRecord(rk0, cudaStreamPerThread));
      if (use_front) {
        CK(root_front_launch(n, g->d_off.as<int32_t>(), g->d_nbr.as<int32_t>(), ws.as<char>(),
                             X.r_front.as<char>(), budget, dout.as<int32_t>(),
                             dret.as<long long>(), first, X.r_fctl.p));
      } else if (use_grid) {
        CK(root_grid_launch(n, g->d_off.as<int32_t>(), g->d_nbr.as<int32_t>(), ws.as<char>(),
                            budget, dout.as<int32_t>(), dret.as<long long>(), first, X.r_gctl.p));
      } else if (fast) {
        k_root_fixpoint_fast<<<1, root_threads, fast_smem>>>(
            n, g->d_off.as<int32_t>(), g->d_nbr.as<int32_t>(), ws.as<uint32_t>(), lo, hi,
            budget, dout.as<int32_t>(), dret.as<long long>(), first);
      } else {
        k_root_fixpoint<<<1, 1024>>>(n, g->d_off.as<int32_t>(), g->d_nbr.as<int32_t>(),
                                     ws.as<char>(), lo, hi, budget,
                                     dout.as<int32_t>(), 0, dret.as<long long>(), first);
      }
      CK(cudaGetLastError());
      CK(cudaEventRecord(rk1, cudaStreamPerThread));
      const auto tl1 = std::chrono::steady_clock::now();
      CK(cudaMemcpy(ret, dret.p, fast ? 144 : use_front ? 208 : use_grid ? 88 : 80,
                    cudaMemcpyDeviceToHost));
      const auto tl2 = std::chrono::steady_clock::now();
      if (first) host_span.tret = tl2;
      if (trace_on())
        fprintf(stderr, "[vcg root] host: entry..launch %.1f us, launch call %.1f us, launch..ret copied %.1f us\n",
                std::chrono::duration<double, std::micro>(tl0 - host_span.t0).count(),
                std::chrono::duration<double, std::micro>(tl1 - tl0).count(),
                std::chrono::duration<double, std::micro>(tl2 - tl0).count());
      {
        float kms = 0.f;
        CK(cudaEventElapsedTime(&kms, rk0, rk1));
        info->kernel_ms += kms;
        info->kernel_launches += 1;
        info->kernel_scans += (use_grid || use_front || fast) ? ret[10] : 0;
        if (use_front) {
          info->kernel_sweeps += ret[11];
          info->kernel_walked += ret[13];
          info->kernel_barriers += ret[25];
        }
      }
      if (fast && trace_on())
        fprintf(stderr, "[vcg root] fixpoint sweeps: scans %lld (%lld cyc) d1 %lld (%lld) tri %lld (%lld) hd %lld (%lld)\n",
                ret[10], ret[14], ret[11], ret[15], ret[12], ret[16], ret[13], ret[17]);
      if (use_front && trace_on())
        fprintf(stderr, "[vcg root] frontier fixpoint (%d blocks): %lld full passes, %lld sweeps "
                "(%lld in one block), %lld adjacency entries, %lld frontier entries, forced %lld; "
                "us: solo %.1f, grid d1 %.1f, grid tri %.1f, hd %.1f\n",
                root_front_blocks(), ret[10], ret[11], ret[12], ret[13], ret[14], ret[0],
                ret[15] * 1e-3, ret[16] * 1e-3, ret[17] * 1e-3, ret[18] * 1e-3);
      if (use_front && trace_on()) root_front_print_log(X.r_fctl.p);
      if (use_front && trace_on())
        fprintf(stderr, "[vcg root] d1 phases us: A %.1f syncA %.1f B %.1f syncB %.1f C %.1f syncC %.1f\n",
                ret[19] * 1e-3, ret[22] * 1e-3, ret[20] * 1e-3, ret[23] * 1e-3, ret[21] * 1e-3,
                ret[24] * 1e-3);
      if (use_grid && trace_on())
        fprintf(stderr, "[vcg root] grid fixpoint (%d blocks): %lld scans, forced %lld\n",
                root_grid_blocks(), ret[10], ret[0]);
      if ((fast || use_grid || use_front) && ret[8])
        return fail(VCG_ECUDA, "root fixpoint: inconsistent degree array");
      if (spec)
        spec_rounds.emplace_back((fast || use_grid || use_front) ? ret[9] : ret[8], forced_count);
      first = 0;
      if (ret[7] > 0 && forced_out)  // straight into the caller's buffer
        CK(cudaMemcpy(forced_out + nforced, dout.p, (size_t)ret[7] * 4, cudaMemcpyDeviceToHost));
      if (ret[7] > 0 && !forced_out) {  // kept on the device for the reduced graph
        if (!facc.p && facc.ensure((size_t)std::max(n, 1) * 4)) return VCG_ERESOURCE;
        CK(cudaMemcpyAsync(facc.as<int32_t>() + nforced, dout.p, (size_t)ret[7] * 4,
                           cudaMemcpyDeviceToDevice, cudaStreamPerThread));
      }
      nforced += ret[7];
      info->rule_counts[0] += ret[1];
      info->rule_counts[1] += ret[2];
      info->rule_counts[2] += ret[3];
      forced_count += ret[0];
      progressed += ret[0];
      lo = (int)ret[5];
      hi = (int)ret[6];
      info->seconds[0] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      tr.mark("  device rules round");
      if (has_bound && forced_count > bound) break;
      if (crown && lo > hi) crown_applied_last = 0;  // an empty residual has no crown
      if (crown && lo <= hi) {
        auto t1 = std::chrono::steady_clock::now();
        // large graphs: the round trip of the degree array goes through a
        // pinned per-thread buffer (pageable copies of 4 MB took ~0.4 ms each
        // way on planted1m with 3x noise)
        int32_t* hd = nullptr;
        if (n > kHostCompactMax) {
          if (int r = pinned_ints(n, &hd)) return r;
        } else {
          hdeg.resize(n);
          hd = hdeg.data();
          hdeg_current = true;
        }
        CK(cudaMemcpy(hd, ws.p, (size_t)n * 4, cudaMemcpyDeviceToHost));
        std::vector<int32_t> heads;
        int64_t er = 0;
        int64_t nh = crown_reduce_host(n, g->hoff, g->hnbr, hd, lo, hi,
                                       &heads, &er);
        crown_applied_last = nh > 0;
        if (nh > 0) {
          info->rule_counts[3] += 1;
          if (forced_out) {
            std::copy(heads.begin(), heads.end(), forced_out + nforced);
          } else if (!heads.empty()) {
            if (!facc.p && facc.ensure((size_t)std::max(n, 1) * 4)) return VCG_ERESOURCE;
            CK(cudaMemcpy(facc.as<int32_t>() + nforced, heads.data(), heads.size() * 4,
                          cudaMemcpyHostToDevice));
          }
          nforced += (int64_t)heads.size();
          forced_count += nh;
          progressed += nh;
          CK(cudaMemcpy(ws.p, hd, (size_t)n * 4, cudaMemcpyHostToDevice));
          int l = -1, h = -1;
          for (int v = lo; v <= hi; ++v)
            if (hd[v] > 0) {
              if (l < 0) l = v;
              h = v;
            }
          if (l < 0) {
            lo = n > 1 ? n : 1;
            hi = 0;
          } else {
            lo = l;
            hi = h;
          }
        }
        info->seconds[1] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
        tr.mark("  crown round");
      }
      if (progressed == 0) break;
    }
    (void)pos;
    residual_empty = lo > hi;
    const char* dc_env = getenv("VCG_DEVICE_COMPACT");
    if (residual_empty) {
      // nothing survives: the empty graph, no flag / scan / gather
    } else if (n <= kHostCompactMax && !(dc_env && atoi(dc_env) == 1)) {
      if (!hdeg_current) {
        hdeg.resize(n);
        CK(cudaMemcpy(hdeg.data(), ws.p, (size_t)n * 4, cudaMemcpyDeviceToHost));
      }
      host_compact = true;
      host_deg.swap(hdeg);
    } else {
      COUNT_LAUNCH(1);
      k_flags_from_deg<<<(n + 256) / 256 + 1, 256>>>(ws.as<uint32_t>(), n, flag.as<int32_t>());
      CK(cudaGetLastError());
    }
  }
  tr.mark("rules+crown");
  auto t2 = std::chrono::steady_clock::now();
  vcg_graph* red = nullptr;
  if (residual_empty) {
    red = new vcg_graph();
    red->n = 0;
    red->m2 = 0;
    if (red->d_off.ensure(4) || red->d_nbr.ensure(4)) {
      delete red;
      return VCG_ERESOURCE;
    }
    CK(cudaMemsetAsync(red->d_off.p, 0, 4, cudaStreamPerThread));
    red->own_off.assign(1, 0);
    red->adopt_owned();
  } else if (host_compact) {
    if (int r = compact_host(g, host_deg.data(), &red, &vmap)) return r;
  } else if (int r = compact_flagged(g, flag, &red, &vmap)) {
    return r;
  }
  info->seconds[2] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t2).count();
  info->forced_count = forced_count;
  info->n_reduced = red->n;
  info->m_reduced = red->m2 / 2;
  int64_t md = 0;
  for (int64_t v = 0; v < red->n; ++v) md = std::max<int64_t>(md, red->hoff[v + 1] - red->hoff[v]);
  info->max_degree_reduced = md;
  tr.mark("compaction");
  info->greedy_reduced = greedy_cover_host(red->n, red->hoff, red->hnbr, nullptr);
  tr.mark("greedy_reduced");
  // VCG_ROOT_LAZY_GREEDY (the MVC solve path): every vertex cover of g has
  // at least forced + (maximal matching of the reduced graph) vertices --
  // the root rules keep an optimal cover -- and so does the greedy one.  If
  // that lower bound already certifies both uses of the greedy value (the
  // speculative high-degree check and best_init = greedy_reduced), the
  // greedy is abandoned and reported as -1.
  if (lazy) {
    // the greedy of g is the MVC bound, >= every cover size: the speculation
    // holds iff greedy_original >= spec_need; the caller checks it against
    // the optimum it finds (a lower bound of the greedy), and only computes
    // the greedy when that does not suffice
    int64_t need = -1;
    for (const auto& sr : spec_rounds) need = std::max<int64_t>(need, sr.first + sr.second);
    info->spec_need = need;
    info->greedy_original = -1;
    if (vertex_map_out)
      for (size_t i = 0; i < vmap.size(); ++i) vertex_map_out[i] = vmap[i];
    attach_forced(red, facc, forced_count, forced_out);
    *reduced_out = red;
    return 0;
  }
  if (greedy_thr.joinable()) greedy_thr.join();
  tr.mark("greedy_original joined");
  info->greedy_original = greedy_orig;
  for (const auto& sr : spec_rounds)
    if (sr.first > greedy_orig - sr.second) {  // the real budget would have fired
      vcg_graph_destroy(red);
      return kSpecFailed;
    }
  if (vertex_map_out)
    for (size_t i = 0; i < vmap.size(); ++i) vertex_map_out[i] = vmap[i];
  attach_forced(red, facc, forced_count, forced_out);
  *reduced_out = red;
  return 0;
}

extern "C" int vcg_graph_forced(const vcg_graph* reduced, int32_t* out, int64_t* count) {
  if (!reduced || !count) return fail(VCG_EINVAL, "bad arguments");
  if (reduced->nforced < 0) return fail(VCG_EINVAL, "not a root reduction's graph");
  *count = reduced->nforced;
  if (out && reduced->nforced > 0)
    CK(cudaMemcpy(out, reduced->d_forced.p, (size_t)reduced->nforced * 4, cudaMemcpyDeviceToHost));
  return 0;
}

extern "C" int vcg_root_reduce(const vcg_graph* g, int enabled, int crown, int has_bound,
                               int64_t bound, vcg_preprocessed* info, int32_t* forced_out,
                               int64_t* vertex_map_out, vcg_graph** reduced_out) {
  if (int r = need_device()) return r;
  if (!g || !info || !reduced_out) return fail(VCG_EINVAL, "bad arguments");
  int r = root_reduce_impl(g, enabled, crown, has_bound, bound, info, forced_out, vertex_map_out,
                           reduced_out, 1);
  if (r == kSpecFailed)
    r = root_reduce_impl(g, enabled, crown, has_bound, bound, info, forced_out, vertex_map_out,
                         reduced_out, 0);
  return r;
}

// -------------------------------------------------------------- expansion --
// FIFO of int32-degree node records in HBM: [S, E, lo, hi, split, pad, pad, pad | deg[n]]

__global__ void k_expand(int n, const int32_t* off, const int32_t* nbr, char* wsmem, char* fifo,
                         long long rec_bytes, long long cap, long long target, int best_init,
                         int use_components, int use_bounds, long long* out) {
  __shared__ BlockScratch bs;
  __shared__ int sh[8];
  init_block_scratch(&bs);
  NodeWs<uint32_t> w = carve_ws<uint32_t>(wsmem, n, &bs, off, nbr);
  w.inc = w.inc2 = nullptr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    w.tmin[i] = kInf;
    w.flag[i] = 0;
    if (i < (n + 31) / 32) w.vbits[i] = 0u;
  }
  __syncthreads();
  long long head = 0, tail = 1, nodes = 0;
  int best = best_init;
  auto rec = [&](long long i) { return fifo + (i % cap) * rec_bytes; };
  // splits stay open: they are moved behind the tail and never expanded
  long long open_splits = 0;
  while (head < tail && (tail - head) < target) {
    int* hd = (int*)rec(head);
    if (hd[4]) {  // an unexpanded split node: rotate it behind the tail
      if (open_splits >= tail - head) break;  // only splits left
      if (tail - head + 1 > cap) break;
      int* dstr = (int*)rec(tail);
      for (long long i = threadIdx.x; i < rec_bytes / 4; i += blockDim.x) dstr[i] = hd[i];
      __syncthreads();
      ++head;
      ++tail;
      ++open_splits;
      continue;
    }
    open_splits = 0;
    const int S0 = hd[0], E0 = hd[1], lo0 = hd[2], hi0 = hd[3];
    uint32_t* dg = (uint32_t*)(hd + 8);
    for (int i = threadIdx.x; i < n; i += blockDim.x) w.deg[i] = dg[i];
    __syncthreads();
    ++head;
    ++nodes;
    long long maxkey;
    FixRet fr = reduce_fixpoint_fast(w, lo0, hi0, best - S0 - 1, &maxkey);
    int S = S0 + fr.forced, E = E0 - fr.edges, lo = fr.lo, hi = fr.hi;
    if (!use_bounds && n) {
      lo = 0;
      hi = n - 1;
    }
    bool prune = S >= best;
    if (!prune) {
      long long rem = (long long)best - S - 1;
      prune = (long long)E > rem * rem;
    }
    if (prune) continue;
    if (E == 0) {
      best = S;  // a leaf: the cover found so far is the new bound
      continue;
    }
    int split = 0;
    if (use_components) {
      int nc = label_components(w, lo, hi, true);
      split = nc > 1;
    }
    if (tail + 2 - head > cap) break;
    int* c1 = (int*)rec(tail);
    uint32_t* d1 = (uint32_t*)(c1 + 8);
    if (split) {  // keep the node (after its reduction) as an open subtree
      for (int i = threadIdx.x; i < n; i += blockDim.x) d1[i] = w.deg[i];
      if (threadIdx.x == 0) {
        c1[0] = S;
        c1[1] = E;
        c1[2] = lo;
        c1[3] = hi;
        c1[4] = 1;
      }
      __syncthreads();
      ++tail;
      continue;
    }
    const int v = maxkey < 0 ? -1 : 0x7fffffff - (int)(maxkey & 0xffffffffLL);
    // exclude child (N(v) forced) first, then include child (v forced)
    for (int i = threadIdx.x; i < n; i += blockDim.x) w.deg2[i] = w.deg[i];
    __syncthreads();
    NodeWs<uint32_t> wx = w;
    wx.deg = w.deg2;
    int removed, edges;
    remove_neighbors_fast(wx, v, w.lst, &removed, &edges);
    for (int i = threadIdx.x; i < n; i += blockDim.x) d1[i] = w.deg2[i];
    if (threadIdx.x == 0) {
      c1[0] = S + removed;
      c1[1] = E - edges;
      c1[2] = lo;
      c1[3] = hi;
      c1[4] = 0;
    }
    int e2 = remove_vertex(w, v);
    int* c2 = (int*)rec(tail + 1);
    uint32_t* d2 = (uint32_t*)(c2 + 8);
    for (int i = threadIdx.x; i < n; i += blockDim.x) d2[i] = w.deg[i];
    if (threadIdx.x == 0) {
      c2[0] = S + 1;
      c2[1] = E - e2;
      c2[2] = lo;
      c2[3] = hi;
      c2[4] = 0;
    }
    __syncthreads();
    tail += 2;
  }
  if (threadIdx.x == 0) {
    out[0] = head;
    out[1] = tail;
    out[2] = best;
    out[3] = nodes;
  }
  (void)sh;
}

extern "C" int vcg_expand(const vcg_graph* g, const vcg_expand_config* cfg, vcg_expand_result* res,
                          int32_t* sub_S, int32_t* sub_deg, int64_t capacity) {
  if (int r = need_device()) return r;
  if (!g || !cfg || !res || cfg->target < 1) return fail(VCG_EINVAL, "bad arguments");
  const int n = (int)g->n;
  const long long rec_bytes = 32 + 4LL * ((n + 3) & ~3);
  const long long cap = 2 * cfg->target + 8;
  SearchCtx& X = search_ctx();
  DevBuf &ws = X.x_ws, &fifo = X.x_fifo, &out = X.x_out;
  if (ws.ensure(ws_total<uint32_t>(n)) || fifo.ensure((size_t)(cap * rec_bytes)) || out.ensure(64))
    return VCG_ERESOURCE;
  std::vector<int32_t> root(rec_bytes / 4, 0);
  int lo = -1, hi = -1;
  for (int v = 0; v < n; ++v) {
    int d = (int)(g->hoff[v + 1] - g->hoff[v]);
    root[8 + v] = d;
    if (d) {
      if (lo < 0) lo = v;
      hi = v;
    }
  }
  root[0] = 0;
  root[1] = (int)(g->m2 / 2);
  root[2] = lo < 0 ? (n > 1 ? n : 1) : lo;
  root[3] = lo < 0 ? 0 : hi;
  CK(cudaMemcpy(fifo.p, root.data(), rec_bytes, cudaMemcpyHostToDevice));
  COUNT_LAUNCH(1);
  k_expand<<<1, 512>>>(n, g->d_off.as<int32_t>(), g->d_nbr.as<int32_t>(), ws.as<char>(),
                       fifo.as<char>(), rec_bytes, cap, cfg->target, (int)cfg->best_init,
                       cfg->use_components, cfg->use_bounds, out.as<long long>());
  CK(cudaGetLastError());
  long long o[4];
  CK(cudaMemcpy(o, out.p, 32, cudaMemcpyDeviceToHost));
  const long long head = o[0], tail = o[1];
  memset(res, 0, sizeof(*res));
  res->best = o[2];
  res->nodes = o[3];
  const long long count = tail - head;
  if (count > capacity) return fail(VCG_ERESOURCE, "expansion capacity too small");
  std::vector<int32_t> buf(rec_bytes / 4);
  for (long long i = 0; i < count; ++i) {
    CK(cudaMemcpy(buf.data(), fifo.as<char>() + ((head + i) % cap) * rec_bytes, rec_bytes,
                  cudaMemcpyDeviceToHost));
    sub_S[i] = buf[0];
    memcpy(sub_deg + i * (int64_t)n, buf.data() + 8, (size_t)n * 4);
  }
  res->count = count;
  return 0;
}

// ----------------------------------------------------------------- search --


template <typename T>
static int search_t(const vcg_graph* gc, const vcg_search_config* cfg, vcg_search_result* res,
                    int64_t* hist_out) {
  vcg_graph* g = const_cast<vcg_graph*>(gc);
  SearchCtx& C = search_ctx();
  Tracer tr("search");
  const int n = (int)g->n;
  DevAttrs* da = nullptr;
  if (int r = dev_attrs(&da)) return r;
  const int sm_count = da->sm_count, smem_optin = da->smem_optin;

  const bool auto_threads = cfg->threads <= 0;
  int threads = cfg->threads;
  if (auto_threads) threads = n <= 256 ? 64 : n <= 512 ? 128 : n <= 32768 ? 256 : 512;
  const long long wsb = ws_total<T>(n);
  const long long smem_limit = (long long)smem_optin - 8192;  // static smem headroom
  const int smem_fits = wsb <= smem_limit && !getenv("VCG_WS_GLOBAL");
  const long long csrb = csr_smem_bytes(n, g->m2);
  // warp tier limit; < 0 = auto: 128-vertex tasks on small dense reduced
  // graphs (average degree >= 8, n <= 256: G(180, 0.08) 7.7 s -> 0.9 s),
  // 64 otherwise -- sparse graphs' component splits already fit 64 and
  // their long 128-vertex tasks would serialise (rgg2000 PVC 1.2 -> 8.9 ms),
  // and on larger dense graphs the search rarely gets down to 128 live
  // vertices while the 128-bit workspaces halve the resident blocks
  // (G(400, 0.1): 15.6 -> 8.7 M nodes/s)
  int warp_limit0 = cfg->warp_limit;
  if (warp_limit0 < 0) {
    const bool dense = g->m2 >= 8LL * g->n;
    warp_limit0 = dense && g->n <= 256 ? 128 : dense && g->n <= 640 ? 256 : 64;
  }
  warp_limit0 = std::min(warp_limit0, kWMax);
  if (cfg->deterministic || cfg->record_cover || !cfg->use_components || cfg->disable_pruning ||
      !cfg->load_balance)
    warp_limit0 = 0;
  // when the wide warp tier carries the search, more warps per block beat
  // the small blocks a small graph's node operations want: 256 threads with
  // 128-vertex tasks (G(180, 0.08): 0.91 -> 0.68 s), 128 with 256-vertex
  // tasks (their workspaces are 4x larger; G(400, 0.1) 15.6 -> 38 M nodes/s)
  if (auto_threads && warp_limit0 > 64) threads = warp_limit0 > 128 ? 128 : 256;
  // launch plan for a block size, workspace placement (shared memory or a
  // per-block slice of HBM) and CSR placement: dynamic shared memory,
  // warp-tier workspace placement and resident blocks per SM
  struct Plan {
    int threads, in_smem, csr_smem, warp_limit, bws_alias, per_sm;
    long long bws_off;
    size_t dsmem;
  };
  // kernel variant: workspace placement x widest warp-task mask (64-bit words)
  auto variant = [](int ws_smem, int wl) -> void (*)(SearchParams) {
    const int ww = wl > 128 ? 4 : wl > 64 ? 2 : 1;
    if (ws_smem)
      return ww == 4 ? search_kernel<T, true, 4>
             : ww == 2 ? search_kernel<T, true, 2> : search_kernel<T, true, 1>;
    return ww == 4 ? search_kernel<T, false, 4>
           : ww == 2 ? search_kernel<T, false, 2> : search_kernel<T, false, 1>;
  };
  auto plan = [&](int th, int ws_smem, int csr, Plan* pl) -> int {
    pl->threads = th;
    pl->in_smem = ws_smem;
    pl->csr_smem = ws_smem && csr;
    pl->dsmem = ws_smem ? (size_t)(wsb + (pl->csr_smem ? csrb : 0)) : 0;
    // warp tier: per-warp workspaces alias the node workspace's int scratch
    // (ia .. par, 7 arrays; the tier runs only while the block holds no node)
    // when that is large enough, else they follow in dynamic shared memory
    pl->warp_limit = th > 32 * kWTierWarps ? 0 : warp_limit0;
    pl->bws_alias = 0;
    pl->bws_off = 0;
    if (pl->warp_limit) {
      const long long need =
          (long long)(th / 32) * (long long)(warp_limit0 > 128  ? sizeof(WarpWs4)
                                             : warp_limit0 > 64 ? sizeof(WarpWs2)
                                                                : sizeof(WarpWs1));
      const long long ni = ((long long)std::max(n, 1) + 3) & ~3LL;
      if (ws_smem && 7 * ni * 4 >= need) {
        pl->bws_alias = 1;
      } else {
        pl->bws_off = ((long long)pl->dsmem + 15) & ~15LL;
        // the wide-tier variants carry more static shared memory (the task
        // packing table): check against the variant's own headroom
        cudaFuncAttributes fa{};
        CK(cudaFuncGetAttributes(&fa, (const void*)variant(ws_smem, pl->warp_limit)));
        const long long lim = std::min<long long>(smem_limit, (long long)smem_optin -
                                                                  (long long)fa.sharedSizeBytes);
        if (pl->bws_off + need <= lim) pl->dsmem = (size_t)(pl->bws_off + need);
        else pl->warp_limit = 0;
      }
    }
    auto kern = variant(ws_smem, pl->warp_limit);
    if (int r = raise_smem_limit((const void*)kern, pl->dsmem)) return r;
    pl->per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl->per_sm, kern, th, pl->dsmem));
    return 0;
  };
  Plan pl;
  const int csr_fits = smem_fits && wsb + csrb <= smem_limit && !getenv("VCG_NO_SMEM_CSR");
  if (int r = plan(threads, smem_fits, csr_fits, &pl)) return r;
  if (!cfg->deterministic && cfg->workers <= 0 && auto_threads) {
    // a staged CSR that dominates the block's shared memory (dense reduced
    // graphs, e.g. G(400, 0.1)) is dropped when that at least doubles the
    // resident blocks: more concurrent nodes beat on-chip adjacency there
    if (pl.csr_smem && csrb > 2 * wsb) {
      Plan alt;
      if (int r = plan(threads, 1, 0, &alt)) return r;
      if (alt.per_sm >= 2 * pl.per_sm) pl = alt;
    }
    // one resident block per SM (large workspaces, e.g. the 60x60 torus):
    // 128-thread blocks with their workspaces in HBM (L1/L2-resident) keep
    // 8x the nodes in flight, which beats on-chip workspaces there
    // (torus60: 5.4 vs 2.7 M nodes/s)
    if (pl.in_smem && pl.per_sm == 1) {
      Plan alt;
      if (int r = plan(128, 0, 0, &alt)) return r;
      if (alt.per_sm >= 4) pl = alt;
    }
  }
  // the chosen plan is the kernel's final attribute setting
  if (int r = plan(pl.threads, pl.in_smem, pl.csr_smem, &pl)) return r;
  auto kern = variant(pl.in_smem, pl.warp_limit);
  const int in_smem = pl.in_smem;
  threads = pl.threads;
  const int csr_smem = pl.csr_smem;
  const int warp_limit = pl.warp_limit;
  const int bws_alias = pl.bws_alias;
  const long long bws_off = pl.bws_off;
  const size_t dsmem = pl.dsmem;
  const int per_sm = pl.per_sm;
  if (per_sm < 1) return fail(VCG_ERESOURCE, "search kernel does not fit on an SM");
  const int share_k = cfg->gpu_share > 1 ? cfg->gpu_share : 1;
  const int resident = std::max(1, per_sm * sm_count / share_k);
  int blocks = cfg->deterministic ? 1 : (cfg->workers > 0 ? cfg->workers : resident);
  // a residual of <= 32 vertices (the ba100k / planted1m root reductions
  // leave 4-21) is one small warp task: one block per SM is plenty, and 16
  // per SM cost their start-up and exit (search kernel 0.048 -> 0.039 ms)
  if (!cfg->deterministic && cfg->workers <= 0 && pl.warp_limit && n <= 32 &&
      blocks > sm_count)
    blocks = sm_count;
  if (blocks > resident) blocks = resident;

  const long long slot = (long long)sizeof(NodeHdr) + deg_bytes<T>(n) +
                         (cfg->record_cover ? bits_bytes(n) : 0);
  // private stack: depth <= n + 1 (SPEC preprocess: stack bound), capped by memory
  long long stack_cap = (long long)n + 2;
  const long long stack_budget = 16LL << 30;
  if (stack_cap * slot * blocks > stack_budget) stack_cap = std::max(16LL, stack_budget / (slot * blocks));
  const int share = cfg->load_balance && !cfg->deterministic;
  long long threshold = cfg->worklist_threshold > 0 ? cfg->worklist_threshold : 2LL * blocks;
  long long qcap = std::max<long long>(4 * threshold + 1024, 4096);
  const long long q_budget = 4LL << 30;
  if (qcap * slot > q_budget) qcap = std::max(4096LL, q_budget / slot);
  const int reg_cap = (int)std::min<long long>(1LL << 23, std::max<long long>(1LL << 16, (long long)n * 1024));

  // warp-task ring: slots sized for the run's limit (576 B at 64 vertices,
  // 8 KB at 256); fewer of the large ones
  const long long bcap = !warp_limit ? 16
                         : warp_limit > 128 ? std::max<long long>(16384, 16LL * blocks)
                                            : std::max<long long>(65536, 64LL * blocks);
  // component subgraph arena: order-preserving compaction of split
  // components (not in record-cover mode, whose witnesses use reduced ids)
  const int compact = !cfg->record_cover && !getenv("VCG_NO_COMPACT");
  const int sg_cap = compact ? (1 << 20) : 1;
  const long long arena_cap = compact ? std::min<long long>(
      (1LL << 28), std::max<long long>(1LL << 22, 64LL * ((long long)n + 1 + g->m2))) : 4;
  if (C.sg.ensure((size_t)sg_cap * 8 + 64) || C.arena.ensure((size_t)arena_cap * 4)) return VCG_ERESOURCE;
  const long long bslot = wslot_bytes(std::max(warp_limit, 1));
  if (C.bseq.ensure((size_t)bcap * 8) || C.bdata.ensure((size_t)(bcap * bslot)) ||
      C.bctl.ensure(64))
    return VCG_ERESOURCE;
  if (C.stacks.ensure((size_t)(stack_cap * slot * blocks)) || C.qseq.ensure((size_t)qcap * 8) ||
      C.qdata.ensure((size_t)(qcap * slot)) || C.qctl.ensure(64) ||
      C.reg.ensure((size_t)reg_cap * (4 * 13 + 8) + 64 + 8 * kFreeClasses * kFreeShards) ||
      C.ctl.ensure(sizeof(Ctl)) ||
      C.hist.ensure((size_t)(n + 2) * 8) ||
      (!in_smem && C.gws.ensure((size_t)(wsb * blocks))))
    return VCG_ERESOURCE;

  tr.mark("alloc");
  SearchParams P;
  memset(&P, 0, sizeof(P));
  P.n = n;
  P.m2 = g->m2;
  P.csr_in_smem = csr_smem;
  P.off = g->d_off.as<int32_t>();
  P.nbr = g->d_nbr.as<int32_t>();
  P.stacks = C.stacks.as<char>();
  P.stack_cap = stack_cap;
  P.slot_bytes = slot;
  P.q.seq = C.qseq.as<unsigned long long>();
  P.q.head = C.qctl.as<unsigned long long>();
  P.q.tail = C.qctl.as<unsigned long long>() + 1;
  P.q.count = C.qctl.as<unsigned long long>() + 2;
  P.q.err = &C.ctl.as<Ctl>()->error;
  P.q.data = C.qdata.as<char>();
  P.q.cap = qcap;
  int* rb = C.reg.as<int>();
  Registry& R = P.reg;
  R.key = rb;
  R.live = rb + reg_cap;
  R.link = rb + 2 * reg_cap;
  R.kind = rb + 3 * reg_cap;
  R.sum = rb + 4 * reg_cap;
  R.sum_ach = rb + 5 * reg_cap;
  R.init_sum = rb + 6 * reg_cap;
  R.folded = rb + 7 * reg_cap;
  R.first_child = rb + 8 * reg_cap;
  R.nchild = rb + 9 * reg_cap;
  R.disc_done = rb + 10 * reg_cap;
  R.child_folded = rb + 11 * reg_cap;
  R.pwrec = rb + 12 * reg_cap;
  R.count = rb + 13 * reg_cap;
  R.wkey = (unsigned long long*)(rb + 13 * reg_cap + 16);  // 64-byte aligned
  R.cap = reg_cap;
  R.fheads = R.wkey + reg_cap;
  const int record = cfg->record_cover != 0;
  // registry reclamation: parallel mode, unless the entries are read back
  // (record-cover witnesses, audits, the registry view) -- VCG_NO_RECLAIM=1 off
  R.reclaim = !record && !cfg->deterministic && !cfg->check_registry && !cfg->registry_out &&
              !getenv("VCG_NO_RECLAIM");
  // recycling starts at half the arena (VCG_RECLAIM_AT: entries, tests use 0)
  R.reclaim_at = getenv("VCG_RECLAIM_AT") ? atoi(getenv("VCG_RECLAIM_AT")) : reg_cap / 2;
  const int nw = (n + 31) / 32;
  int wcap = 0;
  if (record) {
    wcap = (int)std::min<long long>(1LL << 22, std::max<long long>(4096, (1LL << 30) / (nw * 4LL)));
    if (C.wbits.ensure((size_t)wcap * nw * 4) || C.wcount.ensure(64)) return VCG_ERESOURCE;
  }
  P.record = record;
  P.nw = nw;
  P.wbits = C.wbits.as<unsigned>();
  P.wcount = C.wcount.as<int>();
  P.wcap = wcap;
  P.ctl = C.ctl.as<Ctl>();
  P.hist = C.hist.as<unsigned long long>();
  P.gws = C.gws.as<char>();
  P.gws_bytes = wsb;
  P.ws_in_smem = in_smem;
  P.share = share;
  P.batch_live = !cfg->deterministic && !getenv("VCG_NO_BATCH");
  P.par_rules = !cfg->deterministic && !getenv("VCG_EXACT_RULES");
  P.threshold = threshold;
  P.use_components = cfg->use_components;
  P.use_bounds = cfg->use_bounds;
  P.disable_pruning = cfg->disable_pruning;
  P.pvc = cfg->pvc;
  P.k_red = (int)cfg->k_red;
  P.root_index = 0;
  P.root_in_stack = 1;
  P.bq.seq = C.bseq.as<unsigned long long>();
  P.bq.head = C.bctl.as<unsigned long long>();
  P.bq.tail = C.bctl.as<unsigned long long>() + 1;
  P.bq.count = C.bctl.as<unsigned long long>() + 2;
  P.bq.err = &C.ctl.as<Ctl>()->error;
  P.bq.data = C.bdata.as<char>();
  P.bq.cap = bcap;
  P.warp_limit = warp_limit;
  P.bq_slot = bslot;
  P.warp_split_export = !getenv("VCG_NO_WSPLIT");
  P.tma_load = !getenv("VCG_NO_TMA");  // VCG_NO_TMA: per-thread loads instead
  P.bq_low = std::max(8LL, (long long)blocks * (threads / 32) / 4);
  if (const char* e = getenv("VCG_BQLOW")) P.bq_low = atoll(e);  // experiments
  {
    const char* e1 = getenv("VCG_WCHECK");
    const char* e2 = getenv("VCG_WEXPORT");
    P.w_check_mask = e1 ? atoi(e1) : 3;
    P.w_export_after = e2 ? atoi(e2) : 4;
  }
  P.compact = compact;
  P.sg_n = C.sg.as<int>();
  P.sg_base = C.sg.as<int>() + sg_cap;
  P.sg_count = C.sg.as<int>() + 2 * sg_cap;
  P.arena_top = C.sg.as<int>() + 2 * sg_cap + 1;
  P.sg_cap = sg_cap;
  P.arena = C.arena.as<int>();
  P.arena_cap = (int)arena_cap;
  P.bws_alias = bws_alias;
  P.bws_off = bws_off;

  // root scope entry + root node record (engine.py:183-188)
  std::vector<char> rec(slot, 0);
  NodeHdr* hh = (NodeHdr*)rec.data();
  T* rdeg = (T*)(rec.data() + sizeof(NodeHdr));
  int lo = -1, hi = -1;
  int64_t dsum = 0;
  for (int v = 0; v < n; ++v) {
    int64_t d = cfg->root_deg ? cfg->root_deg[v] : g->hoff[v + 1] - g->hoff[v];
    rdeg[v] = (T)d;
    dsum += d;
    if (d) {
      if (lo < 0) lo = v;
      hi = v;
    }
  }
  if (lo < 0 || dsum == 0) {
    lo = n > 1 ? n : 1;
    hi = 0;
  }
  hh->S = 0;
  hh->E = (int)(dsum / 2);
  hh->lo = lo;
  hh->hi = hi;
  hh->scope = 0;
  hh->depth = 0;
  CK(cudaMemcpyAsync(C.stacks.p, rec.data(), slot, cudaMemcpyHostToDevice, 0));
  double limit = cfg->timeout;
  if (limit <= 0) {
    // safety watchdog for test/bench runs: a protocol bug must not hang the GPU
    const char* wd = getenv("VCG_WATCHDOG_S");
    if (wd) limit = atof(wd);
  }
  const unsigned long long timeout_ns = limit > 0 ? (unsigned long long)(limit * 1e9) : 0ull;
  const int root_key = (int)(cfg->best_init * 2 + (cfg->best_init_achieved ? 0 : 1));
  COUNT_LAUNCH(1);
  search_init_kernel<<<256, 256>>>(P, root_key, timeout_ns);
  CK(cudaGetLastError());
  tr.mark("init");

  static thread_local cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (!e0) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
  }
  // debug heartbeat: per-warp progress codes in host-mapped memory, dumped
  // (and the process ended) when the search kernel overruns VCG_HEARTBEAT s
  static thread_local int* hb_host = nullptr;
  static thread_local long long hb_cap = 0;
  const char* hb_env = getenv("VCG_HEARTBEAT");
  P.xch = cfg->exchange ? cfg->exchange->d : nullptr;
  P.gpeer = cfg->peer ? cfg->peer->d : nullptr;
  P.gpeer_off = (int)cfg->peer_offset;
  P.hb = nullptr;
  if (hb_env) {
    const long long need = (long long)blocks * kMaxWarps;
    if (need > hb_cap) {
      if (hb_host) cudaFreeHost(hb_host);
      CK(cudaHostAlloc((void**)&hb_host, (size_t)need * 4, cudaHostAllocMapped));
      hb_cap = need;
    }
    memset(hb_host, 0, (size_t)need * 4);
    CK(cudaHostGetDevicePointer((void**)&P.hb, hb_host, 0));
  }
  cudaEventRecord(e0);
  COUNT_LAUNCH(2);  // search + drain
  kern<<<blocks, threads, dsmem>>>(P);
  cudaEventRecord(e1);
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) return fail(VCG_ECUDA, std::string("search launch: ") + cudaGetErrorString(le));
  if (hb_env) {
    const double lim = atof(hb_env);
    auto t0 = std::chrono::steady_clock::now();
    while (cudaEventQuery(e1) == cudaErrorNotReady) {
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > lim) {
        std::map<std::string, int> hist;
        const int nw = threads / 32;
        for (int b = 0; b < blocks; ++b) {
          std::string key;
          for (int w = 0; w < nw; ++w) key += std::to_string(((volatile int*)hb_host)[b * kMaxWarps + w]) + " ";
          hist[key] += 1;
        }
        fprintf(stderr, "[vcg heartbeat] search kernel still running after %.1f s (%d blocks x %d warps); per-warp codes -> blocks:\n", lim, blocks, nw);
        for (auto& kv : hist) fprintf(stderr, "  %5d x [ %s]\n", kv.second, kv.first.c_str());
        for (int b = 0; b < blocks; ++b) {
          const volatile int* r = hb_host + (long long)b * kMaxWarps;
          if (r[0] == 99) continue;
          fprintf(stderr, "  block %d: d1 ncand=%d applied=%d no-live-nbr=%d | graph=%d lo=%d hi=%d gn=%d cur_graph=%d ws.n=%d\n",
                  b, r[20], r[21], r[22], r[23], r[24], r[25], r[26], r[27], r[28]);
        }
        fflush(stderr);
        _exit(3);
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(50));
    }
  }
  tr.mark("search_kernel");
  drain_kernel<<<1, 32>>>(P);
  CK(cudaStreamSynchronize(cudaStreamPerThread));
  tr.mark("drain");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);

  Ctl ctl;
  CK(cudaMemcpy(&ctl, C.ctl.p, sizeof(Ctl), cudaMemcpyDeviceToHost));
  const int final_key = ctl.root_key, count = ctl.reg_count;
  memset(res, 0, sizeof(*res));
  res->best = final_key >> 1;
  res->best_achieved = !(final_key & 1);
  res->found = ctl.found;
  res->timed_out = ctl.timed_out;
  res->error = ctl.error;
  res->tree_nodes_visited = (int64_t)ctl.nodes;
  res->component_branches = (int64_t)ctl.comp_branches;
  res->worklist_pushes = (int64_t)ctl.pushes;
  res->worklist_pops = (int64_t)ctl.pops;
  res->max_stack_depth = ctl.max_depth;
  for (int i = 0; i < 6; ++i) res->rule_counts[i] = (int64_t)ctl.rules[i];
  res->registry_entries = count;
  res->kernel_ms = ms;
  res->workers = blocks;
  res->threads = threads;
  res->records_loaded = (int64_t)ctl.rec_in;
  res->records_stored = (int64_t)ctl.rec_out;
  res->slot_bytes = slot;
  for (int i = 0; i < 10; ++i) res->phase_cycles[i] = (int64_t)ctl.phase[i];
  res->warp_tasks = (int64_t)ctl.wtasks;
  res->warp_nodes = (int64_t)ctl.wnodes;
  res->warp_cycles = (int64_t)ctl.wcyc;
  res->warp_limit = warp_limit;
  res->warp_epoch_cycles = (int64_t)ctl.wepoch;
  res->warp_task_max_cycles = (int64_t)ctl.wmax;
  auto rel = [&](unsigned long long t) { return t && t != ~0ull ? (int64_t)(t - ctl.t0) : -1; };
  res->trace[0] = rel(ctl.t_node_last);
  res->trace[1] = rel(ctl.t_task_first);
  res->trace[2] = rel(ctl.t_task_last);
  res->trace[3] = (int64_t)ctl.wmax_nodes;
  res->trace[4] = (int64_t)ctl.wmax_n;
  res->trace[5] = (int64_t)ctl.wc_fix;
  res->trace[6] = (int64_t)ctl.wc_comp;
  res->trace[7] = (int64_t)ctl.wc_split;
#ifdef VCG_WARP_PROFILE
  res->trace[3] = (int64_t)ctl.wc_iter;  // profile builds: fixpoint iterations in place of max nodes
#endif
  res->kernel_t0_ns = (int64_t)ctl.t0;
  res->kernel_t1_ns = (int64_t)ctl.t_end;

  for (int i = 0; i < 4; ++i) {
    res->fix_cycles[i] = (int64_t)ctl.rcyc[i];
    res->fix_count[i] = (int64_t)ctl.rcnt[i];
  }
  if (hist_out) {
    std::vector<unsigned long long> h(n + 2);
    CK(cudaMemcpy(h.data(), C.hist.p, (size_t)(n + 2) * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n + 2; ++i) hist_out[i] = (int64_t)h[i];
  }
  tr.mark("readback");
  res->cover_size = -1;
  if (record && cfg->cover_out) {
    // expand the root's witness tree: leaf records are scoped cover bitsets,
    // composite witnesses are a split's record plus its children's witnesses
    std::vector<unsigned long long> wkey(count);
    std::vector<int> pw(count), fc(count), nc(count);
    CK(cudaMemcpy(wkey.data(), R.wkey, (size_t)count * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(pw.data(), R.pwrec, (size_t)count * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(fc.data(), R.first_child, (size_t)count * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(nc.data(), R.nchild, (size_t)count * 4, cudaMemcpyDeviceToHost));
    int wn = 0;
    CK(cudaMemcpy(&wn, P.wcount, 4, cudaMemcpyDeviceToHost));
    wn = std::min(wn, wcap);
    std::vector<unsigned> bits((size_t)wn * nw);
    if (wn) CK(cudaMemcpy(bits.data(), P.wbits, bits.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<unsigned> cover(nw, 0u);
    const unsigned long long root_w = wkey[0];
    bool ok = root_w != kNoWitness && (long long)(root_w >> 32) <= res->best;
    std::vector<int> stack;
    if (ok) stack.push_back(0);
    while (ok && !stack.empty()) {
      const int e = stack.back();
      stack.pop_back();
      const unsigned long long wk = wkey[e];
      if (wk == kNoWitness) {
        ok = false;
        break;
      }
      const unsigned wid = (unsigned)(wk & 0xffffffffu);
      int rec = (int)wid;
      if (wid & kComposite) {
        const int p = (int)(wid & ~kComposite);
        rec = pw[p];
        for (int c = fc[p]; c < fc[p] + nc[p]; ++c) stack.push_back(c);
      }
      if (rec < 0 || rec >= wn) {
        ok = false;
        break;
      }
      for (int i = 0; i < nw; ++i) cover[i] |= bits[(size_t)rec * nw + i];
    }
    if (ok) {
      int64_t k = 0;
      for (int v = 0; v < n; ++v)
        if (cover[v >> 5] >> (v & 31) & 1u) cfg->cover_out[k++] = v;
      res->cover_size = k;
    }
  }
  if (cfg->registry_out && count > 0 && count <= cfg->registry_cap) {
    std::vector<int> f(count);
    for (int k = 0; k < 12; ++k) {
      CK(cudaMemcpy(f.data(), rb + (size_t)k * reg_cap, (size_t)count * 4, cudaMemcpyDeviceToHost));
      for (int i = 0; i < count; ++i) cfg->registry_out[(size_t)i * 12 + k] = f[i];
    }
  }
  if (cfg->check_registry && count > 0) {
    // registry quiescence + conservation (SPEC registry invariants)
    std::vector<int> f[12];
    for (int k = 0; k < 12; ++k) {
      f[k].resize(count);
      CK(cudaMemcpy(f[k].data(), rb + (size_t)k * reg_cap, (size_t)count * 4, cudaMemcpyDeviceToHost));
    }
    int64_t bad = 0;
    for (int i = 0; i < count; ++i) {
      if (f[1][i] != 0) ++bad;  // live counters quiesced
      if (f[3][i] == 1) {
        long long expect = (long long)f[6][i] + f[7][i];
        for (int c = f[8][i]; c < f[8][i] + f[9][i]; ++c) expect += f[0][c] >> 1;
        if (expect != f[4][i]) ++bad;
      }
    }
    res->registry_violations = bad;
  }
  return 0;
}

// ---------------------------------------------------------------- exchange --

struct vcg_exchange {
  int dev = 0;
  int32_t* d = nullptr;  // [0] external bound, [1] external stop, [2] local best, [3] pad
};

extern "C" int vcg_exchange_create(vcg_exchange** out) {
  if (int r = need_device()) return r;
  if (!out) return fail(VCG_EINVAL, "bad arguments");
  auto* x = new vcg_exchange();
  CK(cudaGetDevice(&x->dev));
  if (cudaMalloc(&x->d, 16) != cudaSuccess) {
    delete x;
    return fail(VCG_ERESOURCE, "exchange: cudaMalloc failed");
  }
  *out = x;
  return vcg_exchange_reset(x);
}

extern "C" int vcg_exchange_destroy(vcg_exchange* x) {
  if (!x) return 0;
  if (!g_shutdown.load()) cudaFree(x->d);
  delete x;
  return 0;
}

extern "C" int vcg_exchange_reset(vcg_exchange* x) {
  if (!x) return fail(VCG_EINVAL, "bad arguments");
  const int32_t init[4] = {kInf, 0, kInf, 0};
  CK(cudaMemcpyAsync(x->d, init, 16, cudaMemcpyHostToDevice, cudaStreamPerThread));
  CK(cudaStreamSynchronize(cudaStreamPerThread));
  return 0;
}

extern "C" int vcg_exchange_post(vcg_exchange* x, int64_t bound, int stop) {
  if (!x) return fail(VCG_EINVAL, "bad arguments");
  if (bound >= 0) {
    const int32_t b = (int32_t)std::min<int64_t>(bound, kInf);
    CK(cudaMemcpyAsync(x->d, &b, 4, cudaMemcpyHostToDevice, cudaStreamPerThread));
  }
  if (stop) {
    const int32_t one = 1;
    CK(cudaMemcpyAsync(x->d + 1, &one, 4, cudaMemcpyHostToDevice, cudaStreamPerThread));
  }
  CK(cudaStreamSynchronize(cudaStreamPerThread));
  return 0;
}

extern "C" int vcg_exchange_peek(vcg_exchange* x, int64_t* local_best) {
  if (!x || !local_best) return fail(VCG_EINVAL, "bad arguments");
  int32_t v = kInf;
  CK(cudaMemcpyAsync(&v, x->d + 2, 4, cudaMemcpyDeviceToHost, cudaStreamPerThread));
  CK(cudaStreamSynchronize(cudaStreamPerThread));
  *local_best = v;
  return 0;
}

// ------------------------------------------------------------ peer words --

struct vcg_peer {
  int32_t* d = nullptr;  // [0] best absolute cover, [1] stop, [2..3] pad
  int owner = 0;         // allocated here (else mapped from another process)
};

__global__ void k_peer_offer(int32_t* d, int best, int stop) {
  if (best >= 0) atomicMin_system(d, best);
  if (stop) atomicExch_system(d + 1, 1);
}

extern "C" int vcg_peer_create(vcg_peer** out) {
  if (int r = need_device()) return r;
  if (!out) return fail(VCG_EINVAL, "bad arguments");
  auto* p = new vcg_peer();
  if (cudaMalloc(&p->d, 16) != cudaSuccess) {
    delete p;
    return fail(VCG_ERESOURCE, "peer: cudaMalloc failed");
  }
  p->owner = 1;
  const int32_t init[4] = {kInf, 0, 0, 0};
  CK(cudaMemcpy(p->d, init, 16, cudaMemcpyHostToDevice));
  *out = p;
  return 0;
}

extern "C" int vcg_peer_handle(const vcg_peer* p, void* handle) {
  if (!p || !handle || !p->owner) return fail(VCG_EINVAL, "bad arguments");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, p->d));
  static_assert(sizeof(h) <= VCG_PEER_HANDLE_BYTES, "IPC handle size");
  memset(handle, 0, VCG_PEER_HANDLE_BYTES);
  memcpy(handle, &h, sizeof(h));
  return 0;
}

extern "C" int vcg_peer_open(const void* handle, vcg_peer** out) {
  if (int r = need_device()) return r;
  if (!handle || !out) return fail(VCG_EINVAL, "bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* ptr = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess)
    return fail(VCG_ECUDA, std::string("peer: cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  auto* p = new vcg_peer();
  p->d = (int32_t*)ptr;
  *out = p;
  return 0;
}

extern "C" int vcg_peer_destroy(vcg_peer* p) {
  if (!p) return 0;
  if (!g_shutdown.load()) {
    if (p->owner) cudaFree(p->d);
    else cudaIpcCloseMemHandle(p->d);
  }
  delete p;
  return 0;
}

extern "C" int vcg_peer_offer(vcg_peer* p, int64_t best, int stop) {
  if (!p) return fail(VCG_EINVAL, "bad arguments");
  COUNT_LAUNCH(1);
  k_peer_offer<<<1, 1>>>(p->d, best < 0 ? -1 : (int)std::min<int64_t>(best, kInf), stop);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(cudaStreamPerThread));
  return 0;
}

extern "C" int vcg_peer_read(const vcg_peer* p, int64_t* best, int* stop) {
  if (!p || !best || !stop) return fail(VCG_EINVAL, "bad arguments");
  int32_t w[2] = {kInf, 0};
  CK(cudaMemcpy(w, p->d, 8, cudaMemcpyDeviceToHost));
  *best = w[0];
  *stop = w[1];
  return 0;
}

extern "C" int vcg_search(const vcg_graph* g, const vcg_search_config* cfg, vcg_search_result* res,
                          int64_t* hist_out) {
  if (int r = need_device()) return r;
  if (!g || !cfg || !res) return fail(VCG_EINVAL, "bad arguments");
  if (g->n == 0 || g->m2 == 0) return fail(VCG_EINVAL, "search needs a graph with edges");
  if (cfg->root_deg) {
    int64_t dsum = 0;
    for (int64_t v = 0; v < g->n; ++v) dsum += cfg->root_deg[v];
    if (dsum == 0) return fail(VCG_EINVAL, "subtree root has no edges");
  }
  if (cfg->width == 8) return search_t<uint8_t>(g, cfg, res, hist_out);
  if (cfg->width == 16) return search_t<uint16_t>(g, cfg, res, hist_out);
  if (cfg->width == 32) return search_t<uint32_t>(g, cfg, res, hist_out);
  return fail(VCG_EINVAL, "width must be 8, 16 or 32");
}
