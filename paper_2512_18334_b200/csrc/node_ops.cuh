// Block-level operations on one search-tree node's degree array.
//
// One thread block owns one search node at a time (north star (2)); every
// function here is called by ALL threads of the block with block-uniform
// arguments and returns block-uniform results.  The degree array lives in
// shared memory when it fits (generic pointers, so the same code also runs on
// a global-memory workspace for very large reduced graphs).
//
// Semantics are those of the reference's sequential kernels
// (vcsolver/kernels/pure.py) -- same forced sets, same `out` order, same
// returned counters -- obtained with parallel formulations that are exact,
// not approximate:
//
// * degree-one sweep (pure.py:82-110): a snapshot candidate v (deg 1, unique
//   live neighbour u(v)) applies iff it is the lowest-index candidate
//   targeting u(v) and is not the higher end of an isolated edge whose lower
//   end is also a candidate.  (v can only lose its degree through u(v), so
//   this closed form equals the in-order sweep.)
// * triangle sweep (pure.py:113-155): valid candidates are found in
//   parallel; the in-order conflict resolution is a lane-0 scan over the
//   (short) compacted list; removals are applied in parallel.
// * high-degree sweep (pure.py:158-185): in-order warp scan while the running
//   budget is >= 0; once it is negative the remaining candidates follow the
//   closed form "applies iff it still has a live neighbour that is not an
//   earlier remaining candidate".
//
// Sub-word degree decrements use a 32-bit atomicSub on the containing word:
// a live entry is >= 1, so the subtraction never borrows into the neighbour
// entry (SPEC graph_core design decision on sub-word atomics, §4.4).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vcg {

constexpr int kInf = 0x7fffffff;
// Speculative root budget: the root rules run with this budget while the
// host computes the greedy bound; the high-degree rule cannot fire, and the
// sweeps record in BlockScratch::spec_m the largest (max live degree +
// vertices forced so far) they saw, so the host can verify afterwards that
// the real budget would not have fired it either (capi.cu vcg_root_reduce).
constexpr int kSpecBudget = 1 << 30;
constexpr int kMaxWarps = 32;

// ---------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ int ldv(const T* p, int i) {
  return (int)(*(const volatile T*)(p + i));
}

template <typename T>
__device__ __forceinline__ void deg_dec(T* deg, int x) {
  if constexpr (sizeof(T) == 4) {
    atomicSub((unsigned*)(deg + x), 1u);
  } else {
    uintptr_t a = (uintptr_t)(deg + x);
    unsigned* w = (unsigned*)(a & ~(uintptr_t)3);
    unsigned sh = (unsigned)(a & 3) * 8u;
    atomicSub(w, 1u << sh);
  }
}

// record-cover mode: vertex u joins the node's (scoped) cover
__device__ __forceinline__ void mark_inc(unsigned* inc, int u) {
  if (inc) atomicOr(&inc[u >> 5], 1u << (u & 31));
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// block collectives (all threads call; result is block-uniform)
// ---------------------------------------------------------------------------

struct BlockScratch {
  int v[kMaxWarps + 8];
  long long w[kMaxWarps + 2];
  int v2[kMaxWarps];
  int v3[kMaxWarps];
  long long w2[kMaxWarps];
  int bc[16];  // broadcast slots
  // thread-0 profile of the fixpoint: cycles and counts of scans, degree-one,
  // triangle and high-degree sweeps
  unsigned long long rcyc[4];
  unsigned long long rcnt[4];
  // one-barrier reductions: per-warp partials, double-buffered per call
  // (a warp can only reuse a buffer after the next call's barrier, by which
  // time every warp has read it); the parity is per warp, so no cross-warp race
  int red[2][8][kMaxWarps];
  int wpar[kMaxWarps];
  // debug heartbeat (VCG_HEARTBEAT): this block's row of per-warp codes in
  // host-mapped memory, null when off
  int* hb;
  int spec_m;  // speculative root budget: max(live degree + forced so far)
};

#ifdef VCG_DBG_FENCE
#define VCG_FENCE() __threadfence()
#else
#define VCG_FENCE() \
  do {              \
  } while (0)
#endif

// lane 0 of the calling warp records `code` in the heartbeat row
#define VCG_HB(bs, code)                                                  \
  do {                                                                    \
    if ((bs)->hb && (threadIdx.x & 31) == 0)                              \
      ((volatile int*)(bs)->hb)[threadIdx.x >> 5] = (code);               \
  } while (0)

__device__ __forceinline__ void rprof(BlockScratch* bs, int i, long long* t) {
  if (threadIdx.x == 0) {
    long long now = clock64();
    bs->rcyc[i] += (unsigned long long)(now - *t);
    bs->rcnt[i] += 1;
    *t = now;
  }
}

__device__ __forceinline__ int warp_sum(int x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ int warp_parity(BlockScratch* bs) {
  return ((volatile int*)bs->wpar)[threadIdx.x >> 5];
}
__device__ __forceinline__ void warp_parity_flip(BlockScratch* bs, int p) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) bs->wpar[threadIdx.x >> 5] = p ^ 1;
  __syncwarp();
}

// op: 0 add, 1 min, 2 max.  K values reduced with one block barrier.
template <int K>
__device__ __forceinline__ void block_reduce(int (&x)[K], const int (&op)[K], BlockScratch* bs) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const int p = warp_parity(bs);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    int r = op[k] == 0   ? __reduce_add_sync(0xffffffffu, x[k])
            : op[k] == 1 ? __reduce_min_sync(0xffffffffu, x[k])
                         : __reduce_max_sync(0xffffffffu, x[k]);
    if (lane == 0) bs->red[p][k][wid] = r;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int ident = op[k] == 0 ? 0 : op[k] == 1 ? kInf : -kInf;
    int y = lane < nw ? bs->red[p][k][lane] : ident;
    x[k] = op[k] == 0   ? __reduce_add_sync(0xffffffffu, y)
           : op[k] == 1 ? __reduce_min_sync(0xffffffffu, y)
                        : __reduce_max_sync(0xffffffffu, y);
  }
  warp_parity_flip(bs, p);
}

__device__ __forceinline__ int block_sum(int x, BlockScratch* bs) {
  int v[1] = {x};
  const int op[1] = {0};
  block_reduce<1>(v, op, bs);
  return v[0];
}

__device__ __forceinline__ int block_min(int x, BlockScratch* bs) {
  int v[1] = {x};
  const int op[1] = {1};
  block_reduce<1>(v, op, bs);
  return v[0];
}

__device__ __forceinline__ int block_max(int x, BlockScratch* bs) {
  int v[1] = {x};
  const int op[1] = {2};
  block_reduce<1>(v, op, bs);
  return v[0];
}

__device__ __forceinline__ long long block_max64(long long x, BlockScratch* bs) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y > x ? y : x;
  }
  __syncthreads();
  if (lane == 0) bs->w[wid] = x;
  __syncthreads();
  long long t = bs->w[0];
  for (int i = 1; i < nw; ++i) t = bs->w[i] > t ? bs->w[i] : t;
  return t;
}

// Exclusive prefix of x over threads in threadIdx order; *total = sum.
__device__ __forceinline__ int block_exscan(int x, BlockScratch* bs, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();
  if (lane == 31 || (int)threadIdx.x == (int)blockDim.x - 1) bs->v[wid] = inc;
  __syncthreads();
  int before = 0, tot = 0;
  for (int i = 0; i < nw; ++i) {
    int s = bs->v[i];
    if (i < wid) before += s;
    tot += s;
  }
  *total = tot;
  return before + inc - x;
}

// contiguous chunk [b, e) of [lo, hi] owned by this thread (index order is
// preserved across threads, so chunked scans give in-order compaction)
__device__ __forceinline__ void my_chunk(int lo, int hi, int* b, int* e) {
  int len = hi - lo + 1;
  if (len <= 0) {
    *b = *e = 0;
    return;
  }
  int per = (len + (int)blockDim.x - 1) / (int)blockDim.x;
  long long s = (long long)lo + (long long)threadIdx.x * per;
  long long t = s + per;
  if (s > hi + 1) s = hi + 1;
  if (t > hi + 1) t = hi + 1;
  *b = (int)s;
  *e = (int)t;
}

// ---------------------------------------------------------------------------
// per-node workspace
// ---------------------------------------------------------------------------

template <typename T>
struct NodeWs {
  T* deg;           // current node degree array [n] (4-byte aligned)
  T* deg2;          // second degree buffer [n] (exclude child under construction)
  int* tmin;        // [n], kept == kInf between operations
  int* ia;          // [n] int scratch
  int* ib;          // [n]
  int* ic;          // [n]
  int* lst;         // [n]
  int* id;          // [n]
  int* par;         // [n] union-find parents (component labels)
  unsigned* vbits;  // [ceil(n/32)] candidate bitmap, all-zero between sweeps
  uint8_t* flag;    // [n], kept == 0 between operations
  unsigned* inc;    // cover-membership bitset of the node (record-cover mode), else null
  unsigned* inc2;   // bitset of the exclude child under construction
  BlockScratch* bs;
  const int* off;   // static CSR (reduced graph), int32 offsets
  const int* nbr;
  int n;
};

// every kernel that uses the block collectives calls this first
__device__ __forceinline__ void init_block_scratch(BlockScratch* bs) {
  if (threadIdx.x < kMaxWarps) bs->wpar[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    bs->hb = nullptr;
    bs->spec_m = -1;
  }
  __syncthreads();
}

struct PassRet {
  int applied;
  int forced;
  int edges;
  int pos;
};

template <typename T>
__device__ __forceinline__ bool adjacent_static(const NodeWs<T>& w, int u, int x) {
  int lo = w.off[u], hi = w.off[u + 1] - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int y = w.nbr[mid];
    if (y == x) return true;
    if (y < x) lo = mid + 1;
    else hi = mid - 1;
  }
  return false;
}

// Removal of a vertex u that is part of a set being removed together
// (flag[.] == mark for every member): live neighbours outside the set are
// decremented, an edge inside the set is counted once.  Returns edges.
// deg[u] itself is zeroed by the caller once every member is processed.
template <typename T>
__device__ __forceinline__ int remove_marked_edges(const NodeWs<T>& w, int u, uint8_t mark) {
  int e = 0;
  const int b = w.off[u], end = w.off[u + 1];
  for (int i = b; i < end; ++i) {
    int x = w.nbr[i];
    if (w.flag[x] == mark) {
      if (x > u && ldv(w.deg, x) > 0) ++e;
    } else if (ldv(w.deg, x) > 0) {
      deg_dec(w.deg, x);
      ++e;
    }
  }
  return e;
}

// Parallel removal of the list out[b0, b0+cnt) (all flagged 1 and live).
template <typename T>
__device__ __forceinline__ int remove_list(const NodeWs<T>& w, const int* list, int cnt) {
  int edges = 0;
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) edges += remove_marked_edges(w, list[k], 1);
  VCG_FENCE();
  edges = block_sum(edges, w.bs);  // also a barrier
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
    int u = list[k];
    w.deg[u] = 0;
    w.flag[u] = 0;
    mark_inc(w.inc, u);
  }
  __syncthreads();
  return edges;
}

// ---------------------------------------------------------------------------
// rule sweeps
// ---------------------------------------------------------------------------

// pure.py:82 degree_one_pass.  Returns {applied, forced, edges, new_pos}.
template <typename T>
__device__ PassRet degree_one_pass(const NodeWs<T>& w, int lo, int hi, int* out, int pos) {
  int b, e;
  my_chunk(lo, hi, &b, &e);
  int cnt = 0;
  for (int v = b; v < e; ++v) cnt += (w.deg[v] == 1);
  int ncand;
  int at = block_exscan(cnt, w.bs, &ncand);
  if (ncand == 0) return PassRet{0, 0, 0, pos};
  for (int v = b; v < e; ++v) {
    if (w.deg[v] == 1) {
      int u = -1;
      for (int i = w.off[v]; i < w.off[v + 1]; ++i) {
        int x = w.nbr[i];
        if (w.deg[x] > 0) {
          u = x;
          break;
        }
      }
      w.ia[v] = u;
      w.lst[at++] = v;
      atomicMin(&w.tmin[u], v);
    }
  }
  VCG_FENCE();
  __syncthreads();
  // decide, in candidate order (chunks of the candidate list)
  int cb, ce;
  my_chunk(0, ncand - 1, &cb, &ce);
  int napp = 0;
  for (int k = cb; k < ce; ++k) {
    int v = w.lst[k];
    int u = w.ia[v];
    bool app = (w.tmin[u] == v) && !(w.deg[u] == 1 && w.ia[u] == v && u < v);
    w.ic[k] = app;
    napp += app;
  }
  int total;
  int oat = block_exscan(napp, w.bs, &total);
  for (int k = cb; k < ce; ++k) {
    if (w.ic[k]) {
      int u = w.ia[w.lst[k]];
      out[pos + oat++] = u;
      w.flag[u] = 1;
    }
  }
  __syncthreads();
  int edges = remove_list(w, out + pos, total);
  for (int k = threadIdx.x; k < ncand; k += blockDim.x) w.tmin[w.ia[w.lst[k]]] = kInf;
  __syncthreads();
  return PassRet{total, total, edges, pos + total};
}

// pure.py:113 degree_two_triangle_pass
template <typename T>
__device__ PassRet degree_two_triangle_pass(const NodeWs<T>& w, int lo, int hi, int* out, int pos) {
  int b, e;
  my_chunk(lo, hi, &b, &e);
  int cnt = 0;
  for (int v = b; v < e; ++v) {
    if (w.deg[v] == 2) {
      int u = -1, x2 = -1;
      for (int i = w.off[v]; i < w.off[v + 1]; ++i) {
        int x = w.nbr[i];
        if (w.deg[x] > 0) {
          if (u < 0) {
            u = x;
          } else {
            x2 = x;
            break;
          }
        }
      }
      bool ok = x2 >= 0 && adjacent_static(w, u, x2);
      w.ia[v] = u;
      w.ib[v] = x2;
      w.ic[v] = ok;
      cnt += ok;
    }
  }
  int nvalid;
  int at = block_exscan(cnt, w.bs, &nvalid);
  if (nvalid == 0) return PassRet{0, 0, 0, pos};
  for (int v = b; v < e; ++v)
    if (w.deg[v] == 2 && w.ic[v]) w.lst[at++] = v;
  __syncthreads();
  // in-order conflict resolution (sequential semantics), lane 0
  if (threadIdx.x == 0) {
    int p = pos, applied = 0;
    for (int k = 0; k < nvalid; ++k) {
      int v = w.lst[k];
      int u = w.ia[v], x2 = w.ib[v];
      if (!w.flag[v] && !w.flag[u] && !w.flag[x2]) {
        w.flag[u] = 1;
        w.flag[x2] = 1;
        out[p++] = u;
        out[p++] = x2;
        ++applied;
      }
    }
    w.bs->bc[0] = applied;
  }
  __syncthreads();
  int applied = w.bs->bc[0];
  int edges = remove_list(w, out + pos, 2 * applied);
  return PassRet{applied, 2 * applied, edges, pos + 2 * applied};
}

// pure.py:158 high_degree_pass.
template <typename T>
__device__ PassRet high_degree_pass(const NodeWs<T>& w, int lo, int hi, int budget, int* out,
                                    int pos) {
  VCG_HB(w.bs, 104);
  int b, e;
  my_chunk(lo, hi, &b, &e);
  int cnt = 0, dmax = 0;
  for (int v = b; v < e; ++v) {
    int d = w.deg[v];
    cnt += (d > 0 && d > budget);
    dmax = d > dmax ? d : dmax;
  }
  if (budget > kSpecBudget / 2) {  // speculative: forced so far = kSpecBudget - budget
    dmax = block_max(dmax, w.bs);
    if (threadIdx.x == 0 && dmax + (kSpecBudget - budget) > w.bs->spec_m)
      w.bs->spec_m = dmax + (kSpecBudget - budget);
  }
  int ncand;
  int at = block_exscan(cnt, w.bs, &ncand);
  if (ncand == 0) return PassRet{0, 0, 0, pos};
  for (int v = b; v < e; ++v) {
    int d = w.deg[v];
    if (d > 0 && d > budget) w.lst[at++] = v;
  }
  __syncthreads();
  // sequential phase: warp 0, in candidate order, while the budget is >= 0
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int i = 0, bud = budget, p = pos, applied = 0, edges = 0;
    while (i < ncand && bud >= 0) {
      int c = w.lst[i];
      int d = ldv(w.deg, c);
      if (d > 0 && d > bud) {
        for (int j = w.off[c] + lane; j < w.off[c + 1]; j += 32) {
          int x = w.nbr[j];
          if (ldv(w.deg, x) > 0) deg_dec(w.deg, x);
        }
        VCG_FENCE();
        __syncwarp();
        if (lane == 0) {
          w.deg[c] = 0;
          mark_inc(w.inc, c);
          out[p] = c;
        }
        __syncwarp();
        ++p;
        ++applied;
        edges += d;
        --bud;
      }
      ++i;
    }
    if (lane == 0) {
      w.bs->bc[0] = i;
      w.bs->bc[1] = p;
      w.bs->bc[2] = applied;
      w.bs->bc[3] = edges;
    }
  }
  __syncthreads();
  const int i0 = w.bs->bc[0];
  int p = w.bs->bc[1], applied = w.bs->bc[2], edges = w.bs->bc[3];
  __syncthreads();
  if (i0 < ncand) {
    // closed form for the remaining candidates R = lst[i0:]: c applies iff
    // it has a live neighbour x with x not in R or x > c
    const int nr = ncand - i0;
    for (int k = threadIdx.x; k < nr; k += blockDim.x) w.flag[w.lst[i0 + k]] = 2;
    __syncthreads();
    int cb, ce;
    my_chunk(0, nr - 1, &cb, &ce);
    int napp = 0;
    for (int k = cb; k < ce; ++k) {
      int c = w.lst[i0 + k];
      bool app = false;
      if (w.deg[c] > 0) {
        for (int j = w.off[c]; j < w.off[c + 1]; ++j) {
          int x = w.nbr[j];
          if (w.deg[x] > 0 && (w.flag[x] != 2 || x > c)) {
            app = true;
            break;
          }
        }
      }
      w.ic[k] = app;
      napp += app;
    }
    int total;
    int oat = block_exscan(napp, w.bs, &total);
    for (int k = cb; k < ce; ++k)
      if (w.ic[k]) out[p + oat++] = w.lst[i0 + k];
    __syncthreads();
    for (int k = threadIdx.x; k < nr; k += blockDim.x) w.flag[w.lst[i0 + k]] = w.ic[k] ? 1 : 0;
    __syncthreads();
    edges += remove_list(w, out + p, total);
    p += total;
    applied += total;
  }
  return PassRet{applied, applied, edges, p};
}

// pure.py:230 recompute_bounds -> (lo, hi); empty -> (max(n,1), 0)
template <typename T>
__device__ void recompute_bounds(const NodeWs<T>& w, int* lo, int* hi) {
  int l = *lo, h = *hi;
  int mn = kInf, mx = -1;
  if (l <= h) {
    for (int v = l + threadIdx.x; v <= h; v += blockDim.x) {
      if (w.deg[v] > 0) {
        mn = min(mn, v);
        mx = max(mx, v);
      }
    }
  }
  mn = block_min(mn, w.bs);
  mx = block_max(mx, w.bs);
  if (mx < 0) {
    *lo = w.n > 1 ? w.n : 1;
    *hi = 0;
  } else {
    *lo = mn;
    *hi = mx;
  }
}

struct FixRet {
  int forced, d1, d2t, hd, edges, lo, hi, pos;
};

// pure.py:188 reduce_fixpoint
template <typename T>
__device__ FixRet reduce_fixpoint(const NodeWs<T>& w, int lo, int hi, int budget, int* out,
                                  int pos) {
  FixRet r{0, 0, 0, 0, 0, lo, hi, pos};
  while (true) {
    int cycle = 0;
    while (true) {
      PassRet a = degree_one_pass(w, lo, hi, out, r.pos);
      r.d1 += a.applied;
      r.forced += a.forced;
      r.edges += a.edges;
      r.pos = a.pos;
      cycle += a.applied;
      if (a.applied == 0) break;
    }
    PassRet t = degree_two_triangle_pass(w, lo, hi, out, r.pos);
    r.d2t += t.applied;
    r.forced += t.forced;
    r.edges += t.edges;
    r.pos = t.pos;
    cycle += t.applied;
    PassRet h = high_degree_pass(w, lo, hi, budget - r.forced, out, r.pos);
    r.hd += h.applied;
    r.forced += h.forced;
    r.edges += h.edges;
    r.pos = h.pos;
    cycle += h.applied;
    if (cycle == 0) break;
  }
  int l = lo, h = hi;
  recompute_bounds(w, &l, &h);
  r.lo = l;
  r.hi = h;
  return r;
}

// pure.py:241 select_max_degree: lowest-index live vertex of max degree, or -1
template <typename T>
__device__ int select_max_degree(const NodeWs<T>& w, int lo, int hi) {
  long long best = -1;
  if (lo <= hi) {
    for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x) {
      int d = w.deg[v];
      if (d > 0) {
        long long key = ((long long)d << 32) | (long long)(unsigned)(0x7fffffff - v);
        best = key > best ? key : best;
      }
    }
  }
  best = block_max64(best, w.bs);
  if (best < 0) return -1;
  return 0x7fffffff - (int)(best & 0xffffffffLL);
}

template <typename T>
__device__ int count_live(const NodeWs<T>& w, int lo, int hi) {
  int c = 0;
  if (lo <= hi)
    for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x) c += (w.deg[v] > 0);
  return block_sum(c, w.bs);
}

// pure.py:30 remove_vertex (single vertex, whole block): returns edges removed
template <typename T>
__device__ int remove_vertex(const NodeWs<T>& w, int v) {
  int d = w.deg[v];
  __syncthreads();
  if (d == 0) return 0;
  for (int j = w.off[v] + threadIdx.x; j < w.off[v + 1]; j += blockDim.x) {
    int x = w.nbr[j];
    if (ldv(w.deg, x) > 0) deg_dec(w.deg, x);
  }
  VCG_FENCE();
  __syncthreads();
  if (threadIdx.x == 0) {
    w.deg[v] = 0;
    mark_inc(w.inc, v);
  }
  __syncthreads();
  return d;
}

// pure.py:47 remove_neighbors: force every live neighbour of v; returns
// {removed, edges}; forced ids appended to out[pos..] in adjacency order.
template <typename T>
__device__ void remove_neighbors(const NodeWs<T>& w, int v, int* out, int pos, int* removed,
                                 int* edges) {
  if (w.deg[v] == 0) {  // pure.py:55: a dead vertex has no live neighbours to force
    *removed = 0;
    *edges = 0;
    __syncthreads();
    return;
  }
  const int b = w.off[v], e = w.off[v + 1];
  // compact live neighbours (adjacency order) into out
  int cb, ce;
  my_chunk(b, e - 1, &cb, &ce);
  int cnt = 0;
  for (int j = cb; j < ce; ++j) cnt += (w.deg[w.nbr[j]] > 0);
  int total;
  int at = block_exscan(cnt, w.bs, &total);
  for (int j = cb; j < ce; ++j) {
    int x = w.nbr[j];
    if (w.deg[x] > 0) {
      out[pos + at++] = x;
      w.flag[x] = 1;
    }
  }
  __syncthreads();
  *edges = remove_list(w, out + pos, total);
  *removed = total;
}

// ---------------------------------------------------------------------------
// search-path variants: same forced SETS and counters as the ordered sweeps
// above (so every statistic is unchanged), but the forced ids are appended in
// arbitrary order -- the search only needs the counts -- which removes one
// block scan per sweep, and the candidate counts of all three rules come from
// one fused pass over the window.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void block_scan3(int a, int b, int c, BlockScratch* bs, int* a_before,
                                            int* ta, int* tb, int* tc) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int inc = a;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  int sb = warp_sum(b), sc = warp_sum(c);
  __syncthreads();
  if (lane == 31 || (int)threadIdx.x == (int)blockDim.x - 1) bs->v[wid] = inc;
  if (lane == 0) {
    bs->w[wid] = ((long long)sb << 32) | (unsigned)sc;
  }
  if (threadIdx.x == 0) bs->bc[8] = 0;  // append counter for the pass that follows
  __syncthreads();
  int before = 0, tot = 0;
  long long t2 = 0, t3 = 0;
  for (int i = 0; i < nw; ++i) {
    int s = bs->v[i];
    if (i < wid) before += s;
    tot += s;
    t2 += (int)(bs->w[i] >> 32);
    t3 += (int)(bs->w[i] & 0xffffffffLL);
  }
  *a_before = before + inc - a;
  *ta = tot;
  *tb = (int)t2;
  *tc = (int)t3;
}

// block_scan3 plus the live window (min / max live index) and the
// max-degree key ((deg << 32) | (INT_MAX - v): lowest index on ties) in the
// same two barriers -- the last scan of a fixpoint describes the final state
struct ScanStats {
  int c1, c2, ch, lo, hi;
  long long key;
};

__device__ __forceinline__ ScanStats block_scan_stats(int a, int b, int c, int mn, int mx,
                                                      int dmax, int dmax_v, BlockScratch* bs) {
  {
    int v[6] = {a, b, c, mn, mx, dmax};
    const int op[6] = {0, 0, 0, 1, 2, 2};
    block_reduce<6>(v, op, bs);
    a = v[0];
    b = v[1];
    c = v[2];
    mn = v[3];
    mx = v[4];
    // lowest index among the vertices of maximum degree (pure.py:241 tie-break)
    int w2[1] = {dmax == v[5] ? dmax_v : kInf};
    const int op2[1] = {1};
    block_reduce<1>(w2, op2, bs);
    dmax = v[5];
    dmax_v = w2[0];
  }
  long long key = dmax > 0 ? (((long long)dmax << 32) | (long long)(unsigned)(0x7fffffff - dmax_v))
                           : -1;
  return ScanStats{a, b, c, mn, mx, key};
}

template <typename T>
__device__ __forceinline__ void deg_zero(T* deg, int x) {
  if constexpr (sizeof(T) == 4) {
    atomicExch((unsigned*)(deg + x), 0u);
  } else {
    uintptr_t a = (uintptr_t)(deg + x);
    unsigned* w = (unsigned*)(a & ~(uintptr_t)3);
    unsigned sh = (unsigned)(a & 3) * 8u;
    unsigned mask = (sizeof(T) == 1 ? 0xffu : 0xffffu) << sh;
    atomicAnd(w, ~mask);
  }
}

// Remove the vertices list[0, cnt) (all flagged 1, all live) together.
// Each remover zeroes its own entry atomically (flagged entries are never
// decremented by others); flags are cleared after the barrier inside the
// block_sum, before any later reader (every later reader is behind a barrier).
template <typename T>
__device__ __forceinline__ int remove_list_fast(const NodeWs<T>& w, const int* list, int cnt) {
  VCG_HB(w.bs, 105);
  int edges = 0;
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
    const int u = list[k];
    const int b = w.off[u], end = w.off[u + 1];
    for (int i = b; i < end; ++i) {
      int x = w.nbr[i];
      if (w.flag[x] == 1) {
        if (x > u) ++edges;
      } else if (ldv(w.deg, x) > 0) {
        deg_dec(w.deg, x);
        ++edges;
      }
    }
    deg_zero(w.deg, u);
    mark_inc(w.inc, u);
  }
  VCG_FENCE();
  edges = block_sum(edges, w.bs);
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) w.flag[list[k]] = 0;
  return edges;
}

// degree-one sweep with the candidate count/offsets already known
template <typename T>
__device__ PassRet degree_one_pass_fast(const NodeWs<T>& w, int b, int e, int ncand, int* rem) {
  VCG_HB(w.bs, 102);
  // candidates in any order: the decision below depends only on tmin
  for (int v = b; v < e; ++v) {
    if (w.deg[v] == 1) {
      int u = -1;
      for (int i = w.off[v]; i < w.off[v + 1]; ++i) {
        int x = w.nbr[i];
        if (w.deg[x] > 0) {
          u = x;
          break;
        }
      }
      if (u < 0) {  // inconsistent degree array: report instead of looping
        if (w.bs->hb) atomicAdd(&w.bs->hb[22], 1);
        w.bs->bc[10] = 1;
        continue;
      }
      w.ia[v] = u;
      w.lst[atomicAdd(&w.bs->bc[8], 1)] = v;
      atomicMin(&w.tmin[u], v);
    }
  }
  VCG_FENCE();
  __syncthreads();
  ncand = w.bs->bc[8];
  for (int k = threadIdx.x; k < ncand; k += blockDim.x) {
    int v = w.lst[k];
    int u = w.ia[v];
    if ((w.tmin[u] == v) && !(w.deg[u] == 1 && w.ia[u] == v && u < v)) {
      w.flag[u] = 1;
      rem[atomicAdd(&w.bs->bc[9], 1)] = u;
    }
  }
  __syncthreads();
  const int total = w.bs->bc[9];
  if (threadIdx.x == 0 && w.bs->hb) {
    ((volatile int*)w.bs->hb)[20] = ncand;
    ((volatile int*)w.bs->hb)[21] = total;
  }
  int edges = remove_list_fast(w, rem, total);
  for (int k = threadIdx.x; k < ncand; k += blockDim.x) w.tmin[w.ia[w.lst[k]]] = kInf;
  return PassRet{total, total, edges, 0};
}

// Triangle sweep with the reference's exact outcome, resolved in parallel.
// The in-order walk applies candidate c iff no earlier applied candidate's
// closed triangle T = {v, u, x} meets T(c) (a shared vertex is always a
// removed neighbour of one of them), i.e. the applied set is the
// lexicographically-first maximal independent set of the triangles'
// intersection graph.  Rounds: every undecided candidate claims its three
// vertices (atomicMin); one holding all three claims has no undecided
// earlier conflicting candidate, so it is in; one touching a removed vertex
// is out.  The minimum undecided candidate is decided every round.
template <typename T>
__device__ PassRet degree_two_triangle_pass_lfmis(const NodeWs<T>& w, int b, int e, int* rem) {
  VCG_HB(w.bs, 108);
  int nvalid = 0;
  for (int v = b; v < e; ++v) {
    if (w.deg[v] == 2) {
      int u = -1, x2 = -1;
      for (int i = w.off[v]; i < w.off[v + 1]; ++i) {
        int x = w.nbr[i];
        if (w.deg[x] > 0) {
          if (u < 0) {
            u = x;
          } else {
            x2 = x;
            break;
          }
        }
      }
      if (x2 >= 0 && adjacent_static(w, u, x2)) {
        w.ia[v] = u;
        w.ib[v] = x2;
        const int k = atomicAdd(&w.bs->bc[8], 1);
        w.lst[k] = v;
        w.ic[k] = 0;  // undecided
        ++nvalid;
      }
    }
  }
  nvalid = block_sum(nvalid, w.bs);
  if (nvalid == 0) return PassRet{0, 0, 0, 0};
  while (true) {
    for (int k = threadIdx.x; k < nvalid; k += blockDim.x) {
      if (w.ic[k] != 0) continue;
      const int v = w.lst[k];
      atomicMin(&w.tmin[v], v);
      atomicMin(&w.tmin[w.ia[v]], v);
      atomicMin(&w.tmin[w.ib[v]], v);
    }
    __syncthreads();
    int open = 0;
    for (int k = threadIdx.x; k < nvalid; k += blockDim.x) {
      if (w.ic[k] != 0) continue;
      const int v = w.lst[k], u = w.ia[v], x2 = w.ib[v];
      if (((volatile uint8_t*)w.flag)[v] | ((volatile uint8_t*)w.flag)[u] |
          ((volatile uint8_t*)w.flag)[x2]) {
        w.ic[k] = 2;  // meets an applied triangle's removed vertex
      } else if (w.tmin[v] == v && w.tmin[u] == v && w.tmin[x2] == v) {
        w.ic[k] = 1;
        w.flag[u] = 1;
        w.flag[x2] = 1;
        const int at = atomicAdd(&w.bs->bc[9], 2);
        rem[at] = u;
        rem[at + 1] = x2;
      } else {
        open = 1;
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nvalid; k += blockDim.x) {
      const int v = w.lst[k];
      w.tmin[v] = kInf;
      w.tmin[w.ia[v]] = kInf;
      w.tmin[w.ib[v]] = kInf;
    }
    if (!__syncthreads_or(open)) break;
  }
  const int total = w.bs->bc[9];
  int edges = remove_list_fast(w, rem, total);
  return PassRet{total / 2, total, edges, 0};
}

// Triangle sweep for the parallel search: every valid candidate v (degree
// 2, neighbours u, x adjacent) claims its closed triangle {v, u, x} with
// atomicMin on tmin; v applies iff it holds all three claims.  Applied
// triangles are vertex-disjoint, so applying them together is sound (a
// removal can only invalidate a candidate whose closed triangle it
// touches); the minimum valid candidate always applies, and the rest are
// revisited by the fixpoint's next sweep.  A different (but sound) choice
// than the reference's in-order walk, so only the parallel mode uses it:
// answers are the same, rule counts may differ.
template <typename T>
__device__ PassRet degree_two_triangle_pass_par(const NodeWs<T>& w, int b, int e, int* rem) {
  VCG_HB(w.bs, 107);
  int nvalid = 0;
  for (int v = b; v < e; ++v) {
    if (w.deg[v] == 2) {
      int u = -1, x2 = -1;
      for (int i = w.off[v]; i < w.off[v + 1]; ++i) {
        int x = w.nbr[i];
        if (w.deg[x] > 0) {
          if (u < 0) {
            u = x;
          } else {
            x2 = x;
            break;
          }
        }
      }
      if (x2 >= 0 && adjacent_static(w, u, x2)) {
        w.ia[v] = u;
        w.ib[v] = x2;
        w.lst[atomicAdd(&w.bs->bc[8], 1)] = v;
        atomicMin(&w.tmin[v], v);
        atomicMin(&w.tmin[u], v);
        atomicMin(&w.tmin[x2], v);
        ++nvalid;
      }
    }
  }
  nvalid = block_sum(nvalid, w.bs);
  if (nvalid == 0) return PassRet{0, 0, 0, 0};
  for (int k = threadIdx.x; k < nvalid; k += blockDim.x) {
    const int v = w.lst[k], u = w.ia[v], x2 = w.ib[v];
    if (w.tmin[v] == v && w.tmin[u] == v && w.tmin[x2] == v) {
      w.flag[u] = 1;
      w.flag[x2] = 1;
      const int at = atomicAdd(&w.bs->bc[9], 2);
      rem[at] = u;
      rem[at + 1] = x2;
    }
  }
  __syncthreads();
  const int total = w.bs->bc[9];
  for (int k = threadIdx.x; k < nvalid; k += blockDim.x) {
    const int v = w.lst[k];
    w.tmin[v] = kInf;
    w.tmin[w.ia[v]] = kInf;
    w.tmin[w.ib[v]] = kInf;
  }
  int edges = remove_list_fast(w, rem, total);
  return PassRet{total / 2, total, edges, 0};
}

// reduce_fixpoint (pure.py:188) for the search: identical forced sets and
// counters; one fused scan decides which sweeps have candidates.
template <typename T>
__device__ FixRet reduce_fixpoint_fast(const NodeWs<T>& w, int lo, int hi, int budget,
                                      long long* maxkey, bool par_tri = false) {
  FixRet r{0, 0, 0, 0, 0, lo, hi, 0};
  int b, e;
  my_chunk(lo, hi, &b, &e);
  int* rem = w.id;
  ScanStats st{};
  long long t0 = clock64();
  while (true) {
    int cycle = 0;
    while (true) {
      VCG_HB(w.bs, 101);
      const int bud = budget - r.forced;
      int t1 = 0, t2 = 0, th = 0, mn = kInf, mx = -1, dm = 0, dv = kInf;
      for (int v = b; v < e; ++v) {
        int d = w.deg[v];
        w.par[v] = v;  // union-find init for the component check that follows
        t1 += (d == 1);
        t2 += (d == 2);
        th += (d > 0 && d > bud);
        if (d > 0) {
          mn = min(mn, v);
          mx = v;
          if (d > dm) {  // ascending chunk: first maximum = lowest index
            dm = d;
            dv = v;
          }
        }
      }
      if (threadIdx.x == 0) {  // list cursors of the sweep that follows
        w.bs->bc[8] = 0;
        w.bs->bc[9] = 0;
        w.bs->bc[10] = 0;
      }
      st = block_scan_stats(t1, t2, th, mn, mx, dm, dv, w.bs);
      rprof(w.bs, 0, &t0);
      if (bud > kSpecBudget / 2 && threadIdx.x == 0 && st.key >= 0) {
        const int m = (int)(st.key >> 32) + (kSpecBudget - bud);
        if (m > w.bs->spec_m) w.bs->spec_m = m;
      }
      if (st.c1 == 0) break;
      PassRet a = degree_one_pass_fast(w, b, e, st.c1, rem);
      rprof(w.bs, 1, &t0);
      if (((volatile int*)w.bs->bc)[10]) {  // corrupted node state: give up on it
        r.pos = -1;
        *maxkey = -1;
        return r;
      }
      r.d1 += a.applied;
      r.forced += a.forced;
      r.edges += a.edges;
      cycle += a.applied;
    }
    int tri = 0;
    if (st.c2 > 0) {
      PassRet t = par_tri ? degree_two_triangle_pass_par(w, b, e, rem)
                          : degree_two_triangle_pass_lfmis(w, b, e, rem);
      rprof(w.bs, 2, &t0);
      tri = t.applied;
      r.d2t += t.applied;
      r.forced += t.forced;
      r.edges += t.edges;
      cycle += t.applied;
    }
    if (tri > 0 || st.ch > 0) {
      // the last scan's maximum degree bounds every degree now (degrees only
      // fall): if it is within the budget the sweep could force nothing
      const int bud_now = budget - r.forced;
      const int dmax_ub = st.key >= 0 ? (int)(st.key >> 32) : 0;
      if (st.ch == 0 && dmax_ub <= bud_now) {
        if (bud_now > kSpecBudget / 2 && threadIdx.x == 0 &&
            dmax_ub + (kSpecBudget - bud_now) > w.bs->spec_m)
          w.bs->spec_m = dmax_ub + (kSpecBudget - bud_now);  // speculative-budget record
      } else {
        PassRet h = high_degree_pass(w, lo, hi, bud_now, rem, 0);
        rprof(w.bs, 3, &t0);
        r.hd += h.applied;
        r.forced += h.forced;
        r.edges += h.edges;
        cycle += h.applied;
      }
    }
    if (cycle == 0) break;
  }
  // nothing changed since the last scan: its window and max-degree key are final
  if (st.hi < 0) {  // pure.py:238 empty window
    r.lo = w.n > 1 ? w.n : 1;
    r.hi = 0;
  } else {
    r.lo = st.lo;
    r.hi = st.hi;
  }
  *maxkey = st.key;
  return r;
}

// remove_neighbors (pure.py:47) for the search: forced set and counters only
template <typename T>
__device__ void remove_neighbors_fast(const NodeWs<T>& w, int v, int* rem, int* removed,
                                      int* edges) {
  if (threadIdx.x == 0) w.bs->bc[8] = 0;
  VCG_HB(w.bs, 106);
  __syncthreads();
  for (int j = w.off[v] + threadIdx.x; j < w.off[v + 1]; j += blockDim.x) {
    int x = w.nbr[j];
    if (w.deg[x] > 0) {
      w.flag[x] = 1;
      rem[atomicAdd(&w.bs->bc[8], 1)] = x;
    }
  }
  __syncthreads();
  const int total = w.bs->bc[8];
  *edges = remove_list_fast(w, rem, total);
  *removed = total;
}

// ---------------------------------------------------------------------------
// connected components of the live subgraph (union-find in the workspace)
// ---------------------------------------------------------------------------

__device__ __forceinline__ int uf_find(int* par, int x) {
  int p = ((volatile int*)par)[x];
  unsigned guard = 0;
  while (p != x) {
    if (++guard > (1u << 24)) __trap();  // a cycle in the forest: protocol bug
    int gp = ((volatile int*)par)[p];
    if (gp != p) ((volatile int*)par)[x] = gp;  // path halving, benign race
    x = p;
    p = gp;
  }
  return x;
}

// Labels every live vertex in [lo, hi] with its component's minimum vertex
// (par[v]) and returns the number of components.
// `inited`: par[v] == v already holds on [lo, hi] (the fixpoint's scan sets it).
//
// Min-label hooking with shortcutting (FastSV): per round every live edge
// (u, x) hooks the larger of its endpoints' grandparents under the smaller
// (atomicMin), then every vertex jumps to its grandparent.  Labels only
// decrease and stay inside the component (par[v] <= v), so at the round
// without change every vertex points at a root and both ends of every edge
// share it: the root is the component minimum.  O(log diameter) rounds --
// the earlier union-find hooked ordered paths into chains whose finds walked
// them (42 us to label the 1113-vertex root of rgg2000, now a few us).
template <typename T>
__device__ int label_components(const NodeWs<T>& w, int lo, int hi, bool inited = false) {
  VCG_HB(w.bs, 110);
  volatile int* par = w.par;
  if (!inited) {
    for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x) par[v] = v;
    __syncthreads();
  }
  const int m = (lo <= hi && w.deg[lo] > 0) ? lo : -1;
  while (true) {
    int changed = 0;
    for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x) {
      if (w.deg[v] == 0) continue;
      for (int j = w.off[v]; j < w.off[v + 1]; ++j) {
        const int x = w.nbr[j];
        if (x <= v || w.deg[x] == 0) continue;
        const int pu = par[v], px = par[x];
        const int gu = par[pu], gx = par[px];
        if (gu < gx) {
          atomicMin((int*)&par[px], gu);
          changed = 1;
        } else if (gx < gu) {
          atomicMin((int*)&par[pu], gx);
          changed = 1;
        }
      }
    }
    __syncthreads();
    // every live vertex already labelled with the window's first (= minimum)
    // live vertex: one component, no verification round needed
    int stray = 0;
    for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x) {
      if (w.deg[v] == 0) continue;
      const int p = par[v];
      const int gp = par[p];
      if (gp < p) {
        par[v] = gp;
        changed = 1;
      }
      stray |= (gp < p ? gp : p) != m;
    }
    VCG_HB(w.bs, 111);
    if (m >= 0 && !__syncthreads_or(stray)) return 1;
    if (!__syncthreads_or(changed)) break;
  }
  VCG_HB(w.bs, 112);
  int roots = 0;
  for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x)
    if (w.deg[v] > 0 && par[v] == v) ++roots;
  return block_sum(roots, w.bs);
}

// full path compression: par[v] = component minimum for every live v.
// Two phases: finds (with path halving, which only ever shortcuts to an
// ancestor, so every find still returns the root) into w.ia, a barrier,
// then the writes.  Writing par[v] = root in the same phase races: a
// concurrent find's halving store (par[x] = grandparent) can land after x's
// owner wrote the root and leave par[x] at a non-root ancestor, mislabelling
// x (observed as lost degrees in component children with the workspace in
// HBM, where the window is wide).
template <typename T>
__device__ void compress_labels(const NodeWs<T>& w, int lo, int hi) {
  VCG_HB(w.bs, 113);
  for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x)
    if (w.deg[v] > 0) w.ia[v] = uf_find(w.par, v);
  __syncthreads();
  for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x)
    if (w.deg[v] > 0) w.par[v] = w.ia[v];
  __syncthreads();
}

struct CompInfo {
  int size, degsum, mindeg, maxdeg, vmin, vmax;
};

// After label_components with ncomp > 1: component j (in increasing order of
// its minimum vertex, i.e. the reference's discovery order) gets
//   root lst[j], size ib[j], degsum ic[j], mindeg tmp..., see below.
// Uses ia (labels), id (root -> ordinal), lst (ordinal -> root) and packs the
// four aggregates into ib/ic (size, degsum) and two halves of tmin-free arrays.
// Aggregates are written to agg[5*ncomp] (caller-provided int scratch).
template <typename T>
__device__ void component_aggregates(const NodeWs<T>& w, int lo, int hi, int ncomp, int* agg) {
  VCG_HB(w.bs, 114);
  int b, e;
  my_chunk(lo, hi, &b, &e);
  int cnt = 0;
  for (int v = b; v < e; ++v) cnt += (w.deg[v] > 0 && w.par[v] == v);
  int tot;
  int at = block_exscan(cnt, w.bs, &tot);
  for (int v = b; v < e; ++v) {
    if (w.deg[v] > 0 && w.par[v] == v) {
      w.lst[at] = v;
      w.id[v] = at;
      ++at;
    }
  }
  for (int j = threadIdx.x; j < ncomp; j += blockDim.x) {
    agg[5 * j + 0] = 0;
    agg[5 * j + 1] = 0;
    agg[5 * j + 2] = kInf;
    agg[5 * j + 3] = 0;
    agg[5 * j + 4] = 0;
  }
  __syncthreads();
  for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x) {
    int d = w.deg[v];
    if (d > 0) {
      int j = w.id[w.par[v]];
      atomicAdd(&agg[5 * j + 0], 1);
      atomicAdd(&agg[5 * j + 1], d);
      atomicMin(&agg[5 * j + 2], d);
      atomicMax(&agg[5 * j + 3], d);
      atomicMax(&agg[5 * j + 4], v);
    }
  }
  __syncthreads();
}

}  // namespace vcg
