// Grid-wide root fixpoint (preprocess.py:77 root_reduce -> reductions.py:110
// reduce_to_fixpoint -> kernels/pure.py:188 reduce_fixpoint) for graphs whose
// workspace does not fit one SM's shared memory.
//
// One cooperative launch, every SM resident, runs the whole joint fixpoint of
// the degree-one / degree-two-triangle / high-degree rules on int32 degrees in
// HBM, with grid-wide barriers between the phases of each sweep.  Each thread
// owns a contiguous chunk of vertex ids (index order is preserved across
// threads and blocks), so a sweep's forced vertices are emitted in the
// reference's order with one grid-wide exclusive scan: the forced list is
// identical to the sequential restatement's, id for id, not just as a set.
//
// Sweep semantics (exact, see node_ops.cuh for the derivations):
//  * degree-one (pure.py:82): candidate v (deg 1, unique live neighbour u(v))
//    applies iff v is the lowest-index candidate targeting u(v) and not the
//    higher end of an isolated edge whose lower end is also a candidate;
//    the applied targets are removed together.  3 barriers per sweep.
//  * triangle (pure.py:113): valid candidates resolved as the
//    lexicographically-first maximal independent set of their closed
//    triangles, in claim rounds (atomicMin on tmin), 3 barriers per round.
//  * high-degree (pure.py:158): in-order, budget-dependent -- block 0 runs the
//    block-level sweep on the same HBM workspace (rare at the root: the MVC
//    solve path runs it with the speculative budget under which it cannot
//    fire; only PVC bounds reach it).
// Control flow (which sweeps run, the skip of a high-degree sweep that can
// force nothing, the speculative-budget record) is reduce_fixpoint_fast's.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "root_grid.cuh"
#include "search.cuh"

namespace cg = cooperative_groups;

namespace vcg {

namespace {

struct Slot {  // grid-wide result of one scan (triple-buffered by scan index)
  int c1, c2, ch, mn, mx, nvalid, pad0, pad1;
  unsigned long long key;  // (dmax << 32) | (INT_MAX - lowest index of dmax)
};

struct GridCtl {
  Slot slot[3];
  int open[3];            // triangle claim rounds: undecided candidates left
  int hd[4];              // block 0 -> all: high-degree applied, edges, pos
  unsigned long long edges;
  int error;
  int spec_m;
  int partial[kRootGridMaxBlocks];  // per-block counts of an ordered emission
};

__device__ __forceinline__ Slot load_slot(const Slot* p) {
  const volatile Slot* q = p;
  Slot s;
  s.c1 = q->c1;
  s.c2 = q->c2;
  s.ch = q->ch;
  s.mn = q->mn;
  s.mx = q->mx;
  s.nvalid = q->nvalid;
  s.pad0 = s.pad1 = 0;
  s.key = q->key;
  return s;
}

__device__ __forceinline__ void grid_chunk(int n, int* b, int* e) {
  const long long T = (long long)gridDim.x * blockDim.x;
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (n + T - 1) / T;
  long long s = gt * per, t = s + per;
  if (s > n) s = n;
  if (t > n) t = n;
  *b = (int)s;
  *e = (int)t;
}

// sum of partial[0, blockIdx.x) and of all partials (every thread gets both)
__device__ __forceinline__ void block_base(const volatile int* partial, int* base, int* total,
                                           BlockScratch* bs) {
  if (threadIdx.x < 32) {
    int before = 0, tot = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) {
      const int p = partial[i];
      tot += p;
      if (i < (int)blockIdx.x) before += p;
    }
    before = __reduce_add_sync(0xffffffffu, before);
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (threadIdx.x == 0) {
      bs->bc[12] = before;
      bs->bc[13] = tot;
    }
  }
  __syncthreads();
  *base = bs->bc[12];
  *total = bs->bc[13];
  __syncthreads();
}

// removal of u, a member of the set being removed together (flag == 1):
// live neighbours outside the set lose one degree; an edge inside the set
// is counted once (at its lower end)
__device__ __forceinline__ int remove_member(const NodeWs<uint32_t>& w, int u) {
  int e = 0;
  for (int i = w.off[u]; i < w.off[u + 1]; ++i) {
    const int x = w.nbr[i];
    if (((volatile uint8_t*)w.flag)[x] == 1) {
      if (x > u) ++e;
    } else if (ldv(w.deg, x) > 0) {
      atomicSub((unsigned*)(w.deg + x), 1u);
      ++e;
    }
  }
  return e;
}

}  // namespace

__global__ void __launch_bounds__(kRootGridThreads)
    k_root_grid(int n, const int32_t* off, const int32_t* nbr, char* wsmem, int budget,
                int32_t* out, long long* ret, int init, void* ctl_mem) {
  cg::grid_group grid = cg::this_grid();
  __shared__ BlockScratch bs;
  init_block_scratch(&bs);
  GridCtl* G = (GridCtl*)ctl_mem;
  NodeWs<uint32_t> w = carve_ws<uint32_t>(wsmem, n, &bs, off, nbr);
  int b, e;
  grid_chunk(n, &b, &e);
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;

  for (int v = b; v < e; ++v) {
    if (init) w.deg[v] = (uint32_t)(off[v + 1] - off[v]);
    w.tmin[v] = kInf;
    w.flag[v] = 0;
    w.ic[v] = 0;
  }
  if (leader) {
    for (int s = 0; s < 3; ++s) {
      G->slot[s] = Slot{0, 0, 0, kInf, -1, 0, 0, 0, 0ull};
      G->open[s] = 0;
    }
    G->edges = 0ull;
    G->error = 0;
    G->spec_m = -1;
  }
  grid.sync();

  int forced = 0, d1 = 0, d2t = 0, hd = 0, pos = 0;
  int clear_lo = 0, clear_hi = 0;  // forced ids whose removal flags are still set
  int scan = 0;                    // scans so far (slot rotation)
  Slot st{};
  int spec_m = -1;
  while (true) {
    int cycle = 0;
    // ---- degree-one sweeps to exhaustion; the last scan describes the state
    while (true) {
      const int bud = budget - forced;
      Slot* S = &G->slot[scan % 3];
      if (leader) G->slot[(scan + 2) % 3] = Slot{0, 0, 0, kInf, -1, 0, 0, 0, 0ull};
      for (int k = clear_lo + (int)(blockIdx.x * blockDim.x + threadIdx.x); k < clear_hi;
           k += gridDim.x * blockDim.x)
        w.flag[out[k]] = 0;
      clear_lo = clear_hi = pos;
      int t1 = 0, t2 = 0, th = 0, mn = kInf, mx = -1, dm = 0, dv = kInf;
      for (int v = b; v < e; ++v) {
        const int d = (int)w.deg[v];
        t2 += (d == 2);
        th += (d > 0 && d > bud);
        if (d > 0) {
          mn = min(mn, v);
          mx = v;
          if (d > dm) {
            dm = d;
            dv = v;
          }
        }
        if (d == 1) {
          int u = -1;
          for (int i = off[v]; i < off[v + 1]; ++i) {
            const int x = nbr[i];
            if (w.deg[x] > 0) {
              u = x;
              break;
            }
          }
          if (u < 0) {  // inconsistent degree array: report, never loop
            atomicExch(&G->error, 1);
            continue;
          }
          ++t1;
          w.ia[v] = u;
          atomicMin(&w.tmin[u], v);
        }
      }
      {
        int vals[6] = {t1, t2, th, mn, mx, dm};
        const int op[6] = {0, 0, 0, 1, 2, 2};
        block_reduce<6>(vals, op, &bs);
        int lv[1] = {dm == vals[5] ? dv : kInf};
        const int op1[1] = {1};
        block_reduce<1>(lv, op1, &bs);
        if (threadIdx.x == 0) {
          if (vals[0]) atomicAdd(&S->c1, vals[0]);
          if (vals[1]) atomicAdd(&S->c2, vals[1]);
          if (vals[2]) atomicAdd(&S->ch, vals[2]);
          if (vals[3] != kInf) atomicMin(&S->mn, vals[3]);
          if (vals[4] >= 0) atomicMax(&S->mx, vals[4]);
          if (vals[5] > 0)
            atomicMax(&S->key, ((unsigned long long)vals[5] << 32) |
                                   (unsigned long long)(unsigned)(0x7fffffff - lv[0]));
        }
      }
      grid.sync();
      ++scan;
      st = load_slot(S);
      if (bud > kSpecBudget / 2 && st.key) {
        const int m = (int)(st.key >> 32) + (kSpecBudget - bud);
        spec_m = max(spec_m, m);
      }
      if (*(volatile int*)&G->error) break;
      if (st.c1 == 0) break;
      // decide in candidate order; count this thread's applications
      int cnt = 0;
      for (int v = b; v < e; ++v) {
        if (w.deg[v] != 1) continue;
        const int u = w.ia[v];
        const bool app = (w.tmin[u] == v) && !(w.deg[u] == 1 && w.ia[u] == v && u < v);
        w.ic[v] = app ? 2 : 1;
        if (app) {
          w.flag[u] = 1;
          ++cnt;
        }
      }
      int btot;
      const int at = block_exscan(cnt, &bs, &btot);
      if (threadIdx.x == 0) G->partial[blockIdx.x] = btot;
      grid.sync();
      int base, total;
      block_base(G->partial, &base, &total, &bs);
      int o = pos + base + at, edges = 0;
      for (int v = b; v < e; ++v) {
        const int c = w.ic[v];
        if (!c) continue;
        const int u = w.ia[v];
        w.tmin[u] = kInf;
        w.ic[v] = 0;
        if (c == 2) {
          out[o++] = u;
          edges += remove_member(w, u);
          w.deg[u] = 0;
        }
      }
      edges = block_sum(edges, &bs);
      if (threadIdx.x == 0 && edges) atomicAdd(&G->edges, (unsigned long long)edges);
      clear_lo = pos;
      pos += total;
      clear_hi = pos;
      forced += total;
      d1 += total;
      cycle += total;
      grid.sync();
    }
    if (*(volatile int*)&G->error) break;
    // ---- one triangle sweep
    int tri = 0;
    if (st.c2 > 0) {
      Slot* S = &G->slot[scan % 3];  // zeroed two scans ago: holds nvalid
      for (int v = b; v < e; ++v) {
        if (w.deg[v] != 2) continue;
        int u = -1, x2 = -1;
        for (int i = off[v]; i < off[v + 1]; ++i) {
          const int x = nbr[i];
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
          w.ic[v] = 3;  // undecided
          w.lst[atomicAdd(&S->nvalid, 1)] = v;
        }
      }
      grid.sync();
      const int nvalid = *(volatile int*)&S->nvalid;
      if (leader) G->slot[(scan + 2) % 3] = Slot{0, 0, 0, kInf, -1, 0, 0, 0, 0ull};
      ++scan;
      if (nvalid > 0) {
        const int gt = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
        for (int round = 0;; ++round) {
          int* open = &G->open[round % 3];
          if (leader) G->open[(round + 2) % 3] = 0;
          for (int k = gt; k < nvalid; k += T) {
            const int v = w.lst[k];
            if (w.ic[v] != 3) continue;
            atomicMin(&w.tmin[v], v);
            atomicMin(&w.tmin[w.ia[v]], v);
            atomicMin(&w.tmin[w.ib[v]], v);
          }
          grid.sync();
          int still = 0;
          for (int k = gt; k < nvalid; k += T) {
            const int v = w.lst[k];
            if (w.ic[v] != 3) continue;
            const int u = w.ia[v], x2 = w.ib[v];
            const volatile uint8_t* fl = w.flag;
            if (fl[v] | fl[u] | fl[x2]) {
              w.ic[v] = 4;  // meets an applied triangle's removed vertex: out
            } else if (w.tmin[v] == v && w.tmin[u] == v && w.tmin[x2] == v) {
              w.ic[v] = 5;  // in
              w.flag[u] = 1;
              w.flag[x2] = 1;
            } else {
              still = 1;
            }
          }
          if (__syncthreads_or(still) && threadIdx.x == 0) atomicOr(open, 1);
          grid.sync();
          for (int k = gt; k < nvalid; k += T) {
            const int v = w.lst[k];
            w.tmin[v] = kInf;
            w.tmin[w.ia[v]] = kInf;
            w.tmin[w.ib[v]] = kInf;
          }
          const int more = *(volatile int*)open;
          grid.sync();
          if (!more) break;
        }
        // ordered emission (u then x per applied candidate, in index order)
        int cnt = 0;
        for (int v = b; v < e; ++v) cnt += (w.ic[v] == 5) ? 2 : 0;
        int btot;
        const int at = block_exscan(cnt, &bs, &btot);
        if (threadIdx.x == 0) G->partial[blockIdx.x] = btot;
        grid.sync();
        int base, total;
        block_base(G->partial, &base, &total, &bs);
        int o = pos + base + at, edges = 0;
        for (int v = b; v < e; ++v) {
          const int c = w.ic[v];
          if (!c) continue;
          w.ic[v] = 0;
          if (c == 5) {
            const int u = w.ia[v], x2 = w.ib[v];
            out[o++] = u;
            out[o++] = x2;
            edges += remove_member(w, u) + remove_member(w, x2);
          }
        }
        edges = block_sum(edges, &bs);
        if (threadIdx.x == 0 && edges) atomicAdd(&G->edges, (unsigned long long)edges);
        grid.sync();
        // zero the removed entries once every remover is done reading flags
        for (int k = pos + gt; k < pos + total; k += T) {
          w.deg[out[k]] = 0;
          w.flag[out[k]] = 0;
        }
        tri = total / 2;
        pos += total;
        forced += total;
        d2t += tri;
        cycle += tri;
        clear_lo = clear_hi = pos;
        grid.sync();
      }
    }
    // ---- high-degree sweep (reduce_fixpoint_fast's skip of a sweep that
    // can force nothing; speculative-budget record)
    if (tri > 0 || st.ch > 0) {
      const int bud_now = budget - forced;
      const int dmax_ub = st.key ? (int)(st.key >> 32) : 0;
      if (st.ch == 0 && dmax_ub <= bud_now) {
        if (bud_now > kSpecBudget / 2) spec_m = max(spec_m, dmax_ub + (kSpecBudget - bud_now));
      } else {
        if (blockIdx.x == 0) {
          for (int k = clear_lo + (int)threadIdx.x; k < clear_hi; k += blockDim.x)
            w.flag[out[k]] = 0;
          __syncthreads();
          PassRet h = high_degree_pass(w, 0, n - 1, bud_now, out, pos);
          if (threadIdx.x == 0) {
            G->hd[0] = h.applied;
            G->hd[1] = h.edges;
            G->hd[2] = h.pos;
            if (bs.spec_m > G->spec_m) G->spec_m = bs.spec_m;
          }
        }
        grid.sync();
        const int applied = *(volatile int*)&G->hd[0];
        if (leader) G->edges += (unsigned long long)*(volatile int*)&G->hd[1];
        pos = *(volatile int*)&G->hd[2];
        clear_lo = clear_hi = pos;
        hd += applied;
        forced += applied;
        cycle += applied;
        // the block-level sweep used ic[0, candidates) as scratch
        for (int v = b; v < e; ++v) w.ic[v] = 0;
        grid.sync();
      }
    }
    if (cycle == 0) break;
  }
  if (leader) {
    const int err = *(volatile int*)&G->error;
    const int sm = max(spec_m, *(volatile int*)&G->spec_m);
    ret[0] = forced;
    ret[1] = d1;
    ret[2] = d2t;
    ret[3] = hd;
    ret[4] = (long long)*(volatile unsigned long long*)&G->edges;
    if (st.mx < 0) {  // pure.py:238 empty window
      ret[5] = n > 1 ? n : 1;
      ret[6] = 0;
    } else {
      ret[5] = st.mn;
      ret[6] = st.mx;
    }
    ret[7] = pos;
    ret[8] = err;
    ret[9] = sm;
    ret[10] = scan;
  }
  // leave the workspace's invariants for the next round (flags clear)
  for (int k = clear_lo + (int)(blockIdx.x * blockDim.x + threadIdx.x); k < clear_hi;
       k += gridDim.x * blockDim.x)
    w.flag[out[k]] = 0;
}

size_t root_grid_ctl_bytes() { return sizeof(GridCtl); }

int root_grid_blocks() {
  static thread_local int dev_cached = -1, blocks = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev != dev_cached) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_root_grid, kRootGridThreads, 0);
    per_sm = per_sm > 2 ? 2 : per_sm;
    blocks = sms * per_sm;
    if (blocks > kRootGridMaxBlocks) blocks = kRootGridMaxBlocks;
    dev_cached = dev;
  }
  return blocks;
}

cudaError_t root_grid_launch(int n, const int32_t* off, const int32_t* nbr, char* ws, int budget,
                             int32_t* out, long long* ret, int init, void* ctl) {
  const int blocks = root_grid_blocks();
  if (blocks < 1) return cudaErrorInvalidConfiguration;
  void* args[] = {&n, &off, &nbr, &ws, &budget, &out, &ret, &init, &ctl};
  return cudaLaunchCooperativeKernel((const void*)k_root_grid, dim3(blocks),
                                     dim3(kRootGridThreads), args, 0, cudaStreamPerThread);
}

}  // namespace vcg
