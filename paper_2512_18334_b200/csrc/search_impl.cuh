// Persistent search kernel (template definition): one resident block per
// worker, one search node per block at a time.  See search.cuh for the
// coordination structures and node_ops.cuh for the exact-semantics
// block-parallel node operations.  Instantiated by search.cu (warp tasks of
// <= 64 vertices), search_w2.cu (<= 128) and search_w4.cu (<= 256): each
// variant compiles only its own warp-tier widths, so the wider tiers' code
// and registers never weigh on the sparse workloads' kernel.
#pragma once

#include "search.cuh"
#include "warp_solve.cuh"

#ifndef VCG_SEARCH_MAXT
#define VCG_SEARCH_MAXT 512
#endif
#ifndef VCG_SEARCH_MINB
#define VCG_SEARCH_MINB 2
#endif

namespace vcg {

struct BlockState {
  NodeHdr hdr;   // current node
  int best_s;    // scope best snapshot at node start
  int qpos_lo, qpos_hi;
  int flag;
  int gen;       // number of general components in a split
  int parent;
  int child_base;
  int v;
  int emitted;   // the node went to the warp tier
};

template <typename T>
struct Worker {
  const SearchParams& P;
  NodeWs<T> w;
  BlockState* st;
  char* my_stack;
  int top;   // block-uniform private stack height
  // thread-0 statistics
  unsigned long long nodes, comp_branches, pushes, pops, rules[6], rec_in, rec_out;
  int max_depth;
  LiveBatch lb;  // thread 0
  long long payload;  // bytes of a record after its header: deg (+ inclusion bitset)
  unsigned long long ph[10];
  long long last_clk;
  unsigned long long wep;  // thread 0: cycles in warp-tier epochs that ran tasks
  int* gl;           // per-warp local -> reduced id scratch for task packing
  int gl_stride;     // ints per warp (the variant's task limit)
  int cur_graph;     // graph of the node in the workspace (0: the reduced graph)
  int* soff;         // shared-memory CSR region (null: the CSR is read from HBM/L2)
  int* snbr;
  long long extra;   // record-cover bitset bytes after the degree array

  __device__ void tick(int phase) {
    VCG_HB(w.bs, phase);
    if (threadIdx.x == 0) {
      long long now = clock64();
      ph[phase] += (unsigned long long)(now - last_clk);
      last_clk = now;
    }
  }

  __device__ Worker(const SearchParams& p, NodeWs<T> ws, BlockState* s)
      : P(p), w(ws), st(s), top(0), nodes(0), comp_branches(0), pushes(0), pops(0), rec_in(0),
        rec_out(0), max_depth(0), wep(0) {
    for (int i = 0; i < 6; ++i) rules[i] = 0;
    for (int i = 0; i < 10; ++i) ph[i] = 0;
    last_clk = clock64();
    extra = P.record ? bits_bytes(P.n) : 0;
    payload = deg_bytes<T>(P.n) + extra;
    cur_graph = 0;
    soff = snbr = nullptr;
    lb.enabled = P.batch_live;
    my_stack = P.stacks + (long long)blockIdx.x * P.stack_cap * P.slot_bytes;
  }

  // ------------------------------------------------------- warp tasks --
  // One warp (all lanes) packs the live vertices of the current node in
  // [lo, hi] that belong to component `root` (root < 0: all of them) --
  // `size` of them, <= kWMax -- into a warp-tier task: local ids follow the
  // reduced graph's order (so lowest-index tie-breaks are unchanged), rows
  // are adjacency bitmasks.  Returns false when the task ring is full.
  __device__ bool emit_task(int root, int size, int lo, int hi, int scope, int S, int depth,
                            int counted, long long ticket = -1) {
    const int lane = threadIdx.x & 31;
    int* gv = gl + (threadIdx.x >> 5) * gl_stride;
    long long pos = -1;
    if (lane == 0) {
      if (ticket >= 0) {
        q_wait_free(P.bq, ticket);
        pos = ticket;
      } else {
        pos = q_reserve_push(P.bq, P.bq.cap);
      }
    }
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (pos < 0) return false;
    char* slot = P.bq.data + (pos % P.bq.cap) * P.bq_slot;
    int base = 0;
    for (int c0 = lo; c0 <= hi && base < size; c0 += 32) {
      const int v = c0 + lane;
      const bool in = v <= hi && w.deg[v] > 0 && (root < 0 || w.par[v] == root);
      const unsigned m = __ballot_sync(0xffffffffu, in);
      const int li = base + __popc(m & ((1u << lane) - 1u));
      if (in && li < gl_stride) {
        w.ia[v] = li;
        gv[li] = v;
      }
      base += __popc(m);
    }
    __syncwarp();
    unsigned long long* adj = (unsigned long long*)(slot + kWHdrBytes);
    const int W = wrows(size);  // 64-bit words per row
    for (int i = lane; i < size; i += 32) {
      const int v = gv[i];
      // four named words, not an indexed array (which would live in local memory)
      unsigned long long mk0 = 0ull, mk1 = 0ull, mk2 = 0ull, mk3 = 0ull;
      for (int k = w.off[v]; k < w.off[v + 1]; ++k) {
        const int x = w.nbr[k];
        if (w.deg[x] > 0) {
          const int b = w.ia[x];
          const unsigned long long bit = 1ull << (b & 63);
          const int wi = b >> 6;
          mk0 |= wi == 0 ? bit : 0ull;
          mk1 |= wi == 1 ? bit : 0ull;
          mk2 |= wi == 2 ? bit : 0ull;
          mk3 |= wi == 3 ? bit : 0ull;
        }
      }
      __stcg(adj + W * i, mk0);
      if (W > 1) __stcg(adj + W * i + 1, mk1);
      if (W > 2) {
        __stcg(adj + W * i + 2, mk2);
        __stcg(adj + W * i + 3, mk3);
      }
    }
    if (lane == 0) {
      __stcg((int4*)slot, make_int4(S, scope, size | (counted << 16), depth));
      unsigned long long lv[4];
      for (int j = 0; j < 4; ++j) {
        const int r = size - 64 * j;
        lv[j] = r >= 64 ? ~0ull : r > 0 ? ((1ull << r) - 1) : 0ull;
      }
      __stcg((ulonglong2*)(slot + 16), make_ulonglong2(lv[0], lv[1]));
      if (W > 2) __stcg((ulonglong2*)(adj + size * W), make_ulonglong2(lv[2], lv[3]));
    }
    __syncwarp();
    if (lane == 0) q_publish_push(P.bq, pos);
    return true;
  }

  // Make `graph` (gn vertices) the workspace's graph: restage its CSR in
  // shared memory (every subgraph is smaller than the reduced graph, so it
  // fits the region) or point at it.  All threads, block-uniform arguments.
  __device__ void set_graph(int graph, int gn) {
    if (graph == cur_graph) return;
    const int* goff = P.off;
    const int* gnbr = P.nbr;
    long long m2 = P.m2;
    if (graph) {
      goff = P.arena + __ldcg(&P.sg_base[graph - 1]);
      gnbr = goff + ((gn + 1 + 3) & ~3);
      m2 = __ldcg(goff + gn);
    }
    if (soff) {
      for (int i = threadIdx.x; i <= gn; i += blockDim.x) soff[i] = __ldcg(goff + i);
      for (long long i = threadIdx.x; i < m2; i += blockDim.x) snbr[i] = __ldcg(gnbr + i);
      __syncthreads();
    } else {
      w.off = goff;
      w.nbr = gnbr;
    }
    w.n = gn;
    cur_graph = graph;
    payload = deg_bytes<T>(gn) + extra;
  }

  // Order-preserving compaction of component `root` of the current node
  // (size vertices, degree sum m2c, all in [lo, hi]) into a subgraph in the
  // arena: local ids follow the current graph's order, so every
  // lowest-index rule and tie-break of the reference is unchanged inside the
  // component, while the child's degree array, window and sweeps shrink
  // from the parent's span to the component (graph.py:99 induced_subgraph,
  // applied per component).  Writes the local degrees to dd[0, size).
  // Returns the subgraph's graph number (id + 1), 0 when the arena is full.
  __device__ int compact_component(int root, int size, int m2c, int lo, int hi, T* dd) {
    const int offw = (size + 1 + 3) & ~3;
    if (threadIdx.x == 0) {
      int g = -1;
      const long long words = (long long)offw + m2c;
      long long b = -1;
      // the arena is bump-allocated for the whole search; once it is full
      // (or the subgraph table is), components stay in the parent's graph.
      // Check before claiming: a counter advanced by every failed claim of a
      // long search would overflow int and alias live subgraphs.
      if (ld_relaxed(P.arena_top) + words <= (long long)P.arena_cap &&
          ld_relaxed(P.sg_count) < P.sg_cap) {
        b = atomicAdd(P.arena_top, (int)words);
        if (b + words <= (long long)P.arena_cap) {
          g = atomicAdd(P.sg_count, 1);
          if (g >= P.sg_cap) {
            g = -1;
          } else {
            P.sg_base[g] = (int)b;
            P.sg_n[g] = size;
          }
        }
      }
      st->v = g;
      st->child_base = (int)b;
    }
    __syncthreads();
    const int g = st->v;
    if (g < 0) return 0;
    int* goff = P.arena + st->child_base;
    int* gnbr = goff + offw;
    int b, e;
    my_chunk(lo, hi, &b, &e);
    int cnt = 0, dsum = 0;
    for (int v = b; v < e; ++v) {
      const int d = w.deg[v];
      if (d > 0 && w.par[v] == root) {
        ++cnt;
        dsum += d;
      }
    }
    int tot;
    int li = block_exscan(cnt, w.bs, &tot);
    int dp = block_exscan(dsum, w.bs, &tot);
    for (int v = b; v < e; ++v) {
      const int d = w.deg[v];
      if (d > 0 && w.par[v] == root) {
        w.ia[v] = li;
        dd[li] = (T)d;
        __stcg(goff + li, dp);
        ++li;
        dp += d;
      }
    }
    for (int i = size + threadIdx.x; i < (int)(deg_bytes<T>(size) / sizeof(T)); i += blockDim.x)
      dd[i] = 0;
    if (threadIdx.x == 0) __stcg(goff + size, m2c);
    __syncthreads();
    for (int v = b; v < e; ++v) {
      if (w.deg[v] > 0 && w.par[v] == root) {
        int k = __ldcg(goff + w.ia[v]);
        for (int j = w.off[v]; j < w.off[v + 1]; ++j) {
          const int x = w.nbr[j];
          if (w.deg[x] > 0) __stcg(gnbr + k++, w.ia[x]);
        }
      }
    }
    __syncthreads();
    return g + 1;
  }

  __device__ char* stack_slot(int i) const { return my_stack + (long long)i * P.slot_bytes; }
  __device__ char* queue_slot(long long pos) const {
    return P.q.data + (pos % P.q.cap) * P.slot_bytes;
  }

  // engine.py:413 _offload_or_push: pick where the next child record goes.
  // Returns the destination; *qpos >= 0 means a reserved worklist slot.
  __device__ char* choose_dest(long long* qpos) {
    VCG_HB(w.bs, 30);
    reserve_dest();
    return resolve_dest(qpos);
  }

  // choose_dest in two halves: thread 0 claims the worklist ticket (L2
  // atomics) without a barrier, so the claim overlaps the block's work up
  // to the next barrier; resolve_dest (all threads, after that barrier or
  // its own) reads the outcome.
  __device__ void reserve_dest() {
    if (threadIdx.x == 0) {
      long long pos = -1;
      if (P.share) pos = q_reserve_push(P.q, P.threshold);
      if (pos < 0 && top >= P.stack_cap) {
        // private stack full: the worklist must take it (SPEC offloadOrPush)
        unsigned spins = 0;
        while ((pos = q_reserve_push(P.q, P.q.cap)) < 0) {
          __nanosleep(256);
          if (++spins > (1u << 24)) {
            atomicExch(&P.ctl->error, 2);
            atomicExch(&P.ctl->stop, 1);
            break;
          }
        }
      }
      st->qpos_lo = (int)(pos & 0xffffffffLL);
      st->qpos_hi = (int)(pos >> 32);
    }
  }

  __device__ char* resolve_dest(long long* qpos) {
    VCG_HB(w.bs, 31);
    __syncthreads();
    VCG_HB(w.bs, 32);
    long long pos = ((long long)st->qpos_hi << 32) | (unsigned)st->qpos_lo;
    *qpos = pos;
    if (pos >= 0) return queue_slot(pos);
    if (top >= P.stack_cap) return nullptr;  // error path (stop set)
    return stack_slot(top);
  }

  __device__ void commit_dest(long long qpos, const NodeHdr& h, char* dst) {
    if (threadIdx.x == 0 && dst) {
      *(NodeHdr*)dst = h;
      ++rec_out;
    }
    __syncthreads();
    if (qpos >= 0) {
      if (threadIdx.x == 0) {
        q_publish_push(P.q, qpos);
        ++pushes;
      }
    } else if (dst) {
      ++top;
      if (threadIdx.x == 0 && top > max_depth) max_depth = top;
    }
  }

  // ------------------------------------------------------ record cover --
  // Witness of a split: arena record of the splitting node's scoped cover
  // plus closed-form covers of its clique (all but the root) and chordless
  // cycle (every other vertex) components; one record per general component
  // holding its all-but-one cover (the child's achieved initial bound).
  __device__ void record_split_witness(int ncomp, const int* agg, int parent) {
    const int G = st->gen;
    if (threadIdx.x == 0) {
      int wb = atomicAdd(P.wcount, 1 + G);
      if (wb + 1 + G > P.wcap) {
        atomicExch(&P.ctl->error, 4);
        atomicExch(&P.ctl->stop, 1);
        wb = -1;
      }
      st->child_base = wb;
    }
    __syncthreads();
    const int wb = st->child_base;
    if (wb < 0) return;
    unsigned* rec0 = P.wbits + (long long)wb * P.nw;
    for (int i = threadIdx.x; i < P.nw; i += blockDim.x) rec0[i] = w.inc[i];
    for (long long i = threadIdx.x; i < (long long)G * P.nw; i += blockDim.x) rec0[P.nw + i] = 0u;
    __syncthreads();
    const int lo = st->hdr.lo, hi = st->hdr.hi;
    for (int v = lo + threadIdx.x; v <= hi; v += blockDim.x) {
      if (w.deg[v] == 0) continue;
      const int j = w.id[w.par[v]];
      if (v == w.lst[j]) continue;  // the component root stays out
      const int mark = agg[5 * j + 2];
      unsigned* rec = nullptr;
      if (mark == -1) rec = rec0;
      else if (mark >= 0) rec = rec0 + (long long)(1 + (mark - parent - 1)) * P.nw;
      if (rec) atomicOr(&rec[v >> 5], 1u << (v & 31));
    }
    if (threadIdx.x == 0) {
      for (int j = 0; j < ncomp; ++j) {
        if (agg[5 * j + 2] != -2) continue;
        // chordless cycle: walk it, take positions 0, 2, 4, ... (ceil(L/2))
        const int L = agg[5 * j];
        int prev = -1, v = w.lst[j];
        for (int i = 0; i < L; ++i) {
          if ((i & 1) == 0) atomicOr(&rec0[v >> 5], 1u << (v & 31));
          int nxt = -1;
          for (int k = w.off[v]; k < w.off[v + 1]; ++k) {
            const int x = w.nbr[k];
            if (w.deg[x] > 0 && x != prev) {
              nxt = x;
              break;
            }
          }
          prev = v;
          v = nxt;
        }
      }
      P.reg.pwrec[parent] = wb;
      for (int j = 0; j < ncomp; ++j) {
        const int c = agg[5 * j + 2];
        if (c < 0) continue;
        const int key = P.reg.key[c];
        if (!(key & 1))  // achieved initial bound == all-but-one
          P.reg.wkey[c] = ((unsigned long long)(unsigned)(key >> 1) << 32) |
                          (unsigned)(wb + 1 + (c - parent - 1));
      }
      __threadfence();
    }
    __syncthreads();
  }

  // leaf in record mode: store the scoped cover if it improves the scope
  __device__ unsigned long long record_leaf_witness(int scope, int S) {
    if (threadIdx.x == 0) {
      const int key = ld_relaxed(&P.reg.key[scope]);
      int wid = -1;
      if (S * 2 < key) {
        wid = atomicAdd(P.wcount, 1);
        if (wid >= P.wcap) {
          atomicExch(&P.ctl->error, 4);
          atomicExch(&P.ctl->stop, 1);
          wid = -1;
        }
      }
      st->v = wid;
    }
    __syncthreads();
    const int wid = st->v;
    if (wid < 0) return kNoWitness;
    unsigned* rec = P.wbits + (long long)wid * P.nw;
    for (int i = threadIdx.x; i < P.nw; i += blockDim.x) rec[i] = w.inc[i];
    __syncthreads();
    if (threadIdx.x == 0) __threadfence();
    return (unsigned long long)(unsigned)wid;
  }

  // ---------------------------------------------------------------- split --
  // engine.py:334 _try_component_split
  __device__ bool try_split() {
    NodeHdr& h = st->hdr;
    const int lo = h.lo, hi = h.hi;
    int ncomp = label_components(w, lo, hi, /*inited=*/true);
    if (ncomp <= 1) return false;
    compress_labels(w, lo, hi);
    tick(PH_LABEL);
    int* agg = w.ib;
    component_aggregates(w, lo, hi, ncomp, agg);
    if (threadIdx.x == 0) {
      ++comp_branches;
      atomicAdd(&P.hist[ncomp < P.n + 1 ? ncomp : P.n + 1], 1ull);
      int G = 0, spec = 0;
      for (int j = 0; j < ncomp; ++j) {
        int size = agg[5 * j], mn = agg[5 * j + 2], mx = agg[5 * j + 3];
        // reductions.py:160 classify_special_component
        if (mn == mx && mn == size - 1) {
          spec += size - 1;
          ++rules[4];
          agg[5 * j + 2] = -1;  // mark special
        } else if (mn == mx && mn == 2 && size >= 3) {
          spec += (size + 1) / 2;
          ++rules[5];
          agg[5 * j + 2] = -2;
        } else {
          ++G;
        }
      }
      const Registry& R = P.reg;
      const int scope = h.scope;
      lb.inc(P, scope);  // slot for the parent entry's finalisation
      int base = reg_alloc(R, 1 + G);
      if (base < 0) {
        atomicExch(&P.ctl->error, 1);
        atomicExch(&P.ctl->stop, 1);
        base = -1;
      } else {
        const int p = base;
        R.kind[p] = 1;
        R.sum[p] = h.S + spec;
        R.sum_ach[p] = 1;
        R.init_sum[p] = h.S;
        R.folded[p] = spec;
        R.live[p] = 1 + G;
        R.link[p] = scope;
        R.first_child[p] = p + 1;
        R.nchild[p] = G;
        R.disc_done[p] = 0;
        R.key[p] = 0;
        R.child_folded[p] = 0;
        int running = h.S, g = 0;
        for (int j = 0; j < ncomp; ++j) {
          int size = agg[5 * j];
          int mark = agg[5 * j + 2];
          if (mark == -1) {
            running += size - 1;
          } else if (mark == -2) {
            running += (size + 1) / 2;
          } else {
            int init = st->best_s - running;
            if (size - 1 < init) init = size - 1;
            if (init < 1) init = 1;
            const bool ach = init == size - 1;
            const int c = p + 1 + g;
            R.kind[c] = 0;
            R.key[c] = init * 2 + (ach ? 0 : 1);
            R.live[c] = 1;
            R.link[c] = p;
            R.child_folded[c] = 0;
            R.disc_done[c] = 0;
            if (P.record) R.wkey[c] = kNoWitness;
            agg[5 * j + 2] = c;  // component -> its child entry
            ++g;
          }
        }
        __threadfence();
      }
      st->gen = G;
      st->parent = base;
    }
    __syncthreads();
    const int parent = st->parent;
    if (parent >= 0 && P.record) record_split_witness(ncomp, agg, parent);
    if (parent >= 0 && P.warp_limit) {
      // small general components go to the warp tier, one warp per
      // component: thread 0 numbers them and claims all their ring tickets
      // with one reservation; each task packs only its component's index
      // span [root, vmax]
      if (threadIdx.x == 0) {
        int k = 0;
        for (int j = 0; j < ncomp; ++j) {
          const bool small = agg[5 * j + 2] >= 0 && agg[5 * j] <= P.warp_limit;
          agg[5 * j + 3] = small ? k++ : -1;
        }
        const long long t0 = k ? q_reserve_push_n(P.bq, k, P.bq.cap) : -1;
        st->qpos_lo = (int)(t0 & 0xffffffffLL);
        st->qpos_hi = (int)(t0 >> 32);
      }
      __syncthreads();
      const long long t0 = ((long long)st->qpos_hi << 32) | (unsigned)st->qpos_lo;
      const int nwarps = blockDim.x >> 5;
      for (int j = threadIdx.x >> 5; j < ncomp; j += nwarps) {
        const int c = agg[5 * j + 2];
        const int ord = agg[5 * j + 3];
        if (ord < 0) continue;
        if (emit_task(w.lst[j], agg[5 * j], w.lst[j], agg[5 * j + 4], c, 0, h.depth + 1, 0,
                      t0 >= 0 ? t0 + ord : -1) &&
            (threadIdx.x & 31) == 0)
          agg[5 * j + 1] = -1;  // taken by the warp tier
      }
      __syncthreads();
    }
    if (parent >= 0) {
      for (int j = 0; j < ncomp; ++j) {
        const int c = agg[5 * j + 2];
        if (c < 0) continue;  // special: folded into the parent sum
        if (agg[5 * j + 1] < 0) continue;  // solved by a warp
        const int root = w.lst[j];
        const int size_deg = agg[5 * j + 1];
        const int vmax = agg[5 * j + 4];
        long long qpos;
        char* dst = choose_dest(&qpos);
        if (!dst) break;
        T* dd = (T*)(dst + sizeof(NodeHdr));
        NodeHdr ch;
        const int g = P.compact ? compact_component(root, agg[5 * j], size_deg, lo, hi, dd) : 0;
        if (g) {
          ch.lo = 0;
          ch.hi = agg[5 * j] - 1;
          ch.graph = g;
          ch.gn = agg[5 * j];
        } else {
          for (int v = threadIdx.x; v < w.n; v += blockDim.x) {
            T val = 0;
            if (v >= lo && v <= hi && w.deg[v] > 0 && w.par[v] == root) val = w.deg[v];
            dd[v] = val;
          }
          if (P.record) {  // a component child starts a fresh cover scope
            unsigned* db = (unsigned*)(dst + sizeof(NodeHdr) + deg_bytes<T>(P.n));
            for (int i = threadIdx.x; i < P.nw; i += blockDim.x) db[i] = 0u;
          }
          ch.lo = P.use_bounds ? root : 0;
          ch.hi = P.use_bounds ? vmax : w.n - 1;
          ch.graph = cur_graph;
          ch.gn = w.n;
        }
        ch.S = 0;
        ch.E = size_deg / 2;
        ch.scope = c;
        ch.depth = h.depth + 1;
        commit_dest(qpos, ch, dst);
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        __threadfence();
        st_release(&P.reg.disc_done[parent], 1);
        if (atomicSub(&P.reg.live[parent], 1) == 1) reg_cascade(P, parent);
      }
    }
    if (threadIdx.x == 0) lb.finish(P, h.scope, false);
    __syncthreads();
    tick(PH_SPLIT);
    return true;
  }

  // ------------------------------------------------------------- process --
  // engine.py:277 _process_node.  Returns true when the include child is
  // left in shared memory to be processed next.
  __device__ bool process() {
    NodeHdr& h = st->hdr;
    if (threadIdx.x == 0) ++nodes;  // st->best_s was fetched with the record
    const int best_s = st->best_s;
    const int budget = best_s - h.S - 1;
    long long maxkey;
    FixRet fr = reduce_fixpoint_fast(w, h.lo, h.hi, budget, &maxkey, P.par_rules != 0);
    tick(PH_REDUCE);
    if (fr.pos < 0) {  // inconsistent degree array (a protocol bug): fail loudly
      if (threadIdx.x == 0) {
        atomicExch(&P.ctl->error, 8);
        atomicExch(&P.ctl->stop, 1);
        lb.finish(P, h.scope, false);
      }
      __syncthreads();
      return false;
    }
    if (threadIdx.x == 0) {
      rules[0] += fr.d1;
      rules[1] += fr.d2t;
      rules[2] += fr.hd;
    }
    int S = h.S + fr.forced;
    int E = h.E - fr.edges;
    int lo = fr.lo, hi = fr.hi;
    if (!P.use_bounds && w.n) {
      lo = 0;
      hi = w.n - 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      h.S = S;
      h.E = E;
      h.lo = lo;
      h.hi = hi;
    }
    __syncthreads();
    if (!P.disable_pruning) {
      bool prune = S >= best_s;
      if (!prune) {
        long long rem = (long long)best_s - S - 1;
        prune = (long long)E > rem * rem;
      }
      if (prune) {
        if (threadIdx.x == 0) lb.finish(P, h.scope, false);
        __syncthreads();
        tick(PH_REGISTRY);
        return false;
      }
    }
    if (E == 0) {
      const unsigned long long wid = P.record ? record_leaf_witness(h.scope, S) : kNoWitness;
      if (threadIdx.x == 0) {
        reg_submit(P, h.scope, S, true, wid);
        lb.finish(P, h.scope, true);
      }
      __syncthreads();
      tick(PH_REGISTRY);
      return false;
    }
    if (P.warp_limit) {
      // small enough for one warp: hand the whole node (and its live unit
      // on the scope) to the warp tier, which also splits it if needed
      int b, e, cnt = 0;
      my_chunk(lo, hi, &b, &e);
      for (int u = b; u < e; ++u) cnt += w.deg[u] > 0;
      cnt = block_sum(cnt, w.bs);
      if (cnt <= P.warp_limit) {
        if (threadIdx.x < 32) {
          const bool ok = emit_task(-1, cnt, lo, hi, h.scope, S, h.depth, 1);
          if (threadIdx.x == 0) st->emitted = ok;
        }
        __syncthreads();
        if (st->emitted) {
          tick(PH_SPLIT);
          return false;
        }
      }
    }
    if (P.use_components && try_split()) return false;
    tick(PH_LABEL);
    // pure.py:241 select_max_degree, taken from the fixpoint's final scan
    const int v = maxkey < 0 ? -1 : 0x7fffffff - (int)(maxkey & 0xffffffffLL);
    tick(PH_SELECT);
    if (v < 0) {
      if (threadIdx.x == 0) {
        atomicExch(&P.ctl->error, 3);
        atomicExch(&P.ctl->stop, 1);
      }
      __syncthreads();
      return false;
    }
    // engine.py:319 _branch_on_vertex
    if (threadIdx.x == 0) lb.inc(P, h.scope);
    // exclude child: built in the second shared-memory buffer, then stored;
    // its destination is claimed first so the claim overlaps the build
    reserve_dest();
    {
      const long long words = payload / 16;  // [deg | inc] -> [deg2 | inc2]
      const uint4* a = (const uint4*)w.deg;
      uint4* b2 = (uint4*)w.deg2;
      for (long long i = threadIdx.x; i < words; i += blockDim.x) b2[i] = a[i];
    }
    __syncthreads();
    NodeWs<T> wx = w;
    wx.deg = w.deg2;
    wx.inc = w.inc2;
    int removed, edges;
    remove_neighbors_fast(wx, v, w.lst, &removed, &edges);
    long long qpos;
    char* dst = resolve_dest(&qpos);
    if (dst) {
      store_payload(dst, w.deg2, payload);
      NodeHdr ex = h;
      ex.S = S + removed;
      ex.E = E - edges;
      ex.depth = h.depth + 1;
      commit_dest(qpos, ex, dst);
    }
    __syncthreads();
    tick(PH_EXCLUDE);
    // the include child continues here: its scope best is read now and
    // consumed after the removal (the load overlaps it)
    int kk = 0;
    if (threadIdx.x == 0) kk = ld_relaxed(&P.reg.key[h.scope]);
    int e2 = remove_vertex(w, v);
    if (threadIdx.x == 0) {
      h.S = S + 1;
      h.E = E - e2;
      h.depth += 1;
      if (top + 1 > max_depth) max_depth = top + 1;
      st->best_s = kk >> 1;
    }
    __syncthreads();
    tick(PH_INCLUDE);
    return true;
  }

  // (zero counters are skipped: an idle block of a small search otherwise
  // adds ~30 zeros to the same Ctl words as every other block -- 2368 blocks
  // of a tiny residual's search spent ~50 us queued on them)
  __device__ void flush_stats() {
    if (threadIdx.x != 0) return;
    Ctl* c = P.ctl;
    add_nz(&c->nodes, nodes);
    add_nz(&c->comp_branches, comp_branches);
    add_nz(&c->pushes, pushes);
    add_nz(&c->pops, pops);
    for (int i = 0; i < 6; ++i) add_nz(&c->rules[i], rules[i]);
    if (max_depth) atomicMax(&c->max_depth, max_depth);
    add_nz(&c->rec_in, rec_in);
    add_nz(&c->rec_out, rec_out);
    for (int i = 0; i < 10; ++i) add_nz(&c->phase[i], ph[i]);
    add_nz(&c->wepoch, wep);
    for (int i = 0; i < 4; ++i) {
      add_nz(&c->rcyc[i], w.bs->rcyc[i]);
      add_nz(&c->rcnt[i], w.bs->rcnt[i]);
    }
  }

};

// kSmem: the workspace (and, when it fits, the CSR) lives in shared memory;
// a compile-time choice so every workspace access is an LDS/STS/ATOMS rather
// than a generic-address access.
template <typename T, bool kSmem, int kWW>
__global__ void __launch_bounds__(VCG_SEARCH_MAXT, VCG_SEARCH_MINB) search_kernel(SearchParams P) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  __shared__ BlockScratch bs;
  __shared__ BlockState st;
  // task packing scratch, sized for this variant's widest task (the warp
  // tier runs in blocks of <= 256 threads)
  __shared__ int wgl[kWTierWarps * 64 * kWW];
  __shared__ int wbusy;
  __shared__ __align__(8) unsigned long long tma_bar;  // node-record bulk copies (kSmem)
  unsigned tma_phase = 0;
  if (kSmem && threadIdx.x == 0) mbar_init(&tma_bar);
  char* base = kSmem ? (char*)dsmem : P.gws + (long long)blockIdx.x * P.gws_bytes;
  NodeWs<T> ws = carve_ws<T>(base, P.n, &bs, P.off, P.nbr);
  if (kSmem && P.csr_in_smem) {
    // the reduced CSR is read-only for the whole search: stage it on chip
    int* soff = (int*)((char*)dsmem + ws_bytes<T>(P.n));
    int* snbr = soff + (((P.n + 1) + 3) & ~3);
    for (int i = threadIdx.x; i <= P.n; i += blockDim.x) soff[i] = P.off[i];
    for (long long i = threadIdx.x; i < P.m2; i += blockDim.x) snbr[i] = P.nbr[i];
    ws.off = soff;
    ws.nbr = snbr;
  }
  int* csr_soff = nullptr;
  int* csr_snbr = nullptr;
  if (kSmem && P.csr_in_smem) {
    csr_soff = const_cast<int*>(ws.off);
    csr_snbr = const_cast<int*>(ws.nbr);
  }
  for (int i = threadIdx.x; i < P.n; i += blockDim.x) {
    ws.tmin[i] = kInf;
    if (i < (P.n + 31) / 32) ws.vbits[i] = 0u;
    ws.flag[i] = 0;
  }
  if (threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) bs.rcyc[i] = bs.rcnt[i] = 0;
  init_block_scratch(&bs);
  if (threadIdx.x == 0 && P.hb) bs.hb = P.hb + (long long)blockIdx.x * kMaxWarps;
  if (!P.record) {
    ws.inc = nullptr;
    ws.inc2 = nullptr;
  }
  // zero the degree-array padding once; load_node only overwrites [0, n)
  {
    const long long words = deg_bytes<T>(P.n > 0 ? P.n : 1) / 4;
    for (long long i = threadIdx.x; i < words; i += blockDim.x) ((unsigned*)ws.deg)[i] = 0;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) P.ctl->t0 = globaltimer();
  Worker<T> wk(P, ws, &st);
  wk.gl = wgl;
  wk.gl_stride = 64 * kWW;
  wk.soff = csr_soff;
  wk.snbr = csr_snbr;
  void* wws = nullptr;
  if (P.warp_limit)
    wws = (kSmem && P.bws_alias) ? (void*)ws.ia : (void*)((char*)dsmem + P.bws_off);
  WStats wst;
  memset(&wst, 0, sizeof(wst));
  if (threadIdx.x == 0) wbusy = 0;
  st.emitted = 0;
  if (blockIdx.x == 0 && P.root_in_stack) {
    wk.top = 1;
    wk.max_depth = 1;
  }
  bool cont = false;
  unsigned backoff = 32;
  unsigned iter = 0;
  unsigned xpoll = 0;
  while (true) {
    VCG_HB(&bs, 50);
    // stop / deadline poll: before every pop, and every 4th node of an
    // include chain (the poll is an L2 round trip plus a barrier)
    if (!cont || (++iter & 3) == 0) {
      if (threadIdx.x == 0) {
        const int stop0 = ld_relaxed(&P.ctl->stop);
        const unsigned long long dl = __ldcg(&P.ctl->deadline_ns);
        int stop = stop0;
        if (!stop && dl && globaltimer() > dl) {
          atomicExch(&P.ctl->timed_out, 1);
          atomicExch(&P.ctl->stop, 1);
          stop = 1;
        }
        // in-flight exchange (vcg_exchange): a cover found elsewhere bounds
        // the root scope (not achieved here); an external stop ends the search
        if (!stop && (P.xch || P.gpeer) && (xpoll++ & 15) == 0 && xch_poll(P)) stop = 1;
        st.flag = stop;
      }
      __syncthreads();
      if (st.flag) break;
    }
    wk.tick(PH_OTHER);
    if (!cont) {
      if (wk.top > 0) {
        wk.top -= 1;
        const int gn =
            kSmem && P.tma_load
                ? load_node_tma<T>(wk.stack_slot(wk.top), &st.hdr, ws.deg, wk.extra, P.n, P.reg.key,
                                   &st.best_s, &tma_bar, &tma_phase, &P.ctl->error)
                : load_node<T>(wk.stack_slot(wk.top), &st.hdr, ws.deg, wk.extra, P.n, P.reg.key,
                               &st.best_s);
        if (threadIdx.x == 0) ++wk.rec_in;
        __syncthreads();
        wk.set_graph(st.hdr.graph, gn);
      } else {
        if (threadIdx.x == 0) {
          long long pos = q_reserve_pop(P.q);
          st.qpos_lo = (int)(pos & 0xffffffffLL);
          st.qpos_hi = (int)(pos >> 32);
        }
        __syncthreads();
        long long pos = ((long long)st.qpos_hi << 32) | (unsigned)st.qpos_lo;
        if (pos < 0) {
          if (threadIdx.x == 0) wk.lb.flush(P);  // idle: release every held-back decrement
          if (P.warp_limit) {
            __syncthreads();
            wk.tick(PH_IDLE);
            VCG_HB(&bs, 60);
            const bool ran = warp_epoch<kWW>(P, wws, &wbusy, wst);
            VCG_HB(&bs, 61);
            if (threadIdx.x == 0) {
              const long long now = clock64();
              if (ran) wk.wep += (unsigned long long)(now - wk.last_clk);
              else wk.ph[PH_IDLE] += (unsigned long long)(now - wk.last_clk);
              wk.last_clk = now;
            }
            if (ran) {
              backoff = 32;
              continue;
            }
          }
          if (threadIdx.x == 0) __nanosleep(backoff);
          backoff = backoff < 4096 ? backoff * 2 : 4096;
          __syncthreads();
          wk.tick(PH_IDLE);
          continue;
        }
        backoff = 32;
        const int gn =
            kSmem && P.tma_load
                ? load_node_tma<T>(wk.queue_slot(pos), &st.hdr, ws.deg, wk.extra, P.n, P.reg.key,
                                   &st.best_s, &tma_bar, &tma_phase, &P.ctl->error)
                : load_node<T>(wk.queue_slot(pos), &st.hdr, ws.deg, wk.extra, P.n, P.reg.key,
                               &st.best_s);
        __syncthreads();
        wk.set_graph(st.hdr.graph, gn);
        if (threadIdx.x == 0) {
          q_release_pop(P.q, pos);
          ++wk.pops;
          ++wk.rec_in;
        }
      }
    }
    wk.tick(PH_LOAD);
    if (threadIdx.x == 0 && bs.hb) {
      ((volatile int*)bs.hb)[23] = st.hdr.graph;
      ((volatile int*)bs.hb)[24] = st.hdr.lo;
      ((volatile int*)bs.hb)[25] = st.hdr.hi;
      ((volatile int*)bs.hb)[26] = st.hdr.gn;
      ((volatile int*)bs.hb)[27] = wk.cur_graph;
      ((volatile int*)bs.hb)[28] = wk.w.n;
    }
    cont = wk.process();
    if (threadIdx.x == 0) atomicMax(&P.ctl->t_node_last, globaltimer());
  }
  // stop: release the registry slots of abandoned work (engine.py:235-243)
  VCG_HB(&bs, 70);
  if (threadIdx.x == 0) {
    wk.lb.flush(P);
    if (cont) reg_finish(P, st.hdr.scope);
    for (int i = wk.top - 1; i >= 0; --i) {
      const NodeHdr* hh = (const NodeHdr*)wk.stack_slot(i);
      reg_finish(P, __ldcg(&hh->scope));
    }
    // every block helps empty the worklist (the host drain kernel only picks
    // up records pushed by blocks that were still finishing a node)
    while (true) {
      long long pos = q_reserve_pop(P.q);
      if (pos < 0) break;
      const NodeHdr* hh = (const NodeHdr*)(P.q.data + (pos % P.q.cap) * P.slot_bytes);
      int scope = __ldcg(&hh->scope);
      q_release_pop(P.q, pos);
      reg_finish(P, scope);
    }
    warp_ring_drain(P);
  }
  wk.flush_stats();
  warp_flush_stats(P, wst);
  VCG_HB(&bs, 99);
}

}  // namespace vcg
