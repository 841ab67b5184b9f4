// Persistent component-aware branch-and-reduce search (north star (2)-(4)).
//
// One resident thread block = one worker of the reference engine
// (vcsolver/engine.py:160 _Engine).  Each block loops: take a node (the
// include child it just produced, else the top of its private stack in HBM,
// else the global worklist), reduce it in shared memory, prune / submit /
// split into components / branch on the max-degree vertex.  Coordination is
// only through:
//   * the global worklist -- a bounded MPMC ring (Vyukov sequence numbers)
//     holding whole node records (engine.py:413 _offload_or_push policy);
//   * the component branch registry -- struct-of-arrays entries updated with
//     device-scope atomics (registry.py; SPEC registry module), whose
//     live-descendant counters hand finalisation to the last finisher
//     (engine.py:424-462 _finish/_cascade/_submit, :464 _pvc_propagate);
//   * the stop/found flags.
#pragma once

#include "node_ops.cuh"

namespace vcg {

// node record header, 32 bytes, followed by deg[gn] (padded to 16 B).
// graph 0: the reduced graph (gn = n); graph g + 1: compacted component
// subgraph g (gn vertices, local ids in reduced-graph order).
struct NodeHdr {
  int S, E, lo, hi, scope, depth, graph, gn;
};

struct Registry {
  int* key;           // child: best*2 + !achieved (atomicMin == atomic_min_best)
  int* live;          // child: live_nodes; parent: live_comps
  int* link;          // child: parent entry (-1 at root); parent: ancestor
  int* kind;          // 0 child, 1 parent
  int* sum;           // parent
  int* sum_ach;       // parent: 1 while every folded term was achieved
  int* init_sum;      // parent (diagnostics / conservation check)
  int* folded;        // parent: total of in-place solved (special) components
  int* first_child;   // parent: children are [first_child, first_child+nchild)
  int* nchild;        // parent
  int* disc_done;     // parent
  int* child_folded;  // child: its best has been added to the parent sum
  unsigned long long* wkey;  // record-cover: (value << 32 | witness) of the best achieved
  int* pwrec;         // record-cover: parent entry's arena record (path + special covers)
  int* count;         // arena size (device counter)
  int cap;
  // Reclamation (parallel mode without record-cover / audits): a split's
  // group (parent + its child entries, contiguous) is dead once the parent's
  // cascade has submitted to its ancestor -- every reader holds a live node
  // below it until then -- so it goes on a free stack for groups of its size
  // class (power of two).  Tagged Treiber stacks, next pointer in the free
  // group's link field.  Without reclamation groups are bump-allocated.
  // Recycling starts once the arena is half used (short searches never pay
  // for it) and the stacks are sharded by block to spread the CAS traffic.
  unsigned long long* fheads;  // [kFreeClasses][kFreeShards]: tag << 32 | top (0xffffffff: empty)
  int reclaim;
  int reclaim_at;  // arena entries in use from which groups are recycled
};

constexpr int kFreeClasses = 32;
constexpr int kFreeShards = 16;

__device__ __forceinline__ int reg_class(int sz) { return sz <= 1 ? 0 : 32 - __clz(sz - 1); }

__device__ __forceinline__ bool reg_recycling(const Registry& R) {
  return R.reclaim && ld_relaxed(R.count) >= R.reclaim_at;
}

// base of a group of sz entries, or -1 when the arena is exhausted
__device__ inline int reg_alloc(const Registry& R, int sz) {
  if (R.reclaim) {
    const int c = reg_class(sz);
    if (reg_recycling(R)) {
      for (int k = 0; k < kFreeShards; ++k) {
        unsigned long long* h =
            &R.fheads[c * kFreeShards + (blockIdx.x + k) % kFreeShards];
        while (true) {
          const unsigned long long old = ld_acquire_u64(h);
          const unsigned top = (unsigned)old;
          if (top == 0xffffffffu) break;
          const unsigned nxt = (unsigned)ld_relaxed(&R.link[top]);
          const unsigned long long nw = (((old >> 32) + 1ull) << 32) | nxt;
          if (atomicCAS(h, old, nw) == old) return (int)top;
        }
      }
    }
    sz = 1 << c;  // a recyclable group occupies its whole size class
  }
  const int base = atomicAdd(R.count, sz);
  return base + sz > R.cap ? -1 : base;
}

// the group of parent entry p is dead: recycle it
__device__ inline void reg_free_group(const Registry& R, int p) {
  if (!reg_recycling(R)) return;
  const int c = reg_class(1 + R.nchild[p]);
  unsigned long long* h = &R.fheads[c * kFreeShards + blockIdx.x % kFreeShards];
  while (true) {
    const unsigned long long old = ld_relaxed_u64(h);
    R.link[p] = (int)(unsigned)old;
    __threadfence();
    const unsigned long long nw = (((old >> 32) + 1ull) << 32) | (unsigned)p;
    if (atomicCAS(h, old, nw) == old) return;
  }
}

// counter flush that skips zeros (the idle blocks / warps of a small search)
template <typename U>
__device__ __forceinline__ void add_nz(U* p, U v) {
  if (v) atomicAdd(p, v);
}

struct Ctl {
  int stop, found, timed_out, error;
  int max_depth, pad0, pad1, pad2;
  unsigned long long nodes, comp_branches, pushes, pops;
  unsigned long long rules[6];  // degree_one, d2t, high_degree, crown, clique, cycle
  unsigned long long rec_in, rec_out;  // node records read from / written to HBM
  unsigned long long deadline_ns;      // %globaltimer deadline, 0 = none
  int root_key, reg_count;             // written by the drain kernel for readback
  unsigned long long phase[10];        // SM cycles per phase, summed over blocks (thread 0)
  unsigned long long rcyc[4], rcnt[4]; // fixpoint profile: scan, degree-one, triangle, high-degree
  unsigned long long wtasks, wnodes, wcyc;  // warp tier: tasks, tree nodes, warp cycles in tasks
  unsigned long long wepoch;           // block cycles (thread 0) spent in warp-tier epochs
  unsigned long long wmax;             // longest warp task (cycles)
  unsigned long long wmax_nodes, wmax_n;  // its tree nodes and vertex count
  // %globaltimer trace (ns): search start, last node-level step, first warp
  // task start, last warp task end
  unsigned long long t0, t_node_last, t_task_first, t_task_last;
  unsigned long long t_end;  // %globaltimer when the drain kernel published the result
  unsigned long long wc_fix, wc_comp, wc_split;  // warp-task cycles: fixpoint, component test, splits
  unsigned long long wc_iter;                    // warp fixpoint loop iterations
};

// phases of a block's time (clock64 deltas taken by thread 0)
enum Phase { PH_IDLE = 0, PH_LOAD, PH_REDUCE, PH_LABEL, PH_SPLIT, PH_SELECT, PH_EXCLUDE,
             PH_INCLUDE, PH_REGISTRY, PH_OTHER };

struct Queue {
  unsigned long long* seq;
  unsigned long long* head;
  unsigned long long* tail;
  unsigned long long* count;  // records claimed by producers minus by consumers
  int* err;                   // Ctl::error, for the spin watchdogs
  char* data;
  long long cap;
};

struct SearchParams {
  int n;
  long long m2;           // 2 * edges of the reduced graph
  int csr_in_smem;        // stage off/nbr in shared memory (after the workspace)
  const int* off;
  const int* nbr;
  char* stacks;           // gridDim.x * stack_cap * slot_bytes
  long long stack_cap;
  long long slot_bytes;
  Queue q;
  Registry reg;
  Ctl* ctl;
  unsigned long long* hist;  // [n + 2] components-per-branch histogram
  char* gws;              // global workspace (when the workspace does not fit smem)
  long long gws_bytes;    // per block
  int ws_in_smem;
  int share;              // offload to the worklist at all
  long long threshold;    // worklist length below which nodes are offloaded
  int use_components, use_bounds, disable_pruning;
  int pvc;
  int k_red;
  int root_index;
  int root_in_stack;
  int record;             // record-cover mode: nodes carry inclusion bitsets
  int batch_live;         // parallel mode: LiveBatch decrement batching
  int par_rules;          // parallel mode: claim-based triangle sweep (sound, not in-order)
  int nw;                 // bitset words per record
  unsigned* wbits;        // witness arena [wcap][nw]
  int* wcount;
  int wcap;
  // warp tier (warp_solve.cuh): ring of bitmask tasks, per-warp workspaces
  Queue bq;
  long long bq_slot;      // bytes per warp-task slot (warp_solve.cuh wslot_bytes)
  int warp_split_export;  // wide warp tasks hand frame-0 splits to the registry
  int tma_load;           // node records into shared-memory workspaces by TMA bulk copy
  int warp_limit;         // 0 = off
  long long bq_low;       // a long warp task sheds work while the ring holds fewer
  int w_check_mask;       // a warp task polls stop / bound / ring every (mask + 1) nodes
  int w_export_after;     // and may shed work once it has run this many nodes
  // component subgraphs (order-preserving compaction of split components):
  // subgraph g = CSR at arena[sg_base[g]]: offsets [sg_n[g] + 1] (padded to 4),
  // then neighbours
  int compact;            // compact general components larger than warp_limit
  int* sg_n;
  int* sg_base;
  int* sg_count;
  int sg_cap;
  int* arena;
  int* arena_top;
  int arena_cap;
  int bws_alias;          // warp workspaces alias the node workspace's int scratch
  long long bws_off;      // else: their offset in dynamic shared memory
  int* hb;                // debug heartbeat rows [gridDim.x][kMaxWarps] (host-mapped), or null
  // vcg_exchange words: [0] external root bound (kInf: none), [1] external
  // stop, [2] this search's best achieved root cover (kInf: none); or null
  int* xch;
  // peer exchange (vcg_peer): the distributed solve's global words, in one
  // rank's device memory and mapped into every rank's address space by CUDA
  // IPC (NVLink peer memory across GPUs): [0] best absolute cover, [1] stop.
  // This search's root covers are offset by gpeer_off (the subtree's S).
  int* gpeer;
  int gpeer_off;
};

__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// external bound / stop from the exchange words (thread 0 of a block or lane
// 0 of a warp): true when the search must stop
__device__ inline bool xch_poll(const SearchParams& P, int root_key_idx_unused = 0) {
  (void)root_key_idx_unused;
  bool stop = false;
  int bound = kInf;
  if (P.xch) {
    const int xb = __ldcg(&P.xch[0]), xs = __ldcg(&P.xch[1]);
    stop |= xs != 0;
    bound = xb;
  }
  if (P.gpeer) {
    const int gb = ld_relaxed_sys(&P.gpeer[0]), gs = ld_relaxed_sys(&P.gpeer[1]);
    stop |= gs != 0;
    if (gb < kInf) bound = min(bound, gb - P.gpeer_off);
  }
  if (bound <= 0) stop = true;
  if (stop) {
    atomicExch(&P.ctl->stop, 1);
    return true;
  }
  if (bound < kInf) atomicMin(&P.reg.key[P.root_index], 2 * bound + 1);
  return false;
}

// an achieved root-scope cover of `value` vertices: publish it to the exchange
__device__ __forceinline__ void xch_publish(const SearchParams& P, int idx, int value) {
  if (idx != P.root_index) return;
  if (P.xch) atomicMin(&P.xch[2], value);
  if (P.gpeer) atomicMin_system(&P.gpeer[0], value + P.gpeer_off);
}

template <typename T>
__host__ __device__ inline long long deg_bytes(int n) {
  return (((long long)n * (long long)sizeof(T)) + 15) & ~15LL;
}

// record-cover bitset bytes (one bit per reduced vertex), 16-byte padded
__host__ __device__ inline long long bits_bytes(int n) {
  long long nw = ((long long)(n > 0 ? n : 1) + 31) / 32;
  return (nw * 4 + 15) & ~15LL;
}

// workspace bytes for one block: [deg | inc | deg2 | inc2 | flag | 8 int arrays | bitmap]
template <typename T>
__host__ __device__ inline long long ws_bytes(int n) {
  long long nn = n > 0 ? n : 1;
  return 2 * (deg_bytes<T>((int)nn) + bits_bytes((int)nn)) + ((nn + 15) & ~15LL) +
         8LL * 4LL * ((nn + 3) & ~3LL) + bits_bytes((int)nn);
}

// bytes of the reduced CSR staged in shared memory (int32 offsets + neighbours)
__host__ __device__ inline long long csr_smem_bytes(int n, long long m2) {
  return ((4LL * (n + 1) + 15) & ~15LL) + ((4LL * m2 + 15) & ~15LL);
}

template <typename T>
__device__ inline NodeWs<T> carve_ws(char* base, int n, BlockScratch* bs, const int* off,
                                     const int* nbr) {
  long long nn = n > 0 ? n : 1;
  long long ni = (nn + 3) & ~3LL;
  NodeWs<T> w;
  char* p = base;
  w.deg = (T*)p;
  p += deg_bytes<T>((int)nn);
  w.inc = (unsigned*)p;
  p += bits_bytes((int)nn);
  w.deg2 = (T*)p;
  p += deg_bytes<T>((int)nn);
  w.inc2 = (unsigned*)p;
  p += bits_bytes((int)nn);
  w.flag = (uint8_t*)p;
  p += (nn + 15) & ~15LL;
  int* ip = (int*)p;
  w.tmin = ip;
  w.ia = ip + ni;
  w.id = ip + 2 * ni;
  w.lst = ip + 3 * ni;
  w.ib = ip + 4 * ni;  // ib, ic and the spare that follows are contiguous:
  w.ic = ip + 5 * ni;  // component aggregates (5 ints x <= n/2 comps) use them
  w.par = ip + 7 * ni;
  w.vbits = (unsigned*)(ip + 8 * ni);
  w.bs = bs;
  w.off = off;
  w.nbr = nbr;
  w.n = n;
  return w;
}

// ------------------------------------------------------------------ queue --
// Broker-queue ring (count guard + fetch-and-add tickets): a producer first
// claims a unit of `count` (which doubles as the length check of the offload
// policy), then a tail ticket; a consumer claims a unit of `count` only when
// one is there, then a head ticket, so the ticket's producer is guaranteed to
// be committed.  Per-slot sequence numbers hand each slot between the two.
// No CAS loops: every operation is O(1) atomics, contention-free retries.

__device__ __forceinline__ long long atom_add_ll(unsigned long long* p, long long v) {
  return (long long)atomicAdd(p, (unsigned long long)v);
}

// Claim a push slot if fewer than `limit` records are queued; -1 otherwise.
__device__ inline long long q_reserve_push(const Queue& q, long long limit) {
  if (limit > q.cap) limit = q.cap;
  if ((long long)ld_relaxed_u64(q.count) >= limit) return -1;
  long long c = atom_add_ll(q.count, 1);
  if (c >= limit) {
    atom_add_ll(q.count, -1);
    return -1;
  }
  long long pos = atom_add_ll(q.tail, 1);
  // the slot is free once its previous consumer has released it
  unsigned spins = 0;
  while ((long long)ld_acquire_u64(&q.seq[pos % q.cap]) != pos) {
    __nanosleep(32);
    if (++spins == (1u << 26)) {
      atomicExch(q.err, 6);  // watchdog: slot never released
      break;
    }
  }
  return pos;
}

// Claim k consecutive tickets at once (a split's warp tasks); the caller
// waits for each slot with q_wait_free before writing it.  -1: no room.
__device__ inline long long q_reserve_push_n(const Queue& q, long long k, long long limit) {
  if (limit > q.cap) limit = q.cap;
  if ((long long)ld_relaxed_u64(q.count) + k > limit) return -1;
  long long c = atom_add_ll(q.count, k);
  if (c + k > limit) {
    atom_add_ll(q.count, -k);
    return -1;
  }
  return atom_add_ll(q.tail, k);
}

// the slot of ticket pos is free once its previous consumer released it
__device__ inline void q_wait_free(const Queue& q, long long pos) {
  unsigned spins = 0;
  while ((long long)ld_acquire_u64(&q.seq[pos % q.cap]) != pos) {
    __nanosleep(32);
    if (++spins == (1u << 26)) {
      atomicExch(q.err, 6);
      break;
    }
  }
}

__device__ inline void q_publish_push(const Queue& q, long long pos) {
  __threadfence();
  st_release_u64(&q.seq[pos % q.cap], (unsigned long long)pos + 1);
}

// Claim a queued record; -1 when none.
__device__ inline long long q_reserve_pop(const Queue& q) {
  if ((long long)ld_relaxed_u64(q.count) <= 0) return -1;
  long long c = atom_add_ll(q.count, -1);
  if (c <= 0) {
    atom_add_ll(q.count, 1);
    return -1;
  }
  long long pos = atom_add_ll(q.head, 1);
  // the ticket's producer is committed: wait for its publication
  unsigned spins = 0;
  while ((long long)ld_acquire_u64(&q.seq[pos % q.cap]) != pos + 1) {
    __nanosleep(32);
    if (++spins == (1u << 26)) {
      atomicExch(q.err, 7);  // watchdog: ticket never published
      break;
    }
  }
  return pos;
}

__device__ inline void q_release_pop(const Queue& q, long long pos) {
  st_release_u64(&q.seq[pos % q.cap], (unsigned long long)pos + (unsigned long long)q.cap);
}

// --------------------------------------------------------------- registry --

constexpr unsigned long long kNoWitness = ~0ull;
constexpr unsigned kComposite = 1u << 31;  // witness id tag: "parent entry p + its children"

__device__ inline void reg_submit(const SearchParams& P, int idx, int value, bool achieved,
                                  unsigned long long wid);

__device__ __forceinline__ void note_witness(const SearchParams& P, int idx, int value,
                                             unsigned long long wid) {
  if (P.record && wid != kNoWitness)
    atomicMin(&P.reg.wkey[idx], ((unsigned long long)(unsigned)value << 32) | wid);
}

// engine.py:464 _pvc_propagate.  Children are read before the parent sum so
// a child that finishes concurrently is counted twice (a safe over-estimate)
// rather than not at all.
__device__ inline void pvc_propagate(const SearchParams& P, int idx) {
  const Registry& R = P.reg;
  while (true) {
    int p = ld_relaxed(&R.link[idx]);
    if (p < 0) return;
    if (!ld_acquire(&R.disc_done[p])) return;
    long long total = 0;
    int fc = R.first_child[p], nc = R.nchild[p];
    for (int c = fc; c < fc + nc; ++c) {
      int live = ld_relaxed(&R.live[c]);
      int folded = ld_acquire(&R.child_folded[c]);
      if (live > 0 || !folded) {
        int key = ld_relaxed(&R.key[c]);
        if (key & 1) return;  // live component whose bound is not achieved
        total += key >> 1;
      }
    }
    __threadfence();
    if (!ld_relaxed(&R.sum_ach[p])) return;
    total += ld_relaxed(&R.sum[p]);
    int anc = R.link[p];
    atomicMin(&R.key[anc], (int)(total * 2));
    xch_publish(P, anc, (int)total);
    note_witness(P, anc, (int)total, kComposite | (unsigned)p);
    idx = anc;
  }
}

// engine.py:453 _submit
__device__ inline void reg_submit(const SearchParams& P, int idx, int value, bool achieved,
                                  unsigned long long wid) {
  if (achieved) {
    note_witness(P, idx, value, wid);
    xch_publish(P, idx, value);
  }
  atomicMin(&P.reg.key[idx], value * 2 + (achieved ? 0 : 1));
  if (!P.pvc) return;
  if (idx != P.root_index) pvc_propagate(P, idx);
  int best = ld_relaxed(&P.reg.key[P.root_index]) >> 1;
  if (best <= P.k_red) {
    atomicExch(&P.ctl->found, 1);
    atomicExch(&P.ctl->stop, 1);
    if (P.gpeer) atomicExch_system(&P.gpeer[1], 1);  // PVC answered: every rank stops
  }
}

// engine.py:428 _cascade: run completion upward from a quiesced entry.
__device__ inline void reg_cascade(const SearchParams& P, int idx) {
  const Registry& R = P.reg;
  while (true) {
    if (R.kind[idx] == 0) {
      int p = R.link[idx];
      if (p < 0) {
        atomicExch(&P.ctl->stop, 1);  // root scope finished
        return;
      }
      int key = ld_relaxed(&R.key[idx]);
      atomicAdd(&R.sum[p], key >> 1);
      if (key & 1) atomicAnd(&R.sum_ach[p], 0);
      __threadfence();
      st_release(&R.child_folded[idx], 1);
      if (atomicSub(&R.live[p], 1) != 1) return;
      idx = p;
    } else {
      __threadfence();
      int total = ld_relaxed(&R.sum[idx]);
      int ach = ld_relaxed(&R.sum_ach[idx]);
      int anc = R.link[idx];
      reg_submit(P, anc, total, ach != 0, kComposite | (unsigned)idx);
      reg_free_group(R, idx);
      if (atomicSub(&R.live[anc], 1) != 1) return;
      idx = anc;
    }
  }
}

// release: this node's submissions are visible before its slot is returned;
// acquire: the last finisher sees every other finisher's submissions
__device__ __forceinline__ int atom_dec_acq_rel(int* p) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

__device__ inline void reg_finish(const SearchParams& P, int scope) {
  if (atom_dec_acq_rel(&P.reg.live[scope]) == 1) reg_cascade(P, scope);
}

// Parallel-mode batching of LiveNodes updates (thread 0 of a block).  A
// finished node's decrement is held back and cancelled against the block's
// next increment on the same scope; it is flushed the moment the block
// touches another scope or idles.  While the block works in scope s, s has a
// live node (the block's own), so holding s's decrements delays no cascade.
// Increments are never deferred, so a counter can only read high.
struct LiveBatch {
  int scope = -1;
  int pending = 0;
  int enabled = 0;

  __device__ void flush(const SearchParams& P);
  __device__ void finish(const SearchParams& P, int s, bool submitted);
  __device__ void inc(const SearchParams& P, int s);
};

// a pruned node submitted nothing: no release needed, only the last finisher
// needs to acquire before cascading
__device__ inline void reg_finish_pruned(const SearchParams& P, int scope) {
  if (atomicSub(&P.reg.live[scope], 1) == 1) {
    __threadfence();
    reg_cascade(P, scope);
  }
}



// ------------------------------------------------------------ node moves --

// payload = degree array of the node's graph (+ inclusion bitset in
// record-cover mode, which never compacts: extra = its bytes); the
// shared-memory layout keeps them contiguous, like the record.  Every thread
// reads the header's second half (one broadcast request per warp) to size
// the copy; the scope's best (engine.py:279 best_snapshot) is fetched by
// thread 1, overlapped with the payload copy.  Returns the graph's vertex
// count.
template <typename T>
__device__ inline int load_node(const char* src, NodeHdr* hdr, void* payload, long long extra,
                                int n_root, const int* keys, int* best_out) {
  const uint4* s = (const uint4*)src;
  const uint4 h1 = __ldcg(s + 1);  // scope, depth, graph, gn
  const int gn = h1.z ? (int)h1.w : n_root;
  if (threadIdx.x == 0) ((uint4*)hdr)[0] = __ldcg(s);
  if (threadIdx.x == 1) {
    ((uint4*)hdr)[1] = h1;
    *best_out = ld_relaxed(&keys[(int)h1.x]) >> 1;
  }
  const long long words = (deg_bytes<T>(gn) + extra) / 16;
  const uint4* sd = s + 2;
  uint4* dd = (uint4*)payload;
  for (long long i = threadIdx.x; i < words; i += blockDim.x) dd[i] = __ldcg(sd + i);
  return gn;
}

// The same load with the payload moved by the Tensor Memory Accelerator: one
// thread reads the header's graph fields (the size depends on them), then
// issues a 1-D bulk copy (cp.async.bulk, global -> shared) that completes on
// an mbarrier every thread waits on; the other threads issue no loads.
// Shared-memory payloads only (kSmem search variants).  `phase` is the
// mbarrier's parity, flipped per use.
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
template <typename T>
__device__ inline int load_node_tma(const char* src, NodeHdr* hdr, void* payload, long long extra,
                                    int n_root, const int* keys, int* best_out,
                                    unsigned long long* bar, unsigned* phase, int* err) {
  const uint4* s = (const uint4*)src;
  const uint4 h1 = __ldcg(s + 1);  // scope, depth, graph, gn
  const int gn = h1.z ? (int)h1.w : n_root;
  const unsigned bytes = (unsigned)(deg_bytes<T>(gn) + extra);
  const unsigned ab = (unsigned)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    ((uint4*)hdr)[0] = __ldcg(s);
    // the block's earlier generic-proxy accesses of the payload (ordered
    // before this thread by the caller's barrier) precede the async writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ab), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (unsigned)__cvta_generic_to_shared(payload)),
        "l"(s + 2), "r"(bytes), "r"(ab)
        : "memory");
  }
  if (threadIdx.x == 1) {
    ((uint4*)hdr)[1] = h1;
    *best_out = ld_relaxed(&keys[(int)h1.x]) >> 1;
  }
  unsigned done = 0;
  for (unsigned spin = 0; !done; ++spin) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(ab), "r"(*phase)
        : "memory");
    if (!done && spin > (1u << 24)) {  // never hang the search: report and stop
      atomicExch(err, 1);
      break;
    }
  }
  *phase ^= 1u;
  return gn;
}

__device__ inline void store_payload(char* dst, const void* payload, long long bytes) {
  const long long words = bytes / 16;
  uint4* dd = (uint4*)(dst + sizeof(NodeHdr));
  const uint4* sd = (const uint4*)payload;
  for (long long i = threadIdx.x; i < words; i += blockDim.x) __stcg(dd + i, sd[i]);
}

__device__ inline void LiveBatch::flush(const SearchParams& P) {
  if (pending > 0) {
    const int k = pending;
    pending = 0;
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;"
                 : "=r"(old) : "l"(&P.reg.live[scope]), "r"(-k) : "memory");
    if (old == k) reg_cascade(P, scope);
  }
  scope = -1;
}

__device__ inline void LiveBatch::finish(const SearchParams& P, int s, bool submitted) {
  if (!enabled) {
    if (submitted) reg_finish(P, s);
    else reg_finish_pruned(P, s);
    return;
  }
  if (s != scope) {
    flush(P);
    scope = s;
  }
  ++pending;
}

__device__ inline void LiveBatch::inc(const SearchParams& P, int s) {
  if (enabled) {
    if (s == scope && pending > 0) {
      --pending;
      return;
    }
    flush(P);
  }
  atomicAdd(&P.reg.live[s], 1);
}

}  // namespace vcg
