// Warp tier of the search: a subproblem with at most 64 live vertices is
// solved by ONE warp as bitmask branch-and-reduce.
//
// Why: on the component-splitting workloads (configs[1], the RGG) the search
// nodes hold ~13 live vertices on average while their degree-array window
// spans ~540 vertices of the reduced graph (87% of the nodes have <= 32 live
// vertices, 97.6% <= 64).  A whole thread block sweeping a 1 KB degree
// record per node is the wrong granularity for them.  Here a task is the
// induced subgraph itself -- 64 adjacency bitmasks (512 B) held in
// registers, two rows per lane -- and a search node is a 64-bit live mask
// plus a cover count, so a node costs a few hundred warp instructions and no
// block barrier, HBM record or registry atomic.
//
// Semantics (reference engine.py:277 _process_node, kernels/pure.py rules,
// engine.py:334 _try_component_split) are preserved as sets, not as
// schedules: the same rules are applied to a fixpoint (in a different but
// sound order), the same stopping rule prunes, the same max-degree vertex
// (lowest index on ties, the task keeps the reduced graph's vertex order) is
// branched on, include child first.  A node that splits is handled
// component-aware inside the warp: clique / chordless-cycle components are
// folded in closed form (reductions.py:160), the general ones are solved one
// after another as nested frames whose bounds account for the components
// already solved -- the sequential restatement of the registry's parent /
// child entries, with the cover total submitted to the enclosing scope.
// Parity: answers (cover size, PVC yes/no) equal the reference's; tree-node
// counts differ, as in every parallel schedule.  Deterministic mode and
// record-cover mode do not use this tier.
#pragma once

#include "search.cuh"

namespace vcg {

// per-phase cycle counters of warp tasks (SolveResult.phase_cycles
// warp_*_cycles): build with -DVCG_WARP_PROFILE; off by default, the
// counters live in local memory on the hot path
#ifdef VCG_WARP_PROFILE
#define WPROF(...) __VA_ARGS__
#else
#define WPROF(...)
#endif

constexpr int kWMax = 64;      // vertices per warp task
constexpr int kWStack = 72;    // DFS stack entries per warp (depth <= 64)
constexpr int kWFrames = 24;   // nested component frames (each >= 6 vertices)
constexpr int kWPend = 32;     // pending component masks over all frames

// warp-task record: 32 B header + adjacency rows (n used of 64)
struct WTaskHdr {
  int S;      // cover size of the task's root within its registry scope
  int scope;  // registry entry the task reports to (it holds one live unit)
  int n;      // vertices | (root already counted as a tree node) << 16
  int depth;
  unsigned long long live;  // live vertices of the task's root node
  unsigned long long pad;
};
constexpr long long kWHdrBytes = 32;
constexpr long long kWSlotBytes = kWHdrBytes + 8 * kWMax;
// a task polls every 4 nodes and may shed work after 4 (capi.cu; VCG_WCHECK /
// VCG_WEXPORT override): on rgg2000 PVC(opt-1) 1.40 -> 1.28 ms vs every 16 / after 64

struct WFrame {
  int best;     // looking for covers of this frame's graph smaller than best
  int ach;      // best is the size of a known cover
  int running;  // frames > 0: cover of the enclosing node so far
  int base;     // DFS stack height when the current component started
  int pend_b, pend_e;  // its pending general components: pend[pend_b, pend_e)
  int pad0, pad1;
};

struct WarpWs {
  unsigned long long adj[kWMax];
  unsigned long long stL[kWStack];
  unsigned long long pend[kWPend];
  int stS[kWStack];
  WFrame fr[kWFrames];
};

struct WStats {
  unsigned long long tasks, nodes, splits, cyc, maxcyc, max_nodes, max_n;
  unsigned long long c_fix, c_comp, c_split;  // cycles in the node phases
  unsigned long long c_iter;                   // fixpoint loop iterations
  unsigned long long rules[6];
};

__device__ __forceinline__ unsigned long long wor64(unsigned long long x) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)x);
  const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(x >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

__device__ __forceinline__ unsigned long long ballot64(bool a, bool b) {
  return (unsigned long long)__ballot_sync(0xffffffffu, a) |
         ((unsigned long long)__ballot_sync(0xffffffffu, b) << 32);
}

// Mask helpers for both task widths: tasks of <= 32 vertices run on 32-bit
// masks (one vertex per lane: one ballot / reduction per collective, no
// 64-bit emulation), larger ones on 64-bit masks (two vertices per lane).
__device__ __forceinline__ unsigned wor(unsigned x) { return __reduce_or_sync(0xffffffffu, x); }
__device__ __forceinline__ unsigned long long wor(unsigned long long x) { return wor64(x); }
__device__ __forceinline__ int wpopc(unsigned x) { return __popc(x); }
__device__ __forceinline__ int wpopc(unsigned long long x) { return __popcll(x); }
__device__ __forceinline__ int wlsb(unsigned x) { return __ffs((int)x) - 1; }
__device__ __forceinline__ int wlsb(unsigned long long x) { return __ffsll((long long)x) - 1; }
__device__ __forceinline__ int wmsb(unsigned x) { return 31 - __clz((int)x); }
__device__ __forceinline__ int wmsb(unsigned long long x) { return 63 - __clzll((long long)x); }
template <typename M>
__device__ __forceinline__ M wbit(int i) { return (M)1 << i; }
// vertex v live in L (v >= the mask width: never)
__device__ __forceinline__ bool whas(unsigned L, int v) { return v < 32 && ((L >> v) & 1u); }
__device__ __forceinline__ bool whas(unsigned long long L, int v) { return (L >> v) & 1ull; }
template <typename M>
__device__ __forceinline__ M wballot(bool a, bool b);
template <>
__device__ __forceinline__ unsigned wballot<unsigned>(bool a, bool) {
  return __ballot_sync(0xffffffffu, a);
}
template <>
__device__ __forceinline__ unsigned long long wballot<unsigned long long>(bool a, bool b) {
  return ballot64(a, b);
}

// Per-lane view of the task graph: this lane owns vertices lane and lane+32.
template <typename M>
struct WLane {
  M a0, a1;  // adjacency rows of the two vertices (32-bit tasks: a1 = 0, v1 = 64)
  int v0, v1;
};

// Connected component of the live mask L containing r (frontier BFS, one
// OR-reduction per level).
template <typename M>
__device__ __forceinline__ M w_component(const WLane<M>& q, M L, int r) {
  M comp = wbit<M>(r), fr = comp;
  while (fr) {
    M c = 0;
    if (whas(fr, q.v0)) c |= q.a0;
    if (whas(fr, q.v1)) c |= q.a1;
    fr = wor(c) & L & ~comp;
    comp |= fr;
  }
  return comp;
}

// Rules to a joint fixpoint on (L, S) under the bound `best` (pure.py:188
// reduce_fixpoint: degree-one, degree-two triangle, high degree).  Leaves d0
// / d1 = current degrees of the lane's vertices.  Returns the edge count,
// or -1 when S reached the bound (prune).
template <typename M>
__device__ __forceinline__ int w_fixpoint(const WarpWs& ws, const WLane<M>& q, M& L, int& S,
                                          int best, int& d0, int& d1, WStats& st) {
  while (true) {
    WPROF(++st.c_iter);
    d0 = whas(L, q.v0) ? wpopc(q.a0 & L) : 0;
    d1 = whas(L, q.v1) ? wpopc(q.a1 & L) : 0;
    L = wballot<M>(d0 > 0, d1 > 0);  // isolated vertices leave the graph
    const int k = best - S - 1;    // vertices an improving cover may still take
    if (k < 0) return -1;
    // degree one (pure.py:82): the neighbour of a pendant vertex is forced;
    // of an isolated edge only the higher end (the in-order sweep's choice)
    const M p1 = wballot<M>(d0 == 1, d1 == 1);
    if (p1) {
      M c = 0;
      if (d0 == 1) {
        const int u = wlsb(q.a0 & L);
        if (!(((p1 >> u) & 1) && u < q.v0)) c |= wbit<M>(u);
      }
      if (d1 == 1) {
        const int u = wlsb(q.a1 & L);
        if (!(((p1 >> u) & 1) && u < q.v1)) c |= wbit<M>(u);
      }
      const M F = wor(c);
      L &= ~F;
      S += wpopc(F);
      st.rules[0] += wpopc(F);
      continue;
    }
    // degree-two triangle (pure.py:113): in index order with revalidation.
    // Validity (the two neighbours adjacent) is decided by every lane for
    // its own vertices, fetching the neighbour's row from its owner lane;
    // the in-order walk then only visits valid candidates, and a later
    // candidate stays applicable iff it and its two neighbours are still
    // live (a removal only deletes vertices, so its degree cannot stay 2
    // otherwise).
    {
      int ab0 = -1, ab1 = -1;
      bool t0 = false, t1 = false;
      {
        const M n0 = q.a0 & L, n1 = q.a1 & L;
        const int a0 = wlsb(n0), b0 = wmsb(n0);
        const int a1 = wlsb(n1), b1 = wmsb(n1);
        // row of a0 / a1 from their owner lanes (all lanes shuffle)
        const M r0lo = __shfl_sync(0xffffffffu, q.a0, a0 & 31);
        const M r0hi = __shfl_sync(0xffffffffu, q.a1, a0 & 31);
        const M r1lo = __shfl_sync(0xffffffffu, q.a0, a1 & 31);
        const M r1hi = __shfl_sync(0xffffffffu, q.a1, a1 & 31);
        if (d0 == 2) {
          const M ra = a0 < 32 ? r0lo : r0hi;
          t0 = (ra >> b0) & 1;
          ab0 = a0 | (b0 << 8);
        }
        if (d1 == 2) {
          const M ra = a1 < 32 ? r1lo : r1hi;
          t1 = (ra >> b1) & 1;
          ab1 = a1 | (b1 << 8);
        }
      }
      M T = wballot<M>(t0, t1);
      if (T) {
        M R = 0;  // vertices removed by this sweep
        int applied = 0;
        while (T) {
          const int v = wlsb(T);
          T &= T - 1;
          const int ab = __shfl_sync(0xffffffffu, v < 32 ? ab0 : ab1, v & 31);
          const M tri = wbit<M>(v) | wbit<M>(ab & 255) | wbit<M>(ab >> 8);
          if (tri & R) continue;
          R |= tri & ~wbit<M>(v);
          R |= wbit<M>(v);  // v leaves too (isolated once its neighbours are in)
          ++applied;
        }
        const M nb = R;  // includes the candidates themselves
        // cover gains exactly the two neighbours per applied triangle
        L &= ~nb;
        S += 2 * applied;
        st.rules[1] += applied;
        continue;
      }
    }
    // high degree (pure.py:158): a vertex of degree > k is in every cover
    // that still improves the bound
    const M H = wballot<M>(d0 > k, d1 > k);
    if (H) {
      L &= ~H;
      S += wpopc(H);
      st.rules[2] += wpopc(H);
      continue;
    }
    break;
  }
  return __reduce_add_sync(0xffffffffu, d0 + d1) >> 1;
}

// Push (adjacency of this task, live mask L) as a new task on the same
// scope with cover offset th.S + Sl.  false: ring full.
__device__ inline bool warp_export(const SearchParams& P, const WarpWs& ws, const WTaskHdr& th,
                                   int n, unsigned long long L, int Sl) {
  const int lane = threadIdx.x & 31;
  long long pos = -1;
  if (lane == 0) pos = q_reserve_push(P.bq, P.bq.cap);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  if (pos < 0) return false;
  char* slot = P.bq.data + (pos % P.bq.cap) * kWSlotBytes;
  unsigned long long* dst = (unsigned long long*)(slot + kWHdrBytes);
  for (int i = lane; i < n; i += 32) __stcg(dst + i, ws.adj[i]);
  if (lane == 0) {
    __stcg((int4*)slot, make_int4(th.S + Sl, th.scope, n, th.depth + 1));
    __stcg((unsigned long long*)(slot + 16), L);
    atomicAdd(&P.reg.live[th.scope], 1);  // before the task can finish it
  }
  __syncwarp();
  if (lane == 0) q_publish_push(P.bq, pos);
  return true;
}

// Solve one task to completion (or until the stop flag).  All 32 lanes run
// it with warp-uniform state; returns false when abandoned on stop.
template <typename M>
__device__ inline bool warp_solve_task(const SearchParams& P, WarpWs& ws, const WTaskHdr th,
                                       WStats& st) {
  const int lane = threadIdx.x & 31;
  const int n = th.n & 0xffff;
  constexpr bool kTwo = sizeof(M) == 8;
  WLane<M> q;
  q.v0 = lane;
  q.v1 = kTwo ? lane + 32 : 64;  // 64: never live (whas)
  q.a0 = q.v0 < n ? (M)ws.adj[q.v0] : (M)0;
  q.a1 = kTwo && q.v1 < n ? (M)ws.adj[q.v1] : (M)0;
  bool skip_count = (th.n >> 16) & 1;

  int sb = 0;
  if (lane == 0) sb = ld_relaxed(&P.reg.key[th.scope]) >> 1;
  sb = __shfl_sync(0xffffffffu, sb, 0);
  ws.fr[0].best = sb - th.S;
  ws.fr[0].ach = 0;
  ws.fr[0].base = 0;
  ws.fr[0].pend_b = ws.fr[0].pend_e = 0;
  int nf = 1, sp = 0;
  M L = (M)th.live;
  int S = 0;
  bool have = ws.fr[0].best > 0;
  unsigned tick = 0;

  while (true) {
    if (!have) {
      const int f = nf - 1;
      if (sp > ws.fr[f].base) {
        --sp;
        L = (M)ws.stL[sp];
        S = ws.stS[sp];
        have = true;
      } else if (f == 0) {
        break;  // task exhausted
      } else {
        // the current component of frame f is exhausted
        WFrame& F = ws.fr[f];
        if (!F.ach) {
          --nf;  // nothing below its bound: the enclosing node cannot improve
          continue;
        }
        F.running += F.best;
        if (F.pend_e > F.pend_b) {
          const M c = (M)ws.pend[--F.pend_e];
          const int bound = ws.fr[f - 1].best - F.running - (F.pend_e - F.pend_b);
          const int size = wpopc(c);
          if (bound <= 0) {
            --nf;
            continue;
          }
          if (size - 1 < bound) {
            F.best = size - 1;
            F.ach = 1;
          } else {
            F.best = bound;
            F.ach = 0;
          }
          F.base = sp;
          L = c;
          S = 0;
          have = true;
        } else {
          const int total = F.running;
          --nf;
          WFrame& G = ws.fr[f - 1];
          if (total < G.best) {  // leaf of the enclosing frame
            G.best = total;
            G.ach = 1;
            if (f - 1 == 0 && lane == 0) reg_submit(P, th.scope, th.S + total, true, kNoWitness);
          }
        }
        continue;
      }
    }
    // ------------------------------------------------------------ node --
    const int f = nf - 1;
    if ((++tick & (unsigned)P.w_check_mask) == 0) {
      int stop = 0, shed = 0;
      if (lane == 0) {
        // four independent L2 reads issued together: one round trip
        stop = ld_relaxed(&P.ctl->stop);
        const unsigned long long dl = __ldcg(&P.ctl->deadline_ns);
        const int key = ld_relaxed(&P.reg.key[th.scope]);
        const long long ring = (long long)ld_relaxed_u64(P.bq.count);
        if (!stop && dl && globaltimer() > dl) {
          atomicExch(&P.ctl->timed_out, 1);
          atomicExch(&P.ctl->stop, 1);
          stop = 1;
        }
        if (!stop) {  // the scope may be shared (exports, MVC root): follow its bound
          const int b = (key >> 1) - th.S;
          if (b < ws.fr[0].best) ws.fr[0].best = b;
          shed = tick >= (unsigned)P.w_export_after && ring < P.bq_low;
        }
      }
      __syncwarp();
      if (__shfl_sync(0xffffffffu, stop, 0)) return false;
      // Long task and a short ring: shed the shallowest pending node of
      // frame 0 (the largest open subtree) as a task of its own on the same
      // scope, which takes a live unit there (engine.py:413's offload, for
      // the warp tier).
      const int top0 = nf > 1 ? ws.fr[1].base : sp;
      if (__shfl_sync(0xffffffffu, shed, 0) && top0 > ws.fr[0].base) {
        const int b = ws.fr[0].base;
        if (warp_export(P, ws, th, n, ws.stL[b], ws.stS[b])) ws.fr[0].base = b + 1;
      }
    }
    if (skip_count) skip_count = false;
    else ++st.nodes;
    WFrame& F = ws.fr[f];
    int d0, d1;
    WPROF(long long c0 = clock64());
    const int E = w_fixpoint(ws, q, L, S, F.best, d0, d1, st);
    WPROF(long long c1 = clock64(); st.c_fix += (unsigned long long)(c1 - c0));
    have = false;
    if (E < 0) continue;
    {
      const long long rem = (long long)F.best - S - 1;
      if ((long long)E > rem * rem) continue;  // stopping rule (engine.py:296)
    }
    if (E == 0) {
      if (S < F.best) {
        F.best = S;
        F.ach = 1;
        if (f == 0 && lane == 0) reg_submit(P, th.scope, th.S + S, true, kNoWitness);
      }
      continue;
    }
    // --------------------------------------------------- components --
    M comp = w_component(q, L, wlsb(L));
    WPROF(c0 = clock64(); st.c_comp += (unsigned long long)(c0 - c1));
    if (comp != L) {
      ++st.splits;
      int special = 0, ng = 0, ncomp = 0;
      // pend[] is a stack: frames <= f own everything below F.pend_e; the
      // general components are staged at pend[pbase ..] in discovery order
      const int pbase = F.pend_e;
      M rest = L;
      bool overflow = false;
      while (true) {
        ++ncomp;
        const int size = wpopc(comp);
        const bool in0 = whas(comp, q.v0), in1 = whas(comp, q.v1);
        if (!wballot<M>(in0 && d0 != size - 1, in1 && d1 != size - 1)) {
          special += size - 1;  // clique: all but one vertex
          st.rules[4] += 1;
        } else if (size >= 3 && !wballot<M>(in0 && d0 != 2, in1 && d1 != 2)) {
          special += (size + 1) / 2;  // chordless cycle
          st.rules[5] += 1;
        } else {
          if (pbase + ng < kWPend) ws.pend[pbase + ng] = comp;
          else overflow = true;
          ++ng;
        }
        rest &= ~comp;
        if (!rest) break;
        comp = w_component(q, rest, wlsb(rest));
      }
      if (lane == 0) atomicAdd(&P.hist[ncomp < P.n + 1 ? ncomp : P.n + 1], 1ull);
      WPROF(st.c_split += (unsigned long long)(clock64() - c0));
      const int base_S = S + special;
      if (ng == 0) {
        if (base_S < F.best) {
          F.best = base_S;
          F.ach = 1;
          if (f == 0 && lane == 0) reg_submit(P, th.scope, th.S + base_S, true, kNoWitness);
        }
        continue;
      }
      if (base_S + ng >= F.best) continue;  // every general component needs >= 1
      if (ng == 1) {
        L = (M)ws.pend[pbase];
        S = base_S;
        have = true;
        continue;
      }
      if (overflow || nf >= kWFrames) {
        if (lane == 0) {
          atomicExch(&P.ctl->error, 8);
          atomicExch(&P.ctl->stop, 1);
        }
        return false;
      }
      // new frame: solve pend[pbase] now, the rest afterwards (popped from
      // the end, so store them reversed to keep discovery order)
      const M first = (M)ws.pend[pbase];
      for (int i = 1, j = ng - 1; i < j; ++i, --j) {
        const unsigned long long t = ws.pend[pbase + i];
        ws.pend[pbase + i] = ws.pend[pbase + j];
        ws.pend[pbase + j] = t;
      }
      WFrame& G = ws.fr[nf++];
      G.running = base_S;
      G.pend_b = pbase + 1;
      G.pend_e = pbase + ng;
      const int bound = F.best - base_S - (ng - 1);
      const int size = wpopc(first);
      if (size - 1 < bound) {
        G.best = size - 1;
        G.ach = 1;
      } else {
        G.best = bound;
        G.ach = 0;
      }
      G.base = sp;
      L = first;
      S = 0;
      have = true;
      continue;
    }
    // ------------------------------------------------------- branch --
    // pure.py:241 select_max_degree (lowest index on ties)
    unsigned k0 = d0 > 0 ? ((unsigned)d0 << 7) | (127u - q.v0) : 0u;
    unsigned k1 = d1 > 0 ? ((unsigned)d1 << 7) | (127u - q.v1) : 0u;
    const unsigned key = __reduce_max_sync(0xffffffffu, k0 > k1 ? k0 : k1);
    const int v = 127 - (int)(key & 127u);
    const M nv = (M)ws.adj[v] & L;
    // engine.py:319: exclude child (v out, N(v) in) to the stack, include
    // child (v in) continues here
    const int Sx = S + wpopc(nv);
    if (Sx < F.best) {
      if (sp >= kWStack) {
        if (lane == 0) {
          atomicExch(&P.ctl->error, 8);
          atomicExch(&P.ctl->stop, 1);
        }
        return false;
      }
      ws.stL[sp] = L & ~(nv | wbit<M>(v));
      ws.stS[sp] = Sx;
      ++sp;
    }
    L &= ~wbit<M>(v);
    S += 1;
    have = true;
  }
  return true;
}

// One warp-tier epoch of a block (all threads call it, block-uniformly).
// Every warp takes tasks from the ring and solves them; a warp leaves once
// the ring is empty and no warp of its block is still busy (new tasks can
// only come from busy blocks), or as soon as node-level work is queued (the
// block is needed there), or on stop.  Returns whether the block ran a task.
__device__ inline bool warp_epoch(const SearchParams& P, WarpWs* wws, int* busy, WStats& st) {
  const int lane = threadIdx.x & 31;
  WarpWs& ws = wws[threadIdx.x >> 5];
  bool any = false;
  unsigned backoff = 64;
  while (true) {
    long long pos = -1;
    int stop = 0, node_work = 0;
    if (lane == 0) {
      stop = ld_relaxed(&P.ctl->stop);
      node_work = (long long)ld_relaxed_u64(P.q.count) > 0;
      if (!stop && !node_work) {
        pos = q_reserve_pop(P.bq);
        if (pos >= 0) atomicAdd(busy, 1);
      }
    }
    pos = __shfl_sync(0xffffffffu, pos, 0);
    stop = __shfl_sync(0xffffffffu, stop, 0);
    node_work = __shfl_sync(0xffffffffu, node_work, 0);
    if (stop) break;
    if (pos < 0) {
      int b = 0;
      if (lane == 0) b = *(volatile int*)busy;
      b = __shfl_sync(0xffffffffu, b, 0);
      if (node_work || b == 0) break;
      if (lane == 0) __nanosleep(backoff);
      backoff = backoff < 2048 ? backoff * 2 : 2048;
      __syncwarp();
      continue;
    }
    backoff = 64;
    any = true;
    const char* slot = P.bq.data + (pos % P.bq.cap) * kWSlotBytes;
    const int4 h = __ldcg((const int4*)slot);
    const WTaskHdr th{h.x, h.y, h.z, h.w, __ldcg((const unsigned long long*)(slot + 16)), 0ull};
    const int n = th.n & 0xffff;
    const unsigned long long* src = (const unsigned long long*)(slot + kWHdrBytes);
    for (int i = lane; i < n; i += 32) ws.adj[i] = __ldcg(src + i);
    __syncwarp();
    if (lane == 0) q_release_pop(P.bq, pos);
    const long long t0 = clock64();
    const unsigned long long nodes0 = st.nodes;
    if (lane == 0) atomicMin(&P.ctl->t_task_first, globaltimer());
    if (n <= 32) warp_solve_task<unsigned>(P, ws, th, st);
    else warp_solve_task<unsigned long long>(P, ws, th, st);
    __syncwarp();
    if (lane == 0) {
      reg_finish(P, th.scope);  // the task's live unit on its scope
      atomicSub(busy, 1);
    }
    const unsigned long long dt = (unsigned long long)(clock64() - t0);
    st.tasks += 1;
    st.cyc += dt;
    if (dt > st.maxcyc) {
      st.maxcyc = dt;
      st.max_nodes = st.nodes - nodes0;
      st.max_n = n;
    }
    if (lane == 0) atomicMax(&P.ctl->t_task_last, globaltimer());
  }
  return __syncthreads_or(any);
}

// end of the kernel: lane 0 of every warp adds its counters
__device__ inline void warp_flush_stats(const SearchParams& P, const WStats& st) {
  if ((threadIdx.x & 31) != 0 || !P.warp_limit) return;
  Ctl* c = P.ctl;
  atomicAdd(&c->nodes, st.nodes);
  atomicAdd(&c->comp_branches, st.splits);
  for (int i = 0; i < 6; ++i)
    if (st.rules[i]) atomicAdd(&c->rules[i], st.rules[i]);
  atomicAdd(&c->wtasks, st.tasks);
  atomicAdd(&c->wnodes, st.nodes);
  atomicAdd(&c->wcyc, st.cyc);
  atomicAdd(&c->wc_fix, st.c_fix);
  atomicAdd(&c->wc_comp, st.c_comp);
  atomicAdd(&c->wc_split, st.c_split);
  atomicAdd(&c->wc_iter, st.c_iter);
  if (atomicMax(&c->wmax, st.maxcyc) < st.maxcyc) {
    c->wmax_nodes = st.max_nodes;
    c->wmax_n = st.max_n;
  }
}

// release the live units of tasks still queued after a stop
__device__ inline void warp_ring_drain(const SearchParams& P) {
  while (true) {
    const long long pos = q_reserve_pop(P.bq);
    if (pos < 0) break;
    const int scope = __ldcg((const int*)(P.bq.data + (pos % P.bq.cap) * kWSlotBytes) + 1);
    q_release_pop(P.bq, pos);
    reg_finish(P, scope);
  }
}

}  // namespace vcg
