// Warp tier of the search: a subproblem with at most 128 live vertices is
// solved by ONE warp as bitmask branch-and-reduce.
//
// Why: on the component-splitting workloads (configs[1], the RGG) the search
// nodes hold ~13 live vertices on average while their degree-array window
// spans ~540 vertices of the reduced graph (87% of the nodes have <= 32 live
// vertices, 97.6% <= 64).  A whole thread block sweeping a 1 KB degree
// record per node is the wrong granularity for them.  Here a task is the
// induced subgraph itself -- up to 128 adjacency bitmasks held in registers,
// one to four rows per lane -- and a search node is a live mask plus a
// cover count, so a node costs a few hundred warp instructions and no block
// barrier, HBM record or registry atomic.  Masks are 32, 64 or 128 bits wide
// by task size: dense instances (configs[4]) have most of their search
// nodes at 65-128 live vertices, which the 128-bit tier takes off the block
// tier.
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
// idle warps poll the task ring with exponential backoff (ns)
#ifndef VCG_EPOCH_STICKY
#define VCG_EPOCH_STICKY 1
#endif
#ifndef VCG_WBACKOFF_MIN
#define VCG_WBACKOFF_MIN 64
#endif
#ifndef VCG_WBACKOFF_MAX
#define VCG_WBACKOFF_MAX 2048
#endif
#ifdef VCG_TASK_TRACE  // per-task printf of the slow tasks (diagnostic builds)
#define TTRACE(...) __VA_ARGS__
#else
#define TTRACE(...)
#endif
#ifdef VCG_WARP_PROFILE
#define WPROF(...) __VA_ARGS__
#else
#define WPROF(...)
#endif

constexpr int kWMax = 256;            // vertices per warp task
constexpr int kWFrames = 24;          // nested component frames (each >= 6 vertices)
constexpr int kWTierWarps = 8;        // warps of a block that runs the warp tier (<= 256 threads)
constexpr int kWPend = 32;            // pending component masks over all frames

// warp-task record: 32 B header, adjacency rows of n vertices (each row
// wrows(n) 64-bit words: 1 for n <= 64, 2 up to 128, 4 up to 256), then
// the live mask's words beyond the first two
struct WTaskHdr {  // (the root's live mask follows at +16 / after the rows: WarpWsT::live0)
  int S;      // cover size of the task's root within its registry scope
  int scope;  // registry entry the task reports to (it holds one live unit)
  int n;      // vertices | (root already counted as a tree node) << 16
  int depth;
};
constexpr long long kWHdrBytes = 32;
__host__ __device__ __forceinline__ int wrows(int n) { return n > 128 ? 4 : n > 64 ? 2 : 1; }
// bytes of a ring slot for tasks of up to `limit` vertices
__host__ __device__ __forceinline__ long long wslot_bytes(int limit) {
  return (kWHdrBytes + 8LL * wrows(limit) * limit + 16 + 15) & ~15LL;  // 16 B aligned
}
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

// per-warp shared-memory workspace for tasks of up to 64 * WW vertices;
// masks are stored as WW 64-bit words (the 64-vertex layout keeps the
// round-1 footprint, so the launch plan of sparse workloads is unchanged)
template <int WW>
struct WarpWsT {
  static constexpr int kW = WW;
  static constexpr int kMax = 64 * WW;
  static constexpr int kStack = kMax + 8;  // DFS depth <= kMax
  unsigned long long adj[WW * kMax];
  unsigned long long stL[WW * kStack];
  unsigned long long pend[WW * kWPend];
  int stS[kStack];
  WFrame fr[kWFrames];
  unsigned long long live0[WW];  // the task root's live mask
};
using WarpWs1 = WarpWsT<1>;
using WarpWs2 = WarpWsT<2>;
using WarpWs4 = WarpWsT<4>;

struct WStats {
  unsigned long long tasks, nodes, splits, cyc, maxcyc, max_nodes, max_n;
  unsigned long long c_fix, c_comp, c_split;  // cycles in the node phases
  unsigned long long c_iter;                   // fixpoint loop iterations
  unsigned long long rules[6];
  unsigned long long t_exp, t_rsplit, t_wait, t_rfail;  // VCG_TASK_TRACE, per task
  unsigned long long t_ph[8];                           // split phases (VCG_TASK_TRACE)
};

// ------------------------------------------------------------ masks --
// Three task widths: <= 32 vertices on 32-bit masks (one vertex per lane),
// <= 64 on 64-bit masks (two per lane), <= 128 on 128-bit masks (four per
// lane).  Lane l owns vertices l + 32 r; the ballot of every lane's r-th
// vertex is bits [32 r, 32 r + 32) of a mask, so a collective over the
// warp's vertices is R ballots / OR-reductions, no cross-lane shuffles.
struct W128 {
  unsigned long long lo, hi;
};
__device__ __forceinline__ W128 operator&(W128 a, W128 b) { return {a.lo & b.lo, a.hi & b.hi}; }
__device__ __forceinline__ W128 operator|(W128 a, W128 b) { return {a.lo | b.lo, a.hi | b.hi}; }
__device__ __forceinline__ W128 operator~(W128 a) { return {~a.lo, ~a.hi}; }
__device__ __forceinline__ W128& operator&=(W128& a, W128 b) { a = a & b; return a; }
__device__ __forceinline__ W128& operator|=(W128& a, W128 b) { a = a | b; return a; }
__device__ __forceinline__ bool operator==(W128 a, W128 b) { return a.lo == b.lo && a.hi == b.hi; }
__device__ __forceinline__ bool operator!=(W128 a, W128 b) { return !(a == b); }

struct W256 {
  unsigned long long w[4];
};
__device__ __forceinline__ W256 operator&(const W256& a, const W256& b) {
  return {{a.w[0] & b.w[0], a.w[1] & b.w[1], a.w[2] & b.w[2], a.w[3] & b.w[3]}};
}
__device__ __forceinline__ W256 operator|(const W256& a, const W256& b) {
  return {{a.w[0] | b.w[0], a.w[1] | b.w[1], a.w[2] | b.w[2], a.w[3] | b.w[3]}};
}
__device__ __forceinline__ W256 operator~(const W256& a) {
  return {{~a.w[0], ~a.w[1], ~a.w[2], ~a.w[3]}};
}
__device__ __forceinline__ W256& operator&=(W256& a, const W256& b) { a = a & b; return a; }
__device__ __forceinline__ W256& operator|=(W256& a, const W256& b) { a = a | b; return a; }
__device__ __forceinline__ bool operator==(const W256& a, const W256& b) {
  return a.w[0] == b.w[0] && a.w[1] == b.w[1] && a.w[2] == b.w[2] && a.w[3] == b.w[3];
}
__device__ __forceinline__ bool operator!=(const W256& a, const W256& b) { return !(a == b); }

template <typename M> struct WT;
template <> struct WT<unsigned> { static constexpr int R = 1; };
template <> struct WT<unsigned long long> { static constexpr int R = 2; };
template <> struct WT<W128> { static constexpr int R = 4; };
template <> struct WT<W256> { static constexpr int R = 8; };

__device__ __forceinline__ bool nz(unsigned x) { return x != 0u; }
__device__ __forceinline__ bool nz(unsigned long long x) { return x != 0ull; }
__device__ __forceinline__ bool nz(W128 x) { return (x.lo | x.hi) != 0ull; }
__device__ __forceinline__ bool nz(const W256& x) {
  return (x.w[0] | x.w[1] | x.w[2] | x.w[3]) != 0ull;
}

__device__ __forceinline__ unsigned long long wor64(unsigned long long x) {
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)x);
  const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(x >> 32));
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned wor(unsigned x) { return __reduce_or_sync(0xffffffffu, x); }
__device__ __forceinline__ unsigned long long wor(unsigned long long x) { return wor64(x); }
__device__ __forceinline__ W128 wor(W128 x) { return {wor64(x.lo), wor64(x.hi)}; }
__device__ __forceinline__ W256 wor(const W256& x) {
  return {{wor64(x.w[0]), wor64(x.w[1]), wor64(x.w[2]), wor64(x.w[3])}};
}
__device__ __forceinline__ int wpopc(unsigned x) { return __popc(x); }
__device__ __forceinline__ int wpopc(unsigned long long x) { return __popcll(x); }
__device__ __forceinline__ int wpopc(W128 x) { return __popcll(x.lo) + __popcll(x.hi); }
__device__ __forceinline__ int wpopc(const W256& x) {
  return __popcll(x.w[0]) + __popcll(x.w[1]) + __popcll(x.w[2]) + __popcll(x.w[3]);
}
__device__ __forceinline__ int wlsb(unsigned x) { return __ffs((int)x) - 1; }
__device__ __forceinline__ int wlsb(unsigned long long x) { return __ffsll((long long)x) - 1; }
__device__ __forceinline__ int wlsb(W128 x) {
  return x.lo ? __ffsll((long long)x.lo) - 1 : (x.hi ? 63 + __ffsll((long long)x.hi) : -1);
}
__device__ __forceinline__ int wlsb(const W256& x) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (x.w[i]) return 64 * i + __ffsll((long long)x.w[i]) - 1;
  return -1;
}
__device__ __forceinline__ int wmsb(unsigned x) { return 31 - __clz((int)x); }
__device__ __forceinline__ int wmsb(unsigned long long x) { return 63 - __clzll((long long)x); }
__device__ __forceinline__ int wmsb(W128 x) {
  return x.hi ? 127 - __clzll((long long)x.hi) : 63 - __clzll((long long)x.lo);
}
__device__ __forceinline__ int wmsb(const W256& x) {
#pragma unroll
  for (int i = 3; i >= 0; --i)
    if (x.w[i]) return 64 * i + 63 - __clzll((long long)x.w[i]);
  return -1;
}
__device__ __forceinline__ unsigned wclr(unsigned x) { return x & (x - 1u); }
__device__ __forceinline__ unsigned long long wclr(unsigned long long x) { return x & (x - 1ull); }
__device__ __forceinline__ W128 wclr(W128 x) {
  return x.lo ? W128{x.lo & (x.lo - 1ull), x.hi} : W128{0ull, x.hi & (x.hi - 1ull)};
}
__device__ __forceinline__ W256 wclr(W256 x) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (x.w[i]) {
      x.w[i] &= x.w[i] - 1ull;
      break;
    }
  return x;
}
// set bits of c below position u
__device__ __forceinline__ int wrank(unsigned c, int u) { return __popc(c & ((1u << u) - 1u)); }
__device__ __forceinline__ int wrank(unsigned long long c, int u) {
  return __popcll(c & ((1ull << u) - 1ull));
}
__device__ __forceinline__ int wrank(W128 c, int u) {
  return u < 64 ? __popcll(c.lo & ((1ull << u) - 1ull))
                : __popcll(c.lo) + __popcll(c.hi & ((1ull << (u - 64)) - 1ull));
}
__device__ __forceinline__ int wrank(const W256& c, int u) {
  int r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int lo = 64 * i;
    if (u >= lo + 64) r += __popcll(c.w[i]);
    else if (u > lo) r += __popcll(c.w[i] & ((1ull << (u - lo)) - 1ull));
  }
  return r;
}
template <typename M>
__device__ __forceinline__ M wbit(int i);
template <>
__device__ __forceinline__ unsigned wbit<unsigned>(int i) { return 1u << i; }
template <>
__device__ __forceinline__ unsigned long long wbit<unsigned long long>(int i) { return 1ull << i; }
template <>
__device__ __forceinline__ W128 wbit<W128>(int i) {
  return i < 64 ? W128{1ull << i, 0ull} : W128{0ull, 1ull << (i - 64)};
}
template <>
__device__ __forceinline__ W256 wbit<W256>(int i) {
  const unsigned long long b = 1ull << (i & 63);
  const int k = i >> 6;  // selects, not an indexed store (which would go to local memory)
  return {{k == 0 ? b : 0ull, k == 1 ? b : 0ull, k == 2 ? b : 0ull, k == 3 ? b : 0ull}};
}
// vertex v live in L (v >= the mask width: never)
__device__ __forceinline__ bool whas(unsigned L, int v) { return v < 32 && ((L >> v) & 1u); }
__device__ __forceinline__ bool whas(unsigned long long L, int v) { return v < 64 && ((L >> v) & 1ull); }
__device__ __forceinline__ bool whas(W128 L, int v) {
  return v < 64 ? ((L.lo >> v) & 1ull) : (v < 128 && ((L.hi >> (v - 64)) & 1ull));
}
__device__ __forceinline__ bool whas(const W256& L, int v) {
  const int k = v >> 6;
  const unsigned long long w = k == 0 ? L.w[0] : k == 1 ? L.w[1] : k == 2 ? L.w[2] : L.w[3];
  return v < 256 && ((w >> (v & 63)) & 1ull);
}
// bits [32 j, 32 j + 32) of a mask: the lane-indexed ballot word of the
// lanes' j-th vertices (j is a compile-time constant in the unrolled loops)
__device__ __forceinline__ unsigned wchunk(unsigned x, int) { return x; }
__device__ __forceinline__ unsigned wchunk(unsigned long long x, int j) {
  return (unsigned)(x >> (32 * j));
}
__device__ __forceinline__ unsigned wchunk(W128 x, int j) {
  return (unsigned)((j < 2 ? x.lo : x.hi) >> (32 * (j & 1)));
}
__device__ __forceinline__ unsigned wchunk(const W256& x, int j) {
  return (unsigned)(x.w[j >> 1] >> (32 * (j & 1)));
}
// the lane's own j-th vertex (lane + 32 j) is in x: one shift, no range tests
template <typename M>
__device__ __forceinline__ bool wown(const M& x, int j, int lane) {
  return (wchunk(x, j) >> lane) & 1u;
}
// mask from per-lane predicates p[r] on the lane's r-th vertex
template <typename M>
__device__ __forceinline__ M wballot(const bool (&p)[WT<M>::R]);
template <>
__device__ __forceinline__ unsigned wballot<unsigned>(const bool (&p)[1]) {
  return __ballot_sync(0xffffffffu, p[0]);
}
template <>
__device__ __forceinline__ unsigned long long wballot<unsigned long long>(const bool (&p)[2]) {
  return (unsigned long long)__ballot_sync(0xffffffffu, p[0]) |
         ((unsigned long long)__ballot_sync(0xffffffffu, p[1]) << 32);
}
template <>
__device__ __forceinline__ W128 wballot<W128>(const bool (&p)[4]) {
  return {(unsigned long long)__ballot_sync(0xffffffffu, p[0]) |
              ((unsigned long long)__ballot_sync(0xffffffffu, p[1]) << 32),
          (unsigned long long)__ballot_sync(0xffffffffu, p[2]) |
              ((unsigned long long)__ballot_sync(0xffffffffu, p[3]) << 32)};
}
template <>
__device__ __forceinline__ W256 wballot<W256>(const bool (&p)[8]) {
  W256 r;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    r.w[i] = (unsigned long long)__ballot_sync(0xffffffffu, p[2 * i]) |
             ((unsigned long long)__ballot_sync(0xffffffffu, p[2 * i + 1]) << 32);
  return r;
}
// masks in the workspace: WW 64-bit words each
template <typename M>
__device__ __forceinline__ M wload(const unsigned long long* p);
template <>
__device__ __forceinline__ unsigned wload<unsigned>(const unsigned long long* p) { return (unsigned)p[0]; }
template <>
__device__ __forceinline__ unsigned long long wload<unsigned long long>(const unsigned long long* p) {
  return p[0];
}
template <>
__device__ __forceinline__ W128 wload<W128>(const unsigned long long* p) { return {p[0], p[1]}; }
template <>
__device__ __forceinline__ W256 wload<W256>(const unsigned long long* p) {
  return {{p[0], p[1], p[2], p[3]}};
}
template <int WW>
__device__ __forceinline__ void wstore(unsigned long long* p, unsigned x) {
  p[0] = x;
#pragma unroll
  for (int i = 1; i < WW; ++i) p[i] = 0ull;
}
template <int WW>
__device__ __forceinline__ void wstore(unsigned long long* p, unsigned long long x) {
  p[0] = x;
#pragma unroll
  for (int i = 1; i < WW; ++i) p[i] = 0ull;
}
template <int WW>
__device__ __forceinline__ void wstore(unsigned long long* p, W128 x) {
  p[0] = x.lo;
  if (WW > 1) p[1] = x.hi;
  if (WW > 2) p[2] = p[3] = 0ull;
}
template <int WW>
__device__ __forceinline__ void wstore(unsigned long long* p, const W256& x) {
#pragma unroll
  for (int i = 0; i < WW; ++i) p[i] = x.w[i];
}

// Per-lane view of the task graph: this lane owns vertices lane + 32 r.
// Rows of up to 128-bit tasks are held in registers; the 256-bit tier's
// eight 256-bit rows per lane stay in the workspace and are read on use.
template <typename M>
struct WLane {
  M a[WT<M>::R];    // adjacency rows of the lane's vertices (0 beyond n)
  int v[WT<M>::R];
  __device__ __forceinline__ M row(int j) const { return a[j]; }
};
template <>
struct WLane<W256> {
  const unsigned long long* adj;  // the workspace rows, 4 words each
  int n;
  int v[8];
  __device__ __forceinline__ W256 row(int j) const {
    return v[j] < n ? wload<W256>(adj + 4 * v[j]) : W256{{0ull, 0ull, 0ull, 0ull}};
  }
};

// Connected component of the live mask L containing r (frontier BFS, one
// OR-reduction per level).
template <typename M>
__device__ __forceinline__ M w_component(const WLane<M>& q, M L, int r) {
  M comp = wbit<M>(r), fr = comp;
  while (nz(fr)) {
    M c{};
#pragma unroll
    for (int j = 0; j < WT<M>::R; ++j)
      if (wown(fr, j, q.v[0])) c |= q.row(j);
    fr = wor(c) & L & ~comp;
    comp |= fr;
  }
  return comp;
}

// Rules to a joint fixpoint on (L, S) under the bound `best` (pure.py:188
// reduce_fixpoint: degree-one, degree-two triangle, high degree).  Leaves d
// = current degrees of the lane's vertices.  Returns the edge count, or -1
// when S reached the bound (prune).
template <typename M, typename WS>
__device__ __forceinline__ int w_fixpoint(const WS& ws, const WLane<M>& q, M& L, int& S,
                                          int best, int (&d)[WT<M>::R], WStats& st) {
  constexpr int R = WT<M>::R;
  // Isolated vertices stay in L during the loop (no live row contains them,
  // so no rule sees them) and leave it once, at the fixpoint.
  bool p[R];
  while (true) {
    WPROF(++st.c_iter);
#pragma unroll
    for (int j = 0; j < R; ++j) d[j] = wown(L, j, q.v[0]) ? wpopc(q.row(j) & L) : 0;
    const int k = best - S - 1;  // vertices an improving cover may still take
    if (k < 0) return -1;
    // degree one (pure.py:82): the neighbour of a pendant vertex is forced;
    // of an isolated edge only the higher end (the in-order sweep's choice).
    // High degree (pure.py:158) on the same snapshot: a vertex of degree > k
    // is in every cover that still improves the bound.  Both at once is
    // sound -- every improving cover holds H, and the pendant exchange
    // argument never removes a vertex of H (degree 1 <= k) -- and saves the
    // rescan between them (the node-level sweeps keep the reference's
    // order; the warp tier only runs in parallel mode).
#pragma unroll
    for (int j = 0; j < R; ++j) p[j] = d[j] == 1;
    const M p1 = wballot<M>(p);
#pragma unroll
    for (int j = 0; j < R; ++j) p[j] = d[j] > k;
    const M H = wballot<M>(p);
    if (nz(p1 | H)) {
      M F = H;
      if (nz(p1)) {
        M c{};
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (d[j] == 1) {
            const M nb = q.row(j) & L;  // the single live neighbour
            if (!nz(nb & p1) || wlsb(nb) > q.v[j]) c |= nb;
          }
        F |= wor(c);
      }
      L &= ~F;
      const int nf = wpopc(F), nh = wpopc(H);
      S += nf;
      st.rules[0] += nf - nh;
      st.rules[2] += nh;
      continue;
    }
    // degree-two triangle (pure.py:113): in index order with revalidation.
    // Validity (the two neighbours adjacent) is decided by every lane for
    // its own vertices from the neighbour's row in the workspace; the
    // in-order walk then only visits valid candidates, and a later
    // candidate stays applicable iff it and its two neighbours are still
    // live (a removal only deletes vertices, so its degree cannot stay 2
    // otherwise).
    {
      int ab[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        p[j] = false;
        ab[j] = -1;
        if (d[j] == 2) {
          const M nb = q.row(j) & L;
          const int x = wlsb(nb), y = wmsb(nb);
          p[j] = whas(wload<M>(&ws.adj[WS::kW * x]), y);
          ab[j] = x | (y << 8);
        }
      }
      M T = wballot<M>(p);
      if (nz(T)) {
        M Rm{};  // vertices removed by this sweep
        int applied = 0;
        while (nz(T)) {
          const int v = wlsb(T);
          T = wclr(T);
          int mine = ab[0];
#pragma unroll
          for (int j = 1; j < R; ++j)
            if ((v >> 5) == j) mine = ab[j];
          const int abv = __shfl_sync(0xffffffffu, mine, v & 31);
          // v leaves too (isolated once its neighbours are in)
          const M tri = wbit<M>(v) | wbit<M>(abv & 255) | wbit<M>(abv >> 8);
          if (nz(tri & Rm)) continue;
          Rm |= tri;
          ++applied;
        }
        // cover gains exactly the two neighbours per applied triangle
        L &= ~Rm;
        S += 2 * applied;
        st.rules[1] += applied;
        continue;
      }
    }
    break;
  }
#pragma unroll
  for (int j = 0; j < R; ++j) p[j] = d[j] > 0;
  L = wballot<M>(p);  // isolated vertices leave the graph
  int sum = 0;
#pragma unroll
  for (int j = 0; j < R; ++j) sum += d[j];
  return __reduce_add_sync(0xffffffffu, sum) >> 1;
}

// Push (adjacency of this task, live mask L = two words at Lw) as a new task
// on the same scope with cover offset th.S + Sl.  false: ring full.
template <typename WS>
__device__ inline bool warp_export(const SearchParams& P, const WS& ws, const WTaskHdr& th,
                                   int n, const unsigned long long* Lw, int Sl) {
  const int lane = threadIdx.x & 31;
  long long pos = -1;
  if (lane == 0) pos = q_reserve_push(P.bq, P.bq.cap);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  if (pos < 0) return false;
  char* slot = P.bq.data + (pos % P.bq.cap) * P.bq_slot;
  unsigned long long* dst = (unsigned long long*)(slot + kWHdrBytes);
  const int W = wrows(n);
  for (int i = lane; i < n * W; i += 32) __stcg(dst + i, ws.adj[WS::kW * (i / W) + i % W]);
  if (lane == 0) {
    __stcg((int4*)slot, make_int4(th.S + Sl, th.scope, n, th.depth + 1));
    __stcg((ulonglong2*)(slot + 16), make_ulonglong2(Lw[0], WS::kW > 1 ? Lw[1] : 0ull));
    if (W > 2) __stcg((ulonglong2*)(dst + n * W), make_ulonglong2(Lw[2], Lw[3]));
    atomicAdd(&P.reg.live[th.scope], 1);  // before the task can finish it
  }
  __syncwarp();
  if (lane == 0) q_publish_push(P.bq, pos);
  return true;
}

// Write component c of the current task as a new task at ring ticket pos:
// its vertices renumbered in increasing order (lowest-index tie-breaks are
// unchanged), rows restricted to c and compacted, so a small component runs
// on narrow masks.
template <typename M, typename WS>
__device__ inline long long warp_emit_component(const SearchParams& P, const WS& ws, M c, int scope,
                                                int depth, long long pos) {
  const int lane = threadIdx.x & 31;
  const int sz = wpopc(c);
  const int Wn = wrows(sz);
  char* slot = P.bq.data + (pos % P.bq.cap) * P.bq_slot;
  unsigned long long* dst = (unsigned long long*)(slot + kWHdrBytes);
  // Each lane packs the rows of its own vertices (lane + 32 r), at their
  // ranks in c.  (A walk over c in which lane j % 32 packed row j diverged
  // at every step, so the warp issued the whole walk 32 times over: ~300 k
  // cycles per emitted component in the 256-bit tier.)
#pragma unroll
  for (int r = 0; r < WT<M>::R; ++r) {
    const int v = lane + 32 * r;
    if (!wown(c, r, lane)) continue;
    const int j = wrank(c, v);
    M rw = wload<M>(&ws.adj[WS::kW * v]) & c;
    unsigned long long o0 = 0ull, o1 = 0ull, o2 = 0ull, o3 = 0ull;
    while (nz(rw)) {
      const int b = wrank(c, wlsb(rw));
      rw = wclr(rw);
      const unsigned long long bit = 1ull << (b & 63);
      const int k = b >> 6;
      o0 |= k == 0 ? bit : 0ull;
      o1 |= k == 1 ? bit : 0ull;
      o2 |= k == 2 ? bit : 0ull;
      o3 |= k == 3 ? bit : 0ull;
    }
    __stcg(dst + Wn * j, o0);
    if (Wn > 1) __stcg(dst + Wn * j + 1, o1);
    if (Wn > 2) {
      __stcg(dst + Wn * j + 2, o2);
      __stcg(dst + Wn * j + 3, o3);
    }
  }
  if (lane == 0) {
    __stcg((int4*)slot, make_int4(0, scope, sz, depth));
    unsigned long long lv[4];
    for (int j = 0; j < 4; ++j) {
      const int rr = sz - 64 * j;
      lv[j] = rr >= 64 ? ~0ull : rr > 0 ? ((1ull << rr) - 1) : 0ull;
    }
    __stcg((ulonglong2*)(slot + 16), make_ulonglong2(lv[0], lv[1]));
    if (Wn > 2) __stcg((ulonglong2*)(dst + sz * Wn), make_ulonglong2(lv[2], lv[3]));
  }
  __syncwarp();
  TTRACE(const long long tp = clock64());
  if (lane == 0) q_publish_push(P.bq, pos);
  TTRACE(__syncwarp(); return clock64() - tp);
  return 0;
}

// A frame-0 node of a wide task that splits into ng >= 2 general components
// (staged at pend[pbase, pbase + ng)): hand them to the registry like a
// block-level split (engine.py:334 _try_component_split, search_impl.cuh
// try_split) -- a parent entry on the task's scope holding the node's cover
// S_abs plus the folded special components, one child entry and one compacted
// task per component -- instead of solving them one after another inside this
// warp.  The components then run on any warp in parallel: a wide task's
// subtree no longer serialises on the warp that started it.  false: no ring
// room (the caller solves them in place as nested frames).
template <typename M, typename WS>
__device__ inline bool warp_registry_split(const SearchParams& P, WS& ws, const WTaskHdr& th,
                                           int pbase, int ng, int S_abs, int special,
                                           int best_abs, WStats& st) {
  TTRACE(long long tq = clock64());
  constexpr int K = WS::kW;
  const int lane = threadIdx.x & 31;
  const Registry& R = P.reg;
  // each component may take at most this many vertices for the node to
  // improve the scope's bound (the others need >= 1 each)
  const int room = best_abs - S_abs - special - (ng - 1);
  long long pos = -1;
  int p = -1;
  if (lane == 0) {
    p = reg_alloc(R, 1 + ng);
    if (p < 0) {
      atomicExch(&P.ctl->error, 1);
      atomicExch(&P.ctl->stop, 1);
    } else {
      pos = q_reserve_push_n(P.bq, ng, P.bq.cap);
      if (pos < 0) {
        R.nchild[p] = ng;  // the free list reads the group size from it
        reg_free_group(R, p);
        p = -2;
      }
    }
  }
  p = __shfl_sync(0xffffffffu, p, 0);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  if (p == -2) return false;
  if (p < 0) return true;  // registry exhausted: the search stops
  TTRACE(st.t_ph[0] += clock64() - tq; tq = clock64());
  if (lane == 0) {
    atomicAdd(&R.live[th.scope], 1);  // the parent entry's reference on the scope
    R.kind[p] = 1;
    R.sum[p] = S_abs + special;
    R.sum_ach[p] = 1;
    R.init_sum[p] = S_abs;
    R.folded[p] = special;
    R.live[p] = 1 + ng;
    R.link[p] = th.scope;
    R.first_child[p] = p + 1;
    R.nchild[p] = ng;
    R.disc_done[p] = 0;
    R.key[p] = 0;
    R.child_folded[p] = 0;
    for (int j = 0; j < ng; ++j) {
      const int size = wpopc(wload<M>(&ws.pend[K * (pbase + j)]));
      int init = room < size - 1 ? room : size - 1;
      if (init < 1) init = 1;
      const int c = p + 1 + j;
      R.kind[c] = 0;
      R.key[c] = init * 2 + (init == size - 1 ? 0 : 1);
      R.live[c] = 1;
      R.link[c] = p;
      R.child_folded[c] = 0;
      R.disc_done[c] = 0;
    }
    __threadfence();
  }
  __syncwarp();
  TTRACE(st.t_ph[1] += clock64() - tq; tq = clock64());
  for (int j = 0; j < ng; ++j) {
    if (lane == 0) q_wait_free(P.bq, pos + j);
    __syncwarp();
    TTRACE(st.t_ph[2] += clock64() - tq; tq = clock64());
    const long long tpub = warp_emit_component<M, WS>(P, ws, wload<M>(&ws.pend[K * (pbase + j)]), p + 1 + j,
                               th.depth + 1, pos + j);
    (void)tpub;
    TTRACE(st.t_ph[7] += tpub; st.t_ph[5] += 1; st.t_ph[6] += wpopc(wload<M>(&ws.pend[K * (pbase + j)])));
    TTRACE(st.t_ph[3] += clock64() - tq; tq = clock64());
  }
  if (lane == 0) {
    __threadfence();
    st_release(&R.disc_done[p], 1);
    if (atomicSub(&R.live[p], 1) == 1) reg_cascade(P, p);
  }
  __syncwarp();
  TTRACE(st.t_ph[4] += clock64() - tq);
  return true;
}

// Solve one task to completion (or until the stop flag).  All 32 lanes run
// it with warp-uniform state; returns false when abandoned on stop.
template <typename M, typename WS>
__device__ inline bool warp_solve_task(const SearchParams& P, WS& ws, const WTaskHdr th,
                                       WStats& st) {
  constexpr int K = WS::kW;
  constexpr int R = WT<M>::R;
  const int lane = threadIdx.x & 31;
  const int n = th.n & 0xffff;
  WLane<M> q;
  if constexpr (R == 8) {
    q.adj = ws.adj;
    q.n = n;
#pragma unroll
    for (int j = 0; j < R; ++j) q.v[j] = lane + 32 * j;
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) {
      q.v[j] = lane + 32 * j;
      q.a[j] = q.v[j] < n ? wload<M>(&ws.adj[K * q.v[j]]) : M{};
    }
  }
  bool skip_count = (th.n >> 16) & 1;

  int sb = 0;
  if (lane == 0) sb = ld_relaxed(&P.reg.key[th.scope]) >> 1;
  sb = __shfl_sync(0xffffffffu, sb, 0);
  ws.fr[0].best = sb - th.S;
  ws.fr[0].ach = 0;
  ws.fr[0].base = 0;
  ws.fr[0].pend_b = ws.fr[0].pend_e = 0;
  int nf = 1, sp = 0;
  M L = wload<M>(ws.live0);
  int S = 0;
  bool have = ws.fr[0].best > 0;
  unsigned tick = 0;

  while (true) {
    if (!have) {
      const int f = nf - 1;
      if (sp > ws.fr[f].base) {
        --sp;
        L = wload<M>(&ws.stL[K * sp]);
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
          const M c = wload<M>(&ws.pend[K * --F.pend_e]);
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
        if (warp_export(P, ws, th, n, &ws.stL[K * b], ws.stS[b])) {
          ws.fr[0].base = b + 1;
          TTRACE(++st.t_exp);
        }
      }
    }
    if (skip_count) skip_count = false;
    else ++st.nodes;
    WFrame& F = ws.fr[f];
    int d[R];
    WPROF(long long c0 = clock64());
    const int E = w_fixpoint(ws, q, L, S, F.best, d, st);
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
        bool p[R];
#pragma unroll
        for (int j = 0; j < R; ++j) p[j] = wown(comp, j, q.v[0]) && d[j] != size - 1;
        bool cyc = false;
        if (!nz(wballot<M>(p))) {
          special += size - 1;  // clique: all but one vertex
          st.rules[4] += 1;
        } else {
#pragma unroll
          for (int j = 0; j < R; ++j) p[j] = wown(comp, j, q.v[0]) && d[j] != 2;
          cyc = size >= 3 && !nz(wballot<M>(p));
          if (cyc) {
            special += (size + 1) / 2;  // chordless cycle
            st.rules[5] += 1;
          } else {
            if (pbase + ng < kWPend) wstore<K>(&ws.pend[K * (pbase + ng)], comp);
            else overflow = true;
            ++ng;
          }
        }
        rest &= ~comp;
        if (!nz(rest)) break;
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
        L = wload<M>(&ws.pend[K * pbase]);
        S = base_S;
        have = true;
        continue;
      }
      if constexpr (K > 1) {  // wide-task variants only
        if (f == 0 && n > 64 && !overflow && P.warp_split_export) {
          TTRACE(const long long tw0 = clock64());
          const bool ok =
              warp_registry_split<M, WS>(P, ws, th, pbase, ng, th.S + S, special, th.S + F.best,
                                       st);
          TTRACE(st.t_wait += (unsigned long long)(clock64() - tw0); if (ok) ++st.t_rsplit;
                 else ++st.t_rfail);
          if (ok) continue;  // the components run as tasks of their own
        }
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
      const M first = wload<M>(&ws.pend[K * pbase]);
      for (int i = 1, j = ng - 1; i < j; ++i, --j) {
        for (int w = 0; w < K; ++w) {
          const unsigned long long t = ws.pend[K * (pbase + i) + w];
          ws.pend[K * (pbase + i) + w] = ws.pend[K * (pbase + j) + w];
          ws.pend[K * (pbase + j) + w] = t;
        }
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
    unsigned kmax = 0u;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const unsigned kj = d[j] > 0 ? ((unsigned)d[j] << 8) | (255u - (unsigned)q.v[j]) : 0u;
      kmax = kj > kmax ? kj : kmax;
    }
    const unsigned key = __reduce_max_sync(0xffffffffu, kmax);
    const int v = 255 - (int)(key & 255u);
    const M nv = wload<M>(&ws.adj[K * v]) & L;
    // engine.py:319: exclude child (v out, N(v) in) to the stack, include
    // child (v in) continues here
    const int Sx = S + wpopc(nv);
    if (Sx < F.best) {
      if (sp >= WS::kStack) {
        if (lane == 0) {
          atomicExch(&P.ctl->error, 8);
          atomicExch(&P.ctl->stop, 1);
        }
        return false;
      }
      wstore<K>(&ws.stL[K * sp], L & ~(nv | wbit<M>(v)));
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
// no warp of its block is still busy and either the ring is empty (new tasks
// can only come from busy blocks) or node-level work is queued (the block is
// needed there), or on stop.  Returns whether the block ran a task.
template <int WW>
__device__ inline bool warp_epoch(const SearchParams& P, void* wws_raw, int* busy, WStats& st) {
  using WS = WarpWsT<WW>;
  constexpr bool kSticky = VCG_EPOCH_STICKY && WW > 1;
  const int lane = threadIdx.x & 31;
  WS& ws = ((WS*)wws_raw)[threadIdx.x >> 5];
  bool any = false;
  unsigned backoff = VCG_WBACKOFF_MIN;
  unsigned polls = 0;
  while (true) {
    long long pos = -1;
    int stop = 0, node_work = 0;
    if (lane == 0) {
      // the exchange words are polled here too: a block can stay in the
      // warp tier for the whole search
      if ((P.xch || P.gpeer) && (polls++ & 7) == 0) xch_poll(P);
      stop = ld_relaxed(&P.ctl->stop);
      node_work = (long long)ld_relaxed_u64(P.q.count) > 0;
      // node-level work needs every warp of the block: while a sibling is
      // still inside a wide task (long: up to thousands of nodes) the block
      // cannot take it, so an idle warp keeps taking tasks instead of
      // waiting at the block barrier for that sibling (G(180, 0.08): 386 ->
      // 531 M nodes/s).  With 64-vertex tasks the sibling is done soon and
      // the block is better off returning to the node queue.
      if (!stop && (!node_work || (kSticky && *(volatile int*)busy > 0))) {
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
      if (b == 0 || (node_work && !kSticky)) break;
      if (lane == 0) __nanosleep(backoff);
      backoff = backoff < VCG_WBACKOFF_MAX ? backoff * 2 : VCG_WBACKOFF_MAX;
      __syncwarp();
      continue;
    }
    backoff = VCG_WBACKOFF_MIN;
    any = true;
    const char* slot = P.bq.data + (pos % P.bq.cap) * P.bq_slot;
    const int4 h = __ldcg((const int4*)slot);
    const ulonglong2 lv = __ldcg((const ulonglong2*)(slot + 16));
    const WTaskHdr th{h.x, h.y, h.z, h.w};
    const int n = th.n & 0xffff;
    const int W = wrows(n);
    const unsigned long long* src = (const unsigned long long*)(slot + kWHdrBytes);
    if (lane == 0) {
      ws.live0[0] = lv.x;
      if (WW > 1) ws.live0[1] = W > 1 ? lv.y : 0ull;
      if (WW > 2) {
        const ulonglong2 t = W > 2 ? __ldcg((const ulonglong2*)(src + n * W)) : ulonglong2{0ull, 0ull};
        ws.live0[2] = t.x;
        ws.live0[3] = t.y;
      }
    }
    if (W == WW) {
      for (int i = lane; i < WW * n; i += 32) ws.adj[i] = __ldcg(src + i);
    } else {  // a narrower task in a wider layout: zero-extend its rows
      for (int i = lane; i < WW * n; i += 32) {
        const int r = i / WW, w = i % WW;
        ws.adj[i] = w < W ? __ldcg(src + r * W + w) : 0ull;
      }
    }
    __syncwarp();
    if (lane == 0) q_release_pop(P.bq, pos);
    const long long t0 = clock64();
    const unsigned long long nodes0 = st.nodes;
    if (lane == 0) atomicMin(&P.ctl->t_task_first, globaltimer());
    if (n <= 32) warp_solve_task<unsigned>(P, ws, th, st);
    else if (n <= 64 || WW == 1) warp_solve_task<unsigned long long>(P, ws, th, st);
    else if (n <= 128 || WW == 2) warp_solve_task<W128>(P, ws, th, st);
    else warp_solve_task<W256>(P, ws, th, st);
    __syncwarp();
    if (lane == 0) {
      reg_finish(P, th.scope);  // the task's live unit on its scope
      atomicSub(busy, 1);
    }
    const unsigned long long dt = (unsigned long long)(clock64() - t0);
    TTRACE(if (lane == 0 && dt > 400000ull)
             printf("task n=%d depth=%d nodes=%llu cycles=%llu exports=%llu rsplits=%llu "
                    "rfail=%llu split_cycles=%llu f0best=%d ph=%llu/%llu/%llu/%llu/%llu emits=%llu emitted_v=%llu pub=%llu\n", n,
                    th.depth, st.nodes - nodes0, dt, st.t_exp, st.t_rsplit, st.t_rfail, st.t_wait,
                    ws.fr[0].best, st.t_ph[0], st.t_ph[1], st.t_ph[2], st.t_ph[3], st.t_ph[4], st.t_ph[5],
                    st.t_ph[6], st.t_ph[7]);
           st.t_exp = st.t_rsplit = st.t_wait = st.t_rfail = 0;
           for (int i = 0; i < 8; ++i) st.t_ph[i] = 0);
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
  if (!st.tasks && !st.nodes) return;  // a warp that never ran a task
  Ctl* c = P.ctl;
  add_nz(&c->nodes, st.nodes);
  add_nz(&c->comp_branches, st.splits);
  for (int i = 0; i < 6; ++i) add_nz(&c->rules[i], st.rules[i]);
  add_nz(&c->wtasks, st.tasks);
  add_nz(&c->wnodes, st.nodes);
  add_nz(&c->wcyc, st.cyc);
  add_nz(&c->wc_fix, st.c_fix);
  add_nz(&c->wc_comp, st.c_comp);
  add_nz(&c->wc_split, st.c_split);
  add_nz(&c->wc_iter, st.c_iter);
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
    const int scope = __ldcg((const int*)(P.bq.data + (pos % P.bq.cap) * P.bq_slot) + 1);
    q_release_pop(P.bq, pos);
    reg_finish(P, scope);
  }
}

}  // namespace vcg
