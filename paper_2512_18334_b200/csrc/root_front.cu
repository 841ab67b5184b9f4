// Frontier-driven grid-wide root fixpoint for the solve path
// (preprocess.py:77 root_reduce -> reductions.py:110 reduce_to_fixpoint ->
// kernels/pure.py:188 reduce_fixpoint), any-order variant: the same sweeps,
// the same forced SET and rule counts as the reference, forced ids returned
// in index order (VCG_ROOT_ANY_ORDER).
//
// Why a frontier.  Every sweep of the reference snapshots its candidates with
// a scan of the whole live window.  On the 1M-vertex / 100k-vertex configs
// that is 12 / 66 sweeps of a full scan each (root_grid.cu), although after
// the first sweep only vertices whose degree changed can be candidates:
//  * degree-one (pure.py:82): every candidate of a sweep ends it with degree 0
//    (it applies and its neighbour is removed, or an earlier candidate removed
//    that neighbour), so the candidates of sweep s+1 are exactly the vertices
//    whose degree fell 2 -> 1 since the snapshot of sweep s;
//  * triangle (pure.py:113): validity (two live neighbours, adjacent in the
//    static CSR) only changes with the vertex's degree, and a valid candidate
//    that does not apply meets an applied triangle, i.e. loses degree; so the
//    candidates that can be valid are the vertices whose degree fell 3 -> 2
//    since the previous triangle snapshot.
// Removals push those transitions (the atomicSub's old value) onto
// double-buffered frontier lists, so a sweep costs its frontier plus the
// adjacency of what it removes, not n.  The high-degree sweep (pure.py:158)
// depends on the budget, not on degree changes: it stays a full pass (one
// per fixpoint cycle), which also yields the exact maximum live degree for
// the speculative-budget record.
//
// Latency, not bandwidth, bounds a sweep (a few thousand frontier entries on
// the 100k-vertex config), so every step is shaped for short dependent
// chains spread over the whole grid:
//  * every vertex with a long adjacency (> kTrack) keeps the sum and the sum
//    of squares of its live neighbours' ids: a degree-1 vertex's neighbour
//    is the sum, a degree-2 vertex's two neighbours solve a + b = S1,
//    a^2 + b^2 = S2 -- one load instead of a walk over a mostly dead
//    adjacency; short adjacencies are read whole (all loads in flight);
//  * removals are split into chunks of kChunk adjacency entries, one thread
//    per chunk, loads of a chunk issued before its atomics;
//  * a grid barrier that polls with volatile loads and __nanosleep (the
//    cooperative-groups barrier invalidates L1 on every poll).
//
// Exact parallel sweep semantics (node_ops.cuh): degree-one candidate v with
// target u(v) applies iff v is the lowest-index candidate targeting u(v) and
// not the higher end of an isolated candidate edge; triangles apply as the
// lexicographically-first maximal independent set of the valid candidates'
// intersection graph, resolved in claim rounds.  Claims are 64-bit
// (tag << 32 | INT_MAX - v) atomicMax keys with a fresh tag per round, so no
// reset pass is needed; removal-set membership is a per-vertex sweep tag.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdio>
#include <cstdlib>

#include "root_grid.cuh"
#include "search.cuh"

namespace vcg {

namespace {

// -DVCG_FRONT_PROF: sub-phase timers of the degree-one sweep (diagnostic
// builds; they add block barriers)
#ifdef VCG_FRONT_PROF
#define FPROF(...) __VA_ARGS__
#else
#define FPROF(...)
#endif

constexpr int kSolo = 0;     // default: frontier size below which block 0 sweeps alone
#ifndef VCG_FRONT_CHUNK
#define VCG_FRONT_CHUNK 4  // 4 vs 8 vs 16 vs 2: ba100k 0.85 / 0.90 / 0.97 / 0.99 ms
#endif
constexpr int kChunk = VCG_FRONT_CHUNK;  // adjacency entries per removal work item
#ifndef VCG_FRONT_TRACK
#define VCG_FRONT_TRACK 8  // 8 vs 12 vs 20: planted1m 0.274 / 0.283 / 0.279 ms
#endif
constexpr int kTrack = VCG_FRONT_TRACK;  // adjacencies longer than this keep live-neighbour id sums

enum Phase { F_D1 = 0, F_TRI = 1, F_HD = 2, F_DONE = 3 };
constexpr int kLog = 96;

struct St {  // fixpoint state, replicated in every thread (uniform transitions)
  int phase, p1, p2, s, tg;
  int cycle, d1, d2t, hd, forced, spec_m;
  int sweeps, passes, solo;
};

struct FrontCtl {
  int cnt1[2], cnt2[2];                       // frontier list lengths (index = buffer)
  int nrem[3], ncand[3], ch[3], dmax[3], nchunk[3];  // per step, by step id mod 3
  int ropen[3];                               // triangle claim rounds, by claim tag mod 3
  int err, hd_applied, wlo, whi;  // wlo = max(INT_MAX - lowest live), whi = max(highest live + 1)
  unsigned long long edges, walked, items;
  unsigned bar, nbar;                         // grid_barrier word, barriers passed
  unsigned long long tph[24];                 // phase times (ns, thread 0): A, B, C, barriers, sub-phases
  St st;                                      // block 0 -> grid after a solo segment
  int nlog;                                   // per-sweep log (trace builds read it)
  long long slog[kLog][5];                    // phase, end ns, frontier, removed, chunks
  int partial[kRootGridMaxBlocks];
};

struct Front {  // device arrays (root_front_bytes)
  int n;
  uint32_t* deg;
  unsigned long long* key;          // claims
  unsigned long long *nsum, *nsq;   // live-neighbour id sums
  int *ia, *ib, *st, *rs;           // targets, triangle state, removal tag
  int *l1[2], *l2[2];               // frontier lists (pending / snapshot)
  int *rem, *cand;
  int4* chunk;                      // removal work items (vertex, first entry, end, -)
  uint8_t* forced;
  uint8_t* trk;                     // adjacency longer than kTrack: sums maintained
};

// Per-block copy of FrontCtl's control header (list lengths, step slots,
// claim-round flags, err): refreshed by warp 0 inside every barrier, one word
// per lane.  Every thread used to read these words from L2 after each barrier:
// 2368 warps' loads of one address queue at one L2 slice (ncu: the loop
// bounds after a barrier were the top long-scoreboard lines).
constexpr int kHdr = 32;
__device__ __forceinline__ int* hdr_cache() {
  __shared__ int c[kHdr];
  return c;
}
__device__ __forceinline__ void hdr_refresh(const int* G) {  // warp 0, after the acquire
  if (threadIdx.x < kHdr) hdr_cache()[threadIdx.x] = __ldcg(G + threadIdx.x);
}

// Grid barrier.  cooperative_groups' grid.sync() polls with acquire loads,
// each followed by an L1 invalidate (CCTL.IVALL; ncu: 8.5 M in one launch).
// This one polls with volatile loads and __nanosleep and acquires once, after
// the flip (an acquire fence instead measured slower).  Arrival flips bit 31 of the word (block 0 adds 2^31 - (blocks -
// 1), the others 1), so it needs no reset.  Warp 0 then refreshes the
// block's header copy.
__device__ __forceinline__ void grid_barrier(unsigned* bar, const int* hdr) {
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
      __threadfence();
      const unsigned old = atomicAdd(bar, inc);
      if (blockIdx.x == 0) bar[1] += 1;  // barriers passed (FrontCtl::nbar)
      unsigned ns = 32;
      while (((old ^ *(volatile unsigned*)bar) & 0x80000000u) == 0) {
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      (void)v;
    }
    __syncwarp();
    hdr_refresh(hdr);
  }
  __syncthreads();
}

struct Ex {  // executor: the whole grid, or block 0 alone
  int rank, size;
  bool grid;
  unsigned* bar;
  const int* hdr;
  __device__ void sync() const {
    if (grid) {
      grid_barrier(bar, hdr);
    } else {
      __syncthreads();
      hdr_refresh(hdr);
      __syncthreads();
    }
  }
};

__device__ __forceinline__ int vld(const int* p) { return *(const volatile int*)p; }
// a header word as of the block's last barrier (stable from that barrier to
// the next one: written only by atomics of the phase that ends there)
__device__ __forceinline__ int cld(const void* G, const int* p) {
  return hdr_cache()[p - (const int*)G];
}
// Degree words.  Bit 30 flags a tracked vertex (adjacency > kTrack), so a
// removal's decrement returns the flag with the old degree (one L2 request
// per adjacency entry); the low 30 bits hold the live degree, or, once the
// vertex is dead, kDead -- decremented speculatively by later removals
// (rm_chunk) but never below kDeadMin, so "dead" is low bits >= kDeadMin.
// sweep_hd decodes the array for the block-level high-degree pass (and
// re-encodes it after); the final pass leaves plain degrees for the host
// and the next launch.
constexpr uint32_t kTrkBit = 1u << 30, kLowMask = kTrkBit - 1u;
constexpr uint32_t kDead = 1u << 29, kDeadMin = 1u << 28;
__device__ __forceinline__ int dval(uint32_t w) {
  const uint32_t x = w & kLowMask;
  return x >= kDeadMin ? 0 : (int)x;
}
__device__ __forceinline__ uint32_t denc(int d, bool trk) {
  return (trk ? kTrkBit : 0u) | (d > 0 ? (uint32_t)d : kDead);
}
__device__ __forceinline__ int dget(const uint32_t* d, int v) { return dval(__ldcg(d + v)); }

__device__ __forceinline__ unsigned long long claim_key(int tg, int v) {
  return ((unsigned long long)(unsigned)tg << 32) | (unsigned long long)(unsigned)(kInf - v);
}

// Appends to the global lists go through two block-local staging queues in
// shared memory: one global atomic per block and phase instead of one per
// entry (the list counters are the kernel's only hot words).
// The staging queues live in dynamic shared memory (the kernel runs one
// 512-thread block per SM, so there is room): 8192 appends per list and 4096
// removal chunks per block.  With the 48 KB static limit (2048 / 1024) the
// two heavy planted1m sweeps (600 k transitions, 230 k chunks) overflowed
// into per-entry global appends: 93 / 80 us -> 52 / 56 us, root kernel 0.39 ->
// 0.32 ms.  Larger queues measured slower (12288 / 6144: 0.43 ms, the L1
// carve-out shrinks), fewer staged chunks too (8192 / 2048: 0.43 ms).
#ifndef VCG_FRONT_THREADS  // block size of the frontier kernel (one block per SM)
#define VCG_FRONT_THREADS kRootGridThreads
#endif
#ifndef VCG_FRONT_DYNQ
#define VCG_FRONT_DYNQ 1
#endif
#ifndef VCG_FRONT_KQ
#define VCG_FRONT_KQ 8192
#endif
#ifndef VCG_FRONT_KQC
#define VCG_FRONT_KQC 4096
#endif
constexpr int kQ = VCG_FRONT_KQ;
constexpr int kQC = VCG_FRONT_KQC;  // staged removal chunks (16 B each)
struct BlockQ {
  int cnt[2], base[2];
  int buf[2][kQ];
  int ccnt, cbase, cused;  // removal chunks: reserved, published base, staged
  int4 cbuf[kQC];
};

__device__ __forceinline__ void qpush(BlockQ* q, int which, int* list, int* gcnt, int v) {
  const int pos = atomicAdd(&q->cnt[which], 1);
  if (pos < kQ) q->buf[which][pos] = v;
  else list[atomicAdd(gcnt, 1)] = v;  // staging full: append directly
}

// every thread of the block calls; publishes both staging queues
__device__ __forceinline__ void qflush(BlockQ* q, int* list0, int* cnt0, int* list1, int* cnt1) {
  __syncthreads();
  const int c0 = min(q->cnt[0], kQ), c1 = min(q->cnt[1], kQ);
  if (c0 == 0 && c1 == 0) return;  // nothing staged (block-uniform): no more barriers
  if (threadIdx.x == 0) {
    q->base[0] = c0 ? atomicAdd(cnt0, c0) : 0;
    q->base[1] = c1 ? atomicAdd(cnt1, c1) : 0;
  }
  __syncthreads();
  const int b0 = q->base[0], b1 = q->base[1];
  for (int i = threadIdx.x; i < c0; i += blockDim.x) list0[b0 + i] = q->buf[0][i];
  for (int i = threadIdx.x; i < c1; i += blockDim.x) list1[b1 + i] = q->buf[1][i];
  __syncthreads();
  if (threadIdx.x == 0) q->cnt[0] = q->cnt[1] = 0;
}

// the two live neighbours a < b of a degree-2 vertex from its sums
__device__ __forceinline__ void two_from_sums(const Front& F, int v, int* a, int* b) {
  const unsigned long long s1 = __ldcg(F.nsum + v), s2 = __ldcg(F.nsq + v);
  const unsigned long long d2 = 2ull * s2 - s1 * s1;  // (b - a)^2
  unsigned long long d = (unsigned long long)sqrt((double)d2);
  while (d * d > d2) --d;
  while ((d + 1) * (d + 1) <= d2) ++d;
  *a = (int)((s1 - d) >> 1);
  *b = (int)((s1 + d) >> 1);
}

// u joins the removal set of step s: the rem list, and its adjacency as
// kChunk-entry work items
__device__ __forceinline__ void add_removed_at(const Front& F, FrontCtl* G, BlockQ* q, int s,
                                               int u, int b, int e, long long* walked) {
  F.rs[u] = s;
  qpush(q, 0, F.rem, &G->nrem[s % 3], u);
  *walked += e - b;
  const int nc = (e - b + kChunk - 1) / kChunk;
  if (nc > 0) {
    const int pos = atomicAdd(&q->ccnt, nc);
    if (pos + nc <= kQC) {
      for (int c = 0; c < nc; ++c)
        q->cbuf[pos + c] = make_int4(u, b + c * kChunk, min(e, b + (c + 1) * kChunk), 0);
      atomicMax(&q->cused, pos + nc);
    } else {  // staging full: append directly
      const int at = atomicAdd(&G->nchunk[s % 3], nc);
      for (int c = 0; c < nc; ++c)
        F.chunk[at + c] = make_int4(u, b + c * kChunk, min(e, b + (c + 1) * kChunk), 0);
    }
  }
}

__device__ __forceinline__ void add_removed(const Front& F, FrontCtl* G, BlockQ* q,
                                            const int* off, int s, int u, long long* walked) {
  add_removed_at(F, G, q, s, u, off[u], off[u + 1], walked);
}

// every thread of the block calls: publishes the removal list (staging queue
// 0) and the staged removal chunks with their two reservations in one round
// trip (qflush + cflush back to back cost two)
__device__ __forceinline__ void rflush(BlockQ* q, int* rem, int* nrem, int4* chunks, int* nch) {
  __syncthreads();
  const int c0 = min(q->cnt[0], kQ), c = q->cused;
  if (c0 == 0 && c == 0) {  // nothing staged (block-uniform): no more barriers
    if (q->ccnt) {  // chunk reservations that overflowed: reset after every thread read
      __syncthreads();
      if (threadIdx.x == 0) q->ccnt = 0;
    }
    return;
  }
  if (threadIdx.x == 0) {
    q->base[0] = c0 ? atomicAdd(nrem, c0) : 0;
    q->cbase = c ? atomicAdd(nch, c) : 0;
  }
  __syncthreads();
  const int b0 = q->base[0], b = q->cbase;
  for (int i = threadIdx.x; i < c0; i += blockDim.x) rem[b0 + i] = q->buf[0][i];
  for (int i = threadIdx.x; i < c; i += blockDim.x) chunks[b + i] = q->cbuf[i];
  __syncthreads();
  if (threadIdx.x == 0) q->cnt[0] = q->ccnt = q->cused = 0;
}

// every thread of the block calls: publishes the staged removal chunks
__device__ __forceinline__ void cflush(BlockQ* q, int4* list, int* cnt) {
  __syncthreads();
  const int c = q->cused;
  if (threadIdx.x == 0) q->cbase = c ? atomicAdd(cnt, c) : 0;
  __syncthreads();
  const int b = q->cbase;
  for (int i = threadIdx.x; i < c; i += blockDim.x) list[b + i] = q->cbuf[i];
  __syncthreads();
  if (threadIdx.x == 0) q->ccnt = q->cused = 0;
}

// the first two live neighbours of an untracked vertex (adjacency <= kTrack)
// whose slice [s0, s0 + len) is known: its entries and their degrees loaded
// at once, two dependent round trips
__device__ __forceinline__ void live_short_at(const Front& F, const int* nbr, int s0, int len,
                                              int* a, int* b) {
  int x[kTrack], d[kTrack];
#pragma unroll
  for (int j = 0; j < kTrack; ++j) x[j] = j < len ? __ldg(nbr + s0 + j) : -1;
#pragma unroll
  for (int j = 0; j < kTrack; ++j) d[j] = x[j] >= 0 ? dget(F.deg, x[j]) : 0;
  int u = -1, w = -1;
#pragma unroll
  for (int j = 0; j < kTrack; ++j)
    if (d[j] > 0) {
      if (u < 0) u = x[j];
      else if (w < 0) w = x[j];
    }
  *a = u;
  *b = w;
}

__device__ __forceinline__ void live_short(const Front& F, const int* off, const int* nbr, int v,
                                           int* a, int* b) {
  const int s0 = off[v];
  live_short_at(F, nbr, s0, off[v + 1] - s0, a, b);
}

// one removal work item: the entries [b, min(b + kChunk, end(u))) of removed
// vertex u.  Live neighbours lose a degree and (tracked ones) u from their
// sums; 2 -> 1 and 3 -> 2 transitions are pushed to the pending lists.  The
// decrement is issued without a prior degree read: a dead neighbour's word
// goes negative (harmless, readers clamp) and the atomic's old value says
// whether the neighbour was live.  A neighbour in the same removal set is
// decremented and pushed like a live one -- its word is zeroed by
// remove_set either way and the next sweep drops it by its degree -- so no
// removal-tag load: two L2 requests per entry instead of three (the heavy
// sweeps are L2-request bound).  The solve path does not count removed
// edges (the reduced graph's size comes from the compaction).
__device__ __forceinline__ void rm_chunk(const Front& F, FrontCtl* G, BlockQ* q,
                                         const int* nbr, int s, int p1, int p2, int u, int b,
                                         int e, long long* edges) {
  (void)s;
  (void)edges;
  const int len = e - b;
  int x[kChunk];
  unsigned old[kChunk];
  uint8_t tr[kChunk];
#pragma unroll
  for (int j = 0; j < kChunk; ++j) x[j] = j < len ? __ldg(nbr + b + j) : -1;
#pragma unroll
  for (int j = 0; j < kChunk; ++j) old[j] = x[j] >= 0 ? atomicSub(F.deg + x[j], 1u) : 0u;
  const unsigned long long uu = (unsigned long long)u;
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    tr[j] = (old[j] & kTrkBit) != 0;
    old[j] = (unsigned)dval(old[j]);  // the neighbour's degree before (0: dead)
    if (tr[j] && old[j] > 0u) {  // tracked live neighbour: u leaves its sums
      atomicAdd(F.nsum + x[j], 0ull - uu);
      atomicAdd(F.nsq + x[j], 0ull - uu * uu);
    }
  }
#pragma unroll
  for (int j = 0; j < kChunk; ++j) {
    if (old[j] == 2u) qpush(q, 0, F.l1[p1], &G->cnt1[p1], x[j]);
    else if (old[j] == 3u) qpush(q, 1, F.l2[p2], &G->cnt2[p2], x[j]);
  }
}

struct Timer {  // thread 0's phase clock
  unsigned long long t;
  bool on;
  __device__ explicit Timer(bool o) : t(o ? globaltimer() : 0), on(o) {}
  __device__ void lap(FrontCtl* G, int i) {
    if (on) {
      const unsigned long long now = globaltimer();
      G->tph[i] += now - t;
      t = now;
    }
  }
};

// phase C of a sweep: remove every member of the step's set (rem / chunks);
// transitions go to the pending lists l1[p1] / l2[p2]
__device__ __forceinline__ void remove_set(const Ex& E, const Front& F, FrontCtl* G, BlockQ* q,
                                           const int* off, const int* nbr, int s, int p1, int p2,
                                           long long* edges, long long* walked) {
  FPROF(Timer tm(E.rank == 0));
  const int nrem = cld(G, &G->nrem[s % 3]), nch = cld(G, &G->nchunk[s % 3]);
  FPROF(tm.lap(G, 6));
  for (int k = E.rank; k < nrem; k += E.size) {  // independent of the chunks: issued first
    const int u = F.rem[k];
    F.deg[u] = kDead;
    F.forced[u] = 1;
  }
  for (int c = E.rank; c < nch; c += E.size) {
    const int4 ch = __ldcg(F.chunk + c);
    rm_chunk(F, G, q, nbr, s, p1, p2, ch.x, ch.y, ch.z, edges);
  }
  FPROF(tm.lap(G, 7); __syncthreads(); tm.lap(G, 8));
  qflush(q, F.l1[p1], &G->cnt1[p1], F.l2[p2], &G->cnt2[p2]);
  FPROF(tm.lap(G, 9));
}

// live-neighbour sums of every tracked live vertex.  Each lane reads its own
// vertex's flag, degree and adjacency bounds in one round trip; tracked ones
// with up to 64 entries are then summed by 8-lane groups, four vertices per
// warp at a time (longer ones by the whole warp, one after another),
// each lane loading every 8th entry (all loads of a round in flight) and the
// group reducing with shuffles.  (A whole warp per tracked vertex, one vertex
// after another, cost two dependent round trips per vertex: 36 of the 57 us
// init on planted1m.)
__device__ __forceinline__ void init_sums(const Front& F, const int* off, const int* nbr, int n,
                                          bool all_live) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  for (int base = gt - lane; base < n; base += T) {
    const int v = base + lane;
    int b = 0, e = 0;
    bool tracked = false;
    if (v < n) {
      const uint8_t tr = F.trk[v];
      const int d = dget(F.deg, v);
      b = __ldg(off + v);
      e = __ldg(off + v + 1);
      tracked = tr && d > 0;
    }
    const bool hub = tracked && e - b > 64;  // whole-warp path below
    unsigned m = __ballot_sync(0xffffffffu, tracked && !hub);
    while (m) {
      // group grp takes the (grp + 1)-th remaining tracked vertex
      const unsigned src = __fns(m, 0, grp + 1);
      const bool act = src < 32u;
      const int sl = act ? (int)src : 0;
      const int vb = __shfl_sync(0xffffffffu, b, sl), ve = __shfl_sync(0xffffffffu, e, sl);
      unsigned long long s1 = 0, s2 = 0;
      if (act) {
        int i = vb + sub;
#pragma unroll 4
        for (; i < ve; i += 8) {
          const int x = __ldg(nbr + i);
          if (all_live || dget(F.deg, x) > 0) {
            s1 += (unsigned long long)x;
            s2 += (unsigned long long)x * (unsigned long long)x;
          }
        }
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (act && sub == 0) {
        F.nsum[base + sl] = s1;
        F.nsq[base + sl] = s2;
      }
      // drop the (up to) four vertices taken this round
#pragma unroll
      for (int g = 0; g < 4; ++g) m &= m - 1;
    }
    unsigned h = __ballot_sync(0xffffffffu, hub);  // long adjacencies: a warp each
    while (h) {
      const int src = __ffs(h) - 1;
      h &= h - 1;
      const int vb = __shfl_sync(0xffffffffu, b, src), ve = __shfl_sync(0xffffffffu, e, src);
      unsigned long long s1 = 0, s2 = 0;
#pragma unroll 4
      for (int i = vb + lane; i < ve; i += 32) {
        const int x = __ldg(nbr + i);
        if (all_live || dget(F.deg, x) > 0) {
          s1 += (unsigned long long)x;
          s2 += (unsigned long long)x * (unsigned long long)x;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == 0) {
        F.nsum[base + src] = s1;
        F.nsq[base + src] = s2;
      }
    }
  }
}

// step prologue (rank 0): clear the next step's slots
__device__ __forceinline__ void next_slots(FrontCtl* G, int s) {
  const int z = (s + 1) % 3;
  G->nrem[z] = G->ncand[z] = G->ch[z] = G->dmax[z] = G->nchunk[z] = 0;
}


// thread 0 of the grid appends one record per sweep (after its last barrier)
__device__ __forceinline__ void slog(FrontCtl* G, int rank, int ph, int ncur, int s) {
  if (rank != 0 || G->nlog >= kLog) return;
  long long* r = G->slog[G->nlog++];
  r[0] = ph;
  r[1] = (long long)globaltimer();
  r[2] = ncur;
  r[3] = vld(&G->nrem[s % 3]);
  r[4] = vld(&G->nchunk[s % 3]);
}

// One degree-one sweep (pure.py:82) over the pending list l1[p1].
__device__ __forceinline__ void sweep_d1(const Ex& E, const Front& F, FrontCtl* G, BlockQ* q,
                                         const int* off, const int* nbr, St& S, long long* edges,
                                         long long* walked) {
  const int s = S.s, t = S.tg;
  const int cur = S.p1, nxt = S.p1 ^ 1;
  const int ncur = cld(G, &G->cnt1[cur]);
  if (ncur == 0) {  // nothing to sweep: no barriers, no step slot used
    S.sweeps += 1;
    S.phase = F_TRI;
    return;
  }
  Timer tm(E.rank == 0);
  int* L = F.l1[cur];
  if (E.rank == 0) {
    G->cnt1[nxt] = 0;
    next_slots(G, s);
    G->items += (unsigned long long)ncur;
  }
  FPROF(tm.lap(G, 13));
  // AB: targets and decisions in one phase.  A degree-1 candidate v with
  // live neighbour u removes u unless v is the higher end of an isolated
  // candidate edge (u has degree 1 too: its only live neighbour is v, so u
  // removes v); of the candidates targeting one u the first to tag it adds
  // it to the removal set.  Degrees do not change before phase C, so this
  // is the reference's in-order sweep (the candidate that wins a shared
  // target only changes which thread enqueues it), with one grid barrier
  // less than a claim round.  Everything a candidate needs is loaded in one
  // round trip (degree, tracked flag, id sum, adjacency bounds).
  for (int k = E.rank; k < ncur; k += E.size) {
    const int v = L[k];
    const uint32_t wv = __ldcg(F.deg + v);  // degree and tracked flag, one request
    const int d = dval(wv);
    const bool tr = (wv & kTrkBit) != 0;
    const int o0 = __ldg(off + v), o1 = __ldg(off + v + 1);
    if (d != 1) continue;
    int u, u2;
    if (tr) u = (int)__ldcg(F.nsum + v);  // tracked candidates only (L2 requests)
    else live_short_at(F, nbr, o0, o1 - o0, &u, &u2);
    if (u < 0 || u >= F.n) {  // inconsistent degree array: report, never loop
      atomicExch(&G->err, 1);
      continue;
    }
    const int du = dget(F.deg, u);
    const int ob = __ldg(off + u), oe = __ldg(off + u + 1);
    if (du <= 0) {
      atomicExch(&G->err, 1);
      continue;
    }
    if (du == 1 && u < v) continue;  // isolated candidate edge: u removes v
    if (atomicMax(F.rs + u, s) < s) add_removed_at(F, G, q, s, u, ob, oe, walked);
  }
  (void)t;
  tm.lap(G, 0);
  FPROF(tm.lap(G, 10); __syncthreads(); tm.lap(G, 11));
  rflush(q, F.rem, &G->nrem[s % 3], F.chunk, &G->nchunk[s % 3]);
  FPROF(tm.lap(G, 12));
  tm.lap(G, 1);
  E.sync();
  tm.lap(G, 4);
  // C: removal
  const int nr = cld(G, &G->nrem[s % 3]);
  remove_set(E, F, G, q, off, nbr, s, nxt, S.p2, edges, walked);
  tm.lap(G, 2);
  E.sync();
  tm.lap(G, 5);
  slog(G, E.rank, 1, ncur, s);
  S.p1 = nxt;
  S.d1 += nr;
  S.forced += nr;
  S.cycle += nr;
  S.sweeps += 1;
  S.s += 1;
  S.tg += 1;
  if (nr == 0) S.phase = F_TRI;
}

// static adjacency test, binary search in the shorter slice
__device__ __forceinline__ bool adjacent(const int* off, const int* nbr, int a, int b) {
  if (off[a + 1] - off[a] > off[b + 1] - off[b]) {
    const int t = a;
    a = b;
    b = t;
  }
  int lo = off[a], hi = off[a + 1] - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int y = __ldg(nbr + mid);
    if (y == b) return true;
    if (y < b) lo = mid + 1;
    else hi = mid - 1;
  }
  return false;
}

// One triangle sweep (pure.py:113) over the pending list l2[p2].
__device__ __forceinline__ void sweep_tri(const Ex& E, const Front& F, FrontCtl* G, BlockQ* q,
                                          const int* off, const int* nbr, St& S,
                                          long long* edges, long long* walked) {
  const int lane = threadIdx.x & 31;
  const int s = S.s;
  const int cur = S.p2, nxt = S.p2 ^ 1;
  const int ncur = cld(G, &G->cnt2[cur]);
  if (ncur == 0) {
    S.sweeps += 1;
    S.phase = F_HD;
    return;
  }
  int* L = F.l2[cur];
  int* ncand = &G->ncand[s % 3];
  if (E.rank == 0) {
    G->cnt2[nxt] = 0;
    G->ropen[S.tg % 3] = 0;
    next_slots(G, s);
    G->items += (unsigned long long)ncur;
  }
  // A: valid candidates (degree 2, live neighbours adjacent)
  for (int k = E.rank; k < ncur; k += E.size) {
    const int v = L[k];
    if (dget(F.deg, v) != 2) continue;
    int a, b;
    if (__ldg(F.trk + v)) two_from_sums(F, v, &a, &b);
    else live_short(F, off, nbr, v, &a, &b);
    if (a < 0 || a >= b || dget(F.deg, a) <= 0 || dget(F.deg, b) <= 0) {
      atomicExch(&G->err, 1);
      continue;
    }
    if (adjacent(off, nbr, a, b)) {
      F.ia[v] = a;
      F.ib[v] = b;
      F.st[v] = 3;  // undecided
      qpush(q, 0, F.cand, ncand, v);
    }
  }
  qflush(q, F.cand, ncand, F.cand, ncand);
  E.sync();
  const int nc = cld(G, ncand);
  int tri = 0;
  if (nc > 0) {
    while (true) {
      const int t = S.tg;
      int* open = &G->ropen[t % 3];
      if (E.rank == 0) G->ropen[(t + 1) % 3] = 0;
      for (int k = E.rank; k < nc; k += E.size) {
        const int v = F.cand[k];
        if (__ldcg(F.st + v) != 3) continue;
        const unsigned long long key = claim_key(t, v);
        atomicMax(F.key + v, key);
        atomicMax(F.key + F.ia[v], key);
        atomicMax(F.key + F.ib[v], key);
      }
      E.sync();
      int still = 0;
      for (int k = E.rank; k < nc; k += E.size) {
        const int v = F.cand[k];
        if (__ldcg(F.st + v) != 3) continue;
        const int u = F.ia[v], x = F.ib[v];
        if (__ldcg(F.rs + v) == s || __ldcg(F.rs + u) == s || __ldcg(F.rs + x) == s) {
          F.st[v] = 4;  // meets an applied triangle's removed vertex: out
        } else {
          const unsigned long long key = claim_key(t, v);
          if (__ldcg(F.key + v) == key && __ldcg(F.key + u) == key && __ldcg(F.key + x) == key) {
            F.st[v] = 5;  // in
            add_removed(F, G, q, off, s, u, walked);
            add_removed(F, G, q, off, s, x, walked);
          } else {
            still = 1;
          }
        }
      }
      if (__any_sync(0xffffffffu, still) && lane == 0) atomicOr(open, 1);
      rflush(q, F.rem, &G->nrem[s % 3], F.chunk, &G->nchunk[s % 3]);
      S.tg += 1;
      E.sync();
      if (!cld(G, open)) break;
    }
    const int nr = cld(G, &G->nrem[s % 3]);
    remove_set(E, F, G, q, off, nbr, s, S.p1, nxt, edges, walked);
    E.sync();
    tri = nr / 2;
  }
  slog(G, E.rank, 2, ncur, s);
  S.p2 = nxt;
  S.d2t += tri;
  S.forced += 2 * tri;
  S.cycle += tri;
  S.sweeps += 1;
  S.s += 1;
  S.phase = F_HD;
}

// The high-degree point of a cycle (pure.py:158): a full pass for the
// candidates and the maximum live degree; block 0 applies an in-order sweep
// when a real budget fires it (then the frontier lists and sums are rebuilt).
__device__ __forceinline__ void sweep_hd(const Front& F, FrontCtl* G, BlockQ* q, const int* off,
                                         const int* nbr, char* wsmem, int n, int budget,
                                         int* hd_out, St& S, BlockScratch* bs) {
  const int s = S.s;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  const int bud = budget - S.forced;
  if (gt == 0) next_slots(G, s);
  int ch = 0, dm = 0;
  for (int v = gt; v < n; v += T) {
    const int d = dget(F.deg, v);
    ch += (d > 0 && d > bud);
    dm = d > dm ? d : dm;
  }
  {
    int vals[2] = {ch, dm};
    const int op[2] = {0, 2};
    block_reduce<2>(vals, op, bs);
    if (threadIdx.x == 0) {
      if (vals[0]) atomicAdd(&G->ch[s % 3], vals[0]);
      if (vals[1]) atomicMax(&G->dmax[s % 3], vals[1]);
    }
  }
  grid_barrier(&G->bar, (const int*)G);
  S.passes += 1;
  const int CH = cld(G, &G->ch[s % 3]), DM = cld(G, &G->dmax[s % 3]);
  if (bud > kSpecBudget / 2) S.spec_m = max(S.spec_m, DM + S.forced);
  int applied = 0;
  if (CH > 0) {
    // the block-level pass reads plain degrees: decode, then re-encode below
    for (int v = gt; v < n; v += T) F.deg[v] = (uint32_t)dget(F.deg, v);
    grid_barrier(&G->bar, (const int*)G);
    if (blockIdx.x == 0) {
      NodeWs<uint32_t> w = carve_ws<uint32_t>(wsmem, n, bs, off, nbr);
      PassRet h = high_degree_pass(w, 0, n - 1, bud, hd_out, 0);
      for (int k = threadIdx.x; k < h.pos; k += blockDim.x) F.forced[hd_out[k]] = 1;
      if (threadIdx.x == 0) {
        G->hd_applied = h.applied;
        G->edges += (unsigned long long)h.edges;
        G->cnt1[S.p1] = 0;  // rebuilt below
        G->cnt2[S.p2] = 0;
      }
    }
    grid_barrier(&G->bar, (const int*)G);
    for (int v = gt; v < n; v += T) F.deg[v] = denc((int)__ldcg(F.deg + v), F.trk[v] != 0);
    grid_barrier(&G->bar, (const int*)G);
    applied = cld(G, &G->hd_applied);
    if (applied > 0) {
      for (int v = gt; v < n; v += T) {
        const int d = dget(F.deg, v);
        if (d == 1) qpush(q, 0, F.l1[S.p1], &G->cnt1[S.p1], v);
        else if (d == 2) qpush(q, 1, F.l2[S.p2], &G->cnt2[S.p2], v);
      }
      qflush(q, F.l1[S.p1], &G->cnt1[S.p1], F.l2[S.p2], &G->cnt2[S.p2]);
      init_sums(F, off, nbr, n, false);  // the block-level sweep did not maintain them
      S.passes += 1;
    }
    // the block-level sweep used ic[0, candidates) as scratch
    if (blockIdx.x == 0) {
      NodeWs<uint32_t> w = carve_ws<uint32_t>(wsmem, n, bs, off, nbr);
      for (int v = threadIdx.x; v < n; v += blockDim.x) w.ic[v] = 0;
    }
    grid_barrier(&G->bar, (const int*)G);
  }
  slog(G, gt, 3, CH, s);
  S.hd += applied;
  S.forced += applied;
  S.cycle += applied;
  S.s += 1;
  if (S.cycle == 0) {
    S.phase = F_DONE;
  } else {
    S.cycle = 0;
    S.phase = F_D1;
  }
}

}  // namespace

// One block per SM; 512 threads, or 1024 on graphs of >= kFrontBigN vertices
// (their heavy sweeps are L2-request bound and want more requests in
// flight: planted1m 0.276 -> 0.262 ms; the long cascades of smaller graphs
// want cheaper barriers: ba100k 0.83 ms at 512, 0.86 at 1024, 0.90 at 768).
constexpr int kFrontBigN = 1 << 19;
template <int TH>
__global__ void __launch_bounds__(TH, 1)
    k_root_front(int n, const int32_t* off, const int32_t* nbr, char* wsmem, char* fmem,
                 int budget, int32_t* out, long long* ret, int init, void* ctl_mem,
                 int solo_max) {
  __shared__ BlockScratch bs;
#if VCG_FRONT_DYNQ
  extern __shared__ __align__(16) unsigned char qmem[];  // the staging queues (dynamic)
  BlockQ& q = *(BlockQ*)qmem;
#else
  __shared__ BlockQ q;
#endif
  const unsigned long long t_start = globaltimer();
  if (threadIdx.x == 0) q.cnt[0] = q.cnt[1] = q.ccnt = q.cused = 0;
  init_block_scratch(&bs);
  FrontCtl* G = (FrontCtl*)ctl_mem;  // zeroed by the host before the launch
  Front F;
  {
    const size_t nn = ((size_t)n + 31) & ~(size_t)31;
    F.n = n;
    F.deg = (uint32_t*)wsmem;
    unsigned long long* lp = (unsigned long long*)fmem;
    F.key = lp;
    F.nsum = lp + nn;
    F.nsq = lp + 2 * nn;
    int* ip = (int*)(lp + 3 * nn);
    F.ia = ip;
    F.ib = ip + nn;
    F.st = ip + 2 * nn;
    F.rs = ip + 3 * nn;
    F.l1[0] = ip + 4 * nn;
    F.l1[1] = ip + 5 * nn;
    F.l2[0] = ip + 6 * nn;
    F.l2[1] = ip + 7 * nn;
    F.rem = ip + 8 * nn;
    F.cand = ip + 9 * nn;
    F.forced = (uint8_t*)(ip + 10 * nn);
    F.trk = F.forced + nn;
    F.chunk = (int4*)(((uintptr_t)(F.trk + nn) + 15) & ~(uintptr_t)15);
  }
  int* hd_out = F.cand;  // the high-degree sweep's ids (cand is free outside triangle sweeps)
  const int gt = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  const bool real_budget = budget <= kSpecBudget / 2;
  // init: degrees, tags, the first frontier (every degree-1 / degree-2 vertex)
  for (int v = gt; v < n; v += T) {
    const int len = off[v + 1] - off[v];
    const int d = init ? len : (int)F.deg[v];
    F.deg[v] = denc(d, len > kTrack);
    F.key[v] = 0ull;
    F.rs[v] = 0;
    F.forced[v] = 0;
    F.trk[v] = len > kTrack;
    if (d == 1) qpush(&q, 0, F.l1[0], &G->cnt1[0], v);
    else if (d == 2) qpush(&q, 1, F.l2[0], &G->cnt2[0], v);
  }
  FPROF(Timer ti(gt == 0); ti.t = gt == 0 ? t_start : 0; ti.lap(G, 16));
  qflush(&q, F.l1[0], &G->cnt1[0], F.l2[0], &G->cnt2[0]);
  FPROF(ti.lap(G, 17));
  if (real_budget) {  // scratch of the block-level high-degree sweep
    NodeWs<uint32_t> w = carve_ws<uint32_t>(wsmem, n, &bs, off, nbr);
    for (int v = gt; v < n; v += T) {
      w.flag[v] = 0;
      w.ic[v] = 0;
    }
  }
  grid_barrier(&G->bar, (const int*)G);  // degrees initialised
  FPROF(ti.lap(G, 18));
  init_sums(F, off, nbr, n, init != 0);
  FPROF(ti.lap(G, 19));
  grid_barrier(&G->bar, (const int*)G);
  FPROF(ti.lap(G, 20));
  if (gt == 0) {
    G->slog[0][0] = 0;
    G->slog[0][1] = (long long)globaltimer();
    G->slog[0][2] = (long long)t_start;
    G->nlog = 1;
  }
  St S{F_D1, 0, 0, 1, 1, 0, 0, 0, 0, 0, -1, 0, 1, 0};
  long long edges = 0, walked = 0;
  // grid ranks interleave blocks (rank = thread * blocks + block): a small
  // frontier spreads over every SM instead of filling block 0
  const Ex EG{(int)(threadIdx.x * gridDim.x + blockIdx.x), T, true, &G->bar, (const int*)G};
  const Ex EB{(int)threadIdx.x, (int)blockDim.x, false, &G->bar, (const int*)G};
  // %globaltimer profile (thread 0): ns in solo segments, grid degree-one
  // sweeps, grid triangle sweeps, high-degree points
  unsigned long long tcat[4] = {0, 0, 0, 0}, tprev = gt == 0 ? globaltimer() : 0;
  auto tick = [&](int c) {
    if (gt == 0) {
      const unsigned long long now = globaltimer();
      tcat[c] += now - tprev;
      tprev = now;
    }
  };
  while (S.phase != F_DONE) {
    if (cld(G, &G->err)) break;
    const int work = S.phase == F_D1 ? cld(G, &G->cnt1[S.p1]) : cld(G, &G->cnt2[S.p2]);
    if (S.phase != F_HD && work < solo_max) {
      if (blockIdx.x == 0) {
        while (true) {
          if (S.phase == F_D1) sweep_d1(EB, F, G, &q, off, nbr, S, &edges, &walked);
          else sweep_tri(EB, F, G, &q, off, nbr, S, &edges, &walked);
          S.solo += 1;
          if (S.phase == F_HD || cld(G, &G->err)) break;
          const int wk = S.phase == F_D1 ? cld(G, &G->cnt1[S.p1]) : cld(G, &G->cnt2[S.p2]);
          if (wk >= solo_max) break;
        }
        if (threadIdx.x == 0) G->st = S;
      }
      grid_barrier(&G->bar, (const int*)G);
      {
        const volatile int* r = (const volatile int*)&G->st;
        int* p = (int*)&S;
        for (int i = 0; i < (int)(sizeof(St) / sizeof(int)); ++i) p[i] = r[i];
      }
      tick(0);
      continue;
    }
    const int c = S.phase == F_D1 ? 1 : S.phase == F_TRI ? 2 : 3;
    if (S.phase == F_D1) sweep_d1(EG, F, G, &q, off, nbr, S, &edges, &walked);
    else if (S.phase == F_TRI) sweep_tri(EG, F, G, &q, off, nbr, S, &edges, &walked);
    else sweep_hd(F, G, &q, off, nbr, wsmem, n, budget, hd_out, S, &bs);
    tick(c);
  }
  // forced ids in index order (each thread owns a contiguous chunk), the
  // live window, and the totals
  int b, e;
  {
    const long long per = ((long long)n + T - 1) / T;
    const long long s0 = (long long)gt * per, t0 = s0 + per;
    b = (int)(s0 < n ? s0 : n);
    e = (int)(t0 < n ? t0 : n);
  }
  int cnt = 0, mn = kInf, mx = -1;
  for (int v = b; v < e; ++v) {
    cnt += F.forced[v];
    const uint32_t w = __ldcg(F.deg + v);
    const int dv = dval(w);
    if (w != (uint32_t)dv) F.deg[v] = (uint32_t)dv;  // plain degrees for the host / next launch
    if (dv > 0) {
      mn = min(mn, v);
      mx = v;
    }
  }
  int btot;
  const int at = block_exscan(cnt, &bs, &btot);
  {
    int vals[2] = {mn, mx};
    const int op[2] = {1, 2};
    block_reduce<2>(vals, op, &bs);
    if (threadIdx.x == 0) {
      G->partial[blockIdx.x] = btot;
      if (vals[0] != kInf) atomicMax(&G->wlo, kInf - vals[0]);
      if (vals[1] >= 0) atomicMax(&G->whi, vals[1] + 1);
    }
    long long ew[2] = {edges, walked};
    for (int k = 0; k < 2; ++k) {
      long long x = ew[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) == 0 && x)
        atomicAdd(k ? &G->walked : &G->edges, (unsigned long long)x);
    }
  }
  grid_barrier(&G->bar, (const int*)G);
  int base, total;
  {
    const volatile int* partial = G->partial;
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
        bs.bc[12] = before;
        bs.bc[13] = tot;
      }
    }
    __syncthreads();
    base = bs.bc[12];
    total = bs.bc[13];
  }
  int o = base + at;
  for (int v = b; v < e; ++v)
    if (F.forced[v]) out[o++] = v;
  if (gt == 0) {
    const int whi = vld(&G->whi);
    const int lo = kInf - vld(&G->wlo), hi = whi - 1;
    ret[0] = S.forced;
    ret[1] = S.d1;
    ret[2] = S.d2t;
    ret[3] = S.hd;
    ret[4] = -1;  // removed edges are not counted on the solve path (rm_chunk); unused
    if (hi < 0) {  // pure.py:238 empty window
      ret[5] = n > 1 ? n : 1;
      ret[6] = 0;
    } else {
      ret[5] = lo;
      ret[6] = hi;
    }
    ret[7] = total;
    ret[8] = vld(&G->err);
    ret[9] = S.spec_m;
    ret[10] = S.passes + 1;  // + the final pass
    ret[11] = S.sweeps;
    ret[12] = S.solo;
    ret[13] = (long long)*(volatile unsigned long long*)&G->walked;
    ret[14] = (long long)*(volatile unsigned long long*)&G->items;
    for (int k = 0; k < 4; ++k) ret[15 + k] = (long long)tcat[k];
    for (int k = 0; k < 6; ++k) ret[19 + k] = (long long)G->tph[k];
    ret[25] = (long long)*(volatile unsigned*)&G->nbar;
  }
}

static_assert(offsetof(FrontCtl, edges) <= kHdr * sizeof(int), "control header exceeds the cached words");
size_t root_front_ctl_bytes() { return sizeof(FrontCtl); }

// VCG_TRACE: the per-sweep log of the last launch (ctl on the device)
void root_front_print_log(const void* ctl) {
  FrontCtl h;
  if (cudaMemcpy(&h, ctl, sizeof(FrontCtl), cudaMemcpyDeviceToHost) != cudaSuccess) return;
  static const char* nm[4] = {"init", "d1", "tri", "hd"};
  if (h.tph[16])  // -DVCG_FRONT_PROF builds
    fprintf(stderr, "[vcg root]   init us: pass %.1f qflush %.1f barrier %.1f sums %.1f barrier %.1f\n",
            h.tph[16] * 1e-3, h.tph[17] * 1e-3, h.tph[18] * 1e-3, h.tph[19] * 1e-3, h.tph[20] * 1e-3);
  if (h.tph[7]) fprintf(stderr, "[vcg root]   sub-phases us: C vld %.1f chunks %.1f sync %.1f flush %.1f | B work %.1f sync %.1f qflush %.1f cflush %.1f | pre-A %.1f\n",
          h.tph[6] * 1e-3, h.tph[7] * 1e-3, h.tph[8] * 1e-3, h.tph[9] * 1e-3, h.tph[10] * 1e-3,
          h.tph[11] * 1e-3, h.tph[12] * 1e-3, h.tph[1] * 1e-3, h.tph[13] * 1e-3);
  fprintf(stderr, "[vcg root]   init (degrees, lists, sums) %.1f us\n",
          (h.slog[0][1] - h.slog[0][2]) * 1e-3);
  for (int i = 1; i < h.nlog && i < kLog; ++i)
    fprintf(stderr, "[vcg root]   sweep %2d %-4s %7.1f us  frontier %8lld removed %8lld chunks %8lld\n",
            i, nm[h.slog[i][0] & 3], (h.slog[i][1] - h.slog[i - 1][1]) * 1e-3, h.slog[i][2],
            h.slog[i][3], h.slog[i][4]);
}

size_t root_front_bytes(int n, long long m2) {
  const size_t nn = ((size_t)n + 31) & ~(size_t)31;
  // key, nsum, nsq, 10 int arrays, forced, trk, then the chunk list: every vertex
  // is removed at most once, so a step's chunks number at most n + m2 / kChunk
  return 24 * nn + 40 * nn + 2 * nn + 16 * ((size_t)n + (size_t)m2 / kChunk + 1) + 256;
}

template <int TH>
static int front_blocks() {
  static thread_local int dev_cached = -1, blocks = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev != dev_cached) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#if VCG_FRONT_DYNQ
    cudaFuncSetAttribute((const void*)k_root_front<TH>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BlockQ));
#endif
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_root_front<TH>, TH,
                                                  VCG_FRONT_DYNQ ? sizeof(BlockQ) : 0);
    per_sm = per_sm > 2 ? 2 : per_sm;
    blocks = sms * per_sm;
    if (blocks > kRootGridMaxBlocks) blocks = kRootGridMaxBlocks;
    dev_cached = dev;
  }
  return blocks;
}

int root_front_blocks() { return front_blocks<VCG_FRONT_THREADS>(); }

cudaError_t root_front_launch(int n, const int32_t* off, const int32_t* nbr, char* ws,
                              char* front, int budget, int32_t* out, long long* ret, int init,
                              void* ctl) {
  // VCG_FRONT_BIGBLOCK / VCG_FRONT_SMALLBLOCK force a variant (tests, A/B)
  const bool force_big = getenv("VCG_FRONT_BIGBLOCK") != nullptr;  // read per call (tests)
  const bool force_small = getenv("VCG_FRONT_SMALLBLOCK") != nullptr;
  const bool big = (n >= kFrontBigN || force_big) && !force_small;
  const int blocks = big ? front_blocks<1024>() : front_blocks<VCG_FRONT_THREADS>();
  if (blocks < 1) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(FrontCtl), cudaStreamPerThread);
  if (e != cudaSuccess) return e;
  // VCG_FRONT_SOLO: the frontier size below which one block sweeps alone
  static const int solo_env = getenv("VCG_FRONT_SOLO") ? atoi(getenv("VCG_FRONT_SOLO")) : -1;
  int solo_max = solo_env >= 0 ? solo_env : kSolo;
  void* args[] = {&n, &off, &nbr, &ws, &front, &budget, &out, &ret, &init, &ctl, &solo_max};
  const void* kern = big ? (const void*)k_root_front<1024> : (const void*)k_root_front<VCG_FRONT_THREADS>;
  return cudaLaunchCooperativeKernel(kern, dim3(blocks), dim3(big ? 1024 : VCG_FRONT_THREADS), args,
                                     VCG_FRONT_DYNQ ? sizeof(BlockQ) : 0, cudaStreamPerThread);
}

}  // namespace vcg
