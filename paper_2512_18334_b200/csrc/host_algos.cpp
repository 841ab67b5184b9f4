// Host-side runtime pieces of the root pipeline that are inherently
// sequential and run once per solve: the max-degree greedy bound and the
// crown rule's matching.  Both are native C++ (the reference runs them in
// Python), exact restatements of the reference semantics so the reduced
// graph -- and with it every downstream statistic -- is identical.
#include "host_algos.h"

#include <algorithm>
#include <climits>
#include <cstdint>
#include <vector>

namespace vcg {

// preprocess.py:28 greedy_bound -> pure.py:306 greedy_cover: repeatedly take
// the lowest-index vertex of maximum residual degree.
//
// Level form of the same pick sequence: with D the current maximum degree,
// degrees only fall, so the picks at level D are exactly the vertices of
// degree D visited in ascending index order that still have degree D when
// visited (a pick demotes its degree-D neighbours, nothing enters level D).
// Each level's candidates come from an append-only list (a vertex enters
// list[d] once, when its degree reaches d) and are visited through a
// bitmap over their index span.  O(n + m + sum over levels of span/64)
// time, sequential memory traffic apart from the degree updates.
int64_t greedy_cover_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* members,
                          const std::atomic<bool>* cancel) {
  if (n <= 0) return 0;
  std::vector<int32_t> deg(n);
  int64_t m2 = 0, maxdeg = 0;
  // a cancelled greedy (the solve path's lazy bound) must return promptly
  auto cancelled = [&]() { return cancel && cancel->load(std::memory_order_relaxed); };
  for (int64_t v = 0; v < n; ++v) {
    deg[v] = (int32_t)(off[v + 1] - off[v]);
    m2 += deg[v];
    maxdeg = std::max<int64_t>(maxdeg, deg[v]);
    if ((v & 0xffff) == 0 && cancelled()) return -1;
  }
  if (m2 == 0) return 0;
  std::vector<std::vector<int32_t>> level(maxdeg + 1);
  {
    std::vector<int64_t> cnt(maxdeg + 1, 0);
    for (int64_t v = 0; v < n; ++v) ++cnt[deg[v]];
    for (int64_t d = 1; d <= maxdeg; ++d) level[d].reserve((size_t)cnt[d]);
    for (int64_t v = 0; v < n; ++v)
      if (deg[v]) level[deg[v]].push_back((int32_t)v);
  }
  std::vector<uint64_t> mark((size_t)((n + 63) / 64), 0);
  int64_t size = 0;
  for (int64_t d = maxdeg; d >= 1; --d) {
    std::vector<int32_t>& cand = level[d];
    if (cand.empty()) continue;
    if (cancelled()) return -1;
    int64_t wlo = INT64_MAX, whi = -1;
    for (int32_t v : cand)
      if (deg[v] == d) {
        mark[v >> 6] |= 1ull << (v & 63);
        wlo = std::min<int64_t>(wlo, v >> 6);
        whi = std::max<int64_t>(whi, v >> 6);
      }
    std::vector<int32_t>().swap(cand);
    for (int64_t w = wlo; w <= whi; ++w) {
      uint64_t bits = mark[w];
      mark[w] = 0;
      while (bits) {
        const int64_t v = w * 64 + __builtin_ctzll(bits);
        bits &= bits - 1;
        if (deg[v] != d) continue;  // demoted by an earlier pick of this level
        if ((size & 0xfff) == 0 && cancelled()) return -1;
        for (int64_t i = off[v]; i < off[v + 1]; ++i) {
          const int32_t u = nbr[i];
          if (deg[u] > 0) {
            const int32_t du = --deg[u];
            if (du) level[du].push_back(u);
          }
        }
        deg[v] = 0;
        if (members) members[size] = (int32_t)v;
        ++size;
      }
    }
  }
  return size;
}

int64_t maximal_matching_host(int64_t n, const int64_t* off, const int32_t* nbr) {
  std::vector<uint8_t> matched((size_t)std::max<int64_t>(n, 1), 0);
  int64_t size = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (matched[v]) continue;
    for (int64_t i = off[v]; i < off[v + 1]; ++i) {
      const int32_t x = nbr[i];
      if (x != v && !matched[x]) {
        matched[v] = matched[x] = 1;
        ++size;
        break;
      }
    }
  }
  return size;
}

namespace {

constexpr int kAbsent = -2;
constexpr int kBarred = -1;

// reductions.py:200 _try_augment: iterative alternating DFS restricted to the
// current BFS layering; the per-vertex iterators persist across backtracking.
bool try_augment(int32_t root, const std::vector<std::vector<int32_t>>& adj,
                 const std::vector<int32_t>& left_slot, std::vector<int>& dist,
                 std::vector<int32_t>& pair_left, std::vector<int32_t>& pair_right) {
  struct Frame {
    int32_t v;
    size_t it;
  };
  std::vector<Frame> stack{{root, 0}};
  std::vector<std::pair<int32_t, int32_t>> trail;
  while (!stack.empty()) {
    Frame& f = stack.back();
    const auto& edges = adj[left_slot[f.v]];
    bool advanced = false;
    while (f.it < edges.size()) {
      int32_t h = edges[f.it++];
      int32_t w = pair_right[h];
      if (w < 0) {
        pair_left[f.v] = h;
        pair_right[h] = f.v;
        for (auto& th : trail) {
          pair_left[th.first] = th.second;
          pair_right[th.second] = th.first;
        }
        return true;
      }
      if (dist[w] != kAbsent && dist[w] == dist[f.v] + 1) {
        trail.emplace_back(f.v, h);
        int32_t v = f.v;
        (void)v;
        stack.push_back(Frame{w, 0});
        advanced = true;
        break;
      }
    }
    if (!advanced) {
      dist[stack.back().v] = kBarred;
      stack.pop_back();
      if (!trail.empty()) trail.pop_back();
    }
  }
  return false;
}

}  // namespace

// Per-thread scratch of size n, initialised once and restored after every
// call by walking the entries the call touched: a crown round on a 1M-vertex
// graph with a small live set used to spend ~1 ms allocating and clearing
// seven n-sized arrays.
namespace {
struct CrownScratch {
  std::vector<int32_t> partner, left_slot, pair_left, pair_right;
  std::vector<int> dist;
  std::vector<char> in_crown, is_head;
  void fit(int64_t n) {
    if ((int64_t)partner.size() >= n) return;
    partner.assign(n, -1);
    left_slot.assign(n, -1);
    pair_left.assign(n, -1);
    pair_right.assign(n, -1);
    dist.assign(n, kAbsent);
    in_crown.assign(n, 0);
    is_head.assign(n, 0);
  }
};
thread_local CrownScratch t_crown;
}  // namespace

// reductions.py:263 crown_reduce on a host degree array (int32, in/out).
int64_t crown_reduce_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* deg,
                          int64_t lo, int64_t hi, std::vector<int32_t>* heads_out,
                          int64_t* edges_removed, std::vector<int32_t>* crown_out) {
  heads_out->clear();
  if (crown_out) crown_out->clear();
  *edges_removed = 0;
  if (lo > hi) return 0;
  std::vector<int32_t> live;
  for (int64_t v = lo; v <= hi; ++v)
    if (deg[v] > 0) live.push_back((int32_t)v);
  if (live.empty()) return 0;
  CrownScratch& X = t_crown;
  X.fit(n);
  std::vector<int32_t>& partner = X.partner;
  std::vector<int32_t>& left_slot = X.left_slot;
  std::vector<int32_t>& pair_left = X.pair_left;
  std::vector<int32_t>& pair_right = X.pair_right;
  std::vector<int>& dist = X.dist;
  std::vector<char>& in_crown = X.in_crown;
  std::vector<char>& is_head = X.is_head;
  // every index written below is a live vertex (live vertices lie in the
  // window, and partners, heads and left vertices are live): restore them
  struct Restore {
    CrownScratch& X;
    const std::vector<int32_t>& live;
    ~Restore() {
      for (int32_t v : live) {
        X.partner[v] = X.left_slot[v] = X.pair_left[v] = X.pair_right[v] = -1;
        X.dist[v] = kAbsent;
        X.in_crown[v] = X.is_head[v] = 0;
      }
    }
  } restore{X, live};
  for (int32_t v : live) {
    if (partner[v] >= 0) continue;
    for (int64_t i = off[v]; i < off[v + 1]; ++i) {
      int32_t u = nbr[i];
      if (deg[u] > 0 && partner[u] < 0) {
        partner[v] = u;
        partner[u] = v;
        break;
      }
    }
  }
  std::vector<int32_t> outside;
  for (int32_t v : live)
    if (partner[v] < 0) outside.push_back(v);
  if (outside.empty()) return 0;
  std::vector<std::vector<int32_t>> adj(outside.size());
  for (size_t i = 0; i < outside.size(); ++i) {
    int32_t v = outside[i];
    left_slot[v] = (int32_t)i;
    for (int64_t j = off[v]; j < off[v + 1]; ++j)
      if (deg[nbr[j]] > 0) adj[i].push_back(nbr[j]);
  }
  // reductions.py:229 _hopcroft_karp
  std::vector<int32_t> touched;
  while (true) {
    for (int32_t t : touched) dist[t] = kAbsent;
    touched.clear();
    std::vector<int32_t> queue;
    for (int32_t v : outside) {
      if (pair_left[v] < 0) {
        dist[v] = 0;
        touched.push_back(v);
        queue.push_back(v);
      }
    }
    bool reachable_free = false;
    for (size_t qh = 0; qh < queue.size(); ++qh) {
      int32_t v = queue[qh];
      for (int32_t h : adj[left_slot[v]]) {
        int32_t w = pair_right[h];
        if (w < 0) {
          reachable_free = true;
        } else if (dist[w] == kAbsent) {
          dist[w] = dist[v] + 1;
          touched.push_back(w);
          queue.push_back(w);
        }
      }
    }
    if (!reachable_free) break;
    int augmented = 0;
    for (int32_t root : outside)
      if (pair_left[root] < 0 && try_augment(root, adj, left_slot, dist, pair_left, pair_right))
        ++augmented;
    if (augmented == 0) break;
  }
  std::vector<int32_t> crown;
  for (int32_t v : outside)
    if (pair_left[v] < 0) {
      crown.push_back(v);
      in_crown[v] = 1;
    }
  if (crown.empty()) return 0;
  std::vector<int32_t> heads;
  while (true) {
    for (int32_t h : heads) is_head[h] = 0;
    heads.clear();
    for (int32_t v : crown)
      for (int32_t h : adj[left_slot[v]])
        if (!is_head[h]) {
          is_head[h] = 1;
          heads.push_back(h);
        }
    std::vector<int32_t> fresh;
    for (int32_t h : heads) {
      int32_t w = pair_right[h];
      if (w >= 0 && !in_crown[w]) {
        in_crown[w] = 1;
        fresh.push_back(w);
      }
    }
    if (fresh.empty()) break;
    crown.insert(crown.end(), fresh.begin(), fresh.end());
  }
  std::sort(heads.begin(), heads.end());
  int64_t er = 0;
  for (int32_t h : heads) {
    int32_t d = deg[h];
    if (d == 0) continue;
    for (int64_t i = off[h]; i < off[h + 1]; ++i) {
      int32_t u = nbr[i];
      if (deg[u] > 0) --deg[u];
    }
    deg[h] = 0;
    er += d;
  }
  *heads_out = heads;
  *edges_removed = er;
  if (crown_out) {
    std::sort(crown.begin(), crown.end());
    *crown_out = std::move(crown);
  }
  return (int64_t)heads.size();
}

}  // namespace vcg
