// Host-side runtime pieces of the root pipeline that are inherently
// sequential and run once per solve: the max-degree greedy bound and the
// crown rule's matching.  Both are native C++ (the reference runs them in
// Python), exact restatements of the reference semantics so the reduced
// graph -- and with it every downstream statistic -- is identical.
#include "host_algos.h"

#include <algorithm>
#include <queue>
#include <vector>

namespace vcg {

// preprocess.py:348 greedy_bound -> pure.py:306 greedy_cover: repeatedly take
// the lowest-index vertex of maximum residual degree.
//
// Degree buckets as three-level bitsets (64-bit words, a summary bit per
// word, a summary bit per summary word): the pick is "highest non-empty bucket, lowest set bit", a vertex
// moves one bucket down per removed neighbour.  O(m + picks * n/2^18) time;
// falls back to a lazy max-heap when buckets x n bits would exceed 256 MiB.
namespace {

struct Buckets {
  // per degree bucket: L0 vertex bits, L1 = non-empty L0 words, L2 = non-empty L1 words
  int64_t w0, w1, w2;
  std::vector<uint64_t> b0, b1, b2;
  std::vector<int64_t> count;
  Buckets(int64_t n, int64_t maxdeg)
      : w0((n + 63) / 64), w1((w0 + 63) / 64), w2((w1 + 63) / 64),
        b0((size_t)(maxdeg + 1) * w0, 0), b1((size_t)(maxdeg + 1) * w1, 0),
        b2((size_t)(maxdeg + 1) * w2, 0), count(maxdeg + 1, 0) {}
  void set(int64_t d, int64_t v) {
    const int64_t i0 = v >> 6, i1 = i0 >> 6;
    uint64_t& a = b0[(size_t)d * w0 + i0];
    if (!a) {
      uint64_t& b = b1[(size_t)d * w1 + i1];
      if (!b) b2[(size_t)d * w2 + (i1 >> 6)] |= 1ull << (i1 & 63);
      b |= 1ull << (i0 & 63);
    }
    a |= 1ull << (v & 63);
    ++count[d];
  }
  void clear(int64_t d, int64_t v) {
    const int64_t i0 = v >> 6, i1 = i0 >> 6;
    uint64_t& a = b0[(size_t)d * w0 + i0];
    a &= ~(1ull << (v & 63));
    if (!a) {
      uint64_t& b = b1[(size_t)d * w1 + i1];
      b &= ~(1ull << (i0 & 63));
      if (!b) b2[(size_t)d * w2 + (i1 >> 6)] &= ~(1ull << (i1 & 63));
    }
    --count[d];
  }
  int64_t lowest(int64_t d) const {
    const uint64_t* l2 = &b2[(size_t)d * w2];
    for (int64_t i = 0; i < w2; ++i)
      if (l2[i]) {
        const int64_t i1 = i * 64 + __builtin_ctzll(l2[i]);
        const int64_t i0 = i1 * 64 + __builtin_ctzll(b1[(size_t)d * w1 + i1]);
        return i0 * 64 + __builtin_ctzll(b0[(size_t)d * w0 + i0]);
      }
    return -1;
  }
};

}  // namespace

int64_t greedy_cover_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* members) {
  if (n <= 0) return 0;
  std::vector<uint32_t> deg(n);
  int64_t m2 = 0, maxdeg = 0;
  for (int64_t v = 0; v < n; ++v) {
    deg[v] = (uint32_t)(off[v + 1] - off[v]);
    m2 += deg[v];
    maxdeg = std::max<int64_t>(maxdeg, deg[v]);
  }
  if (m2 == 0) return 0;
  int64_t size = 0;
  if ((maxdeg + 1) * ((n + 63) / 64) * 8 <= (256LL << 20)) {
    Buckets b(n, maxdeg);
    for (int64_t v = 0; v < n; ++v)
      if (deg[v]) b.set(deg[v], v);
    int64_t top = maxdeg;
    while (true) {
      while (top > 0 && b.count[top] == 0) --top;
      if (top == 0) break;
      const int64_t v = b.lowest(top);
      b.clear(top, v);
      for (int64_t i = off[v]; i < off[v + 1]; ++i) {
        const int32_t u = nbr[i];
        if (deg[u] > 0) {
          b.clear(deg[u], u);
          --deg[u];
          if (deg[u]) b.set(deg[u], u);
        }
      }
      deg[v] = 0;
      if (members) members[size] = (int32_t)v;
      ++size;
    }
    return size;
  }
  using Key = std::pair<uint32_t, int64_t>;  // (degree, -index)
  std::priority_queue<Key> heap;
  for (int64_t v = 0; v < n; ++v)
    if (deg[v]) heap.push(Key(deg[v], -v));
  while (!heap.empty()) {
    Key k = heap.top();
    heap.pop();
    int64_t v = -k.second;
    if (deg[v] == 0 || deg[v] != k.first) continue;
    for (int64_t i = off[v]; i < off[v + 1]; ++i) {
      int32_t u = nbr[i];
      if (deg[u] > 0) {
        --deg[u];
        if (deg[u]) heap.push(Key(deg[u], -(int64_t)u));
      }
    }
    deg[v] = 0;
    if (members) members[size] = (int32_t)v;
    ++size;
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

// reductions.py:263 crown_reduce on a host degree array (int32, in/out).
int64_t crown_reduce_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* deg,
                          int64_t lo, int64_t hi, std::vector<int32_t>* heads_out,
                          int64_t* edges_removed) {
  heads_out->clear();
  *edges_removed = 0;
  if (lo > hi) return 0;
  std::vector<int32_t> live;
  for (int64_t v = lo; v <= hi; ++v)
    if (deg[v] > 0) live.push_back((int32_t)v);
  if (live.empty()) return 0;
  std::vector<int32_t> partner(n, -1);
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
  std::vector<int32_t> left_slot(n, -1);
  std::vector<std::vector<int32_t>> adj(outside.size());
  for (size_t i = 0; i < outside.size(); ++i) {
    int32_t v = outside[i];
    left_slot[v] = (int32_t)i;
    for (int64_t j = off[v]; j < off[v + 1]; ++j)
      if (deg[nbr[j]] > 0) adj[i].push_back(nbr[j]);
  }
  // reductions.py:229 _hopcroft_karp
  std::vector<int32_t> pair_left(n, -1), pair_right(n, -1);
  std::vector<int> dist(n, kAbsent);
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
  std::vector<char> in_crown(n, 0), is_head(n, 0);
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
  return (int64_t)heads.size();
}

}  // namespace vcg
