// Persistent search kernel: the warp-tier-64 instantiations (search_impl.cuh
// holds the template), plus the per-solve init and post-stop drain kernels.
#include "search_impl.cuh"

namespace vcg {

// single-thread drain of records pushed after the in-kernel drain
// (engine.py:216), then publish the result words for one readback
__global__ void drain_kernel(SearchParams P) {
  if (threadIdx.x != 0) return;
  P.ctl->t_end = globaltimer();
  while (true) {
    long long pos = q_reserve_pop(P.q);
    if (pos < 0) break;
    const NodeHdr* hh = (const NodeHdr*)(P.q.data + (pos % P.q.cap) * P.slot_bytes);
    int scope = __ldcg(&hh->scope);
    q_release_pop(P.q, pos);
    reg_finish(P, scope);
  }
  warp_ring_drain(P);
  __threadfence();
  P.ctl->root_key = ld_relaxed(&P.reg.key[P.root_index]);
  P.ctl->reg_count = ld_relaxed(P.reg.count);
}

// one launch resets every per-solve structure: root registry entry, arena
// counter, worklist ring, control block (with the deadline) and histogram
__global__ void search_init_kernel(SearchParams P, int root_key, unsigned long long timeout_ns) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < P.q.cap; i += nth) P.q.seq[i] = (unsigned long long)i;
  for (long long i = tid; i < P.bq.cap; i += nth) P.bq.seq[i] = (unsigned long long)i;
  for (long long i = tid; i < P.n + 2; i += nth) P.hist[i] = 0ull;
  if (tid == 0) {
    const Registry& R = P.reg;
    const int r = P.root_index;
    R.key[r] = root_key;
    R.live[r] = 1;
    R.link[r] = -1;
    R.kind[r] = 0;
    R.sum[r] = R.sum_ach[r] = R.init_sum[r] = R.folded[r] = 0;
    R.first_child[r] = R.nchild[r] = R.disc_done[r] = R.child_folded[r] = 0;
    if (P.record) {
      R.wkey[r] = kNoWitness;
      *P.wcount = 0;
    }
    *R.count = 1;
    for (int c = 0; c < kFreeClasses * kFreeShards; ++c) R.fheads[c] = 0xffffffffull;
    *P.q.head = 0ull;
    *P.q.tail = 0ull;
    *P.q.count = 0ull;
    *P.bq.head = 0ull;
    *P.bq.tail = 0ull;
    *P.bq.count = 0ull;
    *P.sg_count = 0;
    *P.arena_top = 0;
    Ctl* c = P.ctl;
    unsigned long long* cw = (unsigned long long*)c;
    for (size_t i = 0; i < sizeof(Ctl) / 8; ++i) cw[i] = 0ull;
    c->deadline_ns = timeout_ns ? globaltimer() + timeout_ns : 0ull;
    c->t_task_first = ~0ull;
  }
}

template __global__ void search_kernel<uint8_t, true, 1>(SearchParams);
template __global__ void search_kernel<uint16_t, true, 1>(SearchParams);
template __global__ void search_kernel<uint32_t, true, 1>(SearchParams);
template __global__ void search_kernel<uint8_t, false, 1>(SearchParams);
template __global__ void search_kernel<uint16_t, false, 1>(SearchParams);
template __global__ void search_kernel<uint32_t, false, 1>(SearchParams);

}  // namespace vcg
