// Exhaustive minimum vertex cover for small graphs (oracle.py:28
// brute_force_mvc), on the device.
//
// The reference branches on edges with memoisation and then builds the
// lexicographically smallest minimum cover by a greedy over vertex ids
// (oracle.py:67-78).  Here every subset S of the n <= 26 vertices is a
// candidate: S is a cover iff its complement is independent.  Among covers,
// the reference's witness is the smallest size first and then the
// lexicographically smallest sorted tuple, i.e. the set that contains the
// smallest element of any symmetric difference -- the largest bit-reversed
// mask.  One 64-bit key (size << 32 | ~reversed mask) per cover, reduced with
// atomicMin over a grid-stride enumeration of the 2^n masks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/vcgpu.h"

namespace {

constexpr int kMaxN = 26;

__global__ void k_brute(int n, const unsigned* adj, unsigned long long* best) {
  __shared__ unsigned sadj[kMaxN];
  if (threadIdx.x < (unsigned)n) sadj[threadIdx.x] = adj[threadIdx.x];
  __syncthreads();
  const unsigned full = n == 32 ? 0xffffffffu : ((1u << n) - 1u);
  const unsigned long long total = 1ull << n;
  unsigned long long mine = ~0ull;
  for (unsigned long long m = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; m < total;
       m += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned s = (unsigned)m;
    const unsigned c = ~s & full;  // complement must be independent
    unsigned rest = c;
    bool ok = true;
    while (rest) {
      const int v = __ffs(rest) - 1;
      rest &= rest - 1;
      if (sadj[v] & c) {
        ok = false;
        break;
      }
    }
    if (!ok) continue;
    const unsigned rev = __brev(s) >> (32 - n);
    const unsigned long long key =
        ((unsigned long long)__popc(s) << 32) | (unsigned long long)(~rev & full);
    mine = key < mine ? key : mine;
  }
  // warp minimum, then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, mine, o);
    mine = y < mine ? y : mine;
  }
  if ((threadIdx.x & 31) == 0 && mine != ~0ull) atomicMin(best, mine);
}

}  // namespace

extern "C" const char* vcg_last_error(void);
int vcg_fail_external(int code, const char* msg);  // capi.cu: records the message
void vcg_note_launch(int k);                       // capi.cu: launch counter

extern "C" int vcg_brute_force_mvc(int64_t n, const int64_t* offsets, const int32_t* neighbors,
                                   int64_t* size, int32_t* witness) {
  if (!offsets || !size || n < 0) return vcg_fail_external(VCG_EINVAL, "bad arguments");
  if (n > kMaxN)
    return vcg_fail_external(VCG_EINVAL, ("oracle limited to 26 vertices, got " +
                                          std::to_string(n)).c_str());
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    return vcg_fail_external(VCG_ENODEV, "no CUDA device available");
  *size = 0;
  if (n == 0) return 0;
  std::vector<unsigned> adj(n, 0u);
  for (int64_t v = 0; v < n; ++v)
    for (int64_t i = offsets[v]; i < offsets[v + 1]; ++i) adj[v] |= 1u << neighbors[i];
  unsigned* dadj = nullptr;
  unsigned long long* dbest = nullptr;
  const unsigned long long init = ~0ull;
  unsigned long long key = 0;
  cudaError_t e = cudaMalloc(&dadj, n * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dbest, 8);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dadj, adj.data(), n * 4, cudaMemcpyHostToDevice, cudaStreamPerThread);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dbest, &init, 8, cudaMemcpyHostToDevice, cudaStreamPerThread);
  if (e == cudaSuccess) {
    const unsigned long long total = 1ull << n;
    const int threads = 256;
    const int blocks = (int)std::min<unsigned long long>((total + threads - 1) / threads, 148 * 32);
    vcg_note_launch(1);
    k_brute<<<blocks, threads, 0, cudaStreamPerThread>>>((int)n, dadj, dbest);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&key, dbest, 8, cudaMemcpyDeviceToHost, cudaStreamPerThread);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamPerThread);
  if (dadj) cudaFree(dadj);
  if (dbest) cudaFree(dbest);
  if (e != cudaSuccess) return vcg_fail_external(VCG_ECUDA, cudaGetErrorString(e));
  const unsigned full = (unsigned)((1ull << n) - 1);
  const unsigned rev = ~(unsigned)(key & 0xffffffffu) & full;
  *size = (int64_t)(key >> 32);
  int64_t k = 0;
  for (int64_t v = 0; v < n; ++v)  // bit (n - 1 - v) of the reversed mask is vertex v
    if (rev >> (n - 1 - v) & 1u) {
      if (witness) witness[k] = (int32_t)v;
      ++k;
    }
  return 0;
}
