// L2 atomic throughput microbenchmark (the denominator for the search and
// root kernels' atomic rates): every thread of a full grid issues atomicAdd
// (with return, ATOM) or red.add (no return, RED) on
//   * distinct words spread over 64 MiB (no contention),
//   * one word per warp (32-way contention),
//   * one word for the whole grid (full contention).
// Also a latency probe: one thread, a dependent chain of atomicAdd returns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_atomic_peak l2_atomic_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_atom(unsigned* p, unsigned mask, int iters, unsigned* sink, int mode) {
  const unsigned gt = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned a;
    if (mode == 0) a = (gt * 33u + (unsigned)i * 7919u * 64u) & mask;  // distinct, scattered
    else if (mode == 1) a = ((gt >> 5) * 32u) & mask;                     // one word per warp
    else a = 0;                                                            // one word
    acc += atomicAdd(p + a, 1u);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

__global__ void k_red(unsigned* p, unsigned mask, int iters, int mode) {
  const unsigned gt = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    unsigned a;
    if (mode == 0) a = (gt * 33u + (unsigned)i * 7919u * 64u) & mask;
    else if (mode == 1) a = ((gt >> 5) * 32u) & mask;
    else a = 0;
    atomicAdd(p + a, 1u);  // result unused: RED
  }
}

__global__ void k_chain(unsigned* p, int iters, unsigned* out) {
  unsigned x = 0;
  for (int i = 0; i < iters; ++i) x = atomicAdd(p + (x & 1023u) * 32u, 1u);
  *out = x;
}

int main() {
  const size_t words = 16u << 20;  // 64 MiB
  unsigned *p, *sink;
  cudaMalloc(&p, words * 4);
  cudaMalloc(&sink, 4);
  cudaMemset(p, 0, words * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 64;
  const double ops = (double)blocks * threads * iters;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[3] = {"distinct", "per-warp word", "single word"};
  printf("{\n \"grid\": \"%d x %d threads, %d atomics each\",\n", blocks, threads, iters);
  for (int red = 0; red < 2; ++red)
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        if (red) k_red<<<blocks, threads>>>(p, (unsigned)words - 1, iters, mode);
        else k_atom<<<blocks, threads>>>(p, (unsigned)words - 1, iters, sink, mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf(" \"%s %s\": {\"ms\": %.4f, \"G_atomics_per_s\": %.2f},\n", red ? "RED" : "ATOM",
             names[mode], best, ops / (best * 1e-3) / 1e9);
    }
  {
    const int n = 4096;
    cudaEventRecord(a);
    k_chain<<<1, 1>>>(p, n, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf(" \"dependent ATOM chain latency_ns\": %.1f\n}\n", ms * 1e6 / n);
  }
  return 0;
}
