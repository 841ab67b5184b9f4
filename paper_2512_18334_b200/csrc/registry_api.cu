// The completion registry's protocol operations (registry.py:79-224) as a
// standalone device object: the same HBM arena layout and the same atomic
// encodings the search kernel uses (search.cuh Registry / reg_submit /
// reg_cascade), exposed one operation per call -- or one operation per
// device thread, all at once, to exercise the lock-free protocol under
// contention the way the reference's threaded tests do.
//
// Encodings (search.cuh):
//   child  key = best * 2 + !achieved; atomicMin on it is atomic_min_best
//          (a smaller candidate wins; an equal achieved candidate lowers the
//          key by one, which is the reference's "achieved upgrade").
//   live   live_nodes (child) / live_comps (parent), plain atomics.
//   parent sum / sum_ach / folded by atomicAdd / atomicAnd.
// The reference's protocol errors (a counter going negative, an increment on
// a finished entry) are detected here the way registry.py raises them: the
// decrement stays applied, the increment is refused.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/vcgpu.h"

int vcg_fail_external(int code, const char* msg);  // capi.cu
void vcg_note_launch(int k);                       // capi.cu

struct vcg_registry {
  int* arena = nullptr;  // 12 fields x cap, then the entry counter
  long long* dret = nullptr;
  int* derr = nullptr;
  int cap = 0;
  int dev = 0;
};

namespace {

constexpr int kFields = 12;
constexpr int kMaxSeq = 8;

struct Reg {
  int *key, *live, *link, *kind, *sum, *sum_ach, *init_sum, *folded, *first_child, *nchild,
      *disc_done, *child_folded, *count;
  int cap;
};

Reg view(const vcg_registry* r) {
  Reg R;
  int* b = r->arena;
  const int c = r->cap;
  R.key = b;
  R.live = b + c;
  R.link = b + 2 * c;
  R.kind = b + 3 * c;
  R.sum = b + 4 * c;
  R.sum_ach = b + 5 * c;
  R.init_sum = b + 6 * c;
  R.folded = b + 7 * c;
  R.first_child = b + 8 * c;
  R.nchild = b + 9 * c;
  R.disc_done = b + 10 * c;
  R.child_folded = b + 11 * c;
  R.count = b + kFields * c;
  R.cap = c;
  return R;
}

// error codes written to *err (first one wins)
enum : int { kOk = 0, kFull = 1, kIncFinished = 2, kNegative = 3 };

__device__ void set_err(int* err, int e) { atomicCAS(err, kOk, e); }

// an increment refused on a finished entry (registry.py:140 / :179)
__device__ long long inc_checked(int* p, int* err) {
  int old = *(volatile int*)p;
  while (true) {
    if (old < 1) {
      set_err(err, kIncFinished);
      return old;
    }
    const int seen = atomicCAS(p, old, old + 1);
    if (seen == old) return old + 1;
    old = seen;
  }
}

// a decrement that stays applied even when it goes negative (registry.py:149)
__device__ long long dec_checked(int* p, int* err) {
  const int now = atomicSub(p, 1) - 1;
  if (now < 0) set_err(err, kNegative);
  return now;
}

__device__ long long apply(const Reg& R, int op, long long idx, long long a, long long b,
                           long long c, int* err, long long* ret2) {
  switch (op) {
    case VCG_REG_NEW_CHILD: {  // a = best_init, b = parent (-1 none), c = achieved
      const int i = atomicAdd(R.count, 1);
      if (i >= R.cap) {
        set_err(err, kFull);
        return -1;
      }
      R.key[i] = (int)a * 2 + (c ? 0 : 1);
      R.live[i] = 1;
      R.link[i] = (int)b;
      R.kind[i] = 0;
      R.child_folded[i] = 0;
      if (b >= 0) atomicAdd(&R.nchild[b], 1);
      return i;
    }
    case VCG_REG_NEW_PARENT: {  // a = initial_sum, b = ancestor
      const int i = atomicAdd(R.count, 1);
      if (i >= R.cap) {
        set_err(err, kFull);
        return -1;
      }
      R.sum[i] = (int)a;
      R.init_sum[i] = (int)a;
      R.sum_ach[i] = 1;
      R.folded[i] = 0;
      R.live[i] = 1;
      R.link[i] = (int)b;
      R.kind[i] = 1;
      R.disc_done[i] = 0;
      R.nchild[i] = 0;
      R.first_child[i] = -1;
      return i;
    }
    case VCG_REG_ATOMIC_MIN_BEST:  // a = candidate, b = achieved; returns the prior best
      return atomicMin(&R.key[idx], (int)a * 2 + (b ? 0 : 1)) >> 1;
    case VCG_REG_BEST_SNAPSHOT: {
      const int k = *(volatile int*)&R.key[idx];
      *ret2 = (k & 1) ? 0 : 1;
      return k >> 1;
    }
    case VCG_REG_INC_LIVE_NODES:
    case VCG_REG_INC_LIVE_COMPS:
      return inc_checked(&R.live[idx], err);
    case VCG_REG_DEC_LIVE_NODES:
    case VCG_REG_DEC_LIVE_COMPS:
      return dec_checked(&R.live[idx], err);
    case VCG_REG_ADD_TO_SUM: {  // a = delta, b = achieved, c = folded
      const int now = atomicAdd(&R.sum[idx], (int)a) + (int)a;
      if (c) atomicAdd(&R.folded[idx], (int)a);
      if (!b) atomicAnd(&R.sum_ach[idx], 0);
      return now;
    }
    case VCG_REG_MARK_DISCOVERY_DONE:
      atomicExch(&R.disc_done[idx], 1);
      return 0;
  }
  return 0;
}

__global__ void k_reg_one(Reg R, int op, long long idx, long long a, long long b, long long c,
                          long long* ret, int* err) {
  long long r2 = 0;
  ret[0] = apply(R, op, idx, a, b, c, err, &r2);
  ret[1] = r2;
}

struct OpSeq {
  int op[kMaxSeq];
  int n;
};

// thread i runs `rounds` passes of the operation sequence on entry idx[i]
// with arguments (a[i], b[i]); ret[i] = the last operation's result
__global__ void k_reg_many(Reg R, OpSeq seq, int rounds, const long long* idx, const long long* a,
                           const long long* b, long long count, long long* ret, int* err) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= count) return;
  long long r2 = 0, last = 0;
  for (int k = 0; k < rounds; ++k)
    for (int j = 0; j < seq.n; ++j)
      last = apply(R, seq.op[j], idx[i], a ? a[i] : 0, b ? b[i] : 0, 0, err, &r2);
  ret[i] = last;
}

const char* err_text(int e) {
  switch (e) {
    case kFull: return "registry arena full";
    case kIncFinished: return "increment on a completed entry";
    case kNegative: return "live count went negative";
  }
  return "";
}

int cuda_fail(cudaError_t e) { return vcg_fail_external(VCG_ECUDA, cudaGetErrorString(e)); }

int read_count(const vcg_registry* r, int* count) {
  cudaError_t e = cudaMemcpy(count, r->arena + (size_t)kFields * r->cap, 4,
                             cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e);
  if (*count > r->cap) *count = r->cap;
  return 0;
}

bool is_index_op(int op) {
  return op != VCG_REG_NEW_CHILD && op != VCG_REG_NEW_PARENT;
}

}  // namespace

extern "C" int vcg_registry_create(int64_t capacity, vcg_registry** out) {
  if (!out || capacity < 1 || capacity > (1 << 26)) return vcg_fail_external(VCG_EINVAL, "bad capacity");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    return vcg_fail_external(VCG_ENODEV, "no CUDA device available");
  auto* r = new vcg_registry;
  r->cap = (int)capacity;
  cudaGetDevice(&r->dev);
  const size_t bytes = ((size_t)kFields * r->cap + 1) * 4;
  cudaError_t e = cudaMalloc(&r->arena, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&r->dret, 16);
  if (e == cudaSuccess) e = cudaMalloc(&r->derr, 4);
  if (e == cudaSuccess) e = cudaMemset(r->arena, 0, bytes);
  if (e != cudaSuccess) {
    cudaFree(r->arena);
    cudaFree(r->dret);
    cudaFree(r->derr);
    delete r;
    return cuda_fail(e);
  }
  *out = r;
  return 0;
}

extern "C" int vcg_registry_destroy(vcg_registry* r) {
  if (!r) return 0;
  cudaFree(r->arena);
  cudaFree(r->dret);
  cudaFree(r->derr);
  delete r;
  return 0;
}

extern "C" int64_t vcg_registry_size(const vcg_registry* r) {
  int c = 0;
  if (!r || read_count(r, &c)) return -1;
  return c;
}

extern "C" int vcg_registry_op(vcg_registry* r, int op, int64_t idx, int64_t a, int64_t b,
                               int64_t c, int64_t* ret) {
  if (!r || !ret || op < VCG_REG_NEW_CHILD || op > VCG_REG_MARK_DISCOVERY_DONE)
    return vcg_fail_external(VCG_EINVAL, "bad arguments");
  int count = 0;
  if (int rc = read_count(r, &count)) return rc;
  if (is_index_op(op) && (idx < 0 || idx >= count))
    return vcg_fail_external(VCG_EINVAL, ("no registry entry " + std::to_string(idx)).c_str());
  if (op == VCG_REG_NEW_CHILD) {
    if (a < 1)
      return vcg_fail_external(VCG_EINVAL,
                               ("child entry needs best >= 1, got " + std::to_string(a)).c_str());
    if (b >= count) return vcg_fail_external(VCG_EINVAL, "parent entry out of range");
  }
  if (op == VCG_REG_NEW_PARENT && a < 0)
    return vcg_fail_external(VCG_EINVAL, "initial sum must be non-negative");
  cudaError_t e = cudaMemset(r->derr, 0, 4);
  if (e != cudaSuccess) return cuda_fail(e);
  vcg_note_launch(1);
  k_reg_one<<<1, 1>>>(view(r), op, idx, a, b, c, r->dret, r->derr);
  long long h[2] = {0, 0};
  int err = 0;
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(h, r->dret, 16, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&err, r->derr, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e);
  ret[0] = h[0];
  ret[1] = h[1];
  if (err == kFull) return vcg_fail_external(VCG_ERESOURCE, err_text(err));
  if (err)
    return vcg_fail_external(VCG_EPROTOCOL,
                             ("entry " + std::to_string(idx) + ": " + err_text(err)).c_str());
  return 0;
}

extern "C" int vcg_registry_concurrent(vcg_registry* r, const int* ops, int nops, int rounds,
                                       const int64_t* idx, const int64_t* a, const int64_t* b,
                                       int64_t count, int64_t* ret, int* protocol_error) {
  if (!r || !ops || nops < 1 || nops > kMaxSeq || rounds < 1 || !idx || !ret || count < 0)
    return vcg_fail_external(VCG_EINVAL, "bad arguments");
  OpSeq seq{};
  seq.n = nops;
  for (int j = 0; j < nops; ++j) {
    if (!is_index_op(ops[j]) || ops[j] > VCG_REG_MARK_DISCOVERY_DONE)
      return vcg_fail_external(VCG_EINVAL, "concurrent operations act on existing entries");
    seq.op[j] = ops[j];
  }
  if (count == 0) return 0;
  int n = 0;
  if (int rc = read_count(r, &n)) return rc;
  for (int64_t i = 0; i < count; ++i)
    if (idx[i] < 0 || idx[i] >= n) return vcg_fail_external(VCG_EINVAL, "entry out of range");
  long long *d = nullptr;
  const size_t bytes = (size_t)count * 8;
  cudaError_t e = cudaMalloc(&d, bytes * 4);
  if (e != cudaSuccess) return cuda_fail(e);
  long long *di = d, *da = d + count, *db = d + 2 * count, *dr = d + 3 * count;
  e = cudaMemcpy(di, idx, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && a) e = cudaMemcpy(da, a, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && b) e = cudaMemcpy(db, b, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(r->derr, 0, 4);
  if (e == cudaSuccess) {
    vcg_note_launch(1);
    const int threads = 256;
    k_reg_many<<<(unsigned)((count + threads - 1) / threads), threads>>>(
        view(r), seq, rounds, di, a ? da : nullptr, b ? db : nullptr, count, dr, r->derr);
    e = cudaGetLastError();
  }
  int err = 0;
  if (e == cudaSuccess) e = cudaMemcpy(ret, dr, bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&err, r->derr, 4, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e);
  if (protocol_error) *protocol_error = err;
  return 0;
}

// entries [0, count) as rows of 12 int32 fields (the vcg_search
// registry_out layout, include/vcgpu.h), children of a parent counted in
// nchild; the per-child parent links give the lists.
extern "C" int vcg_registry_download(const vcg_registry* r, int32_t* rows, int64_t cap,
                                     int64_t* count) {
  if (!r || !count) return vcg_fail_external(VCG_EINVAL, "bad arguments");
  int n = 0;
  if (int rc = read_count(r, &n)) return rc;
  *count = n;
  if (!rows || n == 0) return 0;
  if (n > cap) return vcg_fail_external(VCG_EINVAL, "row buffer too small");
  std::vector<int> f(n);
  for (int k = 0; k < kFields; ++k) {
    cudaError_t e = cudaMemcpy(f.data(), r->arena + (size_t)k * r->cap, (size_t)n * 4,
                               cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e);
    for (int i = 0; i < n; ++i) rows[(size_t)i * kFields + k] = f[i];
  }
  return 0;
}
