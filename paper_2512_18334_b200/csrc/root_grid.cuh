// Host interface of the grid-wide root fixpoint (root_grid.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace vcg {

constexpr int kRootGridThreads = 512;
constexpr int kRootGridMaxBlocks = 2048;

// bytes of the kernel's control block (device memory, no initialisation needed)
size_t root_grid_ctl_bytes();
// cooperative grid size on the current device (all blocks co-resident)
int root_grid_blocks();
// One launch = reduce_fixpoint (pure.py:188) on int32 degrees in the HBM
// workspace `ws` (carve_ws layout, n vertices).  Forced ids are written to
// out[0..) in the reference's order.  ret (int64[11]): forced, degree-one,
// triangle, high-degree applications, edges removed, lo, hi, ids written,
// error, speculative-budget record, scans.  init: take the degrees from the
// CSR offsets instead of the workspace.
cudaError_t root_grid_launch(int n, const int32_t* off, const int32_t* nbr, char* ws, int budget,
                             int32_t* out, long long* ret, int init, void* ctl);

// Frontier-driven any-order variant (root_front.cu, the solve path): same
// forced set and rule counts, forced ids in index order.  `front` holds
// root_front_bytes(n) bytes of scratch, `ctl` root_front_ctl_bytes() (zeroed
// by the launch).  ret (int64[15]): as root_grid_launch's first 11 (ret[10] =
// full passes over the degree array), then sweeps, sweeps run by one block,
// adjacency entries walked, frontier entries examined.
size_t root_front_ctl_bytes();
void root_front_print_log(const void* ctl);
size_t root_front_bytes(int n, long long m2);
int root_front_blocks();
cudaError_t root_front_launch(int n, const int32_t* off, const int32_t* nbr, char* ws,
                              char* front, int budget, int32_t* out, long long* ret, int init,
                              void* ctl);

}  // namespace vcg
