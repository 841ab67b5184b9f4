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

}  // namespace vcg
