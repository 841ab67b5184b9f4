// Persistent search kernel, warp tasks of up to 128 vertices (search_impl.cuh).
#include "search_impl.cuh"

namespace vcg {

template __global__ void search_kernel<uint8_t, true, 2>(SearchParams);
template __global__ void search_kernel<uint16_t, true, 2>(SearchParams);
template __global__ void search_kernel<uint32_t, true, 2>(SearchParams);
template __global__ void search_kernel<uint8_t, false, 2>(SearchParams);
template __global__ void search_kernel<uint16_t, false, 2>(SearchParams);
template __global__ void search_kernel<uint32_t, false, 2>(SearchParams);

}  // namespace vcg
