#pragma once
#include <cstdint>
#include <vector>

namespace vcg {

// greedy max-degree cover of a CSR graph; members (nullable) gets the picks
int64_t greedy_cover_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* members);

// one crown reduction on deg (int32, mutated); returns #heads forced
int64_t crown_reduce_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* deg,
                          int64_t lo, int64_t hi, std::vector<int32_t>* heads_out,
                          int64_t* edges_removed);

}  // namespace vcg
