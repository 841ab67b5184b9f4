#pragma once
#include <atomic>
#include <cstdint>
#include <vector>

namespace vcg {

// greedy max-degree cover of a CSR graph; members (nullable) gets the picks;
// returns -1 if `cancel` (nullable) is raised before it finishes
int64_t greedy_cover_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* members,
                          const std::atomic<bool>* cancel = nullptr);

// size of a greedy maximal matching (a lower bound on every vertex cover)
int64_t maximal_matching_host(int64_t n, const int64_t* off, const int32_t* nbr);

// one crown reduction on deg (int32, mutated); returns #heads forced.
// heads_out gets the sorted heads; crown_out (optional) the sorted
// independent side.
int64_t crown_reduce_host(int64_t n, const int64_t* off, const int32_t* nbr, int32_t* deg,
                          int64_t lo, int64_t hi, std::vector<int32_t>* heads_out,
                          int64_t* edges_removed, std::vector<int32_t>* crown_out = nullptr);

}  // namespace vcg
