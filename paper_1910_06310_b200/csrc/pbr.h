// K2: device partition-based reordering (reorder.py:361-404), bit-exact.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "mgk_dev.cuh"

namespace mgk {
// Computes forward maps (old -> new, local to each graph) for every graph of
// the dataset; returns 0 or an MGK_E_* code with the message in err.
int pbr_device(int G, const std::vector<int64_t>& node_off, const std::vector<int64_t>& edge_off,
               const std::vector<int32_t>& ei, const std::vector<int32_t>& ej, uint64_t seed,
               const Octile* d_tiles, const std::vector<GraphDesc>& graphs, const int32_t* d_trow, int device,
               cudaStream_t stream,
               std::vector<int64_t>& forward, std::string& err);
}  // namespace mgk
