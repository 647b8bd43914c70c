#include "pbr.h"
namespace mgk {
int pbr_device(int G, const std::vector<int64_t>& node_off, const std::vector<int64_t>&, const std::vector<int32_t>&,
               const std::vector<int32_t>&, uint64_t, const Octile*, const std::vector<GraphDesc>&, int, cudaStream_t,
               std::vector<int64_t>& forward, std::string& err) {
  err = "device PBR not built yet";
  return -4;
}
}  // namespace mgk
