// launch_t64.cu -- tiled-kernel instantiations for fp64 matrix replicas (launch_tile.cuh).
#include "launch_tile.cuh"

namespace f3rg {
F3RG_TILE_INSTANTIATE(P64)
}  // namespace f3rg
