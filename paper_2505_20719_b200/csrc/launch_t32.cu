// launch_t32.cu -- tiled-kernel instantiations for fp32 matrix replicas (launch_tile.cuh).
#include "launch_tile.cuh"

namespace f3rg {
F3RG_TILE_INSTANTIATE(P32)
}  // namespace f3rg
