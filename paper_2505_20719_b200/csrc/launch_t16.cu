// launch_t16.cu -- tiled-kernel instantiations for fp16 matrix replicas (launch_tile.cuh).
#include "launch_tile.cuh"

namespace f3rg {
F3RG_TILE_INSTANTIATE(P16)
}  // namespace f3rg
