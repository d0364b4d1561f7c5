// dispatch.cuh -- runtime precision tag -> compile-time template argument, plus
// the launch-geometry helpers shared by the launch_*.cu translation units.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "launch.hpp"
#include "levels.cuh"

namespace f3rg {

template <int P>
using PC = std::integral_constant<int, P>;

template <class F>
inline void with_p(int p, F&& f) {
  switch (p) {
    case P16: f(PC<P16>{}); break;
    case P32: f(PC<P32>{}); break;
    default: f(PC<P64>{}); break;
  }
}

// seq: sequential index-order reductions (validation mode, launch.hpp)
inline Sync to_sync(SyncH s) { return Sync{s.partials, s.counter, seq_reductions()}; }
inline Gate to_gate(GateH g) { return Gate{g.dead, g.n}; }
inline Dist to_dist(DistH d) { return Dist{d.mode, d.P, d.loc, d.all}; }

constexpr int kThreads = 256;

// every kernel is launched with programmatic stream serialization (PDL): it may
// start while its predecessor drains, and waits in pdl_wait() (common.cuh) before
// touching anything another kernel wrote. F3RG_PDL=0 turns it off (A/B runs).
bool pdl_enabled();
template <class... KArgs, class... Args>
inline cudaError_t launch_kt(void (*kern)(KArgs...), int grid, int threads, int smem, cudaStream_t s,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <class... KArgs, class... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), int grid, int smem, cudaStream_t s, Args&&... args) {
  return launch_kt(kern, grid, kThreads, smem, s, std::forward<Args>(args)...);
}
// one-thread scalar kernel (state updates between batched kernels)
template <class... KArgs, class... Args>
inline cudaError_t launch_k1(void (*kern)(KArgs...), cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(1);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// occupancy-derived persistent grid for a tile kernel instantiation (cached per
// instantiation by the caller through a function-local static)
template <class K>
inline int occupancy_blocks(K kernel, int smem, int threads = kThreads) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem);
  return nb < 1 ? 1 : nb;
}

}  // namespace f3rg
