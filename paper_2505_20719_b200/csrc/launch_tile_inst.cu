// launch_tile_inst.cu -- one (matrix precision, kernel family) slice of the tiled-kernel
// launchers of launch_tile.cuh. buildlib.py compiles this file 18 times, with
// -DF3RG_INST_PA=0|1|2 (fp16 / fp32 / fp64 replica) and -DF3RG_INST_FAMILY=0..5, so
// the heavy template bodies (every column stream x tile shape) compile in parallel.
#include "launch_tile.cuh"

#ifndef F3RG_INST_PA
#error "compile with -DF3RG_INST_PA=<0|1|2> -DF3RG_INST_FAMILY=<0..5> (buildlib.py)"
#endif

namespace f3rg {
#if F3RG_INST_FAMILY == 0
template cudaError_t launch_spmv_dots_t<F3RG_INST_PA>(int, int, Launch, const CsrDev&, const TilesDev&, const void*,
                                                      void*, uint64_t, int, LevelState*, GateH, SyncH, double*, int,
                                                      int*, DistH);
#elif F3RG_INST_FAMILY == 1
template cudaError_t launch_residual_t<F3RG_INST_PA>(int, int, Launch, const CsrDev&, const TilesDev&, const void*,
                                                     const double*, void*, LevelState*, double*, SyncH, DistH);
#elif F3RG_INST_FAMILY == 2
template cudaError_t launch_spmv_t<F3RG_INST_PA>(int, int, Launch, const CsrDev&, const TilesDev&, const void*, void*);
#elif F3RG_INST_FAMILY == 3
template cudaError_t launch_richardson_t<F3RG_INST_PA>(int, int, Launch, const CsrDev&, const TilesDev&, const void*,
                                                       const double*, void*, uint64_t, RichState*, GateH, int,
                                                       unsigned long long*, SyncH, unsigned*, unsigned*,
                                                       const IoSlot*, uint64_t, int);
#elif F3RG_INST_FAMILY == 4
template cudaError_t launch_rich_phase_t<F3RG_INST_PA>(int, int, Launch, const CsrDev&, const TilesDev&, int, int,
                                                       const void*, const double*, uint64_t, void*, uint64_t,
                                                       RichState*, void*, void*, GateH, int, unsigned long long*,
                                                       SyncH, DistH);
#elif F3RG_INST_FAMILY == 5
template cudaError_t launch_richm_phase_t<F3RG_INST_PA>(int, int, Launch, const CsrDev&, const TilesDev&, int, int,
                                                        const void*, const double*, void*, uint64_t, RichState*,
                                                        void*, void*, void*, GateH, int, unsigned long long*, SyncH);
#else
#error "F3RG_INST_FAMILY must be 0..5"
#endif
}  // namespace f3rg
