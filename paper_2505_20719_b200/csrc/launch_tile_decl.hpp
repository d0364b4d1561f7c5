// launch_tile_decl.hpp -- declarations of the per-precision tiled-kernel launchers
// (defined in launch_tile.cuh, instantiated by launch_tile_inst.cu).
#pragma once

#include "launch.hpp"
#include "state.hpp"

namespace f3rg {

template <int PA>
cudaError_t launch_spmv_dots_t(int pz, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* z, void* V,
                               uint64_t ld, int j, LevelState* L, GateH gate, SyncH sync, double* dots, int defer,
                               int* grid_out, DistH dist);
template <int PA>
cudaError_t launch_residual_t(int px, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* x,
                              const double* b, void* r, LevelState* L, double* out_norm, SyncH sync, DistH dist);
template <int PA>
cudaError_t launch_spmv_t(int px, int py, Launch l, const CsrDev& A, const TilesDev& T, const void* x, void* y);
template <int PA>
cudaError_t launch_richardson_t(int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, const void* v,
                                const double* v_scale, void* out, uint64_t n, RichState* RS, GateH gate, int level,
                                unsigned long long* cnt, SyncH sync, unsigned* bar_count, unsigned* bar_gen,
                                const IoSlot* io, uint64_t voff, int flags);
template <int PA>
cudaError_t launch_rich_phase_t(int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                                const void* v, const double* v_scale, uint64_t off, void* out, uint64_t n,
                                RichState* RS, void* R, void* Za, GateH gate, int level, unsigned long long* cnt,
                                SyncH sync, DistH dist);
template <int PA>
cudaError_t launch_richm_phase_t(int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                                 const void* v, const double* v_scale, void* out, uint64_t n, RichState* RS, void* R,
                                 void* P, void* Za, GateH gate, int level, unsigned long long* cnt, SyncH sync);

}  // namespace f3rg
