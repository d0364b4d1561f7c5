// launch_rich.cu -- runtime dispatch of the tiled kernels on the matrix precision
// (the instantiations live in launch_tile_inst.cu).
#include "launch_tile_decl.hpp"

namespace f3rg {

#define F3RG_BY_PA(pa, CALL)                              \
  switch (pa) {                                           \
    case 0: return CALL(0);                               \
    case 1: return CALL(1);                               \
    case 2: return CALL(2);                               \
    default: return cudaErrorInvalidValue;                \
  }

cudaError_t launch_spmv_dots(int pa, int pz, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* z,
                             void* V, uint64_t ld, int j, LevelState* L, GateH gate, SyncH sync, double* dots,
                             int defer, int* grid_out, DistH dist) {
#define C_(P) launch_spmv_dots_t<P>(pz, pw, l, A, T, z, V, ld, j, L, gate, sync, dots, defer, grid_out, dist)
  F3RG_BY_PA(pa, C_)
#undef C_
}

cudaError_t launch_residual(int pa, int px, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* x,
                            const double* b, void* r, LevelState* L, double* out_norm, SyncH sync, DistH dist) {
#define C_(P) launch_residual_t<P>(px, pw, l, A, T, x, b, r, L, out_norm, sync, dist)
  F3RG_BY_PA(pa, C_)
#undef C_
}

cudaError_t launch_spmv(int pa, int px, int py, Launch l, const CsrDev& A, const TilesDev& T, const void* x, void* y) {
#define C_(P) launch_spmv_t<P>(px, py, l, A, T, x, y)
  F3RG_BY_PA(pa, C_)
#undef C_
}

cudaError_t launch_richardson(int pa, int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, const void* v,
                              const double* v_scale, void* out, uint64_t n, RichState* RS, GateH gate, int level,
                              unsigned long long* cnt, SyncH sync, unsigned* bar_count, unsigned* bar_gen,
                              const IoSlot* io, uint64_t voff, int flags) {
#define C_(P) \
  launch_richardson_t<P>(pw, pv, l, A, T, v, v_scale, out, n, RS, gate, level, cnt, sync, bar_count, bar_gen, io, voff, flags)
  F3RG_BY_PA(pa, C_)
#undef C_
}

cudaError_t launch_rich_phase(int pa, int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                              const void* v, const double* v_scale, uint64_t off, void* out, uint64_t n,
                              RichState* RS, void* R, void* Za, GateH gate, int level, unsigned long long* cnt,
                              SyncH sync, DistH dist) {
#define C_(P) \
  launch_rich_phase_t<P>(pw, pv, l, A, T, phase, k, v, v_scale, off, out, n, RS, R, Za, gate, level, cnt, sync, dist)
  F3RG_BY_PA(pa, C_)
#undef C_
}

cudaError_t launch_richm_phase(int pa, int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                               const void* v, const double* v_scale, void* out, uint64_t n, RichState* RS, void* R,
                               void* P, void* Za, GateH gate, int level, unsigned long long* cnt, SyncH sync) {
#define C_(PP) launch_richm_phase_t<PP>(pw, pv, l, A, T, phase, k, v, v_scale, out, n, RS, R, P, Za, gate, level, cnt, sync)
  F3RG_BY_PA(pa, C_)
#undef C_
}

}  // namespace f3rg
