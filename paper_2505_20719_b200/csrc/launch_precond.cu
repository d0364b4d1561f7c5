// launch_precond.cu -- launchers of the block-Jacobi ILU(0)/IC(0) sweeps (trsv.cuh).
#include <cstdlib>

#include "dispatch.cuh"
#include "trsv.cuh"

namespace f3rg {

// Persistent grid, capped at the co-resident capacity (the sweeps' progress argument
// needs every CTA to become resident) and at one warp per slice. F3RG_SWEEP_CTAS
// sets CTAs per SM (default 1: ~9 levels of slices in flight already cover the
// latency, and fewer polling warps leave L2 to the critical path; measured).
template <class K>
static int sweep_grid(K kern, uint32_t nslices) {
  static const int per_sm = [] {
    const char* e = std::getenv("F3RG_SWEEP_CTAS");
    const int v = e ? std::atoi(e) : 1;
    return v < 1 ? 1 : v;
  }();
  const int occ = occupancy_blocks(kern, 0);
  long g = (long)std::min(occ, per_sm) * sm_count();
  const long need = ((long)nslices * 32 + kThreads - 1) / kThreads;
  if (g > need) g = need;
  return g < 1 ? 1 : (int)g;
}

cudaError_t launch_sweep_fwd(int pf, int pin, Launch l, const SweepDev& S, const void* r, void* cells,
                             unsigned* level_done, SweepCtl* ctl, GateH gate) {
  cudaError_t err = cudaErrorInvalidValue;
  with_p(pf, [&](auto F) {
    with_p(pin, [&](auto I) {
      auto kern = k_sweep_fwd<decltype(F)::value, decltype(I)::value>;
      const int g = l.grid ? l.grid : sweep_grid(kern, S.nslices);
      launch_k(kern, g, 0, l.stream, S, r, cells, level_done, ctl, to_gate(gate));
      err = cudaGetLastError();
    });
  });
  return err;
}

cudaError_t launch_sweep_bwd(int pf, int pc, int pout, Launch l, const SweepDev& S, const void* fcells, void* cells,
                             void* out, unsigned* level_done, SweepCtl* ctl, GateH gate, RichEpiH re) {
  cudaError_t err = cudaErrorInvalidValue;
  with_p(pf, [&](auto F) {
    constexpr int TF = decltype(F)::value;
    with_p(pc, [&](auto Cc) {
      constexpr int C = decltype(Cc)::value;
      if constexpr (C >= TF) {
        with_p(pout, [&](auto O) {
          auto kern = k_sweep_bwd<TF, C, decltype(O)::value>;
          const int g = l.grid ? l.grid : sweep_grid(kern, S.nslices);
          launch_k(kern, g, 0, l.stream, S, fcells, cells, out, level_done, ctl, to_gate(gate),
                   RichEpi{re.RS, re.k, re.zin, re.zout});
          err = cudaGetLastError();
        });
      }
    });
  });
  return err;
}

}  // namespace f3rg
