// launch_rich.cu -- launcher for the cooperative Richardson kernel (richardson.cuh).
#include "dispatch.cuh"
#include "richardson.cuh"

namespace f3rg {

template <int PA, int PW, int PV>
static int rich_occ() {
  static const int o = occupancy_blocks(k_richardson<PA, PW, PV>, TileCfg<PA>::SMEM_BYTES);
  return o;
}

int richardson_grid(int pa, int pw, int pv, uint32_t ntiles) {
  int occ = 1;
  with_p(pa, [&](auto A) {
    with_p(pw, [&](auto W) {
      with_p(pv, [&](auto V) { occ = rich_occ<decltype(A)::value, decltype(W)::value, decltype(V)::value>(); });
    });
  });
  // every CTA must be co-resident (grid barriers); tiles beyond the grid are
  // processed by the persistent loop
  long g = (long)occ * sm_count();
  (void)ntiles;
  return g < 1 ? 1 : (int)g;
}

cudaError_t launch_richardson(int pa, int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, const void* v,
                              const double* v_scale, void* out, uint64_t n, RichState* RS, GateH gate, int level,
                              unsigned long long* cnt, SyncH sync, unsigned* bar_count, unsigned* bar_gen,
                              const IoSlot* io) {
  cudaError_t err = cudaSuccess;
  with_p(pa, [&](auto PA_) {
    constexpr int PA = decltype(PA_)::value;
    with_p(pw, [&](auto W) {
      with_p(pv, [&](auto V) {
        constexpr int PW = decltype(W)::value, PV = decltype(V)::value;
        const int g = l.grid ? l.grid : richardson_grid(PA, PW, PV, T.ntiles);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = TileCfg<PA>::SMEM_BYTES;
        cfg.stream = l.stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        err = cudaLaunchKernelEx(&cfg, k_richardson<PA, PW, PV>, A, T, v, v_scale, out, n, RS, to_gate(gate), level,
                                 cnt, to_sync(sync), bar_count, bar_gen, io);
      });
    });
  });
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

}  // namespace f3rg
