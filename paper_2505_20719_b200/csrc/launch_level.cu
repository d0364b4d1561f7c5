// launch_level.cu -- launchers for the FGMRES level kernels (levels.cuh).
#include <atomic>
#include <cstdlib>

#include "dispatch.cuh"
#include "levels.cuh"

namespace f3rg {

int sm_count() {
  static int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 1;
  }();
  return sms;
}
int stream_grid() { return sm_count() * 8; }
// tile shape of the host tile builder = the device TileCfg (spmv.cuh)
uint32_t tile_max_rows() { return TileCfg<P16>::NT; }
uint32_t tile_max_nnz(int pa, int shape) {
  if (shape == 1) return pa == P16 ? TileCfg<P16, 4>::TNNZ : pa == P32 ? TileCfg<P32, 4>::TNNZ : TileCfg<P64, 4>::TNNZ;
  if (shape == 2) return pa == P16 ? TileCfg<P16, 8>::TNNZ : pa == P32 ? TileCfg<P32, 8>::TNNZ : TileCfg<P64, 8>::TNNZ;
  return pa == P16 ? TileCfg<P16>::TNNZ : pa == P32 ? TileCfg<P32>::TNNZ : TileCfg<P64>::TNNZ;
}
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}
// CTAs per SM of the reduction kernels with a last-CTA tail (level start, cgs): a
// single wave, few enough partials that the counter atomics and the final
// partial reduction stay short (F3RG_RED_PER_SM / F3RG_CGS_PER_SM for sweeps)
int red_grid() {
  static const int g = sm_count() * env_int("F3RG_RED_PER_SM", 4);
  return g;
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("F3RG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
int max_partial_blocks() { return sm_count() * 8; }
static std::atomic<int>& seq_flag() {
  static std::atomic<int> f{env_int("F3RG_SEQ_REDUCTIONS", 0) != 0};
  return f;
}
int seq_reductions() { return seq_flag().load(std::memory_order_relaxed); }
void set_seq_reductions(int on) { seq_flag().store(on != 0, std::memory_order_relaxed); }

cudaError_t launch_level_start(int ps, int pw, Launch l, void* src, const double* src_scale, int writeback, void* dst,
                               uint64_t n, LevelState* L, int* dead, GateH gate, int level, unsigned long long* cnt,
                               SyncH sync, const IoSlot* io, DistH dist) {
  const int g = dist.mode == 2 ? 1 : l.grid ? l.grid : red_grid();
  with_p(ps, [&](auto S) {
    with_p(pw, [&](auto W) {
      launch_k(k_level_start<decltype(S)::value, decltype(W)::value>, g, 0, l.stream, src, src_scale, writeback, dst, n, L, dead, to_gate(gate), level, cnt, to_sync(sync), io, to_dist(dist));
    });
  });
  return cudaGetLastError();
}

cudaError_t launch_copy_scaled(int pw, Launch l, void* v, const double* scale, void* z, uint64_t n, GateH gate,
                               unsigned long long* cnt) {
  const int g = l.grid ? l.grid : stream_grid();
  with_p(pw, [&](auto W) {
    launch_k(k_copy_scaled<decltype(W)::value>, g, 0, l.stream, v, scale, z, n, to_gate(gate), cnt);
  });
  return cudaGetLastError();
}

cudaError_t launch_multi_dot(int pw, Launch l, const void* V, uint64_t n, int j, int k0, LevelState* L, GateH gate,
                             SyncH sync, uint64_t ldv, DistH dist) {
  const int g = dist.mode == 2 ? 1 : l.grid ? l.grid : stream_grid();
  with_p(pw, [&](auto W) {
    launch_k(k_multi_dot<decltype(W)::value>, g, 0, l.stream, V, n, ldv ? ldv : n, j, k0, L, to_gate(gate),
                                                                  to_sync(sync), to_dist(dist));
  });
  return cudaGetLastError();
}

cudaError_t launch_cgs(int pw, Launch l, void* V, uint64_t n, int j, LevelState* L, int* dead, GateH gate, int level,
                       int outer, int use_tol, StepInfo* info, SyncH sync, const double* dots, int dots_grid,
                       uint64_t ldv, DistH dist) {
  const int nj = j + 1 < 8 ? j + 1 : 8;
  with_p(pw, [&](auto W) {
    constexpr int PW = decltype(W)::value;
    auto go = [&](auto NJ_) {
      constexpr int NJ = decltype(NJ_)::value;
      auto kern = k_cgs<PW, NJ>;
      // all co-resident CTAs, one wave (occupancy-derived per instantiation)
      static const int per = env_int("F3RG_CGS_PER_SM", 0);
      static const int g0 = (per > 0 ? per : occupancy_blocks(kern, 0)) * sm_count();
      const int g = dist.mode == 2 ? 1 : l.grid ? l.grid : (g0 < max_partial_blocks() ? g0 : max_partial_blocks());
      launch_k(kern, g, 0, l.stream, V, n, ldv ? ldv : n, j, L, dead, to_gate(gate), level, outer, use_tol, info,
                                         to_sync(sync), dots, dots_grid, to_dist(dist));
    };
    switch (nj) {
      case 1: go(PC<1>{}); break;
      case 2: go(PC<2>{}); break;
      case 3: go(PC<3>{}); break;
      case 4: go(PC<4>{}); break;
      case 5: go(PC<5>{}); break;
      case 6: go(PC<6>{}); break;
      case 7: go(PC<7>{}); break;
      default: go(PC<8>{}); break;
    }
  });
  return cudaGetLastError();
}

cudaError_t launch_level_finish(int pz, int pw, int px, Launch l, const void* Z, uint64_t n, LevelState* L, void* x,
                                int x_is_zero, GateH gate, int level, unsigned long long* cnt, int count_iterations,
                                const IoSlot* io, uint64_t ldz) {
  const int g = l.grid ? l.grid : red_grid();  // every CTA redoes the back-substitution: keep them few
  with_p(pz, [&](auto PZ) {
    with_p(pw, [&](auto W) {
      with_p(px, [&](auto X) {
        launch_k(k_level_finish<decltype(PZ)::value, decltype(W)::value, decltype(X)::value>, g, 0, l.stream, Z, n, ldz ? ldz : n, L, x, x_is_zero, to_gate(gate), level, cnt, count_iterations, io);
      });
    });
  });
  return cudaGetLastError();
}

__global__ void k_set_outer(LevelState* L, double bnorm, double tol) {
  pdl_wait();
  L->bnorm = bnorm;
  L->tol = tol;
}

cudaError_t launch_set_outer(Launch l, LevelState* L, double bnorm, double tol) {
  k_set_outer<<<1, 1, 0, l.stream>>>(L, bnorm, tol);  // plain launch: fully ordered
  return cudaGetLastError();
}

}  // namespace f3rg
