// launch_tile.cuh -- launchers of every TMA-tiled kernel (SpMV + fused epilogues)
// for ONE matrix precision PA, instantiated per (precision, kernel family) by
// launch_tile_inst.cu so the heavy template bodies compile in parallel. Only
// combinations the engine can produce are instantiated (a child level's vector
// precision never exceeds its parent's); the column format (u32 or D16) follows
// the matrix.
#pragma once

#include "blas1.cuh"
#include "dispatch.cuh"
#include "levels.cuh"
#include "richardson.cuh"

namespace f3rg {

// column stream of a launch: P16 (packed fp16 value + delta) for the fp16 replica
// when present, else D16, else u32; plus the matrix's tile shape (IDX bit 2)
// shape 3: the windowed SELL engine (wsell.cuh), whose own layout replaces the
// column streams
template <int PA, int SH, class F>
inline void dispatch_col(const CsrDev& A, F&& go) {
  if constexpr (PA == P16) {
    if (A.pk) return go(std::integral_constant<int, 2 | SH>{});
  }
  if (A.dcol) go(std::integral_constant<int, 1 | SH>{});
  else go(std::integral_constant<int, 0 | SH>{});
}
template <int PA, class F>
inline void dispatch_idx(const CsrDev& A, const TilesDev& T, F&& go) {
  if (T.shape == 3) go(std::integral_constant<int, 16>{});
  else if (T.shape == 1) dispatch_col<PA, 4>(A, go);
  else if (T.shape == 2) dispatch_col<PA, 8>(A, go);
  else dispatch_col<PA, 0>(A, go);
}

template <class K>
inline int tile_kernel_grid(K kern, int smem, uint32_t ntiles, bool cap_by_tiles, int threads = kThreads) {
  const int occ = occupancy_blocks(kern, smem, threads);
  long g = (long)occ * sm_count();
  if (cap_by_tiles && g > (long)ntiles) g = ntiles;
  return g < 1 ? 1 : (int)g;
}

// grid of one tile-kernel launch: the occupancy-derived persistent grid (capped by
// the tile count, or the caller's override), or, for the windowed engine, exactly
// the CTA count its window split was made for
// (g0: the caller's per-instantiation cached tile_kernel_grid -- it must be a static
// local of the generic lambda that names the kernel, NOT of a helper templated on
// the kernel's pointer type: kernels of one signature would share it and all but
// the first would miss their cudaFuncSetAttribute)
template <int IDX>
inline int tile_launch_grid(int g0, const TilesDev& T, int override_grid) {
  if constexpr (idx_wsell(IDX)) {
    (void)override_grid;
    return (int)T.ws_G;
  } else {
    int g = override_grid ? override_grid : (g0 > (int)T.ntiles ? (int)T.ntiles : g0);
    return g < 1 ? 1 : g;
  }
}

template <int PA>
cudaError_t launch_spmv_dots_t(int pz, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* z, void* V,
                               uint64_t ld, int j, LevelState* L, GateH gate, SyncH sync, double* dots, int defer,
                               int* grid_out, DistH dist) {
  cudaError_t err = cudaErrorInvalidValue;
  auto go = [&](auto IDX_) {
    constexpr int IDX = decltype(IDX_)::value;
    constexpr int SM = TileCfg<PA, IDX>::SMEM_BYTES;
    with_p(pw, [&](auto W) {
      constexpr int PW = decltype(W)::value;
      with_p(pz, [&](auto Z) {
        constexpr int PZ = decltype(Z)::value;
        if constexpr (PZ <= PW) {
          auto kern = k_spmv_dots<PA, PZ, PW, IDX>;
          static const int g0 = tile_kernel_grid(kern, SM, T.ntiles, false, tile_threads(IDX));
          int g = tile_launch_grid<IDX>(g0, T, l.grid);
          if (dist.mode == 2) g = 1;
          if (grid_out) *grid_out = g;
          launch_kt(kern, g, tile_threads(IDX), SM, l.stream, A, T, z, V, ld, j, L, to_gate(gate), to_sync(sync), dots, defer,
                                              to_dist(dist));
          err = cudaGetLastError();
        }
      });
    });
  };
  dispatch_idx<PA>(A, T, go);
  return err;
}

template <int PA>
cudaError_t launch_residual_t(int px, int pw, Launch l, const CsrDev& A, const TilesDev& T, const void* x,
                              const double* b, void* r, LevelState* L, double* out_norm, SyncH sync, DistH dist) {
  cudaError_t err = cudaErrorInvalidValue;
  auto go = [&](auto IDX_) {
    constexpr int IDX = decltype(IDX_)::value;
    constexpr int SM = TileCfg<PA, IDX>::SMEM_BYTES;
    with_p(px, [&](auto X) {
      constexpr int PX = decltype(X)::value;
      with_p(pw, [&](auto W) {
        constexpr int PW = decltype(W)::value;
        if constexpr (PW >= PX) {
          auto kern = k_residual<PA, PX, PW, IDX>;
          static const int g0 = tile_kernel_grid(kern, SM, T.ntiles, false, tile_threads(IDX));
          int g = tile_launch_grid<IDX>(g0, T, l.grid);
          if (dist.mode == 2) g = 1;
          launch_kt(kern, g, tile_threads(IDX), SM, l.stream, A, T, x, b, r, L, out_norm, to_sync(sync), to_dist(dist));
          err = cudaGetLastError();
        }
      });
    });
  };
  dispatch_idx<PA>(A, T, go);
  return err;
}

template <int PA>
cudaError_t launch_spmv_t(int px, int py, Launch l, const CsrDev& A, const TilesDev& T, const void* x, void* y) {
  cudaError_t err = cudaErrorInvalidValue;
  auto go = [&](auto IDX_) {
    constexpr int IDX = decltype(IDX_)::value;
    constexpr int SM = TileCfg<PA, IDX>::SMEM_BYTES;
    with_p(px, [&](auto X) {
      with_p(py, [&](auto Y) {
        auto kern = k_spmv<PA, decltype(X)::value, decltype(Y)::value, IDX>;
        static const int g0 = tile_kernel_grid(kern, SM, T.ntiles, false, tile_threads(IDX));
        const int g = tile_launch_grid<IDX>(g0, T, l.grid);
        launch_kt(kern, g, tile_threads(IDX), SM, l.stream, A, T, x, y);
        err = cudaGetLastError();
      });
    });
  };
  dispatch_idx<PA>(A, T, go);
  return err;
}

// cooperative: grid = co-resident capacity (grid barriers on update calls)
template <int PA>
cudaError_t launch_richardson_t(int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, const void* v,
                                const double* v_scale, void* out, uint64_t n, RichState* RS, GateH gate, int level,
                                unsigned long long* cnt, SyncH sync, unsigned* bar_count, unsigned* bar_gen,
                                const IoSlot* io, uint64_t voff, int flags) {
  cudaError_t err = cudaErrorInvalidValue;
  auto go = [&](auto IDX_) {
    constexpr int IDX = decltype(IDX_)::value;
    constexpr int SM = TileCfg<PA, IDX>::SMEM_BYTES;
    with_p(pv, [&](auto V) {
      constexpr int PV = decltype(V)::value;
      with_p(pw, [&](auto W) {
        constexpr int PW = decltype(W)::value;
        if constexpr (PW <= PV) {
          auto kern = k_richardson<PA, PW, PV, IDX>;
          static const int g0 = tile_kernel_grid(kern, SM, T.ntiles, false, tile_threads(IDX));
          const int g = idx_wsell(IDX) ? (int)T.ws_G : l.grid ? l.grid : g0;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(g);
          cfg.blockDim = dim3(tile_threads(IDX));
          cfg.dynamicSmemBytes = SM;
          cfg.stream = l.stream;
          cudaLaunchAttribute attr[1];
          attr[0].id = cudaLaunchAttributeCooperative;
          attr[0].val.cooperative = 1;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          err = cudaLaunchKernelEx(&cfg, kern, A, T, v, v_scale, out, n, RS, to_gate(gate), level, cnt, to_sync(sync),
                                   bar_count, bar_gen, io, voff, flags);
          if (err == cudaSuccess) err = cudaGetLastError();
        }
      });
    });
  };
  dispatch_idx<PA>(A, T, go);
  return err;
}

template <int PA>
cudaError_t launch_rich_phase_t(int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                                const void* v, const double* v_scale, uint64_t off, void* out, uint64_t n,
                                RichState* RS, void* R, void* Za, GateH gate, int level, unsigned long long* cnt,
                                SyncH sync, DistH dist) {
  cudaError_t err = cudaErrorInvalidValue;
  auto go = [&](auto IDX_) {
    constexpr int IDX = decltype(IDX_)::value;
    constexpr int SM = TileCfg<PA, IDX>::SMEM_BYTES;
    with_p(pv, [&](auto V) {
      constexpr int PV = decltype(V)::value;
      with_p(pw, [&](auto W) {
        constexpr int PW = decltype(W)::value;
        if constexpr (PW <= PV) {
          auto kern = k_rich_phase<PA, PW, PV, IDX>;
          static const int g0 = tile_kernel_grid(kern, SM, T.ntiles, false, tile_threads(IDX));
          int g = tile_launch_grid<IDX>(g0, T, l.grid);
          if (phase == PH_BOOK) g = 1;
          launch_kt(kern, g, tile_threads(IDX), SM, l.stream, A, T, phase, k, v, v_scale, off, out, n, RS, R, Za, to_gate(gate), level,
                                              cnt, to_sync(sync), to_dist(dist));
          err = cudaGetLastError();
        }
      });
    });
  };
  dispatch_idx<PA>(A, T, go);
  return err;
}

template <int PA>
cudaError_t launch_richm_phase_t(int pw, int pv, Launch l, const CsrDev& A, const TilesDev& T, int phase, int k,
                                 const void* v, const double* v_scale, void* out, uint64_t n, RichState* RS, void* R,
                                 void* P, void* Za, GateH gate, int level, unsigned long long* cnt, SyncH sync) {
  cudaError_t err = cudaErrorInvalidValue;
  auto go = [&](auto IDX_) {
    constexpr int IDX = decltype(IDX_)::value;
    constexpr int SM = TileCfg<PA, IDX>::SMEM_BYTES;
    with_p(pv, [&](auto V) {
      constexpr int PV = decltype(V)::value;
      with_p(pw, [&](auto W) {
        constexpr int PW = decltype(W)::value;
        if constexpr (PW <= PV) {
          auto kern = k_richm_phase<PA, PW, PV, IDX>;
          static const int g0 = tile_kernel_grid(kern, SM, T.ntiles, false, tile_threads(IDX));
          int g = tile_launch_grid<IDX>(g0, T, l.grid);
          if (phase == RM_BOOK) g = 1;
          launch_kt(kern, g, tile_threads(IDX), SM, l.stream, A, T, phase, k, v, v_scale, out, n, RS, R, P, Za, to_gate(gate), level, cnt,
                   to_sync(sync));
          err = cudaGetLastError();
        }
      });
    });
  };
  dispatch_idx<PA>(A, T, go);
  return err;
}

}  // namespace f3rg
