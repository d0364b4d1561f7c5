// launch_krylov.cu -- launchers of the fp64 CG / BiCGStab kernels (krylov.cuh).
#include "dispatch.cuh"
#include "krylov.cuh"
#include "launch.hpp"

namespace f3rg {

template <class F>
static void with_idx64(const CsrDev& A, const TilesDev& T, F&& go) {
  if (T.shape == 3) {
    go(PC<16>{});
  } else if (T.shape == 1) {
    if (A.dcol) go(PC<5>{});
    else go(PC<4>{});
  } else if (T.shape == 2) {
    if (A.dcol) go(PC<9>{});
    else go(PC<8>{});
  } else {
    if (A.dcol) go(PC<1>{});
    else go(PC<0>{});
  }
}

// persistent grid: co-resident CTAs (occ, cached by the caller per kernel
// instantiation), capped by the tile count
static int tile_grid(int occ, uint32_t ntiles) {
  long g = (long)occ * sm_count();
  if (g > (long)ntiles) g = ntiles;
  return g < 1 ? 1 : (int)g;
}
// the windowed engine runs exactly the CTA count its windows were split over
template <int IDX>
static int krylov_grid(int occ, const TilesDev& T) {
  return idx_wsell(IDX) ? (int)T.ws_G : tile_grid(occ, T.ntiles);
}

cudaError_t launch_cg_spmv(Launch l, const CsrDev& A, const TilesDev& T, const double* p, double* q, KState* S,
                           SyncH sync) {
  cudaError_t err = cudaSuccess;
  with_idx64(A, T, [&](auto I) {
    constexpr int IDX = decltype(I)::value;
    constexpr int SM = TileCfg<P64, IDX>::SMEM_BYTES;
    auto kern = k_cg_spmv<IDX>;
    static const int occ = occupancy_blocks(kern, SM, tile_threads(IDX));  // also sets the dynamic smem limit
    err = launch_kt(kern, krylov_grid<IDX>(occ, T), tile_threads(IDX), SM, l.stream, A, T, p, q, S, to_sync(sync));
  });
  return err;
}

cudaError_t launch_cg_update(Launch l, double* x, double* r, const double* p, const double* q, uint64_t n, KState* S,
                             SyncH sync) {
  return launch_k(k_cg_update, red_grid(), 0, l.stream, x, r, p, q, n, S, to_sync(sync));
}

cudaError_t launch_cg_next(Launch l, KState* S) { return launch_k1(k_cg_next, l.stream, S); }

cudaError_t launch_cg_rz(Launch l, const double* r, const double* z, uint64_t n, KState* S, SyncH sync) {
  return launch_k(k_cg_rz, red_grid(), 0, l.stream, r, z, n, S, to_sync(sync));
}

cudaError_t launch_cg_p(Launch l, double* p, const double* r, uint64_t n, const KState* S) {
  return launch_k(k_cg_p, stream_grid(), 0, l.stream, p, r, n, S);
}

cudaError_t launch_bi_rho(Launch l, const double* rhat, const double* r, uint64_t n, KState* S, SyncH sync) {
  return launch_k(k_bi_rho, red_grid(), 0, l.stream, rhat, r, n, S, to_sync(sync));
}

cudaError_t launch_bi_p(Launch l, double* p, const double* v, const double* r, uint64_t n, const KState* S) {
  return launch_k(k_bi_p, stream_grid(), 0, l.stream, p, v, r, n, S);
}

cudaError_t launch_bi_v(Launch l, const CsrDev& A, const TilesDev& T, const double* p, double* v, const double* rhat,
                        KState* S, SyncH sync) {
  cudaError_t err = cudaSuccess;
  with_idx64(A, T, [&](auto I) {
    constexpr int IDX = decltype(I)::value;
    constexpr int SM = TileCfg<P64, IDX>::SMEM_BYTES;
    auto kern = k_bi_v<IDX>;
    static const int occ = occupancy_blocks(kern, SM, tile_threads(IDX));  // also sets the dynamic smem limit
    err = launch_kt(kern, krylov_grid<IDX>(occ, T), tile_threads(IDX), SM, l.stream, A, T, p, v, rhat, S, to_sync(sync));
  });
  return err;
}

cudaError_t launch_bi_s(Launch l, double* s, const double* r, const double* v, uint64_t n, const KState* S) {
  return launch_k(k_bi_s, stream_grid(), 0, l.stream, s, r, v, n, S);
}

cudaError_t launch_bi_t(Launch l, const CsrDev& A, const TilesDev& T, const double* s, const double* shat, double* t,
                        KState* S, SyncH sync) {
  cudaError_t err = cudaSuccess;
  with_idx64(A, T, [&](auto I) {
    constexpr int IDX = decltype(I)::value;
    constexpr int SM = TileCfg<P64, IDX>::SMEM_BYTES;
    auto kern = k_bi_t<IDX>;
    static const int occ = occupancy_blocks(kern, SM, tile_threads(IDX));  // also sets the dynamic smem limit
    err = launch_kt(kern, krylov_grid<IDX>(occ, T), tile_threads(IDX), SM, l.stream, A, T, s, shat, t, S, to_sync(sync));
  });
  return err;
}

cudaError_t launch_bi_update(Launch l, double* x, double* r, const double* p, const double* s, const double* shat,
                             const double* t, uint64_t n, KState* S, SyncH sync) {
  return launch_k(k_bi_update, red_grid(), 0, l.stream, x, r, p, s, shat, t, n, S, to_sync(sync));
}

cudaError_t launch_krylov_resume(Launch l, KState* S) { return launch_k1(k_krylov_resume, l.stream, S); }

}  // namespace f3rg
