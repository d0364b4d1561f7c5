// launch_blas.cu -- launchers for the precision-generic BLAS-1 / SpMV kernels (blas1.cuh).
#include "blas1.cuh"
#include "dispatch.cuh"

namespace f3rg {

cudaError_t launch_fill(int p, Launch l, void* x, uint64_t n, double value) {
  const int g = l.grid ? l.grid : stream_grid();
  with_p(p, [&](auto P) { launch_k(k_fill<decltype(P)::value>, g, 0, l.stream, x, n, value); });
  return cudaGetLastError();
}

cudaError_t launch_copy(int px, int py, Launch l, const void* x, void* y, uint64_t n) {
  const int g = l.grid ? l.grid : stream_grid();
  with_p(px, [&](auto X) {
    with_p(py, [&](auto Y) { launch_k(k_copy<decltype(X)::value, decltype(Y)::value>, g, 0, l.stream, x, y, n); });
  });
  return cudaGetLastError();
}

cudaError_t launch_scale(int p, Launch l, double alpha, void* x, uint64_t n) {
  const int g = l.grid ? l.grid : stream_grid();
  with_p(p, [&](auto P) { launch_k(k_scale<decltype(P)::value>, g, 0, l.stream, alpha, x, n); });
  return cudaGetLastError();
}

cudaError_t launch_axpy(int px, int py, Launch l, double alpha, const void* x, void* y, uint64_t n) {
  const int g = l.grid ? l.grid : stream_grid();
  with_p(px, [&](auto X) {
    with_p(py, [&](auto Y) {
      launch_k(k_axpy<decltype(X)::value, decltype(Y)::value>, g, 0, l.stream, alpha, x, y, n);
    });
  });
  return cudaGetLastError();
}

cudaError_t launch_add_scaled(int px, int py, int po, Launch l, const void* x, double alpha, const void* y, void* out,
                              uint64_t n) {
  const int g = l.grid ? l.grid : stream_grid();
  with_p(px, [&](auto X) {
    with_p(py, [&](auto Y) {
      with_p(po, [&](auto O) {
        launch_k(k_add_scaled<decltype(X)::value, decltype(Y)::value, decltype(O)::value>, g, 0, l.stream, x, alpha, y, out, n);
      });
    });
  });
  return cudaGetLastError();
}

cudaError_t launch_dot(int px, int py, int floor_p, Launch l, const void* x, const void* y, uint64_t n, double* out,
                       SyncH sync, DistH dist) {
  const int g = dist.mode == 2 ? 1 : l.grid ? l.grid : stream_grid();
  const int c = floor_p > px ? (floor_p > py ? floor_p : py) : (px > py ? px : py);
  with_p(px, [&](auto X) {
    with_p(py, [&](auto Y) {
      with_p(c, [&](auto C) {
        constexpr int CX = decltype(C)::value, PX = decltype(X)::value, PY = decltype(Y)::value;
        if constexpr (CX >= PX && CX >= PY)
          launch_k(k_dot<PX, PY, CX, false, CX>, g, 0, l.stream, x, y, n, out, to_sync(sync), to_dist(dist));
      });
    });
  });
  return cudaGetLastError();
}

cudaError_t launch_norm2(int px, Launch l, const void* x, uint64_t n, double* out, SyncH sync, DistH dist) {
  const int g = dist.mode == 2 ? 1 : l.grid ? l.grid : stream_grid();
  with_p(px, [&](auto X) {
    constexpr int PX = decltype(X)::value;
    launch_k(k_dot<PX, PX, PX, true, PX>, g, 0, l.stream, x, x, n, out, to_sync(sync), to_dist(dist));
  });
  return cudaGetLastError();
}

cudaError_t launch_gather(int p, Launch l, const void* src, const uint32_t* idx, uint64_t cnt, void* dst) {
  if (cnt == 0) return cudaSuccess;
  const uint64_t want = (cnt + kThreads - 1) / kThreads;
  const int g = l.grid ? l.grid : (int)(want < (uint64_t)stream_grid() ? want : (uint64_t)stream_grid());
  with_p(p, [&](auto P) { launch_k(k_gather<decltype(P)::value>, g, 0, l.stream, src, idx, cnt, dst); });
  return cudaGetLastError();
}

cudaError_t launch_pack16(Launch l, const void* val16, const uint16_t* dcol, uint32_t* out, uint64_t nnz) {
  if (nnz == 0) return cudaSuccess;
  const int g = l.grid ? l.grid : stream_grid();
  return launch_k(k_pack16, g, 0, l.stream, static_cast<const __half*>(val16), dcol, out, nnz);
}

}  // namespace f3rg
