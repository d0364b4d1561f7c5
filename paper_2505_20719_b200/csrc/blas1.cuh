// blas1.cuh -- precision-generic BLAS-1 kernels mirroring src/vector_ops.cpp
// (fill :77, copy_into :87, scale_in_place :104, axpy :114, add_scaled :131,
// dot/dot_at_least :150-164, norm2 :166). Element-wise ops follow the reference's
// per-element rounding sequence exactly; reductions use a fixed-shape tree
// (deterministic, order differs from the reference's sequential sum).
#pragma once

#include "common.cuh"
#include "levels.cuh"

namespace f3rg {

template <int P>
__global__ void __launch_bounds__(256) k_fill(void* x, uint64_t n, double value) {
  pdl_wait();
  const T_<P> v = cvt<P>(value);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) st<P>(x, i, v);
}

template <int PX, int PY>
__global__ void __launch_bounds__(256) k_copy(const void* x, void* y, uint64_t n) {
  pdl_wait();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    st<PY>(y, i, cvt<PY>(ld<PX>(x, i)));
}

template <int P>
__global__ void __launch_bounds__(256) k_scale(double alpha, void* x, uint64_t n) {
  pdl_wait();
  const T_<P> a = cvt<P>(alpha);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    st<P>(x, i, Ar<P>::mul(a, ld<P>(x, i)));
}

// y = fl_C(fl_C(a * x) + y), C = promote(x, y)
template <int PX, int PY>
__global__ void __launch_bounds__(256) k_axpy(double alpha, const void* x, void* y, uint64_t n) {
  pdl_wait();
  constexpr int C = pmax(PX, PY);
  const T_<C> a = cvt<C>(alpha);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    st<PY>(y, i, cvt<PY>(Ar<C>::add(Ar<C>::mul(a, cvt<C>(ld<PX>(x, i))), cvt<C>(ld<PY>(y, i)))));
}

// out = fl_C(x + fl_C(a * y)), C = promote(x, y, out)
template <int PX, int PY, int PO>
__global__ void __launch_bounds__(256) k_add_scaled(const void* x, double alpha, const void* y, void* out,
                                                    uint64_t n) {
  pdl_wait();
  constexpr int C = pmax(pmax(PX, PY), PO);
  const T_<C> a = cvt<C>(alpha);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    st<PO>(out, i, cvt<PO>(Ar<C>::add(cvt<C>(ld<PX>(x, i)), Ar<C>::mul(a, cvt<C>(ld<PY>(y, i))))));
}

// dot at C = max(floor, px, py); result (a C value) in *out; if SQRT, sqrt at
// precision PS of the C value rounded to PS (norm2 semantics).
template <int PX, int PY, int C, bool SQRT, int PS>
__global__ void __launch_bounds__(256) k_dot(const void* x, const void* y, uint64_t n, double* out, Sync sync,
                                             Dist dist) {
  pdl_wait();
  __shared__ double scratch[64];
  __shared__ double tot[1];
  if (dist.mode != 2) {
    T_<C> acc[1] = {Ar<C>::zero()};
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      acc[0] = Ar<C>::add(acc[0], Ar<C>::mul(cvt<C>(ld<PX>(x, i)), cvt<C>(ld<PY>(y, i))));
    pdl_trigger();
    block_sum<C, 1>(acc, scratch);
    if (threadIdx.x == 0) sync.partials[(size_t)blockIdx.x * kMaxPart] = Ar<C>::wide(acc[0]);
    if (!last_block(sync.counter)) return;
    if (sync.seq) {
      seq_sums<C>(n, 1, [&](uint64_t i, int) { return Ar<C>::mul(cvt<C>(ld<PX>(x, i)), cvt<C>(ld<PY>(y, i))); }, tot);
    } else {
      reduce_partials<C, 1>(sync.partials, gridDim.x, kMaxPart, tot, scratch);
    }
    if (publish_local(dist, 1, tot)) return;
  } else {
    combine_ranks<C>(dist, 1, tot);
  }
  if (threadIdx.x == 0) {
    if constexpr (SQRT) {
      *out = Ar<PS>::wide(Ar<PS>::sqrt(cvt<PS>(tot[0])));
    } else {
      *out = tot[0];
    }
  }
}

// halo exchange helper (row-block partition): dst[i] = src[idx[i]], element-wise
// copies at one precision (pack for a send, or a direct gather from a peer's
// owned rows when the peers share an address space)
template <int P>
__global__ void __launch_bounds__(256) k_gather(const void* src, const uint32_t* idx, uint64_t cnt, void* dst) {
  pdl_wait();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride)
    st<P>(dst, i, ld<P>(src, idx[i]));
}

// P16 stream: fp16 value bits | D16 delta << 16, one word per entry
static __global__ void __launch_bounds__(256) k_pack16(const __half* v, const uint16_t* d, uint32_t* out, uint64_t nnz) {
  pdl_wait();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride)
    out[i] = (uint32_t)__half_as_ushort(v[i]) | ((uint32_t)d[i] << 16);
}

// plain y = A x (any precision triple), for the kernel-level entry point
template <int PA, int PX, int PY, int IDX>
__global__ void __launch_bounds__(tile_threads(IDX), tile_minb(IDX)) k_spmv(CsrDev A, TilesDev T, const void* x, void* y) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int C = pmax(PA, PX);
  GatherPlain<PX, C> g{x};
  EpiStore<C, PY> e{y};
  spmv_tiles<PA, C, IDX>(A, T, g, e, smem);
}

}  // namespace f3rg
