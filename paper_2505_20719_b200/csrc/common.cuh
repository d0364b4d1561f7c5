// common.cuh -- precision traits, bit-faithful arithmetic, sm_100a async-copy
// primitives and deterministic reductions shared by every f3rg kernel.
//
// Numeric contract (reference include/f3r/precision.hpp,
// include/f3r/half.hpp, src/vector_ops.cpp): an operation "at precision C"
// widens its operands exactly, performs ONE correctly rounded IEEE op at C and
// never contracts a*b+c into an FMA. We use the explicit _rn intrinsics
// (__dmul_rn/__dadd_rn, __fmul_rn/__fadd_rn, __hmul_rn/__hadd_rn), which nvcc
// never fuses, and additionally build with -fmad=false. binary16 division and
// square root go through binary32 and round once more -- exactly what the
// reference's software Half does (half.hpp:121-124,146), and equal to the
// correctly rounded binary16 result.
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

namespace f3rg {

enum : int { P16 = 0, P32 = 1, P64 = 2 };

template <int P> struct Prec;
template <> struct Prec<P16> { using T = __half; };
template <> struct Prec<P32> { using T = float; };
template <> struct Prec<P64> { using T = double; };
template <int P> using T_ = typename Prec<P>::T;

__host__ __device__ constexpr int pmax(int a, int b) { return a > b ? a : b; }

// ---- conversions (RNE, subnormals kept) -------------------------------------
template <int To> struct Cvt;
template <> struct Cvt<P64> {
  __device__ static double of(double x) { return x; }
  __device__ static double of(float x) { return (double)x; }
  __device__ static double of(__half x) { return (double)__half2float(x); }
};
template <> struct Cvt<P32> {
  __device__ static float of(double x) { return __double2float_rn(x); }
  __device__ static float of(float x) { return x; }
  __device__ static float of(__half x) { return __half2float(x); }
};
template <> struct Cvt<P16> {
  __device__ static __half of(double x) { return __double2half(x); }  // one rounding from binary64
  __device__ static __half of(float x) { return __float2half_rn(x); }
  __device__ static __half of(__half x) { return x; }
};
template <int To, class S>
__device__ __forceinline__ T_<To> cvt(S x) { return Cvt<To>::of(x); }

// ---- hypot as the reference's std::hypot computes it ------------------------------
// The Givens rotations call std::hypot at the basis precision (src/fgmres.cpp:105),
// i.e. glibc's hypot / hypotf on the x86-64 reference build. Both are restated here
// so the device rotations are bit-identical (checked against the host libm over
// 4e7 random pairs, every binade and sign; tests/test_gpu_seq.py):
//  * hypotf: the binary32 result of the binary64 expression sqrt(x*x + y*y) (both
//    squares exact, one rounding each for the sum, the sqrt and the narrowing);
//  * hypot (glibc >= 2.35, dbl-64/e_hypot.c without FMA): Borges' corrected kernel
//    ("An Improved Algorithm for hypot(a,b)", 2019) with range scaling by 2^600.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    const double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}
__device__ __forceinline__ double ref_hypot(double x, double y) {
  if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000ll);
  if (isnan(x) || isnan(y)) return x + y;
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return __ddiv_rn(hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
  }
  if (ay < kTiny) {
    if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
    return __dmul_rn(hypot_kernel(__ddiv_rn(ax, kScale), __ddiv_rn(ay, kScale)), kScale);
  }
  if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
  return hypot_kernel(ax, ay);
}
__device__ __forceinline__ float ref_hypotf(float x, float y) {
  if (isinf(x) || isinf(y)) return __int_as_float(0x7f800000);
  const double xd = x, yd = y;
  return __double2float_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(xd, xd), __dmul_rn(yd, yd))));
}

// ---- one rounded op at precision C --------------------------------------------
template <int C> struct Ar;
template <> struct Ar<P64> {
  using T = double;
  __device__ static T zero() { return 0.0; }
  __device__ static T one() { return 1.0; }
  __device__ static T mul(T a, T b) { return __dmul_rn(a, b); }
  __device__ static T add(T a, T b) { return __dadd_rn(a, b); }
  __device__ static T sub(T a, T b) { return __dsub_rn(a, b); }
  __device__ static T div(T a, T b) { return __ddiv_rn(a, b); }
  __device__ static T sqrt(T a) { return __dsqrt_rn(a); }
  __device__ static T hypot(T a, T b) { return ref_hypot(a, b); }
  __device__ static T neg(T a) { return -a; }
  __device__ static double wide(T a) { return a; }
  __device__ static bool finite(T a) { return isfinite(a); }
};
template <> struct Ar<P32> {
  using T = float;
  __device__ static T zero() { return 0.0f; }
  __device__ static T one() { return 1.0f; }
  __device__ static T mul(T a, T b) { return __fmul_rn(a, b); }
  __device__ static T add(T a, T b) { return __fadd_rn(a, b); }
  __device__ static T sub(T a, T b) { return __fsub_rn(a, b); }
  __device__ static T div(T a, T b) { return __fdiv_rn(a, b); }
  __device__ static T sqrt(T a) { return __fsqrt_rn(a); }
  __device__ static T hypot(T a, T b) { return ref_hypotf(a, b); }
  __device__ static T neg(T a) { return -a; }
  __device__ static double wide(T a) { return (double)a; }
  __device__ static bool finite(T a) { return isfinite(a); }
};
template <> struct Ar<P16> {
  using T = __half;
  __device__ static T zero() { return __ushort_as_half((unsigned short)0); }
  __device__ static T one() { return __ushort_as_half((unsigned short)0x3c00u); }
  __device__ static T mul(T a, T b) { return __hmul_rn(a, b); }
  __device__ static T add(T a, T b) { return __hadd_rn(a, b); }
  __device__ static T sub(T a, T b) { return __hsub_rn(a, b); }
  __device__ static T div(T a, T b) { return __float2half_rn(__fdiv_rn(__half2float(a), __half2float(b))); }
  __device__ static T sqrt(T a) { return __float2half_rn(__fsqrt_rn(__half2float(a))); }
  __device__ static T hypot(T a, T b) { return __float2half_rn(ref_hypotf(__half2float(a), __half2float(b))); }
  __device__ static T neg(T a) { return __hneg(a); }
  __device__ static double wide(T a) { return (double)__half2float(a); }
  __device__ static bool finite(T a) { return (__half_as_ushort(a) & 0x7c00u) != 0x7c00u; }
};

// reinterpret 16 bits as an fp16 value (P16 stream decode)
template <class T>
__device__ __forceinline__ T bits_as(unsigned short b) {
  return __ushort_as_half(b);
}

// generic typed load of element i of a precision-tagged array
template <int P>
__device__ __forceinline__ T_<P> ld(const void* p, uint64_t i) {
  return static_cast<const T_<P>*>(p)[i];
}
template <int P>
__device__ __forceinline__ T_<P> ldg(const void* p, uint64_t i) {
  if constexpr (P == P16) {
    return __ushort_as_half(__ldg(static_cast<const unsigned short*>(p) + i));
  } else {
    return __ldg(static_cast<const T_<P>*>(p) + i);
  }
}
// L2-coherent load (bypasses L1) for data written earlier in the SAME kernel
// (cooperative Richardson passes separated by grid barriers)
template <int P>
__device__ __forceinline__ T_<P> ldcg(const void* p, uint64_t i) {
  if constexpr (P == P16) {
    return __ushort_as_half(__ldcg(static_cast<const unsigned short*>(p) + i));
  } else {
    return __ldcg(static_cast<const T_<P>*>(p) + i);
  }
}
// L1-cached load of data written earlier in the same kernel, after a grid barrier
// (no SM holds a stale line of it: nothing reads it before the barrier)
template <int P>
__device__ __forceinline__ T_<P> ldca(const void* p, uint64_t i) {
  if constexpr (P == P16) {
    return __ushort_as_half(__ldca(static_cast<const unsigned short*>(p) + i));
  } else {
    return __ldca(static_cast<const T_<P>*>(p) + i);
  }
}
template <int P>
__device__ __forceinline__ void st(void* p, uint64_t i, T_<P> v) {
  static_cast<T_<P>*>(p)[i] = v;
}

// 8 consecutive elements (group g) of a precision-tagged array as 16-byte
// transactions (1, 2 or 4 of them); the array must be 16-byte aligned
constexpr int kGroup = 8;
template <int P>
__device__ __forceinline__ void ld8(const void* p, uint64_t g, T_<P> (&out)[kGroup]) {
  constexpr int NQ = kGroup * (int)sizeof(T_<P>) / 16;
  const uint4* q = reinterpret_cast<const uint4*>(p) + g * NQ;
  uint4 t[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) t[k] = q[k];
  memcpy(out, t, sizeof t);
}
template <int P>
__device__ __forceinline__ void st8(void* p, uint64_t g, const T_<P> (&v)[kGroup]) {
  constexpr int NQ = kGroup * (int)sizeof(T_<P>) / 16;
  uint4 t[NQ];
  memcpy(t, v, sizeof t);
  uint4* q = reinterpret_cast<uint4*>(p) + g * NQ;
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = t[k];
}
__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- programmatic dependent launch ------------------------------------------------
// pdl_wait(): returns once the preceding kernel has completed and its writes are
// visible (a no-op without a programmatic dependency). pdl_trigger(): this CTA no
// longer holds the successor back (it may launch once every CTA has triggered or
// exited); called after the main loops, before the reduction tails.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- sm_90+/sm_100a async bulk copy (TMA 1D) + mbarrier ------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier (src/dst 16B aligned, bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- L2 eviction priorities --------------------------------------------------------
// A pass streams the matrix once and gathers a vector many times over (config 5:
// a 40 MB fp16 x, ~37 reads of every element per pass). With the hints on, the
// stream is loaded evict-first and the gathers evict-last, so the vector stays in
// the 126 MB L2 instead of being pushed out by the stream (TilesDev::l2hint).
__device__ __forceinline__ uint64_t l2_policy(int kind) {  // 0 normal, 1 evict-first, 2 evict-last
  uint64_t p;
  if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// element i of a precision-tagged array with an L2 policy; CACHE: "nc" (read-only
// path), "cg" (L2 only) or "ca" (L1-allocating)
#define F3RG_LD_HINT(NAME, QUAL)                                                                              \
  template <int P>                                                                                            \
  __device__ __forceinline__ T_<P> NAME(const void* p, uint64_t i, uint64_t pol) {                            \
    if constexpr (P == P16) {                                                                                 \
      unsigned short v;                                                                                       \
      asm volatile("ld.global." QUAL ".L2::cache_hint.u16 %0, [%1], %2;"                                      \
                   : "=h"(v) : "l"(static_cast<const unsigned short*>(p) + i), "l"(pol));                      \
      return __ushort_as_half(v);                                                                             \
    } else if constexpr (P == P32) {                                                                          \
      float v;                                                                                                \
      asm volatile("ld.global." QUAL ".L2::cache_hint.f32 %0, [%1], %2;"                                      \
                   : "=f"(v) : "l"(static_cast<const float*>(p) + i), "l"(pol));                              \
      return v;                                                                                               \
    } else {                                                                                                  \
      double v;                                                                                               \
      asm volatile("ld.global." QUAL ".L2::cache_hint.f64 %0, [%1], %2;"                                      \
                   : "=d"(v) : "l"(static_cast<const double*>(p) + i), "l"(pol));                             \
      return v;                                                                                               \
    }                                                                                                         \
  }
F3RG_LD_HINT(ldg_hint, "nc")
F3RG_LD_HINT(ldcg_hint, "cg")
F3RG_LD_HINT(ldca_hint, "ca")
#undef F3RG_LD_HINT

// ---- deterministic reductions ----------------------------------------------------
// Fixed-shape trees: the result depends only on the inputs' positions, never on
// scheduling, so repeated solves are bitwise identical (reference
// tests/test_nesting.cpp:152-165 pins determinism).
template <int C>
__device__ __forceinline__ T_<C> warp_sum(T_<C> v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T_<C> w;
    if constexpr (C == P16) {
      w = __ushort_as_half(__shfl_xor_sync(0xffffffffu, __half_as_ushort(v), o));
    } else {
      w = __shfl_xor_sync(0xffffffffu, v, o);
    }
    v = Ar<C>::add(v, w);
  }
  return v;
}

// Block-wide sums of NV values per thread. Result valid in thread 0.
// scratch: >= (blockDim/32) * NV doubles.
template <int C, int NV>
__device__ __forceinline__ void block_sum(T_<C> (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum<C>(v[k]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[k * nw + wid] = Ar<C>::wide(v[k]);
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      T_<C> t = lane < nw ? cvt<C>(scratch[k * nw + lane]) : Ar<C>::zero();
      v[k] = warp_sum<C>(t);
    }
  }
  __syncthreads();
}

// "last block done": every block publishes its partials, the block that arrives
// last returns true (and re-arms the counter for the next launch).
__device__ __forceinline__ bool last_block(unsigned* counter) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    // only thread 0 published data for the last CTA (the block's partials), so
    // only its stores need ordering before the count (a fence by every thread
    // waits out all their outputs: measured as membar stalls in k_cgs)
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    is_last = (t == gridDim.x - 1);
    if (is_last) *counter = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Light variant for bookkeeping that publishes no data between CTAs: one atomic per
// CTA after the CTA's work, no fences; the last CTA to arrive returns true.
__device__ __forceinline__ bool last_block_light(unsigned* counter) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    if (is_last) *counter = 0u;
  }
  __syncthreads();
  return is_last;
}

// Reduce partials[G][stride] columns 0..NV-1 over G blocks in a fixed tree;
// called by one whole block; results (doubles holding C values) in out[] (shared),
// valid for all threads after the call.
template <int C, int NV>
__device__ void reduce_partials(const double* partials, int G, int stride, double* out, double* scratch) {
  T_<C> acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = Ar<C>::zero();
  for (int b = threadIdx.x; b < G; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = Ar<C>::add(acc[k], cvt<C>(__ldcg(partials + (size_t)b * stride + k)));
  }
  block_sum<C, NV>(acc, scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) out[k] = Ar<C>::wide(acc[k]);
  }
  __syncthreads();
}

// ---- sequential reductions (validation mode) --------------------------------------
// The reference sums every dot and norm on one thread in index order (dot_core,
// src/vector_ops.cpp:20-28): acc = fl_C(acc + fl_C(x_i * y_i)), i = 0 .. n-1. With
// sequential reductions on (F3RG_SEQ_REDUCTIONS=1 / f3rg_set_seq_reductions) the
// CTA that completes a reduction recomputes it in exactly that order from the
// operands in memory and replaces the tree result -- slow (one dependent add per
// element), bit-identical to the reference. It exists to validate parity on long
// vectors, where the two orders part.
template <int C>
__device__ __forceinline__ T_<C> shfl_idx(T_<C> v, int src) {
  if constexpr (C == P16) {
    return __ushort_as_half(__shfl_sync(0xffffffffu, __half_as_ushort(v), src));
  } else {
    return __shfl_sync(0xffffffffu, v, src);
  }
}

// One warp: the sequential sum of term(i), i < n. Lanes fetch and form the terms of
// 256 consecutive elements (the next batch's loads are in flight while the current
// one is summed); every lane then carries the same dependent chain, so the result
// is valid in all lanes. Terms past n are skipped, never added as zeros (-0 + +0 = +0).
template <int C, class F>
__device__ __forceinline__ T_<C> warp_seq_sum(uint64_t n, const F& term) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  T_<C> acc = Ar<C>::zero();
  T_<C> cur[U], nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = (uint64_t)u * 32 + lane;
    cur[u] = i < n ? term(i) : Ar<C>::zero();
  }
  for (uint64_t base = 0; base < n; base += 32 * U) {
    const uint64_t nb = base + 32 * U;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = nb + (uint64_t)u * 32 + lane;
      nxt[u] = i < n ? term(i) : Ar<C>::zero();
    }
    const uint64_t lim = n - base;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        const T_<C> t = shfl_idx<C>(cur[u], s);
        if ((uint64_t)(u * 32 + s) < lim) acc = Ar<C>::add(acc, t);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  return acc;
}

// nv <= 8 sequential sums by one whole CTA (warp k runs sum k); term(i, k) is the
// k-th sum's term at element i. out[k] (shared, doubles holding C values) is valid
// for all threads after the call.
template <int C, class F>
__device__ void seq_sums(uint64_t n, int nv, const F& term, double* out) {
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if (w < nv) {
    const T_<C> s = warp_seq_sum<C>(n, [&](uint64_t i) { return term(i, w); });
    if ((threadIdx.x & 31) == 0) out[w] = Ar<C>::wide(s);
  }
  __syncthreads();
}

// Software grid barrier for cooperative launches (all blocks co-resident).
__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0u;
      __threadfence();
      atomicAdd((unsigned*)gen, 1u);
    } else {
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace f3rg
