// wsell.cuh -- windowed SELL-32 SpMV engine for gather-bound matrices (config 5:
// n = 2e7 unstructured rows whose columns scatter +-15,000 around the diagonal plus
// 5 % uniform long-range entries).
//
// Why: with one thread per row and the gathered vector read through L1 (the tile
// engine, spmv.cuh), every entry of such a matrix is its own 128-byte line request;
// the L1 tag stage serves about one line per clock per SM, which is exactly the
// 2 ms the config-5 fp16 pass took (4.1 M lines per SM at 1.965 GHz). Here the
// gathered vector lives in shared memory instead: each persistent CTA (one per SM,
// 1024 threads) owns a contiguous run of rows and keeps the band of x those rows
// can touch in a 128 KB ring, slid forward window by window with plain loads issued
// one window ahead. Gathers inside the band are shared-memory loads; the rest (the
// long-range 5 %) go to L2 with an evict-last policy. Which of the two an entry is
// gets decided once, when the matrix is uploaded (the encoded column stream below).
// The fp16-matrix passes with 2-byte operands run the same engine over a packed
// 4-byte stream: wsell_pk.cuh.
//
// Layout (host: engine.cpp build_wsell; device arrays in TilesDev ws_*):
//  * sort windows of kWsSort = 2048 consecutive rows; inside a window the rows are
//    ordered by length (descending, stable) and cut into 64 slices of 32 rows;
//  * a slice stores its entries chunk-major: chunk q (entries 4q..4q+3 of every
//    lane's row) is 32 lanes x 4 entries, so lane l reads one 16-byte column quad
//    and one 8/16/32-byte value quad per chunk, fully coalesced across the warp;
//    a slice is as wide as its longest row rounded up to 4;
//  * per ring width (state.hpp ws_rn/ws_tw/ws_w) the columns are ENCODED on the
//    device at upload (launch_setup.cu k_ws_encode): the byte offset of the ring slot
//    for an entry inside its window's band, the offset of a slot that holds zero for
//    padding (the padded value is +0 too, and a row accumulator is never -0, so the
//    +-0 product leaves it unchanged), the column with bit 31 set for the rest;
//  * ws_row maps slice lane -> matrix row; ws_cwin splits the windows over the
//    CTAs by stored entries.
// Each row is still summed by one thread in stored column order at
// C = promote(TA, TX), each product and sum rounded to C (src/csr.cpp:23-37), so
// results are bit-identical to the tile engine and to the reference.
//
// Per kernel window of TW rows (TW = a multiple of kWsSort, set by the ring element
// size): warps claim slices in descending-length order (longest processing time
// first, so the window's tail is one short slice), write each row's sum into a
// shared-memory buffer at the row's position, then, after one CTA barrier, the
// epilogue runs over the window's rows in natural order (coalesced row-local
// operands). Ring invariant for the window at rows [B, B+TW): the ring holds
// x[B-W, B+2TW+W) (RN = 2TW + 2W elements): the gathers' band [B-W, B+TW+W) plus
// the top block of the next window's band; the block after that is loaded into
// registers at the window's start and stored after its barrier into the slots the
// window just freed.
#pragma once

#include <type_traits>
#include <utility>

#include "common.cuh"
#include "state.hpp"

namespace f3rg {

constexpr int kWsThreads = 1024;
constexpr int kWsSort = (int)kWsSortRows;   // rows per sort window (layout unit)
constexpr int kWsSlices = kWsSort / 32;     // slices per sort window
constexpr int kWsRingBytes = 128 * 1024;    // the x band
constexpr int kWsYBytes = 64 * 1024;        // two row-sum buffers
constexpr int kWsSmem = kWsRingBytes + kWsYBytes + 64;
constexpr uint32_t kWsPad = kWsPadIdx;
constexpr uint32_t kWsZeroOff = kWsZeroOffset;  // byte offset of the zero slot (after the claim counters)
static_assert(kWsZeroOffset == kWsRingBytes + kWsYBytes + 32, "zero slot offset (state.hpp)");
#ifndef F3RG_WS_U  // column/value quads per lane per pipeline step
#define F3RG_WS_U 2
#endif

// What the ring stores for a gather: its raw load, or (gathers with a per-element
// transform, e.g. Richardson's z1 = w0 * v) the transformed value, so the transform
// runs once per ring element instead of once per gathered entry.
template <class G, class = void>
struct WsRing {
  using R = typename G::Raw;
  __device__ __forceinline__ static R put(const G&, typename G::Raw r) { return r; }
  __device__ __forceinline__ static auto get(const G& g, R r) { return g.value(r); }
};
template <class G>
struct WsRing<G, std::void_t<typename G::RingT>> {
  using R = typename G::RingT;
  __device__ __forceinline__ static R put(const G& g, typename G::Raw r) { return g.ring_put(r); }
  __device__ __forceinline__ static auto get(const G& g, R r) { return g.ring_get(r); }
};

// L2 policy of the engine's vector loads (ring fills, far gathers): the gather's own
// set_policy, or set_ring_policy where the tile engine's gathers take none
// (Richardson's GatherZ1 / GatherRhs read the parent's v)
template <class G, class = void>
struct WsPolicy {
  __device__ __forceinline__ static void set(G& g, uint64_t p) { g.set_policy(p); }
};
template <class G>
struct WsPolicy<G, std::void_t<decltype(std::declval<G&>().set_ring_policy(0ull))>> {
  __device__ __forceinline__ static void set(G& g, uint64_t p) { g.set_ring_policy(p); }
};

// streamed loads: read once, do not allocate in L1, L2 policy from the caller
__device__ __forceinline__ uint4 ws_ld16(const void* p, uint64_t pol) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint2 ws_ld8(const void* p, uint64_t pol) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}

// one lane's 4 values of a chunk
template <int PA>
struct WsVals;
template <>
struct WsVals<P16> {
  uint2 q;
  __device__ __forceinline__ void load(const void* base, uint64_t quad, uint64_t pol) {
    q = ws_ld8(static_cast<const uint2*>(base) + quad, pol);
  }
  __device__ __forceinline__ void zero() { q = make_uint2(0u, 0u); }
  __device__ __forceinline__ __half at(int e) const {
    const uint32_t w = e < 2 ? q.x : q.y;
    return __ushort_as_half((unsigned short)((e & 1) ? (w >> 16) : (w & 0xffffu)));
  }
};
template <>
struct WsVals<P32> {
  uint4 q;
  __device__ __forceinline__ void load(const void* base, uint64_t quad, uint64_t pol) {
    q = ws_ld16(static_cast<const uint4*>(base) + quad, pol);
  }
  __device__ __forceinline__ void zero() { q = make_uint4(0u, 0u, 0u, 0u); }
  __device__ __forceinline__ float at(int e) const {
    return __uint_as_float(e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w);
  }
};
template <>
struct WsVals<P64> {
  uint4 a, b;
  __device__ __forceinline__ void load(const void* base, uint64_t quad, uint64_t pol) {
    a = ws_ld16(static_cast<const uint4*>(base) + 2 * quad, pol);
    b = ws_ld16(static_cast<const uint4*>(base) + 2 * quad + 1, pol);
  }
  __device__ __forceinline__ void zero() { a = b = make_uint4(0u, 0u, 0u, 0u); }
  __device__ __forceinline__ double at(int e) const {
    const uint4& h = e < 2 ? a : b;
    return (e & 1) ? __hiloint2double((int)h.w, (int)h.z) : __hiloint2double((int)h.y, (int)h.x);
  }
};
__device__ __forceinline__ uint32_t quad_at(const uint4& q, int e) {
  return e == 0 ? q.x : e == 1 ? q.y : e == 2 ? q.z : q.w;
}

// Streams this CTA's windows; calls e.prefetch(i); e.row(i, acc) for every row i in
// natural order, acc at C. Launch: gridDim.x == T.ws_G, blockDim.x == kWsThreads,
// kWsSmem bytes of dynamic shared memory. Square matrices on one rank only (x has
// n elements).
template <int PA, int C, class G, class Epi>
__device__ __forceinline__ void wsell_pass(const CsrDev& A, const TilesDev& T, G& g, Epi& e, uint8_t* smem) {
  using RT = WsRing<G>;
  using R = typename RT::R;
  using Raw = typename G::Raw;
  using TA = T_<PA>;
  constexpr int RS = (int)sizeof(R);
  constexpr int RN = kWsRingBytes / RS;  // ring elements (power of two)
  constexpr int CS = (int)sizeof(T_<C>);
  constexpr int CL = RS == 2 ? 0 : RS == 4 ? 1 : 2;  // ring class (state.hpp): fixes the window geometry
  static_assert(RN == ws_rn(CL), "ring size");
  constexpr int TW = ws_tw(CL);     // rows per kernel window
  constexpr int KW = TW / kWsSort;  // sort windows per kernel window
  constexpr int W = ws_w(CL);
  constexpr int PF = TW / kWsThreads;  // ring elements each thread carries one window ahead
  constexpr int U = PA == P64 ? 1 : F3RG_WS_U;
  // two row-sum buffers (the next window's sums land while this one's epilogue runs),
  // or one and a second barrier per window when the accumulator is too wide for two
  constexpr bool YDBL = 2 * TW * CS <= kWsYBytes;
  static_assert(TW % kWsSort == 0 && W > 0 && PF >= 1 && (RN & (RN - 1)) == 0, "window geometry");
  static_assert(TW * CS <= kWsYBytes, "row-sum buffer");
  // the column stream of this ring class, encoded on the host side of the layout
  // (launch_setup.cu k_ws_encode): an entry inside its window's band is the byte
  // offset of its ring slot, a padding entry the offset of a slot that holds zero
  // (its value is +0 too; a row accumulator is never -0, so the +-0 product leaves
  // it unchanged), any other ("far") entry its column with bit 31 set
  const uint32_t* __restrict__ enc = T.ws_enc[CL];

  R* ring = reinterpret_cast<R*>(smem);
  T_<C>* ybuf = reinterpret_cast<T_<C>*>(smem + kWsRingBytes);
  unsigned* claim = reinterpret_cast<unsigned*>(smem + kWsRingBytes + kWsYBytes);
  WsPolicy<G>::set(g, l2_policy(T.l2hint ? 2 : 0));       // ring fills and far gathers: keep x in L2
  const uint64_t spol = l2_policy(T.l2hint ? 1 : 0);     // the matrix stream
  const int64_t n = (int64_t)A.n;
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  const uint32_t sw0 = T.ws_cwin[blockIdx.x], sw1 = T.ws_cwin[blockIdx.x + 1];
  const TA* __restrict__ vals = static_cast<const TA*>(T.ws_val);
  (void)vals;

  __syncthreads();  // a previous pass in the same kernel is done with the ring
  if (tid < 2) claim[tid] = 0u;
  if (tid < 2) reinterpret_cast<uint32_t*>(smem + kWsZeroOff)[tid] = 0u;  // the zero slot
  if (sw0 < sw1) {  // ring for the first window: x[B0-W, B0+2TW+W)
    const int64_t B0 = (int64_t)sw0 * kWsSort;
    int64_t i0 = B0 - W;
    if (i0 < 0) i0 = 0;
    int64_t i1 = B0 + 2 * TW + W;
    if (i1 > n) i1 = n;
    for (int64_t i = i0 + tid; i < i1; i += kWsThreads) ring[i & (RN - 1)] = RT::put(g, g.load((uint32_t)i));
  }
  __syncthreads();

  uint32_t it = 0;
  for (uint32_t sw = sw0; sw < sw1; sw += KW, ++it) {
    const int64_t B = (int64_t)sw * kWsSort;
    const uint32_t kw = (sw1 - sw) < (uint32_t)KW ? (sw1 - sw) : (uint32_t)KW;
    // the ring block two windows ahead, into registers now, into the ring after the barrier
    const int64_t pb = B + 2 * TW + W;
    Raw pf[PF];
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int64_t i = pb + (int64_t)q * kWsThreads + tid;
      if (i < n) pf[q] = g.load((uint32_t)i);
    }
    T_<C>* yb = ybuf + (YDBL ? (it & 1u) * TW : 0u);
    const uint32_t nsl = kw * (uint32_t)kWsSlices;
    unsigned* cl = &claim[it & 1u];
    for (;;) {
      uint32_t j = 0;
      if (lane == 0) j = atomicAdd(cl, 1u);
      j = __shfl_sync(0xffffffffu, j, 0);
      if (j >= nsl) break;
      // claim order: slice rank j / kw of sort window j % kw -- descending length
      const uint32_t s = (sw + j % kw) * (uint32_t)kWsSlices + j / kw;
      const uint32_t e0 = __ldg(T.ws_soff + s), e1 = __ldg(T.ws_soff + s + 1);
      const uint32_t row = __ldg(T.ws_row + (size_t)s * 32 + lane);
      const uint32_t nq = (e1 - e0) >> 7;  // chunks: 32 lanes x 4 entries
      const uint64_t qb = (uint64_t)(e0 >> 2) + lane;  // this lane's quad of chunk 0
      T_<C> acc = Ar<C>::zero();
      uint4 cc[U], cn[U];
      WsVals<PA> vc[U], vn[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if ((uint32_t)u < nq) {
          cc[u] = ws_ld16(reinterpret_cast<const uint4*>(enc) + qb + (uint64_t)u * 32, spol);
          vc[u].load(T.ws_val, qb + (uint64_t)u * 32, spol);
        } else {
          cc[u] = make_uint4(kWsZeroOff, kWsZeroOff, kWsZeroOff, kWsZeroOff);
          vc[u].zero();
        }
      }
      for (uint32_t q0 = 0; q0 < nq; q0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {  // next step's stream, in flight during this one
          const uint32_t q = q0 + U + u;
          if (q < nq) {
            cn[u] = ws_ld16(reinterpret_cast<const uint4*>(enc) + qb + (uint64_t)q * 32, spol);
            vn[u].load(T.ws_val, qb + (uint64_t)q * 32, spol);
          } else {
            cn[u] = make_uint4(kWsZeroOff, kWsZeroOff, kWsZeroOff, kWsZeroOff);
            vn[u].zero();
          }
        }
        R xr[4 * U];
        Raw xf[4 * U];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t c = quad_at(cc[u], k);
            const bool in = (int32_t)c >= 0;
            xr[4 * u + k] = in ? *reinterpret_cast<const R*>(smem + c) : R{};
            xf[4 * u + k] = !in ? g.load(c & 0x7fffffffu) : Raw{};
          }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const bool in = (int32_t)quad_at(cc[u], k) >= 0;
            const T_<C> xv = in ? RT::get(g, xr[4 * u + k]) : RT::get(g, RT::put(g, xf[4 * u + k]));
            acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(vc[u].at(k)), xv));
          }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          cc[u] = cn[u];
          vc[u] = vn[u];
        }
      }
      if (row != kWsPad) yb[(uint32_t)((int64_t)row - B)] = acc;
    }
    __syncthreads();  // every row sum of the window is in yb; the band's bottom block is free
    if (tid == 0) claim[it & 1u] = 0u;  // reused two windows on, after the next barrier
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int64_t i = pb + (int64_t)q * kWsThreads + tid;
      if (i < n) ring[i & (RN - 1)] = RT::put(g, pf[q]);
    }
    int64_t rend = B + (int64_t)kw * kWsSort;
    if (rend > n) rend = n;
    for (int64_t i = B + tid; i < rend; i += kWsThreads) {
      e.prefetch((uint32_t)i);
      e.row((uint32_t)i, yb[(uint32_t)(i - B)]);
    }
    if constexpr (!YDBL) __syncthreads();  // the one row-sum buffer is free again
  }
  pdl_trigger();
}

}  // namespace f3rg
