// wsell_pk.cuh -- the windowed SELL pass over the PACKED stream (wsell_pk_layout.hpp):
// fp16 matrix, 2-byte ring elements (plain Richardson on materialised z1, the L3
// spmv_dots, the fp16 SpMV). Same engine as wsell.cuh -- one 1024-thread CTA per SM,
// the band of x in a shared-memory ring slid window by window, sorted 32-row slices
// claimed longest-first, row sums parked in shared memory for a coalesced epilogue --
// with 4 bytes per slot instead of 6: one 32-bit word holds the slot's 16-bit code and
// its fp16 value, and a far entry is an escape pair of two slots of its own row
// ([kPkEsc + column >> 16, +0], [column & 0xffff, value]), so there is no side list,
// no second stream and no dependent load. Each row is still summed by one thread in
// stored column order at C = promote(f16, TX); the padding and escape slots add +-0
// to an accumulator that is never -0, so the results are bit-identical to wsell.cuh,
// to the row tiles and to the reference (src/csr.cpp:23-37).
//
// Kernel windows lie on a global grid of kPkTW rows; a CTA owns whole sort windows and
// may start and end inside a window. Ring invariant for the window at rows
// [B, B + TW): the ring (kPkRing slots, slot = row mod kPkRing, the last one reserved
// for zero) holds x[B - W, B + 2 TW + W).
#pragma once

#include "wsell.cuh"

namespace f3rg {

constexpr int kPkRingBytes = kPkRing * 2;
constexpr int kPkSmem = kPkRingBytes + kWsYBytes + 64;
static_assert(kPkSmem <= kWsSmem, "the packed pass runs inside the windowed engine's shared memory");

template <int C, class G, class Epi>
__device__ __forceinline__ void wsell_pass_pk(const CsrDev& A, const TilesDev& T, G& g, Epi& e, uint8_t* smem) {
  using RT = WsRing<G>;
  using R = typename RT::R;
  using Raw = typename G::Raw;
  static_assert(sizeof(R) == 2, "the packed stream is cut for 2-byte ring elements");
  constexpr int CS = (int)sizeof(T_<C>);
  constexpr int TW = kPkTW, W = kPkW;
  constexpr uint32_t RN = kPkRing;
  constexpr int KW = TW / kWsSort;
  constexpr int PF = TW / kWsThreads;
  constexpr int U = F3RG_WS_U;
  constexpr bool YDBL = 2 * TW * CS <= kWsYBytes;
  static_assert(TW % kWsSort == 0 && PF >= 1 && TW * CS <= kWsYBytes, "window geometry");

  R* ring = reinterpret_cast<R*>(smem);
  T_<C>* ybuf = reinterpret_cast<T_<C>*>(smem + kPkRingBytes);
  unsigned* claim = reinterpret_cast<unsigned*>(smem + kPkRingBytes + kWsYBytes);
  WsPolicy<G>::set(g, l2_policy(T.l2hint ? 2 : 0));    // ring fills and far gathers: keep x in L2
  const uint64_t spol = l2_policy(T.l2hint ? 1 : 0);  // the matrix stream
  const int64_t n = (int64_t)A.n;
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  const uint32_t sw0 = T.pk_cwin[blockIdx.x], sw1 = T.pk_cwin[blockIdx.x + 1];
  const uint4* __restrict__ words = reinterpret_cast<const uint4*>(T.pk_words);
  const int64_t row0 = (int64_t)sw0 * kWsSort;                                             // this CTA's rows
  const int64_t row1 = (int64_t)sw1 * kWsSort < n ? (int64_t)sw1 * kWsSort : n;

  __syncthreads();  // a previous pass in the same kernel is done with the shared memory
  if (tid < 2) claim[tid] = 0u;
  if (tid == 0) reinterpret_cast<uint16_t*>(ring)[kPkPad] = 0;  // the zero slot
  const int64_t Bfirst = row0 / TW * TW;
  if (sw0 < sw1) {  // ring for the first window: x[B - W, B + 2TW + W)
    int64_t i0 = Bfirst - W;
    if (i0 < 0) i0 = 0;
    int64_t i1 = Bfirst + 2 * TW + W;
    if (i1 > n) i1 = n;
    for (int64_t i = i0 + tid; i < i1; i += kWsThreads) {
      const uint32_t s = (uint32_t)i % RN;
      if (s < kPkLimit) ring[s] = RT::put(g, g.load((uint32_t)i));
    }
  }
  __syncthreads();

  uint32_t it = 0;
  for (int64_t B = Bfirst; sw0 < sw1 && B < row1; B += TW, ++it) {
    // the CTA's sort windows inside this kernel window
    const uint32_t swa = (uint32_t)(B / kWsSort) > sw0 ? (uint32_t)(B / kWsSort) : sw0;
    const uint32_t swb = (uint32_t)((B + TW) / kWsSort) < sw1 ? (uint32_t)((B + TW) / kWsSort) : sw1;
    const uint32_t kw = swb - swa;
    (void)KW;
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
      const uint32_t s = (swa + j % kw) * (uint32_t)kWsSlices + j / kw;
      const uint32_t e0 = __ldg(T.pk_soff + s), e1 = __ldg(T.pk_soff + s + 1);
      const uint32_t row = __ldg(T.pk_row + (size_t)s * 32 + lane);
      const uint32_t nq = (e1 - e0) >> 7;  // chunks: 32 lanes x 4 slots
      const uint64_t qb = (uint64_t)(e0 >> 2) + lane;  // this lane's quad of chunk 0
      T_<C> acc = Ar<C>::zero();
      constexpr uint32_t PADW = kPkPad;  // [pad slot, +0]
      uint4 cc[U], cn[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        cc[u] = (uint32_t)u < nq ? ws_ld16(words + qb + (uint64_t)u * 32, spol) : make_uint4(PADW, PADW, PADW, PADW);
      for (uint32_t q0 = 0; q0 < nq; q0 += U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {  // next step's stream, in flight during this one
          const uint32_t q = q0 + U + u;
          cn[u] = q < nq ? ws_ld16(words + qb + (uint64_t)q * 32, spol) : make_uint4(PADW, PADW, PADW, PADW);
        }
        R xr[4 * U];
        Raw xf[4 * U];
        bool farf[4 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          bool low = false;     // this slot is the low half of a far column
          uint32_t hi = 0;      // (escape code - kPkEsc) << 16 of the slot before
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t w = quad_at(cc[u], k);
            const uint32_t code = w & 0xffffu;
            const uint32_t idx = code < (uint32_t)kPkPad ? code : (uint32_t)kPkPad;  // escape and low-half slots read zero
            farf[4 * u + k] = low;
            xr[4 * u + k] = ring[idx];
            xf[4 * u + k] = low ? g.load(hi | code) : Raw{};
            const bool esc = !low && code >= (uint32_t)kPkEsc;
            hi = (code - (uint32_t)kPkEsc) << 16;
            low = esc;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const __half a = __ushort_as_half((unsigned short)(quad_at(cc[u], k) >> 16));
            const T_<C> xv = !farf[4 * u + k] ? RT::get(g, xr[4 * u + k]) : RT::get(g, RT::put(g, xf[4 * u + k]));
            acc = Ar<C>::add(acc, Ar<C>::mul(cvt<C>(a), xv));
          }
#pragma unroll
        for (int u = 0; u < U; ++u) cc[u] = cn[u];
      }
      if (row != kWsPad) yb[(uint32_t)((int64_t)row - B)] = acc;
    }
    __syncthreads();  // every row sum of the window is in yb; the band's bottom block is free
    if (tid == 0) claim[it & 1u] = 0u;  // reused two windows on, after the next barrier
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int64_t i = pb + (int64_t)q * kWsThreads + tid;
      const uint32_t s = (uint32_t)i % RN;
      if (i < n && s < kPkLimit) ring[s] = RT::put(g, pf[q]);
    }
    const int64_t ra = B > row0 ? B : row0, rb = B + TW < row1 ? B + TW : row1;
    for (int64_t i = ra + tid; i < rb; i += kWsThreads) {
      e.prefetch((uint32_t)i);
      e.row((uint32_t)i, yb[(uint32_t)(i - B)]);
    }
    if constexpr (!YDBL) __syncthreads();  // the one row-sum buffer is free again
  }
  pdl_trigger();
}

}  // namespace f3rg
